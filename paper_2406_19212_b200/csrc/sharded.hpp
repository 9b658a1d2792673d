// A pure state sharded over several devices of ONE process (
// no reference analogue: the reference is single-address-space, so its
// unsharded result is the oracle).
//
// Layout: P = 2^g shards of 2^(n-g) amplitudes; shard r holds the amplitudes
// whose top g physical bits equal r. A logical->physical qubit map starts as
// the identity and changes only through global<->local swaps. Operations run
// on every shard through the fused executor, with their conditions on global
// bits fixed to the shard's values on the host (controls and diagonal phases
// on global qubits need no data movement); a mixing bit on a global qubit
// first swaps k global bits with k free local bits in one all-to-all round:
// shard r (global value a) exchanges its amplitudes whose local bits equal b
// with shard r' (value b) amplitudes whose local bits equal a, in place, by
// kernels that read and write the peer shard directly over NVLink (peer
// access; no staging buffer at all), each pair's range split between the two
// devices. Reductions: per-shard partials summed on the host in shard order
// (deterministic).
#pragma once

#include "engine.hpp"

namespace vqb {

struct Sharded {
    int n = 0, g = 0, n_loc = 0, P = 0;
    std::vector<int> devs;
    std::vector<DeviceState *> shards;
    // extra shard sets moved by every swap (the adjoint costate Psi)
    std::vector<std::vector<DeviceState *>> followers;
    std::vector<cudaEvent_t> events;
    std::vector<int> log2phys; // logical qubit (0-based) -> physical bit
    int64_t rounds = 0, bits_swapped = 0;
    uint64_t bytes_moved = 0;  // over the links, both directions
    int lookahead = 64;
};

Sharded *sharded_create(int n, int num_devices, const int *devices);
void sharded_destroy(Sharded *s);
void sharded_set_zero(Sharded *s);
void sharded_apply_circuit(Sharded *s, const vqb_op *ops, int64_t count);
double sharded_norm(Sharded *s);
cplx sharded_expectation(Sharded *s, const vqb_pauli_term *terms, int64_t nterms);
void sharded_download(Sharded *s, vqb_c128 *host, uint64_t count); // canonical order
void sharded_upload(Sharded *s, const vqb_c128 *host, uint64_t count);
// Exchange physical global bits with local bits (pairs of (global, local)
// physical bit positions) in one all-to-all round.
void sharded_swap(Sharded *s, const std::vector<std::pair<int, int>> &pairs);
void sharded_sync(Sharded *s);
// Restore the canonical layout (logical qubit q at physical bit q): global
// positions by exchange rounds, local ones by SWAP gates (exact data moves).
void sharded_canonicalize(Sharded *s);
// save_state / load_state (io.hpp:56-128) of the whole state: canonical layout
// first, then the shards streamed back to back (the file equals an unsharded
// dump of the same state byte for byte).
void sharded_save(Sharded *s, const char *path);
void sharded_load(Sharded *s, const char *path, int *precision);
// gradient_pure (autodiff.hpp:95-156) on the sharded state, which holds s0:
// forward in place, <H>, Psi = H|Phi> in a second set of shards that follows
// every swap, the reverse sweep per shard through the fused adjoint executor
// (steps restricted to each shard's global bit values, exchange rounds when a
// step mixes a global qubit), per-shard gradient vectors summed in shard
// order. On return the state holds the reverse-swept Phi (= s0 up to the
// reverse residual, which is reported as max |Phi_end - s0| only when
// `residual` is requested -- that needs a copy of s0, one more shard set).
struct ShardedGradient {
    double loss = 0;
    std::vector<double> grads;
};
ShardedGradient sharded_gradient_pure(Sharded *s, const vqb_op *ops, int64_t count,
                                      const vqb_pauli_term *terms, int64_t nterms);

} // namespace vqb
