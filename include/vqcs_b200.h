/*
 * vqcs_b200.h — C-ABI of the B200-native state-vector / density-matrix core.
 *
 * This is the drop-in boundary for the data-parallel path of the C++
 * reference `vqcs` (/root/reference/proj/include/vqcs). The reference has no
 * FFI: its "operator API" is a header-only C++ template API. Every entry point
 * below replaces one function of that API (cited per function) with plain C
 * types, so a maintainer can bind it from the reference's C++ (see
 * include/vqcs_b200.hpp and INTEGRATION.md) or from ctypes.
 *
 * Conventions (identical to the reference):
 *   - complex128 amplitudes, interleaved (re, im) doubles;
 *   - qubit j (1-based) <-> bit j-1 of the flat amplitude index
 *     (state.hpp:17-22);
 *   - a density matrix of n qubits is stored as 4^n entries,
 *     entry(row, col) at row + col * 2^n, i.e. a 2n-qubit pseudo state with
 *     ket qubits 1..n and bra qubits n+1..2n (state.hpp:259-327);
 *   - gate matrices are column-major 2^m x 2^m, first listed position = local
 *     LSB (gates.hpp:18-22).
 *
 * Error handling: every function returns a vqb_status. Nonzero codes 1..11
 * map 1:1 onto the reference exception classes (errors.hpp:23-96); CUDA and
 * NCCL failures get their own codes. vqb_last_error() returns a thread-local
 * message for the last failure on the calling thread.
 *
 * Calls are synchronous at the API (the reference's calls are synchronous,
 * threading.hpp:54-70): a function returns after its device work completed.
 * One CUDA stream per state handle; callers need exclusive access to a state
 * during a call.
 */
#ifndef VQCS_B200_H
#define VQCS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VQB_API __attribute__((visibility("default")))
#else
#define VQB_API
#endif

/* ---- status codes: errors.hpp:23-96, in declaration order ---- */
typedef enum vqb_status {
    VQB_OK = 0,
    VQB_ERR_SIZE = 1,           /* SizeError            errors.hpp:29 */
    VQB_ERR_SHAPE = 2,          /* ShapeError           errors.hpp:35 */
    VQB_ERR_VALIDITY = 3,       /* ValidityError        errors.hpp:42 */
    VQB_ERR_DOMAIN = 4,         /* DomainError          errors.hpp:48 */
    VQB_ERR_INDEX = 5,          /* IndexError           errors.hpp:54 */
    VQB_ERR_TYPE = 6,           /* TypeError            errors.hpp:61 */
    VQB_ERR_UNSUPPORTED = 7,    /* UnsupportedError     errors.hpp:68 */
    VQB_ERR_DEGENERATE = 8,     /* DegenerateStateError errors.hpp:75 */
    VQB_ERR_NONINVERTIBLE = 9,  /* NonInvertibleChannelError errors.hpp:81 */
    VQB_ERR_IO = 10,            /* IoError              errors.hpp:87 */
    VQB_ERR_USAGE = 11,         /* UsageError           errors.hpp:93 */
    VQB_ERR_CUDA = 20,          /* CUDA runtime failure (no reference analogue) */
    VQB_ERR_NCCL = 21,          /* NCCL failure (no reference analogue) */
    VQB_ERR_INTERNAL = 22
} vqb_status;

/* ---- GateKind, same numbering as gates.hpp:38-61 ---- */
typedef enum vqb_gate_kind {
    VQB_GATE_GENERIC = 0,
    VQB_GATE_X, VQB_GATE_Y, VQB_GATE_Z, VQB_GATE_H, VQB_GATE_S, VQB_GATE_T,
    VQB_GATE_SQRTX, VQB_GATE_SQRTY, VQB_GATE_SWAP, VQB_GATE_ISWAP, VQB_GATE_CZ,
    VQB_GATE_CNOT, VQB_GATE_TOFFOLI, VQB_GATE_FREDKIN, VQB_GATE_RX, VQB_GATE_RY,
    VQB_GATE_RZ, VQB_GATE_CRX, VQB_GATE_CRY, VQB_GATE_CRZ, VQB_GATE_FSIM
} vqb_gate_kind;

/* ---- ChannelKind, same numbering as gates.hpp:63-68 ---- */
typedef enum vqb_channel_kind {
    VQB_CHANNEL_GENERIC = 0,
    VQB_CHANNEL_AMPLITUDE_DAMPING = 1,
    VQB_CHANNEL_PHASE_DAMPING = 2,
    VQB_CHANNEL_DEPOLARIZING = 3
} vqb_channel_kind;

enum { VQB_ELEM_GATE = 0, VQB_ELEM_CHANNEL = 1 };
enum { VQB_MAX_POSITIONS = 6, VQB_MAX_PARAMS = 5 };

typedef struct vqb_c128 {
    double re;
    double im;
} vqb_c128;

/*
 * One circuit element: a GateOp (gates.hpp:106-130) or a ChannelOp
 * (gates.hpp:133-141). Nested circuits (circuit.hpp:40) are passed flattened
 * in depth-first order, which is the reference's traversal order
 * (circuit.hpp:69-102).
 */
typedef struct vqb_op {
    int32_t elem;                        /* VQB_ELEM_GATE | VQB_ELEM_CHANNEL */
    int32_t kind;                        /* vqb_gate_kind | vqb_channel_kind */
    int32_t num_positions;               /* m >= 1 */
    int32_t positions[VQB_MAX_POSITIONS];/* 1-based; first = local LSB */
    int32_t num_params;                  /* 0, 1 (rotations) or 5 (FSIM) */
    double params[VQB_MAX_PARAMS];
    int32_t is_param[VQB_MAX_PARAMS];    /* nonzero = variational */
    /* Gate: column-major 2^m x 2^m matrix, or NULL to build it from kind and
     * params exactly as standard_gate/parametric_gate do (gates.hpp:439-533). */
    const vqb_c128 *matrix;
    /* Channel: num_kraus column-major 2^m x 2^m Kraus operators back to back,
     * or NULL for a named channel built from params[0] as standard_channel
     * does (gates.hpp:657-704). */
    int32_t num_kraus;
    const vqb_c128 *kraus;
} vqb_op;

/* One Pauli string (observables.hpp:38-65): product of (qubit, label) factors
 * with distinct 1-based qubits and labels 'x'|'y'|'z' (either case); an empty
 * factor list is the identity term. */
typedef struct vqb_pauli_term {
    vqb_c128 coeff;
    int32_t num_factors;
    const int32_t *qubits;
    const char *labels;
} vqb_pauli_term;

/* Opaque device-resident state (PureState<double> state.hpp:175-256 or
 * MixedState<double> state.hpp:259-349). */
typedef struct vqb_state vqb_state;

/* ---- errors / build info ---- */
VQB_API const char *vqb_last_error(void);
VQB_API const char *vqb_build_info(void);
/* Number of native kernel launches issued by this process so far (evidence
 * counter for benchmarks; incremented on every launch of our kernels). */
VQB_API int64_t vqb_kernel_launch_count(void);
/* Per-launch CUDA-event timing window for benchmarks (no reference analogue;
 * the reference only wall-clocks whole calls, src/bench.cpp:76-87).
 * vqb_profile_end synchronises the device and writes one line per kernel
 * name: "<name> <launches> <total_ms>\n" (truncated to `cap` bytes). */
/* FP64 flops issued by the fused executors so far: the specialised kernels
 * count the FMAs they execute (exact zeros and real/imaginary-only matrix
 * entries are skipped); the interpreter counts a dense complex 2^m x 2^m block
 * as 8 * 2^m flops per amplitude. The FP64 roofline numerator for benchmarks. */
VQB_API double vqb_flop_count(void);
/* Development aid (host only, no device work): the source of the specialised
 * stage kernel for a lowered stage program dumped with VQB_JIT_DUMP=<dir>
 * (`regs` = 16 or 8 amplitudes per thread, `rev` != 0 for adjoint programs).
 * Writes the NUL-terminated source to `out` and the executed FP64 flops per
 * amplitude to `*flops_per_amp`. */
VQB_API int vqb_debug_jit_source(int32_t regs, const void *params, size_t nbytes, int32_t rev, char *out,
                                 size_t cap, double *flops_per_amp);
VQB_API int vqb_profile_begin(void);
VQB_API int vqb_profile_end(char *buf, int64_t cap);

/* ---- allocation bookkeeping: state.hpp:56-83,154-161 ---- */
/* state_alloc_stats(): live and peak counts of full amplitude buffers (every
 * state created by this library, including working states a loss/gradient
 * keeps cached for the next call), plus live/peak device bytes of everything
 * the library allocated (scratch included). Null outputs are skipped. */
VQB_API int vqb_alloc_stats(int64_t *live_states, int64_t *peak_states, uint64_t *live_bytes,
                            uint64_t *peak_bytes);
/* reset_state_alloc_peak(): peak counters <- live counters. */
VQB_API int vqb_reset_alloc_peak(void);
/* Frees every cache the library keeps across calls (working states of
 * losses/gradients, the batch API's rotating states, executor scratch) on
 * every device. No reference analogue (the reference frees its working
 * copies at the end of each call, autodiff.hpp:111-124). Must not run
 * concurrently with any other call. */
VQB_API int vqb_release_caches(void);

/* ---- device state: replaces PureState / MixedState storage ---- */
/* PureState(n) (state.hpp:182-185) when mixed == 0, MixedState(n)
 * (state.hpp:264-268) when mixed != 0; initialised to |0...0> (<0...0|). */
VQB_API int vqb_state_create(int32_t num_qubits, int32_t mixed, vqb_state **out);
/* Non-owning handle over caller-owned device memory holding 2^num_qubits
 * amplitudes (mixed: 4^num_qubits). `global_offset` is the flat index of the
 * buffer's first amplitude inside a larger, sharded state (0 when
 * unsharded): vqb_state_set_zero puts the |0...0> amplitude only into the
 * buffer at offset 0. Operations act on the buffer's own qubits; callers
 * restrict operations on global qubits first (as vqb_sharded_* and
 * paper_2406_19212_b200/distributed.py do). */
VQB_API int vqb_state_wrap(void *device_ptr, int32_t num_qubits, int32_t mixed,
                           uint64_t global_offset, int32_t global_qubits,
                           vqb_state **out);
VQB_API int vqb_state_destroy(vqb_state *st);
VQB_API int vqb_state_info(const vqb_state *st, int32_t *num_qubits, int32_t *mixed,
                           uint64_t *num_amplitudes);
VQB_API int vqb_state_device_ptr(const vqb_state *st, void **ptr);
/* The cudaStream_t all work on this state is issued to (for event timing). */
VQB_API int vqb_state_stream(const vqb_state *st, void **stream);
VQB_API int vqb_state_set_zero(vqb_state *st); /* back to |0...0> */
/* Host <-> device. `count` must equal the number of amplitudes. The host
 * buffer may be pageable or pinned. */
VQB_API int vqb_state_upload(vqb_state *st, const vqb_c128 *host, uint64_t count);
VQB_API int vqb_state_download(const vqb_state *st, vqb_c128 *host, uint64_t count);
/* Upload without waiting: `host` must be page-locked and stay unchanged until
 * the next call on this state that returns a result to the host (every such
 * call synchronises the state's stream, on which the copy is ordered). Lets
 * the host-side planning of the following call overlap the transfer.
 * VQB_ERR_USAGE for pageable memory. No reference counterpart (the
 * reference's states live in host memory, state.hpp:175-256). */
VQB_API int vqb_state_upload_async(vqb_state *st, const vqb_c128 *host, uint64_t count);
VQB_API int vqb_state_copy(vqb_state *dst, const vqb_state *src);
/* Amplitudes [offset, offset + count) in canonical order (the host-side view
 * of a slice of state.hpp's amplitude vector, state.hpp:222-226) — for states
 * too large to download whole (config 4: 128 GiB). INDEX if the range does not
 * fit the state. */
VQB_API int vqb_state_download_range(const vqb_state *st, uint64_t offset, uint64_t count,
                                     vqb_c128 *host);

/* ---- gate / channel application: kernels.hpp, circuit.hpp ---- */
/* apply_gate_fast (kernels.hpp:365-430) on a pure state; apply_gate_mixed
 * (kernels.hpp:434-449) on a mixed state. */
VQB_API int vqb_apply_gate(vqb_state *st, const vqb_op *gate);
/* apply_channel (kernels.hpp:453-461); mixed states only. */
VQB_API int vqb_apply_channel(vqb_state *st, const vqb_op *channel);
/* apply_matrix (kernels.hpp:327-361): arbitrary (not necessarily unitary)
 * m-qubit matrix on the given positions of the (pseudo) state. */
VQB_API int vqb_apply_matrix(vqb_state *st, const int32_t *positions, int32_t m,
                             const vqb_c128 *matrix);
/* apply_circuit (circuit.hpp:110-129) over a flattened element list. Gates
 * are scheduled into fused shared-memory tile passes; results match the
 * reference within 1e-12 max-abs. */
VQB_API int vqb_apply_circuit(vqb_state *st, const vqb_op *ops, int64_t count);
/* apply_circuit_copy (circuit.hpp:132-146) over `batch` host-resident input
 * states of 2^num_qubits amplitudes (mixed: 4^num_qubits entries, the
 * MixedState layout): outputs[j] <- circuit(inputs[j]). Uploads, circuits and
 * downloads of consecutive jobs overlap (three rotating device states on their
 * own streams); use pinned host buffers for the overlap. Synchronous: returns
 * when every output has been written. Same results as vqb_apply_circuit. */
VQB_API int vqb_apply_circuit_copy_batch(int32_t num_qubits, int32_t mixed, const vqb_op *ops, int64_t count,
                                         const vqb_c128 *const *inputs, vqb_c128 *const *outputs,
                                         int64_t batch);
/* Same, gate by gate (one kernel per element, the unfused path). */
VQB_API int vqb_apply_circuit_unfused(vqb_state *st, const vqb_op *ops, int64_t count);

/* ---- reductions: state.hpp, observables.hpp ---- */
VQB_API int vqb_norm(const vqb_state *st, double *out);       /* state.hpp:236-242 */
VQB_API int vqb_trace(const vqb_state *st, vqb_c128 *out);    /* state.hpp:329-336 */
/* expectation (observables.hpp:176-213), pure or mixed. */
VQB_API int vqb_expectation(const vqb_state *st, const vqb_pauli_term *terms,
                            int64_t num_terms, vqb_c128 *out);
/* apply_operator (observables.hpp:216-237): dst <- H src. dst must have the
 * same shape as src. */
VQB_API int vqb_apply_operator(const vqb_state *src, vqb_state *dst,
                               const vqb_pauli_term *terms, int64_t num_terms);
/* bilinear_gate_form (kernels.hpp:466-503): <bra| L |ket>. */
VQB_API int vqb_bilinear_form(const vqb_state *bra, const vqb_state *ket,
                              const int32_t *positions, int32_t m,
                              const vqb_c128 *local, vqb_c128 *out);
/* reverse_sweep_step (kernels.hpp:659-697): phi <- inv phi;
 * out[p] = <psi| dmats[p] |phi>; psi <- inv psi. dmats holds np matrices
 * back to back. */
VQB_API int vqb_reverse_step(vqb_state *phi, vqb_state *psi, const int32_t *positions,
                             int32_t m, const vqb_c128 *inv, const vqb_c128 *dmats,
                             int32_t np, vqb_c128 *out);

/* A batch of reverse steps (the reverse loop of autodiff.hpp:130-150 with
 * explicit matrices): each step is reverse_sweep_step (kernels.hpp:659-697). */
typedef struct vqb_rev_step {
    int32_t num_positions;                /* m, 1..4 (pseudo-state positions) */
    int32_t positions[VQB_MAX_POSITIONS]; /* 1-based; first = local LSB */
    const vqb_c128 *inv;                  /* 2^m x 2^m column-major, applied to phi and psi */
    int32_t num_dmats;                    /* 0..VQB_MAX_PARAMS */
    const vqb_c128 *dmats;                /* num_dmats matrices back to back */
    int64_t grad_index;                   /* first gradient slot of this step */
} vqb_rev_step;
/* Runs steps[0..count) in order through the fused adjoint executor: phi <-
 * inv phi; grads[grad_index + p] += scale * Re <psi| D_p |phi>; psi <- inv psi.
 * Used by sharded gradients (each rank sweeps its shard between global<->local
 * swaps, with controls on global qubits restricted on the host; the per-rank
 * gradients are summed by one all-reduce). */
VQB_API int vqb_reverse_sweep(vqb_state *phi, vqb_state *psi, const vqb_rev_step *steps,
                              int64_t count, double scale, double *grads, int64_t grads_len);

/* ---- losses and gradients: autodiff.hpp ---- */
/* loss_pure (autodiff.hpp:80-89). s0 is not mutated. */
VQB_API int vqb_loss_pure(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                          int64_t num_terms, const vqb_state *s0, double *loss);
/* gradient_pure (autodiff.hpp:95-156): Algorithm 2 with two working states.
 * grads receives one value per active parameter in traversal order;
 * *num_grads is set to that count (an error if it exceeds capacity).
 * reverse_residual (nullable) = max |phi_end - s0| (autodiff.hpp:151-154). */
VQB_API int vqb_gradient_pure(const vqb_op *ops, int64_t count,
                              const vqb_pauli_term *terms, int64_t num_terms,
                              const vqb_state *s0, double *loss, double *grads,
                              int64_t capacity, int64_t *num_grads,
                              double *reverse_residual);
/* loss_mixed (autodiff.hpp:160-167). */
VQB_API int vqb_loss_mixed(const vqb_op *ops, int64_t count, const vqb_pauli_term *terms,
                           int64_t num_terms, const vqb_state *dm0, double *loss);
/* gradient_mixed (autodiff.hpp:184-329): noisy reverse sweep on vec(rho);
 * channels are inverted on the host (LU, condition limit 1e12,
 * autodiff.hpp:51,263-276) and a non-invertible one returns
 * VQB_ERR_NONINVERTIBLE. */
VQB_API int vqb_gradient_mixed(const vqb_op *ops, int64_t count,
                               const vqb_pauli_term *terms, int64_t num_terms,
                               const vqb_state *dm0, double *loss, double *grads,
                               int64_t capacity, int64_t *num_grads,
                               double *reverse_residual);

/* ---- measurement: circuit.hpp:303-375 ---- */
/* measure(state, qubit, rng) (circuit.hpp:303-337 pure, :339-375 mixed):
 * p1 = sum over basis states with bit (qubit-1) set of |a_k|^2 (pure) or
 * rho_kk (mixed), clamped to [0,1]; p0 = clamp(1 - p1); outcome =
 * (uniform < p1); the state collapses in place (scale 1/sqrt(p) pure, 1/p
 * mixed) and *probability = p of the drawn outcome. `uniform` is the value
 * the reference draws from its stream (detail::uniform_unit, circuit.hpp:288:
 * (rng() >> 11) * 2^-53); the C++ facade draws it from the caller's
 * std::mt19937_64, so outcomes follow the same stream. Errors: INDEX (bad
 * qubit), DEGENERATE (both probabilities vanish / drawn outcome has p = 0). */
VQB_API int vqb_measure(vqb_state *st, int32_t qubit, double uniform, int32_t *outcome,
                        double *probability);
/* The two halves of vqb_measure, for sharded states (per-rank partial p1,
 * all-reduced by the caller): the unclamped local p1, and the collapse of
 * qubit to `outcome` with scale 1/sqrt(p) (pure) or 1/p (mixed). */
VQB_API int vqb_measure_probability(const vqb_state *st, int32_t qubit, double *p1);
VQB_API int vqb_collapse(vqb_state *st, int32_t qubit, int32_t outcome, double probability);

/* ---- multi-device sharded pure state (no reference analogue; SURVEY.md
 * §8(e)). The reference is single-address-space (state.hpp:175-256), so its
 * unsharded result is the oracle. ----
 * One process drives P = 2^g devices: shard r (on devices[r]) holds the 2^(n-g)
 * amplitudes whose top g physical bits equal r. Operations on local qubits
 * run on every shard through the fused executor; controls and diagonal phases
 * on global qubits are resolved per shard on the host (no data movement); a
 * mixing operation on a global qubit first swaps global and local qubits in
 * one all-to-all round of in-place peer-to-peer kernels (NVLink loads and
 * stores into the peer shard, no staging buffer). A logical->physical qubit
 * map is kept; download/upload use the canonical order (bit-exact).
 * `devices` may repeat an ordinal (several shards on one device, e.g. to
 * test the exchange logic on one GPU); distinct devices need peer access
 * (UNSUPPORTED otherwise). At least 12 local qubits per shard. */
typedef struct vqb_sharded vqb_sharded;
VQB_API int vqb_sharded_create(int32_t num_qubits, int32_t num_devices, const int32_t *devices,
                               vqb_sharded **out);
VQB_API int vqb_sharded_destroy(vqb_sharded *st);
VQB_API int vqb_sharded_set_zero(vqb_sharded *st);
/* apply_circuit (circuit.hpp:110-129) on the sharded state; pure gates only
 * (TYPE for channels, as for a PureState). */
VQB_API int vqb_sharded_apply_circuit(vqb_sharded *st, const vqb_op *ops, int64_t count);
VQB_API int vqb_sharded_norm(vqb_sharded *st, double *out);
/* expectation (observables.hpp:176-190). A term whose X/Y factors flip
 * global qubits pairs shard r with shard r ^ x_global: its partials read the
 * partner shard directly (peer memory), so no exchange round is needed. */
VQB_API int vqb_sharded_expectation(vqb_sharded *st, const vqb_pauli_term *terms, int64_t num_terms,
                                    vqb_c128 *out);
/* Whole state in canonical order (count = 2^num_qubits). */
VQB_API int vqb_sharded_download(vqb_sharded *st, vqb_c128 *host, uint64_t count);
VQB_API int vqb_sharded_upload(vqb_sharded *st, const vqb_c128 *host, uint64_t count);
/* Exchange counters: all-to-all rounds, global<->local bit exchanges, bytes
 * moved over the links (both directions); the physical bit of each logical
 * qubit (num_qubits entries, 0-based). Null outputs are skipped. */
VQB_API int vqb_sharded_stats(const vqb_sharded *st, int64_t *rounds, int64_t *swapped_bits,
                              uint64_t *bytes_moved, int32_t *log2phys);
/* save_state / load_state (io.hpp:56-128) of the whole sharded state: the
 * layout is made canonical first (exchange rounds + local SWAPs), then the
 * shards are streamed to the file back to back through a pinned chunk, so the
 * dump is byte-identical to an unsharded save of the same state. Load: the
 * file's qubit count must equal the state's (SHAPE otherwise); IO errors as
 * vqb_state_load. */
VQB_API int vqb_sharded_save(vqb_sharded *st, const char *path);
/* gradient_pure (autodiff.hpp:95-156) with the sharded state as s0: the
 * forward pass runs in place, the costate H|Phi> lives in a second set of
 * shards that follows every exchange round, the reverse sweep runs per shard
 * through the fused adjoint executor and the per-shard gradient vectors are
 * summed in shard order. On return the state holds the reverse-swept Phi,
 * i.e. s0 up to rounding (the reference keeps s0 const and works on copies,
 * autodiff.hpp:111-124; a third full-size state per device would not fit at
 * the sizes sharding is for). Outputs as vqb_gradient_pure. */
VQB_API int vqb_sharded_gradient_pure(vqb_sharded *st, const vqb_op *ops, int64_t count,
                                      const vqb_pauli_term *terms, int64_t num_terms, double *loss,
                                      double *grads, int64_t capacity, int64_t *num_grads);
VQB_API int vqb_sharded_load(vqb_sharded *st, const char *path, int32_t *precision);

/* ---- state dump I/O: io.hpp:40-128 ---- */
/* save_state (io.hpp:56-82): "VQCS" | u32 version 1 | u32 n | u8 precision
 * (2 = complex double) | 2^n little-endian (re, im) doubles. Pure states only
 * (TYPE for a density matrix); the state is streamed from the device in
 * chunks through a pinned buffer. IO on open/write failure. */
VQB_API int vqb_state_save(const vqb_state *st, const char *path);
/* load_state (io.hpp:84-128) into a new device pure state; *precision
 * (nullable) receives the file's precision tag (1 or 2). IO errors exactly as
 * the reference: bad magic, unsupported version, qubit count out of range,
 * unknown precision tag, truncated payload. */
VQB_API int vqb_state_load(const char *path, vqb_state **out, int32_t *precision);

/* ---- benchmark records: BenchRecord (bench.hpp:60-72) and emit_report
 * (src/bench.cpp:296-310,329-369) ---- */
typedef struct vqb_bench_record {
    const char *task;              /* e.g. "rqc", "rqc-grad", "noisy-grad" */
    int32_t num_qubits, depth, threads;
    const double *seconds;         /* one entry per repetition (warm-up excluded) */
    int64_t num_seconds;
    double speedup;                /* 0: not a thread sweep (field omitted) */
    int64_t num_info;              /* params: key/value strings */
    const char *const *info_keys;
    const char *const *info_values;
} vqb_bench_record;
/* emit_report: format 0 = JSON array (stable field order, mean and population
 * standard deviation computed as finish_stats does), 1 = CSV
 * (task,n,depth,threads,rep,seconds). Writes at most `cap` bytes (NUL
 * included) to `out` (nullable) and the full length to *length. Output is
 * byte-identical to the reference harness's. USAGE for an empty record list. */
VQB_API int vqb_bench_report(const vqb_bench_record *records, int64_t count, int32_t format, char *out,
                             int64_t cap, int64_t *length);

/* ---- circuit fusion: circuit.hpp:199-276 ---- */
/* fuse_gates: absorbs single-qubit gates into the next (else the previous)
 * two-qubit gate acting on the same qubit; every surviving gate becomes a
 * non-parametric generic gate. UNSUPPORTED for circuits with channels.
 * Two-phase: with cap == 0 only *num_out and *num_entries (total matrix
 * entries) are set; otherwise out_ops[0..*num_out) are written with
 * out_ops[i].matrix pointing into out_matrices (matrices back to back). */
VQB_API int vqb_fuse_gates(const vqb_op *ops, int64_t count, int64_t cap, vqb_op *out_ops,
                           int64_t matrix_cap, vqb_c128 *out_matrices, int64_t *num_out,
                           int64_t *num_entries);

/* ---- host-only planning (no device work; no reference analogue) ---- */
/* Plans the fused execution of a circuit exactly as vqb_apply_circuit does
 * (stage packing into 2^tile_bits tiles, then block fusion on at most
 * max_support qubits) and exports the result as dense blocks in execution
 * order: block b acts on num_positions[b] 1-based positions
 * positions[6*b ...] of the (pseudo) state with the column-major matrix
 * matrices[stride*b ...] (stride = 256, so blocks of at most 4 positions).
 * mixed != 0 plans the density-matrix program of an n-qubit MixedState.
 * With cap == 0 only *num_blocks and *num_stages are computed. */
VQB_API int vqb_plan_blocks(const vqb_op *ops, int64_t count, int32_t num_qubits, int32_t mixed,
                            int32_t tile_bits, int32_t max_support, int64_t cap,
                            int64_t *num_blocks, int64_t *num_stages, int32_t *num_positions,
                            int32_t *positions, vqb_c128 *matrices);

/* ---- host-side gate algebra (gates.hpp), exported for bindings ---- */
/* Matrix of a gate descriptor: the caller's matrix if given, else built from
 * kind/params (gates.hpp:188-259,309-373). out: 4^m entries. */
VQB_API int vqb_gate_matrix(const vqb_op *gate, vqb_c128 *out);
/* gate_derivative (gates.hpp:543-577). */
VQB_API int vqb_gate_derivative(const vqb_op *gate, int32_t param_index, vqb_c128 *out);
/* gate_inverse (gates.hpp:581-619): matrix of the inverse gate. */
VQB_API int vqb_gate_inverse(const vqb_op *gate, vqb_c128 *out);
/* channel_superoperator (gates.hpp:708-732). out: 16^m entries. */
VQB_API int vqb_channel_superop(const vqb_op *channel, vqb_c128 *out);
/* Inverse of the channel's superoperator as gradient_mixed uses it
 * (autodiff.hpp:263-276): closed form for the named 1-qubit channels
 * (gates.hpp:657-704), elimination with partial pivoting for Generic ones
 * (linalg.hpp:140-200). *condition = ||S||_1 ||S^-1||_1; *singular != 0 when
 * a pivot vanishes (out untouched then). Host only. */
VQB_API int vqb_channel_inverse(const vqb_op *channel, vqb_c128 *out, double *condition,
                                int32_t *singular);

#ifdef __cplusplus
}
#endif

#endif /* VQCS_B200_H */
