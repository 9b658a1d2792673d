// Stage planner for the fused tile executor.
//
// Every operation is analysed into
//   * mixing bits    — bits whose values the matrix couples (must live in the
//                      shared-memory tile), at most 4;
//   * condition bits — bits in which the matrix is block diagonal (controls,
//                      diagonal phases); they select one of 2^nc sub-matrices
//                      and are read from the amplitude's global index, so they
//                      may lie anywhere in the state.
// Consecutive operations are greedily packed into stages whose mixing bits
// fit a 2^k tile that always contains the lowest three bits (128-B runs);
// a later operation may overtake a deferred one only if their supports are
// disjoint (they commute), so the stage order reproduces the program exactly.
#pragma once
#include <deque>
#include <functional>
#include <memory>

#include "engine.hpp"

namespace vqb {

constexpr int kMaxMix = 4;
constexpr int kMaxCond = 6;
constexpr int kLowBits = 3;
constexpr int kMaxPlanOps = 96; // per stage, before block fusion (bounds shared memory)

struct FusedOp {
    int nt = 0, nc = 0, np = 0;
    int mix[kMaxMix] = {};   // global bits, local sub-matrix order
    int cnd[kMaxCond] = {};  // global bits, condition index order
    cvec sub_phi;            // 2^nc blocks of (2^nt)^2, column-major
    cvec sub_psi;            // pair ops only (phi and psi matrices differ)
    cvec sub_d;              // np * 2^nc blocks (param ops)
    bool pair = false;
    int64_t grad_base = -1;
    double scale = 1.0;
    uint64_t support = 0;    // all bits touched (commutation test)
    uint64_t mixmask = 0;
    bool fusable = true;
    Gate gate;               // original (fallback path)
    const RevOp *rev = nullptr;
    mutable double cost = -1; // op_cost cache (-1: not computed)
};

struct Stage {
    bool fused = true;       // false: a single unfusable op, run unfused
    int k = 0;
    int bits[24] = {};       // tile bits, ascending (global positions)
    std::vector<int> ops;    // indices into the op list, in execution order
};

FusedOp analyse_gate(const Gate &g);
FusedOp analyse_rev(const RevOp &r);
// seeds: starting points of the tile search per stage (0: 12 for states of
// >= 2^22 amplitudes, 6 below)
std::vector<Stage> plan_stages(const std::vector<FusedOp> &ops, int pn, int k, int max_ops = kMaxPlanOps,
                               int seeds = 0);
// one setting of the greedy packing: the lowest `low_bits` bits are in every
// tile (contiguous runs of 16 * 2^low_bits bytes) + how the tile search weighs the front of the program: an operation
// among the first `window` pending ones scores up to `gamma`/64 of a mixing
// operation extra, falling linearly with its position
struct PlanKnobs {
    int low_bits, gamma, window;
    int max_ops = kMaxPlanOps; // operations per stage (the register executor splits a stage into launches itself)
    int seeds = 0;             // extra starting points of the tile search (pending operations' mixing bits)
};
std::vector<Stage> plan_stages(const std::vector<FusedOp> &ops, int pn, int k, const PlanKnobs &knobs);

// Within one stage, multiply runs of non-parametric operations into dense
// blocks on at most `max_support` qubits (an operation is moved only past
// operations on disjoint qubits). Parametric reverse steps are kept as they
// are. Returns the stage's new operation list (re-analysed).
std::vector<FusedOp> fuse_blocks(const std::vector<FusedOp> &ops, const std::vector<int> &order,
                                 int max_support);
// The same without copying: unmerged operations are returned as pointers into
// `ops`, merged blocks are stored in `store` (stable addresses). With
// `cost_model`, a merge happens only if the merged block's emitted cost
// (op_cost, after scalar factoring) does not exceed the parts' total: the
// structure-aware specialised kernels run a sparse fSim or a factored sqrt(X)
// far cheaper than the dense product of both (the interpreter runs every
// block dense, so it merges whenever it can).
std::vector<const FusedOp *> fuse_blocks_ref(const std::vector<FusedOp> &ops, const std::vector<int> &order,
                                             int max_support, std::deque<FusedOp> &store,
                                             bool cost_model = false);

// ---- emitted-cost model of the structure-aware specialised kernels ----
// Entry class: 0 zero, 1 real, 2 imaginary, 3 complex, 4 exactly +1,
// 5 exactly -1, 6 exactly +i, 7 exactly -i.
int entry_class(const cplx &v);
// Host planning in parallel: fn(0..n-1) on a small persistent pool (the caller
// takes part; several callers may overlap). done(i) is polled by consumers
// that need results in order: wait_for(i) returns once fn(i) has finished,
// running other indices of the job meanwhile.
class StageJob {
  public:
    StageJob(size_t n, std::function<void(size_t)> fn);
    ~StageJob(); // waits for indices still running
    void wait_for(size_t i);
    struct Impl;

  private:
    std::shared_ptr<Impl> impl_;
};

// fn(begin, end) over [0, n) in chunks on the planning pool; returns when all
// chunks are done. Small n runs inline.
void parallel_chunks(size_t n, size_t chunk, const std::function<void(size_t, size_t)> &fn);

// Gradient slots that share a destination, chained in slot order:
// link[j] = (next slot of dst[j], or -1) * 2 + (1 if j is its destination's first slot)
std::vector<long long> slot_links(const std::vector<long long> &dst);
// FP64 instructions per amplitude of an op's register code: per output row
// a unit entry is emitted first and costs nothing (a copy), every other term
// 2 (unit, real, imaginary) or 4 (complex); identity sub-matrices cost
// nothing. Averaged over rows and condition values.
double subs_cost(const cplx *sub, int nt, int nc);
// The scalar s (a nonzero entry, or 1) minimising subs_cost(sub / s); its
// cost in *cost. Dividing every sub-matrix by s is exact for the entries
// equal to s (they become exactly 1).
cplx best_scale(const cplx *sub, int nt, int nc, double *cost);
// subs_cost after best_scale of an analysed op's matrices (cached in f.cost)
double op_cost(const FusedOp &f);
// sub / s entry by entry (textbook complex division, so x / x == 1 exactly)
void divide_by(cplx *sub, size_t count, const cplx &s);

} // namespace vqb
