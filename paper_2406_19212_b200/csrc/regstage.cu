// Register-resident stage executor (forward programs).
//
// A stage's tile (K = 12 tile bits = 4096 amplitudes) is split over 256
// threads x 16 registers. A *layout* assigns 4 tile bits to the register
// index and 8 to the thread index. Within a sub-stage every operation's
// mixing bits are register bits, so the operation is pure register
// arithmetic (FP64 FMA bound, no shared memory, no barrier). Between
// sub-stages the tile is re-laid out once through shared memory, XOR-swizzled
// so the three quarter-warp lane bits always hit distinct bank groups.
//
// The stage program (layouts, operations, sub-matrices) is passed as one
// __grid_constant__ parameter block: every thread reads the same words, so
// the matrices come through the constant cache (LDC) instead of occupying
// registers, which keeps the kernel at <= 128 registers = 2 blocks (16 warps)
// per SM; one block's HBM load overlaps the other's arithmetic.
//
// Host side: sub-stage packing reuses the stage planner's rule (an op may
// overtake a deferred one only if their supports are disjoint), with the
// register-bit budget instead of the tile budget.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"

namespace vqb {

void apply_gate_fast(double2 *a, int pn, const Gate &g, cudaStream_t st);

namespace {

constexpr int RB = 4;       // register bits
constexpr int R = 1 << RB;  // amplitudes per thread
constexpr int TB = 7;       // thread bits (per tile group)
constexpr int TG = 1 << TB; // threads per tile group
constexpr int G = 2;        // independent tile groups per block (named barriers)
constexpr int T = TG * G;   // threads per block
constexpr int K = RB + TB;  // tile bits
constexpr int TS = 1 << K;  // tile size

constexpr int kMaxSubs = 40;
constexpr int kMaxOps = 64;
constexpr int kMaxPool = 1024; // double2 entries

struct RLayout {
    int reg[RB]; // tile-local bit of register bit b
    int thr[TB]; // tile-local bit of thread bit b (thr[0..2]: quarter-warp lanes)
};

struct ROp {
    int nt, nc;
    int code;             // nt = 1: p0; nt = 2: pair index; nt = 3: triple index
    int per_group;        // condition depends on register bits
    int ck[kMaxCond];     // 0: outside tile, 1: thread bit, 2: register bit
    int cp[kMaxCond];     // global bit / thread bit / register bit
    unsigned mat;         // pool offset of 2^nc sub-matrices (ascending register order)
    unsigned nz;          // nt <= 2: union sparsity of the sub-matrices
    unsigned long long ident;
};

struct RSub {
    RLayout L;
    int op_begin, op_count;
};

struct RParams {
    int bits[K];                // tile bits ascending (global); local bit j <-> bits[j]
    unsigned long long ntiles;
    int nsubs;
    RSub subs[kMaxSubs];
    ROp ops[kMaxOps];
    double2 pool[kMaxPool];
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// shared-memory slot of a tile-local index: low 3 bits XOR-folded with the
// three higher 3-bit chunks (local bit l contributes to bank bit l mod 3).
// XOR-linear: swz(a | b) = swz(a) ^ swz(b) for disjoint a, b.
__host__ __device__ __forceinline__ int swz(int l) {
    return l ^ ((l >> 3) & 7) ^ ((l >> 6) & 7) ^ ((l >> 9) & 7);
}

// Per-thread addressing of one layout: slot(i) = st ^ XOR_{b in i} sw[b]
struct Addr {
    int st;
    int sw[RB];
};

__device__ __forceinline__ Addr layout_addr(const RLayout &L, int t) {
    Addr a;
    int td = 0;
#pragma unroll
    for (int b = 0; b < TB; ++b) td |= ((t >> b) & 1) << L.thr[b];
    a.st = swz(td);
#pragma unroll
    for (int b = 0; b < RB; ++b) a.sw[b] = swz(1 << L.reg[b]);
    return a;
}

__device__ __forceinline__ int slot(const Addr &a, int i) {
    int s = a.st;
#pragma unroll
    for (int b = 0; b < RB; ++b)
        if ((i >> b) & 1) s ^= a.sw[b];
    return s;
}

__device__ __forceinline__ int cond_of(const ROp &op, int cbase, int i) {
    int c = cbase;
#pragma unroll
    for (int q = 0; q < kMaxCond; ++q)
        if (q < op.nc && op.ck[q] == 2) c |= ((i >> op.cp[q]) & 1) << q;
    return c;
}

// nt-bit operation on register positions P[0..NT) (ascending). Group-major:
// each group's outputs are formed in a small temporary, entries of the
// sub-matrix are read from the parameter block (constant cache).
template <int NT, int P0, int P1 = 0, int P2 = 0, int P3 = 0>
__device__ __forceinline__ void apply_r(double2 (&v)[R], const ROp &op, const double2 *pool,
                                        int cbase) {
    constexpr int D = 1 << NT;
    constexpr int P[4] = {P0, P1, P2, P3};
    constexpr int MASK = (NT > 0 ? 1 << P0 : 0) | (NT > 1 ? 1 << P1 : 0) | (NT > 2 ? 1 << P2 : 0) |
                         (NT > 3 ? 1 << P3 : 0);
    auto off = [&](int r) constexpr {
        int o = 0;
        for (int q = 0; q < NT; ++q)
            if (r >> q & 1) o |= 1 << P[q];
        return o;
    };
    if (NT <= 2 && !op.per_group) {
        // uniform sub-matrix: loaded once into registers, reused by every group
        if ((op.ident >> cbase) & 1) return;
        const double2 *M = pool + op.mat + cbase * D * D;
        double2 m[D * D];
#pragma unroll
        for (int e = 0; e < D * D; ++e) m[e] = M[e];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & MASK) continue;
            double2 out[D];
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double2 acc = cmul(m[r], v[i | off(0)]);
#pragma unroll
                for (int s = 1; s < D; ++s) acc = cfma(m[r + s * D], v[i | off(s)], acc);
                out[r] = acc;
            }
#pragma unroll
            for (int r = 0; r < D; ++r) v[i | off(r)] = out[r];
        }
        return;
    }
    if (!op.per_group && ((op.ident >> cbase) & 1)) return;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & MASK) continue;
        const int c = op.per_group ? cond_of(op, cbase, i) : cbase;
        if (op.per_group && ((op.ident >> c) & 1)) continue;
        const double2 *M = pool + op.mat + c * D * D;
        double2 out[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double2 acc = cmul(M[r], v[i | off(0)]);
#pragma unroll
            for (int s = 1; s < D; ++s) acc = cfma(M[r + s * D], v[i | off(s)], acc);
            out[r] = acc;
        }
#pragma unroll
        for (int r = 0; r < D; ++r) v[i | off(r)] = out[r];
    }
}

__device__ __forceinline__ void apply_diag(double2 (&v)[R], const ROp &op, const double2 *pool,
                                           int cbase) {
    if (!op.per_group) {
        if ((op.ident >> cbase) & 1) return;
        const double2 ph = pool[op.mat + cbase];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = cmul(ph, v[i]);
        return;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int c = cond_of(op, cbase, i);
        if ((op.ident >> c) & 1) continue;
        v[i] = cmul(pool[op.mat + c], v[i]);
    }
}

__device__ __forceinline__ void dispatch(double2 (&v)[R], const ROp &op, const double2 *pool,
                                         int cbase) {
    switch (op.nt) {
    case 0: apply_diag(v, op, pool, cbase); return;
    case 1:
        switch (op.code) {
        case 0: apply_r<1, 0>(v, op, pool, cbase); return;
        case 1: apply_r<1, 1>(v, op, pool, cbase); return;
        case 2: apply_r<1, 2>(v, op, pool, cbase); return;
        default: apply_r<1, 3>(v, op, pool, cbase); return;
        }
    case 2:
        switch (op.code) {
        case 0: apply_r<2, 0, 1>(v, op, pool, cbase); return;
        case 1: apply_r<2, 0, 2>(v, op, pool, cbase); return;
        case 2: apply_r<2, 0, 3>(v, op, pool, cbase); return;
        case 3: apply_r<2, 1, 2>(v, op, pool, cbase); return;
        case 4: apply_r<2, 1, 3>(v, op, pool, cbase); return;
        default: apply_r<2, 2, 3>(v, op, pool, cbase); return;
        }
    case 3:
        switch (op.code) {
        case 0: apply_r<3, 0, 1, 2>(v, op, pool, cbase); return;
        case 1: apply_r<3, 0, 1, 3>(v, op, pool, cbase); return;
        case 2: apply_r<3, 0, 2, 3>(v, op, pool, cbase); return;
        default: apply_r<3, 1, 2, 3>(v, op, pool, cbase); return;
        }
    default: apply_r<4, 0, 1, 2, 3>(v, op, pool, cbase); return;
    }
}

// barrier over the 128 threads of one tile group
__device__ __forceinline__ void group_sync(int grp) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(grp + 1), "r"(TG) : "memory");
}

__global__ void __launch_bounds__(T, 1)
    k_regstage(double2 *__restrict__ amps, const __grid_constant__ RParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int grp = threadIdx.x / TG;          // tile group: its own tiles, buffers, barrier
    const int t = threadIdx.x % TG;
    double2 *stage_buf = reinterpret_cast<double2 *>(smem_raw) + (size_t)grp * 2 * TS;
    double2 *xbuf = stage_buf + TS;

    // natural tile order j = t + T*s: global offset glo | gh(s), slot swz(j)
    unsigned long long glo = 0;
#pragma unroll
    for (int b = 0; b < TB; ++b)
        if ((t >> b) & 1) glo |= 1ull << P.bits[b];
    unsigned long long gh[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) gh[b] = 1ull << P.bits[TB + b];
    const int nat_st = swz(t);
    int nat_sw[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) nat_sw[b] = swz(TG << b);
    auto tile_base = [&](unsigned long long c) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int s = P.bits[i];
            c = ((c >> s) << (s + 1)) | (c & ((1ull << s) - 1));
        }
        return c;
    };
    auto prefetch = [&](unsigned long long tile) {
        const unsigned long long base = tile_base(tile);
#pragma unroll
        for (int s = 0; s < R; ++s) {
            unsigned long long g = base | glo;
            int sl = nat_st;
#pragma unroll
            for (int b = 0; b < RB; ++b)
                if ((s >> b) & 1) {
                    g |= gh[b];
                    sl ^= nat_sw[b];
                }
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&stage_buf[sl]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(&amps[g]));
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };

    const unsigned long long tstride = (unsigned long long)gridDim.x * G;
    unsigned long long tile = (unsigned long long)blockIdx.x * G + grp;
    if (tile < P.ntiles) prefetch(tile);
    for (; tile < P.ntiles; tile += tstride) {
        const unsigned long long base = tile_base(tile);
        asm volatile("cp.async.wait_group 0;\n" ::);
        group_sync(grp);
        double2 v[R];
        Addr A = layout_addr(P.subs[0].L, t);
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = stage_buf[slot(A, i)];
        group_sync(grp); // staging consumed: refill it with the next tile
        if (tile + tstride < P.ntiles) prefetch(tile + tstride);
        int cur = 0;
        for (int sub = 0; sub < P.nsubs; ++sub) {
            if (sub > 0) {
#pragma unroll
                for (int i = 0; i < R; ++i) xbuf[slot(A, i)] = v[i];
                group_sync(grp);
                A = layout_addr(P.subs[sub].L, t);
#pragma unroll
                for (int i = 0; i < R; ++i) v[i] = xbuf[slot(A, i)];
                group_sync(grp); // xbuf free for the next relayout
                cur = sub;
            }
            const RSub &sb = P.subs[sub];
            for (int o = 0; o < sb.op_count; ++o) {
                const ROp &op = P.ops[sb.op_begin + o];
                int cbase = 0;
                for (int q = 0; q < op.nc; ++q) {
                    if (op.ck[q] == 0) cbase |= (int)((base >> op.cp[q]) & 1) << q;
                    else if (op.ck[q] == 1) cbase |= ((t >> op.cp[q]) & 1) << q;
                }
                dispatch(v, op, P.pool, cbase);
            }
        }
        // store from registers in the final layout
        const RLayout &L = P.subs[cur].L;
        unsigned long long g0 = base;
#pragma unroll
        for (int b = 0; b < TB; ++b)
            if ((t >> b) & 1) g0 |= 1ull << P.bits[L.thr[b]];
        unsigned long long gr[RB];
#pragma unroll
        for (int b = 0; b < RB; ++b) gr[b] = 1ull << P.bits[L.reg[b]];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            unsigned long long g = g0;
#pragma unroll
            for (int b = 0; b < RB; ++b)
                if ((i >> b) & 1) g |= gr[b];
            amps[g] = v[i];
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// ---------------------------------------------------------------- host planning
int pair_code(int a, int b) { // a < b in [0,4)
    static const int code[4][4] = {{-1, 0, 1, 2}, {-1, -1, 3, 4}, {-1, -1, -1, 5}, {}};
    return code[a][b];
}
int triple_code(int a, int b, int c) {
    const int missing = 6 - a - b - c; // {0,1,2}->0, {0,1,3}->1, {0,2,3}->2, {1,2,3}->3
    return 3 - missing;
}

// reorder the local bits of a (2^nt x 2^nt) matrix: new bit q = old bit perm[q]
cvec permute_matrix(const cvec &m, int nt, const int *perm) {
    const int d = 1 << nt;
    auto map = [&](int nidx) {
        int o = 0;
        for (int q = 0; q < nt; ++q)
            if (nidx >> q & 1) o |= 1 << perm[q];
        return o;
    };
    cvec out(m.size());
    for (int c = 0; c < d; ++c)
        for (int r = 0; r < d; ++r) out[r + c * d] = m[map(r) + map(c) * d];
    return out;
}

// Choose thread bits: thr[0..2] with distinct residues mod 3 (bank-conflict
// free under swz), preferring local bits 0,1,2.
void choose_threads(RLayout &L, const std::vector<int> &fb) {
    int lanes[3] = {-1, -1, -1};
    auto used = [&](int b) { return lanes[0] == b || lanes[1] == b || lanes[2] == b; };
    for (int want = 0; want < 3; ++want)
        if (std::find(fb.begin(), fb.end(), want) != fb.end()) lanes[want] = want;
    for (int r = 0; r < 3; ++r)
        if (lanes[r] < 0)
            for (int b : fb)
                if (!used(b) && b % 3 == r) {
                    lanes[r] = b;
                    break;
                }
    for (int r = 0; r < 3; ++r) // fall back: any unused bit (bank conflicts possible)
        if (lanes[r] < 0)
            for (int b : fb)
                if (!used(b)) {
                    lanes[r] = b;
                    break;
                }
    int k = 0;
    for (int r = 0; r < 3; ++r) L.thr[k++] = lanes[r];
    for (int b : fb)
        if (!used(b)) L.thr[k++] = b;
}

// Lower one stage into its parameter block; false if it does not fit.
bool lower_stage_reg(const Stage &sg, const std::vector<FusedOp> &blocks, int pn, RParams &P) {
    std::memset(&P, 0, sizeof P);
    for (int j = 0; j < K; ++j) P.bits[j] = sg.bits[j];
    P.ntiles = 1ull << (pn - K);
    auto local_of = [&](int g) {
        for (int j = 0; j < K; ++j)
            if (sg.bits[j] == g) return j;
        return -1;
    };
    int nops = 0, npool = 0;
    std::vector<int> remaining(blocks.size());
    for (size_t i = 0; i < blocks.size(); ++i) remaining[i] = (int)i;
    while (!remaining.empty()) {
        if (P.nsubs >= kMaxSubs) return false;
        unsigned rset = 0;
        uint64_t blocked = 0;
        std::vector<int> taken, deferred;
        for (int i : remaining) {
            const FusedOp &f = blocks[i];
            unsigned mix = 0;
            for (int q = 0; q < f.nt; ++q) mix |= 1u << local_of(f.mix[q]);
            if ((f.support & blocked) || __builtin_popcount(rset | mix) > RB) {
                deferred.push_back(i);
                blocked |= f.support;
                continue;
            }
            rset |= mix;
            taken.push_back(i);
        }
        // pad the register set: bits the deferred ops need, then high bits
        for (int i : deferred) {
            const FusedOp &f = blocks[i];
            unsigned mix = 0;
            for (int q = 0; q < f.nt; ++q) mix |= 1u << local_of(f.mix[q]);
            if (__builtin_popcount(rset | mix) <= RB) rset |= mix;
        }
        for (int j = K - 1; j >= 0 && __builtin_popcount(rset) < RB; --j) rset |= 1u << j;
        RSub &sb = P.subs[P.nsubs++];
        int nr = 0;
        std::vector<int> free_bits;
        for (int j = 0; j < K; ++j) {
            if (rset >> j & 1) sb.L.reg[nr++] = j;
            else free_bits.push_back(j);
        }
        choose_threads(sb.L, free_bits);
        auto reg_of = [&](int j) {
            for (int b = 0; b < RB; ++b)
                if (sb.L.reg[b] == j) return b;
            return -1;
        };
        auto thr_of = [&](int j) {
            for (int b = 0; b < TB; ++b)
                if (sb.L.thr[b] == j) return b;
            return -1;
        };
        sb.op_begin = nops;
        for (int i : taken) {
            const FusedOp &f = blocks[i];
            if (nops >= kMaxOps) return false;
            ROp &o = P.ops[nops++];
            o.nt = f.nt;
            o.nc = f.nc;
            int rp[kMaxMix], order[kMaxMix];
            for (int q = 0; q < f.nt; ++q) {
                rp[q] = reg_of(local_of(f.mix[q]));
                order[q] = q;
            }
            std::sort(order, order + f.nt, [&](int x, int y) { return rp[x] < rp[y]; });
            int perm[kMaxMix], srp[kMaxMix];
            for (int q = 0; q < f.nt; ++q) {
                perm[q] = order[q];
                srp[q] = rp[order[q]];
            }
            if (f.nt == 1) o.code = srp[0];
            if (f.nt == 2) o.code = pair_code(srp[0], srp[1]);
            if (f.nt == 3) o.code = triple_code(srp[0], srp[1], srp[2]);
            for (int q = 0; q < f.nc; ++q) {
                const int j = local_of(f.cnd[q]);
                if (j < 0) {
                    o.ck[q] = 0;
                    o.cp[q] = f.cnd[q];
                } else if (reg_of(j) >= 0) {
                    o.ck[q] = 2;
                    o.cp[q] = reg_of(j);
                    o.per_group = 1;
                } else {
                    o.ck[q] = 1;
                    o.cp[q] = thr_of(j);
                }
            }
            const int D = 1 << f.nt, dd = D * D;
            if (npool + (dd << f.nc) > kMaxPool) return false;
            o.mat = (unsigned)npool;
            for (int c = 0; c < (1 << f.nc); ++c) {
                const cvec sub(f.sub_phi.begin() + size_t(c) * dd,
                               f.sub_phi.begin() + size_t(c + 1) * dd);
                const cvec pm = f.nt > 1 ? permute_matrix(sub, f.nt, perm) : sub;
                bool ident = true;
                for (int r = 0; r < D; ++r)
                    for (int s = 0; s < D; ++s) {
                        const cplx x = pm[r + s * D];
                        if (x != (r == s ? cplx(1) : cplx(0))) ident = false;
                        if (f.nt <= 2 && x != cplx(0)) o.nz |= 1u << (r + s * D);
                    }
                if (ident) o.ident |= 1ull << c;
                for (const auto &x : pm) P.pool[npool++] = make_double2(x.real(), x.imag());
            }
        }
        sb.op_count = nops - sb.op_begin;
        remaining.swap(deferred);
    }
    return true;
}

} // namespace

bool regstage_available(int pn) { return pn >= K; }

void run_program_fused_smem_stage(DeviceState *s, const std::vector<FusedOp> &fops,
                                  const Stage &sg);

// Forward program on the register-resident executor. Unfusable ops go
// through the element-by-element kernels; a stage whose program does not fit
// the parameter block goes through the shared-memory executor.
void run_program_reg(DeviceState *s, const std::vector<Gate> &prog) {
    std::vector<FusedOp> fops;
    fops.reserve(prog.size());
    for (const auto &g : prog) fops.push_back(analyse_gate(g));
    const auto stages = plan_stages(fops, s->pn, K);
    const char *fq = std::getenv("VQB_FUSE_QUBITS");
    const int max_support = fq ? std::atoi(fq) : 2;
    cudaStream_t st = s->stream;
    const size_t smem = (size_t)G * 2 * TS * sizeof(double2);
    static bool attr = false;
    if (!attr) {
        VQB_CUDA(cudaFuncSetAttribute(k_regstage, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        attr = true;
    }
    int nsm = 148, dev = 0, per_sm = 1;
    VQB_CUDA(cudaGetDevice(&dev));
    VQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    VQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_regstage, T, smem));
    static thread_local RParams P; // ~26 KB, host staging of the parameter block
    for (const Stage &sg : stages) {
        if (!sg.fused) {
            apply_gate_fast(s->amps, s->pn, fops[sg.ops[0]].gate, st);
            continue;
        }
        std::vector<FusedOp> blocks;
        if (max_support > 0) blocks = fuse_blocks(fops, sg.ops, max_support);
        else
            for (int idx : sg.ops) blocks.push_back(fops[idx]);
        if (!lower_stage_reg(sg, blocks, s->pn, P)) {
            run_program_fused_smem_stage(s, fops, sg);
            continue;
        }
        if (std::getenv("VQB_PLAN_STATS")) {
            int nt_hist[5] = {0, 0, 0, 0, 0}, nops = 0;
            for (int i = 0; i < P.nsubs; ++i) nops += P.subs[i].op_count;
            for (int i = 0; i < nops; ++i) nt_hist[std::min(P.ops[i].nt, 4)]++;
            std::fprintf(stderr, "[regstage] gates %zu blocks %zu subs %d ops nt0..4 %d %d %d %d %d\n",
                         sg.ops.size(), blocks.size(), P.nsubs, nt_hist[0], nt_hist[1], nt_hist[2],
                         nt_hist[3], nt_hist[4]);
        }
        const int grid = (int)std::min<unsigned long long>((unsigned long long)nsm * std::max(per_sm, 1),
                                                           (P.ntiles + G - 1) / G);
        const ProfMark pf_ = prof_begin(st);
        k_regstage<<<grid, T, smem, st>>>(s->amps, P);
        check_launch("k_regstage", pf_);
    }
    VQB_CUDA(cudaStreamSynchronize(st));
}

} // namespace vqb
