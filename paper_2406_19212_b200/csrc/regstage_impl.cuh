// Register-resident stage executor (forward programs and adjoint sweeps).
//
// Included once per geometry (regstage.cu, regstage_r8.cu) with
//   VQB_RS_RB  register bits (amplitudes per thread and state = 2^RB)
//   VQB_RS_TB  thread bits (threads per block = 2^TB)
//   VQB_RS_NS  namespace of this instantiation
//   VQB_RS_FWD_BLOCKS / VQB_RS_REV_BLOCKS  target blocks per SM
// e.g. RB = 4, TB = 7: a stage's tile (K = 11 tile bits = 2048 amplitudes per
// state) is split over 128 threads x 16 registers. A *layout* assigns RB tile
// bits to the register index and TB to the thread index. Within a sub-stage every operation's
// mixing bits are register bits, so the operation is pure register arithmetic
// (FP64 FMA bound, no shared memory, no barrier). Between sub-stages the tile
// is re-laid out once through shared memory, XOR-swizzled so the three
// quarter-warp lane bits always hit distinct bank groups. The next tile is
// prefetched with cp.async (LDGSTS) into a staging buffer while the current
// one is computed; results are stored straight from registers. Two blocks run
// per SM, so one block's relayout or load phase overlaps the other's FP64.
//
// The stage program (layouts, operations, sub-matrices) is one
// __grid_constant__ parameter block (read through the constant cache);
// programs that do not fit are split over several launches of the same tile
// bits.
//
// Adjoint mode (REV): each thread holds 16 amplitudes of Phi and of Psi; a
// parametric step computes Phi <- inv Phi, Re <Psi| D_p |Phi>, Psi <- inv Psi
// in registers (reverse_sweep_step kernels.hpp:659-697); contributions are
// reduced per warp into shared-memory slots, per block into a partial row,
// and over blocks in fixed order by k_grads (deterministic for a fixed grid).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

#include "jit.hpp"
#include <map>
#include "plan.hpp"

#define VQB_RS_STR2(x) #x
#define VQB_RS_STR1(x) VQB_RS_STR2(x)
#define VQB_RS_STR VQB_RS_STR1(VQB_RS_NS)
namespace vqb {

void apply_gate_fast(double2 *a, int pn, const Gate &g, cudaStream_t st);
void note_flops(double f);
void reverse_step_async(double2 *phi, double2 *psi, int pn, const int *pos1, int m,
                        const cvec &inv, const std::vector<cvec> &dmats, DeviceState *w,
                        double2 *out_c, double *out_r, double real_scale);

namespace VQB_RS_NS {
namespace {

constexpr int RB = VQB_RS_RB; // register bits
constexpr int R = 1 << RB;  // amplitudes per thread (per state)
constexpr int TB = VQB_RS_TB; // thread bits
constexpr int T = 1 << TB;  // threads per block (one tile per block at a time)
constexpr int NW = T / 32;  // warps per block
constexpr int K = RB + TB;  // tile bits
constexpr int TS = 1 << K;  // tile size

// adjoint gradient partials: lanes reduced by shuffles per partial sum (the
// rest stay separate shared-memory partials, summed once per block)
#ifndef VQB_RS_LANES_PER_PART
#define VQB_RS_LANES_PER_PART 32
#endif
constexpr int LANES_PER_PART = VQB_RS_LANES_PER_PART;
constexpr int NPART = NW * (32 / LANES_PER_PART);

// register bit 3 in the dispatch tables (never selected when RB = 3)
constexpr int B3 = RB > 3 ? 3 : 0;

constexpr int kMaxSubs = 32;
constexpr int kMaxOps = 84; // (ROp is 112 bytes: the parameter block stays under 32 KB)
constexpr int kMaxSlots = 64;
constexpr int kMaxPool = 1072; // double2 entries
constexpr int kMaxTab = 192;   // per-element diagonal tables, copied to shared memory

struct RLayout {
    int reg[RB]; // tile-local bit of register bit b
    int thr[TB]; // tile-local bit of thread bit b (thr[0..2]: quarter-warp lanes)
};

struct ROp {
    int nt, nc, np;
    int code;             // nt = 1: register bit; nt = 2: pair index
    int per_group;        // condition depends on register bits
    int pair;             // psi has its own matrices (channel steps)
    int slot;             // first gradient slot (param ops)
    signed char ck[kMaxCond]; // 0: outside tile, 1: thread bit, 2: register bit
    signed char cp[kMaxCond]; // global bit / thread bit / register bit
    unsigned mat, mat_psi, mat_d; // pool offsets (2^nc sub-matrices each, ascending order)
    unsigned long long ident, ident_psi;
    unsigned char rw[RB]; // condition-index bits contributed by register bit b
    int tab, tab_psi;     // nt = 0 with register conditions: shared-memory tables
    int xoff, nx;         // nt >= 3: XOR patterns of the diagonal-times-permutation terms
    signed char lb[kMaxMix]; // nt >= 3: tile-local mixing bits in matrix bit order
    // nt = 0 adjoint steps: every phase has modulus 1 (conj(psi) phi is then
    // invariant under the step) and, for parametric ones, the tables
    // e_p[c] = D_p[c] * M[c] at pool offset mat_e
    int unit;
    unsigned mat_e;
    // nt >= 3 operation whose mixing bits are all register bits (specialised
    // kernels only): lb[q] is then the register bit of matrix bit q and the
    // XOR-term pool is applied in registers, no shared-memory round trip
    int inreg;
};

struct RSub {
    RLayout L;
    int op_begin, op_count;
};

struct RParams {
    int bits[K];                // tile bits ascending (global); local bit j <-> bits[j]
    unsigned long long ntiles;
    int nsubs, nslots, slot_begin, partial_ld;
    RSub subs[kMaxSubs];
    ROp ops[kMaxOps];
    double2 pool[kMaxPool];
    double2 tab[kMaxTab];
    int ntab, nxpat, npool;
    unsigned char xpat[256];
    // forward fast path: unconditioned 1- and 2-bit register ops packed as
    // (pool offset << 4) | variant (1..4: nt=1 on register bit v-1; 5..10:
    // nt=2 pair code v-5); 0 = general path. One word per op, loaded one op
    // ahead, replaces the dependent descriptor loads of the general path.
    int fast[kMaxOps];
};
static_assert(sizeof(RParams) <= 32000, "kernel parameter block too large");

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// Re(conj(a) * b)
__device__ __forceinline__ double re_cj(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }

// shared-memory slot of a tile-local index: low 3 bits XOR-folded with the
// higher 3-bit chunks (local bit l contributes to bank bit l mod 3).
// XOR-linear: swz(a | b) = swz(a) ^ swz(b) for disjoint a, b.
__host__ __device__ __forceinline__ int swz(int l) {
    return l ^ ((l >> 3) & 7) ^ ((l >> 6) & 7) ^ ((l >> 9) & 7);
}

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

// condition value of register element i (a compile-time constant in the
// unrolled loops): the per-register-bit masks are ORed in
__device__ __forceinline__ int cond_of(const ROp &op, int cbase, int i) {
    int c = cbase;
#pragma unroll
    for (int b = 0; b < RB; ++b)
        if ((i >> b) & 1) c |= op.rw[b];
    return c;
}

template <int NT, int P0, int P1, int P2, int P3> struct Pos {
    static constexpr int D = 1 << NT;
    static constexpr int MASK = (NT > 0 ? 1 << P0 : 0) | (NT > 1 ? 1 << P1 : 0) |
                                (NT > 2 ? 1 << P2 : 0) | (NT > 3 ? 1 << P3 : 0);
    __host__ __device__ static constexpr int off(int r) {
        int o = 0;
        if (NT > 0 && (r & 1)) o |= 1 << P0;
        if (NT > 1 && (r & 2)) o |= 1 << P1;
        if (NT > 2 && (r & 4)) o |= 1 << P2;
        if (NT > 3 && (r & 8)) o |= 1 << P3;
        return o;
    }
};

// out = M * v[group], written back in place; M read element by element.
template <class PS>
__device__ __forceinline__ void group_mv(double2 (&v)[R], int i, const double2 *M) {
    constexpr int D = PS::D;
    double2 out[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double2 acc = cmul(M[r], v[i | PS::off(0)]);
#pragma unroll
        for (int s = 1; s < D; ++s) acc = cfma(M[r + s * D], v[i | PS::off(s)], acc);
        out[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < D; ++r) v[i | PS::off(r)] = out[r];
}

// Apply an nt-bit operation (sub-matrices at `mat`) to one register state.
// HOIST: a uniform sub-matrix of nt <= HOIST is loaded into registers once.
template <int HOIST, int NT, int P0, int P1 = 0, int P2 = 0, int P3 = 0>
__device__ __forceinline__ void apply_r(double2 (&v)[R], const ROp &op, const double2 *pool,
                                        int cbase, unsigned mat, unsigned long long ident) {
    using PS = Pos<NT, P0, P1, P2, P3>;
    constexpr int D = PS::D;
    if (NT <= HOIST && !op.per_group) {
        if ((ident >> cbase) & 1) return;
        const double2 *M = pool + mat + cbase * D * D;
        double2 m[D * D];
#pragma unroll
        for (int e = 0; e < D * D; ++e) m[e] = M[e];
#pragma unroll
        for (int i = 0; i < R; ++i)
            if (!(i & PS::MASK)) group_mv<PS>(v, i, m);
        return;
    }
    if (!op.per_group && ((ident >> cbase) & 1)) return;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & PS::MASK) continue;
        const int c = op.per_group ? cond_of(op, cbase, i) : cbase;
        if (op.per_group && ((ident >> c) & 1)) continue;
        group_mv<PS>(v, i, pool + mat + c * D * D);
    }
}

// Reverse-sweep parametric step on (phi, psi) registers.
template <int NT, int P0, int P1 = 0, int P2 = 0, int P3 = 0>
__device__ __forceinline__ void param_r(double2 (&vf)[R], double2 (&vg)[R], const ROp &op,
                                        const double2 *pool, int cbase, double (&acc)[VQB_MAX_PARAMS]) {
    using PS = Pos<NT, P0, P1, P2, P3>;
    constexpr int D = PS::D;
    const int nsub = 1 << op.nc;
    if (NT == 0 && op.per_group && op.np == 1 && op.tab >= 0) {
        // diagonal step with per-element conditions: tables in shared memory
        // (the first kMaxTab entries of the dynamic shared memory)
        extern __shared__ __align__(16) unsigned char smem_raw[];
        const double2 *stab = reinterpret_cast<const double2 *>(smem_raw);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int c = cond_of(op, cbase, i);
            const double2 m = stab[op.tab + c], d = stab[op.tab + nsub + c];
            const double2 w = cmul(m, vf[i]);
            vf[i] = w;
            acc[0] += re_cj(vg[i], cmul(d, w));
            vg[i] = cmul(m, vg[i]);
        }
        return;
    }
    if (NT <= 1 && !op.per_group && op.np == 1) {
        double2 m[D * D], d[D * D];
#pragma unroll
        for (int e = 0; e < D * D; ++e) {
            m[e] = pool[op.mat + cbase * D * D + e];
            d[e] = pool[op.mat_d + cbase * D * D + e];
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            if (i & PS::MASK) continue;
            group_mv<PS>(vf, i, m);
            double a = 0;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double2 x = cmul(d[r], vf[i | PS::off(0)]);
#pragma unroll
                for (int s = 1; s < D; ++s) x = cfma(d[r + s * D], vf[i | PS::off(s)], x);
                a += re_cj(vg[i | PS::off(r)], x);
            }
            acc[0] += a;
            group_mv<PS>(vg, i, m);
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i & PS::MASK) continue;
        const int c = op.per_group ? cond_of(op, cbase, i) : cbase;
        group_mv<PS>(vf, i, pool + op.mat + c * D * D);
#pragma unroll
        for (int p = 0; p < VQB_MAX_PARAMS; ++p) {
            if (p >= op.np) break;
            const double2 *Dm = pool + op.mat_d + (p * nsub + c) * D * D;
            double a = 0;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double2 x = cmul(Dm[r], vf[i | PS::off(0)]);
#pragma unroll
                for (int s = 1; s < D; ++s) x = cfma(Dm[r + s * D], vf[i | PS::off(s)], x);
                a += re_cj(vg[i | PS::off(r)], x);
            }
            acc[p] += a;
        }
        group_mv<PS>(vg, i, pool + op.mat + c * D * D);
    }
}

__device__ __forceinline__ void apply_diag(double2 (&v)[R], const ROp &op, const double2 *pool,
                                           int cbase, unsigned mat, unsigned long long ident) {
    if (!op.per_group) {
        if ((ident >> cbase) & 1) return;
        const double2 ph = pool[mat + cbase];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = cmul(ph, v[i]);
        return;
    }
    const int tabo = mat == op.mat ? op.tab : op.tab_psi;
    if (tabo >= 0) {
        // per-element phase from the shared-memory copy of the table
        extern __shared__ __align__(16) unsigned char smem_raw[];
        const double2 *stab = reinterpret_cast<const double2 *>(smem_raw) + tabo;
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = cmul(stab[cond_of(op, cbase, i)], v[i]);
        return;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int c = cond_of(op, cbase, i);
        if ((ident >> c) & 1) continue;
        v[i] = cmul(pool[mat + c], v[i]);
    }
}

template <int NT, int P0, int P1 = 0>
__device__ __forceinline__ void apply_hoisted(double2 (&v)[R], const double2 *M) {
    using PS = Pos<NT, P0, P1, 0, 0>;
#if !VQB_RS_HOIST
    // entries re-read per group (broadcast shared-memory loads), no register copy
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (!(i & PS::MASK)) group_mv<PS>(v, i, M);
#else
    constexpr int D = PS::D;
    double2 m[D * D];
#pragma unroll
    for (int e = 0; e < D * D; ++e) m[e] = M[e];
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (!(i & PS::MASK)) group_mv<PS>(v, i, m);
#endif
}

__device__ __forceinline__ void apply_fast(double2 (&v)[R], const double2 *pool, int w) {
    const double2 *M = pool + (w >> 4);
    switch (w & 15) {
    case 1: apply_hoisted<1, 0>(v, M); return;
    case 2: apply_hoisted<1, 1>(v, M); return;
    case 3: apply_hoisted<1, 2>(v, M); return;
    case 4: apply_hoisted<1, B3>(v, M); return;
    case 5: apply_hoisted<2, 0, 1>(v, M); return;
    case 6: apply_hoisted<2, 0, 2>(v, M); return;
    case 7: apply_hoisted<2, 0, B3>(v, M); return;
    case 8: apply_hoisted<2, 1, 2>(v, M); return;
    case 9: apply_hoisted<2, 1, B3>(v, M); return;
    default: apply_hoisted<2, 2, B3>(v, M); return;
    }
}

template <int HOIST, int MAXNT>
__device__ __forceinline__ void dispatch(double2 (&v)[R], const ROp &op, const double2 *pool,
                                         int cbase, unsigned mat, unsigned long long ident) {
    if (op.nt > MAXNT) return; // the caller routes wider ops elsewhere
    switch (op.nt) {
    case 0: apply_diag(v, op, pool, cbase, mat, ident); return;
    case 1:
        switch (op.code) {
        case 0: apply_r<HOIST, 1, 0>(v, op, pool, cbase, mat, ident); return;
        case 1: apply_r<HOIST, 1, 1>(v, op, pool, cbase, mat, ident); return;
        case 2: apply_r<HOIST, 1, 2>(v, op, pool, cbase, mat, ident); return;
        default: apply_r<HOIST, 1, B3>(v, op, pool, cbase, mat, ident); return;
        }
    case 2:
        switch (op.code) {
        case 0: apply_r<HOIST, 2, 0, 1>(v, op, pool, cbase, mat, ident); return;
        case 1: apply_r<HOIST, 2, 0, 2>(v, op, pool, cbase, mat, ident); return;
        case 2: apply_r<HOIST, 2, 0, B3>(v, op, pool, cbase, mat, ident); return;
        case 3: apply_r<HOIST, 2, 1, 2>(v, op, pool, cbase, mat, ident); return;
        case 4: apply_r<HOIST, 2, 1, B3>(v, op, pool, cbase, mat, ident); return;
        default: apply_r<HOIST, 2, 2, B3>(v, op, pool, cbase, mat, ident); return;
        }
    default: return; // nt >= 3 runs through smem_op
    }
}

__device__ __forceinline__ void dispatch_param(double2 (&vf)[R], double2 (&vg)[R], const ROp &op,
                                               const double2 *pool, int cbase,
                                               double (&acc)[VQB_MAX_PARAMS]) {
    switch (op.nt) {
    case 0: param_r<0, 0>(vf, vg, op, pool, cbase, acc); return;
    case 1:
        switch (op.code) {
        case 0: param_r<1, 0>(vf, vg, op, pool, cbase, acc); return;
        case 1: param_r<1, 1>(vf, vg, op, pool, cbase, acc); return;
        case 2: param_r<1, 2>(vf, vg, op, pool, cbase, acc); return;
        default: param_r<1, B3>(vf, vg, op, pool, cbase, acc); return;
        }
    case 2:
        switch (op.code) {
        case 0: param_r<2, 0, 1>(vf, vg, op, pool, cbase, acc); return;
        case 1: param_r<2, 0, 2>(vf, vg, op, pool, cbase, acc); return;
        case 2: param_r<2, 0, B3>(vf, vg, op, pool, cbase, acc); return;
        case 3: param_r<2, 1, 2>(vf, vg, op, pool, cbase, acc); return;
        case 4: param_r<2, 1, B3>(vf, vg, op, pool, cbase, acc); return;
        default: param_r<2, 2, B3>(vf, vg, op, pool, cbase, acc); return;
        }
    default: return; // wider parametric steps are planned as unfusable
    }
}

// Wide (nt >= 3) operation on one state through the relayout buffer: the
// registers go to shared memory in layout L, the operation runs over 2^(K-nt)
// groups per tile with the outputs written straight back, and the registers
// are reloaded. Used by the adjoint kernel, whose two register states leave
// no room for 8- or 16-element groups.
template <int NT>
__device__ __forceinline__ void smem_op(double2 (&v)[R], const Addr &A, const RLayout &L,
                                        double2 *xbuf, const ROp &op, const double2 *pool,
                                        int cbase_uni, unsigned mat, unsigned long long ident,
                                        int t, const unsigned char *P_xpat) {
    constexpr int D = 1 << NT;
    // tile-local mixing bits (matrix bit order; any local bits, not only
    // register bits), then ascending for the group enumeration
    int lb[NT], sorted[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) sorted[q] = lb[q] = op.lb[q];
#pragma unroll
    for (int a = 0; a < NT; ++a)
#pragma unroll
        for (int b = 0; b + 1 < NT - a; ++b)
            if (sorted[b] > sorted[b + 1]) {
                const int x = sorted[b];
                sorted[b] = sorted[b + 1];
                sorted[b + 1] = x;
            }
    int sw_off[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        int o = 0;
#pragma unroll
        for (int q = 0; q < NT; ++q)
            if (r >> q & 1) o |= 1 << lb[q];
        sw_off[r] = swz(o);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) xbuf[slot(A, i)] = v[i];
    __syncthreads();
    for (int g = t; g < (TS >> NT); g += T) {
        int b = g;
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const int s = sorted[q];
            b = ((b >> s) << (s + 1)) | (b & ((1 << s) - 1));
        }
        int c = cbase_uni;
        for (int q = 0; q < op.nc; ++q) {
            const int l = op.ck[q] == 1 ? L.thr[op.cp[q]] : (op.ck[q] == 2 ? L.reg[op.cp[q]] : -1);
            if (l >= 0) c |= ((b >> l) & 1) << q;
        }
        if ((ident >> c) & 1) continue;
        // S = sum_k diag(d_k) P_{x_k}: out[r] = sum_k d_k[r] in[r ^ x_k]; the
        // swizzle is XOR-linear, so slot(r ^ x) = slot(r) ^ slot(x)
        const double2 *Mc = pool + mat + c * op.nx * D;
        const int sb = swz(b);
        double2 out[D];
#pragma unroll
        for (int r = 0; r < D; ++r) out[r] = make_double2(0, 0);
        for (int k = 0; k < op.nx; ++k) {
            const int x = P_xpat[op.xoff + k];
            int sx = 0;
#pragma unroll
            for (int q = 0; q < NT; ++q)
                if ((x >> q) & 1) sx ^= sw_off[1 << q];
            const double2 *dk = Mc + k * D;
#pragma unroll
            for (int r = 0; r < D; ++r) out[r] = cfma(dk[r], xbuf[sb ^ sw_off[r] ^ sx], out[r]);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < D; ++r) xbuf[sb ^ sw_off[r]] = out[r];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = xbuf[slot(A, i)];
    __syncthreads();
}

// WIDE = false: forward stages without nt >= 3 operations (leaner registers).
// Those run unstaged: tiles are loaded straight into registers (coalesced,
// natural order) and re-laid out once, with no cp.async staging tile, so the
// smaller shared-memory footprint fits more blocks per SM and the other
// blocks' arithmetic covers each block's load.
#ifndef VQB_RS_HOIST
#define VQB_RS_HOIST 0
#endif
#ifndef VQB_RS_FWD_STAGED
#define VQB_RS_FWD_STAGED 1
#endif
template <bool REV, bool WIDE> constexpr bool kStaged = REV || WIDE || VQB_RS_FWD_STAGED;
template <bool REV, bool WIDE>
constexpr int kBlocksPerSm = REV ? VQB_RS_REV_BLOCKS : (WIDE ? 2 : VQB_RS_FWD_BLOCKS);

template <bool REV, bool WIDE = true>
__global__ void __launch_bounds__(T, (kBlocksPerSm<REV, WIDE>))
    k_regstage(double2 *__restrict__ phi, double2 *__restrict__ psi,
               double *__restrict__ partial, const __grid_constant__ RParams P) {
    constexpr int NS = REV ? 2 : 1; // states per tile
    constexpr bool STAGED = kStaged<REV, WIDE>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // layout: diagonal tables | NS staging tiles (cp.async target) | relayout tile | slots
    double2 *stab = reinterpret_cast<double2 *>(smem_raw);
    double2 *stage_buf = stab + kMaxTab;
    double2 *xbuf = STAGED ? stage_buf + NS * TS : stage_buf;
    double *pacc = reinterpret_cast<double *>(xbuf + TS); // [nslots][NPART] (REV)
    // the stage's matrix pool, read with broadcast shared-memory loads
    double2 *spool = REV ? reinterpret_cast<double2 *>(pacc + kMaxSlots * NPART) : xbuf + TS;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    if (REV)
        for (int i = t; i < P.nslots * NPART; i += T) pacc[i] = 0;
    for (int i = t; i < P.ntab; i += T) stab[i] = P.tab[i];
    for (int i = t; i < P.npool; i += T) spool[i] = P.pool[i];
    __syncthreads();

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
    for (int b = 0; b < RB; ++b) nat_sw[b] = swz(T << b);
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
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(&stage_buf[q * TS + sl]);
                const double2 *src = (q == 0 ? phi : psi) + g;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    auto relayout = [&](double2 (&v)[R], const Addr &A, const Addr &B) {
#pragma unroll
        for (int i = 0; i < R; ++i) xbuf[slot(A, i)] = v[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = xbuf[slot(B, i)];
        __syncthreads();
    };

    unsigned long long tile = blockIdx.x;
    if (STAGED && tile < P.ntiles) prefetch(tile);
    for (; tile < P.ntiles; tile += gridDim.x) {
        const unsigned long long base = tile_base(tile);
        double2 vf[R], vg[REV ? R : 1];
        Addr A = layout_addr(P.subs[0].L, t);
        if constexpr (STAGED) {
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < R; ++i) vf[i] = stage_buf[slot(A, i)];
            if constexpr (REV) {
#pragma unroll
                for (int i = 0; i < R; ++i) vg[i] = stage_buf[TS + slot(A, i)];
            }
            __syncthreads(); // staging consumed: refill it with the next tile
            if (tile + gridDim.x < P.ntiles) prefetch(tile + gridDim.x);
        } else {
#pragma unroll
            for (int s = 0; s < R; ++s) {
                unsigned long long g = base | glo;
#pragma unroll
                for (int b = 0; b < RB; ++b)
                    if ((s >> b) & 1) g |= gh[b];
                vf[s] = phi[g];
            }
#pragma unroll
            for (int s = 0; s < R; ++s) {
                int sl = nat_st;
#pragma unroll
                for (int b = 0; b < RB; ++b)
                    if ((s >> b) & 1) sl ^= nat_sw[b];
                xbuf[sl] = vf[s];
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < R; ++i) vf[i] = xbuf[slot(A, i)];
            __syncthreads();
        }
        int cur = 0;
        for (int sub = 0; sub < P.nsubs; ++sub) {
            if (sub > 0) {
                const Addr B = layout_addr(P.subs[sub].L, t);
                relayout(vf, A, B);
                if constexpr (REV) relayout(vg, A, B);
                A = B;
                cur = sub;
            }
            const RSub &sb = P.subs[sub];
            int wnext = REV ? 0 : P.fast[sb.op_begin];
            for (int o = 0; o < sb.op_count; ++o) {
                if constexpr (!REV) {
                    const int w = wnext;
                    if (o + 1 < sb.op_count) wnext = P.fast[sb.op_begin + o + 1];
                    if (w) {
                        apply_fast(vf, spool, w);
                        continue;
                    }
                }
                const ROp &op = P.ops[sb.op_begin + o];
                int cuni = 0, cthr = 0;
                for (int q = 0; q < op.nc; ++q) {
                    if (op.ck[q] == 0) cuni |= (int)((base >> op.cp[q]) & 1) << q;
                    else if (op.ck[q] == 1) cthr |= ((t >> op.cp[q]) & 1) << q;
                }
                const int cbase = cuni | cthr;
                if constexpr (!REV) {
                    if (!WIDE || op.nt <= 2) {
                        dispatch<2, 2>(vf, op, spool, cbase, op.mat, op.ident);
                    } else if (op.nt == 3) {
                        smem_op<3>(vf, A, P.subs[sub].L, xbuf, op, spool, cuni, op.mat, op.ident, t,
                                   P.xpat);
                    } else {
                        smem_op<4>(vf, A, P.subs[sub].L, xbuf, op, spool, cuni, op.mat, op.ident, t,
                                   P.xpat);
                    }
                } else if (op.np == 0 && op.nt <= 2) {
                    dispatch<1, 2>(vf, op, spool, cbase, op.mat, op.ident);
                    dispatch<1, 2>(vg, op, spool, cbase, op.pair ? op.mat_psi : op.mat,
                                   op.pair ? op.ident_psi : op.ident);
                } else if (op.np == 0) {
                    const RLayout &Lc = P.subs[sub].L;
                    const unsigned mg = op.pair ? op.mat_psi : op.mat;
                    const unsigned long long ig = op.pair ? op.ident_psi : op.ident;
                    if (op.nt == 3) {
                        smem_op<3>(vf, A, Lc, xbuf, op, spool, cuni, op.mat, op.ident, t, P.xpat);
                        smem_op<3>(vg, A, Lc, xbuf, op, spool, cuni, mg, ig, t, P.xpat);
                    } else {
                        smem_op<4>(vf, A, Lc, xbuf, op, spool, cuni, op.mat, op.ident, t, P.xpat);
                        smem_op<4>(vg, A, Lc, xbuf, op, spool, cuni, mg, ig, t, P.xpat);
                    }
                } else {
                    double acc[VQB_MAX_PARAMS] = {0, 0, 0, 0, 0};
                    dispatch_param(vf, vg, op, spool, cbase, acc);
#pragma unroll
                    for (int p = 0; p < VQB_MAX_PARAMS; ++p) {
                        if (p >= op.np) break;
                        double x = acc[p];
                        // partial warp reduction: LANES_PER_PART lanes per partial
                        // sum, each partial slot owned by one lane (deterministic)
#pragma unroll
                        for (int sh = LANES_PER_PART / 2; sh > 0; sh >>= 1)
                            x += __shfl_down_sync(0xffffffffu, x, sh);
                        if ((lane & (LANES_PER_PART - 1)) == 0)
                            pacc[(op.slot + p) * NPART + warp * (32 / LANES_PER_PART) +
                                 lane / LANES_PER_PART] += x;
                    }
                }
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
            phi[g] = vf[i];
            if constexpr (REV) psi[g] = vg[i];
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    if constexpr (REV) {
        __syncthreads();
        for (int s = t; s < P.nslots; s += T) {
            double x = 0;
            for (int w = 0; w < NPART; ++w) x += pacc[s * NPART + w];
            partial[(size_t)blockIdx.x * P.partial_ld + P.slot_begin + s] = x;
        }
    }
}

// grads[dst] += sum over the slots of that destination (chained in slot order,
// slot_links) of scale[j] * (sum_b partial[b][j] + extra[j]), blocks in fixed
// order: one thread per destination, deterministic
__global__ void k_grads(const double *__restrict__ partial, int nblocks, int ld,
                        const double *__restrict__ scale, const long long *__restrict__ dst,
                        const long long *__restrict__ link, int ncols,
                        const double *__restrict__ extra, double *__restrict__ grads) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols || !(link[j] & 1)) return;
    double acc = 0;
    for (long long k = j; k >= 0; k = link[k] >> 1) {
        double v = 0;
        for (int b = 0; b < nblocks; ++b) v += partial[(size_t)b * ld + k];
        acc += scale[k] * (v + extra[k]);
    }
    grads[dst[j]] += acc;
}

// Specialised adjoint launches write one partial per (slot, tile); this sums a
// slot's row in fixed order (strided per thread, then a fixed tree):
// deterministic. One block per slot of the launch.
// Split over kSlotSplit blocks per slot (blockIdx.y), each summing a
// contiguous share of the row into split[slot][y]; k_slot_final adds the
// shares in fixed order. (One block per slot left most SMs idle: 0.45 ms per
// launch at 2^20 tiles.)
constexpr int kSlotSplit = 16;
__global__ void __launch_bounds__(256) k_slot_sums(const double *__restrict__ partial,
                                                   unsigned long long ntiles,
                                                   double *__restrict__ split) {
    __shared__ double sh[256];
    const double *row = partial + (size_t)blockIdx.x * ntiles;
    const unsigned long long per = (ntiles + gridDim.y - 1) / gridDim.y;
    const unsigned long long lo = per * blockIdx.y, hi = lo + per < ntiles ? lo + per : ntiles;
    double v = 0;
    for (unsigned long long i = lo + threadIdx.x; i < hi; i += 256) v += row[i];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) split[blockIdx.x * gridDim.y + blockIdx.y] = sh[0];
}
__global__ void k_slot_final(const double *__restrict__ split, int nslots, int nsplit,
                             double *__restrict__ out) {
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
        double x = 0;
        for (int y = 0; y < nsplit; ++y) x += split[s * nsplit + y];
        out[s] = x;
    }
}

// ---------------------------------------------------------------- host planning
int pair_code(int a, int b) { // a < b in [0,4)
    static const int code[4][4] = {{-1, 0, 1, 2}, {-1, -1, 3, 4}, {-1, -1, -1, 5}, {}};
    return code[a][b];
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

// thr[0..2] get distinct residues mod 3 (bank-conflict free under swz),
// preferring local bits 0,1,2 (coalesced stores).
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
    for (int r = 0; r < 3; ++r)
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

struct SlotMap {
    std::vector<double> scale;
    std::vector<long long> dst;
};

int env_int(const char *name, int dflt);

// Lower as much of a stage's block list as fits one parameter block.
// `remaining` (block indices, in a valid order) is consumed; what is left
// must run in a following launch with the same tile bits.
// Real scalar and rank-one form of one matrix of a channel step (D x D,
// column-major): M = c (1 + e J_R) up to rounding with J_R the all-ones matrix
// on the index set R (mask; |R| >= 2), or otherwise the real scalar that
// leaves the cheapest M / c (best_scale); c = 1: leave M alone.
struct PairForm {
    double c = 1.0;
    unsigned mask = 0;
    double e = 0.0;
};
PairForm pair_form(const cvec &M, int nt) {
    PairForm pf;
    const int D = 1 << nt;
    for (const cplx &v : M)
        if (v.imag() != 0.0 || v != v) return pf;
    auto at = [&](int r, int c) { return M[r + (size_t)c * D].real(); };
    unsigned rmask = 0; // indices coupled to another one
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c)
            if (r != c && at(r, c) != 0.0) rmask |= (1u << r) | (1u << c);
    bool ok = true;
    double c0 = 0, d = 0, e = 0;
    bool have_c = false, have_d = false, have_e = false;
    auto same = [](double x, double y) { return std::abs(x - y) <= 4e-16 * std::max(std::abs(x), std::abs(y)); };
    for (int r = 0; r < D && ok; ++r) {
        if (rmask >> r & 1) {
            if (!have_d) d = at(r, r), have_d = true;
            else ok = same(at(r, r), d);
            for (int c = 0; c < D && ok; ++c) {
                if (c == r || !(rmask >> c & 1)) continue;
                if (!have_e) e = at(r, c), have_e = true;
                else ok = same(at(r, c), e);
            }
        } else {
            if (!have_c) c0 = at(r, r), have_c = true;
            else ok = same(at(r, r), c0);
        }
    }
    if (ok && rmask == 0 && have_c && c0 != 0.0) { // c * identity
        pf.c = c0;
        return pf;
    }
    if (ok && have_d && have_e && __builtin_popcount(rmask) >= 2) {
        const double c = have_c ? c0 : d - e;
        if (c != 0.0 && std::abs(d - e - c) <= 1e-14 * std::abs(c)) {
            pf.c = c;
            pf.mask = rmask;
            pf.e = e / c;
            return pf;
        }
    }
    double cost = 0;
    const cplx sc = best_scale(M.data(), nt, 0, &cost);
    if (sc.imag() == 0.0 && sc.real() != 0.0) pf.c = sc.real();
    return pf;
}

void lower_stage_reg(const Stage &sg, const std::vector<const FusedOp *> &blocks,
                     std::vector<int> &remaining, int pn, bool rev, RParams &P, SlotMap &slots,
                     bool regwide = false, bool gdiff = false, bool factor = false) {
    // Scalar factoring (forward, specialised kernels): every register op's
    // matrices are divided by the scalar that makes the most entries exact
    // units (sqrt(X) = e^{i pi/4}/sqrt2 [[1, -i], [-i, 1]]: adds only; a
    // rotation diag(e^{-it/2}, e^{it/2}) = e^{-it/2} diag(1, e^{it}): half the
    // elements untouched); the scalars' product is applied once at the end
    // of the launch by one extra op (a 1x1 "diagonal" without conditions).
    // Results equal the unfactored product up to rounding.
    // Adjoint sweeps (same scalar on Phi and Psi, non-pair steps only): the
    // states run as true / c; a parametric step is factored only when its
    // contribution is taken before its update (derivative generator G_p),
    // and that contribution is rescaled by |c|^2 through its slot scale;
    // the launch ends with both states multiplied by c.
    // Channel steps (pair ops: S^-1 on Phi, S^dag on Psi) are factored per
    // state by real scalars ra (Phi) and rb (Psi): Phi runs as true / (c ra),
    // Psi as true / (c rb), later contributions are rescaled by |c|^2 ra rb.
    // A depolarizing superoperator and its inverse are c (1 + e J_R) with J_R
    // the all-ones matrix on the basis states R with equal ket and bra bits:
    // x_i += e * sum_R x for i in R, nothing else (rank_one below; flagged in
    // ROp::unit bits 2 (Phi) and 3 (Psi), R in ROp::slot, e at ROp::mat_d /
    // ROp::mat_e -- fields a non-parametric step does not otherwise use).
    cplx scale = 1.0;
    double ra = 1.0, rb = 1.0;
    const int ops_cap = factor ? kMaxOps - 1 : kMaxOps;
    const int pool_cap = factor ? kMaxPool - 2 : kMaxPool;
    std::memset(&P, 0, sizeof P);
    for (int j = 0; j < K; ++j) P.bits[j] = sg.bits[j];
    P.ntiles = 1ull << (pn - K);
    P.slot_begin = (int)slots.scale.size();
    auto local_of = [&](int g) {
        for (int j = 0; j < K; ++j)
            if (sg.bits[j] == g) return j;
        return -1;
    };
    // register bits an op needs: its mixing bits (wide ops run through the
    // shared-memory tile on any local bits and need none)
    auto wide_in_regs = [&](const FusedOp &f) { return regwide && f.nt >= 3 && f.nt <= RB; };
    auto mixmask = [&](const FusedOp &f) {
        unsigned mix = 0;
        if (f.nt >= 3 && !wide_in_regs(f)) return mix;
        for (int q = 0; q < f.nt; ++q) mix |= 1u << local_of(f.mix[q]);
        return mix;
    };
    auto count_x = [&](const FusedOp &f) { // XOR patterns of a wide op
        if (f.nt < 3) return 0;
        const int D = 1 << f.nt, dd = D * D;
        int nx = 0;
        for (int x = 0; x < D; ++x) {
            bool any = false;
            for (int c = 0; c < (1 << f.nc) && !any; ++c)
                for (int r = 0; r < D && !any; ++r)
                    any = f.sub_phi[size_t(c) * dd + r + size_t(r ^ x) * D] != cplx(0) ||
                          (f.pair && f.sub_psi[size_t(c) * dd + r + size_t(r ^ x) * D] != cplx(0));
            nx += any ? 1 : 0;
        }
        return nx;
    };
    auto pool_need = [&](const FusedOp &f) {
        if (f.nt >= 3) // XOR-term form: |X| * D entries per sub-matrix
            return (count_x(f) * (1 << f.nt) << f.nc) * (1 + (f.pair ? 1 : 0)) + 2;
        const int dd = (1 << (2 * f.nt)) << f.nc;
        return dd * (1 + (f.pair ? 1 : 0) + (rev ? f.np : 0)) + (rev && f.nt == 0 ? f.np << f.nc : 0) +
               2; // + rank-one coefficients
    };
    int nops = 0, npool = 0, nslots = 0;
    // (states below 2^22 amplitudes are host-bound: their relayouts are cheap
    // and the search's host time is not)
    const bool sub_search = env_int("VQB_SUB_SEARCH", pn >= 22 ? 1 : 0) != 0;
    // per-block figures the packing loops below read many times
    std::vector<unsigned> mix_of(blocks.size());
    std::vector<int> nx_of(blocks.size()), need_of(blocks.size());
    // Channel steps that run in rank-one form (both states of an adjoint pair
    // step, or a forward superoperator) read one coefficient each and no
    // matrix: their matrices and XOR patterns are left out of the parameter
    // block, which is what a launch's capacity is mostly spent on in the
    // density-matrix sweeps (130 pool entries per 2-qubit channel otherwise).
    // Such a launch has no interpreter form (ROp::unit bit 4).
    std::vector<char> r1_of(blocks.size(), 0);
    const bool r1_allowed = factor && env_int("VQB_JIT_PAIRFACTOR", 1) != 0 && env_int("VQB_JIT_RANKONE", 1) != 0 &&
                            env_int("VQB_JIT_R1_OMIT", 1) != 0;
    for (int i : remaining) {
        const FusedOp &f = *blocks[i];
        mix_of[i] = mixmask(f);
        nx_of[i] = count_x(f);
        need_of[i] = pool_need(f);
        if (!r1_allowed || f.np != 0 || f.nc != 0 || !(f.nt <= 2 || wide_in_regs(f))) continue;
        if (rev && f.pair && f.nt >= 1) {
            const PairForm a = pair_form(f.sub_phi, f.nt), b = pair_form(f.sub_psi, f.nt);
            r1_of[i] = a.mask && a.mask == b.mask;
        } else if (!rev && !f.pair && f.nt >= 2) {
            r1_of[i] = pair_form(f.sub_phi, f.nt).mask != 0;
        }
        if (r1_of[i]) {
            need_of[i] = 2;
            nx_of[i] = 0;
        }
    }
    while (!remaining.empty()) {
        if (P.nsubs >= kMaxSubs) break;
        unsigned rset = 0;
        uint64_t blocked = 0;
        std::vector<int> taken, deferred;
        int pool_used = 0, ops_used = 0, slots_used = 0, xp_used = 0;
        for (int i : remaining) {
            const FusedOp &f = *blocks[i];
            const unsigned mix = mix_of[i];
            const int nx = nx_of[i];
            const bool fits_res = nops + ops_used < ops_cap &&
                                  npool + pool_used + need_of[i] <= pool_cap &&
                                  nslots + slots_used + (rev ? f.np : 0) <= kMaxSlots &&
                                  P.nxpat + xp_used + nx <= 256;
            if ((f.support & blocked) || __builtin_popcount(rset | mix) > RB || !fits_res) {
                deferred.push_back(i);
                blocked |= f.support;
                continue;
            }
            rset |= mix;
            taken.push_back(i);
            pool_used += need_of[i];
            xp_used += nx;
            ++ops_used;
            slots_used += rev ? f.np : 0;
        }
        if (taken.empty()) break; // parameter block full: continue in the next launch
        for (int i : deferred) {
            const unsigned mix = mix_of[i];
            if (__builtin_popcount(rset | mix) <= RB) rset |= mix;
        }
        for (int j = K - 1; j >= 0 && __builtin_popcount(rset) < RB; --j) rset |= 1u << j;
        // Hill climbing on the register set, as the stage planner does on tiles:
        // swap one register bit for another tile bit while the sub-stage takes
        // more operations (every sub-stage saved is one relayout of the tile
        // through shared memory). VQB_SUB_SEARCH=0: first fit.
        if (sub_search) {
            auto pack = [&](unsigned rs, std::vector<int> *tk, std::vector<int> *df) {
                uint64_t bl = 0;
                int pool_u = 0, ops_u = 0, slots_u = 0, xp_u = 0, score = 0;
                for (int i : remaining) {
                    const FusedOp &f = *blocks[i];
                    const unsigned mix = mix_of[i];
                    const int nx = nx_of[i];
                    const bool fits_res = nops + ops_u < ops_cap && npool + pool_u + need_of[i] <= pool_cap &&
                                          nslots + slots_u + (rev ? f.np : 0) <= kMaxSlots &&
                                          P.nxpat + xp_u + nx <= 256;
                    if ((f.support & bl) || (mix & ~rs) || !fits_res) {
                        if (df) df->push_back(i);
                        bl |= f.support;
                        continue;
                    }
                    if (tk) tk->push_back(i);
                    pool_u += need_of[i];
                    xp_u += nx;
                    ++ops_u;
                    slots_u += rev ? f.np : 0;
                    score += mix ? 4 : 1;
                }
                return score;
            };
            int best = pack(rset, nullptr, nullptr);
            for (int iter = 0; iter < 6; ++iter) {
                unsigned best_rs = rset;
                for (int bo = 0; bo < K; ++bo) {
                    if (!(rset >> bo & 1)) continue;
                    for (int bi = 0; bi < K; ++bi) {
                        if (rset >> bi & 1) continue;
                        const unsigned rs = (rset & ~(1u << bo)) | (1u << bi);
                        const int sc = pack(rs, nullptr, nullptr);
                        if (sc > best) {
                            best = sc;
                            best_rs = rs;
                        }
                    }
                }
                if (best_rs == rset) break;
                rset = best_rs;
            }
            taken.clear();
            deferred.clear();
            pack(rset, &taken, &deferred);
            if (taken.empty()) break;
        }
        RSub &sb = P.subs[P.nsubs++];
        {
            int nr = 0;
            std::vector<int> free_bits;
            for (int j = 0; j < K; ++j) {
                if (rset >> j & 1) sb.L.reg[nr++] = j;
                else free_bits.push_back(j);
            }
            choose_threads(sb.L, free_bits);
        }
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
            const FusedOp &f = *blocks[i];
            ROp &o = P.ops[nops++];
            o.nt = f.nt;
            o.nc = f.nc;
            o.np = rev ? f.np : 0;
            o.pair = f.pair ? 1 : 0;
            // register ops: matrix bits permuted to ascending register order;
            // wide ops keep their own bit order with local bits in o.lb
            int rp[kMaxMix] = {0, 0, 0, 0}, order[kMaxMix] = {0, 1, 2, 3};
            if (f.nt <= 2) {
                for (int q = 0; q < f.nt; ++q) rp[q] = reg_of(local_of(f.mix[q]));
                if (f.nt == 2 && rp[1] < rp[0]) std::swap(order[0], order[1]);
                if (f.nt == 1) o.code = rp[0];
                if (f.nt == 2) o.code = pair_code(rp[order[0]], rp[order[1]]);
            } else if (wide_in_regs(f)) {
                o.inreg = 1;
                for (int q = 0; q < f.nt; ++q) o.lb[q] = reg_of(local_of(f.mix[q]));
            } else {
                for (int q = 0; q < f.nt; ++q) o.lb[q] = local_of(f.mix[q]);
            }
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
            cplx scale_before = scale; // Phi and Psi computed = true / scale before this op
            // Derivative generators: the contribution Re<psi|D_p inv phi>
            // can be taken before the update with G_p = D_p inv; for
            // rotations G_p is a scaled Pauli (dRx inv = -i X / 2), for
            // superoperator steps a diagonal -- much sparser than D_p.
            // Store whichever has fewer nonzero real/imaginary parts
            // (ROp::unit bit 1 marks G; specialised kernels only).
            bool use_g = false;
            cvec G;
            if (o.np > 0 && gdiff && f.nt >= 1 && f.nt <= 2 && !f.pair) {
                const int nsubm = 1 << f.nc;
                G.assign(f.sub_d.size(), cplx(0));
                auto weight = [](const cplx &x) { return (x.real() != 0.0) + (x.imag() != 0.0); };
                int wd = 0, wg = 0;
                for (int p = 0; p < f.np; ++p)
                    for (int c = 0; c < nsubm; ++c) {
                        const cplx *Dm = f.sub_d.data() + ((size_t(p) << f.nc) + c) * dd;
                        const cplx *U = f.sub_phi.data() + size_t(c) * dd;
                        cplx *Gm = G.data() + ((size_t(p) << f.nc) + c) * dd;
                        for (int col = 0; col < D; ++col)
                            for (int row = 0; row < D; ++row) {
                                cplx acc = 0;
                                for (int k2 = 0; k2 < D; ++k2) acc += Dm[row + k2 * D] * U[k2 + col * D];
                                // entries at rounding level of an exact zero are zero
                                if (std::abs(acc.real()) < 1e-15 * 4) acc.real(0.0);
                                if (std::abs(acc.imag()) < 1e-15 * 4) acc.imag(0.0);
                                Gm[row + col * D] = acc;
                                wg += weight(acc);
                                wd += weight(Dm[row + col * D]);
                            }
                    }
                use_g = wg < wd;
            }
            // push 2^nc sub-matrices of `src` (permuted to ascending register
            // order); returns the pool offset and the identity mask
            auto push = [&](const cvec &src, size_t first_block, unsigned long long *ident) {
                const unsigned off = (unsigned)npool;
                for (int c = 0; c < (1 << f.nc); ++c) {
                    const cvec sub(src.begin() + (first_block + c) * dd,
                                   src.begin() + (first_block + c + 1) * dd);
                    const cvec pm = f.nt > 1 ? permute_matrix(sub, f.nt, order) : sub;
                    bool id = true;
                    for (int r = 0; r < D; ++r)
                        for (int s = 0; s < D; ++s)
                            if (pm[r + s * D] != (r == s ? cplx(1) : cplx(0))) id = false;
                    if (ident && id) *ident |= 1ull << c;
                    for (const auto &x : pm) P.pool[npool++] = make_double2(x.real(), x.imag());
                }
                return off;
            };
            // channel steps: per-state real scalars and the rank-one form
            // (detected on the matrices in the op's final bit order)
            cvec pair_phi, pair_psi;
            const cvec *src_phi = &f.sub_phi, *src_psi = &f.sub_psi;
            PairForm fa, fb;
            if (factor && rev && f.pair && f.np == 0 && f.nc == 0 && f.nt >= 1 &&
                (f.nt <= 2 || wide_in_regs(f)) && env_int("VQB_JIT_PAIRFACTOR", 1) != 0) {
                fa = pair_form(f.nt > 1 ? permute_matrix(f.sub_phi, f.nt, order) : f.sub_phi, f.nt);
                fb = pair_form(f.nt > 1 ? permute_matrix(f.sub_psi, f.nt, order) : f.sub_psi, f.nt);
                pair_phi = f.sub_phi;
                pair_psi = f.sub_psi;
                if (fa.c != 1.0) divide_by(pair_phi.data(), pair_phi.size(), cplx(fa.c));
                if (fb.c != 1.0) divide_by(pair_psi.data(), pair_psi.size(), cplx(fb.c));
                ra *= fa.c;
                rb *= fb.c;
                src_phi = &pair_phi;
                src_psi = &pair_psi;
                if (fa.mask && fb.mask && fa.mask != fb.mask) fb.mask = 0;
                if (env_int("VQB_JIT_RANKONE", 1) == 0) fa.mask = fb.mask = 0;
                if (fa.mask) o.unit |= 4;
                if (fb.mask) o.unit |= 8;
                o.slot = (int)(fa.mask ? fa.mask : fb.mask);
            }
            // forward channel superoperators (non-parametric, no conditions): the
            // same scalar / rank-one form, the scalar joins the launch's product
            bool fwd_form = false;
            if (factor && !rev && !f.pair && f.np == 0 && f.nc == 0 && f.nt >= 2 &&
                (f.nt <= 2 || wide_in_regs(f)) && env_int("VQB_JIT_PAIRFACTOR", 1) != 0) {
                fa = pair_form(f.nt > 1 ? permute_matrix(f.sub_phi, f.nt, order) : f.sub_phi, f.nt);
                // register ops keep best_scale's (possibly complex) scalar unless
                // the rank-one form applies; wide ops had no factoring at all
                if (fa.mask || f.nt >= 3) {
                    pair_phi = f.sub_phi;
                    if (fa.c != 1.0) divide_by(pair_phi.data(), pair_phi.size(), cplx(fa.c));
                    scale *= fa.c;
                    src_phi = &pair_phi;
                    if (env_int("VQB_JIT_RANKONE", 1) == 0) fa.mask = 0;
                    if (fa.mask) {
                        o.unit |= 4;
                        o.slot = (int)fa.mask;
                    }
                    fwd_form = true;
                }
            }
            const bool omit = r1_of[i] && (o.unit & 4) && (!f.pair || (o.unit & 8));
            if (omit) {
                o.unit |= 16; // rank-one form only: no matrices in the block
                o.xoff = P.nxpat;
                o.nx = 0;
            } else if (f.nt >= 3) {
                // wide ops run in smem_op as sum_k diag(d_k) P_{x_k}: store the
                // XOR patterns x_k and, per sub-matrix, d_k[r] = S[r, r ^ x_k]
                auto permuted = [&](const cvec &src, int c) {
                    const cvec sub(src.begin() + size_t(c) * dd, src.begin() + size_t(c + 1) * dd);
                    return permute_matrix(sub, f.nt, order);
                };
                std::vector<int> X;
                auto scan = [&](const cvec &src) {
                    for (int c = 0; c < (1 << f.nc); ++c) {
                        const cvec pm = permuted(src, c);
                        for (int x = 0; x < D; ++x) {
                            if (std::find(X.begin(), X.end(), x) != X.end()) continue;
                            for (int r = 0; r < D; ++r)
                                if (pm[r + size_t(r ^ x) * D] != cplx(0)) {
                                    X.push_back(x);
                                    break;
                                }
                        }
                    }
                };
                scan(*src_phi);
                if (f.pair) scan(*src_psi);
                std::sort(X.begin(), X.end());
                o.xoff = P.nxpat;
                o.nx = (int)X.size();
                for (int x : X) P.xpat[P.nxpat++] = (unsigned char)x;
                auto pushx = [&](const cvec &src, unsigned long long *ident) {
                    const unsigned off = (unsigned)npool;
                    for (int c = 0; c < (1 << f.nc); ++c) {
                        const cvec pm = permuted(src, c);
                        bool id = true;
                        for (int r = 0; r < D; ++r)
                            for (int s = 0; s < D; ++s)
                                if (pm[r + s * D] != (r == s ? cplx(1) : cplx(0))) id = false;
                        if (id) *ident |= 1ull << c;
                        for (int x : X)
                            for (int r = 0; r < D; ++r) {
                                const cplx v = pm[r + size_t(r ^ x) * D];
                                P.pool[npool++] = make_double2(v.real(), v.imag());
                            }
                    }
                    return off;
                };
                o.mat = pushx(*src_phi, &o.ident);
                if (f.pair) o.mat_psi = pushx(*src_psi, &o.ident_psi);
            } else if (fwd_form) {
                o.mat = push(*src_phi, 0, &o.ident);
            } else if (factor && !f.pair && (!rev || f.np == 0 || use_g)) {
                cvec sub = f.sub_phi;
                double c = 0;
                const cplx sc = best_scale(sub.data(), f.nt, f.nc, &c);
                scale_before = scale;
                if (sc != cplx(1)) {
                    divide_by(sub.data(), sub.size(), sc);
                    scale *= sc;
                }
                o.mat = push(sub, 0, &o.ident);
            } else {
                o.mat = push(*src_phi, 0, &o.ident);
                if (f.pair) o.mat_psi = push(*src_psi, 0, &o.ident_psi);
            }
            if (o.unit & (4 | 8)) {
                // rank-one coefficients e (Phi at mat_d, Psi at mat_e)
                o.mat_d = (unsigned)npool;
                P.pool[npool++] = make_double2(fa.e, 0.0);
                o.mat_e = (unsigned)npool;
                P.pool[npool++] = make_double2(fb.e, 0.0);
            }
            if (rev && f.nt == 0 && !f.pair) {
                o.unit = 1;
                for (int c = 0; c < (1 << f.nc); ++c)
                    if (std::abs(std::abs(f.sub_phi[c]) - 1.0) > 1e-13) o.unit = 0;
            }
            if (o.np > 0) {
                o.mat_d = (unsigned)npool;
                if (use_g) o.unit |= 2;
                for (int p = 0; p < f.np; ++p) push(use_g ? G : f.sub_d, size_t(p) << f.nc, nullptr);
                if (f.nt == 0) {
                    o.mat_e = (unsigned)npool;
                    for (int p = 0; p < f.np; ++p)
                        for (int c = 0; c < (1 << f.nc); ++c) {
                            cplx e = f.sub_d[(size_t(p) << f.nc) + c] * f.sub_phi[c];
                            // parts at rounding level of an exact zero are zero (a
                            // rotation's e is -i/2 times a sign: imaginary)
                            if (std::abs(e.real()) < 4e-15) e.real(0.0);
                            if (std::abs(e.imag()) < 4e-15) e.imag(0.0);
                            P.pool[npool++] = make_double2(e.real(), e.imag());
                        }
                }
                o.ident = 0;
                o.slot = nslots;
                // contributions of the scaled states: <psi/c|G|phi/c> = |1/c|^2 <psi|G|phi>
                const double corr = std::norm(scale_before) * ra * rb;
                for (int p = 0; p < f.np; ++p) {
                    slots.scale.push_back(f.scale * corr);
                    slots.dst.push_back(f.grad_base + p);
                }
                nslots += f.np;
            }
            // per-register-bit condition masks
            for (int q = 0; q < f.nc; ++q)
                if (o.ck[q] == 2) o.rw[o.cp[q]] |= 1 << q;
            // forward fast path (see RParams::fast)
            P.fast[nops - 1] = 0;
            if (!rev && f.nc == 0 && !f.pair && (f.nt == 1 || f.nt == 2) && o.ident == 0 &&
                o.mat < (1u << 27))
                P.fast[nops - 1] = (int)(o.mat << 4) | (f.nt == 1 ? 1 + o.code : 5 + o.code);
            // diagonal steps with register-bit conditions read their tables
            // from shared memory (phi table, [D table for a parametric step])
            o.tab = o.tab_psi = -1;
            const int nsub = 1 << f.nc;
            auto push_tab = [&](const cvec &src, size_t first) {
                const int off = P.ntab;
                for (int c = 0; c < nsub; ++c)
                    P.tab[P.ntab++] = make_double2(src[first + c].real(), src[first + c].imag());
                return off;
            };
            if (f.nt == 0 && o.per_group) {
                const int need = nsub * (1 + (f.pair ? 1 : 0) + (o.np == 1 ? 1 : 0));
                if (P.ntab + need <= kMaxTab && o.np <= 1) {
                    o.tab = push_tab(f.sub_phi, 0);
                    if (o.np == 1) push_tab(f.sub_d, 0); // at o.tab + nsub
                    if (f.pair) o.tab_psi = push_tab(f.sub_psi, 0);
                }
            }
        }
        sb.op_count = nops - sb.op_begin;
        remaining.swap(deferred);
    }
    if (factor && (scale != cplx(1) || ra != 1.0 || rb != 1.0) && P.nsubs > 0) {
        // the factored scalars, once per amplitude, in the last sub-stage
        ROp &o = P.ops[nops++];
        o.tab = o.tab_psi = -1;
        o.mat = (unsigned)npool;
        const cplx sa = scale * ra, sb2 = scale * rb;
        P.pool[npool++] = make_double2(sa.real(), sa.imag());
        if (ra != rb) {
            o.pair = 1;
            o.mat_psi = (unsigned)npool;
            P.pool[npool++] = make_double2(sb2.real(), sb2.imag());
        }
        P.fast[nops - 1] = 0;
        ++P.subs[P.nsubs - 1].op_count;
    }
    P.nslots = nslots;
    P.npool = npool;
}


int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// dynamic shared memory: tables | staging | relayout tile | slots (REV) or
// the matrix pool (forward, npool entries)
template <bool REV, bool WIDE = true> size_t smem_bytes(int npool = kMaxPool) {
    const int staging = kStaged<REV, WIDE> ? (REV ? 2 : 1) : 0;
    return (size_t)kMaxTab * sizeof(double2) + (size_t)(staging + 1) * TS * sizeof(double2) +
           (REV ? kMaxSlots * NPART * 8 : 0) + (size_t)npool * sizeof(double2);
}

// resident blocks (grid = SMs x blocks per SM) for a launch with `smem` bytes
template <bool REV, bool WIDE> int grid_size(unsigned long long ntiles, size_t smem) {
    static int nsm = -1;
    static int per_sm[64] = {}; // by smem in KiB
    if (nsm < 0) {
        int dev = 0;
        VQB_CUDA(cudaGetDevice(&dev));
        VQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        VQB_CUDA(cudaFuncSetAttribute(k_regstage<REV, WIDE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem_bytes<REV, WIDE>()));
    }
    const size_t kib = std::min<size_t>((smem + 1023) / 1024, 63);
    if (per_sm[kib] == 0) {
        int b = 0;
        VQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_regstage<REV, WIDE>, T,
                                                               kib * 1024));
        per_sm[kib] = std::max(b, 1);
    }
    return (int)std::min<unsigned long long>((unsigned long long)nsm * per_sm[kib], ntiles);
}



// Lanes per warp that keep a partial sum of a gradient slot (the rest of the
// warp reduction happens in the block's final sum): VQB_JIT_REDLANES (1, 2,
// 4, 8); measured best 4 for 8-register adjoints (QAOA 578 -> 556 ms), 2 for
// 16-register ones (noisy 915 -> 898 ms).
int red_lanes_of() {
    int v = env_int("VQB_JIT_REDLANES", R >= 16 ? 2 : 4);
    return v >= 8 ? 8 : v >= 4 ? 4 : v >= 2 ? 2 : 1;
}

// ---------------------------------------------------------------- structure-aware emission
// The specialised kernels read matrix values at run time, but which entries
// are exactly zero, purely real or purely imaginary is structure: channel
// superoperators are real and sparse (a depolarizing channel is
// (1-p) I + p * trace-and-replace), rotations about X/Y and their derivatives
// have purely real / imaginary entries, controlled blocks are mostly zero.
// That class (bit 0: some real part nonzero, bit 1: some imaginary part
// nonzero, over every sub-matrix the code may select) is part of the kernel
// key, and each term is emitted with only the FMAs its class needs. Dropped
// terms are exact zeros, so the result equals the dense product (up to the
// sign of zero).
int pool_cls(const RParams &P, unsigned off, int count, int stride) {
    int c = 0;
    for (int k = 0; k < count; ++k) {
        const double2 v = P.pool[off + (unsigned)(k * stride)];
        if (v.x != 0.0 || v.x != v.x) c |= 1;
        if (v.y != 0.0 || v.y != v.y) c |= 2;
    }
    return c;
}

// pool_cls extended by the unit classes of entry_class (4: +1, 5: -1, 6: +i,
// 7: -i) when every selected entry is the same unit: those terms are adds
// (or plain copies as a row's first term), no multiplications
int pool_ucls(const RParams &P, unsigned off, int count, int stride) {
    int u = -1;
    for (int k = 0; k < count; ++k) {
        const double2 v = P.pool[off + (unsigned)(k * stride)];
        const int c = entry_class(cplx(v.x, v.y));
        if (c < 4 || (u >= 0 && u != c)) return pool_cls(P, off, count, stride);
        u = c;
    }
    return u < 0 ? 0 : u;
}
// class of a term that may take either of two entries (a run-time choice)
int merge_cls(int a, int b) {
    if (a == b) return a;
    auto bits = [](int c) { return c < 4 ? c : (c <= 5 ? 1 : 2); };
    return bits(a) | bits(b);
}

// acc (=|+=) m * x for an entry of class cls; adds the FP64 flops per thread
std::string cterm(const std::string &m, const std::string &x, const std::string &acc, int cls, bool first,
                  double &fl) {
    switch (cls) {
    case 0:
        return "";
    case 1:
        fl += 4;
        return first ? "        " + acc + " = make_double2(" + m + ".x * " + x + ".x, " + m + ".x * " + x + ".y);\n"
                     : "        " + acc + ".x = fma(" + m + ".x, " + x + ".x, " + acc + ".x); " + acc + ".y = fma(" + m +
                           ".x, " + x + ".y, " + acc + ".y);\n";
    case 2:
        fl += 4;
        return first ? "        " + acc + " = make_double2(-" + m + ".y * " + x + ".y, " + m + ".y * " + x + ".x);\n"
                     : "        " + acc + ".x = fma(-" + m + ".y, " + x + ".y, " + acc + ".x); " + acc + ".y = fma(" +
                           m + ".y, " + x + ".x, " + acc + ".y);\n";
    case 4: // +1
        if (first) return "        " + acc + " = " + x + ";\n";
        fl += 2;
        return "        " + acc + ".x += " + x + ".x; " + acc + ".y += " + x + ".y;\n";
    case 5: // -1
        if (first) return "        " + acc + " = make_double2(-" + x + ".x, -" + x + ".y);\n";
        fl += 2;
        return "        " + acc + ".x -= " + x + ".x; " + acc + ".y -= " + x + ".y;\n";
    case 6: // +i
        if (first) return "        " + acc + " = make_double2(-" + x + ".y, " + x + ".x);\n";
        fl += 2;
        return "        " + acc + ".x -= " + x + ".y; " + acc + ".y += " + x + ".x;\n";
    case 7: // -i
        if (first) return "        " + acc + " = make_double2(" + x + ".y, -" + x + ".x);\n";
        fl += 2;
        return "        " + acc + ".x += " + x + ".y; " + acc + ".y -= " + x + ".x;\n";
    default:
        fl += 8;
        return first ? "        " + acc + " = cmul(" + m + ", " + x + ");\n"
                     : "        " + acc + " = cfma(" + m + ", " + x + ", " + acc + ");\n";
    }
}

// v[idx[r]] <- sum_s M[r + s D] v[idx[s]] for one group; M entry k is the
// expression mat(k) of class cls(k)
// a row's terms in emission order: a unit entry first (as the first term it
// is a plain copy), then the others in column order
template <typename ClsF> void term_order(int r, int D, ClsF cls, int *order) {
    int n = 0;
    for (int s = 0; s < D; ++s)
        if (cls(r + s * D) >= 4) {
            order[n++] = s;
            break;
        }
    for (int s = 0; s < D; ++s)
        if (n == 0 || order[0] != s) order[n++] = s;
}

template <typename MatF, typename ClsF>
std::string mv_code(const std::string &v, const int *idx, int D, MatF mat, ClsF cls, double &fl) {
    std::string e = "      {\n";
    for (int s = 0; s < D; ++s)
        e += "        const double2 x" + std::to_string(s) + " = " + v + "[" + std::to_string(idx[s]) + "];\n";
    for (int r = 0; r < D; ++r) {
        e += "        double2 o" + std::to_string(r) + ";\n";
        bool first = true;
        int order[16];
        term_order(r, D, cls, order);
        for (int oi = 0; oi < D; ++oi) {
            const int s = order[oi];
            const int c = cls(r + s * D);
            if (!c) continue;
            e += cterm(mat(r + s * D), "x" + std::to_string(s), "o" + std::to_string(r), c, first, fl);
            first = false;
        }
        if (first) e += "        o" + std::to_string(r) + " = make_double2(0.0, 0.0);\n";
    }
    for (int r = 0; r < D; ++r)
        e += "        " + v + "[" + std::to_string(idx[r]) + "] = o" + std::to_string(r) + ";\n";
    return e + "      }\n";
}

// acc += Re <vg | Dm | vf> over one group (dot_group with structure)
template <typename MatF, typename ClsF>
std::string dot_code(const std::string &acc, const int *idx, int D, MatF mat, ClsF cls, double &fl) {
    std::string e = "      {\n        double a = 0.0;\n";
    bool any = false;
    for (int r = 0; r < D; ++r) {
        std::string row;
        bool first = true;
        int order[16];
        term_order(r, D, cls, order);
        for (int oi = 0; oi < D; ++oi) {
            const int s = order[oi];
            const int c = cls(r + s * D);
            if (!c) continue;
            row += cterm(mat(r + s * D), "vf[" + std::to_string(idx[s]) + "]", "y", c, first, fl);
            first = false;
        }
        if (first) continue;
        any = true;
        fl += 4;
        e += "        {\n          double2 y;\n" + row + "          a += re_cj(vg[" + std::to_string(idx[r]) +
             "], y);\n        }\n";
    }
    if (!any) return "";
    return e + "        " + acc + " += a;\n      }\n";
}

// Factored derivative contraction. The entries of a derivative matrix come in
// few distinct values up to a unit factor: G_p = D_p inv of a rotation is
// -i/2 times a Pauli matrix (one value), D_p of Rx is {-s/2, -i c/2}. With
// the entries partitioned into classes {u_k * m_c} (u_k in {1, -1, i, -i}),
//   Re <psi| D |phi> = sum_c Re(m_c * w_c),  w_c = sum_k u_k conj(psi_r) phi_s,
// so each entry costs two FMAs per needed component of w_c (only Re w_c for a
// real m_c, only Im w_c for an imaginary one) straight into a per-thread
// accumulator, and the products with m_c are taken once per thread and step
// instead of once per row. The partition is structure (part of the kernel
// key, dot_signature); the values m_c stay launch parameters.
struct DotPlan {
    bool ok = false;
    int nclass = 0;
    int ref[4] = {0, 0, 0, 0};  // reference entry of each class
    int need[4] = {0, 0, 0, 0}; // bit 0: Re w needed (m has a real part), bit 1: Im w
    int cls_of[16];             // class of entry k, -1: zero
    int unit_of[16];            // u_k: 0: 1, 1: -1, 2: i, 3: -i
};
// u with v == u * r exactly, or -1
int unit_ratio(double2 v, double2 r) {
    if (v.x == r.x && v.y == r.y) return 0;
    if (v.x == -r.x && v.y == -r.y) return 1;
    if (v.x == -r.y && v.y == r.x) return 2;
    if (v.x == r.y && v.y == -r.x) return 3;
    return -1;
}
// plan over the sub-matrices `sel` (pool offset off, dd entries each) one
// thread may select at run time
DotPlan dot_plan(const RParams &P, unsigned off, int dd, const std::vector<int> &sel) {
    DotPlan pl;
    if (dd > 16) return pl;
    auto val = [&](int cc, int k) { return P.pool[off + (unsigned)(cc * dd + k)]; };
    auto nz = [](double2 v) { return v.x != 0.0 || v.y != 0.0 || v.x != v.x || v.y != v.y; };
    int first = -1;
    for (int cc : sel) {
        for (int k = 0; k < dd && first < 0; ++k)
            if (nz(val(cc, k))) first = cc;
        if (first >= 0) break;
    }
    if (first < 0) return pl;
    for (int k = 0; k < dd; ++k) {
        pl.cls_of[k] = -1;
        pl.unit_of[k] = 0;
        const double2 v = val(first, k);
        if (v.x != v.x || v.y != v.y) return pl;
        if (!nz(v)) continue;
        for (int c = 0; c < pl.nclass && pl.cls_of[k] < 0; ++c) {
            const int u = unit_ratio(v, val(first, pl.ref[c]));
            if (u >= 0) {
                pl.cls_of[k] = c;
                pl.unit_of[k] = u;
            }
        }
        if (pl.cls_of[k] < 0) {
            if (pl.nclass == 4) return pl;
            pl.ref[pl.nclass] = k;
            pl.cls_of[k] = pl.nclass++;
        }
    }
    for (int cc : sel) {
        bool any = false;
        for (int k = 0; k < dd; ++k) any = any || nz(val(cc, k));
        if (!any) continue; // a zero sub-matrix contributes m_c = 0
        for (int k = 0; k < dd; ++k) {
            const double2 v = val(cc, k);
            if (pl.cls_of[k] < 0) {
                if (nz(v)) return pl;
                continue;
            }
            if (unit_ratio(v, val(cc, pl.ref[pl.cls_of[k]])) != pl.unit_of[k]) return pl;
        }
        for (int c = 0; c < pl.nclass; ++c) {
            const double2 m = val(cc, pl.ref[c]);
            if (m.x != 0.0) pl.need[c] |= 1;
            if (m.y != 0.0) pl.need[c] |= 2;
        }
    }
    pl.ok = true;
    return pl;
}
std::string dot_plan_sig(const DotPlan &pl, int dd) {
    if (!pl.ok) return "-";
    std::string s;
    for (int k = 0; k < dd; ++k) s += (char)('a' + (pl.cls_of[k] < 0 ? 0 : 1 + pl.cls_of[k] * 4 + pl.unit_of[k]));
    for (int c = 0; c < pl.nclass; ++c) s += (char)('0' + pl.need[c]);
    return s;
}
// sub-matrices selectable by a thread whose register-bit conditions are cs
std::vector<int> dot_selectable(const ROp &op, int cs) {
    int rmask = 0;
    bool dynamic = false;
    for (int q = 0; q < op.nc; ++q) {
        if (op.ck[q] == 2) rmask |= 1 << q;
        else dynamic = true;
    }
    std::vector<int> sel;
    for (int cc = 0; cc < (1 << op.nc); ++cc)
        if (dynamic ? (cc & rmask) == cs : cc == cs) sel.push_back(cc);
    return sel;
}
// matrices the contraction of a parametric step uses: D_p (with the updated
// Phi), G_p (ROp::unit bit 1, old Phi), or for a unit-modulus diagonal step
// the table e_p = D_p M at mat_e (old Phi: conj(psi) phi is invariant under
// the step, autodiff contribution Re(conj(psi) e phi))
unsigned dot_base(const ROp &op) { return op.nt == 0 && (op.unit & 1) ? op.mat_e : op.mat_d; }

// every plan a parametric 0..2-bit step's code depends on (kernel key)
std::string dot_signature(const RParams &P, const ROp &op) {
    if (op.np <= 0 || op.nt >= 3) return "";
    const int dd = 1 << (2 * op.nt), nsub = 1 << op.nc;
    int rmask = 0;
    for (int q = 0; q < op.nc; ++q)
        if (op.ck[q] == 2) rmask |= 1 << q;
    std::string s;
    for (int p = 0; p < op.np; ++p)
        for (int cs = 0; cs < nsub; ++cs) {
            if (cs & ~rmask) continue;
            s += dot_plan_sig(dot_plan(P, dot_base(op) + (unsigned)(p * nsub * dd), dd, dot_selectable(op, cs)), dd);
            s += ';';
        }
    return s;
}
// one group's terms: w_c (+)= u_k conj(vg[idx[r]]) vf[idx[s]], needed components only
std::string dot_plan_group(const DotPlan &pl, const std::string &wname, const int *idx, int D, double &fl) {
    std::string e;
    for (int s = 0; s < D; ++s)
        for (int r = 0; r < D; ++r) {
            const int k = r + s * D, c = pl.cls_of[k];
            if (c < 0) continue;
            const std::string g = "vg[" + std::to_string(idx[r]) + "]", f = "vf[" + std::to_string(idx[s]) + "]";
            const std::string wr = wname + "r" + std::to_string(c), wi = wname + "i" + std::to_string(c);
            // q = conj(g) f: qr = g.x f.x + g.y f.y, qi = g.x f.y - g.y f.x
            auto add_qr = [&](const std::string &w, bool neg) {
                const std::string sg = neg ? "-" : "";
                e += "        " + w + " = fma(" + sg + g + ".x, " + f + ".x, fma(" + sg + g + ".y, " + f + ".y, " + w + "));\n";
                fl += 4;
            };
            auto add_qi = [&](const std::string &w, bool neg) {
                const std::string sa = neg ? "-" : "", sb = neg ? "" : "-";
                e += "        " + w + " = fma(" + sa + g + ".x, " + f + ".y, fma(" + sb + g + ".y, " + f + ".x, " + w + "));\n";
                fl += 4;
            };
            const int u = pl.unit_of[k];
            if (pl.need[c] & 1) { // Re(u q)
                if (u == 0) add_qr(wr, false);
                else if (u == 1) add_qr(wr, true);
                else if (u == 2) add_qi(wr, true);
                else add_qi(wr, false);
            }
            if (pl.need[c] & 2) { // Im(u q)
                if (u == 0) add_qi(wi, false);
                else if (u == 1) add_qi(wi, true);
                else if (u == 2) add_qr(wi, false);
                else add_qr(wi, true);
            }
        }
    return e;
}

// v[i] += e * sum_{j in R} v[j] for i in R (real e): the rank-one form of a
// depolarizing superoperator (or its inverse) after its scalar is factored
std::string rank_one_code(const std::string &v, const int *ridx, int nr, const std::string &e, double &fl) {
    auto el = [&](int k) { return v + "[" + std::to_string(ridx[k]) + "]"; };
    std::string c = "      {\n        double2 tsum = " + el(0) + ";\n";
    for (int k = 1; k < nr; ++k) {
        c += "        tsum.x += " + el(k) + ".x; tsum.y += " + el(k) + ".y;\n";
        fl += 2;
    }
    for (int k = 0; k < nr; ++k) {
        c += "        " + el(k) + ".x = fma(" + e + ".x, tsum.x, " + el(k) + ".x); " + el(k) + ".y = fma(" + e +
             ".x, tsum.y, " + el(k) + ".y);\n";
        fl += 4;
    }
    return c + "      }\n";
}

// register indices of the matrix rows of group i (Pos<NT, P0, P1>::off)
void group_idx(int nt, int code, int i, int *idx) {
    static const int p0[6] = {0, 0, 0, 1, 1, 2}, p1[6] = {1, 2, 3, 2, 3, 3};
    const int P0 = nt == 1 ? code : p0[code], P1 = nt == 2 ? p1[code] : 0;
    for (int r = 0; r < (1 << nt); ++r)
        idx[r] = i | ((r & 1) ? 1 << P0 : 0) | ((nt > 1 && (r & 2)) ? 1 << P1 : 0);
}

// ---------------------------------------------------------------- specialisation
// Specialised code for a wide (nt >= 3) operation of sub-stage `sub` on the
// register state `v`: through the shared-memory tile as sum_k diag(d_k)
// P_{x_k} (smem_op), with the mixing bits, XOR patterns and slot offsets as
// literals. Matrices come from the shared-memory pool copy (spool).
struct WideState {
    const char *v;   // register array
    const char *buf; // shared-memory tile it goes through
    unsigned mat;
    unsigned long long ident;
};
// One wide operation applied to one or two register states (the adjoint's Phi
// and Psi, each with its own matrices): the states go through their own
// shared-memory tiles in one round trip, and the groups of all states are
// spread over the block's threads. Matrices come from the shared-memory pool
// copy (*needs_spool).
std::string jit_wide_op(const RParams &P, int sub, const ROp &op, const std::vector<WideState> &sts,
                        const char *slot_base, double *wide_fl, bool *needs_spool, bool inplace = false,
                        bool param_ok = false) {
    auto I = [](long long x) { return std::to_string(x); };
    const RLayout &L = P.subs[sub].L;
    const int NT = std::min(std::max(op.nt, 1), kMaxMix), D = 1 << NT;
    const int G = TS >> NT, S = (int)sts.size();
    auto slot_const = [&](int i) {
        int c = 0;
        for (int b = 0; b < RB; ++b)
            if ((i >> b) & 1) c ^= swz(1 << L.reg[b]);
        return c;
    };
    int sorted[kMaxMix];
    for (int q = 0; q < NT; ++q) sorted[q] = op.lb[q];
    std::sort(sorted, sorted + NT);
    int sw_off[16];
    for (int r = 0; r < D; ++r) {
        int o = 0;
        for (int q = 0; q < NT; ++q)
            if ((r >> q) & 1) o |= 1 << op.lb[q];
        sw_off[r] = swz(o);
    }
    // conditioned matrices come from the shared-memory pool copy (run-time
    // sub-matrix index); unconditioned ones are parameter-bank operands at
    // literal offsets where the caller allows it (forward kernels; adjoint
    // pools outgrow the constant cache)
    const bool cond = op.nc > 0 || !param_ok;
    if (cond) *needs_spool = true;
    std::string e = "    {\n";
    if (!inplace) {
        for (const auto &st : sts)
            for (int i = 0; i < R; ++i)
                e += std::string("      ") + st.buf + "[" + slot_base + " ^ " + I(slot_const(i)) + "] = " + st.v +
                     "[" + I(i) + "];\n";
        e += "      __syncthreads();\n";
    }
    e += "      const int cu = 0";
    for (int q = 0; q < op.nc; ++q)
        if (op.ck[q] == 0) e += " | (int)(((base >> " + I(op.cp[q]) + ") & 1) << " + I(q) + ")";
    e += ";\n      for (int w = threadIdx.x; w < " + I(S * G) + "; w += " + I(T) + ") {\n";
    for (int si = 0; si < S; ++si) {
        const WideState &st = sts[si];
        if (S > 1) e += si == 0 ? "       if (w < " + I(G) + ") {\n        int b = w;\n"
                                : "       } else {\n        int b = w - " + I(G) + ";\n";
        else e += "       {\n        int b = w;\n";
        for (int q = 0; q < NT; ++q)
            e += "        b = ((b >> " + I(sorted[q]) + ") << " + I(sorted[q] + 1) + ") | (b & " +
                 I((1 << sorted[q]) - 1) + ");\n";
        e += "        const int c = cu";
        for (int q = 0; q < op.nc; ++q) {
            const int l = op.ck[q] == 1 ? L.thr[op.cp[q]] : (op.ck[q] == 2 ? L.reg[op.cp[q]] : -1);
            if (l >= 0) e += " | (((b >> " + I(l) + ") & 1) << " + I(q) + ")";
        }
        e += ";\n";
        if (st.ident) e += "        if ((" + std::to_string(st.ident) + "ull >> c) & 1) continue;\n";
        if (cond) e += "        const double2 *M = spool + " + I(st.mat) + " + c * " + I(op.nx * D) + ";\n";
        auto Mk = [&](int k) {
            return cond ? "M[" + I(k) + "]" : "P.pool[" + I(st.mat + (unsigned)k) + "]";
        };
        e += "        const int sb = swz(b);\n";
        // per-entry structure over every selectable sub-matrix (pool_cls)
        const int nsubm = 1 << op.nc;
        double fl = 0;
        for (int r = 0; r < D; ++r) {
            bool first = true;
            e += "        double2 o" + I(r) + ";\n";
            for (int k = 0; k < op.nx; ++k) {
                const int x = P.xpat[op.xoff + k];
                const int c = pool_cls(P, st.mat + (unsigned)(k * D + r), nsubm, op.nx * D);
                if (!c) continue;
                e += cterm(Mk(k * D + r), std::string(st.buf) + "[sb ^ " + I(sw_off[r ^ x]) + "]",
                           "o" + I(r), c, first, fl);
                first = false;
            }
            if (first) e += "        o" + I(r) + " = make_double2(0.0, 0.0);\n";
        }
        *wide_fl += fl * G; // per tile
        for (int r = 0; r < D; ++r) e += "        " + std::string(st.buf) + "[sb ^ " + I(sw_off[r]) + "] = o" + I(r) + ";\n";
    }
    e += "       }\n      }\n      __syncthreads();\n";
    if (!inplace) {
        for (const auto &st : sts)
            for (int i = 0; i < R; ++i)
                e += std::string("      ") + st.v + "[" + I(i) + "] = " + st.buf + "[" + slot_base + " ^ " +
                     I(slot_const(i)) + "];\n";
        e += "      __syncthreads();\n";
    }
    e += "    }\n";
    return e;
}

// Relayout of register arrays from layout A to B by warp shuffles, when B is
// A with some register bits exchanged for lane bits (stable layouts): per
// exchanged pair (register bit p, lane bit q) and register pair (i, i | 1<<p),
// lane value l keeps one element and receives the other from lane ^ (1<<q).
// Returns "" when B is not reachable that way (warp bits or other moves).
std::string shuffle_relayout(const RLayout &A, const RLayout &B, const std::vector<std::string> &vs) {
    std::vector<std::pair<int, int>> swaps; // (register position p, lane bit q)
    RLayout C = A;
    for (int p = 0; p < RB; ++p) {
        if (A.reg[p] == B.reg[p]) continue;
        int q = -1;
        for (int b = 0; b < TB; ++b)
            if (A.thr[b] == B.reg[p]) q = b;
        if (q < 0 || q >= 5 || B.thr[q] != A.reg[p]) return "";
        swaps.push_back({p, q});
        C.reg[p] = B.reg[p];
        C.thr[q] = A.reg[p];
    }
    for (int b = 0; b < TB; ++b)
        if (C.thr[b] != B.thr[b]) return "";
    if (swaps.empty()) return " ";
    std::string e = "    {\n";
    for (auto [p, q] : swaps) {
        e += "      {\n        const bool l = (threadIdx.x >> " + std::to_string(q) + ") & 1;\n";
        for (const auto &v : vs)
            for (int i = 0; i < R; ++i) {
                if ((i >> p) & 1) continue;
                const int j = i | (1 << p);
                const std::string vi = v + "[" + std::to_string(i) + "]", vj = v + "[" + std::to_string(j) + "]";
                e += "        { const double2 s = l ? " + vi + " : " + vj +
                     "; const double2 r = make_double2(__shfl_xor_sync(0xffffffffu, s.x, " + std::to_string(1 << q) +
                     "), __shfl_xor_sync(0xffffffffu, s.y, " + std::to_string(1 << q) + ")); if (l) " + vi +
                     " = r; else " + vj + " = r; }\n";
            }
        e += "      }\n";
    }
    return e + "    }\n";
}

// A wide operation on register bits (ROp::inreg): out[r] = sum_k d_k[r]
// v[r ^ x_k] per group of registers, XOR-term pool, register conditions
// resolved per group, run-time ones (cd) select the sub-matrix. `mexpr(off)`
// gives a pool entry expression at a literal offset (static sub-matrix) and
// `dyn` is the run-time condition-index expression ("" if none).
template <typename MExpr>
std::string jit_wide_regs(const RParams &P, const ROp &op, const char *v, unsigned mat, unsigned long long ident,
                          const std::string &dyn, MExpr mexpr, double &fl) {
    auto I = [](long long x) { return std::to_string(x); };
    const int NT = op.nt, D = 1 << NT, stride = op.nx * D;
    int rmask = 0;
    for (int q = 0; q < NT; ++q) rmask |= 1 << op.lb[q];
    auto regidx = [&](int i0, int r) {
        int x = i0;
        for (int q = 0; q < NT; ++q)
            if ((r >> q) & 1) x |= 1 << op.lb[q];
        return x;
    };
    std::string e;
    for (int i0 = 0; i0 < R; ++i0) {
        if (i0 & rmask) continue;
        int cs = 0, rq = 0;
        for (int q = 0; q < op.nc; ++q) {
            if (op.ck[q] == 2) {
                rq |= 1 << q;
                if ((i0 >> op.cp[q]) & 1) cs |= 1 << q;
            }
        }
        if (dyn.empty() && ((ident >> cs) & 1)) continue;
        e += "      {\n";
        if (!dyn.empty())
            e += "        const int cw = " + dyn + " | " + I(cs) + ";\n        if (!((" + std::to_string(ident) +
                 "ull >> cw) & 1)) {\n";
        for (int r = 0; r < D; ++r) e += "        const double2 x" + I(r) + " = " + v + "[" + I(regidx(i0, r)) + "];\n";
        for (int r = 0; r < D; ++r) {
            bool first = true;
            e += "        double2 o" + I(r) + ";\n";
            for (int k = 0; k < op.nx; ++k) {
                const int x = P.xpat[op.xoff + k];
                int c = 0;
                for (int cc = 0; cc < (1 << op.nc); ++cc)
                    if (dyn.empty() ? cc == cs : (cc & rq) == cs)
                        c |= pool_cls(P, mat + (unsigned)(cc * stride + k * D + r), 1, 0);
                if (!c) continue;
                const std::string m = dyn.empty() ? mexpr(mat + (unsigned)(cs * stride + k * D + r))
                                                  : "spool[" + I(mat + (unsigned)(k * D + r)) + " + cw * " + I(stride) + "]";
                e += cterm(m, "x" + I(r ^ x), "o" + I(r), c, first, fl);
                first = false;
            }
            if (first) e += "        o" + I(r) + " = make_double2(0.0, 0.0);\n";
        }
        for (int r = 0; r < D; ++r) e += "        " + std::string(v) + "[" + I(regidx(i0, r)) + "] = o" + I(r) + ";\n";
        if (!dyn.empty()) e += "        }\n";
        e += "      }\n";
    }
    return e;
}

// One-tile-per-block kernels read run-time-indexed matrices (sub-matrices
// selected by conditions on thread or global bits) straight from the
// parameter bank: the constant cache serialises a warp's read only over the
// distinct addresses (at most 2^k for k thread-bit conditions; one for
// global-bit conditions, which are block-uniform), whereas copying the pool
// into shared memory in every block cost a fifth of the QAOA adjoint's stall
// samples (profiles/r2_ncu_qaoa_rev.txt). Kernels with a tile loop keep the
// shared-memory copy (parameter-bank operands would be hoisted out of the
// loop into registers and spill). VQB_JIT_PBANK=0 restores the copy.
bool pool_reads_from_bank(std::string &body) {
    if (env_int("VQB_JIT_PBANK", 1) == 0) return false;
    auto replace_all = [&](const std::string &a, const std::string &b) {
        for (size_t pos = 0; (pos = body.find(a, pos)) != std::string::npos; pos += b.size()) body.replace(pos, a.size(), b);
    };
    replace_all("spool[", "P.pool[");
    replace_all("spool + ", "P.pool + ");
    return true;
}

std::string jit_forward_source_rs16(const RParams &P, bool *uses_spool, bool *per_block, double *flops);
// Source of a kernel equivalent to k_regstage<false, false> on one lowered
// stage program, with every structural quantity a literal: tile bits, layouts
// (shared-memory slot XOR constants), register positions, condition bits,
// identity masks and matrix offsets. Matrices are read from the kernel's
// parameter block at constant offsets; sub-matrices selected by thread or
// tile bits come from a shared-memory copy. Returns "" for programs the
// generator does not cover (wide operations).
std::string jit_forward_source(const RParams &P, bool *uses_spool, bool *per_block, double *flops) {
    if constexpr (RB != 4) return "";
    else return jit_forward_source_rs16(P, uses_spool, per_block, flops);
}

std::string jit_forward_source_rs16(const RParams &P, bool *uses_spool, bool *per_block, double *flops) {
    std::string src;
    auto out = [&](const std::string &x) { src += x; };
    auto num = [](unsigned long long v) { return std::to_string(v) + "ull"; };
    auto thread_expr = [&](const int *lbits, bool global) {
        // sum_b ((t >> b) & 1) << pos(b), pos = local bit or its global bit
        std::string e = "(0";
        for (int b = 0; b < TB; ++b) {
            const int pos = global ? P.bits[lbits[b]] : lbits[b];
            e += " | (" + std::string(global ? "(u64)" : "") + "((t >> " + std::to_string(b) +
                 ") & 1) << " + std::to_string(pos) + ")";
        }
        return e + ")";
    };
    auto slot_const = [&](const RLayout &L, int i) {
        int c = 0;
        for (int b = 0; b < RB; ++b)
            if ((i >> b) & 1) c ^= swz(1 << L.reg[b]);
        return c;
    };
    bool spool = false;
    // where statically indexed matrices are read from: the parameter bank
    // (uniform-register operands; the compiler hoists them) or the
    // shared-memory copy (VQB_JIT_POOL=smem)
    const char *pool_env = std::getenv("VQB_JIT_POOL");
    const bool pool_smem = pool_env && std::strcmp(pool_env, "smem") == 0;
    const std::string MP = pool_smem ? "spool" : "P.pool";
    const int jit_blocks = env_int("VQB_JIT_BLOCKS", TB >= 8 ? 2 : 4);
    const char *mode_env = std::getenv("VQB_JIT_MODE");
    const bool per_block_mode = !(mode_env && std::strcmp(mode_env, "persistent") == 0);
    std::string body;
    auto emit = [&](const std::string &x) { body += x; };
    static const int pair_p0[6] = {0, 0, 0, 1, 1, 2}, pair_p1[6] = {1, 2, 3, 2, 3, 3};
    double fl = 0, wfl = 0; // FP64 flops per thread (register code) / per wide-op group
    // lazy residency (as in the adjoint generator): the tile is in registers
    // in the layout of cur_sub, or in xbuf in tile-index space; wide ops work
    // on xbuf in place, so they share the round trip of a neighbouring
    // relayout. The one-tile-per-block prologue leaves the tile in xbuf.
    // VQB_JIT_DIRECT: the one-tile-per-block prologue loads straight into the
    // first sub-stage's layout (lanes 0-2 on the tile's low bits keep the
    // loads in full sectors) instead of through the shared-memory tile
    const bool direct = per_block_mode && env_int("VQB_JIT_DIRECT", 1) != 0;
    bool in_smem = per_block_mode && !direct;
    int cur_sub = per_block_mode && !direct ? -1 : 0;
    auto to_smem = [&]() {
        if (in_smem) return;
        for (int i = 0; i < R; ++i)
            emit("    xbuf[st" + std::to_string(cur_sub) + " ^ " + std::to_string(slot_const(P.subs[cur_sub].L, i)) +
                 "] = v[" + std::to_string(i) + "];\n");
        emit("    __syncthreads();\n");
        in_smem = true;
    };
    const bool shuffles = env_int("VQB_JIT_SHUFFLE", 1) != 0;
    auto to_regs = [&](int sub) {
        if (!in_smem && cur_sub == sub) return;
        if (!in_smem && shuffles) {
            const std::string sh = shuffle_relayout(P.subs[cur_sub].L, P.subs[sub].L, {"v"});
            if (!sh.empty()) {
                emit(sh);
                cur_sub = sub;
                return;
            }
        }
        to_smem();
        for (int i = 0; i < R; ++i)
            emit("    v[" + std::to_string(i) + "] = xbuf[st" + std::to_string(sub) + " ^ " +
                 std::to_string(slot_const(P.subs[sub].L, i)) + "];\n");
        emit("    __syncthreads();\n");
        in_smem = false;
        cur_sub = sub;
    };
    const bool lazy = env_int("VQB_JIT_LAZY", 1) != 0;
    const bool dotplan_on = env_int("VQB_JIT_DOTPLAN", 1) != 0;
    for (int sub = 0; sub < P.nsubs; ++sub) {
        const RSub &sb = P.subs[sub];
        if (!lazy) to_regs(sub);
        for (int k = 0; k < sb.op_count; ++k) {
            const ROp &op = P.ops[sb.op_begin + k];
            if (op.nt >= 3 && op.inreg) {
                to_regs(sub);
                std::string dyn;
                for (int q = 0; q < op.nc; ++q) {
                    if (op.ck[q] == 0)
                        dyn += " | (int)(((base >> " + std::to_string(op.cp[q]) + ") & 1) << " + std::to_string(q) + ")";
                    else if (op.ck[q] == 1)
                        dyn += " | (((t >> " + std::to_string(op.cp[q]) + ") & 1) << " + std::to_string(q) + ")";
                }
                if (!dyn.empty()) {
                    dyn = "(0" + dyn + ")";
                    spool = true;
                }
                if (dyn.empty() && (op.unit & 4)) { // rank-one form (channel superoperators)
                    if (op.ident & 1) continue;
                    int rm = 0;
                    for (int q = 0; q < op.nt; ++q) rm |= 1 << op.lb[q];
                    for (int i0 = 0; i0 < R; ++i0) {
                        if (i0 & rm) continue;
                        int ridx[16], nr = 0;
                        for (int r = 0; r < (1 << op.nt); ++r) {
                            if (!((op.slot >> r) & 1)) continue;
                            int x = i0;
                            for (int q = 0; q < op.nt; ++q)
                                if ((r >> q) & 1) x |= 1 << op.lb[q];
                            ridx[nr++] = x;
                        }
                        emit(rank_one_code("v", ridx, nr, MP + "[" + std::to_string(op.mat_d) + "]", fl));
                    }
                    continue;
                }
                emit(jit_wide_regs(P, op, "v", op.mat, op.ident, dyn,
                                   [&](unsigned off) { return MP + "[" + std::to_string(off) + "]"; }, fl));
                continue;
            }
            if (op.nt >= 3) {
                to_smem();
                emit(jit_wide_op(P, sub, op, {{"v", "xbuf", op.mat, op.ident}}, ("st" + std::to_string(sub)).c_str(),
                                 &wfl, &spool, true, true));
                if (!lazy) to_regs(sub);
                continue;
            }
            to_regs(sub);
            {
                // a run of diagonal operations (they commute): each one's
                // element depends on register element i only through the
                // register bits among its conditions (mask m, usually none or
                // one bit), so it multiplies one of 2^|m| per-thread phase
                // products PH_m[g]; every element gets its product once at
                // the end of the run
                int run_end = k;
                while (run_end < sb.op_count && P.ops[sb.op_begin + run_end].nt == 0) ++run_end;
                if (run_end - k >= 2 && env_int("VQB_JIT_DIAGRUN", 1)) {
                    auto I = [](long long x) { return std::to_string(x); };
                    auto rmask_of = [&](const ROp &o) {
                        int m = 0;
                        for (int q = 0; q < o.nc; ++q)
                            if (o.ck[q] == 2) m |= 1 << o.cp[q];
                        return m;
                    };
                    auto extract = [](int i, int m) {
                        int g = 0, k2 = 0;
                        for (int b = 0; b < RB; ++b)
                            if ((m >> b) & 1) g |= ((i >> b) & 1) << k2++;
                        return g;
                    };
                    std::vector<int> masks;
                    for (int j = k; j < run_end; ++j) {
                        const int m = rmask_of(P.ops[sb.op_begin + j]);
                        if (std::find(masks.begin(), masks.end(), m) == masks.end()) masks.push_back(m);
                    }
                    emit("    {\n");
                    for (int m : masks)
                        for (int g = 0; g < (1 << __builtin_popcount(m)); ++g)
                            emit("      double2 PH" + I(m) + "_" + I(g) + ";\n");
                    std::map<std::pair<int, int>, bool> ph_set;
                    for (int j = k; j < run_end; ++j) {
                        const ROp &oj = P.ops[sb.op_begin + j];
                        std::string dynx;
                        int rmq = 0;
                        for (int q = 0; q < oj.nc; ++q) {
                            if (oj.ck[q] == 0)
                                dynx += " | (int)(((base >> " + I(oj.cp[q]) + ") & 1) << " + I(q) + ")";
                            else if (oj.ck[q] == 1)
                                dynx += " | (((t >> " + I(oj.cp[q]) + ") & 1) << " + I(q) + ")";
                            else
                                rmq |= 1 << q;
                        }
                        const bool dynj = !dynx.empty();
                        if (dynj) spool = true;
                        const int m = rmask_of(oj);
                        emit("      {\n");
                        if (dynj) emit("        const int cd = 0" + dynx + ";\n");
                        for (int g = 0; g < (1 << __builtin_popcount(m)); ++g) {
                            int cs = 0, k2 = 0, full = 0;
                            for (int b = 0; b < RB; ++b)
                                if ((m >> b) & 1) full |= ((g >> k2++) & 1) << b;
                            for (int q = 0; q < oj.nc; ++q)
                                if (oj.ck[q] == 2 && ((full >> oj.cp[q]) & 1)) cs |= 1 << q;
                            if (!dynj && ((oj.ident >> cs) & 1)) continue;
                            const std::string mm = dynj ? "spool[" + I(oj.mat) + " + (cd | " + I(cs) + ")]"
                                                        : MP + "[" + I(oj.mat + (unsigned)cs) + "]";
                            int c = 0;
                            for (int cc = 0; cc < (1 << oj.nc); ++cc)
                                if (dynj ? (cc & rmq) == cs : cc == cs) c |= pool_cls(P, oj.mat + (unsigned)cc, 1, 0);
                            const std::string PHg = "PH" + I(m) + "_" + I(g);
                            bool &set = ph_set[{m, g}];
                            if (!set) {
                                emit("        " + PHg + " = " + mm + ";\n");
                                set = true;
                            } else if (c == 1) {
                                emit("        " + PHg + ".x *= " + mm + ".x; " + PHg + ".y *= " + mm + ".x;\n");
                                fl += 2;
                            } else if (c == 2) {
                                emit("        " + PHg + " = make_double2(-" + mm + ".y * " + PHg + ".y, " + mm + ".y * " +
                                     PHg + ".x);\n");
                                fl += 2;
                            } else if (c == 0) {
                                emit("        " + PHg + " = make_double2(0.0, 0.0);\n");
                            } else {
                                emit("        " + PHg + " = cmul(" + mm + ", " + PHg + ");\n");
                                fl += 6;
                            }
                        }
                        emit("      }\n");
                    }
                    for (int i = 0; i < R; ++i) {
                        std::string ph;
                        for (int m : masks) {
                            const int g = extract(i, m);
                            if (!ph_set[{m, g}]) continue;
                            const std::string t2 = "PH" + I(m) + "_" + I(g);
                            if (ph.empty()) ph = t2;
                            else {
                                ph = "cmul(" + t2 + ", " + ph + ")";
                                fl += 6;
                            }
                        }
                        if (ph.empty()) continue;
                        emit("      v[" + I(i) + "] = cmul(" + ph + ", v[" + I(i) + "]);\n");
                        fl += 6;
                    }
                    emit("    }\n");
                    k = run_end - 1;
                    continue;
                }
            }
            const int dd = 1 << (2 * op.nt);
            std::string dyn;
            for (int q = 0; q < op.nc; ++q) {
                if (op.ck[q] == 0)
                    dyn += " | (int)(((base >> " + std::to_string(op.cp[q]) + ") & 1) << " +
                           std::to_string(q) + ")";
                else if (op.ck[q] == 1)
                    dyn += " | (((t >> " + std::to_string(op.cp[q]) + ") & 1) << " + std::to_string(q) + ")";
            }
            auto cstat = [&](int i) {
                int c = 0;
                for (int q = 0; q < op.nc; ++q)
                    if (op.ck[q] == 2 && ((i >> op.cp[q]) & 1)) c |= 1 << q;
                return c;
            };
            std::string tmpl;
            int mask = 0;
            if (op.nt == 1) {
                tmpl = "1, " + std::to_string(op.code) + ", 0, " + std::to_string(R);
                mask = 1 << op.code;
            } else if (op.nt == 2) {
                tmpl = "2, " + std::to_string(pair_p0[op.code]) + ", " + std::to_string(pair_p1[op.code]) + ", " +
                       std::to_string(R);
                mask = (1 << pair_p0[op.code]) | (1 << pair_p1[op.code]);
            }
            const std::string ident = num(op.ident);
            // register-condition bits are fixed per group; the others select
            // the sub-matrix at run time (class = union over those)
            int rmask = 0;
            for (int q = 0; q < op.nc; ++q)
                if (op.ck[q] == 2) rmask |= 1 << q;
            auto ecls = [&](unsigned off, int cs, int k) {
                int c = -1;
                for (int cc = 0; cc < (1 << op.nc); ++cc)
                    if ((cc & rmask) == cs) {
                        const int e = pool_ucls(P, off + (unsigned)(cc * dd + k), 1, 0);
                        c = c < 0 ? e : merge_cls(c, e);
                    }
                return c < 0 ? 0 : c;
            };
            const int D = 1 << op.nt;
            if (dyn.empty()) {
                for (int i = 0; i < R; ++i) {
                    if (i & mask) continue;
                    const int c = cstat(i);
                    if ((op.ident >> c) & 1) continue;
                    int idx[4];
                    group_idx(op.nt, op.code, i, idx);
                    if (op.unit & 4) { // rank-one form (channel superoperators)
                        int ridx[16], nr = 0;
                        for (int r = 0; r < D; ++r)
                            if ((op.slot >> r) & 1) ridx[nr++] = idx[r];
                        emit(rank_one_code("v", ridx, nr, MP + "[" + std::to_string(op.mat_d) + "]", fl));
                        continue;
                    }
                    const unsigned base_off = op.mat + (unsigned)(c * dd);
                    emit(mv_code(
                        "v", idx, D, [&](int k) { return MP + "[" + std::to_string(base_off + (unsigned)k) + "]"; },
                        [&](int k) { return pool_ucls(P, base_off + (unsigned)k, 1, 0); }, fl));
                }
                continue;
            }
            spool = true;
            emit("    {\n      const int cd = 0" + dyn + ";\n");
            for (int i = 0; i < R; ++i) {
                if (i & mask) continue;
                const int cs = cstat(i);
                const std::string c = "(cd | " + std::to_string(cs) + ")";
                int idx[4];
                group_idx(op.nt, op.code, i, idx);
                emit("      if (!((" + ident + " >> " + c + ") & 1)) {\n        const double2 *M = spool + " +
                     std::to_string(op.mat) + " + " + c + " * " + std::to_string(dd) + ";\n");
                emit(mv_code(
                    "v", idx, D, [&](int k) { return "M[" + std::to_string(k) + "]"; },
                    [&](int k) { return ecls(op.mat, cs, k); }, fl));
                emit("      }\n");
            }
            emit("    }\n");
        }
    }
    to_regs(P.nsubs - 1);
    const RLayout &Lf = P.subs[P.nsubs - 1].L;
    out("#include \"jit_rt.cuh\"\nusing namespace vqbjit;\n");
    out("struct JP { double2 pool[" + std::to_string(std::max(P.npool, 1)) + "]; };\n");
    out("extern \"C\" __global__ void __launch_bounds__(" + std::to_string(T) + ", " + std::to_string(jit_blocks) + ")\n"
        "vqb_stage(double2 *__restrict__ a, const __grid_constant__ JP P) {\n");
    out(per_block_mode ? "  extern __shared__ __align__(16) double2 sm[];\n  double2 *xbuf = sm;\n"
                       : "  extern __shared__ __align__(16) double2 sm[];\n"
                         "  double2 *stage = sm, *xbuf = sm + " + std::to_string(TS) + ";\n");
    // matrices are read from a shared-memory copy at constant offsets: loads
    // the compiler cannot hoist out of the tile loop (parameter-bank reads
    // would be hoisted into registers and spill)
    if (spool && per_block_mode && !pool_smem && pool_reads_from_bank(body)) spool = false;
    spool = spool || pool_smem;
    if (spool)
        out(std::string("  double2 *spool = sm + ") + std::to_string(per_block_mode ? TS : 2 * TS) +
            ";\n  for (int i = threadIdx.x; i < " + std::to_string(P.npool) +
            "; i += " + std::to_string(T) + ") spool[i] = P.pool[i];\n  __syncthreads();\n");
    out("  const int t = threadIdx.x;\n");
    int nat_local[TB];
    for (int b = 0; b < TB; ++b) nat_local[b] = b;
    out("  const u64 glo = " + thread_expr(nat_local, true) + ";\n");
    // thread-dependent slot bases are recomputed per tile from an opaque copy
    // of t (cheap integer work) instead of being hoisted into registers
    auto opaque_t = [](const char *name) {
        return std::string("int ") + name + "; asm volatile(\"mov.b32 %0, %1;\" : \"=r\"(" + name +
               ") : \"r\"(t));\n";
    };
    out("  const u64 gfin = " + thread_expr(Lf.thr, true) + ";\n");
    out("  const u64 NT = " + num(P.ntiles) + ";\n");
    out("  auto base_of = [&](u64 c) -> u64 {\n");
    for (int j = 0; j < K; ++j) {
        const int sb = P.bits[j];
        out("    c = ((c >> " + std::to_string(sb) + ") << " + std::to_string(sb + 1) + ") | (c & " +
            num((1ull << sb) - 1) + ");\n");
    }
    out("    return c;\n  };\n");
    // per-layout slot bases, with t seen through an opaque copy (so they are
    // recomputed per tile instead of being hoisted into registers)
    std::string slot_bases = "    " + opaque_t("to");
    for (int sub = 0; sub < P.nsubs; ++sub) {
        std::string x = thread_expr(P.subs[sub].L.thr, false);
        for (size_t pos; (pos = x.find("(t >>")) != std::string::npos;) x.replace(pos, 5, "(to >>");
        slot_bases += "    const int st" + std::to_string(sub) + " = swz" + x + ";\n";
    }
    auto natural = [&](int s2, unsigned long long *g, int *sl) {
        *g = 0;
        *sl = 0;
        for (int b = 0; b < RB; ++b)
            if ((s2 >> b) & 1) {
                *g |= 1ull << P.bits[TB + b];
                *sl ^= swz(T << b);
            }
    };
    if (per_block_mode) {
        // one tile per block: coalesced loads straight into registers, one
        // relayout to the first layout; other resident blocks cover latency
        out("  {\n    const u64 tile = blockIdx.x;\n    const u64 base = base_of(tile);\n    double2 v[" + std::to_string(R) + "];\n");
        if (direct) {
            const RLayout &L0 = P.subs[0].L;
            out("    const u64 g0 = " + thread_expr(L0.thr, true) + ";\n");
            for (int i = 0; i < R; ++i) {
                unsigned long long g = 0;
                for (int b = 0; b < RB; ++b)
                    if ((i >> b) & 1) g |= 1ull << P.bits[L0.reg[b]];
                out("    v[" + std::to_string(i) + "] = a[base | g0 | " + num(g) + "];\n");
            }
            out(slot_bases);
        }
        for (int s2 = 0; s2 < R && !direct; ++s2) {
            unsigned long long g;
            int sl;
            natural(s2, &g, &sl);
            out("    v[" + std::to_string(s2) + "] = a[base | glo | " + num(g) + "];\n");
        }
        if (!direct) out(slot_bases + "    const int nat_st = swz(to);\n");
        for (int s2 = 0; s2 < R && !direct; ++s2) {
            unsigned long long g;
            int sl;
            natural(s2, &g, &sl);
            out("    xbuf[nat_st ^ " + std::to_string(sl) + "] = v[" + std::to_string(s2) + "];\n");
        }
        if (!direct) out("    __syncthreads();\n"); // the body starts with the tile in xbuf (lazy residency)
    } else {
        out("  auto prefetch = [&](u64 tile) {\n    const u64 b = base_of(tile) | glo;\n    " + opaque_t("tn") +
            "    const int nat_st = swz(tn);\n");
        for (int s2 = 0; s2 < R; ++s2) {
            unsigned long long g;
            int sl;
            natural(s2, &g, &sl);
            out("    cp_async16(&stage[nat_st ^ " + std::to_string(sl) + "], a + (b | " + num(g) + "));\n");
        }
        out("    cp_async_commit();\n  };\n");
        out("  u64 tile = blockIdx.x;\n  if (tile < NT) prefetch(tile);\n"
            "  for (; tile < NT; tile += gridDim.x) {\n    const u64 base = base_of(tile);\n"
            "    cp_async_wait_all();\n    __syncthreads();\n    double2 v[" + std::to_string(R) + "];\n");
        out(slot_bases);
        for (int i = 0; i < R; ++i)
            out("    v[" + std::to_string(i) + "] = stage[st0 ^ " + std::to_string(slot_const(P.subs[0].L, i)) + "];\n");
        out("    __syncthreads();\n    if (tile + gridDim.x < NT) prefetch(tile + gridDim.x);\n");
    }
    out(body);
    for (int i = 0; i < R; ++i) {
        unsigned long long g = 0;
        for (int b = 0; b < RB; ++b)
            if ((i >> b) & 1) g |= 1ull << P.bits[Lf.reg[b]];
        out("    a[base | gfin | " + num(g) + "] = v[" + std::to_string(i) + "];\n");
    }
    out(per_block_mode ? "  }\n}\n" : "  }\n  cp_async_wait_all();\n}\n");
    if (uses_spool) *uses_spool = spool;
    if (per_block) *per_block = per_block_mode;
    if (flops) *flops = (fl * T + wfl) / TS; // executed FP64 flops per amplitude
    return src;
}


// VQB_JIT_CHECK=1 (debugging aid, stands in for compute-sanitizer, which
// this pool does not allow): every global index of the generated kernel is
// checked against the state size (2^pn amplitudes) and every shared-memory
// tile / pool index against its array, trapping on a violation (the call
// then fails with a CUDA error). Applied to the finished source text.
std::string instrument_checks(const std::string &src, int pn, int tile, int npool) {
    if (env_int("VQB_JIT_CHECK", 0) == 0) return src;
    std::string out;
    out.reserve(src.size() * 2);
    const std::string pre = "#define VQB_GCHK(x) vqbjit::chk_idx((u64)(x), " + std::to_string(1ull << pn) +
                            "ull)\n#define VQB_SCHK(x) ((int)vqbjit::chk_idx((u64)(x), " + std::to_string(tile) +
                            "ull))\n#define VQB_PCHK(x) ((int)vqbjit::chk_idx((u64)(x), " + std::to_string(npool) +
                            "ull))\n";
    size_t i = 0;
    const size_t inc = src.find("using namespace vqbjit;");
    auto wrap_at = [&](size_t pos, size_t open, const char *mac) {
        // copy through `open` ('['), wrap the balanced index expression
        out.append(src, i, open + 1 - i);
        int depth = 1;
        size_t j = open + 1;
        while (j < src.size() && depth > 0) {
            if (src[j] == '[') ++depth;
            else if (src[j] == ']') --depth;
            ++j;
        }
        out += std::string(mac) + "(" + src.substr(open + 1, j - 1 - (open + 1)) + ")]";
        i = j;
        (void)pos;
    };
    while (i < src.size()) {
        size_t best = std::string::npos, open = 0;
        const char *mac = nullptr;
        for (const auto &pm : {std::make_pair("a[", "VQB_GCHK"), std::make_pair("b2[", "VQB_GCHK"),
                               std::make_pair("xbuf[", "VQB_SCHK"), std::make_pair("xbuf2[", "VQB_SCHK"),
                               std::make_pair("spool[", "VQB_PCHK")}) {
            size_t p = src.find(pm.first, i);
            // whole identifiers only
            while (p != std::string::npos && p > 0 && (std::isalnum((unsigned char)src[p - 1]) || src[p - 1] == '_'))
                p = src.find(pm.first, p + 1);
            if (p != std::string::npos && p < best) {
                best = p;
                open = p + std::strlen(pm.first) - 1;
                mac = pm.second;
            }
        }
        if (best == std::string::npos) break;
        wrap_at(best, open, mac);
    }
    out.append(src, i, std::string::npos);
    if (inc != std::string::npos) {
        const size_t at = out.find("using namespace vqbjit;");
        out.insert(at + std::strlen("using namespace vqbjit;") + 1, pre);
    }
    return out;
}

// Source of a specialised adjoint stage kernel (the REV mode of k_regstage on
// one lowered program): Phi and Psi tiles in registers, one tile per block,
// each parametric step's contributions reduced per warp into shared memory and
// written as one partial per (slot, tile) for k_slot_sums. Returns "" for
// programs with wide operations (they stay on the interpreter).
std::string jit_reverse_source(const RParams &P, bool *uses_spool, double *flops, int *xtiles) {
    int nops_total = 0;
    for (int i = 0; i < P.nsubs; ++i)
        for (int o = 0; o < P.subs[i].op_count; ++o) {
            const ROp &op = P.ops[P.subs[i].op_begin + o];
            if (op.nt >= 3 && op.np > 0) return ""; // wide parametric steps are unfusable anyway
            ++nops_total;
        }
    if (nops_total == 0) return "";
    auto num = [](unsigned long long v) { return std::to_string(v) + "ull"; };
    auto I = [](long long v) { return std::to_string(v); };
    auto thread_expr = [&](const int *lbits, bool global, const char *tv) {
        std::string e = "(0";
        for (int b = 0; b < TB; ++b) {
            const int pos = global ? P.bits[lbits[b]] : lbits[b];
            e += std::string(" | (") + (global ? "(u64)" : "") + "((" + tv + " >> " + I(b) + ") & 1) << " +
                 I(pos) + ")";
        }
        return e + ")";
    };
    auto slot_const = [&](const RLayout &L, int i) {
        int c = 0;
        for (int b = 0; b < RB; ++b)
            if ((i >> b) & 1) c ^= swz(1 << L.reg[b]);
        return c;
    };
    static const int pair_p0[6] = {0, 0, 0, 1, 1, 2}, pair_p1[6] = {1, 2, 3, 2, 3, 3};
    const int jit_blocks = env_int("VQB_JIT_REV_BLOCKS", R >= 16 ? 2 : 4);
    bool spool = false;
    double fl = 0, wfl = 0; // FP64 flops per thread (register code) / per tile (wide ops)
    std::string body;
    auto emit = [&](const std::string &x) { body += x; };
    // Gradient accumulators: a slot's per-thread sum is complete after its
    // step; it is warp-reduced into shared memory once more than acc_budget
    // slots are pending, so the reduction overlaps the following steps and at
    // most acc_budget accumulators hold registers (dozens of slots per launch
    // would otherwise spill).
    const int red_lanes = red_lanes_of();
    // measured: 6 for 8-register sweeps, 3 for the register-heavy 16-register ones
    const int acc_budget = env_int("VQB_JIT_ACC", R >= 16 ? 3 : 6);
    std::vector<int> open_slots;
    // Batches of 4 (2) pending slots share their shuffles: at the first two
    // (one) levels each lane keeps half of the batch and sends the other half
    // to its partner, so after them every lane holds one slot's partial and
    // the remaining levels reduce that one value: 4 (5) double shuffles per
    // 4 slots instead of 12 (16). Lane l ends with the slot selected by its
    // top lane bits; the lanes whose middle bits are zero store.
    const int red_batch = env_int("VQB_JIT_REDBATCH", 4);
    auto flush_slots = [&](int keep) {
        while ((int)open_slots.size() > keep) {
            const int avail = (int)open_slots.size();
            const int B = (red_batch >= 4 && avail >= 4 && red_lanes <= 4) ? 4
                          : (red_batch >= 2 && avail >= 2 && red_lanes <= 8) ? 2 : 1;
            std::vector<int> sl(open_slots.begin(), open_slots.begin() + B);
            open_slots.erase(open_slots.begin(), open_slots.begin() + B);
            if (B == 1) {
                // reduce over the lane bits above log2(PL) only; PL lanes per warp
                // store partial sums (fewer dependent shuffles per slot)
                std::string e = "    { double x = acc_s" + I(sl[0]) + ";";
                for (int sh = 16; sh >= red_lanes; sh >>= 1)
                    e += " x += __shfl_xor_sync(0xffffffffu, x, " + I(sh) + ");";
                e += " if (lane < " + I(red_lanes) + ") red[" + I(sl[0] * NW * red_lanes) + " + warp * " + I(red_lanes) +
                     " + lane] = x; }\n";
                emit(e);
                continue;
            }
            std::string e = "    {\n      const bool h4 = (lane & 16) != 0, h3 = (lane & 8) != 0;\n";
            auto xchg = [&](const std::string &dst, const std::string &lo, const std::string &hi, const char *flag,
                            int sh) {
                // the lane with `flag` keeps hi and sends lo, its partner the reverse
                e += "      const double " + dst + " = (" + flag + " ? " + hi + " : " + lo +
                     ") + __shfl_xor_sync(0xffffffffu, " + flag + " ? " + lo + " : " + hi + ", " + I(sh) + ");\n";
            };
            int sh = 16;
            std::string slot_expr;
            if (B == 4) {
                xchg("b0", "acc_s" + I(sl[0]), "acc_s" + I(sl[2]), "h4", 16);
                xchg("b1", "acc_s" + I(sl[1]), "acc_s" + I(sl[3]), "h4", 16);
                xchg("c0", "b0", "b1", "h3", 8);
                e += "      double x = c0;\n";
                slot_expr = "(h4 ? (h3 ? " + I(sl[3]) + " : " + I(sl[2]) + ") : (h3 ? " + I(sl[1]) + " : " + I(sl[0]) + "))";
                sh = 4;
            } else {
                xchg("c0", "acc_s" + I(sl[0]), "acc_s" + I(sl[1]), "h4", 16);
                e += "      double x = c0;\n";
                slot_expr = "(h4 ? " + I(sl[1]) + " : " + I(sl[0]) + ")";
                sh = 8;
            }
            int mid = 0;
            for (; sh >= red_lanes; sh >>= 1) {
                e += "      x += __shfl_xor_sync(0xffffffffu, x, " + I(sh) + ");\n";
                mid |= sh;
            }
            e += "      if ((lane & " + I(mid) + ") == 0) red[" + slot_expr + " * " + I(NW * red_lanes) + " + warp * " +
                 I(red_lanes) + " + (lane & " + I(red_lanes - 1) + ")] = x;\n    }\n";
            emit(e);
        }
    };
    // Where Phi and Psi live: in registers in the layout of sub-stage cur_sub,
    // or in the shared-memory tiles xbuf / xbuf2 in tile-index space (any
    // layout writes and reads the same slots). Register ops pull them into the
    // registers of their layout, wide ops push them to the tiles, so a
    // relayout next to a wide operation shares its shared-memory round trip
    // and sub-stages without register work cost no relayout.
    // the prologue leaves both states in the tiles, or (VQB_JIT_DIRECT) loads
    // them straight into the first sub-stage's layout
    const bool direct = env_int("VQB_JIT_DIRECT", 1) != 0;
    bool in_smem = !direct;
    int cur_sub = direct ? 0 : -1;
    auto to_smem = [&]() {
        if (in_smem) return;
        for (int i = 0; i < R; ++i) {
            const std::string sl = "st" + I(cur_sub) + " ^ " + I(slot_const(P.subs[cur_sub].L, i));
            emit("    xbuf[" + sl + "] = vf[" + I(i) + "]; xbuf2[" + sl + "] = vg[" + I(i) + "];\n");
        }
        emit("    __syncthreads();\n");
        in_smem = true;
    };
    const bool shuffles = env_int("VQB_JIT_SHUFFLE", 1) != 0;
    auto to_regs = [&](int sub) {
        if (!in_smem && cur_sub == sub) return;
        if (!in_smem && shuffles) {
            const std::string sh = shuffle_relayout(P.subs[cur_sub].L, P.subs[sub].L, {"vf", "vg"});
            if (!sh.empty()) {
                emit(sh);
                cur_sub = sub;
                return;
            }
        }
        to_smem();
        for (int i = 0; i < R; ++i) {
            const std::string sl = "st" + I(sub) + " ^ " + I(slot_const(P.subs[sub].L, i));
            emit("    vf[" + I(i) + "] = xbuf[" + sl + "]; vg[" + I(i) + "] = xbuf2[" + sl + "];\n");
        }
        emit("    __syncthreads();\n");
        in_smem = false;
        cur_sub = sub;
    };
    const bool lazy = env_int("VQB_JIT_LAZY", 1) != 0;
    const bool dotplan_on = env_int("VQB_JIT_DOTPLAN", 1) != 0;
    for (int sub = 0; sub < P.nsubs; ++sub) {
        const RSub &sb = P.subs[sub];
        if (!lazy) to_regs(sub);
        for (int k = 0; k < sb.op_count; ++k) {
            if (P.ops[sb.op_begin + k].nt < 3 || P.ops[sb.op_begin + k].inreg) to_regs(sub);
            const ROp &op = P.ops[sb.op_begin + k];
            // development aid: FP64 flops per thread each op's code adds
            struct CostNote {
                const ROp &o;
                const double &f, &w;
                double f0, w0;
                int sub;
                ~CostNote() {
                    if (env_int("VQB_JIT_OPCOST", 0))
                        std::fprintf(stderr, "[opcost] sub %d nt %d nc %d np %d pair %d inreg %d unit %d: %.0f flops/thread %.0f/tile\n",
                                     sub, o.nt, o.nc, o.np, o.pair, o.inreg, o.unit, f - f0, w - w0);
                }
            } cost_note{op, fl, wfl, fl, wfl, sub};
            // a run of unit-modulus diagonal steps: conj(psi) phi is invariant
            // along it, so every contribution is Re(z e_p) with z taken once,
            // and both states get the product of the phases at the end
            int run_end = k;
            while (run_end < sb.op_count && P.ops[sb.op_begin + run_end].nt == 0 &&
                   (P.ops[sb.op_begin + run_end].unit & 1) && !P.ops[sb.op_begin + run_end].pair)
                ++run_end;
            if (run_end - k >= 2 && env_int("VQB_JIT_DIAGRUN", 1)) {
                // Step-major, factored by register conditions. A step's
                // matrix element depends on a register element i only through
                // the register bits among its condition bits (mask rm, usually
                // none or one bit). So its contribution sum_i Re(z_i e(c(i)))
                // = sum_g Re(S_rm[g] e(g)) with S_rm[g] the sum of z over the
                // elements whose rm-bits are g (taken once per run), and its
                // phase multiplies one of 2^|rm| running products PH_rm[g];
                // each element gets the product of its PH's at the end. Phi
                // and Psi wait in thread-private shared-memory slots meanwhile.
                auto rmask_of = [&](const ROp &o) {
                    int m = 0;
                    for (int q = 0; q < o.nc; ++q)
                        if (o.ck[q] == 2) m |= 1 << o.cp[q];
                    return m;
                };
                auto extract = [](int i, int m) { // bits of i under mask m, compressed
                    int g = 0, k2 = 0;
                    for (int b = 0; b < RB; ++b)
                        if ((m >> b) & 1) g |= ((i >> b) & 1) << k2++;
                    return g;
                };
                std::vector<int> masks;
                for (int j = k; j < run_end; ++j) {
                    const int m = rmask_of(P.ops[sb.op_begin + j]);
                    if (std::find(masks.begin(), masks.end(), m) == masks.end()) masks.push_back(m);
                }
                // Phi and Psi stay in registers through the run
                emit("    {\n");
                emit("      double2 z[" + I(R) + "];\n");
                for (int i = 0; i < R; ++i)
                    emit("      z[" + I(i) + "] = make_double2(fma(vg[" + I(i) + "].x, vf[" + I(i) + "].x, vg[" + I(i) +
                         "].y * vf[" + I(i) + "].y), fma(vg[" + I(i) + "].x, vf[" + I(i) + "].y, -vg[" + I(i) +
                         "].y * vf[" + I(i) + "].x));\n");
                fl += 4.0 * R;
                // class sums S_m_g, phase products PH_m_g
                for (int m : masks) {
                    const int ng = 1 << __builtin_popcount(m);
                    for (int g = 0; g < ng; ++g) {
                        std::string e = "      const double2 S" + I(m) + "_" + I(g) + " = make_double2(0.0";
                        std::string ex, ey;
                        for (int i = 0; i < R; ++i)
                            if (extract(i, m) == g) {
                                ex += " + z[" + I(i) + "].x";
                                ey += " + z[" + I(i) + "].y";
                                fl += 2;
                            }
                        emit(e + ex + ", 0.0" + ey + ");\n      double2 PH" + I(m) + "_" + I(g) + ";\n");
                    }
                }
                std::map<std::pair<int, int>, bool> ph_set;
                for (int j = k; j < run_end; ++j) {
                    const ROp &oj = P.ops[sb.op_begin + j];
                    std::string dynx;
                    int rmq = 0;
                    for (int q = 0; q < oj.nc; ++q) {
                        if (oj.ck[q] == 0)
                            dynx += " | (int)(((base >> " + I(oj.cp[q]) + ") & 1) << " + I(q) + ")";
                        else if (oj.ck[q] == 1)
                            dynx += " | (((to >> " + I(oj.cp[q]) + ") & 1) << " + I(q) + ")";
                        else
                            rmq |= 1 << q;
                    }
                    const bool dyn = !dynx.empty();
                    if (dyn) spool = true;
                    const int m = rmask_of(oj);
                    const int ng = 1 << __builtin_popcount(m);
                    const int nsubj = 1 << oj.nc;
                    emit("      {\n");
                    if (dyn) emit("        const int cd = 0" + dynx + ";\n");
                    for (int g = 0; g < ng; ++g) {
                        // condition index bits contributed by the register bits g
                        int cs = 0, k2 = 0, full = 0;
                        for (int b = 0; b < RB; ++b)
                            if ((m >> b) & 1) full |= ((g >> k2++) & 1) << b;
                        for (int q = 0; q < oj.nc; ++q)
                            if (oj.ck[q] == 2 && ((full >> oj.cp[q]) & 1)) cs |= 1 << q;
                        auto elem = [&](unsigned off) {
                            return dyn ? "spool[" + I(off) + " + (cd | " + I(cs) + ")]" : "P.pool[" + I(off + (unsigned)cs) + "]";
                        };
                        auto ucls = [&](unsigned off) {
                            int c = 0;
                            for (int cc = 0; cc < nsubj; ++cc)
                                if (dyn ? (cc & rmq) == cs : cc == cs) c |= pool_cls(P, off + (unsigned)cc, 1, 0);
                            return c;
                        };
                        const std::string Sg = "S" + I(m) + "_" + I(g), PHg = "PH" + I(m) + "_" + I(g);
                        for (int p = 0; p < oj.np; ++p) {
                            const unsigned eo = oj.mat_e + (unsigned)(p << oj.nc);
                            const int c = ucls(eo);
                            const std::string acc = "acc_s" + I(oj.slot + p), e = elem(eo);
                            if (c == 1) { emit("        " + acc + " = fma(" + Sg + ".x, " + e + ".x, " + acc + ");\n"); fl += 2; }
                            else if (c == 2) { emit("        " + acc + " = fma(-" + Sg + ".y, " + e + ".y, " + acc + ");\n"); fl += 2; }
                            else if (c == 3) {
                                emit("        " + acc + " = fma(" + Sg + ".x, " + e + ".x, fma(-" + Sg + ".y, " + e + ".y, " + acc + "));\n");
                                fl += 4;
                            }
                        }
                        if (!dyn && ((oj.ident >> cs) & 1)) continue;
                        const std::string mm = elem(oj.mat);
                        const int c = ucls(oj.mat);
                        bool &set = ph_set[{m, g}];
                        if (!set) {
                            emit("        " + PHg + " = " + mm + ";\n");
                            set = true;
                        } else if (c == 1) {
                            emit("        " + PHg + ".x *= " + mm + ".x; " + PHg + ".y *= " + mm + ".x;\n");
                            fl += 2;
                        } else if (c == 2) {
                            emit("        " + PHg + " = make_double2(-" + mm + ".y * " + PHg + ".y, " + mm + ".y * " + PHg + ".x);\n");
                            fl += 2;
                        } else {
                            emit("        " + PHg + " = cmul(" + mm + ", " + PHg + ");\n");
                            fl += 6;
                        }
                    }
                    emit("      }\n");
                    for (int p = 0; p < oj.np; ++p) open_slots.push_back(oj.slot + p);
                    flush_slots(acc_budget);
                }
                // every element: the product of its phase products
                // (innermost product from the masks with the fewest classes: the
                // partial products shared between elements are then the small ones)
                std::vector<int> by_size(masks);
                std::stable_sort(by_size.begin(), by_size.end(), [](int a, int b) {
                    return __builtin_popcount(a) < __builtin_popcount(b);
                });
                for (int i = 0; i < R; ++i) {
                    std::string ph;
                    for (int m : by_size) {
                        const int g = extract(i, m);
                        if (!ph_set[{m, g}]) continue;
                        const std::string t2 = "PH" + I(m) + "_" + I(g);
                        if (ph.empty()) ph = t2;
                        else {
                            ph = "cmul(" + t2 + ", " + ph + ")";
                            fl += 6;
                        }
                    }
                    if (ph.empty()) continue;
                    emit("      { const double2 ph = " + ph + "; vf[" + I(i) + "] = cmul(ph, vf[" + I(i) +
                         "]); vg[" + I(i) + "] = cmul(ph, vg[" + I(i) + "]); }\n");
                    fl += 12;
                }
                emit("    }\n");
                k = run_end - 1;
                continue;
            }
            if (op.nt >= 3 && op.inreg) {
                std::string dyn;
                for (int q = 0; q < op.nc; ++q) {
                    if (op.ck[q] == 0)
                        dyn += " | (int)(((base >> " + I(op.cp[q]) + ") & 1) << " + I(q) + ")";
                    else if (op.ck[q] == 1)
                        dyn += " | (((to >> " + I(op.cp[q]) + ") & 1) << " + I(q) + ")";
                }
                if (!dyn.empty()) {
                    dyn = "(0" + dyn + ")";
                    spool = true;
                }
                auto pe = [&](unsigned off) { return "P.pool[" + I(off) + "]"; };
                for (int st2 = 0; st2 < 2; ++st2) {
                    const char *v = st2 ? "vg" : "vf";
                    if (dyn.empty() && op.pair && op.np == 0 && (op.unit & (st2 ? 8 : 4))) {
                        if (((st2 ? op.ident_psi : op.ident) & 1)) continue;
                        int rmask = 0;
                        for (int q = 0; q < op.nt; ++q) rmask |= 1 << op.lb[q];
                        for (int i0 = 0; i0 < R; ++i0) {
                            if (i0 & rmask) continue;
                            int ridx[16], nr = 0;
                            for (int r = 0; r < (1 << op.nt); ++r) {
                                if (!((op.slot >> r) & 1)) continue;
                                int x = i0;
                                for (int q = 0; q < op.nt; ++q)
                                    if ((r >> q) & 1) x |= 1 << op.lb[q];
                                ridx[nr++] = x;
                            }
                            emit(rank_one_code(v, ridx, nr, "P.pool[" + I(st2 ? op.mat_e : op.mat_d) + "]", fl));
                        }
                        continue;
                    }
                    if (st2 == 0) emit(jit_wide_regs(P, op, "vf", op.mat, op.ident, dyn, pe, fl));
                    else
                        emit(jit_wide_regs(P, op, "vg", op.pair ? op.mat_psi : op.mat,
                                           op.pair ? op.ident_psi : op.ident, dyn, pe, fl));
                }
                continue;
            }
            if (op.nt >= 3) {
                const std::string sbase = "st" + I(sub);
                const WideState wf{"vf", "xbuf", op.mat, op.ident};
                const WideState wg{"vg", "xbuf2", op.pair ? op.mat_psi : op.mat, op.pair ? op.ident_psi : op.ident};
                to_smem();
                emit(jit_wide_op(P, sub, op, {wf, wg}, sbase.c_str(), &wfl, &spool, true));
                if (!lazy) to_regs(sub);
                continue;
            }
            const int dd = 1 << (2 * op.nt), nsub = 1 << op.nc;
            std::string dyn;
            for (int q = 0; q < op.nc; ++q) {
                if (op.ck[q] == 0)
                    dyn += " | (int)(((base >> " + I(op.cp[q]) + ") & 1) << " + I(q) + ")";
                else if (op.ck[q] == 1)
                    dyn += " | (((to >> " + I(op.cp[q]) + ") & 1) << " + I(q) + ")";
            }
            const bool dynamic = !dyn.empty();
            spool = spool || dynamic;
            auto cstat = [&](int i) {
                int c = 0;
                for (int q = 0; q < op.nc; ++q)
                    if (op.ck[q] == 2 && ((i >> op.cp[q]) & 1)) c |= 1 << q;
                return c;
            };
            std::string tmpl;
            int mask = 0;
            if (op.nt == 1) {
                tmpl = "1, " + I(op.code) + ", 0, " + I(R);
                mask = 1 << op.code;
            } else if (op.nt == 2) {
                tmpl = "2, " + I(pair_p0[op.code]) + ", " + I(pair_p1[op.code]) + ", " + I(R);
                mask = (1 << pair_p0[op.code]) | (1 << pair_p1[op.code]);
            }
            int rmask = 0;
            for (int q = 0; q < op.nc; ++q)
                if (op.ck[q] == 2) rmask |= 1 << q;
            const int D = 1 << op.nt;
            // entry k of the sub-matrix selected by (cd | cs) of the matrix
            // array at `off` (sub-matrix stride dd): expression and class (the
            // union over the run-time selectable sub-matrices)
            auto mexpr = [&](unsigned off, int cs) {
                return [=](int k) {
                    if (dynamic) return "spool[" + I(off) + " + (cd | " + I(cs) + ") * " + I(dd) + " + " + I(k) + "]";
                    return "P.pool[" + I(off + (unsigned)(cs * dd + k)) + "]";
                };
            };
            auto mcls = [&](unsigned off, int cs) {
                return [=, &P](int k) {
                    int c = -1;
                    for (int cc = 0; cc < nsub; ++cc)
                        if (dynamic ? (cc & rmask) == cs : cc == cs) {
                            const int e = pool_ucls(P, off + (unsigned)(cc * dd + k), 1, 0);
                            c = c < 0 ? e : merge_cls(c, e);
                        }
                    return c < 0 ? 0 : c;
                };
            };
            if (dynamic) emit("    {\n      const int cd = 0" + dyn + ";\n");
            else emit("    {\n");
            if (op.np == 0) {
                const unsigned mpsi = op.pair ? op.mat_psi : op.mat;
                const unsigned long long ipsi = op.pair ? op.ident_psi : op.ident;
                for (int st2 = 0; st2 < 2; ++st2) {
                    const char *v = st2 ? "vg" : "vf";
                    const unsigned m = st2 ? mpsi : op.mat;
                    const unsigned long long id = st2 ? ipsi : op.ident;
                    const bool r1 = !dynamic && op.pair && (op.unit & (st2 ? 8 : 4));
                    for (int i = 0; i < R; ++i) {
                        if (i & mask) continue;
                        const int cs = cstat(i);
                        int idx[4];
                        group_idx(op.nt, op.code, i, idx);
                        if (!dynamic && ((id >> cs) & 1)) continue;
                        if (r1) {
                            int ridx[16], nr = 0;
                            for (int r = 0; r < D; ++r)
                                if ((op.slot >> r) & 1) ridx[nr++] = idx[r];
                            emit(rank_one_code(v, ridx, nr, "P.pool[" + I(st2 ? op.mat_e : op.mat_d) + "]", fl));
                            continue;
                        }
                        if (dynamic) emit("      if (!((" + num(id) + " >> (cd | " + I(cs) + ")) & 1))\n");
                        emit(mv_code(v, idx, D, mexpr(m, cs), mcls(m, cs), fl));
                    }
                }
            } else {
                // per-slot accumulators live to the end of the tile; their warp
                // reductions are issued together there (independent shuffle
                // chains overlap instead of stalling each parametric step)
                // factored contraction (DotPlan) per (parameter, register
                // condition): unit-weighted sums w_c over the thread's groups,
                // multiplied by the class values once after the last group
                std::map<std::pair<int, int>, DotPlan> plans;
                if (dotplan_on)
                    for (int i = 0; i < R; ++i) {
                        if (i & mask) continue;
                        const int cs = cstat(i);
                        for (int p = 0; p < op.np; ++p) {
                            if (plans.count({p, cs})) continue;
                            const DotPlan pl =
                                dot_plan(P, dot_base(op) + (unsigned)(p * nsub * dd), dd, dot_selectable(op, cs));
                            plans[{p, cs}] = pl;
                            if (!pl.ok) continue;
                            const std::string w = "w" + I(p) + "_" + I(cs) + "_";
                            for (int c = 0; c < pl.nclass; ++c) {
                                if (pl.need[c] & 1) emit("      double " + w + "r" + I(c) + " = 0.0;\n");
                                if (pl.need[c] & 2) emit("      double " + w + "i" + I(c) + " = 0.0;\n");
                            }
                        }
                    }
                for (int i = 0; i < R; ++i) {
                    if (i & mask) continue;
                    const int cs = cstat(i);
                    int idx[4];
                    group_idx(op.nt, op.code, i, idx);
                    // G_p = D_p inv, or e_p of a unit-modulus diagonal step, on the old Phi
                    const bool gpre = (op.unit & 2) != 0 || dot_base(op) != op.mat_d;
                    if (!gpre) emit(mv_code("vf", idx, D, mexpr(op.mat, cs), mcls(op.mat, cs), fl));
                    for (int p = 0; p < op.np; ++p) {
                        const unsigned dof = dot_base(op) + (unsigned)(p * nsub * dd);
                        auto it = plans.find({p, cs});
                        if (it != plans.end() && it->second.ok)
                            emit(dot_plan_group(it->second, "w" + I(p) + "_" + I(cs) + "_", idx, D, fl));
                        else
                            emit(dot_code("acc_s" + I(op.slot + p), idx, D, mexpr(dof, cs), mcls(dof, cs), fl));
                    }
                    if (gpre) emit(mv_code("vf", idx, D, mexpr(op.mat, cs), mcls(op.mat, cs), fl));
                    emit(mv_code("vg", idx, D, mexpr(op.mat, cs), mcls(op.mat, cs), fl));
                }
                for (const auto &kv : plans) {
                    const DotPlan &pl = kv.second;
                    if (!pl.ok) continue;
                    const int p = kv.first.first, cs = kv.first.second;
                    const unsigned dof = dot_base(op) + (unsigned)(p * nsub * dd);
                    const std::string w = "w" + I(p) + "_" + I(cs) + "_", acc = "acc_s" + I(op.slot + p);
                    for (int c = 0; c < pl.nclass; ++c) {
                        const std::string m = mexpr(dof, cs)(pl.ref[c]);
                        if (pl.need[c] & 1) { emit("      " + acc + " = fma(" + m + ".x, " + w + "r" + I(c) + ", " + acc + ");\n"); fl += 2; }
                        if (pl.need[c] & 2) { emit("      " + acc + " = fma(-" + m + ".y, " + w + "i" + I(c) + ", " + acc + ");\n"); fl += 2; }
                    }
                }
                for (int p = 0; p < op.np; ++p) open_slots.push_back(op.slot + p);
            }
            emit("    }\n");
            flush_slots(acc_budget);
        }
    }
    flush_slots(0);
    to_regs(P.nsubs - 1);
    const RLayout &Lf = P.subs[P.nsubs - 1].L;
    std::string src;
    auto out = [&](const std::string &x) { src += x; };
    out("#include \"jit_rt.cuh\"\nusing namespace vqbjit;\n");
    out("struct JP { double2 pool[" + I(std::max(P.npool, 1)) + "]; };\n");
    out("extern \"C\" __global__ void __launch_bounds__(" + I(T) + ", " + I(jit_blocks) + ")\n"
        "vqb_rev(double2 *__restrict__ a, double2 *__restrict__ b2, double *__restrict__ partial,\n"
        "        const __grid_constant__ JP P) {\n");
    // shared memory: xbuf (relayouts, Phi's wide ops) [| xbuf2 (Psi's wide
    // ops)] [| pool copy] | gradient reduction slots
    const int xt = 2; // xbuf (Phi) and xbuf2 (Psi)
    if (spool && pool_reads_from_bank(body)) spool = false; // one tile per block
    out("  extern __shared__ __align__(16) double2 sm[];\n  double2 *xbuf = sm;\n");
    out("  double2 *xbuf2 = sm + " + I(TS) + ";\n");
    const int red_at = xt * TS + (spool ? P.npool : 0);
    if (spool)
        out("  double2 *spool = sm + " + I(xt * TS) + ";\n  for (int i = threadIdx.x; i < " + I(P.npool) +
            "; i += " + I(T) + ") spool[i] = P.pool[i];\n");
    out("  double *red = reinterpret_cast<double *>(sm + " + I(red_at) + ");\n");
    out("  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;\n");
    for (int sl = 0; sl < P.nslots; ++sl) out("  double acc_s" + I(sl) + " = 0;\n");
    int nat_local[TB];
    for (int b = 0; b < TB; ++b) nat_local[b] = b;
    out("  const u64 glo = " + thread_expr(nat_local, true, "t") + ";\n");
    out("  const u64 gfin = " + thread_expr(Lf.thr, true, "t") + ";\n");
    out("  auto base_of = [&](u64 c) -> u64 {\n");
    for (int j = 0; j < K; ++j) {
        const int sbit = P.bits[j];
        out("    c = ((c >> " + I(sbit) + ") << " + I(sbit + 1) + ") | (c & " + num((1ull << sbit) - 1) + ");\n");
    }
    out("    return c;\n  };\n");
    out("  const u64 tile = blockIdx.x;\n  const u64 base = base_of(tile);\n");
    out("  double2 vf[" + I(R) + "], vg[" + I(R) + "];\n");
    if (direct) {
        const RLayout &L0 = P.subs[0].L;
        out("  const u64 g0 = " + thread_expr(L0.thr, true, "t") + ";\n");
        for (int i = 0; i < R; ++i) {
            unsigned long long g = 0;
            for (int b = 0; b < RB; ++b)
                if ((i >> b) & 1) g |= 1ull << P.bits[L0.reg[b]];
            out("  vf[" + I(i) + "] = a[base | g0 | " + num(g) + "];\n  vg[" + I(i) + "] = b2[base | g0 | " + num(g) +
                "];\n");
        }
    }
    for (int s2 = 0; s2 < R && !direct; ++s2) {
        unsigned long long g = 0;
        for (int b = 0; b < RB; ++b)
            if ((s2 >> b) & 1) g |= 1ull << P.bits[TB + b];
        out("  vf[" + I(s2) + "] = a[base | glo | " + num(g) + "];\n  vg[" + I(s2) + "] = b2[base | glo | " + num(g) +
            "];\n");
    }
    out("  int to; asm volatile(\"mov.b32 %0, %1;\" : \"=r\"(to) : \"r\"(t));\n");
    for (int sub = 0; sub < P.nsubs; ++sub)
        out("  const int st" + I(sub) + " = swz" + thread_expr(P.subs[sub].L.thr, false, "to") + ";\n");
    if (!direct) {
        out("  const int nat_st = swz(to);\n");
        for (int s2 = 0; s2 < R; ++s2) {
            int sl = 0;
            for (int b = 0; b < RB; ++b)
                if ((s2 >> b) & 1) sl ^= swz(T << b);
            out("  xbuf[nat_st ^ " + I(sl) + "] = vf[" + I(s2) + "]; xbuf2[nat_st ^ " + I(sl) + "] = vg[" + I(s2) + "];\n");
        }
        out("  __syncthreads();\n");
    } else if (spool) {
        out("  __syncthreads(); // the pool copy above is read by every thread\n");
    }
    out(body);
    for (int i = 0; i < R; ++i) {
        unsigned long long g = 0;
        for (int b = 0; b < RB; ++b)
            if ((i >> b) & 1) g |= 1ull << P.bits[Lf.reg[b]];
        out("  a[base | gfin | " + num(g) + "] = vf[" + I(i) + "];\n  b2[base | gfin | " + num(g) + "] = vg[" + I(i) +
            "];\n");
    }
    if (P.nslots > 0) {
        // every slot was reduced into red[] by flush_slots
        out("  __syncthreads();\n");
        out("  for (int s = t; s < " + I(P.nslots) + "; s += " + I(T) + ") {\n    double x = 0;\n");
        for (int w = 0; w < NW * red_lanes; ++w) out("    x += red[s * " + I(NW * red_lanes) + " + " + I(w) + "];\n");
        out("    partial[(size_t)s * " + num(P.ntiles) + " + tile] = x;\n  }\n");
    }
    out("}\n");
    if (uses_spool) *uses_spool = spool;
    if (flops) *flops = (fl * T + wfl) / TS; // executed FP64 flops per amplitude (both states)
    if (xtiles) *xtiles = xt;
    return src;
}

// Specialised kernels by stage-program *structure*: everything in RParams but
// the matrix values (pool, tab). A hit skips source generation entirely.
struct JitShape {
    std::string key;
    jit::Kernel k;
    bool spool = false, per_block = false;
    double flops_per_amp = 0; // executed FP64 flops (structure-aware code)
    int xtiles = 1;           // adjoint: shared-memory tiles (2 with wide operations)
};
uint64_t fnv1a(const std::string &s) {
    // word-wise FNV-1a variant (the key is a few KB per launch)
    uint64_t h = 1469598103934665603ull;
    size_t i = 0;
    for (; i + 8 <= s.size(); i += 8) {
        uint64_t w;
        std::memcpy(&w, s.data() + i, 8);
        h = (h ^ w) * 1099511628211ull;
        h ^= h >> 29;
    }
    for (; i < s.size(); ++i) h = (h ^ (unsigned char)s[i]) * 1099511628211ull;
    return h;
}
std::string shape_key(const RParams &P, bool rev) {
    // the used parts of the structural fields (everything but the matrix
    // values; unused array tails are zero by construction)
    int nops = 0;
    for (int i = 0; i < P.nsubs; ++i) nops = std::max(nops, P.subs[i].op_begin + P.subs[i].op_count);
    std::string key(rev ? "R" : "F");
    auto add = [&](const void *p, size_t n) { key.append(static_cast<const char *>(p), n); };
    add(P.bits, sizeof P.bits);
    add(&P.ntiles, sizeof P.ntiles);
    add(&P.nsubs, 2 * sizeof(int)); // nsubs, nslots (slot_begin and partial_ld do not shape the code)
    add(P.subs, sizeof(RSub) * (size_t)P.nsubs);
    add(P.ops, sizeof(ROp) * (size_t)nops);
    add(&P.ntab, 3 * sizeof(int)); // ntab, nxpat, npool
    add(P.xpat, (size_t)P.nxpat);
    add(P.fast, sizeof(int) * (size_t)nops);
    // per-entry structure of the matrices (zero / real / imaginary / complex,
    // pool_cls): the generated code depends on it, the values themselves not
    {
        std::string cls((size_t)(P.npool + 1) / 2, '\0');
        for (int i = 0; i < P.npool; ++i)
            cls[(size_t)i >> 1] = (char)(cls[(size_t)i >> 1] | (pool_ucls(P, (unsigned)i, 1, 0) << (4 * (i & 1))));
        key += cls;
    }
    // partitions of the derivative matrices (DotPlan)
    if (rev)
        for (int i = 0; i < nops; ++i) key += dot_signature(P, P.ops[i]) + "/";
    for (const char *e : {"VQB_JIT_DOTPLAN", "VQB_JIT_REDBATCH", "VQB_JIT_PAIRFACTOR", "VQB_JIT_RANKONE", "VQB_JIT_POOL", "VQB_JIT_BLOCKS", "VQB_JIT_MODE", "VQB_JIT_REV_BLOCKS", "VQB_JIT_DIAGRUN", "VQB_JIT_ACC", "VQB_JIT_WIDE2", "VQB_JIT_LAZY", "VQB_WIDE_REGS", "VQB_JIT_GDIFF", "VQB_JIT_SHUFFLE", "VQB_JIT_REDLANES", "VQB_JIT_DIRECT", "VQB_JIT_FACTOR", "VQB_JIT_CHECK", "VQB_JIT_PBANK"}) {
        const char *v = std::getenv(e);
        key += '|';
        if (v) key += v;
    }
    return key;
}
std::mutex g_shape_mu;
std::unordered_map<uint64_t, JitShape> g_shapes;
// cached kernel for a structure, or nullptr
const JitShape *find_shape(const std::string &key, uint64_t h) {
    std::lock_guard<std::mutex> lk(g_shape_mu);
    auto it = g_shapes.find(h);
    return it != g_shapes.end() && it->second.key == key ? &it->second : nullptr;
}

// Shared driver: stage planning, block fusion, lowering, launches.
template <bool REV, typename Fallback>
void run_reg(DeviceState *sphi, DeviceState *spsi, std::vector<FusedOp> &fops, double *dgrads,
             Fallback &&fallback) {
    HostTimer ht_all(REV ? "run_reg (rev) total" : "run_reg (fwd) total");
    double t_fuse = 0, t_lower = 0, t_key = 0, t_issue = 0;
    struct Report {
        double *a, *b, *c, *d;
        ~Report() {
            static const bool on = std::getenv("VQB_HOST_TIMING") != nullptr;
            if (on) std::fprintf(stderr, "[host]   fuse %.1f lower %.1f key %.1f issue %.1f us\n", *a, *b, *c, *d);
        }
    } report{&t_fuse, &t_lower, &t_key, &t_issue};
    const int pn = sphi->pn;
    cudaStream_t st = sphi->stream;
    std::vector<Stage> stages;
    {
        HostTimer ht(REV ? "plan_stages (rev)" : "plan_stages (fwd)");
        // the executor splits a stage into launches itself (kMaxOps blocks each),
        // and block fusion shrinks runs of gates: stages may hold more operations
        // than the shared-memory interpreter's limit
        // (density-matrix programs pair every ket bit with its bra bit, so good
        // tiles are rarer: their search starts from 24 seeds per stage instead of
        // 12 -- config 3's adjoint 23 -> 21 launches, profiles/r2_ab_plan_seeds.txt)
        stages = plan_stages(fops, pn, K, env_int("VQB_STAGE_OPS", 192), sphi->mixed && pn >= 22 ? 24 : 0);
    }
    const int max_support = env_int("VQB_FUSE_QUBITS", 2);
    const bool stats = std::getenv("VQB_PLAN_STATS") != nullptr;
    const unsigned long long ntiles = 1ull << (pn - K);
    // upper bound of the per-launch grids (no pool): partial rows of blocks a
    // launch does not run stay zero
    const int grid = grid_size<REV, true>(ntiles, smem_bytes<REV>(0));
    // gradient slots of the whole sweep: partial[grid][total slots]
    int total_slots = 0;
    if (REV)
        for (const auto &f : fops) total_slots += f.np;
    static thread_local DevMem m_partial, m_slots;
    // per-block partial rows of the interpreter's launches: zeroed at its first
    // use; a sweep run entirely by specialised kernels (per-slot sums in
    // m_slotsum) leaves them out of the final reduction
    bool partial_rows_used = false;
    auto use_partial_rows = [&] {
        if (partial_rows_used || !REV || total_slots == 0) return;
        VQB_CUDA(cudaMemsetAsync(m_partial.p, 0, sizeof(double) * (size_t)grid * total_slots, st));
        partial_rows_used = true;
    };
    if (REV && total_slots > 0) m_partial.ensure(sizeof(double) * (size_t)grid * total_slots);
    SlotMap slots;
    // Actions (a launch, or an unfusable op) are lowered in program order and
    // issued as soon as their kernel is known, so the host's planning of later
    // stages overlaps the device's work on earlier ones. The first
    // specialisation miss switches to batch mode: the rest is lowered first,
    // all missing kernels are compiled in parallel, then everything pending is
    // issued in order.
    struct Action {
        int fallback_op = -1;
        std::unique_ptr<RParams> P;
        bool wide = false;     // interpreter variant with wide-op support
        bool has_wide = false; // nt >= 3 operations (not specialised)
        const JitShape *jit = nullptr;
        std::string key;
        uint64_t hash = 0;
        double dense_flops_per_amp = 0; // interpreter: dense matrices
    };
    // adjoint specialisation: per-(slot, tile) partials, summed per launch
    static thread_local DevMem m_jpartial, m_slotsum, m_slotsplit;
    // Small sweeps (config 0: 2^10 tiles, 600 slots) keep every slot's tile
    // partials of the whole sweep and sum them in one launch at the end
    // instead of one small launch behind every stage.
    const bool merged_sums = REV && total_slots > 0 && (size_t)total_slots * ntiles <= (size_t(1) << 23) &&
                             ntiles < (1ull << 16);
    const size_t jpartial_bytes =
        sizeof(double) * (size_t)(merged_sums ? std::max(total_slots, kMaxSlots) : kMaxSlots) * ntiles;
    const bool use_jit = jit::enabled(pn) && (!REV || jpartial_bytes <= (size_t(1) << 30));
    bool any_jit_slots = false;
    // wide operations on register bits need the specialised kernels (the
    // interpreter runs them through shared memory only)
    const bool regwide = use_jit && RB >= 4 && env_int("VQB_WIDE_REGS", 1) != 0;
    if (REV && total_slots > 0) {
        m_slotsum.ensure(sizeof(double) * total_slots);
        VQB_CUDA(cudaMemsetAsync(m_slotsum.p, 0, sizeof(double) * total_slots, st));
        if (use_jit) m_jpartial.ensure(jpartial_bytes);
        if (use_jit && merged_sums) VQB_CUDA(cudaMemsetAsync(m_jpartial.p, 0, jpartial_bytes, st));
    }
    // structure-aware kernels: merge blocks only where the emitted cost does
    // not grow, factor scalars out of the forward matrices (VQB_JIT_FACTOR=0:
    // merge whenever possible, no factoring)
    // (auto: states of >= 2^22 amplitudes, where the planning cost -- about
    // 0.5 us per operation -- hides behind the kernels; config 0's 2^20
    // amplitudes are host-bound and measured faster without: 491 vs 414
    // evals/s. VQB_JIT_FACTOR=1 / 0 forces it on / off.)
    const int factor_env = env_int("VQB_JIT_FACTOR", -1);
    const bool factor_on = use_jit && (factor_env < 0 ? pn >= 22 : factor_env != 0);
    const bool cost_fusion = factor_on && !REV;
    bool batching = false;
    std::vector<Action> pending;
    auto issue = [&](Action &act) {
        if (REV) wait_issue_gate();
        if (act.fallback_op >= 0) {
            fallback(fops[act.fallback_op]);
            return;
        }
        RParams &P = *act.P;
        if (!(act.jit && act.jit->k.e)) {
            int nops = 0;
            for (int i = 0; i < P.nsubs; ++i) nops = std::max(nops, P.subs[i].op_begin + P.subs[i].op_count);
            for (int i = 0; i < nops; ++i)
                if (P.ops[i].inreg || (P.ops[i].nt > 0 && (P.ops[i].unit & 2)) || (P.ops[i].unit & 16))
                    raise(VQB_ERR_INTERNAL, "stage program with register-resident wide operations has no "
                                            "specialised kernel (set VQB_WIDE_REGS=0)");
        }
        const double launch_flops =
            (act.jit && act.jit->k.e ? act.jit->flops_per_amp : act.dense_flops_per_amp) * double(1ull << pn);
        note_flops(launch_flops);
        const ProfMark pf_ = prof_begin(st);
        prof_annotate(pf_, launch_flops, 32.0 * (REV ? 2 : 1) * double(1ull << pn));
        if (act.jit && act.jit->k.e && REV) {
            const JitShape &sh = *act.jit;
            const size_t sm = (size_t)(sh.xtiles * TS + (sh.spool ? P.npool : 0)) * sizeof(double2) +
                              sizeof(double) * (size_t)P.nslots * NW * red_lanes_of();
            void *a0 = sphi->amps, *a1 = spsi->amps, *pp = m_jpartial.p;
            if (merged_sums) pp = static_cast<double *>(m_jpartial.p) + (size_t)P.slot_begin * ntiles;
            void *args[4] = {&a0, &a1, &pp, P.pool};
            jit::launch(sh.k, (unsigned)ntiles, T, sm, st, args);
            check_launch("k_regstage_rev_jit", pf_);
            if (P.nslots > 0 && merged_sums) {
                any_jit_slots = true; // summed after the last launch
            } else if (P.nslots > 0) {
                const ProfMark pf2 = prof_begin(st);
                // small sweeps (few tiles): one block per slot, straight to the sums
                double *slot_out = static_cast<double *>(m_slotsum.p) + P.slot_begin;
                if (ntiles >= (1ull << 16)) {
                    m_slotsplit.ensure(sizeof(double) * kMaxSlots * kSlotSplit);
                    k_slot_sums<<<dim3(P.nslots, kSlotSplit), 256, 0, st>>>(
                        static_cast<const double *>(m_jpartial.p), ntiles, static_cast<double *>(m_slotsplit.p));
                    k_slot_final<<<1, 64, 0, st>>>(static_cast<const double *>(m_slotsplit.p), P.nslots,
                                                   kSlotSplit, slot_out);
                    note_launch(1); // k_slot_final (check_launch below counts k_slot_sums)
                } else {
                    k_slot_sums<<<dim3(P.nslots, 1), 256, 0, st>>>(static_cast<const double *>(m_jpartial.p),
                                                                  ntiles, slot_out);
                }
                check_launch("k_slot_sums", pf2);
            }
            return;
        }
        if (act.jit && act.jit->k.e) {
            const JitShape &sh = *act.jit;
            const size_t sm = (size_t)((sh.per_block ? 1 : 2) * TS + (sh.spool ? P.npool : 0)) * sizeof(double2);
            static int nsm = 0;
            if (!nsm) VQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
            const unsigned g = sh.per_block
                                   ? (unsigned)ntiles
                                   : (unsigned)std::min<unsigned long long>(
                                         (unsigned long long)nsm * jit::blocks_per_sm(sh.k, T, sm), ntiles);
            void *amps = sphi->amps;
            void *args[2] = {&amps, P.pool};
            jit::launch(sh.k, g, T, sm, st, args);
            check_launch("k_regstage_jit", pf_);
            return;
        }
        use_partial_rows();
        if (act.wide) {
            const size_t sm = smem_bytes<REV>(P.npool);
            k_regstage<REV, true><<<grid_size<REV, true>(ntiles, sm), T, sm, st>>>(
                sphi->amps, REV ? spsi->amps : nullptr, static_cast<double *>(m_partial.p), P);
        } else {
            const size_t sm = smem_bytes<REV, false>(P.npool);
            k_regstage<REV, false><<<grid_size<REV, false>(ntiles, sm), T, sm, st>>>(
                sphi->amps, REV ? spsi->amps : nullptr, static_cast<double *>(m_partial.p), P);
        }
        check_launch(REV ? "k_regstage_rev" : "k_regstage", pf_);
    };
    // Per stage: block fusion, lowering (one or more launches) and the kernel
    // lookup. Stages are independent once planned, so they are prepared in
    // parallel on the planning pool (plan.hpp StageJob) and issued in program
    // order as they complete; gradient slots are numbered per stage and
    // shifted to their place in the sweep afterwards.
    struct StageOut {
        std::vector<Action> acts;
        SlotMap slots;
        std::exception_ptr err;
    };
    std::vector<StageOut> outs(stages.size());
    auto prepare = [&](size_t si) {
        StageOut &so = outs[si];
        try {
            const Stage &sg = stages[si];
            if (!sg.fused) {
                Action a;
                a.fallback_op = sg.ops[0];
                so.acts.push_back(std::move(a));
                return;
            }
            std::deque<FusedOp> store; // merged blocks (stable addresses)
            std::vector<const FusedOp *> blocks;
            if (max_support > 0) blocks = fuse_blocks_ref(fops, sg.ops, max_support, store, cost_fusion);
            else
                for (int idx : sg.ops) blocks.push_back(&fops[idx]);
            std::vector<int> remaining(blocks.size());
            for (size_t i = 0; i < blocks.size(); ++i) remaining[i] = (int)i;
            while (!remaining.empty()) {
                Action act;
                act.P = std::make_unique<RParams>();
                RParams &P = *act.P;
                lower_stage_reg(sg, blocks, remaining, pn, REV, P, so.slots, regwide,
                                use_jit && env_int("VQB_JIT_GDIFF", 1) != 0, factor_on);
                P.partial_ld = total_slots;
                if (stats) {
                    int nt_hist[5] = {0, 0, 0, 0, 0}, nops = 0;
                    for (int i = 0; i < P.nsubs; ++i) nops += P.subs[i].op_count;
                    for (int i = 0; i < nops; ++i) nt_hist[std::min(P.ops[i].nt, 4)]++;
                    std::string tb;
                    for (int j = 0; j < K; ++j) tb += (j ? "," : "") + std::to_string(sg.bits[j]);
                    std::fprintf(stderr, "[regstage%s] gates %zu blocks %zu subs %d ops nt0..4 %d %d %d %d %d slots %d tile %s\n",
                                 REV ? "-rev" : "", sg.ops.size(), blocks.size(), P.nsubs, nt_hist[0],
                                 nt_hist[1], nt_hist[2], nt_hist[3], nt_hist[4], P.nslots, tb.c_str());
                }
                {
                    // algorithmic FP64 flops of this launch: a dense 2^nt x 2^nt
                    // complex matrix costs 8 * 2^nt flops per amplitude per state;
                    // a parametric step adds the np derivative contractions
                    double per_amp = 0;
                    int nops = 0;
                    for (int i = 0; i < P.nsubs; ++i) nops += P.subs[i].op_count;
                    for (int i = 0; i < nops; ++i) {
                        const ROp &o = P.ops[i];
                        const double mv = o.nt == 0 ? 6.0 : 8.0 * (1 << o.nt);
                        per_amp += (REV ? 2.0 : 1.0) * mv + (REV ? o.np * (mv + 2.0) : 0.0);
                    }
                    act.dense_flops_per_amp = per_amp;
                }
                for (int i = 0; i < P.nsubs; ++i)
                    for (int o = 0; o < P.subs[i].op_count; ++o)
                        act.has_wide = act.has_wide || P.ops[P.subs[i].op_begin + o].nt >= 3;
                act.wide = REV || act.has_wide;
                if (use_jit) {
                    act.key = shape_key(P, REV);
                    act.hash = fnv1a(act.key);
                    act.jit = find_shape(act.key, act.hash);
                }
                so.acts.push_back(std::move(act));
            }
        } catch (...) {
            so.err = std::current_exception();
        }
    };
    {
        HostAcc ha_f(&t_fuse); // fuse + lower + key, wall time of the pipeline
        StageJob job(stages.size(), prepare);
        for (size_t si = 0; si < stages.size(); ++si) {
            job.wait_for(si);
            StageOut &so = outs[si];
            if (so.err) std::rethrow_exception(so.err);
            const int shift = (int)slots.scale.size();
            slots.scale.insert(slots.scale.end(), so.slots.scale.begin(), so.slots.scale.end());
            slots.dst.insert(slots.dst.end(), so.slots.dst.begin(), so.slots.dst.end());
            for (Action &act : so.acts) {
                if (act.P) act.P->slot_begin += shift;
                if (use_jit && act.P && !act.jit) batching = true; // compile later, with the other misses
                if (batching) pending.push_back(std::move(act));
                else {
                    HostAcc ha(&t_issue);
                    issue(act);
                }
            }
        }
    }
    if (!pending.empty()) {
        // compile the missing structures (distinct ones, in parallel), then issue
        std::vector<std::string> srcs;
        std::vector<size_t> which;
        std::vector<std::pair<bool, bool>> flags;
        std::vector<double> fpas;
        std::vector<int> xts;
        std::unordered_map<uint64_t, size_t> first;
        for (size_t i = 0; i < pending.size(); ++i) {
            Action &act = pending[i];
            if (!act.P || act.hash == 0) continue;
            if ((act.jit = find_shape(act.key, act.hash))) continue;
            if (first.count(act.hash)) continue;
            bool sp = false, pb = REV;
            double fpa = 0;
            int xt = 1;
            std::string src = REV ? jit_reverse_source(*act.P, &sp, &fpa, &xt) : jit_forward_source(*act.P, &sp, &pb, &fpa);
            if (!src.empty()) src = instrument_checks(src, pn, TS, std::max(act.P->npool, 1));
            if (src.empty()) {
                // not specialisable: remember that (no kernel), stay on the interpreter
                std::lock_guard<std::mutex> lk(g_shape_mu);
                g_shapes[act.hash].key = act.key;
                continue;
            }
            first[act.hash] = i;
            if (const char *dump = std::getenv("VQB_JIT_DUMP")) {
                // development aid: the lowered program (regenerate the source on
                // the host with vqb_debug_jit_source) and the source itself
                char name[512];
                std::snprintf(name, sizeof name, "%s/%s_%s_%016llx", dump, REV ? "R" : "F", VQB_RS_STR,
                              (unsigned long long)act.hash);
                if (FILE *f = std::fopen((std::string(name) + ".params").c_str(), "wb")) {
                    std::fwrite(act.P.get(), sizeof(RParams), 1, f);
                    std::fclose(f);
                }
                if (FILE *f = std::fopen((std::string(name) + ".cu").c_str(), "w")) {
                    std::fwrite(src.data(), 1, src.size(), f);
                    std::fclose(f);
                }
            }
            srcs.push_back(std::move(src));
            flags.emplace_back(sp, pb);
            fpas.push_back(fpa);
            xts.push_back(xt);
            which.push_back(i);
        }
        if (!srcs.empty()) {
            const auto ks = jit::get(srcs, REV ? "vqb_rev" : "vqb_stage");
            std::lock_guard<std::mutex> lk(g_shape_mu);
            for (size_t k = 0; k < which.size(); ++k) {
                const Action &act = pending[which[k]];
                JitShape &sh = g_shapes[act.hash];
                sh.key = act.key;
                sh.k = ks[k];
                sh.spool = flags[k].first;
                sh.per_block = flags[k].second;
                sh.flops_per_amp = fpas[k];
                sh.xtiles = xts[k];
            }
        }
        for (Action &act : pending) {
            if (act.P && act.hash != 0 && !act.jit) act.jit = find_shape(act.key, act.hash);
            issue(act);
        }
    }
    if (merged_sums && any_jit_slots) {
        // slots of interpreter launches or fallback steps have no tile partials:
        // their rows were zeroed with the buffer and add nothing
        const ProfMark pf2 = prof_begin(st);
        k_slot_sums<<<dim3(total_slots, 1), 256, 0, st>>>(static_cast<const double *>(m_jpartial.p), ntiles,
                                                         static_cast<double *>(m_slotsum.p));
        check_launch("k_slot_sums", pf2);
    }
    if (REV && total_slots > 0) {
        wait_issue_gate();
        if ((int)slots.scale.size() != total_slots) raise(VQB_ERR_INTERNAL, "gradient slot mismatch");
        m_slots.ensure((sizeof(double) + 2 * sizeof(long long)) * total_slots);
        const std::vector<long long> links = slot_links(slots.dst);
        VQB_CUDA(cudaMemcpyAsync(m_slots.p, slots.scale.data(), sizeof(double) * total_slots,
                                 cudaMemcpyHostToDevice, st));
        VQB_CUDA(cudaMemcpyAsync(static_cast<char *>(m_slots.p) + sizeof(double) * total_slots,
                                 slots.dst.data(), sizeof(long long) * total_slots,
                                 cudaMemcpyHostToDevice, st));
        VQB_CUDA(cudaMemcpyAsync(static_cast<char *>(m_slots.p) +
                                     (sizeof(double) + sizeof(long long)) * total_slots,
                                 links.data(), sizeof(long long) * total_slots, cudaMemcpyHostToDevice, st));
        const ProfMark pf_ = prof_begin(st);
        k_grads<<<(total_slots + 127) / 128, 128, 0, st>>>(
            static_cast<const double *>(m_partial.p), partial_rows_used ? grid : 0, total_slots,
            static_cast<const double *>(m_slots.p),
            reinterpret_cast<const long long *>(static_cast<char *>(m_slots.p) +
                                                sizeof(double) * total_slots),
            reinterpret_cast<const long long *>(static_cast<char *>(m_slots.p) +
                                                (sizeof(double) + sizeof(long long)) * total_slots),
            total_slots, static_cast<const double *>(m_slotsum.p), dgrads);
        check_launch("k_grads", pf_);
    }
    // no synchronisation: kernel parameters are copied at launch and the
    // pageable slot vectors are staged by cudaMemcpyAsync before it returns,
    // so the caller's next host work overlaps this program on the device
}

} // namespace

bool regstage_available(int pn) { return pn >= K + 2; }

// Host-only: the specialised source for a dumped lowered program (VQB_JIT_DUMP).
std::string debug_jit_source(const void *params, size_t nbytes, bool rev, double *flops) {
    if (nbytes != sizeof(RParams)) raise(VQB_ERR_SIZE, "params blob size mismatch");
    auto P = std::make_unique<RParams>();
    std::memcpy(P.get(), params, sizeof(RParams));
    bool sp = false, pb = false;
    return rev ? jit_reverse_source(*P, &sp, flops, nullptr) : jit_forward_source(*P, &sp, &pb, flops);
}

void run_program_reg(DeviceState *s, const std::vector<Gate> &prog) {
    std::vector<FusedOp> fops;
    fops.reserve(prog.size());
    {
        HostTimer ht("analyse_gate x n");
        fops.resize(prog.size());
        parallel_chunks(prog.size(), 96, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) fops[i] = analyse_gate(prog[i]);
        });
    }
    run_reg<false>(s, nullptr, fops, nullptr, [&](const FusedOp &f) {
        apply_gate_fast(s->amps, s->pn, f.gate, s->stream);
    });
}

void run_reverse_reg(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog,
                     double *dgrads) {
    HostTimer ht("run_reverse_reg (analyse+run)");
    std::vector<FusedOp> fops;
    fops.reserve(prog.size());
    fops.resize(prog.size());
    parallel_chunks(prog.size(), 96, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            fops[i] = analyse_rev(prog[i]);
            if (fops[i].np > 0 && fops[i].nt > 2) fops[i].fusable = false;
        }
    });
    run_reg<true>(phi, psi, fops, dgrads, [&](const FusedOp &f) {
        const RevOp &r = *f.rev;
        if (r.dmats.empty()) {
            apply_gate_fast(phi->amps, phi->pn, r.phi_op, phi->stream);
            apply_gate_fast(psi->amps, psi->pn, r.psi_op, phi->stream);
        } else {
            reverse_step_async(phi->amps, psi->amps, phi->pn, r.phi_op.pos, r.phi_op.m,
                               r.phi_op.mat, r.dmats, phi, nullptr, dgrads + r.grad_base, r.scale);
        }
    });
}

} // namespace VQB_RS_NS
} // namespace vqb
