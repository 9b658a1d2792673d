// Fused tile executor: one HBM pass per stage.
//
// A stage (plan.hpp) fixes k tile bits. The persistent kernel walks the
// 2^(pn-k) tiles; for each it loads the 2^k amplitudes whose non-tile bits
// equal the tile's base index into shared memory (runs of >= 8 contiguous
// amplitudes = 128-B lines, since the lowest 3 bits are always tile bits),
// applies every operation of the stage in order on the shared-memory copy,
// and writes the tile back. Condition bits (controls / diagonal phases) are
// read from the global index, so they need not be tile bits.
//
// Shared-memory layout: tile bits are placed at local (shared-memory) bit
// positions by ascending use count, so the bits the stage's operations mix
// are the high local bits and consecutive threads touch consecutive 16-B
// words (no bank conflicts); the global<->shared mapping is applied once per
// tile when loading and storing.
//
// The adjoint variant keeps a phi tile and a psi tile and runs the reverse
// sweep (reverse_sweep_step kernels.hpp:659-697) on both; every gradient
// contribution Re <psi| D_p |phi> is reduced per warp into a per-block
// shared-memory slot, written as a per-block partial, and summed over blocks
// in fixed order by a final kernel (deterministic for a fixed grid).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"

namespace vqb {

void apply_gate_fast(double2 *a, int pn, const Gate &g, cudaStream_t st);

namespace {

constexpr int kT = 256;      // threads per block
constexpr int kTBits = 8;    // log2(kT)
constexpr int kMaxStageOps = 2 * kMaxPlanOps + 1;

enum : int { OP_DENSE = 0, OP_PARAM = 1, OP_DIAG_BATCH = 2 };

struct DevOp {
    int type;          // OP_*
    int nt, nc, np;
    int pair;          // psi uses its own matrices
    int count;         // OP_DIAG_BATCH: number of following member ops
    int tb[kMaxMix];   // local bit of each mixing bit (sub-matrix order)
    int ct[kMaxCond];  // local bit of each condition bit, -1 if outside the tile
    int cg[kMaxCond];  // global bit of each condition bit
    unsigned mat_phi, mat_psi, mat_d;  // offsets into the matrix pool (double2)
    unsigned long long id_phi, id_psi; // bit c set: sub-matrix c is the identity
    unsigned nz;       // nt <= 2, uniform sub-matrix: bit (r + s*D) = entry nonzero
    unsigned idrow;    // nt <= 2, uniform sub-matrix: bit r = row r is e_r (skip)
    int slot;          // first gradient slot of this stage (param ops)
    int uniform;       // all condition bits outside the tile
    int sync;          // a block barrier is needed before this op
    int pad_;
};

struct StageArgs {
    int k;
    int bits[24];            // tile bits ascending (global positions)
    int lbit[24];            // local (shared-memory) bit of bits[i]
    unsigned long long ntiles;
    int op_begin, op_count;
    int nslots;              // gradient slots used by this stage
    int slot_begin;          // global gradient column of slot 0
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// Re(conj(a) * b)
__device__ __forceinline__ double re_cjmul(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }

__device__ __forceinline__ unsigned long long expand_bits(unsigned long long c, const int *bits,
                                                          int k) {
    for (int i = 0; i < k; ++i) {
        const int s = bits[i];
        c = ((c >> s) << (s + 1)) | (c & ((1ull << s) - 1));
    }
    return c;
}

template <int NT>
__device__ __forceinline__ int insert_zeros(int g, const int *sorted) {
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        const int s = sorted[i];
        g = ((g >> s) << (s + 1)) | (g & ((1 << s) - 1));
    }
    return g;
}

__device__ __forceinline__ int cond_value(const DevOp &op, int local, int cuni) {
    int c = cuni;
#pragma unroll
    for (int i = 0; i < kMaxCond; ++i)
        if (i < op.nc && op.ct[i] >= 0) c |= ((local >> op.ct[i]) & 1) << i;
    return c;
}

__device__ __forceinline__ int cond_uniform(const DevOp &op, unsigned long long base) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < kMaxCond; ++i)
        if (i < op.nc && op.ct[i] < 0) c |= (int)((base >> op.cg[i]) & 1) << i;
    return c;
}

template <int NT> struct Geometry {
    static constexpr int D = 1 << NT;
    int sorted[NT > 0 ? NT : 1];
    int off[D];
    __device__ __forceinline__ explicit Geometry(const DevOp &op) {
#pragma unroll
        for (int i = 0; i < NT; ++i) sorted[i] = op.tb[i];
#pragma unroll
        for (int i = 0; i < NT; ++i)
#pragma unroll
            for (int j = 0; j + 1 < NT - i; ++j)
                if (sorted[j] > sorted[j + 1]) {
                    const int x = sorted[j];
                    sorted[j] = sorted[j + 1];
                    sorted[j + 1] = x;
                }
#pragma unroll
        for (int r = 0; r < D; ++r) {
            int o = 0;
#pragma unroll
            for (int i = 0; i < NT; ++i)
                if (r >> i & 1) o += 1 << op.tb[i];
            off[r] = o;
        }
    }
};

// Dense/sparse application of one nt <= 2 operation whose sub-matrix is the
// same for the whole tile: the matrix lives in registers, structural zeros
// and identity rows are skipped (uniform branches).
template <int NT>
__device__ __forceinline__ void apply_uniform(double2 *__restrict__ t, const DevOp &op,
                                              const double2 *__restrict__ M, int tsize) {
    constexpr int D = 1 << NT;
    constexpr int U = 1; // groups in flight per thread (more ILP spills registers)
    const Geometry<NT> G(op);
    double2 m[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) m[i] = M[i];
    const unsigned nz = op.nz, idrow = op.idrow;
    const int groups = tsize >> NT;
    for (int g0 = threadIdx.x; g0 < groups; g0 += kT * U) {
        double2 in[U][D];
        int b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int g = g0 + u * kT;
            b[u] = g < groups ? insert_zeros<NT>(g, G.sorted) : -1;
            if (b[u] >= 0) {
#pragma unroll
                for (int r = 0; r < D; ++r) in[u][r] = t[b[u] + G.off[r]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (b[u] < 0) continue;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                if (idrow >> r & 1) continue;
                double2 acc = make_double2(0, 0);
#pragma unroll
                for (int s = 0; s < D; ++s)
                    if (nz >> (r + s * D) & 1) acc = cfma(m[r + s * D], in[u][s], acc);
                t[b[u] + G.off[r]] = acc;
            }
        }
    }
}

// General application (condition bits inside the tile select the sub-matrix
// per group, or nt >= 3): matrices read through L1.
template <int NT>
__device__ __forceinline__ void apply_general(double2 *__restrict__ t, const DevOp &op,
                                              const double2 *__restrict__ pool, unsigned mat,
                                              unsigned long long ident, int tsize, int cuni) {
    constexpr int D = 1 << NT;
    const Geometry<NT> G(op);
    const int groups = tsize >> NT;
    for (int g = threadIdx.x; g < groups; g += kT) {
        const int b = insert_zeros<NT>(g, G.sorted);
        const int c = cond_value(op, b, cuni);
        if ((ident >> c) & 1) continue;
        const double2 *__restrict__ M = pool + mat + (size_t)c * D * D;
        double2 in[D];
#pragma unroll
        for (int r = 0; r < D; ++r) in[r] = t[b + G.off[r]];
#pragma unroll(NT <= 2 ? 4 : 1)
        for (int r = 0; r < D; ++r) {
            double2 acc = cmul(M[r], in[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) acc = cfma(M[r + s * D], in[s], acc);
            t[b + G.off[r]] = acc;
        }
    }
}

__device__ __forceinline__ void apply_any(double2 *t, const DevOp &op, const double2 *pool,
                                          bool psi_side, int tsize, int cuni) {
    const bool ps = psi_side && op.pair;
    const unsigned mat = ps ? op.mat_psi : op.mat_phi;
    const unsigned long long ident = ps ? op.id_psi : op.id_phi;
    if (op.uniform && op.nt <= 2 && !ps) {
        if ((ident >> cuni) & 1) return;
        const double2 *M = pool + mat + (size_t)cuni * (1 << (2 * op.nt));
        switch (op.nt) {
        case 0: apply_uniform<0>(t, op, M, tsize); return;
        case 1: apply_uniform<1>(t, op, M, tsize); return;
        default: apply_uniform<2>(t, op, M, tsize); return;
        }
    }
    switch (op.nt) {
    case 0: apply_general<0>(t, op, pool, mat, ident, tsize, cuni); break;
    case 1: apply_general<1>(t, op, pool, mat, ident, tsize, cuni); break;
    case 2: apply_general<2>(t, op, pool, mat, ident, tsize, cuni); break;
    case 3: apply_general<3>(t, op, pool, mat, ident, tsize, cuni); break;
    default: apply_general<4>(t, op, pool, mat, ident, tsize, cuni); break;
    }
}

// A run of diagonal operations: one shared-memory pass, phases multiplied in
// registers (member ops follow the header in sops[]).
__device__ __forceinline__ void apply_diag_batch(double2 *__restrict__ t, const DevOp *sops,
                                                 int count, const double2 *__restrict__ pool,
                                                 bool psi_side, int tsize,
                                                 unsigned long long base) {
    for (int e = threadIdx.x; e < tsize; e += kT) {
        double2 ph = make_double2(1, 0);
        bool any = false;
        for (int i = 0; i < count; ++i) {
            const DevOp &op = sops[i];
            const int c = cond_value(op, e, cond_uniform(op, base));
            const bool ps = psi_side && op.pair;
            if (((ps ? op.id_psi : op.id_phi) >> c) & 1) continue;
            const double2 v = pool[(ps ? op.mat_psi : op.mat_phi) + c];
            ph = any ? cmul(ph, v) : v;
            any = true;
        }
        if (any) t[e] = cmul(ph, t[e]);
    }
}

// Param op of the reverse sweep on the two tiles; accumulates this thread's
// contributions Re <psi| D_p |phi'> (p < np) in acc[].
template <int NT>
__device__ __forceinline__ void param_op(double2 *__restrict__ tf, double2 *__restrict__ tg,
                                         const DevOp &op, const double2 *__restrict__ pool,
                                         int tsize, int cuni, double *acc) {
    constexpr int D = 1 << NT;
    const Geometry<NT> G(op);
    const int groups = tsize >> NT;
    const size_t blk = (size_t)D * D;
    const size_t nsub = (size_t)1 << op.nc;
    // One register array: phi group -> inv phi (written back), re-read as w
    // for the derivative contractions against psi (read from shared memory),
    // then the psi group -> inv psi.
    for (int g = threadIdx.x; g < groups; g += kT) {
        const int b = insert_zeros<NT>(g, G.sorted);
        const int c = op.nc ? cond_value(op, b, cuni) : 0;
        const double2 *__restrict__ M = pool + op.mat_phi + c * blk;
        double2 v[D];
#pragma unroll
        for (int r = 0; r < D; ++r) v[r] = tf[b + G.off[r]];
#pragma unroll(NT <= 2 ? 4 : 1)
        for (int r = 0; r < D; ++r) {
            double2 x = cmul(M[r], v[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) x = cfma(M[r + s * D], v[s], x);
            tf[b + G.off[r]] = x;
        }
#pragma unroll
        for (int r = 0; r < D; ++r) v[r] = tf[b + G.off[r]];
#pragma unroll
        for (int p = 0; p < VQB_MAX_PARAMS; ++p) {
            if (p >= op.np) break;
            const double2 *__restrict__ Dm = pool + op.mat_d + (p * nsub + c) * blk;
            double a = 0;
#pragma unroll(NT <= 2 ? 4 : 1)
            for (int r = 0; r < D; ++r) {
                double2 x = cmul(Dm[r], v[0]);
#pragma unroll
                for (int s = 1; s < D; ++s) x = cfma(Dm[r + s * D], v[s], x);
                a += re_cjmul(tg[b + G.off[r]], x);
            }
            acc[p] += a;
        }
#pragma unroll
        for (int r = 0; r < D; ++r) v[r] = tg[b + G.off[r]];
#pragma unroll(NT <= 2 ? 4 : 1)
        for (int r = 0; r < D; ++r) {
            double2 x = cmul(M[r], v[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) x = cfma(M[r + s * D], v[s], x);
            tg[b + G.off[r]] = x;
        }
    }
}

__device__ __forceinline__ double2 sel4(const double2 (&v)[4], int c) {
    double2 r = v[0];
    if (c == 1) r = v[1];
    if (c == 2) r = v[2];
    if (c == 3) r = v[3];
    return r;
}

// Fast path for the common one-parameter reverse step (rotations): at most
// four sub-matrix entries for inv and D (nt = 0 with <= 2 condition bits, or
// nt = 1 without), held in registers; the group is never re-read.
template <int NT>
__device__ __forceinline__ double param_small(double2 *__restrict__ tf, double2 *__restrict__ tg,
                                              const DevOp &op, const double2 *__restrict__ pool,
                                              int tsize, int cuni) {
    constexpr int D = 1 << NT;
    constexpr int U = 1;
    const Geometry<NT> G(op);
    const int nent = (1 << op.nc) * D * D;
    double2 mi[4], md[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        mi[i] = i < nent ? pool[op.mat_phi + i] : make_double2(0, 0);
        md[i] = i < nent ? pool[op.mat_d + i] : make_double2(0, 0);
    }
    double a = 0;
    const int groups = tsize >> NT;
    for (int g0 = threadIdx.x; g0 < groups; g0 += kT * U) {
        double2 f[U][D], h[U][D];
        int b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int g = g0 + u * kT;
            b[u] = g < groups ? insert_zeros<NT>(g, G.sorted) : -1;
            if (b[u] >= 0) {
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    f[u][r] = tf[b[u] + G.off[r]];
                    h[u][r] = tg[b[u] + G.off[r]];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (b[u] < 0) continue;
            if constexpr (NT == 0) {
                const int c = op.nc ? cond_value(op, b[u], cuni) : 0;
                const double2 m = sel4(mi, c), d = sel4(md, c);
                const double2 w = cmul(m, f[u][0]);
                tf[b[u]] = w;
                a += re_cjmul(h[u][0], cmul(d, w));
                tg[b[u]] = cmul(m, h[u][0]);
            } else {
                const double2 w0 = cfma(mi[2], f[u][1], cmul(mi[0], f[u][0]));
                const double2 w1 = cfma(mi[3], f[u][1], cmul(mi[1], f[u][0]));
                tf[b[u] + G.off[0]] = w0;
                tf[b[u] + G.off[1]] = w1;
                const double2 x0 = cfma(md[2], w1, cmul(md[0], w0));
                const double2 x1 = cfma(md[3], w1, cmul(md[1], w0));
                a += re_cjmul(h[u][0], x0) + re_cjmul(h[u][1], x1);
                tg[b[u] + G.off[0]] = cfma(mi[2], h[u][1], cmul(mi[0], h[u][0]));
                tg[b[u] + G.off[1]] = cfma(mi[3], h[u][1], cmul(mi[1], h[u][0]));
            }
        }
    }
    return a;
}

template <bool REV>
__global__ void __launch_bounds__(kT, 2) k_stage(double2 *__restrict__ phi, double2 *__restrict__ psi,
                                                 const DevOp *__restrict__ ops,
                                                 const double2 *__restrict__ pool,
                                                 const __grid_constant__ StageArgs S,
                                                 double *__restrict__ partial, int partial_ld) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tsize = 1 << S.k;
    double2 *tf = reinterpret_cast<double2 *>(smem_raw);
    double2 *tg = tf + (REV ? tsize : 0);
    DevOp *sops = reinterpret_cast<DevOp *>(tf + (REV ? 2 : 1) * tsize);
    const int nhi = tsize > kT ? tsize / kT : 1;
    unsigned long long *dep_hi = reinterpret_cast<unsigned long long *>(sops + S.op_count);
    int *sdep_hi = reinterpret_cast<int *>(dep_hi + nhi);
    double *pacc = reinterpret_cast<double *>(sdep_hi + ((nhi + 1) & ~1)); // [nslots][nwarps]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int nw = kT / 32;

    // stage ops -> shared memory
    {
        const int words = S.op_count * (int)(sizeof(DevOp) / 4);
        const int *src = reinterpret_cast<const int *>(ops + S.op_begin);
        int *dst = reinterpret_cast<int *>(sops);
        for (int i = threadIdx.x; i < words; i += kT) dst[i] = src[i];
    }
    // deposit tables: global-order tile index j = t + kT*s ->
    //   global offset my_lo | dep_hi[s], shared slot my_slo | sdep_hi[s]
    const int tb_lo = tsize < kT ? S.k : kTBits;
    unsigned long long my_lo = 0;
    int my_slo = 0;
    for (int i = 0; i < tb_lo; ++i)
        if (threadIdx.x >> i & 1) {
            my_lo |= 1ull << S.bits[i];
            my_slo |= 1 << S.lbit[i];
        }
    for (int s = threadIdx.x; s < nhi; s += kT) {
        unsigned long long o = 0;
        int so = 0;
        for (int i = tb_lo; i < S.k; ++i)
            if ((s >> (i - tb_lo)) & 1) {
                o |= 1ull << S.bits[i];
                so |= 1 << S.lbit[i];
            }
        dep_hi[s] = o;
        sdep_hi[s] = so;
    }
    if (REV)
        for (int i = threadIdx.x; i < S.nslots * nw; i += kT) pacc[i] = 0;
    __syncthreads();
    const bool active = threadIdx.x < tsize;

    for (unsigned long long tile = blockIdx.x; tile < S.ntiles; tile += gridDim.x) {
        const unsigned long long base = expand_bits(tile, S.bits, S.k);
        if (active) {
#pragma unroll 8
            for (int s = 0; s < nhi; ++s) {
                const unsigned long long gi = base | my_lo | dep_hi[s];
                const int li = my_slo | sdep_hi[s];
                tf[li] = phi[gi];
                if (REV) tg[li] = psi[gi];
            }
        }
        __syncthreads();
        for (int o = 0; o < S.op_count; ++o) {
            const DevOp &op = sops[o];
            if (op.sync) __syncthreads();
            if (op.type == OP_DIAG_BATCH) {
                apply_diag_batch(tf, sops + o + 1, op.count, pool, false, tsize, base);
                if (REV) apply_diag_batch(tg, sops + o + 1, op.count, pool, true, tsize, base);
                o += op.count;
            } else if (!REV || op.type == OP_DENSE) {
                const int cuni = op.nc ? cond_uniform(op, base) : 0;
                apply_any(tf, op, pool, false, tsize, cuni);
                if (REV) apply_any(tg, op, pool, true, tsize, cuni);
            } else {
                const int cuni = op.nc ? cond_uniform(op, base) : 0;
                double acc[VQB_MAX_PARAMS] = {0, 0, 0, 0, 0};
                const bool small = op.np == 1 && op.nt <= 1 && ((1 << op.nc) << (2 * op.nt)) <= 4;
                if (small) {
                    acc[0] = op.nt == 0 ? param_small<0>(tf, tg, op, pool, tsize, cuni)
                                        : param_small<1>(tf, tg, op, pool, tsize, cuni);
                } else {
                    switch (op.nt) {
                    case 0: param_op<0>(tf, tg, op, pool, tsize, cuni, acc); break;
                    case 1: param_op<1>(tf, tg, op, pool, tsize, cuni, acc); break;
                    case 2: param_op<2>(tf, tg, op, pool, tsize, cuni, acc); break;
                    case 3: param_op<3>(tf, tg, op, pool, tsize, cuni, acc); break;
                    default: param_op<4>(tf, tg, op, pool, tsize, cuni, acc); break;
                    }
                }
#pragma unroll
                for (int p = 0; p < VQB_MAX_PARAMS; ++p) {
                    if (p >= op.np) break;
                    double v = acc[p];
#pragma unroll
                    for (int sh = 16; sh > 0; sh >>= 1) v += __shfl_down_sync(0xffffffffu, v, sh);
                    if (lane == 0) pacc[(op.slot + p) * nw + warp] += v;
                }
            }
        }
        __syncthreads();
        if (active) {
#pragma unroll 8
            for (int s = 0; s < nhi; ++s) {
                const unsigned long long gi = base | my_lo | dep_hi[s];
                const int li = my_slo | sdep_hi[s];
                phi[gi] = tf[li];
                if (REV) psi[gi] = tg[li];
            }
        }
        __syncthreads();
    }
    if (REV) {
        for (int s = threadIdx.x; s < S.nslots; s += kT) {
            double v = 0;
            for (int w = 0; w < nw; ++w) v += pacc[s * nw + w];
            partial[(size_t)blockIdx.x * partial_ld + S.slot_begin + s] = v;
        }
    }
}

// grads[dst] += sum over the slots of that destination (chained in slot order
// by slot_links) of scale[j] * sum_b partial[b][j] (fixed block order): one
// thread per destination, deterministic
__global__ void k_reduce_grads(const double *__restrict__ partial, int nblocks, int ld,
                               const double *__restrict__ scale, const long long *__restrict__ dst,
                               const long long *__restrict__ link, int ncols,
                               double *__restrict__ grads) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols || !(link[j] & 1)) return;
    double acc = 0;
    for (long long k = j; k >= 0; k = link[k] >> 1) {
        double v = 0;
        for (int b = 0; b < nblocks; ++b) v += partial[(size_t)b * ld + k];
        acc += scale[k] * v;
    }
    grads[dst[j]] += acc;
}

bool is_identity(const cplx *m, int d) {
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c)
            if (m[r + c * d] != (r == c ? cplx(1) : cplx(0))) return false;
    return true;
}

int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

int tile_bits_for(int pn, bool rev) {
    const int kmax = env_int(rev ? "VQB_TILE_BITS_REV" : "VQB_TILE_BITS", rev ? 11 : 12);
    if (pn <= 12) return std::min(pn, kmax);
    return std::min(kmax, std::max(10, pn - 9));
}


size_t smem_bytes(bool rev, int k, int nops, int nslots) {
    const int tsize = 1 << k;
    const int nhi = tsize > kT ? tsize / kT : 1;
    return (size_t)(rev ? 2 : 1) * tsize * sizeof(double2) + (size_t)nops * sizeof(DevOp) +
           (size_t)nhi * 8 + (size_t)((nhi + 1) & ~1) * 4 + (size_t)nslots * (kT / 32) * 8;
}

// One stage's device ops (after block fusion), appended to dops/pool.
template <bool REV>
void lower_stage(const Stage &sg, const std::vector<FusedOp> &sops, std::vector<DevOp> &dops,
                 std::vector<double2> &pool, StageArgs &a, std::vector<double> &slot_scale,
                 std::vector<long long> &slot_dst) {
    auto push_pool = [&](const cvec &v) {
        const unsigned off = (unsigned)pool.size();
        for (const auto &x : v) pool.push_back(make_double2(x.real(), x.imag()));
        return off;
    };
    // local bit order: least-mixed tile bits at the low shared-memory bits
    std::vector<int> use(sg.k, 0);
    for (const FusedOp &f : sops)
        for (int i = 0; i < f.nt; ++i)
            for (int j = 0; j < sg.k; ++j)
                if (sg.bits[j] == f.mix[i]) use[j] += 1 << (2 * f.nt);
    std::vector<int> order(sg.k);
    for (int j = 0; j < sg.k; ++j) order[j] = j;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return use[x] < use[y]; });
    for (int l = 0; l < sg.k; ++l) a.lbit[order[l]] = l;
    auto local_of = [&](int gbit) {
        for (int j = 0; j < sg.k; ++j)
            if (sg.bits[j] == gbit) return a.lbit[j];
        return -1;
    };

    a.op_begin = (int)dops.size();
    a.slot_begin = (int)slot_scale.size();
    int slot = 0;
    int batch_hdr = -1; // index of the open diagonal batch header
    bool first = true, prev_tl = false;
    for (const FusedOp &f : sops) {
        DevOp d{};
        d.nt = f.nt;
        d.nc = f.nc;
        d.np = REV ? f.np : 0;
        d.pair = f.pair ? 1 : 0;
        d.type = d.np > 0 ? OP_PARAM : OP_DENSE;
        for (int i = 0; i < f.nt; ++i) d.tb[i] = local_of(f.mix[i]);
        d.uniform = 1;
        for (int i = 0; i < f.nc; ++i) {
            d.ct[i] = local_of(f.cnd[i]);
            d.cg[i] = f.cnd[i];
            if (d.ct[i] >= 0) d.uniform = 0;
        }
        const int D = 1 << f.nt, dd = D * D;
        d.mat_phi = push_pool(f.sub_phi);
        for (int c = 0; c < (1 << f.nc); ++c)
            if (is_identity(&f.sub_phi[size_t(c) * dd], D)) d.id_phi |= 1ull << c;
        if (f.pair) {
            d.mat_psi = push_pool(f.sub_psi);
            for (int c = 0; c < (1 << f.nc); ++c)
                if (is_identity(&f.sub_psi[size_t(c) * dd], D)) d.id_psi |= 1ull << c;
        }
        if (f.nt <= 2 && d.uniform) {
            // sparsity of the sub-matrices (union over condition values)
            for (int c = 0; c < (1 << f.nc); ++c)
                for (int r = 0; r < D; ++r)
                    for (int s = 0; s < D; ++s)
                        if (f.sub_phi[size_t(c) * dd + r + s * D] != cplx(0)) d.nz |= 1u << (r + s * D);
            d.idrow = (1u << D) - 1;
            for (int c = 0; c < (1 << f.nc); ++c) {
                if (d.id_phi >> c & 1) continue;
                for (int r = 0; r < D; ++r)
                    for (int s = 0; s < D; ++s)
                        if (f.sub_phi[size_t(c) * dd + r + s * D] != (r == s ? cplx(1) : cplx(0)))
                            d.idrow &= ~(1u << r);
            }
        }
        if (d.np > 0) {
            d.mat_d = push_pool(f.sub_d);
            d.id_phi = 0; // the fused param step always runs
            d.slot = slot;
            for (int p = 0; p < f.np; ++p) {
                slot_scale.push_back(f.scale);
                slot_dst.push_back(f.grad_base + p);
            }
            slot += f.np;
        }
        // Barrier elision: an op is thread-local when every thread touches only
        // the elements whose low kTBits local bits equal its thread index
        // (all mixing bits at local bits >= kTBits, or none); two consecutive
        // thread-local ops need no barrier between them.
        bool tl = (1 << sg.k) >= kT;
        for (int i = 0; i < f.nt; ++i) tl = tl && d.tb[i] >= kTBits;
        const bool diag = d.type == OP_DENSE && d.nt == 0;
        if (diag) {
            if (batch_hdr < 0) {
                DevOp h{};
                h.type = OP_DIAG_BATCH;
                h.count = 0;
                h.sync = (first || !(prev_tl && tl)) && !first ? 1 : 0;
                batch_hdr = (int)dops.size();
                dops.push_back(h);
                first = false;
                prev_tl = tl;
            }
            dops[batch_hdr].count += 1;
        } else {
            batch_hdr = -1;
            d.sync = (!first && !(prev_tl && tl)) ? 1 : 0;
            first = false;
            prev_tl = tl;
        }
        dops.push_back(d);
    }
    a.op_count = (int)dops.size() - a.op_begin;
    a.nslots = slot;
}

// Uploads ops + pool, runs the stages; unfusable ops go through `fallback`.
template <bool REV, typename Fallback>
void execute(DeviceState *sphi, DeviceState *spsi, const std::vector<FusedOp> &fops,
             const std::vector<Stage> &stages, int pn, double *dgrads, Fallback &&fallback) {
    cudaStream_t st = sphi->stream;
    std::vector<DevOp> dops;
    std::vector<double2> pool;
    std::vector<StageArgs> sargs(stages.size());
    std::vector<double> slot_scale;
    std::vector<long long> slot_dst;
    const int max_support = env_int("VQB_FUSE_QUBITS", 2);
    for (size_t i = 0; i < stages.size(); ++i) {
        const Stage &sg = stages[i];
        StageArgs &a = sargs[i];
        std::memset(&a, 0, sizeof a);
        if (!sg.fused) continue;
        a.k = sg.k;
        std::memcpy(a.bits, sg.bits, sizeof(a.bits));
        a.ntiles = 1ull << (pn - sg.k);
        std::vector<FusedOp> sops;
        if (max_support > 0) {
            sops = fuse_blocks(fops, sg.ops, max_support);
        } else {
            for (int idx : sg.ops) sops.push_back(fops[idx]);
        }
        lower_stage<REV>(sg, sops, dops, pool, a, slot_scale, slot_dst);
        if (a.op_count > kMaxStageOps) raise(VQB_ERR_INTERNAL, "fused stage has too many ops");
    }
    static thread_local DevMem m_ops, m_pool, m_partial, m_slots;
    m_ops.ensure(sizeof(DevOp) * std::max<size_t>(dops.size(), 1));
    m_pool.ensure(sizeof(double2) * std::max<size_t>(pool.size(), 1));
    VQB_CUDA(cudaMemcpyAsync(m_ops.p, dops.data(), sizeof(DevOp) * dops.size(),
                             cudaMemcpyHostToDevice, st));
    VQB_CUDA(cudaMemcpyAsync(m_pool.p, pool.data(), sizeof(double2) * pool.size(),
                             cudaMemcpyHostToDevice, st));
    const int nslots_total = (int)slot_scale.size();

    // grid: persistent, fixed for the whole program
    int max_k = 0;
    size_t smem_max = 0;
    for (size_t i = 0; i < stages.size(); ++i)
        if (stages[i].fused) {
            max_k = std::max(max_k, sargs[i].k);
            smem_max = std::max(smem_max, smem_bytes(REV, sargs[i].k, sargs[i].op_count,
                                                     sargs[i].nslots));
        }
    if (smem_max > 227 * 1024) raise(VQB_ERR_INTERNAL, "fused stage exceeds shared memory");
    static bool attr_set[2] = {false, false};
    if (!attr_set[REV]) {
        VQB_CUDA(cudaFuncSetAttribute(k_stage<REV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
        attr_set[REV] = true;
    }
    int nsm = 148, dev = 0;
    VQB_CUDA(cudaGetDevice(&dev));
    VQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int per_sm = 1;
    VQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stage<REV>, kT,
                                                           std::max<size_t>(smem_max, 1)));
    per_sm = std::max(per_sm, 1);
    const unsigned long long max_tiles = max_k ? 1ull << (pn - max_k) : 1ull;
    const int grid = (int)std::min<unsigned long long>((unsigned long long)nsm * per_sm, max_tiles);
    if (REV && nslots_total > 0) {
        m_partial.ensure(sizeof(double) * (size_t)grid * nslots_total);
        m_slots.ensure((sizeof(double) + 2 * sizeof(long long)) * nslots_total);
        const std::vector<long long> links = slot_links(slot_dst);
        VQB_CUDA(cudaMemcpyAsync(m_slots.p, slot_scale.data(), sizeof(double) * nslots_total,
                                 cudaMemcpyHostToDevice, st));
        VQB_CUDA(cudaMemcpyAsync(static_cast<char *>(m_slots.p) + sizeof(double) * nslots_total,
                                 slot_dst.data(), sizeof(long long) * nslots_total,
                                 cudaMemcpyHostToDevice, st));
        VQB_CUDA(cudaMemcpyAsync(static_cast<char *>(m_slots.p) +
                                     (sizeof(double) + sizeof(long long)) * nslots_total,
                                 links.data(), sizeof(long long) * nslots_total,
                                 cudaMemcpyHostToDevice, st));
    }
    for (size_t i = 0; i < stages.size(); ++i) {
        if (!stages[i].fused) {
            fallback(fops[stages[i].ops[0]]);
            continue;
        }
        const StageArgs &a = sargs[i];
        if (a.op_count == 0) continue;
        // every block writes its partial columns, so REV stages with slots use the full grid
        const int g = (REV && a.nslots > 0) ? grid
                                            : (int)std::min<unsigned long long>(grid, a.ntiles);
        const ProfMark pf_ = prof_begin(st);
        k_stage<REV><<<g, kT, smem_bytes(REV, a.k, a.op_count, a.nslots), st>>>(
            sphi->amps, REV ? spsi->amps : nullptr, static_cast<const DevOp *>(m_ops.p),
            static_cast<const double2 *>(m_pool.p), a, static_cast<double *>(m_partial.p),
            nslots_total);
        check_launch(REV ? "k_stage_rev" : "k_stage", pf_);
    }
    if (REV && nslots_total > 0) {
        const ProfMark pf_ = prof_begin(st);
        k_reduce_grads<<<(nslots_total + 127) / 128, 128, 0, st>>>(
            static_cast<const double *>(m_partial.p), grid, nslots_total,
            static_cast<const double *>(m_slots.p),
            reinterpret_cast<const long long *>(static_cast<char *>(m_slots.p) +
                                                sizeof(double) * nslots_total),
            reinterpret_cast<const long long *>(static_cast<char *>(m_slots.p) +
                                                (sizeof(double) + sizeof(long long)) * nslots_total),
            nslots_total, dgrads);
        check_launch("k_reduce_grads", pf_);
    }
    // op / pool buffers are reused by the next call on this thread
    VQB_CUDA(cudaStreamSynchronize(st));
}

} // namespace

// register executors (regstage_impl.cuh), one namespace per geometry
#define VQB_DECLARE_REGSTAGE(ns)                                                            \
    namespace ns {                                                                          \
    bool regstage_available(int pn);                                                        \
    void run_program_reg(DeviceState *s, const std::vector<Gate> &prog);                    \
    void run_reverse_reg(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog, \
                         double *dgrads);                                                   \
    std::string debug_jit_source(const void *params, size_t nbytes, bool rev, double *flops); \
    }
VQB_DECLARE_REGSTAGE(rs16)
VQB_DECLARE_REGSTAGE(rs8)
#undef VQB_DECLARE_REGSTAGE

std::string debug_jit_source(int regs, const void *params, size_t nbytes, bool rev, double *flops) {
    return regs == 8 ? rs8::debug_jit_source(params, nbytes, rev, flops)
                     : rs16::debug_jit_source(params, nbytes, rev, flops);
}

namespace {
// register-executor geometry: VQB_REGS / VQB_REV_REGS = 8 or 16 amplitudes per
// thread (defaults: 16 for forward programs, 8 for adjoint sweeps)
bool use_rs8(bool rev, const DeviceState *s = nullptr) {
    const char *v = std::getenv(rev ? "VQB_REV_REGS" : "VQB_REGS");
    if (v && *v) return std::atoi(v) == 8;
    // density-matrix sweeps take 16 registers per state: their 4-bit channel
    // superoperators then run on register bits (ROp::inreg), no shared-memory
    // round trips; pure-state sweeps keep 8 (lighter, 4 blocks per SM)
    if (rev && s && s->mixed && std::getenv("VQB_WIDE_REGS") == nullptr) return false;
    if (rev && s && s->mixed) return std::atoi(std::getenv("VQB_WIDE_REGS")) == 0;
    return rev;
}
bool smem_forced() {
    const char *ex = std::getenv("VQB_EXECUTOR");
    return ex && std::strcmp(ex, "smem") == 0;
}
} // namespace

// One stage through the shared-memory executor (used by the register
// executor when a stage's program exceeds its parameter block).
void run_program_fused_smem_stage(DeviceState *s, const std::vector<FusedOp> &fops,
                                  const Stage &sg) {
    execute<false>(s, nullptr, fops, std::vector<Stage>{sg}, s->pn, nullptr,
                   [&](const FusedOp &f) { apply_gate_fast(s->amps, s->pn, f.gate, s->stream); });
}

void run_program_fused(DeviceState *s, const std::vector<Gate> &prog) {
    // register-resident executor for states of >= 2^12 amplitudes
    // (VQB_EXECUTOR=smem selects the shared-memory interpreter instead)
    if (!smem_forced()) {
        if (use_rs8(false) ? rs8::regstage_available(s->pn) : rs16::regstage_available(s->pn)) {
            if (use_rs8(false)) rs8::run_program_reg(s, prog);
            else rs16::run_program_reg(s, prog);
            return;
        }
    }
    std::vector<FusedOp> fops;
    fops.reserve(prog.size());
    for (const auto &g : prog) fops.push_back(analyse_gate(g));
    const int k = tile_bits_for(s->pn, false);
    const auto stages = plan_stages(fops, s->pn, k);
    execute<false>(s, nullptr, fops, stages, s->pn, nullptr, [&](const FusedOp &f) {
        apply_gate_fast(s->amps, s->pn, f.gate, s->stream);
    });
}

void run_reverse_fused(DeviceState *phi, DeviceState *psi, const std::vector<RevOp> &prog,
                       double *dgrads) {
    if (!smem_forced()) {
        const bool r8 = use_rs8(true, phi);
        if (r8 ? rs8::regstage_available(phi->pn) : rs16::regstage_available(phi->pn)) {
            if (r8) rs8::run_reverse_reg(phi, psi, prog, dgrads);
            else rs16::run_reverse_reg(phi, psi, prog, dgrads);
            return;
        }
    }
    std::vector<FusedOp> fops;
    fops.reserve(prog.size());
    for (const auto &r : prog) fops.push_back(analyse_rev(r));
    const int k = tile_bits_for(phi->pn, true);
    const auto stages = plan_stages(fops, phi->pn, k);
    wait_issue_gate();
    execute<true>(phi, psi, fops, stages, phi->pn, dgrads, [&](const FusedOp &f) {
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

} // namespace vqb
