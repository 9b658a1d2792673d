// Per-element kernels (the unfused path) and the deterministic reductions.
//
// Every kernel here streams the state once per call (HBM-bound, one
// complex128 = 16 B per access, 128-bit loads). Index math follows the
// reference's compressed-base scheme (kernels.hpp:101-169): a group base is a
// compressed index with the target bits inserted as zeros; group members are
// base + offsets[r] with offsets in listed-position order.
//
// Reductions are deterministic: a fixed grid (a function of the problem size
// only), a fixed in-block tree, per-block partials, and the last block to
// finish summing the partials in index order (mirrors the reference's
// segment-ordered sums, kernels.hpp:498-502,690-696).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>

#include "device.hpp"

namespace vqb {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a)*b + c
__device__ __forceinline__ double2 cjfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// Insert zero bits at ascending positions (expand_index kernels.hpp:116-122).
template <int M>
__device__ __forceinline__ uint64_t expand(uint64_t c, const int *sorted) {
#pragma unroll
    for (int k = 0; k < M; ++k) {
        const int s = sorted[k];
        c = ((c >> s) << (s + 1)) | (c & ((1ull << s) - 1));
    }
    return c;
}

__device__ __forceinline__ uint64_t expand_rt(uint64_t c, const int *sorted, int m) {
    for (int k = 0; k < m; ++k) {
        const int s = sorted[k];
        c = ((c >> s) << (s + 1)) | (c & ((1ull << s) - 1));
    }
    return c;
}

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t work, int threads = kThreads, unsigned cap = 148 * 16) {
    const uint64_t b = (work + threads - 1) / threads;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, cap));
}

// ------------------------------------------------------------------ launch accounting

// ------------------------------------------------------------------ dense m-qubit
template <int M> struct DenseArgs {
    int sorted[M];
    unsigned long long off[1 << M];
    double2 mat[(1 << M) * (1 << M)];
};

template <int M>
__global__ void __launch_bounds__(kThreads) k_dense(double2 *__restrict__ a, uint64_t groups,
                                                    const __grid_constant__ DenseArgs<M> A) {
    constexpr int D = 1 << M;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < groups; c += stride) {
        const uint64_t b = expand<M>(c, A.sorted);
        double2 in[D];
#pragma unroll
        for (int r = 0; r < D; ++r) in[r] = a[b + A.off[r]];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double2 acc = cmul(A.mat[r], in[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) acc = cfma(A.mat[r + s * D], in[s], acc);
            a[b + A.off[r]] = acc;
        }
    }
}

// m = 5, 6: matrix in global memory, group in local memory (rare fallback).
struct DenseBigArgs {
    int m;
    int sorted[VQB_MAX_POSITIONS];
    unsigned long long off[64];
};

template <int M>
__global__ void __launch_bounds__(128) k_dense_big(double2 *__restrict__ a, uint64_t groups,
                                                   const double2 *__restrict__ mat,
                                                   const __grid_constant__ DenseBigArgs A) {
    constexpr int D = 1 << M;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < groups; c += stride) {
        const uint64_t b = expand<M>(c, A.sorted);
        double2 in[D], out[D];
        for (int r = 0; r < D; ++r) in[r] = a[b + A.off[r]];
        for (int r = 0; r < D; ++r) {
            double2 acc = cmul(mat[r], in[0]);
            for (int s = 1; s < D; ++s) acc = cfma(mat[r + s * D], in[s], acc);
            out[r] = acc;
        }
        for (int r = 0; r < D; ++r) a[b + A.off[r]] = out[r];
    }
}

static void sorted_bits(const int *bits, int m, int *out) {
    std::copy(bits, bits + m, out);
    std::sort(out, out + m);
}

template <int M>
static void launch_dense_m(double2 *a, int pn, const int *bits, const cvec &mat, cudaStream_t st) {
    DenseArgs<M> A;
    sorted_bits(bits, M, A.sorted);
    for (int r = 0; r < (1 << M); ++r) {
        uint64_t o = 0;
        for (int k = 0; k < M; ++k)
            if ((r >> k) & 1) o += 1ull << bits[k];
        A.off[r] = o;
    }
    for (int i = 0; i < (1 << (2 * M)); ++i) A.mat[i] = make_double2(mat[i].real(), mat[i].imag());
    const uint64_t groups = 1ull << (pn - M);
    const ProfMark pf_ = prof_begin(st);
    k_dense<M><<<grid_for(groups), kThreads, 0, st>>>(a, groups, A);
    check_launch("k_dense", pf_);
}

template <int M>
static void launch_dense_big(double2 *a, int pn, const int *bits, const cvec &mat, cudaStream_t st) {
    DenseBigArgs A;
    A.m = M;
    sorted_bits(bits, M, A.sorted);
    for (int r = 0; r < (1 << M); ++r) {
        uint64_t o = 0;
        for (int k = 0; k < M; ++k)
            if ((r >> k) & 1) o += 1ull << bits[k];
        A.off[r] = o;
    }
    double2 *dm = nullptr;
    const size_t bytes = sizeof(double2) * mat.size();
    VQB_CUDA(cudaMallocAsync((void **)&dm, bytes, st));
    VQB_CUDA(cudaMemcpyAsync(dm, mat.data(), bytes, cudaMemcpyHostToDevice, st));
    const uint64_t groups = 1ull << (pn - M);
    const ProfMark pf_ = prof_begin(st);
    k_dense_big<M><<<grid_for(groups, 128), 128, 0, st>>>(a, groups, dm, A);
    check_launch("k_dense_big", pf_);
    VQB_CUDA(cudaFreeAsync(dm, st));
    VQB_CUDA(cudaStreamSynchronize(st)); // mat (host) must outlive the async copy
}

void launch_dense(double2 *a, int pn, const int *bits, int m, const cvec &mat, cudaStream_t st) {
    switch (m) {
    case 1: launch_dense_m<1>(a, pn, bits, mat, st); return;
    case 2: launch_dense_m<2>(a, pn, bits, mat, st); return;
    case 3: launch_dense_m<3>(a, pn, bits, mat, st); return;
    case 4: launch_dense_m<4>(a, pn, bits, mat, st); return;
    case 5: launch_dense_big<5>(a, pn, bits, mat, st); return;
    case 6: launch_dense_big<6>(a, pn, bits, mat, st); return;
    default: raise(VQB_ERR_UNSUPPORTED, "apply_matrix: at most 6 positions");
    }
}

// ------------------------------------------------------------------ permutations / phases
struct SparseArgs {
    int m;
    int sorted[3];
    unsigned long long base_add;
    unsigned long long delta;
    double2 phase;
};

// swap_pairs_range kernels.hpp:291-299: exact data moves (bit-exact).
__global__ void __launch_bounds__(kThreads) k_swap(double2 *__restrict__ a, uint64_t groups,
                                                   const SparseArgs A) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < groups; c += stride) {
        const uint64_t i = expand_rt(c, A.sorted, A.m) + A.base_add;
        const double2 t = a[i];
        a[i] = a[i + A.delta];
        a[i + A.delta] = t;
    }
}

// phase_range kernels.hpp:301-308.
__global__ void __launch_bounds__(kThreads) k_phase(double2 *__restrict__ a, uint64_t groups,
                                                    const SparseArgs A) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < groups; c += stride) {
        const uint64_t i = expand_rt(c, A.sorted, A.m) + A.base_add;
        a[i] = cmul(a[i], A.phase);
    }
}

static void launch_sparse(bool swap, double2 *a, int pn, const Gate &g, uint64_t base_add,
                          uint64_t delta, cplx phase, cudaStream_t st) {
    SparseArgs A;
    A.m = g.m;
    int bits[3];
    for (int k = 0; k < g.m; ++k) bits[k] = g.pos[k] - 1;
    sorted_bits(bits, g.m, A.sorted);
    A.base_add = base_add;
    A.delta = delta;
    A.phase = make_double2(phase.real(), phase.imag());
    const uint64_t groups = 1ull << (pn - g.m);
    if (swap) {
        const ProfMark pf_ = prof_begin(st);
        k_swap<<<grid_for(groups), kThreads, 0, st>>>(a, groups, A);
        check_launch("k_swap", pf_);
    } else {
        const ProfMark pf_ = prof_begin(st);
        k_phase<<<grid_for(groups), kThreads, 0, st>>>(a, groups, A);
        check_launch("k_phase", pf_);
    }
}

// apply_gate_fast kernels.hpp:365-430
void apply_gate_fast(double2 *a, int pn, const Gate &g, cudaStream_t st) {
    check_fit(g.pos, g.m, pn);
    int bits[VQB_MAX_POSITIONS];
    for (int k = 0; k < g.m; ++k) bits[k] = g.pos[k] - 1;
    if ((1ull << (pn - g.m)) < 8) { // bases < kAggregationBatch: naive path
        launch_dense(a, pn, bits, g.m, g.mat, st);
        return;
    }
    const uint64_t o1 = g.m >= 1 ? 1ull << bits[0] : 0;
    const uint64_t o2 = g.m >= 2 ? 1ull << bits[1] : 0;
    const double isq = 0.70710678118654752440;
    switch (g.kind) {
    case VQB_GATE_X: launch_sparse(true, a, pn, g, 0, o1, 0.0, st); return;
    case VQB_GATE_Z: launch_sparse(false, a, pn, g, o1, 0, -1.0, st); return;
    case VQB_GATE_S: launch_sparse(false, a, pn, g, o1, 0, cplx(0, 1), st); return;
    case VQB_GATE_T: launch_sparse(false, a, pn, g, o1, 0, cplx(isq, isq), st); return;
    case VQB_GATE_CZ: launch_sparse(false, a, pn, g, o1 + o2, 0, -1.0, st); return;
    case VQB_GATE_CNOT: launch_sparse(true, a, pn, g, o1, o2, 0.0, st); return;
    case VQB_GATE_SWAP: {
        const uint64_t lo = std::min(o1, o2), hi = std::max(o1, o2);
        launch_sparse(true, a, pn, g, lo, hi - lo, 0.0, st);
        return;
    }
    default:
        launch_dense(a, pn, bits, g.m, g.mat, st);
    }
}

void apply_gate_both_sides(DeviceState *s, const Gate &g) {
    apply_gate_fast(s->amps, s->pn, g, s->stream);
    Gate bra = g;
    for (int k = 0; k < g.m; ++k) bra.pos[k] = g.pos[k] + s->n;
    bra.mat = conjugated(g.mat);
    bra.np = 0;
    if (bra.mat != g.mat) bra.kind = VQB_GATE_GENERIC;
    apply_gate_fast(s->amps, s->pn, bra, s->stream);
}

void apply_superop(DeviceState *s, const Channel &c) {
    const cvec sop = channel_superop(c);
    int bits[6];
    for (int k = 0; k < c.m; ++k) {
        bits[k] = c.pos[k] - 1;
        bits[k + c.m] = c.pos[k] - 1 + s->n;
    }
    launch_dense(s->amps, s->pn, bits, 2 * c.m, sop, s->stream);
}

// ------------------------------------------------------------------ deterministic reductions
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_down_sync(0xffffffffu, v.x, o);
        v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
    return v;
}

struct Epilogue {
    double2 *out_c;   // complex results [ns] (nullable)
    double *out_r;    // real_scale * Re(result) [ns] (nullable)
    double real_scale;
    bool accumulate = false; // out_r[s] += ... (gradient vectors: several steps may share an entry)
};

// Block-reduce NS complex values, store the block partial, and let the last
// block reduce all partials in index order (deterministic for a fixed grid).
template <int NS>
__device__ void reduce_epilogue(double2 (&v)[NS], int ns, double2 *partials, unsigned *counter,
                                const Epilogue ep) {
    __shared__ double2 sh[kThreads / 32][NS];
    __shared__ bool am_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        if (s >= ns) break;
        double2 w = warp_sum(v[s]);
        if (lane == 0) sh[warp][s] = w;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (s >= ns) break;
            double2 w = lane < nw ? sh[lane][s] : make_double2(0, 0);
            w = warp_sum(w);
            if (lane == 0) partials[(size_t)blockIdx.x * NS + s] = w;
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(counter, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    const volatile double2 *vp = partials;
    for (int s = 0; s < ns; ++s) {
        double2 acc = make_double2(0, 0);
        for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
            const double2 x = make_double2(vp[(size_t)i * NS + s].x, vp[(size_t)i * NS + s].y);
            acc = cadd(acc, x);
        }
        acc = warp_sum(acc);
        __syncthreads();
        if (lane == 0) sh[warp][0] = acc;
        __syncthreads();
        if (warp == 0) {
            double2 w = lane < nw ? sh[lane][0] : make_double2(0, 0);
            w = warp_sum(w);
            if (lane == 0) {
                if (ep.out_c) ep.out_c[s] = w;
                if (ep.out_r) ep.out_r[s] = (ep.accumulate ? ep.out_r[s] : 0.0) + ep.real_scale * w.x;
            }
        }
    }
    if (threadIdx.x == 0) *counter = 0;
}

// Fixed reduction grid: depends on the problem size only.
inline unsigned reduce_grid(uint64_t work) { return grid_for(work, kThreads, kMaxReduceBlocks); }

__global__ void __launch_bounds__(kThreads) k_norm_sq(const double2 *__restrict__ a, uint64_t size,
                                                      double2 *partials, unsigned *counter,
                                                      Epilogue ep) {
    double2 v[1] = {make_double2(0, 0)};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < size; k += stride) {
        const double2 x = a[k];
        v[0].x = fma(x.x, x.x, fma(x.y, x.y, v[0].x));
    }
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

__global__ void __launch_bounds__(kThreads) k_trace(const double2 *__restrict__ a, uint64_t dim,
                                                    double2 *partials, unsigned *counter,
                                                    Epilogue ep) {
    double2 v[1] = {make_double2(0, 0)};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < dim; k += stride)
        v[0] = cadd(v[0], a[k + k * dim]);
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

// <a|b>
__global__ void __launch_bounds__(kThreads) k_dot(const double2 *__restrict__ a,
                                                  const double2 *__restrict__ b, uint64_t size,
                                                  double2 *partials, unsigned *counter,
                                                  Epilogue ep) {
    double2 v[1] = {make_double2(0, 0)};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < size; k += stride)
        v[0] = cjfma(a[k], b[k], v[0]);
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    atomicMax((unsigned long long *)addr, (unsigned long long)__double_as_longlong(v));
}

__global__ void __launch_bounds__(kThreads) k_max_abs_diff(const double2 *__restrict__ a,
                                                           const double2 *__restrict__ b,
                                                           uint64_t size, double *out) {
    double m = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < size; k += stride) {
        const double dx = a[k].x - b[k].x, dy = a[k].y - b[k].y;
        m = fmax(m, hypot(dx, dy));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

static Epilogue ep_result(DeviceState *s) { return Epilogue{s->ws.result, nullptr, 0.0}; }

static cplx fetch_result(DeviceState *s, int slot = 0) {
    VQB_CUDA(cudaMemcpyAsync(s->ws.host_result, s->ws.result, sizeof(double2) * (slot + 1),
                             cudaMemcpyDeviceToHost, s->stream));
    VQB_CUDA(cudaStreamSynchronize(s->stream));
    return cplx(s->ws.host_result[slot].x, s->ws.host_result[slot].y);
}

double norm_sq(DeviceState *s) {
    const unsigned g = reduce_grid(s->size);
    const ProfMark pf_ = prof_begin(s->stream);
    k_norm_sq<<<g, kThreads, 0, s->stream>>>(s->amps, s->size, s->ws.partials, s->ws.counter,
                                             ep_result(s));
    check_launch("k_norm_sq", pf_);
    return fetch_result(s).real();
}

cplx trace(DeviceState *s) {
    const uint64_t dim = 1ull << s->n;
    const unsigned g = reduce_grid(dim);
    const ProfMark pf_ = prof_begin(s->stream);
    k_trace<<<g, kThreads, 0, s->stream>>>(s->amps, dim, s->ws.partials, s->ws.counter,
                                           ep_result(s));
    check_launch("k_trace", pf_);
    return fetch_result(s);
}

// ---- measurement (circuit.hpp:303-375) ----
// P(bit set): pure sum_{k & mask} |a_k|^2; mixed sum_{k & mask} Re rho_kk
// (stride dim + 1 along the diagonal of vec(rho)).
__global__ void __launch_bounds__(kThreads) k_prob_one(const double2 *__restrict__ a,
                                                       uint64_t count, uint64_t stride,
                                                       uint64_t mask, int pure,
                                                       double2 *partials, unsigned *counter,
                                                       Epilogue ep) {
    double2 v[1] = {make_double2(0, 0)};
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += step) {
        if (!(k & mask)) continue;
        const double2 x = a[k * stride];
        v[0].x = pure ? fma(x.x, x.x, fma(x.y, x.y, v[0].x)) : v[0].x + x.x;
    }
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

// Collapse: keep entries whose bits under mask_a and mask_b (the ket and, for
// a density matrix, the bra copy of the qubit) both equal the outcome; scale
// the kept ones, zero the rest.
__global__ void __launch_bounds__(kThreads) k_collapse(double2 *__restrict__ a, uint64_t size,
                                                       uint64_t mask_a, uint64_t mask_b,
                                                       int outcome, double scale) {
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < size; k += step) {
        const bool keep = (((k & mask_a) != 0) == (outcome == 1)) &&
                          (((k & mask_b) != 0) == (outcome == 1));
        const double2 x = a[k];
        a[k] = keep ? make_double2(x.x * scale, x.y * scale) : make_double2(0, 0);
    }
}

double prob_one(DeviceState *s, int qubit) {
    const uint64_t mask = 1ull << (qubit - 1);
    const uint64_t count = s->mixed ? (1ull << s->n) : s->size;
    const uint64_t stride = s->mixed ? (1ull << s->n) + 1 : 1;
    const unsigned g = reduce_grid(count);
    const ProfMark pf_ = prof_begin(s->stream);
    k_prob_one<<<g, kThreads, 0, s->stream>>>(s->amps, count, stride, mask, s->mixed ? 0 : 1,
                                              s->ws.partials, s->ws.counter, ep_result(s));
    check_launch("k_prob_one", pf_);
    return fetch_result(s).real();
}

void collapse(DeviceState *s, int qubit, int outcome, double scale) {
    const uint64_t mask_a = 1ull << (qubit - 1);
    const uint64_t mask_b = s->mixed ? mask_a << s->n : mask_a;
    const ProfMark pf_ = prof_begin(s->stream);
    k_collapse<<<grid_for(s->size, kThreads, 148 * 16), kThreads, 0, s->stream>>>(
        s->amps, s->size, mask_a, mask_b, outcome, scale);
    check_launch("k_collapse", pf_);
    VQB_CUDA(cudaStreamSynchronize(s->stream));
}

void dot_async(DeviceState *s, const double2 *a, const double2 *b, double2 *out_dev) {
    const unsigned g = reduce_grid(s->size);
    const ProfMark pf_ = prof_begin(s->stream);
    k_dot<<<g, kThreads, 0, s->stream>>>(a, b, s->size, s->ws.partials, s->ws.counter,
                                         Epilogue{out_dev, nullptr, 0.0});
    check_launch("k_dot", pf_);
}

cplx dot_async_result(DeviceState *s, const double2 *a, const double2 *b) {
    dot_async(s, a, b, s->ws.result);
    return fetch_result(s);
}

double max_abs_diff(DeviceState *s, const double2 *a, const double2 *b) {
    double *d = reinterpret_cast<double *>(s->ws.result);
    VQB_CUDA(cudaMemsetAsync(d, 0, sizeof(double), s->stream));
    const ProfMark pf_ = prof_begin(s->stream);
    k_max_abs_diff<<<grid_for(s->size), kThreads, 0, s->stream>>>(a, b, s->size, d);
    check_launch("k_max_abs_diff", pf_);
    VQB_CUDA(cudaMemcpyAsync(s->ws.host_result, d, sizeof(double), cudaMemcpyDeviceToHost,
                             s->stream));
    VQB_CUDA(cudaStreamSynchronize(s->stream));
    double r;
    std::memcpy(&r, s->ws.host_result, sizeof(double));
    return r;
}

// ------------------------------------------------------------------ Pauli sums
PauliPack pack_operator(const vqb_pauli_term *terms, int64_t nterms, bool conjugate) {
    struct T {
        uint64_t x, z;
        cplx c;
    };
    std::vector<T> ts;
    PauliPack p;
    for (int64_t t = 0; t < nterms; ++t) {
        uint64_t x = 0, z = 0;
        int ny = 0;
        for (int k = 0; k < terms[t].num_factors; ++k) {
            const int q = terms[t].qubits[k];
            const char l = terms[t].labels[k] | 0x20;
            if (l != 'x' && l != 'y' && l != 'z')
                raise(VQB_ERR_VALIDITY, std::string("unknown Pauli label '") + terms[t].labels[k] + "'");
            if (q < 1) raise(VQB_ERR_VALIDITY, "PauliTerm: qubit indices must be >= 1");
            for (int j = k + 1; j < terms[t].num_factors; ++j)
                if (terms[t].qubits[j] == q)
                    raise(VQB_ERR_VALIDITY, "PauliTerm: duplicate qubit index " + std::to_string(q));
            if (q > 63) raise(VQB_ERR_INDEX, "PauliTerm: qubit index beyond 63");
            p.max_qubit = std::max(p.max_qubit, q);
            const uint64_t bit = 1ull << (q - 1);
            if (l == 'x' || l == 'y') x |= bit;
            if (l == 'y' || l == 'z') z |= bit;
            if (l == 'y') ++ny;
        }
        cplx c(terms[t].coeff.re, terms[t].coeff.im);
        if (conjugate) c = std::conj(c);
        static const cplx ipow[4] = {1.0, cplx(0, 1), -1.0, cplx(0, -1)};
        ts.push_back({x, z, c * ipow[ny & 3]});
    }
    // group by x-mask, stable in first-appearance order
    std::vector<uint64_t> xs;
    for (const auto &t : ts)
        if (std::find(xs.begin(), xs.end(), t.x) == xs.end()) xs.push_back(t.x);
    for (uint64_t x : xs) {
        PauliGroupDev g{x, (int)p.terms.size(), 0};
        for (const auto &t : ts)
            if (t.x == x) {
                p.terms.push_back({t.z, make_double2(t.c.real(), t.c.imag())});
                ++g.count;
            }
        p.groups.push_back(g);
    }
    return p;
}

void upload_operator(DeviceState *s, const PauliPack &p) {
    const size_t gb = sizeof(PauliGroupDev) * p.groups.size();
    const size_t tb = sizeof(PauliTermDev) * p.terms.size();
    const size_t need = gb + tb + 16;
    if (need > s->ws.terms_bytes) {
        if (s->ws.terms) dev_free(s->ws.terms, s->ws.terms_bytes, false);
        s->ws.terms = nullptr;
        s->ws.terms_bytes = 0;
        s->ws.terms = dev_alloc(need, false);
        s->ws.terms_bytes = need;
    }
    std::vector<char> buf(gb + tb);
    std::memcpy(buf.data(), p.groups.data(), gb);
    std::memcpy(buf.data() + gb, p.terms.data(), tb);
    VQB_CUDA(cudaMemcpyAsync(s->ws.terms, buf.data(), buf.size(), cudaMemcpyHostToDevice, s->stream));
    VQB_CUDA(cudaStreamSynchronize(s->stream)); // buf is a stack temporary
}

// Pauli tables staged once per block in shared memory: every thread reads
// every term for every amplitude, so broadcast shared-memory reads replace
// per-thread global loads (the operator is a few KB; larger ones stay global).
struct PauliView {
    const PauliGroupDev *g;
    const PauliTermDev *t;
};
__device__ __forceinline__ PauliView stage_pauli(const PauliGroupDev *g, int ng, const PauliTermDev *t, int nt,
                                                 bool staged) {
    if (!staged) return {g, t};
    extern __shared__ __align__(16) unsigned char pauli_sm[];
    auto *sg = reinterpret_cast<PauliGroupDev *>(pauli_sm);
    auto *st = reinterpret_cast<PauliTermDev *>(pauli_sm + sizeof(PauliGroupDev) * (size_t)ng);
    for (int i = threadIdx.x; i < ng; i += blockDim.x) sg[i] = g[i];
    for (int i = threadIdx.x; i < nt; i += blockDim.x) st[i] = t[i];
    __syncthreads();
    return {sg, st};
}
size_t pauli_smem(const PauliPack &p) {
    const size_t b = sizeof(PauliGroupDev) * p.groups.size() + sizeof(PauliTermDev) * p.terms.size();
    return b <= 40 * 1024 ? b : 0;
}

// Sum over a group's terms of c_t * (-1)^popc(idx & z_t).
__device__ __forceinline__ double2 group_weight(const PauliTermDev *__restrict__ terms, int first,
                                                int count, uint64_t idx) {
    double2 w = make_double2(0, 0);
    for (int t = first; t < first + count; ++t) {
        const PauliTermDev T = terms[t];
        const double sgn = (__popcll(idx & T.zmask) & 1) ? -1.0 : 1.0;
        w.x = fma(sgn, T.coeff.x, w.x);
        w.y = fma(sgn, T.coeff.y, w.y);
    }
    return w;
}

// <psi|H|psi> = sum_g sum_b conj(psi[b^x]) psi[b] W_g(b) (observables.hpp:176-190)
// `ket` (nullable: = a) is the buffer read at b: a different shard for the
// terms of a sharded state whose X/Y factors flip global qubits
__global__ void __launch_bounds__(kThreads) k_expect_pure(const double2 *__restrict__ a, uint64_t size,
                                                          const PauliGroupDev *__restrict__ groups_g,
                                                          int ngroups,
                                                          const PauliTermDev *__restrict__ terms_g, int nterms, int staged,
                                                          double2 *partials, unsigned *counter,
                                                          Epilogue ep, const double2 *__restrict__ ket) {
    const PauliView pv = stage_pauli(groups_g, ngroups, terms_g, nterms, staged != 0);
    const PauliGroupDev *groups = pv.g;
    const PauliTermDev *terms = pv.t;
    double2 v[1] = {make_double2(0, 0)};
    const bool same = ket == nullptr;
    const double2 *k = same ? a : ket;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < size; b += stride) {
        const double2 ab = k[b];
        for (int g = 0; g < ngroups; ++g) {
            const PauliGroupDev G = groups[g];
            const double2 w = group_weight(terms, G.first, G.count, b);
            const double2 ax = (G.xmask || !same) ? a[b ^ G.xmask] : ab;
            const double2 pr = cjfma(ax, ab, make_double2(0, 0));
            v[0] = cfma(pr, w, v[0]);
        }
    }
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

// tr(H rho) = sum_k sum_g rho[(k^x) + k*dim] W_g(k^x) (observables.hpp:194-213)
__global__ void __launch_bounds__(kThreads) k_expect_mixed(const double2 *__restrict__ a, uint64_t dim,
                                                           const PauliGroupDev *__restrict__ groups_g,
                                                           int ngroups,
                                                           const PauliTermDev *__restrict__ terms_g, int nterms, int staged,
                                                           double2 *partials, unsigned *counter,
                                                           Epilogue ep) {
    const PauliView pv = stage_pauli(groups_g, ngroups, terms_g, nterms, staged != 0);
    const PauliGroupDev *groups = pv.g;
    const PauliTermDev *terms = pv.t;
    double2 v[1] = {make_double2(0, 0)};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < dim; k += stride) {
        for (int g = 0; g < ngroups; ++g) {
            const PauliGroupDev G = groups[g];
            const uint64_t r = k ^ G.xmask;
            const double2 w = group_weight(terms, G.first, G.count, r);
            v[0] = cfma(a[r + k * dim], w, v[0]);
        }
    }
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

void expectation_async(DeviceState *s, const PauliPack &p, double2 *out_dev, const double2 *ket) {
    upload_operator(s, p);
    auto *groups = reinterpret_cast<const PauliGroupDev *>(s->ws.terms);
    auto *terms = reinterpret_cast<const PauliTermDev *>(
        reinterpret_cast<const char *>(s->ws.terms) + sizeof(PauliGroupDev) * p.groups.size());
    const int ng = (int)p.groups.size();
    const Epilogue ep{out_dev, nullptr, 0.0};
    if (ng == 0) {
        VQB_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double2), s->stream));
        return;
    }
    if (s->mixed) {
        const uint64_t dim = 1ull << s->n;
        const ProfMark pf_ = prof_begin(s->stream);
        k_expect_mixed<<<reduce_grid(dim), kThreads, pauli_smem(p), s->stream>>>(
            s->amps, dim, groups, ng, terms, (int)p.terms.size(), pauli_smem(p) > 0, s->ws.partials,
            s->ws.counter, ep);
        check_launch("k_expect_mixed", pf_);
    } else {
        const ProfMark pf_ = prof_begin(s->stream);
        k_expect_pure<<<reduce_grid(s->size), kThreads, pauli_smem(p), s->stream>>>(
            s->amps, s->size, groups, ng, terms, (int)p.terms.size(), pauli_smem(p) > 0, s->ws.partials,
            s->ws.counter, ep, ket);
        check_launch("k_expect_pure", pf_);
    }
}

cplx expectation(DeviceState *s, const PauliPack &p) {
    expectation_async(s, p, s->ws.result);
    return fetch_result(s);
}

cplx expectation_cross(DeviceState *bra, const double2 *ket, const PauliPack &p) {
    if (bra->mixed) raise(VQB_ERR_INTERNAL, "expectation_cross: pure states only");
    expectation_async(bra, p, bra->ws.result, ket);
    return fetch_result(bra);
}

// dst[b] = sum_g psi[b^x] W_g(b^x) (apply_operator observables.hpp:216-237)
__global__ void __launch_bounds__(kThreads) k_apply_operator(const double2 *__restrict__ a,
                                                             double2 *__restrict__ out, uint64_t size,
                                                             const PauliGroupDev *__restrict__ groups_g,
                                                             int ngroups,
                                                             const PauliTermDev *__restrict__ terms_g, int nterms, int staged,
                                                             int accumulate) {
    const PauliView pv = stage_pauli(groups_g, ngroups, terms_g, nterms, staged != 0);
    const PauliGroupDev *groups = pv.g;
    const PauliTermDev *terms = pv.t;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < size; b += stride) {
        double2 acc = accumulate ? out[b] : make_double2(0, 0);
        for (int g = 0; g < ngroups; ++g) {
            const PauliGroupDev G = groups[g];
            const uint64_t src = b ^ G.xmask;
            acc = cfma(a[src], group_weight(terms, G.first, G.count, src), acc);
        }
        out[b] = acc;
    }
}

// H|psi> for a diagonal operator with real coefficients (every term a Z
// string: one group, x mask 0), e.g. the QAOA cost Hamiltonian: each thread
// takes the 8 amplitudes b0 | i << 5 (i < 8; a warp's lanes cover bits 0-4, so
// every load is coalesced), so a term's sign is the parity of (b0 & z) flipped
// by the parity of (i & (z >> 5) & 7); terms that miss bits 5-7 add the same
// signed coefficient to all 8 (one scalar), the others flip the sign bit of c
// per element (integer ops, then one DADD). Same sums as group_weight up to
// the summation order.
__global__ void __launch_bounds__(kThreads) k_apply_zdiag(const double2 *__restrict__ a, double2 *__restrict__ out,
                                                          uint64_t size, const PauliTermDev *__restrict__ terms_g,
                                                          int nterms) {
    extern __shared__ __align__(16) unsigned char zsm[];
    auto *zm = reinterpret_cast<unsigned long long *>(zsm);
    auto *cf = reinterpret_cast<double *>(zsm + sizeof(unsigned long long) * (size_t)nterms);
    for (int i = threadIdx.x; i < nterms; i += blockDim.x) {
        zm[i] = terms_g[i].zmask;
        cf[i] = terms_g[i].coeff.x;
    }
    __syncthreads();
    // byte lz of kPar: bit i = parity(i & lz)
    constexpr unsigned long long kPar = 0x963C5AF066CCAA00ull;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (size >> 3); j += stride) {
        const uint64_t b0 = ((j >> 5) << 8) | (j & 31);
        double w[8], wc = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = 0.0;
        for (int t = 0; t < nterms; ++t) {
            const unsigned long long z = zm[t];
            const double c = cf[t];
            const int base = __popcll(b0 & z) & 1;
            const int lz = (int)((z >> 5) & 7);
            if (lz == 0) {
                wc += base ? -c : c;
                continue;
            }
            const unsigned pm = ((unsigned)(kPar >> (8 * lz)) & 0xFFu) ^ (base ? 0xFFu : 0u);
            const int hi = __double2hiint(c), lo = __double2loint(c);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                w[i] += __hiloint2double(hi ^ (int)(((pm >> i) & 1u) << 31), lo);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double2 v = a[b0 | ((uint64_t)i << 5)];
            const double wi = w[i] + wc;
            out[b0 | ((uint64_t)i << 5)] = make_double2(wi * v.x, wi * v.y);
        }
    }
}

void apply_operator(DeviceState *src, double2 *dst, const PauliPack &p, bool) {
    apply_operator_from(src, src->amps, dst, p, false);
}

void apply_operator_from(DeviceState *src, const double2 *src_amps, double2 *dst, const PauliPack &p,
                         bool accumulate) {
    bool zdiag = !accumulate && p.groups.size() == 1 && p.groups[0].xmask == 0 && src->size >= 256 &&
                 p.terms.size() * 16 <= 40 * 1024;
    for (const auto &t : p.terms) zdiag = zdiag && t.coeff.y == 0.0;
    if (zdiag) {
        upload_operator(src, p);
        auto *terms = reinterpret_cast<const PauliTermDev *>(reinterpret_cast<const char *>(src->ws.terms) +
                                                             sizeof(PauliGroupDev) * p.groups.size());
        const ProfMark pf_ = prof_begin(src->stream);
        k_apply_zdiag<<<grid_for(src->size >> 3), kThreads, 16 * p.terms.size(), src->stream>>>(
            src_amps, dst, src->size, terms, (int)p.terms.size());
        check_launch("k_apply_zdiag", pf_);
        return;
    }
    upload_operator(src, p);
    auto *groups = reinterpret_cast<const PauliGroupDev *>(src->ws.terms);
    auto *terms = reinterpret_cast<const PauliTermDev *>(
        reinterpret_cast<const char *>(src->ws.terms) + sizeof(PauliGroupDev) * p.groups.size());
    const ProfMark pf_ = prof_begin(src->stream);
    if (p.groups.empty()) {
        if (!accumulate) VQB_CUDA(cudaMemsetAsync(dst, 0, sizeof(double2) * src->size, src->stream));
        return;
    }
    k_apply_operator<<<grid_for(src->size), kThreads, pauli_smem(p), src->stream>>>(
        src_amps, dst, src->size, groups, (int)p.groups.size(), terms, (int)p.terms.size(), pauli_smem(p) > 0,
        accumulate ? 1 : 0);
    check_launch("k_apply_operator", pf_);
}

// <<I| H as a ket on vec(rho) (autodiff.hpp:241-248): entry (c^x) + c*dim gets
// sum_t conj(coeff_t) i^{#Y} (-1)^popc(c & z_t); everything else is zero.
__global__ void __launch_bounds__(kThreads) k_identity_costate(double2 *__restrict__ out, uint64_t dim,
                                                               const PauliGroupDev *__restrict__ groups_g,
                                                               int ngroups,
                                                               const PauliTermDev *__restrict__ terms_g, int nterms, int staged) {
    const PauliView pv = stage_pauli(groups_g, ngroups, terms_g, nterms, staged != 0);
    const PauliGroupDev *groups = pv.g;
    const PauliTermDev *terms = pv.t;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < dim; c += stride)
        for (int g = 0; g < ngroups; ++g) {
            const PauliGroupDev G = groups[g];
            out[(c ^ G.xmask) + c * dim] = group_weight(terms, G.first, G.count, c);
        }
}

void identity_costate(DeviceState *s, const PauliPack &p) {
    upload_operator(s, p);
    auto *groups = reinterpret_cast<const PauliGroupDev *>(s->ws.terms);
    auto *terms = reinterpret_cast<const PauliTermDev *>(
        reinterpret_cast<const char *>(s->ws.terms) + sizeof(PauliGroupDev) * p.groups.size());
    VQB_CUDA(cudaMemsetAsync(s->amps, 0, sizeof(double2) * s->size, s->stream));
    const uint64_t dim = 1ull << s->n;
    const ProfMark pf_ = prof_begin(s->stream);
    k_identity_costate<<<grid_for(dim), kThreads, pauli_smem(p), s->stream>>>(
        s->amps, dim, groups, (int)p.groups.size(), terms, (int)p.terms.size(), pauli_smem(p) > 0);
    check_launch("k_identity_costate", pf_);
}

// ------------------------------------------------------------------ bilinear form / reverse step
template <int M> struct StepArgs {
    int sorted[M];
    unsigned long long off[1 << M];
    int np;
    double2 inv[(1 << M) * (1 << M)];
    double2 dm[VQB_MAX_PARAMS][(1 << M) * (1 << M)];
};

// bilinear_gate_form kernels.hpp:466-503 (dm[0] = local)
template <int M>
__global__ void __launch_bounds__(kThreads) k_bilinear(const double2 *__restrict__ bra,
                                                       const double2 *__restrict__ ket, uint64_t groups,
                                                       const __grid_constant__ StepArgs<M> A,
                                                       double2 *partials, unsigned *counter,
                                                       Epilogue ep) {
    constexpr int D = 1 << M;
    double2 v[1] = {make_double2(0, 0)};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < groups; c += stride) {
        const uint64_t b = expand<M>(c, A.sorted);
        double2 in[D];
#pragma unroll
        for (int r = 0; r < D; ++r) in[r] = ket[b + A.off[r]];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double2 w = cmul(A.dm[0][r], in[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) w = cfma(A.dm[0][r + s * D], in[s], w);
            v[0] = cjfma(bra[b + A.off[r]], w, v[0]);
        }
    }
    reduce_epilogue<1>(v, 1, partials, counter, ep);
}

// reverse_sweep_step kernels.hpp:659-697: phi <- inv phi; acc_p += <psi|D_p|phi>; psi <- inv psi
template <int M>
__global__ void __launch_bounds__(kThreads) k_reverse_step(double2 *__restrict__ phi,
                                                           double2 *__restrict__ psi, uint64_t groups,
                                                           const __grid_constant__ StepArgs<M> A,
                                                           double2 *partials, unsigned *counter,
                                                           Epilogue ep) {
    constexpr int D = 1 << M;
    double2 acc[VQB_MAX_PARAMS];
#pragma unroll
    for (int p = 0; p < VQB_MAX_PARAMS; ++p) acc[p] = make_double2(0, 0);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < groups; c += stride) {
        const uint64_t b = expand<M>(c, A.sorted);
        double2 f[D], w[D], g[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            f[r] = phi[b + A.off[r]];
            g[r] = psi[b + A.off[r]];
        }
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double2 x = cmul(A.inv[r], f[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) x = cfma(A.inv[r + s * D], f[s], x);
            w[r] = x;
            phi[b + A.off[r]] = x;
        }
        for (int p = 0; p < A.np; ++p) {
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double2 x = cmul(A.dm[p][r], w[0]);
#pragma unroll
                for (int s = 1; s < D; ++s) x = cfma(A.dm[p][r + s * D], w[s], x);
                acc[p] = cjfma(g[r], x, acc[p]);
            }
        }
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double2 x = cmul(A.inv[r], g[0]);
#pragma unroll
            for (int s = 1; s < D; ++s) x = cfma(A.inv[r + s * D], g[s], x);
            psi[b + A.off[r]] = x;
        }
    }
    reduce_epilogue<VQB_MAX_PARAMS>(acc, A.np, partials, counter, ep);
}

template <int M>
static StepArgs<M> make_step_args(const int *pos1, const cvec &inv, const std::vector<cvec> &dm) {
    StepArgs<M> A;
    int bits[M];
    for (int k = 0; k < M; ++k) bits[k] = pos1[k] - 1;
    sorted_bits(bits, M, A.sorted);
    for (int r = 0; r < (1 << M); ++r) {
        uint64_t o = 0;
        for (int k = 0; k < M; ++k)
            if ((r >> k) & 1) o += 1ull << bits[k];
        A.off[r] = o;
    }
    A.np = (int)dm.size();
    const int dd = 1 << (2 * M);
    for (int i = 0; i < dd; ++i) {
        A.inv[i] = inv.empty() ? make_double2(0, 0) : make_double2(inv[i].real(), inv[i].imag());
        for (int p = 0; p < A.np; ++p) A.dm[p][i] = make_double2(dm[p][i].real(), dm[p][i].imag());
    }
    return A;
}

template <int M>
static cplx bilinear_m(DeviceState *bra, DeviceState *ket, const int *pos1, const cvec &local) {
    const auto A = make_step_args<M>(pos1, {}, {local});
    const uint64_t groups = 1ull << (ket->pn - M);
    const ProfMark pf_ = prof_begin(ket->stream);
    k_bilinear<M><<<reduce_grid(groups), kThreads, 0, ket->stream>>>(
        bra->amps, ket->amps, groups, A, ket->ws.partials, ket->ws.counter, ep_result(ket));
    check_launch("k_bilinear", pf_);
    return fetch_result(ket);
}

cplx bilinear_form(DeviceState *bra, DeviceState *ket, const int *pos1, int m, const cvec &local) {
    if (bra->stream != ket->stream) sync(bra);
    switch (m) {
    case 1: return bilinear_m<1>(bra, ket, pos1, local);
    case 2: return bilinear_m<2>(bra, ket, pos1, local);
    case 3: return bilinear_m<3>(bra, ket, pos1, local);
    case 4: return bilinear_m<4>(bra, ket, pos1, local);
    default: raise(VQB_ERR_UNSUPPORTED, "bilinear_form: at most 4 positions on the device path");
    }
}

template <int M>
static void reverse_m(double2 *phi, double2 *psi, int pn, const int *pos1, const cvec &inv,
                      const std::vector<cvec> &dm, DeviceState *w, double2 *out_c, double *out_r,
                      double scale) {
    const auto A = make_step_args<M>(pos1, inv, dm);
    const uint64_t groups = 1ull << (pn - M);
    const ProfMark pf_ = prof_begin(w->stream);
    k_reverse_step<M><<<reduce_grid(groups), kThreads, 0, w->stream>>>(
        phi, psi, groups, A, w->ws.partials, w->ws.counter, Epilogue{out_c, out_r, scale, true});
    check_launch("k_reverse_step", pf_);
}

void reverse_step_async(double2 *phi, double2 *psi, int pn, const int *pos1, int m, const cvec &inv,
                        const std::vector<cvec> &dmats, DeviceState *w, double2 *out_c, double *out_r,
                        double real_scale) {
    if ((int)dmats.size() > VQB_MAX_PARAMS) raise(VQB_ERR_SHAPE, "reverse_step: at most 5 derivative matrices");
    if (dmats.empty()) {
        raise(VQB_ERR_SHAPE, "reverse_step: needs at least one derivative matrix");
    }
    switch (m) {
    case 1: reverse_m<1>(phi, psi, pn, pos1, inv, dmats, w, out_c, out_r, real_scale); return;
    case 2: reverse_m<2>(phi, psi, pn, pos1, inv, dmats, w, out_c, out_r, real_scale); return;
    case 3: reverse_m<3>(phi, psi, pn, pos1, inv, dmats, w, out_c, out_r, real_scale); return;
    case 4: reverse_m<4>(phi, psi, pn, pos1, inv, dmats, w, out_c, out_r, real_scale); return;
    default: raise(VQB_ERR_UNSUPPORTED, "reverse_step: at most 4 positions on the device path");
    }
}

// ------------------------------------------------------------------ state management
// Pinned host staging for small results: one 1-KiB block per thread, shared
// by the states that thread drives (API calls are synchronous per thread).
// Deliberately never freed: a state may outlive the thread that created it.
struct PinnedResults {
    double2 *p = nullptr;
};
static thread_local PinnedResults g_pinned;

constexpr size_t kWorkspaceBytes =
    sizeof(double2) * kMaxReduceBlocks * kMaxReduceSlots + sizeof(double2) * 64 + 64;

static void alloc_workspace(DeviceState *s) {
    // one device allocation: partials | result | counter
    const size_t pb = sizeof(double2) * kMaxReduceBlocks * kMaxReduceSlots;
    char *base = static_cast<char *>(dev_alloc(kWorkspaceBytes, false));
    s->ws.partials = reinterpret_cast<double2 *>(base);
    s->ws.result = reinterpret_cast<double2 *>(base + pb);
    s->ws.counter = reinterpret_cast<unsigned *>(base + pb + sizeof(double2) * 64);
    VQB_CUDA(cudaMemsetAsync(s->ws.counter, 0, sizeof(unsigned) * 4, s->stream));
    if (!g_pinned.p) VQB_CUDA(cudaMallocHost(&g_pinned.p, sizeof(double2) * 64));
    s->ws.host_result = g_pinned.p;
}

DeviceState *state_create(int n, int mixed) {
    const int maxq = mixed ? 20 : 40; // state.hpp:179,261
    if (n < 1) raise(VQB_ERR_SIZE, "state: qubit count must be >= 1, got " + std::to_string(n));
    if (n > maxq)
        raise(VQB_ERR_SIZE, "state: qubit count " + std::to_string(n) +
                                " exceeds the supported maximum of " + std::to_string(maxq));
    auto *s = new DeviceState();
    s->n = n;
    s->mixed = mixed ? 1 : 0;
    s->pn = mixed ? 2 * n : n;
    s->size = 1ull << s->pn;
    s->device = current_device();
    VQB_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->amps = static_cast<double2 *>(dev_alloc(sizeof(double2) * s->size, true, false));
    if (!s->amps) {
        cudaStreamDestroy(s->stream);
        delete s;
        raise(VQB_ERR_SIZE, "state: cannot allocate 2^" + std::to_string(mixed ? 2 * n : n) +
                                " amplitudes on the device");
    }
    alloc_workspace(s);
    state_set_zero(s);
    return s;
}

DeviceState *state_wrap(void *ptr, int n, int mixed, uint64_t global_offset, int global_qubits) {
    cudaPointerAttributes attr{};
    VQB_CUDA(cudaPointerGetAttributes(&attr, ptr));
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
        raise(VQB_ERR_USAGE, "state_wrap: pointer is not device memory");
    DevScope on(attr.device);
    auto *s = new DeviceState();
    s->n = n;
    s->mixed = mixed ? 1 : 0;
    s->pn = mixed ? 2 * n : n;
    s->size = 1ull << s->pn;
    s->amps = static_cast<double2 *>(ptr);
    s->owned = false;
    s->device = attr.device;
    s->global_offset = global_offset;
    s->global_qubits = global_qubits;
    VQB_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    alloc_workspace(s);
    return s;
}

void state_set_zero(DeviceState *s) {
    VQB_CUDA(cudaMemsetAsync(s->amps, 0, sizeof(double2) * s->size, s->stream));
    if (s->global_offset == 0) {
        const double2 one = make_double2(1.0, 0.0);
        VQB_CUDA(cudaMemcpyAsync(s->amps, &one, sizeof(double2), cudaMemcpyHostToDevice, s->stream));
    }
    VQB_CUDA(cudaStreamSynchronize(s->stream));
}

void state_destroy(DeviceState *s) {
    if (!s) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != s->device) cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    if (s->owned && s->amps) dev_free(s->amps, sizeof(double2) * s->size, true);
    dev_free(s->ws.partials, kWorkspaceBytes, false); // partials | result | counter: one allocation
    if (s->ws.terms) dev_free(s->ws.terms, s->ws.terms_bytes, false);
    cudaStreamDestroy(s->stream);
    if (cur >= 0 && cur != s->device) cudaSetDevice(cur);
    delete s;
}

void sync(DeviceState *s) { VQB_CUDA(cudaStreamSynchronize(s->stream)); }

} // namespace vqb
