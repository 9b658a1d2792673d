// jit_rt.cuh — device runtime of the specialised stage kernels.
//
// The register executor (regstage_impl.cuh) interprets a stage program held in
// a __grid_constant__ block: per operation it loads a descriptor, dispatches
// on it and reads its matrix with a computed index. For stage programs that
// are run repeatedly (circuits of the same shape: every step of a benchmark,
// every iteration of a variational loop) the library instead generates one
// kernel per stage program with the layouts, register positions, condition
// bits and matrix offsets as compile-time constants, and compiles it once with
// NVRTC (jit.cpp). Matrices stay launch parameters (values change between
// calls, structure does not), read at constant offsets of the parameter bank
// (constant-bank operands of DFMA, no index arithmetic, no loads). This file is
// the only code the generated kernels include; it is embedded into the
// library as a string and compiled for sm_100a at run time.
#pragma once

typedef unsigned long long u64;

namespace vqbjit {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// Re(conj(a) * b)
__device__ __forceinline__ double re_cj(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }

// swizzled shared-memory slot of a tile-local index (regstage_impl.cuh swz)
__device__ __forceinline__ int swz(int l) {
    return l ^ ((l >> 3) & 7) ^ ((l >> 6) & 7) ^ ((l >> 9) & 7);
}

// index check of the VQB_JIT_CHECK instrumentation: traps when i >= n
__device__ __forceinline__ u64 chk_idx(u64 i, u64 n) {
    if (i >= n) __trap();
    return i;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// register offsets of matrix index r for an op on register bits (P0[, P1])
template <int NT, int P0, int P1> struct Pos {
    static constexpr int D = 1 << NT;
    static constexpr int MASK = (1 << P0) | (NT > 1 ? 1 << P1 : 0);
    __host__ __device__ static constexpr int off(int r) {
        return ((r & 1) ? 1 << P0 : 0) | ((NT > 1 && (r & 2)) ? 1 << P1 : 0);
    }
};

// out = M * v[group i], in place; M column-major D x D
template <int NT, int P0, int P1, int R>
__device__ __forceinline__ void mv_group(double2 (&v)[R], int i, const double2 *__restrict__ M) {
    using PS = Pos<NT, P0, P1>;
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

// the same matrix on every group
template <int NT, int P0, int P1, int R>
__device__ __forceinline__ void mv_all(double2 (&v)[R], const double2 *__restrict__ M) {
    using PS = Pos<NT, P0, P1>;
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (!(i & PS::MASK)) mv_group<NT, P0, P1, R>(v, i, M);
}

// adjoint step on one group: phi <- M phi; acc += Re <psi| D |phi>; psi <- M psi
template <int NT, int P0, int P1, int R>
__device__ __forceinline__ double dot_group(const double2 (&vf)[R], const double2 (&vg)[R], int i,
                                            const double2 *__restrict__ Dm) {
    using PS = Pos<NT, P0, P1>;
    constexpr int D = PS::D;
    double a = 0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double2 x = cmul(Dm[r], vf[i | PS::off(0)]);
#pragma unroll
        for (int s = 1; s < D; ++s) x = cfma(Dm[r + s * D], vf[i | PS::off(s)], x);
        a += re_cj(vg[i | PS::off(r)], x);
    }
    return a;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) x += __shfl_down_sync(0xffffffffu, x, sh);
    return x;
}

} // namespace vqbjit
