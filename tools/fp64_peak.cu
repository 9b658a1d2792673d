// Measures the FP64 ceilings the fused executors are bound by on this GPU:
//   dfma  - CUDA-core DFMA throughput (independent FMA chains per thread)
//   dmma  - FP64 tensor-core throughput (mma.sync m8n8k4 f64, one warp-wide
//           instruction = 256 FMAs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
// Prints one JSON line; used to fill roofline.fp64.peak (bench.py).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

constexpr int kChains = 8;
#ifndef MIXR
#define MIXR 4
#endif

__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}

__global__ void k_dmma(double *out, int iters, double a) {
    const int lane = threadIdx.x & 31;
    double av = a + lane * 1e-3, bv = a - lane * 1e-3;
    double d[kChains][2];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
                         "{%0,%1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(av), "d"(bv));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
    if (s == 1234.5) out[0] = s;
}

// both pipes at once: each warp interleaves DMMA chains with DFMA chains, to
// learn whether the FP64 tensor path and the DFMA pipe issue concurrently
__global__ void k_mixed(double *out, int iters, double a, double b) {
    const int lane = threadIdx.x & 31;
    double av = a + lane * 1e-3, bv = a - lane * 1e-3;
    double d[4][2];
    double x[kChains];
#pragma unroll
    for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = c;
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
                         "{%0,%1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(av), "d"(bv));
#pragma unroll
        for (int r = 0; r < MIXR; ++r)
#pragma unroll
            for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    double *out;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int threads = 256, blocks = nsm * 8, iters = 1 << 14;
    double best_dfma = 0, best_dmma = 0;
    for (int rep = 0; rep < 6; ++rep) {
        float ms;
        CK(cudaEventRecord(e0));
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double f1 = 2.0 * kChains * iters * double(blocks) * threads / (ms * 1e-3) / 1e12;
        if (rep > 0 && f1 > best_dfma) best_dfma = f1;
        CK(cudaEventRecord(e0));
        k_dmma<<<blocks, threads>>>(out, iters / 4, 0.5);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double f2 =
            2.0 * 256 * kChains * (iters / 4) * double(blocks) * (threads / 32) / (ms * 1e-3) / 1e12;
        if (rep > 0 && f2 > best_dmma) best_dmma = f2;
    }
    double best_mixed = 0;
    for (int rep = 0; rep < 6; ++rep) {
        float ms;
        const int it = iters / 8;
        CK(cudaEventRecord(e0));
        k_mixed<<<blocks, threads>>>(out, it, 0.999999, 1e-7);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        // per iteration per warp: 4 DMMA (256 FMA each) + MIXR*kChains*32 DFMA
        const double fl = 2.0 * (4.0 * 256 + MIXR * kChains * 32.0) * it * double(blocks) * (threads / 32);
        const double f3 = fl / (ms * 1e-3) / 1e12;
        if (rep > 0 && f3 > best_mixed) best_mixed = f3;
    }
    CK(cudaGetLastError());
    std::printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"mixed_tflops\": %.3f, \"mixr\": %d, \"sms\": %d, \"clock_mhz\": %d}\n",
                best_dfma, best_dmma, best_mixed, MIXR, nsm, clk / 1000);
    return 0;
}
