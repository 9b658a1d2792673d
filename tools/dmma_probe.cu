// Throughput probe for a tensor-core (DMMA m8n8k4 f64) gate executor:
// one block = 128 threads = one 2048-amplitude tile, 16 amplitudes per
// thread; an op is a dense complex 4x4 matrix on the two tile bits held by
// lane bits 0,1 (2 DMMAs per amplitude register), and every `per_relayout`
// ops the tile is re-laid out through XOR-swizzled shared memory.
// Prints effective FP64 TF/s (32 flops per amplitude per op) per variant.
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

constexpr int R = 16, T = 128, TS = 2048;

__device__ __forceinline__ int swz(int l) {
    return l ^ ((l >> 3) & 7) ^ ((l >> 6) & 7) ^ ((l >> 9) & 7);
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b, double c0,
                                     double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__constant__ double2 cB[64][32]; // per op, per lane: (b0, b1)

template <int MODE> // 0: DMMA only, 1: relayout every op, 2: every 2 ops, 3: DFMA register ops
__global__ void __launch_bounds__(T, 3) k_probe(double2 *amps, long long ntiles, int nops) {
    __shared__ double2 xbuf[TS];
    const int t = threadIdx.x, lane = t & 31;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        double2 *base = amps + tile * TS;
        double2 v[R];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = base[t + T * i];
        for (int o = 0; o < nops; ++o) {
            if ((MODE == 1) || (MODE == 2 && (o & 1))) {
                // relayout: rotate which tile bits are lane bits (cost model only)
                const int rot = (o % 5) + 1;
#pragma unroll
                for (int i = 0; i < R; ++i) xbuf[swz((t + T * i) & (TS - 1))] = v[i];
                __syncthreads();
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const int l = ((t << rot) | (t >> (7 - rot))) & 127;
                    v[i] = xbuf[swz((l + T * i) & (TS - 1))];
                }
                __syncthreads();
            }
            if (MODE == 3) {
                // the DFMA reference: a dense 4x4 on register bits 0,1
                double2 m[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) m[e] = cB[o & 63][e];
#pragma unroll
                for (int g = 0; g < R; g += 4) {
                    double2 out[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        double re = 0, im = 0;
#pragma unroll
                        for (int s = 0; s < 4; ++s) {
                            re = fma(m[r + 4 * s].x, v[g + s].x, fma(-m[r + 4 * s].y, v[g + s].y, re));
                            im = fma(m[r + 4 * s].x, v[g + s].y, fma(m[r + 4 * s].y, v[g + s].x, im));
                        }
                        out[r] = make_double2(re, im);
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) v[g + r] = out[r];
                }
            } else {
                const double2 b = cB[o & 63][lane];
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    double d0, d1;
                    dmma(d0, d1, v[i].x, b.x, 0.0, 0.0);
                    dmma(d0, d1, v[i].y, b.y, d0, d1);
                    v[i] = make_double2(d0, d1);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) base[t + T * i] = v[i];
    }
}

int main() {
    const int pn = 28, nops = 24;
    const long long n = 1ll << pn, ntiles = n / TS;
    double2 *a;
    CK(cudaMalloc(&a, n * sizeof(double2)));
    CK(cudaMemset(a, 0, n * sizeof(double2)));
    static double2 hb[64][32];
    for (int o = 0; o < 64; ++o)
        for (int l = 0; l < 32; ++l) hb[o][l] = make_double2(0.5 * ((l + o) % 3 - 1), 0.25);
    CK(cudaMemcpyToSymbol(cB, hb, sizeof hb));
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const char *names[4] = {"dmma_only", "dmma_relayout_every_op", "dmma_relayout_every_2",
                            "dfma_registers"};
    std::printf("{");
    for (int mode = 0; mode < 4; ++mode) {
        int per_sm = 0;
        void *fn = mode == 0 ? (void *)k_probe<0> : mode == 1 ? (void *)k_probe<1>
                 : mode == 2 ? (void *)k_probe<2> : (void *)k_probe<3>;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, T, 0));
        const int grid = nsm * per_sm;
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(e0));
            if (mode == 0) k_probe<0><<<grid, T>>>(a, ntiles, nops);
            if (mode == 1) k_probe<1><<<grid, T>>>(a, ntiles, nops);
            if (mode == 2) k_probe<2><<<grid, T>>>(a, ntiles, nops);
            if (mode == 3) k_probe<3><<<grid, T>>>(a, ntiles, nops);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0 && ms < best) best = ms;
        }
        CK(cudaGetLastError());
        const double tf = 32.0 * nops * double(n) / (best * 1e-3) / 1e12;
        std::printf("%s\"%s\": {\"ms\": %.3f, \"tflops\": %.2f, \"blocks_per_sm\": %d}",
                    mode ? ", " : "", names[mode], best, tf, per_sm);
    }
    std::printf("}\n");
    return 0;
}
