// Micro-benchmarks of the MIO pipe (B200, sm_100a): do shuffles and shared-memory wavefronts share one issue port, and
// what does a broadcast LDS.64 / LDS.128 (4 distinct 8 / 16-byte addresses per warp) cost next to 64-bit shuffles?
// Throughput per SM with W warps resident; all operations independent (4 chains).
#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
__device__ __forceinline__ double lds64(const double *p) {
    double v; unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds128(const double *p) {
    double2 v; unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
template <int MODE>
__global__ void k(double *out, long long *cyc, int iters, int stride) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, t4 = lane & 3, g8 = lane >> 2;
    double *base = sm + w * 1024;
    for (int i = lane; i < 1024; i += 32) base[i] = i * 0.5 + w;
    __syncthreads();
    double x0 = lane, x1 = 2 * lane, x2 = 3, x3 = 4;
    const double *pb = base + 2 * t4;                 // broadcast: 4 distinct 16-byte chunks
    const double *pd = base + stride * g8 + 2 * t4;   // distinct: 32 distinct 16-byte chunks
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int o = 64 * u + 8 * (i & 7);
            if (MODE == 0) {          // 4 x SHFL.64 (8 SHFL)
                x0 += __shfl_sync(FULL, x0, 4 * u + t4); x1 += __shfl_sync(FULL, x1, 4 * u + t4);
                x2 += __shfl_sync(FULL, x2, 4 * u + t4); x3 += __shfl_sync(FULL, x3, 4 * u + t4);
            } else if (MODE == 1) {   // 4 x broadcast LDS.64
                x0 += lds64(pb + o); x1 += lds64(pb + o + 8); x2 += lds64(pb + o + 16); x3 += lds64(pb + o + 24);
            } else if (MODE == 2) {   // 4 x broadcast LDS.128 (8 doubles)
                const double2 a = lds128(pb + o), b = lds128(pb + o + 8);
                const double2 c = lds128(pb + o + 16), d = lds128(pb + o + 24);
                x0 += a.x + a.y; x1 += b.x + b.y; x2 += c.x + c.y; x3 += d.x + d.y;
            } else if (MODE == 3) {   // 4 x distinct LDS.64 (lane-contiguous)
                const double *q = base + lane + o;
                x0 += lds64(q); x1 += lds64(q + 32); x2 += lds64(q + 64); x3 += lds64(q + 96);
            } else if (MODE == 4) {   // 4 x distinct LDS.128, pitch `stride` doubles between lane groups
                const double2 a = lds128(pd + (o & 63)), b = lds128(pd + (o & 63) + 8);
                const double2 c = lds128(pd + (o & 63) + 16), d = lds128(pd + (o & 63) + 24);
                x0 += a.x + a.y; x1 += b.x + b.y; x2 += c.x + c.y; x3 += d.x + d.y;
            } else if (MODE == 5) {   // 2 x SHFL.64 + 2 x broadcast LDS.128 (shared port?)
                x0 += __shfl_sync(FULL, x0, 4 * u + t4); x1 += __shfl_sync(FULL, x1, 4 * u + t4);
                const double2 c = lds128(pb + o + 16), d = lds128(pb + o + 24);
                x2 += c.x + c.y; x3 += d.x + d.y;
            } else if (MODE == 6) {   // 4 x STS.128 from 4 active lanes
                if (g8 == (i & 7)) {
                    *reinterpret_cast<double2 *>(base + 2 * t4 + o) = make_double2(x0, x1);
                    *reinterpret_cast<double2 *>(base + 2 * t4 + o + 8) = make_double2(x1, x2);
                    *reinterpret_cast<double2 *>(base + 2 * t4 + o + 16) = make_double2(x2, x3);
                    *reinterpret_cast<double2 *>(base + 2 * t4 + o + 24) = make_double2(x3, x0);
                }
            } else if (MODE == 7) {   // 4 x STS.64 from 4 active lanes
                if (g8 == (i & 7)) {
                    base[t4 + o] = x0; base[t4 + o + 8] = x1; base[t4 + o + 16] = x2; base[t4 + o + 24] = x3;
                }
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + base[lane];
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE>
void run(const char *name, int threads, int stride = 8) {
    double *out; long long *cyc, h;
    const int blocks = 148;
    cudaMalloc(&out, sizeof(double) * threads * blocks); cudaMalloc(&cyc, 8);
    const int iters = 4000;
    const size_t smem = (threads / 32) * 1024 * sizeof(double);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<MODE><<<blocks, threads, smem>>>(out, cyc, 10, stride);
    k<MODE><<<blocks, threads, smem>>>(out, cyc, iters, stride);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-52s warps/SM %2d: %.2f cycles per group of 4 per SM\n", name, threads / 32, (double)h / iters / 4 / (threads / 32));
    cudaFree(out); cudaFree(cyc);
}
int main() {
    for (int th : {128, 256, 512}) {
        run<0>("4 x SHFL.64 (idx)", th);
        run<1>("4 x LDS.64 broadcast (4 distinct)", th);
        run<2>("4 x LDS.128 broadcast (4 distinct)", th);
        run<3>("4 x LDS.64 distinct lane-contiguous", th);
        run<4>("4 x LDS.128 distinct pitch 8", th, 8);
        run<4>("4 x LDS.128 distinct pitch 12", th, 12);
        run<5>("2 x SHFL.64 + 2 x LDS.128 broadcast", th);
        run<6>("4 x STS.128 4 lanes", th);
        run<7>("4 x STS.64 4 lanes", th);
    }
    return 0;
}
