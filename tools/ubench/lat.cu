// Micro-benchmarks of the instruction latencies / throughputs the regression kernels depend on (B200, sm_100a).
// One warp per SM sub-partition unless stated; clock64() around unrolled chains.
#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
__device__ __forceinline__ void mma_f64(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double *out, long long *cyc, int iters, double a, double b) {
    double x0 = a + threadIdx.x, x1 = b, x2 = a * 2, x3 = b * 3, y0 = 1, y1 = 2, y2 = 3, y3 = 4;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {          // dependent DFMA chain
#pragma unroll
            for (int u = 0; u < 16; ++u) x0 = fma(x0, a, b);
        } else if (MODE == 1) {   // 4 independent DFMA chains
#pragma unroll
            for (int u = 0; u < 4; ++u) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); }
        } else if (MODE == 2) {   // dependent DMMA chain
#pragma unroll
            for (int u = 0; u < 16; ++u) mma_f64(x0, x1, a, b);
        } else if (MODE == 3) {   // 4 independent DMMA chains
#pragma unroll
            for (int u = 0; u < 4; ++u) { mma_f64(x0, x1, a, b); mma_f64(x2, x3, a, b); mma_f64(y0, y1, a, b); mma_f64(y2, y3, a, b); }
        } else if (MODE == 4) {   // dependent 64-bit shuffle chain
#pragma unroll
            for (int u = 0; u < 16; ++u) x0 = __shfl_xor_sync(FULL, x0, 1);
        } else if (MODE == 5) {   // independent 64-bit shuffles
#pragma unroll
            for (int u = 0; u < 4; ++u) { x0 = __shfl_xor_sync(FULL, x0, 1); x1 = __shfl_xor_sync(FULL, x1, 2); x2 = __shfl_xor_sync(FULL, x2, 4); x3 = __shfl_xor_sync(FULL, x3, 8); }
        } else if (MODE == 6) {   // sqrt + reciprocal chain
#pragma unroll
            for (int u = 0; u < 4; ++u) { x0 = sqrt(x0 + 2.0); x0 = 1.0 / (x0 * (x0 + 1.5)); }
        } else if (MODE == 7) {   // rsqrt chain
#pragma unroll
            for (int u = 0; u < 8; ++u) x0 = rsqrt(x0 + 2.0);
        } else if (MODE == 8) {   // DFMA feeding a shuffle feeding a DFMA (reduction step)
#pragma unroll
            for (int u = 0; u < 8; ++u) { x0 = fma(x0, a, b); x0 += __shfl_xor_sync(FULL, x0, 1); }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + y0 + y1 + y2 + y3;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE>
void run(const char *name, int ops_per_iter, int threads, int blocks) {
    double *out; long long *cyc, h;
    cudaMalloc(&out, sizeof(double) * threads * blocks); cudaMalloc(&cyc, 8);
    const int iters = 2000;
    k<MODE><<<blocks, threads>>>(out, cyc, 10, 1.0000001, 1e-9);
    k<MODE><<<blocks, threads>>>(out, cyc, iters, 1.0000001, 1e-9);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-44s threads/CTA %4d: %.2f cycles per op per warp (%.2f per op per SM with %d warps)\n", name, threads,
           (double)h / iters / ops_per_iter, (double)h / iters / ops_per_iter / (threads / 32), threads / 32);
    cudaFree(out); cudaFree(cyc);
}
int main() {
    for (int th : {32, 128, 256, 512, 1024}) {
        run<0>("DFMA dependent chain", 16, th, 148);
        run<1>("DFMA 4 independent chains", 16, th, 148);
        run<2>("DMMA m8n8k4 dependent chain", 16, th, 148);
        run<3>("DMMA 4 independent chains", 16, th, 148);
        run<4>("SHFL.64 dependent chain", 16, th, 148);
        run<5>("SHFL.64 4 independent", 16, th, 148);
        run<6>("sqrt + 1/(x(x+c)) chain (pairs)", 4, th, 148);
        run<7>("rsqrt chain", 8, th, 148);
        run<8>("DFMA -> SHFL.64 -> DADD chain (steps)", 8, th, 148);
    }
    return 0;
}
