// Latency of the in-register 8x8 Cholesky + inverse used by K3b's warp 0 (one warp, shared-memory input/output).
#include <cstdio>
#include <cfloat>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
#define LP_PITCH 10
template <int VARIANT>
__global__ void k(double *out, long long *cyc, int iters) {
    __shared__ double Dg[8 * 12], Lp[8 * LP_PITCH], invd[8];
    const int lane = threadIdx.x;
    if (lane < 8) for (int c = 0; c < 8; ++c) Dg[lane * 12 + c] = (lane == c ? 10.0 + lane : 1.0 / (1 + lane + c));
    __syncwarp();
    double pivmax = 0.0, sink = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int r = lane & 7;
        double a[8], v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) { a[c] = (c <= r) ? Dg[r * 12 + c] + 1e-9 * it : 0.0; v[c] = (c == r) ? 1.0 : 0.0; }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double piv = __shfl_sync(FULL, a[c], c);
            pivmax = fmax(pivmax, piv);
            const double inv = (VARIANT == 1) ? 1.0 / sqrt(piv) : rsqrt(piv);
            a[c] = (r == c) ? piv * inv : a[c] * inv;
            if (VARIANT != 2) {
#pragma unroll
                for (int k = 0; k <= c; ++k) if (r == c) v[k] *= inv;
            }
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) {
                const double lc2 = __shfl_sync(FULL, a[c], c2);
                if (r >= c2) a[c2] -= a[c] * lc2;
            }
            if (VARIANT != 2) {
#pragma unroll
                for (int k = 0; k <= c; ++k) {
                    const double vk = __shfl_sync(FULL, v[k], c);
                    if (r > c) v[k] -= a[c] * vk;
                }
            }
        }
        if (lane < 8) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (c <= r) Lp[r * LP_PITCH + c] = a[c];
                if (c < r) Lp[c * LP_PITCH + r] = v[c];
            }
            invd[r] = v[r];
        }
        __syncwarp();
        sink += Lp[(lane & 7) * LP_PITCH + (lane >> 3)];
    }
    long long t1 = clock64();
    out[lane] = sink + pivmax + invd[lane & 7];
    if (lane == 0) *cyc = t1 - t0;
}
template <int V> void run(const char *name) {
    double *out; long long *cyc, h;
    cudaMalloc(&out, 256); cudaMalloc(&cyc, 8);
    k<V><<<1, 32>>>(out, cyc, 10);
    k<V><<<1, 32>>>(out, cyc, 1000);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-52s %.0f cycles per 8x8 block\n", name, (double)h / 1000);
}
int main() {
    run<0>("Cholesky + inverse, rsqrt");
    run<1>("Cholesky + inverse, 1/sqrt");
    run<2>("Cholesky only, rsqrt");
    return 0;
}
