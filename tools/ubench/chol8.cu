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

// Variant 3: every lane holds the whole lower triangle and factors it redundantly (no shuffles); lane j solves for
// column j of the inverse.
__global__ void k3(double *out, long long *cyc, int iters) {
    __shared__ double Dg[8 * 12], Lp[8 * LP_PITCH], invd[8];
    const int lane = threadIdx.x;
    if (lane < 8) for (int c = 0; c < 8; ++c) Dg[lane * 12 + c] = (lane == c ? 10.0 + lane : 1.0 / (1 + lane + c));
    __syncwarp();
    double pivmax = 0.0, sink = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int r = lane & 7;
        double a[8][8], li[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int c = 0; c <= i; ++c) a[i][c] = Dg[i * 12 + c] + 1e-9 * it;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double piv = a[c][c];
            pivmax = fmax(pivmax, piv);
            const double inv = rsqrt(piv);
            li[c] = inv;
            a[c][c] = piv * inv;
#pragma unroll
            for (int i = c + 1; i < 8; ++i) a[i][c] *= inv;
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2)
#pragma unroll
                for (int i = c2; i < 8; ++i) a[i][c2] = fma(-a[i][c], a[c2][c], a[i][c2]);
        }
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int kk = 0; kk < i; ++kk) { if (kk & 1) s1 = fma(a[i][kk], x[kk], s1); else s0 = fma(a[i][kk], x[kk], s0); }
            x[i] = (i == r) ? li[i] : -li[i] * (s0 + s1);
        }
        if (lane < 8) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double lv = a[c][c];
#pragma unroll
                for (int i = c + 1; i < 8; ++i) lv = (r == i) ? a[i][c] : lv;
                if (c <= r) Lp[r * LP_PITCH + c] = lv;
            }
#pragma unroll
            for (int i = 1; i < 8; ++i) if (i > r) Lp[r * LP_PITCH + i] = x[i];
            invd[r] = (r == 0) ? x[0] : (r == 1) ? x[1] : (r == 2) ? x[2] : (r == 3) ? x[3] : (r == 4) ? x[4] : (r == 5) ? x[5] : (r == 6) ? x[6] : x[7];
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
    {
        double *out; long long *cyc, h;
        cudaMalloc(&out, 256); cudaMalloc(&cyc, 8);
        k3<<<1, 32>>>(out, cyc, 10);
        k3<<<1, 32>>>(out, cyc, 1000);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-52s %.0f cycles per 8x8 block\n", "every lane the whole triangle + column-wise inverse", (double)h / 1000);
    }
    return 0;
}
