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

// Variant 4: the kernel's factor_diag as it stands (pivot rule, original diagonal, run-time pitch).
__global__ void k4(double *out, long long *cyc, int iters, int pitch, double gmax, unsigned *counter) {
    __shared__ double Aw[8 * 100], Lp[8 * LP_PITCH], invd[8];
    __shared__ int s_fail;
    const int lane = threadIdx.x;
    const int Wr = pitch - 2;
    if (lane == 0) s_fail = 0;
    if (lane < 8) { for (int c = 0; c < 8; ++c) Aw[lane * pitch + c] = (lane == c ? 10.0 + lane : 1.0 / (1 + lane + c)); Aw[lane * pitch + Wr] = 10.0 + lane; }
    __syncwarp();
    double pivmax = 0.0, sink = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double *Dg = Aw;
        const int r = lane & 7;
        double a[8], v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) { a[c] = (c <= r) ? Dg[(size_t)r * pitch + c] + 1e-9 * it : 0.0; v[c] = (c == r) ? 1.0 : 0.0; }
        const double d0 = Aw[(size_t)r * pitch + Wr];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double piv = __shfl_sync(FULL, a[c], c);
            const double orig = __shfl_sync(FULL, d0, c);
            bool pin = false;
            const double scale = fmax(pivmax, orig);
            if (!(piv == piv) || !(fabs(piv) < DBL_MAX)) { if (lane == 0 && s_fail == 0) s_fail = 2; }
            else if (!(piv > 1e-13 * scale)) {
                if ((pivmax == 0.0 && !(piv > 0.0)) || piv < -1e-8 * fmax(scale, gmax)) { if (lane == 0 && s_fail == 0) s_fail = 1; }
                else { pin = true; if (lane == 0) atomicAdd(counter, 1u); }
            }
            pivmax = fmax(pivmax, piv);
            const double inv = pin ? 0.0 : rsqrt(piv);
            a[c] = (r == c) ? (pin ? 1.0 : piv * inv) : a[c] * inv;
#pragma unroll
            for (int k = 0; k <= c; ++k) if (r == c) v[k] *= inv;
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) {
                const double lc2 = __shfl_sync(FULL, a[c], c2);
                if (r >= c2) a[c2] -= a[c] * lc2;
            }
#pragma unroll
            for (int k = 0; k <= c; ++k) {
                const double vk = __shfl_sync(FULL, v[k], c);
                if (r > c) v[k] -= a[c] * vk;
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
        pivmax = 0.0;
    }
    long long t1 = clock64();
    out[lane] = sink + pivmax + invd[lane & 7] + s_fail;
    if (lane == 0) *cyc = t1 - t0;
}
// Variant 5: the same with the pivot rule off the critical path (original diagonals broadcast up front, rsqrt issued before the test).
__global__ void k5(double *out, long long *cyc, int iters, int pitch, double gmax, unsigned *counter) {
    __shared__ double Aw[8 * 100], Lp[8 * LP_PITCH], invd[8];
    __shared__ int s_fail;
    const int lane = threadIdx.x;
    const int Wr = pitch - 2;
    if (lane == 0) s_fail = 0;
    if (lane < 8) { for (int c = 0; c < 8; ++c) Aw[lane * pitch + c] = (lane == c ? 10.0 + lane : 1.0 / (1 + lane + c)); Aw[lane * pitch + Wr] = 10.0 + lane; }
    __syncwarp();
    double pivmax = 0.0, sink = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double *Dg = Aw;
        const int r = lane & 7;
        double a[8], v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) { a[c] = (c <= r) ? Dg[(size_t)r * pitch + c] + 1e-9 * it : 0.0; v[c] = (c == r) ? 1.0 : 0.0; }
        double og[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) og[c] = Aw[(size_t)c * pitch + Wr];       // uniform loads: no shuffle in the chain
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double piv = __shfl_sync(FULL, a[c], c);
            double inv = rsqrt(piv);                                          // speculative: replaced below in the rare cases
            bool pin = false;
            const double scale = fmax(pivmax, og[c]);
            if (!(piv > 1e-13 * scale) || !(piv < DBL_MAX)) {                 // rare (warp-uniform): NaN / inf, noise-level or negative pivot
                if (!(piv == piv) || !(fabs(piv) < DBL_MAX)) { if (lane == 0 && s_fail == 0) s_fail = 2; }
                else if ((pivmax == 0.0 && !(piv > 0.0)) || piv < -1e-8 * fmax(scale, gmax)) { if (lane == 0 && s_fail == 0) s_fail = 1; }
                else { pin = true; if (lane == 0) atomicAdd(counter, 1u); }
                if (pin) inv = 0.0;
            }
            pivmax = fmax(pivmax, piv);
            a[c] = (r == c) ? (pin ? 1.0 : piv * inv) : a[c] * inv;
#pragma unroll
            for (int k = 0; k <= c; ++k) if (r == c) v[k] *= inv;
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) {
                const double lc2 = __shfl_sync(FULL, a[c], c2);
                if (r >= c2) a[c2] -= a[c] * lc2;
            }
#pragma unroll
            for (int k = 0; k <= c; ++k) {
                const double vk = __shfl_sync(FULL, v[k], c);
                if (r > c) v[k] -= a[c] * vk;
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
        pivmax = 0.0;
    }
    long long t1 = clock64();
    out[lane] = sink + pivmax + invd[lane & 7] + s_fail;
    if (lane == 0) *cyc = t1 - t0;
}
// Variant 6: variant 5 + the column broadcasts of the trailing update issued on the unscaled column, next to the pivot's
// (one shuffle latency per column instead of two): a[c2] -= (a[c] / piv) * a_c2[c].
__global__ void k6(double *out, long long *cyc, int iters, int pitch, double gmax, unsigned *counter) {
    __shared__ double Aw[8 * 100], Lp[8 * LP_PITCH], invd[8];
    __shared__ int s_fail;
    const int lane = threadIdx.x;
    const int Wr = pitch - 2;
    if (lane == 0) s_fail = 0;
    if (lane < 8) { for (int c = 0; c < 8; ++c) Aw[lane * pitch + c] = (lane == c ? 10.0 + lane : 1.0 / (1 + lane + c)); Aw[lane * pitch + Wr] = 10.0 + lane; }
    __syncwarp();
    double pivmax = 0.0, sink = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double *Dg = Aw;
        const int r = lane & 7;
        double a[8], v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) { a[c] = (c <= r) ? Dg[(size_t)r * pitch + c] + 1e-9 * it : 0.0; v[c] = (c == r) ? 1.0 : 0.0; }
        double og[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) og[c] = Aw[(size_t)c * pitch + Wr];       // uniform loads: no shuffle in the chain
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double piv = __shfl_sync(FULL, a[c], c);
            double raw[8];
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) raw[c2] = __shfl_sync(FULL, a[c], c2);   // unscaled A[c2][c]
            double inv = rsqrt(piv);                                          // speculative: replaced below in the rare cases
            bool pin = false;
            const double scale = fmax(pivmax, og[c]);
            if (!(piv > 1e-13 * scale) || !(piv < DBL_MAX)) {                 // rare (warp-uniform): NaN / inf, noise-level or negative pivot
                if (!(piv == piv) || !(fabs(piv) < DBL_MAX)) { if (lane == 0 && s_fail == 0) s_fail = 2; }
                else if ((pivmax == 0.0 && !(piv > 0.0)) || piv < -1e-8 * fmax(scale, gmax)) { if (lane == 0 && s_fail == 0) s_fail = 1; }
                else { pin = true; if (lane == 0) atomicAdd(counter, 1u); }
                if (pin) inv = 0.0;
            }
            pivmax = fmax(pivmax, piv);
            const double tsc = a[c] * (inv * inv);                            // a[r][c] / piv (0 for a pinned pivot)
#pragma unroll
            for (int c2 = c + 1; c2 < 8; ++c2) if (r >= c2) a[c2] = fma(-tsc, raw[c2], a[c2]);
            a[c] = (r == c) ? (pin ? 1.0 : piv * inv) : a[c] * inv;
#pragma unroll
            for (int k = 0; k <= c; ++k) if (r == c) v[k] *= inv;
#pragma unroll
            for (int k = 0; k <= c; ++k) {
                const double vk = __shfl_sync(FULL, v[k], c);
                if (r > c) v[k] -= a[c] * vk;
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
        pivmax = 0.0;
    }
    long long t1 = clock64();
    out[lane] = sink + pivmax + invd[lane & 7] + s_fail;
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
    for (int th : {32, 512}) {
        double *out; long long *cyc, h; unsigned *cnt;
        cudaMalloc(&out, 256 * 16); cudaMalloc(&cyc, 8); cudaMalloc(&cnt, 4); cudaMemset(cnt, 0, 4);
        k4<<<1, 32>>>(out, cyc, 10, 98, 1e3, cnt);
        k4<<<1, 32>>>(out, cyc, 1000, 98, 1e3, cnt);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-52s %.0f cycles per 8x8 block\n", "kernel's factor_diag (pivot rule, run-time pitch)", (double)h / 1000);
        k5<<<1, 32>>>(out, cyc, 10, 98, 1e3, cnt);
        k5<<<1, 32>>>(out, cyc, 1000, 98, 1e3, cnt);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-52s %.0f cycles per 8x8 block\n", "the same, pivot rule off the critical path", (double)h / 1000);
        k6<<<1, 32>>>(out, cyc, 10, 98, 1e3, cnt);
        k6<<<1, 32>>>(out, cyc, 1000, 98, 1e3, cnt);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-52s %.0f cycles per 8x8 block\n", "+ trailing-update broadcasts on the unscaled column", (double)h / 1000);
        (void)th;
        break;
    }
    return 0;
}
