// diag_bench.cu -- latency of the 8x8 diagonal-block factorization used by the
// blocked LU (k_band_lu_dmma), one warp, no contention.
#include <cstdio>
__device__ __forceinline__ int afrag(int m, int k) { return (k >> 2) * 32 + m * 4 + (k & 3); }
__device__ __forceinline__ int bfrag(int k, int n) { return (k >> 2) * 32 + n * 4 + (k & 3); }

template <int VAR>
__global__ void k_bench(double* out, long long* cyc, int reps) {
    __shared__ double sm[64 * 4 + 16];
    const int lane = threadIdx.x, gi = lane >> 2, q = lane & 3;
    const unsigned full = 0xffffffffu;
    double lu0 = (gi == 2 * q ? 10.0 : 0.1 * (gi + q)), lu1 = (gi == 2 * q + 1 ? 10.0 : 0.2 * (gi - q));
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double* sDinv = sm + 256;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int src = c * 4 + (c >> 1);
            double pv = __shfl_sync(full, (c & 1) ? lu1 : lu0, src);
            const double lraw = __shfl_sync(full, (c & 1) ? lu1 : lu0, gi * 4 + (c >> 1));
            const double u0 = __shfl_sync(full, lu0, c * 4 + q);
            const double u1 = __shfl_sync(full, lu1, c * 4 + q);
            double inv;
            if (VAR == 0) {
                asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(pv));
                double e = fma(-pv, inv, 1.0);
                inv = fma(inv, e, inv);
                e = fma(-pv, inv, 1.0);
                inv = fma(inv, e, inv);
            } else {
                inv = 1.0 / pv;
            }
            if (lane == 0) sDinv[c] = inv;
            const double lr = lraw * inv;
            if (gi > c) {
                const int c0 = 2 * q, c1 = 2 * q + 1;
                lu0 = c0 > c ? fma(-lr, u0, lu0) : (c0 == c ? lr : lu0);
                lu1 = c1 > c ? fma(-lr, u1, lu1) : (c1 == c ? lr : lu1);
            }
        }
        long long t1 = clock64();
        double x0 = gi == 2 * q, x1 = gi == 2 * q + 1, y0 = x0, y1 = x1;
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            if (s < 7) {
                const int k = s;
                const double lik = __shfl_sync(full, (k & 1) ? lu1 : lu0, gi * 4 + (k >> 1));
                const double xk0 = __shfl_sync(full, x0, k * 4 + q);
                const double xk1 = __shfl_sync(full, x1, k * 4 + q);
                if (gi > k) {
                    x0 = fma(-lik, xk0, x0);
                    x1 = fma(-lik, xk1, x1);
                }
            }
            {
                const int k = 7 - s;
                if (gi == k) {
                    const double dk = sDinv[k];
                    y0 *= dk;
                    y1 *= dk;
                }
                const double yk0 = __shfl_sync(full, y0, k * 4 + q);
                const double yk1 = __shfl_sync(full, y1, k * 4 + q);
                const double uik = __shfl_sync(full, (k & 1) ? lu1 : lu0, gi * 4 + (k >> 1));
                if (gi < k) {
                    y0 = fma(-uik, yk0, y0);
                    y1 = fma(-uik, yk1, y1);
                }
            }
        }
        sm[afrag(gi, 2 * q)] = x0;
        sm[64 + bfrag(gi, 2 * q)] = y0 + x1 + y1;
        long long t2 = clock64();
        if (lane == 0 && r == reps - 1) { cyc[0] = t1; cyc[1] = t2; }
        lu0 += 1e-3 * x0;
        lu1 += 1e-3 * y1;
    }
    long long t3 = clock64();
    if (lane == 0) { cyc[2] = t3 - t0; }
    out[lane] = lu0 + lu1;
}

// lockstep: LU, X = L^-1 and Z = U^-T in one pass over the 8 pivots
__global__ void k_bench2(double* out, long long* cyc, int reps) {
    __shared__ double sm[64 * 4 + 16];
    const int lane = threadIdx.x, gi = lane >> 2, q = lane & 3;
    const unsigned full = 0xffffffffu;
    double lu0 = (gi == 2 * q ? 10.0 : 0.1 * (gi + q)), lu1 = (gi == 2 * q + 1 ? 10.0 : 0.2 * (gi - q));
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double x0 = gi == 2 * q, x1 = gi == 2 * q + 1, z0 = x0, z1 = x1;
        double dinv_mine = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int src = c * 4 + (c >> 1);
            const double pv = __shfl_sync(full, (c & 1) ? lu1 : lu0, src);
            const double lraw = __shfl_sync(full, (c & 1) ? lu1 : lu0, gi * 4 + (c >> 1));
            const double u0 = __shfl_sync(full, lu0, c * 4 + q);
            const double u1 = __shfl_sync(full, lu1, c * 4 + q);
            const double ua = __shfl_sync(full, lu0, c * 4 + (gi >> 1));
            const double ub = __shfl_sync(full, lu1, c * 4 + (gi >> 1));
            const double xk0 = __shfl_sync(full, x0, c * 4 + q);
            const double xk1 = __shfl_sync(full, x1, c * 4 + q);
            double inv;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(pv));
            double e = fma(-pv, inv, 1.0);
            inv = fma(inv, e, inv);
            e = fma(-pv, inv, 1.0);
            inv = fma(inv, e, inv);
            dinv_mine = lane == c ? inv : dinv_mine;
            const double lr = lraw * inv;
            const bool below = gi > c;
            const int c0 = 2 * q, c1 = 2 * q + 1;
            // LU
            const double n0 = fma(-lr, u0, lu0), n1 = fma(-lr, u1, lu1);
            lu0 = below ? (c0 > c ? n0 : (c0 == c ? lr : lu0)) : lu0;
            lu1 = below ? (c1 > c ? n1 : (c1 == c ? lr : lu1)) : lu1;
            // X = L^-1: rows below take -l * (row c of X)
            x0 = below ? fma(-lr, xk0, x0) : x0;
            x1 = below ? fma(-lr, xk1, x1) : x1;
            // Z = U^-T: row c scales by 1/u_cc, rows below take -u(c, gi) * (row c of Z)
            if (gi == c) {
                z0 *= inv;
                z1 *= inv;
            }
            const double zc0 = __shfl_sync(full, z0, c * 4 + q);
            const double zc1 = __shfl_sync(full, z1, c * 4 + q);
            const double ucg = (gi & 1) ? ub : ua;
            z0 = below ? fma(-ucg, zc0, z0) : z0;
            z1 = below ? fma(-ucg, zc1, z1) : z1;
        }
        if (lane < 8) sm[256 + lane] = dinv_mine;
        sm[gi * 8 + 2 * q] = lu0;
        sm[gi * 8 + 2 * q + 1] = lu1;
        sm[64 + afrag(gi, 2 * q)] = x0;
        sm[64 + afrag(gi, 2 * q + 1)] = x1;
        sm[128 + bfrag(2 * q, gi)] = z0;
        sm[128 + bfrag(2 * q + 1, gi)] = z1;
        lu0 += 1e-3 * x0;
        lu1 += 1e-3 * z1;
    }
    long long t3 = clock64();
    if (lane == 0) { cyc[2] = t3 - t0; }
    out[lane] = lu0 + lu1;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 256); cudaMalloc(&cyc, 64);
    long long h[3];
    for (int var = 0; var < 2; ++var) {
        for (int it = 0; it < 2; ++it) {
            if (var == 0) k_bench<0><<<1, 32>>>(out, cyc, 1000); else k_bench<1><<<1, 32>>>(out, cyc, 1000);
            cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
        }
        printf("variant %s: %.0f clk per 8x8 factor+inverses (last: LU %lld, inverses %lld)\n",
               var == 0 ? "rcp+newton" : "ieee div", h[2] / 1000.0, 0LL, h[1] - h[0]);
    }
    for (int it = 0; it < 2; ++it) {
        k_bench2<<<1, 32>>>(out, cyc, 1000);
        cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
    }
    printf("variant lockstep: %.0f clk per 8x8 factor+inverses\n", h[2] / 1000.0);
    return 0;
}
