// spk_verify.cu — verification and refinement on the device (SURVEY.md §8(f)
// rows 1-2): everything the reference does on the host around the solver to
// check or improve a solution, without moving n x nrhs blocks over PCIe.
//
//   k_band_mm_dmma     Y = op(A) X or R = F - op(A) X      band_ops.cpp:11-37 (band_matmul),
//                                                          solve.cpp:412-413 (the refinement residual)
//   k_col_stats(_reduce) per column sum|x|, sum x^2, max|x|  band_ops.cpp:45-57 (frobenius_norm /
//                                                          relative_residual), oracle.cpp:132-166 (|y|_1)
//   k_band_rownorm / k_band_colnorm  ||A||_inf, ||A||_1, max|a|  band_ops.cpp:59-69 (norm1, max_abs)
//   k_axpy, k_sign, k_dot_argmax, k_unit   refinement update (solve.cpp:428-429) and the
//                                          Hager estimator's vector steps (oracle.cpp:132-166)
//
// The band product is a masked GEMM on the tensor cores: the packed band is
// a dense column-major matrix with leading dimension kl+ku once entries
// outside the band are masked (A(i,j) at band[j*ld + ku + i - j]).  A CTA
// computes a 64x64 tile of the result over the K range its rows touch
// (64 + kl + ku columns), staging masked band tiles and X tiles through
// shared memory with cp.async (double buffer), 4 warps x 4x4 DMMA m8n8k4
// accumulators.  All reductions are deterministic: sums in a fixed order
// (per-block partials, then an ordered pass), maxima by atomicMax on the bit
// pattern of non-negative doubles (order-free).
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_sweep_fast.cuh"

#include <algorithm>
#include <cfloat>

namespace spk {

namespace {
constexpr int VM = 64, VN = 64, VK = 16;
constexpr int VSA = VK + 4, VSB = VK + 4;

__device__ __forceinline__ void vdmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
    atomicMax(p, (unsigned long long)__double_as_longlong(v));
}
}  // namespace

// Y = op(A) X (F == nullptr) or Y = F - op(A) X.  grid (ceil(n/64), ceil(ncols/64)).
template <bool TRANS>
__global__ void __launch_bounds__(128) k_band_mm_dmma(const double* __restrict__ band, long long n, int kl, int ku,
                                                      const double* __restrict__ X, long long ldx, int ncols,
                                                      const double* __restrict__ F, long long ldf,
                                                      double* __restrict__ Y, long long ldy) {
    __shared__ __align__(16) double sA[2][VM * VSA];
    __shared__ __align__(16) double sB[2][VN * VSB];
    const int ld = kl + ku + 1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const int g = lane >> 2, q = lane & 3;
    const long long row0 = (long long)blockIdx.x * VM;
    const int col0 = blockIdx.y * VN;
    // op(A)(i, j) != 0 only for j in [i - lo, i + hi]
    const int lo = TRANS ? ku : kl, hi = TRANS ? kl : ku;
    const long long kbeg = max(0LL, row0 - lo), kend = min(n, row0 + VM + hi);
    auto stage = [&](int buf, long long k0) {
        for (int idx = tid; idx < VM * VK; idx += 128) {
            int i, l;
            if (TRANS) {  // row gi of A^T = column gi of A: contiguous over gj
                l = idx % VK;
                i = idx / VK;
            } else {  // column gj of A: contiguous over gi
                i = idx % VM;
                l = idx / VM;
            }
            double* dst = &sA[buf][i * VSA + l];
            const long long gi = row0 + i, gj = k0 + l;
            const long long d = gi - gj;  // op(A)(gi, gj) nonzero for -hi <= d <= lo
            if (gi < n && gj < kend && d <= lo && -d <= hi) {
                const double* src = TRANS ? band + gi * ld + ku + (gj - gi) : band + gj * ld + ku + (gi - gj);
                cp_async8(dst, src);
            } else {
                *dst = 0.0;
            }
        }
        for (int idx = tid; idx < VK * VN; idx += 128) {
            const int l = idx % VK, c = idx / VK;
            double* dst = &sB[buf][c * VSB + l];
            const long long gj = k0 + l;
            const int gc = col0 + c;
            if (gj < kend && gc < ncols) cp_async8(dst, X + (long long)gc * ldx + gj);
            else *dst = 0.0;
        }
        cp_async_commit();
    };
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int nk = kend > kbeg ? (int)((kend - kbeg + VK - 1) / VK) : 0;
    if (nk > 0) stage(0, kbeg);
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nk) {
            stage(buf ^ 1, kbeg + (long long)(kc + 1) * VK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* a_s = sA[buf];
        const double* b_s = sB[buf];
#pragma unroll
        for (int ks = 0; ks < VK; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = a_s[(wm + 8 * a + g) * VSA + ks + q];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = b_s[(wn + 8 * b + g) * VSB + ks + q];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) vdmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const long long i = row0 + wm + 8 * a + g;
        if (i >= n) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = col0 + wn + 8 * b + 2 * q + e;
                if (c >= ncols) continue;
                const double v = acc[a][b][e];
                Y[(long long)c * ldy + i] = F ? F[(long long)c * ldf + i] - v : v;
            }
    }
}

// Per-column statistics, pass 1: block b of column c covers rows
// [b*chunk, (b+1)*chunk); part[(c*nblk + b)*3 + {0,1,2}] = {sum|x|, sum x^2, max|x|}.
__global__ void __launch_bounds__(256) k_col_stats(const double* __restrict__ X, long long ldx, long long n,
                                                   long long chunk, int nblk, double* __restrict__ part) {
    const int b = blockIdx.x, c = blockIdx.y;
    const double* x = X + (long long)c * ldx;
    const long long r0 = (long long)b * chunk, r1 = min(n, r0 + chunk);
    double s1 = 0.0, s2 = 0.0, mx = 0.0;
    for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const double v = x[r];
        s1 += fabs(v);
        s2 += v * v;
        mx = fmax(mx, fabs(v));
    }
    __shared__ double sh[3][256];
    sh[0][threadIdx.x] = s1;
    sh[1][threadIdx.x] = s2;
    sh[2][threadIdx.x] = mx;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {  // fixed tree: deterministic
        if (threadIdx.x < o) {
            sh[0][threadIdx.x] += sh[0][threadIdx.x + o];
            sh[1][threadIdx.x] += sh[1][threadIdx.x + o];
            sh[2][threadIdx.x] = fmax(sh[2][threadIdx.x], sh[2][threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* p = part + ((long long)c * nblk + b) * 3;
        p[0] = sh[0][0];
        p[1] = sh[1][0];
        p[2] = sh[2][0];
    }
}

// pass 2: out[c*3 + ...] = the blocks of column c combined in block order
__global__ void k_col_stats_reduce(const double* __restrict__ part, int nblk, int ncols, double* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    double s1 = 0.0, s2 = 0.0, mx = 0.0;
    for (int b = 0; b < nblk; ++b) {
        const double* p = part + ((long long)c * nblk + b) * 3;
        s1 += p[0];
        s2 += p[1];
        mx = fmax(mx, p[2]);
    }
    out[c * 3 + 0] = s1;
    out[c * 3 + 1] = s2;
    out[c * 3 + 2] = mx;
}

// row abs sums (||A||_inf) and max|a|: thread per row; the CTA walks the
// absolute columns its rows touch, so a warp's loads of one column are
// contiguous.  out[1] = ||A||_inf bits, out[2] = max|a| bits.
__global__ void __launch_bounds__(256) k_band_rownorm(const double* __restrict__ band, long long n, int kl, int ku,
                                                      unsigned long long* __restrict__ out) {
    const int ld = kl + ku + 1;
    const long long i0 = (long long)blockIdx.x * blockDim.x;
    const long long i = i0 + threadIdx.x;
    const long long j0 = max(0LL, i0 - kl), j1 = min(n - 1, i0 + (long long)blockDim.x - 1 + ku);
    double s = 0.0, mx = 0.0;
    for (long long j = j0; j <= j1; ++j) {
        const long long d = i - j;
        if (i < n && d <= kl && -d <= ku) {
            const double v = fabs(band[j * ld + ku + d]);
            s += v;
            mx = fmax(mx, v);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(&out[1], s);
        atomic_max_nonneg(&out[2], mx);
    }
}

// column abs sums (||A||_1): warp per column, lanes over its band rows.
// out[0] = ||A||_1 bits.
__global__ void __launch_bounds__(256) k_band_colnorm(const double* __restrict__ band, long long n, int kl, int ku,
                                                      unsigned long long* __restrict__ out) {
    const int ld = kl + ku + 1;
    const long long j = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    if (j < n)
        for (int r = lane; r < ld; r += 32) {
            const long long i = j + r - ku;
            if (i >= 0 && i < n) s += fabs(band[j * ld + r]);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && j < n) atomic_max_nonneg(&out[0], s);
}

// X[:, c] += D[:, c]
__global__ void k_axpy(double* __restrict__ X, long long ldx, const double* __restrict__ D, long long ldd,
                       long long n, int ncols) {
    const long long total = n * ncols;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / n, r = e - c * n;
        X[c * ldx + r] += D[c * ldd + r];
    }
}

// xi = sign(y) with sign(0) = +1 (oracle.cpp:148)
__global__ void k_sign(const double* __restrict__ y, double* __restrict__ xi, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        xi[i] = y[i] >= 0.0 ? 1.0 : -1.0;
}

// per block: sum z_i x_i (fixed order) and the first argmax |z_i|;
// part[b] = {dot, max, index}
__global__ void __launch_bounds__(256) k_dot_argmax(const double* __restrict__ z, const double* __restrict__ x,
                                                    long long n, long long chunk, double* __restrict__ part) {
    const long long r0 = (long long)blockIdx.x * chunk, r1 = min(n, r0 + chunk);
    double dot = 0.0, best = -1.0;
    long long bi = n;
    for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        dot += z[i] * x[i];
        const double a = fabs(z[i]);
        if (a > best) {
            best = a;
            bi = i;
        }
    }
    __shared__ double sd[256], sb[256];
    __shared__ long long si[256];
    sd[threadIdx.x] = dot;
    sb[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sd[threadIdx.x] += sd[threadIdx.x + o];
            const double ob = sb[threadIdx.x + o];
            const long long oi = si[threadIdx.x + o];
            if (ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x])) {
                sb[threadIdx.x] = ob;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x * 3 + 0] = sd[0];
        part[blockIdx.x * 3 + 1] = sb[0];
        part[blockIdx.x * 3 + 2] = (double)si[0];
    }
}

// x = e_j
__global__ void k_unit(double* __restrict__ x, long long n, long long j) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = i == j ? 1.0 : 0.0;
}

__global__ void k_fill(double* __restrict__ x, long long n, double v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        x[i] = v;
}

// ---------------------------------------------------------------------------
// launchers
static unsigned vgrid(long long work, int per, long long cap) {
    long long g = (work + per - 1) / per;
    return (unsigned)std::max(1LL, std::min(g, cap));
}

void launch_band_mm(const double* band, long long n, int kl, int ku, const double* X, long long ldx, int ncols,
                    int transpose, const double* F, long long ldf, double* Y, long long ldy, cudaStream_t s) {
    if (n <= 0 || ncols <= 0) return;
    const dim3 grid((unsigned)((n + VM - 1) / VM), (unsigned)((ncols + VN - 1) / VN));
    if (transpose) k_band_mm_dmma<true><<<grid, 128, 0, s>>>(band, n, kl, ku, X, ldx, ncols, F, ldf, Y, ldy);
    else k_band_mm_dmma<false><<<grid, 128, 0, s>>>(band, n, kl, ku, X, ldx, ncols, F, ldf, Y, ldy);
    count_launch();
}

int col_stats_blocks(long long n) { return (int)std::min<long long>(std::max<long long>(1, (n + 8191) / 8192), 256); }

void launch_col_stats(const double* X, long long ldx, long long n, int ncols, double* part, double* out,
                      cudaStream_t s) {
    if (n <= 0 || ncols <= 0) return;
    const int nblk = col_stats_blocks(n);
    const long long chunk = (n + nblk - 1) / nblk;
    k_col_stats<<<dim3(nblk, ncols), 256, 0, s>>>(X, ldx, n, chunk, nblk, part);
    count_launch();
    k_col_stats_reduce<<<(ncols + 127) / 128, 128, 0, s>>>(part, nblk, ncols, out);
    count_launch();
}

void launch_band_norms(const double* band, long long n, int kl, int ku, unsigned long long* out, cudaStream_t s) {
    if (n <= 0) return;
    k_band_rownorm<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(band, n, kl, ku, out);
    count_launch();
    k_band_colnorm<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(band, n, kl, ku, out);
    count_launch();
}

void launch_axpy(double* X, long long ldx, const double* D, long long ldd, long long n, int ncols, cudaStream_t s) {
    if (n <= 0 || ncols <= 0) return;
    k_axpy<<<vgrid(n * ncols, 256, 148LL * 16), 256, 0, s>>>(X, ldx, D, ldd, n, ncols);
    count_launch();
}

void launch_sign(const double* y, double* xi, long long n, cudaStream_t s) {
    k_sign<<<vgrid(n, 256, 148LL * 8), 256, 0, s>>>(y, xi, n);
    count_launch();
}

int dot_argmax_blocks(long long n) { return (int)std::min<long long>(std::max<long long>(1, (n + 8191) / 8192), 256); }

void launch_dot_argmax(const double* z, const double* x, long long n, double* part, cudaStream_t s) {
    const int nblk = dot_argmax_blocks(n);
    k_dot_argmax<<<nblk, 256, 0, s>>>(z, x, n, (n + nblk - 1) / nblk, part);
    count_launch();
}

void launch_unit(double* x, long long n, long long j, cudaStream_t s) {
    k_unit<<<vgrid(n, 256, 148LL * 8), 256, 0, s>>>(x, n, j);
    count_launch();
}

void launch_fill(double* x, long long n, double v, cudaStream_t s) {
    k_fill<<<vgrid(n, 256, 148LL * 8), 256, 0, s>>>(x, n, v);
    count_launch();
}

}  // namespace spk
