// spk_smallk_solve.cu — the small-k engine's forward solve (k_sk_solve), see
// spk_smallk.cu for the engine: D-stage per partition, the reduced solve
// level by level, retrieval per partition, one cooperative kernel.
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_smallk.cuh"

#include <cuda_runtime.h>

#include <algorithm>

namespace spk {

// ===========================================================================
// forward solve: D-stage, reduced levels, retrieval (one cooperative kernel)
namespace {
constexpr int kSkSvWarps = 4;

// Forward L then backward U over one partition's rows (LU space) for nr <= 8
// columns.  Lanes hold the window rows (forward: row r in lane r mod 32,
// backward: row r in lane (m-1-r) mod 32), so a step is one shuffle of the
// pivot row's x and one FMA per column on the rows it updates; the factor
// entries of the next kSkPf steps (each lane's own row: L column j / U column
// j, contiguous in the packed factor) and the rows entering the window are
// prefetched into register rings, so no step waits on memory.  x enters from
// load(r, c); the forward results go to the warp's Xs (m x 8); the backward
// value of row j (j >= bwd_lo) goes to store(j, c, v).
constexpr int kSkPf = 8;

template <int NR, class Load, class Store>
__device__ void sk_fwd_bwd(const PartDev& P, const double* fac, double* Xs, int lane, int bwd_lo, Load load,
                           Store store) {
    const unsigned full = 0xffffffffu;
    const int m = P.m, kl = P.kl, ku = P.ku, rows = P.rows, d = P.d;
    const double* F = fac + P.fofs;
    double x[NR];
    double rf[kSkPf];       // factor entry of step j + s for this lane's row
    double rx[kSkPf][NR];   // the row entering at step j + s (only on its lane)
    // ---- forward, rows 0 .. m-1
#pragma unroll
    for (int c = 0; c < NR; ++c) x[c] = lane < m ? load(lane, c) : 0.0;
    auto fpref = [&](int j, int s) {
        const int o = (lane - j) & 31;
        rf[s] = (j < m && o >= 1 && o <= kl && j + o < m) ? F[(long long)j * rows + d + o] : 0.0;
        if (o == 0 && j + 32 < m)
#pragma unroll
            for (int c = 0; c < NR; ++c) rx[s][c] = load(j + 32, c);
    };
#pragma unroll
    for (int s = 0; s < kSkPf; ++s) fpref(s, s);
    for (int j0 = 0; j0 < m; j0 += kSkPf) {
#pragma unroll
        for (int s = 0; s < kSkPf; ++s) {
            const int j = j0 + s;
            if (j >= m) break;
            const int o = (lane - j) & 31;
            double xj[NR];
#pragma unroll
            for (int c = 0; c < NR; ++c) xj[c] = __shfl_sync(full, x[c], j & 31);
            if (o == 0) {
#pragma unroll
                for (int c = 0; c < NR; ++c) {
                    Xs[j * 8 + c] = xj[c];
                    x[c] = j + 32 < m ? rx[s][c] : 0.0;
                }
            } else if (o <= kl) {
#pragma unroll
                for (int c = 0; c < NR; ++c) x[c] = fma(-rf[s], xj[c], x[c]);
            }
            fpref(j + kSkPf, s);
        }
    }
    __syncwarp();
    // ---- backward, rows m-1 .. bwd_lo
    double rd[kSkPf];  // 1 / u_jj of step j
#pragma unroll
    for (int c = 0; c < NR; ++c) x[c] = m - 1 - lane >= 0 ? Xs[(m - 1 - lane) * 8 + c] : 0.0;
    auto bpref = [&](int j, int s) {  // step j = row j (descending)
        const int o = (lane - (m - 1 - j)) & 31;
        rf[s] = (j >= 0 && o >= 1 && o <= ku && j - o >= 0) ? F[(long long)j * rows + d - o] : 0.0;
        rd[s] = j >= 0 ? 1.0 / F[(long long)j * rows + d] : 0.0;
        if (o == 0 && j - 32 >= 0)
#pragma unroll
            for (int c = 0; c < NR; ++c) rx[s][c] = Xs[(j - 32) * 8 + c];
    };
#pragma unroll
    for (int s = 0; s < kSkPf; ++s) bpref(m - 1 - s, s);
    for (int j0 = 0; m - 1 - j0 >= bwd_lo; j0 += kSkPf) {
#pragma unroll
        for (int s = 0; s < kSkPf; ++s) {
            const int j = m - 1 - (j0 + s);
            if (j < bwd_lo) break;
            const int o = (lane - (m - 1 - j)) & 31;
            double xj[NR];
#pragma unroll
            for (int c = 0; c < NR; ++c) xj[c] = __shfl_sync(full, x[c], (m - 1 - j) & 31) * rd[s];
            if (o == 0) {
#pragma unroll
                for (int c = 0; c < NR; ++c) {
                    store(j, c, xj[c]);
                    x[c] = j - 32 >= 0 ? rx[s][c] : 0.0;
                }
            } else if (o <= ku) {
#pragma unroll
                for (int c = 0; c < NR; ++c) x[c] = fma(-rf[s], xj[c], x[c]);
            }
            bpref(j - kSkPf, s);
        }
    }
    __syncwarp();
}
}  // namespace

template <int NR>
__global__ void __launch_bounds__(32 * kSkSvWarps) k_sk_solve(SkSolveArgs A) {
    extern __shared__ __align__(16) double sv_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kSkSvWarps + warp, nwarps = gridDim.x * kSkSvWarps;
    const int k = A.k, p = A.p;
    const long long H = 2LL * p * k, kk = (long long)k * k;
    const int nr = A.nrhs;  // columns < nr exist (NR rounds nrhs up)
    double* Xs = sv_smem + (long long)warp * A.mmax * 8;

    // ---- D-stage: tips of Y = D^-1 F into T0
    for (int i = gw; i < p; i += nwarps) {
        const PartDev P = A.parts[i];
        const int m = P.m;
        const bool first = i == 0, last = i == p - 1;
        auto phys = [&](int r) -> long long { return P.rev ? (long long)(m - 1 - r) : (long long)r; };
        auto load = [&](int r, int c) -> double { return c < nr ? A.F[(long long)c * A.ldf + P.r0 + phys(r)] : 0.0; };
        double* T = A.T0;
        if (first) {
            for (int e = lane; e < k * nr; e += 32) T[(long long)(e / k) * H + (e % k)] = 0.0;  // dead top tip
            sk_fwd_bwd<NR>(P, A.fac, Xs, lane, m - k, load, [&](int j, int c, double v) {
                if (c < nr) T[(long long)c * H + k + (j - (m - k))] = v;
            });
        } else if (last) {
            for (int e = lane; e < k * nr; e += 32) T[(long long)(e / k) * H + (2LL * i + 1) * k + (e % k)] = 0.0;
            sk_fwd_bwd<NR>(P, A.fac, Xs, lane, m - k, load, [&](int j, int c, double v) {
                if (c < nr) T[(long long)c * H + 2LL * i * k + (m - 1 - j)] = v;
            });
        } else {
            sk_fwd_bwd<NR>(P, A.fac, Xs, lane, 0, load, [&](int j, int c, double v) {
                if (c >= nr) return;
                if (j < k) T[(long long)c * H + 2LL * i * k + j] = v;
                else if (j >= m - k) T[(long long)c * H + (2LL * i + 1) * k + (j - (m - k))] = v;
            });
        }
    }
    unsigned target = 0;
    grid_barrier(A.bar, target);

    // ---- reduced solve (solve.cpp:33-43): level by level, ping-pong T; one
    //      CTA per item (pair, kSkChunk rows of the merged unit)
    double* Tin = A.T0;
    double* Tout = A.T1;
    __shared__ double sWt[256], sVb[256], sSi[256], su[16 * 8], sz2[16 * 8], sz1[16 * 8];
    const int tid = threadIdx.x;
    for (int l = 0; l < A.nlevels; ++l) {
        const SkLevel L = A.levels[l];
        for (int it = blockIdx.x; it < L.nitems; it += gridDim.x) {
            const SkItem I = A.items[L.item0 + it];
            if (I.pair < 0) {
                const SkUnit u = A.units[-(I.pair + 1)];
                for (int r = I.row0 + tid; r < u.uh && r < I.row0 + kSkChunk; r += blockDim.x)
#pragma unroll
                    for (int c = 0; c < NR; ++c)
                        if (c < nr) Tout[(long long)c * H + u.uoff + r] = Tin[(long long)c * H + u.uoff + r];
                continue;
            }
            const SkPair pr = A.pairs[I.pair];
            const SkUnit uL = A.units[pr.left], uR = A.units[pr.left + 1];
            const int hL = uL.uh, hR = uR.uh, Hu = hL + hR;
            const long long zb = uL.uoff;
            const double* vl = A.pool + uL.voff;
            const double* wr = A.pool + uR.woff;
            for (int e = tid; e < k * k; e += blockDim.x) {
                const int c = e / k, r = e - c * k;
                sWt[r * 16 + c] = wr[(long long)c * hR + r];
                sVb[r * 16 + c] = vl[(long long)c * hL + hL - k + r];
                sSi[r * 16 + c] = A.pool[pr.sinv + e];
            }
            __syncthreads();
            // z2 = S^-1 (y2 - Wt y1), z1 = y1 - Vb z2: one element per thread
            const int er = tid % 16, ec = tid / 16;
            const bool el = er < k && ec < nr;
            if (el) {
                double v = Tin[(long long)ec * H + zb + hL + er];
                for (int t = 0; t < k; ++t) v = fma(-sWt[er * 16 + t], Tin[(long long)ec * H + zb + hL - k + t], v);
                su[er * 8 + ec] = v;
            }
            __syncthreads();
            if (el) {
                double v = 0.0;
                for (int t = 0; t < k; ++t) v = fma(sSi[er * 16 + t], su[t * 8 + ec], v);
                sz2[er * 8 + ec] = v;
            }
            __syncthreads();
            if (el) {
                double v = Tin[(long long)ec * H + zb + hL - k + er];
                for (int t = 0; t < k; ++t) v = fma(-sVb[er * 16 + t], sz2[t * 8 + ec], v);
                sz1[er * 8 + ec] = v;
            }
            __syncthreads();
            for (int r = I.row0 + tid; r < Hu && r < I.row0 + kSkChunk; r += blockDim.x) {
                if (r < hL - k || r >= hL + k) {
                    const bool left = r < hL - k;
                    const double* M = left ? vl : wr;
                    const int hm = left ? hL : hR, rr = left ? r : r - hL;
                    const double* z = left ? sz2 : sz1;
                    double v[NR];
#pragma unroll
                    for (int c = 0; c < NR; ++c) v[c] = c < nr ? Tin[(long long)c * H + zb + r] : 0.0;
                    for (int t = 0; t < k; ++t) {
                        const double mt = M[(long long)t * hm + rr];
#pragma unroll
                        for (int c = 0; c < NR; ++c) v[c] = fma(-mt, z[t * 8 + c], v[c]);
                    }
#pragma unroll
                    for (int c = 0; c < NR; ++c)
                        if (c < nr) Tout[(long long)c * H + zb + r] = v[c];
                } else {
                    const bool top = r < hL;
                    const int rr = top ? r - (hL - k) : r - hL;
#pragma unroll
                    for (int c = 0; c < NR; ++c)
                        if (c < nr) Tout[(long long)c * H + zb + r] = (top ? sz1 : sz2)[rr * 8 + c];
                }
            }
            __syncthreads();
        }
        grid_barrier(A.bar, target);
        double* tmp = Tin;
        Tin = Tout;
        Tout = tmp;
    }

    // ---- retrieval (solve.cpp:180-223): X_i = A_i^-1 (F_i - B_i xi - C_i eta)
    for (int i = gw; i < p; i += nwarps) {
        const PartDev P = A.parts[i];
        const int m = P.m;
        const bool first = i == 0, last = i == p - 1;
        const double* bh = A.pool + A.off_bhat + i * kk;
        const double* ch = A.pool + A.off_chat + i * kk;
        auto phys = [&](int r) -> int { return P.rev ? m - 1 - r : r; };
        auto load = [&](int r, int c) -> double {
            const int pr = phys(r);
            if (c >= nr) return 0.0;
            double v = A.F[(long long)c * A.ldf + P.r0 + pr];
            if (!last && pr >= m - k) {  // - bhat_i x_top(i+1)
                const int rr = pr - (m - k);
                for (int t = 0; t < k; ++t) v = fma(-bh[(long long)t * k + rr], Tin[(long long)c * H + 2LL * (i + 1) * k + t], v);
            }
            if (!first && pr < k) {  // - chat_i x_bot(i-1)
                for (int t = 0; t < k; ++t) v = fma(-ch[(long long)t * k + pr], Tin[(long long)c * H + (2LL * i - 1) * k + t], v);
            }
            return v;
        };
        sk_fwd_bwd<NR>(P, A.fac, Xs, lane, 0, load,
                       [&](int j, int c, double v) {
                           if (c < nr) A.X[(long long)c * A.ldx + P.r0 + phys(j)] = v;
                       });
    }
}

template <int NR>
static void launch_solve_t(const SkSolveArgs& A, cudaStream_t s) {
    const size_t smem = sizeof(double) * kSkSvWarps * (size_t)A.mmax * 8;
    set_smem_attr((const void*)k_sk_solve<NR>, (int)smem);
    const int grid = sk_coop_grid((const void*)k_sk_solve<NR>, 32 * kSkSvWarps, smem);
    SkSolveArgs a = A;
    void* args[] = {&a};
    (void)cudaLaunchCooperativeKernel((const void*)k_sk_solve<NR>, grid, 32 * kSkSvWarps, args, smem, s);
    count_launch();  // reports a failed launch
}

void launch_sk_solve(const SkSolveArgs& A, cudaStream_t s) {
    if (A.nrhs <= 1) launch_solve_t<1>(A, s);
    else if (A.nrhs <= 2) launch_solve_t<2>(A, s);
    else if (A.nrhs <= 4) launch_solve_t<4>(A, s);
    else launch_solve_t<8>(A, s);
}

}  // namespace spk
