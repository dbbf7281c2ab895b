// spk_smallk.cu — the small-k engine: non-pivoting SPIKE for narrow bands
// (kl, ku <= 31), HBM/latency-bound, in three launches per factorization and
// one per forward solve instead of the general engine's stage programs
// (~250 dependent launches at BASELINE C1).
//
//   k_sk_parts   one warp per partition: the partition's band columns (plus k
//                halo columns each side for the corners) land in shared
//                memory with ONE bulk async copy (cp.async.bulk, TMA 1-D,
//                mbarrier completion); register-window LU with diagonal
//                boosting (LUFactors::factor, src/kernels.cpp:79-118: lanes
//                hold the window rows, registers its columns, the pivot row
//                goes through shared memory); factors written back in the
//                general engine's layouts (packed LU, row-major copy, 1/u_jj);
//                corner blocks B^, C^ (spike2x2.cpp:17-26); spike tips
//                (factorize.cpp:133-257: V = A_i^-1 [0; B^], W = A_i^-1 [C^; 0],
//                truncated forward sweeps and bottom-tip backward sweeps for
//                the first / last partition, the last one through its reversed
//                LU = the reference's UL) by register-window sweeps, lanes =
//                spike columns.
//   k_sk_levels  cooperative persistent kernel: the whole reduced hierarchy
//                (reduce_factorize, factorize.cpp:46-120), one grid barrier
//                per level.  Work items are (pair, 32-row chunk of the merged
//                unit); every item re-derives its pair's S = I - W V, S^-1
//                (Gauss-Jordan, partial pivoting) and the pair-solve tips from
//                the level's read-only inputs, so a level needs no second
//                barrier.  Pairs with max|W| > 1 or a singular S need the
//                pivoted 2k coupling: the kernel raises a fallback flag and the
//                host re-runs the general engine's hierarchy program on the
//                (untouched) level-0 tips.
//   k_sk_solve   cooperative persistent kernel, forward solve with <= 8
//                right-hand sides (solve.cpp:81-223): D-stage per partition
//                (warp per partition, lanes = window rows), grid barrier, the
//                reduced solve level by level (ping-pong tip buffers, one
//                barrier per level), retrieval per partition.
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_smallk.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

namespace spk {

namespace {

constexpr int kSkWarpsMax = 4;

// shared memory per warp (doubles) of k_sk_parts
__host__ __device__ inline long long sk_parts_warp_smem(int mmax, int k, int ld) {
    const long long slab = (long long)(mmax + 2 * k) * ld + 4;  // + alignment slack
    const long long xs = (long long)mmax * 32;                   // forward spike rows, <= 32 columns
    return (slab + xs + 2 * 32 + 8 + 1) / 2 * 2;                 // + U-row buffers, mbarrier
}

}  // namespace

// ===========================================================================
// partitions: LU + factor layouts + corners + level-0 spike tips
//
// Windows of KS = 17 register slots (kl, ku <= 16): the LU holds columns
// j .. j+16 of each window row (column c in slot c mod KS), the spike sweeps
// rows j .. j+16 of each column (row r in slot (r - start) mod KS); the step
// loops are unrolled KS times so every slot index is a constant.  LU-space
// element (li, lj) of the staged band is base[off0 + lj * cj + li * ci]
// (the reversed last partition runs the other way), so addresses step by
// constants.
constexpr int kSkSlots = 17;

template <int CPL>
__global__ void __launch_bounds__(32 * kSkWarpsMax) k_sk_parts(SkPartsArgs A) {
    constexpr int KS = kSkSlots;
    extern __shared__ __align__(16) double sk_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int i = blockIdx.x * nw + warp;
    if (i >= A.p) return;
    const int ld = A.akl + A.aku + 1, k = A.k;
    const long long wsm = sk_parts_warp_smem(A.mmax, k, ld);
    double* const wbase = sk_smem + (long long)warp * wsm;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(wbase + wsm - 2);
    double* const ubuf = wbase + wsm - 2 - 64;  // [2][32]
    double* const Xs = ubuf - (long long)A.mmax * 32;
    const PartDev P = A.parts[i];
    const int m = P.m, rev = P.rev;
    const long long r0 = P.r0;
    const long long c0 = r0 - k > 0 ? r0 - k : 0;
    const long long c1 = r0 + m + k < A.n ? r0 + m + k : A.n;

    // ---- stage the band columns [c0, c1) (contiguous) with one bulk copy
    const long long e0 = c0 * ld, e1 = c1 * ld, etot = A.n * ld;
    const long long a0 = e0 & ~1LL;
    long long a1 = (e1 + 1) & ~1LL;
    if (a1 > etot) a1 -= 2;  // never read past the band
    double* const slab_raw = wbase;
    double* const slab = slab_raw + (e0 - a0);
    if (lane == 0) {
        mbar_init1(mbar);
        const unsigned bytes = (unsigned)((a1 - a0) * 8);
        mbar_expect_tx(mbar, bytes);
        bulk_g2s(slab_raw, A.band + a0, bytes, mbar);
    }
    __syncwarp();
    mbar_wait0(mbar);
    for (long long e = a1 + lane; e < e1; e += 32) slab_raw[e - a0] = A.band[e];  // tail element
    __syncwarp();

    double* const base = slab + (int)(r0 - c0) * ld + A.aku;
    const int kl = P.kl, ku = P.ku;  // LU space (swapped for rev)
    const int ci = rev ? -1 : 1, cj = rev ? -(ld - 1) : ld - 1, off0 = rev ? (m - 1) * ld : 0;
    auto sid = [&](int li, int lj) -> int { return off0 + lj * cj + li * ci; };
    auto inband = [&](int li, int lj) -> bool {
        return li >= 0 && lj >= 0 && li < m && lj < m && li - lj <= kl && lj - li <= ku;
    };

    // boost threshold over the partition block (kernels.cpp:80-85): column pj,
    // packed rows q on the lanes
    double amax = 0.0;
    for (int pj = 0; pj < m; ++pj)
        for (int q = lane; q < ld; q += 32) {
            const int pi = pj + q - A.aku;
            if (pi >= 0 && pi < m) amax = fmax(amax, fabs(base[pj * ld + q - A.aku]));
        }
    amax = warp_max(amax);
    const double scale = amax == 0.0 ? 1.0 : amax;
    const double zero_thresh = DBL_EPSILON * scale, boost_mag = A.boost_eps * scale;

    // ---- register-window LU: lane (row mod 32) holds its row's columns
    //      j .. j+KS-1 (column c in slot c mod KS)
    double W[KS];
#pragma unroll
    for (int c = 0; c < KS; ++c) W[c] = (lane <= kl && inband(lane, c)) ? base[sid(lane, c)] : 0.0;
    int boosts = 0;
    for (int j0 = 0; j0 < m; j0 += KS) {
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int j = j0 + t;
            if (j >= m) break;
            const int o = (lane - j) & 31;
            double* ub = ubuf + (j & 1) * 32;
            const int sjj = sid(j, j);
            if (o == 0) {
                double u = W[t];
                if (fabs(u) < zero_thresh) {
                    u = u == 0.0 ? boost_mag : copysign(boost_mag, u);
                    ++boosts;
                }
                W[t] = u;
                const double inv = 1.0 / u;
                ub[0] = inv;
#pragma unroll
                for (int c = 1; c < KS; ++c) ub[c] = W[(t + c) % KS];
                const int ce = min(ku, m - 1 - j);
                base[sjj] = u;
#pragma unroll
                for (int c = 1; c < KS; ++c)
                    if (c <= ce) base[sjj + c * cj] = W[(t + c) % KS];
                A.dinv[r0 + j] = inv;
            }
            __syncwarp();
            if (o >= 1 && o <= kl) {
                const double l = W[t] * ub[0];
                if (j + o < m) base[sjj + o * ci] = l;
#pragma unroll
                for (int c = 1; c < KS; ++c) W[(t + c) % KS] = fma(-l, ub[c], W[(t + c) % KS]);
                // entering column j + KS: in band iff KS - o <= ku
                const int cn = j + KS;
                W[t] = (KS - o <= ku && cn < m && j + o < m) ? base[sjj + o * ci + KS * cj] : 0.0;
            } else if (o == ((kl + 1) & 31)) {  // entering row j + kl + 1: columns j+1 .. j+KS
                const int r = j + kl + 1;
                const int sb = sid(r, j + 1);
#pragma unroll
                for (int c = 0; c < KS; ++c)
                    W[(t + 1 + c) % KS] = (c <= kl + ku && r < m && j + 1 + c < m) ? base[sb + c * cj] : 0.0;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) boosts += __shfl_xor_sync(0xffffffffu, boosts, o);
    if (lane == 0) A.boost[i] = boosts;
    __syncwarp();

    // ---- factor layouts: packed LU at fofs (column lj, packed rows on the
    //      lanes), row-major copy at tofs (row li)
    {
        double* F = A.fac + P.fofs;
        const int rows = P.rows, d = P.d;
        for (int lj = 0; lj < m; ++lj)
            for (int q = lane; q < rows; q += 32) {
                const int li = lj + q - d;
                F[(long long)lj * rows + q] = inband(li, lj) ? base[sid(li, lj)] : 0.0;
            }
        double* TF = A.tfac + P.tofs;
        const int rt = P.rowsT;
        for (int li = 0; li < m; ++li)
            for (int q = lane; q < rt; q += 32) {
                const int lj = li - kl + q;
                TF[(long long)li * rt + q] = inband(li, lj) ? base[sid(li, lj)] : 0.0;
            }
    }
    if (A.p < 2 || k == 0) return;

    // ---- corners (physical; k_corners, spike2x2.cpp:17-26)
    const bool first = i == 0, last = i == A.p - 1;
    const long long kk = (long long)k * k;
    auto bhat = [&](int rr, int c) -> double {  // A(r0+m-k+rr, r0+m+c)
        const int q = A.aku - k + rr - c;
        const long long pc = r0 + m + c;
        return (pc < c1 && q >= 0 && q < ld) ? slab[(pc - c0) * ld + q] : 0.0;
    };
    auto chat = [&](int rr, int c) -> double {  // A(r0+rr, r0-k+c)
        const int q = A.aku + rr + k - c;
        const long long pc = r0 - k + c;
        return (pc >= c0 && q >= 0 && q < ld) ? slab[(pc - c0) * ld + q] : 0.0;
    };
    for (int e = lane; e < k * k; e += 32) {
        const int c = e / k, rr = e - c * k;
        if (!last) A.pool[A.off_bhat + i * kk + e] = bhat(rr, c);
        if (!first) A.pool[A.off_chat + i * kk + e] = chat(rr, c);
    }

    // ---- spike tips.  Columns: inner partitions V (0..k-1) and W (k..2k-1);
    //      first: V; last (reversed): its W through the reversed LU in the V slot
    const int nc = (!first && !last) ? 2 * k : k;
    const int js = (!first && !last) ? 0 : m - k;  // forward start (trunc_start)
    const SkUnit U0 = A.units[i];
    auto rhs = [&](int r, int col) -> double {
        if (r >= m || col >= nc) return 0.0;
        if (col < k) {
            if (r < m - k) return 0.0;
            return last ? chat(m - 1 - r, col) : bhat(r - (m - k), col);
        }
        return r < k ? chat(r, col - k) : 0.0;
    };
    // forward L (unit lower), push form, rows js .. m-1; row j in slot (j-js) mod KS
    double X[CPL][KS];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int s = 0; s < KS; ++s) X[q][s] = rhs(js + s, lane + 32 * q);
    for (int j0 = js; j0 < m; j0 += KS) {
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int j = j0 + t;
            if (j >= m) break;
            // L column j (broadcast reads, issued together; rows past the band
            // or the partition contribute zero)
            const int sjj = sid(j, j);
            double lv[KS];
#pragma unroll
            for (int o = 1; o < KS; ++o) lv[o] = (o <= kl && j + o < m) ? base[sjj + o * ci] : 0.0;
#pragma unroll
            for (int q = 0; q < CPL; ++q) Xs[(long long)j * 32 * CPL + lane + 32 * q] = X[q][t];
#pragma unroll
            for (int o = 1; o < KS; ++o)
#pragma unroll
                for (int q = 0; q < CPL; ++q) X[q][(t + o) % KS] = fma(-lv[o], X[q][t], X[q][(t + o) % KS]);
#pragma unroll
            for (int q = 0; q < CPL; ++q) X[q][t] = rhs(j + KS, lane + 32 * q);
        }
    }
    __syncwarp();
    // backward U, rows m-1 down to je (inner: 0; first / last: the bottom tip)
    const int je = (!first && !last) ? 0 : m - k;
    auto emit = [&](int j, int col, double v) {
        if (col >= nc) return;
        if (last) {  // reversed W: LU row j in [m-k, m) is physical row m-1-j of wt
            A.pool[U0.woff + (long long)col * 2 * k + (m - 1 - j)] = v;
            return;
        }
        if (j >= k && j < m - k) return;
        const int rr = j >= m - k ? k + j - (m - k) : j;  // bottom tip rows k.., top rows 0..
        if (col < k) A.pool[U0.voff + (long long)col * 2 * k + rr] = v;
        else A.pool[U0.woff + (long long)(col - k) * 2 * k + rr] = v;
    };
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int r = m - 1 - s;
            X[q][s] = r >= js ? Xs[(long long)r * 32 * CPL + lane + 32 * q] : 0.0;
        }
    for (int j0 = 0; m - 1 - j0 >= je; j0 += KS) {
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int j = m - 1 - (j0 + t);
            if (j < je) break;
            const int sjj = sid(j, j);
            double uv[KS];
#pragma unroll
            for (int o = 1; o < KS; ++o) uv[o] = (o <= ku && j - o >= je) ? base[sjj - o * ci] : 0.0;
            const double dv = 1.0 / base[sjj];
            double xj[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                xj[q] = X[q][t] * dv;
                emit(j, lane + 32 * q, xj[q]);
            }
#pragma unroll
            for (int o = 1; o < KS; ++o)
#pragma unroll
                for (int q = 0; q < CPL; ++q) X[q][(t + o) % KS] = fma(-uv[o], xj[q], X[q][(t + o) % KS]);
            const int rn = j - KS;
#pragma unroll
            for (int q = 0; q < CPL; ++q) X[q][t] = rn >= js ? Xs[(long long)rn * 32 * CPL + lane + 32 * q] : 0.0;
        }
    }
}

template <int CPL>
static bool launch_parts_t(const SkPartsArgs& A, cudaStream_t s) {
    const int ld = A.akl + A.aku + 1;
    const size_t wsm = sizeof(double) * sk_parts_warp_smem(A.mmax, A.k, ld);
    int nw = (int)std::min<size_t>(kSkWarpsMax, (227u * 1024) / wsm);
    if (nw < 1) return false;
    const size_t smem = wsm * nw;
    set_smem_attr((const void*)k_sk_parts<CPL>, (int)smem);
    k_sk_parts<CPL><<<(A.p + nw - 1) / nw, 32 * nw, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_sk_parts(const SkPartsArgs& A, cudaStream_t s) {
    if (A.akl > 16 || A.aku > 16 || (reinterpret_cast<uintptr_t>(A.band) & 15)) return false;
    return launch_parts_t<1>(A, s);
}

// ===========================================================================
// reduced hierarchy: per level, items (pair, chunk of kSkLvRows rows of the
// merged unit), one CTA per item
//
// Pair (left unit hL rows: V = vl, W = wl; right unit hR rows: V = vr, W = wr),
// coupling [[I, Vb], [Wt, I]] with Vb = vl[hL-k : hL], Wt = wr[0 : k]; Schur
// complement S = I - Wt Vb.  The merged unit's spikes are the pair solves
// (factorize.cpp:19-32) of [0; vr] and [wl; 0]:
//   z2 = S^-1 (y2 - Wt y1), z1 = y1 - Vb z2,
//   rows [0, hL-k) -= vl[0:hL-k] z2, rows [hL+k, H) -= wr[k:hR] z1.
// The k x k work (S, S^-1 by Gauss-Jordan with partial pivoting, the z
// blocks) runs one element per thread; the rows one row per thread.
namespace {
constexpr int kSkLvThreads = 256;
constexpr int kSkLvRows = 256;  // rows per work item (one per thread)
}  // namespace

__global__ void __launch_bounds__(kSkLvThreads) k_sk_levels(SkLevelsArgs A) {
    // k <= 16: k x k blocks row-major with ld 16
    __shared__ double Wt[256], Vb[256], Si[256], y2v[256], y1w[256], uw[256], z2v[256], z1v[256], z2w[256],
        z1w[256], colj[16];
    __shared__ double aug[16][33], rowp[32];
    __shared__ int s_pr, s_bad, s_perm[16];
    const int tid = threadIdx.x;
    const int k = A.k;
    const int er = tid & 15, ec = tid >> 4;  // element (row, column) of a k x k block
    const bool el = er < k && ec < k;
    unsigned target = 0;
    for (int l = 0; l < A.nlevels; ++l) {
        const SkLevel L = A.levels[l];
        for (int it = blockIdx.x; it < L.nitems; it += gridDim.x) {
            const SkItem I = A.items[L.item0 + it];
            if (I.pair < 0) {  // carried odd unit: spikes move up unchanged
                const SkUnit u = A.units[-(I.pair + 1)], nu = A.units[I.next];
                const int r = I.row0 + tid;
                if (r < u.uh)
                    for (int c = 0; c < k; ++c) {
                        if (u.voff >= 0) A.pool[nu.voff + (long long)c * nu.uh + r] = A.pool[u.voff + (long long)c * u.uh + r];
                        if (u.woff >= 0) A.pool[nu.woff + (long long)c * nu.uh + r] = A.pool[u.woff + (long long)c * u.uh + r];
                    }
                continue;
            }
            const SkPair pr = A.pairs[I.pair];
            const SkUnit uL = A.units[pr.left], uR = A.units[pr.left + 1], nu = A.units[pr.next];
            const int hL = uL.uh, hR = uR.uh, H = hL + hR;
            const bool hv = nu.voff >= 0, hw = nu.woff >= 0;
            const double* vl = A.pool + uL.voff;
            const double* wl = hw ? A.pool + uL.woff : nullptr;
            const double* vr = hv ? A.pool + uR.voff : nullptr;
            const double* wr = A.pool + uR.woff;
            if (tid == 0) s_bad = 0;
            __syncthreads();
            if (el) {
                const double w = wr[(long long)ec * hR + er];
                if (fabs(w) > 1.0) s_bad = 1;
                Wt[er * 16 + ec] = w;
                Vb[er * 16 + ec] = vl[(long long)ec * hL + hL - k + er];
                y2v[er * 16 + ec] = hv ? vr[(long long)ec * hR + er] : 0.0;
                y1w[er * 16 + ec] = hw ? wl[(long long)ec * hL + hL - k + er] : 0.0;
            }
            __syncthreads();
            if (s_bad) {  // |W| > 1: the pivoted 2k coupling (general programs)
                if (tid == 0) {
                    A.flags[pr.gidx] = 0;
                    atomicExch(A.fallback, 1);
                }
                __syncthreads();
                continue;
            }
            // S = I - Wt Vb into aug[:, 0:k], I into aug[:, k:2k]; uw = -Wt y1w
            if (el) {
                double sv = er == ec ? 1.0 : 0.0, u = 0.0;
                for (int t = 0; t < k; ++t) {
                    sv = fma(-Wt[er * 16 + t], Vb[t * 16 + ec], sv);
                    u = fma(-Wt[er * 16 + t], y1w[t * 16 + ec], u);
                }
                aug[er][ec] = sv;
                aug[er][k + ec] = er == ec ? 1.0 : 0.0;
                uw[er * 16 + ec] = u;
            }
            __syncthreads();
            // Gauss-Jordan, partial pivoting: first maximum among unused rows
            unsigned used = 0u;
            int perm = 0;  // thread j: pivot row of step j
            bool sing = false;
            for (int j = 0; j < k; ++j) {
                if (tid < 32) {
                    double best = (tid < k && !((used >> tid) & 1u)) ? fabs(aug[tid][j]) : -1.0;
                    int idx = tid;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
                        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
                        if (ov > best || (ov == best && oi < idx)) {
                            best = ov;
                            idx = oi;
                        }
                    }
                    if (tid == 0) s_pr = best > 0.0 ? idx : -1;
                }
                __syncthreads();
                const int prw = s_pr;
                if (prw < 0) {
                    sing = true;
                    break;
                }
                used |= 1u << prw;
                if (tid == j) perm = prw;
                if (tid < k) colj[tid] = aug[tid][j];
                if (tid < 2 * k) rowp[tid] = aug[prw][tid] / aug[prw][j];
                __syncthreads();
                for (int e = tid; e < k * 2 * k; e += kSkLvThreads) {
                    const int r = e / (2 * k), c = e - r * 2 * k;
                    const double pc = rowp[c];
                    aug[r][c] = r == prw ? pc : fma(-colj[r], pc, aug[r][c]);
                }
                __syncthreads();
            }
            if (sing) {
                if (tid == 0) {
                    A.flags[pr.gidx] = 0;
                    atomicExch(A.fallback, 1);
                }
                __syncthreads();
                continue;
            }
            // S^-1 row j = aug[perm(j)][k:2k]
            if (tid < k) s_perm[tid] = perm;
            __syncthreads();
            if (el) Si[er * 16 + ec] = aug[s_perm[er]][k + ec];
            __syncthreads();
            if (I.row0 == 0) {
                if (el) A.pool[pr.sinv + (long long)ec * k + er] = Si[er * 16 + ec];
                if (tid == 0) A.flags[pr.gidx] = 1;
            }
            // z2 = S^-1 [vr top | uw]; z1 = [0 | y1w] - Vb z2
            if (el) {
                double a = 0.0, b = 0.0;
                for (int t = 0; t < k; ++t) {
                    a = fma(Si[er * 16 + t], y2v[t * 16 + ec], a);
                    b = fma(Si[er * 16 + t], uw[t * 16 + ec], b);
                }
                z2v[er * 16 + ec] = a;
                z2w[er * 16 + ec] = b;
            }
            __syncthreads();
            if (el) {
                double a = 0.0, b = y1w[er * 16 + ec];
                for (int t = 0; t < k; ++t) {
                    a = fma(-Vb[er * 16 + t], z2v[t * 16 + ec], a);
                    b = fma(-Vb[er * 16 + t], z2w[t * 16 + ec], b);
                }
                z1v[er * 16 + ec] = a;
                z1w[er * 16 + ec] = b;
            }
            __syncthreads();
            // rows of the merged unit: one per thread
            const int r = I.row0 + tid;
            if (r < H && r < I.row0 + kSkLvRows) {
                double* nv = hv ? A.pool + nu.voff : nullptr;
                double* nwp = hw ? A.pool + nu.woff : nullptr;
                if (r < hL - k || r >= hL + k) {
                    const bool left = r < hL - k;
                    const int rr = left ? r : r - hL;
                    const double* M = left ? vl : wr;
                    const int hm = left ? hL : hR;
                    const double* zv = left ? z2v : z1v;
                    const double* zw = left ? z2w : z1w;
                    double mrow[16];
#pragma unroll
                    for (int t = 0; t < 16; ++t) mrow[t] = t < k ? M[(long long)t * hm + rr] : 0.0;
                    for (int c = 0; c < k; ++c) {
                        double a = left ? 0.0 : (hv ? vr[(long long)c * hR + rr] : 0.0);
                        double b = left ? (hw ? wl[(long long)c * hL + rr] : 0.0) : 0.0;
#pragma unroll
                        for (int t = 0; t < 16; ++t)
                            if (t < k) {
                                a = fma(-mrow[t], zv[t * 16 + c], a);
                                b = fma(-mrow[t], zw[t * 16 + c], b);
                            }
                        if (hv) nv[(long long)c * H + r] = a;
                        if (hw) nwp[(long long)c * H + r] = b;
                    }
                } else {
                    const bool top = r < hL;  // z1 rows [hL-k, hL), z2 rows [hL, hL+k)
                    const int rr = top ? r - (hL - k) : r - hL;
                    for (int c = 0; c < k; ++c) {
                        if (hv) nv[(long long)c * H + r] = (top ? z1v : z2v)[rr * 16 + c];
                        if (hw) nwp[(long long)c * H + r] = (top ? z1w : z2w)[rr * 16 + c];
                    }
                }
            }
            __syncthreads();
        }
        if (l + 1 < A.nlevels) grid_barrier(A.bar, target);
    }
}

void launch_sk_levels(const SkLevelsArgs& A, cudaStream_t s) {
    if (A.nlevels <= 0) return;
    const int grid = sk_coop_grid((const void*)k_sk_levels, kSkLvThreads, 0);
    SkLevelsArgs a = A;
    void* args[] = {&a};
    (void)cudaLaunchCooperativeKernel((const void*)k_sk_levels, grid, kSkLvThreads, args, 0, s);
    count_launch();  // reports a failed launch
}

}  // namespace spk
