// spk_lu_fast.cu — register-window band LU (non-pivoting, diagonal boosting)
// for SPIKE partitions, one CTA per partition.
//
// Reference: LUFactors::factor, src/kernels.cpp:79-118 (+ the packed copy of
// :29-65, done here on the fly from the input band, reversed for the UL
// partition).  Same arithmetic: multipliers l = a * (1/u_jj), rank-1 update
// of the kl x ku trailing window per column step, boost |u_jj| < eps*max|A_i|
// to +-boost_eps*max|A_i|.
//
// Layout: the K x K active window (K = 32*TR >= max(kl, ku)) lives in
// registers.  Lane l / register a hold row slot 32a+l (row i <-> slot i mod K);
// warp w / register b hold column slot w + NW*b (column c <-> slot c mod K).
// Step j:
//   1. every warp reads l_j (published in shared memory by the owner of column
//      j during step j-1) and shuffles the pivot row u_j out of lane j mod 32;
//   2. the pivot row/column slots are recycled for row/column j+K (gathered
//      from HBM one 32-step round ahead by cp.async);
//   3. rank-1 update of the whole window (DFMA), the owner of column j+1
//      first, which then scales that column and publishes l_{j+1};
//   4. one __syncthreads.
// Factors are written in both layouts the sweeps use (column-major packed LU
// and the row-major copy) plus 1/u_jj.  Boosting is decided optimistically:
// the CTA tracks max|A_i| and min|u_jj| on the fly and, if a boost would have
// fired, re-runs its partition with the now-known threshold (exact reference
// semantics; never taken for diagonally dominant input).
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_sweep_fast.cuh"

#include <cfloat>

namespace spk {

struct FastLuArgs {
    const int* units;
    const PartDev* parts;
    const double* band;  // input band (kl+ku+1) x n, column-major
    int akl, aku;
    double* fac;
    double* tfac;
    double* dinv;
    int* piv;
    double boost_eps;
    int* boost_cnt;
};

template <int TR, int NW>
struct LuGeom {
    static constexpr int K = 32 * TR;
    static constexpr int CPW = K / NW;
    static_assert(32 % NW == 0 && CPW * NW == K, "geometry");
};

inline size_t fast_lu_smem(int K) {
    // 2 stages x (new rows + new columns) + u/extra + l double buffer + U-row buffer
    return (size_t)(2 * 2 * 32 * K + 2 * 2 * 32 + 2 * K + 32 * (K + 1)) * 8 + 64;
}

template <int TR, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_band_lu_fast(FastLuArgs A) {
    constexpr int K = LuGeom<TR, NW>::K;
    constexpr int CPW = LuGeom<TR, NW>::CPW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_nr = reinterpret_cast<double*>(smem_raw);  // [2][32][K] new rows (column-slot order)
    double* s_nc = s_nr + 2 * 32 * K;                    // [2][32][K] new columns (row-slot order)
    double* s_ncu = s_nc + 2 * 32 * K;                   // [2][32]    A(j, j+K)
    double* s_ex = s_ncu + 2 * 32;                       // [2][32]    A(j+1+K, j+1)
    double* s_l = s_ex + 2 * 32;                         // [2][K]     published multipliers
    double* s_ur = s_l + 2 * K;                          // [32][K]    U rows of the round (slot order)
    __shared__ double s_red[2 * 32];

    const int u = A.units[blockIdx.x];
    const PartDev P = A.parts[u];
    const int m = P.m, kl = P.kl, ku = P.ku, rows = P.rows, d = P.d, rowsT = P.rowsT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ald = A.akl + A.aku + 1;
    double* F = A.fac + P.fofs;
    double* TF = A.tfac + P.tofs;

    // address of LU-space entry (i, c) in the input band, or nullptr (zero)
    auto aptr = [&](int i, int c) -> const double* {
        if (i < 0 || c < 0 || i >= m || c >= m) return nullptr;
        if (i - c > kl || c - i > ku) return nullptr;
        if (!P.rev) return A.band + (long long)(P.r0 + c) * ald + A.aku + i - c;
        return A.band + (long long)(P.r0 + m - 1 - c) * ald + A.aku + c - i;
    };
    auto aval = [&](int i, int c) -> double {
        const double* q = aptr(i, c);
        return q ? *q : 0.0;
    };

    // stage round R (steps j = 32R + t): new row j+K for the column slots,
    // new column j+K for the row slots, u entry A(j, j+K), extra A(j+1+K, j+1)
    auto load_round = [&](int R) {
        const int st = R & 1;
        const int j0 = 32 * R;
        if (j0 < m) {
            double* nr = s_nr + st * 32 * K;
            double* nc = s_nc + st * 32 * K;
            for (int idx = threadIdx.x; idx < 32 * K; idx += blockDim.x) {
                const int t = idx & 31, s = idx >> 5;  // t fastest: consecutive rows of one column
                const int j = j0 + t;
                int off = s - (j + 1) % K;
                if (off < 0) off += K;
                const int c = j + 1 + off;
                const double* q = aptr(j + K, c);
                if (q) cp_async8(nr + t * K + s, q);
                else nr[t * K + s] = 0.0;
            }
            for (int idx = threadIdx.x; idx < 32 * K; idx += blockDim.x) {
                const int t = idx / K, s = idx - t * K;  // s fastest: consecutive rows of column j+K
                const int j = j0 + t;
                int off = s - (j + 1) % K;
                if (off < 0) off += K;
                const int i = j + 1 + off;
                const double* q = aptr(i, j + K);
                if (q) cp_async8(nc + t * K + s, q);
                else nc[t * K + s] = 0.0;
            }
            if (threadIdx.x < 64) {
                const int t = threadIdx.x & 31;
                const int j = j0 + t;
                double* dst = threadIdx.x < 32 ? s_ncu + st * 32 + t : s_ex + st * 32 + t;
                const double* q = threadIdx.x < 32 ? aptr(j, j + K) : aptr(j + 1 + K, j + 1);
                if (q) cp_async8(dst, q);
                else *dst = 0.0;
            }
        }
        cp_async_commit();
    };

    double amax = 0.0;
    double minpiv = 1.0 / 0.0;
    int nboost = 0;
    bool boost_mode = false;
    double thresh = 0.0, bmag = 0.0;

    // positions of the packed layouts that no step writes (above row 0 / left
    // of column 0) must read as zero for the sweeps
    for (int idx = threadIdx.x; idx < ku * ku; idx += blockDim.x) {
        const int c = idx / ku, off = idx - c * ku + 1;  // column c, row c - off < 0
        if (c < m && off > c) F[(long long)c * rows + d - off] = 0.0;
    }
    for (int idx = threadIdx.x; idx < kl * kl; idx += blockDim.x) {
        const int r = idx / kl, off = idx - r * kl + 1;  // row r, column r - off < 0
        if (r < m && off > r) TF[(long long)r * rowsT + kl - off] = 0.0;
    }

    for (int attempt = 0; attempt < 2; ++attempt) {
        // ---- initial window: rows 0..K-1, columns 0..K-1
        double W[TR][CPW];
#pragma unroll
        for (int a = 0; a < TR; ++a)
#pragma unroll
            for (int b = 0; b < CPW; ++b) {
                W[a][b] = aval(32 * a + lane, warp + NW * b);
                amax = fmax(amax, fabs(W[a][b]));
            }
        load_round(0);
        // ---- publish l_0 (owner of column 0 = warp 0, register 0)
        if (warp == 0) {
            double pv = __shfl_sync(0xffffffffu, W[0][0], 0);
            minpiv = fmin(minpiv, fabs(pv));
            if (boost_mode && fabs(pv) < thresh) {
                pv = pv == 0.0 ? bmag : copysign(bmag, pv);
                ++nboost;
                if (lane == 0) W[0][0] = pv;
            }
            const double inv = 1.0 / pv;
            const double ex = aval(K, 0);
            amax = fmax(amax, fabs(ex));
#pragma unroll
            for (int a2 = 0; a2 < TR; ++a2) {
                const int r = 32 * a2 + lane;  // row in slot r (rows 0..K-1)
                double lv = (r == 0) ? ex * inv : W[a2][0] * inv;
                s_l[r] = lv;
                const int rr = r == 0 ? K : r;  // row this multiplier belongs to
                if (rr >= 1 && rr <= kl) {
                    F[(long long)0 * rows + d + rr] = rr < m ? lv : 0.0;
                    if (rr < m) TF[(long long)rr * rowsT + kl - rr] = lv;
                }
            }
            if (lane == 0) A.dinv[P.r0] = inv;
        }

        const int nrounds = (m + 31) / 32;
        for (int R0 = 0; R0 < nrounds; R0 += TR) {
#pragma unroll
            for (int a = 0; a < TR; ++a) {
                const int R = R0 + a;
                if (R < nrounds) {
                    cp_async_wait<0>();
                    __syncthreads();
                    load_round(R + 1);
                    const int st = R & 1;
                    const double* nr = s_nr + st * 32 * K;
                    const double* nc = s_nc + st * 32 * K;
                    // max|A_i| over everything this round brings into the window
                    for (int idx = threadIdx.x; idx < 2 * 32 * K; idx += blockDim.x)
                        amax = fmax(amax, fabs((idx < 32 * K ? nr : nc - 32 * K)[idx]));
                    if (threadIdx.x < 64)
                        amax = fmax(amax, fabs((threadIdx.x < 32 ? s_ncu : s_ex)[st * 32 + (threadIdx.x & 31)]));
#pragma unroll
                    for (int q = 0; q < 32 / NW; ++q) {
                        const int bq = (32 * a) / NW + q;  // register column of pivot column j
                        for (int w2 = 0; w2 < NW; ++w2) {
                            const int t = q * NW + w2;
                            const int j = 32 * R + t;
                            if (j >= m) break;
                            double lv[TR];
#pragma unroll
                            for (int a2 = 0; a2 < TR; ++a2) lv[a2] = s_l[(j & 1) * K + 32 * a2 + lane];
                            const bool own = warp == w2;
                            const bool last = w2 == NW - 1;
                            const bool pub = warp == (w2 + 1) % NW && j + 1 < m;
                            const bool mine = lane == t;
                            const double* nrow = nr + t * K + warp;
                            double* urow = s_ur + t * K + warp;  // U row j, column-slot order
#pragma unroll
                            for (int bi = 0; bi < CPW; ++bi) {
                                const int b = (bq + bi) % CPW;
                                double ub = __shfl_sync(0xffffffffu, W[a][b], t);
                                urow[NW * b] = ub;
                                const double nv = nrow[NW * b];
                                W[a][b] = mine ? nv : W[a][b];
                                if (bi == 0 && own) {
                                    // the pivot column's slot becomes column j+K
#pragma unroll
                                    for (int a2 = 0; a2 < TR; ++a2) W[a2][b] = nc[t * K + 32 * a2 + lane];
                                    ub = s_ncu[st * 32 + t];
                                }
#pragma unroll
                                for (int a2 = 0; a2 < TR; ++a2) W[a2][b] = fma(-lv[a2], ub, W[a2][b]);
                                if (pub && ((bi == 0 && !last) || (bi == 1 && last) || (CPW == 1 && last))) {
                                    // owner of column j+1: pivot, scale, publish l_{j+1}
                                    const int tn = (t + 1) & 31;
                                    const bool wrap = t == 31;
                                    const double wsel = wrap ? W[(a + 1) % TR][b] : W[a][b];
                                    double pv = __shfl_sync(0xffffffffu, wsel, tn);
                                    minpiv = fmin(minpiv, fabs(pv));
                                    if (boost_mode && fabs(pv) < thresh) {
                                        pv = pv == 0.0 ? bmag : copysign(bmag, pv);
                                        ++nboost;
                                        if (lane == tn) {
                                            if (wrap) W[(a + 1) % TR][b] = pv;
                                            else W[a][b] = pv;
                                        }
                                    }
                                    const double inv = 1.0 / pv;
                                    const double ex = s_ex[st * 32 + t];
                                    const int jn = j + 1;
                                    const int sn = (32 * a + t + 1) % K;  // pivot slot of step j+1
#pragma unroll
                                    for (int a2 = 0; a2 < TR; ++a2) {
                                        const int sl = 32 * a2 + lane;
                                        const double lval = (sl == sn) ? ex * inv : W[a2][b] * inv;
                                        s_l[(jn & 1) * K + sl] = lval;
                                        int off = sl - sn;  // row jn + off
                                        if (off <= 0) off += K;
                                        const int r = jn + off;
                                        if (off <= kl) {
                                            F[(long long)jn * rows + d + off] = r < m ? lval : 0.0;
                                            if (r < m) TF[(long long)r * rowsT + kl - off] = lval;
                                        }
                                    }
                                    if (lane == 0) A.dinv[P.r0 + jn] = inv;
                                }
                            }
                            __syncthreads();
                        }
                    }
                    // write back the round's U rows (both layouts): slot s of row j
                    // holds column j + ((s - j) mod K); column j+K comes from s_ncu
                    const int nst = min(32, m - 32 * R);
                    for (int idx = threadIdx.x; idx < nst * (K + 1); idx += blockDim.x) {
                        const int t = idx / (K + 1), sl = idx - t * (K + 1);
                        const int j = 32 * R + t;
                        int off = K;
                        double val = s_ncu[st * 32 + t];
                        if (sl < K) {
                            off = sl - (32 * a + t) % K;
                            if (off < 0) off += K;
                            val = s_ur[t * K + sl];
                        }
                        if (off > ku) continue;
                        TF[(long long)j * rowsT + kl + off] = (j + off < m) ? val : 0.0;
                        if (j + off < m) F[(long long)(j + off) * rows + d - off] = val;
                    }
                }
            }
        }
        cp_async_wait<0>();
        // ---- optimistic boosting check (non-pivoting): reduce max|A_i| and min|u_jj|
        double am = amax, mp = minpiv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
            mp = fmin(mp, __shfl_xor_sync(0xffffffffu, mp, o));
        }
        __syncthreads();
        if (lane == 0) {
            s_red[warp] = am;
            s_red[32 + warp] = mp;
        }
        __syncthreads();
        am = 0.0;
        mp = 1.0 / 0.0;
        for (int w = 0; w < NW; ++w) {
            am = fmax(am, s_red[w]);
            mp = fmin(mp, s_red[32 + w]);
        }
        const double scale = am == 0.0 ? 1.0 : am;
        if (boost_mode || !(mp < DBL_EPSILON * scale)) break;
        boost_mode = true;
        thresh = DBL_EPSILON * scale;
        bmag = A.boost_eps * scale;
        nboost = 0;
        __syncthreads();
    }
    // column m-1 has no multipliers (no step publishes it)
    for (int off = threadIdx.x + 1; off <= kl; off += blockDim.x) F[(long long)(m - 1) * rows + d + off] = 0.0;
    // reduce the boost count
    int nb = nboost;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if (lane == 0 && nb) atomicAdd(&A.boost_cnt[u], nb);
    // pivots are the identity in this mode
    for (int j = threadIdx.x; j < m; j += blockDim.x) A.piv[P.r0 + j] = j;
}

bool launch_band_lu_fast(const int* d_units, int nunits, int kmax, const FastLuArgs& A, cudaStream_t s) {
    void (*fn)(FastLuArgs) = nullptr;
    int nw = 0, K = 0;
    if (kmax <= 32) {
        fn = k_band_lu_fast<1, 4>;
        nw = 4;
        K = 32;
    } else if (kmax <= 64) {
        fn = k_band_lu_fast<2, 8>;
        nw = 8;
        K = 64;
    } else if (kmax <= 96) {
        fn = k_band_lu_fast<3, 8>;
        nw = 8;
        K = 96;
    } else if (kmax <= 128) {
        fn = k_band_lu_fast<4, 16>;
        nw = 16;
        K = 128;
    } else if (kmax <= 160) {
        fn = k_band_lu_fast<5, 16>;
        nw = 16;
        K = 160;
    } else {
        return false;
    }
    const size_t smem = fast_lu_smem(K);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<nunits, 32 * nw, smem, s>>>(A);
    count_launch();
    return true;
}

}  // namespace spk
