// spk_sweep_piv_dmma.cu — pivoted forward L sweep (B := L^-1 P B) on the FP64
// tensor cores, 8 rows per step, from the blocked L records the pivoted LU
// writes (spk_piv_blocked.cuh).
//
// Reference: forward_lower / forward_lower_tail, src/kernels.cpp:131-165
// (pivoting: for each row j, interchange B(j) and B(ip), then
// B(j+1 .. j+kl) -= l_j B(j)).  Per 8-row panel J the reference's 8 steps are
// one record: the panel's row permutation of the window rows 8J .. 8J+8TRW-1,
// X = L11^-1 (rows 8J .. 8J+7), then the window below takes -L21 X.  Layout
// follows k_sweep_dmma (spk_sweep_dmma.cuh): each warp owns 8 right-hand-side
// columns and holds the window as TRW DMMA accumulator tiles (lane l: row l>>2,
// columns 2(l&3), 2(l&3)+1), registers rotate one tile per panel.  The
// permutation goes through a per-warp shared-memory scratch (only tile 0 and
// the rows that move); records and entering rows are staged by cp.async one
// 4-panel round ahead, one CTA barrier per round.
//
// A job starting at row lo starts at panel lo/8: rows [8 (lo/8), lo) of its
// right-hand side are zero in every program that emits a pivoted forward
// sweep with lo > 0 (the V spike on the zeroed FS buffer, the edge retrieval
// on the zeroed S buffer), and the reference's steps there are no-ops on zero
// rows (their pivots stay below m - kcorner).  Rows below lo are not written.
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_piv_blocked.cuh"
#include "spk_sweep_fast.cuh"

namespace spk {

__device__ __forceinline__ void ps_dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

constexpr int kPsRound = 4;  // panels per staging round

template <int TRW>
inline size_t piv_sweep_smem(int nwarps) {
    const int ncta = nwarps * 8;
    return sizeof(double) * ((size_t)2 * kPsRound * PivRec<TRW>::SIZE + (size_t)2 * 8 * kPsRound * (ncta + 1) +
                             (size_t)nwarps * 8 * TRW * 8);
}

template <int TRW>
__global__ void __launch_bounds__(512) k_sweep_piv_dmma(PivSweepArgs A) {
    using R = PivRec<TRW>;
    constexpr int RND = kPsRound;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const SweepJob J = A.jobs[blockIdx.x];
    if (!guard_ok(A.B.flags, J.guard)) return;
    const PartDev P = A.parts[J.part];
    const int nc_total = J.nc >= 0 ? J.nc : A.ncols;
    const int nwarps = blockDim.x >> 5, ncta = nwarps * 8, sin_ld = ncta + 1;
    const int colbase = blockIdx.y * ncta;
    if (colbase >= nc_total) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const unsigned full = 0xffffffffu;
    const int m = P.m, lo = J.lo;
    const int J0 = lo / 8, nblk = (m + 7) / 8;
    if (J0 >= nblk) return;
    const int npan = nblk - J0;

    double* s_rec = reinterpret_cast<double*>(smem_raw);         // [2][RND][R::SIZE]
    double* s_in = s_rec + 2 * RND * R::SIZE;                     // [2][8 RND][ncta+1]
    double* xs = s_in + 2 * 8 * RND * sin_ld + warp * 8 * TRW * 8;  // per-warp [8TRW][8]

    const View& v = J.v;
    const long long ld = v.ld >= 0 ? v.ld : A.B.ld[v.buf];
    double* const bbase = A.B.p[v.buf] + v.base;
    auto phys = [&](int r) -> long long {
        return v.rev ? (long long)(v.mrows - 1 - (r - v.off)) : (long long)(r - v.off);
    };
    const int c0 = J.c0 + colbase;
    const int ncta_valid = min(ncta, nc_total - colbase);
    const int lc0 = warp * 8 + 2 * q;
    const bool cv0 = lc0 < ncta_valid, cv1 = lc0 + 1 < ncta_valid;
    double* const cp0 = bbase + (long long)(c0 + (cv0 ? lc0 : 0)) * ld;
    double* const cp1 = bbase + (long long)(c0 + (cv1 ? lc0 + 1 : 0)) * ld;
    const double* recbase = A.lblk + (P.r0 / 8 + J.part) * (long long)R::SIZE;

    // round Rr: records of panels J0 + RND Rr + b and the rows entering at
    // their shifts (8 (Jp + TRW) + t)
    auto load_round = [&](int Rr) {
        const int st = Rr & 1, k0 = RND * Rr;
        if (k0 < npan) {
            const int nb = min(RND, npan - k0);
            double* dr = s_rec + (size_t)st * RND * R::SIZE;
            const double* src = recbase + (long long)(J0 + k0) * R::SIZE;
            for (int idx = threadIdx.x; idx < nb * R::SIZE / 2; idx += blockDim.x)
                cp_async16(dr + 2 * idx, src + 2 * idx);
            double* di = s_in + (size_t)st * 8 * RND * sin_ld;
            for (int idx = threadIdx.x; idx < 8 * RND * ncta; idx += blockDim.x) {
                const int t = idx & 31, col = idx >> 5;  // t = 8 b + row
                const int row = 8 * (J0 + k0 + (t >> 3) + TRW) + (t & 7);
                double* dst = di + t * sin_ld + col;
                if (row < m && col < ncta_valid) cp_async8(dst, bbase + phys(row) + (long long)(c0 + col) * ld);
                else *dst = 0.0;
            }
        }
        cp_async_commit();
    };

    double Wt[TRW][2];
#pragma unroll
    for (int t = 0; t < TRW; ++t) {
        const int row = 8 * (J0 + t) + g;
        const bool ok = row < m;
        const long long pr = ok ? phys(row) : 0;
        Wt[t][0] = (ok && cv0) ? cp0[pr] : 0.0;
        Wt[t][1] = (ok && cv1) ? cp1[pr] : 0.0;
    }
    load_round(0);

    for (int k = 0; k < npan; ++k) {
        const int st = (k / RND) & 1, bb = k % RND, Jp = J0 + k;
        if (bb == 0) {
            cp_async_wait<0>();
            __syncthreads();
            load_round(k / RND + 1);
        }
        const double* rec = s_rec + (size_t)(st * RND + bb) * R::SIZE;
        const int* ri = reinterpret_cast<const int*>(rec + R::SRC);
        // 1. the panel's row permutation (rows move only between tile 0 and the
        //    pivot rows)
#pragma unroll
        for (int t = 0; t < TRW; ++t) {
            const unsigned mo = (unsigned)ri[8 * TRW + ((8 * t) >> 5)];
            if (t == 0 || ((mo >> (((8 * t) & 31) + g)) & 1u))
                *reinterpret_cast<double2*>(&xs[(8 * t + g) * 8 + 2 * q]) = make_double2(Wt[t][0], Wt[t][1]);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < TRW; ++t) {
            const unsigned mi = (unsigned)ri[8 * TRW + R::NSLW + ((8 * t) >> 5)];
            if (t == 0 || ((mi >> (((8 * t) & 31) + g)) & 1u)) {
                // (clamped: a factorization that stopped at an exactly singular
                // column leaves later records unwritten; its status reports it)
                const int sr = min((unsigned)ri[8 * t + g], (unsigned)(8 * TRW - 1));
                const double2 vv = *reinterpret_cast<const double2*>(&xs[sr * 8 + 2 * q]);
                Wt[t][0] = vv.x;
                Wt[t][1] = vv.y;
            }
        }
        __syncwarp();
        // 2. X = L11^-1 (tile 0): B fragments B[k][n] = P[4s+k][n] by shuffles
        double pb[2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int src = 4 * (4 * s2 + q) + (g >> 1);
            const double v0 = __shfl_sync(full, Wt[0][0], src);
            const double v1 = __shfl_sync(full, Wt[0][1], src);
            pb[s2] = (g & 1) ? v1 : v0;
        }
        double x0 = 0.0, x1 = 0.0;
        ps_dmma(x0, x1, rec[lane], pb[0]);
        ps_dmma(x0, x1, rec[32 + lane], pb[1]);
        double xb[2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int src = 4 * (4 * s2 + q) + (g >> 1);
            const double v0 = __shfl_sync(full, x0, src);
            const double v1 = __shfl_sync(full, x1, src);
            xb[s2] = (g & 1) ? v1 : v0;
        }
        // 3. the window below: W_t += (-L21_t) X, next tile first
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int t = 1; t < TRW; ++t) ps_dmma(Wt[t][0], Wt[t][1], rec[64 * t + 32 * s2 + lane], xb[s2]);
        {
            const int row = 8 * Jp + g;
            if (row < m && row >= lo) {
                const long long pr = phys(row);
                if (cv0) cp0[pr] = x0;
                if (cv1) cp1[pr] = x1;
            }
        }
        // 4. rotate; the freed tile takes rows 8 (Jp + TRW) ..
#pragma unroll
        for (int t = 0; t + 1 < TRW; ++t) {
            Wt[t][0] = Wt[t + 1][0];
            Wt[t][1] = Wt[t + 1][1];
        }
        const double* in = s_in + (size_t)st * 8 * RND * sin_ld + (8 * bb + g) * sin_ld + lc0;
        Wt[TRW - 1][0] = in[0];
        Wt[TRW - 1][1] = in[1];
    }
    cp_async_wait<0>();
}

template <int TRW>
static bool launch_piv_sweep(int nwarps, dim3 grid, const PivSweepArgs& A, cudaStream_t s) {
    const size_t smem = piv_sweep_smem<TRW>(nwarps);
    if (smem > 227 * 1024) return false;
    set_smem_attr((const void*)k_sweep_piv_dmma<TRW>, (int)smem);
    k_sweep_piv_dmma<TRW><<<grid, 32 * nwarps, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_sweep_piv_dmma(int trw, int nwarps, dim3 grid, const PivSweepArgs& A, cudaStream_t s) {
    switch (trw) {
        case 5: return launch_piv_sweep<5>(nwarps, grid, A, s);
        case 9: return launch_piv_sweep<9>(nwarps, grid, A, s);
        case 13: return launch_piv_sweep<13>(nwarps, grid, A, s);
        default: return false;
    }
}

// ===========================================================================
// Transposed pivoted L sweep, B := P^T L^-T B (backward_lowerT /
// lowerT_perm_bottom_tip, src/kernels.cpp:219-261: for rows i = m-1 .. lo,
// B(i) -= l_i . B(i+1 .. i+kl), then interchange B(i) and B(ip)).  The forward
// sweep applies panel operators M_J = [[L11^-1, 0], [-L21 L11^-1, I]] P_J in
// increasing J, so the transpose applies M_J^T = P_J^T [[L11^-T, (-L21 L11^-1)^T],
// [0, I]] in decreasing J over the same window: per panel
//   t' = L11^-T (t + (-L21)^T r)      (t = window tile 0, r = tiles 1 ..)
//   window := P_J^T window            (inverse of the record's permutation)
// with the same records read transposed (A fragments gathered from shared
// memory).  The window slides up one tile per panel: its bottom tile is final
// (no earlier panel reaches it) and the rows above enter from B.  Here the
// window lives in DMMA B-fragment layout (lane: rows 4s + (lane&3) of each
// tile, column lane>>2), so the reduction (-L21)^T r needs no shuffles.
// A job with lo not a multiple of 8 ends with the reference's per-row steps
// on panel lo/8 (rows lo .. 8 (lo/8) + 7) from the packed factor and pivots:
// rows below lo are neither read nor written.
template <int TRW>
__global__ void __launch_bounds__(512) k_sweep_piv_dmma_t(PivSweepArgs A) {
    using R = PivRec<TRW>;
    constexpr int RND = kPsRound;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const SweepJob J = A.jobs[blockIdx.x];
    if (!guard_ok(A.B.flags, J.guard)) return;
    const PartDev P = A.parts[J.part];
    const int nc_total = J.nc >= 0 ? J.nc : A.ncols;
    const int nwarps = blockDim.x >> 5, ncta = nwarps * 8, sin_ld = ncta + 1;
    const int colbase = blockIdx.y * ncta;
    if (colbase >= nc_total) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const unsigned full = 0xffffffffu;
    const int m = P.m, lo = max(J.lo, 0);
    const int J0 = lo / 8, nblk = (m + 7) / 8;
    if (J0 >= nblk) return;
    const bool partial = (lo & 7) != 0;
    const int nfull = nblk - J0 - (partial ? 1 : 0);  // DMMA panels nblk-1 .. nblk-nfull

    double* s_rec = reinterpret_cast<double*>(smem_raw);            // [2][RND][R::SIZE]
    double* s_in = s_rec + 2 * RND * R::SIZE;                        // [2][8 RND][ncta+1]
    double* xs = s_in + 2 * 8 * RND * sin_ld + warp * 8 * TRW * 8;  // per-warp [8TRW][8]

    const View& v = J.v;
    const long long ld = v.ld >= 0 ? v.ld : A.B.ld[v.buf];
    double* const bbase = A.B.p[v.buf] + v.base;
    auto phys = [&](int r) -> long long {
        return v.rev ? (long long)(v.mrows - 1 - (r - v.off)) : (long long)(r - v.off);
    };
    const int c0 = J.c0 + colbase;
    const int ncta_valid = min(ncta, nc_total - colbase);
    const int lc = warp * 8 + g;  // this lane's column (B-fragment layout)
    const bool cv = lc < ncta_valid;
    double* const cp = bbase + (long long)(c0 + (cv ? lc : 0)) * ld;
    const double* recbase = A.lblk + (P.r0 / 8 + J.part) * (long long)R::SIZE;

    // round Rr: records of panels nblk-1-(RND Rr + b), b < nb, and the rows
    // entering after each (8 (Jp - 1) + t, t < 8)
    auto load_round = [&](int Rr) {
        const int st = Rr & 1, k0 = RND * Rr;
        if (k0 < nfull) {
            const int nb = min(RND, nfull - k0);
            double* dr = s_rec + (size_t)st * RND * R::SIZE;
            constexpr int H = R::SIZE / 2;
            for (int idx = threadIdx.x; idx < nb * H; idx += blockDim.x) {
                const int b = idx / H, o = idx - b * H;
                cp_async16(dr + (size_t)b * R::SIZE + 2 * o, recbase + (long long)(nblk - 1 - k0 - b) * R::SIZE + 2 * o);
            }
            double* di = s_in + (size_t)st * 8 * RND * sin_ld;
            for (int idx = threadIdx.x; idx < 8 * RND * ncta; idx += blockDim.x) {
                const int t = idx & 31, col = idx >> 5;  // t = 8 b + row
                const int row = 8 * (nblk - 2 - k0 - (t >> 3)) + (t & 7);
                double* dst = di + t * sin_ld + col;
                if ((t >> 3) < nb && row >= lo && row < m && col < ncta_valid)
                    cp_async8(dst, bbase + phys(row) + (long long)(c0 + col) * ld);
                else *dst = 0.0;
            }
        }
        cp_async_commit();
    };

    // window of panel nblk-1: tile 0 = rows 8 (nblk-1) .., the tiles below are
    // past the partition
    double Wt[TRW][2];
#pragma unroll
    for (int t = 0; t < TRW; ++t)
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int row = 8 * (nblk - 1 + t) + 4 * s2 + q;
            Wt[t][s2] = (t == 0 && row >= lo && row < m && cv) ? cp[phys(row)] : 0.0;
        }
    load_round(0);

    int base = 8 * (nblk - 1);  // first row of window tile 0
    for (int k = 0; k < nfull; ++k) {
        const int st = (k / RND) & 1, bb = k % RND;
        if (bb == 0) {
            cp_async_wait<0>();
            __syncthreads();
            load_round(k / RND + 1);
        }
        const double* rec = s_rec + (size_t)(st * RND + bb) * R::SIZE;
        const int* ri = reinterpret_cast<const int*>(rec + R::SRC);
        // 1. u = t + (-L21)^T r: A fragment (i = g, kk = q) of slice s of
        //    (-L21_t)^T is (-L21_t)[4s + q][g]
        double a0 = 0.0, a1 = 0.0;
        const int ao = 32 * (g >> 2) + (g & 3);
#pragma unroll
        for (int t = 1; t < TRW; ++t)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) ps_dmma(a0, a1, rec[64 * t + ao + 4 * (4 * s2 + q)], Wt[t][s2]);
        // accumulator (row g, cols 2q, 2q+1) -> B fragment (row 4s + q, col g)
        double u[2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int src = 4 * (4 * s2 + q) + (g >> 1);
            const double v0 = __shfl_sync(full, a0, src);
            const double v1 = __shfl_sync(full, a1, src);
            u[s2] = Wt[0][s2] + ((g & 1) ? v1 : v0);
        }
        // 2. t' = L11^-T u
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) ps_dmma(x0, x1, rec[ao + 4 * (4 * s2 + q)], u[s2]);
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int src = 4 * (4 * s2 + q) + (g >> 1);
            const double v0 = __shfl_sync(full, x0, src);
            const double v1 = __shfl_sync(full, x1, src);
            Wt[0][s2] = (g & 1) ? v1 : v0;
        }
        // 3. window := P_J^T window.  The record maps each receiving position
        //    (tile 0 and mv_in) to its source (tile 0 and mv_out); the inverse
        //    scatters the receivers back to their sources
#pragma unroll
        for (int t = 0; t < TRW; ++t)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int pos = 8 * t + 4 * s2 + q;
                const unsigned mi = (unsigned)ri[8 * TRW + R::NSLW + (pos >> 5)];
                if (t == 0 || ((mi >> (pos & 31)) & 1u)) {
                    const int sr = min((unsigned)ri[pos], (unsigned)(8 * TRW - 1));
                    xs[sr * 8 + g] = Wt[t][s2];
                }
            }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < TRW; ++t)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int pos = 8 * t + 4 * s2 + q;
                const unsigned mo = (unsigned)ri[8 * TRW + (pos >> 5)];
                if (t == 0 || ((mo >> (pos & 31)) & 1u)) Wt[t][s2] = xs[pos * 8 + g];
            }
        __syncwarp();
        // 4. the bottom tile is final; the window moves up one tile
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int row = base + 8 * (TRW - 1) + 4 * s2 + q;
            if (row < m && cv) cp[phys(row)] = Wt[TRW - 1][s2];
        }
#pragma unroll
        for (int t = TRW - 1; t > 0; --t) {
            Wt[t][0] = Wt[t - 1][0];
            Wt[t][1] = Wt[t - 1][1];
        }
        const double* in = s_in + (size_t)st * 8 * RND * sin_ld + lc;
        Wt[0][0] = in[(8 * bb + q) * sin_ld];
        Wt[0][1] = in[(8 * bb + 4 + q) * sin_ld];
        base -= 8;
    }
    cp_async_wait<0>();
    if (partial) {
        // panel J0 (base == 8 J0): the reference's steps i = 8 J0 + 7 .. lo,
        // window rows in the per-warp scratch; 4 lanes per column share a dot
#pragma unroll
        for (int t = 0; t < TRW; ++t)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) xs[(8 * t + 4 * s2 + q) * 8 + g] = Wt[t][s2];
        __syncwarp();
        const double* F = A.fac + P.fofs;
        const int* piv = A.piv + P.r0;
        const int c = lane >> 2, j = lane & 3;
        for (int i = min(base + 7, m - 1); i >= lo; --i) {
            const int pi = i - base, rl = min(P.kl, m - 1 - i);
            const double* li = F + (long long)i * P.rows + P.d + 1;
            double part = 0.0;
            for (int r = j; r < rl; r += 4) part += li[r] * xs[(pi + 1 + r) * 8 + c];
            part += __shfl_xor_sync(full, part, 1);
            part += __shfl_xor_sync(full, part, 2);
            __syncwarp();
            if (j == 0) xs[pi * 8 + c] -= part;
            __syncwarp();
            const int ip = P.pivoting ? piv[i] : i;
            if (ip != i && j == 0) {
                const int pp = min(ip - base, 8 * TRW - 1);
                const double tmp = xs[pi * 8 + c];
                xs[pi * 8 + c] = xs[pp * 8 + c];
                xs[pp * 8 + c] = tmp;
            }
            __syncwarp();
        }
#pragma unroll
        for (int t = 0; t < TRW; ++t)
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) Wt[t][s2] = xs[(8 * t + 4 * s2 + q) * 8 + g];
    }
    // flush the rest of the window (rows lo .. m-1 only)
#pragma unroll
    for (int t = 0; t < TRW; ++t)
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int row = base + 8 * t + 4 * s2 + q;
            if (row >= lo && row < m && cv) cp[phys(row)] = Wt[t][s2];
        }
}

template <int TRW>
static bool launch_piv_sweep_t(int nwarps, dim3 grid, const PivSweepArgs& A, cudaStream_t s) {
    const size_t smem = piv_sweep_smem<TRW>(nwarps);
    if (smem > 227 * 1024) return false;
    set_smem_attr((const void*)k_sweep_piv_dmma_t<TRW>, (int)smem);
    k_sweep_piv_dmma_t<TRW><<<grid, 32 * nwarps, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_sweep_piv_dmma_t(int trw, int nwarps, dim3 grid, const PivSweepArgs& A, cudaStream_t s) {
    switch (trw) {
        case 5: return launch_piv_sweep_t<5>(nwarps, grid, A, s);
        case 9: return launch_piv_sweep_t<9>(nwarps, grid, A, s);
        case 13: return launch_piv_sweep_t<13>(nwarps, grid, A, s);
        default: return false;
    }
}

}  // namespace spk
