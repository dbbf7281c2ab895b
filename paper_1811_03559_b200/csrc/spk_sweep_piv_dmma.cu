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

}  // namespace spk
