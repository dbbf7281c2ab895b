// spk_sweep_fast.cuh — register-window triangular sweeps for SPIKE partitions.
//
// One CTA per (partition, group of right-hand-side columns); each warp owns NC
// columns.  The active band window of every column (KW = 32*TR rows: the
// current pivot row and the rows it still updates) lives in registers, one
// circular slot per (lane, register).  Per step u of the sweep:
//   x_c   = pivot row value (warp shuffle from the owning lane), scaled by the
//           precomputed reciprocal diagonal for U sweeps;
//   slot  <- next input row (recycled: the pivot row leaves, row u+KW enters);
//   W    -= v_u (x) x   (rank-1 axpy over the window, DFMA)
// where v_u is the step's factor vector (a column of L or U, or a row of L or
// U for the transpose sweeps, read from the row-major factor copy).  Factor
// vectors, reciprocal diagonals, pivots and the incoming rows are staged one
// 32-step round at a time through a 3-stage cp.async ring in shared memory, so
// HBM latency is hidden behind >= 2 rounds of arithmetic.  The pivot slot's
// register index is a compile-time constant inside each round (rounds are
// unrolled TR at a time), so the window never spills to local memory.
//
// Covers (reference /root/reference/proj/src/kernels.cpp):
//   SW_FWD_L   forward_lower (+ LAPACK-style row interchanges)   :131-165
//   SW_BWD_U   backward_upper / upper_bottom_tip                 :167-202
//   SW_FWD_UT  forward_upperT / add_upperT_tail (row-major U)    :204-217, :263-280
//   SW_BWD_LT  backward_lowerT, non-pivoting (row-major L)       :219-234
#pragma once

#include "spk_device.cuh"

namespace spk {


__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
// mbarrier helpers (shared::cta): the DMMA sweeps' producer/consumer rings
// and warp-pair handshakes
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_cp_async_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct FastSweepArgs {
    const SweepJob* jobs;
    const PartDev* parts;
    const double* fac;   // column-major packed LU factors
    const double* tfac;  // row-major copies (transpose sweeps)
    const double* dinv;  // 1/u_jj per partition row
    const int* piv;      // partition-local pivots per row
    Bufs B;
    int ncols;
};

// Window of TW = TR+1 register rows per column (KW = 32*TW slots): during round
// R (32 steps) the pivots are register row R mod TW; the other TR rows cover
// every row the round's pivots update.  A finished pivot row stays untouched
// (its vector slots are zero) until the round ends; then it is written back
// (times 1/u_jj for U sweeps) and refilled with the rows 32*TW further on.  No
// per-step selects or divergent branches.
template <int TR>
struct SweepGeom {
    static constexpr int TW = TR + 1;
    static constexpr int KW = 32 * TW;
    static constexpr int NST = (TR <= 5) ? 3 : 2;
};

inline size_t fast_sweep_smem(int tr, int nwarps, int nc) {
    const int KW = 32 * (tr + 1);
    const int nst = tr <= 5 ? 3 : 2;
    const size_t per_stage = 32 * (size_t)KW * 8 + 32 * 8 + 32 * 4 + 32 * (size_t)nwarps * nc * 8;
    return nst * per_stage + 64;
}

template <int TR, int NC, int MODE, bool PIV>
__global__ void __launch_bounds__(640) k_sweep_fast(FastSweepArgs A) {
    constexpr int TW = SweepGeom<TR>::TW;
    constexpr int KW = SweepGeom<TR>::KW;
    constexpr int NST = SweepGeom<TR>::NST;
    constexpr bool kAsc = (MODE == SW_FWD_L || MODE == SW_FWD_UT);
    constexpr bool kDiag = (MODE == SW_BWD_U || MODE == SW_FWD_UT);
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const SweepJob J = A.jobs[blockIdx.x];
    if (!guard_ok(A.B.flags, J.guard)) return;
    const PartDev P = A.parts[J.part];
    const int nc_total = J.nc >= 0 ? J.nc : A.ncols;
    const int nwarps = blockDim.x >> 5;
    const int ncta = nwarps * NC;
    const int colbase = blockIdx.y * ncta;
    if (colbase >= nc_total) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int lo = J.lo;
    const int hi = (MODE == SW_BWD_U) ? J.hi : P.m - 1;
    const int nsteps = hi - lo + 1;
    if (nsteps <= 0) return;

    int kw;
    const double* vbase;
    long long vstride;
    int vdir;
    if (MODE == SW_FWD_L) {
        kw = P.kl;
        vbase = A.fac + P.fofs + P.d + 1;
        vstride = P.rows;
        vdir = 1;
    } else if (MODE == SW_BWD_U) {
        kw = P.ubw;
        vbase = A.fac + P.fofs + P.d - 1;
        vstride = P.rows;
        vdir = -1;
    } else if (MODE == SW_FWD_UT) {
        kw = P.ubw;
        vbase = A.tfac + P.tofs + P.kl + 1;
        vstride = P.rowsT;
        vdir = 1;
    } else {
        kw = P.kl;
        vbase = A.tfac + P.tofs + P.kl - 1;
        vstride = P.rowsT;
        vdir = -1;
    }

    double* s_vec = reinterpret_cast<double*>(smem_raw);                    // [st][32][KW]
    double* s_dg = s_vec + (size_t)NST * 32 * KW;                           // [st][32]
    double* s_in = s_dg + NST * 32;                                         // [st][32][ncta]
    int* s_pv = reinterpret_cast<int*>(s_in + (size_t)NST * 32 * ncta);     // [st][32]

    const View& v = J.v;
    const long long ld = v.ld >= 0 ? v.ld : A.B.ld[v.buf];
    double* const bbase = A.B.p[v.buf] + v.base;
    auto phys = [&](int r) -> long long {
        return v.rev ? (long long)(v.mrows - 1 - (r - v.off)) : (long long)(r - v.off);
    };
    auto rowof = [&](int u) -> int { return kAsc ? lo + u : hi - u; };

    const int c0 = J.c0 + colbase;
    const int ncta_valid = min(ncta, nc_total - colbase);
    bool cval[NC];
    double* cptr[NC];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
        const int lc = warp * NC + cc;
        cval[cc] = lc < ncta_valid;
        cptr[cc] = bbase + (long long)(c0 + (cval[cc] ? lc : 0)) * ld;
    }

    // stage round R: vectors of steps 32R.. in slot order, 1/u_jj, pivots, and
    // the rows that refill the window at the end of round R (rows 32(R+TW)+l)
    auto load_round = [&](int R) {
        const int st = R % NST;
        const int u0 = 32 * R;
        if (u0 < nsteps) {
            const int pa = 32 * (R % TW);
            double* dv = s_vec + (size_t)st * 32 * KW;
            for (int idx = threadIdx.x; idx < 32 * KW; idx += blockDim.x) {
                const int t = idx / KW, sl = idx - t * KW;
                int dl = sl - pa - t - 1;
                if (dl < 0) dl += KW;
                const int u = u0 + t;
                if (dl < kw && u < nsteps)
                    cp_async8(dv + idx, vbase + (long long)rowof(u) * vstride + vdir * dl);
                else
                    dv[idx] = 0.0;
            }
            if (threadIdx.x < 32) {
                const int u = u0 + threadIdx.x;
                if (u < nsteps) {
                    const int j = rowof(u);
                    if (kDiag) cp_async8(s_dg + st * 32 + threadIdx.x, A.dinv + P.r0 + j);
                    if (PIV) cp_async4(s_pv + st * 32 + threadIdx.x, A.piv + P.r0 + j);
                }
            }
            double* di = s_in + (size_t)st * 32 * ncta;
            for (int idx = threadIdx.x; idx < 32 * ncta; idx += blockDim.x) {
                const int t = idx & 31, col = idx >> 5;
                const int uu = u0 + t + KW;
                double* dst = di + t * ncta + col;
                if (uu < nsteps && col < ncta_valid)
                    cp_async8(dst, bbase + phys(rowof(uu)) + (long long)(c0 + col) * ld);
                else
                    *dst = 0.0;
            }
        }
        cp_async_commit();
    };

    double W[TW][NC];
#pragma unroll
    for (int a = 0; a < TW; ++a) {
        const int u = 32 * a + lane;
        const bool ok = u < nsteps;
        const long long pr = ok ? phys(rowof(u)) : 0;
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) W[a][cc] = (ok && cval[cc]) ? cptr[cc][pr] : 0.0;
    }

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) load_round(s);

    const int nrounds = (nsteps + 31) / 32;
    for (int R0 = 0; R0 < nrounds; R0 += TW) {
#pragma unroll
        for (int a = 0; a < TW; ++a) {
            const int R = R0 + a;
            if (R < nrounds) {
                cp_async_wait<NST - 2>();
                __syncthreads();
                load_round(R + NST - 1);
                const int st = R % NST;
                const double* vec = s_vec + (size_t)st * 32 * KW + lane;
                const double* dg = s_dg + st * 32;
                const int steps = min(32, nsteps - 32 * R);
#pragma unroll 2
                for (int t = 0; t < steps; ++t) {
                    if (PIV) {
                        const int ip = s_pv[st * 32 + t];
                        const int du = ip - rowof(32 * R + t);  // 0..kl
                        int sl = 32 * a + t + du;
                        if (sl >= KW) sl -= KW;
                        const int lip = sl & 31, rip = sl >> 5;
#pragma unroll
                        for (int cc = 0; cc < NC; ++cc) {
                            double wsel = W[0][cc];
#pragma unroll
                            for (int q = 1; q < TW; ++q)
                                if (rip == q) wsel = W[q][cc];
                            const double vp = __shfl_sync(0xffffffffu, W[a][cc], t);
                            const double vi = __shfl_sync(0xffffffffu, wsel, lip);
                            if (lane == lip) {
#pragma unroll
                                for (int q = 0; q < TW; ++q)
                                    if (rip == q) W[q][cc] = vp;
                            }
                            if (lane == t) W[a][cc] = vi;
                        }
                    }
                    double x[NC];
                    const double dgt = kDiag ? dg[t] : 1.0;
#pragma unroll
                    for (int cc = 0; cc < NC; ++cc) {
                        x[cc] = __shfl_sync(0xffffffffu, W[a][cc], t);
                        if (kDiag) x[cc] *= dgt;
                    }
                    const double* vr = vec + t * KW;
                    // the pivot register row first: it feeds the next step's shuffle
                    {
                        const double lv = vr[32 * a];
#pragma unroll
                        for (int cc = 0; cc < NC; ++cc) W[a][cc] = fma(-lv, x[cc], W[a][cc]);
                    }
#pragma unroll
                    for (int a2 = 0; a2 < TW; ++a2) {
                        if (a2 == a) continue;
                        const double lv = vr[32 * a2];
#pragma unroll
                        for (int cc = 0; cc < NC; ++cc) W[a2][cc] = fma(-lv, x[cc], W[a2][cc]);
                    }
                }
                // register row a now holds this round's finished pivot rows:
                // write them back, then refill with the rows 32*TW further on
                if (lane < steps) {
                    const long long pr = phys(rowof(32 * R + lane));
                    const double sc = kDiag ? dg[lane] : 1.0;
#pragma unroll
                    for (int cc = 0; cc < NC; ++cc)
                        if (cval[cc]) cptr[cc][pr] = kDiag ? W[a][cc] * sc : W[a][cc];
                }
                const double* in = s_in + (size_t)st * 32 * ncta + lane * ncta + warp * NC;
#pragma unroll
                for (int cc = 0; cc < NC; ++cc) W[a][cc] = in[cc];
            }
        }
    }
    cp_async_wait<0>();
}

}  // namespace spk
