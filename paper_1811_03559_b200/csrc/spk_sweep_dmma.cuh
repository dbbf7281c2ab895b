// spk_sweep_dmma.cuh — blocked triangular sweeps on the FP64 tensor cores.
//
// Same jobs and semantics as k_sweep_fast (non-pivoting modes), restructured
// for DMMA (mma.sync.m8n8k4.f64): each warp owns 8 right-hand-side columns and
// keeps the active band window as NTW 8x8 tiles in the accumulator (C
// fragment) layout — lane l holds row l>>2, columns 2(l&3), 2(l&3)+1 of every
// tile.  The sweep advances 8 rows per block:
//   1. the pivot tile (rows 8b..8b+7) is solved in place: 8 in-tile steps of
//      x_t = P_t (* 1/u for U sweeps); P_{t'} -= v_t[t'-t-1] x_t   (shuffles);
//   2. its rows become the B operand (8 steps x 8 columns) and every other
//      tile takes a rank-8 update  W_T -= A_T X  with A_T[r][t] = v_{8b+t}[r-t-1]
//      — two DMMA per tile, A fragments loaded from a shared-memory block of
//      factor vectors laid out [step][row] with a row stride = 8 (mod 16)
//      doubles (conflict-free fragment loads);
//   3. the solved tile is written back and its register slot recycled for the
//      rows 8*NTW further on (staged one 32-row round ahead by cp.async).
// Per 8 rows a warp issues 2(NTW-1) DMMA + 2(NTW-1) LDS + ~100 other
// instructions against 8*8*(NTW-1)*8 FMAs, i.e. ~4x fewer issue slots and half
// the shared-memory bytes per FMA of the per-row DFMA kernel.  Row interchanges
// (pivoting) do not commute with the blocked update in gbtf2 storage, so the
// pivoted forward sweep stays on k_sweep_fast.
#pragma once

#include "spk_device.cuh"
#include "spk_sweep_fast.cuh"

namespace spk {

__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NTW>
struct DmmaGeom {
    static constexpr int KWT = 8 * (NTW - 1);                       // longest factor vector
    static constexpr int SR = ((8 + KWT + 15) / 16) * 16 + 4;       // [step][row] stride, = 4 mod 16
};

// PAIR: nwarps counts both warps of each pair (ncta = 4 nwarps columns)
inline size_t dmma_sweep_smem(int ntw, int nwarps, bool pair = false) {
    const int KWT = 8 * (ntw - 1);
    const int SR = ((8 + KWT + 15) / 16) * 16 + 4;
    const int ncta = (pair ? nwarps / 2 : nwarps) * 8;
    const size_t per_stage = (size_t)4 * 8 * SR * 8 + 32 * 8 + (size_t)32 * (ncta + 1) * 8 + 4 * 64 * 8;
    return 2 * per_stage + 64 + (pair ? (size_t)(nwarps / 2) * (4 * 64 * 8 + 16) : 0);
}

// PAIR: two warps per 8 right-hand-side columns split the window (A: tiles
// 0 .. HA-1 and X, B: tiles HA .. NTW-1 and the incoming rows), with the X
// (A -> B) and front-tile (B -> A) handoffs of k_sweep_dmma2's pair mode;
// each warp issues about half the DMMAs of a block (a warp issues at most one
// per ~32 cycles, profiles/r01_dmma_occupancy.txt).
template <int NTW, int MODE, bool PAIR = false>
__global__ void __launch_bounds__(512) k_sweep_dmma(FastSweepArgs A) {
    constexpr int SR = DmmaGeom<NTW>::SR;
    constexpr int KWT = DmmaGeom<NTW>::KWT;
    constexpr bool kAsc = (MODE == SW_FWD_L || MODE == SW_FWD_UT);
    constexpr bool kDiag = (MODE == SW_BWD_U || MODE == SW_FWD_UT);
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const SweepJob J = A.jobs[blockIdx.x];
    if (!guard_ok(A.B.flags, J.guard)) return;
    const PartDev P = A.parts[J.part];
    const int nc_total = J.nc >= 0 ? J.nc : A.ncols;
    const int nwarps = blockDim.x >> 5;
    const int ncta = (PAIR ? nwarps / 2 : nwarps) * 8;
    const int sin_ld = ncta + 1;
    const int colbase = blockIdx.y * ncta;
    if (colbase >= nc_total) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;

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

    double* s_A = reinterpret_cast<double*>(smem_raw);      // [st][4 blocks][8 steps][SR rows]
    double* s_dg = s_A + 2 * 4 * 8 * SR;                     // [st][32]
    double* s_in = s_dg + 2 * 32;                            // [st][32 rows][ncta+1] (odd stride)
    double* s_ti = s_in + 2 * 32 * (ncta + 1);               // [st][4 blocks][8][8] inverse diagonal blocks
    double* s_pair = s_ti + 2 * 4 * 64;                       // PAIR: [pair][xbuf 2x64, tbuf 2x64]
    unsigned long long* s_pbar = reinterpret_cast<unsigned long long*>(s_pair + (size_t)(nwarps / 2) * 4 * 64);
    if (PAIR && threadIdx.x < nwarps) mbar_init(s_pbar + threadIdx.x, 32);

    const View& v = J.v;
    const long long ld = v.ld >= 0 ? v.ld : A.B.ld[v.buf];
    double* const bbase = A.B.p[v.buf] + v.base;
    auto phys = [&](int r) -> long long {
        return v.rev ? (long long)(v.mrows - 1 - (r - v.off)) : (long long)(r - v.off);
    };
    auto rowof = [&](int u) -> int { return kAsc ? lo + u : hi - u; };

    const int c0 = J.c0 + colbase;
    const int ncta_valid = min(ncta, nc_total - colbase);
    const int lc0 = (PAIR ? warp >> 1 : warp) * 8 + 2 * q;  // this lane's two columns (CTA-local)
    const bool cv0 = lc0 < ncta_valid, cv1 = lc0 + 1 < ncta_valid;
    double* const cp0 = bbase + (long long)(c0 + (cv0 ? lc0 : 0)) * ld;
    double* const cp1 = bbase + (long long)(c0 + (cv1 ? lc0 + 1 : 0)) * ld;

    // Staging, a few instructions per entry: a thread keeps one factor vector
    // of the round (step vt, entries vj, vj + nwarps, ...) and one row of the
    // incoming right-hand sides (row rt, columns rc0, rc0 + nwarps, ...), so the
    // stage offsets are fixed and the sources step by constants.  Out-of-band
    // stage slots are zeroed once (both buffers) and never loaded; vectors past
    // the sweep end keep stale finite data that the zero rows of Tinv cancel.
    // (One flat loop over the stage, with a division per entry and the zero
    // slots rewritten every round, was a third of the kernel's instructions.)
    const int vt = threadIdx.x / nwarps, vj = threadIdx.x - vt * nwarps;
    const int sdst = vt * SR + (vt & 7) + 1 + vj;
    const int rt = threadIdx.x & 31, rc0 = threadIdx.x >> 5;
    for (int idx = threadIdx.x; idx < 2 * 4 * 8 * SR; idx += blockDim.x) s_A[idx] = 0.0;
    __syncthreads();
    auto load_round = [&](int R) {
        const int st = R & 1;
        const int u0 = 32 * R;
        if (u0 < nsteps) {
            double* dA = s_A + (size_t)st * 4 * 8 * SR;
            if (u0 + vt < nsteps) {
                const double* src = vbase + (long long)rowof(u0 + vt) * vstride + vdir * vj;
                double* dst = dA + sdst;
                for (int dl = vj; dl < kw; dl += nwarps) {
                    cp_async8(dst, src);
                    dst += nwarps;
                    src += vdir * nwarps;
                }
            }
            if (kDiag && threadIdx.x < 32) {
                const int u = u0 + threadIdx.x;
                if (u < nsteps) cp_async8(s_dg + st * 32 + threadIdx.x, A.dinv + P.r0 + rowof(u));
            }
            double* dst = s_in + (size_t)st * 32 * sin_ld + rt * sin_ld + rc0;
            const int uu = u0 + rt + 8 * NTW;
            const bool ok = uu < nsteps;
            const double* src = bbase + (ok ? phys(rowof(uu)) : 0) + (long long)(c0 + rc0) * ld;
            for (int col = rc0; col < ncta; col += nwarps) {
                if (ok && col < ncta_valid) cp_async8(dst, src);
                else *dst = 0.0;
                dst += nwarps;
                src += (long long)nwarps * ld;
            }
        }
        cp_async_commit();
    };

    load_round(0);

    // Per 8-row block the system is  P = M X  with M the 8x8 diagonal block of
    // the triangular factor (M[r][t] = v_t[r-t-1] below, 1 or u_tt on the
    // diagonal).  At each round start one warp forms Tinv = M^-1 for the
    // round's 4 blocks, so a block is X = Tinv P (2 DMMA) followed by the
    // rank-8 update W_i -= A_i X (2 DMMA per tile): a short shuffle/DMMA chain
    // instead of an 8-step serial in-tile solve.
    auto prep_round = [&](int st, int u0) {
        double* Ar = s_A + (size_t)st * 4 * 8 * SR;
        double* Ti = s_ti + (size_t)st * 4 * 64;
        const double* dg = s_dg + st * 32;
        // Tinv columns: thread (bb, c) solves M y = e_c by forward substitution
        if (threadIdx.x < 32) {
            const int bb = threadIdx.x >> 3, c = threadIdx.x & 7;
            const double* Ab = Ar + (size_t)bb * 8 * SR;
            double y[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double acc = (r == c) ? 1.0 : 0.0;
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (t < r) acc -= Ab[t * SR + r] * y[t];
                // diagonal: 1 for unit sweeps, u_tt = 1/dinv for U sweeps
                y[r] = kDiag ? acc * dg[8 * bb + r] : acc;
                if (u0 + 8 * bb + r >= nsteps) y[r] = 0.0;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) Ti[bb * 64 + r * 8 + c] = y[r];  // Tinv[r][c]
        }
        __syncthreads();
    };

    if constexpr (PAIR) {
        constexpr int HA = (NTW + 1) / 2, HB = NTW - HA;
        const int pr_ = warp >> 1, role = warp & 1;
        double* xbuf = s_pair + (size_t)pr_ * 4 * 64;  // [2][64]: -X as B fragments (A -> B)
        double* tbuf = xbuf + 128;                      // [2][64]: B's front tile (B -> A)
        unsigned long long* mbx = s_pbar + 2 * pr_;
        unsigned long long* mbt = mbx + 1;
        const int nblocks = (nsteps + 7) / 8;
        if (role == 0) {
            double Wt[HA][2];
#pragma unroll
            for (int T = 0; T < HA; ++T) {
                const int u = 8 * T + g;
                const bool ok = u < nsteps;
                const long long pr = ok ? phys(rowof(u)) : 0;
                Wt[T][0] = (ok && cv0) ? cp0[pr] : 0.0;
                Wt[T][1] = (ok && cv1) ? cp1[pr] : 0.0;
            }
            for (int b = 0; b < nblocks; ++b) {
                const int st = (b >> 2) & 1, bb = b & 3;
                if (bb == 0) {
                    cp_async_wait<0>();
                    __syncthreads();
                    prep_round(st, 8 * b);
                    load_round((b >> 2) + 1);
                }
                const double* Ab = s_A + (size_t)((st * 4 + bb) * 8) * SR;
                const double* T = s_ti + (size_t)(st * 4 + bb) * 64;
                double pb[2];
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const int src = 4 * (4 * s2 + q) + (g >> 1);
                    const double v0 = __shfl_sync(0xffffffffu, Wt[0][0], src);
                    const double v1 = __shfl_sync(0xffffffffu, Wt[0][1], src);
                    pb[s2] = (g & 1) ? v1 : v0;
                }
                double x0 = 0.0, x1 = 0.0;
                dmma_acc(x0, x1, T[g * 8 + q], pb[0]);
                dmma_acc(x0, x1, T[g * 8 + 4 + q], pb[1]);
                double nb[2];
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const int src = 4 * (4 * s2 + q) + (g >> 1);
                    const double v0 = __shfl_sync(0xffffffffu, x0, src);
                    const double v1 = __shfl_sync(0xffffffffu, x1, src);
                    nb[s2] = -((g & 1) ? v1 : v0);
                }
                *reinterpret_cast<double2*>(xbuf + (b & 1) * 64 + 2 * lane) = make_double2(nb[0], nb[1]);
                if (b > 0) mbar_wait(mbt, (b - 1) & 1);  // B took X of block b-1: one phase apart
                mbar_arrive(mbx);
                if (b > 0) {  // my last tile is B's front tile of the previous block
                    const double2 t = *reinterpret_cast<const double2*>(tbuf + ((b - 1) & 1) * 64 + 2 * lane);
                    Wt[HA - 1][0] = t.x;
                    Wt[HA - 1][1] = t.y;
                }
                dmma_acc(Wt[1][0], Wt[1][1], Ab[q * SR + 8 + g], nb[0]);
                dmma_acc(Wt[1][0], Wt[1][1], Ab[(4 + q) * SR + 8 + g], nb[1]);
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                    for (int i = 2; i < HA; ++i) dmma_acc(Wt[i][0], Wt[i][1], Ab[(4 * s2 + q) * SR + 8 * i + g], nb[s2]);
                {
                    const int u = 8 * b + g;
                    if (u < nsteps) {
                        const long long pr = phys(rowof(u));
                        if (cv0) cp0[pr] = x0;
                        if (cv1) cp1[pr] = x1;
                    }
                }
#pragma unroll
                for (int i = 0; i < HA - 1; ++i) {
                    Wt[i][0] = Wt[i + 1][0];
                    Wt[i][1] = Wt[i + 1][1];
                }
            }
        } else {
            double Wt[HB][2];
#pragma unroll
            for (int T = 0; T < HB; ++T) {
                const int u = 8 * (HA + T) + g;
                const bool ok = u < nsteps;
                const long long pr = ok ? phys(rowof(u)) : 0;
                Wt[T][0] = (ok && cv0) ? cp0[pr] : 0.0;
                Wt[T][1] = (ok && cv1) ? cp1[pr] : 0.0;
            }
            for (int b = 0; b < nblocks; ++b) {
                const int st = (b >> 2) & 1, bb = b & 3;
                if (bb == 0) {
                    cp_async_wait<0>();
                    __syncthreads();
                    prep_round(st, 8 * b);
                    load_round((b >> 2) + 1);
                }
                const double* Ab = s_A + (size_t)((st * 4 + bb) * 8) * SR;
                mbar_wait(mbx, b & 1);
                const double2 x = *reinterpret_cast<const double2*>(xbuf + (b & 1) * 64 + 2 * lane);
                const double nb[2] = {x.x, x.y};
                dmma_acc(Wt[0][0], Wt[0][1], Ab[q * SR + 8 * HA + g], nb[0]);
                dmma_acc(Wt[0][0], Wt[0][1], Ab[(4 + q) * SR + 8 * HA + g], nb[1]);
                *reinterpret_cast<double2*>(tbuf + (b & 1) * 64 + 2 * lane) = make_double2(Wt[0][0], Wt[0][1]);
                mbar_arrive(mbt);
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                    for (int i = 1; i < HB; ++i)
                        dmma_acc(Wt[i][0], Wt[i][1], Ab[(4 * s2 + q) * SR + 8 * (HA + i) + g], nb[s2]);
#pragma unroll
                for (int i = 0; i < HB - 1; ++i) {
                    Wt[i][0] = Wt[i + 1][0];
                    Wt[i][1] = Wt[i + 1][1];
                }
                const double* in = s_in + (size_t)st * 32 * sin_ld + (8 * bb + g) * sin_ld + lc0;
                Wt[HB - 1][0] = in[0];
                Wt[HB - 1][1] = in[1];
            }
        }
    } else {
    // window: tile slot T <-> rows [8T, 8T+8) of the sweep, initially T = 0..NTW-1
        double Wt[NTW][2];
#pragma unroll
        for (int T = 0; T < NTW; ++T) {
            const int u = 8 * T + g;
            const bool ok = u < nsteps;
            const long long pr = ok ? phys(rowof(u)) : 0;
            Wt[T][0] = (ok && cv0) ? cp0[pr] : 0.0;
            Wt[T][1] = (ok && cv1) ? cp1[pr] : 0.0;
        }
    // The tile registers rotate by one slot per block, so Wt[0] is always the
        // pivot tile and Wt[i] holds rows [8i, 8i+8) past it: one loop body.
        const int nblocks = (nsteps + 7) / 8;
        for (int b = 0; b < nblocks; ++b) {
            const int st = (b >> 2) & 1, bb = b & 3;
            if (bb == 0) {
                cp_async_wait<0>();
                __syncthreads();
                prep_round(st, 8 * b);
                load_round((b >> 2) + 1);
            }
            const double* Ab = s_A + (size_t)((st * 4 + bb) * 8) * SR;
            const double* T = s_ti + (size_t)(st * 4 + bb) * 64;
            // P (C layout: row g, cols 2q..2q+1) -> B fragments: B[k][n] = P[4s+k][n]
            double pb[2];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int src = 4 * (4 * s2 + q) + (g >> 1);
                const double v0 = __shfl_sync(0xffffffffu, Wt[0][0], src);
                const double v1 = __shfl_sync(0xffffffffu, Wt[0][1], src);
                pb[s2] = (g & 1) ? v1 : v0;
            }
            // X = Tinv P : the 8 finished rows (C layout)
            double x0 = 0.0, x1 = 0.0;
            dmma_acc(x0, x1, T[g * 8 + q], pb[0]);
            dmma_acc(x0, x1, T[g * 8 + 4 + q], pb[1]);
            // X -> B fragments (negated)
            double nb[2];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int src = 4 * (4 * s2 + q) + (g >> 1);
                const double v0 = __shfl_sync(0xffffffffu, x0, src);
                const double v1 = __shfl_sync(0xffffffffu, x1, src);
                nb[s2] = -((g & 1) ? v1 : v0);
            }
            // rank-8 update: the next pivot tile first, then k-slice-major so the
            // two DMMAs of a tile are NTW-2 instructions apart
            dmma_acc(Wt[1][0], Wt[1][1], Ab[q * SR + 8 + g], nb[0]);
            dmma_acc(Wt[1][0], Wt[1][1], Ab[(4 + q) * SR + 8 + g], nb[1]);
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                for (int i = 2; i < NTW; ++i) dmma_acc(Wt[i][0], Wt[i][1], Ab[(4 * s2 + q) * SR + 8 * i + g], nb[s2]);
            {
                const int u = 8 * b + g;
                if (u < nsteps) {
                    const long long pr = phys(rowof(u));
                    if (cv0) cp0[pr] = x0;
                    if (cv1) cp1[pr] = x1;
                }
            }
            // rotate; the freed slot takes rows 8(b+NTW)+g
#pragma unroll
            for (int i = 0; i < NTW - 1; ++i) {
                Wt[i][0] = Wt[i + 1][0];
                Wt[i][1] = Wt[i + 1][1];
            }
            const double* in = s_in + (size_t)st * 32 * sin_ld + (8 * bb + g) * sin_ld + lc0;
            Wt[NTW - 1][0] = in[0];
            Wt[NTW - 1][1] = in[1];
        }
    }
    cp_async_wait<0>();
}

}  // namespace spk
