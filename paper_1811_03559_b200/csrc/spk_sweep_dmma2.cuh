// spk_sweep_dmma2.cuh — blocked triangular sweeps on the FP64 tensor cores,
// producer/consumer version.  Exec::run_fast_sweep picks it over k_sweep_dmma
// (spk_sweep_dmma.cuh) when it needs no extra column groups and has >= 6
// compute warps: C3's sweeps 48 -> 41 ms; SPK_SWEEP_V1=1 forces the other.
//
// Same jobs, semantics and 8-row blocking as k_sweep_dmma: each compute warp
// owns 8 right-hand-side columns and keeps the active band window as NTW 8x8
// accumulator tiles; per block, X = M^-1 P for the 8x8 diagonal block M of the
// triangular factor, then the rank-8 update W_i -= A_i X (two DMMA per tile).
// What changes is everything around the DMMAs:
//   * two producer warps stream the factor vectors (32 rows per stage, ring of
//     NST stages, conflict-free [step][row] layout) with cp.async and publish
//     each stage through an mbarrier; compute warps release stages through a
//     second mbarrier -- no CTA-wide barrier inside the sweep, so warps drift
//     apart and keep the tensor pipe fed (k_sweep_dmma synchronised every 32
//     rows and formed the diagonal-block inverses on one warp meanwhile);
//   * the producers also form the stage's diagonal-block inverses (off the
//     compute warps' path), so a block is X = Tinv P (2 DMMA) + the update;
//   * right-hand-side rows entering the window come through a per-warp
//     shared-memory ring filled by cp.async kDmma2Ring blocks ahead (each lane
//     copies and later reads its own two entries: no synchronisation beyond
//     cp.async.wait_group).  A register queue filled by plain loads stalled
//     the warp at the top of every block -- ptxas reuses the load's target
//     register and moves the value out at once, which waits for the load
//     (ncu: 11% of the kernel's samples on that move, long scoreboard).
// Out-of-band stage slots are zeroed once and never loaded; rows past the sweep
// end are masked in the consumer (their window rows are never stored).
#pragma once

#include "spk_device.cuh"
#include "spk_sweep_fast.cuh"

namespace spk {

__device__ __forceinline__ void dmma2_acc(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

constexpr int kDmma2Producers = 2;  // producer warps per CTA
constexpr int kDmma2Stages = 3;     // factor stages in flight
constexpr int kDmma2Ring = 6;       // right-hand-side ring depth per compute warp, blocks (512 B each)

template <int NTW>
struct Dmma2Geom {
    static constexpr int KWT = 8 * (NTW - 1);                  // longest factor vector
    static constexpr int SR = ((8 + KWT + 15) / 16) * 16 + 4;  // [step][row] stride, = 4 mod 16
    static constexpr int STAGE = 32 * SR + 32 + 4 * 64;        // 32 steps x SR rows + 32 x 1/u + 4 inverses
};

// pair mode: + per pair two X buffers, two tile buffers and two mbarriers
inline size_t dmma2_sweep_smem(int ntw, int ncw = 0, bool pair = false) {
    const int KWT = 8 * (ntw - 1);
    const int SR = ((8 + KWT + 15) / 16) * 16 + 4;
    return (size_t)kDmma2Stages * (32 * SR + 32 + 4 * 64) * 8 + 2 * kDmma2Stages * 8 + 16 +
           (pair ? (size_t)(ncw / 2) * (4 * 64 * 8 + 16) : (size_t)ncw * kDmma2Ring * 512);
}

// PAIR (narrow solves, <= 8 right-hand sides): two compute warps share the 8
// columns and split the window: warp A holds tiles 0 .. HA-1 and forms X, warp
// B holds tiles HA .. NTW-1 and the incoming rows.  Per block A publishes -X
// through shared memory and an mbarrier, and B publishes the tile leaving its
// front, which A takes one block later.  A single warp issues a DMMA at most
// every ~32 cycles (profiles/r01_dmma_occupancy.txt): with one column group
// the per-block issue of one warp (2 NTW DMMAs) set the pace; split, each warp
// issues about half.  (For wide solves the pairing measured slower.)
template <int NTW, int MODE, bool PAIR = false>
__global__ void __launch_bounds__(512) k_sweep_dmma2(FastSweepArgs A) {
    constexpr int SR = Dmma2Geom<NTW>::SR;
    constexpr int KWT = Dmma2Geom<NTW>::KWT;
    constexpr int STG = Dmma2Geom<NTW>::STAGE;
    constexpr int NST = kDmma2Stages;
    constexpr bool kAsc = (MODE == SW_FWD_L || MODE == SW_FWD_UT);
    constexpr bool kDiag = (MODE == SW_BWD_U || MODE == SW_FWD_UT);
    constexpr int kV = kAsc ? 1 : -1;  // factor vectors run forward (L columns, U rows) or backward
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_st = reinterpret_cast<double*>(smem_raw);  // [NST][32 steps][SR rows] + [32] 1/u
    unsigned long long* full = reinterpret_cast<unsigned long long*>(s_st + NST * STG);
    unsigned long long* empty = full + NST;

    const SweepJob J = A.jobs[blockIdx.x];
    if (!guard_ok(A.B.flags, J.guard)) return;
    const PartDev P = A.parts[J.part];
    const int nc_total = J.nc >= 0 ? J.nc : A.ncols;
    const int ncw = (blockDim.x >> 5) - kDmma2Producers;  // compute warps
    const int ncta = (PAIR ? ncw / 2 : ncw) * 8;
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
    if (MODE == SW_FWD_L) {
        kw = P.kl;
        vbase = A.fac + P.fofs + P.d + 1;
        vstride = P.rows;
    } else if (MODE == SW_BWD_U) {
        kw = P.ubw;
        vbase = A.fac + P.fofs + P.d - 1;
        vstride = P.rows;
    } else if (MODE == SW_FWD_UT) {
        kw = P.ubw;
        vbase = A.tfac + P.tofs + P.kl + 1;
        vstride = P.rowsT;
    } else {
        kw = P.kl;
        vbase = A.tfac + P.tofs + P.kl - 1;
        vstride = P.rowsT;
    }
    auto rowof = [&](int u) -> int { return kAsc ? lo + u : hi - u; };
    const int nrounds = (nsteps + 31) / 32;

    // stage slot (step t of the round, row r) holds v_{32R + t}[r - (t & 7) - 1]
    // (zero outside 0 <= r - (t&7) - 1 < kw: a fixed set of slots, never loaded)
    for (int idx = threadIdx.x; idx < NST * STG; idx += blockDim.x) s_st[idx] = 0.0;
    if (threadIdx.x < NST) {
        mbar_init(full + threadIdx.x, kDmma2Producers * 32);  // producers arrive after forming the inverses
        mbar_init(empty + threadIdx.x, ncw);
    }
    // pair handshakes (PAIR): per pair, X ready (A -> B) and front tile ready (B -> A)
    unsigned long long* pbar = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<double*>(empty + NST) + (size_t)(ncw / 2) * 4 * 64);
    if (PAIR && threadIdx.x < ncw) mbar_init(pbar + threadIdx.x, 32);
    __syncthreads();

    if (warp >= ncw) {
        // ---- producers: round R -> stage R % NST, loads issued two rounds ahead
        const int pt = threadIdx.x - ncw * 32, npt = blockDim.x - ncw * 32;  // (run-time on purpose: see DESIGN 4)
        auto issue = [&](int R) {
            if (R < nrounds) {
                const int s = R % NST;
                if (R >= NST) mbar_wait(empty + s, ((R / NST) - 1) & 1);
                double* st = s_st + s * STG;
                const int u0 = 32 * R;
                // thread pt copies entries dl = pt, pt + npt, ... of each of the
                // round's 32 vectors: the source steps by one factor vector per
                // t and the slot offsets are compile-time (t unrolled), a few
                // instructions per entry.  (One flat loop over the stage with a
                // division per entry made a producer as busy as a compute warp.)
                const int nv = min(32, nsteps - u0);
                const double* src = vbase + (long long)rowof(u0) * vstride + kV * pt;
                const long long sstep = kAsc ? vstride : -vstride;
                double* dst = st + pt + 1;
#pragma unroll 8
                for (int t = 0; t < 32; ++t) {
                    if (t < nv) {
                        for (int dl = pt, o = 0; dl < kw; dl += npt, o += npt)
                            cp_async8(dst + t * SR + (t & 7) + o, src + kV * o);
                    }
                    src += sstep;
                }
                if (kDiag && pt < 32 && u0 + pt < nsteps)
                    cp_async8(st + 32 * SR + pt, A.dinv + P.r0 + rowof(u0 + pt));
            }
            cp_async_commit();
        };
        issue(0);
        issue(1);
        for (int R = 0; R < nrounds; ++R) {
            const int s = R % NST, u0 = 32 * R;
            double* st = s_st + s * STG;
            cp_async_wait<1>();  // round R has landed (R+1 may still be in flight)
            asm volatile("bar.sync 1, %0;\n" ::"r"(npt) : "memory");  // producers see each other's data
            // the round's 4 diagonal-block inverses Tinv = M^-1: thread (bb, c)
            // solves M y = e_c by forward substitution (M unit, or u_tt on the
            // diagonal for the U sweeps); rows past the sweep end give 0
            if (pt < 32) {
                const int bb = pt >> 3, c = pt & 7;
                const double* Ab = st + (size_t)(8 * bb) * SR;
                double y[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    double a = (r == c) ? 1.0 : 0.0;
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        if (t < r) a -= Ab[t * SR + r] * y[t];
                    y[r] = kDiag ? a * st[32 * SR + 8 * bb + r] : a;
                    if (u0 + 8 * bb + r >= nsteps) y[r] = 0.0;
                }
                double* Ti = st + 32 * SR + 32 + bb * 64;
#pragma unroll
                for (int r = 0; r < 8; ++r) Ti[r * 8 + c] = y[r];  // Tinv[r][c]
            }
            mbar_arrive(full + s);
            issue(R + 2);
        }
        cp_async_wait<0>();
        return;
    }

    // ---- compute warps
    if constexpr (PAIR) {
        constexpr int HA = (NTW + 1) / 2, HB = NTW - HA;
        constexpr int LAP = 4;  // right-hand-side lookahead of warp B, blocks
        const int g = lane >> 2, q = lane & 3;
        const int pr_ = warp >> 1, role = warp & 1;
        double* pbuf = reinterpret_cast<double*>(empty + NST) + (size_t)pr_ * 4 * 64;
        double* xbuf = pbuf;         // [2][64]: -X as B fragments (A -> B)
        double* tbuf = pbuf + 128;   // [2][64]: B's front tile after its update (B -> A)
        unsigned long long* mbx = pbar + 2 * pr_;
        unsigned long long* mbt = mbx + 1;
        const View& v = J.v;
        const long long ld = v.ld >= 0 ? v.ld : A.B.ld[v.buf];
        double* const bbase = A.B.p[v.buf] + v.base;
        auto phys = [&](int r) -> long long {
            return v.rev ? (long long)(v.mrows - 1 - (r - v.off)) : (long long)(r - v.off);
        };
        const int c0 = J.c0 + colbase;
        const int ncta_valid = min(ncta, nc_total - colbase);
        const int lc0 = pr_ * 8 + 2 * q;
        const bool cv0 = lc0 < ncta_valid, cv1 = lc0 + 1 < ncta_valid;
        double* const cp0 = bbase + (long long)(c0 + (cv0 ? lc0 : 0)) * ld;
        double* const cp1 = bbase + (long long)(c0 + (cv1 ? lc0 + 1 : 0)) * ld;
        auto rhs = [&](int u, double& a, double& b) {
            const bool ok = u < nsteps;
            const long long pr = ok ? phys(rowof(u)) : 0;
            a = (ok && cv0) ? cp0[pr] : 0.0;
            b = (ok && cv1) ? cp1[pr] : 0.0;
        };
        const int nblocks = (nsteps + 7) / 8;
        if (role == 0) {
            // ---- warp A: window tiles 0 .. HA-1
            double Wt[HA][2];
#pragma unroll
            for (int T = 0; T < HA; ++T) rhs(8 * T + g, Wt[T][0], Wt[T][1]);
            for (int b = 0; b < nblocks; ++b) {
                const int R = b >> 2, bb = b & 3, s = R % NST;
                if (bb == 0) mbar_wait(full + s, (R / NST) & 1);
                const double* Ab = s_st + s * STG + (size_t)(8 * bb) * SR;
                const int u0 = 8 * b;
                double p0 = 0.0, p1 = 0.0;
                {
                    const double* T = s_st + s * STG + 32 * SR + 32 + bb * 64;
                    double pb[2];
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        const int src = 4 * (4 * s2 + q) + (g >> 1);
                        const double v0 = __shfl_sync(0xffffffffu, Wt[0][0], src);
                        const double v1 = __shfl_sync(0xffffffffu, Wt[0][1], src);
                        pb[s2] = (g & 1) ? v1 : v0;
                    }
                    dmma2_acc(p0, p1, T[g * 8 + q], pb[0]);
                    dmma2_acc(p0, p1, T[g * 8 + 4 + q], pb[1]);
                }
                double nb[2];
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const int src = 4 * (4 * s2 + q) + (g >> 1);
                    const double v0 = __shfl_sync(0xffffffffu, p0, src);
                    const double v1 = __shfl_sync(0xffffffffu, p1, src);
                    nb[s2] = -((g & 1) ? v1 : v0);
                }
                *reinterpret_cast<double2*>(xbuf + (b & 1) * 64 + 2 * lane) = make_double2(nb[0], nb[1]);
                // B has consumed X of block b-1 (and published its front tile)
                // before X of block b is announced: one phase apart at most
                if (b > 0) mbar_wait(mbt, (b - 1) & 1);
                mbar_arrive(mbx);
                if (b > 0) {  // my last tile is B's front tile of the previous block
                    const double2 t = *reinterpret_cast<const double2*>(tbuf + ((b - 1) & 1) * 64 + 2 * lane);
                    Wt[HA - 1][0] = t.x;
                    Wt[HA - 1][1] = t.y;
                }
                {
                    const int u = u0 + g;
                    if (u < nsteps) {
                        const long long pr = phys(rowof(u));
                        if (cv0) cp0[pr] = p0;
                        if (cv1) cp1[pr] = p1;
                    }
                }
                dmma2_acc(Wt[1][0], Wt[1][1], Ab[q * SR + 8 + g], nb[0]);
                dmma2_acc(Wt[1][0], Wt[1][1], Ab[(4 + q) * SR + 8 + g], nb[1]);
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                    for (int i = 2; i < HA; ++i) dmma2_acc(Wt[i][0], Wt[i][1], Ab[(4 * s2 + q) * SR + 8 * i + g], nb[s2]);
                if (bb == 3 || b == nblocks - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + s);
                }
#pragma unroll
                for (int i = 0; i < HA - 1; ++i) {
                    Wt[i][0] = Wt[i + 1][0];
                    Wt[i][1] = Wt[i + 1][1];
                }
            }
        } else {
            // ---- warp B: window tiles HA .. NTW-1 and the incoming rows
            double Wt[HB][2];
#pragma unroll
            for (int T = 0; T < HB; ++T) rhs(8 * (HA + T) + g, Wt[T][0], Wt[T][1]);
            double qv[LAP][2];
#pragma unroll
            for (int j = 0; j < LAP; ++j) rhs(8 * (NTW + j) + g, qv[j][0], qv[j][1]);
            for (int b = 0; b < nblocks; ++b) {
                const int R = b >> 2, bb = b & 3, s = R % NST;
                if (bb == 0) mbar_wait(full + s, (R / NST) & 1);
                const double* Ab = s_st + s * STG + (size_t)(8 * bb) * SR;
                mbar_wait(mbx, b & 1);
                const double2 x = *reinterpret_cast<const double2*>(xbuf + (b & 1) * 64 + 2 * lane);
                const double nb[2] = {x.x, x.y};
                // the front tile first: A takes it next block
                dmma2_acc(Wt[0][0], Wt[0][1], Ab[q * SR + 8 * HA + g], nb[0]);
                dmma2_acc(Wt[0][0], Wt[0][1], Ab[(4 + q) * SR + 8 * HA + g], nb[1]);
                *reinterpret_cast<double2*>(tbuf + (b & 1) * 64 + 2 * lane) = make_double2(Wt[0][0], Wt[0][1]);
                mbar_arrive(mbt);
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                    for (int i = 1; i < HB; ++i)
                        dmma2_acc(Wt[i][0], Wt[i][1], Ab[(4 * s2 + q) * SR + 8 * (HA + i) + g], nb[s2]);
                if (bb == 3 || b == nblocks - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + s);
                }
#pragma unroll
                for (int i = 0; i < HB - 1; ++i) {
                    Wt[i][0] = Wt[i + 1][0];
                    Wt[i][1] = Wt[i + 1][1];
                }
                Wt[HB - 1][0] = qv[0][0];
                Wt[HB - 1][1] = qv[0][1];
#pragma unroll
                for (int j = 0; j + 1 < LAP; ++j) {
                    qv[j][0] = qv[j + 1][0];
                    qv[j][1] = qv[j + 1][1];
                }
                rhs(8 * (b + 1 + NTW + LAP - 1) + g, qv[LAP - 1][0], qv[LAP - 1][1]);
                {
                    constexpr int PF = 8;
                    const int u = 8 * (b + 1 + NTW + LAP - 1 + PF) + g;
                    if (u < nsteps) {
                        const long long pr = phys(rowof(u));
                        if (cv0) asm volatile("prefetch.global.L2 [%0];" ::"l"(cp0 + pr));
                        if (cv1) asm volatile("prefetch.global.L2 [%0];" ::"l"(cp1 + pr));
                    }
                }
            }
        }
        return;
    } else {
    const int g = lane >> 2, q = lane & 3;
    const View& v = J.v;
    const long long ld = v.ld >= 0 ? v.ld : A.B.ld[v.buf];
    double* const bbase = A.B.p[v.buf] + v.base;
    auto phys = [&](int r) -> long long {
        return v.rev ? (long long)(v.mrows - 1 - (r - v.off)) : (long long)(r - v.off);
    };
    const int c0 = J.c0 + colbase;
    const int ncta_valid = min(ncta, nc_total - colbase);
    const int lc0 = warp * 8 + 2 * q;  // this lane's two columns (CTA-local)
    const bool cv0 = lc0 < ncta_valid, cv1 = lc0 + 1 < ncta_valid;
    double* const cp0 = bbase + (long long)(c0 + (cv0 ? lc0 : 0)) * ld;
    double* const cp1 = bbase + (long long)(c0 + (cv1 ? lc0 + 1 : 0)) * ld;
    auto rhs = [&](int u, double& a, double& b) {
        const bool ok = u < nsteps;
        const long long pr = ok ? phys(rowof(u)) : 0;
        a = (ok && cv0) ? cp0[pr] : 0.0;
        b = (ok && cv1) ? cp1[pr] : 0.0;
    };

    // window: tile slot i <-> rows [8(b+i), 8(b+i)+8) of the sweep at block b
    double Wt[NTW][2];
#pragma unroll
    for (int T = 0; T < NTW; ++T) rhs(8 * T + g, Wt[T][0], Wt[T][1]);
    // incoming rows: ring slot j holds this lane's two entries of a block
    // (slot layout [2 columns][32 lanes]: the 8-byte copies of a warp fall on distinct banks)
    double* const ring = reinterpret_cast<double*>(empty + NST) + (size_t)warp * (kDmma2Ring * 64) + lane;
    auto fetch = [&](int blk, int slot) {  // rows 8 blk + g -> slot (zero past the sweep / the columns)
        const int u = 8 * blk + g;
        double* dst = ring + slot * 64;
        const bool ok = u < nsteps;
        const long long pr = ok ? phys(rowof(u)) : 0;
        if (ok && cv0) cp_async8(dst, cp0 + pr);
        else dst[0] = 0.0;
        if (ok && cv1) cp_async8(dst + 32, cp1 + pr);
        else dst[32] = 0.0;
        cp_async_commit();
    };
#pragma unroll
    for (int j = 0; j < kDmma2Ring; ++j) fetch(NTW + j, j);
    int rslot = 0;

    const int nblocks = (nsteps + 7) / 8;
    for (int b = 0; b < nblocks; ++b) {
        const int R = b >> 2, bb = b & 3, s = R % NST;
        if (bb == 0) mbar_wait(full + s, (R / NST) & 1);
        const double* Ab = s_st + s * STG + (size_t)(8 * bb) * SR;
        const int u0 = 8 * b;
        // X = Tinv P (Tinv formed by the producers): P -> B fragments, 2 DMMA
        double p0 = 0.0, p1 = 0.0;
        {
            const double* T = s_st + s * STG + 32 * SR + 32 + bb * 64;
            double pb[2];
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int src = 4 * (4 * s2 + q) + (g >> 1);
                const double v0 = __shfl_sync(0xffffffffu, Wt[0][0], src);
                const double v1 = __shfl_sync(0xffffffffu, Wt[0][1], src);
                pb[s2] = (g & 1) ? v1 : v0;
            }
            dmma2_acc(p0, p1, T[g * 8 + q], pb[0]);
            dmma2_acc(p0, p1, T[g * 8 + 4 + q], pb[1]);
        }
        {
            const int u = u0 + g;
            if (u < nsteps) {
                const long long pr = phys(rowof(u));
                if (cv0) cp0[pr] = p0;
                if (cv1) cp1[pr] = p1;
            }
        }
        // X -> B fragments (negated): B[k][n] = X[4 s2 + k][n]
        double nb[2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int src = 4 * (4 * s2 + q) + (g >> 1);
            const double v0 = __shfl_sync(0xffffffffu, p0, src);
            const double v1 = __shfl_sync(0xffffffffu, p1, src);
            nb[s2] = -((g & 1) ? v1 : v0);
        }
        // rank-8 update: the next pivot tile first, then k-slice-major
        dmma2_acc(Wt[1][0], Wt[1][1], Ab[q * SR + 8 + g], nb[0]);
        dmma2_acc(Wt[1][0], Wt[1][1], Ab[(4 + q) * SR + 8 + g], nb[1]);
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int i = 2; i < NTW; ++i) dmma2_acc(Wt[i][0], Wt[i][1], Ab[(4 * s2 + q) * SR + 8 * i + g], nb[s2]);
        if (bb == 3 || b == nblocks - 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        // rotate; the freed slot takes rows 8(b+NTW)+g from the ring, whose
        // slot is refilled kDmma2Ring blocks ahead
#pragma unroll
        for (int i = 0; i < NTW - 1; ++i) {
            Wt[i][0] = Wt[i + 1][0];
            Wt[i][1] = Wt[i + 1][1];
        }
        cp_async_wait<kDmma2Ring - 1>();
        {
            Wt[NTW - 1][0] = ring[rslot * 64];
            Wt[NTW - 1][1] = ring[rslot * 64 + 32];
        }
        fetch(b + NTW + kDmma2Ring, rslot);
        rslot = rslot + 1 == kDmma2Ring ? 0 : rslot + 1;
    }
    cp_async_wait<0>();
    }
}

}  // namespace spk
