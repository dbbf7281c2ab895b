// spk_lu_piv_dmma.cu — blocked partial-pivoting band LU on the FP64 tensor
// cores, one CTA per SPIKE partition.
//
// Reference: LUFactors::factor, src/kernels.cpp:79-118, pivoting branch
// (gbtf2 semantics): for column j the pivot is the first row of maximal |a| in
// rows j..j+kl, rows j and ip are interchanged in columns j..j+ubw (ubw =
// kl+ku), the multipliers are a * (1/pivot) and the trailing kl x ubw window
// takes a rank-1 update; an exactly zero pivot column throws runtime_error
// (status 2 here).  The packed factor written is the reference's layout
// (kernels.cpp:29-42): L column j holds the multipliers as computed at step j
// (later interchanges are not applied to it), U row j the pivoted row.
//
// Blocked form (8 columns per step, right-looking, like LAPACK gbtrf).  The
// window of step J (columns j0 = 8J ..) is TRW x TCW tiles of 8 x 8: rows
// j0 .. j0+8TRW-1 (covers j0+7+kl) and columns j0 .. j0+8TCW-1 (covers
// j0+7+ubw).  Warp w owns one tile column, the column block J + co with
// co = (w - J) mod TCW, as TRW DMMA accumulator fragments; ownership rotates
// so registers never move between warps.
//   panel (co == 0): the 8TRW x 8 panel goes through shared memory into a
//     row-per-lane layout and is factored column by column: exact argmax by
//     redux.sync over the bits of |a| (hi word, then lo word) and the first
//     position by a min-redux; interchanges only swap the rows' position tags
//     (the rows stay in their lanes), the pivot row is shuffled to all lanes,
//     then multipliers and the rank-1 update of the panel.  Each L column goes
//     to HBM as computed (gbtf2 order); the pivots, L11 and -L21 in final
//     (getrf) order, DMMA A-fragment layout, are published.
//   update (co >= 1): the panel's row permutation on my tile column (through
//     a per-warp shared-memory scratch, only the moving rows), U12 = L11^-1 A12 by a 7-step forward
//     substitution, A22 -= L21 U12 by DMMA (2 per tile), then the window moves
//     down one tile row.  The entering row tile and the entering column block
//     are raw band values, staged in shared memory by cp.async one step ahead
//     (a global load merged into a register by a branch would stall the
//     critical warp for a full memory latency).
// The warp that holds the next panel (co == 1) factors it right after its own
// update, while the other warps are still updating: one CTA barrier per step,
// published data double-buffered by step parity.  The panel warp then takes
// the entering column block (raw band values; no earlier step touched it).
// Rows/columns past m continue as the identity (never selected as pivots).
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_piv_blocked.cuh"
#include "spk_sweep_fast.cuh"  // cp_async8 / commit / wait

#include <algorithm>

namespace spk {

__device__ __forceinline__ void pv_dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}
// A fragment (m x k, row-major): lane = m*4 + k%4, slice k/4
__device__ __forceinline__ int pv_afrag(int mm, int kk) { return (kk >> 2) * 32 + mm * 4 + (kk & 3); }

#ifdef SPK_PIV_PROFILE
// tools/piv_probe.cu: per-phase clock totals of the panel-critical warp of CTA 0
__device__ unsigned long long g_piv_prof[8];
#define PIV_MARK(slot)                                                              \
    do {                                                                            \
        if (blockIdx.x == 0 && lane == 0) {                                         \
            const long long now = clock64();                                       \
            atomicAdd(&g_piv_prof[(slot)], (unsigned long long)(now - tprev));     \
            tprev = now;                                                            \
        }                                                                           \
    } while (0)
#else
#define PIV_MARK(slot) \
    do {               \
    } while (0)
#endif

// Row-exchange scratch per warp: indexed by window position when it fits
// (one slot per row), packed otherwise (piv_xslot: tile 0 plus the <= 8 pivot
// rows outside it) -- the packed slots cost popcounts on every exchange.
template <int TRW, int TCW>
struct PivXs {
    static constexpr bool kFull = (size_t)TCW * 8 * TRW * 8 * 8 <= 96u * 1024;
    static constexpr int kRows = kFull ? 8 * TRW : 16;
};

// shared memory (doubles unless noted)
template <int TRW, int TCW>
struct PivDmmaSmem {
    static constexpr int PTLD = 9;            // panel transpose buffer row stride (bank-conflict free)
    static constexpr int RLD = 8 * TCW + 2;   // staged row tile stride
    double pt[8 * TRW * PTLD];
    double d11[2][64];        // rows 0..7 of the factored panel (L11 strictly below, U11), row-major
    double lbuf[2][8][8 * TRW];  // L columns of the panel in gbtf2 order (offsets 1..kl)
    int spiv[2][8];           // pivot positions of the panel
    double l21[2][TRW * 64];  // -L21 per tile row (tile 0 unused), A-fragment order
    double srow[2][8 * RLD];  // staged entering row tile of step J (rows 8(J+TRW).., window columns)
    double scol[2][8 * TRW * 8];  // staged entering column block for the panel warp of step J+1
    double xs[TCW][PivXs<TRW, TCW>::kRows * 8];  // per-warp row exchange scratch (PivXs)
    int src[2][8 * TRW];          // original position of the row at each final position
    unsigned mv_out[2][(8 * TRW + 31) / 32];  // rows leaving their position (by original position)
    unsigned mv_in[2][(8 * TRW + 31) / 32];   // positions receiving another row
    int sing[2];
};

// Scratch slot of window position pos for a panel's row exchange: tile 0 in
// slots 0..7, the (at most 8) pivot rows outside tile 0 packed after it in
// position order.  Outside tile 0 the rows leaving their position (mv_out)
// are exactly the positions receiving one (a pivot row goes to tile 0 and
// takes a tile-0 row), so one mask serves both directions.
template <int NW>
__device__ __forceinline__ int piv_xslot(const unsigned* mv_out, int pos) {
    if (pos < 8) return pos;
    int c = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const unsigned mk = w == 0 ? (mv_out[0] & ~0xffu) : mv_out[w];
        const int lo = 32 * w;
        if (pos >= lo + 32) c += __popc(mk);
        else if (pos > lo) c += __popc(mk & ((1u << (pos - lo)) - 1u));
    }
    return 8 + c;
}

template <int TRW, int TCW, bool DENSE>
__global__ void __launch_bounds__(32 * TCW, 1) k_band_lu_piv_dmma(PivDmmaArgs A) {
    constexpr int NSL = (8 * TRW + 31) / 32;  // row slots per lane in the panel layout
    extern __shared__ __align__(16) unsigned char piv_smem_raw[];
    PivDmmaSmem<TRW, TCW>& S = *reinterpret_cast<PivDmmaSmem<TRW, TCW>*>(piv_smem_raw);
    const int u = A.units[blockIdx.x];
    const PartDev P = A.parts[u];
    if (DENSE && P.guard >= 0 && !guard_ok(A.flags, P.guard)) return;
    const int m = P.m, kl = P.kl, ku = P.ku, ubw = P.ubw, d = P.d, rows = P.rows;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = lane >> 2, q = lane & 3;
    const unsigned full = 0xffffffffu;
    // dense coupling units read their band in place (fac, layout kernels.cpp:29-42)
    const int ald = DENSE ? rows : A.akl + A.aku + 1;
    double* F = A.fac + P.fofs;
    double* TF = A.tfac + P.tofs;
    const int rowsT = P.rowsT;
    int* piv = A.piv + P.r0;
    const int nblk = (m + 7) / 8;
    const double* bbase = DENSE ? A.fac + P.fofs + d
                                : A.band + (P.rev ? (long long)(P.r0 + m - 1) * ald + A.aku : (long long)P.r0 * ald + A.aku);
    const long long sg = P.rev ? -1 : 1;
    // LU-space entry of the raw band; rows/columns past m continue as the identity
    auto val = [&](int i, int c) -> double {
        if (i < m && c < m) {
            if (i - c > kl || c - i > ku) return 0.0;
            return bbase[sg * ((long long)c * (ald - 1) + i)];
        }
        return i == c ? 1.0 : 0.0;
    };

    // packed positions above row 0 (and row-major positions left of column 0)
    // that no step writes read as zero
    for (int idx = threadIdx.x; idx < ubw * ubw; idx += blockDim.x) {
        const int c = idx / ubw, off = idx - c * ubw + 1;
        if (c < m && off > c) F[(long long)c * rows + d - off] = 0.0;
    }
    for (int idx = threadIdx.x; idx < kl * kl; idx += blockDim.x) {
        const int r = idx / kl, off = idx - r * kl + 1;
        if (!DENSE && r < m && off > r) TF[(long long)r * rowsT + kl - off] = 0.0;
    }
    // row-major U slots right of column m - 1 and the partition's padding: no
    // step writes them, and the truncated U^T sweeps of the edge partitions
    // read them against zero right-hand-side rows -- they must be finite
    // whatever the block held before (found by the SPK_POISON runs of
    // tools/fuzz_parity.py: NaN from transposed pivoted solves)
    for (int idx = threadIdx.x; idx < ubw * ubw; idx += blockDim.x) {
        const int i = m - 1 - idx / ubw, off = idx % ubw + 1;
        if (!DENSE && i >= 0 && i + off >= m) TF[(long long)i * rowsT + kl + off] = 0.0;
    }
    if (!DENSE && threadIdx.x < 8) {
        const long long e = (long long)m * rowsT + threadIdx.x;
        if (e < ((long long)m * rowsT + 7) / 8 * 8) TF[e] = 0.0;
    }

    double acc[TRW][2];
    auto load_block = [&](int r0, int cb) {  // rows r0 .., column block cb (direct, start-up only)
#pragma unroll
        for (int t = 0; t < TRW; ++t) {
            acc[t][0] = val(r0 + 8 * t + gi, 8 * cb + 2 * q);
            acc[t][1] = val(r0 + 8 * t + gi, 8 * cb + 2 * q + 1);
        }
    };
    // Staging for step Jn (buffer Jn & 1), issued one step ahead by all threads:
    // the row tile entering at the shift of step Jn (rows 8(Jn+TRW) .., window
    // columns 8Jn ..) and the column block the panel warp of step Jn+1 takes
    // after its panel (block Jn+1+TCW, rows 8(Jn+2) ..).  Out-of-band slots
    // are stored as zeros, past-m slots as the identity; band values by cp.async.
    // (issued by the TCW-1 warps off the critical path: rank 0 .. TCW-2)
    auto stage = [&](int Jn, int rank) {
        const int b = Jn & 1;
        constexpr int NR = 8 * 8 * TCW, NC = 8 * TRW * 8;
        for (int idx = rank * 32 + lane; idx < NR + NC; idx += 32 * (TCW - 1)) {
            int i, c;
            double* dst;
            if (idx < NR) {
                const int cc = idx >> 3, rr = idx & 7;
                i = 8 * (Jn + TRW) + rr;
                c = 8 * Jn + cc;
                dst = &S.srow[b][rr * S.RLD + cc];
            } else {
                const int e = idx - NR, cc = e / (8 * TRW), rr = e - cc * 8 * TRW;
                i = 8 * (Jn + 2) + rr;
                c = 8 * (Jn + 1 + TCW) + cc;
                dst = &S.scol[b][rr * 8 + cc];
            }
            if (i < m && c < m) {
                if (i - c > kl || c - i > ku) *dst = 0.0;
                else cp_async8(dst, bbase + sg * ((long long)c * (ald - 1) + i));
            } else {
                *dst = i == c ? 1.0 : 0.0;
            }
        }
        cp_async_commit();
    };

    // Factor the panel of step Jp held in acc; publish into buffer Jp & 1.
    // Rows stay where they are (lane, slot); pos[] is the row's position after
    // the interchanges so far, so an interchange is two integer compares.
    auto panel = [&](int Jp, long long& tprev) {
        (void)tprev;
        const int par = Jp & 1, j0 = 8 * Jp;
#pragma unroll
        for (int t = 0; t < TRW; ++t) {
            S.pt[(8 * t + gi) * S.PTLD + 2 * q] = acc[t][0];
            S.pt[(8 * t + gi) * S.PTLD + 2 * q + 1] = acc[t][1];
        }
        __syncwarp();
        double pr[NSL][8];
        int pos[NSL];
#pragma unroll
        for (int s = 0; s < NSL; ++s) {
            const int r = lane + 32 * s;
            pos[s] = r < 8 * TRW ? r : 1 << 20;  // padding slots never take part
#pragma unroll
            for (int t = 0; t < 8; ++t) pr[s][t] = r < 8 * TRW ? S.pt[r * S.PTLD + t] : 0.0;
        }
        __syncwarp();  // the buffer is rewritten by the next panel warp only after a CTA barrier
        PIV_MARK(2);
        int sing = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            // exact argmax of |a(r, c)| over positions c .. c+kl, first position on ties
            double lb = 0.0;
#pragma unroll
            for (int s = 0; s < NSL; ++s) {
                const double a = fabs(pr[s][c]);
                if (pos[s] >= c && pos[s] <= c + kl && a > lb) lb = a;
            }
            const unsigned hi = (unsigned)__double2hiint(lb), lo = (unsigned)__double2loint(lb);
            const unsigned hmax = __reduce_max_sync(full, hi);
            const unsigned lmax = __reduce_max_sync(full, hi == hmax ? lo : 0u);
            const double gmax = __hiloint2double((int)hmax, (int)lmax);
            unsigned mypos = 0xffffffffu;
#pragma unroll
            for (int s = 0; s < NSL; ++s)
                if (pos[s] >= c && pos[s] <= c + kl && fabs(pr[s][c]) == gmax) mypos = min(mypos, (unsigned)pos[s]);
            const int p = (int)__reduce_min_sync(full, mypos);
            if (gmax == 0.0 && j0 + c < m) sing = 1;
            // pivot row (position p) to every lane
            const int holder = __ffs(__ballot_sync(full, mypos == (unsigned)p)) - 1;
            double vp[8];
#pragma unroll
            for (int t = c; t < 8; ++t) {
                double src = pr[0][t];
#pragma unroll
                for (int s = 1; s < NSL; ++s)
                    if (pos[s] == p) src = pr[s][t];
                vp[t] = __shfl_sync(full, src, holder);
            }
            // interchange positions c and p
#pragma unroll
            for (int s = 0; s < NSL; ++s) pos[s] = pos[s] == p ? c : (pos[s] == c ? p : pos[s]);
            // 1 / pivot: hardware estimate + two Newton steps
            double inv;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(vp[c]));
            {
                double e = fma(-vp[c], inv, 1.0);
                inv = fma(inv, e, inv);
                e = fma(-vp[c], inv, 1.0);
                inv = fma(inv, e, inv);
            }
#pragma unroll
            for (int s = 0; s < NSL; ++s) {
                if (pos[s] > c) {  // padding slots hold zeros
                    const double l = pr[s][c] * inv;
                    pr[s][c] = l;
#pragma unroll
                    for (int t = c + 1; t < 8; ++t) pr[s][t] = fma(-l, vp[t], pr[s][t]);
                }
            }
            // L column j0+c as computed at this step (gbtf2 order), to HBM after the publish
#pragma unroll
            for (int s = 0; s < NSL; ++s) {
                const int off = pos[s] - c;
                if (off >= 1 && off <= kl) S.lbuf[par][c][off] = pr[s][c];
            }
            if (lane == 0) S.spiv[par][c] = p;
        }
        PIV_MARK(3);
        // U11 rows, L11 / -L21 / pivots for the update, by final position
#pragma unroll
        for (int s = 0; s < NSL; ++s) {
            const int r = pos[s];
            if (r < 8) {
#pragma unroll
                for (int t = 0; t < 8; t += 2)
                    *reinterpret_cast<double2*>(&S.d11[par][r * 8 + t]) = make_double2(pr[s][t], pr[s][t + 1]);
            } else if (r < 8 * TRW) {
                const int tt = r >> 3, mm = r & 7;
#pragma unroll
                for (int t = 0; t < 8; ++t) S.l21[par][tt * 64 + pv_afrag(mm, t)] = -pr[s][t];
            }
        }
        // the row permutation of this panel: final position -> original position
#pragma unroll
        for (int s = 0; s < NSL; ++s)
            if (pos[s] < 8 * TRW) S.src[par][pos[s]] = lane + 32 * s;
#pragma unroll
        for (int s = 0; s < NSL; ++s) {
            const unsigned b = __ballot_sync(full, pos[s] < 8 * TRW && pos[s] != lane + 32 * s);
            if (lane == 0) S.mv_out[par][s] = b;
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < NSL; ++s) {
            const int f = lane + 32 * s;
            const unsigned b = __ballot_sync(full, f < 8 * TRW && S.src[par][f] != f);
            if (lane == 0) S.mv_in[par][s] = b;
        }
        if (lane == 0) S.sing[par] = sing;
        PIV_MARK(4);
    };

    double u12[2];
    auto write_u12 = [&](int J, int co) {
        const int i = 8 * J + gi;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = 8 * (J + co) + 2 * q + e, off = cc - i;
            if (i < m && off <= ubw) {
                if (cc < m) F[(long long)cc * rows + d - off] = u12[e];
                if (!DENSE) TF[(long long)i * rowsT + kl + off] = cc < m ? u12[e] : 0.0;
            }
        }
    };

    // update of step J on my tile column (column block J + co, co >= 1)
    auto update = [&](int J, int co, long long& tprev) {
        (void)tprev;
        const int par = J & 1, j0 = 8 * J;
        // the panel's row interchanges as one permutation through shared memory:
        // tile 0 and the rows leaving tiles >= 1 go out, every position that
        // receives another row reads it back (rows only move between tile 0 and
        // the pivot rows, so nothing else is touched)
        {
            double* xs = S.xs[w];
            constexpr int NW = (8 * TRW + 31) / 32;
            const unsigned* mvo = S.mv_out[par];
#pragma unroll
            for (int t = 0; t < TRW; ++t) {
                const unsigned mo = S.mv_out[par][(8 * t) >> 5];
                if (t == 0 || ((mo >> (((8 * t) & 31) + gi)) & 1u))
                    *reinterpret_cast<double2*>(
                        &xs[(PivXs<TRW, TCW>::kFull ? 8 * t + gi : piv_xslot<NW>(mvo, 8 * t + gi)) * 8 + 2 * q]) =
                        make_double2(acc[t][0], acc[t][1]);
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < TRW; ++t) {
                const unsigned mi = S.mv_in[par][(8 * t) >> 5];
                if (t == 0 || ((mi >> (((8 * t) & 31) + gi)) & 1u)) {
                    const int sl = PivXs<TRW, TCW>::kFull ? S.src[par][8 * t + gi]
                                                          : piv_xslot<NW>(mvo, S.src[par][8 * t + gi]);
                    const double2 v = *reinterpret_cast<const double2*>(&xs[sl * 8 + 2 * q]);
                    acc[t][0] = v.x;
                    acc[t][1] = v.y;
                }
            }
        }
        if (co == 1) PIV_MARK(0);
        // U12 = L11^-1 A12 (unit lower, forward substitution)
#pragma unroll
        for (int s = 0; s < 7; ++s) {
            const double v0 = __shfl_sync(full, acc[0][0], s * 4 + q);
            const double v1 = __shfl_sync(full, acc[0][1], s * 4 + q);
            const double l = gi > s ? S.d11[par][gi * 8 + s] : 0.0;
            acc[0][0] = fma(-l, v0, acc[0][0]);
            acc[0][1] = fma(-l, v1, acc[0][1]);
        }
        // U rows j0..j0+7 in my columns (the critical warp keeps them for later)
        u12[0] = acc[0][0];
        u12[1] = acc[0][1];
        if (co != 1) write_u12(J, co);
        // U12 as B fragments: B[k][n] = U12[k][n] sits in lane k*4 + n/2, register n&1
        double bf[2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int src = (q + 4 * ks) * 4 + (gi >> 1);
            const double v0 = __shfl_sync(full, acc[0][0], src);
            const double v1 = __shfl_sync(full, acc[0][1], src);
            bf[ks] = (gi & 1) ? v1 : v0;
        }
        if (co == 1) PIV_MARK(7);
        const double* L21 = S.l21[par];
        // k-slice-major: a tile's two DMMAs are TRW-1 instructions apart
#pragma unroll
        for (int t = 1; t < TRW; ++t) pv_dmma(acc[t][0], acc[t][1], L21[t * 64 + lane], bf[0]);
#pragma unroll
        for (int t = 1; t < TRW; ++t) pv_dmma(acc[t][0], acc[t][1], L21[t * 64 + 32 + lane], bf[1]);
        // the window moves down one tile row
#pragma unroll
        for (int t = 0; t + 1 < TRW; ++t) {
            acc[t][0] = acc[t + 1][0];
            acc[t][1] = acc[t + 1][1];
        }
        const double2 v = *reinterpret_cast<const double2*>(&S.srow[par][gi * S.RLD + 8 * co + 2 * q]);
        acc[TRW - 1][0] = v.x;
        acc[TRW - 1][1] = v.y;
    };

    // step 0: warp w holds column block w; warp 0 factors panel 0
    load_block(0, w);
    if (w != 1) stage(0, w == 0 ? 0 : w - 1);
    long long tprev = 0;
#ifdef SPK_PIV_PROFILE
    tprev = clock64();
#endif
    if (w == 0) {
        panel(0, tprev);
        load_block(8, TCW);
    }
    int co = w;
    for (int J = 0; J < nblk; ++J) {
        cp_async_wait<0>();  // staging of step J
        if (co == 1) PIV_MARK(1);
        __syncthreads();
        if (co == 1) PIV_MARK(6);
        if (S.sing[J & 1]) {
            if (threadIdx.x == 0) {
                if (DENSE && P.fallback) A.redo[u] = 2;  // k_band_lu_small redoes it (boosted fallback)
                else atomicMax(A.status, 2);
            }
            return;
        }
        if (co == 0) {
            // factor output of panel J (this warp factored it last step): L
            // columns, U11 and the pivots, and its U12 of step J-1
            const int par = J & 1, j0 = 8 * J;
            if (J > 0) write_u12(J - 1, 1);
            for (int c = 0; c < 8 && j0 + c < m; ++c)
                for (int off = 1 + lane; off <= kl; off += 32)
                    F[(long long)(j0 + c) * rows + d + off] = j0 + c + off < m ? S.lbuf[par][c][off] : 0.0;
            for (int e = lane; e < 64; e += 32) {
                const int r = e >> 3, t = e & 7;
                if (t >= r && t - r <= ubw && j0 + r < m) {
                    const double v = j0 + t < m ? S.d11[par][e] : 0.0;
                    if (j0 + t < m) F[(long long)(j0 + t) * rows + d - (t - r)] = v;
                    if (!DENSE) TF[(long long)(j0 + r) * rowsT + kl + t - r] = v;
                }
            }
            // row-major L: row j0+r takes columns j0+cc, cc < r, within kl (one run)
            for (int r = 1 + lane; !DENSE && r < 8 + kl && j0 + r < m; r += 32) {
                double* dst = TF + (long long)(j0 + r) * rowsT + kl - r;
                const int c0 = max(0, r - kl), c1 = min(7, r - 1);
                for (int cc = c0; cc <= c1; ++cc) dst[cc] = S.lbuf[par][cc][r - cc];
            }
            if (lane < 8 && j0 + lane < m) {
                piv[j0 + lane] = j0 + S.spiv[par][lane];
                if (!DENSE) A.dinv[P.r0 + j0 + lane] = 1.0 / S.d11[par][lane * 9];
            }
            if (!DENSE && A.lblk) {
                // the panel's blocked L record (spk_piv_blocked.cuh)
                using R = PivRec<TRW>;
                double* rec = A.lblk + (P.r0 / 8 + u + J) * (long long)R::SIZE;
                if (lane < 8) {  // column c = lane of L11^-1 by forward substitution
                    const int c = lane;
                    double y[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        double a = r == c ? 1.0 : 0.0;
#pragma unroll
                        for (int t = 0; t < r; ++t) a = fma(-S.d11[par][r * 8 + t], y[t], a);
                        y[r] = r < c ? 0.0 : a;
                    }
#pragma unroll
                    for (int r = 0; r < 8; ++r) rec[pv_afrag(r, c)] = y[r];
                }
                for (int e = 64 + lane; e < 64 * TRW; e += 32) rec[e] = S.l21[par][e];
                int* ri = reinterpret_cast<int*>(rec + R::SRC);
                for (int e = lane; e < 8 * TRW; e += 32) ri[e] = S.src[par][e];
                if (lane < R::NSLW) {
                    ri[8 * TRW + lane] = S.mv_out[par][lane];
                    ri[8 * TRW + R::NSLW + lane] = S.mv_in[par][lane];
                }
            }
            if (J + 1 < nblk) stage(J + 1, 0);
        } else {
            update(J, co, tprev);
            if (co != 1 && J + 1 < nblk) stage(J + 1, co - 1);
            if (co == 1) PIV_MARK(1);
            if (co == 1 && J + 1 < nblk) {
                panel(J + 1, tprev);
                // the entering column block of step J+2
                const int par = J & 1;
#pragma unroll
                for (int t = 0; t < TRW; ++t) {
                    const double2 v = *reinterpret_cast<const double2*>(&S.scol[par][(8 * t + gi) * 8 + 2 * q]);
                    acc[t][0] = v.x;
                    acc[t][1] = v.y;
                }
                PIV_MARK(5);
            }
        }
        co = co == 0 ? TCW - 1 : co - 1;
    }
    cp_async_wait<0>();
}

template <int TRW, int TCW, bool DENSE = false>
static bool launch_piv_dmma(int nunits, const PivDmmaArgs& A, cudaStream_t s) {
    const int smem = (int)sizeof(PivDmmaSmem<TRW, TCW>);
    if (smem > 227 * 1024) return false;
    set_smem_attr((const void*)k_band_lu_piv_dmma<TRW, TCW, DENSE>, (int)smem);
    k_band_lu_piv_dmma<TRW, TCW, DENSE><<<nunits, 32 * TCW, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_band_lu_piv_dmma(int nunits, int kl, int ku, const PivDmmaArgs& A, cudaStream_t s) {
    // the reversed (UL) partition swaps kl and ku: tile rows for the larger
    switch (piv_trw(kl, ku)) {
        case 5: return launch_piv_dmma<5, 9>(nunits, A, s);
        case 9: return launch_piv_dmma<9, 17>(nunits, A, s);
        case 13: return launch_piv_dmma<13, 25>(nunits, A, s);
        default: return false;
    }
}

// Coupling units: a dense 2k x 2k matrix stored as a band with kl = ku = 2k-1
// (kernels.cpp:67-77) is the window itself (8 TRW = 8 TCW >= 2k rows and
// columns; everything past m is identity padding, so no entering blocks are
// read), factored in place.
bool launch_dense_lu_piv_dmma(int nunits, int max_m, const PivDmmaArgs& A, cudaStream_t s) {
    if (nunits <= 0) return true;
    if (max_m <= 64) return launch_piv_dmma<8, 8, true>(nunits, A, s);
    if (max_m <= 128) return launch_piv_dmma<16, 16, true>(nunits, A, s);
    return false;
}

}  // namespace spk
