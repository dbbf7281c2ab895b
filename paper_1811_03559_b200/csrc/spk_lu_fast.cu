// spk_lu_fast.cu — blocked band LU (non-pivoting, diagonal boosting) for SPIKE
// partitions on the FP64 tensor cores, one CTA per partition.
//
// Reference: LUFactors::factor, src/kernels.cpp:79-118 (+ the packed copy of
// :29-65, done here on the fly from the input band, reversed for the UL
// partition).  Same arithmetic: multipliers l = a * (1/u_jj), rank-1 update
// of the kl x ku trailing window per column step, boost |u_jj| < eps*max|A_i|
// to +-boost_eps*max|A_i|.
//
// The kernel (k_band_lu_dmma below) is blocked 8 columns per step on the FP64
// tensor cores.  Factors are written in both layouts the sweeps use
// (column-major packed LU and the row-major copy) plus 1/u_jj.  Boosting is
// decided optimistically: the CTA tracks max|A_i| and min|u_jj| on the fly
// and, if a boost would have fired, re-runs its partition with the now-known
// threshold (exact reference semantics; never taken for diagonally dominant
// input).
#include <cuda.h>

#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_sweep_fast.cuh"

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cstring>

namespace spk {


// ===========================================================================
// Blocked variant on the FP64 tensor cores (kl, ku <= 128).
//
// Same factorization, 8 columns per step instead of 1.  The active window is
// the 8 x 8 tiles of the rows and columns within the band of the current
// 8-column panel: T = 8-blocks of max(kl, ku) + 1 column offsets and T-1 tile
// rows below the panel, held in DMMA accumulator fragments, one warp per tile
// row, indexed by column offset from the panel (registers rotate one tile per
// step).  Step J (columns 8J .. 8J+7):
//   1a. L21 = A21 U11^-1 for each tile row (DMMA with the inverse of the
//       factored 8 x 8 diagonal block);
//   1b. U12 = L11^-1 (A12 - L21' U12') per column offset: the panel row was
//       published before its last (primed) rank-8 update, applied here;
//   2.  the warp of the row right below the panel publishes its far tile, then
//       updates the next diagonal tile and factors it (shuffles: LU with the
//       boosting rule, L11^-1 and U11^-T in lockstep); every other warp applies
//       the rank-8 update A22 -= L21 U12 (DMMA), shifts its row by one tile and
//       takes the entering column block (cp.async staging, triple-buffered),
//       the warp two rows below publishes its row as the panel row of step J+2,
//       and the warp that took the entering row block last step reads it from
//       staging inside its update; then the step's L columns / U rows go out in
//       both packed layouts.
// Tiles outside the band are exact zeros throughout, so no band tests sit in
// the update.  Two CTA barriers per 8 columns (the register-window kernel above
// needs one per column).  Multipliers equal the unblocked ones up to rounding
// (l = a u_jj^-1 through the block inverse); boosting is decided exactly as
// above (optimistic pass, re-run with the known threshold).  tools/lu_probe.cu
// times the phases (the diagonal chain, latency-bound, sets the step time).
__device__ __forceinline__ void lu_dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

template <int T, int TR>
struct LuDmmaSmem {  // offsets in doubles (from a 128-byte aligned base)
    static constexpr int NW = T - 1;
    static constexpr int D = 0;                  // [2][64] factored diagonal block, row-major
    static constexpr int DINV = D + 128;         // [2][8]  1/u_jj
    static constexpr int LI = DINV + 16;         // [2][64] L11^-1, A-fragment order
    static constexpr int UI = LI + 128;          // [2][64] U11^-1, B-fragment order
    static constexpr int PROW = UI + 128;        // [2][T][64] panel row of step J (parity J), accumulator order
    static constexpr int L = PROW + 2 * 64 * T;  // [2][T][64] -L21 by row offset, A-fragment order
    static constexpr int U = L + 2 * 64 * T;     // [2][T][64] U12 by column offset, B-fragment order
    // staging of the entering blocks, in the TMA box layouts (column-major,
    // padded strides: conflict-free fragment reads; both 128-byte aligned):
    // column block [8 columns][SC rows], row block [8T columns][SR rows]
    static constexpr int SC = 8 * T + 2, SR = 10;
    static constexpr int CB = 8 * SC, RB = 8 * T * SR;
    static constexpr int ST = U + 2 * 64 * T;    // [2][CB] column blocks, then [2][RB] row blocks
    static constexpr int NS = T - TR;            // column offsets held in shared memory per tile row
    static constexpr int WIN = ST + 2 * CB + 2 * RB;  // [NW][NS][32] double2, circular by step
    static constexpr int TOTAL = WIN + NW * NS * 64;
    static_assert(ST % 16 == 0 && CB % 16 == 0 && RB % 16 == 0, "TMA destinations must stay 128-byte aligned");
};

// TMA tile load (2-D tensor map) into shared memory, completion on an mbarrier
__device__ __forceinline__ void lu_tma_2d(void* dst, const CUtensorMap* tm, int x, int y, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
        "l"(tm), "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}
__device__ __forceinline__ void lu_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}

#if defined(SPK_LU_PROFILE) || defined(SPK_LU_DBG)
// tools/lu_probe.cu (timing experiments, wrong results): bit 0 no column TMA,
// 1 no row TMA, 2 no zeroing, 3 no TMA waits, 4 no TMA arming, 5 no outputs,
// 6 no diagonal factorization, 7 no trailing update
__device__ int g_lu_dbg;
#define LU_DBG(bit) (g_lu_dbg & (bit))
#else
#define LU_DBG(bit) 0
#endif
#ifdef SPK_LU_PROFILE
// tools/lu_probe.cu: per-phase clock totals of CTA 0 (lane 0 of each warp)
__device__ unsigned long long g_lu_prof[8];
__device__ volatile int* g_lu_where;  // mapped host memory: last (step, mark) per warp
#define LU_MARK(slot)                                                          \
    do {                                                                       \
        if (g_lu_where && lane == 0) g_lu_where[blockIdx.x * 32 + w] = J * 16 + (slot); \
        if (blockIdx.x == 0 && lane == 0) {                                    \
            const long long now = clock64();                                  \
            atomicAdd(&g_lu_prof[(slot)], (unsigned long long)(now - tprev)); \
            tprev = now;                                                       \
        }                                                                      \
    } while (0)
#else
#define LU_MARK(slot) \
    do {              \
    } while (0)
#endif

// fragment orders: A (m x k, row-major): lane = m*4 + k%4, slice k/4;
// B (k x n): lane = n*4 + k%4, slice k/4 -- one conflict-free 8-byte access each
__device__ __forceinline__ int afrag(int m, int k) { return (k >> 2) * 32 + m * 4 + (k & 3); }
__device__ __forceinline__ int bfrag(int k, int n) { return (k >> 2) * 32 + n * 4 + (k & 3); }

// Column offsets < TR of a tile row live in registers; offsets TR..T-1 in a
// per-warp circular shared-memory window (slot (J + o - TR) mod (T-TR) at step
// J), so the per-step rotation moves one tile in and one out.  T = 21 (k <=
// 160) needs it: 20 warps leave 96 registers per thread.
template <int T, int TR>
__global__ void __launch_bounds__(32 * (T - 1), T <= 13 ? 2 : 1) k_band_lu_dmma(FastLuArgs A, const __grid_constant__ CUtensorMap tmc,
                                                                           const __grid_constant__ CUtensorMap tmr,
                                                                           int tma_sh) {
    using S = LuDmmaSmem<T, TR>;
    constexpr int NS = T - TR;
    constexpr int NW = T - 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // 128-byte aligned base (TMA destinations).  The pad is computed from the
    // shared-window offset and added to the array itself: rounding the generic
    // address through an integer hid the address space from the compiler, and
    // every shared access of the kernel became a generic LD/ST (64-bit address
    // arithmetic, long-scoreboard latency; ncu: 17% of the stall samples)
    const unsigned sm_off = static_cast<unsigned>(__cvta_generic_to_shared(smem_raw));
    double* sm = reinterpret_cast<double*>(smem_raw + ((128u - (sm_off & 127u)) & 127u));
    __shared__ unsigned long long s_mb[2];  // TMA staging barriers, by issuing-step parity
    __shared__ double s_red[2 * 32];
    __shared__ int s_cnt[32];

    const int u = A.units[blockIdx.x];
    const PartDev P = A.parts[u];
    const int m = P.m, kl = P.kl, ku = P.ku, rows = P.rows, d = P.d, rowsT = P.rowsT;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gi = lane >> 2, q = lane & 3;  // accumulator fragment: row gi, columns 2q, 2q+1
    const int ald = A.akl + A.aku + 1;
    double* F = A.fac + P.fofs;
    double* TF = A.tfac ? A.tfac + P.tofs : nullptr;
    const int nblk = (m + 7) / 8;
    const unsigned full = 0xffffffffu;
    // LU-space (i, c) -> input band: base + sg * (c * (ald - 1) + i) (UL: reversed)
    const double* bbase = A.band + (P.rev ? (long long)(P.r0 + m - 1) * ald + A.aku : (long long)P.r0 * ald + A.aku);
    const long long sg = P.rev ? -1 : 1;
    auto inband = [&](int i, int c) { return i < m && c < m && i - c <= kl && c - i <= ku; };
    // LU-space entry; rows/columns past m continue as the identity
    auto val = [&](int i, int c) -> double {
        if (i >= 0 && c >= 0 && inband(i, c)) return bbase[sg * ((long long)c * (ald - 1) + i)];
        return (i == c && i >= m) ? 1.0 : 0.0;
    };

    // staging for the recycle at step Jr: the entering block nb = Jr + T as a
    // column (window rows 8(Jr+1) .. x 8 columns; read at step Jr) and as a row
    // (8 rows x the window columns 8(Jr+1) ..; read at step Jr+1 by the warp
    // taking it).  Column block of step J+1 and row block of step J are issued
    // at the start of step J (double buffers: nobody reads the buffer being
    // refilled).  TMA (one thread, two 2-D tiles through the aliased band view
    // of launch_lu_dmma) while both blocks lie inside the partition; the last
    // steps (and bands the view cannot describe) gather element-wise with
    // cp.async.  Buffers hold the TMA box layouts; a reversed (UL) partition's
    // boxes arrive mirrored (index BOX-1-L), and the element path writes them
    // the same way.  Slots outside the band are not cleared: readers mask them.
    const bool mir = P.rev != 0;
    auto tma_ok = [&](int Jr) { return tma_sh >= 0 && Jr >= 0 && Jr < nblk && 8 * (Jr + T) + 8 <= m; };
    // box origins at Jr = 0 (column box x, y; row box x, y), 8 rows / columns
    // further (reversed: back) per step; kept in shared memory, read by the
    // issuing thread only
    // TMA box rows must start on 16-byte boundaries (even x): a box whose
    // first row would be odd starts one row early (reversed: one late), so its
    // data sit one slot later (earlier) in the buffer -- every staging access,
    // the element path's included, is shifted by dsh (the same for both boxes
    // and all steps: x moves by 8 per step)
    int dsh = 0;
    if (tma_sh >= 0 && ((P.r0 + A.aku + A.col0 + tma_sh + (mir ? m : 0)) & 1)) dsh = mir ? -1 : 1;
    __shared__ int s_tc[4];
    if (threadIdx.x == 0 && tma_sh >= 0) {
        const long long xo = A.aku + A.col0 + tma_sh - dsh, yo = A.col0, r0 = P.r0, e = P.r0 + m - 1;
        s_tc[0] = (int)(xo + (mir ? e - 8 - (S::SC - 1) : r0 + 8));
        s_tc[1] = (int)(yo + (mir ? e - 8 * T - 7 : r0 + 8 * T));
        s_tc[2] = (int)(xo + (mir ? e - 8 * T - (S::SR - 1) : r0 + 8 * T));
        s_tc[3] = (int)(yo + (mir ? e - 8 - (8 * T - 1) : r0 + 8));
    }
    auto tma_issue = [&](int Jr, bool rows, unsigned long long* bar) {
        const int dx = (mir ? -8 : 8) * Jr;
        if (!rows) lu_tma_2d(sm + S::ST + (Jr & 1) * S::CB, &tmc, s_tc[0] + dx, s_tc[1] + dx, bar);
        else lu_tma_2d(sm + S::ST + 2 * S::CB + (Jr & 1) * S::RB, &tmr, s_tc[2] + dx, s_tc[3] + dx, bar);
    };
    // readers: column block element (window row ri, column jj), row block
    // element (row ii, window column ci)
    auto colv = [&](const double* buf, int ri, int jj) -> double {
        const int L = jj * S::SC + ri;
        return buf[(mir ? S::CB - 1 - L : L) + dsh];
    };
    auto rowv = [&](const double* buf, int ii, int ci) -> double {
        const int L = ci * S::SR + ii;
        return buf[(mir ? S::RB - 1 - L : L) + dsh];
    };
    // the slots outside the band hold whatever the box covered (other band
    // entries) or stale data: before the readers, the warp taking the entering
    // row this step (ro == NW) zeroes them in the column block of step J (read
    // after the mid-step barrier) and the row block of step J-1 (read by itself)
    auto zero_outside = [&](int J) {
        constexpr int c8 = 8 * (T - 1);
        double* cb = sm + S::ST + (J & 1) * S::CB;
        {
            const int jj = lane & 7, lo = min(jj + c8 - ku, c8);  // rows above the band (readers: < c8)
            for (int ri = lane >> 3; ri < lo; ri += 4) {
                const int L = jj * S::SC + ri;
                cb[(mir ? S::CB - 1 - L : L) + dsh] = 0.0;
            }
        }
        if (J > 0) {
            double* rb = sm + S::ST + 2 * S::CB + ((J + 1) & 1) * S::RB;
            const int ii = lane & 7, lo = min(c8 + ii - kl, 8 * T), hi = ii + c8 + ku;  // left of / right of the band
            for (int ci = lane >> 3; ci < lo; ci += 4) {
                const int L = ci * S::SR + ii;
                rb[(mir ? S::RB - 1 - L : L) + dsh] = 0.0;
            }
            for (int ci = hi + 1 + (lane >> 3); ci < 8 * T; ci += 4) {
                const int L = ci * S::SR + ii;
                rb[(mir ? S::RB - 1 - L : L) + dsh] = 0.0;
            }
        }
        // generic writes before the buffer's next TMA fill (after a CTA barrier)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
    };
    // element path: each warp instruction covers 4 rows x 8 columns of one
    // tile (global sources: 8 sectors, 4 consecutive rows per column); warp
    // `rank` of `nrank` (the diagonal warp of the step stays out)
    auto stage_load = [&](int Jr, bool rows, int rank, int nrank) {
        if (Jr < 0 || Jr >= nblk || rank < 0) return;
        const int cc = lane & 7, r4 = lane >> 3;
        for (int task = rank; task < 2 * T; task += nrank) {
            const int tile = task >> 1, rr = ((task & 1) << 2) + r4;  // row within the tile
            int i, c;
            double* dst;
            if (!rows) {  // entering column block: window rows 8(Jr+1) + 8 tile + rr, column cc
                i = 8 * (Jr + 1) + 8 * tile + rr;
                c = 8 * (Jr + T) + cc;
                const int L = cc * S::SC + 8 * tile + rr;
                dst = sm + S::ST + (Jr & 1) * S::CB + (mir ? S::CB - 1 - L : L) + dsh;
            } else {      // entering row block: row rr, window column 8(Jr+1) + 8 tile + cc
                i = 8 * (Jr + T) + rr;
                c = 8 * (Jr + 1) + 8 * tile + cc;
                const int L = (8 * tile + cc) * S::SR + rr;
                dst = sm + S::ST + 2 * S::CB + (Jr & 1) * S::RB + (mir ? S::RB - 1 - L : L) + dsh;
            }
            if (i - c > kl || c - i > ku) continue;  // outside the band: masked by the readers
            if (i < m && c < m) cp_async8(dst, bbase + sg * ((long long)c * (ald - 1) + i));
            else *dst = i == c ? 1.0 : 0.0;
        }
    };

    double amax = 0.0, minpiv = 1.0 / 0.0;
    int nboost = 0;
    bool boost_mode = false;
    double thresh = 0.0, bmag = 0.0;

    // factor the diagonal block of step Jn held as an accumulator fragment;
    // publish LU, 1/u_jj and both triangular inverses (buffer parity of Jn).
    // One pass over the 8 pivots: the LU, X = L11^-1 (rows below pivot c take
    // -l(gi, c) x row c) and Z = U11^-T (row c scales by 1/u_cc, rows below take
    // -u(c, gi) x row c) advance in lockstep; U11^-1 = Z^T is stored transposed.
    auto diag_factor = [&](double lu0, double lu1, int Jn) {
        const int par = Jn & 1, j0n = 8 * Jn;
        const int c0 = 2 * q, c1 = 2 * q + 1;
        double x0 = gi == c0, x1 = gi == c1, z0 = x0, z1 = x1;
        double dmine = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int src = c * 4 + (c >> 1);
            double pv = __shfl_sync(full, (c & 1) ? lu1 : lu0, src);
            const double lraw = __shfl_sync(full, (c & 1) ? lu1 : lu0, gi * 4 + (c >> 1));
            const double u0 = __shfl_sync(full, lu0, c * 4 + q);
            const double u1 = __shfl_sync(full, lu1, c * 4 + q);
            const double ua = __shfl_sync(full, lu0, c * 4 + (gi >> 1));
            const double ub = __shfl_sync(full, lu1, c * 4 + (gi >> 1));
            const double xk0 = __shfl_sync(full, x0, c * 4 + q);
            const double xk1 = __shfl_sync(full, x1, c * 4 + q);
            if (j0n + c < m) {
                minpiv = fmin(minpiv, fabs(pv));
                if (boost_mode && fabs(pv) < thresh) {
                    pv = pv == 0.0 ? bmag : copysign(bmag, pv);
                    if (lane == 0) ++nboost;
                }
            }
            // the (possibly boosted) pivot in place
            lu0 = (gi == c && c0 == c) ? pv : lu0;
            lu1 = (gi == c && c1 == c) ? pv : lu1;
            // 1/u_cc: hardware estimate + two Newton steps (a zero pivot gives a
            // non-finite inverse; the boosting re-run replaces it)
            double inv;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(pv));
            double e = fma(-pv, inv, 1.0);
            inv = fma(inv, e, inv);
            e = fma(-pv, inv, 1.0);
            inv = fma(inv, e, inv);
            dmine = lane == c ? inv : dmine;
            const double lr = lraw * inv;
            const bool below = gi > c;
            const double n0 = fma(-lr, u0, lu0), n1 = fma(-lr, u1, lu1);
            lu0 = below ? (c0 > c ? n0 : (c0 == c ? lr : lu0)) : lu0;
            lu1 = below ? (c1 > c ? n1 : (c1 == c ? lr : lu1)) : lu1;
            x0 = below ? fma(-lr, xk0, x0) : x0;
            x1 = below ? fma(-lr, xk1, x1) : x1;
            z0 = gi == c ? z0 * inv : z0;
            z1 = gi == c ? z1 * inv : z1;
            const double zc0 = __shfl_sync(full, z0, c * 4 + q);
            const double zc1 = __shfl_sync(full, z1, c * 4 + q);
            const double ucg = (gi & 1) ? ub : ua;
            z0 = below ? fma(-ucg, zc0, z0) : z0;
            z1 = below ? fma(-ucg, zc1, z1) : z1;
        }
        if (lane < 8) sm[S::DINV + par * 8 + lane] = dmine;
        double* sD = sm + S::D + par * 64;
        sD[gi * 8 + c0] = lu0;
        sD[gi * 8 + c1] = lu1;
        // L11^-1 (A-fragment order) and U11^-1 = Z^T (B-fragment order)
        double* sLi = sm + S::LI + par * 64;
        double* sUi = sm + S::UI + par * 64;
        sLi[afrag(gi, c0)] = x0;
        sLi[afrag(gi, c1)] = x1;
        sUi[bfrag(c0, gi)] = z0;
        sUi[bfrag(c1, gi)] = z1;
    };

    // positions of the packed layouts that no step writes must read as zero
    for (int idx = threadIdx.x; idx < ku * ku; idx += blockDim.x) {
        const int c = idx / ku, off = idx - c * ku + 1;
        if (c < m && off > c) F[(long long)c * rows + d - off] = 0.0;
    }
    // the row-major copy is optional (null: the transposed sweeps' copy is
    // made from the packed factor when a transposed solve first needs it)
    const bool wt = A.tfac != nullptr;
    for (int idx = threadIdx.x; idx < kl * kl && wt; idx += blockDim.x) {
        const int r = idx / kl, off = idx - r * kl + 1;
        if (r < m && off > r) TF[(long long)r * rowsT + kl - off] = 0.0;
    }

    double2* prow = reinterpret_cast<double2*>(sm + S::PROW) + lane;  // + parity * T * 32 + offset * 32
    double2* win = reinterpret_cast<double2*>(sm + S::WIN) + (size_t)w * NS * 32 + lane;
    for (int attempt = 0; attempt < 2; ++attempt) {
        double acc[TR][2];  // my tile row, by column offset from the panel (offsets < TR)
        // offset c of my row as seen at step J: registers or window slot
        auto slot = [&](int J, int c) {
            int sl = (J % NS) + c - TR;
            if (sl >= NS) sl -= NS;
            return sl;
        };
        auto get = [&](int J, int c, double& t0, double& t1) {
            if (c < TR) {
                t0 = acc[c < TR ? c : 0][0];
                t1 = acc[c < TR ? c : 0][1];
            } else {
                const double2 v = win[slot(J, c) * 32];
                t0 = v.x;
                t1 = v.y;
            }
        };
        auto put = [&](int J, int c, double t0, double t1) {
            if (c < TR) {
                acc[c < TR ? c : 0][0] = t0;
                acc[c < TR ? c : 0][1] = t1;
            } else {
                win[slot(J, c) * 32] = make_double2(t0, t1);
            }
        };
        auto load_row = [&](int b) {  // row block b over column blocks 0..T-1 (step 0 offsets)
#pragma unroll
            for (int c = 0; c < T; ++c) {
                const int i = 8 * b + gi, cc = 8 * c + 2 * q;
                const double v0 = val(i, cc), v1 = val(i, cc + 1);
                put(0, c, v0, v1);
                if (i < m) amax = fmax(amax, fmax(fabs(v0), fabs(v1)));
            }
        };
        // step 0: warp 0 factors block row 0 and publishes it (nothing
        // pending), warp 1 publishes block row 1 for step 1; warp w holds row
        // block w+1 (row offset ro = ((w - J) mod NW) + 1)
        if (w == 0) {
            load_row(0);
            diag_factor(acc[0][0], acc[0][1], 0);
#pragma unroll
            for (int c = 0; c < T; ++c) {
                double t0, t1;
                get(0, c, t0, t1);
                prow[c * 32] = make_double2(t0, t1);
            }
        }
        load_row(w + 1);
        if (w == 0) {  // panel row of step 1 (block 1) at step-1 offsets, minus the far tile
#pragma unroll
            for (int c = 1; c < T; ++c) {
                double t0, t1;
                get(0, c, t0, t1);
                prow[(T + c - 1) * 32] = make_double2(t0, t1);
            }
        }
        // TMA issues run at steps -1 (column block of step 0, barrier 1), 0, 1,
        // .. while tma_ok holds (monotone in the step), so the issue of step s
        // is phase (s + 1) >> 1 of barrier s & 1; re-armed for each attempt
        if (threadIdx.x == 0) {
            if (attempt > 0) {  // idle since the last step of the first pass
                asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(&s_mb[0])) : "memory");
                asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(&s_mb[1])) : "memory");
            }
            mbar_init(&s_mb[0], 1);
            mbar_init(&s_mb[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tma_ok(0) && threadIdx.x == 0) {
            lu_expect_tx(&s_mb[1], S::CB * 8);
            tma_issue(0, false, &s_mb[1]);
        }
        if (!tma_ok(0)) stage_load(0, false, w, NW);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();

        int ro = w + 1;
#ifdef SPK_LU_PROFILE
        long long tprev = clock64();
#endif
        for (int J = 0; J < nblk; ++J) {
            const int par = J & 1, j0 = 8 * J;
            // the warp that factors the next diagonal block this step (ro == 1)
            // does no staging and no output writes: they are off its chain
            const int orank = ro == 1 ? -1 : ro - 2;
            // the blocks staged by TMA at step J-1 (read this step) have landed
            if (tma_ok(J > 0 ? J - 1 : 0) && !LU_DBG(8)) mbar_wait(&s_mb[(J - 1) & 1], (J >> 1) & 1);
            if (ro == NW && !LU_DBG(4)) zero_outside(J);
            {
                const bool tc = tma_ok(J + 1), trw = tma_ok(J);
                if ((tc || trw) && threadIdx.x == 0 && !LU_DBG(16)) {
                    unsigned long long* bar = &s_mb[J & 1];
                    lu_expect_tx(bar, (tc && !LU_DBG(1) ? S::CB * 8 : 0) + (trw && !LU_DBG(2) ? S::RB * 8 : 0));
                    if (tc && !LU_DBG(1)) tma_issue(J + 1, false, bar);
                    if (trw && !LU_DBG(2)) tma_issue(J, true, bar);
                }
                if (!tc) stage_load(J + 1, false, orank, NW - 1);
                if (!trw) stage_load(J, true, orank, NW - 1);
                cp_async_commit();
            }
            LU_MARK(0);
            double* sLc = sm + S::L + par * 64 * T;
            double* sUc = sm + S::U + par * 64 * T;
            const double* sLp = sm + S::L + (par ^ 1) * 64 * T;
            const double* sUp = sm + S::U + (par ^ 1) * 64 * T;
            // a warp that took the entering row block last step reads it from staging
            const bool fresh = ro == NW && J > 0;
            const double* stp = sm + S::ST + 2 * S::CB + ((J + 1) & 1) * S::RB;  // row block of step J-1
            // 1a. L21 of my tile row: (panel-column tile) x U11^-1
            {
                double a0 = acc[0][0], a1 = acc[0][1];
                if (fresh) {
                    a0 = rowv(stp, gi, 2 * q);
                    a1 = rowv(stp, gi, 2 * q + 1);
                }
                // accumulator -> A fragments: A[gi][q + 4 ks] sits in lane gi*4 + 2ks + q/2
                double af[2];
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int src = gi * 4 + 2 * ks + (q >> 1);
                    const double v0 = __shfl_sync(0xffffffffu, a0, src);
                    const double v1 = __shfl_sync(0xffffffffu, a1, src);
                    af[ks] = (q & 1) ? v1 : v0;
                }
                const double* sUi = sm + S::UI + par * 64;
                double c0 = 0.0, c1 = 0.0;
                lu_dmma(c0, c1, af[0], sUi[lane]);
                lu_dmma(c0, c1, af[1], sUi[32 + lane]);
                sLc[ro * 64 + afrag(gi, 2 * q)] = -c0;
                sLc[ro * 64 + afrag(gi, 2 * q + 1)] = -c1;
            }
            // 1b. U12 of column offset co = w+1: L11^-1 x (panel-row tile with the
            // previous step's pending update -L21'[1] U12'[co+1] applied)
            {
                const int co = w + 1;
                const double2 pv = prow[(par * T + co) * 32];
                double c0 = pv.x, c1 = pv.y;
                if (J > 0 && co + 1 < T) {
                    lu_dmma(c0, c1, sLp[64 + lane], sUp[(co + 1) * 64 + lane]);
                    lu_dmma(c0, c1, sLp[64 + 32 + lane], sUp[(co + 1) * 64 + 32 + lane]);
                }
                // accumulator -> B fragments: B[q + 4 ks][gi] sits in lane (q + 4ks)*4 + gi/2
                double bf[2];
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int src = (q + 4 * ks) * 4 + (gi >> 1);
                    const double v0 = __shfl_sync(0xffffffffu, c0, src);
                    const double v1 = __shfl_sync(0xffffffffu, c1, src);
                    bf[ks] = (gi & 1) ? v1 : v0;
                }
                const double* sLi = sm + S::LI + par * 64;
                double u0 = 0.0, u1 = 0.0;
                lu_dmma(u0, u1, sLi[lane], bf[0]);
                lu_dmma(u0, u1, sLi[32 + lane], bf[1]);
                sUc[co * 64 + bfrag(gi, 2 * q)] = u0;
                sUc[co * 64 + bfrag(gi, 2 * q + 1)] = u1;
            }
            LU_MARK(1);
            __syncthreads();
            LU_MARK(2);

            const double* stc = sm + S::ST + (J & 1) * S::CB;  // column block of step J
            if (ro == 1) {
                // my row is the next panel row, already published one step ago
                // (this step's update is applied by 1b of the next step) except
                // its far tile, the entering column block; then update and factor
                // the next diagonal tile.  Next step I take the entering row block.
                const double2 cv = make_double2(colv(stc, gi, 2 * q), colv(stc, gi, 2 * q + 1));
                prow[((par ^ 1) * T + T - 1) * 32] = cv;
                if (8 * (J + 1) + gi < m) amax = fmax(amax, fmax(fabs(cv.x), fabs(cv.y)));
                double d0 = acc[1][0], d1 = acc[1][1];
                // my tiles are dead from here (next step I take the entering row
                // block): constants free their registers across the chain below
#pragma unroll
                for (int c = 0; c < TR; ++c) acc[c][0] = acc[c][1] = 0.0;
                LU_MARK(3);
                lu_dmma(d0, d1, sLc[64 + lane], sUc[64 + lane]);
                lu_dmma(d0, d1, sLc[64 + 32 + lane], sUc[64 + 32 + lane]);
                if (!LU_DBG(64)) diag_factor(d0, d1, J + 1);
                LU_MARK(4);
            }
            if (ro != 1) {
                // 2. trailing update of my tile row, shifted by one tile; the
                // entering column block comes in at the far end
                const double la0 = sLc[ro * 64 + lane], la1 = sLc[ro * 64 + 32 + lane];
                if (fresh) {
                    const bool live = 8 * (J - 1 + T) + gi < m;
#pragma unroll
                    for (int c = 1; c < T; ++c) {
                        double t0 = rowv(stp, gi, 8 * c + 2 * q), t1 = rowv(stp, gi, 8 * c + 2 * q + 1);
                        if (live) amax = fmax(amax, fmax(fabs(t0), fabs(t1)));
                        lu_dmma(t0, t1, la0, sUc[c * 64 + lane]);
                        lu_dmma(t0, t1, la1, sUc[c * 64 + 32 + lane]);
                        put(J + 1, c - 1, t0, t1);
                    }
                    const double2 v0 = make_double2(rowv(stp, gi, 2 * q), rowv(stp, gi, 2 * q + 1));
                    if (live) amax = fmax(amax, fmax(fabs(v0.x), fabs(v0.y)));
                } else {
                    // register tiles k-slice-major: a tile's two DMMAs are TR-1
                    // instructions apart (back to back they stall on the DMMA latency)
#pragma unroll
                    for (int c = 1; c < TR; ++c)
                        lu_dmma(acc[c][0], acc[c][1], la0, sUc[c * 64 + lane]);
#pragma unroll
                    for (int c = 1; c < TR; ++c)
                        lu_dmma(acc[c][0], acc[c][1], la1, sUc[c * 64 + 32 + lane]);
#pragma unroll
                    for (int c = TR; c < T; ++c) {
                        {
                            double t0, t1;
                            get(J, c, t0, t1);
                            lu_dmma(t0, t1, la0, sUc[c * 64 + lane]);
                            lu_dmma(t0, t1, la1, sUc[c * 64 + 32 + lane]);
                            put(J, c, t0, t1);
                        }
                    }
                    // shift by one tile: registers move down, the window slot of
                    // offset TR comes into the last register (and is refilled below)
#pragma unroll
                    for (int c = 0; c + 1 < TR; ++c) {
                        acc[c][0] = acc[c + 1][0];
                        acc[c][1] = acc[c + 1][1];
                    }
                    if (TR < T) {
                        double t0, t1;
                        get(J, TR, t0, t1);
                        acc[TR - 1][0] = t0;
                        acc[TR - 1][1] = t1;
                    }
                }
                const double2 cv = make_double2(colv(stc, 8 * (ro - 1) + gi, 2 * q), colv(stc, 8 * (ro - 1) + gi, 2 * q + 1));
                put(J + 1, T - 1, cv.x, cv.y);
                if (8 * (J + ro) + gi < m) amax = fmax(amax, fmax(fabs(cv.x), fabs(cv.y)));
                if (ro == 2) {
                    // publish my row (next step's ro = 1) as the panel row of step J+2
#pragma unroll
                    for (int c = 1; c < T; ++c) {
                        double t0, t1;
                        get(J + 1, c, t0, t1);
                        prow[(par * T + c - 1) * 32] = make_double2(t0, t1);
                    }
                }
                LU_MARK(5);
            }
            // write L columns j0.. and U rows j0.. (both packed layouts) and 1/u_jj
            if (j0 < m && !LU_DBG(32)) {
                const double* sD = sm + S::D + par * 64;
                // L columns (packed column-major) and U rows (row-major copy): one
                // contiguous run per warp, its (<= 5) loads issued before its stores
                constexpr int KIT = (8 * (T - 1) + 32) / 32;  // <= k + 1 entries per run
                const int nseg = wt ? 16 : 8;
                for (int sgm = orank; sgm < nseg && orank >= 0; sgm += NW - 1) {
                    const int qq = sgm & 7, c = j0 + qq;
                    if (c >= m) continue;
                    const bool lseg = sgm < 8;
                    double* dst = lseg ? F + (long long)c * rows + d : TF + (long long)c * rowsT + kl;
                    const int o0 = lseg ? 1 : 0, oe = lseg ? kl : ku;
                    double v[KIT];
#pragma unroll
                    for (int it = 0; it < KIT; ++it) {
                        const int off = o0 + lane + 32 * it, rc = qq + off;
                        v[it] = 0.0;
                        if (off <= oe) {
                            if (lseg) v[it] = rc < 8 ? sD[rc * 8 + qq] : -sLc[(rc >> 3) * 64 + afrag(rc & 7, qq)];
                            else v[it] = rc < 8 ? sD[qq * 8 + rc] : sUc[(rc >> 3) * 64 + bfrag(qq, rc & 7)];
                        }
                    }
#pragma unroll
                    for (int it = 0; it < KIT; ++it) {
                        const int off = o0 + lane + 32 * it;
                        if (off <= oe) dst[off] = c + off < m ? v[it] : 0.0;
                    }
                }
                // L rows (row-major copy) and U columns (packed): run x holds the
                // <= 8 entries of rows / columns j0..j0+7 of L row j0+x / U column
                // j0+x; one lane per run (two 4-entry fragment runs in shared
                // memory, 16-byte stores), starting on the warps without a column
                const int nl = wt ? 7 + kl : 0, nrun = nl + 8 + ku;
                const int brank = (orank + (NW - 1) - nseg % (NW - 1)) % (NW - 1);
                for (int t = brank * 32 + lane; t < nrun && orank >= 0; t += 32 * (NW - 1)) {
                    const bool lrun = t < nl;
                    const int x = lrun ? t + 1 : t - nl;
                    if (j0 + x >= m) continue;
                    const int lo = max(0, x - (lrun ? kl : ku)), hi = min(lrun ? x - 1 : x, min(7, m - 1 - j0));
                    double* dst = lrun ? TF + (long long)(j0 + x) * rowsT + kl - x : F + (long long)(j0 + x) * rows + d - x;
                    double v[8];
                    if (x >= 8) {
                        const double* src = (lrun ? sLc : sUc) + (x >> 3) * 64 + (x & 7) * 4;
                        const double2 p0 = *reinterpret_cast<const double2*>(src);
                        const double2 p1 = *reinterpret_cast<const double2*>(src + 2);
                        const double2 p2 = *reinterpret_cast<const double2*>(src + 32);
                        const double2 p3 = *reinterpret_cast<const double2*>(src + 34);
                        const double sg1 = lrun ? -1.0 : 1.0;
                        v[0] = sg1 * p0.x, v[1] = sg1 * p0.y, v[2] = sg1 * p1.x, v[3] = sg1 * p1.y;
                        v[4] = sg1 * p2.x, v[5] = sg1 * p2.y, v[6] = sg1 * p3.x, v[7] = sg1 * p3.y;
                    } else {
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq) v[qq] = lrun ? sD[x * 8 + qq] : sD[qq * 8 + x];
                    }
                    if (lo == 0 && hi == 7) {
                        const bool al = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
                        double* d2 = al ? dst : dst + 1;
                        if (!al) dst[0] = v[0];
                        *reinterpret_cast<double2*>(d2) = al ? make_double2(v[0], v[1]) : make_double2(v[1], v[2]);
                        *reinterpret_cast<double2*>(d2 + 2) = al ? make_double2(v[2], v[3]) : make_double2(v[3], v[4]);
                        *reinterpret_cast<double2*>(d2 + 4) = al ? make_double2(v[4], v[5]) : make_double2(v[5], v[6]);
                        if (al) *reinterpret_cast<double2*>(d2 + 6) = make_double2(v[6], v[7]);
                        else dst[7] = v[7];
                    } else {
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq)
                            if (qq >= lo && qq <= hi) dst[qq] = v[qq];
                    }
                }
                if (threadIdx.x < 8 && j0 + threadIdx.x < m)
                    A.dinv[P.r0 + j0 + threadIdx.x] = sm[S::DINV + par * 8 + threadIdx.x];
            }
            LU_MARK(6);
            ro = ro == 1 ? NW : ro - 1;
            cp_async_wait<0>();  // element-path staging of this step, read next step
            __syncthreads();
            LU_MARK(7);
        }
        cp_async_wait<0>();
        // optimistic boosting check: max|A_i| and min|u_jj| over the CTA
        double am = amax, mp = minpiv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            am = fmax(am, __shfl_xor_sync(full, am, o));
            mp = fmin(mp, __shfl_xor_sync(full, mp, o));
        }
        if (lane == 0) {
            s_red[w] = am;
            s_red[32 + w] = mp;
        }
        __syncthreads();
        am = 0.0;
        mp = 1.0 / 0.0;
        for (int i = 0; i < NW; ++i) {
            am = fmax(am, s_red[i]);
            mp = fmin(mp, s_red[32 + i]);
        }
        __syncthreads();
        const double scale = am == 0.0 ? 1.0 : am;
        if (boost_mode || !(mp < DBL_EPSILON * scale)) break;
        boost_mode = true;
        thresh = DBL_EPSILON * scale;
        bmag = A.boost_eps * scale;
        nboost = 0;
    }
    if (lane == 0) s_cnt[w] = nboost;
    __syncthreads();
    if (threadIdx.x == 0) {
        int nb = 0;
        for (int i = 0; i < NW; ++i) nb += s_cnt[i];
        if (nb) atomicAdd(&A.boost_cnt[u], nb);
    }
    for (int j = threadIdx.x; j < m; j += blockDim.x) A.piv[P.r0 + j] = j;
}

// The band seen by TMA: element (R, C) sits at band[C*ald + aku + R - C] =
// base[(C + col0) * (ald - 1) + (R + aku + col0)], i.e. a 2-D tensor with
// x = R + aku + col0 (contiguous) and y = C + col0 (stride (ald - 1) doubles)
// whose rows overlap in memory -- TMA only computes addresses, so a box is
// "rows x0.. of columns y0..", the band's diagonal structure flattened.  Rows
// past the readable columns come back as zeros (out-of-bounds fill).  Needs
// (ald - 1) * 8 to be a multiple of 16 (kl + ku even); the base is aligned
// down to 16 bytes by shifting x.  tma_sh = -1: no maps, element path only.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static const EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            (void)cudaGetLastError();
            return (EncodeTiledFn) nullptr;
        }
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

static int band_tensor_maps(const FastLuArgs& A, unsigned sc, unsigned sr, unsigned bw, CUtensorMap* tmc,
                            CUtensorMap* tmr) {
    const long long ald = A.akl + A.aku + 1;
    if (A.ncols <= 0 || ((ald - 1) * 8) % 16 != 0) return -1;
    const EncodeTiledFn enc = encode_tiled();
    if (!enc) return -1;
    const double* base = A.band - A.col0 * ald;
    const uintptr_t a = reinterpret_cast<uintptr_t>(base);
    if (a % 8) return -1;
    const int sh = (int)((a % 16) / 8);
    base -= sh;
    const cuuint64_t dims[2] = {(cuuint64_t)(A.ncols + A.aku + sh), (cuuint64_t)A.ncols};
    if (dims[0] >= (1ull << 31) || dims[1] >= (1ull << 31)) return -1;  // int coordinates
    const cuuint64_t strides[1] = {(cuuint64_t)(ald - 1) * 8};
    const cuuint32_t boxc[2] = {sc, 8}, boxr[2] = {sr, bw}, es[2] = {1, 1};
    void* g = const_cast<double*>(base);
    if (enc(tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, boxc, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    if (enc(tmr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, boxr, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    return sh;
}

template <int T, int TR>
static bool launch_lu_dmma(const int* d_units, int nunits, const FastLuArgs& A, cudaStream_t s) {
    using S = LuDmmaSmem<T, TR>;
    const size_t smem = sizeof(double) * S::TOTAL + 128;  // + alignment of the base
    if (smem > 227 * 1024) return false;
    set_smem_attr((const void*)k_band_lu_dmma<T, TR>, (int)smem);
    CUtensorMap tmc, tmr;
    memset(&tmc, 0, sizeof(tmc));
    memset(&tmr, 0, sizeof(tmr));
    const int sh = band_tensor_maps(A, S::SC, S::SR, 8 * T, &tmc, &tmr);
    k_band_lu_dmma<T, TR><<<nunits, 32 * (T - 1), smem, s>>>(A, tmc, tmr, sh);
    count_launch();
    return true;
}

// ===========================================================================
// Partial-pivoting band LU (gbtf2 semantics, kernels.cpp:79-118 pivoting
// branch), one CTA per partition, active window in shared memory.
//
// Step j touches rows j..j+kl and columns j..j+ubw (ubw = kl+ku): that window
// is kept circularly (row r in row slot r mod (kl+1), column c in column slot
// c mod (ubw+1)).  Three CTA barriers per column: (1) warp argmax of |a(r, j)|
// (first index on ties) -> pivot; (2) interchange rows j and ip in columns >=
// j, multipliers l = a(:, j) / a(ip, j) and the pivot row u copied aside;
// (3) rank-1 update a(r, c) -= l(r) u(c) (skipped where u(c) == 0, as the
// reference does), the finished L column / U row go to the packed factor, and
// the slots of column j and row j take the entering column j+ubw+1 and row
// j+kl+1 (raw band values: no earlier step touched them), staged by cp.async
// one step ahead.  An exactly zero pivot column sets status 2 (the
// reference's runtime_error).  tfac / 1/u_jj follow from the transpose stage.
struct PivLuArgs {
    const int* units;
    const PartDev* parts;
    const double* band;
    int akl, aku;
    double* fac;
    int* piv;
    int* status;
};

__global__ void __launch_bounds__(256, 2) k_band_lu_piv(PivLuArgs A) {
    extern __shared__ __align__(16) double psm[];
    const int u = A.units[blockIdx.x];
    const PartDev P = A.parts[u];
    const int m = P.m, kl = P.kl, ku = P.ku, ubw = P.ubw, d = P.d, rows = P.rows;
    const int NR = kl + 1, NC = ubw + 1, LDW = NR + (NR % 2 == 0 ? 1 : 0);  // odd column stride
    double* W = psm;                     // [NC][LDW]
    double* s_l = W + (size_t)NC * LDW;  // [NR] multipliers of the step (row slot order)
    double* s_u = s_l + NR;              // [NC] pivot row (column slot order)
    double* s_st = s_u + NC;             // [4][NR + NC] staging ring: entering column, entering row
    __shared__ int s_ip, s_fail;
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = T >> 5;
    const int ald = A.akl + A.aku + 1;
    double* F = A.fac + P.fofs;
    int* piv = A.piv + P.r0;
    const double* bbase = A.band + (P.rev ? (long long)(P.r0 + m - 1) * ald + A.aku : (long long)P.r0 * ald + A.aku);
    const long long sg = P.rev ? -1 : 1;
    auto aval_ptr = [&](int i, int c) -> const double* {
        if (i < 0 || c < 0 || i >= m || c >= m || i - c > kl || c - i > ku) return nullptr;
        return bbase + sg * ((long long)c * (ald - 1) + i);
    };
    // staging for step js (entering column js+ubw+1 rows js+1..js+kl+1, entering
    // row js+kl+1 columns js+1..js+ubw+1)
    auto stage = [&](int js) {
        double* st = s_st + (js & 3) * (NR + NC);
        for (int e = tid; e < NR + NC; e += T) {
            int i, c;
            if (e < NR) {
                i = js + 1 + e;
                c = js + ubw + 1;
            } else {
                i = js + kl + 1;
                c = js + 1 + (e - NR);
            }
            const double* p = aval_ptr(i, c);
            if (p) cp_async8(st + e, p);
            else st[e] = 0.0;
        }
        cp_async_commit();
    };
    // zero the packed positions no step writes (above row 0)
    for (int idx = tid; idx < ubw * ubw; idx += T) {
        const int c = idx / ubw, off = idx - c * ubw + 1;
        if (c < m && off > c) F[(long long)c * rows + d - off] = 0.0;
    }
    // initial window: rows 0..kl, columns 0..ubw
    for (int e = tid; e < NC * NR; e += T) {
        const int c = e / NR, r = e - c * NR;
        const double* p = aval_ptr(r, c);
        W[(size_t)c * LDW + r] = p ? *p : 0.0;
    }
    stage(0);  // three steps ahead: HBM latency exceeds a step
    stage(1);
    stage(2);
    __syncthreads();
    for (int j = 0; j < m; ++j) {
        const int rl = min(kl, m - 1 - j);    // rows below the pivot
        const int ce = min(ubw, m - 1 - j);   // columns right of the pivot
        const int cs = j % NC;
        // (1) pivot: max |a(r, j)|, r = j..j+rl, first index on ties
        if (wid == 0) {
            double best = -1.0;
            int bi = j;
            int slot = (j + lane) % NR;
            const int step = 32 % NR;
            for (int r = j + lane; r <= j + rl; r += 32) {
                const double a = fabs(W[(size_t)cs * LDW + slot]);
                if (a > best) {
                    best = a;
                    bi = r;
                }
                slot += step;
                if (slot >= NR) slot -= NR;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_ip = bi;
                s_fail = !(best > 0.0);
            }
        }
        __syncthreads();
        if (s_fail) {
            if (tid == 0) atomicMax(A.status, 2);
            return;
        }
        const int ip = s_ip, sj = j % NR, sp = ip % NR;
        // (2) interchange rows j, ip in columns j..j+ce; pivot row aside; multipliers
        for (int cc = tid; cc <= ce; cc += T) {
            int csl = cs + cc;
            if (csl >= NC) csl -= NC;  // cc < T = 512 may exceed NC: reduce fully
            while (csl >= NC) csl -= NC;
            double* col = W + (size_t)csl * LDW;
            const double vj = col[sj], vp = col[sp];
            col[sj] = vp;
            col[sp] = vj;
            s_u[cc] = vp;
        }
        if (tid == 0) piv[j] = ip;
        __syncthreads();
        {
            const double inv = 1.0 / s_u[0];
            double* colj = W + (size_t)cs * LDW;
            for (int r = 1 + tid; r <= rl; r += T) {
                int sl = sj + r;
                while (sl >= NR) sl -= NR;
                const double l = colj[sl] * inv;
                colj[sl] = l;
                s_l[r] = l;
            }
        }
        cp_async_wait<2>();  // this step's staging (issued three steps ago), visible after the barrier
        __syncthreads();
        // (3) rank-1 update (warp -> columns, lane -> rows); outputs; refill
        {
            int sl0 = sj + 1 + lane;  // row slot of row j+1+lane
            while (sl0 >= NR) sl0 -= NR;
            const int rstep = 32 % NR;
            int csl = cs + 1 + wid;  // column slot of column j+1+wid
            while (csl >= NC) csl -= NC;
            const int cstep = nw % NC;
            for (int cc = 1 + wid; cc <= ce; cc += nw) {
                const double uc = s_u[cc];
                double* col = W + (size_t)csl * LDW;
                csl += cstep;
                if (csl >= NC) csl -= NC;
                if (uc == 0.0) continue;
                int sl = sl0;
                for (int r = 1 + lane; r <= rl; r += 32) {
                    double& a = col[sl];
                    a = fma(-s_l[r], uc, a);
                    sl += rstep;
                    if (sl >= NR) sl -= NR;
                }
            }
        }
        // packed factor: L column j (rows j+1..j+kl, zero past m), U row j
        for (int r = 1 + tid; r <= kl; r += T) F[(long long)j * rows + d + r] = r <= rl ? s_l[r] : 0.0;
        for (int cc = tid; cc <= ubw; cc += T)
            if (j + cc < m) F[(long long)(j + cc) * rows + d - cc] = cc <= ce ? s_u[cc] : 0.0;
        // entering column / row into the slots of column j and row j
        {
            const double* st = s_st + (j & 3) * (NR + NC);
            // column j+ubw+1 into slot cs: rows j+1..j+kl+1 -> row slots
            for (int e = tid; e < NR; e += T) {
                int sl = sj + 1 + e;
                while (sl >= NR) sl -= NR;
                W[(size_t)cs * LDW + sl] = st[e];
            }
            // row j+kl+1 into row slot sj: columns j+1..j+ubw (the corner column
            // j+ubw+1 came with the column above)
            for (int e = tid; e < NC - 1; e += T) {
                int csl = cs + 1 + e;
                while (csl >= NC) csl -= NC;
                W[(size_t)csl * LDW + sj] = st[NR + e];
            }
        }
        __syncthreads();
        stage(j + 3);
    }
    cp_async_wait<0>();
}

bool launch_band_lu_piv(const int* d_units, int nunits, int kl, int ku, const PivLuArgs& A, cudaStream_t s) {
    // the reversed (UL) partition swaps kl and ku: size for the larger window
    const int ubw = kl + ku, NR = std::max(kl, ku) + 1, NC = ubw + 1, LDW = NR + (NR % 2 == 0 ? 1 : 0);
    const size_t smem = sizeof(double) * ((size_t)NC * LDW + NR + NC + 4 * (NR + NC));
    if (smem > 200 * 1024) return false;
    set_smem_attr((const void*)k_band_lu_piv, (int)smem);
    k_band_lu_piv<<<nunits, 256, smem, s>>>(A);  // 2 CTAs per SM (registers)
    count_launch();
    return true;
}

bool launch_band_lu_fast(const int* d_units, int nunits, int kmax, const FastLuArgs& A, cudaStream_t s) {
    (void)nunits;
    if (kmax < 1) return false;
    if (kmax <= 32) return launch_lu_dmma<5, 5>(d_units, nunits, A, s);
    if (kmax <= 64) return launch_lu_dmma<9, 9>(d_units, nunits, A, s);
    if (kmax <= 96) return launch_lu_dmma<13, 13>(d_units, nunits, A, s);
    if (kmax <= 128) return launch_lu_dmma<17, 17>(d_units, nunits, A, s);
    if (kmax <= 160) return launch_lu_dmma<21, 12>(d_units, nunits, A, s);
    return false;
}

}  // namespace spk
