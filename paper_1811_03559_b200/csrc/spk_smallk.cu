// spk_smallk.cu — the small-k engine: non-pivoting SPIKE for narrow bands
// (kl, ku <= 31), HBM/latency-bound, in three launches per factorization and
// one per forward solve instead of the general engine's stage programs
// (~250 dependent launches at BASELINE C1).
//
//   k_sk_parts   (spk_smallk_parts.cu) one warp per partition: the partition's band columns (plus k
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

// ===========================================================================
// reduced hierarchy (reduce_factorize, factorize.cpp:46-120), one cooperative
// kernel, one grid barrier per level.
//
// Pair a of level l: left unit (hL rows; V = vl, W = wl), right unit (hR rows;
// V = vr, W = wr).  Coupling [[I, Vb], [Wt, I]] with Vb = vl[hL-k : hL],
// Wt = wr[0 : k]; while max|W| <= 1 partial pivoting on it takes the identity
// pivots (kernels.cpp:94), so it factors through the Schur complement
// S = I - Wt Vb.  The merged unit's spikes are the pair solves of [0; vr] and
// [wl; 0] (factorize.cpp:19-32):
//   z2 = S^-1 (y2 - Wt y1), z1 = y1 - Vb z2,
//   rows [0, hL-k) -= vl[0:hL-k] z2 (left rows), rows [hL+k, H) -= wr[k:hR] z1.
// Phase ph runs two tasks:
//   A (level ph, one warp per pair): the pair's k x k algebra only -- S,
//     S^-1 (Gauss-Jordan in registers, a row of [S | I] per lane pair; no row
//     search when S is column diagonally dominant, where partial pivoting
//     takes the diagonal anyway), z1, z2, and the merged unit's TIP rows (top
//     k, bottom k) straight from the children's tips, so the next level's
//     task A needs nothing else;
//   B (level ph-1, a CTA per row item): the merged units' other rows.
namespace {
constexpr int kLvWarps = 4;
constexpr int kLvThreads = 32 * kLvWarps;
constexpr int kLd = 20;          // 16 x 16 blocks, row-major, ld 20 (16-byte rows; a fragment's 8 rows hit all banks)
constexpr int kBlk = 16 * kLd;
enum { B_WT, B_VB, B_Y2, B_Y1, B_VLT, B_WLT, B_VRB, B_WRB, B_S, B_UW, B_SI, B_Z2V, B_Z2W, B_Z1V, B_Z1W, NBLK };
constexpr int kWarpSmem = NBLK * kBlk;  // doubles per warp

// 16 x 16 products on the FP64 tensor cores (mma.sync m8n8k4): 4 output
// tiles, 4 k-steps; operand fragments are single 8-byte shared loads (row
// pitch kLd = 20 spreads the 8 rows of a fragment over all banks).  Tile
// t = 2 ti + tj holds rows 8ti + (lane>>2), columns 8tj + 2(lane&3) + {0,1}.
__device__ __forceinline__ void sk_dmma(double d[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}
__device__ __forceinline__ void dgemm16(const double* Am, const double* Bm, double d[4][2], int lane) {
    const int g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int t = 0; t < 4; ++t) d[t][0] = d[t][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const double a0 = Am[g * kLd + 4 * kk + q], a1 = Am[(8 + g) * kLd + 4 * kk + q];
        const double b0 = Bm[(4 * kk + q) * kLd + g], b1 = Bm[(4 * kk + q) * kLd + 8 + g];
        sk_dmma(d[0], a0, b0);
        sk_dmma(d[1], a0, b1);
        sk_dmma(d[2], a1, b0);
        sk_dmma(d[3], a1, b1);
    }
}
// element e (0, 1) of tile t: block offset
__device__ __forceinline__ int toff(int t, int lane) {
    return (8 * (t >> 1) + (lane >> 2)) * kLd + 8 * (t & 1) + 2 * (lane & 3);
}
// C = sa * d + (base ? base : 0) into shared memory (C may alias base)
__device__ __forceinline__ void tiles_put(double* C, const double d[4][2], double sa, const double* base, int lane) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int o = toff(t, lane);
        double2 v = make_double2(sa * d[t][0], sa * d[t][1]);
        if (base) {
            const double2 b = *reinterpret_cast<const double2*>(base + o);
            v.x += b.x;
            v.y += b.y;
        }
        *reinterpret_cast<double2*>(C + o) = v;
    }
}
// a k x k block held in shared memory to rows [r0, r0 + k) of a spike
// (column-major, ld h) in global memory
__device__ __forceinline__ void blk_store(double* dst, long long h, int r0, const double* Bm, int k, int lane) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = lane + 32 * i, c = e >> 4, r = e & 15;  // rows fastest: coalesced
        if (r < k && c < k) dst[(long long)c * h + r0 + r] = Bm[r * kLd + c];
    }
}

__device__ __forceinline__ double rcp_nr(double x) {
    // reciprocal: MUFU seed and two Newton steps (no IEEE-division slow path;
    // pivots here are normal numbers)
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ void sk_pair_task(const SkLevelsArgs& A, const SkPair& pr, double* sm, int lane) {
    const unsigned full = 0xffffffffu;
    const int k = A.k;
    const int hL = pr.hL, hR = pr.hR, H = hL + hR;
    const bool hv = pr.nv >= 0, hw = pr.nw >= 0;
    auto B = [&](int i) { return sm + i * kBlk; };
    // the eight k x k tips straight into shared memory (cp.async), zero padding
    {
        const double* vl = A.pool + pr.vl;
        const double* wr = A.pool + pr.wr;
        const double* wl = A.pool + (hw ? pr.wl : 0);
        const double* vr = A.pool + (hv ? pr.vr : 0);
        for (int e = lane; e < 256; e += 32) {
            const int r = e & 15, c = e >> 4, o = r * kLd + c;  // column-major walk: coalesced reads
            if (r < k && c < k) {
                sk_cp8(B(B_WT) + o, wr + (long long)c * hR + r);
                sk_cp8(B(B_VB) + o, vl + (long long)c * hL + hL - k + r);
                sk_cp8(B(B_VLT) + o, vl + (long long)c * hL + r);
                sk_cp8(B(B_WRB) + o, wr + (long long)c * hR + hR - k + r);
                if (hv) {
                    sk_cp8(B(B_Y2) + o, vr + (long long)c * hR + r);
                    sk_cp8(B(B_VRB) + o, vr + (long long)c * hR + hR - k + r);
                } else {
                    B(B_Y2)[o] = 0.0;
                    B(B_VRB)[o] = 0.0;
                }
                if (hw) {
                    sk_cp8(B(B_Y1) + o, wl + (long long)c * hL + hL - k + r);
                    sk_cp8(B(B_WLT) + o, wl + (long long)c * hL + r);
                } else {
                    B(B_Y1)[o] = 0.0;
                    B(B_WLT)[o] = 0.0;
                }
            } else {
#pragma unroll
                for (int b = B_WT; b <= B_WRB; ++b) B(b)[o] = 0.0;
            }
        }
        sk_cp_wait_all();
        __syncwarp();
    }
    // S = I - Wt Vb (padding: identity), UW = -Wt Y1
    {
        double d[4][2], e[4][2];
        dgemm16(B(B_WT), B(B_VB), d, lane);
        dgemm16(B(B_WT), B(B_Y1), e, lane);
#pragma unroll
        for (int t = 0; t < 4; ++t) {  // identity on the diagonal tiles
            const int r = 8 * (t >> 1) + (lane >> 2), c0 = 8 * (t & 1) + 2 * (lane & 3);
            d[t][0] = (r == c0 ? 1.0 : 0.0) - d[t][0];
            d[t][1] = (r == c0 + 1 ? 1.0 : 0.0) - d[t][1];
        }
        tiles_put(B(B_S), d, 1.0, nullptr, lane);
        tiles_put(B(B_UW), e, -1.0, nullptr, lane);
    }
    __syncwarp();
    // column diagonal dominance of S (then partial pivoting takes the diagonal)
    bool dom = true;
    if (lane < 16) {
        double o = 0.0;
#pragma unroll
        for (int i = 0; i < 16; ++i) o += i == lane ? 0.0 : fabs(B(B_S)[i * kLd + lane]);
        dom = fabs(B(B_S)[lane * kLd + lane]) > o;
    }
    dom = __all_sync(full, dom);
    // Gauss-Jordan on [S | I] in registers: lane (r, h) holds row r, columns
    // 16h .. 16h+15 of the augmented matrix
    const int r = lane & 15, h = lane >> 4;
    double a[16];
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(B(B_S) + r * kLd + c);
        a[c] = h == 0 ? v.x : (r == c ? 1.0 : 0.0);
        a[c + 1] = h == 0 ? v.y : (r == c + 1 ? 1.0 : 0.0);
    }
    unsigned used = 0u;
    int jr = r;  // S^-1 row held by this lane's I-part: the step whose pivot row is r
    double boost = 0.0;  // an exactly singular S: zero pivots boosted (kernels.cpp:104-109 rule)
    if (!dom) {
        double mx = 0.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) mx = fmax(mx, h == 0 ? fabs(a[c]) : 0.0);
        boost = A.boost_eps * fmax(warp_max(mx), 1.0);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const double colv = __shfl_sync(full, a[j], r);  // aug[r][j] (S part, lane (r, 0))
        int p = j;
        if (!dom) {
            double v = (lane < 16 && !((used >> lane) & 1u)) ? fabs(colv) : -1.0;
            int idx = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(full, v, o);
                const int oi = __shfl_xor_sync(full, idx, o);
                if (ov > v || (ov == v && oi < idx)) {
                    v = ov;
                    idx = oi;
                }
            }
            // all candidates zero: the first unused row, its pivot boosted
            p = v > 0.0 ? idx : __ffs(~used & 0xffffu) - 1;
        }
        used |= 1u << p;
        if (r == p) jr = j;
        double piv = __shfl_sync(full, a[j], p);  // aug[p][j]
        if (piv == 0.0) piv = boost;
        const double inv = rcp_nr(piv);
        const double g = colv * inv;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const double pv = __shfl_sync(full, a[c], p + 16 * h);
            a[c] = r == p ? pv * inv : fma(-g, pv, a[c]);
        }
    }
    // S^-1 row jr = this lane's I part (h = 1): shared memory and the pool
    if (h == 1) {
        double* d = B(B_SI) + jr * kLd;
#pragma unroll
        for (int c = 0; c < 16; c += 2) *reinterpret_cast<double2*>(d + c) = make_double2(a[c], a[c + 1]);
        if (jr < k) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < k) A.pool[pr.sinv + (long long)c * k + jr] = a[c];
        }
    }
    if (lane == 0) A.flags[pr.gidx] = 1;
    __syncwarp();
    // z2v = S^-1 y2, z2w = S^-1 (-Wt y1): rows [hL, hL+k) of the merged unit
    {
        double d[4][2], e[4][2];
        dgemm16(B(B_SI), B(B_Y2), d, lane);
        dgemm16(B(B_SI), B(B_UW), e, lane);
        tiles_put(B(B_Z2V), d, 1.0, nullptr, lane);
        tiles_put(B(B_Z2W), e, 1.0, nullptr, lane);
    }
    __syncwarp();
    // z1v = -Vb z2v, z1w = y1 - Vb z2w: rows [hL-k, hL); top tips
    // vt' = -vl_top z2v, wt' = wl_top - vl_top z2w: rows [0, k)
    {
        double d[4][2], e[4][2], f[4][2], g4[4][2];
        dgemm16(B(B_VB), B(B_Z2V), d, lane);
        dgemm16(B(B_VB), B(B_Z2W), e, lane);
        dgemm16(B(B_VLT), B(B_Z2V), f, lane);
        dgemm16(B(B_VLT), B(B_Z2W), g4, lane);
        __syncwarp();  // VLT / WLT are rewritten in place
        tiles_put(B(B_Z1V), d, -1.0, nullptr, lane);
        tiles_put(B(B_Z1W), e, -1.0, B(B_Y1), lane);
        tiles_put(B(B_VLT), f, -1.0, nullptr, lane);
        tiles_put(B(B_WLT), g4, -1.0, B(B_WLT), lane);
    }
    __syncwarp();
    // bottom tips: vb' = vr_bot - wr_bot z1v, wb' = -wr_bot z1w: rows [H-k, H)
    {
        double d[4][2], e[4][2];
        dgemm16(B(B_WRB), B(B_Z1V), d, lane);
        dgemm16(B(B_WRB), B(B_Z1W), e, lane);
        __syncwarp();  // WRB is rewritten in place
        tiles_put(B(B_VRB), d, -1.0, B(B_VRB), lane);
        tiles_put(B(B_WRB), e, -1.0, nullptr, lane);
    }
    __syncwarp();
    if (hv) {
        double* nv = A.pool + pr.nv;
        blk_store(nv, H, 0, B(B_VLT), k, lane);
        blk_store(nv, H, hL - k, B(B_Z1V), k, lane);
        blk_store(nv, H, hL, B(B_Z2V), k, lane);
        blk_store(nv, H, H - k, B(B_VRB), k, lane);
    }
    if (hw) {
        double* nw = A.pool + pr.nw;
        blk_store(nw, H, 0, B(B_WLT), k, lane);
        blk_store(nw, H, hL - k, B(B_Z1W), k, lane);
        blk_store(nw, H, hL, B(B_Z2W), k, lane);
        blk_store(nw, H, H - k, B(B_WRB), k, lane);
    }
}

// carried odd unit: its tip rows move up now (the rest in task B)
__device__ void sk_carry_tips(const SkLevelsArgs& A, int u, int nu_i, int lane) {
    const int k = A.k;
    const SkUnit u0 = A.units[u], u1 = A.units[nu_i];
    const int h = u0.uh;
    for (int e = lane; e < 2 * k * k; e += 32) {
        const int c = e / (2 * k), q = e - c * 2 * k;
        const int rr = q < k ? q : h - 2 * k + q;
        if (u0.voff >= 0) A.pool[u1.voff + (long long)c * h + rr] = A.pool[u0.voff + (long long)c * h + rr];
        if (u0.woff >= 0) A.pool[u1.woff + (long long)c * h + rr] = A.pool[u0.woff + (long long)c * h + rr];
    }
}

// task B: rows [k, hL-k) and [hL+k, H-k) of a merged unit, one per thread
__device__ void sk_rows_task(const SkLevelsArgs& A, const SkItem& I, double* zs) {
    const int k = A.k, tid = threadIdx.x;
    if (I.pair < 0) {  // carried unit: the non-tip rows
        const SkUnit u0 = A.units[-(I.pair + 1)], u1 = A.units[I.next];
        const int h = u0.uh;
        for (int rr = I.row0 + tid; rr < h - k && rr < I.row0 + kSkChunk; rr += blockDim.x) {
            if (rr < k) continue;
            for (int c = 0; c < k; ++c) {
                if (u0.voff >= 0) A.pool[u1.voff + (long long)c * h + rr] = A.pool[u0.voff + (long long)c * h + rr];
                if (u0.woff >= 0) A.pool[u1.woff + (long long)c * h + rr] = A.pool[u0.woff + (long long)c * h + rr];
            }
        }
        return;
    }
    const SkPair pr = A.pairs[I.pair];
    const int hL = pr.hL, hR = pr.hR, H = hL + hR;
    const bool hv = pr.nv >= 0, hw = pr.nw >= 0;
    // z blocks from the merged unit's middle rows: zs[0] z2v, [1] z2w, [2] z1v, [3] z1w (row-major ld 16)
    __syncthreads();
    {
        // every load of the thread in one batch (one memory round trip)
        constexpr int kPer = 4 * 256 / kLvThreads;
        double v[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int e = tid + i * kLvThreads;
            const int w = e >> 8, q = e & 255, rr = q & 15, c = q >> 4;
            const int row = (w < 2 ? hL : hL - k) + rr;
            const bool isv = (w & 1) == 0;
            const long long off = isv ? pr.nv : pr.nw;
            v[i] = (rr < k && c < k && off >= 0) ? A.pool[off + (long long)c * H + row] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int e = tid + i * kLvThreads;
            const int w = e >> 8, q = e & 255;
            zs[w * kBlk + (q & 15) * kLd + (q >> 4)] = v[i];
        }
    }
    __syncthreads();
    if (k == 16) {
        // the FP64 tensor cores: 8-row tiles of the item, a warp per tile;
        // D = base - M z as mma.sync with A = -M (fragments straight from the
        // spike's columns), C = the base spike's rows, B = z from shared memory
        const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
        for (int t = warp; t < kSkChunk / 8; t += kLvWarps) {
            const int R0 = I.row0 + 8 * t;
            if (R0 >= H) break;
            const bool left = R0 >= k && R0 + 8 <= hL - k;
            const bool right = R0 >= hL + k && R0 + 8 <= H - k;
            if (!left && !right) continue;
            const double* M = A.pool + (left ? pr.vl : pr.wr);
            const int hm = left ? hL : hR, ro = (left ? R0 : R0 - hL) + g;
            double am[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) am[kk] = -M[(long long)(4 * kk + q) * hm + ro];
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
                const bool isv = pass == 0;
                if (isv ? !hv : !hw) continue;
                const long long bo = isv ? (left ? -1 : pr.vr) : (left ? pr.wl : -1);
                const double* z = zs + ((left ? 0 : 2) + (isv ? 0 : 1)) * kBlk;
                double d[2][2];
#pragma unroll
                for (int tj = 0; tj < 2; ++tj)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        d[tj][e] = bo >= 0 ? A.pool[bo + (long long)(8 * tj + 2 * q + e) * hm + ro] : 0.0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int tj = 0; tj < 2; ++tj) sk_dmma(d[tj], am[kk], z[(4 * kk + q) * kLd + 8 * tj + g]);
                double* dst = A.pool + (isv ? pr.nv : pr.nw);
#pragma unroll
                for (int tj = 0; tj < 2; ++tj)
#pragma unroll
                    for (int e = 0; e < 2; ++e) dst[(long long)(8 * tj + 2 * q + e) * H + R0 + g] = d[tj][e];
            }
        }
        return;
    }
    for (int rr = I.row0 + tid; rr < H && rr < I.row0 + kSkChunk; rr += blockDim.x) {
        const bool left = rr >= k && rr < hL - k;
        const bool right = rr >= hL + k && rr < H - k;
        if (!left && !right) continue;
        const double* M = A.pool + (left ? pr.vl : pr.wr);
        const int hm = left ? hL : hR, ro = left ? rr : rr - hL;
        // merged V: left rows -vl z2v, right rows vr - wr z1v; merged W: left
        // rows wl - vl z2w, right rows -wr z1w.  All loads first.
        const long long bo = left ? (hw ? pr.wl : -1) : (hv ? pr.vr : -1);
        double mrow[16], base[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            mrow[q] = q < k ? M[(long long)q * hm + ro] : 0.0;
            base[q] = (q < k && bo >= 0) ? A.pool[bo + (long long)q * hm + ro] : 0.0;
        }
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            const bool isv = pass == 0;
            if (isv ? !hv : !hw) continue;
            const bool hasb = isv ? !left : left;  // the pass that adds the base spike
            double acc[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[c] = hasb ? base[c] : 0.0;
            const double* z = zs + ((left ? 0 : 2) + (isv ? 0 : 1)) * kBlk;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                if (q >= k) break;
#pragma unroll
                for (int c = 0; c < 16; ++c) acc[c] = fma(-mrow[q], z[q * kLd + c], acc[c]);
            }
            double* dst = A.pool + (isv ? pr.nv : pr.nw);
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < k) dst[(long long)c * H + rr] = acc[c];
        }
    }
}
}  // namespace

__global__ void __launch_bounds__(kLvThreads, 1) k_sk_levels(SkLevelsArgs A) {
    extern __shared__ __align__(16) double lv_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* const wsm = lv_smem + warp * kWarpSmem;
    const int nwarps = gridDim.x * kLvWarps;
    unsigned target = 0;
    for (int ph = 0; ph <= A.nlevels; ++ph) {
        sk_stamp(A.trace, ph, 0);
        // task A on the first CTAs (a warp per pair), task B first on the CTAs
        // that have no pair: the phase costs max(A, B), not A + B
        const int ntask = ph < A.nlevels ? A.levels[ph].npairs + (A.levels[ph].carry >= 0 ? 1 : 0) : 0;
        const int ctasA = min((int)gridDim.x, (ntask + kLvWarps - 1) / kLvWarps);
        if (ph < A.nlevels) {
            const SkLevel L = A.levels[ph];
            for (int a = blockIdx.x * kLvWarps + warp; a < ntask; a += nwarps) {
                if (a < L.npairs) sk_pair_task(A, A.pairs[L.pair0 + a], wsm, lane);
                else sk_carry_tips(A, L.carry, L.carry_next, lane);
                __syncwarp();
            }
        }
        __syncthreads();
        sk_stamp(A.trace, ph, 1);
        if (ph >= 1) {
            const SkLevel L = A.levels[ph - 1];
            const int nb = (int)gridDim.x - ctasA;  // CTAs without a pair
            const int b0 = nb > 0 ? (int)blockIdx.x - ctasA : (int)blockIdx.x;
            if (b0 >= 0)
                for (int it = b0; it < L.nitems; it += (nb > 0 ? nb : (int)gridDim.x))
                    sk_rows_task(A, A.items[L.item0 + it], lv_smem);
        }
        sk_stamp(A.trace, ph, 2);
        if (ph < A.nlevels) grid_barrier(A.bar, target);
        sk_stamp(A.trace, ph, 3);
    }
}

void launch_sk_levels(const SkLevelsArgs& A, cudaStream_t s) {
    if (A.nlevels <= 0) return;
    const int smem = (int)(sizeof(double) * kWarpSmem * kLvWarps);
    set_smem_attr((const void*)k_sk_levels, smem);
    SkLevelsArgs a = A;
    void* args[] = {&a};
    (void)cudaLaunchCooperativeKernel((const void*)k_sk_levels, device_sms(), kLvThreads, args, smem, s);
    count_launch();  // reports a failed launch
}


}  // namespace spk
