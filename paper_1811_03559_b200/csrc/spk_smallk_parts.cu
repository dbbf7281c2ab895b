// spk_smallk_parts.cu — the small-k engine's partition stage (k_sk_parts):
// LU with diagonal boosting, the packed factor, 1/u_jj, corner blocks and the
// level-0 spike tips of every partition, for kl, ku <= 16, non-pivoting.
//
// Two partitions per warp, one per half-warp (16 lanes).  A partition's band
// rows are staged once into shared memory in LU space (the reversed last
// partition is reversed while staging), pitch 34 doubles: row li holds columns
// li-16 .. li+16 at positions 0..32, position 33 holds 1/u_ii.  Everything
// after the staging runs out of shared memory and registers:
//
//   LU (LUFactors::factor, src/kernels.cpp:79-118), lanes = rows: lane hl
//     holds the window rows congruent to hl mod 16, each as 17 register slots
//     (column c in slot c mod 17, the step loop unrolled 17 times so every slot
//     index is a constant).  Step j: the pivot lane boosts u_jj if needed
//     (kernels.cpp:104-109), writes the U row and 1/u_jj back to the staged
//     band and takes over row j+16; every lane reads the U row (a broadcast),
//     forms its multiplier l = a * (1/u_jj), stores it, and applies 16 FMAs.
//   packed factor out (the general engine's layout: column-major, rows
//     ubw+kl+1, diagonal at row ubw), coalesced from the staged band.
//   spike tips (factorize.cpp:133-257), lanes = spike columns: V = A^-1 [0; B^]
//     (truncated forward L sweep over its last k rows), W = A^-1 [C^; 0] (full
//     forward L sweep, results stored over the dead L entries of each row),
//     then one backward U sweep over both (inner partitions: all rows, tips
//     top and bottom; the first partition: V's bottom tip; the last, reversed:
//     its W through the reversed LU = the reference's UL, in the V registers).
//     The L and U columns are shared-memory broadcasts; each step is 16 FMAs
//     per spike column.
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_smallk.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

namespace spk {

namespace {

constexpr int kPitch = 34;  // staged row: 33 band positions + 1/u_ii
constexpr int KS = 17;      // register window slots
constexpr int kPad = 17;    // zero rows before and after a CTA's staged blocks: the sweeps read
                            // window rows past a partition's ends without tests (neighbours'
                            // rows or padding; only rows that are never used are touched)

__device__ __forceinline__ double half_max(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int half_sum(int v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace

size_t sk_parts_smem_per_part(int mmax) { return sizeof(double) * (size_t)mmax * kPitch; }
size_t sk_parts_smem_pad() { return sizeof(double) * (size_t)2 * kPad * kPitch; }

template <int NW>
__global__ void __launch_bounds__(32 * NW) k_sk_parts(SkPartsArgs A) {
    extern __shared__ __align__(16) double sk_slab[];
    const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
    const int warp = threadIdx.x >> 5;
    const int i = (blockIdx.x * NW + warp) * 2 + half;  // partition of this half-warp
    const bool live = i < A.p;
    double* const S = sk_slab + kPad * kPitch + (size_t)(warp * 2 + half) * A.mmax * kPitch;
    {  // zero the CTA's pad rows (front and back)
        double* pf = sk_slab;
        double* pb = sk_slab + kPad * kPitch + (size_t)2 * NW * A.mmax * kPitch;
        for (int e = threadIdx.x; e < kPad * kPitch; e += blockDim.x) {
            pf[e] = 0.0;
            pb[e] = 0.0;
        }
    }

    PartDev P{};
    if (live) P = A.parts[i];
    const int m = live ? P.m : 0;
    const int mo = __shfl_xor_sync(0xffffffffu, m, 16);
    const int mx = max(m, mo);  // loop bound shared by both halves
    const int rev = P.rev;
    const long long r0 = P.r0;
    const int ld = A.akl + A.aku + 1;

    // ---- stage the partition block in LU space: the band is column-major
    //      packed (A(i, j) at band[j * ld + aku + i - j]), read column by
    //      column (contiguous) with cp.async straight into the staged rows;
    //      entries outside the block / band stay zero
    const int k = A.k, aku = A.aku;
    const bool first = i == 0, last = i == A.p - 1;
    {
        for (int e = hl * 2; e < m * kPitch; e += 32)
            *reinterpret_cast<double2*>(S + e) = make_double2(0.0, 0.0);
        __syncwarp();
        const int tot = m * ld;
        int cj = 0, b = hl;
        const double* src = A.band + r0 * ld;
        for (int e = hl; e < tot; e += 16) {
            while (b >= ld) {
                b -= ld;
                ++cj;
            }
            const int ci = cj + b - aku;  // physical row offset in the block
            if (ci >= 0 && ci < m) {
                const int li = rev ? m - 1 - ci : ci, lj = rev ? m - 1 - cj : cj;
                sk_cp8(S + li * kPitch + lj - li + 16, src + e);
            }
            b += 16;
        }
    }
    // corner columns (lane c: column c of B^ and C^, physical; spike2x2.cpp:17-26),
    // in flight with the staging
    double bh[16], ch[16];
    {
        const int c = hl;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            const int bb = aku - k + rr - c, bc = aku + k + rr - c;  // A(r0+m-k+rr, r0+m+c), A(r0+rr, r0-k+c)
            bh[rr] = (live && !last && c < k && rr < k && r0 + m + c < A.n && bb >= 0 && bb < ld)
                         ? A.band[(r0 + m + c) * ld + bb] : 0.0;
            ch[rr] = (live && !first && c < k && rr < k && r0 - k + c >= 0 && bc >= 0 && bc < ld)
                         ? A.band[(r0 - k + c) * ld + bc] : 0.0;
        }
    }
    sk_cp_wait_all();
    __syncwarp();
    double amax = 0.0;
    for (int e = hl * 2; e < m * kPitch; e += 32) {
        const double2 v = *reinterpret_cast<const double2*>(S + e);
        amax = fmax(amax, fmax(fabs(v.x), fabs(v.y)));
    }
    amax = half_max(amax);
    const double scale = amax == 0.0 ? 1.0 : amax;
    const double zero_thresh = DBL_EPSILON * scale, boost_mag = A.boost_eps * scale;

    // ---- LU, lanes = rows
    double R[KS];
#pragma unroll
    for (int c = 0; c < KS; ++c) R[c] = hl < m ? S[hl * kPitch + c - hl + 16] : 0.0;
    int boosts = 0;
    for (int j0 = 0; j0 < mx; j0 += KS) {
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int j = j0 + t;
            if (j >= mx) break;
            const bool act = j < m;
            if (act && hl == (j & 15)) {
                double u = R[t];
                if (fabs(u) < zero_thresh) {
                    u = u == 0.0 ? boost_mag : copysign(boost_mag, u);
                    ++boosts;
                }
                R[t] = u;
                double* row = S + j * kPitch + 16;  // 16-byte aligned (pitch 34, offset 16)
#pragma unroll
                for (int c = 0; c < 16; c += 2)
                    *reinterpret_cast<double2*>(row + c) = make_double2(R[(t + c) % KS], R[(t + c + 1) % KS]);
                *reinterpret_cast<double2*>(row + 16) = make_double2(R[(t + 16) % KS], 1.0 / u);
                // row j+16, columns j .. j+16 (untouched so far)
                const double* nrow = S + (j + 16) * kPitch;
                if (j + 16 < m) {
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(nrow + c);
                        R[(t + c) % KS] = v.x;
                        R[(t + c + 1) % KS] = v.y;
                    }
                    R[(t + 16) % KS] = nrow[16];
                } else {
#pragma unroll
                    for (int c = 0; c < KS; ++c) R[c] = 0.0;
                }
            }
            __syncwarp();
            if (act) {
                const double* urow = S + j * kPitch + 16;
                double uj[KS];
                uj[1] = urow[1];
#pragma unroll
                for (int c = 2; c < 16; c += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(urow + c);
                    uj[c] = v.x;
                    uj[c + 1] = v.y;
                }
                const double2 tail = *reinterpret_cast<const double2*>(urow + 16);
                uj[16] = tail.x;
                const double inv = tail.y;
                const int r = j + 1 + ((hl - j - 1) & 15);
                const bool rv = r < m;
                const double l = R[t] * inv;
                if (rv) S[r * kPitch + j - r + 16] = l;
#pragma unroll
                for (int c = 1; c < KS; ++c) R[(t + c) % KS] = fma(-l, uj[c], R[(t + c) % KS]);
                R[t] = (rv && j + 17 < m) ? S[r * kPitch + j + 33 - r] : 0.0;
            }
        }
    }
    __syncwarp();
    boosts = half_sum(boosts);
    if (!live) return;  // no collective operations below
    if (hl == 0) A.boost[i] = boosts;

    // ---- packed factor (column lj: rows d-ubw .. ; li = lj + q - d) and 1/u
    {
        double* F = A.fac + P.fofs;
        const int rows = P.rows, d = P.d, tot = m * rows;
        int lj = 0, q = hl;
        for (int e = hl; e < tot; e += 16) {
            while (q >= rows) {
                q -= rows;
                ++lj;
            }
            const int li = lj + q - d;
            F[e] = (li >= 0 && li < m) ? S[li * kPitch + lj - li + 16] : 0.0;
            q += 16;
        }
        for (int j = hl; j < m; j += 16) A.dinv[r0 + j] = S[j * kPitch + 33];
    }
    if (A.p < 2 || k == 0) return;

    // ---- corners to the pool
    const long long kk = (long long)k * k;
    if (hl < k) {
#pragma unroll
        for (int rr = 0; rr < 16; ++rr)
            if (rr < k) {  // (zero blocks where the edge is closed: the pool is not cleared)
                A.pool[A.off_bhat + i * kk + hl * k + rr] = bh[rr];
                A.pool[A.off_chat + i * kk + hl * k + rr] = ch[rr];
            }
    }

    // ---- spike sweeps, lanes = spike columns (c = hl < k)
    const bool inner = !first && !last;
    const int c = hl;
    const bool cv = c < k;
    const int mk = m - k;
    // V (first, inner: B^ in rows >= m-k; the last, reversed: C^ reversed):
    // truncated forward sweep over the last k rows, row j in slot m-1-j
    // (distance from the bottom) -- the backward sweep's own slot order.  It
    // reads the L columns before the W sweep overwrites them.
    double V[KS];
    {
#pragma unroll
        for (int u = 0; u < 16; ++u) {  // row m-1-u: B^ row k-1-u, or C^ row u (reversed)
            const int rr = last ? u : k - 1 - u;
            double v = 0.0;
            if (cv && u < k) {
                const int bb = last ? aku + k + rr - c : aku - k + rr - c;
                const long long col = last ? r0 - k + c : r0 + m + c;
                const bool ok = last ? (col >= 0) : (col < A.n);
                if (ok && bb >= 0 && bb < ld) v = A.band[col * ld + bb];
            }
            V[u] = v;
        }
        V[16] = 0.0;
#pragma unroll
        for (int u = 15; u >= 0; --u) {
            if (u >= k) continue;
            const int j = m - 1 - u;
            const double x = V[u];
#pragma unroll
            for (int o = 1; o < 16; ++o)
                if (u - o >= 0) V[u - o] = fma(-S[(j + o) * kPitch + 16 - o], x, V[u - o]);
        }
    }
    // W (inner partitions: C^ in rows < k): full forward L sweep, row r in
    // slot r mod 17; row j's result is stored over its dead L entries
    // (positions 0..15 of staged row j) for the backward sweep
    if (inner) {
        double W[KS];
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) W[s2] = (cv && s2 < k) ? ch[s2] : 0.0;
        for (int j0 = 0; j0 < m; j0 += KS) {
#pragma unroll
            for (int t = 0; t < KS; ++t) {
                const int j = j0 + t;
                if (j >= m) break;
                double lv[KS];  // L(j+o, j); rows past m read a neighbour's rows or padding
#pragma unroll
                for (int o = 1; o < KS; ++o) lv[o] = S[(j + o) * kPitch + 16 - o];
                const double x = W[t];
#pragma unroll
                for (int o = 1; o < KS; ++o) W[(t + o) % KS] = fma(-lv[o], x, W[(t + o) % KS]);
                __syncwarp();  // the L column of row j is read: its slots take W(j, :)
                S[j * kPitch + c] = x;
                W[t] = 0.0;  // entering row j + 17: C^ rows are < k <= 16
            }
        }
        __syncwarp();
    }
    // backward U sweep, rows m-1 .. je (inner: all rows, tips at both ends;
    // first / last: the bottom k), row j in slot (m-1-j) mod 17
    const int je = inner ? 0 : mk;
    const SkUnit U0 = A.units[i];
    const long long twok = 2LL * k;
    if (cv && first) {  // dead top rows of the first partition's V unit
        for (int r = 0; r < k; ++r) A.pool[U0.voff + c * twok + r] = 0.0;
    }
    if (cv && last) {  // dead bottom rows of the last partition's W unit
        for (int r = 0; r < k; ++r) A.pool[U0.woff + c * twok + k + r] = 0.0;
    }
    double W[KS];
#pragma unroll
    for (int s2 = 0; s2 < KS; ++s2) W[s2] = inner ? S[(m - 1 - s2) * kPitch + c] : 0.0;  // (padding above row 0)
    const int ns = m - je;  // backward steps
    for (int s0 = 0; s0 < ns; s0 += KS) {
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int sd = s0 + t;
            if (sd >= ns) break;
            const int j = m - 1 - sd;
            double uv[KS];  // U(j-o, j); rows above 0 read a neighbour's rows or padding
#pragma unroll
            for (int o = 1; o < KS; ++o) uv[o] = S[(j - o) * kPitch + 16 + o];
            const double dv = S[j * kPitch + 33];
            const double xv = V[t] * dv;
            const double xw = W[t] * dv;
            if (cv) {
                if (inner) {
                    if (j < k || j >= mk) {
                        const int rr = j < k ? j : k + j - mk;
                        A.pool[U0.voff + c * twok + rr] = xv;
                        A.pool[U0.woff + c * twok + rr] = xw;
                    }
                } else if (last) {
                    A.pool[U0.woff + c * twok + (m - 1 - j)] = xv;
                } else {
                    A.pool[U0.voff + c * twok + k + (j - mk)] = xv;
                }
            }
            // row j - o sits in slot (sd + o) mod 17
#pragma unroll
            for (int o = 1; o < KS; ++o) V[(t + o) % KS] = fma(-uv[o], xv, V[(t + o) % KS]);
            if (inner) {
#pragma unroll
                for (int o = 1; o < KS; ++o) W[(t + o) % KS] = fma(-uv[o], xw, W[(t + o) % KS]);
            }
            // entering row j - 17 (its slot is row j's): V is zero above m - k;
            // W from its stored forward result (padding above row 0)
            V[t] = 0.0;
            W[t] = inner ? S[(j - KS) * kPitch + c] : 0.0;
        }
    }
}

template <int NW>
static bool launch_parts_t(const SkPartsArgs& A, size_t smem, cudaStream_t s) {
    set_smem_attr((const void*)k_sk_parts<NW>, (int)smem);
    const int per = 2 * NW;
    k_sk_parts<NW><<<(A.p + per - 1) / per, 32 * NW, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_sk_parts(const SkPartsArgs& A, cudaStream_t s) {
    if (A.akl > 16 || A.aku > 16) return false;
    const size_t per = sk_parts_smem_per_part(A.mmax), pad = sk_parts_smem_pad();
    // as many warps per CTA as fit in 227 KB (one CTA per SM)
    const size_t cap = 227u * 1024;
    if (8 * per + pad <= cap) return launch_parts_t<4>(A, 8 * per + pad, s);
    if (4 * per + pad <= cap) return launch_parts_t<2>(A, 4 * per + pad, s);
    if (2 * per + pad <= cap) return launch_parts_t<1>(A, 2 * per + pad, s);
    return false;
}

}  // namespace spk
