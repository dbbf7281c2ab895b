// spk_coupling.cu — reduced-system coupling blocks via their Schur complement.
//
// The reference factors every 2k x 2k coupling C = [[I, V], [W, I]] with a
// pivoted dense LU, falling back to a boosted one on an exactly singular
// column (src/factorize.cpp:94-102, src/kernels.cpp:67-77).  Partial pivoting
// on C takes the identity pivots of its first k columns exactly when every
// |W_ij| <= 1 (ties keep the diagonal, strict '>' at kernels.cpp:94); C then
// factors as [[I, 0], [W, L_S]] [[I, V], [0, U_S]] with P_S S = L_S U_S the
// partially pivoted LU of the k x k Schur complement S = I - W V.  On B200:
//   k_wcheck      flag[pair] = max|W| <= 1            (else: generic 2k path)
//   k_schur_init  S storage := I (dense k x k kept as a full band, so the band
//                 sweep kernels solve with it)      ; then S -= W V on DMMA
//   k_schur_inverse  S^-1 by register-resident Gauss-Jordan with partial
//                 pivoting (the solves apply it as a GEMM); an exactly zero
//                 pivot column clears the flag so the generic path reproduces
//                 the reference's boosted fallback.
//   k_dense_lu    partial-pivot LU of S in shared memory, LAPACK/gbtf2 row
//                 interchange convention (earlier L columns not swapped): the
//                 P_S S = L_S U_S factors spk_fact_coupling reports.
#include "spk_device.cuh"
#include "spk_launch.h"

#include <algorithm>
#include <cfloat>

namespace spk {

// flag[g] = (max |W| <= 1) for the top k x k tip of wr (h x k, ld h).  The
// pair's k columns are split over gridDim.y CTAs (warp per column, lanes over
// rows); flags were set to 1 by k_wcheck_init, and any CTA seeing |w| > 1
// writes 0 (idempotent: deterministic).
__global__ void k_wcheck_init(const CouplingJob* __restrict__ jobs, int njobs, int* __restrict__ flags) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < njobs) flags[jobs[a].guard] = 1;
}

__global__ void __launch_bounds__(256) k_wcheck(const CouplingJob* __restrict__ jobs,
                                                const double* __restrict__ pool, int* __restrict__ flags) {
    const CouplingJob J = jobs[blockIdx.x];
    const int k = J.k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    int bad = 0;
    for (int c = blockIdx.y * W + warp; c < k; c += gridDim.y * W) {
        const double* col = pool + J.wr_off + (long long)c * J.hR;
        for (int r = lane; r < k; r += 32) bad |= fabs(col[r]) > 1.0;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) flags[J.guard] = 0;
}

// S unit storage (dense k x k as a full band: rows 2k-1, diagonal row k-1) := I
__global__ void k_schur_init(const CouplingJob* __restrict__ jobs, const PartDev* __restrict__ parts,
                             double* __restrict__ fac, int* __restrict__ piv_pool, const int* __restrict__ flags) {
    const CouplingJob J = jobs[blockIdx.y];
    if (flags[J.guard] != 1) return;
    const PartDev P = parts[J.part];
    const long long total = (long long)P.m * P.rows;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(e / P.rows);
        const int q = (int)(e - (long long)j * P.rows);
        fac[P.fofs + e] = (q == P.d) ? 1.0 : 0.0;
        (void)j;
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.m; j += gridDim.x * blockDim.x)
        piv_pool[P.r0 + j] = j;
}

// Partial-pivoting dense LU of the k x k S units in shared memory.
__global__ void __launch_bounds__(512) k_dense_lu(const CouplingJob* __restrict__ jobs,
                                                  const PartDev* __restrict__ parts, double* __restrict__ fac,
                                                  int* __restrict__ piv_pool, int* __restrict__ flags) {
    const CouplingJob J = jobs[blockIdx.x];
    if (flags[J.guard] != 1) return;
    const PartDev P = parts[J.part];
    const int n = P.m;
    extern __shared__ double sm[];  // n x n column-major, ld n+1 (odd: the row swap is conflict-free)
    __shared__ int s_ip, s_fail;
    const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31;
    double* F = fac + P.fofs;
    const int ls = n + 1;
    for (int e = tid; e < n * n; e += T) {
        const int c = e / n, r = e - c * n;
        sm[c * ls + r] = F[(long long)c * P.rows + P.d + r - c];
    }
    __syncthreads();
    int* piv = piv_pool + P.r0;
    for (int j = 0; j < n; ++j) {
        if (tid < 32) {
            double best = -1.0;
            int bi = j;
            for (int r = j + lane; r < n; r += 32) {
                const double a = fabs(sm[j * ls + r]);
                if (a > best) {
                    best = a;
                    bi = r;
                }
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
                s_fail = best == 0.0;
            }
        }
        __syncthreads();
        if (s_fail) {
            if (tid == 0) flags[J.guard] = 0;  // generic 2k path takes over (boosted fallback)
            return;
        }
        const int ip = s_ip;
        if (tid == 0) piv[j] = ip;
        if (ip != j)
            for (int c = j + tid; c < n; c += T) {
                const double t = sm[c * ls + j];
                sm[c * ls + j] = sm[c * ls + ip];
                sm[c * ls + ip] = t;
            }
        __syncthreads();
        const double inv = 1.0 / sm[j * ls + j];
        for (int r = j + 1 + tid; r < n; r += T) sm[j * ls + r] *= inv;
        __syncthreads();
        // rank-1 update: warp -> columns, lane -> consecutive rows (no index
        // divisions, conflict-free); zero a(j, c) skipped as in kernels.cpp:108
        const int nw = T >> 5, wid = tid >> 5;
        for (int c = j + 1 + wid; c < n; c += nw) {
            const double ajc = sm[c * ls + j];
            if (ajc == 0.0) continue;
            double* col = sm + (size_t)c * ls;
            const double* lj = sm + (size_t)j * ls;
            for (int r = j + 1 + lane; r < n; r += 32) col[r] -= ajc * lj[r];
        }
        __syncthreads();
    }
    for (int e = tid; e < n * n; e += T) {
        const int c = e / n, r = e - c * n;
        F[(long long)c * P.rows + P.d + r - c] = sm[c * ls + r];
    }
}

// S^-1 of the k x k Schur units by in-place Gauss-Jordan with partial
// pivoting, register resident: thread (warp w of 8, lane l) holds S(r, c) for
// r = l + 32a, c = w + 8b.  Step j: the owner warp of column j (w = j % 8)
// picks the pivot among the rows not yet used (max |s(r, j)|, first index on
// ties: the same choice as the row-interchange LU), publishes the column and
// the pivot through shared memory (double-buffered, one CTA barrier per
// step); every warp takes the pivot row of its own columns by warp shuffle
// and updates in registers:
//   row ip:  s(ip, c) /= p, s(ip, j) = 1/p;  others: s(r, c) -= s(r, j) s(ip, c)/p,
//   s(r, j) = -s(r, j)/p.
// Pivot rows are never moved, so the result M is the inverse up to the
// pivot order: S^-1(q(r), perm(c)) = M(r, c), perm(j) = pivot row of step j,
// q = perm^-1.  An exactly zero pivot column clears the flag (generic 2k path,
// like k_dense_lu).  S itself stays in the factor pool (spk_fact_coupling
// factors it on demand).
template <int RA, int CB, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_schur_inverse(const CouplingJob* __restrict__ jobs,
                                                           const PartDev* __restrict__ parts,
                                                           const double* __restrict__ fac,
                                                           double* __restrict__ pool, int* __restrict__ flags) {
    constexpr int NR = 32 * RA;
    __shared__ double s_col[2][NR];
    __shared__ double s_inv[2];
    __shared__ int s_ip[2];
    __shared__ int s_perm[NR], s_q[NR];
    __shared__ double s_row[NW][CB];
    const CouplingJob J = jobs[blockIdx.x];
    if (flags[J.guard] != 1) return;
    const PartDev P = parts[J.part];
    const int n = P.m;
    const double* F = fac + P.fofs;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double a[RA][CB];
#pragma unroll
    for (int ra = 0; ra < RA; ++ra)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
            const int r = lane + 32 * ra, c = w + NW * cb;
            a[ra][cb] = (r < n && c < n) ? F[(long long)c * P.rows + P.d + r - c] : 0.0;
        }
    unsigned used = 0;
#pragma unroll
    for (int ra = 0; ra < RA; ++ra)
        if (lane + 32 * ra >= n) used |= 1u << ra;
    // Register chunks are only ever selected by warp- or block-uniform indices
    // (column chunk jb of the owner warp, row chunk ia of the pivot), so the
    // selections compile to uniform branches, never to runtime-indexed
    // registers (which would be demoted to local memory).
    auto publish = [&](int j) {  // owner warp of column j
        const int jb = j / NW, buf = j & 1;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb)
            if (cb == jb)
#pragma unroll
                for (int ra = 0; ra < RA; ++ra) s_col[buf][lane + 32 * ra] = a[ra][cb];
        __syncwarp();
        double best = -1.0, bv = 0.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) {
            const double v = s_col[buf][lane + 32 * ra];
            if (!((used >> ra) & 1u) && fabs(v) > best) {
                best = fabs(v);
                bv = v;
                bi = lane + 32 * ra;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_ip[buf] = best > 0.0 ? bi : -1;
            s_inv[buf] = 1.0 / bv;
        }
    };
    // Column diagonal dominance (with a margin): partial pivoting then takes
    // the diagonal at every step, so the owner of column j+1 publishes it --
    // pivot j+1, no search -- right after the multipliers of step j are known,
    // before its bulk update: the search and the update leave the chain.
    bool dom_ok = true;
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
        const int c = w + NW * cb;
        double off = 0.0, dg = 0.0;
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) {
            const int r = lane + 32 * ra;
            if (r == c) dg = fabs(a[ra][cb]);
            else off += fabs(a[ra][cb]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            dg += __shfl_xor_sync(0xffffffffu, dg, o);
        }
        if (c < n && !(dg > 1.0001 * off)) dom_ok = false;
    }
    const bool dom = __syncthreads_and(dom_ok) != 0;
    if (w == 0) publish(0);
    for (int j = 0; j < n; ++j) {
        __syncthreads();
        const int buf = j & 1;
        const int ip = s_ip[buf];
        if (ip < 0) {
            if (threadIdx.x == 0) flags[J.guard] = 0;
            return;
        }
        const double inv = s_inv[buf];
        if (threadIdx.x == 0) s_perm[j] = ip;
        const int ia = ip >> 5, il = ip & 31;
        // pivot row of this warp's columns, scaled, from its holder lane
#pragma unroll
        for (int ra = 0; ra < RA; ++ra)
            if (ra == ia) {
                if (lane == il) {
#pragma unroll
                    for (int cb = 0; cb < CB; ++cb) s_row[w][cb] = a[ra][cb] * inv;
                }
                if (lane == il) used |= 1u << ra;
            }
        __syncwarp();
        double f[RA];
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) f[ra] = s_col[buf][lane + 32 * ra];
        if (dom && j + 1 < n && w == (j + 1) % NW) {
            const int jb1 = (j + 1) / NW, nb = buf ^ 1;
#pragma unroll
            for (int cb = 0; cb < CB; ++cb)
                if (cb == jb1) {
                    const double u = s_row[w][cb];
#pragma unroll
                    for (int ra = 0; ra < RA; ++ra) {
                        const double v = (ra == ia && lane == il) ? u : fma(-f[ra], u, a[ra][cb]);
                        s_col[nb][lane + 32 * ra] = v;
                        if (lane + 32 * ra == j + 1) {
                            s_ip[nb] = j + 1;
                            s_inv[nb] = 1.0 / v;
                        }
                    }
                }
        }
        // rank-1 elimination on every element (pivot row and column j are
        // rewritten below)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
            const double u = s_row[w][cb];
#pragma unroll
            for (int ra = 0; ra < RA; ++ra) a[ra][cb] = fma(-f[ra], u, a[ra][cb]);
        }
        if (w == j % NW) {  // column j := -s(r, j) / p
            const int jb = j / NW;
#pragma unroll
            for (int cb = 0; cb < CB; ++cb)
                if (cb == jb)
#pragma unroll
                    for (int ra = 0; ra < RA; ++ra) a[ra][cb] = -f[ra] * inv;
        }
#pragma unroll
        for (int ra = 0; ra < RA; ++ra)  // pivot row := s(ip, c) / p, s(ip, j) = 1/p
            if (ra == ia && lane == il) {
#pragma unroll
                for (int cb = 0; cb < CB; ++cb) a[ra][cb] = (w + NW * cb == j) ? inv : s_row[w][cb];
            }
        if (!dom && j + 1 < n && w == (j + 1) % NW) publish(j + 1);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) s_q[s_perm[j]] = j;
    __syncthreads();
    double* out = pool + J.aux;
#pragma unroll
    for (int ra = 0; ra < RA; ++ra)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
            const int r = lane + 32 * ra, c = w + NW * cb;
            if (r < n && c < n) out[(long long)s_perm[c] * n + s_q[r]] = a[ra][cb];
        }
}

bool launch_schur_inverse(const CouplingJob* d_jobs, int njobs, int n, const PartDev* d_parts, const double* fac,
                          double* pool, int* flags, cudaStream_t s) {
    if (njobs <= 0) return true;
#define SPK_SINV(RA, CB)                                                                            \
    if (n <= 32 * RA && n <= 8 * CB) {                                                              \
        k_schur_inverse<RA, CB, 8><<<njobs, 256, 0, s>>>(d_jobs, d_parts, fac, pool, flags);      \
        count_launch();                                                                             \
        return true;                                                                                \
    }
    SPK_SINV(1, 4)
    SPK_SINV(2, 8)
    SPK_SINV(3, 12)
    SPK_SINV(4, 16)
    SPK_SINV(5, 20)
#undef SPK_SINV
    return false;
}

void launch_wcheck(const CouplingJob* d_jobs, int njobs, int k, const double* pool, int* flags, cudaStream_t s) {
    if (njobs <= 0) return;
    k_wcheck_init<<<(njobs + 127) / 128, 128, 0, s>>>(d_jobs, njobs, flags);
    count_launch();
    const int ycta = std::max(1, std::min((k + 7) / 8, 16));  // <= 8 columns per CTA
    k_wcheck<<<dim3(njobs, ycta), 256, 0, s>>>(d_jobs, pool, flags);
    count_launch();
}

void launch_schur_init(const CouplingJob* d_jobs, int njobs, long long max_elems, const PartDev* d_parts,
                       double* fac, int* piv, const int* flags, cudaStream_t s) {
    if (njobs <= 0) return;
    dim3 g((unsigned)std::min<long long>((max_elems + 255) / 256, 256), njobs);
    k_schur_init<<<g, 256, 0, s>>>(d_jobs, d_parts, fac, piv, flags);
    count_launch();
}

void launch_dense_lu(const CouplingJob* d_jobs, int njobs, int n, const PartDev* d_parts, double* fac, int* piv,
                     int* flags, cudaStream_t s) {
    if (njobs <= 0) return;
    const size_t smem = (size_t)n * (n + 1) * 8;
    set_smem_attr((const void*)k_dense_lu, (int)smem);
    k_dense_lu<<<njobs, 512, smem, s>>>(d_jobs, d_parts, fac, piv, flags);
    count_launch();
}

}  // namespace spk
