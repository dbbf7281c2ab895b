// spk_smallk_solve.cu — the small-k engine's forward solve (k_sk_solve) for
// nrhs <= 8: one cooperative kernel (solve.cpp:81-223).
//
//   D-stage   a warp per partition: the packed factor block lands in shared
//             memory with one TMA bulk copy (cp.async.bulk, mbarrier
//             completion), the right-hand sides with cp.async; forward L and
//             backward U sweeps with lanes = window rows (a step is one
//             shuffle of the pivot row's x and one FMA per column on the rows
//             it updates, the factor entries are shared-memory reads); the
//             tips of Y = D^-1 F go to T.
//   reduced   (reduced_solve, solve.cpp:33-43) level by level, one grid
//             barrier per level.  Phase ph: task A (level ph, a warp per pair)
//             forms z2 = S^-1 (y2 - Wt y1), z1 = y1 - Vb z2 and the merged
//             unit's boundary rows (top k: y - vl_top z2, bottom k:
//             y - wr_bot z1) straight from k x k blocks, so the next level
//             needs nothing else; task B (level ph-1, a CTA per row item)
//             updates the merged units' other rows.  T is updated in place:
//             the two tasks of a phase touch disjoint rows.
//   retrieval a warp per partition, the factor still in shared memory:
//             X_i = A_i^-1 (F_i - B^_i x_top(i+1) - C^_i x_bot(i-1)).
#include "spk_device.cuh"
#include "spk_launch.h"
#include "spk_smallk.cuh"

#include <cuda_runtime.h>

#include <algorithm>

namespace spk {

namespace {
constexpr int kSvWarps = 8;
constexpr int kSvThreads = 32 * kSvWarps;

__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "SKWP_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra SKWP_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// per-warp shared memory (doubles): factor block (+2 alignment slack), 1/u,
// right-hand-side rows, mbarrier
__host__ __device__ inline long long sv_warp_smem(int mmax, int rmax, int nr) {
    return ((long long)mmax * rmax + 2 + mmax + (long long)mmax * nr + 2 + 1) / 2 * 2;
}

struct SvWarp {
    double* Fs;   // packed factor of the staged partition (column j at j * rows)
    double* dv;   // 1 / u_jj
    double* Ys;   // right-hand-side rows (LU space), then the forward results
    unsigned long long* bar;
    unsigned phase;
};

// Stage partition P: the factor block by one bulk copy (16-byte aligned
// window, the odd tail element by a plain load), 1/u_jj from its diagonal.
__device__ void sv_stage_factor(const SkSolveArgs& A, const PartDev& P, SvWarp& w, double*& Fs, int lane) {
    const long long e0 = P.fofs, e1 = P.fofs + (long long)P.m * P.rows;
    const long long a0 = e0 & ~1LL;
    long long a1 = (e1 + 1) & ~1LL;
    if (a1 > A.fac_size) a1 -= 2;
    Fs = w.Fs + (e0 - a0);
    if (lane == 0) {
        const unsigned bytes = (unsigned)((a1 - a0) * 8);
        mbar_expect_tx(w.bar, bytes);
        bulk_g2s(w.Fs, A.fac + a0, bytes, w.bar);
    }
    for (long long e = a1 + lane; e < e1; e += 32) w.Fs[e - a0] = A.fac[e];
    mbar_wait_parity(w.bar, w.phase);
    w.phase ^= 1u;
    __syncwarp();
    for (int j = lane; j < P.m; j += 32) w.dv[j] = 1.0 / Fs[(long long)j * P.rows + P.d];
    __syncwarp();
}

// Forward L then backward U over the partition (LU space) for NR columns of
// Ys (row-major, NR per row).  Forward: row r in lane r mod 32; backward: row
// r in lane (m-1-r) mod 32.  The forward results overwrite Ys; backward values
// of rows j >= bwd_lo go to store(j, c, v).
template <int NR, class Store>
__device__ __forceinline__ void sv_sweeps(const PartDev& P, const double* Fs, const double* dv, double* Ys, int lane,
                                          int bwd_lo, Store store) {
    const unsigned full = 0xffffffffu;
    const int m = P.m, kl = P.kl, ku = P.ku, rows = P.rows, d = P.d;
    double x[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) x[c] = lane < m ? Ys[lane * NR + c] : 0.0;
#pragma unroll 4
    for (int j = 0; j < m; ++j) {
        const int o = (lane - j) & 31;
        const double l = (o >= 1 && o <= kl) ? Fs[(long long)j * rows + d + o] : 0.0;
        double xj[NR];
#pragma unroll
        for (int c = 0; c < NR; ++c) xj[c] = __shfl_sync(full, x[c], j & 31);
        if (o == 0) {
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                Ys[j * NR + c] = xj[c];
                x[c] = j + 32 < m ? Ys[(j + 32) * NR + c] : 0.0;
            }
        } else {
#pragma unroll
            for (int c = 0; c < NR; ++c) x[c] = fma(-l, xj[c], x[c]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NR; ++c) x[c] = m - 1 - lane >= 0 ? Ys[(m - 1 - lane) * NR + c] : 0.0;
#pragma unroll 4
    for (int j = m - 1; j >= bwd_lo; --j) {
        const int o = (lane - (m - 1 - j)) & 31;
        const double u = (o >= 1 && o <= ku) ? Fs[(long long)j * rows + d - o] : 0.0;
        const double r = dv[j];
        double xj[NR];
#pragma unroll
        for (int c = 0; c < NR; ++c) xj[c] = __shfl_sync(full, x[c], (m - 1 - j) & 31) * r;
        if (o == 0) {
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                store(j, c, xj[c]);
                x[c] = j - 32 >= 0 ? Ys[(j - 32) * NR + c] : 0.0;
            }
        } else {
#pragma unroll
            for (int c = 0; c < NR; ++c) x[c] = fma(-u, xj[c], x[c]);
        }
    }
    __syncwarp();
}

// task A of the reduced solve: one warp per pair, lanes 0..15 = rows
template <int NR>
__device__ void sv_pair_task(const SkSolveArgs& A, const SkPair& pr, int pg, int lane) {
    const unsigned full = 0xffffffffu;
    const int k = A.k, nr = A.nrhs;
    const long long H = 2LL * A.p * k;
    const SkUnit uL = A.units[pr.left], uR = A.units[pr.left + 1];
    const int hL = uL.uh, hR = uR.uh, Hu = hL + hR;
    const long long zb = uL.uoff;
    const double* vl = A.pool + uL.voff;
    const double* wr = A.pool + uR.woff;
    const double* si = A.pool + pr.sinv;
    const int r = lane & 15;
    const bool rv = lane < 16 && r < k;
    // every load first: rows of Wt, Vb, S^-1, vl_top, wr_bot; the four tips
    double Wt[16], Vb[16], Si[16], Vt[16], Wb[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        const bool ok = rv && t < k;
        Wt[t] = ok ? wr[(long long)t * hR + r] : 0.0;
        Vb[t] = ok ? vl[(long long)t * hL + hL - k + r] : 0.0;
        Si[t] = ok ? si[(long long)t * k + r] : 0.0;
        Vt[t] = ok ? vl[(long long)t * hL + r] : 0.0;
        Wb[t] = ok ? wr[(long long)t * hR + hR - k + r] : 0.0;
    }
    double y1[NR], y2[NR], yt[NR], yb[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) {
        const bool ok = rv && c < nr;
        const double* Tc = A.T + (long long)c * H + zb;
        y1[c] = ok ? Tc[hL - k + r] : 0.0;
        y2[c] = ok ? Tc[hL + r] : 0.0;
        yt[c] = ok ? Tc[r] : 0.0;
        yb[c] = ok ? Tc[Hu - k + r] : 0.0;
    }
    // row r of M times the vector v (v[t] on lane t)
    auto mv = [&](const double* M, const double* v, double* out) {
#pragma unroll
        for (int c = 0; c < NR; ++c) out[c] = 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
#pragma unroll
            for (int c = 0; c < NR; ++c) out[c] = fma(M[t], __shfl_sync(full, v[c], t), out[c]);
        }
    };
    double a[NR], z2[NR], z1[NR];
    mv(Wt, y1, a);
#pragma unroll
    for (int c = 0; c < NR; ++c) a[c] = y2[c] - a[c];
    mv(Si, a, z2);
    mv(Vb, z2, a);
#pragma unroll
    for (int c = 0; c < NR; ++c) z1[c] = y1[c] - a[c];
    double b[NR];
    mv(Vt, z2, a);
    mv(Wb, z1, b);
    if (rv) {
        double* zp = A.ZS + (long long)pg * 32 * NR;  // [z2 | z1], row t at t * NR
#pragma unroll
        for (int c = 0; c < NR; ++c) {
            zp[r * NR + c] = z2[c];
            zp[16 * NR + r * NR + c] = z1[c];
            if (c >= nr) continue;
            double* Tc = A.T + (long long)c * H + zb;
            Tc[hL - k + r] = z1[c];
            Tc[hL + r] = z2[c];
            Tc[r] = yt[c] - a[c];
            Tc[Hu - k + r] = yb[c] - b[c];
        }
    }
}

// The tree of pair tasks as dataflow (no grid barrier per level): unit u of
// level l complete -> arrive at the consuming pair's counter; the second
// arrival runs that pair at once on the same warp.  Carried units pass through.
template <int NR>
__device__ void sv_tree_from(const SkSolveArgs& A, int l, int u, int lane) {
    const unsigned full = 0xffffffffu;
    while (l < A.nlevels) {
        const SkLevel L = A.levels[l];
        const int a = u >> 1;
        if (a < L.npairs) {
            __syncwarp();
            __threadfence();  // every lane's writes before the arrival
            unsigned c = 0;
            if (lane == 0) c = atomicAdd(A.cnt + L.pair0 + a, 1u);
            c = __shfl_sync(full, c, 0);
            if (c == 0) return;  // the sibling's warp continues
            __threadfence();
            sv_pair_task<NR>(A, A.pairs[L.pair0 + a], L.pair0 + a, lane);
        }
        u = a;
        ++l;
    }
}

// Deferred row updates, after the tree: reduced row r picks up, in level
// order, the update of every level where it is an interior row of its merged
// unit (once interior, always interior; tip and middle rows were written by
// the pair tasks): y -= vl_row z2 (left rows), y -= wr_row z1 (right rows).
template <int NR>
__device__ void sv_row_pass(const SkSolveArgs& A, long long r) {
    const int k = A.k, nr = A.nrhs;
    const long long H = 2LL * A.p * k;
    double y[NR];
    bool any = false;
#pragma unroll
    for (int c = 0; c < NR; ++c) y[c] = c < nr ? A.T[(long long)c * H + r] : 0.0;
    const int u0 = (int)(r / (2 * k));
    for (int l = 0; l < A.nlevels; ++l) {
        const SkLevel L = A.levels[l];
        const int a = (u0 >> l) >> 1;
        if (a >= L.npairs) continue;  // carried unit
        const SkPair pr = A.pairs[L.pair0 + a];
        const int hL = pr.hL, Hu = hL + pr.hR, ro = (int)(r - pr.zb);
        const bool left = ro >= k && ro < hL - k;
        const bool right = ro >= hL + k && ro < Hu - k;
        if (!left && !right) continue;
        any = true;
        const double* M = A.pool + (left ? pr.vl : pr.wr);
        const int hm = left ? hL : pr.hR, rl = left ? ro : ro - hL;
        const double* z = A.ZS + (long long)(L.pair0 + a) * 32 * NR + (left ? 0 : 16 * NR);
        double mrow[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) mrow[t] = t < k ? M[(long long)t * hm + rl] : 0.0;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= k) break;  // (z rows past k are never written)
#pragma unroll
            for (int c = 0; c < NR; ++c) y[c] = fma(-mrow[t], z[t * NR + c], y[c]);
        }
    }
    if (any) {
#pragma unroll
        for (int c = 0; c < NR; ++c)
            if (c < nr) A.T[(long long)c * H + r] = y[c];
    }
}

}  // namespace

template <int NR>
__global__ void __launch_bounds__(kSvThreads, 1) k_sk_solve(SkSolveArgs A) {
    extern __shared__ __align__(16) double sv_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kSvWarps + warp, nwarps = gridDim.x * kSvWarps;
    const int k = A.k, p = A.p, nr = A.nrhs;
    const long long H = 2LL * p * k, kk = (long long)k * k;
    const long long wsm = sv_warp_smem(A.mmax, A.rmax, NR);
    double* const wb = sv_smem + warp * wsm;
    SvWarp w{wb, wb + (long long)A.mmax * A.rmax + 2, wb + (long long)A.mmax * A.rmax + 2 + A.mmax,
             reinterpret_cast<unsigned long long*>(wb + wsm - 2), 0u};
    if (lane == 0) mbar_init1(w.bar);
    __syncwarp();
    double* Fs = nullptr;
    int staged = -1;

    // the right-hand-side rows of partition i (LU space) into Ys, with cp.async
    auto stage_rhs = [&](const PartDev& P) {
        const int m = P.m;
        for (int e = lane; e < m * NR; e += 32) {
            const int r = e / NR, c = e - r * NR;
            const long long pr = P.rev ? (long long)(m - 1 - r) : (long long)r;
            if (c < nr) sk_cp8(w.Ys + e, A.F + (long long)c * A.ldf + P.r0 + pr);
            else w.Ys[e] = 0.0;
        }
        sk_cp_wait_all();
        __syncwarp();
    };

    // ---- D-stage: tips of Y = D^-1 F into T
    for (int i = gw; i < p; i += nwarps) {
        const PartDev P = A.parts[i];
        const int m = P.m;
        const bool first = i == 0, last = i == p - 1;
        sv_stage_factor(A, P, w, Fs, lane);
        staged = i;
        stage_rhs(P);
        double* T = A.T;
        if (first) {
            for (int e = lane; e < k * nr; e += 32) T[(long long)(e / k) * H + (e % k)] = 0.0;  // dead top tip
            sv_sweeps<NR>(P, Fs, w.dv, w.Ys, lane, m - k, [&](int j, int c, double v) {
                if (c < nr) T[(long long)c * H + k + (j - (m - k))] = v;
            });
        } else if (last) {
            for (int e = lane; e < k * nr; e += 32) T[(long long)(e / k) * H + (2LL * i + 1) * k + (e % k)] = 0.0;
            sv_sweeps<NR>(P, Fs, w.dv, w.Ys, lane, m - k, [&](int j, int c, double v) {
                if (c < nr) T[(long long)c * H + 2LL * i * k + (m - 1 - j)] = v;
            });
        } else {
            sv_sweeps<NR>(P, Fs, w.dv, w.Ys, lane, 0, [&](int j, int c, double v) {
                if (c >= nr) return;
                if (j < k) T[(long long)c * H + 2LL * i * k + j] = v;
                else if (j >= m - k) T[(long long)c * H + (2LL * i + 1) * k + (j - (m - k))] = v;
            });
        }
    }
    unsigned target = 0;
    grid_barrier(A.bar, target);

    // ---- reduced solve (solve.cpp:33-43): the tree of pair tasks (dataflow),
    //      then every row's deferred updates
    sk_stamp(A.trace, 0, 0);
    if (A.nlevels > 0) {
        const SkLevel L0 = A.levels[0];
        const int ntask = L0.npairs + (L0.carry >= 0 ? 1 : 0);
        for (int a = gw; a < ntask; a += nwarps) {
            if (a < L0.npairs) sv_pair_task<NR>(A, A.pairs[L0.pair0 + a], L0.pair0 + a, lane);
            sv_tree_from<NR>(A, 1, a, lane);
        }
    }
    sk_stamp(A.trace, 0, 1);
    grid_barrier(A.bar, target);
    sk_stamp(A.trace, 0, 2);
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < H; r += (long long)gridDim.x * blockDim.x)
        sv_row_pass<NR>(A, r);
    grid_barrier(A.bar, target);
    sk_stamp(A.trace, 0, 3);

    // ---- retrieval (solve.cpp:180-223): X_i = A_i^-1 (F_i - B^_i xi - C^_i eta)
    for (int i = gw; i < p; i += nwarps) {
        const PartDev P = A.parts[i];
        const int m = P.m;
        const bool first = i == 0, last = i == p - 1;
        if (staged != i) {
            sv_stage_factor(A, P, w, Fs, lane);
            staged = i;
        }
        stage_rhs(P);
        // boundary rows: physical rows [m-k, m) -= B^ x_top(i+1), [0, k) -= C^ x_bot(i-1)
        const double* bh = A.pool + A.off_bhat + i * kk;
        const double* ch = A.pool + A.off_chat + i * kk;
        for (int e = lane; e < 2 * k * NR; e += 32) {
            const int side = e / (k * NR), q = e - side * k * NR, rr = q / NR, c = q - rr * NR;
            const bool on = c < nr && (side == 0 ? !last : !first);
            const double* M = side == 0 ? bh : ch;
            const double* Tv = A.T + (long long)c * H + (side == 0 ? 2LL * (i + 1) * k : (2LL * i - 1) * k);
            double mv[16], tv[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                mv[t] = (on && t < k) ? M[(long long)t * k + rr] : 0.0;
                tv[t] = (on && t < k) ? Tv[t] : 0.0;
            }
            double v = 0.0;
#pragma unroll
            for (int t = 0; t < 16; ++t) v = fma(mv[t], tv[t], v);
            const int pr = side == 0 ? m - k + rr : rr;
            const int lr = P.rev ? m - 1 - pr : pr;
            if (c < nr) w.Ys[lr * NR + c] -= v;
        }
        __syncwarp();
        sv_sweeps<NR>(P, Fs, w.dv, w.Ys, lane, 0, [&](int j, int c, double v) {
            if (c < nr) A.X[(long long)c * A.ldx + P.r0 + (P.rev ? m - 1 - j : j)] = v;
        });
    }
}

template <int NR>
static void launch_solve_t(const SkSolveArgs& A, cudaStream_t s) {
    const size_t smem = sizeof(double) * (kSvWarps * (size_t)sv_warp_smem(A.mmax, A.rmax, NR) + 2 * 16 * NR);
    set_smem_attr((const void*)k_sk_solve<NR>, (int)smem);
    SkSolveArgs a = A;
    void* args[] = {&a};
    (void)cudaLaunchCooperativeKernel((const void*)k_sk_solve<NR>, device_sms(), kSvThreads, args, smem, s);
    count_launch();  // reports a failed launch
}

size_t sk_solve_smem(int mmax, int rmax, int nrhs) {
    const int nr = nrhs <= 1 ? 1 : nrhs <= 2 ? 2 : nrhs <= 4 ? 4 : 8;
    return sizeof(double) * (kSvWarps * (size_t)sv_warp_smem(mmax, rmax, nr) + 2 * 16 * nr);
}

void launch_sk_solve(const SkSolveArgs& A, cudaStream_t s) {
    if (A.nrhs <= 1) launch_solve_t<1>(A, s);
    else if (A.nrhs <= 2) launch_solve_t<2>(A, s);
    else if (A.nrhs <= 4) launch_solve_t<4>(A, s);
    else launch_solve_t<8>(A, s);
}

}  // namespace spk
