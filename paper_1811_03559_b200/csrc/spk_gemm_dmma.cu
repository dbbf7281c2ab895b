// spk_gemm_dmma.cu — batched FP64 GEMM on the tensor cores (DMMA).
//
// C[crow0+i, c] (=|-=) sum_l opA(A)[i, l] * B[brow0+l, c] for a batch of jobs
// (GemmJob, row-mapped views), i.e. the reference's gemm_minus / gemm_minus_t
// / block_util mul (src/banded_matrix.cpp:39-51, src/block_util.hpp:29-35)
// for the reduced-system spike updates, the coupling Schur complements and the
// retrieval corner products.
//
// sm_100a has no tcgen05 FP64 kind; FP64 tensor math is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA).  CTA tile 64 x TN, K-chunk 16,
// 4 warps each owning a 32 x TN/2 sub-tile = 4 x NB DMMA accumulators; A and B
// chunks are staged through shared memory (cp.async, double-buffered).  TN is
// 64 (NB = 4) or 80 (NB = 5), whichever pads the job's columns less: k = nrhs
// = 160 is two 80-column tiles instead of three 64-column ones (a sixth of
// the tensor work was padding).
#include "spk_device.cuh"

#include <algorithm>
#include "spk_launch.h"
#include "spk_sweep_fast.cuh"

namespace spk {

namespace {
constexpr int TM = 64, TK = 16;
// padded strides (doubles): 20 = 40 words keeps each 16-lane phase of the
// 8-byte fragment loads on distinct banks
constexpr int SA = TK + 4;  // A tile stored [m][k]
constexpr int SB = TK + 4;  // B tile stored [n][k]

// resolved view: element (L, c) at p + (rev ? mrows-1-(L-off) : L-off) + c*ld
struct RV {
    double* p;
    long long ld;
    int rev, off, mrows;
    __device__ __forceinline__ double* at(int L, int c) const {
        return p + (rev ? (mrows - 1 - (L - off)) : (L - off)) + (long long)c * ld;
    }
};
__device__ __forceinline__ RV resolve(const Bufs& B, const View& v) {
    RV r;
    r.p = B.p[v.buf] + v.base;
    r.ld = v.ld >= 0 ? v.ld : B.ld[v.buf];
    r.rev = v.rev;
    r.off = v.off;
    r.mrows = v.mrows;
    return r;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
}  // namespace

// Split-K (ws != nullptr): blockIdx.z takes K range [z*ks, (z+1)*ks) and writes
// its partial tile to ws[((job * tiles + tile) * nsplit + z) * TM*TN]; the
// reduction kernel sums the splits in order (deterministic, no atomics).
// NS = cp.async stages in flight (dynamic shared memory, NS * (TM*SA + TN*SB)
// doubles).  With two stages the warps of the 64 x 80 variant (three CTAs per
// SM) spend 28-30% of their stall samples on the next chunk's loads
// (profiles/r02_gemm_schur_ncu.txt), but three stages measured slower (C3's
// GEMMs 5.73 -> 6.05 ms): both variants run NS = 2.
template <int NB, int NS>
__global__ void __launch_bounds__(128, NB == 5 ? 3 : 4) k_gemm_dmma(const GemmJob* __restrict__ jobs, Bufs B, int ncols,
                                                   double* __restrict__ ws, int nsplit, int tiles_max) {
    constexpr int TN = 16 * NB;
    const GemmJob& Jg = jobs[blockIdx.x];
    if (!guard_ok(B.flags, Jg.guard)) return;
    const int nc = Jg.nc >= 0 ? Jg.nc : ncols;
    const int jr = Jg.r, jkk = Jg.kk, transA = Jg.transA, op = Jg.op, brow0 = Jg.brow0, crow0 = Jg.crow0;
    const int tiles_r = (jr + TM - 1) / TM;
    const int tr = blockIdx.y % tiles_r;
    const int tc = blockIdx.y / tiles_r;
    if (tc * TN >= nc || jr <= 0) return;
    const RV va = resolve(B, Jg.a), vb = resolve(B, Jg.b), vc = resolve(B, Jg.c);
    extern __shared__ __align__(16) double gemm_sm[];
    double* const sA = gemm_sm;                 // [NS][TM * SA]
    double* const sB = gemm_sm + NS * TM * SA;  // [NS][TN * SB]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * (8 * NB);
    const int g = lane >> 2, q = lane & 3;
    const int row0 = tr * TM, col0 = tc * TN;

    // K range of this CTA (whole K unless split)
    int kbeg = 0, kend = jkk;
    if (ws) {
        const int ks = ((jkk + nsplit - 1) / nsplit + TK - 1) / TK * TK;
        kbeg = blockIdx.z * ks;
        kend = min(jkk, kbeg + ks);
    }
    // Staging: each thread keeps its row pointer(s) and steps through the
    // chunk with a constant stride (one add + one bounds test per element
    // instead of a full view resolution).
    auto rowp = [](const RV& v, int L) -> const double* {
        return v.p + (v.rev ? (v.mrows - 1 - (L - v.off)) : (L - v.off));
    };
    // A, not transposed: thread -> row i = tid & 63, k offsets (tid >> 6) + 2 j
    const int a_i = tid & (TM - 1), a_l = tid >> 6;
    const bool a_rok = row0 + a_i < jr;
    const double* a_row = transA ? nullptr : rowp(va, a_rok ? row0 + a_i : 0);
    // A transposed (A is kk x r): thread -> k offset tid & 15, rows (tid >> 4) + 8 j
    const int t_l = tid & (TK - 1), t_i = tid >> 4;
    // B: thread -> k offset tid & 15, columns (tid >> 4) + 8 j
    const int b_l = tid & (TK - 1), b_c = tid >> 4;
    auto stage = [&](int buf, int k0) {
        if (!transA) {
            const double* src = a_row + (long long)(k0 + a_l) * va.ld;
#pragma unroll
            for (int j = 0; j < TK / 2; ++j) {
                const int l = a_l + 2 * j;
                double* dst = &sA[buf * TM * SA + a_i * SA + l];
                if (a_rok && k0 + l < kend) cp_async8(dst, src + (long long)(2 * j) * va.ld);
                else *dst = 0.0;
            }
        } else {
            const bool lok = k0 + t_l < kend;
            const double* src = rowp(va, lok ? k0 + t_l : 0) + (long long)row0 * va.ld;
#pragma unroll
            for (int j = 0; j < TM / 8; ++j) {
                const int i = t_i + 8 * j;
                double* dst = &sA[buf * TM * SA + i * SA + t_l];
                if (lok && row0 + i < jr) cp_async8(dst, src + (long long)i * va.ld);
                else *dst = 0.0;
            }
        }
        {
            const bool lok = k0 + b_l < kend;
            const double* src = rowp(vb, brow0 + (lok ? k0 + b_l : 0)) + (long long)col0 * vb.ld;
#pragma unroll
            for (int j = 0; j < TN / 8; ++j) {
                const int c = b_c + 8 * j;
                double* dst = &sB[buf * TN * SB + c * SB + b_l];
                if (lok && col0 + c < nc) cp_async8(dst, src + (long long)c * vb.ld);
                else *dst = 0.0;
            }
        }
        cp_async_commit();
    };

    double acc[4][NB][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    const int nk = kend > kbeg ? (kend - kbeg + TK - 1) / TK : 0;
    // NS - 1 chunks in flight; one commit group per chunk slot (empty past the end)
#pragma unroll
    for (int c = 0; c < NS - 1; ++c) {
        if (c < nk) stage(c, kbeg + c * TK);
        else cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc % NS;
        if (kc + NS - 1 < nk) stage((kc + NS - 1) % NS, kbeg + (kc + NS - 1) * TK);
        else cp_async_commit();
        cp_async_wait<NS - 1>();
        __syncthreads();
        const double* a_s = sA + buf * TM * SA;
        const double* b_s = sB + buf * TN * SB;
#pragma unroll
        for (int ks = 0; ks < TK; ks += 4) {
            double af[4], bf[NB];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = a_s[(wm + 8 * a + g) * SA + ks + q];
#pragma unroll
            for (int b = 0; b < NB; ++b) bf[b] = b_s[(wn + 8 * b + g) * SB + ks + q];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < NB; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        __syncthreads();
    }
    if (ws) {
        // split-K: every split stores its partial tile; the last split to
        // arrive (per-tile counter) sums them in split order -- deterministic --
        // and applies the epilogue, then re-arms the counter
        const size_t tile_id = (size_t)blockIdx.x * tiles_max + blockIdx.y;
        double* tile = ws + tile_id * nsplit * (TM * TN);
        double* part = tile + (size_t)blockIdx.z * (TM * TN);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b)
                *reinterpret_cast<double2*>(part + (wm + 8 * a + g) * TN + wn + 8 * b + 2 * q) =
                    make_double2(acc[a][b][0], acc[a][b][1]);
        __threadfence();
        __syncthreads();
        __shared__ int s_last;
        if (tid == 0) {
            int* cnt = reinterpret_cast<int*>(ws + (size_t)gridDim.x * tiles_max * nsplit * (TM * TN)) + tile_id;
            s_last = atomicAdd(cnt, 1) == nsplit - 1;
            if (s_last) *cnt = 0;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        // this thread's fragment positions again, summed over the splits in
        // order (all 32 loads of a split in flight), then the epilogue below
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        for (int z = 0; z < nsplit; ++z) {
            const double* pz = tile + (size_t)z * (TM * TN);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    const double2 v = __ldcg(reinterpret_cast<const double2*>(pz + (wm + 8 * a + g) * TN + wn + 8 * b + 2 * q));
                    acc[a][b][0] += v.x;
                    acc[a][b][1] += v.y;
                }
        }
    }
    // epilogue: C[row, col] with row = wm+8a+g, col = wn+8b+2q+{0,1}.  All of
    // C's old values are loaded before the first store: interleaved
    // load-subtract-store through computed pointers would serialise on
    // possible aliasing, one memory latency per element.
    // element (i0 + 8a, c0 + 8b + e) of C sits at P0 + 8a*sr + (8b+e)*ld
    const int i0 = row0 + wm + g, c0 = col0 + wn + 2 * q;
    const long long ld = vc.ld;
    const int sr = vc.rev ? -1 : 1;
    double* const P0 = vc.p + (vc.rev ? (vc.mrows - 1 - (crow0 + i0 - vc.off)) : (crow0 + i0 - vc.off)) +
                       (long long)c0 * ld;
    if (op != GM_SET) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (i0 + 8 * a < jr && c0 + 8 * b + e < nc)
                        acc[a][b][e] = P0[8 * a * sr + (8 * b + e) * ld] - acc[a][b][e];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (i0 + 8 * a < jr && c0 + 8 * b + e < nc) P0[8 * a * sr + (8 * b + e) * ld] = acc[a][b][e];
}

// the column tile that pads max_nc less (64 on ties)
static int gemm_tn(int max_nc) {
    const int p64 = (max_nc + 63) / 64 * 64, p80 = (max_nc + 79) / 80 * 80;
    return p80 < p64 ? 80 : 64;
}

int gemm_splitk_factor(int njobs, int max_r, int max_nc, int max_kk) {
    // few output tiles over a long K (the transposed reduced-system updates):
    // spread K over CTAs, ~512 per split, enough CTAs for the SMs
    const int TN = gemm_tn(max_nc);
    const long long tiles = (long long)njobs * ((max_r + TM - 1) / TM) * ((max_nc + TN - 1) / TN);
    if (max_kk < 1024 || tiles >= 296) return 1;
    int ns = (max_kk + 511) / 512;
    ns = (int)std::min<long long>(ns, (592 + tiles - 1) / tiles);
    return std::max(1, std::min(ns, 64));
}

// doubles: partial tiles, then one int counter per output tile
size_t gemm_splitk_workspace(int njobs, int max_r, int max_nc, int nsplit) {
    const int TN = gemm_tn(max_nc);
    const size_t tiles = (size_t)((max_r + TM - 1) / TM) * ((max_nc + TN - 1) / TN);
    return (size_t)njobs * tiles * nsplit * TM * TN + ((size_t)njobs * tiles + 1) / 2;
}

void launch_gemm_dmma(const GemmJob* d_jobs, int njobs, int max_r, int max_nc, const Bufs& B, int ncols,
                      cudaStream_t s, double* ws, int nsplit) {
    if (njobs <= 0 || max_r <= 0 || max_nc <= 0) return;
    const int TN = gemm_tn(max_nc);
    const int tr = (max_r + TM - 1) / TM, tc = (max_nc + TN - 1) / TN;
    auto* fn = TN == 80 ? k_gemm_dmma<5, 2> : k_gemm_dmma<4, 2>;
    const int smem = 2 * (TM * SA + TN * SB) * (int)sizeof(double);
    set_smem_attr((const void*)fn, smem);
    if (ws && nsplit > 1) {
        const size_t tiles = (size_t)njobs * tr * tc;
        cudaMemsetAsync(ws + tiles * nsplit * TM * TN, 0, sizeof(int) * tiles, s);  // split counters
        dim3 g(njobs, tr * tc, nsplit);
        fn<<<g, 128, smem, s>>>(d_jobs, B, ncols, ws, nsplit, tr * tc);
        count_launch();
        return;
    }
    dim3 g(njobs, tr * tc);
    fn<<<g, 128, smem, s>>>(d_jobs, B, ncols, nullptr, 1, tr * tc);
    count_launch();
}

}  // namespace spk
