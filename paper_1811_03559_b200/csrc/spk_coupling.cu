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
//   k_dense_lu    partial-pivot LU of S in shared memory, LAPACK/gbtf2 row
//                 interchange convention (earlier L columns not swapped), one
//                 CTA per pair; an exactly zero column clears the flag so the
//                 generic path reproduces the reference's boosted fallback.
#include "spk_device.cuh"
#include "spk_launch.h"

#include <cfloat>

namespace spk {

// flag[g] = (max |W| <= 1) for the top k x k tip of wr (h x k, ld h)
__global__ void k_wcheck(const CouplingJob* __restrict__ jobs, const double* __restrict__ pool,
                         int* __restrict__ flags) {
    const CouplingJob J = jobs[blockIdx.x];
    const int k = J.k;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    int mybad = 0;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int c = e / k, r = e - c * k;
        if (fabs(pool[J.wr_off + (long long)c * J.hR + r]) > 1.0) mybad = 1;
    }
    if (mybad) atomicOr(&bad, 1);
    __syncthreads();
    if (threadIdx.x == 0) flags[J.guard] = bad ? 0 : 1;
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

void launch_wcheck(const CouplingJob* d_jobs, int njobs, const double* pool, int* flags, cudaStream_t s) {
    if (njobs <= 0) return;
    k_wcheck<<<njobs, 256, 0, s>>>(d_jobs, pool, flags);
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
    cudaFuncSetAttribute(k_dense_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_dense_lu<<<njobs, 512, smem, s>>>(d_jobs, d_parts, fac, piv, flags);
    count_launch();
}

}  // namespace spk
