// lu_probe.cu -- phase timing of the blocked DMMA band LU on one partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPK_LU_PROFILE \
//        -o tools/lu_probe tools/lu_probe.cu && tools/lu_probe [m] [k] [parts] [tma 0/1] [row-major copy 0/1]
// Prints the per-step clock totals of CTA 0, summed over its warps (slot 3/4:
// the warp publishing the panel row and factoring the next diagonal block).
#include "../paper_1811_03559_b200/csrc/spk_lu_fast.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace spk {
void count_launch(int) {}
void set_smem_attr(const void* fn, int bytes) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 108108;
    const int k = argc > 2 ? atoi(argv[2]) : 128;
    const int ld = 2 * k + 1, nparts = argc > 3 ? atoi(argv[3]) : 1;
    std::vector<double> band((size_t)ld * m * nparts, 0.0);
    unsigned long long st = 12345;
    auto rnd = [&] { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return (double)(st >> 11) / 9007199254740992.0 * 2 - 1; };
    const long long n = (long long)m * nparts;
    std::vector<double> rs(n, 0.0);
    for (long long j = 0; j < n; ++j)
        for (int q = 0; q < ld; ++q) {
            const long long i = j + q - k;
            if (i < 0 || i >= n || i == j) continue;
            const double v = rnd();
            band[j * ld + q] = v;
            rs[i] += fabs(v);
        }
    for (long long j = 0; j < n; ++j) band[j * ld + k] = 1.5 * rs[j] * (rnd() < 0 ? -1 : 1);
    std::vector<spk::PartDev> parts(nparts);
    std::vector<int> units(nparts);
    for (int i = 0; i < nparts; ++i) {
        spk::PartDev P{};
        P.r0 = (long long)i * m;
        P.m = m;
        P.kl = P.ku = k;
        P.ubw = k;
        P.d = k;
        P.rows = 2 * k + 1;
        P.rowsT = 2 * k + 1;
        P.fofs = (long long)i * m * P.rows;
        P.tofs = (long long)i * m * P.rowsT;
        P.trunc = 0;
        P.bofs = -1;
        P.guard = -1;
        parts[i] = P;
        units[i] = i;
    }
    double *d_band, *d_fac, *d_tfac, *d_dinv;
    int *d_piv, *d_boost, *d_units;
    spk::PartDev* d_parts;
    cudaMalloc(&d_band, sizeof(double) * band.size());
    cudaMalloc(&d_fac, sizeof(double) * n * ld);
    cudaMalloc(&d_tfac, sizeof(double) * n * ld);
    cudaMalloc(&d_dinv, sizeof(double) * n);
    cudaMalloc(&d_piv, sizeof(int) * n);
    cudaMalloc(&d_boost, sizeof(int) * nparts);
    cudaMalloc(&d_units, sizeof(int) * nparts);
    cudaMalloc(&d_parts, sizeof(spk::PartDev) * nparts);
    cudaMemcpy(d_band, band.data(), sizeof(double) * band.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_parts, parts.data(), sizeof(spk::PartDev) * nparts, cudaMemcpyHostToDevice);
    cudaMemcpy(d_units, units.data(), sizeof(int) * nparts, cudaMemcpyHostToDevice);
    cudaMemset(d_boost, 0, sizeof(int) * nparts);
    spk::FastLuArgs A{d_units, d_parts, d_band, k, k, d_fac, d_tfac, d_dinv, d_piv, 1.49e-8, d_boost, n, 0};
    if (argc > 4 && atoi(argv[4]) == 0) A.ncols = 0;  // element-path staging only
    if (argc > 5 && atoi(argv[5]) == 0) A.tfac = nullptr;  // no row-major copy (factorizations without transposed solves)
    {
        CUtensorMap a, b;
        printf("TMA staging: %s\n", spk::band_tensor_maps(A, 170, 10, 168, &a, &b) >= 0 ? "yes" : "no");
    }
#if defined(SPK_LU_PROFILE) || defined(SPK_LU_DBG)
    {
        const int dbg = getenv("LU_DBG") ? atoi(getenv("LU_DBG")) : 0;
        cudaMemcpyToSymbol(spk::g_lu_dbg, &dbg, sizeof(int));
    }
#endif
    int* h_where = nullptr;
#ifdef SPK_LU_PROFILE
    if (getenv("LU_WHERE")) {  // last (step, mark) per warp in mapped host memory (survives a fault)
        cudaHostAlloc(&h_where, sizeof(int) * 32 * nparts, cudaHostAllocMapped);
        for (int i = 0; i < 32 * nparts; ++i) h_where[i] = -1;
        int* dw = nullptr;
        cudaHostGetDevicePointer(&dw, h_where, 0);
        cudaMemcpyToSymbol(spk::g_lu_where, &dw, sizeof(dw));
    }
#endif
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[8] = {0};
#ifdef SPK_LU_PROFILE
        cudaMemcpyToSymbol(spk::g_lu_prof, z, sizeof(z));
#endif
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        spk::launch_band_lu_fast(d_units, nparts, k, A, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long pr[8] = {0};
#ifdef SPK_LU_PROFILE
        cudaMemcpyFromSymbol(pr, spk::g_lu_prof, sizeof(pr));
#endif
        const int steps = (m + 7) / 8, nw = (k + 7) / 8;  // NW = T - 1 warps, T = k/8 + 1
        std::vector<int> bc(nparts);
        cudaMemcpy(bc.data(), d_boost, sizeof(int) * nparts, cudaMemcpyDeviceToHost);
        long long nb = 0;
        for (int v : bc) nb += v;
        if (h_where && cudaGetLastError() != cudaSuccess) {
            for (int b = 0; b < nparts && b < 6; ++b) {
                printf("  cta %d:", b);
                for (int w = 0; w < (k + 7) / 8; ++w) printf(" %d/%d", h_where[b * 32 + w] >> 4, h_where[b * 32 + w] & 15);
                printf("\n");
            }
        }
        printf("m=%d k=%d parts=%d: %.3f ms, %.0f clk/step (wall at 1.965 GHz) boosts=%lld err=%s\n", m, k, nparts, ms,
               ms * 1e-3 * 1.965e9 / steps, nb, cudaGetErrorString(cudaGetLastError()));
        const char* names[8] = {"stage issue", "phase 1 (1a+1b)", "S1 wait", "ro1 publish+reload",
                                "ro1 diag update+factor", "update+shift", "outputs", "S0 wait"};
        for (int i = 0; i < 8; ++i)
            printf("  %-24s %8.0f clk/step per warp\n", names[i], (double)pr[i] / steps / (i == 3 || i == 4 ? 1 : nw));
    }
    return 0;
}
