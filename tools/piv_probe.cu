// piv_probe.cu -- phase timing of the blocked pivoted DMMA band LU (CTA 0's
// panel-critical warp: the one that updates and then factors the next panel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSPK_PIV_PROFILE \
//        -o tools/piv_probe tools/piv_probe.cu && tools/piv_probe [m] [k] [nparts]
// Slots: 6 barrier wait, 0 swaps, 7 U12 solve + B fragments, 1 DMMA update +
// shift, 2 panel -> row layout, 3 panel columns, 4 publish, 5 entering block.
#include "../paper_1811_03559_b200/csrc/spk_lu_piv_dmma.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace spk {
void count_launch(int) {}
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 6757;
    const int k = argc > 2 ? atoi(argv[2]) : 64;
    const int nparts = argc > 3 ? atoi(argv[3]) : 148;
    const int ld = 2 * k + 1;
    const long long n = (long long)m * nparts;
    std::vector<double> band((size_t)ld * n, 0.0);
    unsigned long long st = 12345;
    auto rnd = [&] { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return (double)(st >> 11) / 9007199254740992.0 * 2 - 1; };
    for (long long j = 0; j < n; ++j)
        for (int q = 0; q < ld; ++q) {
            const long long i = j + q - k;
            if (i < 0 || i >= n) continue;
            band[j * ld + q] = rnd();
        }
    const int ubw = 2 * k, rows = ubw + k + 1;
    std::vector<spk::PartDev> parts(nparts);
    std::vector<int> units(nparts);
    for (int i = 0; i < nparts; ++i) {
        spk::PartDev P{};
        P.r0 = (long long)i * m;
        P.m = m;
        P.kl = P.ku = k;
        P.ubw = ubw;
        P.d = ubw;
        P.rows = rows;
        P.fofs = (long long)i * m * rows;
        P.bofs = -1;
        P.tofs = (long long)i * m * (k + ubw + 1);
        P.rowsT = k + ubw + 1;
        P.guard = -1;
        P.pivoting = 1;
        parts[i] = P;
        units[i] = i;
    }
    double *dband, *dfac, *dtfac, *ddinv;
    int *dpiv, *dstatus, *dunits;
    spk::PartDev* dparts;
    cudaMalloc(&dband, band.size() * 8);
    cudaMalloc(&dfac, (size_t)n * rows * 8);
    cudaMalloc(&dpiv, n * 4);
    cudaMalloc(&dtfac, (size_t)n * (k + ubw + 1) * 8);
    cudaMalloc(&ddinv, n * 8);
    cudaMalloc(&dstatus, 4);
    cudaMalloc(&dunits, nparts * 4);
    cudaMalloc(&dparts, nparts * sizeof(spk::PartDev));
    cudaMemcpy(dband, band.data(), band.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dunits, units.data(), nparts * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dparts, parts.data(), nparts * sizeof(spk::PartDev), cudaMemcpyHostToDevice);
    cudaMemset(dstatus, 0, 4);
    spk::PivDmmaArgs A{dunits, dparts, dband, k, k, dfac, dtfac, ddinv, dpiv, dstatus};
    for (int rep = 0; rep < 3; ++rep) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(spk::g_piv_prof, z, sizeof(z));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (!spk::launch_band_lu_piv_dmma(nparts, k, k, A, 0)) return 1;
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[8];
        cudaMemcpyFromSymbol(h, spk::g_piv_prof, sizeof(h));
        int status = 0;
        cudaMemcpy(&status, dstatus, 4, cudaMemcpyDeviceToHost);
        const double steps = (m + 7) / 8;
        printf("m=%d k=%d parts=%d: %.3f ms, status %d (%s); cycles/step:", m, k, nparts, ms, status,
               cudaGetErrorString(cudaGetLastError()));
        const char* nm[8] = {"swaps", "dmma+shift", "toRows", "columns", "publish", "loads", "barrier", "trsm+conv"};
        for (int i = 0; i < 8; ++i) printf(" %s %.0f", nm[i], h[i] / steps);
        printf("\n");
    }
    return 0;
}
