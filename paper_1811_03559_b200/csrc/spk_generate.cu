// spk_generate.cu — seeded BASELINE inputs generated directly in HBM.
//
// Same counter-based generator as the host/oracle side
// (include/spike_b200_gen.h), so device and host materialise bit-identical
// A and F; config 5 (33 GB band) is generated in place with no host copy.
#include "spk_launch.h"

#include "../../include/spike_b200_gen.h"

namespace spk {

__global__ void k_generate_band(unsigned long long seed, long long n, int kl, int ku, double dd,
                                double* __restrict__ band) {
    const int ld = kl + ku + 1;
    const long long total = n * ld;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long j = e / ld;
        const int q = (int)(e - j * ld);
        const long long i = j + q - ku;
        double v = 0.0;
        if (i >= 0 && i < n) v = spk_gen_entry(seed, n, kl, ku, dd, i, j);
        band[e] = v;
    }
}

__global__ void k_generate_rhs(unsigned long long seed, long long n, int ncols,
                               double* __restrict__ F, long long ldf) {
    const long long total = n * ncols;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / n, i = e - c * n;
        F[c * ldf + i] = spk_gen_rhs(seed, i, c);
    }
}

void launch_generate_band(unsigned long long seed, long long n, int kl, int ku, double dd,
                          double* band, cudaStream_t s) {
    k_generate_band<<<148 * 32, 256, 0, s>>>(seed, n, kl, ku, dd, band);
    count_launch();
}

void launch_generate_rhs(unsigned long long seed, long long n, int ncols, double* F, long long ldf,
                         cudaStream_t s) {
    k_generate_rhs<<<148 * 16, 256, 0, s>>>(seed, n, ncols, F, ldf);
    count_launch();
}

}  // namespace spk
