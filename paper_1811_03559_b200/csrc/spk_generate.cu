// spk_generate.cu — seeded BASELINE inputs generated directly in HBM.
//
// Same counter-based generator as the host/oracle side
// (include/spike_b200_gen.h), so device and host materialise bit-identical
// A and F; config 5 (33 GB band) is generated in place with no host copy, and
// each GPU of a multi-GPU run generates its own slab (plus halo columns) of
// the same global matrix.
#include "spk_launch.h"

#include "../../include/spike_b200_gen.h"

namespace spk {

// band columns [col0, col0 + ncols) of the n x n matrix; entries outside the
// matrix (halo columns past either end) are zero
__global__ void k_generate_band(unsigned long long seed, long long n, int kl, int ku, double dd,
                                long long col0, long long ncols, double* __restrict__ band) {
    const int ld = kl + ku + 1;
    const long long total = ncols * ld;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long jl = e / ld, j = col0 + jl;
        const int q = (int)(e - jl * ld);
        const long long i = j + q - ku;
        double v = 0.0;
        if (i >= 0 && i < n && j >= 0 && j < n) v = spk_gen_entry(seed, n, kl, ku, dd, i, j);
        band[e] = v;
    }
}

// F rows [row0, row0 + nrows)
__global__ void k_generate_rhs(unsigned long long seed, long long row0, long long nrows, int ncols,
                               double* __restrict__ F, long long ldf) {
    const long long total = nrows * ncols;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long c = e / nrows, i = e - c * nrows;
        F[c * ldf + i] = spk_gen_rhs(seed, row0 + i, c);
    }
}

void launch_generate_band(unsigned long long seed, long long n, int kl, int ku, double dd, long long col0,
                          long long ncols, double* band, cudaStream_t s) {
    k_generate_band<<<148 * 32, 256, 0, s>>>(seed, n, kl, ku, dd, col0, ncols, band);
    count_launch();
}

void launch_generate_rhs(unsigned long long seed, long long row0, long long nrows, int ncols, double* F,
                         long long ldf, cudaStream_t s) {
    k_generate_rhs<<<148 * 16, 256, 0, s>>>(seed, row0, nrows, ncols, F, ldf);
    count_launch();
}

}  // namespace spk
