// The C++ drop-in surface (include/spike/*.hpp) links against libspike_b200.so:
// every reference entry point of the hot path is referenced by address, none is
// called (no GPU needed).  Reference headers: proj/include/spike/factorize.hpp,
// solve.hpp, partition.hpp, spike2x2.hpp, band_ops.hpp, band_io.hpp.
#include "spike/band_io.hpp"
#include "spike/band_ops.hpp"
#include "spike/banded_matrix.hpp"
#include "spike/factorize.hpp"
#include "spike/partition.hpp"
#include "spike/solve.hpp"
#include "spike/spike2x2.hpp"

#include <cstdio>

using namespace spike;

int main() {
    const void* fns[] = {
        (const void*)static_cast<SpikeFactorization (*)(const BandedMatrix&, const PartitionPlan&, FactorOptions)>(&factorize),
        (const void*)static_cast<DenseBlock (*)(const SpikeFactorization&, const DenseBlock&, SolveStats*)>(&solve),
        (const void*)static_cast<DenseBlock (*)(const SpikeFactorization&, const DenseBlock&, SolveStats*)>(&transpose_solve),
        (const void*)&reduce_factorize,
        (const void*)&reduced_solve,
        (const void*)&reduced_solve_transpose,
        (const void*)&iterative_refine,
        (const void*)&make_plan,
        (const void*)&distribute_threads,
        (const void*)&compute_ratios,
        (const void*)&compute_sizes,
        (const void*)&gpu_plan,
        (const void*)&band_corner,
        (const void*)&factor_2x2,
        (const void*)&solve_2x2,
        (const void*)&spikes_2x2,
        (const void*)&band_matmul,
        (const void*)&relative_residual,
        (const void*)&band_transpose,
        (const void*)&read_matrix,
        (const void*)&write_matrix,
        (const void*)&calibrate_k,
    };
    int n = 0;
    for (const void* f : fns) n += f != nullptr;
    // host-only objects work without a device
    BandedMatrix a(6, 1, 2);
    a.set(2, 3, 1.5);
    Spike2x2Factors empty;
    std::printf("api surface ok: %d entry points, a(2,3)=%.1f, split=%d\n", n, a.at(2, 3), empty.split());
    return (n == (int)(sizeof(fns) / sizeof(fns[0])) && a.at(2, 3) == 1.5) ? 0 : 1;
}
