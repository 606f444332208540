// cbp_kernels_alg1.cu -- instantiations of cbp_kernel for ALG 1: normalized min-sum CBP.
#include "cbp_kernel.cuh"

namespace cbp {

int launch_alg1(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    return dispatch_alg<1, LaunchFn>(g, &a, grid, st);
}

int occupancy_alg1(const Geometry& g, int* out)
{
    return dispatch_alg<1, OccFn>(g, out);
}

}  // namespace cbp
