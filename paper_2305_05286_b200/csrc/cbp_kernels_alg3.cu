// cbp_kernels_alg3.cu -- instantiations of cbp_kernel for ALG 3: flooding BP (comparison schedule).
#include "cbp_kernel.cuh"

namespace cbp {

int launch_alg3(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    return dispatch_alg<3, LaunchFn>(g, &a, grid, st);
}

int occupancy_alg3(const Geometry& g, int* out)
{
    return dispatch_alg<3, OccFn>(g, out);
}

}  // namespace cbp
