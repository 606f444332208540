// cbp_kernels_alg2.cu -- instantiations of cbp_kernel for ALG 2: layered BP (comparison schedule).
#include "cbp_warp.cuh"

namespace cbp {

int launch_alg2(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    if (g.wk) return wdispatch<2>(g, &a, grid, st, nullptr);
    return dispatch_alg<2, LaunchFn>(g, &a, grid, st);
}

int occupancy_alg2(const Geometry& g, int* out)
{
    if (g.wk) return wdispatch<2>(g, nullptr, 0, nullptr, out);
    return dispatch_alg<2, OccFn>(g, out);
}

}  // namespace cbp
