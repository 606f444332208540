// cbp_kernels_alg0.cu -- instantiations of cbp_kernel for ALG 0: CBP log-tanh (producer-side B2V).
#include "cbp_warp.cuh"

namespace cbp {

int launch_alg0(const KernelArgs& a, const Geometry& g, int grid, cudaStream_t st)
{
    if (g.wk) return wdispatch<0>(g, &a, grid, st, nullptr);
    return dispatch_alg<0, LaunchFn>(g, &a, grid, st);
}

int occupancy_alg0(const Geometry& g, int* out)
{
    if (g.wk) return wdispatch<0>(g, nullptr, 0, nullptr, out);
    return dispatch_alg<0, OccFn>(g, out);
}

}  // namespace cbp
