// cbp_kernels.cu -- launch dispatch over the decoding algorithms (the kernels are instantiated
// per algorithm in cbp_kernels_alg{0,1,2,3}.cu) and the contract evaluation kernel.
#include "cbp_kernel.cuh"

namespace cbp {

// element-wise evaluation of the contract functions (pin of device vs oracle bits)
__global__ void contract_eval_kernel(int fn, const float* __restrict__ x, float* __restrict__ y, int64_t n,
                                     const float4* __restrict__ tab)
{
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float v = x[k];
        float out;
        if (fn == 0) {
            out = phi32(v, tab);
        } else if (fn == 1) {
            out = ln32(v);
        } else {
            float sn, cs;
            sincos_quarter32(__float_as_uint(v) & 0xffffffu, sn, cs);
            out = (fn == 2) ? sn : cs;
        }
        y[k] = out;
    }
}

int launch_contract_eval(int fn, const float* x, float* y, int64_t n, const float4* tab, void* stream)
{
    if (n <= 0) return 0;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    contract_eval_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(fn, x, y, n, tab);
    return static_cast<int>(cudaGetLastError());
}

int launch_cbp(const KernelArgs& a, const Geometry& g, int grid, void* stream)
{
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (g.alg) {
    case 1: return launch_alg1(a, g, grid, st);
    case 2: return launch_alg2(a, g, grid, st);
    case 3: return launch_alg3(a, g, grid, st);
    default: return launch_alg0(a, g, grid, st);
    }
}

int occupancy_ctas_per_sm(const Geometry& g, int* out)
{
    switch (g.alg) {
    case 1: return occupancy_alg1(g, out);
    case 2: return occupancy_alg2(g, out);
    case 3: return occupancy_alg3(g, out);
    default: return occupancy_alg0(g, out);
    }
}

}  // namespace cbp
