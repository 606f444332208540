// ubench_lookup.cu -- micro-benchmark: random 16-byte table lookups (the phi
// contract v2 access pattern: 929 segments x float4) through shared memory
// (LDS.128, LSU data pipe) versus the texture path (TEX data pipe), alone and
// mixed, to see whether the two pipes add up.  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_lookup.cu && /tmp/ubench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kSegs = 929;

template <int NS, int NT>
__global__ void __launch_bounds__(448, 1) lookups(const float4* __restrict__ tab_g, cudaTextureObject_t tex, int iters,
                                                  float* out)
{
    __shared__ float4 tab[kSegs];
    for (int k = threadIdx.x; k < kSegs; k += blockDim.x) tab[k] = tab_g[k];
    __syncthreads();
    uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    float acc[3] = {0.f, 0.f, 0.f};
    const bool on = (threadIdx.x & 31) < 27;      // 27 of 32 lanes, as C2
    if (on) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    x = x * 1664525u + 1013904223u;
                    const int seg = min(static_cast<int>(x >> 22), kSegs - 1);
                    const float4 v = tab[seg];
                    acc[c] = fmaf(fmaf(fmaf(v.w, acc[c], v.z), acc[c], v.y), 1e-3f, v.x);
                }
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    x = x * 1664525u + 1013904223u;
                    const int seg = min(static_cast<int>(x >> 22), kSegs - 1);
                    const float4 v = tex1Dfetch<float4>(tex, seg);
                    acc[c] = fmaf(fmaf(fmaf(v.w, acc[c], v.z), acc[c], v.y), 1e-3f, v.x);
                }
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2];
}

template <int NS, int NT>
static void run(const char* name, const float4* d_tab, cudaTextureObject_t tex, float* d_out, int nsm)
{
    const int iters = 2000;
    lookups<NS, NT><<<nsm, 448>>>(d_tab, tex, 10, d_out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    lookups<NS, NT><<<nsm, 448>>>(d_tab, tex, iters, d_out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_lookups = static_cast<double>(nsm) * 14 * iters * 3 * (NS + NT);
    std::printf("%-22s %8.3f ms  %.3e warp-lookups/s  %.2f SM-cycles per warp-lookup (at 1.965 GHz)\n", name, ms,
                warp_lookups / (ms * 1e-3), (ms * 1e-3) * 1.965e9 * nsm / warp_lookups);
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<float4> h(kSegs);
    for (int k = 0; k < kSegs; ++k) h[k] = make_float4(1.0f / (k + 1), 0.5f, 0.25f, 0.125f);
    float4* d_tab;
    float* d_out;
    cudaMalloc(&d_tab, sizeof(float4) * kSegs);
    cudaMalloc(&d_out, sizeof(float) * nsm * 448);
    cudaMemcpy(d_tab, h.data(), sizeof(float4) * kSegs, cudaMemcpyHostToDevice);
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = d_tab;
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = sizeof(float4) * kSegs;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    run<2, 0>("smem x2", d_tab, tex, d_out, nsm);
    run<1, 1>("smem x1 + tex x1", d_tab, tex, d_out, nsm);
    run<0, 2>("tex x2", d_tab, tex, d_out, nsm);
    run<1, 0>("smem x1", d_tab, tex, d_out, nsm);
    run<0, 1>("tex x1", d_tab, tex, d_out, nsm);
    run<2, 1>("smem x2 + tex x1", d_tab, tex, d_out, nsm);
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
