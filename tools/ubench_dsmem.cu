// ubench_dsmem.cu -- micro-benchmark for SURVEY NEXT-2 (C4 state in cluster DSMEM):
// random 4-byte accesses of the C4 state pattern served from (a) the CTA's own shared
// memory, (b) a peer CTA's shared memory in a 4-CTA cluster (distributed shared memory,
// ld.shared::cluster), (c) global memory with an L1-resident footprint, (d) global
// memory with an L2-resident footprint, (e) an HBM footprint (C4's global state, 207 MB, lies between).
// Latency: one warp, dependent pointer chase.  Throughput: 12 warps per SM (one C4
// team) issuing independent loads.  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_dsmem tools/ubench_dsmem.cu && /tmp/ubench_dsmem
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

constexpr int kWords = 48 * 1024;          // 192 KB of shared memory per CTA
constexpr int kClusterSize = 4;

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

// MODE 0 own smem, 1 peer smem (cluster rank + 1), 2 global
template <int MODE, bool CHASE>
__global__ void __cluster_dims__(kClusterSize, 1, 1) __launch_bounds__(384, 1)
    probe(const uint32_t* g, uint32_t gmask, int iters, unsigned long long* cycles, uint32_t* sink)
{
    extern __shared__ uint32_t sm[];
    cg::cluster_group cl = cg::this_cluster();
    if (MODE != 2)
        for (int k = threadIdx.x; k < kWords; k += blockDim.x) sm[k] = hash(k + 17u * blockIdx.x) % kWords;
    cl.sync();
    const uint32_t* src = sm;
    if (MODE == 1) src = cl.map_shared_rank(sm, (cl.block_rank() + 1) % kClusterSize);
    uint32_t x = hash(threadIdx.x + 977u * blockIdx.x) % kWords, acc = 0;
    const long long t0 = clock64();
    if (CHASE) {
        for (int it = 0; it < iters; ++it) {
            if (MODE == 2) {   // volatile asm: not reordered against the clock64 reads
                asm volatile("ld.global.u32 %0, [%1];" : "=r"(x) : "l"(g + (x & gmask)));
            } else {
                x = src[x];
            }
        }
        acc = x;
    } else {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t idx = hash(x + it * 8 + u);
                acc += (MODE == 2) ? g[idx & gmask] : src[idx % kWords];
            }
        }
    }
    const long long t1 = clock64();
    cl.sync();                                   // peers stay resident while read
    if (threadIdx.x == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE, bool CHASE>
static int run(const char* what, const uint32_t* g, uint32_t gmask, int threads, int blocks, int iters, int loads_per_iter)
{
    auto k = probe<MODE, CHASE>;
    const int smem = (MODE == 2) ? 0 : kWords * 4;   // global modes keep the L1 share of the SM's 256 KB
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* cyc;
    uint32_t* sink;
    CK(cudaMalloc(&cyc, sizeof(unsigned long long) * blocks));
    CK(cudaMalloc(&sink, 4));
    k<<<blocks, threads, smem>>>(g, gmask, iters / 10, cyc, sink);   // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, threads, smem>>>(g, gmask, iters, cyc, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(blocks);
    cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto c : h) avg += static_cast<double>(c);
    avg /= blocks;
    const double loads = static_cast<double>(iters) * loads_per_iter;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    if (CHASE)
        std::printf("%-34s latency %7.1f cycles per dependent load (clock64; %.0f from the kernel time)\n", what,
                    avg / loads, ms * 1e-3 * khz * 1e3 / loads);
    else
        std::printf("%-34s %6.2f loads/clk/SM (%d warps/SM)   %.1f G loads/s\n", what,
                    loads * threads / avg, threads / 32, loads * threads * blocks / (ms * 1e6));
    cudaFree(cyc);
    cudaFree(sink);
    return 0;
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = nsm / kClusterSize * kClusterSize;
    // footprints: 64 KB (L1), 32 MB (L2), 512 MB (HBM; C4's 2 x 148 x 0.7 MB = 207 MB lies between)
    const size_t l1_words = 16 * 1024, l2_words = size_t(1) << 23, big_words = size_t(1) << 27;
    uint32_t* g;
    CK(cudaMalloc(&g, big_words * 4));
    std::vector<uint32_t> h(big_words);
    // next index = full-period LCG (chase over the whole footprint, masked per mode)
    for (size_t k = 0; k < big_words; ++k) h[k] = static_cast<uint32_t>((k * 2654435761ull + 12345ull) & (big_words - 1));
    CK(cudaMemcpy(g, h.data(), big_words * 4, cudaMemcpyHostToDevice));
    const int it = 4000;
    // latency: one warp per CTA
    run<0, true>("own smem (LDS)", g, 0, 32, blocks, it, 1);
    run<1, true>("peer smem, 4-CTA cluster (DSMEM)", g, 0, 32, blocks, it, 1);
    run<2, true>("global, 64 KB footprint (L1)", g, l1_words - 1, 32, blocks, it, 1);
    run<2, true>("global, 32 MB footprint (L2)", g, static_cast<uint32_t>(l2_words - 1), 32, blocks, it, 1);
    run<2, true>("global, 512 MB footprint (HBM)", g, static_cast<uint32_t>(big_words - 1), 32, blocks, it / 4, 1);
    // throughput: 12 warps per SM, 8 independent loads per iteration
    run<0, false>("own smem (LDS)", g, 0, 384, blocks, it / 4, 8);
    run<1, false>("peer smem (DSMEM)", g, 0, 384, blocks, it / 4, 8);
    run<2, false>("global, 64 KB footprint (L1)", g, l1_words - 1, 384, blocks, it / 4, 8);
    run<2, false>("global, 32 MB footprint (L2)", g, static_cast<uint32_t>(l2_words - 1), 384, blocks, it / 4, 8);
    run<2, false>("global, 512 MB footprint (HBM)", g, static_cast<uint32_t>(big_words - 1), 384, blocks, it / 4, 8);
    cudaFree(g);
    return 0;
}
