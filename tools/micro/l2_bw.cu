// L2 -> SM read bandwidth microbenchmark: can a lattice-split hash read every
// candidate row three times (once per lattice group) from L2?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/l2_bw tools/micro/l2_bw.cu
// Mode 0: LDG.128, every CTA group of `rep` CTAs reads the same 10 KB tiles
//         (the rows of one tile read by `rep` CTAs close together in time).
// Mode 1: the same with 1-D cp.async.bulk of the whole 10 KB tile into SMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(512) ldg_tiles(const uint4* __restrict__ src, int64_t ntiles,
                                                 int tile_u4, int rep, unsigned long long* sink) {
    // CTA b: group g = b / rep walks tiles g, g + ngroups, ...
    const int ngroups = gridDim.x / rep;
    const int g = blockIdx.x / rep;
    uint32_t acc = 0;
    for (int64_t t = g; t < ntiles; t += ngroups) {
        const uint4* p = src + t * tile_u4;
        for (int i = threadIdx.x; i < tile_u4; i += blockDim.x) {
            uint4 v = __ldg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void __launch_bounds__(128) bulk_tiles(const uint4* __restrict__ src, int64_t ntiles,
                                                  int tile_u4, int rep, int stages,
                                                  unsigned long long* sink) {
    extern __shared__ __align__(128) uint4 buf[];
    __shared__ __align__(8) uint64_t bar[8];
    const int ngroups = gridDim.x / rep;
    const int g = blockIdx.x / rep;
    const uint32_t bytes = (uint32_t)tile_u4 * 16u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    int64_t my = 0;
    for (int64_t t = g; t < ntiles; t += ngroups) ++my;
    uint32_t acc = 0;
    auto issue = [&](int64_t k) {
        const int s = (int)(k % stages);
        const int64_t t = g + k * ngroups;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])),
                     "r"(bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(sa(buf + s * tile_u4)),
            "l"(src + t * tile_u4), "r"(bytes), "r"(sa(&bar[s]))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int64_t k = 0; k < stages && k < my; ++k) issue(k);
    for (int64_t k = 0; k < my; ++k) {
        const int s = (int)(k % stages);
        const uint32_t ph = (uint32_t)((k / stages) & 1);
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                sa(&bar[s])),
            "r"(ph)
            : "memory");
        uint4 v = buf[s * tile_u4 + threadIdx.x];
        acc ^= v.x;
        __syncthreads();
        if (threadIdx.x == 0 && k + stages < my) issue(k + stages);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
    const int64_t n_rows = 1ll << 26, row_bytes = 80;
    const int64_t total = n_rows * row_bytes;  // 5.37 GB
    const int tile_u4 = 128 * 80 / 16;         // 640 x 16 B = 10 KB
    const int64_t ntiles = total / (tile_u4 * 16);
    uint4* src;
    unsigned long long* sink;
    cudaMalloc(&src, total);
    cudaMalloc(&sink, 8);
    cudaMemset(src, 1, total);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep : {1, 2, 3, 4}) {
        for (int per_sm : {1, 2, 3}) {
            const int grid = (sms * per_sm / rep) * rep;
            float best = 1e9f;
            for (int it = 0; it < 3; ++it) {
                cudaEventRecord(a);
                ldg_tiles<<<grid, 512>>>(src, ntiles, tile_u4, rep, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("ldg  rep=%d ctas/sm=%d: %.3f ms, SM ingress %.0f GB/s, HBM-unique %.0f GB/s\n",
                   rep, per_sm, best, rep * total / (best * 1e-3) / 1e9,
                   total / (best * 1e-3) / 1e9);
        }
        for (int stages : {2, 4, 8}) {
            const int grid = (sms * 2 / rep) * rep;
            const size_t sm = (size_t)stages * tile_u4 * 16;
            cudaFuncSetAttribute(bulk_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            float best = 1e9f;
            for (int it = 0; it < 3; ++it) {
                cudaEventRecord(a);
                bulk_tiles<<<grid, 128, sm>>>(src, ntiles, tile_u4, rep, stages, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("bulk rep=%d stages=%d: %.3f ms, SM ingress %.0f GB/s, HBM-unique %.0f GB/s (%s)\n",
                   rep, stages, best, rep * total / (best * 1e-3) / 1e9,
                   total / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
