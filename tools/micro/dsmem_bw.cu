// DSMEM bandwidth microbenchmark (cluster all-to-all 16-byte stores / loads).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) bw_store(int iters, double* sink) {
    extern __shared__ double2 buf[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    const int n = 4096;  // double2 per CTA (64 KB)
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_double2(rank, i);
    cl.sync();
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int dst = (rank + 1 + (it % (CS - 1))) % CS;
        double2* remote = cl.map_shared_rank(buf, dst);
        for (int i = threadIdx.x; i < n; i += blockDim.x) remote[(i + it) & (n - 1)] = make_double2(it, i);
        cl.sync();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += buf[i].x;
    if (acc == -1.0) sink[0] = acc;
}

template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) bw_load(int iters, double* sink) {
    extern __shared__ double2 buf[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    const int n = 4096;
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_double2(rank, i);
    cl.sync();
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int src = (rank + 1 + (it % (CS - 1))) % CS;
        const double2* remote = cl.map_shared_rank(buf, src);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double2 v = remote[(i * 7 + it) & (n - 1)];
            acc += v.x + v.y;
        }
        cl.sync();
    }
    if (acc == -1.0) sink[0] = acc;
}

template <typename K>
void run(K kern, int cs, const char* name) {
    double* sink;
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int blocks = (148 / cs) * cs;
    const int iters = 200;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, 512, 65536>>>(10, sink);
    cudaEventRecord(a);
    kern<<<blocks, 512, 65536>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)blocks * iters * 65536.0;
    printf("%s cluster=%d blocks=%d: %.3f ms, %.1f GB/s total, %.1f B/clk/SM @1.9GHz err=%s\n", name,
           cs, blocks, ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / blocks / 1.9e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run(bw_store<2>, 2, "store");
    run(bw_store<4>, 4, "store");
    run(bw_store<8>, 8, "store");
    run(bw_load<2>, 2, "load");
    run(bw_load<4>, 4, "load");
    run(bw_load<8>, 8, "load");
    return 0;
}
