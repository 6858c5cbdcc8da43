// Modular injectivity of candidate rows (the prime search of next_valid_prime,
// lattice.py:114-125) on the device.
//
// Replaces _core.rows_injective_mod (_core.pyx:103-144: packed int64 codes +
// open addressing) and its numpy lexsort fallback (fallback.py:78-103) with a
// lock-free open-addressing table of row ids: each row's reduced coordinates
// are hashed; a slot is claimed with atomicCAS; a probe that meets an
// occupied slot compares the full reduced rows, so the answer is exact for
// any d and p (no 62-bit packing limit).
#include "common.cuh"

namespace sfftb {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ int64_t redmod(int64_t v, int64_t p) {
    int64_t r = v % p;
    return r < 0 ? r + p : r;
}

__global__ void inject_kernel(const int64_t* __restrict__ elems, int64_t n, int d, int64_t p,
                              unsigned long long* __restrict__ table, uint64_t mask,
                              int* __restrict__ dup) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (*(volatile int*)dup) return;
        const int64_t* row = elems + i * d;
        uint64_t h = 0x9E3779B97F4A7C15ull;
        for (int j = 0; j < d; ++j) h = mix64(h ^ (uint64_t)redmod(row[j], p));
        uint64_t slot = h & mask;
        while (true) {
            const unsigned long long prev =
                atomicCAS(table + slot, 0ull, (unsigned long long)(i + 1));
            if (prev == 0ull) break;
            const int64_t* other = elems + (int64_t)(prev - 1) * d;
            bool same = true;
            for (int j = 0; j < d && same; ++j) same = redmod(row[j], p) == redmod(other[j], p);
            if (same) {
                atomicExch(dup, 1);
                return;
            }
            slot = (slot + 1) & mask;
        }
    }
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int sfftb_injective_mod_dev(const int64_t* elems, int64_t n, int64_t d, int64_t p,
                                       int* injective, void* stream) {
    SFFTB_REQUIRE(p >= 1 && n >= 0 && d >= 0, "injective: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 1) {
        *injective = 1;
        return SFFTB_OK;
    }
    if (d == 0) {
        *injective = 0;
        return SFFTB_OK;
    }
    uint64_t size = 1;
    while (size < (uint64_t)(2 * n)) size <<= 1;
    unsigned long long* table = nullptr;
    int* dup = nullptr;
    SFFTB_CUDA(cudaMallocAsync((void**)&table, size * sizeof(unsigned long long), st));
    SFFTB_CUDA(cudaMallocAsync((void**)&dup, sizeof(int), st));
    SFFTB_CUDA(cudaMemsetAsync(table, 0, size * sizeof(unsigned long long), st));
    SFFTB_CUDA(cudaMemsetAsync(dup, 0, sizeof(int), st));
    const int blocks = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 8);
    inject_kernel<<<blocks, 256, 0, st>>>(elems, n, (int)d, p, table, size - 1, dup);
    SFFTB_CHECK_LAUNCH();
    int h_dup = 0;
    SFFTB_CUDA(cudaMemcpyAsync(&h_dup, dup, sizeof(int), cudaMemcpyDeviceToHost, st));
    SFFTB_CUDA(cudaFreeAsync(table, st));
    SFFTB_CUDA(cudaFreeAsync(dup, st));
    SFFTB_CUDA(cudaStreamSynchronize(st));
    *injective = h_dup ? 0 : 1;
    return SFFTB_OK;
}
