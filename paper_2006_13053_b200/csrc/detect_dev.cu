// detect_frequencies / detect_and_compute on device buffers as ONE C-ABI call
// (reference detect.py:149-169 over _gather, :122-146): finiteness check of
// the samples, zero test (detect.py:42-53), the L prime-length DFTs, nonzero
// bitmaps, hashing + hit counts, ascending compaction and medians -- the same
// entry points the Python engine calls one by one, launched back to back from
// C so a small detection (config 1: 7 kernels, ~150 us of device work) is not
// bound by per-launch host overhead.
#include <algorithm>

#include "common.cuh"

#define SFFTB_TRY_RC(x)                  \
    do {                                 \
        const int rc_ = (x);             \
        if (rc_ != SFFTB_OK) return rc_; \
    } while (0)

namespace sfftb {

__global__ void finite_flag_kernel(const double* __restrict__ x, int64_t n,
                                   int32_t* __restrict__ bad) {
    bool b = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        b |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

static int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

}  // namespace sfftb

using namespace sfftb;

extern "C" int64_t sfftb_detect_dev_workspace_bytes(int64_t L, int64_t M, int64_t n) {
    if (L < 0 || M < 1 || n < 0) return 0;
    const int64_t W = sfftb_bitmap_words(M);
    return align256(16 * L * M) +                         // ghat
           align256(4 * L * W) +                          // bitmaps
           align256(8 * std::max<int64_t>(L, 1)) +        // sum |x|^2 per lattice
           align256(4 * std::max<int64_t>((n + 31) / 32, 1)) +  // detected mask
           align256(sfftb_dft_workspace_bytes(L, M)) +
           align256(sfftb_compact_workspace_bytes(1, std::max<int64_t>(n, 1)));
}

extern "C" int sfftb_detect_dev(const double* samples, int64_t L, int64_t M,
                                const int64_t* rows, int64_t n, int64_t d, const int64_t* zmat,
                                const double* theta_in, int64_t kbound, int64_t min_hits,
                                int want_medians, int64_t* hits, int64_t* idx, int64_t* counts,
                                double* coeffs, double* theta_out, int32_t* bad, void* ws,
                                void* stream) {
    SFFTB_REQUIRE(L >= 1 && M >= 1 && n >= 0 && d >= 1, "detect_dev: bad sizes");
    SFFTB_REQUIRE((int64_t)d * (M - 1) * (M - 1) >= 0, "detect_dev: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t W = sfftb_bitmap_words(M);
    char* w = (char*)ws;
    auto take = [&](int64_t bytes) {
        char* p = w;
        w += align256(bytes);
        return p;
    };
    double* ghat = (double*)take(16 * L * M);
    uint32_t* bits = (uint32_t*)take(4 * L * W);
    double* sumsq = (double*)take(8 * std::max<int64_t>(L, 1));
    uint32_t* detmask = (uint32_t*)take(4 * std::max<int64_t>((n + 31) / 32, 1));
    void* dft_ws = take(sfftb_dft_workspace_bytes(L, M));
    void* cws = take(sfftb_compact_workspace_bytes(1, std::max<int64_t>(n, 1)));
    // samples must be finite (detect.py:98-109): a device flag the caller
    // reads back with the counts
    SFFTB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
    finite_flag_kernel<<<(unsigned)std::min<int64_t>(num_sms() * 4,
                                                     std::max<int64_t>(1, (2 * L * M + 255) / 256)),
                         256, 0, st>>>(samples, 2 * L * M, bad);
    SFFTB_CHECK_LAUNCH();
    if (theta_in) {
        SFFTB_CUDA(cudaMemcpyAsync(theta_out, theta_in, sizeof(double), cudaMemcpyDeviceToDevice,
                                   st));
    } else {
        SFFTB_TRY_RC(sfftb_sumsq(samples, M, L, M, sumsq, st));
        SFFTB_TRY_RC(sfftb_zero_thresholds(sumsq, 1, L, M, theta_out, st));
    }
    SFFTB_TRY_RC(sfftb_dft(samples, M, ghat, M, L, M, 0, 1.0 / (double)M, dft_ws, st));
    SFFTB_TRY_RC(sfftb_nonzero_bitmap(ghat, 1, L, M, theta_out, bits, st));
    if (n == 0) {
        SFFTB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t), st));
        return SFFTB_OK;
    }
    SFFTB_TRY_RC(sfftb_hash_hits(rows, n, d, zmat, 1, L, M, bits, kbound, min_hits, hits,
                                 detmask, st));
    SFFTB_TRY_RC(sfftb_compact_mask(detmask, 1, n, idx, counts, cws, st));
    if (want_medians)
        SFFTB_TRY_RC(sfftb_medians(rows, d, zmat, 1, L, M, ghat, idx, counts, n, coeffs, st));
    return SFFTB_OK;
}
