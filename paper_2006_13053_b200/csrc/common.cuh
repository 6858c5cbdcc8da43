// Shared helpers for the sm_100a kernels of libsfftb200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/sfft_b200.h"

namespace sfftb {

// Thread-local error message behind sfftb_last_error().
void set_error(const std::string& msg);

#define SFFTB_CUDA(call)                                                    \
    do {                                                                    \
        cudaError_t err__ = (call);                                         \
        if (err__ != cudaSuccess) {                                         \
            ::sfftb::set_error(std::string(#call ": ") +                    \
                               cudaGetErrorString(err__));                  \
            return err__ == cudaErrorMemoryAllocation ? SFFTB_ENOMEM        \
                                                      : SFFTB_ECUDA;        \
        }                                                                   \
    } while (0)

// Count of kernels this library launched (sfftb_launch_count()).
void count_launch();
#define SFFTB_CHECK_LAUNCH()          \
    do {                              \
        ::sfftb::count_launch();      \
        SFFTB_CUDA(cudaGetLastError()); \
    } while (0)

#define SFFTB_REQUIRE(cond, msg)                                            \
    do {                                                                    \
        if (!(cond)) {                                                      \
            ::sfftb::set_error(msg);                                        \
            return SFFTB_EINVAL;                                            \
        }                                                                   \
    } while (0)

inline int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// u mod M for u < 2^62 (M < 2^31): the FP64 quotient estimate is off by at
// most a few units, fixed up exactly in integers -- no 64-bit division.
__device__ __forceinline__ uint64_t mod_u64(uint64_t u, uint64_t M, double invM) {
    int64_t q = (int64_t)((double)u * invM);
    int64_t r = (int64_t)u - q * (int64_t)M;
    while (r < 0) r += M;
    while (r >= (int64_t)M) r -= M;
    return (uint64_t)r;
}

// x mod M in [0, M) for any int64 x, skipping the division when |x| < M.
__device__ __forceinline__ int64_t reduce_mod(int64_t x, int64_t M) {
    if (x >= 0 && x < M) return x;
    if (x < 0 && x > -M) return x + M;
    x %= M;
    return x < 0 ? x + M : x;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel)
// and size: launch paths call this every time, the driver call is skipped
// when an equal or larger opt-in is already recorded.
cudaError_t smem_opt_in_raw(const void* kernel, size_t bytes);
template <typename K>
inline cudaError_t smem_opt_in(K kernel, size_t bytes) {
    return smem_opt_in_raw(reinterpret_cast<const void*>(kernel), bytes);
}
// cudaOccupancyMaxActiveBlocksPerMultiprocessor, memoised per (device,
// kernel, threads, smem).
cudaError_t occupancy_raw(int* out, const void* kernel, int threads, size_t smem);
template <typename K>
inline cudaError_t occupancy(int* out, K kernel, int threads, size_t smem) {
    return occupancy_raw(out, reinterpret_cast<const void*>(kernel), threads, smem);
}

// Bluestein chirp of length M from the plan cache (csrc/fft.cu).
int bluestein_chirp(int64_t M, const double2** chirp);

// complex double helpers (interleaved re, im == numpy complex128 layout)
struct cplx {
    double x, y;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) {
    return make_double2(a.x * s, a.y * s);
}

// |v| > theta evaluated exactly as the reference's compiled gather does
// (_core.pyx:195): separately rounded products, one add, IEEE sqrt.
__device__ __forceinline__ bool nonzero_test(double re, double im, double theta) {
    double a = __dmul_rn(re, re);
    double b = __dmul_rn(im, im);
    return __dsqrt_rn(__dadd_rn(a, b)) > theta;
}

// Floor-mod of a signed 64-bit integer by M > 0 (result in [0, M)).
__device__ __forceinline__ int64_t mod_floor(int64_t a, int64_t M) {
    int64_t r = a % M;
    return r < 0 ? r + M : r;
}

}  // namespace sfftb

// ---- harness noise: Philox4x32-10 + 53-bit Box-Muller (oracle/port.py:
// noise_for_call restates it) ----
namespace sfftb {
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        if (r < 9) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
    }
}

// sigma * (N(0,1) + i N(0,1)) for sample m of oracle call `call`
__device__ __forceinline__ double2 harness_noise(uint64_t seed, uint64_t call, int64_t m,
                                                 double sigma) {
    uint32_t c[4] = {(uint32_t)m, (uint32_t)((uint64_t)m >> 32), (uint32_t)call,
                     (uint32_t)(call >> 32)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t ua = ((uint64_t)(c[0] >> 5) << 26) + (c[1] >> 6);
    const uint64_t ub = ((uint64_t)(c[2] >> 5) << 26) + (c[3] >> 6);
    const double u1 = ((double)ua + 1.0) * 0x1.0p-53;
    const double u2 = (double)ub * 0x1.0p-53;
    const double rad = sigma * sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    return make_double2(rad * cs, rad * sn);
}
}  // namespace sfftb

// ---- programmatic dependent launch (sm_90+) ----
// pdl_wait: block until the preceding kernel of the stream has completed and
// its writes are visible (no-op when not launched with PDL); pdl_launch: let
// the next kernel of the stream start launching (its CTAs fill SMs as ours
// exit and run their prologue until their own pdl_wait).
namespace sfftb {
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// <<<>>> or, with pdl, cudaLaunchKernelEx with programmatic stream
// serialization (the kernel must pdl_wait before reading its predecessor's
// output)
template <typename... Exp, typename... Act>
inline cudaError_t launch_maybe_pdl(bool pdl, void (*kern)(Exp...), dim3 grid, dim3 block,
                                    size_t smem, cudaStream_t st, Act&&... args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

// medians on pair tables (hash.cu); dense: most candidates detected
int medians_pairs_launch(const int32_t* P, const int32_t* V, int64_t n1, int64_t n2, int64_t G,
                         int64_t L, int64_t M, const double* ghat, const int64_t* idx,
                         const int64_t* counts, int64_t cap, double* coeffs, void* stream,
                         bool dense);

// mask compaction (hash.cu) with the single-CTA threshold in words per group
int compact_mask_launch(const uint32_t* mask, int64_t G, int64_t n, int64_t cap, int64_t* idx,
                        int64_t* counts, int64_t* totals, void* ws, void* stream,
                        int64_t single_words);

// candidate hashing on the tensor cores (hash_tc.cu): 1 = handled, 0 = shape
// outside the byte-GEMM path (use the CUDA-core kernels), < 0 = -status
int hash_hits_tc(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat, int64_t L,
                 int64_t M, const uint32_t* bits, int64_t min_hits, int64_t* hits64,
                 uint32_t* detmask, cudaStream_t st);

// candidate hashing on the tensor cores, rolling kernel (hash_roll.cu): same
// return convention
int hash_hits_roll(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat, int64_t L,
                   int64_t M, const uint32_t* bits, int64_t min_hits, int64_t* hits64,
                   uint32_t* detmask, cudaStream_t st);
// fp16 variant for small coordinates (csrc/hash_rollf.cu; kbound = sum_j max|k_j| < 2048)
int hash_hits_rollf(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat, int64_t L,
                    int64_t M, const uint32_t* bits, int64_t kbound, int64_t min_hits,
                    int64_t* hits64, uint32_t* detmask, cudaStream_t st);

// zero-test thresholds (hash.cu) launched inside the fused transform chain
int zero_thresholds_launch(const double* sumsq, int64_t G, int64_t L, int64_t M, double* theta,
                           cudaStream_t st, bool pdl);
}  // namespace sfftb

// ---- mbarrier + 1-D bulk copy (TMA engine) helpers, sm_90+/sm_100a ----
namespace sfftb {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_addr(bar)),
        "r"(bytes)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// global -> shared bulk copy (bytes % 16 == 0, 16-B aligned), completes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// same, destination given as a 32-bit shared-window address
__device__ __forceinline__ void bulk_g2s_addr(uint32_t dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem_ptr)),
                 "l"(gptr)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

}  // namespace sfftb
