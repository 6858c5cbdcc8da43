// Step-1 selection of the dimension-incremental driver on the device
// (step1_components, dimincr.py:122-152): for every coordinate line q = (t, i)
// the estimates est[q][v mod K] of the axis values v, their magnitudes
// |.| = hypot (np.abs), the s_local largest by the reference's lexsort key
// (magnitude descending, value ascending, dimincr.py:143-144), the >= theta
// cut (:145), and the union over the r lines of one coordinate (:146,
// np.union1d) as a presence mask over the sorted values.
//
// One CTA per line; the rank of value i is #{j: m_j > m_i} + #{j < i: m_j ==
// m_i} (values are ascending, so a lower index is the smaller value), which
// is exactly its position in the stable lexsort.  K (the line length, 65 or
// 129 at the BASELINE configs) is small, so every thread scans the line's
// magnitudes in shared memory.
#include "common.cuh"

namespace sfftb {

static constexpr int kStep1Threads = 256;
static constexpr int64_t kStep1MaxVals = 8192;  // shared magnitudes: 64 KB

__global__ void __launch_bounds__(kStep1Threads)
    step1_select_kernel(const double2* __restrict__ est, int64_t K,
                        const int64_t* __restrict__ vals, int64_t nv, int64_t r,
                        int64_t s_local, double theta, int32_t* __restrict__ present,
                        int64_t* __restrict__ kept) {
    extern __shared__ double mags[];
    __shared__ int red[kStep1Threads / 32];
    const int64_t q = blockIdx.x;
    const double2* e = est + q * K;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        int64_t h = vals[i] % K;
        if (h < 0) h += K;
        const double2 v = e[h];
        mags[i] = hypot(v.x, v.y);
    }
    __syncthreads();
    int cnt = 0;
    int32_t* pres = present + (q / r) * nv;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const double mi = mags[i];
        int64_t rank = 0;
        for (int64_t j = 0; j < nv; ++j) {
            const double mj = mags[j];
            rank += (mj > mi) || (mj == mi && j < i);
        }
        if (rank < s_local && mi >= theta) {
            pres[i] = 1;  // every line of coordinate q / r writes 1: idempotent
            ++cnt;
        }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < kStep1Threads / 32; ++w) tot += red[w];
        kept[q] = tot;
    }
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int sfftb_step1_select(const double* est, int64_t nlines, int64_t K,
                                  const int64_t* vals, int64_t nv, int64_t r, int64_t s_local,
                                  double theta, int32_t* present, int64_t* kept,
                                  void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SFFTB_REQUIRE(nlines >= 0 && K >= 1 && r >= 1 && nlines % r == 0,
                  "sfftb_step1_select: bad line shape");
    SFFTB_REQUIRE(nv >= 0 && nv <= kStep1MaxVals, "sfftb_step1_select: too many axis values");
    SFFTB_REQUIRE(s_local >= 0 && theta >= 0.0, "sfftb_step1_select: bad s_local / theta");
    if (nlines == 0) return SFFTB_OK;
    SFFTB_CUDA(cudaMemsetAsync(present, 0, sizeof(int32_t) * (nlines / r) * (nv ? nv : 1),
                               stream));
    if (nv == 0) {
        SFFTB_CUDA(cudaMemsetAsync(kept, 0, sizeof(int64_t) * nlines, stream));
        return SFFTB_OK;
    }
    const size_t sm = sizeof(double) * (size_t)nv;
    SFFTB_CUDA(smem_opt_in(step1_select_kernel, sm));
    step1_select_kernel<<<(unsigned)nlines, kStep1Threads, sm, stream>>>(
        reinterpret_cast<const double2*>(est), K, vals, nv, r, s_local, theta, present, kept);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
