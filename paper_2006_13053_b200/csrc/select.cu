// Threshold + top-s selection of detected coefficients (detect_topk,
// detect.py:172-195): keep |c| >= theta; if more than s_tilde survive, keep
// the s_tilde largest by (|c| descending, candidate index ascending) -- the
// reference's lexsort key, since candidate rows are in lexicographic order --
// and return them in ascending candidate order.
//
// One CTA per group: |c| keys (IEEE bits of non-negative doubles are
// monotone) go through an MSB-first 8-bit radix select that finds the
// s_tilde-th largest key T; an order-preserving block scan then emits every
// element with key > T plus the first (s_tilde - #{key > T}) elements equal
// to T.
#include "common.cuh"

namespace sfftb {

static constexpr int kSelThreads = 1024;

__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    int64_t t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (kSelThreads / 32) ? red[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    t = red[0];
    __syncthreads();
    return t;
}

// exclusive prefix over the block of flag (0/1); returns prefix, *total set
__device__ __forceinline__ int block_excl_scan(int flag, int* wsum, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, flag);
    const int within = __popc(b & ((1u << lane) - 1u));
    __syncthreads();
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) {
        if (w < warp) before += wsum[w];
        tot += wsum[w];
    }
    *total = tot;
    return before + within;
}

__global__ void __launch_bounds__(kSelThreads)
    topk_kernel(const int64_t* __restrict__ idx, const double2* __restrict__ coeffs,
                const int64_t* __restrict__ counts, int64_t cap, double theta, int64_t s_tilde,
                int64_t* __restrict__ kidx, double2* __restrict__ kco,
                int64_t* __restrict__ kcounts, uint64_t* __restrict__ keys) {
    const int g = blockIdx.x;
    const int64_t n = counts[g];
    const int64_t* I = idx + (int64_t)g * cap;
    const double2* C = coeffs + (int64_t)g * cap;
    uint64_t* K = keys + (int64_t)g * cap;
    int64_t* OI = kidx + (int64_t)g * cap;
    double2* OC = kco + (int64_t)g * cap;
    __shared__ int64_t red[32];
    __shared__ int wsum[32];
    __shared__ unsigned int hist[256];
    __shared__ uint64_t sh_prefix;
    __shared__ int64_t sh_rank;

    // keys: |c| bits for kept entries, sentinel 0 with a kept flag folded in
    // (|c| >= theta >= 0, so dropped entries get key 0 and are excluded via
    // the kept test below)
    int64_t kept_local = 0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double2 c = C[k];
        const double m = hypot(c.x, c.y);
        const bool keep = m >= theta;
        K[k] = keep ? (__double_as_longlong(m) | 0ull) : ~0ull;  // ~0 marks dropped
        kept_local += keep;
    }
    const int64_t nkeep = block_sum_i64(kept_local, red);

    uint64_t T = 0;
    int64_t need_eq = 0;
    const bool select = nkeep > s_tilde;
    if (select && s_tilde > 0) {
        // find the s_tilde-th largest key among kept (keys != ~0)
        if (threadIdx.x == 0) {
            sh_prefix = 0;
            sh_rank = s_tilde;  // rank from the top, 1-based
        }
        __syncthreads();
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            const uint64_t prefix = sh_prefix;
            const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
            for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
                const uint64_t key = K[k];
                if (key == ~0ull) continue;
                if ((key & hmask) != prefix) continue;
                atomicAdd(&hist[(key >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int64_t rank = sh_rank;
                int digit = 255;
                for (; digit > 0; --digit) {
                    if ((int64_t)hist[digit] >= rank) break;
                    rank -= hist[digit];
                }
                sh_prefix = prefix | ((uint64_t)digit << shift);
                sh_rank = rank;
            }
            __syncthreads();
        }
        T = sh_prefix;
        int64_t gt_local = 0;
        for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
            const uint64_t key = K[k];
            gt_local += (key != ~0ull && key > T);
        }
        need_eq = s_tilde - block_sum_i64(gt_local, red);
    }

    // ordered emission
    int64_t out_pos = 0, eq_seen = 0;
    for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const int64_t k = c0 + threadIdx.x;
        uint64_t key = ~0ull;
        if (k < n) key = K[k];
        const bool kept = key != ~0ull;
        int emit;
        int is_eq = 0;
        if (!select) {
            emit = kept;
        } else if (s_tilde == 0) {
            emit = 0;
        } else {
            is_eq = kept && key == T;
            int tot_eq;
            const int eq_before = block_excl_scan(is_eq, wsum, &tot_eq);
            emit = (kept && key > T) || (is_eq && (eq_seen + eq_before) < need_eq);
            eq_seen += tot_eq;
        }
        int total;
        const int pos = block_excl_scan(emit, wsum, &total);
        if (emit) {
            OI[out_pos + pos] = I[k];
            OC[out_pos + pos] = C[k];
        }
        out_pos += total;
    }
    if (threadIdx.x == 0) kcounts[g] = out_pos;
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int64_t sfftb_topk_workspace_bytes(int64_t G, int64_t cap) {
    return std::max<int64_t>(G * cap, 1) * (int64_t)sizeof(uint64_t);
}

extern "C" int sfftb_topk(const int64_t* idx, const double* coeffs, const int64_t* counts,
                          int64_t G, int64_t cap, double theta, int64_t s_tilde, int64_t* kidx,
                          double* kcoeffs, int64_t* kcounts, void* ws, void* stream) {
    SFFTB_REQUIRE(G >= 1 && G <= 65535 && cap >= 0, "topk: bad sizes");
    SFFTB_REQUIRE(s_tilde >= 0 && theta >= 0, "topk: s_tilde and theta must be >= 0");
    topk_kernel<<<(unsigned)G, kSelThreads, 0, (cudaStream_t)stream>>>(
        idx, (const double2*)coeffs, counts, cap, theta, s_tilde, kidx, (double2*)kcoeffs,
        kcounts, (uint64_t*)ws);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
