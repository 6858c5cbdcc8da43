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

// ---------------------------------------------------------------------------
// Grid-wide path for large groups (noisy data: every candidate detected, 10^5
// per group).  Same selection, spread over the whole GPU:
//   keys + 12-bit top-digit histograms (grid) -> pick digit (CTA per group)
//   -> 12/12/12/12/4-bit refinements over the keys still matching the prefix
//   -> gt / eq masks -> the first need_eq ties by index -> compaction and
//   gathers of (idx, coeff) in ascending candidate order.
// ---------------------------------------------------------------------------
static constexpr int kHistBins = 4096;

struct TopkState {  // per group
    uint64_t prefix;
    int64_t rank;     // remaining rank from the top inside the current prefix
    int64_t nkeep;
    int64_t active;   // selection needed (nkeep > s_tilde > 0); 2: s_tilde == 0
};

__global__ void __launch_bounds__(256)
    topk_keys_kernel(const double2* __restrict__ coeffs, const int64_t* __restrict__ counts,
                     int64_t cap, double theta, uint64_t* __restrict__ keys,
                     uint32_t* __restrict__ hist, TopkState* __restrict__ st) {
    __shared__ uint32_t h[kHistBins];
    const int g = blockIdx.y;
    const int64_t n = counts[g];
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    int64_t kept = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double2 c = coeffs[(int64_t)g * cap + k];
        const double m = hypot(c.x, c.y);
        const bool keep = m >= theta;
        const uint64_t key = keep ? (uint64_t)__double_as_longlong(m) : ~0ull;
        keys[(int64_t)g * cap + k] = key;
        if (keep) {
            atomicAdd(&h[key >> 52], 1u);
            ++kept;
        }
    }
    for (int o = 16; o > 0; o >>= 1) kept += __shfl_down_sync(0xffffffffu, kept, o);
    if ((threadIdx.x & 31) == 0 && kept) atomicAdd((unsigned long long*)&st[g].nkeep,
                                                   (unsigned long long)kept);
    __syncthreads();
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[(int64_t)g * kHistBins + i], h[i]);
}

// one CTA per group: choose the digit at this level.  The 2^width bins are
// summed per thread (16 consecutive bins each), a block suffix scan finds the
// thread whose bins cross the remaining rank from the top, and that thread
// walks its 16 bins.
__global__ void __launch_bounds__(256)
    topk_pick_kernel(uint32_t* __restrict__ hist, TopkState* __restrict__ st, int64_t s_tilde,
                     int shift, int width, int first) {
    __shared__ int64_t suf[257];
    __shared__ int64_t sh_rank;
    const int g = blockIdx.x;
    TopkState& S = st[g];
    uint32_t* h = hist + (int64_t)g * kHistBins;
    if (threadIdx.x == 0) {
        if (first) {
            S.active = (s_tilde == 0) ? 2 : (S.nkeep > s_tilde ? 1 : 0);
            S.rank = s_tilde;
            S.prefix = 0;
        }
        sh_rank = S.rank;
    }
    __syncthreads();
    const int nb = 1 << width;
    const int per = (nb + 255) / 256;  // bins per thread (16 for 12-bit levels)
    const int b0 = threadIdx.x * per;
    uint32_t loc[16];
    int64_t mine = 0;
    for (int q = 0; q < per && q < 16; ++q) {
        loc[q] = b0 + q < nb ? h[b0 + q] : 0u;
        mine += loc[q];
    }
    if (S.active == 1) {
        // suffix sums over threads: suf[t] = sum of bins of threads > t
        suf[threadIdx.x] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t run = 0;
            for (int t = 255; t >= 0; --t) {
                const int64_t v = suf[t];
                suf[t] = run;
                run += v;
            }
        }
        __syncthreads();
        const int64_t above = suf[threadIdx.x], rank = sh_rank;
        if (above < rank && above + mine >= rank) {  // the crossing thread
            int64_t r = rank - above;
            int digit = b0 + per - 1;
            for (int q = per - 1; q > 0; --q, --digit) {
                if ((int64_t)loc[q] >= r) break;
                r -= loc[q];
            }
            S.prefix |= (uint64_t)digit << shift;
            S.rank = r;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) h[i] = 0;  // next level
}

__global__ void __launch_bounds__(256)
    topk_hist_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ counts,
                     int64_t cap, const TopkState* __restrict__ st, int shift, int width,
                     uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kHistBins];
    const int g = blockIdx.y;
    if (st[g].active != 1) return;
    const int64_t n = counts[g];
    const int hi = shift + width;
    const uint64_t pre = st[g].prefix >> hi;
    const uint32_t dmask = (1u << width) - 1u;
    for (int i = threadIdx.x; i < (1 << width); i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[(int64_t)g * cap + k];
        if (key == ~0ull || (hi < 64 && (key >> hi) != pre)) continue;
        atomicAdd(&h[(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (1 << width); i += blockDim.x)
        if (h[i]) atomicAdd(&hist[(int64_t)g * kHistBins + i], h[i]);
}

// emit / tie masks (ballot words per 32 candidates)
__global__ void topk_mask_kernel(const uint64_t* __restrict__ keys,
                                 const int64_t* __restrict__ counts, int64_t cap,
                                 const TopkState* __restrict__ st, uint32_t* __restrict__ emask,
                                 uint32_t* __restrict__ qmask, int64_t nwords) {
    const int g = blockIdx.y;
    const int64_t n = counts[g];
    const TopkState S = st[g];
    const int64_t nb = (n + 31) / 32 * 32;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nwords * 32;
         k += (int64_t)gridDim.x * blockDim.x) {
        bool e = false, q = false;
        if (k < n) {
            const uint64_t key = keys[(int64_t)g * cap + k];
            const bool kept = key != ~0ull;
            if (S.active == 0) e = kept;
            else if (S.active == 1) {
                e = kept && key > S.prefix;
                q = kept && key == S.prefix;
            }
        }
        const unsigned be = __ballot_sync(0xffffffffu, e), bq = __ballot_sync(0xffffffffu, q);
        if ((threadIdx.x & 31) == 0) {
            emask[(int64_t)g * nwords + (k >> 5)] = k < nb ? be : 0u;
            qmask[(int64_t)g * nwords + (k >> 5)] = k < nb ? bq : 0u;
        }
    }
}

// the first `rank` ties (ascending candidate index) join the emitted set
__global__ void topk_ties_kernel(const int64_t* __restrict__ tpos,
                                 const int64_t* __restrict__ tcount, int64_t cap,
                                 const TopkState* __restrict__ st, uint32_t* __restrict__ emask,
                                 int64_t nwords) {
    const int g = blockIdx.y;
    if (st[g].active != 1) return;
    const int64_t take = min(st[g].rank, tcount[g]);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < take;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = tpos[(int64_t)g * cap + j];
        atomicOr(&emask[(int64_t)g * nwords + (k >> 5)], 1u << (k & 31));
    }
}

__global__ void topk_gather_kernel(const int64_t* __restrict__ idx,
                                   const double2* __restrict__ coeffs,
                                   const int64_t* __restrict__ pos,
                                   const int64_t* __restrict__ kcounts, int64_t cap,
                                   int64_t* __restrict__ kidx, double2* __restrict__ kco) {
    const int g = blockIdx.y;
    const int64_t c = kcounts[g];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = pos[(int64_t)g * cap + j];
        kidx[(int64_t)g * cap + j] = idx[(int64_t)g * cap + k];
        kco[(int64_t)g * cap + j] = coeffs[(int64_t)g * cap + k];
    }
}

}  // namespace sfftb

using namespace sfftb;

static int64_t topk_grid_ws(int64_t G, int64_t cap) {
    const int64_t nwords = (cap + 31) / 32;
    const int64_t a = 8 * G * cap;                         // keys
    const int64_t b = 4 * G * kHistBins;                   // histograms
    const int64_t c = (int64_t)sizeof(TopkState) * G;      // states
    const int64_t d = 2 * 4 * G * nwords;                  // emit / tie masks
    const int64_t e = 2 * 8 * G * cap;                     // tie positions, emit positions
    const int64_t f = 8 * G;                               // tie counts
    return a + b + c + d + e + f + sfftb_compact_workspace_bytes(G, cap) + 16 * 256;
}

extern "C" int64_t sfftb_topk_workspace_bytes(int64_t G, int64_t cap) {
    // sized for either path (sfftb_topk or sfftb_topk_grid)
    return std::max(std::max<int64_t>(G * cap, 1) * (int64_t)sizeof(uint64_t),
                    topk_grid_ws(G, cap));
}

static int topk_grid(const int64_t* idx, const double* coeffs, const int64_t* counts, int64_t G,
                     int64_t cap, double theta, int64_t s_tilde, int64_t* kidx,
                     double* kcoeffs, int64_t* kcounts, void* ws, cudaStream_t st) {
    const int64_t nwords = (cap + 31) / 32;
    char* w = (char*)ws;
    auto take = [&](int64_t bytes) {
        char* p = w;
        w += (bytes + 255) & ~int64_t(255);
        return p;
    };
    uint64_t* keys = (uint64_t*)take(8 * G * cap);
    uint32_t* hist = (uint32_t*)take(4 * G * kHistBins);
    TopkState* S = (TopkState*)take((int64_t)sizeof(TopkState) * G);
    uint32_t* emask = (uint32_t*)take(4 * G * nwords);
    uint32_t* qmask = (uint32_t*)take(4 * G * nwords);
    int64_t* tpos = (int64_t*)take(8 * G * cap);
    int64_t* epos = (int64_t*)take(8 * G * cap);
    int64_t* tcount = (int64_t*)take(8 * G);
    void* cws = (void*)take(sfftb_compact_workspace_bytes(G, cap));
    SFFTB_CUDA(cudaMemsetAsync(hist, 0, 4 * G * kHistBins, st));
    SFFTB_CUDA(cudaMemsetAsync(S, 0, sizeof(TopkState) * G, st));
    const unsigned gx = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(cap, 256), ceil_div((int64_t)num_sms() * 8, G)));
    topk_keys_kernel<<<dim3(gx, (unsigned)G), 256, 0, st>>>((const double2*)coeffs, counts, cap,
                                                            theta, keys, hist, S);
    SFFTB_CHECK_LAUNCH();
    // digit levels: 12 bits each from the top, then the last 4
    const int shifts[6] = {52, 40, 28, 16, 4, 0};
    const int widths[6] = {12, 12, 12, 12, 12, 4};
    for (int lv = 0; lv < 6; ++lv) {
        if (lv > 0) {
            topk_hist_kernel<<<dim3(gx, (unsigned)G), 256, 0, st>>>(keys, counts, cap, S,
                                                                    shifts[lv], widths[lv], hist);
            SFFTB_CHECK_LAUNCH();
        }
        topk_pick_kernel<<<(unsigned)G, 256, 0, st>>>(hist, S, s_tilde, shifts[lv], widths[lv],
                                                       lv == 0);
        SFFTB_CHECK_LAUNCH();
    }
    topk_mask_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(
                                ceil_div(nwords * 32, 256), ceil_div((int64_t)num_sms() * 8, G))),
                            (unsigned)G),
                       256, 0, st>>>(keys, counts, cap, S, emask, qmask, nwords);
    SFFTB_CHECK_LAUNCH();
    int rc = sfftb_compact_mask(qmask, G, cap, tpos, tcount, cws, st);
    if (rc) return rc;
    topk_ties_kernel<<<dim3(gx, (unsigned)G), 256, 0, st>>>(tpos, tcount, cap, S, emask, nwords);
    SFFTB_CHECK_LAUNCH();
    rc = sfftb_compact_mask(emask, G, cap, epos, kcounts, cws, st);
    if (rc) return rc;
    topk_gather_kernel<<<dim3(gx, (unsigned)G), 256, 0, st>>>(
        idx, (const double2*)coeffs, epos, kcounts, cap, kidx, (double2*)kcoeffs);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
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

extern "C" int sfftb_topk_grid(const int64_t* idx, const double* coeffs, const int64_t* counts,
                               int64_t G, int64_t cap, double theta, int64_t s_tilde,
                               int64_t* kidx, double* kcoeffs, int64_t* kcounts, void* ws,
                               void* stream) {
    SFFTB_REQUIRE(G >= 1 && G <= 65535 && cap >= 0, "topk: bad sizes");
    SFFTB_REQUIRE(s_tilde >= 0 && theta >= 0, "topk: s_tilde and theta must be >= 0");
    if (cap == 0) {
        SFFTB_CUDA(cudaMemsetAsync(kcounts, 0, sizeof(int64_t) * G, (cudaStream_t)stream));
        return SFFTB_OK;
    }
    return topk_grid(idx, coeffs, counts, G, cap, theta, s_tilde, kidx, kcoeffs, kcounts, ws,
                     (cudaStream_t)stream);
}
