// Candidate-set canonicalisation and generation in HBM.
//
// FreqSet's contract (reference latfft/freqset.py:48-67, :85-155): rows are
// duplicate-free and lexicographically sorted, and the row order IS the
// candidate index.  For candidate sets that are born on the device (2^26 rows
// at config 4) this file sorts and de-duplicates them without a host round
// trip:
//
//  * per-coordinate bounds -> coordinates packed, most significant first,
//    into 64-bit keys of consecutive coordinate groups (each group's bit
//    widths sum to <= 64);
//  * an LSD sort over the groups, last group first, each group by a stable
//    8-bit-digit radix sort of (key, row id) pairs: per-tile digit histograms,
//    a digit-major scan, and a stable scatter whose in-tile ranks come from
//    __match_any_sync peer masks (round by round, warp by warp);
//  * rows gathered in the final order, duplicates (equal neighbours) masked
//    and compacted away.
//
// The generator draws uniform rows of [lo, hi]^d from a counter-based
// Philox4x32-10 stream (row i, coordinate j) -- a seeded synthetic workload,
// not numpy's stream (the reference's _random_from_box stays on the host).
#include <vector>

#include "common.cuh"
#include "../../include/sfft_b200.h"

namespace sfftb {

static constexpr int kSortThreads = 256;
static constexpr int kSortItems = 8;
static constexpr int kSortTile = kSortThreads * kSortItems;

__global__ void init_perm_kernel(uint32_t* perm, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        perm[i] = (uint32_t)i;
}

// key[i] = packed coordinates [j0, j1) of row perm[i] (offset by the minima)
__global__ void pack_keys_kernel(const int64_t* __restrict__ rows, int64_t n, int d,
                                 const uint32_t* __restrict__ perm,
                                 const int64_t* __restrict__ lo, int j0, int j1,
                                 const int* __restrict__ shifts, uint64_t* __restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t* r = rows + (int64_t)perm[i] * d;
        uint64_t k = 0;
        for (int j = j0; j < j1; ++j) k |= (uint64_t)(r[j] - lo[j]) << shifts[j - j0];
        key[i] = k;
    }
}

__global__ void __launch_bounds__(kSortThreads)
    digit_hist_kernel(const uint64_t* __restrict__ key, int64_t n, int shift, int64_t ntiles,
                      uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        h[threadIdx.x] = 0;
        __syncthreads();
        const int64_t base = tile * kSortTile;
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const int64_t i = base + it * kSortThreads + threadIdx.x;
            if (i < n) atomicAdd(&h[(key[i] >> shift) & 255u], 1u);
        }
        __syncthreads();
        hist[(int64_t)threadIdx.x * ntiles + tile] = h[threadIdx.x];
        __syncthreads();
    }
}

// one CTA per digit: exclusive prefix over tiles, digit total
__global__ void __launch_bounds__(1024)
    digit_scan_kernel(uint32_t* __restrict__ hist, int64_t ntiles, uint32_t* __restrict__ total) {
    __shared__ uint32_t warp_sum[32];
    __shared__ uint32_t carry;
    const int dgt = blockIdx.x;
    uint32_t* h = hist + (int64_t)dgt * ntiles;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t c0 = 0; c0 < ntiles; c0 += blockDim.x) {
        const int64_t t = c0 + threadIdx.x;
        const uint32_t v = t < ntiles ? h[t] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) warp_sum[warp] = incl;
        __syncthreads();
        uint32_t before = carry;
        for (int w = 0; w < warp; ++w) before += warp_sum[w];
        if (t < ntiles) h[t] = before + incl - v;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t s = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += warp_sum[w];
            carry += s;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) total[dgt] = carry;
}

__global__ void __launch_bounds__(kSortThreads)
    digit_scatter_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ perm,
                         int64_t n, int shift, int64_t ntiles, const uint32_t* __restrict__ hist,
                         const uint32_t* __restrict__ total, uint64_t* __restrict__ key_out,
                         uint32_t* __restrict__ perm_out) {
    constexpr int W = kSortThreads / 32;
    __shared__ uint32_t base[256];      // digit base + this tile's prefix
    __shared__ uint32_t running[256];   // digit counts of earlier rounds in the tile
    __shared__ uint32_t wcnt[W][256];   // this round's per-warp digit counts
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    // digit bases: exclusive scan of the 256 totals (thread 0, tiny)
    __shared__ uint32_t dbase[256];
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int b = 0; b < 256; ++b) {
            dbase[b] = s;
            s += total[b];
        }
    }
    for (int b = threadIdx.x; b < W * 256; b += blockDim.x) (&wcnt[0][0])[b] = 0;
    __syncthreads();
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        base[threadIdx.x] = dbase[threadIdx.x] + hist[(int64_t)threadIdx.x * ntiles + tile];
        running[threadIdx.x] = 0;
        __syncthreads();
        const int64_t t0 = tile * kSortTile;
        for (int it = 0; it < kSortItems; ++it) {
            const int64_t i = t0 + it * kSortThreads + threadIdx.x;
            const bool ok = i < n;
            const uint64_t k = ok ? key[i] : 0;
            const uint32_t p = ok ? perm[i] : 0;
            const unsigned dg = ok ? (unsigned)((k >> shift) & 255u) : 256u + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, dg);
            const int rank = __popc(peers & lt);
            if (ok && rank == 0) wcnt[warp][dg] = __popc(peers);
            __syncthreads();
            if (ok) {
                uint32_t pos = base[dg] + running[dg] + rank;
                for (int w = 0; w < warp; ++w) pos += wcnt[w][dg];
                key_out[pos] = k;
                perm_out[pos] = p;
            }
            __syncthreads();
            {  // fold this round's counts into running[], clear wcnt
                const int b = threadIdx.x;
                uint32_t s = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    s += wcnt[w][b];
                    wcnt[w][b] = 0;
                }
                running[b] += s;
            }
            __syncthreads();
        }
    }
}

__global__ void gather_perm_kernel(const int64_t* __restrict__ rows, int64_t n, int d,
                                   const uint32_t* __restrict__ perm, int64_t* __restrict__ out,
                                   uint32_t* __restrict__ first) {
    // out[i] = rows[perm[i]]; first bit i = row differs from its predecessor
    const int64_t nb = (n + 31) / 32 * 32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool f = false;
        if (i < n) {
            const int64_t* r = rows + (int64_t)perm[i] * d;
            const int64_t* q = i > 0 ? rows + (int64_t)perm[i - 1] * d : nullptr;
            f = (i == 0);
            for (int j = 0; j < d; ++j) {
                const int64_t v = r[j];
                out[i * d + j] = v;
                if (q && q[j] != v) f = true;
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if ((threadIdx.x & 31) == 0 && i < n) first[i >> 5] = b;
    }
}

__global__ void random_box_kernel(int64_t n, int d, int64_t lo, uint64_t span, uint64_t seed,
                                  int64_t* __restrict__ out) {
    const int64_t total = n * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)((uint64_t)e >> 32), 0x5eedu, 0u};
        philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint64_t u = ((uint64_t)c[0] << 32) | c[1];
        out[e] = lo + (int64_t)(uint64_t)(((unsigned __int128)u * span) >> 64);
    }
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int64_t sfftb_canonicalize_workspace_bytes(int64_t n, int64_t d) {
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    // keys x2, perm x2, hist, totals, first mask, bounds, minima, shifts,
    // compact ws, sorted rows (+ 256-byte alignment of each piece)
    return 16 * n + 8 * n + 4 * 256 * ntiles + 4 * 256 + 4 * ((n + 31) / 32 + 4) + 16 * d +
           8 * d + 4 * 64 + sfftb_compact_workspace_bytes(1, n) + 8 * n * d + 12 * 256;
}

extern "C" int sfftb_canonicalize_rows(const int64_t* rows, int64_t n, int64_t d, int64_t* out,
                                       int64_t* count, void* ws, void* stream) {
    SFFTB_REQUIRE(n >= 0 && d >= 1 && d <= 64, "canonicalize: bad sizes");
    SFFTB_REQUIRE(n < (int64_t(1) << 32), "canonicalize: n must be < 2^32");
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        SFFTB_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
        return SFFTB_OK;
    }
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    char* w = (char*)ws;
    auto take = [&](int64_t bytes) {
        char* p = w;
        w += (bytes + 255) & ~int64_t(255);
        return p;
    };
    uint64_t* keyA = (uint64_t*)take(8 * n);
    uint64_t* keyB = (uint64_t*)take(8 * n);
    uint32_t* permA = (uint32_t*)take(4 * n);
    uint32_t* permB = (uint32_t*)take(4 * n);
    uint32_t* hist = (uint32_t*)take(4 * 256 * ntiles);
    uint32_t* total = (uint32_t*)take(4 * 256);
    uint32_t* first = (uint32_t*)take(4 * ((n + 31) / 32 + 4));
    int64_t* bounds = (int64_t*)take(16 * d);
    int64_t* lo = (int64_t*)take(8 * d);
    int* shifts = (int*)take(4 * 64);
    void* cws = (void*)take(sfftb_compact_workspace_bytes(1, n));

    // bounds -> key plan (host; the lexicographic order needs the spans)
    int rc = sfftb_row_bounds(rows, n, d, bounds, stream);
    if (rc) return rc;
    std::vector<int64_t> hb(2 * d);
    SFFTB_CUDA(cudaMemcpyAsync(hb.data(), bounds, 16 * d, cudaMemcpyDeviceToHost, st));
    SFFTB_CUDA(cudaStreamSynchronize(st));
    std::vector<int> bits(d);
    std::vector<int64_t> hlo(d);
    for (int j = 0; j < d; ++j) {
        hlo[j] = hb[2 * j];
        const uint64_t span = (uint64_t)hb[2 * j + 1] - (uint64_t)hb[2 * j];
        bits[j] = span ? 64 - __builtin_clzll(span) : 0;
    }
    SFFTB_CUDA(cudaMemcpyAsync(lo, hlo.data(), 8 * d, cudaMemcpyHostToDevice, st));
    // groups of consecutive coordinates, <= 64 key bits each
    std::vector<std::pair<int, int>> groups;
    for (int j = 0; j < d;) {
        int acc = 0, k = j;
        while (k < d && acc + bits[k] <= 64) acc += bits[k++];
        if (k == j) {  // a single coordinate wider than 64 bits cannot occur
            set_error("canonicalize: coordinate span exceeds 64 bits");
            return SFFTB_EINVAL;
        }
        groups.push_back({j, k});
        j = k;
    }
    const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 16);
    init_perm_kernel<<<grid, 256, 0, st>>>(permA, n);
    SFFTB_CHECK_LAUNCH();
    const int sgrid = (int)std::min<int64_t>(ntiles, (int64_t)num_sms() * 8);
    std::vector<int> sh(64);
    for (int gi = (int)groups.size() - 1; gi >= 0; --gi) {
        const int j0 = groups[gi].first, j1 = groups[gi].second;
        int pos = 0;
        for (int j = j1 - 1; j >= j0; --j) {  // last coordinate least significant
            sh[j - j0] = pos;
            pos += bits[j];
        }
        if (pos == 0) continue;  // constant coordinates: nothing to order
        SFFTB_CUDA(cudaMemcpyAsync(shifts, sh.data(), 4 * 64, cudaMemcpyHostToDevice, st));
        pack_keys_kernel<<<grid, 256, 0, st>>>(rows, n, (int)d, permA, lo, j0, j1, shifts, keyA);
        SFFTB_CHECK_LAUNCH();
        for (int shift = 0; shift < pos; shift += 8) {
            digit_hist_kernel<<<sgrid, kSortThreads, 0, st>>>(keyA, n, shift, ntiles, hist);
            SFFTB_CHECK_LAUNCH();
            digit_scan_kernel<<<256, 1024, 0, st>>>(hist, ntiles, total);
            SFFTB_CHECK_LAUNCH();
            digit_scatter_kernel<<<sgrid, kSortThreads, 0, st>>>(keyA, permA, n, shift, ntiles,
                                                                 hist, total, keyB, permB);
            SFFTB_CHECK_LAUNCH();
            std::swap(keyA, keyB);
            std::swap(permA, permB);
        }
        // the host-side shift table must outlive the async copy
        SFFTB_CUDA(cudaStreamSynchronize(st));
    }
    int64_t* sorted = (int64_t*)take(8 * n * d);
    gather_perm_kernel<<<grid, 256, 0, st>>>(rows, n, (int)d, permA, sorted, first);
    SFFTB_CHECK_LAUNCH();
    // keep the first of each run of equal rows
    int64_t* kidx = (int64_t*)keyB;  // n int64 of scratch
    rc = sfftb_compact_mask(first, 1, n, kidx, count, cws, stream);
    if (rc) return rc;
    return sfftb_gather_rows(sorted, d, kidx, count, n, out, stream);
}

extern "C" int sfftb_random_box_rows(int64_t n, int64_t d, int64_t lo, int64_t hi, uint64_t seed,
                                     int64_t* out, void* stream) {
    SFFTB_REQUIRE(n >= 0 && d >= 1 && hi >= lo, "random_box_rows: bad arguments");
    if (n == 0) return SFFTB_OK;
    const uint64_t span = (uint64_t)(hi - lo) + 1u;
    const int grid = (int)std::min<int64_t>(ceil_div(n * d, 256), (int64_t)num_sms() * 16);
    random_box_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, (int)d, lo, span, seed, out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
