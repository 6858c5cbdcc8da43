// Lattice sampling of sparse trigonometric polynomials, dense point
// evaluation, and the harness noise stream.
//
// The reference samples a lattice either densely (evaluate_many,
// polyeval.py:66-75 -- what sfft uses through SamplingOracle.sample_many,
// dimincr.py:186-191) or structurally for whole lattices (evaluate_on_lattice,
// polyeval.py:78-87: bincount of coefficients by residue, then M * ifft).
// Here every lattice sampling -- including the fixed-tail lattices of the
// dimension-incremental driver -- is structured: the non-lattice coordinates
// of a node are constant, so they fold into an anchor phase per frequency,
//   p([j z/M | tail]) = sum_h B[h] e^{2 pi i j h/M},
//   B[h] = sum_{k: k_{<t}.z = h mod M} c_k e^{2 pi i k_{>=t}.tail},
// an exact restatement of the dense sum.
#include "common.cuh"

namespace sfftb {

static constexpr int kScatterThreads = 1024;
static constexpr int kScatterChunk = 8192;  // keys per shared-memory sort

__global__ void anchor_kernel(const int64_t* __restrict__ support, int64_t s, int d, int t_dim,
                              const double2* __restrict__ coeffs,
                              const double* __restrict__ tails, int G,
                              double2* __restrict__ out) {
    const int64_t total = s * G;
    const int m = d - t_dim;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = e / s, k = e % s;
        const double2 c = coeffs[k];
        if (m == 0) {
            out[e] = c;
            continue;
        }
        double phi = 0.0;
        for (int j = 0; j < m; ++j)
            phi = fma((double)support[k * d + t_dim + j], tails[g * m + j], phi);
        double sn, cs;
        sincospi(2.0 * phi, &sn, &cs);
        out[e] = cmul(c, make_double2(cs, sn));
    }
}

// One CTA per lattice; bins summed in ascending coefficient order.
__global__ void __launch_bounds__(kScatterThreads)
    scatter_kernel(const int64_t* __restrict__ support, int64_t s, int d, int t_dim,
                   const double2* __restrict__ anchored, const int64_t* __restrict__ zmat,
                   int L, int64_t M, double2* __restrict__ bins) {
    extern __shared__ uint64_t keys[];  // kScatterChunk
    __shared__ uint64_t zs[64];
    const int64_t lat = blockIdx.x;
    const int64_t g = lat / L;
    const double invM = 1.0 / (double)M;
    for (int j = threadIdx.x; j < t_dim; j += blockDim.x) {
        int64_t z = zmat[lat * t_dim + j] % M;
        zs[j] = (uint64_t)(z < 0 ? z + M : z);
    }
    double2* B = bins + lat * M;
    for (int64_t h = threadIdx.x; h < M; h += blockDim.x) B[h] = make_double2(0.0, 0.0);
    __syncthreads();
    const double2* a = anchored + g * s;
    for (int64_t c0 = 0; c0 < s; c0 += kScatterChunk) {
        const int cnt = (int)(s - c0 < kScatterChunk ? s - c0 : kScatterChunk);
        int P = 1;
        while (P < cnt) P <<= 1;
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
            uint64_t key = ~0ull;
            if (i < cnt) {
                const int64_t* row = support + (c0 + i) * d;
                uint64_t r = 0;  // r + e z < M + M^2 < 2^62
                for (int j = 0; j < t_dim; ++j)
                    r = mod_u64(r + (uint64_t)reduce_mod(row[j], M) * zs[j], (uint64_t)M, invM);
                key = (r << 32) | (uint64_t)i;
            }
            keys[i] = key;
        }
        __syncthreads();
        // bitonic sort of P keys (ascending)
        for (int k = 2; k <= P; k <<= 1) {
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                for (int i = threadIdx.x; i < P; i += blockDim.x) {
                    const int ixj = i ^ jj;
                    if (ixj > i) {
                        const uint64_t x = keys[i], y = keys[ixj];
                        const bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            keys[i] = y;
                            keys[ixj] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // run heads accumulate their run in ascending coefficient order
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint64_t r = keys[i] >> 32;
            if (i > 0 && (keys[i - 1] >> 32) == r) continue;
            double2 acc = B[r];
            for (int q = i; q < cnt && (keys[q] >> 32) == r; ++q) {
                const double2 v = a[c0 + (int64_t)(keys[q] & 0xffffffffu)];
                acc.x += v.x;
                acc.y += v.y;
            }
            B[r] = acc;
        }
        __syncthreads();
    }
}

// Same binning with a stable LSD radix sort of the residues (8-bit digits,
// ceil(log2 M / 8) passes) in place of the bitonic network: per pass a digit
// histogram, its scan, and a stable scatter in rounds of 512 items whose
// in-round ranks come from __match_any_sync peer masks -- ~3 barriers per
// round instead of log2(P)^2/2 network stages.  Ties stay in coefficient
// order, so the run heads accumulate exactly like np.bincount.
static constexpr int kScatterRsThreads = 512;
static constexpr int kScatterRsChunk = 4096;

__global__ void __launch_bounds__(kScatterRsThreads)
    scatter_rs_kernel(const int64_t* __restrict__ support, int64_t s, int d, int t_dim,
                      const double2* __restrict__ anchored, const int64_t* __restrict__ zmat,
                      int L, int64_t M, int npass, double2* __restrict__ bins,
                      uint32_t* __restrict__ list_r, double2* __restrict__ list_v,
                      const double2* __restrict__ chirp) {
    constexpr int W = kScatterRsThreads / 32;
    extern __shared__ uint32_t rs_dsm[];
    uint32_t* ra = rs_dsm;
    uint32_t* ia = ra + kScatterRsChunk;
    uint32_t* rb = ia + kScatterRsChunk;
    uint32_t* ib = rb + kScatterRsChunk;
    uint32_t(*wcnt)[256] = reinterpret_cast<uint32_t(*)[256]>(ib + kScatterRsChunk);
    __shared__ uint32_t base[256], running[256];
    __shared__ uint64_t zs[64];
    const int64_t lat = blockIdx.x, g = lat / L;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const double invM = 1.0 / (double)M;
    for (int j = threadIdx.x; j < t_dim; j += blockDim.x)
        zs[j] = (uint64_t)reduce_mod(zmat[lat * t_dim + j], M);
    for (int b = threadIdx.x; b < W * 256; b += blockDim.x) wcnt[0][b] = 0;
    // list mode (s <= one chunk): no dense bins; entry i of the lattice's
    // list is (residue, run sum) at run heads and residue ~0 elsewhere
    const bool listed = list_r != nullptr;
    double2* B = listed ? nullptr : bins + lat * M;
    if (!listed)
        for (int64_t h = threadIdx.x; h < M; h += blockDim.x) B[h] = make_double2(0.0, 0.0);
    __syncthreads();
    const double2* a = anchored + g * s;
    for (int64_t c0 = 0; c0 < s; c0 += kScatterRsChunk) {
        const int cnt = (int)(s - c0 < kScatterRsChunk ? s - c0 : kScatterRsChunk);
        uint32_t *r0 = ra, *i0 = ia, *r1 = rb, *i1 = ib;
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int64_t* row = support + (c0 + i) * d;
            uint64_t r = 0;  // r + e z < M + M^2 < 2^62
            for (int j = 0; j < t_dim; ++j)
                r = mod_u64(r + (uint64_t)reduce_mod(row[j], M) * zs[j], (uint64_t)M, invM);
            r0[i] = (uint32_t)r;
            i0[i] = (uint32_t)i;
        }
        for (int pass = 0; pass < npass; ++pass) {
            const int shift = 8 * pass;
            for (int b = threadIdx.x; b < 256; b += blockDim.x) {
                base[b] = 0;
                running[b] = 0;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += blockDim.x)
                atomicAdd(&base[(r0[i] >> shift) & 255u], 1u);
            __syncthreads();
            if (warp == 0) {  // exclusive scan of the 256 digit counts: 8 per lane
                uint32_t v[8], sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    v[q] = base[lane * 8 + q];
                    sum += v[q];
                }
                uint32_t inc = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                uint32_t run = inc - sum;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    base[lane * 8 + q] = run;
                    run += v[q];
                }
            }
            __syncthreads();
            for (int rr = 0; rr < cnt; rr += blockDim.x) {
                const int i = rr + threadIdx.x;
                const bool ok = i < cnt;
                const unsigned dg = ok ? ((r0[i] >> shift) & 255u) : 256u + lane;
                const unsigned peers = __match_any_sync(0xffffffffu, dg);
                const int rank = __popc(peers & lt);
                if (ok && rank == 0) wcnt[warp][dg] = __popc(peers);
                __syncthreads();
                if (ok) {
                    uint32_t pos = base[dg] + running[dg] + rank;
                    for (int w = 0; w < warp; ++w) pos += wcnt[w][dg];
                    r1[pos] = r0[i];
                    i1[pos] = i0[i];
                }
                __syncthreads();
                if (threadIdx.x < 256) {
                    uint32_t sum = 0;
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        sum += wcnt[w][threadIdx.x];
                        wcnt[w][threadIdx.x] = 0;
                    }
                    running[threadIdx.x] += sum;
                }
                __syncthreads();
            }
            uint32_t* t = r0;
            r0 = r1;
            r1 = t;
            t = i0;
            i0 = i1;
            i1 = t;
        }
        // run heads accumulate their run in ascending coefficient order
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint32_t r = r0[i];
            if (i > 0 && r0[i - 1] == r) {
                if (listed) list_r[lat * s + i] = ~0u;
                continue;
            }
            double2 acc = listed ? make_double2(0.0, 0.0) : B[r];
            for (int q = i; q < cnt && r0[q] == r; ++q) {
                const double2 v = a[c0 + i0[q]];
                acc.x += v.x;
                acc.y += v.y;
            }
            if (listed) {  // the sampler's first Bluestein product, folded in
                list_r[lat * s + i] = r;
                list_v[lat * s + i] = cmul(make_double2(acc.x, -acc.y), chirp[r]);
            } else {
                B[r] = acc;
            }
        }
        __syncthreads();
    }
}

// One warp per point: lane q accumulates coefficients q, q+32, ... in order,
// then a fixed shuffle tree adds the 32 partial sums (deterministic).
static constexpr int kEvalThreads = 256;

// LINES: point p = q*K + j of coordinate line q is base row q with
// coordinate q / r replaced by j / K (step 1's line nodes, dimincr.py:137-141).
template <bool LINES>
__global__ void __launch_bounds__(kEvalThreads)
    eval_dense_kernel(const int64_t* __restrict__ support, int64_t s, int d,
                      const double2* __restrict__ coeffs, const double* __restrict__ X, int64_t m,
                      double2* __restrict__ out, int64_t K, int64_t r) {
    const int lane = threadIdx.x & 31;
    const int64_t p = blockIdx.x * (int64_t)(kEvalThreads / 32) + (threadIdx.x >> 5);
    if (p >= m) return;
    double x[32];
    if (LINES) {
        const int64_t q = p / K, jj = p % K;
        for (int j = 0; j < d; ++j) x[j] = X[q * d + j];
        x[q / r] = (double)jj / (double)K;
    } else {
        for (int j = 0; j < d; ++j) x[j] = X[p * d + j];
    }
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t k = lane; k < s; k += 32) {
        double phi = 0.0;
        for (int j = 0; j < d; ++j) phi = fma((double)support[k * d + j], x[j], phi);
        double sn, c;
        sincospi(2.0 * phi, &sn, &c);
        const double2 t = cmul(coeffs[k], make_double2(c, sn));
        acc.x += t.x;
        acc.y += t.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) out[p] = acc;
}

__global__ void noise_kernel(double2* __restrict__ x, int64_t rows, int64_t M, uint64_t seed,
                             int64_t call0, double sigma) {
    const int64_t total = rows * M;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / M, m = e % M;
        const double2 nz = harness_noise(seed, (uint64_t)(call0 + row), m, sigma);
        double2 v = x[e];
        v.x += nz.x;
        v.y += nz.y;
        x[e] = v;
    }
}

static int grid_1d(int64_t work, int threads) {
    int64_t g = ceil_div(work, threads);
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * 16));
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int sfftb_anchor_coeffs(const int64_t* support, int64_t s, int64_t d, int64_t t_dim,
                                   const double* coeffs, const double* tails, int64_t G,
                                   double* out, void* stream) {
    SFFTB_REQUIRE(t_dim >= 0 && t_dim <= d, "anchor: bad t_dim");
    if (s == 0 || G == 0) return SFFTB_OK;
    anchor_kernel<<<grid_1d(s * G, 256), 256, 0, (cudaStream_t)stream>>>(
        support, s, (int)d, (int)t_dim, (const double2*)coeffs, tails, (int)G, (double2*)out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int64_t sfftb_scatter_workspace_bytes(int64_t lattices, int64_t s) {
    (void)lattices;
    (void)s;
    return 0;
}

extern "C" int sfftb_scatter_bins(const int64_t* support, int64_t s, int64_t d, int64_t t_dim,
                                  const double* anchored, const int64_t* zmat, int64_t G,
                                  int64_t L, int64_t M, double* bins, void* ws, void* stream) {
    (void)ws;
    SFFTB_REQUIRE(t_dim >= 0 && t_dim <= 64 && t_dim <= d, "scatter: bad t_dim");
    SFFTB_REQUIRE(M >= 1 && M < (int64_t(1) << 31), "scatter: bad M");
    const int64_t lat = G * L;
    if (lat == 0) return SFFTB_OK;
    SFFTB_REQUIRE(lat <= 0x7fffffff, "scatter: too many lattices");
    if (M <= (int64_t(1) << 24)) {  // the radix path: <= 3 digit passes
        int npass = 1;
        while (npass < 4 && (int64_t(1) << (8 * npass)) < M) ++npass;
        const size_t rsm = sizeof(uint32_t) * (4 * kScatterRsChunk + 256 * (kScatterRsThreads / 32));
        SFFTB_CUDA(smem_opt_in(scatter_rs_kernel, rsm));
        scatter_rs_kernel<<<(unsigned)lat, kScatterRsThreads, rsm, (cudaStream_t)stream>>>(
            support, s, (int)d, (int)t_dim, (const double2*)anchored, zmat, (int)L, M, npass,
            (double2*)bins, nullptr, nullptr, nullptr);
        SFFTB_CHECK_LAUNCH();
        return SFFTB_OK;
    }
    const size_t sm = sizeof(uint64_t) * kScatterChunk;
    SFFTB_CUDA(smem_opt_in(scatter_kernel, sm));
    scatter_kernel<<<(unsigned)lat, kScatterThreads, sm, (cudaStream_t)stream>>>(
        support, s, (int)d, (int)t_dim, (const double2*)anchored, zmat, (int)L, M,
        (double2*)bins);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_scatter_list(const int64_t* support, int64_t s, int64_t d, int64_t t_dim,
                                  const double* anchored, const int64_t* zmat, int64_t G,
                                  int64_t L, int64_t M, uint32_t* list_r, double* list_v,
                                  void* stream) {
    SFFTB_REQUIRE(t_dim >= 0 && t_dim <= 64 && t_dim <= d, "scatter_list: bad t_dim");
    SFFTB_REQUIRE(M >= 1 && M <= (int64_t(1) << 24), "scatter_list: M must be <= 2^24");
    SFFTB_REQUIRE(s >= 1 && s <= kScatterRsChunk, "scatter_list: 1 <= s <= 4096");
    const int64_t lat = G * L;
    if (lat == 0) return SFFTB_OK;
    int npass = 1;
    while (npass < 4 && (int64_t(1) << (8 * npass)) < M) ++npass;
    const size_t rsm = sizeof(uint32_t) * (4 * kScatterRsChunk + 256 * (kScatterRsThreads / 32));
    SFFTB_CUDA(smem_opt_in(scatter_rs_kernel, rsm));
    const double2* chirp = nullptr;
    const int rc = bluestein_chirp(M, &chirp);
    if (rc != SFFTB_OK) return rc;
    scatter_rs_kernel<<<(unsigned)lat, kScatterRsThreads, rsm, (cudaStream_t)stream>>>(
        support, s, (int)d, (int)t_dim, (const double2*)anchored, zmat, (int)L, M, npass,
        nullptr, list_r, (double2*)list_v, chirp);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_eval_dense(const int64_t* support, int64_t s, int64_t d,
                                const double* coeffs, const double* X, int64_t m, double* out,
                                void* stream) {
    SFFTB_REQUIRE(d >= 1 && d <= 32, "eval_dense: 1 <= d <= 32");
    if (m == 0) return SFFTB_OK;
    eval_dense_kernel<false><<<(unsigned)ceil_div(m, kEvalThreads / 32), kEvalThreads, 0,
                               (cudaStream_t)stream>>>(support, s, (int)d,
                                                       (const double2*)coeffs, X, m,
                                                       (double2*)out, 1, 1);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_eval_lines(const int64_t* support, int64_t s, int64_t d,
                                const double* coeffs, const double* base, int64_t nlines,
                                int64_t K, int64_t r, double* out, void* stream) {
    SFFTB_REQUIRE(d >= 1 && d <= 32, "eval_lines: 1 <= d <= 32");
    SFFTB_REQUIRE(K >= 1 && r >= 1 && nlines <= d * r, "eval_lines: bad sizes");
    const int64_t m = nlines * K;
    if (m == 0) return SFFTB_OK;
    eval_dense_kernel<true><<<(unsigned)ceil_div(m, kEvalThreads / 32), kEvalThreads, 0,
                              (cudaStream_t)stream>>>(support, s, (int)d,
                                                      (const double2*)coeffs, base, m,
                                                      (double2*)out, K, r);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_add_noise(double* x, int64_t rows, int64_t M, uint64_t seed, int64_t call0,
                               double sigma, void* stream) {
    if (rows == 0 || M == 0 || sigma == 0.0) return SFFTB_OK;
    noise_kernel<<<grid_1d(rows * M, 256), 256, 0, (cudaStream_t)stream>>>(
        (double2*)x, rows, M, seed, call0, sigma);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
