// Batched prime-length DFT in FP64: Bluestein chirp-z onto power-of-two FFTs.
//
// Replaces numpy/pocketfft behind dft_forward_normalized (dft.py:18-27) and
// the inverse transform of the lattice sampler (polyeval.py:87).
//
//   X_h = w_h * sum_j (x_j w_j) conj(w_{h-j}),   w_n = exp(-i pi n^2 / M)
//
// The linear convolution runs as FFT_N -> * B^ -> IFFT_N with N >= 2M-1 a
// power of two and B^ = FFT_N(b)/N (b_n = conj(w_|n|), wrapped) precomputed
// once per M on the host in long double.
//
//  * N <= 8192: one CTA per transform, the whole chain in shared memory
//    (bluestein_small).
//  * N >= 16384: four-step N = N1*N2 in three kernels over a device workspace:
//      colA : chirp + length-N2 FFTs down the N1 columns + twiddle
//      rowB : length-N1 FFT of each row, * B^ (stored row-permuted),
//             length-N1 IFFT, conjugate twiddle  (forward pass 2, pointwise
//             product and inverse pass 1 fused in shared memory)
//      colC : length-N2 IFFTs down the columns + chirp + scale -> output
//    Each kernel moves its CTA's tile once in and once out, coalesced in
//    runs of F consecutive complex numbers.
#include <math.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <vector>

#include "fft_core.cuh"

namespace sfftb {

struct BluesteinPlan {
    int64_t M = 0;
    int N = 0, N1 = 0, N2 = 0, logN = 0;
    int P9 = 0;  // single-CTA mixed length N = 9 * P9 (P9 a power of two), else 0
    double2* chirp = nullptr;  // M
    double2* bhat = nullptr;   // N (natural if N <= 8192, else [k2][k1] = B^[k2 + N2 k1])
    double2* tw_hi = nullptr;  // N/64 : e^{-2 pi i 64k/N}
    double2* tw_lo = nullptr;  // 64   : e^{-2 pi i k/N}
    double2* tw_n1 = nullptr;  // N1   : e^{-2 pi i k/N1} (four-step only)
    double2* tw_n2 = nullptr;  // N2   : e^{-2 pi i k/N2}
};

static std::mutex g_plan_mu;
static std::map<std::pair<int, int64_t>, BluesteinPlan*> g_plans;

static constexpr int kSmallMaxLog = 13;  // single-CTA Bluestein up to N = 8192
static constexpr int kMinLog = 8;        // N >= 256
static constexpr int kMaxLog = 20;

static int bluestein_log(int64_t M) {
    int lg = kMinLog;
    while ((int64_t(1) << lg) < 2 * M - 1) ++lg;
    return lg;
}

// Convolution length: the smallest N >= 2M-1 among the powers of two (>= 256)
// and, above the single-CTA sizes, the mixed-radix 192 * {128, 256} of the
// register four-step kernels (N = 3 * 2^k: 25% fewer bytes per pass than the
// next power of two for M in (8192, 12288] and (16384, 24576]).
// Within the single-CTA sizes the smallest 9 * 2^k >= max(2M-1, 576) is used
// when it is below the power of two (bluestein_small9: M = 2069 -> 4608
// instead of 8192, M = 1039 -> 2304 instead of 4096).
static int64_t bluestein_N(int64_t M) {
    const int64_t pow2 = int64_t(1) << bluestein_log(M);
    if (pow2 > (int64_t(1) << kSmallMaxLog)) {
        for (int64_t c : {int64_t(24576), int64_t(49152)})
            if (c >= 2 * M - 1 && c < pow2) return c;
    } else {
        static const bool off = getenv("SFFTB_NO_SMALL9") != nullptr;  // A/B only
        if (!off)
            for (int64_t c : {int64_t(576), int64_t(1152), int64_t(2304), int64_t(4608)})
                if (c >= 2 * M - 1 && c < pow2) return c;
    }
    return pow2;
}

// iterative radix-2 FFT in long double (plan construction only)
static void host_fft_ld(std::vector<long double>& re, std::vector<long double>& im) {
    const size_t n = re.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            std::swap(re[i], re[j]);
            std::swap(im[i], im[j]);
        }
    }
    const long double PI = 3.141592653589793238462643383279502884L;
    std::vector<long double> wr(n / 2), wi(n / 2);
    for (size_t k = 0; k < n / 2; ++k) {
        long double a = -2.0L * PI * (long double)k / (long double)n;
        wr[k] = cosl(a);
        wi[k] = sinl(a);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1, step = n / len;
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < half; ++k) {
                long double xr = re[i + k + half], xi = im[i + k + half];
                long double tr = xr * wr[k * step] - xi * wi[k * step];
                long double ti = xr * wi[k * step] + xi * wr[k * step];
                re[i + k + half] = re[i + k] - tr;
                im[i + k + half] = im[i + k] - ti;
                re[i + k] += tr;
                im[i + k] += ti;
            }
    }
}

// Forward DFT of any length 2^a 3^b in long double by recursive radix-2/3
// decimation in time (plan construction only).
static void host_fft23_ld(std::vector<long double>& re, std::vector<long double>& im) {
    const size_t n = re.size();
    if (n == 1) return;
    const size_t R = (n % 2 == 0) ? 2 : 3, m = n / R;
    std::vector<long double> r[3], i[3];
    for (size_t q = 0; q < R; ++q) {
        r[q].resize(m);
        i[q].resize(m);
        for (size_t j = 0; j < m; ++j) {
            r[q][j] = re[R * j + q];
            i[q][j] = im[R * j + q];
        }
        host_fft23_ld(r[q], i[q]);
    }
    const long double PI = 3.141592653589793238462643383279502884L;
    for (size_t k = 0; k < n; ++k) {
        long double sr = 0.0L, si = 0.0L;
        for (size_t q = 0; q < R; ++q) {
            const long double a = -2.0L * PI * (long double)((q * k) % n) / (long double)n;
            const long double c = cosl(a), sn = sinl(a);
            const long double xr = r[q][k % m], xi = i[q][k % m];
            sr += xr * c - xi * sn;
            si += xr * sn + xi * c;
        }
        re[k] = sr;
        im[k] = si;
    }
}

// B^ of a mixed-radix length N = 3 * 2^k: three decimated power-of-two FFTs
// combined by one radix-3 step, all in long double.
static void host_fft3_ld(std::vector<long double>& re, std::vector<long double>& im) {
    const size_t n = re.size(), m = n / 3;
    std::vector<long double> r[3], i[3];
    for (int q = 0; q < 3; ++q) {
        r[q].resize(m);
        i[q].resize(m);
        for (size_t j = 0; j < m; ++j) {
            r[q][j] = re[3 * j + q];
            i[q][j] = im[3 * j + q];
        }
        host_fft_ld(r[q], i[q]);
    }
    const long double PI = 3.141592653589793238462643383279502884L;
    for (size_t k = 0; k < n; ++k) {
        long double sr = 0.0L, si = 0.0L;
        for (int q = 0; q < 3; ++q) {
            const long double a = -2.0L * PI * (long double)((q * k) % n) / (long double)n;
            const long double c = cosl(a), sn = sinl(a);
            const long double xr = r[q][k % m], xi = i[q][k % m];
            sr += xr * c - xi * sn;
            si += xr * sn + xi * c;
        }
        re[k] = sr;
        im[k] = si;
    }
}

static int build_plan(int64_t M, BluesteinPlan** out) {
    SFFTB_REQUIRE(M >= 1, "DFT length must be >= 1");
    const int lg = bluestein_log(M);
    SFFTB_REQUIRE(lg <= kMaxLog, "DFT length too large for the Bluestein plan (M <= 524288)");
    BluesteinPlan* p = new BluesteinPlan();
    p->M = M;
    p->N = (int)bluestein_N(M);
    const bool mixed = (p->N & (p->N - 1)) != 0;
    p->logN = mixed ? 0 : lg;
    if (mixed && p->N <= (1 << kSmallMaxLog)) {
        p->P9 = p->N / 9;  // bluestein_small9
    } else if (mixed) {
        p->N1 = 192;
        p->N2 = p->N / 192;
    } else if (lg > kSmallMaxLog) {
        p->N1 = 1 << (lg / 2);
        p->N2 = 1 << (lg - lg / 2);
    }
    const int N = p->N;
    const long double PI = 3.141592653589793238462643383279502884L;
    std::vector<double2> chirp(M), thi(N / 64), tlo(64), bh(N);
    std::vector<double2> tn1(p->N1 ? p->N1 : 1), tn2(p->N2 ? p->N2 : 1);
    for (int k = 0; k < p->N1; ++k) {
        long double a = -2.0L * PI * k / p->N1;
        tn1[k] = make_double2((double)cosl(a), (double)sinl(a));
    }
    for (int k = 0; k < p->N2; ++k) {
        long double a = -2.0L * PI * k / p->N2;
        tn2[k] = make_double2((double)cosl(a), (double)sinl(a));
    }
    std::vector<long double> br(N, 0.0L), bi(N, 0.0L);
    for (int64_t j = 0; j < M; ++j) {
        const int64_t q = (int64_t)((__int128)j * j % (2 * M));  // exact j^2 mod 2M
        long double a = -PI * (long double)q / (long double)M;
        long double c = cosl(a), s = sinl(a);
        chirp[j] = make_double2((double)c, (double)s);
        br[j] = c;
        bi[j] = -s;  // conj
        if (j > 0) {
            br[N - j] = c;
            bi[N - j] = -s;
        }
    }
    for (int k = 0; k < 64; ++k) {
        long double a = -2.0L * PI * k / N;
        tlo[k] = make_double2((double)cosl(a), (double)sinl(a));
    }
    for (int k = 0; k < N / 64; ++k) {
        long double a = -2.0L * PI * (64.0L * k) / N;
        thi[k] = make_double2((double)cosl(a), (double)sinl(a));
    }
    if (p->P9)
        host_fft23_ld(br, bi);
    else if (mixed)
        host_fft3_ld(br, bi);
    else
        host_fft_ld(br, bi);
    for (int k = 0; k < N; ++k) {
        int dst = k;
        if (p->N1) {  // B^[k2 + N2 k1] stored at [k2][k1]
            const int k2 = k % p->N2, k1 = k / p->N2;
            dst = k2 * p->N1 + k1;
        } else if (p->P9) {  // B^[k1 + 9 k2] stored at [k1][k2] (bluestein_small9)
            dst = (k % 9) * p->P9 + k / 9;
        }
        bh[dst] = make_double2((double)(br[k] / N), (double)(bi[k] / N));
    }
    auto up = [](double2** d, const std::vector<double2>& h) -> cudaError_t {
        cudaError_t e = cudaMalloc(d, h.size() * sizeof(double2));
        if (e != cudaSuccess) return e;
        return cudaMemcpy(*d, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice);
    };
    cudaError_t e;
    if ((e = up(&p->chirp, chirp)) != cudaSuccess || (e = up(&p->bhat, bh)) != cudaSuccess ||
        (e = up(&p->tw_hi, thi)) != cudaSuccess || (e = up(&p->tw_lo, tlo)) != cudaSuccess ||
        (e = up(&p->tw_n1, tn1)) != cudaSuccess || (e = up(&p->tw_n2, tn2)) != cudaSuccess) {
        cudaFree(p->chirp);
        cudaFree(p->bhat);
        cudaFree(p->tw_hi);
        cudaFree(p->tw_lo);
        cudaFree(p->tw_n1);
        cudaFree(p->tw_n2);
        delete p;
        set_error(std::string("Bluestein plan upload: ") + cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? SFFTB_ENOMEM : SFFTB_ECUDA;
    }
    // the uploads are pageable cudaMemcpy on the legacy stream: such a copy can
    // return before its DMA has finished, and the kernels that read the tables
    // run on non-blocking streams that do not order after the legacy stream.
    // One-time cost per (device, M).
    if ((e = cudaStreamSynchronize(cudaStreamLegacy)) != cudaSuccess) {
        set_error(std::string("Bluestein plan upload: ") + cudaGetErrorString(e));
        return SFFTB_ECUDA;
    }
    *out = p;
    return SFFTB_OK;
}

static int get_plan(int64_t M, BluesteinPlan** out) {
    int dev = 0;
    SFFTB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto key = std::make_pair(dev, M);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
        *out = it->second;
        return SFFTB_OK;
    }
    BluesteinPlan* p = nullptr;
    int rc = build_plan(M, &p);
    if (rc != SFFTB_OK) return rc;
    g_plans[key] = p;
    *out = p;
    return SFFTB_OK;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

struct DftArgs {
    const double2* x;
    int64_t xs;
    double2* y;
    int64_t ys;
    int64_t M;
    double scale;
    const double2* chirp;
    const double2* bhat;
    const double2* tw_hi;
    const double2* tw_lo;
    const double2* tw_n1;
    const double2* tw_n2;
    double2* work;  // four-step workspace, batch * N
    int hi_in_smem;  // four-step: copy tw_hi into shared memory
    int64_t ntiles;  // four-step: tiles of the current kernel (persistent grid)
    // fused sampler -> detection path (sfftb_sample_detect_dft)
    double* sumsq_part;     // [batch][N1/F] partial sums of |sample|^2
    uint64_t noise_seed;
    int64_t noise_call0;
    double noise_sigma;
    const double* theta;    // [batch / L] zero-test thresholds
    int L;
    uint32_t* bits;         // [batch][W] nonzero bitmaps
    int64_t W;
    // sparse sampler input (fs2_colA<.., SPARSE>): per transform a list of
    // ls entries (residue, bin value), residue ~0 = no entry
    const uint32_t* lr;
    const double2* lv;
    int64_t ls;
    int pdl = 0;  // launch the fused chain's kernels with programmatic dependent launch
};

// Grid of the four-step passes: 8 CTAs per SM (2 resident at a time), each
// striding over ~2 tiles at the metric's stage shape.  Measured on B200 against
// fully persistent grids (2 per SM): the reconstruction 4.40 -> 4.17 ms, the
// standalone chain 0.405 -> 0.395 ms -- finer CTA granularity lets the
// high-priority detection kernels of the other stream interleave, and evens
// out the last wave (tools/env_sweep.sh SFFTB_FS_CTAS 2 4 6 8 12 16 100).
static int fs_grid(int64_t ntiles, bool rows = false) {
    static int per_sm = -1, per_sm_rows = -1;
    if (per_sm < 0) {
        const char* e = getenv("SFFTB_FS_CTAS");
        per_sm = e ? std::max(1, atoi(e)) : 8;
        const char* er = getenv("SFFTB_FS_CTAS_ROWS");
        per_sm_rows = er ? std::max(1, atoi(er)) : 16;  // rows: 16 measured ~0.5% better
    }
    const int k = rows ? per_sm_rows : per_sm;
    return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms() * k));
}

// fs2_rowB192 keeps every row inside a warp (no CTA barrier in its tile loop),
// so fewer, longer-lived CTAs pay: their warps drift apart over the tiles and
// hide each other's load latency, and the 16 KB of tables are staged once per
// ~3 tiles.  Measured (profiles/r02/ab_rowB192_warp_rows.txt): 6 CTAs per SM
// 3.94-3.97 ms per reconstruction, 16 per SM 3.98-4.00 ms.
static int fs_grid_rows192(int64_t ntiles) {
    static int per_sm = -1;
    if (per_sm < 0) {
        const char* e = getenv("SFFTB_FS_CTAS_ROWS");
        per_sm = e ? std::max(1, atoi(e)) : 6;
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms() * per_sm));
}

template <bool C>
__device__ __forceinline__ double2 conj_if(double2 v) {
    return C ? make_double2(v.x, -v.y) : v;
}

// cooperative copy of n double2 into shared memory
__device__ __forceinline__ void stage(double2* dst, const double2* __restrict__ src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

// One CTA per transform; N/16 threads.  Shared: data | tw_hi (N/64) | tw_lo (64).
template <int N, bool INV>
__global__ void __launch_bounds__(N / 16) bluestein_small(DftArgs a) {
    extern __shared__ double2 smem[];
    constexpr int DATA = N + N / 16;
    double2* hi = smem + DATA;
    double2* lo = hi + N / 64;
    const int tid = threadIdx.x;
    constexpr int T = N / 16;
    const int64_t b = blockIdx.x;
    stage(hi, a.tw_hi, N / 64);
    stage(lo, a.tw_lo, 64);
    const double2* x = a.x + b * a.xs;
    for (int i = tid; i < N; i += T) {
        double2 v = make_double2(0.0, 0.0);
        if (i < a.M) v = cmul(conj_if<INV>(x[i]), a.chirp[i]);
        smem[pad16(i)] = v;
    }
    __syncthreads();
    const TwTwoLevel tw{hi, lo, 1};
    fft_smem<N, false>(smem, tid, tw);
    for (int i = tid; i < N; i += T) smem[pad16(i)] = cmul(smem[pad16(i)], a.bhat[i]);
    __syncthreads();
    fft_smem<N, true>(smem, tid, tw);
    double2* y = a.y + b * a.ys;
    for (int h = tid; h < a.M; h += T) {
        double2 v = cmul(a.chirp[h], smem[pad16(h)]);
        y[h] = cscale(conj_if<INV>(v), a.scale);
    }
}

// e^{-+2 pi i m/9}, m in {1, 2, 4} (the products b c of the 3 x 3 split)
template <bool INV>
__device__ __forceinline__ double2 w9(int m) {
    double2 w;
    switch (m) {
        case 1: w = make_double2(0.76604444311897803520, -0.64278760968653932632); break;
        case 2: w = make_double2(0.17364817766693034885, -0.98480775301220805936); break;
        default: w = make_double2(-0.93969262078590838405, -0.34202014332566873304); break;
    }
    if (INV) w.y = -w.y;
    return w;
}

// 9-point DFT, natural order: n = 3a + b, k = c + 3d,
// X[c + 3d] = sum_b w3^{bd} w9^{bc} sum_a x[3a + b] w3^{ac}.
template <bool INV>
__device__ __forceinline__ void dft9(double2 (&v)[9]) {
    double2 y[3][3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        double2 p = v[b], q = v[3 + b], r = v[6 + b];
        dft3<INV>(p, q, r);
        y[b][0] = p;
        y[b][1] = b ? cmul(q, w9<INV>(b)) : q;
        y[b][2] = b ? cmul(r, w9<INV>(2 * b)) : r;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double2 p = y[0][c], q = y[1][c], r = y[2][c];
        dft3<INV>(p, q, r);
        v[c] = p;
        v[c + 3] = q;
        v[c + 6] = r;
    }
}

// Single-CTA Bluestein for N = 9 P (P a power of two, 64..512): with
// j = P r + p and k = k1 + 9 k2,
//   X[k1 + 9 k2] = sum_p w_P^{p k2} [w_N^{p k1} sum_r x[P r + p] w_9^{r k1}],
// so the data live as 9 sub-arrays of P (sub-array r holds x[P r + .]): a
// 9-point DFT down every column p with the twiddle w_N^{p k1}, then 9
// concurrent P-point Stockham FFTs (fft_smem, P/16 threads each) leave
// X[k1 + 9 k2] at sub-array k1, position k2 -- the layout B^ is stored in.
// The inverse runs the same steps backwards and ends in natural order.
template <int P, bool INV>
__global__ void __launch_bounds__(9 * P / 16) bluestein_small9(DftArgs a) {
    extern __shared__ double2 smem[];
    constexpr int N = 9 * P, T = N / 16, SUB = P + P / 16, TPF = P / 16;
    double2* hi = smem + 9 * SUB;
    double2* lo = hi + N / 64;
    const int tid = threadIdx.x;
    const int64_t b = blockIdx.x;
    stage(hi, a.tw_hi, N / 64);
    stage(lo, a.tw_lo, 64);
    const double2* x = a.x + b * a.xs;
    for (int i = tid; i < N; i += T) {
        double2 v = make_double2(0.0, 0.0);
        if (i < a.M) v = cmul(conj_if<INV>(x[i]), a.chirp[i]);
        smem[(i / P) * SUB + pad16(i % P)] = v;
    }
    __syncthreads();
    const TwTwoLevel twN{hi, lo, 1};
    const TwTwoLevel twP{hi, lo, 9};
    double2* sub = smem + (tid / TPF) * SUB;
    const int tpf = tid % TPF;
    // forward: radix 9 down the columns, twiddle w_N^{p k1}
    for (int p = tid; p < P; p += T) {
        double2 v[9];
#pragma unroll
        for (int r = 0; r < 9; ++r) v[r] = smem[r * SUB + pad16(p)];
        dft9<false>(v);
#pragma unroll
        for (int k1 = 0; k1 < 9; ++k1)
            smem[k1 * SUB + pad16(p)] = (k1 && p) ? cmul(v[k1], twN.template get<false>(p * k1))
                                                  : v[k1];
    }
    __syncthreads();
    fft_smem<P, false>(sub, tpf, twP);
    for (int i = tid; i < N; i += T) {
        const int k1 = i / P, k2 = i % P;
        double2* e = smem + k1 * SUB + pad16(k2);
        *e = cmul(*e, a.bhat[i]);
    }
    __syncthreads();
    // inverse: P-point IFFTs, twiddle w_N^{-p k1}, radix 9 back to natural order
    fft_smem<P, true>(sub, tpf, twP);
    for (int p = tid; p < P; p += T) {
        double2 v[9];
#pragma unroll
        for (int k1 = 0; k1 < 9; ++k1) {
            const double2 u = smem[k1 * SUB + pad16(p)];
            v[k1] = (k1 && p) ? cmul(u, twN.template get<true>(p * k1)) : u;
        }
        dft9<true>(v);
#pragma unroll
        for (int r = 0; r < 9; ++r) smem[r * SUB + pad16(p)] = v[r];
    }
    __syncthreads();
    double2* y = a.y + b * a.ys;
    for (int h = tid; h < a.M; h += T) {
        double2 v = cmul(a.chirp[h], smem[(h / P) * SUB + pad16(h % P)]);
        y[h] = cscale(conj_if<INV>(v), a.scale);
    }
}

// four-step shared layout: F slots of SLOT (+1 pad slot: the column gathers
// of F lanes then spread over all 16-byte bank groups) | sub-FFT table |
// tw_lo (64) | tw_hi (N/64, when it fits)
template <int LEN>
struct FsLayout {
    static constexpr int TPF = LEN / 16;
    static constexpr int F = 256 / TPF;
    static constexpr int SLOT = LEN + LEN / 16 + 1;
    static constexpr int DATA = F * SLOT;
};

// colA: CTA = F columns n1 of the N1 x N2 view, length-N2 forward FFTs.
template <int N2, bool INV>
__global__ void __launch_bounds__(256, 2) fs_colA(DftArgs a, int N1) {
    using Lay = FsLayout<N2>;
    constexpr int TPF = Lay::TPF, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw2 = smem + Lay::DATA;
    double2* lo = tw2 + N2;
    double2* hi_s = lo + 64;
    const int tid = threadIdx.x;
    const int N = N1 * N2;
    stage(tw2, a.tw_n2, N2);
    stage(lo, a.tw_lo, 64);
    if (a.hi_in_smem) stage(hi_s, a.tw_hi, N / 64);
    const double2* hi = a.hi_in_smem ? hi_s : a.tw_hi;
    constexpr int PER = F * N2 / 256;  // elements per thread
    const int per_b = N1 / F;
    // persistent: tables staged once, then tiles (transform b, columns n1_0..)
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t b = tile / per_b;
    const int n1_0 = (int)(tile % per_b) * F;
    const double2* x = a.x + b * a.xs;
    __syncthreads();
    {
        // all loads of the tile in flight before any use (memory-level parallelism)
        double2 v[PER], c[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            const int64_t j = n1_0 + e % F + (int64_t)N1 * (e / F);
            v[i] = make_double2(0.0, 0.0);
            c[i] = make_double2(0.0, 0.0);
            if (j < a.M) {
                v[i] = __ldg(x + j);
                c[i] = __ldg(a.chirp + j);
            }
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            smem[(e % F) * SLOT + pad16(e / F)] = cmul(conj_if<INV>(v[i]), c[i]);
        }
    }
    __syncthreads();
    const int f_me = tid / TPF;
    fft_smem<N2, false>(smem + f_me * SLOT, tid % TPF, TwDirect{tw2});
    double2* T = a.work + b * (int64_t)N;
    for (int e = tid; e < F * N2; e += 256) {
        const int f = e % F, k2 = e / F;
        const int n1 = n1_0 + f;
        double2 v = smem[f * SLOT + pad16(k2)];
        const int ex = n1 * k2;  // < N
        if (ex) v = cmul(v, twiddle2<false>(hi, lo, ex));
        T[(int64_t)k2 * N1 + n1] = v;
    }
    }
}

// rowB: CTA = F rows k2, forward FFT_N1 -> * B^ -> inverse FFT_N1 -> conj twiddle.
template <int N1>
__global__ void __launch_bounds__(256, 2) fs_rowB(DftArgs a, int N2) {
    using Lay = FsLayout<N1>;
    constexpr int TPF = Lay::TPF, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw1 = smem + Lay::DATA;
    double2* lo = tw1 + N1;
    double2* hi_s = lo + 64;
    const int tid = threadIdx.x;
    const int N = N1 * N2;
    stage(tw1, a.tw_n1, N1);
    stage(lo, a.tw_lo, 64);
    if (a.hi_in_smem) stage(hi_s, a.tw_hi, N / 64);
    const double2* hi = a.hi_in_smem ? hi_s : a.tw_hi;
    constexpr int PER = F * N1 / 256;
    const int per_b = N2 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t b = tile / per_b;
    const int k2_0 = (int)(tile % per_b) * F;
    double2* T = a.work + b * (int64_t)N;
    __syncthreads();
    {
        double2 v[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            v[i] = T[(int64_t)(k2_0 + e / N1) * N1 + e % N1];
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            smem[(e / N1) * SLOT + pad16(e % N1)] = v[i];
        }
    }
    __syncthreads();
    const int f_me = tid / TPF;
    double2* mine = smem + f_me * SLOT;
    const TwDirect tw{tw1};
    fft_smem<N1, false>(mine, tid % TPF, tw);
    {
        double2 bh[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            bh[i] = __ldg(a.bhat + (int64_t)(k2_0 + e / N1) * N1 + e % N1);
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            double2* p = smem + (e / N1) * SLOT + pad16(e % N1);
            *p = cmul(*p, bh[i]);
        }
    }
    __syncthreads();
    fft_smem<N1, true>(mine, tid % TPF, tw);
    for (int e = tid; e < F * N1; e += 256) {
        const int f = e / N1, m1 = e % N1;
        const int k2 = k2_0 + f;
        double2 v = smem[f * SLOT + pad16(m1)];
        const int ex = m1 * k2;
        if (ex) v = cmul(v, twiddle2<true>(hi, lo, ex));
        T[(int64_t)k2 * N1 + m1] = v;
    }
    }
}

// colC: CTA = F columns m1, inverse length-N2 FFTs, chirp, scale, output.
template <int N2, bool INV>
__global__ void __launch_bounds__(256, 2) fs_colC(DftArgs a, int N1) {
    using Lay = FsLayout<N2>;
    constexpr int TPF = Lay::TPF, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw2 = smem + Lay::DATA;
    const int tid = threadIdx.x;
    const int N = N1 * N2;
    stage(tw2, a.tw_n2, N2);
    constexpr int PER = F * N2 / 256;
    const int per_b = N1 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t b = tile / per_b;
    const int m1_0 = (int)(tile % per_b) * F;
    const double2* T = a.work + b * (int64_t)N;
    __syncthreads();
    {
        double2 v[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            v[i] = T[(int64_t)(e / F) * N1 + m1_0 + e % F];
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = tid + i * 256;
            smem[(e % F) * SLOT + pad16(e / F)] = v[i];
        }
    }
    __syncthreads();
    const int f_me = tid / TPF;
    fft_smem<N2, true>(smem + f_me * SLOT, tid % TPF, TwDirect{tw2});
    double2* y = a.y + b * a.ys;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = tid + i * 256;
        const int64_t h = m1_0 + e % F + (int64_t)N1 * (e / F);
        if (h < a.M) {
            double2 v = cmul(__ldg(a.chirp + h), smem[(e % F) * SLOT + pad16(e / F)]);
            y[h] = cscale(conj_if<INV>(v), a.scale);
        }
    }
    }
}

// ---------------------------------------------------------------------------
// Register-pass four-step kernels for sub-FFT lengths 128 and 256 (the sfft
// sizes N = 32768, 65536): global -> registers (pass 1) -> one smem
// transpose -> registers (pass 2) -> global.  rowB keeps the forward
// outputs in registers through the B^ product and the inverse pass 1.
// ---------------------------------------------------------------------------

// smem: F slots | sub-FFT table (LEN) | tw_lo (64) | tw_hi (N/64, optional)
template <int LEN>
struct Fs2Layout {
    static constexpr int T = LEN / 16;
    static constexpr int F = 256 / T;
    static constexpr int SLOT = LEN + LEN / 16 + 1;
    static constexpr int DATA = F * SLOT;
};

template <int N2, bool INV, bool SPARSE = false, int N1C = 0>
__global__ void __launch_bounds__(256, 2) fs2_colA(DftArgs a, int N1_rt) {
    const int N1 = N1C ? N1C : N1_rt;  // compile-time N1: immediate offsets
    using Lay = Fs2Layout<N2>;
    constexpr int T = Lay::T, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw2 = smem + Lay::DATA;
    double2* lo = tw2 + N2;
    double2* hi_s = lo + 64;
    const int tid = threadIdx.x;
    const int f = tid % F, t = tid / F;  // columns fastest: coalesced rows
    const int N = N1 * N2;
    stage(tw2, a.tw_n2, N2);
    stage(lo, a.tw_lo, 64);
    const bool hi_smem = N1C ? true : (bool)a.hi_in_smem;
    if (hi_smem) stage(hi_s, a.tw_hi, N / 64);
    const double2* hi = hi_smem ? hi_s : a.tw_hi;
    pdl_wait();    // the predecessor's output (constant tables staged above)
    pdl_launch();
    double2* slot = smem + f * SLOT;
    const int per_b = N1 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const int64_t b = tile / per_b;
        const int n1 = (int)(tile % per_b) * F + f;
        double2 v[16];
        if (SPARSE) {
            // the tile's columns [n1_0, n1_0 + F) of the N1 x N2 view: zero
            // them in the slots, drop in the listed bins, read them back
            const int n1_0 = n1 - f;
            __syncthreads();  // previous tile done with the slots
            for (int i = tid; i < F * N2; i += 256) smem[(i / N2) * SLOT + (i % N2)] =
                make_double2(0.0, 0.0);
            __syncthreads();
            // list values already carry the chirp product (sfftb_scatter_list);
            // residues and values of U entries per thread are loaded at once
            const uint32_t* lr = a.lr + b * a.ls;
            const double2* lv = a.lv + b * a.ls;
            // r / N1 by multiply-high with ceil(2^32 / N1): exact for r < 2^24
            const uint32_t magic = (uint32_t)((0x100000000ull + (uint32_t)N1 - 1) / (uint32_t)N1);
            constexpr int U = 4;
            for (int64_t k0 = tid; k0 < a.ls; k0 += 256 * U) {
                uint32_t rr[U];
                double2 vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t k = k0 + 256 * u;
                    rr[u] = k < a.ls ? __ldg(lr + k) : ~0u;
                    vv[u] = k < a.ls ? __ldg(lv + k) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (rr[u] == ~0u) continue;
                    const uint32_t q = __umulhi(rr[u], magic);
                    const int c = (int)(rr[u] - q * (uint32_t)N1) - n1_0;
                    if (c >= 0 && c < F) smem[c * SLOT + (int)q] = vv[u];
                }
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = slot[t + r * T];
            __syncthreads();  // fft2pass reuses the slots
        } else {
            const double2* x = a.x + b * a.xs;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int64_t j = n1 + (int64_t)N1 * (t + r * T);
                v[r] = make_double2(0.0, 0.0);
                if (j < a.M) v[r] = cmul(conj_if<INV>(__ldg(x + j)), __ldg(a.chirp + j));
            }
            __syncthreads();  // previous tile done with the slots
        }
        fft2pass<N2, false>(v, slot, t, tw2);
        out_twiddle<N2, false>(v, n1, t, hi, lo);
        double2* Tw = a.work + b * (int64_t)N;
#pragma unroll
        for (int e = 0; e < 16; ++e) Tw[(int64_t)fft2_out_index<N2>(t, e) * N1 + n1] = v[e];
    }
}

template <int N1>
__global__ void __launch_bounds__(256, 2) fs2_rowB(DftArgs a, int N2) {
    using Lay = Fs2Layout<N1>;
    constexpr int T = Lay::T, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw1 = smem + Lay::DATA;
    double2* lo = tw1 + N1;
    double2* hi_s = lo + 64;
    const int tid = threadIdx.x;
    const int f = tid / T, t = tid % T;  // row elements fastest: coalesced
    const int N = N1 * N2;
    stage(tw1, a.tw_n1, N1);
    stage(lo, a.tw_lo, 64);
    if (a.hi_in_smem) stage(hi_s, a.tw_hi, N / 64);
    const double2* hi = a.hi_in_smem ? hi_s : a.tw_hi;
    double2* slot = smem + f * SLOT;
    const int per_b = N2 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const int64_t b = tile / per_b;
        const int k2 = (int)(tile % per_b) * F + f;
        double2* row = a.work + b * (int64_t)N + (int64_t)k2 * N1;
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = row[t + r * T];
        __syncthreads();
        fft2pass<N1, false>(v, slot, t, tw1);
        const double2* bh = a.bhat + (int64_t)k2 * N1;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = cmul(v[e], __ldg(bh + fft2_out_index<N1>(t, e)));
        fft2_out_to_in<N1>(v);
        fft2pass<N1, true>(v, slot, t, tw1);
        out_twiddle<N1, true>(v, k2, t, hi, lo);
#pragma unroll
        for (int e = 0; e < 16; ++e) row[fft2_out_index<N1>(t, e)] = v[e];
    }
}

// Row pass for the mixed-radix length N = 192 * N2 (N1 = 192 = 16 x 12):
// forward 192-point FFT (radix 12 on 16 threads, one transpose, radix 16 on
// 12 threads), x B^, inverse 192-point FFT (radix 16 on the same 12 threads
// straight from registers, one transpose, radix 12 on 16 threads), four-step
// twiddle.  Index maps: j = t + 16 r (t < 16, r < 12), k = s + 12 q
// (s < 12, q < 16); w192^{jk} = w192^{ts} w16^{tq} w12^{rs}.
// Per-row shared slots: 16 x 13 (pass-1 layout [t][s]) and 12 x 17 (inverse
// layout [s][t]) in 212 double2 -- the +4 pad puts neighbouring rows in the
// other half of the banks for the remapped middle pass.
static constexpr int kR192Slot = 212;
template <int N2C = 0>
__global__ void __launch_bounds__(256, 2) fs2_rowB192(DftArgs a, int N2_rt) {
    const int N2 = N2C ? N2C : N2_rt;  // compile-time N2: immediate offsets
    constexpr int N1 = 192, F = 16;
    extern __shared__ double2 smem[];
    double2* tw1 = smem + F * kR192Slot;  // e^{-2 pi i m/192}
    double2* lo = tw1 + N1;
    double2* hi_s = lo + 64;
    const int tid = threadIdx.x;
    const int f = tid >> 4, t = tid & 15;
    // middle passes: the 12 columns of row f on lanes t < 12 of the row's own
    // half-warp, so that a row never leaves its warp: every exchange through the
    // row's slot needs a warp barrier only (no CTA barrier in the tile loop)
    const bool mid = t < 12;
    const int f2 = f, sc = t;
    const int N = N1 * N2;
    stage(tw1, a.tw_n1, N1);
    stage(lo, a.tw_lo, 64);
    // N = 192 * N2 <= 49152: the N / 64 <= 768 high twiddles always fit in
    // shared memory (a.hi_in_smem is set for them), so no generic pointer
    stage(hi_s, a.tw_hi, N / 64);
    const double2* hi = hi_s;
    pdl_wait();    // the predecessor's output (constant tables staged above)
    pdl_launch();
    __syncthreads();  // the staged tables
    double2* slot = smem + f * kR192Slot;
    double2* slot2 = smem + f2 * kR192Slot;
    const int per_b = N2 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const int64_t b = tile / per_b;
        const int kbase = (int)(tile % per_b) * F;
        const int k2 = kbase + f;
        double2* row = a.work + b * (int64_t)N + (int64_t)k2 * N1;
        double2 x[12];
#pragma unroll
        for (int r = 0; r < 12; ++r) x[r] = row[t + 16 * r];
        __syncwarp();  // previous tile done with the row's slot
        // forward pass 1: radix 12 over r, twiddle w192^{t s} (powers of w^t)
        dft12<false>(x);
        {
            const Pow16 p(tw1[t], tw1[2 * t], tw1[4 * t], tw1[8 * t]);
#pragma unroll
            for (int sI = 0; sI < 12; ++sI) slot[t * 13 + sI] = sI ? cmul(x[sI], p(sI)) : x[sI];
        }
        __syncwarp();
        double2 u[16];
        if (mid) {
            // forward pass 2: radix 16 over t' for column sc of row f2
#pragma unroll
            for (int tp = 0; tp < 16; ++tp) u[tp] = slot2[tp * 13 + sc];
            dft_reg<16, false>(u);  // u[q] = X[sc + 12 q]
            const double2* bh = a.bhat + (int64_t)(kbase + f2) * N1;
#pragma unroll
            for (int q = 0; q < 16; ++q) u[q] = cmul(u[q], __ldg(bh + sc + 12 * q));
            // inverse pass A: radix 16 over q
            dft_reg<16, true>(u);  // u[t'] = sum_q X w16^{-t' q}
        }
        __syncwarp();  // pass-2 loads done before the slot is rewritten
        if (mid) {
            // twiddle w192^{-t' s} from the powers of conj(w^s)
            const Pow16 p(conj_if_b(tw1[sc], true), conj_if_b(tw1[2 * sc], true),
                          conj_if_b(tw1[4 * sc], true), conj_if_b(tw1[8 * sc], true));
#pragma unroll
            for (int tp = 0; tp < 16; ++tp)
                slot2[sc * 17 + tp] = tp ? cmul(u[tp], p(tp)) : u[tp];
        }
        __syncwarp();
        // inverse pass B: radix 12 over s for t' = t
#pragma unroll
        for (int sI = 0; sI < 12; ++sI) x[sI] = slot[sI * 17 + t];
        dft12<true>(x);  // x[r] = y[t + 16 r]
        // four-step twiddle w^{-(t + 16 r) k2}: base w^{-t k2} x (w^{-16 k2})^r
        if (k2) {
            const Pow16 p(twiddle2<true>(hi, lo, 16 * k2), twiddle2<true>(hi, lo, 32 * k2),
                          twiddle2<true>(hi, lo, 64 * k2), twiddle2<true>(hi, lo, 128 * k2));
            const double2 base = twiddle2<true>(hi, lo, t * k2);
            x[0] = cmul(x[0], base);
#pragma unroll
            for (int r = 1; r < 12; ++r) x[r] = cmul(x[r], cmul(base, p(r)));
        }
#pragma unroll
        for (int r = 0; r < 12; ++r) row[t + 16 * r] = x[r];
    }
}

template <int N2, bool INV>
__global__ void __launch_bounds__(256, 2) fs2_colC(DftArgs a, int N1) {
    using Lay = Fs2Layout<N2>;
    constexpr int T = Lay::T, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw2 = smem + Lay::DATA;
    const int tid = threadIdx.x;
    const int f = tid % F, t = tid / F;
    const int N = N1 * N2;
    stage(tw2, a.tw_n2, N2);
    double2* slot = smem + f * SLOT;
    const int per_b = N1 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const int64_t b = tile / per_b;
        const int m1 = (int)(tile % per_b) * F + f;
        const double2* Tw = a.work + b * (int64_t)N;
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = Tw[(int64_t)(t + r * T) * N1 + m1];
        __syncthreads();
        fft2pass<N2, true>(v, slot, t, tw2);
        double2* y = a.y + b * a.ys;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int64_t h = m1 + (int64_t)N1 * fft2_out_index<N2>(t, e);
            if (h < a.M) {
                const double2 w = cmul(__ldg(a.chirp + h), v[e]);
                y[h] = cscale(conj_if<INV>(w), a.scale);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Fused sampler -> detection chain for the register-pass sizes.
//
// colCA = (sampler inverse colC) + (detection forward colA) on the same
// column tile: inverse column FFT -> samples y = conj(w c) (+ harness noise)
// -> per-tile sum |y|^2 for the zero test -> x = y w -> forward column FFT ->
// four-step twiddle.  Samples never reach HBM.  colC_bits = detection colC
// that also emits the nonzero bitmap (|ghat| > theta, _core.pyx:195).
// ---------------------------------------------------------------------------
// N1C: the row length N1 as a compile-time constant (0: runtime N1); with it
// every load/store offset of a thread folds into an immediate, which keeps
// the kernel inside its 128 registers without spilling addresses
template <int N2, bool NOISE, int N1C = 0>
__global__ void __launch_bounds__(256, 2) fs2_colCA(DftArgs a, int N1_rt) {
    const int N1 = N1C ? N1C : N1_rt;
    using Lay = Fs2Layout<N2>;
    constexpr int T = Lay::T, F = Lay::F, SLOT = Lay::SLOT;
    extern __shared__ double2 smem[];
    double2* tw2 = smem + Lay::DATA;
    double2* lo = tw2 + N2;
    double2* hi_s = lo + 64;
    __shared__ double red[8];
    const int tid = threadIdx.x;
    const int f = tid % F, t = tid / F;
    const int N = N1 * N2;
    stage(tw2, a.tw_n2, N2);
    stage(lo, a.tw_lo, 64);
    // compile-time N1: N <= 256 * 256, so N / 64 <= 2048 twiddles always fit
    const bool hi_smem = N1C ? true : (bool)a.hi_in_smem;
    if (hi_smem) stage(hi_s, a.tw_hi, N / 64);
    const double2* hi = hi_smem ? hi_s : a.tw_hi;
    pdl_wait();    // the predecessor's output (constant tables staged above)
    pdl_launch();
    double2* slot = smem + f * SLOT;
    const int per_b = N1 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const int64_t b = tile / per_b;
        const int m1 = (int)(tile % per_b) * F + f;
        double2* Tw = a.work + b * (int64_t)N;
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = Tw[(int64_t)(t + r * T) * N1 + m1];
        __syncthreads();
        fft2pass<N2, true>(v, slot, t, tw2);
        double ss = 0.0;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int64_t h = m1 + (int64_t)N1 * fft2_out_index<N2>(t, e);
            double2 x = make_double2(0.0, 0.0);
            if (h < a.M) {
                const double2 w = __ldg(a.chirp + h);
                double2 y = cmul(w, v[e]);
                y.y = -y.y;  // sample: conj(w c), the M*ifft of the bins
                if (NOISE) {
                    const double2 nz = harness_noise(a.noise_seed,
                                                     (uint64_t)(a.noise_call0 + b), h,
                                                     a.noise_sigma);
                    y.x += nz.x;
                    y.y += nz.y;
                }
                ss = fma(y.x, y.x, fma(y.y, y.y, ss));
                x = cmul(y, w);  // detection chirp
            }
            v[e] = x;
        }
        // per-tile sum of |y|^2 in a fixed order (deterministic zero test)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
        if ((tid & 31) == 0) red[tid >> 5] = ss;
        fft2_out_to_in<N2>(v);
        fft2pass<N2, false>(v, slot, t, tw2);  // (its syncs also publish red[])
        if (tid == 0) {
            double s8 = 0.0;
            for (int w8 = 0; w8 < 8; ++w8) s8 += red[w8];
            a.sumsq_part[b * per_b + tile % per_b] = s8;
        }
        out_twiddle<N2, false>(v, m1, t, hi, lo);
#pragma unroll
        for (int e = 0; e < 16; ++e) Tw[(int64_t)fft2_out_index<N2>(t, e) * N1 + m1] = v[e];
    }
}

template <int N2, int N1C = 0>
__global__ void __launch_bounds__(256, 2) fs2_colC_bits(DftArgs a, int N1_rt) {
    const int N1 = N1C ? N1C : N1_rt;
    using Lay = Fs2Layout<N2>;
    constexpr int T = Lay::T, F = Lay::F, SLOT = Lay::SLOT;
    static_assert(F == 16 || F == 32, "bit groups of F consecutive bins");
    extern __shared__ double2 smem[];
    double2* tw2 = smem + Lay::DATA;
    const int tid = threadIdx.x;
    const int f = tid % F, t = tid / F;
    const int lane = tid & 31;
    const int N = N1 * N2;
    stage(tw2, a.tw_n2, N2);
    pdl_wait();    // the predecessor's output (constant tables staged above)
    pdl_launch();
    double2* slot = smem + f * SLOT;
    const int per_b = N1 / F;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const int64_t b = tile / per_b;
        const int m1_0 = (int)(tile % per_b) * F;
        const int m1 = m1_0 + f;
        const double th = a.theta[b / a.L];
        const double2* Tw = a.work + b * (int64_t)N;
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = Tw[(int64_t)(t + r * T) * N1 + m1];
        __syncthreads();
        fft2pass<N2, true>(v, slot, t, tw2);
        double2* y = a.y + b * a.ys;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int64_t m2 = fft2_out_index<N2>(t, e);
            const int64_t h = m1 + (int64_t)N1 * m2;
            bool nz = false;
            if (h < a.M) {
                const double2 g = cscale(cmul(__ldg(a.chirp + h), v[e]), a.scale);
                y[h] = g;
                nz = nonzero_test(g.x, g.y, th);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, nz);
            // lanes hold F consecutive bins of 32/F rows m2: bins m1_0 + N1*m2
            // start on an F-aligned bit, so each F-bit group is one store
            if (F == 32) {
                if (lane == 0 && (m1_0 + (int64_t)N1 * m2) < a.M)
                    a.bits[b * a.W + ((m1_0 + (int64_t)N1 * m2) >> 5)] = bal;
            } else if (f == 0) {
                const int64_t h0 = m1_0 + (int64_t)N1 * m2;
                if (h0 < a.M) {
                    uint16_t* b16 = reinterpret_cast<uint16_t*>(a.bits + b * a.W);
                    b16[h0 >> 4] = (uint16_t)(bal >> (lane & 16));
                }
            }
        }
    }
}

__global__ void partial_sumsq_reduce(const double* __restrict__ part, int64_t rows, int per_b,
                                     double* __restrict__ out) {
    pdl_wait();
    pdl_launch();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < per_b; ++k) s += part[r * per_b + k];
        out[r] = s;
    }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------

template <typename K>
static cudaError_t allow_smem(K kernel, size_t bytes) {
    return smem_opt_in(kernel, bytes);
}

template <int N, bool INV>
static int launch_small(const DftArgs& a, int64_t batch, cudaStream_t st) {
    const size_t sm = sizeof(double2) * (N + N / 16 + N / 64 + 64);
    SFFTB_CUDA(allow_smem(bluestein_small<N, INV>, sm));
    bluestein_small<N, INV><<<(unsigned)batch, N / 16, sm, st>>>(a);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

template <int P, bool INV>
static int launch_small9(const DftArgs& a, int64_t batch, cudaStream_t st) {
    constexpr int N = 9 * P;
    const size_t sm = sizeof(double2) * (9 * (P + P / 16) + N / 64 + 64);
    SFFTB_CUDA(allow_smem(bluestein_small9<P, INV>, sm));
    bluestein_small9<P, INV><<<(unsigned)batch, N / 16, sm, st>>>(a);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

template <bool INV>
static int small9_dispatch(int P, const DftArgs& a, int64_t batch, cudaStream_t st) {
    switch (P) {
        case 64: return launch_small9<64, INV>(a, batch, st);
        case 128: return launch_small9<128, INV>(a, batch, st);
        case 256: return launch_small9<256, INV>(a, batch, st);
        case 512: return launch_small9<512, INV>(a, batch, st);
    }
    set_error("internal: bad 9 * 2^k Bluestein size");
    return SFFTB_EINVAL;
}

template <bool INV>
static int small_dispatch(int lg, const DftArgs& a, int64_t batch, cudaStream_t st) {
    switch (lg) {
        case 8: return launch_small<256, INV>(a, batch, st);
        case 9: return launch_small<512, INV>(a, batch, st);
        case 10: return launch_small<1024, INV>(a, batch, st);
        case 11: return launch_small<2048, INV>(a, batch, st);
        case 12: return launch_small<4096, INV>(a, batch, st);
        case 13: return launch_small<8192, INV>(a, batch, st);
    }
    set_error("internal: bad small Bluestein size");
    return SFFTB_EINVAL;
}

template <int N2, bool INV>
static int launch_cols(const DftArgs& a, int64_t batch, int N1, cudaStream_t st, bool first) {
    using Lay = FsLayout<N2>;
    constexpr int F = Lay::F;
    const size_t hi = a.hi_in_smem ? (size_t)(N1 * N2 / 64) : 0;
    const size_t sm = sizeof(double2) * (Lay::DATA + N2 + (first ? 64 + hi : 0));
    DftArgs c = a;
    c.ntiles = (int64_t)(N1 / F) * batch;
    const int grid = fs_grid(c.ntiles);
    if (first) {
        SFFTB_CUDA(allow_smem(fs_colA<N2, INV>, sm));
        fs_colA<N2, INV><<<grid, 256, sm, st>>>(c, N1);
    } else {
        SFFTB_CUDA(allow_smem(fs_colC<N2, INV>, sm));
        fs_colC<N2, INV><<<grid, 256, sm, st>>>(c, N1);
    }
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

template <int N1>
static int launch_rows(const DftArgs& a, int64_t batch, int N2, cudaStream_t st) {
    using Lay = FsLayout<N1>;
    constexpr int F = Lay::F;
    const size_t hi = a.hi_in_smem ? (size_t)(N1 * N2 / 64) : 0;
    const size_t sm = sizeof(double2) * (Lay::DATA + N1 + 64 + hi);
    SFFTB_CUDA(allow_smem(fs_rowB<N1>, sm));
    DftArgs c = a;
    c.ntiles = (int64_t)(N2 / F) * batch;
    const int grid = fs_grid(c.ntiles);
    fs_rowB<N1><<<grid, 256, sm, st>>>(c, N2);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

template <bool INV>
static int cols_dispatch(int N2, const DftArgs& a, int64_t batch, int N1, cudaStream_t st,
                         bool first) {
    switch (N2) {
        case 128: return launch_cols<128, INV>(a, batch, N1, st, first);
        case 256: return launch_cols<256, INV>(a, batch, N1, st, first);
        case 512: return launch_cols<512, INV>(a, batch, N1, st, first);
        case 1024: return launch_cols<1024, INV>(a, batch, N1, st, first);
    }
    set_error("internal: bad four-step column size");
    return SFFTB_EINVAL;
}

static int rows_dispatch(int N1, const DftArgs& a, int64_t batch, int N2, cudaStream_t st) {
    switch (N1) {
        case 128: return launch_rows<128>(a, batch, N2, st);
        case 256: return launch_rows<256>(a, batch, N2, st);
        case 512: return launch_rows<512>(a, batch, N2, st);
        case 1024: return launch_rows<1024>(a, batch, N2, st);
    }
    set_error("internal: bad four-step row size");
    return SFFTB_EINVAL;
}

template <int N2, bool INV, bool SPARSE = false>
static int fs2_cols(const DftArgs& a, int64_t batch, int N1, cudaStream_t st, bool first) {
    using Lay = Fs2Layout<N2>;
    const size_t hi = a.hi_in_smem ? (size_t)(N1 * N2 / 64) : 0;
    const size_t sm = sizeof(double2) * (Lay::DATA + N2 + (first ? 64 + hi : 0));
    DftArgs c = a;
    c.ntiles = (int64_t)(N1 / Lay::F) * batch;
    const int grid = fs_grid(c.ntiles);
    if (first) {
        if (N1 == 192) {
            SFFTB_CUDA(allow_smem(fs2_colA<N2, INV, SPARSE, 192>, sm));
            SFFTB_CUDA(launch_maybe_pdl(c.pdl, fs2_colA<N2, INV, SPARSE, 192>, dim3(grid),
                                        dim3(256), sm, st, c, N1));
        } else {
            SFFTB_CUDA(allow_smem(fs2_colA<N2, INV, SPARSE>, sm));
            fs2_colA<N2, INV, SPARSE><<<grid, 256, sm, st>>>(c, N1);
        }
    } else {
        SFFTB_CUDA(allow_smem(fs2_colC<N2, INV>, sm));
        fs2_colC<N2, INV><<<grid, 256, sm, st>>>(c, N1);
    }
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

static int fs2_rows192(const DftArgs& a, int64_t batch, int N2, cudaStream_t st) {
    const size_t hi = (size_t)(192 * N2 / 64);  // always staged (fs2_rowB192)
    const size_t sm = sizeof(double2) * (16 * kR192Slot + 192 + 64 + hi);
    DftArgs c = a;
    c.ntiles = (int64_t)(N2 / 16) * batch;
    const int grid = fs_grid_rows192(c.ntiles);
    // (a compile-time N2 spills more here and is no faster: runtime N2)
    SFFTB_CUDA(allow_smem(fs2_rowB192<>, sm));
    SFFTB_CUDA(launch_maybe_pdl(c.pdl, fs2_rowB192<>, dim3(grid), dim3(256), sm, st, c, N2));
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

template <int N1>
static int fs2_rows(const DftArgs& a, int64_t batch, int N2, cudaStream_t st) {
    if constexpr (N1 == 192) {
        return fs2_rows192(a, batch, N2, st);
    } else {
    using Lay = Fs2Layout<N1>;
    const size_t hi = a.hi_in_smem ? (size_t)(N1 * N2 / 64) : 0;
    const size_t sm = sizeof(double2) * (Lay::DATA + N1 + 64 + hi);
    DftArgs c = a;
    c.ntiles = (int64_t)(N2 / Lay::F) * batch;
    const int grid = fs_grid(c.ntiles, true);
    SFFTB_CUDA(allow_smem(fs2_rowB<N1>, sm));
    fs2_rowB<N1><<<grid, 256, sm, st>>>(c, N2);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
    }
}

// the row pass for any supported N1 (128, 192, 256)
static int fs2_rows_any(const DftArgs& a, int64_t batch, int N1, int N2, cudaStream_t st) {
    if (N1 == 256) return fs2_rows<256>(a, batch, N2, st);
    if (N1 == 192) return fs2_rows<192>(a, batch, N2, st);
    return fs2_rows<128>(a, batch, N2, st);
}

static bool fs2_supported(const BluesteinPlan* p) {
    return (p->N1 == 128 || p->N1 == 192 || p->N1 == 256) && (p->N2 == 128 || p->N2 == 256);
}

template <bool INV>
static int fs2_all(const BluesteinPlan* p, const DftArgs& a, int64_t batch, cudaStream_t st) {
    int rc = p->N2 == 256 ? fs2_cols<256, INV>(a, batch, p->N1, st, true)
                          : fs2_cols<128, INV>(a, batch, p->N1, st, true);
    if (rc) return rc;
    rc = fs2_rows_any(a, batch, p->N1, p->N2, st);
    if (rc) return rc;
    return p->N2 == 256 ? fs2_cols<256, INV>(a, batch, p->N1, st, false)
                        : fs2_cols<128, INV>(a, batch, p->N1, st, false);
}

static int fs2_dispatch(const BluesteinPlan* p, const DftArgs& a, int64_t batch, bool inverse,
                        cudaStream_t st) {
    return inverse ? fs2_all<true>(p, a, batch, st) : fs2_all<false>(p, a, batch, st);
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int64_t sfftb_dft_workspace_bytes(int64_t batch, int64_t M) {
    if (batch <= 0 || M <= 0) return 0;
    const int64_t N = bluestein_N(M);
    if (N <= (int64_t(1) << kSmallMaxLog)) return 0;
    return batch * N * (int64_t)sizeof(double2);
}

extern "C" int sfftb_dft(const double* x, int64_t x_stride, double* y, int64_t y_stride,
                         int64_t batch, int64_t M, int inverse, double scale, void* ws,
                         void* stream) {
    SFFTB_REQUIRE(batch >= 0 && M >= 1, "dft: bad sizes");
    if (batch == 0) return SFFTB_OK;
    SFFTB_REQUIRE(batch <= 65535 || bluestein_N(M) <= (int64_t(1) << kSmallMaxLog),
                  "dft: batch too large for one launch");
    BluesteinPlan* p = nullptr;
    int rc = get_plan(M, &p);
    if (rc != SFFTB_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    DftArgs a;
    a.x = (const double2*)x;
    a.xs = x_stride;
    a.y = (double2*)y;
    a.ys = y_stride;
    a.M = M;
    a.scale = scale;
    a.chirp = p->chirp;
    a.bhat = p->bhat;
    a.tw_hi = p->tw_hi;
    a.tw_lo = p->tw_lo;
    a.tw_n1 = p->tw_n1;
    a.tw_n2 = p->tw_n2;
    a.work = (double2*)ws;
    a.hi_in_smem = p->N / 64 <= 2048;  // <= 32 KB of shared memory
    if (p->P9)
        return inverse ? small9_dispatch<true>(p->P9, a, batch, st)
                       : small9_dispatch<false>(p->P9, a, batch, st);
    if (p->N <= (1 << kSmallMaxLog))
        return inverse ? small_dispatch<true>(p->logN, a, batch, st)
                       : small_dispatch<false>(p->logN, a, batch, st);
    SFFTB_REQUIRE(ws != nullptr, "dft: workspace required");
    if (fs2_supported(p)) return fs2_dispatch(p, a, batch, inverse != 0, st);
    // Run the three passes over L2-sized slices of the batch so the
    // four-step intermediate (16*N bytes per transform) is re-read from L2,
    // not HBM: <= 48 MiB of workspace live per slice (L2 is ~126 MB).
    const int64_t per = (int64_t)p->N * (int64_t)sizeof(double2);
    // (measured: slicing to 48 MiB made the launches too small and was
    // slower than one launch over the batch, so the slice is the batch)
    const int64_t chunk = std::max<int64_t>(batch, ((int64_t)48 << 20) / per);
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int64_t nb = std::min<int64_t>(chunk, batch - b0);
        DftArgs c = a;
        c.x = a.x + b0 * a.xs;
        c.y = a.y + b0 * a.ys;
        rc = inverse ? cols_dispatch<true>(p->N2, c, nb, p->N1, st, true)
                     : cols_dispatch<false>(p->N2, c, nb, p->N1, st, true);
        if (rc != SFFTB_OK) return rc;
        rc = rows_dispatch(p->N1, c, nb, p->N2, st);
        if (rc != SFFTB_OK) return rc;
        rc = inverse ? cols_dispatch<true>(p->N2, c, nb, p->N1, st, false)
                     : cols_dispatch<false>(p->N2, c, nb, p->N1, st, false);
        if (rc != SFFTB_OK) return rc;
    }
    return SFFTB_OK;
}

extern "C" int64_t sfftb_sample_detect_workspace_bytes(int64_t batch, int64_t M) {
    if (batch <= 0 || M <= 0) return 0;
    const int64_t N = bluestein_N(M);
    if (N <= (int64_t(1) << kSmallMaxLog)) return 0;
    return batch * N * (int64_t)sizeof(double2) + batch * 64 * (int64_t)sizeof(double) +
           batch * (int64_t)sizeof(double);
}

static int sample_detect(const double* bins, const uint32_t* lr, const double* lv, int64_t ls,
                         int64_t G, int64_t L, int64_t M, uint64_t seed, int64_t call0,
                         double sigma, double* ghat, double* theta, uint32_t* bits, void* ws,
                         void* stream) {
    SFFTB_REQUIRE(G >= 1 && L >= 1 && M >= 1, "sample_detect: bad sizes");
    BluesteinPlan* p = nullptr;
    int rc = get_plan(M, &p);
    if (rc != SFFTB_OK) return rc;
    if (!fs2_supported(p)) {
        set_error("sample_detect: fused path needs N1 in {128, 192, 256}, N2 in {128, 256}");
        return SFFTB_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t batch = G * L;
    SFFTB_REQUIRE(batch <= 65535, "sample_detect: batch too large");
    const int64_t N = p->N;
    DftArgs a;
    a.x = (const double2*)bins;
    a.xs = M;
    a.y = (double2*)ghat;
    a.ys = M;
    a.M = M;
    a.chirp = p->chirp;
    a.bhat = p->bhat;
    a.tw_hi = p->tw_hi;
    a.tw_lo = p->tw_lo;
    a.tw_n1 = p->tw_n1;
    a.tw_n2 = p->tw_n2;
    a.work = (double2*)ws;
    a.hi_in_smem = p->N / 64 <= 2048;
    a.sumsq_part = (double*)((char*)ws + batch * N * sizeof(double2));
    double* sumsq = a.sumsq_part + batch * 64;
    a.noise_seed = seed;
    a.noise_call0 = call0;
    a.noise_sigma = sigma;
    a.theta = theta;
    a.L = (int)L;
    a.bits = bits;
    a.W = sfftb_bitmap_words(M);
    a.lr = lr;
    a.lv = (const double2*)lv;
    a.ls = ls;
    {
        const char* e = getenv("SFFTB_PDL");
        a.pdl = (!e || atoi(e) != 0) && p->N1 == 192 && p->N2 == 256;
    }
    SFFTB_CUDA(cudaMemsetAsync(bits, 0, sizeof(uint32_t) * batch * a.W, st));
    // sampler: inverse DFT (scale 1) -- colA (conj input) and rowB
    a.scale = 1.0;
    if (lr)
        rc = p->N2 == 256 ? fs2_cols<256, true, true>(a, batch, p->N1, st, true)
                          : fs2_cols<128, true, true>(a, batch, p->N1, st, true);
    else
        rc = p->N2 == 256 ? fs2_cols<256, true>(a, batch, p->N1, st, true)
                          : fs2_cols<128, true>(a, batch, p->N1, st, true);
    if (rc) return rc;
    rc = fs2_rows_any(a, batch, p->N1, p->N2, st);
    if (rc) return rc;
    // fused colC(sampler) + colA(detection)
    {
        const int F = p->N2 == 256 ? Fs2Layout<256>::F : Fs2Layout<128>::F;
        DftArgs c = a;
        c.ntiles = (int64_t)(p->N1 / F) * batch;
        const int grid = fs_grid(c.ntiles);
        const size_t hi = a.hi_in_smem ? (size_t)(N / 64) : 0;
        auto launch_ca = [&](auto kern, size_t sm) -> int {
            SFFTB_CUDA(allow_smem(kern, sm));
            SFFTB_CUDA(launch_maybe_pdl(c.pdl, kern, dim3(grid), dim3(256), sm, st, c, (int)p->N1));
            return SFFTB_OK;
        };
        const size_t sm256 = sizeof(double2) * (Fs2Layout<256>::DATA + 256 + 64 + hi);
        const size_t sm128 = sizeof(double2) * (Fs2Layout<128>::DATA + 128 + 64 + hi);
        int rcl = SFFTB_OK;
        if (p->N2 == 256 && p->N1 == 192)
            rcl = sigma > 0.0 ? launch_ca(fs2_colCA<256, true, 192>, sm256)
                              : launch_ca(fs2_colCA<256, false, 192>, sm256);
        else if (p->N2 == 256)
            rcl = sigma > 0.0 ? launch_ca(fs2_colCA<256, true>, sm256)
                              : launch_ca(fs2_colCA<256, false>, sm256);
        else if (p->N1 == 192)
            rcl = sigma > 0.0 ? launch_ca(fs2_colCA<128, true, 192>, sm128)
                              : launch_ca(fs2_colCA<128, false, 192>, sm128);
        else
            rcl = sigma > 0.0 ? launch_ca(fs2_colCA<128, true>, sm128)
                              : launch_ca(fs2_colCA<128, false>, sm128);
        if (rcl) return rcl;
        SFFTB_CHECK_LAUNCH();
        const int per_b = p->N1 / F;
        SFFTB_CUDA(launch_maybe_pdl(a.pdl, partial_sumsq_reduce, dim3((unsigned)ceil_div(batch, 128)),
                                    dim3(128), 0, st, (const double*)a.sumsq_part, batch, per_b,
                                    sumsq));
        SFFTB_CHECK_LAUNCH();
    }
    rc = zero_thresholds_launch(sumsq, G, L, M, theta, st, a.pdl != 0);
    if (rc) return rc;
    // detection: rowB, then colC emitting ghat (scale 1/M) and the bitmap
    // (bits zeroed at the start of the chain, so the two kernels are adjacent)
    rc = fs2_rows_any(a, batch, p->N1, p->N2, st);
    if (rc) return rc;
    {
        DftArgs c = a;
        c.scale = 1.0 / (double)M;
        const int F = p->N2 == 256 ? Fs2Layout<256>::F : Fs2Layout<128>::F;
        c.ntiles = (int64_t)(p->N1 / F) * batch;
        const int grid = fs_grid(c.ntiles);
        if (p->N2 == 256) {
            const size_t sm = sizeof(double2) * (Fs2Layout<256>::DATA + 256);
            if (p->N1 == 192) {
                SFFTB_CUDA(allow_smem(fs2_colC_bits<256, 192>, sm));
                SFFTB_CUDA(launch_maybe_pdl(c.pdl, fs2_colC_bits<256, 192>, dim3(grid), dim3(256),
                                            sm, st, c, (int)p->N1));
            } else {
                SFFTB_CUDA(allow_smem(fs2_colC_bits<256>, sm));
                fs2_colC_bits<256><<<grid, 256, sm, st>>>(c, p->N1);
            }
        } else {
            const size_t sm = sizeof(double2) * (Fs2Layout<128>::DATA + 128);
            SFFTB_CUDA(allow_smem(fs2_colC_bits<128>, sm));
            fs2_colC_bits<128><<<grid, 256, sm, st>>>(c, p->N1);
        }
        SFFTB_CHECK_LAUNCH();
    }
    return SFFTB_OK;
}

extern "C" int sfftb_sample_detect_dft(const double* bins, int64_t G, int64_t L, int64_t M,
                                       uint64_t seed, int64_t call0, double sigma,
                                       double* ghat, double* theta, uint32_t* bits,
                                       void* ws, void* stream) {
    return sample_detect(bins, nullptr, nullptr, 0, G, L, M, seed, call0, sigma, ghat, theta,
                         bits, ws, stream);
}

extern "C" int sfftb_sample_detect_dft_list(const uint32_t* list_r, const double* list_v,
                                            int64_t ls, int64_t G, int64_t L, int64_t M,
                                            uint64_t seed, int64_t call0, double sigma,
                                            double* ghat, double* theta, uint32_t* bits,
                                            void* ws, void* stream) {
    SFFTB_REQUIRE(list_r && list_v && ls >= 1, "sample_detect_list: empty list");
    return sample_detect(nullptr, list_r, list_v, ls, G, L, M, seed, call0, sigma, ghat, theta,
                         bits, ws, stream);
}

namespace sfftb {
// The Bluestein chirp of length M (plan cache), for producers that fold the
// sampler's chirp product into their output (sfftb_scatter_list).
int bluestein_chirp(int64_t M, const double2** chirp) {
    BluesteinPlan* p = nullptr;
    const int rc = get_plan(M, &p);
    if (rc != SFFTB_OK) return rc;
    *chirp = p->chirp;
    return SFFTB_OK;
}
}  // namespace sfftb

extern "C" int sfftb_plan_cache_clear(void) {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    for (auto& kv : g_plans) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first.first);
        cudaFree(kv.second->chirp);
        cudaFree(kv.second->bhat);
        cudaFree(kv.second->tw_hi);
        cudaFree(kv.second->tw_lo);
        cudaFree(kv.second->tw_n1);
        cudaFree(kv.second->tw_n2);
        cudaSetDevice(cur);
        delete kv.second;
    }
    g_plans.clear();
    return SFFTB_OK;
}
