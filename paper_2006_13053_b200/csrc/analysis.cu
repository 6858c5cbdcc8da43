// K12: worst-case alias accounting of the experiment harness
// (reference latfft/analysis.py:67-104 pfp_pfn_count, :218-250 _trial), and
// K13: the tensor-product B-spline test function f10 (polyeval.py:216-272)
// evaluated on device, so black-box sfft runs on it sample on the GPU.
//
// K12 runs after detection of G independent trials that share one candidate
// set (the "lattices" redraw protocol batches every trial of one L into one
// launch chain):
//   rows_in_sorted   in_I[i] = Gamma row i is a member of the support I
//                    (FreqSet.contains_rows, binary search in the sorted rows)
//   alias_classify   per detected (group, row, median): integral / rounded /
//                    class code, and per-group tallies of the five counts the
//                    reference's masks sum (analysis.py:88-101).
#include "common.cuh"

namespace sfftb {

// -1 / 0 / 1: lexicographic order of two d-vectors
__device__ __forceinline__ int lex_cmp(const int64_t* a, const int64_t* b, int d) {
    for (int j = 0; j < d; ++j) {
        const int64_t x = a[j], y = b[j];
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

__global__ void rows_in_sorted_kernel(const int64_t* __restrict__ rows, int64_t n, int d,
                                      const int64_t* __restrict__ pool, int64_t m,
                                      uint32_t* __restrict__ mask) {
    const int64_t nblk = (n + 31) / 32 * 32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nblk;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool hit = false;
        if (i < n) {
            const int64_t* r = rows + i * d;
            int64_t lo = 0, hi = m;  // first pool row >= r
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (lex_cmp(pool + mid * d, r, d) < 0) lo = mid + 1;
                else hi = mid;
            }
            hit = lo < m && lex_cmp(pool + lo * d, r, d) == 0;
        }
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if ((threadIdx.x & 31) == 0 && i < n) mask[i >> 5] = b;
    }
}

// Tallies per group: [0] detected & in_I, [1] detected & ~integral,
// [2] detected & integral & rounded < 1, [3] pfn (in_I & integral &
// rounded >= 2), [4] pfp (~in_I & integral & rounded >= 1).
// Class code per entry: bit 0 = in_I, bits 1..3 = 0 clean (in_I, rounded
// == 1), 1 non-integral, 2 rounded < 1, 3 pfn, 4 pfp.
constexpr int kTallies = 5;

__global__ void alias_classify_kernel(const int64_t* __restrict__ idx,
                                      const double2* __restrict__ med,
                                      const int64_t* __restrict__ counts, int64_t cap,
                                      const uint32_t* __restrict__ in_mask, double tol,
                                      uint8_t* __restrict__ cls,
                                      unsigned long long* __restrict__ tallies) {
    const int g = blockIdx.y;
    const int64_t cnt = counts[g];
    unsigned t[kTallies] = {0, 0, 0, 0, 0};
    const int64_t span = (cnt + 31) / 32 * 32;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < span;
         j += (int64_t)gridDim.x * blockDim.x) {
        if (j < cnt) {
            const int64_t e = (int64_t)g * cap + j;
            const int64_t row = idx[e];
            const bool in_i = (in_mask[row >> 5] >> (row & 31)) & 1u;
            const double2 v = med[e];
            // np.rint (half to even) and the reference's integrality test
            const double rounded = rint(v.x);
            const bool integral = fabs(v.x - rounded) <= tol && fabs(v.y) <= tol;
            int code;
            if (!integral) code = 1;
            else if (rounded < 1.0) code = 2;
            else if (in_i) code = rounded >= 2.0 ? 3 : 0;
            else code = 4;
            t[0] += in_i;
            t[1] += code == 1;
            t[2] += code == 2;
            t[3] += code == 3;
            t[4] += code == 4;
            if (cls) cls[e] = (uint8_t)((code << 1) | (in_i ? 1 : 0));
        }
    }
#pragma unroll
    for (int k = 0; k < kTallies; ++k) {
        const unsigned s = __reduce_add_sync(0xffffffffu, t[k]);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(tallies + (int64_t)g * kTallies + k, s);
    }
}

// ---------------------------------------------------------------------------
// K13: sum over groups of products of periodised B-splines (f10_values)
// ---------------------------------------------------------------------------

constexpr int kMaxSplineDim = 32;
constexpr int kMaxSplineGroups = 8;

struct SplineSum {
    int d, ngroups;
    int axis_group[kMaxSplineDim];  // -1: axis unused
    int order[kMaxSplineGroups];
    double scale[kMaxSplineGroups];  // C_m * m (bspline_values' prefactor)
};

// Centered cardinal B-spline of order m at t (polyeval.py:206-213):
// sum_j (-1)^j C(m, j) max(0, t + m/2 - j)^(m-1) / (m-1)!
__device__ __forceinline__ double cardinal_bspline(int m, double t) {
    double acc = 0.0;
    double binom = 1.0;  // C(m, j), exact in binary
    double fact = 1.0;   // (m-1)!
    for (int k = 2; k < m; ++k) fact *= (double)k;
    for (int j = 0; j <= m; ++j) {
        const double u = t + 0.5 * (double)m - (double)j;
        double p = 0.0;
        if (u > 0.0) {
            p = 1.0;
            for (int e = 0; e < m - 1; ++e) p *= u;
        }
        acc += ((j & 1) ? -binom : binom) * p;
        binom = binom * (double)(m - j) / (double)(j + 1);
    }
    return acc / fact;
}

// bspline_values(m, x) (polyeval.py:216-225) without its C_m * m prefactor
__device__ __forceinline__ double spline_at(int m, double x) {
    const double u = x - floor(x) - 0.5;
    return cardinal_bspline(m, (double)m * u);
}

__device__ __forceinline__ double spline_sum(const SplineSum& f, const double* x) {
    double prod[kMaxSplineGroups];
    for (int g = 0; g < f.ngroups; ++g) prod[g] = 1.0;
    for (int a = 0; a < f.d; ++a) {
        const int g = f.axis_group[a];
        if (g < 0) continue;
        prod[g] *= f.scale[g] * spline_at(f.order[g], x[a]);
    }
    double total = 0.0;
    for (int g = 0; g < f.ngroups; ++g) total += prod[g];
    return total;
}

// values at lattice nodes [(j z mod M)/M | tail_g] (dimincr.py:186-191),
// out[(gi*L + l)*M + j] as complex128 (imaginary part 0)
__global__ void spline_lattice_kernel(SplineSum f, const int64_t* __restrict__ zmat, int G,
                                      int L, int64_t M, int t_dim,
                                      const double* __restrict__ tails,
                                      double2* __restrict__ out) {
    const int64_t total = (int64_t)G * L * M;
    const int tail_w = max(f.d - t_dim, 1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gl = e / M;
        const int64_t j = e - gl * M;
        const int gi = (int)(gl / L);
        double x[kMaxSplineDim];
        for (int a = 0; a < t_dim; ++a) {
            const int64_t z = reduce_mod(zmat[gl * t_dim + a], M);
            // (j * z) mod M exactly (j, z < M < 2^31), then the float division
            const int64_t r = (int64_t)(((uint64_t)j * (uint64_t)z) % (uint64_t)M);
            x[a] = (double)r / (double)M;
        }
        for (int a = t_dim; a < f.d; ++a) x[a] = tails[(int64_t)gi * tail_w + (a - t_dim)];
        out[e] = make_double2(spline_sum(f, x), 0.0);
    }
}

__global__ void spline_points_kernel(SplineSum f, const double* __restrict__ X, int64_t m,
                                     double2* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x[kMaxSplineDim];
        for (int a = 0; a < f.d; ++a) x[a] = X[i * f.d + a];
        out[i] = make_double2(spline_sum(f, x), 0.0);
    }
}

static int grid_of(int64_t work, int threads) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads),
                                                       (int64_t)num_sms() * 16));
}

static int make_spline(SplineSum& f, int64_t d, const int32_t* axis_group, int64_t ngroups,
                       const int32_t* order, const double* scale) {
    SFFTB_REQUIRE(d >= 1 && d <= kMaxSplineDim, "spline sum: 1 <= d <= 32");
    SFFTB_REQUIRE(ngroups >= 1 && ngroups <= kMaxSplineGroups, "spline sum: 1..8 groups");
    f.d = (int)d;
    f.ngroups = (int)ngroups;
    for (int a = 0; a < d; ++a) {
        SFFTB_REQUIRE(axis_group[a] >= -1 && axis_group[a] < ngroups, "spline sum: bad axis group");
        f.axis_group[a] = axis_group[a];
    }
    for (int g = 0; g < ngroups; ++g) {
        SFFTB_REQUIRE(order[g] >= 1 && order[g] <= 16, "spline sum: order must be 1..16");
        f.order[g] = order[g];
        f.scale[g] = scale[g];
    }
    return SFFTB_OK;
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int sfftb_rows_in_sorted(const int64_t* rows, int64_t n, int64_t d,
                                    const int64_t* pool, int64_t m, uint32_t* mask,
                                    void* stream) {
    SFFTB_REQUIRE(n >= 0 && d >= 1 && m >= 0, "rows_in_sorted: bad sizes");
    if (n == 0) return SFFTB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (m == 0) {
        SFFTB_CUDA(cudaMemsetAsync(mask, 0, sizeof(uint32_t) * (size_t)ceil_div(n, 32), st));
        return SFFTB_OK;
    }
    rows_in_sorted_kernel<<<grid_of((n + 31) / 32 * 32, 256), 256, 0, st>>>(rows, n, (int)d,
                                                                            pool, m, mask);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_alias_classify(const int64_t* idx, const double* med, const int64_t* counts,
                                    int64_t G, int64_t cap, const uint32_t* in_mask, double tol,
                                    uint8_t* cls, int64_t* tallies, void* stream) {
    SFFTB_REQUIRE(G >= 1 && G <= 65535 && cap >= 0, "alias_classify: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    SFFTB_CUDA(cudaMemsetAsync(tallies, 0, sizeof(int64_t) * kTallies * (size_t)G, st));
    if (cap == 0) return SFFTB_OK;
    const int bx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, 256),
                                                               std::max(1, num_sms() * 8 / (int)std::min<int64_t>(G, 1024))));
    alias_classify_kernel<<<dim3((unsigned)bx, (unsigned)G), 256, 0, st>>>(
        idx, (const double2*)med, counts, cap, in_mask, tol, cls,
        (unsigned long long*)tallies);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_spline_sum_lattice(int64_t d, const int32_t* axis_group, int64_t ngroups,
                                        const int32_t* order, const double* scale,
                                        const int64_t* zmat, int64_t G, int64_t L, int64_t M,
                                        int64_t t_dim, const double* tails, double* out,
                                        void* stream) {
    SplineSum f;
    const int rc = make_spline(f, d, axis_group, ngroups, order, scale);
    if (rc != SFFTB_OK) return rc;
    SFFTB_REQUIRE(G >= 1 && L >= 1 && M >= 1 && M < (1ll << 31), "spline lattice: bad sizes");
    SFFTB_REQUIRE(t_dim >= 1 && t_dim <= d, "spline lattice: 1 <= t_dim <= d");
    const int64_t total = G * L * M;
    spline_lattice_kernel<<<grid_of(total, 256), 256, 0, (cudaStream_t)stream>>>(
        f, zmat, (int)G, (int)L, M, (int)t_dim, tails, (double2*)out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_spline_sum_points(int64_t d, const int32_t* axis_group, int64_t ngroups,
                                       const int32_t* order, const double* scale,
                                       const double* X, int64_t m, double* out, void* stream) {
    SplineSum f;
    const int rc = make_spline(f, d, axis_group, ngroups, order, scale);
    if (rc != SFFTB_OK) return rc;
    SFFTB_REQUIRE(m >= 0, "spline points: bad sizes");
    if (m == 0) return SFFTB_OK;
    spline_points_kernel<<<grid_of(m, 256), 256, 0, (cudaStream_t)stream>>>(f, X, m,
                                                                           (double2*)out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
