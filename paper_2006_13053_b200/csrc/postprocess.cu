// K9: rank-1-lattice coefficient refinement (postprocess_r1l, reference
// latfft/detect.py:198-228).
//
// For the n detected rows and each of the L lattices: the residue of every
// row, a per-lattice histogram of those residues (np.bincount), and for each
// row the lattices on which its residue is unique among the detected rows.
// The refined value is the mean of the per-lattice estimates over those
// lattices, accumulated in lattice order like the reference's
// `unique_sum[is_unique] += vals[is_unique, col]`, then divided the way numpy
// divides complex128 by an integer count (c -> c + 0j, Smith's branch:
// re * (1/c), im * (1/c)); rows without such a lattice keep their median.
// keep bit = |refined| > theta0 (np.abs of complex128 = hypot).
#include "common.cuh"

namespace sfftb {

__device__ __forceinline__ int64_t residue_rows(const int64_t* row, const int64_t* z, int d,
                                                int64_t M) {
    uint64_t acc = 0;  // d (M-1)^2 < 2^62: the caller's bound (detect.py:128-129)
    for (int j = 0; j < d; ++j)
        acc += (uint64_t)reduce_mod(row[j], M) * (uint64_t)reduce_mod(z[j], M);
    return (int64_t)mod_u64(acc, (uint64_t)M, 1.0 / (double)M);
}

// e = l * n + i: residues and histogram, lattice-major (coalesced per lattice)
__global__ void r1l_hist_kernel(const int64_t* __restrict__ rows, int64_t n, int d,
                                const int64_t* __restrict__ zmat,
                                const int64_t* __restrict__ offs, int L,
                                int32_t* __restrict__ res, int32_t* __restrict__ cnt) {
    const int64_t total = n * L;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(e / n);
        const int64_t i = e % n;
        const int64_t M = offs[l + 1] - offs[l];
        const int64_t r = residue_rows(rows + i * d, zmat + (int64_t)l * d, d, M);
        res[e] = (int32_t)r;
        atomicAdd(cnt + offs[l] + r, 1);
    }
}

__global__ void r1l_refine_kernel(int64_t n, int L, const int64_t* __restrict__ offs,
                                  const int32_t* __restrict__ res,
                                  const int32_t* __restrict__ cnt,
                                  const double2* __restrict__ vals,
                                  const double2* __restrict__ medians, double theta0,
                                  double2* __restrict__ refined, uint32_t* __restrict__ keep) {
    const int64_t nblk = (n + 31) / 32 * 32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nblk;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool k = false;
        if (i < n) {
            double2 acc = make_double2(0.0, 0.0);
            int64_t c = 0;
            for (int l = 0; l < L; ++l) {
                const int64_t e = (int64_t)l * n + i;
                if (cnt[offs[l] + res[e]] == 1) {
                    const double2 v = vals[e];
                    acc.x += v.x;
                    acc.y += v.y;
                    ++c;
                }
            }
            double2 out = medians[i];
            if (c > 0) {
                const double scl = 1.0 / (double)c;
                out = make_double2(acc.x * scl, acc.y * scl);
            }
            refined[i] = out;
            k = hypot(out.x, out.y) > theta0;
        }
        const unsigned b = __ballot_sync(0xffffffffu, k);
        if ((threadIdx.x & 31) == 0 && i < n) keep[i >> 5] = b;
    }
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int64_t sfftb_r1l_workspace_bytes(int64_t n, int64_t L, int64_t Msum) {
    return 4 * (n * L + Msum) + 16;
}

extern "C" int sfftb_postprocess_r1l(const int64_t* rows, int64_t n, int64_t d,
                                     const int64_t* zmat, const int64_t* offs, int64_t L,
                                     int64_t Msum, const double* vals, const double* medians,
                                     double theta0, double* refined, uint32_t* keep, void* ws,
                                     void* stream) {
    SFFTB_REQUIRE(n >= 0 && d >= 1 && L >= 1 && Msum >= L, "postprocess_r1l: bad sizes");
    if (n == 0) return SFFTB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t* res = (int32_t*)ws;
    int32_t* cnt = res + n * L;
    SFFTB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)Msum, st));
    const int64_t total = n * L;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 16);
    r1l_hist_kernel<<<grid, 256, 0, st>>>(rows, n, (int)d, zmat, offs, (int)L, res, cnt);
    SFFTB_CHECK_LAUNCH();
    const int grid2 = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 8);
    r1l_refine_kernel<<<grid2, 256, 0, st>>>(n, (int)L, offs, res, cnt, (const double2*)vals,
                                             (const double2*)medians, theta0,
                                             (double2*)refined, keep);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
