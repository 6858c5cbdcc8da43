// The drop-in plugin API of latfft._kernels (host buffers in and out) and the
// library's error/version plumbing.
//
//   sfftb_detect_gather       <- _kernels/__init__.py:54-70, _core.pyx:164-202
//   sfftb_rows_injective_mod  <- _kernels/__init__.py:45-51, _core.pyx:103-144
//   sfftb_hc_count/enumerate  <- _kernels/__init__.py:29-42, _core.pyx:24-96
//
// detect_gather runs the same device pipeline as the drivers: upload, bitmap
// of |ghat| > theta, hashing with hit counts, compaction of the detected
// rows, medians, download.  Everything is stream-ordered on the calling
// thread's per-thread default stream, so calls are reentrant like the
// reference's nogil kernels.
#include <math.h>

#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "common.cuh"

namespace sfftb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::mutex g_attr_mu;
static std::map<std::pair<int, const void*>, size_t> g_smem_set;
static std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;

cudaError_t smem_opt_in_raw(const void* kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto key = std::make_pair(dev, kernel);
    auto it = g_smem_set.find(key);
    if (it != g_smem_set.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e =
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) g_smem_set[key] = bytes;
    return e;
}

cudaError_t occupancy_raw(int* out, const void* kernel, int threads, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto key = std::make_tuple(dev, kernel, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, threads, smem);
    if (e == cudaSuccess) g_occ[key] = *out;
    return e;
}

__global__ void scatter_medians_kernel(const int64_t* __restrict__ idx,
                                       const int64_t* __restrict__ count,
                                       const double2* __restrict__ vals,
                                       double2* __restrict__ full) {
    const int64_t c = count[0];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < c;
         k += (int64_t)gridDim.x * blockDim.x)
        full[idx[k]] = vals[k];
}

// RAII bundle of stream-ordered device allocations
struct DevBufs {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit DevBufs(cudaStream_t s) : st(s) {}
    cudaError_t alloc(void** p, size_t bytes) {
        cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~DevBufs() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
    }
};

// ---- hyperbolic cross (host recursion; same floating-point steps as
// _core.pyx:24-96 so the enumerated sets agree exactly) ----
static inline double hc_factor(double w, double k) {
    double f = w * fabs(k);
    return f > 1.0 ? f : 1.0;
}
static inline int64_t hc_cap(double bound, double prod, double w) {
    int64_t k = (int64_t)floor((bound / prod) / w);
    if (k < 0) k = 0;
    while (k > 0 && prod * hc_factor(w, (double)k) > bound) --k;
    while (prod * hc_factor(w, (double)(k + 1)) <= bound) ++k;
    return k;
}
static int64_t hc_walk(int t, int d, double prod, double bound, const double* w, int64_t* buf,
                       int64_t* out, int64_t pos, int64_t capacity, bool count_only) {
    const int64_t cap = hc_cap(bound, prod, w[t]);
    if (t == d - 1 && count_only) return pos + 2 * cap + 1;
    for (int64_t k = -cap; k <= cap; ++k) {
        buf[t] = k;
        if (t == d - 1) {
            if (pos < capacity)
                for (int j = 0; j < d; ++j) out[pos * d + j] = buf[j];
            ++pos;
        } else {
            pos = hc_walk(t + 1, d, prod * hc_factor(w[t], (double)k), bound, w, buf, out, pos,
                          capacity, count_only);
        }
    }
    return pos;
}

}  // namespace sfftb

using namespace sfftb;

extern "C" const char* sfftb_version(void) { return "sfftb200 0.1.0 (sm_100a)"; }
extern "C" const char* sfftb_last_error(void) { return g_err.c_str(); }
extern "C" int64_t sfftb_launch_count(void) { return g_launches.load(); }

extern "C" int sfftb_hc_count(int d, double bound, const double* weights, int64_t* count) {
    SFFTB_REQUIRE(d >= 1 && d <= 64, "hc_count: 1 <= d <= 64");
    std::vector<int64_t> buf(d);
    *count = hc_walk(0, d, 1.0, bound, weights, buf.data(), nullptr, 0, 0, true);
    return SFFTB_OK;
}

extern "C" int sfftb_hc_enumerate(int d, double bound, const double* weights, int64_t* out,
                                  int64_t capacity) {
    SFFTB_REQUIRE(d >= 1 && d <= 64, "hc_enumerate: 1 <= d <= 64");
    std::vector<int64_t> buf(d);
    const int64_t n = hc_walk(0, d, 1.0, bound, weights, buf.data(), out, 0, capacity, false);
    SFFTB_REQUIRE(n <= capacity, "hc_enumerate: output capacity too small");
    return SFFTB_OK;
}

extern "C" int sfftb_rows_injective_mod(const int64_t* elems, int64_t n, int64_t d, int64_t p,
                                        int* injective) {
    SFFTB_REQUIRE(p >= 1, "rows_injective_mod: p must be >= 1");
    if (n <= 1) {
        *injective = 1;
        return SFFTB_OK;
    }
    cudaStream_t st = cudaStreamPerThread;
    DevBufs bufs(st);
    void* de = nullptr;
    SFFTB_CUDA(bufs.alloc(&de, sizeof(int64_t) * n * d));
    SFFTB_CUDA(cudaMemcpyAsync(de, elems, sizeof(int64_t) * n * d, cudaMemcpyHostToDevice, st));
    return sfftb_injective_mod_dev((const int64_t*)de, n, d, p, injective, st);
}

// Largest lattice count the reference's compiled gather serves
// (_kernels/__init__.py:26 _MAX_COMPILED_L); beyond it the numpy path applies.
static constexpr int64_t kMaxCompiledL = 128;

extern "C" int sfftb_detect_gather(const int64_t* elems, int64_t n, int64_t d,
                                   const int64_t* zmat, int64_t L, int64_t M, const double* ghat,
                                   double theta, double hit_threshold, int want_medians,
                                   int64_t* hits, double* medians) {
    SFFTB_REQUIRE(n >= 0 && d >= 0 && L >= 0 && M >= 1, "detect_gather: bad sizes");
    if (want_medians && (L % 2) == 0) {
        set_error("medians require an odd lattice count");
        return SFFTB_EINVAL;
    }
    if (n == 0) return SFFTB_OK;
    cudaStream_t st = cudaStreamPerThread;
    // detected iff (double)hits >= hit_threshold  <=>  hits >= ceil(thr)
    int64_t min_hits;
    if (std::isnan(hit_threshold) || hit_threshold > (double)L)
        min_hits = L + 1;
    else if (hit_threshold <= 0.0)
        min_hits = 0;
    else
        min_hits = (int64_t)ceil(hit_threshold);

    const int64_t W = sfftb_bitmap_words(M);
    const int64_t nwords = (n + 31) / 32;
    DevBufs b(st);
    void *de, *dz, *dg, *dbits, *dth, *dhits, *dmask, *dbnd;
    SFFTB_CUDA(b.alloc(&de, sizeof(int64_t) * n * std::max<int64_t>(d, 1)));
    SFFTB_CUDA(b.alloc(&dz, sizeof(int64_t) * std::max<int64_t>(L * d, 1)));
    SFFTB_CUDA(b.alloc(&dg, sizeof(double2) * std::max<int64_t>(L * M, 1)));
    SFFTB_CUDA(b.alloc(&dbits, sizeof(uint32_t) * std::max<int64_t>(L * W, 4)));
    SFFTB_CUDA(b.alloc(&dth, sizeof(double)));
    SFFTB_CUDA(b.alloc(&dhits, sizeof(int64_t) * n));
    SFFTB_CUDA(b.alloc(&dmask, sizeof(uint32_t) * nwords));
    SFFTB_CUDA(b.alloc(&dbnd, sizeof(int64_t) * 2 * std::max<int64_t>(d, 1)));
    if (d > 0)
        SFFTB_CUDA(cudaMemcpyAsync(de, elems, sizeof(int64_t) * n * d, cudaMemcpyHostToDevice,
                                   st));
    if (L * d > 0)
        SFFTB_CUDA(cudaMemcpyAsync(dz, zmat, sizeof(int64_t) * L * d, cudaMemcpyHostToDevice,
                                   st));
    if (L > 0)
        SFFTB_CUDA(cudaMemcpyAsync(dg, ghat, sizeof(double2) * L * M, cudaMemcpyHostToDevice,
                                   st));
    SFFTB_CUDA(cudaMemcpyAsync(dth, &theta, sizeof(double), cudaMemcpyHostToDevice, st));
    int rc;
    if (L > kMaxCompiledL) {
        // the reference's numpy path for L > _MAX_COMPILED_L (_kernels/__init__.py:62,
        // fallback.py:106-131): per row the L values ghat[l, r_l], hits by
        // np.abs (hypot) > theta, np.median of real and imaginary parts; rows
        // in chunks of <= 256 MB of values
        const int64_t chunk = std::max<int64_t>(1, ((int64_t)256 << 20) / (16 * L));
        void *dv, *dm;
        SFFTB_CUDA(b.alloc(&dv, sizeof(double2) * std::min(n, chunk) * L));
        SFFTB_CUDA(b.alloc(&dm, sizeof(double2) * n));
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            const int64_t cn = std::min(chunk, n - c0);
            rc = sfftb_lattice_values((const int64_t*)de + c0 * d, d, (const int64_t*)dz, L, M,
                                      (const double*)dg, nullptr, cn, (double*)dv, st);
            if (rc) return rc;
            rc = sfftb_rows_hits_medians((const double*)dv, cn, L, theta, hit_threshold,
                                         want_medians, (int64_t*)dhits + c0,
                                         (double*)((double2*)dm + c0), st);
            if (rc) return rc;
        }
        SFFTB_CUDA(cudaMemcpyAsync(hits, dhits, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
        if (want_medians)
            SFFTB_CUDA(cudaMemcpyAsync(medians, dm, sizeof(double2) * n, cudaMemcpyDeviceToHost,
                                       st));
        else
            memset(medians, 0, sizeof(double) * 2 * n);
        SFFTB_CUDA(cudaStreamSynchronize(st));
        return SFFTB_OK;
    }
    if (L > 0) {
        rc = sfftb_nonzero_bitmap((const double*)dg, 1, L, M, (const double*)dth,
                                  (uint32_t*)dbits, st);
        if (rc) return rc;
    }
    // exact magnitude bound of the rows enables the 32-bit residue path
    int64_t kbound = -1;
    if (d >= 1 && d <= 256) {
        rc = sfftb_row_bounds((const int64_t*)de, n, d, (int64_t*)dbnd, st);
        if (rc) return rc;
        std::vector<int64_t> bnd(2 * d);
        SFFTB_CUDA(cudaMemcpyAsync(bnd.data(), dbnd, sizeof(int64_t) * 2 * d,
                                   cudaMemcpyDeviceToHost, st));
        SFFTB_CUDA(cudaStreamSynchronize(st));
        __int128 kb = 0;
        for (int64_t j = 0; j < d; ++j) {
            const __int128 lo = bnd[2 * j], hi = bnd[2 * j + 1];
            kb += std::max(lo < 0 ? -lo : lo, hi < 0 ? -hi : hi);
        }
        if (kb < ((__int128)1 << 62)) kbound = (int64_t)kb;
    }
    if (L == 0) {
        SFFTB_CUDA(cudaMemsetAsync(dhits, 0, sizeof(int64_t) * n, st));
        SFFTB_CUDA(cudaMemsetAsync(dmask, min_hits <= 0 ? 0xff : 0, sizeof(uint32_t) * nwords, st));
    } else {
        rc = sfftb_hash_hits((const int64_t*)de, n, d, (const int64_t*)dz, 1, L, M,
                             (const uint32_t*)dbits, kbound, min_hits, (int64_t*)dhits,
                             (uint32_t*)dmask, st);
        if (rc) return rc;
    }
    SFFTB_CUDA(cudaMemcpyAsync(hits, dhits, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
    if (want_medians) {
        void *didx, *dcnt, *dws, *dvals, *dfull;
        SFFTB_CUDA(b.alloc(&didx, sizeof(int64_t) * n));
        SFFTB_CUDA(b.alloc(&dcnt, sizeof(int64_t)));
        SFFTB_CUDA(b.alloc(&dws, (size_t)sfftb_compact_workspace_bytes(1, n)));
        SFFTB_CUDA(b.alloc(&dvals, sizeof(double2) * n));
        SFFTB_CUDA(b.alloc(&dfull, sizeof(double2) * n));
        rc = sfftb_compact_mask((const uint32_t*)dmask, 1, n, (int64_t*)didx, (int64_t*)dcnt, dws,
                                st);
        if (rc) return rc;
        rc = sfftb_medians((const int64_t*)de, d, (const int64_t*)dz, 1, L, M,
                           (const double*)dg, (const int64_t*)didx, (const int64_t*)dcnt, n,
                           (double*)dvals, st);
        if (rc) return rc;
        SFFTB_CUDA(cudaMemsetAsync(dfull, 0, sizeof(double2) * n, st));
        scatter_medians_kernel<<<num_sms() * 4, 256, 0, st>>>(
            (const int64_t*)didx, (const int64_t*)dcnt, (const double2*)dvals, (double2*)dfull);
        SFFTB_CHECK_LAUNCH();
        SFFTB_CUDA(cudaMemcpyAsync(medians, dfull, sizeof(double2) * n, cudaMemcpyDeviceToHost,
                                   st));
    } else {
        memset(medians, 0, sizeof(double) * 2 * n);
    }
    SFFTB_CUDA(cudaStreamSynchronize(st));
    return SFFTB_OK;
}
