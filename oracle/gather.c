/*
 * CPU oracle (TEST INFRASTRUCTURE ONLY -- never linked into the product).
 *
 * Plain-C restatement of the reference's native kernels, used by tests/ and
 * bench.py's cpu_baseline leg to check the CUDA path:
 *
 *   oracle_detect_gather      <- latfft/_kernels/_core.pyx:164-202 (semantics of
 *                                fallback.py:106-131; odd-L medians per
 *                                _core.pyx:151-161)
 *   oracle_rows_injective_mod <- _core.pyx:103-144 / fallback.py:78-103 (the
 *                                boolean answer; computed here by sorting the
 *                                reduced rows instead of hashing packed codes,
 *                                so it has no 62-bit packing limit)
 *
 * Build: make -C oracle  (gcc -O2 -ffp-contract=off).  Single-threaded and
 * reentrant; callers parallelise over row chunks (ctypes drops the GIL).  The hit test
 * is sqrt(re*re + im*im) > theta with separately rounded products, exactly as
 * the reference's default x86-64 build evaluates _core.pyx:195.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* middle element of L (odd) doubles by insertion sort, _core.pyx:151-161 */
static double median_odd(const double *src, double *tmp, int64_t L)
{
    for (int64_t i = 0; i < L; ++i) {
        double v = src[i];
        int64_t j = i;
        while (j > 0 && tmp[j - 1] > v) {
            tmp[j] = tmp[j - 1];
            --j;
        }
        tmp[j] = v;
    }
    return tmp[L >> 1];
}

/*
 * elems: (n, d) int64 already reduced mod M (detect.py:132); zmat: (L, d);
 * ghat: (L, M) complex128 as interleaved doubles.  hits: (n,) int64;
 * med: (n,) complex128 interleaved, zero where hits < hit_threshold.
 * Returns 0, or 2 on allocation failure.
 */
int oracle_detect_gather(const int64_t *elems, int64_t n, int64_t d,
                         const int64_t *zmat, int64_t L, int64_t M,
                         const double *ghat, double theta, double hit_threshold,
                         int want_medians, int64_t *hits, double *med)
{
    memset(med, 0, sizeof(double) * 2 * (size_t)n);
    double *re = (double *)malloc(sizeof(double) * 3 * (size_t)(L ? L : 1));
    if (!re)
        return 2;
    double *im = re + L, *tmp = re + 2 * L;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t *row = elems + i * d;
        int64_t cnt = 0;
        for (int64_t l = 0; l < L; ++l) {
            const int64_t *z = zmat + l * d;
            int64_t r = 0;
            for (int64_t j = 0; j < d; ++j)
                r += row[j] * z[j];
            r %= M;
            const double *v = ghat + 2 * (l * M + r);
            re[l] = v[0];
            im[l] = v[1];
            double a = re[l] * re[l];
            double b = im[l] * im[l];
            if (sqrt(a + b) > theta)
                ++cnt;
        }
        hits[i] = cnt;
        if (want_medians && (double)cnt >= hit_threshold) {
            med[2 * i] = median_odd(re, tmp, L);
            med[2 * i + 1] = median_odd(im, tmp, L);
        }
    }
    free(re);
    return 0;
}

static int64_t g_cmp_d;
static int cmp_rows(const void *a, const void *b)
{
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    for (int64_t j = 0; j < g_cmp_d; ++j) {
        if (x[j] < y[j]) return -1;
        if (x[j] > y[j]) return 1;
    }
    return 0;
}

/* 1 when rows reduced componentwise mod p are pairwise distinct, else 0;
 * -1 on allocation failure.  Not thread-safe (qsort comparator state). */
int oracle_rows_injective_mod(const int64_t *elems, int64_t n, int64_t d,
                              int64_t p)
{
    if (n <= 1)
        return 1;
    int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * d));
    if (!buf)
        return -1;
    for (int64_t i = 0; i < n * d; ++i) {
        int64_t r = elems[i] % p;
        buf[i] = r < 0 ? r + p : r;
    }
    g_cmp_d = d;
    qsort(buf, (size_t)n, sizeof(int64_t) * (size_t)d, cmp_rows);
    int ok = 1;
    for (int64_t i = 1; i < n && ok; ++i)
        if (cmp_rows(buf + (i - 1) * d, buf + i * d) == 0)
            ok = 0;
    free(buf);
    return ok;
}
