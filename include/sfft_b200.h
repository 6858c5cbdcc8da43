/*
 * libsfftb200 -- C ABI of the B200-native multiple-rank-1-lattice sparse FFT
 * hot path (arXiv 2006.13053, reference package latfft 0.1.0).
 *
 * Two layers:
 *
 *  1. The drop-in plugin API.  These four functions are exactly what the
 *     reference's kernel dispatch module binds (latfft/_kernels/__init__.py,
 *     reference file:line cited per function).  Host buffers in, host buffers
 *     out; the host<->device copies happen inside.  INTEGRATION.md shows the
 *     ctypes stub a maintainer adds to latfft/_kernels/__init__.py.
 *
 *  2. Device-resident entry points used by the Python drivers
 *     (paper_2006_13053_b200.detect / .dimincr).  Device pointers, sizes and
 *     an explicit cudaStream_t (passed as void*); stream-ordered and
 *     reentrant.  Buffers are owned by the caller; functions that need
 *     scratch take a caller-provided workspace whose size a *_workspace_bytes
 *     query returns.  The only library-owned device state is the Bluestein
 *     plan cache (chirps / filter spectra keyed by device and M, guarded by
 *     a mutex), released by sfftb_plan_cache_clear().
 *
 * Complex numbers are interleaved (re, im) doubles: numpy complex128 layout.
 * Every function returns a status code; sfftb_last_error() describes the
 * last failure on the calling thread.
 */
#ifndef SFFT_B200_H
#define SFFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFFTB_OK 0
#define SFFTB_EINVAL 1 /* -> ParameterError / ValueError */
#define SFFTB_ENOMEM 2 /* -> MemoryError (the reference's _core.pyx:89-90) */
#define SFFTB_ECUDA 3  /* -> RuntimeError */

const char *sfftb_version(void);
const char *sfftb_last_error(void);
/* Number of CUDA kernels the library has launched so far (all threads). */
int64_t sfftb_launch_count(void);
/* Release the cached Bluestein plans of every device. */
int sfftb_plan_cache_clear(void);

/* ------------------------------------------------------------------ */
/* 1. plugin API (host buffers)                                        */
/* ------------------------------------------------------------------ */

/*
 * Per-candidate hit counts and odd-L coefficient medians.
 * Replaces latfft._kernels.detect_gather (_kernels/__init__.py:54-70), i.e.
 * _core.detect_gather (_core.pyx:164-202) / fallback.detect_gather
 * (fallback.py:106-131).  elems (n, d) int64 must already be reduced mod M
 * (the reference's precondition, fallback.py:109-110); zmat (L, d) int64;
 * ghat (L, M) complex128.  hits[i] = #{l : |ghat[l, r_l(i)]| > theta},
 * r_l(i) = elems[i] . zmat[l] mod M; medians[i] = median_l Re + i median_l Im
 * when want_medians and hits[i] >= hit_threshold, else 0.  Medians need odd L
 * (SFFTB_EINVAL otherwise, the reference's ValueError, __init__.py:60-61).
 */
int sfftb_detect_gather(const int64_t *elems, int64_t n, int64_t d,
                        const int64_t *zmat, int64_t L, int64_t M,
                        const double *ghat, double theta, double hit_threshold,
                        int want_medians, int64_t *hits, double *medians);

/*
 * *injective = 1 iff the rows of elems (n, d), reduced componentwise mod p,
 * are pairwise distinct.  Replaces latfft._kernels.rows_injective_mod
 * (_kernels/__init__.py:45-51; _core.pyx:103-144 / fallback.py:78-103) with
 * no 62-bit packing limit (the compiled core's -1 case is handled here).
 */
int sfftb_rows_injective_mod(const int64_t *elems, int64_t n, int64_t d,
                             int64_t p, int *injective);

/*
 * |{k in Z^d : prod_t max(1, w_t |k_t|) <= bound}| and its lexicographic
 * enumeration.  Replaces latfft._kernels.hc_count / hc_enumerate
 * (_kernels/__init__.py:29-42; _core.pyx:24-96).  Host C++ (the recursion
 * is not data-parallel work).  hc_enumerate writes count*d int64 into out,
 * which must hold `capacity` rows.
 */
int sfftb_hc_count(int d, double bound, const double *weights, int64_t *count);
int sfftb_hc_enumerate(int d, double bound, const double *weights, int64_t *out,
                       int64_t capacity);

/* ------------------------------------------------------------------ */
/* 2. device-resident entry points                                     */
/* ------------------------------------------------------------------ */

/*
 * Batched prime-length (any length) DFT by Bluestein chirp-z onto
 * power-of-two FFTs in FP64 complex.  Row b of x (stride x_stride complex
 * elements) maps to row b of y:
 *   y[h] = scale * sum_j x[j] exp(-+2 pi i j h / M)   (sign - forward, + inverse)
 * dft_forward_normalized (dft.py:18-27) is inverse=0, scale=1/M; the
 * lattice sampler's M*ifft (polyeval.py:87) is inverse=1, scale=1.
 * ws: sfftb_dft_workspace_bytes(batch, M) bytes of device memory.
 */
int64_t sfftb_dft_workspace_bytes(int64_t batch, int64_t M);
int sfftb_dft(const double *x, int64_t x_stride, double *y, int64_t y_stride,
              int64_t batch, int64_t M, int inverse, double scale, void *ws,
              void *stream);

/*
 * Fused sampler -> detection transforms for G groups of L lattices (the
 * dimension-incremental stage): samples = M*ifft(bins) (+ harness noise for
 * oracle call call0 + row, sigma > 0), theta[g] = default zero test of the
 * group's samples, ghat = fft(samples)/M, bits = |ghat| > theta[g].  The
 * samples themselves stay on chip.  Only for Bluestein sizes whose four-step
 * factors are 128/256 (M in [8192, 32768]); SFFTB_EINVAL otherwise (use the
 * unfused sfftb_dft / sfftb_sumsq / sfftb_zero_thresholds / bitmap chain).
 * ws: sfftb_sample_detect_workspace_bytes(G*L, M).
 */
int64_t sfftb_sample_detect_workspace_bytes(int64_t batch, int64_t M);
int sfftb_sample_detect_dft(const double *bins, int64_t G, int64_t L, int64_t M,
                            uint64_t seed, int64_t call0, double sigma, double *ghat,
                            double *theta, uint32_t *bits, void *ws, void *stream);

/*
 * The same with the sampler's bins given sparsely (sfftb_scatter_list): per
 * transform b, ls entries list_r[b*ls + k] (residue, ~0 = none) and list_v
 * (complex128 bin value).  The first column pass drops the listed bins into
 * its shared-memory tile instead of reading a dense (G*L x M) bins array.
 */
int sfftb_sample_detect_dft_list(const uint32_t *list_r, const double *list_v,
                                 int64_t ls, int64_t G, int64_t L, int64_t M,
                                 uint64_t seed, int64_t call0, double sigma,
                                 double *ghat, double *theta, uint32_t *bits,
                                 void *ws, void *stream);

/* out[b] = sum_j |x[b, j]|^2 (for default_zero_test, detect.py:42-53). */
int sfftb_sumsq(const double *x, int64_t stride, int64_t batch, int64_t M,
                double *out, void *stream);

/*
 * theta[g] = max(1e-12, 1e-10 * median_l sqrt(sumsq[g*L + l] / M)) for each of
 * G groups of L lattices (default_zero_test, detect.py:42-53; even-L median
 * averages the middle pair).
 */
int sfftb_zero_thresholds(const double *sumsq, int64_t G, int64_t L, int64_t M,
                          double *theta, void *stream);

/* Words per lattice bitmap: ceil(M/32) rounded up to a multiple of 4. */
int64_t sfftb_bitmap_words(int64_t M);

/*
 * bits[(g*L + l)*W + w] bit b = |ghat[g*L + l, 32w + b]| > theta[g] (device
 * theta, one per group), W = sfftb_bitmap_words(M).  The predicate is
 * _core.pyx:195's.
 */
int sfftb_nonzero_bitmap(const double *ghat, int64_t G, int64_t L, int64_t M,
                         const double *theta, uint32_t *bits, void *stream);

/*
 * Candidate hashing + hit counting for G groups of L lattices (shared M):
 *   hits[g*n + i] = sum_l bit(g, l, elems[i] . zmat[g*L + l] mod M)
 * elems (n, d) int64 with ARBITRARY signs/magnitudes (the % M of detect.py:132
 * is fused).  kbound = sum_j max_i |elems[i, j]| when known (enables the
 * 32-bit residue path), else -1.  hits64 (G*n int64) may be NULL;
 * detmask[g*ceil(n/32) + w] bit b is set when hits of row 32w+b >= min_hits.
 * Replaces _core.pyx:164-197 (the hit half of detect_gather).
 *
 * G == 1 sets of >= 2^21 rows with even d <= 14, L <= 60 and M <= ~1.2e5 run
 * on the tensor cores: rows packed into tensor memory as the A operand of an
 * exact GEMM against per-lattice coefficient limbs, bitmaps streamed in
 * lattice groups over the resident rows; exact for ANY int64 rows (rows
 * outside the limb range are redone by an exact 64-bit kernel).
 *   csrc/hash_rollf.cu (L <= 48, M <= ~1.04e5): 8 lattices per group;
 *     kbound in [0, 2048), even d <= 12: f16 x f16 -> f32 (tcgen05.mma
 *     kind::f16, two limbs per lattice, accumulators seeded into [2^23, 2^24)
 *     and combined from their bit patterns by one integer multiply-add);
 *     otherwise, even d <= 10: u8 x u8 -> s32 (kind::i8, rows in [-2^13,
 *     2^13); kbound is not needed) -- two limbs per lattice on residues scaled
 *     by a per-lattice multiplier against bitmaps permuted to match when every
 *     lattice has such a multiplier (found on the device per call), three
 *     limbs otherwise (SFFTB_HASH_ROLLW2=0 forces three).
 *   csrc/hash_roll.cu: the other shapes (u8 x u8 -> s32, 5 lattices per group).
 * SFFTB_HASH_ROLL=0 keeps the CUDA-core kernel, SFFTB_HASH_ROLLF=0 /
 * SFFTB_HASH_ROLLW=0 skip hash_rollf.cu / its byte mode; SFFTB_HASH_TC=1
 * selects the earlier byte-GEMM kernel (csrc/hash_tc.cu).
 */
int sfftb_hash_hits(const int64_t *elems, int64_t n, int64_t d,
                    const int64_t *zmat, int64_t G, int64_t L, int64_t M,
                    const uint32_t *bits, int64_t kbound, int64_t min_hits,
                    int64_t *hits64, uint32_t *detmask, void *stream);

/* Rows the tensor-core hash sent to its exact 64-bit path since the last
 * reset (reset != 0 zeroes the counter); synchronous, for tests. */
int64_t sfftb_hash_tc_recomputed(int reset);

/* The same counter of the rolling tensor-core kernel (csrc/hash_roll.cu): rows
 * with a coordinate outside [-2^13, 2^13) that took its exact 64-bit path. */
int64_t sfftb_hash_roll_recomputed(int reset);

/* Calls served by the fp16 rolling tensor-core kernel (csrc/hash_rollf.cu:
 * single group, n >= 2^21, kbound = sum_j max|k_j| < 2048, even d <= 12,
 * L <= 48) since the last reset; for tests and the bench's kernel label. */
int64_t sfftb_hash_rollf_calls(int reset);

/* Of those, the calls its scaled two-limb byte kernel served (every lattice had
 * a multiplier t with all byte-limb coefficients t c mod M < 2^16); synchronous,
 * for tests and the bench's kernel label. */
int64_t sfftb_hash_rollf_scaled_runs(int reset);

/*
 * Ascending indices of set bits per group: idx[g*n + k], counts[g].
 * ws: sfftb_compact_workspace_bytes(G, n).
 */
int64_t sfftb_compact_workspace_bytes(int64_t G, int64_t n);
int sfftb_compact_mask(const uint32_t *mask, int64_t G, int64_t n, int64_t *idx,
                       int64_t *counts, void *ws, void *stream);

/*
 * sfftb_compact_mask with at most cap indices kept per group: idx[g*cap + k],
 * counts[g] = min(set bits, cap), totals[g] = set bits (totals may be NULL).
 * Same workspace.  Used by batched trials whose detected sets are far
 * smaller than the candidate set (analysis.py:218-250).
 */
int sfftb_compact_mask_cap(const uint32_t *mask, int64_t G, int64_t n,
                           int64_t cap, int64_t *idx, int64_t *counts,
                           int64_t *totals, void *ws, void *stream);

/*
 * Distinct lattice sizes (detect.py:134-145): for each row of vals (n, L)
 * complex128, hits[i] = #{l: hypot(vals[i, l]) > theta} and, when
 * want_medians and hits[i] >= thr, medians[i] = np.median of the real and
 * imaginary parts (mean of the two middle values for even L).
 */
int sfftb_rows_hits_medians(const double *vals, int64_t n, int64_t L, double theta,
                            double thr, int want_medians, int64_t *hits,
                            double *medians, void *stream);

/* mask bit i = hits[i] >= thr (the detection threshold nu*L, a double). */
int sfftb_threshold_mask(const int64_t *hits, int64_t n, double thr, uint32_t *mask,
                         void *stream);

/*
 * Residue tables of a Cartesian candidate set J = prefix (n1 x t) x vals (n2)
 * (pair_candidates, dimincr.py:155-175; row i = i1*n2 + i2) for GL lattices
 * with generators zmat (GL x (t+1)):  P[l*n1 + i1] = prefix[i1] . z_l[0:t]
 * mod M,  V[l*n2 + i2] = vals[i2] * z_l[t] mod M;  r_l(i) = (P + V) mod M.
 */
int sfftb_pair_residues(const int64_t *prefix, int64_t n1, int64_t t,
                        const int64_t *vals, int64_t n2, const int64_t *zmat,
                        int64_t GL, int64_t M, int32_t *P, int32_t *V, void *stream);

/* sfftb_hash_hits on a Cartesian J from its residue tables (same outputs):
 * bitmaps + tables in shared memory, sfftb_hash_pairs_smem_bytes(L, M, n2)
 * <= 200 KB. */
int64_t sfftb_hash_pairs_smem_bytes(int64_t L, int64_t M, int64_t n2);
int sfftb_hash_pairs(const int32_t *P, const int32_t *V, int64_t n1, int64_t n2,
                     int64_t G, int64_t L, int64_t M, const uint32_t *bits,
                     int64_t min_hits, int64_t *hits64, uint32_t *detmask, void *stream);

/* sfftb_medians on a Cartesian J from its residue tables (same outputs). */
int sfftb_medians_pairs(const int32_t *P, const int32_t *V, int64_t n1, int64_t n2,
                        int64_t G, int64_t L, int64_t M, const double *ghat,
                        const int64_t *idx, const int64_t *counts, int64_t cap,
                        double *coeffs, void *stream);

/*
 * Odd-L componentwise medians of the L per-lattice values of the compacted
 * rows: coeffs[g*cap + k] for row idx[g*cap + k], k < counts[g] (device).
 * The middle element of a stable sort, i.e. the reference's insertion-sort
 * median (_core.pyx:151-161, :198-200) bit for bit.
 */
int sfftb_medians(const int64_t *elems, int64_t d, const int64_t *zmat,
                  int64_t G, int64_t L, int64_t M, const double *ghat,
                  const int64_t *idx, const int64_t *counts, int64_t cap,
                  double *coeffs, void *stream);

/*
 * Gather the per-lattice values ghat[l, r_l(row)] for listed rows:
 * out[k*L + l] (per_lattice_coefficients, detect.py:112-119).
 */
int sfftb_lattice_values(const int64_t *elems, int64_t d, const int64_t *zmat,
                         int64_t L, int64_t M, const double *ghat,
                         const int64_t *rows, int64_t nrows, double *out,
                         void *stream);

/*
 * Threshold + top-s selection (detect_topk, detect.py:184-193), per group:
 * keep |c| >= theta; if more than s_tilde remain keep the s_tilde largest by
 * (|c| descending, candidate index ascending); output in ascending candidate
 * order.  In: idx/coeffs[g*cap + k], k < counts[g].  Out: kidx/kcoeffs[g*cap
 * + k], k < kcounts[g].  ws: sfftb_topk_workspace_bytes(G, cap).
 */
int64_t sfftb_topk_workspace_bytes(int64_t G, int64_t cap);
int sfftb_topk(const int64_t *idx, const double *coeffs, const int64_t *counts,
               int64_t G, int64_t cap, double theta, int64_t s_tilde,
               int64_t *kidx, double *kcoeffs, int64_t *kcounts, void *ws,
               void *stream);

/*
 * sfftb_topk for large groups (10^4 - 10^6 detected rows each, e.g. noisy
 * data where every candidate passes the zero test): the same selection and
 * output, spread over the whole GPU (grid-wide key histograms, a 12/12/12/
 * 12/12/4-bit radix select, tie masks, compaction).  Same workspace size.
 */
int sfftb_topk_grid(const int64_t *idx, const double *coeffs, const int64_t *counts,
                    int64_t G, int64_t cap, double theta, int64_t s_tilde,
                    int64_t *kidx, double *kcoeffs, int64_t *kcounts, void *ws,
                    void *stream);

/* Step-1 selection (step1_components, dimincr.py:122-152) for nlines = d*r
 * coordinate lines of K estimates each (est (nlines, K) complex128 row-major,
 * line q = (t, i) = divmod(q, r)): per line the values v of vals (nv,
 * ascending) ranked by (|est[q][v mod K]| descending, v ascending), the first
 * s_local with magnitude >= theta kept (kept[q] = their count); present
 * (d, nv) int32 = 1 where any line of coordinate t kept vals[j] (the
 * np.union1d over i).  nv <= 8192.  Replaces the host lexsort of
 * dimincr.py:143-146. */
int sfftb_step1_select(const double *est, int64_t nlines, int64_t K,
                       const int64_t *vals, int64_t nv, int64_t r, int64_t s_local,
                       double theta, int32_t *present, int64_t *kept, void *stream);

/* detect_frequencies / detect_and_compute (detect.py:149-169) on device
 * buffers in one call: samples (L, M) complex128, rows (n, d) int64, zmat
 * (L, d).  theta_in: device theta0, or NULL for the default zero test
 * (detect.py:42-53).  Outputs: hits (n), idx (n) ascending with counts[0]
 * entries, coeffs (n) medians of the detected rows when want_medians,
 * theta_out (1), bad (1) = 1 when the samples hold NaN or Inf (detect.py:
 * 98-109; the caller raises).  ws: sfftb_detect_dev_workspace_bytes(L, M, n). */
int64_t sfftb_detect_dev_workspace_bytes(int64_t L, int64_t M, int64_t n);
int sfftb_detect_dev(const double *samples, int64_t L, int64_t M, const int64_t *rows,
                     int64_t n, int64_t d, const int64_t *zmat, const double *theta_in,
                     int64_t kbound, int64_t min_hits, int want_medians, int64_t *hits,
                     int64_t *idx, int64_t *counts, double *coeffs, double *theta_out,
                     int32_t *bad, void *ws, void *stream);

/* Set mask bit i for every listed index (group union, dimincr.py:239-240). */
int sfftb_mark_indices(const int64_t *idx, const int64_t *counts, int64_t G,
                       int64_t cap, uint32_t *mask, int64_t n, void *stream);

/* dst[k] = src[rows[k]] for k < *count (device count), rows of d int64. */
int sfftb_gather_rows(const int64_t *src, int64_t d, const int64_t *rows,
                      const int64_t *count, int64_t cap, int64_t *dst,
                      void *stream);

/*
 * Cartesian candidate builder J = I_prev x I_t in lexicographic order
 * (pair_candidates, dimincr.py:155-175): out[i*n2 + j] = (prev[i], vals[j]).
 */
int sfftb_pair_product(const int64_t *prev, int64_t n1, int64_t t,
                       const int64_t *vals, int64_t n2, int64_t *out,
                       void *stream);

/* Per-coordinate (min, max) of n rows: out[2j] = min, out[2j+1] = max. */
int sfftb_row_bounds(const int64_t *elems, int64_t n, int64_t d, int64_t *out,
                     void *stream);

/*
 * Lattice sampler, step 1: anchored coefficients for G fixed tails
 *   out[g*s + k] = c_k * exp(2 pi i sum_{j >= t_dim} support[k, j] tail[g, j - t_dim])
 * (the non-lattice coordinates of dimincr.py:188-190 folded into a phase).
 */
int sfftb_anchor_coeffs(const int64_t *support, int64_t s, int64_t d,
                        int64_t t_dim, const double *coeffs, const double *tails,
                        int64_t G, double *out, void *stream);

/*
 * Lattice sampler, step 2: residue bins for G*L lattices,
 *   bins[(g*L + l)*M + h] = sum_{k : support[k, :t_dim] . z[g*L + l] = h mod M} anchored[g*s + k]
 * summed in ascending k order (deterministic; np.bincount's order,
 * polyeval.py:85-86).  ws: sfftb_scatter_workspace_bytes(G*L, s).
 */
int64_t sfftb_scatter_workspace_bytes(int64_t lattices, int64_t s);
int sfftb_scatter_bins(const int64_t *support, int64_t s, int64_t d,
                       int64_t t_dim, const double *anchored,
                       const int64_t *zmat, int64_t G, int64_t L, int64_t M,
                       double *bins, void *ws, void *stream);

/*
 * The sampler bins as per-lattice lists instead of a dense array (s <= 4096,
 * M <= 2^24): list_r[(g*L + l)*s + k], list_v[...] = (residue, bin sum) for
 * the k-th coefficient in residue order when it heads its residue's run (the
 * run summed in ascending coefficient order, like np.bincount), residue ~0
 * otherwise.  Bins without coefficients are implicit zeros.  The values carry
 * the sampler's first Bluestein product, conj(bin) * chirp_M[residue] (the
 * input sfftb_sample_detect_dft_list expects).
 */
int sfftb_scatter_list(const int64_t *support, int64_t s, int64_t d, int64_t t_dim,
                       const double *anchored, const int64_t *zmat, int64_t G,
                       int64_t L, int64_t M, uint32_t *list_r, double *list_v,
                       void *stream);

/*
 * Dense evaluation p(x) = sum_k c_k exp(2 pi i k . x) at m points X (m, d)
 * (evaluate_many, polyeval.py:66-75).
 */
int sfftb_eval_dense(const int64_t *support, int64_t s, int64_t d,
                     const double *coeffs, const double *X, int64_t m,
                     double *out, void *stream);

/*
 * Step 1's coordinate-line samples (dimincr.py:137-141) without building the
 * nodes on the host: out[q*K + j] = p(x) with x = base row q (nlines x d)
 * and coordinate q / r set to j / K.  Same arithmetic as sfftb_eval_dense on
 * those nodes.
 */
int sfftb_eval_lines(const int64_t *support, int64_t s, int64_t d,
                     const double *coeffs, const double *base, int64_t nlines,
                     int64_t K, int64_t r, double *out, void *stream);

/*
 * Harness noise: rows r of x (length M each) get sigma*(N(0,1) + i N(0,1))
 * from Philox4x32-10 keyed by seed with counter (m, call0 + r)  (the config-5
 * noise stream; restated in oracle/port.py:noise_for_call).
 */
int sfftb_add_noise(double *x, int64_t rows, int64_t M, uint64_t seed,
                    int64_t call0, double sigma, void *stream);

/* Device injectivity test of n rows mod p; result written to *injective. */
int sfftb_injective_mod_dev(const int64_t *elems, int64_t n, int64_t d,
                            int64_t p, int *injective, void *stream);

/*
 * K9 rank-1-lattice refinement (postprocess_r1l, detect.py:198-228) of n
 * detected rows (rows (n, d) int64): lattice l has generator zmat[l] and
 * size offs[l+1] - offs[l] (offs: L+1 prefix sums on the device, Msum =
 * offs[L]); vals (L, n) complex128 are the per-lattice estimates
 * ghat_l[r_l(row)] (lattice-major), medians (n) the median estimates.
 * refined[i] = mean of vals[l, i] over the lattices where row i's residue is
 * unique among the n rows (lattice order; numpy's complex/int division), else
 * medians[i]; keep bit i = |refined[i]| > theta0.
 * ws: sfftb_r1l_workspace_bytes(n, L, Msum).
 */
int64_t sfftb_r1l_workspace_bytes(int64_t n, int64_t L, int64_t Msum);
int sfftb_postprocess_r1l(const int64_t *rows, int64_t n, int64_t d,
                          const int64_t *zmat, const int64_t *offs, int64_t L,
                          int64_t Msum, const double *vals, const double *medians,
                          double theta0, double *refined, uint32_t *keep,
                          void *ws, void *stream);

/*
 * Device canonicalisation of a candidate set (FreqSet, freqset.py:48-67):
 * rows (n, d) int64 in any order, with duplicates -> out (first *count rows,
 * *count on the device) lexicographically sorted and duplicate-free.
 * Synchronises the stream once per key group (the packing plan needs the
 * per-coordinate spans).  ws: sfftb_canonicalize_workspace_bytes(n, d).
 */
int64_t sfftb_canonicalize_workspace_bytes(int64_t n, int64_t d);
int sfftb_canonicalize_rows(const int64_t *rows, int64_t n, int64_t d,
                            int64_t *out, int64_t *count, void *ws, void *stream);

/*
 * Seeded synthetic candidate rows: out (n, d) uniform on [lo, hi]^d from a
 * counter-based Philox4x32-10 stream (entry e = i*d + j, key = seed).  Not
 * numpy's stream: the reference-identical _random_from_box stays on the host.
 */
int sfftb_random_box_rows(int64_t n, int64_t d, int64_t lo, int64_t hi,
                          uint64_t seed, int64_t *out, void *stream);

/* ---------------------------------------------------------------------
 * One dimension-incremental detection stage (dimincr.py:178-192 + the union
 * of :239-240) as ONE host call: the r iterations of coordinate t share M and
 * L and run as a batch of G groups.  The call enqueues, on `stream`:
 *   prefix  = gather_rows(prev_J, prev_uidx, prev_ucount)     if prev_J
 *   J       = prefix x vals (lexicographic)                     if vals
 *   zmat, tails <- host (pinned) copies
 *   anchored/bins = structured sampler of the polynomial (support, coeffs)
 *   ghat, theta0, bits = fused sampler->detection transforms, or the unfused
 *       inverse DFT / noise / zero test / forward DFT / bitmap chain
 *   detmask = hash(J, zmat, bits); idx, counts = compaction; medians
 *   kidx, kcoeffs, kcounts = threshold + top-s_tilde per group
 *   uidx, ucount = ascending union of the kept indices      if uidx
 *   host_counts[0:G] = kcounts, host_counts[G] = ucount   (async D2H)
 * Every buffer is caller-owned (device unless noted); sizes in the comments.
 * The caller synchronises the stream before reading host_counts.
 * ------------------------------------------------------------------- */
typedef struct {
    /* candidates: J (n x tdim), n = n1 * n2, tdim = t + 1 */
    const int64_t *prev_J;      /* (n_prev x t) or NULL: prefix given */
    const int64_t *prev_uidx;   /* indices into prev_J */
    const int64_t *prev_ucount; /* device count (1) */
    int64_t *prefix;            /* (n1 x t) */
    const int64_t *vals;        /* (n2) or NULL: J given */
    int64_t n1, n2, t;
    int64_t *J;                 /* (n x tdim) */
    int64_t n, tdim;
    /* polynomial of the structured oracle (support (s x d), coeffs (s) c128) */
    const int64_t *support;
    const double *coeffs;
    int64_t s, d;
    /* lattices: G groups x L, shared M */
    int64_t G, L, M;
    const int64_t *zmat_host;   /* pinned (G*L x tdim) */
    const double *tails_host;   /* pinned (G x tail_w) */
    int64_t tail_w;             /* max(d - tdim, 1) */
    int64_t *zmat;              /* (G*L x tdim) */
    double *tails;              /* (G x tail_w) */
    uint64_t noise_seed;
    int64_t call0;
    double sigma;
    int fused;                  /* 1: sfftb_sample_detect_dft */
    /* detection */
    int64_t kbound, min_hits, s_tilde;
    double theta;
    /* buffers */
    double *anchored;           /* (G x s) c128 */
    double *bins;               /* (G*L x M) c128 */
    double *samples;            /* (G*L x M) c128, unfused only */
    double *ghat;               /* (G*L x M) c128 */
    double *theta0;             /* (G) */
    double *sumsq;              /* (G*L), unfused only */
    uint32_t *bits;             /* (G*L x W) */
    void *ws_dft;               /* max(sample_detect, dft) workspace */
    uint32_t *detmask;          /* (G x ceil(n/32)) */
    int64_t *idx;               /* (G x n) */
    int64_t *counts;            /* (G) */
    double *med;                /* (G x n) c128 */
    void *ws_compact;           /* compact_workspace_bytes(G, n) */
    int64_t *kidx;              /* (G x n) */
    double *kco;                /* (G x n) c128 */
    int64_t *kcounts;           /* (G) */
    void *ws_topk;              /* topk_workspace_bytes(G, n) */
    uint32_t *umask;            /* (ceil(n/32)) or NULL: no union */
    int64_t *uidx;              /* (n) */
    int64_t *ucount;            /* (1) */
    int64_t *host_counts;       /* pinned (G + 1) */
    /* optional: 9 cudaEvent_t recorded at the phase boundaries: candidates
     * start, end | sampler start | transforms start, end | hashing start, end
     * | compaction+medians end | top-s+union end */
    void *const *events;
    /* elements between consecutive groups in zmat_host (0: dense G*L*tdim);
     * lets the host pre-draw L_cap >= L generators per group before L is known */
    int64_t zmat_host_ld;
    /* optional residue tables of the Cartesian J (pair stages): ptab
     * (G*L x n1) and vtab (G*L x n2) int32; NULL: generic hashing/medians */
    int32_t *ptab;
    int32_t *vtab;
    /* 1: the top-s selection runs grid-wide (sfftb_topk_grid) -- set when
     * large detected sets are expected (the previous stage saturated) */
    int64_t topk_grid;
    /* 0: the whole stage.  1: spectra only -- the zmat/tails copies, the
     * sampler and the transforms (ghat, theta0, bits), which do not depend on
     * the candidate set, so the driver enqueues them for stage t+1 before it
     * waits for stage t's counts.  2: the rest (candidates, hashing,
     * compaction, medians, top-s, union) on the spectra of an earlier phase-1
     * call with the same G, L, M, zmat and call0.  3 and 4 split phase 1: the
     * sampler (zmat/tails copies, anchor, scatter into bins) and the
     * transforms on those bins, so the sampler can run on another stream. */
    int64_t phase;
} sfftb_stage_t;

int sfftb_sfft_stage(const sfftb_stage_t *st, void *stream);

/* ---------------------------------------------------------------------
 * Experiment harness (csrc/analysis.cu; reference latfft/analysis.py and
 * the f10 test function of polyeval.py:216-277).
 * ------------------------------------------------------------------- */

/*
 * mask bit i = (rows[i] is a row of pool), pool lexicographically sorted and
 * duplicate-free (FreqSet.contains_rows, freqset.py:139-142).  Device.
 */
int sfftb_rows_in_sorted(const int64_t *rows, int64_t n, int64_t d,
                         const int64_t *pool, int64_t m, uint32_t *mask,
                         void *stream);

/*
 * Alias classification of pfp_pfn_count (analysis.py:67-104) for G groups of
 * detected rows idx/med[g*cap + k], k < counts[g], against in_mask (bit per
 * candidate: member of I).  rounded = rint(Re), integral = |Re - rounded| <=
 * tol and |Im| <= tol.  tallies[g*5 + c]: c = 0 detected & in_I, 1 not
 * integral, 2 integral & rounded < 1, 3 pfn (in_I & rounded >= 2), 4 pfp
 * (not in_I & rounded >= 1).  cls[g*cap + k] (may be NULL): bit 0 = in_I,
 * bits 1-3 = 0 clean, 1 not integral, 2 rounded < 1, 3 pfn, 4 pfp.
 */
int sfftb_alias_classify(const int64_t *idx, const double *med,
                         const int64_t *counts, int64_t G, int64_t cap,
                         const uint32_t *in_mask, double tol, uint8_t *cls,
                         int64_t *tallies, void *stream);

/*
 * Sum over groups of products of periodised B-splines (f10_values,
 * polyeval.py:261-272): value(x) = sum_g prod_{a: axis_group[a] == g}
 * scale[g] * N_{order[g]}(x_a), N_m the centred cardinal B-spline of
 * bspline_values (polyeval.py:216-225) without its prefactor scale = C_m * m.
 * axis_group[a] = -1 leaves axis a out.  d <= 32, ngroups <= 8.
 * _lattice: out (G*L, M) complex128 at the nodes [(j z mod M)/M | tail_g]
 * (zmat (G*L, t_dim), tails (G, max(d - t_dim, 1))).  _points: out (m,) at X
 * (m, d).  Device.
 */
int sfftb_spline_sum_lattice(int64_t d, const int32_t *axis_group,
                             int64_t ngroups, const int32_t *order,
                             const double *scale, const int64_t *zmat,
                             int64_t G, int64_t L, int64_t M, int64_t t_dim,
                             const double *tails, double *out, void *stream);
int sfftb_spline_sum_points(int64_t d, const int32_t *axis_group,
                            int64_t ngroups, const int32_t *order,
                            const double *scale, const double *X, int64_t m,
                            double *out, void *stream);

/* ---------------------------------------------------------------------
 * Host seed streams (csrc/hostrng.cpp): numpy Generator(PCG64(SeedSequence(
 * entropy))) restated, for the driver's per-iteration streams
 * (dimincr.py:99-100).  State = 6 x uint64 per stream (state hi/lo, inc
 * hi/lo, has_uint32, uinteger).  Host memory only; no device work.
 * ------------------------------------------------------------------- */

/* rows streams; row r's SeedSequence entropy words (uint32, assembled as
 * numpy's _coerce_to_uint32_array) are words[r*nwords:(r+1)*nwords]. */
int sfftb_pcg64_seed(const uint32_t *words, int64_t rows, int64_t nwords,
                     uint64_t *states);

/* out (rows, count): Generator.random() / uniform(0, 1) draws per stream. */
int sfftb_pcg64_random(uint64_t *states, int64_t rows, int64_t count,
                       double *out);

/* out (rows, count): Generator.integers(low, high_incl + 1, dtype=int64). */
int sfftb_pcg64_integers(uint64_t *states, int64_t rows, int64_t low,
                         int64_t high_incl, int64_t count, int64_t *out);

/* Advance one stream's PCG64 by `delta` 64-bit outputs (LCG jump-ahead).
 * tables (may be NULL): the jump-by-2^i maps s -> A_i s + C_i, i < 64, as
 * (A hi, A lo, C hi, C lo) -- the input of sfftb_box_integers. */
int sfftb_pcg64_advance(uint64_t *state, uint64_t delta, uint64_t *tables);

/* Generator.choice(pop, size, replace=False) in numpy's tail-shuffle regime
 * (pop > 10000 and size > pop // 50; _generator.pyx _shuffle_int from the
 * top of arange(pop)): out (size) the chosen indices in numpy's order, the
 * state advanced exactly.  final_shuffle must be 0 to match numpy 2.x. */
int sfftb_pcg64_choice_tail(uint64_t *state, int64_t pop, int64_t size,
                            int final_shuffle, int64_t *out);

/*
 * Generator.integers(low, high_incl + 1, size=n, dtype=int64) on the DEVICE
 * in numpy's exact stream (freqset.py:273-275; csrc/boxgen.cu), for
 * high_incl - low < 2^32 - 1: out (device, n).  state6 (host) is the stream
 * before the draw and is not modified; jump = sfftb_pcg64_advance tables of
 * it.  extra = spare 32-bit words for Lemire rejections.  Synchronous: on
 * return *words_used = 32-bit words consumed, *last_hi = the high half of the
 * 64-bit output that held the last one (the caller rebuilds the state).
 */
int64_t sfftb_box_integers_workspace_bytes(int64_t n, int64_t extra);
int sfftb_box_integers(const uint64_t *state6, const uint64_t *jump, int64_t low,
                       int64_t high_incl, int64_t n, int64_t extra, int64_t *out,
                       void *ws, int64_t *words_used, uint64_t *last_hi,
                       void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SFFT_B200_H */
