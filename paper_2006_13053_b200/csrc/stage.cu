// One detection stage of the dimension-incremental driver as a single host
// call (include/sfft_b200.h: sfftb_sfft_stage), or its two halves: the
// spectra (phase 1: sampler + transforms, independent of the candidate set)
// and the detection on them (phase 2).  No new device code: the
// stage is the sequence of the library's own entry points that the Python
// driver issued one ctypes call at a time (dimincr.py _detect_stage +
// _engine), composed here so the ~12 launches of a stage cost microseconds
// of host time instead of ~0.3 ms of interpreter overhead while the GPU idles
// between stages.
#include <stdlib.h>

#include <mutex>

#include "common.cuh"
#include "../../include/sfft_b200.h"

#define SFFTB_TRY(x)                    \
    do {                                \
        const int rc_ = (x);            \
        if (rc_ != SFFTB_OK) return rc_; \
    } while (0)

namespace {

struct Marks {
    const sfftb_stage_t* a;
    cudaStream_t st;
    int operator()(int k) const {
        if (a->events && a->events[k])
            SFFTB_CUDA(cudaEventRecord((cudaEvent_t)a->events[k], st));
        return SFFTB_OK;
    }
};

// prefix gather + pair product
int stage_candidates(const sfftb_stage_t* a, void* stream, const Marks& mark) {
    SFFTB_TRY(mark(0));
    if (a->prev_J) {
        SFFTB_TRY(sfftb_gather_rows(a->prev_J, a->t, a->prev_uidx, a->prev_ucount, a->n1,
                                    a->prefix, stream));
    }
    if (a->vals) {
        SFFTB_REQUIRE(a->n1 * a->n2 == a->n && a->t + 1 == a->tdim, "stage: pair sizes");
        SFFTB_TRY(sfftb_pair_product(a->prefix, a->n1, a->t, a->vals, a->n2, a->J, stream));
    }
    SFFTB_TRY(mark(1));
    return SFFTB_OK;
}

// generators/tails H2D, structured sampler (parts & 1), transforms -> ghat,
// theta0, bits (parts & 2)
int stage_spectra(const sfftb_stage_t* a, void* stream, const Marks& mark, int parts) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t G = a->G, L = a->L, M = a->M, tdim = a->tdim;
    const int64_t rows = G * L;
    // fused path with few coefficients: sparse bins (residue lists) in the
    // bins buffer -- no dense zero fill, the first column pass drops them in
    static const bool lists_on = [] {
        const char* e = getenv("SFFTB_LISTS");
        return !e || atoi(e) != 0;
    }();
    const bool listed = lists_on && a->fused && a->s >= 1 && a->s <= 4096 &&
                        M <= (int64_t(1) << 24) && M >= 2 * a->s;
    uint32_t* list_r = reinterpret_cast<uint32_t*>(a->bins + 2 * rows * a->s);
    if (parts & 1) {
    SFFTB_TRY(mark(2));
    if (a->zmat_host_ld > 0 && a->zmat_host_ld != L * tdim) {
        SFFTB_REQUIRE(a->zmat_host_ld >= L * tdim, "stage: zmat_host_ld < L*tdim");
        SFFTB_CUDA(cudaMemcpy2DAsync(a->zmat, (size_t)(L * tdim) * sizeof(int64_t), a->zmat_host,
                                     (size_t)a->zmat_host_ld * sizeof(int64_t),
                                     (size_t)(L * tdim) * sizeof(int64_t), (size_t)G,
                                     cudaMemcpyHostToDevice, st));
    } else {
        SFFTB_CUDA(cudaMemcpyAsync(a->zmat, a->zmat_host,
                                   (size_t)(rows * tdim) * sizeof(int64_t),
                                   cudaMemcpyHostToDevice, st));
    }
    SFFTB_CUDA(cudaMemcpyAsync(a->tails, a->tails_host,
                               (size_t)(G * a->tail_w) * sizeof(double),
                               cudaMemcpyHostToDevice, st));

    // structured sampler: anchored coefficients -> residue bins
    if (a->s > 0)
        SFFTB_TRY(sfftb_anchor_coeffs(a->support, a->s, a->d, tdim, a->coeffs, a->tails, G,
                                      a->anchored, stream));
    if (listed)
        SFFTB_TRY(sfftb_scatter_list(a->support, a->s, a->d, tdim, a->anchored, a->zmat, G, L,
                                     M, list_r, a->bins, stream));
    else
        SFFTB_TRY(sfftb_scatter_bins(a->support, a->s, a->d, tdim, a->anchored, a->zmat, G, L,
                                     M, a->bins, nullptr, stream));

    SFFTB_TRY(mark(3));
    }
    if (!(parts & 2)) return SFFTB_OK;

    // samples -> zero test, spectra, bitmaps
    if (!(parts & 1)) SFFTB_TRY(mark(3));
    const char* split_env = getenv("SFFTB_SPLIT_GROUPS");
    const bool split = listed && G >= 2 && split_env && atoi(split_env) > 0;
    if (split) {
        // one transform chain per group, alternating between this stream and a
        // second one: a group's 5 passes stay in L2 and the two chains fill
        // each other's kernel tails
        // per-device second stream and events, created once under a lock (the
        // driver runs one arena per host thread); the events are recorded and
        // waited on under the same lock so that two threads never interleave
        // their record/wait pairs
        static std::mutex split_mu;
        static cudaStream_t st2[64] = {nullptr};
        static cudaEvent_t evs[64][2];
        int dev = 0;
        SFFTB_CUDA(cudaGetDevice(&dev));
        SFFTB_REQUIRE(dev >= 0 && dev < 64, "stage: device index out of range");
        std::lock_guard<std::mutex> split_lock(split_mu);
        if (!st2[dev]) {
            SFFTB_CUDA(cudaStreamCreateWithFlags(&st2[dev], cudaStreamNonBlocking));
            SFFTB_CUDA(cudaEventCreateWithFlags(&evs[dev][0], cudaEventDisableTiming));
            SFFTB_CUDA(cudaEventCreateWithFlags(&evs[dev][1], cudaEventDisableTiming));
        }
        SFFTB_CUDA(cudaEventRecord(evs[dev][0], st));
        SFFTB_CUDA(cudaStreamWaitEvent(st2[dev], evs[dev][0], 0));
        const int64_t W = sfftb_bitmap_words(M);
        // per-group workspace regions, 256-B aligned (the caller's buffer has
        // G * 256 bytes of slack: sfftb_stage_t.ws_dft)
        const int64_t wsg = (sfftb_sample_detect_workspace_bytes(L, M) + 255) & ~int64_t(255);
        for (int64_t g = 0; g < G; ++g) {
            cudaStream_t sg = (g & 1) ? st2[dev] : st;
            SFFTB_TRY(sfftb_sample_detect_dft_list(
                list_r + g * L * a->s, a->bins + 2 * g * L * a->s, a->s, 1, L, M, a->noise_seed,
                a->call0 + g * L, a->sigma, a->ghat + 2 * g * L * M, a->theta0 + g,
                a->bits + g * L * W, (char*)a->ws_dft + g * wsg, sg));
        }
        SFFTB_CUDA(cudaEventRecord(evs[dev][1], st2[dev]));
        SFFTB_CUDA(cudaStreamWaitEvent(st, evs[dev][1], 0));
    } else if (listed) {
        SFFTB_TRY(sfftb_sample_detect_dft_list(list_r, a->bins, a->s, G, L, M, a->noise_seed,
                                               a->call0, a->sigma, a->ghat, a->theta0, a->bits,
                                               a->ws_dft, stream));
    } else if (a->fused) {
        SFFTB_TRY(sfftb_sample_detect_dft(a->bins, G, L, M, a->noise_seed, a->call0, a->sigma,
                                          a->ghat, a->theta0, a->bits, a->ws_dft, stream));
    } else {
        const int64_t step = 65535;
        for (int64_t b0 = 0; b0 < rows; b0 += step) {
            const int64_t nb = rows - b0 < step ? rows - b0 : step;
            SFFTB_TRY(sfftb_dft(a->bins + 2 * b0 * M, M, a->samples + 2 * b0 * M, M, nb, M, 1,
                                1.0, a->ws_dft, stream));
        }
        if (a->sigma > 0)
            SFFTB_TRY(sfftb_add_noise(a->samples, rows, M, a->noise_seed, a->call0, a->sigma,
                                      stream));
        SFFTB_TRY(sfftb_sumsq(a->samples, M, rows, M, a->sumsq, stream));
        SFFTB_TRY(sfftb_zero_thresholds(a->sumsq, G, L, M, a->theta0, stream));
        for (int64_t b0 = 0; b0 < rows; b0 += step) {
            const int64_t nb = rows - b0 < step ? rows - b0 : step;
            SFFTB_TRY(sfftb_dft(a->samples + 2 * b0 * M, M, a->ghat + 2 * b0 * M, M, nb, M, 0,
                                1.0 / (double)M, a->ws_dft, stream));
        }
        SFFTB_TRY(sfftb_nonzero_bitmap(a->ghat, G, L, M, a->theta0, a->bits, stream));
    }
    SFFTB_TRY(mark(4));
    return SFFTB_OK;
}

// hashing, compaction, medians, top-s, union, count read-back
int stage_detect(const sfftb_stage_t* a, void* stream, const Marks& mark) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t G = a->G, L = a->L, M = a->M, n = a->n, tdim = a->tdim;
    const int64_t rows = G * L;
    SFFTB_TRY(mark(5));
    // Cartesian J (pair stages): residues from per-lattice tables of the
    // prefix and value parts -- n1 + n2 dot products per lattice, not n1*n2
    // (table hashing beats the resident dot-product kernel from ~8 coordinates
    // on: measured 23+7 vs 29 us at 7, 48+11 vs 117 us at 19; tools/prof_pairs.py)
    const bool pairs = a->vals && a->ptab && a->vtab && a->n2 >= 1;
    const bool hash_pairs =
        pairs && tdim >= 8 && sfftb_hash_pairs_smem_bytes(L, M, a->n2) <= 200 * 1024;
    if (n > 0) {
        if (pairs)
            SFFTB_TRY(sfftb_pair_residues(a->prefix, a->n1, a->t, a->vals, a->n2, a->zmat, rows,
                                          M, a->ptab, a->vtab, stream));
        if (hash_pairs) {
            SFFTB_TRY(sfftb_hash_pairs(a->ptab, a->vtab, a->n1, a->n2, G, L, M, a->bits,
                                       a->min_hits, nullptr, a->detmask, stream));
        } else {
            SFFTB_TRY(sfftb_hash_hits(a->J, n, tdim, a->zmat, G, L, M, a->bits, a->kbound,
                                      a->min_hits, nullptr, a->detmask, stream));
        }
        SFFTB_TRY(mark(6));
        // noisy data detects (nearly) every candidate: dense masks compact
        // faster over many blocks
        SFFTB_TRY(sfftb::compact_mask_launch(a->detmask, G, n, n, a->idx, a->counts, nullptr,
                                             a->ws_compact, stream,
                                             a->sigma > 0.0 ? 1024 : 8192));
        if (pairs)  // noisy data: (nearly) every candidate detected
            SFFTB_TRY(sfftb::medians_pairs_launch(a->ptab, a->vtab, a->n1, a->n2, G, L, M,
                                                  a->ghat, a->idx, a->counts, n, a->med, stream,
                                                  a->sigma > 0.0));
        else
            SFFTB_TRY(sfftb_medians(a->J, tdim, a->zmat, G, L, M, a->ghat, a->idx, a->counts,
                                    n, a->med, stream));
    } else {
        SFFTB_TRY(mark(6));
        SFFTB_CUDA(cudaMemsetAsync(a->counts, 0, (size_t)G * sizeof(int64_t), st));
    }
    SFFTB_TRY(mark(7));
    const int64_t cap = n > 0 ? n : 1;
    if (a->topk_grid && cap >= 16384)
        SFFTB_TRY(sfftb_topk_grid(a->idx, a->med, a->counts, G, cap, a->theta, a->s_tilde,
                                  a->kidx, a->kco, a->kcounts, a->ws_topk, stream));
    else
        SFFTB_TRY(sfftb_topk(a->idx, a->med, a->counts, G, cap, a->theta, a->s_tilde, a->kidx,
                             a->kco, a->kcounts, a->ws_topk, stream));
    SFFTB_CUDA(cudaMemcpyAsync(a->host_counts, a->kcounts, (size_t)G * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));

    // union of the kept indices (ascending)
    if (a->umask && G == 1) {
        // one group: its kept indices are already the ascending union (the
        // top-s emits in candidate order) -- two copies instead of mark +
        // compaction on the latency-bound tail stages
        const int64_t keep = std::min<int64_t>(cap, std::max<int64_t>(a->s_tilde, 1));
        SFFTB_CUDA(cudaMemcpyAsync(a->uidx, a->kidx, (size_t)keep * sizeof(int64_t),
                                   cudaMemcpyDeviceToDevice, st));
        SFFTB_CUDA(cudaMemcpyAsync(a->ucount, a->kcounts, sizeof(int64_t),
                                   cudaMemcpyDeviceToDevice, st));
        SFFTB_CUDA(cudaMemcpyAsync(a->host_counts + G, a->ucount, sizeof(int64_t),
                                   cudaMemcpyDeviceToHost, st));
    } else if (a->umask) {
        const int64_t nwords = (n + 31) / 32 > 0 ? (n + 31) / 32 : 1;
        SFFTB_CUDA(cudaMemsetAsync(a->umask, 0, (size_t)nwords * sizeof(uint32_t), st));
        SFFTB_TRY(sfftb_mark_indices(a->kidx, a->kcounts, G, cap, a->umask, n, stream));
        if (n > 0) {
            SFFTB_TRY(sfftb_compact_mask(a->umask, 1, n, a->uidx, a->ucount, a->ws_compact,
                                         stream));
        } else {
            SFFTB_CUDA(cudaMemsetAsync(a->ucount, 0, sizeof(int64_t), st));
        }
        SFFTB_CUDA(cudaMemcpyAsync(a->host_counts + G, a->ucount, sizeof(int64_t),
                                   cudaMemcpyDeviceToHost, st));
    }
    SFFTB_TRY(mark(8));
    return SFFTB_OK;
}

}  // namespace

extern "C" int sfftb_sfft_stage(const sfftb_stage_t* a, void* stream) {
    SFFTB_REQUIRE(a != nullptr, "stage: null descriptor");
    SFFTB_REQUIRE(a->G >= 1 && a->L >= 1 && a->M >= 1 && a->tdim >= 1 && a->n >= 0,
                  "stage: bad sizes");
    SFFTB_REQUIRE(a->d >= a->tdim && a->tail_w >= 1, "stage: bad dimensions");
    SFFTB_REQUIRE(a->phase >= 0 && a->phase <= 4, "stage: phase must be 0 .. 4");
    const Marks mark{a, (cudaStream_t)stream};
    if (a->phase == 1) return stage_spectra(a, stream, mark, 3);
    if (a->phase == 3) return stage_spectra(a, stream, mark, 1);
    if (a->phase == 4) return stage_spectra(a, stream, mark, 2);
    SFFTB_TRY(stage_candidates(a, stream, mark));
    if (a->phase == 0) SFFTB_TRY(stage_spectra(a, stream, mark, 3));
    return stage_detect(a, stream, mark);
}
