// Candidate hashing, hit counting, detected-row compaction and medians.
//
// Replaces the reference's per-candidate gather (latfft/_kernels/_core.pyx:
// 164-202; semantics of fallback.py:106-131) and the index bookkeeping of
// detect.py:122-169.
//
// Design:
//  * the L*M per-lattice values are reduced once to nonzero BITMAPS
//    (bit = |ghat| > theta, the exact predicate of _core.pyx:195) which live
//    in shared memory, W = ceil(M/32) words per lattice;
//  * each thread keeps R candidate rows in registers and walks the lattices:
//    residue by 32-bit IMAD chain (exact when sum_j max|k_j| * M/2 fits, the
//    common case, checked on the host) or a 64-bit chain otherwise, then a
//    multiply-high modular reduction and one bitmap probe per (row, lattice);
//  * when the bitmaps of all L lattices exceed the shared-memory budget they
//    are streamed through shared memory in lattice chunks per row tile;
//  * detected rows (hits >= nu*L) leave a warp-ballot bitmask that
//    sfftb_compact_mask turns into ascending indices; medians are computed
//    only for those rows, one warp per row.
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "median_nets.cuh"

namespace sfftb {

static constexpr int kHashThreads = 512;
static constexpr size_t kBitmapSmemBudget = 224 * 1024;
static constexpr size_t kStreamSmemBudget = 160 * 1024;

struct HashArgs {
    const int64_t* elems;
    int64_t n;
    int d;
    const int64_t* zmat;  // G*L*d
    int G, L;
    int64_t M;
    const uint32_t* bits;  // G*L*W
    int64_t W;
    int Lc;              // lattices per shared-memory chunk
    int nbuf;            // 1 (all bitmaps resident) or 2 (double-buffered chunks)
    int slot_words;      // power-of-two smem stride per lattice bitmap (>= W)
    uint32_t offset;     // multiple of M >= |residue sum| (32-bit path)
    uint32_t magic;      // floor((2^32-1)/M)
    int64_t min_hits;
    int64_t* hits64;     // may be null
    uint32_t* detmask;   // G * ceil(n/32)
    int64_t nwords;
    int xsplit;          // FP64 coordinates of the 32-bit path (0: all IMAD)
    int variant;         // tuning-table entry (d = 10)
    int64_t auto_sum;    // AUTO: rows with sum_j |k_j| <= auto_sum take the 32-bit path
    int64_t auto_bias;   // AUTO: multiple of M >= d * M * (M/2), keeps 64-bit sums >= 0
};

// FP64/IMAD split of the 32-bit dot product (see hash_rows): opt-in only
static int hash_x_for(int d, int variant) {
    return (d == 10 && (variant == 1 || variant == 2)) ? 5 : 0;
}

// r = u mod M for u < 2^32: q = umulhi(u, floor((2^32-1)/M)) is floor(u/M)
// or one less, so u + q*(-M) lies in [0, 2M) and one unsigned min finishes.
__device__ __forceinline__ uint32_t mod_u32(uint32_t u, uint32_t M, uint32_t negM,
                                            uint32_t magic) {
    const uint32_t q = __umulhi(u, magic);
    uint32_t r;
    // one IMAD with the precomputed -M (keeps ptxas from negating q first)
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(negM), "r"(u));
    return min(r, r - M);
}

// Bit r of a bitmap whose shared address `slot` is aligned to a power of two
// larger than its size: the word address is slot | ((r >> 3) & ~3), two ALU
// ops (SHF + LOP3) and no IMAD-pipe add.
__device__ __forceinline__ uint32_t probe_slot(uint32_t slot, uint32_t r) {
    uint32_t w;
    asm volatile("{\n\t.reg .u32 a;\n\t"
                 "shr.u32 a, %1, 3;\n\t"
                 "lop3.b32 a, a, 0xFFFFFFFC, %2, 0xEA;\n\t"
                 "ld.shared.u32 %0, [a];\n\t}"
                 : "=r"(w)
                 : "r"(r), "r"(slot));
    return __funnelshift_r(w, w, r) & 1u;
}

// The probed words themselves (bit r & 31 is the answer): the caller shifts
// that bit into a per-row bit accumulator instead of adding it.
__device__ __forceinline__ uint32_t word_slot(uint32_t slot, uint32_t r) {
    uint32_t w;
    asm volatile("{\n\t.reg .u32 a;\n\t"
                 "shr.u32 a, %1, 3;\n\t"
                 "lop3.b32 a, a, 0xFFFFFFFC, %2, 0xEA;\n\t"
                 "ld.shared.u32 %0, [a];\n\t}"
                 : "=r"(w)
                 : "r"(r), "r"(slot));
    return w;
}

__device__ __forceinline__ uint32_t word_bit(uint32_t base, uint32_t r) {
    uint32_t w;
    asm volatile("{\n\t.reg .u32 a;\n\t"
                 "shr.u32 a, %1, 5;\n\t"
                 "shl.b32 a, a, 2;\n\t"
                 "add.u32 a, a, %2;\n\t"
                 "ld.shared.u32 %0, [a];\n\t}"
                 : "=r"(w)
                 : "r"(r), "r"(base));
    return w;
}

// acc' = (acc >> 1) | (bit r of w) << 31: rotate bit r down to position 0,
// funnel it in from the top -- two shifts on the ALU pipe (the per-lattice hit
// add would otherwise be an IMAD on the already saturated FMA-heavy pipe);
// popc every 32 lattices.
__device__ __forceinline__ uint32_t shift_in_bit(uint32_t acc, uint32_t w, uint32_t r) {
    const uint32_t rot = __funnelshift_r(w, w, r);  // bit r & 31 -> bit 0
    return __funnelshift_r(acc, rot, 1);            // (rot:acc) >> 1
}

// Bit r of the bitmap at shared address `base`: word (r >> 5), bit r & 31.
__device__ __forceinline__ uint32_t probe_bit(uint32_t base, uint32_t r) {
    uint32_t w;
    asm volatile("{\n\t.reg .u32 a;\n\t"
                 "shr.u32 a, %1, 3;\n\t"
                 "and.b32 a, a, 0xFFFFFFFC;\n\t"
                 "add.u32 a, a, %2;\n\t"
                 "ld.shared.u32 %0, [a];\n\t}"
                 : "=r"(w)
                 : "r"(r), "r"(base));
    return __funnelshift_r(w, w, r) & 1u;
}


// Synchronous cooperative copy (generic fallback kernel only).
__device__ __forceinline__ void load_bits(uint32_t* dst, const HashArgs& a, int g, int l0,
                                          int cnt) {
    const uint4* src = reinterpret_cast<const uint4*>(a.bits + ((int64_t)g * a.L + l0) * a.W);
    const int64_t words = (int64_t)cnt * a.W;
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t i = threadIdx.x; i < words / 4; i += blockDim.x) d4[i] = __ldg(src + i);
}

// Candidate rows of one warp slice into registers (row = base + q*32 + lane).
template <int D, int R, bool WIDE>
__device__ __forceinline__ void load_rows(const HashArgs& a, int64_t base, int lane,
                                          int32_t (&k)[R][D], uint32_t (&ku)[WIDE ? R : 1][WIDE ? D : 1],
                                          bool (&valid)[R], bool* all_safe = nullptr) {
    bool safe = true;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int64_t i = base + q * 32 + lane;
        valid[q] = i < a.n;
        const int64_t* row = a.elems + (valid[q] ? i : 0) * D;
        int64_t v[D];
        if (D % 2 == 0) {
#pragma unroll
            for (int j = 0; j < D; j += 2) {
                const longlong2 p = __ldg(reinterpret_cast<const longlong2*>(row + j));
                v[j] = p.x;
                v[j + 1] = p.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < D; ++j) v[j] = __ldg(row + j);
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (!valid[q]) v[j] = 0;
            if (WIDE) {
                int64_t m = v[j] % a.M;
                if (m < 0) m += a.M;
                ku[WIDE ? q : 0][WIDE ? j : 0] = (uint32_t)m;
                k[q][j] = 0;
            } else {
                k[q][j] = (int32_t)v[j];
            }
        }
        if (all_safe) {  // AUTO: the 32-bit path is exact for this row?
            int64_t sum = 0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const uint64_t m = v[j] < 0 ? (uint64_t)0 - (uint64_t)v[j] : (uint64_t)v[j];
                sum += m >= ((uint64_t)1 << 40) ? ((int64_t)1 << 40) : (int64_t)m;
            }
            safe = safe && sum <= a.auto_sum;
        }
    }
    if (all_safe) *all_safe = __all_sync(0xffffffffu, safe);
}

// AUTO tiles with a row outside the 32-bit bound: the rows again, reduced mod M
// (exact for any int64), into the same registers.
template <int D, int R>
__device__ __forceinline__ void load_rows_reduced(const HashArgs& a, int64_t base, int lane,
                                                  int32_t (&k)[R][D]) {
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int64_t i = base + q * 32 + lane;
        const int64_t* row = a.elems + (i < a.n ? i : 0) * D;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            int64_t m = __ldg(row + j) % a.M;
            if (m < 0) m += a.M;
            k[q][j] = (int32_t)m;
        }
    }
}

// WIDE = false: 32-bit residue path (values truncated to int32, exact by the
// host's bound check); WIDE = true: exact 64-bit path for any int64 input.
//
// Shared memory: [z (L*D int32)] [2 mbarriers] [bitmap buffer 0] [buffer 1].
// With nbuf == 2 the bitmaps of Lc lattices at a time stream through two
// buffers: thread 0 issues a 1-D bulk copy (TMA engine, completion on an
// mbarrier) for chunk q+2 as soon as every warp is done with chunk q, so the
// L2 -> SMEM transfer overlaps the hashing of chunk q+1.
// X > 0 (32-bit path only): the first X coordinates of each dot product run
// as FP64 FMAs on the FP64 pipe, the remaining D - X as IMADs on the FMA-heavy
// pipe, so the two pipes share the multiply work.  The FP64 accumulator starts
// at 1.5*2^52 + offset: every partial sum is an exact integer in [2^52, 2^53)
// whose low 32 mantissa bits are (offset + sum_{j<X} k_j z_j) mod 2^32, and
// that word seeds the integer chain -- bit-identical to the all-IMAD sum.
// AUTO (32-bit instantiation only): no host bound on the rows; each warp
// checks its rows (sum_j |k_j| <= auto_sum) and takes the 32-bit chain when
// all pass, otherwise the exact 64-bit chain on rows reduced mod M.
template <int D, int R, bool WIDE, int NT = kHashThreads, bool SLOT = false, int X = 0,
          bool AUTO = false>
__global__ void __launch_bounds__(NT, 1) hash_rows(HashArgs a) {
    extern __shared__ __align__(16) uint32_t smem_u32[];
    const int g = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int WARPS = NT / 32;
    constexpr int TILE = WARPS * 32 * R;
    const uint32_t M32 = (uint32_t)a.M, negM = 0u - M32;

    int32_t* zc = reinterpret_cast<int32_t*>(smem_u32);
    const int zwords = ((a.L * D + 3) & ~3);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_u32 + zwords);
    double* zd = reinterpret_cast<double*>(smem_u32 + zwords + 4);
    const int zdwords = X > 0 ? ((a.L * X * 2 + 3) & ~3) : 0;
    // bitmap slots: one per lattice, stride slot_words (a power of two >= W),
    // from the first shared address aligned to the stride
    const uint32_t slot_bytes = (uint32_t)a.slot_words * 4u;
    const uint32_t after = smem_addr(smem_u32 + zwords + 4 + zdwords);
    const uint32_t slot0 = SLOT ? (after + slot_bytes - 1) & ~(slot_bytes - 1) : after;
    const uint32_t slot1 = slot0 + (uint32_t)a.Lc * slot_bytes;
    for (int i = threadIdx.x; i < a.L * D; i += blockDim.x) {
        int64_t z = a.zmat[(int64_t)g * a.L * D + i] % a.M;
        if (z < 0) z += a.M;
        if (!WIDE && z > a.M / 2) z -= a.M;
        zc[i] = (int32_t)z;
        if (X > 0 && (i % D) < X) zd[(i / D) * X + (i % D)] = (double)z;
    }
    const double dmagic = 6755399441055744.0 + (double)a.offset;  // 1.5*2^52 + offset
    const int nchunks = (a.L + a.Lc - 1) / a.Lc;
    const bool resident = nchunks == 1;
    const int64_t ntiles = (a.n + TILE - 1) / TILE;
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total_q = resident ? (my_tiles ? 1 : 0) : my_tiles * nchunks;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t qi) {
        const int c = resident ? 0 : (int)(qi % nchunks);
        const int l0 = c * a.Lc;
        const int cnt = min(a.L, l0 + a.Lc) - l0;
        const uint32_t bytes = (uint32_t)(a.W * 4);
        uint64_t* bar = &bars[qi & 1];
        mbar_arrive_expect_tx(bar, bytes * (uint32_t)cnt);
        const uint32_t dst0 = (qi & 1) ? slot1 : slot0;
        for (int l = 0; l < cnt; ++l)
            bulk_g2s_addr(dst0 + (uint32_t)l * slot_bytes,
                          a.bits + ((int64_t)g * a.L + l0 + l) * a.W, bytes, bar);
    };
    if (threadIdx.x == 0) {
        if (total_q > 0) issue(0);
        if (total_q > 1) issue(1);
    }

    const double invM = 1.0 / (double)a.M;
    int64_t qc = 0;  // chunk counter of this CTA
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * TILE + (int64_t)warp * 32 * R;
        int32_t k[R][D];
        uint32_t ku[WIDE ? R : 1][WIDE ? D : 1];
        bool valid[R];
        bool all_safe = true;
        load_rows<D, R, WIDE>(a, base, lane, k, ku, valid, AUTO ? &all_safe : nullptr);
        if (AUTO && !all_safe) load_rows_reduced<D, R>(a, base, lane, k);
        double kd[R][X > 0 ? X : 1];
#pragma unroll
        for (int q = 0; q < R; ++q)
#pragma unroll
            for (int j = 0; j < X; ++j) kd[q][j] = (double)k[q][j];
        {  // warm L2 with the next tile's rows while this one is hashed
            const int64_t nb = (tile + gridDim.x) * TILE + (int64_t)warp * 32 * R;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t i = nb + q * 32 + lane;
                if (i < a.n) prefetch_l2(a.elems + i * D);
            }
        }
        int hits[R];
        uint32_t bacc[R];
        auto run = [&](auto wide_tag) {
        constexpr bool WT = decltype(wide_tag)::value;
        int nbits = 0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            hits[q] = 0;
            bacc[q] = 0;
        }

        for (int c = 0; c < nchunks; ++c) {
            const int64_t qq = resident ? 0 : qc;
            mbar_wait(&bars[qq & 1], (uint32_t)((qq >> 1) & 1));
            const int l0 = c * a.Lc;
            const int lend = min(a.L, l0 + a.Lc);
            const uint32_t bbase = (qq & 1) ? slot1 : slot0;
            for (int l = l0; l < lend; ++l) {
                int32_t zr[D];
#pragma unroll
                for (int j = X; j < D; ++j) zr[j] = zc[l * D + j];
                double zdr[X > 0 ? X : 1];
#pragma unroll
                for (int j = 0; j < X; ++j) zdr[j] = zd[l * X + j];
                const uint32_t lb = bbase + (uint32_t)(l - l0) * slot_bytes;
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    uint32_t r;
                    if (!WIDE && WT) {  // AUTO tile with wide rows: exact signed 64-bit
                        int64_t acc = a.auto_bias;
#pragma unroll
                        for (int j = 0; j < D; ++j) acc += (int64_t)k[q][j] * (int64_t)zr[j];
                        r = (uint32_t)mod_u64((uint64_t)acc, (uint64_t)a.M, invM);
                    } else if (!WIDE) {
                        uint32_t u = a.offset;
                        if (X > 0) {
                            double acc = dmagic;
#pragma unroll
                            for (int j = 0; j < X; ++j) acc = __fma_rn(kd[q][j], zdr[j], acc);
                            u = (uint32_t)__double2loint(acc);
                        }
#pragma unroll
                        for (int j = X; j < D; ++j) u += (uint32_t)k[q][j] * (uint32_t)zr[j];
                        r = mod_u32(u, M32, negM, a.magic);
                    } else {
                        uint64_t acc = 0;
#pragma unroll
                        for (int j = 0; j < D; ++j)
                            acc += (uint64_t)ku[WIDE ? q : 0][WIDE ? j : 0] * (uint32_t)zr[j];
                        r = (uint32_t)mod_u64(acc, (uint64_t)a.M, invM);
                    }
                    const uint32_t w = SLOT ? word_slot(lb, r) : word_bit(lb, r);
                    bacc[q] = shift_in_bit(bacc[q], w, r);
                }
                if (++nbits == 32) {
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        hits[q] += __popc(bacc[q]);
                        bacc[q] = 0;
                    }
                    nbits = 0;
                }
            }
            if (!resident) {
                __syncthreads();  // every warp is done with this buffer
                if (threadIdx.x == 0 && qc + 2 < total_q) issue(qc + 2);
                ++qc;
            }
        }
        };
        if (AUTO && !all_safe) run(std::true_type{});
        else run(std::false_type{});
#pragma unroll
        for (int q = 0; q < R; ++q) hits[q] += __popc(bacc[q]);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int64_t i = base + q * 32 + lane;
            const unsigned det = __ballot_sync(0xffffffffu, valid[q] && hits[q] >= a.min_hits);
            if (valid[q] && a.hits64) a.hits64[(int64_t)g * a.n + i] = hits[q];
            if (lane == 0 && (base + q * 32) < a.n)
                a.detmask[(int64_t)g * a.nwords + ((base + q * 32) >> 5)] = det;
        }
    }
}

// Generic fallback: any d (runtime), one row per thread, exact 64-bit.
__global__ void __launch_bounds__(kHashThreads) hash_rows_generic(HashArgs a) {
    extern __shared__ uint32_t smem_u32[];
    const int g = blockIdx.y;
    uint32_t* bm = smem_u32;
    const int nchunks = (a.L + a.Lc - 1) / a.Lc;
    if (nchunks == 1) load_bits(bm, a, g, 0, a.L);
    __syncthreads();
    const int64_t ntiles = (a.n + kHashThreads - 1) / kHashThreads;
    const int lane = threadIdx.x & 31;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t i = tile * kHashThreads + threadIdx.x;
        const bool valid = i < a.n;
        int hits = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int l0 = c * a.Lc;
            const int lend = min(a.L, l0 + a.Lc);
            if (nchunks > 1) {
                __syncthreads();
                load_bits(bm, a, g, l0, lend - l0);
                __syncthreads();
            }
            if (!valid) continue;
            for (int l = l0; l < lend; ++l) {
                const int64_t* z = a.zmat + ((int64_t)g * a.L + l) * a.d;
                unsigned __int128 acc = 0;
                for (int j = 0; j < a.d; ++j) {
                    int64_t e = a.elems[i * a.d + j] % a.M;
                    if (e < 0) e += a.M;
                    int64_t zz = z[j] % a.M;
                    if (zz < 0) zz += a.M;
                    acc += (unsigned __int128)((uint64_t)e * (uint64_t)zz);
                }
                const uint32_t r = (uint32_t)(acc % (unsigned __int128)a.M);
                const uint32_t w = bm[(int64_t)(l - l0) * a.W + (r >> 5)];
                hits += (w >> (r & 31)) & 1u;
            }
        }
        const unsigned det = __ballot_sync(0xffffffffu, valid && hits >= a.min_hits);
        if (valid && a.hits64) a.hits64[(int64_t)g * a.n + i] = hits;
        if (lane == 0 && (tile * kHashThreads + (threadIdx.x & ~31)) < a.n)
            a.detmask[(int64_t)g * a.nwords + ((tile * kHashThreads + (threadIdx.x & ~31)) >> 5)] =
                det;
    }
}

// ---------------------------------------------------------------------------

__global__ void nonzero_bitmap_kernel(const double2* __restrict__ ghat, int64_t rows, int L,
                                      int64_t M, int64_t W, const double* __restrict__ theta,
                                      uint32_t* __restrict__ bits) {
    const int64_t total = rows * W;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / W, w = e % W;
        const double th = theta[row / L];
        uint32_t word = 0;
        const int64_t h0 = w * 32;
        const double2* src = ghat + row * M;
#pragma unroll 4
        for (int b = 0; b < 32; ++b) {
            const int64_t h = h0 + b;
            if (h < M) {
                const double2 v = src[h];
                word |= (uint32_t)nonzero_test(v.x, v.y, th) << b;
            }
        }
        bits[e] = word;
    }
}

// ---------------------------------------------------------------------------
// compaction of a per-row bitmask into ascending indices
// ---------------------------------------------------------------------------

static constexpr int kCompactWordsPerBlock = 512;  // 16k rows per block
static constexpr int kCompactThreads = 256;
static constexpr int64_t kCompactSingleWords = 8192;  // one 1024-thread CTA per group

__global__ void compact_count(const uint32_t* __restrict__ mask, int64_t nwords,
                              int64_t nblk, int64_t* __restrict__ blocksum) {
    const int g = blockIdx.y;
    const int64_t w0 = blockIdx.x * (int64_t)kCompactWordsPerBlock;
    int64_t s = 0;
    for (int64_t w = w0 + threadIdx.x; w < min(nwords, w0 + kCompactWordsPerBlock);
         w += blockDim.x)
        s += __popc(mask[(int64_t)g * nwords + w]);
    __shared__ int64_t red[kCompactThreads];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) blocksum[(int64_t)g * nblk + blockIdx.x] = red[0];
}

// Exclusive scan of a group's per-block counts, one CTA of kCompactScanThreads
// per group: chunks of blockDim entries, warp shuffles + one shared pass each.
static constexpr int kCompactScanThreads = 1024;

__global__ void __launch_bounds__(kCompactScanThreads)
    compact_scan(int64_t* blocksum, int64_t nblk, int64_t* counts, int64_t cap,
                 int64_t* totals) {
    const int g = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int64_t wsum[kCompactScanThreads / 32];
    __shared__ int64_t carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    int64_t* bs = blocksum + (int64_t)g * nblk;
    for (int64_t c0 = 0; c0 < nblk; c0 += blockDim.x) {
        const int64_t b = c0 + threadIdx.x;
        const int64_t v = b < nblk ? bs[b] : 0;
        int64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int64_t x = lane < (int)(blockDim.x / 32) ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t t = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += t;
            }
            if (lane < (int)(blockDim.x / 32)) wsum[lane] = x;  // inclusive warp prefix
        }
        __syncthreads();
        const int64_t base = carry_s + (warp ? wsum[warp - 1] : 0);
        if (b < nblk) bs[b] = base + incl - v;
        __syncthreads();
        if (threadIdx.x == 0) carry_s += wsum[blockDim.x / 32 - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        counts[g] = min(carry_s, cap);
        if (totals) totals[g] = carry_s;
    }
}

// SINGLE: one CTA per group walks all words with a running carry and writes
// counts[g] itself -- one launch instead of count/scan/write for the small
// masks of the sfft stages (nwords <= kCompactSingleWords).
template <bool SINGLE, int NT = kCompactThreads>
__global__ void __launch_bounds__(NT)
    compact_write(const uint32_t* __restrict__ mask, int64_t nwords, int64_t n, int64_t nblk,
                  const int64_t* __restrict__ blocksum, int64_t* __restrict__ idx,
                  int64_t* __restrict__ counts, int64_t cap, int64_t* __restrict__ totals) {
    const int g = blockIdx.y;
    const int64_t w0 = SINGLE ? 0 : blockIdx.x * (int64_t)kCompactWordsPerBlock;
    const int64_t wend = SINGLE ? nwords : min(nwords, w0 + kCompactWordsPerBlock);
    __shared__ int64_t warp_tot[NT / 32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = SINGLE ? 0 : blocksum[(int64_t)g * nblk + blockIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t c0 = w0; c0 < wend; c0 += blockDim.x) {
        const int64_t w = c0 + threadIdx.x;
        const uint32_t bitsw = w < wend ? mask[(int64_t)g * nwords + w] : 0u;
        int cnt = __popc(bitsw);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        int64_t before = carry;
        for (int k = 0; k < warp; ++k) before += warp_tot[k];
        const int64_t pos = before + incl - cnt;
        // expand the warp's 32 words cooperatively: for each word, lane j
        // writes row 32 w + j when bit j is set -- one coalesced store per
        // word instead of a lane writing its own word's rows one by one
        // (dense masks: every candidate detected); set bits are rows < n
        const unsigned below = (1u << lane) - 1u;
        unsigned any = __ballot_sync(0xffffffffu, bitsw != 0u);
        while (any) {
            const int src = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t wb = __shfl_sync(0xffffffffu, bitsw, src);
            const int64_t p0 = __shfl_sync(0xffffffffu, pos, src);
            const int64_t ws = __shfl_sync(0xffffffffu, w, src);
            if ((wb >> lane) & 1u) {
                const int64_t q = p0 + __popc(wb & below);
                const int64_t row = ws * 32 + lane;
                if (row < n && q < cap) idx[(int64_t)g * cap + q] = row;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t t = 0;
            for (int k = 0; k < NT / 32; ++k) t += warp_tot[k];
            carry += t;
        }
        __syncthreads();
    }
    if (SINGLE && threadIdx.x == 0) {
        counts[g] = min(carry, cap);
        if (totals) totals[g] = carry;
    }
}

// ---------------------------------------------------------------------------
// medians (one warp per detected row, L <= 128)
// ---------------------------------------------------------------------------

__device__ __forceinline__ int64_t residue_exact(const int64_t* row, const int64_t* z, int d,
                                                 int64_t M) {
    // sum_j (row_j mod M)(z_j mod M) < d (M-1)^2 < 2^62 (the caller's bound,
    // detect.py:128-129), so one 64-bit accumulation and a final mod suffice
    // (the 64-bit divisions are skipped for entries already in (-M, M), the
    // common case, and the final reduction uses the FP64 quotient estimate)
    uint64_t acc = 0;
    for (int j = 0; j < d; ++j) {
        acc += (uint64_t)reduce_mod(row[j], M) * (uint64_t)reduce_mod(z[j], M);
    }
    return (int64_t)mod_u64(acc, (uint64_t)M, 1.0 / (double)M);
}

// Componentwise median of the L complex values a warp holds (lane + 32 s).
// Fast path: ranks lt = #{v_j < v_i} for both components in one pass over the
// warp's values in shared memory (broadcast double2 reads); the stable-sort
// position floor(L/2) is held by the lowest-index element with lt ==
// floor(L/2) -- unless that position falls strictly inside a run of equal
// values, which no lane can then claim; that component then falls back to
// full stable ranks #{v_j < v_i} + #{j < i: v_j == v_i} (bit-identical to the
// reference's insertion-sort median, _core.pyx:151-161, including the order
// of +0.0 and -0.0).
template <int S>
__device__ __forceinline__ double median_claim(const double (&v)[S], const int (&lt)[S], int L,
                                               int lane, bool& found) {
    const int target = L >> 1;
    double val = 0.0;
    found = false;
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {  // lowest claiming index wins
        const int i = lane + 32 * s;
        const unsigned b = __ballot_sync(0xffffffffu, i < L && lt[s] == target);
        if (b) {
            val = __shfl_sync(0xffffffffu, v[s], __ffs(b) - 1);
            found = true;
        }
    }
    return val;
}

template <int S>
__device__ __forceinline__ double median_stable(const double (&v)[S], const double2* sv, bool im,
                                                int L, int lane) {
    const int target = L >> 1;
    int rk[S];
#pragma unroll
    for (int s = 0; s < S; ++s) rk[s] = 0;
    for (int j = 0; j < L; ++j) {
        const double o = im ? sv[j].y : sv[j].x;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = lane + 32 * s;
            rk[s] += (o < v[s]) || (o == v[s] && j < i);
        }
    }
    double val = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int i = lane + 32 * s;
        const unsigned b = __ballot_sync(0xffffffffu, i < L && rk[s] == target);
        if (b) val = __shfl_sync(0xffffffffu, v[s], __ffs(b) - 1);
    }
    return val;
}

template <int S>
__device__ __forceinline__ double2 warp_median2_exact(const double (&re)[S], const double (&im)[S],
                                                      const double2* sv, int L, int lane) {
    int lr[S], li[S];
#pragma unroll
    for (int s = 0; s < S; ++s) lr[s] = li[s] = 0;
    for (int j = 0; j < L; ++j) {
        const double2 o = sv[j];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            lr[s] += o.x < re[s];
            li[s] += o.y < im[s];
        }
    }
    bool fr, fi;
    double mr = median_claim<S>(re, lr, L, lane, fr);
    double mi = median_claim<S>(im, li, L, lane, fi);
    if (!fr) mr = median_stable<S>(re, sv, false, L, lane);
    if (!fi) mi = median_stable<S>(im, sv, true, L, lane);
    return make_double2(mr, mi);
}

// Top 31 bits of an order-preserving integer image of a double: monotone,
// not strictly, in the double order (-0.0 sorts below +0.0 here; the exact
// check below decides).
__device__ __forceinline__ int32_t order_key31(double x) {
    const long long b = __double_as_longlong(x);
    return (int32_t)((b ^ ((b >> 63) & 0x7FFFFFFFFFFFFFFFLL)) >> 33);
}

// acc + (a < b) for |a|, |b| < 2^30: the sign bit of a - b, added with one
// LEA.HI (the compiler's own lowering is a compare, a select and moves)
__device__ __forceinline__ unsigned add_sign_bit(unsigned acc, int a, int b) {
    unsigned d, r;
    asm("sub.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    asm("{\n\t.reg .u32 t;\n\tshr.u32 t, %1, 31;\n\tadd.u32 %0, %2, t;\n\t}"
        : "=r"(r) : "r"(d), "r"(acc));
    return r;
}

// The lowest-index value whose approximate rank is floor(L/2), accepted only
// when its exact rank is floor(L/2) and no other value compares equal to it:
// then it is the stable-sort median whatever the approximate ranks were.
template <int S>
__device__ __forceinline__ bool median_verified(const double (&v)[S], const unsigned (&lt)[S],
                                                int L, int lane, double& out) {
    const int target = L >> 1;
    bool found = false;
    double p = 0.0;
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {
        const unsigned b = __ballot_sync(0xffffffffu, lane + 32 * s < L && (int)lt[s] == target);
        if (b) {
            p = __shfl_sync(0xffffffffu, v[s], __ffs(b) - 1);
            found = true;
        }
    }
    if (!found) return false;
    int nlt = 0, neq = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const bool ok = lane + 32 * s < L;
        nlt += __popc(__ballot_sync(0xffffffffu, ok && v[s] < p));
        neq += __popc(__ballot_sync(0xffffffffu, ok && v[s] == p));
    }
    out = p;
    return nlt == target && neq == 1;
}

// Componentwise median: ranks from 31-bit integer keys (two integer ops per
// comparison instead of a DSETP and a select), each candidate verified
// exactly; a component that fails verification (near-ties in the top bits,
// equal values, signed zeros) takes the exact path.
template <int S>
__device__ __forceinline__ double2 warp_median2(const double (&re)[S], const double (&im)[S],
                                                const double2* sv, const int2* sk, int L,
                                                int lane) {
    int kr[S], ki[S];
    unsigned lr[S], li[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        kr[s] = order_key31(re[s]);
        ki[s] = order_key31(im[s]);
        lr[s] = li[s] = 0u;
    }
#pragma unroll 4
    for (int j = 0; j < L; ++j) {
        const int2 o = sk[j];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            lr[s] = add_sign_bit(lr[s], o.x, kr[s]);
            li[s] = add_sign_bit(li[s], o.y, ki[s]);
        }
    }
    double mr, mi;
    const bool okr = median_verified<S>(re, lr, L, lane, mr);
    const bool oki = median_verified<S>(im, li, L, lane, mi);
    if (okr && oki) return make_double2(mr, mi);
    const double2 e = warp_median2_exact<S>(re, im, sv, L, lane);
    return make_double2(okr ? mr : e.x, oki ? mi : e.y);
}

// Residue tables of a Cartesian candidate set J = prefix x vals (the
// dimension-incremental pairing, dimincr.py:155-175): row i = i1 * n2 + i2
// has residue (P[l][i1] + V[l][i2]) mod M on lattice l.
struct PairTables {
    const int32_t* P;  // [G*L][n1]
    const int32_t* V;  // [G*L][n2]
    int64_t n1, n2;
};

// SMALL (pair tables): every table / spectrum offset < 2^31, so the per-row
// index arithmetic is 32-bit
template <int S, bool PAIRS = false, bool SMALL = false>
__global__ void __launch_bounds__(256) medians_kernel(const int64_t* __restrict__ elems, int d,
                                                      const int64_t* __restrict__ zmat, int G,
                                                      int L, int64_t M,
                                                      const double2* __restrict__ ghat,
                                                      const int64_t* __restrict__ idx,
                                                      const int64_t* __restrict__ counts,
                                                      int64_t cap, double2* __restrict__ coeffs,
                                                      PairTables pt = PairTables{}) {
    __shared__ double2 sv[8][32 * S];
    __shared__ int2 sk[8][32 * S];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // one flat work list over the groups' detected rows (g, k), so small
    // groups do not serialise one latency-bound round per group
    __shared__ int64_t cnt_s[32];
    const bool cnt_in_smem = G <= 32;
    if (cnt_in_smem && threadIdx.x < G) cnt_s[threadIdx.x] = counts[threadIdx.x];
    __syncthreads();
    const int64_t* cnt = cnt_in_smem ? cnt_s : counts;
    int64_t total = 0;
    for (int g = 0; g < G; ++g) total += cnt[g];
    for (int64_t w = gwarp; w < total; w += nwarps) {
        int g = 0;
        int64_t k = w;
        while (k >= cnt[g]) k -= cnt[g++];
        const int64_t row = idx[(int64_t)g * cap + k];
        int64_t i1 = 0, i2 = 0;
        if (PAIRS) {  // row = i1 * n2 + i2 (< 2^32: 32-bit division)
            const uint32_t q = (uint32_t)row / (uint32_t)pt.n2;
            i1 = q;
            i2 = row - (int64_t)q * pt.n2;
        }
        double re[S], im[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int l = lane + 32 * s;
            re[s] = 0.0;
            im[s] = 0.0;
            if (l < L) {
                int64_t r;
                double2 v;
                if (PAIRS && SMALL) {
                    const uint32_t gl = (uint32_t)(g * L + l);
                    uint32_t r32 = (uint32_t)pt.P[gl * (uint32_t)pt.n1 + (uint32_t)i1] +
                                   (uint32_t)pt.V[gl * (uint32_t)pt.n2 + (uint32_t)i2];
                    if (r32 >= (uint32_t)M) r32 -= (uint32_t)M;
                    v = ghat[gl * (uint32_t)M + r32];
                } else {
                    if (PAIRS) {
                        const int64_t gl = (int64_t)g * L + l;
                        r = (int64_t)pt.P[gl * pt.n1 + i1] + pt.V[gl * pt.n2 + i2];
                        if (r >= M) r -= M;
                    } else {
                        r = residue_exact(elems + row * d, zmat + ((int64_t)g * L + l) * d, d,
                                          M);
                    }
                    v = ghat[((int64_t)g * L + l) * M + r];
                }
                re[s] = v.x;
                im[s] = v.y;
            }
            sv[wib][l] = make_double2(re[s], im[s]);
            sk[wib][l] = make_int2(order_key31(re[s]), order_key31(im[s]));
        }
        __syncwarp();
        const double2 m = warp_median2<S>(re, im, sv[wib], sk[wib], L, lane);
        if (lane == 0) coeffs[(int64_t)g * cap + k] = m;
        __syncwarp();  // the next row's stores wait for these reads
    }
}

// Two rows per warp for 32 < L <= 48 on pair tables (noisy stages detect
// every candidate): each half-warp holds one row's L values in 3 slots of 16
// lanes, so a broadcast comparison serves 2 rows x 48 slots instead of 1 row
// x 64 slots.  Ranks on the 31-bit order keys; each half's candidate median
// is verified exactly (exact rank floor(L/2), no other equal value); if either
// half fails, both rows are redone by the one-row-per-warp path.
__global__ void __launch_bounds__(256) medians2_pairs_kernel(
    int G, int L, int64_t M, const double2* __restrict__ ghat, const int64_t* __restrict__ idx,
    const int64_t* __restrict__ counts, int64_t cap, double2* __restrict__ coeffs,
    PairTables pt) {
    constexpr int S = 3;
    __shared__ int2 sk[8][2][48];
    __shared__ double2 fv[8][64];
    __shared__ int2 fk[8][64];
    __shared__ int64_t cnt_s[32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int half = lane >> 4, hl = lane & 15;
    const unsigned hmask = half ? 0xFFFF0000u : 0x0000FFFFu;
    const bool cnt_in_smem = G <= 32;
    if (cnt_in_smem && threadIdx.x < G) cnt_s[threadIdx.x] = counts[threadIdx.x];
    __syncthreads();
    const int64_t* cnt = cnt_in_smem ? cnt_s : counts;
    int64_t total = 0;
    for (int g = 0; g < G; ++g) total += cnt[g];
    const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int target = L >> 1;
    auto locate = [&](int64_t w, int& g, int64_t& k) {
        g = 0;
        k = w;
        while (k >= cnt[g]) k -= cnt[g++];
    };
    auto value = [&](int g, int64_t row, int l) -> double2 {
        const uint32_t q = (uint32_t)row / (uint32_t)pt.n2;
        const uint32_t i2 = (uint32_t)(row - (int64_t)q * pt.n2);
        const uint32_t gl = (uint32_t)(g * L + l);
        uint32_t r32 = (uint32_t)pt.P[gl * (uint32_t)pt.n1 + q] +
                       (uint32_t)pt.V[gl * (uint32_t)pt.n2 + i2];
        if (r32 >= (uint32_t)M) r32 -= (uint32_t)M;
        return ghat[gl * (uint32_t)M + r32];
    };
    for (int64_t w2 = gwarp * 2; w2 < total; w2 += nwarps * 2) {
        const int64_t wmine = w2 + half;
        const bool live = wmine < total;
        int g = 0;
        int64_t k = 0, row = 0;
        if (live) {
            locate(wmine, g, k);
            row = idx[(int64_t)g * cap + k];
        }
        double re[S], im[S];
        int kr[S], ki[S];
        unsigned lr[S], li[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int l = hl + 16 * s;
            double2 v = make_double2(0.0, 0.0);
            if (live && l < L) v = value(g, row, l);
            re[s] = v.x;
            im[s] = v.y;
            kr[s] = order_key31(v.x);
            ki[s] = order_key31(v.y);
            lr[s] = li[s] = 0u;
            if (l < 48) sk[wib][half][l] = make_int2(kr[s], ki[s]);
        }
        __syncwarp();
#pragma unroll 4
        for (int j = 0; j < L; ++j) {
            const int2 o = sk[wib][half][j];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                lr[s] = add_sign_bit(lr[s], o.x, kr[s]);
                li[s] = add_sign_bit(li[s], o.y, ki[s]);
            }
        }
        // per half: the lowest-index claimant, then its exact rank
        double mr = 0.0, mi = 0.0;
        bool okr = false, oki = false;
#pragma unroll
        for (int comp = 0; comp < 2; ++comp) {
            const double(&v)[S] = comp ? im : re;
            const unsigned(&lt)[S] = comp ? li : lr;
            bool found = false;
            double p = 0.0;
#pragma unroll
            for (int s = S - 1; s >= 0; --s) {
                const unsigned b =
                    __ballot_sync(0xffffffffu, hl + 16 * s < L && (int)lt[s] == target) & hmask;
                const int src = b ? __ffs(b) - 1 : lane;
                const double cand = __shfl_sync(0xffffffffu, v[s], src);
                if (b) {
                    p = cand;
                    found = true;
                }
            }
            int nlt = 0, neq = 0;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool okl = hl + 16 * s < L;
                nlt += __popc(__ballot_sync(0xffffffffu, okl && v[s] < p) & hmask);
                neq += __popc(__ballot_sync(0xffffffffu, okl && v[s] == p) & hmask);
            }
            const bool ok = found && nlt == target && neq == 1;
            if (comp) {
                mi = p;
                oki = ok;
            } else {
                mr = p;
                okr = ok;
            }
        }
        const bool good = __all_sync(0xffffffffu, !live || (okr && oki));
        if (good) {
            if (live && hl == 0) coeffs[(int64_t)g * cap + k] = make_double2(mr, mi);
            __syncwarp();
            continue;
        }
        // rare: both rows again, one at a time, on the full warp
        for (int h = 0; h < 2; ++h) {
            const int64_t wr = w2 + h;
            if (wr >= total) break;
            int g2;
            int64_t k2;
            locate(wr, g2, k2);
            const int64_t row2 = idx[(int64_t)g2 * cap + k2];
            double r2[2], i2v[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int l = lane + 32 * s;
                double2 v = make_double2(0.0, 0.0);
                if (l < L) v = value(g2, row2, l);
                r2[s] = v.x;
                i2v[s] = v.y;
                fv[wib][l] = v;
                fk[wib][l] = make_int2(order_key31(v.x), order_key31(v.y));
            }
            __syncwarp();
            const double2 m = warp_median2<2>(r2, i2v, fv[wib], fk[wib], L, lane);
            if (lane == 0) coeffs[(int64_t)g2 * cap + k2] = m;
            __syncwarp();
        }
    }
}

// Thread-pair per detected row on pair tables, L odd <= 63: lane pair (2i,
// 2i + 1) takes the real and the imaginary part of work item i, gathers its
// L values in lattice order into registers and selects the median with the
// pruned network of median_nets.cuh (DSETP/FSEL comparators, no ranks, no
// shared memory).  Min/max networks agree bit for bit with the reference's
// stable insertion sort (_core.pyx:151-161) except when -0.0 and +0.0 are
// both present; a component holding a zero takes that insertion sort
// itself, in lattice order.
template <int L>
__global__ void __launch_bounds__(256) medians_net_pairs_kernel(
    int G, int64_t M, const double2* __restrict__ ghat, const int64_t* __restrict__ idx,
    const int64_t* __restrict__ counts, int64_t cap, double2* __restrict__ coeffs,
    PairTables pt) {
    __shared__ int64_t cnt_s[32];
    const bool cnt_in_smem = G <= 32;
    if (cnt_in_smem && threadIdx.x < G) cnt_s[threadIdx.x] = counts[threadIdx.x];
    __syncthreads();
    const int64_t* cnt = cnt_in_smem ? cnt_s : counts;
    int64_t total = 0;
    for (int g = 0; g < G; ++g) total += cnt[g];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w2 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w2 < 2 * total;
         w2 += stride) {
        const int64_t w = w2 >> 1;
        const int comp = (int)(w2 & 1);
        int g = 0;
        int64_t k = w;
        while (k >= cnt[g]) k -= cnt[g++];
        const int64_t row = idx[(int64_t)g * cap + k];
        const uint32_t q = (uint32_t)row / (uint32_t)pt.n2;
        const uint32_t i2 = (uint32_t)(row - (int64_t)q * pt.n2);
        double a[L];
        bool zero = false;
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const uint32_t gl = (uint32_t)(g * L + l);
            uint32_t r32 = (uint32_t)__ldg(pt.P + gl * (uint32_t)pt.n1 + q) +
                           (uint32_t)__ldg(pt.V + gl * (uint32_t)pt.n2 + i2);
            if (r32 >= (uint32_t)M) r32 -= (uint32_t)M;
            a[l] = __ldg(reinterpret_cast<const double*>(ghat + gl * (uint32_t)M + r32) + comp);
            zero |= a[l] == 0.0;
        }
        double m;
        if (!zero) {
            m = median_net<L>(a);
        } else {  // signed zeros: the reference's insertion sort, in lattice order
            double t[L];
#pragma unroll
            for (int l = 0; l < L; ++l) t[l] = a[l];
            for (int i = 1; i < L; ++i) {
                const double v = t[i];
                int j = i;
                while (j > 0 && t[j - 1] > v) {
                    t[j] = t[j - 1];
                    --j;
                }
                t[j] = v;
            }
            m = t[L >> 1];
        }
        reinterpret_cast<double*>(coeffs + (int64_t)g * cap + k)[comp] = m;
    }
}

__global__ void lattice_values_kernel(const int64_t* __restrict__ elems, int d,
                                      const int64_t* __restrict__ zmat, int L, int64_t M,
                                      const double2* __restrict__ ghat,
                                      const int64_t* __restrict__ rows, int64_t nrows,
                                      double2* __restrict__ out) {
    const int64_t total = nrows * L;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / L;
        const int l = (int)(e % L);
        const int64_t row = rows ? rows[k] : k;
        const int64_t r = residue_exact(elems + row * d, zmat + (int64_t)l * d, d, M);
        out[e] = ghat[(int64_t)l * M + r];
    }
}

// Distinct lattice sizes (reference detect.py:134-145, numpy path): per row of
// vals (n, L) the hits count #{l: |v_l| > theta} with |.| = hypot (np.abs) and,
// for rows with hits >= thr, np.median of the real and imaginary parts: the
// middle element (odd L) or the mean of the two middle elements (even L).
// One warp per row; values staged in shared memory (L <= 128) or read from
// the row itself in global memory (any L: the reference's numpy fallback,
// _kernels/__init__.py:62, serves every L > _MAX_COMPILED_L = 128), stable
// ranks.
__global__ void __launch_bounds__(256)
    rows_hits_medians_kernel(const double2* __restrict__ vals, int64_t n, int L, double theta,
                             double thr, int want_medians, int64_t* __restrict__ hits,
                             double2* __restrict__ med) {
    __shared__ double2 sv[8][128];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool staged = L <= 128;
    for (int64_t i = gw; i < n; i += nw) {
        int h = 0;
        for (int l = lane; l < L; l += 32) {
            const double2 v = vals[i * L + l];
            if (staged) sv[wib][l] = v;
            h += hypot(v.x, v.y) > theta;
        }
        for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
        __syncwarp();
        const double2* row = staged ? sv[wib] : vals + i * L;
        double2 m = make_double2(0.0, 0.0);
        if (want_medians && (double)h >= thr) {
            const int lo = (L - 1) / 2, hi = L / 2;
            double lo_re = 0.0, hi_re = 0.0, lo_im = 0.0, hi_im = 0.0;
            for (int l = lane; l < L; l += 32) {
                const double2 v = row[l];
                int rr = 0, ri = 0;
                for (int j = 0; j < L; ++j) {
                    const double2 o = row[j];
                    rr += (o.x < v.x) || (o.x == v.x && j < l);
                    ri += (o.y < v.y) || (o.y == v.y && j < l);
                }
                if (rr == lo) lo_re = v.x;
                if (rr == hi) hi_re = v.x;
                if (ri == lo) lo_im = v.y;
                if (ri == hi) hi_im = v.y;
            }
            for (int o = 16; o > 0; o >>= 1) {  // exactly one lane holds each
                lo_re += __shfl_xor_sync(0xffffffffu, lo_re, o);
                hi_re += __shfl_xor_sync(0xffffffffu, hi_re, o);
                lo_im += __shfl_xor_sync(0xffffffffu, lo_im, o);
                hi_im += __shfl_xor_sync(0xffffffffu, hi_im, o);
            }
            m = (L & 1) ? make_double2(lo_re, lo_im)
                        : make_double2((lo_re + hi_re) / 2.0, (lo_im + hi_im) / 2.0);
        }
        if (lane == 0) {
            hits[i] = h;
            if (want_medians) med[i] = m;
        }
        __syncwarp();
    }
}

// P[gl][i1] = prefix[i1] . z_gl[0:t] mod M;  V[gl][i2] = vals[i2] * z_gl[t] mod M
__global__ void pair_residues_kernel(const int64_t* __restrict__ prefix, int64_t n1, int t,
                                     const int64_t* __restrict__ vals, int64_t n2,
                                     const int64_t* __restrict__ zmat, int64_t GL, int64_t M,
                                     int32_t* __restrict__ P, int32_t* __restrict__ V) {
    const int td = t + 1;
    const int64_t np = GL * n1, total = np + GL * n2;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < np) {
            const int64_t gl = e / n1, i1 = e % n1;
            P[e] = (int32_t)residue_exact(prefix + i1 * t, zmat + gl * td, t, M);
        } else {
            const int64_t f = e - np, gl = f / n2, i2 = f % n2;
            const uint64_t a = (uint64_t)reduce_mod(vals[i2], M);
            const uint64_t b = (uint64_t)reduce_mod(zmat[gl * td + t], M);
            V[f] = (int32_t)mod_u64(a * b, (uint64_t)M, 1.0 / (double)M);
        }
    }
}

// Hashing of a Cartesian J from its residue tables.  The group's bitmaps
// arrive in shared memory by one bulk copy (TMA engine, mbarrier), the V table
// by an unrolled loop; per tile of kPairRows * 256 rows the P entries of the
// tile's i1 range are staged too.  Each thread owns kPairRows rows
// (independent chains); per (row, lattice): two shared loads (P broadcast, V
// contiguous), an add, an unsigned-min reduction and the bit probe -- no dot
// product, no multiply-high.  (Probing the bitmaps from L1 instead: ~16
// wavefronts per random warp probe vs ~4 in shared memory, measured slower.)
static constexpr int kPairRows = 8;
static constexpr int kPairThreads = 256;
static constexpr int kPairTile = kPairRows * kPairThreads;

__global__ void __launch_bounds__(kPairThreads)
    hash_pairs_kernel(const int32_t* __restrict__ P, const int32_t* __restrict__ V, int64_t n1,
                      int64_t n2, int L, int64_t M, const uint32_t* __restrict__ bits, int64_t W,
                      int64_t min_hits, int64_t* __restrict__ hits64,
                      uint32_t* __restrict__ detmask, int span) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint64_t bar;
    const int g = blockIdx.y;
    const int64_t n = n1 * n2, nwords = (n + 31) / 32;
    uint32_t* bm = sm;                                     // L * W words
    uint32_t* vs = sm + (int64_t)L * W;                    // L * n2
    uint32_t* ps = vs + (((int64_t)L * n2 + 3) & ~int64_t(3));  // L * span
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)((int64_t)L * W * 4);
        mbar_arrive_expect_tx(&bar, bytes);
        bulk_g2s(bm, bits + (int64_t)g * L * W, bytes, &bar);
    }
    const uint32_t* gV = (const uint32_t*)V + (int64_t)g * L * n2;
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < (int64_t)L * n2; i += blockDim.x) vs[i] = __ldg(gV + i);
    const uint32_t* gP = (const uint32_t*)P + (int64_t)g * L * n1;
    const uint32_t M32 = (uint32_t)M;
    const int64_t ntiles = (n + kPairTile - 1) / kPairTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bool waited = false;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t t0 = tile * kPairTile;
        const int64_t i1lo = t0 / n2;
        __syncthreads();  // previous tile done with ps
#pragma unroll 4
        for (int64_t e = threadIdx.x; e < (int64_t)L * span; e += blockDim.x) {
            const int l = (int)(e / span);
            const int64_t i1 = i1lo + e % span;
            ps[e] = i1 < n1 ? __ldg(gP + (int64_t)l * n1 + i1) : 0u;
        }
        if (!waited) {
            mbar_wait(&bar, 0);
            waited = true;
        }
        __syncthreads();
        int pi[kPairRows], vi[kPairRows], hits[kPairRows];
        bool valid[kPairRows];
#pragma unroll
        for (int q = 0; q < kPairRows; ++q) {
            const int64_t i = t0 + (int64_t)warp * 32 * kPairRows + q * 32 + lane;
            valid[q] = i < n;
            const int64_t ii = valid[q] ? i : t0;
            const int64_t i1 = ii / n2;
            pi[q] = (int)(i1 - i1lo);
            vi[q] = (int)(ii - i1 * n2);
            hits[q] = 0;
        }
        for (int l = 0; l < L; ++l) {
            const uint32_t* pl = ps + (int64_t)l * span;
            const uint32_t* vl = vs + (int64_t)l * n2;
            const uint32_t* bl = bm + (int64_t)l * W;
#pragma unroll
            for (int q = 0; q < kPairRows; ++q) {
                uint32_t r = pl[pi[q]] + vl[vi[q]];
                r = min(r, r - M32);  // r < 2M: one unsigned min reduces it
                hits[q] += (bl[r >> 5] >> (r & 31)) & 1u;
            }
        }
#pragma unroll
        for (int q = 0; q < kPairRows; ++q) {
            const int64_t i = t0 + (int64_t)warp * 32 * kPairRows + q * 32 + lane;
            const unsigned det = __ballot_sync(0xffffffffu, valid[q] && hits[q] >= min_hits);
            if (valid[q] && hits64) hits64[(int64_t)g * n + i] = hits[q];
            if (lane == 0 && i < n) detmask[(int64_t)g * nwords + (i >> 5)] = det;
        }
    }
    if (!waited) mbar_wait(&bar, 0);  // never leave a bulk copy in flight
}

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------

__global__ void sumsq_kernel(const double2* __restrict__ x, int64_t stride, int64_t M,
                             double* __restrict__ out) {
    const int64_t b = blockIdx.x;
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < M; j += blockDim.x) {
        const double2 v = x[b * stride + j];
        s = fma(v.x, v.x, fma(v.y, v.y, s));
    }
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b] = red[0];
}

// One warp per group: lane l owns rms of lattices l, l+32, ...; the median
// is found by stable ranking (L <= 256).
// One CTA per group: the L per-lattice RMS values in shared memory, each
// thread ranks its values against all L (stable rank: #{v_j < v_i} +
// #{j < i : v_j == v_i}), the holders of ranks (L-1)/2 and L/2 publish them.
__global__ void zero_threshold_kernel(const double* __restrict__ sumsq, int G, int L, int64_t M,
                                      double* __restrict__ theta) {
    pdl_wait();  // inside the fused chain: the partial sums of the previous kernel
    pdl_launch();
    extern __shared__ double zt_v[];
    __shared__ double mids[2];
    const int g = blockIdx.x;
    for (int l = threadIdx.x; l < L; l += blockDim.x)
        zt_v[l] = sqrt(sumsq[(int64_t)g * L + l] / (double)M);
    __syncthreads();
    const int lo = (L - 1) / 2, hi = L / 2;  // middle pair (equal when L is odd)
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const double vi = zt_v[i];
        int rank = 0;
        for (int j = 0; j < L; ++j) {
            const double o = zt_v[j];
            rank += (o < vi) || (o == vi && j < i);
        }
        if (rank == lo) mids[0] = vi;
        if (rank == hi) mids[1] = vi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double mid = (L % 2 == 1) ? mids[0] : 0.5 * (mids[0] + mids[1]);
        theta[g] = fmax(1e-12, 1e-10 * mid);
    }
}

__global__ void mark_kernel(const int64_t* __restrict__ idx, const int64_t* __restrict__ counts,
                            int G, int64_t cap, uint32_t* __restrict__ mask) {
    for (int g = 0; g < G; ++g) {
        const int64_t c = counts[g];
        for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < c;
             k += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i = idx[(int64_t)g * cap + k];
            atomicOr(mask + (i >> 5), 1u << (i & 31));
        }
    }
}

__global__ void gather_rows_kernel(const int64_t* __restrict__ src, int d,
                                   const int64_t* __restrict__ rows,
                                   const int64_t* __restrict__ count, int64_t* __restrict__ dst) {
    const int64_t total = count[0] * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / d;
        dst[e] = src[rows[k] * d + (e % d)];
    }
}

__global__ void pair_kernel(const int64_t* __restrict__ prev, int64_t n1, int t,
                            const int64_t* __restrict__ vals, int64_t n2,
                            int64_t* __restrict__ out) {
    const int64_t total = n1 * n2 * (t + 1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / (t + 1);
        const int c = (int)(e % (t + 1));
        const int64_t i = row / n2, j = row % n2;
        out[e] = c < t ? prev[i * t + c] : vals[j];
    }
}

__global__ void row_bounds_kernel(const int64_t* __restrict__ elems, int64_t n, int d,
                                  int64_t* __restrict__ out) {
    // blockDim is a multiple of d: each thread always sees the same coordinate
    const int per = blockDim.x / d;
    if (threadIdx.x >= per * d) return;
    const int coord = threadIdx.x % d;
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    const int64_t total = n * d;
    for (int64_t e = blockIdx.x * (int64_t)(per * d) + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * per * d) {
        const int64_t v = elems[e];
        lo = min(lo, v);
        hi = max(hi, v);
    }
    atomicMin((long long*)&out[2 * coord], (long long)lo);
    atomicMax((long long*)&out[2 * coord + 1], (long long)hi);
}

__global__ void init_bounds_kernel(int64_t* out, int d) {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        out[2 * j] = INT64_MAX;
        out[2 * j + 1] = INT64_MIN;
    }
}

static int grid_for(int64_t work, int threads) {
    int64_t g = ceil_div(work, threads);
    const int64_t cap = (int64_t)num_sms() * 16;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

// ---------------------------------------------------------------------------
// hash dispatch
// ---------------------------------------------------------------------------

// CTAs per group (grid.x): every CTA of a group strides over the same number
// of row tiles, so the launch runs in ceil(gx*G / slots) equal waves.  Pick
// the smallest gx >= ceil(slots/G) whose last wave is >= 95% full (e.g. G =
// 198 trial groups on 148 SMs: gx = 7, 9.4 waves, instead of gx = 1 and a
// one-third-full second wave).
static int hash_grid_x(int64_t ntiles, int64_t G, int64_t slots) {
    const int64_t lo = std::max<int64_t>(1, ceil_div(slots, G));
    int64_t best = lo;
    double best_eff = 0.0;
    for (int64_t gx = lo; gx <= lo * 16 && gx <= ntiles; ++gx) {
        const int64_t ctas = gx * G;
        const double eff = (double)ctas / (double)(slots * ceil_div(ctas, slots));
        if (eff > best_eff + 1e-9) {
            best = gx;
            best_eff = eff;
        }
        if (eff >= 0.95) break;
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, best));
}

template <int D, int R, bool WIDE, int NT, bool SLOT, int X, bool AUTO = false>
static int launch_hash_s(HashArgs& a, size_t smem, cudaStream_t st) {
    auto kern = hash_rows<D, R, WIDE, NT, SLOT, X, AUTO>;
    SFFTB_CUDA(smem_opt_in(kern, smem));
    int per_sm = 0;
    SFFTB_CUDA(occupancy(&per_sm, kern, NT, smem));
    per_sm = std::max(per_sm, 1);
    constexpr int TILE = (NT / 32) * 32 * R;
    const int64_t ntiles = ceil_div(a.n, TILE);
    const int gx = hash_grid_x(ntiles, a.G, (int64_t)num_sms() * per_sm);
    kern<<<dim3(gx, a.G), NT, smem, st>>>(a);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

template <int D, int R, bool WIDE, int NT = kHashThreads, int X = 0, bool AUTO = false>
static int launch_hash_t(HashArgs& a, size_t smem, cudaStream_t st) {
    const bool pow2 = (a.slot_words & (a.slot_words - 1)) == 0;
    return pow2 ? launch_hash_s<D, R, WIDE, NT, true, X, AUTO>(a, smem, st)
                : launch_hash_s<D, R, WIDE, NT, false, X, AUTO>(a, smem, st);
}

// 640 threads (20 warps) per SM with R rows per thread, R*D <= ~60 int32
// registers of candidate rows: measured on B200 (cfg4 shape, 2^26 rows):
// 512x8 4.57 ms, 768x4 4.05 ms, 640x6 4.00 ms, 256x16 4.87 ms.
template <int D, bool WIDE, bool AUTO = false>
static int launch_hash_d(HashArgs& a, size_t smem, cudaStream_t st) {
    constexpr int R = D <= 5 ? 12 : (D <= 7 ? 8 : (D <= 10 ? 6 : (D <= 15 ? 4 : 3)));
    constexpr int RW = R / 2 > 0 ? R / 2 : 1;  // the 64-bit path needs wider temporaries
    if constexpr (AUTO) {
        return launch_hash_t<D, R, false, 640, 0, true>(a, smem, st);
    }
    if constexpr (D == 10 && !WIDE) {
        // opt-in FP64/IMAD split (SFFTB_HASH_VARIANT=1|2); measured slower
        // than the all-IMAD default on B200 (profiles/r01/SUMMARY.md)
        if (a.xsplit > 0) {
            if (a.variant == 2) return launch_hash_t<D, 3, false, 640, 5>(a, smem, st);
            return launch_hash_t<D, 4, false, 640, 5>(a, smem, st);
        }
    }
    return launch_hash_t<D, (WIDE ? RW : R), WIDE, 640>(a, smem, st);
}

template <bool WIDE, bool AUTO = false>
static int hash_dispatch(int d, HashArgs& a, size_t smem, cudaStream_t st) {
    switch (d) {
#define SFFTB_HD(X) \
    case X: return launch_hash_d<X, WIDE, AUTO>(a, smem, st);
        SFFTB_HD(1) SFFTB_HD(2) SFFTB_HD(3) SFFTB_HD(4) SFFTB_HD(5) SFFTB_HD(6) SFFTB_HD(7)
        SFFTB_HD(8) SFFTB_HD(9) SFFTB_HD(10) SFFTB_HD(11) SFFTB_HD(12) SFFTB_HD(13)
        SFFTB_HD(14) SFFTB_HD(15) SFFTB_HD(16) SFFTB_HD(17) SFFTB_HD(18) SFFTB_HD(19)
        SFFTB_HD(20)
#undef SFFTB_HD
    }
    return -1;
}

}  // namespace sfftb

using namespace sfftb;

extern "C" int64_t sfftb_bitmap_words(int64_t M) {
    return ((M + 31) / 32 + 3) & ~int64_t(3);
}

extern "C" int sfftb_nonzero_bitmap(const double* ghat, int64_t G, int64_t L, int64_t M,
                                    const double* theta, uint32_t* bits, void* stream) {
    SFFTB_REQUIRE(G >= 0 && L >= 0 && M >= 1, "bitmap: bad sizes");
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    const int64_t rows = G * L;
    if (rows == 0) return SFFTB_OK;
    nonzero_bitmap_kernel<<<grid_for(rows * W, 256), 256, 0, (cudaStream_t)stream>>>(
        (const double2*)ghat, rows, (int)L, M, W, theta, bits);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_hash_hits(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat,
                               int64_t G, int64_t L, int64_t M, const uint32_t* bits,
                               int64_t kbound, int64_t min_hits, int64_t* hits64,
                               uint32_t* detmask, void* stream) {
    SFFTB_REQUIRE(n >= 0 && d >= 0 && G >= 1 && L >= 0 && M >= 1, "hash: bad sizes");
    SFFTB_REQUIRE(G <= 65535, "hash: too many groups");
    SFFTB_REQUIRE(M < (int64_t(1) << 31), "hash: M must be < 2^31");
    if (n == 0) return SFFTB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    // tensor-core path (csrc/hash_tc.cu): exact for any int64 rows, no bound
    if (G == 1) {
        const int rf = hash_hits_rollf(elems, n, d, zmat, L, M, bits, kbound, min_hits, hits64,
                                       detmask, st);
        if (rf < 0) return -rf;
        if (rf == 1) return SFFTB_OK;
        const int rr = hash_hits_roll(elems, n, d, zmat, L, M, bits, min_hits, hits64, detmask, st);
        if (rr < 0) return -rr;
        if (rr == 1) return SFFTB_OK;
        const int rc = hash_hits_tc(elems, n, d, zmat, L, M, bits, min_hits, hits64, detmask, st);
        if (rc < 0) return -rc;
        if (rc == 1) return SFFTB_OK;
    }
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    HashArgs a;
    a.elems = elems;
    a.n = n;
    a.d = (int)d;
    a.zmat = zmat;
    a.G = (int)G;
    a.L = (int)L;
    a.M = M;
    a.bits = bits;
    a.W = W;
    a.min_hits = min_hits;
    a.hits64 = hits64;
    a.detmask = detmask;
    a.nwords = (n + 31) / 32;
    a.magic = (uint32_t)(0xFFFFFFFFull / (uint64_t)M);
    const int64_t lat_bytes = W * 4;
    int64_t pow2_words = 4;
    while (pow2_words < W) pow2_words <<= 1;
    // 32-bit path: u = offset + sum_j k_j zc_j stays in [0, 2^32)
    const int64_t zmax = M / 2;
    bool fast = false;
    if (kbound >= 0 && d >= 1 && d <= 20) {
        const __int128 B = (__int128)kbound * zmax;
        const __int128 off = ((B + M - 1) / M) * M;
        if (off + B < ((__int128)1 << 32) && kbound < (int64_t(1) << 31)) {
            fast = true;
            a.offset = (uint32_t)off;
        }
    }
    {
        const char* v = getenv("SFFTB_HASH_VARIANT");
        a.variant = v ? atoi(v) : 0;  // 0: all-IMAD default
    }
    a.xsplit = fast ? hash_x_for((int)d, a.variant) : 0;
    const int64_t zbytes = ((L * std::max<int64_t>(d, 1) + 3) & ~int64_t(3)) * 4 + 16 +
                           ((L * a.xsplit * 2 + 3) & ~int64_t(3)) * 4;
    int64_t slot_bytes, smem_i;
    // (a) resident: power-of-two slots (OR addressing) when all L fit
    const int64_t pow2_bytes = pow2_words * 4;
    if (zbytes + pow2_bytes + L * pow2_bytes <= (int64_t)kBitmapSmemBudget) {
        slot_bytes = pow2_bytes;
        a.Lc = (int)std::max<int64_t>(L, 1);
        a.nbuf = 1;
        smem_i = zbytes + slot_bytes + (int64_t)a.Lc * slot_bytes;
    } else if (zbytes + L * lat_bytes <= (int64_t)kBitmapSmemBudget) {
        slot_bytes = lat_bytes;  // (b) resident, dense
        a.Lc = (int)std::max<int64_t>(L, 1);
        a.nbuf = 1;
        smem_i = zbytes + (int64_t)a.Lc * slot_bytes;
    } else {
        // (c) streamed, dense, in two buffers; leave L1 room for the row
        // loads (measured: 160 KB of bitmaps beats 224 KB at cfg4)
        slot_bytes = lat_bytes;
        const int64_t budget = (int64_t)kStreamSmemBudget - zbytes;
        SFFTB_REQUIRE(budget >= 2 * slot_bytes, "hash: one lattice bitmap exceeds shared memory");
        a.Lc = (int)(budget / (2 * slot_bytes));
        a.nbuf = 2;
        smem_i = zbytes + 2 * (int64_t)a.Lc * slot_bytes;
    }
    a.slot_words = (int)(slot_bytes / 4);
    const size_t smem = (size_t)smem_i;

    if (fast) return hash_dispatch<false>((int)d, a, smem, st);
    // 64-bit path: exact while d*(M-1)^2 < 2^62 (the reference's own bound,
    // detect.py:128-129); beyond that the 128-bit generic kernel
    const bool wide_ok = (__int128)d * (M - 1) * (M - 1) < ((__int128)1 << 62);
    if (kbound < 0 && d >= 1 && d <= 20 && wide_ok && M <= ((int64_t)1 << 30)) {
        // no host bound: the rows themselves pick the chain, warp by warp
        a.offset = (uint32_t)((((int64_t)1 << 31) / M) * M);
        const int64_t room = std::min<int64_t>(a.offset, (int64_t)0xFFFFFFFF - a.offset);
        a.auto_sum = room / std::max<int64_t>(zmax, 1);
        a.auto_bias = d * (M / 2 + 1) * M;
        return hash_dispatch<false, true>((int)d, a, smem, st);
    }
    if (d >= 1 && d <= 20 && wide_ok) {
        a.offset = 0;
        return hash_dispatch<true>((int)d, a, smem, st);
    }
    a.Lc = (int)std::max<int64_t>(
        1, std::min<int64_t>(std::max<int64_t>(L, 1),
                             ((int64_t)kBitmapSmemBudget - 16) / lat_bytes));
    const size_t smem_g = (size_t)((int64_t)a.Lc * lat_bytes);
    SFFTB_CUDA(smem_opt_in(hash_rows_generic, smem_g));
    const int64_t ntiles = ceil_div(n, kHashThreads);
    const int gx = (int)std::max<int64_t>(
        1, std::min<int64_t>(ntiles, ceil_div((int64_t)num_sms(), G)));
    hash_rows_generic<<<dim3(gx, (unsigned)G), kHashThreads, smem_g, st>>>(a);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int64_t sfftb_compact_workspace_bytes(int64_t G, int64_t n) {
    const int64_t nwords = (n + 31) / 32;
    const int64_t nblk = std::max<int64_t>(1, ceil_div(nwords, kCompactWordsPerBlock));
    return G * nblk * (int64_t)sizeof(int64_t);
}

namespace sfftb {
// single_words: masks up to this many words per group compact in one
// 1024-thread CTA per group (one launch); larger ones in count / scan / write
// passes over 512-word blocks.  Measured: 8192 for sparse masks (the metric
// instance, 4.02 vs 4.06 ms), 1024 for dense ones (config 5, 8.55 vs 8.65 ms).
int compact_mask_launch(const uint32_t* mask, int64_t G, int64_t n, int64_t cap, int64_t* idx,
                        int64_t* counts, int64_t* totals, void* ws, void* stream,
                        int64_t single_words);
}

extern "C" int sfftb_compact_mask_cap(const uint32_t* mask, int64_t G, int64_t n, int64_t cap,
                                      int64_t* idx, int64_t* counts, int64_t* totals, void* ws,
                                      void* stream) {
    return compact_mask_launch(mask, G, n, cap, idx, counts, totals, ws, stream,
                               kCompactSingleWords);
}

int sfftb::compact_mask_launch(const uint32_t* mask, int64_t G, int64_t n, int64_t cap,
                               int64_t* idx, int64_t* counts, int64_t* totals, void* ws,
                               void* stream, int64_t single_words) {
    SFFTB_REQUIRE(G >= 1 && n >= 0 && G <= 65535 && cap >= 0, "compact: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nwords = (n + 31) / 32;
    const int64_t nblk = std::max<int64_t>(1, ceil_div(nwords, kCompactWordsPerBlock));
    int64_t* bs = (int64_t*)ws;
    if (nwords <= single_words) {
        compact_write<true, 1024><<<dim3(1, (unsigned)G), 1024, 0, st>>>(
            mask, nwords, n, 1, nullptr, idx, counts, cap, totals);
        SFFTB_CHECK_LAUNCH();
        return SFFTB_OK;
    }
    compact_count<<<dim3((unsigned)nblk, (unsigned)G), kCompactThreads, 0, st>>>(mask, nwords,
                                                                                 nblk, bs);
    SFFTB_CHECK_LAUNCH();
    compact_scan<<<(unsigned)G, kCompactScanThreads, 0, st>>>(bs, nblk, counts, cap, totals);
    SFFTB_CHECK_LAUNCH();
    compact_write<false><<<dim3((unsigned)nblk, (unsigned)G), kCompactThreads, 0, st>>>(
        mask, nwords, n, nblk, bs, idx, counts, cap, totals);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_compact_mask(const uint32_t* mask, int64_t G, int64_t n, int64_t* idx,
                                  int64_t* counts, void* ws, void* stream) {
    return sfftb_compact_mask_cap(mask, G, n, n, idx, counts, nullptr, ws, stream);
}

extern "C" int sfftb_medians(const int64_t* elems, int64_t d, const int64_t* zmat, int64_t G,
                             int64_t L, int64_t M, const double* ghat, const int64_t* idx,
                             const int64_t* counts, int64_t cap, double* coeffs, void* stream) {
    SFFTB_REQUIRE(L >= 1 && L <= 128 && (L % 2) == 1, "medians require odd L <= 128");
    SFFTB_REQUIRE(G >= 1 && M >= 1, "medians: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = num_sms() * 8;
    if (L <= 32)
        medians_kernel<1><<<blocks, 256, 0, st>>>(elems, (int)d, zmat, (int)G, (int)L, M,
                                                  (const double2*)ghat, idx, counts, cap,
                                                  (double2*)coeffs);
    else if (L <= 64)
        medians_kernel<2><<<blocks, 256, 0, st>>>(elems, (int)d, zmat, (int)G, (int)L, M,
                                                  (const double2*)ghat, idx, counts, cap,
                                                  (double2*)coeffs);
    else
        medians_kernel<4><<<blocks, 256, 0, st>>>(elems, (int)d, zmat, (int)G, (int)L, M,
                                                  (const double2*)ghat, idx, counts, cap,
                                                  (double2*)coeffs);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

__global__ void threshold_mask_kernel(const int64_t* __restrict__ hits, int64_t n, double thr,
                                      uint32_t* __restrict__ mask) {
    const int64_t nb = (n + 31) / 32 * 32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool d = i < n && (double)hits[i] >= thr;
        const unsigned b = __ballot_sync(0xffffffffu, d);
        if ((threadIdx.x & 31) == 0) mask[i >> 5] = b;
    }
}

extern "C" int sfftb_threshold_mask(const int64_t* hits, int64_t n, double thr, uint32_t* mask,
                                    void* stream) {
    if (n <= 0) return SFFTB_OK;
    threshold_mask_kernel<<<grid_for((n + 31) / 32 * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        hits, n, thr, mask);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_rows_hits_medians(const double* vals, int64_t n, int64_t L, double theta,
                                       double thr, int want_medians, int64_t* hits,
                                       double* medians, void* stream) {
    SFFTB_REQUIRE(n >= 0 && L >= 1 && L < (int64_t(1) << 30), "rows_hits_medians: bad L");
    if (n == 0) return SFFTB_OK;
    rows_hits_medians_kernel<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        (const double2*)vals, n, (int)L, theta, thr, want_medians, hits, (double2*)medians);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_pair_residues(const int64_t* prefix, int64_t n1, int64_t t,
                                   const int64_t* vals, int64_t n2, const int64_t* zmat,
                                   int64_t GL, int64_t M, int32_t* P, int32_t* V,
                                   void* stream) {
    SFFTB_REQUIRE(n1 >= 0 && n2 >= 0 && t >= 1 && GL >= 1, "pair_residues: bad sizes");
    SFFTB_REQUIRE(M >= 1 && M < (int64_t(1) << 30), "pair_residues: M must be < 2^30");
    const int64_t total = GL * (n1 + n2);
    if (total == 0) return SFFTB_OK;
    pair_residues_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
        prefix, n1, (int)t, vals, n2, zmat, GL, M, P, V);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

static int64_t pair_span(int64_t n2) { return kPairTile / n2 + 2; }

extern "C" int64_t sfftb_hash_pairs_smem_bytes(int64_t L, int64_t M, int64_t n2) {
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    return 4 * (L * W + ((L * n2 + 3) & ~int64_t(3)) + L * pair_span(n2));
}

extern "C" int sfftb_hash_pairs(const int32_t* P, const int32_t* V, int64_t n1, int64_t n2,
                                int64_t G, int64_t L, int64_t M, const uint32_t* bits,
                                int64_t min_hits, int64_t* hits64, uint32_t* detmask,
                                void* stream) {
    SFFTB_REQUIRE(n1 >= 0 && n2 >= 1 && G >= 1 && G <= 65535 && L >= 1, "hash_pairs: bad sizes");
    SFFTB_REQUIRE(M >= 1 && M < (int64_t(1) << 30), "hash_pairs: M must be < 2^30");
    const int64_t n = n1 * n2;
    if (n == 0) return SFFTB_OK;
    const size_t sm = (size_t)sfftb_hash_pairs_smem_bytes(L, M, n2);
    SFFTB_REQUIRE(sm <= 200 * 1024, "hash_pairs: bitmaps + tables exceed shared memory");
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    SFFTB_CUDA(smem_opt_in(hash_pairs_kernel, sm));
    int per_sm = 1;
    SFFTB_CUDA(occupancy(&per_sm, hash_pairs_kernel, kPairThreads, sm));
    const int64_t want =
        std::max<int64_t>(1, ceil_div((int64_t)num_sms() * std::max(per_sm, 1), G));
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kPairTile), want));
    hash_pairs_kernel<<<dim3(gx, (unsigned)G), kPairThreads, sm, (cudaStream_t)stream>>>(
        P, V, n1, n2, (int)L, M, bits, W, min_hits, hits64, detmask, (int)pair_span(n2));
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

namespace sfftb {
int medians_pairs_launch(const int32_t* P, const int32_t* V, int64_t n1, int64_t n2, int64_t G,
                         int64_t L, int64_t M, const double* ghat, const int64_t* idx,
                         const int64_t* counts, int64_t cap, double* coeffs, void* stream,
                         bool dense);
}

extern "C" int sfftb_medians_pairs(const int32_t* P, const int32_t* V, int64_t n1, int64_t n2,
                                   int64_t G, int64_t L, int64_t M, const double* ghat,
                                   const int64_t* idx, const int64_t* counts, int64_t cap,
                                   double* coeffs, void* stream) {
    return medians_pairs_launch(P, V, n1, n2, G, L, M, ghat, idx, counts, cap, coeffs, stream,
                                false);
}

namespace sfftb {
// dense: most candidates detected (noisy data) -- then two rows per warp pays
// off (cfg5 9.33 -> 8.55 ms); with sparse detections the one-row kernel is
// lighter next to the concurrent transforms (metric 4.10 -> 4.05 ms)
int medians_pairs_launch(const int32_t* P, const int32_t* V, int64_t n1, int64_t n2, int64_t G,
                         int64_t L, int64_t M, const double* ghat, const int64_t* idx,
                         const int64_t* counts, int64_t cap, double* coeffs, void* stream,
                         bool dense) {
    SFFTB_REQUIRE(L >= 1 && L <= 128 && (L % 2) == 1, "medians require odd L <= 128");
    SFFTB_REQUIRE(G >= 1 && M >= 1 && n2 >= 1, "medians_pairs: bad sizes");
    SFFTB_REQUIRE(n1 * n2 < (int64_t(1) << 32), "medians_pairs: n1 * n2 must be < 2^32");
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = num_sms() * 8;
    const PairTables pt{P, V, n1, n2};
    const int64_t lim = int64_t(1) << 31;
    const bool small = G * L * std::max<int64_t>(std::max<int64_t>(n1, n2), M) < lim;
    auto go = [&](auto kern) {
        kern<<<blocks, 256, 0, st>>>(nullptr, 0, nullptr, (int)G, (int)L, M,
                                     (const double2*)ghat, idx, counts, cap, (double2*)coeffs,
                                     pt);
    };
    // pair-table medians by selection network (medians_net_pairs_kernel):
    // config 5 8.62 -> 7.75 ms, the metric instance unchanged (A/B on one box,
    // profiles/r02/ab_mednet.txt); SFFTB_MEDNET=0 restores the rank kernels,
    // 1 uses the network for dense detections only
    static const int mednet = [] {
        const char* e = getenv("SFFTB_MEDNET");
        return e ? atoi(e) : 2;
    }();
    if (small && L <= 63 && mednet > 0 && (mednet > 1 || dense)) {
        const int nb = num_sms() * 8;
        switch (L) {
#define SFFTB_MN(LL)                                                                        \
    case LL:                                                                                \
        medians_net_pairs_kernel<LL><<<nb, 256, 0, st>>>((int)G, M, (const double2*)ghat, \
                                                         idx, counts, cap,                \
                                                         (double2*)coeffs, pt);           \
        break;
            SFFTB_MN(1) SFFTB_MN(3) SFFTB_MN(5) SFFTB_MN(7) SFFTB_MN(9) SFFTB_MN(11)
            SFFTB_MN(13) SFFTB_MN(15) SFFTB_MN(17) SFFTB_MN(19) SFFTB_MN(21) SFFTB_MN(23)
            SFFTB_MN(25) SFFTB_MN(27) SFFTB_MN(29) SFFTB_MN(31) SFFTB_MN(33) SFFTB_MN(35)
            SFFTB_MN(37) SFFTB_MN(39) SFFTB_MN(41) SFFTB_MN(43) SFFTB_MN(45) SFFTB_MN(47)
            SFFTB_MN(49) SFFTB_MN(51) SFFTB_MN(53) SFFTB_MN(55) SFFTB_MN(57) SFFTB_MN(59)
            SFFTB_MN(61) SFFTB_MN(63)
#undef SFFTB_MN
        }
    } else if (L <= 32)
        small ? go(medians_kernel<1, true, true>) : go(medians_kernel<1, true>);
    else if (L <= 64)
    {
        static const int two_rows = [] {
            const char* e = getenv("SFFTB_MEDIANS2");
            return e ? atoi(e) : -1;  // -1: by the caller's density hint
        }();
        if (small && L <= 48 && (two_rows > 0 || (two_rows < 0 && dense))) {
            medians2_pairs_kernel<<<blocks, 256, 0, st>>>((int)G, (int)L, M,
                                                          (const double2*)ghat, idx, counts,
                                                          cap, (double2*)coeffs, pt);
        } else {
            small ? go(medians_kernel<2, true, true>) : go(medians_kernel<2, true>);
        }
    }
    else
        small ? go(medians_kernel<4, true, true>) : go(medians_kernel<4, true>);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
}  // namespace sfftb

extern "C" int sfftb_lattice_values(const int64_t* elems, int64_t d, const int64_t* zmat,
                                    int64_t L, int64_t M, const double* ghat,
                                    const int64_t* rows, int64_t nrows, double* out,
                                    void* stream) {
    if (nrows == 0 || L == 0) return SFFTB_OK;
    lattice_values_kernel<<<grid_for(nrows * L, 256), 256, 0, (cudaStream_t)stream>>>(
        elems, (int)d, zmat, (int)L, M, (const double2*)ghat, rows, nrows, (double2*)out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_sumsq(const double* x, int64_t stride, int64_t batch, int64_t M,
                           double* out, void* stream) {
    if (batch == 0) return SFFTB_OK;
    sumsq_kernel<<<(unsigned)batch, 256, 0, (cudaStream_t)stream>>>((const double2*)x, stride, M,
                                                                    out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

namespace sfftb {
int zero_thresholds_launch(const double* sumsq, int64_t G, int64_t L, int64_t M, double* theta,
                           cudaStream_t st, bool pdl) {
    SFFTB_REQUIRE(L >= 1 && L <= 256, "zero test: 1 <= L <= 256");
    const size_t zsm = sizeof(double) * (size_t)L;
    SFFTB_CUDA(smem_opt_in(zero_threshold_kernel, zsm));
    SFFTB_CUDA(launch_maybe_pdl(pdl, zero_threshold_kernel, dim3((unsigned)G), dim3(128), zsm, st,
                                sumsq, (int)G, (int)L, M, theta));
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
}  // namespace sfftb

extern "C" int sfftb_zero_thresholds(const double* sumsq, int64_t G, int64_t L, int64_t M,
                                     double* theta, void* stream) {
    return zero_thresholds_launch(sumsq, G, L, M, theta, (cudaStream_t)stream, false);
}

extern "C" int sfftb_mark_indices(const int64_t* idx, const int64_t* counts, int64_t G,
                                  int64_t cap, uint32_t* mask, int64_t n, void* stream) {
    (void)n;
    mark_kernel<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(idx, counts, (int)G, cap, mask);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_gather_rows(const int64_t* src, int64_t d, const int64_t* rows,
                                 const int64_t* count, int64_t cap, int64_t* dst, void* stream) {
    if (cap == 0 || d == 0) return SFFTB_OK;
    gather_rows_kernel<<<grid_for(cap * d, 256), 256, 0, (cudaStream_t)stream>>>(
        src, (int)d, rows, count, dst);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_pair_product(const int64_t* prev, int64_t n1, int64_t t,
                                  const int64_t* vals, int64_t n2, int64_t* out, void* stream) {
    const int64_t total = n1 * n2 * (t + 1);
    if (total == 0) return SFFTB_OK;
    pair_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(prev, n1, (int)t, vals,
                                                                        n2, out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

extern "C" int sfftb_row_bounds(const int64_t* elems, int64_t n, int64_t d, int64_t* out,
                                void* stream) {
    SFFTB_REQUIRE(d >= 1 && d <= 256, "row bounds: 1 <= d <= 256");
    cudaStream_t st = (cudaStream_t)stream;
    init_bounds_kernel<<<1, 256, 0, st>>>(out, (int)d);
    SFFTB_CHECK_LAUNCH();
    if (n == 0) return SFFTB_OK;
    const int threads = (int)(256 / d) * (int)d;
    row_bounds_kernel<<<grid_for(n * d, threads), threads, 0, st>>>(elems, n, (int)d, out);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}
