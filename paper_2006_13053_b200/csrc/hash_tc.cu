// K3 on the tensor cores: candidate residues k . z mod M as an exact u8 x u8
// -> s32 GEMM (tcgen05.mma kind::i8, accumulators in TMEM), then the
// reference's hit counting (_core.pyx:185-197: residue, |ghat| > theta probe,
// hits >= nu*L) in the epilogue.
//
// Why a GEMM is exact here.  A candidate row is d int64 coordinates, 8d bytes
// in HBM (row-major, FreqSet layout).  For |k| < 2^(8P) the two's-complement
// bytes b_0..b_7 of k satisfy
//     k = b_0 + 256 b_1 + ... + 256^(P-1) b_(P-1) - 2^(8P) [k < 0],
// with b_P = ... = b_7 = 255 [k < 0].  So, modulo the prime M,
//     k z = sum_{p<P} b_p (256^p z mod M) + b_P (-(2^(8P)/255) z mod M),
// a dot product of the RAW row bytes with per-lattice coefficients in [0, M).
// The A operand of the MMA is therefore the candidate tile exactly as it sits
// in HBM (TMA, no conversion pass); the B operand holds, per lattice, the
// three base-256 limbs of every coefficient (u8), so the MMA produces three
// s32 partial sums v_0..v_2 per (row, lattice) and
//     x = v_0 + 256 v_1 + 65536 v_2 = sum_{j,p} b_{jp} c_{jp}  <  2^32
// (d (P+1) 255 (M-1) < 2^32 is required), x == k.z (mod M).  One multiply-
// high reduction gives r = x mod M, then the bitmap probe.  Rows whose bytes
// P..7 are not a sign extension (|k| >= 2^(8P)) are caught by extra "validity"
// columns (sum of bytes P..7 of one coordinate must be 0 or 255 (8-P)) and
// recomputed exactly (64-bit) by the finalising thread from global memory.
//
// Cluster layout.  The nonzero bitmaps of all L lattices (L*M bits, 607 KB at
// config 4) do not fit one SM's shared memory, so a cluster of C CTAs splits
// the lattices: CTA c keeps the bitmaps of lattices [c*Lp, (c+1)*Lp) resident
// and computes those residues for EVERY row of the cluster's tiles.  Row
// tiles (128 rows) are TMA-multicast into all C CTAs (each CTA issues some of
// the 16-byte column chunks), so HBM/L2 read each candidate byte once.  Each
// CTA's epilogue produces a partial hit count per row and st.async's it into
// the finalising CTA (tile k -> CTA k mod C), which sums the C partials,
// writes hits (int64) and the detected bitmask word.
//
// Warp roles (608 threads): warp 0 = TMA producer (+ TMEM allocation), warp 1
// = MMA issuer, warp 2 = finaliser (sums the partials of the tiles this CTA
// owns), warps 3..18 = four epilogue groups of four warps (a group covers the
// 128 TMEM lanes; group e takes the cluster's tiles k = e mod 4).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <map>
#include <mutex>

#include "common.cuh"

namespace sfftb {

namespace tc {

constexpr int kEpiGroups = 4;
constexpr int kThreads = 96 + kEpiGroups * 128;  // producer, MMA, finaliser + epilogue
constexpr int kTileRows = 128;
constexpr int kTmemBufs = 8;        // accumulator buffers, 64 columns each
constexpr int kTmemStride = 64;
constexpr int kPSlotsMax = 8;       // partial-count slots per finalising CTA
constexpr int kPrefetch = 16;       // L2 prefetch distance in tiles
constexpr int kCols = 64;           // MMA N: 3 limbs x <= 16 lattices, validity at 48..63
constexpr int kValCol = 48;
constexpr int kLpMax = 16;
constexpr uint32_t kBadFlag = 1u << 16;  // partial-count flag: row outside the byte-GEMM range

struct Args {
    const int64_t* elems;  // (n, d) int64, for the exact recompute path
    int64_t n;
    int d;
    const int64_t* zmat;   // (L, d)
    int L, Lp, ncols, sw, nbox, nmma, P, stages, pslots, prefetch;
    uint32_t tile_bytes, guard;
    int nomc, dbg;  // diagnostics: per-CTA (unicast) tile loads; epilogue skipped
    unsigned long long* trace;  // diagnostics: event times of cluster 0's first tiles
    uint32_t M, magic, csign;
    uint32_t pw[8];        // 256^p mod M
    const uint32_t* bits;  // (L, W) nonzero bitmaps
    int W;
    int64_t ntiles;
    int64_t min_hits;
    int64_t* hits64;       // may be null
    uint32_t* detmask;     // ceil(n/32)
    unsigned long long* recomputed;  // rows taken by the exact path (diagnostic)
    uint32_t smem_bytes;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init_a(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_a(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// arrive on the barrier at cluster address `bar` (any CTA of the cluster)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// acquire at cluster scope: data written by other CTAs (st.async, multicast)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, int x, int y,
                                               uint32_t bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(map), "r"(x),
                 "r"(y)
                 : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(
                     raddr),
                 "r"(v), "r"(rbar)
                 : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of
// 8 rows x 16 B stored as 128 contiguous bytes; `lbo` = byte distance between
// the two K-adjacent core matrices, `sbo` = between M/N-adjacent ones.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t desc = 0;
    desc |= (uint64_t)((addr >> 4) & 0x3FFF);
    desc |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    desc |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    desc |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return desc;                // base offset 0, layout SWIZZLE_NONE
}

// A-operand descriptor of the m-th K = 32 slice of a tile of `sw`-byte TMA
// boxes (K-major): sw = 16 unswizzled chunk-major [box][128 rows][16 B];
// sw = 32/64/128 the TMA's SWIZZLE_32B/64B/128B rows, 8-row atoms of 8*sw B.
__device__ __forceinline__ uint64_t a_desc(uint32_t tile, int m, int sw) {
    if (sw == 16) return umma_desc(tile + (uint32_t)m * 4096u, 2048u, 128u);
    const int lg = sw == 32 ? 0 : (sw == 64 ? 1 : 2);  // log2 of the K slices per box
    const uint32_t addr = tile + (uint32_t)(m >> lg) * (uint32_t)sw * kTileRows +
                          (uint32_t)(m & ((1 << lg) - 1)) * 32u;
    const uint64_t layout = sw == 32 ? 6 : (sw == 64 ? 4 : 2);
    return umma_desc(addr, 16u, 8u * (uint32_t)sw) | (layout << 61);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define SFFTB_TMEM_LD16(taddr, v, o)                                                          \
    asm volatile(                                                                            \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15}, [%16];"                                                                   \
        : "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]),     \
          "=r"(v[o + 5]), "=r"(v[o + 6]), "=r"(v[o + 7]), "=r"(v[o + 8]), "=r"(v[o + 9]),     \
          "=r"(v[o + 10]), "=r"(v[o + 11]), "=r"(v[o + 12]), "=r"(v[o + 13]),                 \
          "=r"(v[o + 14]), "=r"(v[o + 15])                                                   \
        : "r"(taddr))

__device__ __forceinline__ uint32_t mod_m(uint32_t u, uint32_t M, uint32_t negM, uint32_t magic) {
    const uint32_t q = __umulhi(u, magic);
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(negM), "r"(u));
    return min(r, r - M);
}

// Exact hits of one row over all L lattices from global memory (rows whose
// coordinates exceed the byte-GEMM range).
__device__ int exact_row_hits(const Args& a, int64_t row) {
    int h = 0;
    for (int l = 0; l < a.L; ++l) {
        uint64_t acc = 0;
        for (int j = 0; j < a.d; ++j) {
            int64_t e = a.elems[row * a.d + j] % (int64_t)a.M;
            if (e < 0) e += a.M;
            int64_t z = a.zmat[(int64_t)l * a.d + j] % (int64_t)a.M;
            if (z < 0) z += a.M;
            acc = (acc + (uint64_t)e * (uint64_t)z) % a.M;
        }
        const uint32_t r = (uint32_t)acc;
        h += (a.bits[(int64_t)l * a.W + (r >> 5)] >> (r & 31)) & 1u;
    }
    return h;
}

// Shared-memory map (byte offsets from a 1024-aligned base).
struct Smem {
    uint32_t a, b, bits, pbuf, bars, tmem_holder;
    uint32_t full, aempty, tfull, tempty, pfull, pempty, bbar;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem smem_map(int stages, uint32_t tile_bytes, uint32_t guard, int nmma,
                                         int ncols, int Lp, int W, int C, int pslots) {
    Smem s;
    uint32_t o = 0;
    s.a = o;
    o += (uint32_t)stages * tile_bytes;
    o += guard;  // the last MMA of an unswizzled odd-chunk tile reads past it (zero weights)
    s.b = o;
    o += (uint32_t)(2 * nmma) * ncols * 16u;
    s.bits = align_up(o, 16);
    o = s.bits + (uint32_t)Lp * W * 4u;
    s.pbuf = align_up(o, 16);
    o = s.pbuf + (uint32_t)pslots * C * kTileRows * 4u;
    s.bars = align_up(o, 8);
    s.full = s.bars;
    s.aempty = s.full + 8u * stages;
    s.tfull = s.aempty + 8u * stages;
    s.tempty = s.tfull + 8u * kTmemBufs;
    s.pfull = s.tempty + 8u * kTmemBufs;
    s.pempty = s.pfull + 8u * pslots;
    s.bbar = s.pempty + 8u * pslots * C;
    s.tmem_holder = s.bbar + 8u;
    return s;
}

inline uint32_t smem_total(const Smem& s) { return s.tmem_holder + 16u + 1024u; }

// diagnostic event trace (SFFTB_HASH_TC_TRACE): cluster 0, CTA 0, tiles < 512
#define TRACE(ev, k)                                                                \
    do {                                                                            \
        if (a.trace && cid == 0 && rank == 0 && (k) < 512 && (k) >= 0) {                        \
            unsigned long long t_;                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
            a.trace[(ev) * 512 + (k)] = t_;                                         \
        }                                                                           \
    } while (0)

template <int C, int LP>
__global__ void __launch_bounds__(kThreads, 1)
    hash_tc_kernel(const __grid_constant__ CUtensorMap tmap, Args a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t raw = smem_addr(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const Smem S = smem_map(a.stages, a.tile_bytes, a.guard, a.nmma, kCols, LP, a.W, C, a.pslots);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t cid = cluster_id_x(), ncl = nclusters_x();
    const int64_t my_tiles = a.ntiles > cid ? (a.ntiles - 1 - cid) / ncl + 1 : 0;
    const int l0 = (int)rank * LP;
    const int Lc = max(0, min(a.L, l0 + LP) - l0);  // lattices of this CTA
    const uint16_t all_mask = (uint16_t)((1u << C) - 1u);
    const uint32_t a_stage_bytes = a.tile_bytes;
    const uint32_t box_bytes = (uint32_t)a.sw * kTileRows;

    // ---- setup: barriers, TMEM, B operand, resident bitmaps ----
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init_a(base + S.full + 8u * s, 1);
            mbar_init_a(base + S.aempty + 8u * s, a.nomc ? 1 : C);
        }
        for (int b = 0; b < kTmemBufs; ++b) {
            mbar_init_a(base + S.tfull + 8u * b, 1);
            mbar_init_a(base + S.tempty + 8u * b, 4);
        }
        for (int p = 0; p < a.pslots; ++p) mbar_init_a(base + S.pfull + 8u * p, 1);
        for (int p = 0; p < a.pslots * C; ++p) mbar_init_a(base + S.pempty + 8u * p, 1);
        mbar_init_a(base + S.bbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         base + S.tmem_holder)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // B operand: [2*nmma chunks][ncols][16 B], K index = 16*chunk + byte.
    {
        const uint32_t nB = (uint32_t)(2 * a.nmma) * kCols * 16u;
        const int nval = (a.d - (int)rank + C - 1) / C;  // validity columns
        for (uint32_t e = threadIdx.x; e < nB / 4; e += blockDim.x) {
            uint32_t word = 0;
            for (int t = 0; t < 4; ++t) {
                const uint32_t idx = e * 4 + t;
                const int q = (int)(idx / (kCols * 16u));
                const int col = (int)((idx / 16u) % kCols);
                const int kb = q * 16 + (int)(idx % 16u);
                const int j = kb >> 3, p = kb & 7;
                uint32_t v = 0;
                if (j < a.d) {
                    if (col < 3 * Lc) {
                        const int l = l0 + col / 3, limb = col % 3;
                        int64_t z = a.zmat[(int64_t)l * a.d + j] % (int64_t)a.M;
                        if (z < 0) z += a.M;
                        uint64_t c = 0;
                        if (p < a.P) c = ((uint64_t)z * a.pw[p]) % a.M;
                        else if (p == a.P) c = ((uint64_t)z * a.csign) % a.M;
                        v = (uint32_t)(c >> (8 * limb)) & 255u;
                    } else if (col >= kValCol && col < kValCol + nval) {
                        const int jv = (int)rank + (col - kValCol) * C;
                        v = (j == jv && p >= a.P) ? 1u : 0u;
                    }
                }
                word |= v << (8 * t);
            }
            *reinterpret_cast<uint32_t*>(smem_raw + (base - raw) + S.b + e * 4) = word;
        }
    }
    {  // unused lattice slots probe an all-zero bitmap
        uint32_t* z = reinterpret_cast<uint32_t*>(smem_raw + (base - raw) + S.bits);
        for (int e = Lc * a.W + threadIdx.x; e < LP * a.W; e += blockDim.x) z[e] = 0u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0 && Lc > 0) {
        const uint32_t bytes = (uint32_t)a.W * 4u;
        mbar_expect_tx_a(base + S.bbar, bytes * (uint32_t)Lc);
        for (int i = 0; i < Lc; ++i)
            bulk_g2s_addr(base + S.bits + (uint32_t)i * bytes, a.bits + (int64_t)(l0 + i) * a.W,
                          bytes, reinterpret_cast<uint64_t*>(smem_raw + (base - raw) + S.bbar));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync_all();  // every CTA's barriers are initialised before any remote traffic
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (base - raw) +
                                                                S.tmem_holder);

    if (warp == 0) {
        // ================= TMA producer (whole warp, one elected lane issues) =================
        const bool leader = elect_one();
        int s = 0;
        uint32_t ph = 0;  // parity of the current round of the A ring
        int y = (int)cid * kTileRows;
        const int ystep = (int)ncl * kTileRows;
        for (int k = 0; k < (int)my_tiles; ++k, y += ystep) {
            if (k >= a.stages) mbar_wait_a(base + S.aempty + 8u * s, ph ^ 1u);
            if (leader) {
                TRACE(7, k);
                const uint32_t full = base + S.full + 8u * s;
                TRACE(0, k);
                mbar_expect_tx_a(full, a_stage_bytes);
                const uint32_t dst = base + S.a + (uint32_t)s * a_stage_bytes;
                if (a.nomc) {
                    for (int bx = 0; bx < a.nbox; ++bx)
                        tma_load_2d(dst + (uint32_t)bx * box_bytes, &tmap, bx * a.sw, y, full);
                } else {
                    for (int bx = (int)rank; bx < a.nbox; bx += C)
                        tma_load_2d_mc(dst + (uint32_t)bx * box_bytes, &tmap, bx * a.sw, y, full,
                                       all_mask);
                }
                if (a.prefetch > 0 && k + a.prefetch < (int)my_tiles) {
                    const int yp = y + a.prefetch * ystep;
                    for (int bx = (int)rank; bx < a.nbox; bx += C)
                        tma_prefetch_2d(&tmap, bx * a.sw, yp);
                }
            }
            __syncwarp();
            if (++s == a.stages) {
                s = 0;
                ph ^= 1u;
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (whole warp, one elected lane issues) =================
        const bool leader = elect_one();
        const uint32_t idesc = (2u << 4)                           // D = s32
                               | ((uint32_t)(kCols >> 3) << 17)  // N
                               | ((uint32_t)(kTileRows >> 4) << 24);  // M = 128
        // descriptors of stage 0 (stage s adds s * a_stage_bytes to the 14-bit
        // start-address field, which cannot carry: SMEM < 256 KB)
        uint64_t ad0[4], bd[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            ad0[m] = a_desc(base + S.a, m, a.sw);
            bd[m] = umma_desc(base + S.b + (uint32_t)m * 2u * kCols * 16u, kCols * 16u, 128u);
        }
        const int nmma = (a.dbg & 2) ? 1 : a.nmma;
        const uint64_t sinc = (uint64_t)(a_stage_bytes >> 4);
        int s = 0, b = 0;
        uint32_t ph = 0, tph = 0;
        uint64_t soff = 0;
        for (int k = 0; k < (int)my_tiles; ++k) {
            if (k >= kTmemBufs) mbar_wait_a(base + S.tempty + 8u * b, tph ^ 1u);
            if (leader) TRACE(1, k);
            mbar_wait_a(base + S.full + 8u * s, ph);
            tc_fence_after();
            if (leader) {
                TRACE(2, k);
                const uint32_t dt = tmem + (uint32_t)b * kTmemStride;
                umma_i8(dt, ad0[0] + soff, bd[0], idesc, 0u);
                if (nmma > 1) umma_i8(dt, ad0[1] + soff, bd[1], idesc, 1u);
                if (nmma > 2) umma_i8(dt, ad0[2] + soff, bd[2], idesc, 1u);
                if (nmma > 3) umma_i8(dt, ad0[3] + soff, bd[3], idesc, 1u);
                umma_commit(base + S.tfull + 8u * b);
                if (a.nomc) umma_commit(base + S.aempty + 8u * s);
                else umma_commit_mc(base + S.aempty + 8u * s, all_mask);
                TRACE(3, k);
            }
            __syncwarp();
            soff += sinc;
            if (++s == a.stages) {
                s = 0;
                ph ^= 1u;
                soff = 0;
            }
            if (++b == kTmemBufs) {
                b = 0;
                tph ^= 1u;
            }
        }
    } else if (warp == 2) {
        // ============ finaliser: tiles k = rank (mod C) of the cluster ============
        int my_tiles_fin = (int)my_tiles;
        if (a.dbg & 4) my_tiles_fin = 0;
        const uint32_t* pb = reinterpret_cast<const uint32_t*>(smem_raw + (base - raw) + S.pbuf);
        const int plog = a.pslots == 8 ? 3 : 2;  // pslots is 4 or 8
        for (int k = (int)rank, m = 0; k < my_tiles_fin; k += C, ++m) {
            const int ps = m & (a.pslots - 1);
            const uint32_t pf = base + S.pfull + 8u * ps;
            if (lane == 0) mbar_expect_tx_a(pf, (uint32_t)C * kTileRows * 4u);
            mbar_wait_cluster(pf, (uint32_t)((m >> plog) & 1));
            if (lane == 0) TRACE(4, k);
            uint32_t hsum[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                hsum[q] = 0;
#pragma unroll
                for (int c = 0; c < C; ++c) hsum[q] += pb[(ps * C + c) * kTileRows + q * 32 + lane];
            }
            __syncwarp();
            if (lane < C)  // slot ps of this CTA is free again for every writer
                mbar_arrive_remote(mapa(base + S.pempty + 8u * (rank * a.pslots + ps), (uint32_t)lane));
            const int64_t t = (int64_t)cid + (int64_t)k * ncl;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t row0 = t * kTileRows + q * 32;
                const int64_t row = row0 + lane;
                const bool valid = row < a.n;
                int64_t hits = (int64_t)(hsum[q] & (kBadFlag - 1u));
                if (hsum[q] >= kBadFlag && valid) {
                    hits = exact_row_hits(a, row);
                    atomicAdd(a.recomputed, 1ull);
                }
                const unsigned det = __ballot_sync(0xffffffffu, valid && hits >= a.min_hits);
                if (valid && a.hits64) a.hits64[row] = hits;
                if (lane == 0 && row0 < a.n) a.detmask[row0 >> 5] = det;
            }
        }
    } else {
        // ================= epilogue =================
        const int ew = warp - 3;
        const int grp = ew >> 2;
        const int quad = warp & 3;  // TMEM lane quadrant this warp may access
        const int row_in_tile = quad * 32 + lane;
        const uint32_t M = a.M, negM = 0u - a.M, magic = a.magic;
        const uint32_t vgood = 255u * (uint32_t)(8 - a.P);
        const int nval = (a.d - (int)rank + C - 1) / C;
        if (Lc > 0) mbar_wait_a(base + S.bbar, 0);
        const uint32_t* bm = reinterpret_cast<const uint32_t*>(smem_raw + (base - raw) + S.bits);
        const int plog = a.pslots == 8 ? 3 : 2;  // pslots is 4 or 8
        for (int k = grp; k < (int)my_tiles; k += kEpiGroups) {
            const int b = k & (kTmemBufs - 1);
            mbar_wait_a(base + S.tfull + 8u * b, (uint32_t)((k / kTmemBufs) & 1));
            if (lane == 0 && quad == 0) TRACE(5, k);
            tc_fence_after();
            uint32_t v[kCols];
            const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)b * kTmemStride;
            SFFTB_TMEM_LD16(taddr, v, 0);
            SFFTB_TMEM_LD16(taddr + 16, v, 16);
            if (LP > 10) SFFTB_TMEM_LD16(taddr + 32, v, 32);
            SFFTB_TMEM_LD16(taddr + 48, v, 48);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_a(base + S.tempty + 8u * b);
            if (a.dbg & 4) continue;  // diagnostic: TMA + MMA + TMEM drain only

            // slots i >= Lc hold an all-zero bitmap and zero B columns
            uint32_t bacc = 0;
#pragma unroll
            for (int i = 0; i < LP; ++i) {
                if (a.dbg & 1) break;  // diagnostic: TMA + MMA + exchange without the probes
                uint32_t x;
                asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(x) : "r"(v[3 * i + 1]), "r"(v[3 * i]));
                asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(x) : "r"(v[3 * i + 2]), "r"(x));
                const uint32_t r = mod_m(x, M, negM, magic);
                const uint32_t w = bm[(uint32_t)i * a.W + (r >> 5)];
                bacc = __funnelshift_r(bacc, __funnelshift_r(w, w, r), 1);
            }
            uint32_t partial = __popc(bacc);
            bool bad = false;
#pragma unroll
            for (int i = 0; i < kCols - kValCol; ++i) {
                if (i < nval) {
                    const uint32_t vv = v[kValCol + i];
                    bad |= (vv != 0u) & (vv != vgood);
                }
            }
            if (bad) partial |= kBadFlag;

            // ---- send the partial to the finalising CTA (tile k -> CTA k mod C) ----
            const int f = k & (C - 1);
            const int m = k / C;  // round of this tile at CTA f
            const int ps = m & (a.pslots - 1);
            if (m >= a.pslots)
                mbar_wait_cluster(base + S.pempty + 8u * (f * a.pslots + ps),
                                  (uint32_t)(((m >> plog) - 1) & 1));
            const uint32_t slot_off =
                S.pbuf + (uint32_t)((ps * C + (int)rank) * kTileRows + row_in_tile) * 4u;
            st_async_u32(mapa(base + slot_off, (uint32_t)f), partial,
                         mapa(base + S.pfull + 8u * ps, (uint32_t)f));
            if (lane == 0 && quad == 0) TRACE(6, k);
        }
    }
    __syncwarp();

    // ---- teardown: no CTA leaves while others may still write into it ----
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                     : "memory");
    }
}

// ---- host side ----

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

static int64_t inv_mod(int64_t a, int64_t m) {  // a^-1 mod m, or -1
    int64_t t = 0, nt = 1, r = m, nr = a % m;
    while (nr != 0) {
        const int64_t q = r / nr;
        int64_t tmp = t - q * nt;
        t = nt;
        nt = tmp;
        tmp = r - q * nr;
        r = nr;
        nr = tmp;
    }
    if (r != 1) return -1;
    return t < 0 ? t + m : t;
}

template <int C, int LP>
static int launch_c(const CUtensorMap& map, Args& a, uint32_t smem, cudaStream_t st) {
    auto kern = hash_tc_kernel<C, LP>;
    SFFTB_CUDA(smem_opt_in(kern, smem));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent grid: as many clusters as fit at once (memoised per shape)
    static std::mutex mu;
    static std::map<std::pair<int, uint32_t>, int> ncl_cache;
    int ncl_max = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        int dev = 0;
        cudaGetDevice(&dev);
        const auto key = std::make_pair(dev * 1024 + C * 32 + LP, smem);
        auto it = ncl_cache.find(key);
        if (it == ncl_cache.end()) {
            cfg.gridDim = dim3((unsigned)(C * num_sms()));
            int ncl = 0;
            SFFTB_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
            it = ncl_cache.emplace(key, std::max(ncl, 1)).first;
        }
        ncl_max = it->second;
    }
    if (const char* e = getenv("SFFTB_HASH_TC_CLUSTERS")) ncl_max = std::max(1, atoi(e));
    const int64_t ncl = std::min<int64_t>(ncl_max, std::max<int64_t>(a.ntiles, 1));
    cfg.gridDim = dim3((unsigned)(ncl * C));
    if (getenv("SFFTB_HASH_TC_DEBUG"))
        fprintf(stderr, "hash_tc: C=%d LP=%d sw=%d stages=%d pslots=%d P=%d clusters=%lld smem=%u tiles=%lld\n",
                C, LP, a.sw, a.stages, a.pslots, a.P, (long long)ncl, smem, (long long)a.ntiles);
    SFFTB_CUDA(cudaLaunchKernelEx(&cfg, kern, map, a));
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

static unsigned long long* recomputed_counter() {
    static unsigned long long* p = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        if (cudaMalloc(&p, sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(p, 0, sizeof(unsigned long long));
        else
            p = nullptr;
    });
    return p;
}

}  // namespace tc

// Returns 1 when the tensor-core path handled the call, 0 when the shape is
// outside it (the caller takes the CUDA-core kernels), <0 on error.
int hash_hits_tc(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat, int64_t L,
                 int64_t M, const uint32_t* bits, int64_t min_hits, int64_t* hits64,
                 uint32_t* detmask, cudaStream_t st) {
    using namespace tc;
    {
        // opt-in: measured slower than the CUDA-core kernel at config 4
        // (6.2 vs 3.8 ms, profiles/r02/SUMMARY.md: every row tile must reach
        // all C SMs of the cluster, and the TMA delivers 16-32 B row segments)
        const char* e = getenv("SFFTB_HASH_TC");
        if (!e || e[0] != '1') return 0;
    }
    const char* mr = getenv("SFFTB_HASH_TC_MINROWS");
    const int64_t min_rows = mr ? atoll(mr) : (int64_t)1 << 16;
    // int32 tile/row coordinates in the kernel (TMA coordinates are int32 too)
    if (n < min_rows || n > ((int64_t)1 << 31) - (int64_t)1024 * kTileRows || d < 2 || d > 16 ||
        (d & 1) || L < 1 || M < 2 || M >= (1 << 24))
        return 0;
    if (((uintptr_t)elems & 15) != 0 || ((uintptr_t)bits & 15) != 0) return 0;
    const int64_t inv255 = inv_mod(255 % M, M);
    if (inv255 < 0) return 0;
    // weighted bytes P: the largest in [2, 7] with d (P+1) 255 (M-1) < 2^32
    int P = 0;
    for (int p = 7; p >= 2; --p)
        if ((__int128)d * (p + 1) * 255 * (M - 1) < ((__int128)1 << 32)) {
            P = p;
            break;
        }
    if (P == 0) return 0;
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    // TMA box width sw (bytes of a row per box): 16 = unswizzled 16-B chunks,
    // 32/64/128 = swizzled boxes (fewer, wider TMA row requests); boxes past
    // the 8d-byte row are zero-filled by the TMA
    int sw = 32;
    if (const char* e = getenv("SFFTB_HASH_TC_SW")) sw = atoi(e);
    if (sw != 16 && sw != 32 && sw != 64 && sw != 128) return 0;
    const int nbox = (int)((8 * d + sw - 1) / sw);
    const int nmma = (nbox * sw + 31) / 32;
    const uint32_t tile_bytes = (uint32_t)nbox * sw * kTileRows;
    const uint32_t guard = (uint32_t)(nmma * 32 - nbox * sw) * kTileRows;  // sw = 16, odd nbox
    int prefetch = kPrefetch;
    if (const char* e = getenv("SFFTB_HASH_TC_PF")) prefetch = atoi(e);
    static int prop_smem = 0;
    if (prop_smem == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&prop_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (prop_smem <= 0) prop_smem = 232448;
    }
    // cluster size C and lattices per CTA LP (instantiated: LP in {4,8,12,16}):
    // the smallest C whose resident bitmaps leave room for >= 3 A stages
    int C = 0, LP = 0, stages = 0, pslots = 0;
    uint32_t smem = 0;
    const char* ce = getenv("SFFTB_HASH_TC_CLUSTER");
    for (int c : {4, 8, 2}) {
        if (ce && atoi(ce) != c) continue;
        int lp = (int)((L + c - 1) / c);
        lp = (lp + 3) / 4 * 4;
        if (lp > kLpMax) continue;
        if ((d + c - 1) / c > kCols - kValCol) continue;
        // deepest A ring (<= 8 stages) with >= 4 partial slots, then more slots
        for (int s = 8; s >= 3 && !C; --s)
            for (int ps = kPSlotsMax; ps >= 4; ps /= 2) {
                const uint32_t tot =
                    smem_total(smem_map(s, tile_bytes, guard, nmma, kCols, lp, (int)W, c, ps));
                if (tot <= (uint32_t)prop_smem) {
                    C = c;
                    LP = lp;
                    stages = s;
                    pslots = ps;
                    smem = tot;
                    break;
                }
            }
        if (C) break;
    }
    if (C == 0) return 0;
    auto enc = encode_fn();
    if (!enc) return 0;
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)(8 * d), (cuuint64_t)n};
    cuuint64_t gstride[1] = {(cuuint64_t)(8 * d)};
    cuuint32_t box[2] = {(cuuint32_t)sw, (cuuint32_t)kTileRows};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)elems, gdim, gstride, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      sw == 16 ? CU_TENSOR_MAP_SWIZZLE_NONE
                      : sw == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                      : sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return 0;
    unsigned long long* rec = recomputed_counter();
    if (!rec) return 0;

    Args a;
    a.elems = elems;
    a.n = n;
    a.d = (int)d;
    a.zmat = zmat;
    a.L = (int)L;
    a.Lp = LP;
    a.ncols = kCols;
    a.sw = sw;
    a.nbox = nbox;
    a.tile_bytes = tile_bytes;
    a.guard = guard;
    a.prefetch = prefetch;
    a.nomc = getenv("SFFTB_HASH_TC_NOMC") ? 1 : 0;
    a.dbg = getenv("SFFTB_HASH_TC_DBG") ? atoi(getenv("SFFTB_HASH_TC_DBG")) : 0;
    static unsigned long long* trace = nullptr;
    a.trace = nullptr;
    if (getenv("SFFTB_HASH_TC_TRACE")) {
        if (!trace) SFFTB_CUDA(cudaMalloc(&trace, 8 * 512 * sizeof(unsigned long long)));
        SFFTB_CUDA(cudaMemset(trace, 0, 8 * 512 * sizeof(unsigned long long)));
        a.trace = trace;
    }
    a.nmma = nmma;
    a.P = P;
    a.stages = stages;
    a.pslots = pslots;
    a.M = (uint32_t)M;
    a.magic = (uint32_t)(0xFFFFFFFFull / (uint64_t)M);
    uint64_t pw = 1 % (uint64_t)M;
    for (int p = 0; p < 8; ++p) {
        a.pw[p] = (uint32_t)pw;
        pw = (pw * 256) % (uint64_t)M;
    }
    // csign = -(256^P / 255) mod M
    const uint64_t t = ((uint64_t)a.pw[P] * (uint64_t)inv255) % (uint64_t)M;
    a.csign = (uint32_t)(((uint64_t)M - t) % (uint64_t)M);
    a.bits = bits;
    a.W = (int)W;
    a.ntiles = (n + kTileRows - 1) / kTileRows;
    a.min_hits = min_hits;
    a.hits64 = hits64;
    a.detmask = detmask;
    a.recomputed = rec;
    a.smem_bytes = smem;
    int rc = SFFTB_EINVAL;
#define SFFTB_TC_CASE(CC, LL) \
    if (C == CC && LP == LL) rc = launch_c<CC, LL>(map, a, smem, st);
    SFFTB_TC_CASE(2, 4) SFFTB_TC_CASE(2, 8) SFFTB_TC_CASE(2, 12) SFFTB_TC_CASE(2, 16)
    SFFTB_TC_CASE(4, 4) SFFTB_TC_CASE(4, 8) SFFTB_TC_CASE(4, 12) SFFTB_TC_CASE(4, 16)
    SFFTB_TC_CASE(8, 4) SFFTB_TC_CASE(8, 8) SFFTB_TC_CASE(8, 12) SFFTB_TC_CASE(8, 16)
#undef SFFTB_TC_CASE
    if (a.trace && rc == SFFTB_OK) {
        unsigned long long h[8 * 512];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost);
        const unsigned long long t0 = h[0];
        fprintf(stderr, "k  issue mma_wait full_ok committed fin tfull_epi sent aempty_done (ns)\n");
        for (int k = 0; k < 512; k += (k < 40 ? 1 : 37)) {
            fprintf(stderr, "%3d", k);
            for (int e = 0; e < 8; ++e)
                fprintf(stderr, " %8lld", h[e * 512 + k] ? (long long)(h[e * 512 + k] - t0) : -1LL);
            fprintf(stderr, "\n");
        }
    }
    return rc == SFFTB_OK ? 1 : -rc;
}

}  // namespace sfftb

// Rows the tensor-core hash sent to its exact 64-bit path (|coordinate| beyond
// the byte-GEMM range) since the last reset; tests use it to prove both paths.
extern "C" int64_t sfftb_hash_tc_recomputed(int reset) {
    unsigned long long* p = sfftb::tc::recomputed_counter();
    if (!p) return -1;
    unsigned long long v = 0;
    if (cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    if (reset) cudaMemset(p, 0, sizeof(v));
    return (int64_t)v;
}
