// K3 on the tensor cores, second design ("rolling" kernel): candidate residues
// k . z mod M as an exact u8 x u8 -> s32 GEMM whose A operand (the candidate
// rows) lives in TENSOR MEMORY, and the per-lattice nonzero bitmaps streamed
// through shared memory in lattice groups while ~6000 rows stay resident.
// Same semantics as hash_rows (hash.cu): the reference's per-candidate loop of
// _core.pyx:185-197 (residue, |ghat| > theta probe, hits >= nu*L).
//
// Why this shape.  The CUDA-core kernel spends 10 IMADs per (row, lattice) on
// the dot product (IMAD-pipe floor 2.08 ms at config 4) and re-streams the
// 607 KB of bitmaps per 2048-row tile (L2 -> SM ingress).  Here
//  * a row is packed ONCE into 2d+2 bytes (u = k + 2^13 = a + 128 b, limbs a, b
//    < 128, a constant 1 and an out-of-range flag) and stored by its loader
//    thread into TMEM (tcgen05.st): 8 columns hold a 128-row tile, 50 tiles
//    (6400 rows) stay resident in 400 of the 512 columns;
//  * one tcgen05.mma (kind::i8, A from TMEM, B = the base-256 limbs of the
//    per-lattice coefficients z_j 128^p mod M in shared memory) gives, for a
//    128-row tile and a group of 5 lattices, three s32 partial sums per (row,
//    lattice): x = v0 + 256 v1 + 65536 v2 == k.z (mod M), x < 2^32;
//  * the epilogue reduces x with ONE multiply-high (q = umulhi(x, 2^32/M) is
//    floor(x/M) or one less, so x - qM < M + ext with ext = ceil(M x_max /
//    2^32)) and probes a bitmap whose first ext bits are repeated after bit
//    M (roll_extend_kernel writes these once per call);
//  * bitmaps arrive by 1-D bulk copies, one group (5 lattices) per step,
//    double buffered; a step applies its group to every resident tile.  Tiles
//    are organised in NG cohorts (NG = groups per pass): at step s the cohort
//    s mod NG is reborn with fresh rows and every cohort sees the groups in
//    rotated order, so loading, hashing and retiring all overlap and each
//    group of bitmaps is brought in once per ~6400 rows instead of once per
//    2048.
//
// Warp roles (832 threads, one CTA per SM): warp 0 bitmap producer (+ TMEM
// allocation), warp 1 MMA issuer, warps 2-9 row loaders (two per TMEM lane
// quadrant), warps 10-25 epilogue (four groups of four quadrant warps).
#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"
#include "roll_ptx.cuh"

namespace sfftb {

namespace roll {

constexpr int kThreads = 832;
constexpr int kTile = 128;
constexpr int kLG = 5;          // lattices per group (15 of the 16 MMA columns)
constexpr int kNC = 16;         // MMA N
constexpr int kACols = 8;       // TMEM columns of one A tile (K = 32 bytes)
constexpr int kSP = 4;          // tiles per cohort (one per epilogue warp group)
constexpr int kMaxNG = 12;      // 8*4*NG A columns + two 64-column accumulator buffers
constexpr int kLoaders = 8;
constexpr int kEpiWarp0 = 2 + kLoaders;
constexpr int kEpiWarps = 16;
constexpr int64_t kOffset = 8192;  // u = k + kOffset must lie in [0, 2^14)

struct Args {
    const int64_t* elems;
    int64_t n;
    const int64_t* zmat;  // (L, d)
    int d, L, NG;
    uint32_t M, negM, magic;
    const uint32_t* bits;  // (L, W)
    int W;                 // words per lattice in global memory
    const uint32_t* xbits; // (L, Wx) wrap-extended bitmaps (roll_extend_kernel)
    int Wx;
    int ext_words;         // words rewritten/appended from word M >> 5 on
    uint32_t S2;           // shared-memory stride per lattice bitmap (power of two)
    int64_t ntiles;
    int64_t min_hits;
    int64_t* hits64;   // may be null
    uint32_t* detmask;
    unsigned long long* recomputed;
    unsigned int* nbad;  // warps that met a row outside the limb range (this launch)
    int32_t* dbg;  // diagnostics: the 128 x 16 accumulators of tile 0, step 0
    long long* prof;  // diagnostics: cycle counters of CTA 0 (SFFTB_HASH_ROLL_PROF)
};

using namespace rollptx;

// Exact hits of one row from global memory (a coordinate outside the limb range).
__device__ int exact_row_hits(const Args& a, int d, int64_t row) {
    int h = 0;
    for (int l = 0; l < a.L; ++l) {
        uint64_t acc = 0;
        for (int j = 0; j < d; ++j) {
            int64_t e = a.elems[row * d + j] % (int64_t)a.M;
            if (e < 0) e += a.M;
            int64_t z = a.zmat[(int64_t)l * d + j] % (int64_t)a.M;
            if (z < 0) z += a.M;
            acc = (acc + (uint64_t)e * (uint64_t)z) % a.M;
        }
        const uint32_t r = (uint32_t)acc;
        h += (a.bits[(int64_t)l * a.W + (r >> 5)] >> (r & 31)) & 1u;
    }
    return h;
}

// Runs after every hash_roll_kernel launch: exits at once unless the main
// kernel met a row outside the limb range; otherwise finds those rows again
// (same range test), recomputes their hits exactly and repairs hits64 and the
// detected bit.
__global__ void __launch_bounds__(256) roll_fixup_kernel(Args a) {
    if (*reinterpret_cast<volatile unsigned int*>(a.nbad) == 0u) return;
    const int d = a.d;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < a.n;
         row += (int64_t)gridDim.x * blockDim.x) {
        bool bad = false;
        for (int j = 0; j < d; ++j)
            bad |= ((uint64_t)(a.elems[row * d + j] + kOffset) >> 14) != 0;
        if (!bad) continue;
        const int64_t hits = exact_row_hits(a, d, row);
        atomicAdd(a.recomputed, 1ull);
        if (a.hits64) a.hits64[row] = hits;
        const uint32_t bit = 1u << (row & 31);
        if (hits >= a.min_hits) atomicOr(a.detmask + (row >> 5), bit);
        else atomicAnd(a.detmask + (row >> 5), ~bit);
    }
}

// Shared-memory map: byte offsets from the dynamic base (the two bitmap ring
// slots follow at the next S2-aligned address).
struct Smem {
    uint32_t bm_raw, bm_full, bm_empty, d_full, d_empty, a_full, a_empty, tmem_holder;
    uint32_t bop, stage, end;
};
__host__ __device__ inline Smem smem_map(int NG) {
    Smem s;
    uint32_t o = 0;
    s.bm_raw = o;   o += 16;
    s.bm_full = o;  o += 16;
    s.bm_empty = o; o += 16;
    s.d_full = o;   o += 32;
    s.d_empty = o;  o += 32;
    s.a_full = o;   o += 8u * kMaxNG;
    s.a_empty = o;  o += 8u * kMaxNG;
    s.tmem_holder = o; o += 16;
    o = (o + 127u) & ~127u;
    s.bop = o;      o += (uint32_t)NG * 512u;                 // B operand: NG x [2][16][16 B]
    s.stage = o;    o += (uint32_t)kLoaders * 32u * 7u * 4u;  // loader transposition (RS <= 7)
    s.end = (o + 15u) & ~15u;
    return s;
}

#define ROLL_T(acc, ...)                         \
    do {                                         \
        if (PROF) {                              \
            const long long t0_ = clock64();     \
            __VA_ARGS__;                         \
            acc += clock64() - t0_;              \
        } else {                                 \
            __VA_ARGS__;                         \
        }                                        \
    } while (0)

struct Ctx {
    uint32_t raw, tmem;
    int lane, warp, nb, NG;
    int64_t cta, ncta;
};

// Row loader of one warp: lane quadrant q = warp & 3, tiles k = hsel, hsel + 2
// of every birth.  Coalesced 16-byte loads (a coordinate pair each), packed
// to one word per pair, transposed through shared memory to thread-per-row,
// stored into the cohort's A tiles in tensor memory.
template <int D, bool PROF>
__device__ __forceinline__ void run_loader(const Args& a, const Smem& S, const Ctx& x,
                                           uint8_t* smem_raw) {
    constexpr int H = D / 2;   // 16-byte chunks (coordinate pairs) per row
    constexpr int RS = H | 1;  // odd row stride of the transposition buffer
    const int lane = x.lane, q = x.warp & 3, hsel = (x.warp - 2) >> 2;
    const uint32_t raw = x.raw;
    uint32_t* stg = reinterpret_cast<uint32_t*>(smem_raw + S.stage) + (x.warp - 2) * 32 * RS;
    const int4* gbase = reinterpret_cast<const int4*>(a.elems);
    // unit = (birth b, tile k): rows [t*128 + q*32, +32) of tile t = cta + (4b + k) ncta
    auto unit_rows = [&](int b, int k) -> int64_t {
        return ((x.cta + (int64_t)(b * kSP + k) * x.ncta) * kTile + q * 32);
    };
    auto load = [&](int4 (&rawv)[H], int b, int k) {
        const int64_t r0 = unit_rows(b, k);
        const int4* src = gbase + r0 * H + lane;
        if (r0 + 32 <= a.n) {  // the whole unit is inside the set
#pragma unroll
            for (int i = 0; i < H; ++i) rawv[i] = __ldg(src + 32 * i);
        } else {
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const int64_t row = r0 + (lane + 32 * i) / H;
                rawv[i] = row < a.n ? __ldg(src + 32 * i) : make_int4(0, 0, 0, 0);
            }
        }
    };
    // word (row, pair) of chunk lane + 32 i in the transposition buffer
    const uint32_t stg_a = smem_addr(stg);
    uint32_t sdst[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
        const int ch = lane + 32 * i;
        sdst[i] = stg_a + 4u * (uint32_t)((ch / H) * RS + (ch % H));
    }
    auto prefetch = [&](int b, int k) {
        const int64_t r0 = unit_rows(b, k);
        const char* p = reinterpret_cast<const char*>(a.elems) + r0 * (8 * D);
        if (lane * 128 < 32 * 8 * D && r0 + 32 <= a.n) prefetch_l2(p + lane * 128);
    };
    long long pt[2] = {0, 0};
    const long long tstart = clock64();
    // two register buffers, used alternately (no copies): tile hsel of a birth
    // is packed from bufA while tile hsel + 2 loads into bufB, and vice versa
    int4 bufA[H], bufB[H];
    if (x.nb > 0) load(bufA, 0, hsel);
    for (int u = 1; u <= 4; ++u)
        if ((u >> 1) < x.nb) prefetch(u >> 1, hsel + 2 * (u & 1));
    int c = 0, beta = 0;
    auto pack_store = [&](const int4 (&cur)[H], int k, bool first, bool last) {
#pragma unroll
        for (int i = 0; i < H; ++i) {
            // u = k + 2^13 as 64 bits: in range <=> high word 0 and low < 2^14;
            // a + 256 b for u = a + 128 b is u + (u & ~127)
            uint32_t l0, h0, l1, h1;
            asm("add.cc.u32 %0, %2, 8192;\n\taddc.u32 %1, %3, 0;"
                : "=r"(l0), "=r"(h0)
                : "r"(cur[i].x), "r"(cur[i].y));
            asm("add.cc.u32 %0, %2, 8192;\n\taddc.u32 %1, %3, 0;"
                : "=r"(l1), "=r"(h1)
                : "r"(cur[i].z), "r"(cur[i].w));
            const uint32_t p0 = (l0 & 0x3FFFu) + (l0 & 0x3F80u);
            const uint32_t p1 = (l1 & 0x3FFFu) + (l1 & 0x3F80u);
            uint32_t w = (p1 << 16) + p0;
            if ((h0 | h1) | ((l0 | l1) >> 14)) w |= 0x80u;
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(sdst[i]), "r"(w) : "memory");
        }
        __syncwarp();
        uint32_t r[8];
        uint32_t bad = 0;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            if (p < H) {
                const uint32_t w = stg[lane * RS + p];
                bad |= w;
                r[p] = w & ~0x80u;
            } else {
                r[p] = 0u;
            }
        }
        // K = 2D: the constant 1; K = 2D + 1: the out-of-range flag
        if (H < 8) r[H] = 1u + ((bad & 0x80u) << 1);
        __syncwarp();
        if (first && beta >= 1)  // the cohort's previous occupants have retired
            ROLL_T(pt[0], bar_wait(raw + S.a_empty + 8u * c, (uint32_t)((beta - 1) & 1)));
        tc_fence_after();
        ROLL_T(pt[1], tmem_st8(x.tmem + ((uint32_t)(q * 32) << 16) +
                                   (uint32_t)((c * kSP + k) * kACols), r));
        if (last) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(raw + S.a_full + 8u * c);
        }
    };
    for (int b = 0; b < x.nb; ++b) {
        // the next unit's rows are requested before this one is packed
        load(bufB, b, hsel + 2);
        if (b + 3 < x.nb) prefetch(b + 3, hsel);
        pack_store(bufA, hsel, true, false);
        if (b + 1 < x.nb) load(bufA, b + 1, hsel);
        if (b + 3 < x.nb) prefetch(b + 3, hsel + 2);
        pack_store(bufB, hsel + 2, false, true);
        if (++c == x.NG) {
            c = 0;
            ++beta;
        }
    }
    if (PROF && x.cta == 0 && lane == 0 && x.warp == 2) {
        a.prof[16] = pt[0];
        a.prof[17] = pt[1];
        a.prof[19] = clock64() - tstart;
    }
}

// NG = lattice groups per pass = cohorts.  Every step runs the same NG items
// (cohorts 0..NG-1 in index order, four tiles each, accumulator buffer c & 1):
// cohorts not yet born or past the end of the rows are processed as dummies
// (their outputs are never written), so the whole schedule is static.
template <int NG, bool PROF>
__global__ void __launch_bounds__(kThreads, 1) hash_roll_kernel(Args a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t raw = smem_addr(smem_raw);
    const Smem S = smem_map(NG);
    const uint32_t ring0 = (raw + S.end + a.S2 - 1u) & ~(a.S2 - 1u);
    const uint32_t ring_bytes = (uint32_t)kLG * a.S2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cta = blockIdx.x, ncta = gridDim.x;
    const int my_tiles = a.ntiles > cta ? (int)((a.ntiles - 1 - cta) / ncta + 1) : 0;
    const int nb = (my_tiles + kSP - 1) / kSP;  // births
    const int nsteps = nb > 0 ? nb + NG - 1 : 0;
    constexpr int dcol0 = NG * kSP * kACols;
    constexpr int dstride = kNC * kSP;  // accumulator columns of one cohort
    // accumulator buffers: cohort c uses buffer c % ND (static; when NG is not
    // a multiple of ND the step boundary reuses one buffer back to back)
    constexpr int ND = (dcol0 + 3 * dstride <= 512 && NG >= 3) ? 3 : 2;
    const int D = a.d;

    // ---- setup ----
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            bar_init(raw + S.bm_raw + 8u * i, 1);
            bar_init(raw + S.bm_full + 8u * i, 1);
            bar_init(raw + S.bm_empty + 8u * i, kEpiWarps);
        }
        for (int i = 0; i < ND; ++i) {
            bar_init(raw + S.d_full + 8u * i, 1);
            bar_init(raw + S.d_empty + 8u * i, kEpiWarps);
        }
        for (int i = 0; i < NG; ++i) {
            bar_init(raw + S.a_full + 8u * i, kLoaders);
            bar_init(raw + S.a_empty + 8u * i, kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         raw + S.tmem_holder)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // B operand of group g: [2 K-chunks][16 columns][16 B]; column 3i + limb
    // for lattice g*kLG + i, column 15 = the out-of-range flag.  K bytes:
    // 4p + e = coordinate 2p + (e >> 1), limb weight (e & 1) ? 128 : 1;
    // 2D = the constant (k = u - kOffset); 2D + 1 = the flag.
    for (uint32_t e4 = threadIdx.x; e4 < (uint32_t)NG * 128u; e4 += blockDim.x) {
        uint32_t word = 0;
        for (int t = 0; t < 4; ++t) {
            const uint32_t idx = e4 * 4 + t;
            const int g = (int)(idx / 512u);
            const uint32_t in = idx % 512u;
            const int col = (int)((in / 16u) % 16u);
            const int kb = (int)(in / 256u) * 16 + (int)(in % 16u);
            uint32_t v = 0;
            const int i = col / 3, limb = col % 3;
            const int l = g * kLG + i;
            if (col < 3 * kLG && l < a.L) {
                uint64_t c = 0;
                bool have = false;
                if (kb < 2 * D) {
                    int64_t z = a.zmat[(int64_t)l * D + (kb >> 1)] % (int64_t)a.M;
                    if (z < 0) z += a.M;
                    c = ((uint64_t)z * ((kb & 1) ? 128u : 1u)) % a.M;
                    have = true;
                } else if (kb == 2 * D) {
                    uint64_t zs = 0;
                    for (int j = 0; j < D; ++j) {
                        int64_t z = a.zmat[(int64_t)l * D + j] % (int64_t)a.M;
                        if (z < 0) z += a.M;
                        zs += (uint64_t)z;
                    }
                    const uint64_t t2 = ((zs % a.M) * (uint64_t)(kOffset % (int64_t)a.M)) % a.M;
                    c = (a.M - t2) % a.M;
                    have = true;
                }
                if (have) v = (uint32_t)(c >> (8 * limb)) & 255u;
            } else if (col == 15 && kb == 2 * D + 1) {
                v = 1u;
            }
            word |= v << (8 * t);
        }
        *reinterpret_cast<uint32_t*>(smem_raw + S.bop + e4 * 4) = word;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + S.tmem_holder);

    if (warp == 0) {
        // ================= bitmap producer =================
        long long pt[4] = {0, 0, 0, 0};
        const long long tstart = clock64();
        const uint32_t wbytes = (uint32_t)a.Wx * 4u;
        auto issue = [&](int s) {
            const int ring = s & 1;
            const int l0 = (s % NG) * kLG;
            const int cnt = min(a.L, l0 + kLG) - l0;
            if (lane == 0) {
                const uint32_t bar = raw + S.bm_full + 8u * ring;
                bar_expect_tx(bar, wbytes * (uint32_t)cnt);
                for (int i = 0; i < cnt; ++i)
                    bulk_g2s_a(ring0 + (uint32_t)ring * ring_bytes + (uint32_t)i * a.S2,
                               a.xbits + (int64_t)(l0 + i) * a.Wx, wbytes, bar);
            }
        };
        if (nsteps > 0) issue(0);
        if (nsteps > 1) issue(1);
        for (int s = 0; s + 2 < nsteps; ++s) {
            ROLL_T(pt[2], bar_wait(raw + S.bm_empty + 8u * (uint32_t)(s & 1),
                                   (uint32_t)((s >> 1) & 1)));
            issue(s + 2);
        }
        if (PROF && cta == 0 && lane == 0) {
            a.prof[0] = pt[0];
            a.prof[1] = pt[1];
            a.prof[2] = pt[2];
            a.prof[3] = clock64() - tstart;
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        const bool leader = elect_one();
        const uint32_t idesc = (2u << 4) | ((uint32_t)(kNC >> 3) << 17) | ((uint32_t)(kTile >> 4) << 24);
        uint32_t epar[3] = {1u, 1u, 1u};  // parity of the d_empty phase before the next use
        bool used[3] = {false, false, false};
        int sm = 0, beta = 0;
        long long pt[4] = {0, 0, 0, 0};
        const long long tstart = clock64();
        for (int s = 0; s < nsteps; ++s) {
            const uint64_t bdesc = umma_desc(raw + S.bop + (uint32_t)sm * 512u, 256u, 128u);
#pragma unroll
            for (int c = 0; c < NG; ++c) {
                const int buf = c % ND;
                if (used[buf]) ROLL_T(pt[0], bar_wait(raw + S.d_empty + 8u * buf, epar[buf]));
                used[buf] = true;
                epar[buf] ^= 1u;
                if (c == sm && s < nb)  // newborn cohort: its rows are in tensor memory
                    ROLL_T(pt[1], bar_wait(raw + S.a_full + 8u * c, (uint32_t)(beta & 1)));
                tc_fence_after();
                if (leader) {
#pragma unroll
                    for (int k = 0; k < kSP; ++k)
                        umma_i8_ts(tmem + (uint32_t)(dcol0 + dstride * buf + kNC * k),
                                   tmem + (uint32_t)((c * kSP + k) * kACols), bdesc, idesc);
                    umma_commit(raw + S.d_full + 8u * buf);
                }
                __syncwarp();
            }
            if (++sm == NG) {
                sm = 0;
                ++beta;
            }
        }
        if (PROF && cta == 0 && lane == 0) {
            a.prof[8] = pt[0];
            a.prof[9] = pt[1];
            a.prof[11] = clock64() - tstart;
        }
    } else if (warp < kEpiWarp0) {
        // ================= row loaders =================
        Ctx x;
        x.raw = raw;
        x.tmem = tmem;
        x.lane = lane;
        x.warp = warp;
        x.nb = nb;
        x.NG = NG;
        x.cta = cta;
        x.ncta = ncta;
        switch (D) {
            case 4: run_loader<4, PROF>(a, S, x, smem_raw); break;
            case 6: run_loader<6, PROF>(a, S, x, smem_raw); break;
            case 8: run_loader<8, PROF>(a, S, x, smem_raw); break;
            case 10: run_loader<10, PROF>(a, S, x, smem_raw); break;
            case 12: run_loader<12, PROF>(a, S, x, smem_raw); break;
            default: run_loader<14, PROF>(a, S, x, smem_raw); break;
        }
    } else {
        // ================= epilogue =================
        const int ew = warp - kEpiWarp0;
        const int grp = ew >> 2;  // the cohort's tile this warp probes
        const int q = warp & 3;
        const uint32_t negM = a.negM, magic = a.magic;
        uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(dcol0 + kNC * grp);
        asm volatile("" : "+r"(tlane));
        const bool lane0 = lane == 0;
        uint32_t dfull = raw + S.d_full, dempty = raw + S.d_empty;
        asm volatile("" : "+r"(dfull), "+r"(dempty));  // not rematerialised per item
        // running hit counts of this thread's row in every cohort, one byte each
        uint32_t hp[(NG + 3) / 4];
#pragma unroll
        for (int i = 0; i < (NG + 3) / 4; ++i) hp[i] = 0;
        uint32_t par[3] = {0u, 0u, 0u};
        int sm = 0;
        long long pt[4] = {0, 0, 0, 0};
        const long long tstart = clock64();
        uint32_t va[16], vb[16];
        for (int s = 0; s < nsteps; ++s) {
            const int ring = s & 1;
            const int lcg = min(a.L, sm * kLG + kLG) - sm * kLG;
            // pair i's bit ends at position 32 - kLG + i of the accumulator
            const uint32_t lmask = ((1u << lcg) - 1u) << (32 - kLG);
            uint32_t lb[kLG];
#pragma unroll
            for (int i = 0; i < kLG; ++i) {
                uint32_t t = ring0 + (uint32_t)ring * ring_bytes + (uint32_t)i * a.S2;
                asm volatile("" : "+r"(t));  // keep the five slot bases in registers
                lb[i] = t;
            }
            ROLL_T(pt[0], bar_wait(raw + S.bm_full + 8u * ring, (uint32_t)((s >> 1) & 1)));
            // Software pipeline over the step's cohorts: while cohort c is
            // probed (address, shared load, bit), the residues of cohort c + 1
            // are computed and the accumulators of cohort c + 2 are in flight.
            auto residues = [&](const uint32_t (&v)[16], uint32_t (&r)[kLG]) {
                // residues in [0, M + ext): x - umulhi(x, 2^32/M) M
#pragma unroll
                for (int i = 0; i < kLG; ++i) {
                    uint32_t xx = (v[3 * i + 1] << 8) + v[3 * i];
                    xx = (v[3 * i + 2] << 16) + xx;
                    const uint32_t qq = __umulhi(xx, magic);
                    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r[i]) : "r"(qq), "r"(negM), "r"(xx));
                }
            };
            uint32_t rr[2][kLG], flag[2];
            ROLL_T(pt[1], bar_wait(dfull, par[0]));
            par[0] ^= 1u;
            tc_fence_after();
            tmem_ld16_async(tlane, va);
            tmem_wait_ld16(va);
            tc_fence_before();
            __syncwarp();
            if (lane0) bar_arrive(dempty);
            if (NG > 1) {
                ROLL_T(pt[1], bar_wait(dfull + 8u * (1 % ND), par[1 % ND]));
                par[1 % ND] ^= 1u;
                tc_fence_after();
                tmem_ld16_async(tlane + (uint32_t)(dstride * (1 % ND)), vb);
            }
            residues(va, rr[0]);
            flag[0] = va[15];
#pragma unroll
            for (int c = 0; c < NG; ++c) {
                uint32_t(&vc)[16] = (c & 1) ? vb : va;  // cohort c: consumed, reused for c + 2
                uint32_t(&vn)[16] = (c & 1) ? va : vb;  // cohort c + 1: in flight
                const int b1 = (c + 1) % ND, b2 = (c + 2) % ND;
                if (c + 1 < NG) {
                    tmem_wait_ld16(vn);
                    tc_fence_before();
                    __syncwarp();
                    if (lane0) bar_arrive(dempty + 8u * b1);
                }
                if (c + 2 < NG) {
                    ROLL_T(pt[1], bar_wait(dfull + 8u * b2, par[b2]));
                    par[b2] ^= 1u;
                    tc_fence_after();
                    tmem_ld16_async(tlane + (uint32_t)(dstride * b2), vc);
                }
                if (c + 1 < NG) {
                    residues(vn, rr[(c + 1) & 1]);
                    flag[(c + 1) & 1] = vn[15];
                }
                uint32_t w[kLG];
#pragma unroll
                for (int i = 0; i < kLG; ++i) {
                    asm volatile("{\n\t.reg .u32 t;\n\t"
                                 "shr.u32 t, %1, 3;\n\t"
                                 "lop3.b32 t, t, 0xFFFFFFFC, %2, 0xEA;\n\t"
                                 "ld.shared.u32 %0, [t];\n\t}"
                                 : "=r"(w[i])
                                 : "r"(rr[c & 1][i]), "r"(lb[i]));
                }
                uint32_t bacc = 0;
#pragma unroll
                for (int i = 0; i < kLG; ++i)
                    bacc = __funnelshift_r(bacc, __funnelshift_r(w[i], w[i], rr[c & 1][i]), 1);
                hp[c >> 2] += __popc(bacc & lmask) << (8 * (c & 3));
                if (sm == (c + NG - 1) % NG) {  // the cohort born at step s - (NG - 1) retires
                    const int b = s - (NG - 1);
                    const uint32_t hc = (hp[c >> 2] >> (8 * (c & 3))) & 255u;
                    hp[c >> 2] &= ~(255u << (8 * (c & 3)));
                    if (b >= 0) {  // b < nb holds: s < nb + NG - 1
                        const int64_t t = cta + (int64_t)(b * kSP + grp) * ncta;
                        const int64_t row0 = t * kTile + q * 32;
                        const int64_t row = row0 + lane;
                        const bool valid = row < a.n;
                        const int64_t hits = (int64_t)hc;
                        // rows outside the limb range: counted here, redone
                        // exactly by roll_fixup_kernel
                        if (__any_sync(0xffffffffu, flag[c & 1] != 0u && valid) && lane0)
                            atomicAdd(a.nbad, 1u);
                        const unsigned det =
                            __ballot_sync(0xffffffffu, valid && hits >= a.min_hits);
                        if (valid && a.hits64) a.hits64[row] = hits;
                        if (lane0 && row0 < a.n) a.detmask[row0 >> 5] = det;
                        __syncwarp();
                        if (lane0) bar_arrive(raw + S.a_empty + 8u * c);
                    }
                }
            }
            __syncwarp();
            if (lane0) bar_arrive(raw + S.bm_empty + 8u * ring);
            if (++sm == NG) sm = 0;
        }
        if (PROF && cta == 0 && lane == 0 && (ew == 0 || ew == 15)) {
            long long* o = a.prof + (ew == 0 ? 24 : 32);
            o[0] = pt[0];
            o[1] = pt[1];
            o[2] = pt[2];
            o[3] = clock64() - tstart;
        }
    }

    // ---- teardown ----
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                     : "memory");
    }
}

// Keeps freed stream-ordered allocations in the device's default pool across
// synchronisations (release threshold 64 MB) instead of returning them to the
// driver after every call: a cudaMallocAsync after a synchronisation otherwise
// costs ~0.2 ms of host time in front of the kernels.  Once per device.
void keep_async_pool() {
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64)
        std::call_once(once[dev], [dev] {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                unsigned long long thr = 0;
                if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) ==
                        cudaSuccess &&
                    thr < (64ull << 20)) {
                    thr = 64ull << 20;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                }
            }
        });
}

unsigned long long* recomputed_counter() {
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

template <int NG>
static int launch_ng(Args& a, uint32_t smem, int grid, cudaStream_t st) {
    if (NG == 10 && a.prof) {
        auto kp = hash_roll_kernel<10, true>;
        SFFTB_CUDA(smem_opt_in(kp, smem));
        kp<<<grid, kThreads, smem, st>>>(a);
        SFFTB_CHECK_LAUNCH();
        return SFFTB_OK;
    }
    auto kern = hash_roll_kernel<NG, false>;
    SFFTB_CUDA(smem_opt_in(kern, smem));
    kern<<<grid, kThreads, smem, st>>>(a);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

}  // namespace roll

// Returns 1 when the rolling tensor-core kernel handled the call, 0 when the
// shape is outside it (the caller takes the other kernels), < 0 = -status.
int hash_hits_roll(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat, int64_t L,
                   int64_t M, const uint32_t* bits, int64_t min_hits, int64_t* hits64,
                   uint32_t* detmask, cudaStream_t st) {
    using namespace roll;
    {
        // on by default; SFFTB_HASH_ROLL=0 keeps the CUDA-core kernel
        const char* e = getenv("SFFTB_HASH_ROLL");
        if (e && e[0] == '0') return 0;
    }
    const char* mr = getenv("SFFTB_HASH_ROLL_MINROWS");
    // measured break-even against hash_rows at the config-4 shape: ~2^21 rows
    const int64_t min_rows = mr ? atoll(mr) : (int64_t)1 << 21;
    if (n < min_rows || n > ((int64_t)1 << 36) || L < 1 || L > 255 || M < 64 ||
        M >= ((int64_t)1 << 24))
        return 0;
    if (d != 4 && d != 6 && d != 8 && d != 10 && d != 12 && d != 14) return 0;
    if (((uintptr_t)elems & 15) != 0 || ((uintptr_t)bits & 15) != 0) return 0;
    // x = sum of 2d limb products + the constant, must stay below 2^32
    const __int128 xmax = ((__int128)(2 * d) * 127 + 1) * (M - 1);
    if (xmax >= ((__int128)1 << 32)) return 0;
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    // q = umulhi(x, floor(2^32/M)) >= floor(x/M) - 1, and is one short only
    // when x mod M < M x / 2^32: residues land in [0, M + ext)
    const int64_t ext = (int64_t)(((__int128)M * xmax) >> 32) + 2;
    const int64_t ext_words = (ext + 31) / 32 + 1;
    if (ext_words >= (M >> 5)) return 0;
    const int64_t Wx = ((M >> 5) + ext_words + 1 + 3) & ~int64_t(3);
    uint32_t S2 = 64;
    while ((int64_t)S2 < Wx * 4) S2 <<= 1;
    const int NG = (int)((L + kLG - 1) / kLG);
    if (NG > kMaxNG) return 0;
    const Smem S = smem_map(NG);
    const uint32_t smem = S.end + S2 + 2u * kLG * S2;
    static int prop_smem = 0;
    if (prop_smem == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&prop_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (prop_smem <= 0) prop_smem = 232448;
    }
    if (smem > (uint32_t)prop_smem) return 0;
    unsigned long long* rec = recomputed_counter();
    if (!rec) return 0;

    Args a;
    a.elems = elems;
    a.n = n;
    a.zmat = zmat;
    a.d = (int)d;
    a.L = (int)L;
    a.NG = NG;
    a.M = (uint32_t)M;
    a.negM = 0u - (uint32_t)M;
    a.magic = (uint32_t)(((uint64_t)1 << 32) / (uint64_t)M);
    a.bits = bits;
    a.W = (int)W;
    // stream-ordered scratch (reentrant); freed blocks stay in the device's
    // default pool across synchronisations
    keep_async_pool();
    // per-call scratch: the extended bitmaps and, behind them, this call's
    // out-of-range flag (private to the call: concurrent calls on other
    // streams must not share it)
    uint32_t* xbits = nullptr;
    SFFTB_CUDA(cudaMallocAsync(&xbits, ((size_t)L * Wx + 4) * sizeof(uint32_t), st));
    a.xbits = xbits;
    a.Wx = (int)Wx;
    a.nbad = xbits + (size_t)L * Wx;
    SFFTB_CUDA(cudaMemsetAsync(a.nbad, 0, sizeof(unsigned int), st));
    a.ext_words = (int)ext_words;
    a.S2 = S2;
    a.ntiles = (n + kTile - 1) / kTile;
    a.min_hits = min_hits;
    a.hits64 = hits64;
    a.detmask = detmask;
    a.recomputed = rec;
    a.dbg = nullptr;
    static int32_t* dbg = nullptr;
    if (getenv("SFFTB_HASH_ROLL_DUMP") && getenv("SFFTB_HASH_ROLL_PROF")) {
        if (!dbg) SFFTB_CUDA(cudaMalloc(&dbg, 128 * 16 * sizeof(int32_t)));
        SFFTB_CUDA(cudaMemsetAsync(dbg, 0xFF, 128 * 16 * sizeof(int32_t), st));
        a.dbg = dbg;
    }
    a.prof = nullptr;
    static long long* prof = nullptr;
    if (getenv("SFFTB_HASH_ROLL_PROF")) {
        if (!prof) SFFTB_CUDA(cudaMalloc(&prof, 40 * sizeof(long long)));
        SFFTB_CUDA(cudaMemsetAsync(prof, 0, 40 * sizeof(long long), st));
        a.prof = prof;
    }
    int grid = num_sms();
    if (const char* e = getenv("SFFTB_HASH_ROLL_GRID")) grid = std::max(1, atoi(e));
    grid = (int)std::min<int64_t>(grid, a.ntiles);
    if (getenv("SFFTB_HASH_ROLL_DEBUG"))
        fprintf(stderr, "hash_roll: d=%d L=%d NG=%d S2=%u ext_words=%d smem=%u grid=%d\n",
                (int)d, (int)L, NG, S2, (int)ext_words, smem, grid);
    roll_extend_kernel<0><<<(unsigned)((L * Wx + 255) / 256), 256, 0, st>>>(
        bits, (int)L, (int)W, (int)Wx, (uint32_t)M, (int)ext_words, xbits);
    count_launch();
    int rc = SFFTB_EINVAL;
    switch (NG) {
        case 1: rc = launch_ng<1>(a, smem, grid, st); break;
        case 2: rc = launch_ng<2>(a, smem, grid, st); break;
        case 3: rc = launch_ng<3>(a, smem, grid, st); break;
        case 4: rc = launch_ng<4>(a, smem, grid, st); break;
        case 5: rc = launch_ng<5>(a, smem, grid, st); break;
        case 6: rc = launch_ng<6>(a, smem, grid, st); break;
        case 7: rc = launch_ng<7>(a, smem, grid, st); break;
        case 8: rc = launch_ng<8>(a, smem, grid, st); break;
        case 9: rc = launch_ng<9>(a, smem, grid, st); break;
        case 10: rc = launch_ng<10>(a, smem, grid, st); break;
        case 11: rc = launch_ng<11>(a, smem, grid, st); break;
        case 12: rc = launch_ng<12>(a, smem, grid, st); break;
    }
    if (rc == SFFTB_OK) {
        roll_fixup_kernel<<<4 * num_sms(), 256, 0, st>>>(a);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) rc = SFFTB_ECUDA;
    }
    cudaFreeAsync(xbits, st);
    if (a.dbg && rc == SFFTB_OK) {
        static int32_t h[128 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost);
        for (int r : {0, 1, 33, 127}) {
            fprintf(stderr, "roll dbg row %3d:", r);
            for (int i = 0; i < 16; ++i) fprintf(stderr, " %d", h[r * 16 + i]);
            fprintf(stderr, "\n");
        }
    }
    if (a.prof && rc == SFFTB_OK) {
        long long h[40];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "roll prof (cycles, CTA 0): producer raw_wait %lld extend %lld empty_wait %lld total %lld\n",
                h[0], h[1], h[2], h[3]);
        fprintf(stderr, "  mma: d_empty_wait %lld a_full_wait %lld total %lld\n", h[8], h[9], h[11]);
        fprintf(stderr, "  loader w2: a_empty_wait %lld tmem_st %lld total %lld\n", h[16], h[17], h[19]);
        fprintf(stderr, "  epi w0: bm_wait %lld d_full_wait %lld tmem_ld %lld total %lld\n", h[24], h[25], h[26], h[27]);
        fprintf(stderr, "  epi w15: bm_wait %lld d_full_wait %lld tmem_ld %lld total %lld\n", h[32], h[33], h[34], h[35]);
    }
    return rc == SFFTB_OK ? 1 : -rc;
}

}  // namespace sfftb

// Rows the rolling tensor-core hash sent to its exact 64-bit path (a
// coordinate outside [-2^13, 2^13)) since the last reset.
extern "C" int64_t sfftb_hash_roll_recomputed(int reset) {
    unsigned long long* p = sfftb::roll::recomputed_counter();
    if (!p) return -1;
    unsigned long long v = 0;
    if (cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    if (reset) cudaMemset(p, 0, sizeof(v));
    return (int64_t)v;
}
