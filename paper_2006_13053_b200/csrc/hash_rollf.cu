// K3 on the tensor cores, third design: the rolling kernel of hash_roll.cu with
// 8 lattices per group instead of 5 (6 groups cover L <= 48 where it needs 10:
// fewer, larger work items per row), in two modes.  Same semantics as
// hash_rows (hash.cu) / _core.pyx:185-197 (residue, |ghat| > theta probe,
// hits >= nu*L); same rolling schedule, warp roles and wrap-extended bitmaps
// as hash_roll.cu.
//
// fp16 mode -- candidate sets whose coordinates are small (kbound = sum_j
// max|k_j| known and < 2048, the case of the boxes and hyperbolic crosses of the
// reference's workloads): an exact FP16 x FP16 -> FP32 GEMM.
//  * the A operand is the row itself, k_j as signed fp16 (exact for |k_j| <
//    2048), K = 16 = d coordinates + three constant slots (2048, 2048, 1);
//  * the 17-bit coefficients z_j mod M are split in TWO limbs c = c0 + 2^s c1
//    (both exact in fp16), so a lattice takes two accumulator columns instead
//    of three and a 16-column tile serves 8 lattices;
//  * the constant slots seed every accumulator with 1.5 * 2^23 (+ kbound * M
//    split over the two limbs, so x' = k.z + kbound M >= 0): the FP32 result
//    lies in [2^23, 2^24), where its bit pattern is 0x4B000000 + integer.  The
//    second limb's seed carries one more constant chosen so that
//        x' = bits1 * 2^s + bits0   (mod 2^32)
//    exactly: ONE integer multiply-add combines the limbs straight from the raw
//    accumulator bits (the byte kernel needs two).  Every partial sum is an
//    integer below 2^24, so the FP32 accumulation is exact in any order.
// Byte modes -- coordinates in [-2^13, 2^13), any kbound (see hash_rollf_kernel):
// byte limbs of the rows against THREE base-256 limbs of the coefficients (kind::i8,
// N = 24), or -- the default when every lattice has a multiplier t with all its
// coefficients t c mod M below 2^16 -- TWO limbs on the residues scaled by t against
// bitmaps permuted to match (N = 16, the fp16 mode's pipeline).  The three-limb
// kernel is bound by its tensor-memory reads (12 B per pair at 63 of 64 B/clk), the
// two-limb kernel by the shared-memory data pipe (the random bitmap probes).
//
// Both modes:
//  * two cohorts are born per step (12 cohorts of 4 tiles for 6 groups: 6144
//    rows resident in 384 TMEM columns, accumulator buffers behind them);
//  * a group's 8 bitmaps sit in 13 824-byte slots, two buffers (see Smem); a
//    probe address is ((r >> 3) & 0x3FFC) | buffer offset with the slot and
//    the window base as the load's immediate, which also bounds the address
//    for any accumulator content;
//  * the bitmap words of cohort c + 1 are requested before the bits of cohort
//    c are counted;
//  * rows outside the mode's range are flagged by the loaders (one vote per 32
//    rows) and redone exactly by rollf_fixup_kernel.
// Per (row, lattice) the epilogue issues IMAD (limbs; two with three limbs),
// IMAD.HI + IMAD (reduction), SHF + LOP3 (address), LDS, 2 funnel shifts.
#include <stdio.h>
#include <stdlib.h>

#include <cuda_fp16.h>

#include <atomic>
#include <mutex>

#include "common.cuh"
#include "roll_ptx.cuh"

namespace sfftb {

namespace rollf {

using namespace rollptx;

constexpr int kThreads = 832;
constexpr int kTile = 128;
constexpr int kLG = 8;          // lattices per group (two accumulator columns each)
constexpr int kNC = 16;         // MMA N, fp16 mode: 8 lattices x 2 limbs
constexpr int kNCW = 24;        // MMA N, byte mode: 8 lattices x 3 limbs
constexpr int64_t kOffsetW = 8192;  // byte mode: u = k + kOffsetW must lie in [0, 2^14)
constexpr int kACols = 8;       // TMEM columns of one A tile (K = 16 halves)
constexpr int kSP = 4;          // tiles per cohort (one per epilogue warp group)
constexpr int kBPS = 2;         // cohorts born per step
constexpr int kMaxNG = 6;
constexpr int kLoaders = 8;
constexpr int kEpiWarp0 = 2 + kLoaders;
constexpr int kEpiWarps = 16;
constexpr uint32_t kSlot = 13824;           // bytes per lattice bitmap slot (M + ext <= 110592 bits)
constexpr uint32_t kBuf = kLG * kSlot;      // one ring buffer: a group of 8 bitmaps
constexpr uint32_t kBufStride = 0x1C000u;   // buffer 1 starts here (low 14 bits zero: OR-able)
constexpr int kRing = 2;
constexpr int32_t kCoordLim = 2048;         // |k_j| < kCoordLim (fp16-exact)
constexpr uint32_t kSeedBits = 0x4B400000u; // float bits of 1.5 * 2^23

struct Args {
    const int64_t* elems;
    int64_t n;
    const int64_t* zmat;  // (L, d)
    int d, L, NG;
    uint32_t M, negM, magic;
    int wide;              // byte mode (see hash_rollf_kernel)
    // scaled byte mode: per-lattice multipliers t (0 = none), their inverses, and the
    // number of lattices that have one (the two-limb kernel runs when it equals L,
    // the three-limb kernel when it does not)
    const uint32_t* tmul;
    const uint32_t* tinv;
    const unsigned int* nfound;
    unsigned long long* scaled_runs;  // launches the two-limb kernel served (persistent counter)
    int s;                 // limb split: c = c0 + 2^s c1
    uint32_t pow2s;
    // B-operand constants of the seed slots (A = 2048, 2048, 1), per limb
    uint32_t seed0[3], seed1[3];
    const uint32_t* bits;  // (L, W)
    int W;
    const uint32_t* xbits; // (L, Wx) wrap-extended bitmaps
    int Wx;
    int64_t ntiles;
    int64_t min_hits;
    int64_t* hits64;   // may be null
    uint32_t* detmask;
    unsigned long long* recomputed;
    unsigned int* nbad;  // warps that met a coordinate outside (-2048, 2048)
    uint32_t* dbg;       // diagnostics: raw accumulators of tile 0, step 0
};

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

// Runs after every launch: exits at once unless a loader met a coordinate
// outside the fp16 range; otherwise redoes those rows exactly.
__global__ void __launch_bounds__(256) rollf_fixup_kernel(Args a) {
    const unsigned int nbad = *reinterpret_cast<volatile unsigned int*>(a.nbad);
    if (nbad == 0u) return;
    const int d = a.d;
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < a.n;
         row += (int64_t)gridDim.x * blockDim.x) {
        bool bad = (nbad & 0x80000000u) != 0u;  // the main kernel did not run
        for (int j = 0; j < d; ++j)
            bad |= a.wide ? ((uint64_t)(a.elems[row * d + j] + kOffsetW) >> 14) != 0
                          : ((uint64_t)(a.elems[row * d + j] + kCoordLim) >> 12) != 0;
        if (!bad) continue;
        const int64_t hits = exact_row_hits(a, d, row);
        atomicAdd(a.recomputed, 1ull);
        if (a.hits64) a.hits64[row] = hits;
        const uint32_t bit = 1u << (row & 31);
        if (hits >= a.min_hits) atomicOr(a.detmask + (row >> 5), bit);
        else atomicAnd(a.detmask + (row >> 5), ~bit);
        // the main kernel did not write the mask: clear the bits past the last row
        if ((nbad & 0x80000000u) && row == a.n - 1 && (a.n & 31))
            atomicAnd(a.detmask + (row >> 5), (1u << (a.n & 31)) - 1u);
    }
}

// x mod M for x < 2^63 with magic = floor(2^64 / M): one multiply-high, one
// multiply-subtract, one correction.
__device__ __forceinline__ uint32_t mod_magic(uint64_t x, uint32_t M, uint64_t magic) {
    const uint64_t q = __umul64hi(x, magic);
    uint64_t r = x - q * M;
    if (r >= M) r -= M;
    return (uint32_t)r;
}

constexpr int kTSplit = 16;  // blocks per lattice in the multiplier search

// Scaled byte mode, step 1a: the smallest multiplier t of lattice l = blockIdx.x
// with t c mod M < 2^16 for all 2d + 1 byte-mode coefficients c (the same
// values hash_rollf_kernel's B-operand setup computes).  blockIdx.y splits the
// range of t; tbest[l] (preset to 0xFFFFFFFF) takes the minimum.
__global__ void __launch_bounds__(256) rollf_tsearch_kernel(const int64_t* __restrict__ zmat,
                                                            int D, uint32_t M, uint64_t magic,
                                                            uint32_t* __restrict__ tbest) {
    __shared__ uint32_t c[32];
    const int l = blockIdx.x, nc = 2 * D + 1;
    if ((int)threadIdx.x < nc) {
        const int kb = threadIdx.x;
        uint64_t v;
        if (kb < 2 * D) {
            int64_t z = zmat[(int64_t)l * D + (kb >> 1)] % (int64_t)M;
            if (z < 0) z += M;
            v = ((uint64_t)z * ((kb & 1) ? 128u : 1u)) % M;
        } else {
            uint64_t zs = 0;
            for (int j = 0; j < D; ++j) {
                int64_t z = zmat[(int64_t)l * D + j] % (int64_t)M;
                if (z < 0) z += M;
                zs += (uint64_t)z;
            }
            const uint64_t t2 = ((zs % M) * (uint64_t)(kOffsetW % (int64_t)M)) % M;
            v = (M - t2) % M;
        }
        c[kb] = (uint32_t)v;
    }
    __syncthreads();
    const uint32_t chunk = (M + kTSplit - 1) / kTSplit;
    const uint32_t t0 = max(1u, blockIdx.y * chunk), t1 = min(M, (blockIdx.y + 1) * chunk);
    uint32_t mine = 0xFFFFFFFFu;
    const volatile uint32_t* best = tbest + l;
    for (uint32_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
        if (t >= *best) break;  // a smaller multiplier is known: the minimum is not here
        bool ok = true;
        for (int j = 0; j < nc && ok; ++j) ok = mod_magic((uint64_t)t * c[j], M, magic) < 65536u;
        if (ok) {
            mine = t;
            break;
        }
    }
    if (mine != 0xFFFFFFFFu) atomicMin(tbest + l, mine);
}

// Step 1b (one thread per lattice): the inverse of the multiplier mod M;
// tmul[l] = 0 when there is no multiplier or it is not invertible (composite
// M); *nfound counts the lattices that have one.
__global__ void rollf_tfinish_kernel(int L, uint32_t M, uint32_t* __restrict__ tmul,
                                     uint32_t* __restrict__ tinv, unsigned int* nfound) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= L) return;
    uint32_t t = tmul[l], inv = 0;
    if (t != 0xFFFFFFFFu) {
        int64_t r0 = M, r1 = t, s0 = 0, s1 = 1;  // extended Euclid
        while (r1 != 0) {
            const int64_t q = r0 / r1;
            const int64_t r2 = r0 - q * r1;
            r0 = r1;
            r1 = r2;
            const int64_t s2 = s0 - q * s1;
            s0 = s1;
            s1 = s2;
        }
        if (r0 == 1) {
            inv = (uint32_t)(((s0 % (int64_t)M) + (int64_t)M) % (int64_t)M);
            if (((uint64_t)inv * t) % M != 1u) inv = 0;
        }
    }
    const bool have = inv != 0;
    tmul[l] = have ? t : 0u;
    tinv[l] = inv;
    if (have) atomicAdd(nfound, 1u);
}

// Scaled byte mode, step 2: the wrap-extended bitmaps (roll_extend_kernel's
// layout).  When every lattice has a multiplier they are PERMUTED: bit p of
// lattice l is bit (tinv[l] (p mod M)) mod M of the input, so that the probe of
// the scaled residue t r mod M finds the bit of r.  One thread per output word.
__global__ void __launch_bounds__(256) rollf_extend_kernel(const uint32_t* __restrict__ bits,
                                                           int L, int W, int Wx, uint32_t M,
                                                           uint64_t magic, int ext_words,
                                                           const uint32_t* __restrict__ tinv,
                                                           const unsigned int* __restrict__ nfound,
                                                           uint32_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L * Wx) return;
    const int l = i / Wx, w = i % Wx;
    const uint32_t* bm = bits + (int64_t)l * W;
    const bool two = *nfound == (unsigned int)L;
    const uint32_t inv = two ? tinv[l] : 1u;
    const uint32_t lim = ((M >> 5) + (uint32_t)ext_words + 1u) * 32u;  // bits the kernels may probe
    uint32_t v = 0;
    const uint32_t p0 = 32u * (uint32_t)w;
    // q = p mod M and r = inv q mod M, advanced by additions (lim < 2 M)
    uint32_t q = p0 >= M ? p0 - M : p0;
    uint32_t r = mod_magic((uint64_t)inv * q, M, magic);
    for (int b = 0; b < 32 && p0 + (uint32_t)b < lim; ++b) {
        v |= ((bm[r >> 5] >> (r & 31u)) & 1u) << b;
        if (++q == M) {
            q = 0;
            r = 0;
        } else {
            r += inv;
            if (r >= M) r -= M;
        }
    }
    out[i] = v;
}

// Shared-memory map: byte offsets from the dynamic base.
//   [0, 110592)        bitmap buffer 0 (8 slots of 13824 B)
//   [110592, 114688)   barriers, TMEM address, B operands (the gap up to kBufStride)
//   [114688, 225280)   bitmap buffer 1
//   [225280, 232448)   loader transposition buffers
// = the 227 KB a CTA can have.  A probe offset is masked to 16 KB, so a
// residue computed from a garbage accumulator (a row outside the fp16 range)
// can read up to 2.5 KB past its 13.5 KB slot: from the last slot of a buffer
// that lands in the tables behind it, never outside the CTA's window.
struct Smem {
    uint32_t bm_full, bm_empty, d_full, d_empty, a_full, a_empty, tmem_holder;
    uint32_t bop, stage, end;
};
__host__ __device__ inline Smem smem_map(int NG) {
    Smem s;
    uint32_t o = kBuf;
    s.bm_full = o;  o += 8u * kRing;
    s.bm_empty = o; o += 8u * kRing;
    s.d_full = o;   o += 32;
    s.d_empty = o;  o += 32;
    s.a_full = o;   o += 8u * kMaxNG * kBPS;
    s.a_empty = o;  o += 8u * kMaxNG * kBPS;
    s.tmem_holder = o; o += 16;
    o = (o + 127u) & ~127u;
    s.bop = o;      o += (uint32_t)kMaxNG * 512u;  // B operand: NG x [2][16][16 B]
    (void)NG;  // byte mode (768 B per group): groups 0-3 here, 4-5 behind the loader buffers
    s.stage = kBufStride + kBuf;                   // loader transposition (RS <= 7)
    s.end = s.stage + (uint32_t)kLoaders * 32u * 7u * 4u;
    return s;
}
static_assert(kBuf + 512u + kMaxNG * 512u <= kBufStride, "tables fit the gap between the buffers");
static_assert(kBuf + 512u + 4u * 768u <= kBufStride, "byte-mode B operands of groups 0-3 fit the gap");
// byte mode is limited to d <= 10 (RS = 5): its loaders use 5120 B, groups 4-5 follow
__host__ __device__ inline uint32_t bop_wide(const Smem& S, int g) {
    return g < 4 ? S.bop + (uint32_t)g * 768u
                 : S.stage + (uint32_t)kLoaders * 32u * 5u * 4u + (uint32_t)(g - 4) * 768u;
}
static_assert(kBuf % 16u == 0 && (kBufStride & 0x3FFFu) == 0, "buffer alignment");
static_assert((kLG - 1) * kSlot + 16384u <= kBufStride, "probe overrun of buffer 0 stays in the gap");
static_assert((kLG - 1) * kSlot + 16384u <= kBuf + kLoaders * 32u * 7u * 4u,
              "probe overrun of buffer 1 stays in the loader buffers");

struct Ctx {
    uint32_t raw, tmem;
    int lane, warp, nb, NG;
    int64_t cta, ncta;
};

__device__ __forceinline__ uint32_t half_bits(float v) {
    return (uint32_t)__half_as_ushort(__float2half_rn(v));
}

// Bitmap word of residue r in slot I of the ring buffer at byte offset boff
// (0 or kBufStride) of the dynamic window: the mask keeps the offset below
// 16 KB for any r (see Smem).  SHF + LOP3 + LDS with the window base and the
// slot as the load's immediate: the dynamic shared memory of a kernel without
// static shared memory starts at address kWin of the shared window (the
// compiler itself materialises that constant); the kernel checks it and
// leaves the whole call to the exact follow-up kernel if it ever differs.
constexpr uint32_t kWin = 0x400u;
constexpr unsigned int kAllRows = 0x80000000u;
template <int I>
__device__ __forceinline__ uint32_t probe(uint32_t r, uint32_t boff) {
    uint32_t w;
    asm volatile("{\n\t.reg .u32 t;\n\t"
                 "shr.u32 t, %1, 3;\n\t"
                 "lop3.b32 t, t, 0x3FFC, %2, 0xEA;\n\t"
                 "ld.shared.u32 %0, [t+%3];\n\t}"
                 : "=r"(w)
                 : "r"(r), "r"(boff), "n"(kWin + I * kSlot));
    return w;
}

// Row loader of one warp: lane quadrant q = warp & 3, tiles k = hsel, hsel + 2
// of both cohorts of every birth.  Coalesced 16-byte loads (a coordinate pair
// each), converted to an fp16 pair, transposed through shared memory to
// thread-per-row, stored into the cohort's A tiles in tensor memory.
template <int D, bool WIDE>
__device__ __forceinline__ void run_loader(const Args& a, const Smem& S, const Ctx& x,
                                           uint8_t* smem_raw) {
    constexpr int H = D / 2;   // 16-byte chunks (coordinate pairs) per row
    constexpr int RS = H | 1;  // odd row stride of the transposition buffer
    static_assert(H + 2 <= 8, "d + 3 constant slots must fit K = 16");
    const int lane = x.lane, q = x.warp & 3, hsel = (x.warp - 2) >> 2;
    const uint32_t raw = x.raw;
    uint32_t* stg = reinterpret_cast<uint32_t*>(smem_raw + S.stage) + (x.warp - 2) * 32 * RS;
    const int4* gbase = reinterpret_cast<const int4*>(a.elems);
    // unit u of birth b: cohort j = u >> 1, tile k = hsel + 2 (u & 1); rows
    // [t*128 + q*32, +32) of tile t = cta + ((b kBPS + j) kSP + k) ncta
    auto unit_rows = [&](int b, int u) -> int64_t {
        const int j = u >> 1, k = hsel + 2 * (u & 1);
        return ((x.cta + (int64_t)((b * kBPS + j) * kSP + k) * x.ncta) * kTile + q * 32);
    };
    auto load = [&](int4 (&rawv)[H], int b, int u) {
        const int64_t r0 = unit_rows(b, u);
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
    const uint32_t stg_a = smem_addr(stg);
    uint32_t sdst[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
        const int ch = lane + 32 * i;
        sdst[i] = stg_a + 4u * (uint32_t)((ch / H) * RS + (ch % H));
    }
    auto prefetch = [&](int b, int u) {
        const int64_t r0 = unit_rows(b, u);
        const char* p = reinterpret_cast<const char*>(a.elems) + r0 * (8 * D);
        if (lane * 128 < 32 * 8 * D && r0 + 32 <= a.n) prefetch_l2(p + lane * 128);
    };
    int c0 = 0, beta = 0;  // first cohort of the current birth slot, its generation
    auto pack_store = [&](const int4 (&cur)[H], int u) {
        uint32_t bad = 0;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            uint32_t l0, h0, l1, h1, w;
            if (WIDE) {
                // u = k + 2^13 as 64 bits: in range <=> high word 0 and low < 2^14;
                // a + 256 b for u = a + 128 b is u + (u & ~127): bytes a0 b0 a1 b1
                asm("add.cc.u32 %0, %2, 8192;\n\taddc.u32 %1, %3, 0;"
                    : "=r"(l0), "=r"(h0)
                    : "r"(cur[i].x), "r"(cur[i].y));
                asm("add.cc.u32 %0, %2, 8192;\n\taddc.u32 %1, %3, 0;"
                    : "=r"(l1), "=r"(h1)
                    : "r"(cur[i].z), "r"(cur[i].w));
                bad |= (h0 | h1) | ((l0 | l1) >> 14);
                // (no mask on u: a row outside the range is flagged and redone, and
                // its garbage stays in its own lane of tensor memory)
                const uint32_t p0 = l0 + (l0 & 0x3F80u);
                const uint32_t p1 = l1 + (l1 & 0x3F80u);
                w = (p1 << 16) + p0;
            } else {
                // in range <=> k + 2048 as 64 bits < 4096
                asm("add.cc.u32 %0, %2, 2048;\n\taddc.u32 %1, %3, 0;"
                    : "=r"(l0), "=r"(h0)
                    : "r"(cur[i].x), "r"(cur[i].y));
                asm("add.cc.u32 %0, %2, 2048;\n\taddc.u32 %1, %3, 0;"
                    : "=r"(l1), "=r"(h1)
                    : "r"(cur[i].z), "r"(cur[i].w));
                bad |= (h0 | h1) | ((l0 | l1) >> 12);
                const __half2 hh = __floats2half2_rn((float)cur[i].x, (float)cur[i].z);
                w = *reinterpret_cast<const uint32_t*>(&hh);
            }
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(sdst[i]), "r"(w) : "memory");
        }
        if (__any_sync(0xffffffffu, bad != 0u)) {  // also orders the stores (warp-convergent)
            if (lane == 0) atomicAdd(a.nbad, 1u);
        }
        __syncwarp();
        uint32_t r[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) r[p] = p < H ? stg[lane * RS + p] : 0u;
        if (WIDE) {
            r[H] = 1u;  // byte K = 2D: the constant 1 (k = u - 2^13)
        } else {
            r[H] = 0x68006800u;      // K = D, D + 1: the constants 2048, 2048
            r[H + 1] = 0x00003C00u;  // K = D + 2: the constant 1
        }
        __syncwarp();
        const int c = c0 + (u >> 1);
        if (!(u & 1) && beta >= 1)  // the cohort's previous occupants have retired
            bar_wait(raw + S.a_empty + 8u * c, (uint32_t)((beta - 1) & 1));
        tc_fence_after();
        const int k = hsel + 2 * (u & 1);
        tmem_st8(x.tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((c * kSP + k) * kACols), r);
        if (u & 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(raw + S.a_full + 8u * c);
        }
    };
    // two register buffers used alternately: unit u packs from one while unit
    // u + 1 loads into the other
    int4 bufA[H], bufB[H];
    if (x.nb > 0) load(bufA, 0, 0);
    for (int v = 1; v <= 8; ++v)
        if ((v >> 2) < x.nb) prefetch(v >> 2, v & 3);
    for (int b = 0; b < x.nb; ++b) {
        load(bufB, b, 1);
        if (b + 2 < x.nb) prefetch(b + 2, 1);
        pack_store(bufA, 0);
        load(bufA, b, 2);
        if (b + 2 < x.nb) prefetch(b + 2, 2);
        pack_store(bufB, 1);
        load(bufB, b, 3);
        if (b + 2 < x.nb) prefetch(b + 2, 3);
        pack_store(bufA, 2);
        if (b + 1 < x.nb) load(bufA, b + 1, 0);
        if (b + 3 < x.nb) prefetch(b + 3, 0);
        pack_store(bufB, 3);
        c0 += kBPS;
        if (c0 == x.NG * kBPS) {
            c0 = 0;
            ++beta;
        }
    }
}

// NG = lattice groups per pass; NCH = kBPS * NG cohorts.  Every step runs the
// same NCH items (cohorts in index order, four tiles each, accumulator buffer
// c % ND): cohorts not yet born or past the end of the rows are processed as
// dummies (their outputs are never written), so the schedule is static.
//
// WIDE = byte mode for coordinates in [-2^13, 2^13) (any kbound), the limb
// scheme of hash_roll.cu on this kernel's schedule: u = k + 2^13 = a + 128 b
// packed as bytes, tcgen05 kind::i8 with THREE base-256 limbs per lattice
// (N = 24 for the same 8 lattices per group), x = v0 + 256 v1 + 65536 v2.
// The 24-column accumulators leave room for two HALF-cohort buffers (tiles
// 0-1 and 2-3: 2 x 48 columns behind the 384 A columns); epilogue warp groups
// 0-1 and 2-3 each wait on their own buffer, loaded one cohort ahead.
//
// MODE 2 = scaled byte mode: when every lattice has a multiplier t with all its
// 2d + 1 byte-limb coefficients t c mod M below 2^16 (rollf_tsearch_kernel: ~7
// such t per lattice at d = 10, M ~ 1e5), the residues t (k.z) mod M -- a
// permutation of the true ones, the bitmaps are permuted to match
// (rollf_extend_kernel) -- need only TWO limbs: N = 16, 8 bytes of accumulator
// per pair instead of 12, and the fp16 mode's pipeline.  Both byte kernels are
// launched; each returns at once unless it is the one to run (Args::nfound).
template <int NG, int MODE>
__global__ void __launch_bounds__(kThreads, 1) hash_rollf_kernel(Args a) {
    constexpr bool WIDE = MODE == 1;    // three limbs, half-cohort accumulator buffers
    constexpr bool LOADW = MODE != 0;   // byte-limb rows
    extern __shared__ __align__(16) uint8_t smem_raw[];
    constexpr int NCH = NG * kBPS;
    const uint32_t raw = smem_addr(smem_raw);
    const Smem S = smem_map(NG);
    const uint32_t ring0 = raw;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cta = blockIdx.x, ncta = gridDim.x;
    const int my_tiles = a.ntiles > cta ? (int)((a.ntiles - 1 - cta) / ncta + 1) : 0;
    const int nb = (my_tiles + kSP * kBPS - 1) / (kSP * kBPS);  // births (kBPS cohorts each)
    const int nsteps = nb > 0 ? nb + NG - 1 : 0;
    constexpr int dcol0 = NCH * kSP * kACols;
    // fp16 mode: ND buffers of one cohort's accumulators (4 tiles x 16 columns);
    // byte mode: 2 buffers of half a cohort's (2 tiles x 24 columns)
    constexpr int dstride = WIDE ? kNCW * 2 : kNC * kSP;
    constexpr int ND = WIDE ? 2 : ((dcol0 + 3 * dstride <= 512) ? 3 : 2);
    static_assert(dcol0 + ND * dstride <= 512, "tensor memory");
    const int D = a.d;
    if (MODE != 0 && a.nfound) {  // which byte kernel serves this call
        const bool two = *a.nfound == (unsigned int)a.L;
        if (two != (MODE == 2)) return;
        if (MODE == 2 && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.scaled_runs, 1ull);
    }
    if (raw != kWin) {  // see probe(): never on current toolchains; exact path for every row
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(a.nbad, kAllRows);
        return;
    }

    // ---- setup ----
    if (threadIdx.x == 0) {
        for (int i = 0; i < kRing; ++i) {
            bar_init(raw + S.bm_full + 8u * i, 1);
            bar_init(raw + S.bm_empty + 8u * i, kEpiWarps);
        }
        for (int i = 0; i < ND; ++i) {
            bar_init(raw + S.d_full + 8u * i, 1);
            bar_init(raw + S.d_empty + 8u * i, WIDE ? kEpiWarps / 2 : kEpiWarps);
        }
        for (int i = 0; i < NCH; ++i) {
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
    if (WIDE) {
        // B operand of group g: [2 K-chunks][24 columns][16 B]; column 3i + limb for
        // lattice g*kLG + i.  K bytes: 4p + e = coordinate 2p + (e >> 1), limb
        // weight (e & 1) ? 128 : 1; 2D = the constant (k = u - 2^13).
        for (uint32_t e = threadIdx.x; e < (uint32_t)NG * 768u; e += blockDim.x) {
            const int g = (int)(e / 768u);
            const uint32_t in = e % 768u;
            const int col = (int)((in / 16u) % 24u);
            const int kb = (int)(in / 384u) * 16 + (int)(in % 16u);
            const int i = col / 3, limb = col % 3;
            const int l = g * kLG + i;
            uint32_t v = 0;
            if (l < a.L) {
                uint64_t c = 0;
                if (kb < 2 * D) {
                    int64_t z = a.zmat[(int64_t)l * D + (kb >> 1)] % (int64_t)a.M;
                    if (z < 0) z += a.M;
                    c = ((uint64_t)z * ((kb & 1) ? 128u : 1u)) % a.M;
                } else if (kb == 2 * D) {
                    uint64_t zs = 0;
                    for (int j = 0; j < D; ++j) {
                        int64_t z = a.zmat[(int64_t)l * D + j] % (int64_t)a.M;
                        if (z < 0) z += a.M;
                        zs += (uint64_t)z;
                    }
                    const uint64_t t2 = ((zs % a.M) * (uint64_t)(kOffsetW % (int64_t)a.M)) % a.M;
                    c = (a.M - t2) % a.M;
                }
                v = (uint32_t)(c >> (8 * limb)) & 255u;
            }
            smem_raw[bop_wide(S, g) + in] = (uint8_t)v;
        }
    } else if (MODE == 2) {
        // [2 K-chunks][16 columns][16 B]; column 2i + limb for lattice g*kLG + i; the
        // coefficients of the byte mode times the lattice's multiplier, < 2^16
        for (uint32_t e = threadIdx.x; e < (uint32_t)NG * 512u; e += blockDim.x) {
            const int g = (int)(e / 512u);
            const uint32_t in = e % 512u;
            const int col = (int)((in / 16u) % 16u);
            const int kb = (int)(in / 256u) * 16 + (int)(in % 16u);
            const int i = col >> 1, limb = col & 1;
            const int l = g * kLG + i;
            uint32_t v = 0;
            if (l < a.L && kb <= 2 * D) {
                uint64_t c = 0;
                if (kb < 2 * D) {
                    int64_t z = a.zmat[(int64_t)l * D + (kb >> 1)] % (int64_t)a.M;
                    if (z < 0) z += a.M;
                    c = ((uint64_t)z * ((kb & 1) ? 128u : 1u)) % a.M;
                } else {
                    uint64_t zs = 0;
                    for (int j = 0; j < D; ++j) {
                        int64_t z = a.zmat[(int64_t)l * D + j] % (int64_t)a.M;
                        if (z < 0) z += a.M;
                        zs += (uint64_t)z;
                    }
                    const uint64_t t2 = ((zs % a.M) * (uint64_t)(kOffsetW % (int64_t)a.M)) % a.M;
                    c = (a.M - t2) % a.M;
                }
                c = (c * (uint64_t)a.tmul[l]) % a.M;  // < 2^16 by the search
                v = (uint32_t)(c >> (8 * limb)) & 255u;
            }
            smem_raw[S.bop + e] = (uint8_t)v;
        }
    } else {
        // B operand of group g: [2 K-chunks][16 columns][8 halves]; column 2i +
        // limb for lattice g*kLG + i.  K index kb: < D the coordinate, D and D + 1
        // the 2048 slots, D + 2 the unit slot.
        for (uint32_t e = threadIdx.x; e < (uint32_t)NG * 256u; e += blockDim.x) {
            const int g = (int)(e / 256u);
            const uint32_t in = e % 256u;
            const int col = (int)((in / 8u) % 16u);
            const int kb = (int)(in / 128u) * 8 + (int)(in % 8u);
            const int i = col >> 1, limb = col & 1;
            const int l = g * kLG + i;
            float v = 0.f;
            if (l < a.L) {
                if (kb < D) {
                    int64_t z = a.zmat[(int64_t)l * D + kb] % (int64_t)a.M;
                    if (z < 0) z += a.M;
                    const uint32_t c = (uint32_t)z;
                    v = (float)(limb ? (c >> a.s) : (c & (a.pow2s - 1u)));
                } else if (kb < D + 3) {
                    v = (float)(limb ? a.seed1[kb - D] : a.seed0[kb - D]);
                }
            }
            reinterpret_cast<uint16_t*>(smem_raw + S.bop)[e] = (uint16_t)half_bits(v);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + S.tmem_holder);

    if (warp == 0) {
        // ================= bitmap producer =================
        const uint32_t wbytes = (uint32_t)a.Wx * 4u;
        auto issue = [&](int s) {
            const int ring = s & 1;
            const int l0 = (s % NG) * kLG;
            const int cnt = min(a.L, l0 + kLG) - l0;
            if (lane == 0) {
                const uint32_t bar = raw + S.bm_full + 8u * ring;
                bar_expect_tx(bar, wbytes * (uint32_t)cnt);
                for (int i = 0; i < cnt; ++i)
                    bulk_g2s_a(ring0 + (uint32_t)ring * kBufStride + (uint32_t)i * kSlot,
                               a.xbits + (int64_t)(l0 + i) * a.Wx, wbytes, bar);
            }
        };
        if (nsteps > 0) issue(0);
        if (nsteps > 1) issue(1);
        for (int s = 0; s + 2 < nsteps; ++s) {
            bar_wait(raw + S.bm_empty + 8u * (uint32_t)(s & 1), (uint32_t)((s >> 1) & 1));
            issue(s + 2);
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        const bool leader = elect_one();
        // kind::f16: D = f32 (1 << 4), A = B = f16 (0); kind::i8: D = s32 (2 << 4),
        // A = B = u8 (0); K-major, N >> 3, M >> 4
        constexpr int NCOL = WIDE ? kNCW : kNC;
        const uint32_t idesc = ((MODE ? 2u : 1u) << 4) | ((uint32_t)(NCOL >> 3) << 17) |
                               ((uint32_t)(kTile >> 4) << 24);
        uint32_t epar[3] = {1u, 1u, 1u};
        bool used[3] = {false, false, false};
        int sm = 0, beta = 0;
        for (int s = 0; s < nsteps; ++s) {
            const uint64_t bdesc =
                WIDE ? umma_desc(raw + bop_wide(S, sm), 384u, 128u)
                     : umma_desc(raw + S.bop + (uint32_t)sm * 512u, 256u, 128u);
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (WIDE) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {  // tiles 2h, 2h + 1 into half buffer h
                        if (used[h]) bar_wait(raw + S.d_empty + 8u * h, epar[h]);
                        used[h] = true;
                        epar[h] ^= 1u;
                        if (h == 0 && (c / kBPS) == sm && s < nb)
                            bar_wait(raw + S.a_full + 8u * c, (uint32_t)(beta & 1));
                        tc_fence_after();
                        if (leader) {
#pragma unroll
                            for (int k = 0; k < 2; ++k)
                                umma_i8_ts(tmem + (uint32_t)(dcol0 + dstride * h + kNCW * k),
                                           tmem + (uint32_t)((c * kSP + 2 * h + k) * kACols),
                                           bdesc, idesc);
                            umma_commit(raw + S.d_full + 8u * h);
                        }
                        __syncwarp();
                    }
                } else {
                    const int buf = c % ND;
                    if (used[buf]) bar_wait(raw + S.d_empty + 8u * buf, epar[buf]);
                    used[buf] = true;
                    epar[buf] ^= 1u;
                    if ((c / kBPS) == sm && s < nb)  // newborn cohort: its rows are in tensor memory
                        bar_wait(raw + S.a_full + 8u * c, (uint32_t)(beta & 1));
                    tc_fence_after();
                    if (leader) {
#pragma unroll
                        for (int k = 0; k < kSP; ++k) {
                            const uint32_t td = tmem + (uint32_t)(dcol0 + dstride * buf + kNC * k);
                            const uint32_t ta = tmem + (uint32_t)((c * kSP + k) * kACols);
                            if (MODE == 2) umma_i8_ts(td, ta, bdesc, idesc);
                            else umma_f16_ts(td, ta, bdesc, idesc);
                        }
                        umma_commit(raw + S.d_full + 8u * buf);
                    }
                    __syncwarp();
                }
            }
            if (++sm == NG) {
                sm = 0;
                ++beta;
            }
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
        if (LOADW) {
            switch (D) {
                case 4: run_loader<4, true>(a, S, x, smem_raw); break;
                case 6: run_loader<6, true>(a, S, x, smem_raw); break;
                case 8: run_loader<8, true>(a, S, x, smem_raw); break;
                default: run_loader<10, true>(a, S, x, smem_raw); break;
            }
        } else {
            switch (D) {
                case 4: run_loader<4, false>(a, S, x, smem_raw); break;
                case 6: run_loader<6, false>(a, S, x, smem_raw); break;
                case 8: run_loader<8, false>(a, S, x, smem_raw); break;
                case 10: run_loader<10, false>(a, S, x, smem_raw); break;
                default: run_loader<12, false>(a, S, x, smem_raw); break;
            }
        }
    } else {
        // ================= epilogue =================
        const int ew = warp - kEpiWarp0;
        const int grp = ew >> 2;  // the cohort's tile this warp probes
        const int q = warp & 3;
        const uint32_t negM = a.negM, magic = a.magic, pow2s = a.pow2s;
        uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(dcol0 + kNC * grp);
        asm volatile("" : "+r"(tlane));
        const bool lane0 = lane == 0;
        uint32_t dfull = raw + S.d_full, dempty = raw + S.d_empty;
        asm volatile("" : "+r"(dfull), "+r"(dempty));  // not rematerialised per item
        // running hit counts of this thread's row in every cohort, one byte each
        uint32_t hp[(NCH + 3) / 4];
#pragma unroll
        for (int i = 0; i < (NCH + 3) / 4; ++i) hp[i] = 0;
        uint32_t par[3] = {0u, 0u, 0u};
        int sm = 0;
        // byte mode: this warp's half buffer (tiles 0-1 / 2-3) and its tile's columns
        const int hb = grp >> 1;
        uint32_t tlw = tmem + ((uint32_t)(q * 32) << 16) +
                       (uint32_t)(dcol0 + dstride * hb + kNCW * (grp & 1));
        uint32_t dfullw = raw + S.d_full + 8u * hb, demptyw = raw + S.d_empty + 8u * hb;
        asm volatile("" : "+r"(tlw), "+r"(dfullw), "+r"(demptyw));
        uint32_t parw = 0u;
        for (int s = 0; s < nsteps; ++s) {
            const int lcg = max(0, min(a.L, sm * kLG + kLG) - sm * kLG);
            // pair i's bit ends at position 32 - kLG + i of the accumulator
            const uint32_t lmask = ((1u << lcg) - 1u) << (32 - kLG);
            const int ring = s & 1;
            uint32_t boff = (uint32_t)ring * kBufStride;
            asm volatile("" : "+r"(boff));  // one register per step, not rematerialised per probe
            bar_wait(raw + S.bm_full + 8u * ring, (uint32_t)((s >> 1) & 1));
            // residues in [0, M + ext): x - umulhi(x, 2^32/M) M
            auto reduce = [&](uint32_t xx) -> uint32_t {
                const uint32_t qq = __umulhi(xx, magic);
                uint32_t r;
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(qq), "r"(negM), "r"(xx));
                return r;
            };
            auto probes = [&](const uint32_t (&r)[kLG], uint32_t (&w)[kLG]) {
                w[0] = probe<0>(r[0], boff);
                w[1] = probe<1>(r[1], boff);
                w[2] = probe<2>(r[2], boff);
                w[3] = probe<3>(r[3], boff);
                w[4] = probe<4>(r[4], boff);
                w[5] = probe<5>(r[5], boff);
                w[6] = probe<6>(r[6], boff);
                w[7] = probe<7>(r[7], boff);
            };
            // the bits of cohort c (words wc, residues rc) into its hit counter;
            // a cohort that has now seen every group retires
            auto count_retire = [&](const int c, const uint32_t (&rc)[kLG],
                                    const uint32_t (&wc)[kLG]) {
                uint32_t bacc = 0;
#pragma unroll
                for (int i = 0; i < kLG; ++i)
                    bacc = __funnelshift_r(bacc, __funnelshift_r(wc[i], wc[i], rc[i]), 1);
                hp[c >> 2] += __popc(bacc & lmask) << (8 * (c & 3));
                if (sm == ((c / kBPS) + NG - 1) % NG) {  // born at step s - (NG - 1): retires
                    const int b = s - (NG - 1);
                    const uint32_t hc = (hp[c >> 2] >> (8 * (c & 3))) & 255u;
                    hp[c >> 2] &= ~(255u << (8 * (c & 3)));
                    if (b >= 0) {  // b < nb holds: s < nb + NG - 1
                        const int64_t t =
                            cta + (int64_t)((b * kBPS + (c % kBPS)) * kSP + grp) * ncta;
                        const int64_t row0 = t * kTile + q * 32;
                        const int64_t row = row0 + lane;
                        const bool valid = row < a.n;
                        const int64_t hits = (int64_t)hc;
                        const unsigned det =
                            __ballot_sync(0xffffffffu, valid && hits >= a.min_hits);
                        if (valid && a.hits64) a.hits64[row] = hits;
                        if (lane0 && row0 < a.n) a.detmask[row0 >> 5] = det;
                        __syncwarp();
                        if (lane0) bar_arrive(raw + S.a_empty + 8u * c);
                    }
                }
            };
            uint32_t rr[2][kLG], ww[2][kLG];
            if (WIDE) {
                // Software pipeline: while the bits of cohort c are counted, the
                // accumulators of cohort c + 1 come from tensor memory; its
                // bitmap words are requested before cohort c + 1 is counted.
                uint32_t v[24];
                auto residues = [&](uint32_t (&r)[kLG]) {
#pragma unroll
                    for (int i = 0; i < kLG; ++i) {
                        uint32_t xx = (v[3 * i + 1] << 8) + v[3 * i];
                        xx = (v[3 * i + 2] << 16) + xx;
                        r[i] = reduce(xx);
                    }
                };
                bar_wait(dfullw, parw);
                parw ^= 1u;
                tc_fence_after();
                tmem_ld24_async(tlw, v);
                tmem_wait_ld24(v);  // .sync.aligned: every lane's load has completed
                tc_fence_before();
                if (lane0) bar_arrive(demptyw);
                if (a.dbg && s == 0 && cta == 0 && grp == 0) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) a.dbg[(q * 32 + lane) * 16 + i] = v[i];
                }
                residues(rr[0]);
                probes(rr[0], ww[0]);
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    if (c + 1 < NCH) {
                        bar_wait(dfullw, parw);
                        parw ^= 1u;
                        tc_fence_after();
                        tmem_ld24_async(tlw, v);
                    }
                    if (c + 1 < NCH) {
                        tmem_wait_ld24(v);
                        tc_fence_before();
                        if (lane0) bar_arrive(demptyw);
                        residues(rr[(c + 1) & 1]);
                        probes(rr[(c + 1) & 1], ww[(c + 1) & 1]);
                    }
                    // after the release: the MMA of cohort c + 2 runs behind this
                    count_retire(c, rr[c & 1], ww[c & 1]);
                }
            } else {
                // Software pipeline over the step's cohorts: while the bits of
                // cohort c are counted, the bitmap words of cohort c + 1 are on
                // their way from shared memory and the accumulators of cohort
                // c + 2 on their way from tensor memory.
                uint32_t va[16], vb[16];
                auto residues = [&](const uint32_t (&v)[16], uint32_t (&r)[kLG]) {
#pragma unroll
                    for (int i = 0; i < kLG; ++i) {
                        uint32_t xx;
                        asm("mad.lo.u32 %0, %1, %2, %3;"
                            : "=r"(xx)
                            : "r"(v[2 * i + 1]), "r"(pow2s), "r"(v[2 * i]));
                        r[i] = reduce(xx);
                    }
                };
                bar_wait(dfull, par[0]);
                par[0] ^= 1u;
                tc_fence_after();
                tmem_ld16_async(tlane, va);
                tmem_wait_ld16(va);  // .sync.aligned: every lane's load has completed
                tc_fence_before();
                if (lane0) bar_arrive(dempty);
                if (a.dbg && s == 0 && cta == 0 && grp == 0) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) a.dbg[(q * 32 + lane) * 16 + i] = va[i];
                }
                if (NCH > 1) {
                    bar_wait(dfull + 8u * (1 % ND), par[1 % ND]);
                    par[1 % ND] ^= 1u;
                    tc_fence_after();
                    tmem_ld16_async(tlane + (uint32_t)(dstride * (1 % ND)), vb);
                }
                residues(va, rr[0]);
                probes(rr[0], ww[0]);
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    uint32_t(&vc)[16] = (c & 1) ? vb : va;  // cohort c: consumed, reused for c + 2
                    uint32_t(&vn)[16] = (c & 1) ? va : vb;  // cohort c + 1: in flight
                    const int b1 = (c + 1) % ND, b2 = (c + 2) % ND;
                    if (c + 1 < NCH) {
                        tmem_wait_ld16(vn);
                        tc_fence_before();
                        if (lane0) bar_arrive(dempty + 8u * b1);
                    }
                    if (c + 2 < NCH) {
                        bar_wait(dfull + 8u * b2, par[b2]);
                        par[b2] ^= 1u;
                        tc_fence_after();
                        tmem_ld16_async(tlane + (uint32_t)(dstride * b2), vc);
                    }
                    if (c + 1 < NCH) {
                        residues(vn, rr[(c + 1) & 1]);
                        probes(rr[(c + 1) & 1], ww[(c + 1) & 1]);
                    }
                    count_retire(c, rr[c & 1], ww[c & 1]);
                }
            }
            __syncwarp();
            if (lane0) bar_arrive(raw + S.bm_empty + 8u * ring);  // (the probes are volatile asm: done)
            if (++sm == NG) sm = 0;
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

static std::atomic<long long> g_calls{0};

static unsigned long long* scaled_counter() {
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

template <int NG, int MODE>
static int launch_ng(Args& a, uint32_t smem, int grid, cudaStream_t st) {
    auto kern = hash_rollf_kernel<NG, MODE>;
    SFFTB_CUDA(smem_opt_in(kern, smem));
    kern<<<grid, kThreads, smem, st>>>(a);
    SFFTB_CHECK_LAUNCH();
    return SFFTB_OK;
}

}  // namespace rollf

namespace roll {
unsigned long long* recomputed_counter();
void keep_async_pool();
}

// Returns 1 when the fp16 rolling kernel handled the call, 0 when the shape is
// outside it (the caller takes the other kernels), < 0 = -status.
int hash_hits_rollf(const int64_t* elems, int64_t n, int64_t d, const int64_t* zmat, int64_t L,
                    int64_t M, const uint32_t* bits, int64_t kbound, int64_t min_hits,
                    int64_t* hits64, uint32_t* detmask, cudaStream_t st) {
    using namespace rollf;
    {
        const char* e = getenv("SFFTB_HASH_ROLL");
        if (e && e[0] == '0') return 0;
        e = getenv("SFFTB_HASH_ROLLF");
        if (e && e[0] == '0') return 0;
    }
    const char* mr = getenv("SFFTB_HASH_ROLL_MINROWS");
    const int64_t min_rows = mr ? atoll(mr) : (int64_t)1 << 21;
    if (n < min_rows || n > ((int64_t)1 << 36) || L < 1 || L > kLG * kMaxNG || M < 4096 ||
        M >= ((int64_t)1 << 22))
        return 0;
    if (d != 4 && d != 6 && d != 8 && d != 10 && d != 12) return 0;
    if (((uintptr_t)elems & 15) != 0 || ((uintptr_t)bits & 15) != 0) return 0;
    // fp16 mode: x' = k.z + J M with J = kbound: 0 <= x' <= 2 kbound M
    const int64_t J = std::max<int64_t>(kbound, 1);
    __int128 xmax = (__int128)2 * J * M;
    const bool f16_ok = kbound >= 0 && kbound < kCoordLim && xmax < ((__int128)1 << 31);
    const int64_t JM = f16_ok ? J * M : 0;
    int bitsM = 0;
    while (((int64_t)1 << bitsM) < M) ++bitsM;
    // limb split c = c0 + 2^s c1 with both limbs < 2048 (fp16-exact), and
    //   bits0 = C0 + e0 + v0,  bits1 = C0 + T1 + v1,  e0 + 2^s e1 = J M,
    //   T1 = off1 + e1 with 2^s (C0 + off1) + C0 == 0 (mod 2^32),
    // both accumulators inside [2^23, 2^24): |v| + constants < 2^22.  Not
    // every s has a small enough off1: take the most balanced one that does.
    const uint64_t C0 = kSeedBits;
    const int64_t half = (int64_t)1 << 22;
    int s = -1;
    int64_t e0 = 0, T1 = 0;
    for (int dist = 0; f16_ok && dist <= 11 && s < 0; ++dist) {
        for (int sign = 0; sign < 2 && s < 0; ++sign) {
            const int st_ = (bitsM + 1) / 2 + (sign ? -dist : dist);
            if (st_ < 1 || st_ > 11 || bitsM - st_ > 11 || (sign && dist == 0)) continue;
            const int64_t c0max = ((int64_t)1 << st_) - 1, c1max = (M - 1) >> st_;
            const uint64_t mod = (uint64_t)1 << (32 - st_);
            const uint64_t X = ((((uint64_t)1 << 32) - C0) >> st_) % mod;  // 2^st_ divides C0
            const uint64_t off1 = (X + mod - (C0 % mod)) % mod;
            const int64_t e0_ = JM & c0max, e1_ = JM >> st_;
            const int64_t T1_ = (int64_t)off1 + e1_;
            if (e0_ + kbound * c0max >= half) continue;
            if (T1_ + kbound * c1max >= half) continue;
            s = st_;
            e0 = e0_;
            T1 = T1_;
        }
    }
    // byte mode (any kbound): x = sum of 2d limb products + the constant < 2^32
    const bool wide = s < 0;
    if (wide) {
        const char* e = getenv("SFFTB_HASH_ROLLW");
        if (e && e[0] == '0') return 0;
        if (d > 10) return 0;  // its B operands use the tail of the loader buffers (RS = 5)
        xmax = ((__int128)(2 * d) * 127 + 1) * (M - 1);
        if (xmax >= ((__int128)1 << 32)) return 0;
    }
    const int64_t W = ((M + 31) / 32 + 3) & ~int64_t(3);
    const int64_t ext = (int64_t)(((__int128)M * xmax) >> 32) + 2;
    const int64_t ext_words = (ext + 31) / 32 + 1;
    if (ext_words >= (M >> 5)) return 0;
    const int64_t Wx = ((M >> 5) + ext_words + 1 + 3) & ~int64_t(3);
    if (Wx * 4 > (int64_t)kSlot) return 0;
    const int NG = (int)((L + kLG - 1) / kLG);
    const Smem S = smem_map(NG);
    const uint32_t smem = S.end;
    static int prop_smem = 0;
    if (prop_smem == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&prop_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (prop_smem <= 0) prop_smem = 232448;
    }
    if (smem > (uint32_t)prop_smem) return 0;
    unsigned long long* rec = roll::recomputed_counter();
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
    a.wide = wide ? 1 : 0;
    a.s = wide ? 0 : s;
    a.pow2s = wide ? 256u : 1u << s;  // byte modes: limbs in base 256
    // A slots (2048, 2048, 1): limb 0 gets 2048 * 6144 = 1.5 * 2^23 and e0;
    // limb 1 gets 1.5 * 2^23 + T1 with T1 = 2048 t1h + t1l
    a.seed0[0] = 6144u;
    a.seed0[1] = 0u;
    a.seed0[2] = (uint32_t)e0;
    a.seed1[0] = 6144u;
    a.seed1[1] = (uint32_t)(T1 >> 11);
    a.seed1[2] = (uint32_t)(T1 & 2047);
    a.bits = bits;
    a.W = (int)W;
    roll::keep_async_pool();
    bool try2 = wide;  // the scaled two-limb byte mode when every lattice has a multiplier
    if (const char* e = getenv("SFFTB_HASH_ROLLW2")) try2 = try2 && e[0] != '0';
    // scratch: extended bitmaps | nbad, nfound, pad, pad | tmul[L] | tinv[L]
    uint32_t* xbits = nullptr;
    SFFTB_CUDA(cudaMallocAsync(&xbits, ((size_t)L * Wx + 4 + 2 * (size_t)L) * sizeof(uint32_t), st));
    a.xbits = xbits;
    a.Wx = (int)Wx;
    a.nbad = xbits + (size_t)L * Wx;
    SFFTB_CUDA(cudaMemsetAsync(a.nbad, 0, 4 * sizeof(unsigned int), st));
    unsigned int* nfound = a.nbad + 1;
    uint32_t* tmul = xbits + (size_t)L * Wx + 4;
    uint32_t* tinv = tmul + L;
    a.tmul = try2 ? tmul : nullptr;
    a.tinv = try2 ? tinv : nullptr;
    a.nfound = try2 ? nfound : nullptr;
    a.scaled_runs = scaled_counter();
    if (!a.scaled_runs) try2 = false, a.tmul = a.tinv = nullptr, a.nfound = nullptr;
    a.ntiles = (n + kTile - 1) / kTile;
    a.min_hits = min_hits;
    a.hits64 = hits64;
    a.detmask = detmask;
    a.recomputed = rec;
    a.dbg = nullptr;
    static uint32_t* dbg = nullptr;
    if (getenv("SFFTB_HASH_ROLL_DUMP")) {
        if (!dbg) SFFTB_CUDA(cudaMalloc(&dbg, 128 * 16 * sizeof(uint32_t)));
        SFFTB_CUDA(cudaMemsetAsync(dbg, 0xFF, 128 * 16 * sizeof(uint32_t), st));
        a.dbg = dbg;
    }
    int grid = num_sms();
    if (const char* e = getenv("SFFTB_HASH_ROLL_GRID")) grid = std::max(1, atoi(e));
    grid = (int)std::min<int64_t>(grid, a.ntiles);
    if (getenv("SFFTB_HASH_ROLL_DEBUG"))
        fprintf(stderr,
                "hash_rollf: d=%d L=%d NG=%d wide=%d s=%d kbound=%lld e0=%lld T1=%lld ext_words=%d "
                "smem=%u grid=%d\n",
                (int)d, (int)L, NG, (int)wide, s, (long long)kbound, (long long)e0, (long long)T1,
                (int)ext_words, smem, grid);
    if (try2) {
        const uint64_t magic64 = ~0ull / (uint64_t)M;  // floor((2^64 - 1) / M) = floor(2^64 / M), M odd or not a power of two
        SFFTB_CUDA(cudaMemsetAsync(tmul, 0xFF, sizeof(uint32_t) * (size_t)L, st));
        rollf_tsearch_kernel<<<dim3((unsigned)L, kTSplit), 256, 0, st>>>(zmat, (int)d, (uint32_t)M,
                                                                        magic64, tmul);
        count_launch();
        rollf_tfinish_kernel<<<(unsigned)((L + 63) / 64), 64, 0, st>>>((int)L, (uint32_t)M, tmul,
                                                                      tinv, nfound);
        count_launch();
        rollf_extend_kernel<<<(unsigned)((L * Wx + 255) / 256), 256, 0, st>>>(
            bits, (int)L, (int)W, (int)Wx, (uint32_t)M, magic64, (int)ext_words, tinv, nfound,
            xbits);
    } else {
        rollptx::roll_extend_kernel<0><<<(unsigned)((L * Wx + 255) / 256), 256, 0, st>>>(
            bits, (int)L, (int)W, (int)Wx, (uint32_t)M, (int)ext_words, xbits);
    }
    count_launch();
    int rc = SFFTB_EINVAL;
    if (getenv("SFFTB_HASH_ROLLF_FORCE_EXACT")) {
        // tests: take the path of a kernel that declined the call (see probe()):
        // every row through the exact follow-up kernel
        const unsigned int all = kAllRows;
        SFFTB_CUDA(cudaMemcpyAsync(a.nbad, &all, sizeof(all), cudaMemcpyHostToDevice, st));
        SFFTB_CUDA(cudaStreamSynchronize(st));  // `all` is a stack variable
        rc = SFFTB_OK;
    } else if (wide) {
        if (try2) {  // returns at once unless every lattice has a multiplier
            switch (NG) {
                case 1: rc = launch_ng<1, 2>(a, smem, grid, st); break;
                case 2: rc = launch_ng<2, 2>(a, smem, grid, st); break;
                case 3: rc = launch_ng<3, 2>(a, smem, grid, st); break;
                case 4: rc = launch_ng<4, 2>(a, smem, grid, st); break;
                case 5: rc = launch_ng<5, 2>(a, smem, grid, st); break;
                case 6: rc = launch_ng<6, 2>(a, smem, grid, st); break;
            }
            if (rc != SFFTB_OK) {
                cudaFreeAsync(xbits, st);
                return -rc;
            }
        }
        switch (NG) {  // returns at once when the two-limb kernel ran
            case 1: rc = launch_ng<1, 1>(a, smem, grid, st); break;
            case 2: rc = launch_ng<2, 1>(a, smem, grid, st); break;
            case 3: rc = launch_ng<3, 1>(a, smem, grid, st); break;
            case 4: rc = launch_ng<4, 1>(a, smem, grid, st); break;
            case 5: rc = launch_ng<5, 1>(a, smem, grid, st); break;
            case 6: rc = launch_ng<6, 1>(a, smem, grid, st); break;
        }
    } else {
        switch (NG) {
            case 1: rc = launch_ng<1, 0>(a, smem, grid, st); break;
            case 2: rc = launch_ng<2, 0>(a, smem, grid, st); break;
            case 3: rc = launch_ng<3, 0>(a, smem, grid, st); break;
            case 4: rc = launch_ng<4, 0>(a, smem, grid, st); break;
            case 5: rc = launch_ng<5, 0>(a, smem, grid, st); break;
            case 6: rc = launch_ng<6, 0>(a, smem, grid, st); break;
        }
    }
    if (rc == SFFTB_OK) {
        rollf_fixup_kernel<<<4 * num_sms(), 256, 0, st>>>(a);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) rc = SFFTB_ECUDA;
    }
    cudaFreeAsync(xbits, st);
    if (a.dbg && rc == SFFTB_OK) {
        static uint32_t h[128 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost);
        for (int r : {0, 1, 33, 127}) {
            fprintf(stderr, "rollf dbg row %3d:", r);
            for (int i = 0; i < 16; ++i) fprintf(stderr, " %08x", h[r * 16 + i]);
            fprintf(stderr, "\n");
        }
    }
    if (rc == SFFTB_OK) rollf::g_calls.fetch_add(1, std::memory_order_relaxed);
    return rc == SFFTB_OK ? 1 : -rc;
}

}  // namespace sfftb

extern "C" int64_t sfftb_hash_rollf_scaled_runs(int reset) {
    unsigned long long* p = sfftb::rollf::scaled_counter();
    if (!p) return -1;
    unsigned long long v = 0;
    if (cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    if (reset) cudaMemset(p, 0, sizeof(v));
    return (int64_t)v;
}

extern "C" int64_t sfftb_hash_rollf_calls(int reset) {
    return reset ? sfftb::rollf::g_calls.exchange(0) : sfftb::rollf::g_calls.load();
}
