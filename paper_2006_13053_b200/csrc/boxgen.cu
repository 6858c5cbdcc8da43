// numpy Generator.integers(low, high, size=N, dtype=int64) on the device, in
// numpy's exact stream (the draw of freqset._random_from_box, reference
// freqset.py:273-275), so a seeded candidate set can be born in HBM.
//
// numpy draws int64 values with range rng = high - 1 - low < 2^32 - 1 by
// Lemire's method on 32-bit words taken from PCG64 64-bit outputs through a
// one-word buffer (low half first, then the high half).  A word x is accepted
// iff the low 32 bits of x * (rng + 1) are >= (2^32 - 1 - rng) mod (rng + 1);
// the value is low + the high 32 bits.  Acceptance depends on the word alone,
// so the stream parallelises as: every thread jumps its PCG64 copy to its
// block of outputs (LCG jump tables from the host, csrc/hostrng.cpp), counts
// the accepted words of its block (pass 1), the host scans the per-CTA
// counts, and pass 2 rewrites the accepted values at their stream positions.
// The host rebuilds the generator's final state from the index of the last
// consumed word (sfftb_box_integers returns it).
#include "common.cuh"

namespace sfftb {

namespace {

typedef unsigned __int128 u128;

constexpr int kOutPerThread = 32;  // 64-bit outputs (64 words) per thread
constexpr int kGenThreads = 256;

struct Jump {
    uint64_t a_hi[64], a_lo[64], c_hi[64], c_lo[64];
};

struct GenArgs {
    uint64_t s_hi, s_lo;  // state before the first output
    int64_t q_total;      // 64-bit outputs covered by the grid
    int has0;             // 1: word 0 is the buffered high half `u0`
    uint32_t u0;
    uint32_t excl, thr;   // rng + 1, rejection threshold
    int64_t low;
    int64_t n;            // values wanted
    const int64_t* block_off;  // pass 2: values before each CTA
    int* block_cnt;            // pass 1 output
    int64_t* out;
    unsigned long long* last;  // pass 2: [word index of value n-1, its output's high half]
};

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ bool accept(uint32_t w, uint32_t excl, uint32_t thr, uint32_t* v) {
    const uint64_t m = (uint64_t)w * excl;
    *v = (uint32_t)(m >> 32);
    return (uint32_t)m >= thr;
}

template <bool WRITE>
__global__ void __launch_bounds__(kGenThreads) box_integers_kernel(const __grid_constant__ Jump J,
                                                                   GenArgs a) {
    __shared__ int warp_tot[kGenThreads / 32];
    const int64_t t = (int64_t)blockIdx.x * kGenThreads + threadIdx.x;
    const int64_t q0 = t * kOutPerThread;
    // state before output q0: s_q0 = A^q0 s_0 + C_q0
    u128 s = mk(a.s_hi, a.s_lo);
    if (q0 < a.q_total) {
        for (int i = 0; i < 40; ++i)
            if ((q0 >> i) & 1) s = mk(J.a_hi[i], J.a_lo[i]) * s + mk(J.c_hi[i], J.c_lo[i]);
    }
    const u128 A1 = mk(J.a_hi[0], J.a_lo[0]), C1 = mk(J.c_hi[0], J.c_lo[0]);
    const int64_t left = a.q_total - q0;
    const int nq = left <= 0 ? 0 : (left < kOutPerThread ? (int)left : kOutPerThread);
    const bool first = t == 0 && a.has0;
    int cnt = 0;
    {
        u128 s1 = s;
        uint32_t v;
        if (first) cnt += accept(a.u0, a.excl, a.thr, &v);
        for (int q = 0; q < nq; ++q) {
            s1 = A1 * s1 + C1;
            const uint64_t o = xsl_rr(s1);
            cnt += accept((uint32_t)o, a.excl, a.thr, &v);
            cnt += accept((uint32_t)(o >> 32), a.excl, a.thr, &v);
        }
    }
    // block-exclusive offsets of the per-thread counts
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (!WRITE) {
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < kGenThreads / 32; ++w) tot += warp_tot[w];
            a.block_cnt[blockIdx.x] = tot;
        }
        return;
    }
    int before = 0;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    int64_t pos = a.block_off[blockIdx.x] + before + incl - cnt;
    if (pos >= a.n || cnt == 0) return;
    // word index of this thread's first word in the stream
    int64_t word = (a.has0 ? 1 : 0) + 2 * q0 - (first ? 1 : 0);
    uint32_t v;
    if (first) {
        if (accept(a.u0, a.excl, a.thr, &v)) {
            a.out[pos] = a.low + (int64_t)v;
            if (pos == a.n - 1) {
                a.last[0] = 0;
                a.last[1] = a.u0;
            }
            ++pos;
        }
        ++word;
    }
    for (int q = 0; q < nq && pos < a.n; ++q) {
        s = A1 * s + C1;
        const uint64_t o = xsl_rr(s);
        for (int h = 0; h < 2 && pos < a.n; ++h, ++word) {
            if (accept(h ? (uint32_t)(o >> 32) : (uint32_t)o, a.excl, a.thr, &v)) {
                a.out[pos] = a.low + (int64_t)v;
                if (pos == a.n - 1) {
                    a.last[0] = (unsigned long long)word;
                    a.last[1] = o >> 32;
                }
                ++pos;
            }
        }
    }
}

}  // namespace
}  // namespace sfftb

using namespace sfftb;

// Generator.integers(low, high_incl + 1, size=n, dtype=int64) from the PCG64
// state `state6` (hostrng.cpp layout), written to the device array out (n).
// Requires high_incl - low < 2^32 - 1.  jump: the 64 jump-by-2^i pairs of
// sfftb_pcg64_advance(state, 0, jump) (4 uint64 each).  ws: device workspace
// of sfftb_box_integers_workspace_bytes(n) bytes.  On return (synchronous)
// *words_used = the stream words consumed and *last_hi = the high half of the
// 64-bit output holding the last one (for the caller to rebuild the state);
// SFFTB_EINVAL when the draw needs more words than the margin allowed for
// (the caller retries with a larger `extra`).
extern "C" int64_t sfftb_box_integers_workspace_bytes(int64_t n, int64_t extra) {
    const int64_t q = (n + extra + 1) / 2 + 1;
    const int64_t blocks = (q + (int64_t)kGenThreads * kOutPerThread - 1) /
                           ((int64_t)kGenThreads * kOutPerThread);
    return blocks * (4 + 8) + 16 + 256;
}

extern "C" int sfftb_box_integers(const uint64_t* state6, const uint64_t* jump, int64_t low,
                                  int64_t high_incl, int64_t n, int64_t extra, int64_t* out,
                                  void* ws, int64_t* words_used, uint64_t* last_hi,
                                  void* stream) {
    SFFTB_REQUIRE(n >= 0 && extra >= 0 && high_incl >= low, "box_integers: bad sizes");
    const uint64_t rng = (uint64_t)high_incl - (uint64_t)low;
    SFFTB_REQUIRE(rng < 0xFFFFFFFFull, "box_integers: range needs 64-bit words");
    *words_used = 0;
    *last_hi = state6[5];
    if (n == 0) return SFFTB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Jump J;
    for (int i = 0; i < 64; ++i) {
        J.a_hi[i] = jump[4 * i + 0];
        J.a_lo[i] = jump[4 * i + 1];
        J.c_hi[i] = jump[4 * i + 2];
        J.c_lo[i] = jump[4 * i + 3];
    }
    const int has0 = state6[4] ? 1 : 0;
    const int64_t words = n + extra;
    const int64_t q = (words - has0 + 1) / 2 + 1;
    const int64_t per_block = (int64_t)kGenThreads * kOutPerThread;
    const int64_t blocks = (q + per_block - 1) / per_block;
    SFFTB_REQUIRE(blocks < (int64_t)1 << 31, "box_integers: too many values");
    char* w = (char*)ws;
    int* cnt = (int*)w;
    int64_t* off = (int64_t*)(w + ((blocks * 4 + 15) & ~int64_t(15)));
    unsigned long long* last =
        (unsigned long long*)(w + ((blocks * 4 + 15) & ~int64_t(15)) + blocks * 8);
    GenArgs a;
    a.s_hi = state6[0];
    a.s_lo = state6[1];
    a.q_total = q;
    a.has0 = has0;
    a.u0 = (uint32_t)state6[5];
    a.excl = (uint32_t)(rng + 1);
    a.thr = (uint32_t)((0xFFFFFFFFull - rng) % (rng + 1));
    a.low = low;
    a.n = n;
    a.block_cnt = cnt;
    a.block_off = off;
    a.out = out;
    a.last = last;
    box_integers_kernel<false><<<(unsigned)blocks, kGenThreads, 0, st>>>(J, a);
    SFFTB_CHECK_LAUNCH();
    int* hc = new int[blocks];
    int64_t* ho = new int64_t[blocks];
    SFFTB_CUDA(cudaMemcpyAsync(hc, cnt, blocks * sizeof(int), cudaMemcpyDeviceToHost, st));
    SFFTB_CUDA(cudaStreamSynchronize(st));
    int64_t acc = 0;
    for (int64_t b = 0; b < blocks; ++b) {
        ho[b] = acc;
        acc += hc[b];
    }
    delete[] hc;
    if (acc < n) {
        delete[] ho;
        set_error("box_integers: not enough accepted words, raise extra");
        return SFFTB_EINVAL;
    }
    SFFTB_CUDA(cudaMemcpyAsync(off, ho, blocks * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    box_integers_kernel<true><<<(unsigned)blocks, kGenThreads, 0, st>>>(J, a);
    SFFTB_CHECK_LAUNCH();
    unsigned long long hl[2];
    SFFTB_CUDA(cudaMemcpyAsync(hl, last, sizeof(hl), cudaMemcpyDeviceToHost, st));
    SFFTB_CUDA(cudaStreamSynchronize(st));
    delete[] ho;
    *words_used = (int64_t)hl[0] + 1;
    *last_hi = hl[1];
    return SFFTB_OK;
}
