// Host-side seed streams of the sfft driver, restated natively.
//
// The reference draws every lattice generator, coordinate-line node and fixed
// tail from numpy Generator(PCG64(SeedSequence((master, tag, t, i))))
// (latfft/dimincr.py:99-100, :137-141, :231-235; lattice.py:225-227).  The
// driver needs ~10^2 such streams per reconstruction; building them through
// numpy costs ~25 us each on the host critical path, so this file restates
// the three published algorithms involved, bit-for-bit:
//
//  * SeedSequence entropy pooling (O'Neill's seed_seq_fe with 4 words):
//    hashmix/mix over the uint32 words of the entropy integers, then
//    generate_state(4, uint64) -> (state, increment) of the 128-bit PCG;
//  * PCG64 = PCG-XSL-RR 128/64 (LCG multiplier 0x2360ED051FC65DA4_4385DF649FCCF645),
//    seeded with pcg_setseq_128_srandom_r, with numpy's one-word buffer for
//    32-bit draws (has_uint32 / uinteger);
//  * Generator.random / uniform(0, 1): (next64 >> 11) * 2^-53;
//    Generator.integers(low, high) for int64: Lemire's nearly-divisionless
//    bounded draw on 32-bit words when high - low - 1 < 2^32 - 1, on 64-bit
//    words above, no masking.
//
// State layout (6 x uint64): state_hi, state_lo, inc_hi, inc_lo, has_uint32,
// uinteger.  tests/test_host.py checks every entry point against numpy.
#include <stdint.h>
#include <string.h>

#include <new>

namespace {

typedef unsigned __int128 u128;

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kPool = 4;

inline uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    v ^= v >> 16;
    return v;
}

inline uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    r ^= r >> 16;
    return r;
}

struct Pcg {
    u128 state, inc;
    uint64_t has32, uint32v;
};

const u128 kMult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;

inline void load(const uint64_t* s, Pcg& p) {
    p.state = ((u128)s[0] << 64) | s[1];
    p.inc = ((u128)s[2] << 64) | s[3];
    p.has32 = s[4];
    p.uint32v = s[5];
}

inline void store(const Pcg& p, uint64_t* s) {
    s[0] = (uint64_t)(p.state >> 64);
    s[1] = (uint64_t)p.state;
    s[2] = (uint64_t)(p.inc >> 64);
    s[3] = (uint64_t)p.inc;
    s[4] = p.has32;
    s[5] = p.uint32v;
}

inline uint64_t next64(Pcg& p) {
    p.state = p.state * kMult + p.inc;
    const uint64_t x = (uint64_t)(p.state >> 64) ^ (uint64_t)p.state;
    const unsigned rot = (unsigned)(p.state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

inline uint32_t next32(Pcg& p) {
    if (p.has32) {
        p.has32 = 0;
        return (uint32_t)p.uint32v;
    }
    const uint64_t n = next64(p);
    p.has32 = 1;
    p.uint32v = n >> 32;
    return (uint32_t)n;
}

void seed_one(const uint32_t* words, int64_t nwords, uint64_t* out) {
    uint32_t pool[kPool];
    uint32_t hc = kInitA;
    for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < nwords ? words[i] : 0u, hc);
    for (int s = 0; s < kPool; ++s)
        for (int d = 0; d < kPool; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (int64_t s = kPool; s < nwords; ++s)
        for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hashmix(words[s], hc));
    // generate_state(4, uint64): 8 words cycling the pool, little-endian pairs
    uint32_t st[8];
    uint32_t hb = kInitB;
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i % kPool];
        v ^= hb;
        hb *= kMultB;
        v *= hb;
        v ^= v >> 16;
        st[i] = v;
    }
    uint64_t val[4];
    for (int i = 0; i < 4; ++i) val[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
    // pcg64_set_seed: state = val[0]:val[1], initseq = val[2]:val[3]
    Pcg p;
    const u128 initstate = ((u128)val[0] << 64) | val[1];
    const u128 initseq = ((u128)val[2] << 64) | val[3];
    p.state = 0;
    p.inc = (initseq << 1) | 1u;
    p.state = p.state * kMult + p.inc;
    p.state += initstate;
    p.state = p.state * kMult + p.inc;
    p.has32 = 0;
    p.uint32v = 0;
    store(p, out);
}

inline uint32_t lemire32(Pcg& p, uint32_t rng) {
    const uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)next32(p) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        const uint32_t thr = (UINT32_MAX - rng) % excl;
        while (left < thr) {
            m = (uint64_t)next32(p) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

inline uint64_t lemire64(Pcg& p, uint64_t rng) {
    const uint64_t excl = rng + 1u;
    u128 m = (u128)next64(p) * excl;
    uint64_t left = (uint64_t)m;
    if (left < excl) {
        const uint64_t thr = (UINT64_MAX - rng) % excl;
        while (left < thr) {
            m = (u128)next64(p) * excl;
            left = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

void fill_int(Pcg& p, int64_t low, uint64_t rng, int64_t count, int64_t* out) {
    const uint64_t off = (uint64_t)low;
    if (rng == 0) {
        for (int64_t i = 0; i < count; ++i) out[i] = low;
    } else if (rng < 0xFFFFFFFFull) {
        for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)(off + lemire32(p, (uint32_t)rng));
    } else if (rng == 0xFFFFFFFFull) {
        for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)(off + next32(p));
    } else if (rng == UINT64_MAX) {
        for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)(off + next64(p));
    } else {
        for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)(off + lemire64(p, rng));
    }
}

}  // namespace

extern "C" {

// rows seed streams; row r's entropy is words[r*nwords : (r+1)*nwords]
// (the uint32 words of SeedSequence's entropy, already assembled).
int sfftb_pcg64_seed(const uint32_t* words, int64_t rows, int64_t nwords, uint64_t* states) {
    if (rows < 0 || nwords < 0) return 1;
    for (int64_t r = 0; r < rows; ++r) seed_one(words + r * nwords, nwords, states + 6 * r);
    return 0;
}

// count doubles of Generator.random() from each of rows streams -> out (rows, count)
int sfftb_pcg64_random(uint64_t* states, int64_t rows, int64_t count, double* out) {
    if (rows < 0 || count < 0) return 1;
    for (int64_t r = 0; r < rows; ++r) {
        Pcg p;
        load(states + 6 * r, p);
        for (int64_t i = 0; i < count; ++i)
            out[r * count + i] = (double)(next64(p) >> 11) * (1.0 / 9007199254740992.0);
        store(p, states + 6 * r);
    }
    return 0;
}

// count int64 of Generator.integers(low, high_incl + 1) from each stream
int sfftb_pcg64_integers(uint64_t* states, int64_t rows, int64_t low, int64_t high_incl,
                         int64_t count, int64_t* out) {
    if (rows < 0 || count < 0 || high_incl < low) return 1;
    const uint64_t rng = (uint64_t)high_incl - (uint64_t)low;
    for (int64_t r = 0; r < rows; ++r) {
        Pcg p;
        load(states + 6 * r, p);
        fill_int(p, low, rng, count, out + r * count);
        store(p, states + 6 * r);
    }
    return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Candidate-set generation in the reference's stream (freqset.py:266-280:
// integers -> _canonicalize -> Generator.choice(replace=False) -> sort).
// ---------------------------------------------------------------------------

namespace {

// bounded draw in [0, rng] as numpy's random_bounded_uint64(off=0, rng, mask,
// use_masked=0): nothing for rng == 0, Lemire on buffered 32-bit words up to
// 2^32 - 2, one raw 32-bit word at 2^32 - 1, Lemire on 64-bit words above.
inline uint64_t bounded(Pcg& p, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng < 0xFFFFFFFFull) return lemire32(p, (uint32_t)rng);
    if (rng == 0xFFFFFFFFull) return next32(p);
    if (rng == UINT64_MAX) return next64(p);
    return lemire64(p, rng);
}

// Fisher-Yates of _generator.pyx's _shuffle_int: i from n-1 down to first.
void shuffle_int(Pcg& p, int64_t n, int64_t first, int64_t* data) {
    for (int64_t i = n - 1; i >= first; --i) {
        const int64_t j = (int64_t)bounded(p, (uint64_t)i);
        const int64_t t = data[j];
        data[j] = data[i];
        data[i] = t;
    }
}

}  // namespace

extern "C" {

// Advance a PCG64 state by `delta` 64-bit outputs (LCG jump-ahead; the
// 32-bit buffer is untouched).  tables: if non-null, receives the 128 pairs
// (A_i, C_i) of the jump by 2^i as 4 uint64 each (hi, lo of A, hi, lo of C).
int sfftb_pcg64_advance(uint64_t* state, uint64_t delta, uint64_t* tables) {
    Pcg p;
    load(state, p);
    u128 A = kMult, C = p.inc;  // jump by 2^i: s -> A s + C
    u128 accA = 1, accC = 0;
    for (int i = 0; i < 64; ++i) {
        if (tables) {
            tables[4 * i + 0] = (uint64_t)(A >> 64);
            tables[4 * i + 1] = (uint64_t)A;
            tables[4 * i + 2] = (uint64_t)(C >> 64);
            tables[4 * i + 3] = (uint64_t)C;
        }
        if ((delta >> i) & 1u) {
            accA = A * accA;
            accC = A * accC + C;
        }
        C = A * C + C;
        A = A * A;
    }
    p.state = accA * p.state + accC;
    store(p, state);
    return 0;
}

// Generator.choice(pop, size, replace=False) in numpy's tail-shuffle regime
// (pop > 10000 and size > pop // 50): arange(pop), _shuffle_int(pop,
// max(pop - size, 1)), keep the last `size`, and -- when final_shuffle --
// _shuffle_int(size, 1) of those.  out (size) gets the chosen indices in
// numpy's order; the state advances exactly as numpy's does.
int sfftb_pcg64_choice_tail(uint64_t* state, int64_t pop, int64_t size, int final_shuffle,
                            int64_t* out) {
    if (pop < 0 || size < 0 || size > pop) return 1;
    Pcg p;
    load(state, p);
    int64_t* data = new (std::nothrow) int64_t[pop > 0 ? pop : 1];
    if (!data) return 2;
    for (int64_t i = 0; i < pop; ++i) data[i] = i;
    const int64_t first = pop - size > 1 ? pop - size : 1;
    shuffle_int(p, pop, first, data);
    memcpy(out, data + (pop - size), (size_t)size * sizeof(int64_t));
    delete[] data;
    if (final_shuffle) shuffle_int(p, size, 1, out);
    store(p, state);
    return 0;
}

}  // extern "C"
