// Power-of-two FP64 complex FFTs held in shared memory (Stockham autosort,
// radix 16/8/4/2 butterflies in registers).  Building block of the Bluestein
// prime-length DFT in fft.cu.
//
// Layout: one FFT of length n occupies n*17/16 double2 slots (one pad slot
// per 16 elements, pad(i) = i + i/16) so that the stride-R stores of the
// first Stockham pass do not serialise on shared-memory banks.
#pragma once

#include "common.cuh"

namespace sfftb {

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

// e^{-2 pi i k / 16}, k < 16, correctly rounded literals.
__device__ __forceinline__ double2 w16(int k) {
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
    constexpr double c2 = 0.70710678118654752440;
    switch (k & 15) {
        case 0: return make_double2(1.0, 0.0);
        case 1: return make_double2(c1, -s1);
        case 2: return make_double2(c2, -c2);
        case 3: return make_double2(s1, -c1);
        case 4: return make_double2(0.0, -1.0);
        case 5: return make_double2(-s1, -c1);
        case 6: return make_double2(-c2, -c2);
        case 7: return make_double2(-c1, -s1);
        case 8: return make_double2(-1.0, 0.0);
        case 9: return make_double2(-c1, s1);
        case 10: return make_double2(-c2, c2);
        case 11: return make_double2(-s1, c1);
        case 12: return make_double2(0.0, 1.0);
        case 13: return make_double2(s1, c1);
        case 14: return make_double2(c2, c2);
        default: return make_double2(c1, s1);
    }
}

// multiply by e^{-+2 pi i k/16} with the trivial factors special-cased
template <bool INV>
__device__ __forceinline__ double2 mul_w16(double2 v, int k) {
    k &= 15;
    if (k == 0) return v;
    if (k == 4) return INV ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
    if (k == 8) return make_double2(-v.x, -v.y);
    if (k == 12) return INV ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
    double2 w = w16(k);
    if (INV) w.y = -w.y;
    return cmul(v, w);
}

// In-register radix-R DFT (R in {2,4,8,16}), natural order in and out,
// iterative radix-2 DIT on bit-reversed inputs; all indices compile-time.
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(double2 (&v)[R]) {
    constexpr int LR = ilog2c(R);
    double2 t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        int rev = 0;
#pragma unroll
        for (int b = 0; b < LR; ++b) rev |= ((i >> b) & 1) << (LR - 1 - b);
        t[rev] = v[i];
    }
#pragma unroll
    for (int s = 1; s <= LR; ++s) {
        constexpr int dummy = 0;
        (void)dummy;
        const int m = 1 << s, h = m >> 1;
#pragma unroll
        for (int k = 0; k < R; k += m) {
#pragma unroll
            for (int j = 0; j < h; ++j) {
                // twiddle e^{-2 pi i j/m} = w16(j * 16/m)
                double2 u = t[k + j];
                double2 x = mul_w16<INV>(t[k + j + h], j * (16 / m));
                t[k + j] = cadd(u, x);
                t[k + j + h] = csub(u, x);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = t[i];
}

// Twiddle e^{-+2 pi i e / NT} from a two-level table:
// tw_hi[e >> 6] * tw_lo[e & 63] (both tables hold e^{-2 pi i (.)/NT}).
template <bool INV>
__device__ __forceinline__ double2 twiddle2(const double2* __restrict__ tw_hi,
                                            const double2* __restrict__ tw_lo, int e) {
    double2 a = tw_hi[e >> 6];
    double2 w = (e & 63) ? cmul(a, tw_lo[e & 63]) : a;
    if (INV) w.y = -w.y;
    return w;
}

// Largest radix (<= 16) for the next Stockham pass given remaining log2 size.
__host__ __device__ constexpr int pass_radix(int rem_log) {
    return rem_log >= 4 ? 16 : (1 << rem_log);
}

// Twiddle sources for a length-N sub-FFT:
//  * TwDirect: shared-memory table tw[m] = e^{-2 pi i m/N}, m < N (one load)
//  * TwTwoLevel: e^{-2 pi i e/NT} = hi[e >> 6] * lo[e & 63] (tables of the
//    full transform length NT; e = m * (NT/N)) for lengths whose direct table
//    would not fit next to the data.
struct TwDirect {
    const double2* tw;
    template <bool INV>
    __device__ __forceinline__ double2 get(int m) const {
        double2 w = tw[m];
        if (INV) w.y = -w.y;
        return w;
    }
};
struct TwTwoLevel {
    const double2* hi;
    const double2* lo;
    int scale;
    template <bool INV>
    __device__ __forceinline__ double2 get(int m) const {
        return twiddle2<INV>(hi, lo, m * scale);
    }
};

// One Stockham pass of radix R over a length-N FFT held at buf (threads per
// FFT TPF = N/16, each thread owns 16 elements = 16/R butterflies).  The
// twiddle of butterfly j, output r is e^{-+2 pi i (j mod Ns) r / (Ns R)}.
template <int N, int R, bool INV, class TW>
__device__ __forceinline__ void stockham_pass(double2* __restrict__ buf, int tpf_id, int Ns,
                                              const TW& tw) {
    constexpr int TPF = N / 16;
    constexpr int BPT = 16 / R;  // butterflies per thread
    double2 v[BPT][R];
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int j = tpf_id + q * TPF;
#pragma unroll
        for (int r = 0; r < R; ++r) v[q][r] = buf[pad16(j + r * (N / R))];
        if (Ns > 1) {
            const int jm = j % Ns;
            const int step = jm * (N / (Ns * R));
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const int m = (step * r) & (N - 1);
                if (m) v[q][r] = cmul(v[q][r], tw.template get<INV>(m));
            }
        }
        dft_reg<R, INV>(v[q]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int j = tpf_id + q * TPF;
        const int base = (j / Ns) * Ns * R + (j % Ns);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pad16(base + r * Ns)] = v[q][r];
    }
    __syncthreads();
}

template <int N, int NS, int REM, bool INV, class TW>
struct StockhamRun {
    __device__ __forceinline__ static void run(double2* buf, int tpf_id, const TW& tw) {
        constexpr int R = pass_radix(REM);
        stockham_pass<N, R, INV, TW>(buf, tpf_id, NS, tw);
        StockhamRun<N, NS * R, REM - ilog2c(R), INV, TW>::run(buf, tpf_id, tw);
    }
};
template <int N, int NS, bool INV, class TW>
struct StockhamRun<N, NS, 0, INV, TW> {
    __device__ __forceinline__ static void run(double2*, int, const TW&) {}
};

// Full length-N FFT on buf (caller syncs before; ends synced).  N >= 16.
template <int N, bool INV, class TW>
__device__ __forceinline__ void fft_smem(double2* buf, int tpf_id, const TW& tw) {
    StockhamRun<N, 1, ilog2c(N), INV, TW>::run(buf, tpf_id, tw);
}

}  // namespace sfftb

namespace sfftb {

// ---------------------------------------------------------------------------
// Two-pass register FFT of length N = 16 * R2 (R2 in {8, 16}) by T = N/16
// threads holding 16 elements each.  Pass 1 (radix 16) runs on the inputs
// the thread loaded itself, one shared-memory transpose feeds pass 2
// (radix R2), and the outputs stay in registers -- one smem round trip per
// FFT instead of one per pass plus staging.
//
//   in : v[r]  = x[t + r*T],            r < 16
//   out: v[e]  = X[fft2_out_index<N>(t, e)] = X[t + (e / R2) * T + 16 * (e % R2)]
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ int fft2_out_index(int t, int e) {
    constexpr int R2 = N / 16, T = N / 16;
    return t + (e / R2) * T + 16 * (e % R2);
}

// Reorder pass outputs (index fft2_out_index) into the next FFT's pass-1
// input order (x[t + r*T]) -- the same set of indices, permuted.
template <int N>
__device__ __forceinline__ void fft2_out_to_in(double2 (&v)[16]) {
    constexpr int R2 = N / 16, T = N / 16;
    if constexpr (R2 == 16) {
        return;  // k = t + 16 e == t + T e
    } else {
        // out e = q*R2 + r holds t + q*T + 16 r; input slot rr holds t + rr*T,
        // so rr = q + r * (16 / T)
        double2 w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int q = e / R2, r = e % R2;
            w[q + r * (16 / T)] = v[e];
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = w[e];
    }
}

// p[r] = s^r, r < R (R in {2, 4, 8, 16}), from s, s^2, s^4, s^8 by binary
// powers: at most three complex products (roundings) per entry.  Replaces R
// table loads per thread by four -- the twiddle lookups were the largest
// share of the shared-memory traffic (and of its bank conflicts).
template <int R>
__device__ __forceinline__ void pow_table(double2 s1, double2 s2, double2 s4, double2 s8,
                                          double2 (&p)[R]) {
    p[0] = make_double2(1.0, 0.0);
    if constexpr (R > 1) p[1] = s1;
    if constexpr (R > 2) {
        p[2] = s2;
        p[3] = cmul(s1, s2);
    }
    if constexpr (R > 4) {
        p[4] = s4;
        p[5] = cmul(s1, s4);
        p[6] = cmul(s2, s4);
        p[7] = cmul(p[3], s4);
    }
    if constexpr (R > 8) {
        p[8] = s8;
#pragma unroll
        for (int r = 9; r < 16; ++r) p[r] = cmul(p[r - 8], s8);
    }
}

// s^r, r < 16, as q4[r >> 2] * q1[r & 3] with q1 = {1, s, s^2, s^3} and
// q4 = {1, s^4, s^8, s^12}: 8 live values instead of pow_table's 16, at most
// three roundings per power.
struct Pow16 {
    double2 q1[4], q4[4];
    __device__ __forceinline__ Pow16(double2 s1, double2 s2, double2 s4, double2 s8) {
        q1[0] = q4[0] = make_double2(1.0, 0.0);
        q1[1] = s1;
        q1[2] = s2;
        q1[3] = cmul(s1, s2);
        q4[1] = s4;
        q4[2] = s8;
        q4[3] = cmul(s4, s8);
    }
    __device__ __forceinline__ double2 operator()(int r) const {
        const int a = r >> 2, c = r & 3;
        return a ? (c ? cmul(q4[a], q1[c]) : q4[a]) : q1[c];
    }
};

__device__ __forceinline__ double2 conj_if_b(double2 w, bool c) {
    if (c) w.y = -w.y;
    return w;
}

template <int N, bool INV>
__device__ __forceinline__ void fft2pass(double2 (&v)[16], double2* __restrict__ slot, int t,
                                         const double2* __restrict__ tw) {
    constexpr int R2 = N / 16, T = N / 16, BPT = 16 / R2;
    dft_reg<16, INV>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) slot[pad16(t * 16 + r)] = v[r];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int j = t + q * T;
        double2 u[R2];
#pragma unroll
        for (int r = 0; r < R2; ++r) u[r] = slot[pad16(j + 16 * r)];
        // twiddles e^{-+2 pi i jm r / N}, r < R2, from the powers of tw[jm]
        // (jm = 0 gives exact ones: the products of (1, 0) are exact)
        const int jm = j & 15;
        const double2 one = make_double2(1.0, 0.0);
        const double2 s1 = conj_if_b(tw[jm], INV);
        const double2 s2 = conj_if_b(tw[2 * jm], INV);
        const double2 s4 = R2 > 4 ? conj_if_b(tw[4 * jm], INV) : one;
        const double2 s8 = R2 > 8 ? conj_if_b(tw[8 * jm], INV) : one;
        const Pow16 p(s1, s2, s4, s8);
#pragma unroll
        for (int r = 1; r < R2; ++r) u[r] = cmul(u[r], p(r));
        dft_reg<R2, INV>(u);
#pragma unroll
        for (int r = 0; r < R2; ++r) v[q * R2 + r] = u[r];
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Radix-3 and radix-12 register DFTs (natural order in and out), for the
// mixed-radix four-step length N = 3 * 2^k (row FFTs of length 192).
// ---------------------------------------------------------------------------
template <bool INV>
__device__ __forceinline__ void dft3(double2& a, double2& b, double2& c) {
    constexpr double h = 0.86602540378443864676;  // sqrt(3)/2
    const double2 s = cadd(b, c), d = csub(b, c);
    const double2 m = make_double2(a.x - 0.5 * s.x, a.y - 0.5 * s.y);
    // forward: X1 = m - i h d, X2 = m + i h d (e^{-2 pi i/3} = -1/2 - i h)
    const double2 rot = INV ? make_double2(-h * d.y, h * d.x) : make_double2(h * d.y, -h * d.x);
    a = cadd(a, s);
    b = cadd(m, rot);
    c = csub(m, rot);
}

// e^{-+2 pi i k/12}, k in [0, 12)
template <bool INV>
__device__ __forceinline__ double2 w12(int k) {
    constexpr double h = 0.86602540378443864676;
    double2 w;
    switch (k) {
        case 0: w = make_double2(1.0, 0.0); break;
        case 1: w = make_double2(h, -0.5); break;
        case 2: w = make_double2(0.5, -h); break;
        case 3: w = make_double2(0.0, -1.0); break;
        case 4: w = make_double2(-0.5, -h); break;
        case 5: w = make_double2(-h, -0.5); break;
        default: w = make_double2(-1.0, 0.0); break;  // 6
    }
    if (INV) w.y = -w.y;
    return w;
}

// 12-point DFT: n = 4a + b, k = c + 3d (a, c < 3; b, d < 4):
// X[c + 3d] = sum_b w4^{bd} w12^{bc} (sum_a x[4a + b] w3^{ac}).
template <bool INV>
__device__ __forceinline__ void dft12(double2 (&v)[12]) {
    double2 y[4][3];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        double2 p = v[b], q = v[4 + b], r = v[8 + b];
        dft3<INV>(p, q, r);
        y[b][0] = p;
        y[b][1] = b ? cmul(q, w12<INV>(b)) : q;
        y[b][2] = b ? cmul(r, w12<INV>(2 * b)) : r;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double2 u[4] = {y[0][c], y[1][c], y[2][c], y[3][c]};
        dft_reg<4, INV>(u);
#pragma unroll
        for (int d = 0; d < 4; ++d) v[c + 3 * d] = u[d];
    }
}

// Four-step twiddle of pass outputs: v[e] *= w^(a * fft2_out_index<N>(t, e)),
// w = e^{-+2 pi i / NT} from the two-level tables of the full length NT.
// Per output group g the base w^(a (t + g T)) times (w^(16 a))^r, the powers
// by pow_table: 5-6 table lookups per thread instead of 16 pairs.
template <int N, bool INV>
__device__ __forceinline__ void out_twiddle(double2 (&v)[16], int a, int t,
                                            const double2* __restrict__ hi,
                                            const double2* __restrict__ lo) {
    constexpr int R2 = N / 16, T = N / 16, BPT = 16 / R2;
    if (a == 0) return;  // every exponent is 0
    const double2 one = make_double2(1.0, 0.0);
    const double2 s1 = twiddle2<INV>(hi, lo, 16 * a);
    const double2 s2 = twiddle2<INV>(hi, lo, 32 * a);
    const double2 s4 = R2 > 4 ? twiddle2<INV>(hi, lo, 64 * a) : one;
    const double2 s8 = R2 > 8 ? twiddle2<INV>(hi, lo, 128 * a) : one;
    const Pow16 p(s1, s2, s4, s8);
#pragma unroll
    for (int g = 0; g < BPT; ++g) {
        const int e0 = a * (t + g * T);
        const double2 b = twiddle2<INV>(hi, lo, e0);  // e0 == 0: exactly (1, 0)
        v[g * R2] = cmul(v[g * R2], b);
#pragma unroll
        for (int r = 1; r < R2; ++r) v[g * R2 + r] = cmul(v[g * R2 + r], cmul(b, p(r)));
    }
}

}  // namespace sfftb
