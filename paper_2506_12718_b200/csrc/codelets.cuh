// In-register DFT codelets for the sm_100a pass kernels.
//
// Dft<P, S>::run(z) replaces the P complex values held in registers by their
// DFT, natural order in and out:  Z[k] = sum_m z[m] * w^(S*m*k),
// w = exp(-2 pi i / P).  S = +1 is the forward kernel F_P used by the DIF
// ladder A^T (butterfly.cpp:58-75 / :155-193 / :307-379 combine with F_r);
// S = -1 is conj(F_P), used by the conjugate ladder A-bar (butterfly.cpp:39-56).
// Primitive sizes 2, 3, 4, 5, 8 are written out (Eq. 25);
// composite sizes are in-register Cooley-Tukey with compile-time constant
// twiddles from roots.h (trivial quarter/eighth turns are folded exactly).
// Everything is fully unrolled: indices are compile-time, so the arrays live
// in registers and the data movement between sub-DFTs is free renaming.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "roots.h"

namespace pafft_b200 {

// Compile-time loop: f(std::integral_constant<int, I>) for I in [Begin, End).
template <int Begin, int End, typename F> __device__ __forceinline__ void static_for(F&& f) {
    if constexpr (Begin < End) {
        f(std::integral_constant<int, Begin>{});
        static_for<Begin + 1, End>(f);
    }
}

template <typename T> struct Cplx;
template <> struct Cplx<double> { using type = double2; };
template <> struct Cplx<float> { using type = float2; };
template <typename T> using cplx = typename Cplx<T>::type;

// fp32 complex arithmetic on Blackwell's packed fp32 pipe: one complex value is
// one 64-bit register pair, add.f32x2 / mul.f32x2 / fma.f32x2 (FADD2, FMUL2,
// FFMA2) work on both halves at once and take broadcast, swap and per-half sign
// operand modifiers, so a complex add is one instruction instead of two, a
// real-constant multiply-add one instead of two and a complex multiply two or
// three instead of four.  The pipe's lane throughput is that of scalar FFMA
// (tools/probes/ffma2.cu): what is saved is issue slots, which bound the fp32
// passes (85% of the fp32 CONV's instructions were FFMA/FADD/FMUL).
#ifndef PAFFT_F32X2
#define PAFFT_F32X2 1
#endif
#if PAFFT_F32X2
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, float2{-b.x, -b.y}); }
// a * b = a.x (b.x, b.y) + (-s.x, s.y), s = a.y (b.y, b.x): FMUL2 with a
// broadcast and a swapped operand, then FFMA2 whose addend takes the per-half
// sign as an operand modifier -- two instructions, no register moves
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    const float2 s = __fmul2_rn(float2{a.y, a.y}, float2{b.y, b.x});
    return __ffma2_rn(float2{a.x, a.x}, b, float2{-s.x, s.y});
}
// a * conj(b) = a.y (b.y, b.x) + (t.x, -t.y), t = a.x (b.x, b.y)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    const float2 t = __fmul2_rn(float2{a.x, a.x}, b);
    return __ffma2_rn(float2{a.y, a.y}, float2{b.y, b.x}, float2{t.x, -t.y});
}
#endif
// a + s b, a - s b, s b for a real s (both halves the same factor)
template <typename V, typename T> __device__ __forceinline__ V caxpy(V a, T s, V b) {
    if constexpr (PAFFT_F32X2 && sizeof(T) == 4) return __ffma2_rn(float2{s, s}, b, a);
    else return V{a.x + s * b.x, a.y + s * b.y};
}
template <typename V, typename T> __device__ __forceinline__ V cscale(T s, V b) {
    if constexpr (PAFFT_F32X2 && sizeof(T) == 4) return __fmul2_rn(float2{s, s}, b);
    else return V{s * b.x, s * b.y};
}
// a - i s b = (a.x + s b.y, a.y - s b.x)  and  a + i s b
template <typename V, typename T> __device__ __forceinline__ V caxpy_mi(V a, T s, V b) {
    if constexpr (PAFFT_F32X2 && sizeof(T) == 4) return __ffma2_rn(float2{s, -s}, float2{b.y, b.x}, a);
    else return V{a.x + s * b.y, a.y - s * b.x};
}
template <typename V, typename T> __device__ __forceinline__ V caxpy_pi(V a, T s, V b) {
    if constexpr (PAFFT_F32X2 && sizeof(T) == 4) return __ffma2_rn(float2{-s, s}, float2{b.y, b.x}, a);
    else return V{a.x - s * b.y, a.y + s * b.x};
}
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return V{a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return V{a.x - b.x, a.y - b.y}; }
// a * b
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    return V{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
    return V{a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
// a * w^S with w given (S = -1 uses conj(w))
template <int S, typename V> __device__ __forceinline__ V cmul_s(V a, V w) {
    if constexpr (S > 0) return cmul(a, w);
    else return cmulc(a, w);
}
// a * (-i)^S : S=+1 -> -i a = (a.y, -a.x); S=-1 -> +i a = (-a.y, a.x)
template <int S, typename V> __device__ __forceinline__ V rot_mi(V a) {
    if constexpr (S > 0) return V{a.y, -a.x};
    else return V{-a.y, a.x};
}

// a * exp(-2 pi i S e / 8) for e in [0, 8), exact at quarter turns.
template <int E, int S, typename V> __device__ __forceinline__ V rot8(V a) {
    using T = decltype(a.x);
    constexpr int e = ((E * S) % 8 + 8) % 8;
    const T h = (T)PAFFT_SQRTH;
    if constexpr (PAFFT_F32X2 && sizeof(T) == 4) {
        // odd eighth turns as h (a +- (-i a)): two packed instructions
        if constexpr (e == 0) return a;
        else if constexpr (e == 1) return cscale(h, cadd(a, V{a.y, -a.x}));    // (1 - i)/sqrt2
        else if constexpr (e == 2) return V{a.y, -a.x};                          // -i
        else if constexpr (e == 3) return cscale(h, csub(V{a.y, -a.x}, a));    // (-1 - i)/sqrt2
        else if constexpr (e == 4) return V{-a.x, -a.y};
        else if constexpr (e == 5) return cscale((T)-h, cadd(a, V{a.y, -a.x}));  // (-1 + i)/sqrt2
        else if constexpr (e == 6) return V{-a.y, a.x};                          // +i
        else return cscale(h, csub(a, V{a.y, -a.x}));                           // (1 + i)/sqrt2
    } else {
        if constexpr (e == 0) return a;
        else if constexpr (e == 1) return V{(a.x + a.y) * h, (a.y - a.x) * h};    // (1 - i)/sqrt2
        else if constexpr (e == 2) return V{a.y, -a.x};                            // -i
        else if constexpr (e == 3) return V{(a.y - a.x) * h, -(a.x + a.y) * h};   // (-1 - i)/sqrt2
        else if constexpr (e == 4) return V{-a.x, -a.y};
        else if constexpr (e == 5) return V{-(a.x + a.y) * h, (a.x - a.y) * h};   // (-1 + i)/sqrt2
        else if constexpr (e == 6) return V{-a.y, a.x};                            // +i
        else return V{(a.x - a.y) * h, (a.x + a.y) * h};                           // (1 + i)/sqrt2
    }
}

// a * exp(-2 pi i S e / P) with compile-time P, e.
template <int P, int E, int S, typename V> __device__ __forceinline__ V twiddle_const(V a) {
    using T = decltype(a.x);
    constexpr int e = E % P;
    if constexpr (e == 0) return a;
    else if constexpr ((8 * e) % P == 0) return rot8<(8 * e) / P, S>(a);
    else {
        const V w{RootTable<P, T>::re(e), RootTable<P, T>::im(e)};
        return cmul_s<S>(a, w);
    }
}

// Codelets work in place on a register array z at compile-time positions
// z[OFF + i*ST], i < P: input index i, output frequency k left at
// z[OFF + pos(k)*ST].  Primitive sizes have pos(k) = k; composite sizes keep
// their sub-results where they were computed (no transposition moves), so the
// live register set stays ~P complex values.
template <int P, int S> struct Dft;

template <int S> struct Dft<1, S> {
    static constexpr int pos(int k) { return k; }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&)[N]) {}
};

template <int S> struct Dft<2, S> {
    static constexpr int pos(int k) { return k; }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&z)[N]) {
        const V a = z[OFF], b = z[OFF + ST];
        z[OFF] = cadd(a, b);
        z[OFF + ST] = csub(a, b);
    }
};

template <int S> struct Dft<3, S> {
    static constexpr int pos(int k) { return k; }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&z)[N]) {
        using T = decltype(z[0].x);
        const T s = (T)(S * PAFFT_SIN60);
        const V a = z[OFF];
        const V t1 = cadd(z[OFF + ST], z[OFF + 2 * ST]);
        const V t2 = csub(z[OFF + ST], z[OFF + 2 * ST]);
        if constexpr (PAFFT_F32X2 && sizeof(T) == 4) {
            const V m = caxpy(a, (T)-0.5, t1);
            z[OFF] = cadd(a, t1);
            z[OFF + ST] = caxpy_mi(m, s, t2);
            z[OFF + 2 * ST] = caxpy_pi(m, s, t2);
        } else {
            const V m{a.x - (T)0.5 * t1.x, a.y - (T)0.5 * t1.y};
            z[OFF] = cadd(a, t1);
            z[OFF + ST] = V{m.x + s * t2.y, m.y - s * t2.x};
            z[OFF + 2 * ST] = V{m.x - s * t2.y, m.y + s * t2.x};
        }
    }
};

template <int S> struct Dft<4, S> {
    static constexpr int pos(int k) { return k; }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&z)[N]) {
        const V t0 = cadd(z[OFF], z[OFF + 2 * ST]), t1 = csub(z[OFF], z[OFF + 2 * ST]);
        const V t2 = cadd(z[OFF + ST], z[OFF + 3 * ST]);
        const V t3 = rot_mi<S>(csub(z[OFF + ST], z[OFF + 3 * ST]));
        z[OFF] = cadd(t0, t2);
        z[OFF + 2 * ST] = csub(t0, t2);
        z[OFF + ST] = cadd(t1, t3);
        z[OFF + 3 * ST] = csub(t1, t3);
    }
};

template <int S> struct Dft<5, S> {
    static constexpr int pos(int k) { return k; }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&z)[N]) {
        using T = decltype(z[0].x);
        const T c1 = (T)PAFFT_C51, c2 = (T)PAFFT_C52;
        const T s1 = (T)(S * PAFFT_S51), s2 = (T)(S * PAFFT_S52);
        const V a = z[OFF];
        const V t1 = cadd(z[OFF + ST], z[OFF + 4 * ST]), t2 = cadd(z[OFF + 2 * ST], z[OFF + 3 * ST]);
        const V t3 = csub(z[OFF + ST], z[OFF + 4 * ST]), t4 = csub(z[OFF + 2 * ST], z[OFF + 3 * ST]);
        // Z1 = m1 - i n1, Z4 = m1 + i n1, Z2 = m2 - i n2, Z3 = m2 + i n2
        if constexpr (PAFFT_F32X2 && sizeof(T) == 4) {
            const V m1 = caxpy(caxpy(a, c1, t1), c2, t2);
            const V m2 = caxpy(caxpy(a, c2, t1), c1, t2);
            const V n1 = caxpy(cscale(s1, t3), s2, t4);
            const V n2 = caxpy(cscale(s2, t3), (T)-s1, t4);
            z[OFF] = cadd(cadd(a, t1), t2);
            z[OFF + ST] = caxpy_mi(m1, (T)1, n1);
            z[OFF + 4 * ST] = caxpy_pi(m1, (T)1, n1);
            z[OFF + 2 * ST] = caxpy_mi(m2, (T)1, n2);
            z[OFF + 3 * ST] = caxpy_pi(m2, (T)1, n2);
        } else {
            const V m1{a.x + c1 * t1.x + c2 * t2.x, a.y + c1 * t1.y + c2 * t2.y};
            const V m2{a.x + c2 * t1.x + c1 * t2.x, a.y + c2 * t1.y + c1 * t2.y};
            const V n1{s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y};
            const V n2{s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y};
            z[OFF] = V{a.x + t1.x + t2.x, a.y + t1.y + t2.y};
            z[OFF + ST] = V{m1.x + n1.y, m1.y - n1.x};
            z[OFF + 4 * ST] = V{m1.x - n1.y, m1.y + n1.x};
            z[OFF + 2 * ST] = V{m2.x + n2.y, m2.y - n2.x};
            z[OFF + 3 * ST] = V{m2.x - n2.y, m2.y + n2.x};
        }
    }
};

template <int S> struct Dft<8, S> {
    static constexpr int pos(int k) { return k; }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&z)[N]) {
        V e[4] = {z[OFF], z[OFF + 2 * ST], z[OFF + 4 * ST], z[OFF + 6 * ST]};
        V o[4] = {z[OFF + ST], z[OFF + 3 * ST], z[OFF + 5 * ST], z[OFF + 7 * ST]};
        Dft<4, S>::template run<1, 0>(e);
        Dft<4, S>::template run<1, 0>(o);
        o[1] = rot8<1, S>(o[1]);
        o[2] = rot8<2, S>(o[2]);
        o[3] = rot8<3, S>(o[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            z[OFF + k * ST] = cadd(e[k], o[k]);
            z[OFF + (k + 4) * ST] = csub(e[k], o[k]);
        }
    }
};

// Composite split P = A * B used by the generic Cooley-Tukey codelet.
template <int P> struct Split;
template <> struct Split<9> { static constexpr int A = 3; };
template <> struct Split<16> { static constexpr int A = 4; };
template <> struct Split<25> { static constexpr int A = 5; };
template <> struct Split<27> { static constexpr int A = 3; };
template <> struct Split<32> { static constexpr int A = 4; };
template <> struct Split<64> { static constexpr int A = 8; };
template <> struct Split<81> { static constexpr int A = 9; };
template <> struct Split<125> { static constexpr int A = 5; };

// In-place Cooley-Tukey: index m = m1*B + m2, frequency k = k1 + A*k2.
//   (1) for each column m2: A-point DFT over m1 (stride B), in place;
//       twiddle the result for k1 by w_P^{m2 k1};
//   (2) for each k1 (row at A-position pos_A(k1)): B-point DFT over m2.
// Frequency k1 + A k2 ends at pos_A(k1) * B + pos_B(k2).
template <int P, int S> struct Dft {
    static constexpr int A = Split<P>::A;
    static constexpr int B = P / A;
    static constexpr int pos(int k) { return Dft<A, S>::pos(k % A) * B + Dft<B, S>::pos(k / A); }
    template <int ST, int OFF, typename V, int N> static __device__ __forceinline__ void run(V (&z)[N]) {
        static_for<0, B>([&](auto m2c) {
            constexpr int m2 = decltype(m2c)::value;
            Dft<A, S>::template run<ST * B, OFF + m2 * ST>(z);
            static_for<1, A>([&](auto k1c) {
                constexpr int k1 = decltype(k1c)::value;
                constexpr int slot = OFF + (Dft<A, S>::pos(k1) * B + m2) * ST;
                z[slot] = twiddle_const<P, k1 * m2, S>(z[slot]);
            });
        });
        static_for<0, A>([&](auto k1c) {
            constexpr int k1 = decltype(k1c)::value;
            Dft<B, S>::template run<ST, OFF + Dft<A, S>::pos(k1) * B * ST>(z);
        });
    }
};

// Whole-array transform with natural-order result (z[k] = frequency k): the
// in-place codelet followed by a compile-time renaming (no data movement).
template <int P, int S, typename V> __device__ __forceinline__ void dft(V (&z)[P]) {
    Dft<P, S>::template run<1, 0>(z);
    if constexpr (P > 1) {
        V w[P];
#pragma unroll
        for (int k = 0; k < P; ++k) w[k] = z[Dft<P, S>::pos(k)];
#pragma unroll
        for (int k = 0; k < P; ++k) z[k] = w[k];
    }
}

// z[k] *= w^(k) for k = 1 .. F-1 (S = -1: conj(w)^k).  Codelets of fewer
// than PAFFT_CHEB_MIN points build w^k by binary powering in registers (error
// ~ log2(F) roundings); larger ones by the Chebyshev three-term recurrence
// w^{k+1} = 2 cos(theta) w^k - w^{k-1} (|w| = 1): two FMAs per power instead
// of a complex multiply, on a longer dependency chain.  Measured on B200 with
// the threshold at 16: config 1 +4%, config 5 +2.3%, config 2 neutral, but
// config 3 -2.8% and config 4 -10% (16-point CONV tiles at 12 warps/SM cannot
// hide the chain), so it is used from 25 points on (config 5's codelets), and
// from 16 points in contiguous tiles of >= 256 threads (CHEB16: config 1,
// +3.3%, 5.2e-15 relative L2).
// The recurrence's error grows ~k cot(theta) ulps: config 5 1.1e-14 relative
// L2 vs 1.9e-15 with binary powering, against the 1e-12 bar
// (tools/accuracy_probe.py).
#ifndef PAFFT_CHEB_MIN
#define PAFFT_CHEB_MIN 25
#endif
// fp32 twiddle powers by binary powering only: the Chebyshev recurrence's
// error growth (~k cot(theta) ulps) costs 7x accuracy in fp32 (config 5 fp32:
// 7.0e-6 relative L2 against the 1e-5 bar, 1.0e-6 with binary powers;
// configs 1/3/4 fp32 3x) for 2% of config 5 fp32 speed (config 1 fp32 +2%)
#ifndef PAFFT_CHEB_F32
#define PAFFT_CHEB_F32 0
#endif
template <int F, int S, bool CHEB16 = false, typename V>
__device__ __forceinline__ void twiddle_powers(V (&z)[F], V w) {
    if constexpr (F > 1) {
        if constexpr (S < 0) w.y = -w.y;
        if constexpr ((F >= PAFFT_CHEB_MIN || (CHEB16 && F >= 16)) && (PAFFT_CHEB_F32 || sizeof(w.x) == 8)) {
            using T = decltype(w.x);
            const T c2 = w.x + w.x;
            V pm{(T)1, (T)0}, pc = w;
            z[1] = cmul(z[1], w);
#pragma unroll
            for (int k = 2; k < F; ++k) {
                const V pn{c2 * pc.x - pm.x, c2 * pc.y - pm.y};
                z[k] = cmul(z[k], pn);
                pm = pc;
                pc = pn;
            }
        } else {
            V p[F];
            p[1] = w;
#pragma unroll
            for (int k = 2; k < F; ++k) p[k] = (k & 1) ? cmul(p[k - 1], p[1]) : cmul(p[k / 2], p[k / 2]);
#pragma unroll
            for (int k = 1; k < F; ++k) z[k] = cmul(z[k], p[k]);
        }
    }
}

}  // namespace pafft_b200
