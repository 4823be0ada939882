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
    if constexpr (e == 0) return a;
    else if constexpr (e == 1) return V{(a.x + a.y) * h, (a.y - a.x) * h};    // (1 - i)/sqrt2
    else if constexpr (e == 2) return V{a.y, -a.x};                            // -i
    else if constexpr (e == 3) return V{(a.y - a.x) * h, -(a.x + a.y) * h};   // (-1 - i)/sqrt2
    else if constexpr (e == 4) return V{-a.x, -a.y};
    else if constexpr (e == 5) return V{-(a.x + a.y) * h, (a.x - a.y) * h};   // (-1 + i)/sqrt2
    else if constexpr (e == 6) return V{-a.y, a.x};                            // +i
    else return V{(a.x - a.y) * h, (a.x + a.y) * h};                           // (1 + i)/sqrt2
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

template <int P, int S> struct Dft;

template <int S> struct Dft<1, S> {
    template <typename V> static __device__ __forceinline__ void run(V (&)[1]) {}
};

template <int S> struct Dft<2, S> {
    template <typename V> static __device__ __forceinline__ void run(V (&z)[2]) {
        const V a = z[0], b = z[1];
        z[0] = cadd(a, b);
        z[1] = csub(a, b);
    }
};

template <int S> struct Dft<3, S> {
    template <typename V> static __device__ __forceinline__ void run(V (&z)[3]) {
        using T = decltype(z[0].x);
        const T s = (T)(S * PAFFT_SIN60);
        const V t1 = cadd(z[1], z[2]);
        const V t2 = csub(z[1], z[2]);
        const V m{z[0].x - (T)0.5 * t1.x, z[0].y - (T)0.5 * t1.y};
        z[0] = cadd(z[0], t1);
        z[1] = V{m.x + s * t2.y, m.y - s * t2.x};
        z[2] = V{m.x - s * t2.y, m.y + s * t2.x};
    }
};

template <int S> struct Dft<4, S> {
    template <typename V> static __device__ __forceinline__ void run(V (&z)[4]) {
        const V t0 = cadd(z[0], z[2]), t1 = csub(z[0], z[2]);
        const V t2 = cadd(z[1], z[3]), t3 = rot_mi<S>(csub(z[1], z[3]));
        z[0] = cadd(t0, t2);
        z[2] = csub(t0, t2);
        z[1] = cadd(t1, t3);
        z[3] = csub(t1, t3);
    }
};

template <int S> struct Dft<5, S> {
    template <typename V> static __device__ __forceinline__ void run(V (&z)[5]) {
        using T = decltype(z[0].x);
        const T c1 = (T)PAFFT_C51, c2 = (T)PAFFT_C52;
        const T s1 = (T)(S * PAFFT_S51), s2 = (T)(S * PAFFT_S52);
        const V t1 = cadd(z[1], z[4]), t2 = cadd(z[2], z[3]);
        const V t3 = csub(z[1], z[4]), t4 = csub(z[2], z[3]);
        const V a = z[0];
        const V m1{a.x + c1 * t1.x + c2 * t2.x, a.y + c1 * t1.y + c2 * t2.y};
        const V m2{a.x + c2 * t1.x + c1 * t2.x, a.y + c2 * t1.y + c1 * t2.y};
        const V n1{s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y};
        const V n2{s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y};
        z[0] = V{a.x + t1.x + t2.x, a.y + t1.y + t2.y};
        // Z1 = m1 - i n1, Z4 = m1 + i n1, Z2 = m2 - i n2, Z3 = m2 + i n2
        z[1] = V{m1.x + n1.y, m1.y - n1.x};
        z[4] = V{m1.x - n1.y, m1.y + n1.x};
        z[2] = V{m2.x + n2.y, m2.y - n2.x};
        z[3] = V{m2.x - n2.y, m2.y + n2.x};
    }
};

template <int S> struct Dft<8, S> {
    template <typename V> static __device__ __forceinline__ void run(V (&z)[8]) {
        V e[4] = {z[0], z[2], z[4], z[6]};
        V o[4] = {z[1], z[3], z[5], z[7]};
        Dft<4, S>::run(e);
        Dft<4, S>::run(o);
        o[1] = rot8<1, S>(o[1]);
        o[2] = rot8<2, S>(o[2]);
        o[3] = rot8<3, S>(o[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            z[k] = cadd(e[k], o[k]);
            z[k + 4] = csub(e[k], o[k]);
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

template <int P, int S> struct Dft {
    static constexpr int A = Split<P>::A;
    static constexpr int B = P / A;
    // m = m1*B + m2, k = k1 + A*k2:
    // Z[k1 + A k2] = sum_m2 w_B^{m2 k2} [ w_P^{m2 k1} sum_m1 w_A^{m1 k1} z[m1 B + m2] ]
    template <typename V> static __device__ __forceinline__ void run(V (&z)[P]) {
        V v[P];
        static_for<0, B>([&](auto m2c) {
            constexpr int m2 = decltype(m2c)::value;
            V u[A];
#pragma unroll
            for (int m1 = 0; m1 < A; ++m1) u[m1] = z[m1 * B + m2];
            Dft<A, S>::run(u);
            static_for<0, A>([&](auto k1c) {
                constexpr int k1 = decltype(k1c)::value;
                v[k1 * B + m2] = twiddle_const<P, k1 * m2, S>(u[k1]);
            });
        });
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) {
            V t[B];
#pragma unroll
            for (int m2 = 0; m2 < B; ++m2) t[m2] = v[k1 * B + m2];
            Dft<B, S>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) z[k1 + A * k2] = t[k2];
        }
    }
};

}  // namespace pafft_b200
