// Stage-group pass kernels: the sm_100a replacement for pafft's in-place
// stage ladders (butterfly.cpp:20-379), tensor driver (butterfly.cpp:423-466),
// pointwise product (convolution.cpp:23-35) and 1/n sweep (core.cpp:79-82).
//
// A pass runs s consecutive radix-r stages of one axis.  With a stages already
// done, block size K0 = n_q / r^a, R = r^s and L = K0 / R, the stages act on
// closed sets {j + m L} (m < R) inside each block, so the signal is viewed as
//     [panel][R rows][C = L * sq columns]      (sq = stride of axis q)
// and a pass is an R-point transform down every column:
//   DIF  (A^T group, butterfly.cpp:58-75):  out[rev(k)] = w_K0^{jj k} DFT_R(col)[k]
//   DIT  (A / A-bar group, :20-56):         out[m] = sum_k w_R^{+-mk} w_K0^{+-jj k} in[rev(k)]
// where jj = column / sq and rev is the base-r digit reversal of s digits
// (permutation.cpp:27-37).  The DIF output is therefore already in the
// reference's index-reversed order: no permutation is ever executed.
//   CONV (the middle pass) = DIF group, x ghat (the reversed filter, 1/N folded
// in on the device), DIT-conj group, all on one contiguous block in one kernel
// (convolve_permfree, convolution.cpp:45-52, north_star item 3).
//
// Inside a tile the R-point column transform is R = R1 * R2 * R3 with
// in-register codelets (codelets.cuh) and shared-memory exchanges between
// steps (four-step decomposition with internal twiddles w_R, w_{R2 R3} from
// L1-resident tables laid out for the access pattern).  Each codelet size is a
// power of r, so rev(k) splits per step.  Layout is interleaved complex
// (double2 / float2): every element is one 16-byte (8-byte) vector access.
#pragma once

#include "codelets.cuh"

namespace pafft_b200 {

enum PassKind : int { KIND_DIF = 0, KIND_DIT_FWD = 1, KIND_DIT_CONJ = 2, KIND_CONV = 3 };

template <typename T> struct PassArgs {
    const cplx<T>* src;
    cplx<T>* dst;
    long long tiles;
    long long panels;        // total panels over the batch
    long long panel_elems;   // R * C
    int C;                   // columns per panel (contiguous)
    int W;                   // tile width: columns (strided) or panels (contig)
    int contig;              // 1: C == 1, tile = W consecutive panels
    int tiles_per_panel;     // ceil(C / W) for strided tiles
    // external twiddle w_K0^{jj k}, jj = column / sq, two-level table
    int ext;
    unsigned sq;
    unsigned ext_bits;
    const cplx<T>* ext_lo;   // w_K0^{e},           e < 2^bits
    const cplx<T>* ext_hi;   // w_K0^{h * 2^bits},  h < ceil(K0 / 2^bits)
    // internal twiddles
    const cplx<T>* tw1;      // [k1][m23] = w_R^{k1 m23}
    const cplx<T>* tw2;      // [k2][m3]  = w_{R2 R3}^{k2 m3}
    // CONV filter (digit-reversed, pre-scaled by 1/N) and signal period
    const cplx<T>* ghat;
    long long N;
    // DIT epilogue: natural-order multiplier (period N) and/or scale
    const cplx<T>* mul;
    T scale;
    int has_scale;
};

// Base-r digit reversal over the digits of P = r^s (permutation.cpp:27-37).
template <int RADIX, int P> __device__ __forceinline__ int revd(int k) {
    int o = 0;
#pragma unroll
    for (int p = 1; p < P; p *= RADIX) {
        o = o * RADIX + k % RADIX;
        k /= RADIX;
    }
    return o;
}

template <typename T>
__device__ __forceinline__ cplx<T> ext_root(const PassArgs<T>& a, unsigned long long e) {
    const cplx<T> lo = __ldg(a.ext_lo + (e & ((1ull << a.ext_bits) - 1)));
    const cplx<T> hi = __ldg(a.ext_hi + (e >> a.ext_bits));
    return cmul(lo, hi);
}

template <typename T, int RADIX, int R1, int R2, int R3, int KIND>
__global__ void __launch_bounds__(256) pass_kernel(PassArgs<T> a) {
    using V = cplx<T>;
    constexpr int R = R1 * R2 * R3;
    constexpr int R23 = R2 * R3;
    constexpr int NSTEP = 1 + (R2 > 1 ? 1 : 0) + (R3 > 1 ? 1 : 0);
    static_assert(R3 == 1 || R2 > 1, "R3 > 1 requires R2 > 1");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* sm = reinterpret_cast<V*>(smem_raw);

    const int W = a.W;
    const int NT = blockDim.x;
    const int tid = threadIdx.x;
    const bool contig = a.contig != 0;

    for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        // ---- tile geometry: element (row m, tile column c) at base + m*rs + c*cs
        long long base, first;  // first: first panel (contig) or column (strided)
        int nvalid;
        long long rs, cs;
        if (contig) {
            first = tile * W;
            const long long left = a.panels - first;
            nvalid = left < W ? (int)left : W;
            base = first * (long long)R;
            rs = 1;
            cs = R;
        } else {
            const long long p = tile / a.tiles_per_panel;
            first = (tile - p * a.tiles_per_panel) * (long long)W;
            const long long left = a.C - first;
            nvalid = left < W ? (int)left : W;
            base = p * a.panel_elems + first;
            rs = a.C;
            cs = 1;
        }
        const V* __restrict__ src = a.src;
        V* __restrict__ dst = a.dst;
        auto sidx = [&](int j, int c) -> int { return contig ? c * R + j : j * W + c; };
        auto item = [&](int w, int G, int& g, int& c) {
            if (contig) { g = w % G; c = w / G; }
            else { c = w % W; g = w / W; }
        };
        // external twiddle base/step for column c: w_K0^{jj kf}, w_K0^{jj S}
        auto ext_pair = [&](int c, int kf, int S, V& t, V& s) {
            const unsigned long long col = (unsigned long long)(first + c);
            const unsigned long long jj = col / a.sq;
            t = ext_root(a, jj * (unsigned long long)kf);
            s = ext_root(a, jj * (unsigned long long)S);
        };

        if constexpr (KIND == KIND_DIF || KIND == KIND_CONV) {
            // ------------------------------------------------ DIF step 1
            {
                constexpr int G = R23;
                for (int w = tid; w < G * W; w += NT) {
                    int g, c;
                    item(w, G, g, c);
                    const bool ok = c < nvalid;
                    V z[R1];
#pragma unroll
                    for (int m1 = 0; m1 < R1; ++m1)
                        z[m1] = ok ? src[base + (long long)(m1 * R23 + g) * rs + c * cs] : V{0, 0};
                    Dft<R1, 1>::run(z);
                    if constexpr (NSTEP == 1) {
                        if constexpr (KIND == KIND_DIF) {
                            if (ok) {
                                V t{1, 0}, s{1, 0};
                                if (a.ext) ext_pair(c, 0, 1, t, s);
#pragma unroll
                                for (int k1 = 0; k1 < R1; ++k1) {
                                    const V y = a.ext ? cmul(z[k1], t) : z[k1];
                                    dst[base + (long long)revd<RADIX, R1>(k1) * rs + c * cs] = y;
                                    if (a.ext) t = cmul(t, s);
                                }
                            }
                        } else {  // CONV with a single codelet: x ghat, inverse, store
                            if (ok) {
                                const long long gofs = ((first + c) % (a.N / R)) * (long long)R;
#pragma unroll
                                for (int k1 = 0; k1 < R1; ++k1)
                                    z[k1] = cmul(z[k1], __ldg(a.ghat + gofs + revd<RADIX, R1>(k1)));
                                Dft<R1, -1>::run(z);
#pragma unroll
                                for (int m1 = 0; m1 < R1; ++m1) dst[base + (long long)m1 * rs + c * cs] = z[m1];
                            }
                        }
                    } else {
#pragma unroll
                        for (int k1 = 1; k1 < R1; ++k1) z[k1] = cmul(z[k1], __ldg(a.tw1 + k1 * R23 + g));
#pragma unroll
                        for (int k1 = 0; k1 < R1; ++k1) sm[sidx(k1 * R23 + g, c)] = z[k1];
                    }
                }
            }
            if constexpr (NSTEP >= 2) {
                __syncthreads();
                // -------------------------------------------- DIF step 2
                constexpr int G = R1 * R3;
                for (int w = tid; w < G * W; w += NT) {
                    int g, c;
                    item(w, G, g, c);
                    const int k1 = g / R3, m3 = g - (g / R3) * R3;
                    V z[R2];
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) z[m2] = sm[sidx(k1 * R23 + m2 * R3 + m3, c)];
                    Dft<R2, 1>::run(z);
                    if constexpr (NSTEP == 2) {
                        const bool ok = c < nvalid;
                        const int pfix = revd<RADIX, R1>(k1) * R23;
                        if constexpr (KIND == KIND_DIF) {
                            if (ok) {
                                V t{1, 0}, s{1, 0};
                                if (a.ext) ext_pair(c, k1, R1, t, s);
#pragma unroll
                                for (int k2 = 0; k2 < R2; ++k2) {
                                    const V y = a.ext ? cmul(z[k2], t) : z[k2];
                                    dst[base + (long long)(pfix + revd<RADIX, R2>(k2)) * rs + c * cs] = y;
                                    if (a.ext) t = cmul(t, s);
                                }
                            }
                        } else {  // CONV: x ghat, DIT-conj step B, back to smem
                            const long long gofs = ok ? ((first + c) % (a.N / R)) * (long long)R : 0;
#pragma unroll
                            for (int k2 = 0; k2 < R2; ++k2)
                                z[k2] = cmul(z[k2], __ldg(a.ghat + gofs + pfix + revd<RADIX, R2>(k2)));
                            Dft<R2, -1>::run(z);
#pragma unroll
                            for (int m2 = 1; m2 < R2; ++m2) z[m2] = cmulc(z[m2], __ldg(a.tw1 + k1 * R23 + m2));
#pragma unroll
                            for (int m2 = 0; m2 < R2; ++m2) sm[sidx(k1 * R23 + m2, c)] = z[m2];
                        }
                    } else {
#pragma unroll
                        for (int k2 = 1; k2 < R2; ++k2) z[k2] = cmul(z[k2], __ldg(a.tw2 + k2 * R3 + m3));
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2) sm[sidx(k1 * R23 + k2 * R3 + m3, c)] = z[k2];
                    }
                }
            }
            if constexpr (NSTEP == 3) {
                __syncthreads();
                // -------------------------------------------- DIF step 3
                constexpr int G = R1 * R2;
                for (int w = tid; w < G * W; w += NT) {
                    int g, c;
                    item(w, G, g, c);
                    const int k1 = g / R2, k2 = g - (g / R2) * R2;
                    const bool ok = c < nvalid;
                    V z[R3];
#pragma unroll
                    for (int m3 = 0; m3 < R3; ++m3) z[m3] = sm[sidx(k1 * R23 + k2 * R3 + m3, c)];
                    Dft<R3, 1>::run(z);
                    const int pfix = revd<RADIX, R1>(k1) * R23 + revd<RADIX, R2>(k2) * R3;
                    if constexpr (KIND == KIND_DIF) {
                        if (ok) {
                            V t{1, 0}, s{1, 0};
                            if (a.ext) ext_pair(c, k1 + R1 * k2, R1 * R2, t, s);
#pragma unroll
                            for (int k3 = 0; k3 < R3; ++k3) {
                                const V y = a.ext ? cmul(z[k3], t) : z[k3];
                                dst[base + (long long)(pfix + revd<RADIX, R3>(k3)) * rs + c * cs] = y;
                                if (a.ext) t = cmul(t, s);
                            }
                        }
                    } else {  // CONV: x ghat, DIT-conj step A
                        const long long gofs = ok ? ((first + c) % (a.N / R)) * (long long)R : 0;
#pragma unroll
                        for (int k3 = 0; k3 < R3; ++k3)
                            z[k3] = cmul(z[k3], __ldg(a.ghat + gofs + pfix + revd<RADIX, R3>(k3)));
                        Dft<R3, -1>::run(z);
                        if (k2 != 0) {
#pragma unroll
                            for (int m3 = 1; m3 < R3; ++m3) z[m3] = cmulc(z[m3], __ldg(a.tw2 + k2 * R3 + m3));
                        }
#pragma unroll
                        for (int m3 = 0; m3 < R3; ++m3) sm[sidx(k1 * R23 + k2 * R3 + m3, c)] = z[m3];
                    }
                }
            }
        }

        if constexpr (KIND == KIND_DIT_FWD || KIND == KIND_DIT_CONJ || KIND == KIND_CONV) {
            constexpr int S = (KIND == KIND_DIT_FWD) ? 1 : -1;
            constexpr bool FROM_GLOBAL = KIND != KIND_CONV;
            auto tw = [&](V x, V w) -> V { return S > 0 ? cmul(x, w) : cmulc(x, w); };
            // ---------------------------------------- DIT step A (R3 > 1)
            if constexpr (NSTEP == 3 && FROM_GLOBAL) {
                constexpr int G = R1 * R2;
                for (int w = tid; w < G * W; w += NT) {
                    int g, c;
                    item(w, G, g, c);
                    const int k1 = g / R2, k2 = g - (g / R2) * R2;
                    const bool ok = c < nvalid;
                    const int pfix = revd<RADIX, R1>(k1) * R23 + revd<RADIX, R2>(k2) * R3;
                    V z[R3];
#pragma unroll
                    for (int k3 = 0; k3 < R3; ++k3)
                        z[k3] = ok ? src[base + (long long)(pfix + revd<RADIX, R3>(k3)) * rs + c * cs] : V{0, 0};
                    if (a.ext && ok) {
                        V t, s;
                        ext_pair(c, k1 + R1 * k2, R1 * R2, t, s);
#pragma unroll
                        for (int k3 = 0; k3 < R3; ++k3) {
                            z[k3] = tw(z[k3], t);
                            t = cmul(t, s);
                        }
                    }
                    Dft<R3, S>::run(z);
                    if (k2 != 0) {
#pragma unroll
                        for (int m3 = 1; m3 < R3; ++m3) z[m3] = tw(z[m3], __ldg(a.tw2 + k2 * R3 + m3));
                    }
#pragma unroll
                    for (int m3 = 0; m3 < R3; ++m3) sm[sidx(k1 * R23 + k2 * R3 + m3, c)] = z[m3];
                }
            }
            // ---------------------------------------- DIT step B (R2 > 1)
            if constexpr (NSTEP >= 2 && !(KIND == KIND_CONV && NSTEP == 2)) {
                if constexpr (NSTEP == 3) __syncthreads();
                constexpr int G = R1 * R3;
                for (int w = tid; w < G * W; w += NT) {
                    int g, c;
                    item(w, G, g, c);
                    const int k1 = g / R3, m3 = g - (g / R3) * R3;
                    V z[R2];
                    if constexpr (NSTEP == 2 && FROM_GLOBAL) {
                        const bool ok = c < nvalid;
                        const int pfix = revd<RADIX, R1>(k1) * R23;
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2)
                            z[k2] = ok ? src[base + (long long)(pfix + revd<RADIX, R2>(k2)) * rs + c * cs] : V{0, 0};
                        if (a.ext && ok) {
                            V t, s;
                            ext_pair(c, k1, R1, t, s);
#pragma unroll
                            for (int k2 = 0; k2 < R2; ++k2) {
                                z[k2] = tw(z[k2], t);
                                t = cmul(t, s);
                            }
                        }
                    } else {
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2) z[k2] = sm[sidx(k1 * R23 + k2 * R3 + m3, c)];
                    }
                    Dft<R2, S>::run(z);
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) {
                        const int m23 = m2 * R3 + m3;
                        if (m23 != 0) z[m2] = tw(z[m2], __ldg(a.tw1 + k1 * R23 + m23));
                    }
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) sm[sidx(k1 * R23 + m2 * R3 + m3, c)] = z[m2];
                }
            }
            // ---------------------------------------- DIT step C (always)
            if constexpr (!(KIND == KIND_CONV && NSTEP == 1)) {
                if constexpr (NSTEP >= 2) __syncthreads();
                constexpr int G = R23;
                for (int w = tid; w < G * W; w += NT) {
                    int g, c;
                    item(w, G, g, c);
                    const bool ok = c < nvalid;
                    V z[R1];
                    if constexpr (NSTEP == 1) {
                        // single codelet straight from global (DIT kinds only)
#pragma unroll
                        for (int k1 = 0; k1 < R1; ++k1)
                            z[k1] = ok ? src[base + (long long)revd<RADIX, R1>(k1) * rs + c * cs] : V{0, 0};
                        if (a.ext && ok) {
                            V t, s;
                            ext_pair(c, 0, 1, t, s);
#pragma unroll
                            for (int k1 = 0; k1 < R1; ++k1) {
                                z[k1] = tw(z[k1], t);
                                t = cmul(t, s);
                            }
                        }
                    } else {
#pragma unroll
                        for (int k1 = 0; k1 < R1; ++k1) z[k1] = sm[sidx(k1 * R23 + g, c)];
                    }
                    Dft<R1, S>::run(z);
                    if (ok) {
#pragma unroll
                        for (int m1 = 0; m1 < R1; ++m1) {
                            const long long e = base + (long long)(m1 * R23 + g) * rs + c * cs;
                            V y = z[m1];
                            if (a.mul) y = cmul(y, __ldg(a.mul + (e % a.N)));
                            if (a.has_scale) y = V{y.x * a.scale, y.y * a.scale};
                            dst[e] = y;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace pafft_b200
