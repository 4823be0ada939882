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
// steps (four-step decomposition; internal twiddles w_R, w_{R2 R3} from
// L1-resident tables laid out for the access pattern; the external twiddle
// w_K0^{jj k} by a per-thread recurrence from a two-level table).  Each codelet
// size is a power of r, so rev(k) splits per step.
//
// Tile geometry is compile-time: W columns (STRIDED map: W adjacent columns
// of one panel, so every row segment is a W*16-byte coalesced run and each
// shared-memory row is conflict-free) or W panels (CONTIG map: C == 1, W
// consecutive contiguous blocks).  Every thread owns one (column, group-slot)
// pair; step i handles G_i / GMIN groups per thread at compile-time offsets,
// so all shared/global index arithmetic folds to per-thread bases plus
// immediates.  Layout is interleaved complex (double2 / float2).
#pragma once

#include "codelets.cuh"

namespace pafft_b200 {

enum PassKind : int { KIND_DIF = 0, KIND_DIT_FWD = 1, KIND_DIT_CONJ = 2, KIND_CONV = 3 };
enum PassMap : int { MAP_STRIDED = 0, MAP_CONTIG = 1 };

template <typename T> struct PassArgs {
    const cplx<T>* src;
    cplx<T>* dst;
    long long tiles;
    long long panels;        // total panels over the batch
    long long panel_elems;   // R * C
    int C;                   // columns per panel (contiguous)
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
template <int RADIX, int P> __host__ __device__ constexpr int revd(int k) {
    int o = 0;
    for (int p = 1; p < P; p *= RADIX) {
        o = o * RADIX + k % RADIX;
        k /= RADIX;
    }
    return o;
}

template <int R1, int R2, int R3> struct Shape {
    static constexpr int R = R1 * R2 * R3;
    static constexpr int R23 = R2 * R3;
    static constexpr int NSTEP = 1 + (R2 > 1 ? 1 : 0) + (R3 > 1 ? 1 : 0);
    static constexpr int G1 = R23;       // step 1 groups: m23
    static constexpr int G2 = R1 * R3;   // step 2 groups: (k1, m3)
    static constexpr int G3 = R1 * R2;   // step 3 groups: (k1, k2)
    static constexpr int gmin() {
        int g = G1;
        if (NSTEP >= 2 && G2 < g) g = G2;
        if (NSTEP == 3 && G3 < g) g = G3;
        return g;
    }
    static constexpr int GMIN = gmin();
};

// Compile-time tile policy shared by kernels and host plan (registry).
template <typename T, int R1, int R2, int R3, int MAP> struct TilePolicy {
    using S = Shape<R1, R2, R3>;
    static constexpr int ESZ = (int)sizeof(cplx<T>);
    static constexpr int SMEM_BUDGET = 112 * 1024;
    // STRIDED: 8 (fp64) / 16 (fp32) columns = one 128-byte row segment; more
    // columns for single-codelet passes (no shared memory, tiny groups).
    static constexpr int MAXW = MAP == MAP_STRIDED ? (S::NSTEP == 1 ? 64 : (ESZ == 16 ? 8 : 16)) : 64;
    static constexpr int wcalc() {
        int w = MAXW;
        while (w > 1 && S::GMIN * w > 512) --w;
        if (MAP == MAP_CONTIG)
            while (w > 1 && S::GMIN * w > 256) --w;
        if (S::NSTEP > 1)
            while (w > 1 && S::R * w * ESZ > SMEM_BUDGET) --w;
        return w;
    }
    static constexpr int W = wcalc();
    static constexpr int NT = S::GMIN * W;
    static constexpr int SMEM = S::NSTEP > 1 ? S::R * W * ESZ : 0;
};

template <typename T>
__device__ __forceinline__ cplx<T> ext_root(const PassArgs<T>& a, unsigned long long e) {
    const cplx<T> lo = __ldg(a.ext_lo + (e & ((1ull << a.ext_bits) - 1)));
    const cplx<T> hi = __ldg(a.ext_hi + (e >> a.ext_bits));
    return cmul(lo, hi);
}

template <typename T, int RADIX, int R1, int R2, int R3, int KIND, int MAP>
__global__ void __launch_bounds__(TilePolicy<T, R1, R2, R3, MAP>::NT)
    pass_kernel(const PassArgs<T> a) {
    using V = cplx<T>;
    using Sh = Shape<R1, R2, R3>;
    using Pol = TilePolicy<T, R1, R2, R3, MAP>;
    constexpr int R = Sh::R, R23 = Sh::R23, NSTEP = Sh::NSTEP, GMIN = Sh::GMIN;
    constexpr int W = Pol::W;
    constexpr bool STRIDED = MAP == MAP_STRIDED;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* const sm = reinterpret_cast<V*>(smem_raw);

    const int t = threadIdx.x;
    // thread -> (tile column c, group slot gt); STRIDED: c fastest (coalesced
    // W-wide row segments, conflict-free smem rows); CONTIG: group fastest.
    const int c = STRIDED ? t % W : t / GMIN;
    const int gt = STRIDED ? t / W : t % GMIN;
    // shared element (j, c): STRIDED sm[j*W + c], CONTIG sm[c*R + j]
    V* const scol = STRIDED ? sm + c : sm + c * R;
    constexpr int SS = STRIDED ? W : 1;  // shared stride between consecutive j

    for (long long tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        long long base, first;
        int nvalid;
        if (!STRIDED) {
            first = tile * W;
            const long long left = a.panels - first;
            nvalid = left < W ? (int)left : W;
            base = first * (long long)R + (long long)c * R;
        } else {
            const long long p = tile / a.tiles_per_panel;
            first = (tile - p * a.tiles_per_panel) * (long long)W;
            const long long left = a.C - first;
            nvalid = left < W ? (int)left : W;
            base = p * a.panel_elems + first + c;
        }
        const bool ok = c < nvalid;
        const long long rs = STRIDED ? (long long)a.C : 1;  // global row stride
        const V* __restrict__ gsrc = a.src + base;
        V* __restrict__ gdst = a.dst + base;
        // external twiddle base/step for this column: w_K0^{jj kf}, w_K0^{jj S}
        auto ext_pair = [&](int kf, int S, V& tw, V& st) {
            const unsigned long long jj = (unsigned long long)(first + c) / a.sq;
            tw = ext_root(a, jj * (unsigned long long)kf);
            st = ext_root(a, jj * (unsigned long long)S);
        };

        if constexpr (KIND == KIND_DIF || KIND == KIND_CONV) {
            // ------------------------------------------------ DIF step 1
#pragma unroll
            for (int j = 0; j < Sh::G1 / GMIN; ++j) {
                const int g = gt + j * GMIN;  // m23
                V z[R1];
#pragma unroll
                for (int m1 = 0; m1 < R1; ++m1)
                    z[m1] = ok ? gsrc[(long long)(m1 * R23 + g) * rs] : V{0, 0};
                dft<R1, 1>(z);
                if constexpr (NSTEP == 1) {
                    if constexpr (KIND == KIND_DIF) {
                        if (ok) {
                            V tw{1, 0}, st{1, 0};
                            if (a.ext) ext_pair(0, 1, tw, st);
#pragma unroll
                            for (int k1 = 0; k1 < R1; ++k1) {
                                gdst[(long long)revd<RADIX, R1>(k1) * rs] = a.ext ? cmul(z[k1], tw) : z[k1];
                                if (a.ext) tw = cmul(tw, st);
                            }
                        }
                    } else {  // CONV with a single codelet: x ghat, inverse, store
                        if (ok) {
                            const V* gh = a.ghat + ((first + c) % (a.N / R)) * (long long)R;
#pragma unroll
                            for (int k1 = 0; k1 < R1; ++k1) z[k1] = cmul(z[k1], __ldg(gh + revd<RADIX, R1>(k1)));
                            dft<R1, -1>(z);
#pragma unroll
                            for (int m1 = 0; m1 < R1; ++m1) gdst[(long long)m1 * rs] = z[m1];
                        }
                    }
                } else {
                    const V* tw1 = a.tw1 + g;
#pragma unroll
                    for (int k1 = 1; k1 < R1; ++k1) z[k1] = cmul(z[k1], __ldg(tw1 + k1 * R23));
#pragma unroll
                    for (int k1 = 0; k1 < R1; ++k1) scol[(k1 * R23 + g) * SS] = z[k1];
                }
            }
            if constexpr (NSTEP >= 2) {
                __syncthreads();
                // -------------------------------------------- DIF step 2
#pragma unroll
                for (int j = 0; j < Sh::G2 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R3, m3 = g - (g / R3) * R3;
                    V* sp = scol + (k1 * R23 + m3) * SS;
                    V z[R2];
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) z[m2] = sp[m2 * R3 * SS];
                    dft<R2, 1>(z);
                    if constexpr (NSTEP == 2) {
                        const int pfix = revd<RADIX, R1>(k1) * R23;
                        if constexpr (KIND == KIND_DIF) {
                            if (ok) {
                                V tw{1, 0}, st{1, 0};
                                if (a.ext) ext_pair(k1, R1, tw, st);
#pragma unroll
                                for (int k2 = 0; k2 < R2; ++k2) {
                                    gdst[(long long)(pfix + revd<RADIX, R2>(k2)) * rs] = a.ext ? cmul(z[k2], tw) : z[k2];
                                    if (a.ext) tw = cmul(tw, st);
                                }
                            }
                        } else {  // CONV: x ghat, DIT-conj step B (in registers), back to smem
                            if (ok) {
                                const V* gh = a.ghat + ((first + c) % (a.N / R)) * (long long)R + pfix;
#pragma unroll
                                for (int k2 = 0; k2 < R2; ++k2) z[k2] = cmul(z[k2], __ldg(gh + revd<RADIX, R2>(k2)));
                            }
                            dft<R2, -1>(z);
                            const V* tw1 = a.tw1 + k1 * R23;
#pragma unroll
                            for (int m2 = 1; m2 < R2; ++m2) z[m2] = cmulc(z[m2], __ldg(tw1 + m2));
#pragma unroll
                            for (int m2 = 0; m2 < R2; ++m2) sp[m2 * SS] = z[m2];
                        }
                    } else {
                        const V* tw2 = a.tw2 + m3;
#pragma unroll
                        for (int k2 = 1; k2 < R2; ++k2) z[k2] = cmul(z[k2], __ldg(tw2 + k2 * R3));
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2) sp[k2 * R3 * SS] = z[k2];
                    }
                }
            }
            if constexpr (NSTEP == 3) {
                __syncthreads();
                // -------------------------------------------- DIF step 3
#pragma unroll
                for (int j = 0; j < Sh::G3 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R2, k2 = g - (g / R2) * R2;
                    V* sp = scol + (k1 * R23 + k2 * R3) * SS;
                    V z[R3];
#pragma unroll
                    for (int m3 = 0; m3 < R3; ++m3) z[m3] = sp[m3 * SS];
                    dft<R3, 1>(z);
                    const int pfix = revd<RADIX, R1>(k1) * R23 + revd<RADIX, R2>(k2) * R3;
                    if constexpr (KIND == KIND_DIF) {
                        if (ok) {
                            V tw{1, 0}, st{1, 0};
                            if (a.ext) ext_pair(k1 + R1 * k2, R1 * R2, tw, st);
                            V* gp = gdst + (long long)pfix * rs;
#pragma unroll
                            for (int k3 = 0; k3 < R3; ++k3) {
                                gp[(long long)revd<RADIX, R3>(k3) * rs] = a.ext ? cmul(z[k3], tw) : z[k3];
                                if (a.ext) tw = cmul(tw, st);
                            }
                        }
                    } else {  // CONV: x ghat, DIT-conj step A
                        if (ok) {
                            const V* gh = a.ghat + ((first + c) % (a.N / R)) * (long long)R + pfix;
#pragma unroll
                            for (int k3 = 0; k3 < R3; ++k3) z[k3] = cmul(z[k3], __ldg(gh + revd<RADIX, R3>(k3)));
                        }
                        dft<R3, -1>(z);
                        if (k2 != 0) {
                            const V* tw2 = a.tw2 + k2 * R3;
#pragma unroll
                            for (int m3 = 1; m3 < R3; ++m3) z[m3] = cmulc(z[m3], __ldg(tw2 + m3));
                        }
#pragma unroll
                        for (int m3 = 0; m3 < R3; ++m3) sp[m3 * SS] = z[m3];
                    }
                }
            }
        }

        if constexpr (KIND == KIND_DIT_FWD || KIND == KIND_DIT_CONJ || KIND == KIND_CONV) {
            constexpr int S = (KIND == KIND_DIT_FWD) ? 1 : -1;
            constexpr bool FROM_GLOBAL = KIND != KIND_CONV;
            auto tw = [](V x, V w) -> V { return S > 0 ? cmul(x, w) : cmulc(x, w); };
            // ---------------------------------------- DIT step A (R3 > 1)
            if constexpr (NSTEP == 3 && FROM_GLOBAL) {
#pragma unroll
                for (int j = 0; j < Sh::G3 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R2, k2 = g - (g / R2) * R2;
                    const int pfix = revd<RADIX, R1>(k1) * R23 + revd<RADIX, R2>(k2) * R3;
                    const V* gp = gsrc + (long long)pfix * rs;
                    V z[R3];
#pragma unroll
                    for (int k3 = 0; k3 < R3; ++k3) z[k3] = ok ? gp[(long long)revd<RADIX, R3>(k3) * rs] : V{0, 0};
                    if (a.ext && ok) {
                        V w, st;
                        ext_pair(k1 + R1 * k2, R1 * R2, w, st);
#pragma unroll
                        for (int k3 = 0; k3 < R3; ++k3) {
                            z[k3] = tw(z[k3], w);
                            w = cmul(w, st);
                        }
                    }
                    dft<R3, S>(z);
                    if (k2 != 0) {
                        const V* tw2 = a.tw2 + k2 * R3;
#pragma unroll
                        for (int m3 = 1; m3 < R3; ++m3) z[m3] = tw(z[m3], __ldg(tw2 + m3));
                    }
                    V* sp = scol + (k1 * R23 + k2 * R3) * SS;
#pragma unroll
                    for (int m3 = 0; m3 < R3; ++m3) sp[m3 * SS] = z[m3];
                }
            }
            // ---------------------------------------- DIT step B (R2 > 1)
            if constexpr (NSTEP >= 2 && !(KIND == KIND_CONV && NSTEP == 2)) {
                if constexpr (NSTEP == 3) __syncthreads();
#pragma unroll
                for (int j = 0; j < Sh::G2 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R3, m3 = g - (g / R3) * R3;
                    V* sp = scol + (k1 * R23 + m3) * SS;
                    V z[R2];
                    if constexpr (NSTEP == 2 && FROM_GLOBAL) {
                        const V* gp = gsrc + (long long)(revd<RADIX, R1>(k1) * R23) * rs;
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2) z[k2] = ok ? gp[(long long)revd<RADIX, R2>(k2) * rs] : V{0, 0};
                        if (a.ext && ok) {
                            V w, st;
                            ext_pair(k1, R1, w, st);
#pragma unroll
                            for (int k2 = 0; k2 < R2; ++k2) {
                                z[k2] = tw(z[k2], w);
                                w = cmul(w, st);
                            }
                        }
                    } else {
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2) z[k2] = sp[k2 * R3 * SS];
                    }
                    dft<R2, S>(z);
                    const V* tw1 = a.tw1 + k1 * R23 + m3;
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2)
                        if (m2 * R3 != 0 || m3 != 0) z[m2] = tw(z[m2], __ldg(tw1 + m2 * R3));
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) sp[m2 * R3 * SS] = z[m2];
                }
            }
            // ---------------------------------------- DIT step C (always)
            if constexpr (!(KIND == KIND_CONV && NSTEP == 1)) {
                if constexpr (NSTEP >= 2) __syncthreads();
#pragma unroll
                for (int j = 0; j < Sh::G1 / GMIN; ++j) {
                    const int g = gt + j * GMIN;  // m23
                    V z[R1];
                    if constexpr (NSTEP == 1) {
#pragma unroll
                        for (int k1 = 0; k1 < R1; ++k1)
                            z[k1] = ok ? gsrc[(long long)revd<RADIX, R1>(k1) * rs] : V{0, 0};
                        if (a.ext && ok) {
                            V w, st;
                            ext_pair(0, 1, w, st);
#pragma unroll
                            for (int k1 = 0; k1 < R1; ++k1) {
                                z[k1] = tw(z[k1], w);
                                w = cmul(w, st);
                            }
                        }
                    } else {
#pragma unroll
                        for (int k1 = 0; k1 < R1; ++k1) z[k1] = scol[(k1 * R23 + g) * SS];
                    }
                    dft<R1, S>(z);
                    if (ok) {
                        V* gp = gdst + (long long)g * rs;
#pragma unroll
                        for (int m1 = 0; m1 < R1; ++m1) {
                            V y = z[m1];
                            if (a.mul) {
                                const long long e = (gp - a.dst) + (long long)(m1 * R23) * rs;
                                y = cmul(y, __ldg(a.mul + (e % a.N)));
                            }
                            if (a.has_scale) y = V{y.x * a.scale, y.y * a.scale};
                            gp[(long long)(m1 * R23) * rs] = y;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace pafft_b200
