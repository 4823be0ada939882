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

#include <cuda.h>

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
    // STRIDED staging through a 2-D tensor map (boxes of rb rows), else one
    // bulk copy per row
    int use_tmap;
    int rb;
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
    static constexpr int SMEM_BUDGET = 110 * 1024;  // per tile buffer (two are resident)
    // STRIDED: 8 (fp64) / 16 (fp32) columns = one 128-byte row segment; more
    // columns for single-codelet passes (no shared memory, tiny groups).
    static constexpr int MAXW = MAP == MAP_STRIDED ? (S::NSTEP == 1 ? 64 : (ESZ == 16 ? 8 : 16)) : 64;
    // fp32 strided rows may start 8 bytes off a 16-byte boundary (odd C):
    // each shared row then holds W + 2 slots and the data sits at a per-row
    // shift of 0 or 1 element (see stage_tile).
    static constexpr bool SHIFT = MAP == MAP_STRIDED && ESZ == 8;
    static constexpr int rowslots(int w) { return SHIFT ? w + 2 : w; }
    static constexpr int wcalc() {
        int w = MAXW;
        while (w > 1 && S::GMIN * w > 512) --w;
        if (MAP == MAP_CONTIG)
            while (w > 1 && S::GMIN * w > 256) --w;
        while (w > 1 && S::R * rowslots(w) * ESZ > SMEM_BUDGET) --w;
        // at least one full warp: warp 0 issues the bulk copies
        while (S::GMIN * w < 32 && S::R * rowslots(w + 1) * ESZ <= SMEM_BUDGET) ++w;
        if (SHIFT && (w & 1)) ++w;  // even W keeps rows 16-byte sized
        // fp32 contiguous tiles start at first*R elements: even W keeps every
        // tile start 16-byte aligned for the bulk copy
        if (MAP == MAP_CONTIG && ESZ == 8 && (w & 1)) w = (w > 1 && S::R * (w + 1) * ESZ > SMEM_BUDGET) ? w - 1 : w + 1;
        return w;
    }
    static constexpr int W = wcalc();
    static constexpr int SW = rowslots(W);  // shared row stride (STRIDED)
    static constexpr int NT = S::GMIN * W;
    static_assert(NT >= 32, "tile policy needs a full warp");
    // two tile buffers (TMA double buffering) + two mbarriers
    static constexpr int BUF = ((MAP == MAP_STRIDED ? S::R * SW : S::R * W) * ESZ + 15) / 16 * 16;
    static constexpr int SMEM = 2 * BUF + 16;
};

template <typename T>
__device__ __forceinline__ cplx<T> ext_root(const PassArgs<T>& a, unsigned long long e) {
    const cplx<T> lo = __ldg(a.ext_lo + (e & ((1ull << a.ext_bits) - 1)));
    const cplx<T> hi = __ldg(a.ext_hi + (e >> a.ext_bits));
    return cmul(lo, hi);
}

// ---------------------------------------------------------------- TMA/mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    unsigned ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!ok);
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_load_1d(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Tile geometry: element (row j, tile column c) lives at
// src + base + j*rs + c*cs; STRIDED: cs = 1, rs = C; CONTIG: cs = R, rs = 1.
struct TileGeo {
    long long base;   // element offset of (row 0, column 0)
    long long first;  // first column (STRIDED) or first panel (CONTIG)
    int nvalid;
};

template <int R, int W, bool STRIDED, typename T>
__device__ __forceinline__ TileGeo tile_geo(const PassArgs<T>& a, long long tile) {
    TileGeo g;
    if (!STRIDED) {
        g.first = tile * W;
        const long long left = a.panels - g.first;
        g.nvalid = left < W ? (int)left : W;
        g.base = g.first * (long long)R;
    } else {
        const long long p = tile / a.tiles_per_panel;
        g.first = (tile - p * a.tiles_per_panel) * (long long)W;
        const long long left = a.C - g.first;
        g.nvalid = left < W ? (int)left : W;
        g.base = p * a.panel_elems + g.first;
    }
    return g;
}

// Issue the bulk copies that stage one tile into `buf` (called by warp 0).
// STRIDED: one copy per row (rows land at buf[j*SW + shift_j]); CONTIG: the
// tile is one contiguous run of nvalid*R elements.  Bulk copies need 16-byte
// aligned addresses and sizes: fp64 always satisfies this; fp32 rows copy the
// enclosing 16-byte-aligned window (shift_j = 1 when the row starts 8 bytes
// into it), and an odd fp32 contiguous tail element is moved by one thread.
__device__ __forceinline__ void tma_load_2d(void* sdst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(sdst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

template <int R, int W, int SW, bool STRIDED, typename T>
__device__ __forceinline__ void stage_tile(const PassArgs<T>& a, const CUtensorMap* map, long long tile,
                                           cplx<T>* buf, unsigned long long* bar, int lane) {
    using V = cplx<T>;
    const TileGeo g = tile_geo<R, W, STRIDED>(a, tile);
    if (STRIDED && a.use_tmap) {
        // boxes of rb rows x SW columns (out-of-range columns zero-filled);
        // the tile lands densely as [row][SW]
        if (lane == 0) {
            const long long p = tile / a.tiles_per_panel;
            const int nb = R / a.rb;
            mbar_expect_tx(bar, (unsigned)(R * SW * sizeof(V)));
            for (int i = 0; i < nb; ++i)
                tma_load_2d(buf + i * a.rb * SW, map, (int)(2 * g.first), (int)(p * R + i * a.rb), bar);
        }
    } else if (STRIDED) {
        const V* src = a.src + g.base;
        if constexpr (sizeof(V) == 16) {
            const unsigned rb = (unsigned)(g.nvalid * sizeof(V));
            if (lane == 0) mbar_expect_tx(bar, rb * R);
            __syncwarp();
            for (int j = lane; j < R; j += 32) tma_load_1d(buf + j * SW, src + (long long)j * a.C, rb, bar);
        } else {
            // total bytes: sum over rows of round16(shift_j*8 + nvalid*8)
            const long long b0 = g.base & 1;
            const unsigned odd = (unsigned)(a.C & 1);
            const unsigned n8 = (unsigned)g.nvalid * 8u;
            const unsigned sz0 = (n8 + 15u) & ~15u;              // shift 0
            const unsigned sz1 = (n8 + 8u + 15u) & ~15u;         // shift 1
            const unsigned rows_shift1 = odd ? (unsigned)(b0 ? (R + 1) / 2 : R / 2) : (unsigned)(b0 ? R : 0);
            if (lane == 0) mbar_expect_tx(bar, rows_shift1 * sz1 + ((unsigned)R - rows_shift1) * sz0);
            __syncwarp();
            for (int j = lane; j < R; j += 32) {
                const unsigned sh = (unsigned)(b0 ^ (j & odd));
                const V* row = src + (long long)j * a.C - sh;
                tma_load_1d(buf + j * SW, row, sh ? sz1 : sz0, bar);
            }
        }
    } else if (lane == 0) {
        const long long n = (long long)g.nvalid * R;
        unsigned bytes = (unsigned)(n * sizeof(V));
        if constexpr (sizeof(V) == 8) {
            if (bytes & 15u) {  // odd element count: tail element by hand
                bytes -= 8u;
                buf[n - 1] = a.src[g.base + n - 1];
            }
        }
        mbar_expect_tx(bar, bytes);
        if (bytes) tma_load_1d(buf, a.src + g.base, bytes, bar);
    }
}

// Persistent pass kernel: each CTA walks tiles blockIdx.x + i * gridDim.x.
// Tile i+1 streams into the other shared buffer (TMA, mbarrier) while tile i
// is transformed in place in its buffer; results go straight from registers
// to global memory in their final order (rev-ordered rows for DIF).
template <typename T, int RADIX, int R1, int R2, int R3, int KIND, int MAP>
__global__ void __launch_bounds__(TilePolicy<T, R1, R2, R3, MAP>::NT, 1)
    pass_kernel(const PassArgs<T> a, const __grid_constant__ CUtensorMap tmap) {
    using V = cplx<T>;
    using Sh = Shape<R1, R2, R3>;
    using Pol = TilePolicy<T, R1, R2, R3, MAP>;
    constexpr int R = Sh::R, R23 = Sh::R23, NSTEP = Sh::NSTEP, GMIN = Sh::GMIN;
    constexpr int W = Pol::W;
    constexpr int SW = Pol::SW;
    constexpr int BUFE = Pol::BUF / (int)sizeof(V);  // elements per tile buffer
    constexpr bool STRIDED = MAP == MAP_STRIDED;
    constexpr bool SHIFT = Pol::SHIFT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V* const bufs = reinterpret_cast<V*>(smem_raw);
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(smem_raw + 2 * Pol::BUF);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    // thread -> (tile column c, group slot gt); STRIDED: c fastest (coalesced
    // W-wide row segments, conflict-free smem rows); CONTIG: group fastest.
    const int c = STRIDED ? t % W : t / GMIN;
    const int gt = STRIDED ? t / W : t % GMIN;
    constexpr int SS = STRIDED ? SW : 1;  // shared stride between consecutive rows
    const long long rs = STRIDED ? (long long)a.C : 1;  // global row stride

    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = blockIdx.x, ts = gridDim.x;
    if (warp == 0) {
        if (t0 < a.tiles) stage_tile<R, W, SW, STRIDED>(a, &tmap, t0, bufs, &bars[0], lane);
        if (t0 + ts < a.tiles) stage_tile<R, W, SW, STRIDED>(a, &tmap, t0 + ts, bufs + BUFE, &bars[1], lane);
    }
    __syncthreads();  // hand-copied fp32 tail elements of the first tiles

    int it = 0;
    for (long long tile = t0; tile < a.tiles; tile += ts, ++it) {
        const int b = it & 1;
        V* const buf = bufs + b * BUFE;
        const TileGeo geo = tile_geo<R, W, STRIDED>(a, tile);
        const long long first = geo.first;
        const bool ok = c < geo.nvalid;
        V* const scol = STRIDED ? buf + c : buf + c * R;
        // shared element of tile row `row` for this thread's column
        const int codd = SHIFT && !a.use_tmap ? (a.C & 1) : 0;
        const int b0 = SHIFT && !a.use_tmap ? (int)(geo.base & 1) : 0;
        auto sref = [&](int row) -> V& { return scol[row * SS + (SHIFT ? ((row & codd) ^ b0) : 0)]; };
        V* __restrict__ gdst = a.dst + geo.base + (STRIDED ? c : (long long)c * R);
        auto ext_pair = [&](int kf, int S, V& tw, V& st) {
            const unsigned long long jj = (unsigned long long)(first + c) / a.sq;
            tw = ext_root(a, jj * (unsigned long long)kf);
            st = ext_root(a, jj * (unsigned long long)S);
        };
        mbar_wait(&bars[b], (it >> 1) & 1);

        if constexpr (KIND == KIND_DIF || KIND == KIND_CONV) {
            // ------------------------------------------------ DIF step 1
#pragma unroll
            for (int j = 0; j < Sh::G1 / GMIN; ++j) {
                const int g = gt + j * GMIN;  // m23
                V z[R1];
#pragma unroll
                for (int m1 = 0; m1 < R1; ++m1) z[m1] = sref(m1 * R23 + g);
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
                    for (int k1 = 0; k1 < R1; ++k1) sref(k1 * R23 + g) = z[k1];
                }
            }
            if constexpr (NSTEP >= 2) {
                __syncthreads();
                // -------------------------------------------- DIF step 2
#pragma unroll
                for (int j = 0; j < Sh::G2 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R3, m3 = g - (g / R3) * R3;
                    const int sb = k1 * R23 + m3;
                    V z[R2];
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) z[m2] = sref(sb + m2 * R3);
                    dft<R2, 1>(z);
                    if constexpr (NSTEP == 2) {
                        const int pfix = revd<RADIX, R1>(k1) * R23;
                        if constexpr (KIND == KIND_DIF) {
                            if (ok) {
                                V tw{1, 0}, st{1, 0};
                                if (a.ext) ext_pair(k1, R1, tw, st);
                                V* gp = gdst + (long long)pfix * rs;
#pragma unroll
                                for (int k2 = 0; k2 < R2; ++k2) {
                                    gp[(long long)revd<RADIX, R2>(k2) * rs] = a.ext ? cmul(z[k2], tw) : z[k2];
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
                            for (int m2 = 0; m2 < R2; ++m2) sref(sb + m2) = z[m2];
                        }
                    } else {
                        const V* tw2 = a.tw2 + m3;
#pragma unroll
                        for (int k2 = 1; k2 < R2; ++k2) z[k2] = cmul(z[k2], __ldg(tw2 + k2 * R3));
#pragma unroll
                        for (int k2 = 0; k2 < R2; ++k2) sref(sb + k2 * R3) = z[k2];
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
                    const int sb = k1 * R23 + k2 * R3;
                    V z[R3];
#pragma unroll
                    for (int m3 = 0; m3 < R3; ++m3) z[m3] = sref(sb + m3);
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
                        for (int m3 = 0; m3 < R3; ++m3) sref(sb + m3) = z[m3];
                    }
                }
            }
        }

        if constexpr (KIND == KIND_DIT_FWD || KIND == KIND_DIT_CONJ || KIND == KIND_CONV) {
            constexpr int S = (KIND == KIND_DIT_FWD) ? 1 : -1;
            constexpr bool FIRST = KIND != KIND_CONV;  // DIT kinds start from the staged input
            auto tw = [](V x, V w) -> V { return S > 0 ? cmul(x, w) : cmulc(x, w); };
            // ---------------------------------------- DIT step A (R3 > 1)
            if constexpr (NSTEP == 3 && FIRST) {
#pragma unroll
                for (int j = 0; j < Sh::G3 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R2, k2 = g - (g / R2) * R2;
                    const int pfix = revd<RADIX, R1>(k1) * R23 + revd<RADIX, R2>(k2) * R3;
                    V z[R3];
#pragma unroll
                    for (int k3 = 0; k3 < R3; ++k3) z[k3] = sref(pfix + revd<RADIX, R3>(k3));
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
                    // in place: the rows pfix + rev(k3) just read are rows pfix + m3
#pragma unroll
                    for (int m3 = 0; m3 < R3; ++m3) sref(pfix + m3) = z[m3];
                }
            }
            // ---------------------------------------- DIT step B (R2 > 1)
            // Slot convention: DIT kinds keep the staged (digit-reversed) row
            // order, so group k1 lives at rev(k1)*R23 and index k2 at rev(k2)*R3;
            // CONV continues from the DIF's natural frequency slots.  Every step
            // then reads and writes the same slot set (in place).
            if constexpr (NSTEP >= 2 && !(KIND == KIND_CONV && NSTEP == 2)) {
                if constexpr (NSTEP == 3) __syncthreads();
#pragma unroll
                for (int j = 0; j < Sh::G2 / GMIN; ++j) {
                    const int g = gt + j * GMIN;
                    const int k1 = g / R3, m3 = g - (g / R3) * R3;
                    const int sk1 = FIRST ? revd<RADIX, R1>(k1) : k1;
                    const int sb = sk1 * R23 + m3;
                    V z[R2];
#pragma unroll
                    for (int k2 = 0; k2 < R2; ++k2) z[k2] = sref(sb + (FIRST ? revd<RADIX, R2>(k2) : k2) * R3);
                    if constexpr (NSTEP == 2 && FIRST) {
                        if (a.ext && ok) {
                            V w, st;
                            ext_pair(k1, R1, w, st);
#pragma unroll
                            for (int k2 = 0; k2 < R2; ++k2) {
                                z[k2] = tw(z[k2], w);
                                w = cmul(w, st);
                            }
                        }
                    }
                    dft<R2, S>(z);
                    const V* tw1 = a.tw1 + k1 * R23 + m3;
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2)
                        if (m2 * R3 != 0 || m3 != 0) z[m2] = tw(z[m2], __ldg(tw1 + m2 * R3));
#pragma unroll
                    for (int m2 = 0; m2 < R2; ++m2) sref(sb + m2 * R3) = z[m2];
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
                        for (int k1 = 0; k1 < R1; ++k1) z[k1] = sref(revd<RADIX, R1>(k1));
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
                        for (int k1 = 0; k1 < R1; ++k1)
                            z[k1] = sref((FIRST ? revd<RADIX, R1>(k1) : k1) * R23 + g);
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
        // all reads of this buffer are done: refill it with tile it + 2
        __syncthreads();
        if (warp == 0 && tile + 2 * ts < a.tiles) {
            fence_proxy_async();
            stage_tile<R, W, SW, STRIDED>(a, &tmap, tile + 2 * ts, buf, &bars[b], lane);
        }
    }
}

}  // namespace pafft_b200
