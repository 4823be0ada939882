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

// cap on resident CTAs per SM the register allocation is sized for
#ifndef PAFFT_MAX_MINB
#define PAFFT_MAX_MINB 4
#endif
// Contiguous tiles single-buffered: more resident CTAs per SM instead of
// double buffering inside one CTA.  0 = never, 1 = when double buffering
// leaves one CTA per SM (measured on B200: config 1's R=4096 CONV, 1 -> 2 CTAs,
// +5.6% conv/s; forcing it where two or more CTAs fit spills and loses 6-25%),
// 2 = always (experiments).
#ifndef PAFFT_SB
#define PAFFT_SB 1
#endif
// Tuning switches (defaults = measured best on B200; DESIGN.md §3 has the A/B
// numbers).  PAFFT_EXT_HOIST: DIT passes load the first step's external
// twiddles before waiting for the tile, for codelets of <= PAFFT_HOIST_FMAX
// points (config 1's 16-point DIT measured 0.5% faster without it).
// PAFFT_OK_CT: one-block double-buffered contiguous tiles skip the
// column-in-range test (always full).  PAFFT_GHAT_PF: L2 prefetch of the next
// CONV tile's filter blocks.
#ifndef PAFFT_EXT_HOIST
#define PAFFT_EXT_HOIST 1
#endif
#ifndef PAFFT_HOIST_FMAX
#define PAFFT_HOIST_FMAX 9
#endif
#ifndef PAFFT_OK_CT
#define PAFFT_OK_CT 1
#endif
#ifndef PAFFT_GHAT_PF
#define PAFFT_GHAT_PF 1
#endif
// profiling build: per-CTA retire times of every pass launch (PAFFT_PASS_TRACE=1
// at run time); off in the product build, where it would cost registers
#ifndef PAFFT_TRACE
#define PAFFT_TRACE 0
#endif
#ifndef PAFFT_SB_MAX_MINB
#define PAFFT_SB_MAX_MINB 8
#endif


// PAFFT_DEBUG builds (tools/debug_build.sh) check tile geometry and
// shared-memory indices on the device; release builds compile them out.
#ifdef PAFFT_DEBUG
#include <cassert>
#define PAFFT_DASSERT(c) assert(c)
#else
#define PAFFT_DASSERT(c) ((void)0)
#endif

namespace pafft_b200 {

enum PassKind : int { KIND_DIF = 0, KIND_DIT_FWD = 1, KIND_DIT_CONJ = 2, KIND_CONV = 3 };
enum PassMap : int { MAP_STRIDED = 0, MAP_CONTIG = 1 };

template <typename T> struct PassArgs {
    const cplx<T>* src;
    cplx<T>* dst;
    long long tiles;
    // CONTIG tiles are ordered block-major across the batch: tile t covers
    // signal t % nsig, blocks [(t / nsig) W, +W) of it, so concurrently running
    // CTAs share the filter block (reused from L2 across the batch)
    long long nsig;
    long long bps;           // blocks (panels) per signal
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
    // internal twiddles of step i (i < nsteps - 1): tw[i][k * Q_i + lo] =
    // w_{P_i}^{k lo}, P_i = R_i ... R_last, Q_i = P_i / R_i
    const cplx<T>* tw[3];
    // CONV filter (pre-scaled by 1/N, each R-block in the pass's slot order:
    // see pafft_b200.cu kernel_ghat) and signal period
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
    // CONTIG tiles of power-of-two radix: staged through a 128-byte-swizzled
    // tensor map (rows of 128 B; 16-byte chunk index XOR row index), which
    // removes the 8-way bank conflicts of power-of-two slot strides
    int swz;
    int swz_b1;   // box rows per row group
    // dynamic tile order: the CTA's first tile is blockIdx.x, later ones are
    // gridDim.x + atomicAdd(&ctr[0], 1); ctr[1] counts retired CTAs and the last
    // one zeroes both, so the pair is clean for the stream's next launch;
    // nullptr = the static order blockIdx.x + i * gridDim.x
    unsigned* ctr;
#if PAFFT_TRACE
    // profiling build (-DPAFFT_TRACE=1, tools/trace_build.sh): per CTA {start,
    // retire time, tiles done, time waiting for tile arrival} in globaltimer ns; nullptr = off
    unsigned long long* trace;
#endif
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

// The same at run time (power-of-radix P, small: unrolled).
template <int RADIX, int P> __device__ __forceinline__ int revd_rt_dev(int k) {
    int o = 0;
#pragma unroll
    for (int p = 1; p < P; p *= RADIX) {
        o = o * RADIX + k % RADIX;
        k /= RADIX;
    }
    return o;
}

// Codelet split R = F0 * F1 * F2 * F3 (trailing 1s unused).  Step i works on
// digit i of the row index m = sum_i m_i wt(i), wt(i) = F_{i+1} ... F_last:
// groups are all combinations of the other digits, G(i) = R / F_i of them.
template <int F0, int F1, int F2, int F3> struct Fac {
    static constexpr int NS = 1 + (F1 > 1) + (F2 > 1) + (F3 > 1);
    static constexpr int R = F0 * F1 * F2 * F3;
    static constexpr int f(int i) { return i == 0 ? F0 : i == 1 ? F1 : i == 2 ? F2 : F3; }
    // P(i) = F_i ... F_last;  wt(i) = Q(i) = P(i + 1)
    static constexpr int P(int i) { return i >= NS ? 1 : f(i) * P(i + 1); }
    static constexpr int Q(int i) { return P(i + 1); }
    static constexpr int G(int i) { return R / f(i); }
    // product F_0 ... F_{i-1} (weight of digit i in the frequency index)
    static constexpr int L(int i) { return i == 0 ? 1 : L(i - 1) * f(i - 1); }
    static constexpr int gmin() {
        int g = G(0);
        for (int i = 1; i < NS; ++i)
            if (G(i) < g) g = G(i);
        return g;
    }
    static constexpr int GMIN = gmin();
    static constexpr int FMAX = R / GMIN;
};

// Compile-time tile policy shared by kernels and host plan (registry).
template <typename T, typename FAC, int MAP, int WOVR = 0> struct TilePolicy {
    static constexpr int ESZ = (int)sizeof(cplx<T>);
    static constexpr int SMEM_BUDGET = 110 * 1024;  // per tile buffer (two are resident)
    // STRIDED: 8 (fp64) / 16 (fp32) columns = one 128-byte row segment; more
    // columns for single-codelet passes (no shared-memory exchange).
    static constexpr int MAXW = MAP == MAP_STRIDED ? (FAC::NS == 1 ? 64 : (ESZ == 16 ? 8 : 16)) : 64;
    // fp32 strided rows may start 8 bytes off a 16-byte boundary (odd C):
    // each shared row then holds W + 2 slots and the data sits at a per-row
    // shift of 0 or 1 element (see stage_tile).
    // (WOVR < 0: the dense fp32 strided instance for even row lengths -- rows are
    // 16-byte aligned, the tile comes and goes through tensor maps like an fp64
    // one, no spare slots, no per-row copies, no register stores)
    static constexpr bool SHIFT = MAP == MAP_STRIDED && ESZ == 8 && WOVR >= 0;
    static constexpr int rowslots(int w) { return SHIFT ? w + 2 : w; }
    static constexpr int wcalc() {
        if (MAP == MAP_STRIDED && FAC::NS > 1) {
            // powers of two up to one 128-byte row segment (measured on B200:
            // full 128-byte rows beat 64-byte rows with twice the residency)
            int w = MAXW;
            while (w > 1 && 2 * FAC::R * rowslots(w) * ESZ > 220 * 1024) w /= 2;
            while (w > 1 && FAC::GMIN * w > 1024) w /= 2;
            if (SHIFT && (w & 1)) ++w;
            return w;
        }
        int w = MAXW;
        while (w > 1 && FAC::GMIN * w > 512) --w;
        if (MAP == MAP_CONTIG) {
            while (w > 1 && FAC::GMIN * w > 256) --w;
            // ~36 KB tiles: three double-buffered CTAs per SM
            while (w > 1 && FAC::NS > 1 && FAC::R * w * ESZ > 36 * 1024) --w;
            // power-of-two blocks: power-of-two W, so tiles divide the batch and
            // stay 1 KB multiples (swizzled staging)
            if ((FAC::R & (FAC::R - 1)) == 0)
                while (w & (w - 1)) --w;
        }
        while (w > 1 && FAC::R * rowslots(w) * ESZ > SMEM_BUDGET) --w;
        // at least one full warp: warp 0 issues the bulk copies
        while (FAC::GMIN * w < 32 && FAC::R * rowslots(w + 1) * ESZ <= SMEM_BUDGET) ++w;
        if (SHIFT && (w & 1)) ++w;  // even W keeps rows 16-byte sized
        // fp32 contiguous tiles start at first*R elements: even W keeps every
        // tile start 16-byte aligned for the bulk copy
        if (MAP == MAP_CONTIG && ESZ == 8 && (w & 1))
            w = (w > 1 && FAC::R * (w + 1) * ESZ > SMEM_BUDGET) ? w - 1 : w + 1;
        return w;
    }
    static constexpr int W = WOVR > 0 ? WOVR : wcalc();
    static constexpr int SW = rowslots(W);  // shared row stride (STRIDED)
    static constexpr int NT = FAC::GMIN * W;
    static_assert(NT >= 32, "tile policy needs a full warp");
    // two tile buffers (TMA double buffering) + two mbarriers
    // (tensor-map destinations must be 128-byte aligned)
    // (tensor-map destinations 128-byte aligned, 128B-swizzled ones 1024)
    static constexpr int BUF = ((MAP == MAP_STRIDED ? FAC::R * SW : FAC::R * W) * ESZ + 1023) / 1024 * 1024;
    static constexpr int MINB_DB = (227 * 1024) / (2 * BUF + 16 + 1024);
    static constexpr int NBUF = (MAP == MAP_CONTIG && (PAFFT_SB == 2 || (PAFFT_SB == 1 && MINB_DB <= 1))) ? 1 : 2;
    static constexpr int SMEM = NBUF * BUF + 32;
    // resident CTAs per SM the shared memory allows (registers are capped to match)
    static constexpr int MINB_SMEM = (227 * 1024) / (SMEM + 1024);
    // single-buffered CTAs are capped by registers instead: at least ~4 per
    // complex value a thread holds (F_max of them) plus addressing
    static constexpr int REG_FLOOR = FAC::FMAX >= 25 ? 128 : (FAC::FMAX >= 16 ? 96 : (FAC::FMAX >= 9 ? 72 : 64));
    static constexpr int MINB_REG = 65536 / (((NT + 31) / 32 * 32) * REG_FLOOR);
    static constexpr int MAXB = NBUF == 1 ? (MINB_REG < PAFFT_SB_MAX_MINB ? MINB_REG : PAFFT_SB_MAX_MINB)
                                          : PAFFT_MAX_MINB;
    static constexpr int MINB0 = MINB_SMEM < 1 ? 1 : (MINB_SMEM > MAXB ? MAXB : MINB_SMEM);
    // fp32 contiguous tiles of many threads: do not let the occupancy the shared
    // memory allows push the register allocation below ~2/3 of the fp64 floor
    // (config 2 fp32's 486-thread CONV tiles at three CTAs per SM got 40
    // registers and spilled 84 bytes per thread into an L1 that is the pass's
    // limiter)
#ifndef PAFFT_F32_REGCAP
#define PAFFT_F32_REGCAP 1
#endif
    static constexpr int MINB_F32 = 65536 / (((NT + 31) / 32 * 32) * (REG_FLOOR * 2 / 3));
    static constexpr int MINB = (PAFFT_F32_REGCAP && ESZ == 8 && MAP == MAP_CONTIG && NBUF == 2 && MINB_F32 >= 1 &&
                                 MINB_F32 < MINB0)
                                    ? MINB_F32
                                    : MINB0;
    static constexpr int NTB = NT;  // threads per block
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
    // tile, nsig, bps, tiles_per_panel, C all fit 32 bits (checked on the host):
    // 32-bit divisions keep the per-tile bookkeeping cheap
    const unsigned t32 = (unsigned)tile;
    TileGeo g;
    if (!STRIDED) {
        const unsigned ns = (unsigned)a.nsig;
        const unsigned tb = t32 / ns, sig = t32 - tb * ns;
        const long long left = a.bps - (long long)tb * W;
        g.nvalid = left < W ? (int)left : W;
        g.first = (long long)sig * a.bps + (long long)tb * W;
        g.base = g.first * (long long)R;
    } else {
        const unsigned tpp = (unsigned)a.tiles_per_panel;
        const unsigned p = t32 / tpp;
        g.first = (long long)(t32 - p * tpp) * W;
        const long long left = a.C - g.first;
        g.nvalid = left < W ? (int)left : W;
        g.base = (long long)p * a.panel_elems + g.first;
    }
    PAFFT_DASSERT(g.nvalid >= 1 && g.nvalid <= W);
    PAFFT_DASSERT(STRIDED ? (g.first + g.nvalid <= a.C && g.base + (long long)(R - 1) * a.C + g.nvalid <=
                                                              a.panels * a.panel_elems)
                          : (g.base + (long long)g.nvalid * R <= a.panels * a.panel_elems));
    return g;
}

// Issue the bulk copies that stage one tile into `buf` (called by warp 0).
// STRIDED: one copy per row (rows land at buf[j*SW + shift_j]); CONTIG: the
// tile is one contiguous run of nvalid*R elements.  Bulk copies need 16-byte
// aligned addresses and sizes: fp64 always satisfies this; fp32 rows copy the
// enclosing 16-byte-aligned window (shift_j = 1 when the row starts 8 bytes
// into it), and an odd fp32 contiguous tail element is moved by one thread.
__device__ __forceinline__ void tma_load_3d(void* sdst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(sdst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* ssrc, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(ssrc))
                 : "memory");
}
__device__ __forceinline__ void bulk_store_1d(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int R, int W, int SW, typename T>
__device__ __noinline__ void stage_rows(const PassArgs<T>& a, const TileGeo g, cplx<T>* buf, unsigned long long* bar,
                                        int lane) {
    using V = cplx<T>;
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
}

template <int R, int W, int SW, bool STRIDED, typename T>
__device__ __forceinline__ void stage_tile(const PassArgs<T>& a, const CUtensorMap* map, long long tile,
                                           cplx<T>* buf, unsigned long long* bar, int lane) {
    using V = cplx<T>;
    const TileGeo g = tile_geo<R, W, STRIDED>(a, tile);
    if (STRIDED && a.use_tmap) {
        // one 3-D box {SW columns, rb rows, R/rb row groups} = the whole tile,
        // landing densely as [row][SW] (out-of-range columns zero-filled)
        if (lane == 0) {
            const unsigned p = (unsigned)tile / (unsigned)a.tiles_per_panel;
            mbar_expect_tx(bar, (unsigned)(R * SW * sizeof(V)));
            tma_load_3d(buf, map, (int)(2 * g.first), 0, (int)(p * (R / a.rb)), bar);
        }
    } else if (STRIDED) {
        // one bulk copy per row (tiles a tensor map cannot describe): out of
        // line, fp64 tiles always take the tensor-map path
        stage_rows<R, W, SW>(a, g, buf, bar, lane);
    } else if (a.swz) {
        if (lane == 0) {
            mbar_expect_tx(bar, (unsigned)(R * W * sizeof(V)));
            tma_load_3d(buf, map, 0, 0, (int)(g.base * (long long)sizeof(V) / 128 / a.swz_b1), bar);
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
// to global memory in their final order (digit-reversed rows for DIF).
//
// DIF step i (i = 0 .. NS-1): group g = hi * Q_i + lo (hi: digits 0..i-1,
// already frequency; lo: digits i+1.., still spatial); DFT_{F_i} over digit
// i at slots hi * P_i + r * Q_i + lo; then twiddle w_{P_i}^{k lo} (i < last).
// The last step holds frequency k = kf_hi + (R / F_last) * k_last with
// position pos(k) = sum_j rev(k_j) wt(j): DIF stores it there (times the
// external twiddle w_K0^{jj k}); CONV multiplies by ghat[pos] and turns round.
// DIT step i (i = NS-1 .. 0) is the transpose: DFT over digit i (frequency ->
// space), then twiddle w_{P_{i-1}}^{k_{i-1} (m Q_i + lo)} with conj for A-bar.
// DIT kinds read the staged tile in its digit-reversed row order, so digit j
// of a frequency index sits at rev(k_j) wt(j); CONV continues from the DIF's
// natural frequency slots.  Every step reads and writes one slot set (in
// place); the final spatial rows go to global memory with the epilogue.
// The tile's bulk/tensor store from shared memory, committed as one bulk group
// (called by one thread).
template <typename T, int R, int W, bool STRIDED>
__device__ __forceinline__ void issue_tile_store(const PassArgs<T>& a, const CUtensorMap* tmap_dst, long long tile,
                                                 cplx<T>* buf) {
    using V = cplx<T>;
    const TileGeo geo = tile_geo<R, W, STRIDED>(a, tile);
    fence_proxy_async();
    if constexpr (STRIDED) {
        const unsigned p = (unsigned)tile / (unsigned)a.tiles_per_panel;
        tma_store_3d(tmap_dst, buf, (int)(2 * geo.first), 0, (int)(p * (R / a.rb)));
    } else if (a.swz) {
        (void)W;
        tma_store_3d(tmap_dst, buf, 0, 0, (int)(geo.base * (long long)sizeof(V) / 128 / a.swz_b1));
    } else {
        const long long n = (long long)geo.nvalid * R;
        unsigned bytes = (unsigned)(n * sizeof(V));
        if constexpr (sizeof(V) == 8) {
            if (bytes & 15u) {  // odd fp32 element count: tail by hand
                bytes -= 8u;
                a.dst[geo.base + n - 1] = buf[n - 1];
            }
        }
        if (bytes) bulk_store_1d(a.dst + geo.base, buf, bytes);
    }
    bulk_commit();
}

// Steps whose inner index lo = g mod Q_I takes only a few values (Q_I <= 3,
// codelets of <= 9 points, one group per thread): threads are mapped lo-major,
// so lo is uniform across most warps, and the twiddle w_{P_I}^{k lo} is applied
// as compile-time constants for each lo (none for lo = 0) instead of powers of
// a table value.  Measured on B200: config 2's CONV pass -3.5% time; with
// 25-point codelets (config 5) the per-lo code copies cost more than they save.
#ifndef PAFFT_SMALLQ
#define PAFFT_SMALLQ 1
#endif
template <typename FA, int I> struct SmallQ {
    static constexpr bool on = PAFFT_SMALLQ && I < FA::NS - 1 && FA::Q(I) > 1 && FA::Q(I) <= 3 &&
                               FA::f(I) <= 9 && FA::G(I) == FA::GMIN;
};
// The lo-major thread map alone (no constant twiddles) for fp32 steps of odd
// P_I with a short inner run Q_I: in the natural map a half-warp reads
// Q_I-long runs that start P_I elements apart, and for 5 <= Q_I < 16 those runs
// land on overlapping 8-byte bank pairs (config 5 fp32's 25-point step with
// Q = 5: 37% of the CONV pass's shared wavefronts were conflicts); lo-major,
// consecutive lanes are P_I elements apart, and an odd P_I visits 16 distinct
// bank pairs.  (fp64 tiles of these shapes measured conflict-free as they are.)
#ifndef PAFFT_LOMAJOR
#define PAFFT_LOMAJOR 1
#endif
template <typename FA, int I, int ESZ> struct LoMajor {
    static constexpr bool on = PAFFT_LOMAJOR && ESZ == 8 && !SmallQ<FA, I>::on && I < FA::NS - 1 && FA::Q(I) > 1 &&
                               FA::Q(I) < 16 && (FA::P(I) & 1) && FA::G(I) == FA::GMIN;
};
template <int F, int P, int L, int S, typename V> __device__ __forceinline__ void twiddle_lo(V (&z)[F]) {
    static_for<1, F>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        z[k] = twiddle_const<P, k * L, S>(z[k]);
    });
}
template <int F, int P, int Q, int S, typename V> __device__ __forceinline__ void twiddle_small_q(V (&z)[F], int lo) {
    static_for<1, Q>([&](auto lc) {
        constexpr int L = decltype(lc)::value;
        if (lo == L) twiddle_lo<F, P, L, S>(z);
    });
}

// Lane-rotated access for strided tiles of narrow rows.  In a step with
// Q = 1 a group's F rows are consecutive, so with rows of 16*SW < 128 bytes the
// GQ = 128 / (16*SW) groups of a quarter-warp read and write rows that are all
// F rows apart -- the same banks, a GQ-way conflict (config 3's 32-byte rows:
// 4-way on every access of its last step).  Each group instead walks its rows
// starting at a lane-dependent offset (q for natural row order, q * F / GQ for
// digit-reversed order, which spreads the rows over all banks), and the
// registers are rotated back with a log2(GQ)-stage select network.
#ifndef PAFFT_ROT
#define PAFFT_ROT 1
#endif
// z[j] = t[(j - s) mod F] for s = q * unit, q < 2^BITS (barrel shifter of selects)
template <int F, int UNIT, int BITS, typename V> __device__ __forceinline__ void rotate_right(V (&z)[F], int q) {
    static_for<0, BITS>([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        constexpr int sh = (UNIT << b) % F;
        const bool on = (q >> b) & 1;
        V u[F];
#pragma unroll
        for (int j = 0; j < F; ++j) u[j] = on ? z[(j - sh + F) % F] : z[j];
#pragma unroll
        for (int j = 0; j < F; ++j) z[j] = u[j];
    });
}
template <int F, int UNIT, int BITS, typename V> __device__ __forceinline__ void rotate_left(V (&z)[F], int q) {
    static_for<0, BITS>([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        constexpr int sh = (UNIT << b) % F;
        const bool on = (q >> b) & 1;
        V u[F];
#pragma unroll
        for (int j = 0; j < F; ++j) u[j] = on ? z[(j + sh) % F] : z[j];
#pragma unroll
        for (int j = 0; j < F; ++j) z[j] = u[j];
    });
}

// DIT epilogue of the transforms and the standard-order comparator (natural-
// order multiplier of period N, then a scale), kept out of line.
#ifndef PAFFT_EPI_CALL
#define PAFFT_EPI_CALL 1
#endif
template <typename T>
__device__ __noinline__ cplx<T> dit_epilogue(const PassArgs<T>& a, cplx<T> y, long long e, bool ok) {
    if (a.mul && ok) y = cmul(y, __ldg(a.mul + (e % a.N)));
    if (a.has_scale) y = cplx<T>{y.x * a.scale, y.y * a.scale};
    return y;
}

// Warp-local DIF scatter.  The last DIF step writes group g's outputs into the
// input block of g' = digitwise rev(g) (an involution on the last step's
// groups), so a thread map under which every warp's groups are closed under
// g -> g' lets the scatter synchronise with __syncwarp instead of a CTA
// barrier.  ScatterMap packs the orbits (pairs and fixed points) into blocks of
// GPW groups (the groups one warp holds); ok = false when they do not pack.
#ifndef PAFFT_WARP_SCATTER
#define PAFFT_WARP_SCATTER 1
#endif
template <typename FA, int RADIX, int GPW> struct ScatterMap {
    static constexpr int NG = FA::G(FA::NS - 1);
    int sigma[NG];
    bool ok;
    constexpr ScatterMap() : sigma{}, ok(true) {
        int partner[NG] = {};
        for (int g = 0; g < NG; ++g) {
            int hi = g, rv = 0, w = 1;
            for (int jj = FA::NS - 2; jj >= 0; --jj) {  // least significant digit first
                const int fj = FA::f(jj), d = hi % fj;
                hi /= fj;
                rv += revd_rt(d, fj) * w;
                w *= fj;
            }
            partner[g] = rv;
        }
        bool used[NG] = {};
        int pos = 0;
        while (pos < NG && ok) {
            const int room = GPW - pos % GPW;
            int pick = -1;
            for (int g = 0; g < NG && pick < 0; ++g)
                if (!used[g] && partner[g] != g && room >= 2) pick = g;
            if (pick < 0)
                for (int g = 0; g < NG && pick < 0; ++g)
                    if (!used[g] && partner[g] == g) pick = g;
            if (pick < 0) {
                ok = false;
                break;
            }
            used[pick] = true;
            sigma[pos++] = pick;
            if (partner[pick] != pick) {
                used[partner[pick]] = true;
                sigma[pos++] = partner[pick];
            }
        }
    }
    static constexpr int revd_rt(int k, int P) {
        int o = 0;
        for (int p = 1; p < P; p *= RADIX) {
            o = o * RADIX + k % RADIX;
            k /= RADIX;
        }
        return o;
    }
};
template <typename FA, int RADIX, int GPW> __constant__ ScatterMap<FA, RADIX, GPW> kScatter{};

// One tile of a pass (the tile is staged in `buf`; the caller waited for it):
// the column transforms, the epilogue, and the issue of the tile's bulk/tensor
// store (committed as one bulk group by warp 0 lane 0).  `service` is called by
// every thread after the tile's first internal barrier (the deferred refill).
// Threads t >= Pol::NT (a CTA wider than the tile needs) only join the barriers.
template <typename T, int RADIX, typename FA, int KIND, int MAP, typename Pol, bool ALL_ACTIVE, typename Svc>
__device__ __forceinline__ void run_tile(const PassArgs<T>& a, const CUtensorMap* tmap_dst, long long tile,
                                         cplx<T>* buf, const cplx<T>* buf_end, int t, Svc&& service,
                                         unsigned long long* tile_bar = nullptr, unsigned tile_phase = 0) {
    using V = cplx<T>;
    constexpr int R = FA::R, NS = FA::NS, GMIN = FA::GMIN;
    constexpr int W = Pol::W;
    constexpr int SW = Pol::SW;
    constexpr int BUFE = Pol::BUF / (int)sizeof(V);
    constexpr bool STRIDED = MAP == MAP_STRIDED;
    constexpr bool SHIFT = Pol::SHIFT;
    constexpr int FL = FA::f(NS - 1);  // last codelet
    // Results leave through shared memory and one bulk/tensor store per tile
    // (scattered 128-byte STG rows reach ~2 TB/s on B200, bulk stores ~6);
    // fp32 strided tiles (per-row shifted layout) keep register stores.
    constexpr bool TSTORE = !SHIFT;
    constexpr int NGL = FA::G(NS - 1) / GMIN;  // last-step groups per thread
    // warp-local DIF scatter (ScatterMap): strided DIF, one last-step group per
    // thread, whole warps of W-column groups
    constexpr int GPWS = (STRIDED && W <= 32) ? 32 / W : 1;  // groups per warp
    constexpr bool WSCAT = PAFFT_WARP_SCATTER && KIND == KIND_DIF && STRIDED && !SHIFT && NGL == 1 && NS >= 2 &&
                           W <= 32 && 32 % W == 0 && ScatterMap<FA, RADIX, GPWS>().ok;
    // Chebyshev twiddle powers for 16-point steps (codelets.cuh) where enough
    // warps hide its longer chain: contiguous tiles of >= 256 threads
    constexpr bool CHEB16 = !STRIDED && Pol::NT >= 256;
    // lane-rotated Q = 1 steps (PAFFT_ROT): fp64 strided rows narrower than 128 B
    constexpr int GQ = (STRIDED && !SHIFT && SW * (int)sizeof(V) < 128) ? 128 / (SW * (int)sizeof(V)) : 1;
    constexpr int GQB = GQ >= 8 ? 3 : GQ >= 4 ? 2 : GQ >= 2 ? 1 : 0;
    constexpr bool ROT = PAFFT_ROT && sizeof(V) == 16 && GQ > 1 && (FL & (FL - 1)) == 0 && FL >= GQ && (32 % W == 0);
    (void)BUFE;
    (void)buf_end;
    const int warp = t >> 5, lane = t & 31;
    const bool act = ALL_ACTIVE || t < Pol::NT;
    // thread -> (tile column c, group slot gt); STRIDED: c fastest (coalesced
    // W-wide row segments, conflict-free smem rows); CONTIG: group fastest.
    const int c = STRIDED ? t % W : t / GMIN;
    const int gt = STRIDED ? t / W : t % GMIN;
    const int rq = ROT ? gt % GQ : 0;  // this thread's rotation (the group's place in its quarter-warp)
    constexpr int SS = STRIDED ? SW : 1;  // shared stride between consecutive rows
    const long long rs = STRIDED ? (long long)a.C : 1;  // global row stride
    const TileGeo geo = tile_geo<R, W, STRIDED>(a, tile);
    const long long first = geo.first;
    // CONV: this column's filter block (the panel's position inside its signal)
    const V* const gblk =
        KIND == KIND_CONV ? a.ghat + (long long)((unsigned)(first + c) % (unsigned)(a.N / R)) * R : nullptr;
    // one-block double-buffered contiguous tiles are always full: ok is the
    // activity flag (PAFFT_OK_CT)
    const bool ok = (PAFFT_OK_CT && !STRIDED && W == 1 && Pol::NBUF == 2) ? act : (act && c < geo.nvalid);
    V* const scol = STRIDED ? buf + c : buf + c * R;
    // shared element of tile row `row` for this thread's column
    const int codd = SHIFT && !a.use_tmap ? (a.C & 1) : 0;
    const int b0 = SHIFT && !a.use_tmap ? (int)(geo.base & 1) : 0;
    const int swx = a.swz;  // 0/1
    // CONV tiles in the 128B-swizzled layout with a 16-point last step: the
    // group bases gt*16 map a quarter-warp's 8 groups onto 4 swizzle phases
    // (2-way conflicts); groups with bit 2 of gt set walk their 16 rows from
    // the upper half (m ^ 8), which separates the pairs (PAFFT_ROT)
    constexpr bool ROTC = PAFFT_ROT && !STRIDED && KIND == KIND_CONV && sizeof(V) == 16 &&
                          (RADIX == 2 || RADIX == 4 || RADIX == 8) && FL == 16;
    const int rqc = ROTC ? (swx & (gt >> 2) & 1) : 0;
    auto sref = [&](int row) -> V& {
        PAFFT_DASSERT(row >= 0 && row < R);
        if constexpr (!STRIDED && (RADIX == 2 || RADIX == 4 || RADIX == 8)) {
            const int e = c * R + row;
            const int sw = sizeof(V) == 16 ? ((e >> 3) & 7) : (((e >> 4) & 7) << 1);
            PAFFT_DASSERT((e ^ (sw & -swx)) < BUFE);
            return buf[e ^ (sw & -swx)];
        } else {
            PAFFT_DASSERT(&scol[row * SS + (SHIFT ? ((row & codd) ^ b0) : 0)] < buf_end);
            return scol[row * SS + (SHIFT ? ((row & codd) ^ b0) : 0)];
        }
    };
    V* __restrict__ gdst = a.dst + geo.base + (STRIDED ? c : (long long)c * R);
    // external twiddle base/step for this column: w_K0^{jj kf}, w_K0^{jj S}
    auto ext_pair = [&](int kf, int S, V& tw, V& st) {
        const unsigned long long jj = (unsigned long long)(first + c) / a.sq;
        tw = ext_root(a, jj * (unsigned long long)kf);
        st = ext_root(a, jj * (unsigned long long)S);
    };

    // hi index (digits 0..I-1 of a group) -> frequency offset sum k_j L(j)
    // and digit-reversed slot offset sum rev(k_j) wt(j); `rev_in` says the
    // slot digits are already reversed (DIT kinds).
    auto hi_decode = [&](auto Ic, int hi, bool rev_in, int& kf, int& pos) {
        constexpr int I = decltype(Ic)::value;
        kf = 0;
        pos = 0;
        static_for<0, I>([&](auto jc) {
            constexpr int jj = I - 1 - decltype(jc)::value;  // least significant digit first
            constexpr int fj = FA::f(jj);
            const int d = hi % fj;
            hi /= fj;
            const int k = rev_in ? revd<RADIX, fj>(d) : d;
            kf += k * FA::L(jj);
            pos += (rev_in ? d : revd<RADIX, fj>(d)) * FA::Q(jj);
        });
    };

    // DIT kinds: the first step's external twiddle pair w_K0^{jj kf}, w_K0^{jj S}
    // is loaded before waiting for the tile, so the table latency hides under
    // the TMA wait (PAFFT_EXT_HOIST)
    constexpr int NJF = FA::G(NS - 1) / GMIN;
    // (fp64 tiles of full 128-byte rows only: config 3's 2-column tiles, which
    // never carry an external twiddle, measured 2% slower from the extra code,
    // and config 5's fp32 DIT 12% slower)
    constexpr bool HOIST = PAFFT_EXT_HOIST && STRIDED && sizeof(V) == 16 &&
                           (KIND == KIND_DIT_FWD || KIND == KIND_DIT_CONJ) && NJF <= 2 && W >= 8 &&
                           FA::FMAX <= PAFFT_HOIST_FMAX;
    V hw[HOIST ? NJF : 1], hs[HOIST ? NJF : 1];
    if constexpr (HOIST) {
        if (a.ext && ok) {
#pragma unroll
            for (int j = 0; j < NJF; ++j) {
                int kf, pos;
                hi_decode(std::integral_constant<int, NS - 1>{}, gt + j * GMIN, true, kf, pos);
                ext_pair(kf, R / FL, hw[j], hs[j]);
            }
        }
    }
#if PAFFT_TRACE
    // profiling build: time thread 0 spends waiting for the tile to arrive
    // (accumulated in trace[4 bid + 3])
    unsigned long long tw0 = 0;
    if (a.trace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw0));
#endif
    if (tile_bar) mbar_wait(tile_bar, tile_phase);
#if PAFFT_TRACE
    if (a.trace && t == 0) {
        unsigned long long tw1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw1));
        a.trace[4 * blockIdx.x + 3] += tw1 - tw0;
    }
#endif

    // DIF results of the last step, held until every thread has read its
    // last-step inputs (the output rows pos(k) belong to other groups)
    V zl[KIND == KIND_DIF ? NGL : 1][KIND == KIND_DIF ? FL : 1];
    int pl[KIND == KIND_DIF ? NGL : 1];
    if constexpr (KIND == KIND_DIF || KIND == KIND_CONV) {
        static_for<0, NS>([&](auto Ic) {
            constexpr int I = decltype(Ic)::value;
            constexpr int FI = FA::f(I), PI = FA::P(I), QI = FA::Q(I);
            if constexpr (I > 0) __syncthreads();
            if constexpr (I == 1) service();
#pragma unroll
            for (int j = 0; j < (act ? FA::G(I) / GMIN : 0); ++j) {
                constexpr bool SQ = SmallQ<FA, I>::on;
                constexpr bool LM = SQ || (!STRIDED && LoMajor<FA, I, (int)sizeof(V)>::on);
                int g = LM ? (gt % (FA::G(I) / QI)) * QI + gt / (FA::G(I) / QI) : gt + j * GMIN;
                if constexpr (WSCAT && I == NS - 1) g = kScatter<FA, RADIX, GPWS>.sigma[gt];
                const int hi = g / QI, lo = g - (g / QI) * QI;
                const int sb = hi * PI + lo;
                V z[FI];
                if constexpr (ROT && KIND == KIND_DIF && I == NS - 1) {
                    // rows sb + (m + q) mod F, then rotate back
#pragma unroll
                    for (int m = 0; m < FI; ++m) z[m] = sref(sb + ((m + rq) & (FI - 1)));
                    rotate_right<FI, 1, GQB>(z, rq);
                } else if constexpr (ROTC && I == NS - 1) {
#pragma unroll
                    for (int m = 0; m < FI; ++m) z[m] = sref(sb + (m ^ (rqc << 3)));
                    rotate_right<FI, 8, 1>(z, rqc);
                } else {
#pragma unroll
                    for (int m = 0; m < FI; ++m) z[m] = sref(sb + m * QI);
                }
                dft<FI, 1>(z);
                if constexpr (I < NS - 1) {
                    // w_{P_I}^{k lo}: powers of tw[I][Q_I + lo] = w_{P_I}^{lo}
                    if constexpr (SQ) twiddle_small_q<FI, PI, QI, 1>(z, lo);
                    else twiddle_powers<FI, 1, CHEB16>(z, __ldg(a.tw[I] + QI + lo));
#pragma unroll
                    for (int k = 0; k < FI; ++k) sref(sb + k * QI) = z[k];
                } else {
                    // last DIF step (QI == 1, lo == 0): frequency kf + (R/FL) k
                    int kf, pos;
                    hi_decode(Ic, hi, false, kf, pos);
                    if constexpr (KIND == KIND_DIF) {
                        // external twiddle w_K0^{jj k} (a uniform branch: passes
                        // over a whole axis have none)
                        if (a.ext) {
                            V tw{1, 0}, st{1, 0};
                            if (ok) ext_pair(kf, R / FL, tw, st);
#pragma unroll
                            for (int k = 0; k < FI; ++k) {
                                zl[j][k] = cmul(z[k], tw);
                                tw = cmul(tw, st);
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < FI; ++k) zl[j][k] = z[k];
                        }
                        pl[j] = pos;
                    } else {
                        // CONV: x ghat (digit-reversed, 1/N folded in), then the
                        // first DIT-conj step on the same registers
                        if (ok) {
                            // the kernel copy of ghat is stored in this pass's slot
                            // order (ghat[pos(k)] at slot sum k_j wt(j)), k-major:
                            // slot g*FL + k at k*(R/FL) + g, so each load is one
                            // lane-contiguous run (measured: config 3 CONV -15%)
#pragma unroll
                            for (int k = 0; k < FI; ++k) z[k] = cmul(z[k], __ldg(gblk + k * (R / FI) + g));
                        }
                        dft<FI, -1>(z);
                        if constexpr (NS == 1) {
                            if constexpr (TSTORE) {
#pragma unroll
                                for (int m = 0; m < FI; ++m) sref(m) = z[m];
                            } else if (ok) {
#pragma unroll
                                for (int m = 0; m < FI; ++m) gdst[(long long)m * rs] = z[m];
                            }
                        } else {
                            if constexpr (ROTC) {
                                rotate_left<FI, 8, 1>(z, rqc);
#pragma unroll
                                for (int m = 0; m < FI; ++m) sref(sb + (m ^ (rqc << 3))) = z[m];
                            } else {
#pragma unroll
                                for (int m = 0; m < FI; ++m) sref(sb + m) = z[m];
                            }
                        }
                    }
                }
            }
        });
    }

    if constexpr (KIND == KIND_DIF) {
        if constexpr (TSTORE) {
            if constexpr (WSCAT) __syncwarp();
            else __syncthreads();
#pragma unroll
            for (int j = 0; j < (act ? NGL : 0); ++j) {
                if constexpr (ROT) {
                    // frequency (k + q F/GQ) mod F at instruction k: digit-reversed rows spread over the banks
                    rotate_left<FL, FL / GQ, GQB>(zl[j], rq);
#pragma unroll
                    for (int k = 0; k < FL; ++k) sref(pl[j] + revd_rt_dev<RADIX, FL>((k + rq * (FL / GQ)) & (FL - 1))) = zl[j][k];
                } else {
#pragma unroll
                    for (int k = 0; k < FL; ++k) sref(pl[j] + revd<RADIX, FL>(k)) = zl[j][k];
                }
            }
        } else if (ok) {
#pragma unroll
            for (int j = 0; j < NGL; ++j)
#pragma unroll
                for (int k = 0; k < FL; ++k) gdst[(long long)(pl[j] + revd<RADIX, FL>(k)) * rs] = zl[j][k];
        }
    }

    if constexpr (KIND == KIND_DIT_FWD || KIND == KIND_DIT_CONJ || KIND == KIND_CONV) {
        constexpr int S = (KIND == KIND_DIT_FWD) ? 1 : -1;
        constexpr bool FIRST = KIND != KIND_CONV;  // slots hold digit-reversed frequency digits
        auto tw = [](V x, V w) -> V { return S > 0 ? cmul(x, w) : cmulc(x, w); };
        // DIT steps I = NS-1 .. 0 (CONV already did NS-1 in registers)
        static_for<0, NS>([&](auto Rc) {
            constexpr int I = NS - 1 - decltype(Rc)::value;
            constexpr int FI = FA::f(I), PI = FA::P(I), QI = FA::Q(I);
            if constexpr (!(KIND == KIND_CONV && I == NS - 1)) {
                if constexpr (KIND == KIND_CONV || I < NS - 1) __syncthreads();
                if constexpr (KIND != KIND_CONV && I == NS - 2) service();
#pragma unroll
                for (int j = 0; j < (act ? FA::G(I) / GMIN : 0); ++j) {
                    constexpr bool SQ = SmallQ<FA, I>::on;
                    constexpr bool LM = SQ || (!STRIDED && LoMajor<FA, I, (int)sizeof(V)>::on);
                    const int g = LM ? (gt % (FA::G(I) / QI)) * QI + gt / (FA::G(I) / QI) : gt + j * GMIN;
                    const int hi = g / QI, lo = g - (g / QI) * QI;
                    const int sb = hi * PI + lo;
                    V z[FI];
                    constexpr bool RL = ROT && FIRST && I == NS - 1;  // rotated Q = 1 step
                    if constexpr (RL) {
#pragma unroll
                        for (int k = 0; k < FI; ++k)
                            z[k] = sref(sb + revd_rt_dev<RADIX, FI>((k + rq * (FI / GQ)) & (FI - 1)));
                        rotate_right<FI, FI / GQ, GQB>(z, rq);
                    } else {
#pragma unroll
                        for (int k = 0; k < FI; ++k) z[k] = sref(sb + (FIRST ? revd<RADIX, FI>(k) : k) * QI);
                    }
                    if constexpr (FIRST && I == NS - 1) {
                        // pre-twiddle w_K0^{+-jj k} on the first DIT step
                        if (a.ext && ok) {
                            V w, st;
                            if constexpr (HOIST) {
                                w = hw[j];
                                st = hs[j];
                            } else {
                                int kf, pos;
                                hi_decode(std::integral_constant<int, I>{}, hi, true, kf, pos);
                                ext_pair(kf, R / FL, w, st);
                            }
#pragma unroll
                            for (int k = 0; k < FI; ++k) {
                                z[k] = tw(z[k], w);
                                w = cmul(w, st);
                            }
                        }
                    }
                    // pre-twiddle: the transpose of DIF step I's w_{P_I}^{k lo}
                    if constexpr (I < NS - 1) {
                        if constexpr (SQ) twiddle_small_q<FI, PI, QI, S>(z, lo);
                        else twiddle_powers<FI, S, CHEB16>(z, __ldg(a.tw[I] + QI + lo));
                    }
                    dft<FI, S>(z);
                    if constexpr (I > 0) {
                        if constexpr (RL) {
                            rotate_left<FI, 1, GQB>(z, rq);
#pragma unroll
                            for (int m = 0; m < FI; ++m) sref(sb + ((m + rq) & (FI - 1))) = z[m];
                        } else {
#pragma unroll
                            for (int m = 0; m < FI; ++m) sref(sb + m * QI) = z[m];
                        }
                    } else {
                        // final spatial rows m * Q_0 + lo (hi == 0), epilogue in registers
                        V* gp = gdst + (long long)lo * rs;
#pragma unroll
                        for (int m = 0; m < FI; ++m) {
                            V y = z[m];
                            // (the CONV pass never has an epilogue: 1/N is in its filter copy)
                            if constexpr (KIND != KIND_CONV) {
#if PAFFT_EPI_CALL
                                // out of line: the permutation-free passes never take it
                                if (a.mul || a.has_scale)
                                    y = dit_epilogue(a, y, (gp - a.dst) + (long long)(m * QI) * rs, ok);
#else
                                if (a.mul && ok) {
                                    const long long e = (gp - a.dst) + (long long)(m * QI) * rs;
                                    y = cmul(y, __ldg(a.mul + (e % a.N)));
                                }
                                if (a.has_scale) y = V{y.x * a.scale, y.y * a.scale};
#endif
                            }
                            if constexpr (TSTORE) sref(sb + m * QI) = y;
                            else if (ok) gp[(long long)(m * QI) * rs] = y;
                        }
                    }
                }
            }
        });
    }
    // the tile is final in shared memory: one bulk/tensor store by warp 0
    __syncthreads();
    if (warp == 0) {
        if constexpr (TSTORE) {
            if (lane == 0) issue_tile_store<T, R, W, STRIDED>(a, tmap_dst, tile, buf);
            __syncwarp();
        }
    }
}

// L2 prefetch of bytes [lo, hi) of a buffer (one thread): the bulk prefetch
// needs a 16-byte aligned address and size, so the range is widened to 16-byte
// bounds and clipped to `limit` (fp32 blocks of odd length start 8 bytes off).
__device__ __forceinline__ void l2_prefetch_range(const void* base, long long lo, long long hi, long long limit) {
    lo &= ~15ll;
    hi = (hi + 15) & ~15ll;
    if (hi > (limit & ~15ll)) hi = limit & ~15ll;
    if (hi > lo)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(base) + lo),
                     "r"((unsigned)(hi - lo))
                     : "memory");
}

// The filter blocks a CONV tile will multiply by, into L2 ahead of the
// multiply: measured on B200 config 4 (256 MiB filter) CONV -9%, config 2
// (24 MiB) -2%; a filter of a few MiB stays in L2 anyway (size floor).
template <int R, int W, typename T>
__device__ __forceinline__ void prefetch_filter_blocks(const PassArgs<T>& a, long long tile) {
    using V = cplx<T>;
    if (a.N * (long long)sizeof(V) < (8ll << 20)) return;
    const TileGeo g = tile_geo<R, W, false>(a, tile);
    const long long nb = a.N / R, b0 = g.first % nb;
    const long long nblk = b0 + g.nvalid <= nb ? g.nvalid : nb - b0;
    l2_prefetch_range(a.ghat, b0 * R * (long long)sizeof(V), (b0 + nblk) * R * (long long)sizeof(V),
                      a.N * (long long)sizeof(V));
}

// WOVR > 0: an instance with W = WOVR columns per tile (the wide strided
// variants of inst/inst_wide.cu, taken by launches with many tiles).
template <typename T, int RADIX, int F0, int F1, int F2, int F3, int KIND, int MAP, int WOVR = 0>
__global__ void __launch_bounds__(TilePolicy<T, Fac<F0, F1, F2, F3>, MAP, WOVR>::NTB,
                                  TilePolicy<T, Fac<F0, F1, F2, F3>, MAP, WOVR>::MINB)
    pass_kernel(const PassArgs<T> a, const __grid_constant__ CUtensorMap tmap,
                const __grid_constant__ CUtensorMap tmap_dst) {
    using V = cplx<T>;
    using FA = Fac<F0, F1, F2, F3>;
    using Pol = TilePolicy<T, FA, MAP, WOVR>;
    constexpr int R = FA::R, NS = FA::NS;
    constexpr int W = Pol::W;
    constexpr int SW = Pol::SW;
    constexpr int BUFE = Pol::BUF / (int)sizeof(V);  // elements per tile buffer
    constexpr bool STRIDED = MAP == MAP_STRIDED;
    constexpr bool TSTORE = !Pol::SHIFT;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    V* const bufs = reinterpret_cast<V*>(smem_raw);
    constexpr int NBUF = Pol::NBUF;
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(smem_raw + NBUF * Pol::BUF);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;

    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = blockIdx.x, ts = gridDim.x;
    // tile sequence T_0 = t0, T_i = t0 + i ts (static) or ts + atomicAdd(ctr, 1)
    // (dynamic: CTAs that run faster take more tiles, so the launch has no
    // ragged tail).  Warp 0 fetches T_i when it issues that tile's staging and
    // leaves it in nxt[i & 1] for the other warps (read after a CTA barrier).
    int* const nxt = reinterpret_cast<int*>(bars + 2);
    const bool dyn = a.ctr != nullptr;
    // (lane 0 keeps one ticket in hand, taken at the previous staging, so the
    // atomic's round trip is off the refill's critical path)
    unsigned ahead = 0;
    if (dyn && t == 0) ahead = atomicAdd(a.ctr, 1u);
    auto fetch = [&](int i) -> long long {  // warp 0, all lanes
        if (!dyn) return t0 + (long long)i * ts;
        unsigned v = 0;
        if (lane == 0) {
            const unsigned long long w = (unsigned long long)ts + ahead;
            ahead = atomicAdd(a.ctr, 1u);
            v = w < (unsigned long long)a.tiles ? (unsigned)w : (unsigned)a.tiles;
            nxt[i & 1] = (int)v;
        }
        return (long long)__shfl_sync(0xffffffffu, v, 0);
    };
    if (warp == 0) {
        if (t0 < a.tiles) stage_tile<R, W, SW, STRIDED>(a, &tmap, t0, bufs, &bars[0], lane);
        if constexpr (NBUF == 2) {
            const long long t1 = fetch(1);
            if (t1 < a.tiles) stage_tile<R, W, SW, STRIDED>(a, &tmap, t1, bufs + BUFE, &bars[1], lane);
        }
    }
    __syncthreads();  // hand-copied fp32 tail elements of the first tiles

    // Deferred refill: after storing tile i from buffer b, the refill of b
    // with tile i+2 waits for the store to drain shared memory; warp 0 does
    // that after the next tile's first barrier instead of stalling the CTA.
    int pend = -1;  // sequence index of the tile to stage, -1 = none
    V* pbuf = nullptr;
    unsigned long long* pbar = nullptr;
    auto service = [&]() {
        if (warp == 0 && pend >= 0) {
            const long long nt = fetch(pend);
            if (nt < a.tiles) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
                fence_proxy_async();
                stage_tile<R, W, SW, STRIDED>(a, &tmap, nt, pbuf, pbar, lane);
                // (the instruction-cache-bound 25-point kernels, config 5, lose ~1%
                // to the extra code, so they skip it)
                if constexpr (KIND == KIND_CONV && PAFFT_GHAT_PF && FA::FMAX < 25) {
                    if (lane == 0) prefetch_filter_blocks<R, W>(a, nt);
                }
            }
        }
        pend = -1;
    };
#if PAFFT_TRACE
    if (a.trace && t == 0) {  // straight to memory: no register lives across the tile loop
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        a.trace[4 * blockIdx.x] = now;
    }
#endif
    int it = 0;
    for (long long tile = t0; tile < a.tiles; ++it) {
        const int b = NBUF == 2 ? (it & 1) : 0;
        V* const buf = bufs + b * BUFE;
        run_tile<T, RADIX, FA, KIND, MAP, Pol, Pol::NTB == Pol::NT>(a, &tmap_dst, tile, buf, bufs + NBUF * BUFE, t,
                                                                    service, &bars[b],
                                                                    NBUF == 2 ? ((it >> 1) & 1) : (it & 1));
        // this buffer's next tile is T_{it + NBUF} (staged only if it exists)
        if (dyn || tile + NBUF * ts < a.tiles) {
            pend = it + NBUF;
            pbuf = buf;
            pbar = &bars[b];
        }
        // no later barrier in the next tile (or the next tile is this refill)
        if constexpr (!TSTORE || NS == 1 || NBUF == 1) service();
        // single buffer: an fp32 tail element hand-copied by the refill must be
        // visible before the next tile's first shared-memory reads (and, in
        // dynamic order, the next tile's index)
        if constexpr (NBUF == 1) {
            if (sizeof(V) == 8 || dyn) __syncthreads();
        }
        // T_{it+1}: fetched by the prologue or by a service() that ran before
        // this tile's last barrier (NBUF == 1: the barrier above)
        tile = dyn ? (long long)nxt[(it + 1) & 1] : tile + ts;
    }
    service();
    if constexpr (TSTORE) {
        if (t == 0) bulk_wait0();  // stores complete before the CTA retires
    }
#if PAFFT_TRACE
    if (a.trace && t == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        a.trace[4 * blockIdx.x + 1] = t1;
        a.trace[4 * blockIdx.x + 2] = (unsigned long long)it;
    }
#endif
    if (dyn && t == 0) {
        // every fetch of this CTA precedes this increment: the last CTA to
        // arrive resets the pair
        __threadfence();
        if (atomicAdd(a.ctr + 1, 1u) == gridDim.x - 1) {
            a.ctr[0] = 0;
            a.ctr[1] = 0;
        }
    }
}

}  // namespace pafft_b200
