// libpafft_b200: host runtime behind include/pafft_b200.h.
//
// Owns plans (device twiddle tables + pass schedule, replacing Plan::Plan,
// core.cpp:93-127), prepared filters (prepare_filter, convolution.cpp:9-14),
// and issues the pass kernels (pass.cuh) for convolve_permfree
// (convolution.cpp:45-52), convolve_standard (:37-43) and the transforms
// (transform.cpp:8-26).  No CPU compute fallback exists: every transform runs
// in the sm_100a kernels; the host only builds tables and moves buffers.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/pafft_b200.h"
#include "pass.cuh"
#include "registry.h"

using namespace pafft_b200;

namespace {

// ------------------------------------------------------------ errors --
thread_local std::string g_err;
thread_local size_t g_err_dim = 0, g_err_extent = 0;
thread_local uint64_t g_perm_passes = 0;
thread_local uint64_t g_launches = 0;
thread_local uint64_t g_dynamic_launches = 0;  // pass launches that handed tiles out dynamically

pafft_status fail(pafft_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(PAFFT_CUDA_ERROR, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                        __FILE__, __LINE__);                                                        \
    } while (0)

#define ST_TRY(expr)                      \
    do {                                  \
        pafft_status s_ = (expr);         \
        if (s_ != PAFFT_OK) return s_;    \
    } while (0)

// ---------------------------------------------------------- registry --
Registry& registry() {
    static Registry reg;
    static std::once_flag once;
    std::call_once(once, [] {
        register_r2_f64(reg);
        register_r3_f64(reg);
        register_r4_f64(reg);
        register_r5_f64(reg);
        register_r8_f64(reg);
        register_r2_f32(reg);
        register_r3_f32(reg);
        register_r4_f32(reg);
        register_r5_f32(reg);
        register_r8_f32(reg);
        register_wide_f64(reg);
    });
    return reg;
}

const KernelEntry* find_kernel(int prec, int radix, int R, int kind, int map, int wide = 0) {
    for (const auto& e : registry())
        if (e.prec == prec && e.radix == radix && e.R == R && e.kind == kind && e.map == map && e.wide == wide)
            return &e;
    return nullptr;
}

int max_stages_compiled(int prec, int radix, int kind, int map) {
    int best = 0;
    for (const auto& e : registry()) {
        if (e.radix != radix || e.prec != prec || e.kind != kind || e.map != map || e.wide) continue;
        int s = 0;
        for (int v = e.R; v > 1; v /= radix) ++s;
        best = std::max(best, s);
    }
    return best;
}

bool radix_ok(unsigned r) { return r == 2 || r == 3 || r == 4 || r == 5 || r == 8; }

// ------------------------------------------------------------- tables --
// exp(-2 pi i e / K) in long double, rounded once (TwiddleTable semantics,
// core.cpp:84-91, at higher internal precision).
inline void root(unsigned long long e, unsigned long long K, long double& c, long double& s) {
    const long double pi = 3.141592653589793238462643383279502884L;
    const unsigned long long g = e % K;
    const long double a = -2.0L * pi * (long double)g / (long double)K;
    c = cosl(a);
    s = sinl(a);
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// Per-call scratch, stream-ordered (cudaMallocAsync / cudaFreeAsync on the
// call's stream): Plan stays immutable, so calls on distinct buffers may run
// concurrently from several threads and streams.
struct AsyncBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~AsyncBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

struct PassDesc {
    int kind = 0;
    int axis = 0, a = 0, s = 0;
    int R = 0, F[4] = {1, 1, 1, 1}, nsteps = 1;
    long long K0 = 0, L = 0, sq = 1, C = 1;
    int contig = 0, W = 1, NT = 32;
    size_t smem = 0;
    long long max_ctas = 1;
    int occ = 1;  // resident CTAs per SM
    int dense = 0;  // fp32 strided tile without spare row slots (even row lengths, tensor maps)
    int use_tmap = 0, rb = 0, sw = 0;  // STRIDED tensor-map staging
    int swz = 0, swz_b1 = 0;           // CONTIG 128B-swizzled staging (power-of-two radix)
    int ext = 0;
    unsigned ext_bits = 0;
    const void* ext_lo = nullptr;
    const void* ext_hi = nullptr;
    const void* tw[3] = {nullptr, nullptr, nullptr};
    const void* fn = nullptr;
    // wide strided variant (16 columns, 256-byte rows), taken by launches
    // with many tiles (use_wide)
    std::shared_ptr<PassDesc> wide;
};

struct Group {
    int axis, a, s;
};

}  // namespace

struct pafft_plan_s {
    unsigned radix = 0;          // radix of axis 0 (the pafft Radix when uniform)
    unsigned radices[8] = {0};   // per-axis radix
    int rank = 0;
    size_t dims[8] = {0};
    unsigned depth[8] = {0};
    size_t total = 0;
    int prec = 0;
    int device = 0;
    size_t esize = 16;  // bytes per complex element
    std::vector<Group> groups;                 // DIF order; last = contiguous axis-0 group
    std::vector<std::unique_ptr<DevBuf>> owned;
    std::map<long long, std::pair<const void*, const void*>> ext_tables;  // K0 -> (lo, hi)
    std::map<std::string, std::vector<const void*>> int_tables;            // split -> step tables
    std::map<long long, unsigned> ext_bits;
    std::vector<uint32_t*> rev_dev;            // per-axis digit reversal maps (device)
    std::unique_ptr<DevBuf> stage[4];
    cudaStream_t streams[4] = {nullptr, nullptr, nullptr, nullptr};
    std::mutex mu;
    std::mutex host_mu;  // serialises the host-buffer pipeline (plan-owned streams + staging)
    // pass schedules, built once at plan creation (immutable afterwards)
    std::vector<PassDesc> pf, dif, dit_fwd, dit_conj;
    // slot layout of the filter's kernel copy: the CONV pass's (axis, R,
    // F0..F3) -- set by the pass schedule, which depends on PAFFT_* tuning
    // variables read at plan creation, so it is part of the filter key
    long long layout[6] = {0, 0, 0, 0, 0, 0};
    std::map<std::string, CUtensorMap> tmaps;
};

struct pafft_filter_s {
    pafft_plan_t plan = nullptr;  // key: (radices, dims, precision, device)
    unsigned radix = 0;
    unsigned radices[8] = {0};
    int rank = 0;
    size_t dims[8] = {0};
    int prec = 0, device = 0;
    long long layout[6] = {0, 0, 0, 0, 0, 0};  // kernel-copy slot layout (plan's CONV pass)
    std::shared_ptr<DevBuf> ghat;         // unscaled, plan precision
    std::shared_ptr<DevBuf> ghat_scaled;  // x (1/N), plan precision (shared by cached filters)
};

namespace {

pafft_status alloc(pafft_plan_t p, size_t bytes, void** out) {
    auto b = std::make_unique<DevBuf>();
    CUDA_TRY(cudaMalloc(&b->p, bytes ? bytes : 16));
    b->bytes = bytes;
    *out = b->p;
    p->owned.push_back(std::move(b));
    return PAFFT_OK;
}

template <typename T>
pafft_status upload_roots(pafft_plan_t p, const std::vector<long double>& re, const std::vector<long double>& im,
                          const void** out) {
    std::vector<cplx<T>> h(re.size());
    for (size_t i = 0; i < re.size(); ++i) h[i] = cplx<T>{(T)re[i], (T)im[i]};
    void* d;
    ST_TRY(alloc(p, h.size() * sizeof(cplx<T>), &d));
    CUDA_TRY(cudaMemcpy(d, h.data(), h.size() * sizeof(cplx<T>), cudaMemcpyHostToDevice));
    *out = d;
    return PAFFT_OK;
}

pafft_status upload(pafft_plan_t p, const std::vector<long double>& re, const std::vector<long double>& im,
                    const void** out) {
    return p->prec == 0 ? upload_roots<double>(p, re, im, out) : upload_roots<float>(p, re, im, out);
}

pafft_status ext_table(pafft_plan_t p, long long K0, PassDesc& d) {
    auto it = p->ext_tables.find(K0);
    if (it == p->ext_tables.end()) {
        unsigned lg = 0;
        while ((1ll << lg) < K0) ++lg;
        const unsigned bits = (lg + 1) / 2;
        const long long nlo = 1ll << bits;
        const long long nhi = (K0 + nlo - 1) / nlo;
        std::vector<long double> lr(nlo), li(nlo), hr(nhi), hi(nhi);
        for (long long e = 0; e < nlo; ++e) root(e, K0, lr[e], li[e]);
        for (long long h = 0; h < nhi; ++h) root((unsigned long long)h * nlo, K0, hr[h], hi[h]);
        const void *lo, *hip;
        ST_TRY(upload(p, lr, li, &lo));
        ST_TRY(upload(p, hr, hi, &hip));
        p->ext_tables[K0] = {lo, hip};
        p->ext_bits[K0] = bits;
        it = p->ext_tables.find(K0);
    }
    d.ext_lo = it->second.first;
    d.ext_hi = it->second.second;
    d.ext_bits = p->ext_bits[K0];
    return PAFFT_OK;
}

// Internal twiddles of step i: tw[i][k * Q_i + lo] = w_{P_i}^{k lo}
// (P_i = F_i ... F_last, Q_i = P_i / F_i), keyed by the split.
pafft_status int_table(pafft_plan_t p, PassDesc& d) {
    char key[64];
    snprintf(key, sizeof key, "%d/%d/%d/%d", d.F[0], d.F[1], d.F[2], d.F[3]);
    auto it = p->int_tables.find(key);
    if (it == p->int_tables.end()) {
        std::vector<const void*> tabs;
        for (int i = 0; i + 1 < d.nsteps; ++i) {
            long long P = 1;
            for (int j = i; j < d.nsteps; ++j) P *= d.F[j];
            const long long Q = P / d.F[i];
            std::vector<long double> re(P), im(P);
            for (long long k = 0; k < d.F[i]; ++k)
                for (long long lo = 0; lo < Q; ++lo) root((unsigned long long)(k * lo), P, re[k * Q + lo], im[k * Q + lo]);
            const void* t;
            ST_TRY(upload(p, re, im, &t));
            tabs.push_back(t);
        }
        p->int_tables[key] = tabs;
        it = p->int_tables.find(key);
    }
    for (size_t i = 0; i < 3; ++i) d.tw[i] = i < it->second.size() ? it->second[i] : nullptr;
    return PAFFT_OK;
}

long long ipow(long long b, int e) {
    long long v = 1;
    while (e-- > 0) v *= b;
    return v;
}

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

// Stage groups in DIF order (north_star item 4: per-axis passes, no global
// transposes).  Strided axes first (any order is valid: modes commute,
// SPEC.md:226), then axis 0 split so its last group is a contiguous block.
void build_groups(pafft_plan_t p) {
    p->groups.clear();
    for (int q = p->rank - 1; q >= 0; --q) {
        const int t = (int)p->depth[q];
        if (t == 0) continue;
        const unsigned radix = p->radices[q];
        const int maxs = max_stages_compiled(p->prec, (int)radix, KIND_CONV, MAP_CONTIG);
        const int max_mid = std::min(maxs, env_int("PAFFT_MAX_MID_STAGES", maxs));
        int max_str = max_stages_compiled(p->prec, (int)radix, KIND_DIF, MAP_STRIDED);
        if (radix == 2) max_str = std::min(max_str, 11);
        // fp32 strided rows of an odd number of elements (odd radix, all lower
        // extents odd) alternate between 16-byte aligned and misaligned starts, so
        // no tensor map describes them and each row is staged by its own bulk
        // copy.  That needs long rows: the 729- and 625-row groups (81 / 125
        // threads per column) are held to 8 columns by the 1024-thread limit, 80-byte
        // copies that run at ~0.5 TB/s, while 16-column groups reach ~3 TB/s and
        // single-codelet ones (64 columns) the HBM roof.  Such axes therefore stop
        // at 81 / 125 rows per strided pass (measured: 243 rows in one pass is 21%
        // slower than 9 + 27) and take one more round trip each way instead:
        // config 2 in fp32 9.6k -> 38.0k conv/s, 5^9 2.6x, 729 x 729 3.9x
        // (profiles/r02_f32_odd_schedule.log).
        {
            unsigned long long sq = 1;
            for (int i = 0; i < q; ++i) sq *= (unsigned long long)p->dims[i];
            if (p->esize == 8 && (radix & 1) && (sq & 1) && env_int("PAFFT_F32_ODD_SINGLE", 1))
                max_str = std::min(max_str, radix == 3 ? 4 : 3);
        }
        max_str = std::min(max_str, env_int("PAFFT_MAX_STRIDED_STAGES", max_str));
        const int lim = (q == 0) ? std::max(max_mid, 1) : std::max(max_str, 1);
        const int forced_mid = env_int("PAFFT_MID_STAGES", 0);
        int mid_pref = 1;
        while (mid_pref + 1 <= max_mid && ipow(radix, mid_pref + 1) * (long long)p->esize <= 64 * 1024) ++mid_pref;
        if (q == 0 && forced_mid > 0 && forced_mid < t && forced_mid <= max_mid) {
            // tuning override: contiguous group of exactly forced_mid stages,
            // the rest split evenly into strided groups
            const int rest = t - forced_mid;
            const int npass = (rest + max_str - 1) / max_str;
            int a = 0;
            for (int i = 0; i < npass; ++i) {
                const int s = rest / npass + (i >= npass - rest % npass ? 1 : 0);
                p->groups.push_back({q, a, s});
                a += s;
            }
            p->groups.push_back({q, a, forced_mid});
        } else if (q == 0 && t > mid_pref) {
            // Contiguous (CONV) group: the largest block of <= 64 KB (measured on
            // B200: 2^12 fp64 for config 1, 3^7 for config 2, 5^5 for config 5);
            // the remaining stages split evenly into strided groups.
            const int mid = mid_pref;
            const int rest = t - mid;
            const int npass = (rest + max_str - 1) / max_str;
            int a = 0;
            for (int i = 0; i < npass; ++i) {
                const int s = rest / npass + (i >= npass - rest % npass ? 1 : 0);
                p->groups.push_back({q, a, s});
                a += s;
            }
            p->groups.push_back({q, a, mid});
        } else {
            const int npass = (t + lim - 1) / lim;
            int rem = t, a = 0;
            for (int i = 0; i < npass; ++i) {
                const int s = (rem + (npass - i) - 1) / (npass - i);
                p->groups.push_back({q, a, s});
                a += s;
                rem -= s;
            }
        }
    }
    // The CONV pass needs the last group to be contiguous (axis 0, L == 1).
    // Axis-0 groups are emitted last, in ascending stage order; ensure the
    // contiguous one ends the list even if axis 0 has extent 1.
}

// The kernel-instance part of a pass: entry point, codelet split, tile
// policy, and the persistent grid (every resident CTA slot, no more).
pafft_status bind_kernel(pafft_plan_t p, const KernelEntry& ke, PassDesc& d) {
    d.fn = ke.fn;
    d.F[0] = ke.F0;
    d.F[1] = ke.F1;
    d.F[2] = ke.F2;
    d.F[3] = ke.F3;
    d.nsteps = 1 + (d.F[1] > 1) + (d.F[2] > 1) + (d.F[3] > 1);
    d.W = ke.W;
    d.NT = ke.NT;
    d.smem = (size_t)ke.smem;
    if (d.smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(d.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem));
    int occ = 0, sms = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, d.fn, d.NT, d.smem));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
    if (occ < 1) return fail(PAFFT_CUDA_ERROR, "pass kernel R=%d cannot be resident (smem %zu)", d.R, d.smem);
    d.max_ctas = (long long)occ * sms;
    d.occ = occ;
    d.dense = ke.wide == 2;
    if (!d.contig) d.sw = (p->esize == 8 && !d.dense) ? d.W + 2 : d.W;
    return PAFFT_OK;
}

pafft_status make_pass(pafft_plan_t p, const Group& g, int kind, PassDesc& d) {
    const long long n = (long long)p->dims[g.axis];
    long long sq = 1;
    for (int q = 0; q < g.axis; ++q) sq *= (long long)p->dims[q];
    d.kind = kind;
    d.axis = g.axis;
    d.a = g.a;
    d.s = g.s;
    const unsigned radix = p->radices[g.axis];
    d.R = (int)ipow(radix, g.s);
    d.K0 = n / ipow(radix, g.a);
    d.L = d.K0 / d.R;
    d.sq = sq;
    d.C = d.L * sq;
    d.contig = d.C == 1;
    const KernelEntry* ke = find_kernel(p->prec, (int)radix, d.R, kind, d.contig ? MAP_CONTIG : MAP_STRIDED);
    // 2-D tensor map staging: row groups of rb rows, at most 256 groups per box
    int rb = 1;
    for (int v = 1; v <= 256 && v <= d.R; ++v)
        if (d.R % v == 0) rb = v;
    // fp32 strided tiles of even row length whose box a tensor map can describe
    // take the dense instance (PAFFT_F32_DENSE=0: the spare-slot one everywhere)
    if (ke && !d.contig && p->esize == 8 && d.C % 2 == 0 && d.R / rb <= 256 && env_int("PAFFT_F32_DENSE", 1) &&
        env_int("PAFFT_NO_TMAP", 0) == 0) {
        const KernelEntry* de = find_kernel(p->prec, (int)radix, d.R, kind, MAP_STRIDED, 2);
        if (de && de->F0 == ke->F0 && de->F1 == ke->F1 && de->F2 == ke->F2 && de->F3 == ke->F3) ke = de;
    }
    if (!ke)
        return fail(PAFFT_INVALID_ARGUMENT, "no kernel for radix %u R=%d kind %d map %d", radix, d.R, kind,
                    d.contig);
    ST_TRY(bind_kernel(p, *ke, d));
    if (d.contig && (radix == 2 || radix == 4 || radix == 8) && env_int("PAFFT_NO_SWIZZLE", 0) == 0) {
        const long long tile_bytes = (long long)d.R * d.W * (long long)p->esize;
        if (tile_bytes % 1024 == 0) {
            const long long tr = tile_bytes / 128;
            d.swz_b1 = (int)std::min<long long>(tr, 256);
            d.swz = (tr % d.swz_b1 == 0 && tr / d.swz_b1 <= 256) ? 1 : 0;
        }
    }
    if (!d.contig) {
        // 2-D tensor map staging needs 16-byte row strides (always for fp64,
        // even C for fp32); otherwise one bulk copy per row (d.sw: bind_kernel).
        // fp64 strided tiles always stage and store through tensor maps (their
        // tile store is a tensor store); fp32 ones may use per-row copies
        d.use_tmap = p->esize == 16 || ((d.C % 2) == 0 && env_int("PAFFT_NO_TMAP", 0) == 0);
        int rb = 1;
        for (int v = 1; v <= 256 && v <= d.R; ++v)
            if (d.R % v == 0) rb = v;
        d.rb = rb;
        if (d.R / rb > 256) {
            if (p->esize == 16) return fail(PAFFT_INVALID_ARGUMENT, "strided tile of %d rows has no tensor-map box", d.R);
            d.use_tmap = 0;
        }
    }
    d.ext = d.L > 1;
    if (d.ext) ST_TRY(ext_table(p, d.K0, d));
    if (d.nsteps > 1) ST_TRY(int_table(p, d));
    if (!d.contig) {
        const KernelEntry* we = find_kernel(p->prec, (int)radix, d.R, kind, MAP_STRIDED, 1);
        if (we && we->W > d.W && we->F0 == d.F[0] && we->F1 == d.F[1] && we->F2 == d.F[2] && we->F3 == d.F[3] &&
            env_int("PAFFT_WIDE", 1)) {
            auto wd = std::make_shared<PassDesc>(d);
            wd->wide.reset();
            ST_TRY(bind_kernel(p, *we, *wd));
            d.wide = wd;
        }
    }
    return PAFFT_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
    });
    return fn;
}

// 2-D view of a pass input: rows of C complex (2C reals), box = rb rows x sw
// complex columns.  Cached per (buffer, geometry).
pafft_status tensor_map(pafft_plan_t p, const PassDesc& d, const void* src, size_t batch, CUtensorMap* out) {
    const unsigned long long rows = (unsigned long long)p->total * batch / (unsigned long long)d.C;
    char key[160];
    snprintf(key, sizeof key, "%p/%lld/%llu/%d/%d/%d", src, d.C, rows, d.sw, d.rb, p->prec);
    {
        std::lock_guard<std::mutex> lk(p->mu);
        auto it = p->tmaps.find(key);
        if (it != p->tmaps.end()) {
            *out = it->second;
            return PAFFT_OK;
        }
    }
    auto enc = encode_fn();
    if (!enc) return fail(PAFFT_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    // 3-D view {2C reals, rb rows, (rows / rb) row groups}: one box = one tile
    const unsigned long long nb = (unsigned long long)(d.R / d.rb);
    const cuuint64_t dims[3] = {(cuuint64_t)(2 * d.C), (cuuint64_t)d.rb, (cuuint64_t)(rows / d.rb)};
    const cuuint64_t strides[2] = {(cuuint64_t)(d.C * p->esize), (cuuint64_t)(d.rb * d.C * p->esize)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * d.sw), (cuuint32_t)d.rb, (cuuint32_t)nb};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    const CUresult r = enc(&m, p->prec == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(src), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PAFFT_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    std::lock_guard<std::mutex> lk(p->mu);
    if (p->tmaps.size() > 4096) p->tmaps.clear();
    p->tmaps[key] = m;
    *out = m;
    return PAFFT_OK;
}

// Contiguous tiles as rows of 128 bytes, SWIZZLE_128B: 3-D view
// {128 B of reals, b1 rows, row groups}; one box = one tile.
pafft_status tensor_map_swz(pafft_plan_t p, const PassDesc& d, const void* src, size_t batch, CUtensorMap* out) {
    const unsigned long long rows = (unsigned long long)p->total * batch * p->esize / 128;
    char key[160];
    snprintf(key, sizeof key, "swz/%p/%llu/%d/%d/%d", src, rows, d.R * d.W, d.swz_b1, p->prec);
    {
        std::lock_guard<std::mutex> lk(p->mu);
        auto it = p->tmaps.find(key);
        if (it != p->tmaps.end()) {
            *out = it->second;
            return PAFFT_OK;
        }
    }
    auto enc = encode_fn();
    if (!enc) return fail(PAFFT_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const unsigned long long tr = (unsigned long long)d.R * d.W * p->esize / 128;
    const unsigned inner = p->prec == 0 ? 16u : 32u;  // reals per 128-byte row
    const cuuint64_t dims[3] = {inner, (cuuint64_t)d.swz_b1, (cuuint64_t)(rows / d.swz_b1)};
    const cuuint64_t strides[2] = {128, (cuuint64_t)128 * d.swz_b1};
    const cuuint32_t box[3] = {inner, (cuuint32_t)d.swz_b1, (cuuint32_t)(tr / d.swz_b1)};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    const CUresult r = enc(&m, p->prec == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(src), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PAFFT_CUDA_ERROR, "cuTensorMapEncodeTiled (swizzled) failed (%d)", (int)r);
    std::lock_guard<std::mutex> lk(p->mu);
    if (p->tmaps.size() > 4096) p->tmaps.clear();
    p->tmaps[key] = m;
    *out = m;
    return PAFFT_OK;
}

// Dynamic tile order (pass.cuh): a {next tile, retired CTAs} counter pair per
// (device, stream).  Launches on one stream run one after another and each
// leaves its pair zeroed, so the pair needs no host-side reset; streams run
// concurrently, so each has its own.  Launches that cannot be tied to one
// stream keep the static order: a capturing stream (the graph may replay on
// any stream, next to other graphs captured on the same one) and the
// per-thread default stream (one handle, a different stream per thread).
unsigned* tile_counters(int device, cudaStream_t st) {
    if (st == cudaStreamPerThread) return nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return nullptr;
    }
    if (st == cudaStreamLegacy) st = nullptr;
    constexpr int kSlots = 4096;
    struct Slab {
        unsigned* base = nullptr;
        int used = 0;
        std::map<cudaStream_t, int> slot;
    };
    static std::mutex mu;
    static std::map<int, Slab> slabs;
    std::lock_guard<std::mutex> lk(mu);
    Slab& sl = slabs[device];
    if (!sl.base) {
        if (cudaMalloc(&sl.base, kSlots * 2 * sizeof(unsigned)) != cudaSuccess ||
            cudaMemset(sl.base, 0, kSlots * 2 * sizeof(unsigned)) != cudaSuccess) {
            cudaGetLastError();
            sl.base = nullptr;
            return nullptr;
        }
    }
    auto it = sl.slot.find(st);
    if (it == sl.slot.end()) {
        if (sl.used == kSlots) return nullptr;
        it = sl.slot.emplace(st, sl.used++).first;
    }
    return sl.base + 2 * it->second;
}

template <typename T>
pafft_status launch_t(pafft_plan_t p, const PassDesc& d, const void* src, void* dst, size_t batch,
                      const void* ghat, const void* mul, double scale, cudaStream_t st, long long grid_cap) {
    if (((uintptr_t)src | (uintptr_t)dst) & 15u)
        return fail(PAFFT_INVALID_ARGUMENT, "device buffers must be 16-byte aligned (TMA staging)");
    PassArgs<T> a;
    memset(&a, 0, sizeof a);
    a.src = (const cplx<T>*)src;
    a.dst = (cplx<T>*)dst;
    const long long per_signal = (long long)p->total / ((long long)d.R * d.C);
    a.panels = per_signal * (long long)batch;
    a.panel_elems = (long long)d.R * d.C;
    a.C = (int)d.C;
    a.tiles_per_panel = d.contig ? 1 : (int)((d.C + d.W - 1) / d.W);
    a.nsig = (long long)batch;
    a.bps = per_signal;
    if (((long long)p->total * (long long)p->esize) % 16 != 0) {
        // fp32 signals of odd length: per-signal tile starts would break the
        // bulk copies' 16-byte alignment; walk the batch as one run instead
        a.nsig = 1;
        a.bps = a.panels;
    }
    a.tiles = d.contig ? a.nsig * ((a.bps + d.W - 1) / d.W) : a.panels * a.tiles_per_panel;
    a.ext = d.ext;
    a.sq = (unsigned)d.sq;
    a.ext_bits = d.ext_bits;
    a.ext_lo = (const cplx<T>*)d.ext_lo;
    a.ext_hi = (const cplx<T>*)d.ext_hi;
    for (int i = 0; i < 3; ++i) a.tw[i] = (const cplx<T>*)d.tw[i];
    a.ghat = (const cplx<T>*)ghat;
    a.N = (long long)p->total;
    a.mul = (const cplx<T>*)mul;
    a.scale = (T)scale;
    a.has_scale = scale != 1.0;
    if (a.tiles == 0) return PAFFT_OK;
    if (a.tiles > 0x7fffffffll || a.nsig > 0x7fffffffll)
        return fail(PAFFT_INVALID_ARGUMENT, "batch too large for one launch (%lld tiles); split the call", a.tiles);
    CUtensorMap map, map_dst;
    memset(&map, 0, sizeof map);
    memset(&map_dst, 0, sizeof map_dst);
    a.use_tmap = d.use_tmap;
    a.rb = d.rb;
    // swizzled staging needs every tile start on a box-row group boundary
    a.swz = d.swz && (per_signal % d.W == 0) &&
            (((long long)p->total * (long long)p->esize / 128) % d.swz_b1 == 0);
    a.swz_b1 = d.swz_b1;
    if (d.use_tmap) {
        ST_TRY(tensor_map(p, d, src, batch, &map));
        ST_TRY(tensor_map(p, d, dst, batch, &map_dst));
    } else if (a.swz) {
        ST_TRY(tensor_map_swz(p, d, src, batch, &map));
        ST_TRY(tensor_map_swz(p, d, dst, batch, &map_dst));
    }
    const long long grid = std::max<long long>(1, std::min<long long>(a.tiles, grid_cap > 0 ? std::min(grid_cap, d.max_ctas) : d.max_ctas));
    // Launches with several tiles per CTA and several CTAs per SM hand the tiles
    // out dynamically.  Co-resident CTAs do not share an SM evenly (measured on
    // B200, PAFFT_PASS_TRACE: with equal tile counts the three CTAs of config 2's
    // CONV pass retire at 0.71, 0.88 and 1.06 ms, config 5's strided CTAs between
    // 1.1 and 1.9 ms), so the static order leaves SMs part empty for the last
    // third of the launch; one-CTA-per-SM launches finish within 2% of each other
    // and keep the static order (dynamic: config 2's DIF +6% time).
    // PAFFT_DYN_MIN_TILES: tiles per CTA from which the order is dynamic (0 = never),
    // PAFFT_DYN_MIN_OCC: resident CTAs per SM from which it is.
    const int dyn_min = env_int("PAFFT_DYN_MIN_TILES", 4);
    if (dyn_min > 0 && a.tiles >= (long long)dyn_min * grid && d.occ >= env_int("PAFFT_DYN_MIN_OCC", 2))
        a.ctr = tile_counters(p->device, st);
    if (a.ctr) ++g_dynamic_launches;
#if PAFFT_TRACE
    // profiling build: per-CTA start/retire times and tile counts of this launch
    // (synchronous; prints one line to stderr)
    DevBuf trace;
    if (env_int("PAFFT_PASS_TRACE", 0)) {
        trace.bytes = (size_t)grid * 4 * sizeof(unsigned long long);
        CUDA_TRY(cudaMalloc(&trace.p, trace.bytes));
        CUDA_TRY(cudaMemsetAsync(trace.p, 0, trace.bytes, st));
        a.trace = (unsigned long long*)trace.p;
    }
#endif
    void* args[] = {&a, &map, &map_dst};
    CUDA_TRY(cudaLaunchKernel(d.fn, dim3((unsigned)grid), dim3(d.NT), args, d.smem, st));
    ++g_launches;
#if PAFFT_TRACE
    if (a.trace) {
        std::vector<unsigned long long> h((size_t)grid * 4);
        CUDA_TRY(cudaStreamSynchronize(st));
        CUDA_TRY(cudaMemcpy(h.data(), trace.p, trace.bytes, cudaMemcpyDeviceToHost));
        unsigned long long b0 = ~0ull, e1 = 0, tmin = ~0ull, tmax = 0;
        std::vector<unsigned long long> ends;
        double wait_frac = 0;
        for (long long i = 0; i < grid; ++i) {
            b0 = std::min(b0, h[4 * i]);
            e1 = std::max(e1, h[4 * i + 1]);
            tmin = std::min(tmin, h[4 * i + 2]);
            tmax = std::max(tmax, h[4 * i + 2]);
            ends.push_back(h[4 * i + 1]);
            wait_frac += (double)h[4 * i + 3] / (double)std::max<unsigned long long>(1, h[4 * i + 1] - h[4 * i]);
        }
        wait_frac /= (double)grid;
        std::sort(ends.begin(), ends.end());
        auto q = [&](double f) { return (double)(ends[(size_t)(f * (ends.size() - 1))] - b0) * 1e-3; };
        fprintf(stderr,
                "[pass trace] kind %d R %d grid %lld tiles %lld dyn %d: span %.1f us; CTA retire times (us after first "
                "start) min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f; tiles per CTA %llu..%llu; waiting for tile "
                "arrival %.1f%% of CTA time\n",
                d.kind, d.R, grid, a.tiles, a.ctr ? 1 : 0, (double)(e1 - b0) * 1e-3, q(0), q(0.1), q(0.5), q(0.9), q(1.0),
                tmin, tmax, 100.0 * wait_frac);
    }
#endif
    return PAFFT_OK;
}

// A strided launch takes its wide variant when that still gives at least four
// tiles per resident CTA slot (a full pipeline on every SM); batch-1 signals
// keep the 8-column tiles (config 1: 256 wide tiles for 148 slots).
bool use_wide(const PassDesc& d, const pafft_plan_s* p, size_t batch) {
    if (!d.wide) return false;
    const long long per_signal = (long long)p->total / ((long long)d.R * d.C);
    const long long tiles = per_signal * (long long)batch * ((d.C + d.wide->W - 1) / d.wide->W);
    return tiles >= 4 * d.wide->max_ctas;
}

pafft_status launch(pafft_plan_t p, const PassDesc& d0, const void* src, void* dst, size_t batch,
                    const void* ghat, const void* mul, double scale, cudaStream_t st, long long grid_cap = 0) {
    const PassDesc& d = use_wide(d0, p, batch) ? *d0.wide : d0;
    return p->prec == 0 ? launch_t<double>(p, d, src, dst, batch, ghat, mul, scale, st, grid_cap)
                        : launch_t<float>(p, d, src, dst, batch, ghat, mul, scale, st, grid_cap);
}

// ---------------------------------------------------- helper kernels --
// Out-of-place digit-reversal gather: y[i] = x[(rev_1(i_1), ..., rev_d(i_d))]
// (permute_tensor, permutation.cpp:46-90, as a pure gather; an involution).
struct PermArgs {
    int rank;
    unsigned long long dims[8];
    const uint32_t* rev[8];
};

template <typename V>
__global__ void permute_kernel(const V* __restrict__ x, V* __restrict__ y, unsigned long long total,
                               unsigned long long count, PermArgs pa) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < count;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long sig = i / total;
        unsigned long long r = i - sig * total, src = 0, w = 1;
        for (int q = 0; q < pa.rank; ++q) {
            const unsigned long long n = pa.dims[q];
            const unsigned long long iq = r % n;
            r /= n;
            src += (unsigned long long)__ldg(pa.rev[q] + iq) * w;
            w *= n;
        }
        y[i] = x[sig * total + src];
    }
}

template <typename T>
__global__ void scale_convert_kernel(const double2* __restrict__ in, cplx<T>* __restrict__ out,
                                     cplx<T>* __restrict__ out_scaled, double s, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const double2 v = in[i];
        if (out) out[i] = cplx<T>{(T)v.x, (T)v.y};
        out_scaled[i] = cplx<T>{(T)(v.x * s), (T)(v.y * s)};
    }
}

// Kernel copy of ghat, per R-block: slot sum_j d_j wt(j) (natural digit
// order of the CONV pass) holds s * ghat[b*R + sum_j rev_{F_j}(d_j) wt(j)], and
// slot g*FL + k (last-step group g, frequency k) is stored at k*(R/FL) + g.
struct SlotPerm {
    int radix, ns, R;
    int F[4], wt[4];
};

__device__ __forceinline__ int rev_rt(int d, int radix, int f) {
    int o = 0;
    for (int p = 1; p < f; p *= radix) {
        o = o * radix + d % radix;
        d /= radix;
    }
    return o;
}

template <typename T>
__global__ void kernel_ghat_kernel(const cplx<T>* __restrict__ in, cplx<T>* __restrict__ out, double s,
                                   unsigned long long n, SlotPerm sp) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long blk = i / sp.R;
        const int o = (int)(i - blk * sp.R);
        // k-major within the block: the CONV's last step reads, for each of
        // its FL frequencies k, one lane-contiguous run over the groups g
        const int G = sp.ns ? sp.R / sp.F[sp.ns - 1] : 1;
        int rem = sp.ns ? (o % G) * sp.F[sp.ns - 1] + o / G : o, src = 0;
        for (int j = 0; j < sp.ns; ++j) {
            const int d = rem / sp.wt[j];
            rem -= d * sp.wt[j];
            src += rev_rt(d, sp.radix, sp.F[j]) * sp.wt[j];
        }
        const cplx<T> v = in[blk * sp.R + src];
        out[i] = cplx<T>{(T)(v.x * s), (T)(v.y * s)};
    }
}

template <typename T>
__global__ void scale_kernel(const cplx<T>* __restrict__ in, cplx<T>* __restrict__ out, double s,
                             unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const cplx<T> v = in[i];
        out[i] = cplx<T>{(T)(v.x * s), (T)(v.y * s)};
    }
}

// y[i] = x[i] * g[i mod N]  (hadamard_inplace, convolution.cpp:23-35), used only
// when the plan has no stages at all (every extent 1).
template <typename T>
__global__ void hadamard_kernel(const cplx<T>* __restrict__ x, const cplx<T>* __restrict__ g, cplx<T>* __restrict__ y,
                                unsigned long long N, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        y[i] = cmul(x[i], g[i % N]);
}

unsigned grid_for(unsigned long long n, int threads) {
    const unsigned long long b = (n + threads - 1) / threads;
    return (unsigned)std::min<unsigned long long>(std::max<unsigned long long>(b, 1), 148ull * 32);
}

// Tiled digit reversal (the explicit P of the standard-order comparator and
// of prepare_filter; permute_tensor, permutation.cpp:46-90).  Axis-0 index
// j = A r^(t0-d) + B r^d + Cc reverses to rev(Cc) r^(t0-d) + rev(B) r^d + rev(A),
// so the output block of fixed (row, B) -- TD x TD elements, TD = r^d -- comes
// from the source block of middle rev(B): read as rows a' (contiguous runs of
// TD), written as rows A (contiguous runs over Cc), transposed through padded
// shared memory.  Higher axes only relocate whole axis-0 rows.
struct TPermArgs {
    int rank, radix, d, t0;
    unsigned long long n0, rows, mids, total;
    unsigned long long dims[8];
    const uint32_t* rev[8];
};

__device__ __forceinline__ int rev_digits(int v, int radix, int ndig) {
    int o = 0;
    for (int i = 0; i < ndig; ++i) {
        o = o * radix + v % radix;
        v /= radix;
    }
    return o;
}

template <typename V, int RADIX, int D>
__global__ void __launch_bounds__(256) permute_tiled_kernel(const V* __restrict__ x, V* __restrict__ y,
                                                            unsigned long long batch, TPermArgs pa) {
    constexpr int TD = RADIX == 2 ? (1 << D) : (RADIX == 3 ? 27 : (RADIX == 4 ? 16 : (RADIX == 5 ? 25 : 8)));
    constexpr int TP = TD + 1;
    __shared__ V sm[TD * TP];
    __shared__ int rv[TD];
    if (threadIdx.x < TD) rv[threadIdx.x] = revd<RADIX, TD>(threadIdx.x);
    __syncthreads();
    const unsigned long long hs = pa.n0 / (unsigned long long)TD;  // r^(t0-d)
    const unsigned long long units = batch * pa.rows * pa.mids;
    for (unsigned long long u = blockIdx.x; u < units; u += gridDim.x) {
        const unsigned long long B = u % pa.mids;
        const unsigned long long rowg = u / pa.mids;
        const unsigned long long sig = rowg / pa.rows;
        const unsigned long long row = rowg - sig * pa.rows;
        unsigned long long srow = 0, w = 1, r = row;
        for (int q = 1; q < pa.rank; ++q) {
            const unsigned long long n = pa.dims[q];
            const unsigned long long iq = r % n;
            r /= n;
            srow += (unsigned long long)__ldg(pa.rev[q] + iq) * w;
            w *= n;
        }
        unsigned long long rB = 0, v = B;
        for (int i = 0; i < pa.t0 - 2 * D; ++i) {
            rB = rB * RADIX + v % RADIX;
            v /= RADIX;
        }
        const V* src = x + sig * pa.total + srow * pa.n0 + rB * TD;
        V* dst = y + sig * pa.total + row * pa.n0 + B * TD;
#pragma unroll 4
        for (int e = threadIdx.x; e < TD * TD; e += 256) {
            const int ap = e / TD, cp = e - ap * TD;
            sm[ap * TP + cp] = src[(unsigned long long)ap * hs + cp];
        }
        __syncthreads();
#pragma unroll 4
        for (int e = threadIdx.x; e < TD * TD; e += 256) {
            const int A = e / TD, Cc = e - A * TD;
            dst[(unsigned long long)A * hs + Cc] = sm[rv[Cc] * TP + rv[A]];
        }
        __syncthreads();
    }
}

template <typename V>
void launch_permute_tiled(int radix, unsigned grid, cudaStream_t st, const V* x, V* y, unsigned long long batch,
                          const TPermArgs& ta) {
    switch (radix) {
        case 2: permute_tiled_kernel<V, 2, 5><<<grid, 256, 0, st>>>(x, y, batch, ta); break;
        case 3: permute_tiled_kernel<V, 3, 3><<<grid, 256, 0, st>>>(x, y, batch, ta); break;
        case 4: permute_tiled_kernel<V, 4, 2><<<grid, 256, 0, st>>>(x, y, batch, ta); break;
        case 5: permute_tiled_kernel<V, 5, 2><<<grid, 256, 0, st>>>(x, y, batch, ta); break;
        default: permute_tiled_kernel<V, 8, 1><<<grid, 256, 0, st>>>(x, y, batch, ta); break;
    }
}

pafft_status permute_dev(pafft_plan_t p, const void* x, void* y, size_t batch, cudaStream_t st) {
    {
        // tiled path when axis 0 has at least 2d digits
        const int r = (int)p->radix;
        const int d = r == 2 ? 5 : r == 3 ? 3 : r == 4 ? 2 : r == 5 ? 2 : 1;
        const int t0 = (int)p->depth[0];
        // (radix 4/8: the L2-cached gather measured faster than 16/8-wide tiles)
        if (t0 >= 2 * d && r != 4 && r != 8 && env_int("PAFFT_NAIVE_PERMUTE", 0) == 0) {
            TPermArgs ta;
            memset(&ta, 0, sizeof ta);
            ta.rank = p->rank;
            ta.radix = r;
            ta.d = d;
            ta.t0 = t0;
            ta.n0 = p->dims[0];
            ta.total = p->total;
            ta.rows = p->total / p->dims[0];
            ta.mids = (unsigned long long)ipow(r, t0 - 2 * d);
            for (int q = 0; q < p->rank; ++q) {
                ta.dims[q] = p->dims[q];
                ta.rev[q] = p->rev_dev[q];
            }
            const unsigned long long units = (unsigned long long)batch * ta.rows * ta.mids;
            const unsigned grid = (unsigned)std::min<unsigned long long>(units, 148ull * 16);
            if (p->prec == 0)
                launch_permute_tiled<double2>(r, grid, st, (const double2*)x, (double2*)y, batch, ta);
            else
                launch_permute_tiled<float2>(r, grid, st, (const float2*)x, (float2*)y, batch, ta);
            CUDA_TRY(cudaGetLastError());
            ++g_launches;
            g_perm_passes += batch;
            return PAFFT_OK;
        }
    }
    PermArgs pa;
    memset(&pa, 0, sizeof pa);
    pa.rank = p->rank;
    for (int q = 0; q < p->rank; ++q) {
        pa.dims[q] = p->dims[q];
        pa.rev[q] = p->rev_dev[q];
    }
    const unsigned long long count = (unsigned long long)p->total * batch;
    if (count == 0) return PAFFT_OK;
    if (p->prec == 0)
        permute_kernel<double2><<<grid_for(count, 256), 256, 0, st>>>((const double2*)x, (double2*)y, p->total,
                                                                      count, pa);
    else
        permute_kernel<float2><<<grid_for(count, 256), 256, 0, st>>>((const float2*)x, (float2*)y, p->total,
                                                                     count, pa);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    g_perm_passes += batch;
    return PAFFT_OK;
}

pafft_status hadamard_dev(pafft_plan_t p, const void* x, const void* g, void* y, size_t batch, cudaStream_t st) {
    const unsigned long long n = (unsigned long long)p->total * batch;
    if (p->prec == 0)
        hadamard_kernel<double><<<grid_for(n, 256), 256, 0, st>>>((const double2*)x, (const double2*)g, (double2*)y,
                                                                  p->total, n);
    else
        hadamard_kernel<float><<<grid_for(n, 256), 256, 0, st>>>((const float2*)x, (const float2*)g, (float2*)y,
                                                                 p->total, n);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    return PAFFT_OK;
}

pafft_status async_alloc(pafft_plan_t p, AsyncBuf& b, size_t bytes, cudaStream_t st) {
    static std::once_flag once[64];
    if (p->device >= 0 && p->device < 64)
        std::call_once(once[p->device], [&] {
            // keep freed blocks in the device pool (no OS round trip per call)
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, p->device) == cudaSuccess) {
                uint64_t thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        });
    b.st = st;
    CUDA_TRY(cudaMallocAsync(&b.p, bytes ? bytes : 16, st));
    return PAFFT_OK;
}

pafft_status ensure(std::unique_ptr<DevBuf>& b, size_t bytes) {
    if (b && b->bytes >= bytes) return PAFFT_OK;
    b.reset();
    auto nb = std::make_unique<DevBuf>();
    CUDA_TRY(cudaMalloc(&nb->p, bytes ? bytes : 16));
    nb->bytes = bytes;
    b = std::move(nb);
    return PAFFT_OK;
}

// Pass kernels stage tiles with TMA, which needs 16-byte aligned global
// addresses: fp64 element pointers always are; fp32 views may sit 8 bytes off.
bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; }
#define ALIGN_TRY(ptr)                                                                                       \
    do {                                                                                                     \
        if (!aligned16(ptr))                                                                                 \
            return fail(PAFFT_INVALID_ARGUMENT, "device buffer %s=%p is not 16-byte aligned (TMA staging)", \
                        #ptr, (const void*)(ptr));                                                           \
    } while (0)

pafft_status set_device(pafft_plan_t p) {
    CUDA_TRY(cudaSetDevice(p->device));
    return PAFFT_OK;
}

bool key_match(pafft_filter_t f, pafft_plan_t p) {
    if (f->radix != p->radix || f->rank != p->rank || f->prec != p->prec || f->device != p->device) return false;
    for (int q = 0; q < p->rank; ++q)
        if (f->radices[q] != p->radices[q]) return false;
    for (int q = 0; q < p->rank; ++q)
        if (f->dims[q] != p->dims[q]) return false;
    for (int i = 0; i < 6; ++i)
        if (f->layout[i] != p->layout[i]) return false;
    return true;
}

// Pass sequences (built on demand from the stage groups).
pafft_status passes_permfree(pafft_plan_t p, std::vector<PassDesc>& out) {
    out.clear();
    const size_t ng = p->groups.size();
    if (ng == 0) return PAFFT_OK;
    for (size_t i = 0; i + 1 < ng; ++i) {
        PassDesc d;
        ST_TRY(make_pass(p, p->groups[i], KIND_DIF, d));
        out.push_back(d);
    }
    {
        PassDesc d;
        ST_TRY(make_pass(p, p->groups[ng - 1], KIND_CONV, d));
        out.push_back(d);
    }
    for (size_t i = ng - 1; i-- > 0;) {
        PassDesc d;
        ST_TRY(make_pass(p, p->groups[i], KIND_DIT_CONJ, d));
        out.push_back(d);
    }
    return PAFFT_OK;
}

// Ladders over every mode in the reference's mode order (butterfly_tensor,
// butterfly.cpp:423-466: mode 0 first, ascending), so a tensor ladder is
// bitwise the 1-D ladder applied line by line (test_butterfly.cpp:198-215).
// A (DIT_FWD) / A-bar (DIT_CONJ): reverse group order (axis 0 first, its
// stage groups descending).  A^T (DIF): axes ascending, each axis's stage
// groups ascending (the permutation-free schedule keeps its own order: there
// axis 0's contiguous group must come last to merge with the filter).
pafft_status passes_ladder(pafft_plan_t p, int kind, std::vector<PassDesc>& out) {
    out.clear();
    std::vector<Group> order(p->groups.begin(), p->groups.end());
    if (kind == KIND_DIF)
        std::stable_sort(order.begin(), order.end(), [](const Group& x, const Group& y) { return x.axis < y.axis; });
    else
        std::reverse(order.begin(), order.end());
    for (const Group& g : order) {
        PassDesc d;
        ST_TRY(make_pass(p, g, kind, d));
        out.push_back(d);
    }
    return PAFFT_OK;
}

// Runs a ladder (list of passes) src -> dst; the first pass reads src, the
// rest run in place on dst.  Epilogue (mul / scale) on the last pass.
pafft_status run_ladder(pafft_plan_t p, const std::vector<PassDesc>& ps, const void* src, void* dst, size_t batch,
                        const void* mul, double scale, cudaStream_t st) {
    if (ps.empty()) {
        // n == 1 everywhere: identity transform (plus epilogue)
        if (src != dst)
            CUDA_TRY(cudaMemcpyAsync(dst, src, p->total * batch * p->esize, cudaMemcpyDeviceToDevice, st));
        if (scale != 1.0 || mul) return fail(PAFFT_INVALID_ARGUMENT, "epilogue on an empty ladder");
        return PAFFT_OK;
    }
    for (size_t i = 0; i < ps.size(); ++i) {
        const bool last = i + 1 == ps.size();
        ST_TRY(launch(p, ps[i], i == 0 ? src : dst, dst, batch, nullptr, last ? mul : nullptr, last ? scale : 1.0,
                      st));
    }
    return PAFFT_OK;
}

}  // namespace

// ===================================================================== ABI
// ------------------------------------------------ split (drop-in) I/O
// The reference API holds a signal as split host arrays (ComplexBuffer re/im,
// core.hpp:48-63).  The synchronous split entry points copy re and im as two
// plain host->device copies into stream-ordered pool scratch and (de)interleave
// on the device (converting to fp32 for fp32 plans), on a thread-local stream
// per device: no cudaMalloc, no stream creation and no host interleave loop per
// call, and calls from distinct threads run concurrently.
template <typename T>
__global__ void split_to_cplx_kernel(const double* __restrict__ re, const double* __restrict__ im,
                                     cplx<T>* __restrict__ out, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        out[i] = cplx<T>{(T)re[i], (T)im[i]};
}
template <typename T>
__global__ void cplx_to_split_kernel(const cplx<T>* __restrict__ in, double* __restrict__ re,
                                     double* __restrict__ im, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const cplx<T> v = in[i];
        re[i] = (double)v.x;
        im[i] = (double)v.y;
    }
}

static pafft_status call_stream(int device, cudaStream_t* out) {
    thread_local std::vector<cudaStream_t> streams;  // never destroyed: live for the thread
    if ((int)streams.size() <= device) streams.resize(device + 1, nullptr);
    if (!streams[device]) CUDA_TRY(cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking));
    *out = streams[device];
    return PAFFT_OK;
}

template <typename T>
static pafft_status upload_split_as(pafft_plan_t p, const double* re, const double* im, size_t n, cplx<T>* dev,
                                    cudaStream_t st) {
    AsyncBuf sc;
    ST_TRY(async_alloc(p, sc, 2 * n * sizeof(double), st));
    double* dre = (double*)sc.p;
    double* dim = dre + n;
    CUDA_TRY(cudaMemcpyAsync(dre, re, n * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dim, im, n * sizeof(double), cudaMemcpyHostToDevice, st));
    split_to_cplx_kernel<T><<<grid_for(n, 256), 256, 0, st>>>(dre, dim, dev, n);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    return PAFFT_OK;
}
template <typename T>
static pafft_status download_split_as(pafft_plan_t p, const cplx<T>* dev, size_t n, double* re, double* im,
                                      cudaStream_t st) {
    AsyncBuf sc;
    ST_TRY(async_alloc(p, sc, 2 * n * sizeof(double), st));
    double* dre = (double*)sc.p;
    double* dim = dre + n;
    cplx_to_split_kernel<T><<<grid_for(n, 256), 256, 0, st>>>(dev, dre, dim, n);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    CUDA_TRY(cudaMemcpyAsync(re, dre, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(im, dim, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return PAFFT_OK;
}
// plan precision
static pafft_status upload_split(pafft_plan_t p, const double* re, const double* im, size_t n, void* dev,
                                 cudaStream_t st) {
    return p->prec == 0 ? upload_split_as<double>(p, re, im, n, (double2*)dev, st)
                        : upload_split_as<float>(p, re, im, n, (float2*)dev, st);
}
static pafft_status download_split(pafft_plan_t p, const void* dev, size_t n, double* re, double* im,
                                   cudaStream_t st) {
    return p->prec == 0 ? download_split_as<double>(p, (const double2*)dev, n, re, im, st)
                        : download_split_as<float>(p, (const float2*)dev, n, re, im, st);
}

extern "C" {

const char* pafft_last_error(void) { return g_err.c_str(); }

void pafft_last_error_dim(size_t* dim, size_t* extent) {
    if (dim) *dim = g_err_dim;
    if (extent) *extent = g_err_extent;
}

const char* pafft_build_info(void) {
    return "pafft_b200 sm_100a (" __DATE__ " " __TIME__ ")";
}

uint64_t pafft_permutation_pass_count(void) { return g_perm_passes; }
void pafft_reset_permutation_pass_count(void) { g_perm_passes = 0; }
uint64_t pafft_kernel_launch_count(void) { return g_launches; }
uint64_t pafft_dynamic_launch_count(void) { return g_dynamic_launches; }

pafft_status pafft_digit_reverse(uint64_t j, unsigned radix, unsigned digits, uint64_t* out) {
    uint64_t bound = 1;
    for (unsigned s = 0; s < digits; ++s) bound *= radix;
    if (j >= bound)
        return fail(PAFFT_INDEX_OUT_OF_RANGE, "index %llu outside [0, %llu)", (unsigned long long)j,
                    (unsigned long long)bound);
    uint64_t o = 0;
    for (unsigned s = 0; s < digits; ++s) {
        o = o * radix + j % radix;
        j /= radix;
    }
    *out = o;
    return PAFFT_OK;
}

pafft_status pafft_plan_create(unsigned radix, const size_t* dims, int rank, int precision, int device,
                               pafft_plan_t* out) {
    if (!out) return fail(PAFFT_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    if (!radix_ok(radix))
        return fail(PAFFT_INVALID_ARGUMENT, "radix must be 2, 3, 4, 5, or 8 (got %u)", radix);
    if (rank <= 0) return fail(PAFFT_EMPTY_SHAPE, "shape has no dimensions");
    if (rank > 8) return fail(PAFFT_INVALID_ARGUMENT, "rank %d exceeds 8", rank);
    unsigned radices[8];
    for (int q = 0; q < 8; ++q) radices[q] = radix;
    return pafft_plan_create_mixed(radices, dims, rank, precision, device, out);
}

pafft_status pafft_plan_create_mixed(const unsigned* radices, const size_t* dims, int rank, int precision,
                                     int device, pafft_plan_t* out) {
    if (!out) return fail(PAFFT_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    if (rank <= 0) return fail(PAFFT_EMPTY_SHAPE, "shape has no dimensions");
    if (rank > 8) return fail(PAFFT_INVALID_ARGUMENT, "rank %d exceeds 8", rank);
    if (!radices || !dims) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    for (int q = 0; q < rank; ++q)
        if (!radix_ok(radices[q]))
            return fail(PAFFT_INVALID_ARGUMENT, "radix must be 2, 3, 4, 5, or 8 (got %u on axis %d)", radices[q], q);
    if (precision != PAFFT_F64 && precision != PAFFT_F32)
        return fail(PAFFT_INVALID_ARGUMENT, "unknown precision %d", precision);
    for (int q = 0; q < rank; ++q) {
        const unsigned radix = radices[q];
        size_t n = dims[q];
        bool pow = n != 0;
        while (pow && n % radix == 0) n /= radix;
        pow = pow && n == 1;
        if (!pow) {
            g_err_dim = (size_t)q;
            g_err_extent = dims[q];
            return fail(PAFFT_NOT_A_POWER_OF_RADIX, "dimension %d has extent %zu, not a power of radix %u", q,
                        dims[q], radix);
        }
        if (dims[q] > 0xffffffffull) return fail(PAFFT_INVALID_ARGUMENT, "dimension extent exceeds 32-bit range");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(PAFFT_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    }
    if (device < 0) CUDA_TRY(cudaGetDevice(&device));
    CUDA_TRY(cudaSetDevice(device));
    auto p = std::make_unique<pafft_plan_s>();
    p->radix = radices[0];
    for (int q = 0; q < rank; ++q) p->radices[q] = radices[q];
    p->rank = rank;
    p->prec = precision;
    p->device = device;
    p->esize = precision == PAFFT_F64 ? 16 : 8;
    p->total = 1;
    for (int q = 0; q < rank; ++q) {
        p->dims[q] = dims[q];
        p->total *= dims[q];
        unsigned t = 0;
        for (size_t n = dims[q]; n > 1; n /= radices[q]) ++t;
        p->depth[q] = t;
    }
    build_groups(p.get());
    // all pass schedules now, so missing kernels surface at plan time
    ST_TRY(passes_permfree(p.get(), p->pf));
    if (!p->pf.empty()) {
        const PassDesc& cv = p->pf[p->pf.size() / 2];  // the CONV pass
        const long long lay[6] = {cv.axis, cv.R, cv.F[0], cv.F[1], cv.F[2], cv.F[3]};
        for (int i = 0; i < 6; ++i) p->layout[i] = lay[i];
    }
    ST_TRY(passes_ladder(p.get(), KIND_DIF, p->dif));
    ST_TRY(passes_ladder(p.get(), KIND_DIT_FWD, p->dit_fwd));
    ST_TRY(passes_ladder(p.get(), KIND_DIT_CONJ, p->dit_conj));
    for (int q = 0; q < rank; ++q) {
        const unsigned radix = radices[q];
        std::vector<uint32_t> rev(dims[q]);
        for (size_t j = 0; j < dims[q]; ++j) {
            size_t v = j, o = 0;
            for (unsigned s = 0; s < p->depth[q]; ++s) {
                o = o * radix + v % radix;
                v /= radix;
            }
            rev[j] = (uint32_t)o;
        }
        void* d;
        ST_TRY(alloc(p.get(), rev.size() * 4, &d));
        CUDA_TRY(cudaMemcpy(d, rev.data(), rev.size() * 4, cudaMemcpyHostToDevice));
        p->rev_dev.push_back((uint32_t*)d);
    }
    for (auto& s : p->streams) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    // table uploads above used pageable cudaMemcpy; make them visible to
    // every stream (including non-blocking ones) before the plan is used
    CUDA_TRY(cudaDeviceSynchronize());
    *out = p.release();
    return PAFFT_OK;
}

pafft_status pafft_plan_destroy(pafft_plan_t plan) {
    if (!plan) return PAFFT_OK;
    cudaSetDevice(plan->device);
    for (auto& s : plan->streams)
        if (s) cudaStreamDestroy(s);
    delete plan;
    return PAFFT_OK;
}

pafft_status pafft_plan_radices(pafft_plan_t p, unsigned* radices) {
    if (!p || !radices) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    for (int q = 0; q < p->rank; ++q) radices[q] = p->radices[q];
    return PAFFT_OK;
}

pafft_status pafft_plan_info(pafft_plan_t p, unsigned* radix, int* rank, size_t* dims, unsigned* depths,
                             size_t* total, int* precision, int* device) {
    if (!p) return fail(PAFFT_INVALID_ARGUMENT, "null plan");
    if (radix) *radix = p->radix;
    if (rank) *rank = p->rank;
    for (int q = 0; q < p->rank; ++q) {
        if (dims) dims[q] = p->dims[q];
        if (depths) depths[q] = p->depth[q];
    }
    if (total) *total = p->total;
    if (precision) *precision = p->prec;
    if (device) *device = p->device;
    return PAFFT_OK;
}

pafft_status pafft_plan_num_passes(pafft_plan_t p, int* n) {
    *n = p->pf.empty() ? 1 : (int)p->pf.size();
    return PAFFT_OK;
}

pafft_status pafft_plan_describe(pafft_plan_t p, char* buf, size_t len) {
    const std::vector<PassDesc>& ps = p->pf;
    std::string s;
    const char* kn[] = {"DIF", "DIT_FWD", "DIT_CONJ", "CONV"};
    for (const auto& d : ps) {
        char line[256];
        snprintf(line, sizeof line,
                 "%s axis=%d stages=[%d,%d) R=%d(%dx%dx%dx%d) K0=%lld L=%lld C=%lld %s W=%d NT=%d smem=%zu ext=%d\n",
                 kn[d.kind], d.axis, d.a, d.a + d.s, d.R, d.F[0], d.F[1], d.F[2], d.F[3], d.K0, d.L, d.C,
                 d.contig ? "contig" : "strided", d.W, d.NT, d.smem, d.ext);
        s += line;
        if (d.wide) {
            snprintf(line, sizeof line, "  (many tiles: W=%d NT=%d smem=%zu)\n", d.wide->W, d.wide->NT, d.wide->smem);
            s += line;
        }
    }
    if (buf && len) {
        strncpy(buf, s.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return PAFFT_OK;
}

// --------------------------------------------------------------- filters
static pafft_status new_filter(pafft_plan_t p, pafft_filter_t* out) {
    auto f = std::make_unique<pafft_filter_s>();
    f->plan = p;
    f->radix = p->radix;
    for (int q = 0; q < p->rank; ++q) f->radices[q] = p->radices[q];
    f->rank = p->rank;
    for (int q = 0; q < p->rank; ++q) f->dims[q] = p->dims[q];
    f->prec = p->prec;
    f->device = p->device;
    for (int i = 0; i < 6; ++i) f->layout[i] = p->layout[i];
    for (std::shared_ptr<DevBuf>* b : {&f->ghat, &f->ghat_scaled}) {
        auto nb = std::make_shared<DevBuf>();
        CUDA_TRY(cudaMalloc(&nb->p, p->total * p->esize ? p->total * p->esize : 16));
        nb->bytes = p->total * p->esize;
        *b = std::move(nb);
    }
    *out = f.release();
    return PAFFT_OK;
}

pafft_status pafft_filter_create_empty(pafft_plan_t p, pafft_filter_t* out) {
    if (!p || !out) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ST_TRY(set_device(p));
    return new_filter(p, out);
}

pafft_status pafft_filter_sync_scaled(pafft_filter_t f, void* stream) {
    pafft_plan_t p = f->plan;
    ST_TRY(set_device(p));
    cudaStream_t st = (cudaStream_t)stream;
    const double s = 1.0 / (double)p->total;
    SlotPerm sp;
    memset(&sp, 0, sizeof sp);
    sp.radix = (int)p->radix;
    sp.R = 1;
    sp.ns = 0;
    if (!p->pf.empty()) {
        const PassDesc& cv = p->pf[p->pf.size() / 2];  // the CONV pass
        // the CONV pass's own axis radix: it is axis 0's only when axis 0 has
        // extent > 1 (with leading extent-1 axes it is the first longer axis)
        sp.radix = (int)p->radices[cv.axis];
        sp.R = cv.R;
        sp.ns = cv.nsteps;
        int w = 1;
        for (int j = cv.nsteps - 1; j >= 0; --j) {
            sp.F[j] = cv.F[j];
            sp.wt[j] = w;
            w *= cv.F[j];
        }
    }
    if (p->prec == 0)
        kernel_ghat_kernel<double><<<grid_for(p->total, 256), 256, 0, st>>>(
            (const double2*)f->ghat->p, (double2*)f->ghat_scaled->p, s, p->total, sp);
    else
        kernel_ghat_kernel<float><<<grid_for(p->total, 256), 256, 0, st>>>(
            (const float2*)f->ghat->p, (float2*)f->ghat_scaled->p, s, p->total, sp);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    return PAFFT_OK;
}

pafft_status pafft_prepare_filter_device(pafft_plan_t p, const void* g_dev, void* stream, pafft_filter_t* out) {
    if (!p || !out || !g_dev) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ST_TRY(set_device(p));
    pafft_filter_t f;
    ST_TRY(new_filter(p, &f));
    std::unique_ptr<pafft_filter_s> guard(f);
    cudaStream_t st = (cudaStream_t)stream;
    ST_TRY(permute_dev(p, g_dev, f->ghat->p, 1, st));  // the one offline reordering pass
    ST_TRY(pafft_filter_sync_scaled(f, stream));
    CUDA_TRY(cudaStreamSynchronize(st));
    *out = guard.release();
    return PAFFT_OK;
}

pafft_status pafft_prepare_filter_split(pafft_plan_t p, const double* g_re, const double* g_im,
                                        pafft_filter_t* out) {
    if (!p || !out || !g_re || !g_im) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ST_TRY(set_device(p));
    cudaStream_t st;
    ST_TRY(call_stream(p->device, &st));
    const size_t n = p->total;
    // the observable ghat stays bit-exact: permute in double, convert after
    AsyncBuf g64, gh64;
    ST_TRY(async_alloc(p, g64, n * 16, st));
    ST_TRY(async_alloc(p, gh64, n * 16, st));
    ST_TRY(upload_split_as<double>(p, g_re, g_im, n, (double2*)g64.p, st));
    pafft_filter_t f;
    ST_TRY(new_filter(p, &f));
    std::unique_ptr<pafft_filter_s> guard(f);
    {
        PermArgs pa;
        memset(&pa, 0, sizeof pa);
        pa.rank = p->rank;
        for (int q = 0; q < p->rank; ++q) {
            pa.dims[q] = p->dims[q];
            pa.rev[q] = p->rev_dev[q];
        }
        permute_kernel<double2><<<grid_for(n, 256), 256, 0, st>>>((const double2*)g64.p, (double2*)gh64.p, n, n, pa);
        CUDA_TRY(cudaGetLastError());
        ++g_launches;
        ++g_perm_passes;  // the one offline reordering pass (convolution.cpp:9-14)
    }
    if (p->prec == 0)
        CUDA_TRY(cudaMemcpyAsync(f->ghat->p, gh64.p, n * 16, cudaMemcpyDeviceToDevice, st));
    else {
        scale_convert_kernel<float><<<grid_for(n, 256), 256, 0, st>>>((const double2*)gh64.p, (float2*)f->ghat->p,
                                                                      (float2*)f->ghat_scaled->p, 1.0, n);
        CUDA_TRY(cudaGetLastError());
        ++g_launches;
    }
    ST_TRY(pafft_filter_sync_scaled(f, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    *out = guard.release();
    return PAFFT_OK;
}

pafft_status pafft_filter_from_prepared_split(pafft_plan_t p, const double* ghat_re, const double* ghat_im,
                                              pafft_filter_t* out) {
    if (!p || !out || !ghat_re || !ghat_im) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ST_TRY(set_device(p));
    cudaStream_t st;
    ST_TRY(call_stream(p->device, &st));
    pafft_filter_t f;
    ST_TRY(new_filter(p, &f));
    std::unique_ptr<pafft_filter_s> guard(f);
    // already digit-reversed: no reordering pass
    ST_TRY(upload_split(p, ghat_re, ghat_im, p->total, f->ghat->p, st));
    ST_TRY(pafft_filter_sync_scaled(f, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    *out = guard.release();
    return PAFFT_OK;
}

pafft_status pafft_prepare_filter_from_impulse_device(pafft_plan_t p, const void* h_dev, void* stream,
                                                      pafft_filter_t* out) {
    if (!p || !out || !h_dev) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ALIGN_TRY(h_dev);
    ST_TRY(set_device(p));
    pafft_filter_t f;
    ST_TRY(new_filter(p, &f));
    std::unique_ptr<pafft_filter_s> guard(f);
    cudaStream_t st = (cudaStream_t)stream;
    ST_TRY(run_ladder(p, p->dif, h_dev, f->ghat->p, 1, nullptr, 1.0, st));  // ghat = A^T h, no permutation
    ST_TRY(pafft_filter_sync_scaled(f, stream));
    CUDA_TRY(cudaStreamSynchronize(st));
    *out = guard.release();
    return PAFFT_OK;
}

// ------------------------------------------------- multi-GPU filter --
// NCCL is resolved at first use with dlopen("libnccl.so.2"): inside a process
// that already loaded NCCL (torch.distributed) the loader returns that copy,
// so the library never brings a second NCCL into the process.
namespace {
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            a.why = std::string("cannot load NCCL: ") + (e ? e : "libnccl.so.2 not found");
            return a;
        }
        a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
        a.comm_init_all = (decltype(a.comm_init_all))dlsym(h, "ncclCommInitAll");
        a.comm_user_rank = (decltype(a.comm_user_rank))dlsym(h, "ncclCommUserRank");
        a.broadcast = (decltype(a.broadcast))dlsym(h, "ncclBroadcast");
        a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
        a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
        a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
        a.ok = a.comm_init_all && a.comm_user_rank && a.broadcast && a.group_start && a.group_end && a.error_string;
        if (!a.ok) a.why = "libnccl.so.2 lacks the collective entry points";
        return a;
    }();
    return api;
}

#define NCCL_TRY(x)                                                                                   \
    do {                                                                                              \
        const ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) return fail(PAFFT_NCCL_ERROR, "%s: %s", #x, nccl().error_string(r_)); \
    } while (0)

// communicator cliques the library created for single-process broadcasts,
// keyed by the device list (kept for the life of the process)
std::mutex g_clique_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_cliques;
}  // namespace

pafft_status pafft_filter_broadcast(pafft_filter_t* filters, int ndev, int root, void* const* comms,
                                    void* const* streams) {
    if (!filters || ndev < 1) return fail(PAFFT_INVALID_ARGUMENT, "need at least one filter");
    for (int i = 0; i < ndev; ++i) {
        if (!filters[i]) return fail(PAFFT_INVALID_ARGUMENT, "null filter %d", i);
        const pafft_filter_s& a = *filters[i];
        const pafft_filter_s& b = *filters[0];
        bool same = a.radix == b.radix && a.rank == b.rank && a.prec == b.prec;
        for (int q = 0; same && q < a.rank; ++q) same = a.dims[q] == b.dims[q] && a.radices[q] == b.radices[q];
        for (int k = 0; same && k < 6; ++k) same = a.layout[k] == b.layout[k];
        if (!same) return fail(PAFFT_FILTER_PLAN_MISMATCH, "filter %d does not match filter 0's plan key", i);
        for (int j = 0; j < i; ++j)
            if (filters[j]->device == a.device)
                return fail(PAFFT_INVALID_ARGUMENT, "filters %d and %d share device %d", j, i, a.device);
    }
    const NcclApi& api = nccl();
    if (!api.ok) return fail(PAFFT_NCCL_ERROR, "%s", api.why.c_str());
    std::vector<ncclComm_t> cs(ndev);
    if (comms) {
        for (int i = 0; i < ndev; ++i) cs[i] = (ncclComm_t)comms[i];
    } else {
        if (root < 0 || root >= ndev) return fail(PAFFT_INVALID_ARGUMENT, "root %d out of range", root);
        std::vector<int> devs(ndev);
        for (int i = 0; i < ndev; ++i) devs[i] = filters[i]->device;
        std::lock_guard<std::mutex> lk(g_clique_mu);
        auto it = g_cliques.find(devs);
        if (it == g_cliques.end()) {
            std::vector<ncclComm_t> fresh(ndev);
            NCCL_TRY(api.comm_init_all(fresh.data(), ndev, devs.data()));
            it = g_cliques.emplace(devs, fresh).first;
        }
        cs = it->second;
    }
    const size_t count = filters[0]->plan->total * 2;  // reals
    const ncclDataType_t dt = filters[0]->prec == 0 ? ncclFloat64 : ncclFloat32;
    std::vector<int> is_root(ndev);
    for (int i = 0; i < ndev; ++i) {
        int r = 0;
        NCCL_TRY(api.comm_user_rank(cs[i], &r));
        is_root[i] = r == root;
    }
    // the unscaled ghat travels; receivers rebuild their kernel copy locally
    NCCL_TRY(api.group_start());
    for (int i = 0; i < ndev; ++i) {
        CUDA_TRY(cudaSetDevice(filters[i]->device));
        void* buf = filters[i]->ghat->p;
        const ncclResult_t r =
            api.broadcast(buf, buf, count, dt, root, cs[i], streams ? (cudaStream_t)streams[i] : (cudaStream_t)0);
        if (r != ncclSuccess) {
            api.group_end();
            return fail(PAFFT_NCCL_ERROR, "ncclBroadcast: %s", api.error_string(r));
        }
    }
    NCCL_TRY(api.group_end());
    for (int i = 0; i < ndev; ++i)
        if (!is_root[i]) ST_TRY(pafft_filter_sync_scaled(filters[i], streams ? streams[i] : nullptr));
    return PAFFT_OK;
}

// ------------------------------------------ filter-spectrum cache --
// Prepared spectra keyed by (plan key, 128-bit content hash of the impulse),
// shared across plans with the same key.  Entries are
// weak: a spectrum lives as long as some filter handle uses it.
namespace {
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// order-dependent sums of two independent word mixes (commutative reductions)
__global__ void content_hash_kernel(const unsigned long long* __restrict__ w, unsigned long long n,
                                    unsigned long long* out) {
    unsigned long long h1 = 0, h2 = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long v = w[i];
        h1 += mix64(v + 0x9e3779b97f4a7c15ULL * (i + 1));
        h2 += mix64((v ^ 0xd6e8feb86659fd93ULL) + 0xc2b2ae3d27d4eb4fULL * (i + 7)) | 1ull;
    }
    for (int o = 16; o > 0; o >>= 1) {
        h1 += __shfl_xor_sync(0xffffffffu, h1, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, h1);
        atomicAdd(out + 1, h2);
    }
}

struct CacheKey {
    std::vector<unsigned> radices;
    std::vector<size_t> dims;
    int prec, device;
    std::vector<long long> layout;  // the kernel copy's slot layout (plan's CONV pass)
    unsigned long long h1, h2;
    bool operator<(const CacheKey& o) const {
        return std::tie(radices, dims, prec, device, layout, h1, h2) <
               std::tie(o.radices, o.dims, o.prec, o.device, o.layout, o.h1, o.h2);
    }
};
struct CacheEntry {
    std::weak_ptr<DevBuf> ghat, ghat_scaled;
};
std::mutex g_cache_mu;
std::map<CacheKey, CacheEntry> g_cache;
std::atomic<unsigned long long> g_cache_hits{0}, g_cache_misses{0};
}  // namespace

pafft_status pafft_prepare_filter_from_impulse_cached(pafft_plan_t p, const void* h_dev, void* stream,
                                                      pafft_filter_t* out, int* hit) {
    if (!p || !out || !h_dev) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ALIGN_TRY(h_dev);
    ST_TRY(set_device(p));
    cudaStream_t st = (cudaStream_t)stream;
    AsyncBuf hb;
    ST_TRY(async_alloc(p, hb, 16, st));
    CUDA_TRY(cudaMemsetAsync(hb.p, 0, 16, st));
    const unsigned long long words = (unsigned long long)p->total * p->esize / 8;
    content_hash_kernel<<<(unsigned)std::min<unsigned long long>((words + 255) / 256, 148ull * 8), 256, 0, st>>>(
        (const unsigned long long*)h_dev, words, (unsigned long long*)hb.p);
    CUDA_TRY(cudaGetLastError());
    unsigned long long hh[2];
    CUDA_TRY(cudaMemcpyAsync(hh, hb.p, 16, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    CacheKey key{std::vector<unsigned>(p->radices, p->radices + p->rank), std::vector<size_t>(p->dims, p->dims + p->rank),
                 p->prec, p->device, std::vector<long long>(p->layout, p->layout + 6), hh[0], hh[1]};
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            auto g = it->second.ghat.lock();
            auto gs = it->second.ghat_scaled.lock();
            if (g && gs) {
                auto f = std::make_unique<pafft_filter_s>();
                f->plan = p;
                f->radix = p->radix;
                f->rank = p->rank;
                for (int q = 0; q < p->rank; ++q) {
                    f->dims[q] = p->dims[q];
                    f->radices[q] = p->radices[q];
                }
                f->prec = p->prec;
                f->device = p->device;
                for (int i = 0; i < 6; ++i) f->layout[i] = p->layout[i];
                f->ghat = std::move(g);
                f->ghat_scaled = std::move(gs);
                *out = f.release();
                if (hit) *hit = 1;
                ++g_cache_hits;
                return PAFFT_OK;
            }
            g_cache.erase(it);
        }
    }
    pafft_filter_t f = nullptr;
    ST_TRY(pafft_prepare_filter_from_impulse_device(p, h_dev, stream, &f));
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        // drop expired entries, then publish this one
        for (auto it = g_cache.begin(); it != g_cache.end();)
            it = it->second.ghat.expired() ? g_cache.erase(it) : std::next(it);
        g_cache[key] = CacheEntry{f->ghat, f->ghat_scaled};
    }
    ++g_cache_misses;
    if (hit) *hit = 0;
    *out = f;
    return PAFFT_OK;
}

void pafft_filter_cache_stats(uint64_t* hits, uint64_t* misses, uint64_t* live) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (hits) *hits = g_cache_hits.load();
    if (misses) *misses = g_cache_misses.load();
    if (live) {
        uint64_t n = 0;
        for (auto& e : g_cache) n += e.second.ghat.expired() ? 0 : 1;
        *live = n;
    }
}

pafft_status pafft_filter_destroy(pafft_filter_t f) {
    if (!f) return PAFFT_OK;
    cudaSetDevice(f->device);
    delete f;
    return PAFFT_OK;
}

pafft_status pafft_filter_ghat_split(pafft_filter_t f, double* re, double* im) {
    if (!f || !re || !im) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    pafft_plan_t p = f->plan;
    ST_TRY(set_device(p));
    cudaStream_t st;
    ST_TRY(call_stream(p->device, &st));
    return download_split(p, f->ghat->p, p->total, re, im, st);
}

void* pafft_filter_device_ghat(pafft_filter_t f) { return f ? f->ghat->p : nullptr; }
void* pafft_filter_device_ghat_scaled(pafft_filter_t f) { return f ? f->ghat_scaled->p : nullptr; }

int pafft_filter_matches(pafft_filter_t f, pafft_plan_t p) { return f && p && key_match(f, p) ? 1 : 0; }

// ------------------------------------------------------------- hot path
pafft_status pafft_convolve_permfree_oop(pafft_plan_t p, pafft_filter_t f, const void* x_dev, void* y_dev,
                                         size_t batch, void* stream) {
    if (!p || !f) return fail(PAFFT_INVALID_ARGUMENT, "null plan or filter");
    if (!key_match(f, p)) return fail(PAFFT_FILTER_PLAN_MISMATCH, "prepared filter does not belong to this plan");
    if (batch == 0) return PAFFT_OK;
    if (!x_dev || !y_dev) return fail(PAFFT_INVALID_ARGUMENT, "null buffer");
    ALIGN_TRY(x_dev);
    ALIGN_TRY(y_dev);
    ST_TRY(set_device(p));
    cudaStream_t st = (cudaStream_t)stream;
    const std::vector<PassDesc>& ps = p->pf;
    if (ps.empty()) return hadamard_dev(p, x_dev, f->ghat_scaled->p, y_dev, batch, st);
    for (size_t i = 0; i < ps.size(); ++i)
        ST_TRY(launch(p, ps[i], i == 0 ? x_dev : y_dev, y_dev, batch,
                      ps[i].kind == KIND_CONV ? f->ghat_scaled->p : nullptr, nullptr, 1.0, st));
    return PAFFT_OK;
}

pafft_status pafft_convolve_permfree_pass(pafft_plan_t p, pafft_filter_t f, const void* x_dev, void* y_dev,
                                          size_t batch, int i, void* stream) {
    if (!p || !f) return fail(PAFFT_INVALID_ARGUMENT, "null plan or filter");
    if (!key_match(f, p)) return fail(PAFFT_FILTER_PLAN_MISMATCH, "prepared filter does not belong to this plan");
    const std::vector<PassDesc>& ps = p->pf;
    if (ps.empty()) {
        if (i != 0) return fail(PAFFT_INVALID_ARGUMENT, "pass index %d out of range", i);
        return hadamard_dev(p, x_dev, f->ghat_scaled->p, y_dev, batch, (cudaStream_t)stream);
    }
    if (i < 0 || i >= (int)ps.size()) return fail(PAFFT_INVALID_ARGUMENT, "pass index %d out of range", i);
    ST_TRY(set_device(p));
    // profiling aid: PAFFT_PASS_GRID_CAP limits the persistent grid (co-running
    // passes on disjoint SM sets, tools/corun_probe.py)
    return launch(p, ps[i], i == 0 ? x_dev : y_dev, y_dev, batch, ps[i].kind == KIND_CONV ? f->ghat_scaled->p : nullptr,
                  nullptr, 1.0, (cudaStream_t)stream, env_int("PAFFT_PASS_GRID_CAP", 0));
}

pafft_status pafft_plan_pass_info(pafft_plan_t p, int i, int* kind, int* axis, int* R, int* stages) {
    if (!p) return fail(PAFFT_INVALID_ARGUMENT, "null plan");
    if (i < 0 || i >= (int)p->pf.size()) return fail(PAFFT_INVALID_ARGUMENT, "pass index %d out of range", i);
    const PassDesc& d = p->pf[i];
    if (kind) *kind = d.kind;
    if (axis) *axis = d.axis;
    if (R) *R = d.R;
    if (stages) *stages = d.s;
    return PAFFT_OK;
}

pafft_status pafft_convolve_permfree(pafft_plan_t p, pafft_filter_t f, void* x_dev, size_t batch, void* stream) {
    return pafft_convolve_permfree_oop(p, f, x_dev, x_dev, batch, stream);
}

pafft_status pafft_convolve_permfree_split_if(pafft_plan_t p, pafft_filter_t f, double* re, double* im,
                                              size_t batch, int (*commit)(void*), void* ctx, int* committed) {
    if (committed) *committed = 0;
    if (!p || !f) return fail(PAFFT_INVALID_ARGUMENT, "null plan or filter");
    if (!key_match(f, p)) return fail(PAFFT_FILTER_PLAN_MISMATCH, "prepared filter does not belong to this plan");
    if (batch == 0) {
        if (committed) *committed = 1;
        return PAFFT_OK;
    }
    if (!re || !im) return fail(PAFFT_INVALID_ARGUMENT, "null buffer");
    ST_TRY(set_device(p));
    cudaStream_t st;
    ST_TRY(call_stream(p->device, &st));
    const size_t n = p->total * batch;
    AsyncBuf x;
    ST_TRY(async_alloc(p, x, n * p->esize, st));
    ST_TRY(upload_split(p, re, im, n, x.p, st));
    ST_TRY(pafft_convolve_permfree(p, f, x.p, batch, st));
    // the caller's veto (the C++ shim's check that the filter's spectrum still
    // equals PreparedFilter::ghat, run on another thread while the upload and
    // the convolution were in flight): the host arrays are written only on commit
    if (commit && !commit(ctx)) {
        CUDA_TRY(cudaStreamSynchronize(st));
        return PAFFT_OK;
    }
    ST_TRY(download_split(p, x.p, n, re, im, st));
    if (committed) *committed = 1;
    return PAFFT_OK;
}

pafft_status pafft_convolve_permfree_split(pafft_plan_t p, pafft_filter_t f, double* re, double* im,
                                           size_t batch) {
    return pafft_convolve_permfree_split_if(p, f, re, im, batch, nullptr, nullptr, nullptr);
}

pafft_status pafft_convolve_permfree_host_oop(pafft_plan_t p, pafft_filter_t f, const void* x_host, void* y_host,
                                              size_t batch) {
    if (!p || !f) return fail(PAFFT_INVALID_ARGUMENT, "null plan or filter");
    if (!key_match(f, p)) return fail(PAFFT_FILTER_PLAN_MISMATCH, "prepared filter does not belong to this plan");
    if (batch == 0) return PAFFT_OK;
    ST_TRY(set_device(p));
    // the pipeline's streams and staging buffers belong to the plan: one
    // host-buffer call at a time per plan (each call is synchronous)
    std::lock_guard<std::mutex> lk(p->host_mu);
    const size_t sig_bytes = p->total * p->esize;
    // chunks of ~64 MiB pipelined over three streams: H2D(i+1) || conv(i) || D2H(i-1)
    const int ns = std::min(4, std::max(2, env_int("PAFFT_HOST_STREAMS", 3)));
    size_t chunk = std::max<size_t>(1, ((size_t)env_int("PAFFT_HOST_CHUNK_MB", 64) << 20) / sig_bytes);
    chunk = std::min(chunk, batch);
    for (int i = 0; i < ns; ++i) ST_TRY(ensure(p->stage[i], chunk * sig_bytes));
    const char* src = (const char*)x_host;
    char* dst = (char*)y_host;
    size_t done = 0;
    int k = 0;
    while (done < batch) {
        const size_t nb = std::min(chunk, batch - done);
        cudaStream_t st = p->streams[k % ns];
        void* buf = p->stage[k % ns]->p;
        CUDA_TRY(cudaMemcpyAsync(buf, src + done * sig_bytes, nb * sig_bytes, cudaMemcpyHostToDevice, st));
        ST_TRY(pafft_convolve_permfree(p, f, buf, nb, st));
        CUDA_TRY(cudaMemcpyAsync(dst + done * sig_bytes, buf, nb * sig_bytes, cudaMemcpyDeviceToHost, st));
        done += nb;
        ++k;
    }
    for (auto& s : p->streams) CUDA_TRY(cudaStreamSynchronize(s));
    return PAFFT_OK;
}

pafft_status pafft_convolve_permfree_host(pafft_plan_t p, pafft_filter_t f, void* x_host, size_t batch) {
    return pafft_convolve_permfree_host_oop(p, f, x_host, x_host, batch);
}

// ------------------------------------------------ comparator / transforms
pafft_status pafft_permute(pafft_plan_t p, void* x, size_t batch, void* stream) {
    if (!p) return fail(PAFFT_INVALID_ARGUMENT, "null plan");
    ST_TRY(set_device(p));
    cudaStream_t st = (cudaStream_t)stream;
    AsyncBuf scratch;
    ST_TRY(async_alloc(p, scratch, p->total * batch * p->esize, st));
    ST_TRY(permute_dev(p, x, scratch.p, batch, st));
    CUDA_TRY(cudaMemcpyAsync(x, scratch.p, p->total * batch * p->esize, cudaMemcpyDeviceToDevice, st));
    return PAFFT_OK;
}

static pafft_status ladder_op(pafft_plan_t p, int kind, bool permute_first, double scale, const void* mul,
                              void* x, size_t batch, cudaStream_t st) {
    ALIGN_TRY(x);
    const std::vector<PassDesc>& ps = kind == KIND_DIF ? p->dif : kind == KIND_DIT_FWD ? p->dit_fwd : p->dit_conj;
    if (permute_first) {
        AsyncBuf scratch;
        ST_TRY(async_alloc(p, scratch, p->total * batch * p->esize, st));
        ST_TRY(permute_dev(p, x, scratch.p, batch, st));
        if (ps.empty()) {
            CUDA_TRY(cudaMemcpyAsync(x, scratch.p, p->total * batch * p->esize, cudaMemcpyDeviceToDevice, st));
            if (scale != 1.0) {
                const unsigned long long n = p->total * batch;
                if (p->prec == 0)
                    scale_kernel<double><<<grid_for(n, 256), 256, 0, st>>>((const double2*)x, (double2*)x, scale, n);
                else
                    scale_kernel<float><<<grid_for(n, 256), 256, 0, st>>>((const float2*)x, (float2*)x, scale, n);
            }
            return PAFFT_OK;
        }
        return run_ladder(p, ps, scratch.p, x, batch, mul, scale, st);
    }
    if (ps.empty() && scale != 1.0) {
        const unsigned long long n = p->total * batch;
        if (p->prec == 0)
            scale_kernel<double><<<grid_for(n, 256), 256, 0, st>>>((const double2*)x, (double2*)x, scale, n);
        else
            scale_kernel<float><<<grid_for(n, 256), 256, 0, st>>>((const float2*)x, (float2*)x, scale, n);
        return PAFFT_OK;
    }
    return run_ladder(p, ps, x, x, batch, mul, scale, st);
}

pafft_status pafft_fft_forward(pafft_plan_t p, void* x, size_t batch, void* stream) {
    ST_TRY(set_device(p));
    return ladder_op(p, KIND_DIT_FWD, true, 1.0, nullptr, x, batch, (cudaStream_t)stream);
}
pafft_status pafft_fft_backward(pafft_plan_t p, void* x, size_t batch, void* stream) {
    ST_TRY(set_device(p));
    return ladder_op(p, KIND_DIT_CONJ, true, 1.0 / (double)p->total, nullptr, x, batch, (cudaStream_t)stream);
}
pafft_status pafft_fft_forward_unordered(pafft_plan_t p, void* x, size_t batch, void* stream) {
    ST_TRY(set_device(p));
    return ladder_op(p, KIND_DIT_FWD, false, 1.0, nullptr, x, batch, (cudaStream_t)stream);
}
pafft_status pafft_fft_backward_unordered(pafft_plan_t p, void* x, size_t batch, void* stream) {
    ST_TRY(set_device(p));
    return ladder_op(p, KIND_DIT_CONJ, false, 1.0 / (double)p->total, nullptr, x, batch, (cudaStream_t)stream);
}
pafft_status pafft_fft_transposed(pafft_plan_t p, void* x, size_t batch, void* stream) {
    ST_TRY(set_device(p));
    return ladder_op(p, KIND_DIF, false, 1.0, nullptr, x, batch, (cudaStream_t)stream);
}

pafft_status pafft_convolve_standard(pafft_plan_t p, const void* g_dev, void* x, size_t batch, void* stream) {
    if (!p || !g_dev) return fail(PAFFT_INVALID_ARGUMENT, "null argument");
    ALIGN_TRY(x);
    ST_TRY(set_device(p));
    cudaStream_t st = (cudaStream_t)stream;
    // fft_forward (permute #1 + A), o g fused into A's last pass, fft_backward (permute #2 + A-bar + 1/N)
    if (p->groups.empty()) {  // 1-element transform: both reorderings are identities
        g_perm_passes += 2 * batch;
        return hadamard_dev(p, x, g_dev, x, batch, st);
    }
    ST_TRY(ladder_op(p, KIND_DIT_FWD, true, 1.0, g_dev, x, batch, st));
    ST_TRY(ladder_op(p, KIND_DIT_CONJ, true, 1.0 / (double)p->total, nullptr, x, batch, st));
    return PAFFT_OK;
}

pafft_status pafft_convolve_standard_split(pafft_plan_t p, const double* g_re, const double* g_im, double* re,
                                           double* im, size_t batch) {
    if (!p) return fail(PAFFT_INVALID_ARGUMENT, "null plan");
    if (batch == 0) return PAFFT_OK;
    ST_TRY(set_device(p));
    cudaStream_t st;
    ST_TRY(call_stream(p->device, &st));
    const size_t n = p->total;
    AsyncBuf g, x;
    ST_TRY(async_alloc(p, g, n * p->esize, st));
    ST_TRY(async_alloc(p, x, n * batch * p->esize, st));
    ST_TRY(upload_split(p, g_re, g_im, n, g.p, st));
    ST_TRY(upload_split(p, re, im, n * batch, x.p, st));
    ST_TRY(pafft_convolve_standard(p, g.p, x.p, batch, st));
    return download_split(p, x.p, n * batch, re, im, st);
}

pafft_status pafft_transform_split(pafft_plan_t p, int op, double* re, double* im, size_t batch) {
    if (!p) return fail(PAFFT_INVALID_ARGUMENT, "null plan");
    if (batch == 0) return PAFFT_OK;
    if (op < 0 || op > 6) return fail(PAFFT_INVALID_ARGUMENT, "unknown transform op %d", op);
    ST_TRY(set_device(p));
    cudaStream_t st;
    ST_TRY(call_stream(p->device, &st));
    const size_t n = p->total * batch;
    AsyncBuf x;
    ST_TRY(async_alloc(p, x, n * p->esize, st));
    ST_TRY(upload_split(p, re, im, n, x.p, st));
    switch (op) {
        case 0: ST_TRY(pafft_fft_forward(p, x.p, batch, st)); break;
        case 1: ST_TRY(pafft_fft_backward(p, x.p, batch, st)); break;
        case 2: ST_TRY(pafft_fft_forward_unordered(p, x.p, batch, st)); break;
        case 3: ST_TRY(pafft_fft_backward_unordered(p, x.p, batch, st)); break;
        case 4: ST_TRY(pafft_fft_transposed(p, x.p, batch, st)); break;
        case 5: ST_TRY(pafft_permute(p, x.p, batch, st)); break;
        case 6: ST_TRY(ladder_op(p, KIND_DIT_CONJ, false, 1.0, nullptr, x.p, batch, st)); break;
    }
    return download_split(p, x.p, n, re, im, st);
}

pafft_status pafft_filter_from_impulse_split(pafft_plan_t p, const double* h_re, const double* h_im, double* g_re,
                                             double* g_im) {
    if (!p) return fail(PAFFT_INVALID_ARGUMENT, "null plan");
    memcpy(g_re, h_re, p->total * sizeof(double));
    memcpy(g_im, h_im, p->total * sizeof(double));
    return pafft_transform_split(p, 0, g_re, g_im, 1);
}

// ------------------------------------------------------------ workload
static inline uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void pafft_fill_uniform(uint64_t seed, size_t n, double* out) {
    uint64_t st = seed;
    for (size_t i = 0; i < n; ++i) {
        out[2 * i] = 2.0 * ((double)(splitmix64(st) >> 11) / 9007199254740991.0) - 1.0;
        out[2 * i + 1] = 2.0 * ((double)(splitmix64(st) >> 11) / 9007199254740991.0) - 1.0;
    }
}

void pafft_fill_normal(uint64_t seed, size_t n, double* out) {
    uint64_t st = seed;
    const double inv53 = 1.0 / 9007199254740992.0;
    const double two_pi = 2.0 * 3.14159265358979323846264338327950288;
    for (size_t i = 0; i < n; ++i) {
        const double u1 = (double)((splitmix64(st) >> 11) + 1) * inv53;
        const double u2 = (double)(splitmix64(st) >> 11) * inv53;
        const double rho = sqrt(-2.0 * log(u1));
        out[2 * i] = rho * cos(two_pi * u2);
        out[2 * i + 1] = rho * sin(two_pi * u2);
    }
}

}  // extern "C"
