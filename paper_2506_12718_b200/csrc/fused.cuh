// Fused permutation-free convolution: the three passes of a 1-D plan
// (DIF strided -> CONV contiguous -> DIT-conj strided, convolve_permfree,
// convolution.cpp:45-52) in ONE persistent launch.
//
// Every CTA takes jobs (pass, signal, tile) from a global ticket counter.  The
// tickets run in steps k = 0, 1, ...; step k holds the DIT tiles of signal
// k - 2D, the CONV tiles of signal k - D and the DIF tiles of signal k (D =
// lag), so a signal's intermediate is re-read by the next pass about D steps
// after it was written -- while it is still in L2 -- instead of after the whole
// batch went through HBM, and HBM-bound (DIF/DIT) and FP64-bound (CONV) tiles
// run side by side on the machine.  A CONV tile of signal s starts only when
// all DIF tiles of s are stored (per-(pass, signal) counters, release/acquire),
// a DIT tile only when all CONV tiles of s are.
//
// Deadlock freedom: a CTA blocks on a dependency only while it holds no
// unfinished job (its previous store is completed and counted first), and
// dependencies point to strictly smaller tickets, which running CTAs finish.
// The tile bodies are the pass kernels' own (run_tile, pass.cuh); the CTA is
// as wide as the widest of the two tile shapes, narrower tiles idle the rest.
#pragma once

#include "pass.cuh"

namespace pafft_b200 {

template <typename T> struct FusedArgs {
    PassArgs<T> p[3];   // 0 = DIF (strided), 1 = CONV (contiguous), 2 = DIT-conj (strided)
    unsigned* ticket;   // job ticket counter (zeroed per call)
    unsigned* done;     // [3][nsig] stored tiles per (pass, signal) (zeroed per call)
    int nsig;
    int lag;
    int U[3];           // tiles per signal of each pass
    long long nticket;  // (nsig + 2 lag) * (U0 + U1 + U2)
};

struct FusedMaps {
    CUtensorMap src[3];
    CUtensorMap dst[3];
};

struct FusedJob {
    int p;        // pass, -1 = no more work
    int s;        // signal
    long long tile;
    int staged;   // 1: the TMA load is issued; 0: waits for its dependency
    int pad;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait2() { asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

// Bounded waits: a dependency that never completes (a scheduling bug) traps
// the launch (an error the host reports) instead of hanging the device.
#ifndef PAFFT_FUSED_SPIN_LIMIT
#define PAFFT_FUSED_SPIN_LIMIT (1u << 25)
#endif
__device__ __forceinline__ void mbar_wait_bounded(unsigned long long* bar, unsigned phase) {
    unsigned ok;
    unsigned n = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (++n > PAFFT_FUSED_SPIN_LIMIT) __trap();
    } while (!ok);
}

template <typename T, int RADIX, int D0, int D1, int D2, int D3, int WD, int C0, int C1, int C2, int C3, int WC>
struct FusedShape {
    using FD = Fac<D0, D1, D2, D3>;
    using FC = Fac<C0, C1, C2, C3>;
    using PD = TilePolicy<T, FD, MAP_STRIDED, WD>;
    using PC = TilePolicy<T, FC, MAP_CONTIG, WC>;
    static constexpr int NT = ((PD::NT > PC::NT ? PD::NT : PC::NT) + 31) / 32 * 32;
    static constexpr int BUF = PD::BUF > PC::BUF ? PD::BUF : PC::BUF;
    static constexpr int SMEM = 2 * BUF + 16 + 2 * (int)sizeof(FusedJob);
    static constexpr int MINB_SMEM = (227 * 1024) / (SMEM + 1024);
    static constexpr int MINB = MINB_SMEM < 1 ? 1 : (MINB_SMEM > 4 ? 4 : MINB_SMEM);
};

template <typename T, int RADIX, int D0, int D1, int D2, int D3, int WD, int C0, int C1, int C2, int C3, int WC>
__global__ void __launch_bounds__((FusedShape<T, RADIX, D0, D1, D2, D3, WD, C0, C1, C2, C3, WC>::NT),
                                  (FusedShape<T, RADIX, D0, D1, D2, D3, WD, C0, C1, C2, C3, WC>::MINB))
    fused_conv_kernel(const FusedArgs<T> fa, const __grid_constant__ FusedMaps maps) {
    using V = cplx<T>;
    using SH = FusedShape<T, RADIX, D0, D1, D2, D3, WD, C0, C1, C2, C3, WC>;
    using FD = typename SH::FD;
    using FC = typename SH::FC;
    using PD = typename SH::PD;
    using PC = typename SH::PC;
    constexpr int BUFE = SH::BUF / (int)sizeof(V);
    static_assert(!PD::SHIFT, "fused kernel: fp64 / tensor-map strided tiles only");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    V* const bufs = reinterpret_cast<V*>(smem_raw);
    unsigned long long* const bars = reinterpret_cast<unsigned long long*>(smem_raw + 2 * SH::BUF);
    FusedJob* const jobs = reinterpret_cast<FusedJob*>(smem_raw + 2 * SH::BUF + 16);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int SU = fa.U[0] + fa.U[1] + fa.U[2];

    // ---- scheduler (thread 0 only) ------------------------------------------
    // The next ticket is fetched one job ahead (its atomic's latency hides
    // behind a tile); a (pass, signal) seen complete is cached (counters only
    // grow), so most readiness checks cost no memory round trip.
    unsigned long long q_pre = 0;
    int rc_p = -1, rc_s = -1;
    auto take = [&]() -> FusedJob {
        FusedJob j{-1, 0, 0, 0, 0};
        for (;;) {
            const long long q = (long long)q_pre;
            if (q >= fa.nticket) return j;
            q_pre = atomicAdd(fa.ticket, 1u);
            const long long k = q / SU;
            int r = (int)(q - k * SU);
            int p, s;
            if (r < fa.U[2]) {
                p = 2;
                s = (int)(k - 2 * fa.lag);
            } else if ((r -= fa.U[2]) < fa.U[1]) {
                p = 1;
                s = (int)(k - fa.lag);
            } else {
                r -= fa.U[1];
                p = 0;
                s = (int)k;
            }
            if (s < 0 || s >= fa.nsig) continue;  // pipeline fill / drain slot
            j.p = p;
            j.s = s;
            j.tile = (long long)s * fa.U[p] + r;
            return j;
        }
    };
    auto ready = [&](const FusedJob& j) -> bool {
        if (j.p == 0 || (j.p == rc_p && j.s == rc_s)) return true;
        if (ld_acquire(fa.done + (long long)(j.p - 1) * fa.nsig + j.s) >= (unsigned)fa.U[j.p - 1]) {
            rc_p = j.p;
            rc_s = j.s;
            return true;
        }
        return false;
    };
    auto wait_ready = [&](const FusedJob& j) {
        for (unsigned n = 0; !ready(j); ++n) {
            if (n > PAFFT_FUSED_SPIN_LIMIT / 16) __trap();
            __nanosleep(128);
        }
    };
    auto stage = [&](const FusedJob& j, V* buf, unsigned long long* bar) {
        fence_proxy_async_global();  // the producer's stores (async proxy) before our TMA reads
        if (j.p == 1)
            stage_tile<FC::R, PC::W, PC::SW, false>(fa.p[1], &maps.src[1], j.tile, buf, bar, 0);
        else
            stage_tile<FD::R, PD::W, PD::SW, true>(fa.p[j.p], &maps.src[j.p], j.tile, buf, bar, 0);
    };
    auto signal = [&](const FusedJob& j) {
        fence_proxy_async_global();
        __threadfence();
        atomicAdd(fa.done + (long long)j.p * fa.nsig + j.s, 1u);
    };

    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        q_pre = atomicAdd(fa.ticket, 1u);
        FusedJob j0 = take();
        if (j0.p >= 0) {
            wait_ready(j0);
            stage(j0, bufs, &bars[0]);
            j0.staged = 1;
        }
        jobs[0] = j0;  // buffer 1 is filled by the first tile's service
    }
    __syncthreads();

    // thread 0: jobs whose stores are committed but not yet counted (A older);
    // a job is counted one tile after its store left shared memory, when its
    // global writes are complete (bulk wait_group), so nobody stalls on them
    FusedJob pa{-1, 0, 0, 0, 0}, pb{-1, 0, 0, 0, 0};
    unsigned uses0 = 0, uses1 = 0;
    for (int it = 0;; ++it) {
        const int b = it & 1;
        V* const buf = bufs + b * BUFE;
        const FusedJob J = jobs[b];
        if (J.p < 0) break;
        if (t == 0 && !J.staged) {
            // blocking: first count every finished job (one may be J's dependency)
            bulk_wait0();
            if (pa.p >= 0) signal(pa);
            if (pb.p >= 0) signal(pb);
            pa.p = pb.p = -1;
            wait_ready(J);
            stage(J, buf, &bars[b]);
        }
        const unsigned ph = (b ? uses1++ : uses0++) & 1;
        mbar_wait_bounded(&bars[b], ph);

        // count job i-2, free the other buffer (job i-1's store has read it) and
        // fill it with the next job: inside the tile after its first barrier,
        // or after the tile (POST: this tile's store is committed too)
        bool serviced = false;
        auto service_impl = [&](auto post) {
            serviced = true;
            if (t == 0) {
                constexpr bool POST = decltype(post)::value;
                if (pa.p >= 0) {
                    if constexpr (POST) bulk_wait2();
                    else bulk_wait1();
                    signal(pa);
                }
                if constexpr (POST) bulk_wait_read1();
                else bulk_wait_read0();
                pa = pb;
                pb.p = -1;
                FusedJob n = take();
                if (n.p >= 0 && ready(n)) {
                    stage(n, bufs + (b ^ 1) * BUFE, &bars[b ^ 1]);
                    n.staged = 1;
                }
                jobs[b ^ 1] = n;
            }
        };
        auto service = [&]() { service_impl(std::false_type{}); };
        if (J.p == 1)
            run_tile<T, RADIX, FC, KIND_CONV, MAP_CONTIG, PC, PC::NT == SH::NT>(fa.p[1], &maps.dst[1], J.tile, buf,
                                                                               bufs + 2 * BUFE, t, service);
        else if (J.p == 0)
            run_tile<T, RADIX, FD, KIND_DIF, MAP_STRIDED, PD, PD::NT == SH::NT>(fa.p[0], &maps.dst[0], J.tile, buf,
                                                                               bufs + 2 * BUFE, t, service);
        else
            run_tile<T, RADIX, FD, KIND_DIT_CONJ, MAP_STRIDED, PD, PD::NT == SH::NT>(fa.p[2], &maps.dst[2], J.tile,
                                                                                    buf, bufs + 2 * BUFE, t, service);
        if (!serviced) service_impl(std::true_type{});
        if (t == 0) pb = J;
        // the next job's descriptor (written by thread 0) before anyone reads it
        __syncthreads();
    }
    if (t == 0) {
        bulk_wait0();
        if (pa.p >= 0) signal(pa);
        if (pb.p >= 0) signal(pb);
    }
    (void)warp;
    (void)lane;
}

}  // namespace pafft_b200
