// ref_capi.cpp -- a thin extern "C" shim over the UNMODIFIED reference
// library (pafft, compiled from /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/libpafft_ref.so).  TEST INFRASTRUCTURE ONLY: it exists so
// the oracle restatement can be pinned against the reference's own results
// (tests/golden/make_golden.py) and so bench.py can time the reference CPU
// path (cpu_baseline kind "reference") on radix 2/4/8 workloads.
//
// Every call goes through pafft's public API (convolution.hpp, core.hpp,
// permutation.hpp, butterfly.hpp, oracle.hpp); the shim only moves split
// re/im arrays in and out of pafft::ComplexBuffer.
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "pafft/butterfly.hpp"
#include "pafft/convolution.hpp"
#include "pafft/core.hpp"
#include "pafft/oracle.hpp"
#include "pafft/permutation.hpp"
#include "pafft/transform.hpp"

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const pafft::NotAPowerOfRadix*>(&e)) return 1;
    if (dynamic_cast<const pafft::EmptyShape*>(&e)) return 2;
    if (dynamic_cast<const pafft::LengthMismatch*>(&e)) return 3;
    if (dynamic_cast<const pafft::ShapeMismatch*>(&e)) return 4;
    if (dynamic_cast<const pafft::FilterPlanMismatch*>(&e)) return 5;
    if (dynamic_cast<const pafft::IndexOutOfRange*>(&e)) return 6;
    return 7;
}

pafft::ComplexBuffer load(const double* re, const double* im, std::size_t n) {
    pafft::ComplexBuffer b(n);
    std::memcpy(b.re.data(), re, n * sizeof(double));
    std::memcpy(b.im.data(), im, n * sizeof(double));
    return b;
}

void store(const pafft::ComplexBuffer& b, double* re, double* im) {
    std::memcpy(re, b.re.data(), b.size() * sizeof(double));
    std::memcpy(im, b.im.data(), b.size() * sizeof(double));
}

struct Batch {
    const pafft::Plan* plan;
    pafft::PreparedFilter filter;
    std::vector<pafft::ComplexBuffer> signals;
};

}  // namespace

#define GUARD(...)                                    \
    try {                                             \
        __VA_ARGS__;                                      \
        return 0;                                     \
    } catch (const std::exception& e) {               \
        return code_of(e);                            \
    }

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_plan_create(unsigned radix, const std::size_t* dims, int rank, void** out) {
    GUARD({
        std::vector<std::size_t> d(dims, dims + rank);
        *out = new pafft::Plan(pafft::plan_create(pafft::radix_from_value(radix), pafft::TensorShape(d)));
    })
}

void ref_plan_destroy(void* p) { delete static_cast<pafft::Plan*>(p); }

int ref_digit_reverse(std::uint64_t j, unsigned radix, unsigned digits, std::uint64_t* out) {
    GUARD(*out = pafft::digit_reverse(j, radix, digits))
}

std::uint64_t ref_permutation_pass_count() { return pafft::permutation_pass_count(); }
void ref_reset_permutation_pass_count() { pafft::reset_permutation_pass_count(); }

int ref_permute_tensor(void* p, double* re, double* im) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        auto b = load(re, im, plan.total());
        pafft::permute_tensor(b, plan);
        store(b, re, im);
    })
}

// variant: 0 forward, 1 conjugate, 2 transposed (butterfly.hpp:12-16)
int ref_butterfly_line(void* p, std::size_t dim, int variant, double* re, double* im, std::size_t len) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        auto b = load(re, im, len);
        if (variant == 0) pafft::butterfly_forward(b, plan, dim);
        else if (variant == 1) pafft::butterfly_conjugate(b, plan, dim);
        else pafft::butterfly_transposed(b, plan, dim);
        store(b, re, im);
    })
}

int ref_butterfly_tensor(void* p, int variant, double* re, double* im) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        auto b = load(re, im, plan.total());
        const auto v = variant == 0 ? pafft::ButterflyVariant::forward
                       : variant == 1 ? pafft::ButterflyVariant::conjugate
                                      : pafft::ButterflyVariant::transposed;
        pafft::butterfly_tensor(b, plan, v);
        store(b, re, im);
    })
}

int ref_prepare_filter(void* p, const double* gr, const double* gi, double* outr, double* outi) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        const auto f = pafft::prepare_filter(load(gr, gi, plan.total()), plan);
        store(f.ghat, outr, outi);
    })
}

int ref_filter_from_impulse(void* p, const double* hr, const double* hi, double* gr, double* gi) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        store(pafft::filter_from_impulse(load(hr, hi, plan.total()), plan), gr, gi);
    })
}

int ref_convolve_permfree(void* p, const double* ghr, const double* ghi, double* re, double* im) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        const pafft::PreparedFilter f{load(ghr, ghi, plan.total()), plan.key()};
        auto b = load(re, im, plan.total());
        pafft::convolve_permfree(b, f, plan);
        store(b, re, im);
    })
}

int ref_convolve_standard(void* p, const double* gr, const double* gi, double* re, double* im) {
    GUARD({
        const auto& plan = *static_cast<pafft::Plan*>(p);
        auto b = load(re, im, plan.total());
        pafft::convolve_standard(b, load(gr, gi, plan.total()), plan);
        store(b, re, im);
    })
}

int ref_naive_circular_convolution(const std::size_t* dims, int rank, const double* xr, const double* xi,
                                   const double* hr, const double* hi, double* yr, double* yi) {
    GUARD({
        pafft::TensorShape shape(std::vector<std::size_t>(dims, dims + rank));
        const auto y = pafft::oracle::naive_circular_convolution(load(xr, xi, shape.total()),
                                                                 load(hr, hi, shape.total()), shape);
        store(y, yr, yi);
    })
}

int ref_naive_dft_tensor(const std::size_t* dims, int rank, int backward, const double* xr, const double* xi,
                         double* yr, double* yi) {
    GUARD({
        pafft::TensorShape shape(std::vector<std::size_t>(dims, dims + rank));
        const auto y = pafft::oracle::naive_dft_tensor(
            load(xr, xi, shape.total()), shape,
            backward ? pafft::oracle::Direction::backward : pafft::oracle::Direction::forward);
        store(y, yr, yi);
    })
}

// Batched comparator for bench.py: buffers are staged once outside timing;
// ref_batch_run times only convolve_permfree calls (threads share the
// immutable Plan/PreparedFilter) and returns wall seconds.
void* ref_batch_create(void* p, const double* ghr, const double* ghi, const double* re, const double* im,
                       std::size_t batch) {
    try {
        const auto& plan = *static_cast<pafft::Plan*>(p);
        auto* b = new Batch{&plan, pafft::PreparedFilter{load(ghr, ghi, plan.total()), plan.key()}, {}};
        b->signals.reserve(batch);
        for (std::size_t i = 0; i < batch; ++i)
            b->signals.push_back(load(re + i * plan.total(), im + i * plan.total(), plan.total()));
        return b;
    } catch (const std::exception& e) {
        code_of(e);
        return nullptr;
    }
}

double ref_batch_run(void* h, int threads) {
    auto* b = static_cast<Batch*>(h);
    const std::size_t n = b->signals.size();
    if (threads < 1) threads = 1;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([b, t, threads, n] {
            for (std::size_t i = static_cast<std::size_t>(t); i < n; i += static_cast<std::size_t>(threads))
                pafft::convolve_permfree(b->signals[i], b->filter, *b->plan);
        });
    }
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void ref_batch_read(void* h, std::size_t i, double* re, double* im) {
    store(static_cast<Batch*>(h)->signals[i], re, im);
}

void ref_batch_destroy(void* h) { delete static_cast<Batch*>(h); }

}  // extern "C"
