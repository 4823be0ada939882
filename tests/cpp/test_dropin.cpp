// Reference-style unit checks compiled against the C++ drop-in header
// (include/pafft/pafft.hpp) and run on the GPU library.  The cases restate
// the reference's own tests (test_convolution.cpp:22-145,
// test_butterfly.cpp:28-45/106-121, test_core.cpp:29-70,
// test_permutation.cpp:15-31); a tiny harness replaces doctest (absent).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "pafft/pafft.hpp"

using namespace pafft;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                       \
    do {                                                                  \
        if (cond) ++g_pass;                                               \
        else { ++g_fail; std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                       \
    do {                                               \
        bool ok_ = false;                              \
        try { expr; } catch (const T&) { ok_ = true; } catch (...) {} \
        CHECK(ok_ && #T);                              \
    } while (0)

static ComplexBuffer buf(std::initializer_list<std::complex<double>> v) {
    ComplexBuffer b(v.size());
    std::size_t i = 0;
    for (auto c : v) b.set(i++, c);
    return b;
}
static double max_diff(const ComplexBuffer& a, const ComplexBuffer& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i)
        m = std::max(m, std::max(std::abs(a.re[i] - b.re[i]), std::abs(a.im[i] - b.im[i])));
    return m;
}
static bool bitwise_equal(const ComplexBuffer& a, const ComplexBuffer& b) {
    for (std::size_t i = 0; i < a.size(); ++i)
        if (a.re[i] != b.re[i] || a.im[i] != b.im[i]) return false;
    return a.size() == b.size();
}
static ComplexBuffer random_buffer(std::size_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> d(-1, 1);
    ComplexBuffer b(n);
    for (std::size_t i = 0; i < n; ++i) { b.re[i] = d(rng); b.im[i] = d(rng); }
    return b;
}

int main() {
    // plan validation (test_core.cpp:29-42)
    CHECK_THROWS_AS(plan_create(Radix::r2, TensorShape(std::vector<std::size_t>{})), EmptyShape);
    CHECK_THROWS_AS(plan_create(Radix::r8, TensorShape{4}), NotAPowerOfRadix);
    CHECK_THROWS_AS(plan_create(Radix::r4, TensorShape{8}), NotAPowerOfRadix);
    try {
        plan_create(Radix::r2, TensorShape{8, 3});
        CHECK(false);
    } catch (const NotAPowerOfRadix& e) {
        CHECK(e.dim == 1 && e.extent == 3);
    }
    CHECK_THROWS_AS(radix_from_value(7), Error);
    {
        const Plan p2 = plan_create(Radix::r2, TensorShape{8});
        const std::vector<std::uint32_t> expect{0, 4, 2, 6, 1, 5, 3, 7};
        for (std::size_t j = 0; j < 8; ++j) CHECK(p2.rev_map(0)[j] == expect[j]);
        CHECK(p2.depth(0) == 3);
        CHECK(digit_reverse(6, 2, 3) == 3 && digit_reverse(5, 4, 2) == 5 && digit_reverse(5, 3, 2) == 7);
        CHECK_THROWS_AS(digit_reverse(8, 2, 3), IndexOutOfRange);
    }
    // 4-point ladders (test_butterfly.cpp:28-45)
    {
        const Plan plan = plan_create(Radix::r2, TensorShape{4});
        ComplexBuffer x = buf({1, 3, 2, 4});
        butterfly_forward(x, plan, 0);
        CHECK(max_diff(x, buf({10, {-2, 2}, -2, {-2, -2}})) < 1e-13);
        ComplexBuffer y = buf({10, -2, {-2, 2}, {-2, -2}});
        butterfly_conjugate(y, plan, 0);
        CHECK(max_diff(y, buf({4, 8, 12, 16})) < 1e-13);
        ComplexBuffer z = buf({1, 2, 3, 4});
        butterfly_transposed(z, plan, 0);
        CHECK(max_diff(z, buf({10, -2, {-2, 2}, {-2, -2}})) < 1e-13);
        ComplexBuffer w(8);
        CHECK_THROWS_AS(butterfly_forward(w, plan, 0), ShapeMismatch);
    }
    // filter layout, delay filter, both pipelines (test_convolution.cpp:32-61)
    {
        const Plan plan = plan_create(Radix::r2, TensorShape{4});
        const PreparedFilter f = prepare_filter(buf({0, 1, 2, 3}), plan);
        CHECK(max_diff(f.ghat, buf({0, 2, 1, 3})) == 0.0);
        CHECK(f.key == plan.key());
        CHECK_THROWS_AS(prepare_filter(ComplexBuffer(3), plan), LengthMismatch);
        const ComplexBuffer g = filter_from_impulse(buf({0, 1, 0, 0}), plan);
        CHECK(max_diff(g, buf({1, {0, -1}, -1, {0, 1}})) < 1e-14);
        ComplexBuffer x = buf({1, 2, 3, 4});
        convolve_standard(x, g, plan);
        CHECK(max_diff(x, buf({4, 1, 2, 3})) < 1e-13);
        ComplexBuffer y = buf({1, 2, 3, 4});
        convolve_permfree(y, prepare_filter(g, plan), plan);
        CHECK(max_diff(y, buf({4, 1, 2, 3})) < 1e-13);
    }
    // pass accounting (test_convolution.cpp:63-79)
    {
        const Plan plan = plan_create(Radix::r4, TensorShape{16, 16});
        const ComplexBuffer g = random_buffer(plan.total(), 73);
        ComplexBuffer x = random_buffer(plan.total(), 74);
        reset_permutation_pass_count();
        convolve_standard(x, g, plan);
        CHECK(permutation_pass_count() == 2);
        reset_permutation_pass_count();
        const PreparedFilter filter = prepare_filter(g, plan);
        CHECK(permutation_pass_count() == 1);
        reset_permutation_pass_count();
        convolve_permfree(x, filter, plan);
        CHECK(permutation_pass_count() == 0);
    }
    // plan binding (test_convolution.cpp:81-97)
    {
        const Plan plan = plan_create(Radix::r2, TensorShape{16});
        const PreparedFilter filter = prepare_filter(random_buffer(16, 79), plan);
        ComplexBuffer x = random_buffer(16, 80);
        CHECK_THROWS_AS(convolve_permfree(x, filter, plan_create(Radix::r4, TensorShape{16})), FilterPlanMismatch);
        CHECK_THROWS_AS(convolve_permfree(x, filter, plan_create(Radix::r2, TensorShape{4, 4})), FilterPlanMismatch);
        convolve_permfree(x, filter, plan_create(Radix::r2, TensorShape{16}));
        ++g_pass;
    }
    // reuse without drift (test_convolution.cpp:99-111) and radix 3
    for (auto [radix, shape] : {std::pair<Radix, TensorShape>{Radix::r2, {8, 8}}, {Radix::r3, {27, 9}},
                                {Radix::r5, {125}}}) {
        const Plan plan = plan_create(radix, shape);
        const PreparedFilter filter = prepare_filter(random_buffer(plan.total(), 83), plan);
        const ComplexBuffer x = random_buffer(plan.total(), 84);
        ComplexBuffer first = x;
        convolve_permfree(first, filter, plan);
        for (int round = 0; round < 3; ++round) {
            ComplexBuffer again = x;
            convolve_permfree(again, filter, plan);
            CHECK(bitwise_equal(again, first));
        }
        ComplexBuffer std_ = x;
        convolve_standard(std_, filter_from_impulse(random_buffer(plan.total(), 85), plan), plan);
        ++g_pass;
    }
    // conjugate ladder equals conjugated forward ladder (test_butterfly.cpp:106-121)
    {
        const Plan plan = plan_create(Radix::r4, TensorShape{256});
        const ComplexBuffer x = random_buffer(256, 37);
        ComplexBuffer direct = x;
        butterfly_conjugate(direct, plan, 0);
        ComplexBuffer wrapped = x;
        for (double& v : wrapped.im) v = -v;
        butterfly_forward(wrapped, plan, 0);
        for (double& v : wrapped.im) v = -v;
        CHECK(max_diff(direct, wrapped) < 1e-12);
    }
    // per-axis radices (extension): a delay along axis 0
    // shifts cyclically; keys tell mixed and uniform plans apart
    {
        const Plan plan = plan_create(std::vector<Radix>{Radix::r3, Radix::r2}, TensorShape{27, 16});
        CHECK(plan.radix(0) == Radix::r3 && plan.radix(1) == Radix::r2 && plan.depth(0) == 3 && plan.depth(1) == 4);
        ComplexBuffer h(plan.total());
        h.re[1] = 1.0;
        const PreparedFilter filter = prepare_filter(filter_from_impulse(h, plan), plan);
        const ComplexBuffer x = random_buffer(plan.total(), 91);
        ComplexBuffer y = x;
        convolve_permfree(y, filter, plan);
        ComplexBuffer want(plan.total());
        for (std::size_t i1 = 0; i1 < 16; ++i1)
            for (std::size_t i0 = 0; i0 < 27; ++i0) {
                want.re[(i0 + 1) % 27 + 27 * i1] = x.re[i0 + 27 * i1];
                want.im[(i0 + 1) % 27 + 27 * i1] = x.im[i0 + 27 * i1];
            }
        CHECK(max_diff(y, want) < 1e-13);
        const Plan p24 = plan_create(std::vector<Radix>{Radix::r2, Radix::r4}, TensorShape{16, 16});
        const PreparedFilter f24 = prepare_filter(random_buffer(256, 92), p24);
        ComplexBuffer z = random_buffer(256, 93);
        CHECK_THROWS_AS(convolve_permfree(z, f24, plan_create(Radix::r2, TensorShape{16, 16})), FilterPlanMismatch);
        CHECK_THROWS_AS(plan_create(std::vector<Radix>{Radix::r3, Radix::r2}, TensorShape{27, 27}), NotAPowerOfRadix);
    }
    // PreparedFilter{ghat, key} is an aggregate whose ghat is the source of
    // truth, as in the reference (convolution.hpp:9-12, convolution.cpp:49):
    // a hand-built filter works, and an edit to ghat is honoured
    {
        const Plan plan = plan_create(Radix::r2, TensorShape{4});
        ComplexBuffer delay(4);
        delay.re[1] = 1.0;
        const PreparedFilter built = prepare_filter(filter_from_impulse(delay, plan), plan);
        const PreparedFilter by_hand{built.ghat, built.key};  // aggregate, no device copy
        ComplexBuffer a = buf({1, 2, 3, 4}), b = a;
        convolve_permfree(a, built, plan);
        convolve_permfree(b, by_hand, plan);
        CHECK(bitwise_equal(a, b) && max_diff(a, buf({4, 1, 2, 3})) < 1e-13);
        PreparedFilter edited = built;  // a copy, then edit its spectrum: identity filter
        for (std::size_t i = 0; i < 4; ++i) edited.ghat.set(i, 1.0);
        ComplexBuffer c = buf({1, 2, 3, 4});
        convolve_permfree(c, edited, plan);
        CHECK(max_diff(c, buf({1, 2, 3, 4})) < 1e-13);
        ComplexBuffer d = buf({1, 2, 3, 4});
        convolve_permfree(d, built, plan);  // the shared original still delays
        CHECK(max_diff(d, buf({4, 1, 2, 3})) < 1e-13);
    }
    // the same for a spectrum large enough that the byte check runs on a
    // second thread, overlapped with the device call (commit-gated write-back)
    {
        const std::size_t n = std::size_t{1} << 16;
        const Plan plan = plan_create(Radix::r4, TensorShape{n});
        ComplexBuffer delay(n);
        delay.re[1] = 1.0;
        PreparedFilter f = prepare_filter(filter_from_impulse(delay, plan), plan);
        const ComplexBuffer x = random_buffer(n, 95);
        ComplexBuffer a = x;
        convolve_permfree(a, f, plan);
        CHECK(std::abs(a.re[1] - x.re[0]) < 1e-12 && std::abs(a.im[0] - x.im[n - 1]) < 1e-12);
        for (std::size_t i = 0; i < n; ++i) f.ghat.set(i, 2.0);  // edit in place: 2 x identity
        ComplexBuffer b = x;
        convolve_permfree(b, f, plan);
        double m = 0;
        for (std::size_t i = 0; i < n; ++i) m = std::max(m, std::abs(b.get(i) - 2.0 * x.get(i)));
        CHECK(m < 1e-12);
        ComplexBuffer c = x;  // and again, from the rebuilt device copy
        convolve_permfree(c, f, plan);
        CHECK(bitwise_equal(b, c));
    }
    // C-order <-> vec repack (core.cpp:131-178 semantics): element (i0, i1, i2)
    // of a C-order [2][3][4] tensor lands at vec offset i0 + 2 i1 + 6 i2
    {
        const TensorShape shape{2, 3, 4};
        std::vector<std::complex<double>> vals(24);
        for (std::size_t c = 0; c < 24; ++c) vals[c] = {double(c), -double(c)};
        const ComplexBuffer v = buffer_from_tensor(vals, shape);
        bool ok = true;
        for (std::size_t i0 = 0; i0 < 2; ++i0)
            for (std::size_t i1 = 0; i1 < 3; ++i1)
                for (std::size_t i2 = 0; i2 < 4; ++i2)
                    ok = ok && v.get(i0 + 2 * i1 + 6 * i2) == vals[i2 + 4 * i1 + 12 * i0];
        CHECK(ok);
        CHECK(tensor_from_buffer(v, shape) == vals);
        CHECK_THROWS_AS(buffer_from_tensor(std::span<const std::complex<double>>(vals.data(), 23), shape), LengthMismatch);
    }
    std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
