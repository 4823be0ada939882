// pafft/pafft.hpp -- C++ drop-in for the reference library's public API
// (namespace pafft: core.hpp, errors.hpp, convolution.hpp, permutation.hpp,
// transform.hpp, butterfly.hpp), header-only over the C ABI
// (include/pafft_b200.h, libpafft_b200.so).  Same names, argument meanings,
// exception classes and ownership as the reference, so caller code
// (e.g. bench.cpp:169-180, verify.cpp:117-125, the unit tests) compiles
// unchanged against it; every transform and convolution runs on the B200.
//
// Differences, all supersets: Radix also has r3 and r5; Plan takes an
// optional precision/device; PreparedFilter additionally owns the device copy
// of ghat (its public `ghat`/`key` fields keep the reference meaning,
// convolution.hpp:9-12).  Link with -lpafft_b200.
#pragma once

#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <memory>
#include <numbers>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../pafft_b200.h"

namespace pafft {

// ------------------------------------------------------------ errors.hpp
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NotAPowerOfRadix : Error {
    NotAPowerOfRadix(std::size_t dim_, std::size_t extent_, const std::string& msg)
        : Error(msg), dim(dim_), extent(extent_) {}
    std::size_t dim;
    std::size_t extent;
};
struct EmptyShape : Error {
    using Error::Error;
};
struct LengthMismatch : Error {
    using Error::Error;
    LengthMismatch(std::size_t expected, std::size_t got)
        : Error("buffer length mismatch: expected " + std::to_string(expected) + ", got " + std::to_string(got)) {}
};
struct ShapeMismatch : Error {
    using Error::Error;
    ShapeMismatch(std::size_t expected, std::size_t got)
        : Error("line length mismatch: expected " + std::to_string(expected) + ", got " + std::to_string(got)) {}
};
struct FilterPlanMismatch : Error {
    FilterPlanMismatch() : Error("prepared filter does not belong to this plan") {}
    using Error::Error;
};
struct IndexOutOfRange : Error {
    using Error::Error;
};

namespace detail {
// Rethrows a C-ABI status as the matching reference exception class.
inline void check(pafft_status st) {
    if (st == PAFFT_OK) return;
    const std::string msg = pafft_last_error();
    switch (st) {
        case PAFFT_NOT_A_POWER_OF_RADIX: {
            std::size_t d = 0, e = 0;
            pafft_last_error_dim(&d, &e);
            throw NotAPowerOfRadix(d, e, msg);
        }
        case PAFFT_EMPTY_SHAPE: throw EmptyShape(msg);
        case PAFFT_LENGTH_MISMATCH: throw LengthMismatch(msg);
        case PAFFT_SHAPE_MISMATCH: throw ShapeMismatch(msg);
        case PAFFT_FILTER_PLAN_MISMATCH: throw FilterPlanMismatch(msg);
        case PAFFT_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
        default: throw Error(msg);
    }
}
}  // namespace detail

// -------------------------------------------------------------- core.hpp
enum class Radix : unsigned { r2 = 2, r3 = 3, r4 = 4, r5 = 5, r8 = 8 };

constexpr unsigned radix_value(Radix r) { return static_cast<unsigned>(r); }

inline Radix radix_from_value(unsigned value) {
    switch (value) {
        case 2: return Radix::r2;
        case 3: return Radix::r3;
        case 4: return Radix::r4;
        case 5: return Radix::r5;
        case 8: return Radix::r8;
        default: throw Error("radix must be 2, 3, 4, 5, or 8 (got " + std::to_string(value) + ")");
    }
}

class TensorShape {
public:
    TensorShape() = default;
    TensorShape(std::initializer_list<std::size_t> extents) : dims_(extents) {}
    explicit TensorShape(std::vector<std::size_t> extents) : dims_(std::move(extents)) {}
    std::size_t rank() const { return dims_.size(); }
    std::size_t dim(std::size_t q) const { return dims_[q]; }
    const std::vector<std::size_t>& dims() const { return dims_; }
    std::size_t total() const {
        std::size_t n = 1;
        for (std::size_t e : dims_) n *= e;
        return n;
    }
    bool operator==(const TensorShape&) const = default;

private:
    std::vector<std::size_t> dims_;
};

struct ComplexBuffer {
    std::vector<double> re;
    std::vector<double> im;
    ComplexBuffer() = default;
    explicit ComplexBuffer(std::size_t n) : re(n, 0.0), im(n, 0.0) {}
    std::size_t size() const { return re.size(); }
    std::complex<double> get(std::size_t i) const { return {re[i], im[i]}; }
    void set(std::size_t i, std::complex<double> v) {
        re[i] = v.real();
        im[i] = v.imag();
    }
};

inline double max_abs(const ComplexBuffer& x) {
    double m = 0.0;
    for (std::size_t i = 0; i < x.size(); ++i) m = std::max(m, std::sqrt(x.re[i] * x.re[i] + x.im[i] * x.im[i]));
    return m;
}

inline void scale_inplace(ComplexBuffer& x, double s) {
    for (double& v : x.re) v *= s;
    for (double& v : x.im) v *= s;
}

// Host copy of the reference's master table w[j] = exp(-2 pi i j / n)
// (core.hpp:71-88); the device uses its own per-pass tables.
class TwiddleTable {
public:
    explicit TwiddleTable(std::size_t n) : n_(n), re_(n), im_(n) {
        const double step = -2.0 * std::numbers::pi / static_cast<double>(n);
        for (std::size_t j = 0; j < n; ++j) {
            re_[j] = std::cos(step * static_cast<double>(j));
            im_[j] = std::sin(step * static_cast<double>(j));
        }
    }
    std::size_t length() const { return n_; }
    double re(std::size_t j) const { return re_[j]; }
    double im(std::size_t j) const { return im_[j]; }
    std::size_t stage_stride(std::size_t k) const { return n_ / k; }

private:
    std::size_t n_;
    std::vector<double> re_, im_;
};

struct PlanKey {
    Radix radix;
    std::vector<std::size_t> dims;
    std::vector<Radix> radices = {};  // per-axis radices of a mixed plan (empty: all == radix)
    bool operator==(const PlanKey&) const = default;
};

class Plan {
public:
    Plan(Radix radix, TensorShape shape, int precision = PAFFT_F64, int device = -1)
        : radix_(radix), shape_(std::move(shape)) {
        pafft_plan_t h = nullptr;
        detail::check(pafft_plan_create(radix_value(radix), shape_.dims().data(), static_cast<int>(shape_.rank()),
                                        precision, device, &h));
        init(h, std::vector<Radix>(shape_.rank(), radix));
        key_ = PlanKey{radix_, shape_.dims()};
    }
    // Extension: one radix per axis.
    Plan(const std::vector<Radix>& radices, TensorShape shape, int precision = PAFFT_F64, int device = -1)
        : radix_(radices.empty() ? Radix::r2 : radices[0]), shape_(std::move(shape)) {
        if (radices.size() != shape_.rank()) throw Error("one radix per axis required");
        std::vector<unsigned> rs;
        for (Radix r : radices) rs.push_back(radix_value(r));
        pafft_plan_t h = nullptr;
        detail::check(pafft_plan_create_mixed(rs.data(), shape_.dims().data(), static_cast<int>(shape_.rank()),
                                              precision, device, &h));
        init(h, radices);
        key_ = PlanKey{radix_, shape_.dims(), radices};
    }
    Radix radix() const { return radix_; }
    Radix radix(std::size_t q) const { return radices_[q]; }
    const TensorShape& shape() const { return shape_; }
    std::size_t total() const { return shape_.total(); }
    unsigned depth(std::size_t q) const { return depths_[q]; }
    const TwiddleTable& twiddles(std::size_t q) const { return twiddles_[q]; }
    std::span<const std::uint32_t> rev_map(std::size_t q) const { return rev_maps_[q]; }
    const PlanKey& key() const { return key_; }
    pafft_plan_t handle() const { return h_.get(); }
    const std::shared_ptr<pafft_plan_s>& shared_handle() const { return h_; }

private:
    void init(pafft_plan_t h, const std::vector<Radix>& radices) {
        h_ = std::shared_ptr<pafft_plan_s>(h, [](pafft_plan_t p) { pafft_plan_destroy(p); });
        radices_ = radices;
        for (std::size_t q = 0; q < shape_.rank(); ++q) {
            const unsigned r = radix_value(radices[q]);
            const std::size_t n = shape_.dim(q);
            unsigned t = 0;
            for (std::size_t v = n; v > 1; v /= r) ++t;
            depths_.push_back(t);
            twiddles_.emplace_back(n);
            std::vector<std::uint32_t> rev(n);
            for (std::size_t j = 0; j < n; ++j) {
                std::uint64_t o = 0;
                pafft_digit_reverse(j, r, t, &o);
                rev[j] = static_cast<std::uint32_t>(o);
            }
            rev_maps_.push_back(std::move(rev));
        }
    }

    Radix radix_;
    std::vector<Radix> radices_;
    TensorShape shape_;
    std::shared_ptr<pafft_plan_s> h_;
    std::vector<unsigned> depths_;
    std::vector<TwiddleTable> twiddles_;
    std::vector<std::vector<std::uint32_t>> rev_maps_;
    PlanKey key_;
};

inline Plan plan_create(Radix radix, const TensorShape& shape) { return Plan(radix, shape); }
inline Plan plan_create(const std::vector<Radix>& radices, const TensorShape& shape) { return Plan(radices, shape); }

inline ComplexBuffer buffer_from_tensor(std::span<const std::complex<double>> values, const TensorShape& shape) {
    const std::size_t total = shape.total();
    if (values.size() != total) throw LengthMismatch(total, values.size());
    const std::size_t d = shape.rank();
    ComplexBuffer out(total);
    std::vector<std::size_t> row_stride(d, 1), idx(d, 0);
    for (std::size_t q = d; q-- > 1;) row_stride[q - 1] = row_stride[q] * shape.dim(q);
    std::size_t src = 0;
    for (std::size_t dst = 0; dst < total; ++dst) {
        out.re[dst] = values[src].real();
        out.im[dst] = values[src].imag();
        for (std::size_t q = 0; q < d; ++q) {
            src += row_stride[q];
            if (++idx[q] < shape.dim(q)) break;
            idx[q] = 0;
            src -= row_stride[q] * shape.dim(q);
        }
    }
    return out;
}

inline std::vector<std::complex<double>> tensor_from_buffer(const ComplexBuffer& x, const TensorShape& shape) {
    const std::size_t total = shape.total();
    if (x.size() != total) throw LengthMismatch(total, x.size());
    const std::size_t d = shape.rank();
    std::vector<std::complex<double>> out(total);
    std::vector<std::size_t> row_stride(d, 1), idx(d, 0);
    for (std::size_t q = d; q-- > 1;) row_stride[q - 1] = row_stride[q] * shape.dim(q);
    std::size_t dst = 0;
    for (std::size_t src = 0; src < total; ++src) {
        out[dst] = {x.re[src], x.im[src]};
        for (std::size_t q = 0; q < d; ++q) {
            dst += row_stride[q];
            if (++idx[q] < shape.dim(q)) break;
            idx[q] = 0;
            dst -= row_stride[q] * shape.dim(q);
        }
    }
    return out;
}

// ------------------------------------------------------- permutation.hpp
inline std::uint64_t digit_reverse(std::uint64_t j, unsigned radix, unsigned digits) {
    std::uint64_t out = 0;
    detail::check(pafft_digit_reverse(j, radix, digits, &out));
    return out;
}

inline void permute_tensor(ComplexBuffer& x, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), 5, x.re.data(), x.im.data(), 1));
}

inline void permute_1d(ComplexBuffer& x, const Plan& plan, std::size_t dim) {
    const std::size_t n = plan.shape().dim(dim);
    if (x.size() != n) throw ShapeMismatch(n, x.size());
    Plan line(plan.radix(), TensorShape{n});
    detail::check(pafft_transform_split(line.handle(), 5, x.re.data(), x.im.data(), 1));
}

inline std::uint64_t permutation_pass_count() { return pafft_permutation_pass_count(); }
inline void reset_permutation_pass_count() { pafft_reset_permutation_pass_count(); }

// --------------------------------------------------------- butterfly.hpp
enum class ButterflyVariant { forward, conjugate, transposed };

namespace detail {
inline int ladder_op(ButterflyVariant v) {
    return v == ButterflyVariant::forward ? 2 : v == ButterflyVariant::transposed ? 4 : 6;
}
}  // namespace detail

inline void butterfly_tensor(ComplexBuffer& x, const Plan& plan, ButterflyVariant variant) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), detail::ladder_op(variant), x.re.data(), x.im.data(), 1));
}

inline void butterfly_line(ComplexBuffer& x, const Plan& plan, std::size_t dim, ButterflyVariant variant) {
    const std::size_t n = plan.shape().dim(dim);
    if (x.size() != n) throw ShapeMismatch(n, x.size());
    if (n == 1) return;
    Plan line(plan.radix(), TensorShape{n});
    detail::check(pafft_transform_split(line.handle(), detail::ladder_op(variant), x.re.data(), x.im.data(), 1));
}
inline void butterfly_forward(ComplexBuffer& x, const Plan& p, std::size_t d) {
    butterfly_line(x, p, d, ButterflyVariant::forward);
}
inline void butterfly_conjugate(ComplexBuffer& x, const Plan& p, std::size_t d) {
    butterfly_line(x, p, d, ButterflyVariant::conjugate);
}
inline void butterfly_transposed(ComplexBuffer& x, const Plan& p, std::size_t d) {
    butterfly_line(x, p, d, ButterflyVariant::transposed);
}

// --------------------------------------------------------- transform.hpp
inline void fft_forward(ComplexBuffer& x, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), 0, x.re.data(), x.im.data(), 1));
}
inline void fft_backward(ComplexBuffer& x, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), 1, x.re.data(), x.im.data(), 1));
}
inline void fft_forward_unordered(ComplexBuffer& x, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), 2, x.re.data(), x.im.data(), 1));
}
inline void fft_backward_unordered(ComplexBuffer& x, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), 3, x.re.data(), x.im.data(), 1));
}

// ------------------------------------------------------- convolution.hpp
struct PreparedFilter {
    ComplexBuffer ghat;
    PlanKey key;
    std::shared_ptr<pafft_filter_s> device;  // the device copy the kernels read
};

inline PreparedFilter prepare_filter(const ComplexBuffer& g, const Plan& plan) {
    if (g.size() != plan.total()) throw LengthMismatch(plan.total(), g.size());
    pafft_filter_t f = nullptr;
    detail::check(pafft_prepare_filter_split(plan.handle(), g.re.data(), g.im.data(), &f));
    // the deleter keeps the creating plan alive as long as the filter
    auto keep = plan.shared_handle();
    PreparedFilter out{ComplexBuffer(plan.total()), plan.key(),
                       std::shared_ptr<pafft_filter_s>(f, [keep](pafft_filter_t h) { pafft_filter_destroy(h); })};
    detail::check(pafft_filter_ghat_split(f, out.ghat.re.data(), out.ghat.im.data()));
    return out;
}

inline ComplexBuffer filter_from_impulse(const ComplexBuffer& h, const Plan& plan) {
    if (h.size() != plan.total()) throw LengthMismatch(plan.total(), h.size());
    ComplexBuffer g(plan.total());
    detail::check(pafft_filter_from_impulse_split(plan.handle(), h.re.data(), h.im.data(), g.re.data(), g.im.data()));
    return g;
}

inline void hadamard_inplace(ComplexBuffer& x, const ComplexBuffer& y) {
    if (x.size() != y.size()) throw LengthMismatch(x.size(), y.size());
    for (std::size_t i = 0; i < x.size(); ++i) {
        const double r = x.re[i] * y.re[i] - x.im[i] * y.im[i];
        const double m = x.re[i] * y.im[i] + x.im[i] * y.re[i];
        x.re[i] = r;
        x.im[i] = m;
    }
}

inline void convolve_standard(ComplexBuffer& x, const ComplexBuffer& g, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    if (g.size() != plan.total()) throw LengthMismatch(plan.total(), g.size());
    detail::check(pafft_convolve_standard_split(plan.handle(), g.re.data(), g.im.data(), x.re.data(), x.im.data(), 1));
}

inline void convolve_permfree(ComplexBuffer& x, const PreparedFilter& filter, const Plan& plan) {
    if (!(filter.key == plan.key()) || !filter.device || !pafft_filter_matches(filter.device.get(), plan.handle()))
        throw FilterPlanMismatch();
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_convolve_permfree_split(plan.handle(), filter.device.get(), x.re.data(), x.im.data(), 1));
}

}  // namespace pafft
