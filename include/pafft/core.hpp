// pafft/core.hpp -- drop-in for the reference's core types (reference
// include/pafft/core.hpp:14-139): Radix, TensorShape, ComplexBuffer,
// TwiddleTable, PlanKey, Plan, plan_create and the C-order <-> vec repack.
// Header-only over the C ABI (include/pafft_b200.h, libpafft_b200.so): a Plan
// owns a device plan (twiddle tables and pass schedule in HBM) and keeps the
// reference's host-side accessors (depth, twiddles, rev_map, key).
//
// Supersets of the reference, none of which change its behaviour: Radix also
// has r3 and r5; Plan takes an optional precision and device, and a per-axis
// radix list.  Link with -lpafft_b200 -lcudart.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <memory>
#include <numbers>
#include <span>
#include <string>
#include <vector>

#include "../pafft_b200.h"
#include "errors.hpp"

namespace pafft {

namespace detail {
// A C-ABI status rethrown as the matching reference exception class.
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

enum class Radix : unsigned { r2 = 2, r3 = 3, r4 = 4, r5 = 5, r8 = 8 };

constexpr unsigned radix_value(Radix r) { return static_cast<unsigned>(r); }

inline Radix radix_from_value(unsigned value) {
    switch (value) {
        case 2: return Radix::r2;
        case 3: return Radix::r3;
        case 4: return Radix::r4;
        case 5: return Radix::r5;
        case 8: return Radix::r8;
        default: throw Error("unsupported radix " + std::to_string(value) + " (2, 3, 4, 5 or 8)");
    }
}

// Extents n_1..n_d; the FIRST index varies fastest in memory (vec layout).
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

// Split-complex host storage of vec(X).
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
    for (std::size_t i = 0; i < x.size(); ++i) m = std::max(m, std::hypot(x.re[i], x.im[i]));
    return m;
}

inline void scale_inplace(ComplexBuffer& x, double s) {
    std::transform(x.re.begin(), x.re.end(), x.re.begin(), [s](double v) { return v * s; });
    std::transform(x.im.begin(), x.im.end(), x.im.begin(), [s](double v) { return v * s; });
}

// Host copy of the reference's master root table w[j] = exp(-2 pi i j / n);
// the device kernels use their own per-pass tables.
class TwiddleTable {
public:
    explicit TwiddleTable(std::size_t n) : n_(n), re_(n), im_(n) {
        for (std::size_t j = 0; j < n; ++j) {
            const double a = -2.0 * std::numbers::pi * static_cast<double>(j) / static_cast<double>(n);
            re_[j] = std::cos(a);
            im_[j] = std::sin(a);
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
    std::vector<Radix> radices = {};  // per-axis radices of a mixed plan (empty: every axis uses `radix`)
    bool operator==(const PlanKey&) const = default;
};

// A device plan plus the reference's host accessors.  Immutable; copies
// share the device plan; safe to use from several threads at once.
class Plan {
public:
    Plan(Radix radix, TensorShape shape, int precision = PAFFT_F64, int device = -1)
        : radix_(radix), shape_(std::move(shape)) {
        pafft_plan_t h = nullptr;
        detail::check(pafft_plan_create(radix_value(radix), shape_.dims().data(), static_cast<int>(shape_.rank()),
                                        precision, device, &h));
        adopt(h, std::vector<Radix>(shape_.rank(), radix));
        key_ = PlanKey{radix_, shape_.dims()};
    }
    Plan(const std::vector<Radix>& radices, TensorShape shape, int precision = PAFFT_F64, int device = -1)
        : radix_(radices.empty() ? Radix::r2 : radices.front()), shape_(std::move(shape)) {
        if (radices.size() != shape_.rank()) throw Error("a mixed plan needs one radix per axis");
        std::vector<unsigned> rs(radices.size());
        std::transform(radices.begin(), radices.end(), rs.begin(), radix_value);
        pafft_plan_t h = nullptr;
        detail::check(pafft_plan_create_mixed(rs.data(), shape_.dims().data(), static_cast<int>(shape_.rank()),
                                              precision, device, &h));
        adopt(h, radices);
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
    void adopt(pafft_plan_t h, const std::vector<Radix>& radices) {
        h_ = std::shared_ptr<pafft_plan_s>(h, [](pafft_plan_t p) { pafft_plan_destroy(p); });
        radices_ = radices;
        std::vector<unsigned> depth(shape_.rank());
        detail::check(pafft_plan_info(h, nullptr, nullptr, nullptr, depth.data(), nullptr, nullptr, nullptr));
        for (std::size_t q = 0; q < shape_.rank(); ++q) {
            const std::size_t n = shape_.dim(q);
            depths_.push_back(depth[q]);
            twiddles_.emplace_back(n);
            std::vector<std::uint32_t> rev(n);
            for (std::size_t j = 0; j < n; ++j) {
                std::uint64_t o = 0;
                detail::check(pafft_digit_reverse(j, radix_value(radices[q]), depth[q], &o));
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

// Throws EmptyShape / NotAPowerOfRadix like the reference (core.cpp:93-129).
inline Plan plan_create(Radix radix, const TensorShape& shape) { return Plan(radix, shape); }
inline Plan plan_create(const std::vector<Radix>& radices, const TensorShape& shape) { return Plan(radices, shape); }

namespace detail {
// Walks a shape's multi-indices in C order (last index fastest) and calls
// f(c_offset, vec_offset) for each, where vec_offset = sum_q i_q * prod_{p<q} n_p.
template <class F>
void walk_c_order(const TensorShape& shape, F&& f) {
    const std::size_t d = shape.rank(), total = shape.total();
    std::vector<std::size_t> vstride(d), idx(d, 0);
    std::size_t acc = 1;
    for (std::size_t q = 0; q < d; ++q) {
        vstride[q] = acc;
        acc *= shape.dim(q);
    }
    std::size_t v = 0;
    for (std::size_t c = 0; c < total; ++c) {
        f(c, v);
        for (std::size_t q = d; q-- > 0;) {  // advance the C-order counter
            if (++idx[q] < shape.dim(q)) {
                v += vstride[q];
                break;
            }
            v -= vstride[q] * (shape.dim(q) - 1);
            idx[q] = 0;
        }
    }
}
}  // namespace detail

// C-order (numpy) values -> vec-order buffer, and back.
inline ComplexBuffer buffer_from_tensor(std::span<const std::complex<double>> values, const TensorShape& shape) {
    if (values.size() != shape.total()) throw LengthMismatch(shape.total(), values.size());
    ComplexBuffer out(shape.total());
    detail::walk_c_order(shape, [&](std::size_t c, std::size_t v) { out.set(v, values[c]); });
    return out;
}

inline std::vector<std::complex<double>> tensor_from_buffer(const ComplexBuffer& x, const TensorShape& shape) {
    if (x.size() != shape.total()) throw LengthMismatch(shape.total(), x.size());
    std::vector<std::complex<double>> out(shape.total());
    detail::walk_c_order(shape, [&](std::size_t c, std::size_t v) { out[c] = x.get(v); });
    return out;
}

}  // namespace pafft
