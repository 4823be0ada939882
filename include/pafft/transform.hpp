// pafft/transform.hpp -- drop-in for the reference's transforms (reference
// include/pafft/transform.hpp:7-19, transform.cpp:8-26): natural-order
// forward/backward DFTs (one digit-reversal pass + ladders; backward scaled by
// 1/N) and the ladder-only "unordered" forms.  fft_forward(x) is bit-for-bit
// permute_tensor(x) followed by fft_forward_unordered(x): the device runs the
// same reordering kernel and the same pass kernels in both.
#pragma once

#include "core.hpp"

namespace pafft {

namespace detail {
inline void transform(ComplexBuffer& x, const Plan& plan, int op) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    check(pafft_transform_split(plan.handle(), op, x.re.data(), x.im.data(), 1));
}
}  // namespace detail

inline void fft_forward(ComplexBuffer& x, const Plan& plan) { detail::transform(x, plan, 0); }
inline void fft_backward(ComplexBuffer& x, const Plan& plan) { detail::transform(x, plan, 1); }
inline void fft_forward_unordered(ComplexBuffer& x, const Plan& plan) { detail::transform(x, plan, 2); }
inline void fft_backward_unordered(ComplexBuffer& x, const Plan& plan) { detail::transform(x, plan, 3); }

}  // namespace pafft
