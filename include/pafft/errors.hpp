// pafft/errors.hpp -- drop-in for the reference's error classes
// (reference include/pafft/errors.hpp:10-44): every error is a pafft::Error,
// with the same class names, constructor arguments and public fields, so
// caller code that throws or catches them compiles unchanged.  Each class
// also takes a ready message: the C-ABI status (include/pafft_b200.h) is
// rethrown with the library's own text by pafft::detail::check (core.hpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace pafft {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// An extent n_q that is not a power of the plan radix (dim is 0-based).
struct NotAPowerOfRadix : Error {
    NotAPowerOfRadix(std::size_t dim_, std::size_t extent_, unsigned radix)
        : Error("extent " + std::to_string(extent_) + " of dimension " + std::to_string(dim_) +
                " is not a power of radix " + std::to_string(radix)),
          dim(dim_),
          extent(extent_) {}
    NotAPowerOfRadix(std::size_t dim_, std::size_t extent_, const std::string& message)
        : Error(message), dim(dim_), extent(extent_) {}
    std::size_t dim;
    std::size_t extent;
};

// A rank-0 shape where a tensor is required.
struct EmptyShape : Error {
    EmptyShape() : Error("a tensor shape needs at least one dimension") {}
    explicit EmptyShape(const std::string& message) : Error(message) {}
};

// Buffer length differs from the plan total (or from the other operand).
struct LengthMismatch : Error {
    LengthMismatch(std::size_t expected, std::size_t got)
        : Error("length mismatch: want " + std::to_string(expected) + " elements, have " + std::to_string(got)) {}
    explicit LengthMismatch(const std::string& message) : Error(message) {}
};

// A line buffer whose length is not the extent of the dimension it is run as.
struct ShapeMismatch : Error {
    ShapeMismatch(std::size_t expected, std::size_t got)
        : Error("line length mismatch: dimension extent " + std::to_string(expected) + ", line has " +
                std::to_string(got)) {}
    explicit ShapeMismatch(const std::string& message) : Error(message) {}
};

// A prepared filter used under a plan it was not prepared for.
struct FilterPlanMismatch : Error {
    FilterPlanMismatch() : Error("prepared filter belongs to a different plan") {}
    explicit FilterPlanMismatch(const std::string& message) : Error(message) {}
};

// An index outside [0, bound) of a digit permutation.
struct IndexOutOfRange : Error {
    IndexOutOfRange(std::uint64_t index, std::uint64_t bound)
        : Error("index " + std::to_string(index) + " outside [0, " + std::to_string(bound) + ")") {}
    explicit IndexOutOfRange(const std::string& message) : Error(message) {}
};

}  // namespace pafft
