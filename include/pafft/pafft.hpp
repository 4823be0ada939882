// pafft/pafft.hpp -- umbrella header of the C++ drop-in for the reference
// library's public API.  The per-module headers mirror the reference's
// (include/pafft/{errors,core,permutation,butterfly,transform,convolution}.hpp),
// so reference code that includes "pafft/convolution.hpp" etc. compiles
// unchanged against them; everything runs on the B200 through the C ABI
// (include/pafft_b200.h).  Link with -lpafft_b200 -lcudart.
#pragma once

#include "butterfly.hpp"
#include "convolution.hpp"
#include "core.hpp"
#include "errors.hpp"
#include "permutation.hpp"
#include "transform.hpp"
