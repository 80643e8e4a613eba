// sketchcp drop-in (B200 build) — FFT entry points of proj/include/sketchcp/fft.hpp.
// Same semantics (forward unnormalised e^{-2 pi i tk/b}; inverse scaled by 1/b or
// unscaled; power-of-two lengths), executed by the sm_100a residue-split FFT.
#pragma once

#include <cstdint>

#include "sketchcp/common.hpp"

namespace sketchcp::fft {

void forward_inplace(cvec& x);
void inverse_inplace(cvec& x);
void inverse_inplace_unscaled(cvec& x);
cvec circular_convolve(const cvec& x, const cvec& y);
std::uint64_t transform_count();

}  // namespace sketchcp::fft
