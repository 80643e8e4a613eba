// sketchcp drop-in (B200 build) — fast robust tensor power method of
// proj/include/sketchcp/decompose.hpp (Algorithm 1): batched restarts on the device,
// lowest-tau tie rule, rank-1 sketch deflation. (ALS and the exact drivers are outside
// this build's scope.)
#pragma once

#include "sketchcp/contraction.hpp"
#include "sketchcp/tensor.hpp"

namespace sketchcp {

struct PowerConfig {
    int k = 1;
    int L = 30;
    int T_iters = 30;
    std::uint32_t b = 4096;
    int B = 20;
    std::uint64_t seed = 0;
    double tol = 1e-12;
};

CpDecomposition robust_tpm_fast(SymTensorSketchSet& set, const PowerConfig& cfg);

}  // namespace sketchcp
