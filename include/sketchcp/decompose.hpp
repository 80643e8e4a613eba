// sketchcp drop-in (B200 build) — fast drivers of proj/include/sketchcp/decompose.hpp:
// the robust tensor power method (Algorithm 1: batched restarts on the device, lowest-tau
// tie rule, rank-1 sketch deflation) and fast CP-ALS on the asymmetric sketch set
// (batched sketched mode contractions). The exact O(n^3) drivers are outside this build.
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

struct AlsConfig {
    int k = 1;
    int max_iters = 1000;
    double tol = 1e-6;  // relative change of the lambda vector
    std::uint32_t b = 4096;
    int B = 40;
    std::uint64_t seed = 0;
};

CpDecomposition robust_tpm_fast(SymTensorSketchSet& set, const PowerConfig& cfg);

/// CP-ALS where each factor column update reads T(., b_i, c_i) off the asymmetric
/// sketch set (decompose.cpp:117-205).
CpDecomposition als_fast(const AsymTensorSketchSet& set, const AlsConfig& cfg);

/// Symmetric pseudoinverse with spectral truncation at 1e-10 of the largest |eigenvalue|
/// (decompose.cpp:44-51).
Eigen::MatrixXd pinv_spectral(const Eigen::MatrixXd& G);

}  // namespace sketchcp
