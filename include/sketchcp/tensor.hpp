// sketchcp drop-in (B200 build) — tensor input/output types of the hot path.
// Layout and semantics of proj/include/sketchcp/tensor.hpp: DenseTensor3 is row-major
// (i,j,k) at (i*n + j)*n + k; CpDecomposition stores lambda and unit factor columns.
// (The exact O(n^3) contractions, synthetic generators and COO I/O of the reference are
// outside this build's scope.)
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <vector>

#include <Eigen/Core>

#include "sketchcp/common.hpp"

namespace sketchcp {

struct DenseTensor3 {
    int n = 0;
    std::vector<double> entries;

    DenseTensor3() = default;
    explicit DenseTensor3(int dim)
        : n(dim), entries(static_cast<std::size_t>(dim) * dim * dim, 0.0) {}
    double& at(int i, int j, int k) { return entries[(static_cast<std::size_t>(i) * n + j) * n + k]; }
    double at(int i, int j, int k) const { return entries[(static_cast<std::size_t>(i) * n + j) * n + k]; }
    double frobenius_sq() const;
    bool is_symmetric(double tol = 0.0) const;
    std::optional<std::array<int, 3>> first_asymmetric_triple(double tol = 0.0) const;
};

struct Triple {
    int i, j, k;
    double value;
};

struct FactoredTensor {
    struct Component {
        double weight;
        Eigen::VectorXd u, v, w;
    };
    int n = 0;
    bool symmetric = false;
    std::vector<Component> components;

    void add(double a, Eigen::VectorXd u, Eigen::VectorXd v, Eigen::VectorXd w);
    void add_symmetric(double a, Eigen::VectorXd u);
};

struct CpDecomposition {
    Eigen::VectorXd lambda;
    Eigen::MatrixXd A, B, C;

    int rank() const { return static_cast<int>(lambda.size()); }
    int dim() const { return static_cast<int>(A.rows()); }
    bool symmetric() const { return B.size() == 0 || B.data() == A.data(); }
    static CpDecomposition symmetric_of(Eigen::VectorXd lambda, Eigen::MatrixXd V);
};

}  // namespace sketchcp
