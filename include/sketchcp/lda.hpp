// sketchcp drop-in (B200 build) — whitened third-moment sketch of
// proj/include/sketchcp/lda.hpp (sketch_whitened_m3 and the corpus types it consumes).
#pragma once

#include <vector>

#include "sketchcp/sketch.hpp"
#include "sketchcp/tensor.hpp"

namespace sketchcp {

struct Document {
    std::vector<int> word;
    std::vector<int> count;
    long long total = 0;
};

struct Corpus {
    int V = 0;
    std::vector<Document> docs;
    long long total_tokens() const;
};

struct WhiteningMap {
    Eigen::MatrixXd W;
    Eigen::MatrixXd unwhiten;
    Eigen::VectorXd singular_values;
};

struct StreamStats {
    long long used = 0;
    long long skipped = 0;
};

struct LdaModel {
    Eigen::MatrixXd Phi;    // V x k, column-stochastic
    Eigen::VectorXd alpha;  // positive
    double alpha0() const { return alpha.sum(); }
    int vocab() const { return static_cast<int>(Phi.rows()); }
    int topics() const { return static_cast<int>(Phi.cols()); }
};

/// Mean normalized word frequency over documents (lda.cpp:88-100; GPU).
Eigen::VectorXd compute_m1(const Corpus& c);

/// Unbiased within-document pair moment minus the alpha0/(alpha0+1) rank-1 correction
/// (lda.cpp:102-123). Dense V x V like the reference: formed on the GPU by applying the
/// implicit operator to identity blocks. Prefer whiten_corpus for large vocabularies.
Eigen::MatrixXd compute_m2(const Corpus& c, double alpha0);

/// whiten(m2hat, k) (lda.cpp:125-143): top-k eigenpairs by randomized subspace iteration
/// (GPU, DGEMM operator); eigenvector signs are unpinned as in Eigen.
WhiteningMap whiten(const Eigen::MatrixXd& m2hat, int k);

/// B200 extension: whiten(compute_m2(c, alpha0), k) without forming M2 (V up to ~1e5+).
WhiteningMap whiten_corpus(const Corpus& c, double alpha0, int k);

StreamStats sketch_whitened_m3(const Corpus& c, const WhiteningMap& wm, double alpha0, SymTensorSketchSet& set);

/// lda.cpp:228-248
LdaModel recover_params(const CpDecomposition& D, const WhiteningMap& wm, double alpha0);

/// lda.cpp:250-271
Eigen::VectorXd project_to_simplex(const Eigen::VectorXd& y);

/// lda.cpp:273-320
double heldout_likelihood(const LdaModel& m, const Corpus& held, long long* floored_words = nullptr);

}  // namespace sketchcp
