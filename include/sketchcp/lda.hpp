// sketchcp drop-in (B200 build) — whitened third-moment sketch of
// proj/include/sketchcp/lda.hpp (sketch_whitened_m3 and the corpus types it consumes).
#pragma once

#include <vector>

#include "sketchcp/sketch.hpp"

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

StreamStats sketch_whitened_m3(const Corpus& c, const WhiteningMap& wm, double alpha0, SymTensorSketchSet& set);

}  // namespace sketchcp
