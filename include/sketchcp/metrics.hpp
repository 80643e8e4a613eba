// sketchcp drop-in (B200 build) — recovery metrics of proj/include/sketchcp/metrics.hpp.
#pragma once

#include <vector>

#include <Eigen/Core>

namespace sketchcp {

struct VectorMatch {
    int recovered;
    int truth;
    double cosine;
    double sq_distance;
};

std::vector<VectorMatch> greedy_match(const Eigen::MatrixXd& recovered, const Eigen::MatrixXd& truth);
int wrong_vector_count(const std::vector<VectorMatch>& matches, double threshold = 0.1);

}  // namespace sketchcp
