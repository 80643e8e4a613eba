// sketchcp drop-in (B200 build) — sketched contractions of
// proj/include/sketchcp/contraction.hpp, evaluated by the fused sm_100a kernels. The
// cached forward transform of each replicate is kept on the device and refreshed when
// the set's version moves; cached_transform(m) returns a host copy in natural order.
#pragma once

#include <vector>

#include "sketchcp/sketch.hpp"

namespace sketchcp {

class SymContractionWorkspace {
public:
    explicit SymContractionWorkspace(const SymTensorSketchSet& set);
    double vvv(const Eigen::VectorXd& u);
    Eigen::VectorXd Ivv(const Eigen::VectorXd& u);
    const cvec& cached_transform(int m);
    const SymTensorSketchSet& set() const { return *set_; }

private:
    const SymTensorSketchSet* set_;
    std::vector<cvec> spectra_;
};

class AsymContractionWorkspace {
public:
    explicit AsymContractionWorkspace(const AsymTensorSketchSet& set);
    double vvv(const Eigen::VectorXd& u);
    Eigen::VectorXd Ivv(const Eigen::VectorXd& u);
    Eigen::VectorXd Ibc(const Eigen::VectorXd& bvec, const Eigen::VectorXd& cvec_);
    Eigen::VectorXd mode_contraction(int free_mode, const Eigen::VectorXd& x, const Eigen::VectorXd& y);
    const cvec& cached_transform(int m);
    const AsymTensorSketchSet& set() const { return *set_; }

private:
    const AsymTensorSketchSet* set_;
    std::vector<cvec> spectra_;
};

}  // namespace sketchcp
