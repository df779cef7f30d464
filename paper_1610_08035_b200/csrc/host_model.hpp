// host_model.hpp — host-side model setup for the device kernels (compiled by g++,
// C++20; used by the nvcc-compiled launch code through this plain interface).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "model_desc.h"
#include "spingp_c.h"

namespace spingp_host {

// Error carried to the C ABI boundary (status code + failing block).
struct ApiError {
    int status;
    int64_t block;
    std::string what;
};

struct HostModel {
    spingp_dev::ModelDesc desc{};
    int b = 0, nt = 0, rec_stride = 0;
    bool single_matern = false;
    std::vector<double> eqconst;  // shared per-model constants (EQ leaves)
};

// Validates the leaves and builds the device description (state_space_of,
// kernels.hpp:326-381, in the form the closed-form device discretisation needs).
HostModel build_model(const spingp_leaf* leaves, int32_t n_leaves, int32_t n_theta);

// Per-series record: sigma, jitter, d jitter / d theta, leaf params.
// Throws std::invalid_argument on non-positive hyperparameters (kernels.hpp:132-135).
void fill_record(const HostModel& hm, const double* theta, double sigma, double* rec);

// Level structure of the hierarchical reduction for S series of n points.
// tree: levels >= 1 are shared-memory tree groups of tree_group_size(Bsz) records
// (tree.cuh) and there is always at least one such level; otherwise the per-thread
// 4-record chunks of k_fwdL / k_revL (the materialised btd_core path, and the
// SPINGP_UPPER=coop|levels comparison knob).
struct Plan {
    spingp_dev::Geom geo{};
    bool tree = false;
};
// Upper-level scheme of the eval path: true = trees (default), false when
// SPINGP_UPPER=coop|levels.
bool upper_tree();
// g_override (testing knob): a smaller tree group size than tree_group_size(Bsz).
Plan make_plan(int64_t n, int64_t S, int Bsz, int64_t m0_override = 0, int tree = -1, int64_t g_override = 0);
// Resident threads of one level-0 reverse wave on the current device (occupancy query at
// context creation); make_plan's wave rule uses it.
void set_plan_wave(int64_t threads);

// predict at test times: the merged grid of n training points (strictly
// increasing t) and m test times (any order).  Test points carry no observation term
// (obs = 0, y = 0).  A test time at or before the previous grid time is nudged to that
// time + eps_t, eps_t = 1e-9 * (time span); a nudge that would reach the
// next grid time throws std::invalid_argument.
struct PredictGrid {
    std::vector<double> t, y;
    std::vector<unsigned char> obs;
    std::vector<int64_t> test_pos;  // merged index of test point k (input order)
};
PredictGrid predict_grid(const double* t, const double* y, int64_t n, const double* test_t, int64_t m);

// Padded block size with a kernel instantiation (1, 2, 3, 4, 6, 8, 12, 16).
int pad_b(int b);

// Models with a static-structure (compile-time offsets) instantiation.
enum StaticModel { SM_NONE = 0, SM_EQ6 = 1, SM_EQ10 = 2, SM_M32_QP6 = 3, SM_M32_EQ10 = 4 };
StaticModel static_model(const HostModel& hm);

}  // namespace spingp_host
