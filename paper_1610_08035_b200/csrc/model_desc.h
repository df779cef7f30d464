// model_desc.h — plain-C++ description of a state-space model as the device
// kernels see it (shared by the g++-compiled host model code and the nvcc
// device code; no CUDA types).
#pragma once

namespace spingp_dev {

constexpr int kMaxLeaves = 8;
constexpr int kMaxB = 16;
constexpr int kMaxTheta = 2 + 4 * kMaxLeaves;

enum LeafType { MATERN12 = 0, MATERN32 = 1, MATERN52 = 2, EQ = 3, QP = 4 };

struct ModelDesc {
    int b;           // true state dimension (kernels may be instantiated for a padded B)
    int nleaves;
    int nt;          // kernel hyperparameters (sigma excluded)
    int rec_stride;  // doubles per series record
    int type[kMaxLeaves], off[kMaxLeaves], dim[kMaxLeaves], order[kMaxLeaves];
    int rec[kMaxLeaves], th[kMaxLeaves], eqc[kMaxLeaves];
    double H[kMaxB];
    const double* eqconst;  // per EQ leaf at eqc[l]: (a_p, c_p) p < J/2, then P1[J*J]
};

constexpr int kMaxLev = 24;

// Level structure of the hierarchical reduction (host-planned, passed to kernels).
struct Geom {
    int nlev;                  // number of reduction levels (level nlev-1 has K = 1)
    int S;                     // independent series
    long long n[kMaxLev + 1];  // blocks per series at each level (n[0] = points)
    long long K[kMaxLev];      // chunks per series at each level
    int m[kMaxLev];            // chunk length at each level
    // segment mode (multi-GPU partition of one long series): the first
    // block couples to a left separator held by the previous rank (segL) and the last
    // block's diagonal includes the step to the next rank's first time (segR).
    int segL, segR;
};

// Levels >= 1 as CTA-wide binary trees in shared memory (tree.cuh): a level-l group is
// G(B) consecutive level-(l-1) records of one series.  G is the largest power of two
// (<= 512, two records per thread of a 256-thread CTA) whose records plus separators fit
// the 227 KB opt-in shared memory of a CTA (component-major rows of even length).
constexpr long long kTreeSmemCap = 232448 - 2048;
constexpr long long tree_row(long long n) { return (n + 1) & ~1LL; }
constexpr long long tree_smem_bytes(int B, long long G) {
    return 8 * ((3 * B * B + 2 * B + 1) * tree_row(G) + (B + 2 * B * B) * tree_row(G + 1));
}
constexpr int tree_group_size(int B) {
    int G = 512;
    while (G > 2 && tree_smem_bytes(B, G) > kTreeSmemCap) G >>= 1;
    return G;
}

}  // namespace spingp_dev
