// Kernel instantiation: single Matérn leaf with state dimension 1 (registers only).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_matern_1(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<MaternTraits<1>>(ctx, a); }
}  // namespace spingp_host
