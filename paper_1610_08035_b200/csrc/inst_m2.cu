// Kernel instantiation: single Matérn leaf with state dimension 2 (registers only).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_matern_2(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<MaternTraits<2>>(ctx, a); }
}  // namespace spingp_host
