// Kernel instantiation: single Matérn leaf with state dimension 3 (registers only).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_matern_3(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<MaternTraits<3>>(ctx, a); }
}  // namespace spingp_host
