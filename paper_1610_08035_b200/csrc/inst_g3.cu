// Kernel instantiation: generic sum of leaves padded to B = 3.
#include "launch_eval.cuh"

namespace spingp_host {
void eval_generic_3(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<GenericTraits<3>>(ctx, a); }
}  // namespace spingp_host
