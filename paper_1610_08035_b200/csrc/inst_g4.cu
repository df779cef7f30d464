// Kernel instantiation: generic sum of leaves padded to B = 4.
#include "launch_eval.cuh"

namespace spingp_host {
void eval_generic_4(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<GenericTraits<4>>(ctx, a); }
}  // namespace spingp_host
