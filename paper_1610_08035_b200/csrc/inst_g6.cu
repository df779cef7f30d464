// Kernel instantiation: generic sum of leaves padded to B = 6.
#include "launch_eval.cuh"

namespace spingp_host {
void eval_generic_6(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<GenericTraits<6>>(ctx, a); }
}  // namespace spingp_host
