// Kernel instantiation: generic sum of leaves padded to B = 12.
#include "launch_eval.cuh"

namespace spingp_host {
void eval_generic_12(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<GenericTraits<12>>(ctx, a); }
}  // namespace spingp_host
