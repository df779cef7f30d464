// Kernel instantiation: generic sum of leaves padded to B = 16.
#include "launch_eval.cuh"

namespace spingp_host {
void eval_generic_16(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<GenericTraits<16>>(ctx, a); }
}  // namespace spingp_host
