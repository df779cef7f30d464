// Kernel instantiation: generic sum of leaves padded to B = 8.
#include "launch_eval.cuh"

namespace spingp_host {
void eval_generic_8(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<GenericTraits<8>>(ctx, a); }
}  // namespace spingp_host
