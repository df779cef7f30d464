// Kernel instantiation: static-structure model StaticTraits<SMatern<2>, SQP<6>> (compile-time leaf offsets).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_s_m32qp6(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<StaticTraits<SMatern<2>, SQP<6>>>(ctx, a); }
}  // namespace spingp_host
