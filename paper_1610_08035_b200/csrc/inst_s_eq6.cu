// Kernel instantiation: static-structure model StaticTraits<SEQ<6>> (compile-time leaf offsets).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_s_eq6(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<StaticTraits<SEQ<6>>>(ctx, a); }
}  // namespace spingp_host
