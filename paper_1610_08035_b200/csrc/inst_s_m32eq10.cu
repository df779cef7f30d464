// Kernel instantiation: static-structure model StaticTraits<SMatern<2>, SEQ<10>> (compile-time leaf offsets).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_s_m32eq10(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<StaticTraits<SMatern<2>, SEQ<10>>>(ctx, a); }
}  // namespace spingp_host
