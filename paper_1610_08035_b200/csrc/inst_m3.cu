// Kernel instantiation: single Matérn leaf with state dimension 3 (registers only).
#include "launch_eval.cuh"

namespace spingp_host {
void eval_matern_3(spingp_ctx* ctx, const EvalArgs& a) { launch_eval<MaternTraits<3>>(ctx, a); }
// resident threads of one k_rev0 wave at b = 3 on the current device (make_plan's wave rule)
int64_t rev0_wave_threads_m3() {
    int per = 0, dev = 0, sms = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rev0<MaternTraits<3>>, 128, 0));
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return static_cast<int64_t>(std::max(1, per)) * sms * 128;
}
}  // namespace spingp_host
