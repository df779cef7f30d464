// btd_core instantiation for blocks padded to B = 8.
#include "btd_ops.cuh"

namespace spingp_host {
void btd_run_8(spingp_ctx* ctx, int64_t n, int b, const double* diag, const double* upper, const double* rhs,
              int k, int col, double* x, double* cdiag, double* cupper, double* logdet, bool needC) {
    launch_btd<8>(ctx, n, b, diag, upper, rhs, k, col, x, cdiag, cupper, logdet, needC);
}
}  // namespace spingp_host
