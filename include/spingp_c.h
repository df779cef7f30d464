/*
 * spingp_c.h — the C ABI of the B200-native SpInGP sparse-precision inference path.
 *
 * This is the drop-in boundary: plain pointers, sizes and
 * status codes, no C++ or torch types.  The C++ header API in include/spingp/
 * (the reference's `spingp` namespace) is implemented on top of it, and any
 * FFI (ctypes, cgo, JNI) binds these symbols directly.
 *
 * Which reference interface each entry point replaces (file:line under the
 * read-only reference tree):
 *   spingp_state_space        state_space_of            proj/include/spingp/kernels.hpp:326-381
 *   (discretize / discretize_with_grad, kernels.hpp:392-443, stay host-side C++ in
 *    include/spingp/kernels.hpp; on the device they are fused into spingp_eval)
 *   spingp_eval[_device]      log_marginal_likelihood + mll_gradient + predict (training grid)
 *                                                       SPEC.md:280-306 (assemble :262-279)
 *   spingp_eval_batched[...]  the same over many independent series (BASELINE cfg3)
 *   spingp_assemble[_device]  assemble_prior_precision + add_observation_term
 *   spingp_btd_cr_solve[...]  cr_solve (+ solve/logdet)
 *   spingp_btd_selinv[...]    selective_inverse
 *   spingp_btd_matvec[...]    matvec
 *   spingp_mctx_create + spingp_eval_partitioned   the multi-GPU (NCCL) partition of one
 *                             long series; data-parallel cr_solve contract SPEC.md:200,224
 *   spingp_btd_factorize / _factor_{solve,selinv,blocks}   BTDFactor + factorize / solve /
 *                             selective_inverse on a kept factor
 * Error convention: every function returns a spingp_status; NOT_PD carries the
 * failing block index through `fail_block` (errors.hpp:12-20 NotPositiveDefinite),
 * SINGULAR_Q likewise (errors.hpp:23-27 SingularProcessNoise).  The C++ layer
 * rethrows the reference exception types.
 *
 * Memory: the caller owns every buffer.  Functions without a `_device` suffix
 * take HOST pointers and are synchronous (host->device copies, kernels,
 * device->host copies inside the call).  `_device` variants take DEVICE
 * pointers, enqueue on the context's stream and return immediately; device-side
 * failures are then reported by spingp_ctx_status().
 *
 * Layouts: all matrices are row-major; a block-tridiagonal (BTD) matrix of n
 * blocks of size b is stored as diag[n][b][b] and upper[n-1][b][b] (upper[i] is
 * the (i, i+1) block; the (i+1, i) block is its transpose) — SPEC.md:129-134,220.
 * Vectors over blocks are x[n][b] (times k right-hand sides: x[n*b][k]).
 */
#ifndef SPINGP_C_H
#define SPINGP_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPINGP_ABI_VERSION 1

typedef enum {
    SPINGP_OK = 0,
    SPINGP_NOT_PD = 1,          /* a Cholesky pivot failed (NotPositiveDefinite)            */
    SPINGP_SINGULAR_Q = 2,      /* a process-noise block stayed singular after jitter       */
    SPINGP_BAD_ARG = 3,         /* invalid argument (std::invalid_argument)                 */
    SPINGP_CUDA_ERR = 4,        /* CUDA runtime failure                                     */
    SPINGP_NCCL_ERR = 5,        /* NCCL failure                                             */
    SPINGP_DUPLICATE_TIME = 6,  /* two training times coincide (DuplicateTimestamp)         */
    SPINGP_UNSUPPORTED = 7,     /* configuration not implemented by this build              */
    SPINGP_NEG_VARIANCE = 8     /* a posterior variance fell below -1e-10     */
} spingp_status;

/* Kernel leaves.  Matérn-ν and EQ follow kernels.hpp:17-49; QP (quasi-periodic:
 * periodic with J harmonics x Matérn-1/2 envelope, Solin & Särkkä 2014) is the
 * extension BASELINE cfg5 needs and the reference lacks. */
typedef enum {
    SPINGP_MATERN12 = 0,
    SPINGP_MATERN32 = 1,
    SPINGP_MATERN52 = 2,
    SPINGP_EQ = 3,
    SPINGP_QP = 4
} spingp_leaf_type;

/* One leaf of a sum kernel.  `order`: EQ approximation order (even, 2..16);
 * QP number of harmonics J (state dimension 2(J+1)); ignored for Matérn.
 * Hyperparameters, in the reference's traversal order (kernels.hpp:84-107):
 *   Matérn, EQ : (var, len)
 *   QP         : (var, len, period, env)   len = periodic smoothness ℓ_p,
 *                                          env = envelope lengthscale ℓ_e      */
typedef struct {
    int32_t type;
    int32_t order;
} spingp_leaf;

/* flags for the evaluation entry points */
#define SPINGP_WANT_LOGLIK 0u      /* always computed                                   */
#define SPINGP_WANT_GRAD 1u        /* d loglik / d(theta..., sigma), raw parameters     */
#define SPINGP_WANT_MEAN 2u        /* posterior mean H mu_i at the training times       */
#define SPINGP_WANT_VAR 4u         /* posterior latent variance H C_ii H^T              */
#define SPINGP_INCLUDE_NOISE 8u    /* add sigma^2 to the variances                      */

typedef struct spingp_ctx spingp_ctx;

int spingp_abi_version(void);
const char* spingp_status_string(int status);
/* Message of the last failure on the calling thread. */
const char* spingp_last_error(void);

/* ---- host-side model setup (no GPU needed) ------------------------------------ */

/* b (state dimension) and n_theta (kernel hyperparameters, excluding sigma). */
int spingp_kernel_dims(const spingp_leaf* leaves, int32_t n_leaves, int32_t* b, int32_t* n_theta);

/* state_space_of (kernels.hpp:326-381): F[b*b], H[b], Pinf[b*b], dF[n_theta*b*b],
 * dPinf[n_theta*b*b], f_constant[n_theta]; any output may be NULL. */
int spingp_state_space(const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                       int32_t n_theta, double* F, double* H, double* Pinf, double* dF,
                       double* dPinf, int32_t* f_constant);

/* ---- context ------------------------------------------------------------------- */

int spingp_ctx_create(int32_t device, spingp_ctx** out);
int spingp_ctx_destroy(spingp_ctx* ctx);
/* Use an external CUDA stream (cudaStream_t passed as void*).  As in the CUDA
 * runtime, NULL is the legacy default stream (torch's default current stream). */
int spingp_ctx_set_stream(spingp_ctx* ctx, void* stream);
/* Go back to the context's own private non-blocking stream. */
int spingp_ctx_use_own_stream(spingp_ctx* ctx);
void* spingp_ctx_get_stream(spingp_ctx* ctx);
/* Synchronise the context's stream and return the first device-side failure of
 * the work enqueued since the previous call (and its block index). */
int spingp_ctx_status(spingp_ctx* ctx, int64_t* fail_block);
/* Number of kernel launches this context has issued so far. */
int64_t spingp_ctx_launch_count(spingp_ctx* ctx);
/* Tuning/testing knob: force the level-0 chunk length (0 = automatic). */
int spingp_ctx_set_chunk(spingp_ctx* ctx, int64_t m0);
/* Testing knob: cap the records per shared-memory tree group of levels >= 1
 * (0 = automatic, the largest that fits a CTA; >= 2 forces more tree levels). */
int spingp_ctx_set_tree_group(spingp_ctx* ctx, int64_t g);
/* Diagnostics: bracket every kernel launch with CUDA events (on the context's
 * stream) and report them: spingp_ctx_kernel_times synchronises, returns up to
 * `cap` (name, milliseconds) pairs in launch order and clears the record. */
int spingp_ctx_set_profiling(spingp_ctx* ctx, int on);
/* Diagnostics: a device buffer of >= 64 uint64 that the fused upper-level kernel fills
 * with %globaltimer stamps at every phase boundary (NULL = off). */
int spingp_ctx_set_phase_stamps(spingp_ctx* ctx, void* d_stamps);
int spingp_ctx_kernel_times(spingp_ctx* ctx, const char** names, double* ms, int32_t cap,
                            int32_t* count);

/* ---- the hot path: discretise -> assemble -> partitioned BTD factor/solve/selinv
 *      -> loglik, gradient, posterior mean/var, fused on the device ------------- */

int spingp_eval(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                const double* theta, int32_t n_theta, const double* t, const double* y,
                int64_t n, double sigma, uint32_t flags, double* out_loglik,
                double* out_grad /* n_theta+1 */, double* out_mean /* n */,
                double* out_var /* n */, int64_t* fail_block);

int spingp_eval_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                       const double* theta, int32_t n_theta, const double* d_t,
                       const double* d_y, int64_t n, double sigma, uint32_t flags,
                       double* d_loglik /* 1 */, double* d_grad, double* d_mean, double* d_var);

/* S independent series of n points each, series-major t[S][n], y[S][n];
 * per-series hyperparameters theta[S][n_theta] and noise sigma[S];
 * outputs loglik[S], grad[S][n_theta+1], mean[S][n], var[S][n]. */
int spingp_eval_batched(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                        const double* theta, int32_t n_theta, int64_t S, int64_t n,
                        const double* t, const double* y, const double* sigma, uint32_t flags,
                        double* out_loglik, double* out_grad, double* out_mean, double* out_var,
                        int64_t* fail_block);

/* Device variant: t, y and every output are device pointers; the per-series
 * hyperparameters theta[S][n_theta] and sigma[S] stay HOST arrays (control data,
 * turned into per-series device records by the library). */
int spingp_eval_batched_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                               const double* theta, int32_t n_theta, int64_t S, int64_t n,
                               const double* d_t, const double* d_y, const double* sigma,
                               uint32_t flags, double* d_loglik, double* d_grad, double* d_mean,
                               double* d_var);

/* predict at arbitrary test times: posterior
 * mean H mu and latent variance H C H^T (+ sigma^2 with SPINGP_INCLUDE_NOISE) at test_t[m]
 * (any order, outputs in input order), plus the training-data loglik and, with
 * SPINGP_WANT_GRAD, its gradient.  The test points join the n training points in one
 * sorted grid without an observation term (Sigma'^{-1} = 0 there); a test
 * time at or before the previous grid time is nudged by 1e-9 x (time span).
 * Host pointers; fail_block indexes the merged grid. */
int spingp_predict(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                   int32_t n_theta, const double* t, const double* y, int64_t n, const double* test_t,
                   int64_t m, double sigma, uint32_t flags, double* out_loglik, double* out_grad,
                   double* out_mean, double* out_var, int64_t* fail_block);

/* assemble_prior_precision + add_observation_term with the jitter
 * of SPEC.md:328 and Q_0 := Pinf: diag[n*b*b], upper[(n-1)*b*b], rhs[n*b]
 * (rhs_i = H^T y_i / sigma^2). */
int spingp_assemble(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                    const double* theta, int32_t n_theta, const double* t, const double* y,
                    int64_t n, double sigma, double* diag, double* upper, double* rhs,
                    int64_t* fail_block);

/* ---- multi-GPU partition of one long series -----------------
 * Rank r of P owns the contiguous time segment t[s_r .. e_r) (n_local points, device
 * pointers).  t_left = the last time of rank r-1 (ignored on rank 0), t_right = the
 * first time of rank r+1 (ignored on the last rank).  Protocol:
 *   1. spingp_seg_forward_device   -> d_record (n_record doubles): the segment reduced
 *      to its two boundary separators (Schur complement + logdet partial);
 *   2. caller all-gathers the P records (rank order) into d_records (e.g. NCCL);
 *   3. spingp_seg_reverse_device   -> d_partials (n_partials doubles): the P-block
 *      reduced system is solved redundantly, the segment back-substituted (selected
 *      inverse, gradient terms, optional per-point mean/var of the segment);
 *   4. caller all-reduces (sum) d_partials across ranks;
 *   5. spingp_seg_finalize_device  -> loglik, gradient (identical on every rank).
 * Steps 1 and 3 must run on the same context with no other evaluation in between. */
int spingp_seg_sizes(const spingp_leaf* leaves, int32_t n_leaves, int32_t* n_record, int32_t* n_partials);
int spingp_seg_forward_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                              const double* theta, int32_t n_theta, const double* d_t, const double* d_y,
                              int64_t n_local, double t_left, double t_right, int32_t rank, int32_t nranks,
                              double sigma, uint32_t flags, double* d_record);
int spingp_seg_reverse_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                              const double* theta, int32_t n_theta, const double* d_t, const double* d_y,
                              int64_t n_local, double t_left, double t_right, int32_t rank, int32_t nranks,
                              double sigma, uint32_t flags, const double* d_records, double* d_partials,
                              double* d_mean, double* d_var);
int spingp_seg_finalize_device(spingp_ctx* ctx, int32_t n_theta, int64_t n_total, double sigma, uint32_t flags,
                               const double* d_partials, double* d_loglik, double* d_grad);

/* K hyperparameter vectors theta[K][n_theta] (noise std-devs sigma[K]) on ONE series:
 * the optimizer's line-search probes in one batched evaluation.
 * t, y are uploaded once.  out_loglik[K], out_grad[K][n_theta+1]; on failure
 * fail_series = the first failing probe (its loglik is not meaningful). */
int spingp_eval_multi_theta(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                            int32_t n_theta, int64_t K, const double* t, const double* y, int64_t n,
                            const double* sigma, uint32_t flags, double* out_loglik, double* out_grad,
                            int64_t* fail_series);

/* ---- multi-GPU inside the library -----------------------
 * A multi-device context: one spingp_ctx per device plus an NCCL communicator
 * (ncclCommInitAll; NCCL is dlopen'ed on first use — SPINGP_NCCL_ERR without it).
 * spingp_eval_partitioned evaluates ONE long series over the P devices: contiguous time
 * segments, each reduced to a 2-separator Schur record, NCCL all-gather of the records,
 * the P-block reduced system solved on every device, back substitution + selected
 * inverse per segment, NCCL all-reduce of the partial sums.  Host pointers, synchronous;
 * results equal spingp_eval's to rounding.  Replaces the data-parallel cr_solve
 * contract of SPEC.md:200,224 at the scale of one box. */
typedef struct spingp_mctx spingp_mctx;
int spingp_mctx_create(int32_t n_gpus, const int32_t* device_ids, spingp_mctx** out);
int spingp_mctx_destroy(spingp_mctx* m);
int32_t spingp_mctx_size(const spingp_mctx* m);
spingp_ctx* spingp_mctx_rank_ctx(spingp_mctx* m, int32_t rank);
int spingp_eval_partitioned(spingp_mctx* m, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                            int32_t n_theta, const double* t, const double* y, int64_t n, double sigma,
                            uint32_t flags, double* out_loglik, double* out_grad, double* out_mean, double* out_var,
                            int64_t* fail_block);

/* ---- btd_core on a materialised symmetric BTD --------------- */

/* cr_solve: x = M^{-1} rhs for k right-hand sides, plus log det M. */
int spingp_btd_cr_solve(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag,
                        const double* upper, const double* rhs, int32_t k, double* x,
                        double* logdet, int64_t* fail_block);
int spingp_btd_cr_solve_device(spingp_ctx* ctx, int64_t n, int32_t b, const double* d_diag,
                               const double* d_upper, const double* d_rhs, int32_t k,
                               double* d_x, double* d_logdet);

/* selective_inverse: the BTD-pattern blocks of M^{-1}: cdiag[n*b*b], cupper[(n-1)*b*b]. */
int spingp_btd_selinv(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag,
                      const double* upper, double* cdiag, double* cupper, double* logdet,
                      int64_t* fail_block);
int spingp_btd_selinv_device(spingp_ctx* ctx, int64_t n, int32_t b, const double* d_diag,
                             const double* d_upper, double* d_cdiag, double* d_cupper,
                             double* d_logdet);

/* ---- BTDFactor: factorize once, reuse ------------------------
 * spingp_btd_factorize    factorize(SymBTD) -> BTDFactor
 *   A device-resident factor: the pivot Cholesky factors L_i (lower, positive
 *   diagonal, [n][b][b]), the multipliers M_i = U_i^T S_i^{-1} ([n-1][b][b]), the
 *   cached log det and the selected inverse.  One partitioned
 *   elimination pass, then every L_i, M_i in parallel from the Takahashi identities.
 * spingp_btd_factor_solve  solve(BTDFactor, rhs[(n b) x k])
 * spingp_btd_factor_selinv selective_inverse(BTDFactor)
 * spingp_btd_factor_blocks the L_i, M_i blocks (host copies)
 * Block size b <= 16.  The factor is bound to the context's device. */
typedef struct spingp_btd_factor spingp_btd_factor;
int spingp_btd_factorize(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag, const double* upper,
                         spingp_btd_factor** out, double* logdet, int64_t* fail_block);
int spingp_btd_factor_destroy(spingp_btd_factor* f);
int spingp_btd_factor_info(const spingp_btd_factor* f, int64_t* n, int32_t* b, double* logdet);
int spingp_btd_factor_blocks(spingp_ctx* ctx, const spingp_btd_factor* f, double* L, double* M);
int spingp_btd_factor_solve(spingp_ctx* ctx, const spingp_btd_factor* f, const double* rhs, int32_t k, double* x);
int spingp_btd_factor_selinv(spingp_ctx* ctx, const spingp_btd_factor* f, double* cdiag, double* cupper);

/* matvec: y = M v (one vector). */
int spingp_btd_matvec(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag,
                      const double* upper, const double* v, double* out);

#ifdef __cplusplus
}
#endif

#endif /* SPINGP_C_H */
