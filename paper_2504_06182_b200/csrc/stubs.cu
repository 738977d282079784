// Temporary: entry points whose kernels are not built yet fail loudly.
#include "capi_internal.cuh"
extern "C" {
recon_status recon_assign_1d(recon_ctx *, int32_t, const int32_t *, int32_t, const int32_t *, int32_t, int64_t *,
                             int64_t *, int64_t *, int32_t *, int32_t *) { return RECON_ERR_ARGUMENT; }
recon_status recon_assign_1d_generalized(recon_ctx *, int32_t, const int64_t *, const int32_t *, const int32_t *,
                                         int32_t, const int64_t *, int64_t *, int64_t *, int64_t *, int32_t *,
                                         int32_t *) { return RECON_ERR_ARGUMENT; }
recon_status recon_solve_1d(recon_ctx *, int32_t, const int32_t *, int32_t, const int32_t *, int32_t, int32_t *,
                            int32_t *, int32_t *, int32_t *, int32_t *, int64_t, int64_t *, int64_t *, int32_t *,
                            int32_t *) { return RECON_ERR_ARGUMENT; }
recon_status recon_solve_1d_batch(recon_ctx *, const recon_chain_batch *) { return RECON_ERR_ARGUMENT; }
recon_status recon_solve_1d_batch_host(recon_ctx *, const recon_chain_batch *) { return RECON_ERR_ARGUMENT; }
recon_status recon_batch_moves(recon_ctx *, int32_t, int32_t, const uint64_t *, int32_t, const int64_t *,
                               const int32_t *, int64_t, const int32_t *, const int32_t *, int32_t, int32_t,
                               int32_t *, int64_t *, int32_t *) { return RECON_ERR_ARGUMENT; }
recon_status recon_pipeline_batch_run(recon_ctx *, const recon_pipeline_batch *) { return RECON_ERR_ARGUMENT; }
recon_status recon_pipeline_batch_run_host(recon_ctx *, const recon_pipeline_batch *) { return RECON_ERR_ARGUMENT; }
}
