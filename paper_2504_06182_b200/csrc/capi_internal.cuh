// Internal host-side context for the C-ABI implementation.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "recon_b200.h"

namespace rb {

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};
struct HostBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// Workspace slots (grow-only device buffers owned by a context).
enum Slot {
    S_OCC, S_PSRC, S_PDST, S_PEV, S_PCNT, S_TDISP, S_STATUS, S_DETAIL, S_EVENTS,
    S_SRCOF, S_TGTOF, S_DCNT, S_DOFF, S_KEYS, S_KEYS2, S_TEMP, S_EA, S_EB,
    S_CHAIN_A, S_CHAIN_B, S_CHAIN_C, S_CHAIN_D, S_CHAIN_E,
    S_BM_OFF, S_BM_VERT, S_BM_ES, S_BM_ED, S_BM_OUT, S_BM_AUX0, S_BM_AUX1, S_BM_AUX2, S_BM_AUX3,
    S_BM_AUX4, S_BM_AUX5, S_BM_AUX6, S_BM_AUX7, S_STAGE, S_WORK, S_PLAN,
    S_V_VERDICT, S_V_STATE, S_V_SRCOF, S_V_DSTOF, S_V_FIN, S_V_LEN, S_V_MB, S_V_EV, S_V_EV2, S_V_BCNT,
    S_V_BMIN, S_V_BMAX, S_V_ECNT, S_V_ALIVE, S_V_PRED, S_V_TOK, S_V_BEGAN,
    S_W_LEN, S_W_OUT, S_W_MOFF, S_W_VOFF, S_W_MB, S_W_K0, S_W_K1, S_W_I0, S_W_I1,
    S_SIM_OCC, S_SIM_CUR, S_SIM_NXT, S_SIM_CYC, S_SIM_ST, S_SIM_SUC, S_SIM_ACC, S_SIM_EL, S_SIM_LIVE, S_SIM_CODE,
    S_SIM_CEL, S_SIM_PDEC, S_SIM_SRC, S_SIM_DST, S_SIM_PC, S_SIM_PST, S_SIM_DET, S_SIM_NB, S_SIM_TD, S_SIM_OFF,
    S_SIM_MB, S_SIM_BCNT, S_SIM_RUN, S_SIM_ALLC, S_PPACK, S_BM_WSTATE, S_BM_VMIN, S_BM_PREC,
    S_PH_OCC0, S_PH_OCC1, S_PH_SRC0, S_PH_SRC1, S_PH_DST0, S_PH_DST1, S_PH_EV0, S_PH_EV1, S_PH_I32_0, S_PH_I32_1,
    S_PH_I64_0, S_PH_I64_1, S_PH_MB0, S_PH_MB1, S_PH_RS0, S_PH_RS1, S_PH_RC0, S_PH_RC1,
    S_NSLOTS
};

struct Ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    bool timing = false;          // recon_ctx_set_kernel_timing
    bool timed_plan = false;      // the last timed solve launched the planner
    cudaEvent_t tev[3] = {};      // before planner, before executor, after executor
    cudaEvent_t pev[5] = {};      // pipeline phases: solve | dag | wide | batching (recon_ctx_phase_times)
    bool timed_pipeline = false;
    cudaStream_t copy_stream = nullptr;  // device-to-host copies overlapping the next chunk's solve
    cudaEvent_t cev[64] = {};            // chunk-done events (reused round robin)
    int cev_next = 0;
    cudaEvent_t chunk_event() {
        cudaEvent_t &e = cev[cev_next++ % 64];
        if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        return e;
    }
    DevBuf buf[S_NSLOTS];
    HostBuf hbuf[8];
    void *get(int slot, size_t bytes);
    void *host(int slot, size_t bytes);
    template <class T>
    T *dev(int slot, size_t count) {
        return static_cast<T *>(get(slot, count * sizeof(T)));
    }
    ~Ctx();
};

Ctx *resolve(recon_ctx *ctx);
// stats.cu: the run-length schedule of a device pipeline batch, enqueued on st
cudaError_t launch_schedule_runs(const recon_pipeline_batch &pb, const recon_schedule_runs &runs, int sms,
                                 cudaStream_t st);
void set_cuda_error(cudaError_t e, const char *where);
recon_status cuda_fail(cudaError_t e, const char *where, int32_t *detail);

}  // namespace rb
