// ls_api_internal.h -- host-side pieces shared by ls_api.cu and ls_multi.cu.
#pragma once
#include <cuda_runtime.h>

#include <memory>

#include "ls.h"
#include "ls_common.cuh"

namespace ls {

// State of an enqueued sort whose status/stats are collected after a sync.
struct Pending {
    bool active = false;
    Ctl ctl_host;
    Ctl *ctl_dev = nullptr;
    DevModel *model_dev = nullptr;
    std::unique_ptr<DevModel> model_host;
    ls_model *model_out = nullptr;
    uint64_t launches = 0;
    int dtype = 0;
    bool timer_on = false;
    bool own_events = true;  // false: the events belong to a cached graph
    cudaEvent_t ev[LS_NUM_PHASES + 1];
    int phase_of[LS_NUM_PHASES + 1];
    int nmarks = 0;
};

void set_error(const char *msg);
// LS_OK or LS_E_INVALID (with ls_last_error set) for a bad ls_config.
ls_status check_config(const ls_config &c);
ls_status enqueue_sort(void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg,
                       const ls_model *inject, void *d_ws, size_t ws_bytes, cudaStream_t st,
                       ls_stats *stats, const ls_dumps *dumps, Pending *pend);
ls_status finish_sort(Pending *pend, cudaStream_t st, ls_stats *stats);
size_t workspace_bytes(uint64_t n, const ls_config &cfg);

}  // namespace ls
