// capi_internal.h — library-internal interface between capi.cu (contexts,
// transport, finalize) and multi.cu (NCCL communicator, device groups).
// Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <functional>

#include "../../include/xscat_gpu.h"

namespace xsi {

// NVTX range for Nsight timelines (header-only NVTX 3: a no-op unless a tool
// is attached).
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};

// The correction loop's scans, delegated (xs_group_run_iterative_correction
// shards them by angle over the group's devices).  Outputs are device
// buffers of the calling context.
using ScanHook = std::function<void(const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                                    const int32_t* subset, int32_t n, int32_t what, double* d_primary,
                                    double* d_scatter)>;

// Runs f with the context's device current; errors become the context's
// xs_last_error and the returned xs_status.
int run(xs_context* c, const std::function<void()>& f);

int device(const xs_context* c);
cudaStream_t stream(const xs_context* c);
void*& mgpu_slot(xs_context* c);       // owned by multi.cu
void mgpu_release(xs_context* c);      // multi.cu: frees the communicator (xs_ctx_destroy)
void set_scan_hook(xs_context* c, ScanHook h);

uint64_t history_count(const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg);
xs_accum_layout layout(const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg);
unsigned long long* own_accum(xs_context* c, size_t words); // the context's accumulator buffer

// validate + transport of histories [h0, h1) into d_accum (on c's device)
void accumulate(xs_context* c, const xs_geometry& g, int angle, const xs_spectrum& spec, const xs_sim_config& cfg,
                uint64_t h0, uint64_t h1, unsigned long long* d_accum);
// SimResult of the sum of n_src accumulators (local or peer device memory)
void finalize(xs_context* c, const xs_geometry& g, const xs_spectrum& spec, const xs_sim_config& cfg,
              const unsigned long long* const* srcs, int n_src, uint64_t h0, uint64_t h1, xs_scatter_result* out,
              double* d_image);
void scan_device(xs_context* c, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                 const int32_t* subset, int32_t n, int32_t what, double* d_primary, double* d_scatter,
                 double* seconds);
void check_scan_args(const xs_geometry* g, const xs_sim_config* cfg, const int32_t* subset, int32_t n);
void cuda(cudaError_t e, const char* what); // throws XS_E_CUDA

} // namespace xsi
