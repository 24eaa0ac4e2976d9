// Shared helpers for libhrt_b200: error plumbing and handle types.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hrt_b200.h"

namespace hrt {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

struct Stream {
    cudaStream_t s = nullptr;
    int gpu = 0;
    // hrt_bytes_equal's result word (device) and its pinned host mirror,
    // allocated on first use, freed with the handle
    unsigned long long* cmp_d = nullptr;
    unsigned long long* cmp_h = nullptr;
};

// NVTX range over a host entry point (header-only NVTX 3: a null check when
// no profiler is attached); shows the enqueue side of runs, uploads and
// messages on an Nsight Systems timeline next to the kernels they launch
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline Stream* as_stream(void* h) { return reinterpret_cast<Stream*>(h); }

// Make `gpu` current for the calling thread (cheap when already current).
int use_device(int gpu);

// Streaming multiprocessors of `gpu` (queried once per device, cached);
// gpu < 0 means the calling thread's current device.  Grid sizes derive
// from it instead of a hard-coded 148 (other SKUs, MIG slices).
inline int sm_count(int gpu = -1) {
    static int cache[64] = {0};
    if (gpu < 0 && cudaGetDevice(&gpu) != cudaSuccess) gpu = 0;
    if (gpu >= 64) gpu = 63;
    if (cache[gpu] <= 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, gpu) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;  // B200
        }
        cache[gpu] = n;
    }
    return cache[gpu];
}

}  // namespace hrt

#define HRT_CUDA(call)                                              \
    do {                                                            \
        cudaError_t _e = (call);                                    \
        if (_e != cudaSuccess) return hrt::cuda_fail(_e, #call);    \
    } while (0)

#define HRT_CHECK_ARG(cond, msg)                                    \
    do {                                                            \
        if (!(cond)) {                                              \
            hrt::set_error("%s", msg);                              \
            return HRT_E_INVALID;                                   \
        }                                                           \
    } while (0)
