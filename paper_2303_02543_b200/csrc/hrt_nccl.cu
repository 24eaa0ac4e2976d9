// libhrt_b200 — cross-process halo exchange over NCCL send/recv.
//
// The reference moves halo objects between ranks with mp_send
// (/root/reference/pkg/src/hrt/bench/jacobi.py:237) over a loopback or TCP
// transport (transport.py:62-278), staging through host memory
// (comm.py:419-466).  Here one process drives one B200 and the faces that
// cross a process boundary go GPU->GPU with grouped ncclSend/ncclRecv over
// NVLink/NVSwitch, enqueued on the step stream (and therefore capturable in
// the step's CUDA graph).  NCCL is dlopen'ed so the library loads on hosts
// without it; whichever libnccl.so.2 the process already loaded (torch's)
// is reused.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "hrt_common.cuh"

namespace {

// minimal NCCL ABI (stable across 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
enum { ncclUint64 = 5, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };

struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(ncclUniqueId*);
    int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    int (*CommDestroy)(ncclComm_t);
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
    int (*GroupStart)();
    int (*GroupEnd)();
    int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(int);
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

int load_nccl() {
    std::lock_guard<std::mutex> g(g_nccl_mu);
    if (g_nccl.h) return HRT_OK;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names) {
        h = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        hrt::set_error("cannot load libnccl.so.2: %s", dlerror());
        return HRT_E_NCCL;
    }
#define SYM(field, name)                                                     \
    *(void**)(&g_nccl.field) = dlsym(h, name);                               \
    if (!g_nccl.field) {                                                     \
        hrt::set_error("libnccl is missing %s", name);                       \
        return HRT_E_NCCL;                                                   \
    }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(AllReduce, "ncclAllReduce");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    g_nccl.h = h;
    return HRT_OK;
}

int nccl_fail(int r, const char* what) {
    hrt::set_error("%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
    return HRT_E_NCCL;
}

}  // namespace

extern "C" {

int hrt_nccl_unique_id(uint8_t* out128) {
    int rc = load_nccl();
    if (rc) return rc;
    ncclUniqueId id;
    int r = g_nccl.GetUniqueId(&id);
    if (r) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(out128, id.internal, 128);
    return HRT_OK;
}

int hrt_nccl_init(int gpu, int rank, int world, const uint8_t* id128, void** comm) {
    HRT_CHECK_ARG(comm && id128, "null argument");
    int rc = load_nccl();
    if (rc) return rc;
    rc = hrt::use_device(gpu);
    if (rc) return rc;
    ncclUniqueId id;
    memcpy(id.internal, id128, 128);
    ncclComm_t c = nullptr;
    int r = g_nccl.CommInitRank(&c, world, id, rank);
    if (r) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return HRT_OK;
}

int hrt_nccl_destroy(void* comm) {
    if (!comm) return HRT_OK;
    int r = g_nccl.CommDestroy(reinterpret_cast<ncclComm_t>(comm));
    if (r) return nccl_fail(r, "ncclCommDestroy");
    return HRT_OK;
}

// Grouped send/recv of every remote face for one step parity.
int hrt_nccl_exchange(void* comm, void* stream, const hrt_remote_seg_t* segs, int n, int parity) {
    HRT_CHECK_ARG(comm && stream, "remote faces need an NCCL communicator");
    if (n == 0) return HRT_OK;
    cudaStream_t s = hrt::as_stream(stream)->s;
    ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
    int r = g_nccl.GroupStart();
    if (r) return nccl_fail(r, "ncclGroupStart");
    for (int i = 0; i < n; ++i) {
        const hrt_remote_seg_t& g = segs[i];
        if (g.kind == 0)
            r = g_nccl.Send(reinterpret_cast<const void*>(g.buf[parity]), (size_t)g.count,
                            ncclFloat64, g.peer, c, s);
        else
            r = g_nccl.Recv(reinterpret_cast<void*>(g.buf[parity]), (size_t)g.count, ncclFloat64,
                            g.peer, c, s);
        if (r) break;
    }
    int r2 = g_nccl.GroupEnd();
    if (r) return nccl_fail(r, "ncclSend/ncclRecv");
    if (r2) return nccl_fail(r2, "ncclGroupEnd");
    return HRT_OK;
}

// In-place max all-reduce of uint64 words (the residual history bit
// patterns: non-negative doubles order like their bits).
int hrt_nccl_allreduce_max_u64(void* comm, void* stream, uint64_t* buf, int64_t count) {
    HRT_CHECK_ARG(comm && stream && buf, "null argument");
    int r = g_nccl.AllReduce(buf, buf, (size_t)count, ncclUint64, ncclMax,
                             reinterpret_cast<ncclComm_t>(comm), hrt::as_stream(stream)->s);
    if (r) return nccl_fail(r, "ncclAllReduce");
    return HRT_OK;
}

// Plain sum all-reduce of doubles (checksums of disjoint partial sums are
// not used for parity; this serves the ping-pong/bench plumbing).
int hrt_nccl_allreduce_sum_f64(void* comm, void* stream, double* buf, int64_t count) {
    HRT_CHECK_ARG(comm && stream && buf, "null argument");
    int r = g_nccl.AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum,
                             reinterpret_cast<ncclComm_t>(comm), hrt::as_stream(stream)->s);
    if (r) return nccl_fail(r, "ncclAllReduce");
    return HRT_OK;
}

}  // extern "C"
