// libhrt_b200 — device layer: first-fit pools over HBM arenas, CUDA streams,
// cudaEvent-backed completion tokens and asynchronous copies (H2D, D2H, D2D
// and peer).  This replaces the reference's simulated device layer
// (/root/reference/pkg/src/hrt/devices.py): FreeListAllocator (89-154),
// DeviceBackend.attach/region (285-308), CompletionToken (199-222) and
// DeviceRegistry.enqueue_transfer (446-496), whose D2D rejection
// (devices.py:456-457) is lifted here.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "hrt_common.cuh"

namespace hrt {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // clear the sticky-free allocation error
        return HRT_E_OOM;
    }
    return HRT_E_CUDA;
}

int use_device(int gpu) {
    int cur = -1;
    HRT_CUDA(cudaGetDevice(&cur));
    if (cur != gpu) HRT_CUDA(cudaSetDevice(gpu));
    return HRT_OK;
}

// ---------------------------------------------------------------------------
// First-fit free list (FreeListAllocator, devices.py:89-154): address-ordered
// free blocks, sizes rounded up to the alignment, first fit, coalescing with
// the successor and then the predecessor on free.

struct FreeList {
    uint64_t capacity, alignment;
    std::map<uint64_t, uint64_t> free_blocks;  // offset -> size (address order)
    std::unordered_map<uint64_t, uint64_t> live;
    std::mutex mu;

    FreeList(uint64_t cap, uint64_t align) : capacity(cap), alignment(align) {
        free_blocks[0] = cap;
    }

    int alloc(uint64_t size, uint64_t* off, uint64_t* granted) {
        if (size == 0) {
            set_error("allocation size must be positive, got 0");
            return HRT_E_INVALID;
        }
        uint64_t need = (size + alignment - 1) / alignment * alignment;
        std::lock_guard<std::mutex> g(mu);
        for (auto it = free_blocks.begin(); it != free_blocks.end(); ++it) {
            if (it->second >= need) {
                uint64_t o = it->first, avail = it->second;
                free_blocks.erase(it);
                if (avail > need) free_blocks[o + need] = avail - need;
                live[o] = need;
                *off = o;
                *granted = need;
                return HRT_OK;
            }
        }
        set_error("no free block fits %llu bytes", (unsigned long long)need);
        return HRT_E_OOM;
    }

    int free(uint64_t off, uint64_t* size_out) {
        std::lock_guard<std::mutex> g(mu);
        auto lv = live.find(off);
        if (lv == live.end()) {
            set_error("offset %llu is not a live allocation", (unsigned long long)off);
            return HRT_E_DOUBLE_FREE;
        }
        uint64_t size = lv->second;
        live.erase(lv);
        if (size_out) *size_out = size;
        auto it = free_blocks.emplace(off, size).first;
        auto nx = std::next(it);
        if (nx != free_blocks.end() && off + size == nx->first) {
            it->second += nx->second;
            free_blocks.erase(nx);
        }
        if (it != free_blocks.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == off) {
                pv->second += it->second;
                free_blocks.erase(it);
            }
        }
        return HRT_OK;
    }

    void stats(uint64_t* lb, uint64_t* fb, uint64_t* nb) {
        std::lock_guard<std::mutex> g(mu);
        uint64_t l = 0, f = 0;
        for (auto& kv : live) l += kv.second;
        for (auto& kv : free_blocks) f += kv.second;
        if (lb) *lb = l;
        if (fb) *fb = f;
        if (nb) *nb = free_blocks.size();
    }

    int check() {
        std::lock_guard<std::mutex> g(mu);
        std::vector<std::pair<uint64_t, uint64_t>> spans;
        uint64_t total = 0;
        for (auto& kv : live) { spans.push_back({kv.first, kv.first + kv.second}); total += kv.second; }
        for (auto& kv : free_blocks) { spans.push_back({kv.first, kv.first + kv.second}); total += kv.second; }
        if (total != capacity) {
            set_error("live + free = %llu != capacity %llu", (unsigned long long)total,
                      (unsigned long long)capacity);
            return HRT_E_INVALID;
        }
        std::sort(spans.begin(), spans.end());
        for (size_t i = 1; i < spans.size(); ++i)
            if (spans[i - 1].second > spans[i].first) {
                set_error("overlapping regions at %llu", (unsigned long long)spans[i].first);
                return HRT_E_INVALID;
            }
        return HRT_OK;
    }
};

struct Pool {
    int gpu;
    void* base;
    FreeList fl;
    Pool(int g, void* b, uint64_t cap) : gpu(g), base(b), fl(cap, HRT_ALIGNMENT) {}
};

// ---------------------------------------------------------------------------
// Completion tokens: one cudaEvent each, recycled through a per-device pool.

struct Token {
    cudaEvent_t ev;
    int gpu;
};

static std::mutex g_tok_mu;
static std::unordered_map<uint64_t, Token> g_tokens;
static std::unordered_map<int, std::vector<cudaEvent_t>> g_event_pool;
static uint64_t g_next_token = 0;

static int take_event(int gpu, unsigned flags, cudaEvent_t* ev) {
    {
        std::lock_guard<std::mutex> g(g_tok_mu);
        auto& v = g_event_pool[gpu * 4 + (flags == cudaEventDefault ? 0 : 1)];
        if (!v.empty()) {
            *ev = v.back();
            v.pop_back();
            return HRT_OK;
        }
    }
    HRT_CUDA(cudaEventCreateWithFlags(ev, flags));
    return HRT_OK;
}

}  // namespace hrt

using namespace hrt;

extern "C" {

const char* hrt_last_error(void) { return hrt::g_err; }

int hrt_version(void) { return HRT_ABI_VERSION; }

int hrt_device_count(int* n) {
    HRT_CHECK_ARG(n, "null out pointer");
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return HRT_OK;
}

int hrt_device_info(int gpu, char* name, int name_len, int* sm_count, uint64_t* hbm_bytes,
                    int* cc_major, int* cc_minor) {
    cudaDeviceProp p;
    HRT_CUDA(cudaGetDeviceProperties(&p, gpu));
    if (name && name_len > 0) snprintf(name, name_len, "%s", p.name);
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (hbm_bytes) *hbm_bytes = p.totalGlobalMem;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    return HRT_OK;
}

int hrt_enable_peer_access(int gpu, int peer) {
    if (gpu == peer) return HRT_OK;
    int can = 0;
    HRT_CUDA(cudaDeviceCanAccessPeer(&can, gpu, peer));
    if (!can) {
        set_error("device %d cannot access peer %d", gpu, peer);
        return HRT_E_UNSUPPORTED;
    }
    int rc = use_device(gpu);
    if (rc) return rc;
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return HRT_OK;
    }
    HRT_CUDA(e);
    return HRT_OK;
}

// ---- first-fit allocator (host logic) ----

int hrt_fl_create(uint64_t capacity, uint64_t alignment, void** fl) {
    HRT_CHECK_ARG(fl, "null out pointer");
    HRT_CHECK_ARG(capacity > 0, "allocator capacity must be positive");
    HRT_CHECK_ARG(alignment > 0 && (alignment & (alignment - 1)) == 0,
                  "alignment must be a power of two");
    *fl = new FreeList(capacity, alignment);
    return HRT_OK;
}

int hrt_fl_alloc(void* fl, uint64_t size, uint64_t* offset, uint64_t* granted) {
    HRT_CHECK_ARG(fl && offset && granted, "null argument");
    return reinterpret_cast<FreeList*>(fl)->alloc(size, offset, granted);
}

int hrt_fl_free(void* fl, uint64_t offset, uint64_t* size) {
    HRT_CHECK_ARG(fl, "null allocator");
    return reinterpret_cast<FreeList*>(fl)->free(offset, size);
}

int hrt_fl_stats(void* fl, uint64_t* live_bytes, uint64_t* free_bytes, uint64_t* free_blocks) {
    HRT_CHECK_ARG(fl, "null allocator");
    reinterpret_cast<FreeList*>(fl)->stats(live_bytes, free_bytes, free_blocks);
    return HRT_OK;
}

int hrt_fl_check(void* fl) {
    HRT_CHECK_ARG(fl, "null allocator");
    return reinterpret_cast<FreeList*>(fl)->check();
}

void hrt_fl_destroy(void* fl) { delete reinterpret_cast<FreeList*>(fl); }

// ---- device pools ----

int hrt_pool_create(int gpu, uint64_t capacity, void** pool) {
    HRT_CHECK_ARG(pool && capacity > 0, "bad pool arguments");
    int rc = use_device(gpu);
    if (rc) return rc;
    void* base = nullptr;
    HRT_CUDA(cudaMalloc(&base, capacity));
    *pool = new Pool(gpu, base, capacity);
    return HRT_OK;
}

int hrt_pool_alloc(void* pool, uint64_t size, uint64_t* offset, uint64_t* granted, void** dptr) {
    HRT_CHECK_ARG(pool && offset && granted, "null argument");
    Pool* p = reinterpret_cast<Pool*>(pool);
    int rc = p->fl.alloc(size, offset, granted);
    if (rc) return rc;
    if (dptr) *dptr = static_cast<char*>(p->base) + *offset;
    return HRT_OK;
}

int hrt_pool_free(void* pool, uint64_t offset) {
    HRT_CHECK_ARG(pool, "null pool");
    return reinterpret_cast<Pool*>(pool)->fl.free(offset, nullptr);
}

int hrt_pool_stats(void* pool, uint64_t* live_bytes, uint64_t* free_bytes) {
    HRT_CHECK_ARG(pool, "null pool");
    reinterpret_cast<Pool*>(pool)->fl.stats(live_bytes, free_bytes, nullptr);
    return HRT_OK;
}

int hrt_pool_base(void* pool, void** base) {
    HRT_CHECK_ARG(pool && base, "null argument");
    *base = reinterpret_cast<Pool*>(pool)->base;
    return HRT_OK;
}

int hrt_pool_destroy(void* pool) {
    if (!pool) return HRT_OK;
    Pool* p = reinterpret_cast<Pool*>(pool);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    cudaError_t e = cudaFree(p->base);
    delete p;
    HRT_CUDA(e);
    return HRT_OK;
}

// ---- streams ----

int hrt_stream_create(int gpu, int priority, void** stream) {
    HRT_CHECK_ARG(stream, "null out pointer");
    int rc = use_device(gpu);
    if (rc) return rc;
    Stream* s = new Stream();
    s->gpu = gpu;
    cudaError_t e = cudaStreamCreateWithPriority(&s->s, cudaStreamNonBlocking, priority);
    if (e != cudaSuccess) {
        delete s;
        return cuda_fail(e, "cudaStreamCreateWithPriority");
    }
    *stream = s;
    return HRT_OK;
}

int hrt_stream_wrap(int gpu, void* cuda_stream, void** stream) {
    HRT_CHECK_ARG(stream, "null out pointer");
    Stream* s = new Stream();
    s->gpu = gpu;
    s->s = reinterpret_cast<cudaStream_t>(cuda_stream);
    *stream = s;
    return HRT_OK;
}

void* hrt_stream_handle(void* stream) { return stream ? as_stream(stream)->s : nullptr; }

int hrt_stream_destroy(void* stream, int owned) {
    if (!stream) return HRT_OK;
    Stream* s = as_stream(stream);
    cudaError_t e = cudaSuccess;
    if (owned || s->cmp_d) use_device(s->gpu);
    if (s->cmp_d) {
        cudaStreamSynchronize(s->s);
        cudaFree(s->cmp_d);
        cudaFreeHost(s->cmp_h);
    }
    if (owned) e = cudaStreamDestroy(s->s);
    delete s;
    HRT_CUDA(e);
    return HRT_OK;
}

int hrt_stream_synchronize(void* stream) {
    HRT_CHECK_ARG(stream, "null stream");
    HRT_CUDA(cudaStreamSynchronize(as_stream(stream)->s));
    return HRT_OK;
}

int hrt_device_synchronize(int gpu) {
    int rc = use_device(gpu);
    if (rc) return rc;
    HRT_CUDA(cudaDeviceSynchronize());
    return HRT_OK;
}

// ---- tokens ----

int hrt_token_record(void* stream, uint64_t* token) {
    HRT_CHECK_ARG(stream && token, "null argument");
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    cudaEvent_t ev;
    rc = take_event(s->gpu, cudaEventDefault, &ev);
    if (rc) return rc;
    HRT_CUDA(cudaEventRecord(ev, s->s));
    std::lock_guard<std::mutex> g(g_tok_mu);
    uint64_t id = ++g_next_token;
    g_tokens[id] = Token{ev, s->gpu};
    *token = id;
    return HRT_OK;
}

static int find_token(uint64_t token, Token* out) {
    std::lock_guard<std::mutex> g(g_tok_mu);
    auto it = g_tokens.find(token);
    if (it == g_tokens.end()) {
        set_error("unknown token %llu", (unsigned long long)token);
        return HRT_E_UNKNOWN_TOKEN;
    }
    *out = it->second;
    return HRT_OK;
}

int hrt_token_query(uint64_t token) {
    Token t;
    int rc = find_token(token, &t);
    if (rc) return rc;
    cudaError_t e = cudaEventQuery(t.ev);
    if (e == cudaSuccess) return 1;
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        return 0;
    }
    set_error("token %llu failed: %s", (unsigned long long)token, cudaGetErrorString(e));
    return 2;
}

// Waits poll the event for up to HRT_SPIN_US (default 2000) before the
// blocking cudaEventSynchronize: a blocking wake-up costs the OS timer slack
// (~50 us), which doubled small-message round trips whenever the CUDA
// scheduling heuristic chose to yield.
int hrt_token_wait(uint64_t token) {
    Token t;
    int rc = find_token(token, &t);
    if (rc) return rc;
    static const long long spin_ns = [] {
        const char* e = getenv("HRT_SPIN_US");
        return (e ? atoll(e) : 2000LL) * 1000LL;
    }();
    if (spin_ns > 0) {
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t e = cudaEventQuery(t.ev);
            if (e == cudaSuccess) return HRT_OK;
            if (e != cudaErrorNotReady) HRT_CUDA(e);
            if (std::chrono::duration_cast<std::chrono::nanoseconds>(
                    std::chrono::steady_clock::now() - t0).count() > spin_ns)
                break;
        }
        cudaGetLastError();  // clear the sticky not-ready status
    }
    HRT_CUDA(cudaEventSynchronize(t.ev));
    return HRT_OK;
}

int hrt_stream_wait_token(void* stream, uint64_t token) {
    HRT_CHECK_ARG(stream, "null stream");
    Token t;
    int rc = find_token(token, &t);
    if (rc) return rc;
    Stream* s = as_stream(stream);
    rc = use_device(s->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaStreamWaitEvent(s->s, t.ev, 0));
    return HRT_OK;
}

int hrt_token_elapsed_ms(uint64_t start, uint64_t end, float* ms) {
    HRT_CHECK_ARG(ms, "null out pointer");
    Token a, b;
    int rc = find_token(start, &a);
    if (rc) return rc;
    rc = find_token(end, &b);
    if (rc) return rc;
    HRT_CUDA(cudaEventElapsedTime(ms, a.ev, b.ev));
    return HRT_OK;
}

int hrt_token_release(uint64_t token) {
    std::lock_guard<std::mutex> g(g_tok_mu);
    auto it = g_tokens.find(token);
    if (it == g_tokens.end()) {
        set_error("unknown token %llu", (unsigned long long)token);
        return HRT_E_UNKNOWN_TOKEN;
    }
    g_event_pool[it->second.gpu * 4].push_back(it->second.ev);
    g_tokens.erase(it);
    return HRT_OK;
}

// ---- host memory and copies ----

int hrt_host_alloc(uint64_t bytes, void** ptr) {
    HRT_CHECK_ARG(ptr && bytes > 0, "bad host allocation");
    HRT_CUDA(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable));
    return HRT_OK;
}

int hrt_host_free(void* ptr) {
    if (!ptr) return HRT_OK;
    HRT_CUDA(cudaFreeHost(ptr));
    return HRT_OK;
}

int hrt_host_register(void* ptr, uint64_t bytes) {
    HRT_CHECK_ARG(ptr && bytes > 0, "bad host registration");
    HRT_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
    return HRT_OK;
}

int hrt_host_unregister(void* ptr) {
    HRT_CUDA(cudaHostUnregister(ptr));
    return HRT_OK;
}

int hrt_copy_async(void* stream, void* dst, const void* src, uint64_t bytes) {
    HRT_CHECK_ARG(stream, "null stream");
    if (bytes == 0) return HRT_OK;
    HRT_CHECK_ARG(dst && src, "null copy pointer");
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s->s));
    return HRT_OK;
}

int hrt_copy_peer_async(void* stream, void* dst, int dst_gpu, const void* src, int src_gpu,
                        uint64_t bytes) {
    HRT_CHECK_ARG(stream, "null stream");
    if (bytes == 0) return HRT_OK;
    HRT_CHECK_ARG(dst && src, "null copy pointer");
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaMemcpyPeerAsync(dst, dst_gpu, src, src_gpu, bytes, s->s));
    return HRT_OK;
}

}  // extern "C"

namespace hrt {
// SM-driven copy over NVLink (either pointer may live on a peer GPU): each
// thread moves 4 x 16 bytes per iteration with independent loads in flight;
// a head/tail in 8-byte then 1-byte units covers unaligned sizes.
__global__ void __launch_bounds__(512) sm_copy_kernel(uint8_t* __restrict__ dst,
                                                      const uint8_t* __restrict__ src,
                                                      uint64_t n16, uint64_t tail_from,
                                                      uint64_t bytes) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        const uint4 a = __ldcs(s + i), b = __ldcs(s + i + stride), c = __ldcs(s + i + 2 * stride),
                    e = __ldcs(s + i + 3 * stride);
        __stcs(d + i, a);
        __stcs(d + i + stride, b);
        __stcs(d + i + 2 * stride, c);
        __stcs(d + i + 3 * stride, e);
    }
    for (; i < n16; i += stride) __stcs(d + i, __ldcs(s + i));
    const uint64_t t = tail_from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < bytes) dst[t] = src[t];
}
// counts differing bytes of a and b (16-byte words, then the tail)
__global__ void __launch_bounds__(512) bytes_diff_kernel(const uint8_t* __restrict__ a,
                                                         const uint8_t* __restrict__ b,
                                                         uint64_t n16, uint64_t bytes,
                                                         unsigned long long* diff) {
    const uint4* x = reinterpret_cast<const uint4*>(a);
    const uint4* y = reinterpret_cast<const uint4*>(b);
    unsigned long long d = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4 u = x[i], v = y[i];
        d += (u.x != v.x) + (u.y != v.y) + (u.z != v.z) + (u.w != v.w);
    }
    const uint64_t t = n16 * 16 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < bytes) d += a[t] != b[t];
    if (d) atomicAdd(diff, d);
}
}  // namespace hrt

extern "C" {

// *equal = 1 when the n bytes at a and b (device or peer addresses, 16-byte
// aligned) are identical.  Synchronises `stream`.
int hrt_bytes_equal(void* stream, const void* a, const void* b, uint64_t bytes, int* equal) {
    HRT_CHECK_ARG(stream && equal, "null argument");
    *equal = 1;
    if (bytes == 0) return HRT_OK;
    HRT_CHECK_ARG(a && b && ((uintptr_t)a | (uintptr_t)b) % 16 == 0,
                  "bytes_equal needs 16-byte aligned pointers");
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    if (!s->cmp_d) {
        // one word per stream handle, kept: a cudaMallocAsync per call went
        // back to the OS at every synchronize (~1.4 ms per compare)
        HRT_CUDA(cudaMalloc(&s->cmp_d, sizeof(unsigned long long)));
        cudaError_t he = cudaHostAlloc(&s->cmp_h, sizeof(unsigned long long), cudaHostAllocDefault);
        if (he != cudaSuccess) {
            cudaFree(s->cmp_d);
            s->cmp_d = nullptr;
            HRT_CUDA(he);
        }
    }
    unsigned long long* d = s->cmp_d;
    HRT_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s->s));
    const uint64_t n16 = bytes / 16;
    const uint64_t nb = std::min<uint64_t>((uint64_t)hrt::sm_count(s->gpu) * 4, (n16 + 511) / 512 + 1);
    hrt::bytes_diff_kernel<<<(unsigned)nb, 512, 0, s->s>>>(
        reinterpret_cast<const uint8_t*>(a), reinterpret_cast<const uint8_t*>(b), n16, bytes, d);
    HRT_CUDA(cudaGetLastError());
    HRT_CUDA(cudaMemcpyAsync(s->cmp_h, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->s));
    HRT_CUDA(cudaStreamSynchronize(s->s));
    *equal = *s->cmp_h == 0;
    return HRT_OK;
}

// cudaMemcpyPeerAsync replacement for GPU<->GPU messages: an SM copy kernel
// on `stream`'s GPU (peer access to the other side must be enabled).  Needs
// 16-byte aligned pointers for the vector part.
int hrt_copy_sm_async(void* stream, void* dst, const void* src, uint64_t bytes, int blocks) {
    HRT_CHECK_ARG(stream, "null stream");
    if (bytes == 0) return HRT_OK;
    HRT_CHECK_ARG(dst && src, "null copy pointer");
    HRT_CHECK_ARG(((uintptr_t)dst | (uintptr_t)src) % 16 == 0, "sm copy needs 16-byte alignment");
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    const uint64_t n16 = bytes / 16;
    const uint64_t nb = blocks > 0 ? (uint64_t)blocks
                                   : std::min<uint64_t>((uint64_t)hrt::sm_count(s->gpu) * 4, (n16 + 511) / 512 + 1);
    hrt::sm_copy_kernel<<<(unsigned)nb, 512, 0, s->s>>>(
        reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src), n16, n16 * 16,
        bytes);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

// One call for a message/transfer copy (the registry's enqueue_transfer,
// devices.py:446-496): GPU-side waits on `waits`, the copy, and a completion
// token recorded behind it.  method 0: copy engine (cudaMemcpyAsync over
// UVA; peer copies ride NVLink), 1: SM pull/push kernel on the stream's GPU
// (16-byte aligned pointers), 2: automatic — SM kernel for aligned GPU<->GPU
// copies of at most HRT_SM_COPY_MAX bytes (it beats the copy engine's
// per-copy latency there, profiles/copy_methods_r01.txt), else the copy
// engine.  One device switch for the whole sequence: the Python path paid
// one per native call.
int hrt_copy_ordered(void* stream, void* dst, const void* src, uint64_t bytes, int peer,
                     const uint64_t* waits, int nwait, int method, uint64_t* token) {
    hrt::NvtxRange nvtx_("hrt_copy_ordered");
    HRT_CHECK_ARG(stream && token, "null argument");
    HRT_CHECK_ARG(nwait >= 0 && (nwait == 0 || waits), "bad wait list");
    HRT_CHECK_ARG(bytes == 0 || (dst && src), "null copy pointer");
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    for (int k = 0; k < nwait; ++k) {
        Token t;
        rc = find_token(waits[k], &t);
        if (rc == HRT_E_UNKNOWN_TOKEN) {  // retired already: nothing to order after
            continue;
        }
        if (rc) return rc;
        HRT_CUDA(cudaStreamWaitEvent(s->s, t.ev, 0));
    }
    if (bytes) {
        const bool aligned = (((uintptr_t)dst | (uintptr_t)src) % 16) == 0;
        static const uint64_t sm_max = [] {
            const char* e = getenv("HRT_SM_COPY_MAX");
            return e ? (uint64_t)strtoull(e, nullptr, 10) : (uint64_t)(64ull << 20);
        }();
        const bool sm = method == 1 || (method == 2 && peer && aligned && bytes <= sm_max);
        if (sm) {
            HRT_CHECK_ARG(aligned, "sm copy needs 16-byte alignment");
            const uint64_t n16 = bytes / 16;
            const uint64_t nb = std::min<uint64_t>((uint64_t)hrt::sm_count(s->gpu) * 4, (n16 + 511) / 512 + 1);
            hrt::sm_copy_kernel<<<(unsigned)nb, 512, 0, s->s>>>(
                reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src), n16,
                n16 * 16, bytes);
            HRT_CUDA(cudaGetLastError());
        } else {
            HRT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s->s));
        }
    }
    cudaEvent_t ev;
    rc = take_event(s->gpu, cudaEventDefault, &ev);
    if (rc) return rc;
    HRT_CUDA(cudaEventRecord(ev, s->s));
    std::lock_guard<std::mutex> g(g_tok_mu);
    const uint64_t id = ++g_next_token;
    g_tokens[id] = Token{ev, s->gpu};
    *token = id;
    return HRT_OK;
}

int hrt_copy2d_async(void* stream, void* dst, uint64_t dpitch, const void* src, uint64_t spitch,
                     uint64_t width, uint64_t height) {
    HRT_CHECK_ARG(stream, "null stream");
    if (width == 0 || height == 0) return HRT_OK;
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault, s->s));
    return HRT_OK;
}

int hrt_memset_async(void* stream, void* dst, int value, uint64_t bytes) {
    HRT_CHECK_ARG(stream, "null stream");
    if (bytes == 0) return HRT_OK;
    Stream* s = as_stream(stream);
    int rc = use_device(s->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaMemsetAsync(dst, value, bytes, s->s));
    return HRT_OK;
}

// ---- CUDA IPC: map another process's device allocation (same node) ----

int hrt_ipc_get_handle(const void* base, uint8_t* out64) {
    HRT_CHECK_ARG(base && out64, "null argument");
    cudaIpcMemHandle_t h;
    HRT_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(base)));
    memcpy(out64, &h, sizeof(h));
    return HRT_OK;
}

int hrt_ipc_open_handle(int gpu, const uint8_t* in64, void** ptr) {
    HRT_CHECK_ARG(in64 && ptr, "null argument");
    int rc = use_device(gpu);
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    memcpy(&h, in64, sizeof(h));
    HRT_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return HRT_OK;
}

int hrt_ipc_close_handle(void* ptr) {
    if (!ptr) return HRT_OK;
    HRT_CUDA(cudaIpcCloseMemHandle(ptr));
    return HRT_OK;
}

int hrt_pointer_device(const void* ptr, int* gpu) {
    HRT_CHECK_ARG(gpu, "null out pointer");
    cudaPointerAttributes a;
    HRT_CUDA(cudaPointerGetAttributes(&a, ptr));
    *gpu = (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? a.device : -1;
    return HRT_OK;
}

}  // extern "C"
