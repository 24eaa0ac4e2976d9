// libhrt_b200 — the Jacobi hot path on sm_100a.
//
// Reference behaviour (paths under /root/reference/pkg/src/hrt):
//   bench/jacobi.py:70-79   _update_body: 7-point update, sum order
//                           (((((xm+xp)+ym)+yp)+zm)+zp) and IEEE /6.0
//   bench/jacobi.py:102-124 halo pack/unpack bodies (plane copies)
//   bench/jacobi.py:219-273 per-step protocol: pack, send, unpack, update
//   bench/jacobi.py:425-436 gather and checksum float(np.sum(assembled))
//
// B200 design:
//   * every chunk lives in HBM as two ghosted float64 buffers; same-GPU halo
//     exchange is one launch of `halo_copy_kernel` that reads the neighbour's
//     boundary plane in place and writes this chunk's ghost plane (pack +
//     message + unpack fused into one plane copy; cross-GPU planes are read
//     over NVLink by the same kernel or exchanged with NCCL send/recv);
//   * one `slab_update_kernel` launch per step covers every chunk on the GPU
//     (block table), marching rows with a register window, 128-bit loads and
//     warp shuffles for the y neighbours, a fused L-inf residual
//     (warp-shuffle max + one 64-bit atomicMax per CTA);
//   * the division is Markstein's correction q=s*r; e=fma(-q,6,s); q=fma(e,r,q)
//     with r=RN(1/6), which is correctly rounded (== IEEE s/6.0) whenever
//     s/6 is normal; tiny/special inputs take the IEEE path.  Parity tests
//     check it bitwise against IEEE division on the GPU.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "hrt_common.cuh"


namespace hrt {

// ---------------------------------------------------------------------------
// arithmetic

// Out of line on purpose: inlined, ptxas if-converts the IEEE division and
// runs its Newton sequence for every cell (measured: the 3D kernel executed
// MUFU.RCP64H + 6 DFMA per cell and was issue-bound at 3.1 TB/s).
__device__ __noinline__ double div6_ieee(double s) { return __ddiv_rn(s, 6.0); }

__device__ __forceinline__ double div6(double s) {
#if HRT_IEEE_DIV
    return __ddiv_rn(s, 6.0);
#else
    const double r = 0x1.5555555555555p-3;  // RN(1/6)
    double q = __dmul_rn(s, r);
    const double e = -__fma_rn(q, 6.0, -s);  // exact remainder (sign of zero kept: -0/6 = -0)
    q = __fma_rn(e, r, q);
    const double a = fabs(s);
    if ((a < 0x1p-1019 && a != 0.0) || !(a <= 0x1p1000)) q = div6_ieee(s);
    return q;
#endif
}

// variant 3 (the independent check path of run_jacobi3d(check=True)):
// plain IEEE division, no Markstein correction
__device__ __forceinline__ double div6_sel(double s, int ieee) {
    return ieee ? __ddiv_rn(s, 6.0) : div6(s);
}

__device__ __forceinline__ double sum6(double xm, double xp, double ym, double yp, double zm,
                                       double zp) {
    double acc = __dadd_rn(xm, xp);
    acc = __dadd_rn(acc, ym);
    acc = __dadd_rn(acc, yp);
    acc = __dadd_rn(acc, zm);
    return __dadd_rn(acc, zp);
}

// running max of |differences| (never NaN for finite fields): one compare
// and a select, where fmax's NaN/signed-zero handling costs ~8 instructions
__device__ __forceinline__ double rmax_acc(double r, double a) { return a > r ? a : r; }

// non-negative doubles order like their bit patterns
__device__ __forceinline__ void resid_max(unsigned long long* slot, double v) {
    atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct ChunkBufs {
    double* b[2];
};

// ---------------------------------------------------------------------------
// slab update: (X,Y,1) domains.  Chunk layout: element (i,j) of the ghosted
// (ex+2, ey+2) chunk at base + origin + i*sx + j, with (1,1) 16-byte aligned
// and sx even, so every interior row starts 16-byte aligned.
//
// CTA = SLAB_THREADS threads covering 2*SLAB_THREADS columns; each thread owns
// two adjacent columns (one double2) and marches `rows` rows keeping the row
// above/at/below in registers; rows are fetched SLAB_U at a time.

constexpr int SLAB_THREADS = 128;
constexpr int SLAB_COLS = 2 * SLAB_THREADS;
constexpr int SLAB_U = 4;

// per chunk: where its boundary planes go for each buffer parity (fused
// halo push), face order FACES 0..3; stride = element step along the plane
struct ChunkPush {
    double* ptr[4][2];
    int64_t stride[4];
};
static_assert(sizeof(ChunkPush) == sizeof(hrt_push_t), "ChunkPush layout");

// per chunk: its own contiguous west/east ghost columns per parity (null:
// domain face, constant boundary value)
struct ChunkSide {
    const double* w[2];
    const double* e[2];
};
static_assert(sizeof(ChunkSide) == sizeof(hrt_side_t), "ChunkSide layout");

struct SlabArgs {
    const ChunkBufs* chunks;
    const ChunkPush* push;  // null unless the plan pushes its halo
    const ChunkSide* sides; // null: ghost columns in-buffer (read via the row span)
    const int* tiles;       // null: all tiles (dense); else (chunk, rb, cb) triples
    // cross-process IPC push sync (null arrived: none).  Tiles [0, n_edge)
    // of the tile list touch remote faces.
    unsigned long long* arrived;                 // [n_nbr] steps published to us
    unsigned long long* const* remote_slots;     // [n_nbr] our slot in each neighbour
    int n_nbr;
    unsigned int* edge_done;                     // per-parity edge-tile counter
    int64_t n_edge;
    unsigned long long tag;                      // this step + 1
    unsigned long long timeout_ns;
    int* err;
    int parity;
    int64_t ex, ey, sx, origin;
    int64_t rows;          // rows per CTA tile
    int64_t tiles_r, tiles_c;
    unsigned long long* resid;  // nullable: L-inf residual slot for this step
    double zghost;         // the two constant z ghosts (BOUNDARY)
    int ieee;              // LDG kernel: IEEE __ddiv_rn instead of Markstein (variant 3)
};

__global__ void __launch_bounds__(SLAB_THREADS)
slab_update_kernel(SlabArgs a) {
    const int64_t per_chunk = a.tiles_r * a.tiles_c;
    const int64_t t = blockIdx.x;
    const int64_t c = t / per_chunk;
    const int64_t rem = t - c * per_chunk;
    const int64_t rb = rem / a.tiles_c;
    const int64_t cb = rem - rb * a.tiles_c;
    const int tid = threadIdx.x;
    const int lane = tid & 31;

    const double* __restrict__ u = a.chunks[c].b[a.parity] + a.origin;
    double* __restrict__ w = a.chunks[c].b[a.parity ^ 1] + a.origin;

    const int64_t j = 1 + cb * SLAB_COLS + 2 * tid;   // ghosted column of .x
    const bool act = j <= a.ey;                       // .x is interior
    const bool both = j + 1 <= a.ey;                  // .y is interior
    const bool right_mem = (lane == 31) || (j + 2 > a.ey);  // next lane idle
    const int64_t i0 = 1 + rb * a.rows;
    const int64_t i1 = min(a.ex, i0 + a.rows - 1);
    const double zg = a.zghost;

    auto ld2 = [&](int64_t i) -> double2 {
        return act ? __ldg(reinterpret_cast<const double2*>(u + i * a.sx + j))
                   : make_double2(0.0, 0.0);
    };
    auto ldl = [&](int64_t i) -> double {
        return (act && lane == 0) ? __ldg(u + i * a.sx + j - 1) : 0.0;
    };
    auto ldr = [&](int64_t i) -> double {
        return (both && right_mem) ? __ldg(u + i * a.sx + j + 2) : 0.0;
    };
    // y-neighbours of a row: left of .x and right of .y
    auto nbrs = [&](double2 v, double el, double er, double& lx, double& ry) {
        double l = __shfl_up_sync(0xffffffffu, v.y, 1);
        double r = __shfl_down_sync(0xffffffffu, v.x, 1);
        lx = (lane == 0) ? el : l;
        ry = right_mem ? er : r;
    };

    double2 up = ld2(i0 - 1);
    double2 mid = ld2(i0);
    double lx, ry;
    {
        double el = ldl(i0), er = ldr(i0);
        nbrs(mid, el, er, lx, ry);
    }
    double rmax = 0.0;

    for (int64_t i = i0; i <= i1; i += SLAB_U) {
        double2 nb[SLAB_U];
        double el[SLAB_U], er[SLAB_U];
#pragma unroll
        for (int k = 0; k < SLAB_U; ++k) {
            const int64_t r = i + 1 + k;
            if (r <= i1 + 1) {
                nb[k] = ld2(r);
                el[k] = ldl(r);
                er[k] = ldr(r);
            } else {
                nb[k] = make_double2(0.0, 0.0);
                el[k] = er[k] = 0.0;
            }
        }
#pragma unroll
        for (int k = 0; k < SLAB_U; ++k) {
            const int64_t r = i + k;
            if (r > i1) break;  // uniform across the CTA
            const double2 dn = nb[k];
            if (act) {
                double2 o;
                o.x = div6_sel(sum6(up.x, dn.x, lx, mid.y, zg, zg), a.ieee);
                o.y = div6_sel(sum6(up.y, dn.y, mid.x, ry, zg, zg), a.ieee);
                double* dst = w + r * a.sx + j;
                if (both) {
                    *reinterpret_cast<double2*>(dst) = o;
                    rmax = rmax_acc(rmax_acc(rmax, fabs(__dsub_rn(o.x, mid.x))), fabs(__dsub_rn(o.y, mid.y)));
                } else {
                    dst[0] = o.x;
                    rmax = rmax_acc(rmax, fabs(__dsub_rn(o.x, mid.x)));
                }
            }
            double nlx, nry;
            nbrs(dn, el[k], er[k], nlx, nry);
            up = mid;
            mid = dn;
            lx = nlx;
            ry = nry;
        }
    }

    if (a.resid) {
        __shared__ double red[SLAB_THREADS / 32];
        rmax = warp_max(rmax);
        if (lane == 0) red[tid >> 5] = rmax;
        __syncthreads();
        if (tid == 0) {
            double m = red[0];
#pragma unroll
            for (int k = 1; k < SLAB_THREADS / 32; ++k) m = fmax(m, red[k]);
            resid_max(a.resid, m);
        }
    }
}

// ---------------------------------------------------------------------------
// slab update, TMA variant: one producer thread streams the tile's rows
// (each row segment incl. the two neighbour columns is one contiguous
// 16-byte-aligned span) global -> shared with cp.async.bulk into a ring of
// TMA_STAGES stages guarded by mbarriers (full: transaction bytes;
// empty: one arrival per consumer warp).  Consumer warps read a row once
// (double2 + left + right from shared memory: no shuffles, no edge loads),
// release the stage, and keep the 3-row window in registers.

constexpr int TMA_CONSUMER_WARPS = 4;
constexpr int TMA_THREADS = 32 * (TMA_CONSUMER_WARPS + 1);
constexpr int TMA_COLS = 64 * TMA_CONSUMER_WARPS;    // 2 columns per consumer thread
constexpr int TMA_ROW = TMA_COLS + 4;                // + cols j0-2, j0-1 .. j0+W, j0+W+1
constexpr int TMA_STAGES = 12;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Watchdog: a barrier that has not completed for 20 s means a protocol bug
// (or a stalled peer); trap so the launch fails loudly instead of hanging
// the GPU.  The clock is read once per 64 Ki polls.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    unsigned long long t0 = 0;
    unsigned n = 0;
    while (!mbar_try(bar, parity)) {
        if ((++n & 0xFFFFu) == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t0 == 0) t0 = t;
            else if (t - t0 > 20000000000ULL) __trap();
        }
    }
}
// A waiter that has nothing else to do (the producer thread when the ring is
// full): try_wait with a suspend-time hint parks the thread in hardware
// until the phase completes instead of spinning on issue slots the
// consumer warps need.
__device__ __forceinline__ bool mbar_try_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    unsigned long long t0 = 0;
    while (!mbar_try_sleep(bar, parity)) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t0 == 0) t0 = t;
        else if (t - t0 > 20000000000ULL) __trap();
    }
}
__device__ __forceinline__ void tma_row_load(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(TMA_THREADS)
slab_update_tma_kernel(SlabArgs a) {
    __shared__ alignas(128) double ring[TMA_STAGES][TMA_ROW];
    __shared__ alignas(8) uint64_t full[TMA_STAGES], empty[TMA_STAGES];
    __shared__ double red[TMA_CONSUMER_WARPS];

    const int64_t per_chunk = a.tiles_r * a.tiles_c;
    const int64_t t = blockIdx.x;
    const int64_t c = t / per_chunk;
    const int64_t rem = t - c * per_chunk;
    const int64_t rb = rem / a.tiles_c;
    const int64_t cb = rem - rb * a.tiles_c;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    const double* __restrict__ u = a.chunks[c].b[a.parity] + a.origin;
    double* __restrict__ w = a.chunks[c].b[a.parity ^ 1] + a.origin;
    const int64_t j0 = 1 + cb * TMA_COLS;
    const int64_t last = min(j0 + TMA_COLS - 1, a.ey);
    const uint32_t nload = (uint32_t)(((last - j0 + 4) + 1) & ~int64_t(1));
    const uint32_t bytes = nload * 8u;
    const int64_t i0 = 1 + rb * a.rows;
    const int64_t i1 = min(a.ex, i0 + a.rows - 1);
    const int nrows = (int)(i1 - i0 + 3);  // rows i0-1 .. i1+1

    if (tid == 0) {
        for (int s = 0; s < TMA_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TMA_CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    if (warp == TMA_CONSUMER_WARPS) {
        // producer
        if (lane == 0) {
            const double* src = u + (i0 - 1) * a.sx + (j0 - 2);
            for (int q = 0; q < nrows; ++q) {
                const int s = q % TMA_STAGES;
                if (q >= TMA_STAGES) mbar_wait(&empty[s], ((q / TMA_STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], bytes);
                tma_row_load(&ring[s][0], src + (int64_t)q * a.sx, bytes, &full[s]);
            }
        }
        return;
    }

    // consumers: thread owns columns j, j+1 -> ring positions p = 2*tid+2, +3
    const int64_t j = j0 + 2 * tid;
    const bool act = j <= a.ey;
    const bool both = j + 1 <= a.ey;
    const int p = 2 * tid + 2;
    const double zg = a.zghost;
    double rmax = 0.0;

    auto take = [&](int q, double2& v, double& l, double& r) {
        const int s = q % TMA_STAGES;
        mbar_wait(&full[s], (q / TMA_STAGES) & 1);
        v = *reinterpret_cast<const double2*>(&ring[s][p]);
        l = ring[s][p - 1];
        r = ring[s][p + 2];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs next TMA
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    };

    double2 up, mid, dn;
    double lx, ry, dl, dr, tl, tr;
    take(0, up, tl, tr);
    take(1, mid, lx, ry);
    for (int q = 2; q < nrows; ++q) {
        take(q, dn, dl, dr);
        if (act) {
            const int64_t r = i0 - 2 + q;
            double2 o;
            o.x = div6(sum6(up.x, dn.x, lx, mid.y, zg, zg));
            o.y = div6(sum6(up.y, dn.y, mid.x, ry, zg, zg));
            double* dst = w + r * a.sx + j;
            if (both) {
                *reinterpret_cast<double2*>(dst) = o;
                rmax = rmax_acc(rmax_acc(rmax, fabs(__dsub_rn(o.x, mid.x))), fabs(__dsub_rn(o.y, mid.y)));
            } else {
                dst[0] = o.x;
                rmax = rmax_acc(rmax, fabs(__dsub_rn(o.x, mid.x)));
            }
        }
        up = mid;
        mid = dn;
        lx = dl;
        ry = dr;
    }

    if (a.resid) {
        rmax = warp_max(rmax);
        if (lane == 0) red[warp] = rmax;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * TMA_CONSUMER_WARPS));
        if (tid == 0) {
            double m = red[0];
#pragma unroll
            for (int k = 1; k < TMA_CONSUMER_WARPS; ++k) m = fmax(m, red[k]);
            resid_max(a.resid, m);
        }
    }
}

// ---------------------------------------------------------------------------
// slab update, TMA variant with four columns per consumer thread (variant 2).
// Same ring protocol as above; per row a consumer thread does one barrier
// wait, two 16-byte + two 8-byte shared loads and two 16-byte global stores
// for four cells, with row pointers advanced by increments.
//
// GUARD=false is used when the solver guarantees a non-negative finite field
// (the reference's problem: interior >= 0, Dirichlet 1.0): the six-term sum
// then includes +1.0+1.0 and is >= 2, so s/6 >= 1/3 is a normal number and
// Markstein's correction is exactly IEEE division without the range check.

constexpr int T4_CONSUMER_WARPS = 4;
constexpr int T4_COLS = 128 * T4_CONSUMER_WARPS;  // 4 columns per consumer thread
constexpr int T4_STAGES = 11;  // 11 x 4128 B ring: within the 48 KB static limit

__device__ __forceinline__ double div6_fast(double s) {
    const double r = 0x1.5555555555555p-3;
    double q = __dmul_rn(s, r);
    const double e = -__fma_rn(q, 6.0, -s);  // see div6
    return __fma_rn(e, r, q);
}

template <bool GUARD>
__device__ __forceinline__ double div6_t(double s) {
    if constexpr (GUARD) return div6(s);
    else return div6_fast(s);
}

// ---- cross-process step flags (IPC push mode) ----
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// step tag-1 published by every neighbour = its edge tiles of the previous
// step are done.  A stuck neighbour raises *err after timeout_ns instead of
// hanging the GPU.
__device__ void sync_wait_neighbours(const SlabArgs& a) {
    const unsigned long long need = a.tag - 1;
    const unsigned long long t0 = globaltimer_ns();
    for (int k = 0; k < a.n_nbr; ++k) {
        while (ld_acquire_sys(a.arrived + k) < need) {
            if (globaltimer_ns() - t0 > a.timeout_ns) {
                atomicExch(a.err, 1);
                return;
            }
            __nanosleep(100);
        }
    }
    // peers wrote our ghost planes with generic stores; the producer reads
    // them with TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// the last edge tile of this step publishes tag to every neighbour
__device__ void sync_signal_neighbours(const SlabArgs& a) {
    unsigned int* cnt = a.edge_done + a.parity;
    const unsigned int old = atomicAdd(cnt, 1u);
    if (old == (unsigned int)(a.n_edge - 1)) {
        *cnt = 0;  // reused two steps later, after this kernel has ended
        __threadfence_system();
        for (int k = 0; k < a.n_nbr; ++k) st_release_sys(a.remote_slots[k], a.tag);
    }
}

// Producer side of the ring for one (chunk c, column block cb) strip, rows
// i0-1 .. i1+1 of buffer `parity`: one bulk copy per row into stage s.
template <int CW, int STAGES>
__device__ __forceinline__ void t4_produce(const SlabArgs& a, double (*ring)[128 * CW + 4],
                                           uint64_t* full, uint64_t* empty, int& s, uint32_t& ph,
                                           int64_t c, int64_t cb, int64_t i0, int64_t i1,
                                           int parity) {
    const int64_t j0 = 1 + cb * (128 * CW);
    const int64_t last = min(j0 + (128 * CW) - 1, a.ey);
    const int nrows = (int)(i1 - i0 + 3);
    const int64_t sx = a.sx;
    // Side-array mode: at a chunk's west/east face the neighbour value comes
    // from a contiguous ghost column, so the bulk copy covers only the
    // 16-byte-aligned interior span (no partial 128-byte lines) and this
    // thread writes the two neighbour values into the ring slots the span
    // would have used (positions 1 and last-j0+3; the copy never touches
    // them because chunk widths are even in this mode).  Loads run AH rows
    // ahead (ld.global.cg: L2, coherent with the pushing CTAs).
    const bool wside = a.sides != nullptr && cb == 0;
    const bool eside = a.sides != nullptr && last == a.ey;
    const double* sw = wside ? a.sides[c].w[parity] : nullptr;
    const double* se = eside ? a.sides[c].e[parity] : nullptr;
    const int64_t lo = wside ? j0 : j0 - 2;
    const int64_t hi = eside ? last : last + 2;
    const uint32_t bytes = (uint32_t)((((hi - lo + 1) + 1) & ~int64_t(1)) * 8);
    const int dst0 = wside ? 2 : 0;
    const int epos = (int)(last - j0) + 3;
    const double* src = a.chunks[c].b[parity] + a.origin + (i0 - 1) * sx + lo;
    // row of ring position q is i0-1+q; side element of row r is [r-1]
    constexpr int AH = 4;  // rows of look-ahead (~1.5 us at the per-CTA row rate)
    double wv[AH], ev[AH];
    const bool sides = wside || eside;
    if (sides) {
#pragma unroll
        for (int u = 0; u < AH; ++u) {
            const int64_t r = i0 - 1 + u;  // rows outside 1..ex are never used
            const bool ok = u < nrows && r >= 1 && r <= a.ex;
            wv[u] = !wside ? 0.0 : (sw && ok ? __ldcg(sw + r - 1) : HRT_BOUNDARY);
            ev[u] = !eside ? 0.0 : (se && ok ? __ldcg(se + r - 1) : HRT_BOUNDARY);
        }
    }
    for (int qb = 0; qb < nrows; qb += AH) {
#pragma unroll
        for (int u = 0; u < AH; ++u) {
            const int q = qb + u;
            if (q >= nrows) break;
            mbar_wait(&empty[s], ph ^ 1);  // (a fresh barrier passes parity 1 at once)
            if (sides) {
                if (wside) ring[s][1] = wv[u];
                if (eside) ring[s][epos] = ev[u];
                const int64_t r = i0 - 1 + q + AH;  // refill this slot AH rows ahead
                const bool ok = q + AH < nrows && r >= 1 && r <= a.ex;
                if (wside) wv[u] = (sw && ok) ? __ldcg(sw + r - 1) : HRT_BOUNDARY;
                if (eside) ev[u] = (se && ok) ? __ldcg(se + r - 1) : HRT_BOUNDARY;
            }
            mbar_expect_tx(&full[s], bytes);
            tma_row_load(&ring[s][dst0], src, bytes, &full[s]);
            src += sx;
            if (++s == STAGES) {
                s = 0;
                ph ^= 1;
            }
        }
    }
}

// Consumer side for the same strip: output rows i0 .. i1 into buffer
// parity^1 (+ the fused halo push), residual folded into rmax.
template <bool GUARD, bool RESID, int CW, bool PUSH, int STAGES>
__device__ __forceinline__ void t4_consume(const SlabArgs& a, double (*ring)[128 * CW + 4],
                                           uint64_t* full, uint64_t* empty, int& s, uint32_t& ph,
                                           int64_t c, int64_t cb, int64_t i0, int64_t i1,
                                           int parity, double& rmax) {
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int64_t j0 = 1 + cb * (128 * CW);
    const int nrows = (int)(i1 - i0 + 3);
    const int64_t sx = a.sx;
    const int64_t j = j0 + 4 * tid;
    const int64_t nv64 = a.ey - j + 1;
    const int nv = nv64 <= 0 ? 0 : (nv64 >= 4 ? 4 : (int)nv64);  // valid columns
    const int p = 4 * tid + 2;
    double* __restrict__ wr = a.chunks[c].b[parity ^ 1] + a.origin + i0 * sx + j;
    // push targets of this chunk for the buffer being written (face order
    // north, south, west, east = FACES 0..3); null: domain face
    // (row planes are contiguous in both targets: in-buffer ghost rows and
    // staging slots; column planes step by sx or 1)
    double *pn = nullptr, *ps = nullptr, *pwp = nullptr, *pep = nullptr;
    int64_t sw = 0, se = 0;
    bool pw_on = false, pe_on = false;
    int qrow_n = -1, qrow_s = -1, ke = 0;
    if (PUSH) {
        const ChunkPush* cp = a.push + c;
        const int wp = parity ^ 1;
        pn = cp->ptr[0][wp];
        ps = cp->ptr[1][wp];
        double* pw = cp->ptr[2][wp];
        double* pe = cp->ptr[3][wp];
        sw = cp->stride[2];
        se = cp->stride[3];
        if (pn && i0 == 1) qrow_n = 2;                      // output row 1 is this strip's first
        if (ps && i1 == a.ex) qrow_s = (int)(i1 - i0) + 2;  // output row ex is its last
        pw_on = pw != nullptr && j == 1;
        pe_on = pe != nullptr && nv > 0 && j + nv - 1 == a.ey;
        ke = nv - 1;
        if (pw_on) pwp = pw + (i0 - 1) * sw;
        if (pe_on) pep = pe + (i0 - 1) * se;
    }

    auto take = [&](double (&v)[4], double& l, double& r) {
        mbar_wait(&full[s], ph);
        const double2 v01 = *reinterpret_cast<const double2*>(&ring[s][p]);
        const double2 v23 = *reinterpret_cast<const double2*>(&ring[s][p + 2]);
        l = ring[s][p - 1];
        r = ring[s][p + 4];
        // the next TMA write into this stage is an async-proxy access: order
        // this warp's generic-proxy reads before it (without this fence the
        // ring races; measured on B200)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == STAGES) {
            s = 0;
            ph ^= 1;
        }
        v[0] = v01.x;
        v[1] = v01.y;
        v[2] = v23.x;
        v[3] = v23.y;
    };

    double up[4], mid[4], dn[4], lx, ry, dl, dr, tl, tr;
    take(up, tl, tr);
    take(mid, lx, ry);
    const double zg = a.zghost;
    for (int q = 2; q < nrows; ++q) {
        take(dn, dl, dr);
        double o[4];
        o[0] = div6_t<GUARD>(sum6(up[0], dn[0], lx, mid[1], zg, zg));
        o[1] = div6_t<GUARD>(sum6(up[1], dn[1], mid[0], mid[2], zg, zg));
        o[2] = div6_t<GUARD>(sum6(up[2], dn[2], mid[1], mid[3], zg, zg));
        o[3] = div6_t<GUARD>(sum6(up[3], dn[3], mid[2], ry, zg, zg));
        if (nv == 4) {
            *reinterpret_cast<double2*>(wr) = make_double2(o[0], o[1]);
            *reinterpret_cast<double2*>(wr + 2) = make_double2(o[2], o[3]);
            if (RESID) {
#pragma unroll
                for (int k = 0; k < 4; ++k) rmax = rmax_acc(rmax, fabs(__dsub_rn(o[k], mid[k])));
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < nv) {
                    wr[k] = o[k];
                    if (RESID) rmax = rmax_acc(rmax, fabs(__dsub_rn(o[k], mid[k])));
                }
        }
        if (PUSH) {
            // fused halo: boundary rows/columns of the new field go straight
            // into the neighbours' ghost planes of the same buffer parity
            // (same GPU, a peer GPU over NVLink, or a packed NCCL staging
            // slot) — the reference's pack -> mp_send -> unpack (jacobi.py:
            // 102-124, 237) as extra stores of the producing kernel.  All
            // predicates are hoisted; per row this is two predicated stores.
            if (pw_on) {
                *pwp = o[0];
                pwp += sw;
            }
            if (pe_on) {
                *pep = ke == 3 ? o[3] : (ke == 2 ? o[2] : (ke == 1 ? o[1] : o[0]));
                pep += se;
            }
            if (q == qrow_n) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < nv) pn[j - 1 + k] = o[k];
            }
            if (q == qrow_s) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < nv) ps[j - 1 + k] = o[k];
            }
        }
        wr += sx;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            up[k] = mid[k];
            mid[k] = dn[k];
        }
        lx = dl;
        ry = dr;
    }
}

template <bool GUARD, bool RESID, int CW = T4_CONSUMER_WARPS, bool PUSH = false,
          int STAGES = T4_STAGES>
__global__ void __launch_bounds__(32 * (CW + 1), CW == 2 ? 9 : 1)
slab_update_tma4_kernel(SlabArgs a) {
    __shared__ alignas(128) double ring[STAGES][(128 * CW + 4)];
    __shared__ alignas(8) uint64_t full[STAGES], empty[STAGES];
    __shared__ double red[CW];

    int64_t c, rb, cb;
    if (a.tiles) {  // explicit tile subset (split schedule)
        const int* tt = a.tiles + 3 * (int64_t)blockIdx.x;
        c = tt[0];
        rb = tt[1];
        cb = tt[2];
    } else {
        const int64_t per_chunk = a.tiles_r * a.tiles_c;
        const int64_t t = blockIdx.x;
        c = t / per_chunk;
        const int64_t rem = t - c * per_chunk;
        rb = rem / a.tiles_c;
        cb = rem - rb * a.tiles_c;
    }
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    const int64_t j0 = 1 + cb * (128 * CW);
    if (j0 > a.ey) return;  // (uniform) no interior columns in this tile
    const int64_t i0 = 1 + rb * a.rows;
    const int64_t i1 = min(a.ex, i0 + a.rows - 1);
    // cross-process edge tile (IPC push mode): wait until every remote
    // neighbour finished its edge tiles of the previous step — their pushes
    // into our ghost planes have landed (RAW) and they no longer read the
    // ghost planes we are about to push into (WAR).  Inner tiles never wait.
    const bool xedge = a.arrived != nullptr && (int64_t)blockIdx.x < a.n_edge;

    if (tid == 0) {
        if (xedge) sync_wait_neighbours(a);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    int s = 0;
    uint32_t ph = 0;
    if (warp == CW) {
        if (lane == 0) t4_produce<CW, STAGES>(a, ring, full, empty, s, ph, c, cb, i0, i1, a.parity);
        return;
    }
    double rmax = 0.0;
    t4_consume<GUARD, RESID, CW, PUSH, STAGES>(a, ring, full, empty, s, ph, c, cb, i0, i1,
                                               a.parity, rmax);

    if (RESID) {
        rmax = warp_max(rmax);
        if (lane == 0) red[warp] = rmax;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * CW));
        if (tid == 0) {
            double m = red[0];
#pragma unroll
            for (int k = 1; k < CW; ++k) m = fmax(m, red[k]);
            resid_max(a.resid, m);
        }
    }
    if (xedge) {
        // our pushes (peer stores over NVLink) are visible system-wide before
        // the last edge tile of this step publishes the step to neighbours
        __threadfence_system();
        asm volatile("bar.sync 2, %0;" ::"n"(32 * CW));
        if (tid == 0) sync_signal_neighbours(a);
    }
}

// ---------------------------------------------------------------------------
// Persistent wavefront slab kernel (many steps per launch).  Resident CTAs
// claim tickets from one global counter; ticket t is tile (t mod T) of step
// (t div T), tiles as in slab_update_tma4_kernel (chunk, row block, column
// block).  A tile of step k runs once it and its four stencil neighbours —
// across chunk faces through the plan's neighbour table, whose halo pushes
// it receives — have published step k-1 in their per-tile counters: RAW on
// their new values and pushed ghosts, WAR on the buffer it overwrites.
// Dynamic claiming balances fast and slow SMs like a normal launch, there is
// no grid barrier and no per-step launch ramp/tail, and the producer warp
// prefetches the next tile into the ring while the consumers finish the
// current one.  Deadlock-free: tickets are claimed in order by co-resident
// CTAs (cooperative launch), so the oldest unfinished tile's dependencies
// have all been claimed earlier and finish.  Every dependency spin has a
// globaltimer timeout that sets *err (the producer then stops waiting but
// keeps feeding the ring, so the kernel always terminates).

struct WaveArgs {
    SlabArgs s;
    const int* nbr;               // [nchunks][4] neighbour chunk (N,S,W,E) or -1
    unsigned int* done;           // [T] steps completed per tile (absolute)
    unsigned long long* ticket;   // claim counter, 0 at launch
    unsigned int base;            // every done[] at launch
    int nsteps;
    int parity0;
    int64_t ntiles;               // T
    unsigned long long* resid;    // nullable: slots for this launch's steps
    // cross-process faces (CUDA IPC, same tiling on every rank); null: none
    const int* rnbr;              // [nchunks][4] chunk index in the neighbour rank's plan
    const int* rpeer;             // [nchunks][4] peer slot or -1
    unsigned int* const* peer_done;  // [peers] mapped tile counters of each peer
};

__device__ __forceinline__ unsigned int ld_acquire_gpu_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Wait until every counter q[d] (null: none) reaches `need`.  The loads are
// relaxed and independent, so all round trips overlap; one fence afterwards
// gives them acquire semantics (system scope when any counter lives in
// another process's memory).  Returns false after a timeout (sets *err).
template <int ND>
__device__ __forceinline__ bool wait_counters(const unsigned int* const (&q)[ND],
                                              const bool (&sys)[ND], unsigned need,
                                              unsigned long long timeout_ns, int* err) {
    unsigned v[ND];
    bool any_sys = false;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        any_sys |= q[d] != nullptr && sys[d];
        if (!q[d]) v[d] = need;
        else if (sys[d])
            asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v[d]) : "l"(q[d]) : "memory");
        else
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v[d]) : "l"(q[d]) : "memory");
    }
    unsigned long long t0 = 0;
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int d = 0; d < ND; ++d) ok &= v[d] >= need;
        if (ok) break;
        if (t0 == 0) t0 = globaltimer_ns();
        else if (globaltimer_ns() - t0 > timeout_ns) {
            atomicExch(err, 2);
            return false;
        }
#pragma unroll
        for (int d = 0; d < ND; ++d)
            if (v[d] < need) {
                if (sys[d])
                    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v[d]) : "l"(q[d]) : "memory");
                else
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v[d]) : "l"(q[d]) : "memory");
            }
    }
    if (any_sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return true;
}

constexpr int WAVE_TQ = 4;  // tile descriptors in flight between producer and consumers

template <bool GUARD, bool RESID, int CW, int STAGES = T4_STAGES>
__global__ void __launch_bounds__(32 * (CW + 1), CW == 2 ? 9 : 1)
slab_wave_kernel(WaveArgs wa) {
    __shared__ alignas(128) double ring[STAGES][(128 * CW + 4)];
    __shared__ alignas(8) uint64_t full[STAGES], empty[STAGES], tq_full[WAVE_TQ],
        tq_empty[WAVE_TQ];
    __shared__ long long tq[WAVE_TQ];
    const SlabArgs& a = wa.s;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int64_t T = wa.ntiles;
    const int64_t per_chunk = a.tiles_r * a.tiles_c;
    const long long total = (long long)T * wa.nsteps;

    if (tid == 0) {
        for (int k = 0; k < STAGES; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], CW);
        }
        for (int k = 0; k < WAVE_TQ; ++k) {
            mbar_init(&tq_full[k], 1);
            mbar_init(&tq_empty[k], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    int s = 0;
    uint32_t ph = 0;
    if (warp == CW) {
        if (lane != 0) return;
        bool dead = false;
        int slot = 0;
        uint32_t tph = 0;
        for (;;) {
            const long long t = (long long)atomicAdd(wa.ticket, 1ull);
            mbar_wait(&tq_empty[slot], tph ^ 1);
            tq[slot] = t < total ? t : -1;
            mbar_arrive(&tq_full[slot]);
            if (++slot == WAVE_TQ) {
                slot = 0;
                tph ^= 1;
            }
            if (t >= total) break;
            const int k = (int)(t / T);
            const int64_t tile = t - (long long)k * T;
            const int64_t c = tile / per_chunk;
            const int64_t rem = tile - c * per_chunk;
            const int64_t rb = rem / a.tiles_c;
            const int64_t cb = rem - rb * a.tiles_c;
            if (!dead) {
                // this tile and its N/S/W/E neighbours must have finished step k-1
                const int* nb = wa.nbr + 4 * c;
                const unsigned need = wa.base + (unsigned)k;
                // this tile + its N/S/W/E neighbours (inside the chunk, the
                // adjacent chunk's boundary tile, or another rank's)
                const int64_t offN = (a.tiles_r - 1) * a.tiles_c + cb, offS = cb;
                const int64_t offW = rb * a.tiles_c + (a.tiles_c - 1), offE = rb * a.tiles_c;
                const unsigned int* q[5] = {wa.done + tile, nullptr, nullptr, nullptr, nullptr};
                bool sys[5] = {false, false, false, false, false};
                auto face = [&](int d, int f, bool inside, int64_t in_tile, int64_t off) {
                    if (inside) q[d] = wa.done + in_tile;
                    else if (nb[f] >= 0) q[d] = wa.done + nb[f] * per_chunk + off;
                    else if (wa.rpeer && wa.rpeer[4 * c + f] >= 0) {
                        q[d] = wa.peer_done[wa.rpeer[4 * c + f]] +
                               (int64_t)wa.rnbr[4 * c + f] * per_chunk + off;
                        sys[d] = true;
                    }
                };
                face(1, 0, rb > 0, tile - a.tiles_c, offN);
                face(2, 1, rb < a.tiles_r - 1, tile + a.tiles_c, offS);
                face(3, 2, cb > 0, tile - 1, offW);
                face(4, 3, cb < a.tiles_c - 1, tile + 1, offE);
                dead = !wait_counters<5>(q, sys, need, a.timeout_ns, a.err);
                // other CTAs' generic-proxy stores -> our async-proxy reads
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            const int64_t i0 = 1 + rb * a.rows;
            const int64_t i1 = min(a.ex, i0 + a.rows - 1);
            t4_produce<CW, STAGES>(a, ring, full, empty, s, ph, c, cb, i0, i1,
                                   (wa.parity0 + k) & 1);
        }
        return;
    }
    int slot = 0;
    uint32_t tph = 0;
    for (;;) {
        mbar_wait(&tq_full[slot], tph);
        const long long t = tq[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&tq_empty[slot]);
        if (++slot == WAVE_TQ) {
            slot = 0;
            tph ^= 1;
        }
        if (t < 0) break;
        const int k = (int)(t / T);
        const int64_t tile = t - (long long)k * T;
        const int64_t c = tile / per_chunk;
        const int64_t rem = tile - c * per_chunk;
        const int64_t rb = rem / a.tiles_c;
        const int64_t cb = rem - rb * a.tiles_c;
        const int64_t i0 = 1 + rb * a.rows;
        const int64_t i1 = min(a.ex, i0 + a.rows - 1);
        double rmax = 0.0;
        t4_consume<GUARD, RESID, CW, true, STAGES>(a, ring, full, empty, s, ph, c, cb, i0, i1,
                                                   (wa.parity0 + k) & 1, rmax);
        if (RESID && wa.resid) {
            rmax = warp_max(rmax);
            if (lane == 0) resid_max(wa.resid + k, rmax);
        }
        // our stores -> later async-proxy reads (TMA of any CTA); then one
        // thread publishes the tile's step once every consumer warp is done.
        // Tiles on a cross-process face pushed over NVLink into a neighbour
        // rank's memory: system-scope fence + release for those.
        const int* rp = wa.rpeer ? wa.rpeer + 4 * c : nullptr;
        const bool xedge = rp && ((rb == 0 && rp[0] >= 0) || (rb == a.tiles_r - 1 && rp[1] >= 0) ||
                                  (cb == 0 && rp[2] >= 0) || (cb == a.tiles_c - 1 && rp[3] >= 0));
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (xedge) __threadfence_system();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * CW));
        if (tid == 0) {
            const unsigned v = wa.base + (unsigned)k + 1u;
            if (xedge) {
                __threadfence_system();
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(wa.done + tile), "r"(v)
                             : "memory");
            } else {
                __threadfence();
                st_release_gpu_u32(wa.done + tile, v);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Two steps per pass (temporal blocking) for slabs of one GPU.  A tile of
// fused step k reads u(t) once — its rows i0-2 .. i1+2 and columns
// j0-2 .. j0+W+1, straight from whichever chunk owns them (the 3 x 3 chunk
// neighbourhood: no ghost planes, no pushes) — computes u(t+1) on the tile
// plus a one-cell rim in registers (cells outside the domain keep the
// Dirichlet value, as the reference's ghost shell does), then u(t+2) on the
// tile, and writes only u(t+2): 8 B of HBM per lattice update instead of 16.
// Every value is produced by the same IEEE operations in the reference's
// order (the rim cells exactly as their owner computes them), so the field
// and both residuals per pass stay bitwise identical.  Dependencies: a tile
// of fused step k needs its 3 x 3 tile neighbourhood done with step k-1
// (RAW on u(t), and WAR on the buffer it overwrites, which those tiles read
// as rim); counters count steps (2 per pass).

// The 3 x 3 chunk neighbourhood of a chunk, (di+1)*3+(dj+1): the buffers
// (this process's, or another process's mapped over CUDA IPC) and the base
// of that chunk's tile counters; null outside the domain.
struct Nbr9 {
    double* b[9][2];
    unsigned int* cnt[9];
    unsigned int sysmask;        // bit d: counters in another process (system scope)
    unsigned int pad_;
};

struct Wave2Args {
    const Nbr9* n9;              // [nchunks]
    unsigned int* done;          // [T] steps completed per tile (absolute)
    unsigned long long* ticket;
    unsigned int base;           // every done[] at launch
    int nfused;                  // passes (2 steps each)
    int parity0;                 // buffer holding u(first)
    int64_t ntiles, ex, ey, sx, origin, rows, tiles_r, tiles_c;
    unsigned long long* resid;   // nullable: 2 * nfused slots
    const double* ones;          // a BOUNDARY row source for rows outside the domain
    unsigned long long timeout_ns;
    int* err;
    double zghost;
};

// rows i0-2 .. i1+2 of u(t) into the ring: the span j0-2 .. j0+W+1 (or the
// owning chunk's part of it at a chunk's west/east edge, plus 16 bytes from
// the west/east neighbour chunk's same row), BOUNDARY where outside.
template <int W, int STAGES>
__device__ __forceinline__ void w2_produce(const Wave2Args& a, double (*ring)[W + 4],
                                           uint64_t* full, uint64_t* empty, int& s,
                                           uint32_t& ph, int64_t c, int64_t cb, int64_t i0,
                                           int64_t i1, int parity) {
    const int64_t j0 = 1 + cb * W;
    const int64_t last = min(j0 + W - 1, a.ey);
    const Nbr9* n9 = a.n9 + c;
    const bool wedge = cb == 0, eedge = last == a.ey;
    const int64_t lo = wedge ? 1 : j0 - 2;
    const int64_t hi = eedge ? a.ey : last + 2;
    const uint32_t mbytes = (uint32_t)((hi - lo + 1) * 8);  // even count: ey even
    const int mpos = (int)(lo - (j0 - 2));
    const int epos = (int)(last - j0 + 3);
    // three row segments (north chunk rows, own rows, south chunk rows):
    // the sources are fixed per segment, so the row loop only advances
    // pointers (a table load per row stalled the producer thread)
    int64_t r = i0 - 2;
    const int64_t rend = i1 + 2;
#pragma unroll 1
    for (int di = -1; di <= 1; ++di) {
        const int64_t cap = di < 0 ? 0 : (di == 0 ? a.ex : rend);
        const int64_t seg_end = rend < cap ? rend : cap;
        if (r > seg_end) continue;
        const double* br = n9->b[(di + 1) * 3 + 1][parity];
        const double* bw = (br && wedge) ? n9->b[(di + 1) * 3 + 0][parity] : nullptr;
        const double* be = (br && eedge) ? n9->b[(di + 1) * 3 + 2][parity] : nullptr;
        const int64_t rr = r - di * a.ex;
        const double* msrc = br ? br + a.origin + rr * a.sx + lo : a.ones;
        const double* wsrc = bw ? bw + a.origin + rr * a.sx + (a.ey - 1) : nullptr;
        const double* esrc = be ? be + a.origin + rr * a.sx + 1 : nullptr;
        const int64_t mstep = br ? a.sx : 0;
        const uint32_t bytes = mbytes + (wsrc ? 16u : 0u) + (esrc ? 16u : 0u);
        const bool wfill = wedge && !wsrc, efill = eedge && !esrc;
#pragma unroll 1
        for (; r <= seg_end; ++r) {
            mbar_wait_sleep(&empty[s], ph ^ 1);
            if (wfill) {
                ring[s][0] = HRT_BOUNDARY;
                ring[s][1] = HRT_BOUNDARY;
            }
            if (efill) {
                ring[s][epos] = HRT_BOUNDARY;
                ring[s][epos + 1] = HRT_BOUNDARY;
            }
            mbar_expect_tx(&full[s], bytes);
            tma_row_load(&ring[s][mpos], msrc, mbytes, &full[s]);
            if (wsrc) {
                tma_row_load(&ring[s][0], wsrc, 16, &full[s]);
                wsrc += a.sx;
            }
            if (esrc) {
                tma_row_load(&ring[s][epos], esrc, 16, &full[s]);
                esrc += a.sx;
            }
            msrc += mstep;
            if (++s == STAGES) {
                s = 0;
                ph ^= 1;
            }
        }
    }
}

// ---- shared-memory helpers on 32-bit shared addresses (computed once per
// tile: a generic->shared conversion per row cost an S2R of the CTA id, a
// LEA and an IMAD on every row) ----
__device__ __forceinline__ bool mbar_try_u32(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __noinline__ void mbar_wait_u32_slow(uint32_t bar, uint32_t parity) {
    unsigned long long t0 = 0;
    unsigned n = 0;
    while (!mbar_try_u32(bar, parity)) {
        if ((++n & 0xFFFFu) == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t0 == 0) t0 = t;
            else if (t - t0 > 20000000000ULL) __trap();
        }
    }
}
// one lane arrives (a predicated instruction: no divergent branch)
__device__ __forceinline__ void mbar_arrive_lane0_u32(uint32_t bar, int lane) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.eq.s32 p, %1, 0;\n\t"
        "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(bar),
        "r"(lane)
        : "memory");
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}
// |x| on the integer pipe (a DADD with |.| would take an FP64 issue slot)
__device__ __forceinline__ double abs_bits(double x) {
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// Per-thread state of the two-step consumer (one tile).
struct W2Ctx {
    uint32_t ring;          // shared address of this thread's column span in stage 0
    uint32_t full, empty;   // shared addresses of the barrier arrays
    int s;
    uint32_t ph;
    bool ready;             // the current stage's full barrier was seen complete
    int lane, nv;
    unsigned cghost;
    bool mask, out_n, out_s;
    int qlast;              // last ring row whose u(t+1) row is inside the tile
    int64_t i0, ex, sx;
    double* wr;
    double zg, r1, r2;
};

// Take the next ring row: wait for its stage (unless an earlier poll saw it
// complete), read this thread's span, hand the stage back to the producer,
// and poll the following stage now so its barrier latency overlaps this
// row's arithmetic instead of stalling the next take.
template <int RS, int STAGES, int NP>
__device__ __forceinline__ void w2_take(W2Ctx& x, double2 (&v)[NP]) {
    const uint32_t fb = x.full + 8u * (uint32_t)x.s;
    if (!x.ready && !mbar_try_u32(fb, x.ph)) mbar_wait_u32_slow(fb, x.ph);
    const uint32_t row = x.ring + (uint32_t)(x.s * RS * 8);
#pragma unroll
    for (int k = 0; k < NP; ++k) v[k] = lds_f64x2(row + 16u * k);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs the next TMA
    __syncwarp();
    mbar_arrive_lane0_u32(x.empty + 8u * (uint32_t)x.s, x.lane);
    if (++x.s == STAGES) {
        x.s = 0;
        x.ph ^= 1;
    }
    x.ready = mbar_try_u32(x.full + 8u * (uint32_t)x.s, x.ph);
}

template <int NP>
__device__ __forceinline__ double w2_e(const double2 (&v)[NP], int m) {
    return (m & 1) ? v[m >> 1].y : v[m >> 1].x;
}

// one ring row q: u(t) row r+1 arrives in `dn`; u(t+1) row r (r = i0-3+q)
// goes into `u1n` (the slot of row r-3); u(t+2) row r-1 from u(t+1) rows
// r-2 (`u1a`), r-1 (`u1b`), r (`u1n`).  Per-row residual maxima are folded
// as a tree (two independent compares, then one into the running max).
template <bool GUARD, bool RESID, bool FULL, int RS, int STAGES, int CPT>
__device__ __forceinline__ void w2_row(W2Ctx& x, const double2 (&up)[CPT / 2 + 2],
                                       const double2 (&mid)[CPT / 2 + 2],
                                       double2 (&dn)[CPT / 2 + 2], const double (&u1a)[CPT + 2],
                                       const double (&u1b)[CPT + 2], double (&u1n)[CPT + 2],
                                       int q) {
    static_assert(CPT == 4, "the residual tree assumes four columns per thread");
    w2_take<RS, STAGES, CPT / 2 + 2>(x, dn);
    const double zg = x.zg;
#pragma unroll
    for (int m = 0; m < CPT + 2; ++m)
        u1n[m] = div6_t<GUARD>(sum6(w2_e(up, m + 1), w2_e(dn, m + 1), w2_e(mid, m),
                                    w2_e(mid, m + 2), zg, zg));
    if (x.mask) {
        const int64_t r = x.i0 - 3 + q;
        const bool rghost = (r < 1 && x.out_n) || (r > x.ex && x.out_s);
#pragma unroll
        for (int m = 0; m < CPT + 2; ++m)
            if (rghost || ((x.cghost >> m) & 1u)) u1n[m] = HRT_BOUNDARY;
    }
    if (RESID && q >= 3 && q <= x.qlast) {  // u(t+1) row r = i0-3+q inside [i0, i1]
        double d[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k)
            d[k] = (FULL || k < x.nv) ? abs_bits(__dsub_rn(u1n[k + 1], w2_e(mid, k + 2))) : 0.0;
        x.r1 = dmax(x.r1, dmax(dmax(d[0], d[1]), dmax(d[2], d[3])));
    }
    if (q >= 4) {
        double o[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k)
            o[k] = div6_t<GUARD>(sum6(u1a[k + 1], u1n[k + 1], u1b[k], u1b[k + 2], zg, zg));
        if (FULL) {
#pragma unroll
            for (int k = 0; k < CPT; k += 2)
                *reinterpret_cast<double2*>(x.wr + k) = make_double2(o[k], o[k + 1]);
        } else {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                if (k < x.nv) x.wr[k] = o[k];
        }
        if (RESID) {
            double d[CPT];
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                d[k] = (FULL || k < x.nv) ? abs_bits(__dsub_rn(o[k], u1b[k + 1])) : 0.0;
            x.r2 = dmax(x.r2, dmax(dmax(d[0], d[1]), dmax(d[2], d[3])));
        }
        x.wr += x.sx;
    }
}

template <bool GUARD, bool RESID, bool FULL, int RS, int STAGES, int CPT>
__device__ __forceinline__ void w2_rows(W2Ctx& x, int nrows) {
    double2 x0[CPT / 2 + 2], x1[CPT / 2 + 2], x2[CPT / 2 + 2];  // u(t) rows, rotating
    double y0[CPT + 2], y1[CPT + 2], y2[CPT + 2];              // u(t+1) rows, rotating
    w2_take<RS, STAGES, CPT / 2 + 2>(x, x0);                     // row i0-2
    w2_take<RS, STAGES, CPT / 2 + 2>(x, x1);                     // row i0-1
    int q = 2;
    for (; q + 2 < nrows; q += 3) {
        w2_row<GUARD, RESID, FULL, RS, STAGES, CPT>(x, x0, x1, x2, y1, y2, y0, q);
        w2_row<GUARD, RESID, FULL, RS, STAGES, CPT>(x, x1, x2, x0, y2, y0, y1, q + 1);
        w2_row<GUARD, RESID, FULL, RS, STAGES, CPT>(x, x2, x0, x1, y0, y1, y2, q + 2);
    }
    if (q < nrows) w2_row<GUARD, RESID, FULL, RS, STAGES, CPT>(x, x0, x1, x2, y1, y2, y0, q);
    if (q + 1 < nrows)
        w2_row<GUARD, RESID, FULL, RS, STAGES, CPT>(x, x1, x2, x0, y2, y0, y1, q + 1);
}

// u(t+1) on rows i0-1 .. i1+1, columns j-1 .. j+4 of this thread (j = its
// first column), then u(t+2) on rows i0 .. i1, columns j .. j+3 -> buffer
// parity^1.  r1 / r2: max |u(t+1)-u(t)| / |u(t+2)-u(t+1)| over own cells.
// The row loop is unrolled by three with the u(t) and u(t+1) row windows
// rotating through three register arrays each (no moves); cells outside the
// domain are masked only in tiles that touch it (a uniform branch).
template <bool GUARD, bool RESID, bool FULL, int CW, int CPT, int STAGES>
__device__ __forceinline__ void w2_consume(const Wave2Args& a, uint32_t ring_u32,
                                           uint32_t full_u32, uint32_t empty_u32, int& s,
                                           uint32_t& ph, int64_t c, int64_t cb, int64_t i0,
                                           int64_t i1, int parity, double& r1, double& r2) {
    constexpr int W = 32 * CPT * CW;
    constexpr int RS = W + 4;
    const int tid = threadIdx.x;
    W2Ctx x;
    x.full = full_u32;
    x.empty = empty_u32;
    x.s = s;
    x.ph = ph;
    x.ready = false;
    x.lane = tid & 31;
    const int64_t j0 = 1 + cb * W;
    const int64_t j = j0 + CPT * tid;
    const int64_t nv64 = a.ey - j + 1;
    x.nv = nv64 <= 0 ? 0 : (nv64 >= CPT ? CPT : (int)nv64);
    x.ring = ring_u32 + 8u * (uint32_t)(CPT * tid);  // ring position of column j-2
    const int nrows = (int)(i1 - i0 + 5);
    const Nbr9& n9 = a.n9[c];
    x.out_n = !n9.b[1][0];
    x.out_s = !n9.b[7][0];
    const bool out_w = !n9.b[3][0], out_e = !n9.b[5][0];
    // u(t+1) columns j-1+m (m = 0..CPT+1) outside the domain keep BOUNDARY
    unsigned cghost = 0;
#pragma unroll
    for (int m = 0; m < CPT + 2; ++m) {
        const int64_t cc = j - 1 + m;
        if ((cc < 1 && out_w) || (cc > a.ey && out_e)) cghost |= 1u << m;
    }
    x.cghost = cghost;
    // does any u(t+1) value of this tile fall outside the domain?
    x.mask = __any_sync(0xffffffffu, cghost != 0) || (x.out_n && i0 <= 1) ||
             (x.out_s && i1 >= a.ex);
    x.i0 = i0;
    x.qlast = (int)(i1 - i0) + 3;
    x.ex = a.ex;
    x.sx = a.sx;
    x.wr = n9.b[4][parity ^ 1] + a.origin + i0 * a.sx + j;
    x.zg = a.zghost;
    x.r1 = r1;
    x.r2 = r2;

    w2_rows<GUARD, RESID, FULL, RS, STAGES, CPT>(x, nrows);
    s = x.s;
    ph = x.ph;
    r1 = x.r1;
    r2 = x.r2;
}

#ifndef HRT_W2_MINB4
#define HRT_W2_MINB4 3   // resident CTAs/SM the registers target: 512-wide tiles
#endif
#ifndef HRT_W2_MINB2
#define HRT_W2_MINB2 5   // 256-wide tiles (chunks at most 256 wide)
#endif
// CW consumer warps (4 columns per thread) + one producer warp
__host__ __device__ constexpr int w2_threads(int cw) { return 32 * (cw + 1); }
constexpr int w2_minb(int cw) { return cw == 2 ? HRT_W2_MINB2 : HRT_W2_MINB4; }
constexpr int W2_STAGES = T4_STAGES;
// FULL: the chunk width is a multiple of the tile width, so every thread
// owns CPT columns inside the chunk and the row body needs no column masks
template <bool GUARD, bool RESID, int CW, bool FULL = false, int CPT = 4,
          int STAGES = W2_STAGES>
__global__ void __launch_bounds__(w2_threads(CW), w2_minb(CW))
slab_wave2_kernel(Wave2Args wa) {
    __shared__ alignas(128) double ring[STAGES][(32 * CPT * CW + 4)];
    __shared__ alignas(8) uint64_t full[STAGES], empty[STAGES], tq_full[WAVE_TQ],
        tq_empty[WAVE_TQ];
    __shared__ long long tq[WAVE_TQ];
    __shared__ double red[2][CW];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int64_t T = wa.ntiles;
    const int64_t tr = wa.tiles_r, tc = wa.tiles_c;
    const int64_t per_chunk = tr * tc;
    const long long total = (long long)T * wa.nfused;

    if (tid == 0) {
        for (int k = 0; k < STAGES; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], CW);
        }
        for (int k = 0; k < WAVE_TQ; ++k) {
            mbar_init(&tq_full[k], 1);
            mbar_init(&tq_empty[k], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    int s = 0;
    uint32_t ph = 0;
    if (warp >= CW) {
        if (lane != 0) return;
        bool dead = false;
        int slot = 0;
        uint32_t tph = 0;
        for (;;) {
            const long long t = (long long)atomicAdd(wa.ticket, 1ull);
            mbar_wait(&tq_empty[slot], tph ^ 1);
            tq[slot] = t < total ? t : -1;
            mbar_arrive(&tq_full[slot]);
            if (++slot == WAVE_TQ) {
                slot = 0;
                tph ^= 1;
            }
            if (t >= total) break;
            const int k = (int)(t / T);
            const int64_t tile = t - (long long)k * T;
            const int64_t c = tile / per_chunk;
            const int64_t rem = tile - c * per_chunk;
            const int64_t rb = rem / tc;
            const int64_t cb = rem - rb * tc;
            if (!dead) {
                // the 3 x 3 tile neighbourhood must be done with step base+2k
                const unsigned need = wa.base + 2u * (unsigned)k;
                const Nbr9& n9 = wa.n9[c];
                const unsigned int* q[9];
                bool sys[9];
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    const int64_t r2 = rb + d / 3 - 1, c2 = cb + d % 3 - 1;
                    const int ci = r2 < 0 ? -1 : (r2 >= tr ? 1 : 0);
                    const int cj = c2 < 0 ? -1 : (c2 >= tc ? 1 : 0);
                    const int e = (ci + 1) * 3 + (cj + 1);
                    const unsigned int* base = n9.cnt[e];
                    q[d] = base ? base + (r2 - ci * tr) * tc + (c2 - cj * tc) : nullptr;
                    sys[d] = (n9.sysmask >> e) & 1u;
                }
                dead = !wait_counters<9>(q, sys, need, wa.timeout_ns, wa.err);
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            const int64_t i0 = 1 + rb * wa.rows;
            const int64_t i1 = min(wa.ex, i0 + wa.rows - 1);
            w2_produce<32 * CPT * CW, STAGES>(wa, ring, full, empty, s, ph, c, cb, i0, i1,
                                   (wa.parity0 + k) & 1);
        }
        return;
    }
    const uint32_t ring_u32 = smem_u32(&ring[0][0]);
    const uint32_t full_u32 = smem_u32(&full[0]), empty_u32 = smem_u32(&empty[0]);
    int slot = 0;
    uint32_t tph = 0;
    for (;;) {
        mbar_wait(&tq_full[slot], tph);
        const long long t = tq[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&tq_empty[slot]);
        if (++slot == WAVE_TQ) {
            slot = 0;
            tph ^= 1;
        }
        if (t < 0) break;
        const int k = (int)(t / T);
        const int64_t tile = t - (long long)k * T;
        const int64_t c = tile / per_chunk;
        const int64_t rem = tile - c * per_chunk;
        const int64_t rb = rem / tc;
        const int64_t cb = rem - rb * tc;
        const int64_t i0 = 1 + rb * wa.rows;
        const int64_t i1 = min(wa.ex, i0 + wa.rows - 1);
        double r1 = 0.0, r2 = 0.0;
        w2_consume<GUARD, RESID, FULL, CW, CPT, STAGES>(wa, ring_u32, full_u32, empty_u32, s, ph, c,
                                                  cb, i0, i1, (wa.parity0 + k) & 1, r1, r2);
        if (RESID && wa.resid) {
            r1 = warp_max(r1);
            r2 = warp_max(r2);
            if (lane == 0) {
                red[0][warp] = r1;
                red[1][warp] = r2;
            }
        }
        // a tile another process reads as rim (chunk edge facing it): its
        // stores must be visible system-wide before the counter says so
        const unsigned sm = wa.n9[c].sysmask;
        const bool xedge = sm && ((rb == 0 && (sm & 0x7u)) || (rb == tr - 1 && (sm & 0x1C0u)) ||
                                  (cb == 0 && (sm & 0x49u)) || (cb == tc - 1 && (sm & 0x124u)));
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (xedge) __threadfence_system();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * CW));
        if (tid == 0) {
            if (RESID && wa.resid) {
                double m1 = red[0][0], m2 = red[1][0];
#pragma unroll
                for (int w = 1; w < CW; ++w) {
                    m1 = fmax(m1, red[0][w]);
                    m2 = fmax(m2, red[1][w]);
                }
                resid_max(wa.resid + 2 * k, m1);
                resid_max(wa.resid + 2 * k + 1, m2);
            }
            const unsigned v = wa.base + 2u * (unsigned)k + 2u;
            if (xedge) {
                __threadfence_system();
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(wa.done + tile), "r"(v)
                             : "memory");
            } else {
                __threadfence();
                st_release_gpu_u32(wa.done + tile, v);
            }
        }
    }
}


// ---------------------------------------------------------------------------
// volume update, TMA variant.  Tile: V_CW consumer warps = V_CW y-rows
// (j0 .. j0+V_CW-1) x 64 z-columns (two per lane), marching planes i along x.
// Stage q holds plane i0-1+q of the tile plus its y/z halo: V_CW+2 row spans
// of z = k0-2 .. k0+65, one 1D bulk copy each (rows 16-byte aligned by the
// layout).  A thread keeps the x window (plane i-1, i, i+1 at its (j,k)) in
// registers and reads the y/z neighbours of plane i from its stage, which is
// released once plane i is computed.  Sum order (((((xm+xp)+ym)+yp)+zm)+zp).

// Fused halo push for volumes: per chunk, face f (FACES order -x,+x,-y,+y,
// -z,+z) and parity of the buffer being written, the address that
// corresponds to this chunk's element offset 0 in the neighbour's ghost
// plane: target(i,j,k) = ptr[f][p] + (i*sx + j*sy + k).  Null: domain face.
struct VolPush {
    double* ptr[6][2];
};
static_assert(sizeof(VolPush) == sizeof(hrt_vpush_t), "VolPush layout");

struct VolArgs {
    const ChunkBufs* chunks;   // block table, or null: single chunk (du -> dw)
    const double* du;
    double* dw;
    int parity;
    int64_t ex, ey, ez, sx, sy, origin;
    int64_t rows;
    int64_t tiles_i, tiles_j, tiles_k;
    int flat;                  // ez == 1 stored with z ghosts: threads tile j only
    int ieee;                  // LDG kernel: IEEE __ddiv_rn instead of Markstein (variant 3)
    unsigned long long* resid;
    const VolPush* vpush;      // null: no fused push
};

#ifndef HRT_V_CW
#define HRT_V_CW 8        // consumer warps = y rows per volume tile
#endif
#ifndef HRT_V_STAGES
#define HRT_V_STAGES 8    // ring stages (planes in flight per CTA)
#endif
#ifndef HRT_V_MINB
#define HRT_V_MINB 4      // resident CTAs per SM the register budget targets
#endif
constexpr int V_CW = HRT_V_CW;
constexpr int V_ZW = 64;               // z columns per tile
constexpr int V_ZROW = V_ZW + 4;       // + k0-2, k0-1, k0+64, k0+65
constexpr int V_ROWS = V_CW + 2;       // y rows per stage (with halo)
constexpr int V_STAGES = HRT_V_STAGES;
// the ring lives in dynamic shared memory (more than the 48 KB static cap
// for taller tiles / deeper rings)
constexpr size_t V_SMEM = sizeof(double) * V_STAGES * V_ROWS * V_ZROW;

// Producer for one volume tile: planes i0-1 .. i1+1, each stage = the tile's
// V_CW+2 y-rows of z = k0-2 .. k0+65 (one bulk copy per row).
__device__ __forceinline__ void v_produce(const VolArgs& a, double (*ring)[V_ROWS][V_ZROW],
                                          uint64_t* full, uint64_t* empty, int& s, uint32_t& ph,
                                          int64_t c, int64_t i0, int64_t i1, int64_t j0,
                                          int64_t k0, int parity) {
    const int64_t klast = min(k0 + V_ZW - 1, a.ez);
    const uint32_t bytes = (uint32_t)((((klast - k0 + 4) + 1) & ~int64_t(1)) * 8);
    // stage rows j0-1 .. j0+V_CW, but never beyond the ghost row ey+1
    const int64_t nyr64 = a.ey + 2 - (j0 - 1);
    const int nyr = nyr64 < V_ROWS ? (int)nyr64 : V_ROWS;
    const int nplanes = (int)(i1 - i0 + 3);
    const double* src = a.chunks[c].b[parity] + a.origin + (i0 - 1) * a.sx + (j0 - 1) * a.sy +
                        (k0 - 2);
    for (int q = 0; q < nplanes; ++q) {
        mbar_wait(&empty[s], ph ^ 1);  // (a fresh barrier passes parity 1 at once)
        mbar_expect_tx(&full[s], bytes * (uint32_t)nyr);
        for (int r = 0; r < nyr; ++r) tma_row_load(&ring[s][r][0], src + r * a.sy, bytes, &full[s]);
        src += a.sx;
        if (++s == V_STAGES) {
            s = 0;
            ph ^= 1;
        }
    }
}

// Consumer for the same tile (warp = y-row, lane = 2 z-columns): output
// planes i0..i1 into buffer parity^1, plus the fused push of boundary cells.
template <bool GUARD, bool RESID, bool PUSH>
__device__ __forceinline__ void v_consume(const VolArgs& a, double (*ring)[V_ROWS][V_ZROW],
                                          uint64_t* full, uint64_t* empty, int& s, uint32_t& ph,
                                          int64_t c, int64_t i0, int64_t i1, int64_t j0,
                                          int64_t k0, int parity, double& rmax) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nplanes = (int)(i1 - i0 + 3);
    const int64_t j = j0 + warp;
    const int64_t k = k0 + 2 * lane;
    const bool act = (j <= a.ey) && (k <= a.ez);
    const bool both = act && (k + 1 <= a.ez);
    const int r = warp + 1;   // this thread's row in a stage
    const int p = 2 * lane + 2;
    const int64_t off0 = i0 * a.sx + j * a.sy + k;  // element offset of the first output
    double* __restrict__ wr = a.chunks[c].b[parity ^ 1] + a.origin + off0;
    // push faces of this thread as a bitmask (registers are what limits the
    // volume kernels' occupancy); targets are rebuilt at the rare boundary
    // stores: x faces at the chunk's first/last plane, y faces for the
    // boundary rows, z faces for the boundary columns (k = 1 is .x; k = ez
    // is .x or .y)
    unsigned pm = 0;
    if (PUSH && act) {
        const VolPush* vp = a.vpush + c;
        const int wp = parity ^ 1;
        if (i0 == 1 && vp->ptr[0][wp]) pm |= 1u;
        if (i1 == a.ex && vp->ptr[1][wp]) pm |= 2u;
        if (j == 1 && vp->ptr[2][wp]) pm |= 4u;
        if (j == a.ey && vp->ptr[3][wp]) pm |= 8u;
        if (k == 1 && vp->ptr[4][wp]) pm |= 16u;
        if ((k == a.ez || k + 1 == a.ez) && vp->ptr[5][wp]) pm |= 32u;
    }
    auto center = [&](int st) -> double2 {
        return *reinterpret_cast<const double2*>(&ring[st][r][p]);
    };
    auto advance = [&]() {
        if (++s == V_STAGES) {
            s = 0;
            ph ^= 1;
        }
    };
    auto release = [&](int st) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs next TMA
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    };

    mbar_wait(&full[s], ph);
    double2 up = center(s);  // plane i0-1: only its centre is needed
    release(s);
    advance();
    mbar_wait(&full[s], ph);
    double2 mid = center(s);
    int sm = s;
    advance();
    for (int q = 2; q < nplanes; ++q) {
        mbar_wait(&full[s], ph);
        const double2 dn = center(s);
        const double2 ym = *reinterpret_cast<const double2*>(&ring[sm][r - 1][p]);
        const double2 yp = *reinterpret_cast<const double2*>(&ring[sm][r + 1][p]);
        const double zm = ring[sm][r][p - 1];
        const double zp = ring[sm][r][p + 2];
        release(sm);
        sm = s;
        advance();
        if (act) {
            const double ox = div6_t<GUARD>(sum6(up.x, dn.x, ym.x, yp.x, zm, mid.y));
            double oy = 0.0;
            if (both) {
                oy = div6_t<GUARD>(sum6(up.y, dn.y, ym.y, yp.y, mid.x, zp));
                *reinterpret_cast<double2*>(wr) = make_double2(ox, oy);
                if (RESID)
                    rmax = rmax_acc(rmax_acc(rmax, fabs(__dsub_rn(ox, mid.x))), fabs(__dsub_rn(oy, mid.y)));
            } else {
                wr[0] = ox;
                if (RESID) rmax = rmax_acc(rmax, fabs(__dsub_rn(ox, mid.x)));
            }
            if (PUSH && pm) {
                // the reference's pack -> mp_send -> unpack of all six faces
                // (jacobi.py:102-124, 237) as stores of the producing kernel
                const VolPush* vp = a.vpush + c;
                const int wp = parity ^ 1;
                const int64_t off = off0 + (int64_t)(q - 2) * a.sx;
                const bool xf = ((pm & 1u) && q == 2) || ((pm & 2u) && q == nplanes - 1);
                if (xf || (pm & 12u)) {
                    auto put2 = [&](double* t) {
                        if (both) *reinterpret_cast<double2*>(t) = make_double2(ox, oy);
                        else t[0] = ox;
                    };
                    if ((pm & 1u) && q == 2) put2(vp->ptr[0][wp] + off);
                    if ((pm & 2u) && q == nplanes - 1) put2(vp->ptr[1][wp] + off);
                    if (pm & 4u) put2(vp->ptr[2][wp] + off);
                    if (pm & 8u) put2(vp->ptr[3][wp] + off);
                }
                if (pm & 16u) vp->ptr[4][wp][off] = ox;
                if (pm & 32u) {
                    const bool z1y = k + 1 == a.ez;
                    vp->ptr[5][wp][off + (z1y ? 1 : 0)] = z1y ? oy : ox;
                }
            }
        }
        wr += a.sx;
        up = mid;
        mid = dn;
    }
    release(sm);  // the tile's last plane (the ring continues with the next tile)
}

template <bool RESID>
__global__ void __launch_bounds__(32 * (V_CW + 1), HRT_V_MINB)
volume_update_tma_kernel(VolArgs a) {
    extern __shared__ __align__(128) unsigned char v_dyn_smem[];
    auto ring = reinterpret_cast<double (*)[V_ROWS][V_ZROW]>(v_dyn_smem);
    __shared__ alignas(8) uint64_t full[V_STAGES], empty[V_STAGES];
    __shared__ double red[V_CW];

    const int64_t per_chunk = a.tiles_i * a.tiles_j * a.tiles_k;
    const int64_t t = blockIdx.x;
    const int64_t c = t / per_chunk;
    int64_t rem = t - c * per_chunk;
    const int64_t ti = rem / (a.tiles_j * a.tiles_k);
    rem -= ti * a.tiles_j * a.tiles_k;
    const int64_t tj = rem / a.tiles_k;
    const int64_t tk = rem - tj * a.tiles_k;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    const int64_t k0 = 1 + tk * V_ZW;
    const int64_t j0 = 1 + tj * V_CW;
    const int64_t i0 = 1 + ti * a.rows;
    const int64_t i1 = min(a.ex, i0 + a.rows - 1);

    if (tid == 0) {
        for (int s = 0; s < V_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], V_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    int s = 0;
    uint32_t ph = 0;
    if (warp == V_CW) {
        if (lane == 0) v_produce(a, ring, full, empty, s, ph, c, i0, i1, j0, k0, a.parity);
        return;
    }
    double rmax = 0.0;
    if (a.vpush)
        v_consume<true, RESID, true>(a, ring, full, empty, s, ph, c, i0, i1, j0, k0, a.parity,
                                     rmax);
    else
        v_consume<true, RESID, false>(a, ring, full, empty, s, ph, c, i0, i1, j0, k0, a.parity,
                                      rmax);

    if (RESID) {
        rmax = warp_max(rmax);
        if (lane == 0) red[warp] = rmax;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * V_CW));
        if (tid == 0) {
            double m2 = red[0];
#pragma unroll
            for (int q = 1; q < V_CW; ++q) m2 = fmax(m2, red[q]);
            resid_max(a.resid, m2);
        }
    }
}

// Persistent wavefront for volumes: the slab protocol (tickets, per-tile
// step counters, tile-descriptor queue, timeouts) with 6-neighbour tile
// dependencies — (i, j, k) block neighbours inside a chunk, the adjacent
// chunk's boundary tile across a face — and the fused 6-face push.
struct VolWaveArgs {
    VolArgs v;
    const int* nbr;               // [nchunks][6] neighbour chunk or -1
    unsigned int* done;           // [T]
    unsigned long long* ticket;
    unsigned int base;
    int nsteps;
    int parity0;
    int64_t ntiles;
    unsigned long long* resid;
    unsigned long long timeout_ns;
    int* err;
    const int* rnbr;              // [nchunks][6] (cross-process faces) or null
    const int* rpeer;
    unsigned int* const* peer_done;
};

template <bool RESID>
__global__ void __launch_bounds__(32 * (V_CW + 1), HRT_V_MINB)
volume_wave_kernel(VolWaveArgs wa) {
    extern __shared__ __align__(128) unsigned char v_dyn_smem[];
    auto ring = reinterpret_cast<double (*)[V_ROWS][V_ZROW]>(v_dyn_smem);
    __shared__ alignas(8) uint64_t full[V_STAGES], empty[V_STAGES], tq_full[WAVE_TQ],
        tq_empty[WAVE_TQ];
    __shared__ long long tq[WAVE_TQ];
    __shared__ double red[V_CW];
    const VolArgs& a = wa.v;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int64_t T = wa.ntiles;
    const int64_t tjk = a.tiles_j * a.tiles_k;
    const int64_t per_chunk = a.tiles_i * tjk;
    const long long total = (long long)T * wa.nsteps;

    if (tid == 0) {
        for (int k = 0; k < V_STAGES; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], V_CW);
        }
        for (int k = 0; k < WAVE_TQ; ++k) {
            mbar_init(&tq_full[k], 1);
            mbar_init(&tq_empty[k], V_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    auto decode = [&](int64_t tile, int64_t& c, int64_t& ti, int64_t& tj, int64_t& tk) {
        c = tile / per_chunk;
        int64_t rem = tile - c * per_chunk;
        ti = rem / tjk;
        rem -= ti * tjk;
        tj = rem / a.tiles_k;
        tk = rem - tj * a.tiles_k;
    };

    int s = 0;
    uint32_t ph = 0;
    if (warp == V_CW) {
        if (lane != 0) return;
        bool dead = false;
        int slot = 0;
        uint32_t tph = 0;
        for (;;) {
            const long long t = (long long)atomicAdd(wa.ticket, 1ull);
            mbar_wait(&tq_empty[slot], tph ^ 1);
            tq[slot] = t < total ? t : -1;
            mbar_arrive(&tq_full[slot]);
            if (++slot == WAVE_TQ) {
                slot = 0;
                tph ^= 1;
            }
            if (t >= total) break;
            const int k = (int)(t / T);
            const int64_t tile = t - (long long)k * T;
            int64_t c, ti, tj, tk;
            decode(tile, c, ti, tj, tk);
            if (!dead) {
                const int* nb = wa.nbr + 6 * c;
                const unsigned need = wa.base + (unsigned)k;
                auto tix = [&](int64_t cc, int64_t i, int64_t j, int64_t kk) {
                    return cc * per_chunk + i * tjk + j * a.tiles_k + kk;
                };
                const unsigned int* q[7] = {wa.done + tile, nullptr, nullptr, nullptr,
                                            nullptr, nullptr, nullptr};
                bool sys[7] = {false, false, false, false, false, false, false};
                // face f: the adjacent tile inside the chunk if any, else the
                // neighbour chunk's boundary tile (local or another rank's)
                auto face = [&](int f, bool inside, int64_t ii, int64_t jj, int64_t kk, int64_t bi,
                                int64_t bj, int64_t bk) {
                    const int d = f + 1;
                    if (inside) q[d] = wa.done + tix(c, ii, jj, kk);
                    else if (nb[f] >= 0) q[d] = wa.done + tix(nb[f], bi, bj, bk);
                    else if (wa.rpeer && wa.rpeer[6 * c + f] >= 0) {
                        q[d] = wa.peer_done[wa.rpeer[6 * c + f]] +
                               tix(wa.rnbr[6 * c + f], bi, bj, bk);
                        sys[d] = true;
                    }
                };
                face(0, ti > 0, ti - 1, tj, tk, a.tiles_i - 1, tj, tk);
                face(1, ti < a.tiles_i - 1, ti + 1, tj, tk, 0, tj, tk);
                face(2, tj > 0, ti, tj - 1, tk, ti, a.tiles_j - 1, tk);
                face(3, tj < a.tiles_j - 1, ti, tj + 1, tk, ti, 0, tk);
                face(4, tk > 0, ti, tj, tk - 1, ti, tj, a.tiles_k - 1);
                face(5, tk < a.tiles_k - 1, ti, tj, tk + 1, ti, tj, 0);
                dead = !wait_counters<7>(q, sys, need, wa.timeout_ns, wa.err);
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            const int64_t i0 = 1 + ti * a.rows;
            v_produce(a, ring, full, empty, s, ph, c, i0, min(a.ex, i0 + a.rows - 1),
                      1 + tj * V_CW, 1 + tk * V_ZW, (wa.parity0 + k) & 1);
        }
        return;
    }
    int slot = 0;
    uint32_t tph = 0;
    for (;;) {
        mbar_wait(&tq_full[slot], tph);
        const long long t = tq[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&tq_empty[slot]);
        if (++slot == WAVE_TQ) {
            slot = 0;
            tph ^= 1;
        }
        if (t < 0) break;
        const int k = (int)(t / T);
        const int64_t tile = t - (long long)k * T;
        int64_t c, ti, tj, tk;
        decode(tile, c, ti, tj, tk);
        const int64_t i0 = 1 + ti * a.rows;
        const int64_t i1 = min(a.ex, i0 + a.rows - 1);
        double rmax = 0.0;
        v_consume<true, RESID, true>(a, ring, full, empty, s, ph, c, i0, i1, 1 + tj * V_CW,
                                     1 + tk * V_ZW, (wa.parity0 + k) & 1, rmax);
        if (RESID && wa.resid) {  // one atomic per tile (folded at the barrier below)
            rmax = warp_max(rmax);
            if (lane == 0) red[warp] = rmax;
        }
        const int* rp = wa.rpeer ? wa.rpeer + 6 * c : nullptr;
        const bool xedge = rp && ((ti == 0 && rp[0] >= 0) || (ti == a.tiles_i - 1 && rp[1] >= 0) ||
                                  (tj == 0 && rp[2] >= 0) || (tj == a.tiles_j - 1 && rp[3] >= 0) ||
                                  (tk == 0 && rp[4] >= 0) || (tk == a.tiles_k - 1 && rp[5] >= 0));
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (xedge) __threadfence_system();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * V_CW));
        if (tid == 0) {
            if (RESID && wa.resid) {
                double m2 = red[0];
#pragma unroll
                for (int w = 1; w < V_CW; ++w) m2 = fmax(m2, red[w]);
                resid_max(wa.resid + k, m2);
            }
            const unsigned v = wa.base + (unsigned)k + 1u;
            if (xedge) {
                __threadfence_system();
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(wa.done + tile), "r"(v)
                             : "memory");
            } else {
                __threadfence();
                st_release_gpu_u32(wa.done + tile, v);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// volume update: general (X,Y,Z) domains; element (i,j,k) at
// base + origin + i*sx + j*sy + k.  Threads tile (j,k), march i.

constexpr int VOL_TX = 32, VOL_TY = 4;

__global__ void __launch_bounds__(VOL_TX * VOL_TY)
volume_update_kernel(VolArgs a) {
    const int64_t per_chunk = a.tiles_i * a.tiles_j * a.tiles_k;
    const int64_t t = blockIdx.x;
    const int64_t c = t / per_chunk;
    int64_t rem = t - c * per_chunk;
    const int64_t ti = rem / (a.tiles_j * a.tiles_k);
    rem -= ti * a.tiles_j * a.tiles_k;
    const int64_t tj = rem / a.tiles_k;
    const int64_t tk = rem - tj * a.tiles_k;

    const double* __restrict__ u = (a.chunks ? a.chunks[c].b[a.parity] : a.du) + a.origin;
    double* __restrict__ w = (a.chunks ? a.chunks[c].b[a.parity ^ 1] : a.dw) + a.origin;
    const int64_t k = a.flat ? 1 : 1 + tk * VOL_TX + threadIdx.x;
    const int64_t j = a.flat ? 1 + tj * (VOL_TX * VOL_TY) + threadIdx.y * VOL_TX + threadIdx.x
                             : 1 + tj * VOL_TY + threadIdx.y;
    const bool act = (k <= a.ez) && (j <= a.ey);
    const int64_t i0 = 1 + ti * a.rows;
    const int64_t i1 = min(a.ex, i0 + a.rows - 1);
    double rmax = 0.0;
    if (act) {
        const int64_t col = j * a.sy + k;
        double up = __ldg(u + (i0 - 1) * a.sx + col);
        double mid = __ldg(u + i0 * a.sx + col);
        for (int64_t i = i0; i <= i1; ++i) {
            const double* p = u + i * a.sx + col;
            const double dn = __ldg(p + a.sx);
            const double nv = div6_sel(sum6(up, dn, __ldg(p - a.sy), __ldg(p + a.sy),
                                            __ldg(p - 1), __ldg(p + 1)), a.ieee);
            w[i * a.sx + col] = nv;
            rmax = rmax_acc(rmax, fabs(__dsub_rn(nv, mid)));
            up = mid;
            mid = dn;
        }
    }
    if (a.resid) {
        __shared__ double red[VOL_TX * VOL_TY / 32];
        const int tid = threadIdx.y * VOL_TX + threadIdx.x;
        rmax = warp_max(rmax);
        if ((tid & 31) == 0) red[tid >> 5] = rmax;
        __syncthreads();
        if (tid == 0) {
            double m = red[0];
            for (int q = 1; q < VOL_TX * VOL_TY / 32; ++q) m = fmax(m, red[q]);
            resid_max(a.resid, m);
        }
    }
}

// ---------------------------------------------------------------------------
// halo plane copies: dst[o*ds0 + i*ds1] = src[o*ss0 + i*ss1] for every
// segment.  One launch per step moves every face of every chunk on the GPU:
// same-GPU faces read the neighbour's boundary plane in place, peer faces
// read it over NVLink, remote (NCCL) faces pack/unpack staging buffers.

constexpr int HALO_THREADS = 256;
constexpr int HALO_PER_THREAD = 4;

__global__ void __launch_bounds__(HALO_THREADS)
halo_copy_kernel(const hrt_halo_seg_t* __restrict__ segs, int parity, int64_t blocks_per_seg) {
    const int64_t s = blockIdx.x / blocks_per_seg;
    const int64_t b = blockIdx.x - s * blocks_per_seg;
    const hrt_halo_seg_t g = segs[s];
    const double* __restrict__ src = reinterpret_cast<const double*>(g.src[parity]);
    double* __restrict__ dst = reinterpret_cast<double*>(g.dst[parity]);
    const int64_t n = g.n0 * g.n1;
    const int64_t stride = blocks_per_seg * HALO_THREADS;
    for (int64_t e = b * HALO_THREADS + threadIdx.x; e < n; e += stride) {
        const int64_t o = e / g.n1, i = e - o * g.n1;
        dst[o * g.ds0 + i * g.ds1] = src[o * g.ss0 + i * g.ss1];
    }
}

// field scan at upload (volume plans): smallest positive value (as ~bits,
// max-reduced: 0 = none yet) and a flag for any value the unguarded
// division cannot take (negative, non-finite, > 2^997; -0.0 is fine)
__device__ __forceinline__ void range_acc(unsigned long long& key, bool& bad, double v) {
    const bool b = !(v >= 0.0) || v > 0x1p997;
    bad |= b;
    const unsigned long long k =
        (v > 0.0 && !b) ? ~(unsigned long long)__double_as_longlong(v) : 0ull;
    key = k > key ? k : key;
}
// whole warp
__device__ __forceinline__ void range_flush(unsigned long long* range, unsigned long long key,
                                            bool bad) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, key, o);
        key = x > key ? x : key;
    }
    const bool anybad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        if (anybad) atomicOr(range + 1, 1ull);
        if (key > *reinterpret_cast<volatile unsigned long long*>(range)) atomicMax(range, key);
    }
}

// contiguous (FX, FY, FZ) field <-> every chunk interior of a plan, one CTA
// per interior row: upload scatter / gather (jacobi.py:425-435) in one launch
__global__ void __launch_bounds__(256)
field_copy_kernel(const ChunkBufs* __restrict__ chunks, const int64_t* __restrict__ offs, int parity,
                  int ndim, int64_t ex, int64_t ey, int64_t ez, int64_t sx, int64_t sy,
                  int64_t origin, double* __restrict__ field, int64_t FY, int64_t FZ,
                  int to_chunks, unsigned long long* __restrict__ range) {
    const int64_t rows = ndim == 2 ? ex : ex * ey;
    const int64_t c = blockIdx.x / rows;
    const int64_t r = blockIdx.x - c * rows;
    const int64_t ox = offs[3 * c], oy = offs[3 * c + 1], oz = offs[3 * c + 2];
    double* base = chunks[c].b[parity] + origin;
    double* crow;
    double* frow;
    int64_t n;
    if (ndim == 2) {
        crow = base + (r + 1) * sx + 1;
        frow = field + (ox + r) * FY + oy;
        n = ey;
    } else {
        const int64_t i = r / ey, j = r - i * ey;
        crow = base + (i + 1) * sx + (j + 1) * sy + 1;
        frow = field + ((ox + i) * FY + (oy + j)) * FZ + oz;
        n = ez;
    }
    if (to_chunks && range) {
        unsigned long long key = 0;
        bool bad = false;
        for (int64_t k = threadIdx.x; k < n; k += 256) {
            const double v = frow[k];
            crow[k] = v;
            range_acc(key, bad, v);
        }
        range_flush(range, key, bad);
    } else if (to_chunks)
        for (int64_t k = threadIdx.x; k < n; k += 256) crow[k] = frow[k];
    else
        for (int64_t k = threadIdx.x; k < n; k += 256) frow[k] = crow[k];
}

// one plane copy passed by value (standalone pack/unpack tasks)
__global__ void __launch_bounds__(HALO_THREADS) plane_copy_kernel(hrt_halo_seg_t g) {
    const double* __restrict__ src = reinterpret_cast<const double*>(g.src[0]);
    double* __restrict__ dst = reinterpret_cast<double*>(g.dst[0]);
    const int64_t n = g.n0 * g.n1;
    for (int64_t e = blockIdx.x * (int64_t)HALO_THREADS + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * HALO_THREADS) {
        const int64_t o = e / g.n1, i = e - o * g.n1;
        dst[o * g.ds0 + i * g.ds1] = src[o * g.ss0 + i * g.ss1];
    }
}

// ghost shell carry of _update_body (jacobi.py:80-86): nxt's six ghost
// planes = u's, for a volume-layout chunk (z ghosts stored)
__global__ void ghost_shell_copy_kernel(const double* __restrict__ u, double* __restrict__ w,
                                        int64_t ex, int64_t ey, int64_t ez, int64_t sx,
                                        int64_t sy) {
    const int64_t gx = ex + 2, gy = ey + 2, gz = ez + 2;
    const int64_t n = gx * gy * gz;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / (gy * gz);
        const int64_t r = e - i * gy * gz;
        const int64_t j = r / gz;
        const int64_t k = r - j * gz;
        if (i == 0 || i == gx - 1 || j == 0 || j == gy - 1 || k == 0 || k == gz - 1) {
            const int64_t off = i * sx + j * sy + k;
            w[off] = u[off];
        }
    }
}

// ---------------------------------------------------------------------------
// ghost initialisation: set the ghost shell of a chunk buffer to `value`
// for faces in `mask` (bit f = face f of jacobi.py:41 FACES) and 0 elsewhere.

__global__ void ghost_fill_kernel(double* __restrict__ base, int64_t origin, int64_t ex,
                                  int64_t ey, int64_t ez, int64_t sx, int64_t sy, int ndim,
                                  int mask, double value) {
    // iterate over the full ghosted box; write only ghost cells
    const int64_t gx = ex + 2, gy = ey + 2, gz = (ndim == 3) ? ez + 2 : 1;
    const int64_t n = gx * gy * gz;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / (gy * gz);
        const int64_t r = e - i * gy * gz;
        const int64_t jj = r / gz;
        const int64_t kk = r - jj * gz;
        int face = -1;
        if (i == 0) face = 0;
        else if (i == gx - 1) face = 1;
        else if (jj == 0) face = 2;
        else if (jj == gy - 1) face = 3;
        else if (ndim == 3 && kk == 0) face = 4;
        else if (ndim == 3 && kk == gz - 1) face = 5;
        if (face < 0) continue;
        // a ghost cell on several faces (edges/corners) is never read by the
        // 7-point stencil; give it the value of any domain face it touches
        bool dom = (mask >> face) & 1;
        if (!dom) {
            dom = ((i == 0) && (mask & 1)) || ((i == gx - 1) && (mask & 2)) ||
                  ((jj == 0) && (mask & 4)) || ((jj == gy - 1) && (mask & 8)) ||
                  (ndim == 3 && kk == 0 && (mask & 16)) ||
                  (ndim == 3 && kk == gz - 1 && (mask & 32));
        }
        base[origin + i * sx + jj * sy + kk] = dom ? value : 0.0;
    }
}

// ---------------------------------------------------------------------------
// exact float(np.sum(a)): numpy's pairwise summation (PW_BLOCKSIZE 128, eight
// partial sums), evaluated as one CTA per subtree of <= SEG elements; the top
// of the recursion tree is combined on the host in the same order.

constexpr int PW_SEG = 16384;
constexpr int PW_THREADS = 256;
constexpr int PW_MAX_LEAVES = 512;

__device__ double pw_leaf(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = a[q];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], a[i + q]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// enumerate leaves (n <= 128) of the subtree rooted at (off, n) in order
__device__ void pw_leaves(int64_t off, int64_t n, int64_t* lo, int64_t* ln, int* cnt) {
    // explicit stack: depth <= log2(PW_SEG/64)+1
    int64_t so[32], sn[32];
    int sp = 0;
    so[sp] = off;
    sn[sp] = n;
    ++sp;
    while (sp) {
        --sp;
        int64_t o = so[sp], m = sn[sp];
        if (m <= 128) {
            lo[*cnt] = o;
            ln[*cnt] = m;
            ++*cnt;
        } else {
            int64_t m2 = m / 2;
            m2 -= m2 % 8;
            // push right first so the left subtree is visited first
            so[sp] = o + m2; sn[sp] = m - m2; ++sp;
            so[sp] = o; sn[sp] = m2; ++sp;
        }
    }
}

__device__ double pw_combine(int64_t n, const double* leaf, int* next) {
    if (n <= 128) return leaf[(*next)++];
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    double l = pw_combine(n2, leaf, next);
    double r = pw_combine(n - n2, leaf, next);
    return __dadd_rn(l, r);
}

__global__ void __launch_bounds__(PW_THREADS)
pairwise_seg_kernel(const double* __restrict__ a, const int64_t* __restrict__ seg_off,
                    const int64_t* __restrict__ seg_len, double* __restrict__ out) {
    __shared__ int64_t lo[PW_MAX_LEAVES], ln[PW_MAX_LEAVES];
    __shared__ double leaf[PW_MAX_LEAVES];
    __shared__ int cnt;
    const int64_t off = seg_off[blockIdx.x], n = seg_len[blockIdx.x];
    if (threadIdx.x == 0) {
        cnt = 0;
        pw_leaves(off, n, lo, ln, &cnt);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < cnt; q += PW_THREADS) leaf[q] = pw_leaf(a + lo[q], ln[q]);
    __syncthreads();
    if (threadIdx.x == 0) {
        int next = 0;
        out[blockIdx.x] = pw_combine(n, leaf, &next);
    }
}

// ---------------------------------------------------------------------------
// division self-check: Markstein div6 vs IEEE on a counter-hashed sweep

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

__global__ void div6_sweep_kernel(uint64_t seed, int64_t n, int mode,
                                  unsigned long long* mismatches, double* first_bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = mix64(seed + (uint64_t)e * 0x9e3779b97f4a7c15ULL);
        double x;
        if (mode == 0) {  // uniform [0, 6): the Jacobi range of a six-term sum
            x = (double)(h >> 11) * 0x1p-53 * 6.0;
        } else if (mode == 1) {  // doubles within 2^-40 of 1.0 and of 6.0, 3.0
            const double centre = (h & 3) == 0 ? 1.0 : ((h & 3) == 1 ? 6.0 : ((h & 3) == 2 ? 3.0 : 2.0));
            x = centre + ((double)((int64_t)(h >> 24) - (int64_t)(1ULL << 39)) * 0x1p-80);
        } else {  // random finite bit patterns, positive
            uint64_t bits = h & 0x7fffffffffffffffULL;
            x = __longlong_as_double((long long)bits);
            if (!(fabs(x) <= 0x1p1000)) x = 1.0;
        }
        const double q = div6(x);
        const double ref = __ddiv_rn(x, 6.0);
        if (__double_as_longlong(q) != __double_as_longlong(ref)) {
            unsigned long long k = atomicAdd(mismatches, 1ULL);
            if (k == 0) *first_bad = x;
        }
    }
}

// ---------------------------------------------------------------------------
// TWO Jacobi steps per pass for volumes split along x (volume_wave2_kernel):
// the 3D form of slab_wave2_kernel.  A tile is (all planes of a chunk) x
// (VW_R y-rows) x (VW_TZ z-columns); pass k reads u(t) once — planes -1 ..
// ex+2 (the first and last two from the x-neighbour chunks, in place), rows
// j0-2 .. j0+VW_R+1, columns k0-2 .. k0+VW_TZ+1 — and writes only u(t+2).
// 8 algorithmic bytes per lattice update instead of 16.
//
// Producer: one 3D TMA tensor copy per plane (box 124 x 8 x 1 of the chunk
// buffer seen as a (ex+2, ey+2, sy) tensor); coordinates outside the buffer
// (plane -1 / ex+2 at a domain face, row -1 / ey+2) are zero-filled by the
// TMA unit and only ever feed values the consumer masks.
// Consumer thread (warp w, lane L) owns column k = k0-1+30w+L and the
// tile's VW_R rows; lanes 0 and 31 are rim columns (their u(t+2) is never
// stored), so a warp outputs 30 columns and computes u(t+1) on 32.  u(t) of
// the planes x-1, x, x+1 at the own column lives in registers (8 rows); its
// z neighbours come from the ring stage of plane x; u(t+1) of three planes
// lives in registers (6 rows) and its z neighbours come from the adjacent
// lanes by shuffles.  Every value is computed with the reference's
// operations in the reference's order (xm, xp, ym, yp, zm, zp), so the field
// and both per-step residuals stay bitwise equal.
// Dependencies: a tile of pass k needs its 3 x 3 x 3 neighbourhood — the
// chunk and its x neighbours, y and z blocks +-1 — done with pass k-1 (RAW
// on the rims it reads; WAR on the buffer it overwrites, which those tiles
// read as rim).  Only chunks whose y and z faces are all domain faces.
// Division: Markstein's sequence without a range check when the launch is
// proven safe (vw2_fast below); otherwise the same sequence plus an integer
// range test per sum, and a rare per-group recomputation with IEEE division
// (no branch per cell: branches split the dependency chains the scheduler
// interleaves).

#ifndef HRT_VW_MINB
#define HRT_VW_MINB 3  // resident CTAs per SM the register budget targets
#endif
#ifndef HRT_VW_CW
#define HRT_VW_CW 4
#endif
constexpr int VW_CW = HRT_VW_CW;      // consumer warps, side by side in z
#ifndef HRT_VW_R
#define HRT_VW_R 4
#endif
constexpr int VW_R = HRT_VW_R;        // y rows per tile (per thread)
constexpr int VW_ZO = 30;             // output columns per warp (lanes 1..30)
constexpr int VW_TZ = VW_CW * VW_ZO;  // output columns per tile
constexpr int VW_RS = VW_TZ + 4;      // ring row: columns k0-2 .. k0+VW_TZ+1
constexpr int VW_RR = VW_R + 4;       // ring rows per plane: j0-2 .. j0+VW_R+1
#ifndef HRT_VW_STAGES
#define HRT_VW_STAGES 5
#endif
constexpr int VW_STAGES = HRT_VW_STAGES;  // 5 x 8 x 124 doubles = 39.7 KB
constexpr uint32_t VW_STAGE_BYTES = (uint32_t)(VW_RR * VW_RS * 8);
constexpr size_t VW_SMEM = (size_t)VW_STAGES * VW_STAGE_BYTES;  // the ring (dynamic)
static_assert(VW_STAGE_BYTES % 128 == 0, "TMA tensor destinations must stay 128-byte aligned");

// x neighbours of a chunk (faces -x, +x): the tensor maps their planes are
// read through (null: a domain face, whose ghost plane is read from the own
// buffer), the step counter of their tile 0 (this plan's, or mapped from
// the neighbour process over CUDA IPC) and which of them live in another
// process (system-scope counters)
struct VW2Nbr {
    const CUtensorMap* map[2][2];   // [face][parity]
    const unsigned int* cnt[2];     // [face]
    unsigned sys;                   // bit f: face f's neighbour is in another process
    unsigned pad_;
};

struct VolW2Args {
    const CUtensorMap* maps;   // [nchunks][2] tensor map of buffer 0 / 1
    const ChunkBufs* chunks;
    const VW2Nbr* nbr;         // [nchunks]
    // chains: maximal runs of this plan's chunks linked along +x; a tile is
    // (chain, y block, z block) and streams every plane of its chain
    const int2* chains;        // [nchains] (offset into clist, length)
    const int* clist;          // chunk indices in +x order, chain after chain
    int64_t cdelta;            // output pointer step at a chunk boundary of a chain:
                               // (next chunk's buffer - this one's) - ex * sx
    unsigned int* done;        // [T] steps completed per tile (absolute: base at launch)
    unsigned int base;
    unsigned long long* ticket;
    const unsigned long long* range;  // field scan: [0] ~bits(min positive), [1] bad flag
    double need;               // unguarded division is exact if min positive >= need
    int nfused;                // passes (2 steps each)
    int parity0;
    int64_t ntiles, ex, ey, ez, sx, sy, origin, tiles_j, tiles_k;
    unsigned long long* resid; // nullable: 2 * nfused slots
    unsigned long long timeout_ns;
    int* err;
};

__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// |s| outside the range where Markstein's quotient is IEEE's: nonzero below
// 2^-1019, or 2^1000 and above (incl. inf / NaN) — integer ops on the bits
__device__ __forceinline__ bool div6_out_of_range(double s) {
    const uint32_t h = (uint32_t)__double2hiint(s) & 0x7fffffffu;
    const uint32_t l = (uint32_t)__double2loint(s);
    return (h - 0x00400000u) >= (0x7E700000u - 0x00400000u) && (h | l) != 0u;
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

// planes -1 .. m*ex+2 of tile (chain, j0, k0) into the ring, one tensor
// copy each: the chain's chunks in turn, the first and last two from the
// x neighbours of its end chunks (in place) or their own ghost planes
__device__ __forceinline__ void vw2_produce(const VolW2Args& a, uint32_t ring, uint64_t* full,
                                            uint64_t* empty, int& s, uint32_t& ph, int2 ch,
                                            int64_t j0, int64_t k0, int parity) {
    const int* cl = a.clist + ch.x;
    const int cf = cl[0], cz = cl[ch.y - 1];
    const CUtensorMap* mm = a.nbr[cf].map[0][parity];
    const CUtensorMap* pm = a.nbr[cz].map[1][parity];
    const int c0 = (int)(a.origin + k0 - 2), c1 = (int)(j0 - 2);
    const int ex = (int)a.ex;
    const int nx = ex * ch.y;  // planes of the chain
    const int nplanes = nx + 4;
    int j = 0, ii0 = 0;  // chunk of the chain and its plane, for planes 1 .. nx
    for (int q = 0; q < nplanes; ++q) {
        const int i = q - 1;  // plane of the chain
        const CUtensorMap* m;
        int ii;
        if (i < 1) {
            m = mm ? mm : a.maps + 2 * cf + parity;
            ii = mm ? i + ex : i;
        } else if (i > nx) {
            m = pm ? pm : a.maps + 2 * cz + parity;
            ii = pm ? i - nx : i - (nx - ex);
        } else {
            if (++ii0 > ex) {
                ii0 = 1;
                ++j;
            }
            m = a.maps + 2 * cl[j] + parity;
            ii = ii0;
        }
        mbar_wait_sleep(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], VW_STAGE_BYTES);
        tma_load_3d(ring + (uint32_t)s * VW_STAGE_BYTES, m, c0, c1, ii, smem_u32(&full[s]));
        if (++s == VW_STAGES) {
            s = 0;
            ph ^= 1;
        }
    }
}

// Per-thread state of the volume two-step consumer (one tile).
// the ring's barriers (full, then empty) at file scope: their shared
// addresses are link-time constants, so the consumer keeps no register
// for them
__shared__ alignas(8) uint64_t vw2_fe[2 * VW_STAGES];
__device__ __forceinline__ uint32_t vw2_bar(int k) { return smem_u32(&vw2_fe[k]); }

struct VW2Ctx {
    uint32_t ring;        // shared address of this thread's column in stage 0, row 0
    int s;
    uint32_t ph;
    bool ready;
    bool tmask;           // some row or column of this warp's tile lies outside the domain
    bool xlo, xhi;        // the x faces are domain faces
    unsigned vrow;        // bit r: ring row r (0..7) inside the domain rows
    bool colok;           // this lane's column is inside the domain
    bool own;             // lane 1..30 with an inside column: stores + residuals
    int ex;               // planes of the chain
    double* wr;           // plane 1, row j0, this column, buffer parity^1
    int rem;              // output planes left in the current chunk
    double r1, r2;
};

// next output plane: within a chunk one x stride, across a chain's chunk
// boundary the step to the next chunk's buffer (strides and extents come
// from the kernel parameters, not registers: the consumer runs at the
// register limit)
template <bool CHAIN>
__device__ __forceinline__ void vw2_next_plane(VW2Ctx& x, const VolW2Args& a) {
    x.wr += a.sx;
    if (CHAIN && --x.rem == 0) {
        x.wr += a.cdelta;
        x.rem = (int)a.ex;
    }
}

template <int NP>
__device__ __forceinline__ void vw2_take(VW2Ctx& x, double (&v)[NP], int& st) {
    const uint32_t fb = vw2_bar(x.s);
    if (!x.ready && !mbar_try_u32(fb, x.ph)) mbar_wait_u32_slow(fb, x.ph);
    st = x.s;
    const uint32_t base = x.ring + (uint32_t)x.s * VW_STAGE_BYTES;
#pragma unroll
    for (int r = 0; r < NP; ++r) v[r] = lds_f64(base + (uint32_t)(r * VW_RS * 8));
    if (++x.s == VW_STAGES) {
        x.s = 0;
        x.ph ^= 1;
    }
    x.ready = false;
}

// Poll the next stage once the step's shared loads are issued: try_wait
// acquires, so shared loads after it wait for its ~90-cycle round trip.
__device__ __forceinline__ void vw2_poll(VW2Ctx& x) {
    x.ready = mbar_try_u32(vw2_bar(x.s), x.ph);
}

__device__ __forceinline__ void vw2_release(VW2Ctx& x, int st) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // WAR vs the next TMA
    __syncwarp();
    // lane 0 arrives (%laneid read in place: no register for it across the loop)
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .u32 l;\n\t"
        "mov.u32 l, %%laneid;\n\t"
        "setp.eq.u32 p, l, 0;\n\t"
        "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(vw2_bar(VW_STAGES + st))
        : "memory");
}

// one pipeline step q (ring plane q = u(t) plane i = q-1 arrives as dn):
// u(t+1) at plane q-2 (ring rows 1..6) -> u1n; u(t+2) at plane q-3 from
// u(t+1) planes q-4 (u1a), q-3 (u1b), q-2 (u1n), stored.
template <bool GUARD, bool RESID, bool CHAIN>
__device__ __forceinline__ void vw2_step(VW2Ctx& x, const VolW2Args& a, const double (&up)[VW_RR],
                                         const double (&mid)[VW_RR], double (&dn)[VW_RR],
                                         int& smid, const double (&u1a)[VW_R + 2],
                                         const double (&u1b)[VW_R + 2], double (&u1n)[VW_R + 2],
                                         int q) {
    int sdn;
    vw2_take<VW_RR>(x, dn, sdn);
    const int64_t i = q - 2;
    // ---- u(t+1) at plane i, ring rows 1 .. VW_R+2 ----
    {
        const uint32_t mb = x.ring + (uint32_t)smid * VW_STAGE_BYTES;
        bool bad = false;
#pragma unroll
        for (int m = 0; m < VW_R + 2; ++m) {
            const uint32_t ra = mb + (uint32_t)((m + 1) * VW_RS * 8);
            const double s = sum6(up[m + 1], dn[m + 1], mid[m], mid[m + 2], lds_f64(ra - 8u),
                                  lds_f64(ra + 8u));
            u1n[m] = div6_fast(s);
            if (GUARD) bad |= div6_out_of_range(s);
        }
        if (GUARD && bad) {  // rare: redo the group with IEEE division (unrolled:
                             // a dynamic index would put the arrays in local memory)
#pragma unroll
            for (int m = 0; m < VW_R + 2; ++m) {
                const uint32_t ra = mb + (uint32_t)((m + 1) * VW_RS * 8);
                u1n[m] = __ddiv_rn(sum6(up[m + 1], dn[m + 1], mid[m], mid[m + 2],
                                        lds_f64(ra - 8u), lds_f64(ra + 8u)),
                                   6.0);
            }
        }
        vw2_release(x, smid);  // the stage of plane q-2 has served as mid: done
        smid = sdn;
        const bool xghost = (i < 1 && x.xlo) || (i > x.ex && x.xhi);
        if (x.tmask || xghost) {  // edge tiles only (warp-uniform)
            double d = 0.0;
#pragma unroll
            for (int m = 0; m < VW_R + 2; ++m) {
                const bool in = !xghost && x.colok && ((x.vrow >> (m + 1)) & 1u);
                if (!in) u1n[m] = HRT_BOUNDARY;
                if (RESID && in && m >= 1 && m <= VW_R)
                    d = dmax(d, abs_bits(__dsub_rn(u1n[m], mid[m + 1])));
            }
            if (RESID && x.own && i >= 1 && i <= x.ex) x.r1 = dmax(x.r1, d);
        } else if (RESID) {
            // every value here is an interior cell's u(t+1): the rim rows /
            // lanes belong to neighbour tiles, and max is idempotent
            double d = abs_bits(__dsub_rn(u1n[0], mid[1]));
#pragma unroll
            for (int m = 1; m < VW_R + 2; ++m) d = dmax(d, abs_bits(__dsub_rn(u1n[m], mid[m + 1])));
            x.r1 = dmax(x.r1, d);
        }
    }
    // ---- u(t+2) at plane q-3 (1 .. ex) -> HBM ----
    if (q >= 4) {
        double o[VW_R];
        bool bad = false;
#pragma unroll
        for (int m = 1; m <= VW_R; ++m) {
            const double s =
                sum6(u1a[m], u1n[m], u1b[m - 1], u1b[m + 1], shfl_up1(u1b[m]), shfl_dn1(u1b[m]));
            o[m - 1] = div6_fast(s);
            if (GUARD) bad |= div6_out_of_range(s);
        }
        if (GUARD && __any_sync(0xffffffffu, bad)) {  // shuffles: the whole warp redoes it
#pragma unroll
            for (int m = 1; m <= VW_R; ++m)
                o[m - 1] = __ddiv_rn(sum6(u1a[m], u1n[m], u1b[m - 1], u1b[m + 1],
                                          shfl_up1(u1b[m]), shfl_dn1(u1b[m])),
                                     6.0);
        }
        if (x.tmask) {
            if (x.own) {
                double d = 0.0;
#pragma unroll
                for (int m = 0; m < VW_R; ++m)
                    if ((x.vrow >> (m + 2)) & 1u) {
                        x.wr[m * a.sy] = o[m];
                        if (RESID) d = dmax(d, abs_bits(__dsub_rn(o[m], u1b[m + 1])));
                    }
                if (RESID) x.r2 = dmax(x.r2, d);
            }
        } else {
            if (x.own) {
#pragma unroll
                for (int m = 0; m < VW_R; ++m) x.wr[m * a.sy] = o[m];
            }
            if (RESID) {
                double d = abs_bits(__dsub_rn(o[0], u1b[1]));
#pragma unroll
                for (int m = 1; m < VW_R; ++m) d = dmax(d, abs_bits(__dsub_rn(o[m], u1b[m + 1])));
                if (x.own) x.r2 = dmax(x.r2, d);
            }
        }
        vw2_next_plane<CHAIN>(x, a);
    }
    vw2_poll(x);
}

// The same step for planes 2 .. ex of a tile with nothing outside the domain
// (no masks; q >= 4): one basic block apart from the barrier waits, so the
// scheduler interleaves the ten independent sums.  The residual of u(t+1)
// is taken on every lane — rim lanes hold neighbour tiles' interior values,
// and max is idempotent — that of u(t+2) on the owning lanes only.
template <bool GUARD, bool RESID, bool CHAIN>
__device__ __forceinline__ void vw2_step_fast(VW2Ctx& x, const VolW2Args& a,
                                              const double (&up)[VW_RR],
                                              const double (&mid)[VW_RR], double (&dn)[VW_RR],
                                              int& smid, const double (&u1a)[VW_R + 2],
                                              const double (&u1b)[VW_R + 2],
                                              double (&u1n)[VW_R + 2]) {
    int sdn;
    vw2_take<VW_RR>(x, dn, sdn);
    const uint32_t mb = x.ring + (uint32_t)smid * VW_STAGE_BYTES;
    bool bad = false;
#pragma unroll
    for (int m = 0; m < VW_R + 2; ++m) {
        const uint32_t ra = mb + (uint32_t)((m + 1) * VW_RS * 8);
        const double s = sum6(up[m + 1], dn[m + 1], mid[m], mid[m + 2], lds_f64(ra - 8u),
                              lds_f64(ra + 8u));
        u1n[m] = div6_fast(s);
        if (GUARD) bad |= div6_out_of_range(s);
    }
    if (GUARD && bad) {
#pragma unroll
        for (int m = 0; m < VW_R + 2; ++m) {
            const uint32_t ra = mb + (uint32_t)((m + 1) * VW_RS * 8);
            u1n[m] = __ddiv_rn(sum6(up[m + 1], dn[m + 1], mid[m], mid[m + 2], lds_f64(ra - 8u),
                                    lds_f64(ra + 8u)),
                               6.0);
        }
    }
    vw2_release(x, smid);
    smid = sdn;
    double o[VW_R];
    bool bad2 = false;
#pragma unroll
    for (int m = 1; m <= VW_R; ++m) {
        const double s =
            sum6(u1a[m], u1n[m], u1b[m - 1], u1b[m + 1], shfl_up1(u1b[m]), shfl_dn1(u1b[m]));
        o[m - 1] = div6_fast(s);
        if (GUARD) bad2 |= div6_out_of_range(s);
    }
    if (GUARD && __any_sync(0xffffffffu, bad2)) {
#pragma unroll
        for (int m = 1; m <= VW_R; ++m)
            o[m - 1] = __ddiv_rn(sum6(u1a[m], u1n[m], u1b[m - 1], u1b[m + 1], shfl_up1(u1b[m]),
                                      shfl_dn1(u1b[m])),
                                 6.0);
    }
    if (x.own) {
#pragma unroll
        for (int m = 0; m < VW_R; ++m) x.wr[m * a.sy] = o[m];
    }
    if (RESID) {
        double e1[VW_R], e2[VW_R];
#pragma unroll
        for (int m = 0; m < VW_R; ++m) {
            e1[m] = abs_bits(__dsub_rn(u1n[m + 1], mid[m + 2]));
            e2[m] = abs_bits(__dsub_rn(o[m], u1b[m + 1]));
        }
#pragma unroll
        for (int w = 1; w < VW_R; w *= 2)  // pairwise tree
#pragma unroll
            for (int m = 0; m + w < VW_R; m += 2 * w) {
                e1[m] = dmax(e1[m], e1[m + w]);
                e2[m] = dmax(e2[m], e2[m + w]);
            }
        x.r1 = dmax(x.r1, e1[0]);
        if (x.own) x.r2 = dmax(x.r2, e2[0]);
    }
    vw2_next_plane<CHAIN>(x, a);
    vw2_poll(x);
}

template <bool GUARD, bool RESID, bool CHAIN>
__device__ __forceinline__ void vw2_consume(const VolW2Args& a, uint32_t ring_u32,
                                            uint32_t full_u32, uint32_t empty_u32, int& s,
                                            uint32_t& ph, int2 ch, int64_t j0, int64_t k0,
                                            int parity, double& r1, double& r2) {
    const int cf = a.clist[ch.x], cz = a.clist[ch.x + ch.y - 1];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    VW2Ctx x;
    (void)full_u32;  // (vw2_fe: full barriers, then the empty ones)
    (void)empty_u32;
    x.s = s;
    x.ph = ph;
    x.ready = false;
    const int lane = tid & 31;
    const int pc = 1 + VW_ZO * warp + lane;  // ring column of k
    const int64_t k = k0 - 2 + pc;
    x.ring = ring_u32 + 8u * (uint32_t)pc;
    x.ex = (int)a.ex * ch.y;
    x.rem = (int)a.ex;
    x.xlo = a.nbr[cf].map[0][0] == nullptr;
    x.xhi = a.nbr[cz].map[1][0] == nullptr;
    unsigned vrow = 0;
#pragma unroll
    for (int r = 0; r < VW_RR; ++r) {
        const int64_t j = j0 - 2 + r;
        if (j >= 1 && j <= a.ey) vrow |= 1u << r;
    }
    x.vrow = vrow;
    x.colok = k >= 1 && k <= a.ez;
    x.own = lane >= 1 && lane <= VW_ZO && x.colok;
    x.tmask = __any_sync(0xffffffffu, !x.colok) || vrow != (1u << VW_RR) - 1u;
    x.wr = a.chunks[cf].b[parity ^ 1] + a.origin + a.sx + j0 * a.sy + k;
    x.r1 = r1;
    x.r2 = r2;
    const int nplanes = (int)(x.ex + 4);

    double t0[VW_RR], t1[VW_RR], t2[VW_RR];           // u(t) planes, rotating
    double y0[VW_R + 2], y1[VW_R + 2], y2[VW_R + 2];  // u(t+1) planes, rotating
    int st0, smid;
    vw2_take<VW_RR>(x, t0, st0);  // plane -1: only ever "up"
    vw2_release(x, st0);
    vw2_take<VW_RR>(x, t1, smid);  // plane 0
    // register roles rotate with period 3: step q uses set (q-2) % 3
    vw2_step<GUARD, RESID, CHAIN>(x, a, t0, t1, t2, smid, y1, y2, y0, 2);  // u(t+1) at plane 0
    vw2_step<GUARD, RESID, CHAIN>(x, a, t1, t2, t0, smid, y2, y0, y1, 3);
    int q = 4;
    if (!x.tmask)  // planes 2 .. ex: nothing outside the domain
        for (; q + 2 <= (int)x.ex + 2; q += 3) {
            vw2_step_fast<GUARD, RESID, CHAIN>(x, a, t2, t0, t1, smid, y0, y1, y2);
            vw2_step_fast<GUARD, RESID, CHAIN>(x, a, t0, t1, t2, smid, y1, y2, y0);
            vw2_step_fast<GUARD, RESID, CHAIN>(x, a, t1, t2, t0, smid, y2, y0, y1);
        }
    for (; q + 2 < nplanes; q += 3) {
        vw2_step<GUARD, RESID, CHAIN>(x, a, t2, t0, t1, smid, y0, y1, y2, q);
        vw2_step<GUARD, RESID, CHAIN>(x, a, t0, t1, t2, smid, y1, y2, y0, q + 1);
        vw2_step<GUARD, RESID, CHAIN>(x, a, t1, t2, t0, smid, y2, y0, y1, q + 2);
    }
    if (q < nplanes) vw2_step<GUARD, RESID, CHAIN>(x, a, t2, t0, t1, smid, y0, y1, y2, q);
    if (q + 1 < nplanes) vw2_step<GUARD, RESID, CHAIN>(x, a, t0, t1, t2, smid, y1, y2, y0, q + 1);
    vw2_release(x, smid);  // the last plane only served as dn
    s = x.s;
    ph = x.ph;
    r1 = x.r1;
    r2 = x.r2;
}

// Unguarded division is exact for this launch: the uploaded field was
// finite, >= 0 and <= 2^997 (so sums stay <= 2^1000), and its smallest
// positive value m0 (or the 1.0 boundary) shrinks by at most a factor
// 6(1+2^-52) per step, so every nonzero sum of the run is >= 2^-1019 as
// long as m0 >= need = 2^-1019 * 6.000001^(steps since the scan + this run)
// (computed by the host).  Non-negative sums cannot cancel to something
// smaller than their largest term.
__device__ __forceinline__ bool vw2_fast(const VolW2Args& a) {
    if (!a.range || a.range[1] != 0ull) return false;
    const unsigned long long key = a.range[0];
    const double m0 = key == 0ull ? 1.0 : fmin(1.0, __longlong_as_double((long long)~key));
    return m0 >= a.need;
}

// Launched as a pair on one stream: the FAST instance runs when vw2_fast
// holds, the guarded one otherwise; the other returns at once (the decision
// is on the device: the scan it reads was written by an upload kernel).
// CHAIN: the output pointer steps between the buffers of a chain's chunks
// (the product launches CHAIN = true only: an instance without that
// bookkeeping measured no faster — 492 vs 510 GLUPS on paper3d — its
// register allocation spilled more)
template <bool FAST, bool RESID, bool CHAIN>
__global__ void __launch_bounds__(32 * (VW_CW + 1), HRT_VW_MINB)
volume_wave2_kernel(VolW2Args wa) {
    if (vw2_fast(wa) != FAST) return;
    extern __shared__ __align__(128) unsigned char vw2_dyn[];  // the ring: VW_SMEM bytes
    __shared__ alignas(8) uint64_t tq_full[WAVE_TQ], tq_empty[WAVE_TQ];
    uint64_t* full = vw2_fe;            // ring barriers: full, then empty
    uint64_t* empty = vw2_fe + VW_STAGES;
    __shared__ long long tq[WAVE_TQ];
    __shared__ double red[2][VW_CW];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int64_t T = wa.ntiles;
    const int64_t tj = wa.tiles_j, tk = wa.tiles_k;
    const int64_t per_chunk = tj * tk;
    const long long total = (long long)T * wa.nfused;

    if (tid == 0) {
        for (int k = 0; k < VW_STAGES; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], VW_CW);
        }
        for (int k = 0; k < WAVE_TQ; ++k) {
            mbar_init(&tq_full[k], 1);
            mbar_init(&tq_empty[k], VW_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    int s = 0;
    uint32_t ph = 0;
    const uint32_t ring_u32 = smem_u32(vw2_dyn);
    if (warp >= VW_CW) {
        if (lane != 0) return;
        bool dead = false;
        int slot = 0;
        uint32_t tph = 0;
        for (;;) {
            const long long t = (long long)atomicAdd(wa.ticket, 1ull);
            mbar_wait(&tq_empty[slot], tph ^ 1);
            tq[slot] = t < total ? t : -1;
            mbar_arrive(&tq_full[slot]);
            if (++slot == WAVE_TQ) {
                slot = 0;
                tph ^= 1;
            }
            if (t >= total) break;
            const int k = (int)(t / T);
            const int64_t tile = t - (long long)k * T;
            const int64_t h = tile / per_chunk;  // chain
            const int64_t rem = tile - h * per_chunk;
            // z fastest in ticket order (y fastest cuts the DRAM re-reads of
            // the rows y-adjacent tiles share, 39 vs 47 GB per 4 paper3d
            // passes, at the same speed on one GPU, but ran 3.5 % slower on
            // 4: 1450 vs 1502 GLUPS)
            const int64_t yb = rem / tk;
            const int64_t zb = rem - yb * tk;
            const int2 ch = wa.chains[h];
            if (!dead) {
                // the 3 x 3 x 3 tile neighbourhood must be done with step 2k:
                // y / z blocks +-1 of this chain (every chunk of a chain
                // publishes together: its first chunk's counters stand for
                // all) and of the x neighbours of its end chunks
                const unsigned need = wa.base + 2u * (unsigned)k;
                const unsigned int* q[27];
                bool sys[27];
                const int cf = wa.clist[ch.x], cz = wa.clist[ch.x + ch.y - 1];
                const unsigned int* cx[3] = {wa.nbr[cf].cnt[0], wa.done + cf * per_chunk,
                                             wa.nbr[cz].cnt[1]};
                const bool sx[3] = {(wa.nbr[cf].sys & 1u) != 0, false,
                                    (wa.nbr[cz].sys & 2u) != 0};
#pragma unroll
                for (int d = 0; d < 27; ++d) {
                    const unsigned int* cc = cx[d / 9];
                    const int64_t y2 = yb + (d / 3) % 3 - 1, z2 = zb + d % 3 - 1;
                    const bool in = cc && y2 >= 0 && y2 < tj && z2 >= 0 && z2 < tk;
                    q[d] = in ? cc + y2 * tk + z2 : nullptr;
                    sys[d] = sx[d / 9];
                }
                dead = !wait_counters<27>(q, sys, need, wa.timeout_ns, wa.err);
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            vw2_produce(wa, ring_u32, full, empty, s, ph, ch, 1 + yb * VW_R, 1 + zb * VW_TZ,
                        (wa.parity0 + k) & 1);
        }
        return;
    }
    const uint32_t full_u32 = smem_u32(&full[0]), empty_u32 = smem_u32(&empty[0]);
    int slot = 0;
    uint32_t tph = 0;
    for (;;) {
        mbar_wait(&tq_full[slot], tph);
        const long long t = tq[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&tq_empty[slot]);
        if (++slot == WAVE_TQ) {
            slot = 0;
            tph ^= 1;
        }
        if (t < 0) break;
        const int k = (int)(t / T);
        const int64_t tile = t - (long long)k * T;
        const int64_t h = tile / per_chunk;
        const int64_t rem = tile - h * per_chunk;
        const int64_t yb = rem / tk;  // z fastest (see the producer)
        const int64_t zb = rem - yb * tk;
        const int64_t cidx = yb * tk + zb;  // the tile's counter within a chunk
        const int2 ch = wa.chains[h];
        double r1 = 0.0, r2 = 0.0;
        vw2_consume<!FAST, RESID, CHAIN>(wa, ring_u32, full_u32, empty_u32, s, ph, ch, 1 + yb * VW_R,
                                  1 + zb * VW_TZ, (wa.parity0 + k) & 1, r1, r2);
        if (RESID && wa.resid) {
            r1 = warp_max(r1);
            r2 = warp_max(r2);
            if (lane == 0) {
                red[0][warp] = r1;
                red[1][warp] = r2;
            }
        }
        // a chain whose end chunk faces another device is read by it (a tile
        // spans all planes): the consumers' stores are ordered before the
        // counter by the CTA barrier and thread 0's system-scope fence +
        // release (cumulative; a fence in every thread measured 4 % slower
        // on 4 GPUs and adds nothing)
        const bool xsys = (wa.nbr[wa.clist[ch.x]].sys | wa.nbr[wa.clist[ch.x + ch.y - 1]].sys) != 0;
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"n"(32 * VW_CW));
        if (tid == 0) {
            if (RESID && wa.resid) {
                double m1 = red[0][0], m2 = red[1][0];
#pragma unroll
                for (int w = 1; w < VW_CW; ++w) {
                    m1 = fmax(m1, red[0][w]);
                    m2 = fmax(m2, red[1][w]);
                }
                resid_max(wa.resid + 2 * k, m1);
                resid_max(wa.resid + 2 * k + 1, m2);
            }
            // the tile's (y, z) block of every chunk of the chain
            const unsigned v = wa.base + 2u * (unsigned)k + 2u;
            if (xsys) __threadfence_system();
            else __threadfence();
            for (int j = 0; j < ch.y; ++j) {
                unsigned int* d = wa.done + wa.clist[ch.x + j] * per_chunk + cidx;
                if (xsys)
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(d), "r"(v) : "memory");
                else
                    st_release_gpu_u32(d, v);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// plan: the per-GPU step engine

struct Plan {
    int gpu;
    hrt_chunk_layout_t L;
    int nchunks;
    ChunkBufs* d_chunks = nullptr;
    std::vector<ChunkBufs> h_chunks;
    hrt_halo_seg_t* d_segs = nullptr;
    int nsegs = 0;
    int64_t seg_blocks = 1;
    hrt_halo_seg_t* d_post = nullptr;
    int64_t* d_offs = nullptr;  // chunk origins in the field (field_copy)
    ChunkPush* d_push = nullptr;  // fused halo push table (slab variant 2)
    ChunkSide* d_sides = nullptr; // contiguous west/east ghost columns (push mode)
    VolPush* d_vpush = nullptr;   // fused 6-face halo push (volume plans, TMA kernel)
    bool ghosts_ready = false;    // ghost planes of the next buffer are current
    bool push_on() const { return d_push != nullptr && L.ndim == 2 && variant == 2; }
    bool vpush_on() const {
        return d_vpush != nullptr && L.ndim == 3 && variant != 0 && variant != 3 && L.origin % 2 == 1 &&
               L.stride[1] % 2 == 0;
    }
    bool any_push() const { return push_on() || vpush_on(); }
    // split schedule (push mode with remote faces): edge tiles first, the
    // NCCL exchange on `side` overlapped with the inner tiles
    int* d_tiles_edge = nullptr;
    int* d_tiles_inner = nullptr;
    int64_t n_edge = 0, n_inner = 0;
    int64_t split_rows = 0;  // rows value the tile lists were built for
    std::vector<int> remote_mask;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool split_on() const { return push_on() && side != nullptr && !remote.empty() && !ipc; }
    // IPC push mode: remote faces are pushed straight into the neighbour
    // processes' ghost planes (CUDA IPC mappings); per-step flags replace
    // the NCCL exchange (which only primes ghosts after an upload)
    bool ipc = false;
    unsigned long long* d_arrived = nullptr;          // owned by the caller
    unsigned long long** d_remote_slots = nullptr;    // device array (plan-owned)
    unsigned int* d_edge_done = nullptr;              // plan-owned, 2 slots
    int* d_err = nullptr;                             // plan-owned
    int n_nbr = 0;
    unsigned long long gstep = 0;                     // global step counter (tags)
    unsigned long long timeout_ns = 30000000000ULL;
    int* d_tiles_all = nullptr;                       // edge tiles then inner tiles
    bool ipc_on() const { return ipc && push_on(); }
    int npost = 0;
    int64_t post_blocks = 1;
    std::vector<hrt_remote_seg_t> remote;
    void* comm = nullptr;
    int64_t rows = 64;
    bool rows_explicit = false;   // set by hrt_jacobi_plan_set_rows
    int variant = 2;  // slab kernel: 0 LDG register march, 1 TMA ring, 2 TMA ring x4 cols
    bool nonneg = false;  // caller guarantees a finite field >= 0 (unguarded division)
    // graph of two steps (parity 0 then 1) per residual base pointer
    cudaGraphExec_t graph = nullptr;
    unsigned long long* graph_resid = nullptr;
    cudaStream_t graph_stream = nullptr;
    std::vector<cudaEvent_t> events;  // run_timed's per-launch events
    // persistent dataflow mode (single plan, no remote faces): see
    // slab_wave_kernel
    bool persist = false;
    std::vector<int> nbr;          // [nchunks][4] plan-local neighbour chunk or -1
    int* d_pnbr = nullptr;
    unsigned int* d_pdone = nullptr;   // per-tile step counters
    unsigned long long* d_pticket = nullptr;
    int pgrid = 0;                 // resident CTA slots of the current build (0: not built)
    int64_t ptiles = 0, pkey = -1;
    unsigned int pbase = 0;
    // wavefront across processes: neighbour ranks' tile counters (IPC)
    bool wave_ipc = false;
    int* d_rnbr = nullptr;
    int* d_rpeer = nullptr;
    unsigned int** d_peer_done = nullptr;
    unsigned long long persist_timeout_ns = 10000000000ULL;
    // chunks at most 256 wide run the 2-consumer-warp instances (no idle
    // threads); HRT_NARROW=0 forces the 4-warp ones (experiments)
    bool narrow_ok = true;
    bool narrow_chunk() const { return narrow_ok && L.ext[1] <= 256; }
    // two steps per pass (slab_wave2_kernel): one GPU, no faces to other
    // processes; HRT_FUSE2=0 turns it off
    int fuse2 = 1;  // 0 off, 1 when the problem has enough tiles, 2 always (tests)
    // Chunk count the tiling decisions (tile rows, two-step or not) are made
    // for: the largest chunk count per GPU over the whole decomposition, so
    // every GPU and rank of a run picks the same tiling — neighbours index
    // each other's tile counters with their own tiling and read each
    // other's buffers by pass parity (hrt_jacobi_plan_set_tiling_chunks;
    // 0 = this plan's own count)
    int64_t tiling_chunks = 0;
    int64_t tn() const { return tiling_chunks > 0 ? tiling_chunks : (int64_t)nchunks; }
    Nbr9* d_n9 = nullptr;          // [nchunks] 3 x 3 chunk neighbourhood
    int64_t n9_key = -1;           // tiles per chunk the table was built for
    // faces to other processes (hrt_jacobi_plan_set_wave2_remote): per chunk
    // and face N,S,W,E the mapped buffers and tile-counter base, or null
    // 3 x 3 chunk neighbourhood of the two-step slab passes when some of it
    // lives on other GPUs or in other processes ([nchunks][9], row-major
    // NW N NE W C E SW S SE; empty = all local, derived from nbr)
    struct R9 {
        int32_t kind;   // 0 none (domain), 1 this plan's chunk idx, 2 another device's
        int32_t idx;    // plan-local index, or the chunk's index in its own plan
        uint64_t cnt;   // kind 2: that plan's tile counters (mapped)
        uint64_t b[2];  // kind 2: its buffers (mapped)
    };
    std::vector<R9> r9;
    double* d_ones = nullptr;      // BOUNDARY row (rows outside the domain)
    // two steps per pass for x-band volumes (volume_wave2_kernel)
    std::vector<hrt_vpush_t> h_vpush;  // host copy of the push table (face kinds)
    unsigned int* d_v2done = nullptr;  // per-tile step counters (absolute; IPC-exported)
    unsigned int v2base = 0;           // every d_v2done entry between launches
    VW2Nbr* d_v2nbr = nullptr;         // [nchunks] x-neighbour table
    int2* d_v2chains = nullptr;        // chains of chunks linked along +x
    int* d_v2clist = nullptr;
    int v2nchains = 0;
    int64_t v2cdelta = 0;
    bool v2chained = false;            // some chain has more than one chunk
    bool v2dirty = true;               // maps / table to (re)build
    CUtensorMap* d_v2maps = nullptr;   // own [nchunks][2], then remote [nchunks][2 faces][2]
    // x faces to another process (hrt_jacobi_plan_set_vw2_remote): mapped
    // buffers [nchunks][2 faces][2 parities] and tile-0 counters [nchunks][2]
    std::vector<uint64_t> v2rbuf, v2rcnt;
    // field scan of the last upload (volume plans; see vw2_fast) and the
    // steps run since (saturating; "unknown" until the first scan)
    unsigned long long* d_range = nullptr;
    int64_t since_scan = int64_t(1) << 40;
    void count_steps(int64_t n) { since_scan = std::min<int64_t>(since_scan + n, int64_t(1) << 40); }
    int64_t v2_tiles = 0;
    int pgrid3 = 0;                    // resident CTA slots of volume_wave2_kernel
    int pgrid2 = 0;                // resident CTA slots of slab_wave2_kernel
    int64_t pkey2 = -1;
    bool fuse2_on() const {
        const bool local = !wave_ipc && remote.empty() && !ipc;
        return fuse2 && persist_on() && L.ndim == 2 && (local || !r9.empty()) &&
               L.ext[0] >= 2 && L.ext[1] >= 2 && L.ext[1] % 2 == 0 && rows >= 2 &&
               L.ext[0] % rows != 1 && (int64_t)nbr.size() == 4 * (int64_t)nchunks;
    }
    bool persist_on() const {
        return persist && any_push() && !nbr.empty() && (wave_ipc || (remote.empty() && !ipc));
    }
};

static int64_t blocks_for(const hrt_halo_seg_t* segs, int n) {
    int64_t mx = 1;
    for (int i = 0; i < n; ++i) mx = std::max<int64_t>(mx, segs[i].n0 * segs[i].n1);
    return std::max<int64_t>(1, (mx + HALO_THREADS * HALO_PER_THREAD - 1) /
                                    (HALO_THREADS * HALO_PER_THREAD));
}

}  // namespace hrt

using namespace hrt;

// NCCL hooks (hrt_nccl.cu)
extern "C" int hrt_nccl_exchange(void* comm, void* stream, const hrt_remote_seg_t* segs, int n,
                                 int parity);

// subset: 0 every tile, 1 the edge tiles (they feed remote faces), 2 the rest
static int launch_update(Plan* p, cudaStream_t s, int parity, unsigned long long* resid,
                         int subset = 0) {
    const hrt_chunk_layout_t& L = p->L;
    if (L.ndim == 2) {
        SlabArgs a{};
        a.chunks = p->d_chunks;
        a.push = p->push_on() ? p->d_push : nullptr;
        a.sides = p->push_on() && p->variant == 2 ? p->d_sides : nullptr;
        a.tiles = subset == 1   ? p->d_tiles_edge
                  : subset == 2 ? p->d_tiles_inner
                  : subset == 3 ? p->d_tiles_all
                                : nullptr;
        if (subset == 3 && p->ipc_on()) {
            a.arrived = p->d_arrived;
            a.remote_slots = p->d_remote_slots;
            a.n_nbr = p->n_nbr;
            a.edge_done = p->d_edge_done;
            a.n_edge = p->n_edge;
            a.tag = p->gstep + 1;
            a.timeout_ns = p->timeout_ns;
            a.err = p->d_err;
        }
        a.parity = parity;
        a.ex = L.ext[0];
        a.ey = L.ext[1];
        a.sx = L.stride[0];
        a.origin = L.origin;
        a.rows = p->rows;
        a.tiles_r = (a.ex + a.rows - 1) / a.rows;
        // chunks at most 256 wide (e.g. cfg5's 256^2 blocks) use 2 consumer
        // warps per CTA so no thread is idle
        const bool narrow = p->variant == 2 && p->narrow_chunk();
        const int cols = p->variant == 2 ? (narrow ? 256 : T4_COLS) : SLAB_COLS;
        a.tiles_c = (a.ey + cols - 1) / cols;
        a.resid = resid;
        a.zghost = HRT_BOUNDARY;
        a.ieee = p->variant == 3;
        const int64_t grid = subset == 1   ? p->n_edge
                             : subset == 2 ? p->n_inner
                             : subset == 3 ? p->n_edge + p->n_inner
                                           : (int64_t)p->nchunks * a.tiles_r * a.tiles_c;
        if (grid == 0) return HRT_OK;
        if (p->variant == 2) {
            const bool guard = !p->nonneg;
            const unsigned g = (unsigned)grid;
#define T4_LAUNCH(G, R, CW)                                                              \
    do {                                                                                 \
        if (a.push) slab_update_tma4_kernel<G, R, CW, true><<<g, 32 * (CW + 1), 0, s>>>(a); \
        else slab_update_tma4_kernel<G, R, CW, false><<<g, 32 * (CW + 1), 0, s>>>(a);      \
    } while (0)
            if (narrow) {
                if (guard && resid) T4_LAUNCH(true, true, 2);
                else if (guard) T4_LAUNCH(true, false, 2);
                else if (resid) T4_LAUNCH(false, true, 2);
                else T4_LAUNCH(false, false, 2);
            } else {
                if (guard && resid) T4_LAUNCH(true, true, 4);
                else if (guard) T4_LAUNCH(true, false, 4);
                else if (resid) T4_LAUNCH(false, true, 4);
                else T4_LAUNCH(false, false, 4);
            }
#undef T4_LAUNCH
        } else if (p->variant == 1) {
            slab_update_tma_kernel<<<(unsigned)grid, TMA_THREADS, 0, s>>>(a);
        } else {
            slab_update_kernel<<<(unsigned)grid, SLAB_THREADS, 0, s>>>(a);
        }
    } else {
        VolArgs a{};
        a.chunks = p->d_chunks;
        a.parity = parity;
        a.ex = L.ext[0];
        a.ey = L.ext[1];
        a.ez = L.ext[2];
        a.sx = L.stride[0];
        a.sy = L.stride[1];
        a.origin = L.origin;
        a.rows = p->rows;
        a.tiles_i = (a.ex + a.rows - 1) / a.rows;
        a.tiles_j = (a.ey + VOL_TY - 1) / VOL_TY;
        a.tiles_k = (a.ez + VOL_TX - 1) / VOL_TX;
        a.du = nullptr;
        a.dw = nullptr;
        a.flat = 0;
        a.ieee = p->variant == 3;
        a.resid = resid;
        a.vpush = p->vpush_on() ? p->d_vpush : nullptr;
        // TMA ring variant needs 16-byte aligned z rows (origin odd, sy even)
        const bool tma = p->variant != 0 && p->variant != 3 && (L.origin % 2 == 1) &&
                         (L.stride[1] % 2 == 0);
        if (tma) {
            a.tiles_j = (a.ey + V_CW - 1) / V_CW;
            a.tiles_k = (a.ez + V_ZW - 1) / V_ZW;
        }
        const int64_t grid = (int64_t)p->nchunks * a.tiles_i * a.tiles_j * a.tiles_k;
        if (grid == 0) return HRT_OK;
        if (tma && resid)
            volume_update_tma_kernel<true><<<(unsigned)grid, 32 * (V_CW + 1), V_SMEM, s>>>(a);
        else if (tma)
            volume_update_tma_kernel<false><<<(unsigned)grid, 32 * (V_CW + 1), V_SMEM, s>>>(a);
        else
            volume_update_kernel<<<(unsigned)grid, dim3(VOL_TX, VOL_TY), 0, s>>>(a);
    }
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

template <typename K>
static void carveout(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
}

static void set_carveouts() {
    // function attributes are per device context: once per GPU of the process
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (dev < 64 && (done >> dev) & 1) return;
    if (dev < 64) done |= 1ull << dev;
#define C4(G, R, CW)                                       \
    carveout(slab_update_tma4_kernel<G, R, CW, false>);   \
    carveout(slab_update_tma4_kernel<G, R, CW, true>)
    C4(true, true, 4); C4(true, false, 4); C4(false, true, 4); C4(false, false, 4);
    C4(true, true, 2); C4(true, false, 2); C4(false, true, 2); C4(false, false, 2);
#undef C4
    carveout(slab_wave_kernel<true, true, 4>);
    carveout(slab_wave_kernel<true, false, 4>);
    carveout(slab_wave_kernel<false, true, 4>);
    carveout(slab_wave_kernel<false, false, 4>);
    carveout(slab_wave_kernel<true, true, 2>);
    carveout(slab_wave_kernel<true, false, 2>);
    carveout(slab_wave_kernel<false, true, 2>);
    carveout(slab_wave_kernel<false, false, 2>);
#define C2(CW)                                    \
    carveout(slab_wave2_kernel<true, true, CW, false>);    \
    carveout(slab_wave2_kernel<true, false, CW, false>);   \
    carveout(slab_wave2_kernel<false, true, CW, false>);   \
    carveout(slab_wave2_kernel<false, false, CW, false>);  \
    carveout(slab_wave2_kernel<true, true, CW, true>);     \
    carveout(slab_wave2_kernel<true, false, CW, true>);    \
    carveout(slab_wave2_kernel<false, true, CW, true>);    \
    carveout(slab_wave2_kernel<false, false, CW, true>)
    C2(4);
    C2(2);
#undef C2
    carveout(slab_update_tma_kernel);
    carveout(volume_update_tma_kernel<true>);
    carveout(volume_wave_kernel<true>);
    carveout(volume_wave_kernel<false>);
    carveout(volume_update_tma_kernel<false>);
    cudaFuncSetAttribute(volume_update_tma_kernel<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V_SMEM);
    cudaFuncSetAttribute(volume_update_tma_kernel<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V_SMEM);
    cudaFuncSetAttribute(volume_wave_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)V_SMEM);
    cudaFuncSetAttribute(volume_wave_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)V_SMEM);
    cudaGetLastError();
}

static int launch_halo(Plan* p, cudaStream_t s, int parity) {
    if (p->nsegs > 0) {
        halo_copy_kernel<<<(unsigned)(p->nsegs * p->seg_blocks), HALO_THREADS, 0, s>>>(
            p->d_segs, parity, p->seg_blocks);
        HRT_CUDA(cudaGetLastError());
    }
    if (!p->remote.empty()) {
        Stream tmp;
        tmp.s = s;
        tmp.gpu = p->gpu;
        int rc = hrt_nccl_exchange(p->comm, &tmp, p->remote.data(), (int)p->remote.size(), parity);
        if (rc) return rc;
        if (p->npost > 0) {
            halo_copy_kernel<<<(unsigned)(p->npost * p->post_blocks), HALO_THREADS, 0, s>>>(
                p->d_post, parity, p->post_blocks);
            HRT_CUDA(cudaGetLastError());
        }
    }
    return HRT_OK;
}

// cross-process faces only: NCCL exchange of the (pushed or packed) staging
// buffers, then unpack into the ghost planes of `parity`
static int launch_remote(Plan* p, cudaStream_t s, int parity) {
    if (p->remote.empty()) return HRT_OK;
    Stream tmp;
    tmp.s = s;
    tmp.gpu = p->gpu;
    int rc = hrt_nccl_exchange(p->comm, &tmp, p->remote.data(), (int)p->remote.size(), parity);
    if (rc) return rc;
    if (p->npost > 0) {
        halo_copy_kernel<<<(unsigned)(p->npost * p->post_blocks), HALO_THREADS, 0, s>>>(
            p->d_post, parity, p->post_blocks);
        HRT_CUDA(cudaGetLastError());
    }
    return HRT_OK;
}

// Push mode: the update kernel writes the next buffer's ghost planes (and
// the remote send staging) itself, so a step is update + remote exchange;
// the full halo pass runs only when the ghosts are stale (after an upload).
static int prime_ghosts(Plan* p, cudaStream_t s, int parity) {
    if (!p->any_push() || p->ghosts_ready) return HRT_OK;
    int rc = launch_halo(p, s, parity);
    if (rc) return rc;
    p->ghosts_ready = true;
    return HRT_OK;
}

// (Re)build the edge / inner tile lists for the current tiling.
static int build_split(Plan* p) {
    const hrt_chunk_layout_t& L = p->L;
    const int64_t ex = L.ext[0], ey = L.ext[1];
    const int64_t tr = (ex + p->rows - 1) / p->rows;
    const int cols = p->narrow_chunk() ? 256 : T4_COLS;
    const int64_t tc = (ey + cols - 1) / cols;
    std::vector<int> edge, inner;
    for (int64_t c = 0; c < p->nchunks; ++c) {
        const int m = p->remote_mask[c];
        for (int64_t rb = 0; rb < tr; ++rb)
            for (int64_t cb = 0; cb < tc; ++cb) {
                const bool e = ((m & 1) && rb == 0) || ((m & 2) && rb == tr - 1) ||
                               ((m & 4) && cb == 0) || ((m & 8) && cb == tc - 1);
                auto& v = e ? edge : inner;
                v.push_back((int)c);
                v.push_back((int)rb);
                v.push_back((int)cb);
            }
    }
    cudaFree(p->d_tiles_edge);
    cudaFree(p->d_tiles_inner);
    cudaFree(p->d_tiles_all);
    p->d_tiles_edge = p->d_tiles_inner = p->d_tiles_all = nullptr;
    p->n_edge = (int64_t)edge.size() / 3;
    p->n_inner = (int64_t)inner.size() / 3;
    {
        std::vector<int> all(edge);
        all.insert(all.end(), inner.begin(), inner.end());
        if (!all.empty()) {
            HRT_CUDA(cudaMalloc(&p->d_tiles_all, all.size() * sizeof(int)));
            HRT_CUDA(cudaMemcpy(p->d_tiles_all, all.data(), all.size() * sizeof(int),
                                cudaMemcpyHostToDevice));
        }
    }
    if (!edge.empty()) {
        HRT_CUDA(cudaMalloc(&p->d_tiles_edge, edge.size() * sizeof(int)));
        HRT_CUDA(cudaMemcpy(p->d_tiles_edge, edge.data(), edge.size() * sizeof(int),
                            cudaMemcpyHostToDevice));
    }
    if (!inner.empty()) {
        HRT_CUDA(cudaMalloc(&p->d_tiles_inner, inner.size() * sizeof(int)));
        HRT_CUDA(cudaMemcpy(p->d_tiles_inner, inner.data(), inner.size() * sizeof(int),
                            cudaMemcpyHostToDevice));
    }
    p->split_rows = p->rows;
    return HRT_OK;
}

template <int CW>
static int wave_occupancy(bool guard) {
    int dev = 0, sms = 0, a = 0, b = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (guard) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, slab_wave_kernel<true, true, CW>,
                                                      32 * (CW + 1), 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, slab_wave_kernel<true, false, CW>,
                                                      32 * (CW + 1), 0);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, slab_wave_kernel<false, true, CW>,
                                                      32 * (CW + 1), 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, slab_wave_kernel<false, false, CW>,
                                                      32 * (CW + 1), 0);
    }
    return std::min(a, b) * sms;
}

// (Re)build the wavefront tables: per-tile counters and the neighbour table
static int build_wave(Plan* p, int64_t ntiles) {
    // the counters keep their values (all == pbase between launches) unless
    // the tile count changes; with cross-process waves they are IPC-mapped
    // by the neighbours and must never move
    if (p->d_pdone && p->ptiles != ntiles) {
        if (p->wave_ipc) {
            set_error("wavefront tiling changed after the counters were shared over IPC");
            return HRT_E_INVALID;
        }
        cudaFree(p->d_pdone);
        p->d_pdone = nullptr;
    }
    p->pgrid = 0;
    const bool narrow = p->narrow_chunk();
    int G = 0;
    if (p->L.ndim == 3) {
        int dev = 0, sms = 0, a = 0, b = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, volume_wave_kernel<true>, 32 * (V_CW + 1), V_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, volume_wave_kernel<false>, 32 * (V_CW + 1), V_SMEM);
        G = std::min(a, b) * sms;
    } else {
        G = narrow ? wave_occupancy<2>(!p->nonneg) : wave_occupancy<4>(!p->nonneg);
    }
    HRT_CUDA(cudaGetLastError());
    if (G <= 0) {
        set_error("persistent kernel: no resident CTA slots");
        return HRT_E_CUDA;
    }
    if (!p->d_pdone) {
        HRT_CUDA(cudaMalloc(&p->d_pdone, sizeof(unsigned int) * std::max<int64_t>(1, ntiles)));
        HRT_CUDA(cudaMemset(p->d_pdone, 0, sizeof(unsigned int) * std::max<int64_t>(1, ntiles)));
        p->pbase = 0;
    }
    if (!p->d_pnbr) {
        HRT_CUDA(cudaMalloc(&p->d_pnbr, sizeof(int) * p->nbr.size()));
        HRT_CUDA(cudaMemcpy(p->d_pnbr, p->nbr.data(), sizeof(int) * p->nbr.size(),
                            cudaMemcpyHostToDevice));
    }
    if (!p->d_pticket) HRT_CUDA(cudaMalloc(&p->d_pticket, sizeof(unsigned long long)));
    if (!p->d_err) {
        HRT_CUDA(cudaMalloc(&p->d_err, sizeof(int)));
        HRT_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
    }
    p->pgrid = G;
    p->pkey = ntiles * 4 + (p->nonneg ? 1 : 0);
    p->ptiles = ntiles;
    return HRT_OK;
}

static int64_t wave_tiles(const Plan* p, int64_t* tiles_c_out = nullptr) {
    const int64_t ex = p->L.ext[0], ey = p->L.ext[1];
    if (p->L.ndim == 3)
        return (int64_t)p->nchunks * ((ex + p->rows - 1) / p->rows) * ((ey + V_CW - 1) / V_CW) *
               ((p->L.ext[2] + V_ZW - 1) / V_ZW);
    const int cols = p->narrow_chunk() ? 256 : T4_COLS;
    const int64_t tc = (ey + cols - 1) / cols;
    if (tiles_c_out) *tiles_c_out = tc;
    return (int64_t)p->nchunks * ((ex + p->rows - 1) / p->rows) * tc;
}

static SlabArgs slab_args(Plan* p, int parity, unsigned long long* resid) {
    const hrt_chunk_layout_t& L = p->L;
    SlabArgs a{};
    a.chunks = p->d_chunks;
    a.push = p->push_on() ? p->d_push : nullptr;
    a.sides = p->push_on() ? p->d_sides : nullptr;
    a.parity = parity;
    a.ex = L.ext[0];
    a.ey = L.ext[1];
    a.sx = L.stride[0];
    a.origin = L.origin;
    a.rows = p->rows;
    a.tiles_r = (a.ex + a.rows - 1) / a.rows;
    a.resid = resid;
    a.zghost = HRT_BOUNDARY;
    return a;
}

// volume plans: steps [first, first+n) in one volume_wave_kernel launch
static int launch_persist3(Plan* p, cudaStream_t s, int64_t first, int64_t n,
                           unsigned long long* resid_base) {
    const hrt_chunk_layout_t& L = p->L;
    const int64_t T = wave_tiles(p);
    if (T == 0) return HRT_OK;
    int rc;
    if (p->pgrid == 0 || p->ptiles != T || p->pkey != T * 4 + (p->nonneg ? 1 : 0)) {
        HRT_CUDA(cudaStreamSynchronize(s));
        rc = build_wave(p, T);
        if (rc) return rc;
    }
    HRT_CUDA(cudaMemsetAsync(p->d_pticket, 0, sizeof(unsigned long long), s));
    VolWaveArgs wa{};
    VolArgs& a = wa.v;
    a.chunks = p->d_chunks;
    a.parity = (int)(first & 1);
    a.ex = L.ext[0];
    a.ey = L.ext[1];
    a.ez = L.ext[2];
    a.sx = L.stride[0];
    a.sy = L.stride[1];
    a.origin = L.origin;
    a.rows = p->rows;
    a.tiles_i = (a.ex + a.rows - 1) / a.rows;
    a.tiles_j = (a.ey + V_CW - 1) / V_CW;
    a.tiles_k = (a.ez + V_ZW - 1) / V_ZW;
    a.vpush = p->d_vpush;
    wa.nbr = p->d_pnbr;
    wa.done = p->d_pdone;
    wa.ticket = p->d_pticket;
    wa.base = p->pbase;
    wa.nsteps = (int)n;
    wa.parity0 = (int)(first & 1);
    wa.ntiles = T;
    wa.resid = resid_base ? resid_base + first : nullptr;
    wa.timeout_ns = p->persist_timeout_ns;
    wa.err = p->d_err;
    if (p->wave_ipc) {
        wa.rnbr = p->d_rnbr;
        wa.rpeer = p->d_rpeer;
        wa.peer_done = p->d_peer_done;
    }
    void* fn = resid_base ? (void*)volume_wave_kernel<true> : (void*)volume_wave_kernel<false>;
    const unsigned grid = (unsigned)std::min<int64_t>(p->pgrid, T);
    void* args[] = {&wa};
    HRT_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(32 * (V_CW + 1)), args, V_SMEM, s));
    p->pbase += (unsigned)n;
    return HRT_OK;
}

static int launch_persist1(Plan* p, cudaStream_t s, int64_t first, int64_t n,
                           unsigned long long* resid_base);

// resident CTAs of the two-step kernel on this GPU (3 per SM for 512-wide
// tiles, 5 for 256-wide; from the occupancy API once known)
// (a function of the layout and the SM count only — not of launch history —
// so the decision is the same before and after the first launch)
static int64_t fuse2_slots(const Plan* p) {
    return (int64_t)sm_count(p->gpu) * (p->narrow_chunk() ? HRT_W2_MINB2 : HRT_W2_MINB4);
}

// two-step passes pay off only with at least one tile per resident CTA
// (smaller problems: a two-step tile pass is twice as long and too few run
// at once — 2048^2 in 8x8 chunks: 64 vs 129 GLUPS one step per pass);
// counted for tn() chunks so every GPU of a decomposition decides alike
static bool fuse2_use(const Plan* p) {
    if (!p->fuse2_on()) return false;
    if (p->fuse2 == 2) return true;
    // with tile heights chosen for parallelism (hrt_jacobi_plan_set_persistent)
    // two-step passes measured faster at every size, also where tiles are
    // fewer than CTA slots (1024^2: 110 vs 85 GLUPS one step per pass);
    // explicitly tall tiles on a small problem keep one step per pass
    const int64_t per_chunk = wave_tiles(p) / std::max(1, p->nchunks);
    return p->rows <= 16 || per_chunk * p->tn() >= fuse2_slots(p);
}

// steps per fused pass this plan runs (0: one step per pass)
static bool vfuse2_use(const Plan* p);
static int pass_steps_of(const Plan* p) {
    return (p->L.ndim == 3 ? vfuse2_use(p) : fuse2_use(p)) ? 2 : 0;
}

template <bool G, bool R, int CW, bool F>
static int w2_blocks_per_sm() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, slab_wave2_kernel<G, R, CW, F>,
                                                  w2_threads(CW), 0);
    return n;
}

// co-resident CTAs of every instance a launch may pick (cooperative launch)
template <int CW>
static int wave2_occupancy(bool guard) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int n = guard ? std::min(std::min(w2_blocks_per_sm<true, true, CW, false>(),
                                            w2_blocks_per_sm<true, false, CW, false>()),
                                   std::min(w2_blocks_per_sm<true, true, CW, true>(),
                                            w2_blocks_per_sm<true, false, CW, true>()))
                        : std::min(std::min(w2_blocks_per_sm<false, true, CW, false>(),
                                            w2_blocks_per_sm<false, false, CW, false>()),
                                   std::min(w2_blocks_per_sm<false, true, CW, true>(),
                                            w2_blocks_per_sm<false, false, CW, true>()));
    return n * sm_count(dev);
}

// nf passes (2 steps each) from step `first` in one slab_wave2_kernel launch
static int launch_fused(Plan* p, cudaStream_t s, int64_t first, int64_t nf,
                        unsigned long long* resid_base) {
    if (nf <= 0) return HRT_OK;
    const bool narrow = p->narrow_chunk();
    int64_t tc = 0;
    const int64_t T = wave_tiles(p, &tc);
    if (T == 0) return HRT_OK;
    int rc;
    if (p->pgrid == 0 || p->ptiles != T || p->pkey != T * 4 + (p->nonneg ? 1 : 0)) {
        HRT_CUDA(cudaStreamSynchronize(s));  // counters reset: nothing may be in flight
        rc = build_wave(p, T);
        if (rc) return rc;
    }
    const int64_t per_chunk = T / std::max(1, p->nchunks);
    if (!p->d_n9 || p->n9_key != per_chunk) {
        std::vector<Nbr9> n9((size_t)p->nchunks);
        auto at = [&](int c, int f) { return c < 0 ? -1 : p->nbr[4 * (size_t)c + f]; };
        for (int c = 0; c < p->nchunks; ++c) {
            Nbr9& o = n9[c];
            memset(&o, 0, sizeof(o));
            if (!p->r9.empty()) {  // neighbourhood given, partly on other devices
                for (int e = 0; e < 9; ++e) {
                    const Plan::R9& r = p->r9[9 * (size_t)c + e];
                    if (r.kind == 1) {
                        o.b[e][0] = p->h_chunks[r.idx].b[0];
                        o.b[e][1] = p->h_chunks[r.idx].b[1];
                        o.cnt[e] = p->d_pdone + (int64_t)r.idx * per_chunk;
                    } else if (r.kind == 2) {
                        o.b[e][0] = reinterpret_cast<double*>(r.b[0]);
                        o.b[e][1] = reinterpret_cast<double*>(r.b[1]);
                        o.cnt[e] = reinterpret_cast<unsigned int*>(r.cnt) + (int64_t)r.idx * per_chunk;
                        o.sysmask |= 1u << e;
                    }
                }
                continue;
            }
            const int n = at(c, 0), so = at(c, 1);
            const int idx[9] = {at(n, 2), n, at(n, 3), at(c, 2), c, at(c, 3),
                                at(so, 2), so, at(so, 3)};
            for (int e = 0; e < 9; ++e) {
                if (idx[e] < 0) continue;
                o.b[e][0] = p->h_chunks[idx[e]].b[0];
                o.b[e][1] = p->h_chunks[idx[e]].b[1];
                o.cnt[e] = p->d_pdone + (int64_t)idx[e] * per_chunk;
            }
        }
        cudaFree(p->d_n9);
        p->d_n9 = nullptr;
        HRT_CUDA(cudaMalloc(&p->d_n9, sizeof(Nbr9) * n9.size()));
        HRT_CUDA(cudaMemcpy(p->d_n9, n9.data(), sizeof(Nbr9) * n9.size(), cudaMemcpyHostToDevice));
        p->n9_key = per_chunk;
    }
    if (!p->d_ones) {
        std::vector<double> ones(T4_COLS + 8, HRT_BOUNDARY);
        HRT_CUDA(cudaMalloc(&p->d_ones, sizeof(double) * ones.size()));
        HRT_CUDA(cudaMemcpy(p->d_ones, ones.data(), sizeof(double) * ones.size(),
                            cudaMemcpyHostToDevice));
    }
    const int64_t key2 = T * 4 + (p->nonneg ? 1 : 0);
    int& pg = p->pgrid2;
    if (pg == 0 || p->pkey2 != key2) {
        pg = narrow ? wave2_occupancy<2>(!p->nonneg) : wave2_occupancy<4>(!p->nonneg);
        HRT_CUDA(cudaGetLastError());
        if (pg <= 0) {
            set_error("two-step kernel: no resident CTA slots");
            return HRT_E_CUDA;
        }
        p->pkey2 = key2;
    }
    HRT_CUDA(cudaMemsetAsync(p->d_pticket, 0, sizeof(unsigned long long), s));
    const hrt_chunk_layout_t& L = p->L;
    Wave2Args wa{};
    wa.n9 = p->d_n9;
    wa.done = p->d_pdone;
    wa.ticket = p->d_pticket;
    wa.base = p->pbase;
    wa.nfused = (int)nf;
    wa.parity0 = (int)(first & 1);
    wa.ntiles = T;
    wa.ex = L.ext[0];
    wa.ey = L.ext[1];
    wa.sx = L.stride[0];
    wa.origin = L.origin;
    wa.rows = p->rows;
    wa.tiles_r = (L.ext[0] + p->rows - 1) / p->rows;
    wa.tiles_c = tc;
    wa.resid = resid_base ? resid_base + first : nullptr;
    wa.ones = p->d_ones;
    wa.timeout_ns = p->persist_timeout_ns;
    wa.err = p->d_err;
    wa.zghost = HRT_BOUNDARY;
    const bool guard = !p->nonneg, res = resid_base != nullptr;
    void* fn;
    int threads;
    // every column tile full: the chunk width is a multiple of the tile's
    const bool full = L.ext[1] % (narrow ? 256 : T4_COLS) == 0;
#define WK2(G, R, CW, F) (void*)slab_wave2_kernel<G, R, CW, F>
#define PICKF(CW, F)                                                    \
    (guard ? (res ? WK2(true, true, CW, F) : WK2(true, false, CW, F))    \
           : (res ? WK2(false, true, CW, F) : WK2(false, false, CW, F)))
#define PICK(CW) (full ? PICKF(CW, true) : PICKF(CW, false))
    const size_t smem = 0;
    fn = narrow ? PICK(2) : PICK(4);
    threads = w2_threads(narrow ? 2 : 4);
#undef PICK
#undef PICKF
#undef WK2
    const unsigned grid = (unsigned)std::min<int64_t>(pg, T);
    void* args[] = {&wa};
    HRT_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3((unsigned)threads), args, smem, s));
    p->pbase += 2u * (unsigned)nf;
    p->ghosts_ready = false;  // passes read neighbours in place; ghost planes went stale
    return HRT_OK;
}

// ---- two steps per pass for volumes (volume_wave2_kernel) ----
// x-band volumes on one GPU: every y and z face a domain face, x faces to
// chunks of this plan or the domain (never to another GPU or process)
static bool vfuse2_on(const Plan* p) {
    const hrt_chunk_layout_t& L = p->L;
    if (!p->fuse2 || L.ndim != 3 || !p->persist_on() || p->ipc) return false;
    if (!p->wave_ipc && !p->remote.empty()) return false;
    if (L.ext[0] < 2 || L.origin % 2 != 1 || L.stride[0] % 2 != 0 || L.stride[1] % 2 != 0)
        return false;
    if ((int64_t)p->nbr.size() != 6 * (int64_t)p->nchunks ||
        (int64_t)p->h_vpush.size() != (int64_t)p->nchunks)
        return false;
    for (int c = 0; c < p->nchunks; ++c)
        for (int f = 0; f < 6; ++f) {
            const int n = p->nbr[6 * (size_t)c + f];
            const hrt_vpush_t& v = p->h_vpush[c];
            const bool other_gpu = n < 0 && (v.ptr[f][0] || v.ptr[f][1]);
            if (f >= 2 && (n >= 0 || other_gpu)) return false;  // y / z: domain faces only
            if (!other_gpu) continue;
            // x face to another GPU: only another process's chunk whose
            // buffers and counters are mapped (hrt_jacobi_plan_set_vw2_remote)
            if (!p->wave_ipc || p->v2rcnt.empty() || !p->v2rcnt[2 * (size_t)c + f] ||
                !p->v2rbuf[4 * (size_t)c + 2 * f] || !p->v2rbuf[4 * (size_t)c + 2 * f + 1])
                return false;
        }
    return true;
}

static int64_t vw2_tiles(const Plan* p, int64_t* tj = nullptr, int64_t* tk = nullptr) {
    const int64_t a = (p->L.ext[1] + VW_R - 1) / VW_R, b = (p->L.ext[2] + VW_TZ - 1) / VW_TZ;
    if (tj) *tj = a;
    if (tk) *tk = b;
    return (int64_t)p->nchunks * a * b;
}

template <bool F, bool R, bool C>
static int vw2_blocks_per_sm() {
    int n = 0;
    cudaFuncSetAttribute(volume_wave2_kernel<F, R, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)VW_SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, volume_wave2_kernel<F, R, C>,
                                                  32 * (VW_CW + 1), VW_SMEM);
    return n;
}

// 3D tensor maps of every chunk buffer: dims (sy, ey+2, ex+2) from the
// buffer base, box 124 x 8 x 1 (one plane of a tile), out-of-range
// coordinates zero-filled
static int build_vw2_maps(Plan* p) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        HRT_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000,
                                                  cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return HRT_E_UNSUPPORTED;
        }
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const hrt_chunk_layout_t& L = p->L;
    std::vector<CUtensorMap> maps(6 * (size_t)p->nchunks);
    memset(maps.data(), 0, sizeof(CUtensorMap) * maps.size());
    const cuuint64_t dims[3] = {(cuuint64_t)L.stride[1], (cuuint64_t)(L.ext[1] + 2),
                                (cuuint64_t)(L.ext[0] + 2)};
    const cuuint64_t strides[2] = {(cuuint64_t)L.stride[1] * 8, (cuuint64_t)L.stride[0] * 8};
    const cuuint32_t box[3] = {VW_RS, VW_RR, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    auto enc = [&](CUtensorMap* m, void* base) -> int {
        CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
            return HRT_E_CUDA;
        }
        return HRT_OK;
    };
    const size_t R = 2 * (size_t)p->nchunks;  // remote maps start here
    for (int c = 0; c < p->nchunks; ++c)
        for (int par = 0; par < 2; ++par) {
            int rc = enc(&maps[2 * (size_t)c + par], p->h_chunks[c].b[par]);
            if (rc) return rc;
            for (int f = 0; f < 2 && !p->v2rbuf.empty(); ++f) {
                const uint64_t b = p->v2rbuf[4 * (size_t)c + 2 * f + par];
                if (!b) continue;
                rc = enc(&maps[R + 4 * (size_t)c + 2 * f + par], reinterpret_cast<void*>(b));
                if (rc) return rc;
            }
        }
    cudaFree(p->d_v2maps);
    p->d_v2maps = nullptr;
    HRT_CUDA(cudaMalloc(&p->d_v2maps, sizeof(CUtensorMap) * maps.size()));
    HRT_CUDA(cudaMemcpy(p->d_v2maps, maps.data(), sizeof(CUtensorMap) * maps.size(),
                        cudaMemcpyHostToDevice));
    return HRT_OK;
}

// per-tile step counters of the volume two-step passes: allocated once
// (zero), absolute (v2base between launches), exported over CUDA IPC to the
// neighbour processes, so never reset or reallocated
static int ensure_vw2_counters(Plan* p) {
    const int64_t T = vw2_tiles(p);
    if (p->d_v2done) {
        if (p->v2_tiles != T) {
            set_error("volume two-step tiling changed after the counters were allocated");
            return HRT_E_INVALID;
        }
        return HRT_OK;
    }
    HRT_CUDA(cudaMalloc(&p->d_v2done, sizeof(unsigned int) * std::max<int64_t>(1, T)));
    HRT_CUDA(cudaMemset(p->d_v2done, 0, sizeof(unsigned int) * std::max<int64_t>(1, T)));
    p->v2_tiles = T;
    p->v2base = 0;
    return HRT_OK;
}

// x-neighbour table of the volume two-step kernel (maps already built)
static int build_vw2_nbr(Plan* p) {
    const int64_t per_chunk = vw2_tiles(p) / std::max(1, p->nchunks);
    const size_t R = 2 * (size_t)p->nchunks;
    std::vector<VW2Nbr> t((size_t)std::max(1, p->nchunks));
    for (int c = 0; c < p->nchunks; ++c) {
        VW2Nbr& o = t[c];
        memset(&o, 0, sizeof(o));
        for (int f = 0; f < 2; ++f) {
            const int n = p->nbr[6 * (size_t)c + f];
            if (n >= 0) {
                o.map[f][0] = p->d_v2maps + 2 * (size_t)n;
                o.map[f][1] = p->d_v2maps + 2 * (size_t)n + 1;
                o.cnt[f] = p->d_v2done + (int64_t)n * per_chunk;
            } else if (!p->v2rcnt.empty() && p->v2rcnt[2 * (size_t)c + f]) {
                o.map[f][0] = p->d_v2maps + R + 4 * (size_t)c + 2 * f;
                o.map[f][1] = p->d_v2maps + R + 4 * (size_t)c + 2 * f + 1;
                o.cnt[f] = reinterpret_cast<const unsigned int*>(p->v2rcnt[2 * (size_t)c + f]);
                o.sys |= 1u << f;
            }
        }
    }
    cudaFree(p->d_v2nbr);
    p->d_v2nbr = nullptr;
    HRT_CUDA(cudaMalloc(&p->d_v2nbr, sizeof(VW2Nbr) * t.size()));
    HRT_CUDA(cudaMemcpy(p->d_v2nbr, t.data(), sizeof(VW2Nbr) * t.size(), cudaMemcpyHostToDevice));
    // chains: from each chunk without a -x neighbour in this plan, follow
    // the +x neighbours.  A tile streams a whole chain (no rim planes and
    // no tile start-up between its chunks: 32-plane chunks ran at 315
    // GLUPS one by one vs 526 for 128-plane ones); the output pointer steps
    // from chunk to chunk by one constant, so chains need equally spaced
    // buffers (the solver allocates them in order) — else single chunks
    std::vector<std::vector<int>> chains;
    std::vector<char> seen((size_t)p->nchunks, 0);
    for (int c = 0; c < p->nchunks; ++c) {
        if (p->nbr[6 * (size_t)c] >= 0) continue;
        std::vector<int> ch;
        for (int x = c; x >= 0 && !seen[x]; x = p->nbr[6 * (size_t)x + 1]) {
            seen[x] = 1;
            ch.push_back(x);
        }
        chains.push_back(ch);
    }
    for (int c = 0; c < p->nchunks; ++c)
        if (!seen[c]) chains.push_back({c});  // (a cycle cannot occur; defensive)
    {
        // chains of up to ~256 planes: long enough that short chunks pay
        // no per-tile start-up, short enough that adjacent tiles do not
        // drift apart by more than L2 keeps their shared rows (1028-plane
        // chains read 39 GB of DRAM per 4 paper3d passes, 256-plane ones
        // less at the same speed); HRT_VW2_CHAIN overrides (experiments)
        size_t cap = (size_t)std::max<int64_t>(1, 256 / std::max<int64_t>(1, p->L.ext[0]));
        if (const char* e = getenv("HRT_VW2_CHAIN")) cap = (size_t)std::max(1, atoi(e));
        std::vector<std::vector<int>> cut;
        for (const auto& ch : chains)
            for (size_t j = 0; j < ch.size(); j += cap)
                cut.emplace_back(ch.begin() + j, ch.begin() + std::min(ch.size(), j + cap));
        chains.swap(cut);
    }
    const hrt_chunk_layout_t& L = p->L;
    int64_t cstride = 0;
    bool uniform = true;
    for (const auto& ch : chains)
        for (size_t j = 0; j + 1 < ch.size(); ++j)
            for (int par = 0; par < 2; ++par) {
                const int64_t d = (reinterpret_cast<intptr_t>(p->h_chunks[ch[j + 1]].b[par]) -
                                   reinterpret_cast<intptr_t>(p->h_chunks[ch[j]].b[par]));
                if (d % 8 != 0 || (cstride != 0 && d != cstride)) uniform = false;
                cstride = d;
            }
    if (!uniform) {
        std::vector<std::vector<int>> single;
        for (const auto& ch : chains)
            for (int c : ch) single.push_back({c});
        chains.swap(single);
        cstride = 0;
    }
    std::vector<int2> ctab;
    std::vector<int> clist;
    for (const auto& ch : chains) {
        ctab.push_back(make_int2((int)clist.size(), (int)ch.size()));
        clist.insert(clist.end(), ch.begin(), ch.end());
    }
    p->v2nchains = (int)ctab.size();
    p->v2cdelta = cstride / 8 - L.ext[0] * L.stride[0];
    p->v2chained = false;
    for (const auto& c : ctab) p->v2chained |= c.y > 1;
    cudaFree(p->d_v2chains);
    cudaFree(p->d_v2clist);
    p->d_v2chains = nullptr;
    p->d_v2clist = nullptr;
    HRT_CUDA(cudaMalloc(&p->d_v2chains, sizeof(int2) * std::max<size_t>(1, ctab.size())));
    HRT_CUDA(cudaMalloc(&p->d_v2clist, sizeof(int) * std::max<size_t>(1, clist.size())));
    if (!ctab.empty()) {
        HRT_CUDA(cudaMemcpy(p->d_v2chains, ctab.data(), sizeof(int2) * ctab.size(),
                            cudaMemcpyHostToDevice));
        HRT_CUDA(cudaMemcpy(p->d_v2clist, clist.data(), sizeof(int) * clist.size(),
                            cudaMemcpyHostToDevice));
    }
    return HRT_OK;
}

// volume tiles are 2 x 4 x 120 (a pass is one tile per CTA slot at least)
static bool vfuse2_use(const Plan* p) {
    if (!vfuse2_on(p)) return false;
    if (p->fuse2 == 2) return true;
    const int64_t per_chunk = vw2_tiles(p) / std::max(1, p->nchunks);
    return per_chunk * p->tn() >= (int64_t)sm_count(p->gpu) * 3;
}

static int launch_vfused(Plan* p, cudaStream_t s, int64_t first, int64_t nf,
                         unsigned long long* resid_base) {
    if (nf <= 0) return HRT_OK;
    const hrt_chunk_layout_t& L = p->L;
    int64_t tj = 0, tk = 0;
    if (vw2_tiles(p, &tj, &tk) == 0) return HRT_OK;
    int rc = ensure_vw2_counters(p);
    if (rc) return rc;
    if (p->v2dirty) {
        HRT_CUDA(cudaStreamSynchronize(s));  // the table of a launch in flight
        rc = build_vw2_maps(p);
        if (rc) return rc;
        rc = build_vw2_nbr(p);
        if (rc) return rc;
        p->v2dirty = false;
    }
    const int64_t T = (int64_t)p->v2nchains * tj * tk;  // tiles: (chain, y block, z block)
    if (!p->d_range) {  // never scanned: "unknown" (guarded division)
        HRT_CUDA(cudaMalloc(&p->d_range, 2 * sizeof(unsigned long long)));
        const unsigned long long h[2] = {0ull, 1ull};
        HRT_CUDA(cudaMemcpy(p->d_range, h, sizeof(h), cudaMemcpyHostToDevice));
        p->since_scan = int64_t(1) << 40;
    }
    if (!p->d_pticket) HRT_CUDA(cudaMalloc(&p->d_pticket, sizeof(unsigned long long)));
    if (!p->d_err) {
        HRT_CUDA(cudaMalloc(&p->d_err, sizeof(int)));
        HRT_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
    }
    if (p->pgrid3 == 0) {
        const int n = std::min(std::min(vw2_blocks_per_sm<true, true, true>(), vw2_blocks_per_sm<true, false, true>()),
                               std::min(vw2_blocks_per_sm<false, true, true>(), vw2_blocks_per_sm<false, false, true>()));
        HRT_CUDA(cudaGetLastError());
        if (n <= 0) {
            set_error("volume two-step kernel: no resident CTA slots");
            return HRT_E_CUDA;
        }
        p->pgrid3 = n * sm_count(p->gpu);
    }
    HRT_CUDA(cudaMemsetAsync(p->d_pticket, 0, sizeof(unsigned long long), s));
    VolW2Args wa{};
    wa.chunks = p->d_chunks;
    wa.nbr = p->d_v2nbr;
    wa.chains = p->d_v2chains;
    wa.clist = p->d_v2clist;
    wa.cdelta = p->v2cdelta;
    wa.done = p->d_v2done;
    wa.base = p->v2base;
    wa.ticket = p->d_pticket;
    wa.nfused = (int)nf;
    wa.parity0 = (int)(first & 1);
    wa.ntiles = T;
    wa.ex = L.ext[0];
    wa.ey = L.ext[1];
    wa.ez = L.ext[2];
    wa.sx = L.stride[0];
    wa.sy = L.stride[1];
    wa.origin = L.origin;
    wa.tiles_j = tj;
    wa.tiles_k = tk;
    wa.resid = resid_base ? resid_base + first : nullptr;
    wa.maps = p->d_v2maps;
    wa.range = p->d_range;
    // exact unguarded division needs min positive >= 2^-1019 * 6.000001^n
    // for n = steps since the scan, this run included (see vw2_fast)
    wa.need = p->since_scan > 400 ? HUGE_VAL
                                  : std::ldexp(1.0, -1019) * std::pow(6.000001, (double)p->since_scan);
    wa.timeout_ns = p->persist_timeout_ns;
    wa.err = p->d_err;
    // the unguarded instance, then the guarded one: exactly one of them
    // works (vw2_fast), the other returns at entry
#define VW2K(F, R) ((void*)volume_wave2_kernel<F, R, true>)
    void* fns[2] = {resid_base ? VW2K(true, true) : VW2K(true, false),
                    resid_base ? VW2K(false, true) : VW2K(false, false)};
#undef VW2K
    const unsigned grid = (unsigned)std::min<int64_t>(p->pgrid3, T);
    void* args[] = {&wa};
    for (void* fn : fns)
        HRT_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(32 * (VW_CW + 1)), args, VW_SMEM, s));
    p->v2base += 2u * (unsigned)nf;
    p->ghosts_ready = false;  // passes read neighbours in place; ghost planes went stale
    return HRT_OK;
}

// steps [first, first+n): on a single-GPU slab plan, passes of two steps
// (after n mod 4 single steps, so the result lands in the buffer of parity
// (first+n) mod 2 like single steps); otherwise one wavefront launch
static int launch_persist(Plan* p, cudaStream_t s, int64_t first, int64_t n,
                          unsigned long long* resid_base) {
    if (n <= 0) return HRT_OK;
    const bool vol = p->L.ndim == 3;
    // volume single steps and passes keep separate counters: with
    // neighbours on other devices the caller issues them as separate
    // launches with a fence between (jacobi.py _run_segments); a mixed run
    // arriving here anyway runs as single steps
    const bool mixed_ok = !vol || !p->wave_ipc || n % 4 == 0;
    if ((vol ? vfuse2_use(p) : fuse2_use(p)) && n >= 4 && mixed_ok) {
        const int64_t nf = (n / 4) * 2, nr = n - 2 * nf;
        int rc = nr ? launch_persist1(p, s, first, nr, resid_base) : HRT_OK;
        if (rc) return rc;
        return vol ? launch_vfused(p, s, first + nr, nf, resid_base)
                   : launch_fused(p, s, first + nr, nf, resid_base);
    }
    return launch_persist1(p, s, first, n, resid_base);
}

// steps [first, first+n) in one persistent wavefront launch
static int launch_persist1(Plan* p, cudaStream_t s, int64_t first, int64_t n,
                           unsigned long long* resid_base) {
    if (n <= 0) return HRT_OK;
    const int parity0 = (int)(first & 1);
    int rc = prime_ghosts(p, s, parity0);
    if (rc) return rc;
    if (p->L.ndim == 3) return launch_persist3(p, s, first, n, resid_base);
    const bool narrow = p->narrow_chunk();
    SlabArgs a = slab_args(p, parity0, nullptr);
    const int64_t T = wave_tiles(p, &a.tiles_c);
    if (T == 0) return HRT_OK;
    if (p->pgrid == 0 || p->ptiles != T || p->pkey != T * 4 + (p->nonneg ? 1 : 0)) {
        HRT_CUDA(cudaStreamSynchronize(s));  // counters reset: nothing may be in flight
        rc = build_wave(p, T);
        if (rc) return rc;
    }
    HRT_CUDA(cudaMemsetAsync(p->d_pticket, 0, sizeof(unsigned long long), s));
    WaveArgs wa{};
    wa.s = a;
    wa.s.timeout_ns = p->persist_timeout_ns;
    wa.s.err = p->d_err;
    wa.nbr = p->d_pnbr;
    wa.done = p->d_pdone;
    wa.ticket = p->d_pticket;
    wa.base = p->pbase;
    wa.nsteps = (int)n;
    wa.parity0 = parity0;
    wa.ntiles = T;
    wa.resid = resid_base ? resid_base + first : nullptr;
    if (p->wave_ipc) {
        wa.rnbr = p->d_rnbr;
        wa.rpeer = p->d_rpeer;
        wa.peer_done = p->d_peer_done;
    }
    const bool guard = !p->nonneg, res = resid_base != nullptr;
    void* fn;
    int threads;
#define WK(G, R, CW) (void*)slab_wave_kernel<G, R, CW>
    if (narrow) {
        fn = guard ? (res ? WK(true, true, 2) : WK(true, false, 2))
                   : (res ? WK(false, true, 2) : WK(false, false, 2));
        threads = 96;
    } else {
        fn = guard ? (res ? WK(true, true, 4) : WK(true, false, 4))
                   : (res ? WK(false, true, 4) : WK(false, false, 4));
        threads = 160;
    }
#undef WK
    const unsigned grid = (unsigned)std::min<int64_t>(p->pgrid, T);
    void* args[] = {&wa};
    HRT_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3((unsigned)threads), args, 0, s));
    p->pbase += (unsigned)n;
    return HRT_OK;
}

static int do_step(Plan* p, cudaStream_t s, int64_t step, unsigned long long* resid_base) {
    const int parity = (int)(step & 1);
    unsigned long long* slot = resid_base ? resid_base + step : nullptr;
    // persistent mode: a single step is a one-step wavefront launch, so the
    // tile counters (shared with neighbour ranks) stay the only protocol
    if (p->persist_on()) return launch_persist(p, s, step, 1, resid_base);
    if (p->ipc_on()) {
        // one launch, edge tiles first: they wait for / signal the
        // neighbour processes and push over NVLink; no NCCL in the step
        int rc = prime_ghosts(p, s, parity);
        if (rc) return rc;
        if (p->split_rows != p->rows) {
            rc = build_split(p);
            if (rc) return rc;
        }
        rc = launch_update(p, s, parity, slot, 3);
        if (rc) return rc;
        ++p->gstep;
        return HRT_OK;
    }
    if (p->split_on()) {
        // edge tiles (they push into the NCCL staging) -> fork: exchange +
        // unpack on the side stream || inner tiles on the main stream -> join
        int rc = prime_ghosts(p, s, parity);
        if (rc) return rc;
        if (p->split_rows != p->rows) {
            rc = build_split(p);
            if (rc) return rc;
        }
        rc = launch_update(p, s, parity, slot, 1);
        if (rc) return rc;
        HRT_CUDA(cudaEventRecord(p->ev_fork, s));
        HRT_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
        rc = launch_remote(p, p->side, parity ^ 1);
        if (rc) return rc;
        HRT_CUDA(cudaEventRecord(p->ev_join, p->side));
        rc = launch_update(p, s, parity, slot, 2);
        if (rc) return rc;
        HRT_CUDA(cudaStreamWaitEvent(s, p->ev_join, 0));
        return HRT_OK;
    }
    if (p->any_push()) {
        int rc = prime_ghosts(p, s, parity);
        if (rc) return rc;
        rc = launch_update(p, s, parity, slot);
        if (rc) return rc;
        return launch_remote(p, s, parity ^ 1);
    }
    int rc = launch_halo(p, s, parity);
    if (rc) return rc;
    return launch_update(p, s, parity, slot);
}

extern "C" {

int hrt_jacobi_plan_create(int gpu, const hrt_chunk_layout_t* layout, int nchunks,
                           const uint64_t* bufs, const hrt_halo_seg_t* segs, int nsegs,
                           void** plan) {
    HRT_CHECK_ARG(layout && plan && (nchunks == 0 || bufs) && (nsegs == 0 || segs),
                  "null plan argument");
    HRT_CHECK_ARG(layout->ndim == 2 || layout->ndim == 3, "layout.ndim must be 2 or 3");
    if (layout->ndim == 2) {
        HRT_CHECK_ARG(layout->stride[1] == 1, "slab layout needs unit y stride");
        HRT_CHECK_ARG(layout->stride[0] % 2 == 0 && (layout->origin + 1) % 2 == 0,
                      "slab layout: interior rows must start 16-byte aligned");
        for (int c = 0; c < nchunks; ++c)
            for (int b = 0; b < 2; ++b)
                HRT_CHECK_ARG(bufs[2 * c + b] % 16 == 0, "chunk buffers must be 16-byte aligned");
    } else {
        HRT_CHECK_ARG(layout->stride[2] == 1, "volume layout needs unit z stride");
    }
    int rc = use_device(gpu);
    if (rc) return rc;
    Plan* p = new Plan();
    p->gpu = gpu;
    p->L = *layout;
    p->nchunks = nchunks;
    p->h_chunks.resize(nchunks);
    for (int c = 0; c < nchunks; ++c) {
        p->h_chunks[c].b[0] = reinterpret_cast<double*>(bufs[2 * c]);
        p->h_chunks[c].b[1] = reinterpret_cast<double*>(bufs[2 * c + 1]);
    }
    cudaError_t e = cudaSuccess;
    if (nchunks) {
        e = cudaMalloc(&p->d_chunks, sizeof(ChunkBufs) * nchunks);
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_chunks, p->h_chunks.data(), sizeof(ChunkBufs) * nchunks,
                           cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && nsegs) {
        e = cudaMalloc(&p->d_segs, sizeof(hrt_halo_seg_t) * nsegs);
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_segs, segs, sizeof(hrt_halo_seg_t) * nsegs, cudaMemcpyHostToDevice);
        p->nsegs = nsegs;
        p->seg_blocks = blocks_for(segs, nsegs);
    }
    if (e != cudaSuccess) {
        cudaFree(p->d_chunks);
        cudaFree(p->d_segs);
        delete p;
        return cuda_fail(e, "plan tables");
    }
    // Ring kernels are smem-limited (4-5 CTAs/SM): ask for the max shared
    // carveout explicitly so graph-launched nodes get the same residency as
    // stream launches (measured: a graph replay of the push kernel ran 40 %
    // slower without this).
    set_carveouts();
    // rows (slab) / planes (volume) per CTA tile.  Volumes: 64 planes halves
    // the x-halo planes re-read from DRAM (x-adjacent tiles run ~tiles_j *
    // tiles_k tiles apart, after L2 has dropped them): paper3d 344.6 -> 352
    // GLUPS; 128 planes leaves too few tiles (319)
    p->rows = 64;
    if (const char* e = getenv("HRT_NARROW")) p->narrow_ok = e[0] != '0';
    if (const char* e = getenv("HRT_FUSE2")) p->fuse2 = e[0] == '0' ? 0 : (e[0] == '2' ? 2 : 1);

    *plan = p;
    return HRT_OK;
}

// chunk origins (3 int64 per chunk, plan order) inside the process's field
int hrt_jacobi_plan_set_offsets(void* plan, const int64_t* offs3) {
    HRT_CHECK_ARG(plan && offs3, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    cudaFree(p->d_offs);
    p->d_offs = nullptr;
    if (p->nchunks == 0) return HRT_OK;
    HRT_CUDA(cudaMalloc(&p->d_offs, sizeof(int64_t) * 3 * p->nchunks));
    HRT_CUDA(cudaMemcpy(p->d_offs, offs3, sizeof(int64_t) * 3 * p->nchunks, cudaMemcpyHostToDevice));
    return HRT_OK;
}

// field (FX x FY x FZ, contiguous float64, any GPU reachable from this one)
// -> buffer `parity` of every chunk (to_chunks=1), or back (0)
int hrt_jacobi_plan_field_copy(void* plan, void* stream, double* field, int64_t FY, int64_t FZ,
                               int parity, int to_chunks) {
    hrt::NvtxRange nvtx_("hrt_jacobi_plan_field_copy");
    HRT_CHECK_ARG(plan && stream && field, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG(p->d_offs || p->nchunks == 0, "set the chunk offsets first");
    if (p->nchunks == 0) return HRT_OK;
    int rc = use_device(p->gpu);
    if (rc) return rc;
    const hrt_chunk_layout_t& L = p->L;
    const int64_t rows = L.ndim == 2 ? L.ext[0] : L.ext[0] * L.ext[1];
    const int64_t grid = rows * p->nchunks;
    cudaStream_t cs = as_stream(stream)->s;
    unsigned long long* range = nullptr;
    if (to_chunks && L.ndim == 3) {
        if (!p->d_range) HRT_CUDA(cudaMalloc(&p->d_range, 2 * sizeof(unsigned long long)));
        HRT_CUDA(cudaMemsetAsync(p->d_range, 0, 2 * sizeof(unsigned long long), cs));
        range = p->d_range;
        p->since_scan = 0;
    }
    field_copy_kernel<<<(unsigned)grid, 256, 0, cs>>>(
        p->d_chunks, p->d_offs, parity & 1, L.ndim, L.ext[0], L.ext[1], L.ext[2], L.stride[0],
        L.stride[1], L.origin, field, FY, FZ, to_chunks, range);
    HRT_CUDA(cudaGetLastError());
    if (to_chunks) p->ghosts_ready = false;  // new interiors: ghost planes are stale
    return HRT_OK;
}

// Enable the fused halo push (slab variant 2): per chunk (plan order) the
// ghost-plane targets of its four faces for both parities; null = domain face.
int hrt_jacobi_plan_set_push(void* plan, const hrt_push_t* table) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    cudaFree(p->d_push);
    p->d_push = nullptr;
    p->ghosts_ready = false;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    if (!table || p->nchunks == 0) return HRT_OK;
    HRT_CUDA(cudaMalloc(&p->d_push, sizeof(ChunkPush) * p->nchunks));
    HRT_CUDA(cudaMemcpy(p->d_push, table, sizeof(ChunkPush) * p->nchunks, cudaMemcpyHostToDevice));
    return HRT_OK;
}

int hrt_jacobi_plan_set_sides(void* plan, const hrt_side_t* table) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    HRT_CHECK_ARG(!table || (p->L.ndim == 2 && p->L.ext[1] % 2 == 0),
                  "side arrays need a slab layout with an even chunk width");
    cudaFree(p->d_sides);
    p->d_sides = nullptr;
    p->ghosts_ready = false;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    if (!table || p->nchunks == 0) return HRT_OK;
    HRT_CUDA(cudaMalloc(&p->d_sides, sizeof(ChunkSide) * p->nchunks));
    HRT_CUDA(cudaMemcpy(p->d_sides, table, sizeof(ChunkSide) * p->nchunks,
                        cudaMemcpyHostToDevice));
    return HRT_OK;
}

int hrt_jacobi_plan_set_vpush(void* plan, const hrt_vpush_t* table) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    HRT_CHECK_ARG(!table || p->L.ndim == 3, "vpush is for volume plans");
    cudaFree(p->d_vpush);
    p->d_vpush = nullptr;
    p->ghosts_ready = false;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    p->h_vpush.clear();
    p->pgrid3 = 0;
    if (!table || p->nchunks == 0) return HRT_OK;
    p->h_vpush.assign(table, table + p->nchunks);
    HRT_CUDA(cudaMalloc(&p->d_vpush, sizeof(VolPush) * p->nchunks));
    HRT_CUDA(cudaMemcpy(p->d_vpush, table, sizeof(VolPush) * p->nchunks, cudaMemcpyHostToDevice));
    return HRT_OK;
}

// Split schedule for push mode with remote faces: remote_mask[c] has bit f
// set when face f of chunk c (plan order) crosses a process boundary; tiles
// touching such faces run first, the NCCL exchange overlaps the rest.
// NULL disables.
int hrt_jacobi_plan_set_split(void* plan, const int32_t* remote_mask) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    if (!remote_mask) {
        if (p->side) cudaStreamDestroy(p->side);
        if (p->ev_fork) cudaEventDestroy(p->ev_fork);
        if (p->ev_join) cudaEventDestroy(p->ev_join);
        p->side = nullptr;
        p->ev_fork = p->ev_join = nullptr;
        return HRT_OK;
    }
    p->remote_mask.assign(remote_mask, remote_mask + p->nchunks);
    if (!p->side) {
        int lo = 0, hi = 0;
        HRT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        HRT_CUDA(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, hi));
        HRT_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
        HRT_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    }
    return build_split(p);
}

// IPC push mode for cross-process faces (the push table's remote entries
// must point into the neighbours' IPC-mapped ghost planes).  remote_mask as
// for set_split; arrived: this process's n_nbr flag slots (device, zeroed,
// IPC-exported so neighbours can publish into them); remote_slots: host array
// of the n_nbr device addresses of our slot in each neighbour's flags.
int hrt_jacobi_plan_set_ipc(void* plan, const int32_t* remote_mask, uint64_t* arrived, int n_nbr,
                            const uint64_t* remote_slots, uint64_t timeout_ns) {
    HRT_CHECK_ARG(plan && remote_mask && arrived && remote_slots && n_nbr > 0, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    p->remote_mask.assign(remote_mask, remote_mask + p->nchunks);
    rc = build_split(p);
    if (rc) return rc;
    cudaFree(p->d_remote_slots);
    p->d_remote_slots = nullptr;
    HRT_CUDA(cudaMalloc(&p->d_remote_slots, sizeof(uint64_t) * n_nbr));
    HRT_CUDA(cudaMemcpy(p->d_remote_slots, remote_slots, sizeof(uint64_t) * n_nbr,
                        cudaMemcpyHostToDevice));
    if (!p->d_edge_done) {
        HRT_CUDA(cudaMalloc(&p->d_edge_done, 2 * sizeof(unsigned int)));
        HRT_CUDA(cudaMalloc(&p->d_err, sizeof(int)));
    }
    HRT_CUDA(cudaMemset(p->d_edge_done, 0, 2 * sizeof(unsigned int)));
    HRT_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
    p->d_arrived = reinterpret_cast<unsigned long long*>(arrived);
    p->n_nbr = n_nbr;
    p->timeout_ns = timeout_ns ? timeout_ns : 30000000000ULL;
    p->ipc = true;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    return HRT_OK;
}

// Synchronises; *err = 1 if an edge tile timed out waiting for a neighbour.
int hrt_jacobi_plan_ipc_error(void* plan, int* err) {
    HRT_CHECK_ARG(plan && err, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    *err = 0;
    if (!p->d_err) return HRT_OK;
    int rc = use_device(p->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaMemcpy(err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    return HRT_OK;
}

// Mark the ghost planes stale (the next step runs the full halo pass first).
int hrt_jacobi_plan_invalidate_ghosts(void* plan) {
    HRT_CHECK_ARG(plan, "null plan");
    reinterpret_cast<Plan*>(plan)->ghosts_ready = false;
    return HRT_OK;
}

int hrt_jacobi_plan_set_rows(void* plan, int64_t rows) {
    HRT_CHECK_ARG(plan && rows > 0, "bad rows");
    Plan* p = reinterpret_cast<Plan*>(plan);
    p->rows = rows;
    p->rows_explicit = true;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    return HRT_OK;
}

int hrt_jacobi_plan_set_variant(void* plan, int variant) {
    HRT_CHECK_ARG(plan && variant >= 0 && variant <= 3, "variant must be 0, 1, 2 or 3");
    Plan* p = reinterpret_cast<Plan*>(plan);
    p->variant = variant;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    return HRT_OK;
}

// The caller guarantees every field value is finite and >= 0 (true for the
// reference's problem and preserved by the update), which makes the slab
// kernel's division range check dead code.
int hrt_jacobi_plan_set_nonneg(void* plan, int nonneg) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    p->nonneg = nonneg != 0;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    return HRT_OK;
}

// Persistent dataflow mode (slab push mode, one plan, no cross-process
// faces): nbr4 = per chunk (plan order) the plan-local index of its north,
// south, west, east neighbour or -1.  Runs of steps then execute as one
// cooperative launch of slab_wave_kernel.  NULL disables.
// Two-step passes across processes: per chunk and face (N, S, W, E) the
// neighbour chunk's two buffers and the base of its rank's tile counters as
// mapped here (CUDA IPC; 0 = not another process's) and its index in that
// rank's plan.  Only row faces qualify (a chunk facing another process
// north/south must have no west/east neighbours, so no diagonal chunk lives
// in a third place); otherwise the plan keeps one step per pass.
int hrt_jacobi_plan_set_wave2_remote(void* plan, const uint64_t* bufs8, const uint64_t* cnt4,
                                     const int32_t* idx4) {
    HRT_CHECK_ARG(plan && bufs8 && cnt4 && idx4, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG((int64_t)p->nbr.size() == 4 * (int64_t)p->nchunks && p->L.ndim == 2,
                  "set the slab plan persistent first");
    p->r9.clear();
    cudaFree(p->d_n9);
    p->d_n9 = nullptr;
    for (int c = 0; c < p->nchunks; ++c) {
        const uint64_t* k = cnt4 + 4 * (size_t)c;
        if (k[2] || k[3]) return HRT_OK;  // column faces: use hrt_jacobi_plan_set_wave2_nbr9
        if ((k[0] || k[1]) && (p->nbr[4 * (size_t)c + 2] >= 0 || p->nbr[4 * (size_t)c + 3] >= 0))
            return HRT_OK;  // diagonal chunks on another device: likewise
    }
    // row faces only: the N / S positions from the table, the rest local
    auto at = [&](int c, int f) { return c < 0 ? -1 : p->nbr[4 * (size_t)c + f]; };
    p->r9.assign(9 * (size_t)p->nchunks, Plan::R9{0, -1, 0, {0, 0}});
    for (int c = 0; c < p->nchunks; ++c) {
        const int n = at(c, 0), so = at(c, 1);
        const int idx[9] = {at(n, 2), n, at(n, 3), at(c, 2), c, at(c, 3),
                            at(so, 2), so, at(so, 3)};
        for (int e = 0; e < 9; ++e)
            if (idx[e] >= 0) p->r9[9 * (size_t)c + e] = Plan::R9{1, idx[e], 0, {0, 0}};
        const int pos[2] = {1, 7};
        for (int f = 0; f < 2; ++f) {
            const size_t k = 4 * (size_t)c + f;
            if (!cnt4[k]) continue;
            p->r9[9 * (size_t)c + pos[f]] =
                Plan::R9{2, idx4[k], cnt4[k], {bufs8[2 * k], bufs8[2 * k + 1]}};
        }
    }
    return HRT_OK;
}

int hrt_jacobi_plan_set_wave2_nbr9(void* plan, const int32_t* kind9, const int32_t* idx9,
                                   const uint64_t* cnt9, const uint64_t* bufs18) {
    HRT_CHECK_ARG(plan && kind9 && idx9 && cnt9 && bufs18, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG((int64_t)p->nbr.size() == 4 * (int64_t)p->nchunks && p->L.ndim == 2,
                  "set the slab plan persistent first");
    int rc = use_device(p->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaDeviceSynchronize());  // no launch reads the old table
    std::vector<Plan::R9> t(9 * (size_t)p->nchunks);
    for (int c = 0; c < p->nchunks; ++c)
        for (int e = 0; e < 9; ++e) {
            const size_t k = 9 * (size_t)c + e;
            Plan::R9& r = t[k];
            r.kind = kind9[k];
            r.idx = idx9[k];
            r.cnt = cnt9[k];
            r.b[0] = bufs18[2 * k];
            r.b[1] = bufs18[2 * k + 1];
            HRT_CHECK_ARG(r.kind >= 0 && r.kind <= 2, "bad neighbour kind");
            HRT_CHECK_ARG(r.kind != 1 || (r.idx >= 0 && r.idx < p->nchunks), "bad local index");
            HRT_CHECK_ARG(r.kind != 2 || (r.idx >= 0 && r.cnt && r.b[0] && r.b[1]),
                          "remote neighbour without buffers or counters");
            HRT_CHECK_ARG(e != 4 || (r.kind == 1 && r.idx == c), "position 4 is the chunk itself");
        }
    // a corner exists exactly when both faces next to it do (regular grid)
    for (int c = 0; c < p->nchunks; ++c) {
        auto has = [&](int e) { return t[9 * (size_t)c + e].kind != 0; };
        const int corner[4][3] = {{0, 1, 3}, {2, 1, 5}, {6, 7, 3}, {8, 7, 5}};
        for (const auto& q : corner)
            HRT_CHECK_ARG(has(q[0]) == (has(q[1]) && has(q[2])), "inconsistent 3x3 neighbourhood");
    }
    p->r9 = std::move(t);
    cudaFree(p->d_n9);
    p->d_n9 = nullptr;
    return HRT_OK;
}

int hrt_jacobi_plan_set_persistent(void* plan, const int32_t* nbr4, uint64_t timeout_ns) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    if (!nbr4) {
        p->persist = false;
        return HRT_OK;
    }
    const int nf = 2 * p->L.ndim;  // faces per chunk: 4 (slab) or 6 (volume)
    for (int i = 0; i < nf * p->nchunks; ++i)
        HRT_CHECK_ARG(nbr4[i] >= -1 && nbr4[i] < p->nchunks, "neighbour index out of range");
    int coop = 0;
    HRT_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, p->gpu));
    if (!coop) {
        set_error("persistent mode needs cooperative launch support");
        return HRT_E_UNSUPPORTED;
    }
    HRT_CUDA(cudaDeviceSynchronize());  // no launch of the old build in flight
    p->nbr.assign(nbr4, nbr4 + nf * p->nchunks);
    p->v2dirty = true;
    cudaFree(p->d_pnbr);
    p->d_pnbr = nullptr;
    // two-step passes run best with 256-row tiles (rim rows 4/256 of the
    // reads, fewer tile hand-offs: cfg2 591 -> 620 GLUPS); every rank of a
    // decomposition derives the same tiling from the same layout
    if (!p->rows_explicit && p->L.ndim == 2 && p->fuse2) {
        // the tallest tiles (256, 64, 32 or 16 rows) that still leave at
        // least one tile per resident CTA of the two-step kernel; 16-row
        // tiles when none does (small problems live in L2 and are bound by
        // parallelism: 1024^2 in 4x4 chunks 36 -> 110 GLUPS, 2048^2 in 8x8
        // 130 -> 315, 4096^2 in 8x8 590 -> 596; 8192^2 and up keep 256)
        const int64_t ex = p->L.ext[0];
        const int64_t w = p->narrow_chunk() ? 256 : T4_COLS;
        const int64_t tc = (p->L.ext[1] + w - 1) / w;
        const int64_t slots = fuse2_slots(p);
        int64_t pick = 0;
        for (int64_t R : {256, 64, 32, 16}) {
            if (ex % R == 1) continue;  // a 1-row last tile (two-step tiles need 2)
            if (p->tn() * ((ex + R - 1) / R) * tc >= slots) {
                pick = R;
                break;
            }
        }
        if (!pick)
            for (int64_t R : {16, 32, 64})
                if (ex % R != 1) {
                    pick = R;
                    break;
                }
        p->rows = pick ? pick : 64;
        if (p->graph) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
    }
    cudaFree(p->d_n9);
    p->d_n9 = nullptr;
    p->persist = true;
    p->pgrid = 0;  // rebuilt at the next launch
    if (timeout_ns) p->persist_timeout_ns = timeout_ns;
    return HRT_OK;
}

// Synchronises `plan`'s GPU; *err: 0 ok, 1 an IPC edge tile timed out, 2 a
// persistent-kernel dependency wait timed out (the result is void).
int hrt_jacobi_plan_error(void* plan, int* err) {
    HRT_CHECK_ARG(plan && err, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    *err = 0;
    if (!p->d_err) return HRT_OK;
    int rc = use_device(p->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaMemcpy(err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    return HRT_OK;
}

// The plan's wavefront tile counters (allocated now if needed) for export to
// neighbour ranks over CUDA IPC; *ntiles = their count.
// *on = 1 when persistent runs of >= 4 steps use two-step passes
// (slab_wave2_kernel) on this plan.
int hrt_jacobi_plan_two_step(void* plan, int* on) {
    HRT_CHECK_ARG(plan && on, "null argument");
    const Plan* p = reinterpret_cast<Plan*>(plan);
    *on = pass_steps_of(p) == 2 ? 1 : 0;  // slab or volume two-step passes
    return HRT_OK;
}

int hrt_jacobi_plan_set_tiling_chunks(void* plan, int64_t n) {
    HRT_CHECK_ARG(plan && n >= 0, "bad argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG(!p->persist, "set the tiling chunk count before persistent mode");
    p->tiling_chunks = n;
    return HRT_OK;
}

int hrt_jacobi_plan_set_fuse2(void* plan, int mode) {
    HRT_CHECK_ARG(plan && mode >= 0 && mode <= 2, "bad argument");
    reinterpret_cast<Plan*>(plan)->fuse2 = mode;
    return HRT_OK;
}

int hrt_jacobi_plan_tiling(void* plan, int64_t* rows, int64_t* tiles_per_chunk, int* two_step) {
    HRT_CHECK_ARG(plan && rows && tiles_per_chunk && two_step, "null argument");
    const Plan* p = reinterpret_cast<Plan*>(plan);
    *rows = p->rows;
    *tiles_per_chunk = wave_tiles(p) / std::max(1, p->nchunks);
    *two_step = pass_steps_of(p);
    return HRT_OK;
}

int hrt_jacobi_plan_vw2_counters(void* plan, uint64_t* ptr, int64_t* ntiles) {
    HRT_CHECK_ARG(plan && ptr && ntiles, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG(p->L.ndim == 3, "volume plans only");
    int rc = use_device(p->gpu);
    if (rc) return rc;
    rc = ensure_vw2_counters(p);
    if (rc) return rc;
    *ptr = reinterpret_cast<uint64_t>(p->d_v2done);
    *ntiles = p->v2_tiles;
    return HRT_OK;
}

int hrt_jacobi_plan_set_vw2_remote(void* plan, const uint64_t* bufs4, const uint64_t* cnt2,
                                   const int32_t* idx2) {
    HRT_CHECK_ARG(plan && bufs4 && cnt2 && idx2, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG(p->L.ndim == 3, "volume plans only");
    int rc = use_device(p->gpu);
    if (rc) return rc;
    HRT_CUDA(cudaDeviceSynchronize());  // no launch reads the old table
    const int64_t per_chunk = vw2_tiles(p) / std::max(1, p->nchunks);
    p->v2rbuf.assign(bufs4, bufs4 + 4 * (size_t)p->nchunks);
    p->v2rcnt.assign(2 * (size_t)p->nchunks, 0);
    for (size_t k = 0; k < p->v2rcnt.size(); ++k)
        if (cnt2[k]) {
            HRT_CHECK_ARG(idx2[k] >= 0, "remote chunk index missing");
            p->v2rcnt[k] = cnt2[k] + sizeof(unsigned int) * (uint64_t)(idx2[k] * per_chunk);
        }
    p->v2dirty = true;
    return HRT_OK;
}

int hrt_jacobi_plan_range(void* plan, uint64_t* ptr) {
    HRT_CHECK_ARG(plan && ptr, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    *ptr = reinterpret_cast<uint64_t>(p->d_range);
    return HRT_OK;
}

int hrt_jacobi_plan_wave_counters(void* plan, uint64_t* ptr, int64_t* ntiles) {
    HRT_CHECK_ARG(plan && ptr && ntiles, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG(p->persist, "enable persistent mode first");
    int rc = use_device(p->gpu);
    if (rc) return rc;
    const int64_t T = wave_tiles(p);
    if (!p->d_pdone || p->ptiles != T) {
        rc = build_wave(p, T);
        if (rc) return rc;
    }
    *ptr = reinterpret_cast<uint64_t>(p->d_pdone);
    *ntiles = T;
    return HRT_OK;
}

// Cross-process wavefront: for each chunk (plan order) and face, the peer
// slot (or -1) and the neighbour chunk's index in that peer's plan;
// peer_done[slot] = the peer's tile counters mapped into this process.
// Every rank must use the same layout, rows and chunk order per rank.
int hrt_jacobi_plan_set_wave_ipc(void* plan, const int32_t* rpeer4, const int32_t* rnbr4,
                                 const uint64_t* peer_done, int n_peers, uint64_t timeout_ns) {
    HRT_CHECK_ARG(plan && rpeer4 && rnbr4 && peer_done && n_peers > 0, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    HRT_CHECK_ARG(p->persist && p->d_pdone, "export the wave counters first");
    int rc = use_device(p->gpu);
    if (rc) return rc;
    const int nf = 2 * p->L.ndim;
    for (int i = 0; i < nf * p->nchunks; ++i)
        HRT_CHECK_ARG(rpeer4[i] >= -1 && rpeer4[i] < n_peers, "peer slot out of range");
    cudaFree(p->d_rnbr);
    cudaFree(p->d_rpeer);
    cudaFree(p->d_peer_done);
    const size_t n4 = sizeof(int) * nf * (size_t)std::max(1, p->nchunks);
    HRT_CUDA(cudaMalloc(&p->d_rnbr, n4));
    HRT_CUDA(cudaMalloc(&p->d_rpeer, n4));
    HRT_CUDA(cudaMalloc(&p->d_peer_done, sizeof(void*) * n_peers));
    HRT_CUDA(cudaMemcpy(p->d_rnbr, rnbr4, n4, cudaMemcpyHostToDevice));
    HRT_CUDA(cudaMemcpy(p->d_rpeer, rpeer4, n4, cudaMemcpyHostToDevice));
    HRT_CUDA(cudaMemcpy(p->d_peer_done, peer_done, sizeof(void*) * n_peers,
                        cudaMemcpyHostToDevice));
    p->wave_ipc = true;
    if (timeout_ns) p->persist_timeout_ns = timeout_ns;
    return HRT_OK;
}

int hrt_jacobi_plan_set_remote(void* plan, void* comm, const hrt_remote_seg_t* remote,
                               int nremote, const hrt_halo_seg_t* post, int npost) {
    HRT_CHECK_ARG(plan, "null plan");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    p->comm = comm;
    p->remote.assign(remote, remote + nremote);
    cudaFree(p->d_post);
    p->d_post = nullptr;
    p->npost = 0;
    if (npost) {
        HRT_CUDA(cudaMalloc(&p->d_post, sizeof(hrt_halo_seg_t) * npost));
        HRT_CUDA(cudaMemcpy(p->d_post, post, sizeof(hrt_halo_seg_t) * npost,
                            cudaMemcpyHostToDevice));
        p->npost = npost;
        p->post_blocks = blocks_for(post, npost);
    }
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
    return HRT_OK;
}

int hrt_jacobi_plan_step(void* plan, void* stream, int64_t step, uint64_t* resid) {
    HRT_CHECK_ARG(plan && stream, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    p->count_steps(1);
    return do_step(p, as_stream(stream)->s, step, reinterpret_cast<unsigned long long*>(resid));
}

int hrt_jacobi_plan_update(void* plan, void* stream, int parity, uint64_t* resid_slot) {
    HRT_CHECK_ARG(plan && stream, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    return launch_update(p, as_stream(stream)->s, parity & 1,
                         reinterpret_cast<unsigned long long*>(resid_slot));
}

int hrt_jacobi_plan_halo(void* plan, void* stream, int parity) {
    HRT_CHECK_ARG(plan && stream, "null argument");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    return launch_halo(p, as_stream(stream)->s, parity & 1);
}

// Run steps [first, first+n).  mode 0: direct launches; mode 1: replay a
// captured two-step CUDA graph (the residual slot advances with the step, so
// with a residual the graph is re-instantiated per pair — use mode 0 then).
int hrt_jacobi_plan_run(void* plan, void* stream, int64_t first, int64_t n, uint64_t* resid,
                        int mode) {
    hrt::NvtxRange nvtx_("hrt_jacobi_plan_run");
    HRT_CHECK_ARG(plan && stream && n >= 0, "bad run arguments");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream)->s;
    unsigned long long* r = reinterpret_cast<unsigned long long*>(resid);
    p->count_steps(n);
    if (p->persist_on()) return launch_persist(p, s, first, n, r);
    // IPC step tags are per launch; in push mode graph replays measured 40 %
    // slower than direct launches on B200 (cause not yet identified; the
    // max-shared carveout did not change it), so push mode launches directly
    if (mode == 0 || r != nullptr || p->ipc_on() || p->any_push()) {
        for (int64_t k = 0; k < n; ++k) {
            rc = do_step(p, s, first + k, r);
            if (rc) return rc;
        }
        return HRT_OK;
    }
    int64_t k = 0;
    if (first & 1) {  // align to an even step
        rc = do_step(p, s, first, nullptr);
        if (rc) return rc;
        k = 1;
    }
    if (n - k >= 2) {
        rc = prime_ghosts(p, s, 0);  // outside the graph: replays assume current ghosts
        if (rc) return rc;
        if (!p->graph || p->graph_stream != s) {
            if (p->graph) cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
            cudaGraph_t g;
            HRT_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            int rc0 = do_step(p, s, 0, nullptr);
            int rc1 = rc0 ? rc0 : do_step(p, s, 1, nullptr);
            cudaError_t e = cudaStreamEndCapture(s, &g);
            if (rc1) return rc1;
            HRT_CUDA(e);
            e = cudaGraphInstantiate(&p->graph, g, 0);
            cudaGraphDestroy(g);
            HRT_CUDA(e);
            p->graph_stream = s;
        }
        for (; k + 2 <= n; k += 2) HRT_CUDA(cudaGraphLaunch(p->graph, s));
    }
    for (; k < n; ++k) {
        rc = do_step(p, s, first + k, nullptr);
        if (rc) return rc;
    }
    return HRT_OK;
}

// Steps [first, first+n) with CUDA events bracketing every update and halo
// launch on `stream`; returns the summed device durations.  Synchronises.
int hrt_jacobi_plan_run_timed(void* plan, void* stream, int64_t first, int64_t n, uint64_t* resid,
                              double* update_ms, double* halo_ms, double* total_ms) {
    hrt::NvtxRange nvtx_("hrt_jacobi_plan_run_timed");
    HRT_CHECK_ARG(plan && stream && n >= 0, "bad run arguments");
    Plan* p = reinterpret_cast<Plan*>(plan);
    int rc = use_device(p->gpu);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream)->s;
    unsigned long long* r = reinterpret_cast<unsigned long long*>(resid);
    p->count_steps(n);
    // events are cached on the plan: creating thousands per call would leave
    // the GPU idle while the host allocates them
    std::vector<cudaEvent_t>& ev = p->events;
    while ((int64_t)ev.size() < 3 * n + 1) {
        cudaEvent_t x;
        HRT_CUDA(cudaEventCreate(&x));
        ev.push_back(x);
    }
    if (p->persist_on()) {
        // one launch for all n steps: "update" is the launch, "halo" the
        // priming pass (only after an upload)
        HRT_CUDA(cudaEventRecord(ev[0], s));
        rc = prime_ghosts(p, s, (int)(first & 1));
        if (rc) return rc;
        HRT_CUDA(cudaEventRecord(ev[1], s));
        rc = launch_persist(p, s, first, n, r);
        if (rc) return rc;
        HRT_CUDA(cudaEventRecord(ev[2], s));
        HRT_CUDA(cudaStreamSynchronize(s));
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        if (update_ms) *update_ms = b;
        if (halo_ms) *halo_ms = a;
        if (total_ms) *total_ms = n ? a + b : 0.0;
        return HRT_OK;
    }
    HRT_CUDA(cudaEventRecord(ev[0], s));
    const bool push = p->any_push();
    const bool split = p->split_on() || p->ipc_on();
    for (int64_t k = 0; k < n; ++k) {
        const int64_t step = first + k;
        const int parity = (int)(step & 1);
        rc = push ? prime_ghosts(p, s, parity) : launch_halo(p, s, parity);
        if (rc) break;
        HRT_CUDA(cudaEventRecord(ev[3 * k + 1], s));
        if (split) {
            // "update" here spans edge tiles + overlapped exchange + inner tiles
            rc = do_step(p, s, step, r);
            if (rc) break;
            HRT_CUDA(cudaEventRecord(ev[3 * k + 2], s));
            HRT_CUDA(cudaEventRecord(ev[3 * k + 3], s));
            continue;
        }
        rc = launch_update(p, s, parity, r ? r + step : nullptr);
        if (rc) break;
        HRT_CUDA(cudaEventRecord(ev[3 * k + 2], s));
        if (push) {
            rc = launch_remote(p, s, parity ^ 1);
            if (rc) break;
        }
        HRT_CUDA(cudaEventRecord(ev[3 * k + 3], s));
    }
    cudaError_t e = cudaStreamSynchronize(s);
    double up = 0, ha = 0;
    float ms = 0;
    if (!rc && e == cudaSuccess) {
        for (int64_t k = 0; k < n; ++k) {
            cudaEventElapsedTime(&ms, ev[3 * k + 1], ev[3 * k + 2]);
            up += ms;
            cudaEventElapsedTime(&ms, ev[3 * k], ev[3 * k + 1]);  // halo before the update
            ha += ms;
            cudaEventElapsedTime(&ms, ev[3 * k + 2], ev[3 * k + 3]);  // exchange after it
            ha += ms;
        }
        cudaEventElapsedTime(&ms, ev[0], ev[3 * n]);
    }
    if (rc) return rc;
    HRT_CUDA(e);
    if (update_ms) *update_ms = up;
    if (halo_ms) *halo_ms = ha;
    if (total_ms) *total_ms = n ? ms : 0.0;
    return HRT_OK;
}

int hrt_jacobi_plan_destroy(void* plan) {
    if (!plan) return HRT_OK;
    Plan* p = reinterpret_cast<Plan*>(plan);
    use_device(p->gpu);
    if (p->graph) cudaGraphExecDestroy(p->graph);
    for (auto& x : p->events) cudaEventDestroy(x);
    cudaFree(p->d_chunks);
    cudaFree(p->d_segs);
    cudaFree(p->d_post);
    cudaFree(p->d_offs);
    cudaFree(p->d_push);
    cudaFree(p->d_sides);
    cudaFree(p->d_vpush);
    cudaFree(p->d_tiles_edge);
    cudaFree(p->d_tiles_inner);
    cudaFree(p->d_tiles_all);
    cudaFree(p->d_remote_slots);
    cudaFree(p->d_edge_done);
    cudaFree(p->d_err);
    cudaFree(p->d_pnbr);
    cudaFree(p->d_pdone);
    cudaFree(p->d_pticket);
    cudaFree(p->d_rnbr);
    cudaFree(p->d_rpeer);
    cudaFree(p->d_peer_done);
    cudaFree(p->d_n9);
    cudaFree(p->d_ones);
    cudaFree(p->d_v2done);
    cudaFree(p->d_v2nbr);
    cudaFree(p->d_v2chains);
    cudaFree(p->d_v2clist);
    cudaFree(p->d_v2maps);
    cudaFree(p->d_range);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    delete p;
    return HRT_OK;
}

// Standalone plane copies (the reference's halo_pack_f / halo_unpack_f
// bodies, jacobi.py:102-124, and any generic strided copy).
int hrt_halo_copy(void* stream, const hrt_halo_seg_t* segs_dev, int nsegs, int parity,
                  int64_t max_elems) {
    HRT_CHECK_ARG(stream && (nsegs == 0 || segs_dev), "null argument");
    if (nsegs == 0) return HRT_OK;
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    int64_t bps = std::max<int64_t>(
        1, (max_elems + HALO_THREADS * HALO_PER_THREAD - 1) / (HALO_THREADS * HALO_PER_THREAD));
    halo_copy_kernel<<<(unsigned)(nsegs * bps), HALO_THREADS, 0, st->s>>>(segs_dev, parity & 1, bps);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

int hrt_plane_copy(void* stream, const hrt_halo_seg_t* seg) {
    HRT_CHECK_ARG(stream && seg, "null argument");
    const int64_t n = seg->n0 * seg->n1;
    if (n == 0) return HRT_OK;
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    const int64_t blocks = std::min<int64_t>((n + HALO_THREADS - 1) / HALO_THREADS, (int64_t)sm_count() * 8);
    plane_copy_kernel<<<(unsigned)blocks, HALO_THREADS, 0, st->s>>>(*seg);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

// One chunk in the reference's own layout — a dense ghosted (ex+2, ey+2,
// ez+2) float64 C-order object (jacobi.py:383) — updated u -> nxt exactly as
// _update_body (jacobi.py:70-86): 7-point interior update, then the ghost
// shell carried forward.  resid_slot (nullable) receives max|nxt-u|.
int hrt_jacobi_chunk_update(void* stream, const double* u, double* nxt, int64_t ex, int64_t ey,
                            int64_t ez, uint64_t* resid_slot) {
    HRT_CHECK_ARG(stream && u && nxt && ex > 0 && ey > 0 && ez > 0, "bad chunk update arguments");
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    VolArgs a{};
    a.chunks = nullptr;
    a.du = u;
    a.dw = nxt;
    a.parity = 0;
    a.ex = ex;
    a.ey = ey;
    a.ez = ez;
    a.sy = ez + 2;
    a.sx = (ey + 2) * a.sy;
    a.origin = 0;
    a.rows = 16;
    a.flat = ez == 1;
    a.tiles_i = (ex + a.rows - 1) / a.rows;
    a.tiles_j = a.flat ? (ey + VOL_TX * VOL_TY - 1) / (VOL_TX * VOL_TY) : (ey + VOL_TY - 1) / VOL_TY;
    a.tiles_k = a.flat ? 1 : (ez + VOL_TX - 1) / VOL_TX;
    a.resid = reinterpret_cast<unsigned long long*>(resid_slot);
    const int64_t grid = a.tiles_i * a.tiles_j * a.tiles_k;
    volume_update_kernel<<<(unsigned)grid, dim3(VOL_TX, VOL_TY), 0, st->s>>>(a);
    HRT_CUDA(cudaGetLastError());
    const int64_t n = (ex + 2) * (ey + 2) * (ez + 2);
    ghost_shell_copy_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8), 256, 0,
                              st->s>>>(u, nxt, ex, ey, ez, a.sx, a.sy);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

int hrt_jacobi_ghost_fill(void* stream, double* base, const hrt_chunk_layout_t* L, int mask,
                          double value) {
    HRT_CHECK_ARG(stream && base && L, "null argument");
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    const int64_t n = (L->ext[0] + 2) * (L->ext[1] + 2) * (L->ndim == 3 ? L->ext[2] + 2 : 1);
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
    ghost_fill_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st->s>>>(
        base, L->origin, L->ext[0], L->ext[1], L->ext[2], L->stride[0], L->stride[1], L->ndim,
        mask, value);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

// float(np.sum(a)) of n contiguous device doubles, bit-exact with numpy.
// Synchronises `stream`.
int hrt_np_sum(void* stream, const double* a, int64_t n, double* out) {
    HRT_CHECK_ARG(stream && out && (n == 0 || a), "null argument");
    if (n == 0) {
        *out = 0.0;
        return HRT_OK;
    }
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    // top of the tree on the host: subtrees of <= PW_SEG elements are leaves
    std::vector<int64_t> off, len;
    std::vector<std::pair<int64_t, int64_t>> stack{{0, n}};
    while (!stack.empty()) {
        auto [o, m] = stack.back();
        stack.pop_back();
        if (m <= PW_SEG) {
            off.push_back(o);
            len.push_back(m);
        } else {
            int64_t m2 = m / 2;
            m2 -= m2 % 8;
            stack.push_back({o + m2, m - m2});
            stack.push_back({o, m2});
        }
    }
    const size_t ns = off.size();
    int64_t* d_tab = nullptr;
    double* d_out = nullptr;
    HRT_CUDA(cudaMallocAsync(&d_tab, sizeof(int64_t) * 2 * ns, st->s));
    HRT_CUDA(cudaMallocAsync(&d_out, sizeof(double) * ns, st->s));
    std::vector<int64_t> tab(2 * ns);
    std::copy(off.begin(), off.end(), tab.begin());
    std::copy(len.begin(), len.end(), tab.begin() + ns);
    HRT_CUDA(cudaMemcpyAsync(d_tab, tab.data(), sizeof(int64_t) * 2 * ns, cudaMemcpyHostToDevice,
                             st->s));
    pairwise_seg_kernel<<<(unsigned)ns, PW_THREADS, 0, st->s>>>(a, d_tab, d_tab + ns, d_out);
    cudaError_t le = cudaGetLastError();
    std::vector<double> seg(ns);
    HRT_CUDA(cudaMemcpyAsync(seg.data(), d_out, sizeof(double) * ns, cudaMemcpyDeviceToHost, st->s));
    cudaFreeAsync(d_tab, st->s);
    cudaFreeAsync(d_out, st->s);
    HRT_CUDA(cudaStreamSynchronize(st->s));
    HRT_CUDA(le);
    // combine with the same recursion
    size_t next = 0;
    struct Rec {
        static double go(int64_t m, const std::vector<double>& s, size_t& i) {
            if (m <= PW_SEG) return s[i++];
            int64_t m2 = m / 2;
            m2 -= m2 % 8;
            volatile double l = go(m2, s, i);
            volatile double r = go(m - m2, s, i);
            return l + r;
        }
    };
    volatile double total = Rec::go(n, seg, next);
    *out = 0.0 + total;
    return HRT_OK;
}

// dst[i] = dst[i]*7 + src[i] + salt (mod 256): a read-modify-write task body
// for the runtime's randomized serial-equivalence tests (the reference's
// writer_body, test_acceptance.py:310-312, on device)
__global__ void mix_u8_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                              int64_t n, int salt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (uint8_t)(dst[i] * 7u + (src ? src[i] : 0u) + (unsigned)salt);
}

int hrt_mix_u8(void* stream, uint8_t* dst, const uint8_t* src, int64_t n, int salt) {
    HRT_CHECK_ARG(stream && dst && n >= 0, "bad mix arguments");
    if (n == 0) return HRT_OK;
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
    mix_u8_kernel<<<(unsigned)blocks, 256, 0, st->s>>>(dst, src, n, salt);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

// executor witness kernel: spins `ns` nanoseconds and stores its own
// [start, end] %globaltimer interval (one GPU's clock) into slot[0..1]
__global__ void spin_stamp_kernel(unsigned long long* slot, unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
    slot[0] = t0;
    slot[1] = t;
}

int hrt_spin_stamp(void* stream, uint64_t* slot, uint64_t ns) {
    HRT_CHECK_ARG(stream && slot && ns <= 10000000000ull, "bad spin arguments");
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    spin_stamp_kernel<<<1, 1, 0, st->s>>>(reinterpret_cast<unsigned long long*>(slot), ns);
    HRT_CUDA(cudaGetLastError());
    return HRT_OK;
}

int hrt_div6_sweep(void* stream, uint64_t seed, int64_t n, int mode, uint64_t* mismatches,
                   double* first_bad) {
    HRT_CHECK_ARG(stream && mismatches, "null argument");
    Stream* st = as_stream(stream);
    int rc = use_device(st->gpu);
    if (rc) return rc;
    unsigned long long* d_cnt = nullptr;
    double* d_bad = nullptr;
    HRT_CUDA(cudaMallocAsync(&d_cnt, sizeof(unsigned long long), st->s));
    HRT_CUDA(cudaMallocAsync(&d_bad, sizeof(double), st->s));
    HRT_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), st->s));
    HRT_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(double), st->s));
    div6_sweep_kernel<<<sm_count() * 8, 256, 0, st->s>>>(seed, n, mode, d_cnt, d_bad);
    cudaError_t le = cudaGetLastError();
    unsigned long long cnt = 0;
    double bad = 0;
    HRT_CUDA(cudaMemcpyAsync(&cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, st->s));
    HRT_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st->s));
    cudaFreeAsync(d_cnt, st->s);
    cudaFreeAsync(d_bad, st->s);
    HRT_CUDA(cudaStreamSynchronize(st->s));
    HRT_CUDA(le);
    *mismatches = cnt;
    if (first_bad) *first_bad = bad;
    return HRT_OK;
}

}  // extern "C"
