/*
 * hrt_b200.h — C ABI of libhrt_b200.so, the B200 (sm_100a) backend for the
 * Jacobi / halo-exchange / device-message hot path of the reference `hrt`
 * runtime (arXiv 2303.02543, /root/reference/pkg/src/hrt).
 *
 * Plain C types only (pointers, sizes, integers); no torch types.  Every
 * function returns 0 (HRT_OK) on success or a negative HRT_E_* code; the
 * message for the calling thread is in hrt_last_error().  Error codes map
 * onto the reference's exception tree (errors.py:4-65) — see
 * paper_2303_02543_b200/errors.py.
 *
 * The reference has no native ABI: its seams are Python classes.  Each
 * entry point below names the reference interface it replaces.  The ctypes
 * binding a maintainer would add to the reference is shown in
 * INTEGRATION.md; paper_2303_02543_b200/_native.py is this repo's binding.
 */
#ifndef HRT_B200_H
#define HRT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HRT_ABI_VERSION 1
#define HRT_ALIGNMENT 256      /* devices.py:35 ALIGNMENT */
#define HRT_BOUNDARY 1.0       /* bench/jacobi.py:38 BOUNDARY */

/* error codes */
#define HRT_OK 0
#define HRT_E_INVALID (-1)        /* HrtError */
#define HRT_E_OOM (-2)            /* OutOfDeviceMemory   devices.py:122 */
#define HRT_E_DOUBLE_FREE (-3)    /* DoubleFree          devices.py:127 */
#define HRT_E_LOCATION (-4)       /* InvalidLocation     devices.py:423-457 */
#define HRT_E_UNKNOWN_TOKEN (-5)  /* UnknownToken        devices.py:564 */
#define HRT_E_CUDA (-6)           /* failed launch/copy -> FAILED token -> TaskFailed runtime.py:507 */
#define HRT_E_NCCL (-7)           /* transport failure   (TransportClosed / ProtocolError) */
#define HRT_E_UNSUPPORTED (-8)

const char *hrt_last_error(void);
int hrt_version(void);

/* ---- devices (DeviceRegistry.register_device devices.py:364-380) ---- */
int hrt_device_count(int *n);
int hrt_device_info(int gpu, char *name, int name_len, int *sm_count, uint64_t *hbm_bytes,
                    int *cc_major, int *cc_minor);
/* enable NVLink peer access gpu -> peer (lifts devices.py:456-457) */
int hrt_enable_peer_access(int gpu, int peer);
int hrt_device_synchronize(int gpu);
int hrt_pointer_device(const void *ptr, int *gpu);
/* CUDA IPC (same node): export a cudaMalloc base (64-byte handle), map a
 * handle from another process on `gpu` (peer access over NVLink), unmap */
int hrt_ipc_get_handle(const void *base, uint8_t *out64);
int hrt_ipc_open_handle(int gpu, const uint8_t *in64, void **ptr);
int hrt_ipc_close_handle(void *ptr);

/* ---- first-fit free list: FreeListAllocator devices.py:89-154 (host logic) ---- */
int hrt_fl_create(uint64_t capacity, uint64_t alignment, void **fl);
int hrt_fl_alloc(void *fl, uint64_t size, uint64_t *offset, uint64_t *granted);   /* alloc 108-122 */
int hrt_fl_free(void *fl, uint64_t offset, uint64_t *size);                       /* free 124-137 */
int hrt_fl_stats(void *fl, uint64_t *live_bytes, uint64_t *free_bytes, uint64_t *free_blocks);
int hrt_fl_check(void *fl);                                                       /* check 147-154 */
void hrt_fl_destroy(void *fl);

/* ---- device pools: DeviceBackend.attach/region devices.py:299-305 +
 *      DeviceRegistry.pool_alloc/pool_free devices.py:398-404 ---- */
int hrt_pool_create(int gpu, uint64_t capacity, void **pool);
int hrt_pool_alloc(void *pool, uint64_t size, uint64_t *offset, uint64_t *granted, void **dptr);
int hrt_pool_free(void *pool, uint64_t offset);
int hrt_pool_stats(void *pool, uint64_t *live_bytes, uint64_t *free_bytes);
int hrt_pool_base(void *pool, void **base);
int hrt_pool_destroy(void *pool);

/* ---- streams (_Device.compute_streams/h2d/d2h devices.py:322-329) ---- */
int hrt_stream_create(int gpu, int priority, void **stream);
int hrt_stream_wrap(int gpu, void *cuda_stream, void **stream);   /* adopt an external cudaStream_t */
void *hrt_stream_handle(void *stream);                              /* the cudaStream_t */
int hrt_stream_destroy(void *stream, int owned);
int hrt_stream_synchronize(void *stream);

/* ---- completion tokens: CompletionToken devices.py:199-222, poll 560-567 ---- */
int hrt_token_record(void *stream, uint64_t *token);
int hrt_token_query(uint64_t token);              /* 0 pending, 1 complete, 2 failed, <0 error */
int hrt_token_wait(uint64_t token);
int hrt_stream_wait_token(void *stream, uint64_t token);   /* GPU-side dependency edge */
int hrt_token_elapsed_ms(uint64_t start, uint64_t end, float *ms);
int hrt_token_release(uint64_t token);

/* ---- transfers: DeviceRegistry.enqueue_transfer devices.py:446-496,
 *      HostPinnedPool devices.py:167-196 ---- */
int hrt_host_alloc(uint64_t bytes, void **ptr);     /* page-locked */
int hrt_host_free(void *ptr);
int hrt_host_register(void *ptr, uint64_t bytes);
int hrt_host_unregister(void *ptr);
int hrt_copy_async(void *stream, void *dst, const void *src, uint64_t bytes);   /* H2D/D2H/D2D (UVA) */
/* *equal = 1 when n bytes at a and b (device/peer, 16-byte aligned) are
 * identical (ping-pong byte identity, pingpong.py:135-138).  Synchronises.
 * Uses a result word owned by the stream handle: one caller per handle at
 * a time. */
int hrt_bytes_equal(void *stream, const void *a, const void *b, uint64_t bytes, int *equal);
/* SM-driven copy kernel on stream's GPU; dst/src may be peer (NVLink)
 * addresses, 16-byte aligned.  blocks <= 0: automatic. */
int hrt_copy_sm_async(void *stream, void *dst, const void *src, uint64_t bytes, int blocks);
int hrt_copy_peer_async(void *stream, void *dst, int dst_gpu, const void *src, int src_gpu,
                        uint64_t bytes);                                         /* NVLink peer copy */
/* enqueue_transfer in one call (devices.py:446-496): GPU-side waits on the
 * tokens in waits[0..nwait) (retired tokens are skipped), the copy (method
 * 0 copy engine, 1 SM kernel, 2 auto: SM kernel for 16-byte aligned
 * GPU<->GPU copies <= HRT_SM_COPY_MAX bytes, default 64 MiB), then a new
 * completion token behind it.  peer != 0: src and dst are on different GPUs. */
int hrt_copy_ordered(void *stream, void *dst, const void *src, uint64_t bytes, int peer,
                     const uint64_t *waits, int nwait, int method, uint64_t *token);
int hrt_copy2d_async(void *stream, void *dst, uint64_t dpitch, const void *src, uint64_t spitch,
                     uint64_t width, uint64_t height);
int hrt_memset_async(void *stream, void *dst, int value, uint64_t bytes);

/* ---- Jacobi hot path: bench/jacobi.py ---- */

/* Ghosted chunk layout.  Element (i,j,k) of the ghosted (ex+2, ey+2, ez+2)
 * chunk (jacobi.py:383) lives at base + origin + i*stride[0] + j*stride[1]
 * + k*stride[2] (float64 elements).  ndim 2 is the (X,Y,1) slab: no z ghosts
 * are stored, the two z neighbours are the constant BOUNDARY. */
typedef struct hrt_chunk_layout {
    int32_t ndim;
    int32_t pad_;
    int64_t ext[3];
    int64_t stride[3];
    int64_t origin;
    int64_t elems;
} hrt_chunk_layout_t;

/* One face copy (pack+send+unpack fused, jacobi.py:102-124 + 237):
 * dst[o*ds0 + i*ds1] = src[o*ss0 + i*ss1] for o < n0, i < n1, with separate
 * addresses for step parity 0 and 1 (the alternating buffers, jacobi.py:213-217). */
typedef struct hrt_halo_seg {
    uint64_t src[2];
    uint64_t dst[2];
    int64_t n0, n1;
    int64_t ss0, ss1;
    int64_t ds0, ds1;
} hrt_halo_seg_t;

/* One half of a face crossing a process boundary: `count` contiguous
 * float64 at buf[parity] sent to (kind 0) or received from (kind 1) NCCL
 * rank `peer`.  Both ranks list their ops in one canonical global order
 * (destination chunk, face), so NCCL's in-order pairing matches them. */
typedef struct hrt_remote_seg {
    uint64_t buf[2];
    int64_t count;
    int32_t peer;
    int32_t kind;
} hrt_remote_seg_t;

/* Fused halo push, per chunk: where the update kernel stores the chunk's
 * new boundary plane of face f (FACES order north, south, west, east) when
 * it writes buffer parity p — the neighbour's ghost plane (same GPU, or a
 * peer GPU over NVLink), or a packed NCCL staging slot; null for a domain
 * face.  stride[f] = element step along that plane. */
typedef struct hrt_push {
    uint64_t ptr[4][2];
    int64_t stride[4];
} hrt_push_t;

/* Step engine for all chunks of one GPU (replaces the per-chunk task chain
 * of _RankDriver.start_step/_try_finish_step jacobi.py:219-273).
 * bufs: 2*nchunks device addresses (buffer 0, buffer 1 per chunk).
 * segs: same-GPU / peer faces, executed before every update. */
int hrt_jacobi_plan_create(int gpu, const hrt_chunk_layout_t *layout, int nchunks,
                           const uint64_t *bufs, const hrt_halo_seg_t *segs, int nsegs,
                           void **plan);
/* faces that cross ranks: NCCL exchange, then `post` (unpack) copies */
int hrt_jacobi_plan_set_remote(void *plan, void *comm, const hrt_remote_seg_t *remote,
                               int nremote, const hrt_halo_seg_t *post, int npost);
int hrt_jacobi_plan_set_rows(void *plan, int64_t rows);
/* chunk origins (3 int64 per chunk, plan order) inside the process's
 * contiguous field, then one-launch scatter (upload, jacobi.py:382-395) /
 * gather (jacobi.py:425-435) between the field and buffer `parity` */
int hrt_jacobi_plan_set_offsets(void *plan, const int64_t *offs3);
/* enable (table != NULL) / disable the fused halo push for slab variant 2:
 * a step is then one update launch (+ the NCCL exchange of pushed staging);
 * the full halo pass runs only when ghosts are stale (after an upload) */
int hrt_jacobi_plan_set_push(void *plan, const hrt_push_t *table);
/* Contiguous west/east ghost columns ("side arrays", push mode, even chunk
 * width): per chunk, the arrays holding its own west and east ghost column
 * for each buffer parity (element i-1 = row i), or null for a domain face
 * (constant boundary value).  The halo push and the priming pass then
 * target these instead of the strided in-buffer ghost columns, and the
 * update kernel streams only the 16-byte-aligned interior row span.
 * NULL disables. */
typedef struct hrt_side {
    uint64_t w[2];
    uint64_t e[2];
} hrt_side_t;
int hrt_jacobi_plan_set_sides(void *plan, const hrt_side_t *table);
/* Fused halo push for volume (3D) plans: per chunk, face f (-x,+x,-y,+y,
 * -z,+z) and parity of the buffer being written, the address matching this
 * chunk's element offset 0 in the neighbour's ghost plane (the kernel stores
 * boundary cell (i,j,k) at ptr[f][p] + 8*(i*sx + j*sy + k)); 0 for a domain
 * face.  NULL disables. */
typedef struct hrt_vpush {
    uint64_t ptr[6][2];
} hrt_vpush_t;
int hrt_jacobi_plan_set_vpush(void *plan, const hrt_vpush_t *table);
int hrt_jacobi_plan_invalidate_ghosts(void *plan);
/* overlap for cross-process faces (push mode): remote_mask[c] bit f = face f
 * of chunk c crosses a process; tiles touching such faces run first, then
 * the NCCL exchange runs on a side stream while the other tiles compute.
 * NULL disables. */
int hrt_jacobi_plan_set_split(void *plan, const int32_t *remote_mask);
/* fused compute + communication across processes: the push table's remote
 * entries point into the neighbours' IPC-mapped ghost planes; edge tiles
 * (remote_mask as above) wait in-kernel for the neighbours' previous step
 * (flags in `arrived`, written by them over NVLink), push, and the last one
 * publishes the step into each neighbour's slot (remote_slots[k]).  No NCCL
 * in the step; a neighbour silent for timeout_ns sets an error instead of
 * hanging (hrt_jacobi_plan_ipc_error). */
int hrt_jacobi_plan_set_ipc(void *plan, const int32_t *remote_mask, uint64_t *arrived, int n_nbr,
                            const uint64_t *remote_slots, uint64_t timeout_ns);
int hrt_jacobi_plan_ipc_error(void *plan, int *err);
/* Persistent dataflow mode for one-plan slab push runs (replaces the
 * reference's per-step barrier `_try_finish_step`, jacobi.py:241-273, with
 * per-CTA step counters on the device): nbr4[4*c + f] = plan-local index of
 * chunk c's neighbour across face f (N,S,W,E; the reference's FACES order,
 * jacobi.py:41-46) or -1.  NULL disables.  timeout_ns 0 = 10 s per wait. */
int hrt_jacobi_plan_set_persistent(void *plan, const int32_t *nbr4, uint64_t timeout_ns);
/* The plan's wavefront tile counters (device address, for CUDA IPC export
 * to neighbour ranks) and their count. */
int hrt_jacobi_plan_wave_counters(void *plan, uint64_t *ptr, int64_t *ntiles);
/* Volume two-step passes across processes (x-band volumes split between
 * ranks; replaces the per-step halo messages of _RankDriver jacobi.py:
 * 219-273 like the slab wave).  vw2_counters: the plan's per-tile step
 * counters of volume_wave2_kernel (allocated on first use, never moved)
 * for CUDA IPC export.  set_vw2_remote: per chunk and x face (-x, +x) the
 * neighbour process's chunk buffers for parity 0/1 (bufs4, mapped here; 0 =
 * no such face), the base of that process's vw2 counters (cnt2, mapped)
 * and the chunk's index in its plan (idx2).  range: device address of the
 * upload scan (2 x uint64: ~bits of the smallest positive value, bad flag)
 * that ranks max-reduce so every rank picks the division from the global
 * field. */
int hrt_jacobi_plan_vw2_counters(void *plan, uint64_t *ptr, int64_t *ntiles);
int hrt_jacobi_plan_set_vw2_remote(void *plan, const uint64_t *bufs4, const uint64_t *cnt2,
                                   const int32_t *idx2);
int hrt_jacobi_plan_range(void *plan, uint64_t *ptr);
/* Cross-process wavefront (the reference's halo messages between ranks,
 * jacobi.py:237 mp_send, as NVLink pushes + per-tile counters): per chunk and
 * face the peer slot (-1 none) and the neighbour chunk's index in that
 * peer's plan; peer_done = each peer's counters mapped here. */
int hrt_jacobi_plan_set_wave_ipc(void *plan, const int32_t *rpeer4, const int32_t *rnbr4,
                                 const uint64_t *peer_done, int n_peers, uint64_t timeout_ns);
/* Two steps per pass across processes (slab_wave2_kernel reads a 2-cell rim
 * straight from the neighbour's chunk): per chunk and face N,S,W,E the
 * neighbour chunk's two buffers (bufs8, mapped here), the base of its
 * rank's tile counters (cnt4, mapped; 0 = not another process) and its
 * index in that rank's plan.  Only row faces qualify; otherwise a no-op.
 * (Kept for callers with row faces only; hrt_jacobi_plan_set_wave2_nbr9
 * below covers every decomposition and is what the Python layer uses.) */
int hrt_jacobi_plan_set_wave2_remote(void *plan, const uint64_t *bufs8, const uint64_t *cnt4,
                                     const int32_t *idx4);
/* The whole 3 x 3 chunk neighbourhood of every chunk for two-step slab
 * passes whose neighbours (faces or corners) live on other GPUs or in other
 * processes — e.g. column faces between ranks (cfg5's y-bands).  Per chunk
 * (plan order) and position e (row-major NW N NE W C E SW S SE): kind9 0 =
 * none (domain), 1 = this plan's chunk idx9, 2 = another device's chunk
 * idx9 (its index in its own plan) with that plan's tile counters cnt9 and
 * buffers bufs18 (both mapped: peer or CUDA IPC).  A corner must exist
 * exactly when both faces next to it do. */
int hrt_jacobi_plan_set_wave2_nbr9(void *plan, const int32_t *kind9, const int32_t *idx9,
                                   const uint64_t *cnt9, const uint64_t *bufs18);
/* *on = 1 when runs of >= 4 steps use two-step passes: slab_wave2_kernel
 * (slabs) or volume_wave2_kernel (x-band volumes on one GPU). */
int hrt_jacobi_plan_two_step(void *plan, int *on);
/* Chunk count the tiling decisions (tile rows, two-step passes or not) are
 * made for: pass the largest chunk count per GPU of the whole
 * decomposition (every GPU and rank of a run), before persistent mode, so
 * neighbouring GPUs agree on the tiling whose counters they index.
 * 0 = the plan's own chunk count. */
int hrt_jacobi_plan_set_tiling_chunks(void *plan, int64_t n);
/* Two-step passes: 0 off, 1 when the decomposition has at least one tile
 * per resident CTA (default; HRT_FUSE2 overrides at plan creation), 2
 * always.  Multi-GPU runs turn them off on every GPU when not every GPU
 * can run them (a one-step neighbour would read ghosts nobody pushed). */
int hrt_jacobi_plan_set_fuse2(void *plan, int mode);
/* The plan's tiling: rows per tile, tiles per chunk, and the Jacobi steps
 * per fused pass runs of several steps use (0 = one step per pass). */
int hrt_jacobi_plan_tiling(void *plan, int64_t *rows, int64_t *tiles_per_chunk, int *steps_per_pass);
/* Synchronises; *err = 0 ok, 1 IPC edge wait timed out, 2 persistent
 * dependency wait timed out (results void). */
int hrt_jacobi_plan_error(void *plan, int *err);
int hrt_jacobi_plan_field_copy(void *plan, void *stream, double *field, int64_t FY, int64_t FZ,
                               int parity, int to_chunks);
/* slab update kernel: 0 = LDG register march, 1 = TMA bulk-copy ring,
 * 2 = TMA ring with four columns per thread (default) */
int hrt_jacobi_plan_set_variant(void *plan, int variant);
/* caller guarantees a finite, non-negative field bounded by 2^997 (the
 * reference's problem): the slab kernel's six-term sum is then in
 * [2, 2^1000] and the division needs no subnormal/overflow guard */
int hrt_jacobi_plan_set_nonneg(void *plan, int nonneg);
/* one step: halo faces, then the 7-point update of every chunk (_update_body
 * jacobi.py:70-79); resid (nullable, device, uint64 bit patterns of float64)
 * receives max|u'-u| at index `step` via atomicMax (must start zeroed). */
int hrt_jacobi_plan_step(void *plan, void *stream, int64_t step, uint64_t *resid);
int hrt_jacobi_plan_update(void *plan, void *stream, int parity, uint64_t *resid_slot);
int hrt_jacobi_plan_halo(void *plan, void *stream, int parity);
/* steps [first, first+n); mode 0 direct launches, 1 CUDA-graph replay */
int hrt_jacobi_plan_run(void *plan, void *stream, int64_t first, int64_t n, uint64_t *resid,
                        int mode);
/* as run(mode 0) with events around every launch; synchronises */
int hrt_jacobi_plan_run_timed(void *plan, void *stream, int64_t first, int64_t n, uint64_t *resid,
                              double *update_ms, double *halo_ms, double *total_ms);
int hrt_jacobi_plan_destroy(void *plan);

/* standalone plane copies (halo_pack_f / halo_unpack_f bodies); segs on device */
int hrt_halo_copy(void *stream, const hrt_halo_seg_t *segs_dev, int nsegs, int parity,
                  int64_t max_elems);
/* one plane copy described by value (uses src[0]/dst[0]) — a pack or unpack
 * task body (jacobi.py:102-124) */
int hrt_plane_copy(void *stream, const hrt_halo_seg_t *seg);
/* one chunk in the reference's dense ghosted (ex+2,ey+2,ez+2) layout,
 * u -> nxt exactly as _update_body (jacobi.py:70-86): interior update + ghost
 * shell carry; resid_slot (nullable) gets max|nxt-u| via atomicMax */
int hrt_jacobi_chunk_update(void *stream, const double *u, double *nxt, int64_t ex, int64_t ey,
                            int64_t ez, uint64_t *resid_slot);
/* ghost shell of one chunk buffer: faces in `mask` (bit f = FACES[f],
 * jacobi.py:41) get `value` (Dirichlet, jacobi.py:386-393), others 0 */
int hrt_jacobi_ghost_fill(void *stream, double *base, const hrt_chunk_layout_t *layout,
                          int mask, double value);
/* float(np.sum(a)) bit-exact (jacobi.py:436): numpy pairwise summation on
 * the GPU; synchronises the stream */
int hrt_np_sum(void *stream, const double *a, int64_t n, double *out);
/* dst[i] = dst[i]*7 + src[i] + salt (mod 256), src nullable: a
 * read-modify-write task body for runtime ordering tests (the reference's
 * writer_body, test_acceptance.py:310-312) */
int hrt_mix_u8(void *stream, uint8_t *dst, const uint8_t *src, int64_t n, int salt);
/* one-thread kernel that spins `ns` ns and stores its [start, end]
 * %globaltimer interval at slot[0..1] (device memory): the executor's
 * overlap witness (AC-02 analogue, test_acceptance.py:67-96) */
int hrt_spin_stamp(void *stream, uint64_t *slot, uint64_t ns);
/* self-check of the Markstein division used by the update kernel against
 * IEEE division: n hashed samples (mode 0 uniform [0,6), 1 near 1/2/3/6,
 * 2 random finite bit patterns); synchronises */
int hrt_div6_sweep(void *stream, uint64_t seed, int64_t n, int mode, uint64_t *mismatches,
                   double *first_bad);

/* ---- NCCL (cross-process faces; replaces Transport transport.py:40-278
 *      for payloads) ---- */
int hrt_nccl_unique_id(uint8_t *out128);
int hrt_nccl_init(int gpu, int rank, int world, const uint8_t *id128, void **comm);
int hrt_nccl_destroy(void *comm);
int hrt_nccl_exchange(void *comm, void *stream, const hrt_remote_seg_t *segs, int n, int parity);
int hrt_nccl_allreduce_max_u64(void *comm, void *stream, uint64_t *buf, int64_t count);
int hrt_nccl_allreduce_sum_f64(void *comm, void *stream, double *buf, int64_t count);

#ifdef __cplusplus
}
#endif
#endif /* HRT_B200_H */
