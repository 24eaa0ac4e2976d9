"""One process per B200: torch.distributed for the plumbing (rendezvous,
barriers, max-over-ranks timing), libhrt_b200's own NCCL communicator for
the data path (halo faces that cross processes, residual all-reduce), so
the whole step — NCCL send/recv included — stays inside libhrt_b200 and
its CUDA graph.

The reference runs ranks as in-process loopback endpoints or TCP peers
(/root/reference/pkg/src/hrt/transport.py:62-278, comm.py:1053-1082
init_from_env); here ``RANK``/``WORLD_SIZE``/``LOCAL_RANK`` come from
torchrun.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

from . import _native as N
from .devices import DevicePool
from .errors import HrtError
from .jacobi import ChunkGrid, JacobiSolver, _arr, face_plane, opposite, persist_timeout_ns


def env_rank() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_process(backend: str = "nccl"):
    """Initialise torch.distributed from the torchrun environment; returns
    (rank, world, local_rank).  A no-op for world size 1."""
    rank, world, local = env_rank()
    if world > 1:
        import torch
        import torch.distributed as dist

        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def nccl_comm(rank: int, world: int, gpu: int) -> int:
    """libhrt_b200 NCCL communicator; the unique id is broadcast over the
    torch.distributed default group."""
    import torch.distributed as dist

    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        N.call("hrt_nccl_unique_id", uid)
    obj = [uid.raw]
    dist.broadcast_object_list(obj, src=0)
    comm = ctypes.c_void_p()
    N.call("hrt_nccl_init", gpu, rank, world, ctypes.create_string_buffer(obj[0], 128),
           ctypes.byref(comm))
    return comm.value


class DistributedJacobi(JacobiSolver):
    """The chunks of ``grid.per_rank[rank]`` (jacobi.py:325-339) on this
    process's GPU; cross-rank faces by NCCL send/recv inside the step."""

    def __init__(self, grid: ChunkGrid, rank: int, world: int, gpu: int,
                 comm: Optional[int] = None, rows: Optional[int] = None,
                 variant: Optional[int] = None, vpush: Optional[bool] = None):
        if grid.ranks != world:
            raise ValueError("grid.ranks must equal the world size")
        if comm is None and world > 1:
            comm = nccl_comm(rank, world, gpu)
        self.world = world
        self._ipc_maps: list[int] = []
        self._fence_buf = None
        super().__init__(grid, gpus=[gpu], rank=rank, comm=comm, rows=rows, variant=variant)
        self.ipc = False
        # decided from the global decomposition so every rank agrees: IPC
        # push for contiguous (row) faces between processes; strided column
        # faces stay on packed NCCL messages (scattered 8-byte NVLink stores
        # measured 25 % slower than pack + send on 2 B200s)
        cross = [(f, ch.rank, grid.chunks[nb].rank) for ch in grid.chunks
                 for f, nb in ch.neighbors.items() if grid.chunks[nb].rank != ch.rank]
        rows_only = bool(cross) and all(f in (0, 1) for f, _, _ in cross)
        # column faces qualify once they are contiguous (side arrays)
        slab_ok = bool(cross) and self.push and (rows_only or self.side_mode)
        # volumes split along x only: the cross-process wavefront, with
        # two-step passes (volume_wave2_kernel) reading the neighbour rank's
        # planes in place, by default
        xband3 = (self.layout.ndim == 3 and rows_only and grid.grid[1] == 1 and grid.grid[2] == 1
                  and os.environ.get("HRT_FUSE2", "1") != "0")
        if world > 1 and os.environ.get("HRT_IPC", "1") != "0" and (slab_ok or rows_only):
            if self.push:
                self._setup_ipc(gpu)
            elif (self.layout.ndim == 3 and variant != 0
                  and (vpush if vpush is not None
                       else (os.environ.get("HRT_VPUSH", "0") == "1" or xband3))
                  and os.environ.get("HRT_PUSH", "1") != "0"
                  and os.environ.get("HRT_PERSIST", "1") != "0"):
                self._setup_ipc3(gpu)

    def _setup_ipc(self, gpu: int) -> None:
        """Fused compute + communication across processes: map the neighbour
        ranks' chunk arenas with CUDA IPC, point the push table's remote faces
        at their ghost rows or (columns) contiguous side arrays (stores over
        NVLink from the update kernel) and
        give every rank one flag slot per neighbour for the per-step
        handshake.  NCCL remains only for priming ghosts after an upload and
        for the residual all-reduce."""
        import torch.distributed as dist

        L = self.layout
        g = self.used_gpus[0]
        mine = [lin for lin in self.owned if self.placement[lin] == g]
        nbr_ranks = sorted({self.rank_of[nb] for lin in mine
                            for nb in self.grid.chunks[lin].neighbors.values()
                            if nb not in self.placement})
        self._flags = DevicePool(g, 4096)
        N.call("hrt_memset_async", self.streams[g].h, ctypes.c_void_p(self._flags.base), 0, 4096)
        self.streams[g].synchronize()
        h_pool = ctypes.create_string_buffer(64)
        h_flags = ctypes.create_string_buffer(64)
        N.call("hrt_ipc_get_handle", ctypes.c_void_p(self.pools[g].base), h_pool)
        N.call("hrt_ipc_get_handle", ctypes.c_void_p(self._flags.base), h_flags)
        info = (self.rank, h_pool.raw, self.pools[g].base, h_flags.raw,
                {lin: self.bufs[lin] for lin in mine}, nbr_ranks,
                {lin: self.sides.get(lin, {}) for lin in mine})
        every = [None] * self.world
        dist.all_gather_object(every, info)
        mapped_pool, mapped_flags = {}, {}
        for q in nbr_ranks:
            _, hp, base_q, hf = every[q][:4]
            pp, pf = ctypes.c_void_p(), ctypes.c_void_p()
            N.call("hrt_ipc_open_handle", g, ctypes.create_string_buffer(hp, 64), ctypes.byref(pp))
            N.call("hrt_ipc_open_handle", g, ctypes.create_string_buffer(hf, 64), ctypes.byref(pf))
            mapped_pool[q] = (pp.value, base_q)
            mapped_flags[q] = pf.value
            self._ipc_maps += [pp.value, pf.value]
        # ranks holding only corner chunks of this rank's 3 x 3 neighbourhoods
        # (two-step passes read their rims too): arenas mapped, no flags
        diag_ranks = sorted({self.rank_of[q] for lin in mine for q in self.grid.nbhd9(lin)
                             if q is not None and q not in self.placement} - set(nbr_ranks))
        for q in diag_ranks:
            _, hp, base_q = every[q][:3]
            pp = ctypes.c_void_p()
            N.call("hrt_ipc_open_handle", g, ctypes.create_string_buffer(hp, 64), ctypes.byref(pp))
            mapped_pool[q] = (pp.value, base_q)
            self._ipc_maps.append(pp.value)

        def remote_buf(nb: int, p: int) -> int:
            q = self.rank_of[nb]
            mp, base_q = mapped_pool[q]
            return mp + (every[q][4][nb][p] - base_q)

        def remote_ghost(nb: int, face: int, p: int):
            """(address, stride) of remote chunk nb's ghost plane `face`:
            its mapped side array (west/east, side mode) or ghost row."""
            q = self.rank_of[nb]
            side = every[q][6].get(nb, {}).get(face)
            if side is not None:
                mp, base_q = mapped_pool[q]
                return mp + (side[p] - base_q), 1
            addr, _, _, _, s1 = face_plane(L, remote_buf(nb, p), face, ghost=True)
            return addr, s1

        table = (N.Push * max(len(mine), 1))()
        masks = []
        for i, lin in enumerate(mine):
            m = 0
            for f in range(4):
                nb = self.grid.chunks[lin].neighbors.get(f)
                if nb is None:
                    continue
                for p in (0, 1):
                    if nb in self.placement:  # (side array or in-buffer ghost plane)
                        addr, _, _, _, s1 = self._ghost_target(nb, opposite(f), p)
                    else:  # another process: mapped ghost row or side array
                        addr, s1 = remote_ghost(nb, opposite(f), p)
                    table[i].ptr[f][p] = addr
                table[i].stride[f] = s1
                if nb not in self.placement:
                    m |= 1 << f
            masks.append(m)
        N.call("hrt_jacobi_plan_set_push", self.plans[g], ctypes.byref(table))
        slots = [mapped_flags[q] + 8 * every[q][5].index(self.rank) for q in nbr_ranks]
        N.call("hrt_jacobi_plan_set_ipc", self.plans[g], _arr(ctypes.c_int32, masks),
               ctypes.c_void_p(self._flags.base), len(nbr_ranks), _arr(ctypes.c_uint64, slots),
               ctypes.c_uint64(30_000_000_000))
        self.ipc = True
        if os.environ.get("HRT_PERSIST", "1") != "0":
            self._setup_wave_ipc(g, mine, nbr_ranks, remote_buf, diag_ranks)
        dist.barrier()

    def _setup_ipc3(self, gpu: int) -> None:
        """Volumes split along x between processes: map the neighbour ranks'
        chunk arenas, push boundary planes into their ghost planes from the
        update kernel (6-face vpush table) and run the persistent wavefront
        with cross-process tile counters.  NCCL primes ghosts after uploads
        and reduces the residual."""
        import torch.distributed as dist

        g = self.used_gpus[0]
        mine = [lin for lin in self.owned if self.placement[lin] == g]
        nbr_ranks = sorted({self.rank_of[nb] for lin in mine
                            for nb in self.grid.chunks[lin].neighbors.values()
                            if nb not in self.placement})
        h_pool = ctypes.create_string_buffer(64)
        N.call("hrt_ipc_get_handle", ctypes.c_void_p(self.pools[g].base), h_pool)
        every = [None] * self.world
        dist.all_gather_object(every, (h_pool.raw, self.pools[g].base,
                                       {lin: self.bufs[lin] for lin in mine}))
        mapped = {}
        for q in nbr_ranks:
            hp, base_q, _ = every[q]
            pp = ctypes.c_void_p()
            N.call("hrt_ipc_open_handle", g, ctypes.create_string_buffer(hp, 64), ctypes.byref(pp))
            mapped[q] = (pp.value, base_q)
            self._ipc_maps.append(pp.value)

        def remote_buf(nb: int, p: int) -> int:
            q = self.rank_of[nb]
            mp, base_q = mapped[q]
            return mp + (every[q][2][nb][p] - base_q)

        self._setup_vpush(remote_buf)
        self.vpush = True
        self.ipc = True
        self._setup_wave_ipc(g, mine, nbr_ranks, remote_buf)
        dist.barrier()

    def _setup_wave_ipc(self, g: int, mine: list, nbr_ranks: list, remote_buf=None,
                        diag_ranks=()) -> None:
        """Persistent wavefront across processes: every rank exports its
        per-tile step counters over CUDA IPC; an edge tile waits on the
        neighbour rank's adjacent tile counter (system scope) instead of a
        per-step launch + flag handshake.  Tilings agree on all ranks (same
        layout and rows), chunk order per rank is ``grid.per_rank``."""
        import torch.distributed as dist

        plan = self.plans[g]
        index = {lin: i for i, lin in enumerate(mine)}
        nf = 2 * self.layout.ndim
        nbr = [index.get(self.grid.chunks[lin].neighbors.get(f), -1)
               if self.grid.chunks[lin].neighbors.get(f) is not None else -1
               for lin in mine for f in range(nf)]
        N.call("hrt_jacobi_plan_set_persistent", plan, _arr(ctypes.c_int32, nbr),
               persist_timeout_ns())
        ptr, ntiles = ctypes.c_uint64(), ctypes.c_int64()
        N.call("hrt_jacobi_plan_wave_counters", plan, ctypes.byref(ptr), ctypes.byref(ntiles))
        h = ctypes.create_string_buffer(64)
        N.call("hrt_ipc_get_handle", ctypes.c_void_p(ptr.value), h)
        every = [None] * self.world
        dist.all_gather_object(every, (h.raw, self.tiling()[g][:2]))
        # neighbours index each other's tile counters with their own tiling:
        # (rows, tiles per chunk) agree by construction (decided from the
        # grid's largest per-rank chunk count); checked again after the
        # two-step set-up below
        if len({t for _, t in every}) != 1:
            raise HrtError(f"per-chunk tilings differ across ranks: {[t for _, t in every]}")
        peer_ptrs = []
        all_ranks = list(nbr_ranks) + list(diag_ranks)  # face ranks first (rpeer indexes them)
        for q in all_ranks:
            pq = ctypes.c_void_p()
            N.call("hrt_ipc_open_handle", g, ctypes.create_string_buffer(every[q][0], 64),
                   ctypes.byref(pq))
            self._ipc_maps.append(pq.value)
            peer_ptrs.append(pq.value)
        rpeer, rnbr = [], []
        for lin in mine:
            for f in range(nf):
                nb = self.grid.chunks[lin].neighbors.get(f)
                if nb is None or nb in self.placement:
                    rpeer.append(-1)
                    rnbr.append(-1)
                else:
                    q = self.rank_of[nb]
                    rpeer.append(nbr_ranks.index(q))
                    rnbr.append(list(self.grid.per_rank[q]).index(nb))
        N.call("hrt_jacobi_plan_set_wave_ipc", plan, _arr(ctypes.c_int32, rpeer),
               _arr(ctypes.c_int32, rnbr), _arr(ctypes.c_uint64, peer_ptrs), len(peer_ptrs),
               ctypes.c_uint64(30_000_000_000))
        if remote_buf is not None and nf == 4:
            # two steps per pass read the rims of the whole 3 x 3 chunk
            # neighbourhood in place: faces and corners on other ranks
            # through their IPC-mapped arenas and tile counters
            kinds, idxs, cnts, bufs = [], [], [], []
            for lin in mine:
                for q in self.grid.nbhd9(lin):
                    if q is None:
                        kinds.append(0)
                        idxs.append(-1)
                        cnts.append(0)
                        bufs += [0, 0]
                    elif q in self.placement:
                        kinds.append(1)
                        idxs.append(index[q])
                        cnts.append(0)
                        bufs += [0, 0]
                    else:
                        r = self.rank_of[q]
                        kinds.append(2)
                        idxs.append(list(self.grid.per_rank[r]).index(q))
                        cnts.append(peer_ptrs[all_ranks.index(r)])
                        bufs += [remote_buf(q, 0), remote_buf(q, 1)]
            N.call("hrt_jacobi_plan_set_wave2_nbr9", plan, _arr(ctypes.c_int32, kinds),
                   _arr(ctypes.c_int32, idxs), _arr(ctypes.c_uint64, cnts),
                   _arr(ctypes.c_uint64, bufs))
        if remote_buf is not None and nf == 6:
            # volume two-step passes read the neighbour rank's x planes in
            # place and wait on its tile counters (both mapped over IPC)
            ptr2, n2 = ctypes.c_uint64(), ctypes.c_int64()
            N.call("hrt_jacobi_plan_vw2_counters", plan, ctypes.byref(ptr2), ctypes.byref(n2))
            h2 = ctypes.create_string_buffer(64)
            N.call("hrt_ipc_get_handle", ctypes.c_void_p(ptr2.value), h2)
            every2 = [None] * self.world
            dist.all_gather_object(every2, h2.raw)
            cnt_of = {}
            for q in nbr_ranks:
                pq = ctypes.c_void_p()
                N.call("hrt_ipc_open_handle", g, ctypes.create_string_buffer(every2[q], 64),
                       ctypes.byref(pq))
                self._ipc_maps.append(pq.value)
                cnt_of[q] = pq.value
            bufs, cnts, idxs = [], [], []
            for k, lin in enumerate(mine):
                for f in (0, 1):
                    p = rpeer[nf * k + f]
                    nb = self.grid.chunks[lin].neighbors.get(f)
                    if p < 0:
                        bufs += [0, 0]
                        cnts.append(0)
                        idxs.append(-1)
                    else:
                        bufs += [remote_buf(nb, 0), remote_buf(nb, 1)]
                        cnts.append(cnt_of[nbr_ranks[p]])
                        idxs.append(rnbr[nf * k + f])
            N.call("hrt_jacobi_plan_set_vw2_remote", plan, _arr(ctypes.c_uint64, bufs),
                   _arr(ctypes.c_uint64, cnts), _arr(ctypes.c_int32, idxs))
        # a rank with a column face to another process keeps one step per
        # pass; then no rank may run two-step passes (see _agree_tiling)
        tilings = [None] * self.world
        dist.all_gather_object(tilings, self.tiling()[g])
        self._agree_tiling(tilings)
        self.persistent = True

    def check_ipc(self) -> None:
        """Raise if an edge tile timed out waiting for a neighbour rank."""
        if self.ipc:
            err = ctypes.c_int()
            N.call("hrt_jacobi_plan_ipc_error", self.plans[self.used_gpus[0]], ctypes.byref(err))
            if err.value:
                raise HrtError("IPC step handshake timed out (a neighbour rank stalled)")

    def global_residual_history(self) -> np.ndarray:
        """Per-step max over all ranks (one NCCL max all-reduce of the
        uint64 bit patterns, then one D2H)."""
        n = self._resid_steps
        g = self.used_gpus[0]
        if self.world > 1 and n:
            N.call("hrt_nccl_allreduce_max_u64", ctypes.c_void_p(self.comm), self.streams[g].h,
                   ctypes.c_void_p(self.resid[g]), n)
        return self.residual_history()

    def _rank_fence(self) -> None:
        """Device-side barrier across ranks on the solver stream (a one-word
        NCCL max all-reduce): what this rank enqueues after it runs only
        once every rank has finished what it enqueued before."""
        g = self.used_gpus[0]
        if self._fence_buf is None:
            self._fence_buf = DevicePool(g, 256)
        N.call("hrt_nccl_allreduce_max_u64", ctypes.c_void_p(self.comm), self.streams[g].h,
               ctypes.c_void_p(self._fence_buf.base), 1)

    def _segment_fence(self) -> None:
        if self._fenced():
            self._rank_fence()

    def _fenced(self) -> bool:
        """Neighbour ranks read this rank's chunks in place (IPC: two-step
        passes and their rims), so host-initiated writes need fences."""
        return bool(self.world > 1 and self.comm and self.ipc)

    def _chunk_copies(self, to_chunks: bool, parity: int, field_ptr: int, stream_of=None) -> None:
        # new interiors: the previous job's kernels of the neighbour ranks
        # may still read this rank's chunks in place — fence before
        # overwriting them (and, in _after_scatter, before anyone reads the
        # new ones: a two-step launch right after an upload has no ghost
        # exchange that would order it after the neighbours' uploads)
        if to_chunks and self._fenced():
            self._rank_fence()
        super()._chunk_copies(to_chunks, parity, field_ptr, stream_of)

    def _after_scatter(self) -> None:
        """Volumes: every rank's upload scan (smallest positive value, bad
        flag) max-reduced over all ranks on the solver stream, so each
        rank's two-step launch picks its division from the global field —
        tiny values of one rank reach its neighbours within a few steps.
        The reduction (or a fence) also orders every rank's next launch
        after all ranks' uploads."""
        if self.world > 1 and self.layout.ndim == 3 and self.comm:
            g = self.used_gpus[0]
            ptr = ctypes.c_uint64()
            N.call("hrt_jacobi_plan_range", self.plans[g], ctypes.byref(ptr))
            if ptr.value:
                N.call("hrt_nccl_allreduce_max_u64", ctypes.c_void_p(self.comm),
                       self.streams[g].h, ctypes.c_void_p(ptr.value), 2)
                return
        if self._fenced():
            self._rank_fence()

    def allreduce_residual(self) -> None:
        """Enqueue the cross-rank max of this run's residual history on the
        solver stream (no host sync; run_jobs' ``after_run`` hook)."""
        n = self._resid_steps
        g = self.used_gpus[0]
        if self.world > 1 and n:
            N.call("hrt_nccl_allreduce_max_u64", ctypes.c_void_p(self.comm), self.streams[g].h,
                   ctypes.c_void_p(self.resid[g]), n)

    def close(self) -> None:
        if self._ipc_maps:
            import torch.distributed as dist

            self.sync()
            dist.barrier()  # nobody still pushes into memory about to be unmapped/freed
        super().close()
        for ptr in self._ipc_maps:
            N.lib().hrt_ipc_close_handle(ctypes.c_void_p(ptr))
        if self._ipc_maps:
            dist.barrier()  # every mapping closed before any arena is freed
        self._ipc_maps = []
        if self.comm:
            N.lib().hrt_nccl_destroy(ctypes.c_void_p(self.comm))
            self.comm = None
