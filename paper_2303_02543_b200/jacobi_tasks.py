"""The reference's Jacobi task protocol executed by the B200 runtime
(``run_jacobi3d(..., engine="tasks")``).

Same protocol as _RankDriver (/root/reference/pkg/src/hrt/bench/jacobi.py:
143-278): chunks are mobile objects whose state carries the chunk id; each
chunk owns two dense ghosted (ex+2, ey+2, ez+2) float64 objects; every step
a pack task per face writes a halo object that is ``mp_send``-ed to the
neighbour's face handler and destroyed (deferred); once all faces of step s
arrived, unpack tasks write the ghost planes and the update task writes the
other buffer; finally every chunk ships its buffer to a collector on rank 0.

What runs where: pack/unpack/update are native launchers (native_kernels);
tasks are issued to CUDA streams as soon as their prerequisites are
*launched*, so a chunk's pack -> send (device copy) -> unpack -> update chain
is ordered on the GPU by events, with several chunks in flight per device;
halo messages take the direct device path (no host staging) when the
transport is device-aware, or the host-staged path otherwise.

This engine is the API-fidelity path (handlers, objects, messages); the
native engine (jacobi.JacobiSolver) is the performance path.
"""

from __future__ import annotations

import struct
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .comm import MobileRef, drive, exchange_all, shutdown_all
from .devices import DeviceType
from .errors import HrtError
from .jacobi import BOUNDARY, FACES, ChunkGrid, opposite
from .native_kernels import HaloPack, HaloUnpack, JacobiUpdate
from .reporting import BenchReport
from .worlds import WorldConfig, device_id_for, make_loopback_world


@dataclass
class _Chunk:
    lin: int
    coord: tuple
    extents: tuple
    offsets: tuple
    device_id: int
    bufs: list = field(default_factory=list)
    neighbors: dict = field(default_factory=dict)
    step: int = 0
    sent_step: int = -1
    recv_count: dict = field(default_factory=dict)
    inbox: dict = field(default_factory=dict)
    done: bool = False


class _RankDriver:
    def __init__(self, comm, steps: int):
        self.comm = comm
        self.rt = comm.runtime
        self.steps = steps
        self.chunks: dict[int, _Chunk] = {}
        self.ref_of: dict[int, MobileRef] = {}
        self.completed = 0
        self.gathered: dict[int, object] = {}
        self._gather_meta: dict[int, list[int]] = {}
        self._collector_ref = None
        rt = self.rt
        self.k_update = rt.register_kernel("jacobi_update", gpu_sim=JacobiUpdate())
        self.k_pack = [rt.register_kernel(f"halo_pack_{f}", gpu_sim=HaloPack(f)) for f in range(6)]
        self.k_unpack = [rt.register_kernel(f"halo_unpack_{f}", gpu_sim=HaloUnpack(f))
                         for f in range(6)]
        self.h_halo = [comm.register_handler(self._halo_handler(f)) for f in range(6)]
        self.h_gather_meta = comm.register_handler(self._on_gather_meta)
        self.h_gather_obj = comm.register_handler(self._on_gather_obj)

    def _halo_handler(self, face: int):
        def handler(mobile, arg, ctx) -> None:
            ch = self.chunks[struct.unpack("<I", bytes(mobile.state[:4]))[0]]
            s = ch.recv_count.get(face, 0)
            ch.recv_count[face] = s + 1
            ch.inbox.setdefault(s, {})[face] = arg
            self._try_finish_step(ch)

        return handler

    def _on_gather_meta(self, mobile, arg, ctx) -> None:
        self._gather_meta.setdefault(ctx.src_rank, []).append(struct.unpack("<I", arg)[0])

    def _on_gather_obj(self, mobile, arg, ctx) -> None:
        self.gathered[self._gather_meta[ctx.src_rank].pop(0)] = arg

    def start_step(self, ch: _Chunk) -> None:
        s = ch.step
        if ch.sent_step >= s or ch.done:
            return
        ch.sent_step = s
        u = ch.bufs[s % 2]
        nx, ny, nz = ch.extents
        for face, nbr in sorted(ch.neighbors.items()):
            axis = FACES[face][0]
            shape = [nx, ny, nz]
            del shape[axis]
            halo = self.rt.create_object(tuple(shape), dtype=np.float64)
            t = self.rt.task().device(DeviceType.GPU_SIM)
            t.arg(u).read()
            t.arg(halo).write()
            t.set_threads((shape[0] * shape[1], 1, 1), (1, 1, 1))
            t.submit(self.k_pack[face])
            self.comm.mp_send(self.ref_of[nbr], self.h_halo[opposite(face)], halo)
            self.rt.destroy_object(halo)
        self._try_finish_step(ch)

    def _try_finish_step(self, ch: _Chunk) -> None:
        s = ch.step
        if ch.done or ch.sent_step < s:
            return
        if not set(ch.neighbors) <= set(ch.inbox.get(s, {})):
            return
        u, nxt = ch.bufs[s % 2], ch.bufs[(s + 1) % 2]
        nx, ny, nz = ch.extents
        for face in sorted(ch.inbox.get(s, {})):
            wrapper = ch.inbox[s][face]
            t = self.rt.task().device(DeviceType.GPU_SIM)
            t.arg(wrapper).read()
            t.arg(u).write()
            t.submit(self.k_unpack[face])
            self.rt.destroy_object(wrapper)
        ch.inbox.pop(s, None)
        t = self.rt.task().device(DeviceType.GPU_SIM)
        t.arg(u).read()
        t.arg(nxt).write()
        t.set_threads((nx * ny * nz, 1, 1), (1, 1, 1))
        t.submit(self.k_update)
        ch.step = s + 1
        if ch.step >= self.steps:
            ch.done = True
            self.completed += 1
            self.comm.mp_send(self._collector_ref, self.h_gather_meta, struct.pack("<I", ch.lin))
            self.comm.mp_send(self._collector_ref, self.h_gather_obj, ch.bufs[self.steps % 2])
        else:
            self.start_step(ch)


def run_jacobi3d_tasks(domain, ranks: int = 1, devices_per_rank: int = 1, od: int = 1,
                       steps: int = 10, grid=None, streams: int = 5, device_aware: bool = False,
                       check: bool = False, tracer=None, gpus=None, capacity: Optional[int] = None):
    cg = ChunkGrid(domain, ranks, devices_per_rank, od, grid)
    ex, ey, ez = cg.ext
    buf_bytes = (ex + 2) * (ey + 2) * (ez + 2) * 8
    per_dev = -(-cg.nchunks // (ranks * devices_per_rank))
    cap = capacity or max(64 << 20, per_dev * (2 * buf_bytes + 8 * buf_bytes // max(ex, 1)) * 2
                          + (32 << 20))
    cfg = WorldConfig(ranks=ranks, devices_per_rank=devices_per_rank, streams=streams,
                      device_aware=device_aware, capacity=cap, gpus=gpus)
    comms = make_loopback_world(cfg, tracer)
    drivers = [_RankDriver(c, steps) for c in comms]
    for r in range(ranks):
        for pos, lin in enumerate(cg.per_rank[r]):
            ch = cg.chunks[lin]
            comms[r].create_mobile_object(struct.pack("<I", lin),
                                          device_hint=device_id_for(r, ch.device_local))
    comms[0].create_mobile_object(b"collector")
    exchange_all(comms)
    ref_of = {lin: MobileRef(r, pos) for r in range(ranks) for pos, lin in enumerate(cg.per_rank[r])}
    collector = MobileRef(0, len(cg.per_rank[0]))
    for r, d in enumerate(drivers):
        d.ref_of = ref_of
        d._collector_ref = collector
        rt = comms[r].runtime
        for lin in cg.per_rank[r]:
            c = cg.chunks[lin]
            ch = _Chunk(lin, c.coord, cg.ext, c.offsets, device_id_for(r, c.device_local),
                        neighbors=dict(c.neighbors))
            for b in range(2):
                obj = rt.create_object((ex + 2, ey + 2, ez + 2), dtype=np.float64)
                view = rt.request_data(obj, write=True).get()
                view[:] = 0.0
                if b == 0:
                    for f, (axis, side) in enumerate(FACES):
                        if f not in ch.neighbors:
                            sl = [slice(None)] * 3
                            sl[axis] = 0 if side == 0 else view.shape[axis] - 1
                            view[tuple(sl)] = BOUNDARY
                rt.release(obj)
                ch.bufs.append(obj)
            d.chunks[lin] = ch
    t0 = time.perf_counter()
    for d in drivers:
        for ch in d.chunks.values():
            d.start_step(ch)
    drive(comms, until=lambda: len(drivers[0].gathered) == cg.nchunks, timeout=600.0)
    rt0 = comms[0].runtime
    assembled = np.empty(cg.domain, dtype=np.float64)
    for lin in range(cg.nchunks):
        w = drivers[0].gathered[lin]
        drive(comms, until=lambda w=w: w.written, timeout=120.0)
        raw = rt0.peek(w).reshape(-1).view(np.float64).reshape(ex + 2, ey + 2, ez + 2)
        ox, oy, oz = cg.chunks[lin].offsets
        assembled[ox:ox + ex, oy:oy + ey, oz:oz + ez] = raw[1:-1, 1:-1, 1:-1]
    makespan = time.perf_counter() - t0
    checksum = float(np.sum(assembled))  # jacobi.py:436 (reporting, on the result)
    report = BenchReport("jacobi3d", columns=["step", "virtual_makespan_s"],
                         meta={"domain": list(cg.domain), "grid": list(cg.grid), "ranks": ranks,
                               "devices_per_rank": devices_per_rank, "od": od, "steps": steps,
                               "checksum": checksum, "makespan_s": makespan, "engine": "tasks",
                               "stats": [vars(c.stats).copy() for c in comms],
                               "tasks": [c.runtime.stats["tasks_completed"] for c in comms]})
    for s in range(1, steps + 1):  # wall clock: the makespan for every step (jacobi.py:453-454)
        report.add(step=s, virtual_makespan_s=makespan)
    if check:
        from .jacobi import jacobi_single_array

        if not np.array_equal(assembled, jacobi_single_array(cg.domain, steps)):
            raise HrtError("jacobi3d result differs from the single-array reference")
    shutdown_all(comms)
    return report, checksum, assembled
