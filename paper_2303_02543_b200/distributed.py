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
from .jacobi import ChunkGrid, JacobiSolver


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
                 variant: Optional[int] = None):
        if grid.ranks != world:
            raise ValueError("grid.ranks must equal the world size")
        if comm is None and world > 1:
            comm = nccl_comm(rank, world, gpu)
        self.world = world
        super().__init__(grid, gpus=[gpu], rank=rank, comm=comm, rows=rows, variant=variant)

    def global_residual_history(self) -> np.ndarray:
        """Per-step max over all ranks (one NCCL max all-reduce of the
        uint64 bit patterns, then one D2H)."""
        n = self._resid_steps
        g = self.used_gpus[0]
        if self.world > 1 and n:
            N.call("hrt_nccl_allreduce_max_u64", ctypes.c_void_p(self.comm), self.streams[g].h,
                   ctypes.c_void_p(self.resid[g]), n)
        return self.residual_history()

    def close(self) -> None:
        super().close()
        if self.comm:
            N.lib().hrt_nccl_destroy(ctypes.c_void_p(self.comm))
            self.comm = None
