"""World construction (/root/reference/pkg/src/hrt/bench/worlds.py:23-95):
per-rank B200 device registry + runtime + comm endpoint over an in-process
loopback fabric.  Device ids are ``rank*100 + local`` (worlds.py:39-41);
virtual device ``rank*devices_per_rank + local`` is placed on physical GPU
``gpus[index % len(gpus)]``.  This is where the B200 backend is selected
(SURVEY.md §8(b) item 5)."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

from . import _native as N
from .comm import Comm, LoopbackFabric
from .devices import ClockMode, DeviceClock, DeviceDescriptor, DeviceRegistry, DeviceType
from .runtime import Runtime


@dataclass
class WorldConfig:
    ranks: int = 1
    devices_per_rank: int = 1
    clock: ClockMode = ClockMode.WALL
    capacity: int = 256 << 20
    latency: float = 1e-5        # simulator parameters, accepted and unused
    bandwidth: float = 1e9
    streams: int = 5
    device_aware: bool = False
    recv_cache_bytes: Optional[int] = None
    shared_host_bus: bool = False
    with_host_device: bool = False  # host copies live in the pinned pool
    host_capacity: int = 64 << 20
    gpus: Optional[Sequence[int]] = None


def device_id_for(rank: int, local_index: int) -> int:
    return rank * 100 + local_index


def build_rank_runtime(cfg: WorldConfig, rank: int, clock=None, tracer=None) -> Runtime:
    gpus = list(cfg.gpus) if cfg.gpus is not None else list(range(max(1, N.gpu_count())))
    reg = DeviceRegistry(clock_mode=cfg.clock, shared_host_bus=cfg.shared_host_bus,
                         tracer=tracer, clock=clock)
    for j in range(cfg.devices_per_rank):
        idx = rank * cfg.devices_per_rank + j
        reg.register_device(DeviceDescriptor(
            device_id=device_id_for(rank, j), device_type=DeviceType.GPU_SIM,
            memory_capacity=cfg.capacity, compute_stream_count=cfg.streams,
            transfer_latency=cfg.latency, transfer_bandwidth=cfg.bandwidth,
            clock_mode=cfg.clock, gpu=gpus[idx % len(gpus)]))
    return Runtime(reg)


def make_loopback_world(cfg: WorldConfig, tracer=None) -> list[Comm]:
    N.require_gpu(0)
    clock = DeviceClock()
    fabric = LoopbackFabric(cfg.ranks)
    return [Comm(fabric.endpoint(r, device_aware=cfg.device_aware),
                 build_rank_runtime(cfg, r, clock, tracer), recv_cache_bytes=cfg.recv_cache_bytes)
            for r in range(cfg.ranks)]


make_world = make_loopback_world
