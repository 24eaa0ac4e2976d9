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


def _free_ports(n: int) -> list:
    import socket

    socks, ports = [], []
    for _ in range(n):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        socks.append(s)
        ports.append(s.getsockname()[1])
    for s in socks:
        s.close()
    return ports


def make_tcp_world(cfg: WorldConfig, tracer=None) -> list[Comm]:
    """All ranks in this process over localhost TCP (worlds.py:110-123):
    the byte protocol end to end — reference headers, data frames, and for
    device-aware sends a CUDA-IPC device locator instead of payload bytes."""
    from .transport import TcpTransport

    peers = [f"127.0.0.1:{p}" for p in _free_ports(cfg.ranks)]
    ts = [TcpTransport(r, peers, device_aware=cfg.device_aware) for r in range(cfg.ranks)]
    while not all([t.establish() for t in ts]):  # every endpoint, every round
        pass
    return [Comm(ts[r], build_rank_runtime(cfg, r, DeviceClock(), tracer),
                 recv_cache_bytes=cfg.recv_cache_bytes) for r in range(cfg.ranks)]


def init_from_env(runtime: Runtime, recv_cache_bytes=None) -> Comm:
    """This process's endpoint from HRT_* variables (comm.py:1053-1082):
    HRT_TRANSPORT=tcp with HRT_RANK and HRT_PEERS (host:port list) joins a
    multi-process world; HRT_DEVICE_AWARE=1 selects device locators (CUDA
    IPC, same node).  Default: a single-rank loopback."""
    import os

    from .config import env_bool
    from .errors import HrtError
    from .transport import TcpTransport

    aware = env_bool("HRT_DEVICE_AWARE")
    if os.environ.get("HRT_TRANSPORT", "loopback") == "tcp":
        rank = int(os.environ["HRT_RANK"])
        peers = [p.strip() for p in os.environ["HRT_PEERS"].split(",") if p.strip()]
        t = TcpTransport(rank, peers, device_aware=aware)
        t.establish_blocking()
        return Comm(t, runtime, recv_cache_bytes=recv_cache_bytes)
    if int(os.environ.get("HRT_RANKS", "1")) != 1:
        raise HrtError("multi-rank loopback worlds are built with make_loopback_world")
    return Comm(LoopbackFabric(1).endpoint(0, device_aware=aware), runtime,
                recv_cache_bytes=recv_cache_bytes)
