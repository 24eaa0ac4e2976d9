"""paper_2303_02543_b200 — B200-native backend for the Jacobi / halo-exchange /
device-message hot path of the PREMA heterogeneous runtime (arXiv 2303.02543;
reference package ``hrt`` at /root/reference/pkg/src/hrt).

The public names mirror the reference's (``run_jacobi3d``, ``run_pingpong``,
``Runtime``, ``Comm``, ``DeviceRegistry`` ...); the compute path is
libhrt_b200.so (include/hrt_b200.h): hand-written sm_100a kernels, CUDA
streams/events/graphs, NVLink peer copies and NCCL send/recv.
"""

from .errors import (  # noqa: F401
    DeadlockError,
    DependencyCycle,
    DoubleFree,
    HrtError,
    InvalidLocation,
    KernelError,
    LeaseConflict,
    NotOwner,
    OutOfDeviceMemory,
    ProtocolError,
    SchedulerBusy,
    TaskFailed,
    TransportClosed,
    UnknownToken,
    UnsatisfiableEviction,
)

__version__ = "0.1.0"

_LAZY = {
    "run_jacobi3d": ".jacobi",
    "ChunkGrid": ".jacobi",
    "JacobiSolver": ".jacobi",
    "FACES": ".jacobi",
    "opposite": ".jacobi",
    "DistributedJacobi": ".distributed",
    "run_pingpong": ".pingpong",
    "parse_sizes": ".pingpong",
    "BenchReport": ".reporting",
    "Tracer": ".trace",
    "ClockMode": ".devices",
    "DeviceType": ".devices",
    "DeviceDescriptor": ".devices",
    "DeviceRegistry": ".devices",
    "DeviceAllocation": ".devices",
    "CompletionToken": ".devices",
    "TokenKind": ".devices",
    "TokenStatus": ".devices",
    "HostPinnedPool": ".devices",
    "Runtime": ".runtime",
    "HeteroTask": ".runtime",
    "TaskState": ".runtime",
    "TaskBuilder": ".builder",
    "KernelRegistry": ".kernels",
    "KernelRef": ".kernels",
    "ThreadGeometry": ".kernels",
    "HeteroObject": ".objects",
    "AccessMode": ".objects",
    "CopyState": ".objects",
    "Comm": ".comm",
    "MobileRef": ".comm",
    "drive": ".comm",
    "exchange_all": ".comm",
    "shutdown_all": ".comm",
    "WorldConfig": ".worlds",
    "make_world": ".worlds",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(mod, __name__), name)
