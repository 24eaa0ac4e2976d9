"""B200 device layer: HBM pools, CUDA streams, event-backed completion
tokens, pinned host staging and asynchronous transfers.

Mirrors the surface of the reference's simulated device layer
(/root/reference/pkg/src/hrt/devices.py) — ``DeviceType``, ``ClockMode``,
``TokenKind``/``TokenStatus``, ``DeviceDescriptor``, ``DeviceAllocation``,
``CompletionToken``, ``HostPinnedPool``, ``DeviceRegistry`` with
``register_device``/``pool_alloc``/``pool_free``/``enqueue_transfer``/
``enqueue_kernel``/``poll`` — but every device is a real B200:

* device arenas are one ``cudaMalloc`` per device managed by the native
  first-fit list (the reference's ``FreeListAllocator``, devices.py:89-154);
* tokens are cudaEvents recorded on the operation's stream; ``status``
  queries the event lazily (the reference fires tokens from a clock,
  devices.py:199-252);
* transfers are real ``cudaMemcpyAsync`` on per-direction streams, and
  device-to-device / peer transfers are allowed (the reference rejects them,
  devices.py:456-457);
* kernels are native launchers enqueued on a compute stream after waiting
  (GPU-side) on the tokens of their prerequisites.

``DeviceType.GPU_SIM`` is kept as the accelerator type name so drivers
written against the reference (which hard-code it, e.g.
bench/jacobi.py:232) target the B200; ``DeviceType.B200`` is an alias.
"""

from __future__ import annotations

import ctypes
from collections import deque
import os
import time
from dataclasses import dataclass, field
from enum import Enum
from typing import Any, Callable, Optional, Union

import numpy as np

from . import _native as N
from .errors import DoubleFree, HrtError, InvalidLocation, OutOfDeviceMemory, UnknownToken
from .trace import NullTracer, Tracer

ALIGNMENT = 256  # devices.py:35


class DeviceType(Enum):
    HOST = "host"
    GPU_SIM = "gpu_sim"
    B200 = "gpu_sim"  # alias: the accelerator type is a real B200 here


class ClockMode(Enum):
    WALL = "wall"
    VIRTUAL = "virtual"  # accepted for signature compatibility; B200 runs in real time


class TokenKind(Enum):
    TRANSFER = "transfer"
    KERNEL = "kernel"


class TokenStatus(Enum):
    PENDING = "pending"
    COMPLETE = "complete"
    FAILED = "failed"


def default_compute_streams() -> int:
    from .config import env_int

    return env_int("HRT_STREAMS", 5)


@dataclass
class DeviceDescriptor:
    """devices.py:59-78; ``gpu`` selects the physical B200 (default: the
    device id modulo the visible GPU count)."""

    device_id: int
    device_type: DeviceType
    memory_capacity: int
    compute_stream_count: int = field(default_factory=default_compute_streams)
    transfer_stream_count: int = 2
    transfer_latency: float = 0.0
    transfer_bandwidth: float = float("inf")
    clock_mode: ClockMode = ClockMode.WALL
    gpu: Optional[int] = None

    def validate(self) -> None:
        if self.device_id < 0:
            raise HrtError(f"device_id must be >= 0, got {self.device_id}")
        if self.memory_capacity <= 0:
            raise HrtError("memory_capacity must be positive")
        if self.compute_stream_count < 1:
            raise HrtError("compute_stream_count must be >= 1")
        if self.transfer_stream_count != 2:
            raise HrtError("transfer_stream_count is fixed at 2 (one per direction)")


@dataclass(frozen=True)
class DeviceAllocation:
    device_id: int
    offset: int
    size: int
    alignment: int = ALIGNMENT
    ptr: int = 0  # device byte address (UVA)


# ---------------------------------------------------------------------------
# native handles


class Stream:
    """A CUDA stream on one GPU (owned unless wrapped)."""

    def __init__(self, gpu: int, priority: int = 0, handle: Optional[int] = None,
                 name: str = ""):
        self.gpu = gpu
        self.name = name
        h = ctypes.c_void_p()
        if handle is None:
            N.require_gpu(gpu)
            N.call("hrt_stream_create", gpu, priority, ctypes.byref(h))
            self._owned = 1
        else:
            N.call("hrt_stream_wrap", gpu, ctypes.c_void_p(handle), ctypes.byref(h))
            self._owned = 0
        self.h = h

    @property
    def cuda_stream(self) -> int:
        return N.lib().hrt_stream_handle(self.h) or 0

    def synchronize(self) -> None:
        N.call("hrt_stream_synchronize", self.h)

    def record(self, kind: TokenKind = TokenKind.KERNEL, device_id: int = -1) -> "CompletionToken":
        t = ctypes.c_uint64()
        N.call("hrt_token_record", self.h, ctypes.byref(t))
        return CompletionToken(t.value, kind, device_id if device_id >= 0 else self.gpu,
                               stream=self.h.value)

    def wait(self, token: "CompletionToken") -> None:
        """GPU-side edge: later work on this stream waits for ``token``."""
        if token is not None and token._native:
            N.call("hrt_stream_wait_token", self.h, ctypes.c_uint64(token.token_id))

    def close(self) -> None:
        if self.h:
            N.lib().hrt_stream_destroy(self.h, self._owned)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CompletionToken:
    """Handle for one asynchronous device operation (devices.py:199-222).

    Backed by a cudaEvent; ``status`` queries it (non-blocking) and latches
    COMPLETE/FAILED exactly once.  Host-only operations complete at creation.
    """

    __slots__ = ("token_id", "kind", "device_id", "_status", "error", "end_time", "_native",
                 "stream", "__weakref__")

    def __init__(self, token_id: int, kind: TokenKind, device_id: int, native: bool = True,
                 stream=None):
        self.stream = stream  # the recording stream's handle (events complete in stream order)
        self.token_id = token_id
        self.kind = kind
        self.device_id = device_id
        self._native = native
        self._status = TokenStatus.PENDING if native else TokenStatus.COMPLETE
        self.error: Optional[BaseException] = None
        self.end_time = 0.0

    @classmethod
    def completed(cls, kind: TokenKind, device_id: int = -1) -> "CompletionToken":
        return cls(0, kind, device_id, native=False)

    @property
    def status(self) -> TokenStatus:
        if self._status is TokenStatus.PENDING:
            rc = N.lib().hrt_token_query(ctypes.c_uint64(self.token_id))
            if rc == 1:
                self._finish(TokenStatus.COMPLETE)
            elif rc == 2 or rc < 0:
                self.error = HrtError(N.last_error())
                self._finish(TokenStatus.FAILED)
        return self._status

    def _finish(self, st: TokenStatus) -> None:
        self._status = st
        self.end_time = time.perf_counter()
        if self._native:
            N.lib().hrt_token_release(ctypes.c_uint64(self.token_id))
            self._native = False

    def fail(self, error: BaseException) -> None:
        self.error = error
        if self._native:
            N.lib().hrt_token_release(ctypes.c_uint64(self.token_id))
            self._native = False
        self._status = TokenStatus.FAILED

    def wait(self) -> TokenStatus:
        if self._status is TokenStatus.PENDING and self._native:
            rc = N.lib().hrt_token_wait(ctypes.c_uint64(self.token_id))
            if rc != 0:
                self.error = HrtError(N.last_error())
                self._finish(TokenStatus.FAILED)
            else:
                self._finish(TokenStatus.COMPLETE)
        return self._status

    def __repr__(self) -> str:
        return f"<token {self.token_id} {self.kind.value} {self._status.value}>"

    def __del__(self):
        try:
            if self._native:
                N.lib().hrt_token_release(ctypes.c_uint64(self.token_id))
        except Exception:
            pass


class DevicePool:
    """One HBM arena per device, carved by the native first-fit list
    (pool_alloc/pool_free, devices.py:398-404)."""

    def __init__(self, gpu: int, capacity: int):
        N.require_gpu(gpu)
        self.gpu = gpu
        self.capacity = int(capacity)
        h = ctypes.c_void_p()
        N.call("hrt_pool_create", gpu, ctypes.c_uint64(self.capacity), ctypes.byref(h))
        self.h = h
        base = ctypes.c_void_p()
        N.call("hrt_pool_base", h, ctypes.byref(base))
        self.base = base.value

    def alloc(self, size: int) -> tuple[int, int, int]:
        if size <= 0:
            raise HrtError(f"allocation size must be positive, got {size}")
        off, granted, ptr = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_void_p()
        N.call("hrt_pool_alloc", self.h, ctypes.c_uint64(size), ctypes.byref(off),
               ctypes.byref(granted), ctypes.byref(ptr))
        return off.value, granted.value, ptr.value

    def free(self, offset: int) -> None:
        N.call("hrt_pool_free", self.h, ctypes.c_uint64(offset))

    @property
    def free_bytes(self) -> int:
        live, free = ctypes.c_uint64(), ctypes.c_uint64()
        N.call("hrt_pool_stats", self.h, ctypes.byref(live), ctypes.byref(free))
        return free.value

    def close(self) -> None:
        if self.h:
            N.lib().hrt_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host memory exposed to numpy (``array(dtype, shape)``)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        N.call("hrt_host_alloc", ctypes.c_uint64(max(self.nbytes, 1)), ctypes.byref(p))
        self.ptr = p.value

    def array(self, dtype=np.uint8, shape=None) -> np.ndarray:
        dtype = np.dtype(dtype)
        count = self.nbytes // dtype.itemsize
        raw = (ctypes.c_char * self.nbytes).from_address(self.ptr)
        arr = np.frombuffer(raw, dtype=dtype, count=count)
        return arr.reshape(shape) if shape is not None else arr

    def close(self) -> None:
        if self.ptr:
            N.lib().hrt_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class HostRegion:
    """A host-memory window; ``pooled`` means it came from the pinned pool."""

    array: np.ndarray
    nbytes: int
    offset: Optional[int] = None
    pooled: bool = False

    @property
    def ptr(self) -> int:
        return self.array.ctypes.data


class FirstFit:
    """Python handle on the native first-fit list (hrt_fl_*), the exact
    semantics of FreeListAllocator (devices.py:89-154)."""

    def __init__(self, capacity: int, alignment: int = ALIGNMENT):
        if capacity <= 0:
            raise HrtError("allocator capacity must be positive")
        h = ctypes.c_void_p()
        N.call("hrt_fl_create", ctypes.c_uint64(capacity), ctypes.c_uint64(alignment),
               ctypes.byref(h))
        self.h = h
        self.capacity = capacity
        self.alignment = alignment

    def alloc(self, size: int) -> tuple[int, int]:
        if size <= 0:
            raise HrtError(f"allocation size must be positive, got {size}")
        off, granted = ctypes.c_uint64(), ctypes.c_uint64()
        N.call("hrt_fl_alloc", self.h, ctypes.c_uint64(size), ctypes.byref(off),
               ctypes.byref(granted))
        return off.value, granted.value

    def free(self, offset: int) -> int:
        size = ctypes.c_uint64()
        N.call("hrt_fl_free", self.h, ctypes.c_uint64(offset), ctypes.byref(size))
        return size.value

    def _stats(self):
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        N.call("hrt_fl_stats", self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        return a.value, b.value, c.value

    @property
    def live_bytes(self) -> int:
        return self._stats()[0]

    @property
    def free_bytes(self) -> int:
        return self._stats()[1]

    def check(self) -> None:
        N.call("hrt_fl_check", self.h)

    def __del__(self):
        try:
            if self.h:
                N.lib().hrt_fl_destroy(self.h)
                self.h = None
        except Exception:
            pass


class HostPinnedPool:
    """Page-locked staging pool (devices.py:167-196), allocated once and
    carved first-fit; exhaustion falls back to pageable memory and bumps
    ``misses``."""

    def __init__(self, capacity: Optional[int] = None):
        from .config import default_pinned_pool_bytes

        self.capacity = capacity if capacity is not None else default_pinned_pool_bytes()
        self._buf = PinnedBuffer(self.capacity)
        self.arena = self._buf.array(np.uint8)
        self._alloc = FirstFit(self.capacity)
        self.misses = 0

    def alloc(self, nbytes: int) -> HostRegion:
        try:
            off, _ = self._alloc.alloc(max(nbytes, 1))
        except OutOfDeviceMemory:
            self.misses += 1
            return HostRegion(np.zeros(nbytes, dtype=np.uint8), nbytes, None, False)
        return HostRegion(self.arena[off: off + nbytes], nbytes, off, True)

    def free(self, region: HostRegion) -> None:
        if region.pooled and region.offset is not None:
            self._alloc.free(region.offset)
            region.offset = None
            region.pooled = False

    def note_unpinned_use(self) -> None:
        self.misses += 1


# ---------------------------------------------------------------------------
# clocks


class DeviceClock:
    """Real-time clock with the reference clock surface (devices.py:225-274).

    ``advance_one`` blocks on the oldest outstanding device token and returns
    it, so ``Runtime.wait``/``drive`` make progress while GPU work is in
    flight instead of declaring a deadlock (runtime.py:503-506)."""

    def __init__(self) -> None:
        self._t0 = time.perf_counter()
        self._outstanding: deque = deque()

    @property
    def now(self) -> float:
        return time.perf_counter() - self._t0

    def track(self, token: CompletionToken) -> None:
        if token.status is TokenStatus.PENDING:
            self._outstanding.append(token)

    def schedule(self, token: CompletionToken, end_time: float) -> None:
        self.track(token)

    def track_pending(self, token: CompletionToken) -> None:
        """A token recorded just now (no status query: it is pending or
        will be found complete by the next service pass).  Settled tokens at
        the front are dropped here, so the queue stays as long as the work
        actually in flight."""
        q = self._outstanding
        while q and q[0]._status is not TokenStatus.PENDING:
            q.popleft()
        q.append(token)

    def advance_one(self) -> Optional[CompletionToken]:
        while self._outstanding:
            tok = self._outstanding.popleft()
            if tok.status is TokenStatus.PENDING:
                tok.wait()
                return tok
        return None

    @property
    def pending_events(self) -> int:
        self._outstanding = deque(t for t in self._outstanding if t.status is TokenStatus.PENDING)
        return len(self._outstanding)


WallClock = DeviceClock
VirtualClock = DeviceClock


# ---------------------------------------------------------------------------
# registry


class _Device:
    def __init__(self, descriptor: DeviceDescriptor, gpu: int):
        self.descriptor = descriptor
        self.gpu = gpu
        self.pool = DevicePool(gpu, descriptor.memory_capacity)
        self.compute_streams = [Stream(gpu, name=f"c{i}")
                                for i in range(descriptor.compute_stream_count)]
        # stream handle -> compute stream index (tokens carry their stream)
        self.stream_index = {st.h.value: i for i, st in enumerate(self.compute_streams)}
        self.h2d = Stream(gpu, name="h2d")
        self.d2h = Stream(gpu, name="d2h")

    @property
    def device_id(self) -> int:
        return self.descriptor.device_id


@dataclass(frozen=True)
class ForeignAllocation:
    """A device allocation owned by another rank's registry in this process
    (the direct message path reads it as a peer-copy source)."""

    alloc: DeviceAllocation
    gpu: int


Location = Union[DeviceAllocation, HostRegion, np.ndarray, ForeignAllocation]


class DeviceRegion:
    """A device-resident byte window (the reference's ``backend.region``,
    devices.py:302-305, returned a numpy view of the arena).  Supports the
    operations the reference performs on regions: ``region[:] = ndarray``
    (H2D), ``tobytes()``/``copy()`` (D2H), ``view(dtype).reshape(...)``
    bookkeeping, and exposes the raw device pointer for kernels."""

    def __init__(self, registry: "DeviceRegistry", alloc: DeviceAllocation, nbytes: int,
                 dtype=np.uint8, shape=None):
        self.registry = registry
        self.alloc = alloc
        self.nbytes = int(nbytes)
        self.dtype = np.dtype(dtype)
        self.shape = tuple(shape) if shape is not None else (self.nbytes // self.dtype.itemsize,)

    @property
    def ptr(self) -> int:
        return self.alloc.ptr

    @property
    def device_id(self) -> int:
        return self.alloc.device_id

    def view(self, dtype) -> "DeviceRegion":
        return DeviceRegion(self.registry, self.alloc, self.nbytes, dtype)

    def reshape(self, *shape) -> "DeviceRegion":
        if len(shape) == 1 and isinstance(shape[0], tuple):
            shape = shape[0]
        return DeviceRegion(self.registry, self.alloc, self.nbytes, self.dtype, shape)

    def __setitem__(self, key, value) -> None:
        if key != slice(None) and key != Ellipsis:
            raise HrtError("device regions support whole-region assignment only")
        src = np.ascontiguousarray(value)
        if src.nbytes == 0:
            return
        if np.ndim(value) == 0 or src.size == 1 and src.nbytes != self.nbytes:
            src = np.full(self.shape, value, dtype=self.dtype)
        raw = src.reshape(-1).view(np.uint8)
        if raw.nbytes != self.nbytes:
            raise InvalidLocation(f"assignment of {raw.nbytes} B into a {self.nbytes} B region")
        dev = self.registry.device(self.device_id)
        N.call("hrt_copy_async", dev.h2d.h, ctypes.c_void_p(self.ptr),
               ctypes.c_void_p(raw.ctypes.data), ctypes.c_uint64(self.nbytes))
        dev.h2d.synchronize()

    def tobytes(self) -> bytes:
        return self.copy().tobytes()

    def copy(self) -> np.ndarray:
        out = np.empty(self.nbytes, dtype=np.uint8)
        dev = self.registry.device(self.device_id)
        N.call("hrt_copy_async", dev.d2h.h, ctypes.c_void_p(out.ctypes.data),
               ctypes.c_void_p(self.ptr), ctypes.c_uint64(self.nbytes))
        dev.d2h.synchronize()
        return out.view(self.dtype).reshape(self.shape)

    def __array__(self, dtype=None, copy=None):
        a = self.copy()
        return a.astype(dtype) if dtype is not None else a

    def __len__(self) -> int:
        return self.shape[0]


_PLACED: dict[int, int] = {}


def _placement(device_id: int, ngpu: int) -> int:
    """Process-wide round robin: the k-th distinct accelerator device id
    (rank*100+local, worlds.py:39-41) lands on GPU k mod ngpu."""
    if device_id not in _PLACED:
        _PLACED[device_id] = len(_PLACED) % ngpu
    return _PLACED[device_id]


class DeviceRegistry:
    """Owner of all B200 devices, the pinned pool, the clock and the tokens
    (devices.py:336-574)."""

    def __init__(
        self,
        clock_mode: ClockMode = ClockMode.WALL,
        pinned_pool_bytes: Optional[int] = None,
        shared_host_bus: bool = False,
        tracer: Optional[Tracer] = None,
        clock: Optional[DeviceClock] = None,
    ):
        self.clock_mode = clock_mode
        self.clock = clock if clock is not None else DeviceClock()
        self._pinned_bytes = pinned_pool_bytes
        self._pinned: Optional[HostPinnedPool] = None
        self.tracer = tracer if tracer is not None else NullTracer()
        self.shared_host_bus = shared_host_bus
        self._devices: dict[int, _Device] = {}
        self._tokens: dict[int, CompletionToken] = {}
        self._peer_enabled: set[tuple[int, int]] = set()
        # hrt_copy_ordered method: 0 copy engine, 1 SM kernel, 2 auto
        self.copy_method = int(os.environ.get("HRT_COPY_METHOD", "2"))

    # -- registration ----------------------------------------------------

    def register_device(self, descriptor: DeviceDescriptor, backend: Any = None) -> int:
        descriptor.validate()
        if descriptor.device_id in self._devices:
            raise HrtError(f"device id {descriptor.device_id} already registered")
        if descriptor.device_type is DeviceType.HOST:
            raise HrtError("the B200 registry manages accelerator devices only")
        n = N.gpu_count()
        if n == 0:
            N.require_gpu(0)
        gpu = descriptor.gpu if descriptor.gpu is not None else _placement(descriptor.device_id, n)
        self._devices[descriptor.device_id] = _Device(descriptor, gpu)
        return descriptor.device_id

    def device(self, device_id: int) -> _Device:
        dev = self._devices.get(device_id)
        if dev is None:
            raise HrtError(f"unknown device {device_id}")
        return dev

    def gpu_of(self, device_id: int) -> int:
        return self.device(device_id).gpu

    @property
    def device_ids(self) -> list[int]:
        return list(self._devices)

    def devices_of_type(self, device_type: DeviceType) -> list[int]:
        return [d for d, dev in self._devices.items()
                if dev.descriptor.device_type is device_type]

    @property
    def pinned_pool(self) -> HostPinnedPool:
        if self._pinned is None:
            self._pinned = HostPinnedPool(self._pinned_bytes)
        return self._pinned

    def enable_peer(self, gpu: int, peer: int) -> bool:
        if gpu == peer or (gpu, peer) in self._peer_enabled:
            return True
        rc = N.lib().hrt_enable_peer_access(gpu, peer)
        if rc == 0:
            self._peer_enabled.add((gpu, peer))
            return True
        return False

    # -- memory ----------------------------------------------------------

    def pool_alloc(self, device_id: int, size: int) -> DeviceAllocation:
        dev = self.device(device_id)
        off, granted, ptr = dev.pool.alloc(size)
        return DeviceAllocation(device_id, off, granted, ALIGNMENT, ptr)

    def pool_free(self, alloc: DeviceAllocation) -> None:
        self.device(alloc.device_id).pool.free(alloc.offset)

    def free_bytes(self, device_id: int) -> int:
        return self.device(device_id).pool.free_bytes

    def region(self, alloc: DeviceAllocation, nbytes: Optional[int] = None) -> DeviceRegion:
        return DeviceRegion(self, alloc, alloc.size if nbytes is None else nbytes)

    # -- async operations ---------------------------------------------------

    def _resolve(self, loc: Location, nbytes: int) -> tuple[int, Optional[int]]:
        """(byte address, device_id or None for host) of a location.  A
        :class:`ForeignAllocation` (another rank's registry, same process)
        resolves to its physical GPU."""
        if isinstance(loc, ForeignAllocation):
            return loc.alloc.ptr, ("gpu", loc.gpu)
        if isinstance(loc, DeviceAllocation):
            self.device(loc.device_id)
            if nbytes > loc.size:
                raise InvalidLocation(f"transfer of {nbytes} B exceeds allocation of {loc.size} B")
            return loc.ptr, loc.device_id
        if isinstance(loc, HostRegion):
            if nbytes > loc.nbytes:
                raise InvalidLocation("transfer exceeds host region")
            if not loc.pooled:
                self.pinned_pool.note_unpinned_use()
            return loc.array.ctypes.data, None
        if isinstance(loc, np.ndarray):
            if not loc.flags["C_CONTIGUOUS"]:
                raise InvalidLocation("host array location must be C-contiguous")
            if nbytes > loc.nbytes:
                raise InvalidLocation("transfer exceeds destination array")
            self.pinned_pool.note_unpinned_use()
            return loc.ctypes.data, None
        raise InvalidLocation(f"unsupported location {type(loc).__name__}")

    def enqueue_transfer(self, src: Location, dst: Location, size: int,
                         wait: Optional[list] = None) -> CompletionToken:
        """Asynchronous copy (devices.py:446-496).  H2D runs on the
        destination's h2d stream, D2H on the source's d2h stream, D2D and
        peer copies on the destination's h2d stream.  ``wait`` tokens become
        GPU-side dependencies.  Host buffers must stay alive until the token
        completes (the runtime's access ops guarantee it)."""
        if size < 0:
            raise InvalidLocation("negative transfer size")
        sp, sd = self._resolve(src, size)
        dp, dd = self._resolve(dst, size)
        if sd is None and dd is None:
            if size:
                ctypes.memmove(dp, sp, size)
            return CompletionToken.completed(TokenKind.TRANSFER)
        if isinstance(dd, tuple):
            raise InvalidLocation("a foreign allocation can only be a transfer source")
        if dd is not None:
            dev = self.device(dd)
            stream = dev.h2d
        else:
            dev = self.device(sd)
            stream = dev.d2h
        t0 = self.clock.now
        peer = 0
        if size:
            g_s = sd[1] if isinstance(sd, tuple) else (self.gpu_of(sd) if sd is not None else None)
            g_d = dev.gpu if dd is not None else None
            if g_s is not None and g_d is not None and g_s != g_d:
                # SM copies need the mapping; without it the copy engine
                # still moves the bytes (staged by the driver)
                peer = 1 if self.enable_peer(g_d, g_s) else 0
        # waits + copy + token in one native call (hrt_copy_ordered); GPU<->GPU
        # copies up to 64 MiB run as an SM pull/push kernel (lower latency
        # than the copy engine there), larger ones on the copy engine
        waits = [t.token_id for t in (wait or ()) if t is not None and t._native]
        tid = ctypes.c_uint64()
        N.call("hrt_copy_ordered", stream.h, ctypes.c_void_p(dp), ctypes.c_void_p(sp),
               ctypes.c_uint64(size), peer, (ctypes.c_uint64 * len(waits))(*waits) if waits else None,
               len(waits), self.copy_method, ctypes.byref(tid))
        token = CompletionToken(tid.value, TokenKind.TRANSFER, dev.device_id)
        self._tokens[token.token_id] = token
        self.clock.track_pending(token)
        if self.tracer.enabled:
            self.tracer.emit("transfer", device=dev.device_id, stream=stream.name, start=t0,
                             end=t0, size=size)
        return token

    def enqueue_kernel(
        self,
        device_id: int,
        kernel_ref: Any,
        args: list,
        thread_dims: Any,
        stream_index: int = 0,
        scratch: Optional[DeviceAllocation] = None,
        label: Optional[str] = None,
        wait: Optional[list] = None,
    ) -> CompletionToken:
        """Launch a registered native kernel (devices.py:502-558) on compute
        stream ``stream_index`` after GPU-side waits on ``wait`` tokens.
        ``args`` are (DeviceAllocation, DeviceRegion) pairs; the body is a
        launcher ``body(views, geometry, scratch, stream)``."""
        dev = self.device(device_id)
        body = kernel_ref.body_for(dev.descriptor.device_type)
        for alloc, _ in args:
            if alloc.device_id != device_id:
                raise InvalidLocation(
                    f"kernel argument lives on device {alloc.device_id}, not {device_id}")
        if not 0 <= stream_index < len(dev.compute_streams):
            raise HrtError(f"stream index {stream_index} out of range")
        stream = dev.compute_streams[stream_index]
        here = stream.h.value
        for t in wait or ():
            if t is not None and t.stream != here:  # same stream: ordered already
                stream.wait(t)
        views = [v for _, v in args]
        t0 = self.clock.now
        try:
            body(views, thread_dims, scratch, stream)
        except Exception as exc:  # launch failure surfaces on the task handle
            token = CompletionToken.completed(TokenKind.KERNEL, device_id)
            token.fail(exc)
            return token
        token = stream.record(TokenKind.KERNEL, device_id)
        self._tokens[token.token_id] = token
        self.clock.track_pending(token)
        if self.tracer.enabled:
            self.tracer.emit("kernel", device=device_id, stream=stream.name, start=t0, end=t0,
                             label=label or kernel_ref.name)
        return token

    def poll(self, token: Union[int, CompletionToken]) -> TokenStatus:
        """Non-blocking status check (devices.py:560-567)."""
        tok = token if isinstance(token, CompletionToken) else self._tokens.get(token)
        if tok is None:
            raise UnknownToken(f"unknown token {token}")
        st = tok.status
        if st is not TokenStatus.PENDING:
            self._tokens.pop(tok.token_id, None)
        return st

    def advance(self) -> Optional[CompletionToken]:
        return self.clock.advance_one()

    @property
    def pinned_pool_misses(self) -> int:
        return self.pinned_pool.misses

    def synchronize(self) -> None:
        for dev in self._devices.values():
            N.call("hrt_device_synchronize", dev.gpu)
