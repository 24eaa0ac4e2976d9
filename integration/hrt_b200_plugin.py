"""B200 backend for the reference ``hrt`` package — the drop-in of
SURVEY.md §8(b), written as the reference-side binding a maintainer would
add to ``hrt`` (it imports the UNMODIFIED reference and libhrt_b200.so
through the C ABI in include/hrt_b200.h; nothing of
``paper_2303_02543_b200``'s Python is used).

Seams (paths relative to /root/reference/pkg/src/hrt):

* ``DeviceBackend`` (devices.py:285-308) -> :class:`B200Backend`: the device
  arena is a ``cudaMalloc`` pool on a B200 (``hrt_pool_create``);
  ``region()`` returns a :class:`DeviceRegion`, which supports what the
  reference does to regions — ``[:] = 0`` (runtime.py:653), ``[:] =
  np.frombuffer(...)`` (comm.py:833, 878), ``.tobytes()`` (comm.py:366,
  547), ``.view(dtype).reshape(dims)`` (runtime.py:296-300) and ``.copy()``
  (jacobi.py:470, pingpong.py:32) — as synchronous H2D/D2H copies.
  ``run_kernel`` is never called: kernel bodies are not executed.
* ``DeviceRegistry`` (devices.py:336-574) -> :class:`B200Registry`:
  ``pool_alloc``/``pool_free`` use the native first fit inside the pool
  (devices.py:89-154 semantics, OutOfDeviceMemory / DoubleFree);
  ``enqueue_transfer`` (446-496) issues a real async copy on the device's
  H2D or D2H stream and also allows device-to-device and peer copies
  (456-457 rejects them in the simulator); ``enqueue_kernel`` (502-558)
  dispatches on the kernel NAME to a native launch (``jacobi_update`` ->
  ``hrt_jacobi_chunk_update``, ``halo_pack_f``/``halo_unpack_f`` ->
  ``hrt_plane_copy``, ping-pong's ``touch`` -> nothing to do) on the
  compute stream the runtime picked; an unknown name yields a FAILED token
  (-> ``TaskFailed``), never a numpy body.
* ``CompletionToken`` (199-222) -> :class:`DeviceToken`: ``status`` is read
  lazily from a CUDA event (``hrt_token_query``) because
  ``Runtime._service_tokens`` reads ``token.status`` directly
  (runtime.py:806-809).
* the clock (225-274) -> :class:`DeviceClock`, a ``WallClock`` whose
  ``advance_one()`` blocks on the oldest outstanding device operation and
  returns its token, so ``Runtime.progress``/``wait`` (runtime.py:503-527)
  and ``drive`` (comm.py:1028-1050) wait for the GPU instead of declaring a
  deadlock.
* the world builder (bench/worlds.py:44-95) -> :func:`b200_worlds`, a
  backend selector: inside it ``make_loopback_world`` /
  ``make_inprocess_tcp_world`` build B200 registries.  ``run_jacobi3d``
  (bench/jacobi.py:281-462) and ``run_pingpong`` (bench/pingpong.py:48-152)
  then run unmodified on the GPUs.

Usage::

    from hrt.bench.jacobi import run_jacobi3d
    from hrt.devices import ClockMode
    with b200_worlds(gpus=[0]):
        report, checksum, field = run_jacobi3d((32, 32, 1), grid=(4, 4, 1), steps=20,
                                               clock=ClockMode.WALL)
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading
from collections import deque
from typing import Optional, Sequence

import numpy as np

from hrt import devices as D
from hrt.bench import worlds as W
from hrt.errors import DoubleFree, HrtError, InvalidLocation, OutOfDeviceMemory
from hrt.runtime import Runtime

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get(
    "HRT_B200_LIB", os.path.join(os.path.dirname(_HERE), "paper_2303_02543_b200", "libhrt_b200.so"))

HRT_E_OOM, HRT_E_DOUBLE_FREE = -2, -3
FACES = [(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1)]  # bench/jacobi.py:41
F64 = 8

_vp, _u64, _i64, _int = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
_P = ctypes.POINTER


class _HaloSeg(ctypes.Structure):  # hrt_halo_seg_t
    _fields_ = [("src", _u64 * 2), ("dst", _u64 * 2), ("n0", _i64), ("n1", _i64),
                ("ss0", _i64), ("ss1", _i64), ("ds0", _i64), ("ds1", _i64)]


_SIGNATURES = {
    "hrt_last_error": (ctypes.c_char_p, []),
    "hrt_device_count": (_int, [_P(_int)]),
    "hrt_enable_peer_access": (_int, [_int, _int]),
    "hrt_pool_create": (_int, [_int, _u64, _P(_vp)]),
    "hrt_pool_alloc": (_int, [_vp, _u64, _P(_u64), _P(_u64), _P(_vp)]),
    "hrt_pool_free": (_int, [_vp, _u64]),
    "hrt_pool_stats": (_int, [_vp, _P(_u64), _P(_u64)]),
    "hrt_pool_base": (_int, [_vp, _P(_vp)]),
    "hrt_pool_destroy": (_int, [_vp]),
    "hrt_stream_create": (_int, [_int, _int, _P(_vp)]),
    "hrt_stream_synchronize": (_int, [_vp]),
    "hrt_stream_destroy": (_int, [_vp, _int]),
    "hrt_token_record": (_int, [_vp, _P(_u64)]),
    "hrt_token_query": (_int, [_u64]),
    "hrt_token_wait": (_int, [_u64]),
    "hrt_token_release": (_int, [_u64]),
    "hrt_copy_async": (_int, [_vp, _vp, _vp, _u64]),
    "hrt_memset_async": (_int, [_vp, _vp, _int, _u64]),
    "hrt_plane_copy": (_int, [_vp, _P(_HaloSeg)]),
    "hrt_jacobi_chunk_update": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
}


class _Lib:
    """ctypes binding of the libhrt_b200.so entry points this backend uses."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise HrtError(f"libhrt_b200.so not found at {path} (build it first)")
        self.dll = ctypes.CDLL(path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(self.dll, name)
            fn.restype, fn.argtypes = res, args
        n = _int()
        if self.dll.hrt_device_count(ctypes.byref(n)) != 0 or n.value < 1:
            raise HrtError("no CUDA device visible: the B200 backend has no CPU fallback")
        self.ngpu = n.value

    def __call__(self, name: str, *args) -> int:
        rc = getattr(self.dll, name)(*args)
        if rc < 0:
            msg = (self.dll.hrt_last_error() or b"").decode()
            exc = {HRT_E_OOM: OutOfDeviceMemory, HRT_E_DOUBLE_FREE: DoubleFree}.get(rc, HrtError)
            raise exc(f"{name}: {msg} (code {rc})")
        return rc


_lib: Optional[_Lib] = None
_lib_lock = threading.Lock()


def lib() -> _Lib:
    global _lib
    with _lib_lock:
        if _lib is None:
            _lib = _Lib()
        return _lib


class _Stream:
    def __init__(self, gpu: int):
        self.gpu = gpu
        h = _vp()
        lib()("hrt_stream_create", gpu, 0, ctypes.byref(h))
        self.h = h.value

    def sync(self) -> None:
        lib()("hrt_stream_synchronize", self.h)


# ---------------------------------------------------------------------------
# tokens and clock

_STATUS = D.CompletionToken.__dict__["status"]  # the base class's slot descriptor


class DeviceToken(D.CompletionToken):
    """CompletionToken whose status follows a CUDA event (devices.py:199-222):
    PENDING until the event completes, then COMPLETE (or FAILED)."""

    __slots__ = ("event",)

    def __init__(self, token_id: int, kind: D.TokenKind, device_id: int, event: int = 0):
        self.event = 0
        super().__init__(token_id, kind, device_id)
        self.event = event

    @property
    def status(self) -> D.TokenStatus:
        st = _STATUS.__get__(self, DeviceToken)
        if st is D.TokenStatus.PENDING and self.event:
            q = lib().dll.hrt_token_query(self.event)
            if q == 1:
                self._settle(self._final)
            elif q != 0:
                self.error = HrtError((lib().dll.hrt_last_error() or b"").decode())
                self._settle(D.TokenStatus.FAILED)
        return _STATUS.__get__(self, DeviceToken)

    @status.setter
    def status(self, value: D.TokenStatus) -> None:
        _STATUS.__set__(self, value)

    def _settle(self, value: D.TokenStatus) -> None:
        _STATUS.__set__(self, value)
        ev, self.event = self.event, 0
        lib().dll.hrt_token_release(ev)

    def wait(self) -> None:
        if self.event:
            lib().dll.hrt_token_wait(self.event)
        _ = self.status


class DeviceClock(D.WallClock):
    """Wall time; ``advance_one()`` waits for the oldest outstanding device
    operation of any registry sharing this clock and returns its token
    (WallClock.advance_one returns None: work there is synchronous)."""

    def __init__(self) -> None:
        super().__init__()
        self._pending: deque = deque()
        self._lock = threading.Lock()

    def track(self, token: DeviceToken) -> None:
        with self._lock:
            self._pending.append(token)

    def advance_one(self) -> Optional[D.CompletionToken]:
        while True:
            with self._lock:
                if not self._pending:
                    return None
                tok = self._pending.popleft()
            if _STATUS.__get__(tok, DeviceToken) is not D.TokenStatus.PENDING:
                continue
            tok.wait()
            return tok

    @property
    def pending_events(self) -> int:
        return len(self._pending)


# ---------------------------------------------------------------------------
# device memory


class DeviceRegion:
    """A window of a B200 pool: what ``DeviceBackend.region`` returns.
    Element access is a synchronous copy (the reference's runtime only
    touches regions whose producers have completed — access ops and task
    retirement order every read and write, runtime.py:414-423, 748-768)."""

    def __init__(self, backend: "B200Backend", ptr: int, nbytes: int, dtype=np.uint8,
                 shape: Optional[tuple] = None):
        self.backend = backend
        self.ptr = int(ptr)
        self.nbytes = int(nbytes)
        self.dtype = np.dtype(dtype)
        self.shape = tuple(shape) if shape is not None else (self.nbytes // self.dtype.itemsize,)

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))

    @property
    def ndim(self) -> int:
        return len(self.shape)

    def view(self, dtype) -> "DeviceRegion":
        dt = np.dtype(dtype)
        if self.nbytes % dt.itemsize:
            raise ValueError("region size is not a multiple of the new itemsize")
        return DeviceRegion(self.backend, self.ptr, self.nbytes, dt, (self.nbytes // dt.itemsize,))

    def reshape(self, *shape) -> "DeviceRegion":
        if len(shape) == 1 and isinstance(shape[0], (tuple, list)):
            shape = tuple(shape[0])
        shape = [int(d) for d in shape]
        if shape.count(-1) == 1:
            known = int(np.prod([d for d in shape if d != -1]))
            shape[shape.index(-1)] = self.size // known if known else 0
        if int(np.prod(shape)) != self.size:
            raise ValueError(f"cannot reshape region of {self.size} elements into {tuple(shape)}")
        return DeviceRegion(self.backend, self.ptr, self.nbytes, self.dtype, tuple(shape))

    def copy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        self.backend.d2h(out, self.ptr, self.nbytes)
        return out

    def __array__(self, dtype=None, copy=None):
        a = self.copy()
        return a if dtype is None else a.astype(dtype)

    def tobytes(self) -> bytes:
        return self.copy().tobytes()

    def __getitem__(self, key):
        return self.copy()[key]

    def __setitem__(self, key, value) -> None:
        whole = (isinstance(key, slice) and key == slice(None)) or key is Ellipsis
        if whole and np.isscalar(value) and value == 0:
            self.backend.memset(self.ptr, 0, self.nbytes)
            return
        if whole:
            src = np.ascontiguousarray(np.broadcast_to(np.asarray(value, dtype=self.dtype),
                                                       self.shape))
        else:  # partial assignment: read, modify, write back
            src = self.copy()
            src[key] = value
        self.backend.h2d(self.ptr, src, self.nbytes)

    def __len__(self) -> int:
        return self.shape[0]

    def __repr__(self) -> str:
        return f"<DeviceRegion gpu{self.backend.gpu} 0x{self.ptr:x} {self.shape} {self.dtype}>"


class _PoolAllocator:
    """FreeListAllocator surface (devices.py:89-154) over the native first
    fit of a B200 pool: granted offsets are arena offsets."""

    def __init__(self, backend: "B200Backend", capacity: int):
        self.backend = backend
        self.capacity = capacity
        self.alignment = D.ALIGNMENT
        self._live: dict[int, int] = {}

    def alloc(self, size: int) -> tuple[int, int]:
        if size <= 0:
            raise HrtError(f"allocation size must be positive, got {size}")
        off, granted, ptr = _u64(), _u64(), _vp()
        lib()("hrt_pool_alloc", self.backend.pool, size, ctypes.byref(off), ctypes.byref(granted),
              ctypes.byref(ptr))
        self._live[off.value] = granted.value
        return off.value, granted.value

    def free(self, offset: int) -> int:
        if offset not in self._live:
            raise DoubleFree(f"offset {offset} is not a live allocation")
        lib()("hrt_pool_free", self.backend.pool, offset)
        return self._live.pop(offset)

    @property
    def live_bytes(self) -> int:
        live, free = _u64(), _u64()
        lib()("hrt_pool_stats", self.backend.pool, ctypes.byref(live), ctypes.byref(free))
        return live.value

    @property
    def free_bytes(self) -> int:
        live, free = _u64(), _u64()
        lib()("hrt_pool_stats", self.backend.pool, ctypes.byref(live), ctypes.byref(free))
        return free.value

    def check(self) -> None:
        assert self.live_bytes + self.free_bytes == self.capacity


class B200Backend(D.GpuSimBackend):
    """One B200 behind a reference device id.  ``device_type`` stays
    GPU_SIM: the Jacobi and ping-pong drivers hard-code it
    (bench/jacobi.py:232,255,262; bench/pingpong.py:121)."""

    device_type = D.DeviceType.GPU_SIM

    def __init__(self, gpu: int):
        super().__init__()
        self.gpu = gpu
        self.pool = None
        self.base = 0
        self.sync_stream: Optional[_Stream] = None
        self.kernel_runs = 0  # numpy bodies executed (must stay 0)

    def attach(self, descriptor: D.DeviceDescriptor) -> None:
        p, b = _vp(), _vp()
        lib()("hrt_pool_create", self.gpu, descriptor.memory_capacity, ctypes.byref(p))
        lib()("hrt_pool_base", p, ctypes.byref(b))
        self.pool, self.base = p.value, b.value
        self.sync_stream = _Stream(self.gpu)
        self.arena = None  # no host arena: bytes live in HBM

    def region(self, alloc: D.DeviceAllocation, nbytes: Optional[int] = None) -> DeviceRegion:
        n = alloc.size if nbytes is None else nbytes
        return DeviceRegion(self, self.base + alloc.offset, n)

    def run_kernel(self, body, views, geometry, scratch) -> None:
        self.kernel_runs += 1
        raise HrtError("B200Backend never runs host kernel bodies")

    # synchronous helpers for DeviceRegion
    def h2d(self, dst: int, src: np.ndarray, nbytes: int) -> None:
        if nbytes:
            lib()("hrt_copy_async", self.sync_stream.h, _vp(dst), _vp(src.ctypes.data), nbytes)
            self.sync_stream.sync()

    def d2h(self, dst: np.ndarray, src: int, nbytes: int) -> None:
        if nbytes:
            lib()("hrt_copy_async", self.sync_stream.h, _vp(dst.ctypes.data), _vp(src), nbytes)
            self.sync_stream.sync()

    def memset(self, dst: int, value: int, nbytes: int) -> None:
        if nbytes:
            lib()("hrt_memset_async", self.sync_stream.h, _vp(dst), value, nbytes)
            self.sync_stream.sync()


# ---------------------------------------------------------------------------
# kernels: the reference's numpy bodies as native launches, keyed by name


def _plane(shape, face: int, interior: bool):
    """(element offset, n0, n1, s0, s1) of the boundary-adjacent interior
    plane (pack source) or the ghost plane (unpack target) of a dense
    ghosted C-order chunk (bench/jacobi.py:89-99)."""
    strides = (shape[1] * shape[2], shape[2], 1)
    axis, side = FACES[face]
    idx = (1 if side == 0 else shape[axis] - 2) if interior else \
        (0 if side == 0 else shape[axis] - 1)
    start = [1, 1, 1]
    start[axis] = idx
    o = [a for a in range(3) if a != axis]
    off = sum(s * st for s, st in zip(start, strides))
    return off, shape[o[0]] - 2, shape[o[1]] - 2, strides[o[0]], strides[o[1]]


def _plane_copy(stream: int, src: int, dst: int, n0, n1, ss0, ss1, ds0, ds1) -> None:
    g = _HaloSeg()
    g.src[0] = g.src[1] = src
    g.dst[0] = g.dst[1] = dst
    g.n0, g.n1, g.ss0, g.ss1, g.ds0, g.ds1 = n0, n1, ss0, ss1, ds0, ds1
    lib()("hrt_plane_copy", stream, ctypes.byref(g))


def _jacobi_update(stream: int, views) -> None:
    """_update_body (bench/jacobi.py:70-86): interior 7-point update in the
    reference's sum order + IEEE /6.0, ghost shell carried u -> nxt."""
    u, nxt = views
    gx, gy, gz = u.shape
    if nxt.shape != u.shape or u.dtype != np.float64:
        raise HrtError(f"jacobi_update: bad views {u!r} {nxt!r}")
    lib()("hrt_jacobi_chunk_update", stream, _vp(u.ptr), _vp(nxt.ptr), gx - 2, gy - 2, gz - 2,
          None)


def _halo_pack(face: int):
    def launch(stream: int, views) -> None:  # bench/jacobi.py:102-110
        u, halo = views
        off, n0, n1, s0, s1 = _plane(u.shape, face, interior=True)
        if halo.nbytes < n0 * n1 * F64:
            raise HrtError(f"halo_pack_{face}: halo of {halo.nbytes} B < plane")
        _plane_copy(stream, u.ptr + F64 * off, halo.ptr, n0, n1, s0, s1, n1, 1)
    return launch


def _halo_unpack(face: int):
    def launch(stream: int, views) -> None:  # bench/jacobi.py:113-124 (raw wrappers too)
        halo, u = views
        off, n0, n1, s0, s1 = _plane(u.shape, face, interior=False)
        if halo.nbytes < n0 * n1 * F64:
            raise HrtError(f"halo_unpack_{face}: wrapper of {halo.nbytes} B < plane")
        _plane_copy(stream, halo.ptr, u.ptr + F64 * off, n0, n1, n1, 1, s0, s1)
    return launch


def _touch(stream: int, views) -> None:
    """pingpong.py:99-103 ``views[0][:] = views[0]``: no bytes change."""


NATIVE_KERNELS = {"jacobi_update": _jacobi_update, "touch": _touch}
for _f in range(6):
    NATIVE_KERNELS[f"halo_pack_{_f}"] = _halo_pack(_f)
    NATIVE_KERNELS[f"halo_unpack_{_f}"] = _halo_unpack(_f)


# ---------------------------------------------------------------------------
# registry


class B200Registry(D.DeviceRegistry):
    """DeviceRegistry on B200s (devices.py:336-574)."""

    def __init__(self, *args, gpu_of: Optional[dict] = None, **kwargs):
        super().__init__(*args, **kwargs)
        self.gpu_of = dict(gpu_of or {})
        self._streams: dict[int, list[_Stream]] = {}
        self._copy_streams: dict[int, tuple[_Stream, _Stream]] = {}
        self.native_launches = 0
        self.copies = {"h2d": 0, "d2h": 0, "d2d": 0, "peer": 0}

    def register_device(self, descriptor: D.DeviceDescriptor,
                        backend: Optional[D.DeviceBackend] = None) -> int:
        if descriptor.device_type is not D.DeviceType.GPU_SIM or backend is not None:
            return super().register_device(descriptor, backend)
        gpu = self.gpu_of.get(descriptor.device_id, 0)
        did = super().register_device(descriptor, B200Backend(gpu))
        dev = self.device(did)
        dev.allocator = _PoolAllocator(dev.backend, descriptor.memory_capacity)
        self._streams[did] = [_Stream(gpu) for _ in range(descriptor.compute_stream_count)]
        self._copy_streams[did] = (_Stream(gpu), _Stream(gpu))
        return did

    def _b200(self, device_id: Optional[int]) -> Optional[B200Backend]:
        if device_id is None:
            return None
        b = self.device(device_id).backend
        return b if isinstance(b, B200Backend) else None

    def _token(self, kind: D.TokenKind, device_id: int, stream: _Stream) -> DeviceToken:
        ev = _u64()
        lib()("hrt_token_record", stream.h, ctypes.byref(ev))
        self._next_token += 1
        tok = DeviceToken(self._next_token, kind, device_id, ev.value)
        self._tokens[tok.token_id] = tok
        if isinstance(self.clock, DeviceClock):
            self.clock.track(tok)
        return tok

    def _address(self, loc, nbytes: int) -> tuple[int, Optional[int]]:
        """(address, device id or None) of a Location (devices.py:418-439)."""
        if isinstance(loc, D.DeviceAllocation):
            if nbytes > loc.size:
                raise InvalidLocation(f"transfer of {nbytes} B exceeds allocation of {loc.size} B")
            b = self._b200(loc.device_id)
            if b is None:
                view, _ = self._resolve(loc, nbytes)
                return view.ctypes.data, None
            return b.base + loc.offset, loc.device_id
        view, _ = self._resolve(loc, nbytes)  # host region / array checks + miss counting
        return view.ctypes.data, None

    def enqueue_transfer(self, src, dst, size: int) -> D.CompletionToken:
        """devices.py:446-496 on the GPU: an async copy on the device's H2D
        (or D2H) stream with a completion token.  Host sources in pageable
        memory are captured when the call returns (the reference copies at
        enqueue); device-to-device and peer copies are allowed."""
        if size < 0:
            raise InvalidLocation("negative transfer size")
        sdev = src.device_id if isinstance(src, D.DeviceAllocation) else None
        ddev = dst.device_id if isinstance(dst, D.DeviceAllocation) else None
        if self._b200(sdev) is None and self._b200(ddev) is None:
            return super().enqueue_transfer(src, dst, size)
        if size == 0:
            tok = DeviceToken(self._next_token + 1, D.TokenKind.TRANSFER, ddev if ddev is not None
                              else sdev)
            self._next_token += 1
            self._tokens[tok.token_id] = tok
            _STATUS.__set__(tok, D.TokenStatus.COMPLETE)
            return tok
        sp, sdev = self._address(src, size)
        dp, ddev = self._address(dst, size)
        device_id = ddev if ddev is not None else sdev
        h2d, d2h = self._copy_streams[device_id]
        stream = h2d if ddev is not None else d2h
        if sdev is not None and ddev is not None:
            gs, gd = self.device(sdev).backend.gpu, self.device(ddev).backend.gpu
            if gs != gd:
                lib()("hrt_enable_peer_access", gd, gs)
                self.copies["peer"] += 1
            else:
                self.copies["d2d"] += 1
        else:
            self.copies["h2d" if ddev is not None else "d2h"] += 1
        lib()("hrt_copy_async", stream.h, _vp(dp), _vp(sp), size)
        tok = self._token(D.TokenKind.TRANSFER, device_id, stream)
        self.tracer.emit("transfer", device=device_id, stream="h2d" if stream is h2d else "d2h",
                         start=self.clock.now, end=self.clock.now, size=size)
        return tok

    def enqueue_kernel(self, device_id: int, kernel_ref, args, thread_dims, stream_index: int = 0,
                       scratch=None, label: Optional[str] = None) -> D.CompletionToken:
        """devices.py:502-558: the kernel's native entry point, by name, on
        compute stream ``stream_index``; the body is never executed."""
        if self._b200(device_id) is None:
            return super().enqueue_kernel(device_id, kernel_ref, args, thread_dims, stream_index,
                                          scratch, label)
        dev = self.device(device_id)
        kernel_ref.body_for(dev.descriptor.device_type)  # the reference's entry-point check
        for alloc, _ in args:
            if alloc.device_id != device_id:
                raise InvalidLocation(
                    f"kernel argument lives on device {alloc.device_id}, not {device_id}")
        if not 0 <= stream_index < len(dev.compute_streams):
            raise HrtError(f"stream index {stream_index} out of range")
        stream = self._streams[device_id][stream_index]
        launch = NATIVE_KERNELS.get(kernel_ref.name)
        error = None
        if launch is None:
            error = HrtError(f"kernel {kernel_ref.name!r} has no B200 entry point")
        else:
            try:
                launch(stream.h, [v for _, v in args])
                self.native_launches += 1
            except Exception as exc:  # recorded, surfaces on the task handle
                error = exc
        tok = self._token(D.TokenKind.KERNEL, device_id, stream)
        if error is not None:
            tok._final = D.TokenStatus.FAILED
            tok.error = error
        self.tracer.emit("kernel", device=device_id, stream=dev.compute_streams[stream_index].name,
                         start=self.clock.now, end=self.clock.now,
                         label=label or kernel_ref.name)
        return tok


# ---------------------------------------------------------------------------
# world builder: the backend selector


_ACTIVE: list = [[]]  # registries built inside the innermost b200_worlds() block


def _build_rank_runtime(cfg: W.WorldConfig, rank: int, clock, tracer=None,
                        gpus: Sequence[int] = (0,)) -> Runtime:
    """bench/worlds.py:44-75 with B200 registries: device rank*100+j maps
    to GPU gpus[(rank*devices_per_rank + j) % len(gpus)]."""
    gpu_of = {W.device_id_for(rank, j): gpus[(rank * cfg.devices_per_rank + j) % len(gpus)]
              for j in range(cfg.devices_per_rank)}
    registry = B200Registry(clock_mode=cfg.clock, shared_host_bus=cfg.shared_host_bus,
                            tracer=tracer, clock=clock, gpu_of=gpu_of)
    for j in range(cfg.devices_per_rank):
        registry.register_device(D.DeviceDescriptor(
            device_id=W.device_id_for(rank, j), device_type=D.DeviceType.GPU_SIM,
            memory_capacity=cfg.capacity, compute_stream_count=cfg.streams,
            transfer_latency=cfg.latency, transfer_bandwidth=cfg.bandwidth,
            clock_mode=cfg.clock))
    if cfg.with_host_device:
        registry.register_device(D.DeviceDescriptor(
            device_id=W.device_id_for(rank, 99), device_type=D.DeviceType.HOST,
            memory_capacity=cfg.host_capacity, compute_stream_count=cfg.streams,
            clock_mode=cfg.clock))
    _ACTIVE[-1].append(registry)
    return Runtime(registry)


@contextlib.contextmanager
def b200_worlds(gpus: Optional[Sequence[int]] = None):
    """Inside the block every world the reference builds (make_loopback_world,
    make_inprocess_tcp_world) runs on B200s; yields the list of registries
    built so far (for counters).  The clock is a DeviceClock whatever
    ClockMode is passed."""
    gpus = list(gpus) if gpus is not None else list(range(lib().ngpu))
    saved = (W.build_rank_runtime, W.make_clock)
    W.build_rank_runtime = lambda cfg, rank, clock, tracer=None: _build_rank_runtime(
        cfg, rank, clock, tracer, gpus)
    W.make_clock = lambda cfg: DeviceClock()
    built: list = []
    _ACTIVE.append(built)
    try:
        yield built
    finally:
        W.build_rank_runtime, W.make_clock = saved
        _ACTIVE.remove(built)
