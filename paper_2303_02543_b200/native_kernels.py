"""Native B200 entry points for the task runtime (kernels.py registry).

Each launcher enqueues libhrt_b200 work on the stream the executor picked,
for device-resident views (DeviceRegion).  They restate the reference's
numpy kernel bodies (/root/reference/pkg/src/hrt/bench/jacobi.py and
bench/pingpong.py) as CUDA launches:

* :class:`JacobiUpdate`  — ``_update_body`` (jacobi.py:70-86)
* :class:`HaloPack`      — ``_make_pack_body(face)`` (jacobi.py:102-110)
* :class:`HaloUnpack`    — ``_make_unpack_body(face)`` (jacobi.py:113-124);
  raw-byte wrappers are reinterpreted as float64 like jacobi.py:120-121
* :class:`Touch`         — ping-pong's ``fill_kernel`` (pingpong.py:99-103):
  no bytes change; the executor's argument staging makes the copy VALID
* :class:`Fill`          — set every byte / element of the first view
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .errors import HrtError
from .kernels import NativeKernel

F64 = 8
FACES = [(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1)]


def _ghosted_dims(view, what: str) -> tuple[int, int, int]:
    shape = tuple(view.shape)
    if len(shape) != 3:
        raise HrtError(f"{what}: expected a ghosted (ex+2, ey+2, ez+2) chunk, got {shape}")
    return shape


def _plane(shape, face: int, interior: bool):
    """(element offset, n0, n1, s0, s1) of a face plane of a dense ghosted
    C-order chunk: the boundary-adjacent interior plane (pack source) or the
    ghost plane (unpack target) — jacobi.py:89-99."""
    gx, gy, gz = shape
    strides = (gy * gz, gz, 1)
    axis, side = FACES[face]
    if interior:
        idx = 1 if side == 0 else shape[axis] - 2
    else:
        idx = 0 if side == 0 else shape[axis] - 1
    start = [1, 1, 1]
    start[axis] = idx
    others = [a for a in range(3) if a != axis]
    off = sum(s * st for s, st in zip(start, strides))
    return (off, shape[others[0]] - 2, shape[others[1]] - 2, strides[others[0]],
            strides[others[1]])


def _seg(src, dst, n0, n1, ss0, ss1, ds0, ds1) -> N.HaloSeg:
    g = N.HaloSeg()
    g.src[0] = g.src[1] = src
    g.dst[0] = g.dst[1] = dst
    g.n0, g.n1, g.ss0, g.ss1, g.ds0, g.ds1 = n0, n1, ss0, ss1, ds0, ds1
    return g


class JacobiUpdate(NativeKernel):
    name = "jacobi_update"

    def __init__(self, residual_slot: int = 0):
        self.residual_slot = residual_slot

    def __call__(self, views, geometry, scratch, stream) -> None:
        u, nxt = views
        gx, gy, gz = _ghosted_dims(u, "jacobi_update")
        N.call("hrt_jacobi_chunk_update", stream.h, ctypes.c_void_p(u.ptr),
               ctypes.c_void_p(nxt.ptr), gx - 2, gy - 2, gz - 2,
               ctypes.c_void_p(self.residual_slot))


class HaloPack(NativeKernel):
    def __init__(self, face: int):
        self.face = face
        self.name = f"halo_pack_{face}"

    def __call__(self, views, geometry, scratch, stream) -> None:
        u, halo = views
        shape = _ghosted_dims(u, self.name)
        off, n0, n1, s0, s1 = _plane(shape, self.face, interior=True)
        if halo.nbytes < n0 * n1 * F64:
            raise HrtError(f"{self.name}: halo of {halo.nbytes} B < plane {n0 * n1 * F64} B")
        g = _seg(u.ptr + F64 * off, halo.ptr, n0, n1, s0, s1, n1, 1)
        N.call("hrt_plane_copy", stream.h, ctypes.byref(g))


class HaloUnpack(NativeKernel):
    def __init__(self, face: int):
        self.face = face
        self.name = f"halo_unpack_{face}"

    def __call__(self, views, geometry, scratch, stream) -> None:
        halo, u = views
        shape = _ghosted_dims(u, self.name)
        off, n0, n1, s0, s1 = _plane(shape, self.face, interior=False)
        if halo.nbytes < n0 * n1 * F64:
            raise HrtError(f"{self.name}: wrapper of {halo.nbytes} B < plane {n0 * n1 * F64} B")
        g = _seg(halo.ptr, u.ptr + F64 * off, n0, n1, n1, 1, s0, s1)
        N.call("hrt_plane_copy", stream.h, ctypes.byref(g))


class Touch(NativeKernel):
    name = "touch"

    def __call__(self, views, geometry, scratch, stream) -> None:
        return None


class Fill(NativeKernel):
    """Every byte of the first view := ``value`` (0..255)."""

    name = "fill"

    def __init__(self, value: int = 0):
        self.value = int(value) & 0xFF

    def __call__(self, views, geometry, scratch, stream) -> None:
        v = views[0]
        N.call("hrt_memset_async", stream.h, ctypes.c_void_p(v.ptr), self.value,
               ctypes.c_uint64(v.nbytes))


class Mix(NativeKernel):
    """views [dst] or [src, dst]: dst = dst*7 + src + salt (mod 256)."""

    name = "mix"

    def __init__(self, salt: int = 0):
        self.salt = int(salt) & 0xFF

    def __call__(self, views, geometry, scratch, stream) -> None:
        dst = views[-1]
        src = views[0].ptr if len(views) > 1 else 0
        if len(views) > 1 and views[0].nbytes < dst.nbytes:
            raise HrtError("mix: source smaller than destination")
        N.call("hrt_mix_u8", stream.h, ctypes.c_void_p(dst.ptr), ctypes.c_void_p(src),
               ctypes.c_int64(dst.nbytes), self.salt)


def dtype_of(view) -> np.dtype:
    return np.dtype(getattr(view, "dtype", np.uint8))


class Stamp(NativeKernel):
    """Spin ``ns`` nanoseconds on the GPU and record the kernel's own
    [start, end] %globaltimer interval at device address ``slot`` (two
    uint64): the witness that conflicting tasks never overlap and
    independent ones do (AC-02, test_acceptance.py:67-96).  Touches no view."""

    name = "stamp"

    def __init__(self, slot: int, ns: int = 100_000):
        self.slot = int(slot)
        self.ns = int(ns)

    def __call__(self, views, geometry, scratch, stream) -> None:
        N.call("hrt_spin_stamp", stream.h, ctypes.c_void_p(self.slot), ctypes.c_uint64(self.ns))

