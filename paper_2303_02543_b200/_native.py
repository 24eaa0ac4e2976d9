"""ctypes binding of libhrt_b200.so (include/hrt_b200.h).

There is no CPU fallback: importing works anywhere (so the CPU test suite
can check exports and the host-side allocator), but every device call goes
through the CUDA library and raises if it is missing or no GPU is present.
"""

from __future__ import annotations

import ctypes
import os

from .errors import raise_for

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhrt_b200.so")

c_int, c_i64, c_u64, c_f, c_d = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_double
c_void_p, c_char_p = ctypes.c_void_p, ctypes.c_char_p
P = ctypes.POINTER


class ChunkLayout(ctypes.Structure):
    """hrt_chunk_layout_t"""

    _fields_ = [("ndim", ctypes.c_int32), ("pad_", ctypes.c_int32), ("ext", c_i64 * 3),
                ("stride", c_i64 * 3), ("origin", c_i64), ("elems", c_i64)]


class HaloSeg(ctypes.Structure):
    """hrt_halo_seg_t"""

    _fields_ = [("src", c_u64 * 2), ("dst", c_u64 * 2), ("n0", c_i64), ("n1", c_i64),
                ("ss0", c_i64), ("ss1", c_i64), ("ds0", c_i64), ("ds1", c_i64)]


class Push(ctypes.Structure):
    """hrt_push_t"""

    _fields_ = [("ptr", (c_u64 * 2) * 4), ("stride", c_i64 * 4)]


class Side(ctypes.Structure):
    """hrt_side_t"""

    _fields_ = [("w", c_u64 * 2), ("e", c_u64 * 2)]


class VPush(ctypes.Structure):
    """hrt_vpush_t"""

    _fields_ = [("ptr", (c_u64 * 2) * 6)]


class RemoteSeg(ctypes.Structure):
    """hrt_remote_seg_t"""

    _fields_ = [("buf", c_u64 * 2), ("count", c_i64), ("peer", ctypes.c_int32),
                ("kind", ctypes.c_int32)]


# name -> (restype, argtypes); every symbol include/hrt_b200.h declares
SIGNATURES = {
    "hrt_last_error": (c_char_p, []),
    "hrt_version": (c_int, []),
    "hrt_device_count": (c_int, [P(c_int)]),
    "hrt_device_info": (c_int, [c_int, c_char_p, c_int, P(c_int), P(c_u64), P(c_int), P(c_int)]),
    "hrt_enable_peer_access": (c_int, [c_int, c_int]),
    "hrt_device_synchronize": (c_int, [c_int]),
    "hrt_pointer_device": (c_int, [c_void_p, P(c_int)]),
    "hrt_fl_create": (c_int, [c_u64, c_u64, P(c_void_p)]),
    "hrt_fl_alloc": (c_int, [c_void_p, c_u64, P(c_u64), P(c_u64)]),
    "hrt_fl_free": (c_int, [c_void_p, c_u64, P(c_u64)]),
    "hrt_fl_stats": (c_int, [c_void_p, P(c_u64), P(c_u64), P(c_u64)]),
    "hrt_fl_check": (c_int, [c_void_p]),
    "hrt_fl_destroy": (None, [c_void_p]),
    "hrt_pool_create": (c_int, [c_int, c_u64, P(c_void_p)]),
    "hrt_pool_alloc": (c_int, [c_void_p, c_u64, P(c_u64), P(c_u64), P(c_void_p)]),
    "hrt_pool_free": (c_int, [c_void_p, c_u64]),
    "hrt_pool_stats": (c_int, [c_void_p, P(c_u64), P(c_u64)]),
    "hrt_pool_base": (c_int, [c_void_p, P(c_void_p)]),
    "hrt_pool_destroy": (c_int, [c_void_p]),
    "hrt_stream_create": (c_int, [c_int, c_int, P(c_void_p)]),
    "hrt_stream_wrap": (c_int, [c_int, c_void_p, P(c_void_p)]),
    "hrt_stream_handle": (c_void_p, [c_void_p]),
    "hrt_stream_destroy": (c_int, [c_void_p, c_int]),
    "hrt_stream_synchronize": (c_int, [c_void_p]),
    "hrt_token_record": (c_int, [c_void_p, P(c_u64)]),
    "hrt_token_query": (c_int, [c_u64]),
    "hrt_token_wait": (c_int, [c_u64]),
    "hrt_stream_wait_token": (c_int, [c_void_p, c_u64]),
    "hrt_token_elapsed_ms": (c_int, [c_u64, c_u64, P(c_f)]),
    "hrt_token_release": (c_int, [c_u64]),
    "hrt_host_alloc": (c_int, [c_u64, P(c_void_p)]),
    "hrt_host_free": (c_int, [c_void_p]),
    "hrt_host_register": (c_int, [c_void_p, c_u64]),
    "hrt_host_unregister": (c_int, [c_void_p]),
    "hrt_copy_async": (c_int, [c_void_p, c_void_p, c_void_p, c_u64]),
    "hrt_bytes_equal": (c_int, [c_void_p, c_void_p, c_void_p, c_u64, P(c_int)]),
    "hrt_copy_sm_async": (c_int, [c_void_p, c_void_p, c_void_p, c_u64, c_int]),
    "hrt_copy_peer_async": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_u64]),
    "hrt_copy_ordered": (c_int, [c_void_p, c_void_p, c_void_p, c_u64, c_int, P(c_u64), c_int,
                                 c_int, P(c_u64)]),
    "hrt_copy2d_async": (c_int, [c_void_p, c_void_p, c_u64, c_void_p, c_u64, c_u64, c_u64]),
    "hrt_memset_async": (c_int, [c_void_p, c_void_p, c_int, c_u64]),
    "hrt_jacobi_plan_create": (c_int, [c_int, P(ChunkLayout), c_int, P(c_u64), P(HaloSeg), c_int,
                                       P(c_void_p)]),
    "hrt_jacobi_plan_set_remote": (c_int, [c_void_p, c_void_p, P(RemoteSeg), c_int, P(HaloSeg),
                                           c_int]),
    "hrt_jacobi_plan_set_rows": (c_int, [c_void_p, c_i64]),
    "hrt_jacobi_plan_set_offsets": (c_int, [c_void_p, P(c_i64)]),
    "hrt_jacobi_plan_set_push": (c_int, [c_void_p, c_void_p]),
    "hrt_jacobi_plan_invalidate_ghosts": (c_int, [c_void_p]),
    "hrt_jacobi_plan_set_split": (c_int, [c_void_p, c_void_p]),
    "hrt_jacobi_plan_set_ipc": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_u64]),
    "hrt_jacobi_plan_ipc_error": (c_int, [c_void_p, P(c_int)]),
    "hrt_jacobi_plan_set_persistent": (c_int, [c_void_p, P(ctypes.c_int32), c_u64]),
    "hrt_jacobi_plan_error": (c_int, [c_void_p, P(c_int)]),
    "hrt_jacobi_plan_set_sides": (c_int, [c_void_p, c_void_p]),
    "hrt_jacobi_plan_set_vpush": (c_int, [c_void_p, c_void_p]),
    "hrt_jacobi_plan_wave_counters": (c_int, [c_void_p, P(c_u64), P(c_i64)]),
    "hrt_jacobi_plan_vw2_counters": (c_int, [c_void_p, P(c_u64), P(c_i64)]),
    "hrt_jacobi_plan_set_vw2_remote": (c_int, [c_void_p, P(c_u64), P(c_u64), P(ctypes.c_int32)]),
    "hrt_jacobi_plan_range": (c_int, [c_void_p, P(c_u64)]),
    "hrt_jacobi_plan_two_step": (c_int, [c_void_p, P(c_int)]),
    "hrt_jacobi_plan_set_tiling_chunks": (c_int, [c_void_p, c_i64]),
    "hrt_jacobi_plan_set_fuse2": (c_int, [c_void_p, c_int]),
    "hrt_jacobi_plan_tiling": (c_int, [c_void_p, P(c_i64), P(c_i64), P(c_int)]),
    "hrt_jacobi_plan_set_wave2_remote": (c_int, [c_void_p, P(c_u64), P(c_u64), P(ctypes.c_int32)]),
    "hrt_jacobi_plan_set_wave2_nbr9": (c_int, [c_void_p, P(ctypes.c_int32), P(ctypes.c_int32),
                                              P(c_u64), P(c_u64)]),
    "hrt_jacobi_plan_set_wave_ipc": (c_int, [c_void_p, P(ctypes.c_int32), P(ctypes.c_int32),
                                             P(c_u64), c_int, c_u64]),
    "hrt_ipc_get_handle": (c_int, [c_void_p, c_char_p]),
    "hrt_ipc_open_handle": (c_int, [c_int, c_char_p, P(c_void_p)]),
    "hrt_ipc_close_handle": (c_int, [c_void_p]),
    "hrt_jacobi_plan_field_copy": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_int,
                                           c_int]),
    "hrt_jacobi_plan_set_variant": (c_int, [c_void_p, c_int]),
    "hrt_jacobi_plan_set_nonneg": (c_int, [c_void_p, c_int]),
    "hrt_jacobi_plan_step": (c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "hrt_jacobi_plan_update": (c_int, [c_void_p, c_void_p, c_int, c_void_p]),
    "hrt_jacobi_plan_halo": (c_int, [c_void_p, c_void_p, c_int]),
    "hrt_jacobi_plan_run": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p, c_int]),
    "hrt_jacobi_plan_run_timed": (c_int, [c_void_p, c_void_p, c_i64, c_i64, c_void_p, P(c_d),
                                          P(c_d), P(c_d)]),
    "hrt_jacobi_plan_destroy": (c_int, [c_void_p]),
    "hrt_halo_copy": (c_int, [c_void_p, c_void_p, c_int, c_int, c_i64]),
    "hrt_plane_copy": (c_int, [c_void_p, P(HaloSeg)]),
    "hrt_jacobi_chunk_update": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_i64, c_i64,
                                        c_void_p]),
    "hrt_jacobi_ghost_fill": (c_int, [c_void_p, c_void_p, P(ChunkLayout), c_int, c_d]),
    "hrt_np_sum": (c_int, [c_void_p, c_void_p, c_i64, P(c_d)]),
    "hrt_div6_sweep": (c_int, [c_void_p, c_u64, c_i64, c_int, P(c_u64), P(c_d)]),
    "hrt_mix_u8": (c_int, [c_void_p, c_void_p, c_void_p, c_i64, c_int]),
    "hrt_spin_stamp": (c_int, [c_void_p, c_void_p, c_u64]),
    "hrt_nccl_unique_id": (c_int, [c_char_p]),
    "hrt_nccl_init": (c_int, [c_int, c_int, c_int, c_char_p, P(c_void_p)]),
    "hrt_nccl_destroy": (c_int, [c_void_p]),
    "hrt_nccl_exchange": (c_int, [c_void_p, c_void_p, P(RemoteSeg), c_int, c_int]),
    "hrt_nccl_allreduce_max_u64": (c_int, [c_void_p, c_void_p, c_void_p, c_i64]),
    "hrt_nccl_allreduce_sum_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_i64]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libhrt_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2303_02543_b200.build` "
                "(the B200 backend has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().hrt_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        raise_for(rc, f"{what}: {last_error()}" if what else last_error())


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


_gpu_count = None


def gpu_count() -> int:
    """Visible CUDA devices (0 when the driver reports none)."""
    global _gpu_count
    if _gpu_count is None:
        n = c_int(0)
        rc = lib().hrt_device_count(ctypes.byref(n))
        _gpu_count = n.value if rc == 0 else 0
    return _gpu_count


def require_gpu(gpu: int = 0) -> None:
    n = gpu_count()
    if n == 0:
        raise RuntimeError("no CUDA device visible: the B200 backend has no CPU fallback "
                           f"({last_error()})")
    if not 0 <= gpu < n:
        raise RuntimeError(f"GPU {gpu} not visible ({n} devices)")
