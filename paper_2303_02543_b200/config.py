"""Environment configuration, same variable names as the reference
(/root/reference/pkg/src/hrt/config.py:1-14):

    HRT_STREAMS            compute streams per device (default 5)
    HRT_PINNED_POOL_MB     page-locked staging pool size (default 64)
    HRT_RECV_CACHE_MB      per-device receive slab pool (default 16)
    HRT_DEVICE_AWARE       0/1, device-to-device message payloads
    HRT_GRAPH              0/1, replay the Jacobi step as a CUDA graph (default 1)
"""

from __future__ import annotations

import os


def env_int(name: str, default: int) -> int:
    raw = os.environ.get(name)
    return default if raw in (None, "") else int(raw)


def env_bool(name: str, default: bool = False) -> bool:
    raw = os.environ.get(name)
    if raw in (None, ""):
        return default
    return raw.strip().lower() not in ("0", "false", "no")


def default_compute_streams() -> int:
    return env_int("HRT_STREAMS", 5)


def default_pinned_pool_bytes() -> int:
    return env_int("HRT_PINNED_POOL_MB", 64) << 20


def default_recv_cache_bytes() -> int:
    return env_int("HRT_RECV_CACHE_MB", 16) << 20
