"""Message wire format (/root/reference/pkg/src/hrt/wire.py:1-138): a fixed
64-byte little-endian header, byte-compatible with the reference.

    0 magic "HRTM" | 4 version | 5 kind | 6 inline | 7 source device type
    8 handler_id u32 | 12 target_rank u32 | 16 target_index u64
    24 payload_size u64 | 32 correlation_id u64 | 40 element_size u32
    44/48/52 dims u32 x3 | 56 reserved (8 zero bytes)

A payload travels inline when header + payload fit in 512 bytes, otherwise
as one data frame ``u64 correlation id + payload``.  For device-aware frames
this backend puts a *device locator* (:class:`DeviceLocator`) in the data
frame instead of the payload bytes: the bytes go GPU->GPU (CUDA IPC + peer
copy) and the header stays the reference's.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from enum import IntEnum

from .errors import ProtocolError

MAGIC = b"HRTM"
VERSION = 1
HEADER_SIZE = 64
INLINE_LIMIT = 512
MAX_INLINE_PAYLOAD = INLINE_LIMIT - HEADER_SIZE
NO_DEVICE = 0xFF
_HDR = struct.Struct("<4s4B2I3Q4I8s")
assert _HDR.size == HEADER_SIZE


class MsgKind(IntEnum):
    HANDLER = 1
    HANDLER_HETERO_META = 2
    PUT_META = 3
    GET_REQ = 4
    ACK = 5


@dataclass
class MessageHeader:
    msg_kind: MsgKind
    handler_id: int = 0
    target_rank: int = 0
    target_index: int = 0
    payload_size: int = 0
    inline_flag: bool = False
    correlation_id: int = 0
    element_size: int = 0
    dims: tuple = (0, 0, 0)
    source_device_type: int = NO_DEVICE
    version: int = VERSION

    def encode(self) -> bytes:
        d0, d1, d2 = self.dims
        return _HDR.pack(MAGIC, self.version, int(self.msg_kind), int(bool(self.inline_flag)),
                         self.source_device_type, self.handler_id, self.target_rank,
                         self.target_index, self.payload_size, self.correlation_id,
                         self.element_size, d0, d1, d2, bytes(8))


def decode_header(data: bytes) -> MessageHeader:
    """Parse and validate (wire.py:90-134): magic, version, kind, inline flag
    and zero reserved bytes; ProtocolError otherwise."""
    if len(data) < HEADER_SIZE:
        raise ProtocolError(f"header truncated: {len(data)} bytes")
    (magic, version, kind, inline, sdt, handler, rank, index, size, corr, esize, d0, d1, d2,
     reserved) = _HDR.unpack_from(data)
    if magic != MAGIC:
        raise ProtocolError(f"bad magic {magic!r}")
    if version != VERSION:
        raise ProtocolError(f"unsupported version {version}")
    try:
        k = MsgKind(kind)
    except ValueError:
        raise ProtocolError(f"unknown message kind {kind}") from None
    if inline not in (0, 1):
        raise ProtocolError(f"bad inline flag {inline}")
    if reserved != bytes(8):
        raise ProtocolError("reserved header bytes must be zero")
    return MessageHeader(k, handler, rank, index, size, bool(inline), corr, esize, (d0, d1, d2),
                         sdt, version)


def should_inline(payload_size: int) -> bool:
    """wire.py:137-138"""
    return HEADER_SIZE + payload_size <= INLINE_LIMIT


# ---------------------------------------------------------------------------
# device locator (this backend's data-frame body for device-aware sends)

_LOC = struct.Struct("<4sII64sQQQ")
LOC_MAGIC = b"HRTL"


@dataclass
class DeviceLocator:
    """Where the payload lives on the sender: a CUDA IPC handle of the
    sender's device arena, the byte offset inside it, the size, the sender's
    GPU ordinal, the arena's address in the sender and the sender's pid (a
    receiver in the same process uses the address directly)."""

    ipc_handle: bytes
    offset: int
    size: int
    gpu: int
    arena_base: int = 0
    pid: int = 0

    def encode(self) -> bytes:
        return _LOC.pack(LOC_MAGIC, self.gpu, self.pid, self.ipc_handle, self.offset, self.size,
                         self.arena_base)

    @staticmethod
    def decode(data: bytes) -> "DeviceLocator":
        if len(data) != _LOC.size:
            raise ProtocolError(f"device locator of {len(data)} bytes")
        magic, gpu, pid, handle, off, size, base = _LOC.unpack(data)
        if magic != LOC_MAGIC:
            raise ProtocolError("bad device locator magic")
        return DeviceLocator(handle, off, size, gpu, base, pid)
