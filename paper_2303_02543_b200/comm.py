"""Distributed layer on B200s: mobile objects, handler invocation and
device-to-device message transfer (/root/reference/pkg/src/hrt/comm.py).

Kept: mobile objects addressed by (owner rank, index) and the reference
exchange (comm.py:206-256), handler ids in registration order, per-source
FIFO handler queues run round-robin (comm.py:899-926), every send holding
an access operation on its object in the runtime's dependency graph so
transfers never overlap conflicting tasks and objects live until
transmission completes (comm.py:12-14, 322-466), wrapper objects on the
receive side with a per-device receive slab cache (comm.py:94-131, 650-697),
and the three send paths:

* **direct** (``device_aware`` transport; comm.py:331-372, 826-839): no host
  staging.  The frame carries a *device locator* (the source allocation and
  the event of its producer) instead of bytes; the receiver copies the
  payload GPU->GPU (cudaMemcpyPeerAsync over NVLink, or D2D on one GPU) into
  a receive slab, ordered on the device after the producer, and runs the
  handler before the bytes land (tasks on the wrapper are ordered behind the
  copy, as in the reference).  The sender's read access completes with the
  copy.
* **staged** (comm.py:419-466, 840-859): D2H into pinned host memory, bytes
  in the frame, H2D upload on the receiver (two staging copies).
* **inline** (<= 512 B with the 64-byte header, wire.py:137-138): one frame.

Two transports.  The in-process loopback fabric (transport.py:62-101):
ranks share a process and frames are Python objects.  Byte transports
(:class:`~paper_2303_02543_b200.transport.TcpTransport`, transport.py:
104-278): frames are the reference's 64-byte headers plus data frames
(wire.py); a device-aware send puts a :class:`DeviceLocator` (CUDA IPC
handle of the sender's arena + offset) in the data frame, the receiver
copies GPU->GPU from the mapped arena and answers with a copy ACK (header
kind ACK, source device type 1) that completes the sender's read access.
Either way device payloads never touch the host on the direct path.
"""

from __future__ import annotations

import ctypes
import os
import struct
import time
from collections import deque
from dataclasses import dataclass
from typing import Callable, Optional, Union

import numpy as np

from .config import default_recv_cache_bytes
from .devices import DeviceAllocation, DeviceType, ForeignAllocation, HostRegion, TokenStatus
from .errors import DeadlockError, HrtError, NotOwner, ProtocolError, TransportClosed
from .objects import AccessMode, CopyInfo, CopyState, HeteroObject
from . import _native as N
from .runtime import AccessOp, Runtime
from .transport import FT_DATA, FT_HEADER
from .wire import HEADER_SIZE, DeviceLocator, MessageHeader, MsgKind, decode_header, should_inline

NONE_INDEX = 0xFFFFFFFFFFFFFFFF
_CORR = struct.Struct("<Q")
_DEVICE_SRC = 1  # header source_device_type of device-locator frames and their ACKs


@dataclass(frozen=True)
class MobileRef:
    owner_rank: int
    local_index: int


@dataclass(frozen=True)
class GlobalObjectId:
    owner_rank: int
    object_id: int


class MobileObject:
    __slots__ = ("index", "state", "device_hint")

    def __init__(self, index: int, state: bytes, device_hint: Optional[int] = None):
        self.index = index
        self.state = bytearray(state)
        self.device_hint = device_hint


class HandlerContext:
    __slots__ = ("comm", "src_rank", "mobile", "arg")

    def __init__(self, comm, src_rank, mobile, arg):
        self.comm = comm
        self.src_rank = src_rank
        self.mobile = mobile
        self.arg = arg


@dataclass
class CommStats:
    sends: int = 0
    inline_sends: int = 0
    split_sends: int = 0
    staging_copies: int = 0
    device_copies: int = 0
    handlers_run: int = 0
    puts: int = 0
    gets: int = 0
    wrapper_reuses: int = 0
    recv_cache_hits: int = 0
    recv_cache_misses: int = 0


class ReceiveCache:
    """Per-device slabs reserved for incoming payloads (comm.py:94-131)."""

    def __init__(self, runtime: Runtime, capacity: int, slab: int = 1 << 20):
        self.runtime = runtime
        self.capacity = capacity
        self.slab = slab
        self._free: dict[int, list[DeviceAllocation]] = {}
        self._owned: dict[int, set[int]] = {}

    def _install(self, device_id: int) -> None:
        if device_id in self._free:
            return
        self._free[device_id] = []
        self._owned[device_id] = set()
        if self.capacity < self.slab:
            return
        try:
            base = self.runtime.registry.pool_alloc(device_id, self.capacity)
        except HrtError:
            return
        for i in range(self.capacity // self.slab):
            a = DeviceAllocation(device_id, base.offset + i * self.slab, self.slab,
                                 ptr=base.ptr + i * self.slab)
            self._free[device_id].append(a)
            self._owned[device_id].add(a.offset)

    def acquire(self, device_id: int, nbytes: int) -> Optional[DeviceAllocation]:
        self._install(device_id)
        if nbytes <= self.slab and self._free[device_id]:
            return self._free[device_id].pop()
        return None

    def release(self, alloc: DeviceAllocation) -> None:
        self._free[alloc.device_id].append(alloc)

    def owns(self, alloc: DeviceAllocation) -> bool:
        return alloc.offset in self._owned.get(alloc.device_id, set())


# ---------------------------------------------------------------------------
# transport


class LoopbackFabric:
    """Shared per-pair FIFO mailboxes of one in-process world."""

    def __init__(self, world_size: int):
        self.world_size = world_size
        self.queues = {(s, d): deque() for s in range(world_size) for d in range(world_size)}

    def endpoint(self, rank: int, device_aware: bool = False) -> "LoopbackTransport":
        return LoopbackTransport(self, rank, device_aware)


class LoopbackTransport:
    def __init__(self, fabric: LoopbackFabric, rank: int, device_aware: bool = False):
        self._fabric = fabric
        self.rank = rank
        self.world_size = fabric.world_size
        self.device_aware = device_aware
        self._closed = False

    def send(self, dst: int, frame) -> None:
        if self._closed:
            raise TransportClosed("loopback endpoint is closed")
        if not 0 <= dst < self.world_size:
            raise HrtError(f"unknown target rank {dst}")
        self._fabric.queues[(self.rank, dst)].append(frame)

    def poll(self):
        out = []
        for src in range(self.world_size):
            q = self._fabric.queues[(src, self.rank)]
            while q:
                out.append((src, q.popleft()))
        return out

    def flushed(self) -> bool:
        return True

    def close(self) -> None:
        self._closed = True


# ---------------------------------------------------------------------------


class _Outgoing:
    __slots__ = ("dst", "ready", "frame", "op", "label")

    def __init__(self, dst: int, label: str):
        self.dst = dst
        self.ready = False
        self.frame = None
        self.op: Optional[AccessOp] = None
        self.label = label


@dataclass
class _Locator:
    """Where a direct-path payload lives: the sender's newest copy."""

    registry: object
    alloc: Optional[DeviceAllocation]     # device source (None: host or zeros)
    host: Optional[np.ndarray]            # host source bytes view
    token: object                         # producer event of the source copy
    on_copied: Callable                   # sender callback(copy_token)
    ipc: Optional[DeviceLocator] = None   # device source in another process


class Comm:
    """One rank's endpoint of the distributed runtime."""

    def __init__(self, transport: LoopbackTransport, runtime: Runtime,
                 recv_cache_bytes: Optional[int] = None, recv_slab_bytes: int = 1 << 20):
        self.transport = transport
        self.runtime = runtime
        self.rank = transport.rank
        self.world_size = transport.world_size
        self.stats = CommStats()
        cache = recv_cache_bytes if recv_cache_bytes is not None else default_recv_cache_bytes()
        self.recv_cache = ReceiveCache(runtime, cache, recv_slab_bytes)
        runtime._cache_release = self.recv_cache.release
        self._handlers: list[Callable] = []
        self._mobiles: list[MobileObject] = []
        self._outgoing: dict[int, deque] = {}
        self._hq: dict[int, deque] = {}
        self._rr = 0
        self._recv_rr = 0
        self._peer_counts: dict[int, int] = {}
        self._exchange_started = False
        self._closed = False
        self._inflight = 0
        self._pending_gets: dict[int, tuple] = {}
        self._next_corr = 0
        self._bytes = getattr(transport, "bytes_frames", False)
        self._pending_in: dict = {}
        self._await_ack: dict = {}
        self._ipc_maps: dict = {}
        self._acks: set = set()
        self._h_exchange = self.register_handler(self._handle_exchange)

    # -- registration / world setup ----------------------------------------

    def register_handler(self, fn: Callable) -> int:
        """Next handler id; registration order must match on every rank."""
        self._handlers.append(fn)
        return len(self._handlers) - 1

    def create_mobile_object(self, state: bytes = b"", device_hint: Optional[int] = None) -> MobileRef:
        m = MobileObject(len(self._mobiles), state, device_hint)
        self._mobiles.append(m)
        return MobileRef(self.rank, m.index)

    def mobile(self, ref: MobileRef) -> MobileObject:
        if ref.owner_rank != self.rank:
            raise NotOwner(f"mobile object owned by rank {ref.owner_rank}, not {self.rank}")
        return self._mobiles[ref.local_index]

    def resolve(self, ref: MobileRef) -> bytes:
        return bytes(self.mobile(ref).state)

    def begin_exchange(self) -> None:
        if self._exchange_started:
            return
        self._exchange_started = True
        for r in range(self.world_size):
            self._send_bytes(r, self._h_exchange, len(self._mobiles).to_bytes(4, "little"))

    def exchange_complete(self) -> bool:
        return len(self._peer_counts) == self.world_size

    def collect_refs(self) -> list[list[MobileRef]]:
        return [[MobileRef(r, i) for i in range(self._peer_counts[r])]
                for r in range(self.world_size)]

    def _handle_exchange(self, mobile, arg: bytes, ctx: HandlerContext) -> None:
        self._peer_counts[ctx.src_rank] = int.from_bytes(arg[:4], "little")

    def global_id(self, obj: HeteroObject) -> GlobalObjectId:
        return GlobalObjectId(self.rank, obj.object_id)

    # -- sending ---------------------------------------------------------------

    def _check(self, rank: int, handler_id: int) -> None:
        if self._closed:
            raise TransportClosed("communication layer is shut down")
        if not 0 <= rank < self.world_size:
            raise HrtError(f"unknown target rank {rank}")
        if not 0 <= handler_id < len(self._handlers):
            raise HrtError(f"unknown handler id {handler_id}")

    def _queue(self, entry: _Outgoing) -> None:
        self._outgoing.setdefault(entry.dst, deque()).append(entry)

    def _send_bytes(self, dst: int, handler_id: int, data: bytes, index: int = NONE_INDEX) -> None:
        e = _Outgoing(dst, "handler")
        e.frame = ("bytes", handler_id, index, bytes(data))
        e.ready = True
        self.stats.sends += 1
        if should_inline(len(data)):
            self.stats.inline_sends += 1
        else:
            self.stats.split_sends += 1
        self._queue(e)

    def mp_send(self, target: MobileRef, handler_id: int,
                payload: Union[bytes, bytearray, memoryview, HeteroObject, None] = None) -> None:
        """Invoke ``handler_id`` on the target mobile object with an optional
        byte payload or data object (comm.py:303-316)."""
        self._check(target.owner_rank, handler_id)
        if payload is None or isinstance(payload, (bytes, bytearray, memoryview)):
            self._send_bytes(target.owner_rank, handler_id, bytes(payload or b""),
                             target.local_index)
            return
        self._send_object(target.owner_rank, handler_id, payload, target.local_index)

    @staticmethod
    def _meta(obj: HeteroObject):
        return obj.element_size, tuple(obj.dims), obj.dtype

    def _send_object(self, dst: int, handler_id: int, obj: HeteroObject, index: int) -> None:
        obj.check_not_destroyed()
        self.stats.sends += 1
        rt = self.runtime
        meta = self._meta(obj)

        if self.transport.device_aware:
            e = _Outgoing(dst, "hetero_direct")
            self.stats.split_sends += 1

            def granted_direct(r: Runtime, op: AccessOp) -> None:
                r._tick(obj)
                valid = obj.valid_devices()
                if valid:
                    # prefer a copy already on the destination's GPU side is
                    # unknown here; take the first VALID device copy
                    ci = obj.copies[valid[0]]
                    loc = _Locator(r.registry, ci.allocation, None, ci.token, None)
                elif obj.host_state is CopyState.VALID:
                    loc = _Locator(r.registry, None, obj.host_region.array[: obj.total_size],
                                   None, None)
                else:
                    loc = _Locator(r.registry, None, None, None, None)
                wait = list(op.wait_tokens)

                def copied(tok) -> None:
                    if tok is None:
                        r.complete_access(op)
                    else:
                        r.access_launched(op, tok)

                loc.on_copied = copied
                e.frame = ("hetero", handler_id, index, meta, obj.total_size, loc, wait)
                e.ready = True

            e.op = rt.register_access(obj, AccessMode.READ, granted_direct, label="send",
                                      gpu_ordered=True)
            self._queue(e)
            return

        # staged / inline: newest bytes to (pinned) host first
        inline = should_inline(obj.total_size)
        e = _Outgoing(dst, "hetero_inline" if inline else "hetero_staged")
        if inline:
            self.stats.inline_sends += 1
        else:
            self.stats.split_sends += 1

        def granted_staged(r: Runtime, op: AccessOp) -> None:
            r._tick(obj)

            def ready(_tok=None) -> None:
                data = r._ensure_host_region(obj).array[: obj.total_size].tobytes()
                obj.host_state = CopyState.VALID
                e.frame = ("staged", handler_id, index, meta, data)
                e.ready = True
                r.complete_access(op)

            if obj.host_state is CopyState.VALID:
                ready()
                return
            valid = obj.valid_devices()
            region = r._ensure_host_region(obj)
            if not valid:
                region.array[: obj.total_size] = 0
                ready()
                return
            ci = obj.copies[valid[0]]
            self.stats.staging_copies += 1
            tok = r.registry.enqueue_transfer(ci.allocation, region, obj.total_size,
                                              wait=[ci.token] if ci.token else None)
            r._watch(tok, ready)

        e.op = rt.register_access(obj, AccessMode.READ, granted_staged, label="send")
        self._queue(e)

    # -- put / get (comm.py:471-645) ----------------------------------------

    def hetero_put(self, gid: GlobalObjectId, source, completion_handler_id: int) -> None:
        """Overwrite a (possibly remote) object with the source bytes; the
        completion handler fires on the owner."""
        self._check(gid.owner_rank, completion_handler_id)
        self.stats.puts += 1
        if isinstance(source, HeteroObject):
            src = source
            rt = self.runtime

            def granted(r: Runtime, op: AccessOp) -> None:
                valid = src.valid_devices()
                if valid:
                    ci = src.copies[valid[0]]
                    loc = _Locator(r.registry, ci.allocation, None, ci.token, None)
                elif src.host_state is CopyState.VALID:
                    loc = _Locator(r.registry, None, src.host_region.array[: src.total_size],
                                   None, None)
                else:
                    loc = _Locator(r.registry, None, None, None, None)
                loc.on_copied = (lambda tok: r.complete_access(op) if tok is None
                                 else r.access_launched(op, tok))
                e.frame = ("put", completion_handler_id, gid.object_id, src.total_size, loc,
                           list(op.wait_tokens))
                e.ready = True

            e = _Outgoing(gid.owner_rank, "put_obj")
            e.op = rt.register_access(src, AccessMode.READ, granted, label="put", gpu_ordered=True)
            self._queue(e)
        else:
            data = bytes(source)
            e = _Outgoing(gid.owner_rank, "put_bytes")
            e.frame = ("put", completion_handler_id, gid.object_id, len(data),
                       _Locator(None, None, np.frombuffer(data, np.uint8), None, lambda t: None),
                       [])
            e.ready = True
            self._queue(e)

    def hetero_get(self, gid: GlobalObjectId, destination: HeteroObject,
                   completion_handler_id: int) -> None:
        """Fetch a (possibly remote) object's newest bytes into a local one;
        the completion handler fires here once they land."""
        self._check(gid.owner_rank, completion_handler_id)
        destination.check_not_destroyed()
        self.stats.gets += 1
        self._next_corr += 1
        corr = self._next_corr
        self._pending_gets[corr] = (destination, completion_handler_id)
        e = _Outgoing(gid.owner_rank, "get_req")
        e.frame = ("get", completion_handler_id, gid.object_id, destination.total_size, corr)
        e.ready = True
        self._queue(e)

    # -- receiving -----------------------------------------------------------

    def _choose_device(self, mobile: Optional[MobileObject]) -> Optional[int]:
        if mobile is not None and mobile.device_hint is not None:
            return mobile.device_hint
        reg = self.runtime.registry
        cands = reg.devices_of_type(DeviceType.GPU_SIM)
        if not cands:
            return None
        d = cands[self._recv_rr % len(cands)]
        self._recv_rr += 1
        return d

    def _alloc_for_receive(self, device_id: int, nbytes: int):
        slab = self.recv_cache.acquire(device_id, nbytes)
        if slab is not None:
            self.stats.recv_cache_hits += 1
            return slab, True
        self.stats.recv_cache_misses += 1
        return self.runtime.registry.pool_alloc(device_id, nbytes), False

    def _make_wrapper(self, meta, size: int) -> HeteroObject:
        esize, dims, dtype = meta
        rt = self.runtime
        if dtype is not None:
            obj = HeteroObject(rt.new_uid(), dims, dtype=dtype)
        else:
            obj = HeteroObject(rt.new_uid(), dims, esize)
        rt.adopt_object(obj)
        return obj

    def _device_copy(self, device_id: int, dst: DeviceAllocation, loc: _Locator, size: int,
                     wait: list):
        """Payload -> dst on device_id, ordered after the producer; returns
        the copy token (None when nothing needed copying)."""
        reg = self.runtime.registry
        waits = list(wait) + ([loc.token] if loc.token is not None else [])
        if loc.ipc is not None:  # another process's device memory, mapped over CUDA IPC
            self.stats.device_copies += 1
            src = ForeignAllocation(DeviceAllocation(-1, 0, size, ptr=self._ipc_ptr(loc.ipc)),
                                    loc.ipc.gpu)
            return reg.enqueue_transfer(src, dst, size, wait=waits)
        if loc.alloc is not None:
            self.stats.device_copies += 1
            src = loc.alloc
            if loc.registry is not reg:  # another rank's device memory (same process)
                src = ForeignAllocation(loc.alloc, loc.registry.gpu_of(loc.alloc.device_id))
            return reg.enqueue_transfer(src, dst, size, wait=waits)
        if loc.host is not None:
            self.stats.staging_copies += 1
            return reg.enqueue_transfer(np.ascontiguousarray(loc.host), dst, size, wait=waits)
        dev = reg.device(device_id)
        from . import _native as N

        for t in waits:
            dev.h2d.wait(t)
        N.call("hrt_memset_async", dev.h2d.h, ctypes.c_void_p(dst.ptr), 0, ctypes.c_uint64(size))
        return dev.h2d.record(device_id=device_id)

    def _on_frame(self, src: int, frame) -> None:
        kind = frame[0]
        rt = self.runtime
        if kind == "bytes":
            _, hid, index, data = frame
            mobile = self._mobiles[index] if index != NONE_INDEX else None
            self._enqueue_handler(src, hid, mobile, data)
        elif kind == "hetero":
            _, hid, index, meta, size, loc, wait = frame
            mobile = self._mobiles[index] if index != NONE_INDEX else None
            wrapper = self._make_wrapper(meta, size)
            device = self._choose_device(mobile)
            alloc, slab = self._alloc_for_receive(device, size)
            ci = CopyInfo(alloc, CopyState.ABSENT, cache_slab=slab)
            wrapper.copies[device] = ci

            def granted(r: Runtime, op: AccessOp) -> None:
                tok = self._device_copy(device, alloc, loc, size, wait + op.wait_tokens)
                ci.catch_up(tok)   # the wrapper's first bytes (written flips on landing)
                r.access_launched(op, tok)
                # ``written`` flips once the bytes have landed (comm.py:837)
                r._watch(tok, lambda t: setattr(wrapper, "written", True))
                loc.on_copied(tok)

            rt.register_access(wrapper, AccessMode.WRITE, granted, label="recv", gpu_ordered=True)
            # handler may run before the payload lands; tasks on the wrapper
            # are ordered behind the receive (comm.py:743-746)
            self._enqueue_handler(src, hid, mobile, wrapper)
        elif kind == "staged":
            _, hid, index, meta, data = frame
            mobile = self._mobiles[index] if index != NONE_INDEX else None
            wrapper = self._make_wrapper(meta, len(data))
            device = self._choose_device(mobile)

            def granted_s(r: Runtime, op: AccessOp) -> None:
                region = r._ensure_host_region(wrapper)
                region.array[: wrapper.total_size] = np.frombuffer(data, dtype=np.uint8)
                wrapper.host_state = CopyState.VALID
                wrapper.written = True
                if device is None:
                    r.complete_access(op)
                    return
                alloc, slab = self._alloc_for_receive(device, wrapper.total_size)
                ci = CopyInfo(alloc, CopyState.ABSENT, cache_slab=slab)
                wrapper.copies[device] = ci
                self.stats.staging_copies += 1
                tok = r.registry.enqueue_transfer(region, alloc, wrapper.total_size)
                ci.catch_up(tok)   # the wrapper's first bytes (written flips on landing)
                r.access_launched(op, tok)

            rt.register_access(wrapper, AccessMode.WRITE, granted_s, label="recv",
                               gpu_ordered=True)
            self._enqueue_handler(src, hid, mobile, wrapper)
        elif kind == "put":
            _, hid, oid, size, loc, wait = frame
            obj = rt._objects.get(oid)
            if obj is None:
                raise ProtocolError(f"put targets unknown object {oid}")
            if size != obj.total_size:
                raise ProtocolError(f"put size mismatch: payload {size} B vs object "
                                    f"{obj.total_size} B")
            self._apply_put(src, hid, obj, loc, wait)
        elif kind == "get":
            _, hid, oid, size, corr = frame
            obj = rt._objects.get(oid)
            if obj is None:
                raise ProtocolError(f"get targets unknown object {oid}")
            if size != obj.total_size:
                raise ProtocolError(f"get size mismatch: destination {size} B vs object "
                                    f"{obj.total_size} B")

            def granted_g(r: Runtime, op: AccessOp) -> None:
                valid = obj.valid_devices()
                if valid:
                    ci = obj.copies[valid[0]]
                    loc = _Locator(r.registry, ci.allocation, None, ci.token, None)
                elif obj.host_state is CopyState.VALID:
                    loc = _Locator(r.registry, None, obj.host_region.array[: obj.total_size],
                                   None, None)
                else:
                    loc = _Locator(r.registry, None, None, None, None)
                loc.on_copied = (lambda tok: r.complete_access(op) if tok is None
                                 else r.access_launched(op, tok))
                e = _Outgoing(src, "get_resp")
                e.frame = ("get_resp", hid, corr, size, loc, list(op.wait_tokens))
                e.ready = True
                self._queue(e)

            rt.register_access(obj, AccessMode.READ, granted_g, label="get", gpu_ordered=True)
        elif kind == "get_resp":
            _, hid, corr, size, loc, wait = frame
            dest, handler = self._pending_gets.pop(corr)
            self._apply_put(src, handler, dest, loc, wait)
        else:
            raise ProtocolError(f"unknown frame kind {kind!r}")

    def _apply_put(self, src: int, hid: int, obj: HeteroObject, loc: _Locator, wait) -> None:
        """Overwrite ``obj`` (comm.py:863-894): into its newest device copy
        (or first allocated one) on the device path, else its host copy."""
        rt = self.runtime

        def granted(r: Runtime, op: AccessOp) -> None:
            allocated = sorted(d for d, c in obj.copies.items() if c.allocation is not None)
            valid = [d for d in allocated if obj.copies[d].state is CopyState.VALID]
            target = valid[0] if valid else (allocated[0] if allocated else None)
            if target is None:
                cands = r.registry.devices_of_type(DeviceType.GPU_SIM)
                target = cands[0]
                obj.copies[target] = CopyInfo(r.registry.pool_alloc(target, obj.total_size))
            ci = obj.copies[target]
            tok = self._device_copy(target, ci.allocation, loc, obj.total_size,
                                    list(wait) + op.wait_tokens)
            obj.publish(target, tok)
            r.access_launched(op, tok)
            loc.on_copied(tok)
            self._enqueue_handler(src, hid, None, obj)

        rt.register_access(obj, AccessMode.WRITE, granted, label="put_recv", gpu_ordered=True)

    # -- handlers / progress ---------------------------------------------------

    def _enqueue_handler(self, src: int, handler_id: int, mobile, arg) -> None:
        self._hq.setdefault(src, deque()).append((handler_id, mobile, arg))

    def _run_handlers(self) -> int:
        sources = sorted(self._hq)
        if not sources:
            return 0
        start = self._rr % len(sources)
        order = sources[start:] + sources[:start]
        budget = {s: len(self._hq[s]) for s in order}
        ran = 0
        progressed = True
        while progressed:
            progressed = False
            for s in order:
                q = self._hq.get(s)
                if q and budget[s] > 0:
                    hid, mobile, arg = q.popleft()
                    budget[s] -= 1
                    self._handlers[hid](mobile, arg, HandlerContext(self, s, mobile, arg))
                    self.stats.handlers_run += 1
                    ran += 1
                    progressed = True
        self._rr += 1
        for s in [s for s, q in self._hq.items() if not q]:
            del self._hq[s]
        return ran

    def network_progress(self) -> int:
        work = 0
        for dst in sorted(self._outgoing):
            q = self._outgoing[dst]
            while q and q[0].ready:
                e = q.popleft()
                if self._bytes:
                    for ftype, data in self._encode(e.dst, e.frame):
                        self.transport.send(e.dst, ftype, data)
                else:
                    self.transport.send(e.dst, e.frame)
                work += 1
        if self._bytes:
            for src, ftype, data in self.transport.poll():
                self._decode(src, ftype, data)
                work += 1
        else:
            for src, frame in self.transport.poll():
                self._on_frame(src, frame)
                work += 1
        work += self._run_handlers()
        return work

    # -- byte transports: reference headers + data frames -------------------

    def _arena_locator(self, reg, alloc: DeviceAllocation) -> DeviceLocator:
        dev = reg.device(alloc.device_id)
        pool = dev.pool
        handle = getattr(pool, "_ipc_handle", None)
        if handle is None:
            buf = ctypes.create_string_buffer(64)
            N.call("hrt_ipc_get_handle", ctypes.c_void_p(pool.base), buf)
            handle = pool._ipc_handle = buf.raw
        return DeviceLocator(handle, alloc.ptr - pool.base, alloc.size, dev.gpu, pool.base,
                             os.getpid())

    def _ipc_ptr(self, loc: DeviceLocator) -> int:
        if loc.pid == os.getpid():  # same process: the arena address is ours too
            return loc.arena_base + loc.offset
        base = self._ipc_maps.get(loc.ipc_handle)
        if base is None:
            p = ctypes.c_void_p()
            dev_ids = self.runtime.registry.device_ids
            gpu = self.runtime.registry.gpu_of(dev_ids[0]) if dev_ids else 0
            N.call("hrt_ipc_open_handle", gpu, ctypes.create_string_buffer(loc.ipc_handle, 64),
                   ctypes.byref(p))
            base = self._ipc_maps[loc.ipc_handle] = p.value
        return base + loc.offset

    def _host_bytes(self, loc: _Locator, size: int) -> bytes:
        """Payload bytes of a locator (device sources are read back)."""
        if loc.alloc is not None:
            if loc.token is not None:
                loc.token.wait()
            return np.asarray(loc.registry.region(loc.alloc, size).copy()).tobytes()
        if loc.host is not None:
            return np.ascontiguousarray(loc.host).tobytes()[:size]
        return bytes(size)

    def _frames(self, hdr: MessageHeader, body: bytes):
        hdr.payload_size = len(body) if hdr.payload_size == 0 else hdr.payload_size
        if hdr.inline_flag:
            return [(FT_HEADER, hdr.encode() + body)]
        return [(FT_HEADER, hdr.encode()), (FT_DATA, _CORR.pack(hdr.correlation_id) + body)]

    def _encode(self, dst: int, frame):
        kind = frame[0]
        self._next_corr += 1
        corr = self._next_corr
        if kind == "bytes":
            _, hid, index, data = frame
            h = MessageHeader(MsgKind.HANDLER, hid, dst, index, len(data), should_inline(len(data)),
                              corr)
            return self._frames(h, data)
        if kind in ("staged", "hetero"):
            esize, dims, _dtype = frame[3]
            d3 = tuple(dims) + (0,) * (3 - len(dims))
            if kind == "staged":
                data = frame[4]
                h = MessageHeader(MsgKind.HANDLER_HETERO_META, frame[1], dst, frame[2], len(data),
                                  should_inline(len(data)), corr, esize, d3)
                return self._frames(h, data)
            _, hid, index, meta, size, loc, wait = frame
            for t in wait:
                t.wait()
            if loc.alloc is None:  # host-resident or untouched source: ship bytes
                data = self._host_bytes(loc, size)
                loc.on_copied(None)
                h = MessageHeader(MsgKind.HANDLER_HETERO_META, hid, dst, index, size,
                                  should_inline(size), corr, esize, d3)
                return self._frames(h, data)
            if loc.token is not None:
                loc.token.wait()  # the receiver copies as soon as the frame arrives
            dl = self._arena_locator(loc.registry, loc.alloc)
            dl.size = size
            self._await_ack[corr] = loc.on_copied
            h = MessageHeader(MsgKind.HANDLER_HETERO_META, hid, dst, index, size, False, corr,
                              esize, d3, source_device_type=1)
            return [(FT_HEADER, h.encode()), (FT_DATA, _CORR.pack(corr) + dl.encode())]
        if kind == "put":
            _, hid, oid, size, loc, wait = frame
            for t in wait:
                t.wait()
            data = self._host_bytes(loc, size)
            loc.on_copied(None)
            h = MessageHeader(MsgKind.PUT_META, hid, dst, oid, size, should_inline(size), corr)
            return self._frames(h, data)
        if kind == "get":
            _, hid, oid, size, gcorr = frame
            return [(FT_HEADER, MessageHeader(MsgKind.GET_REQ, hid, dst, oid, size, False,
                                              gcorr).encode())]
        if kind == "get_resp":
            _, hid, gcorr, size, loc, wait = frame
            for t in wait:
                t.wait()
            data = self._host_bytes(loc, size)
            loc.on_copied(None)
            h = MessageHeader(MsgKind.PUT_META, hid, dst, NONE_INDEX, size, should_inline(size),
                              gcorr)
            return self._frames(h, data)
        if kind == "ack":  # copy completion of a device-locator message
            return [(FT_HEADER, MessageHeader(MsgKind.ACK, 0, dst, 0, 0, False, frame[1],
                                              source_device_type=_DEVICE_SRC).encode())]
        raise ProtocolError(f"cannot encode frame kind {kind!r}")

    def _decode(self, src: int, ftype: int, data: bytes) -> None:
        if ftype == FT_HEADER:
            hdr = decode_header(data)
            body = data[HEADER_SIZE:HEADER_SIZE + hdr.payload_size] if hdr.inline_flag else None
            if hdr.msg_kind is MsgKind.ACK:
                if hdr.source_device_type != _DEVICE_SRC:  # shutdown barrier (comm.py:718)
                    self._acks.add(src)
                    return
                cb = self._await_ack.pop(hdr.correlation_id, None)
                if cb is None:
                    raise ProtocolError(f"ACK for unknown message {hdr.correlation_id}")
                cb(None)
                return
            if hdr.msg_kind is MsgKind.GET_REQ:
                self._on_frame(src, ("get", hdr.handler_id, hdr.target_index, hdr.payload_size,
                                     hdr.correlation_id))
                return
            if body is None:
                self._pending_in[(src, hdr.correlation_id)] = hdr
                return
            self._deliver(src, hdr, body)
        else:
            (corr,) = _CORR.unpack_from(data)
            hdr = self._pending_in.pop((src, corr), None)
            if hdr is None:
                raise ProtocolError(f"data frame with unmatched correlation id {corr} from {src}")
            self._deliver(src, hdr, data[8:])

    def _deliver(self, src: int, hdr: MessageHeader, body: bytes) -> None:
        k = hdr.msg_kind
        if k is MsgKind.HANDLER:
            if len(body) != hdr.payload_size:
                raise ProtocolError("payload size does not match the header")
            self._on_frame(src, ("bytes", hdr.handler_id, hdr.target_index, body))
            return
        dims = tuple(d for d in hdr.dims if d > 0)
        if not dims:
            dims = (max(1, hdr.payload_size // max(1, hdr.element_size)),)
        meta = (hdr.element_size or 1, dims, None)
        if k is MsgKind.HANDLER_HETERO_META:
            if hdr.source_device_type == _DEVICE_SRC:  # device locator: GPU->GPU copy, then ACK
                dl = DeviceLocator.decode(body)
                corr = hdr.correlation_id

                def copied(tok, src=src, corr=corr):
                    if tok is None:
                        self._queue_ack(src, corr)
                    else:
                        self.runtime._watch(tok, lambda t: self._queue_ack(src, corr))

                loc = _Locator(None, None, None, None, copied, ipc=dl)
                self._on_frame(src, ("hetero", hdr.handler_id, hdr.target_index, meta,
                                     hdr.payload_size, loc, []))
            else:
                self._on_frame(src, ("staged", hdr.handler_id, hdr.target_index, meta, body))
            return
        if k is MsgKind.PUT_META:
            loc = _Locator(None, None, np.frombuffer(body, np.uint8), None, lambda t: None)
            if hdr.target_index == NONE_INDEX:
                self._on_frame(src, ("get_resp", hdr.handler_id, hdr.correlation_id,
                                     hdr.payload_size, loc, []))
            else:
                self._on_frame(src, ("put", hdr.handler_id, hdr.target_index, hdr.payload_size,
                                     loc, []))
            return
        raise ProtocolError(f"unexpected message kind {k!r}")

    def _queue_ack(self, dst: int, corr: int) -> None:
        e = _Outgoing(dst, "ack")
        e.frame = ("ack", corr)
        e.ready = True
        self._queue(e)

    def progress(self, advance: bool = True) -> int:
        work = self.runtime.progress(advance=False)
        work += self.network_progress()
        if work == 0 and advance:
            work += self.runtime.progress(advance=True)
        return work

    def _outgoing_pending(self) -> bool:
        return any(q for q in self._outgoing.values())

    @property
    def quiescent(self) -> bool:
        return (not self._outgoing_pending() and not self._hq and not self._pending_gets
                and not self._await_ack and not self._pending_in)

    def flush(self, timeout: float = 60.0) -> None:
        drive([self], until=lambda: not self._outgoing_pending(), timeout=timeout)

    def _send_barrier(self) -> None:
        self._next_corr += 1
        hdr = MessageHeader(MsgKind.ACK, 0, self.rank, 0, 0, False, self._next_corr)
        for r in range(self.world_size):
            if r != self.rank:
                self.transport.send(r, FT_HEADER, hdr.encode())

    def _barrier_done(self) -> bool:
        return self._acks >= set(range(self.world_size)) - {self.rank} and self.transport.flushed()

    def shutdown(self, barrier: Optional[bool] = None, timeout: float = 60.0) -> None:
        """Flush, then close (comm.py:1003-1025).  With ``barrier`` (default
        for byte transports) every rank first waits for the copy ACKs of its
        device-locator sends, then sends a barrier ACK to each peer and waits
        for one from each, so no peer closes while others expect traffic."""
        if self._closed:
            return
        self.flush(timeout)
        if barrier is None:
            barrier = self._bytes
        if barrier and self.world_size > 1:
            drive([self], until=lambda: not self._await_ack and not self._outgoing_pending(),
                  timeout=timeout)
            self._send_barrier()
            drive([self], until=self._barrier_done, timeout=timeout)
        self._closed = True
        self.transport.close()


def drive(comms: list[Comm], until: Callable[[], bool], timeout: float = 120.0) -> None:
    """Advance in-process ranks together until ``until()`` holds
    (comm.py:1028-1050).  When no rank can make host-side progress, block on
    the oldest outstanding device event of any rank; deadlock only when
    nothing is in flight anywhere."""
    deadline = time.monotonic() + timeout
    # over sockets, bytes can be in flight in the kernel (or in another
    # process) with nothing to do here: wait for them until the deadline
    # (busy-poll for a few ms after the last useful work: a sleep costs the
    # kernel's timer slack, ~50 us, on every message of a round trip)
    patient = any(c._bytes for c in comms)
    busy_since = time.monotonic()
    while not until():
        work = 0
        for c in comms:
            work += c.progress(advance=False)
        if work:
            busy_since = time.monotonic()
            continue
        for c in comms:
            work += c.runtime.progress(advance=True)
            if work:
                break
        if work:
            busy_since = time.monotonic()
            continue
        now = time.monotonic()
        if patient and now <= deadline:
            if now - busy_since > 5e-3:
                time.sleep(100e-6)
            continue
        state = "; ".join(
            f"rank {c.rank}: {c.runtime.debug_state()} outgoing="
            f"{[(d, [e.label + ('+' if e.ready else '-') for e in q][:4]) for d, q in c._outgoing.items() if q]}"
            f" handlers={sum(len(q) for q in c._hq.values())}" for c in comms)
        if time.monotonic() > deadline:
            raise DeadlockError(f"drive timed out ({state})")
        raise DeadlockError(f"no progress possible across ranks ({state})")


def exchange_all(comms: list[Comm]) -> list[list[MobileRef]]:
    for c in comms:
        c.begin_exchange()
    drive(comms, until=lambda: all(c.exchange_complete() for c in comms))
    return comms[0].collect_refs()


def shutdown_all(comms: list[Comm], timeout: float = 60.0) -> None:
    drive(comms, until=lambda: all(c.quiescent for c in comms), timeout=timeout)
    for c in comms:
        c.runtime.synchronize()
    if any(c._bytes for c in comms) and len(comms) > 1:  # in-process byte world: joint barrier
        for c in comms:
            c._send_barrier()
        drive(comms, until=lambda: all(c._barrier_done() for c in comms), timeout=timeout)
    for c in comms:
        c.shutdown(barrier=False, timeout=timeout)
