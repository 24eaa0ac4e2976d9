"""Byte transport and the Comm byte protocol over localhost TCP, CPU only
(the reference's transport tests: pkg/tests/test_transport.py,
test_comm_tcp.py).  Ranks run in this process with empty device registries:
handler messages, the exchange, framing (inline vs header + data frame),
malformed input and the shutdown barrier."""

import socket
import struct

import pytest

from paper_2303_02543_b200.comm import Comm, drive, exchange_all, shutdown_all
from paper_2303_02543_b200.devices import DeviceRegistry
from paper_2303_02543_b200.errors import HrtError, ProtocolError, TransportClosed
from paper_2303_02543_b200.runtime import Runtime
from paper_2303_02543_b200.transport import FT_DATA, FT_HEADER, TcpTransport
from paper_2303_02543_b200.wire import (HEADER_SIZE, MAX_INLINE_PAYLOAD, MessageHeader, MsgKind,
                                        decode_header)
from paper_2303_02543_b200.worlds import _free_ports


def _endpoints(n):
    peers = [f"127.0.0.1:{p}" for p in _free_ports(n)]
    ts = [TcpTransport(r, peers) for r in range(n)]
    for _ in range(20000):
        if all([t.establish() for t in ts]):
            return ts
    raise AssertionError("endpoints did not connect")


def _poll_until(ts, want, limit=200000):
    got = {t.rank: [] for t in ts}
    for _ in range(limit):
        for t in ts:
            got[t.rank].extend(t.poll())
        if all(len(got[r]) >= want.get(r, 0) for r in got):
            return got
    raise AssertionError(f"frames missing: {({r: len(v) for r, v in got.items()})}")


def test_tcp_frames_fifo_and_large():
    ts = _endpoints(3)
    try:
        big = bytes(range(256)) * (16 << 10)  # 4 MiB: many partial socket sends
        for i in range(5):
            ts[0].send(2, FT_HEADER, b"m%d" % i)
        ts[0].send(2, FT_DATA, big)
        ts[1].send(2, FT_HEADER, b"")
        ts[2].send(2, FT_HEADER, b"self")
        got = _poll_until(ts, {2: 8})[2]
        from0 = [(f, d) for s, f, d in got if s == 0]
        assert [d for f, d in from0[:5]] == [b"m%d" % i for i in range(5)]
        assert from0[5] == (FT_DATA, big)
        assert (1, FT_HEADER, b"") in got and (2, FT_HEADER, b"self") in got
        assert all(t.flushed() for t in ts)
    finally:
        for t in ts:
            t.close()
    with pytest.raises(TransportClosed):
        ts[0].send(1, FT_HEADER, b"x")


def test_tcp_rejects_bad_hello_and_rank():
    peers = [f"127.0.0.1:{p}" for p in _free_ports(2)]
    t0 = TcpTransport(0, peers)
    try:
        host, port = peers[0].split(":")
        s = socket.create_connection((host, int(port)))
        s.sendall(struct.pack("<4sI", b"XXXX", 1))
        for _ in range(2000):
            t0.establish()
        assert not t0.ready
        with pytest.raises(HrtError):
            t0.send(5, FT_HEADER, b"")
        s.close()
    finally:
        t0.close()


def _comms(n, **kw):
    ts = _endpoints(n)
    return [Comm(t, Runtime(DeviceRegistry()), **kw) for t in ts]


def test_comm_over_tcp_handlers_inline_and_split():
    comms = _comms(3)
    got = {c.rank: [] for c in comms}
    for c in comms:
        c._h = c.register_handler(
            lambda m, arg, ctx, c=c: got[c.rank].append((ctx.src_rank, m.index, bytes(arg))))
        c.create_mobile_object(b"a")
        c.create_mobile_object(b"b")
    refs = exchange_all(comms)
    assert [len(r) for r in refs] == [2, 2, 2]
    small = b"s" * MAX_INLINE_PAYLOAD          # exactly the inline limit
    large = bytes(range(256)) * 40             # header + data frame
    comms[0].mp_send(refs[1][1], comms[0]._h, small)
    comms[0].mp_send(refs[2][0], comms[0]._h, large)
    comms[2].mp_send(refs[1][0], comms[2]._h, b"")
    comms[1].mp_send(refs[1][1], comms[1]._h, large)   # to itself
    drive(comms, until=lambda: len(got[1]) == 3 and len(got[2]) == 1, timeout=30)
    assert sorted(got[1]) == sorted([(0, 1, small), (2, 0, b""), (1, 1, large)])
    assert got[2] == [(0, 0, large)]
    assert comms[0].stats.inline_sends >= 1 and comms[0].stats.split_sends >= 1
    shutdown_all(comms, timeout=30)   # barrier ACKs over the sockets
    assert all(c._acks == set(range(3)) - {c.rank} for c in comms)


def test_comm_wire_bytes_are_reference_headers():
    """A Comm rank talking to a raw endpoint: what goes on the wire is the
    reference's header (kind HANDLER, handler id, target index, inline flag)
    and, above the inline limit, a data frame ``u64 corr + payload``."""
    ts = _endpoints(2)
    c0 = Comm(ts[0], Runtime(DeviceRegistry()))
    raw = ts[1]
    h = c0.register_handler(lambda *a: None)
    from paper_2303_02543_b200.comm import MobileRef

    c0.mp_send(MobileRef(1, 7), h, b"tiny")
    c0.mp_send(MobileRef(1, 3), h, b"x" * 1000)
    frames = []
    for _ in range(200000):
        c0.progress()
        frames.extend(raw.poll())
        if len(frames) == 3:
            break
    assert [f for _, f, _ in frames] == [FT_HEADER, FT_HEADER, FT_DATA]
    h1 = decode_header(frames[0][2])
    assert (h1.msg_kind, h1.handler_id, h1.target_index, h1.payload_size, h1.inline_flag) == \
        (MsgKind.HANDLER, h, 7, 4, True)
    assert frames[0][2][HEADER_SIZE:] == b"tiny"
    h2 = decode_header(frames[1][2])
    assert (h2.target_index, h2.payload_size, h2.inline_flag) == (3, 1000, False)
    (corr,) = struct.unpack_from("<Q", frames[2][2])
    assert corr == h2.correlation_id and frames[2][2][8:] == b"x" * 1000
    c0.shutdown(barrier=False)
    raw.close()


def test_comm_rejects_malformed_frames():
    ts = _endpoints(2)
    c1 = Comm(ts[1], Runtime(DeviceRegistry()))
    c1.register_handler(lambda *a: None)
    try:
        ts[0].send(1, FT_DATA, struct.pack("<Q", 99) + b"orphan")
        with pytest.raises(ProtocolError, match="unmatched"):
            for _ in range(200000):
                c1.progress()
        bad = bytearray(MessageHeader(MsgKind.HANDLER, 1, 1, 0, 0, True, 5).encode())
        bad[0:4] = b"NOPE"
        ts[0].send(1, FT_HEADER, bytes(bad))
        with pytest.raises(ProtocolError, match="magic"):
            for _ in range(200000):
                c1.progress()
    finally:
        ts[0].close()
        ts[1].close()
