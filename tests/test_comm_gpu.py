"""Message path and task-protocol Jacobi on B200s: mp_send (direct device
copies vs host staging), ping-pong byte identity (AC-08 analogue), put/get,
and run_jacobi3d(engine="tasks") — the reference's own per-chunk protocol
(pack -> mp_send -> unpack -> update tasks) — bitwise against the goldens."""

import hashlib

import numpy as np
import pytest

from conftest import kwargs_of, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    from paper_2303_02543_b200 import _native as N

    N.require_gpu(0)


@pytest.mark.parametrize("path", ["direct", "staging"])
def test_pingpong_byte_identity(path):
    from paper_2303_02543_b200.pingpong import run_pingpong

    sizes = [8, 448, 449, 4096, 1 << 20, 3 << 20]
    rep = run_pingpong(sizes, iterations=3, path=path, verify=True, warmup=1)
    assert [r["size_bytes"] for r in rep.rows] == sizes
    for r in rep.rows:
        assert r["mean_latency_s"] > 0
        assert r["bandwidth_Bps"] == pytest.approx(r["size_bytes"] / r["mean_latency_s"])
    if path == "direct":
        assert rep.meta["staging_copies"] == 0  # AC-08: no host staging on the device path
        assert rep.meta["device_copies"] == 2 * (3 + 1) * len(sizes)  # incl. the warm-up
    else:
        assert rep.meta["staging_copies"] > 0


@pytest.mark.parametrize("path", ["direct", "staging"])
def test_pingpong_over_tcp_world(path):
    """Same ping-pong through the byte protocol (reference headers over
    localhost TCP); direct payloads still go GPU->GPU (device locators)."""
    from paper_2303_02543_b200.pingpong import run_pingpong

    sizes = [8, 448, 449, 4096, 1 << 20]
    rep = run_pingpong(sizes, iterations=3, path=path, transport="tcp", verify=True, warmup=1)
    assert [r["size_bytes"] for r in rep.rows] == sizes
    if path == "direct":
        # device sources ship as locators; host-resident payloads never occur here
        assert rep.meta["staging_copies"] == 0
        assert rep.meta["device_copies"] == 2 * (3 + 1) * len(sizes)  # incl. the warm-up
    else:
        assert rep.meta["staging_copies"] > 0


def test_pingpong_payload_sequence_is_the_references():
    """The payload bytes are the reference's (default_rng(99), pingpong.py:107,115)."""
    g = load_golden("pingpong.json")
    rng = np.random.default_rng(g["seed"])
    for p in g["payloads"][:12]:
        b = rng.integers(0, 256, size=p["size"], dtype=np.uint8)
        assert hashlib.sha256(b.tobytes()).hexdigest() == p["sha256"]


@pytest.mark.parametrize("transport", ["loopback", "tcp"])
def test_mp_send_bytes_ordering_and_objects(transport):
    from paper_2303_02543_b200.comm import MobileRef, drive, exchange_all, shutdown_all
    from paper_2303_02543_b200.devices import DeviceType
    from paper_2303_02543_b200.native_kernels import Fill
    from paper_2303_02543_b200.worlds import WorldConfig, make_loopback_world, make_tcp_world

    make = make_tcp_world if transport == "tcp" else make_loopback_world
    for aware in (True, False):
        comms = make(WorldConfig(ranks=2, device_aware=aware))
        got = []
        hid = [c.register_handler(lambda m, a, ctx: got.append(a)) for c in comms][0]
        for c in comms:
            c.create_mobile_object(b"m")
        exchange_all(comms)
        for k in range(20):
            comms[0].mp_send(MobileRef(1, 0), hid, bytes([k]) * (k * 40))
        drive(comms, until=lambda: len(got) == 20)
        assert [len(g) for g in got] == [k * 40 for k in range(20)]
        assert all(g == bytes([k]) * (k * 40) for k, g in enumerate(got))
        # object sends are ordered after the writer task (GPU-side edge)
        rt0 = comms[0].runtime
        rt0.register_kernel("fill9", gpu_sim=Fill(9))
        obj = rt0.create_object((5000,), dtype=np.uint8)
        t = rt0.task().device(DeviceType.GPU_SIM)
        t.arg(obj).write()
        t.submit("fill9")
        got.clear()
        comms[0].mp_send(MobileRef(1, 0), hid, obj)
        drive(comms, until=lambda: len(got) == 1)
        w = got[0]
        drive(comms, until=lambda: w.written or w.host_state.value == "valid")
        assert np.array_equal(comms[1].runtime.peek(w).reshape(-1), np.full(5000, 9, np.uint8))
        shutdown_all(comms)


@pytest.mark.parametrize("transport", ["loopback", "tcp"])
def test_put_get_roundtrip(transport):
    from paper_2303_02543_b200.comm import GlobalObjectId, drive, exchange_all, shutdown_all
    from paper_2303_02543_b200.worlds import WorldConfig, make_loopback_world, make_tcp_world

    make = make_tcp_world if transport == "tcp" else make_loopback_world
    comms = make(WorldConfig(ranks=2, device_aware=True))
    for c in comms:
        c.create_mobile_object(b"m")
    exchange_all(comms)
    done = []
    hid = [c.register_handler(lambda m, a, ctx: done.append(a)) for c in comms][0]
    rt1 = comms[1].runtime
    target = rt1.create_object((256,), dtype=np.uint8)
    v = rt1.request_data(target, write=True).get()
    v[:] = 3
    rt1.release(target)
    comms[0].hetero_put(GlobalObjectId(1, target.object_id), bytes(range(256)), hid)
    drive(comms, until=lambda: len(done) == 1)
    rt1.synchronize()
    assert np.array_equal(rt1.peek(target), np.arange(256, dtype=np.uint8))
    dest = comms[0].runtime.create_object((256,), dtype=np.uint8)
    comms[0].hetero_get(GlobalObjectId(1, target.object_id), dest, hid)
    drive(comms, until=lambda: len(done) == 2)
    comms[0].runtime.synchronize()
    assert np.array_equal(comms[0].runtime.peek(dest), np.arange(256, dtype=np.uint8))
    shutdown_all(comms)


TASK_LADDER = ["cube8_s3", "ac10_g222", "ac10_r2d2", "slab64_s10", "halo32_s20",
               "halo32_s20_r2d2", "halo32_s20_direct", "halo16_cube_s12", "zero_steps",
               "rect_slab", "thin_x", "zslab_3d"]


@pytest.mark.parametrize("name", TASK_LADDER)
def test_task_engine_ladder_bitwise(ladder, name):
    from paper_2303_02543_b200.jacobi import run_jacobi3d

    e = ladder[name]
    rep, cs, arr = run_jacobi3d(tuple(e["domain"]), steps=e["steps"], engine="tasks",
                                **kwargs_of(e))
    assert hashlib.sha256(arr.tobytes()).hexdigest() == e["sha256"]
    assert repr(cs) == e["checksum"]
    if e["kwargs"].get("device_aware"):
        assert sum(s["staging_copies"] for s in rep.meta["stats"]) == 0


@pytest.mark.parametrize("push", [False, True])
def test_sm_copy_kernel_bytes(push):
    """hrt_copy_sm_async (SM copy over NVLink, pull on the destination or
    push from the source) moves exactly the bytes, odd sizes included."""
    import ctypes

    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import DevicePool, Stream

    n = N.gpu_count()
    src_gpu, dst_gpu = 0, (1 if n > 1 else 0)
    if src_gpu != dst_gpu:
        N.call("hrt_enable_peer_access", dst_gpu, src_gpu)
        N.call("hrt_enable_peer_access", src_gpu, dst_gpu)
    rng = np.random.default_rng(3)
    for size in (1, 17, 4096 + 9, (3 << 20) + 5):
        data = rng.integers(0, 256, size=size, dtype=np.uint8)
        sp, dp = DevicePool(src_gpu, size + 4096), DevicePool(dst_gpu, size + 4096)
        s_ptr, d_ptr = sp.alloc(size)[2], dp.alloc(size)[2]
        st_src, st_dst = Stream(src_gpu), Stream(dst_gpu)
        N.call("hrt_copy_async", st_src.h, ctypes.c_void_p(s_ptr),
               ctypes.c_void_p(data.ctypes.data), size)
        st_src.synchronize()
        st = st_src if push else st_dst
        N.call("hrt_copy_sm_async", st.h, ctypes.c_void_p(d_ptr), ctypes.c_void_p(s_ptr),
               ctypes.c_uint64(size), 0)
        st.synchronize()
        out = np.empty(size, np.uint8)
        N.call("hrt_copy_async", st_dst.h, ctypes.c_void_p(out.ctypes.data),
               ctypes.c_void_p(d_ptr), size)
        st_dst.synchronize()
        assert np.array_equal(out, data), size


@pytest.mark.parametrize("method", [0, 1, 2])
def test_copy_ordered_waits_and_bytes(method):
    """hrt_copy_ordered (enqueue_transfer in one call): the copy runs after
    its wait tokens — a producer on another stream writes the source first —
    and moves exactly the bytes with the copy engine (0), the SM kernel (1)
    or the automatic choice (2); retired wait tokens are skipped."""
    import ctypes

    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import DevicePool, Stream

    n = N.gpu_count()
    src_gpu, dst_gpu = 0, (1 if n > 1 else 0)
    if src_gpu != dst_gpu:
        N.call("hrt_enable_peer_access", dst_gpu, src_gpu)
        N.call("hrt_enable_peer_access", src_gpu, dst_gpu)
    rng = np.random.default_rng(5)
    for size in (16, 4096, (2 << 20) + 16, 3 << 20):
        data = rng.integers(0, 256, size=size, dtype=np.uint8)
        sp, dp = DevicePool(src_gpu, size + 4096), DevicePool(dst_gpu, size + 4096)
        s_ptr, d_ptr = sp.alloc(size)[2], dp.alloc(size)[2]
        st_src, st_dst = Stream(src_gpu), Stream(dst_gpu)
        # producer: memset then upload on the source's stream, not synchronised
        N.call("hrt_memset_async", st_src.h, ctypes.c_void_p(s_ptr), 0, ctypes.c_uint64(size))
        N.call("hrt_copy_async", st_src.h, ctypes.c_void_p(s_ptr),
               ctypes.c_void_p(data.ctypes.data), size)
        prod = st_src.record()
        done = ctypes.c_uint64()
        # a retired token in the list (released) must be skipped
        old = st_dst.record()
        old.wait()
        old_id = old.token_id
        _ = old.status  # latches and releases the native token
        waits = (ctypes.c_uint64 * 2)(prod.token_id, old_id)
        N.call("hrt_copy_ordered", st_dst.h, ctypes.c_void_p(d_ptr), ctypes.c_void_p(s_ptr),
               ctypes.c_uint64(size), int(src_gpu != dst_gpu), waits, 2, method,
               ctypes.byref(done))
        assert N.lib().hrt_token_wait(done) == 0
        N.lib().hrt_token_release(done)
        out = np.empty(size, np.uint8)
        N.call("hrt_copy_async", st_dst.h, ctypes.c_void_p(out.ctypes.data),
               ctypes.c_void_p(d_ptr), size)
        st_dst.synchronize()
        assert np.array_equal(out, data), (method, size)
