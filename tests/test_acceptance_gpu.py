"""GPU analogues of the reference's remaining acceptance criteria on the
B200 runtime and message layer:

* AC-02 conflict safety (test_acceptance.py:67-96): tasks' kernels record
  their own device-clock intervals (%globaltimer); kernels of conflicting
  tasks (a shared object, at least one writer) never overlap, and at least
  one pair of independent kernels does — the "several blocks in flight per
  GPU" witness.
* AC-09 put/get ordering (test_acceptance.py:299-387): a remote put racing
  a writer task, in both registration orders, ends in the
  registration-order result; a later get observes post-write bytes.
* ReceiveCache (comm.py:94-131, test_comm.py:297-316): hits, misses, slab
  return on wrapper destruction, transparency of the bytes."""

import ctypes
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    from paper_2303_02543_b200 import _native as N

    N.require_gpu(0)


def _overlap(a, b) -> bool:
    return a[0] < b[1] and b[0] < a[1]


@pytest.mark.parametrize("seed", range(6))
def test_ac02_conflicting_kernels_never_overlap(seed):
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import (DeviceDescriptor, DevicePool, DeviceRegistry,
                                               DeviceType, Stream)
    from paper_2303_02543_b200.native_kernels import Stamp
    from paper_2303_02543_b200.objects import AccessMode
    from paper_2303_02543_b200.runtime import Runtime

    rnd = random.Random(seed)
    reg = DeviceRegistry()
    reg.register_device(DeviceDescriptor(device_id=0, device_type=DeviceType.GPU_SIM,
                                         memory_capacity=16 << 20, compute_stream_count=5, gpu=0))
    rt = Runtime(reg)
    ntask = 40
    stamps = DevicePool(0, ntask * 16 + 256)
    base = stamps.alloc(ntask * 16)[2]
    objs = [rt.create_object((4096,), dtype=np.uint8) for _ in range(6)]
    tasks, access = [], []
    for i in range(ntask):
        rt.register_kernel(f"stamp{i}", gpu_sim=Stamp(base + 16 * i, ns=rnd.choice([60, 150]) * 1000))
        args = []
        for o in rnd.sample(range(len(objs)), rnd.randint(1, 2)):
            args.append((o, rnd.choice([AccessMode.READ, AccessMode.WRITE,
                                        AccessMode.READ_WRITE])))
        t = rt.task().device(DeviceType.GPU_SIM)
        for o, m in args:
            {AccessMode.READ: t.arg(objs[o]).read, AccessMode.WRITE: t.arg(objs[o]).write,
             AccessMode.READ_WRITE: t.arg(objs[o]).read_write}[m]()
        tasks.append(t.submit(f"stamp{i}"))
        access.append(dict(args))
    rt.wait_all(tasks)
    rt.synchronize()
    iv = np.empty(2 * ntask, dtype=np.uint64)
    st = Stream(0)
    N.call("hrt_copy_async", st.h, ctypes.c_void_p(iv.ctypes.data), ctypes.c_void_p(base),
           iv.nbytes)
    st.synchronize()
    iv = iv.reshape(ntask, 2).astype(np.int64)
    assert np.all(iv[:, 1] > iv[:, 0])

    def conflict(a, b):
        return any(o in access[b] and (m is not AccessMode.READ or
                                       access[b][o] is not AccessMode.READ)
                   for o, m in access[a].items())

    witnesses = 0
    for a in range(ntask):
        for b in range(a + 1, ntask):
            if conflict(a, b):
                assert not _overlap(iv[a], iv[b]), f"conflicting tasks {a},{b} overlapped"
            elif _overlap(iv[a], iv[b]):
                witnesses += 1
    assert witnesses >= 1, "no independent kernels ever overlapped"


@pytest.mark.parametrize("seed", range(24))
def test_ac09_put_vs_writer_race_and_get(seed):
    """A put racing a writer task on the owner, both orders; then a get."""
    from paper_2303_02543_b200.comm import GlobalObjectId, drive, exchange_all, shutdown_all
    from paper_2303_02543_b200.devices import DevicePool, DeviceType
    from paper_2303_02543_b200.native_kernels import Mix, Stamp
    from paper_2303_02543_b200.worlds import WorldConfig, make_loopback_world

    rnd = random.Random(seed)
    comms = make_loopback_world(WorldConfig(ranks=2, device_aware=bool(seed % 2)))
    for c in comms:
        c.create_mobile_object(b"m")
    exchange_all(comms)
    rt1 = comms[1].runtime
    size = rnd.choice([64, 256, 1024, 65536])
    initial = rnd.randrange(256)
    put_bytes = bytes([rnd.randrange(256)]) * size
    salt = rnd.randrange(200)
    target = rt1.create_object((size,), dtype=np.uint8)
    rt1.request_data(target, write=True).get()[:] = initial
    rt1.release(target)
    # the writer (dst = dst*7 + salt) and a long-running kernel to hold it back
    rt1.register_kernel("writer", gpu_sim=Mix(salt))
    # the stamp slots live on rank 1's GPU (the kernels run there)
    gpu1 = rt1.registry.gpu_of(rt1.registry.devices_of_type(DeviceType.GPU_SIM)[0])
    scratch = DevicePool(gpu1, 4096)
    rt1.register_kernel("blocker", gpu_sim=Stamp(scratch.alloc(16)[2], ns=500_000))
    blocker_obj = rt1.create_object((8,), dtype=np.uint8)
    done = []
    hid = [c.register_handler(lambda m, a, ctx: done.append(a)) for c in comms][0]
    gid = GlobalObjectId(1, target.object_id)
    shadow = np.full(size, initial, dtype=np.uint8)

    if rnd.random() < 0.5:
        # writer registered first (held by an explicit dependency on a slow
        # kernel); the put arrives later and must still land after it
        b = rt1.task().device(DeviceType.GPU_SIM)
        b.arg(blocker_obj).write()
        blocker = b.submit("blocker")
        t = rt1.task().device(DeviceType.GPU_SIM)
        t.arg(target).read_write()
        t.depends_on(blocker)
        handle = t.submit("writer")
        comms[0].hetero_put(gid, put_bytes, hid)
        shadow = ((shadow.astype(np.uint64) * 7 + salt) % 256).astype(np.uint8)
        shadow[:] = np.frombuffer(put_bytes, dtype=np.uint8)
    else:
        # put registered first (held behind a long reader), writer second
        rt1.register_kernel("reader", gpu_sim=Stamp(scratch.alloc(16)[2], ns=500_000))
        r = rt1.task().device(DeviceType.GPU_SIM)
        r.arg(target).read()
        r.submit("reader")
        comms[0].hetero_put(gid, put_bytes, hid)
        comms[0].network_progress()   # frame out
        comms[1].network_progress()   # owner registers the put's write access
        t = rt1.task().device(DeviceType.GPU_SIM)
        t.arg(target).read_write()
        handle = t.submit("writer")
        shadow[:] = np.frombuffer(put_bytes, dtype=np.uint8)
        shadow = ((shadow.astype(np.uint64) * 7 + salt) % 256).astype(np.uint8)
    drive(comms, until=lambda: len(done) == 1 and handle.done)
    rt1.synchronize()
    assert np.array_equal(rt1.peek(target).reshape(-1), shadow), "put/task order mismatch"
    # a get issued after the writer observes post-write bytes
    dest = comms[0].runtime.create_object((size,), dtype=np.uint8)
    got = []
    gdone = [c.register_handler(lambda m, a, ctx: got.append(a)) for c in comms][0]
    comms[0].hetero_get(gid, dest, gdone)
    drive(comms, until=lambda: len(got) == 1)
    comms[0].runtime.synchronize()
    assert np.array_equal(comms[0].runtime.peek(dest).reshape(-1), shadow)
    shutdown_all(comms)


def _device_resident(rt, data):
    from paper_2303_02543_b200.devices import DeviceType
    from paper_2303_02543_b200.native_kernels import Touch

    obj = rt.create_object((data.size,), dtype=np.uint8)
    np.copyto(rt.request_data(obj, write=True).get(), data)
    rt.release(obj)
    if "touch" not in rt.kernels:
        rt.register_kernel("touch", gpu_sim=Touch())
    t = rt.task().device(DeviceType.GPU_SIM)
    t.arg(obj).read_write()
    rt.wait(t.submit("touch"))
    return obj


@pytest.mark.parametrize("aware", [True, False])
def test_receive_cache_hits_misses_and_reuse(aware):
    """comm.py:94-131: a payload <= slab lands in a cache slab (hit), a
    larger one or a disabled cache allocates from the pool (miss); slabs
    return to the cache when the wrapper is destroyed and are reused; the
    bytes are identical either way."""
    from paper_2303_02543_b200.comm import MobileRef, drive, exchange_all, shutdown_all
    from paper_2303_02543_b200.worlds import WorldConfig, make_loopback_world

    rng = np.random.default_rng(11)
    data = rng.integers(0, 256, 64 << 10, dtype=np.uint8)
    big = rng.integers(0, 256, 3 << 20, dtype=np.uint8)
    results = {}
    for cache_bytes in (2 << 20, 0):
        comms = make_loopback_world(WorldConfig(ranks=2, device_aware=aware,
                                                recv_cache_bytes=cache_bytes))
        for c in comms:
            c.create_mobile_object(b"m")
        exchange_all(comms)
        rt0, rt1 = comms[0].runtime, comms[1].runtime
        got = []
        hid = [c.register_handler(lambda m, a, ctx: got.append(a)) for c in comms][0]
        small, large = _device_resident(rt0, data), _device_resident(rt0, big)
        outs = []
        for k, obj in enumerate([small, small, small, large]):
            comms[0].mp_send(MobileRef(1, 0), hid, obj)
            drive(comms, until=lambda: len(got) == k + 1 and got[-1].written)
            rt1.synchronize()
            outs.append(rt1.peek(got[-1]).reshape(-1).copy())
            w = got[-1]
            rt1.destroy_object(w)   # the slab goes back to the cache
            drive(comms, until=lambda: w.destroyed)
        st = comms[1].stats
        if cache_bytes:
            # two 1 MiB slabs: the three small payloads reuse returned slabs
            assert st.recv_cache_hits == 3 and st.recv_cache_misses == 1, vars(st)
            assert len(comms[1].recv_cache._free[next(iter(comms[1].recv_cache._free))]) == 2
        else:
            assert st.recv_cache_hits == 0 and st.recv_cache_misses == 4, vars(st)
        for o, ref in zip(outs, [data, data, data, big]):
            assert np.array_equal(o, ref)
        results[cache_bytes] = outs
        shutdown_all(comms)
    assert all(np.array_equal(a, b) for a, b in zip(results[2 << 20], results[0]))
