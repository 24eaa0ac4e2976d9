"""Randomized serial equivalence of the B200 task runtime — the analogue of
the reference's AC-01/AC-02 suites (test_acceptance.py:49-163, conftest.py
RandomCase): random streams of read/write tasks (real device kernels) over
shared objects on several devices, interleaved with host read/write leases,
must leave exactly the bytes a serial interpreter computes.  Exercises
GPU-side dependency edges (tasks issued before their prerequisites
finish), program-order coherence, peer/D2D copies between devices and
lease ordering."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def make_runtime(ndev):
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import DeviceDescriptor, DeviceRegistry, DeviceType
    from paper_2303_02543_b200.native_kernels import Fill, Mix
    from paper_2303_02543_b200.runtime import Runtime

    N.require_gpu(0)
    reg = DeviceRegistry()
    for j in range(ndev):
        reg.register_device(DeviceDescriptor(device_id=j, device_type=DeviceType.GPU_SIM,
                                             memory_capacity=32 << 20, compute_stream_count=3,
                                             gpu=j % N.gpu_count()))
    rt = Runtime(reg)
    for salt in range(8):
        rt.register_kernel(f"mix{salt}", gpu_sim=Mix(salt))
        rt.register_kernel(f"fill{salt}", gpu_sim=Fill(salt * 29))
    return rt


def run_case(seed, nobj=5, nops=60, size=4099, ndev=3):
    from paper_2303_02543_b200.devices import DeviceType

    rnd = random.Random(seed)
    rt = make_runtime(ndev)
    objs = [rt.create_object((size,), dtype=np.uint8) for _ in range(nobj)]
    shadow = [np.zeros(size, np.uint8) for _ in range(nobj)]
    for _ in range(nops):
        op = rnd.random()
        d = rnd.randrange(nobj)
        if op < 0.45:  # dst = dst*7 + src + salt
            s = rnd.randrange(nobj)
            salt = rnd.randrange(8)
            t = rt.task().device(DeviceType.GPU_SIM)
            if s != d:
                t.arg(objs[s]).read()
                t.arg(objs[d]).read_write()
                shadow[d] = (shadow[d].astype(np.uint32) * 7 + shadow[s] + salt).astype(np.uint8)
            else:
                t.arg(objs[d]).read_write()
                shadow[d] = (shadow[d].astype(np.uint32) * 7 + salt).astype(np.uint8)
            t.submit(f"mix{salt}")
        elif op < 0.6:  # overwrite
            salt = rnd.randrange(8)
            t = rt.task().device(DeviceType.GPU_SIM)
            t.arg(objs[d]).write()
            t.submit(f"fill{salt}")
            shadow[d][:] = (salt * 29) & 0xFF
        elif op < 0.8:  # host read lease sees the serial state
            v = rt.request_data(objs[d]).get()
            assert np.array_equal(v, shadow[d]), f"seed {seed}: host read mismatch"
            rt.release(objs[d])
        else:  # host write lease
            v = rt.request_data(objs[d], write=True).get()
            v[: size // 3] = rnd.randrange(256)
            shadow[d][: size // 3] = v[: size // 3]
            rt.release(objs[d])
    rt.synchronize()
    for i, o in enumerate(objs):
        assert np.array_equal(rt.peek(o).reshape(-1), shadow[i]), f"seed {seed}: object {i}"
    return rt.stats


def test_random_task_streams_serial_equivalence():
    copies = 0
    for seed in range(40):
        st = run_case(seed)
        copies += st["peer_copies"]
    assert copies > 0  # the streams did move data between devices


def test_deep_dependency_chain_without_host_waits():
    """1000 dependent tasks issued back to back (each waits on the previous
    kernel's event on the GPU, none on the host)."""
    from paper_2303_02543_b200.devices import DeviceType

    rt = make_runtime(2)
    a = rt.create_object((1 << 16,), dtype=np.uint8)
    b = rt.create_object((1 << 16,), dtype=np.uint8)
    sa, sb = np.zeros(1 << 16, np.uint8), np.zeros(1 << 16, np.uint8)
    for k in range(1000):
        src, dst, s_src, s_dst = (a, b, sa, sb) if k % 2 else (b, a, sb, sa)
        t = rt.task().device(DeviceType.GPU_SIM)
        t.arg(src).read()
        t.arg(dst).read_write()
        t.submit(f"mix{k % 8}")
        s_dst[:] = (s_dst.astype(np.uint32) * 7 + s_src + k % 8).astype(np.uint8)
    rt.synchronize()
    assert np.array_equal(rt.peek(a).reshape(-1), sa)
    assert np.array_equal(rt.peek(b).reshape(-1), sb)
