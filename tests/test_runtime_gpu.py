"""The task runtime on B200s (runtime.py): dependency ordering, coherence
across devices, host leases, deferred destruction, failure propagation —
the reference's L1 semantics (runtime.py, objects.py) with GPU-side
ordering."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture()
def rt():
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import DeviceDescriptor, DeviceRegistry, DeviceType
    from paper_2303_02543_b200.runtime import Runtime

    N.require_gpu(0)
    reg = DeviceRegistry()
    for j in range(2):
        reg.register_device(DeviceDescriptor(device_id=j, device_type=DeviceType.GPU_SIM,
                                             memory_capacity=64 << 20, compute_stream_count=3,
                                             gpu=j % N.gpu_count()))
    r = Runtime(reg)
    return r


def _kernels(rt):
    from paper_2303_02543_b200.native_kernels import Fill, HaloPack, HaloUnpack, JacobiUpdate, Touch

    rt.register_kernel("fill7", gpu_sim=Fill(7))
    rt.register_kernel("touch", gpu_sim=Touch())
    rt.register_kernel("upd", gpu_sim=JacobiUpdate())
    for f in range(6):
        rt.register_kernel(f"pack{f}", gpu_sim=HaloPack(f))
        rt.register_kernel(f"unpack{f}", gpu_sim=HaloUnpack(f))


def test_host_lease_roundtrip_and_zero_default(rt):
    from paper_2303_02543_b200.devices import DeviceType

    _kernels(rt)
    obj = rt.create_object((1000,), dtype=np.uint8)
    assert np.array_equal(rt.request_data(obj).get(), np.zeros(1000, np.uint8))
    rt.release(obj)
    v = rt.request_data(obj, write=True).get()
    v[:] = np.arange(1000) % 251
    rt.release(obj)
    t = rt.task().device(DeviceType.GPU_SIM)
    t.arg(obj).read_write()
    rt.wait(t.submit("touch"))
    assert obj.valid_devices() and np.array_equal(rt.peek(obj), np.arange(1000) % 251)
    w = rt.task().device(DeviceType.GPU_SIM)
    w.arg(obj).write()
    rt.wait(w.submit("fill7"))
    assert np.array_equal(rt.request_data(obj).get(), np.full(1000, 7, np.uint8))
    rt.release(obj)


def test_jacobi_chunk_chain_matches_oracle(rt, oracle):
    """A single chunk stepped by a chain of dependent tasks issued without
    host waits (each waits on the previous kernel's event on the GPU)."""
    from paper_2303_02543_b200.devices import DeviceType

    _kernels(rt)
    ex, ey, ez, steps = 20, 18, 6, 25
    bufs = [rt.create_object((ex + 2, ey + 2, ez + 2), dtype=np.float64) for _ in range(2)]
    for b in bufs:
        v = rt.request_data(b, write=True).get()
        v[:] = 0.0
        v[0], v[-1], v[:, 0], v[:, -1], v[:, :, 0], v[:, :, -1] = 1, 1, 1, 1, 1, 1
        rt.release(b)
    last = None
    for s in range(steps):
        t = rt.task().device(DeviceType.GPU_SIM)
        t.arg(bufs[s % 2]).read()
        t.arg(bufs[(s + 1) % 2]).write()
        last = t.submit("upd")
    rt.wait(last)
    got = rt.request_data(bufs[steps % 2]).get()[1:-1, 1:-1, 1:-1]
    assert np.array_equal(got, oracle.jacobi_c((ex, ey, ez), steps))


def test_cross_device_coherence_and_pack_unpack(rt):
    """Writer on device 0, reader on device 1: the reader's copy comes over
    NVLink (peer copy) ordered after the writer; pack/unpack plane copies."""
    from paper_2303_02543_b200.devices import DeviceType

    _kernels(rt)
    shape = (6, 5, 4)
    u = rt.create_object(shape, dtype=np.float64)
    v = rt.request_data(u, write=True).get()
    v[:] = np.arange(np.prod(shape), dtype=np.float64).reshape(shape)
    rt.release(u)
    halos = []
    for f in range(6):
        axis = f // 2
        hs = [shape[a] - 2 for a in range(3) if a != axis]
        h = rt.create_object(tuple(hs), dtype=np.float64)
        t = rt.task().device(DeviceType.GPU_SIM)
        t.arg(u).read()
        t.arg(h).write()
        t.submit(f"pack{f}")
        halos.append(h)
    rt.synchronize()
    full = np.arange(np.prod(shape), dtype=np.float64).reshape(shape)
    idx = {0: 1, 1: shape[0] - 2}
    got0 = rt.request_data(halos[0]).get()
    assert np.array_equal(got0, full[1, 1:-1, 1:-1])
    rt.release(halos[0])
    got3 = rt.request_data(halos[3]).get()
    assert np.array_equal(got3, full[1:-1, shape[1] - 2, 1:-1])
    rt.release(halos[3])
    # unpack every halo into a fresh object's ghost planes
    w = rt.create_object(shape, dtype=np.float64)
    for f in range(6):
        t = rt.task().device(DeviceType.GPU_SIM)
        t.arg(halos[f]).read()
        t.arg(w).read_write()
        t.submit(f"unpack{f}")
    out = rt.request_data(w).get()
    assert np.array_equal(out[0, 1:-1, 1:-1], full[1, 1:-1, 1:-1])
    assert np.array_equal(out[1:-1, -1, 1:-1], full[1:-1, shape[1] - 2, 1:-1])
    assert idx[0] == 1


def test_destroy_is_deferred_until_tasks_finish(rt):
    from paper_2303_02543_b200.devices import DeviceType

    _kernels(rt)
    free0 = rt.registry.free_bytes(0)
    objs = [rt.create_object((1 << 20,), dtype=np.uint8) for _ in range(4)]
    for o in objs:
        t = rt.task().device(DeviceType.GPU_SIM)
        t.arg(o).write()
        t.submit("fill7")
        rt.destroy_object(o)
        assert not o.destroyed
    rt.synchronize()
    assert all(o.destroyed for o in objs)
    assert rt.registry.free_bytes(0) == free0


def test_python_bodies_rejected_no_fallback(rt):
    from paper_2303_02543_b200.errors import HrtError

    with pytest.raises(HrtError, match="native launchers"):
        rt.register_kernel("py", gpu_sim=lambda v, g, s: None)
