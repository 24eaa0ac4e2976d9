"""The drop-in, proven against the reference itself: the
UNMODIFIED reference package (installed into baseline/_ref by
integration/install_reference.sh) runs its own ``run_jacobi3d``
(bench/jacobi.py:281-462) and ``run_pingpong`` (bench/pingpong.py:48-152)
with integration/hrt_b200_plugin.py selected as the device backend — its
DeviceRegistry / DeviceBackend / CompletionToken / clock subclasses over
libhrt_b200.so.  Results are compared bitwise with the goldens the
reference produced on its simulator, and the reference's numpy kernel
bodies are replaced by tripwires: none may execute."""

import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, kwargs_of

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def plugin():
    if not os.path.isdir(os.path.join(REF, "hrt")):
        if os.path.isdir("/root/reference/pkg"):
            subprocess.run(["sh", os.path.join(ROOT, "integration", "install_reference.sh")],
                           check=True, capture_output=True)
        else:
            pytest.skip("baseline/_ref (the reference install) is absent")
    for p in (REF, os.path.join(ROOT, "integration")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import hrt_b200_plugin as P

    P.lib()
    return P


@pytest.fixture
def tripwires(monkeypatch):
    """Replace the reference's numpy kernel bodies by bodies that count and
    fail: the drivers register whatever the module holds at run time."""
    import hrt.bench.jacobi as J

    calls = []

    def trip(name):
        def body(views, geom, scratch):
            calls.append(name)
            raise AssertionError(f"reference numpy body {name} executed")
        return body

    monkeypatch.setattr(J, "_update_body", trip("jacobi_update"))
    monkeypatch.setattr(J, "_make_pack_body", lambda f: trip(f"halo_pack_{f}"))
    monkeypatch.setattr(J, "_make_unpack_body", lambda f: trip(f"halo_unpack_{f}"))
    return calls


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["halo32_s20", "halo16_cube_s12", "ac10_r2d2",
                                  "halo32_s20_direct", "halo32_s20_r2d2", "cube24_s30",
                                  "slab96x80_s13", "unit_chunks_cube", "zero_steps"])
def test_reference_run_jacobi3d_on_b200(plugin, tripwires, ladder, name):
    """hrt.bench.jacobi.run_jacobi3d, unmodified, through the B200 backend:
    every pack / mp_send / unpack / update task of the reference's protocol
    runs as a libhrt_b200 launch; field SHA-256 and checksum repr equal the
    reference's simulator goldens; no numpy body ran."""
    from hrt.bench.jacobi import run_jacobi3d
    from hrt.devices import ClockMode

    e = ladder[name]
    kw = kwargs_of(e)
    with plugin.b200_worlds(gpus=[0]) as regs:
        rep, cs, arr = run_jacobi3d(tuple(e["domain"]), steps=e["steps"], clock=ClockMode.WALL,
                                    **kw)
    assert tripwires == []
    assert sha(arr) == e["sha256"]
    assert repr(cs) == e["checksum"]
    assert len(rep.rows) == e["steps"]
    assert regs and all(isinstance(r, plugin.B200Registry) for r in regs)
    launches = sum(r.native_launches for r in regs)
    assert launches >= e["steps"] * (1 if e["steps"] else 0)
    for r in regs:
        for did in r.device_ids:
            assert r.device(did).backend.kernel_runs == 0


def test_reference_check_mode_and_virtual_clock(plugin, tripwires):
    """The reference's own ``check=True`` (numpy jacobi_reference vs the
    assembled field, jacobi.py:456-459) passes with the B200 backend, also
    under the default ClockMode.VIRTUAL argument (the device clock serves
    both)."""
    from hrt.bench.jacobi import run_jacobi3d

    with plugin.b200_worlds(gpus=[0]):
        _, cs, arr = run_jacobi3d((12, 10, 6), steps=15, grid=(2, 1, 3), check=True)
    assert tripwires == []
    assert 0.0 < arr.mean() < 1.0


@pytest.mark.parametrize("path", ["direct", "staging"])
def test_reference_run_pingpong_on_b200(plugin, path):
    """hrt.bench.pingpong.run_pingpong, unmodified, 8 B .. 8 MiB: the object
    is parked on the B200 by the ``touch`` task (native, no body), sent
    both ways through the reference's mp_send, and verified byte-identical
    by the reference itself (pingpong.py:135-138)."""
    from hrt.bench.pingpong import parse_sizes, run_pingpong
    from hrt.devices import ClockMode

    sizes = parse_sizes("8..8388608")
    with plugin.b200_worlds(gpus=[0]) as regs:
        rep = run_pingpong(sizes, iterations=3, path=path, clock=ClockMode.WALL)
    assert [r["size_bytes"] for r in rep.rows] == sizes
    assert all(r["mean_latency_s"] > 0 for r in rep.rows)
    assert sum(r.native_launches for r in regs) == len(sizes)  # one touch per size
    assert sum(r.copies["h2d"] for r in regs) > 0
    if path == "direct":
        assert rep.meta["staging_copies"] == 0


def test_unknown_kernel_fails_loudly(plugin):
    """A kernel with no native entry point FAILS its token (-> TaskFailed):
    there is no fallback to the Python body."""
    from hrt.bench.worlds import WorldConfig, make_loopback_world
    from hrt.devices import ClockMode, DeviceType
    from hrt.errors import TaskFailed

    ran = []
    with plugin.b200_worlds(gpus=[0]):
        (comm,) = make_loopback_world(WorldConfig(ranks=1, clock=ClockMode.WALL,
                                                  with_host_device=False))
    rt = comm.runtime
    rt.register_kernel("python_only", body=lambda v, g, s: ran.append(1))
    obj = rt.create_object((64,), dtype=np.float64)
    t = rt.task().device(DeviceType.GPU_SIM)
    t.arg(obj).read_write()
    task = t.submit("python_only")
    with pytest.raises(TaskFailed):
        rt.wait(task)
    assert ran == []


def test_device_tokens_follow_events(plugin):
    """DeviceToken.status is PENDING until its CUDA event completes;
    DeviceClock.advance_one blocks on the oldest one (runtime.py:525-527)."""
    from hrt.devices import DeviceAllocation, DeviceDescriptor, DeviceType, TokenStatus

    clock = plugin.DeviceClock()
    reg = plugin.B200Registry(clock=clock, gpu_of={0: 0})
    reg.register_device(DeviceDescriptor(0, DeviceType.GPU_SIM, 512 << 20))
    a = reg.pool_alloc(0, 256 << 20)
    b = reg.pool_alloc(0, 256 << 20)
    src = np.random.default_rng(1).integers(0, 256, 256 << 20, dtype=np.uint8)
    t1 = reg.enqueue_transfer(src, a, src.nbytes)
    t2 = reg.enqueue_transfer(a, b, src.nbytes)  # D2D: the simulator rejects this
    assert clock.advance_one() is t1 and t1.status is TokenStatus.COMPLETE
    assert clock.advance_one() is t2 and t2.status is TokenStatus.COMPLETE
    assert clock.advance_one() is None
    out = reg.device(0).backend.region(b).copy()
    assert np.array_equal(out, src)
    assert reg.copies["d2d"] == 1
    reg.pool_free(a)
    with pytest.raises(Exception):
        reg.pool_free(a)
