"""Small-message anatomy of a direct-path ping-pong round trip: host
timestamps (perf_counter, µs from the mp_send) of every stage the message
passes — access grant, frame out, frame in, handler, copy enqueue, copy
completion seen — averaged over many round trips.

python tools/pingpong_anatomy.py [size_bytes] [iterations]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200 import comm as C  # noqa: E402
from paper_2303_02543_b200.devices import DeviceRegistry, DeviceType  # noqa: E402
from paper_2303_02543_b200.native_kernels import Touch  # noqa: E402
from paper_2303_02543_b200.worlds import WorldConfig, make_loopback_world  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
marks = []


def mark(name):
    marks.append((name, time.perf_counter()))


def wrap(cls, name, label=None):
    orig = getattr(cls, name)

    def w(*a, **k):
        mark((label or name) + ">")
        r = orig(*a, **k)
        mark((label or name) + "<")
        return r

    setattr(cls, name, w)


wrap(C.Comm, "_on_frame")
wrap(C.Comm, "_device_copy")
wrap(DeviceRegistry, "enqueue_transfer")
if os.environ.get("PP_DETAIL"):
    from paper_2303_02543_b200 import runtime as RT
    wrap(C.Comm, "mp_send")
    wrap(C.Comm, "network_progress")
    wrap(RT.Runtime, "destroy_object")
    wrap(RT.Runtime, "register_access")
    wrap(RT.Runtime, "progress", "rt.progress")
    wrap(C.LoopbackTransport, "send", "tr.send")
ncalls = collections.Counter()
orig_call = N.call


def counted(name, *a):
    ncalls[name] += 1
    t = time.perf_counter()
    r = orig_call(name, *a)
    ncalls[name + " us"] += round((time.perf_counter() - t) * 1e6, 1)
    return r


N.call = counted
orig_progress = C.Comm.progress


def counted_progress(self, *a, **k):
    ncalls["Comm.progress"] += 1
    t = time.perf_counter()
    r = orig_progress(self, *a, **k)
    ncalls["Comm.progress us"] += round((time.perf_counter() - t) * 1e6)
    return r


C.Comm.progress = counted_progress
ngpu = N.gpu_count()
cfg = WorldConfig(ranks=2, device_aware=True, capacity=64 << 20, gpus=[0, 1 if ngpu > 1 else 0])
comms = make_loopback_world(cfg)
arrived = []


def h_pong(m, arg, ctx):
    mark("pong-handler")
    ctx.comm.mp_send(C.MobileRef(0, 0), h_ping, arg)
    ctx.comm.runtime.destroy_object(arg)


def h_ping(m, arg, ctx):
    mark("ping-handler")
    arrived.append(arg)


ids = [(c.register_handler(h_pong), c.register_handler(h_ping)) for c in comms]
h_pong_id, h_ping = ids[0]
for c in comms:
    c.create_mobile_object(b"pp")
    c.runtime.register_kernel("touch", gpu_sim=Touch(), cost=1e-6)
C.exchange_all(comms)
rt0 = comms[0].runtime
obj = rt0.create_object((size,), dtype=np.uint8)
np.copyto(rt0.request_data(obj, write=True).get(), np.zeros(size, np.uint8))
rt0.release(obj)
t = rt0.task().device(DeviceType.GPU_SIM)
t.arg(obj).read_write()
rt0.wait(t.submit("touch"))
acc = collections.defaultdict(list)
rts = []
for it in range(-20, iters):
    marks.clear()
    arrived.clear()
    ncalls.clear()
    t0 = time.perf_counter()
    comms[0].mp_send(C.MobileRef(1, 0), h_pong_id, obj)
    mark("sent")
    C.drive(comms, until=lambda: len(arrived) == 1)
    w = arrived[0]
    C.drive(comms, until=lambda: w.written)
    t1 = time.perf_counter()
    mark("written")
    if it >= 0:
        rts.append(t1 - t0)
        seen = collections.Counter()
        for name, ts in marks:
            seen[name] += 1
            acc[f"{name}#{seen[name]}"].append((ts - t0) * 1e6)
    rt0.destroy_object(w)
print(f"size {size} B, {iters} round trips: median round trip {np.median(rts) * 1e6:.1f} us "
      f"(one-way {np.median(rts) * 5e5:.1f} us)")
for k, v in sorted(acc.items(), key=lambda kv: np.median(kv[1])):
    print(f"  {k:28s} {np.median(v):8.1f} us")
print("native calls / progress passes per round trip (last):", dict(ncalls))
C.shutdown_all(comms)
