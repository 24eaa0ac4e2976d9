"""Where does a direct-path ping-pong round trip spend its time?  Runs the
cfg4 ping-pong at a few sizes with the device registry's transfers
instrumented: host timestamps of each enqueue and device time of each
copy (CUDA events), printed per iteration.

python tools/pingpong_trace.py [size_bytes ...]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.comm import MobileRef, drive, exchange_all, shutdown_all  # noqa: E402
from paper_2303_02543_b200.devices import DeviceRegistry, DeviceType  # noqa: E402
from paper_2303_02543_b200.native_kernels import Touch  # noqa: E402
from paper_2303_02543_b200.worlds import WorldConfig, make_loopback_world  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [1 << 20, 16 << 20, 128 << 20]
log = []
orig = DeviceRegistry.enqueue_transfer


def traced(self, src, dst, size, wait=None):
    t_host = time.perf_counter()
    dev = None
    tok = orig(self, src, dst, size, wait=wait)
    log.append((t_host, size, tok))
    return tok


DeviceRegistry.enqueue_transfer = traced
ngpu = N.gpu_count()
cfg = WorldConfig(ranks=2, device_aware=True, capacity=4 * max(sizes) + (64 << 20),
                  gpus=[0, 1 if ngpu > 1 else 0])
comms = make_loopback_world(cfg)
arrived = []


def h_pong(m, arg, ctx):
    ctx.comm.mp_send(MobileRef(0, 0), h_ping, arg)
    ctx.comm.runtime.destroy_object(arg)


def h_ping(m, arg, ctx):
    arrived.append((time.perf_counter(), arg))


ids = [(c.register_handler(h_pong), c.register_handler(h_ping)) for c in comms]
h_pong_id, h_ping = ids[0]
for c in comms:
    c.create_mobile_object(b"pp")
    c.runtime.register_kernel("touch", gpu_sim=Touch(), cost=1e-6)
exchange_all(comms)
rt0 = comms[0].runtime
for size in sizes:
    obj = rt0.create_object((size,), dtype=np.uint8)
    np.copyto(rt0.request_data(obj, write=True).get(), np.zeros(size, np.uint8))
    rt0.release(obj)
    t = rt0.task().device(DeviceType.GPU_SIM)
    t.arg(obj).read_write()
    rt0.wait(t.submit("touch"))
    for it in range(6):
        log.clear()
        arrived.clear()
        t0 = time.perf_counter()
        comms[0].mp_send(MobileRef(1, 0), h_pong_id, obj)
        drive(comms, until=lambda: len(arrived) == 1)
        t_arr = arrived[0][0]
        w = arrived[0][1]
        drive(comms, until=lambda: w.written)
        t1 = time.perf_counter()
        for (_, _, tok) in log:
            tok.wait()
        # device durations of the copies: events recorded before/after are
        # not available, so time each copy against the previous token
        parts = [f"{(th - t0) * 1e6:.0f}us" for (th, _, _) in log]
        print(f"size {size} it {it}: round trip {(t1 - t0) * 1e6:.0f} us, handler(ping) at "
              f"{(t_arr - t0) * 1e6:.0f} us, copies enqueued at {parts}", flush=True)
        rt0.destroy_object(w)
    rt0.destroy_object(obj)
shutdown_all(comms)
