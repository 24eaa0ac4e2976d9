"""Generic task path throughput (no messages): submit + issue + retire of
native-kernel tasks through Runtime, tasks/s.  Independent chains over
`nobj` objects (each task READ_WRITEs one object: RAW/WAW chains per object,
independent across objects), optionally under cProfile.

python tools/task_rate.py [ntasks] [nobj] [--profile]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2303_02543_b200.devices import DeviceDescriptor, DeviceRegistry, DeviceType  # noqa: E402
from paper_2303_02543_b200.native_kernels import Mix  # noqa: E402
from paper_2303_02543_b200.runtime import Runtime  # noqa: E402

ntasks = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20000
nobj = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 8
reg = DeviceRegistry()
reg.register_device(DeviceDescriptor(device_id=0, device_type=DeviceType.GPU_SIM,
                                     memory_capacity=64 << 20, compute_stream_count=5, gpu=0))
rt = Runtime(reg)
rt.register_kernel("mix", gpu_sim=Mix(3))
objs = [rt.create_object((4096,), dtype=np.uint8) for _ in range(nobj)]


def run(n):
    tasks = []
    for i in range(n):
        t = rt.task().device(DeviceType.GPU_SIM)
        t.arg(objs[i % nobj]).read_write()
        tasks.append(t.submit("mix"))
        if len(tasks) >= 256:
            rt.progress(advance=False)
            tasks = [x for x in tasks if not x.done]
    rt.wait_all(tasks)
    rt.synchronize()


run(2000)
t0 = time.perf_counter()
if "--profile" in sys.argv:
    pr = cProfile.Profile()
    pr.enable()
    run(ntasks)
    pr.disable()
else:
    run(ntasks)
dt = time.perf_counter() - t0
print(f"tasks {ntasks}, objects {nobj}: {ntasks / dt:,.0f} tasks/s ({dt / ntasks * 1e6:.1f} us/task)")
if "--profile" in sys.argv:
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
