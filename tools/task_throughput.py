"""Task-protocol throughput: run_jacobi3d(engine="tasks") — the reference's
own per-chunk protocol (pack -> mp_send -> unpack -> update tasks, handlers,
wrappers) executed by the B200 runtime.  Reports tasks/s (every pack,
unpack and update is one task) next to the reference's CPU figures
(1,372-6,021 tasks/s, ~166 us/task).  Writes JSON to argv[1].
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.jacobi import run_jacobi3d  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "task_throughput.json"
rows = []
for dom, grid, steps, aware in [((1024, 1024, 1), (16, 16, 1), 10, True),
                                ((1024, 1024, 1), (16, 16, 1), 10, False),
                                ((4096, 4096, 1), (16, 16, 1), 10, True),
                                ((512, 512, 512), (4, 4, 4), 10, True)]:
    run_jacobi3d(dom, steps=2, grid=grid, engine="tasks", device_aware=aware)  # warm-up
    t0 = time.perf_counter()
    rep, cs, arr = run_jacobi3d(dom, steps=steps, grid=grid, engine="tasks", device_aware=aware)
    dt = time.perf_counter() - t0
    tasks = sum(rep.meta["tasks"])
    cells = dom[0] * dom[1] * dom[2]
    row = dict(domain=dom, grid=grid, steps=steps, device_aware=aware, tasks=tasks,
               seconds=round(dt, 3), tasks_per_s=round(tasks / dt, 1),
               us_per_task=round(dt / tasks * 1e6, 2), glups=round(cells * steps / dt / 1e9, 3))
    rows.append(row)
    print(row, flush=True)
json.dump(rows, open(out, "w"), indent=1)
