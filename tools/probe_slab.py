"""Quick device timing of the slab update kernel on cfg2 (development probe).

python tools/probe_slab.py [steps] [rows...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rows_list = [int(r) for r in sys.argv[2:]] or [64]
X = Y = 16384
cells = X * Y
variants = [int(v) for v in os.environ.get("PROBE_VARIANTS", "0,1").split(",")]
for variant, rows in [(v, r) for v in variants for r in rows_list]:
    print(f"variant {variant}", end=" ")
    s = JacobiSolver(ChunkGrid((X, Y, 1), grid=(8, 8, 1)), rows=rows, variant=variant)
    s.upload()
    s.run_timed(5)
    up, ha, tot = s.run_timed(steps)
    glups = cells * steps / (tot / 1e3) / 1e9
    upd_gbs = 16 * cells * steps / (up / 1e3) / 1e9
    print(f"rows={rows}: total {tot/steps:.3f} ms/step  update {up/steps:.3f} ms  halo {ha/steps:.4f} ms"
          f"  GLUPS {glups:.1f}  update-kernel {upd_gbs:.0f} GB/s", flush=True)
    for resid, graph in ((False, True), (False, False), (True, False)):
        s.run(2, residual=resid, graph=graph)
        s.sync()
        t0 = time.perf_counter()
        s.run(steps, residual=resid, graph=graph)
        s.sync()
        dt = time.perf_counter() - t0
        print(f"   run(residual={resid}, graph={graph}): {dt/steps*1e3:.3f} ms/step "
              f"GLUPS {cells*steps/dt/1e9:.1f}", flush=True)
    s.close()
