"""Device timing of the 3D volume update (development probe).

python tools/probe_3d.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rows_list = [int(r) for r in os.environ.get("ROWS", "0").split(",")]
cases = [((512, 512, 512), (2, 2, 2)), ((1024, 1024, 768), (2, 2, 2)),
         ((1024, 1024, 768), (1, 1, 1))]
if os.environ.get("QUICK"):
    cases = cases[1:2]
for (dom, grid), rows in [(c, r) for c in cases for r in rows_list]:
    print(f"rows={rows or 'default'}", end=" ")
    s = JacobiSolver(ChunkGrid(dom, grid=grid), rows=rows or None)
    s.upload()
    s.run_timed(3)
    up, ha, tot = s.run_timed(steps)
    cells = dom[0] * dom[1] * dom[2]
    print(f"{dom} grid {grid}: {tot / steps:.3f} ms/step  update {up / steps:.3f} ms  "
          f"halo {ha / steps:.3f} ms  GLUPS {cells * steps / (tot / 1e3) / 1e9:.1f}  "
          f"update-kernel {16 * cells * steps / (up / 1e3) / 1e9:.0f} GB/s", flush=True)
    s.close()
