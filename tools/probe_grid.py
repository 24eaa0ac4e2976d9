"""Device timing of one step engine across decompositions (development probe):
which chunk shapes / push settings cost kernel efficiency.

PROBE_DOMAIN=16384x16384 PROBE_GRIDS=8x8,64x1,1x64 PROBE_PUSH=1,0 python tools/probe_grid.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
X, Y = (int(v) for v in os.environ.get("PROBE_DOMAIN", "16384x16384").split("x"))
grids = [tuple(int(v) for v in g.split("x")) for g in
         os.environ.get("PROBE_GRIDS", "8x8,64x1,1x64,1x1").split(",")]
pushes = [p != "0" for p in os.environ.get("PROBE_PUSH", "1,0").split(",")]
rows = int(os.environ.get("PROBE_ROWS", "0")) or None
cells = X * Y
for g in grids:
    for push in pushes:
        s = JacobiSolver(ChunkGrid((X, Y, 1), grid=(g[0], g[1], 1)), rows=rows, push=push)
        s.upload()
        s.run_timed(5)
        up, ha, tot = s.run_timed(steps)
        print(f"grid {g[0]}x{g[1]} push={int(push)}: {tot / steps:.4f} ms/step "
              f"update {up / steps:.4f} halo {ha / steps:.4f}  GLUPS {cells * steps / tot / 1e6:.1f}"
              f"  kernel {16 * cells * steps / up / 1e6:.0f} GB/s", flush=True)
        s.close()
