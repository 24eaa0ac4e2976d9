"""One volume_wave2_kernel launch at paper3d shape for ncu (steps passes / 2):

    ncu --set full --import-source on -k regex:volume_wave2 -c 1 \
        python tools/ncu_vol2.py [steps] [X,Y,Z] [grid]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dom = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1024,1024,768").split(","))
grid = tuple(int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "8,1,1").split(","))
s = JacobiSolver(ChunkGrid(dom, grid=grid))
s.upload()
s.run(steps, residual=True)
s.sync()
k = s.steps_per_pass
s.close()
print("ok", steps, dom, grid, k)
