"""One slab_wave2_kernel launch at cfg2 shape for ncu (steps passes / 2):

    ncu --set full --import-source on -k regex:slab_wave -c 1 \
        python tools/ncu_wave2.py [steps] [grid]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
grid = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "8,8,1").split(","))
X = int(os.environ.get("NCU_X", "16384"))
s = JacobiSolver(ChunkGrid((X, X, 1), grid=grid))
s.upload()
s.run(steps, residual=True)
s.sync()
s.close()
print("ok", steps, grid)
