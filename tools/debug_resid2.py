"""Residual-history debugging probe 2: long runs, (8,8,1) vs (2,32,1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

dom = (16384, 16384, 1)
for steps in (3, 10, 100, 1000):
    hist = {}
    for grid in ((8, 8, 1), (2, 32, 1), (8, 8, 1)):
        s = JacobiSolver(ChunkGrid(dom, grid=grid))
        s.upload()
        s.run(steps, residual=True)
        r = s.residual_history()
        s.close()
        key = grid if grid not in hist else (grid, "again")
        hist[key] = r
        print(steps, grid, r[:4].tolist(), flush=True)
    vals = list(hist.values())
    print("steps", steps, "equal:", [np.array_equal(vals[0], v) for v in vals], flush=True)
