"""Residual-history debugging probe: per-step residual and field vs oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

for dom, grid in [((2048, 2048, 1), (8, 8, 1)), ((2048, 2048, 1), (2, 2, 1)),
                  ((1024, 2048, 1), (1, 2, 1)), ((4096, 4096, 1), (8, 8, 1)),
                  ((16384, 16384, 1), (8, 8, 1)), ((16384, 16384, 1), (2, 32, 1))]:
    for variant in (1, 2):
        for steps in (2, 4):
            s = JacobiSolver(ChunkGrid(dom, grid=grid), variant=variant)
            s.upload()
            s.run(steps, residual=True)
            f = s.download()
            r = s.residual_history()
            s.close()
            ref, rr = O.jacobi_c(dom, steps, residual=True)
            print(dom, grid, "v", variant, "steps", steps, "field_ok", np.array_equal(f, ref),
                  "resid", r.tolist(), "ref", rr.tolist(), flush=True)
