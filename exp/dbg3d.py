import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver
from oracle import oracle as O
for dom, grid in [((12, 20, 10), (1, 1, 1)), ((40, 36, 70), (2, 1, 1))]:
    rng = np.random.default_rng(1)
    init = rng.random(dom) * 4.0 - 1.0
    s = JacobiSolver(ChunkGrid(dom, grid=grid))
    print("two_step", s.two_step)
    s.upload(init); s.run(4, residual=True); got = s.download(); res = s.residual_history(); s.close()
    resid = []
    ref = O.jacobi_reference(dom, 4, initial=init, residuals=resid)
    bad = np.argwhere(got != ref)
    print(dom, grid, "bad", len(bad), "of", got.size)
    if len(bad):
        for ax in range(3):
            print("  axis", ax, "values", np.unique(bad[:, ax])[:20], "...", len(np.unique(bad[:, ax])))
        i, j, k = bad[0]
        print("  first", bad[0], got[i, j, k], ref[i, j, k])
    print("  resid", np.array_equal(res, np.array(resid)), res, resid)
