"""Race hunt: repeat short runs per kernel variant and compare field and
residual with a reference run of the LDG variant on one chunk."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

dom = (int(os.environ.get("DOM", "16384")),) * 2 + (1,)
steps = int(os.environ.get("STEPS", "10"))
reps = int(os.environ.get("REPS", "4"))


def run(grid, variant, halo_sync=False):
    s = JacobiSolver(ChunkGrid(dom, grid=grid), variant=variant)
    s.upload()
    s.run(steps, residual=True, graph=False)
    f, r = s.download(), s.residual_history()
    s.close()
    return f, r


ref_f, ref_r = run((1, 1, 1), 0)
print("ref resid", ref_r[:5].tolist(), flush=True)
for variant in [int(v) for v in os.environ.get("VARIANTS", "0,1,2").split(",")]:
    for grid in ((8, 8, 1), (2, 32, 1), (1, 1, 1)):
        bad = 0
        for _ in range(reps):
            f, r = run(grid, variant)
            ok = np.array_equal(f, ref_f) and np.array_equal(r, ref_r)
            if not ok:
                bad += 1
                nd = int((f != ref_f).sum())
                print(f"  v{variant} {grid}: field diff cells {nd}, resid diff idx "
                      f"{np.nonzero(r != ref_r)[0][:5].tolist()}", flush=True)
        print(f"variant {variant} grid {grid}: {bad}/{reps} bad", flush=True)
