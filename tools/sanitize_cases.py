"""Small runs of every bulk-copy (TMA) / mbarrier kernel for
compute-sanitizer (racecheck, synccheck, memcheck): tools/sanitize.sh
runs this file under each tool.  Each case is checked against the C oracle
too, so a sanitizer-clean run is also a correct one.

    python tools/sanitize_cases.py [case ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

# name -> (domain, grid, steps, env, solver kwargs)
CASES = {
    # slab_wave2_kernel (two steps per pass), 512- and 256-wide tiles
    "wave2": ((260, 1030, 1), (2, 2, 1), 6, {"HRT_FUSE2": "2"}, {}),
    "wave2_narrow": ((200, 512, 1), (2, 2, 1), 5, {"HRT_FUSE2": "2"}, {}),
    # slab_wave_kernel (persistent, one step per pass, side arrays)
    "wave": ((260, 1030, 1), (2, 2, 1), 3, {"HRT_FUSE2": "0"}, {}),
    # slab_update_tma4_kernel (tile launches with fused push)
    "tma4": ((130, 1030, 1), (2, 2, 1), 3, {}, {"persistent": False}),
    # slab_update_tma_kernel (variant 1)
    "tma": ((130, 600, 1), (2, 2, 1), 3, {}, {"variant": 1}),
    # volume_update_tma_kernel (3D ring)
    "volume_tma": ((40, 36, 70), (2, 1, 1), 3, {}, {}),
}


def run(name):
    dom, grid, steps, env, kw = CASES[name]
    os.environ.update(env)
    try:
        s = JacobiSolver(ChunkGrid(dom, grid=grid), **kw)
        init = np.random.default_rng(3).random(dom) * 2.0
        s.upload(init)
        s.run(steps, residual=True)
        got, res = s.download(), s.residual_history()
        s.close()
    finally:
        for k in env:
            os.environ.pop(k, None)
    rr = []
    ref = O.jacobi_reference(dom, steps, initial=init, residuals=rr)
    ok = np.array_equal(got, ref) and np.array_equal(res, np.array(rr))
    print(f"case {name}: {'OK' if ok else 'DIFF'}", flush=True)
    return ok


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    sys.exit(0 if all([run(n) for n in names]) else 1)
