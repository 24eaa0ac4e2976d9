"""One process driving several GPUs (the reference's in-process ranks):
cfg3-style x-bands, device-timed steps, vs the same work on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

n = N.gpu_count()
dom, steps = (32768, 32768, 1), int(sys.argv[1]) if len(sys.argv) > 1 else 200
for g in sorted({1, n}):
    grid = ChunkGrid(dom, ranks=g, grid=(8 * g, 1, 1))
    s = JacobiSolver(grid, gpus=list(range(g)))
    s.upload()
    s.run(20, residual=False)
    s.sync()
    t0 = time.perf_counter()
    s.run(steps, residual=True)
    s.sync()
    dt = time.perf_counter() - t0
    print(f"{g} GPU(s) in one process: {dom[0] * dom[1] * steps / dt / 1e9:.1f} GLUPS "
          f"(persistent={s.persistent})", flush=True)
    s.close()
