"""Single small run of one slab kernel variant (for compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

n = int(os.environ.get("DOM", "2048"))
g = int(os.environ.get("G", "8"))
variant = int(os.environ.get("VARIANT", "3"))
steps = int(os.environ.get("STEPS", "3"))
s = JacobiSolver(ChunkGrid((n, n, 1), grid=(g, g, 1)), variant=variant)
s.upload()
s.run(steps, residual=True, graph=False)
f = s.download()
s.close()
print("variant", variant, "ok", np.array_equal(f, O.jacobi_c((n, n, 1), steps)))
