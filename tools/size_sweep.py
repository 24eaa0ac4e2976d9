"""GLUPS of the default engine vs domain size (square slabs, 8x8 chunks,
device-timed run of `steps` iterations after a warm-up) — where the
two-step wavefront saturates, and the one-step kernel beside it
(HRT_FUSE2=0 in a second process).  python tools/size_sweep.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for n in (1024, 2048, 4096, 8192, 16384, 32768):
    s = JacobiSolver(ChunkGrid((n, n, 1), grid=(8, 8, 1)))
    s.upload()
    s.run_timed(8)
    up, ha, tot = s.run_timed(steps)
    print(f"{n}x{n} 8x8 chunks two_step={s.two_step}: {n * n * steps / tot / 1e6:.1f} GLUPS "
          f"({tot / steps * 1e3:.1f} us/step)", flush=True)
    s.close()
