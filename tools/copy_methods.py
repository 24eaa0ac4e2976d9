"""GPU->GPU copy methods over NVLink: copy engine vs SM copy kernels (pull
on the destination, push from the source), CUDA-event timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.pingpong import peer_copy_sweep  # noqa: E402

sizes = [1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]
for method, blocks in (("ce", 0), ("sm_pull", 0), ("sm_push", 0), ("sm_pull", 1184),
                       ("sm_push", 1184), ("sm_push", 296)):
    rep = peer_copy_sweep(sizes, 0, 1, iterations=20, method=method, blocks=blocks)
    print(method, blocks, " ".join(f"{r['size_bytes'] >> 20}M:{r['bandwidth_Bps'] / 1e9:.0f}"
                                  for r in rep.rows), flush=True)
