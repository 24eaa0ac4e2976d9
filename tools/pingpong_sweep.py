"""cfg4: device-to-device message ping-pong sweep 8 B .. 256 MiB between two
GPUs — the B200 direct path (device locators + cudaMemcpyPeerAsync) vs the
reference's host-staged protocol on the same hardware — plus the raw
cudaMemcpyPeerAsync sweep (achievable peak).  Writes JSON to argv[1].

The reference's own CPU numbers (loopback, wall clock, this container) are
in BASELINE.md §2: staging 0.26-0.79 GB/s, direct 0.33-0.86 GB/s.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.pingpong import parse_sizes, peer_copy_sweep, run_pingpong  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "pingpong_sweep.json"
top = int(os.environ.get("PP_TOP", str(256 << 20)))
sizes = parse_sizes(f"8..{top}")
n = N.gpu_count()
gpus = [0, 1 if n > 1 else 0]
res = {"gpus": gpus, "rows": {}}
for path in ("direct", "staging"):
    iters = [100 if s < (64 << 20) else 20 for s in sizes]
    rows = []
    for s, it in zip(sizes, iters):
        rep = run_pingpong([s], iterations=it, path=path, gpus=gpus, verify=True)
        rows.append(rep.rows[0])
        print(path, s, f"{rep.rows[0]['mean_latency_s'] * 1e6:.1f} us",
              f"{rep.rows[0]['bandwidth_Bps'] / 1e9:.2f} GB/s", flush=True)
    res["rows"][path] = rows
raw = peer_copy_sweep(sizes, gpus[0], gpus[1], iterations=50)
res["rows"]["raw_peer_copy"] = raw.rows
for r in raw.rows:
    print("raw", r["size_bytes"], f"{r['mean_latency_s'] * 1e6:.2f} us",
          f"{r['bandwidth_Bps'] / 1e9:.1f} GB/s", flush=True)
with open(out_path, "w") as fh:
    json.dump(res, fh, indent=1)
