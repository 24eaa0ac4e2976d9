"""Repeatability of small-message ping-pong latency across worlds: runs
run_pingpong on a few sizes, several fresh worlds each, and prints the
one-way latency of every world (µs).  python tools/pingpong_modes.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.pingpong import run_pingpong  # noqa: E402

n = N.gpu_count()
gpus = [0, 1 if n > 1 else 0]
for size in (8, 4096, 1 << 20):
    lat = []
    for rep in range(6):
        r = run_pingpong([size], iterations=200, path="direct", gpus=gpus, verify=os.environ.get("PP_VERIFY", "0") == "1")
        lat.append(round(r.rows[0]["mean_latency_s"] * 1e6, 1))
    print(f"spin={os.environ.get('HRT_SPIN_US', 'default')} size {size}: one-way us per world {lat}",
          flush=True)
