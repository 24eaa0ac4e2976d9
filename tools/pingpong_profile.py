"""cProfile of the direct-path ping-pong host code (4 KiB, 300 round trips)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.pingpong import run_pingpong  # noqa: E402

run_pingpong([4096], iterations=50, path="direct", verify=False)  # warm-up
pr = cProfile.Profile()
pr.enable()
rep = run_pingpong([4096], iterations=300, path="direct", verify=False)
pr.disable()
print("one-way us:", rep.rows[0]["mean_latency_s"] * 1e6)
pstats.Stats(pr).sort_stats("tottime").print_stats(28)
