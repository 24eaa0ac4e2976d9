"""cProfile of the direct-path ping-pong host code (8 B, 300 round trips):
tottime and cumtime views."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200.pingpong import run_pingpong  # noqa: E402

size = int(os.environ.get("PP_SIZE", "8"))
run_pingpong([size], iterations=50, path="direct", verify=False)  # warm-up
pr = cProfile.Profile()
pr.enable()
rep = run_pingpong([size], iterations=300, path="direct", verify=False)
pr.disable()
print("one-way us (under cProfile):", rep.rows[0]["mean_latency_s"] * 1e6)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(40)
st.sort_stats("cumulative").print_stats(60)
