import cProfile, pstats, sys, os
sys.path.insert(0, "/root/repo")
from paper_2303_02543_b200.pingpong import run_pingpong
run_pingpong([8], iterations=50, path="direct", verify=False, gpus=[0,1])
pr = cProfile.Profile(); pr.enable()
rep = run_pingpong([8], iterations=1000, path="direct", verify=False, gpus=[0,1])
pr.disable()
print("one-way us:", rep.rows[0]["mean_latency_s"] * 1e6)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(45)
