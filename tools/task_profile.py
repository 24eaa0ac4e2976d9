import cProfile, pstats, sys
sys.path.insert(0, "/root/repo")
from paper_2303_02543_b200.jacobi import run_jacobi3d
run_jacobi3d((1024, 1024, 1), steps=2, grid=(16, 16, 1), engine="tasks", device_aware=True)
pr = cProfile.Profile(); pr.enable()
run_jacobi3d((1024, 1024, 1), steps=5, grid=(16, 16, 1), engine="tasks", device_aware=True)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(30)
