"""Two-process message ping-pong over the TCP byte transport, one GPU per
process (torchrun --nproc-per-node 2).  Payloads go GPU->GPU through CUDA
IPC device locators when HRT_DEVICE_AWARE=1 (the default here), else they
are staged through host memory and the socket.  Rank 0 prints one JSON
line per transport mode; argv[1] (optional) is an output JSON path.

Env: MP_SIZES ("8..16777216" powers of two, default 8..16777216), MP_ITERS (default 50),
MP_MODES ("direct,staged").
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.pingpong import parse_sizes, pingpong_process  # noqa: E402
from paper_2303_02543_b200.worlds import WorldConfig, build_rank_runtime, init_from_env  # noqa: E402

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
base_port = int(os.environ.get("MASTER_PORT", "29500")) + 17
sizes = parse_sizes(os.environ.get("MP_SIZES", "8..16777216"))
iters = int(os.environ.get("MP_ITERS", "50"))
ngpu = N.gpu_count()
out = {"rows": {}}
for k, mode in enumerate(os.environ.get("MP_MODES", "direct,staged").split(",")):
    os.environ.update(HRT_TRANSPORT="tcp", HRT_RANK=str(rank),
                      HRT_PEERS=",".join(f"127.0.0.1:{base_port + 8 * k + r}" for r in range(world)),
                      HRT_DEVICE_AWARE="1" if mode == "direct" else "0")
    cfg = WorldConfig(ranks=world, gpus=list(range(ngpu)),
                      capacity=max(64 << 20, 4 * max(sizes) + (32 << 20)))
    comm = init_from_env(build_rank_runtime(cfg, rank))
    rep = pingpong_process(comm, sizes, iterations=iters, verify=True)
    if rep is not None:
        out["rows"][mode] = rep.rows
        out["stats_" + mode] = rep.meta["stats"]
        for r in rep.rows:
            print(json.dumps({"mode": mode, "size": r["size_bytes"],
                              "us": round(r["mean_latency_s"] * 1e6, 2),
                              "GBps": round(r["bandwidth_Bps"] / 1e9, 3)}), flush=True)
if rank == 0 and len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
if rank == 0:
    st = out.get("stats_direct", {})
    print(f"MP_PINGPONG PASS direct_staging_copies={st.get('staging_copies', -1)} "
          f"direct_device_copies={st.get('device_copies', -1)}", flush=True)
