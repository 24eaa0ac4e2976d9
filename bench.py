"""Headline benchmark: Jacobi GLUPS on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One bench *step* is one complete job of the workload: the chunked field is
reset to the reference's initial state (interior 0.0, Dirichlet 1.0,
jacobi.py:382-395) and advanced ``iters`` Jacobi iterations (halo faces +
7-point update + L-inf residual per iteration), exactly as
run_jacobi3d(domain, grid=..., steps=iters) does (jacobi.py:281-462).

* N=1: cfg2 — 16384^2 float64, 8x8 chunks, 1000 iterations (BASELINE
  configs[1]).  N>1: cfg3 — 32768^2 float64, 8 chunks per GPU, 1000
  iterations, one process per GPU, faces between processes by NCCL
  send/recv inside libhrt_b200 (strong scaling).
* ``value``: GLUPS with the field resident in HBM, CUDA events on the solver
  stream, max over ranks.  ``e2e``: the same job through the public API
  (JacobiSolver.upload from pinned host memory -> run -> download to pinned
  host memory + residual history), H2D/D2H inside the timed region.
* ``roofline``: the slab update kernel, 16 algorithmic bytes per lattice
  update (read u, write u'), CUDA events around every update launch.
* ``cpu_baseline``: the C/OpenMP oracle (oracle/, a port of the reference's
  jacobi_reference) on this host's cores, bounded sample, rank 0 at N=1.
* ``--impl reference``: the reference CPU path (the oracle port, all host
  threads) on the same workload, bounded samples per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Jacobi GLUPS at 1/2/4/8 B200 (% HBM roofline); halo msg GB/s vs size"
UNIT = "GLUPS"
BYTES_PER_UPDATE = 16  # read u once, write u' once (float64)
# cfg3: 8 chunks per GPU as x-bands (the reference's rank = lin*ranks//n with
# x-fastest lin): faces between processes are contiguous rows, pushed by the
# update kernel straight into the neighbour's ghost row over NVLink (IPC)
CFG3_GRIDS = {n: (8 * n, 1, 1) for n in (1, 2, 4, 8)}


def workload(name: str, n: int):
    if name == "auto":
        name = "cfg2" if n == 1 else "cfg3"
    if name == "cfg1":
        return dict(name="cfg1", desc="Jacobi 2D 1024x1024 float64, 4x4 blocks, 100 iterations",
                    domain=(1024, 1024, 1), grid=(4, 4, 1), iters=100)
    if name == "cfg2":
        return dict(name="cfg2",
                    desc="Jacobi 2D 16384x16384 float64, 8x8 blocks, 1000 iterations on 1 B200",
                    domain=(16384, 16384, 1), grid=(8, 8, 1), iters=1000)
    if name == "cfg3":
        grid = CFG3_GRIDS.get(n, (8, n, 1))
        return dict(name="cfg3",
                    desc=f"Jacobi 2D 32768x32768 float64 strong scaling, 8 blocks per GPU "
                         f"(grid {grid[0]}x{grid[1]}), 1000 iterations on {n} B200",
                    domain=(32768, 32768, 1), grid=grid, iters=1000)
    if name == "cfg5":
        return dict(name="cfg5",
                    desc=f"many-small-tasks: 65536 blocks of 256x256 (grid 256x256), dependency "
                         f"chains (each block-step needs its neighbours' previous step), 100 "
                         f"iterations on {n} B200",
                    domain=(65536, 65536, 1), grid=(256, 256, 1), iters=100)
    if name == "paper3d":
        # the paper's Jacobi3D size, x-bands of 8 chunks per GPU
        grid = (8 * n, 1, 1)
        return dict(name="paper3d",
                    desc=f"Jacobi 3D 1024x1024x768 float64 (7-point), 8 chunks per GPU "
                         f"(grid {grid[0]}x1x1), 100 iterations on {n} B200",
                    domain=(1024, 1024, 768), grid=grid, iters=100)
    raise SystemExit(f"unknown workload {name}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                mx = max(mx, float(f[2].split()[0]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(wl, budget_s: float = 15.0):
    """The C/OpenMP oracle (oracle/jacobi_oracle.c, port of jacobi.py:49-67)
    on a bounded sample of the workload: the full domain, k sweeps."""
    from oracle import oracle as O

    O.build()
    O.use_all_host_threads()
    X, Y, Z = wl["domain"]
    if Z != 1:  # 3D: the C oracle on the full volume, 2 sweeps
        t0 = time.perf_counter()
        O.jacobi_c(wl["domain"], 2)
        dt = time.perf_counter() - t0
        return {"value": round(X * Y * Z * 2 / dt / 1e9, 4), "unit": UNIT,
                "cores": O.cpu_threads(), "kind": "port",
                "sample": f"{X}x{Y}x{Z} volume, 2 of the {wl['iters']} sweeps incl. allocation "
                          f"({dt:.1f} s), oracle/jacobi_oracle.c OpenMP, host of the GPU box"}
    slab = O.CpuSlab(X, Y)
    t0 = time.perf_counter()
    slab.sweep(1)
    t1 = time.perf_counter() - t0
    k = max(2, min(wl["iters"], int(budget_s / max(t1, 1e-4))))
    t0 = time.perf_counter()
    slab.sweep(k)
    dt = time.perf_counter() - t0
    slab.close()
    return {"value": round(X * Y * k / dt / 1e9, 4), "unit": UNIT, "cores": O.cpu_threads(),
            "kind": "port",
            "sample": f"{X}x{Y} slab, {k} of the {wl['iters']} sweeps ({dt:.1f} s, setup "
                      f"excluded), oracle/jacobi_oracle.c OpenMP, host of the GPU box"}


def reduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


_JSON_FD = None  # the real stdout while library chatter is routed to stderr


def quiet_stdout():
    """Route fd 1 to stderr so library banners printed during communicator
    setup (e.g. NCCL's version line) do not share stdout with the JSON line."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict):
    text = json.dumps(line) + "\n"
    if _JSON_FD is None:
        print(text, end="", flush=True)
    else:
        os.write(_JSON_FD, text.encode())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


MSG_SIZES = [8, 64 << 10, 1 << 20, 8 << 20, 64 << 20, 256 << 20]
NVLINK_GBS = 900.0  # NVLink 5, per direction (nominal)


def messages_record():
    """The metric's second half, "halo msg GB/s vs size" (SURVEY.md §8(d),
    pingpong.py:126-147): one-way latency and GB/s of a device-resident
    object through the public message path (``run_pingpong``, path
    "direct": mp_send with device locators, the copy ordered on the GPU,
    byte identity verified every round trip), beside the raw copy of the
    same size timed with CUDA events.  GPU0 <-> GPU1 over NVLink when two
    GPUs are visible, else a same-GPU D2D copy."""
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.pingpong import peer_copy_sweep, run_pingpong

    n = N.gpu_count()
    gpus = [0, 1] if n >= 2 else [0, 0]
    peer = gpus[0] != gpus[1]
    hbm, _ = peaks()
    # a peer copy moves each byte once over the link; a D2D copy reads and
    # writes HBM, so its size/time ceiling is half the copy peak
    peak = NVLINK_GBS if peer else hbm / 2
    raw = peer_copy_sweep(MSG_SIZES, gpus[0], gpus[1], iterations=20)
    rows = []
    for size, rr in zip(MSG_SIZES, raw.rows):
        it = 40 if size < (64 << 20) else 10
        rep = run_pingpong([size], iterations=it, path="direct", gpus=gpus)
        r = rep.rows[0]
        gbs = r["bandwidth_Bps"] / 1e9
        raw_gbs = rr["bandwidth_Bps"] / 1e9
        rows.append({"size_bytes": size, "iters": it,
                     "one_way_us": round(r["mean_latency_s"] * 1e6, 2), "gbs": round(gbs, 3),
                     "raw_copy_us": round(rr["mean_latency_s"] * 1e6, 2),
                     "raw_copy_gbs": round(raw_gbs, 2),
                     "share_of_raw": round(gbs / raw_gbs, 4) if raw_gbs else None,
                     "frac_of_peak": round(gbs / peak, 4)})
    return {"path": "mp_send direct (device locator + GPU-ordered copy), run_pingpong",
            "gpus": gpus, "link": "NVLink 5 peer" if peer else "same-GPU D2D (one GPU visible)",
            "peak_gbs": peak,
            "peak_source": "NVLink 5 nominal 900 GB/s per direction" if peer else
                           "MEASURED_PEAKS.json hbm_gbs / 2 (a D2D copy reads and writes)",
            "raw": "cudaMemcpyAsync/cudaMemcpyPeerAsync on one stream, CUDA events",
            "rows": rows}


def config_for(wl: dict, world: int, iters: int) -> dict:
    """The ``config`` object of both arms (ours and --impl reference)."""
    X, Y, Z = wl["domain"]
    nchunks = wl["grid"][0] * wl["grid"][1] * wl["grid"][2]
    return {"workload": wl["desc"], "domain": list(wl["domain"]), "grid": list(wl["grid"]),
            "iterations_per_step": iters, "chunks_per_gpu": nchunks // world,
            "parallelism": f"domain decomposition over {world} GPU(s), one process each",
            "l2": f"no flush needed: field {X * Y * Z * 8 / 2**30:.2f} GiB >> 126 MB L2",
            "bitexact": "float64 bitwise == reference (Markstein /6 == IEEE, sum order kept)",
            "residual": "L-inf per iteration, fused"}


def run_ours(args):
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import PinnedBuffer
    from paper_2303_02543_b200.distributed import DistributedJacobi, init_process
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    if args.gpus > 1:
        quiet_stdout()
    rank, world, local = init_process("nccl") if args.gpus > 1 else (0, 1, 0)
    N.require_gpu(local)
    wl = workload(args.workload, world)
    if args.grid:
        wl["grid"] = tuple(int(x) for x in args.grid.split(","))
        wl["desc"] += f" [grid override {args.grid}]"
    iters = args.iters or wl["iters"]
    X, Y, Z = wl["domain"]
    cells = X * Y * Z
    grid = ChunkGrid(wl["domain"], ranks=world, grid=wl["grid"])
    if world == 1:
        solver = JacobiSolver(grid, gpus=[local], variant=args.variant, rows=args.rows)
    else:
        solver = DistributedJacobi(grid, rank, world, local, variant=args.variant, rows=args.rows)
    my_cells = solver.field_elems
    nbytes = my_cells * 8
    g = solver.used_gpus[0]
    st = solver.streams[g]

    solver.upload(nonneg=True)  # the reference's initial state (interior 0.0)
    # the resident initial state for the device-timed job: keep a copy on HBM
    init_field = solver._field()

    def device_job():
        """reset to the initial state (device-resident) + iters iterations;
        returns (update_ms, halo_ms, total_ms) from CUDA events."""
        solver._chunk_copies(True, 0, init_field, lambda gg: solver.streams[gg])
        solver.steps_done = 0
        return solver.run_timed(iters, residual=True)

    # warm-up (also instantiates plans/graphs, faults in pages)
    for _ in range(args.warmup):
        device_job()
    barrier(world)
    st.synchronize()
    upd = halo = tot = 0.0
    with ClockSampler(local) as clk:
        t_start = st.record()
        for _ in range(args.steps):
            u, h, t = device_job()
            upd += u
            halo += h
            tot += t
        t_end = st.record()
        st.synchronize()
    region_ms = t_start_elapsed = 0.0
    import ctypes

    ms = ctypes.c_float()
    N.call("hrt_token_elapsed_ms", ctypes.c_uint64(t_start.token_id), ctypes.c_uint64(t_end.token_id),
           ctypes.byref(ms))
    region_ms = reduce_max(ms.value, world)
    barrier(world)
    value = cells * iters * args.steps / (region_ms / 1e3) / 1e9

    # roofline of the dominant kernel: per-launch algorithmic bytes / average
    # launch duration (CUDA events around every launch on the solver stream).
    # Persistent mode runs all iterations of a job in one wavefront launch.
    # Two-step passes (slab_wave2_kernel) read u and write u'' once per TWO
    # updates: their algorithmic bytes are 8 per lattice update; the naive
    # one-step algorithm's 16 B/update is reported beside it.
    persistent = bool(getattr(solver, "persistent", False))
    # steps one fused pass covers (2: slab_wave2_kernel, 1:
    # one step per pass); a run of `iters` steps is n_single one-step sweeps
    # plus n_pass fused passes, each reading u once and writing once: 16
    # algorithmic bytes per cell and sweep/pass
    k = solver.steps_per_pass
    if k == 2 and iters >= 4:
        n_pass = (iters // 4) * 2
        n_single = iters - 2 * n_pass
    else:
        k, n_pass, n_single = 1, 0, iters
    two_step = k > 1
    launches_per_job = (int(n_single > 0) + int(n_pass > 0)) if persistent else \
        (n_pass + n_single)
    steps_per_launch = iters / launches_per_job
    avg_upd_ms = upd / (args.steps * launches_per_job)
    bytes_per_job = BYTES_PER_UPDATE * my_cells * (n_single + n_pass)
    bytes_per_update = bytes_per_job / (my_cells * iters)
    bytes_per_launch = bytes_per_job / launches_per_job
    achieved = bytes_per_launch / (avg_upd_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    cw = 2 if grid.ext[1] <= 256 else 4
    kname = (f"slab_wave2_kernel<false,true,{cw}>" if k == 2 else
             f"slab_wave_kernel<false,true,{cw}>" if persistent else
             {None: f"slab_update_tma4_kernel<false,true,{cw},push>",
              2: f"slab_update_tma4_kernel<false,true,{cw},push>",
              1: "slab_update_tma_kernel", 0: "slab_update_kernel"}[args.variant])
    if grid.slab is False:
        kname = ("volume_wave2_kernel<true,true>" if k == 2 else
                 "volume_wave_kernel<true>" if persistent else "volume_update_tma_kernel<true>")
    traffic = (args.traffic if args.traffic is not None else
               _recorded_traffic(wl["name"] + ("_two_step" if k == 2 else ""), world))
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": traffic * steps_per_launch if traffic else None,
                "kernel": kname, "steps_per_launch": round(steps_per_launch, 3),
                "steps_per_pass": k, "passes_per_job": n_pass, "single_steps_per_job": n_single,
                "bytes_per_launch": round(bytes_per_launch),
                "avg_launch_ms": round(avg_upd_ms, 5), "peak_source": peak_src,
                "bytes_per_update": round(bytes_per_update, 4),
                "one_step_equivalent": {"bytes_per_update": BYTES_PER_UPDATE,
                                        "achieved": round(achieved * BYTES_PER_UPDATE
                                                          / bytes_per_update, 1),
                                        "frac": round(achieved * BYTES_PER_UPDATE
                                                      / bytes_per_update / peak, 4)},
                "update_share_of_step": round(upd / tot, 4) if tot else None,
                "halo_share_of_step": round(halo / tot, 4) if tot else None}

    # end to end through the public API with pinned host buffers: a stream
    # of e2e_steps jobs, each upload(pinned) -> run(iters) -> download(pinned)
    # + residual history, via JacobiSolver.run_jobs (next job's H2D and the
    # previous job's D2H on copy streams while the current job computes)
    e2e_ms = e2e_serial_ms = 0.0
    e2e_value = e2e_serial = None
    if args.e2e_steps > 0:
        K = args.e2e_steps
        # every job reads the same pinned input (the reference's initial
        # state) and writes one pinned output buffer (D2Hs are in order)
        host_in = [PinnedBuffer(nbytes)]
        host_in[0].array(dtype="float64")[:] = 0.0      # the reference's initial interior
        host_out = [PinnedBuffer(nbytes)]
        hook = (lambda s: s.allreduce_residual()) if world > 1 else None
        ins = [host_in[0]] * K
        outs = [host_out[0]] * K
        solver.run_jobs(ins[:1], outs[:1], iters, residual=True, nonneg=True, after_run=hook)
        barrier(world)
        st.synchronize()
        t0 = st.record()
        solver.run_jobs(ins, outs, iters, residual=True, nonneg=True, after_run=hook, start=t0)
        N.call("hrt_token_elapsed_ms", ctypes.c_uint64(t0.token_id),
               ctypes.c_uint64(solver.jobs_done_token.token_id), ctypes.byref(ms))
        e2e_ms = reduce_max(ms.value, world)
        e2e_value = cells * iters * K / (e2e_ms / 1e3) / 1e9
        # the same jobs one after another (no copy/compute overlap), for reference
        for k in range(min(K, 2)):
            barrier(world)
            st.synchronize()
            t0 = st.record()
            solver.upload(host=host_in[0], sync=False, nonneg=True)
            solver.run(iters, residual=True)
            solver.download(host=host_out[0])
            if world > 1:
                solver.global_residual_history()
            else:
                solver.residual_history()
            t1 = st.record()
            st.synchronize()
            N.call("hrt_token_elapsed_ms", ctypes.c_uint64(t0.token_id),
                   ctypes.c_uint64(t1.token_id), ctypes.byref(ms))
            if k == min(K, 2) - 1:
                e2e_serial_ms = reduce_max(ms.value, world)
        e2e_serial = cells * iters / (e2e_serial_ms / 1e3) / 1e9 if e2e_serial_ms else None
    h2d = nbytes * world
    d2h = nbytes * world + 8 * iters * world

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(region_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's initial state (interior 0.0, Dirichlet faces 1.0)",
        "config": config_for(wl, world, iters),
        "roofline": roofline,
        "e2e": {"value": round(e2e_value, 2) if e2e_value else None, "unit": UNIT,
                "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "what": "JacobiSolver.run_jobs: per step (job) H2D of the full field from pinned "
                        "host memory + iters iterations + D2H of the full field and the "
                        "residual history; copies of neighbouring jobs overlap compute on "
                        "separate copy streams",
                "serial_value": round(e2e_serial, 2) if e2e_serial else None,
                "serial_what": "one job with no overlap: upload + run + download + residual"},
        # per job: field_copy_kernel (reset) + halo_copy_kernel (ghost
        # priming) + the update launches
        "gpu_launches": (2 + launches_per_job) * args.steps,
        "halo_faces_per_gpu": solver.n_faces, "remote_messages_per_gpu": solver.n_remote,
        "tasks_per_s": round(len(grid.chunks) * iters * args.steps / (region_ms / 1e3), 1),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, args.cpu_budget)
    else:
        line["cpu_baseline"] = None
    solver.close()
    if world == 1 and not args.no_messages:
        line["messages"] = messages_record()
    if world == 1 and args.workload == "auto" and not args.no_scaling_baseline:
        # N>1 lines measure cfg3 (strong scaling); give the same workload at
        # N=1 so per-N efficiency can be read on one configuration
        line["scaling_baseline"] = scaling_baseline(args, local)
    if rank == 0:
        emit(line)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def scaling_baseline(args, gpu: int):
    """cfg3 (the N>1 workload) on this one GPU, device-timed, 2 jobs."""
    import ctypes

    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    wl = workload("cfg3", 1)
    s = JacobiSolver(ChunkGrid(wl["domain"], grid=wl["grid"]), gpus=[gpu])
    s.upload(nonneg=True)
    f = s._field()
    st = s.streams[gpu]

    def job():
        s._chunk_copies(True, 0, f)
        s.steps_done = 0
        return s.run_timed(wl["iters"], residual=True)

    job()
    t0 = st.record()
    n = 2
    for _ in range(n):
        job()
    t1 = st.record()
    st.synchronize()
    ms = ctypes.c_float()
    N.call("hrt_token_elapsed_ms", ctypes.c_uint64(t0.token_id), ctypes.c_uint64(t1.token_id),
           ctypes.byref(ms))
    s.close()
    X, Y, _ = wl["domain"]
    return {"workload": wl["desc"], "value": round(X * Y * wl["iters"] * n / (ms.value / 1e3) / 1e9, 2),
            "unit": UNIT, "note": "the N>1 bench lines run this workload; read scaling "
                                  "efficiency against this value, not against cfg2's"}


def run_reference(args):
    """Reference CPU path = the oracle port (the reference is pure Python and
    cannot be compiled), all host threads, bounded samples."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    O.use_all_host_threads()
    wl = workload(args.workload, world if args.gpus > 1 else 1)
    X, Y, _ = wl["domain"]
    slab = O.CpuSlab(X, Y)
    t0 = time.perf_counter()
    slab.sweep(1)
    t1 = time.perf_counter() - t0
    per_step = max(1, min(wl["iters"], int(args.ref_step_budget / max(t1, 1e-4))))
    for _ in range(args.warmup):
        slab.sweep(per_step)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        slab.sweep(per_step)
    dt = time.perf_counter() - t0
    slab.close()
    value = X * Y * per_step * args.steps / dt / 1e9
    cores = O.cpu_threads()
    sample = (f"{X}x{Y} slab, {per_step} of the {wl["iters"]} sweeps per step (field setup "
              f"excluded; GLUPS is a per-update rate, so the bounded sample measures the same "
              f"quantity), oracle/jacobi_oracle.c OpenMP port of jacobi.py:49-67")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's initial state (interior 0.0, Dirichlet faces 1.0)",
        "config": config_for(wl, world, args.iters or wl["iters"]),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "cfg1", "cfg2", "cfg3", "cfg5", "paper3d"])
    ap.add_argument("--iters", type=int, default=0, help="override iterations per job")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="jobs in the e2e stream (default: --steps)")
    ap.add_argument("--variant", type=int, default=None, help="slab kernel: 0 LDG, 1 TMA")
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--grid", default=None, help="chunk grid override, e.g. 16,1,1")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per update launch (from profiles/)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scaling-baseline", action="store_true")
    ap.add_argument("--no-messages", action="store_true",
                    help="skip the message-bandwidth record (N=1)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-step-budget", type=float, default=3.0)
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("need --steps >= 1")
    if args.e2e_steps is None:
        args.e2e_steps = args.steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def _recorded_traffic(workload: str, world: int):
    """DRAM read+write bytes per iteration of the dominant kernel from the
    committed ncu capture of the same workload on one GPU
    (profiles/traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            entry = json.load(fh).get(workload)
        if not entry or world != 1:
            return None
        return entry["bytes_per_launch"] / entry.get("steps_per_launch", 1)
    except Exception:
        return None


if __name__ == "__main__":
    main()
