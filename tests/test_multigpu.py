"""Multi-GPU paths (skipped on single-GPU boxes): one process driving several
B200s with chunk faces read over NVLink (peer access), and one process per
GPU under torchrun with faces exchanged by NCCL send/recv inside
libhrt_b200 — both bitwise against the oracle."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def ngpu():
    from paper_2303_02543_b200 import _native as N

    return N.gpu_count()


@pytest.fixture(scope="module", autouse=True)
def need_two():
    if ngpu() < 2:
        pytest.skip("needs >= 2 GPUs")


@pytest.mark.parametrize("persistent", [True, False])
@pytest.mark.parametrize("dom,grid,steps", [((1024, 1024, 1), (4, 4, 1), 50),
                                            ((300, 700, 1), (3, 7, 1), 64),
                                            ((2048, 512, 1), (16, 1, 1), 33),
                                            ((40, 36, 30), (2, 3, 2), 17)])
def test_single_process_peer_faces(oracle, dom, grid, steps, persistent):
    """Several GPUs in one process (the reference's in-process ranks): tile
    launches with per-step stream waits, or one wavefront launch per GPU
    with cross-GPU tile counters; runs split over launches."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    n = min(ngpu(), 4)
    s = JacobiSolver(ChunkGrid(dom, ranks=1, devices_per_rank=n, grid=grid),
                     gpus=list(range(n)), persistent=persistent)
    assert len(s.used_gpus) == n
    assert s.persistent == (persistent and dom[2] == 1)
    s.upload()
    s.run(steps // 2)
    s.run(steps - steps // 2)
    got = s.download()
    s.upload()
    s.run(steps)
    assert np.array_equal(got, s.download())
    res = s.residual_history()
    cs = s.checksum()
    s.close()
    ref, rres = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got, ref)
    assert np.array_equal(res, rres)
    assert cs == oracle.checksum(ref)


@pytest.mark.parametrize("persist", ["1", "0"])
def test_torchrun_nccl_faces(persist):
    """One process per GPU: the cross-process wavefront (default) or, with
    HRT_PERSIST=0, per-step tile launches with IPC step flags / NCCL; the
    full-size cfg3 comparison only in the default mode."""
    n = min(ngpu(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "2953" + persist,
           os.path.join(ROOT, "tests", "dist_check.py")]
    env = dict(os.environ, HRT_PERSIST=persist, DIST_CHECK_FULL=persist)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert "DIST_CHECK PASS" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


def test_two_process_pingpong_over_tcp():
    """Two processes, TCP byte transport with the reference's headers;
    direct mode moves payloads GPU->GPU through CUDA IPC device locators
    (no staging copies on the sender), staged mode through the socket."""
    env = dict(os.environ, MP_SIZES="8,448,449,65536,4194304", MP_ITERS="3")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29541",
           os.path.join(ROOT, "tools", "mp_pingpong.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert "MP_PINGPONG PASS direct_staging_copies=0" in out.stdout, \
        out.stdout[-3000:] + out.stderr[-3000:]
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith('{"mode"')]
    assert sorted({(r["mode"], r["size"]) for r in rows}) == sorted(
        (m, s) for m in ("direct", "staged") for s in (8, 448, 449, 65536, 4194304))


@pytest.mark.parametrize("fuse", ["1", "2"])
@pytest.mark.parametrize("dom,grid,ngpus", [((3 * 4096, 8192, 1), (3, 1, 1), 2),
                                            ((10240, 20480, 1), (8, 1, 1), 3),
                                            ((2048, 3 * 512, 1), (1, 3, 1), 2)])
def test_uneven_chunks_per_gpu(oracle, dom, grid, ngpus, fuse, monkeypatch):
    """Uneven chunk counts per GPU in one process (the reference's device
    assignment pos*dpr//len gives 2/1, 3/3/2, ...): every GPU must pick the
    same tile rows and the same one-step/two-step decision — from the
    largest per-GPU chunk count — since neighbours index each other's tile
    counters with their own tiling and a two-step GPU pushes no ghosts.
    4096x8192 chunks sit exactly at the 256-row and two-step thresholds
    for 2 vs 1 chunks per GPU."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    if ngpu() < ngpus:
        pytest.skip(f"needs {ngpus} GPUs")
    monkeypatch.setenv("HRT_FUSE2", fuse)
    steps = 19
    s = JacobiSolver(ChunkGrid(dom, ranks=1, devices_per_rank=ngpus, grid=grid),
                     gpus=list(range(ngpus)))
    counts = sorted({sum(1 for lin in s.owned if s.placement[lin] == g) for g in s.used_gpus})
    assert len(counts) > 1, "the placement must be uneven"
    til = s.tiling()
    assert len(set(til.values())) == 1, til
    s.upload()
    s.run(steps, residual=True)
    got, res = s.download(), s.residual_history()
    s.close()
    ref, rres = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
    assert np.array_equal(res, rres)


@pytest.mark.parametrize("signed", [True, False])
def test_single_process_volume_two_step(oracle, signed, monkeypatch):
    """x-band volumes on several GPUs of one process: volume_wave2_kernel
    reads the other GPU's x planes through tensor maps of its buffers (peer
    access) and waits on its tile counters; guarded (signed data) and
    unguarded instances, runs split over launches, a re-upload between
    jobs; bitwise vs the oracle."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")
    n = min(ngpu(), 4)
    dom, grid = (6 * 2 * n, 20, 130), (2 * n, 1, 1)
    s = JacobiSolver(ChunkGrid(dom, ranks=1, devices_per_rank=n, grid=grid), gpus=list(range(n)))
    assert len(s.used_gpus) == n and s.persistent and s.steps_per_pass == 2
    for job in range(2):
        rng = np.random.default_rng(31 + job)
        init = rng.random(dom) * 4.0 - (1.0 if signed else 0.0)
        s.upload(init)
        for k in (5, 1, 8):
            s.run(k, residual=False)
        got = s.download()
        ref = oracle.jacobi_reference(dom, 14, initial=init)
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (job, np.argwhere(got != ref)[:4])
    s.upload(init)
    s.run(13, residual=True)
    res = s.residual_history()
    s.close()
    rr = []
    oracle.jacobi_reference(dom, 13, initial=init, residuals=rr)
    assert np.array_equal(res, np.array(rr))


@pytest.mark.parametrize("dom,grid", [((300, 700, 1), (3, 7, 1)),     # staircase: corners on other GPUs
                                      ((64, 256, 1), (2, 8, 1))])      # y-bands: column faces
def test_single_process_slab_two_step_nbr9(oracle, dom, grid, monkeypatch):
    """Two-step slab passes on several GPUs of one process where faces AND
    corners of the 3 x 3 chunk neighbourhood live on other GPUs (peer
    pointers through hrt_jacobi_plan_set_wave2_nbr9): random signed data,
    runs split over launches, bitwise vs the oracle."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")
    n = min(ngpu(), 4)
    s = JacobiSolver(ChunkGrid(dom, ranks=1, devices_per_rank=n, grid=grid), gpus=list(range(n)))
    assert s.persistent and s.steps_per_pass == 2
    init = np.random.default_rng(5).random(dom) * 4.0 - 1.0
    s.upload(init)
    for k in (5, 8):
        s.run(k, residual=False)
    got = s.download()
    s.close()
    ref = oracle.jacobi_reference(dom, 13, initial=init)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
