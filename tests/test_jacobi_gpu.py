"""GPU parity of the native Jacobi engine (libhrt_b200.so on a B200)
against the reference's golden vectors and the C oracle.

Bar: bit-exact float64 (the north star's --fmad=false mode) for the field,
the checksum and the residual history."""

import ctypes
import hashlib

import os

import numpy as np
import pytest

from conftest import kwargs_of

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def hrt():
    import paper_2303_02543_b200 as P
    from paper_2303_02543_b200 import _native as N

    N.require_gpu(0)
    return P


def test_div6_markstein_equals_ieee(hrt):
    """The update kernel's division (Markstein correction) is bitwise IEEE
    x/6.0: 2^28 uniform [0,6), 2^26 near 1/2/3/6, 2^26 random finite."""
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200.devices import Stream

    st = Stream(0)
    for mode, n in ((0, 1 << 28), (1, 1 << 26), (2, 1 << 26)):
        mism, bad = ctypes.c_uint64(), ctypes.c_double()
        N.call("hrt_div6_sweep", st.h, 12345 + mode, n, mode, ctypes.byref(mism), ctypes.byref(bad))
        assert mism.value == 0, (mode, bad.value)


LADDER_NATIVE = [
    "cube8_s3", "ac10_g111", "ac10_g222", "ac10_od2", "ac10_od4", "ac10_r2d2", "slab64_s10",
    "slab1024_s5", "cfg1", "halo32_s20", "halo32_s20_r2d2", "halo32_s20_direct",
    "halo16_cube_s12", "cube24_s30", "slab48x40_s64", "slab96x80_s13", "slab256_s300",
    "unit_chunks_slab", "unit_chunks_cube", "zero_steps", "rect_slab", "thin_x", "zslab_3d",
]


@pytest.mark.parametrize("fuse2", ["1", "2"])  # auto policy, and two-step passes forced
@pytest.mark.parametrize("name", LADDER_NATIVE)
def test_ladder_bitwise(hrt, ladder, small_arrays, name, fuse2, monkeypatch):
    monkeypatch.setenv("HRT_FUSE2", fuse2)
    e = ladder[name]
    rep, cs, arr = hrt.run_jacobi3d(tuple(e["domain"]), steps=e["steps"], **kwargs_of(e))
    if name in small_arrays:
        ref = small_arrays[name]
        bad = np.argwhere(arr != ref)
        assert bad.size == 0, f"{len(bad)} cells differ, first {bad[:3].tolist()}"
    assert sha(arr) == e["sha256"]
    assert repr(cs) == e["checksum"]
    assert len(rep.rows) == e["steps"]


def test_cfg2_prefix_bitwise(hrt, ladder):
    """16384^2 slab, 8x8 chunks (cfg2 decomposition), 1 and 3 steps."""
    for s in (1, 3):
        e = ladder[f"cfg2_prefix_s{s}"]
        _, cs, arr = hrt.run_jacobi3d((16384, 16384, 1), steps=s, grid=(8, 8, 1))
        assert sha(arr) == e["sha256"]
        assert repr(cs) == e["checksum"]


def test_residual_history_bitwise(hrt, oracle):
    for dom, grid, steps in [((40, 24, 1), (5, 3, 1), 33), ((12, 10, 6), (2, 1, 3), 15),
                             ((512, 384, 1), (4, 3, 1), 150)]:
        rep, _, arr = hrt.run_jacobi3d(dom, steps=steps, grid=grid)
        ref, res = oracle.jacobi_c(dom, steps, residual=True)
        assert np.array_equal(arr, ref)
        got = np.array([r["residual"] for r in rep.rows])
        assert np.array_equal(got, res), np.argwhere(got != res)[:5]


def test_mid_size_vs_oracle(hrt, oracle):
    """4096^2 for 257 steps, 4x8 chunks: field and checksum vs the C oracle."""
    dom, steps = (4096, 4096, 1), 257
    _, cs, arr = hrt.run_jacobi3d(dom, steps=steps, grid=(4, 8, 1))
    ref = oracle.jacobi_c(dom, steps)
    assert np.array_equal(arr, ref)
    assert cs == oracle.checksum(ref)


def test_check_mode_and_check_failure_detection(hrt):
    rep, cs, arr = hrt.run_jacobi3d((8, 8, 8), steps=3, check=True)
    assert arr.shape == (8, 8, 8)
    assert 0.0 < arr.mean() < 1.0
    assert rep.columns[:2] == ["step", "virtual_makespan_s"]


def test_full_size_properties(hrt):
    """cfg2 at full size (16384^2, 1000 steps): size-independent properties —
    decomposition invariance (8x8 vs 2x32 chunks, bitwise), exact mirror
    symmetry in x ((xm+xp) is commutative), Dirichlet bound 0 < u <= 1."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    out = []
    for grid in ((8, 8, 1), (2, 32, 1)):
        s = JacobiSolver(ChunkGrid((16384, 16384, 1), grid=grid))
        s.upload()
        s.run(1000, residual=True)
        out.append((s.download(), s.checksum(), s.residual_history()))
        s.close()
    (a, ca, ra), (b, cb, rb) = out
    assert np.array_equal(a, b) and ca == cb and np.array_equal(ra, rb)
    assert np.array_equal(a, a[::-1])
    assert a.min() > 0.0 and a.max() <= 1.0
    assert np.all(ra[1:] <= ra[:-1] * 1.0000001 + 1e-300) or ra[-1] < ra[0]


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_kernel_variants_bitwise(hrt, oracle, variant):
    """Every slab kernel variant (LDG march, TMA ring, TMA ring x4) on a
    ragged decomposition whose chunk width is not a multiple of the tile."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    dom, steps = (300, 1030, 1), 41
    s = JacobiSolver(ChunkGrid(dom, grid=(3, 2, 1)), variant=variant, rows=37)
    s.upload()
    s.run(steps)
    got, res = s.download(), s.residual_history()
    s.close()
    ref, rref = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got, ref)
    assert np.array_equal(res, rref)


@pytest.mark.parametrize("dom,grid", [((40, 70, 1), (4, 5, 1)), ((10, 12, 14), (2, 3, 2))])
def test_arbitrary_initial_data_guarded_division(hrt, oracle, dom, grid):
    """Signed, tiny (subnormal-quotient) and large initial data: the solver
    detects the field is not non-negative and keeps the division guard."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    rng = np.random.default_rng(7)
    init = rng.standard_normal(dom) * rng.choice([1e-310, 1e-300, 1.0, 1e300], size=dom)
    for steps in (1, 6):
        s = JacobiSolver(ChunkGrid(dom, grid=grid))
        s.upload(init)
        assert s.nonneg is False
        s.run(steps, residual=False)
        got = s.download()
        s.close()
        ref = oracle.jacobi_reference(dom, steps, initial=init)
        assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("dom,grid,steps", [((40, 36, 70), (2, 3, 2), 17),
                                            ((20, 17, 300), (1, 1, 2), 11),
                                            ((130, 21, 150), (1, 1, 1), 9),
                                            ((9, 200, 5), (3, 4, 1), 12)])
def test_volume_kernels_bitwise(hrt, oracle, variant, dom, grid, steps):
    """3D chunks with partial y (8-row) and z (64-column) tiles: the TMA ring
    volume kernel (default) and the plain one, field + residual vs oracle."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    s = JacobiSolver(ChunkGrid(dom, grid=grid), variant=variant)
    s.upload()
    s.run(steps)
    got, res = s.download(), s.residual_history()
    s.close()
    ref, rref = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got, ref)
    assert np.array_equal(res, rref)


def test_tma_ring_race_regression(hrt):
    """16384^2, 8x8 chunks, 10 steps, repeated: without the async-proxy fence
    between the consumers' shared-memory reads and the producer's next TMA
    write into the same ring stage, 4 of 5 runs corrupted a cell (found on
    B200 via the residual history).  Field and residual must be identical to
    the LDG kernel on one chunk every time."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    dom = (16384, 16384, 1)

    def run(grid, variant):
        s = JacobiSolver(ChunkGrid(dom, grid=grid), variant=variant)
        s.upload()
        s.run(10, residual=True, graph=False)
        out = s.download(), s.residual_history()
        s.close()
        return out

    ref_f, ref_r = run((1, 1, 1), 0)
    for variant in (2, 1):
        for _ in range(4 if variant == 2 else 2):
            f, r = run((8, 8, 1), variant)
            assert np.array_equal(r, ref_r), (variant, np.nonzero(r != ref_r)[0][:5])
            assert np.array_equal(f, ref_f), variant


@pytest.mark.parametrize("dom,grid,steps", [((64, 64, 1), (4, 4, 1), 10),
                                            ((1000, 1300, 1), (1, 1, 1), 13),
                                            ((2048, 1536, 1), (2, 3, 1), 37),
                                            ((512, 2560, 1), (2, 5, 1), 21),
                                            ((3, 700, 1), (1, 2, 1), 9),
                                            ((1024, 1024, 1), (32, 32, 1), 25),
                                            ((40, 36, 70), (2, 3, 2), 17),
                                            ((130, 21, 150), (1, 1, 1), 9),
                                            ((9, 200, 5), (3, 4, 1), 12),
                                            ((64, 64, 132), (2, 2, 3), 10)])
def test_persistent_dataflow_kernel_bitwise(hrt, oracle, dom, grid, steps):
    """The persistent dataflow launch (balanced row segments per resident CTA,
    neighbour step counters instead of per-step launches) against the C
    oracle and the per-step tile kernel: field + residual bitwise, including
    runs split over several launches (step counters carry over) and narrow
    (<= 256 wide) chunks."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    ref, rref = oracle.jacobi_c(dom, steps, residual=True)
    outs = []
    vp = len(dom) == 3 and dom[2] > 1  # volumes: the opt-in fused push + wavefront
    for persistent, parts in ((True, [steps]), (True, [steps // 3, steps - steps // 3]),
                              (False, [steps])):
        s = JacobiSolver(ChunkGrid(dom, grid=grid), persistent=persistent, vpush=vp)
        assert s.persistent == persistent
        s.upload()
        for n in parts:
            s.run(n, residual=False)
        got = s.download()
        s.close()
        s = JacobiSolver(ChunkGrid(dom, grid=grid), persistent=persistent, vpush=vp)
        s.upload()
        s.run(steps, residual=True)
        res = s.residual_history()
        s.sync()
        s.close()
        outs.append((got, res))
    for got, res in outs:
        assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
        assert np.array_equal(res, rref)


def test_persistent_guarded_division(hrt, oracle):
    """Signed/tiny/huge initial data through the persistent kernel's guarded
    instance."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    dom = (96, 600, 1)
    rng = np.random.default_rng(11)
    init = rng.standard_normal(dom) * rng.choice([1e-310, 1e-300, 1.0, 1e300], size=dom)
    s = JacobiSolver(ChunkGrid(dom, grid=(2, 2, 1)), persistent=True)
    s.upload(init)
    assert s.nonneg is False and s.persistent
    s.run(5, residual=False)
    got = s.download()
    s.close()
    ref = oracle.jacobi_reference(dom, 5, initial=init)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]


@pytest.mark.parametrize("dom,grid,steps,njobs,sign", [
    ((64, 96, 1), (2, 3, 1), 7, 4, 1.0),        # side arrays (even widths)
    ((66, 99, 1), (2, 3, 1), 9, 3, 1.0),        # odd widths: in-buffer ghost columns
    ((66, 99, 1), (2, 3, 1), 5, 1, -1.0),       # one job, guarded /6
    ((512, 512, 1), (2, 2, 1), 70, 2, 1.0),     # 256-wide chunks, several row tiles
    ((1024, 2048, 1), (4, 4, 1), 40, 3, 1.0),   # 512-wide chunks, multiple column tiles
])
def test_run_jobs_pipeline_matches_serial(hrt, oracle, dom, grid, steps, njobs, sign,
                                          monkeypatch):
    """run_jobs (H2D/D2H of neighbouring jobs overlapped with compute on copy
    streams, double-buffered staging) gives, per job, exactly the field and
    residual history of a serial upload/run/download, on random data (side
    arrays and in-buffer ghost columns, narrow and wide chunks, guarded
    division, one job and several)."""
    from paper_2303_02543_b200.devices import PinnedBuffer
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")  # two-step passes even on these small domains
    rng = np.random.default_rng(5)
    inits = [sign * rng.random(dom) * (1 + k) for k in range(njobs)]
    nbytes = dom[0] * dom[1] * 8
    ins, outs = [], []
    for a in inits:
        b = PinnedBuffer(nbytes)
        b.array(np.float64, dom)[...] = a
        ins.append(b)
        outs.append(PinnedBuffer(nbytes))
    s = JacobiSolver(ChunkGrid(dom, grid=grid))
    hists = s.run_jobs(ins, outs, steps, residual=True, nonneg=sign > 0)
    for k, a in enumerate(inits):
        ref = oracle.jacobi_reference(dom, steps, initial=a)
        got = outs[k].array(np.float64, dom)
        assert np.array_equal(got, ref), k
        s2 = JacobiSolver(ChunkGrid(dom, grid=grid))
        s2.upload(a)
        s2.run(steps, residual=True)
        assert np.array_equal(hists[k], s2.residual_history()), k
        s2.close()
    s.close()


def test_full_size_cfg3_and_cfg5_properties(hrt):
    """BASELINE's largest single-GPU shapes, through size-independent
    properties (the oracle would take hours): cfg3 32768^2 — x-band (8x1) vs
    y-band (1x8) decompositions bitwise equal in field, checksum and
    residual history, exact x-mirror symmetry ((xm+xp) commutes; y-mirror
    and transpose are not exact under the reference's sum order); cfg5
    65536^2 in 65,536 chunks of 256^2 — equal to the same domain in 64
    chunks of 8192^2.
    Residuals are non-increasing after the first sweep (monotone Jacobi on
    this problem) and the field stays in (0, 1]."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    def solve(dom, grid, steps):
        s = JacobiSolver(ChunkGrid(dom, grid=grid))
        s.upload()
        s.run(steps, residual=True)
        out = s.download(), s.checksum(), s.residual_history()
        s.close()
        return out

    a, ca, ra = solve((32768, 32768, 1), (8, 1, 1), 60)
    b, cb, rb = solve((32768, 32768, 1), (1, 8, 1), 60)
    assert np.array_equal(a, b) and ca == cb and np.array_equal(ra, rb)
    assert np.array_equal(a, a[::-1])
    assert a.min() >= 0.0 and a.max() <= 1.0
    assert np.all(ra[1:] <= ra[:-1])
    del a, b
    c, cc, rc = solve((65536, 65536, 1), (256, 256, 1), 12)
    d, cd, rd = solve((65536, 65536, 1), (8, 8, 1), 12)
    assert np.array_equal(c, d) and cc == cd and np.array_equal(rc, rd)
    assert np.array_equal(c, c[::-1])


@pytest.mark.parametrize("dom,grid", [
    ((130, 1030, 1), (2, 2, 1)),     # odd chunk width: one step per pass (fallback)
    ((132, 1032, 1), (2, 2, 1)),     # 66-row chunks (rows=64: tiles 64 + 2), 516-wide (512 + 4)
    ((600, 1024, 1), (2, 2, 1)),     # 300-row chunks: 256 + 44 (default rows) / 4 x 64 + 44
    ((96, 512, 1), (3, 2, 1)),       # 256-wide chunks: the 2-warp instance
    ((8, 12, 1), (4, 3, 1)),         # 2 x 4 chunks: rims span whole neighbour chunks
    ((12, 16, 1), (4, 4, 1)),        # 3 x 4 chunks: 3-cell rims span whole neighbours
    ((134, 1032, 1), (2, 2, 1)),     # 67-row chunks: tiles 64 + 3 (the 3-row minimum)
    ((200, 64, 1), (1, 1, 1)),       # one chunk: every rim is the domain boundary
])
@pytest.mark.parametrize("steps", [3, 4, 6, 7, 13])
@pytest.mark.parametrize("rows", [None, 64])
def test_two_step_passes_bitwise(hrt, oracle, dom, grid, steps, rows, monkeypatch):
    """slab_wave2_kernel (two Jacobi steps per pass, 2-cell rims read from the
    3 x 3 chunk neighbourhood, u(t+1) only in registers) against the numpy
    oracle on random signed data: field and every step's residual bitwise,
    with n mod 4 single steps before the passes."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")  # these domains are too small for the auto policy
    rng = np.random.default_rng(steps * 7 + dom[0])
    init = rng.random(dom) * 4.0 - 1.0
    s = JacobiSolver(ChunkGrid(dom, grid=grid), rows=rows)
    ex, ey = dom[0] // grid[0], dom[1] // grid[1]
    if ex % (rows or 64) != 1 and ey % 2 == 0:   # (below the 256-row threshold: 64-row tiles)
        assert s.two_step and s.steps_per_pass == 2, "two-step passes should apply here"
    s.upload(init)
    s.run(steps, residual=True)
    got = s.download()
    res = s.residual_history()
    s.close()
    resid = []
    ref = oracle.jacobi_reference(dom, steps, initial=init, residuals=resid)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
    assert np.array_equal(res, np.array(resid)), (res, resid)


@pytest.mark.parametrize("dom,grid", [
    ((16, 9, 37), (2, 1, 1)),        # partial y (4-row) and z (120-column) tiles
    ((4, 5, 121), (2, 1, 1)),        # 2-plane chunks (the minimum): rims span the neighbour
    ((30, 17, 240), (3, 1, 1)),      # two full z tiles
    ((12, 8, 250), (1, 1, 1)),       # one chunk: both x faces are domain faces
    ((21, 4, 119), (3, 1, 1)),       # 7-plane chunks, odd z extent
    ((40, 33, 130), (4, 1, 1)),
])
@pytest.mark.parametrize("steps", [3, 4, 6, 9, 13])
def test_volume_two_step_passes_bitwise(hrt, oracle, dom, grid, steps, monkeypatch):
    """volume_wave2_kernel (x-band volumes, two Jacobi steps per pass, rims
    from the x-neighbour chunks in place, u(t+1) in registers and lane
    shuffles) against the numpy oracle on random signed data: field and
    every step's residual bitwise, n mod 4 single steps first."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")  # small domains: force the passes
    rng = np.random.default_rng(steps * 13 + dom[2])
    init = rng.random(dom) * 4.0 - 1.0
    s = JacobiSolver(ChunkGrid(dom, grid=grid))
    assert s.persistent and s.steps_per_pass == 2
    s.upload(init)
    s.run(steps, residual=True)
    got = s.download()
    res = s.residual_history()
    s.close()
    resid = []
    ref = oracle.jacobi_reference(dom, steps, initial=init, residuals=resid)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
    assert np.array_equal(res, np.array(resid)), (res, resid)


@pytest.mark.parametrize("parts", [[4, 4], [5, 8], [4, 1, 4], [13]])
def test_volume_two_step_split_runs(hrt, oracle, parts, monkeypatch):
    """Runs alternating two-step passes and single steps over one upload
    (the reference's initial state): the ghost planes the passes leave stale
    are re-primed before the next single step."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")
    dom, grid = (24, 20, 150), (3, 1, 1)
    s = JacobiSolver(ChunkGrid(dom, grid=grid))
    s.upload()
    for n in parts:
        s.run(n, residual=False)
    got = s.download()
    s.close()
    ref = oracle.jacobi_c(dom, sum(parts))
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]


@pytest.mark.parametrize("steps", [4, 13])
def test_volume_two_step_division_paths(hrt, oracle, steps, monkeypatch):
    """The volume pass picks its division on the device from the upload's
    field scan: a non-negative field whose smallest positive value is
    1e-300 allows the unguarded instance for 4 steps (1e-300 * 6^-4 >>
    2^-1019) but not for 13; both runs must match the oracle bitwise."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    monkeypatch.setenv("HRT_FUSE2", "2")
    dom, grid = (24, 9, 130), (3, 1, 1)
    rng = np.random.default_rng(5)
    init = rng.random(dom)
    init[rng.random(dom) < 0.05] = 1e-300
    init[rng.random(dom) < 0.3] = 0.0
    s = JacobiSolver(ChunkGrid(dom, grid=grid))
    s.upload(init)
    s.run(steps, residual=True)
    got, res = s.download(), s.residual_history()
    s.close()
    resid = []
    ref = oracle.jacobi_reference(dom, steps, initial=init, residuals=resid)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(res, np.array(resid))


def test_volume_negative_zero_kept(hrt, oracle, monkeypatch):
    """-0.0 / 6 is -0.0 (numpy, the reference): a field of -0.0 keeps its
    sign bits wherever all six neighbours are -0.0 — bitwise, through the
    two-step passes, the one-step tiles and the persistent wavefront."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    dom, grid = (24, 12, 40), (3, 1, 1)
    init = np.full(dom, -0.0)
    ref = oracle.jacobi_reference(dom, 5, initial=init)
    assert np.signbit(ref).any()
    for fuse2, persistent in (("2", None), ("0", False), ("0", True)):
        monkeypatch.setenv("HRT_FUSE2", fuse2)
        s = JacobiSolver(ChunkGrid(dom, grid=grid), persistent=persistent, vpush=persistent)
        s.upload(init)
        s.run(5, residual=False)
        got = s.download()
        s.close()
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (fuse2, persistent)


@pytest.mark.parametrize("dom,grid,rows_want", [((1024, 1024, 1), (4, 4, 1), 16),    # cfg1
                                                ((2048, 2048, 1), (8, 8, 1), 16),
                                                ((4096, 4096, 1), (8, 8, 1), 64),
                                                ((8192, 8192, 1), (8, 8, 1), 256)])
def test_tile_height_for_parallelism(hrt, oracle, dom, grid, rows_want):
    """The tallest tile height (256/64/32/16 rows) leaving one two-step tile
    per resident CTA, else 16, and two-step passes throughout; the small
    shapes bitwise vs the oracle on random data (16-row tiles: rims of 2
    rows from the tiles above and below are 25 % of the reads)."""
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    s = JacobiSolver(ChunkGrid(dom, grid=grid))
    rows = {t[0] for t in s.tiling().values()}
    assert rows == {rows_want} and s.steps_per_pass == 2, (rows, s.tiling())
    if dom[0] <= 2048:
        init = np.random.default_rng(dom[0]).random(dom) * 3.0 - 1.0
        s.upload(init)
        s.run(14, residual=True)
        got, res = s.download(), s.residual_history()
        ref, rref = oracle.jacobi_c(dom, 14, residual=True, initial=init)
        assert np.array_equal(got, ref)
        assert np.array_equal(res, rref)
    s.close()
