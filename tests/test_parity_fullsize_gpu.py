"""Full-size parity against the C oracle at the shapes bench.py measures,
and the overflow edge of the unguarded division.

The reference's own initial state makes cfg2/cfg3 near-degenerate (three
distinct values after ~100 steps), so besides the exact
benched runs a random non-negative field at full cfg2 shape drives the
default two-step instance (slab_wave2_kernel<false, R, 4, 4>, 256-row
tiles) on non-degenerate data.  The oracle (oracle/jacobi_oracle.c, OpenMP
on the box's host cores) restates jacobi_reference (jacobi.py:49-67); the
bar is bitwise equality of the field and of every step's residual."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver_mod():
    from paper_2303_02543_b200 import _native as N
    from paper_2303_02543_b200 import jacobi as J

    N.require_gpu(0)
    return J


def _solve(J, dom, grid, steps, init=None, nonneg=None):
    s = J.JacobiSolver(J.ChunkGrid(dom, grid=grid))
    try:
        s.upload(init, nonneg=nonneg)
        s.run(steps, residual=True)
        return s.download(), s.residual_history(), s.checksum(), s.two_step, s.tiling(), s.nonneg
    finally:
        s.close()


def test_cfg2_as_benched_vs_oracle(solver_mod, oracle):
    """BASELINE configs[1] exactly as bench.py runs it (16384^2, 8x8 chunks,
    1000 iterations, default policy: two-step passes, 256-row tiles): field,
    checksum and residual history vs the C oracle (~40 s of host time)."""
    dom, steps = (16384, 16384, 1), 1000
    got, res, cs, two, tiling, _ = _solve(solver_mod, dom, (8, 8, 1), steps)
    assert two, "the benched configuration runs two-step passes"
    assert all(t[0] == 256 for t in tiling.values()), tiling
    ref, rref = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
    assert np.array_equal(res, rref), np.nonzero(res != rref)[0][:4]
    assert cs == oracle.checksum(ref)


@pytest.mark.parametrize("steps", [17, 6])
def test_cfg2_shape_random_nonneg_vs_oracle(solver_mod, oracle, steps):
    """A random non-negative field at full cfg2 shape: 17 steps = 1 single
    step + 4 two-step passes of the unguarded instance (the benched one);
    6 steps = 2 single steps + 2 passes.  Non-degenerate data: every cell
    differs, so sum order, division and rims are all exercised."""
    dom = (16384, 16384, 1)
    init = np.random.default_rng(20261019 + steps).random(dom) * 3.0
    got, res, _, two, tiling, nonneg = _solve(solver_mod, dom, (8, 8, 1), steps, init)
    assert two and nonneg, "unguarded two-step instance expected"
    assert all(t[0] == 256 for t in tiling.values()), tiling
    ref, rref = oracle.jacobi_c(dom, steps, residual=True, initial=init)
    assert np.array_equal(got, ref), np.argwhere(got != ref)[:4]
    assert np.array_equal(res, rref), np.nonzero(res != rref)[0][:4]


def test_cfg3_full_size_vs_oracle(solver_mod, oracle):
    """cfg3's domain on one GPU (32768^2, x-bands of 8 chunks, 60 steps)."""
    dom, steps = (32768, 32768, 1), 60
    got, res, cs, two, _, _ = _solve(solver_mod, dom, (8, 1, 1), steps)
    assert two
    ref, rref = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got, ref)
    assert np.array_equal(res, rref)
    del got
    assert cs == oracle.checksum(ref)


def test_paper3d_as_benched_vs_oracle(solver_mod, oracle):
    """The paper's Jacobi3D size as bench.py's paper3d runs it (1024x1024x768,
    x-bands of 8 chunks, 100 iterations: 50 two-step passes of
    volume_wave2_kernel, unguarded instance chosen on the device): field,
    checksum and residual history vs the C oracle."""
    dom, steps = (1024, 1024, 768), 100
    got, res, cs, two, _, _ = _solve(solver_mod, dom, (8, 1, 1), steps)
    assert two, "paper3d runs two-step passes"
    ref, rref = oracle.jacobi_c(dom, steps, residual=True)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(res, rref), np.nonzero(res != rref)[0][:4]
    del got
    assert cs == oracle.checksum(ref)


def test_paper3d_shape_random_signed_vs_oracle(solver_mod, oracle):
    """Random signed data at the paper3d shape: the guarded volume instance
    (the upload scan flags negatives), 9 steps = 1 single + 4 passes."""
    dom, steps = (1024, 1024, 768), 9
    init = np.random.default_rng(7).random(dom) * 4.0 - 2.0
    got, res, _, two, _, _ = _solve(solver_mod, dom, (8, 1, 1), steps, init)
    assert two
    ref, rref = oracle.jacobi_c(dom, steps, residual=True, initial=init)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    assert np.array_equal(res, rref)


@pytest.mark.parametrize("dom,grid", [((40, 70, 1), (4, 5, 1)), ((600, 1024, 1), (2, 2, 1)),
                                      ((10, 12, 14), (2, 3, 2))])
@pytest.mark.parametrize("steps", [1, 2, 5])
def test_overflowing_nonneg_field_matches_reference(solver_mod, oracle, dom, grid, steps,
                                                    monkeypatch):
    """A finite non-negative field with entries near DBL_MAX: the six-term
    sum overflows to inf, and IEEE (the reference) gives inf/6 = inf where
    Markstein's unguarded correction would give NaN.  The solver must see
    that the field exceeds the unguarded bound and keep the guarded
    instance; field and residual (inf, then NaN-ignoring max) match the
    oracle, through the default policy and forced two-step passes."""
    monkeypatch.setenv("HRT_FUSE2", "2")
    rng = np.random.default_rng(steps * 131 + dom[0])
    init = rng.random(dom)
    hot = rng.random(dom) < 0.05
    init[hot] = 1e308 * rng.random(int(hot.sum()))
    init[2:5, 3:6, :] = 1.5e308   # a hot block: neighbour sums overflow at step 1
    got, res, _, _, _, nonneg = _solve(solver_mod, dom, grid, steps, init)
    assert nonneg is False
    ref, rref = oracle.jacobi_c(dom, steps, residual=True, initial=init)
    assert np.isinf(ref).any(), "the case must actually overflow"
    assert np.array_equal(got, ref, equal_nan=True), np.argwhere(~((got == ref) | (
        np.isnan(got) & np.isnan(ref))))[:4]
    assert np.array_equal(res, rref, equal_nan=True), (res, rref)
    if dom[2] == 1:
        # the hazard the bound removes: forcing the unguarded instance on
        # this field gives NaN where the reference has inf
        bad = _solve(solver_mod, dom, grid, steps, init, nonneg=True)[0]
        assert np.isnan(bad).any() and not np.isnan(ref).any()


def test_overflow_through_run_jobs_default_check(solver_mod, oracle):
    """run_jobs(nonneg=None) checks its inputs on the host too."""
    from paper_2303_02543_b200.devices import PinnedBuffer

    J = solver_mod
    dom, steps = (64, 96, 1), 5
    init = np.random.default_rng(3).random(dom)
    init[10:20, 30:40] = 1.5e308
    b_in, b_out = PinnedBuffer(init.nbytes), PinnedBuffer(init.nbytes)
    b_in.array(np.float64, dom)[...] = init
    s = J.JacobiSolver(J.ChunkGrid(dom, grid=(2, 3, 1)))
    try:
        (hist,) = s.run_jobs([b_in], [b_out], steps, residual=True)
        assert s.nonneg is False
        got = b_out.array(np.float64, dom).copy()
    finally:
        s.close()
    ref, rref = oracle.jacobi_c(dom, steps, residual=True, initial=init)
    assert np.array_equal(got, ref, equal_nan=True)
    assert np.array_equal(hist, rref, equal_nan=True)
