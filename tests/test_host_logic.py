"""Host-side logic on CPU (no device calls): chunk decomposition vs the
reference's rules, HBM layout and face-plane address math, the dependency
tracker's edges, ping-pong size parsing, report writers and error mapping."""

import json

import numpy as np
import pytest

from paper_2303_02543_b200 import errors as E
from paper_2303_02543_b200.jacobi import (FACES, ChunkGrid, _contiguous, chunk_layout, face_plane,
                                          opposite, remote_faces, remote_ops)
from paper_2303_02543_b200.objects import AccessMode, HeteroObject
from paper_2303_02543_b200.pingpong import parse_sizes
from paper_2303_02543_b200.reporting import BenchReport
from paper_2303_02543_b200.runtime import DependencyTracker, _DepNode


def test_opposite_faces():
    assert [opposite(f) for f in range(6)] == [1, 0, 3, 2, 5, 4]  # jacobi.py:44-46
    assert FACES[3] == (1, 1)


def test_chunk_grid_matches_oracle_decomposition(oracle):
    for dom, kw in [((8, 8, 8), dict(ranks=2, devices_per_rank=2, od=2)),
                    ((48, 40, 1), dict(grid=(6, 5, 1), devices_per_rank=8)),
                    ((64, 64, 64), dict(grid=(2, 2, 2), ranks=3))]:
        g = ChunkGrid(dom, **kw)
        ref = oracle.chunk_layout(dom, **kw)
        for ch, r in zip(g.chunks, ref):
            assert ch.lin == r["lin"] and ch.coord == r["coord"] and ch.offsets == r["offsets"]
            assert ch.rank == r["rank"] and ch.device_local == r["device_local"]
            assert ch.neighbors == r["neighbors"]


def test_chunk_grid_errors():
    with pytest.raises(E.HrtError, match="not divisible"):
        ChunkGrid((10, 10, 1), grid=(3, 1, 1))
    with pytest.raises(E.HrtError):
        ChunkGrid((0, 10, 1))


def _element(L, base, i, j, k):
    kk = k * L.stride[2] if L.ndim == 3 else 0
    return (base // 8) + L.origin + i * L.stride[0] + j * L.stride[1] + kk


@pytest.mark.parametrize("ext,slab", [((7, 33, 1), True), ((2048, 2048, 1), True),
                                      ((5, 6, 7), False), ((3, 4, 130), False)])
def test_layout_alignment_and_planes(ext, slab):
    L = chunk_layout(ext, slab)
    ex, ey, ez = ext
    # interior (1,1[,1]) 16-byte aligned, every row stride even (16-byte rows)
    assert (L.origin + L.stride[0] + L.stride[1] + (L.stride[2] if not slab else 0)) % 2 == 0
    assert L.stride[0] % 2 == 0 and (slab or L.stride[1] % 2 == 0)
    # TMA spans reach element ey+2 (slab) / ez+2 (volume) inside the row
    fast = ey if slab else ez
    row = L.stride[0] if slab else L.stride[1]
    assert L.origin + fast + 2 < row
    base = 4096
    for f in range(4 if slab else 6):
        axis, side = FACES[f]
        for ghost in (True, False):
            addr, n0, n1, s0, s1 = face_plane(L, base, f, ghost)
            idx = (0 if side == 0 else ext[axis] + 1) if ghost else (1 if side == 0 else ext[axis])
            start = [1, 1, 1]
            start[axis] = idx
            if slab:
                start[2] = 0
            assert addr // 8 == _element(L, base, *start)
            others = [a for a in range(2 if slab else 3) if a != axis]
            assert n1 == ext[others[-1]]
            assert s1 == L.stride[others[-1]]
            if not slab:
                assert n0 == ext[others[0]] and s0 == L.stride[others[0]]
    # the ghost row of a slab (x face) is contiguous, the ghost column is not
    if slab:
        assert _contiguous(*face_plane(L, base, 0, True)[1:])
        assert not _contiguous(*face_plane(L, base, 2, True)[1:]) or ex == 1


def test_remote_faces_x_bands_are_rows():
    g = ChunkGrid((32768, 32768, 1), ranks=4, grid=(32, 1, 1))
    for r in range(4):
        ops = remote_ops(g, r)
        assert all(FACES[f][0] == 0 for _, _, _, f, _ in ops)  # rows only
        assert all(n == 32768 for *_, n in ops)
    assert remote_faces(g, 0) == [(7, 1, 8), (8, 0, 7)]


def test_dependency_tracker_edges():
    """RAW, WAR, WAW per object (runtime.py:167-190)."""
    t = DependencyTracker()
    obj = HeteroObject(1, (4,), dtype=np.float64)
    w1, r1, r2, w2, r3 = (_DepNode(i, True) for i in range(5))
    assert t.register(w1, obj, AccessMode.WRITE) == set()
    assert t.register(r1, obj, AccessMode.READ) == {w1}          # RAW
    assert t.register(r2, obj, AccessMode.READ) == {w1}
    assert t.register(w2, obj, AccessMode.WRITE) == {w1, r1, r2}  # WAW + WAR
    r1.done = True
    assert t.register(r3, obj, AccessMode.READ) == {w2}
    w2.done = True
    other = HeteroObject(2, (4,), dtype=np.float64)
    assert t.register(_DepNode(9, True), other, AccessMode.READ_WRITE) == set()


def test_hetero_object_sizes_and_errors():
    o = HeteroObject(3, (10, 4, 2), dtype=np.float64)
    assert o.total_size == 640 and o.element_size == 8
    with pytest.raises(E.HrtError):
        HeteroObject(4, (0,), dtype=np.uint8)
    with pytest.raises(E.HrtError):
        HeteroObject(5, (1, 2, 3, 4), dtype=np.uint8)
    with pytest.raises(E.HrtError):
        HeteroObject(6, (3,))


def test_parse_sizes():
    assert parse_sizes("8..64") == [8, 16, 32, 64]          # pingpong.py:35-45
    assert parse_sizes("8,100,4096") == [8, 100, 4096]


def test_bench_report_writers(tmp_path):
    rep = BenchReport("pingpong", columns=["size_bytes", "iters"])
    rep.add(size_bytes=8, iters=3, extra="ignored")
    p = tmp_path / "r.csv"
    rep.write(str(p))
    assert p.read_text().splitlines() == ["size_bytes,iters", "8,3"]
    q = tmp_path / "r.json"
    rep.write(str(q))
    assert json.loads(q.read_text())["rows"][0]["size_bytes"] == 8
    assert rep.csv_text() == "size_bytes,iters\n8,3\n"


def test_error_codes_map_to_reference_exceptions():
    for rc, cls in [(-2, E.OutOfDeviceMemory), (-3, E.DoubleFree), (-4, E.InvalidLocation),
                    (-5, E.UnknownToken), (-6, E.KernelError), (-1, E.HrtError)]:
        with pytest.raises(cls):
            E.raise_for(rc, "x")
    assert issubclass(E.OutOfDeviceMemory, E.HrtError)


def test_nonneg_bound_selects_guarded_division():
    """The unguarded division (Markstein without range checks) is exact only
    while every six-term sum stays <= 2^1000: fields above 2^997, negative
    or non-finite keep the guarded instance (reference: inf/6 = inf)."""
    import numpy as np

    from paper_2303_02543_b200.jacobi import NONNEG_MAX, _nonneg

    assert _nonneg(np.zeros((4, 4, 1)))
    assert _nonneg(np.full((3, 3, 1), NONNEG_MAX))
    assert not _nonneg(np.full((3, 3, 1), np.nextafter(NONNEG_MAX, np.inf)))
    assert not _nonneg(np.array([[[1e308]]]))
    assert not _nonneg(np.array([[[-0.5]]]))
    assert not _nonneg(np.array([[[np.inf]]]))
    assert not _nonneg(np.array([[[np.nan]]]))
    assert 6 * NONNEG_MAX + 2 <= 2.0 ** 1000


@pytest.mark.parametrize("grid", [(3, 5, 1), (4, 4, 1), (1, 7, 1), (6, 1, 1)])
def test_nbhd9_is_the_3x3_block(grid):
    """ChunkGrid.nbhd9 (the table behind hrt_jacobi_plan_set_wave2_nbr9):
    row-major NW N NE W C E SW S SE by chunk coordinates, None off the
    domain, and a corner present exactly when both faces next to it are
    (the C side rejects anything else)."""
    from paper_2303_02543_b200.jacobi import ChunkGrid

    cx, cy, _ = grid
    cg = ChunkGrid((cx * 8, cy * 8, 1), grid=grid)
    for lin in range(cg.nchunks):
        ix, iy = lin % cx, lin // cx
        want = []
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                x, y = ix + dx, iy + dy
                want.append(x + cx * y if 0 <= x < cx and 0 <= y < cy else None)
        got = cg.nbhd9(lin)
        assert got == want, (lin, got, want)
        for corner, a, b in ((0, 1, 3), (2, 1, 5), (6, 7, 3), (8, 7, 5)):
            assert (got[corner] is not None) == (got[a] is not None and got[b] is not None)


def test_run_segments_split_mixed_volume_runs_across_devices():
    """Volume one-step and two-step launches keep separate counters: with
    neighbours on other devices a run becomes the n mod 4 single steps, then
    the passes (a fence between them); slabs, single devices and runs that
    are all passes or all single steps stay whole."""
    from types import SimpleNamespace

    from paper_2303_02543_b200.jacobi import JacobiSolver

    def solver(ndim, ngpu, world=1, persistent=True, k=2):
        s = SimpleNamespace(used_gpus=list(range(ngpu)), world=world, persistent=persistent,
                            layout=SimpleNamespace(ndim=ndim), steps_per_pass=k)
        return s

    seg = JacobiSolver._run_segments
    assert seg(solver(3, 2), 10, 13) == [(10, 1), (11, 12)]
    assert seg(solver(3, 1, world=4), 0, 6) == [(0, 2), (2, 4)]
    assert seg(solver(3, 2), 0, 8) == [(0, 8)]        # passes only
    assert seg(solver(3, 2), 0, 3) == [(0, 3)]        # single steps only
    assert seg(solver(3, 1), 0, 13) == [(0, 13)]      # one device: stream order suffices
    assert seg(solver(2, 2), 0, 13) == [(0, 13)]      # slabs share one counter array
    assert seg(solver(3, 2, k=1), 0, 13) == [(0, 13)]  # no two-step passes


def test_device_view_cached_per_allocation():
    """A copy's task-argument view is built once per allocation and rebuilt
    when the copy moves to another allocation."""
    from paper_2303_02543_b200.devices import DeviceAllocation, DeviceRegistry
    from paper_2303_02543_b200.objects import DeviceCopy
    from paper_2303_02543_b200.runtime import Runtime

    rt = Runtime(DeviceRegistry())
    obj = HeteroObject(1, (16,), dtype=np.float64)
    obj.copies[0] = DeviceCopy(DeviceAllocation(0, 0, 128, ptr=4096))
    v = rt.device_view(obj, 0)
    assert rt.device_view(obj, 0) is v
    assert (v.ptr, v.shape, v.dtype) == (4096, (16,), np.dtype(np.float64))
    obj.copies[0].allocation = DeviceAllocation(0, 128, 128, ptr=8192)
    w = rt.device_view(obj, 0)
    assert w is not v and w.ptr == 8192
