"""Multi-process parity check (run under torchrun, one process per GPU):
DistributedJacobi with NCCL faces vs the C oracle, field and residual.

torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2303_02543_b200.distributed import DistributedJacobi, init_process  # noqa: E402
from paper_2303_02543_b200.jacobi import ChunkGrid  # noqa: E402
from oracle import oracle as O  # noqa: E402

rank, world, local = init_process("nccl")


def owned(s, band):
    """This rank's owned cells of its bounding box (a staircase split's box
    also covers other ranks' chunks): NaN elsewhere, so assembling boxes
    never overwrites a neighbour's cells."""
    out = np.full(band.shape, np.nan)
    for lin in s.owned:
        ch = s.grid.chunks[lin]
        a = [ch.offsets[k] - s.box_lo[k] for k in range(3)]
        e = s.grid.ext
        out[a[0]:a[0] + e[0], a[1]:a[1] + e[1], a[2]:a[2] + e[2]] = \
            band[a[0]:a[0] + e[0], a[1]:a[1] + e[1], a[2]:a[2] + e[2]]
    return out


def place(full, l0, b):
    view = full[l0[0]:l0[0] + b.shape[0], l0[1]:l0[1] + b.shape[1], l0[2]:l0[2] + b.shape[2]]
    m = ~np.isnan(b)
    view[m] = b[m]
# y faces (strided: packed), x faces (contiguous rows: direct), 3D z faces
cases = [((1024, 1024, 1), (4, 4, 1), 60), ((600, 520, 1), (3, 2 * world, 1), 77),
         ((512, 300, 1), (2 * world, 1, 1), 45), ((48, 40, 32), (2, 2, world), 21),
         ((4096, 4096, 1), (8, 8, 1), 130), ((64, 40, 48), (2 * world, 1, 1), 15)]
ok_all = True
for dom, grid, steps in cases:
    cg = ChunkGrid(dom, ranks=world, grid=grid)
    # 3D x-bands: the opt-in fused push + cross-process wavefront
    s = DistributedJacobi(cg, rank, world, local, vpush=(grid == (2 * world, 1, 1) and dom[2] > 1))
    boxes = []
    for job in range(2):  # two jobs: re-priming and monotone step tags / counters
        s.upload()
        if job == 0:
            s.run(steps, residual=True)
            res = s.global_residual_history()
        else:  # several launches per job: counters carry across launches
            for n in (steps // 3, 1, steps - steps // 3 - 1):
                s.run(n, residual=False)
        boxes.append(s.download())
        s.check_ipc()
    box = owned(s, boxes[0])
    same = np.array_equal(boxes[0], boxes[1])
    lo = s.box_lo
    ipc = (s.ipc, s.persistent)
    s.close()
    flags = [None] * world
    dist.all_gather_object(flags, (same, ipc))
    if rank == 0:
        print(f"  jobs identical on all ranks: {all(f[0] for f in flags)}; "
              f"(ipc push, wavefront): {[f[1] for f in flags]}", flush=True)
        ok_all &= all(f[0] for f in flags)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, box))
    if rank == 0:
        from oracle import oracle as O

        full = np.empty(dom)
        for (l0, b) in parts:
            place(full, l0, b)
        ref, rres = O.jacobi_c(dom, steps, residual=True)
        ok = np.array_equal(full, ref) and np.array_equal(res, rres)
        ok_all &= ok
        print(f"dist_check world={world} dom={dom} grid={grid} steps={steps}: "
              f"field {'OK' if np.array_equal(full, ref) else 'DIFF'} "
              f"resid {'OK' if np.array_equal(res, rres) else 'DIFF'}", flush=True)
# random signed data through the cross-process two-step passes (x-bands:
# rim rows read over NVLink from the neighbour rank's IPC-mapped chunks):
# every rank uploads its band of one seeded field; the gathered field and
# the residual history vs the numpy oracle
os.environ["HRT_FUSE2"] = "2"  # small domains: force two-step passes
for dom, grid, steps in [((256, 130, 1), (2 * world, 1, 1), 14),
                         ((96, 64, 1), (4 * world, 1, 1), 9),
                         # y-bands (column faces and corners on other ranks,
                         # cfg5's decomposition) and a 2D block staircase
                         ((64, 96 * world, 1), (2, 2 * world, 1), 13),
                         ((120, 16 * (2 * world + 1), 1), (3, 2 * world + 1, 1), 10),
                         # volumes: volume_wave2_kernel (guarded instance)
                         ((12 * world, 20, 130), (2 * world, 1, 1), 13)]:
    cg = ChunkGrid(dom, ranks=world, grid=grid)
    s = DistributedJacobi(cg, rank, world, local)
    full_init = np.random.default_rng(7).random(dom) * 4.0 - 1.0
    lo, bx = s.box_lo, s.box
    s.upload(full_init[lo[0]:lo[0] + bx[0], lo[1]:lo[1] + bx[1], lo[2]:lo[2] + bx[2]])
    s.run(steps, residual=True)
    res = s.global_residual_history()
    band = owned(s, s.download())
    two = s.two_step
    s.check_ipc()
    s.close()
    parts = [None] * world
    dist.all_gather_object(parts, (lo, band, two))
    if rank == 0:
        full = np.empty(dom)
        for (l0, b, _) in parts:
            place(full, l0, b)
        rr = []
        ref = O.jacobi_reference(dom, steps, initial=full_init, residuals=rr)
        ok = np.array_equal(full, ref) and np.array_equal(res, np.array(rr))
        if os.environ.get("HRT_PERSIST", "1") != "0":  # (tile launches have no passes)
            ok &= all(p[2] for p in parts)  # two-step passes were in use on every rank
        ok_all &= ok
        print(f"dist_check world={world} random {dom} grid={grid} steps={steps} two-step="
              f"{[p[2] for p in parts]}: {'OK' if ok else 'DIFF'}", flush=True)
# two-step passes across processes split over several run() calls, with a
# re-upload between jobs: single steps -> fused passes -> the next run's
# ghost priming after stale ghosts (what bench's job stream does)
for dom, grid, parts in [((256, 130, 1), (2 * world, 1, 1), (5, 1, 9)),
                         ((96, 64, 1), (4 * world, 1, 1), (4, 7, 2)),
                         # volumes, non-negative: the unguarded instance
                         ((12 * world, 20, 130), (2 * world, 1, 1), (5, 1, 9))]:
    cg = ChunkGrid(dom, ranks=world, grid=grid)
    s = DistributedJacobi(cg, rank, world, local)
    lo, bx = s.box_lo, s.box
    outs = []
    for job in range(2):
        full_init = np.random.default_rng(70 + job).random(dom) * 2.0
        s.upload(full_init[lo[0]:lo[0] + bx[0], lo[1]:lo[1] + bx[1], lo[2]:lo[2] + bx[2]])
        for n in parts:
            s.run(n, residual=False)
        outs.append((full_init, owned(s, s.download())))
    two = s.two_step
    s.check_ipc()
    s.close()
    parts_all = [None] * world
    dist.all_gather_object(parts_all, (lo, [o[1] for o in outs], two))
    if rank == 0:
        ok = True
        for job, (full_init, _) in enumerate(outs):
            full = np.empty(dom)
            for (l0, bands, _) in parts_all:
                place(full, l0, bands[job])
            ref = O.jacobi_reference(dom, sum(parts), initial=full_init)
            ok &= np.array_equal(full, ref)
        ok_all &= ok
        print(f"dist_check world={world} split runs {dom} grid={grid} parts={parts} two-step="
              f"{[p[2] for p in parts_all]}: {'OK' if ok else 'DIFF'}", flush=True)
del os.environ["HRT_FUSE2"]
# uneven chunk counts per rank ((2*world-1) x-bands: one rank holds one chunk
# fewer): every rank must pick the same tiling (rows, two-step) from the
# grid's largest per-rank chunk count, or neighbours index each other's
# tile counters wrongly (4096 x 8192 chunks sit at the 256-row / two-step
# thresholds for 2 vs 1 chunks per GPU)
for fuse in ("1", "2"):
    os.environ["HRT_FUSE2"] = fuse
    nb = 2 * world - 1
    dom, steps = (nb * 4096, 8192, 1), 21
    cg = ChunkGrid(dom, ranks=world, grid=(nb, 1, 1))
    s = DistributedJacobi(cg, rank, world, local)
    s.upload()
    s.run(steps, residual=True)
    res = s.global_residual_history()
    band, lo = s.download(), s.box_lo
    til = s.tiling()[local]
    s.check_ipc()
    s.close()
    parts = [None] * world
    dist.all_gather_object(parts, (lo, band, til, len(cg.per_rank[rank])))
    if rank == 0:
        from oracle import oracle as O

        full = np.empty(dom)
        for (l0, b, _, _) in parts:
            full[l0[0]:l0[0] + b.shape[0]] = b
        ref, rres = O.jacobi_c(dom, steps, residual=True)
        ok = np.array_equal(full, ref) and np.array_equal(res, rres)
        ok &= len({p[2] for p in parts}) == 1
        ok_all &= ok
        print(f"dist_check world={world} uneven {dom} chunks/rank={[p[3] for p in parts]} "
              f"HRT_FUSE2={fuse} tilings={[p[2] for p in parts]}: {'OK' if ok else 'DIFF'}",
              flush=True)
    del os.environ["HRT_FUSE2"]
# full cfg3 size: the N-rank x-band run (IPC wavefront) against one GPU,
# field bands and residual history bitwise (rank 0 solves the whole domain
# on its own GPU after the distributed run)
if os.environ.get("DIST_CHECK_FULL", "1") != "0":
    dom, steps = (32768, 32768, 1), 40
    cg = ChunkGrid(dom, ranks=world, grid=(8 * world, 1, 1))
    s = DistributedJacobi(cg, rank, world, local)
    s.upload()
    s.run(steps, residual=True)
    band, lo = s.download(), s.box_lo
    res = s.global_residual_history()
    ipc = (s.ipc, s.persistent)
    s.close()
    parts = [None] * world
    dist.all_gather_object(parts, (lo, band.shape, float(band.sum()), band[::97, ::89].copy()))
    if rank == 0:
        from paper_2303_02543_b200.jacobi import JacobiSolver

        one = JacobiSolver(ChunkGrid(dom, grid=(8, 1, 1)), gpus=[local])
        one.upload()
        one.run(steps, residual=True)
        full = one.download()
        r1 = one.residual_history()
        one.close()
        ok = np.array_equal(res, r1)
        for (l0, shape, ssum, sample) in parts:
            ref = full[l0[0]:l0[0] + shape[0], l0[1]:l0[1] + shape[1]]
            ok &= float(ref.sum()) == ssum and np.array_equal(ref[::97, ::89], sample)
        ok &= np.array_equal(band, full[lo[0]:lo[0] + band.shape[0]])
        ok_all &= ok
        print(f"dist_check world={world} full cfg3 {dom} steps={steps} (ipc, wavefront)={ipc}: "
              f"{'OK' if ok else 'DIFF'}", flush=True)
# full paper3d size: the N-rank x-band volume run (cross-process two-step
# passes through chains) against one GPU (itself bitwise vs the oracle in
# test_parity_fullsize_gpu), field samples, sums and residual history
if os.environ.get("DIST_CHECK_FULL", "1") != "0" and os.environ.get("HRT_PERSIST", "1") != "0":
    dom, steps = (1024, 1024, 768), 100
    cg = ChunkGrid(dom, ranks=world, grid=(8 * world, 1, 1))
    s = DistributedJacobi(cg, rank, world, local)
    s.upload()
    s.run(steps, residual=True)
    band, lo = s.download(), s.box_lo
    res = s.global_residual_history()
    two = s.two_step
    s.close()
    parts = [None] * world
    dist.all_gather_object(parts, (lo, band.shape, float(band.sum()), band[::31, ::29, ::7].copy(), two))
    if rank == 0:
        from paper_2303_02543_b200.jacobi import JacobiSolver

        one = JacobiSolver(ChunkGrid(dom, grid=(8, 1, 1)), gpus=[local])
        one.upload()
        one.run(steps, residual=True)
        full = one.download()
        r1 = one.residual_history()
        one.close()
        ok = np.array_equal(res, r1) and all(p[4] for p in parts)
        for (l0, shape, ssum, sample, _) in parts:
            ref = full[l0[0]:l0[0] + shape[0]]
            ok &= float(ref.sum()) == ssum and np.array_equal(ref[::31, ::29, ::7], sample)
        ok &= np.array_equal(band.view(np.uint64), full[lo[0]:lo[0] + band.shape[0]].view(np.uint64))
        ok_all &= ok
        print(f"dist_check world={world} full paper3d {dom} steps={steps} two-step="
              f"{[p[4] for p in parts]}: {'OK' if ok else 'DIFF'}", flush=True)
        del full
dist.barrier()
if rank == 0:
    print("DIST_CHECK", "PASS" if ok_all else "FAIL", flush=True)
dist.destroy_process_group()
