"""Host logic of the multi-process path, on CPU: world_size-2 (and 4) gloo
process groups check that every rank derives NCCL send/recv lists that
pair one-to-one in order (the cross-rank face exchange of DistributedJacobi,
the reference's per-face mp_send, jacobi.py:227-237), and that the
decomposition matches the reference's rank assignment (jacobi.py:325-339)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_02543_b200.jacobi import ChunkGrid, remote_ops

CASES = [((32768, 32768, 1), (4, 4, 1)), ((32768, 32768, 1), (8, 4, 1)),
         ((32768, 32768, 1), (64, 1, 1)), ((32768, 32768, 1), (8, 8, 1)),
         ((64, 64, 64), (2, 2, 2)), ((48, 40, 1), (6, 5, 1)), ((8, 8, 8), None)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for dom, grid in CASES:
            g = ChunkGrid(dom, ranks=world, grid=grid)
            mine = remote_ops(g, rank)
            everyone = [None] * world
            dist.all_gather_object(everyone, mine)
            for a in range(world):
                for b in range(world):
                    if a == b:
                        continue
                    sends = [(c, f, n) for k, p, c, f, n in everyone[a] if k == "send" and p == b]
                    recvs = [(c, f, n) for k, p, c, f, n in everyone[b] if k == "recv" and p == a]
                    assert sends == recvs, (dom, grid, a, b)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_remote_face_pairing_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in results), results


def test_rank_assignment_matches_reference():
    g = ChunkGrid((32768, 32768, 1), ranks=8, grid=(8, 8, 1))
    # lin = ix + cx*iy (jacobi.py:334-335); rank = lin*ranks//nchunks (325-326)
    for ch in g.chunks:
        assert ch.rank == ch.lin * 8 // 64
        assert ch.coord[1] == ch.rank
    ops = remote_ops(g, 3)
    assert {p for _, p, *_ in ops} == {2, 4}
    # y faces (strided columns) of 4096 cells: 8 chunks x 2 sides x send+recv
    assert len(ops) == 32 and all(n == 4096 for *_, n in ops)
