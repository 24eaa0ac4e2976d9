"""Pin the oracle (CPU restatement, oracle/) to the reference's own outputs
(tests/golden/, produced by tests/golden/make_golden.py running
/root/reference/pkg/src/hrt).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _entries(ladder, big=False):
    return [e for e in ladder.values() if e["name"].startswith("cfg2_prefix") == big]


def test_c_oracle_matches_reference_ladder(oracle, ladder):
    """Every ladder entry: C restatement of jacobi_reference == run_jacobi3d
    output bit for bit, and np.sum restatement == the reference checksum."""
    for e in _entries(ladder):
        arr = oracle.jacobi_c(tuple(e["domain"]), e["steps"])
        assert sha(arr) == e["sha256"], e["name"]
        assert repr(oracle.checksum(arr)) == e["checksum"], e["name"]
        assert int(np.unique(arr).size) == e["distinct"], e["name"]


def test_c_oracle_cfg2_prefix(oracle, ladder):
    """16384^2 slab, 1 and 3 steps (the cfg2 shape)."""
    for e in _entries(ladder, big=True):
        arr = oracle.jacobi_c(tuple(e["domain"]), e["steps"])
        assert sha(arr) == e["sha256"], e["name"]
        assert repr(oracle.checksum(arr)) == e["checksum"], e["name"]


def test_numpy_oracle_matches_small_fixtures(oracle, ladder, small_arrays):
    for name, ref in small_arrays.items():
        e = ladder[name]
        got = oracle.jacobi_reference(tuple(e["domain"]), e["steps"])
        assert np.array_equal(got, ref), name
        assert np.array_equal(oracle.jacobi_c(tuple(e["domain"]), e["steps"]), ref), name


def test_residual_definition(oracle):
    """Residual history = max|u_{s+1}-u_s| (builder-defined):
    C oracle vs a direct numpy evaluation."""
    dom, steps = (12, 10, 6), 9
    _, res = oracle.jacobi_c(dom, steps, residual=True)
    prev = np.zeros(dom)
    for s in range(steps):
        cur = oracle.jacobi_reference(dom, s + 1)
        assert res[s] == np.max(np.abs(cur - prev)), s
        prev = cur
    _, res2 = oracle.jacobi_c((20, 16, 1), 7, residual=True)
    prev = np.zeros((20, 16, 1))
    for s in range(7):
        cur = oracle.jacobi_reference((20, 16, 1), s + 1)
        assert res2[s] == np.max(np.abs(cur - prev))
        prev = cur


def test_np_sum_restatement_matches_numpy(oracle):
    g = load_golden("np_sum.json")
    rng = np.random.default_rng(g["seed"])
    for case in g["cases"]:
        a = rng.random(case["n"]) * rng.choice([1.0, 1e-3, 1e6])
        assert hashlib.sha256(a.tobytes()).hexdigest() == case["sha256"]
        assert repr(oracle.checksum(a)) == case["sum"], case["n"]
        assert repr(float(np.sum(a))) == case["sum"]


def test_allocator_restatement_replays_reference_trace(oracle):
    g = load_golden("allocator.json")
    a = oracle.FirstFitAllocator(g["capacity"], g["alignment"])
    for op in g["trace"]:
        if op[0] == "alloc":
            if op[2] == "OutOfDeviceMemory":
                with pytest.raises(MemoryError):
                    a.alloc(op[1])
            else:
                assert a.alloc(op[1]) == (op[2], op[3])
        elif op[0] == "free":
            assert a.free(op[1]) == op[2]
        else:
            # double free: first free succeeds, second raises
            a.free(op[1])
            with pytest.raises(KeyError):
                a.free(op[1])
    assert a.free_bytes == g["final_free"]


def test_pingpong_payload_sequence(oracle):
    g = load_golden("pingpong.json")
    sizes = [p["size"] for p in g["payloads"] if p["size"] <= (1 << 20)]
    for (size, payload), p in zip(oracle.pingpong_payloads(sizes, g["seed"]), g["payloads"]):
        assert size == p["size"]
        assert hashlib.sha256(payload.tobytes()).hexdigest() == p["sha256"]


def test_chunk_layout_matches_reference_decomposition(oracle):
    """Ranks/devices/neighbour assignment restated from jacobi.py:300-380."""
    chunks = oracle.chunk_layout((8, 8, 8), ranks=2, devices_per_rank=2, od=2)
    assert [c["rank"] for c in chunks] == [0] * 4 + [1] * 4
    assert [c["device_local"] for c in chunks] == [0, 0, 1, 1] * 2
    assert chunks[0]["neighbors"] == {5: 1}
    assert chunks[3]["neighbors"] == {4: 2, 5: 4}
