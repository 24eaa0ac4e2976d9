"""Generate the golden vectors that pin the oracle (tests/test_oracle.py) and
the CUDA path (tests/test_jacobi_gpu.py) to the reference's own outputs.

Runs the UNMODIFIED reference (``/root/reference/pkg/src/hrt``) in this
container; the fixtures it writes are committed so that nothing on the GPU
box needs /root/reference.  Usage (from the repo root):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Outputs (tests/golden/):
    jacobi_ladder.json   run_jacobi3d results: checksum (repr), sha256 of the
                         C-order float64 interior, distinct-value count
    jacobi_small.npz     full interiors for the small ladder entries
    np_sum.json          np.sum of seeded float64 arrays (pins the checksum
                         restatement of numpy's pairwise summation)
    allocator.json       a seeded alloc/free trace through the reference
                         FreeListAllocator (devices.py:89-154)
    pingpong.json        sha256 of the ping-pong payload sequence
                         (pingpong.py:107,115) for 8 B .. 256 MiB
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

from hrt.bench.jacobi import jacobi_reference, run_jacobi3d
from hrt.devices import ClockMode, FreeListAllocator
from hrt.errors import DoubleFree, OutOfDeviceMemory

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, domain, steps, run_jacobi3d kwargs) — SURVEY.md §8(c) ladder plus
# edge cases: unit-extent chunks, zero steps, non-square chunk grids.
LADDER = [
    ("cube8_s3", (8, 8, 8), 3, {}),
    ("ac10_g111", (64, 64, 64), 10, dict(grid=(1, 1, 1))),
    ("ac10_g222", (64, 64, 64), 10, dict(grid=(2, 2, 2))),
    ("ac10_od2", (64, 64, 64), 10, dict(od=2)),
    ("ac10_od4", (64, 64, 64), 10, dict(od=4)),
    ("ac10_r2d2", (64, 64, 64), 10, dict(ranks=2, devices_per_rank=2)),
    ("slab64_s10", (64, 64, 1), 10, dict(grid=(4, 4, 1))),
    ("slab1024_s5", (1024, 1024, 1), 5, dict(grid=(4, 4, 1))),
    ("cfg1", (1024, 1024, 1), 100, dict(grid=(4, 4, 1), clock=ClockMode.WALL)),
    ("halo32_s20", (32, 32, 1), 20, dict(grid=(4, 4, 1))),
    ("halo32_s20_r2d2", (32, 32, 1), 20, dict(grid=(4, 4, 1), ranks=2, devices_per_rank=2)),
    ("halo32_s20_direct", (32, 32, 1), 20, dict(grid=(4, 4, 1), device_aware=True)),
    ("halo16_cube_s12", (16, 16, 16), 12, dict(grid=(4, 4, 4))),
    ("cube24_s30", (24, 24, 24), 30, dict(grid=(3, 3, 3))),
    ("slab48x40_s64", (48, 40, 1), 64, dict(grid=(6, 5, 1), devices_per_rank=8)),
    ("slab96x80_s13", (96, 80, 1), 13, dict(grid=(3, 5, 1))),
    ("slab256_s300", (256, 256, 1), 300, dict(grid=(8, 8, 1), devices_per_rank=8)),
    ("unit_chunks_slab", (8, 6, 1), 7, dict(grid=(8, 6, 1))),
    ("unit_chunks_cube", (5, 7, 3), 6, dict(grid=(5, 7, 3))),
    ("zero_steps", (8, 8, 1), 0, dict(grid=(2, 2, 1))),
    ("rect_slab", (40, 24, 1), 33, dict(grid=(5, 3, 1))),
    ("thin_x", (4, 64, 1), 9, dict(grid=(4, 2, 1))),
    ("zslab_3d", (12, 10, 6), 15, dict(grid=(2, 1, 3))),
]
SMALL_LIMIT = 40_000  # elements: store full arrays below this


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def ladder(big: bool):
    out, arrays = [], {}
    for name, domain, steps, kw in LADDER:
        t0 = time.time()
        kw = dict(kw)
        kw.setdefault("capacity", 1 << 30)
        _, cs, arr = run_jacobi3d(domain, steps=steps, **kw)
        ref = jacobi_reference(domain, steps)
        assert np.array_equal(arr, ref), name
        entry = dict(
            name=name, domain=list(domain), steps=steps,
            kwargs={k: (v.value if isinstance(v, ClockMode) else v) for k, v in kw.items()
                    if k != "capacity"},
            checksum=repr(cs), sha256=sha(arr), distinct=int(np.unique(arr).size),
            source="run_jacobi3d",
        )
        out.append(entry)
        if arr.size <= SMALL_LIMIT:
            arrays[name] = arr
        print(f"{name}: {cs!r} {entry['sha256'][:16]} ({time.time() - t0:.1f}s)", flush=True)
    if big:
        # cfg2 prefix: the chunked run needs ~55 GB here; jacobi_reference is
        # bitwise equal to run_jacobi3d by construction (asserted above on
        # every ladder entry), so the single-array solver produces the golden.
        for steps in (1, 3):
            t0 = time.time()
            # contiguous, as run_jacobi3d assembles it (jacobi.py:427-436);
            # np.sum over the strided interior view sums in another order
            arr = np.ascontiguousarray(jacobi_reference((16384, 16384, 1), steps))
            cs = float(np.sum(arr))
            out.append(dict(
                name=f"cfg2_prefix_s{steps}", domain=[16384, 16384, 1], steps=steps,
                kwargs=dict(grid=[8, 8, 1]), checksum=repr(cs), sha256=sha(arr),
                distinct=int(np.unique(arr).size), source="jacobi_reference",
            ))
            del arr
            print(f"cfg2_prefix_s{steps}: {cs!r} ({time.time() - t0:.1f}s)", flush=True)
    return out, arrays


def np_sums():
    rng = np.random.default_rng(2303_02543)
    out = []
    for n in [0, 1, 5, 7, 8, 9, 15, 16, 127, 128, 129, 255, 256, 1000, 4097, 65536 + 3,
              1_000_003, 7_340_033]:
        a = rng.random(n) * rng.choice([1.0, 1e-3, 1e6])
        out.append(dict(n=n, seed_index=len(out), sum=repr(float(np.sum(a))),
                        sha256=hashlib.sha256(a.tobytes()).hexdigest()))
    return out


def allocator_trace(seed=7, ops=4000, capacity=1 << 20):
    rnd = random.Random(seed)
    alloc = FreeListAllocator(capacity)
    live, trace = [], []
    for _ in range(ops):
        if live and rnd.random() < 0.45:
            off = live.pop(rnd.randrange(len(live)))
            size = alloc.free(off)
            trace.append(["free", off, size])
        elif rnd.random() < 0.02 and live:
            # double free of a freed offset is an error in the reference
            off = rnd.choice(live)
            alloc.free(off)
            live.remove(off)
            try:
                alloc.free(off)
                trace.append(["double_free", off, "accepted"])
            except DoubleFree:
                trace.append(["double_free", off, "DoubleFree"])
        else:
            size = rnd.choice([1, 100, 256, 257, 1000, 4096, 12345, 65536, 200000])
            try:
                off, granted = alloc.alloc(size)
                live.append(off)
                trace.append(["alloc", size, off, granted])
            except OutOfDeviceMemory:
                trace.append(["alloc", size, "OutOfDeviceMemory"])
        alloc.check()
    return dict(capacity=capacity, alignment=256, seed=seed, trace=trace,
                final_free=alloc.free_bytes)


def pingpong_payloads():
    rng = np.random.default_rng(99)
    out = []
    size = 8
    while size <= 256 << 20:
        payload = rng.integers(0, 256, size=size, dtype=np.uint8)
        out.append(dict(size=size, sha256=hashlib.sha256(payload.tobytes()).hexdigest()))
        size *= 2
    return out


def main():
    big = "--big" in sys.argv
    entries, arrays = ladder(big)
    if not big and os.path.exists(os.path.join(HERE, "jacobi_ladder.json")):
        # keep previously generated big entries
        old = json.load(open(os.path.join(HERE, "jacobi_ladder.json")))
        entries += [e for e in old["entries"] if e["name"].startswith("cfg2_prefix")]
    json.dump(dict(generator="tests/golden/make_golden.py", reference="/root/reference/pkg",
                   entries=entries),
              open(os.path.join(HERE, "jacobi_ladder.json"), "w"), indent=1)
    np.savez_compressed(os.path.join(HERE, "jacobi_small.npz"), **arrays)
    json.dump(dict(seed=2303_02543, cases=np_sums()),
              open(os.path.join(HERE, "np_sum.json"), "w"), indent=1)
    json.dump(allocator_trace(), open(os.path.join(HERE, "allocator.json"), "w"))
    json.dump(dict(seed=99, payloads=pingpong_payloads()),
              open(os.path.join(HERE, "pingpong.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
