"""Where a direct-path ping-pong hop spends host time: every libhrt_b200
call made through _native.call / CompletionToken, timed per function name
(perf_counter around the ctypes call), for 8 B and 1 MiB round trips.

python tools/pingpong_calls.py
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.pingpong import run_pingpong  # noqa: E402

acc = collections.defaultdict(lambda: [0, 0.0])
real_call = N.call


def timed_call(name, *args):
    t0 = time.perf_counter()
    try:
        return real_call(name, *args)
    finally:
        a = acc[name]
        a[0] += 1
        a[1] += time.perf_counter() - t0


L = N.lib()


class Timed:
    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        fn = getattr(self._lib, name)

        def w(*args):
            t0 = time.perf_counter()
            try:
                return fn(*args)
            finally:
                a = acc["lib." + name]
                a[0] += 1
                a[1] += time.perf_counter() - t0
        return w


for size in (8, 1 << 20):
    run_pingpong([size], iterations=20, path="direct", verify=False)  # warm-up
    acc.clear()
    N.call = timed_call
    N._lib = Timed(L)
    t0 = time.perf_counter()
    rep = run_pingpong([size], iterations=200, path="direct", verify=False)
    wall = time.perf_counter() - t0
    N.call = real_call
    N._lib = L
    print(f"size {size}: one-way {rep.rows[0]['mean_latency_s'] * 1e6:.1f} us; run wall {wall:.3f} s")
    for k, (n, t) in sorted(acc.items(), key=lambda x: -x[1][1])[:12]:
        print(f"   {k:32s} n={n:6d} total {t * 1e3:8.2f} ms  per call {t / n * 1e6:7.2f} us")
