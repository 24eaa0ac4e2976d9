"""Host cost of the message path's native calls (µs per call, 8 B copies
GPU1 <- GPU0) and the device-side latency of one small peer copy seen from
the host (enqueue -> event query reports complete), per copy method.

python tools/msg_micro.py
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2303_02543_b200 import _native as N  # noqa: E402
from paper_2303_02543_b200.devices import DevicePool, Stream  # noqa: E402

n = N.gpu_count()
g0, g1 = 0, (1 if n > 1 else 0)
N.lib().hrt_enable_peer_access(g1, g0)
N.lib().hrt_enable_peer_access(g0, g1)
p0, p1 = DevicePool(g0, 1 << 22), DevicePool(g1, 1 << 22)
src = p0.alloc(1 << 20)[2]
dst = p1.alloc(1 << 20)[2]
st = Stream(g1)
L = N.lib()
R = 2000


def per_call(fn, reps=R):
    fn()
    st.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    st.synchronize()
    return (t1 - t0) / reps * 1e6


sz = ctypes.c_uint64(8)
d, s = ctypes.c_void_p(dst), ctypes.c_void_p(src)
tok = ctypes.c_uint64()
print(f"GPUs {g0}->{g1}")
print(f"  ctypes no-op (hrt_device_count)   {per_call(lambda: L.hrt_device_count(ctypes.byref(ctypes.c_int()))):6.2f} us")
print(f"  hrt_copy_peer_async 8B            {per_call(lambda: L.hrt_copy_peer_async(st.h, d, g1, s, g0, sz)):6.2f} us")
print(f"  hrt_copy_async (UVA) 8B           {per_call(lambda: L.hrt_copy_async(st.h, d, s, sz)):6.2f} us")
print(f"  hrt_copy_sm_async 16B             {per_call(lambda: L.hrt_copy_sm_async(st.h, d, s, ctypes.c_uint64(16), 0)):6.2f} us")


def ordered(method, b=8):
    L.hrt_copy_ordered(st.h, d, s, ctypes.c_uint64(b), 1, None, 0, method, ctypes.byref(tok))
    L.hrt_token_release(tok)


print(f"  hrt_copy_ordered CE 8B (+token)   {per_call(lambda: ordered(0)):6.2f} us")
print(f"  hrt_copy_ordered SM 16B (+token)  {per_call(lambda: ordered(1, 16)):6.2f} us")


def rec():
    L.hrt_token_record(st.h, ctypes.byref(tok))
    L.hrt_token_release(tok)


print(f"  hrt_token_record+release          {per_call(rec):6.2f} us")
L.hrt_token_record(st.h, ctypes.byref(tok))
st.synchronize()
print(f"  hrt_token_query (complete)        {per_call(lambda: L.hrt_token_query(tok)):6.2f} us")
L.hrt_token_release(tok)

for name, fn in [("peer CE", lambda b: L.hrt_copy_peer_async(st.h, d, g1, s, g0, ctypes.c_uint64(b))),
                 ("UVA CE", lambda b: L.hrt_copy_async(st.h, d, s, ctypes.c_uint64(b))),
                 ("SM pull", lambda b: L.hrt_copy_sm_async(st.h, d, s, ctypes.c_uint64(b), 0))]:
    for b in (16, 65536, 1 << 20):
        lat = []
        for it in range(300):
            t0 = time.perf_counter()
            fn(b)
            L.hrt_token_record(st.h, ctypes.byref(tok))
            while L.hrt_token_query(tok) == 0:
                pass
            lat.append(time.perf_counter() - t0)
            L.hrt_token_release(tok)
        print(f"  {name:8s} {b:8d} B enqueue->complete seen: median {np.median(lat[20:]) * 1e6:6.2f} us")

# alternating directions (a ping-pong's two copies): GPU1<-GPU0 on GPU1's
# stream, then GPU0<-GPU1 on GPU0's stream ordered after the first
st0 = Stream(g0)
src1 = p1.alloc(1 << 20)[2]
dst0 = p0.alloc(1 << 20)[2]
t1, t2 = ctypes.c_uint64(), ctypes.c_uint64()
for method in (0, 1):
    def pair(wait):
        L.hrt_copy_ordered(st.h, d, s, ctypes.c_uint64(16), 1, None, 0, method, ctypes.byref(t1))
        w = (ctypes.c_uint64 * 1)(t1.value)
        L.hrt_copy_ordered(st0.h, ctypes.c_void_p(dst0), ctypes.c_void_p(src1), ctypes.c_uint64(16), 1,
                           w if wait else None, 1 if wait else 0, method, ctypes.byref(t2))
        L.hrt_token_release(t1)
        L.hrt_token_release(t2)
    for wait in (False, True):
        us = per_call(lambda: pair(wait), 1000)
        st0.synchronize()
        print(f"  alternating pair method {method} cross-wait {wait}: {us / 2:6.2f} us per copy")
