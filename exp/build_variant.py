"""Experiment builds: libhrt_b200.so with extra -D flags into exp/<name>/
(never used by the product; copied over the package library on a GPU box
only for A/B measurements)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_02543_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), name)
os.makedirs(out, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.run([B.nvcc(), *B.flags([f"-D{d}" for d in defs]), "-c",
                    os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", os.path.join(out, "libhrt_b200.so"), *objs,
                "-lcudart", "-ldl"], check=True)
print(os.path.join(out, "libhrt_b200.so"))
