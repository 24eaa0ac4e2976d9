"""Warp-stall samples of an ncu report grouped by instruction execution
count (separates e.g. a producer's per-row loop from the consumers' per-plane
code):   python tools/ncu_buckets.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "(Not" not in h]
b = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in rows[2:]:
    try:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    e = b[ex]
    e[0] += n
    e[1] += 1
    for s in stalls:
        e[2][s] += int(r[ix[s]] or 0)
tot = sum(v[0] for v in b.values())
for ex, (n, k, c) in sorted(b.items(), key=lambda x: -x[1][0])[:14]:
    top = ", ".join(f"{s[6:]} {v / max(n, 1):.2f}" for s, v in c.most_common(3))
    print(f"exec {ex:10d}  instrs {k:4d}  samples {n:8d} ({n / tot:.3f})  {top}")
