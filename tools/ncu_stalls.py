"""Summarise an ncu report's source page: stall reasons (all samples) and
the hottest SASS lines.   python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "(Not" not in h]
tot = dict.fromkeys(stalls, 0)
n_all, per = 0, []
for r in rows[2:]:
    try:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    n_all += n
    for s in stalls:
        tot[s] += int(r[ix[s]] or 0)
    per.append((n, r[ix["Source"]][:70], int(r[ix["Instructions Executed"]] or 0)))
print("samples", n_all)
for s, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print(f"  {s:24s} {v:8d} {v / n_all:.3f}")
per.sort(key=lambda x: -x[0])
for n, src, ex in per[:top]:
    print(f"{n:7d} {ex:10d}  {src}")
