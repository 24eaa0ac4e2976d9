"""Print selected keys of the last JSON line on stdin (bench.py output).

python bench.py ... | python tools/jline.py value tasks_per_s roofline.frac
"""
import json
import sys

lines = [l for l in sys.stdin.read().splitlines() if l.startswith("{")]
if not lines:
    print("no JSON line")
    sys.exit(1)
d = json.loads(lines[-1])
out = []
for key in sys.argv[1:]:
    v = d
    for part in key.split("."):
        v = v.get(part) if isinstance(v, dict) else None
    out.append(f"{key}={v}")
print(" ".join(out))
