"""Aggregate an ncu report's SASS source page: samples and stall reasons per instruction class,
and the hottest instructions. Usage: ncu_sass_hot.py report.ncu-rep [kernel_regex] [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
regex = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if regex:
    cmd += ["-k", f"regex:{regex}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
by_op = defaultdict(lambda: defaultdict(float))
hot = []
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    try:
        n = float(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    tot += n
    by_op[op]["samples"] += n
    by_op[op]["executed"] += float(r[ix["Instructions Executed"]] or 0)
    for c in stall_cols:
        try:
            by_op[op][c] += float(r[ix[c]] or 0)
        except ValueError:
            pass
    hot.append((n, r[ix["Address"]][-5:], src[:70], {c[6:]: r[ix[c]] for c in stall_cols if r[ix[c]] not in ("0", "")}))
print(f"total samples {tot:.0f}")
for op, d in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:25]:
    st = sorted(((v, k[6:]) for k, v in d.items() if k.startswith("stall_")), reverse=True)[:4]
    print(f"{op:12s} {100 * d['samples'] / tot:5.1f}%  exec {d['executed']:.3g}  " + ", ".join(f"{k} {v:.0f}" for v, k in st))
print("--- hottest instructions")
for n, a, s, st in sorted(hot, reverse=True)[:top]:
    print(f"{100 * n / tot:5.2f}% {a} {s:70s} {st}")
