"""Top SASS lines by warp-stall samples from an ncu report: ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = r[1]; rows = r[2:]
i = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[i] or 0) for x in rows)
print("total samples", tot)
order = sorted(range(len(rows)), key=lambda k: -int(rows[k][i] or 0))[:n]
for k in order:
    x = rows[k]
    print(f"{int(x[i]):7d} {100*int(x[i])/tot:5.1f}%  {x[0][-5:]}  {x[1][:90]}")
