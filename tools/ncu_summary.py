"""Summarise `ncu --set full` reports into markdown (for profiles/) and per-launch DRAM traffic
(profiles/traffic.json, read by bench.py). Usage:
  ncu_summary.py OUT.md TRAFFIC.json NAME=report.ncu-rep:kernel_regex [...]"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep, regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{regex}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stalls(d):
    st = []
    for k, (v, _) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    st.sort(reverse=True)
    return ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in st[:6])


def main():
    out_md, out_json = sys.argv[1], sys.argv[2]
    lines, traffic = [], {}
    for spec in sys.argv[3:]:
        name, rest = spec.split("=", 1)
        rep, regex = rest.split(":", 1)
        d = raw(rep, regex)
        lines.append(f"## {name}\n")
        lines.append(f"source: `{rep}` (kernel regex `{regex}`)\n")
        for m in METRICS:
            if m in d:
                v, u = d[m]
                lines.append(f"- {m}: {v} {u}")
        lines.append(f"- top stall reasons (pc sampling): {stalls(d)}\n")

        def as_bytes(m):
            v, u = d[m]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[name] = as_bytes("dram__bytes_read.sum") + as_bytes("dram__bytes_write.sum")
    open(out_md, "a").write("\n".join(lines) + "\n")
    traffic["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), ncu --set full, "
                       "C2 hybrid with the measured cost model, tools/profile_run.py")
    json.dump(traffic, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main()
