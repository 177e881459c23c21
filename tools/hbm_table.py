"""Per-kernel HBM traffic and achieved GB/s of one evaluation, from an ncu launch list captured
with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (serialised,
cold-cache launches). Kernels are grouped by the SURVEY §8(a) row they implement.
Usage: hbm_table.py launches.csv [hbm_peak_GBps] > table.md"""
import csv
import sys
from collections import defaultdict

ROWS = [  # (row, kernel-name prefixes)
    ("a1 bbox + root cube", ["k_bbox", "k_root"]),
    ("a2 Morton keys", ["k_keys"]),
    ("a3 sort + gather", ["k_gather", "k_sort_fixup"]),
    ("a4/a5 octree + geometry", ["k_tree_coop", "k_split", "k_emit", "k_level_total", "k_leaf_", "k_root_cell",
                                 ]),
    ("a7 P2M", ["k_p2m"]),
    ("a8 M2M (shift GEMM levels + reduce)", ["k_shift_m2m", "k_m2m"]),
    ("a9 traversal", ["k_traverse", "k_pack_cells"]),
    ("a10 M2L class prep", ["k_m2l_keys", "k_m2l_pair", "k_m2l_class", "k_m2l_run", "k_m2l_gather",
                            "k_m2l_build_T", "k_shift_items", "k_shift_keys"]),
    ("a10 M2L + a8/a13 shift GEMMs (tcgen05)", ["k_m2l_tc"]),
    ("a12 P2P", ["k_p2p"]),
    ("a13 L2L (shift add)", ["k_shift_l2l", "k_l2l"]),
    ("a14/a15 L2P + un-permute", ["k_l2p"]),
]


def main():
    path = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6458.4
    per = defaultdict(lambda: {"us": 0.0, "rd": 0.0, "wr": 0.0})
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        key = (r["ID"], name)
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            per[key]["us"] += v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            per[key]["rd" if "read" in m else "wr"] += v * scale
    agg = defaultdict(lambda: {"us": 0.0, "bytes": 0.0, "n": 0})
    phase = "a3"  # CUB sorts / scans belong to the phase of the last named kernel launched before
    for (lid, name), d in sorted(per.items(), key=lambda kv: int(kv[0][0])):
        if name.startswith("k_m2l_keys"):
            phase = "m2l"
        elif name.startswith("k_shift_keys"):
            phase = "shift"
        elif name.startswith(("k_split", "k_leaf_flags")):
            phase = "a4"
        elif name.startswith(("k_m2l_class_flags", "k_shift_items", "k_m2l_run_items", "k_gather")):
            pass
        if name.startswith("cub::"):
            row = {"a3": "a3 sort + gather", "a4": "a4/a5 octree + geometry",
                   "m2l": "a10 M2L class prep", "shift": "a10 M2L class prep"}[phase]
            if "RadixSort" in name and phase == "a4":
                row = "a3 sort + gather"
        else:
            row = next((rw for rw, pre in ROWS if any(name.startswith(p) for p in pre)), "other: " + name[:40])
        agg[row]["us"] += d["us"]
        agg[row]["bytes"] += d["rd"] + d["wr"]
        agg[row]["n"] += 1
    print(f"| §8(a) row | launches | us (serialised) | DRAM MB | GB/s | of measured HBM ({peak:.0f} GB/s) |")
    print("|---|---|---|---|---|---|")
    order = [rw for rw, _ in ROWS] + sorted(k for k in agg if k.startswith("other"))
    for rw in order:
        if rw not in agg:
            continue
        d = agg[rw]
        gbs = d["bytes"] / (d["us"] * 1e-6) / 1e9 if d["us"] > 0 else 0.0
        print(f"| {rw} | {d['n']} | {d['us']:.1f} | {d['bytes'] / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.3f} |")


if __name__ == "__main__":
    main()
