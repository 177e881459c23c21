"""Print the A/B lines written by tools/ab_bench.sh: ms per step, phases, P2P/M2L roofline fractions."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_*.json")):
    try:
        d = json.loads([x for x in open(f) if x.startswith("{")][-1])
    except (IndexError, ValueError):
        print(f, "NO RESULT")
        continue
    r = d["roofline"]
    fr = {r["kernel"]: round(r["frac"], 3), r["secondary"]["kernel"]: round(r["secondary"]["frac"], 3)}
    print(f.split("/")[-1], round(d["ms_per_step"], 3), {k[3:]: round(v, 3) for k, v in d["phases_ms"].items()}, fr,
          d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
