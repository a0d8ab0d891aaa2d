"""Step anatomy from the ncu launch list (profiles/r01_launches.csv) next to the bench's own
CUDA-event split (profiles/r01_bench.json) -> profiles/r01_ncu_step_summary.json."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
launches = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles/r01_launches.csv")
bench = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles/r01_bench.json")
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
step_kernels = ("vtx_kernel", "treduce_kernel", "tgather_kernel", "seg_tma_kernel")
tail = [(k, v) for k, v in recs if k.split("<")[0].split("(")[0].replace("void ", "").split("::")[-1]
        in step_kernels]
last = tail[-4 * 20:]
tot = sum(v for _, v in last)
share = {}
for k, v in last:
    name = k.replace("void ", "").split("(")[0].split("::")[-1]
    share[name] = share.get(name, 0.0) + v / tot
b = json.load(open(bench))
pk = b["roofline"]["per_kernel"]
ev = {k: pk[k]["ms"] for k in pk}
s = sum(ev.values())
traffic = json.load(open(os.path.join(ROOT, "profiles/ncu_traffic.json")))
out = {
    "source": "profiles/r01_launches.csv (ncu --metrics gpu__time_duration.sum --clock-control none; "
              "cold-cache, serialised)",
    "last_steps": 20,
    "step_us_under_ncu": tot / 20 / 1e3 if tot > 1e5 else tot / 20,
    "share": {k: round(v, 4) for k, v in share.items()},
    "bench_event_share": {k: round(v / s, 4) for k, v in ev.items()},
    "full_capture": "profiles/r01_step_prof.ncu-rep (ncu --set full of seg_tma_kernel and vtx_kernel<8>)",
    "dram_bytes_per_launch": traffic,
}
json.dump(out, open(os.path.join(ROOT, "profiles/r01_ncu_step_summary.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
