"""Step anatomy from the ncu launch list (profiles/rNN_launches.csv: cold-cache, serialised
per-launch times) next to the bench's own CUDA-event split -> profiles/rNN_ncu_step_summary.json.

    python tools/step_summary.py [launches.csv] [bench.json] [round tag, default r02]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[3] if len(sys.argv) > 3 else "r02"
launches = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, f"profiles/{TAG}_launches.csv")
bench = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, f"profiles/{TAG}_bench.json")
STEP = ("seg_tma_kernel", "h2_leaf_kernel", "h2_up_kernel", "h2_couple_kernel", "h2_down_kernel")


def short(k):
    k = k.replace("void ", "").split("(")[0].split("::")[-1]
    return k.split("<")[0] if k.startswith("h2s_") else k  # h2s_down_kernel<stages, slot bytes>


rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
recs = [(short(r[ki]), float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
# device steps: the consecutive launch sequence of one step (the e2e steps copy x in by memcpy
# and are excluded): two-kernel H2 step (round 2) or the five-launch walk + segment step (round 1)
SEQS = [["h2s_up_kernel", "h2s_down_kernel"],
        ["xpad_kernel", "h2s_up_kernel", "h2s_down_kernel"],
        ["h2_leaf_kernel", "h2_up_kernel", "h2_couple_kernel", "h2_down_kernel", "seg_tma_kernel<5, 512>"]]
for SEQ in SEQS:
    L = len(SEQ)
    steps = [recs[i:i + L] for i in range(len(recs) - L + 1) if [k for k, _ in recs[i:i + L]] == SEQ]
    if steps:
        break
nsteps = len(steps)
per = {k: sorted(st[j][1] for st in steps)[nsteps // 2] / 1e3 for j, k in enumerate(SEQ)}
tot = sum(per.values())
share = {k: v / tot for k, v in per.items()}
b = json.load(open(bench))
pk = b["roofline"]["per_kernel"]
ev = {k: pk[k]["ms"] for k in pk}
s = sum(ev.values())
tp = os.path.join(ROOT, f"profiles/{TAG}_ncu_traffic.json")
out = {
    "source": f"profiles/{TAG}_launches.csv (ncu --metrics gpu__time_duration.sum --clock-control none; "
              "cold-cache, serialised)",
    "device_steps_in_list": nsteps,
    "step_us_under_ncu": round(tot, 2),
    "us_per_step_median": {k: round(v, 2) for k, v in per.items()},
    "share": {k: round(v, 4) for k, v in share.items()},
    "bench_event_share": {k: round(v / s, 4) for k, v in ev.items()},
    "full_capture": f"profiles/{TAG}_step_prof.ncu-rep (ncu --set full of the step kernels)",
    "dram_bytes_per_launch": json.load(open(tp)) if os.path.exists(tp) else None,
}
json.dump(out, open(os.path.join(ROOT, f"profiles/{TAG}_ncu_step_summary.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
