"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the step
kernels from an `ncu --set full` capture -> profiles/ncu_traffic.json, keyed by the names
bench.py uses in its roofline table.

    python tools/ncu_traffic.py gpurun_out/step_prof.ncu-rep [profiles/ncu_traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

NAMES = {"seg_tma_kernel": "seg(Z)", "vtx_kernel<8>": "vtx(Z)", "h2_leaf_kernel": "h2_leaf",
         "h2_up_kernel": "h2_up", "h2_couple_kernel": "h2_couple", "h2_down_kernel": "h2_down",
         "h2s_up_kernel": "h2s_up(K1)", "h2s_down_kernel": "h2s_down(K2)", "xpad_kernel": "xpad"}


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        key = next((v for k, v in NAMES.items() if k in name.split("(")[0]), None)
        if key is None or key in res:
            continue
        rd = float(r[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
        res[key] = rd + wr
    json.dump(res, open(out, "w"), indent=1)
    print(res)


if __name__ == "__main__":
    main()
