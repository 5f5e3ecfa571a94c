"""roofline.traffic evidence: DRAM bytes (dram__bytes_read.sum +
dram__bytes_write.sum, one `ncu --set full` capture) of the longest dense
GEMM launch of a profiled step, next to its algorithmic bytes (operands read
once + output written once, from the same step's per-launch event CSV - the
two lists are in the same launch order). Writes / updates
profiles/traffic.json, which bench.py reports as roofline.traffic.

python tools/ncu_traffic.py NCU_RAW_CSV EVENTS_CSV PRESET SOURCE_NAME
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(raw, events, preset, source):
    rows = list(csv.reader(open(raw)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, units, data = rows[hi], rows[hi + 1], rows[hi + 2:]
    k = hdr.index("Kernel Name")
    t = hdr.index("gpu__time_duration.sum")
    rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    gemms = [r for r in data if "gemm_bf16_tn_kernel" in r[k]]
    ev = [r for r in csv.DictReader(open(events)) if r["class"].startswith("gemm")]
    best = max(range(len(gemms)), key=lambda i: float(gemms[i][t].replace(",", "")))
    g = gemms[best]
    dram = (float(g[rd].replace(",", "")) * SCALE[units[rd]]
            + float(g[wr].replace(",", "")) * SCALE[units[wr]])
    e = ev[best] if best < len(ev) else None
    rec = {"dram_bytes": dram,
           "algorithmic_bytes": float(e["bytes"]) if e else None,
           "launch": g[k].split("(")[0].replace("void ", "") + (f" [{e['desc']}]" if e else ""),
           "ncu_us": float(g[t].replace(",", "")) / (1000.0 if units[t] == "nsecond" else 1.0),
           "source": source}
    path = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[preset] = rec
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main(*sys.argv[1:5])
