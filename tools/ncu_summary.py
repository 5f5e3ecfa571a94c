"""Key metrics per kernel from an `ncu --page raw --csv` dump (one line per
launch): duration, DRAM bytes read / written, tensor-pipe activity, DRAM
throughput, issue activity, grid."""
import csv
import sys

WANT = [("kernel", "Kernel Name"), ("us", "gpu__time_duration.sum"),
        ("dram_rd_MB", "dram__bytes_read.sum"), ("dram_wr_MB", "dram__bytes_write.sum"),
        ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("grid", "launch__grid_size")]


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, units, data = rows[hi], rows[hi + 1], rows[hi + 2:]
    idx = [hdr.index(m) for _, m in WANT]
    print(" | ".join(k for k, _ in WANT))
    for r in data:
        out = []
        for (k, m), i in zip(WANT, idx):
            v = r[i]
            if k.endswith("_MB"):
                u = units[i]
                scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                v = f"{float(v.replace(',', '')) * scale:.1f}"
            elif k == "us":
                u = units[i]
                v = f"{float(v.replace(',', '')) / (1000.0 if u == 'nsecond' else 1.0):.2f}"
            elif k == "kernel":
                v = v.split("(")[0].replace("void ", "").replace("mimose_dev::", "")
            out.append(v)
        print(" | ".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
