"""Instructions executed and stall samples per CUDA source line from an
`ncu --page source --csv --print-source cuda,sass` dump:
python tools/ncu_lines.py X_source.csv [top]"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    lines = open(path).read().splitlines()
    hi = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    hdr = next(csv.reader([lines[hi]]))
    rows = []
    for row in csv.reader(lines[hi + 1:]):
        if len(row) != len(hdr) or row[2] != "-":
            continue
        d = dict(zip(hdr, row))
        try:
            n = int(d["Instructions Executed"] or 0)
            smp = int(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        rows.append((n, smp, row[0], row[1].strip()[:100]))
    tot = sum(r[0] for r in rows) or 1
    tots = sum(r[1] for r in rows) or 1
    print(f"total {tot} warp instructions, {tots} stall samples")
    for n, smp, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{n:10d} {100 * n / tot:5.1f}%  samples {100 * smp / tots:5.1f}%  L{ln}: {src}")


if __name__ == "__main__":
    main()
