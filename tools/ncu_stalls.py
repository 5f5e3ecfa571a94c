"""Aggregate the warp-stall samples of an `ncu --page source --csv
--print-source cuda,sass` dump by stall reason and by SASS opcode (and list
the hottest instructions): python tools/ncu_stalls.py X_source.csv [top]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    lines = open(path).read().splitlines()
    hi = next(i for i, l in enumerate(lines) if l.startswith('"Line No"') or '"Address"' in l)
    hdr = next(csv.reader([lines[hi]]))
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_reason = collections.Counter()
    by_op = collections.Counter()
    hot = []
    seen = set()
    src = ""
    by_src = collections.Counter()
    for row in csv.reader(lines[hi + 1:]):
        if len(row) != len(hdr) or row[0] == "Line No":
            continue
        d = dict(zip(hdr, row))
        addr = d.get("Address", "")
        if not addr:
            # a CUDA source line (the SASS rows that follow belong to it)
            src = (row[0] + ": " + (row[1] if len(row) > 1 else "")).strip()[:90]
            continue
        if addr in seen:
            continue
        seen.add(addr)
        sass = row[3]
        try:
            n = int(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        op = sass.split()[0] if sass else "?"
        if op.startswith("@"):
            op = sass.split()[1]
        by_op[op.split(".")[0]] += n
        for r in reasons:
            try:
                by_reason[r] += int(d[r] or 0)
            except ValueError:
                pass
        by_src[src] += n
        hot.append((n, addr, sass, {r: d[r] for r in reasons if d[r] not in ("", "0")}, src))
    tot = sum(by_reason.values()) or 1
    print("samples by stall reason:")
    for r, n in by_reason.most_common():
        if n:
            print(f"  {r:24s} {n:8d} {100 * n / tot:5.1f}%")
    print("samples by opcode:")
    for o, n in by_op.most_common(top):
        print(f"  {o:12s} {n:8d} {100 * n / tot:5.1f}%")
    print("hottest source lines:")
    for s, n in by_src.most_common(top):
        print(f"  {n:7d} {100 * n / tot:5.1f}%  {s}")
    print("hottest instructions:")
    for n, a, s, r, src in sorted(hot, reverse=True)[:top]:
        print(f"  {n:7d} {a} {s[:60]:60s} {r}  <- {src[:60]}")


if __name__ == "__main__":
    main()
