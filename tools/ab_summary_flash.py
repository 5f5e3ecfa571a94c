"""Median per-kernel times of two bench_flash.py logs (A/B): python tools/ab_summary_flash.py DIR"""
import collections
import json
import statistics
import sys

out = sys.argv[1]
for V in "AB":
    agg = collections.defaultdict(list)
    for l in open(f"{out}/{V}.log"):
        try:
            d = json.loads(l)
        except Exception:
            continue
        for k, v in d.get("kernels_us", {}).items():
            agg[(d["S"], k)].append(v)
    print(V, " ".join(f"S{S}:{k.replace('attn_flash_', '')}={statistics.median(v):.1f}"
                      for (S, k), v in sorted(agg.items())))
