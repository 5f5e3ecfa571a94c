"""Markdown table of bench_matrix.sh lines: python tools/matrix_table.py OUT.md FILE..."""
import json
import os
import sys


def row(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    m, o, c = d["mimose"], d.get("mimose_other_basis") or {}, d["config"]
    name = os.path.basename(path)[3:-5]
    of = o.get("frac_of_no_ckpt")
    other = (f"{o['value']:.0f} ({of:.3f})" if o.get("value") else
             ("infeasible" if o.get("infeasible") else "-"))
    return (f"| {name} | {c['workload'].split(':')[0]} | {m.get('planner', 'mimose')} | "
            f"{c['seq_len']} | {c['budget_frac_of_no_ckpt_peak']:.0%} {m['basis']} | "
            f"{d['value']:.0f} | {d['e2e']['value']:.0f} | {m['no_ckpt_samples_per_s'] or 0:.0f} | "
            f"**{m['frac_of_no_ckpt'] or 0:.3f}** | {other} | {m['avg_dropped_units']:.2f} | "
            f"{m['steps_over_budget']}/{m['arena_failures']} | "
            f"{(m['mem_pred_err_max'] or 0):.4f} | {(m['planning_overhead_frac'] or 0):.1e} | "
            f"{m['cache_hits']}/{m['cache_misses']} | {d['roofline']['frac']:.3f} |")


def main(out, *files):
    lines = ["| run | workload | planner | S | budget | samples/s | e2e | no-ckpt | frac | "
             "other basis (frac) | dropped units | over budget / arena fails | pred err max | "
             "planning / step | cache hit/miss | GEMM roofline |",
             "|" + "---|" * 16]
    for f in files:
        try:
            lines.append(row(f))
        except Exception as e:  # noqa: BLE001
            lines.append(f"| {os.path.basename(f)} | failed: {e} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
