"""Per-sequence-length cost of checkpointing under a budget: for S on a grid,
the planned step (Mimose trainer after its calibration window) against the
no-checkpoint step, with the plan it ran (attention / FFN units dropped),
its measured peak and the reserve it was planned with. Budget = frac x the
measured configuration's own no-checkpoint peak at S_max (bench.py
--budget-basis self) unless --basis materialised.

python tools/budget_sweep.py --preset bert-base-mc --frac 0.4 [--unit 0|1]
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="bert-base-mc")
    ap.add_argument("--frac", type=float, default=0.4)
    ap.add_argument("--basis", default="self", choices=["self", "materialised"])
    ap.add_argument("--unit", type=int, default=1)
    ap.add_argument("--grid", default="64,128,192,256,320,384,448,512")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2209_02478_b200.trainer import PRESETS, DeviceBatch, Trainer, synthetic_task_batch
    m, t = PRESETS[args.preset]
    t = dataclasses.replace(t, ckpt_unit=args.unit)
    GiB = 1 << 30
    rng = np.random.default_rng(0)
    probe_t = dataclasses.replace(t, planner="none")
    if args.basis == "materialised":
        probe_t = dataclasses.replace(probe_t, attn_fused=2)
    probe = Trainer(m, probe_t, 100 * GiB)
    probe.step(*synthetic_task_batch(rng, m, t.batch, t.seq_max), optimizer=False)
    peak = probe.rows[-1]["peak_reserved"]
    probe.close()
    budget = int(args.frac * peak)
    tr = Trainer(m, dataclasses.replace(t, planner="mimose"), budget)
    base = Trainer(m, dataclasses.replace(t, planner="none"), int(1.3 * peak) + GiB)
    lo, hi = t.seq_min, t.seq_max
    for f in [0.0, 1.0, 0.3, 0.6, 0.15, 0.9, 0.5, 0.05, 0.8, 0.4, 0.2, 0.7]:
        tr.step(*synthetic_task_batch(rng, m, t.batch, int(lo + f * (hi - lo))))
    out = []
    for S in [int(s) for s in args.grid.split(",")]:
        db = DeviceBatch.from_host(*synthetic_task_batch(rng, m, t.batch, S), m.vocab)
        res = {}
        for name, x in (("mimose", tr), ("none", base)):
            x.step_device(db)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                r = x.step_device(db)
            e1.record()
            torch.cuda.synchronize()
            res[name] = (e0.elapsed_time(e1) / args.reps, r)
        ms, r = res["mimose"]
        ms0, _ = res["none"]
        units = r["dropped"]
        row = {"S": S, "ms": round(ms, 3), "ms_none": round(ms0, 3), "ratio": round(ms0 / ms, 4),
               "dropped": len(units),
               "attn_dropped": sum(1 for u in units if args.unit == 1 and u % 2 == 0),
               "ffn_dropped": sum(1 for u in units if args.unit == 1 and u % 2 == 1),
               "peak_frac": round(r["peak_reserved"] / budget, 4),
               "reserve_mb": round(r["reserve_bytes"] / 2**20, 1)}
        out.append(row)
        print(json.dumps(row), flush=True)
    summary = {"preset": args.preset, "frac": args.frac, "basis": args.basis, "unit": args.unit,
               "budget": budget, "peak_none": peak, "constant": tr.info()["constant_bytes"],
               "rows": out}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(summary, f, indent=1)
    tr.close()
    base.close()


if __name__ == "__main__":
    main()
