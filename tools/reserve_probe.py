"""Per-step memory accounting of a planned run: how much of the scheduler
reserve (transients outside the planned blocks) the real step actually used.
Prints one row per planned step: S, dropped blocks, arena peak, the
scheduler's predicted kept bytes (constant + kept blocks), reserve, budget."""
import argparse
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="bert-base-mc")
    ap.add_argument("--budget-frac", type=float, default=0.4)
    ap.add_argument("--steps", type=int, default=40)
    args = ap.parse_args()
    import numpy as np
    from paper_2209_02478_b200.trainer import PRESETS, PRESET_INFO, Trainer, synthetic_task_batch
    from paper_2209_02478_b200 import planner as host
    m, t = PRESETS[args.preset]
    GiB = 1 << 30
    rng = np.random.default_rng(0)
    probe = Trainer(m, dataclasses.replace(t, planner="none"), 60 * GiB)
    probe.step(*synthetic_task_batch(rng, m, t.batch, t.seq_max), optimizer=False)
    peak = probe.rows[-1]["peak_reserved"]
    probe.close()
    tr = Trainer(m, dataclasses.replace(t, planner="mimose"), int(args.budget_frac * peak))
    seqs = [int(x) for x in host.host_lib().workload(PRESET_INFO[args.preset][1], 1,
                                                      args.steps, 2024)]
    print("S,plan,peak,pred_kept,reserve,budget,slack")
    for S in seqs:
        r = tr.step(*synthetic_task_batch(rng, m, t.batch, S))
        if r["phase_name"] != "planned":
            continue
        used = r["peak_reserved"] - r["predicted_kept"]
        print(f"{S},{r['plan_size']},{r['peak_reserved']},{r['predicted_kept']},{r['reserve_bytes']},"
              f"{r['budget']},{r['budget'] - r['peak_reserved']}")
    tr.close()


if __name__ == "__main__":
    main()
