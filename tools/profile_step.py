"""One steady-state planned training step under the bench's budget, for ncu
and for the per-GEMM breakdown. The profiled step is wrapped in an NVTX range
'timed_step' (ncu --nvtx --nvtx-include 'timed_step/')."""
import argparse
import ctypes as C
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def summarize(text, top=30):
    """Per-(class, shape) aggregate of the profiler CSV: ms, share, TFLOP/s
    (GEMMs) or algorithmic GB/s (memory-bound stages)."""
    import csv
    import io
    rows = list(csv.DictReader(io.StringIO(text)))
    agg = {}
    for r in rows:
        key = (r["class"], r["desc"])
        a = agg.setdefault(key, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += float(r["ms"])
        a[2] += float(r["flops"])
        a[3] += float(r["bytes"])
    tot = sum(v[1] for v in agg.values())
    out = [f"instrumented total {tot:.3f} ms over {len(rows)} launches"]
    cls = {}
    for (c, _), (n, ms, fl, by) in agg.items():
        x = cls.setdefault(c, [0, 0.0, 0.0, 0.0])
        x[0] += n; x[1] += ms; x[2] += fl; x[3] += by
    for c, (n, ms, fl, by) in sorted(cls.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{ms:8.3f} ms {100 * ms / tot:5.1f}%  x{n:4d}  {c:18s} "
                   f"{fl / (ms * 1e-3) / 1e12:7.1f} TFLOP/s  {by / (ms * 1e-3) / 1e9:7.0f} GB/s")
    out.append("-- per shape --")
    for (c, d), (n, ms, fl, by) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        out.append(f"{ms:8.3f} ms  x{n:3d}  {c:18s} {d:48s} "
                   f"{fl / (ms * 1e-3) / 1e12:7.1f} TFLOP/s  {by / (ms * 1e-3) / 1e9:7.0f} GB/s")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="bert-base-mc")
    ap.add_argument("--budget-frac", type=float, default=0.4)
    ap.add_argument("--seq", type=int, default=288)
    ap.add_argument("--planner", default="mimose")
    ap.add_argument("--gemm-csv", default="")
    ap.add_argument("--attn-fused", action="store_true", help="(default) fused score kernels")
    ap.add_argument("--attn-unfused", action="store_true", help="GEMM + softmax kernel pair")
    ap.add_argument("--attn-mode", type=int, default=3,
                    help="TrainConfig.attn_fused when fused: 3 flash, 2 single-row fused scores")
    ap.add_argument("--time-steps", type=int, default=0, help="also time N steps at --seq")
    ap.add_argument("--hidden-dropout", type=float, default=None,
                    help="override the preset's hidden dropout (A/B of the Philox stages)")
    ap.add_argument("--attn-dropout", type=float, default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2209_02478_b200 import _lib
    from paper_2209_02478_b200.trainer import PRESETS, DeviceBatch, Trainer, synthetic_task_batch
    m, t = PRESETS[args.preset]
    if args.hidden_dropout is not None:
        m = dataclasses.replace(m, hidden_dropout=args.hidden_dropout)
    if args.attn_dropout is not None:
        m = dataclasses.replace(m, attn_dropout=args.attn_dropout)
    GiB = 1 << 30
    rng = np.random.default_rng(0)
    # budget basis: the materialised-attention model's no-ckpt peak (as bench.py)
    probe = Trainer(m, dataclasses.replace(t, planner="none", attn_fused=2), 60 * GiB)
    probe.step(*synthetic_task_batch(rng, m, t.batch, t.seq_max), optimizer=False)
    peak = probe.rows[-1]["peak_reserved"]
    probe.close()
    budget = int(args.budget_frac * peak) if args.planner == "mimose" else int(1.2 * peak)
    fused = 0 if args.attn_unfused else args.attn_mode
    tr = Trainer(m, dataclasses.replace(t, planner=args.planner, attn_fused=fused),
                 budget)
    lo, hi = t.seq_min, t.seq_max
    for f in [0.0, 1.0, 0.3, 0.6, 0.15, 0.9, 0.5, 0.05, 0.8, 0.4, 0.2, 0.7]:
        tr.step(*synthetic_task_batch(rng, m, t.batch, int(lo + f * (hi - lo)) // 8 * 8 or 8))
    db = DeviceBatch.from_host(*synthetic_task_batch(rng, m, t.batch, args.seq), m.vocab)
    tr.step_device(db)  # warm
    torch.cuda.synchronize()
    lib = _lib.cuda_lib()
    if args.gemm_csv:
        lib.mimose_profile_enable(1)
    torch.cuda.nvtx.range_push("timed_step")
    r = tr.step_device(db)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print({k: r[k] for k in ("seq", "phase_name", "plan_size", "peak_reserved")})
    if args.gemm_csv:
        p = C.c_void_p()
        lib.mimose_profile_csv(C.byref(p))
        text = _lib.take_string(lib, p)
        lib.mimose_profile_enable(0)
        with open(args.gemm_csv, "w") as f:
            f.write(text)
        print(summarize(text))
    if args.time_steps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.time_steps):
            tr.step_device(db)
        e1.record()
        torch.cuda.synchronize()
        print(f"seq {args.seq} attn_fused={fused}: "
              f"{e0.elapsed_time(e1) / args.time_steps:.3f} ms/step (plan_size {r['plan_size']})")
    tr.close()


if __name__ == "__main__":
    main()
