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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="bert-base-mc")
    ap.add_argument("--budget-frac", type=float, default=0.4)
    ap.add_argument("--seq", type=int, default=288)
    ap.add_argument("--planner", default="mimose")
    ap.add_argument("--gemm-csv", default="")
    ap.add_argument("--attn-fused", action="store_true")
    ap.add_argument("--time-steps", type=int, default=0, help="also time N steps at --seq")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2209_02478_b200 import _lib
    from paper_2209_02478_b200.trainer import PRESETS, DeviceBatch, Trainer, synthetic_batch
    m, t = PRESETS[args.preset]
    GiB = 1 << 30
    rng = np.random.default_rng(0)
    probe = Trainer(m, dataclasses.replace(t, planner="none"), 60 * GiB)
    probe.step(*synthetic_batch(rng, t.batch, t.seq_max, m.vocab, m.num_choices), optimizer=False)
    peak = probe.rows[-1]["peak_reserved"]
    probe.close()
    budget = int(args.budget_frac * peak) if args.planner == "mimose" else int(1.2 * peak)
    tr = Trainer(m, dataclasses.replace(t, planner=args.planner, attn_fused=args.attn_fused),
                 budget)
    for s in [64, 512, 200, 350, 128, 480, 300, 96, 420, 256, 160, 384]:
        tr.step(*synthetic_batch(rng, t.batch, s, m.vocab, m.num_choices))
    db = DeviceBatch.from_host(*synthetic_batch(rng, t.batch, args.seq, m.vocab, m.num_choices),
                               m.vocab)
    tr.step_device(db)  # warm
    torch.cuda.synchronize()
    lib = _lib.cuda_lib()
    if args.gemm_csv:
        lib.mimose_gemm_profile_enable(1)
    torch.cuda.nvtx.range_push("timed_step")
    r = tr.step_device(db)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print({k: r[k] for k in ("seq", "phase_name", "plan_size", "peak_reserved")})
    if args.time_steps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.time_steps):
            tr.step_device(db)
        e1.record()
        torch.cuda.synchronize()
        print(f"seq {args.seq} attn_fused={args.attn_fused}: "
              f"{e0.elapsed_time(e1) / args.time_steps:.3f} ms/step (plan_size {r['plan_size']})")
    if args.gemm_csv:
        p = C.c_void_p()
        lib.mimose_gemm_profile_csv(C.byref(p))
        text = _lib.take_string(lib, p)
        lib.mimose_gemm_profile_enable(0)
        with open(args.gemm_csv, "w") as f:
            f.write(text)
        rows = [l.split(",") for l in text.strip().splitlines()[1:]]
        agg = {}
        for row in rows:
            key = tuple(row[:9])
            a = agg.setdefault(key, [0, 0.0])
            a[0] += 1
            a[1] += float(row[9])
        tot = sum(v[1] for v in agg.values())
        print(f"GEMM total {tot:.3f} ms over {len(rows)} launches")
        for key, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
            M, N, K, b = map(int, key[:4])
            tf = 2.0 * M * N * K * b * n / (ms * 1e-3) / 1e12
            print(f"{ms:8.3f} ms  x{n:3d}  M={M:6d} N={N:5d} K={K:6d} batch={b:4d} bn={key[4]} "
                  f"amn={key[5]} bmn={key[6]} epi={key[7]} grid={key[8]}  {tf:7.1f} TFLOP/s")
    tr.close()


if __name__ == "__main__":
    main()
