"""Kernel-level timing of the flash attention operator (forward incl. the
keep-bit pass when dropout is on, backward = dQ kernel + dK/dV kernel) with
algorithmic TFLOP/s (forward 4*64*S^2 per (b, h), x 0.5 causal; backward 2.5x
forward) and the fraction of the measured bf16 burst peak.

python tools/bench_flash.py [--shapes 64x12x288,8x16x1024,8x16x2048] [--p 0.1] [--classes]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2209_02478_b200 import ops


def t(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="64x12x288,8x16x1024,8x16x2048")
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--causal", default="0,1")
    ap.add_argument("--classes", action="store_true")
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        peak = 2250.0
    out = []
    for shp in args.shapes.split(","):
        B, nh, S = (int(v) for v in shp.split("x"))
        for causal in (bool(int(c)) for c in args.causal.split(",")):
            qkv = torch.randn(B * S, 3 * 64 * nh, device="cuda").to(torch.bfloat16)
            f = lambda: ops.flash_attn_fwd(qkv, B, S, nh, causal=causal, dropout_p=args.p, seed=1,
                                           stream_id=2)
            us = t(f)
            fl = 4 * 64 * S * S * B * nh * (0.5 if causal else 1.0)
            ctx, lse, mask = f()
            d = torch.randn_like(ctx)
            ub = t(lambda: ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, causal=causal,
                                              dropout_p=args.p, seed=1, stream_id=2))
            row = {"B": B, "nh": nh, "S": S, "causal": causal, "p": args.p,
                   "fwd_us": us, "fwd_tflops": fl / us / 1e6, "fwd_frac": fl / us / 1e6 / peak,
                   "bwd_us": ub, "bwd_tflops": 2.5 * fl / ub / 1e6,
                   "bwd_frac": 2.5 * fl / ub / 1e6 / peak,
                   "fwd_bwd_frac": 3.5 * fl / (us + ub) / 1e6 / peak}
            if args.classes:
                import ctypes as C
                from paper_2209_02478_b200 import _lib
                lib = _lib.cuda_lib()
                lib.mimose_profile_enable(1)
                ctx, lse, mask = f()
                ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, causal=causal,
                                   dropout_p=args.p, seed=1, stream_id=2)
                torch.cuda.synchronize()
                p = C.c_void_p()
                lib.mimose_profile_csv(C.byref(p))
                text = _lib.take_string(lib, p)
                lib.mimose_profile_enable(0)
                row["kernels_us"] = {c.split(",")[0]: float(c.split(",")[-1]) * 1e3
                                     for c in text.strip().splitlines()[1:]}
            out.append(row)
            print(json.dumps(row), flush=True)
    if args.json:
        json.dump({"peak_bf16_tflops_burst": peak, "rows": out}, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
