"""Times the flash attention operator against the materialised path's kernels
(fused score kernel + P V contraction) at the BERT-base shape (B = 64, 12
heads) -- kernel-level; the step-level comparison is attn_fused 3 vs 2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    B, nh = 64, 12
    for S in (128, 288, 512, 1024):
        for causal in (False, True):
            qkv = torch.randn(B * S, 3 * 64 * nh, device="cuda").to(torch.bfloat16)
            f = lambda: ops.flash_attn_fwd(qkv, B, S, nh, causal=causal, dropout_p=0.1, seed=1,
                                           stream_id=2)
            us = t(f)
            fl = 4 * 64 * S * S * B * nh * (0.5 if causal else 1.0)
            line = f"S={S:5d} causal={int(causal)} fwd {us:8.1f} us {fl / us / 1e6:7.1f} TFLOP/s"
            if "--bwd" in sys.argv:
                ctx, lse, mask = f()
                d = torch.randn_like(ctx)
                ub = t(lambda: ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, causal=causal,
                                                  dropout_p=0.1, seed=1, stream_id=2))
                line += f"  bwd {ub:8.1f} us {2.5 * fl / ub / 1e6:7.1f} TFLOP/s"
            print(line, flush=True)
            if "--classes" in sys.argv:
                import ctypes as C
                from paper_2209_02478_b200 import _lib
                lib = _lib.cuda_lib()
                lib.mimose_profile_enable(1)
                ctx, lse, mask = f()
                d = torch.randn_like(ctx)
                ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, causal=causal, dropout_p=0.1,
                                   seed=1, stream_id=2)
                torch.cuda.synchronize()
                p = C.c_void_p()
                lib.mimose_profile_csv(C.byref(p))
                text = _lib.take_string(lib, p)
                lib.mimose_profile_enable(0)
                for row in text.strip().splitlines()[1:]:
                    c = row.split(",")
                    print(f"    {c[0]:22s} {float(c[-1]) * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
