"""One flash-attention forward + backward at a given shape (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2209_02478_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="64x12x288")
ap.add_argument("--p", type=float, default=0.1)
ap.add_argument("--causal", type=int, default=0)
a = ap.parse_args()
B, nh, S = (int(v) for v in a.shape.split("x"))
qkv = torch.randn(B * S, 3 * 64 * nh, device="cuda").to(torch.bfloat16)
for _ in range(2):
    ctx, lse, mask = ops.flash_attn_fwd(qkv, B, S, nh, causal=bool(a.causal), dropout_p=a.p,
                                        seed=1, stream_id=2)
    d = torch.randn_like(ctx)
    ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, causal=bool(a.causal), dropout_p=a.p,
                       seed=1, stream_id=2)
torch.cuda.synchronize()
print("ok")
