"""Small launches of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): tcgen05 GEMMs (each epilogue, 1-SM and
CTA-pair tiles, K- and MN-major operands, split-K), flash attention forward +
backward (dropout on / off, causal / not, several items per CTA), and one
tiny training step with every unit dropped (recompute path, LN / softmax /
embedding / head / AdamW kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2209_02478_b200 import ops
from paper_2209_02478_b200.trainer import ModelConfig, TrainConfig, Trainer, synthetic_batch


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.manual_seed(0)
    if which in ("all", "gemm"):
        for (M, N, K) in [(256, 256, 128), (200, 72, 80)]:
            for bn in (128, 256):
                for cg in (1, 2):
                    if cg == 2 and (bn != 256 or M <= 128):
                        continue
                    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
                    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
                    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                    ops.gemm(A, B, out, force_bn=bn, force_cg=cg)
                    o2 = torch.empty_like(out)
                    bias = torch.randn(N, device="cuda")
                    ops.gemm(A, B, out, epi=ops.EPI_BIAS_GELU, out2=o2, bias=bias, force_bn=bn,
                             force_cg=cg)
                    ops.gemm(A, B, o2, epi=ops.EPI_DGELU, aux=out, force_bn=bn, force_cg=cg)
                    f = torch.zeros(M, N, device="cuda")
                    ops.gemm(A.t().contiguous(), B, f, a_mn=True, epi=ops.EPI_F32, force_bn=bn,
                             force_cg=cg)
        torch.cuda.synchronize()
        print("gemm ok", flush=True)
    if which in ("all", "flash"):
        for S, B, nh in [(200, 2, 2), (64, 12, 4)]:
            for p in (0.0, 0.1):
                for causal in (False, True):
                    qkv = torch.randn(B * S, 3 * 64 * nh, device="cuda").to(torch.bfloat16)
                    ctx, lse, mask = ops.flash_attn_fwd(qkv, B, S, nh, causal=causal, dropout_p=p,
                                                        seed=1, stream_id=2)
                    d = torch.randn_like(ctx)
                    ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, causal=causal,
                                       dropout_p=p, seed=1, stream_id=2)
        torch.cuda.synchronize()
        print("flash ok", flush=True)
    if which in ("all", "step"):
        m = ModelConfig(layers=2, hidden=256, heads=4, ffn=1024, vocab=512, max_pos=128,
                        hidden_dropout=0.1, attn_dropout=0.1)
        tr = Trainer(m, TrainConfig(planner="none", batch=8, seq_min=16, seq_max=96), 1 << 30)
        tr.force_plan([0, 1, 2, 3])
        tr.step(*synthetic_batch(np.random.default_rng(0), 8, 40, 512, 4))
        tr.close()
        torch.cuda.synchronize()
        print("step ok", flush=True)


if __name__ == "__main__":
    main()
