import sys, torch
sys.path.insert(0, '.')
from paper_2209_02478_b200 import ops
sys.path.insert(0, 'tests')
import test_flash_gpu as T
for S in [64, 200, 256, 288, 320, 384, 512]:
    B, nh = 2, 3
    g = torch.Generator(device="cpu").manual_seed(S * 11)
    qkv = (torch.randn(B * S, 3 * 64 * nh, generator=g) * 1.5).to(torch.bfloat16).cuda()
    dctx = torch.randn(B * S, 64 * nh, generator=g).to(torch.bfloat16).cuda()
    ctx, lse, mask = ops.flash_attn_fwd(qkv, B, S, nh, causal=False, dropout_p=0.0, seed=99, stream_id=5)
    dqkv = ops.flash_attn_bwd(qkv, ctx, lse, mask, dctx, B, S, nh, causal=False, dropout_p=0.0, seed=99, stream_id=5)
    torch.cuda.synchronize()
    ref = T._ref_grads(qkv, dctx, B, S, nh, False, 0.0, 99, 5)
    dq = dqkv[:, :64*nh].float(); rq = ref[:, :64*nh]
    bad = ~torch.isfinite(dq)
    err = (dq - rq).abs()
    err[bad] = 1e9
    rows = (err.max(dim=1).values > 0.05 * rq.abs().max()).nonzero().flatten().tolist()
    print(S, "nan", int(bad.sum()), "badrows", len(rows), rows[:10], rows[-5:] if rows else None,
          "cols", (err.max(dim=0).values > 0.05 * rq.abs().max()).nonzero().flatten().tolist()[:12])
