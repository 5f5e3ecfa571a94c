"""Per-block pipeline trace of the flash dK/dV backward kernel (CTA 0, SM
clocks). Needs the traced build (tools/trace_flash.sh builds it in a scratch
copy): python tools/flash_trace_bwd.py S..."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2209_02478_b200 import _lib, ops

lib = _lib.cuda_lib()
buf = np.zeros(4096, dtype=np.uint64)
for S in [int(a) for a in sys.argv[1:]] or [288, 1024]:
    B, nh = (64, 12) if S <= 512 else (8, 16)
    qkv = torch.randn(B * S, 3 * 64 * nh, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        ctx, lse, mask = ops.flash_attn_fwd(qkv, B, S, nh, dropout_p=0.1, seed=1, stream_id=2)
        d = torch.randn_like(ctx)
        ops.flash_attn_bwd(qkv, ctx, lse, mask, d, B, S, nh, dropout_p=0.1, seed=1, stream_id=2)
    lib.mimose_debug_flash_trace(buf.ctypes.data_as(C.c_void_p))
    b = buf.astype(np.int64)
    t0 = b[0]
    nblk = (S + 127) // 128
    print(f"== dK/dV S={S} B={B} nh={nh} (cycles from the first S/dP issue; {nblk} query blocks per item)")
    print("  blk | SdP_issue acc_start acc_issued | w0: wait_s  s_in  comp_done  pfull")
    for k in range(min(40, 256)):
        m = [b[k * 4 + i] - t0 for i in range(3)]
        e = [b[1024 + k * 4 + i] - t0 for i in range(4)]
        print(f" {k:4d} | {m[0]:9d} {m[1]:9d} {m[2]:10d} | {e[0]:9d} {e[1]:6d} {e[2]:9d} {e[3]:6d}")
    print("  item | item_start  accfull_wait  accfull_seen  drained")
    for ic in range(min(12, 40 // nblk + 1)):
        v = [b[2048 + ic * 4 + k] - t0 for k in range(4)]
        print(f"  {ic:4d} | {v[3]:10d} {v[0]:12d} {v[1]:12d} {v[2]:9d}")
