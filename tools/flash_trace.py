"""Per-block pipeline trace of the flash forward (CTA 0, SM clocks). Needs the
traced build: make clean && make NVFLAGS="$(make -s print-nvflags) -DMIMOSE_FLASH_TRACE"."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2209_02478_b200 import _lib, ops

lib = _lib.cuda_lib()
buf = np.zeros(4096, dtype=np.uint64)
for S in [int(a) for a in sys.argv[1:]] or [128, 512]:
    B, nh = 64, 12
    qkv = torch.randn(B * S, 3 * 64 * nh, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        ops.flash_attn_fwd(qkv, B, S, nh, dropout_p=0.1, seed=1, stream_id=2)
    lib.mimose_debug_flash_trace(buf.ctypes.data_as(C.c_void_p))
    b = buf.astype(np.int64)
    t0 = b[0]
    nkb = (S + 127) // 128
    print(f"== S={S} (cycles from first S issue)")
    print("  jb | S_issue PV_start PV_issued | w0: wait_s  s_in  exps  pfull | w15: wait_s s_in exps pfull")
    for jb in range(min(24, 128)):
        m = [b[jb * 4 + k] - t0 for k in range(3)]
        e0 = [b[1024 + jb * 8 + k] - t0 for k in range(4)]
        e1 = [b[1024 + jb * 8 + 4 + k] - t0 for k in range(4)]
        print(f" {jb:3d} | {m[0]:7d} {m[1]:8d} {m[2]:8d} | {e0[0]:7d} {e0[1]:6d} {e0[2]:6d} {e0[3]:6d} |"
              f" {e1[0]:7d} {e1[1]:6d} {e1[2]:6d} {e1[3]:6d}")
    print("  tile | wait_o  o_seen  done")
    for tc in range(min(8, 24 // nkb + 1)):
        f = [b[2048 + tc * 4 + k] - t0 for k in range(3)]
        print(f"  {tc:4d} | {f[0]:7d} {f[1]:7d} {f[2]:7d}")
