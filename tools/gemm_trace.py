"""Per-tile pipeline trace of the FFN GEMMs (CTA 0, SM clock cycles): when the
MMA warp starts / finishes issuing each tile and how long it waited for
operands, and when the epilogue warps see the accumulator and release it.
Needs the traced build:
  make clean && make NVFLAGS="$(make -s print-nvflags) -DMIMOSE_GEMM_TRACE"
(restore with make clean && make). Findings: profiles/README.md."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_02478_b200 import ops, _lib
lib = _lib.cuda_lib()
T, H, F = 18432, 768, 3072
r = lambda *s: (torch.randn(*s, device="cuda") * 0.1).to(torch.bfloat16)
X, W1, W2 = r(T, H), r(F, H), r(H, F)
U = r(T, F); dY = r(T, H)
b1 = torch.randn(F, device="cuda")
out_f = torch.empty(T, F, device="cuda", dtype=torch.bfloat16); out2 = torch.empty_like(out_f)
buf = np.zeros(1 << 15, dtype=np.uint64)
cases = {
  "gelu": lambda: ops.gemm(X, W1, out_f, epi=ops.EPI_BIAS_GELU, out2=out2, bias=b1, force_cg=1),
  "gelu_cg2": lambda: ops.gemm(X, W1, out_f, epi=ops.EPI_BIAS_GELU, out2=out2, bias=b1, force_cg=2),
  "plain16": lambda: ops.gemm(X, W1, out_f, force_ew=16, force_cg=1),
  "dgelu": lambda: ops.gemm(dY, W2, out_f, b_mn=True, epi=ops.EPI_DGELU, aux=U, force_cg=1),
}
for name, fn in cases.items():
    for _ in range(3): fn()
    lib.mimose_debug_trace(buf.ctypes.data_as(C.c_void_p), 1 << 15, 1)
    fn()
    lib.mimose_debug_trace(buf.ctypes.data_as(C.c_void_p), 1 << 15, 1)
    b = buf.astype(np.int64)
    n = 12
    t0 = b[0]
    print(f"== {name} (cycles rel. to first MMA start; per tile)")
    print(" tile  mma_start mma_issued full_wait | epi_wait_begin(min/max) tfull_seen(min/max) epi_end(min/max)")
    for i in range(n):
        ms, mi, fw = b[i*8+0]-t0, b[i*8+1]-t0, b[i*8+2]
        ew = [(b[4096+(i*16+e)*2]-t0, b[4096+(i*16+e)*2+1]-t0, b[8192+i*16+e]-t0) for e in range(16)]
        ew = [x for x in ew if x[2] > -1e12 and b[8192+i*16] != 0]
        if not ew: 
            print(i, ms, mi, fw); continue
        wb = [x[0] for x in ew]; ts = [x[1] for x in ew]; ee = [x[2] for x in ew]
        print(f" {i:3d} {ms:9d} {mi:9d} {fw:8d} | {min(wb):8d} {max(wb):8d}  {min(ts):8d} {max(ts):8d}  {min(ee):8d} {max(ee):8d}")
