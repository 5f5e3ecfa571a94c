"""Times individual GEMM shapes / epilogues of the training step with CUDA events
(kernel-level roofline check; not the headline bench)."""
import sys, os
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
    return e0.elapsed_time(e1) / reps


def main():
    T, H, F = 18432, 768, 3072
    r = lambda *s: (torch.randn(*s, device="cuda") * 0.1).to(torch.bfloat16)
    X, W1, W2 = r(T, H), r(F, H), r(H, F)
    G, U = r(T, F), r(T, F)
    b1, b2 = torch.randn(F, device="cuda"), torch.randn(H, device="cuda")
    out_f = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
    out2 = torch.empty_like(out_f)
    out_h = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    dY = r(T, H)
    cases = {
        "ffn1 bias+gelu  [T,H]x[F,H]^T": (lambda: ops.gemm(X, W1, out_f, epi=ops.EPI_BIAS_GELU, out2=out2, bias=b1), 2 * T * F * H),
        "ffn1 bias only  [T,H]x[F,H]^T": (lambda: ops.gemm(X, W1, out_f, bias=b1), 2 * T * F * H),
        "ffn1 plain      [T,H]x[F,H]^T": (lambda: ops.gemm(X, W1, out_f), 2 * T * F * H),
        "ffn2 fwd        [T,F]x[H,F]^T": (lambda: ops.gemm(G, W2, out_h, bias=b2), 2 * T * F * H),
        "ffn2 dgrad dGELU[T,H]x[H,F]":   (lambda: ops.gemm(dY, W2, out_f, b_mn=True, epi=ops.EPI_DGELU, aux=U), 2 * T * F * H),
    }
    for name, (fn, fl) in cases.items():
        ms = t(fn)
        print(f"{name}: {ms*1e3:8.1f} us  {fl / ms / 1e9:8.1f} TFLOP/s")
    if "--splitk" in sys.argv:
        # weight-gradient shapes (fp32 out, K = tokens) against the split-K factor
        ws = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
        for (m, n) in ((2304, 768), (768, 3072), (3072, 768), (768, 768)):
            dO, Xin = r(T, m), r(T, n)
            o = torch.empty(m, n, device="cuda", dtype=torch.float32)
            line = []
            for sk in (0, 1, 2, 3, 4, 5, 6, 8):
                ms = t(lambda: ops.gemm(dO, Xin, o, a_mn=True, b_mn=True, epi=ops.EPI_F32,
                                        workspace=ws, split_k=sk))
                line.append(f"s{sk}:{ms*1e3:6.1f}")
            print(f"wgrad {m}x{n}x{T}: " + "  ".join(line) + "  (us; s0 = cost model)")
    if "--direct" in sys.argv:
        # epilogue output path: smem staging + TMA store (default) vs per-thread
        # global stores (no staging traffic in shared memory)
        for name, mk in (
                ("ffn1 gelu", lambda d: ops.gemm(X, W1, out_f, epi=ops.EPI_BIAS_GELU, out2=out2,
                                                 bias=b1, direct_store=d)),
                ("ffn1 plain", lambda d: ops.gemm(X, W1, out_f, direct_store=d)),
                ("dgelu", lambda d: ops.gemm(dY, W2, out_f, b_mn=True, epi=ops.EPI_DGELU, aux=U,
                                             direct_store=d))):
            for d in (False, True):
                ms = t(lambda: mk(d))
                print(f"{name:10s} direct={int(d)}: {ms*1e3:8.1f} us  "
                      f"{2 * T * F * H / ms / 1e9:8.1f} TFLOP/s")
    if "--variants" in sys.argv:
        # epilogue-warp count x CTA pairing for the epilogue-heavy shapes
        for cg in (1, 2):
            for ew in (8, 16):
                for name, fn in (
                        ("ffn1 gelu", lambda: ops.gemm(X, W1, out_f, epi=ops.EPI_BIAS_GELU, out2=out2,
                                                       bias=b1, force_ew=ew, force_cg=cg)),
                        ("ffn1 plain", lambda: ops.gemm(X, W1, out_f, force_ew=ew, force_cg=cg)),
                        ("dgelu", lambda: ops.gemm(dY, W2, out_f, b_mn=True, epi=ops.EPI_DGELU,
                                                   aux=U, force_ew=ew, force_cg=cg))):
                    try:
                        ms = t(fn)
                    except Exception as e:  # configuration not instantiated
                        print(f"{name:10s} cg{cg} ew{ew}: n/a ({e})")
                        continue
                    print(f"{name:10s} cg{cg} ew{ew}: {ms*1e3:8.1f} us  "
                          f"{2 * T * F * H / ms / 1e9:8.1f} TFLOP/s")


if __name__ == "__main__":
    main()
