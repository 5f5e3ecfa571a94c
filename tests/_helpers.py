"""Shared helpers of the GPU parity tests (not a test module)."""
import numpy as np


def oracle_params(tr):
    """The trainer's parameters as the oracle consumes them: GEMM operands and
    embedding tables in bf16 (what the kernels read), biases, LayerNorm
    parameters and the classifier / QA vectors in fp32."""
    import torch
    torch.cuda.synchronize()
    p32 = tr.params().cpu().numpy()
    p16 = tr.params_bf16().float().cpu().numpy()
    out = {}
    for name, (off, n) in tr.param_table().items():
        bf16_used = (name.endswith(".weight") and ("ln" not in name)
                     and name not in ("classifier.weight", "qa.weight"))
        bf16_used = bf16_used or name.startswith("embeddings.") and "ln" not in name
        src = p16 if bf16_used else p32
        out[name] = src[off:off + n].copy()
    return out


def grads_by_name(tr):
    import torch
    torch.cuda.synchronize()
    g = tr.grads().cpu().numpy()
    return {name: g[off:off + n].copy() for name, (off, n) in tr.param_table().items()}


def check_grads(got, ref_grads, rel, floor=5e-4, min_cos=0.995):
    """Every gradient within rel * ||ref|| + floor (L2) and cosine >= min_cos.
    Returns the worst relative error seen (for the failure message / logs)."""
    worst = (0.0, None)
    import os
    log = os.environ.get("MIMOSE_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            for name, ref in ref_grads.items():
                nr = float(np.linalg.norm(ref))
                f.write(f"{name} {float(np.linalg.norm(got[name] - ref)) / max(nr, 1e-12):.4e} {nr:.4e}\n")
    for name, ref in ref_grads.items():
        g = got[name]
        nr = np.linalg.norm(ref)
        err = np.linalg.norm(g - ref)
        r = err / max(nr, 1e-12)
        if nr > 1e-3 and r > worst[0]:
            worst = (r, name)
        assert err <= rel * nr + floor, f"{name}: rel err {r:.3e} (|ref| {nr:.3e})"
        if nr > 1e-6:
            cos = float(np.dot(g, ref) / (np.linalg.norm(g) * nr + 1e-30))
            assert cos >= min_cos, f"{name}: cosine {cos}"
    return worst
