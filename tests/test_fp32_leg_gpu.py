"""The fp32 leg of the north-star tolerance statement ("loss and gradients
match the CPU reference within a stated fp32 and bf16 tolerance").

The training step runs bf16 activations / GEMM operands (the bf16 leg,
tests/test_trainer_gpu.py, tests/test_parity_baseline_shapes_gpu.py); what
the step keeps in fp32 is held to fp32 tolerances here and in
tests/test_gemm_gpu.py (_check_f32: fp32-output GEMMs, the weight gradients,
within 1e-4 * rms * sqrt(K / 64) of the fp32 contraction of the same bf16
operands):

* the optimizer: fp32 master weights, global gradient-norm clipping and
  AdamW (decoupled decay, bias corrections) against torch.optim.AdamW +
  torch.nn.utils.clip_grad_norm_ (the optimizer of the paper's HF Trainer
  runs) in float64 -- within 4 fp32 ulps of each weight plus
  1e-5 of the learning rate, over steps with and without clipping;
* the bf16 GEMM copy is exactly the round-to-nearest bf16 of the fp32 master.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TINY = dict(layers=2, hidden=256, heads=4, ffn=1024, vocab=512, max_pos=128, type_vocab=2,
            num_choices=4)


def _decayed(name):
    return not (name.endswith("bias") or ".ln." in name or name.startswith("final_ln")
                or name.endswith("ln.weight"))


def test_adamw_clipping_fp32_leg(cuda_device):
    from paper_2209_02478_b200.trainer import ModelConfig, TrainConfig, Trainer
    lr, wd, clip = 1e-3, 0.01, 1.0
    m = ModelConfig(seed=5, **TINY)
    t = TrainConfig(planner="none", batch=8, seq_min=16, seq_max=64, lr=lr, weight_decay=wd,
                    max_grad_norm=clip)
    tr = Trainer(m, t, 2 << 30)
    try:
        table = tr.param_table()
        torch.cuda.synchronize()
        p0 = tr.params().cpu().double()
        params = {k: torch.nn.Parameter(p0[off:off + n].clone()) for k, (off, n) in table.items()}
        groups = [{"params": [p for k, p in params.items() if _decayed(k)], "weight_decay": wd},
                  {"params": [p for k, p in params.items() if not _decayed(k)],
                   "weight_decay": 0.0}]
        opt = torch.optim.AdamW(groups, lr=lr, betas=(t.beta1, t.beta2), eps=t.adam_eps)
        gen = torch.Generator().manual_seed(11)
        n_all = tr.params().numel()
        # grad scales: clipping active (norm >> 1), inactive (norm << 1), active
        for step, scale in enumerate([3e-2, 1e-5, 1e-1]):
            g = torch.zeros(n_all, dtype=torch.float32)
            for k, (off, n) in table.items():
                g[off:off + n] = torch.randn(n, generator=gen) * scale
            tr.grads().copy_(g.to(cuda_device))
            tr.optimizer_step(1.0)
            for k, (off, n) in table.items():
                params[k].grad = g[off:off + n].double().clone()
            norm = torch.nn.utils.clip_grad_norm_(list(params.values()), clip)
            assert (norm.item() > clip) == (step != 1)
            opt.step()
            torch.cuda.synchronize()
            p32 = tr.params().cpu()
            for k, (off, n) in table.items():
                got = p32[off:off + n].double()
                ref = params[k].detach()
                ulp = torch.from_numpy(np.spacing(ref.float().abs().numpy())).double()
                err = (got - ref).abs()
                bound = 4 * ulp + 1e-5 * lr
                assert torch.all(err <= bound), (step, k, err.max().item(),
                                                 (err / bound).max().item())
        # the bf16 operand copy is the RN bf16 of the fp32 master, bit for bit
        p16 = tr.params_bf16().cpu()
        assert torch.equal(p16, tr.params().cpu().to(torch.bfloat16))
    finally:
        tr.close()
