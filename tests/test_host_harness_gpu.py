"""The compiled C++ host (tests/host/harness_gpu.cpp) runs the reference's
Mimose training loop (harness.hpp:215-296) itself, over the two C ABIs only
(include/mimose_cuda.h layer-level calls, include/mimose_planner.h fit and
planning session). It must reproduce the in-library Trainer's run on the same
inputs: the phase of every iteration (collect / sheltered / fallback /
planned), every plan, every cache hit, the fitted estimator, and every loss
bit for bit (same kernels, same Philox streams, same AdamW)."""
import os
import shutil
import struct
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

GiB = 1 << 30
SHAPE = dict(layers=4, hidden=256, heads=4, ffn=1024, vocab=512, max_pos=256, type_vocab=2,
             num_choices=4)


def _harness(tmp):
    """Build the host against the in-tree libraries (g++, no CUDA compiler)."""
    out = os.path.join(str(tmp), "harness_gpu")
    cuda = os.path.dirname(os.path.dirname(shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"))
    pkg = os.path.join(ROOT, "paper_2209_02478_b200")
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-Werror",
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"),
           os.path.join(ROOT, "tests", "host", "harness_gpu.cpp"), "-o", out,
           "-L" + pkg, "-lmimose_cuda", "-lmimose_host", "-L" + os.path.join(cuda, "lib64"),
           "-lcudart", "-Wl,-rpath," + pkg, "-Wl,-rpath," + os.path.join(cuda, "lib64")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


@pytest.mark.parametrize("unit,every_new", [(1, 0), (0, 0), (1, 1)])
def test_host_loop_reproduces_trainer(cuda_device, tmp_path, unit, every_new):
    from paper_2209_02478_b200.trainer import ModelConfig, TrainConfig, Trainer, synthetic_batch
    exe = _harness(tmp_path)
    B = 32
    m = ModelConfig(hidden_dropout=0.1, attn_dropout=0.1, seed=123, **SHAPE)
    probe = Trainer(m, TrainConfig(planner="none", batch=B, seq_min=32, seq_max=256,
                                   ckpt_unit=unit), 8 * GiB)
    rng = np.random.default_rng(2)
    peak = probe.step(*synthetic_batch(rng, B, 256, SHAPE["vocab"], 4))["peak_reserved"]
    probe.close()
    budget = int(0.55 * peak)
    t = TrainConfig(planner="mimose", batch=B, seq_min=32, seq_max=256, max_sheltered_iters=4,
                    reserve_per_size=0, ckpt_unit=unit, collect_new_sizes_always=bool(every_new),
                    lr=1e-3)
    seqs = [64, 64, 200, 256, 128, 96, 256, 200, 160, 64, 240, 128, 256, 40]
    batches = [synthetic_batch(rng, B, s, SHAPE["vocab"], 4) for s in seqs]

    tr = Trainer(m, t, budget)
    rows = [tr.step(*b) for b in batches]
    est = tr.estimator_text()
    tr.close()

    with open(tmp_path / "steps.bin", "wb") as f:
        f.write(struct.pack("<ii", len(batches), B))
        for (tok, typ, lab), s in zip(batches, seqs):
            f.write(struct.pack("<i", s))
            f.write(np.ascontiguousarray(tok, np.int32).tobytes())
            f.write(np.ascontiguousarray(typ, np.int32).tobytes())
            f.write(struct.pack("<i", lab.size))
            f.write(np.ascontiguousarray(lab, np.int32).tobytes())
    cfg = dict(SHAPE, hidden_dropout=m.hidden_dropout, attn_dropout=m.attn_dropout,
               ln_eps=m.ln_eps, init_std=m.init_std, seed=m.seed, arch=m.arch, head=m.head,
               causal=m.causal, gelu_tanh=m.gelu_tanh, pad_token_id=m.pad_token_id,
               batch=B, seq_min=t.seq_min, seq_max=t.seq_max,
               bucket_tolerance=t.bucket_tolerance, cache_tolerance=t.cache_tolerance,
               max_sheltered_iters=t.max_sheltered_iters,
               collect_new_sizes_always=int(t.collect_new_sizes_always),
               estimator_order=t.estimator_order, lr=t.lr, attn_fused=t.attn_fused,
               ckpt_unit=t.ckpt_unit, budget=budget, device=0)
    (tmp_path / "cfg.txt").write_text("".join(f"{k} {float(v)!r}\n" for k, v in cfg.items()))
    r = subprocess.run([exe, str(tmp_path / "cfg.txt"), str(tmp_path / "steps.bin")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.splitlines()
    k = lines.index("estimator")
    host_rows = [l.split() for l in lines[:k]]
    assert "\n".join(lines[k + 1:]).strip() == est.strip()
    assert len(host_rows) == len(rows)
    phases = set()
    for row, h in zip(rows, host_rows):
        it, x, phase, hit, ins, mask, bits = h
        assert int(it) == row["iter"] and int(x) == row["x"]
        assert phase == row["phase_name"], (row["iter"], phase, row["phase_name"])
        assert int(hit) == row["cache_hit"] and int(ins) == row["insufficient"]
        assert int(mask, 16) == row["dropped_mask_lo"], (row["iter"], mask, row["dropped_mask_lo"])
        assert int(bits, 16) == struct.unpack("<I", struct.pack("<f", row["loss"]))[0], \
            (row["iter"], bits, row["loss"])
        phases.add(phase)
    assert {"collect", "planned"} <= phases
    assert any(r["phase_name"] == "planned" and r["plan_size"] > 0 for r in rows)
