"""Pins the CPU numerics oracle (oracle/bert_ref.py) before it is trusted.

* Philox4x32-10 restatement == the published Random123 known-answer vectors
  (the kernels' dropout RNG; the GPU side is checked against this oracle in
  tests/test_trainer_gpu.py with dropout on);
* dropout keep-rate and scale;
* the oracle's autograd gradients agree with central finite differences in
  float64 on a tiny model (the oracle differentiates what it claims to);
* bf16 rounding helper == torch's bf16 cast.
"""
import numpy as np
import pytest
import torch

from oracle import bert_ref


def test_philox_known_answers():
    # Random123 philox4x32_10 KAT (kat_vectors): (ctr, key) -> out
    cases = [
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for ctr, key, want in cases:
        group = ctr[0] | (ctr[1] << 32)
        stream = ctr[2] | (ctr[3] << 32)
        seed = key[0] | (key[1] << 32)
        got = bert_ref.philox4x32_10(seed, stream, np.array([group], dtype=np.uint64))[0]
        assert tuple(int(v) for v in got) == want


def test_dropout_mask_rate():
    idx = np.arange(1 << 18, dtype=np.uint64)
    m = bert_ref.keep_mask(0.1, 1234, bert_ref.stream_id(3, 5, 1), idx)
    assert abs(m.mean() - 0.9) < 0.005
    m2 = bert_ref.keep_mask(0.1, 1234, bert_ref.stream_id(3, 5, 1), idx)
    assert np.array_equal(m, m2)
    m3 = bert_ref.keep_mask(0.1, 1234, bert_ref.stream_id(4, 5, 1), idx)
    assert not np.array_equal(m, m3)


class _Cfg:
    layers, hidden, heads, ffn, vocab, max_pos, type_vocab = 1, 128, 2, 64, 20, 16, 2
    num_choices, hidden_dropout, attn_dropout, ln_eps, seed = 2, 0.0, 0.0, 1e-5, 3
    arch, head, causal, gelu_tanh = 0, 0, 0, 0


def _labels(cfg, rng, B, S):
    if cfg.head == 0:
        return rng.integers(0, cfg.num_choices, size=B // cfg.num_choices).astype(np.int32)
    if cfg.head == 1:
        return rng.integers(0, S, size=2 * B).astype(np.int32)
    lab = rng.integers(0, cfg.vocab, size=B * S).astype(np.int32)
    lab[rng.random(B * S) < (0.2 if cfg.head == 2 else 0.7)] = -1
    return lab


VARIANTS = {
    "bert-mc": dict(),
    "bert-qa": dict(head=1),
    "bert-mlm": dict(head=3),
    "gpt2-lm": dict(arch=1, head=2, causal=1, gelu_tanh=1, type_vocab=0),
}
CHECK = {
    "bert-mc": ["layer.0.attn.qkv.weight", "layer.0.ffn.in.bias", "pooler.weight",
                "embeddings.ln.weight", "classifier.bias"],
    "bert-qa": ["layer.0.attn.out.weight", "qa.weight", "qa.bias", "embeddings.token_type"],
    "bert-mlm": ["mlm.transform.weight", "mlm.ln.weight", "mlm.decoder.bias", "embeddings.word"],
    "gpt2-lm": ["layer.0.attn.qkv.weight", "layer.0.ffn.out.weight", "final_ln.weight",
                "embeddings.word", "embeddings.position"],
}


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_oracle_gradients_match_finite_differences(variant):
    cfg = _Cfg()
    for k, v in VARIANTS[variant].items():
        setattr(cfg, k, v)
    rng = np.random.default_rng(0)
    shapes = bert_ref.param_shapes(cfg)
    params = {k: rng.standard_normal(int(np.prod(s))) * (0.5 if "ln.weight" not in k else 0.1)
              + (1.0 if "ln.weight" in k else 0.0) for k, s in shapes.items()}
    tok = rng.integers(0, cfg.vocab, size=(4, 6)).astype(np.int32)
    typ = (rng.random((4, 6)) > 0.5).astype(np.int32)
    lab = _labels(cfg, rng, 4, 6)
    loss, _, grads = bert_ref.loss_and_grads(params, tok, typ, lab, cfg, dtype=torch.float64)
    for name in CHECK[variant]:
        for j in rng.choice(params[name].size, size=min(3, params[name].size), replace=False):
            p2 = {k: v.copy() for k, v in params.items()}
            h = 1e-6
            p2[name][j] += h
            lp, _, _ = bert_ref.loss_and_grads(p2, tok, typ, lab, cfg, dtype=torch.float64)
            p2[name][j] -= 2 * h
            lm, _, _ = bert_ref.loss_and_grads(p2, tok, typ, lab, cfg, dtype=torch.float64)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grads[name][j]) <= 1e-6 + 1e-4 * abs(fd), (name, j, fd, grads[name][j])


def test_bf16_round_matches_torch():
    x = np.random.default_rng(1).standard_normal(10000).astype(np.float32) * 37
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(bert_ref.numpy_bf16_round(x), want)
