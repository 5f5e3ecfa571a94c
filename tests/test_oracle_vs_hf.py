"""Pins the numerics oracle (oracle/bert_ref.py) to the third-party
implementation the paper trained with.

The reference repository has no tensor code; the paper's training math is
HuggingFace transformers 4.18 on PyTorch 1.11 (reference PAPER.md:390,
PAPER.md:419-421). transformers 5.5.0 is what this image ships (same BERT /
GPT-2 module math: post-LN BertLayer with exact-erf GELU, pre-LN GPT2Block
with gelu_new, tied decoders). For each task head the GPU path implements we
load IDENTICAL weights into

    BertForMultipleChoice     (configs[1], multiple choice)
    BertForQuestionAnswering  (configs[2], extractive QA)
    BertForMaskedLM           (configs[4], MLM)
    GPT2LMHeadModel           (configs[3], causal LM)

run one forward + backward in float64 with dropout 0 and eager attention,
and require the oracle's loss and EVERY parameter gradient to agree to
~1e-9 relative. The oracle's fused-QKV / tied-decoder parameterisation is
mapped onto HF's separate query/key/value Linear (BERT) and transposed
Conv1D (GPT-2) tensors by `_to_hf` below.
"""
import numpy as np
import pytest
import torch

from oracle import bert_ref

transformers = pytest.importorskip("transformers")

H, NH, F, V, P, L = 64, 4, 128, 97, 40, 2


class _Cfg:
    layers, hidden, heads, ffn, vocab, max_pos, type_vocab = L, H, NH, F, V, P, 2
    num_choices, hidden_dropout, attn_dropout, ln_eps, seed = 4, 0.0, 0.0, 1e-12, 3
    arch, head, causal, gelu_tanh, init_std = 0, 0, 0, 0, 0.02
    pad_token_id = 0  # BertConfig.pad_token_id: the word embedding's padding_idx


VARIANTS = {
    "mc": dict(),
    "qa": dict(head=1),
    "mlm": dict(head=3),
    "gpt2-lm": dict(arch=1, head=2, causal=1, gelu_tanh=1, type_vocab=0, ln_eps=1e-5,
                    pad_token_id=-1),
}


def _cfg(variant):
    c = _Cfg()
    for k, v in VARIANTS[variant].items():
        setattr(c, k, v)
    return c


def _params(cfg, rng):
    # LayerNorm weights away from 1 and non-zero biases so a swapped or
    # dropped tensor cannot hide
    out = {}
    for k, s in bert_ref.param_shapes(cfg).items():
        n = int(np.prod(s))
        if k.endswith("ln.weight"):
            out[k] = 1.0 + 0.2 * rng.standard_normal(n)
        elif k.endswith("bias"):
            out[k] = 0.05 * rng.standard_normal(n)
        else:
            out[k] = 0.08 * rng.standard_normal(n)
    return out


def _hf_model(cfg):
    if cfg.arch == 1:
        hc = transformers.GPT2Config(vocab_size=V, n_positions=P, n_embd=H, n_layer=L, n_head=NH,
                                     n_inner=F, activation_function="gelu_new",
                                     resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0,
                                     layer_norm_epsilon=cfg.ln_eps)
        hc._attn_implementation = "eager"
        return transformers.GPT2LMHeadModel(hc)
    hc = transformers.BertConfig(vocab_size=V, hidden_size=H, num_hidden_layers=L,
                                 num_attention_heads=NH, intermediate_size=F,
                                 max_position_embeddings=P, type_vocab_size=cfg.type_vocab,
                                 hidden_act="gelu", hidden_dropout_prob=0.0,
                                 attention_probs_dropout_prob=0.0, layer_norm_eps=cfg.ln_eps)
    hc._attn_implementation = "eager"
    cls = {0: transformers.BertForMultipleChoice, 1: transformers.BertForQuestionAnswering,
           3: transformers.BertForMaskedLM}[cfg.head]
    return cls(hc)


def _to_hf(cfg, p):
    """oracle parameter name -> [(hf name, transform(oracle tensor) -> hf tensor)]."""
    t = {k: torch.tensor(v, dtype=torch.float64).reshape(s)
         for (k, s), v in zip(bert_ref.param_shapes(cfg).items(),
                              (p[k] for k in bert_ref.param_shapes(cfg)))}
    m = {}
    if cfg.arch == 1:
        m["transformer.wte.weight"] = t["embeddings.word"]
        m["transformer.wpe.weight"] = t["embeddings.position"]
        m["transformer.ln_f.weight"] = t["final_ln.weight"]
        m["transformer.ln_f.bias"] = t["final_ln.bias"]
        for l in range(L):
            a, h = f"layer.{l}.", f"transformer.h.{l}."
            m[h + "ln_1.weight"], m[h + "ln_1.bias"] = t[a + "attn.ln.weight"], t[a + "attn.ln.bias"]
            m[h + "ln_2.weight"], m[h + "ln_2.bias"] = t[a + "ffn.ln.weight"], t[a + "ffn.ln.bias"]
            # Conv1D stores [in, out]: y = x W + b
            m[h + "attn.c_attn.weight"] = t[a + "attn.qkv.weight"].T
            m[h + "attn.c_attn.bias"] = t[a + "attn.qkv.bias"]
            m[h + "attn.c_proj.weight"] = t[a + "attn.out.weight"].T
            m[h + "attn.c_proj.bias"] = t[a + "attn.out.bias"]
            m[h + "mlp.c_fc.weight"] = t[a + "ffn.in.weight"].T
            m[h + "mlp.c_fc.bias"] = t[a + "ffn.in.bias"]
            m[h + "mlp.c_proj.weight"] = t[a + "ffn.out.weight"].T
            m[h + "mlp.c_proj.bias"] = t[a + "ffn.out.bias"]
        return m
    e = "bert.embeddings."
    m[e + "word_embeddings.weight"] = t["embeddings.word"]
    m[e + "position_embeddings.weight"] = t["embeddings.position"]
    m[e + "token_type_embeddings.weight"] = t["embeddings.token_type"]
    m[e + "LayerNorm.weight"], m[e + "LayerNorm.bias"] = t["embeddings.ln.weight"], t["embeddings.ln.bias"]
    for l in range(L):
        a, h = f"layer.{l}.", f"bert.encoder.layer.{l}."
        for i, part in enumerate(("query", "key", "value")):
            m[h + f"attention.self.{part}.weight"] = t[a + "attn.qkv.weight"][i * H:(i + 1) * H]
            m[h + f"attention.self.{part}.bias"] = t[a + "attn.qkv.bias"][i * H:(i + 1) * H]
        m[h + "attention.output.dense.weight"] = t[a + "attn.out.weight"]
        m[h + "attention.output.dense.bias"] = t[a + "attn.out.bias"]
        m[h + "attention.output.LayerNorm.weight"] = t[a + "attn.ln.weight"]
        m[h + "attention.output.LayerNorm.bias"] = t[a + "attn.ln.bias"]
        m[h + "intermediate.dense.weight"] = t[a + "ffn.in.weight"]
        m[h + "intermediate.dense.bias"] = t[a + "ffn.in.bias"]
        m[h + "output.dense.weight"] = t[a + "ffn.out.weight"]
        m[h + "output.dense.bias"] = t[a + "ffn.out.bias"]
        m[h + "output.LayerNorm.weight"] = t[a + "ffn.ln.weight"]
        m[h + "output.LayerNorm.bias"] = t[a + "ffn.ln.bias"]
    if cfg.head == 0:
        m["bert.pooler.dense.weight"] = t["pooler.weight"]
        m["bert.pooler.dense.bias"] = t["pooler.bias"]
        m["classifier.weight"] = t["classifier.weight"].reshape(1, H)
        m["classifier.bias"] = t["classifier.bias"]
    elif cfg.head == 1:
        m["qa_outputs.weight"] = t["qa.weight"]
        m["qa_outputs.bias"] = t["qa.bias"]
    else:
        c = "cls.predictions."
        m[c + "transform.dense.weight"] = t["mlm.transform.weight"]
        m[c + "transform.dense.bias"] = t["mlm.transform.bias"]
        m[c + "transform.LayerNorm.weight"] = t["mlm.ln.weight"]
        m[c + "transform.LayerNorm.bias"] = t["mlm.ln.bias"]
        m[c + "bias"] = t["mlm.decoder.bias"]
    return m


def _hf_grad_to_oracle(cfg, g):
    """HF gradients -> oracle names (inverse of _to_hf; tied decoders already
    accumulated into the word embedding by autograd)."""
    out = {}
    if cfg.arch == 1:
        out["embeddings.word"] = g["transformer.wte.weight"]
        out["embeddings.position"] = g["transformer.wpe.weight"]
        out["final_ln.weight"], out["final_ln.bias"] = g["transformer.ln_f.weight"], g["transformer.ln_f.bias"]
        for l in range(L):
            a, h = f"layer.{l}.", f"transformer.h.{l}."
            out[a + "attn.ln.weight"], out[a + "attn.ln.bias"] = g[h + "ln_1.weight"], g[h + "ln_1.bias"]
            out[a + "ffn.ln.weight"], out[a + "ffn.ln.bias"] = g[h + "ln_2.weight"], g[h + "ln_2.bias"]
            out[a + "attn.qkv.weight"] = g[h + "attn.c_attn.weight"].T
            out[a + "attn.qkv.bias"] = g[h + "attn.c_attn.bias"]
            out[a + "attn.out.weight"] = g[h + "attn.c_proj.weight"].T
            out[a + "attn.out.bias"] = g[h + "attn.c_proj.bias"]
            out[a + "ffn.in.weight"] = g[h + "mlp.c_fc.weight"].T
            out[a + "ffn.in.bias"] = g[h + "mlp.c_fc.bias"]
            out[a + "ffn.out.weight"] = g[h + "mlp.c_proj.weight"].T
            out[a + "ffn.out.bias"] = g[h + "mlp.c_proj.bias"]
        return out
    e = "bert.embeddings."
    out["embeddings.word"] = g[e + "word_embeddings.weight"]
    out["embeddings.position"] = g[e + "position_embeddings.weight"]
    out["embeddings.token_type"] = g[e + "token_type_embeddings.weight"]
    out["embeddings.ln.weight"], out["embeddings.ln.bias"] = g[e + "LayerNorm.weight"], g[e + "LayerNorm.bias"]
    for l in range(L):
        a, h = f"layer.{l}.", f"bert.encoder.layer.{l}."
        out[a + "attn.qkv.weight"] = torch.cat(
            [g[h + f"attention.self.{x}.weight"] for x in ("query", "key", "value")])
        out[a + "attn.qkv.bias"] = torch.cat(
            [g[h + f"attention.self.{x}.bias"] for x in ("query", "key", "value")])
        out[a + "attn.out.weight"] = g[h + "attention.output.dense.weight"]
        out[a + "attn.out.bias"] = g[h + "attention.output.dense.bias"]
        out[a + "attn.ln.weight"] = g[h + "attention.output.LayerNorm.weight"]
        out[a + "attn.ln.bias"] = g[h + "attention.output.LayerNorm.bias"]
        out[a + "ffn.in.weight"] = g[h + "intermediate.dense.weight"]
        out[a + "ffn.in.bias"] = g[h + "intermediate.dense.bias"]
        out[a + "ffn.out.weight"] = g[h + "output.dense.weight"]
        out[a + "ffn.out.bias"] = g[h + "output.dense.bias"]
        out[a + "ffn.ln.weight"] = g[h + "output.LayerNorm.weight"]
        out[a + "ffn.ln.bias"] = g[h + "output.LayerNorm.bias"]
    if cfg.head == 0:
        out["pooler.weight"], out["pooler.bias"] = g["bert.pooler.dense.weight"], g["bert.pooler.dense.bias"]
        out["classifier.weight"] = g["classifier.weight"].reshape(-1)
        out["classifier.bias"] = g["classifier.bias"]
    elif cfg.head == 1:
        out["qa.weight"], out["qa.bias"] = g["qa_outputs.weight"], g["qa_outputs.bias"]
    else:
        c = "cls.predictions."
        out["mlm.transform.weight"] = g[c + "transform.dense.weight"]
        out["mlm.transform.bias"] = g[c + "transform.dense.bias"]
        out["mlm.ln.weight"] = g[c + "transform.LayerNorm.weight"]
        out["mlm.ln.bias"] = g[c + "transform.LayerNorm.bias"]
        out["mlm.decoder.bias"] = g[c + "bias"]
    return out


def _labels(cfg, rng, tok):
    B, S = tok.shape
    if cfg.head == 0:
        return rng.integers(0, cfg.num_choices, size=B // cfg.num_choices).astype(np.int32)
    if cfg.head == 1:
        return rng.integers(0, S, size=2 * B).astype(np.int32)
    if cfg.head == 2:
        lab = np.full((B, S), -1, np.int32)
        lab[:, :-1] = tok[:, 1:]
        return lab.reshape(-1)
    lab = np.where(rng.random((B, S)) < 0.3, tok, -1).astype(np.int32).reshape(-1)
    lab[0] = tok[0, 0]
    return lab


def _hf_loss(cfg, model, tok, typ, lab):
    B, S = tok.shape
    ids = torch.from_numpy(tok.astype(np.int64))
    tt = torch.from_numpy(typ.astype(np.int64))
    if cfg.arch == 1:
        # GPT2LMHeadModel(labels=ids) shifts (logits[:, :-1] vs ids[:, 1:]) but
        # upcasts the logits to fp32 first (ForCausalLMLoss); the same shifted
        # mean CE is taken here on its fp64 logits
        logits = model(input_ids=ids).logits
        return torch.nn.functional.cross_entropy(logits[:, :-1].reshape(-1, V),
                                                 ids[:, 1:].reshape(-1))
    if cfg.head == 0:
        C = cfg.num_choices
        return model(input_ids=ids.reshape(B // C, C, S), token_type_ids=tt.reshape(B // C, C, S),
                     labels=torch.from_numpy(lab.astype(np.int64))).loss
    if cfg.head == 1:
        se = torch.from_numpy(lab.astype(np.int64)).reshape(B, 2)
        return model(input_ids=ids, token_type_ids=tt, start_positions=se[:, 0],
                     end_positions=se[:, 1]).loss
    lb = torch.from_numpy(lab.astype(np.int64)).reshape(B, S)
    lb[lb < 0] = -100
    return model(input_ids=ids, token_type_ids=tt, labels=lb).loss


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_oracle_matches_hf_transformers_fp64(variant):
    cfg = _cfg(variant)
    rng = np.random.default_rng(17)
    params = _params(cfg, rng)
    B, S = 8, 13
    tok = rng.integers(0, V, size=(B, S)).astype(np.int32)
    tok[:, -2:] = 0  # padding tokens present: their embedding row gets no gradient
    typ = (rng.random((B, S)) > 0.6).astype(np.int32) if cfg.type_vocab > 1 else np.zeros((B, S), np.int32)
    lab = _labels(cfg, rng, tok)

    loss, _, grads = bert_ref.loss_and_grads(params, tok, typ, lab, cfg, dtype=torch.float64)

    model = _hf_model(cfg).double()
    model.eval()  # dropout modules are p = 0 anyway; eval removes any doubt
    sd = model.state_dict()
    mapped = _to_hf(cfg, params)
    for k, v in mapped.items():
        assert k in sd, f"unmapped HF tensor {k}"
        assert tuple(sd[k].shape) == tuple(v.shape), (k, sd[k].shape, v.shape)
    model.load_state_dict(mapped, strict=False)
    # every trainable HF tensor is covered by the mapping (tied decoder weights
    # alias the word embedding)
    named = dict(model.named_parameters())
    for k in named:
        assert k in mapped, f"HF parameter {k} has no oracle counterpart"
    ref_loss = _hf_loss(cfg, model, tok, typ, lab)
    ref_loss = ref_loss
    ref_loss.backward()
    ref_grads = _hf_grad_to_oracle(cfg, {k: p.grad for k, p in named.items()})

    rl = float(ref_loss.detach())
    assert abs(loss - rl) <= 1e-10 * max(1.0, abs(rl)), (loss, rl)
    assert set(ref_grads) == set(grads)
    for name, g in grads.items():
        r = ref_grads[name].detach().reshape(-1).numpy()
        nr = np.linalg.norm(r)
        err = np.linalg.norm(g - r)
        assert err <= 1e-9 * max(nr, 1e-3), f"{name}: |d| {err:.3e} vs |g| {nr:.3e}"
