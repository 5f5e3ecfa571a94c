"""CPU numerics oracle for the B200 training step (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker / the timed CPU baseline - never as the
product path.

What it restates: the transformer-block training step the north star puts on
the GPU (post-LN BERT encoder block with materialised
attention, GELU FFN, multiple-choice head, AdamW-free fwd+bwd), in plain
PyTorch-CPU fp32/fp64 with autograd. The reference has no tensor code (its
layer is the byte polynomial of reference proj/include/mimose/model_spec.hpp:
76-78, its iteration the replay of simulator.hpp:104-160), so numerical
parity here is anchored on the paper's framework - HuggingFace
BertForMultipleChoice as of transformers v4.18 on PyTorch 1.11
 - whose block structure this follows:
  embeddings = dropout(LN(word + position + token_type))
  block:  h1 = LN(h + dropout(Wo . attn(h)))  attn probs dropped out
          h2 = LN(h1 + dropout(W2 . gelu(W1 . h1)))       (exact erf GELU)
  head:   logits = dropout(tanh(Wp . h[:, 0])) . wc + bc ; CE over choices
Pinned to the third-party implementation itself: tests/test_oracle_vs_hf.py
loads identical weights into HF BertForMultipleChoice /
BertForQuestionAnswering / BertForMaskedLM / GPT2LMHeadModel (transformers
5.5.0, float64, dropout 0) and requires this oracle's loss and every
gradient to agree to 1e-9 relative; the reference repository itself has no
tensor vectors. Loss/grad agreement with the GPU is checked at stated
tolerances in tests/test_trainer_gpu.py and
tests/test_parity_baseline_shapes_gpu.py.

Dropout masks are reproduced bit-exactly with a numpy restatement of the
Philox4x32-10 counter scheme the kernels use, so parity holds with dropout on.
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np
import torch

SITE_ATTN_PROBS, SITE_ATTN_OUT, SITE_FFN_OUT, SITE_EMBED, SITE_POOL = 0, 1, 2, 3, 4

# ----------------------------------------------------------------- Philox
_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(seed: int, stream: int, groups: np.ndarray) -> np.ndarray:
    """Philox4x32-10 with key=seed, counter=(group_lo, group_hi, stream_lo, stream_hi).

    Returns uint32 [len(groups), 4]. Restates mimose_dev::Philox (csrc/common.cuh).
    """
    g = groups.astype(np.uint64)
    c0 = (g & _MASK32).astype(np.uint32)
    c1 = (g >> np.uint64(32)).astype(np.uint32)
    c2 = np.full_like(c0, np.uint32(stream & 0xFFFFFFFF))
    c3 = np.full_like(c0, np.uint32((stream >> 32) & 0xFFFFFFFF))
    k0 = np.uint32(seed & 0xFFFFFFFF)
    k1 = np.uint32((seed >> 32) & 0xFFFFFFFF)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = c0.astype(np.uint64) * _M0
            p1 = c2.astype(np.uint64) * _M1
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & _MASK32).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & _MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
    return np.stack([c0, c1, c2, c3], axis=-1)


def dropout_threshold(p: float) -> int:
    """16-bit keep threshold round(p * 65536), clamped to [1, 65535] (0 = off)."""
    if p <= 0.0:
        return 0
    t = p * 65536.0 + 0.5
    thr = 65535 if t >= 65535.0 else int(t)
    return max(thr, 1)


def keep_mask(p: float, seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Boolean keep mask for element indices `idx` (any shape).

    Element i uses the 16-bit half (i & 1) of word ((i & 7) >> 1) of
    Philox4x32-10(seed, stream, i >> 3) - one Philox call per 8 elements
    (restates mimose_dev::dropout_mask8, csrc/common.cuh)."""
    thr = dropout_threshold(p)
    if thr == 0:
        return np.ones(idx.shape, dtype=bool)
    flat = idx.reshape(-1)
    out = np.empty(flat.size, dtype=bool)
    chunk = 1 << 23  # bounded temporaries for S x S masks at S = 2048
    for c0 in range(0, flat.size, chunk):
        f = flat[c0:c0 + chunk].astype(np.uint64)
        groups = f >> np.uint64(3)
        g0, g1 = int(groups.min()), int(groups.max())
        if g1 - g0 < 2 * f.size:  # dense index range: one Philox call per group in it
            r = philox4x32_10(seed, stream, np.arange(g0, g1 + 1, dtype=np.uint64))
            inv = (groups - np.uint64(g0)).astype(np.int64)
        else:
            ug, inv = np.unique(groups, return_inverse=True)
            r = philox4x32_10(seed, stream, ug)
        e = (f & np.uint64(7)).astype(np.int64)
        words = r[inv, e >> 1].astype(np.uint64)
        half = (words >> (np.uint64(16) * (e & 1).astype(np.uint64))) & np.uint64(0xFFFF)
        out[c0:c0 + chunk] = half >= np.uint64(thr)
    return out.reshape(idx.shape)


def stream_id(step: int, layer: int, site: int) -> int:
    return (step << 20) | ((layer & 0xFFFF) << 4) | site


# ----------------------------------------------------------------- model
ARCH_BERT, ARCH_GPT2 = 0, 1
HEAD_MC, HEAD_QA, HEAD_LM, HEAD_MLM = 0, 1, 2, 3


def _c(cfg, name, default=0):
    return getattr(cfg, name, default)


def param_shapes(cfg) -> Dict[str, tuple]:
    H, F, V, P, Ty = cfg.hidden, cfg.ffn, cfg.vocab, cfg.max_pos, cfg.type_vocab
    arch, head = _c(cfg, "arch"), _c(cfg, "head")
    shp = {"embeddings.word": (V, H), "embeddings.position": (P, H)}
    if Ty > 0:
        shp["embeddings.token_type"] = (Ty, H)
    if arch == ARCH_BERT:
        shp.update({"embeddings.ln.weight": (H,), "embeddings.ln.bias": (H,)})
    else:
        shp.update({"final_ln.weight": (H,), "final_ln.bias": (H,)})
    if head == HEAD_MC:
        shp.update({"pooler.weight": (H, H), "pooler.bias": (H,),
                    "classifier.weight": (H,), "classifier.bias": (1,)})
    elif head == HEAD_QA:
        shp.update({"qa.weight": (2, H), "qa.bias": (2,)})
    elif head == HEAD_MLM:
        shp.update({"mlm.transform.weight": (H, H), "mlm.transform.bias": (H,),
                    "mlm.ln.weight": (H,), "mlm.ln.bias": (H,), "mlm.decoder.bias": (V,)})
    for l in range(cfg.layers):
        p = f"layer.{l}."
        shp.update({
            p + "attn.qkv.weight": (3 * H, H), p + "attn.qkv.bias": (3 * H,),
            p + "attn.out.weight": (H, H), p + "attn.out.bias": (H,),
            p + "attn.ln.weight": (H,), p + "attn.ln.bias": (H,),
            p + "ffn.in.weight": (F, H), p + "ffn.in.bias": (F,),
            p + "ffn.out.weight": (H, F), p + "ffn.out.bias": (H,),
            p + "ffn.ln.weight": (H,), p + "ffn.ln.bias": (H,),
        })
    return shp


def _drop(x: torch.Tensor, p: float, seed: int, stream: int, idx: np.ndarray) -> torch.Tensor:
    if p <= 0.0:
        return x
    m = torch.from_numpy(keep_mask(p, seed, stream, idx)).to(x.dtype)
    return x * m * (1.0 / (1.0 - p))


def loss_and_grads(params: Dict[str, np.ndarray], tokens: np.ndarray, types: np.ndarray,
                   labels: np.ndarray, cfg, step: int = 0, dtype=torch.float32,
                   checkpoint_layers=()):
    """Forward + backward on CPU. Returns (loss, logits, {name: grad ndarray}).

    checkpoint_layers: blocks run under torch.utils.checkpoint (the paper's
    mechanism) - forward without saving, recomputed in the
    backward; the Philox masks are regenerated identically, so the result
    does not change (the CPU arm of bench.py times Mimose plans this way).

    Architectures (cfg.arch): 0 post-LN BERT block, 1 pre-LN GPT-2 block
    (attention causal when cfg.causal). Heads (cfg.head) and label layouts:
      0 multiple choice  labels [B / C]
      1 extractive QA    labels [2 B] = (start, end) per sequence
      2 causal LM (tied) labels [B * S] next-token ids, -1 ignored
      3 masked LM (tied) labels [B * S] original ids at masked positions, -1 elsewhere
    """
    shapes = param_shapes(cfg)
    P = {k: torch.tensor(np.asarray(v, dtype=np.float64).reshape(shapes[k]), dtype=dtype,
                         requires_grad=True) for k, v in params.items() if k in shapes}
    B, S = tokens.shape
    H, nh, L = cfg.hidden, cfg.heads, cfg.layers
    arch, head = _c(cfg, "arch"), _c(cfg, "head")
    causal = bool(_c(cfg, "causal"))
    gelu_kind = "tanh" if _c(cfg, "gelu_tanh") else "none"
    d = H // nh
    T = B * S
    ld = (S + 7) // 8 * 8
    seed = cfg.seed
    ph, pa = cfg.hidden_dropout, cfg.attn_dropout
    tok = torch.from_numpy(tokens.astype(np.int64)).reshape(-1)
    pos = torch.arange(S).repeat(B)
    hid_idx = (np.arange(T, dtype=np.uint64)[:, None] * np.uint64(H)
               + np.arange(H, dtype=np.uint64)[None, :])

    def ln(x, w, b):
        return torch.nn.functional.layer_norm(x, (H,), P[w], P[b], eps=cfg.ln_eps)

    # HF BertEmbeddings: nn.Embedding(..., padding_idx=pad_token_id) - the
    # padding row gets no gradient from the lookup (a tied decoder still
    # contributes to it); GPT-2 has no padding index (pad_token_id -1)
    pad = _c(cfg, "pad_token_id", -1)
    e = torch.nn.functional.embedding(tok, P["embeddings.word"],
                                      padding_idx=pad if pad >= 0 else None) \
        + P["embeddings.position"][pos]
    if cfg.type_vocab > 0:
        typ = torch.from_numpy(types.astype(np.int64)).reshape(-1)
        e = e + P["embeddings.token_type"][typ]
    if arch == ARCH_BERT:
        e = ln(e, "embeddings.ln.weight", "embeddings.ln.bias")
    h = _drop(e, ph, seed, stream_id(step, L, SITE_EMBED), hid_idx)
    rows = np.arange(B * nh * S, dtype=np.uint64).reshape(B, nh, S, 1)
    att_idx = rows * np.uint64(ld) + np.arange(S, dtype=np.uint64)[None, None, None, :]
    cmask = torch.triu(torch.ones(S, S, dtype=torch.bool), diagonal=1) if causal else None

    def attention(x, p, l):
        qkv = x @ P[p + "attn.qkv.weight"].T + P[p + "attn.qkv.bias"]
        q, k, v = (qkv[:, i * H:(i + 1) * H].reshape(B, S, nh, d).permute(0, 2, 1, 3)
                   for i in range(3))
        sc = (q @ k.transpose(-1, -2)) / math.sqrt(d)
        if cmask is not None:
            sc = sc.masked_fill(cmask, float("-inf"))
        pr = torch.softmax(sc, dim=-1)
        pr = _drop(pr, pa, seed, stream_id(step, l, SITE_ATTN_PROBS), att_idx)
        ctx = (pr @ v).permute(0, 2, 1, 3).reshape(T, H)
        return ctx @ P[p + "attn.out.weight"].T + P[p + "attn.out.bias"]

    def ffn(x, p):
        u = x @ P[p + "ffn.in.weight"].T + P[p + "ffn.in.bias"]
        return torch.nn.functional.gelu(u, approximate=gelu_kind) @ P[p + "ffn.out.weight"].T \
            + P[p + "ffn.out.bias"]

    def block(h, l):
        p = f"layer.{l}."
        if arch == ARCH_BERT:
            a = attention(h, p, l)
            h1 = ln(h + _drop(a, ph, seed, stream_id(step, l, SITE_ATTN_OUT), hid_idx),
                    p + "attn.ln.weight", p + "attn.ln.bias")
            return ln(h1 + _drop(ffn(h1, p), ph, seed, stream_id(step, l, SITE_FFN_OUT), hid_idx),
                      p + "ffn.ln.weight", p + "ffn.ln.bias")
        a = attention(ln(h, p + "attn.ln.weight", p + "attn.ln.bias"), p, l)
        h1 = h + _drop(a, ph, seed, stream_id(step, l, SITE_ATTN_OUT), hid_idx)
        f = ffn(ln(h1, p + "ffn.ln.weight", p + "ffn.ln.bias"), p)
        return h1 + _drop(f, ph, seed, stream_id(step, l, SITE_FFN_OUT), hid_idx)

    ckpt = set(checkpoint_layers)
    for l in range(L):
        if l in ckpt:
            import torch.utils.checkpoint as tuc
            h = tuc.checkpoint(block, h, l, use_reentrant=False)
        else:
            h = block(h, l)
    if arch == ARCH_GPT2:
        h = ln(h, "final_ln.weight", "final_ln.bias")

    lab = torch.from_numpy(labels.astype(np.int64))
    if head == HEAD_MC:
        cls = h.reshape(B, S, H)[:, 0, :]
        pooled = torch.tanh(cls @ P["pooler.weight"].T + P["pooler.bias"])
        pool_idx = (np.arange(B, dtype=np.uint64)[:, None] * np.uint64(H)
                    + np.arange(H, dtype=np.uint64)[None, :])
        pooled = _drop(pooled, ph, seed, stream_id(step, L, SITE_POOL), pool_idx)
        logits = pooled @ P["classifier.weight"] + P["classifier.bias"]
        C = cfg.num_choices
        loss = torch.nn.functional.cross_entropy(logits.reshape(B // C, C), lab)
    elif head == HEAD_QA:
        logits = (h @ P["qa.weight"].T + P["qa.bias"]).reshape(B, S, 2)
        st, en = lab.reshape(B, 2)[:, 0], lab.reshape(B, 2)[:, 1]
        loss = 0.5 * (torch.nn.functional.cross_entropy(logits[..., 0], st)
                      + torch.nn.functional.cross_entropy(logits[..., 1], en))
    elif head == HEAD_LM:
        logits = h @ P["embeddings.word"].T
        loss = torch.nn.functional.cross_entropy(logits, lab, ignore_index=-1)
    else:
        sel = lab >= 0
        x = h[sel]
        t = x @ P["mlm.transform.weight"].T + P["mlm.transform.bias"]
        t = torch.nn.functional.gelu(t, approximate=gelu_kind)
        t = torch.nn.functional.layer_norm(t, (H,), P["mlm.ln.weight"], P["mlm.ln.bias"],
                                           eps=cfg.ln_eps)
        logits = t @ P["embeddings.word"].T + P["mlm.decoder.bias"]
        loss = torch.nn.functional.cross_entropy(logits, lab[sel])
    loss.backward()
    grads = {k: t.grad.detach().numpy().reshape(-1).copy() for k, t in P.items()}
    return float(loss.detach()), logits.detach().numpy(), grads


def numpy_bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to bf16 (round-to-nearest-even), returned as fp32."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + np.uint64(0x7FFF) + ((a >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return (r & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
