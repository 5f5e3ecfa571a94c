"""Python facade over the C-ABI trainer (libmimose_cuda.so).

This mirrors the reference's experiment surface (reference
proj/include/mimose/harness.hpp:48-118 ``ExperimentConfig`` / ``IterationRow``)
for a real GPU training run: every step returns an IterationRow-shaped dict
with the measured peak bytes instead of simulated ones. All compute happens in
the sm_100a kernels behind the C ABI; torch is used only to hand over device
pointers / streams and to view device buffers.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Callable, Dict, Optional

import numpy as np

from . import _lib
from ._lib import MimoseError, check, cuda_lib

PLANNERS = {"mimose": 0, "none": 1, "all": 2, "static-max": 3, "dtr": 4}
PHASES = {0: "planned", 1: "collect", 2: "sheltered", 3: "plain", 4: "fallback-collect"}


@dataclasses.dataclass
class ModelConfig:
    layers: int = 12
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    vocab: int = 30522
    max_pos: int = 512
    type_vocab: int = 2
    num_choices: int = 4
    hidden_dropout: float = 0.1
    attn_dropout: float = 0.1
    ln_eps: float = 1e-12
    init_std: float = 0.02
    seed: int = 1234
    arch: int = 0        # 0 post-LN BERT block, 1 pre-LN GPT-2 block
    head: int = 0        # 0 multiple choice, 1 extractive QA, 2 causal LM (tied), 3 masked LM (tied)
    causal: int = 0
    gelu_tanh: int = 0
    # HF BertEmbeddings: nn.Embedding(vocab, H, padding_idx=pad_token_id = 0) -
    # the padding row never receives a gradient; GPT-2 has none (-1)
    pad_token_id: int = 0

    def to_c(self):
        c = _lib.ModelCfg()
        for f in dataclasses.fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c

    def labels_count(self, B: int, S: int) -> int:
        return {0: B // self.num_choices, 1: 2 * B, 2: B * S, 3: B * S}[self.head]


@dataclasses.dataclass
class TrainConfig:
    planner: str = "mimose"
    batch: int = 64
    seq_min: int = 64
    seq_max: int = 512
    reserve_bytes: int = -1
    bucket_tolerance: float = 0.10
    cache_tolerance: float = 0.0
    max_sheltered_iters: int = 10
    collect_new_sizes_always: bool = False
    estimator_order: int = 2
    lr: float = 5e-5
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    weight_decay: float = 0.01
    max_grad_norm: float = 1.0
    # attention kernels: 3 (default) = flash attention (flash_sm100.cuh: no
    # S x S tensor saved or written -- lse per row + keep bits; any S);
    # 2 = single-row fused score kernels (attn_sm100.cuh: the key row of a
    # 128-query tile in TMEM, softmax / dropout / softmax-backward in the
    # epilogue; S <= 512, causal too, longer rows as 0); 0 = QK^T GEMM +
    # softmax kernels. 2 and 0 materialise P and dropout(P) like the
    # reference model (HF BERT / GPT-2, bert12.model).
    attn_fused: int = 3
    # automatic reserve sized for each step's S (extras_bytes(S) + 2 %) instead
    # of seq_max: short inputs then keep more blocks (fewer recomputes)
    reserve_per_size: int = 1
    # checkpoint unit the planner schedules: 0 = whole transformer block (the
    # reference's layer granularity), 1 = block half (attention half / FFN
    # half, 2 x layers units): an FFN half frees ~60 % of a block's bytes for
    # ~45 % of its forward time, so tight budgets recompute less
    ckpt_unit: int = 1
    # kept FFN halves save u only; the backward regenerates g = GELU(u)
    # (bit-identical) for the W2 gradient: 8 H fewer saved bytes per token and
    # block for one elementwise pass
    ffn_regen_g: int = 0

    def to_c(self):
        c = _lib.TrainCfg()
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            if f.name == "planner":
                v = PLANNERS[v]
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


# Named configurations of BASELINE.json configs[0..4].
PRESETS = {
    # configs[0]: small BERT-like encoder, 4 layers, hidden 256, S 32-256
    "small4-h256": (ModelConfig(layers=4, hidden=256, heads=4, ffn=1024),
                    TrainConfig(batch=8, seq_min=32, seq_max=256)),
    # configs[1]: BERT-base multiple choice (SWAG-shaped 16 x 4 choices), S 64-512
    "bert-base-mc": (ModelConfig(), TrainConfig(batch=64, seq_min=64, seq_max=512)),
    # configs[2]: RoBERTa-base / -large extractive QA (SQuAD-shaped), S up to 512
    "roberta-base-qa": (ModelConfig(vocab=50265, max_pos=514, type_vocab=1, ln_eps=1e-5, head=1),
                        TrainConfig(batch=12, seq_min=153, seq_max=512)),
    "roberta-large-qa": (ModelConfig(layers=24, hidden=1024, heads=16, ffn=4096, vocab=50265,
                                     max_pos=514, type_vocab=1, ln_eps=1e-5, head=1),
                         TrainConfig(batch=12, seq_min=153, seq_max=512)),
    # configs[3]: GPT-2 medium causal LM, S 128-1024
    "gpt2-medium-lm": (ModelConfig(layers=24, hidden=1024, heads=16, ffn=4096, vocab=50257,
                                   max_pos=1024, type_vocab=0, ln_eps=1e-5, arch=1, head=2,
                                   causal=1, gelu_tanh=1, pad_token_id=-1),
                       TrainConfig(batch=8, seq_min=128, seq_max=1024)),
    # configs[4]: BERT-large MLM pretraining-shaped, S 128-2048 (extended position table)
    "bert-large-mlm": (ModelConfig(layers=24, hidden=1024, heads=16, ffn=4096, max_pos=2048,
                                   head=3),
                       TrainConfig(batch=8, seq_min=128, seq_max=2048)),
}

# Workload description, default size distribution (reference workload.hpp
# syntax) and default budget fraction per preset. QA runs at
# 60 %: with B = 12 the constant footprint (weights, grads, AdamW state) is
# already ~40 % of the no-checkpoint peak, so 40 % is infeasible.
PRESET_INFO = {
    "small4-h256": ("small BERT-like encoder L4 H256 A4 F1024, MC head, B=8 (BASELINE configs[0])",
                    "uniform:32:256", 0.8),
    "bert-base-mc": ("bert-base-mc: BERT-base (L12 H768 A12 F3072 V30522) multiple-choice "
                     "fine-tune, SWAG-shaped 16x4 choices (BASELINE configs[1])",
                     "uniform:64:512", 0.4),
    "roberta-base-qa": ("roberta-base-qa: RoBERTa-base (L12 H768 V50265) extractive QA, "
                        "SQuAD-shaped B=12 (BASELINE configs[2])", "normal:300:100:153:512", 0.6),
    "roberta-large-qa": ("roberta-large-qa: RoBERTa-large (L24 H1024 V50265) extractive QA, "
                         "SQuAD-shaped B=12 (BASELINE configs[2])", "normal:300:100:153:512", 0.6),
    "gpt2-medium-lm": ("gpt2-medium-lm: GPT-2 medium (L24 H1024 A16 V50257) causal LM, B=8 "
                       "(BASELINE configs[3])", "uniform:128:1024", 0.4),
    "bert-large-mlm": ("bert-large-mlm: BERT-large (L24 H1024 A16 V30522) MLM 15%, B=8, "
                       "positions to 2048 (BASELINE configs[4])", "uniform:128:2048", 0.3),
}


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class Context:
    """One device + its budget arena (every byte the trainer uses lives here)."""

    def __init__(self, budget_bytes: int, device: int = 0):
        self.lib = cuda_lib()
        h = C.c_void_p()
        check(self.lib.mimose_ctx_create(device, int(budget_bytes), C.byref(h)))
        self.handle = h
        self.device = device

    def mem_stats(self) -> dict:
        st = _lib.MemStats()
        check(self.lib.mimose_mem_stats_get(self.handle, C.byref(st)))
        return st.as_dict()

    def close(self):
        if self.handle:
            self.lib.mimose_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Trainer:
    def __init__(self, model: ModelConfig, train: TrainConfig, budget_bytes: int,
                 device: int = 0):
        self.model = model
        self.train = train
        self.ctx = Context(budget_bytes, device)
        self.lib = self.ctx.lib
        h = C.c_void_p()
        try:
            check(self.lib.mimose_trainer_create(self.ctx.handle, C.byref(model.to_c()),
                                                 C.byref(train.to_c()), C.byref(h)))
        except Exception:
            self.ctx.close()  # the arena goes back now, not at garbage collection
            raise
        self.handle = h
        self._hook = None
        self.rows = []

    # ------------------------------------------------------------ steps
    def step(self, tokens, types, labels, *, optimizer: bool = True, stream=None) -> dict:
        """Host inputs (numpy / CPU torch, int32): H2D + fwd + bwd (+ AdamW) + loss D2H."""
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        B, S = tokens.shape
        types = np.ascontiguousarray(
            types if types is not None else np.zeros_like(tokens), dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        rep = _lib.StepReport()
        fn = self.lib.mimose_trainer_step if optimizer else self.lib.mimose_trainer_forward_backward
        check(fn(self.handle, tokens.ctypes.data, types.ctypes.data, labels.ctypes.data, B, S,
                 _stream_handle(stream), C.byref(rep)))
        d = self._row(rep)
        self.rows.append(d)
        return d

    def step_pinned(self, tokens, types, labels, *, optimizer: bool = True, stream=None) -> dict:
        """Host inputs already in pinned torch tensors (async H2D inside the step)."""
        B, S = tokens.shape
        rep = _lib.StepReport()
        fn = self.lib.mimose_trainer_step if optimizer else self.lib.mimose_trainer_forward_backward
        check(fn(self.handle, tokens.data_ptr(), types.data_ptr(), labels.data_ptr(), B, S,
                 _stream_handle(stream), C.byref(rep)))
        d = self._row(rep)
        self.rows.append(d)
        return d

    def step_async(self, tokens, types, labels, *, stream=None) -> dict:
        """Pinned host inputs; returns without waiting for the loss (see loss())."""
        B, S = tokens.shape
        rep = _lib.StepReport()
        check(self.lib.mimose_trainer_step_async(self.handle, tokens.data_ptr(), types.data_ptr(),
                                                 labels.data_ptr(), B, S, _stream_handle(stream),
                                                 C.byref(rep)))
        d = self._row(rep)
        self.rows.append(d)
        return d

    def loss(self, iteration: int) -> float:
        out = C.c_float()
        check(self.lib.mimose_trainer_loss(self.handle, iteration, C.byref(out)))
        return float(out.value)

    def step_device(self, batch: "DeviceBatch", *, optimizer: bool = True, stream=None) -> dict:
        """Device-resident inputs; no host synchronisation (loss stays on device)."""
        rep = _lib.StepReport()
        check(self.lib.mimose_trainer_step_device(
            self.handle, batch.tokens.data_ptr(), batch.types.data_ptr(), batch.labels.data_ptr(),
            batch.perm.data_ptr(), batch.seg.data_ptr(), batch.uid.data_ptr(), batch.n_unique,
            batch.B, batch.S, int(optimizer), _stream_handle(stream), C.byref(rep)))
        d = self._row(rep)
        self.rows.append(d)
        return d

    def optimizer_step(self, grad_scale: float = 1.0, stream=None):
        check(self.lib.mimose_trainer_optimizer_step(self.handle, grad_scale,
                                                     _stream_handle(stream)))

    @staticmethod
    def _row(rep) -> dict:
        d = rep.as_dict()
        d["phase_name"] = PHASES.get(d["phase"], str(d["phase"]))
        d["dropped"] = [i for i in range(64) if (d["dropped_mask_lo"] >> i) & 1]
        return d

    # ------------------------------------------------------------ control
    def force_plan(self, ids, active: bool = True):
        ids = list(ids)
        arr = (C.c_int * max(1, len(ids)))(*ids)
        check(self.lib.mimose_trainer_force_plan(self.handle, arr, len(ids), int(active)))

    def set_grad_hook(self, fn: Optional[Callable]):
        """fn(grads_tensor, stream_handle) runs after backward, before AdamW."""
        if fn is None:
            self._hook = None
            check(self.lib.mimose_trainer_set_grad_hook(self.handle, _lib.GRAD_HOOK(), None))
            return
        grads = self.grads()

        def _cb(user, ptr, n, stream):
            fn(grads, stream)

        self._hook = _lib.GRAD_HOOK(_cb)
        check(self.lib.mimose_trainer_set_grad_hook(self.handle, self._hook, None))

    def attach_dp(self, dp, bucket_mb: float = 32.0):
        """Native bucketed all-reduce during backward (dp: dp.NativeDP or None).
        With it attached, optimizer steps average over ranks by themselves."""
        self._dp = dp
        check(self.lib.mimose_trainer_attach_dp(self.handle, dp.handle if dp else None,
                                                int(bucket_mb * (1 << 20))))

    def dp_buckets(self):
        """[(after_unit, begin, end)] of the attached schedule (flat grad elements)."""
        out = (C.c_int64 * (3 * 512))()
        n = C.c_int()
        check(self.lib.mimose_trainer_dp_buckets(self.handle, out, 512, C.byref(n)))
        return [tuple(out[3 * i:3 * i + 3]) for i in range(min(n.value, 512))]

    # ------------------------------------------------------------ buffers
    def _buffers(self):
        p32, p16, g32, dl, dlg = (C.c_void_p() for _ in range(5))
        n = C.c_int64()
        check(self.lib.mimose_trainer_buffers(self.handle, C.byref(p32), C.byref(p16),
                                              C.byref(g32), C.byref(n), C.byref(dl),
                                              C.byref(dlg)))
        return p32.value, p16.value, g32.value, n.value, dl.value, dlg.value

    def params(self):
        import torch
        p32, _, _, n, _, _ = self._buffers()
        return torch.as_tensor(_DevArray(p32, n, "<f4"), device="cuda")

    def params_bf16(self):
        import torch
        _, p16, _, n, _, _ = self._buffers()
        return torch.as_tensor(_DevArray(p16, n, "<i2"), device="cuda").view(torch.bfloat16)

    def grads(self):
        import torch
        _, _, g32, n, _, _ = self._buffers()
        return torch.as_tensor(_DevArray(g32, n, "<f4"), device="cuda")

    def loss_device(self):
        import torch
        _, _, _, _, dl, _ = self._buffers()
        return torch.as_tensor(_DevArray(dl, 1, "<f4"), device="cuda")

    def logits_device(self):
        """Last step's head logits (fp32): MC [B] per choice, QA [B * S][2]
        (start, end). The tied token decoders (LM / MLM) keep no logits."""
        import torch
        _, _, _, _, _, dlg = self._buffers()
        if self.model.head == 0:
            return torch.as_tensor(_DevArray(dlg, self.train.batch, "<f4"), device="cuda")
        if self.model.head == 1:
            S = self.rows[-1]["seq"]
            n = 2 * self.train.batch * S
            return torch.as_tensor(_DevArray(dlg, n, "<f4"), device="cuda").reshape(-1, 2)
        raise ValueError("token heads (LM / MLM) do not retain logits")

    def param_table(self) -> Dict[str, tuple]:
        out = {}
        for i in range(self.lib.mimose_trainer_param_count(self.handle)):
            name = C.c_char_p()
            off = C.c_int64()
            n = C.c_int64()
            check(self.lib.mimose_trainer_param_info(self.handle, i, C.byref(name), C.byref(off),
                                                     C.byref(n)))
            out[name.value.decode()] = (off.value, n.value)
        return out

    def sync_params(self, stream=None):
        check(self.lib.mimose_trainer_sync_params(self.handle, _stream_handle(stream)))

    # ------------------------------------------------------------ planner state
    def _text(self, fn) -> str:
        p = C.c_void_p()
        check(fn(self.handle, C.byref(p)))
        return _lib.take_string(self.lib, p)

    def samples_csv(self) -> str:
        return self._text(self.lib.mimose_trainer_samples_csv)

    def estimator_text(self) -> str:
        return self._text(self.lib.mimose_trainer_estimator_text)

    def model_text(self) -> str:
        return self._text(self.lib.mimose_trainer_model_text)

    def report(self):
        """(summary, csv) in the reference's report formats (harness.hpp:339-379)."""
        a, b = C.c_void_p(), C.c_void_p()
        check(self.lib.mimose_trainer_report(self.handle, C.byref(a), C.byref(b)))
        return _lib.take_string(self.lib, a), _lib.take_string(self.lib, b)

    def info(self) -> dict:
        c, r, b = C.c_int64(), C.c_int64(), C.c_int64()
        t = C.c_int()
        h, m = C.c_int64(), C.c_int64()
        check(self.lib.mimose_trainer_info(self.handle, C.byref(c), C.byref(r), C.byref(b),
                                           C.byref(t), C.byref(h), C.byref(m)))
        return {"constant_bytes": c.value, "reserve_bytes": r.value, "budget": b.value,
                "trained": bool(t.value), "cache_hits": h.value, "cache_misses": m.value}

    def mem_stats(self) -> dict:
        return self.ctx.mem_stats()

    def close(self):
        if getattr(self, "handle", None):
            if getattr(self, "_dp", None) is not None:
                self.lib.mimose_trainer_attach_dp(self.handle, None, 0)
                self._dp = None
            self.lib.mimose_trainer_destroy(self.handle)
            self.handle = None
        self.ctx.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def token_tables(tokens: np.ndarray, vocab: int):
    """Host counting sort for the deterministic word-embedding gradient."""
    lib = cuda_lib()
    tokens = np.ascontiguousarray(tokens, dtype=np.int32).ravel()
    T = tokens.size
    perm = np.empty(T, np.int32)
    seg = np.empty(T + 1, np.int32)
    uid = np.empty(max(T, 1), np.int32)
    nu = C.c_int()
    check(lib.mimose_build_token_tables(tokens.ctypes.data, T, vocab, perm.ctypes.data,
                                        seg.ctypes.data, uid.ctypes.data, C.byref(nu)))
    return perm, seg[: nu.value + 1].copy(), uid[: nu.value].copy(), nu.value


@dataclasses.dataclass
class DeviceBatch:
    """One step's inputs resident on the device (torch int32 tensors)."""
    tokens: "object"
    types: "object"
    labels: "object"
    perm: "object"
    seg: "object"
    uid: "object"
    n_unique: int
    B: int
    S: int

    @staticmethod
    def from_host(tokens, types, labels, vocab, device="cuda"):
        import torch
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        B, S = tokens.shape
        perm, seg, uid, nu = token_tables(tokens, vocab)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)
        return DeviceBatch(t(tokens), t(types), t(labels), t(perm), t(seg),
                           t(uid if nu else np.zeros(1, np.int32)), nu, B, S)


def synthetic_batch(rng: np.random.Generator, B: int, S: int, vocab: int, num_choices: int,
                    type_vocab: int = 2):
    """SWAG-shaped synthetic multiple-choice batch (uniform token ids)."""
    tokens = rng.integers(0, vocab, size=(B, S), dtype=np.int32)
    types = np.zeros((B, S), np.int32)
    if type_vocab > 1:
        split = rng.integers(1, S, size=B)
        types[np.arange(S)[None, :] >= split[:, None]] = 1
    labels = rng.integers(0, num_choices, size=B // num_choices, dtype=np.int32)
    return tokens, types, labels


def synthetic_task_batch(rng: np.random.Generator, cfg: ModelConfig, B: int, S: int,
                         mask_prob: float = 0.15):
    """Synthetic batch for cfg.head with the label layout the head expects.

    MC: [B / C] choice ids; QA: [2 B] (start, end) spans; LM: [B * S] next-token
    ids with the last position of each sequence ignored (-1); MLM: [B * S]
    original ids at ~mask_prob of the positions (at least one), -1 elsewhere.
    """
    if cfg.head == 0:
        return synthetic_batch(rng, B, S, cfg.vocab, cfg.num_choices, max(cfg.type_vocab, 1))
    tokens = rng.integers(0, cfg.vocab, size=(B, S), dtype=np.int32)
    types = np.zeros((B, S), np.int32)
    if cfg.head == 1:
        st = rng.integers(0, S, size=B)
        en = np.minimum(S - 1, st + rng.integers(0, 8, size=B))
        labels = np.stack([st, en], axis=1).reshape(-1).astype(np.int32)
    elif cfg.head == 2:
        labels = np.full((B, S), -1, np.int32)
        labels[:, :-1] = tokens[:, 1:]
        labels = labels.reshape(-1)
    else:
        sel = rng.random((B, S)) < mask_prob
        sel.reshape(-1)[rng.integers(0, B * S)] = True
        labels = np.where(sel, tokens, -1).astype(np.int32).reshape(-1)
    return tokens, types, labels
