#!/usr/bin/env python
"""Benchmark: samples/s of Mimose input-aware checkpointing training on B200
under a fixed per-GPU memory budget with dynamic sequence lengths.

Workload (BASELINE.json configs[1]): BERT-base multiple-choice fine-tune,
SWAG-shaped synthetic data (16 questions x 4 choices = 64 sequences per rank
per step), sequence length S drawn per step from uniform:64:512 with the
reference's own sampler (include/mimose/workload.hpp sample_workload, seed
base+rank), random-init weights (N(0, 0.02)), AdamW, dropout 0.1, bf16
compute. Budget = 40 % of the measured no-checkpoint peak at S_max
(everything - weights, grads, AdamW state, activations, workspace - lives in
the budget arena). The peak is measured twice: for the materialised-
attention model (the reference's / HF's memory semantics, --budget-basis
materialised, the headline default) and for the measured flash-attention
configuration itself ("self"); the line carries the Mimose run on BOTH
budgets (mimose / mimose_other_basis) against the same no-checkpoint
throughput. --preset picks the other BASELINE configs (parity / reporting
runs): small4-h256, roberta-{base,large}-qa, gpt2-medium-lm, bert-large-mlm,
each with its own default size distribution and budget; --planner static-max
| dtr runs the reference's baseline planners under the same budget.

N > 1: one rank per GPU, each drawing its own sequence lengths (seed base +
rank) and planning under its own budget; the gradient exchange is the
library's own NCCL communicator (mimose_dp_*) with bucketed all-reduce
issued as the backward finishes each block (MIMOSE_DP=torch: one torch
all-reduce after backward). NCCL's own device buffers are measured and
taken off each rank's arena.

Arms
  default            this repo's B200 path (python bench.py --gpus N ...)
  --impl reference   the CPU path: sizes and plans from the compiled
                     UNMODIFIED reference (oracle/_ref), the oracle's
                     PyTorch-CPU fp32 restatement of the step with the
                     planned blocks under torch.utils.checkpoint (the
                     reference itself is a byte/ms simulator with no tensor
                     code), all host cores, bounded sub-batch per step, rank 0
                     only.

One JSON line on rank 0. Timing: W untimed warm-up steps after the planner's
sheltered calibration window, then exactly K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec under fixed GPU mem budget, dynamic seqlen, 1/2/4/8 B200; mem-pred err"
GiB = 1 << 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--budget-frac", type=float, default=None,
                    help="budget as a fraction of the no-ckpt peak (default: per preset)")
    ap.add_argument("--preset", default="bert-base-mc")
    ap.add_argument("--dist", default=None, help="size distribution (default: per preset)")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--no-baseline", action="store_true", help="skip no-ckpt throughput arm")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--size-stream", default="grouped", choices=["shared", "per-rank", "grouped"],
                    help="DP length policy: 'grouped' (default) = length-grouped per-rank "
                         "sampling: every step's length group comes from the seeded reference "
                         "stream and each rank draws its own S within +-GROUP_JITTER of it from "
                         "its own RNG (seed base+rank), so ranks train different lengths under "
                         "their own plans without waiting for the longest of N independent "
                         "draws (HF group_by_length practice); 'per-rank' = independent "
                         "streams seed base+rank (max-over-ranks straggler cost); 'shared' = "
                         "every rank the same S")
    ap.add_argument("--group-jitter", type=float, default=0.05,
                    help="relative per-rank spread of S inside a length group ('grouped')")
    ap.add_argument("--attn", default="flash", choices=["flash", "materialised"],
                    help="attention kernels of the measured runs: flash (attn_fused 3, no S x S "
                         "tensor) or materialised (attn_fused 2, P / Pd saved like the reference "
                         "model). The budget denominator is always the materialised model's "
                         "no-ckpt peak (the reference model's memory semantics)")
    ap.add_argument("--budget-basis", default="materialised", choices=["materialised", "self"],
                    help="no-ckpt peak the budget fraction applies to: the materialised-attention "
                         "model's (reference memory semantics, default) or the measured "
                         "configuration's own")
    ap.add_argument("--planner", default="mimose", choices=["mimose", "static-max", "dtr"],
                    help="planner of the measured runs under the budget: Mimose (the product), "
                         "static-max (plan once for S_max, reference baselines.hpp:20-23) or "
                         "dtr (reactive eviction on the real arena, baselines.hpp:62-159)")
    ap.add_argument("--cache-tol", type=float, default=0.0,
                    help="plan-cache tolerance (reference scheduler.hpp:27, 204-221)")
    ap.add_argument("--ffn-regen-g", type=int, default=0, choices=[0, 1],
                    help="Mimose runs: kept FFN halves save u only and regenerate GELU(u) in the "
                         "backward (the no-checkpoint baseline always saves both)")
    ap.add_argument("--ckpt-unit", type=int, default=1, choices=[0, 1],
                    help="checkpoint unit: 1 = block half (attention / FFN, default), 0 = block")
    ap.add_argument("--profile-only", action="store_true",
                    help="short run for ncu (no comparison arms, no cpu baseline)")
    args = ap.parse_args()
    from paper_2209_02478_b200.trainer import PRESET_INFO
    _, dist_default, frac_default = PRESET_INFO[args.preset]
    if args.dist is None:
        args.dist = dist_default
    if args.budget_frac is None:
        args.budget_frac = frac_default
    return args


# ----------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) >= 7:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def sizes_for(dist, batch, iters, seed):
    """Per-step sequence lengths from the product's copy of the reference
    sampler (include/mimose/workload.hpp sample_workload, bit-exact with it:
    tests/test_planner_golden.py)."""
    from paper_2209_02478_b200 import planner
    xs = planner.host_lib().workload(dist, 1, iters, seed)
    return [int(x) for x in xs]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def dist_init(n):
    if n <= 1 and "WORLD_SIZE" not in os.environ:
        return 0, 1, 0
    import torch.distributed as dist
    import torch
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", n))
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    # NCCL over NVLink on real multi-GPU runs; MIMOSE_DIST_BACKEND=gloo lets the
    # N>1 code path be exercised with several ranks sharing one GPU (tests).
    backend = os.environ.get("MIMOSE_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def allmax(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------- CPU arm
def ref_planner_lib():
    """The UNMODIFIED reference planner (proj/include compiled by
    oracle/Makefile into oracle/_ref/libmimose_ref.so; built here, shipped to
    the GPU box with the snapshot) - the reference arm's sizes and plans come
    from it, not from this repo's product libraries."""
    from paper_2209_02478_b200.planner import PlannerLib
    path = os.path.join(ROOT, "oracle", "_ref", "libmimose_ref.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/libmimose_ref.so"],
                       check=True, capture_output=True)
    return PlannerLib(path, "ref_planner_")


def cpu_model_document(model_cfg, batch, s_min, s_max):
    """The CPU step's memory profile in the reference's own `.model` format,
    with the reference's own per-block semantics (proj/models/bert12.model:
    fp32 BERT block = 16 hidden-sized fp32 tensors per token + 3 S x S fp32
    tensors per head, output = one fp32 hidden state; constant = 16 B/param)."""
    H, nh, L = model_cfg.hidden, model_cfg.heads, model_cfg.layers
    from oracle import bert_ref
    n_param = sum(int(np.prod(s)) for s in bert_ref.param_shapes(model_cfg).values())
    lines = ["version: 1", f"constant_footprint: {16 * n_param}",
             f"input_range: {batch * s_min} {batch * s_max}", ""]
    for l in range(L):
        lines += ["[layer]", f"id: {l}", f"position: {l}", f"stage: {l}",
                  "category: quadratic-structure",
                  f"activation_coeffs: 0 {16 * H * 4} {3 * nh * 4 / batch!r}",
                  f"boundary_coeffs: 0 {H * 4}", "forward_time_coeffs: 1 0.0006", ""]
    return "\n".join(lines)


def cpu_plans(model_cfg, batch, s_min, s_max, xs, frac):
    """Mimose on the CPU path: the reference's fit + lookup_or_plan over the
    CPU model document at a budget of frac x its no-checkpoint peak at S_max."""
    import numpy as np  # noqa: F401
    from paper_2209_02478_b200.planner import SchedCfg
    ref = ref_planner_lib()
    doc = cpu_model_document(model_cfg, batch, s_min, s_max)
    # the sheltered collector's samples of this profile at three sizes (exact)
    H, nh = model_cfg.hidden, model_cfg.heads
    rows = ["layer_id,input_size,bytes,ms,valid"]
    for S in (s_min, (s_min + s_max) // 2, s_max):
        x = batch * S
        a = round(16 * H * 4 * x + 3 * nh * 4 / batch * x * x)
        rows += [f"{l},{x},{a},{1 + 0.0006 * x!r},1" for l in range(model_cfg.layers)]
    est = ref.fit_text("\n".join(rows) + "\n", 2)
    peak, _, _ = ref.simulate_plan(doc, [], batch * s_max)
    cfg = SchedCfg(budget_bytes=int(frac * peak))
    masks, _, _ = ref.plan_seq(est, doc, cfg, [batch * S for S in xs], model_cfg.layers)
    return [[l for l in range(model_cfg.layers) if (m >> l) & 1] for m in masks], int(frac * peak)


def cpu_step_sample(model_cfg, S, sub_batch, rng, threads, ckpt=()):
    """One bounded CPU training step (oracle fp32 fwd+bwd with the planned
    blocks under torch.utils.checkpoint, + AdamW) of `sub_batch` sequences of
    length S; returns seconds."""
    import numpy as np
    import torch
    from oracle import bert_ref
    from paper_2209_02478_b200.trainer import synthetic_task_batch
    torch.set_num_threads(threads)
    shapes = bert_ref.param_shapes(model_cfg)
    g = np.random.default_rng(0)
    params = {k: (g.standard_normal(int(np.prod(s))).astype(np.float32) * 0.02
                  if (k.endswith("weight") and "ln" not in k) or k.startswith("embeddings.")
                  and "ln" not in k else
                  (np.ones(int(np.prod(s)), np.float32) if "ln.weight" in k
                   else np.zeros(int(np.prod(s)), np.float32)))
              for k, s in shapes.items()}
    tok, typ, lab = synthetic_task_batch(rng, model_cfg, sub_batch, S)
    t0 = time.perf_counter()
    _, _, grads = bert_ref.loss_and_grads(params, tok, typ, lab, model_cfg, step=0,
                                          checkpoint_layers=ckpt)
    # AdamW update of every parameter (what the GPU step also does)
    for k, gr in grads.items():
        p = torch.from_numpy(params[k])
        gt = torch.from_numpy(gr)
        m = torch.zeros_like(p)
        v = torch.zeros_like(p)
        m.mul_(0.9).add_(gt, alpha=0.1)
        v.mul_(0.999).addcmul_(gt, gt, value=0.001)
        p.mul_(1 - 5e-5 * 0.01).addcdiv_(m, v.sqrt().add_(1e-8), value=-5e-5)
    return time.perf_counter() - t0


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    import numpy as np
    from paper_2209_02478_b200.trainer import PRESETS, PRESET_INFO
    model_cfg, train_cfg = PRESETS[args.preset]
    threads = os.cpu_count() or 1
    sub = model_cfg.num_choices if model_cfg.head == 0 else 1  # one question / sequence
    # sizes: the reference's own sampler (workload.hpp sample_workload), seed base
    xs = [int(x) for x in ref_planner_lib().workload(args.dist, 1, args.warmup + args.steps,
                                                     args.seed)]
    plans, cpu_budget = cpu_plans(model_cfg, sub, train_cfg.seq_min, train_cfg.seq_max, xs,
                                  args.budget_frac)
    rng = np.random.default_rng(args.seed)
    for S, ck in zip(xs[:args.warmup], plans[:args.warmup]):
        cpu_step_sample(model_cfg, S, sub, rng, threads, ck)
    tot = 0.0
    for S, ck in zip(xs[args.warmup:], plans[args.warmup:]):
        tot += cpu_step_sample(model_cfg, S, sub, rng, threads, ck)
    value = sub * args.steps / tot
    timed_plans = plans[args.warmup:]
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"{PRESET_INFO[args.preset][0]} - CPU path", "global_batch": sub,
                   "seq_len": args.dist, "parallelism": "cpu",
                   "budget_frac_of_no_ckpt_peak": args.budget_frac,
                   "cpu_budget_bytes": cpu_budget},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
                         "sample": f"{sub} sequence(s) per step at the step's drawn S "
                                   f"(reference sampler, oracle/_ref); plans from the compiled "
                                   f"reference planner (fit + lookup_or_plan) over the fp32 CPU "
                                   f"profile in bert12.model semantics; oracle/bert_ref.py fp32 "
                                   f"fwd+bwd with the planned blocks under torch.utils.checkpoint "
                                   f"+ AdamW",
                         "avg_checkpointed_blocks": sum(len(p) for p in timed_plans) /
                                                    max(1, len(timed_plans)),
                         "seqs": xs[args.warmup:]},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def traffic_record(preset):
    """ncu --set full DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
    of the dominant dense-GEMM launch, captured at this commit by
    tools/ncu_traffic.py into profiles/traffic.json (None when absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(preset)
    except Exception:
        return None


def run_gpu_arm(args, rank, world, local):
    import torch
    from paper_2209_02478_b200 import _lib
    from paper_2209_02478_b200.trainer import (PRESETS, PRESET_INFO, DeviceBatch, Trainer,
                                               synthetic_task_batch)
    import dataclasses

    lib = _lib.cuda_lib()
    model_cfg, train_cfg = PRESETS[args.preset]
    train_cfg = dataclasses.replace(train_cfg, attn_fused=3 if args.attn == "flash" else 2,
                                    ckpt_unit=args.ckpt_unit, cache_tolerance=args.cache_tol)
    B = train_cfg.batch
    S_max = train_cfg.seq_max
    stream = torch.cuda.current_stream()
    pk, pk_kind = peaks()

    # gradient exchange for N > 1: the library's own NCCL communicator with
    # bucketed all-reduce overlapping the backward (MIMOSE_DP=native, default
    # on NCCL), or one torch.distributed all-reduce after backward (=torch,
    # and always under the gloo test backend). Its device buffers live
    # outside the arena, so they are taken off each rank's budget.
    dp = None
    if world > 1 and os.environ.get("MIMOSE_DP", "native") == "native":
        import torch.distributed as dist
        if dist.get_backend() == "nccl":
            from paper_2209_02478_b200.dp import NativeDP
            dp = NativeDP(local, rank, world)
    nccl_bytes = int(allmax(dp.device_bytes(), world)) if dp is not None else 0
    bucket_mb = float(os.environ.get("MIMOSE_DP_BUCKET_MB", "32"))

    # 1. no-checkpoint peaks at S_max: the measured configuration's own
    #    (flash attention: "self") and the materialised-attention model's
    #    (attention probabilities and their dropout output saved, as HF BERT /
    #    GPT-2 and the reference's bert12.model do). The budget is
    #    budget_frac x the --budget-basis one; the other basis is measured too.
    free, total = torch.cuda.mem_get_info()
    ranks_here = max(1, world // max(1, torch.cuda.device_count()))
    probe_budget = int(min(free * 0.85 / ranks_here, 150 * GiB))
    rng = np.random.default_rng(args.seed + 1000 * rank)
    probe_batch = synthetic_task_batch(rng, model_cfg, B, S_max)

    def probe_peak(attn_fused):
        p = Trainer(model_cfg, dataclasses.replace(train_cfg, planner="none", attn_fused=attn_fused),
                    probe_budget, local)
        p.step(*probe_batch, optimizer=False, stream=stream)
        v = int(allmax(p.rows[-1]["peak_reserved"], world))
        p.close()
        return v

    peak_self = probe_peak(train_cfg.attn_fused)
    peak_mat = probe_peak(2) if train_cfg.attn_fused != 2 else peak_self
    bases = {"materialised": peak_mat, "self": peak_self}
    peak_none = bases[args.budget_basis]
    budget = int(args.budget_frac * peak_none)

    n_total = args.warmup + args.steps
    # sizes: reference sampler; 'per-rank' seeds base + rank, 'shared' /
    # 'grouped' seed base ('grouped' then jitters each step's S per rank)
    if args.size_stream == "grouped":
        from paper_2209_02478_b200.dp import rank_sizes_grouped
        seqs = rank_sizes_grouped(args.dist, 10_000, args.seed, rank, args.group_jitter)
    else:
        seqs = sizes_for(args.dist, B, 10_000,
                         args.seed + (rank if args.size_stream == "per-rank" else 0))

    def batches(seq_list, seed):
        g = np.random.default_rng(seed)
        return [synthetic_task_batch(g, model_cfg, B, s) for s in seq_list]

    def allreduce_hook(tr):
        if world == 1 or dp is not None:
            return None
        import torch.distributed as dist
        grads = tr.grads()

        def hook():
            dist.all_reduce(grads)
        return hook

    def timed_run(tr, dev_batches):
        """W warm-up + K timed device-input steps; returns (ms, launches)."""
        hook = allreduce_hook(tr)
        scale = 1.0 / world if hook else 1.0  # native DP averages by itself

        def one(db):
            tr.step_device(db, optimizer=False, stream=stream)
            if hook:
                hook()
            tr.optimizer_step(scale, stream=stream)

        for db in dev_batches[:args.warmup]:
            one(db)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        l0 = lib.mimose_launch_count()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for db in dev_batches[args.warmup:]:
            one(db)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        ms = ev0.elapsed_time(ev1)
        launches = lib.mimose_launch_count() - l0
        return ms, launches

    calib = train_cfg.max_sheltered_iters + 2
    run_seqs = seqs[calib:calib + n_total]
    hb = batches(run_seqs, args.seed + 7 * rank + 2)
    db = [DeviceBatch.from_host(t, ty, lb, model_cfg.vocab) for (t, ty, lb) in hb]
    samples = B * args.steps * world

    def mimose_run(run_budget, clocks=False):
        """Mimose trainer under run_budget: sheltered calibration window, then
        W + K timed steps; returns (trainer, value, ms, launches, summary, clk)."""
        tr = Trainer(model_cfg, dataclasses.replace(train_cfg, planner=args.planner,
                                                    ffn_regen_g=args.ffn_regen_g),
                     run_budget - nccl_bytes, local)
        try:
            if dp is not None:
                tr.attach_dp(dp, bucket_mb)
            t_cal0 = time.perf_counter()
            for b in batches(seqs[:calib], args.seed + 7 * rank + 1):
                tr.step(*b, stream=stream)
            calib_s = time.perf_counter() - t_cal0
            torch.cuda.synchronize()
            clk = None
            if clocks:
                with ClockSampler(local) as clk:
                    ms, launches = timed_run(tr, db)
            else:
                ms, launches = timed_run(tr, db)
        except Exception:
            tr.close()
            raise
        ms = allmax(ms, world)
        rows = tr.rows[-args.steps:]
        over = [r for r in rows if r["peak_reserved"] > r["budget"]]
        pred = [r["pred_err_max"] for r in rows if r["pred_layers"] > 0]
        plan_us = sum(r["plan_us"] + r["fit_us"] for r in rows)
        units = sum(r["plan_size"] for r in rows) / len(rows)
        info = tr.info()
        summary = {
            "budget_bytes": run_budget, "arena_bytes": run_budget - nccl_bytes,
            "max_peak_bytes": max(r["peak_reserved"] for r in rows),
            "steps_over_budget": len(over), "arena_failures": tr.mem_stats()["n_failures"],
            "mem_pred_err_max": max(pred) if pred else None,
            "mem_pred_err_mean": (sum(pred) / len(pred)) if pred else None,
            "planning_overhead_frac": (plan_us / 1000.0) / ms if ms else None,
            "avg_dropped_units": units,
            "avg_dropped_blocks": units / (2 if train_cfg.ckpt_unit == 1 else 1),
            "constant_bytes": info["constant_bytes"], "reserve_bytes_seq_max": info["reserve_bytes"],
            "cache_hits": info["cache_hits"], "cache_misses": info["cache_misses"],
            "calibration_s": calib_s,
        }
        return tr, samples / (ms / 1000.0), ms, launches, summary, clk

    # 2. Mimose under the headline budget. A budget below what even the
    #    all-units-dropped iteration needs (e.g. fp32 master weights + AdamW
    #    state of a 30-50 k vocabulary model >= the fraction of the flash
    #    configuration's own peak) fails in the arena, which refuses to exceed
    #    it: report the configuration as infeasible instead of a number.
    try:
        tr, value, ms_max, launches, summ, clk = mimose_run(budget, clocks=True)
    except _lib.MimoseError as e:
        if world > 1 or "budget exceeded" not in str(e):
            raise
        print(json.dumps({
            "metric": METRIC, "value": None, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "infeasible": str(e)[:300],
            "config": {"workload": PRESET_INFO[args.preset][0], "seq_len": args.dist,
                       "budget_frac_of_no_ckpt_peak": args.budget_frac, "budget_bytes": budget,
                       "budget_basis": args.budget_basis, "no_ckpt_peak_bytes": peak_none}}),
              flush=True)
        return

    # 3. roofline: every instrumented launch timed by CUDA events on 4 extra steps
    #    (their S drawn from the same stream; fewer steps make the family's
    #    efficiency depend on which lengths happened to be drawn)
    extra = batches(seqs[calib + n_total:calib + n_total + 4], args.seed + 99)
    extra_db = [DeviceBatch.from_host(t, ty, lb, model_cfg.vocab) for (t, ty, lb) in extra]
    import ctypes as C
    lib.mimose_profile_enable(1)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for d in extra_db:
        tr.step_device(d, optimizer=True, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    step_ms_prof = e0.elapsed_time(e1)

    def prof(prefix):
        fl, by, pms, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        _lib.check(lib.mimose_profile_read(prefix.encode(), C.byref(fl), C.byref(by),
                                           C.byref(pms), C.byref(n)))
        return fl.value, by.value, pms.value, n.value

    pcsv = C.c_void_p()
    lib.mimose_profile_csv(C.byref(pcsv))
    classes = sorted({l.split(",", 1)[0] for l in _lib.take_string(lib, pcsv).splitlines()[1:]})
    peak_tf = float(pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1400.0)))
    peak_tf_burst = float(pk.get("bf16_tflops", peak_tf))
    peak_bw = float(pk.get("hbm_gbs", 6547.0))
    # dominant kernel family: the dense (projection / FFN / weight-gradient)
    # tcgen05 GEMMs, tensor-bound; every other class against HBM (and the
    # attention kernels also against the tensor burst peak)
    dfl, dby, dms, dn = prof("gemm_dense")
    achieved_tflops = dfl / (dms / 1000.0) / 1e12 if dms > 0 else 0.0
    stages = {}
    for c in classes:
        fl, by, cms, n = prof(c)
        if cms <= 0:
            continue
        st = {"ms_share_of_step": cms / step_ms_prof, "launches": n}
        if c == "gemm_dense":
            st.update(bound="tensor", achieved_tflops=fl / (cms / 1e3) / 1e12,
                      frac=fl / (cms / 1e3) / 1e12 / peak_tf)
        else:
            st.update(bound="hbm", achieved_gbs=by / (cms / 1e3) / 1e9,
                      frac=by / (cms / 1e3) / 1e9 / peak_bw)
            if fl > 0:
                st["achieved_tflops"] = fl / (cms / 1e3) / 1e12
                st["tensor_frac_burst"] = fl / (cms / 1e3) / 1e12 / peak_tf_burst
        stages[c] = st
    lib.mimose_profile_enable(0)  # (clears the records: read everything first)

    # 4. e2e: public API with HOST (pinned) inputs, H2D + loss D2H inside the region.
    #    N=1: mimose_trainer_step_async + mimose_trainer_loss with a one-step lag
    #    (the host issues step i+1 while step i runs; every step's loss is read
    #    back inside the timed region). N>1: forward_backward + all-reduce + AdamW.
    e2e_batches = batches(run_seqs, args.seed + 5)  # same sizes as the device-resident run
    pinned = [tuple(torch.from_numpy(a).pin_memory() for a in b) for b in e2e_batches]
    losses = []

    def e2e_run(group):
        if world == 1 or dp is not None:
            prev = None
            for b in group:
                row = tr.step_async(*b, stream=stream)
                if prev is not None:
                    losses.append(tr.loss(prev))
                prev = row["iter"]
            if prev is not None:
                losses.append(tr.loss(prev))
        else:
            import torch.distributed as dist
            for b in group:
                row = tr.step_pinned(*b, optimizer=False, stream=stream)
                dist.all_reduce(tr.grads())
                tr.optimizer_step(1.0 / world, stream=stream)
                losses.append(row["loss"])

    e2e_run(pinned[:args.warmup])
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    e2e_run(pinned[args.warmup:])
    torch.cuda.synchronize()
    e2e_s = allmax(time.perf_counter() - t0, world)
    e2e_value = samples / e2e_s
    h2d_per_step = sum(x.numel() * 4 for b in pinned[args.warmup:] for x in b) // args.steps
    host_ms = [r["host_ms"] for r in tr.rows[-args.steps:]]
    tr.close()

    # 5. the other budget basis, same size stream (the claim on both bases).
    #    N = 1 only: an infeasible budget fails on each rank at a step that
    #    depends on its own lengths, and a rank leaving the collectives early
    #    would hang the others.
    other = {}
    if not args.profile_only and world == 1:
        ob = "self" if args.budget_basis == "materialised" else "materialised"
        ob_budget = int(args.budget_frac * bases[ob])
        try:
            t2, v2, _, _, s2, _ = mimose_run(ob_budget)
            t2.close()
            other = {"basis": ob, "value": v2, "no_ckpt_peak_bytes": bases[ob], **s2}
        except _lib.MimoseError as e:
            # e.g. QA / LM presets: the constant footprint (weights, grads, AdamW
            # state) alone is >= the fraction of the smaller (flash) peak
            torch.cuda.synchronize()
            other = {"basis": ob, "value": None, "no_ckpt_peak_bytes": bases[ob],
                     "budget_bytes": ob_budget, "infeasible": str(e)[:200]}

    # 6. no-checkpoint, unlimited-memory throughput on the same size stream
    nock = None
    if not args.no_baseline and not args.profile_only:
        base = Trainer(model_cfg, dataclasses.replace(train_cfg, planner="none"),
                       int(max(peak_self, peak_mat) * 1.15) + GiB, local)
        if dp is not None:
            base.attach_dp(dp, bucket_mb)
        ms_none, _ = timed_run(base, db)
        ms_none = allmax(ms_none, world)
        nock = samples / (ms_none / 1000.0)
        base.close()
    if other and nock and other.get("value"):
        other["frac_of_no_ckpt"] = other["value"] / nock

    # 7. CPU baseline (rank 0, N=1 only): bounded sample of the same workload
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile_only:
        threads = os.cpu_count() or 1
        g = np.random.default_rng(1)
        S_s = run_seqs[:3]
        sub = model_cfg.num_choices if model_cfg.head == 0 else 1
        plans, _ = cpu_plans(model_cfg, sub, train_cfg.seq_min, train_cfg.seq_max, S_s,
                             args.budget_frac)
        tot = sum(cpu_step_sample(model_cfg, S, sub, g, threads, ck) for S, ck in zip(S_s, plans))
        cpu = {"value": sub * len(S_s) / tot, "unit": "samples/s", "cores": threads,
               "kind": "port",
               "sample": f"3 steps x {sub} sequence(s) at S={S_s}; oracle/bert_ref.py "
                         f"PyTorch-CPU fp32 fwd+bwd (reference-planned blocks under "
                         f"torch.utils.checkpoint) + AdamW, {threads} threads"}

    timed_S = run_seqs[args.warmup:]
    if rank == 0:
        traffic = traffic_record(args.preset)
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (uniform token ids, N(0,0.02) random-init weights)",
            "config": {
                "workload": PRESET_INFO[args.preset][0],
                "global_batch": B * world, "seq_len": args.dist, "parallelism": f"dp{world}",
                "dp_size_stream": args.size_stream,
                **({"dp_group_jitter": args.group_jitter} if args.size_stream == "grouped" else {}),
                "budget_frac_of_no_ckpt_peak": args.budget_frac, "budget_bytes": budget,
                "no_ckpt_peak_bytes": peak_none, "seed": args.seed,
                "attention": args.attn,
                "ckpt_unit": "block half (attention / FFN)" if train_cfg.ckpt_unit == 1
                             else "transformer block",
                "budget_basis": ("no-ckpt peak of the materialised-attention model at S_max "
                                 "(reference memory semantics)"
                                 if args.budget_basis == "materialised"
                                 else "no-ckpt peak of the measured configuration at S_max"),
                "nccl_bytes_outside_arena": nccl_bytes,
                "timed_seq_lens": {"values": timed_S, "mean": sum(timed_S) / len(timed_S),
                                   "distribution_mean": _dist_mean(args.dist)},
                "l2": "not flushed: per-step working set (GBs of activations) >> 126 MB L2",
                "calibration": f"{calib} planner-calibration steps (sheltered collection window "
                               f"+ fit) run before warm-up, {summ['calibration_s']:.2f} s",
            },
            "roofline": {"bound": "tensor", "achieved": achieved_tflops, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved_tflops / peak_tf,
                         "traffic": traffic["dram_bytes"] if traffic else None,
                         "traffic_detail": traffic,
                         "kernel": "gemm_bf16_tn_kernel (tcgen05) dense GEMMs: QKV / out-proj / "
                                   "FFN forward, dgrad, split-K wgrad",
                         "ms_share_of_step": dms / step_ms_prof if step_ms_prof else None,
                         "launches": dn, "peak_kind": pk_kind + " sustained",
                         "stages": stages, "hbm_peak_gbs": peak_bw,
                         "profiled": "4 extra planned steps, every launch bracketed by CUDA "
                                     "events on its stream; algorithmic flops / bytes per "
                                     "launch (DESIGN.md §2)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d_per_step,
                    "d2h_bytes_per_step": 4,
                    "api": "mimose_trainer_step_async + mimose_trainer_loss (1-step lag)"
                    if world == 1 or dp is not None else
                    "mimose_trainer_forward_backward + NCCL all-reduce + "
                    "mimose_trainer_optimizer_step",
                    "dp": ("native bucketed NCCL all-reduce overlapping backward "
                           f"({bucket_mb:g} MB buckets)") if dp is not None else
                          ("torch.distributed all-reduce after backward" if world > 1 else None),
                    "host_ms_per_step": sum(host_ms) / len(host_ms),
                    "losses_finite": all(l == l for l in losses)},
            "gpu_launches": int(launches),
            "clocks": clk.summary() if clk else None,
            "mimose": {"planner": args.planner, "cache_tolerance": args.cache_tol,
                       "ffn_regen_g": args.ffn_regen_g,
                       "no_ckpt_samples_per_s": nock,
                       "frac_of_no_ckpt": (value / nock) if nock else None,
                       "basis": args.budget_basis, **summ},
            "mimose_other_basis": other or None,
        }
        print(json.dumps(line), flush=True)
    if dp is not None:
        dp.close()


def _dist_mean(dist):
    f = dist.split(":")
    if f[0] == "uniform":
        return (float(f[1]) + float(f[2])) / 2
    if f[0] == "normal":
        return float(f[1])
    return None


def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", 0))
        world = int(os.environ.get("WORLD_SIZE", args.gpus))
        run_reference_arm(args, rank, world)
        return
    rank, world, local = dist_init(args.gpus)
    run_gpu_arm(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
