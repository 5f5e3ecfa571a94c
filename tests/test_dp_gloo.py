"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel host
logic: per-rank size streams, per-rank plans from the host planner, the flat
gradient all-reduce + 1/world scaling, and max-over-ranks timing."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2209_02478_b200 import dp, planner
        # 1. per-rank variable-length streams (seed = base + rank)
        seqs = dp.rank_sizes("uniform:64:512", 50, 2024, rank)
        # 2. per-rank plans from the host planner for each rank's own sizes
        import json
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "planner_golden.json")))
        f = g["fits"][0]
        cfg = planner.SchedCfg(budget_bytes=6 << 30)
        xs = [32 * (30 + (s - 64) * 302 // 448) for s in seqs[:10]]  # onto bert12 range
        masks, _, _ = planner.host_lib().plan_seq(f["estimator"], g["models"]["bert12"], cfg, xs, 12)
        # 3. gradient all-reduce on a flat fp32 buffer + 1/world scaling
        grads = torch.full((1000,), float(rank + 1))
        dpt = dp.DataParallelTrainer(trainer=None, world=world, rank=rank)
        dpt._allreduce(grads)
        scaled = grads * (1.0 / world)
        # 4. max over ranks
        mx = dp.max_over_ranks(10.0 * (rank + 1))
        out_q.put((rank, seqs, masks, scaled[:3].tolist(), mx))
    finally:
        dist.destroy_process_group()


def test_data_parallel_host_logic_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (s0, m0, g0, mx0), (s1, m1, g1, mx1) = res[0], res[1]
    from paper_2209_02478_b200 import planner
    assert s0 == [int(x) for x in planner.host_lib().workload("uniform:64:512", 1, 50, 2024)]
    assert s1 == [int(x) for x in planner.host_lib().workload("uniform:64:512", 1, 50, 2025)]
    assert s0 != s1                      # ranks draw different lengths
    assert m0 != m1                      # ... and therefore plan differently
    assert g0 == g1 == [1.5, 1.5, 1.5]   # (1 + 2) / 2 on both ranks
    assert mx0 == mx1 == 20.0            # step time = slowest rank


def test_length_grouped_rank_sizes():
    """bench.py's default DP length policy: each rank its own S inside the
    step's length group (the shared reference stream), +-jitter, clamped."""
    from paper_2209_02478_b200 import dp, planner
    shared = planner.host_lib().workload("uniform:64:512", 1, 200, 2024)
    ranks = [dp.rank_sizes_grouped("uniform:64:512", 200, 2024, r, 0.05) for r in range(8)]
    assert ranks[3] == dp.rank_sizes_grouped("uniform:64:512", 200, 2024, 3, 0.05)  # deterministic
    for r in ranks:
        assert all(64 <= s <= 512 for s in r)
        assert all(abs(s - g) <= 0.05 * g + 1 for s, g in zip(r, shared))
    # ranks differ (own mini-batch lengths) but stay grouped: the step's
    # longest rank is within ~5-8 % of its mean (independent streams: ~1.6x)
    assert any(ranks[0][i] != ranks[1][i] for i in range(200))
    spread = [max(r[i] for r in ranks) / (sum(r[i] for r in ranks) / 8) for i in range(200)]
    assert max(spread) < 1.08
