"""Planner parity (CPU): product host planner vs the reference's golden vectors.

Three implementations are compared on the same inputs:
  * product   - include/mimose/*.hpp through libmimose_host.so (what the B200
                trainer links);
  * C oracle  - oracle/planner_oracle.c, a plain-C restatement;
  * reference - the unmodified reference headers compiled by oracle/Makefile
                (only where /root/reference exists; its outputs are frozen in
                tests/golden/planner_golden.json by tests/golden/make_golden.py).
The bar is bit-exact: identical integers, identical text dumps.
"""
import json
import os
import random

import pytest

from conftest import REFERENCE, ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden", "planner_golden.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def host():
    from paper_2209_02478_b200 import planner
    return planner.host_lib()


@pytest.fixture(scope="module")
def orc():
    from oracle import planner_oracle
    planner_oracle.lib()
    return planner_oracle


def _cfg(p):
    from paper_2209_02478_b200.planner import SchedCfg
    return SchedCfg(budget_bytes=p["budget"], reserve_bytes=p["reserve"],
                    bucket_tolerance=p["bucket_tolerance"], cache_tolerance=p["cache_tolerance"])


# ------------------------------------------------------------ hand goldens
def test_reference_test_goldens_workload(host, orc):
    # reference proj/tests/test_harness.cpp:31-40 (and cli_checks.cmake:30)
    want = [186, 33, 231, 147, 133, 195, 57, 43, 234, 104]
    assert host.workload("uniform:30:332", 1, 10, 7) == want
    assert orc.sample_workload("uniform:30:332", 1, 10, 7) == want


def test_reference_test_goldens_scheduler(orc):
    # test_scheduler.cpp:13-24: 12 x (a=100), budget 950, reserve 0 -> {0,1,2}
    assert orc.generate_plan([100] * 12, list(range(12)), 950, reserve=0) == ([0, 1, 2], False)
    # :36-50 a bucket that covers the excess alone wins -> {4}
    assert orc.generate_plan([100, 100, 100, 100, 200], list(range(5)), 450, reserve=0) == ([4], False)
    # :52-61 insufficient -> flagged, all layers
    assert orc.generate_plan([100] * 4, list(range(4)), 900, reserve=0, constant=1000) == \
        ([0, 1, 2, 3], True)
    # :26-33 no excess -> empty plan
    assert orc.generate_plan([100] * 12, list(range(12)), 1700, reserve=0, constant=500) == ([], False)


def test_reference_test_goldens_simulator(orc):
    # test_simulator.cpp:35-90
    act, bnd, fwd = [10, 20, 30], [1, 1, 1], [5.0, 5.0, 5.0]
    assert orc.simulate(act, bnd, fwd, [], 0)[:2] == (60, 45.0)
    assert orc.simulate(act, bnd, fwd, [2], 0)[:2] == (60, 50.0)
    h_act, h_bnd, h_fwd = [100] * 12, [10] * 12, [5.0] * 12
    assert orc.simulate(h_act, h_bnd, h_fwd, [0], 0)[0] == 1110
    assert orc.simulate(h_act, h_bnd, h_fwd, [11], 0)[0] == 1200
    assert orc.simulate(h_act, h_bnd, h_fwd, [], 500)[0] == 1700
    assert orc.simulate(h_act, h_bnd, h_fwd, list(range(12)), 0)[0] == 210


def test_reference_test_goldens_estimator(orc):
    # test_estimator.cpp:25-35: three points of 2 + 3x + 0.5x^2 -> (2, 3, 0.5)
    xs = [10, 20, 30]
    ys = [orc.layer_bytes((2, 3, 0.5), x) for x in xs]
    c = orc.fit_layer(xs, ys, 2)
    assert abs(c[0] - 2.0) <= 1e-9 and abs(c[1] - 3.0) <= 3e-9 and abs(c[2] - 0.5) <= 5e-10


# ------------------------------------------------------------ frozen reference outputs
def test_workloads_match_reference(golden, host, orc):
    for w in golden["workloads"]:
        assert host.workload(w["dist"], w["mult"], w["iters"], w["seed"]) == w["xs"], w["dist"]
        assert orc.sample_workload(w["dist"], w["mult"], w["iters"], w["seed"]) == w["xs"], w["dist"]


def test_fits_match_reference_bit_exact(golden, host):
    for f in golden["fits"]:
        assert host.fit_text(f["samples_csv"], f["order"]) == f["estimator"]


def _est_coeffs(text):
    out = {}
    for line in text.splitlines():
        if line.startswith("layer:"):
            v = line.split(":", 1)[1].split()
            out[int(v[0])] = [float(t) for t in v[5:]]
    return out


def test_c_oracle_fit_matches_reference(golden, orc):
    for f in golden["fits"]:
        per = {}
        for row in f["samples_csv"].strip().splitlines()[1:]:
            lid, x, b, _, _ = row.split(",")
            per.setdefault(int(lid), ([], []))
            per[int(lid)][0].append(int(x))
            per[int(lid)][1].append(int(b))
        ref = _est_coeffs(f["estimator"])
        for lid, (xs, ys) in per.items():
            assert orc.fit_layer(xs, ys, f["order"]) == ref[lid]


def test_plans_match_reference_bit_exact(golden, host, orc):
    for p in golden["plans"]:
        f = golden["fits"][p["fit"]]
        model = golden["models"][f["model"]]
        masks, ins, hits = host.plan_seq(f["estimator"], model, _cfg(p), p["xs"], 64)
        assert (masks, ins, hits) == (p["masks"], p["insufficient"], p["hits"])
        # C oracle (no cache): generate_plan from the same predictions
        if p["cache_tolerance"] == 0.0:
            coeffs = _est_coeffs(f["estimator"])
            const = int([l for l in model.splitlines() if l.startswith("constant_footprint")][0]
                        .split(":")[1])
            for x, m, i in zip(p["xs"], p["masks"], p["insufficient"]):
                est = [orc.predict(coeffs[l], x) for l in sorted(coeffs)]
                d, flag = orc.generate_plan(est, list(range(len(est))), p["budget"],
                                            reserve=p["reserve"], tol=p["bucket_tolerance"],
                                            constant=const)
                assert sum(1 << k for k in d) == m and int(flag) == i


def test_simulation_matches_reference(golden, host):
    for s in golden["simulate"]:
        peak, it, rc = host.simulate_plan(golden["models"][s["model"]], s["dropped"], s["x"])
        assert (peak, it, rc) == (s["peak"], s["iteration_ms"], s["recompute_ms"])


def test_experiments_match_reference(golden, host):
    import hashlib
    from paper_2209_02478_b200.planner import SchedCfg
    for e in golden["experiments"]:
        summary, csv = host.experiment(golden["models"][e["model"]], e["dist"], e["mult"],
                                       e["iters"], e["seed"], SchedCfg(budget_bytes=e["budget"]),
                                       e["planner"])
        assert summary == e["summary"], e["planner"]
        assert hashlib.sha256(csv.encode()).hexdigest() == e["csv_sha256"]


# ------------------------------------------------------------ randomised vs compiled reference
@pytest.mark.skipif(not os.path.isdir(os.path.join(REFERENCE, "proj", "include")),
                    reason="reference not mounted")
def test_randomised_plans_vs_compiled_reference(host):
    import subprocess
    from oracle.planner_oracle import REF_LIB
    from paper_2209_02478_b200.planner import PlannerLib, SchedCfg
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/libmimose_ref.so"],
                   check=True, capture_output=True)
    ref = PlannerLib(REF_LIB, "ref_planner_")
    rng = random.Random(1234)
    for trial in range(60):
        L = rng.randint(1, 24)
        lines = ["version: 1", f"constant_footprint: {rng.randint(0, 10**9)}",
                 "input_range: 100 20000"]
        samples = ["layer_id,input_size,bytes,ms,valid"]
        sizes = sorted(rng.sample(range(100, 20001), rng.randint(3, 12)))
        for l in range(L):
            c0 = rng.uniform(1e5, 1e7)
            c1 = rng.choice([0.0, rng.uniform(10, 5e4)])
            c2 = rng.choice([0.0, rng.uniform(0.01, 5.0)])
            cat = "quadratic-structure" if c2 > 0 else ("fixed-output" if c1 == 0 else "implicit-reduction")
            b1 = min(c1, rng.uniform(1, 3000)) if c1 > 0 else 0.0
            b0 = 0.5 * c0 if b1 == 0 else 0.0
            lines += ["", "[layer]", f"id: {l}", f"position: {l}", f"stage: {l % 3}",
                      f"category: {cat}", f"activation_coeffs: {c0!r} {c1!r} {c2!r}",
                      f"boundary_coeffs: {b0!r} {b1!r}", "forward_time_coeffs: 1 0.0001"]
            for x in sizes:
                y = int(round(c0 + c1 * x + c2 * x * x) * (1 + rng.uniform(-0.02, 0.02)))
                samples.append(f"{l},{x},{y},{rng.uniform(0.1, 5)!r},1")
        model = "\n".join(lines) + "\n"
        csv = "\n".join(samples) + "\n"
        order = rng.choice([0, 1, 2, 2, 3])
        if len(sizes) < order + 1:
            order = len(sizes) - 1
        est_h = host.fit_text(csv, order)
        assert est_h == ref.fit_text(csv, order)
        total = sum(1e7 + 5e4 * 20000 + 5.0 * 20000 ** 2 for _ in range(L))
        cfg = SchedCfg(budget_bytes=int(rng.uniform(0.05, 1.0) * total) + 10**9,
                       reserve_bytes=rng.choice([-1, 0, 10**6]),
                       bucket_tolerance=rng.choice([0.0, 0.1, 0.3]),
                       cache_tolerance=rng.choice([0.0, 0.02, 0.1]))
        xs = [rng.randint(100, 20000) for _ in range(25)]
        xs += xs[:5]
        assert host.plan_seq(est_h, model, cfg, xs, L) == ref.plan_seq(est_h, model, cfg, xs, L)
        dropped = sorted(rng.sample(range(L), rng.randint(0, L)))
        for x in xs[:5]:
            assert host.simulate_plan(model, dropped, x) == ref.simulate_plan(model, dropped, x)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REFERENCE, "proj", "include")),
                    reason="reference not mounted")
def test_golden_fixture_is_current(golden):
    """The committed fixture equals what the reference produces today."""
    import subprocess
    import sys
    import tempfile
    env = dict(os.environ)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "g.json")
        subprocess.run([sys.executable, os.path.join(ROOT, "tests", "golden", "make_golden.py"),
                        out], check=True, capture_output=True, env=env, cwd=ROOT)
        with open(out) as f:
            fresh = json.load(f)
    assert fresh == golden
