"""Regenerates tests/golden/planner_golden.json from the REFERENCE planner.

Runs in the build container only (needs /root/reference): compiles the
unmodified reference headers through oracle/Makefile into
oracle/_ref/libmimose_ref.so and records its outputs on fixed inputs. The
fixture is then the pinned truth for the product planner (include/mimose via
libmimose_host.so) and for the C restatement (oracle/planner_oracle.c), on
boxes where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

REF_MODELS = "/root/reference/proj/models"
OUT = os.path.join(HERE, "planner_golden.json")


def splitmix64(z):
    M = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def noise_delta(eps, seed, layer, x):
    """reference collector.hpp:34-46 NoiseModel::delta, restated."""
    M = (1 << 64) - 1
    if eps == 0.0:
        return 0.0
    h = splitmix64(seed ^ splitmix64((layer & M) ^ splitmix64(x & M)))
    u = float(h >> 11) * 2.0 ** -53
    return eps * (2.0 * u - 1.0)


def parse_model(text):
    layers = []
    cur = None
    head = {}
    for line in text.splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line == "[layer]":
            cur = {}
            layers.append(cur)
            continue
        k, v = [s.strip() for s in line.split(":", 1)]
        (cur if cur is not None else head)[k] = v
    return head, layers


def samples_csv(model_text, xs, eps=0.0, seed=0):
    from oracle.planner_oracle import llround
    _, layers = parse_model(model_text)
    rows = ["layer_id,input_size,bytes,ms,valid"]
    for x in xs:
        for l in layers:
            a = [float(v) for v in l["activation_coeffs"].split()]
            t = [float(v) for v in l["forward_time_coeffs"].split()]
            xf = float(x)
            act = llround(a[0] + a[1] * xf + a[2] * xf * xf)
            meas = llround(float(act) * (1.0 + noise_delta(eps, seed, int(l["id"]), x)))
            ms = t[0] + t[1] * xf
            rows.append(f"{l['id']},{x},{meas},{repr(ms)},1")
    return "\n".join(rows) + "\n"


def main():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/libmimose_ref.so"],
                   check=True)
    from paper_2209_02478_b200.planner import PlannerLib, SchedCfg
    from oracle.planner_oracle import REF_LIB
    ref = PlannerLib(REF_LIB, "ref_planner_")
    models = {}
    for name in ("bert12", "heterostage"):
        with open(os.path.join(REF_MODELS, name + ".model")) as f:
            models[name] = f.read()

    g = {"generator": "tests/golden/make_golden.py (reference planner compiled from "
                      "/root/reference/proj/include via oracle/Makefile)",
         "models": models, "workloads": [], "fits": [], "plans": [], "simulate": [],
         "experiments": []}

    for dist, mult, iters, seed in [("uniform:30:332", 1, 10, 7), ("uniform:30:332", 32, 200, 11),
                                    ("normal:180:60:30:332", 32, 200, 2024),
                                    ("powerlaw:1.5:30:332", 32, 200, 3),
                                    ("powerlaw:1:30:332", 32, 50, 5),
                                    ("uniform:64:512", 1, 300, 2024),
                                    ("normal:300:100:153:512", 12, 100, 9)]:
        g["workloads"].append({"dist": dist, "mult": mult, "iters": iters, "seed": seed,
                               "xs": ref.workload(dist, mult, iters, seed)})

    for name, xs, eps, seed, order in [
            ("bert12", [960 + i * 1024 for i in range(10)], 0.0, 0, 2),
            ("bert12", [960 + i * 1024 for i in range(10)], 0.01, 2024, 2),
            ("heterostage", [1000, 2500, 4000, 5500, 7000, 8500, 10000], 0.0, 0, 2),
            ("heterostage", [1000, 4000, 7000, 10000], 0.02, 77, 1),
            ("bert12", [960, 5000, 10624], 0.0, 0, 2)]:
        csv = samples_csv(models[name], xs, eps, seed)
        g["fits"].append({"model": name, "order": order, "samples_csv": csv,
                          "estimator": ref.fit_text(csv, order)})

    for fit_i, budget, reserve, btol, ctol, xs in [
            (0, 6 << 30, -1, 0.10, 0.0, [10624, 960, 4096, 10624, 7000, 4096]),
            (1, 6 << 30, -1, 0.10, 0.02, [10624, 10500, 9000, 8900, 4096, 4000, 4100]),
            (2, 3 << 30, -1, 0.10, 0.0, [1000, 5500, 10000, 10000, 3000]),
            (2, 2 << 30, 0, 0.30, 0.05, [1000, 5500, 10000, 9800, 3000]),
            (0, 2 << 30, -1, 0.10, 0.0, [10624, 8000])]:
        f = g["fits"][fit_i]
        cfg = SchedCfg(budget_bytes=budget, reserve_bytes=reserve, bucket_tolerance=btol,
                       cache_tolerance=ctol)
        masks, ins, hits = ref.plan_seq(f["estimator"], models[f["model"]], cfg, xs, 64)
        g["plans"].append({"fit": fit_i, "budget": budget, "reserve": reserve,
                           "bucket_tolerance": btol, "cache_tolerance": ctol, "xs": xs,
                           "masks": masks, "insufficient": ins, "hits": hits})

    for name, dropped, x in [("bert12", [], 10624), ("bert12", list(range(9)), 10624),
                             ("bert12", [11], 960), ("heterostage", [1, 3, 7], 5000),
                             ("heterostage", list(range(8)), 10624)]:
        peak, it, rc = ref.simulate_plan(models[name], dropped, x)
        g["simulate"].append({"model": name, "dropped": dropped, "x": x, "peak": peak,
                              "iteration_ms": it, "recompute_ms": rc})

    for name, dist, mult, iters, seed, budget, planner in [
            ("bert12", "normal:180:60:30:332", 32, 300, 2024, 6 << 30, "mimose"),
            ("bert12", "normal:180:60:30:332", 32, 300, 2024, 6 << 30, "static-max"),
            ("bert12", "normal:180:60:30:332", 32, 300, 2024, 6 << 30, "dtr"),
            ("heterostage", "uniform:30:332", 32, 200, 1, 3 << 30, "mimose"),
            ("bert12", "uniform:30:332", 32, 100, 4, 16 << 30, "none")]:
        cfg = SchedCfg(budget_bytes=budget)
        summary, csv = ref.experiment(models[name], dist, mult, iters, seed, cfg, planner)
        g["experiments"].append({"model": name, "dist": dist, "mult": mult, "iters": iters,
                                 "seed": seed, "budget": budget, "planner": planner,
                                 "summary": summary,
                                 "csv_sha256": hashlib.sha256(csv.encode()).hexdigest()})

    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        OUT = sys.argv[1]
    main()
