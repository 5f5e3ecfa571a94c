"""The GPU command-line front end (paper_2209_02478_b200/cli/mimose_gpu.cpp)
keeps the reference CLI's subcommands, flags and exit codes
(reference proj/tools/mimose_main.cpp:22-24, 254-319) and writes its reports
with the reference's writers (harness.hpp:339-379).

CPU: argument handling, exit codes, and gen-workload against the reference's
own CLI check (proj/tests/cli_checks.cmake:19-33: seed 7 -> "186 ...").
GPU: `run` / `compare` / `fit` on a real B200 with the reference's flags; the
planner-determined fields of the GPU report (phases, cache hits, plans,
fit point) equal the reference harness replaying the GPU-measured profile
(run_experiment over the dumped .model document) field for field."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2209_02478_b200")


@pytest.fixture(scope="module")
def cli(tmp_path_factory):
    """Build the CLI against the in-tree libraries (g++, no CUDA compiler)."""
    if not os.path.exists(os.path.join(PKG, "libmimose_cuda.so")):
        pytest.skip("libmimose_cuda.so not built (make)")
    out = str(tmp_path_factory.mktemp("cli") / "mimose_gpu")
    cuda = os.path.dirname(os.path.dirname(shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"))
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-Werror",
           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(cuda, "include"),
           os.path.join(PKG, "cli", "mimose_gpu.cpp"), "-o", out,
           "-L" + PKG, "-lmimose_cuda", "-lmimose_host", "-L" + os.path.join(cuda, "lib64"),
           "-lcudart", "-Wl,-rpath," + PKG, "-Wl,-rpath," + os.path.join(cuda, "lib64")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def run(cli, *args, cwd=None):
    p = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, cwd=cwd,
                       timeout=900)
    return p.returncode, p.stdout, p.stderr


# ------------------------------------------------------------------ CPU
def test_gen_workload_reference_golden(cli, tmp_path):
    # cli_checks.cmake:19-33: deterministic per seed, golden head 186
    for name in ("a", "b"):
        code, _, err = run(cli, "gen-workload", "--dist", "uniform:30:332", "--seed", 7,
                           "--iters", 10, "--batch-multiplier", 1, "--out", f"wl_{name}.txt",
                           cwd=tmp_path)
        assert code == 0, err
    a = (tmp_path / "wl_a.txt").read_text()
    assert a == (tmp_path / "wl_b.txt").read_text()
    # the full sequence of reference tests/test_harness.cpp:31-40
    assert [int(v) for v in a.split()] == [186, 33, 231, 147, 133, 195, 57, 43, 234, 104]
    # --batch-multiplier scales sizes into elements (workload.hpp)
    code, out, _ = run(cli, "gen-workload", "--dist", "uniform:30:332", "--seed", 7, "--iters", 3,
                       "--batch-multiplier", 64)
    assert code == 0 and [int(v) for v in out.split()] == [186 * 64, 33 * 64, 231 * 64]


def test_exit_codes_and_flag_errors(cli):
    assert run(cli)[0] == 1                                   # no subcommand
    assert run(cli, "--help")[0] == 0
    assert run(cli, "frobnicate")[0] == 1                     # unknown subcommand
    assert run(cli, "run", "--bogus", 1)[0] == 1              # unknown flag
    assert run(cli, "run", "--iters")[0] == 1                 # missing value
    assert run(cli, "run", "--format", "xml")[0] == 1         # bad report format
    assert run(cli, "run", "--planner", "greedy", "--iters", 0)[0] == 1
    assert run(cli, "run", "--budget", "6q", "--iters", 0)[0] == 1   # bad byte suffix
    assert run(cli, "gen-workload", "--dist", "zipf:1:2")[0] == 1
    # host-only subcommands point at the reference CLI
    code, _, err = run(cli, "simulate", "--model", "x.model", "--x", 10)
    assert code == 1 and "reference CLI" in err


# ------------------------------------------------------------------ GPU
def _summary(text):
    out = {}
    for line in text.splitlines():
        k, _, v = line.partition(": ")
        out[k] = v
    return out


def _rows(csv):
    lines = csv.strip().splitlines()
    head = lines[0].split(",")
    return head, [dict(zip(head, ln.split(","))) for ln in lines[1:]]


COMMON = ["--model", "small4-h256", "--dist", "uniform:32:256", "--batch-multiplier", 64]


@pytest.mark.gpu
def test_run_matches_reference_replay_of_measured_profile(cli, cuda_device, tmp_path):
    from paper_2209_02478_b200 import planner
    # no-checkpoint peak at S_max -> a budget that forces drops
    code, out, err = run(cli, "run", "--planner", "none", "--budget", "6g", "--iters", 1,
                         "--dist", "uniform:256:256", "--model", "small4-h256",
                         "--batch-multiplier", 64, "--format", "summary")
    assert code == 0, err
    peak = int(float(_summary(out)["mean_peak_bytes"]))
    budget = int(0.6 * peak)
    # one automatic reserve for every size, so the reference can replay the
    # plans with the same (budget, reserve) pair
    args = ["run", *COMMON, "--planner", "mimose", "--budget", budget, "--reserve", "auto",
            "--seed", 13, "--iters", 40]
    code, csv_a, err = run(cli, *args, "--format", "csv", "--out", "a.csv",
                           "--dump-model", "gpu.model", "--dump-estimator", "gpu.est",
                           cwd=tmp_path)
    assert code == 0, err
    code, _, err = run(cli, *args, "--format", "summary", "--out", "a.txt", cwd=tmp_path)
    assert code == 0, err
    head, rows = _rows((tmp_path / "a.csv").read_text())
    assert head == ["iter", "x", "planner", "cache_hit", "peak_bytes", "iteration_ms",
                    "recompute_ms", "sheltered", "plan_size", "insufficient"]
    assert len(rows) == 40
    assert max(int(r["plan_size"]) for r in rows if r["sheltered"] == "0") > 0  # budget binds
    assert all(int(r["peak_bytes"]) <= budget for r in rows)                     # measured
    gpu = _summary((tmp_path / "a.txt").read_text())
    assert int(gpu["oom_risk_iterations"]) == 0

    # the reference harness replaying the GPU-measured profile, same flags
    model_text = (tmp_path / "gpu.model").read_text()
    ref_sum, ref_csv = planner.host_lib().experiment(
        model_text, "uniform:32:256", 64, 40, 13,
        planner.SchedCfg(budget_bytes=budget, reserve_bytes=int(gpu["reserve_bytes"])), "mimose")
    ref = _summary(ref_sum)
    _, ref_rows = _rows(ref_csv)
    for k in ("iterations", "budget_bytes", "reserve_bytes", "planner_invocations",
              "collector_iterations", "sheltered_iterations", "fallback_sheltered_iterations",
              "cache_hits", "cache_misses", "distinct_sizes", "insufficient_budget_iterations",
              "fit_order", "fit_at_iter"):
        assert gpu[k] == ref[k], (k, gpu[k], ref[k])
    for g, r in zip(rows, ref_rows):
        for k in ("iter", "x", "planner", "cache_hit", "sheltered", "plan_size", "insufficient"):
            assert g[k] == r[k], (g["iter"], k, g[k], r[k])


@pytest.mark.gpu
def test_compare_fit_and_infeasible_exit(cli, cuda_device, tmp_path):
    # compare: the reference's grid CSV over planners x budgets
    code, out, err = run(cli, "compare", *COMMON, "--budgets", "2g,3g", "--planners",
                         "mimose,static-max,dtr,none", "--iters", 12, "--seed", 5)
    assert code == 0, err
    lines = out.strip().splitlines()
    assert lines[0].startswith("planner,budget_bytes,total_time_ms,mean_peak_bytes")
    assert [ln.split(",")[0] for ln in lines[1:]] == ["mimose", "static-max", "dtr", "none"] * 2
    assert [int(ln.split(",")[1]) for ln in lines[1:]] == [2 << 30] * 4 + [3 << 30] * 4
    # every cell ran all 12 iterations inside its budget (oom_risk column 0)
    assert all(ln.split(",")[8] == "0" for ln in lines[1:])
    # fit: GPU-measured samples in the reference CSV format + an estimator dump
    code, _, err = run(cli, "fit", *COMMON, "--seed", 3, "--iters", 12, "--budget", "2g",
                       "--dump-estimator", "est.txt", "--dump-samples", "samples.csv",
                       cwd=tmp_path)
    assert code == 0, err
    assert (tmp_path / "samples.csv").read_text().startswith("layer_id,input_size,bytes,ms,valid")
    assert (tmp_path / "est.txt").stat().st_size > 0
    assert "distinct_sizes:" in err
    # a budget below the constant footprint (weights + grads + AdamW state,
    # ~0.2 GB here) is infeasible -> exit 2, as the reference's insufficient plans
    code, out, err = run(cli, "run", *COMMON, "--planner", "mimose", "--budget", "64m",
                         "--iters", 14, "--seed", 13, "--format", "summary")
    assert code == 2, (code, out, err)
    # in a grid the infeasible cell is an empty row, the others still run
    code, out, err = run(cli, "compare", *COMMON, "--budgets", "64m,2g", "--planners", "mimose",
                         "--iters", 12, "--seed", 5)
    assert code == 2, (code, out, err)
    rows = [ln.split(",") for ln in out.strip().splitlines()[1:]]
    assert [r[1] for r in rows] == [str(64 << 20), str(2 << 30)]
    assert rows[0][2] == "" and rows[1][2] != ""
