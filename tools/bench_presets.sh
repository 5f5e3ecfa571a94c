# bench line per BASELINE config preset (N=1); outputs gpurun_out/bench_<preset>.json
set -u
for P in ${PRESETS:-gpt2-medium-lm bert-large-mlm roberta-large-qa roberta-base-qa small4-h256}; do
  timeout 900 python bench.py --preset $P --no-cpu > gpurun_out/bench_$P.log 2>&1
  tail -1 gpurun_out/bench_$P.log > gpurun_out/bench_$P.json
  python - "$P" <<'PY'
import json, sys
p = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{p}.json"))
    m = d["mimose"]
    print(p, round(d["value"], 1), d["unit"], "e2e", round(d["e2e"]["value"], 1), "frac_nock",
          round(m["frac_of_no_ckpt"] or 0, 3), "over", m["steps_over_budget"], "pred_err",
          m["mem_pred_err_max"], "roof", round(d["roofline"]["frac"], 3), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(p, "FAILED", e)
PY
done
