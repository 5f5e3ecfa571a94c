import sys, os, dataclasses, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2209_02478_b200.trainer import PRESETS, Trainer, synthetic_task_batch
for name in sys.argv[1:]:
    m, t = PRESETS[name]
    for af in (2, 3):
        for unit in (0, 1):
            tr = Trainer(m, dataclasses.replace(t, planner="none", attn_fused=af, ckpt_unit=unit), 60 << 30)
            r = tr.step(*synthetic_task_batch(np.random.default_rng(0), m, t.batch, t.seq_max), optimizer=False)
            print(json.dumps({"preset": name, "attn_fused": af, "unit": unit, "peak": r["peak_reserved"], "const": tr.info()["constant_bytes"]}), flush=True)
            tr.close()
