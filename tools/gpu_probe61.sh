#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python bench.py --precision fp64 --no-cpu-baseline --steps 2 --warmup 3 --e2e-shots 1000 > $out/p61_bench128.json 2> $out/p61.err
QG_KW="dict()" timeout 300 python - >> $out/p61.txt 2>&1 <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays
for n in (30, 31):
    gt, gp = random_arrays(RandomSpec(n, 1000, 0))
    for cfg in (0, 1):
        try:
            plan = sv.CompiledCircuit(gt, gp, n, "fp64", jit=1, kernel_cfg=cfg)
        except Exception as e:
            print(n, cfg, "ERR", e); continue
        js = plan.jit_status(wait=True)
        st = sv.init_zero_state(n, "fp64", 1 << 40)
        plan.execute(st); torch.cuda.synchronize()
        best = min(plan.execute(st, timed=True).pass_ms for _ in range(2))
        S = (1 << n) * 16
        print(n, "cfg", cfg, "passes", plan.info["n_passes"], "jit", js["n_jit"], "ms", round(best, 1),
              "ms/pass", round(best / plan.info["n_passes"], 3), "GB/s", round(2 * S * plan.info["n_passes"] / best / 1e6), flush=True)
PY
echo done
