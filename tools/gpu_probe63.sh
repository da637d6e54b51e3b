#!/bin/bash
# complex128: default JIT (k=13, 32 amps, 1 CTA/SM) vs k=12 / 16 amps / 2 CTAs/SM (dev knob)
out=gpurun_out; mkdir -p $out
QG_DEV_JIT_CFG0=1 timeout 600 python - > $out/p63.txt 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays, qft_arrays
for n in (28, 30, 32):
    gt, gp = random_arrays(RandomSpec(n, 1000, 0))
    ref = None
    for cfg in (0, 1):
        plan = sv.CompiledCircuit(gt, gp, n, "fp64", jit=1, kernel_cfg=cfg)
        js = plan.jit_status(wait=True)
        st = sv.init_zero_state(n, "fp64", 1 << 40)
        plan.execute(st); torch.cuda.synchronize()
        a = st.amplitudes[:1 << 20].clone()
        best = min(plan.execute(st, timed=True).pass_ms for _ in range(2))
        if ref is None: ref = a
        d = (a - ref).abs().max().item()
        S = (1 << n) * 16
        print(n, "cfg", cfg, "passes", plan.info["n_passes"], "jit", js["n_jit"], "ms", round(best, 1),
              "ms/pass", round(best / plan.info["n_passes"], 3), "frac", round(2 * S * plan.info["n_passes"] / best / 1e6 / 6471.4, 3),
              "maxdiff_vs_cfg0", f"{d:.2e}", flush=True)
        del st, plan
        torch.cuda.empty_cache()
PY
echo done
