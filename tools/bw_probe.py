"""HBM bandwidth of one fused pass vs the tile's qubit layout (dev probe): the
pass applies one H per listed qubit, so its time is the tile's memory pattern."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402

n = 32
cases = {
    "contig0-12": [12],
    "hi8": [31, 30, 29, 28, 27, 26, 25, 24],
    "mid8": [20, 17, 15, 13, 11, 9, 7, 5],
    "lo3_hi5": [5, 6, 7, 31, 29, 27, 25, 23],
    "lo5_hi3": [5, 6, 7, 8, 9, 31, 27, 23],
    "r256_q10-17": list(range(10, 18)),     # 256 B runs, all in one 2 MB page per tile
    "r256_q18-25": list(range(18, 26)),     # 256 B runs, 256 pages per tile, 512 MB span
    "r256_q6-20even": [6, 8, 10, 12, 14, 16, 18, 20],
    "r512_q24-31": [5] + list(range(25, 32)),
    "r256_q20-27": list(range(20, 28)),
    "r256_q22-29": list(range(22, 30)),
    "r256_q23-30": list(range(23, 31)),
    "r256_q24-31": list(range(24, 32)),
    "r256_q16-19_28-31": [16, 17, 18, 19, 28, 29, 30, 31],
    "r256_q8-11_28-31": [8, 9, 10, 11, 28, 29, 30, 31],
    "r256_q12-17_30-31": [12, 13, 14, 15, 16, 17, 30, 31],
    "r256_q19-26": list(range(19, 27)),
    "r256_q21-28": list(range(21, 29)),
    "r256_q20-23_28-31": [20, 21, 22, 23, 28, 29, 30, 31],
    "r256_q12-15_24-27": [12, 13, 14, 15, 24, 25, 26, 27],
    "r256_odd13-27": [13, 15, 17, 19, 21, 23, 25, 27],
    "r256_q6_q25-31": [6] + list(range(25, 32)),
    "r256_q7_q25-31": [7] + list(range(25, 32)),
    "r256_q10_q25-31": [10] + list(range(25, 32)),
}
import os
only = os.environ.get("QG_BW_CASES")
if only:
    cases = {k: v for k, v in cases.items() if k in only.split(",")}
state = sv.init_zero_state(n, "fp32", 1 << 40)
for name, qs in cases.items():
    for jit in (1,):
        gt = np.array([[0, -1, q] for q in qs], dtype=np.int32)
        gp = np.zeros(len(qs))
        plan = sv.CompiledCircuit(gt, gp, n, "fp32", jit=jit)
        plan.jit_status(wait=True)
        plan.execute(state)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            best = min(best, plan.execute(state, timed=True).pass_ms)
        S = (1 << n) * 8
        print(f"{name:10s} jit={jit:2d} passes {plan.info['n_passes']} {best:.2f} ms "
              f"{2 * S * plan.info['n_passes'] / best / 1e6:.0f} GB/s", flush=True)
