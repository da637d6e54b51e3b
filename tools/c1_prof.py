"""CUDA-graph replay of config C1 (16q c128 x 100 blocks + 3000 shots) for an ncu launch list (dev tool)."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays
gt, gp = random_arrays(RandomSpec(16, 100, 0))
plan = sv.CompiledCircuit(gt, gp, 16, "fp64")
g = sv.CircuitGraph(plan, 3000, 0)
for _ in range(5): g.replay()
torch.cuda.synchronize()
