"""CPU oracle for the Q-Gear state-vector hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference's CPU algorithm for the path
named by BASELINE.json:north_star (/root/reference/pkg/src/qgear/statevec.py
and partition.py).  It is the CHECKER, never the product:

* only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
  ``--impl reference`` leg may import it;
* the product package (paper_2504_03967_b200) never imports it and fails
  loudly when its CUDA library is missing.

Parity pin: every function here is checked against golden vectors produced by
the reference itself (tests/golden/make_golden.py -> tests/golden/golden.npz,
test tests/test_oracle_golden.py): fp64 states bit-identical, fp32 states
bit-identical, counts identical for the same seed.
"""

from .statevec_oracle import (  # noqa: F401
    NORM_TOL,
    apply_cr1_phase,
    apply_cx_swap,
    apply_pair_matrix,
    exact_probabilities,
    gate_matrix,
    run_arrays,
    sample_counts_arrays,
)
from .partition_oracle import execute_partitioned  # noqa: F401
