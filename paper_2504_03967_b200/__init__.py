"""paper_2504_03967_b200 — B200-native executor for the Q-Gear state-vector hot path.

Public API mirrors the reference package (/root/reference/pkg/src/qgear):
  ir          GateKind, GateRecord, CircuitTensor, CircuitSet, encode/decode, set_to/from_arrays
  generators  RandomSpec, QftSpec, generate_random_gate_list, build_qft, random_qubit_pairs
  statevec    init_zero_state, run_circuit, run_circuit_timed, sample_counts, exact_probabilities,
              apply_matrix_array / swap_target_pairs_array / phase_pairs_array, ...
  partition   execute_distributed (sharded over torch.distributed ranks or in-process shards)
The compute runs in libqgear_b200.so (hand-written sm_100a CUDA); see DESIGN.md.
"""

from . import errors, generators, ir  # noqa: F401

__all__ = ["errors", "generators", "ir", "statevec", "partition"]


def __getattr__(name):  # torch-dependent modules load lazily
    if name in ("statevec", "partition"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
