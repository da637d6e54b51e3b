"""paper_2504_03967_b200 — B200-native executor for the Q-Gear state-vector hot path.

Public API mirrors the reference package (/root/reference/pkg/src/qgear):
  ir          GateKind, GateRecord, CircuitTensor, CircuitSet, encode/decode, set_to/from_arrays
  generators  RandomSpec, QftSpec, generate_random_gate_list, build_qft, random_qubit_pairs
  statevec    init_zero_state, run_circuit, run_circuit_timed, sample_counts, exact_probabilities,
              apply_matrix_array / swap_target_pairs_array / phase_pairs_array, ...
  partition   execute_distributed (sharded over torch.distributed ranks or in-process shards)
  batch       run_circuit_set(_distributed): CircuitSet batches, plan reuse via qg_plan_rebind
  qcrank      QCrank image encoding / decoding, one-pass UCRY execution
  container   QGIR1 circuit-set files: native parse / write, zero-copy array views
The compute runs in libqgear_b200.so (hand-written sm_100a CUDA); see DESIGN.md.
"""

from . import errors, generators, ir  # noqa: F401

__all__ = ["errors", "generators", "ir", "statevec", "partition", "batch", "qcrank", "container"]


def __getattr__(name):  # torch- / library-dependent modules load lazily
    if name in ("statevec", "partition", "batch", "qcrank", "container"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
