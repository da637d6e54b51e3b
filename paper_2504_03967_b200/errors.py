"""Exception taxonomy — same class names and meaning as the reference
(/root/reference/pkg/src/qgear/errors.py:6-110) so callers can catch the
same types.  ``raise_for_status`` maps the C-ABI's negative status codes
(include/qgear_b200.h, QG_E_*) onto these classes.
"""

from __future__ import annotations


class QgearError(Exception):
    """Base class for all package-specific errors (errors.py:6)."""


class EmptyInputError(QgearError):
    pass


class InvalidQubitIndexError(QgearError):
    pass


class SelfPairError(QgearError):
    pass


class NonFiniteParamError(QgearError):
    pass


class InvalidGateError(QgearError):
    pass


class CorruptTensorError(QgearError):
    pass


class CapacityExceededError(QgearError):
    pass


class ContainerFormatError(QgearError):
    pass


class TooManyQubitsError(QgearError):
    """errors.py:47-57 — carries the byte figures."""

    def __init__(self, n_qubits: int, required_bytes: int, budget_bytes: int):
        self.n_qubits = n_qubits
        self.required_bytes = required_bytes
        self.budget_bytes = budget_bytes
        super().__init__(
            f"{n_qubits} qubits need {required_bytes} bytes of amplitudes, budget is {budget_bytes} bytes"
        )


class IndexOutOfRangeError(QgearError):
    pass


class MeasureMidCircuitError(QgearError):
    pass


class UnnormalizedStateError(QgearError):
    pass


class BadWorkerCountError(QgearError):
    pass


class ProtocolViolationError(QgearError):
    pass


class SequenceMismatchError(QgearError):
    pass


class TooFewQubitsError(QgearError):
    pass


class PlanTooSmallError(QgearError):
    pass


class LengthMismatchError(QgearError):
    pass


class EmptySpecError(QgearError):
    pass


class InsufficientDataError(QgearError):
    pass


class CudaError(QgearError):
    """A CUDA runtime / launch failure inside libqgear_b200 (no reference analogue)."""


# C-ABI status codes (include/qgear_b200.h) -> exception class
_BY_CODE = {
    -1: ValueError,                 # QG_E_INVALID_ARG
    -2: IndexOutOfRangeError,       # QG_E_INDEX_OUT_OF_RANGE
    -3: SelfPairError,              # QG_E_SELF_PAIR
    -4: MeasureMidCircuitError,     # QG_E_MEASURE_MID_CIRCUIT
    -5: TooManyQubitsError,         # QG_E_TOO_MANY_QUBITS (constructed specially)
    -6: UnnormalizedStateError,     # QG_E_UNNORMALIZED
    -7: BadWorkerCountError,        # QG_E_BAD_WORKER_COUNT
    -8: CorruptTensorError,         # QG_E_CORRUPT_TENSOR
    -9: ProtocolViolationError,     # QG_E_PROTOCOL
    -10: CudaError,                 # QG_E_CUDA
    -11: NonFiniteParamError,       # QG_E_NONFINITE_PARAM
    -12: InvalidGateError,          # QG_E_INVALID_GATE
    -13: MemoryError,               # QG_E_OUT_OF_MEMORY
    -14: ContainerFormatError,      # QG_E_CONTAINER_FORMAT
}


def raise_for_status(code: int, message: str) -> None:
    if code >= 0:
        return
    cls = _BY_CODE.get(code, QgearError)
    raise cls(message)
