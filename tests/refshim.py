"""The reference-side ctypes binding of INTEGRATION.md ("qgear/_b200.py"), verbatim
in structure: what a reference maintainer adds so that qgear's run_circuit runs
on libqgear_b200.so.  Exercised by tests/test_gpu_reference_binding.py with the
reference's own CircuitTensor objects (baseline/_ref)."""
import ctypes as C
import os

import numpy as np
import torch

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2504_03967_b200",
                   "libqgear_b200.so")
lib = C.CDLL(LIB)


class PlanOpts(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("log2_ranks", C.c_int32), ("fuse", C.c_int32), ("tile_qubits", C.c_int32),
                ("max_stages", C.c_int32), ("max_cost", C.c_int32), ("kernel_cfg", C.c_int32),
                ("reserved", C.c_int32 * 5)]


lib.qg_plan_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(PlanOpts),
                               C.POINTER(C.c_void_p)]
lib.qg_plan_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
lib.qg_plan_destroy.argtypes = [C.c_void_p]
lib.qg_state_init_zero.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
lib.qg_last_error.restype = C.c_char_p


class B200Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"QG error {code}: {msg}")
        self.code = code


def run_circuit(circuit, options):  # replaces statevec.py:200-212
    gates = list(circuit.active_gates)
    gt = np.array([(int(g.kind), -1 if g.control is None or g.control < 0 else g.control, g.target)
                   for g in gates], dtype=np.int32).reshape(-1, 3)  # ir.py:281-303 layout
    gp = np.array([g.param for g in gates], dtype=np.float64)
    dtype = 0 if options.precision == "fp32" else 1
    plan = C.c_void_p()
    rc = lib.qg_plan_create(gt.ctypes.data, gp.ctypes.data, len(gt), circuit.n_qubits,
                            C.byref(PlanOpts(dtype=dtype, fuse=1)), C.byref(plan))
    if rc:
        raise B200Error(rc, lib.qg_last_error().decode())
    amps = torch.empty(1 << circuit.n_qubits, dtype=torch.complex64 if dtype == 0 else torch.complex128,
                       device="cuda")
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib.qg_state_init_zero(amps.data_ptr(), circuit.n_qubits, dtype, 0, stream)
    rc = lib.qg_plan_execute(plan, amps.data_ptr(), stream, 0, None)
    lib.qg_plan_destroy(plan)
    if rc:
        raise B200Error(rc, lib.qg_last_error().decode())
    return amps
