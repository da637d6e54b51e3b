"""GPU: size-independent properties at full scale (32-33 qubits, complex64),
where the oracle cannot run: QFT of |0> is the uniform state (analytic), and a
random CX-block circuit followed by its inverse returns |0...0> (round trip).
33 qubits (64 GiB) puts qubit 32 inside fused-pass tiles, exercising the 64-bit
in-tile addressing path (tile_lo32 = 0); 32 qubits the 32-bit path."""

import math

import numpy as np
import pytest
import torch

from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays
from paper_2504_03967_b200.ir import GateKind

pytestmark = pytest.mark.gpu


def inverse(gt, gp):
    """Reverse order; RX/RY/RZ/CR1 angles negated; H and CX are self-inverse."""
    it, ip = gt[::-1].copy(), gp[::-1].copy()
    neg = np.isin(it[:, 0], [GateKind.RX, GateKind.RY, GateKind.RZ, GateKind.CR1])
    ip[neg] = -ip[neg]
    return it, ip


def free_gib():
    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


@pytest.mark.parametrize("n", [32, 33])
def test_random_then_inverse_is_identity(n):
    if free_gib() < (1 << n) * 8 / 2**30 + 4:
        pytest.skip("not enough device memory")
    gt, gp = random_arrays(RandomSpec(n, 120, 3))
    it, ip = inverse(gt, gp)
    plan = sv.CompiledCircuit(np.concatenate([gt, it]), np.concatenate([gp, ip]), n, "fp32")
    st = sv.init_zero_state(n, "fp32", 1 << 40)
    plan.execute(st)
    amp0 = complex(st.amplitudes[0].item())
    a = st.amplitudes
    rest = max(float(a[max(i, 1):i + (1 << 28)].abs().max().item()) for i in range(0, a.numel(), 1 << 28))
    assert abs(abs(amp0) - 1) < 1e-4 and rest < 1e-4
    assert abs(st.norm_sq() - 1) < 1e-4
    del st
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [32, 33])
def test_qft_of_zero_is_uniform(n):
    if free_gib() < (1 << n) * 8 / 2**30 + 4:
        pytest.skip("not enough device memory")
    gt, gp = qft_arrays(n)
    plan = sv.CompiledCircuit(gt, gp, n, "fp32")
    st = sv.init_zero_state(n, "fp32", 1 << 40)
    plan.execute(st)
    u = 2.0 ** (-n / 2)
    a = st.amplitudes
    dev = max(float((a[i:i + (1 << 28)] - u).abs().max().item()) for i in range(0, a.numel(), 1 << 28))
    assert dev < 1e-5 * u * 10
    assert abs(st.norm_sq() - 1) < 1e-4
    del st
    torch.cuda.empty_cache()
