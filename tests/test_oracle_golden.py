"""Pin the CPU oracle to the reference's own outputs (tests/golden/golden.npz).

The fixtures were produced by tests/golden/make_golden.py importing the
reference package; here the oracle must reproduce them bit for bit.
"""

import numpy as np
import pytest

import oracle
from oracle import statevec_oracle as so


def test_oracle_states_bit_identical(golden):
    for name in golden["state_cases"]:
        nq, ng = (int(v) for v in golden[f"state_{name}_hdr"])
        for prec in ("fp64", "fp32"):
            psi = oracle.run_arrays(golden[f"state_{name}_type"], golden[f"state_{name}_param"], nq, ng, prec)
            ref = golden[f"state_{name}_{prec}"]
            assert psi.dtype == ref.dtype
            assert np.array_equal(psi, ref), (name, prec)


def test_oracle_cfg1_state_and_counts(golden):
    gt, gp = golden["gen_random_16_100_0_0_type"], golden["gen_random_16_100_0_0_param"]
    psi = oracle.run_arrays(gt, gp, 16, gt.shape[0], "fp64")
    assert np.array_equal(psi, golden["cfg1_state_fp64"])
    idx, cnt = oracle.sample_counts_arrays(psi, 3000, 0, "fp64")
    assert np.array_equal(idx, golden["cfg1_count_index"])
    assert np.array_equal(cnt, golden["cfg1_count_value"])
    keys = [so.bitstring(int(i), 16) for i in idx]
    assert keys == list(golden["cfg1_count_keys"])


@pytest.mark.parametrize("j", range(4))
def test_oracle_sampling(golden, j):
    n, shots, seed = (int(v) for v in golden[f"sample{j}_meta"])
    idx, cnt = oracle.sample_counts_arrays(golden[f"sample{j}_amps"], shots, seed, "fp64")
    assert np.array_equal(idx, golden[f"sample{j}_index"])
    assert np.array_equal(cnt, golden[f"sample{j}_value"])


@pytest.mark.parametrize("j", range(3))
def test_oracle_partitioned(golden, j):
    nq, ng, w = (int(v) for v in golden[f"part{j}_meta"])
    st, counts, sent, masks = oracle.execute_partitioned(
        golden[f"part{j}_type"], golden[f"part{j}_param"], nq, ng, w, "fp64", 2000, 5)
    assert np.array_equal(st, golden[f"part{j}_state"])
    assert list(sent) == list(golden[f"part{j}_sent"])
    assert np.array_equal(masks, golden[f"part{j}_masks"])
    assert np.array_equal(counts[0], golden[f"part{j}_cidx"])
    assert np.array_equal(counts[1], golden[f"part{j}_cval"])
    # single worker gives the same amplitudes (partition.py docstring, SPEC AC4)
    single = oracle.run_arrays(golden[f"part{j}_type"], golden[f"part{j}_param"], nq, ng, "fp64")
    assert np.array_equal(single, st)


def test_oracle_qft_closed_form():
    # build_qft(n) on |0..0> is the uniform state (generators.py:82-101)
    from paper_2504_03967_b200.generators import qft_arrays

    gt, gp = qft_arrays(9)
    psi = oracle.run_arrays(gt, gp, 9, gt.shape[0], "fp64")
    assert np.allclose(psi, 2 ** -4.5, atol=1e-14)
