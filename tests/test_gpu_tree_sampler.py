"""GPU: the tree (binomial-split) sampler — its binomial generator against the
exact pmf, multinomial counts against the oracle's exact probabilities (TV +
per-qubit 5 sigma, the bound of test_gpu_parity), int64 shot counts far beyond
2^31, and sharded sampling without a state gather."""

import math

import numpy as np
import pytest
import torch
from scipy import stats

import oracle
from paper_2504_03967_b200 import _native as N
from paper_2504_03967_b200 import partition as pt
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.errors import UnnormalizedStateError
from paper_2504_03967_b200.generators import RandomSpec, random_arrays
from paper_2504_03967_b200.ir import CircType, CircuitTensor

pytestmark = pytest.mark.gpu


def _binom(n, p, count, seed=1):
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    N.call("qg_binomial_test", float(n), float(p), seed, count, sv.C.c_void_p(out.data_ptr()),
           sv._stream(out.device))
    return out.cpu().numpy()


@pytest.mark.parametrize("n,p", [(5, 0.3), (100, 0.05), (40, 0.9), (1000, 0.3), (10**6, 0.5), (3 * 10**10, 1e-3),
                                 (10**9, 2e-9), (12, 0.5)])
def test_binomial_matches_pmf(n, p):
    count = 400_000
    x = _binom(n, p, count)
    assert x.min() >= 0 and x.max() <= n
    mu, var = n * p, n * p * (1 - p)
    # mean within 5 sigma of the sample mean's sd; variance within 5 %
    assert abs(x.mean() - mu) <= 5 * math.sqrt(var / count) + 1e-12
    assert abs(x.var() / var - 1) <= 0.05
    # TV distance to the exact pmf over the support carrying 1 - 1e-9 of the mass
    lo, hi = int(stats.binom.ppf(1e-10, n, p)), int(stats.binom.ppf(1 - 1e-10, n, p))
    ks = np.arange(lo, hi + 1)
    if ks.size <= 20_000:
        pmf = stats.binom.pmf(ks, n, p)
        emp = np.bincount(x - lo, minlength=ks.size)[: ks.size] / count
        tv = 0.5 * np.abs(emp - pmf).sum()
        assert tv <= 4 * 0.5 * math.sqrt(ks.size / count), tv


def _state(n, blocks, seed, prec):
    gt, gp = random_arrays(RandomSpec(n, blocks, seed))
    st, _ = sv.run_circuit(CircuitTensor.from_arrays(CircType.RANDOM, n, gt, gp), sv.SimOptions(precision=prec))
    p = oracle.exact_probabilities(oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64"))
    return st, p


def _check_counts(idx, cnt, p, n, shots):
    idx, cnt = np.asarray(idx), np.asarray(cnt)
    assert int(cnt.sum()) == shots and (cnt > 0).all()
    assert (np.diff(idx) > 0).all()  # unique, ascending
    b = min(n, int(math.log2(shots / 64)))
    emp = np.bincount(idx & ((1 << b) - 1), weights=cnt, minlength=1 << b) / shots
    exact = np.bincount(np.arange(1 << n) & ((1 << b) - 1), weights=p, minlength=1 << b)
    assert 0.5 * np.abs(emp - exact).sum() <= 4 * 0.5 * math.sqrt((1 << b) / shots)
    for q in range(n):
        pq = float(p[(np.arange(1 << n) >> q) & 1 == 1].sum())
        eq = float(cnt[((idx >> q) & 1) == 1].sum()) / shots
        assert abs(eq - pq) <= 5 * math.sqrt(max(pq * (1 - pq), 1e-12) / shots) + 1e-9, q


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("n", [3, 7, 12, 20])
def test_tree_sampler_statistics(precision, n):
    st, p = _state(n, 60 if n > 3 else 5, 2, precision)
    shots = 300_000
    t = sv.sample_counts(st, shots, 11, sampler="tree")
    _check_counts(t.indices, t.values, p, n, shots)
    # deterministic per seed; a different seed moves the counts
    t2 = sv.sample_counts(st, shots, 11, sampler="tree")
    assert t.counts == t2.counts
    assert sv.sample_counts(st, shots, 12, sampler="tree").counts != t.counts
    # dense mode (level-synchronous kernels) and the warp-per-leaf compact mode draw the
    # same counts bit for bit (few shots per outcome keeps the compact mode on its own path)
    ts = sv.TreeSampler(st.amplitudes)
    ts.prepare()
    few = max(1, (1 << n) // 16)
    dense = ts.draw(few, 11, dense=True).cpu().numpy()
    ci, cc = ts.draw(few, 11)
    nz = np.flatnonzero(dense)
    assert np.array_equal(nz, ci.cpu().numpy()) and np.array_equal(dense[nz], cc.cpu().numpy())
    dense = ts.draw(shots, 11, dense=True).cpu().numpy()
    nz = np.flatnonzero(dense)
    assert np.array_equal(nz, t.indices) and np.array_equal(dense[nz], t.values)


def test_tree_sampler_int64_shots():
    n = 22
    st, p = _state(n, 40, 4, "fp32")
    shots = 50_000_000_000  # QCrank's s * 2^m scale: far beyond int32, never materialised
    idx, cnt = sv.sample_indices(st.amplitudes, shots, 3)  # "philox" switches to the tree above 2^31 - 1
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    assert int(cnt.sum()) == shots
    # outcomes with a large expectation: each count within 6 sigma of its binomial mean
    # (p from the fp64 oracle); the rest through the per-qubit marginals (5 sigma)
    exp = shots * p[idx]
    big = exp >= 1000
    assert big.sum() > 1000
    z = (cnt[big] - exp[big]) / np.sqrt(exp[big] * (1 - p[idx][big]))
    assert np.max(np.abs(z)) <= 6.0
    for q in range(n):
        pq = float(p[(np.arange(1 << n) >> q) & 1 == 1].sum())
        eq = float(cnt[((idx >> q) & 1) == 1].sum()) / shots
        assert abs(eq - pq) <= 5 * math.sqrt(max(pq * (1 - pq), 1e-12) / shots) + 1e-9, q
    assert idx.size > 0.4 * (1 << n)  # most outcomes of a 22-qubit Porter-Thomas-like state are drawn


def test_tree_sampler_edge_cases():
    st = sv.init_zero_state(1, "fp64")
    t = sv.sample_counts(st, 10**12, 0, sampler="tree")
    assert t.counts == {"0": 10**12}
    st = sv.init_zero_state(17, "fp32")
    sv.apply_1q(st, sv.GateKind.H, 16)
    t = sv.sample_counts(st, 1_000_000, 1, sampler="tree")
    assert set(t.indices.tolist()) <= {0, 1 << 16}
    assert abs(t.values.sum() - 1_000_000) == 0 and abs(t.values[0] / 1e6 - 0.5) < 5 * 0.5 / 1000
    ts = sv.TreeSampler(st.amplitudes)
    ts.prepare()
    idx, cnt = ts.draw(0, 1)
    assert idx.numel() == 0
    big = sv.init_zero_state(4, "fp32")
    big.amplitudes.mul_(2.0)
    with pytest.raises(UnnormalizedStateError):
        sv.sample_counts(big, 10, 0, sampler="tree")


@pytest.mark.parametrize("workers", [2, 8])
def test_sharded_sampling_without_gather(workers):
    n = 18
    gt, gp = random_arrays(RandomSpec(n, 200, workers))
    p = oracle.exact_probabilities(oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64"))
    c = CircuitTensor.from_arrays(CircType.RANDOM, n, gt, gp)
    shots = 400_000
    res = pt.execute_distributed(c, workers, sv.SimOptions("fp32", shots, 5), gather=False)
    assert res.state is None and res.tasks["n_remaps"] >= 1
    _check_counts(res.counts.indices, res.counts.values, p, n, shots)
    # the same with the state gathered (tree sampler on the shards either way)
    res2 = pt.execute_distributed(c, workers, sv.SimOptions("fp32", shots, 5, sampler="tree"))
    assert res2.counts.counts == res.counts.counts


def test_split_shots():
    m = [0.1, 0.2, 0.0, 0.7]
    a = sv.split_shots(m, 10**9, 3)
    assert sum(a) == 10**9 and a[2] == 0 and a == sv.split_shots(m, 10**9, 3)
    for i, mi in enumerate(m):
        assert abs(a[i] - mi * 1e9) <= 6 * math.sqrt(1e9 * mi * (1 - mi)) + 1e-9


def test_circuit_graph_config1():
    """BASELINE configs[0] (16 q x 100 blocks, complex128, 3000 shots) as one CUDA
    graph replay: state vs the oracle at 1e-12, counts of 3000 shots, identical on
    replay (same seed)."""
    n = 16
    gt, gp = random_arrays(RandomSpec(n, 100, 0))
    plan = sv.CompiledCircuit(gt, gp, n, "fp64")
    g = sv.CircuitGraph(plan, 3000, 0)
    g.replay()
    st, c1 = g.result()
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    got = st.to_numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
    assert c1.total == 3000 and sum(c1.counts.values()) == 3000
    g.replay()
    _, c2 = g.result()
    assert c1.counts == c2.counts
    shots = 300_000
    g = sv.CircuitGraph(plan, shots, 4)
    g.replay()
    _, c = g.result()
    _check_counts(c.indices, c.values, oracle.exact_probabilities(ref), n, shots)
