"""GPU activation statistics bit-exact against the reference
ActivationStats (oracle/_ref, experts.cpp:11-62) and the oracle restatement."""
import numpy as np
import pytest
import torch

import paper_2512_13525_b200 as J
from paper_2512_13525_b200.moe import ActivationStats
from routing import RoutingPattern, gen_batch

pytestmark = pytest.mark.gpu


def _steps(E, k, n, seed, T_choices=(0, 1, 3, 17, 64, 300)):
    rng = np.random.default_rng(seed)
    pats = [RoutingPattern.uniform(E), RoutingPattern.zipf(E, 1.2),
            RoutingPattern.gaussian(E, 0.1)]
    out = []
    for i in range(n):
        T = int(rng.choice(T_choices))
        out.append(gen_batch(pats[i % 3], T, k, seed, i).experts)
    return out


@pytest.mark.parametrize("E,k,W", [(8, 2, 1), (64, 8, 3), (128, 8, 8), (256, 8, 5), (40, 4, 2)])
def test_stats_bit_exact_vs_reference(ref, oracle, E, k, W):
    steps = _steps(E, k, 3 * W + 4, E * 7 + W)
    st = ActivationStats(E, W)
    dev = torch.device("cuda", 0)
    for ex in steps:
        st.record_batch(torch.from_numpy(np.ascontiguousarray(ex, np.int32)).to(dev), k)
    counts, coact, rec = st.read()
    activated = [np.unique(ex) for ex in steps]
    rc, rco = ref.stats(E, W, activated)
    np.testing.assert_array_equal(counts, rc)
    np.testing.assert_array_equal(coact.reshape(-1), rco)
    assert rec == min(len(steps), W)
    o = oracle.stats_new(E, W)
    for a in activated:
        oracle.stats_record(o, a)
    np.testing.assert_array_equal(o["counts"], rc)
    np.testing.assert_array_equal(o["coact"], rco)


def test_stats_rejects_out_of_range_step(ref):
    E, k, W = 16, 2, 2
    st = ActivationStats(E, W)
    dev = torch.device("cuda", 0)
    good = np.array([1, 2, 3, 4], np.int32)
    st.record_batch(torch.from_numpy(good).to(dev), k)
    st.record_batch(torch.from_numpy(np.array([5, 16, 2, -3], np.int32)).to(dev), k)
    with pytest.raises(J.ValidationError, match="stats: activated expert -3 out of range"):
        st.check()
    counts, coact, rec = st.read()
    rc, rco = ref.stats(E, W, [np.unique(good)])
    np.testing.assert_array_equal(counts, rc)
    np.testing.assert_array_equal(coact.reshape(-1), rco)
    assert rec == 1
    with pytest.raises(J.ValidationError, match="window must be > 0"):
        ActivationStats(E, 0)
