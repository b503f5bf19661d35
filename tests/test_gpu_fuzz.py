"""Seeded fuzz against the oracle.  The whole layer (K1 -> K3 -> K4 -> K5) vs
the fp32 oracle over random shapes, replica maps, instance filters, shared
experts and step sizes — both GEMM regimes (64- and 256-row tiles), ragged
groups, empty instances (tolerances as in test_gpu_moe.py); the scheduler
bit-exact over random maps and step sizes; the gating kernel over random
shapes; the activation statistics bit-exact vs the reference.
JANUS_FUZZ_CASES sets the case count per test (default 64, seconds; on a
B200 3000 layer, 1000 scheduler, 400 gate and 300 stats cases ran clean)."""
import os

import numpy as np
import pytest

from test_gpu_moe import check_close, make_layer, oracle_layer_out, run, u16  # noqa: F401
from oracle import bf16_to_f32
from routing import RoutingPattern, gen_batch

pytestmark = pytest.mark.gpu
CASES = int(os.environ.get("JANUS_FUZZ_CASES", "64"))


def random_map(J, rng, E, N):
    """Every expert on 1..min(3, N) distinct instances, capacity = the most
    loaded instance (a valid reference ReplicaMap)."""
    hosts = []
    for _ in range(E):
        r = int(rng.integers(1, min(3, N) + 1))
        hosts.append(sorted(rng.choice(N, r, replace=False).tolist()))
    cap = max(1, max(sum(g in h for h in hosts) for g in range(N)))
    return J.ReplicaMap.from_hosts(N, cap, hosts)


@pytest.fixture(scope="module")
def J():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2512_13525_b200 as J
    return J


@pytest.mark.parametrize("case", range(CASES))
def test_layer_fuzz(J, oracle, case):
    import torch
    from paper_2512_13525_b200.moe import expert_weights
    rng = np.random.default_rng(1000 + case)
    E = int(rng.choice([8, 16, 40, 64, 128]))
    k = int(rng.choice([k_ for k_ in (1, 2, 4, 6, 8) if k_ <= E]))
    d_h = int(rng.choice([256, 512, 768]))
    d_e = int(rng.choice([128, 256, 384]))
    # step sizes on both sides of the 28-rows-per-expert tile crossover
    T = int(rng.choice([1, 3, int(rng.integers(4, 120)), int(rng.integers(120, 900))]))
    N = int(rng.choice([1, 2, 3]))
    rm = random_map(J, rng, E, N)
    instance = -1 if N == 1 or rng.random() < 0.5 else int(rng.integers(0, N))
    shared = bool(rng.random() < 0.25) and instance <= 0
    pat = (RoutingPattern.zipf(E, float(rng.choice([0.0, 1.0, 1.5]))) if rng.random() < 0.7
           else RoutingPattern.gaussian(E, 0.2))
    b = gen_batch(pat, T, k, int(rng.integers(1 << 30)), case)
    layer = make_layer(J, rm, d_h, d_e, max(T, 1), k, seed=case + 1, instance=instance)
    if shared:
        wg, wu, wd = expert_weights(E + 1, d_h, d_e, case + 3, "cuda")
        layer.set_shared(torch.cat([wg, wu]).contiguous(), wd.contiguous())
    x, ex, gw, out = run(J, layer, b.experts, T, seed=case + 7)
    tokens = np.unique(np.concatenate([[0, T - 1], rng.integers(0, T, 24)]))
    what = (f"case {case}: E={E} k={k} d_h={d_h} d_e={d_e} T={T} N={N} instance={instance} "
            f"shared={shared}")
    for round_h in (True, False):  # h rounded like the device, and the pure fp32 layer
        ref = oracle_layer_out(oracle, layer, x, ex, gw, tokens, round_h=round_h)
        if shared:
            ref += oracle.expert_swiglu(u16(x)[tokens], u16(wg), u16(wu), u16(wd),
                                        round_h=round_h, nthreads=8)
        check_close(bf16_to_f32(u16(out))[tokens], ref, what + f" round_h={round_h}")


@pytest.mark.parametrize("case", range(CASES))
def test_scheduler_fuzz(J, oracle, case):
    """K1+K2 bit-exact vs the oracle over random maps (1-40 instances, so the
    warp greedy and the N > 32 path), expert counts and step sizes spanning
    every cluster size (1-16 CTAs), AEBS and the random policy."""
    from oracle import POLICY_RANDOM, CSRMap
    rng = np.random.default_rng(5000 + case)
    E = int(rng.choice([8, 16, 64, 128, 200, 256]))
    N = int(rng.choice([1, 2, 3, 6, 8, 16, 33, 40]))
    k = int(rng.choice([k_ for k_ in (1, 2, 4, 8) if k_ <= E]))
    T = int(rng.choice([0, 1, int(rng.integers(2, 300)), int(rng.integers(300, 6000))]))
    rm = random_map(J, rng, E, N)
    pat = RoutingPattern.zipf(E, float(rng.choice([0.0, 1.0, 1.2])))
    b = gen_batch(pat, T, k, int(rng.integers(1 << 30)), case)
    m = CSRMap(rm.num_experts, rm.num_instances, rm.slots_per_instance, *rm.csr())
    sched = J.Scheduler(rm)
    try:
        what = f"case {case}: E={E} N={N} k={k} T={T}"
        a = sched.schedule(b)
        ref = oracle.schedule(b.experts, T, k, m)
        for f in ("instance", "replica", "expert_instance", "load", "routed_tokens"):
            assert np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(ref, f))), \
                f"{what}: {f}"
        seed = int(rng.integers(1 << 30))
        a = sched.schedule_random(b, seed)
        ref = oracle.schedule(b.experts, T, k, m, policy=POLICY_RANDOM, seed=seed)
        for f in ("instance", "replica", "expert_instance", "load", "routed_tokens"):
            assert np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(ref, f))), \
                f"{what} (random): {f}"
    finally:
        sched.close()


@pytest.mark.parametrize("case", range(CASES))
def test_gate_fuzz(J, oracle, case):
    """The gating kernel over random (E, k, d_h, T): every split-K cluster
    size and both epilogues, against the oracle's definition."""
    import torch
    from test_gpu_gate import _check
    from paper_2512_13525_b200.moe import MoELayer, make_inputs, router_weights
    rng = np.random.default_rng(9000 + case)
    E = int(rng.choice([16, 32, 48, 64, 128, 160, 256]))
    k = int(rng.choice([k_ for k_ in (1, 2, 4, 8, 16) if k_ <= E]))
    d_h = int(rng.choice([256, 512, 1024, 2048]))
    T = int(rng.choice([1, int(rng.integers(2, 200)), int(rng.integers(200, 3000))]))
    rm = J.ReplicaMap.from_hosts(1, E, [[0]] * E)
    layer = MoELayer(rm, 256, 128, max(T, 1), k, device=0)
    x, _ = make_inputs(T, k, d_h, case + 5, "cuda")
    wr = router_weights(E, d_h, case + 9, "cuda")
    ex, gw = layer.gate(x, wr)
    torch.cuda.synchronize()
    _check(oracle, x, wr, k, ex, gw)


@pytest.mark.parametrize("case", range(CASES))
def test_stats_fuzz(J, ref, case):
    """Device ActivationStats bit-exact vs the compiled reference over random
    expert counts, windows and step sequences (empty steps included)."""
    import torch
    from test_gpu_stats import _steps
    from paper_2512_13525_b200.moe import ActivationStats
    rng = np.random.default_rng(12000 + case)
    E = int(rng.choice([1, 2, 7, 32, 33, 100, 128, 256]))
    k = int(rng.choice([k_ for k_ in (1, 2, 4, 8) if k_ <= E]))
    W = int(rng.integers(1, 10))
    steps = _steps(E, k, int(rng.integers(1, 3 * W + 6)), case)
    st = ActivationStats(E, W)
    dev = torch.device("cuda", 0)
    for ex in steps:
        st.record_batch(torch.from_numpy(np.ascontiguousarray(ex, np.int32)).to(dev), k)
    counts, coact, rec = st.read()
    rc, rco = ref.stats(E, W, [np.unique(ex) for ex in steps])
    np.testing.assert_array_equal(counts, rc)
    np.testing.assert_array_equal(coact.reshape(-1), rco)
    assert rec == min(len(steps), W)
