"""Oracle restatement vs the reference compiled from /root/reference (oracle/_ref).

Skips where oracle/_ref is absent.  CPU only.
"""
import numpy as np
import pytest

from _cases import aebs_random_case
from oracle import POLICY_RANDOM, CSRMap

FIELDS = ("instance", "replica", "expert_instance", "load", "routed_tokens")


def eq(a, b):
    return all(np.array_equal(getattr(a, f), getattr(b, f)) for f in FIELDS)


@pytest.mark.parametrize("kind,sigma", [("uniform", 0), ("gaussian", 0.15), ("gaussian", 0.02)])
def test_gen_batch_bit_exact(oracle, ref, kind, sigma):
    for E, T, k in ((64, 300, 8), (16, 40, 7), (200, 512, 8), (8, 20, 8)):
        _, cdf = oracle.pattern(kind, E, sigma)
        _, cdf_r = ref.pattern(kind, E, sigma)
        assert np.array_equal(cdf, cdf_r)
        for step in (0, 3, 1256):
            a = oracle.gen_batch(cdf, T, k, 0xBE5C, step)
            b = ref.gen_batch(kind, E, T, k, 0xBE5C, step, sigma=sigma)
            assert np.array_equal(a, b)


def test_gen_batch_zipf_and_cover_all(oracle, ref):
    for s in (1.0, 1.2, 3.0):
        w = np.array([1.0 / (e + 1) ** s for e in range(128)])
        _, cdf = oracle.pattern("pmf", 128, weights=w)
        for T in (32, 256, 1024):
            assert np.array_equal(oracle.gen_batch(cdf, T, 8, 0x30, T),
                                  ref.gen_batch("pmf", 128, T, 8, 0x30, T, weights=w))
    _, cdf = oracle.pattern("gaussian", 64, 0.05)
    assert np.array_equal(oracle.gen_batch(cdf, 40, 4, 9, 1, cover_all=True),
                          ref.gen_batch("gaussian", 64, 40, 4, 9, 1, sigma=0.05, cover_all=True))


def test_schedule_small_cases_vs_ref(oracle, ref):
    for s in range(300):
        c = aebs_random_case(s)
        m = CSRMap.from_lists(c["N"], c["C"], c["hosts"], c["rids"])
        for pol in ("schedule", "reference"):
            assert eq(oracle.schedule(c["experts"], c["T"], c["k"], m),
                      ref.schedule(c["experts"], c["T"], c["k"], m, pol))
        assert eq(oracle.schedule(c["experts"], c["T"], c["k"], m, policy=POLICY_RANDOM, seed=s),
                  ref.schedule(c["experts"], c["T"], c["k"], m, "random", seed=s))


@pytest.mark.parametrize("name", ["c1_uniform", "c1_gaussian", "c2", "c3", "c4_n2", "c4_n4",
                                  "c4_n8", "c5"])
def test_schedule_configs_vs_ref(oracle, ref, name):
    from paper_maps import CONFIG_PATTERNS, load_map_csr
    m = load_map_csr(name)
    kind, kw, seed = CONFIG_PATTERNS[name]
    _, cdf = oracle.pattern(kind, m.E, **kw)
    for T in (1, 32, 256, 1024, 4096):
        ex = oracle.gen_batch(cdf, T, 8, seed, T)
        assert eq(oracle.schedule(ex, T, 8, m), ref.schedule(ex, T, 8, m, "schedule"))
        assert eq(oracle.schedule(ex, T, 8, m, policy=POLICY_RANDOM, seed=T),
                  ref.schedule(ex, T, 8, m, "random", seed=T))


def test_bench_schedule_map(oracle, ref):
    # tools/bench_schedule.cpp:18-38 make_map (per-instance ids, NOT re-ordered with sorted hosts)
    E, N, R = 200, 16, 2
    hosts, rids, nxt, cur = [], [], [0] * N, 0
    for e in range(E):
        hs, rs = [], []
        for r in range(R):
            g = (cur + r * (N // R)) % N
            hs.append(g)
            rs.append(nxt[g])
            nxt[g] += 1
        hosts.append(sorted(hs))
        rids.append(rs)
        cur = (cur + 1) % N
    m = CSRMap.from_lists(N, (E * R + N - 1) // N + 1, hosts, rids)
    _, cdf = oracle.pattern("gaussian", E, 0.15)
    for T in (16, 64, 128, 512):
        ex = oracle.gen_batch(cdf, T, 8, 0xBE5C, T)
        assert eq(oracle.schedule(ex, T, 8, m), ref.schedule(ex, T, 8, m, "schedule"))


def test_latency_model_vs_ref(oracle, ref):
    rng = np.random.default_rng(1)
    for _ in range(50):
        N = int(rng.integers(1, 9))
        load = rng.integers(0, 40, N).astype(np.int32)
        routed = rng.integers(0, 5000, N).astype(np.int64)
        assert oracle.moe_layer_latency(load, routed, 4096, 1536) == \
            ref.moe_layer_latency(load, routed, 4096, 1536)


@pytest.mark.parametrize("E,W", [(8, 1), (40, 3), (256, 6)])
def test_activation_stats_restatement(oracle, ref, E, W):
    """or_stats_record (the device algorithm: a ring of bitmasks) equals the
    reference ActivationStats (experts.cpp:30-57) on random windows."""
    rng = np.random.default_rng(E + W)
    steps = [np.sort(rng.choice(E, int(rng.integers(0, min(E, 20) + 1)), replace=False))
             for _ in range(4 * W + 3)]
    st = oracle.stats_new(E, W)
    for a in steps:
        oracle.stats_record(st, a)
    rc, rco = ref.stats(E, W, steps)
    np.testing.assert_array_equal(st["counts"], rc)
    np.testing.assert_array_equal(st["coact"], rco)
    with pytest.raises(ValueError, match="out of range"):
        ref.stats(E, W, [np.array([E], np.int32)])
    with pytest.raises(ValueError, match="ascending"):
        ref.stats(E, W, [np.array([1, 1], np.int32)])
