"""K1+K2 on the GPU vs the CPU oracle: bit-exact scheduling and dispatch layout.

Mirrors the reference's own scheduler tests (tests/test_aebs.cpp,
tests/acceptance.cpp C02/C11) through the public API (the C ABI via the
Python mirror), plus every BASELINE config at full sizes.
"""
import json
import os
import threading

import numpy as np
import pytest

from _cases import aebs_random_case, c02_instance
from oracle import POLICY_BRUTE, POLICY_RANDOM, CSRMap

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIELDS = ("instance", "replica", "expert_instance", "load", "routed_tokens")


@pytest.fixture(scope="module")
def J():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2512_13525_b200 as J
    return J


def to_rmap(J, m: CSRMap):
    hosts = [m.hosts_of(e).tolist() for e in range(m.E)]
    rids = [m.rids_of(e).tolist() for e in range(m.E)]
    return J.ReplicaMap(m.E, m.N, m.C, hosts, rids)


def assert_same(a, b, ctx=""):
    for f in FIELDS:
        x = np.asarray(getattr(a, f))
        y = np.asarray(b[f] if isinstance(b, dict) else getattr(b, f))
        assert np.array_equal(x, y), f"{ctx}: field {f} differs"


def test_worked_example(J):
    # tests/test_aebs.cpp:83-103
    m = J.ReplicaMap.from_hosts(2, 4, [[0], [0, 1], [1], [0, 1]])
    b = J.ActivationBatch(3, 2, [0, 1, 2, 1, 3, 0])
    a = J.schedule(b, m)
    assert a.expert_instance.tolist() == [0, 0, 1, 1]
    assert a.load.tolist() == [2, 2]
    assert a.routed_tokens.tolist() == [4, 2]
    assert a.max_load() == 2


def test_sample_fixture_golden(J):
    g = json.load(open(os.path.join(GOLD, "sample_fixture.json")))
    mj = g["map"]
    m = CSRMap(mj["E"], mj["N"], mj["C"], *(np.array(mj[x], np.int32)
                                          for x in ("off", "hosts", "rid")))
    rm = to_rmap(J, m)
    b = J.ActivationBatch(g["T"], g["k"], g["experts"])
    a = J.schedule(b, rm)
    assert_same(a, g["schedule"], "sample")
    assert J.dump_assignment(a, b) == g["dump_assignment"]  # C11-style string equality
    assert_same(J.schedule_random(b, rm, 7), g["schedule_random_seed7"], "sample random")


def test_random_small_cases_vs_oracle(J, oracle):
    # tests/test_aebs.cpp:116-145 (300 seeded instances)
    exact = 0
    for s in range(300):
        c = aebs_random_case(s)
        m = CSRMap.from_lists(c["N"], c["C"], c["hosts"], c["rids"])
        rm = to_rmap(J, m)
        sched = J.Scheduler(rm)
        b = J.ActivationBatch(c["T"], c["k"], c["experts"])
        a = sched.schedule(b)
        assert_same(a, oracle.schedule(c["experts"], c["T"], c["k"], m), f"case {s}")
        assert_same(sched.schedule_random(b, s),
                    oracle.schedule(c["experts"], c["T"], c["k"], m, policy=POLICY_RANDOM,
                                    seed=s), f"random case {s}")
        opt = oracle.schedule(c["experts"], c["T"], c["k"], m, policy=POLICY_BRUTE)
        assert a.max_load() <= opt.max_load() + 2
        exact += a.max_load() == opt.max_load()
        sched.close()
    assert exact >= 240


def test_c02_gap_histogram_on_gpu(J, oracle):
    # tests/acceptance.cpp:84,108-136: frozen {496,4,0}, GPU greedy vs exhaustive oracle
    hist = [0, 0, 0]
    for i in range(500):
        E, N, C, T, k, hosts, rids, gseed = c02_instance(i)
        m = CSRMap.from_lists(N, C, hosts, rids)
        _, cdf = oracle.pattern("uniform", E)
        ex = oracle.gen_batch(cdf, T, k, gseed, i)
        sched = J.Scheduler(to_rmap(J, m))
        a = sched.schedule(J.ActivationBatch(T, k, ex))
        sched.close()
        assert_same(a, oracle.schedule(ex, T, k, m), f"C02 {i}")
        gap = a.max_load() - oracle.schedule(ex, T, k, m, policy=POLICY_BRUTE).max_load()
        hist[gap] += 1
    assert hist == [496, 4, 0]


def test_config_cases_golden(J):
    from paper_maps import load_map_csr
    g = json.load(open(os.path.join(GOLD, "config_cases.json")))
    scheds = {}
    for c in g["cases"]:
        if c["name"] not in scheds:
            scheds[c["name"]] = J.Scheduler(to_rmap(J, load_map_csr(c["name"])))
        s = scheds[c["name"]]
        b = J.ActivationBatch(c["T"], c["k"], c["experts"])
        assert_same(s.schedule(b), c["schedule"], c["name"])
        assert_same(s.schedule_random(b, 7), c["schedule_random_seed7"], c["name"])


@pytest.mark.parametrize("name", ["c1_uniform", "c1_gaussian", "c2", "c3", "c4_n2", "c4_n4",
                                  "c4_n8", "c5"])
def test_configs_full_sizes_vs_oracle(J, oracle, name):
    from paper_maps import CONFIG_PATTERNS, load_map_csr
    m = load_map_csr(name)
    kind, kw, seed = CONFIG_PATTERNS[name]
    _, cdf = oracle.pattern(kind, m.E, **kw)
    s = J.Scheduler(to_rmap(J, m))
    for T in (1, 7, 32, 64, 128, 256, 512, 1000, 1024, 2048, 4096):
        ex = oracle.gen_batch(cdf, T, 8, seed, T)
        b = J.ActivationBatch(T, 8, ex)
        assert_same(s.schedule(b), oracle.schedule(ex, T, 8, m), f"{name} T={T}")
        assert_same(s.schedule_random(b, T), oracle.schedule(ex, T, 8, m, policy=POLICY_RANDOM,
                                                             seed=T), f"{name} random T={T}")


def test_c10_and_bench_maps_n16(J, oracle):
    # tests/acceptance.cpp:328-335 (C10 map) and tools/bench_schedule.cpp:18-38
    E, N = 200, 16
    hosts = [sorted({e % N, (e + N // 2) % N}) for e in range(E)]
    nxt = [0] * N
    rids = []
    for h in hosts:
        rids.append([nxt[g] for g in h])
        for g in h:
            nxt[g] += 1
    m = CSRMap.from_lists(N, max(nxt), hosts, rids)
    s = J.Scheduler(to_rmap(J, m))
    _, cdf = oracle.pattern("uniform", E)
    for T in (16, 512, 4096):
        ex = oracle.gen_batch(cdf, T, 8, 0xBE, T)
        assert_same(s.schedule(J.ActivationBatch(T, 8, ex)), oracle.schedule(ex, T, 8, m))


def test_many_instances_general_path(J, oracle):
    # N > 32 takes the smem-load greedy path
    rng = np.random.default_rng(5)
    for N in (33, 64, 200):
        E = 256
        hosts = [sorted(rng.choice(N, size=int(rng.integers(1, 6)), replace=False).tolist())
                 for _ in range(E)]
        m = CSRMap.from_lists(N, E, hosts)
        s = J.Scheduler(to_rmap(J, m))
        _, cdf = oracle.pattern("gaussian", E, 0.1)
        for T in (5, 300, 2000):
            ex = oracle.gen_batch(cdf, T, 8, N, T)
            assert_same(s.schedule(J.ActivationBatch(T, 8, ex)), oracle.schedule(ex, T, 8, m))
            assert_same(s.schedule_random(J.ActivationBatch(T, 8, ex), 3),
                        oracle.schedule(ex, T, 8, m, policy=POLICY_RANDOM, seed=3))


def test_unknown_expert_message(J):
    # tests/test_aebs.cpp:160-167; schedule() reports the minimum bad id
    m = J.ReplicaMap.from_hosts(2, 2, [[0], [1]])
    with pytest.raises(J.ValidationError, match="unknown-expert: batch references expert -4 "
                                                "with no replica in the map"):
        J.schedule(J.ActivationBatch(4, 1, [0, 3, -4, 2]), m)
    with pytest.raises(J.ValidationError, match="expert 2 with no replica"):
        J.schedule(J.ActivationBatch(4, 1, [0, 3, 5, 2]), m)


def test_empty_batch(J):
    m = J.ReplicaMap.from_hosts(2, 2, [[0], [1]])
    a = J.schedule(J.ActivationBatch(0, 2, []), m)
    assert a.instance.size == 0 and a.load.tolist() == [0, 0]
    assert a.expert_instance.tolist() == [-1, -1]


def test_concurrent_invocation_deterministic(J, oracle):
    # tests/test_aebs.cpp:182-192 and acceptance C11: repeated and concurrent calls agree
    from paper_maps import load_map_csr
    m = load_map_csr("c3")
    _, cdf = oracle.pattern("uniform", m.E)
    ex = oracle.gen_batch(cdf, 512, 8, 0xDE7, 0)
    b = J.ActivationBatch(512, 8, ex)
    ref = oracle.schedule(ex, 512, 8, m)
    errs = []

    def worker():
        s = J.Scheduler(to_rmap(J, m))
        for _ in range(20):
            try:
                assert_same(s.schedule(b), ref, "concurrent")
            except AssertionError as e:  # pragma: no cover
                errs.append(e)
        s.close()

    th = [threading.Thread(target=worker) for _ in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs


def test_dispatch_layout_vs_oracle(J, oracle):
    import torch
    from paper_maps import CONFIG_PATTERNS, load_map_csr
    for name in ("c1_gaussian", "c3", "c4_n8", "c5"):
        m = load_map_csr(name)
        kind, kw, seed = CONFIG_PATTERNS[name]
        _, cdf = oracle.pattern(kind, m.E, **kw)
        s = J.Scheduler(to_rmap(J, m))
        qidx_dev, qbase_dev = s.replica_order()
        qidx, _, qbase = oracle.replica_order(m)
        assert np.array_equal(qidx_dev, qidx) and np.array_equal(qbase_dev, qbase)
        R = int(m.off[-1])
        for T in (1, 256, 4096):
            ex = oracle.gen_batch(cdf, T, 8, seed, T)
            S = T * 8
            d = lambda n, dt=torch.int32: torch.full((n,), -7, dtype=dt, device="cuda")
            out = dict(instance=d(S), replica=d(S), expert_instance=d(m.E), load=d(m.N),
                       routed_tokens=d(m.N, torch.int64), expert_tokens=d(m.E, torch.int64),
                       slot_row=d(S), row_slot=d(S), group_off=d(R + 1), status=d(2))
            s.schedule_async(torch.from_numpy(ex).cuda(), T, 8, out)
            torch.cuda.synchronize()
            a = oracle.schedule(ex, T, 8, m)
            goff, srow, rslot = oracle.dispatch_layout(ex, T, 8, m, qidx, a.expert_instance)
            assert out["status"].tolist() == [0, 0]
            assert np.array_equal(out["group_off"].cpu().numpy(), goff), name
            assert np.array_equal(out["slot_row"].cpu().numpy(), srow), name
            assert np.array_equal(out["row_slot"].cpu().numpy(), rslot), name
            assert np.array_equal(out["expert_tokens"].cpu().numpy(), a.expert_tokens)


def test_scheduler_timing_sane(J, oracle):
    import torch
    from paper_maps import load_map_csr
    m = load_map_csr("c1_uniform")
    s = J.Scheduler(to_rmap(J, m))
    _, cdf = oracle.pattern("uniform", m.E)
    ex = torch.from_numpy(oracle.gen_batch(cdf, 256, 8, 0x5EED, 1256)).cuda()
    us = s.time_schedule(ex, 256, 8, reps=21)
    assert 0 < us < 100, us
