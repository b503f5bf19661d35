"""Pin the CPU oracle (oracle/oracle.c) before trusting it.

Against the reference's own golden vectors and known-answer tests, and against
the reference itself compiled from /root/reference (oracle/_ref).  CPU only.
"""
import json
import os

import numpy as np
import pytest

from _cases import aebs_random_case, c02_instance
from oracle import POLICY_AEBS, POLICY_BRUTE, POLICY_RANDOM, CSRMap, ScheduleError

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIELDS = ("instance", "replica", "expert_instance", "load", "routed_tokens")


def same(a, b):
    return all(np.array_equal(np.asarray(getattr(a, f)), np.asarray(b[f] if isinstance(b, dict)
                                                                      else getattr(b, f)))
               for f in FIELDS)


def test_splitmix64_frozen(oracle):
    # tests/test_rng.cpp:17-18
    assert oracle.splitmix64(0, 2) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]


def test_derive_seed_separates(oracle):
    # tests/test_rng.cpp:21-28
    seen = {oracle.derive_seed(r, l, x) for r in (0, 1, 42) for l in ("a", "b", "workload/step")
            for x in (0, 1, 2)}
    assert len(seen) == 27


def test_worked_two_instance_example(oracle):
    # tests/test_aebs.cpp:83-103
    m = CSRMap.from_lists(2, 4, [[0], [0, 1], [1], [0, 1]])
    ex = np.array([0, 1, 2, 1, 3, 0], np.int32)
    a = oracle.schedule(ex, 3, 2, m)
    assert a.expert_instance.tolist() == [0, 0, 1, 1]
    assert a.max_load() == 2
    assert a.load.tolist() == [2, 2]
    assert a.routed_tokens.tolist() == [4, 2]
    for s in range(6):
        assert a.instance[s] == a.expert_instance[ex[s]]


def test_greedy_gap_vs_brute_force(oracle):
    # tests/test_aebs.cpp:105-114
    m = CSRMap.from_lists(3, 3, [[0, 1, 2], [0, 1], [0, 1]])
    ex = np.array([0, 1, 2], np.int32)
    g = oracle.schedule(ex, 3, 1, m)
    opt = oracle.schedule(ex, 3, 1, m, policy=POLICY_BRUTE)
    assert g.max_load() == 2 and opt.max_load() == 1


def test_random_small_instances(oracle):
    # tests/test_aebs.cpp:116-145: 300 seeded instances, gap <= 2, >= 240 optimal,
    # every slot on a genuine replica
    exact = 0
    for s in range(300):
        c = aebs_random_case(s)
        m = CSRMap.from_lists(c["N"], c["C"], c["hosts"], c["rids"])
        a = oracle.schedule(c["experts"], c["T"], c["k"], m)
        opt = oracle.schedule(c["experts"], c["T"], c["k"], m, policy=POLICY_BRUTE)
        assert a.max_load() <= opt.max_load() + 2
        exact += a.max_load() == opt.max_load()
        for si, e in enumerate(c["experts"]):
            g = a.instance[si]
            assert g == a.expert_instance[e]
            hs = list(m.hosts_of(e))
            assert g in hs
            assert a.replica[si] == m.rids_of(e)[hs.index(g)]
    assert exact >= 240


def test_c02_frozen_gap_histogram(oracle):
    # tests/acceptance.cpp:84,108-136: frozen {496,4,0}
    hist = [0, 0, 0]
    for i in range(500):
        E, N, C, T, k, hosts, rids, gseed = c02_instance(i)
        m = CSRMap.from_lists(N, C, hosts, rids)
        _, cdf = oracle.pattern("uniform", E)
        ex = oracle.gen_batch(cdf, T, k, gseed, i)
        gap = (oracle.schedule(ex, T, k, m).max_load()
               - oracle.schedule(ex, T, k, m, policy=POLICY_BRUTE).max_load())
        assert 0 <= gap <= 2
        hist[gap] += 1
    assert hist == [496, 4, 0]


def test_sample_fixture_known_answer(oracle):
    # configs/sample-batch.txt x sample-replicas.txt (README.md:57-58); expected
    # values from SURVEY.md §8(c)(4), reproduced by the reference (golden JSON)
    g = json.load(open(os.path.join(GOLD, "sample_fixture.json")))
    mj = g["map"]
    m = CSRMap(mj["E"], mj["N"], mj["C"], *(np.array(mj[x], np.int32)
                                          for x in ("off", "hosts", "rid")))
    a = oracle.schedule(np.array(g["experts"], np.int32), g["T"], g["k"], m)
    assert a.load.tolist() == [3, 3, 3, 2, 2, 2]
    assert a.routed_tokens.tolist() == [12, 11, 8, 8, 3, 6]
    assert a.expert_instance.tolist() == [0, 0, 1, 2, -1, 1, 2, 3, 4, 5, 0, 1, 2, 3, 4, 5]
    assert same(a, g["schedule"])
    r = oracle.schedule(np.array(g["experts"], np.int32), g["T"], g["k"], m,
                        policy=POLICY_RANDOM, seed=7)
    assert same(r, g["schedule_random_seed7"])


def test_config_cases_golden(oracle):
    from paper_maps import load_map_csr
    g = json.load(open(os.path.join(GOLD, "config_cases.json")))
    for c in g["cases"]:
        m = load_map_csr(c["name"])
        ex = np.array(c["experts"], np.int32)
        assert same(oracle.schedule(ex, c["T"], c["k"], m), c["schedule"]), c["name"]
        assert same(oracle.schedule(ex, c["T"], c["k"], m, policy=POLICY_RANDOM, seed=7),
                    c["schedule_random_seed7"]), c["name"]


def test_unknown_expert_min_id(oracle):
    # tests/test_aebs.cpp:160-167 and aebs.cpp:137-162 (min bad id for schedule())
    m = CSRMap.from_lists(2, 2, [[0], [1]])
    with pytest.raises(ScheduleError) as ei:
        oracle.schedule(np.array([0, 3, 5, 2], np.int32), 4, 1, m)
    assert ei.value.bad == 2
    with pytest.raises(ScheduleError) as ei:
        oracle.schedule(np.array([0, 3, 5, 2], np.int32), 4, 1, m, bad_mode=1)
    assert ei.value.bad == 3


def test_dispatch_layout_definition(oracle):
    # A9: rows grouped by (instance, replica id, expert), slots ascending
    g = json.load(open(os.path.join(GOLD, "sample_fixture.json")))
    mj = g["map"]
    m = CSRMap(mj["E"], mj["N"], mj["C"], *(np.array(mj[x], np.int32)
                                          for x in ("off", "hosts", "rid")))
    ex = np.array(g["experts"], np.int32)
    a = oracle.schedule(ex, g["T"], g["k"], m)
    qidx, qexp, qbase = oracle.replica_order(m)
    goff, slot_row, row_slot = oracle.dispatch_layout(ex, g["T"], g["k"], m, qidx,
                                                      a.expert_instance)
    S = len(ex)
    assert sorted(slot_row.tolist()) == list(range(S))
    assert np.array_equal(row_slot[slot_row], np.arange(S))
    # per-instance row ranges hold exactly that instance's slots, routed_tokens rows each
    for gi in range(m.N):
        lo, hi = goff[qbase[gi]], goff[qbase[gi + 1]]
        assert hi - lo == a.routed_tokens[gi]
        assert all(a.instance[row_slot[r]] == gi for r in range(lo, hi))
    # keys non-decreasing along rows
    keys = [(a.instance[s], int(a.replica[s]), int(ex[s]), s) for s in row_slot]
    assert keys == sorted(keys)


def test_gate_definition(oracle):
    """or_gate (§8(f) 1) against a numpy restatement: logits in float64 over
    the bf16 inputs, top-k by (logit desc, id asc), softmax of the selected."""
    rng = np.random.default_rng(3)
    T, d_h, E, k = 40, 64, 32, 4
    x = rng.standard_normal((T, d_h)).astype(np.float32)
    w = (rng.standard_normal((E, d_h)) / 8).astype(np.float32)
    w[5] = w[9]  # an exact tie: experts 5 and 9 always share a logit
    xb, wb = oracle.f32_to_bf16(x), oracle.f32_to_bf16(w)
    ex, gw, lg = oracle.gate(xb, wb, k, want_logits=True)
    xf = (xb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    wf = (wb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    ref = xf @ wf.T
    np.testing.assert_allclose(lg, ref, rtol=1e-12, atol=1e-12)
    for t in range(T):
        order = sorted(range(E), key=lambda e: (-ref[t, e], e))[:k]
        assert list(ex[t * k:(t + 1) * k]) == order
        z = np.exp(ref[t, order] - ref[t, order[0]])
        np.testing.assert_allclose(gw[t * k:(t + 1) * k], z / z.sum(), rtol=1e-6)
        if 5 in order and 9 in order:
            assert order.index(5) < order.index(9)
