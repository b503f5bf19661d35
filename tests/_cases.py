"""Case generators restated from the reference's own tests (test helpers).

* :func:`aebs_random_case`  — tests/test_aebs.cpp:47-78 ``random_case`` (300 seeded
  small instances, :116-145).
* :func:`c02_instance`      — tests/acceptance.cpp:108-136 C02 (500 seeded instances,
  frozen gap histogram {496,4,0} at :84), with ``Draw`` (:29-35), ``make_map``
  (:37-51) and ``pick_distinct`` (:53-61).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def hash_label(label: str) -> int:
    h = 0xCBF29CE484222325
    for c in label.encode():
        h ^= c
        h = (h * 0x100000001B3) & M64
    return h


def derive_seed(root: int, label: str, extra: int = 0) -> int:
    s, _ = splitmix64(root)
    s ^= hash_label(label)
    s, _ = splitmix64(s)
    _, e = splitmix64(extra)
    s ^= e
    _, out = splitmix64(s)
    return out


class Rng:
    def __init__(self, seed: int):
        self.s = seed

    def next_u64(self) -> int:
        self.s, v = splitmix64(self.s)
        return v

    def next_below(self, n: int) -> int:
        if n == 0:
            return 0
        threshold = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= threshold:
                return r % n


def map_lists_dealt(N, C, hosts):
    """test_aebs.cpp:18-31 map_from: hosts sorted, ids g*slots + next[g]."""
    hosts = [sorted(h) for h in hosts]
    nxt = [0] * N
    rids = []
    for h in hosts:
        rr = []
        for g in h:
            rr.append(g * C + nxt[g])
            nxt[g] += 1
        rids.append(rr)
    return hosts, rids


def aebs_random_case(seed: int):
    rng = Rng(derive_seed(seed, "aebs/case"))
    E = 2 + rng.next_below(5)
    N = 1 + rng.next_below(3)
    T = 1 + rng.next_below(8)
    k = 1 + rng.next_below(min(E, 3))
    hosts = []
    for _ in range(E):
        r = 1 + rng.next_below(N)
        allg = list(range(N))
        for i in range(r):
            j = i + rng.next_below(N - i)
            allg[i], allg[j] = allg[j], allg[i]
        hosts.append(allg[:r])
    C = E + 2
    hosts, rids = map_lists_dealt(N, C, hosts)
    ex = []
    for _ in range(T):
        alle = list(range(E))
        for j in range(k):
            jj = j + rng.next_below(E - j)
            alle[j], alle[jj] = alle[jj], alle[j]
            ex.append(alle[j])
    return dict(E=E, N=N, C=C, T=T, k=k, hosts=hosts, rids=rids,
                experts=np.array(ex, np.int32))


class Draw:
    def __init__(self, seed):
        self.s = seed

    def u(self):
        self.s, v = splitmix64(self.s)
        return v

    def range(self, lo, hi):
        return lo + self.u() % (hi - lo + 1)


def c02_instance(i: int):
    """Returns (E, N, C, T, k, hosts, rids, gen_seed) for acceptance C02 instance i.
    The batch is gen_batch(uniform(E), T, k, gen_seed, step=i)."""
    d = Draw(derive_seed(0xACCE, "oracle-gap", i))
    e_cnt = d.range(1, 6)
    n_inst = d.range(1, 3)
    k = d.range(1, min(e_cnt, 3))
    tokens = d.range(1, 8)
    hosts = []
    for _ in range(e_cnt):
        r = d.range(1, n_inst)
        idx = list(range(n_inst))
        for j in range(r):
            jj = j + d.u() % (n_inst - j)
            idx[j], idx[jj] = idx[jj], idx[j]
        hosts.append(sorted(idx[:r]))
    nxt = [0] * n_inst
    rids = []
    for h in hosts:
        rr = []
        for g in h:
            rr.append(nxt[g])
            nxt[g] += 1
        rids.append(rr)
    C = max(1, max(nxt))
    gen_seed = d.u()
    return e_cnt, n_inst, C, tokens, k, hosts, rids, gen_seed
