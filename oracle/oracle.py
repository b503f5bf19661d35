"""ctypes front end to the parity checkers.

TEST INFRASTRUCTURE ONLY — imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline / ``--impl reference`` leg.  The product package never
imports this module.

* :class:`Oracle` wraps ``oracle/liboracle.so`` — the C restatement in
  ``oracle/oracle.c`` (each function cites the reference file:line it follows).
* :class:`Ref` wraps ``oracle/_ref/libmoesim_ref.so`` — the reference library
  itself compiled from ``/root/reference/proj/src`` by ``oracle/Makefile``
  (present wherever it was built; it travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoesim_ref.so")

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")

POLICY_AEBS, POLICY_RANDOM, POLICY_BRUTE = 0, 1, 2
OK, EINVAL, EUNKNOWN_EXPERT, EINFEASIBLE = 0, 1, 2, 3


@dataclass
class CSRMap:
    """ReplicaMap (include/moesim/aebs.hpp:29-38) in CSR form."""

    E: int
    N: int
    C: int
    off: np.ndarray
    hosts: np.ndarray
    rid: np.ndarray

    @staticmethod
    def from_lists(N: int, C: int, hosts, rids=None) -> "CSRMap":
        off = np.zeros(len(hosts) + 1, np.int32)
        for e, h in enumerate(hosts):
            off[e + 1] = off[e] + len(h)
        flat_h = np.array([g for h in hosts for g in h], np.int32)
        if rids is None:  # dealt per instance in ascending expert order (aebs.cpp:437-446)
            nxt = [0] * N
            flat_r = []
            for h in hosts:
                for g in h:
                    flat_r.append(g * C + nxt[g])
                    nxt[g] += 1
            rids_arr = np.array(flat_r, np.int32)
        else:
            rids_arr = np.array([r for rr in rids for r in rr], np.int32)
        return CSRMap(len(hosts), N, C, off, flat_h, rids_arr)

    @staticmethod
    def from_map_text(text: str) -> "CSRMap":
        """The committed config maps (``paper_2512_13525_b200/maps/*.map``):
        the reference replica-map text format (aebs.cpp:381-449) with explicit
        physical ids ``e: g:rid ...``, or dealt ids ``e: g ...`` (aebs.cpp:437-446).
        Test/bench infrastructure: lets the bench's reference arm read the maps
        without importing the product."""
        N = C_ = 0
        rows = {}
        for raw in text.splitlines():
            s = raw.split("#", 1)[0].strip()
            if not s:
                continue
            if "=" in s and (":" not in s or s.index("=") < s.index(":")):
                key, val = (x.strip() for x in s.split("=", 1))
                if key == "instances":
                    N = int(val)
                elif key == "slots_per_instance":
                    C_ = int(val)
                continue
            e, rest = s.split(":", 1)
            rows[int(e)] = sorted((int(t.split(":")[0]), int(t.split(":")[1]) if ":" in t else None)
                                  for t in rest.split())
        hosts = [[g for g, _ in rows[e]] for e in range(len(rows))]
        rids = [[r for _, r in rows[e]] for e in range(len(rows))]
        if any(r is None for rr in rids for r in rr):
            return CSRMap.from_lists(N, C_, hosts)
        return CSRMap.from_lists(N, C_, hosts, rids)

    def hosts_of(self, e):
        return self.hosts[self.off[e]:self.off[e + 1]]

    def rids_of(self, e):
        return self.rid[self.off[e]:self.off[e + 1]]


@dataclass
class Sched:
    instance: np.ndarray
    replica: np.ndarray
    expert_instance: np.ndarray
    load: np.ndarray
    routed_tokens: np.ndarray
    expert_tokens: np.ndarray | None = None

    def max_load(self) -> int:
        return int(self.load.max()) if self.load.size else 0


class ScheduleError(Exception):
    def __init__(self, code, bad, msg=""):
        super().__init__(msg or f"status {code} bad={bad}")
        self.code = code
        self.bad = bad


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.or_derive_seed.restype = C.c_uint64
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        for n in ("or_pattern_uniform",):
            getattr(L, n).argtypes = [C.c_int, f64p, f64p]
        L.or_pattern_gaussian.argtypes = [C.c_int, C.c_double, f64p, f64p]
        L.or_pattern_from_pmf.argtypes = [f64p, C.c_int, f64p, f64p]
        L.or_gen_batch.argtypes = [f64p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                   C.c_int, i32p]
        L.or_schedule.argtypes = [C.c_int, C.c_int, C.c_uint64, i32p, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, i32p, i32p, i32p, i32p, i32p, i32p, i32p,
                                  i64p, i64p, C.POINTER(C.c_int32)]
        L.or_replica_order.argtypes = [C.c_int, C.c_int, i32p, i32p, i32p, i32p, i32p, i32p]
        L.or_dispatch_layout.argtypes = [i32p, C.c_int, C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                         i32p, i32p, i32p]
        L.or_moe_layer_latency.restype = C.c_double
        L.or_moe_layer_latency.argtypes = [C.c_int, i32p, i64p, C.c_int, C.c_int, C.c_int,
                                           C.c_double, C.c_double, C.c_double]
        L.or_expert_swiglu.argtypes = [u16p, C.c_int, u16p, u16p, u16p, C.c_int, C.c_int, C.c_int,
                                       C.c_int, f32p]
        L.or_combine.argtypes = [f32p, i32p, f32p, C.c_int, C.c_int, C.c_int, f32p]
        L.or_f32_to_bf16.argtypes = [f32p, u16p, C.c_longlong]
        L.or_stats_record.argtypes = [C.c_int, C.c_int, C.c_longlong, u32p, i64p, i64p, i32p,
                                      C.c_int]
        L.or_gate.argtypes = [u16p, u16p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, f32p,
                              C.c_void_p]
        L.or_num_threads.restype = C.c_int

    # --- rng / routing ------------------------------------------------------
    def splitmix64(self, state: int, n: int = 1):
        s = C.c_uint64(state)
        return [self.L.or_splitmix64(C.byref(s)) for _ in range(n)]

    def derive_seed(self, root: int, label: str, extra: int = 0) -> int:
        return self.L.or_derive_seed(root, label.encode(), extra)

    def pattern(self, kind: str, E: int, sigma: float = 0.15, weights=None):
        pmf = np.zeros(E, np.float64)
        cdf = np.zeros(E, np.float64)
        if kind == "uniform":
            rc = self.L.or_pattern_uniform(E, pmf, cdf)
        elif kind == "gaussian":
            rc = self.L.or_pattern_gaussian(E, sigma, pmf, cdf)
        else:
            rc = self.L.or_pattern_from_pmf(np.ascontiguousarray(weights, np.float64), E, pmf, cdf)
        if rc:
            raise ValueError("invalid routing pattern")
        return pmf, cdf

    def gen_batch(self, cdf: np.ndarray, T: int, k: int, seed: int, step: int,
                  cover_all: bool = False) -> np.ndarray:
        out = np.zeros(T * k, np.int32)
        rc = self.L.or_gen_batch(cdf, len(cdf), T, k, seed, step, int(cover_all), out)
        if rc:
            raise ValueError(f"gen_batch status {rc}")
        return out

    # --- scheduler ----------------------------------------------------------
    def schedule(self, experts: np.ndarray, T: int, k: int, m: CSRMap, policy=POLICY_AEBS,
                 seed: int = 0, bad_mode: int = 0) -> Sched:
        S = T * k
        out = Sched(np.zeros(S, np.int32), np.zeros(S, np.int32), np.zeros(m.E, np.int32),
                    np.zeros(m.N, np.int32), np.zeros(m.N, np.int64), np.zeros(m.E, np.int64))
        bad = C.c_int32(0)
        ex = np.ascontiguousarray(experts, np.int32)
        rc = self.L.or_schedule(policy, bad_mode, seed, ex, T, k, m.E, m.N, m.C, m.off, m.hosts,
                                m.rid, out.instance, out.replica, out.expert_instance, out.load,
                                out.routed_tokens, out.expert_tokens, C.byref(bad))
        if rc:
            raise ScheduleError(rc, bad.value)
        return out

    def replica_order(self, m: CSRMap):
        R = int(m.off[-1])
        qidx = np.zeros(R, np.int32)
        qexp = np.zeros(R, np.int32)
        qbase = np.zeros(m.N + 1, np.int32)
        self.L.or_replica_order(m.E, m.N, m.off, m.hosts, m.rid, qidx, qexp, qbase)
        return qidx, qexp, qbase

    def dispatch_layout(self, experts, T, k, m: CSRMap, qidx, expert_instance):
        R = int(m.off[-1])
        group_off = np.zeros(R + 1, np.int32)
        slot_row = np.zeros(T * k, np.int32)
        row_slot = np.zeros(T * k, np.int32)
        self.L.or_dispatch_layout(np.ascontiguousarray(experts, np.int32), T, k, m.E, m.off,
                                  m.hosts, qidx, np.ascontiguousarray(expert_instance, np.int32),
                                  group_off, slot_row, row_slot)
        return group_off, slot_row, row_slot

    def moe_layer_latency(self, load, routed, d_h, d_e, bpp=2, peak_flops=1401.8e12,
                          hbm_bw=6372.5e9, t_launch=5e-6):
        return self.L.or_moe_layer_latency(len(load), np.ascontiguousarray(load, np.int32),
                                           np.ascontiguousarray(routed, np.int64), d_h, d_e, bpp,
                                           peak_flops, hbm_bw, t_launch)

    # --- FFN / combine ------------------------------------------------------
    def expert_swiglu(self, x_bf16, wg, wu, wd, round_h=True, nthreads=1):
        n, d_h = x_bf16.shape
        d_e = wg.shape[0]
        y = np.zeros((n, d_h), np.float32)
        if n:
            self.L.or_expert_swiglu(np.ascontiguousarray(x_bf16), n, np.ascontiguousarray(wg),
                                    np.ascontiguousarray(wu), np.ascontiguousarray(wd), d_h, d_e,
                                    int(round_h), nthreads, y)
        return y

    def combine(self, y, slot_row, w, T, k):
        d_h = y.shape[1]
        out = np.zeros((T, d_h), np.float32)
        self.L.or_combine(np.ascontiguousarray(y, np.float32),
                          np.ascontiguousarray(slot_row, np.int32),
                          np.ascontiguousarray(w, np.float32), T, k, d_h, out)
        return out

    def stats_new(self, E, window):
        """ActivationStats restatement state: (E, window, step, ring, counts, coact)."""
        words = (E + 31) // 32
        return {"E": E, "W": window, "step": 0, "ring": np.zeros(window * words, np.uint32),
                "counts": np.zeros(E, np.int64), "coact": np.zeros(E * E, np.int64)}

    def stats_record(self, st, activated):
        a = np.ascontiguousarray(activated, np.int32)
        r = self.L.or_stats_record(st["E"], st["W"], st["step"], st["ring"], st["counts"],
                                   st["coact"], a, len(a))
        if r:
            raise ValueError(f"stats: bad activated set at {r - 1}")
        st["step"] += 1

    def gate(self, x_bf16, wr_bf16, k, want_logits=False):
        """Router logits (double), top-k ids by descending logit (ties: lower
        id), softmax over the selected — the gating definition (§8(f) 1)."""
        T, d_h = x_bf16.shape
        E = wr_bf16.shape[0]
        ex = np.zeros(T * k, np.int32)
        gw = np.zeros(T * k, np.float32)
        lg = np.zeros((T, E), np.float64) if want_logits else None
        self.L.or_gate(np.ascontiguousarray(x_bf16), np.ascontiguousarray(wr_bf16), T, d_h, E, k,
                       ex, gw, lg.ctypes.data if want_logits else None)
        return (ex, gw, lg) if want_logits else (ex, gw)

    def f32_to_bf16(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        out = np.zeros(a.shape, np.uint16)
        self.L.or_f32_to_bf16(a.reshape(-1), out.reshape(-1), a.size)
        return out

    def num_threads(self) -> int:
        return self.L.or_num_threads()


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


class Ref:
    """The reference library compiled from /root/reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_pattern.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, f64p, f64p]
        L.ref_gen_batch.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int, C.c_int,
                                    C.c_uint64, C.c_uint64, C.c_int, i32p]
        L.ref_schedule.argtypes = [C.c_int, C.c_uint64, i32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int, i32p, i32p, i32p, i32p, i32p, i32p, i32p, i64p]
        L.ref_map_validate.argtypes = [C.c_int, C.c_int, C.c_int, i32p, i32p, i32p]
        L.ref_time_schedule.restype = C.c_double
        L.ref_time_schedule.argtypes = [C.c_int, C.c_uint64, i32p, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, i32p, i32p, i32p, C.c_int,
                                        C.c_int, C.POINTER(C.c_longlong)]
        L.ref_placement.argtypes = [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_int, C.c_uint64, i32p, i32p, i32p]
        L.ref_stats_new.restype = C.c_void_p
        L.ref_stats_new.argtypes = [C.c_int, C.c_int]
        L.ref_stats_free.argtypes = [C.c_void_p]
        L.ref_stats_record.argtypes = [C.c_void_p, i32p, C.c_int]
        L.ref_stats_read.argtypes = [C.c_void_p, i64p, i64p]
        L.ref_moe_layer_latency.restype = C.c_double
        L.ref_moe_layer_latency.argtypes = [C.c_int, i32p, i64p, C.c_int, C.c_int, C.c_int,
                                            C.c_double, C.c_double, C.c_double]
        L.ref_load_replica_map_text.argtypes = [C.c_char_p, C.POINTER(C.c_int),
                                                C.POINTER(C.c_int), C.POINTER(C.c_int), i32p,
                                                i32p, i32p, C.c_int]
        L.ref_load_batch_text.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          i32p, C.c_int]
        L.ref_dump_assignment.argtypes = [i32p, C.c_int, C.c_int, C.c_int, i32p, i32p, i64p,
                                          C.c_char_p, C.c_int, C.POINTER(C.c_int)]

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    @staticmethod
    def _kind(kind):
        return {"uniform": 0, "gaussian": 1, "pmf": 2}[kind]

    def pattern(self, kind, E, sigma=0.15, weights=None):
        pmf = np.zeros(E, np.float64)
        cdf = np.zeros(E, np.float64)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        rc = self.L.ref_pattern(self._kind(kind), E, sigma,
                                None if w is None else w.ctypes.data, pmf, cdf)
        if rc:
            raise ValueError(self.err())
        return pmf, cdf

    def gen_batch(self, kind, E, T, k, seed, step, sigma=0.15, weights=None, cover_all=False):
        out = np.zeros(T * k, np.int32)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        rc = self.L.ref_gen_batch(self._kind(kind), E, sigma, None if w is None else w.ctypes.data,
                                  T, k, seed, step, int(cover_all), out)
        if rc:
            raise ValueError(self.err())
        return out

    def schedule(self, experts, T, k, m: CSRMap, policy="schedule", seed=0) -> Sched:
        p = {"schedule": 0, "reference": 1, "random": 2, "brute": 3}[policy]
        S = T * k
        out = Sched(np.zeros(S, np.int32), np.zeros(S, np.int32), np.zeros(m.E, np.int32),
                    np.zeros(m.N, np.int32), np.zeros(m.N, np.int64))
        rc = self.L.ref_schedule(p, seed, np.ascontiguousarray(experts, np.int32), T, k, m.E, m.N,
                                 m.C, m.off, m.hosts, m.rid, out.instance, out.replica,
                                 out.expert_instance, out.load, out.routed_tokens)
        if rc:
            raise ScheduleError(rc, None, self.err())
        return out

    def time_schedule(self, batches: np.ndarray, T, k, m: CSRMap, policy="schedule", seed=0,
                      reps=101, warmup=3) -> float:
        p = {"schedule": 0, "reference": 1, "random": 2}[policy]
        nb = batches.size // (T * k)
        sink = C.c_longlong(0)
        return self.L.ref_time_schedule(p, seed, np.ascontiguousarray(batches, np.int32), nb, T, k,
                                        m.E, m.N, m.C, m.off, m.hosts, m.rid, reps, warmup,
                                        C.byref(sink))

    def placement(self, kind, E, k, N, C_, seed, warm_steps=32, warm_tokens=256, sigma=0.15,
                  weights=None) -> CSRMap:
        off = np.zeros(E + 1, np.int32)
        hosts = np.zeros(N * C_, np.int32)
        rid = np.zeros(N * C_, np.int32)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        rc = self.L.ref_placement(self._kind(kind), E, sigma, None if w is None else w.ctypes.data,
                                  k, N, C_, warm_steps, warm_tokens, seed, off, hosts, rid)
        if rc:
            raise ValueError(self.err())
        R = int(off[-1])
        return CSRMap(E, N, C_, off, hosts[:R].copy(), rid[:R].copy())

    def stats(self, E, window, steps):
        """The reference ActivationStats fed `steps` (lists of activated ids):
        (counts [E], coact [E*E]); raises ValueError with the reference's
        message on a rejected step."""
        h = self.L.ref_stats_new(E, window)
        if not h:
            raise ValueError(self.err())
        try:
            for a in steps:
                a = np.ascontiguousarray(a, np.int32)
                if self.L.ref_stats_record(h, a, len(a)):
                    raise ValueError(self.err())
            counts = np.zeros(E, np.int64)
            coact = np.zeros(E * E, np.int64)
            self.L.ref_stats_read(h, counts, coact)
            return counts, coact
        finally:
            self.L.ref_stats_free(h)

    def moe_layer_latency(self, load, routed, d_h, d_e, bpp=2, peak_flops=1401.8e12,
                          hbm_bw=6372.5e9, t_launch=5e-6):
        return self.L.ref_moe_layer_latency(len(load), np.ascontiguousarray(load, np.int32),
                                            np.ascontiguousarray(routed, np.int64), d_h, d_e, bpp,
                                            peak_flops, hbm_bw, t_launch)

    def load_replica_map_text(self, text: str, cap: int = 1 << 16) -> CSRMap:
        E, N, C_ = C.c_int(), C.c_int(), C.c_int()
        off = np.zeros(cap + 1, np.int32)
        hosts = np.zeros(cap, np.int32)
        rid = np.zeros(cap, np.int32)
        rc = self.L.ref_load_replica_map_text(text.encode(), C.byref(E), C.byref(N), C.byref(C_),
                                              off, hosts, rid, cap)
        if rc:
            raise ValueError(self.err())
        R = int(off[E.value])
        return CSRMap(E.value, N.value, C_.value, off[:E.value + 1].copy(), hosts[:R].copy(),
                      rid[:R].copy())

    def load_batch_text(self, text: str, cap: int = 1 << 20):
        T, k = C.c_int(), C.c_int()
        ex = np.zeros(cap, np.int32)
        rc = self.L.ref_load_batch_text(text.encode(), C.byref(T), C.byref(k), ex, cap)
        if rc:
            raise ValueError(self.err())
        return ex[:T.value * k.value].copy(), T.value, k.value

    def dump_assignment(self, experts, T, k, a: Sched) -> str:
        cap = 64 + 12 * T * k + 64 * len(a.load) + 1024
        buf = C.create_string_buffer(cap)
        ln = C.c_int()
        rc = self.L.ref_dump_assignment(np.ascontiguousarray(experts, np.int32), T, k, len(a.load),
                                        a.replica, a.load, a.routed_tokens, buf, cap, C.byref(ln))
        if rc:
            raise ValueError("buffer")
        return buf.value.decode()
