"""Python mirror of the reference moesim API for the hot path, backed by the C ABI.

Same names, argument meaning and error behaviour as the reference C++ library
(paths relative to /root/reference/proj):

* :class:`ActivationBatch`, :class:`ReplicaMap`, :class:`Assignment`
  (include/moesim/aebs.hpp:15-50) with ``validate`` raising
  :class:`ValidationError` (include/moesim/types.hpp:20-22).
* :func:`schedule`, :func:`schedule_random` (aebs.hpp:63-71) — run on the GPU by
  the fused sm_100a scheduler kernel; there is no CPU path.
* synthetic routing (RoutingPattern / gen_batch, workload.hpp:14-32) is not
  part of the product: tests and the bench use oracle/routing.py.
* text formats :func:`load_batch`, :func:`load_replica_map`,
  :func:`dump_assignment` (src/aebs.cpp:338-479); ``load_replica_map`` also reads
  the explicit-id extension ``expert: instance:replica_id ...`` used by the
  committed config maps.
* :func:`moe_layer_latency` (include/moesim/latency.hpp:25-35).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from ._lib import (EINVAL, EUNKNOWN_EXPERT, OK, POLICY_AEBS, POLICY_RANDOM, STATUS_NAMES,
                   JanusAssignment, LatencyModel, lib)

MAPS_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "maps")


class ParseError(RuntimeError):
    """types.hpp:13-16"""


class ValidationError(RuntimeError):
    """types.hpp:18-22"""


class JanusError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ------------------------------------------------------------------ types --

@dataclass
class ActivationBatch:
    """aebs.hpp:15-24; experts[t*k+j] is token t's j-th activation."""

    num_tokens: int
    top_k: int
    experts: np.ndarray

    def __post_init__(self):
        self.experts = np.ascontiguousarray(self.experts, dtype=np.int32).reshape(-1)

    def at(self, t: int, j: int) -> int:
        return int(self.experts[t * self.top_k + j])

    def slots(self) -> int:
        return self.num_tokens * self.top_k

    def validate(self, num_experts: int) -> None:
        """aebs.cpp:29-47."""
        if self.num_tokens < 0 or self.top_k <= 0:
            raise ValidationError("batch: num_tokens must be >= 0 and top_k >= 1")
        if self.experts.size != self.slots():
            raise ValidationError("batch: expert list length != num_tokens * top_k")
        ex = self.experts.reshape(self.num_tokens, self.top_k)
        for t in range(self.num_tokens):
            for j in range(self.top_k):
                e = int(ex[t, j])
                if e < 0 or e >= num_experts:
                    raise ValidationError(
                        f"batch: token {t} names expert {e} outside [0, {num_experts})")
                if e in ex[t, :j]:
                    raise ValidationError(f"batch: token {t} lists expert {e} twice")


@dataclass
class ReplicaMap:
    """aebs.hpp:29-38: hosts[e] ascending instance ids, replica_ids[e] opaque ids."""

    num_experts: int
    num_instances: int
    slots_per_instance: int
    hosts: list
    replica_ids: list

    def replica_count(self, e: int) -> int:
        return len(self.hosts[e])

    def csr(self):
        off = np.zeros(self.num_experts + 1, np.int32)
        for e in range(self.num_experts):
            off[e + 1] = off[e] + len(self.hosts[e])
        hosts = np.array([g for h in self.hosts for g in h], np.int32)
        rid = np.array([r for rr in self.replica_ids for r in rr], np.int32)
        return off, hosts, rid

    def validate(self) -> None:
        """aebs.cpp:49-77 (same messages)."""
        if self.num_experts <= 0 or self.num_instances <= 0 or self.slots_per_instance <= 0:
            raise ValidationError("replica map: dimensions must be positive")
        if len(self.hosts) != self.num_experts or len(self.replica_ids) != len(self.hosts):
            raise ValidationError("replica map: per-expert tables sized wrong")
        used = [0] * self.num_instances
        for e in range(self.num_experts):
            hs = self.hosts[e]
            if not hs:
                raise ValidationError(f"replica map: expert {e} has no replica")
            if len(self.replica_ids[e]) != len(hs):
                raise ValidationError(f"replica map: expert {e} replica id list sized wrong")
            for i, g in enumerate(hs):
                if g < 0 or g >= self.num_instances:
                    raise ValidationError(f"replica map: expert {e} hosted on invalid instance {g}")
                if i > 0 and hs[i - 1] >= g:
                    raise ValidationError(
                        f"replica map: expert {e} host list not strictly ascending")
                used[g] += 1
        for g, u in enumerate(used):
            if u > self.slots_per_instance:
                raise ValidationError(f"replica map: instance {g} holds {u} replicas, capacity "
                                      f"{self.slots_per_instance}")

    @staticmethod
    def from_hosts(num_instances: int, slots_per_instance: int, hosts) -> "ReplicaMap":
        """Replica ids dealt per instance in ascending expert order (aebs.cpp:437-446)."""
        hosts = [sorted(int(g) for g in h) for h in hosts]
        nxt = [0] * num_instances
        rids = []
        for h in hosts:
            rr = []
            for g in h:
                rr.append(g * slots_per_instance + nxt[g])
                nxt[g] += 1
            rids.append(rr)
        m = ReplicaMap(len(hosts), num_instances, slots_per_instance, hosts, rids)
        m.validate()
        return m


@dataclass
class Assignment:
    """aebs.hpp:42-50."""

    instance: np.ndarray
    replica: np.ndarray
    expert_instance: np.ndarray
    load: np.ndarray
    routed_tokens: np.ndarray
    expert_tokens: np.ndarray | None = field(default=None, repr=False)

    def max_load(self) -> int:
        return int(self.load.max()) if self.load.size else 0


def max_activated_load(a: Assignment) -> int:
    return a.max_load()


# -------------------------------------------------------------- scheduler --

class Scheduler:
    """A device context holding one uploaded replica map (re-pushed only on
    reconfiguration).  Every call runs the sm_100a kernel."""

    def __init__(self, rmap: ReplicaMap, device: int = 0):
        self.map = rmap
        self.device = device
        self.ctx = C.c_void_p()
        st = lib.janus_create(C.byref(self.ctx), device)
        if st != OK:
            raise JanusError(st, f"janus_create(device={device}) failed (is a GPU visible?)")
        off, hosts, rid = rmap.csr()
        self._csr = (off, hosts, rid)
        st = lib.janus_set_replica_map(self.ctx, rmap.num_experts, rmap.num_instances,
                                       rmap.slots_per_instance, _ptr(off), _ptr(hosts), _ptr(rid))
        if st == EINVAL:
            raise ValidationError(self.last_error())
        if st != OK:
            raise JanusError(st, self.last_error())

    def set_map(self, rmap: ReplicaMap) -> None:
        """Reconfiguration: upload a new replica map (janus_set_replica_map)."""
        off, hosts, rid = rmap.csr()
        st = lib.janus_set_replica_map(self.ctx, rmap.num_experts, rmap.num_instances,
                                       rmap.slots_per_instance, _ptr(off), _ptr(hosts), _ptr(rid))
        if st == EINVAL:
            raise ValidationError(self.last_error())
        if st != OK:
            raise JanusError(st, self.last_error())
        self.map = rmap
        self._csr = (off, hosts, rid)

    def last_error(self) -> str:
        return lib.janus_last_error(self.ctx).decode()

    def close(self):
        if self.ctx:
            lib.janus_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def replica_order(self):
        R = int(self._csr[0][-1])
        qidx = np.zeros(R, np.int32)
        qbase = np.zeros(self.map.num_instances + 1, np.int32)
        lib.janus_replica_order(self.ctx, _ptr(qidx), _ptr(qbase))
        return qidx, qbase

    def _run(self, batch: ActivationBatch, policy: int, seed: int) -> Assignment:
        S = batch.slots()
        E, N = self.map.num_experts, self.map.num_instances
        a = Assignment(np.zeros(S, np.int32), np.zeros(S, np.int32), np.zeros(E, np.int32),
                       np.zeros(N, np.int32), np.zeros(N, np.int64), np.zeros(E, np.int64))
        ex = batch.experts
        st = lib.janus_schedule(self.ctx, _ptr(ex), batch.num_tokens, batch.top_k, policy,
                                seed, _ptr(a.instance), _ptr(a.replica), _ptr(a.expert_instance),
                                _ptr(a.load), _ptr(a.routed_tokens), _ptr(a.expert_tokens))
        if st in (EUNKNOWN_EXPERT, EINVAL):
            raise ValidationError(self.last_error())
        if st != OK:
            raise JanusError(st, self.last_error())
        return a

    def schedule(self, batch: ActivationBatch) -> Assignment:
        return self._run(batch, POLICY_AEBS, 0)

    def schedule_random(self, batch: ActivationBatch, seed: int) -> Assignment:
        return self._run(batch, POLICY_RANDOM, seed)

    def schedule_async(self, d_experts, num_tokens: int, top_k: int, out: dict,
                       policy: int = POLICY_AEBS, seed: int = 0, stream: int = 0) -> None:
        """Device-pointer variant: d_experts and every value of ``out`` are torch
        CUDA tensors (keys as janus_assignment fields)."""
        a = JanusAssignment(**{k: (v.data_ptr() if v is not None else None)
                               for k, v in out.items()})
        st = lib.janus_schedule_async(self.ctx, d_experts.data_ptr(), num_tokens, top_k, policy,
                                      seed, C.byref(a), stream)
        if st != OK:
            raise JanusError(st, self.last_error())

    def time_schedule(self, d_experts, num_tokens: int, top_k: int, policy: int = POLICY_AEBS,
                      reps: int = 101) -> float:
        us = C.c_double()
        st = lib.janus_time_schedule(self.ctx, d_experts.data_ptr(), num_tokens, top_k, policy,
                                     reps, C.byref(us))
        if st != OK:
            raise JanusError(st, self.last_error())
        return us.value

    def launches(self) -> int:
        return int(lib.janus_launch_count(self.ctx))


_SCHEDULERS: dict = {}


def _scheduler_for(rmap: ReplicaMap) -> Scheduler:
    key = id(rmap)
    s = _SCHEDULERS.get(key)
    if s is None or s.map is not rmap:
        s = Scheduler(rmap)
        _SCHEDULERS[key] = s
    return s


def schedule(batch: ActivationBatch, rmap: ReplicaMap) -> Assignment:
    """moesim::schedule (aebs.hpp:63) on the GPU."""
    return _scheduler_for(rmap).schedule(batch)


schedule_reference = schedule  # identical outputs by contract (aebs.hpp:65-67)


def schedule_random(batch: ActivationBatch, rmap: ReplicaMap, seed: int) -> Assignment:
    """moesim::schedule_random (aebs.hpp:69-71) on the GPU."""
    return _scheduler_for(rmap).schedule_random(batch, seed)


# --------------------------------------------------------------- workload --

def derive_seed(root: int, label: str, extra: int = 0) -> int:
    return int(lib.janus_derive_seed(root, label.encode(), extra))


# ------------------------------------------------------------ text formats --

def _strip(line: str) -> str:
    return line.split("#", 1)[0].strip()


def load_batch(text: str) -> ActivationBatch:
    """aebs.cpp:338-365."""
    rows, k, max_e = [], 0, -1
    for ln, raw in enumerate(text.splitlines(), 1):
        s = _strip(raw)
        if not s:
            continue
        try:
            ids = [int(x) for x in s.split()]
        except ValueError:
            raise ParseError(f"batch line {ln}: expected integers") from None
        if k == 0:
            k = len(ids)
        if len(ids) != k:
            raise ParseError(f"batch line {ln}: expected {k} experts, got {len(ids)}")
        max_e = max([max_e, *ids])
        rows.extend(ids)
    if not rows:
        raise ParseError("batch file: no tokens")
    b = ActivationBatch(len(rows) // k, k, np.array(rows, np.int32))
    b.validate(max_e + 1)
    return b


def load_replica_map(text: str) -> ReplicaMap:
    """aebs.cpp:381-449, plus explicit ids ``e: g:rid ...``."""
    N = C_ = 0
    rows = []
    for ln, raw in enumerate(text.splitlines(), 1):
        s = _strip(raw)
        if not s:
            continue
        eq, colon = s.find("="), s.find(":")
        if eq >= 0 and (colon < 0 or eq < colon):
            key, val = s[:eq].strip(), s[eq + 1:].strip()
            try:
                v = int(val)
            except ValueError:
                raise ParseError(f"replica map line {ln}: bad value for '{key}'") from None
            if key == "instances":
                N = v
            elif key == "slots_per_instance":
                C_ = v
            else:
                raise ParseError(f"replica map line {ln}: unknown key '{key}'")
            continue
        if colon < 0:
            raise ParseError(f"replica map line {ln}: expected 'expert: instance...'")
        try:
            e = int(s[:colon])
        except ValueError:
            raise ParseError(f"replica map line {ln}: bad expert id") from None
        toks = s[colon + 1:].split()
        if not toks:
            raise ParseError(f"replica map line {ln}: expected instance ids after ':'")
        try:
            pairs = [(int(t.split(":")[0]), int(t.split(":")[1]) if ":" in t else None)
                     for t in toks]
        except ValueError:
            raise ParseError(f"replica map line {ln}: expected instance ids after ':'") from None
        rows.append((e, pairs))
    if N <= 0 or C_ <= 0:
        raise ParseError("replica map: missing instances/slots_per_instance header")
    E = len(rows)
    hosts = [None] * E
    rids = [None] * E
    for e, pairs in rows:
        if e < 0 or e >= E or hosts[e] is not None:
            raise ParseError(f"replica map: expert ids must cover 0..{E - 1} exactly once "
                             f"(got {e})")
        pairs = sorted(pairs, key=lambda p: p[0])
        hosts[e] = [g for g, _ in pairs]
        rids[e] = [r for _, r in pairs]
    if any(r is None for rr in rids for r in rr):  # dealt ids (reference format)
        nxt = [0] * N
        for e in range(E):
            for i, g in enumerate(hosts[e]):
                if g < 0 or g >= N:
                    raise ParseError(f"replica map: expert {e} placed on invalid instance {g}")
                rids[e][i] = g * C_ + nxt[g]
                nxt[g] += 1
    m = ReplicaMap(E, N, C_, hosts, rids)
    m.validate()
    return m


def load_replica_map_file(path: str) -> ReplicaMap:
    with open(path) as f:
        return load_replica_map(f.read())


def config_map(name: str) -> ReplicaMap:
    """A committed replica map for one of BASELINE.json's configs (maps/*.map)."""
    return load_replica_map_file(os.path.join(MAPS_DIR, f"{name}.map"))


def dump_assignment(a: Assignment, b: ActivationBatch) -> str:
    """aebs.cpp:468-479 (byte-identical output)."""
    out = [f"# assignment: tokens={b.num_tokens} top_k={b.top_k}\n",
           "# per-token physical replica ids\n"]
    rep = a.replica.reshape(b.num_tokens, b.top_k) if b.num_tokens else []
    for t in range(b.num_tokens):
        out.append(" ".join(str(int(x)) for x in rep[t]) + "\n")
    out.append("# instance activated_replicas routed_tokens\n")
    for g in range(len(a.load)):
        out.append(f"load {g} {int(a.load[g])} {int(a.routed_tokens[g])}\n")
    return "".join(out)


# ------------------------------------------------------------ cost model --

@dataclass
class InstanceLoad:
    """latency.hpp:28-31"""

    activated_experts: int = 0
    routed_tokens: int = 0


def moe_layer_latency(loads, hidden_dim: int, expert_dim: int, bytes_per_param: int = 2,
                      peak_flops: float = 989e12, hbm_bandwidth: float = 3.35e12,
                      kernel_launch_overhead: float = 5e-6) -> float:
    """latency.hpp:34-35 (the reference's 2-matrix accounting)."""
    load = np.array([l.activated_experts for l in loads], np.int32)
    routed = np.array([l.routed_tokens for l in loads], np.int64)
    return float(lib.janus_moe_layer_latency(len(load), _ptr(load), _ptr(routed), hidden_dim,
                                             expert_dim, bytes_per_param, peak_flops,
                                             hbm_bandwidth, kernel_launch_overhead))


def shard_tokens(num_tokens: int, attn_instances: int, a: int):
    """comm.cpp:76-81 token ownership: (first, count) of attention shard a."""
    first, count = C.c_int64(), C.c_int64()
    lib.janus_shard_tokens(num_tokens, attn_instances, a, C.byref(first), C.byref(count))
    return first.value, count.value


# ---------------------------------------------- calibrated latency model --

def reference_latency_model(peak_flops: float = 989e12, hbm_bandwidth: float = 3.35e12,
                            kernel_launch_overhead: float = 5e-6,
                            bytes_per_param: int = 2) -> LatencyModel:
    """The reference's model (latency.cpp:17-24) as a janus_latency_model:
    two matrices, max of the memory and compute terms (p = 0)."""
    return LatencyModel(kernel_launch_overhead, hbm_bandwidth, peak_flops, 0.0, 2,
                        bytes_per_param, 1)


def fit_latency_model(activated, routed_tokens, seconds, hidden_dim: int, expert_dim: int,
                      start: LatencyModel | None = None, matrices: int = 3):
    """Fit (t_launch, beta, pi, p) to measured layer times (janus_latency_fit).
    Returns (model, mean absolute relative error)."""
    A = np.ascontiguousarray(activated, np.int32)
    b = np.ascontiguousarray(routed_tokens, np.int64)
    t = np.ascontiguousarray(seconds, np.float64)
    m = start if start is not None else LatencyModel(20e-6, 6.5e12, 1.4e15, 4.0, matrices, 2,
                                                     matrices)
    err = C.c_double()
    st = lib.janus_latency_fit(len(A), _ptr(A), _ptr(b), _ptr(t), hidden_dim, expert_dim,
                               C.byref(m), C.byref(err))
    if st != OK:
        raise JanusError(st, "latency fit: need >= 4 points with positive times")
    return m, err.value


def layer_latency(model: LatencyModel, loads, hidden_dim: int, expert_dim: int) -> float:
    """max over instances of the (calibrated) instance time (janus_latency_layer)."""
    load = np.array([l.activated_experts for l in loads], np.int32)
    routed = np.array([l.routed_tokens for l in loads], np.int64)
    return float(lib.janus_latency_layer(C.byref(model), len(load), _ptr(load), _ptr(routed),
                                         hidden_dim, expert_dim))
