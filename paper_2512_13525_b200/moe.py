"""The MoE layer on one GPU: K1 schedule -> K3 permute -> K4 grouped SwiGLU GEMMs
-> K5 combine, all in libjanus_b200.so.  torch is used only for device memory
and streams.

Weight store: replicas in the replica order the dispatch layout uses
(``Scheduler.replica_order``): for the replicas hosted on an instance, sorted
by (replica id, expert).  ``w13[q] = [Wg; Wu]`` (2*d_e x d_h), ``w2[q] = Wd``
(d_h x d_e), bf16.  A replica holds its logical expert's weights.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import EINVAL, OK, EUNKNOWN_EXPERT, JanusAssignment, lib
from .moesim import JanusError, ReplicaMap, Scheduler, ValidationError, derive_seed


def _cur_stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class MoELayer:
    def __init__(self, rmap: ReplicaMap, d_hidden: int, d_expert: int, max_tokens: int,
                 top_k: int, instance: int = -1, device: int = 0):
        self.sched = Scheduler(rmap, device)
        self.map = rmap
        self.d_h, self.d_e, self.k = d_hidden, d_expert, top_k
        self.max_tokens = max_tokens
        self.instance = instance
        self.device = torch.device("cuda", device)
        st = lib.janus_moe_configure(self.ctx, d_hidden, d_expert, max_tokens, top_k)
        if st != OK:
            raise JanusError(st, self.sched.last_error())
        self._derive_order()
        self.w13 = self.w2 = None

    def _derive_order(self):
        self.qidx, self.qbase = self.sched.replica_order()
        off, _, _ = self.sched._csr
        # expert held at each replica-order index q
        self.q_expert = np.zeros(int(off[-1]), np.int32)
        for e in range(self.map.num_experts):
            for p in range(off[e], off[e + 1]):
                self.q_expert[self.qidx[p]] = e

    def set_map(self, rmap: ReplicaMap) -> None:
        """Replica-map reconfiguration: re-upload the CSR; the
        weight store must be set again (replica order changes)."""
        self.sched.set_map(rmap)
        self.map = rmap
        self._derive_order()
        self.w13 = self.w2 = None

    @property
    def ctx(self):
        return self.sched.ctx

    def local_experts(self) -> np.ndarray:
        """Logical expert of each local weight slot (replica order)."""
        if self.instance < 0:
            return self.q_expert.copy()
        return self.q_expert[self.qbase[self.instance]:self.qbase[self.instance + 1]].copy()

    def set_weights(self, w13: torch.Tensor, w2: torch.Tensor) -> None:
        Q = len(self.local_experts())
        assert w13.shape == (Q, 2 * self.d_e, self.d_h) and w13.dtype == torch.bfloat16
        assert w2.shape == (Q, self.d_h, self.d_e) and w2.dtype == torch.bfloat16
        assert w13.is_cuda and w2.is_cuda and w13.is_contiguous() and w2.is_contiguous()
        self.w13, self.w2 = w13, w2  # keep alive: the context stores raw pointers
        st = lib.janus_moe_set_weights(self.ctx, self.instance, w13.data_ptr(), w2.data_ptr())
        if st != OK:
            raise JanusError(st, self.sched.last_error())

    def forward(self, x: torch.Tensor, experts: torch.Tensor, gate_w: torch.Tensor,
                out: torch.Tensor | None = None, assign: dict | None = None) -> torch.Tensor:
        """Device call on torch's current stream (asynchronous)."""
        T = x.shape[0]
        assert x.dtype == torch.bfloat16 and x.shape[1] == self.d_h and x.is_contiguous()
        assert experts.dtype == torch.int32 and experts.numel() == T * self.k
        assert gate_w.dtype == torch.float32 and gate_w.numel() == T * self.k
        if out is None:
            out = torch.empty_like(x)
        a = None
        if assign is not None:
            a = JanusAssignment(**{k: (v.data_ptr() if v is not None else None)
                                   for k, v in assign.items()})
        st = lib.janus_moe_layer_async(self.ctx, x.data_ptr(), experts.data_ptr(),
                                       gate_w.data_ptr(), T, out.data_ptr(),
                                       C.byref(a) if a is not None else None,
                                       _cur_stream(self.device))
        if st != OK:
            raise JanusError(st, self.sched.last_error())
        return out

    def forward_host(self, x: torch.Tensor, experts: torch.Tensor, gate_w: torch.Tensor,
                     out: torch.Tensor) -> torch.Tensor:
        """End to end from (pinned) host tensors: H2D, layer, D2H, synchronise."""
        T = x.shape[0]
        st = lib.janus_moe_layer(self.ctx, x.data_ptr(), experts.data_ptr(), gate_w.data_ptr(), T,
                                 out.data_ptr())
        if st == EUNKNOWN_EXPERT:
            raise ValidationError(self.sched.last_error())
        if st != OK:
            raise JanusError(st, self.sched.last_error())
        return out

    # --- MoE-side gating ----------------------------------------
    def set_router(self, wr: torch.Tensor) -> None:
        """Router weights [E][d_h] bf16 for :meth:`forward_gated`."""
        assert wr.shape == (self.map.num_experts, self.d_h) and wr.dtype == torch.bfloat16
        assert wr.is_cuda and wr.is_contiguous()
        self.wr = wr  # keep alive: the context stores the raw pointer
        st = lib.janus_moe_set_router(self.ctx, wr.data_ptr())
        if st != OK:
            raise JanusError(st, self.sched.last_error())

    def gate(self, x: torch.Tensor, wr: torch.Tensor | None = None, top_k: int | None = None):
        """(experts int32 [T*k], gate_w fp32 [T*k]) from the gating kernel."""
        wr = self.wr if wr is None else wr
        k = self.k if top_k is None else top_k
        T = x.shape[0]
        ex = torch.empty(T * k, dtype=torch.int32, device=x.device)
        gw = torch.empty(T * k, dtype=torch.float32, device=x.device)
        st = lib.janus_gate_async(self.ctx, x.data_ptr(), wr.data_ptr(), T, x.shape[1],
                                  wr.shape[0], k, ex.data_ptr(), gw.data_ptr(),
                                  _cur_stream(self.device))
        if st != OK:
            raise JanusError(st, self.sched.last_error())
        return ex, gw

    def forward_gated(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Gate on this GPU, then the layer (device call, current stream)."""
        T = x.shape[0]
        assert x.dtype == torch.bfloat16 and x.shape[1] == self.d_h and x.is_contiguous()
        if out is None:
            out = torch.empty_like(x)
        st = lib.janus_moe_layer_gated_async(self.ctx, x.data_ptr(), T, out.data_ptr(),
                                             _cur_stream(self.device))
        if st != OK:
            raise JanusError(st, self.sched.last_error())
        return out

    def set_shared(self, w13: torch.Tensor | None, w2: torch.Tensor | None = None,
                   split: bool = False) -> None:
        """DeepSeek-V3-style shared expert on every token (weight 1):
        w13 [2*d_e][d_h] = [Wg; Wu], w2 [d_h][d_e] bf16; None disables.
        split (box MoE instances): every instance takes an even share of the
        tokens instead of instance 0 taking all (janus_moe_set_shared_split)."""
        if w13 is None:
            self.shared_w = None
            st = lib.janus_moe_set_shared(self.ctx, None, None)
        else:
            assert w13.shape == (2 * self.d_e, self.d_h) and w2.shape == (self.d_h, self.d_e)
            assert w13.dtype == w2.dtype == torch.bfloat16 and w13.is_contiguous()
            assert w2.is_contiguous() and w13.is_cuda and w2.is_cuda
            self.shared_w = (w13, w2)  # keep alive: the context stores raw pointers
            st = lib.janus_moe_set_shared(self.ctx, w13.data_ptr(), w2.data_ptr())
        if st == OK:
            st = lib.janus_moe_set_shared_split(self.ctx, 1 if split else 0)
        if st != OK:
            raise JanusError(st, self.sched.last_error())

    def forward_host_async(self, x: torch.Tensor, experts: torch.Tensor, gate_w: torch.Tensor,
                           out: torch.Tensor) -> None:
        """Pipelined host call (janus_moe_layer_host_async): enqueue H2D, the
        layer and D2H; the copies of neighbouring calls overlap the layer.
        Call :meth:`host_sync` before reading ``out``."""
        T = x.shape[0]
        st = lib.janus_moe_layer_host_async(self.ctx, x.data_ptr(), experts.data_ptr(),
                                            gate_w.data_ptr(), T, out.data_ptr())
        if st != OK:
            raise JanusError(st, self.sched.last_error())

    def host_sync(self) -> None:
        st = lib.janus_moe_host_sync(self.ctx)
        if st == EUNKNOWN_EXPERT:
            raise ValidationError(self.sched.last_error())
        if st != OK:
            raise JanusError(st, self.sched.last_error())

    def launches(self) -> int:
        return self.sched.launches()


def expert_weights(e: int, d_h: int, d_e: int, seed: int, device) -> tuple:
    """Random-init SwiGLU expert e: N(0, 1/sqrt(fan_in)) bf16, seeded by
    derive_seed(seed, "w", e).  Returns (wg [d_e,d_h], wu [d_e,d_h], wd [d_h,d_e])."""
    g = torch.Generator(device=device)
    g.manual_seed(derive_seed(seed, "w", e) & ((1 << 63) - 1))
    wg = torch.randn(d_e, d_h, generator=g, device=device) * (d_h ** -0.5)
    wu = torch.randn(d_e, d_h, generator=g, device=device) * (d_h ** -0.5)
    wd = torch.randn(d_h, d_e, generator=g, device=device) * (d_e ** -0.5)
    return wg.bfloat16(), wu.bfloat16(), wd.bfloat16()


def build_weight_store(layer: MoELayer, seed: int) -> tuple:
    """Weight store for ``layer`` from :func:`expert_weights` (replicas of one
    expert share its weights)."""
    experts = layer.local_experts()
    Q = len(experts)
    w13 = torch.empty(Q, 2 * layer.d_e, layer.d_h, dtype=torch.bfloat16, device=layer.device)
    w2 = torch.empty(Q, layer.d_h, layer.d_e, dtype=torch.bfloat16, device=layer.device)
    cache = {}
    for q, e in enumerate(experts):
        if e not in cache:
            cache = {e: expert_weights(int(e), layer.d_h, layer.d_e, seed, layer.device)}
        wg, wu, wd = cache[e]
        w13[q, :layer.d_e] = wg
        w13[q, layer.d_e:] = wu
        w2[q] = wd
    return w13, w2


def router_weights(E: int, d_h: int, seed: int, device) -> torch.Tensor:
    """Random-init router [E][d_h] bf16, N(0, 1/sqrt(d_h)), seeded by
    derive_seed(seed, "router", E)."""
    g = torch.Generator(device=device)
    g.manual_seed(derive_seed(seed, "router", E) & ((1 << 63) - 1))
    return (torch.randn(E, d_h, generator=g, device=device) * (d_h ** -0.5)).bfloat16()


def make_inputs(T: int, k: int, d_h: int, seed: int, device) -> tuple:
    """x ~ N(0,1) bf16 [T, d_h]; gate weights softmax of seeded N(0,1) logits over
    the k slots, fp32 [T*k]."""
    g = torch.Generator(device=device)
    g.manual_seed(derive_seed(seed, "x", T) & ((1 << 63) - 1))
    x = torch.randn(T, d_h, generator=g, device=device).bfloat16()
    logits = torch.randn(T, k, generator=g, device=device)
    gw = torch.softmax(logits, dim=1).reshape(-1).contiguous()
    return x, gw


class ActivationStats:
    """Device mirror of the reference's ActivationStats (experts.hpp:18-43):
    windowed per-expert activation counts and co-activation matrix, updated
    from a step's routing on the GPU (janus_stats_*)."""

    def __init__(self, num_experts: int, window_steps: int, device: int = 0):
        self.device = torch.device("cuda", device)
        self.ctx = C.c_void_p()
        st = lib.janus_create(C.byref(self.ctx), device)
        if st != OK:
            raise JanusError(st, "janus_create")
        st = lib.janus_stats_configure(self.ctx, num_experts, window_steps)
        if st == EINVAL:
            raise ValidationError(lib.janus_last_error(self.ctx).decode())
        if st != OK:
            raise JanusError(st, lib.janus_last_error(self.ctx).decode())
        self.E, self.W = num_experts, window_steps

    def record_batch(self, experts: torch.Tensor, top_k: int) -> None:
        """record_step(activated set of this routing), asynchronously on the
        current stream."""
        assert experts.dtype == torch.int32 and experts.is_cuda and experts.is_contiguous()
        st = lib.janus_stats_record_async(self.ctx, experts.data_ptr(), experts.numel() // top_k,
                                          top_k, _cur_stream(self.device))
        if st != OK:
            raise JanusError(st, lib.janus_last_error(self.ctx).decode())

    def check(self) -> None:
        """Raise the reference's ValidationError if the last step was rejected."""
        bad = C.c_int()
        if lib.janus_stats_status(self.ctx, C.byref(bad)) == EINVAL:
            raise ValidationError(lib.janus_last_error(self.ctx).decode())

    def read(self):
        """(counts int64 [E], coact int64 [E, E], recorded_steps)."""
        counts = np.zeros(self.E, np.int64)
        coact = np.zeros((self.E, self.E), np.int64)
        rec = C.c_int()
        st = lib.janus_stats_read(self.ctx, counts.ctypes.data_as(C.POINTER(C.c_int64)),
                                  coact.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(rec))
        if st != OK:
            raise JanusError(st, lib.janus_last_error(self.ctx).decode())
        return counts, coact, rec.value

    def __del__(self):
        try:
            if self.ctx:
                lib.janus_destroy(self.ctx)
        except Exception:
            pass
