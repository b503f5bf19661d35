"""One NVLink box split into an attention sub-group and an MoE sub-group.

Ranks ``[0, A)`` own token shards (the attention side: even split, remainder to
the lowest ids, src/comm.cpp:76-81); ranks ``[A, A+M)`` are MoE instances
``g = rank - A``, each holding the replicas AEBS may pick on instance g.  A
decode step's MoE layer is

  attention a:  janus_attn_dispatch_async  — push shard rows + routing + gate
                weights into every MoE rank's memory (NVLink P2P stores), flag
  MoE g:        janus_moe_layer_xfer_async — wait for all shards, K1 schedule
                (replicated, identical on every MoE GPU: no count exchange),
                K3/K4 on this instance's groups, K5 partial sums pushed straight
                into the owners' memory, flag
  attention a:  janus_attn_combine_async   — wait for the M partials, reduce
                (fixed instance order) into the shard's output rows.

torch.distributed is plumbing only: the one-time exchange of CUDA IPC handles.
The data path is libjanus_b200.so's kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._lib import EUNKNOWN_EXPERT, OK, lib
from .moesim import JanusError, ValidationError, shard_tokens


@dataclass(frozen=True)
class BoxPlan:
    """Roles and token ownership of an A-attention + M-MoE box (pure host logic).
    ``colocated``: the MoE-only box — every rank owns a token shard and is MoE
    instance ``rank`` (n_attn == n_moe == world)."""

    n_attn: int
    n_moe: int
    colocated: bool = False

    @property
    def world(self) -> int:
        return self.n_attn if self.colocated else self.n_attn + self.n_moe

    def role(self, rank: int) -> str:
        if self.colocated:
            return "both"
        return "attention" if rank < self.n_attn else "moe"

    def is_attention(self, rank: int) -> bool:
        return self.colocated or rank < self.n_attn

    def is_moe(self, rank: int) -> bool:
        return self.colocated or rank >= self.n_attn

    def instance(self, rank: int) -> int:
        if self.colocated:
            return rank
        return rank - self.n_attn if rank >= self.n_attn else -1

    def shard(self, num_tokens: int, rank: int):
        """(first, count) of attention rank's token shard (comm.cpp:76-81)."""
        assert self.is_attention(rank)
        return shard_tokens(num_tokens, self.n_attn, rank)

    def owner(self, num_tokens: int, t: int) -> int:
        for a in range(self.n_attn):
            first, count = self.shard(num_tokens, a)
            if first <= t < first + count:
                return a
        raise ValueError(t)

    def bytes_per_step(self, num_tokens: int, d_h: int, k: int):
        """NVLink bytes each attention rank sends / receives per step."""
        out = {}
        for a in range(self.n_attn):
            _, ta = self.shard(num_tokens, a)
            send = self.n_moe * ta * (2 * d_h + 8 * k)
            recv = self.n_moe * ta * 2 * d_h
            out[a] = (send, recv)
        return out

    @staticmethod
    def for_gpus(n: int) -> "BoxPlan":
        """Default split used by the benches: 1 attention GPU per 4 (the paper's
        example box is 2 attention + 6 MoE of 8)."""
        a = max(1, n // 4)
        return BoxPlan(a, n - a)

    @staticmethod
    def moe_only(n: int) -> "BoxPlan":
        return BoxPlan(n, n, colocated=True)


class _Ctx:
    """A bare device context (attention ranks of a broadcast box hold no
    replica map; the routed transport gives them one, see JanusBox)."""

    def __init__(self, device: int):
        self.ctx = C.c_void_p()
        st = lib.janus_create(C.byref(self.ctx), device)
        if st != OK:
            raise JanusError(st, f"janus_create(device={device})")

    def last_error(self) -> str:
        return lib.janus_last_error(self.ctx).decode()

    def __del__(self):
        try:
            if self.ctx:
                lib.janus_destroy(self.ctx)
        except Exception:
            pass


TRANSPORTS = ("auto", "p2p", "nvls", "routed", "ce")


class JanusBox:
    """This rank's endpoint of the box exchange.

    For an MoE rank pass ``layer`` (a :class:`paper_2512_13525_b200.moe.MoELayer`
    built with ``instance = rank - n_attn`` and its weight store set).
    ``transport``: ``p2p`` / ``nvls`` broadcast every token to every MoE rank
    (the reference's semantics, comm.hpp:12-14) by SM stores; ``ce`` is the P2P
    broadcast moved by the copy engines (no dispatch kernel: a colocated rank's
    MoE kernels keep every SM); ``routed`` sends a row only to
    the MoE ranks its slots are scheduled on — attention ranks then also need
    the replica map (``rmap``) to run the scheduler; ``auto`` = NVLS when every
    rank supports it, else P2P.  ``combine`` (NVLS only): ``push`` (default) —
    MoE ranks push their partial sums point to point; ``switch`` — the owner
    reads them summed by the NVSwitch (multimem.ld_reduce).

    Multi-process (one rank per GPU): the constructor exchanges the CUDA IPC
    handles over torch.distributed.  One process driving every rank (e.g. all on
    one GPU): :meth:`local`."""

    def __init__(self, plan: BoxPlan, rank: int, max_tokens: int, d_hidden: int, top_k: int,
                 layer=None, device: int = 0, group=None, transport: str = "auto", rmap=None,
                 combine: str = "push", _connect: bool = True):
        if transport not in TRANSPORTS:
            raise ValueError(transport)
        self.plan, self.rank = plan, rank
        self.max_tokens, self.d_h, self.k = max_tokens, d_hidden, top_k
        if plan.is_moe(rank):
            if layer is None or layer.instance != plan.instance(rank):
                raise ValueError("an MoE rank needs its MoELayer with instance = rank - n_attn")
            self.layer = layer
            self._ctx = layer.ctx
            self._err = layer.sched.last_error
        else:
            self.layer = None
            if transport == "routed":  # the attention rank schedules the step too
                if rmap is None:
                    raise ValueError("the routed transport needs the replica map on attention ranks")
                from .moesim import Scheduler
                self._c = Scheduler(rmap, device)
            else:
                self._c = _Ctx(device)
            self._ctx = self._c.ctx
            self._err = self._c.last_error
        if plan.colocated:
            self._check(lib.janus_xfer_configure_colocated(self._ctx, plan.world, rank, max_tokens,
                                                           d_hidden, top_k))
        else:
            self._check(lib.janus_xfer_configure(self._ctx, plan.n_attn, plan.n_moe, rank,
                                                 max_tokens, d_hidden, top_k))
        self.transport = transport if transport in ("routed", "ce") else "p2p"
        if transport in ("routed", "ce"):
            self._check(lib.janus_xfer_set_transport(self._ctx, 1 if transport == "routed" else 2))
        if not _connect:
            return
        import torch.distributed as dist
        h = C.create_string_buffer(64)
        self._check(lib.janus_xfer_handle(self._ctx, h))
        handles = [None] * plan.world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        self._check(lib.janus_xfer_connect(self._ctx, b"".join(handles)))
        dist.barrier(group=group)
        if transport in ("auto", "nvls"):
            yes = C.c_int()
            self._check(lib.janus_xfer_mc_supported(self._ctx, C.byref(yes)))
            every = [None] * plan.world
            dist.all_gather_object(every, bool(yes.value), group=group)
            if all(every):
                self._setup_multicast(dist, group)
                self.transport = "nvls"
                if combine == "switch":  # default: point-to-point push combine
                    self._check(lib.janus_xfer_set_combine(self._ctx, 1))
            elif transport == "nvls":
                raise JanusError(5, "xfer: NVLS multicast not supported on every rank")

    @classmethod
    def local(cls, plan: BoxPlan, max_tokens: int, d_hidden: int, top_k: int, layers: dict,
              devices=None, transport: str = "p2p", rmap=None) -> list:
        """Every rank's endpoint in this process (``layers``: rank -> MoELayer
        of the MoE ranks; ``devices``: rank -> device, default 0), connected
        with raw pointers (janus_xfer_connect_local).  P2P, routed or copy-engine transport.
        Calls into ranks that wait on one another must be enqueued in causal
        order (e.g. on one stream: every dispatch, then every MoE step, then
        every combine)."""
        if transport not in ("p2p", "routed", "ce"):
            raise ValueError("a same-process box uses the p2p, routed or ce transport")
        devices = devices or {}
        boxes = [cls(plan, r, max_tokens, d_hidden, top_k, layer=layers.get(r),
                     device=devices.get(r, 0), transport=transport, rmap=rmap, _connect=False)
                 for r in range(plan.world)]
        arr = (C.c_void_p * plan.world)(*[b._ctx.value for b in boxes])
        for b in boxes:
            b._check(lib.janus_xfer_connect_local(b._ctx, arr))
        return boxes

    def _setup_multicast(self, dist, group) -> None:
        """Rank 0 creates the multicast object; its POSIX fd reaches the other
        ranks over a Unix socket (SCM_RIGHTS); all join, then all bind."""
        import os
        import socket
        import tempfile
        if self.rank == 0:
            fd = C.c_int(-1)
            self._check(lib.janus_xfer_mc_create(self._ctx, C.byref(fd)))
            path = os.path.join(tempfile.gettempdir(), f"janus_mc_{os.getpid()}.sock")
            if os.path.exists(path):
                os.unlink(path)
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(path)
            srv.listen(self.plan.world)
            dist.broadcast_object_list([path], src=0, group=group)
            for _ in range(self.plan.world - 1):
                conn, _ = srv.accept()
                socket.send_fds(conn, [b"fd"], [fd.value])
                conn.close()
            srv.close()
            os.unlink(path)
            os.close(fd.value)
        else:
            obj = [None]
            dist.broadcast_object_list(obj, src=0, group=group)
            cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            cli.connect(obj[0])
            _, fds, _, _ = socket.recv_fds(cli, 16, 1)
            cli.close()
            self._check(lib.janus_xfer_mc_join(self._ctx, fds[0]))
            os.close(fds[0])
        dist.barrier(group=group)
        self._check(lib.janus_xfer_mc_bind(self._ctx))
        dist.barrier(group=group)

    def _check(self, st):
        if st != OK:
            raise JanusError(st, self._err())

    def _check_status(self, st):
        if st == EUNKNOWN_EXPERT:
            raise ValidationError(self._err())
        self._check(st)

    def set_timeout(self, seconds: float) -> None:
        self._check(lib.janus_xfer_set_timeout(self._ctx, int(seconds * 1e9)))

    def check(self) -> None:
        """Raise the first failed step this rank saw since the last check: the
        reference's ValidationError for an unknown expert (on the attention
        side, reported by any MoE rank), JanusError(EPEER) for a peer that
        never published."""
        self._check_status(lib.janus_xfer_check(self._ctx))

    # --- attention rank ------------------------------------------------------
    def route(self, experts_shard, gate_w_shard, num_tokens: int, epoch: int,
              stream: int) -> None:
        """Routed transport: push the routing phase ahead of :meth:`dispatch`."""
        self._check(lib.janus_attn_route_async(self._ctx, experts_shard.data_ptr(),
                                               gate_w_shard.data_ptr(), num_tokens, epoch, stream))

    def dispatch(self, x_shard, experts_shard, gate_w_shard, num_tokens: int, epoch: int,
                 stream: int) -> None:
        """experts / gate_w None: rows only, the MoE ranks gate (set_router)."""
        self._check(lib.janus_attn_dispatch_async(
            self._ctx, x_shard.data_ptr(),
            experts_shard.data_ptr() if experts_shard is not None else None,
            gate_w_shard.data_ptr() if gate_w_shard is not None else None, num_tokens, epoch,
            stream))

    def combine(self, out_shard, num_tokens: int, epoch: int, stream: int) -> None:
        self._check(lib.janus_attn_combine_async(self._ctx, out_shard.data_ptr(), num_tokens,
                                                 epoch, stream))

    # --- MoE rank ---------------------------------------------------------------
    def moe_step(self, num_tokens: int, epoch: int, stream: int) -> None:
        self._check(lib.janus_moe_layer_xfer_async(self._ctx, num_tokens, epoch, stream))

    def recv_rows(self, epoch: int, num_tokens: int):
        """This rank's receive buffer of token rows for ``epoch``'s slot as an
        int16 torch view [num_tokens, d_h] (instrumentation: tests)."""
        import torch
        ptr = C.c_void_p()
        self._check(lib.janus_xfer_recv_rows(self._ctx, epoch, C.byref(ptr)))

        class _Dev:  # __cuda_array_interface__ over the exchange region
            __cuda_array_interface__ = {"data": (ptr.value, False), "typestr": "<i2",
                                        "shape": (num_tokens, self.d_h), "version": 3}
        return torch.as_tensor(_Dev(), device="cuda")

    def timed_out(self) -> bool:
        v = C.c_int()
        self._check(lib.janus_xfer_status(self._ctx, C.byref(v)))
        return bool(v.value)

    def launches(self) -> int:
        return int(lib.janus_launch_count(self._ctx))

