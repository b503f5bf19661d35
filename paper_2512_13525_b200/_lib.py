"""ctypes binding of libjanus_b200.so (the C ABI in include/janus_b200.h).

The library is built in-tree by ``paper_2512_13525_b200/build.py`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing,
importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JANUS_LIB") or os.path.join(PKG, "libjanus_b200.so")  # override: A/B runs

OK, EINVAL, EUNKNOWN_EXPERT, ECUDA, ESTATE, EUNSUPPORTED, EPEER = range(7)
POLICY_AEBS, POLICY_RANDOM = 0, 1
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "EUNKNOWN_EXPERT", 3: "ECUDA", 4: "ESTATE",
                5: "EUNSUPPORTED", 6: "EPEER"}

# Every entry point include/janus_b200.h declares (checked by tests/test_abi.py).
SYMBOLS = (
    "janus_create", "janus_destroy", "janus_last_error", "janus_launch_count",
    "janus_set_replica_map", "janus_replica_order", "janus_schedule_async", "janus_schedule",
    "janus_time_schedule", "janus_moe_configure", "janus_moe_set_weights",
    "janus_moe_layer_async", "janus_moe_layer", "janus_shard_tokens",
    "janus_moe_layer_latency", "janus_derive_seed", "janus_profile",
    "janus_profile_read", "janus_trace_schedule", "janus_xfer_configure", "janus_xfer_handle",
    "janus_xfer_connect", "janus_attn_dispatch_async", "janus_moe_layer_xfer_async",
    "janus_attn_combine_async", "janus_xfer_status", "janus_xfer_mc_supported",
    "janus_xfer_mc_create", "janus_xfer_mc_join", "janus_xfer_mc_bind", "janus_gate_async",
    "janus_moe_set_router", "janus_moe_layer_gated_async", "janus_stats_configure",
    "janus_stats_record_async", "janus_stats_read", "janus_stats_status",
    "janus_moe_layer_host_async", "janus_moe_host_sync", "janus_moe_set_shared",
    "janus_moe_set_shared_split",
    "janus_xfer_configure_colocated", "janus_xfer_check", "janus_xfer_set_timeout",
    "janus_xfer_connect_local", "janus_xfer_set_transport", "janus_attn_route_async",
    "janus_xfer_recv_rows", "janus_xfer_set_combine", "janus_latency_instance",
    "janus_latency_layer", "janus_latency_fit", "janus_debug_ffn_trace",
)


class LatencyModel(C.Structure):
    """janus_latency_model (janus_b200.h)."""
    _fields_ = [("t_launch", C.c_double), ("hbm_bandwidth", C.c_double),
                ("peak_flops", C.c_double), ("p", C.c_double), ("matrices", C.c_int),
                ("bytes_per_param", C.c_int), ("flop_matrices", C.c_int)]


class JanusAssignment(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "instance", "replica", "expert_instance", "load", "routed_tokens", "expert_tokens",
        "slot_row", "row_slot", "group_off", "status")]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
    P = C.POINTER
    L.janus_create.argtypes = [P(vp), i32]
    L.janus_destroy.argtypes = [vp]
    L.janus_destroy.restype = None
    L.janus_last_error.argtypes = [vp]
    L.janus_last_error.restype = C.c_char_p
    L.janus_launch_count.argtypes = [vp]
    L.janus_launch_count.restype = u64
    L.janus_set_replica_map.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    L.janus_replica_order.argtypes = [vp, vp, vp]
    L.janus_schedule_async.argtypes = [vp, vp, i32, i32, i32, u64, P(JanusAssignment), vp]
    L.janus_schedule.argtypes = [vp, vp, i32, i32, i32, u64, vp, vp, vp, vp, vp, vp]
    L.janus_time_schedule.argtypes = [vp, vp, i32, i32, i32, i32, P(dbl)]
    L.janus_moe_configure.argtypes = [vp, i32, i32, i32, i32]
    L.janus_moe_set_weights.argtypes = [vp, i32, vp, vp]
    L.janus_moe_layer_async.argtypes = [vp, vp, vp, vp, i32, vp, P(JanusAssignment), vp]
    L.janus_moe_layer.argtypes = [vp, vp, vp, vp, i32, vp]
    L.janus_shard_tokens.argtypes = [i64, i32, i32, P(i64), P(i64)]
    L.janus_shard_tokens.restype = None
    L.janus_moe_layer_latency.argtypes = [i32, vp, vp, i32, i32, i32, dbl, dbl, dbl]
    L.janus_moe_layer_latency.restype = dbl
    L.janus_derive_seed.argtypes = [u64, C.c_char_p, u64]
    L.janus_derive_seed.restype = u64
    L.janus_profile.argtypes = [vp, i32]
    L.janus_profile_read.argtypes = [vp, P(dbl), P(dbl), P(i32)]
    L.janus_trace_schedule.argtypes = [vp, vp, i32, i32, P(i64)]
    L.janus_debug_ffn_trace.argtypes = [vp, i32]
    L.janus_debug_ffn_trace.restype = i32
    L.janus_xfer_configure.argtypes = [vp, i32, i32, i32, i32, i32, i32]
    L.janus_xfer_handle.argtypes = [vp, C.c_char_p]
    L.janus_xfer_connect.argtypes = [vp, C.c_char_p]
    L.janus_attn_dispatch_async.argtypes = [vp, vp, vp, vp, i64, u64, vp]
    L.janus_moe_layer_xfer_async.argtypes = [vp, i64, u64, vp]
    L.janus_attn_combine_async.argtypes = [vp, vp, i64, u64, vp]
    L.janus_xfer_status.argtypes = [vp, P(i32)]
    L.janus_xfer_mc_supported.argtypes = [vp, P(i32)]
    L.janus_xfer_mc_create.argtypes = [vp, P(i32)]
    L.janus_xfer_mc_join.argtypes = [vp, i32]
    L.janus_xfer_mc_bind.argtypes = [vp]
    L.janus_gate_async.argtypes = [vp, vp, vp, i64, i32, i32, i32, vp, vp, vp]
    L.janus_moe_set_router.argtypes = [vp, vp]
    L.janus_moe_layer_gated_async.argtypes = [vp, vp, i32, vp, vp]
    L.janus_stats_configure.argtypes = [vp, i32, i32]
    L.janus_stats_record_async.argtypes = [vp, vp, i64, i32, vp]
    L.janus_stats_read.argtypes = [vp, P(i64), P(i64), P(i32)]
    L.janus_stats_status.argtypes = [vp, P(i32)]
    L.janus_moe_layer_host_async.argtypes = [vp, vp, vp, vp, i32, vp]
    L.janus_moe_host_sync.argtypes = [vp]
    L.janus_moe_set_shared.argtypes = [vp, vp, vp]
    L.janus_moe_set_shared_split.argtypes = [vp, i32]
    L.janus_xfer_configure_colocated.argtypes = [vp, i32, i32, i32, i32, i32]
    L.janus_xfer_check.argtypes = [vp]
    L.janus_xfer_set_timeout.argtypes = [vp, u64]
    L.janus_xfer_connect_local.argtypes = [vp, vp]
    L.janus_xfer_set_transport.argtypes = [vp, i32]
    L.janus_attn_route_async.argtypes = [vp, vp, vp, i64, u64, vp]
    L.janus_xfer_recv_rows.argtypes = [vp, u64, P(vp)]
    L.janus_xfer_set_combine.argtypes = [vp, i32]
    L.janus_latency_instance.argtypes = [P(LatencyModel), i32, i64, i32, i32]
    L.janus_latency_instance.restype = dbl
    L.janus_latency_layer.argtypes = [P(LatencyModel), i32, vp, vp, i32, i32]
    L.janus_latency_layer.restype = dbl
    L.janus_latency_fit.argtypes = [i32, vp, vp, vp, i32, i32, P(LatencyModel), P(dbl)]
    return L


lib = _load()
