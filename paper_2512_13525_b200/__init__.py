"""B200-native MoE-side hot path of Janus (arXiv 2512.13525).

A drop-in for the reference moesim library's scheduling / MoE-layer path:
``include/janus_b200.h`` is the C ABI, ``include/janus_moesim_compat.hpp`` the
C++ ``moesim::schedule`` shim, :mod:`.moesim` the Python mirror.  All compute
runs in ``libjanus_b200.so`` (sm_100a); there is no CPU fallback.
"""
from .moesim import (ActivationBatch, Assignment, InstanceLoad, ParseError,  # noqa: F401
                     ReplicaMap, Scheduler, ValidationError, config_map,
                     derive_seed, dump_assignment, load_batch, load_replica_map,
                     load_replica_map_file, max_activated_load, moe_layer_latency, schedule,
                     schedule_random, schedule_reference, shard_tokens,
                     reference_latency_model, fit_latency_model, layer_latency)

__all__ = [n for n in dir() if not n.startswith("_")]
