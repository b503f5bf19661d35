"""Synthetic routing for tests, tools and the bench's input generation — TEST
INFRASTRUCTURE, backed by the oracle's gen_batch restatement (oracle.c
or_gen_batch, pinned bit-exact to the reference's gen_batch,
workload.cpp:56-130, by tests/test_oracle_vs_ref.py).  The product does not
generate routing ("do not port; call the oracle").

Same names and meaning as the reference (workload.hpp:14-32): RoutingPattern
uniform / gaussian / from_pmf (+ zipf = from_pmf(1/(e+1)^s)), and gen_batch
returning the package's ActivationBatch.
"""
from __future__ import annotations

import numpy as np

from oracle import Oracle

_ORC = None


def _orc() -> Oracle:
    global _ORC
    if _ORC is None:
        _ORC = Oracle()
    return _ORC


class RoutingPattern:
    def __init__(self, pmf: np.ndarray, cdf: np.ndarray):
        self.pmf, self.cdf = pmf, cdf

    @staticmethod
    def uniform(num_experts: int) -> "RoutingPattern":
        return RoutingPattern(*_orc().pattern("uniform", num_experts))

    @staticmethod
    def gaussian(num_experts: int, sigma: float) -> "RoutingPattern":
        return RoutingPattern(*_orc().pattern("gaussian", num_experts, sigma=sigma))

    @staticmethod
    def from_pmf(weights) -> "RoutingPattern":
        w = np.ascontiguousarray(weights, np.float64)
        return RoutingPattern(*_orc().pattern("pmf", len(w), weights=w))

    @staticmethod
    def zipf(num_experts: int, s: float) -> "RoutingPattern":
        return RoutingPattern.from_pmf([1.0 / (e + 1) ** s for e in range(num_experts)])

    def num_experts(self) -> int:
        return len(self.pmf)


def gen_batch(pattern: RoutingPattern, num_tokens: int, top_k: int, seed: int, step: int):
    """workload.hpp:29-32 -> the package's ActivationBatch."""
    import paper_2512_13525_b200 as J
    ex = _orc().gen_batch(pattern.cdf, num_tokens, top_k, seed, step)
    return J.ActivationBatch(num_tokens, top_k, ex)
