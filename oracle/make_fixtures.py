"""Generate committed fixtures from the reference itself (run where /root/reference exists).

TEST INFRASTRUCTURE / DATA GENERATION.  Writes

* ``paper_2512_13525_b200/maps/*.map`` — replica maps for BASELINE.json's
  configs, produced by the reference placement pipeline (the
  ``DecodeEngine::rebuild_placement`` recipe, src/sim.cpp:107-122,134-148:
  32 x 256-token warmup -> allocate_replicas -> cap_allocation ->
  place_replicas -> to_replica_map).  Placement is the reference's cold path
  (hours scale, SURVEY.md §2 "OUT OF SCOPE"); its output is an INPUT to the hot
  path, like a checkpoint, and is stored with explicit replica ids.
* ``tests/golden/*.json`` — golden vectors: the shipped sample fixture
  (configs/sample-batch.txt x configs/sample-replicas.txt) with the
  reference's assignment, and reference assignments for config c1..c5 batches.

Usage:  python oracle/make_fixtures.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from oracle import CSRMap, Ref  # noqa: E402

REF_CFG = "/root/reference/proj/configs"
MAPS = os.path.join(ROOT, "paper_2512_13525_b200", "maps")
GOLD = os.path.join(ROOT, "tests", "golden")

# BASELINE.json configs.  kind, E, k, N, C, seed, zipf s.
CONFIGS = {
    "c1_uniform": dict(kind="uniform", E=64, k=8, N=4, C=20, seed=0x5EED),
    "c1_gaussian": dict(kind="gaussian", E=64, k=8, N=4, C=20, seed=0x5EED, sigma=0.15),
    "c2": dict(kind="zipf", E=128, k=8, N=1, C=128, seed=0x30, s=1.0),
    "c3": dict(kind="zipf", E=128, k=8, N=6, C=27, seed=0x235, s=1.0),
    "c4_n2": dict(kind="zipf", E=256, k=8, N=2, C=160, seed=0xD5, s=1.0),
    "c4_n4": dict(kind="zipf", E=256, k=8, N=4, C=80, seed=0xD5, s=1.0),
    "c4_n8": dict(kind="zipf", E=256, k=8, N=8, C=40, seed=0xD5, s=1.0),
    "c5": dict(kind="zipf", E=256, k=8, N=6, C=54, seed=0x5A, s=1.2),
    # MoE sub-groups of M GPUs for the box benches (same routing as c2 / c3,
    # C = ceil(1.25 * E / M) as in c3's 6 x 27)
    "c2_m2": dict(kind="zipf", E=128, k=8, N=2, C=80, seed=0x30, s=1.0),
    "c2_m3": dict(kind="zipf", E=128, k=8, N=3, C=54, seed=0x30, s=1.0),
    "c2_m4": dict(kind="zipf", E=128, k=8, N=4, C=40, seed=0x30, s=1.0),
    "c2_m6": dict(kind="zipf", E=128, k=8, N=6, C=27, seed=0x30, s=1.0),
    "c2_m8": dict(kind="zipf", E=128, k=8, N=8, C=20, seed=0x30, s=1.0),
    "c3_m1": dict(kind="zipf", E=128, k=8, N=1, C=128, seed=0x235, s=1.0),
    "c3_m2": dict(kind="zipf", E=128, k=8, N=2, C=80, seed=0x235, s=1.0),
    "c3_m3": dict(kind="zipf", E=128, k=8, N=3, C=54, seed=0x235, s=1.0),
    "c3_m4": dict(kind="zipf", E=128, k=8, N=4, C=40, seed=0x235, s=1.0),
    "c3_m6": dict(kind="zipf", E=128, k=8, N=6, C=27, seed=0x235, s=1.0),  # = c3 (2A+6E)
    "c3_m8": dict(kind="zipf", E=128, k=8, N=8, C=20, seed=0x235, s=1.0),
}


def zipf_weights(E, s):
    return np.array([1.0 / (e + 1) ** s for e in range(E)], np.float64)


def pattern_args(cfg):
    if cfg["kind"] == "zipf":
        return "pmf", dict(weights=zipf_weights(cfg["E"], cfg["s"]))
    if cfg["kind"] == "gaussian":
        return "gaussian", dict(sigma=cfg["sigma"])
    return "uniform", {}


def dump_map(m: CSRMap, path: str, note: str):
    with open(path, "w") as f:
        f.write(f"# replica map: experts={m.E}  ({note})\n")
        f.write("# format: 'expert: instance:replica_id ...' (explicit physical replica ids)\n")
        f.write(f"instances = {m.N}\nslots_per_instance = {m.C}\n")
        for e in range(m.E):
            pairs = " ".join(f"{g}:{r}" for g, r in zip(m.hosts_of(e), m.rids_of(e)))
            f.write(f"{e}: {pairs}\n")


def csr_json(m: CSRMap):
    return dict(E=m.E, N=m.N, C=m.C, off=m.off.tolist(), hosts=m.hosts.tolist(),
                rid=m.rid.tolist())


def sched_json(a):
    return dict(instance=a.instance.tolist(), replica=a.replica.tolist(),
                expert_instance=a.expert_instance.tolist(), load=a.load.tolist(),
                routed_tokens=a.routed_tokens.tolist())


def main():
    ref = Ref()
    os.makedirs(MAPS, exist_ok=True)
    os.makedirs(GOLD, exist_ok=True)

    # 1. the shipped sample fixture, parsed by the reference's own loaders
    with open(os.path.join(REF_CFG, "sample-batch.txt")) as f:
        ex, T, k = ref.load_batch_text(f.read())
    with open(os.path.join(REF_CFG, "sample-replicas.txt")) as f:
        m = ref.load_replica_map_text(f.read())
    a = ref.schedule(ex, T, k, m, "schedule")
    rnd = ref.schedule(ex, T, k, m, "random", seed=7)
    gold = dict(source="reference configs/sample-batch.txt x sample-replicas.txt, "
                       "assignment by reference schedule() (oracle/_ref)",
                T=T, k=k, experts=ex.tolist(), map=csr_json(m), schedule=sched_json(a),
                schedule_random_seed7=sched_json(rnd),
                dump_assignment=ref.dump_assignment(ex, T, k, a))
    with open(os.path.join(GOLD, "sample_fixture.json"), "w") as f:
        json.dump(gold, f)

    # 2. config maps + golden batches/assignments
    cases = []
    for name, cfg in CONFIGS.items():
        kind, kw = pattern_args(cfg)
        mp = ref.placement(kind, cfg["E"], cfg["k"], cfg["N"], cfg["C"], cfg["seed"], **kw)
        dump_map(mp, os.path.join(MAPS, f"{name}.map"),
                 f"reference placement pipeline, {kind}, seed {cfg['seed']:#x}")
        for T in (32, 256) if name != "c1_uniform" else (256,):
            step = 1256 if name.startswith("c1") else T
            ex = ref.gen_batch(kind, cfg["E"], T, cfg["k"], cfg["seed"], step, **kw)
            a = ref.schedule(ex, T, cfg["k"], mp, "schedule")
            r = ref.schedule(ex, T, cfg["k"], mp, "random", seed=7)
            cases.append(dict(name=name, T=T, k=cfg["k"], seed=cfg["seed"], step=step,
                              experts=ex.tolist(), schedule=sched_json(a),
                              schedule_random_seed7=sched_json(r)))
    with open(os.path.join(GOLD, "config_cases.json"), "w") as f:
        json.dump(dict(source="reference gen_batch + schedule()/schedule_random(7) via oracle/_ref;"
                              " maps in paper_2512_13525_b200/maps", cases=cases), f)
    print("wrote", MAPS, GOLD)


if __name__ == "__main__":
    main()
