"""Test helper: read the committed config replica maps and name their routing patterns."""
import os

import numpy as np

from oracle import CSRMap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAPS = os.path.join(ROOT, "paper_2512_13525_b200", "maps")


def zipf(E, s):
    return np.array([1.0 / (e + 1) ** s for e in range(E)], np.float64)


# name -> (pattern kind, kwargs, routing seed)
CONFIG_PATTERNS = {
    "c1_uniform": ("uniform", {}, 0x5EED),
    "c1_gaussian": ("gaussian", {"sigma": 0.15}, 0x5EED),
    "c2": ("pmf", {"weights": zipf(128, 1.0)}, 0x30),
    "c3": ("pmf", {"weights": zipf(128, 1.0)}, 0x235),
    "c4_n2": ("pmf", {"weights": zipf(256, 1.0)}, 0xD5),
    "c4_n4": ("pmf", {"weights": zipf(256, 1.0)}, 0xD5),
    "c4_n8": ("pmf", {"weights": zipf(256, 1.0)}, 0xD5),
    "c5": ("pmf", {"weights": zipf(256, 1.2)}, 0x5A),
}


def load_map_csr(name: str) -> CSRMap:
    N = C = None
    hosts, rids = [], []
    with open(os.path.join(MAPS, f"{name}.map")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            if "=" in line:
                k, v = (x.strip() for x in line.split("="))
                if k == "instances":
                    N = int(v)
                else:
                    C = int(v)
                continue
            e, rest = line.split(":", 1)
            assert int(e) == len(hosts)
            pairs = [p.split(":") for p in rest.split()]
            hosts.append([int(g) for g, _ in pairs])
            rids.append([int(r) for _, r in pairs])
    return CSRMap.from_lists(N, C, hosts, rids)
