"""The attention -> MoE box exchange on real GPUs (needs >= 2 visible GPUs; the
round-end single-GPU run skips it — it is exercised with `gpurun --gpus 2/4`)."""
import glob
import json
import os
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("transport,inflight", [("p2p", 1), ("p2p", 2), ("nvls", 1), ("nvls", 2),
                                               ("routed", 1), ("routed", 2), ("ce", 1), ("ce", 2)])
@pytest.mark.parametrize("attn,moe", [(1, 1), (1, 3), (2, 2)])
def test_box_exchange_matches_single_gpu_layer(attn, moe, transport, inflight):
    if gpus() < attn + moe:
        pytest.skip(f"needs {attn + moe} GPUs (one rank per GPU)")
    out = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={attn + moe}", "--master-addr", "127.0.0.1", "--master-port",
           str(29500 + 10 * attn + moe + {"p2p": 0, "nvls": 50, "routed": 300, "ce": 400}[transport] +
               100 * inflight),
           os.path.join(ROOT, "tests", "dist_worker.py"),
           "--attn", str(attn), "--moe", str(moe), "--out", out, "--transport", transport,
           "--inflight", str(inflight)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(out, "*.json")))]
    assert len(res) == attn + moe
    for r in res:
        assert not r["timed_out"], r
        assert r["check"] == "ok", r
        assert r["transport"] == transport
        if r["role"] in ("attention", "both"):
            for s in r["steps"]:
                assert s["bad"] == 0, s


@pytest.mark.parametrize("attn,moe", [(1, 3), (2, 2)])
def test_box_exchange_nvls_switch_combine(attn, moe):
    """NVLS dispatch with the in-switch combine (multimem.ld_reduce) instead of
    the default point-to-point push, two steps in flight."""
    if gpus() < attn + moe:
        pytest.skip(f"needs {attn + moe} GPUs (one rank per GPU)")
    out = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={attn + moe}", "--master-addr", "127.0.0.1", "--master-port",
           str(29950 + 10 * attn + moe), os.path.join(ROOT, "tests", "dist_worker.py"),
           "--attn", str(attn), "--moe", str(moe), "--out", out, "--transport", "nvls",
           "--combine", "switch", "--inflight", "2"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(out, "*.json")))]
    assert len(res) == attn + moe
    for r in res:
        assert not r["timed_out"], r
        assert r["check"] == "ok", r
        if r["role"] in ("attention", "both"):
            for s_ in r["steps"]:
                assert s_["bad"] == 0, s_


@pytest.mark.parametrize("flag", ["--shared", "--shared-split", "--gate"])
def test_box_exchange_shared_expert_and_moe_side_gating(flag):
    """--shared: the shared expert in a box (MoE instance 0 adds it to its
    partials); --shared-split: every MoE instance adds it for its share of the
    tokens.  --gate: rows only are dispatched and every MoE rank computes
    the routing with the gating kernel (Janus gates on the MoE side).  NVLS
    transport, two steps in flight."""
    attn, moe = 1, 3
    if gpus() < attn + moe:
        pytest.skip(f"needs {attn + moe} GPUs (one rank per GPU)")
    out = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={attn + moe}", "--master-addr", "127.0.0.1", "--master-port",
           str(29777 + ["--shared", "--shared-split", "--gate"].index(flag)), os.path.join(ROOT, "tests", "dist_worker.py"),
           "--attn", str(attn), "--moe",
           str(moe), "--out", out, "--transport", "nvls", "--inflight", "2", flag]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(out, "*.json")))]
    assert len(res) == attn + moe
    for r in res:
        assert not r["timed_out"], r
        if r["role"] in ("attention", "both"):
            for s_ in r["steps"]:
                assert s_["bad"] == 0, s_


@pytest.mark.parametrize("n,transport", [(2, "nvls"), (4, "nvls"), (4, "p2p"), (4, "routed"),
                                         (2, "ce"), (4, "ce")])
def test_moe_only_colocated_box(n, transport):
    """The MoE-only box (every rank owns a shard and is an MoE instance), two
    steps in flight."""
    if gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    out = tempfile.mkdtemp()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
           str(29800 + 10 * n + {"nvls": 0, "p2p": 1, "routed": 2, "ce": 3}[transport]),
           os.path.join(ROOT, "tests", "dist_worker.py"),
           "--attn", str(n), "--moe", str(n), "--out", out, "--transport", transport,
           "--inflight", "2", "--colocated"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(out, "*.json")))]
    assert len(res) == n
    for r in res:
        assert not r["timed_out"], r
        assert r["role"] == "both"
        for s_ in r["steps"]:
            assert s_["bad"] == 0, s_


@pytest.mark.parametrize("n,transport,colocated,inflight", [
    (2, "routed", True, 2), (4, "routed", True, 2), (4, "p2p", True, 2), (4, "ce", True, 2),
    (4, "nvls", True, 2), (4, "routed", False, 2), (4, "p2p", False, 2),
    (4, "routed", True, 3), (4, "p2p", False, 3)])
def test_box_split_streams(n, transport, colocated, inflight):
    """Dispatch, MoE step and combine each on a stream of their own (as
    bench.py runs the box), two or three steps in flight (dispatches one or
    two steps ahead), seven steps: the three epoch slots are kept safe by the
    library's events and flags, not stream order.  Every shard vs the fp32
    oracle."""
    if gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    out = tempfile.mkdtemp()
    roles = ["--attn", str(n), "--moe", str(n), "--colocated"] if colocated else \
        ["--attn", "1", "--moe", str(n - 1)]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port",
           str(29600 + 10 * n + {"routed": 0, "p2p": 1, "ce": 2, "nvls": 3}[transport] +
               (5 if colocated else 0) + 50 * (inflight - 2)),
           os.path.join(ROOT, "tests", "dist_worker.py"), *roles, "--out", out,
           "--transport", transport, "--inflight", str(inflight), "--steps", "7",
           "--split-streams"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(out, "*.json")))]
    assert len(res) == n
    for r in res:
        assert not r["timed_out"], r
        assert r["check"] == "ok", r
        if r["role"] in ("both", "attention"):
            assert len(r["steps"]) == 7
            for s_ in r["steps"]:
                assert s_["bad"] == 0, s_


@pytest.mark.parametrize("box,transport", [("moe-only", "routed"), ("moe-only", "ce"),
                                           ("2a6e", "routed"), ("2a6e", "p2p")])
def test_box_8_ranks_oversubscribed(box, transport):
    """The 8-rank boxes — MoE-only (the 8-GPU bench's default) and the
    north_star split 2A+6E (BASELINE c3) — as 8 processes on the GPUs there are
    (rank r on GPU r % n; CUDA IPC between processes, also on one device):
    every shard vs the fp32 oracle, two steps in flight.  Every phase ends
    with a device sync and a barrier of all ranks, so no wait kernel relies on
    a kernel of another process on its GPU running beside it."""
    n = max(1, min(gpus(), 8))
    out = tempfile.mkdtemp()
    roles = (["--attn", "8", "--moe", "8", "--colocated"] if box == "moe-only"
             else ["--attn", "2", "--moe", "6"])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port",
           str(29950 + {"routed": 0, "ce": 1, "p2p": 2}[transport] + (5 if box == "2a6e" else 0)),
           os.path.join(ROOT, "tests", "dist_worker.py"), *roles, "--out", out,
           "--transport", transport, "--inflight", "2", "--steps", "3", "--tokens", "160"]
    env = dict(os.environ, JANUS_TEST_GPUS=str(n))
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(out, "*.json")))]
    assert len(res) == 8
    for r in res:
        assert not r["timed_out"], r
        if box == "moe-only":
            assert r["role"] == "both"
        if r["role"] in ("both", "attention"):  # the shard owners check their outputs
            assert len(r["steps"]) == 3
            for s_ in r["steps"]:
                assert s_["bad"] == 0, s_
