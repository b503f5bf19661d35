"""A small run of every library kernel for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per gpurun call):
  K1 scheduler — the decode-size single-CTA kernel and the cluster kernel
  (2..16 CTAs, DSMEM exchange), AEBS and random policy, an unknown expert;
  K3 permute, K4 grouped GEMMs (64- and 256-row tiles, shared expert),
  K5 combine; the gating kernel; the activation-statistics kernels; the box
  exchange on one GPU (dispatch, wait, push combine, signal, reduce — P2P and
  routed).  Small shapes: the sanitizers slow kernels down ~100x.

  python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from routing import RoutingPattern, gen_batch  # noqa: E402
import paper_2512_13525_b200 as J  # noqa: E402
from paper_2512_13525_b200.moe import (ActivationStats, MoELayer, build_weight_store,  # noqa: E402
                                       expert_weights, make_inputs, router_weights)


def main():
    torch.cuda.set_device(0)
    # K1: small kernel (S <= 2048), cluster kernel (S > 2048), random policy, error path
    rm = J.config_map("c5")
    sch = J.Scheduler(rm)
    for T in (32, 256, 600, 2100):
        b = gen_batch(RoutingPattern.zipf(256, 1.2), T, 8, 0x5A, T)
        sch.schedule(b)
        sch.schedule_random(b, 7)
    bad = gen_batch(RoutingPattern.zipf(256, 1.2), 64, 8, 1, 1)
    bad.experts[17] = 999
    try:
        sch.schedule(bad)
    except J.ValidationError:
        pass
    # K3/K4/K5 (decode 64-row tiles and 256-row tiles), shared expert, unknown expert
    hosts = [[0, 1], [1, 2], [0, 2], [0], [1], [2], [0, 1, 2], [2]] * 2
    rm3 = J.ReplicaMap.from_hosts(3, 12, hosts)
    layer = MoELayer(rm3, 256, 128, 1200, 4)
    layer.set_weights(*build_weight_store(layer, 1))
    wg, wu, wd = expert_weights(99, 256, 128, 5, "cuda")
    for T, shared in ((40, False), (1200, False), (300, True)):
        if shared:
            layer.set_shared(torch.cat([wg, wu]).contiguous(), wd.contiguous())
        b = gen_batch(RoutingPattern.gaussian(16, 0.2), T, 4, 3, T)
        x, gw = make_inputs(T, 4, 256, 3, "cuda")
        layer.forward(x, torch.from_numpy(b.experts).cuda(), gw)
    ex = torch.from_numpy(gen_batch(RoutingPattern.uniform(16), 40, 4, 2, 2).experts).cuda()
    ex[5] = 77
    x, gw = make_inputs(40, 4, 256, 3, "cuda")
    layer.forward(x, ex, gw)
    torch.cuda.synchronize()
    # gating kernel + gated layer
    wr = router_weights(16, 256, 13, "cuda")
    layer.set_router(wr)
    layer.forward_gated(make_inputs(200, 4, 256, 4, "cuda")[0])
    # activation statistics
    st = ActivationStats(16, 4)
    for i in range(6):
        st.record_batch(torch.from_numpy(gen_batch(RoutingPattern.uniform(16), 64, 4, 9, i).experts)
                        .cuda(), 4)
    st.read()
    # the box exchange on one GPU, causal order on one stream
    from paper_2512_13525_b200.dist import BoxPlan, JanusBox
    for transport in ("p2p", "routed"):
        plan = BoxPlan(1, 2)
        rmb = J.ReplicaMap.from_hosts(2, 16, [sorted({e % 2, (e + 1) % 2}) for e in range(16)])
        layers = {}
        for r in (1, 2):
            lay = MoELayer(rmb, 256, 128, 200, 4, instance=r - 1)
            lay.set_weights(*build_weight_store(lay, 1))
            layers[r] = lay
        boxes = JanusBox.local(plan, 200, 256, 4, layers, transport=transport, rmap=rmb)
        s = torch.cuda.current_stream().cuda_stream
        for e in (1, 2):
            T = 200 - 37 * e
            b = gen_batch(RoutingPattern.gaussian(16, 0.2), T, 4, 7, e)
            x, gw = make_inputs(T, 4, 256, e, "cuda")
            exs = torch.from_numpy(b.experts).cuda()
            boxes[0].dispatch(x, exs, gw, T, e, s)
            boxes[1].moe_step(T, e, s)
            boxes[2].moe_step(T, e, s)
            out = torch.empty(T, 256, dtype=torch.bfloat16, device="cuda")
            boxes[0].combine(out, T, e, s)
        torch.cuda.synchronize()
        for bx in boxes:
            bx.check()
        del boxes
    torch.cuda.synchronize()
    print("sanitize probe done", flush=True)


if __name__ == "__main__":
    main()
