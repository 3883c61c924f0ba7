"""Device-side batch-1 latency: R single-image forwards captured back to back in ONE CUDA graph (torch.cuda.graph),
so the host launch cost (~16 us per cudaGraphLaunch, which bounds the per-image replay loop of the config-1 protocol)
is paid once per R images.  Compares the layer-by-layer PDL path with the whole-network cluster kernel (f1).
usage: python tools/time_latency_dev.py [R]"""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
imgs = synth.images(R, 96, 96, 3, 6).cuda()
res = {}
for name, fused in (("graph (5 kernels, PDL)", 0), ("cluster kernel (f1)", 8)):
    bnn.set_option("fused_max_n", fused)
    net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8)
    lg = torch.empty((R, 4), dtype=torch.int32, device="cuda")
    cls = torch.empty((R * 4,), dtype=torch.int32, device="cuda")  # image i's class at 4 i (16-byte aligned pointers)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            net.forward(imgs[i:i + 1], lg[i:i + 1], cls[4 * i:4 * i + 1])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(R):
            net.forward(imgs[i:i + 1], lg[i:i + 1], cls[4 * i:4 * i + 1])
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) * 1e3 / (reps * R)
    res[name + " classes"] = cls[::4].clone()
    net.close()
bnn.set_option("fused_max_n", 12)
same = torch.equal(res["graph (5 kernels, PDL) classes"], res["cluster kernel (f1) classes"])
for k, v in res.items():
    if not k.endswith("classes"):
        print("%-26s %.2f us per image on the device (%d single-image forwards per CUDA graph)" % (k, v, R))
print("identical classes:", same)
