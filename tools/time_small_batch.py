"""Device time per forward of small batches (B images per forward; R forwards captured in ONE CUDA graph so the
host launch cost is amortised): the whole-network cluster kernel with one cluster per image (fused_multi = 1),
with one cluster for the batch (fused_multi = 0), and the layer-by-layer PDL path (fused_max_n = 0; with gemv_max_n 16 and 255).
usage: python tools/time_small_batch.py [R] [B,B,...]  The three
must agree on every class."""
import json
import os
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

R = int(sys.argv[1]) if len(sys.argv) > 1 else 50
layers = synth.make_weights(synth.VEHICLE, 1, 5)
bnn.set_option("fused_cs", int(os.environ.get("BNN_FUSED_CS", "0")))  # 8: force 8-CTA clusters
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
out = []
for B in [int(b) for b in (sys.argv[2].split(",") if len(sys.argv) > 2 else "1,2,4,8,9,16,32".split(","))]:
    imgs = synth.images(R * B, 96, 96, 3, 60 + B).cuda()
    row = {"batch": B}
    classes = []
    for name, fmax, multi, gemv in (("cluster_per_image", 64, 1, 255), ("one_cluster", 64, 0, 255), ("layers_pdl_gemv16", 0, 1, 16),
                                    ("layers_pdl", 0, 1, 255)):
        if B > 64 and fmax:
            continue
        bnn.set_option("fused_max_n", fmax)
        bnn.set_option("fused_multi", multi)
        bnn.set_option("gemv_max_n", gemv)
        net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=max(64, B))
        lg = torch.empty((R * B, 4), dtype=torch.int32, device="cuda")
        cb = (B + 3) // 4 * 4  # 16-byte aligned class slices
        cls = torch.empty((R * cb,), dtype=torch.int32, device="cuda")
        s = torch.cuda.Stream()
        fwd = lambda i: net.forward(imgs[i * B:(i + 1) * B], lg[i * B:(i + 1) * B], cls[i * cb:i * cb + B])
        with torch.cuda.stream(s):
            for i in range(3):
                fwd(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                fwd(i)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        row[name + "_us"] = round(e0.elapsed_time(e1) * 1e3 / (10 * R), 2)
        row[name + "_launches"] = bnn.forward_launches(net, B)
        classes.append(torch.cat([cls[i * cb:i * cb + B] for i in range(R)]).clone())
        net.close()
    row["classes_identical"] = all(torch.equal(classes[0], c) for c in classes[1:])
    print(json.dumps(row), flush=True)
    out.append(row)
bnn.set_option("fused_max_n", 12)
bnn.set_option("fused_multi", 1)
bnn.set_option("gemv_max_n", 255)
bnn.set_option("fused_cs", 0)
