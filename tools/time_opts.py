"""A/B of library options on the vehicle net (RGB, 16384-image chunks, 32768 images): per-layer live times
(library events, one stream) and the two-stream step for each option setting, outputs checked identical.
usage: python tools/time_opts.py KEY=V[,KEY=V...] [KEY=V...]   e.g.  conv_pair=0 conv_pair=1"""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

B, CHUNK = 32768, 16384
settings = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in a.split(",")) for a in sys.argv[1:]] or [{}]
x = synth.images(B, 96, 96, 3, 6).cuda()
lg = torch.empty((B, 4), dtype=torch.int32, device="cuda")
cls = torch.empty((B,), dtype=torch.int32, device="cuda")
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
ref = None
names = ["pack", "conv1", "conv2", "fc1", "fc2", "fc3", "argmax"]
for rep in range(2):
    for opts in settings:
        for k, v in opts.items():
            bnn.set_option(k, v)
        net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=CHUNK)
        bnn.set_option("streams", 1)
        for _ in range(3):
            net.forward(x, lg, cls)
        torch.cuda.synchronize()
        if ref is None:
            ref = lg.clone()
        same = torch.equal(ref, lg)
        net.profile(True)
        for _ in range(10):
            net.forward(x, lg, cls)
        ms, cnt = net.profile_read()
        net.profile(False)
        bnn.set_option("streams", 2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            net.forward(x, lg, cls)
        e0.record()
        for _ in range(20):
            net.forward(x, lg, cls)
        e1.record()
        torch.cuda.synchronize()
        st = e0.elapsed_time(e1) / 20
        print("%-28s" % ",".join("%s=%d" % kv for kv in opts.items()),
              " ".join("%s=%.4f" % (nm, m / c) for nm, m, c in zip(names, ms, cnt) if c),
              "| step %.3f ms %.2f M img/s" % (st, B / st / 1e3), "same" if same else "DIFFERENT", flush=True)
        net.close()
