"""Batch-1 latency (config 1 protocol: one CUDA-graph replay per image) for option settings given as
key=value pairs: python tools/time_latency.py [fused_max_n=8] ..."""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

opts = dict(kv.split("=") for kv in sys.argv[1:])
for k, v in opts.items():
    bnn.set_option(k, int(v))
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=64)
st_in, st_lg, st_cls = net.staging(1)
imgs = synth.images(300, 96, 96, 3, 6).cuda()
for i in range(20):
    st_in.copy_(imgs[i:i + 1])
    net.forward_staged(1)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(300)]
for i in range(300):
    st_in.copy_(imgs[i:i + 1])
    ev[i][0].record()
    net.forward_staged(1)
    ev[i][1].record()
torch.cuda.synchronize()
per = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(500):
    net.forward_staged(1)
e1.record()
torch.cuda.synchronize()
print(opts, "median %.1f us, mean %.1f us, back-to-back %.1f us; layer0 %s" % (
    per[len(per) // 2], sum(per) / len(per), e0.elapsed_time(e1) * 1e3 / 500, net.layer_kernel(0, 1)), flush=True)
