"""One vehicle-net forward (RGB, one 16384-image chunk) under the given options, for ncu captures.
usage: python tools/one_forward.py KEY=V ..."""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[1:])
for k, v in opts.items():
    bnn.set_option(k, v)
B = 16384
x = synth.images(B, 96, 96, 3, 6).cuda()
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=B)
lg, cls = net.forward(x)
torch.cuda.synchronize()
print("one forward ok", opts)
