"""One vehicle-net forward (RGB, one 16384-image chunk) under the given options, for ncu captures.
usage: python tools/one_forward.py [mode=M] KEY=V ..."""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

opts = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[1:])
mode = opts.pop("mode", 1)  # input binarization (1 RGB, 2 GRAY, 3 LBP, 0 SIGN, -1 NONE)
for k, v in opts.items():
    bnn.set_option(k, v)
B = 16384
x = synth.images(B, 96, 96, 3, 6).cuda()
layers = synth.make_weights(synth.VEHICLE, mode, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
T = {1: synth.thresholds(3, 5).cuda(), 2: torch.tensor([-127.0]).cuda()}.get(mode)
net = bnn.Net(96, 96, 3, bnn.U8, mode, T, dl, max_batch=B)
lg, cls = net.forward(x)
torch.cuda.synchronize()
print("one forward ok", opts)
