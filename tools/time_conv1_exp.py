"""conv1_fp4 role experiments (diagnostics build only; WRONG results by design):
BNN_TRACE_LIB=1 python tools/time_conv1_exp.py [conv_pair] [exp ...] -> conv1 ms/launch per exp bit set: 1 epilogue
skips the drain, 2 builders skip the strips, 4 no data MMAs, 8 no offset MMA, 16 MMA thread skips the
accumulator wait, 32 ... the A-ready wait (default: 0 1 2 3 4 8 16 32 48 0)."""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

B, CHUNK = 32768, 16384
x = synth.images(B, 96, 96, 3, 6).cuda()
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
pair = int(sys.argv[1]) if len(sys.argv) > 1 else 1
exps = [int(e) for e in sys.argv[2:]] or [0, 1, 2, 3, 4, 8, 16, 32, 48, 0]
bnn.set_option("conv_pair", pair)
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=CHUNK)
bnn.set_option("streams", 1)
for e in exps:
    bnn.set_option("first_exp", e)
    for _ in range(2):
        net.forward(x)
    torch.cuda.synchronize()
    net.profile(True)
    for _ in range(6):
        net.forward(x)
    ms, cnt = net.profile_read()
    net.profile(False)
    print("pair=%d exp=%d conv1 %.4f ms/launch" % (pair, e, ms[1] / cnt[1]), flush=True)
bnn.set_option("first_exp", 0)
