"""conv1 per-launch live time (library events, one stream) and the two-stream step for each first_fp4
variant given on the command line (vehicle net, RGB, 16384-image chunks, 32768 images).
usage: python tools/time_conv1.py [first_fp4 values, default 0 1 2]"""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

B, CHUNK = 32768, 16384
variants = [int(v) for v in sys.argv[1:]] or [0, 1, 2]
x = synth.images(B, 96, 96, 3, 6).cuda()
lg = torch.empty((B, 4), dtype=torch.int32, device="cuda")
cls = torch.empty((B,), dtype=torch.int32, device="cuda")
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
ref = None
for v in variants:
    bnn.set_option("first_fp4", v)
    net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=CHUNK)
    bnn.set_option("streams", 1)
    for _ in range(3):
        net.forward(x, lg, cls)
    torch.cuda.synchronize()
    if ref is None:
        ref = lg.clone()
    assert torch.equal(ref, lg), "variant %d differs" % v
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
    print("first_fp4=%d %s | conv1 %.4f ms/launch | step %.3f ms %.2f M img/s" % (
        v, net.layer_kernel(0, CHUNK), ms[1] / cnt[1], st, B / st / 1e3), flush=True)
    net.close()
bnn.set_option("first_fp4", 1)
