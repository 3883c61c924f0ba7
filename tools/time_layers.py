"""Per-layer live times of the vehicle forward (library events, one stream) and the two-stream step,
batch 32768.  usage: python tools/time_layers.py [chunk]"""
import torch
import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth
import sys
B = 32768
CHUNK = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=CHUNK)
x = synth.images(B, 96, 96, 3, 6).cuda()
lg = torch.empty((B, 4), dtype=torch.int32, device="cuda"); cls = torch.empty((B,), dtype=torch.int32, device="cuda")
for rep in range(2):
    bnn.set_option("streams", 1)
    for _ in range(3):
        net.forward(x, lg, cls)
    torch.cuda.synchronize()
    net.profile(True)
    for _ in range(10):
        net.forward(x, lg, cls)
    ms, cnt = net.profile_read()
    net.profile(False)
    print("per launch ms:", " ".join("%s=%.4f" % (n, m / max(c, 1)) for n, m, c in zip(["pack", "conv1", "conv2", "fc1", "fc2", "fc3", "argmax"], ms, cnt)))
    bnn.set_option("streams", 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        net.forward(x, lg, cls)
    e1.record()
    torch.cuda.synchronize()
    print("step %.3f ms  %.2f M img/s" % (e0.elapsed_time(e1) / 20, B / (e0.elapsed_time(e1) / 20) / 1e3))
