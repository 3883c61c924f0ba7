"""CIFAR BinaryNet per-layer live times (library events, one stream) under a list of options.
usage: python tools/time_cifar.py key=value[,key=value] ..."""
import sys
import torch
import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth
B = 16384
layers = synth.make_weights(synth.CIFAR, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
for chunk in (4096, 8192, 16384):
    n2 = bnn.Net(32, 32, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=chunk)
    xx = synth.images(B, 32, 32, 3, 6).cuda()
    for _ in range(3):
        n2.forward(xx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        n2.forward(xx)
    e1.record()
    torch.cuda.synchronize()
    print("chunk %d: step %.3f ms  %.3f M img/s" % (chunk, e0.elapsed_time(e1) / 10, B / (e0.elapsed_time(e1) / 10) / 1e3))
    n2.close()
net = bnn.Net(32, 32, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8192)
bnn.set_option("streams", 1)  # per-layer events are only meaningful on one stream
x = synth.images(B, 32, 32, 3, 6).cuda()
ref = None
for arg in sys.argv[1:] or [""]:
    opts = dict(kv.split("=") for kv in arg.split(",") if kv)
    for k, v in opts.items():
        bnn.set_option(k, int(v))
    lg, cls = net.forward(x)
    torch.cuda.synchronize()
    if ref is None:
        ref = lg.clone()
    assert torch.equal(ref, lg), "results changed"
    net.profile(True)
    for _ in range(5):
        net.forward(x)
    ms, cnt = net.profile_read()
    net.profile(False)
    print("%-30s" % arg, " ".join("%.3f" % (m / 5) for m in ms[1:10]), " total %.3f ms" % (sum(ms) / 5), flush=True)
