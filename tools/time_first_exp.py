"""Decompose the TMA first layer's time: conv1 per-launch time (library events, one stream) with
timing-experiment bits (bnn_set_option "first_exp"; results are wrong unless 0):
  1 = epilogue reads 2 of the 4 pool-offset accumulator blocks, 2 = epilogue reads none,
  4 = builders skip the strips, 8 = one MMA per tile instead of K + 1."""
import sys
import torch
import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth
B = 32768
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8192)
x = synth.images(B, 96, 96, 3, 6).cuda()
lg = torch.empty((B, 4), dtype=torch.int32, device="cuda"); cls = torch.empty((B,), dtype=torch.int32, device="cuda")
bnn.set_option("streams", 1)
exps = sys.argv[1:] or ["0", "1", "2", "4", "8", "6", "10", "12", "0"]
for a in exps:  # "d<bits>": the same with double-buffered TMEM accumulators (first_db = 1)
    db = a.startswith("d")
    fp4 = a.startswith("f")
    e = int(a.lstrip("df"))
    bnn.set_option("first_db", 1 if db else 0)
    bnn.set_option("first_fp4", 1 if fp4 else 0)
    bnn.set_option("first_exp", e)
    for _ in range(3):
        net.forward(x, lg, cls)
    torch.cuda.synchronize()
    net.profile(True)
    for _ in range(10):
        net.forward(x, lg, cls)
    ms, cnt = net.profile_read()
    net.profile(False)
    print("fp4=%d db=%d first_exp=%2d  conv1 %.4f ms/launch  (launches %d)" % (fp4, db, e, ms[1] / cnt[1], cnt[1]), flush=True)
bnn.set_option("first_exp", 0)
bnn.set_option("first_fp4", 0)
bnn.set_option("first_db", 1)
