"""Role timeline of conv_tc4_pool_kernel (vehicle conv2; bnn_set_trace, diagnostics build): CTA (0,0), SM clock
per tile.  usage: BNN_TRACE_LIB=1 python tools/trace_conv2.py [conv_pair = 0 | 1]
(after `python -m paper_1808_00209_b200._build --trace`).  Events per tile it: 0 MMA thread before the A wait,
1 after it, 2 after the accumulator wait, 3 after the commit; 4 loader warp 0 after its A-buffer wait, 5 at its
A-ready arrive; 6 epilogue (quarter 0) at accumulator ready, 7 at release."""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

v = int(sys.argv[1]) if len(sys.argv) > 1 else 0
B = 8192
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
bnn.set_option("conv_pair", v)
bnn.set_option("trace_layer", 1)
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=B)
x = synth.images(B, 96, 96, 3, 6).cuda()
bnn.set_option("streams", 1)
net.forward(x)
torch.cuda.synchronize()
tr = torch.zeros(16 * 2000, dtype=torch.int64, device="cuda")
bnn.set_trace(tr)
net.forward(x)
torch.cuda.synchronize()
bnn.set_trace(None)
t = tr.view(-1, 16).cpu().to(torch.float64)
n = int((t[:, 7] > 0).sum())
t = t[:n]
t0 = float(t[0, 0])
print("conv_pair=%d tiles traced %d (clk relative to the MMA thread's first event)" % (v, n))
print("  it  mma:wait_a  got_a  got_acc  commit | ld:go  ld:rdy | epi:rdy  release")
for i in list(range(min(n, 8))) + list(range(max(8, n - 4), n)):
    r = [int(x - t0) for x in t[i]]
    print("%4d %10d %6d %8d %7d | %6d %7d | %7d %8d" % (i, *r[0:8]))
s = slice(4, n)
d = lambda a, b: float((t[s, b] - t[s, a]).median())  # noqa: E731
print("median period (commit to commit) %.0f clk" % float((t[5:n, 3] - t[4:n - 1, 3]).median()))
print("median MMA: A wait %.0f, acc wait %.0f, issue+commit %.0f clk" % (d(0, 1), d(1, 2), d(2, 3)))
print("median loader: go -> ready %.0f clk" % d(4, 5))
print("median epilogue: ready -> release %.0f clk; commit -> epi ready %.0f clk; release -> MMA got_acc(next) %.0f" % (
    d(6, 7), d(3, 6), float((t[5:n, 2] - t[4:n - 1, 7]).median())))
