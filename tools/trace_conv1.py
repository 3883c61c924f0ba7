"""Role timeline of conv1_fp4_pool_kernel (bnn_set_trace; diagnostics build): CTA (0,0), SM clock per tile.
usage: BNN_TRACE_LIB=1 python tools/trace_conv1.py [first_fp4 = 1 (sleep waits) | 2 (spin waits)]
(after `python -m paper_1808_00209_b200._build --trace`).  Events per tile it: 0 MMA thread before the
ready wait (A built + accumulator set drained), 2 after it, 3 after the commit; 4 builder (group leader)
after its waits, 5 / 6 builder warps 1 / 5 of the group at A ready; 7 epilogue (quarter 0) at accumulator
ready, 8 at release."""
import sys

import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

v = int(sys.argv[1]) if len(sys.argv) > 1 else 1
B = 8192
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
bnn.set_option("first_fp4", v)
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
bnn.set_option("first_fp4", 1)
t = tr.view(-1, 16).cpu().to(torch.float64)
n = int((t[:, 3] > 0).sum())
t = t[:n]
t0 = float(t[0, 0])
print("first_fp4=%d tiles traced %d (clk relative to the MMA thread's first event)" % (v, n))
print("  it  mma:wait_a  got_a  got_acc  commit | bld:go  w1_rdy  w5_rdy | epi:rdy  release")
for i in list(range(min(n, 12))) + list(range(max(12, n - 6), n)):
    r = [int(x - t0) for x in t[i]]
    print("%4d %10d %6d %8d %7d | %7d %7d %7d | %7d %8d" % (i, *r[0:9]))
s = slice(8, n)
d = lambda a, b: float((t[s, b] - t[s, a]).median())  # noqa: E731
print("median period (commit to commit) %.0f clk" % float((t[9:n, 3] - t[8:n - 1, 3]).median()))
print("median MMA wait (A ready + accumulator free) %.0f, issue+commit %.0f clk" % (d(0, 2), d(2, 3)))
print("median builder: go -> warp1 ready %.0f, go -> warp5 ready %.0f clk" % (d(4, 5), d(4, 6)))
print("median epilogue: ready -> release %.0f clk; commit -> epi ready %.0f clk" % (d(7, 8), d(3, 7)))
