"""Role timeline of the TMA first layer (bnn_set_trace): CTA (0,0), SM clocks per tile iteration.
usage: BNN_TRACE_LIB=1 python tools/trace_first.py [first_db] [first_exp]
(after `python -m paper_1808_00209_b200._build --trace`)"""
import sys
import torch
import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth
db = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ex = int(sys.argv[2]) if len(sys.argv) > 2 else 0
B = 8192
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8192)
x = synth.images(B, 96, 96, 3, 6).cuda()
bnn.set_option("streams", 1)
bnn.set_option("first_db", db)
bnn.set_option("first_exp", ex)
net.forward(x)
torch.cuda.synchronize()
tr = torch.zeros(16 * 400, dtype=torch.int64, device="cuda")
bnn.set_trace(tr)
net.forward(x)
torch.cuda.synchronize()
bnn.set_trace(None)
bnn.set_option("first_exp", 0)
bnn.set_option("first_db", 1)
t = tr.view(-1, 16).cpu().to(torch.float64)
n = int((t[:, 2] > 0).sum())
t = t[:n]
t0 = float(t[0, 12])
print("db=%d exp=%d tiles traced %d; clk relative to builder warp 1's first A-free" % (db, ex, n))
print("it   mma:ardy  mma:iss  mma:cmt | bld1..5 A ready                      | epi6..9 acc ready            | bld1 afree  epi rel")
for i in range(min(n, 24)):
    r = [int(v - t0) for v in t[i]]
    print("%2d %9d %8d %8d | %s | %s | %8d %8d" % (i, r[0], r[1], r[2], " ".join("%7d" % v for v in r[3:8]),
                                                   " ".join("%7d" % v for v in r[8:12]), r[12], r[13]))
s = slice(4, n)
b = t[s, 3:8]
e = t[s, 8:12]
print("median per-tile period %.0f clk" % float((t[5:n, 1] - t[4:n - 1, 1]).median()))
print("median spread of builder A-ready (last - first warp) %.0f clk" % float((b.max(1).values - b.min(1).values).median()))
print("median last builder A-ready -> MMA sees A-ready %.0f clk" % float((t[s, 0] - b.max(1).values).median()))
print("median MMA commit -> first / last epilogue wake %.0f / %.0f clk" % (
    float((e.min(1).values - t[s, 2]).median()), float((e.max(1).values - t[s, 2]).median())))
print("median MMA issue -> commit %.0f clk" % float((t[s, 2] - t[s, 1]).median()))
