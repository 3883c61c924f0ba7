"""Role timeline of the TMA first layer (bnn_set_trace): CTA (0,0), SM clocks per tile iteration.
usage: BNN_TRACE_LIB=1 python tools/trace_first.py [first_db] [first_exp]  (after `python -m paper_1808_00209_b200._build --trace`)"""
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
tr = torch.zeros(8 * 400, dtype=torch.int64, device="cuda")
bnn.set_trace(tr)
net.forward(x)
torch.cuda.synchronize()
bnn.set_trace(None)
bnn.set_option("first_exp", 0)
t = tr.view(-1, 8).cpu()
n = int((t[:, 2] > 0).sum())
t0 = int(t[0, 3])
names = ["mma:a_rdy", "mma:issue", "mma:commit", "bld:raw", "bld:afree", "bld:a_rdy", "epi:acc", "epi:rel"]
print("db=%d exp=%d tiles traced %d (clk relative to the first builder raw wait)" % (db, ex, n))
print("it " + " ".join("%10s" % s for s in names))
for i in range(min(n, 40)):
    print("%2d " % i + " ".join("%10d" % (int(v) - t0) for v in t[i]))
d = t[1:n] - t[:n - 1]
print("median per-tile period by event:", [int(v) for v in d.median(0).values])
lat = {"issue->acc ready (epi wake)": (t[:n, 6] - t[:n, 1]), "a_rdy(bld)->a_rdy(mma)": (t[:n, 0] - t[:n, 5]),
       "epi acc->rel": (t[:n, 7] - t[:n, 6]), "bld afree->a_rdy": (t[:n, 5] - t[:n, 4])}
for k, v in lat.items():
    print("median %-28s %d clk" % (k, int(v.median())))
