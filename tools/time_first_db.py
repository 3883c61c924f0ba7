"""Vehicle forward with the first layer's TMEM accumulators single- vs double-buffered."""
import torch
import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth
B = 32768
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8192)
x = synth.images(B, 96, 96, 3, 6).cuda()
lg = torch.empty((B, 4), dtype=torch.int32, device="cuda"); cls = torch.empty((B,), dtype=torch.int32, device="cuda")
ref = None
for db in (0, 1, 0, 1):
    bnn.set_option("first_db", db)
    for _ in range(3):
        net.forward(x, lg, cls)
    torch.cuda.synchronize()
    if ref is None:
        ref = lg.clone()
    assert torch.equal(ref, lg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        net.forward(x, lg, cls)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("first_db=%d  %.3f ms/step  %.2f M img/s" % (db, ms, B / ms / 1e3))
