"""Phase times of fused_cluster_kernel (whole vehicle net in one 16-CTA cluster) for a few single-image forwards
(diagnostics build: BNN_TRACE_LIB=1 python tools/trace_cluster.py, after `python -m paper_1808_00209_b200._build
--trace`).  Stamps (CTA 0, %globaltimer): 0 image start, 1 after conv1, 2 after conv2, 3 after FC1, 4 after FC2/3."""
import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8)
x = synth.images(4, 96, 96, 3, 6).cuda()
bnn.set_option("fused_max_n", 8)
bnn.set_option("trace_layer", 2)
tr = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
for n in (1, 1, 1, 4):
    tr.zero_()
    bnn.set_trace(tr)
    net.forward(x[:n])
    torch.cuda.synchronize()
    bnn.set_trace(None)
    t = tr.view(64, 8)[:n].cpu()
    for i in range(n):
        d = [int(t[i, k + 1] - t[i, k]) for k in range(4)]
        print("n=%d img %d: conv1 %d ns, conv2 %d ns, FC1 %d ns, FC2+FC3+argmax %d ns, total %d ns" % (n, i, *d, sum(d)))
bnn.set_option("fused_max_n", 0)
