"""Phase times of fused_cluster_kernel (whole vehicle net in one 16-CTA cluster) for a few single-image forwards
(diagnostics build: BNN_TRACE_LIB=1 python tools/trace_cluster.py, after `python -m paper_1808_00209_b200._build
--trace`).  Stamps (CTA 0, %globaltimer): 0 image start, 5 raw rows staged, 6 bit image built, 1 after conv1, 2 after conv2,
3 after FC1, 7 after FC2, 4 after FC3 + argmax."""
import torch

import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth

layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
net = bnn.Net(96, 96, 3, bnn.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8)
x = synth.images(4, 96, 96, 3, 6).cuda()
bnn.set_option("fused_max_n", 8)
bnn.set_option("trace_layer", 2)
tr = torch.zeros(65 * 8, dtype=torch.int64, device="cuda")
for n in (1, 1, 1, 4):
    tr.zero_()
    bnn.set_trace(tr)
    net.forward(x[:n])
    torch.cuda.synchronize()
    bnn.set_trace(None)
    t = tr.view(65, 8)[:n].cpu()
    for i in range(n):
        d = [int(t[i, k + 1] - t[i, k]) for k in range(4)]
        print("n=%d img %d: conv1 %d ns (raw staged +%d, warp 0 pixels done +%d), conv2 %d ns, FC1 %d ns, FC2+FC3+argmax %d ns (FC2 +%d),"
              " total %d ns" % (n, i, d[0], int(t[i, 5] - t[i, 0]), int(t[i, 6] - t[i, 0]), d[1], d[2], d[3],
                                int(t[i, 7] - t[i, 3]), sum(d)))
    k = tr.view(65, 8)[64].cpu()
    print("   kernel: entry -> prologue done %d ns, -> image 0 start %d ns, last image end -> exit barrier done %d ns" % (
        int(k[1] - k[0]), int(t[0, 0] - k[0]), int(k[3] - k[2])))
bnn.set_option("fused_max_n", 0)
