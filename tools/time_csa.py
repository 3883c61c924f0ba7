"""POPC-engine conv2 of the vehicle net with and without the carry-save popcount."""
import torch
import paper_1808_00209_b200 as bnn
from paper_1808_00209_b200 import synth
n = 8192
x = bnn.pack(synth.pm1((n, 48, 48, 32), 1).cuda())
w = bnn.pack_weights(synth.pm1((32, 5, 5, 32), 2).cuda())
bnn.set_option("conv_tc", 0)
for csa in (0, 1, 0, 1):
    bnn.set_option("csa", csa)
    for _ in range(2):
        bnn.conv2d(x, bnn.BITS, 32, w, 32, 5, pool=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        bnn.conv2d(x, bnn.BITS, 32, w, 32, 5, pool=2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    popc = n * 48 * 48 * 32 * 25
    print("csa=%d  %.3f ms  %.2f Tpopc-equivalent/s  (POPC roofline 4.65)" % (csa, ms, popc / ms / 1e9))
