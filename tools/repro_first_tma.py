"""Tiny repro of the fused pooled first layer (TMA kernel) for compute-sanitizer runs."""
import torch

from paper_1808_00209_b200 import bnn as cuda, synth

spec = synth.VEHICLE
layers = synth.make_weights(spec, 1, 5)
dl = [dict(L, wt=cuda.pack_weights(L["wt"].cuda())) for L in layers]
net = cuda.Net(96, 96, 3, cuda.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8)
print(net.layer_kernel(0, 2))
lg, cls = net.forward(synth.images(1, 96, 96, 3, 6).cuda())
torch.cuda.synchronize()
print(lg.cpu(), cls.cpu())
