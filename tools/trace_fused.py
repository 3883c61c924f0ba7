import torch
from paper_1808_00209_b200 import bnn as cuda, synth
layers = synth.make_weights(synth.VEHICLE, 1, 5)
dl = [dict(L, wt=cuda.pack_weights(L["wt"].cuda())) for L in layers]
net = cuda.Net(96, 96, 3, cuda.U8, 1, synth.thresholds(3, 5).cuda(), dl, max_batch=8)
x = synth.images(1, 96, 96, 3, 6).cuda()
for i in range(4):
    net.forward(x)
    torch.cuda.synchronize()
st_in, st_lg, st_cls = net.staging(1)
st_in.copy_(x)
for i in range(3):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); net.forward_staged(1); e.record(); torch.cuda.synchronize(); print("graph us", s.elapsed_time(e) * 1000)
