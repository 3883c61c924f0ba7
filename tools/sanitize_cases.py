"""Small forward passes through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck; SURVEY §4 layer 4, §5 race detection).  Results are checked for determinism
between two runs; parity itself is tests/test_gpu_parity.py's job.
usage: compute-sanitizer --tool <tool> python tools/sanitize_cases.py [quick]"""
import sys
import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_00209_b200 as bnn  # noqa: E402
from paper_1808_00209_b200 import synth  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"


def run(spec, mode, n, opts, max_batch=4096):
    for k, v in opts.items():
        bnn.set_option(k, v)
    try:
        layers = synth.make_weights(spec, mode, 77)
        dl = [dict(L, wt=bnn.pack_weights(L["wt"].cuda())) for L in layers]
        T = synth.thresholds(3, 78).cuda() if mode in (1,) else (torch.tensor([-120.0]).cuda() if mode == 2 else None)
        in_dt = bnn.U8
        net = bnn.Net(spec["h"], spec["w"], spec["c"], in_dt, mode, T, dl, max_batch=max_batch)
        x = synth.images(n, spec["h"], spec["w"], spec["c"], 79).cuda()
        l1, c1 = net.forward(x)
        l2, c2 = net.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(l1, l2) and torch.equal(c1, c2), "nondeterministic forward"
        net.close()
    finally:
        for k in opts:
            bnn.set_option(k, {"conv_tc": 1, "first_db": 1, "first_tma": 1, "conv_tc_fp4": 1, "dense_tc": 1,
                               "streams": 2, "first_fp4": 0, "fused_max_n": 0}.get(k, 0))
    print("ok", spec["h"], mode, n, opts, flush=True)


run(synth.VEHICLE, 1, 260, {})                              # TMA first layer (db), pool-in-N mxf4 conv2, mxf4 dense
run(synth.VEHICLE, 1, 260, {"first_db": 0})                 # single accumulator set
if not quick:
    run(synth.VEHICLE, 0, 40, {"conv_tc": 0, "dense_tc": 0})  # integer-pipe (POPC) conv / dense
    run(synth.VEHICLE, -1, 40, {})                            # real-input first layer (kind::i8)
    run(synth.VEHICLE, 3, 40, {})                             # LBP pack + packed first layer
    run(synth.VEHICLE, 1, 6, {"fused_max_n": 8})              # whole-network cooperative kernel
    run(synth.CIFAR, 1, 20, {})                               # streamed wide-channel conv, two-image tiles
print("sanitize cases done")
