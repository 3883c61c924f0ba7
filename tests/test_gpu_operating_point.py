"""Oracle parity of the CUDA path at the bench operating point and at the config-3 extremes.

The end-to-end tests in test_gpu_parity.py use <= 40 images, so each persistent CTA of the
first layer sees <= 3 tiles.  Here the vehicle net runs at bench.py's chunk size (16384 images per
chunk, two full chunks on two streams plus a ragged third): ~1000 conv1 tiles per CTA, so the
8-deep TMA raw ring, both TMEM accumulator sets and every mbarrier phase wrap many times, and
pooled conv2 runs hundreds of tiles per CTA.  Sampled images spread over the batch (first, last,
chunk boundaries) are compared bit-exactly with the oracle (Eq. 1-4, PAPER.md:108-110, 186-195,
212-219, 263-267); every image is compared with a differently tiled run of the same library.

The wide single layers of config 3 (C = 1024, k in {3, 5}; the streamed kernel with 8 / 16 stages
per tile and several tiles per CTA) are compared at sampled outputs through orc_conv_binary_point,
FC1 at the operating point through orc_dense on sampled images.
"""
import numpy as np
import pytest
import torch

from paper_1808_00209_b200 import synth

from test_gpu_parity import build_net, oracle_net, u32

pytestmark = pytest.mark.gpu

CHUNK = 16384
N_OP = 2 * CHUNK + 1000  # two full chunks (one per internal stream) + a ragged third


def _sample_idx(n, chunk, extra, seed):
    rng = np.random.default_rng(seed)
    fixed = [0, 1, chunk - 1, chunk, 2 * chunk - 1, 2 * chunk, n - 2, n - 1]
    rand = rng.choice(n, extra, replace=False).tolist()
    return sorted(set(i for i in fixed + rand if 0 <= i < n))


@pytest.fixture(scope="module")
def op_images():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return synth.images_chunked(0, N_OP, 96, 96, 3, 7001, device="cuda")


@pytest.mark.parametrize("mode,thr,fp4", [(1, False, 1), (1, True, 1), (1, True, 0), (2, False, 1), (3, False, 1),
                                          (-1, True, 1), (0, False, 1)])
def test_forward_operating_point(cuda, orc, op_images, mode, thr, fp4):
    cuda.set_option("first_fp4", fp4)  # 1: conv1_fp4_pool_kernel (default), 0: the int8 TMA kernel
    try:
        _operating_point(cuda, orc, op_images, mode, thr, fp4)
    finally:
        cuda.set_option("first_fp4", 1)


def _operating_point(cuda, orc, op_images, mode, thr, fp4):
    net, layers, T = build_net(cuda, synth.VEHICLE, mode, 7100 + mode, max_batch=CHUNK, thr=thr)
    assert net.layer_kernel(0, CHUNK) == ("conv1_fp4_pool_kernel" if fp4 and mode != -1 else "conv_first_tma_pool_kernel")
    assert net.layer_kernel(1, CHUNK) == "conv_tc4_pool3_kernel"
    logits, cls = net.forward(op_images)
    torch.cuda.synchronize()
    idx = _sample_idx(N_OP, CHUNK, 12, 7200 + mode)
    ref_l, ref_c = oracle_net(orc, synth.VEHICLE, mode, layers, T).forward(op_images[idx].cpu().numpy(), threads=8)
    got_l, got_c = logits[idx].cpu().numpy(), cls[idx].cpu().numpy()
    bad = [i for j, i in enumerate(idx) if not (np.array_equal(got_l[j], ref_l[j]) and got_c[j] == ref_c[j])]
    assert not bad, "images differing from the oracle: %s" % bad
    # every image: a differently tiled run (512-image chunks, one stream, other CTA/tile assignment)
    net2, _, _ = build_net(cuda, synth.VEHICLE, mode, 7100 + mode, max_batch=512, thr=thr)
    lo, hi = CHUNK - 700, CHUNK + 900  # straddles the first chunk boundary of the big run
    l2, c2 = net2.forward(op_images[lo:hi])
    torch.cuda.synchronize()
    assert torch.equal(l2, logits[lo:hi]) and torch.equal(c2, cls[lo:hi])
    net.close()
    net2.close()


@pytest.mark.parametrize("k,c,hw,n,pool", [(3, 1024, 32, 12, 1), (5, 1024, 16, 16, 1), (3, 512, 8, 64, 2),
                                           (5, 256, 24, 24, 2)])
def test_conv_wide_sampled(cuda, orc, k, c, hw, n, pool):
    """bnn_conv2d on config-3-wide layers (streamed conv_tc4_big_kernel: c / 32 words per pixel in
    stages, several tiles per CTA) at ~250 sampled outputs against orc_conv_binary_point (Eq. 3),
    packed bits (Eq. 1, pooled as OR) at every sampled pooled pixel."""
    xs = synth.pm1((n, hw, hw, c), 8000 + k + c)
    ws = synth.pm1((c, k, k, c), 8100 + k + c)
    xp = cuda.pack(xs.cuda())
    wp = cuda.pack_weights(ws.cuda())
    y, acc = cuda.conv2d(xp, cuda.BITS, c, wp, c, k, pool=pool, want_y=True, want_acc=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(k * c + hw)
    xs_np, ws_np = xs.numpy(), ws.numpy()
    pts = [(n - 1, hw - 1, hw - 1, c - 1), (0, 0, 0, 0), (n - 1, 0, hw - 1, 1)]
    pts += [(int(rng.integers(n)), int(rng.integers(hw)), int(rng.integers(hw)), int(rng.integers(c))) for _ in range(250)]
    acc_np = acc.cpu().numpy()
    for (i, yy, xx, o) in pts:
        ref = orc.conv_binary_point(xs_np[i], ws_np[o], yy, xx)
        assert acc_np[i, yy, xx, o] == ref, "acc mismatch at %s" % ((i, yy, xx, o),)
    # packed output at sampled (pooled) pixels: every channel from the oracle's points
    yw = u32(y)
    for (i, yy, xx, _) in pts[:24]:
        py, px = yy // pool, xx // pool
        win = [(py * pool + a, px * pool + b) for a in range(pool) for b in range(pool)]
        bits = np.full(c, -1, np.int8)
        for o in range(c):
            v = max(orc.sign(orc.conv_binary_point(xs_np[i], ws_np[o], wy, wx)) for (wy, wx) in win)
            bits[o] = v
        assert np.array_equal(yw[i, py, px], orc.pack(bits)), "packed mismatch at %s" % ((i, py, px),)


def test_dense_operating_point_sampled(cuda, orc):
    """FC1 of the vehicle net at bench.py's chunk (16384 images, d = 18432, l = 100: dense_tc4_kernel)
    on 48 sampled images against orc_dense, bits and accumulators."""
    n, d, l = CHUNK, 18432, 100
    x = synth.words((n, d // 32), 8300, device="cuda")
    ws = synth.pm1((l, d), 8301)
    wp = cuda.pack_weights(ws.cuda())
    y, acc, _ = cuda.dense(x, d, wp, l, want_y=True, want_acc=True)
    torch.cuda.synchronize()
    idx = _sample_idx(n, 4096, 40, 8302)
    xw = u32(x[idx])
    acc_np, yw = acc.cpu().numpy(), u32(y)
    W = ws.numpy()
    for j, i in enumerate(idx):
        xv = orc.unpack(xw[j], d)
        ra = orc.dense(xv, W)
        assert np.array_equal(acc_np[i], ra.astype(np.int32)), "acc mismatch image %d" % i
        assert np.array_equal(yw[i], orc.pack(orc.binarize(ra[None])[0])), "bits mismatch image %d" % i


def test_forward_bench_chunk(cuda, orc):
    """The vehicle net at bench.py's default chunk (65536 images: FC1 in the two-CTAs-per-SM form,
    512 conv tiles per CTA pair wave) with a ragged second chunk on the other stream: sampled images
    against the oracle, and every image against a 16384-image-chunk run of the same net (the one-CTA
    FC1 form, other tile assignment)."""
    big, n = 65536, 65536 + 1000
    imgs = synth.images_chunked(0, n, 96, 96, 3, 7301, device="cuda")
    net, layers, T = build_net(cuda, synth.VEHICLE, 1, 7302, max_batch=big)
    logits, cls = net.forward(imgs)
    torch.cuda.synchronize()
    idx = _sample_idx(n, big, 8, 7303)
    ref_l, ref_c = oracle_net(orc, synth.VEHICLE, 1, layers, T).forward(imgs[idx].cpu().numpy(), threads=8)
    got_l, got_c = logits[idx].cpu().numpy(), cls[idx].cpu().numpy()
    bad = [i for j, i in enumerate(idx) if not (np.array_equal(got_l[j], ref_l[j]) and got_c[j] == ref_c[j])]
    assert not bad, "images differing from the oracle: %s" % bad
    net2, _, _ = build_net(cuda, synth.VEHICLE, 1, 7302, max_batch=CHUNK)
    l2, c2 = net2.forward(imgs)
    torch.cuda.synchronize()
    assert torch.equal(l2, logits) and torch.equal(c2, cls)
    net.close()
    net2.close()
