"""Parity of the CUDA path (libbnn.so through the C ABI) with the CPU oracle, element by element.

Binary layers must match bit-exactly: packed words, int32 accumulators and logits (north_star).
The f32 real first layer must match within 1e-5 relative error (reading R18).
Inputs come from paper_1808_00209_b200.synth (seeded, CPU generator), are copied to the GPU for the
CUDA path and handed unchanged to the oracle.  Sizes span several tiles and ragged tails.
"""
import numpy as np
import pytest
import torch

from paper_1808_00209_b200 import synth

pytestmark = pytest.mark.gpu


def u32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


def dev(t):
    return t.contiguous().cuda()


# ------------------------------------------------------------------------------------ pack
@pytest.mark.parametrize("dtype", [torch.uint8, torch.int8, torch.float32, torch.int32])
@pytest.mark.parametrize("c", [1, 3, 32, 33, 70])
def test_pack_sign(cuda, orc, dtype, c):
    g = torch.Generator().manual_seed(c)
    if dtype == torch.float32:
        x = torch.randn((2, 5, 7, c), generator=g)
        x[0, 0, 0, 0] = 0.0
        x[0, 0, 1, 0] = -0.0
    elif dtype == torch.uint8:
        x = torch.randint(0, 3, (2, 5, 7, c), generator=g, dtype=torch.uint8)
    else:
        x = torch.randint(-3, 4, (2, 5, 7, c), generator=g).to(dtype)
    y = u32(cuda.pack(dev(x), cuda.SIGN))
    ref = np.stack([orc.pack_channels(orc.binarize_input(x[i].numpy().astype(np.float64), orc.SIGN))
                    for i in range(2)])
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("n,h,w", [(3, 96, 96), (1, 5, 7), (2, 3, 3), (1, 1, 1)])
@pytest.mark.parametrize("mode", ["rgb", "rgb_int", "gray", "lbp"])
def test_pack_input_modes(cuda, orc, n, h, w, mode):
    x = synth.images(n, h, w, 3, 1000 + h + n)
    if mode == "rgb":
        T = synth.thresholds(3, 5)
        m = cuda.THRESH_RGB
    elif mode == "rgb_int":
        T = torch.tensor([-128.0, -100.0, -1.0])  # X + T = 0 ties occur
        m = cuda.THRESH_RGB
    elif mode == "gray":
        T = torch.tensor([-120.0])
        m = cuda.THRESH_GRAY
    else:
        T = None
        m = cuda.LBP
    y = u32(cuda.pack(dev(x), m, None if T is None else dev(T)))
    om = {cuda.THRESH_RGB: orc.THRESH_RGB, cuda.THRESH_GRAY: orc.THRESH_GRAY, cuda.LBP: orc.LBP}[m]
    ref = np.stack([orc.pack_channels(orc.binarize_input(x[i].numpy(), om, None if T is None else T.numpy()))
                    for i in range(n)])
    assert np.array_equal(y, ref)


def test_pack_rgb_f32(cuda, orc):
    x = torch.rand((2, 9, 11, 3)) * 300 - 20
    T = torch.tensor([-128.5, 3.25, -0.0])
    y = u32(cuda.pack(dev(x), cuda.THRESH_RGB, dev(T)))
    ref = np.stack([orc.pack_channels(orc.binarize_input(x[i].numpy(), orc.THRESH_RGB, T.numpy())) for i in range(2)])
    assert np.array_equal(y, ref)


# ------------------------------------------------------------------------------------ conv
def conv_case(cuda, orc, n, h, w, cin, cout, k, pool, thr=False, flip=False, seed=0):
    xs = synth.pm1((n, h, w, cin), 10 + seed)
    ws = synth.pm1((cout, k, k, cin), 20 + seed)
    t = synth.int_thresholds(cout, 30 + seed, -2 * k, 2 * k + 1) if thr else None
    f = synth.flips(cout, 40 + seed) if flip else None
    xp = cuda.pack(dev(xs))
    wp = cuda.pack_weights(dev(ws))
    y, acc = cuda.conv2d(xp, cuda.BITS, cin, wp, cout, k, None if t is None else dev(t), None if f is None else dev(f),
                         pool=pool, want_y=True, want_acc=True)
    torch.cuda.synchronize()
    acc = acc.cpu().numpy()
    y = u32(y)
    for i in range(n):
        ra = orc.conv_binary(xs[i].numpy(), ws.numpy())
        assert np.array_equal(acc[i], ra), "acc mismatch image %d" % i
        b = orc.binarize(ra, None if t is None else t.numpy(), None if f is None else f.numpy())
        if pool == 2:
            b = orc.maxpool2(b)
        assert np.array_equal(y[i], orc.pack_channels(b)), "packed mismatch image %d" % i


@pytest.mark.parametrize("n,h,w,cin,cout,k,pool", [
    (2, 48, 48, 32, 32, 5, 2),    # vehicle conv2
    (2, 96, 96, 3, 32, 5, 2),     # vehicle conv1 (dense-patch kernel)
    (1, 96, 96, 1, 32, 5, 2),     # gray conv1
    (3, 10, 14, 32, 32, 3, 1),    # ragged tiles
    (2, 12, 20, 40, 40, 3, 2),    # ragged channels (pad bits in and out, 2 groups)
    (1, 9, 7, 64, 33, 1, 1),      # k = 1, odd map
    (1, 16, 16, 300, 70, 3, 1),   # multi-chunk (cw = 10 > 8)
    (1, 13, 11, 16, 8, 7, 1),     # k = 7 patch path (7*7*16 > 256 -> generic)
    (1, 14, 18, 5, 20, 7, 2),     # k = 7 dense patch (245 bits = 8 words)
    (2, 8, 8, 128, 64, 3, 2),     # small map tile
    (1, 4, 6, 32, 32, 5, 1),      # map smaller than the kernel reach
    (1, 32, 32, 3, 128, 3, 1),    # CIFAR conv1 (27-bit patch)
])
@pytest.mark.parametrize("tc", [1, 0])
def test_conv_binary(cuda, orc, n, h, w, cin, cout, k, pool, tc):
    """tc = 1: layers with c_in >= 32 run on the tensor cores (tcgen05 kind::mxf4 by default, kind::i8 with
    conv_tc_fp4 = 0) where an instantiation exists; tc = 0: everything on the XOR-popcount integer path."""
    try:
        cuda.set_option("conv_tc", tc)
        conv_case(cuda, orc, n, h, w, cin, cout, k, pool, seed=h + cin + k)
    finally:
        cuda.set_option("conv_tc", 1)


@pytest.mark.parametrize("pool_tc", [1, 0])
@pytest.mark.parametrize("n,h,w,cin,cout,k,thr", [
    (2, 96, 96, 3, 32, 5, True),   # vehicle conv1 (with thresholds + flips)
    (2, 96, 96, 3, 32, 5, False),
    (1, 36, 20, 1, 40, 5, True),   # gray, c_out > 32 (NT = 64), ragged tiles
    (1, 34, 18, 2, 64, 7, False),  # k = 7
    (2, 32, 32, 5, 33, 3, True),   # c_in = 5, k = 3
])
def test_conv_first_layer_pooled_tc(cuda, orc, pool_tc, n, h, w, cin, cout, k, thr):
    """pool = 2 first layers: the pool-window-ordered tensor-core kernel (max of the 4 window sums,
    flips by negation) vs the unordered one, both against the oracle."""
    try:
        cuda.set_option("first_pool_tc", pool_tc)
        conv_case(cuda, orc, n, h, w, cin, cout, k, 2, thr=thr, flip=thr, seed=1700 + h + k + cin)
    finally:
        cuda.set_option("first_pool_tc", 1)


@pytest.mark.parametrize("n,h,w,cin,cout,k,pool", [
    (3, 48, 48, 32, 32, 5, 2),    # vehicle conv2 on tcgen05
    (1, 16, 16, 64, 70, 5, 2),    # c_out > NT: two channel tiles, ragged
    (1, 13, 11, 40, 36, 3, 1),    # cw = 2 with pad channels, ragged map
    (1, 16, 24, 128, 128, 3, 2),  # cw = 4, NT = 128
    (1, 14, 10, 32, 33, 7, 1),    # k = 7
    (5, 24, 16, 64, 64, 5, 1),    # many tiles per CTA (double-buffered TMEM accumulators)
    (2, 16, 16, 300, 70, 3, 1),   # streamed (big) kernel: cw = 10, partial last stage, pad channels
    (1, 12, 20, 256, 130, 5, 2),  # big k = 5: cw = 8, two N = 128 channel groups, ragged c_out
    (1, 10, 10, 64, 40, 7, 1),    # big k = 7
    (3, 8, 8, 512, 512, 3, 2),    # CIFAR conv6 shape (8-wide map: two images per tile, odd n)
    (5, 8, 8, 256, 130, 3, 1),    # two images per tile, ragged c_out, no pool
    (2, 12, 8, 256, 64, 3, 2),    # two images per tile, ragged tile rows
])
@pytest.mark.parametrize("fp4", [2, 1, 0])
def test_conv_tensor_core(cuda, orc, n, h, w, cin, cout, k, pool, fp4):
    """fp4 = 1: kind::mxf4 (packed e2m1, two taps per MMA; the streamed wide kernel stages a per-call
    weight image); fp4 = 2: the same with the weights expanded in-kernel; fp4 = 0: kind::i8."""
    try:
        cuda.set_option("conv_tc_fp4", 1 if fp4 else 0)
        cuda.set_option("big_img", 0 if fp4 == 2 else 1)
        conv_case(cuda, orc, n, h, w, cin, cout, k, pool, thr=True, flip=True, seed=900 + h + k)
    finally:
        cuda.set_option("conv_tc_fp4", 1)
        cuda.set_option("big_img", 1)


@pytest.mark.parametrize("n,h,w,cout,k,thr", [
    (3, 48, 48, 32, 5, True),    # vehicle conv2
    (2, 20, 36, 70, 5, True),    # ragged pooled tiles (10 x 18 pooled), three channel groups
    (1, 34, 18, 33, 3, False),   # k = 3, a 1-channel last group
    (4, 8, 16, 32, 5, True),     # map smaller than the 32 x 16 tile
    (1, 64, 64, 16, 3, True),    # c_out < 16: the second channel half stores zero pad bits
])
@pytest.mark.parametrize("pool_tc", [1, 0])
def test_conv_pool_tensor_core(cuda, orc, pool_tc, n, h, w, cout, k, thr):
    """Pooled 32-channel binary conv with the pool window folded into the MMA N dimension (4 shifted
    weight copies, thresholds as accumulator start values, flips as negated weights) vs the
    per-pixel tensor-core kernel, both against the oracle (sums, packed pooled bits)."""
    try:
        cuda.set_option("conv_pool_tc", pool_tc)
        conv_case(cuda, orc, n, h, w, 32, cout, k, 2, thr=thr, flip=thr, seed=2100 + h + w + k + cout)
    finally:
        cuda.set_option("conv_pool_tc", 1)


@pytest.mark.parametrize("csa", [1, 0])
@pytest.mark.parametrize("n,h,w,cin,cout,k,pool", [
    (2, 48, 48, 32, 32, 5, 2), (1, 13, 11, 64, 40, 3, 1), (1, 14, 10, 32, 33, 7, 2), (1, 9, 7, 300, 70, 1, 1)])
def test_conv_popc_csa(cuda, orc, csa, n, h, w, cin, cout, k, pool):
    """The XOR-popcount engine (Eq. 4) with and without the carry-save compression of each kernel
    row's K words equals the oracle bit for bit."""
    try:
        cuda.set_option("conv_tc", 0)
        cuda.set_option("csa", csa)
        conv_case(cuda, orc, n, h, w, cin, cout, k, pool, thr=True, flip=True, seed=2500 + h + k + cin)
    finally:
        cuda.set_option("conv_tc", 1)
        cuda.set_option("csa", 1)


@pytest.mark.parametrize("cin,k", [(3, 5), (32, 3)])
def test_conv_threshold_flip(cuda, orc, cin, k):
    conv_case(cuda, orc, 2, 16, 16, cin, 40, k, 2, thr=True, flip=True, seed=7)


@pytest.mark.parametrize("algo,tpc", [(1, 0), (2, 0), (3, 0), (4, 0), (5, 0), (0, 1), (0, 3), (1, 7), (3, 5), (4, 2)])
def test_conv_tiling_invariance(cuda, orc, algo, tpc):
    """Launch configuration does not change a single bit (and the generic kernel agrees with
    the dense-patch kernel on the first layer)."""
    try:
        cuda.set_option("conv_algo", algo)
        cuda.set_option("tiles_per_cta", tpc)
        conv_case(cuda, orc, 2, 24, 40, 3, 32, 5, 2, seed=3)
        conv_case(cuda, orc, 3, 16, 32, 32, 32, 3, 1, seed=4)
    finally:
        cuda.set_option("conv_algo", 0)
        cuda.set_option("tiles_per_cta", 0)


def test_conv_empty_batch(cuda):
    xp = torch.zeros((0, 8, 8, 1), dtype=torch.int32, device="cuda")
    wp = cuda.pack_weights(dev(synth.pm1((32, 3, 3, 32), 1)))
    y, _ = cuda.conv2d(xp, cuda.BITS, 32, wp, 32, 3)
    assert y.shape == (0, 8, 8, 1)


@pytest.mark.parametrize("tc", [1, 0])
@pytest.mark.parametrize("k,pool", [(5, 2), (3, 1), (1, 1), (7, 2)])
@pytest.mark.parametrize("cin", [3, 1])
def test_conv_real_u8(cuda, orc, k, pool, cin, tc):
    """Real u8 first layer: tc = 1 runs k in {3, 5} on tcgen05 with unsigned int8 A operands."""
    try:
        cuda.set_option("conv_tc", tc)
        _conv_real_u8_case(cuda, orc, k, pool, cin)
    finally:
        cuda.set_option("conv_tc", 1)


def _conv_real_u8_case(cuda, orc, k, pool, cin):
    n, h, w, cout = 2, 20, 24, 40
    x = synth.images(n, h, w, cin, 50 + k)
    ws = synth.pm1((cout, k, k, cin), 60 + k)
    t = synth.int_thresholds(cout, 61, -300, 300)
    y, acc = cuda.conv2d(dev(x), cuda.U8, cin, cuda.pack_weights(dev(ws)), cout, k, dev(t), None, pool=pool,
                         want_acc=True)
    torch.cuda.synchronize()
    acc = acc.cpu().numpy()
    y = u32(y)
    for i in range(n):
        ra = orc.conv_real(x[i].numpy().astype(np.float64), ws.numpy())
        assert np.array_equal(acc[i], ra.astype(np.int64))
        b = orc.binarize(ra, t.numpy())
        if pool == 2:
            b = orc.maxpool2(b)
        assert np.array_equal(y[i], orc.pack_channels(b))


def test_conv_real_f32(cuda, orc):
    n, h, w, cin, cout, k = 2, 12, 10, 3, 36, 5
    x = torch.randn((n, h, w, cin), generator=torch.Generator().manual_seed(3)) * 50
    ws = synth.pm1((cout, k, k, cin), 70)
    y, acc = cuda.conv2d(dev(x), cuda.F32, cin, cuda.pack_weights(dev(ws)), cout, k, None, None, pool=2, want_acc=True)
    torch.cuda.synchronize()
    acc = acc.cpu().numpy().astype(np.float64)
    y = u32(y)
    exempt = 0
    for i in range(n):
        ra = orc.conv_real(x[i].numpy().astype(np.float64), ws.numpy())
        scale = orc.conv_real(np.abs(x[i].numpy().astype(np.float64)), np.ones_like(ws.numpy()))[..., :1]
        assert np.all(np.abs(acc[i] - ra) <= 1e-5 * np.maximum(np.abs(ra), scale))
        ref_bits = orc.maxpool2(orc.binarize(ra))
        tiny = np.abs(ra) <= 1e-5 * scale  # sign decided by rounding: exempt (reading R18)
        tiny_any = tiny.reshape(h // 2, 2, w // 2, 2, cout).any(axis=(1, 3))
        mismatch = orc.unpack_channels(y[i], cout) != ref_bits
        assert not np.any(mismatch & ~tiny_any)
        exempt += int(mismatch.sum())
    assert exempt <= 4


# ------------------------------------------------------------------------------------ pool, dense
@pytest.mark.parametrize("n,h,w,c", [(2, 96, 96, 32), (3, 6, 10, 70), (1, 2, 2, 1)])
def test_maxpool(cuda, orc, n, h, w, c):
    xs = synth.pm1((n, h, w, c), 80 + c)
    y = u32(cuda.maxpool(cuda.pack(dev(xs)), c))
    for i in range(n):
        assert np.array_equal(y[i], orc.pack_channels(orc.maxpool2(xs[i].numpy())))


@pytest.mark.parametrize("n,d,l", [(5, 18432, 100), (130, 100, 100), (70, 100, 4), (33, 4096, 10), (1, 37, 1),
                                   (64, 2048, 1024)])
def test_dense(cuda, orc, n, d, l):
    xs = synth.pm1((n, d), 90 + d)
    ws = synth.pm1((l, d), 91 + l)
    t = synth.int_thresholds(l, 92, -4, 5)
    xp = cuda.pack(dev(xs).view(n, 1, 1, d)).view(n, -1)
    y, acc, cls = cuda.dense(xp, d, cuda.pack_weights(dev(ws)), l, dev(t), None, want_acc=True, want_cls=True)
    torch.cuda.synchronize()
    acc, y, cls = acc.cpu().numpy(), u32(y), cls.cpu().numpy()
    for i in range(n):
        ra = orc.dense(xs[i].numpy(), ws.numpy())
        assert np.array_equal(acc[i], ra)
        assert np.array_equal(y[i], orc.pack(orc.binarize(ra[None], t.numpy())[0], 32))
        assert cls[i] == orc.argmax(ra)


@pytest.mark.parametrize("n,d,l,flip", [(300, 18432, 100, False), (256, 2040, 10, True), (400, 1024, 300, True),
                                        (129, 4096, 129, False), (8192, 18432, 100, True)])
@pytest.mark.parametrize("ksplit,tma", [(1, 1), (0, 1), (1, 0), (0, 0)])
def test_dense_tensor_core(cuda, orc, n, d, l, flip, ksplit, tma):
    """Large-batch dense on tcgen05 (kind::mxf4): ragged image tiles, d with a partial last word,
    l > 256 (two output groups), thresholds + flips, fused argmax (l <= NT) or the argmax kernel;
    ksplit = 1: K split over grid.z + the reduction kernel where the tile grid is small (FC1 shapes);
    tma = 1: activation stages by TMA into a shared ring (out-of-range rows / words zero-filled)."""
    xs = synth.pm1((n, d), 95 + d)
    ws = synth.pm1((l, d), 96 + l)
    t = synth.int_thresholds(l, 97, -40, 41)
    f = synth.flips(l, 98) if flip else None
    xp = cuda.pack(dev(xs).view(n, 1, 1, d)).view(n, -1)
    try:
        cuda.set_option("dense_ksplit", ksplit)
        cuda.set_option("dense_tma", tma)
        y, acc, cls = cuda.dense(xp, d, cuda.pack_weights(dev(ws)), l, dev(t), None if f is None else dev(f),
                                 want_acc=True, want_cls=True)
        torch.cuda.synchronize()
    finally:
        cuda.set_option("dense_ksplit", 1)
        cuda.set_option("dense_tma", 1)
    acc, y, cls = acc.cpu().numpy(), u32(y), cls.cpu().numpy()
    for i in range(0, n, 7 if n < 1000 else 331):
        ra = orc.dense(xs[i].numpy(), ws.numpy())
        assert np.array_equal(acc[i], ra)
        b = orc.binarize(ra[None], t.numpy(), None if f is None else f.numpy())[0]
        assert np.array_equal(y[i], orc.pack(b, 32))
        assert cls[i] == orc.argmax(ra)


@pytest.mark.parametrize("gemv_max", [0, 1000])
@pytest.mark.parametrize("n,d,l", [(3, 18432, 100), (20, 100, 4), (7, 37, 40), (2, 4096, 10)])
def test_dense_gemv_and_gemm_paths(cuda, orc, gemv_max, n, d, l):
    try:
        cuda.set_option("gemv_max_n", gemv_max)
        test_dense(cuda, orc, n, d, l)
    finally:
        cuda.set_option("gemv_max_n", 255)  # (the default)


# ------------------------------------------------------------------------------------ forward
def build_net(cuda, spec, mode, seed, max_batch=4096, thr=False):
    layers = synth.make_weights(spec, mode, seed)
    dev_layers = []
    for i, L in enumerate(layers):
        D = dict(L)
        D["wt"] = cuda.pack_weights(dev(L["wt"]))
        if thr and i < len(layers) - 1:
            nout = L["c_out"] if L["kind"] == "conv" else L["l"]
            L["thr"] = synth.int_thresholds(nout, seed + i, -3, 4)
            L["flip"] = synth.flips(nout, seed + 50 + i)
            D["thr"], D["flip"] = dev(L["thr"]), dev(L["flip"])
        dev_layers.append(D)
    T = {1: synth.thresholds(3, seed), 2: torch.tensor([-127.0])}.get(mode)
    net = cuda.Net(spec["h"], spec["w"], spec["c"], cuda.U8, mode, None if T is None else dev(T), dev_layers,
                   max_batch=max_batch)
    return net, layers, T


def oracle_net(orc, spec, mode, layers, T):
    ol = []
    for L in layers:
        D = dict(L)
        D["wt"] = L["wt"].numpy()
        if L.get("thr") is not None:
            D["thr"] = L["thr"].numpy()
            D["flip"] = L["flip"].numpy()
        ol.append(D)
    om = {0: orc.SIGN, 1: orc.THRESH_RGB, 2: orc.THRESH_GRAY, 3: orc.LBP, -1: orc.NONE}[mode]
    return orc.Net(spec["h"], spec["w"], spec["c"], om, None if T is None else T.numpy(), ol)


@pytest.mark.parametrize("fused", [8, -8, 0])
@pytest.mark.parametrize("mode", [1, 2, 3, -1, 0])
def test_forward_vehicle(cuda, orc, mode, fused):
    """All input modes end to end; fused = 8: batches of <= 8 images run as one thread-block cluster
    (whole network, activations in DSMEM; RGB / SIGN), -8: the cooperative whole-network kernel,
    0: layer by layer."""
    forward_vehicle_case(cuda, orc, mode, fused)


def forward_vehicle_case(cuda, orc, mode, fused):
    net, layers, T = build_net(cuda, synth.VEHICLE, mode, 500 + mode)
    imgs = synth.images(6, 96, 96, 3, 600 + mode)
    try:
        cuda.set_option("fused_max_n", abs(fused))
        cuda.set_option("fused_cluster", 0 if fused < 0 else 1)
        logits, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
    finally:
        cuda.set_option("fused_max_n", 12)  # (the default)
        cuda.set_option("fused_cluster", 1)
    ref_logits, ref_cls = oracle_net(orc, synth.VEHICLE, mode, layers, T).forward(imgs.numpy(), threads=6)
    assert np.array_equal(logits.cpu().numpy(), ref_logits)
    assert np.array_equal(cls.cpu().numpy(), ref_cls)


@pytest.mark.parametrize("k1,k2,hw", [(3, 5, 64), (5, 3, 48), (5, 5, 96)])
def test_forward_fused_cluster_shapes(cuda, orc, k1, k2, hw):
    """The whole-network cluster kernel (f1) on vehicle-shaped nets other than the vehicle: conv1 k = 3 / 5, conv2
    k = 3 / 5, 64 / 48 / 96-pixel images (1 .. 3 pooled conv1 rows per CTA), thresholds and flips on every hidden
    layer; batches of 1 and 5 images against the oracle."""
    spec = dict(h=hw, w=hw, c=3, layers=[dict(kind="conv", k=k1, c_out=32, pool=2), dict(kind="conv", k=k2, c_out=32, pool=2),
                                         dict(kind="dense", l=100), dict(kind="dense", l=100), dict(kind="dense", l=4)])
    net, layers, T = build_net(cuda, spec, 1, 4400 + 10 * k1 + k2, max_batch=8, thr=True)
    imgs = synth.images(5, hw, hw, 3, 4401 + hw)
    try:
        cuda.set_option("fused_max_n", 8)
        assert cuda.forward_launches(net, 1) == 1, "the whole-network kernel must take this net"
        outs = [net.forward(dev(imgs[:1])), net.forward(dev(imgs))]
        torch.cuda.synchronize()
    finally:
        cuda.set_option("fused_max_n", 12)  # (the default)
    onet = oracle_net(orc, spec, 1, layers, T)
    for (lg, cls), x in zip(outs, (imgs[:1], imgs)):
        ref_l, ref_c = onet.forward(x.numpy(), threads=5)
        assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)


@pytest.mark.parametrize("algo", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", [1, 0])
def test_forward_vehicle_unfused_first_layer(cuda, orc, mode, algo):
    """The same net through the separate pack kernel + generic (1) / dense-patch (2) first layer."""
    try:
        cuda.set_option("conv_algo", algo)
        forward_vehicle_case(cuda, orc, mode, 0)
    finally:
        cuda.set_option("conv_algo", 0)


@pytest.mark.parametrize("algo", [3, 4, 5])
@pytest.mark.parametrize("k", [3, 5, 7])
@pytest.mark.parametrize("cin", [1, 2, 3, 4, 6])
def test_conv_strip_shapes(cuda, orc, k, cin, algo):
    if k * cin > 32:
        pytest.skip("strip wider than a word")
    try:
        cuda.set_option("conv_algo", algo)
        conv_case(cuda, orc, 2, 18, 20, cin, 36, k, 2, thr=True, seed=k * 10 + cin)
    finally:
        cuda.set_option("conv_algo", 0)


@pytest.mark.parametrize("algo", [0, 4, 1])
@pytest.mark.parametrize("T", [[-128.0, -0.5, -255.25], [float("nan"), float("inf"), -float("inf")], [0.0, -1e-7, 1e30]])
def test_forward_input_threshold_edges(cuda, orc, algo, T):
    """R14: the GPU's x > -T (integer compare on u8 in the fused first layer, fp32 in bnn_pack) equals
    the oracle's (double)x + T > 0 for integer, fractional, huge, infinite and NaN thresholds."""
    try:
        cuda.set_option("conv_algo", algo)
        layers = synth.make_weights(synth.VEHICLE, 1, 1500)
        Tt = torch.tensor(T, dtype=torch.float32)
        dl = [dict(L, wt=cuda.pack_weights(dev(L["wt"]))) for L in layers]
        net = cuda.Net(96, 96, 3, cuda.U8, 1, dev(Tt), dl, max_batch=8)
        imgs = synth.images(3, 96, 96, 3, 1501)
        imgs[0, :4, :4] = 128  # x + T = 0 ties for T = -128
        imgs[1, :4, :4] = 0
        imgs[2, :4, :4] = 255
        lg, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
        ref_l, ref_c = oracle_net(orc, synth.VEHICLE, 1, layers, Tt).forward(imgs.numpy(), threads=3)
        assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)
    finally:
        cuda.set_option("conv_algo", 0)


@pytest.mark.parametrize("tma", [3, 2, 1, 0])  # 3: mxf4 conv1_fp4 (default); 2 / 1: int8 TMA double / single buffered; 0: no TMA
@pytest.mark.parametrize("h,w,k,cout,T,mode", [
    (96, 96, 5, 32, None, 1),
    (34, 48, 5, 32, [-128.0, 3.0, -0.5], 1),   # t = (127, -1, 0): out-of-image bytes patched to -1
    (32, 16, 3, 40, None, 1),                  # NT = 64 group, partial second word
    (18, 32, 3, 96, [-20.0, -200.0, -90.0], 1),  # two channel groups (64 + 32), ragged tile rows
    (40, 64, 5, 64, None, 0),                  # SIGN mode: x > 0
    (2, 16, 5, 32, [1.0, 1.0, 1.0], 1),        # every in-image pixel +1, padding -1
])
def test_first_layer_fused_pooled(cuda, orc, tma, h, w, k, cout, T, mode):
    """The fused u8 -> threshold -> conv -> pool first layer (TMA-fed kernel with the thresholds and
    flips folded into the MMA, and the register-staged kernel) against the oracle, read out through a
    dense layer whose integer logits change by 2 for any wrong conv output bit."""
    tail = [dict(kind="conv", k=1, c_out=32, pool=1)] if cout % 32 else []  # dense needs C % 32 == 0
    spec = dict(h=h, w=w, c=3, layers=[dict(kind="conv", k=k, c_out=cout, pool=2)] + tail + [dict(kind="dense", l=8)])
    seed = h * 7 + w + k + cout
    layers = synth.make_weights(spec, mode, seed)
    layers[0]["thr"] = synth.int_thresholds(cout, seed, -30, 31)
    layers[0]["flip"] = synth.flips(cout, seed + 1)
    dl = [dict(L, wt=cuda.pack_weights(dev(L["wt"]))) for L in layers]
    dl[0]["thr"], dl[0]["flip"] = dev(layers[0]["thr"]), dev(layers[0]["flip"])
    Tt = None if mode == 0 else (synth.thresholds(3, seed) if T is None else torch.tensor(T, dtype=torch.float32))
    imgs = synth.images(5, h, w, 3, seed + 2)
    try:
        cuda.set_option("first_tma", 1 if tma else 0)
        cuda.set_option("first_fp4", 1 if tma == 3 else 0)
        cuda.set_option("first_db", 0 if tma == 1 else 1)
        net = cuda.Net(h, w, 3, cuda.U8, mode, None if Tt is None else dev(Tt), dl, max_batch=8)
        if tma:
            assert net.layer_kernel(0, 5) == ("conv1_fp4_pool_kernel" if tma == 3 else "conv_first_tma_pool_kernel")
        lg, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
    finally:
        cuda.set_option("first_tma", 1)
        cuda.set_option("first_fp4", 1)
        cuda.set_option("first_db", 1)
    ref_l, ref_c = oracle_net(orc, spec, mode, layers, Tt).forward(imgs.numpy(), threads=5)
    assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)


@pytest.mark.parametrize("pair", [1, 0])
@pytest.mark.parametrize("k2,h,w,n", [(3, 32, 32, 7), (5, 40, 80, 9), (5, 96, 96, 5)])
def test_forward_pooled_layers_weight_images(cuda, orc, pair, k2, h, w, n):
    """Nets whose pool-in-N layers stage weight images prepared once by bnn_net_create (first layer
    with two channel groups, a 32-channel conv with two channel groups), thresholds and flips on
    every hidden layer, integer logits out of a dense layer.  pair = 1: the 32-channel conv runs as CTA
    pairs (cta_group::2, M = 256; odd tile counts per chunk leave the last pair's second half empty)."""
    spec = dict(h=h, w=w, c=3, layers=[dict(kind="conv", k=5, c_out=32, pool=2), dict(kind="conv", k=k2, c_out=64, pool=2),
                                       dict(kind="dense", l=8)])
    net, layers, T = build_net(cuda, spec, 1, 3100 + k2, max_batch=4, thr=True)
    assert net.layer_kernel(0, 4) == "conv1_fp4_pool_kernel" and net.layer_kernel(1, 4) == "conv_tc4_pool3_kernel"
    imgs = synth.images(n, h, w, 3, 3101 + h)  # several chunks, the last one ragged
    cuda.set_option("conv_pair", pair)
    try:
        lg, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
    finally:
        cuda.set_option("conv_pair", 1)
    ref_l, ref_c = oracle_net(orc, spec, 1, layers, T).forward(imgs.numpy(), threads=7)
    assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)


@pytest.mark.parametrize("spec_name,mode,n", [("vehicle", 1, 3), ("vehicle", 0, 2), ("small_cifar", 1, 3)])
def test_forward_alg1_pipeline(cuda, orc, spec_name, mode, n):
    """The paper's own design (Alg. 1 im2col + packing, tiled XOR-popcount GEMM, int32 max-pool,
    64-segment FC) run through bnn_forward equals the oracle bit for bit."""
    spec = synth.VEHICLE if spec_name == "vehicle" else dict(h=16, w=16, c=3, layers=[
        dict(kind="conv", k=3, c_out=40, pool=1), dict(kind="conv", k=3, c_out=64, pool=2),
        dict(kind="conv", k=5, c_out=32, pool=2), dict(kind="dense", l=70), dict(kind="dense", l=10)])
    net, layers, T = build_net(cuda, spec, mode, 3300 + n)
    imgs = synth.images(n, spec["h"], spec["w"], 3, 3301 + n)
    try:
        cuda.set_option("alg1", 1)
        lg, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
    finally:
        cuda.set_option("alg1", 0)
    ref_l, ref_c = oracle_net(orc, spec, mode, layers, T).forward(imgs.numpy(), threads=n)
    assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)


@pytest.mark.parametrize("fused,streams", [(8, 2), (0, 2), (0, 1)])
def test_forward_thresholds_and_chunking(cuda, orc, fused, streams):
    """BN-folded integer thresholds + flips, and n > max_batch (chunked, ragged last chunk)."""
    net, layers, T = build_net(cuda, synth.VEHICLE, 1, 777, max_batch=2, thr=True)
    imgs = synth.images(5, 96, 96, 3, 778)
    try:
        cuda.set_option("fused_max_n", fused)
        cuda.set_option("streams", streams)  # chunks alternate over two streams / workspaces
        logits, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
    finally:
        cuda.set_option("fused_max_n", 12)  # (the default)
        cuda.set_option("streams", 2)
    ref_logits, ref_cls = oracle_net(orc, synth.VEHICLE, 1, layers, T).forward(imgs.numpy(), threads=5)
    assert np.array_equal(logits.cpu().numpy(), ref_logits)
    assert np.array_equal(cls.cpu().numpy(), ref_cls)


def test_forward_host_equals_forward(cuda):
    net, _, _ = build_net(cuda, synth.VEHICLE, 1, 900, max_batch=4096)
    imgs = synth.images(9000, 96, 96, 3, 901)  # 3 host chunks of <= 4096, ragged
    lg_d, cls_d = net.forward(dev(imgs))
    torch.cuda.synchronize()
    lg_h, cls_h = net.forward_host(imgs.pin_memory())
    assert torch.equal(lg_h, lg_d.cpu()) and torch.equal(cls_h, cls_d.cpu())
    assert cuda.forward_launches(net, 9000) == 3 * 6  # pack-fused conv1, conv2, FC1 (+ K-split reduction), FC2, FC3


@pytest.mark.parametrize("fused", [8, -8, 0])
@pytest.mark.parametrize("pdl", [1, 0])
def test_forward_staged_graph(cuda, orc, pdl, fused):
    """The graph-replayed latency path (config 1) equals the oracle, for n = 1 and n = 3, and a
    replay after new images were staged uses the new images."""
    cuda.set_option("pdl", pdl)  # programmatic dependent launch between the graph's kernels
    cuda.set_option("fused_max_n", abs(fused))  # one whole-network kernel per replay
    cuda.set_option("fused_cluster", 0 if fused < 0 else 1)  # cluster (8) or cooperative (-8) kernel
    try:
        net, layers, T = build_net(cuda, synth.VEHICLE, 1, 1400, max_batch=64)
        onet = oracle_net(orc, synth.VEHICLE, 1, layers, T)
        st_in, st_lg, st_cls = net.staging(4)
        for n, seed in [(1, 1401), (3, 1402), (1, 1403), (3, 1404)]:
            imgs = synth.images(n, 96, 96, 3, seed)
            st_in[:n].copy_(imgs.cuda())
            net.forward_staged(n)
            torch.cuda.synchronize()
            ref_l, ref_c = onet.forward(imgs.numpy(), threads=n)
            assert np.array_equal(st_lg[:n].cpu().numpy(), ref_l)
            assert np.array_equal(st_cls[:n].cpu().numpy(), ref_c)
    finally:
        cuda.set_option("pdl", 1)
        cuda.set_option("fused_max_n", 12)  # (the default)
        cuda.set_option("fused_cluster", 1)


def test_forward_cifar(cuda, orc):
    net, layers, T = build_net(cuda, synth.CIFAR, 1, 1200)
    imgs = synth.images(3, 32, 32, 3, 1201)
    logits, cls = net.forward(dev(imgs))
    torch.cuda.synchronize()
    ref_logits, ref_cls = oracle_net(orc, synth.CIFAR, 1, layers, T).forward(imgs.numpy(), threads=3)
    assert np.array_equal(logits.cpu().numpy(), ref_logits)
    assert np.array_equal(cls.cpu().numpy(), ref_cls)


def test_forward_fault_injection(cuda, orc):
    """Flipping one conv2 weight bit must change the GPU result exactly as it changes the
    oracle's (the parity check is sensitive)."""
    net, layers, T = build_net(cuda, synth.VEHICLE, 1, 1300)
    layers[1]["wt"][5, 2, 2, 7] *= -1
    dl = []
    for L in layers:
        D = dict(L)
        D["wt"] = cuda.pack_weights(dev(L["wt"]))
        dl.append(D)
    net2 = cuda.Net(96, 96, 3, cuda.U8, 1, dev(T), dl, max_batch=64)
    imgs = synth.images(4, 96, 96, 3, 1301)
    lg, _ = net2.forward(dev(imgs))
    torch.cuda.synchronize()
    ref, _ = oracle_net(orc, synth.VEHICLE, 1, layers, T).forward(imgs.numpy(), threads=4)
    assert np.array_equal(lg.cpu().numpy(), ref)


# ------------------------------------------------------------------------------------ f4 output scaling
@pytest.mark.parametrize("n,l", [(0, 4), (1, 4), (37, 10), (300, 100), (5, 1024)])
def test_affine(cuda, orc, n, l):
    """bnn_affine: fp32 scores bit-identical to the oracle's single-rounding fmaf value, within 1e-5
    relative of the fp64 value (north_star), and the first-maximum class of the fp32 scores (R25)."""
    g = torch.Generator().manual_seed(n * 1000 + l)
    acc = (torch.randint(-60, 61, (n, l), generator=g) * 2).to(torch.int32)
    if n > 1 and l > 3:
        acc[1, 2] = acc[1, 3] = 500  # a tie under any positive scale with equal bias
    scale = torch.rand(l, generator=g) * 2 + 0.01
    bias = torch.randn(l, generator=g)
    if l > 3:
        scale[3], bias[3] = scale[2], bias[2]
    scale[0] = -scale[0]  # a negative per-class scale (flipped BN)
    score, cls = cuda.affine(dev(acc), dev(scale), dev(bias))
    torch.cuda.synchronize()
    s64, s32, rcls = orc.affine(acc.numpy(), scale.numpy(), bias.numpy())
    if n == 0:
        return
    got = score.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), s32.view(np.uint32))
    assert np.all(np.abs(got - s64) <= 1e-5 * np.maximum(np.abs(s64), 1e-30) + 1e-30)
    assert np.array_equal(cls.cpu().numpy(), rcls)


@pytest.mark.parametrize("mode", [1, -1])
def test_forward_scores_vehicle(cuda, orc, mode):
    """bnn_forward_scores = oracle forward pass -> per-class affine (XNOR-Net alpha / folded output BN)."""
    net, layers, T = build_net(cuda, synth.VEHICLE, mode, 1700 + mode)
    imgs = synth.images(40, 96, 96, 3, 1710)
    g = torch.Generator().manual_seed(1720)
    scale = torch.rand(4, generator=g) + 0.5
    bias = torch.randn(4, generator=g) * 3
    logits, scores, cls = net.forward_scores(dev(imgs), dev(scale), dev(bias))
    torch.cuda.synchronize()
    ref_logits, _ = oracle_net(orc, synth.VEHICLE, mode, layers, T).forward(imgs.numpy(), threads=8)
    assert np.array_equal(logits.cpu().numpy(), ref_logits)
    _, s32, rcls = orc.affine(ref_logits, scale.numpy(), bias.numpy())
    assert np.array_equal(scores.cpu().numpy().view(np.uint32), s32.view(np.uint32))
    assert np.array_equal(cls.cpu().numpy(), rcls)


# ------------------------------------------------------------------------------------ GRAY / LBP first layer
@pytest.mark.parametrize("tma", [2, 1, 3, 0])
@pytest.mark.parametrize("h,w,k,cout,T", [(32, 48, 5, 32, -100.0), (18, 16, 3, 40, -100.0), (34, 64, 5, 64, -100.0),
                                          (32, 48, 5, 32, 5.0), (32, 16, 3, 32, -255.5)])
@pytest.mark.parametrize("mode", [2, 3])
def test_first_layer_luma_tma(cuda, orc, mode, h, w, k, cout, T, tma):
    """THRESH_GRAY (c_in = 1: zero weights on the two dummy channels) and LBP: luma (and the LBP neighbour
    bits, replicate border) computed inside the TMA-fed first layer (tma = 2), the row-band pre-pass
    luma_band_kernel (tma = 1; ragged last band) or luma_u8img4_kernel (tma = 3) + the TMA-fed first layer, or the
    packed-bit path (tma = 0), with BN thresholds / flips on the first layer, ragged tiles and channel
    groups, against the oracle.  GRAY T = -100 (Y + T = 0 ties), 5 (every pixel +1: the out-of-image
    bytes must still be -1), -255.5 (every pixel -1)."""
    if mode == 3 and T != -100.0:
        pytest.skip("T applies to THRESH_GRAY only")
    cin = 1 if mode == 2 else 3
    tail = [dict(kind="conv", k=1, c_out=32, pool=1)] if cout % 32 else []
    spec = dict(h=h, w=w, c=3, layers=[dict(kind="conv", k=k, c_out=cout, pool=2)] + tail + [dict(kind="dense", l=10)])
    seed = 1900 + h + k + mode
    layers = synth.make_weights(spec, mode, seed)
    assert layers[0]["wt"].shape[-1] == cin
    layers[0]["thr"] = synth.int_thresholds(cout, seed, -6, 7)
    layers[0]["flip"] = synth.flips(cout, seed + 1)
    dl = [dict(L, wt=cuda.pack_weights(dev(L["wt"]))) for L in layers]
    dl[0]["thr"], dl[0]["flip"] = dev(layers[0]["thr"]), dev(layers[0]["flip"])
    T = torch.tensor([T]) if mode == 2 else None  # integer T: Y + T = 0 ties occur
    imgs = synth.images(5, h, w, 3, seed + 2)
    imgs[0, :3, :3] = 100
    try:
        cuda.set_option("first_tma", 1 if tma else 0)
        cuda.set_option("luma_fused", 2 if tma == 2 else 0)
        cuda.set_option("luma_band", 0 if tma == 3 else 1)
        net = cuda.Net(h, w, 3, cuda.U8, mode, None if T is None else dev(T), dl, max_batch=8)
        if tma:
            assert net.layer_kernel(0, 5) == "conv1_fp4_pool_kernel"
        lg, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
        if tma == 2:
            assert cuda.forward_launches(net, 5) == len(spec["layers"]), "no luma pre-pass"
    finally:
        cuda.set_option("first_tma", 1)
        cuda.set_option("luma_fused", 1)
        cuda.set_option("luma_band", 1)
    ref_l, ref_c = oracle_net(orc, spec, mode, layers, T).forward(imgs.numpy(), threads=5)
    assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)


# ------------------------------------------------------------------------------------ real u8 first layer (TMA)
@pytest.mark.parametrize("tma", [1, 0])
@pytest.mark.parametrize("h,w,k,cout,fill", [(32, 48, 5, 32, None), (18, 16, 3, 40, None), (34, 64, 5, 64, None),
                                             (16, 16, 5, 32, 255)])
def test_first_layer_real_u8_tma(cuda, orc, h, w, k, cout, fill, tma):
    """Mode NONE (R5): real u8 pixels x +/-1 weights with zero padding on the TMA kernel (unsigned int8 A
    operand, bias r + 255 q in two slots) or the register-staged kernel: exact int32 accumulators,
    thresholds spanning the +/-K^2*3*255 range, flips, fused 2x2 pool; fill = 255: the extreme sums."""
    seed = 2100 + h + k + cout
    x = synth.images(3, h, w, 3, seed)
    if fill is not None:
        x[:] = fill
    wt = synth.pm1((cout, k, k, 3), seed + 1)
    thr = synth.int_thresholds(cout, seed + 2, -4000, 4001)
    thr[0], thr[1] = 19200, -19200  # beyond |acc| <= 19125: constant bits
    flip = synth.flips(cout, seed + 3)
    try:
        cuda.set_option("first_real_tma", tma)
        y, acc = cuda.conv2d(dev(x), cuda.U8, 3, cuda.pack_weights(dev(wt)), cout, k, dev(thr), dev(flip), pool=2,
                             want_acc=True)
        torch.cuda.synchronize()
    finally:
        cuda.set_option("first_real_tma", 1)
    for i in range(3):
        ra = orc.conv_real(x[i].numpy().astype(np.float64), wt.numpy())
        assert np.array_equal(acc[i].cpu().numpy(), ra.astype(np.int32))
        b = orc.maxpool2(orc.binarize(ra, thr.numpy(), flip.numpy()))
        assert np.array_equal(u32(y[i]), orc.pack_channels(b))


@pytest.mark.parametrize("mode", [2, 3, -1])
def test_forward_chunked_two_streams_modes(cuda, orc, mode):
    """GRAY / LBP / NONE nets over several chunks alternating between the two internal streams
    (max_batch 16, 37 images: 3 chunks, ragged last) equal the oracle; launch accounting matches."""
    net, layers, T = build_net(cuda, synth.VEHICLE, mode, 2300 + mode, max_batch=16)
    imgs = synth.images(37, 96, 96, 3, 2310 + mode)
    lg, cls = net.forward(dev(imgs))
    torch.cuda.synchronize()
    ref_l, ref_c = oracle_net(orc, synth.VEHICLE, mode, layers, T).forward(imgs.numpy(), threads=8)
    assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)
    assert net.layer_kernel(0, 16) == ("conv_first_tma_pool_kernel" if mode == -1 else "conv1_fp4_pool_kernel")
    # per chunk: 5 layers (+ LBP's luma pre-pass; GRAY computes its luma inside conv1; NONE reads the pixels)
    per_chunk = 6 if mode == 3 else 5
    assert cuda.forward_launches(net, 37) == 3 * per_chunk


def test_forward_scores_chunked(cuda, orc):
    """bnn_forward_scores over 3 chunks on two streams: scores / classes of every image."""
    net, layers, T = build_net(cuda, synth.VEHICLE, 1, 2400, max_batch=16)
    imgs = synth.images(40, 96, 96, 3, 2401)
    scale = torch.tensor([0.5, -1.25, 2.0, 1.0])
    bias = torch.tensor([3.0, 0.0, -2.5, 0.125])
    logits, scores, cls = net.forward_scores(dev(imgs), dev(scale), dev(bias))
    torch.cuda.synchronize()
    ref_l, _ = oracle_net(orc, synth.VEHICLE, 1, layers, T).forward(imgs.numpy(), threads=8)
    _, s32, rcls = orc.affine(ref_l, scale.numpy(), bias.numpy())
    assert np.array_equal(logits.cpu().numpy(), ref_l)
    assert np.array_equal(scores.cpu().numpy().view(np.uint32), s32.view(np.uint32))
    assert np.array_equal(cls.cpu().numpy(), rcls)


@pytest.mark.parametrize("mode", [2, 3, -1, 0])
def test_forward_staged_graph_modes(cuda, orc, mode):
    """The CUDA-graph latency path for GRAY / LBP (luma kernel + TMA first layer), NONE (real-u8 TMA
    first layer) and SIGN nets: replays with newly staged images equal the oracle."""
    net, layers, T = build_net(cuda, synth.VEHICLE, mode, 2500 + mode, max_batch=64)
    onet = oracle_net(orc, synth.VEHICLE, mode, layers, T)
    st_in, st_lg, st_cls = net.staging(4)
    for n, seed in [(1, 2501), (3, 2502), (1, 2503)]:
        imgs = synth.images(n, 96, 96, 3, seed + mode)
        st_in[:n].copy_(imgs.cuda())
        net.forward_staged(n)
        torch.cuda.synchronize()
        ref_l, ref_c = onet.forward(imgs.numpy(), threads=n)
        assert np.array_equal(st_lg[:n].cpu().numpy(), ref_l)
        assert np.array_equal(st_cls[:n].cpu().numpy(), ref_c)


@pytest.mark.parametrize("n,d,l,flip", [(40000, 4096, 100, True), (37889, 2040, 10, False)])
@pytest.mark.parametrize("tma", [1, 0])
def test_dense_tensor_core_two_cta_form(cuda, orc, n, d, l, flip, tma):
    """Batches with at least 2 x 148 image tiles run dense_tc4_kernel's two-CTAs-per-SM form (8-word
    stages, 2-slot weight ring; bnn_api.cu `two`): ragged last tile (37889 = 296 tiles + 1 image),
    a partial last word (d = 2040), thresholds + flips, fused argmax; sampled images against
    orc_dense including the first and last image of the batch."""
    xs = synth.pm1((n, d), 195 + d)
    ws = synth.pm1((l, d), 196 + l)
    t = synth.int_thresholds(l, 197, -40, 41)
    f = synth.flips(l, 198) if flip else None
    xp = cuda.pack(dev(xs).view(n, 1, 1, d)).view(n, -1)
    try:
        cuda.set_option("dense_tma", tma)
        y, acc, cls = cuda.dense(xp, d, cuda.pack_weights(dev(ws)), l, dev(t), None if f is None else dev(f),
                                 want_acc=True, want_cls=True)
        torch.cuda.synchronize()
    finally:
        cuda.set_option("dense_tma", 1)
    acc, y, cls = acc.cpu().numpy(), u32(y), cls.cpu().numpy()
    W = ws.numpy()
    for i in sorted(set(list(range(0, n, 997)) + [127, 128, n - 2, n - 1])):
        ra = orc.dense(xs[i].numpy(), W)
        assert np.array_equal(acc[i], ra), "acc mismatch image %d" % i
        b = orc.binarize(ra[None], t.numpy(), None if f is None else f.numpy())[0]
        assert np.array_equal(y[i], orc.pack(b, 32)), "bits mismatch image %d" % i
        assert cls[i] == orc.argmax(ra), "argmax mismatch image %d" % i


@pytest.mark.parametrize("n", [2, 7, 9, 12, 20])
@pytest.mark.parametrize("multi", [1, 0])
def test_forward_fused_multi_cluster(cuda, orc, n, multi):
    """The whole-network cluster kernel (f1) over a small batch: multi = 1 launches one 16-CTA cluster per image up
    to the clusters the device holds at once -- 16-CTA clusters while the images fit in one wave of them (n = 2, 7),
    8-CTA clusters beyond (n = 9, 12, 20; n = 20: each cluster serves every ncl-th image, so the per-cluster
    image count, barrier phases and box prefetch stride are exercised) -- multi = 0 one cluster for all images;
    thresholds and flips, against the oracle."""
    net, layers, T = build_net(cuda, synth.VEHICLE, 1, 4600 + n, max_batch=32, thr=True)
    imgs = synth.images(n, 96, 96, 3, 4601 + n)
    try:
        cuda.set_option("fused_max_n", 32)
        cuda.set_option("fused_multi", multi)
        assert cuda.forward_launches(net, n) == 1, "the whole-network kernel must take this batch"
        lg, cls = net.forward(dev(imgs))
        torch.cuda.synchronize()
    finally:
        cuda.set_option("fused_max_n", 12)  # (the default)
        cuda.set_option("fused_multi", 1)
    ref_l, ref_c = oracle_net(orc, synth.VEHICLE, 1, layers, T).forward(imgs.numpy(), threads=8)
    assert np.array_equal(lg.cpu().numpy(), ref_l) and np.array_equal(cls.cpu().numpy(), ref_c)
