"""Pins of the CPU oracle against things other than itself (CPU only, -m "not gpu").

Each test fixes the oracle to something the paper or mathematics determines independently:
hand-derived worked values (tests/golden/spec_examples.json, cited), closed forms, invariants,
exhaustive brute force on tiny inputs, and special cases that reduce to library routines
(torch float64 conv2d / max_pool2d / matmul, exact for integers below 2^53).  The tests are
chosen so that a dropped term, a wrong sign or index, a transposed operand, a wrong padding
value or a wrong bit order fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_1808_00209_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _expand(x):
    if isinstance(x, str):
        n, v = x.split("x")
        return [int(v)] * int(n)
    return x


def popcount(v: int) -> int:
    return bin(int(v)).count("1")


# ----------------------------------------------------------------------------- Eq. (1), (2)
def test_sign_eq1(orc):
    """Eq. (1): zero maps to -1."""
    assert orc.sign(0.0) == -1 and orc.sign(-0.0) == -1
    assert orc.sign(1e-300) == 1 and orc.sign(3.7) == 1 and orc.sign(-2.0) == -1


@pytest.mark.parametrize("case", GOLD["pack"])
def test_pack_golden(orc, case):
    x = _expand(case["x"])
    assert list(orc.pack(np.array(x, np.int8), case["B"])) == case["words"]
    assert list(orc.unpack(np.array(case["words"], np.uint32), len(x), case["B"])) == x


def test_pack_msb_first_matches_alg1_shift(orc):
    """Alg. 1 line 10: v |= s << (B - 1 - i) -- element i (0-based) of a word is
    bit B-1-i.  One-hot +1 vectors pin the bit order of Eq. (2) for every B."""
    for B in (1, 2, 9, 25, 32):
        for i in range(B):
            x = -np.ones(B, np.int8)
            x[i] = 1
            assert int(orc.pack(x, B)[0]) == 1 << (B - 1 - i)


def test_pack_partial_last_word(orc):
    """Reading R12: D not divisible by B -> the last word holds D mod B elements at the top
    positions, pad bits 0 (3 channels with B = 32 -> bits 31, 30, 29)."""
    assert int(orc.pack(np.array([1, 1, 1], np.int8), 32)[0]) == 0xE0000000
    assert int(orc.pack(np.array([1, -1, 1], np.int8), 32)[0]) == 0xA0000000
    w = orc.pack(np.ones(40, np.int8), 32)
    assert list(w) == [0xFFFFFFFF, 0xFF000000]


def test_unpack_rejects_pad_bits(orc):
    with pytest.raises(ValueError):
        orc.unpack(np.array([0xE0000001], np.uint32), 3, 32)
    with pytest.raises(ValueError):
        orc.unpack(np.array([1 << 9], np.uint32), 9, 9)


def test_pack_roundtrip_random(orc):
    rng = np.random.default_rng(1)
    for B in range(1, 33):
        for D in (1, B - 1 if B > 1 else 1, B, 3 * B + 1, 97):
            x = rng.choice(np.array([-1, 1], np.int8), D)
            assert np.array_equal(orc.unpack(orc.pack(x, B), D, B), x)


# ----------------------------------------------------------------------------- Eq. (4) identity
def _all_pm1(W):
    return np.array(list(itertools.product([-1, 1], repeat=W)), np.int8)


@pytest.mark.parametrize("W", range(1, 9))
def test_eq4_identity_exhaustive(orc, W):
    """Eq. (4) PAPER.md:265-267 for every pair of +/-1 vectors of length W <= 8: the oracle's
    +/-1 dot product equals W - 2 popc(pack(a) XOR pack(b)) with the oracle's own packer."""
    allv = _all_pm1(W)
    packed = [int(orc.pack(v, 32)[0]) for v in allv]
    for i, a in enumerate(allv):
        dots = orc.dense(a, allv)  # all 2^W dot products with a at once
        for j in range(len(allv)):
            assert dots[j] == W - 2 * popcount(packed[i] ^ packed[j])


@pytest.mark.parametrize("W", [25, 32, 64, 100])
def test_eq4_identity_random(orc, W):
    rng = np.random.default_rng(W)
    A = rng.choice(np.array([-1, 1], np.int8), (2000, W))
    Bm = rng.choice(np.array([-1, 1], np.int8), (50, W))
    pa = [orc.pack(a, 32) for a in A]
    pb = [orc.pack(b, 32) for b in Bm]
    for i in range(len(A)):
        dots = orc.dense(A[i], Bm)
        for j in range(len(Bm)):
            pc = sum(popcount(int(u) ^ int(v)) for u, v in zip(pa[i], pb[j]))
            assert dots[j] == W - 2 * pc
            assert abs(dots[j]) <= W and (dots[j] - W) % 2 == 0


@pytest.mark.parametrize("case", GOLD["xnor_dot"])
def test_xnor_dot_golden(orc, case):
    assert orc.dense(np.array(case["a"], np.int8), np.array([case["b"]], np.int8))[0] == case["dot"]


def test_weight_pack_golden(orc):
    case = GOLD["weight_pack"][0]
    k = np.array(case["kernel3x3"], np.float64).reshape(-1)
    signs = np.array([orc.sign(v) for v in k], np.int8)
    assert int(orc.pack(signs, case["B"])[0]) == case["word"]


# ----------------------------------------------------------------------------- Eq. (3) binary conv
def _torch_conv_pm1(x, wt):
    """Library special case: -1 padding + cross-correlation, float64 (exact)."""
    k = wt.shape[1]
    R = (k - 1) // 2
    xt = torch.from_numpy(x.astype(np.float64)).permute(2, 0, 1)[None]
    xt = F.pad(xt, (R, R, R, R), value=-1.0)
    wt_t = torch.from_numpy(wt.astype(np.float64)).permute(0, 3, 1, 2)
    return F.conv2d(xt, wt_t)[0].permute(1, 2, 0).numpy()


@pytest.mark.parametrize("h,w,cin,cout,k", [(3, 3, 1, 1, 3), (4, 4, 2, 3, 3), (5, 5, 3, 2, 5), (5, 7, 1, 4, 5),
                                            (6, 4, 5, 2, 1), (7, 7, 2, 2, 7), (2, 9, 3, 3, 5)])
def test_conv_binary_vs_torch(orc, h, w, cin, cout, k):
    x = synth.numpy(synth.pm1((h, w, cin), 10 + h * w + cin))
    wt = synth.numpy(synth.pm1((cout, k, k, cin), 20 + k + cout))
    acc = orc.conv_binary(x, wt)
    ref = _torch_conv_pm1(x, wt)
    assert np.array_equal(acc, ref.astype(np.int64))


@pytest.mark.parametrize("k,cin,h,w", [(3, 1, 4, 4), (5, 3, 6, 7), (5, 32, 7, 5), (7, 2, 9, 9), (1, 4, 3, 2)])
def test_conv_binary_closed_form_all_ones(orc, k, cin, h, w):
    """All-(+1) map and kernel with -1 padding: acc = c_in (2 n_in - K^2), n_in = in-map taps
    (reading R4: out-of-bounds taps count as -1 and in N = K^2 c_in).  All-(-1) kernel negates."""
    R = (k - 1) // 2
    x = np.ones((h, w, cin), np.int8)
    wt = np.ones((2, k, k, cin), np.int8)
    wt[1] = -1
    acc = orc.conv_binary(x, wt)
    for y in range(h):
        for xx in range(w):
            rows = sum(1 for d in range(-R, R + 1) if 0 <= y + d < h)
            cols = sum(1 for d in range(-R, R + 1) if 0 <= xx + d < w)
            n_in = rows * cols
            assert acc[y, xx, 0] == cin * (2 * n_in - k * k)
            assert acc[y, xx, 1] == -cin * (2 * n_in - k * k)
    if h > 2 * R and w > 2 * R:
        assert acc[R, R, 0] == k * k * cin


def test_conv_golden(orc):
    g = {c["name"]: c for c in GOLD["conv"]}
    c = g["checkerboard_vs_ones_3x3_centre"]
    x = np.array(c["x"], np.int8)[:, :, None]
    wt = np.array(c["w"], np.int8)[None, :, :, None]
    assert orc.conv_binary(x, wt)[c["at"][0], c["at"][1], 0] == c["acc"]
    c = g["corner_patch_27"]
    h, w = c["map_hw"]
    k = c["k"]
    kernel = orc.unpack(np.array([c["patch_word_B9"]], np.uint32), k * k, k * k).reshape(1, k, k, 1)
    acc = orc.conv_binary(np.ones((h, w, 1), np.int8), kernel)
    assert acc[0, 0, 0] == k * k  # the kernel equals the corner patch: perfect match
    assert np.all(acc <= k * k)
    c = g["all_ones_k5_c3_interior"]
    acc = orc.conv_binary(np.ones((7, 7, c["c_in"]), np.int8), np.ones((1, c["k"], c["k"], c["c_in"]), np.int8))
    assert acc[3, 3, 0] == c["acc_interior"]


def test_conv_orientation_not_transposed(orc):
    """Cross-correlation, not convolution and no (ky,kx) transposition
    (reading R3): a one-hot kernel at tap (ky,kx) reads x[y+ky-R, x+kx-R]."""
    rng = np.random.default_rng(5)
    h, w, k = 6, 7, 3
    x = rng.choice(np.array([-1, 1], np.int8), (h, w, 1))
    for ky in range(k):
        for kx in range(k):
            # kernel = +1 at (ky,kx), and +1/-1 pairs elsewhere cancel? use c_in=1: sum of 9 terms;
            # compare the difference of two kernels that differ only at (ky,kx)
            w1 = np.ones((1, k, k, 1), np.int8)
            w2 = w1.copy()
            w2[0, ky, kx, 0] = -1
            d = (orc.conv_binary(x, w1) - orc.conv_binary(x, w2))[:, :, 0]
            for y in range(h):
                for xx in range(w):
                    yy, xs = y + ky - 1, xx + kx - 1
                    v = x[yy, xs, 0] if 0 <= yy < h and 0 <= xs < w else -1
                    assert d[y, xx] == 2 * v


def test_conv_parity_and_range(orc):
    x = synth.numpy(synth.pm1((9, 8, 7), 3))
    wt = synth.numpy(synth.pm1((5, 3, 3, 7), 4))
    acc = orc.conv_binary(x, wt)
    N = 9 * 7
    assert np.all(np.abs(acc) <= N) and np.all((acc - N) % 2 == 0)


def test_conv_fault_injection_localised(orc):
    """flipping one weight changes only that output channel."""
    x = synth.numpy(synth.pm1((8, 8, 4), 6))
    wt = synth.numpy(synth.pm1((6, 3, 3, 4), 7))
    a0 = orc.conv_binary(x, wt)
    wt2 = wt.copy()
    wt2[3, 1, 2, 1] *= -1
    a1 = orc.conv_binary(x, wt2)
    diff = np.nonzero(np.any(a0 != a1, axis=(0, 1)))[0]
    assert list(diff) == [3]


# ----------------------------------------------------------------------------- real first layer
def test_conv_real_vs_torch_zero_pad(orc):
    x = synth.numpy(synth.images(1, 7, 6, 3, 11))[0].astype(np.float64)
    wt = synth.numpy(synth.pm1((4, 5, 5, 3), 12))
    acc = orc.conv_real(x, wt)
    ref = F.conv2d(torch.from_numpy(x).permute(2, 0, 1)[None], torch.from_numpy(wt.astype(np.float64)).permute(0, 3, 1, 2),
                   padding=2)[0].permute(1, 2, 0).numpy()
    assert np.array_equal(acc, ref)


def test_conv_real_closed_form(orc):
    """Constant image v, all-(+1) kernel, zero padding: acc = v c_in n_in (reading R5)."""
    v, k, cin, h, w = 7.0, 3, 2, 4, 5
    acc = orc.conv_real(np.full((h, w, cin), v), np.ones((1, k, k, cin), np.int8))
    for y in range(h):
        for xx in range(w):
            n_in = sum(1 for a in (-1, 0, 1) if 0 <= y + a < h) * sum(1 for b in (-1, 0, 1) if 0 <= xx + b < w)
            assert acc[y, xx, 0] == v * cin * n_in
    c = GOLD["real_conv"][0]
    acc = orc.conv_real(np.full((5, 5, 1), c["value"]), np.ones((1, c["k"], c["k"], 1), np.int8))
    assert acc[2, 2, 0] == c["acc_interior"]


# ----------------------------------------------------------------------------- threshold, pool, dense
def test_binarize_golden(orc):
    c = GOLD["binarize"][0]
    b = orc.binarize(np.array([c["acc"]], np.int64).reshape(1, -1)).reshape(-1)
    assert int(orc.pack(b, 4)[0]) == c["bits_B4"]


def test_binarize_threshold_flip(orc):
    acc = np.array([[-3, 0, 2, 7]], np.int64)
    assert list(orc.binarize(acc, thr=[2, -1, 2, 6])[0]) == [-1, 1, -1, 1]
    assert list(orc.binarize(acc, thr=[2, -1, 2, 6], flip=[1, 0, 0, 1])[0]) == [1, 1, -1, -1]


def test_maxpool_vs_torch_and_or(orc):
    x = synth.numpy(synth.pm1((6, 8, 5), 13))
    y = orc.maxpool2(x)
    ref = F.max_pool2d(torch.from_numpy(x.astype(np.float64)).permute(2, 0, 1)[None], 2)[0].permute(1, 2, 0).numpy()
    assert np.array_equal(y, ref.astype(np.int8))
    for case in GOLD["maxpool"]:
        b = np.array(case["bits"]).reshape(2, 2, 1) * 2 - 1
        assert (orc.maxpool2(b.astype(np.int8))[0, 0, 0] + 1) // 2 == case["out"]
    # OR of packed words == packed max (Table 2 pooling as a bitwise OR)
    px = orc.pack_channels(x)
    py = orc.pack_channels(y)
    por = px[0::2, 0::2] | px[0::2, 1::2] | px[1::2, 0::2] | px[1::2, 1::2]
    assert np.array_equal(py, por)


def test_sign_pool_commute(orc):
    """sign is monotone: binarize(maxpool_int(acc)) == maxpool(binarize(acc)) (reading R9)."""
    rng = np.random.default_rng(9)
    acc = rng.integers(-5, 6, (8, 6, 3)).astype(np.int64)
    a = orc.maxpool2(orc.binarize(acc))
    mp = F.max_pool2d(torch.from_numpy(acc.astype(np.float64)).permute(2, 0, 1)[None], 2)[0].permute(1, 2, 0).numpy()
    b = orc.binarize(mp.astype(np.int64))
    assert np.array_equal(a, b)


def test_dense_vs_matmul(orc):
    x = synth.numpy(synth.pm1((77,), 14))
    W = synth.numpy(synth.pm1((9, 77), 15))
    assert np.array_equal(orc.dense(x, W), W.astype(np.int64) @ x.astype(np.int64))
    assert orc.dense(x, x[None])[0] == 77 and orc.dense(x, -x[None])[0] == -77


@pytest.mark.parametrize("case", GOLD["argmax"])
def test_argmax_golden(orc, case):
    assert orc.argmax(case["v"]) == case["cls"]


# ----------------------------------------------------------------------------- input binarization
@pytest.mark.parametrize("case", GOLD["threshold"])
def test_threshold_golden(orc, case):
    x = np.full((1, 1, 1), case["x"], np.float64)
    assert orc.binarize_input(x, orc.THRESH_RGB, [case["T"]])[0, 0, 0] == case["out"]


def test_threshold_monotone_in_T(orc):
    x = synth.numpy(synth.images(1, 5, 5, 3, 21))[0]
    prev = None
    for t in range(-260, 10, 7):
        b = orc.binarize_input(x, orc.THRESH_RGB, [t, t + 1, t - 1])
        if prev is not None:
            assert np.all(b >= prev)  # raising T never flips +1 -> -1
        prev = b


@pytest.mark.parametrize("case", GOLD["luma"])
def test_luma_golden(orc, case):
    assert orc.luma(*case["rgb"]) == case["y"]


def test_gray_threshold(orc):
    x = np.zeros((1, 2, 3))
    x[0, 0] = [255, 0, 0]  # luma 76
    x[0, 1] = [0, 0, 255]  # luma 29
    assert list(orc.binarize_input(x, orc.THRESH_GRAY, [-50])[0, :, 0]) == [1, -1]
    assert list(orc.binarize_input(x, orc.THRESH_GRAY, [-76])[0, :, 0]) == [-1, -1]  # 76 - 76 = 0 -> -1


@pytest.mark.parametrize("case", GOLD["lbp"])
def test_lbp_golden(orc, case):
    g = np.array(case["gray3x3"], np.float64)
    x = np.repeat(g[:, :, None], 3, axis=2)  # R = G = B = v has luma v
    out = orc.binarize_input(x, orc.LBP)
    assert list(out[1, 1]) == case["centre_out"]


def test_lbp_orientation_and_border(orc):
    """Reading R16: channel j <- neighbour n_{3j} clockwise from top-left (TL, R, BL);
    replicate border (a corner pixel compares against itself for missing neighbours)."""
    g = np.zeros((3, 3))
    g[1, 2] = 9  # only R is brighter
    x = np.repeat(g[:, :, None], 3, axis=2)
    assert list(orc.binarize_input(x, orc.LBP)[1, 1]) == [-1, 1, -1]
    g = np.zeros((3, 3))
    g[2, 0] = 9  # only BL
    x = np.repeat(g[:, :, None], 3, axis=2)
    assert list(orc.binarize_input(x, orc.LBP)[1, 1]) == [-1, -1, 1]
    g = np.arange(9, dtype=np.float64).reshape(3, 3)
    x = np.repeat(g[:, :, None], 3, axis=2)
    # top-left corner (0,0): TL/BL clamp to itself or (1,0); R = (0,1) = 1 > 0
    assert list(orc.binarize_input(x, orc.LBP)[0, 0]) == [-1, 1, 1]


# ----------------------------------------------------------------------------- whole network
def _torch_forward(images, mode, T, layers):
    """Library composition of the Section 2 pipeline in float64 (independent of the oracle's
    code): input binarization written with torch ops (integer luma R15 as int64 tensor arithmetic,
    LBP R16 as comparisons against a replicate-padded luma plane, mode NONE as a zero-padded
    conv2d of the raw pixels, R5), conv2d with -1 padding, the threshold (acc > thr) XOR flip
    with acc <= thr -> -1 (Eq. 1, R23), max_pool2d, HWC flatten, matmul."""
    def binar(a, L, ax):
        t = torch.zeros(a.shape[ax], dtype=torch.float64) if L.get("thr") is None else \
            torch.as_tensor(np.asarray(L["thr"]), dtype=torch.float64)
        f = torch.zeros(a.shape[ax], dtype=torch.bool) if L.get("flip") is None else \
            torch.as_tensor(np.asarray(L["flip"]) != 0)
        shape = [1] * a.dim()
        shape[ax] = -1
        pos = (a > t.view(shape)) ^ f.view(shape)
        return pos.double() * 2 - 1

    x = torch.from_numpy(images.astype(np.float64))  # [n,h,w,c]
    xi = torch.from_numpy(images.astype(np.int64))
    if mode == 1:
        x = (x + torch.from_numpy(np.asarray(T, np.float32).astype(np.float64)) > 0).double() * 2 - 1
    elif mode == 0:
        x = (x > 0).double() * 2 - 1
    elif mode in (2, 3):
        Y = torch.div(299 * xi[..., 0] + 587 * xi[..., 1] + 114 * xi[..., 2] + 500, 1000, rounding_mode="floor")
        if mode == 2:
            x = ((Y.double() + float(np.float32(T[0]))) > 0).double()[..., None] * 2 - 1
        else:
            Yp = F.pad(Y.double()[:, None], (1, 1, 1, 1), mode="replicate")[:, 0]  # [n, h+2, w+2]
            h, w = Y.shape[1], Y.shape[2]
            tl = Yp[:, 0:h, 0:w]            # n0: top-left
            r = Yp[:, 1:h + 1, 2:w + 2]     # n3: right
            bl = Yp[:, 2:h + 2, 0:w]        # n6: bottom-left
            x = torch.stack([(nb > Y.double()).double() * 2 - 1 for nb in (tl, r, bl)], dim=-1)
    x = x.permute(0, 3, 1, 2)
    flat = None
    for i, L in enumerate(layers):
        wt = torch.from_numpy(L["wt"].astype(np.float64))
        last = i == len(layers) - 1
        if L["kind"] == "conv":
            R = (L["k"] - 1) // 2
            pad = 0.0 if (i == 0 and mode == -1) else -1.0
            a = F.conv2d(F.pad(x, (R, R, R, R), value=pad), wt.permute(0, 3, 1, 2))
            x = binar(a, L, 1)
            if L.get("pool", 1) == 2:
                x = F.max_pool2d(x, 2)
        else:
            if flat is None:
                flat = x.permute(0, 2, 3, 1).reshape(x.shape[0], -1)
            a = flat @ wt.T
            if last:
                return a.numpy().astype(np.int64)
            flat = binar(a, L, 1)
    raise AssertionError


@pytest.mark.parametrize("mode", [0, 1, 2, 3, -1])
@pytest.mark.parametrize("bn", [False, True])
def test_forward_vs_torch_composition(orc, mode, bn):
    """orc_forward for every input mode (SIGN, THRESH_RGB, THRESH_GRAY, LBP, NONE), with and without
    BN-folded thresholds / flips, against the torch composition above.  Odd map sizes (10x6 after
    the first pool: 5x3) and a c_out that is not a multiple of 32 exercise the HWC flatten."""
    spec = dict(h=10, w=6, c=3, layers=[dict(kind="conv", k=3, c_out=4, pool=2), dict(kind="conv", k=5, c_out=6, pool=1),
                                        dict(kind="dense", l=7), dict(kind="dense", l=5)])
    seed = 100 + 10 * mode + bn
    layers = synth.make_weights(spec, mode, seed, small_layers=spec["layers"])
    layers = [dict(L, wt=synth.numpy(L["wt"])) for L in layers]
    if bn:
        for j, L in enumerate(layers[:-1]):
            c = L["wt"].shape[0]
            lo, hi = (-300, 300) if (j == 0 and mode == -1) else (-6, 7)
            L["thr"] = synth.numpy(synth.int_thresholds(c, seed + j, lo, hi))
            L["flip"] = synth.numpy(synth.flips(c, seed + 50 + j))
    imgs = synth.numpy(synth.images(4, 10, 6, 3, 30 + mode))
    imgs[0] = 128  # flat image: every LBP comparison is a tie (-> -1), luma 128, X + T = 0 at T = -128
    T = {1: [-128.0, -100.0, -140.0], 2: [-128.0]}.get(mode)
    net = orc.Net(10, 6, 3, mode, T, layers)
    logits, cls = net.forward(imgs)
    ref = _torch_forward(imgs, mode, T, layers)
    assert np.array_equal(logits, ref)
    assert list(cls) == [int(np.argmax(r)) for r in ref]


@pytest.mark.parametrize("case", GOLD["binarize_real"])
def test_binarize_real_golden(orc, case):
    """orc_binarize_f64 (the real first layer's threshold, R5/R23) on hand-derived values: ties at
    acc == thr -> -1, signed zeros -> -1, thr / flip."""
    acc = np.array(case["acc"], np.float64).reshape(1, -1)
    out = orc.binarize(acc, thr=case["thr"], flip=case["flip"])[0]
    assert list(out) == case["out"]


def test_binarize_real_closed_form_none_layer(orc):
    """Mode NONE closed form: a constant image v with all-(+1) weights gives acc = v * C * n_in(y,x)
    (zero padding, R5).  With thr = v * C * 9 (the interior value, k = 3) every interior pixel is a
    tie -> -1, every border pixel is below -> -1; with thr = v * C * 6 - 1 the edge (non-corner)
    pixels and the interior are +1 and the corners (4 taps) are -1."""
    h, w, c, v = 5, 6, 3, 7.0
    wt = np.ones((1, 3, 3, c), np.int8)
    acc = orc.conv_real(np.full((h, w, c), v), wt)
    b = orc.binarize(acc, thr=[int(v * c * 9)])[..., 0]
    assert np.all(b == -1)
    b = orc.binarize(acc, thr=[int(v * c * 6) - 1])[..., 0]
    corner = np.zeros((h, w), bool)
    corner[[0, 0, -1, -1], [0, -1, 0, -1]] = True
    assert np.all(b[corner] == -1) and np.all(b[~corner] == 1)
    b = orc.binarize(acc, thr=[int(v * c * 6) - 1], flip=[1])[..., 0]
    assert np.all(b[corner] == 1) and np.all(b[~corner] == -1)


def test_forward_equals_layer_composition(orc):
    """orc_forward == the per-layer oracle functions chained by hand (NONE mode included)."""
    spec = dict(h=6, w=6, c=3, layers=[dict(kind="conv", k=3, c_out=5, pool=2), dict(kind="dense", l=4)])
    layers = synth.make_weights(spec, -1, 7, small_layers=spec["layers"])
    layers = [dict(L, wt=synth.numpy(L["wt"])) for L in layers]
    img = synth.numpy(synth.images(1, 6, 6, 3, 8))[0].astype(np.float64)
    net = orc.Net(6, 6, 3, orc.NONE, None, layers)
    logits, cls = net.forward_one(img)
    a = orc.conv_real(img, layers[0]["wt"])
    b = orc.maxpool2(orc.binarize(a))
    ref = orc.dense(b.reshape(-1), layers[1]["wt"])
    assert np.array_equal(logits, ref) and cls == orc.argmax(ref)


def test_conv_point_equals_full(orc):
    x = synth.numpy(synth.pm1((7, 9, 5), 40))
    wt = synth.numpy(synth.pm1((3, 5, 5, 5), 41))
    acc = orc.conv_binary(x, wt)
    for (y, xx, o) in [(0, 0, 0), (3, 4, 1), (6, 8, 2), (0, 8, 1), (6, 0, 0)]:
        assert orc.conv_binary_point(x, wt[o], y, xx) == acc[y, xx, o]


# ----------------------------------------------------------------------------- f4 output scaling
def test_affine_identity_and_integer_argmax(orc):
    """scale = 1, bias = 0 reproduces the integer logits and the integer argmax (R19), ties included."""
    rng = np.random.default_rng(7)
    acc = rng.integers(-100, 101, size=(200, 10)) * 2
    acc[:, 3] = acc[:, 7]  # ties -> first maximum
    s64, s32, cls = orc.affine(acc, np.ones(10), np.zeros(10))
    assert np.array_equal(s64, acc.astype(np.float64)) and np.array_equal(s32, acc.astype(np.float32))
    assert np.array_equal(cls, np.array([orc.argmax(a) for a in acc]))


def test_affine_negative_scale_is_argmin(orc):
    """A uniform negative scale turns the decision into the first minimum."""
    rng = np.random.default_rng(8)
    acc = rng.integers(-50, 51, size=(100, 4))
    _, _, cls = orc.affine(acc, np.full(4, -0.25), np.zeros(4))
    assert np.array_equal(cls, np.argmin(acc, axis=1))


def test_affine_closed_form_dyadic(orc):
    """Dyadic scale/bias (exact in fp32 and fp64): score = scale*acc + bias in closed form, per class."""
    acc = np.array([[7, -3, 0, 12]])
    scale = np.array([0.5, -2.0, 4.0, 0.125])
    bias = np.array([1.25, 0.5, -3.0, 0.0])
    s64, s32, cls = orc.affine(acc, scale, bias)
    want = [4.75, 6.5, -3.0, 1.5]
    assert s64[0].tolist() == want and s32[0].tolist() == want and cls[0] == 1


def test_affine_fp32_single_rounding(orc):
    """score32 is the fp64 value rounded once to fp32 (|acc| < 2^24, so the product is exact in
    fp64 and the fp64 sum of two fp32-exact terms rounds at most at 2^-53 relative)."""
    rng = np.random.default_rng(9)
    acc = rng.integers(-20000, 20001, size=(50, 16))
    scale = rng.standard_normal(16).astype(np.float32)
    bias = rng.standard_normal(16).astype(np.float32)
    s64, s32, _ = orc.affine(acc, scale, bias)
    exact = scale.astype(np.float64)[None] * acc + bias.astype(np.float64)[None]
    assert np.array_equal(s64, exact)
    assert np.max(np.abs(s32.astype(np.float64) - exact) / np.maximum(np.abs(exact), 1e-30)) < 2 ** -23
