"""ctypes binding of the CPU oracle (oracle/bnn_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It never imports
the CUDA package (paper_1808_00209_b200) and the CUDA package never imports it.

All arrays are numpy.  +/-1 tensors are int8; accumulators int64 (float64 for the
real first layer); images are passed to C as float64 (exact for u8/i8/f32/i32).
Every wrapper names the PAPER.md passage its C function writes out; see
bnn_oracle.h for the definitions.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bnn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

SIGN, THRESH_RGB, THRESH_GRAY, LBP, NONE = 0, 1, 2, 3, -1

_c_i8p = ctypes.POINTER(ctypes.c_int8)
_c_u8p = ctypes.POINTER(ctypes.c_uint8)
_c_u32p = ctypes.POINTER(ctypes.c_uint32)
_c_i32p = ctypes.POINTER(ctypes.c_int32)
_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_f64p = ctypes.POINTER(ctypes.c_double)
_c_f32p = ctypes.POINTER(ctypes.c_float)


class OrcLayer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("k", ctypes.c_int), ("c_out", ctypes.c_int),
                ("pool", ctypes.c_int), ("l", ctypes.c_int), ("wt", _c_i8p),
                ("thr", _c_i32p), ("flip", _c_u8p)]


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no -march tuning: it is a checker)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "bnn_oracle.h"))):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.orc_sign.argtypes = [ctypes.c_double]
        L.orc_sign.restype = ctypes.c_int
        L.orc_pack.argtypes = [_c_i8p, ctypes.c_int64, ctypes.c_int, _c_u32p]
        L.orc_pack.restype = ctypes.c_int64
        L.orc_unpack.argtypes = [_c_u32p, ctypes.c_int64, ctypes.c_int, _c_i8p]
        L.orc_unpack.restype = ctypes.c_int
        L.orc_luma.argtypes = [ctypes.c_int] * 3
        L.orc_luma.restype = ctypes.c_int
        L.orc_binarize_input.argtypes = [_c_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         _c_f64p, _c_i8p]
        L.orc_binarize_input.restype = ctypes.c_int
        L.orc_conv_binary.argtypes = [_c_i8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i8p, ctypes.c_int,
                                      ctypes.c_int, _c_i64p]
        L.orc_conv_binary.restype = None
        L.orc_conv_binary_point.argtypes = [_c_i8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i8p, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int]
        L.orc_conv_binary_point.restype = ctypes.c_int64
        L.orc_conv_real.argtypes = [_c_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i8p, ctypes.c_int,
                                    ctypes.c_int, _c_f64p]
        L.orc_conv_real.restype = None
        L.orc_binarize_i64.argtypes = [_c_i64p, ctypes.c_int64, ctypes.c_int, _c_i32p, _c_u8p, _c_i8p]
        L.orc_binarize_i64.restype = None
        L.orc_binarize_f64.argtypes = [_c_f64p, ctypes.c_int64, ctypes.c_int, _c_i32p, _c_u8p, _c_i8p]
        L.orc_binarize_f64.restype = None
        L.orc_maxpool2.argtypes = [_c_i8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_i8p]
        L.orc_maxpool2.restype = None
        L.orc_dense.argtypes = [_c_i8p, ctypes.c_int64, _c_i8p, ctypes.c_int, _c_i64p]
        L.orc_dense.restype = None
        L.orc_argmax_i64.argtypes = [_c_i64p, ctypes.c_int]
        L.orc_argmax_i64.restype = ctypes.c_int
        L.orc_affine.argtypes = [_c_i64p, ctypes.c_int, _c_f32p, _c_f32p, _c_f64p, _c_f32p]
        L.orc_affine.restype = None
        L.orc_argmax_f32.argtypes = [_c_f32p, ctypes.c_int]
        L.orc_argmax_f32.restype = ctypes.c_int
        L.orc_forward.argtypes = [_c_f64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_f64p,
                                  ctypes.POINTER(OrcLayer), ctypes.c_int, _c_i64p, _c_i32p]
        L.orc_forward.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray | None, ct):
    if a is None:
        return ctypes.cast(None, ct)
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ct)


def _pm1(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int8)
    assert np.all((a == 1) | (a == -1)), "oracle takes +/-1 values"
    return a


# ---- Eq. (1), Eq. (2) -------------------------------------------------------------------------
def sign(x: float) -> int:
    """Eq. (1)."""
    return lib().orc_sign(float(x))


def pack(x, B: int = 32) -> np.ndarray:
    """Eq. (2), PAPER.md:186-195 (element i -> bit B-1-mod(i-1,B) of word ceil(i/B))."""
    x = _pm1(np.asarray(x).reshape(-1))
    nw = (x.size + B - 1) // B
    out = np.zeros(max(nw, 1), dtype=np.uint32)
    r = lib().orc_pack(_p(x, _c_i8p), x.size, B, _p(out, _c_u32p))
    if r < 0:
        raise ValueError("bad packing bitwidth B=%d" % B)
    return out[:nw]


def unpack(words, D: int, B: int = 32) -> np.ndarray:
    """Inverse of Eq. (2); raises on nonzero pad bits."""
    words = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1)
    out = np.zeros(max(D, 1), dtype=np.int8)
    r = lib().orc_unpack(_p(words, _c_u32p), D, B, _p(out, _c_i8p))
    if r == -2:
        raise ValueError("nonzero pad bits")
    if r != 0:
        raise ValueError("bad unpack arguments")
    return out[:D]


def pack_channels(x) -> np.ndarray:
    """Pack the last (channel) axis of a +/-1 tensor with B = 32 (Eq. 2 per pixel):
    [..., C] int8 -> [..., ceil(C/32)] uint32 (channel c -> word c//32, bit 31 - c%32)."""
    x = _pm1(x)
    lead = x.shape[:-1]
    C = x.shape[-1]
    cw = (C + 31) // 32
    flat = x.reshape(-1, C)
    out = np.zeros((flat.shape[0], cw), dtype=np.uint32)
    for i in range(flat.shape[0]):
        out[i] = pack(flat[i], 32)
    return out.reshape(*lead, cw)


def unpack_channels(words, C: int) -> np.ndarray:
    """Inverse of pack_channels: [..., ceil(C/32)] uint32 -> [..., C] int8 +/-1."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    lead = words.shape[:-1]
    flat = words.reshape(-1, words.shape[-1])
    out = np.zeros((flat.shape[0], C), dtype=np.int8)
    for i in range(flat.shape[0]):
        out[i] = unpack(flat[i], C, 32)
    return out.reshape(*lead, C)


def luma(r: int, g: int, b: int) -> int:
    return lib().orc_luma(int(r), int(g), int(b))


# ---- Section 2.3 input binarization -----------------------------------------------------------
def binarize_input(x, mode: int, T=None) -> np.ndarray:
    """Section 2.3 on ONE HWC image -> +/-1 int8 HWC'."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    h, w, c = x.shape
    cout = {SIGN: c, THRESH_RGB: c, THRESH_GRAY: 1, LBP: 3}[mode]
    out = np.zeros((h, w, cout), dtype=np.int8)
    Td = None if T is None else np.ascontiguousarray(np.asarray(T, dtype=np.float32).astype(np.float64))
    r = lib().orc_binarize_input(_p(x, _c_f64p), h, w, c, mode, _p(Td, _c_f64p), _p(out, _c_i8p))
    if r != cout:
        raise ValueError("bad binarize_input arguments")
    return out


# ---- Eq. (3) ---------------------------------------------------------------------------------
def conv_binary(x, wt) -> np.ndarray:
    """Eq. (3) on one +/-1 HWC map, -1 padding: x [h,w,cin], wt [cout,k,k,cin] -> int64 [h,w,cout]."""
    x, wt = _pm1(x), _pm1(wt)
    h, w, cin = x.shape
    cout, k, k2, cin2 = wt.shape
    assert k == k2 and cin == cin2 and k % 2 == 1
    acc = np.zeros((h, w, cout), dtype=np.int64)
    lib().orc_conv_binary(_p(x, _c_i8p), h, w, cin, _p(wt, _c_i8p), cout, k, _p(acc, _c_i64p))
    return acc


def conv_binary_point(x, wt_o, y: int, xx: int) -> int:
    """One output of Eq. (3): x [h,w,cin] +/-1, wt_o [k,k,cin] (one output channel)."""
    x, wt_o = _pm1(x), _pm1(wt_o)
    h, w, cin = x.shape
    k = wt_o.shape[0]
    return int(lib().orc_conv_binary_point(_p(x, _c_i8p), h, w, cin, _p(wt_o, _c_i8p), k, int(y), int(xx)))


def conv_real(x, wt) -> np.ndarray:
    """Eq. (3) on one real HWC image with zero padding -> float64 [h,w,cout]."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    wt = _pm1(wt)
    h, w, cin = x.shape
    cout, k, _, cin2 = wt.shape
    assert cin == cin2
    acc = np.zeros((h, w, cout), dtype=np.float64)
    lib().orc_conv_real(_p(x, _c_f64p), h, w, cin, _p(wt, _c_i8p), cout, k, _p(acc, _c_f64p))
    return acc


def binarize(acc, thr=None, flip=None) -> np.ndarray:
    """Eq. (1) per channel (last axis) with optional integer threshold / flip."""
    acc = np.asarray(acc)
    c = acc.shape[-1]
    out = np.zeros(acc.shape, dtype=np.int8)
    thr_a = None if thr is None else np.ascontiguousarray(thr, dtype=np.int32)
    flip_a = None if flip is None else np.ascontiguousarray(flip, dtype=np.uint8)
    if acc.dtype == np.float64 or acc.dtype == np.float32:
        a = np.ascontiguousarray(acc, dtype=np.float64)
        lib().orc_binarize_f64(_p(a, _c_f64p), a.size, c, _p(thr_a, _c_i32p), _p(flip_a, _c_u8p),
                               _p(out, _c_i8p))
    else:
        a = np.ascontiguousarray(acc, dtype=np.int64)
        lib().orc_binarize_i64(_p(a, _c_i64p), a.size, c, _p(thr_a, _c_i32p), _p(flip_a, _c_u8p),
                               _p(out, _c_i8p))
    return out


def maxpool2(x) -> np.ndarray:
    """2x2/2 max-pool of one +/-1 HWC map (Table 2)."""
    x = _pm1(x)
    h, w, c = x.shape
    y = np.zeros((h // 2, w // 2, c), dtype=np.int8)
    lib().orc_maxpool2(_p(x, _c_i8p), h, w, c, _p(y, _c_i8p))
    return y


def dense(x, W) -> np.ndarray:
    """Fully connected layer: x [d] +/-1, W [l, d] +/-1 -> int64 [l]."""
    x = _pm1(np.asarray(x).reshape(-1))
    W = _pm1(W)
    l, d = W.shape
    assert d == x.size
    acc = np.zeros(l, dtype=np.int64)
    lib().orc_dense(_p(x, _c_i8p), d, _p(W, _c_i8p), l, _p(acc, _c_i64p))
    return acc


def argmax(v) -> int:
    v = np.ascontiguousarray(v, dtype=np.int64)
    return lib().orc_argmax_i64(_p(v, _c_i64p), v.size)


def affine(acc, scale, bias):
    """Float output scaling of the last layer (f4: BinaryNet output BN folded / XNOR-Net alpha,
    PAPER.md:74): acc int [..., l] -> (score float64, score float32 with one rounding, class).
    The class is the first maximum of the fp32 scores (R19, R25)."""
    acc = np.ascontiguousarray(np.atleast_2d(acc), dtype=np.int64)
    scale = np.ascontiguousarray(scale, dtype=np.float32)
    bias = np.ascontiguousarray(bias, dtype=np.float32)
    n, l = acc.shape
    assert scale.shape == (l,) and bias.shape == (l,)
    s64 = np.zeros((n, l), dtype=np.float64)
    s32 = np.zeros((n, l), dtype=np.float32)
    cls = np.zeros(n, dtype=np.int32)
    for i in range(n):
        lib().orc_affine(_p(acc[i], _c_i64p), l, _p(scale, _c_f32p), _p(bias, _c_f32p), _p(s64[i], _c_f64p),
                         _p(s32[i], _c_f32p))
        cls[i] = lib().orc_argmax_f32(_p(s32[i], _c_f32p), l)
    return s64, s32, cls


# ---- whole network -----------------------------------------------------------------------------
class Net:
    """A network for the oracle: layers are dicts {kind: 'conv'|'dense', ...} with UNPACKED
    +/-1 weights (conv: [cout,k,k,cin] int8; dense: [l, d] int8, d in HWC flatten order)."""

    def __init__(self, h, w, c, mode, T, layers):
        self.h, self.w, self.c, self.mode = h, w, c, mode
        self.T = None if T is None else np.ascontiguousarray(np.asarray(T, np.float32).astype(np.float64))
        self._keep = []
        arr = (OrcLayer * len(layers))()
        for i, L in enumerate(layers):
            wt = _pm1(L["wt"])
            self._keep.append(wt)
            thr = None if L.get("thr") is None else np.ascontiguousarray(L["thr"], dtype=np.int32)
            flip = None if L.get("flip") is None else np.ascontiguousarray(L["flip"], dtype=np.uint8)
            self._keep += [thr, flip]
            if L["kind"] == "conv":
                arr[i] = OrcLayer(1, wt.shape[1], wt.shape[0], L.get("pool", 1), 0, _p(wt, _c_i8p),
                                  _p(thr, _c_i32p), _p(flip, _c_u8p))
            else:
                arr[i] = OrcLayer(2, 0, 0, 1, wt.shape[0], _p(wt, _c_i8p), _p(thr, _c_i32p), _p(flip, _c_u8p))
        self._arr = arr
        self.n_layers = len(layers)
        self.n_classes = layers[-1]["wt"].shape[0]

    def forward_one(self, img):
        """Oracle forward pass of ONE HWC image -> (int64 logits [L], class)."""
        x = np.ascontiguousarray(img, dtype=np.float64)
        logits = np.zeros(self.n_classes, dtype=np.int64)
        cls = ctypes.c_int32(0)
        r = lib().orc_forward(_p(x, _c_f64p), self.h, self.w, self.c, self.mode, _p(self.T, _c_f64p),
                              self._arr, self.n_layers, _p(logits, _c_i64p), ctypes.byref(cls))
        if r != 0:
            raise ValueError("oracle forward failed")
        return logits, cls.value

    def forward(self, images, threads: int = 1):
        """images [n,h,w,c] -> (int64 logits [n,L], int32 classes [n]); one image per thread."""
        n = images.shape[0]
        logits = np.zeros((n, self.n_classes), dtype=np.int64)
        cls = np.zeros(n, dtype=np.int32)

        def one(i):
            logits[i], cls[i] = self.forward_one(images[i])

        if threads <= 1:
            for i in range(n):
                one(i)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(one, range(n)))
        return logits, cls
