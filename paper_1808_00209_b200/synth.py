"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no sign, packing, convolution, popcount):
it only draws random numbers and describes layer shapes.  Both sides consume its output:
the oracle takes the unpacked +/-1 int8 tensors and u8 images as they are, the CUDA path
packs them itself with bnn_pack on the device.

Input recipe:
  * images: u8 NHWC, i.i.d. uniform over [0, 255] ("randomly generated");
  * weights: i.i.d. +/-1 with p = 1/2 (the configs say "random +/-1 weights");
  * thresholds T_c ~ U(-160, -96) so that about half of the input bits are set; integer
    T (e.g. -128) in parity runs so that X + T = 0 ties occur;
  * multi-GPU: images are drawn per fixed 4096-image chunk with seed base + chunk id, so
    the data is identical for every GPU count.
"""
from __future__ import annotations

import numpy as np
import torch

CHUNK = 4096


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def images(n: int, h: int, w: int, c: int, seed: int, device="cpu") -> torch.Tensor:
    """u8 [n, h, w, c], uniform bytes."""
    return torch.randint(0, 256, (n, h, w, c), generator=_gen(seed, device), dtype=torch.uint8, device=device)


def images_chunked(start: int, n: int, h: int, w: int, c: int, seed: int, device="cpu") -> torch.Tensor:
    """Images [start, start+n) of an infinite seeded stream drawn in CHUNK-image chunks
    (chunk j uses seed + 1000003 * (j + 1)); any shard of it is identical for any GPU count."""
    out = torch.empty((n, h, w, c), dtype=torch.uint8, device=device)
    i = start
    while i < start + n:
        j = i // CHUNK
        lo, hi = j * CHUNK, (j + 1) * CHUNK
        chunk = images(CHUNK, h, w, c, seed + 1000003 * (j + 1), device)
        a, b = max(lo, i), min(hi, start + n)
        out[a - start:b - start] = chunk[a - lo:b - lo]
        i = b
    return out


def pm1(shape, seed: int, device="cpu") -> torch.Tensor:
    """int8 tensor of i.i.d. +/-1 (p = 1/2)."""
    b = torch.randint(0, 2, tuple(shape), generator=_gen(seed, device), dtype=torch.int8, device=device)
    return b * 2 - 1


def words(shape, seed: int, device="cpu") -> torch.Tensor:
    """int32 tensor of uniform random 32-bit words (every bit valid: use with c % 32 == 0)."""
    return torch.randint(-(2 ** 31), 2 ** 31, tuple(shape), generator=_gen(seed, device), dtype=torch.int32,
                         device=device)


def thresholds(c: int, seed: int, lo: float = -160.0, hi: float = -96.0) -> torch.Tensor:
    """float32 [c] uniform in [lo, hi)."""
    g = _gen(seed, "cpu")
    return (torch.rand(c, generator=g, dtype=torch.float64) * (hi - lo) + lo).to(torch.float32)


def int_thresholds(c: int, seed: int, lo: int = -8, hi: int = 9) -> torch.Tensor:
    """int32 [c] uniform integers in [lo, hi) (batch-norm-folded integer thresholds)."""
    return torch.randint(lo, hi, (c,), generator=_gen(seed, "cpu"), dtype=torch.int32)


def flips(c: int, seed: int) -> torch.Tensor:
    return torch.randint(0, 2, (c,), generator=_gen(seed, "cpu"), dtype=torch.uint8)


# ------------------------------------------------------------------------ network shapes
# Vehicle classifier, Table 2: conv 32x5x5 (same) -> 2x2 pool -> conv
# 32x5x5 -> 2x2 pool -> FC 100 over 24x24x32 -> FC2, FC3 (sizes unstated: reading R10 =
# 100 -> 100 -> 4 classes).
VEHICLE = dict(h=96, w=96, c=3, layers=[
    dict(kind="conv", k=5, c_out=32, pool=2),
    dict(kind="conv", k=5, c_out=32, pool=2),
    dict(kind="dense", l=100),
    dict(kind="dense", l=100),
    dict(kind="dense", l=4),
])

# CIFAR-10-shaped BinaryNet VGG (reading R22): 2x128C3-MP2-2x256C3-MP2-2x512C3-MP2-1024FC-1024FC-10FC.
CIFAR = dict(h=32, w=32, c=3, layers=[
    dict(kind="conv", k=3, c_out=128, pool=1),
    dict(kind="conv", k=3, c_out=128, pool=2),
    dict(kind="conv", k=3, c_out=256, pool=1),
    dict(kind="conv", k=3, c_out=256, pool=2),
    dict(kind="conv", k=3, c_out=512, pool=1),
    dict(kind="conv", k=3, c_out=512, pool=2),
    dict(kind="dense", l=1024),
    dict(kind="dense", l=1024),
    dict(kind="dense", l=10),
])


def input_channels(c: int, mode: int) -> int:
    """Channels the first layer sees: GRAY -> 1, LBP -> 3, otherwise c (mode ids as bnn.h)."""
    return {2: 1, 3: 3}.get(mode, c)


def make_weights(spec: dict, mode: int, seed: int, device="cpu", small_layers=None):
    """+/-1 int8 weights for every layer of `spec` (conv [c_out, k, k, c_in], dense [l, d]).
    Layer i uses seed + 7919 * (i + 1).  Returns a list of dicts (the spec's layers + 'wt')."""
    layers = small_layers if small_layers is not None else spec["layers"]
    h, w, c = spec["h"], spec["w"], input_channels(spec["c"], mode)
    d = None
    out = []
    for i, L in enumerate(layers):
        s = seed + 7919 * (i + 1)
        L = dict(L)
        if L["kind"] == "conv":
            L["wt"] = pm1((L["c_out"], L["k"], L["k"], c), s, device)
            c = L["c_out"]
            h //= L.get("pool", 1)
            w //= L.get("pool", 1)
        else:
            if d is None:
                d = h * w * c
            L["wt"] = pm1((L["l"], d), s, device)
            d = L["l"]
        out.append(L)
    return out


def numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
