"""ctypes binding of libbnn.so (include/bnn.h) -- argument marshalling only.

Every function here has the name of the C entry point it calls and does nothing but turn
torch tensors into pointers / sizes and raise BnnError on a non-OK status.  PyTorch is used
for device memory and streams (tensor.data_ptr(), torch.cuda.current_stream()).  There is no
Python or CPU implementation of any step of the method in this module.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _build

BITS, U8, F32, I32, I8 = 0, 1, 2, 3, 4
SIGN, THRESH_RGB, THRESH_GRAY, LBP, MODE_NONE = 0, 1, 2, 3, -1

_DTYPES = {torch.uint8: U8, torch.float32: F32, torch.int32: I32, torch.int8: I8}
_STATUS = {0: "BNN_OK", 1: "BNN_E_ARG", 2: "BNN_E_SHAPE", 3: "BNN_E_UNSUPPORTED", 4: "BNN_E_ALIGN",
           5: "BNN_E_CONFIG", 6: "BNN_E_PADBITS", 7: "BNN_E_CUDA", 8: "BNN_E_NOMEM"}


class BnnError(RuntimeError):
    def __init__(self, status: int, func: str, msg: str):
        super().__init__("%s -> %s: %s" % (func, _STATUS.get(status, status), msg))
        self.status = status


class _Layer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("k", ctypes.c_int), ("c_out", ctypes.c_int), ("pool", ctypes.c_int),
                ("l", ctypes.c_int), ("wt", ctypes.c_void_p), ("thr", ctypes.c_void_p), ("flip", ctypes.c_void_p)]


_lib = None


def lib_path() -> str:
    # BNN_TRACE_LIB=1 selects the diagnostics build (tools/trace_first.py); same kernels + role timestamps
    return _build.TRACE_LIB if os.environ.get("BNN_TRACE_LIB") == "1" else _build.LIB


def lib():
    """Load libbnn.so (in-tree).  Raises if it has not been built: there is no fallback."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError("libbnn.so is not built (%s); run `python -m paper_1808_00209_b200._build` -- "
                               "there is no CPU fallback" % path)
        L = ctypes.CDLL(path)
        vp, i, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        L.bnn_last_error.restype = ctypes.c_char_p
        L.bnn_version.restype = i
        L.bnn_set_option.argtypes = [ctypes.c_char_p, i]
        L.bnn_set_trace.argtypes = [vp, i]
        L.bnn_set_trace.restype = i
        L.bnn_set_option.restype = i
        L.bnn_pack.argtypes = [vp, i, i, i, i, i, i, vp, vp, vp]
        L.bnn_pack.restype = i
        L.bnn_conv2d.argtypes = [vp, i, i, i, i, i, vp, i, i, vp, vp, i, vp, vp, vp]
        L.bnn_conv2d.restype = i
        L.bnn_maxpool.argtypes = [vp, i, i, i, i, vp, vp]
        L.bnn_maxpool.restype = i
        L.bnn_dense.argtypes = [vp, i, i64, vp, i, vp, vp, vp, vp, vp, vp]
        L.bnn_dense.restype = i
        L.bnn_affine.argtypes = [vp, i, i, vp, vp, vp, vp, vp]
        L.bnn_affine.restype = i
        L.bnn_forward_scores.argtypes = [vp, vp, i, vp, vp, vp, vp, vp, vp]
        L.bnn_forward_scores.restype = i
        L.bnn_net_create.argtypes = [i, i, i, i, i, vp, ctypes.POINTER(_Layer), i, i, ctypes.POINTER(vp)]
        L.bnn_net_create.restype = i
        L.bnn_forward.argtypes = [vp, vp, i, vp, vp, vp]
        L.bnn_forward.restype = i
        L.bnn_forward_host.argtypes = [vp, vp, i, vp, vp, vp]
        L.bnn_forward_host.restype = i
        L.bnn_forward_launches.argtypes = [vp, i]
        L.bnn_forward_launches.restype = i
        L.bnn_net_staging.argtypes = [vp, i, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.bnn_net_staging.restype = i
        L.bnn_forward_staged.argtypes = [vp, i, vp]
        L.bnn_forward_staged.restype = i
        L.bnn_net_layer_kernel.argtypes = [vp, i, i]
        L.bnn_net_layer_kernel.restype = ctypes.c_char_p
        L.bnn_net_profile.argtypes = [vp, i]
        L.bnn_net_profile.restype = i
        L.bnn_net_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), i]
        L.bnn_net_profile_read.restype = i
        L.bnn_net_destroy.argtypes = [vp]
        L.bnn_net_destroy.restype = None
        _lib = L
    return _lib


def _check(status: int, func: str):
    if status != 0:
        raise BnnError(status, func, lib().bnn_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    return t.data_ptr()


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError("%s must be a CUDA tensor (libbnn takes device pointers)" % name)
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)


def _dev_typed(t: torch.Tensor | None, name: str, dtypes, numel: int | None = None):
    """t is None, or a contiguous CUDA tensor of one of `dtypes` (and `numel` elements if given)."""
    if t is None:
        return
    _dev(t, name)
    if t.dtype not in dtypes:
        raise TypeError("%s must be %s, got %s" % (name, " / ".join(str(d) for d in dtypes), t.dtype))
    if numel is not None and t.numel() != numel:
        raise ValueError("%s must have %d elements, got %d" % (name, numel, t.numel()))


_WORDS = (torch.int32, torch.uint32) if hasattr(torch, "uint32") else (torch.int32,)
_IN_TORCH = {U8: torch.uint8, F32: torch.float32}


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def set_option(key: str, value: int):
    _check(lib().bnn_set_option(key.encode(), int(value)), "bnn_set_option")


def set_trace(buf: torch.Tensor | None):
    """bnn_set_trace: register an int64 CUDA tensor as the role-timestamp trace buffer (None disables)."""
    if buf is None:
        _check(lib().bnn_set_trace(None, 0), "bnn_set_trace")
    else:
        _dev(buf, "trace")
        _check(lib().bnn_set_trace(_ptr(buf), buf.numel()), "bnn_set_trace")


def pack(x: torch.Tensor, mode: int = SIGN, T: torch.Tensor | None = None, out: torch.Tensor | None = None,
         stream=None) -> torch.Tensor:
    """bnn_pack: x [n, h, w, c] (u8 / i8 / f32 / i32, CUDA) -> int32-viewed packed words
    [n, h, w, ceil(c_out/32)] (c_out = c, 1 for GRAY, 3 for LBP)."""
    _dev(x, "x")
    n, h, w, c = x.shape
    c_out = {THRESH_GRAY: 1, LBP: 3}.get(mode, c)
    if out is None:
        out = torch.empty((n, h, w, (c_out + 31) // 32), dtype=torch.int32, device=x.device)
    if T is not None:
        _dev(T, "T")
    _check(lib().bnn_pack(_ptr(x), _DTYPES[x.dtype], n, h, w, c, mode, _ptr(T), _ptr(out), _stream(stream)),
           "bnn_pack")
    return out


def pack_weights(wt: torch.Tensor, stream=None) -> torch.Tensor:
    """Packs +/-1 weights with bnn_pack(SIGN): conv [c_out, k, k, c_in] -> [c_out, k, k, cw];
    dense [l, d] -> [l, dw]."""
    if wt.dim() == 4:
        return pack(wt.contiguous(), SIGN, stream=stream)
    l, d = wt.shape
    return pack(wt.contiguous().view(l, 1, 1, d), SIGN, stream=stream).view(l, -1)


def conv2d(x: torch.Tensor, x_dt: int, c_in: int, wt: torch.Tensor, c_out: int, k: int, thr=None, flip=None,
           pool: int = 1, want_y: bool = True, want_acc: bool = False, stream=None):
    """bnn_conv2d.  x: packed [n,h,w,cw] (x_dt=BITS) or real [n,h,w,c_in] (U8/F32).
    Returns (y packed [n,h/pool,w/pool,cwo] or None, acc [n,h,w,c_out] or None)."""
    _dev(x, "x")
    _dev(wt, "wt")
    n, h, w = x.shape[0], x.shape[1], x.shape[2]
    y = torch.empty((n, h // pool, w // pool, (c_out + 31) // 32), dtype=torch.int32, device=x.device) if want_y else None
    acc = None
    if want_acc:
        acc = torch.empty((n, h, w, c_out), dtype=torch.float32 if x_dt == F32 else torch.int32, device=x.device)
    _check(lib().bnn_conv2d(_ptr(x), x_dt, n, h, w, c_in, _ptr(wt), c_out, k, _ptr(thr), _ptr(flip), pool,
                            _ptr(y), _ptr(acc), _stream(stream)), "bnn_conv2d")
    return y, acc


def maxpool(x: torch.Tensor, c: int, stream=None) -> torch.Tensor:
    """bnn_maxpool: packed [n, h, w, cw] -> packed [n, h/2, w/2, cw]."""
    _dev(x, "x")
    n, h, w, cw = x.shape
    y = torch.empty((n, h // 2, w // 2, cw), dtype=torch.int32, device=x.device)
    _check(lib().bnn_maxpool(_ptr(x), n, h, w, c, _ptr(y), _stream(stream)), "bnn_maxpool")
    return y


def dense(x: torch.Tensor, d: int, wt: torch.Tensor, l: int, thr=None, flip=None, want_y=True, want_acc=False,
          want_cls=False, stream=None):
    """bnn_dense: x packed [n, dw] -> (y packed [n, lw] | None, acc int32 [n, l] | None, cls int32 [n] | None)."""
    _dev(x, "x")
    _dev(wt, "wt")
    n = x.shape[0]
    y = torch.empty((n, (l + 31) // 32), dtype=torch.int32, device=x.device) if want_y else None
    acc = torch.empty((n, l), dtype=torch.int32, device=x.device) if want_acc else None
    cls = torch.empty((n,), dtype=torch.int32, device=x.device) if want_cls else None
    _check(lib().bnn_dense(_ptr(x), n, d, _ptr(wt), l, _ptr(thr), _ptr(flip), _ptr(y), _ptr(acc), _ptr(cls),
                           _stream(stream)), "bnn_dense")
    return y, acc, cls


def affine(acc: torch.Tensor, scale: torch.Tensor, bias: torch.Tensor, want_score=True, want_cls=True, stream=None):
    """bnn_affine: int32 logits [n, l] -> (fp32 scores [n, l] | None, int32 cls [n] | None)."""
    for t, nm in ((acc, "acc"), (scale, "scale"), (bias, "bias")):
        _dev(t, nm)
    n, l = acc.shape
    score = torch.empty((n, l), dtype=torch.float32, device=acc.device) if want_score else None
    cls = torch.empty((n,), dtype=torch.int32, device=acc.device) if want_cls else None
    _check(lib().bnn_affine(_ptr(acc), n, l, _ptr(scale), _ptr(bias), _ptr(score), _ptr(cls), _stream(stream)),
           "bnn_affine")
    return score, cls


class _DeviceBuffer:
    """A library-owned device buffer exposed through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _alias(ptr: int, shape, typestr: str, device) -> torch.Tensor:
    return torch.as_tensor(_DeviceBuffer(ptr, shape, typestr), device=device)


def forward_launches(net: "Net", n: int) -> int:
    return lib().bnn_forward_launches(net.handle, n)


class Net:
    """bnn_net: the whole forward pass.  `layers` are dicts like synth.VEHICLE['layers'] with
    PACKED device weights under 'wt' (see pack_weights) and optional 'thr' / 'flip' device tensors."""

    def __init__(self, h: int, w: int, c: int, in_dtype: int, mode: int, T: torch.Tensor | None, layers,
                 max_batch: int = 8192):
        arr = (_Layer * len(layers))()
        self._keep = [T]
        if in_dtype not in _IN_TORCH:
            raise ValueError("in_dtype must be U8 or F32")
        if mode == THRESH_RGB:
            _dev_typed(T, "T", (torch.float32,), c)
        elif mode == THRESH_GRAY:
            _dev_typed(T, "T", (torch.float32,), 1)
        for i, L in enumerate(layers):
            _dev_typed(L["wt"], "layers[%d].wt" % i, _WORDS)
            n_out = L["c_out"] if L["kind"] == "conv" else L["l"]
            _dev_typed(L.get("thr"), "layers[%d].thr" % i, (torch.int32,), n_out)
            _dev_typed(L.get("flip"), "layers[%d].flip" % i, (torch.uint8,), n_out)
            self._keep += [L["wt"], L.get("thr"), L.get("flip")]
            if L["kind"] == "conv":
                arr[i] = _Layer(1, L["k"], L["c_out"], L.get("pool", 1), 0, _ptr(L["wt"]), _ptr(L.get("thr")),
                                _ptr(L.get("flip")))
            else:
                arr[i] = _Layer(2, 0, 0, 1, L["l"], _ptr(L["wt"]), _ptr(L.get("thr")), _ptr(L.get("flip")))
        h_ = ctypes.c_void_p()
        _check(lib().bnn_net_create(h, w, c, in_dtype, mode, _ptr(T), arr, len(layers), max_batch, ctypes.byref(h_)),
               "bnn_net_create")
        self.handle = h_
        self._n_layers = len(layers)
        self.h, self.w, self.c, self.in_dtype = h, w, c, in_dtype
        self.n_classes = layers[-1]["l"]
        self.device = layers[0]["wt"].device

    def _check_images(self, images: torch.Tensor, host: bool = False):
        """The C ABI receives only a pointer and n: the shape and dtype are checked here."""
        if host:
            if images.is_cuda or not images.is_contiguous():
                raise ValueError("forward_host takes a contiguous CPU tensor (pinned for full speed)")
        else:
            _dev(images, "images")
        if images.dim() != 4 or tuple(images.shape[1:]) != (self.h, self.w, self.c):
            raise ValueError("images must be [n, %d, %d, %d], got %s" % (self.h, self.w, self.c, tuple(images.shape)))
        if images.dtype != _IN_TORCH[self.in_dtype]:
            raise TypeError("images must be %s for this net, got %s" % (_IN_TORCH[self.in_dtype], images.dtype))

    def _check_out(self, n: int, logits, cls, host: bool = False):
        for t, nm, shape in ((logits, "logits", (n, self.n_classes)), (cls, "cls", (n,))):
            if t is None:
                continue
            if host:
                if t.is_cuda or not t.is_contiguous():
                    raise ValueError("%s must be a contiguous CPU tensor" % nm)
            else:
                _dev(t, nm)
            if t.dtype != torch.int32 or tuple(t.shape) != shape:
                raise ValueError("%s must be int32 %s, got %s %s" % (nm, shape, t.dtype, tuple(t.shape)))

    def forward(self, images: torch.Tensor, logits: torch.Tensor | None = None, cls: torch.Tensor | None = None,
                stream=None):
        """bnn_forward: images [n,h,w,c] (CUDA) -> (int32 logits [n, L], int32 cls [n])."""
        self._check_images(images)
        n = images.shape[0]
        self._check_out(n, logits, cls)
        if logits is None:
            logits = torch.empty((n, self.n_classes), dtype=torch.int32, device=images.device)
        if cls is None:
            cls = torch.empty((n,), dtype=torch.int32, device=images.device)
        _check(lib().bnn_forward(self.handle, _ptr(images), n, _ptr(logits), _ptr(cls), _stream(stream)),
               "bnn_forward")
        return logits, cls

    def forward_scores(self, images: torch.Tensor, scale: torch.Tensor, bias: torch.Tensor, stream=None):
        """bnn_forward_scores: images -> (int32 logits [n, L], fp32 scores [n, L], int32 cls [n])."""
        self._check_images(images)
        _dev_typed(scale, "scale", (torch.float32,), self.n_classes)
        _dev_typed(bias, "bias", (torch.float32,), self.n_classes)
        n = images.shape[0]
        logits = torch.empty((n, self.n_classes), dtype=torch.int32, device=images.device)
        scores = torch.empty((n, self.n_classes), dtype=torch.float32, device=images.device)
        cls = torch.empty((n,), dtype=torch.int32, device=images.device)
        _check(lib().bnn_forward_scores(self.handle, _ptr(images), n, _ptr(scale), _ptr(bias), _ptr(logits),
                                        _ptr(scores), _ptr(cls), _stream(stream)), "bnn_forward_scores")
        return logits, scores, cls

    def forward_host(self, images: torch.Tensor, logits: torch.Tensor | None = None, cls: torch.Tensor | None = None,
                     stream=None):
        """bnn_forward_host: HOST images (pinned CPU tensor) -> HOST (logits, cls); synchronous."""
        self._check_images(images, host=True)
        n = images.shape[0]
        self._check_out(n, logits, cls, host=True)
        if logits is None:
            logits = torch.empty((n, self.n_classes), dtype=torch.int32, pin_memory=True)
        if cls is None:
            cls = torch.empty((n,), dtype=torch.int32, pin_memory=True)
        _check(lib().bnn_forward_host(self.handle, _ptr(images), n, _ptr(logits), _ptr(cls), _stream(stream)),
               "bnn_forward_host")
        return logits, cls

    def staging(self, max_staged: int):
        """bnn_net_staging: the net's device staging buffers as torch tensors (aliases, no copy):
        (images [m, h, w, c], logits int32 [m, L], cls int32 [m])."""
        pin, plog, pcls = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().bnn_net_staging(self.handle, max_staged, ctypes.byref(pin), ctypes.byref(plog),
                                     ctypes.byref(pcls)), "bnn_net_staging")
        itype = "|u1" if self.in_dtype == U8 else "<f4"
        dev = self.device
        return (_alias(pin.value, (max_staged, self.h, self.w, self.c), itype, dev),
                _alias(plog.value, (max_staged, self.n_classes), "<i4", dev),
                _alias(pcls.value, (max_staged,), "<i4", dev))

    def forward_staged(self, n: int, stream=None):
        """bnn_forward_staged: graph-replayed forward of the first n staged images."""
        _check(lib().bnn_forward_staged(self.handle, n, _stream(stream)), "bnn_forward_staged")

    def layer_kernel(self, layer: int, n: int) -> str:
        """bnn_net_layer_kernel: the kernel family layer `layer` runs on for a batch of n."""
        return lib().bnn_net_layer_kernel(self.handle, layer, n).decode()

    def profile(self, enable: bool = True) -> int:
        """bnn_net_profile: reset and start (or stop) per-stage event timing."""
        r = lib().bnn_net_profile(self.handle, 1 if enable else 0)
        if r < 0:
            _check(-r, "bnn_net_profile")
        return r

    def profile_read(self):
        """bnn_net_profile_read -> (ms per stage, launches per stage); stage 0 = pack,
        i + 1 = layer i, last = argmax."""
        ns = self.profile_read_count()
        ms = (ctypes.c_double * ns)()
        cnt = (ctypes.c_int64 * ns)()
        r = lib().bnn_net_profile_read(self.handle, ms, cnt, ns)
        if r < 0:
            _check(-r, "bnn_net_profile_read")
        return list(ms), list(cnt)

    def profile_read_count(self) -> int:
        return self._n_layers + 2

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().bnn_net_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
