"""The C ABI (include/bnn.h) on CPU: the library builds, loads, exports every declared symbol, and
its argument validation rejects bad calls before any CUDA work (no GPU needed for these)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bnn.h")).read()
    return sorted(set(re.findall(r"BNN_API\s+[\w\s\*]*?\b(bnn_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_1808_00209_b200 import _build
    _build.build()
    import paper_1808_00209_b200 as b
    return b.lib()


def test_header_declares_the_five_entry_points():
    syms = declared_symbols()
    for s in ["bnn_pack", "bnn_conv2d", "bnn_maxpool", "bnn_dense", "bnn_forward", "bnn_net_create",
              "bnn_net_destroy", "bnn_last_error", "bnn_forward_host"]:
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_only_declared_symbols_are_exported():
    out = os.popen("nm -D --defined-only %s" % os.path.join(ROOT, "paper_1808_00209_b200", "libbnn.so")).read()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == set(declared_symbols())


def test_library_is_sm100a_only():
    out = os.popen("cuobjdump --list-elf %s 2>&1" % os.path.join(ROOT, "paper_1808_00209_b200", "libbnn.so")).read()
    assert "sm_100a" in out
    for other in ["sm_80", "sm_90", "sm_103"]:
        assert other + "." not in out and other + "a." not in out
    ptx = os.popen("cuobjdump --list-ptx %s 2>&1" % os.path.join(ROOT, "paper_1808_00209_b200", "libbnn.so")).read()
    assert ".ptx" not in ptx  # no JIT fallback


def test_version(L):
    assert L.bnn_version() == 101


def _err(L):
    return L.bnn_last_error().decode()


def test_validation_errors(L):
    import paper_1808_00209_b200 as b
    fake = 1 << 20  # never dereferenced: validation fails first
    # bnn_pack: negative size
    assert L.bnn_pack(fake, b.U8, -1, 2, 2, 3, b.SIGN, None, fake, None) == 1
    assert "bad sizes" in _err(L)
    # LBP needs u8 x 3 channels
    assert L.bnn_pack(fake, b.F32, 1, 2, 2, 3, b.LBP, None, fake, None) == 5
    # threshold mode without T
    assert L.bnn_pack(fake, b.U8, 1, 2, 2, 3, b.THRESH_RGB, None, fake, None) == 1
    # misaligned pointer
    assert L.bnn_pack(fake + 4, b.U8, 1, 2, 2, 3, b.SIGN, None, fake, None) == 4
    # conv: even k is unsupported
    assert L.bnn_conv2d(fake, b.BITS, 1, 4, 4, 32, fake, 32, 4, None, None, 1, fake, None, None) == 3
    # pool 2 on an odd map
    assert L.bnn_conv2d(fake, b.BITS, 1, 5, 4, 32, fake, 32, 3, None, None, 2, fake, None, None) == 2
    # real first layer with c_in > 32
    assert L.bnn_conv2d(fake, b.U8, 1, 4, 4, 33, fake, 32, 3, None, None, 1, fake, None, None) == 5
    # no outputs
    assert L.bnn_conv2d(fake, b.BITS, 1, 4, 4, 32, fake, 32, 3, None, None, 1, None, None, None) == 1
    # maxpool odd
    assert L.bnn_maxpool(fake, 1, 3, 4, 32, fake, None) == 2
    # dense: cls with l > 32 needs acc
    assert L.bnn_dense(fake, 2, 64, fake, 40, None, None, None, None, fake, None) == 1
    # net: last layer must be dense
    lay = (b.bnn._Layer * 1)(b.bnn._Layer(1, 3, 32, 1, 0, fake, None, None))
    out = ctypes.c_void_p()
    assert L.bnn_net_create(8, 8, 3, b.U8, b.SIGN, None, lay, 1, 16, ctypes.byref(out)) == 5
    assert out.value is None
    # mode NONE with f32 ok but bad max_batch
    assert L.bnn_net_create(8, 8, 3, b.U8, b.SIGN, None, lay, 1, 0, ctypes.byref(out)) == 1
    assert L.bnn_forward(None, fake, 1, fake, fake, None) == 1
    assert L.bnn_set_option(b"nope", 1) == 1
    # every knob the header documents is accepted (and restored to its default)
    hdr = open(os.path.join(ROOT, "include", "bnn.h")).read()
    doc = hdr[hdr.index("Process-wide tuning"):hdr.index("BNN_API int bnn_set_option")]
    keys = re.findall(r'\*\s+"(\w+)"', doc)
    assert {"conv_algo", "conv_tc", "conv_tc_fp4", "conv_pool_tc", "first_tma", "pdl"} <= set(keys)
    defaults = {"conv_algo": 0, "tiles_per_cta": 0, "gemv_max_n": 255, "fused_max_n": 12, "fused_cs": 0, "alg1": 0, "first_fp4": 1, "streams": 2, "csa": 1, "big_img": 1, "first_db": 1, "dense_ksplit": 1}
    for k in keys:
        if k == "first_exp":
            continue
        assert L.bnn_set_option(k.encode(), defaults.get(k, 1)) == 0, k
    # the production library has no knob that skips work: the timing-experiment key exists only in
    # the diagnostics build (libbnn_trace.so), and a trace buffer is refused
    assert "first_exp" in keys
    for v in (0, 1, 15):
        assert L.bnn_set_option(b"first_exp", v) == 1
    assert L.bnn_set_trace(ctypes.c_void_p(16), 16) == 3
    assert L.bnn_forward_launches(None, 5) == 0


def test_no_oracle_in_product_path():
    """The product package never imports, loads or links the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_1808_00209_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|bnn_oracle|orc_)", src), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_1808_00209_b200" not in src and "bnn.h" not in src.replace("include/bnn.h", "")
    libs = os.popen("ldd %s" % os.path.join(pkg, "libbnn.so")).read()
    assert "oracle" not in libs


def test_binding_validates_before_the_c_call():
    """The C ABI takes only pointers and n, so the binding checks shapes / dtypes / devices first
    (a wrong image size would otherwise be read out of bounds)."""
    import torch
    import paper_1808_00209_b200 as b
    net = object.__new__(b.Net)
    net.h, net.w, net.c, net.in_dtype, net.n_classes = 96, 96, 3, b.U8, 4
    with pytest.raises(ValueError):  # not a CUDA tensor
        net._check_images(torch.zeros((2, 96, 96, 3), dtype=torch.uint8))
    net._check_images(torch.zeros((2, 96, 96, 3), dtype=torch.uint8), host=True)
    with pytest.raises(ValueError):  # lower resolution
        net._check_images(torch.zeros((2, 48, 48, 3), dtype=torch.uint8), host=True)
    with pytest.raises(TypeError):  # f32 pixels for a u8 net
        net._check_images(torch.zeros((2, 96, 96, 3), dtype=torch.float32), host=True)
    with pytest.raises(ValueError):  # logits of the wrong width
        net._check_out(2, torch.zeros((2, 5), dtype=torch.int32), None, host=True)
    with pytest.raises(ValueError):  # weights must be device tensors: nothing reaches bnn_net_create
        b.Net(8, 8, 3, b.U8, b.SIGN, None, [dict(kind="conv", k=3, c_out=32, pool=2, wt=torch.zeros((32, 3, 3, 1),
                                                                                                   dtype=torch.int32))])
