"""paper_1808_00209_b200 -- B200 (sm_100a) bit-packed XNOR-popcount forward pass of the binarized
CNN of Khan, Huttunen, Boutellier (arXiv 1808.00209).

The compute lives in libbnn.so (hand-written CUDA for sm_100a behind the C ABI include/bnn.h);
`bnn` is a thin ctypes binding with the same names.  There is NO CPU fallback: importing the
binding on a machine without the built library raises, and every call fails loudly on error.
"""
from .bnn import (BITS, U8, F32, I32, I8, SIGN, THRESH_RGB, THRESH_GRAY, LBP, MODE_NONE, BnnError, Net,  # noqa: F401
                  affine, conv2d, dense, forward_launches, lib, lib_path, maxpool, pack, pack_weights, set_option, set_trace)

__all__ = ["BITS", "U8", "F32", "I32", "I8", "SIGN", "THRESH_RGB", "THRESH_GRAY", "LBP", "MODE_NONE", "BnnError",
           "Net", "affine", "conv2d", "dense", "forward_launches", "lib", "lib_path", "maxpool", "pack", "pack_weights",
           "set_option", "set_trace"]
