"""fp32 3x3 stride-1 C->C convolutions on the library's own kernels
(``csrc/conv_f32.cu``) — the CNN forward/backward of SURVEY §8 a6 in fp32.

``Conv3x3`` is an ``nn.Conv2d`` (same parameters, init and state-dict
names) whose forward runs ``lpp_conv3x3_f32`` / ``lpp_conv3x3_wgrad_f32``
when the activation is fp32 on a CUDA device and the (channels, size) pair
has a kernel — CIFAR ResNet-20's 16 stride-1 3x3 convolutions — and is
cuDNN's ``F.conv2d`` otherwise (bf16 compute or autocast, other shapes).  The kernels
take NHWC activations (torch channels_last) and OHWI weights (the arena's
channels_last view, ``objectives.py`` ``_view``), so no layout change runs
around them.  Launches go to torch's current stream: they are captured into
the step graphs like cuDNN's.
"""

from __future__ import annotations

import os

import torch
import torch.nn as nn
import torch.nn.functional as F

_CL = torch.channels_last


def enabled() -> bool:
    """``LPP_CONV=cudnn`` routes every convolution to cuDNN (A/B runs)."""
    return os.environ.get("LPP_CONV", "native") != "cudnn"


def _lib():
    from . import _native

    return _native


def supported(c_in: int, c_out: int, hw: int, stride: int, k: int) -> bool:
    N = _lib()
    return k == 3 and stride == 1 and c_in == c_out and bool(N.lib.lpp_conv3x3_supported(c_in, hw))


def _ohwi(w: torch.Tensor) -> torch.Tensor:
    """w [co, ci, 3, 3] whose memory is OHWI (a channels_last view)."""
    if w.is_contiguous(memory_format=_CL):
        return w
    return w.contiguous(memory_format=_CL)


def conv_fwd(x: torch.Tensor, w: torch.Tensor, dgrad: bool = False) -> torch.Tensor:
    N = _lib()
    n, c, h, _ = x.shape
    x = x.contiguous(memory_format=_CL)
    w = _ohwi(w)
    y = torch.empty_like(x, memory_format=_CL)
    N.check(N.lib.lpp_conv3x3_f32(x.data_ptr(), w.data_ptr(), y.data_ptr(), n, c, h, int(dgrad),
                                  torch.cuda.current_stream(x.device).cuda_stream), "conv3x3_f32")
    return y


def conv_wgrad(x: torch.Tensor, dy: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    N = _lib()
    n, c, h, _ = x.shape
    x = x.contiguous(memory_format=_CL)
    dy = dy.contiguous(memory_format=_CL)
    dw = torch.empty_like(like, memory_format=_CL)
    nbytes = int(N.lib.lpp_conv3x3_wgrad_workspace(n, c, h))
    ws = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device)
    N.check(N.lib.lpp_conv3x3_wgrad_f32(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), nbytes,
                                        n, c, h, torch.cuda.current_stream(x.device).cuda_stream),
            "conv3x3_wgrad_f32")
    return dw


class _Conv3x3Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w):
        ctx.save_for_backward(x, w)
        return conv_fwd(x, w)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        gx = conv_fwd(gy, w, dgrad=True) if ctx.needs_input_grad[0] else None
        gw = conv_wgrad(x, gy, w) if ctx.needs_input_grad[1] else None
        return gx, gw


def conv3x3(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """y = conv2d(x, w, stride 1, padding 1) on the library's kernels."""
    return _Conv3x3Fn.apply(x, w)


class Conv3x3(nn.Conv2d):
    """nn.Conv2d(cin, cout, 3, stride, 1, bias=False) with the native fp32
    path for the shapes that have a kernel."""

    def __init__(self, cin: int, cout: int, stride: int = 1):
        super().__init__(cin, cout, 3, stride, 1, bias=False)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if (x.dtype == torch.float32 and x.is_cuda and self.weight.dtype == torch.float32
                and not torch.is_autocast_enabled("cuda") and x.shape[2] == x.shape[3] and enabled()
                and supported(self.in_channels, self.out_channels, x.shape[2], self.stride[0], 3)):
            return conv3x3(x, self.weight)
        return F.conv2d(x, self.weight, None, self.stride, self.padding)
