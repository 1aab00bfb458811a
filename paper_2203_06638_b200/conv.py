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


ARRIVALS = 8   # LPP_CONV_ARRIVALS


def arrival_cells(device) -> torch.Tensor:
    """Zeroed counters for lpp_conv3x3_wgrad_f32 (every call leaves them
    zero; calls sharing a set must be stream-ordered)."""
    return torch.zeros(ARRIVALS, dtype=torch.int32, device=device)


def conv_wgrad(x: torch.Tensor, dy: torch.Tensor, like: torch.Tensor,
               arrivals: torch.Tensor | None = None) -> torch.Tensor:
    N = _lib()
    n, c, h, _ = x.shape
    x = x.contiguous(memory_format=_CL)
    dy = dy.contiguous(memory_format=_CL)
    dw = torch.empty_like(like, memory_format=_CL)
    nbytes = int(N.lib.lpp_conv3x3_wgrad_workspace(n, c, h))
    ws = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device)
    if arrivals is None:
        arrivals = arrival_cells(x.device)
    N.check(N.lib.lpp_conv3x3_wgrad_f32(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), nbytes,
                                        arrivals.data_ptr(), n, c, h,
                                        torch.cuda.current_stream(x.device).cuda_stream),
            "conv3x3_wgrad_f32")
    return dw


def _will_run(node) -> bool:
    """Whether the current backward pass executes ``node`` (a non-leaf
    autograd node): the input gradient of a block's input-most layer is not
    needed under partial backprop."""
    if node is None:
        return False
    try:
        return bool(torch._C._will_engine_execute_node(node))
    except RuntimeError:
        return True


def _strided(kind: str, x: torch.Tensor, w: torch.Tensor, mode: int, other: torch.Tensor | None,
             arrivals: torch.Tensor | None) -> torch.Tensor:
    """The stride-2 kernels (kind "1x1" or "3x3s2"): mode 0 y = conv(x, w);
    1 dX of dY = x; 2 dW of (x, dY = other)."""
    N = _lib()
    fn = N.lib.lpp_conv1x1s2_f32 if kind == "1x1" else N.lib.lpp_conv3x3s2_f32
    wsq = N.lib.lpp_conv1x1s2_wgrad_workspace if kind == "1x1" else N.lib.lpp_conv3x3s2_wgrad_workspace
    co, ci = w.shape[0], w.shape[1]
    x = x.contiguous(memory_format=_CL)
    w = _ohwi(w)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    what = f"conv{kind}_f32"
    if mode == 0:
        n, _, hw, _ = x.shape
        out = torch.empty((n, co, hw // 2, hw // 2), device=x.device, memory_format=_CL)
        N.check(fn(x.data_ptr(), w.data_ptr(), out.data_ptr(), n, ci, co, hw, 0, None, 0, None, stream), what)
    elif mode == 1:
        n, _, ho, _ = x.shape
        out = torch.empty((n, ci, 2 * ho, 2 * ho), device=x.device, memory_format=_CL)
        N.check(fn(x.data_ptr(), w.data_ptr(), out.data_ptr(), n, ci, co, 2 * ho, 1, None, 0, None, stream), what)
    else:
        n, _, hw, _ = x.shape
        dy = other.contiguous(memory_format=_CL)
        out = torch.empty_like(w, memory_format=_CL)
        nbytes = int(wsq(n, ci, co, hw))
        ws = torch.empty(max(nbytes // 4, 1), dtype=torch.float32, device=x.device)
        if arrivals is None:
            arrivals = arrival_cells(x.device)
        N.check(fn(x.data_ptr(), dy.data_ptr(), out.data_ptr(), n, ci, co, hw, 2, ws.data_ptr(), nbytes,
                   arrivals.data_ptr(), stream), what)
    return out


def conv1x1s2(x: torch.Tensor, w: torch.Tensor, mode: int, other: torch.Tensor | None = None,
              arrivals: torch.Tensor | None = None) -> torch.Tensor:
    """The projection shortcut's kernels (1x1, stride 2)."""
    return _strided("1x1", x, w, mode, other, arrivals)


def conv3x3s2(x: torch.Tensor, w: torch.Tensor, mode: int, other: torch.Tensor | None = None,
              arrivals: torch.Tensor | None = None) -> torch.Tensor:
    """The stage-opening 3x3 stride-2 convolution's kernels."""
    return _strided("3x3s2", x, w, mode, other, arrivals)


class _StridedFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, arrivals, want_w, kind):
        ctx.save_for_backward(x, w)
        ctx.arrivals, ctx.want_w, ctx.kind = arrivals, want_w, kind
        return _strided(kind, x, w, 0, None, None)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        gx = gw = None
        if ctx.needs_input_grad[0] and _will_run(ctx.next_functions[0][0]):
            gx = _strided(ctx.kind, gy, w, 1, None, None)
        if ctx.needs_input_grad[1] and ctx.want_w:
            gw = _strided(ctx.kind, x, w, 2, gy, ctx.arrivals)
        return gx, gw, None, None, None


class _Conv3x3Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, arrivals, want_w):
        ctx.save_for_backward(x, w)
        ctx.arrivals, ctx.want_w = arrivals, want_w
        return conv_fwd(x, w)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        gx = gw = None
        if ctx.needs_input_grad[0] and _will_run(ctx.next_functions[0][0]):
            gx = conv_fwd(gy, w, dgrad=True)
        if ctx.needs_input_grad[1] and ctx.want_w:
            gw = conv_wgrad(x, gy, w, ctx.arrivals)
        return gx, gw, None, None


def conv3x3(x: torch.Tensor, w: torch.Tensor, arrivals: torch.Tensor | None = None,
            want_w: bool = True) -> torch.Tensor:
    """y = conv2d(x, w, stride 1, padding 1) on the library's kernels.
    ``want_w=False``: the weight gradient is not wanted (a layer above the
    partial-backprop block; autograd.grad cannot tell a custom function)."""
    if arrivals is None:
        arrivals = arrival_cells(x.device)
    return _Conv3x3Fn.apply(x, w, arrivals, want_w)


def mark_weight_grads(module: nn.Module, leaves) -> None:
    """Set which ``Conv3x3`` weights the next backward differentiates (the
    block's leaves): the others skip their weight-gradient kernels."""
    ids = {id(p) for p in leaves}
    for m in module.modules():
        if isinstance(m, (Conv3x3, Conv1x1)):
            m.want_w = id(m.weight) in ids


class Conv3x3(nn.Conv2d):
    """nn.Conv2d(cin, cout, 3, stride, 1, bias=False) with the native fp32
    path for the shapes that have a kernel."""

    def __init__(self, cin: int, cout: int, stride: int = 1):
        super().__init__(cin, cout, 3, stride, 1, bias=False)
        self.want_w = True
        self._arrivals = None   # wgrad arrival counters; this module's launches are stream-ordered

    def _arrival_cells(self, device) -> torch.Tensor:
        if self._arrivals is None or self._arrivals.device != device:
            self._arrivals = arrival_cells(device)
        return self._arrivals

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        native = (x.dtype == torch.float32 and x.is_cuda and self.weight.dtype == torch.float32
                  and not torch.is_autocast_enabled("cuda") and x.shape[2] == x.shape[3] and enabled())
        if native and supported(self.in_channels, self.out_channels, x.shape[2], self.stride[0], 3):
            return conv3x3(x, self.weight, self._arrival_cells(x.device), self.want_w)
        if (native and self.stride == (2, 2)
                and _lib().lib.lpp_conv3x3s2_supported(self.in_channels, self.out_channels, x.shape[2])):
            return _StridedFn.apply(x, self.weight, self._arrival_cells(x.device), self.want_w, "3x3s2")
        return F.conv2d(x, self.weight, None, self.stride, self.padding)


class Conv1x1(nn.Conv2d):
    """nn.Conv2d(cin, cout, 1, stride, bias=False) — the projection shortcut —
    with the native fp32 path for stride 2 at the shapes with a kernel."""

    def __init__(self, cin: int, cout: int, stride: int = 1):
        super().__init__(cin, cout, 1, stride, 0, bias=False)
        self.want_w = True
        self._arrivals = None

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if (x.dtype == torch.float32 and x.is_cuda and self.weight.dtype == torch.float32
                and not torch.is_autocast_enabled("cuda") and x.shape[2] == x.shape[3] and enabled()
                and self.stride[0] == 2 and self.stride[1] == 2
                and _lib().lib.lpp_conv1x1s2_supported(self.in_channels, self.out_channels, x.shape[2])):
            if self._arrivals is None or self._arrivals.device != x.device:
                self._arrivals = arrival_cells(x.device)
            return _StridedFn.apply(x, self.weight, self._arrivals, self.want_w, "1x1")
        return F.conv2d(x, self.weight, None, self.stride, self.padding)
