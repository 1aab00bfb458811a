"""The fp32 CNN forward/backward on the library's own kernels
(``csrc/conv_f32.cu``) — the gradient step of SURVEY §8 a6 in fp32.

* ``Conv3x3`` / ``Conv1x1`` are ``nn.Conv2d``s (same parameters, init and
  state-dict names) whose forward runs our kernels when the activation is
  fp32 on a CUDA device and the shape has one — every convolution of CIFAR
  ResNet-20: the stem (on the gathered NCHW batch), the 3x3 stride-1 and
  stride-2 convolutions and the 1x1 stride-2 projections — and cuDNN's
  ``F.conv2d`` otherwise (bf16 compute or autocast, other shapes,
  ``LPP_CONV=cudnn``).  Forward (optionally with the output's BatchNorm
  statistics in the epilogue), input gradient (optionally adding the
  residual branch's gradient), weight gradient (one deterministic launch).
* ``bn_act`` is BatchNorm2d (train) [+ residual] [+ ReLU] in one pass each
  way from those statistics, torch's modules when they are absent.

NHWC activations (torch channels_last) and OHWI weights (the arena's
channels_last view, ``objectives.py`` ``_view``): no layout change runs
around the kernels.  Launches go to torch's current stream, so they are
captured into the step graphs like cuDNN's.
"""

from __future__ import annotations

import os

import torch
import torch.nn as nn
import torch.nn.functional as F

_CL = torch.channels_last
# forward convolutions with at least this many channels stage tap-major
# weights made once per call (LPP_CONV_TAPMAJOR_MIN_C; A/B runs)
_TAPMAJOR_MIN_C = int(os.environ.get("LPP_CONV_TAPMAJOR_MIN_C", "32"))


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


def conv_fwd(x: torch.Tensor, w: torch.Tensor, dgrad: bool = False, stats: torch.Tensor | None = None,
             addend: torch.Tensor | None = None):
    """y = conv(x, w) (dgrad: the input gradient for dY = x, plus
    ``addend`` when given).  With ``stats`` (LPP_CONV_ARRIVALS zeroed
    cells) also the fused BatchNorm statistics of y: returns (y, sums)."""
    N = _lib()
    n, c, h, _ = x.shape
    x = x.contiguous(memory_format=_CL)
    w = _ohwi(w)
    y = torch.empty_like(x, memory_format=_CL)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    mode = int(dgrad)
    if not dgrad and c >= _TAPMAJOR_MIN_C:
        # one tap-major copy of the weights per call instead of every CTA
        # transposing its slice while staging (~5 µs per launch at C = 64)
        wt = torch.empty(9 * c * c, dtype=torch.float32, device=x.device)
        N.check(N.lib.lpp_conv3x3_tapmajor(w.data_ptr(), wt.data_ptr(), c, stream), "conv3x3_tapmajor")
        w, mode = wt, 2
    if stats is None:
        add = None
        if addend is not None:
            add = addend.contiguous(memory_format=_CL)
        N.check(N.lib.lpp_conv3x3_f32(x.data_ptr(), w.data_ptr(), y.data_ptr(), n, c, h, mode,
                                      add.data_ptr() if add is not None else None,
                                      add.numel() * 4 if add is not None else 0, None, None, stream),
                "conv3x3_f32")
        return y
    nbytes = int(N.lib.lpp_conv3x3_stats_workspace(n, c, h))
    ws = torch.empty(max(nbytes // 4, 1), dtype=torch.float32, device=x.device)
    sums = torch.empty(2 * c, dtype=torch.float32, device=x.device)
    N.check(N.lib.lpp_conv3x3_f32(x.data_ptr(), w.data_ptr(), y.data_ptr(), n, c, h, mode, ws.data_ptr(), nbytes,
                                  sums.data_ptr(), stats.data_ptr(), stream), "conv3x3_f32")
    return y, sums


ARRIVALS = 8   # LPP_CONV_ARRIVALS


def arrival_cells(device, sets: int = 1) -> torch.Tensor:
    """Zeroed counters for the one-launch reductions (weight gradients, the
    fused BatchNorm statistics); every call leaves them zero; calls sharing
    a set must be stream-ordered.  ``sets`` sets of LPP_CONV_ARRIVALS."""
    return torch.zeros(ARRIVALS * sets, dtype=torch.int32, device=device)


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


# residual-branch gradients waiting for the dgrad of the block's first
# convolution to add them in its epilogue (instead of an autograd add
# kernel): {data_ptr of the block input: gradient}; set by _BnActFn's
# backward, consumed by _Conv3x3Fn's, always within one backward pass
_PENDING_RESID: dict[int, torch.Tensor] = {}


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
             arrivals: torch.Tensor | None, stats: torch.Tensor | None = None):
    """The stride-2 kernels (kind "1x1" or "3x3s2"): mode 0 y = conv(x, w)
    (with ``stats`` cells: (y, BatchNorm sums)); 1 dX of dY = x; 2 dW of
    (x, dY = other)."""
    N = _lib()
    fn = N.lib.lpp_conv1x1s2_f32 if kind == "1x1" else N.lib.lpp_conv3x3s2_f32
    wsq = N.lib.lpp_conv1x1s2_wgrad_workspace if kind == "1x1" else N.lib.lpp_conv3x3s2_wgrad_workspace
    ssq = N.lib.lpp_conv1x1s2_stats_workspace if kind == "1x1" else N.lib.lpp_conv3x3s2_stats_workspace
    co, ci = w.shape[0], w.shape[1]
    x = x.contiguous(memory_format=_CL)
    w = _ohwi(w)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    what = f"conv{kind}_f32"
    if mode == 0:
        n, _, hw, _ = x.shape
        out = torch.empty((n, co, hw // 2, hw // 2), device=x.device, memory_format=_CL)
        if stats is None:
            N.check(fn(x.data_ptr(), w.data_ptr(), out.data_ptr(), n, ci, co, hw, 0, None, 0, None, None, stream),
                    what)
            return out
        nbytes = int(ssq(n, ci, co, hw))
        ws = torch.empty(max(nbytes // 4, 1), dtype=torch.float32, device=x.device)
        sums = torch.empty(2 * co, dtype=torch.float32, device=x.device)
        N.check(fn(x.data_ptr(), w.data_ptr(), out.data_ptr(), n, ci, co, hw, 0, ws.data_ptr(), nbytes,
                   stats.data_ptr(), sums.data_ptr(), stream), what)
        return out, sums
    if mode == 1:
        n, _, ho, _ = x.shape
        out = torch.empty((n, ci, 2 * ho, 2 * ho), device=x.device, memory_format=_CL)
        N.check(fn(x.data_ptr(), w.data_ptr(), out.data_ptr(), n, ci, co, 2 * ho, 1, None, 0, None, None, stream),
                what)
        return out
    n, _, hw, _ = x.shape
    dy = other.contiguous(memory_format=_CL)
    out = torch.empty_like(w, memory_format=_CL)
    nbytes = int(wsq(n, ci, co, hw))
    ws = torch.empty(max(nbytes // 4, 1), dtype=torch.float32, device=x.device)
    if arrivals is None:
        arrivals = arrival_cells(x.device)
    N.check(fn(x.data_ptr(), dy.data_ptr(), out.data_ptr(), n, ci, co, hw, 2, ws.data_ptr(), nbytes,
               arrivals.data_ptr(), None, stream), what)
    return out


def conv1x1s2(x: torch.Tensor, w: torch.Tensor, mode: int, other: torch.Tensor | None = None,
              arrivals: torch.Tensor | None = None, stats: torch.Tensor | None = None):
    """The projection shortcut's kernels (1x1, stride 2)."""
    return _strided("1x1", x, w, mode, other, arrivals, stats)


def conv3x3s2(x: torch.Tensor, w: torch.Tensor, mode: int, other: torch.Tensor | None = None,
              arrivals: torch.Tensor | None = None, stats: torch.Tensor | None = None):
    """The stage-opening 3x3 stride-2 convolution's kernels."""
    return _strided("3x3s2", x, w, mode, other, arrivals, stats)


def _stat_cells(arrivals):
    return arrivals[ARRIVALS:2 * ARRIVALS] if arrivals.numel() >= 2 * ARRIVALS else None


class _StridedFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, arrivals, want_w, kind, with_stats):
        ctx.set_materialize_grads(False)    # no zero-filled gradient for the statistics output
        ctx.save_for_backward(x, w)
        ctx.arrivals, ctx.want_w, ctx.kind = arrivals, want_w, kind
        if with_stats:
            y, sums = _strided(kind, x, w, 0, None, None, _stat_cells(arrivals))
            ctx.mark_non_differentiable(sums)
            return y, sums
        return _strided(kind, x, w, 0, None, None), None

    @staticmethod
    def backward(ctx, gy, _gsums):
        x, w = ctx.saved_tensors
        gx = gw = None
        if gy is None:
            return (None,) * len(ctx.needs_input_grad)
        if ctx.needs_input_grad[0] and _will_run(ctx.next_functions[0][0]):
            gx = _strided(ctx.kind, gy, w, 1, None, None)
        if ctx.needs_input_grad[1] and ctx.want_w:
            gw = _strided(ctx.kind, x, w, 2, gy, ctx.arrivals)
        return gx, gw, None, None, None, None


def stem(x: torch.Tensor, w: torch.Tensor, mode: int, dy: torch.Tensor | None = None,
         arrivals: torch.Tensor | None = None, stats: torch.Tensor | None = None):
    """The CIFAR stem (3 -> 16, 3x3, 32 x 32) on NCHW input: mode 0 y
    (channels-last; with ``stats`` cells: (y, BatchNorm sums)); mode 2 dW."""
    N = _lib()
    n = x.shape[0]
    x = x.contiguous()                                  # NCHW, as gathered
    stream = torch.cuda.current_stream(x.device).cuda_stream
    nbytes = int(N.lib.lpp_stem_workspace(n))
    if mode == 0:
        y = torch.empty((n, 16, 32, 32), device=x.device, memory_format=_CL)
        if stats is None:
            N.check(N.lib.lpp_stem_f32(x.data_ptr(), w.data_ptr(), y.data_ptr(), n, 0, None, 0, None, None, stream),
                    "stem_f32")
            return y
        ws = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device)
        sums = torch.empty(32, dtype=torch.float32, device=x.device)
        N.check(N.lib.lpp_stem_f32(x.data_ptr(), _ohwi(w).data_ptr(), y.data_ptr(), n, 0, ws.data_ptr(), nbytes,
                                   stats.data_ptr(), sums.data_ptr(), stream), "stem_f32")
        return y, sums
    dy = dy.contiguous(memory_format=_CL)
    ws = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device)
    # OHWI, like the weight's arena view: the step's one multi-tensor gradient
    # copy keeps its fast path only when every gradient is dense
    dw = torch.empty((16, 3, 3, 3), dtype=torch.float32, device=x.device, memory_format=_CL)
    if arrivals is None:
        arrivals = arrival_cells(x.device)
    N.check(N.lib.lpp_stem_f32(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), n, 2, ws.data_ptr(), nbytes,
                               arrivals.data_ptr(), None, stream), "stem_f32")
    return dw


class _StemFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, arrivals, want_w, with_stats):
        ctx.set_materialize_grads(False)
        ctx.save_for_backward(x)
        ctx.arrivals, ctx.want_w = arrivals, want_w
        w = _ohwi(w)
        if with_stats:
            y, sums = stem(x, w, 0, stats=_stat_cells(arrivals))
            ctx.mark_non_differentiable(sums)
            return y, sums
        return stem(x, w, 0), None

    @staticmethod
    def backward(ctx, gy, _gsums):
        (x,) = ctx.saved_tensors
        if gy is None or not (ctx.needs_input_grad[1] and ctx.want_w):
            return None, None, None, None, None
        return None, stem(x, None, 2, gy, ctx.arrivals), None, None, None


class _Conv3x3Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, arrivals, want_w, with_stats):
        ctx.set_materialize_grads(False)    # no zero-filled gradient for the statistics output
        ctx.save_for_backward(x, w)
        ctx.arrivals, ctx.want_w = arrivals, want_w
        # a residual gradient left for an earlier tensor at this address (a
        # backward that raised between the hand-off and this dgrad) is stale
        _PENDING_RESID.pop(x.data_ptr(), None)
        if with_stats:
            y, sums = conv_fwd(x, w, stats=_stat_cells(arrivals))
            ctx.mark_non_differentiable(sums)
            return y, sums
        return conv_fwd(x, w), None

    @staticmethod
    def backward(ctx, gy, _gsums):
        x, w = ctx.saved_tensors
        gx = gw = None
        pending = _PENDING_RESID.pop(x.data_ptr(), None)
        if gy is None:
            return (pending,) + (None,) * (len(ctx.needs_input_grad) - 1)
        if ctx.needs_input_grad[0] and _will_run(ctx.next_functions[0][0]):
            gx = conv_fwd(gy, w, dgrad=True, addend=pending)
        elif pending is not None:
            gx = pending
        if ctx.needs_input_grad[1] and ctx.want_w:
            gw = conv_wgrad(x, gy, w, ctx.arrivals)
        return gx, gw, None, None, None


def conv3x3(x: torch.Tensor, w: torch.Tensor, arrivals: torch.Tensor | None = None,
            want_w: bool = True, with_stats: bool = False):
    """y = conv2d(x, w, stride 1, padding 1) on the library's kernels.
    ``want_w=False``: the weight gradient is not wanted (a layer above the
    partial-backprop block; autograd.grad cannot tell a custom function).
    ``with_stats``: returns (y, BatchNorm sums of y) — y's statistics fused
    into the forward's epilogue."""
    if arrivals is None:
        arrivals = arrival_cells(x.device, 2)
    y, sums = _Conv3x3Fn.apply(x, w, arrivals, want_w, with_stats)
    return (y, sums) if with_stats else y


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
        # bn_stats: a BatchNorm consumes the output (bn_act) — compute its
        # statistics in the forward's epilogue
        self.bn_stats = False
        self._arrivals = None   # arrival counters; this module's launches are stream-ordered

    def _arrival_cells(self, device) -> torch.Tensor:
        if self._arrivals is None or self._arrivals.device != device:
            self._arrivals = arrival_cells(device, 2)
        return self._arrivals

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        native = (x.dtype == torch.float32 and x.is_cuda and self.weight.dtype == torch.float32
                  and not torch.is_autocast_enabled("cuda") and x.shape[2] == x.shape[3] and enabled())
        if native and supported(self.in_channels, self.out_channels, x.shape[2], self.stride[0], 3):
            y, sums = _Conv3x3Fn.apply(x, self.weight, self._arrival_cells(x.device), self.want_w, self.bn_stats)
            y._lpp_input_ptr = x.data_ptr()
            return _with_sums(y, sums)
        if (native and self.stride == (2, 2)
                and _lib().lib.lpp_conv3x3s2_supported(self.in_channels, self.out_channels, x.shape[2])):
            y, sums = _StridedFn.apply(x, self.weight, self._arrival_cells(x.device), self.want_w, "3x3s2",
                                       self.bn_stats)
            return _with_sums(y, sums)
        if (native and self.stride == (1, 1) and (self.in_channels, self.out_channels) == (3, 16)
                and x.shape[2] == 32 and not x.requires_grad):
            y, sums = _StemFn.apply(x, self.weight, self._arrival_cells(x.device), self.want_w, self.bn_stats)
            return _with_sums(y, sums)
        if self.weight.is_contiguous(memory_format=_CL) and not x.is_contiguous(memory_format=_CL):
            x = x.contiguous(memory_format=_CL)
        return F.conv2d(x, self.weight, None, self.stride, self.padding)


class Conv1x1(nn.Conv2d):
    """nn.Conv2d(cin, cout, 1, stride, bias=False) — the projection shortcut —
    with the native fp32 path for stride 2 at the shapes with a kernel."""

    def __init__(self, cin: int, cout: int, stride: int = 1):
        super().__init__(cin, cout, 1, stride, 0, bias=False)
        self.want_w = True
        self.bn_stats = False
        self._arrivals = None

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if (x.dtype == torch.float32 and x.is_cuda and self.weight.dtype == torch.float32
                and not torch.is_autocast_enabled("cuda") and x.shape[2] == x.shape[3] and enabled()
                and self.stride[0] == 2 and self.stride[1] == 2
                and _lib().lib.lpp_conv1x1s2_supported(self.in_channels, self.out_channels, x.shape[2])):
            if self._arrivals is None or self._arrivals.device != x.device:
                self._arrivals = arrival_cells(x.device, 2)
            y, sums = _StridedFn.apply(x, self.weight, self._arrivals, self.want_w, "1x1", self.bn_stats)
            return _with_sums(y, sums)
        return F.conv2d(x, self.weight, None, self.stride, self.padding)


def _with_sums(y: torch.Tensor, sums: torch.Tensor | None) -> torch.Tensor:
    if sums is not None:
        y._lpp_bn_sums = sums
    return y


class _BnActFn(torch.autograd.Function):
    """BatchNorm2d (training) [+ residual] [+ ReLU] from the statistics the
    producing convolution fused into its epilogue: forward one
    ``lpp_bn_apply_f32`` pass; backward ``lpp_bn_backward_f32`` (ReLU mask,
    per-channel sums, dx / residual gradient / dgamma / dbeta: the formulas
    of torch.native_batch_norm_backward in train mode)."""

    @staticmethod
    def forward(ctx, x, gamma, beta, resid, sums, running_mean, running_var, eps, momentum, relu, cells,
                resid_consumer=None):
        N = _lib()
        n, c, h, w_ = x.shape
        y = torch.empty_like(x, memory_format=_CL)
        mean = torch.empty(c, dtype=torch.float32, device=x.device)
        invstd = torch.empty(c, dtype=torch.float32, device=x.device)
        rm = running_mean.data_ptr() if running_mean is not None else None
        rv = running_var.data_ptr() if running_var is not None else None
        # the ReLU mask (1 bit per element) is what the backward reads instead of y
        mask = torch.empty(n * c * h * w_ // 32 if relu else 1, dtype=torch.int32, device=x.device)
        N.check(N.lib.lpp_bn_apply_f32(x.data_ptr(), sums.data_ptr(), gamma.data_ptr(), beta.data_ptr(),
                                       resid.data_ptr() if resid is not None else None, y.data_ptr(),
                                       mean.data_ptr(), invstd.data_ptr(), rm, rv,
                                       mask.data_ptr() if relu else None, n * h * w_, c, float(eps),
                                       float(momentum), int(relu),
                                       torch.cuda.current_stream(x.device).cuda_stream), "bn_apply_f32")
        ctx.save_for_backward(x, gamma, mean, invstd, mask)
        ctx.relu, ctx.has_resid, ctx.cells = relu, resid is not None, cells
        ctx.resid_ptr = resid.data_ptr() if resid is not None else None
        ctx.resid_consumer = resid_consumer
        return y

    @staticmethod
    def backward(ctx, gy):
        N = _lib()
        x, gamma, mean, invstd, mask = ctx.saved_tensors
        n, c, h, w_ = x.shape
        need = ctx.needs_input_grad
        gy = gy.contiguous(memory_format=_CL)
        gx = torch.empty_like(x, memory_format=_CL) if need[0] and _will_run(ctx.next_functions[0][0]) else None
        gres = torch.empty_like(x, memory_format=_CL) if ctx.has_resid and need[3] else None
        gg = torch.empty_like(gamma) if need[1] else None
        gb = torch.empty_like(gamma) if need[2] else None
        nbytes = int(N.lib.lpp_bn_backward_workspace(n * h * w_, c))
        ws = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device)
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        N.check(N.lib.lpp_bn_backward_f32(gy.data_ptr(), mask.data_ptr() if ctx.relu else None, x.data_ptr(),
                                          mean.data_ptr(),
                                          invstd.data_ptr(), gamma.data_ptr(), ptr(gx), ptr(gres), ptr(gg), ptr(gb),
                                          ws.data_ptr(), nbytes, ctx.cells.data_ptr(), n * h * w_, c, int(ctx.relu),
                                          torch.cuda.current_stream(x.device).cuda_stream), "bn_backward_f32")
        consumer = ctx.resid_consumer
        if (gres is not None and consumer is not None and _will_run(consumer)
                and _will_run(consumer.next_functions[0][0])):
            # the block's first convolution adds it in its dgrad epilogue
            _PENDING_RESID[ctx.resid_ptr] = gres
            gres = None
        return gx, gg, gb, gres, None, None, None, None, None, None, None, None


def bn_act(x: torch.Tensor, bn: nn.BatchNorm2d, relu: bool = True, resid: torch.Tensor | None = None,
           resid_consumer: torch.Tensor | None = None):
    """``[relu](bn(x) [+ resid])``: one fused pass when x came from one of
    our convolutions with its statistics (``bn_stats``) and bn trains;
    torch's modules otherwise (cuDNN BatchNorm, eval mode, bf16, ...)."""
    sums = getattr(x, "_lpp_bn_sums", None)
    if (sums is None or not bn.training or not bn.affine or not bn.track_running_stats
            or bn.momentum is None or x.dtype != torch.float32 or not enabled()):
        out = bn(x)
        if resid is not None:
            out = out + resid
        return F.relu(out) if relu else out
    if resid is not None:
        resid = resid.contiguous(memory_format=_CL)
    cells = getattr(bn, "_lpp_arrivals", None)
    if cells is None or cells.device != x.device:
        # the backward's one-launch reduction; this module's launches are stream-ordered
        cells = bn._lpp_arrivals = arrival_cells(x.device)
    node = None
    if resid_consumer is not None and resid is not None:
        # resid_consumer: the output of the block's first convolution, whose
        # input is resid — on our kernel its dgrad adds the residual gradient
        fn = resid_consumer.grad_fn
        if fn is not None and type(fn).__name__ == "_Conv3x3FnBackward" and \
                resid.data_ptr() == resid_consumer._lpp_input_ptr:
            node = fn
    return _BnActFn.apply(x, bn.weight, bn.bias, resid, sums, bn.running_mean, bn.running_var, bn.eps,
                          bn.momentum, relu, cells, node)
