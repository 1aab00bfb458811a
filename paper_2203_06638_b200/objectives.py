"""Torch-backed objectives whose parameters are views into a flat arena.

The reference's ``Objective`` protocol (``objectives.py:33-63``) is kept:
``dim``, ``n_samples``, ``layer_param_counts``, ``init_params(seed)``,
``loss``, ``grad_block(x, block, batch) -> GradResult``, ``full_loss``,
``full_grad``, ``backward_cost``.  On top of it every objective can *bind* a
replica arena (parameters) and a gradient arena to a model, which is what
the engine's captured CUDA-graph steps run (``bind`` / ``loss_on``).

* ``MlpObjective`` — the reference MLP (``objectives.py:200-319``) with the
  reference flat layout ``[W1, b1, ...]``, ``W_l`` of shape (in, out),
  ``z = a @ W + b``; used for the deterministic parity gate.
* ``ResNetObjective`` — the small CNN of BASELINE config 0 (``smallcnn``),
  CIFAR ResNet-20 (d=272,474, 65 tensors), CIFAR
  ResNet-18 (d=11,220,132, 62 tensors), ImageNet ResNet-50 (d=25,557,032,
  161 tensors) on synthetic data.  The CNN
  forward/backward stays in PyTorch, as in the paper; partial
  backprop is autograd restricted to the block's leaf tensors.

Parameters are fp32 views into the replica arena; gradients are fp32 views
into the gradient arena, so one apply launch covers any block range.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .conv import Conv1x1, Conv3x3, bn_act, mark_weight_grads
from .conv import enabled as conv_enabled
from .partition import Block


@dataclass(frozen=True)
class GradResult:
    """``objectives.py:23-30``; ``values`` is a device tensor here."""

    values: torch.Tensor
    flops: int
    backward_flops: int
    batch_size: int


class Bound:
    """A model whose parameters / grads are views into two arenas.

    ``grad_views[i]`` is where the gradient of ``params[i]`` belongs in the
    fp32 gradient arena (by default ``params[i].grad``; a bf16 shadow weight
    has an fp32 view here instead).  ``mixed`` is False when the bound model
    already computes in its compute dtype (no autocast needed)."""

    def __init__(self, params: list[torch.Tensor], forward, grad_views=None, mixed: bool = True):
        self.params = params
        self.forward = forward  # forward(xb) -> logits
        self.grad_views = grad_views if grad_views is not None else [p.grad for p in params]
        self.mixed = mixed


class ArenaObjective:
    """Common machinery: dataset on device, layer edges, grad_block."""

    dim: int
    n_samples: int
    n_classes: int
    layer_param_counts: tuple[int, ...]
    autocast_dtype: torch.dtype | None = None

    def _finish_layout(self) -> None:
        edges = [0]
        for c in self.layer_param_counts:
            edges.append(edges[-1] + int(c))
        self.edges = tuple(edges)
        self.dim = edges[-1]

    # -- data --------------------------------------------------------------

    def features_on(self, device) -> torch.Tensor:
        key = str(torch.device(device))
        if key not in self._feat_cache:
            self._feat_cache[key] = self.features.to(device, non_blocking=False)
            self._lab_cache[key] = self.labels.to(device, non_blocking=False)
        return self._feat_cache[key]

    def labels_on(self, device) -> torch.Tensor:
        self.features_on(device)
        return self._lab_cache[str(torch.device(device))]

    # -- blocks -------------------------------------------------------------

    def tensors_of_block(self, block: Block) -> tuple[int, int]:
        """[first, last] tensor indices covered by a layer-aligned block."""
        if block.start == 0 and block.stop == self.dim:
            return 0, len(self.layer_param_counts) - 1
        try:
            first = self.edges.index(block.start)
            last = self.edges.index(block.stop) - 1
        except ValueError:
            raise ValueError(f"block {block} does not align to layer boundaries") from None
        return first, last

    def check_block(self, block: Block) -> None:
        if not (0 <= block.start < block.stop <= self.dim):
            raise ValueError(f"block {block} outside [0, {self.dim})")

    # -- reference protocol --------------------------------------------------

    def _as_device_params(self, x, device) -> torch.Tensor:
        t = torch.as_tensor(x)
        return t.to(device=device, dtype=torch.float32).contiguous()

    def loss_on(self, bound: Bound, xb: torch.Tensor, yb: torch.Tensor) -> torch.Tensor:
        if self.autocast_dtype is not None and bound.mixed:
            with torch.autocast("cuda", dtype=self.autocast_dtype):
                logits = bound.forward(xb)
            return F.cross_entropy(logits.float(), yb)
        return F.cross_entropy(bound.forward(xb).float(), yb)

    def loss(self, x, batch) -> float:
        device = torch.device("cuda", torch.cuda.current_device())
        xp = self._as_device_params(x, device)
        bound = self.bind(xp, None)
        idx = torch.as_tensor(np.asarray(batch), device=device, dtype=torch.long)
        with torch.no_grad():
            return float(self.loss_on(bound, self.features_on(device)[idx], self.labels_on(device)[idx]))

    def grad_block(self, x, block: Block, batch) -> GradResult:
        self.check_block(block)
        first, last = self.tensors_of_block(block)
        device = torch.device("cuda", torch.cuda.current_device())
        xp = self._as_device_params(x, device)
        g = torch.zeros_like(xp)
        bound = self.bind(xp, g)
        idx = torch.as_tensor(np.asarray(batch), device=device, dtype=torch.long)
        if getattr(bound, "module", None) is not None:
            mark_weight_grads(bound.module, bound.params[first:last + 1])
        loss = self.loss_on(bound, self.features_on(device)[idx], self.labels_on(device)[idx])
        grads = torch.autograd.grad(loss, bound.params[first:last + 1])
        torch._foreach_copy_(bound.grad_views[first:last + 1], list(grads))
        n = len(idx)
        back = n * self.backward_cost(block)
        return GradResult(g[block.start:block.stop], n * self.forward_cost() + back, back, n)

    def full_loss(self, x) -> float:
        return self.loss(x, np.arange(self.n_samples))

    def full_grad(self, x) -> torch.Tensor:
        return self.grad_block(x, Block(0, self.dim), np.arange(self.n_samples)).values

    # cost model hooks (per sample, multiply-adds)
    def forward_cost(self) -> int:
        return 0

    def backward_cost(self, block: Block) -> int:
        return 0


# ---------------------------------------------------------------------------
# the reference MLP


class MlpObjective(ArenaObjective):
    """Reference MLP, flat layout [W1, b1, ...], W_l (in, out) (objectives.py:200-250)."""

    def __init__(self, features, labels, hidden: tuple[int, ...], n_classes: int):
        feats = torch.as_tensor(np.asarray(features), dtype=torch.float32)
        labs = torch.as_tensor(np.asarray(labels), dtype=torch.long)
        if feats.dim() != 2 or feats.shape[0] == 0:
            raise ValueError("features must be a non-empty (n, f) array")
        if int(labs.min()) < 0 or int(labs.max()) >= n_classes:
            raise ValueError("labels outside [0, n_classes)")
        self.features, self.labels = feats, labs
        self._feat_cache, self._lab_cache = {}, {}
        self.n_samples = feats.shape[0]
        self.n_classes = n_classes
        self.widths = (feats.shape[1], *hidden, n_classes)
        self.n_layers = len(self.widths) - 1
        self.layer_param_counts = tuple(
            self.widths[l] * self.widths[l + 1] + self.widths[l + 1] for l in range(self.n_layers))
        self._finish_layout()
        # tensor-level edges: W and b of each layer are separate leaves
        self.tensor_sizes = []
        for l in range(self.n_layers):
            self.tensor_sizes += [self.widths[l] * self.widths[l + 1], self.widths[l + 1]]

    def init_params(self, seed: int) -> np.ndarray:
        """Bitwise the reference init (objectives.py:235-240), fp64 host vector."""
        gen = np.random.default_rng(np.random.SeedSequence([seed, self.dim]))
        x = np.zeros(self.dim)
        for l in range(self.n_layers):
            lo = self.edges[l]
            a, b = self.widths[l], self.widths[l + 1]
            x[lo:lo + a * b] = gen.normal(scale=1.0 / np.sqrt(a), size=(a, b)).reshape(-1)
        return x

    def _views(self, arena: torch.Tensor):
        out = []
        for l in range(self.n_layers):
            lo = self.edges[l]
            a, b = self.widths[l], self.widths[l + 1]
            out.append((arena[lo:lo + a * b].view(a, b), arena[lo + a * b:self.edges[l + 1]]))
        return out

    def bind(self, arena: torch.Tensor, grad_arena: torch.Tensor | None) -> Bound:
        pv = self._views(arena)
        gv = self._views(grad_arena) if grad_arena is not None else None
        params = []
        for l, (w, b) in enumerate(pv):
            w = w.detach().requires_grad_(grad_arena is not None)
            b = b.detach().requires_grad_(grad_arena is not None)
            if gv is not None:
                w.grad, b.grad = gv[l][0], gv[l][1]
            params += [w, b]
        L = self.n_layers

        def forward(xb):
            a = xb
            for l in range(L):
                a = torch.addmm(params[2 * l + 1], a, params[2 * l])
                if l < L - 1:
                    a = torch.tanh(a)
            return a

        return Bound(params, forward)

    def tensors_of_block(self, block: Block) -> tuple[int, int]:
        first_layer, last_layer = self._layers_of_block(block)
        return 2 * first_layer, 2 * last_layer + 1

    def _layers_of_block(self, block: Block) -> tuple[int, int]:
        if block.start == 0 and block.stop == self.dim:
            return 0, self.n_layers - 1
        try:
            return self.edges.index(block.start), self.edges.index(block.stop) - 1
        except ValueError:
            raise ValueError(f"block {block} does not align to layer boundaries") from None

    def forward_cost(self) -> int:
        return sum(self.widths[l] * self.widths[l + 1] for l in range(self.n_layers))

    def backward_cost(self, block: Block) -> int:
        first, _ = self._layers_of_block(block)
        return sum(2 * self.widths[l] * self.widths[l + 1] for l in range(first, self.n_layers))


def flops_savings_ratio(obj: ArenaObjective, partition) -> float:
    """Backward work saved by cycling partial blocks instead of full passes:
    ``1 - sum_i cost(block_i) / (U * cost(full))`` (objectives.py:326-337)."""
    if obj.layer_param_counts is None:
        raise ValueError("truncated-backprop savings need a layered objective")
    full = obj.backward_cost(Block(0, obj.dim))
    blocks = partition.blocks()
    return 1.0 - sum(obj.backward_cost(b) for b in blocks) / (len(blocks) * full)


# ---------------------------------------------------------------------------
# desk-scale objectives of the reference (objectives.py:111-193): one flat
# parameter tensor, blocks may split it anywhere (layer_param_counts = None)


class _FlatObjective(ArenaObjective):
    layer_param_counts = None

    def _flat_init(self, features, labels):
        self.features = torch.as_tensor(np.asarray(features), dtype=torch.float32)
        self.labels = torch.as_tensor(np.asarray(labels))
        self._feat_cache, self._lab_cache = {}, {}
        self.n_samples = int(self.features.shape[0])
        self.edges = (0, self.dim)

    def tensors_of_block(self, block: Block) -> tuple[int, int]:
        self.check_block(block)
        return 0, 0          # the block is a range inside the single tensor

    def init_params(self, seed: int) -> np.ndarray:
        return np.zeros(self.dim)

    def bind(self, arena: torch.Tensor, grad_arena: torch.Tensor | None) -> Bound:
        w = arena.detach().requires_grad_(grad_arena is not None)
        if grad_arena is not None:
            w.grad = grad_arena
        return Bound([w], lambda xb: xb)

    def forward_cost(self) -> int:
        return self.dim

    def backward_cost(self, block: Block) -> int:
        return self.dim


class QuadraticObjective(_FlatObjective):
    """f(x) = mean_n 0.5 ||x - t_n||^2 (objectives.py:111-145)."""

    def __init__(self, targets):
        t = np.asarray(targets, dtype=np.float64)
        if t.ndim != 2 or t.shape[0] == 0:
            raise ValueError("targets must be a non-empty (n, d) array")
        self.dim = int(t.shape[1])
        self.n_classes = 0
        self._flat_init(t, np.zeros(t.shape[0], dtype=np.int64))
        self.minimizer = t.mean(axis=0)

    def loss_on(self, bound: Bound, xb: torch.Tensor, yb: torch.Tensor) -> torch.Tensor:
        diff = bound.params[0].unsqueeze(0) - xb
        return 0.5 * (diff * diff).sum(dim=1).mean()


class LogisticObjective(_FlatObjective):
    """Binary logistic loss over +-1 labels (objectives.py:152-193)."""

    def __init__(self, features, labels):
        f = np.asarray(features, dtype=np.float64)
        lab = np.asarray(labels)
        if f.ndim != 2 or f.shape[0] == 0:
            raise ValueError("features must be a non-empty (n, f) array")
        if set(np.unique(lab)) - {-1, 1}:
            raise ValueError("labels must be +-1")
        self.dim = int(f.shape[1])
        self.n_classes = 2
        self._flat_init(f, lab.astype(np.float64))
        self.labels = self.labels.to(torch.float32)

    def loss_on(self, bound: Bound, xb: torch.Tensor, yb: torch.Tensor) -> torch.Tensor:
        margin = yb * (xb @ bound.params[0])
        return F.softplus(-margin).mean()           # log(1 + exp(-margin))


# ---------------------------------------------------------------------------
# ResNets (CIFAR ResNet-20 / ResNet-18, ImageNet ResNet-50)


class _Basic(nn.Module):
    expansion = 1

    def __init__(self, cin, cout, stride):
        super().__init__()
        # 3x3 convolutions: fp32 stride-1 C->C ones at the CIFAR ResNet-20
        # shapes run on the library's kernels (conv.py), the rest on cuDNN
        self.conv1 = Conv3x3(cin, cout, stride)
        self.bn1 = nn.BatchNorm2d(cout)
        self.conv2 = Conv3x3(cout, cout, 1)
        self.bn2 = nn.BatchNorm2d(cout)
        self.shortcut = None
        if stride != 1 or cin != cout:
            self.shortcut = nn.Sequential(Conv1x1(cin, cout, stride), nn.BatchNorm2d(cout))
            self.shortcut[0].bn_stats = True
        # the convolutions' epilogues compute their BatchNorm statistics and
        # bn_act applies BatchNorm (+ residual) + ReLU in one pass (conv.py)
        self.conv1.bn_stats = self.conv2.bn_stats = True

    def forward(self, x):
        c1 = self.conv1(x)
        out = bn_act(c1, self.bn1, relu=True)
        sc = x if self.shortcut is None else bn_act(self.shortcut[0](x), self.shortcut[1], relu=False)
        # identity blocks: conv1's dgrad adds the residual gradient of x
        return bn_act(self.conv2(out), self.bn2, relu=True, resid=sc,
                      resid_consumer=c1 if self.shortcut is None else None)


class _Bottleneck(nn.Module):
    expansion = 4

    def __init__(self, cin, width, stride):
        super().__init__()
        cout = width * 4
        self.conv1 = nn.Conv2d(cin, width, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(width)
        self.conv2 = nn.Conv2d(width, width, 3, stride, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(width)
        self.conv3 = nn.Conv2d(width, cout, 1, bias=False)
        self.bn3 = nn.BatchNorm2d(cout)
        self.shortcut = None
        if stride != 1 or cin != cout:
            self.shortcut = nn.Sequential(nn.Conv2d(cin, cout, 1, stride, bias=False),
                                          nn.BatchNorm2d(cout))

    def forward(self, x):
        out = F.relu(self.bn1(self.conv1(x)))
        out = F.relu(self.bn2(self.conv2(out)))
        out = self.bn3(self.conv3(out))
        return F.relu(out + (x if self.shortcut is None else self.shortcut(x)))


class CifarResNet20(nn.Module):
    """He et al. CIFAR ResNet-20 with 1x1-conv+BN projection shortcuts:
    272,474 parameters in 65 tensors (SURVEY §2 notes, d20)."""

    def __init__(self, num_classes=10):
        super().__init__()
        self.conv1 = Conv3x3(3, 16, 1)        # the stem: native on NCHW input in fp32 (conv.py)
        self.conv1.bn_stats = True
        self.bn1 = nn.BatchNorm2d(16)
        layers, cin = [], 16
        for cout, stride in ((16, 1), (32, 2), (64, 2)):
            for i in range(3):
                layers.append(_Basic(cin, cout, stride if i == 0 else 1))
                cin = cout
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(64, num_classes)

    def forward(self, x):
        out = bn_act(self.conv1(x), self.bn1, relu=True)
        out = self.layers(out)
        out = F.adaptive_avg_pool2d(out, 1).flatten(1)
        return self.fc(out)


class CifarResNet18(nn.Module):
    """CIFAR ResNet-18 (3x3 stem, no max-pool): 11,220,132 parameters in 62
    tensors at 100 classes (d18)."""

    def __init__(self, num_classes=100):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 64, 3, 1, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(64)
        layers, cin = [], 64
        for cout, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
            for i in range(2):
                layers.append(_Basic(cin, cout, stride if i == 0 else 1))
                cin = cout
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(512, num_classes)

    def forward(self, x):
        out = F.relu(self.bn1(self.conv1(x)))
        out = self.layers(out)
        out = F.adaptive_avg_pool2d(out, 1).flatten(1)
        return self.fc(out)


class ResNet50(nn.Module):
    """ImageNet ResNet-50 (v1.5: stride on the 3x3): 25,557,032 parameters in
    161 tensors (d50)."""

    def __init__(self, num_classes=1000):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 64, 7, 2, 3, bias=False)
        self.bn1 = nn.BatchNorm2d(64)
        layers, cin = [], 64
        for width, n, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
            for i in range(n):
                layers.append(_Bottleneck(cin, width, stride if i == 0 else 1))
                cin = width * 4
        self.layers = nn.Sequential(*layers)
        self.fc = nn.Linear(2048, num_classes)

    def forward(self, x):
        out = F.relu(self.bn1(self.conv1(x)))
        out = F.max_pool2d(out, 3, 2, 1)
        out = self.layers(out)
        out = F.adaptive_avg_pool2d(out, 1).flatten(1)
        return self.fc(out)


class SmallCnn(nn.Module):
    """The "small CNN" of BASELINE config 0 (the reference's CPU-runnable
    case): conv 3->16 s2 -> tanh -> conv 16->32 s2 -> tanh -> 2x2 average
    pool -> linear 512->10; 6 tensors, 10,218 parameters.  Smooth (tanh,
    average pooling) so fp32-vs-fp64 parity has no kink flips."""

    def __init__(self, num_classes=10):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 16, 3, stride=2, padding=1)
        self.conv2 = nn.Conv2d(16, 32, 3, stride=2, padding=1)
        self.fc = nn.Linear(32 * 4 * 4, num_classes)

    def forward(self, x):
        x = torch.tanh(self.conv1(x))
        x = torch.tanh(self.conv2(x))
        return self.fc(F.avg_pool2d(x, 2).flatten(1))


_ARCHS = {
    "smallcnn": (SmallCnn, (3, 32, 32), 10),
    "resnet20": (CifarResNet20, (3, 32, 32), 10),
    "resnet18": (CifarResNet18, (3, 32, 32), 100),
    "resnet50": (ResNet50, (3, 224, 224), 1000),
}


def _conv_macs(model: nn.Module, shape) -> dict[str, int]:
    """Per-sample forward multiply-adds of each parameterised module."""
    macs: dict[str, int] = {}
    hooks = []
    for name, mod in model.named_modules():
        if isinstance(mod, nn.Conv2d):
            def hook(m, i, o, name=name):
                macs[name] = int(o[0].numel() * m.in_channels // m.groups * m.kernel_size[0] * m.kernel_size[1])
            hooks.append(mod.register_forward_hook(hook))
        elif isinstance(mod, nn.Linear):
            def hook(m, i, o, name=name):
                macs[name] = int(m.in_features * m.out_features)
            hooks.append(mod.register_forward_hook(hook))
    with torch.no_grad():
        model.eval()
        model(torch.zeros(1, *shape))
        model.train()
    for h in hooks:
        h.remove()
    return macs


class ResNetObjective(ArenaObjective):
    """A ResNet over a synthetic image dataset, parameters in a flat arena.

    ``data`` is "device" (synthetic N(0,1) images generated on the GPU, the
    HBM-resident throughput configuration) or "host" (pinned host tensors,
    for the end-to-end measurement with per-step H2D copies).
    """

    def __init__(self, arch: str = "resnet20", n_samples: int = 8192, seed: int = 0,
                 channels_last: bool = True, autocast: str | None = "bf16",
                 data: str = "device", n_classes: int | None = None,
                 pattern_scale: float = 0.0, shadow_weights: bool = True):
        if arch not in _ARCHS:
            raise ValueError(f"unknown arch {arch!r}")
        cls, shape, k = _ARCHS[arch]
        self.arch = arch
        self.n_classes = int(n_classes or k)
        self.image_shape = shape
        self.n_samples = int(n_samples)
        self.seed = seed
        self.channels_last = channels_last
        self.autocast_dtype = {"bf16": torch.bfloat16, "fp16": torch.float16, None: None}[autocast]
        self.data_mode = data
        # 0: N(0,1) images, uniform labels; > 0: a fixed
        # random pattern per class times pattern_scale plus N(0,1) noise —
        # make_blobs (data.py:34-52) in image space, a learnable task
        self.pattern_scale = float(pattern_scale)
        self._feat_cache, self._lab_cache = {}, {}
        self._template = cls(self.n_classes)
        self.param_names = [n for n, _ in self._template.named_parameters()]
        # bf16 compute: conv / linear parameters live in a bf16 shadow (the
        # tensors autocast would cast); BatchNorm parameters stay fp32
        self.shadow_weights = shadow_weights and self.autocast_dtype is not None
        self._compute_in_shadow = [
            isinstance(self._template.get_submodule(n.rsplit(".", 1)[0]), (nn.Conv2d, nn.Linear))
            for n in self.param_names]
        self.param_shapes = [tuple(p.shape) for p in self._template.parameters()]
        self.layer_param_counts = tuple(int(p.numel()) for p in self._template.parameters())
        self._finish_layout()
        macs = _conv_macs(self._template, shape)
        # cost model: forward MACs per sample; backward of a tensor's module = 2x
        self._fwd_macs = sum(macs.values())
        owner = []
        for name in self.param_names:
            mod = name.rsplit(".", 1)[0]
            owner.append(macs.get(mod, 0))
        self._tensor_macs = owner
        self._features = None

    # synthetic dataset: N(0,1) images, uniform labels
    def _patterns(self) -> torch.Tensor:
        g = torch.Generator().manual_seed(self.seed + 7919)
        return torch.randn(self.n_classes, *self.image_shape, generator=g) * self.pattern_scale

    @property
    def features(self) -> torch.Tensor:
        if self._features is None:
            g = torch.Generator().manual_seed(self.seed)
            self._labels = torch.randint(0, self.n_classes, (self.n_samples,), generator=g)
            if self.data_mode == "host":
                f = torch.randn(self.n_samples, *self.image_shape, generator=g)
                if self.pattern_scale:
                    f += self._patterns()[self._labels]
                self._features = f.pin_memory() if torch.cuda.is_available() else f
            else:
                self._features = "device"
        return self._features

    @property
    def labels(self) -> torch.Tensor:
        self.features
        return self._labels

    def features_on(self, device) -> torch.Tensor:
        key = str(torch.device(device))
        if key not in self._feat_cache:
            self.features
            if self.data_mode == "host":
                self._feat_cache[key] = self._features.to(device)
            else:
                g = torch.Generator(device=device).manual_seed(self.seed)
                f = torch.randn(self.n_samples, *self.image_shape, generator=g, device=device)
                if self.pattern_scale:
                    f += self._patterns().to(device)[self._labels.to(device)]
                if self.shadow_weights and self.channels_last:
                    # stored as the first conv consumes it: NHWC in the compute
                    # dtype (the values the per-step cast + layout change would
                    # produce), so a step gathers 2 B/value and runs no cast
                    f = f.permute(0, 2, 3, 1).to(self.autocast_dtype).contiguous()
                self._feat_cache[key] = f
            self._lab_cache[key] = self._labels.to(device)
        return self._feat_cache[key]

    def init_params(self, seed: int) -> np.ndarray:
        torch.manual_seed(seed)
        m = type(self._template)(self.n_classes)
        return torch.cat([p.detach().reshape(-1) for p in m.parameters()]).double().numpy()

    def make_module(self, device) -> nn.Module:
        m = type(self._template)(self.n_classes).to(device)
        # BatchNorm's num_batches_tracked counter only matters for
        # momentum=None (cumulative averaging); with the fixed momentum used
        # here it is an extra int64 add kernel per BN layer per step
        for mod in m.modules():
            if isinstance(mod, nn.modules.batchnorm._BatchNorm) and mod.momentum is not None:
                mod.num_batches_tracked = None
        if self.channels_last:
            m = m.to(memory_format=torch.channels_last)
        return m

    def bind(self, arena: torch.Tensor, grad_arena: torch.Tensor | None, module: nn.Module | None = None) -> Bound:
        """Parameters become views into ``arena`` (fp32).  With bf16 compute
        (``autocast="bf16"``) the conv / linear weights are instead views
        into a bf16 shadow of the arena that the forward refreshes with ONE
        cast kernel, and the model runs natively in bf16: the same values
        autocast produces (round-to-nearest casts of the same fp32 weights,
        bf16 grads widened exactly into the fp32 gradient arena) without its
        per-tensor cast kernels in forward and backward (44 -> 1 per step)."""
        device = arena.device
        if module is None:
            module = self.make_module(device)
        params = list(module.parameters())
        shadow_dtype = self.autocast_dtype if self.shadow_weights else None
        shadow = (torch.empty(arena.shape[0], dtype=shadow_dtype, device=device)
                  if shadow_dtype is not None else None)
        grad_views = []
        for i, p in enumerate(params):
            lo, hi = self.edges[i], self.edges[i + 1]
            shape = self.param_shapes[i]
            gview = self._view(grad_arena[lo:hi], shape) if grad_arena is not None else None
            if shadow is not None and self._compute_in_shadow[i]:
                p.data = self._view(shadow[lo:hi], shape)
                p.grad = None
            else:
                p.data = self._view(arena[lo:hi], shape)
                if gview is not None:
                    p.grad = gview
            grad_views.append(gview)
            p.requires_grad_(grad_arena is not None)
        cl = self.channels_last

        image_shape = tuple(self.image_shape)
        stem_nchw = self.arch == "resnet20"

        def forward(xb):
            if shadow is not None:
                shadow.copy_(arena)                 # fp32 arena -> bf16 weights, one kernel
            if tuple(xb.shape[1:]) != image_shape:  # NHWC device dataset: a free view
                xb = xb.permute(0, 3, 1, 2)
            if shadow is not None:
                xb = xb.to(shadow_dtype)
            if cl and not (stem_nchw and xb.dtype == torch.float32 and conv_enabled()):
                # (the fp32 ResNet-20 stem reads the gathered NCHW batch itself)
                xb = xb.contiguous(memory_format=torch.channels_last)
            return module(xb)

        b = Bound(params, forward, grad_views=grad_views, mixed=shadow is None)
        b.module = module
        return b

    def _view(self, flat: torch.Tensor, shape):
        if self.channels_last and len(shape) == 4:
            o, i, kh, kw = shape
            return flat.view(o, kh, kw, i).permute(0, 3, 1, 2)
        return flat.view(shape)

    def forward_cost(self) -> int:
        return self._fwd_macs

    def backward_cost(self, block: Block) -> int:
        first, _ = self.tensors_of_block(block)
        # activation grads of every module above the block + weight grads of the block
        return int(sum(2 * m for m in self._tensor_macs[first:]))
