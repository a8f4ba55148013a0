"""Models the schedules run on.

* The reference's synthetic graphs (graph.py:295-342) ported to torch modules
  with the reference's exact initialisation (PCG64 uniform fills seeded by
  ``SeedSequence([seed, pid])``, tensor.py:78-83, graph.py:291-292).  With
  ``exact=True`` the linear layers use the reference's fixed rank-1
  accumulation order (tensor.py:91-104) as separate IEEE multiply and add
  kernels, so a GPU training trajectory is bit-identical to the reference's
  CPU trajectory -- the strongest parity check of the fused path.  With
  ``exact=False`` they use cuBLAS (tolerance parity).
* The benchmark networks named by BASELINE.json (not in the reference, which
  replaces them by synthetic chains): MobileNetV2 / ResNet-18 on
  CIFAR-10 shapes, VGG-16 / ResNet-50 on ImageNet shapes (torchvision), and
  BERT-base pre-training (transformers), all randomly initialised.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F
from torch import nn

from .errors import ConfigError, ShapeError
from .graph import Graph

SYNTHETIC = ("chain", "shared-chain", "mul-probe")
_TORCH_DT = {"f32": torch.float32, "f64": torch.float64}
_NP_DT = {"f32": np.float32, "f64": np.float64}


def _param_seed(seed: int, pid: int) -> int:
    return int(np.random.SeedSequence([seed, pid]).generate_state(1)[0])


def seeded_uniform(shape, lo: float, hi: float, seed: int, precision: str = "f32") -> np.ndarray:
    """Seeded PCG64 uniform fill; bitwise identical to the reference's."""
    if precision not in _NP_DT:
        raise ShapeError(f"unknown precision {precision!r}, expected one of {sorted(_NP_DT)}")
    rng = np.random.Generator(np.random.PCG64(seed))
    vals = rng.uniform(lo, hi, size=int(np.prod(shape)))
    return vals.astype(_NP_DT[precision]).reshape(shape)


def fixed_order_matmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a @ b accumulated one rank-1 product per contraction index, ascending,
    each product and sum a separately rounded IEEE operation (tensor.py:91-105
    order).  On the GPU one kernel (``of_exact_matmul``) computes it; the host
    loop serves the CPU-side tests of the synthetic graphs."""
    if a.is_cuda and a.dtype in (torch.float32, torch.float64) and a.shape[0] <= 65535:
        from . import _native as nat
        from .kernels import _handle
        a = a.contiguous()
        b = b.contiguous()
        out = torch.empty(a.shape[0], b.shape[1], dtype=a.dtype, device=a.device)
        code = nat.OF_F32 if a.dtype == torch.float32 else nat.OF_F64
        st = nat.lib().of_exact_matmul(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.shape[0],
                                       a.shape[1], b.shape[1], code, _handle(None))
        nat.check(st, "of_exact_matmul")
        return out
    out = torch.zeros(a.shape[0], b.shape[1], dtype=a.dtype, device=a.device)
    for k in range(a.shape[1]):
        out = out + a[:, k:k + 1] * b[k:k + 1, :]
    return out


class _ExactLinearReLU(torch.autograd.Function):
    """relu(x @ W) with the reference's arithmetic (graph.py:220-231, :105-124)."""

    @staticmethod
    def forward(ctx, x, w):
        pre = fixed_order_matmul(x, w)
        mask = (pre > 0).to(pre.dtype)
        ctx.save_for_backward(x, w, mask)
        return pre * mask

    @staticmethod
    def backward(ctx, gout):
        x, w, mask = ctx.saved_tensors
        gm = gout * mask
        gw = fixed_order_matmul(x.t(), gm)
        gx = fixed_order_matmul(gm, w.t()) if ctx.needs_input_grad[0] else None
        return gx, gw


class SyntheticLinear(nn.Module):
    """One chain layer: relu(x @ W) (W bound, possibly shared)."""

    def __init__(self, weight: nn.Parameter, exact: bool):
        super().__init__()
        self.weight = weight
        self.exact = exact

    def forward(self, x):
        if self.exact:
            return _ExactLinearReLU.apply(x, self.weight)
        return F.relu(x @ self.weight)


class SyntheticMul(nn.Module):
    """mul-probe node: loss = sum(theta * x) (graph.py:227-229)."""

    def __init__(self, theta: nn.Parameter):
        super().__init__()
        self.theta = theta

    def forward(self, x):
        return self.theta * x


class SyntheticNet(nn.Module):
    def __init__(self, layers):
        super().__init__()
        self.layers = nn.ModuleList(layers)

    def forward(self, x):
        for layer in self.layers:
            x = layer(x)
        return x.sum()


def build_model(model: str, layers: int = 1, width: int = 1, share_groups=None, seed: int = 0,
                precision: str = "f32", init_range=None, device="cuda", exact: bool = True,
                track_input_grad: bool = True) -> Graph:
    """The reference's synthetic graphs (graph.py:295-342) as a torch Graph."""
    if model not in SYNTHETIC:
        raise ConfigError(f"unknown model {model!r}, expected one of {SYNTHETIC}")
    if layers < 1 or width < 1:
        raise ConfigError(f"layers and width must be >= 1, got {layers}, {width}")
    if precision not in _TORCH_DT:
        raise ShapeError(f"unknown precision {precision!r}, expected one of {sorted(_TORCH_DT)}")

    def make(shape, lo, hi, pid):
        arr = seeded_uniform(shape, lo, hi, _param_seed(seed, pid), precision)
        return nn.Parameter(torch.from_numpy(arr).to(device))

    if model == "mul-probe":
        lo, hi = init_range if init_range else (0.5, 1.5)
        net = SyntheticNet([SyntheticMul(make((width,), lo, hi, 0))])
        return Graph(net, None, model=model, precision=precision, width=width,
                     track_input_grad=track_input_grad)

    owner = list(range(layers))
    if model == "shared-chain":
        groups = share_groups if share_groups is not None else [[0, min(2, layers - 1)]]
        seen: set = set()
        for group in groups:
            if len(group) < 2:
                raise ConfigError(f"share group {group} needs at least two layers")
            for idx in group:
                if not 0 <= idx < layers:
                    raise ConfigError(f"share group index {idx} out of range for {layers} layers")
                if idx in seen:
                    raise ConfigError(f"layer {idx} appears in more than one share group")
                seen.add(idx)
            for idx in group:
                owner[idx] = min(group)
    elif share_groups is not None:
        raise ConfigError("share_groups only applies to model 'shared-chain'")

    lo, hi = init_range if init_range else (-1.0 / width ** 0.5, 1.0 / width ** 0.5)
    weights: dict = {}
    mods = []
    for i in range(layers):
        if owner[i] not in weights:
            weights[owner[i]] = make((width, width), lo, hi, len(weights))
        mods.append(SyntheticLinear(weights[owner[i]], exact))
    return Graph(SyntheticNet(mods), None, model=model, precision=precision, width=width,
                 track_input_grad=track_input_grad)


def input_shape(graph: Graph, batch: int = 1) -> tuple:
    return (graph.width,) if graph.model == "mul-probe" else (batch, graph.width)


def make_input(graph: Graph, batch: int, seed: int, device=None) -> torch.Tensor:
    """bench.py:102-103: seeded uniform(0.1, 1.0) input."""
    arr = seeded_uniform(input_shape(graph, batch), 0.1, 1.0, seed, graph.precision)
    return torch.from_numpy(arr).to(device or graph.device)


def iteration_inputs(graph: Graph, batch: int, seed: int, iters: int, device=None) -> list:
    """bench.py:226-228: the verify grid's per-iteration inputs."""
    base = int(np.random.SeedSequence([seed, 9173]).generate_state(1)[0])
    return [make_input(graph, batch, base + i, device) for i in range(iters)]


# ---------------------------------------------------------------------------
# Benchmark networks (BASELINE.json configs)
# ---------------------------------------------------------------------------

def _mobilenet_v2_cifar():
    import torchvision
    return torchvision.models.mobilenet_v2(num_classes=10)


def _resnet18_cifar():
    import torchvision
    m = torchvision.models.resnet18(num_classes=10)
    m.conv1 = nn.Conv2d(3, 64, kernel_size=3, stride=1, padding=1, bias=False)
    m.maxpool = nn.Identity()
    return m


def _vgg16():
    import torchvision
    return torchvision.models.vgg16()


def _resnet50():
    import torchvision
    return torchvision.models.resnet50()


# name -> (constructor, per-sample input shape, number of classes)
CLASSIFIERS = {
    "mobilenet_v2_cifar": (_mobilenet_v2_cifar, (3, 32, 32), 10),
    "resnet18_cifar": (_resnet18_cifar, (3, 32, 32), 10),
    "vgg16": (_vgg16, (3, 224, 224), 1000),
    "resnet50": (_resnet50, (3, 224, 224), 1000),
}


class BertPretraining(nn.Module):
    """BERT-base pre-training model (C5): ``transformers.BertForPreTraining``
    with the default BertConfig (12 layers, hidden 768, vocab 30522), random
    init, returning both heads' logits.  The MLM decoder weight is tied to the
    word embeddings (and the decoder bias to the head bias): one Parameter
    bound to two layers, the reference's shared-parameter case."""

    def __init__(self, **config):
        super().__init__()
        from transformers import BertConfig, BertForPreTraining
        self.net = BertForPreTraining(BertConfig(**config))

    def forward(self, ids):
        out = self.net(input_ids=ids, return_dict=True)
        return out.prediction_logits, out.seq_relationship_logits


def bert_pretraining_loss(out, target):
    """Masked-LM cross entropy (label -100 = not masked) + next-sentence CE."""
    mlm, nsp = out
    labels, nsp_labels = target
    return (F.cross_entropy(mlm.reshape(-1, mlm.shape[-1]).float(), labels.reshape(-1),
                            ignore_index=-100)
            + F.cross_entropy(nsp.float(), nsp_labels))


BERT_SEQ = 128
BERT_VOCAB = 30522

# non-classifier networks: name -> (constructor, loss)
NETWORKS = {"bert_base": (BertPretraining, bert_pretraining_loss)}


def build_classifier(name: str, device="cuda", dtype=torch.float32, seed: int = 0,
                     channels_last: bool = False, **graph_kw) -> Graph:
    """A randomly initialised benchmark network as a Graph: the CNNs with a
    cross-entropy loss, ``bert_base`` with the pre-training loss."""
    if name not in CLASSIFIERS and name not in NETWORKS:
        raise ConfigError(f"unknown network {name!r}, expected one of "
                          f"{sorted(CLASSIFIERS) + sorted(NETWORKS)}")
    torch.manual_seed(seed)
    if name in NETWORKS:
        ctor, loss = NETWORKS[name]
        cfg = graph_kw.pop("config", None) or {}
        return Graph(ctor(**cfg).to(device=device, dtype=dtype), loss, model=name, **graph_kw)
    net = CLASSIFIERS[name][0]().to(device=device, dtype=dtype)
    if channels_last:
        net = net.to(memory_format=torch.channels_last)
    return Graph(net, F.cross_entropy, model=name, **graph_kw)


def synthetic_batch(name: str, batch: int, device="cuda", dtype=torch.float32, seed: int = 0,
                    seq: int = BERT_SEQ, vocab: int = BERT_VOCAB):
    """CNNs: x ~ N(0, 1), y ~ U{0..classes-1}.
    bert_base: ids ~ U{0..30521} [b, 128], 15% of positions carry an MLM label
    (the original id), the rest -100; next-sentence labels ~ U{0, 1}."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    if name == "bert_base":
        ids = torch.randint(0, vocab, (batch, seq), generator=g)
        masked = torch.rand((batch, seq), generator=g) < 0.15
        labels = torch.where(masked, ids, torch.full_like(ids, -100))
        nsp = torch.randint(0, 2, (batch,), generator=g)
        return ids.to(device), (labels.to(device), nsp.to(device))
    _, shape, classes = CLASSIFIERS[name]
    x = torch.randn((batch,) + shape, generator=g).to(device=device, dtype=dtype)
    y = torch.randint(0, classes, (batch,), generator=g).to(device)
    return x, y
