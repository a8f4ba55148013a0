"""Workloads for ncu captures of the update kernel (run under ncu, never timed).

    python tools/profile_kernels.py bf      # MobileNetV2 b128 backward fusion, bucketed launches
    python tools/profile_kernels.py vgg     # one multi-tensor Adam launch over VGG-16 (138 M params)
    python tools/profile_kernels.py bert    # one AdamW launch over BERT-base (206 tensors, 110 M)
    python tools/profile_kernels.py r50mixed  # ResNet-50 bf16 + fp32 masters, AdamW, one launch
    python tools/profile_kernels.py c2full  # one SGD-momentum launch over MobileNetV2 (158 tensors, 2.24 M)
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def bf(iters=6):
    g = of.build_classifier("mobilenet_v2_cifar", device="cuda", channels_last=True)
    g.track_counts = False
    pol = of.OptimizerPolicy("sgd-momentum", eta=0.1, alpha=0.9, weight_decay=5e-4, grad_reset="none")
    x, y = synthetic_batch("mobilenet_v2_cifar", 128, device="cuda")
    x = x.contiguous(memory_format=torch.channels_last)
    for _ in range(iters):
        of.run_backward_fusion(g, pol, (x, y), workers=2, bucket_elems=1 << 20, timing=False)  # headline groups
    torch.cuda.synchronize()


def vgg(iters=3, model="vgg16", kind="adam", mixed=False):
    g = of.build_classifier(model, device="cuda")
    if mixed:
        g.use_master_weights()
    pol = of.OptimizerPolicy(kind, eta=1e-4, grad_reset="none")
    for p in g.parameters:
        p.value.grad = torch.randn_like(p.value) * 0.01
    for _ in range(iters):
        pol.begin_iteration()
        for p in g.parameters:
            if p.value.grad is None:
                p.value.grad = torch.randn_like(p.value) * 0.01
        pol.step_params(g.parameters)
    torch.cuda.synchronize()


def bert(iters=3):
    vgg(iters, "bert_base", "adamw")


def r50mixed(iters=3):
    vgg(iters, "resnet50", "adamw", mixed=True)


def c2full(iters=3):
    vgg(iters, "mobilenet_v2_cifar", "sgd-momentum")


if __name__ == "__main__":
    {"bf": bf, "vgg": vgg, "bert": bert, "r50mixed": r50mixed, "c2full": c2full}[sys.argv[1]]()
