"""Quick start: the reference's fused-optimizer API on a torch model, on a B200.

    python examples/quickstart.py

Backward fusion (updates on a side stream as each layer's gradients complete),
the whole iteration captured as a CUDA graph, a checkpoint, and a resume.
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2104_00237_b200 as optfuse  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def main():
    torch.backends.cudnn.benchmark = True
    # any torch.nn.Module works: optfuse.Graph(module, loss_fn); here a benchmark CNN
    graph = optfuse.build_classifier("mobilenet_v2_cifar", device="cuda", channels_last=True)
    graph.track_counts = False                    # no per-layer Python hooks needed
    policy = optfuse.OptimizerPolicy("sgd-momentum", eta=0.1, alpha=0.9, weight_decay=5e-4,
                                     grad_reset="none")
    x, y = synthetic_batch("mobilenet_v2_cifar", 128, device="cuda")
    x = x.contiguous(memory_format=torch.channels_last)

    def step(inp):
        return optfuse.run_backward_fusion(graph, policy, inp, workers=2, timing=False,
                                           bucket_elems=1 << 20).loss

    cap = optfuse.CapturedStep(step, (x, y), policy=policy, graph=graph)   # warm-up + capture
    for i in range(20):
        loss = cap((x, y))                        # copies the batch in, replays the iteration
    print(f"step {policy.t}: loss {float(loss):.4f}")

    state = optfuse.checkpoint.state_dict(graph, policy)    # flushes pending updates first
    graph2 = optfuse.build_classifier("mobilenet_v2_cifar", device="cuda", channels_last=True)
    policy2 = optfuse.OptimizerPolicy("sgd-momentum", eta=0.1, alpha=0.9, weight_decay=5e-4,
                                      grad_reset="none")
    optfuse.checkpoint.load_state_dict(graph2, policy2, state)
    print(f"resumed at step {policy2.t}")


if __name__ == "__main__":
    main()
