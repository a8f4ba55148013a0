"""Where does the per-instance step-time spread come from (diagnostic)?  One
model instance, captured several times (fresh CUDA graph each time) vs
fresh instances; graphed channels-last MobileNetV2, forward+backward only."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import bench  # noqa: E402
import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.graphs import CapturedStep  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def main():
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda", 0)
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    x, y = synthetic_batch("mobilenet_v2_cifar", 128, device=dev)
    x = x.contiguous(memory_format=torch.channels_last)
    out = {"same_instance_recaptured": [], "fresh_instances": []}
    g = of.build_classifier("mobilenet_v2_cifar", device=dev, channels_last=True)
    net = g.module

    def run(inp):
        for p in net.parameters():
            p.grad = None
        loss = F.cross_entropy(net(inp[0]), inp[1])
        loss.backward()
        return loss
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    keep = []
    for _ in range(n):
        cap = CapturedStep(run, (x, y), warmup=3)
        out["same_instance_recaptured"].append(round(bench.timed(cap, 30, 10, dist, buf.zero_), 4))
        keep.append(cap)       # alive: every capture gets its own pool and stream
    # the captures again, in order: is the mode a property of the captured graph?
    out["recaptured_retimed"] = [round(bench.timed(c, 30, 10, dist, buf.zero_), 4) for c in keep]
    del keep
    for _ in range(n):
        g2 = of.build_classifier("mobilenet_v2_cifar", device=dev, channels_last=True)
        net = g2.module
        cap = CapturedStep(run, (x, y), warmup=3)
        out["fresh_instances"].append(round(bench.timed(cap, 30, 10, dist, buf.zero_), 4))
        del cap, g2
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
