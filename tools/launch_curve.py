"""Update-kernel duration vs launch size (single fp32 tensor, SGD-momentum and
Adam), back-to-back launches on one stream, L2 flushed before each timed
sequence: where the multi-tensor kernel leaves the latency floor and reaches
the HBM roofline.  Prints one JSON line.

    python tools/launch_curve.py
"""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.optim import bytes_per_element  # noqa: E402


def main():
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for kind in ("sgd-momentum", "adam"):
        bpe = bytes_per_element(kind, 4)
        rows = []
        for mb in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024):
            n = (mb << 20) // bpe // 4 * 4
            # distinct parameters covering >= 384 MiB, launched round-robin: every
            # launch finds its operands cold (out of the 126 MB L2)
            k = max(1, (384 << 20) // (mb << 20))
            ps = [of.Parameter(i, torch.nn.Parameter(torch.randn(n, device=dev))) for i in range(k)]
            pol = of.OptimizerPolicy(kind, eta=1e-4, grad_reset="none")   # no extra zero write
            grads = [torch.randn(n, device=dev) * 0.01 for _ in ps]

            def step(i):
                ps[i].value.grad = grads[i]
                pol.step(ps[i])
            for i in range(k):
                pol.begin_iteration()
                step(i)
            reps = max(k, 8)
            ts = []
            for _ in range(3):
                flush.zero_()
                flush.sum()
                torch.cuda._sleep(200_000_000)   # ~0.1 s: the host enqueues the whole sequence first
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for r in range(reps):
                    step(r % k)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / reps * 1e3)
            us = statistics.median(ts)
            rows.append({"MB": round(n * bpe / 1e6, 2), "us": round(us, 2),
                         "GBs": round(n * bpe / us / 1e3, 1)})
            del ps
            torch.cuda.empty_cache()
        out[kind] = rows
    print(json.dumps(out))


if __name__ == "__main__":
    main()
