"""One training iteration per schedule under an NVTX range, for ncu's
whole-iteration DRAM-traffic accounting (the GPU form of the reference's
locality model, locality.py:66-89 simulate_cache / transaction_count, and
SPEC acceptance #5: fused schedules touch fewer parameter lines).

    python tools/iter_dram.py <config> <schedule>
      config:   c3 (VGG-16 Adam b32) | c4 (ResNet-50 bf16+master AdamW b64)
                | c5 (BERT-base AdamW b32) | c2 (MobileNetV2 SGD-m b128)
      schedule: baseline | bf1 (inline, per layer) | bf2 (side stream, per layer)
                | ff (per layer)

Three warm-up iterations, then ONE iteration inside the NVTX range "iter"
(start/end range: process-wide, so autograd's thread is included).  Run it
under tools/iter_dram.sh (ncu --nvtx --nvtx-include "iter" ... with
--cache-control none, so each kernel sees the L2 its predecessors left).
True fp32 (TF32 off) like the headline.
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def main():
    cfg, sched = sys.argv[1], sys.argv[2]
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    wl = bench.WORKLOADS[cfg]
    g = of.build_classifier(wl["model"], device="cuda", channels_last=cfg in ("c2", "c4"))
    g.track_counts = False
    x, y = synthetic_batch(wl["model"], wl["batch"], device="cuda")
    if cfg in ("c2", "c4") and x.dim() == 4:
        x = x.contiguous(memory_format=torch.channels_last)
    if wl.get("mixed"):
        g.use_master_weights()
        x = x.to(torch.bfloat16)
    pol = of.OptimizerPolicy(wl["kind"], **wl["hp"], grad_reset="none")
    inp = (x, y)

    def step():
        if sched == "baseline":
            of.run_baseline(g, pol, inp, timing=False)
        elif sched == "bf1":
            of.run_backward_fusion(g, pol, inp, workers=1, timing=False)
        elif sched == "bf2":
            of.run_backward_fusion(g, pol, inp, workers=2, timing=False)
        elif sched == "ff":
            of.run_forward_fusion(g, pol, inp, timing=False)
        else:
            raise SystemExit(f"unknown schedule {sched}")
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    r = torch.cuda.nvtx.range_start("iter")
    step()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_end(r)
    from paper_2104_00237_b200.optim import algorithmic_bytes
    print(f"{cfg} {sched}: update algorithmic bytes {algorithmic_bytes(pol.kind, g.parameters)}")


if __name__ == "__main__":
    main()
