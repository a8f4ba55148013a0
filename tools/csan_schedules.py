"""Run the fused schedules under PyTorch's CUDA stream sanitizer (CSAN).

    TORCH_CUDA_SANITIZER=1 python tools/csan_schedules.py

CSAN intercepts every torch operator and checks that no tensor is read on one
stream while another stream may still be writing it (and vice versa) without
an event/stream dependency.  What it sees here: every torch-side access of
the fused schedules -- the forward/backward kernels on the compute stream,
gradient allocation and release around the side-stream updates, the
forward-fusion lookahead, the data-parallel flat-buffer copies and NCCL
collectives on the communication stream.  What it cannot see: the update
kernels themselves (launched through the C ABI, not the dispatcher) --
tests/test_race_guard_gpu.py covers those adversarially.  CSAN raises on the
first unsynchronized access; a clean run prints one line per workload.
"""

import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402

TINY_BERT = dict(num_hidden_layers=2, hidden_size=64, num_attention_heads=4, intermediate_size=128,
                 vocab_size=512, max_position_embeddings=64, attn_implementation="sdpa")


def workloads():
    def mobilenet():
        g = of.build_classifier("mobilenet_v2_cifar", device="cuda", channels_last=True)
        g.track_counts = False
        x, y = synthetic_batch("mobilenet_v2_cifar", 32, device="cuda")
        return g, (x.contiguous(memory_format=torch.channels_last), y), "sgd-momentum"

    def bert():
        g = of.build_classifier("bert_base", device="cuda", config=TINY_BERT)
        g.track_counts = False
        inp = synthetic_batch("bert_base", 4, device="cuda", seq=32, vocab=512)
        return g, inp, "adamw"
    return {"mobilenet_v2": mobilenet, "tiny_bert": bert}


def main() -> int:
    assert os.environ.get("TORCH_CUDA_SANITIZER") == "1", "run with TORCH_CUDA_SANITIZER=1"
    for name, make in workloads().items():
        for sched in ("backward-fusion w=2", "backward-fusion w=2 bucketed",
                      "forward-fusion prefetch", "baseline"):
            g, inp, kind = make()
            pol = of.OptimizerPolicy(kind, eta=1e-3, weight_decay=1e-4, grad_reset="none")
            for _ in range(4):
                if sched.startswith("backward"):
                    of.run_backward_fusion(g, pol, inp, workers=2, timing=False,
                                           bucket_elems=(1 << 18) if "bucketed" in sched else 0)
                elif sched.startswith("forward"):
                    of.run_forward_fusion(g, pol, inp, timing=False, bucket_elems=1 << 18,
                                          prefetch=1)
                else:
                    of.run_baseline(g, pol, inp, timing=False)
            of.flush_pending_updates(g, pol)
            torch.cuda.synchronize()
            print(f"csan clean: {name} {sched}", flush=True)
    # data parallel (world 1, NCCL): flat buffers + collectives on the comm stream
    import torch.distributed as dist

    from paper_2104_00237_b200.dp import DataParallelFusion
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for name, make in workloads().items():
            for sched in ("backward-fusion", "forward-fusion"):
                g, inp, kind = make()
                pol = of.OptimizerPolicy(kind, eta=1e-3, weight_decay=1e-4)
                dpf = DataParallelFusion(g, pol, bucket_elems=1 << 18)
                run = dpf.run_backward_fusion if sched == "backward-fusion" else dpf.run_forward_fusion
                for _ in range(4):
                    run(inp)
                dpf.flush()
                torch.cuda.synchronize()
                print(f"csan clean: {name} data-parallel {sched}", flush=True)
    finally:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
