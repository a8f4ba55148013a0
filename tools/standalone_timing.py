"""How the standalone update-kernel timing depends on the method (diagnostic):
one pass after a 2 ms or 10 ms GPU sleep (the host builds the tensor list
meanwhile), and 3 back-to-back passes per event pair (parameter sets >> L2)."""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.optim import algorithmic_bytes  # noqa: E402


def main():
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for name, model, kind in (("vgg16_adam", "vgg16", "adam"), ("bert_base_adamw", "bert_base", "adamw")):
        g = of.build_classifier(model, device=dev)
        pol = of.OptimizerPolicy(kind, eta=1e-4, weight_decay=0.01 if kind == "adamw" else 0.0,
                                 grad_reset="zero")
        params = g.parameters
        for p in params:
            p.value.grad = torch.randn_like(p.value) * 0.01
        nbytes = algorithmic_bytes(kind, params)
        row = {}
        for label, sleep, passes in (("sleep2ms_x1", 4_000_000, 1), ("sleep10ms_x1", 20_000_000, 1),
                                     ("sleep10ms_x3", 20_000_000, 3)):
            ts = []
            for i in range(6):
                flush.zero_()
                flush.sum()
                torch.cuda._sleep(sleep)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(passes):
                    pol.begin_iteration()
                    pol.step_params(params)
                e1.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1) / passes)
            us = statistics.median(ts) * 1e3
            row[label] = {"us": round(us, 1), "TBps": round(nbytes / us / 1e6, 3)}
        out[name] = row
        del g, params
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def torch_fused():
    """torch.optim.Adam(fused=True) / SGD(fused) one step over the same sets, same protocol."""
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for name, model, opt_name, kw, bpe in (("vgg16_adam", "vgg16", "Adam", {"lr": 1e-4}, 28),
                                          ("bert_base_adamw", "bert_base", "AdamW",
                                           {"lr": 1e-4, "weight_decay": 0.01}, 28)):
        g = of.build_classifier(model, device=dev)
        ps = [p.value for p in g.parameters]
        for p in ps:
            p.grad = torch.randn_like(p) * 0.01
        opt = getattr(torch.optim, opt_name)(ps, fused=True, **kw)
        opt.step()
        n = sum(p.numel() for p in ps)
        ts = []
        for i in range(6):
            flush.zero_()
            flush.sum()
            torch.cuda._sleep(20_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            opt.step()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        us = statistics.median(ts) * 1e3
        out[name + "_torch_fused"] = {"us": round(us, 1), "TBps": round(n * bpe / us / 1e6, 3)}
        del g, ps, opt
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "torch":
    torch_fused()
