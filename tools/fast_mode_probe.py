"""Diagnostic: what puts a model instance in the ~7% "fast mode"?  Builds the
headline step (graphed BF) repeatedly, each after an allocator perturbation,
times it three times (is the mode a property of the instance?) and records the
addresses of a few of its buffers and the memory clock."""
import gc
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import pynvml  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    args = bench.parse_args([])
    args.world, args.dp = 1, False
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    keep = []
    out = []
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
    for i in range(n):
        if i % 2 == 1:      # perturb the allocator: a live block of i MiB
            keep.append(torch.empty(i << 20, dtype=torch.uint8, device=dev))
        step, g, pol = bench.make_runner(args, args.batch, args.schedule, dev)
        ts = [bench.timed(step, 20, 5, dist, buf.zero_) for _ in range(3)]
        ps = g.parameters
        p0 = ps[0] if ps else None
        rec = {"i": i, "ms": [round(t, 4) for t in ts],
               "mem_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
               "sm_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
               "alloc_mb": torch.cuda.memory_allocated() >> 20,
               "reserved_mb": torch.cuda.memory_reserved() >> 20}
        if p0 is not None:
            rec["param0"] = hex(getattr(p0, "value", p0).data_ptr())
        sx = getattr(step, "static_inputs", None) or getattr(step, "_static", None)
        if sx is not None:
            try:
                rec["x"] = hex(sx[0].data_ptr())
            except Exception:  # noqa: BLE001
                pass
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del step, g, pol
        if "--gc" in sys.argv:
            gc.collect()
            rec["alloc_mb_after_gc"] = torch.cuda.memory_allocated() >> 20
            by_stream = {}
            for seg in torch.cuda.memory._snapshot()["segments"]:
                live = sum(b["size"] for b in seg["blocks"] if b["state"] == "active_allocated")
                if live:
                    k = hex(seg["stream"])
                    by_stream[k] = by_stream.get(k, 0) + (live >> 20)
            rec["live_mb_by_stream"] = by_stream
            print(json.dumps(rec), flush=True)
        if i % 3 == 2:
            torch.cuda.empty_cache()
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/fmode.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
