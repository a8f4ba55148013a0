import sys, torch
print("start", flush=True)
import paper_2104_00237_b200 as of
from paper_2104_00237_b200 import _native
print("lib", _native.lib(), flush=True)
p = torch.randn(1000, device="cuda"); p.grad = torch.randn(1000, device="cuda")
pol = of.OptimizerPolicy("sgd-momentum", eta=0.1, alpha=0.9)
class P: pass
print("step...", flush=True)
g = of.build_model("chain", layers=3, width=8, seed=0, device="cuda:0")
print("model", flush=True)
x = of.iteration_inputs(g, 4, 0, 1)[0]
of.run_baseline(g, pol, x)
torch.cuda.synchronize()
print("baseline ok", flush=True)
of.run_backward_fusion(g, pol, x, workers=2)
torch.cuda.synchronize()
print("bf ok", flush=True)
