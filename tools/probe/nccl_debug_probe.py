import os, torch, torch.distributed as dist
os.environ.setdefault("NCCL_DEBUG", "INFO"); os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
if len(os.sys.argv) > 1: os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29577", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
t = torch.ones(4, device="cuda"); dist.all_reduce(t); torch.cuda.synchronize()
print("done", t.sum().item())
dist.destroy_process_group()
