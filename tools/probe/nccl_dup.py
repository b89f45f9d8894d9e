"""Probe: can two NCCL ranks share one GPU (ncclCommInitRank on the same device)?"""
import os, torch, torch.distributed as dist
rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
x = torch.full((4,), rank + 1.0, device="cuda")
try:
    dist.all_reduce(x)
    torch.cuda.synchronize()
    print(f"rank {rank}: all_reduce ok -> {x.tolist()}", flush=True)
except Exception as e:
    print(f"rank {rank}: FAILED {type(e).__name__}: {e}", flush=True)
dist.destroy_process_group()
