"""Can two NCCL ranks share one GPU on this box?  (For exercising the
multi-rank path with the single GPU gpurun provides.)"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
t = torch.ones(4, device="cuda") * (rank + 1)
try:
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print(f"rank {rank}: all_reduce ok -> {t.tolist()}", flush=True)
except Exception as e:
    print(f"rank {rank}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)
dist.destroy_process_group()
