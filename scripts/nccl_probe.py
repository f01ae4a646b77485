import os, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
t = torch.tensor([float(rank + 1)], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
print("rank", rank, "allreduce", t.item(), flush=True)
dist.destroy_process_group()
