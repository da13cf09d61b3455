"""Host<->device copy bandwidth per rank with all ranks copying at once
(torchrun; pinned host buffers): the ceiling of bench.py's e2e number."""
import json
import os

import torch
import torch.distributed as dist

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
world = int(os.environ.get("WORLD_SIZE", 1))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
M = 1_300_004_864
res = {"world": world}
for name, nbytes, mode in (("h2d_shard", 2 * M // world, "h2d"), ("d2h_full", 2 * M, "d2h"),
                           ("both", 2 * M, "both")):
    h = torch.empty(nbytes // 2, dtype=torch.float16).pin_memory()
    d = torch.empty(nbytes // 2, dtype=torch.float16, device="cuda")
    h2 = torch.empty(M // world, dtype=torch.float16).pin_memory() if mode == "both" else None
    d2 = torch.empty(M // world, dtype=torch.float16, device="cuda") if mode == "both" else None
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def step():
        if mode == "h2d":
            d.copy_(h, non_blocking=True)
        elif mode == "d2h":
            h.copy_(d, non_blocking=True)
        else:
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s1):
                h.copy_(d, non_blocking=True)
            with torch.cuda.stream(s2):
                d2.copy_(h2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(3):
        step()
    b.record()
    b.synchronize()
    tt = torch.tensor([a.elapsed_time(b) / 3 / 1e3], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    res[name] = {"ms": t * 1e3, "GBps_per_rank": nbytes / t / 1e9}
    del h, d, h2, d2
if local == 0:
    print(json.dumps(res), flush=True)
if world > 1:
    dist.destroy_process_group()
