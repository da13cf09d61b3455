"""qwZ fused all-gather sweep (torchrun): step time and NVLink ingress per GPU."""
import json, os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp
from paper_2306_10209_b200.dist import Communicator, nccl_allgather
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
M = 1_300_004_864; n = M // world
comm = Communicator(qwz_shard=n)
x = (torch.randn(n, device="cuda") * 0.02).half(); out = torch.empty(M, dtype=torch.float16, device="cuda")
def timed(fn, steps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); dist.barrier()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record()
    for _ in range(steps): fn()
    e.record(); e.synchronize()
    t = torch.tensor([s.elapsed_time(e) / steps], device="cuda", dtype=torch.float64); dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
t = timed(lambda: comm.qwz_allgather(x, out=out)); comm.check()
ingress = (world - 1) * (n + n // 2048 * 4)
if rank == 0:
    print(json.dumps({"world": world, "ms": t,
                      "GBps_value": world * 2 * M / t / 1e6, "ingress_GBps_step": ingress / t / 1e6}), flush=True)
comm.close(); dist.destroy_process_group()
