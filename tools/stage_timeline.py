"""Per-stage device timeline of the fused collectives (run under torchrun):
qwZ (quantize | barrier | NVLink gather) and qgZ at S=1 (K1 | group barrier |
K2 | cross barrier | K3), from the communicator's stage tracer (CUDA events
between the launches, on the collective's stream).  Prints one JSON object
per rank: the median over 10 traced calls of each stage's duration.

    python -m torch.distributed.run --nproc-per-node N tools/stage_timeline.py [group_size]
"""

import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp  # noqa: E402
from paper_2306_10209_b200.dist import Communicator  # noqa: E402

M = 1_300_004_864
BUCKET = 134_217_728


def stages(trace):
    out, prev = [], 0.0
    for name, t in trace[1:]:
        out.append((name, t - prev))
        prev = t
    return out


def med(runs):
    keys = [f"{i}:{n}" for i, (n, _) in enumerate(runs[0])]
    return {k: round(statistics.median(r[i][1] for r in runs) * 1e3, 1) for i, k in enumerate(keys)} | \
        {"total_us": round(statistics.median(sum(d for _, d in r) for r in runs) * 1e3, 1)}


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    X = int(sys.argv[1]) if len(sys.argv) > 1 else min(world, 4)
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(rank)
    comm = Communicator(group_size=X, qwz_shard=M // world, qgz_elems=BUCKET, qgz_stages=1,
                        qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    shard = (torch.randn(M // world, generator=g, device=dev) * 0.02).half()
    out = torch.empty(M, dtype=torch.float16, device=dev)
    grad = (torch.randn(BUCKET, generator=g, device=dev) * 1e-3).bfloat16()
    part = torch.empty(BUCKET // world, dtype=torch.float32, device=dev)
    res = {"rank": rank, "world": world, "groups": f"{world // X}x{X}"}
    for name, fn in (("qwz_us", lambda: comm.qwz_allgather(shard, out=out)),
                     ("qgz_us", lambda: comm.qgz_reduce_scatter(grad, out=part))):
        for _ in range(3):
            fn()
        comm.trace(True)
        runs = []
        for _ in range(10):
            dist.barrier()
            torch.cuda.synchronize()
            fn()
            runs.append(stages(comm.trace_read()))
        comm.trace(False)
        res[name] = med(runs)
    comm.check()
    comm.close()
    outs = [None] * world
    dist.all_gather_object(outs, res)
    if rank == 0:
        for r in outs:
            print(json.dumps(r), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
