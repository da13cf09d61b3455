"""Forward qwZ over a GPT-13B layer stack (40 layers, h = 5120): every layer
gathered with (prefetch) or without (plain) the next layer's quantization
prefetched on the side stream.  Max over ranks, CUDA events; sampled parity
of the last layer.  Env ZPP_QWZ_PREFETCH_SMS sets the prefetch SM budget
(tools/prefetch_sweep.sh).

    torchrun --nproc-per-node N tools/qwz_layers_probe.py
"""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp  # noqa: E402
from oracle import sampled, synth  # noqa: E402
from paper_2306_10209_b200.dist import Communicator  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    h, n_layers = 5120, 40
    layer = 12 * h * h + 13 * h
    layer_p = -(-layer // (world * 8192)) * world * 8192
    shard = layer_p // world
    comm = Communicator(group_size=min(world, 4), qwz_shard=shard, qwz_cfg=zpp.QuantConfig(bit_width=8, block_size=2048))
    ws = [synth.device(3000 + 100 * i + rank, 0, shard, torch.float16, "weight", device=dev) for i in range(n_layers)]
    out = torch.empty(layer_p, dtype=torch.float16, device=dev)

    def fwd(prefetch):
        for i in range(n_layers):
            comm.qwz_allgather(ws[i], out=out, next_shard=ws[i + 1] if prefetch and i + 1 < n_layers else None)

    res = {}
    for name, pf in (("plain", False), ("prefetch", True), ("plain2", False), ("prefetch2", True)):
        fwd(pf)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            fwd(pf)
        e.record()
        e.synchronize()
        t = torch.tensor([s.elapsed_time(e) / 3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = t.item()
    comm.check()
    c, b = sampled.qwz_check(out, world, shard, seed_base=3000 + 100 * (n_layers - 1), samples=512, rng_seed=rank)
    v = torch.tensor([c, b], dtype=torch.float64, device=dev)
    dist.all_reduce(v)
    if rank == 0:
        alg = n_layers * (world - 1) * (shard + shard // 2048 * 4)
        print(json.dumps({"world": world, "sms": os.environ.get("ZPP_QWZ_PREFETCH_SMS", "default"),
                          "ms": res, "ingress_GBps_prefetch": alg / (min(res["prefetch"], res["prefetch2"]) * 1e-3) / 1e9,
                          "checked": int(v[0]), "mismatches": int(v[1])}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
