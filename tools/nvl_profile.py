"""Workload for the one-rank ncu capture under real peer traffic
(tools/ncu_rank0.sh): the qwZ gather at the GPT-13B-layer shard, the qgZ
256 MiB bucket (pull K2 with one group, push K1 with two).  Every rank runs the
same calls; a host barrier (gloo, no GPU kernels) follows each call so peers
sit idle on the host while rank 0's kernels are replayed by ncu, and their
symmetric buffers stay unchanged during the replays.

    RANK=r WORLD_SIZE=N LOCAL_RANK=r MASTER_ADDR=127.0.0.1 MASTER_PORT=P python tools/nvl_profile.py X
"""

import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp  # noqa: E402
from oracle import synth  # noqa: E402
from paper_2306_10209_b200.dist import Communicator  # noqa: E402

BUCKET = 134_217_728


def say(msg):
    print(f"[rank {os.environ.get('RANK')}] {msg}", flush=True)


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    say("init")
    dist.init_process_group("gloo")
    say("gloo up")
    rank, world = dist.get_rank(), dist.get_world_size()
    X = int(sys.argv[1]) if len(sys.argv) > 1 else world
    dev = torch.device("cuda", local)
    h = 5120
    layer_p = -(-(12 * h * h + 13 * h) // (world * 8192)) * world * 8192
    comm = Communicator(group_size=X, qwz_shard=layer_p // world, qgz_elems=BUCKET, qgz_stages=1,
                        qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    w = synth.device(3000 + rank, 0, layer_p // world, torch.float16, "weight", device=dev)
    g = synth.device(2000 + 1000 * rank, 0, BUCKET, torch.bfloat16, "grad", device=dev)
    out = torch.empty(layer_p, dtype=torch.float16, device=dev)
    part = torch.empty(BUCKET // world, dtype=torch.float32, device=dev)

    def fence():
        torch.cuda.synchronize()
        dist.barrier()

    say("inputs ready")
    for _ in range(2):  # warm-up (not profiled: ncu -k filters + launch skip in ncu_rank0.sh)
        comm.qwz_allgather(w, out=out)
        comm.qgz_reduce_scatter(g, out=part)
    fence()
    say("warm-up done")
    comm.qwz_allgather(w, out=out)
    fence()
    say("gather done")
    comm.qgz_reduce_scatter(g, out=part)
    fence()
    say("qgz done")
    comm.check()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
