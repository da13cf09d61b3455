"""Time Communicator.qgz_reduce_scatter_stream over NB 256 MiB bf16 buckets
(INT4/512, S = 1) at the torchrun world size, max over ranks, and check a
sample of the outputs bitwise against the oracle.  Env ZPP_QGZ_XB /
ZPP_QGZ_K1_XB_SMS select the cross-bucket overlap (tools/qgz_xb_sweep.sh).

    torchrun --nproc-per-node N tools/qgz_stream_probe.py X NB
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

BUCKET = 134_217_728


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    X = int(sys.argv[1]) if len(sys.argv) > 1 else world
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    comm = Communicator(group_size=X, qgz_elems=BUCKET, qgz_stages=S, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    grads = torch.empty(nb * BUCKET, dtype=torch.bfloat16, device=dev)
    for b in range(nb):
        synth.device(2000 + 1000 * rank + b, 0, BUCKET, torch.bfloat16, "grad", out=grads[b * BUCKET:(b + 1) * BUCKET])
    out = torch.empty(nb * BUCKET // world, dtype=torch.float32, device=dev)
    for _ in range(2):
        comm.qgz_reduce_scatter_stream(grads, out=out)
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    s.record()
    for _ in range(reps):
        comm.qgz_reduce_scatter_stream(grads, out=out)
    e.record()
    e.synchronize()
    t = torch.tensor([s.elapsed_time(e) / reps / nb * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    comm.check()
    per = BUCKET // world
    chk = bad = 0
    for b in range(nb):
        c, m = sampled.qgz_check(out[b * per:(b + 1) * per], rank, world, X, BUCKET, stages=S, seed_base=2000 + b,
                                 samples=128, rng_seed=b)
        chk, bad = chk + c, bad + m
    v = torch.tensor([chk, bad], dtype=torch.float64, device=dev)
    dist.all_reduce(v)
    if rank == 0:
        print(json.dumps({"world": world, "X": X, "buckets": nb, "stages": S, "xb": os.environ.get("ZPP_QGZ_XB", "1"),
                          "k1_sms": os.environ.get("ZPP_QGZ_K1_XB_SMS", "default"),
                          "k1_stage_sms": os.environ.get("ZPP_QGZ_K1_SMS", "default"), "us_per_bucket": t.item(),
                          "checked": int(v[0]), "mismatches": int(v[1])}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
