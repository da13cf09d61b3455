"""Per-rank worker: the fused NVLink collectives at the BASELINE shapes, with
sampled bitwise parity against the oracle (launched by torchrun from
tests/test_gpu_dist.py, one process per GPU).

* qwZ INT8/2048 all-gather of the 1.3B fp16 buffer (configs[1]),
* qgZ INT4/512 2-hop reduce-scatter of a 256 MiB bf16 bucket (configs[3]),
* one GPT-13B layer (configs[4]): qwZ with the hpZ write-through, the hpZ
  group gather, and qgZ with S = 2.

Inputs come from the counter-based generator (oracle/synth.py) on the device;
every rank checks >= 4096 random 2048-blocks of its gathered weights and
>= 4096 random 512-element slices of its reduced gradients bitwise against the
oracle recomputed from the seeded inputs of exactly those positions
(oracle/sampled.py).  Each collective runs several times back to back with no
host synchronisation in between, so both halves of every double buffer are
exercised under real concurrency before the check."""

import argparse
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_10209_b200 as zpp  # noqa: E402
from oracle import sampled, synth  # noqa: E402
from paper_2306_10209_b200.dist import Communicator  # noqa: E402

M_PARAMS = 1_300_004_864
QGZ_BUCKET = 134_217_728


def _pad(n, a):
    return (n + a - 1) // a * a


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--group", type=int, default=2)
    ap.add_argument("--samples", type=int, default=4096)
    ap.add_argument("--cases", default="qwz,qgz,layer,stream")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    oversub = os.environ.get("ZPP_OVERSUBSCRIBE") == "1"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", local)
    X = args.group
    cases = args.cases.split(",")
    report = []

    def record(name, checked, bad):
        report.append((name, checked, bad))

    # ---- qwZ: 1.3B fp16, INT8/2048 ------------------------------------------------
    if "qwz" in cases:
        shard_len = M_PARAMS // world
        comm = Communicator(group_size=X, qwz_shard=shard_len, qwz_cfg=zpp.QuantConfig(bit_width=8, block_size=2048))
        shard = synth.device(1000 + rank, 0, shard_len, torch.float16, "weight", device=dev)
        out = torch.empty(M_PARAMS, dtype=torch.float16, device=dev)
        for _ in range(3):
            comm.qwz_allgather(shard, out=out)
        comm.check()
        record("qwz 1.3B", *sampled.qwz_check(out, world, shard_len, samples=args.samples, rng_seed=rank))
        del out, shard
        comm.close()
        torch.cuda.empty_cache()

    # ---- qgZ: 256 MiB bf16 bucket, INT4/512 --------------------------------------
    if "qgz" in cases:
        comm = Communicator(group_size=X, qgz_elems=QGZ_BUCKET, qgz_stages=1,
                            qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
        grad = synth.device(2000 + 1000 * rank, 0, QGZ_BUCKET, torch.bfloat16, "grad", device=dev)
        o32 = torch.empty(QGZ_BUCKET // world, dtype=torch.float32, device=dev)
        o64 = torch.empty(QGZ_BUCKET // world, dtype=torch.float64, device=dev)
        for _ in range(2):
            comm.qgz_reduce_scatter(grad, out=o64)
            comm.qgz_reduce_scatter(grad, out=o32)
        comm.check()
        record("qgz 256MiB f64", *sampled.qgz_check(o64, rank, world, X, QGZ_BUCKET, samples=args.samples))
        record("qgz 256MiB f32", *sampled.qgz_check(o32, rank, world, X, QGZ_BUCKET, samples=args.samples,
                                                    rng_seed=7))
        del grad, o32, o64
        comm.close()
        torch.cuda.empty_cache()

    # ---- one GPT-13B layer: qwZ (+hpZ write-through), hpZ gather, qgZ S=2 --------
    if "layer" in cases:
        h = 5120
        layer = 12 * h * h + 13 * h
        layer_p = _pad(layer, world * 2048 * 4)
        shard_len = layer_p // world
        comm = Communicator(group_size=X, qwz_shard=shard_len, hpz_sec=layer_p // X, qgz_elems=layer_p,
                            qgz_stages=2, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
        w = synth.device(3000 + rank, 0, shard_len, torch.float16, "weight", device=dev)
        g = synth.device(5000 + 1000 * rank, 0, layer_p, torch.bfloat16, "grad", device=dev)
        wout = torch.empty(layer_p, dtype=torch.float16, device=dev)
        hout = torch.empty(layer_p, dtype=torch.float16, device=dev)
        gout = torch.empty(layer_p // world, dtype=torch.float32, device=dev)
        for _ in range(3):
            comm.qwz_allgather(w, out=wout, write_secondary=True)
            comm.hpz_allgather(out=hout[: (layer_p // X) * X])
            comm.qgz_reduce_scatter(g, out=gout)
        comm.check()
        record("layer qwz", *sampled.qwz_check(wout, world, shard_len, seed_base=3000, samples=args.samples,
                                               rng_seed=rank))
        # the group gather holds the group's secondary shards = gathered weights
        # [node*X*sec, (node+1)*X*sec) with sec = layer_p/X ... i.e. the whole layer
        record("layer hpz", *sampled.qwz_check(hout, world, shard_len, seed_base=3000, samples=args.samples,
                                               rng_seed=100 + rank))
        record("layer qgz S=2", *sampled.qgz_check(gout, rank, world, X, layer_p, stages=2, seed_base=5000,
                                                   samples=args.samples))
        comm.close()

    # ---- a bucketed gradient stream: 3 x 256 MiB buckets + the 7B stream's
    # 20,678,144-element tail, zero-padded (configs[3], zs/engine.py:465-466) --
    if "stream" in cases:
        tail = 20_678_144
        n_total = 3 * QGZ_BUCKET + tail
        comm = Communicator(group_size=X, qgz_elems=QGZ_BUCKET, qgz_stages=1,
                            qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
        grads = torch.empty(n_total, dtype=torch.bfloat16, device=dev)
        for b in range(4):
            lo = b * QGZ_BUCKET
            synth.device(2000 + 1000 * rank + b, 0, min(QGZ_BUCKET, n_total - lo), torch.bfloat16, "grad",
                         out=grads[lo:lo + QGZ_BUCKET])
        full, tl, tail_pad, n_out = comm.stream_layout(n_total)
        out = comm.qgz_reduce_scatter_stream(grads)
        out = comm.qgz_reduce_scatter_stream(grads, out=out)
        comm.check()
        per = QGZ_BUCKET // world
        for b in range(full):
            record(f"stream bucket {b}", *sampled.qgz_check(out[b * per:(b + 1) * per], rank, world, X, QGZ_BUCKET,
                                                            seed_base=2000 + b, samples=args.samples // 4))
        record("stream tail", *sampled.qgz_check(out[full * per:], rank, world, X, tail_pad, seed_base=2000 + full,
                                                 samples=args.samples, valid=tl))
        del grads, out
        comm.close()

    bad = sum(b for _, _, b in report)
    for name, checked, b in report:
        print(f"rank {rank} {name}: checked {checked} mismatches {b}", flush=True)
    flag = torch.tensor([bad], device="cpu" if oversub else dev)
    dist.all_reduce(flag)
    if rank == 0 and int(flag.item()) == 0:
        print(f"large parity ok: world={world} groups={world // X}x{X}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(flag.item()) else 0)


if __name__ == "__main__":
    main()
