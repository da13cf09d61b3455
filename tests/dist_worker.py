"""Per-rank worker for the multi-GPU parity test (launched by torchrun from
tests/test_gpu_dist.py, one process per GPU).  Every rank regenerates all
ranks' seeded inputs on the host, runs the fused NVLink collectives, and
checks its own outputs bit-exactly against the CPU oracle."""

import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import golden_util as gu  # noqa: E402
import paper_2306_10209_b200 as zpp  # noqa: E402
from oracle import zpp_oracle as O  # noqa: E402
from paper_2306_10209_b200.dist import Communicator, make_groups, nccl_allgather  # noqa: E402


def bf16_bits(v):
    return (np.asarray(v, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def same_bits(a, b):
    """Bitwise equality (np.array_equal would accept -0.0 for +0.0)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    return bool(np.array_equal(a.view(f"u{a.dtype.itemsize}"), b.view(f"u{b.dtype.itemsize}")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--group", type=int, default=2)
    ap.add_argument("--stages", type=int, default=2)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    # ZPP_OVERSUBSCRIBE=1: more ranks than GPUs (e.g. the 2x4 layout on a 4-GPU
    # box).  Ranks sharing a GPU map each other's workspace through CUDA IPC
    # like any peer and their kernels time-slice; NCCL refuses duplicate
    # devices, so the host plumbing runs on gloo and the NCCL comparator is off.
    oversub = os.environ.get("ZPP_OVERSUBSCRIBE") == "1"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    X = args.group
    Y = world // X
    failures = []

    def check(name, ok):
        if not ok:
            failures.append(name)

    # ---- qwZ + hpZ -----------------------------------------------------------
    shard_len = 3 * 2048 + 1024  # ragged last block in every shard
    total = shard_len * world
    spec = zpp.PartitionSpec(total_elems=total, world=world, group_size=X)
    lo, hi = spec.secondary_range(rank)
    shards = [(np.random.default_rng(100 + r).normal(size=shard_len) * 0.02).astype(np.float16) for r in range(world)]
    comm = Communicator(group_size=X, qwz_shard=shard_len, qwz_cfg=zpp.QuantConfig(bit_width=8, block_size=2048),
                        hpz_sec=hi - lo, qgz_elems=args.stages * world * 1024, qgz_stages=args.stages,
                        qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    want, _ = O.all_gather_qwz([s.astype(np.float64) for s in shards], 8, 2048)
    want16 = want.astype(np.float16)
    mine = torch.from_numpy(shards[rank]).cuda()
    for it in range(3):  # exercise both halves of the double buffer
        out = comm.qwz_allgather(mine, write_secondary=True)
        comm.check()
        check(f"qwz it{it}", same_bits(out.cpu().numpy(), want16))
        check(f"hpz secondary it{it}", same_bits(comm.secondary.cpu().numpy(), want16[lo:hi]))
        g = comm.hpz_allgather()
        comm.check()
        check(f"hpz gather it{it}", same_bits(g.cpu().numpy(), want16))
    # host-buffer API with transfer/compute overlap (chunked sub-collectives)
    h_in = torch.from_numpy(shards[rank]).pin_memory()
    h_out = torch.empty(total, dtype=torch.float16).pin_memory()
    comm.qwz_allgather_host(h_in, h_out, chunks=3)
    torch.cuda.synchronize()
    comm.check()
    check("qwz host chunked", same_bits(h_out.numpy(), want16))
    # f32 output of the same gather
    out32 = comm.qwz_allgather(mine, out_dtype=torch.float32)
    comm.check()
    check("qwz fp32", same_bits(out32.cpu().numpy(), want.astype(np.float32)))
    # back-to-back calls with different shard lengths and no host sync in
    # between: the half boundaries of the qwZ double buffer move, so K0 of a
    # call must not overwrite codes peers still pull for the previous one
    lens = [shard_len, 4096, shard_len, 2048 + 512, 1024, shard_len, 4096]
    outs = [comm.qwz_allgather(mine[:m]) for m in lens]
    comm.check()
    for i, m in enumerate(lens):
        wm, _ = O.all_gather_qwz([s[:m].astype(np.float64) for s in shards], 8, 2048)
        check(f"qwz varying length #{i} ({m})", same_bits(outs[i].cpu().numpy(), wm.astype(np.float16)))
    # a device barrier that times out: this rank's data kernels stop, the
    # communicator refuses further calls, and recover() (collective) restores it
    if rank == 0:
        comm.barrier("world", timeout_ms=200)  # the other ranks never arrive
        try:
            comm.check()
            check("timeout raised", False)
        except zpp.DeviceError:
            pass
        try:
            comm.qwz_allgather(mine)
            check("broken communicator refuses calls", False)
        except zpp.DeviceError:
            pass
    comm.recover()
    out = comm.qwz_allgather(mine, write_secondary=True)
    comm.check()
    check("qwz after recover", same_bits(out.cpu().numpy(), want16))
    g = comm.hpz_allgather()
    comm.check()
    check("hpz after recover", same_bits(g.cpu().numpy(), want16))
    # NCCL comparator gathers the raw shards
    if not oversub:
        raw = nccl_allgather(mine)
        check("nccl allgather", same_bits(raw.cpu().numpy(), np.concatenate(shards)))

    # ---- qgZ -----------------------------------------------------------------
    n = args.stages * world * 1024
    grads = [bf16_bits(np.random.default_rng(200 + r).normal(size=n) * np.exp(np.random.default_rng(300 + r).normal(size=n)) * 1e-3)
             for r in range(world)]
    ref = O.qgz_2hop([gu.as_f64(g, "bf16") for g in grads], X, Y, args.stages, 4, 512)[rank]
    gt = gu.to_torch(grads[rank], "bf16")
    for it in range(3):
        o64 = comm.qgz_reduce_scatter(gt, out_dtype=torch.float64)
        comm.check()
        check(f"qgz f64 it{it}", same_bits(o64.cpu().numpy(), ref))
        o32 = comm.qgz_reduce_scatter(gt)
        comm.check()
        check(f"qgz f32 it{it}", same_bits(o32.cpu().numpy(), ref.astype(np.float32)))
    # a second communicator and bucket size: 83 blocks per slice, stages 1
    L2 = 2 * 16384 + 17 * 512
    n2 = world * L2
    grads2 = [bf16_bits(np.random.default_rng(400 + r).normal(size=n2) * 1e-3) for r in range(world)]
    ref2 = O.qgz_2hop([gu.as_f64(g, "bf16") for g in grads2], X, Y, 1, 4, 512)[rank]
    comm2 = Communicator(group_size=X, qgz_elems=n2, qgz_stages=1, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    gt2 = gu.to_torch(grads2[rank], "bf16")
    for it in range(3):
        o2 = comm2.qgz_reduce_scatter(gt2, out_dtype=torch.float64)
        comm2.check()
        check(f"qgz bucket2 it{it}", same_bits(o2.cpu().numpy(), ref2))
    comm2.close()
    # ---- cross-layer prefetch-quantize ---------------------
    n_layers = 4
    lshard = 2 * 2048 + 512
    spec_l = zpp.PartitionSpec(total_elems=lshard * world, world=world, group_size=X)
    llo, lhi = spec_l.secondary_range(rank)
    lay = [[(np.random.default_rng(500 + 10 * i + r).normal(size=lshard) * 0.02).astype(np.float16)
            for r in range(world)] for i in range(n_layers)]
    lwant = [O.all_gather_qwz([s.astype(np.float64) for s in lay[i]], 8, 2048)[0].astype(np.float16)
             for i in range(n_layers)]
    comm3 = Communicator(group_size=X, qwz_shard=lshard, hpz_sec=lhi - llo, hpz_layers=n_layers)
    mine_l = [torch.from_numpy(lay[i][rank]).cuda() for i in range(n_layers)]
    for prefetch in (True, False, True):
        outs = comm3.qwz_allgather_layers(mine_l, write_secondary=True, prefetch=prefetch)
        gs = [comm3.hpz_allgather(layer=i) for i in reversed(range(n_layers))][::-1]  # backward order
        comm3.check()
        for i in range(n_layers):
            check(f"prefetch={prefetch} qwz layer {i}", same_bits(outs[i].cpu().numpy(), lwant[i]))
            check(f"prefetch={prefetch} hpz layer {i}", same_bits(gs[i].cpu().numpy(), lwant[i]))
    # a prefetched shard that the next call does not use (it passes another
    # tensor): the prefetch is waited for and the shard quantized as usual
    o0 = comm3.qwz_allgather(mine_l[0], next_shard=mine_l[1])
    o2 = comm3.qwz_allgather(mine_l[2], next_shard=mine_l[3])
    o3 = comm3.qwz_allgather(mine_l[3])
    comm3.check()
    check("prefetch mismatch 0", same_bits(o0.cpu().numpy(), lwant[0]))
    check("prefetch mismatch 2", same_bits(o2.cpu().numpy(), lwant[2]))
    check("prefetch used 3", same_bits(o3.cpu().numpy(), lwant[3]))
    comm3.close()

    # ---- bucketed gradient stream with a zero-padded tail (configs[3]) --------
    # five buckets (one zpp_qgz_reduce_scatter_buckets call: K1 of bucket b+1
    # beside K2/K3 of bucket b) and a ragged tail, with 1 and 2 stages per bucket
    for S2 in (1, 2):
        bucket = S2 * world * 2048
        n_stream = 5 * bucket + 3 * 512 + 77
        gs_host = [bf16_bits(np.random.default_rng(700 + 10 * S2 + r).normal(size=n_stream) * 1e-3)
                   for r in range(world)]
        comm4 = Communicator(group_size=X, qgz_elems=bucket, qgz_stages=S2,
                             qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
        full, tail, tail_pad, n_out = comm4.stream_layout(n_stream)
        check("stream layout", full == 5 and tail == 3 * 512 + 77 and tail_pad % (world * S2 * 512) == 0)
        want_parts = []
        for b in range(full + 1):
            lo_b = b * bucket
            hi_b = min(lo_b + bucket, n_stream)
            nb = bucket if b < full else tail_pad
            srcs = []
            for r in range(world):
                v = np.zeros(nb)
                v[:hi_b - lo_b] = gu.as_f64(gs_host[r][lo_b:hi_b], "bf16")
                srcs.append(v)
            want_parts.append(O.qgz_2hop(srcs, X, Y, S2, 4, 512)[rank])
        want_s = np.concatenate(want_parts)
        gts = gu.to_torch(gs_host[rank], "bf16")
        for it in range(2):
            o_s = comm4.qgz_reduce_scatter_stream(gts, out_dtype=torch.float64)
            comm4.check()
            check(f"qgz stream S={S2} it{it}", o_s.numel() == n_out and same_bits(o_s.cpu().numpy(), want_s))
        comm4.close()

    # ---- process groups for the staged comparators ---------------------------
    mine_pg, cross_pg = make_groups(X)
    check("groups", dist.get_world_size(mine_pg) == X and dist.get_world_size(cross_pg) == Y)

    comm.close()
    flag = torch.tensor([len(failures)], device="cpu" if oversub else "cuda")
    dist.all_reduce(flag)
    if failures:
        print(f"rank {rank} FAILED: {failures}", flush=True)
    elif rank == 0:
        print(f"dist parity ok: world={world} groups={Y}x{X} stages={args.stages}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(flag.item()) else 0)


if __name__ == "__main__":
    main()
