"""Multi-GPU sweep of the secondary BASELINE configs (run under torchrun):

  configs[2] hpZ: GPT-1.3B layer (12h^2+13h, h=2048, padded) gathered inside a
             group vs the full-box fp16 all-gather
  configs[3] qgZ: 256 MiB bf16 bucket, INT4/512, stages S in {1, 2, 4}, vs NCCL
             bf16 reduce-scatter
  configs[4] one GPT-13B layer (h=5120) of ZeRO++ step communication:
             fwd qwZ + bwd hpZ + grad qgZ vs fp16 all-gather x2 + bf16 RS

Prints one JSON object on rank 0.  Device time, CUDA events, max over ranks.
"""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp  # noqa: E402
from paper_2306_10209_b200.dist import Communicator, nccl_allgather, nccl_reduce_scatter, make_groups  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    X = min(world, 4) if len(sys.argv) < 2 else int(sys.argv[1])
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(rank)

    def timed(fn, steps=20, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(steps):
            fn()
        e.record()
        e.synchronize()
        t = torch.tensor([s.elapsed_time(e) / steps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())  # ms

    sections = os.environ.get("ZPP_BENCH_SECTIONS", "qgz,hpz,step").split(",")
    res = {"world": world, "group_size": X, "k1_sms": os.environ.get("ZPP_QGZ_K1_SMS")}
    group_pg, _ = make_groups(X)

    # ---- qgZ stage sweep --------------------------------------------------------
    if "qgz" in sections:
        qgz_sweep(res, X, world, dev, g, timed)
    if "hpz" in sections:
        hpz_layer(res, X, world, dev, g, timed, group_pg)
    if "step" in sections:
        step_13b(res, X, world, dev, g, timed)
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


def qgz_sweep(res, X, world, dev, g, timed):
    bucket = 134_217_728
    grad = (torch.randn(bucket, generator=g, device=dev) * 1e-3).bfloat16()
    q = {}
    for S in [int(v) for v in os.environ.get("ZPP_BENCH_STAGES", "1,2,4,8").split(",")]:
        comm = Communicator(group_size=X, qgz_elems=bucket, qgz_stages=S,
                            qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
        out = torch.empty(bucket // world, dtype=torch.float32, device=dev)
        q[f"S{S}_ms"] = timed(lambda: comm.qgz_reduce_scatter(grad, out=out))
        comm.check()
        comm.close()
    pb = torch.empty(bucket // world, dtype=torch.bfloat16, device=dev)
    q["nccl_bf16_rs_ms"] = timed(lambda: nccl_reduce_scatter(grad, out=pb))
    res["qgz_256MiB"] = q


def hpz_layer(res, X, world, dev, g, timed, group_pg):
    # ---- hpZ: GPT-1.3B layer ----------------------------------------------------
    h = 2048
    layer = 12 * h * h + 13 * h
    align = world * 2048
    layer_p = (layer + align - 1) // align * align
    sec = layer_p // X
    comm = Communicator(group_size=X, qwz_shard=layer_p // world, hpz_sec=sec)
    w = (torch.randn(layer_p // world, generator=g, device=dev) * 0.02).half()
    comm.qwz_allgather(w, write_secondary=True)
    comm.check()
    hp = {"layer_params": layer, "padded": layer_p,
          "hpz_group_gather_ms": timed(lambda: comm.hpz_allgather())}
    full_shard = torch.empty(layer_p // world, dtype=torch.float16, device=dev)
    full_out = torch.empty(layer_p, dtype=torch.float16, device=dev)
    hp["nccl_fullbox_fp16_ag_ms"] = timed(lambda: nccl_allgather(full_shard, out=full_out))
    grp_shard = torch.empty(sec, dtype=torch.float16, device=dev)
    grp_out = torch.empty(sec * X, dtype=torch.float16, device=dev)
    hp["nccl_group_fp16_ag_ms"] = timed(lambda: nccl_allgather(grp_shard, out=grp_out, group=group_pg))
    comm.close()
    res["hpz_gpt1.3b_layer"] = hp


def step_13b(res, X, world, dev, g, timed):
    # ---- combined ZeRO++ step communication, one GPT-13B layer --------------------
    h = 5120
    layer = 12 * h * h + 13 * h
    align = world * 2048 * 4
    layer_p = (layer + align - 1) // align * align
    comm = Communicator(group_size=X, qwz_shard=layer_p // world, hpz_sec=layer_p // X, qgz_elems=layer_p,
                        qgz_stages=2, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    w = (torch.randn(layer_p // world, generator=g, device=dev) * 0.02).half()
    gl = (torch.randn(layer_p, generator=g, device=dev) * 1e-3).bfloat16()
    wout = torch.empty(layer_p, dtype=torch.float16, device=dev)
    gout = torch.empty(layer_p // world, dtype=torch.float32, device=dev)

    def zeropp_layer():
        comm.qwz_allgather(w, out=wout, write_secondary=True)   # forward gather
        comm.hpz_allgather(out=wout)                              # backward gather inside the group
        comm.qgz_reduce_scatter(gl, out=gout)                     # gradient reduce

    t_zpp = timed(zeropp_layer, steps=10)
    t_qwz = timed(lambda: comm.qwz_allgather(w, out=wout, write_secondary=True), steps=10)
    t_hpz = timed(lambda: comm.hpz_allgather(out=wout), steps=10)
    t_qgz = timed(lambda: comm.qgz_reduce_scatter(gl, out=gout), steps=10)
    comm.check()
    comm.close()
    bout = torch.empty(layer_p // world, dtype=torch.bfloat16, device=dev)

    def zero3_layer():
        nccl_allgather(w, out=wout)
        nccl_allgather(w, out=wout)
        nccl_reduce_scatter(gl, out=bout)

    t_z3 = timed(zero3_layer, steps=10)
    t_ag = timed(lambda: nccl_allgather(w, out=wout), steps=10)
    t_rs = timed(lambda: nccl_reduce_scatter(gl, out=bout), steps=10)
    res["gpt13b_layer_step_comm"] = {"layer_params": layer, "padded": layer_p, "zeropp_ms": t_zpp, "parts_ms": {"qwz": t_qwz, "hpz": t_hpz, "qgz": t_qgz},
                                     "zero3_nccl_ms": t_z3, "zero3_parts_ms": {"ag": t_ag, "rs": t_rs}, "speedup": t_z3 / t_zpp,
                                     "zeropp_40_layers_ms": 40 * t_zpp, "zero3_40_layers_ms": 40 * t_z3}


if __name__ == "__main__":
    main()
