"""NVLink bytes per collective call, from the NVML per-link byte counters
(NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES summed over the GPU's
links), read before and after CALLS back-to-back calls on every rank.  The
counters count bytes on the wire (payload plus protocol overhead), so
measured / algorithmic > 1 is the link-level overhead, and >> 1 would be
re-reads.  No profiler: the collectives run at full speed on every rank.

    torchrun --nproc-per-node N tools/nvl_counters.py [X]
"""

import json
import os
import sys

import pynvml
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp  # noqa: E402
from oracle import synth  # noqa: E402
from paper_2306_10209_b200.dist import Communicator  # noqa: E402

BUCKET = 134_217_728
M = 1_300_004_864
CALLS = 10
XMIT, RCV = 202, 204  # NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES


def nvml_handle(dev):
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    return pynvml.nvmlDeviceGetHandleByPciBusId(bus)


def link_bytes(h, links):
    vals = []
    for fid in (XMIT, RCV):
        tot = 0
        res = pynvml.nvmlDeviceGetFieldValues(h, [(fid, l) for l in links])
        for r in res:
            if r.nvmlReturn == 0:
                tot += r.value.ullVal
        vals.append(tot)
    return vals


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    X = int(sys.argv[1]) if len(sys.argv) > 1 else world
    pynvml.nvmlInit()
    h = nvml_handle(dev)
    links = []
    for l in range(18):
        try:
            if pynvml.nvmlDeviceGetNvLinkState(h, l) == pynvml.NVML_FEATURE_ENABLED:
                links.append(l)
        except pynvml.NVMLError:
            break
    shard = M // world
    comm = Communicator(group_size=X, qwz_shard=shard, qwz_cfg=zpp.QuantConfig(bit_width=8, block_size=2048),
                        qgz_elems=BUCKET, qgz_stages=1, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512),
                        hpz_sec=M // X)
    w = synth.device(1000 + rank, 0, shard, torch.float16, "weight", device=dev)
    g = synth.device(2000 + 1000 * rank, 0, BUCKET, torch.bfloat16, "grad", device=dev)
    out = torch.empty(M, dtype=torch.float16, device=dev)
    part = torch.empty(BUCKET // world, dtype=torch.float32, device=dev)
    hout = torch.empty(M, dtype=torch.float16, device=dev)
    Y = world // X
    L = BUCKET // world
    qcodes = shard + shard // 2048 * 4
    cases = {
        # algorithmic NVLink ingress per GPU per call (egress is the same by symmetry)
        "qwz_allgather_1.3B": (lambda: comm.qwz_allgather(w, out=out, write_secondary=True), (world - 1) * qcodes),
        "hpz_allgather_1.3B": (lambda: comm.hpz_allgather(out=hout), (X - 1) * (M // X) * 2),
        "qgz_256MiB": (lambda: comm.qgz_reduce_scatter(g, out=part),
                       (X - 1) * (Y * L // 2 + Y * L // 512 * 4) + (Y - 1) * (L // 2 + L // 512 * 8)),
    }
    res = {}
    for name, (fn, alg) in cases.items():
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        b0 = link_bytes(h, links)
        for _ in range(CALLS):
            fn()
        torch.cuda.synchronize()
        b1 = link_bytes(h, links)
        dist.barrier()
        tx, rx = (b1[0] - b0[0]) / CALLS, (b1[1] - b0[1]) / CALLS
        res[name] = {"alg_ingress_bytes": alg, "nvl_rx_bytes": rx, "nvl_tx_bytes": tx,
                     "rx_per_alg": rx / alg if alg else None, "tx_per_alg": tx / alg if alg else None}
    comm.check()
    allres = [None] * world
    dist.all_gather_object(allres, {"rank": rank, "links": links, "per_call": res})
    if rank == 0:
        print(json.dumps({"world": world, "X": X, "calls": CALLS, "ranks": allres}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
