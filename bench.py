"""Benchmark of the ZeRO++ hot path on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[1]): qwZ INT8/2048 quantized all-gather of a
1.3B-parameter fp16 flat weight buffer (M = 1,300,004,864, block-aligned),
sharded over the N GPUs of one box.  One step = one fused qwZ all-gather:
every rank quantizes its M/N shard and ends with all M weights dequantized to
fp16 in its HBM.  At N = 1 the step is the quantize -> dequantize round trip of
the whole buffer.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value = whole-job qwZ effective GB/s = N * (2*M fp16 bytes delivered per rank)
/ step time (max over ranks, CUDA events).  Extra keys: the roofline of the
dominant kernel, the CPU reference timed on this host, an end-to-end number
through host buffers, clocks during the timed region, the NCCL fp16
all-gather comparator, and the qgZ 256 MiB bf16 gradient bucket (configs[3]).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: everything else that writes to fd 1
# (NCCL's version banner, library warnings) is sent to stderr, and the line is
# written to a duplicate of the original stdout.
_JSON_FD = None


def _claim_stdout():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict) -> None:
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())

METRIC = "qwZ/qgZ effective GB/s at 1/2/4/8 B200; quant kernel HBM GB/s vs 8 TB/s"
M_PARAMS = 1_300_004_864           # 1.3e9 rounded up to a multiple of 8 * 2048
QGZ_BUCKET = 134_217_728           # 256 MiB of bf16 gradients
NVLINK_PEER_GBS = 770.0            # measured peer copy per direction (B200_PROFILING.md)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("pci.bus_id,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, pci=None):
        self.proc = None
        self.lines = []
        self.pci = pci  # {(domain, bus, device)} of the job's GPUs; None = all

    def _ours(self, bus_id: str) -> bool:
        if self.pci is None:
            return True
        try:
            dom, bus, devfn = bus_id.split(":")
            return (int(dom, 16), int(bus, 16), int(devfn.split(".")[0], 16)) in self.pci
        except ValueError:
            return False

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # first sample before the timed region
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, name):
        setattr(self, name, time.time())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = getattr(self, "t_load", 0.0), getattr(self, "t_end", 1e30)
        rows = []
        for ts, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if lo <= ts <= hi and len(parts) >= 8:  # only samples taken while the step was running
                rows.append(parts)
        ours = [r for r in rows if self._ours(r[0])]
        which = "the job's GPUs (matched by PCI bus id)"
        if not ours:
            ours, which = rows, "all GPUs (no PCI bus id match)"
        sm, smax, reasons = [], [], set()
        for parts in ours:
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "gpus": which}


def cpu_reference(sample_elems: int, steps: int, warmup: int, threads: int):
    """The reference algorithm on the host (oracle port of zs/quantizer.py
    quantize + dequantize, numpy, block-parallel over host threads) on a
    bounded sample of the fp16 weight buffer; same metric definition."""
    from oracle import zpp_oracle as O
    rng = np.random.default_rng(1000)
    x = (rng.normal(size=sample_elems) * 0.02).astype(np.float16)
    for _ in range(warmup):
        O.qwz_roundtrip_threaded(x, 8, 2048, threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.qwz_roundtrip_threaded(x, 8, 2048, threads=threads)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return 2 * sample_elems / t / 1e9, t


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    sample = 1 << 24
    gbs, t = cpu_reference(sample, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": {"workload": "qwZ INT8/2048 quantize->dequantize of fp16 weights (reference CPU algorithm)",
                   "M": M_PARAMS, "sample_elems": sample},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} fp16 elements of the 1.3B buffer per step, numpy oracle port of "
                                   "zs/quantizer.py quantize+dequantize, block-parallel over host threads"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200 import _lib
    from paper_2306_10209_b200.dist import Communicator, nccl_allgather, nccl_reduce_scatter

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # ZPP_OVERSUBSCRIBE=1 (functional check only, never a bench number): more
    # ranks than GPUs, e.g. the 8-rank 2x4 layout on a 4-GPU box.  NCCL refuses
    # duplicate devices, so the host plumbing runs on gloo and the NCCL
    # comparators are skipped.
    oversub = os.environ.get("ZPP_OVERSUBSCRIBE") == "1"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    dev = torch.device("cuda", local)
    shard_len = M_PARAMS // world
    cfg = zpp.QuantConfig(bit_width=8, block_size=2048)
    qgz_cfg = zpp.QuantConfig(bit_width=4, block_size=512)
    comm = Communicator(group_size=min(world, 4), qwz_shard=shard_len, qwz_cfg=cfg, qgz_elems=QGZ_BUCKET,
                        qgz_stages=1, qgz_cfg=qgz_cfg)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    shard = (torch.randn(shard_len, generator=g, device=dev) * 0.02).half()
    out = torch.empty(M_PARAMS, dtype=torch.float16, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if oversub else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(steps):
            fn()
        e.record(stream)
        e.synchronize()
        barrier()
        return max_over_ranks(s.elapsed_time(e) / steps * 1e-3)

    # ---- headline: fused qwZ all-gather -----------------------------------
    step = lambda: comm.qwz_allgather(shard, out=out)
    p = torch.cuda.get_device_properties(dev)
    mine = (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    pci = [None] * world
    if world > 1:
        dist.all_gather_object(pci, mine)
    else:
        pci = [mine]
    clocks = ClockSampler(set(pci))  # samples of the job's GPUs only
    if rank == 0:
        clocks.start()  # sampling spans warmup + the timed region
    for _ in range(args.warmup):
        step()
    comm.check()
    barrier()
    # clock window: keep the GPU on this step for ~0.5 s right before the timed
    # region so the 50 ms nvidia-smi samples see it under load
    t_est = timed(step, 3, 0)  # same value on every rank (max over ranks)
    clocks.mark("t_load")
    for _ in range(int(0.5 / max(t_est, 1e-4)) + 1):  # identical step count on all ranks
        step()
    torch.cuda.synchronize()
    t_step = timed(step, args.steps, 0)
    clocks.mark("t_end")
    if rank == 0:
        time.sleep(0.06)
    clk = clocks.stop() if rank == 0 else None
    comm.check()
    # N = 1: one fused quantize->dequantize kernel; N > 1: quantize, barrier, TMA gather
    launches_per_step = 1 if world == 1 else 3
    value = world * 2 * M_PARAMS / t_step / 1e9

    # ---- per-kernel roofline (CUDA events around each kernel alone) ----------
    hbm_peak, peak_kind = peaks()
    sym0 = [lib.zpp_comm_sym_ptr(comm.handle, r) for r in range(world)]
    qbytes = shard_len + shard_len // 2048 * 4
    codes_off, abs_off = comm.layout.qwz, comm.layout.qwz + ((shard_len + 255) // 256 * 256)
    st = stream.cuda_stream
    qcodes = sym0[rank] + codes_off
    qabs = sym0[rank] + abs_off

    def k_quant():
        lib.zpp_quantize(shard.data_ptr(), _lib.F16, shard_len, 8, 2048, qcodes, qabs, comm.flag.data_ptr(), st)

    cp, _k1 = _lib.ptr_array([p + codes_off for p in sym0])
    ap, _k2 = _lib.ptr_array([p + abs_off for p in sym0])

    def k_gather():
        lib.zpp_gather_dequantize(cp, ap, _lib.F32, world, rank, shard_len, 8, 2048, out.data_ptr(), _lib.F16,
                                  shard_len, None, 0, 0, comm.flag.data_ptr(), st)

    kq = timed(k_quant, args.steps, 2)
    comm.barrier()
    barrier()
    kg = timed(k_gather, args.steps, 2)
    comm.check()
    q_alg = 2 * shard_len + qbytes                       # read fp16 shard, write codes + absmax
    g_alg = world * qbytes + 2 * M_PARAMS                # read all codes (local + peers), write fp16
    kern = {"quantize_reg_kernel": {"us": kq * 1e6, "alg_bytes": q_alg, "GBps": q_alg / kq / 1e9},
            "dequant16_kernel (gather)": {"us": kg * 1e6, "alg_bytes": g_alg, "GBps": g_alg / kg / 1e9}}
    traffic = ncu_traffic()
    if world == 1:
        fused_alg = 4 * shard_len + qbytes  # read fp16, write codes + absmax, write fp16
        kern["quantize_reg_kernel<deq> (fused qwZ self-gather)"] = {"us": t_step * 1e6, "alg_bytes": fused_alg,
                                                                   "GBps": fused_alg / t_step / 1e9}
        dom = "quantize_reg_kernel<deq> (fused qwZ self-gather)"
        d = kern[dom]
        roof = {"kernel": dom, "bound": "hbm", "achieved": d["GBps"], "peak": hbm_peak, "unit": "GB/s",
                "frac": d["GBps"] / hbm_peak, "traffic": traffic.get(dom), "peak_kind": peak_kind,
                "alg_bytes_per_launch": d["alg_bytes"], "launch_us": d["us"], "kernels": kern}
    else:
        ingress = (world - 1) * qbytes
        ach = ingress / kg / 1e9
        roof = {"kernel": "dequant16_tma_kernel (gather over NVLink)", "bound": "nvlink", "achieved": ach,
                "peak": NVLINK_PEER_GBS, "unit": "GB/s", "frac": ach / NVLINK_PEER_GBS,
                # ncu cannot profile a multi-rank launch; the 1-GPU capture of the same
                # kernel (4 local sources -> 1.3B fp16) is reported under "hbm" instead
                "traffic": None,
                "peak_kind": "measured peer copy, per direction",
                "alg_bytes_per_launch": ingress, "launch_us": kg * 1e6, "kernels": kern,
                "hbm": {"achieved": kern["dequant16_kernel (gather)"]["GBps"], "peak": hbm_peak,
                        "frac": kern["dequant16_kernel (gather)"]["GBps"] / hbm_peak,
                        "traffic_1gpu_capture": traffic.get("dequant16_tma_kernel (gather over NVLink)"),
                        "alg_bytes_1gpu_capture": 4 * (M_PARAMS // 4 + M_PARAMS // 4 // 2048 * 4) + 2 * M_PARAMS}}

    # ---- end to end through host buffers ------------------------------------
    h_in = torch.empty(shard_len, dtype=torch.float16, pin_memory=True)
    h_in.copy_(shard.cpu())
    h_out = torch.empty(M_PARAMS, dtype=torch.float16, pin_memory=True)

    d_in = torch.empty_like(shard)

    def e2e_step():  # host -> device -> fused qwZ -> host, chunk-pipelined over 3 streams
        comm.qwz_allgather_host(h_in, h_out, chunks=16, d_shard=d_in, d_out=out)

    e2e_steps = max(3, min(args.steps, 5))
    t_e2e = timed(e2e_step, e2e_steps, 1)
    comm.check()
    e2e = {"value": world * 2 * M_PARAMS / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 2 * shard_len,
           "d2h_bytes_per_step": 2 * M_PARAMS, "ms_per_step": t_e2e * 1e3,
           "path": "pinned host shard -> Communicator.qwz_allgather_host (H2D, fused qwZ and D2H overlapped in "
                   "16 chunks) -> pinned host gathered fp16 weights"}
    del h_out, h_in

    # ---- comparators and qgZ ---------------------------------------------------
    extra = {}
    if world > 1 and not oversub:
        t_nccl = timed(lambda: nccl_allgather(shard, out=out), args.steps, 2)
        extra["nccl_fp16_allgather"] = {"value": world * 2 * M_PARAMS / t_nccl / 1e9, "unit": "GB/s",
                                        "ms_per_step": t_nccl * 1e3}
    grad = (torch.randn(QGZ_BUCKET, generator=g, device=dev) * 1e-3).bfloat16()
    part = torch.empty(QGZ_BUCKET // world, dtype=torch.float32, device=dev)
    t_qgz = timed(lambda: comm.qgz_reduce_scatter(grad, out=part), args.steps, 2)
    comm.check()
    X, Y = comm.group_size, world // comm.group_size
    L = QGZ_BUCKET // world
    wire = (X - 1) * (Y * L // 2 + Y * L // 512 * 4) + (Y - 1) * (L // 2 + L // 512 * 8)
    extra["qgz"] = {"workload": "qgZ INT4/512 2-hop reduce-scatter of a 256 MiB bf16 bucket", "groups": f"{Y}x{X}",
                    "ms_per_bucket": t_qgz * 1e3,
                    "effective_GBps": world * 2 * QGZ_BUCKET * (world - 1) / world / t_qgz / 1e9 if world > 1 else
                    2 * QGZ_BUCKET / t_qgz / 1e9,
                    "wire_bytes_per_gpu": wire}
    if world > 1 and not oversub:
        gb = grad.clone()
        pb = torch.empty(QGZ_BUCKET // world, dtype=torch.bfloat16, device=dev)
        t_rs = timed(lambda: nccl_reduce_scatter(gb, out=pb), args.steps, 2)
        extra["nccl_bf16_reduce_scatter"] = {"ms_per_bucket": t_rs * 1e3,
                                             "effective_GBps": world * 2 * QGZ_BUCKET * (world - 1) / world / t_rs / 1e9}

    extra["hpz"] = hpz_leg(comm_cls=Communicator, world=world, dev=dev, g=g, timed=lambda f: timed(f, args.steps, 2),
                           oversub=oversub, nccl_allgather=nccl_allgather)
    extra["zeropp_step_13b_layer"] = step_leg(world=world, dev=dev, g=g, timed=lambda f: timed(f, max(5, args.steps // 2), 2),
                                              oversub=oversub, comm_cls=Communicator, zpp=zpp,
                                              nccl_allgather=nccl_allgather, nccl_reduce_scatter=nccl_reduce_scatter)
    kq_gbs = kern["quantize_reg_kernel"]["GBps"]
    extra["quant_kernel_hbm"] = {"kernel": "quantize_reg_kernel (K0: fp16 shard -> INT8/2048 codes + absmax)",
                                 "achieved_GBps": kq_gbs, "frac_of_8TBs_nominal": kq_gbs / 8000.0,
                                 "frac_of_measured_peak": kq_gbs / hbm_peak, "shard_elems": shard_len}
    extra["params_per_s"] = {"qwz": world * M_PARAMS / t_step, "qgz": world * QGZ_BUCKET / t_qgz,
                             "note": "whole-job parameters (or gradients) delivered per second"}
    if world > 1:
        extra["nvlink_nominal"] = {"peak": 900.0, "unit": "GB/s", "qwz_ingress_frac": (world - 1) * qbytes / kg / 1e9 / 900.0,
                                   "qgz_wire_frac": wire / t_qgz / 1e9 / 900.0}

    line = None
    if rank == 0:
        threads = os.cpu_count() or 1
        cpu_gbs, cpu_t = cpu_reference(1 << 25, 3, 1, threads)
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": f"qwZ INT8/2048 fused all-gather of a 1.3B fp16 weight buffer over {world} GPU(s)"
                                   + (" (W=1: quantize->dequantize round trip)" if world == 1 else " (NVLink P2P)"),
                       "M": M_PARAMS, "shard_elems": shard_len, "quant": "int8/2048", "out_dtype": "fp16",
                       "parallelism": f"zero3-dp{world}", "groups": f"{world // comm.group_size}x{comm.group_size}",
                       "l2": "inputs and outputs larger than L2 (shard + 2.6 GB fp16 output per step), no flush"}
                      | ({"oversubscribed": "functional check, ranks share GPUs: not a measurement"} if oversub else {}),
            "roofline": roof,
            "cpu_baseline": {"value": cpu_gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"{1 << 25} fp16 elements, numpy oracle port of zs/quantizer.py "
                                       "quantize+dequantize, block-parallel over host threads, median of 3"},
            "e2e": e2e, "clocks": clk, "gpu_launches": launches_per_step * args.steps,
            "qwz": {"ms_per_step": t_step * 1e3,
                    "wire_ingress_bytes_per_gpu": (world - 1) * qbytes,
                    "fp16_allgather_ingress_bytes_per_gpu": (world - 1) * 2 * shard_len},
        }
        line.update(extra)
        emit(line)
    comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _pad(n: int, align: int) -> int:
    return (n + align - 1) // align * align


def hpz_leg(*, comm_cls, world, dev, g, timed, oversub, nccl_allgather):
    """BASELINE configs[2]: hpZ gather of one GPT-1.3B layer (12h^2+13h, h=2048)
    inside a group of min(N, 4) consecutive GPUs, vs NCCL's full-box and group
    fp16 all-gathers.  The secondary shard is written through by the qwZ gather
    (zs/engine.py:364-370)."""
    import torch

    from paper_2306_10209_b200.dist import make_groups

    X = min(world, 4)
    h = 2048
    layer = 12 * h * h + 13 * h
    layer_p = _pad(layer, world * 2048)
    sec = layer_p // X
    comm = comm_cls(group_size=X, qwz_shard=layer_p // world, hpz_sec=sec)
    w = (torch.randn(layer_p // world, generator=g, device=dev) * 0.02).half()
    comm.qwz_allgather(w, write_secondary=True)
    comm.check()
    out = torch.empty(layer_p, dtype=torch.float16, device=dev)
    t = timed(lambda: comm.hpz_allgather(out=out))
    comm.check()
    comm.close()
    ingress = (X - 1) * sec * 2
    res = {"workload": "hpZ fp16 gather of one GPT-1.3B layer inside a group", "layer_params": layer,
           "padded": layer_p, "group_size": X, "ms": t * 1e3, "ingress_bytes_per_gpu": ingress,
           "ingress_GBps": ingress / t / 1e9, "cross_group_bytes": 0}
    if world > 1 and not oversub:
        full_out = torch.empty(layer_p, dtype=torch.float16, device=dev)
        res["nccl_fullbox_fp16_ag_ms"] = timed(lambda: nccl_allgather(w, out=full_out)) * 1e3
        if X < world:
            group_pg, _ = make_groups(X)
            gs = torch.empty(sec, dtype=torch.float16, device=dev)
            res["nccl_group_fp16_ag_ms"] = timed(lambda: nccl_allgather(gs, out=out, group=group_pg)) * 1e3
    return res


def step_leg(*, world, dev, g, timed, oversub, comm_cls, zpp, nccl_allgather, nccl_reduce_scatter):
    """BASELINE configs[4]: the communication of one GPT-13B layer (h=5120) of a
    ZeRO++ step -- forward qwZ (INT8/2048, writes the hpZ secondary), backward
    hpZ gather inside the group, gradient qgZ (INT4/512, S=2) -- vs ZeRO-3's
    fp16 all-gather x2 + bf16 reduce-scatter (NCCL)."""
    import torch

    X = min(world, 4)
    h = 5120
    layer = 12 * h * h + 13 * h
    layer_p = _pad(layer, world * 2048 * 4)
    comm = comm_cls(group_size=X, qwz_shard=layer_p // world, hpz_sec=layer_p // X, qgz_elems=layer_p,
                    qgz_stages=2, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    w = (torch.randn(layer_p // world, generator=g, device=dev) * 0.02).half()
    gl = (torch.randn(layer_p, generator=g, device=dev) * 1e-3).bfloat16()
    wout = torch.empty(layer_p, dtype=torch.float16, device=dev)
    gout = torch.empty(layer_p // world, dtype=torch.float32, device=dev)

    def zeropp_layer():
        comm.qwz_allgather(w, out=wout, write_secondary=True)
        comm.hpz_allgather(out=wout)
        comm.qgz_reduce_scatter(gl, out=gout)

    t = timed(zeropp_layer)
    comm.check()
    comm.close()
    res = {"workload": "fwd qwZ + bwd hpZ + grad qgZ of one GPT-13B layer", "layer_params": layer,
           "padded": layer_p, "groups": f"{world // X}x{X}", "zeropp_ms": t * 1e3, "zeropp_40_layers_ms": 40e3 * t}
    if world > 1 and not oversub:
        bout = torch.empty(layer_p // world, dtype=torch.bfloat16, device=dev)

        def zero3_layer():
            nccl_allgather(w, out=wout)
            nccl_allgather(w, out=wout)
            nccl_reduce_scatter(gl, out=bout)

        t3 = timed(zero3_layer)
        res.update({"zero3_nccl_ms": t3 * 1e3, "speedup_vs_zero3": t3 / t})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    args = ap.parse_args()
    _claim_stdout()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
