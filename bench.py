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
dominant kernel (NVLink 900 GB/s at N > 1), busbw, sampled bitwise parity of
every leg against the oracle, the CPU reference timed on this host, an
end-to-end number through host buffers, clocks during the timed region, the
NCCL comparators, and one leg per other BASELINE config: config-1 16M fp32
round trip, the qgZ 256 MiB bucket with its roofline, the hpZ group gather,
the 7B qgZ gradient stream, and the 40-layer GPT-13B ZeRO++ step with and
without cross-layer prefetch.  ZPP_BENCH_LEGS selects legs.
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
NVLINK_NOMINAL_GBS = 900.0         # NVLink 5 per direction per GPU (north_star's roofline)
NVLINK_PEER_GBS = 770.0            # measured peer copy per direction (B200_PROFILING.md)
TMA_PULL_GBS = {2: 644.0, 4: 662.0}  # measured TMA bulk-pull ingress ceiling (profiles/p2p_bw_r1_n{2,4}.txt)


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
    from oracle import sampled, synth
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
    sections = set(os.environ.get("ZPP_BENCH_LEGS", "qgz,config1,hpz,stream,step").split(","))
    lib = _lib.load()
    dev = torch.device("cuda", local)
    # SURVEY 8d's hierarchy: two groups of W/2 consecutive GPUs stand in for
    # two nodes (W = 8: 2x4, W = 4: 2x2, W = 2: 2x1)
    X = group_size_for(world)
    shard_len = M_PARAMS // world
    cfg = zpp.QuantConfig(bit_width=8, block_size=2048)
    qgz_cfg = zpp.QuantConfig(bit_width=4, block_size=512)
    comm = Communicator(group_size=X, qwz_shard=shard_len, qwz_cfg=cfg, qgz_elems=QGZ_BUCKET, qgz_stages=1,
                        qgz_cfg=qgz_cfg)
    # seeded counter-based inputs (oracle/synth.py): any element of any rank's
    # input can be recomputed on the host for the sampled parity check below
    shard = synth.device(1000 + rank, 0, shard_len, torch.float16, "weight", device=dev)
    out = torch.empty(M_PARAMS, dtype=torch.float16, device=dev)
    stream = torch.cuda.current_stream()
    hbm_peak, peak_kind = peaks()
    parity = {}

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

    def sum_over_ranks(vals):
        if world == 1:
            return list(vals)
        t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if oversub else dev)
        dist.all_reduce(t)
        return [int(v) for v in t.tolist()]

    def add_parity(name, checked, bad):
        c, b = sum_over_ranks([checked, bad])
        parity[name] = {"checked": int(c), "mismatches": int(b)}

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
    # sampled bitwise parity of the gathered weights after the timed region
    add_parity("qwz", *sampled.qwz_check(out, world, shard_len, samples=4096, rng_seed=rank))
    # N = 1: one fused quantize->dequantize kernel; N > 1: quantize, barrier, TMA gather
    launches_per_step = 1 if world == 1 else 3
    value = world * 2 * M_PARAMS / t_step / 1e9
    qbytes = shard_len + shard_len // 2048 * 4
    busbw_qwz = 2 * M_PARAMS * (world - 1) / world / t_step / 1e9 if world > 1 else None

    # ---- per-kernel roofline (CUDA events around each kernel alone) ----------
    sym0 = [lib.zpp_comm_sym_ptr(comm.handle, r) for r in range(world)]
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
        nvl = traffic.get(f"nvlink_n{world}", {})
        roof = {"kernel": "dequant16_tma_kernel (gather over NVLink)", "bound": "nvlink", "achieved": ach,
                "peak": NVLINK_NOMINAL_GBS, "unit": "GB/s", "frac": ach / NVLINK_NOMINAL_GBS,
                # ncu of one rank under real peer traffic (tools/ncu_rank0.sh): NVLink rx
                # bytes of the gather per launch, at the GPT-13B-layer shape it was captured
                # at, scaled to this launch's algorithmic ingress
                "traffic": nvl.get("gather_nvlrx_per_alg_byte", None) and nvl["gather_nvlrx_per_alg_byte"] * ingress,
                "traffic_source": nvl.get("source"),
                "peak_kind": "NVLink 5 nominal, per direction (north_star)",
                "secondary": {"measured_peer_copy_gbs": NVLINK_PEER_GBS, "frac_peer_copy": ach / NVLINK_PEER_GBS,
                              "measured_tma_pull_gbs": TMA_PULL_GBS.get(world),
                              "frac_tma_pull": ach / TMA_PULL_GBS[world] if world in TMA_PULL_GBS else None},
                "alg_bytes_per_launch": ingress, "launch_us": kg * 1e6, "kernels": kern,
                "hbm": {"achieved": kern["dequant16_kernel (gather)"]["GBps"], "peak": hbm_peak,
                        "frac": kern["dequant16_kernel (gather)"]["GBps"] / hbm_peak}}

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
    del h_out, h_in, d_in

    # ---- comparators and qgZ ---------------------------------------------------
    extra = {}
    if world > 1 and not oversub:
        t_nccl = timed(lambda: nccl_allgather(shard, out=out), args.steps, 2)
        extra["nccl_fp16_allgather"] = {"value": world * 2 * M_PARAMS / t_nccl / 1e9, "unit": "GB/s",
                                        "ms_per_step": t_nccl * 1e3,
                                        "busbw_GBps": 2 * M_PARAMS * (world - 1) / world / t_nccl / 1e9}
    del out
    torch.cuda.empty_cache()
    def leg(name, fn):
        """Run one secondary leg; a failure is recorded in the line instead of
        losing the headline (the legs' arguments are identical on every rank,
        so a validation error is raised on all of them alike)."""
        try:
            extra[name] = fn()
        except Exception as e:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            extra[name] = {"error": f"{type(e).__name__}: {e}"[:400]}
            torch.cuda.synchronize()
        torch.cuda.empty_cache()

    kw = dict(world=world, rank=rank, dev=dev, timed=timed, steps=args.steps, hbm_peak=hbm_peak, synth=synth,
              sampled=sampled, add_parity=add_parity)
    if "qgz" in sections:
        leg("qgz", lambda: qgz_leg(comm=comm, X=X, oversub=oversub, nccl_reduce_scatter=nccl_reduce_scatter,
                                   traffic=traffic, **kw))
        if world >= 2 and X != world:
            # the same bucket with the whole box as one group (hop 2 a self-send)
            def one_group():
                c1g = Communicator(group_size=world, qgz_elems=QGZ_BUCKET, qgz_stages=1, qgz_cfg=qgz_cfg)
                try:
                    return qgz_leg(comm=c1g, X=world, oversub=oversub, nccl_reduce_scatter=None, traffic=traffic,
                                   parity_name="qgz_one_group", **kw)
                finally:
                    c1g.close()
            leg("qgz_one_group", one_group)
    comm.close()
    torch.cuda.empty_cache()
    if "config1" in sections:
        leg("config1_roundtrip_16M_fp32",
            lambda: config1_leg(lib=lib, dev=dev, rank=rank, timed_flush=None, steps=args.steps, hbm_peak=hbm_peak,
                                add_parity=add_parity, max_over_ranks=max_over_ranks, barrier=barrier, _lib=_lib))
    if "hpz" in sections:
        leg("hpz", lambda: hpz_leg(comm_cls=Communicator, world=world, dev=dev,
                                   timed=lambda f: timed(f, args.steps, 2), oversub=oversub,
                                   nccl_allgather=nccl_allgather, synth=synth, sampled=sampled,
                                   add_parity=add_parity, rank=rank))
    if "stream" in sections:
        leg("qgz_stream_7b", lambda: stream_leg(comm_cls=Communicator, X=X, zpp=zpp, **kw))
        if world >= 2 and X != world:
            # the whole box as one group: buckets pipelined (K1 of bucket b+1
            # beside the pull K2 of bucket b)
            leg("qgz_stream_7b_one_group", lambda: stream_leg(comm_cls=Communicator, X=world, zpp=zpp,
                                                              parity_name="qgz_stream_one_group", **kw))
    if "step" in sections:
        leg("zeropp_step_13b", lambda: step_leg(world=world, rank=rank, dev=dev, timed=timed, steps=args.steps,
                                                oversub=oversub, comm_cls=Communicator, zpp=zpp, synth=synth,
                                                sampled=sampled, add_parity=add_parity,
                                                nccl_allgather=nccl_allgather,
                                                nccl_reduce_scatter=nccl_reduce_scatter))
    kq_gbs = kern["quantize_reg_kernel"]["GBps"]
    extra["quant_kernel_hbm"] = {"kernel": "quantize_reg_kernel (K0: fp16 shard -> INT8/2048 codes + absmax)",
                                 "achieved_GBps": kq_gbs, "frac_of_8TBs_nominal": kq_gbs / 8000.0,
                                 "frac_of_measured_peak": kq_gbs / hbm_peak, "shard_elems": shard_len}
    extra["params_per_s"] = {"qwz": world * M_PARAMS / t_step,
                             "note": "whole-job parameters delivered per second (qgZ: see qgz.params_per_s)"}

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
                       "parallelism": f"zero3-dp{world}", "groups": f"{world // X}x{X}",
                       "inputs": "seeded counter-based generator (oracle/synth.py), generated on the device",
                       "l2": "inputs and outputs larger than L2 (shard + 2.6 GB fp16 output per step), no flush"}
                      | ({"oversubscribed": "functional check, ranks share GPUs: not a measurement"} if oversub else {}),
            "roofline": roof,
            "cpu_baseline": {"value": cpu_gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"{1 << 25} fp16 elements, numpy oracle port of zs/quantizer.py "
                                       "quantize+dequantize, block-parallel over host threads, median of 3"},
            "e2e": e2e, "clocks": clk, "gpu_launches": launches_per_step * args.steps,
            "busbw": {"qwz_GBps": busbw_qwz, "qgz_GBps": extra.get("qgz", {}).get("busbw_GBps"),
                      "definition": "SURVEY 8d collective effective GB/s: 2*M*(W-1)/W / t (fp16/bf16-equivalent "
                                    "bytes per GPU), NCCL busbw for the same collective; null at W=1"},
            "parity": parity | {"total_checked": sum(v["checked"] for v in parity.values()),
                                "total_mismatches": sum(v["mismatches"] for v in parity.values()),
                                "how": "after the timed regions: sampled outputs (whole 2048-blocks / 512-slices, "
                                       "summed over ranks) recomputed bitwise by the oracle from the seeded inputs"},
            "qwz": {"ms_per_step": t_step * 1e3,
                    "wire_ingress_bytes_per_gpu": (world - 1) * qbytes,
                    "fp16_allgather_ingress_bytes_per_gpu": (world - 1) * 2 * shard_len},
        }
        line.update(extra)
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def group_size_for(world: int) -> int:
    return world // 2 if world >= 2 else 1


def _pad(n: int, align: int) -> int:
    return (n + align - 1) // align * align


def qgz_bytes(n, world, X, in_block=512, out_block=512, final_bytes=4):
    """Per-GPU wire and algorithmic HBM bytes of one INT4 qgZ reduce-scatter of
    an n-element bf16 bucket: K1 reads bf16 and writes INT4 codes
    + fp32 absmax; K2 reads X messages of Y*L and writes Y*L INT4 codes + f64
    absmax (or, with one group, the fp32 partition); K3 reads Y segments of L
    and writes the fp32 partition."""
    Y = world // X
    L = n // world
    c4 = lambda m, b, a: m // 2 + m // b * a
    wire = (X - 1) * c4(Y * L, in_block, 4) + (Y - 1) * c4(L, out_block, 8)
    k1 = 2 * n + c4(n, in_block, 4)
    if Y == 1:
        k2 = X * c4(L, in_block, 4) + final_bytes * L
        k3 = 0
    else:
        k2 = X * c4(Y * L, in_block, 4) + c4(Y * L, out_block, 8)
        k3 = Y * c4(L, out_block, 8) + final_bytes * L
    return wire, k1 + k2 + k3


def qgz_leg(*, comm, world, rank, X, dev, timed, steps, hbm_peak, oversub, add_parity, synth, sampled,
            nccl_reduce_scatter, traffic, parity_name="qgz"):
    """BASELINE configs[3], one bucket: qgZ INT4/512 2-hop reduce-scatter of a
    256 MiB bf16 gradient bucket (S = 1), with its roofline
    t_roof = max(wire / 900 GB/s, HBM / peak)."""
    import torch

    grad = synth.device(2000 + 1000 * rank, 0, QGZ_BUCKET, torch.bfloat16, "grad", device=dev)
    part = torch.empty(QGZ_BUCKET // world, dtype=torch.float32, device=dev)
    t_qgz = timed(lambda: comm.qgz_reduce_scatter(grad, out=part), steps, 3)
    comm.check()
    add_parity(parity_name, *sampled.qgz_check(part, rank, world, X, QGZ_BUCKET, samples=4096))
    wire, hbm = qgz_bytes(QGZ_BUCKET, world, X)
    t_roof = max(wire / (NVLINK_NOMINAL_GBS * 1e9), hbm / (hbm_peak * 1e9))
    res = {"workload": "qgZ INT4/512 2-hop reduce-scatter of a 256 MiB bf16 bucket, S=1", "groups": f"{world // X}x{X}",
           "hop1": "K1 pushes (TMA bulk stores)" if world // X > 1 else "K2 pulls (TMA ring)",
           "ms_per_bucket": t_qgz * 1e3,
           "effective_GBps": world * 2 * QGZ_BUCKET / t_qgz / 1e9,
           "busbw_GBps": 2 * QGZ_BUCKET * (world - 1) / world / t_qgz / 1e9 if world > 1 else None,
           "params_per_s": world * QGZ_BUCKET / t_qgz,
           "wire_bytes_per_gpu": wire, "hbm_alg_bytes_per_gpu": hbm,
           "roofline": {"t_roof_us": t_roof * 1e6, "bound": "nvlink" if wire / 900e9 > hbm / (hbm_peak * 1e9) else "hbm",
                        "frac": t_roof / t_qgz, "nvlink_wire_GBps": wire / t_qgz / 1e9 if wire else None,
                        "nvlink_frac_of_900": wire / t_qgz / 1e9 / NVLINK_NOMINAL_GBS if wire else None,
                        "hbm_GBps": hbm / t_qgz / 1e9, "hbm_frac": hbm / t_qgz / 1e9 / hbm_peak,
                        "note": "t_roof = max(wire/900 GB/s, HBM/peak); the path is bound by neither: the bit-exact "
                                "f64 fold and the tie-checked quantizer are issue-bound (DESIGN.md, qgZ)"},
           "bf16_reduce_scatter_wire_bytes_per_gpu": 2 * QGZ_BUCKET * (world - 1) // world}
    if world > 1 and not oversub and nccl_reduce_scatter is not None:
        gb = grad.clone()
        pb = torch.empty(QGZ_BUCKET // world, dtype=torch.bfloat16, device=dev)
        t_rs = timed(lambda: nccl_reduce_scatter(gb, out=pb), steps, 3)
        res["nccl_bf16_reduce_scatter"] = {"ms_per_bucket": t_rs * 1e3,
                                           "busbw_GBps": 2 * QGZ_BUCKET * (world - 1) / world / t_rs / 1e9,
                                           "speedup_qgz_vs_nccl": t_rs / t_qgz}
        del gb, pb
    del grad, part
    return res


def config1_leg(*, lib, dev, rank, timed_flush, steps, hbm_peak, add_parity, max_over_ranks, barrier, _lib):
    """BASELINE configs[0]: INT8/2048 quantize -> dequantize round trip of a
    16M-element fp32 tensor (two kernels, fp32 out).  One set of buffers
    (64 MiB in, 16 MiB codes, 64 MiB out) fits in L2, so the round trips
    rotate over SETS independent buffer sets (> 6x L2 in total) and run back
    to back: every round trip reads inputs that left L2 long ago, and the
    write-back of its outputs is paid in the steady state, as in a stream."""
    import torch

    from oracle import synth, zpp_oracle as O

    n = 1 << 24
    nb = n // 2048
    SETS = 6
    xs = [synth.device(10 + rank + 100 * k, 0, n, torch.float32, "weight", device=dev) for k in range(SETS)]
    codes = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(SETS)]
    absmax = [torch.empty(nb, dtype=torch.float32, device=dev) for _ in range(SETS)]
    ys = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(SETS)]
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream

    def rt(k):
        lib.zpp_quantize(xs[k].data_ptr(), _lib.F32, n, 8, 2048, codes[k].data_ptr(), absmax[k].data_ptr(),
                         flag.data_ptr(), sp)
        lib.zpp_dequantize(codes[k].data_ptr(), absmax[k].data_ptr(), _lib.F32, n, 8, 2048, ys[k].data_ptr(), _lib.F32,
                           flag.data_ptr(), sp)

    for k in range(SETS):
        rt(k)
    barrier()
    reps = max(steps, 5) * SETS
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for i in range(reps):
        rt(i % SETS)
    e.record(st)
    e.synchronize()
    t = max_over_ranks(s.elapsed_time(e) / reps * 1e-3)
    if int(flag.item()):
        raise RuntimeError("config-1 round trip raised a device flag")
    alg = 2 * (4 * n + n + nb * 4)  # quantize: read fp32 + write codes + absmax; dequantize: the reverse
    # full-size parity on the host (rank 0's first set): codes and fp32 output bitwise
    if rank == 0:
        xh = synth.host(10, 0, n, "fp32", "weight")
        c_ref, s_ref, _ = O.quantize(xh, 8, 2048)
        y_ref = O.dequantize(c_ref, s_ref, n, 8, 2048).astype(np.float32)
        bad = int(np.count_nonzero(codes[0].cpu().numpy() != c_ref)) + \
            int(np.count_nonzero(ys[0].cpu().numpy().view(np.uint32) != y_ref.view(np.uint32)))
        add_parity("config1", 2 * n, bad)
    else:
        add_parity("config1", 0, 0)
    del xs, codes, absmax, ys
    torch.cuda.empty_cache()
    return {"workload": "INT8/2048 quantize->dequantize of 16,777,216 fp32 (zpp_quantize + zpp_dequantize)",
            "us_per_roundtrip": t * 1e6, "alg_bytes": alg,
            "roofline": {"bound": "hbm", "achieved": alg / t / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": alg / t / 1e9 / hbm_peak},
            "l2": f"{reps} back-to-back round trips rotating over {SETS} buffer sets ({SETS * 144} MiB > L2)"}


def hpz_leg(*, comm_cls, world, dev, timed, oversub, nccl_allgather, synth, sampled, add_parity, rank):
    """BASELINE configs[2]: hpZ gather of one GPT-1.3B layer (12h^2+13h, h=2048)
    inside a group of N/2 consecutive GPUs (2x4 on 8 GPUs), vs NCCL's full-box
    and group fp16 all-gathers.  The secondary shard is written through by the qwZ gather
    (zs/engine.py:364-370)."""
    import torch

    from paper_2306_10209_b200.dist import make_groups

    X = group_size_for(world)
    h = 2048
    layer = 12 * h * h + 13 * h
    layer_p = _pad(layer, world * 2048)
    sec = layer_p // X
    comm = comm_cls(group_size=X, qwz_shard=layer_p // world, hpz_sec=sec)
    w = synth.device(3000 + rank, 0, layer_p // world, torch.float16, "weight", device=dev)
    comm.qwz_allgather(w, write_secondary=True)
    comm.check()
    out = torch.empty(layer_p, dtype=torch.float16, device=dev)
    t = timed(lambda: comm.hpz_allgather(out=out))
    comm.check()
    # every group holds a full replica of the layer split over its X members
    # (zs/partitioner.py:67-82), so the group gather returns the whole layer
    add_parity("hpz", *sampled.qwz_check(out, world, layer_p // world, seed_base=3000, samples=2048, rng_seed=rank))
    comm.close()
    ingress = (X - 1) * sec * 2
    res = {"workload": "hpZ fp16 gather of one GPT-1.3B layer inside a group", "layer_params": layer,
           "padded": layer_p, "group_size": X, "ms": t * 1e3, "ingress_bytes_per_gpu": ingress,
           "ingress_GBps": ingress / t / 1e9, "nvlink_frac_of_900": ingress / t / 1e9 / NVLINK_NOMINAL_GBS,
           "cross_group_bytes": 0}
    if world > 1 and not oversub:
        full_out = torch.empty(layer_p, dtype=torch.float16, device=dev)
        res["nccl_fullbox_fp16_ag_ms"] = timed(lambda: nccl_allgather(w, out=full_out)) * 1e3
        if X < world:
            group_pg, _ = make_groups(X)
            gs = torch.empty(sec, dtype=torch.float16, device=dev)
            res["nccl_group_fp16_ag_ms"] = timed(lambda: nccl_allgather(gs, out=out, group=group_pg)) * 1e3
    return res


def stream_leg(*, comm_cls, world, rank, X, dev, timed, steps, hbm_peak, synth, sampled, add_parity, zpp,
               parity_name="qgz_stream"):
    """BASELINE configs[3] as written: qgZ INT4/512 over a 7B-parameter bf16
    gradient stream -- 52 buckets of 256 MiB plus a 20,678,144-element tail
    zero-padded to W*S*512 (zs/engine.py:465-466) -- back to back through
    Communicator.qgz_reduce_scatter_stream."""
    import torch

    n_total = 7_000_000_000
    comm = comm_cls(group_size=X, qgz_elems=QGZ_BUCKET, qgz_stages=1,
                    qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    full, tail, tail_pad, n_out = comm.stream_layout(n_total)
    grads = torch.empty(n_total, dtype=torch.bfloat16, device=dev)
    for b in range(full + 1):
        lo = b * QGZ_BUCKET
        synth.device(2000 + 1000 * rank + b, 0, min(QGZ_BUCKET, n_total - lo), torch.bfloat16, "grad",
                     out=grads[lo:lo + QGZ_BUCKET])
    out = torch.empty(n_out, dtype=torch.float32, device=dev)
    t = timed(lambda: comm.qgz_reduce_scatter_stream(grads, out=out), max(2, min(steps // 5, 4)), 1)
    comm.check()
    per = QGZ_BUCKET // world
    chk = bad = 0
    for b in range(0, full, 13):  # a few buckets, and the padded tail
        c, m = sampled.qgz_check(out[b * per:(b + 1) * per], rank, world, X, QGZ_BUCKET, seed_base=2000 + b,
                                 samples=256, rng_seed=b)
        chk, bad = chk + c, bad + m
    c, m = sampled.qgz_check(out[full * per:], rank, world, X, tail_pad, seed_base=2000 + full, samples=512,
                             valid=tail)
    add_parity(parity_name, chk + c, bad + m)
    comm.close()
    del grads, out
    torch.cuda.empty_cache()
    wire_b, hbm_b = qgz_bytes(QGZ_BUCKET, world, X)
    wire_t, hbm_t = qgz_bytes(tail_pad, world, X)
    wire, hbm = full * wire_b + wire_t, full * hbm_b + hbm_t
    t_roof = max(wire / (NVLINK_NOMINAL_GBS * 1e9), hbm / (hbm_peak * 1e9))
    return {"workload": "qgZ INT4/512 over a 7B bf16 gradient stream: 52 x 256 MiB buckets + padded tail",
            "params": n_total, "buckets": full, "tail": tail, "tail_padded": tail_pad, "groups": f"{world // X}x{X}",
            "buckets_pipelined": world > 1 and X == world,
            "ms_per_step": t * 1e3, "effective_GBps": world * 2 * n_total / t / 1e9,
            "busbw_GBps": 2 * n_total * (world - 1) / world / t / 1e9 if world > 1 else None,
            "params_per_s": world * n_total / t,
            "roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof / t,
                         "nvlink_frac_of_900": wire / t / 1e9 / NVLINK_NOMINAL_GBS if wire else None,
                         "hbm_frac": hbm / t / 1e9 / hbm_peak},
            "wire_bytes_per_gpu": wire, "bf16_reduce_scatter_wire_bytes_per_gpu": 2 * n_total * (world - 1) // world}


def step_leg(*, world, rank, dev, timed, steps, oversub, comm_cls, zpp, synth, sampled, add_parity, nccl_allgather,
             nccl_reduce_scatter):
    """BASELINE configs[4]: the communication of a ZeRO++ step over a GPT-13B
    layer stack (h = 5120, 40 layers; zs/engine.py:345-398 order): forward qwZ
    (INT8/2048) layer by layer writing each layer's hpZ secondary, backward hpZ
    gathers inside the group in reverse layer order, gradient qgZ (INT4/512,
    S = 1, the measured optimum) per layer -- with and without the cross-layer prefetch of the next
    layer's quantization -- vs ZeRO-3's fp16 all-gather x2 + bf16
    reduce-scatter per layer (NCCL)."""
    import torch

    X = group_size_for(world)
    h = 5120
    n_layers = 40
    layer = 12 * h * h + 13 * h
    layer_p = _pad(layer, world * 2048 * 4)
    shard = layer_p // world
    comm = comm_cls(group_size=X, qwz_shard=shard, hpz_sec=layer_p // X, hpz_layers=n_layers, qgz_elems=layer_p,
                    qgz_stages=1, qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    ws = [synth.device(3000 + 100 * i + rank, 0, shard, torch.float16, "weight", device=dev) for i in range(n_layers)]
    g = synth.device(5000 + 1000 * rank, 0, layer_p, torch.bfloat16, "grad", device=dev)
    wout = torch.empty(layer_p, dtype=torch.float16, device=dev)
    hout = torch.empty(layer_p, dtype=torch.float16, device=dev)
    gout = torch.empty(layer_p // world, dtype=torch.float32, device=dev)

    def zeropp_step(prefetch):
        for i in range(n_layers):  # forward
            comm.qwz_allgather(ws[i], out=wout, write_secondary=True, layer=i,
                               next_shard=ws[i + 1] if prefetch and i + 1 < n_layers else None)
        for i in reversed(range(n_layers)):  # backward
            comm.hpz_allgather(out=hout, layer=i)
            comm.qgz_reduce_scatter(g, out=gout)

    n_steps = max(2, min(steps // 5, 3))
    t_pf = timed(lambda: zeropp_step(True), n_steps, 1)
    t_no = timed(lambda: zeropp_step(False), n_steps, 1)
    comm.check()
    # after the last step: wout = layer 39 (forward), hout = layer 0 (backward)
    c1, b1 = sampled.qwz_check(wout, world, shard, seed_base=3000 + 100 * (n_layers - 1), samples=1024, rng_seed=rank)
    c2, b2 = sampled.qwz_check(hout, world, shard, seed_base=3000, samples=1024, rng_seed=rank + 7)
    c3, b3 = sampled.qgz_check(gout, rank, world, X, layer_p, stages=1, seed_base=5000, samples=1024)
    add_parity("step_13b", c1 + c2 + c3, b1 + b2 + b3)
    comm.close()
    res = {"workload": "fwd qwZ (prefetched) + bwd hpZ + grad qgZ (S=1) over 40 GPT-13B layers", "layers": n_layers,
           "layer_params": layer, "padded": layer_p, "groups": f"{world // X}x{X}",
           "zeropp_ms": t_pf * 1e3, "zeropp_no_prefetch_ms": t_no * 1e3, "prefetch_gain": t_no / t_pf}
    if world > 1 and not oversub:
        bout = torch.empty(layer_p // world, dtype=torch.bfloat16, device=dev)
        gb = g.clone()

        def zero3_step():
            for i in range(n_layers):
                nccl_allgather(ws[i], out=wout)
            for i in reversed(range(n_layers)):
                nccl_allgather(ws[i], out=hout)
                nccl_reduce_scatter(gb, out=bout)

        t3 = timed(zero3_step, n_steps, 1)
        res.update({"zero3_nccl_ms": t3 * 1e3, "speedup_vs_zero3": t3 / t_pf})
        del bout, gb
    del ws, g, wout, hout, gout
    torch.cuda.empty_cache()
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
