"""Runs ONE hot-path kernel at its benchmark size (2 warm-up launches + 1
measured launch) so that `ncu -k regex:<kernel> -s 2 -c 1` captures exactly
that kernel.  Used by tools/profile_round.sh; also prints CUDA-event timings
and algorithmic GB/s when run without ncu.

    python tools/profile_kernels.py <case>

cases:
  qwz1     fused quantize->dequantize of the 1.3B fp16 buffer (bench N = 1 step)
  k0       K0 quantize of a 1.3B/4 fp16 shard, INT8/2048 (qwZ at N = 4)
  gather4  K4 TMA gather-dequantize of 4 INT8/2048 shards -> 1.3B fp16
           (the N = 4 gather with local instead of peer sources)
  k1       K1 swizzle-quantize of a 256 MiB bf16 bucket, INT4/512, 2x4 layout
  k2       K2 dequant->f64 fold->requant of 4 INT4/512 messages of 33.5M
  k3       K3 dequant->f64 fold of 2 INT4/512 (f64 absmax) segments -> fp32
  c1q      config 1: quantize 16M fp32 -> INT8/2048
  c1d      config 1: dequantize 16M INT8/2048 -> fp32
  qgz1     qgZ of one 256 MiB bf16 bucket in a 1-GPU world (K1 + K2 with the
           final fp32 output), INT4/512
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_10209_b200 as zpp  # noqa: E402
from paper_2306_10209_b200 import _lib  # noqa: E402
from paper_2306_10209_b200.dist import Communicator  # noqa: E402

M = 1_300_004_864
BUCKET = 134_217_728


def timed(fn, reps):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    case = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    if case == "qwz1":
        comm = Communicator(group_size=1, qwz_shard=M, qwz_cfg=zpp.QuantConfig(bit_width=8, block_size=2048))
        x = (torch.randn(M, generator=g, device=dev) * 0.02).half()
        out = torch.empty(M, dtype=torch.float16, device=dev)
        fn = lambda: comm.qwz_allgather(x, out=out)  # noqa: E731
        alg = 4 * M + M + M // 2048 * 4
    elif case == "k0":
        n = M // 4
        x = (torch.randn(n, generator=g, device=dev) * 0.02).half()
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        am = torch.empty(n // 2048, dtype=torch.float32, device=dev)
        fn = lambda: lib.zpp_quantize(x.data_ptr(), _lib.F16, n, 8, 2048, codes.data_ptr(), am.data_ptr(),  # noqa: E731
                                      flag.data_ptr(), st)
        alg = 2 * n + n + n // 2048 * 4
    elif case == "gather4":
        n = M // 4
        x = (torch.randn(n, generator=g, device=dev) * 0.02).half()
        codes = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
        ams = [torch.empty(n // 2048, dtype=torch.float32, device=dev) for _ in range(4)]
        for c, a in zip(codes, ams):
            lib.zpp_quantize(x.data_ptr(), _lib.F16, n, 8, 2048, c.data_ptr(), a.data_ptr(), flag.data_ptr(), st)
        out = torch.empty(M, dtype=torch.float16, device=dev)
        cp, _k1 = _lib.ptr_array([c.data_ptr() for c in codes])
        ap, _k2 = _lib.ptr_array([a.data_ptr() for a in ams])
        fn = lambda: lib.zpp_gather_dequantize(cp, ap, _lib.F32, 4, 0, n, 8, 2048, out.data_ptr(), _lib.F16, n,  # noqa: E731
                                               None, 0, 0, flag.data_ptr(), st)
        alg = 4 * (n + n // 2048 * 4) + 2 * M
    elif case == "k1":
        x = (torch.randn(BUCKET, generator=g, device=dev) * 1e-3).bfloat16()
        codes = torch.empty(BUCKET // 2, dtype=torch.uint8, device=dev)
        am = torch.empty(BUCKET // 512, dtype=torch.float32, device=dev)
        fn = lambda: lib.zpp_swizzle_quantize(x.data_ptr(), _lib.BF16, BUCKET, 4, 2, 1, 0, 1, 4, 512,  # noqa: E731
                                              codes.data_ptr(), am.data_ptr(), flag.data_ptr(), st)
        alg = 2 * BUCKET + BUCKET // 2 + BUCKET // 512 * 4
    elif case in ("k2", "k3"):
        n_src, n = (4, BUCKET // 4) if case == "k2" else (2, BUCKET // 8)
        cfg = zpp.QuantConfig(bit_width=4, block_size=512)
        qs = [zpp.quantize((torch.randn(n, generator=g, device=dev) * 1e-3).float(), cfg) for _ in range(n_src)]
        if case == "k2":
            fn = lambda: zpp.fused_dequant_reduce_quant(qs, cfg, flag=flag)  # noqa: E731
            alg = n_src * (n // 2 + n // 512 * 4) + n // 2 + n // 512 * 8
        else:
            q64 = [zpp.fused_dequant_reduce_quant([q], cfg) for q in qs]  # f64 absmax, as in hop 2
            out = torch.empty(n, dtype=torch.float32, device=dev)
            fn = lambda: zpp.dequant_reduce(q64, torch.float32, out=out, flag=flag)  # noqa: E731
            alg = n_src * (n // 2 + n // 512 * 8) + 4 * n
    elif case == "qgz1":
        comm = Communicator(group_size=1, qgz_elems=BUCKET, qgz_stages=1,
                            qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
        gr = (torch.randn(BUCKET, generator=g, device=dev) * 1e-3).bfloat16()
        part = torch.empty(BUCKET, dtype=torch.float32, device=dev)
        fn = lambda: comm.qgz_reduce_scatter(gr, out=part)  # noqa: E731
        alg = 2 * BUCKET + BUCKET // 2 + BUCKET // 512 * 4 + BUCKET // 2 + BUCKET // 512 * 4 + 4 * BUCKET
    elif case in ("c1q", "c1d"):
        n = 1 << 24
        x = torch.randn(n, generator=g, device=dev) * 0.02
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        am = torch.empty(n // 2048, dtype=torch.float32, device=dev)
        y = torch.empty(n, dtype=torch.float32, device=dev)
        q = lambda: lib.zpp_quantize(x.data_ptr(), _lib.F32, n, 8, 2048, codes.data_ptr(), am.data_ptr(),  # noqa: E731
                                     flag.data_ptr(), st)
        q()
        if case == "c1q":
            fn = q
        else:
            fn = lambda: lib.zpp_dequantize(codes.data_ptr(), am.data_ptr(), _lib.F32, n, 8, 2048,  # noqa: E731
                                            y.data_ptr(), _lib.F32, flag.data_ptr(), st)
        alg = 5 * n + n // 2048 * 4
    else:
        raise SystemExit(f"unknown case {case}")
    fn()
    fn()
    torch.cuda.synchronize()
    t = timed(fn, reps)
    if int(flag.item()):
        raise SystemExit(f"device flag {int(flag.item())}")
    print(json.dumps({"case": case, "us": t * 1e6, "alg_bytes": alg, "GBps": alg / t / 1e9}), flush=True)


if __name__ == "__main__":
    main()
