"""Per-kernel device timings (CUDA events on the launching stream) for the
codec kernels at BASELINE shapes.  Prints algorithmic GB/s and the fraction of
the measured HBM copy peak.  Development aid; bench.py is the contract."""

from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_10209_b200 as zpp  # noqa: E402
from paper_2306_10209_b200 import _lib  # noqa: E402

PEAK = 6539.2
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass


def timeit(fn, iters=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def report(name, sec, nbytes):
    gbs = nbytes / sec / 1e9
    print(f"{name:48s} {sec * 1e6:10.1f} us {gbs:9.1f} GB/s  {gbs / PEAK:6.1%} of HBM")


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else "all"
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    if only == "fused":
        return fused_n1(lib, st, flag)
    cases = [(torch.float16, 1_300_004_864, 8, 2048), (torch.float32, 1 << 24, 8, 2048),
             (torch.bfloat16, 134_217_728, 4, 512), (torch.float16, 134_217_728, 8, 2048)]
    if only == "qgz":
        cases = []
    elif only == "codec":
        cases = cases[2:4]
    for (dt, n, bits, block) in cases:
        x = (torch.randn(n, device="cuda", dtype=torch.float32) * 0.02).to(dt)
        q = zpp.quantize(x, zpp.QuantConfig(bit_width=bits, block_size=block))
        code = zpp.quantizer.dtype_code(dt)
        esz = x.element_size()
        nb = q.n_blocks

        def qfn():
            lib.zpp_quantize(x.data_ptr(), code, n, bits, block, q.codes.data_ptr(), q.absmax.data_ptr(),
                             flag.data_ptr(), st)
        t = timeit(qfn)
        report(f"quantize {dt} n={n} int{bits}/{block}", t, n * esz + q.codes.numel() + nb * 4)
        for odt in (torch.float16, torch.float32):
            out = torch.empty(n, dtype=odt, device="cuda")

            def dfn():
                lib.zpp_dequantize(q.codes.data_ptr(), q.absmax.data_ptr(), _lib.F32, n, bits, block,
                                   out.data_ptr(), zpp.quantizer.dtype_code(odt), flag.data_ptr(), st)
            t = timeit(dfn)
            report(f"dequantize -> {odt}", t, n * out.element_size() + q.codes.numel() + nb * 4)
            del out
        del x, q
        torch.cuda.empty_cache()
    if only == "codec":
        return
    # qgZ kernels at the bucket shapes of W=8 (X=4, Y=2) and W=4 (2x2), emulated
    # on one GPU (all sources local)
    for X, Y in ((4, 2), (2, 2)):
        qgz_shape(lib, st, flag, X, Y)
    torch.cuda.synchronize()
    print("flag", int(flag.item()))


def fused_n1(lib, st, flag):
    """The N = 1 qwZ step (one fused quantize -> dequantize pass over the 1.3B
    fp16 buffer) on two input distributions: torch.randn * 0.02 and the
    bench's counter-based synthetic weights (oracle/synth.py), 20 back-to-back
    launches each, like bench.py's timed region."""
    from oracle import synth
    from paper_2306_10209_b200.dist import Communicator

    M = 1_300_004_864
    comm = Communicator(group_size=1, qwz_shard=M, qwz_cfg=zpp.QuantConfig(bit_width=8, block_size=2048))
    out = torch.empty(M, dtype=torch.float16, device="cuda")
    for name, mk in (("randn*0.02", lambda: (torch.randn(M, device="cuda") * 0.02).half()),
                     ("synth", lambda: synth.device(1000, 0, M, torch.float16, "weight", device=torch.device("cuda")))):
        x = mk()
        # ZPP_MB_WARM_S: keep the GPU busy on the same pass for that many
        # seconds first (bench.py runs ~0.5 s of steps before its timed region)
        warm = 5 + int(float(os.environ.get("ZPP_MB_WARM_S", "0")) / 1.1e-3)
        t = timeit(lambda: comm.qwz_allgather(x, out=out), iters=20, warm=warm)
        report(f"fused N=1 qwZ pass, {name}", t, 5 * M + M // 2048 * 4)
        del x
        torch.cuda.empty_cache()
    comm.check()
    comm.close()


def qgz_shape(lib, st, flag, X, Y):
    n = 134_217_728
    g = (torch.randn(n, device="cuda") * 1e-3).bfloat16()
    S = 1
    L = n // (S * X * Y)
    send = zpp.quantizer.alloc_quantized(X * Y * L, zpp.QuantConfig(bit_width=4, block_size=512))

    def k1():
        lib.zpp_swizzle_quantize(g.data_ptr(), _lib.BF16, n, X, Y, S, 0, 1, 4, 512, send.codes.data_ptr(),
                                 send.absmax.data_ptr(), flag.data_ptr(), st)
    t = timeit(k1)
    report("K1 swizzle-quantize bf16 134M int4/512", t, n * 2 + send.codes.numel() + send.n_blocks * 4)
    msg = Y * L
    ins = [send.slice_blocks(j * msg, msg) for j in range(X)]
    out = zpp.quantizer.alloc_quantized(msg, zpp.QuantConfig(bit_width=4, block_size=512), torch.float64)
    cp, k_a = _lib.ptr_array([q.codes.data_ptr() for q in ins])
    ap, k_b = _lib.ptr_array([q.absmax.data_ptr() for q in ins])

    def k2():
        lib.zpp_dequant_reduce_quant(cp, ap, _lib.F32, X, msg, 4, 512, 4, 512, out.codes.data_ptr(),
                                     out.absmax.data_ptr(), None, 0, flag.data_ptr(), st)
    t = timeit(k2)
    report(f"K2 dequant-reduce-requant X={X} n={msg}", t,
           X * (msg // 2 + msg // 512 * 4) + msg // 2 + msg // 512 * 8)
    segs = [out.slice_blocks(c * L, L) for c in range(Y)]
    res = torch.empty(L, dtype=torch.float32, device="cuda")
    cp3, k_c = _lib.ptr_array([q.codes.data_ptr() for q in segs])
    ap3, k_d = _lib.ptr_array([q.absmax.data_ptr() for q in segs])

    def k3():
        lib.zpp_dequant_reduce(cp3, ap3, _lib.F64, Y, L, 4, 512, res.data_ptr(), _lib.F32, 1.0, flag.data_ptr(), st)
    t = timeit(k3)
    report(f"K3 dequant-reduce Y={Y} n={L}", t, Y * (L // 2 + L // 512 * 8) + L * 4)


if __name__ == "__main__":
    main()
