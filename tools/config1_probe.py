"""Config 1 (16M fp32, INT8/2048 quantize -> dequantize) split per kernel and
per L2-flush method: CUDA events around each kernel after (a) a 512 MiB
write flush (dirty L2 lines), (b) a 512 MiB read flush (clean lines), (c) no
flush.  Development aid for bench.py's config-1 leg."""

from __future__ import annotations

import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_10209_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    n = 1 << 24
    nb = n // 2048
    x = torch.randn(n, device="cuda") * 0.02
    codes = torch.empty(n, dtype=torch.uint8, device="cuda")
    absmax = torch.empty(nb, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    bigf = big.view(torch.float32)
    st = torch.cuda.current_stream().cuda_stream

    def q():
        lib.zpp_quantize(x.data_ptr(), _lib.F32, n, 8, 2048, codes.data_ptr(), absmax.data_ptr(), flag.data_ptr(), st)

    def d():
        lib.zpp_dequantize(codes.data_ptr(), absmax.data_ptr(), _lib.F32, n, 8, 2048, y.data_ptr(), _lib.F32,
                           flag.data_ptr(), st)

    def rt():
        q()
        d()

    flushes = {"write": lambda: big.fill_(1), "read": lambda: bigf.sum(), "write+read": lambda: (big.fill_(1), bigf[: (256 << 20) // 4].sum()),
               "none": lambda: None}
    for fname, fl in flushes.items():
        for kname, fn, alg in (("quantize", q, 5 * n + 4 * nb), ("dequantize", d, 5 * n + 4 * nb),
                               ("round trip", rt, 10 * n + 8 * nb)):
            for _ in range(3):
                fl()
                fn()
            ts = []
            for _ in range(20):
                fl()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fn()
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e) * 1e-3)
            t = statistics.median(ts)
            print(f"flush={fname:10s} {kname:11s} {t * 1e6:8.1f} us  {alg / t / 1e9:8.1f} GB/s")
    assert int(flag.item()) == 0


if __name__ == "__main__":
    main()
