"""The fused-collective code path on one GPU (world = 1, no torch.distributed):
symmetric workspace, double buffering and the three collectives, bit-exact vs
the oracle."""

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle import zpp_oracle as O

pytestmark = pytest.mark.gpu


def test_world1_collectives():
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200.dist import Communicator

    n = 5 * 2048 + 777
    comm = Communicator(qwz_shard=n, hpz_sec=n, qgz_elems=4096, qgz_stages=2,
                        qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    assert comm.world == 1 and comm.group_size == 1
    x = (np.random.default_rng(0).normal(size=n) * 0.05).astype(np.float16)
    want, _ = O.all_gather_qwz([x.astype(np.float64)], 8, 2048)
    for _ in range(3):
        out = comm.qwz_allgather(torch.from_numpy(x).cuda(), write_secondary=True)
        comm.check()
        assert np.array_equal(out.cpu().numpy(), want.astype(np.float16))
        assert np.array_equal(comm.secondary.cpu().numpy(), want.astype(np.float16))
        assert np.array_equal(comm.hpz_allgather().cpu().numpy(), want.astype(np.float16))
    h_out = torch.empty(n, dtype=torch.float16).pin_memory()
    comm.qwz_allgather_host(torch.from_numpy(x).pin_memory(), h_out, chunks=4)
    torch.cuda.synchronize()
    assert np.array_equal(h_out.numpy(), want.astype(np.float16))
    g = (np.random.default_rng(1).normal(size=4096) * 1e-3).astype(np.float32)
    ref = O.qgz_2hop([g.astype(np.float64)], 1, 1, 2, 4, 512)[0]
    for _ in range(3):
        o = comm.qgz_reduce_scatter(torch.from_numpy(g).cuda(), out_dtype=torch.float64)
        comm.check()
        assert np.array_equal(o.cpu().numpy(), ref)
    bad = torch.from_numpy(x).cuda()
    bad[7] = float("nan")
    comm.qwz_allgather(bad)
    with pytest.raises(zpp.ValidationError):
        comm.check()
    with pytest.raises(zpp.ValidationError):
        comm.qwz_allgather(torch.zeros(n + 8, device="cuda", dtype=torch.float16))
    # raw-pointer boundary: undersized / host / strided buffers are rejected before launch
    xs = torch.from_numpy(x).cuda()
    with pytest.raises(zpp.ValidationError):
        comm.qwz_allgather(xs, out=torch.empty(n - 1, dtype=torch.float16, device="cuda"))
    with pytest.raises(zpp.ValidationError):
        comm.qwz_allgather(torch.from_numpy(x))
    with pytest.raises(zpp.ValidationError):
        comm.qgz_reduce_scatter(torch.zeros(8192, device="cuda")[::2])
    with pytest.raises(zpp.ValidationError):
        comm.hpz_allgather(out=torch.empty(n, dtype=torch.float32, device="cuda"))
    comm.close()


@pytest.mark.parametrize("dtype,bits,block", [("fp16", 8, 2048), ("bf16", 8, 2048), ("fp16", 4, 512),
                                              ("bf16", 4, 1024)])
def test_world1_fused_round_trip(dtype, bits, block):
    """1-GPU qwZ takes the fused quantize->dequantize pass (codes still land in
    the symmetric buffer); output = the reference's value rounded once."""
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200.dist import Communicator

    n = 37 * block + 776  # partial last block, n % 8 == 0
    rng = np.random.default_rng(bits * block)
    v = rng.normal(size=n) * np.exp(rng.normal(size=n) * 2) * 0.02
    arr = v.astype(np.float16) if dtype == "fp16" else (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    x = gu.to_torch(arr, dtype)
    comm = Communicator(qwz_shard=n, qwz_cfg=zpp.QuantConfig(bit_width=bits, block_size=block))
    out = comm.qwz_allgather(x, out_dtype=x.dtype)
    comm.check()
    want, _ = O.all_gather_qwz([gu.as_f64(arr, dtype)], bits, block)
    got = out.to(torch.float64).cpu().numpy()
    assert np.array_equal(got, gu.round_to(want, dtype))
    comm.close()


def test_stage_tracer():
    """zpp_comm_trace: one event per launched stage of the last qgZ / qwZ
    call, in launch order, with non-decreasing times (diagnostics used by
    tools/stage_timeline.py)."""
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200.dist import Communicator

    comm = Communicator(qwz_shard=4096, qgz_elems=8192, qgz_stages=2,
                        qgz_cfg=zpp.QuantConfig(bit_width=4, block_size=512))
    g = torch.randn(8192, device="cuda").bfloat16()
    comm.qgz_reduce_scatter(g)
    assert comm.trace_read() == []  # tracing off: nothing recorded
    comm.trace(True)
    comm.qgz_reduce_scatter(g)
    tr = comm.trace_read()
    assert [s for s, _ in tr] == ["begin", "K1", "barrier", "K2", "K1", "barrier", "K2"]
    assert all(b >= a for (_, a), (_, b) in zip(tr, tr[1:]))
    comm.qwz_allgather(torch.randn(4096, device="cuda").half())
    assert [s for s, _ in comm.trace_read()] == ["begin"]  # world of 1: one fused launch
    comm.trace(False)
    comm.check()
    comm.close()
