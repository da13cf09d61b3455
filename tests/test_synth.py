"""CPU checks of the sampled-parity machinery used at full BASELINE sizes:
the counter-based input generator (oracle/synth.py) gives the same bits from
torch and numpy, and the per-slice qgZ oracle equals the whole-tensor oracle
(which the reference goldens pin, tests/test_oracle.py)."""

import numpy as np
import pytest
import torch

from oracle import synth as S
from oracle import zpp_oracle as O


@pytest.mark.parametrize("kind,dt,tdt", [("weight", "fp16", torch.float16), ("grad", "bf16", torch.bfloat16),
                                         ("weight", "fp32", torch.float32), ("grad", "fp16", torch.float16)])
def test_generator_torch_equals_numpy(kind, dt, tdt):
    for seed, lo in ((0, 0), (7, 123_456_789), (3005, (1 << 33) + 17)):
        a = S.host(seed, lo, 200_000, dt, kind)
        b = S.device(seed, lo, 200_000, tdt, kind, device="cpu", chunk=65_536).double().numpy()
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        idx = np.array([lo, lo + 5, lo + 199_999])
        assert np.array_equal(S.host_at(seed, idx, dt, kind), a[[0, 5, 199_999]])
    assert np.all(np.isfinite(a)) and np.abs(a).max() > 0


def test_generator_has_ties_and_spread():
    g = S.host(1, 0, 1 << 16, "bf16", "grad")
    assert len(np.unique(np.abs(g))) > 1000
    assert np.abs(g).max() / np.median(np.abs(g)) > 10  # heavy-ish tail


@pytest.mark.parametrize("x,y,s", [(2, 2, 1), (4, 2, 1), (1, 2, 2), (2, 1, 2), (4, 1, 1), (2, 2, 2)])
@pytest.mark.parametrize("bits", [(4, 512, 4, 512), (8, 256, 4, 512)])
def test_slice_oracle_equals_whole_tensor_oracle(x, y, s, bits):
    intra_bits, intra_block, inter_bits, inter_block = bits
    w = x * y
    L = 3 * 512
    n = s * w * L
    grads = [S.host(2000 + 1000 * r, 0, n, "bf16", "grad") for r in range(w)]
    whole = O.qgz_2hop(grads, x, y, s, inter_bits, inter_block, intra_bits, intra_block)
    part = s * L
    rng = np.random.default_rng(0)
    for r in range(w):
        # sampled 512-element output slices of rank r (any order, any subset)
        sl = rng.choice(part // 512, size=min(4, part // 512), replace=False)
        pos = (sl[:, None] * 512 + np.arange(512)[None, :]).reshape(-1)
        src = np.stack([grads[q][r * part + pos] for q in range(w)])
        got = O.qgz_2hop_slices(src, x, y, inter_bits, inter_block, intra_bits, intra_block)
        assert np.array_equal(got.view(np.uint64), whole[r][pos].view(np.uint64))


def test_sampled_checks_on_host_tensors():
    """The sampled checkers' index logic against whole-tensor oracle outputs
    held in CPU tensors (the GPU workers pass CUDA tensors)."""
    from oracle import sampled

    world, shard = 3, 5 * 2048 + 1000
    shards = [S.host(1000 + r, 0, shard, "fp16", "weight") for r in range(world)]
    want, _ = O.all_gather_qwz(shards, 8, 2048)
    out = torch.from_numpy(want.astype(np.float16))
    checked, bad = sampled.qwz_check(out, world, shard, samples=64)
    assert checked > 0 and bad == 0
    # hpZ view: elements [lo, hi) only
    lo, hi = shard, 3 * shard
    checked, bad = sampled.qwz_check(out[lo:hi], world, shard, samples=64, lo=lo, hi=hi)
    assert checked > 0 and bad == 0
    flip = out.clone()
    flip[2048 * 2 + 7] = -flip[2048 * 2 + 7] + 1
    _, bad = sampled.qwz_check(flip, world, shard, samples=4096)
    assert bad == 1
    # qgZ partitions of a 2x2 run, S = 2
    x, y, s = 2, 2, 2
    n = s * x * y * 4 * 512
    grads = [S.host(2000 + 1000 * q, 0, n, "bf16", "grad") for q in range(x * y)]
    parts = O.qgz_2hop(grads, x, y, s, 4, 512)
    for r in range(x * y):
        for dt in (np.float64, np.float32):
            checked, bad = sampled.qgz_check(torch.from_numpy(parts[r].astype(dt)), r, x * y, x, n, stages=s,
                                             samples=3)
            assert checked >= 512 and bad == 0
