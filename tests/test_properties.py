"""Property tests (hypothesis, CPU) of the host-side invariants the kernels rely
on: partitions tile the buffer, the qgZ reorder map is a permutation whose
inverse undoes it and that groups destinations by local rank, the wire
accounting agrees with the oracle for any length, and the oracle's quantizer
respects its own error bound."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import zpp_oracle as O

settings.register_profile("zpp", max_examples=60, deadline=None)
settings.load_profile("zpp")


@given(total=st.integers(1, 10_000), nodes=st.integers(1, 4), gpn=st.integers(1, 4))
def test_partitions_tile_the_buffer(total, nodes, gpn):
    import paper_2306_10209_b200 as zpp

    world = nodes * gpn
    spec = zpp.PartitionSpec(total_elems=total, world=world, group_size=gpn)
    prim = [spec.primary_range(r) for r in range(world)]
    assert prim[0][0] == 0 and prim[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(prim, prim[1:]))
    sizes = [hi - lo for lo, hi in prim]
    assert max(sizes) - min(sizes) <= 1
    for g in spec.groups():
        sec = [spec.secondary_range(r) for r in g]
        assert sec[0][0] == 0 and sec[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(sec, sec[1:]))
    assert [spec.primary_range(r) for r in range(world)] == [O.primary_range(total, world, r) for r in range(world)]


@given(x=st.integers(1, 8), y=st.integers(1, 8), s=st.integers(1, 4))
def test_reorder_mapping_is_an_invertible_grouping(x, y, s):
    import paper_2306_10209_b200 as zpp

    p = zpp.reorder_mapping(x, y, s)
    n = x * y * s
    assert sorted(p.forward.tolist()) == list(range(n))
    assert np.array_equal(p.forward[p.inverse], np.arange(n)) and np.array_equal(p.inverse[p.forward], np.arange(n))
    fwd, inv = O.reorder_mapping(x, y, s)
    assert np.array_equal(p.forward, fwd) and np.array_equal(p.inverse, inv)


@given(n=st.integers(0, 50_000), bits=st.sampled_from([4, 8]), block=st.integers(1, 512).map(lambda b: 8 * b),
       mode=st.sampled_from(["blocked", "full_tensor"]))
def test_wire_accounting_matches_oracle(n, bits, block, mode):
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200.accounting import encode_sizes

    codec = zpp.BlockCodec(zpp.QuantConfig(bit_width=bits, block_size=block, mode=mode))
    assert encode_sizes(codec, n) == O.accounting(n, bits, block, mode)


@given(seed=st.integers(0, 2**31 - 1), bits=st.sampled_from([4, 8]), block=st.sampled_from([8, 24, 64, 512]),
       n=st.integers(1, 3000), scale=st.floats(1e-30, 1e30))
def test_oracle_round_trip_error_is_half_a_step(seed, bits, block, n, scale):
    """|dequant(quant(x)) - x| <= scale_b / 2 per block (zs/quantizer.py:204-238)."""
    x = np.random.default_rng(seed).normal(size=n) * scale
    codes, scales, _ = O.quantize(x, bits, block)
    y = O.dequantize(codes, scales, n, bits, block)
    per_elem = np.repeat(scales, block)[:n]
    assert np.all(np.abs(y - x) <= per_elem / 2 * (1 + 1e-12))
    assert np.all(np.abs(O.unpack(codes, bits, len(scales) * block)) <= (1 << (bits - 1)) - 1)


@pytest.mark.parametrize("bits", [4, 8])
def test_pack_unpack_are_inverse(bits):
    q = (1 << (bits - 1)) - 1
    c = np.random.default_rng(bits).integers(-q, q + 1, size=4096)
    assert np.array_equal(O.unpack(O.pack(c, bits), bits, len(c)), c)
