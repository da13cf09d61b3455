"""Pin the CPU oracle (oracle/zpp_oracle.py) against the reference's golden
vectors and its own known-answer tests.  CPU only."""

import numpy as np
import pytest

import golden_util as gu
from oracle import zpp_oracle as O


def test_canonical_known_answer():
    # pkg/tests/test_quantizer.py:51-60
    codes, scales, _ = O.quantize([1.0, -1.0, 0.5, -0.5], 8, 8)
    assert scales.tolist() == [1.0 / 127.0]
    assert O.unpack(codes, 8, 4).tolist() == [127, -127, 64, -64]
    back = O.dequantize(codes, scales, 4, 8, 8)
    assert back[2] == np.float64(64) / np.float64(127)


def test_wire_size_formula():
    # pkg/tests/test_quantizer.py:122-129
    assert O.accounting(1021, 4, 512) == (511, 4, 1)


@pytest.mark.parametrize("case", range(len(gu.load("quant")[1])))
def test_quantize_matches_reference(case):
    z, meta = gu.load("quant")
    m = meta[case]
    vals = gu.as_f64(z[f"{case}_input"], m["dtype"])
    codes, scales, b = O.quantize(vals, m["bits"], m["block"], m["mode"])
    assert b == m["eff_block"]
    assert np.array_equal(codes, z[f"{case}_codes"])
    assert np.array_equal(scales, z[f"{case}_scales"])
    deq = O.dequantize(codes, scales, len(vals), m["bits"], b)
    assert np.array_equal(deq, z[f"{case}_deq"])
    assert O.accounting(len(vals), m["bits"], m["block"], m["mode"]) == (m["payload"], m["metadata"], m["padding"])


def test_fused_matches_reference():
    z, meta = gu.load("fused")
    for m in meta:
        i = m["idx"]
        ins = []
        for j in range(m["k"]):
            c, s, _ = O.quantize(z[f"{i}_in{j}_values"], m["in_bits"], m["in_block"])
            assert np.array_equal(c, z[f"{i}_in{j}_codes"])
            ins.append((c, s, m["n"], m["in_bits"], m["in_block"]))
        codes, scales, _ = O.fused_dequant_reduce_quant(ins, m["out_bits"], m["out_block"])
        assert np.array_equal(codes, z[f"{i}_codes"]), i
        assert np.array_equal(scales, z[f"{i}_scales"]), i


def test_reorder_and_partitions_match_reference():
    z, meta = gu.load("collectives")
    for x, y, s in meta["reorder"]:
        f, inv = O.reorder_mapping(x, y, s)
        assert np.array_equal(f, z[f"reorder_{x}_{y}_{s}_fwd"])
        assert np.array_equal(inv, z[f"reorder_{x}_{y}_{s}_inv"])
    for total, world, group in meta["partition"]:
        key = f"part_{total}_{world}_{group}"
        prim = [O.primary_range(total, world, r) for r in range(world)]
        sec = [O.secondary_range(total, group, r) for r in range(world)]
        assert np.array_equal(np.array(prim), z[key + "_primary"])
        assert np.array_equal(np.array(sec), z[key + "_secondary"])


def test_qwz_matches_reference():
    z, meta = gu.load("collectives")
    for m in meta["qwz"]:
        i, world = m["idx"], m["nodes"] * m["gpn"]
        shards = [gu.as_f64(z[f"qwz{i}_in{r}"], m["dtype"]) for r in range(world)]
        gathered, enc = O.all_gather_qwz(shards, m["bits"], m["block"])
        assert np.array_equal(gathered, z[f"qwz{i}_gathered"])
        for r, (c, s, _) in enumerate(enc):
            assert np.array_equal(c, z[f"qwz{i}_codes{r}"])
            assert np.array_equal(s, z[f"qwz{i}_scales{r}"])


def test_qgz_matches_reference():
    z, meta = gu.load("collectives")
    for m in meta["qgz"]:
        i, x, y, s = m["idx"], m["x"], m["y"], m["s"]
        world = x * y
        ins = [gu.as_f64(z[f"qgz{i}_in{r}"], m["dtype"]) for r in range(world)]
        outs = O.qgz_2hop(ins, x, y, s, m["bits"], m["block"], m["ibits"], m["iblock"], reorder=m["reorder"])
        for r in range(world):
            assert np.array_equal(outs[r], z[f"qgz{i}_out{r}"]), (i, r)


def test_ring_and_groups_match_reference():
    z, meta = gu.load("collectives")
    for m in meta["ring"]:
        i, world = m["idx"], m["nodes"] * m["gpn"]
        outs = O.reduce_scatter_ring([z[f"ring{i}_in{r}"] for r in range(world)], world)
        for r in range(world):
            assert np.array_equal(outs[r], z[f"ring{i}_out{r}"])
    for m in meta["groups"]:
        i, gpn, world = m["idx"], m["gpn"], m["nodes"] * m["gpn"]
        groups = [list(range(g * gpn, (g + 1) * gpn)) for g in range(m["nodes"])]
        outs = O.all_gather_groups([z[f"grp{i}_in{r}"] for r in range(world)], groups)
        for r in range(world):
            assert np.array_equal(outs[r], z[f"grp{i}_out{r}"])


def test_threaded_roundtrip_equals_serial():
    rng = np.random.default_rng(0)
    x = (rng.normal(size=3 * 2048 + 77) * 0.02).astype(np.float16)
    c, s, b = O.quantize(x, 8, 2048)
    serial = O.dequantize(c, s, x.size, 8, b).astype(np.float16)
    par = O.qwz_roundtrip_threaded(x, 8, 2048, threads=3)
    assert np.array_equal(serial, par)
