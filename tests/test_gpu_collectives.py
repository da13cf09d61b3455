"""GPU parity of the single-process collectives (all ranks of a virtual
cluster on one GPU) against the reference's golden vectors, plus the
reference's own collective tests (pkg/tests/test_collectives.py) restated on
the GPU codec."""

import itertools

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle import zpp_oracle as O

pytestmark = pytest.mark.gpu

Z, MC = gu.load("collectives")


def _zpp():
    import paper_2306_10209_b200 as zpp
    return zpp


def _vol(ledger):
    return {f"{lb}|{cls}": [b.payload, b.metadata, b.padding] for (lb, cls), b in ledger.volume.items()}


def random_tensors(world, n, seed, scale=1.0, integers=False):
    rng = np.random.default_rng(seed)
    if integers:
        return [torch.from_numpy(rng.integers(-40, 41, size=n).astype(np.float64)).cuda() for _ in range(world)]
    return [torch.from_numpy(rng.normal(size=n) * scale).cuda() for _ in range(world)]


@pytest.mark.parametrize("case", range(len(MC["qwz"])))
def test_qwz_golden(case):
    zpp = _zpp()
    m = MC["qwz"][case]
    world = m["nodes"] * m["gpn"]
    shards = [gu.to_torch(Z[f"qwz{case}_in{r}"], m["dtype"]) for r in range(world)]
    topo = zpp.ClusterTopology(nodes=m["nodes"], gpus_per_node=m["gpn"])
    ledger = zpp.TrafficLedger()
    res = zpp.all_gather_qwz(shards, zpp.QuantConfig(bit_width=m["bits"], block_size=m["block"]), topo, ledger)
    assert res.codec_depth == m["depth"]
    for r in range(world):
        assert np.array_equal(res.quantized[r].codes.cpu().numpy(), Z[f"qwz{case}_codes{r}"])
        assert np.array_equal(res.quantized[r].scales.cpu().numpy(), Z[f"qwz{case}_scales{r}"])
        assert np.array_equal(res.gathered[r].values.cpu().numpy(), Z[f"qwz{case}_gathered"])
    assert _vol(ledger) == m["volume"]
    assert ledger.conservation_holds()
    # the fp16 output the engine consumes (zs/engine.py:353 half_round)
    res16 = zpp.all_gather_qwz(shards, zpp.BlockCodec(zpp.QuantConfig(bit_width=m["bits"], block_size=m["block"]),
                                                       out_dtype=torch.float16), topo, zpp.TrafficLedger())
    assert np.array_equal(res16.gathered[0].values.double().cpu().numpy(),
                          gu.round_to(Z[f"qwz{case}_gathered"], "fp16"))


@pytest.mark.parametrize("case", range(len(MC["groups"])))
def test_hpz_groups_golden(case):
    zpp = _zpp()
    m = MC["groups"][case]
    world = m["nodes"] * m["gpn"]
    shards = [gu.to_torch(Z[f"grp{case}_in{r}"], "fp16") for r in range(world)]
    topo = zpp.ClusterTopology(nodes=m["nodes"], gpus_per_node=m["gpn"])
    spec = zpp.build_partitions(m["shard_len"] * m["gpn"], topo)
    ledger = zpp.TrafficLedger()
    res = zpp.all_gather_baseline(shards, topo, ledger, groups=spec.groups())
    for r in range(world):
        assert np.array_equal(res.gathered[r].values.double().cpu().numpy(), Z[f"grp{case}_out{r}"])
    assert _vol(ledger) == m["volume"]
    phys = {f"{lb}|{cls}": [b.payload, b.messages] for (lb, cls), b in ledger.physical.items()}
    assert phys == m["physical"]
    assert ledger.physical_bytes(cls=zpp.INTER) == 0


@pytest.mark.parametrize("case", range(len(MC["qgz"])))
def test_qgz_golden(case):
    zpp = _zpp()
    m = MC["qgz"][case]
    x, y, s = m["x"], m["y"], m["s"]
    world = x * y
    topo = zpp.ClusterTopology(nodes=y, gpus_per_node=x)
    ins = [gu.to_torch(Z[f"qgz{case}_in{r}"], m["dtype"]) for r in range(world)]
    cfg = zpp.QuantConfig(bit_width=m["bits"], block_size=m["block"])
    icfg = zpp.QuantConfig(bit_width=m["ibits"], block_size=m["iblock"]) if m["ibits"] else None
    ledger = zpp.TrafficLedger()
    res = zpp.qgz_2hop(ins, cfg, topo, ledger, stages=s, intra_codec=icfg, reorder=m["reorder"])
    assert res.codec_depth == m["depth"]
    for r in range(world):
        assert np.array_equal(res.shards[r].values.cpu().numpy(), Z[f"qgz{case}_out{r}"]), (case, r)
    assert _vol(ledger) == m["volume"]
    phys = {f"{lb}|{cls}": [b.payload, b.messages] for (lb, cls), b in ledger.physical.items()}
    assert phys == m["physical"]
    # fp32 output (the B200 default) = the reference's f64 rounded once
    res32 = zpp.qgz_2hop(ins, zpp.BlockCodec(cfg, out_dtype=torch.float32), topo, zpp.TrafficLedger(), stages=s,
                         intra_codec=icfg, reorder=m["reorder"])
    for r in range(world):
        assert np.array_equal(res32.shards[r].values.double().cpu().numpy(),
                              gu.round_to(Z[f"qgz{case}_out{r}"], "fp32"))
    # passthrough routing = ring fold
    ints = [torch.from_numpy(Z[f"qgz{case}_int_in{r}"]).cuda() for r in range(world)]
    pt = zpp.qgz_2hop(ints, zpp.PassthroughCodec(), topo, zpp.TrafficLedger(), stages=s, reorder=m["reorder"])
    for r in range(world):
        assert np.array_equal(pt.shards[r].values.cpu().numpy(), Z[f"qgz{case}_int_out{r}"])


def test_ring_golden():
    zpp = _zpp()
    for m in MC["ring"]:
        i, world = m["idx"], m["nodes"] * m["gpn"]
        topo = zpp.ClusterTopology(nodes=m["nodes"], gpus_per_node=m["gpn"])
        res = zpp.reduce_scatter_ring([torch.from_numpy(Z[f"ring{i}_in{r}"]).cuda() for r in range(world)], topo,
                                      zpp.TrafficLedger())
        for r in range(world):
            assert np.array_equal(res.shards[r].values.cpu().numpy(), Z[f"ring{i}_out{r}"])


# --- restated from pkg/tests/test_collectives.py ---------------------------


def test_qgz_placement_grid_matches_ring():
    zpp = _zpp()
    for x, y, s in itertools.product((2, 4), (2, 3), (1, 2, 4)):
        topo = zpp.ClusterTopology(nodes=y, gpus_per_node=x)
        world = x * y
        n = s * world * 8
        ins = random_tensors(world, n, seed=100 + x + 10 * y + 100 * s, integers=True)
        ring = zpp.reduce_scatter_ring(ins, topo, zpp.TrafficLedger())
        hier = zpp.qgz_2hop(ins, zpp.PassthroughCodec(), topo, zpp.TrafficLedger(), stages=s)
        for got, want in zip(hier.shards, ring.shards):
            assert torch.equal(got.values, want.values), (x, y, s)


def test_qgz_skipping_reorder_misplaces_partitions():
    zpp = _zpp()
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    ins = random_tensors(4, 16, seed=13, integers=True)
    oracle = O.reduce_scatter_ring([t.cpu().numpy() for t in ins], 4)
    res = zpp.qgz_2hop(ins, zpp.PassthroughCodec(), topo, zpp.TrafficLedger(), reorder=False)
    got = [s.values.cpu().numpy() for s in res.shards]
    assert np.array_equal(got[0], oracle[0]) and np.array_equal(got[3], oracle[3])
    assert np.array_equal(got[1], oracle[2]) and np.array_equal(got[2], oracle[1])


def test_qgz_codec_depth_is_two_everywhere():
    zpp = _zpp()
    cfg = zpp.QuantConfig(bit_width=4, block_size=8)
    for x, y in ((1, 1), (2, 2), (4, 3)):
        topo = zpp.ClusterTopology(nodes=y, gpus_per_node=x)
        world = x * y
        res = zpp.qgz_2hop(random_tensors(world, world * 8, seed=14, scale=2.0), cfg, topo, zpp.TrafficLedger())
        assert res.codec_depth == 2


def test_qgz_error_bounds_hold():
    zpp = _zpp()
    cfg = zpp.QuantConfig(bit_width=8, block_size=8)
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    ins = random_tensors(4, 64, seed=16, scale=5.0)
    oracle = O.reduce_scatter_ring([t.cpu().numpy() for t in ins], 4)
    res = zpp.qgz_2hop(ins, cfg, topo, zpp.TrafficLedger(), collect_bounds=True)
    for got, want, bound in zip(res.shards, oracle, res.error_bounds):
        b = bound.cpu().numpy()
        assert np.all(np.isfinite(b))
        assert np.all(np.abs(got.values.cpu().numpy() - want) <= b + 1e-12)
    with pytest.raises(zpp.ValidationError):
        zpp.qgz_2hop(ins, zpp.PassthroughCodec(), topo, zpp.TrafficLedger(), collect_bounds=True)


def test_qgz_traffic_split():
    zpp = _zpp()
    cfg = zpp.QuantConfig(bit_width=4, block_size=8)
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    ledger = zpp.TrafficLedger()
    n = 64
    res = zpp.qgz_2hop(random_tensors(4, n, seed=17), cfg, topo, ledger)
    x, y, sl = 2, 2, n // 4
    assert ledger.physical[("reduce_scatter", zpp.INTRA)].messages == 4 * (x - 1)
    assert ledger.physical[("reduce_scatter", zpp.INTER)].messages == 4 * (y - 1)
    assert ledger.physical_bytes(cls=zpp.INTER) == 4 * (y - 1) * (sl // 2)
    assert ledger.volume_bytes(zpp.INTRA, label="reduce_scatter/intra") == x * (n // 2)
    assert ledger.volume_bytes(zpp.INTER, label="reduce_scatter") == n // 2
    assert ledger.volume_bytes(zpp.INTER, label="reduce_scatter", kind="metadata") == (n // 8) * 2
    im, ib, em, eb, _ = res.trace.totals()
    assert (im, em) == (4 * (x - 1), 4 * (y - 1))
    assert ledger.conservation_holds()


def test_qgz_single_node_has_no_cross_traffic():
    zpp = _zpp()
    topo = zpp.ClusterTopology(nodes=1, gpus_per_node=4)
    ledger = zpp.TrafficLedger()
    zpp.qgz_2hop(random_tensors(4, 64, seed=18), zpp.QuantConfig(bit_width=8, block_size=8), topo, ledger)
    assert ledger.physical_bytes(cls=zpp.INTER) == 0 and ledger.volume_bytes(zpp.INTER) == 0


def test_qgz_validation():
    zpp = _zpp()
    cfg = zpp.QuantConfig(bit_width=8, block_size=8)
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    with pytest.raises(zpp.ValidationError):
        zpp.qgz_2hop(random_tensors(4, 20, seed=19), cfg, topo, zpp.TrafficLedger())
    with pytest.raises(zpp.ValidationError):
        zpp.qgz_2hop(random_tensors(4, 16, seed=20), cfg, topo, zpp.TrafficLedger())
    with pytest.raises(zpp.ValidationError):
        zpp.qgz_2hop(random_tensors(4, 32, seed=21), cfg, topo, zpp.TrafficLedger(), stages=0)
    with pytest.raises(zpp.ValidationError):
        zpp.qgz_2hop(random_tensors(4, 32, seed=22), cfg, topo, zpp.TrafficLedger(),
                     intra_codec=zpp.PassthroughCodec())


def test_qwz_passthrough_equals_baseline():
    zpp = _zpp()
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    shards = random_tensors(4, 16, seed=5)
    base = zpp.all_gather_baseline(shards, topo, zpp.TrafficLedger())
    quant = zpp.all_gather_qwz(shards, zpp.PassthroughCodec(), topo, zpp.TrafficLedger())
    for a, b in zip(base.gathered, quant.gathered):
        assert torch.equal(a.values, b.values)
    assert quant.codec_depth == 0


def test_qgz_large_bucket_vs_oracle():
    """A 2x4 cluster, INT4/512, bf16 grads, 2 stages: bit-exact vs the oracle."""
    zpp = _zpp()
    x, y, s = 4, 2, 2
    world = x * y
    n = s * world * 512 * 16
    rng = np.random.default_rng(2024)
    raw = [(rng.normal(size=n) * np.exp(rng.normal(size=n)) * 1e-3).astype(np.float32) for _ in range(world)]
    bf = [(a.view(np.uint32) >> 16).astype(np.uint16) for a in raw]
    ins = [gu.to_torch(b, "bf16") for b in bf]
    cfg = zpp.QuantConfig(bit_width=4, block_size=512)
    res = zpp.qgz_2hop(ins, cfg, zpp.ClusterTopology(nodes=y, gpus_per_node=x), zpp.TrafficLedger(), stages=s)
    want = O.qgz_2hop([gu.as_f64(b, "bf16") for b in bf], x, y, s, 4, 512)
    for r in range(world):
        assert np.array_equal(res.shards[r].values.cpu().numpy(), want[r])


# --- comparators (pkg/tests/test_collectives.py:164-187, :230-249, :291-302) ---


def test_naive_quant_ring_depth_and_volume():
    zpp = _zpp()
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    ledger = zpp.TrafficLedger()
    cfg = zpp.QuantConfig(bit_width=8, block_size=8)
    ins = random_tensors(4, 32, seed=9, scale=2.0)
    res = zpp.reduce_scatter_ring_naive_quant(ins, cfg, topo, ledger)
    assert res.codec_depth == 3
    oracle = O.reduce_scatter_ring([t.cpu().numpy() for t in ins], 4)
    for got, want in zip(res.shards, oracle):
        assert np.max(np.abs(got.values.cpu().numpy() - want)) < 1.0
    assert ledger.volume_bytes(zpp.INTER, label="reduce_scatter") == 4 * 8
    assert ledger.volume_bytes(zpp.INTER, label="reduce_scatter", kind="metadata") == 4 * 2
    pt = zpp.reduce_scatter_ring_naive_quant(random_tensors(4, 16, seed=10, integers=True), zpp.PassthroughCodec(),
                                             topo, zpp.TrafficLedger())
    assert pt.codec_depth == 0


def test_qgz_1hop_passthrough_and_volume():
    zpp = _zpp()
    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=2)
    ins = random_tensors(4, 16, seed=11, integers=True)
    res = zpp.qgz_1hop(ins, zpp.PassthroughCodec(), topo, zpp.TrafficLedger())
    oracle = O.reduce_scatter_ring([t.cpu().numpy() for t in ins], 4)
    for got, want in zip(res.shards, oracle):
        assert np.array_equal(got.values.cpu().numpy(), want)
    ledger = zpp.TrafficLedger()
    res = zpp.qgz_1hop(random_tensors(4, 32, seed=12), zpp.QuantConfig(bit_width=8, block_size=8), topo, ledger)
    assert res.codec_depth == 1
    assert ledger.volume_bytes(zpp.INTER, label="reduce_scatter") == 2 * 32
    assert ledger.volume_bytes(zpp.INTER, label="reduce_scatter", kind="metadata") == 2 * 8


def test_two_hop_beats_naive_ring_and_depth_is_two():
    """Acceptance c05 (pkg/tests/test_acceptance.py:190-224)."""
    zpp = _zpp()
    cfg = zpp.QuantConfig(bit_width=4, block_size=8)
    depths = {}
    for nodes, gpus in ((2, 2), (4, 2), (4, 4)):
        topo = zpp.ClusterTopology(nodes=nodes, gpus_per_node=gpus)
        world = nodes * gpus
        ins = random_tensors(world, world * 64, seed=50 + world, scale=2.0)
        hier = zpp.qgz_2hop(ins, cfg, topo, zpp.TrafficLedger())
        naive = zpp.reduce_scatter_ring_naive_quant(ins, cfg, topo, zpp.TrafficLedger())
        assert hier.codec_depth == 2
        depths[world] = naive.codec_depth
        if world == 16:
            oracle = O.reduce_scatter_ring([t.cpu().numpy() for t in ins], world)
            rh = np.sqrt(np.mean([(g.values.cpu().numpy() - w) ** 2 for g, w in zip(hier.shards, oracle)]))
            rn = np.sqrt(np.mean([(g.values.cpu().numpy() - w) ** 2 for g, w in zip(naive.shards, oracle)]))
            assert rh < rn
    assert depths == {4: 3, 8: 7, 16: 15}
