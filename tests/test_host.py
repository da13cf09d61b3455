"""CPU tests of the host side: the C ABI loads and exports every symbol
include/zpp.h declares (no compute calls), configs/partitions/reorder maps
against the reference goldens, and the analytic ledger rows."""

import ctypes
import os
import re

import numpy as np
import pytest

import golden_util as gu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "zpp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zpp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2306_10209_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.zpp_version() >= 10000


def test_status_codes_map_to_reference_exceptions():
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200 import _lib

    assert issubclass(zpp.ValidationError, zpp.SimError)
    for rc, exc in ((_lib.ERR_CONFIG, zpp.ConfigError), (_lib.ERR_VALIDATION, zpp.ValidationError),
                    (_lib.ERR_INTEGRITY, zpp.IntegrityError), (_lib.ERR_CUDA, zpp.DeviceError)):
        with pytest.raises(exc):
            _lib.check(rc, "x")
    with pytest.raises(zpp.ValidationError):
        _lib.raise_for_flags(_lib.FLAG_NONFINITE)
    with pytest.raises(zpp.IntegrityError):
        _lib.raise_for_flags(_lib.FLAG_BADCODE)
    _lib.raise_for_flags(0)


def test_c_abi_rejects_bad_configs_without_launching():
    from paper_2306_10209_b200 import _lib

    lib = _lib.load()
    assert lib.zpp_quantize(None, 0, 16, 16, 8, None, None, None, None) == _lib.ERR_CONFIG
    assert lib.zpp_quantize(None, 0, 16, 8, 12, None, None, None, None) == _lib.ERR_CONFIG
    assert lib.zpp_quantize(None, 9, 16, 8, 8, None, None, None, None) == _lib.ERR_VALIDATION
    assert lib.zpp_quantize(None, 0, 16, 8, 8, None, None, None, None) == _lib.ERR_VALIDATION  # null pointers
    assert lib.zpp_quantize(None, 0, 0, 8, 8, None, None, None, None) == _lib.OK  # empty is a no-op
    assert lib.zpp_swizzle_quantize(None, 0, 20, 2, 2, 1, 0, 1, 8, 8, None, None, None, None) == _lib.ERR_VALIDATION
    assert lib.zpp_swizzle_quantize(None, 0, 16, 2, 2, 1, 0, 1, 8, 8, None, None, None, None) == _lib.ERR_VALIDATION
    assert "block" in _lib.last_error() or "slice" in _lib.last_error()
    assert lib.zpp_drq_workspace_bytes(1000, 512) == 1024 * 8


def test_quant_config_validation_matches_reference():
    import paper_2306_10209_b200 as zpp

    for kwargs in ({"bit_width": 16}, {"bit_width": 8, "block_size": 0}, {"bit_width": 8, "block_size": 12},
                   {"bit_width": 8, "mode": "rowwise"}, {"bit_width": 8, "rounding": "away-from-zero"}):
        with pytest.raises(zpp.ConfigError):
            zpp.QuantConfig(**kwargs)
    assert zpp.QuantConfig(bit_width=4).qmax == 7 and zpp.QuantConfig(bit_width=8).qmax == 127
    with pytest.raises(zpp.ValidationError):
        zpp.FlatTensor(np.array([1.0, np.nan]))
    with pytest.raises(zpp.ValidationError):
        zpp.FlatTensor(np.zeros((2, 2)))


def test_partitions_and_reorder_match_reference_goldens():
    import paper_2306_10209_b200 as zpp

    z, meta = gu.load("collectives")
    for total, world, group in meta["partition"]:
        spec = zpp.PartitionSpec(total_elems=total, world=world, group_size=group)
        key = f"part_{total}_{world}_{group}"
        assert np.array_equal(np.array([spec.primary_range(r) for r in range(world)]), z[key + "_primary"])
        assert np.array_equal(np.array([spec.secondary_range(r) for r in range(world)]), z[key + "_secondary"])
        assert np.array_equal(np.array(spec.groups()), z[key + "_groups"])
    for x, y, s in meta["reorder"]:
        p = zpp.reorder_mapping(x, y, s)
        assert np.array_equal(p.forward, z[f"reorder_{x}_{y}_{s}_fwd"])
        assert np.array_equal(p.inverse, z[f"reorder_{x}_{y}_{s}_inv"])
    with pytest.raises(zpp.ValidationError):
        zpp.PartitionSpec(total_elems=10, world=4, group_size=3)
    with pytest.raises(zpp.ValidationError):
        zpp.reorder_mapping(0, 2, 1)


def test_wire_accounting_matches_reference():
    from paper_2306_10209_b200.collectives import BlockCodec, _encode_sizes
    import paper_2306_10209_b200 as zpp

    _, meta = gu.load("quant")
    for m in meta:
        cfg = zpp.QuantConfig(bit_width=m["bits"], block_size=m["block"], mode=m["mode"])
        assert _encode_sizes(BlockCodec(cfg), m["n"]) == (m["payload"], m["metadata"], m["padding"])


def test_topology_and_ledger_basics():
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200.topology import account_phase

    topo = zpp.ClusterTopology(nodes=2, gpus_per_node=4)
    assert topo.world == 8 and topo.node_of(5) == 1
    led = zpp.TrafficLedger()
    tr = zpp.CollectiveTrace(label="x")
    account_phase(led, tr, topo, "x", "p", [(0, 0, 10, 1, 0), (0, 1, 10, 1, 0), (0, 4, 10, 1, 0)])
    assert led.physical_bytes(cls=zpp.INTRA) == 10 and led.physical_bytes(cls=zpp.INTER) == 10
    assert tr.totals()[:4] == (1, 11, 1, 11)
    led.record_volume("x", zpp.INTER, payload=2 << 20)
    assert zpp.normalized_cross_node_volume(led, 1 << 20, label="x") == 1.0
    assert led.conservation_holds()


def test_step_volumes_match_reference_ledger():
    """Comm-only ZeRO/ZeRO++ step (zs/engine.py:455-506): the ledger CSV and the
    normalised cross-node volumes equal the reference's for 15 switch settings."""
    import paper_2306_10209_b200 as zpp

    for row in gu.volumes():
        cfg = zpp.StepConfig(nodes=row["nodes"], gpus_per_node=row["gpn"], quantized_weight_gather=row["qw"],
                             hierarchical_secondary_gather=row["hp"], quantized_grad_reduce=row["qg"])
        ledger, vols, traces = zpp.step_volumes(cfg, row["m"])
        assert ledger.to_csv(row["m"]) == row["csv"], row
        assert vols == row["vols"], row
        assert ledger.conservation_holds()


def test_step_volume_table_headline():
    """Acceptance c01 (pkg/tests/test_acceptance.py:67-93): 8 nodes x 4 GPUs, 2^20
    params: ZeRO-3 moves (1, 1, 1) fp16 model copies across nodes, ZeRO++ (0.5, 0,
    0.25); scale metadata stays under 2% of payload."""
    import paper_2306_10209_b200 as zpp

    m = 1 << 20
    _, base, _ = zpp.step_volumes(zpp.StepConfig(nodes=8, gpus_per_node=4), m)
    led, comp, _ = zpp.step_volumes(zpp.StepConfig(nodes=8, gpus_per_node=4, quantized_weight_gather=True,
                                                   hierarchical_secondary_gather=True,
                                                   quantized_grad_reduce=True), m)
    assert base == {zpp.FWD_GATHER: 1.0, zpp.BWD_GATHER: 1.0, zpp.GRAD_REDUCE: 1.0}
    assert comp == {zpp.FWD_GATHER: 0.5, zpp.BWD_GATHER: 0.0, zpp.GRAD_REDUCE: 0.25}
    assert max(b.metadata / b.payload for b in led.volume.values() if b.payload) < 0.02


def test_secondary_gather_stays_on_node():
    """Acceptance c07: hpZ's backward gather moves zero cross-node bytes."""
    import paper_2306_10209_b200 as zpp

    for nodes, gpus in ((2, 2), (2, 4), (3, 2), (4, 4)):
        led, _, _ = zpp.step_volumes(zpp.StepConfig(nodes=nodes, gpus_per_node=gpus,
                                                    hierarchical_secondary_gather=True), 1 << 16)
        assert led.physical_bytes(label=zpp.BWD_GATHER, cls=zpp.INTER) == 0
    off, _, _ = zpp.step_volumes(zpp.StepConfig(nodes=2, gpus_per_node=2), 1 << 16)
    assert off.physical_bytes(label=zpp.BWD_GATHER, cls=zpp.INTER) > 0


def test_engine_mlp_gradient_matches_central_differences():
    """The toy engine's analytic MLP gradient (zs/engine.py:196-220, checked
    there by gradient_check :223-243) against central differences."""
    import engine_harness as E

    rng = np.random.default_rng(0)
    dims = [4, 5, 3]
    p = E.init_params(dims, rng)
    x, y = rng.normal(size=(2, 4)), rng.normal(size=(2, 3))
    _, g = E.mlp_loss_and_grad(p, x, y, dims)
    num = np.zeros_like(g)
    for i in range(len(p)):
        d = np.zeros_like(p)
        d[i] = 1e-6
        num[i] = (E.mlp_loss_and_grad(p + d, x, y, dims)[0] - E.mlp_loss_and_grad(p - d, x, y, dims)[0]) / 2e-6
    assert np.max(np.abs(g - num) / np.maximum(np.abs(num), 1e-8)) < 1e-4
    assert E.param_count(E.ToyTaskConfig().layer_dims()) == 9928  # padded to 10240 over 4 ranks


def test_engine_config_validation():
    import engine_harness as E
    import paper_2306_10209_b200 as zpp

    for kw in (dict(nodes=0), dict(steps=0), dict(lr=0.0), dict(grad_quant_fraction=1.5), dict(grad_stages=0)):
        with pytest.raises(zpp.ValidationError):
            E.ZeroConfig(**kw)


def test_c10_latency_pipeline_model():
    """Acceptance c10 (pkg/tests/test_acceptance.py:344-380): one stage is the
    plain two-phase sum, equal phases with free messages make two stages cost
    75%, and optimal_stages matches a brute-force sweep with an interior optimum."""
    import paper_2306_10209_b200 as zpp

    trace = zpp.CollectiveTrace(label="step", phases=[zpp.PhaseStats(
        "p", intra_messages=8, intra_bytes=300 * 10**9, inter_messages=8, inter_bytes=25 * 10**9)])
    free = zpp.LinkParams(intra_alpha=0.0, intra_beta=300e9, inter_alpha=0.0, inter_beta=25e9)
    t1 = zpp.estimate_latency(trace, free, stages=1).total_seconds
    assert t1 == 2.0 and zpp.estimate_latency(trace, free, stages=2).total_seconds == 0.75 * t1
    links = zpp.LinkParams(intra_alpha=1e-6, intra_beta=300e9, inter_alpha=1.25e-2, inter_beta=25e9)
    im, ib, em, eb, _ = trace.totals()

    def by_hand(s):
        ti = links.intra_alpha * im * s + ib / links.intra_beta
        te = links.inter_alpha * em * s + eb / links.inter_beta
        return (ti + te) / s + (s - 1) * max(ti, te) / s

    sweep = [by_hand(s) for s in range(1, 9)]
    s_best, t_best = zpp.optimal_stages(trace, links, max_stages=8)
    assert s_best == sweep.index(min(sweep)) + 1 and t_best == min(sweep) and 1 < s_best < 8
    assert all(zpp.pipelined_seconds(trace, links, s) == sweep[s - 1] for s in range(1, 9))
    with pytest.raises(zpp.ValidationError):
        zpp.LinkParams(intra_beta=0.0)


def test_engine_parts_on_the_host():
    """Engine pieces that need no GPU: layer views share the flat vector,
    forward shapes and tanh range, per-rank gradient shards sum to the full
    batch, the input-scale ramp, and the up-front codec check
    (pkg/tests/test_engine.py restated)."""
    import paper_2306_10209_b200 as zpp
    import engine_harness as E

    flat = np.zeros(E.param_count([3, 4, 2]))
    (w0, _), (_, b1) = E._layers(flat, [3, 4, 2])
    w0[1, 2], b1[0] = 7.0, -1.0
    assert flat[6] == 7.0 and flat[3 * 4 + 4 + 4 * 2] == -1.0
    rng = np.random.default_rng(0)
    p = E.init_params([5, 8, 2], rng)
    out, acts = E.mlp_forward(p, rng.normal(size=(7, 5)), [5, 8, 2])
    assert out.shape == (7, 2) and len(acts) == 3 and np.all(np.abs(acts[1]) <= 1.0)
    p = E.init_params([4, 6, 3], rng)
    x, y = rng.normal(size=(8, 4)), rng.normal(size=(8, 3))
    full = E.mlp_loss_and_grad(p, x, y, [4, 6, 3])[1]
    parts = sum(E.mlp_loss_and_grad(p, x[i:i + 2], y[i:i + 2], [4, 6, 3], denom=8)[1] for i in range(0, 8, 2))
    assert np.allclose(parts, full, rtol=0, atol=1e-12)
    task = E.ToyTaskConfig(in_dim=8, hidden=(8,), out_dim=2, input_scale_range=16.0, eval_samples=16)
    s = E.TrainingEngine(task, E.ZeroConfig(steps=1)).input_scales
    assert s[-1] / s[0] == pytest.approx(16.0) and np.sum(s * s) == pytest.approx(8)
    with pytest.raises(zpp.ValidationError):
        E.TrainingEngine(E.ToyTaskConfig(input_scale_range=0.5), E.ZeroConfig(steps=1))
    whole = zpp.QuantConfig(bit_width=4, mode="full_tensor")
    with pytest.raises(zpp.ConfigError):
        E.TrainingEngine(task, E.ZeroConfig(quantized_grad_reduce=True, grad_quant=whole))
    E.TrainingEngine(task, E.ZeroConfig(grad_quant=whole))
    eng = E.TrainingEngine(E.ToyTaskConfig(), E.ZeroConfig(steps=1))
    assert (eng.m_params, eng.padded) == (9928, 10240)
