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
