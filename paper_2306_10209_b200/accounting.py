"""Wire-byte accounting of the collectives, from sizes alone.

The reference's simulated fabric records every message it moves
(zs/simnet.py:37-88) and each collective adds one idealised volume row
(zs/collectives.py:180-195, :236-240, :269-275, :329-330, :548-563).  Here the
same books are filled analytically -- the GPU collectives (collectives.py)
and the comm-only ``step_volumes`` (zs/engine.py:455-506) both call these
functions, so the ledger a GPU run produces is the reference's ledger for the
same call.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .partitioner import build_partitions
from .quantizer import QuantConfig, effective_block
from .topology import INTER, INTRA, ClusterTopology, CollectiveTrace, TrafficLedger, account_phase, span_class

FP16_BYTES = 2
FWD_GATHER = "fwd_allgather"    # zs/engine.py:45-47
BWD_GATHER = "bwd_allgather"
GRAD_REDUCE = "reduce_scatter"


def encode_sizes(codec, k: int):
    """(payload, metadata, padding) bytes of one encode of k elements
    (zs/collectives.py:186-195)."""
    if codec.is_passthrough:
        return k * FP16_BYTES, 0, 0
    cfg = codec.cfg
    eff = effective_block(cfg, k)
    blocks = math.ceil(k / eff)
    payload = math.ceil(k * cfg.bit_width / 8)
    return payload, blocks * 2, blocks * eff * cfg.bit_width // 8 - payload


def volume_valid_adjust(ledger, label, cls, payload, metadata, padding, payload_valid):
    """zs/collectives.py:180-183: bytes beyond the valid payload count as padding."""
    extra = payload - min(payload, payload_valid)
    ledger.record_volume(label, cls, payload=payload - extra, metadata=metadata, padding=padding + extra)


def account_allgather(ledger: TrafficLedger, topo: ClusterTopology, label: str, shard_len: int, web: int,
                      groups=None, valid_elems=None) -> CollectiveTrace:
    """Full-precision (optionally grouped: hpZ) all-gather -- zs/collectives.py:202-241."""
    world = topo.world
    if groups is None:
        groups = [list(range(world))]
    group_of = {r: g for g, members in enumerate(groups) for r in members}
    trace = CollectiveTrace(label=label)
    account_phase(ledger, trace, topo, label, "allgather",
                  ((r, m, shard_len * web, 0, 0) for r in range(world) for m in groups[group_of[r]]))
    cls = INTER if any(span_class(m, topo) == INTER for m in groups) else INTRA
    gathered = shard_len * len(groups[0])
    valid = gathered if valid_elems is None else valid_elems
    volume_valid_adjust(ledger, label, cls, gathered * web, 0, 0, valid * web)
    return trace


def account_qwz(ledger: TrafficLedger, topo: ClusterTopology, label: str, codec, shard_len: int,
                valid_elems=None) -> CollectiveTrace:
    """Quantized all-gather -- zs/collectives.py:244-282."""
    world = topo.world
    pb, mb, padb = encode_sizes(codec, shard_len)
    trace = CollectiveTrace(label=label)
    account_phase(ledger, trace, topo, label, "allgather",
                  ((r, d, pb, mb, padb) for r in range(world) for d in range(world)))
    valid = shard_len * world if valid_elems is None else valid_elems
    volume_valid_adjust(ledger, label, span_class(range(world), topo), world * pb, world * mb, world * padb,
                        codec.payload_bytes_for(valid))
    return trace


def account_ring(ledger: TrafficLedger, topo: ClusterTopology, label: str, n: int, web: int,
                 valid_elems=None) -> CollectiveTrace:
    """Ring reduce-scatter -- zs/collectives.py:289-331."""
    world = topo.world
    chunk = n // world
    trace = CollectiveTrace(label=label)
    for step in range(world - 1):
        account_phase(ledger, trace, topo, label, f"ring{step}",
                      ((r, (r + 1) % world, chunk * web, 0, 0) for r in range(world)))
    valid = n if valid_elems is None else valid_elems
    volume_valid_adjust(ledger, label, span_class(range(world), topo), n * web, 0, 0, valid * web)
    return trace


def account_qgz(ledger: TrafficLedger, topo: ClusterTopology, label: str, codec, intra, n: int, stages: int,
                valid_elems=None) -> CollectiveTrace:
    """Two-hop reduce-scatter -- messages zs/collectives.py:509-534, volume rows :548-563."""
    x, y, s = topo.gpus_per_node, topo.nodes, stages
    world = x * y
    L = n // (s * world)
    trace = CollectiveTrace(label=label)
    m1 = encode_sizes(intra, y * L)
    m2 = encode_sizes(codec, L)
    for st in range(s):
        account_phase(ledger, trace, topo, label, f"s{st}.intra",
                      ((r, (r // x) * x + j, *m1) for r in range(world) for j in range(x)))
        account_phase(ledger, trace, topo, label, f"s{st}.inter",
                      ((r, c * x + (r % x), *m2) for r in range(world) for c in range(y)))
    valid = n if valid_elems is None else valid_elems
    pb1, mb1, padb1 = m1
    volume_valid_adjust(ledger, label + "/intra", INTRA, x * x * s * pb1, x * x * s * mb1, x * x * s * padb1,
                        x * intra.payload_bytes_for(valid))
    pb2, mb2, padb2 = m2
    volume_valid_adjust(ledger, label, INTER if y > 1 else INTRA, x * y * s * pb2, x * y * s * mb2,
                        x * y * s * padb2, codec.payload_bytes_for(valid))
    return trace


def account_qgz_1hop(ledger: TrafficLedger, topo: ClusterTopology, label: str, codec, n: int,
                     valid_elems=None) -> CollectiveTrace:
    """Single all-to-all quantized reduce-scatter -- zs/collectives.py:420-461."""
    world = topo.world
    chunk = n // world
    pb, mb, padb = encode_sizes(codec, chunk)
    trace = CollectiveTrace(label=label)
    account_phase(ledger, trace, topo, label, "alltoall", ((r, d, pb, mb, padb) for r in range(world)
                                                            for d in range(world)))
    x = topo.gpus_per_node
    valid = n if valid_elems is None else valid_elems
    volume_valid_adjust(ledger, label, span_class(range(world), topo), x * world * pb, x * world * mb,
                        x * world * padb, x * codec.payload_bytes_for(valid))
    return trace


def account_ring_naive_quant(ledger: TrafficLedger, topo: ClusterTopology, label: str, codec,
                             n: int) -> CollectiveTrace:
    """Re-quantizing ring -- zs/collectives.py:334-381 (every hop one encode of a chunk)."""
    world = topo.world
    chunk = n // world
    pb, mb, padb = encode_sizes(codec, chunk)
    trace = CollectiveTrace(label=label)
    for step in range(world - 1):
        account_phase(ledger, trace, topo, label, f"ring{step}",
                      ((r, (r + 1) % world, pb, mb, padb) for r in range(world)))
    ledger.record_volume(label, span_class(range(world), topo), payload=world * pb, metadata=world * mb,
                         padding=world * padb)
    return trace


# ---------------------------------------------------------------------------
# comm-only ZeRO(++) step


@dataclass(frozen=True)
class StepConfig:
    """The communication switches of the reference's ZeroConfig
    (zs/engine.py:80-115); any object with these attributes (including a
    zerosim ZeroConfig) is accepted by ``step_volumes``."""

    nodes: int = 2
    gpus_per_node: int = 2
    quantized_weight_gather: bool = False
    hierarchical_secondary_gather: bool = False
    quantized_grad_reduce: bool = False
    weight_quant: QuantConfig = field(default_factory=lambda: QuantConfig(bit_width=8, block_size=2048))
    grad_quant: QuantConfig = field(default_factory=lambda: QuantConfig(bit_width=4, block_size=512))
    grad_intra_quant: QuantConfig | None = None
    grad_stages: int = 1


def step_volumes(cfg, m_params: int):
    """Comm-only pass of one training step -- zs/engine.py:455-506.

    Returns (ledger, {label: normalized cross-node volume}, [(trace, stages)]).
    Padding and partitions follow the reference exactly (align = world *
    stages * max grad block)."""
    from .collectives import BlockCodec, PassthroughCodec  # noqa: F401  (codec accounting)
    from .topology import normalized_cross_node_volume

    topo = ClusterTopology(nodes=cfg.nodes, gpus_per_node=cfg.gpus_per_node)
    world = topo.world
    intra_q = cfg.grad_intra_quant or cfg.grad_quant
    align = world * cfg.grad_stages * max(cfg.grad_quant.block_size, intra_q.block_size)
    padded = math.ceil(m_params / align) * align
    spec = build_partitions(padded, topo)
    shard = padded // world
    ledger = TrafficLedger()
    traces = []
    if cfg.quantized_weight_gather:
        tr = account_qwz(ledger, topo, FWD_GATHER, BlockCodec(cfg.weight_quant), shard, valid_elems=m_params)
    else:
        tr = account_allgather(ledger, topo, FWD_GATHER, shard, FP16_BYTES, valid_elems=m_params)
    traces.append((tr, 1))
    if cfg.hierarchical_secondary_gather:
        lo, hi = spec.secondary_range(0)
        tr = account_allgather(ledger, topo, BWD_GATHER, hi - lo, FP16_BYTES, groups=spec.groups(),
                               valid_elems=m_params)
    elif cfg.quantized_weight_gather:
        tr = account_qwz(ledger, topo, BWD_GATHER, BlockCodec(cfg.weight_quant), shard, valid_elems=m_params)
    else:
        tr = account_allgather(ledger, topo, BWD_GATHER, shard, FP16_BYTES, valid_elems=m_params)
    traces.append((tr, 1))
    if cfg.quantized_grad_reduce:
        intra = BlockCodec(intra_q)
        tr = account_qgz(ledger, topo, GRAD_REDUCE, BlockCodec(cfg.grad_quant), intra, padded, cfg.grad_stages,
                         valid_elems=m_params)
        traces.append((tr, cfg.grad_stages))
    else:
        tr = account_ring(ledger, topo, GRAD_REDUCE, padded, FP16_BYTES, valid_elems=m_params)
        traces.append((tr, 1))
    vols = {label: normalized_cross_node_volume(ledger, m_params, label=label)
            for label in (FWD_GATHER, BWD_GATHER, GRAD_REDUCE)}
    return ledger, vols, traces
