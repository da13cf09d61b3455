"""ZeRO++ collectives on B200 -- drop-in for zs/collectives.py.

Single-process form: like the reference, every function takes the per-rank
inputs of a whole (virtual) cluster and returns every rank's output, so the
reference's tests and callers run unchanged; all ranks' data sit on the
current GPU and each rank's exchange is a pointer hand-off to the next kernel
instead of a simulated message.  The multi-GPU form (one process per GPU,
NVLink P2P) of the same three collectives is ``paper_2306_10209_b200.dist``.

Hot kernels per collective (csrc/zpp_kernels.cuh):

* ``all_gather_qwz``  K0 per rank, then ONE K4 launch decoding all W payloads
  (zs/collectives.py:244-282);
* ``all_gather_baseline(groups=...)`` hpZ routing, bit-identical copies
  (zs/collectives.py:202-241);
* ``qgz_2hop`` K1 (slice reorder fused into quantize) -> K2 (dequant -> f64
  fold -> requant) -> K3 (dequant -> f64 fold) per stage and rank
  (zs/collectives.py:464-569).

Reduction order is pinned exactly as in the reference: every f64 fold runs
from +0.0 over ascending source rank.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ValidationError
from .quantizer import (
    FlatTensor,
    QuantConfig,
    QuantizedTensor,
    alloc_quantized,
    as_flat,
    check_flag,
    dequant_reduce,
    dequantize,
    device,
    dtype_code,
    effective_block,
    fused_dequant_reduce_quant,
    new_flag,
    quantize,
    stream_ptr,
)
from .accounting import (
    account_allgather,
    account_qgz,
    account_qgz_1hop,
    account_qwz,
    account_ring,
    account_ring_naive_quant,
)
from .accounting import encode_sizes as _encode_sizes  # noqa: F401  (re-exported for callers/tests)
from .accounting import volume_valid_adjust as _volume_valid_adjust  # noqa: F401
from .topology import ClusterTopology, CollectiveTrace, TrafficLedger

FP16_BYTES = 2


# ---------------------------------------------------------------------------
# codecs (zs/collectives.py:42-148)


@dataclass
class WirePayload:
    """Encoded data plus the number of sequential quantize passes behind it."""

    data: object
    n: int
    depth: int = 0


def _flat_values(values) -> torch.Tensor:
    if isinstance(values, FlatTensor):
        return values.cuda_values()
    if isinstance(values, torch.Tensor):
        return values if values.is_cuda else values.to(device())
    return as_flat(values).cuda_values()


class BlockCodec:
    """Quantizing codec backed by the sm_100a kernels (zs/collectives.py:51-91).

    ``out_dtype`` is the dtype ``decode``/``reduce_final`` produce; the default
    float64 is the reference's, each element correctly rounded either way.
    """

    is_passthrough = False

    def __init__(self, cfg: QuantConfig, out_dtype: torch.dtype = torch.float64):
        self.cfg = cfg
        self.out_dtype = out_dtype

    def encode(self, values, prior_depth: int = 0) -> WirePayload:
        q = quantize(FlatTensor(_flat_values(values)), self.cfg)
        return WirePayload(data=q, n=q.original_len, depth=prior_depth + 1)

    def decode(self, wp: WirePayload) -> torch.Tensor:
        return dequantize(wp.data, self.out_dtype).values

    def fuse(self, wps) -> WirePayload:
        wps = list(wps)
        fused = fused_dequant_reduce_quant([wp.data for wp in wps], self.cfg)
        return WirePayload(data=fused, n=wps[0].n, depth=max(wp.depth for wp in wps) + 1)

    def reduce_final(self, wps) -> torch.Tensor:
        return dequant_reduce([wp.data for wp in wps], self.out_dtype)

    def slice(self, wp: WirePayload, start: int, length: int) -> WirePayload:
        return WirePayload(data=wp.data.slice_blocks(start, length), n=length, depth=wp.depth)

    def accounting(self, wp: WirePayload):
        q = wp.data
        return q.payload_bytes, q.metadata_bytes, q.padding_bytes

    def payload_bytes_for(self, n_elems: int) -> int:
        return math.ceil(n_elems * self.cfg.bit_width / 8)

    def check_slice_len(self, length: int):
        if self.cfg.mode == "blocked" and length % self.cfg.block_size:
            raise ValidationError(f"slice length {length} is not a multiple of block_size {self.cfg.block_size}")


@dataclass
class _Contribs:
    parts: list


class PassthroughCodec:
    """Identity codec for routing tests (zs/collectives.py:101-142): fusing
    concatenates contribution lists; the single final f64 fold runs in
    ascending source order whatever the route."""

    is_passthrough = True

    def encode(self, values, prior_depth: int = 0) -> WirePayload:
        v = _flat_values(values).to(torch.float64)
        return WirePayload(data=_Contribs([v]), n=int(v.numel()), depth=prior_depth)

    def decode(self, wp: WirePayload) -> torch.Tensor:
        acc = wp.data.parts[0].clone()
        for p in wp.data.parts[1:]:
            acc += p
        return acc

    def fuse(self, wps) -> WirePayload:
        wps = list(wps)
        return WirePayload(data=_Contribs([p for wp in wps for p in wp.data.parts]), n=wps[0].n,
                           depth=max(wp.depth for wp in wps))

    def reduce_final(self, wps) -> torch.Tensor:
        return self.decode(self.fuse(list(wps)))

    def slice(self, wp: WirePayload, start: int, length: int) -> WirePayload:
        return WirePayload(data=_Contribs([p[start:start + length] for p in wp.data.parts]), n=length,
                           depth=wp.depth)

    def accounting(self, wp: WirePayload):
        return wp.n * FP16_BYTES, 0, 0

    def payload_bytes_for(self, n_elems: int) -> int:
        return n_elems * FP16_BYTES

    def check_slice_len(self, length: int):
        pass


def as_codec(codec_or_cfg):
    """zs/collectives.py:145-148."""
    if isinstance(codec_or_cfg, QuantConfig):
        return BlockCodec(codec_or_cfg)
    return codec_or_cfg


@dataclass
class GatherResult:
    gathered: list  # per-rank FlatTensor (ranks of one group share one tensor)
    trace: object
    codec_depth: int = 0
    quantized: list | None = None


@dataclass
class ReduceResult:
    shards: list
    trace: object
    codec_depth: int = 0
    error_bounds: list | None = None


def _check_equal_inputs(tensors, world):
    if len(tensors) != world:
        raise ValidationError(f"expected {world} per-rank inputs, got {len(tensors)}")
    n = len(tensors[0])
    if any(len(t) != n for t in tensors):
        raise ValidationError("per-rank inputs must have equal length")
    return n


def _check_scheduler(scheduler):
    if scheduler not in ("serial", "threads"):
        raise ValidationError(f"unknown scheduler {scheduler!r}")


def _wrap(t: torch.Tensor, web: int = FP16_BYTES) -> FlatTensor:
    ft = FlatTensor.__new__(FlatTensor)
    ft.values, ft.wire_element_bytes = t, web
    return ft


# ---------------------------------------------------------------------------
# all-gathers


def all_gather_baseline(shards, topo: ClusterTopology, ledger: TrafficLedger, *, label="allgather", groups=None,
                        valid_elems=None, scheduler="serial"):
    """Full-precision all-gather of equal shards, optionally per group -- the hpZ
    secondary gather when ``groups=PartitionSpec.groups()`` (zs/collectives.py:202-241).
    Values are copied bit-identically; ranks of one group share one output tensor."""
    _check_scheduler(scheduler)
    world = topo.world
    if len(shards) != world:
        raise ValidationError(f"expected {world} shards, got {len(shards)}")
    if groups is None:
        groups = [list(range(world))]
    group_of = {}
    for g, members in enumerate(groups):
        for r in members:
            if r in group_of:
                raise ValidationError(f"rank {r} in two gather groups")
            group_of[r] = g
    if sorted(group_of) != list(range(world)):
        raise ValidationError("groups must cover every rank exactly once")
    shards = [as_flat(s) for s in shards]
    shard_len = len(shards[0])
    if any(len(s) != shard_len for s in shards):
        raise ValidationError("shards must have equal length")
    web = shards[0].wire_element_bytes
    trace = account_allgather(ledger, topo, label, shard_len, web, groups=groups, valid_elems=valid_elems)
    outs = []
    for members in groups:
        cat = torch.cat([shards[m].cuda_values() for m in members]) if members else None
        outs.append(_wrap(cat, web))
    gathered = [outs[group_of[r]] for r in range(world)]
    return GatherResult(gathered=gathered, trace=trace)


def all_gather_qwz(shards, codec, topo: ClusterTopology, ledger: TrafficLedger, *, label="allgather",
                   valid_elems=None, scheduler="serial"):
    """qwZ (zs/collectives.py:244-282): each rank quantizes its shard once (K0,
    blocks restart at the shard start); the receive side decodes all W payloads,
    own included, with one gather-dequantize launch (K4).  Every rank's result
    equals the concatenation of ``dequantize(quantize(shard_r))``."""
    _check_scheduler(scheduler)
    codec = as_codec(codec)
    world = topo.world
    shards = [as_flat(s) for s in shards]
    shard_len = _check_equal_inputs(shards, world)
    encoded = [codec.encode(s) for s in shards]
    trace = account_qwz(ledger, topo, label, codec, shard_len, valid_elems=valid_elems)
    if codec.is_passthrough:
        out = torch.cat([codec.decode(wp) for wp in encoded])
    else:
        out = _gather_decode([wp.data for wp in encoded], codec.out_dtype)
    g = _wrap(out)
    return GatherResult(gathered=[g] * world, trace=trace, codec_depth=max(wp.depth for wp in encoded),
                        quantized=None if codec.is_passthrough else [wp.data for wp in encoded])


def _gather_decode(qs: list[QuantizedTensor], out_dtype: torch.dtype) -> torch.Tensor:
    """One K4 launch decoding every shard into the concatenated output."""
    q0 = qs[0]
    n = q0.original_len
    out = torch.empty(n * len(qs), dtype=out_dtype, device=device())
    if n == 0:
        return out
    cfgs = {(q.config, q.absmax.dtype, q.original_len) for q in qs}
    if len(cfgs) != 1:
        raise ValidationError("qwZ shards must share config, dtype and length")
    f = new_flag()
    cp, _k1 = _lib.ptr_array([q.codes.data_ptr() for q in qs])
    ap, _k2 = _lib.ptr_array([q.absmax.data_ptr() for q in qs])
    _lib.check(_lib.load().zpp_gather_dequantize(cp, ap, q0.absmax_code, len(qs), 0, n, q0.config.bit_width,
                                                 q0.config.block_size, out.data_ptr(), dtype_code(out_dtype), n,
                                                 None, 0, 0, f.data_ptr(), stream_ptr()), "all_gather_qwz")
    check_flag(f, "all_gather_qwz")
    return out


# ---------------------------------------------------------------------------
# reduce-scatters


def reduce_scatter_ring(inputs, topo: ClusterTopology, ledger: TrafficLedger, *, label="reduce_scatter",
                        valid_elems=None, scheduler="serial"):
    """Full-precision reduce-scatter baseline (zs/collectives.py:289-331): rank r
    gets the f64 fold over ascending source of chunk r.  (Across GPUs the
    comparator is NCCL's bf16 reduce-scatter, see dist.py.)"""
    _check_scheduler(scheduler)
    world = topo.world
    inputs = [as_flat(t) for t in inputs]
    n = _check_equal_inputs(inputs, world)
    if n % world:
        raise ValidationError(f"input length {n} not divisible by world {world}")
    chunk = n // world
    web = inputs[0].wire_element_bytes
    trace = account_ring(ledger, topo, label, n, web, valid_elems=valid_elems)
    vals = [t.cuda_values().to(torch.float64) for t in inputs]
    shards = []
    for r in range(world):
        if world == 1:
            total = vals[0][r * chunk:(r + 1) * chunk].clone()
        else:
            total = torch.zeros(chunk, dtype=torch.float64, device=device())
            for v in vals:
                total += v[r * chunk:(r + 1) * chunk]
        shards.append(_wrap(total, web))
    return ReduceResult(shards=shards, trace=trace)


@dataclass
class ReorderPermutation:
    """Slice permutation that makes the two-hop all-to-all land correctly
    (zs/collectives.py:388-404)."""

    gpus_per_node: int
    nodes: int
    stages: int
    forward: np.ndarray
    inverse: np.ndarray


def reorder_mapping(gpus_per_node: int, nodes: int, stages: int = 1) -> ReorderPermutation:
    """Closed-form pre-transpose (zs/collectives.py:407-417; paper Eq. 1-2):
    within each stage's block of T = X*Y slices, slice X*c + j moves to position
    Y*j + c, so the intra-node message to local peer j carries the partitions of
    ranks {c*X + j : c < Y}."""
    if min(gpus_per_node, nodes, stages) < 1:
        raise ValidationError("reorder_mapping arguments must be >= 1")
    x, y = gpus_per_node, nodes
    t = x * y
    ids = np.arange(stages * t)
    base, pos = (ids // t) * t, ids % t
    forward = base + (pos % x) * y + pos // x
    inverse = base + (pos % y) * x + pos // y
    return ReorderPermutation(x, y, stages, forward=forward, inverse=inverse)


def qgz_2hop(inputs, codec, topo: ClusterTopology, ledger: TrafficLedger, *, stages: int = 1, intra_codec=None,
             reorder: bool = True, label="reduce_scatter", valid_elems=None, collect_bounds: bool = False,
             scheduler="serial"):
    """Hierarchical two-hop quantized reduce-scatter (zs/collectives.py:464-569).

    Per stage and rank: K1 quantizes the reordered slices straight into the
    hop-1 send buffer [j][c][e]; K2 fuses the X messages a rank receives
    (ascending local source) into one requantized tensor; K3 folds the Y
    segments it receives (ascending node) in f64.  Each element passes through
    exactly two codec round trips (``codec_depth == 2``)."""
    _check_scheduler(scheduler)
    codec = as_codec(codec)
    intra = codec if intra_codec is None else as_codec(intra_codec)
    if codec.is_passthrough != intra.is_passthrough:
        raise ValidationError("intra and inter codecs must both be real or both passthrough")
    if collect_bounds and codec.is_passthrough:
        raise ValidationError("error bounds require a quantizing codec")
    world = topo.world
    x, y, s = topo.gpus_per_node, topo.nodes, stages
    if s < 1:
        raise ValidationError("stages must be >= 1")
    inputs = [as_flat(t) for t in inputs]
    n = _check_equal_inputs(inputs, world)
    t = x * y
    if n % (s * t):
        raise ValidationError(f"input length {n} not divisible by stages*world = {s * t}")
    L = n // (s * t)
    intra.check_slice_len(L)
    codec.check_slice_len(L)
    if not codec.is_passthrough and (codec.cfg.mode != "blocked" or intra.cfg.mode != "blocked"):
        raise ValidationError("slice_blocks requires block-aligned bounds")  # what the reference hits
    trace = account_qgz(ledger, topo, label, codec, intra, n, s, valid_elems=valid_elems)
    if codec.is_passthrough:
        shards = _qgz_protocol(inputs, codec, intra, topo, s, L, reorder)
        depth, bounds = 0, None
    else:
        shards, bounds = _qgz_kernels(inputs, codec, intra, topo, s, L, reorder, collect_bounds)
        depth = 2
    return ReduceResult(shards=shards, trace=trace, codec_depth=depth, error_bounds=bounds)


def _qgz_kernels(inputs, codec, intra, topo, s, L, reorder, collect_bounds):
    x, y = topo.gpus_per_node, topo.nodes
    world = x * y
    lib = _lib.load()
    icfg, ocfg = intra.cfg, codec.cfg
    vals = [t.cuda_values() for t in inputs]
    n = int(vals[0].numel())
    f = new_flag()
    outs = [torch.empty(s * L, dtype=codec.out_dtype, device=device()) for _ in range(world)]
    bounds = [torch.empty(s * L, dtype=torch.float64, device=device()) for _ in range(world)] if collect_bounds else None
    msg = y * L
    for st in range(s):
        # K1: hop-1 send buffers
        sends = []
        for r in range(world):
            v = vals[r]
            q = alloc_quantized(world * L, icfg, torch.float64 if v.dtype == torch.float64 else torch.float32)
            _lib.check(lib.zpp_swizzle_quantize(v.data_ptr(), dtype_code(v.dtype), n, x, y, s, st, int(reorder),
                                                icfg.bit_width, icfg.block_size, q.codes.data_ptr(),
                                                q.absmax.data_ptr(), f.data_ptr(), stream_ptr()), "qgz_2hop")
            sends.append([q.slice_blocks(j * msg, msg) for j in range(x)])
        # K2 at every receiver: messages in ascending local source order
        fused = []
        for r in range(world):
            node, loc = divmod(r, x)
            hop1 = [sends[node * x + j][loc] for j in range(x)]
            fused.append(fused_dequant_reduce_quant(hop1, ocfg, flag=f))
        # K3 at every receiver: segments in ascending node order
        for r in range(world):
            node, loc = divmod(r, x)
            segs = [fused[c * x + loc].slice_blocks(node * L, L) for c in range(y)]
            dequant_reduce(segs, out=outs[r][st * L:(st + 1) * L], flag=f)
            if collect_bounds:
                s1 = []
                for c in range(y):
                    src = c * x + loc
                    sn, sl = divmod(src, x)
                    blk = torch.stack([sends[sn * x + j][sl].scales for j in range(x)]).max(0).values
                    s1.append(torch.repeat_interleave(blk, icfg.block_size)[node * L:(node + 1) * L])
                s1max = torch.stack(s1).max(0).values
                s2max = torch.stack([torch.repeat_interleave(g.scales, ocfg.block_size)[:L] for g in segs]).max(0).values
                bounds[r][st * L:(st + 1) * L] = y * (x * s1max / 2 + s2max / 2)
    check_flag(f, "qgz_2hop")
    return [_wrap(o) for o in outs], bounds


def _qgz_protocol(inputs, codec, intra, topo, s, L, reorder):
    """Codec-protocol route (used with PassthroughCodec), zs/collectives.py:502-544."""
    x, y = topo.gpus_per_node, topo.nodes
    world = x * y
    perm = reorder_mapping(x, y, 1)
    resid_at = perm.inverse if reorder else np.arange(x * y)
    part = s * L
    vals = [t.cuda_values().to(torch.float64) for t in inputs]
    outs = [torch.empty(part, dtype=torch.float64, device=device()) for _ in range(world)]
    for st in range(s):
        sent = {}
        for r in range(world):
            node = r // x
            for j in range(x):
                parts = [vals[r][int(resid_at[j * y + c]) * part + st * L:][:L] for c in range(y)]
                sent[(r, node * x + j)] = intra.encode(torch.cat(parts))
        fused = {}
        for r in range(world):
            node = r // x
            fused[r] = codec.fuse([sent[(node * x + j, r)] for j in range(x)])
        segs = {}
        for r in range(world):
            loc = r % x
            for c in range(y):
                segs[(r, c * x + loc)] = codec.slice(fused[r], c * L, L)
        for r in range(world):
            loc = r % x
            received = [segs[(c * x + loc, r)] for c in range(y)]
            outs[r][st * L:(st + 1) * L] = codec.reduce_final(received)
    return [_wrap(o) for o in outs]


# ---------------------------------------------------------------------------
# comparators the paper argues against (zs/collectives.py:334-381, :420-461)


def qgz_1hop(inputs, codec, topo: ClusterTopology, ledger: TrafficLedger, *, label="reduce_scatter",
             valid_elems=None, scheduler="serial"):
    """Single all-to-all quantized reduce-scatter (zs/collectives.py:420-461):
    each rank encodes every destination chunk once, destinations fold in
    ascending source order.  One codec pass, but X-fold cross-node volume."""
    _check_scheduler(scheduler)
    codec = as_codec(codec)
    world = topo.world
    inputs = [as_flat(t) for t in inputs]
    n = _check_equal_inputs(inputs, world)
    if n % world:
        raise ValidationError(f"input length {n} not divisible by world {world}")
    chunk = n // world
    trace = account_qgz_1hop(ledger, topo, label, codec, n, valid_elems=valid_elems)
    vals = [t.cuda_values() for t in inputs]
    sent = [[codec.encode(vals[r][d * chunk:(d + 1) * chunk]) for d in range(world)] for r in range(world)]
    shards = [_wrap(codec.reduce_final([sent[r][d] for r in range(world)])) for d in range(world)]
    depth = max(wp.depth for row in sent for wp in row)
    return ReduceResult(shards=shards, trace=trace, codec_depth=depth)


def reduce_scatter_ring_naive_quant(inputs, codec, topo: ClusterTopology, ledger: TrafficLedger, *,
                                    label="reduce_scatter", scheduler="serial"):
    """Ring reduce-scatter that re-quantizes the running partial at every hop
    (zs/collectives.py:334-381): codec depth world-1, the error the two-hop
    scheme removes."""
    _check_scheduler(scheduler)
    codec = as_codec(codec)
    world = topo.world
    inputs = [as_flat(t) for t in inputs]
    n = _check_equal_inputs(inputs, world)
    if n % world:
        raise ValidationError(f"input length {n} not divisible by world {world}")
    chunk = n // world
    trace = account_ring_naive_quant(ledger, topo, label, codec, n)
    vals = [t.cuda_values().to(torch.float64) for t in inputs]
    shards, depth = [], 0
    for dst in range(world):
        # the partial for chunk dst starts at rank dst+1 and travels the ring to dst
        order = [(dst + 1 + k) % world for k in range(world)]
        wp = None
        for r in order[:-1]:
            piece = vals[r][dst * chunk:(dst + 1) * chunk]
            if wp is None:
                wp = codec.encode(piece.clone())
            else:
                wp = codec.encode(codec.decode(wp).to(torch.float64) + piece, prior_depth=wp.depth)
        own = vals[dst][dst * chunk:(dst + 1) * chunk]
        if wp is None:
            shards.append(_wrap(own.clone()))
        else:
            shards.append(_wrap(codec.decode(wp).to(torch.float64) + own))
            depth = max(depth, wp.depth)
    return ReduceResult(shards=shards, trace=trace, codec_depth=depth)
