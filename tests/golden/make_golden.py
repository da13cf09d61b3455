"""Generate golden vectors by running the REAL reference (zerosim) in the build
container.  The reference cannot travel to the GPU box, so its outputs are
committed as small ``.npz`` fixtures next to this script.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Inputs are generated in the dtype the GPU path consumes (fp16 / bf16 / fp32 /
f64) and handed to the reference as the exactly-equal float64 values, which is
what ``zerosim.FlatTensor`` does with any array (zs/quantizer.py:69-70).
bf16 arrays are stored as their uint16 bit patterns (numpy has no bf16).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("ZEROSIM_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import zerosim as zs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_bits_from_f32(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def as_f64(arr: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return bf16_bits_to_f64(arr)
    return np.asarray(arr).astype(np.float64)


# ---------------------------------------------------------------------------
# quantize / dequantize cases


def quant_cases():
    rng = np.random.default_rng(20230617)
    cases = []

    def add(name, arr, dtype, bits, block, mode="blocked"):
        cases.append((name, arr, dtype, bits, block, mode))

    # known answers from pkg/tests/test_quantizer.py
    add("kat_canonical_int8", np.array([1.0, -1.0, 0.5, -0.5]), "f64", 8, 8)
    add("kat_zero_int4", np.zeros(16), "f64", 4, 8)
    sc = np.float64(3.7) / 127
    lat = np.random.default_rng(7).integers(-127, 128, size=300).astype(np.float64) * sc
    lat[np.argmax(np.abs(lat))] = 127 * sc
    add("kat_lattice_full_tensor", lat, "f64", 8, 2048, "full_tensor")
    for bits, block in [(8, 64), (8, 2048), (4, 8), (4, 512)]:
        r = np.random.default_rng(bits * 1000 + block)
        add(f"kat_scalar_oracle_{bits}_{block}", r.normal(size=block * 3 + 5), "f64", bits, block)
    add("kat_wire_1021_int4", np.ones(1021), "f64", 4, 512)
    add("kat_full_tensor_100", np.random.default_rng(11).normal(size=100), "f64", 8, 2048, "full_tensor")
    add("kat_blocked_104", np.random.default_rng(11).normal(size=100), "f64", 8, 104)

    # the dtypes the hot path consumes
    w = (rng.normal(size=20000) * 0.02).astype(np.float16)
    add("fp16_weights_int8_2048", w, "fp16", 8, 2048)
    add("fp16_weights_int4_512", w, "fp16", 4, 512)
    g = rng.normal(size=9000) * np.exp(rng.normal(size=9000)) * 1e-3
    add("bf16_grads_int4_512", bf16_bits_from_f32(g), "bf16", 4, 512)
    add("bf16_grads_int8_2048", bf16_bits_from_f32(g), "bf16", 8, 2048)
    x = (rng.normal(size=70001) * np.exp(rng.normal(size=70001))).astype(np.float32)
    add("fp32_heavy_int8_2048", x, "fp32", 8, 2048)
    add("fp32_heavy_int4_512", x, "fp32", 4, 512)
    add("fp32_heavy_int8_24", x[:6000], "fp32", 8, 24)
    add("fp32_heavy_int4_full", x[:5003], "fp32", 4, 2048, "full_tensor")
    add("f64_normal_int8_256", rng.normal(size=4099) * 5, "f64", 8, 256)
    add("f64_normal_int4_16", rng.normal(size=777), "f64", 4, 16)

    # every positive fp16 value <= m in one block, both signs, for several m:
    # exercises every rounding tie the fp16 grid can produce
    allpos = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16)
    for m_bits in (0x3C00, 0x3555, 0x2E66, 0x0400):  # 1.0, ~0.333, ~0.1, min normal
        m = np.uint16(m_bits).view(np.float16)
        vals = allpos[allpos <= m]
        vals = np.concatenate([vals, -vals])
        blk = 1 << int(np.ceil(np.log2(vals.size)))
        add(f"fp16_exhaustive_m{m_bits:04x}_int8", vals, "fp16", 8, blk)
        add(f"fp16_exhaustive_m{m_bits:04x}_int4", vals, "fp16", 4, blk)
    # exact ties: x = (k + 0.5) * m / 127 in fp32 where representable
    m = np.float32(1.0)
    ties = (np.arange(-127, 127, dtype=np.float64) + 0.5) / 127.0
    t32 = np.concatenate([[m], ties.astype(np.float32)])
    add("fp32_ties_int8", np.resize(t32, 2048), "fp32", 8, 2048)
    ties4 = ((np.arange(-7, 7) + 0.5) / 7.0).astype(np.float32)
    add("fp32_ties_int4", np.resize(np.concatenate([[m], ties4]), 512), "fp32", 4, 512)
    # subnormal blocks (fp32 and bf16): the reciprocal overflows fp32
    sub = (rng.normal(size=1024) * 1e-39).astype(np.float32)
    add("fp32_subnormal_int8_512", sub, "fp32", 8, 512)
    add("fp32_subnormal_int4_512", sub, "fp32", 4, 512)
    add("bf16_tiny_int8_512", bf16_bits_from_f32(rng.normal(size=1024) * 1e-36), "bf16", 8, 512)
    # zero blocks mixed in, ragged tail
    zb = rng.normal(size=5000).astype(np.float32)
    zb[512:1024] = 0
    add("fp32_zero_block_int8_512", zb, "fp32", 8, 512)
    add("fp16_ragged_int4_512", (rng.normal(size=513)).astype(np.float16), "fp16", 4, 512)
    add("fp16_ragged_int8_2048", (rng.normal(size=2049)).astype(np.float16), "fp16", 8, 2048)
    add("fp16_tiny_n3", np.array([0.5, -0.25, 0.125], dtype=np.float16), "fp16", 4, 8)
    add("empty", np.zeros(0, dtype=np.float32), "fp32", 8, 2048)
    return cases


def build_quant():
    out = {}
    meta = []
    for i, (name, arr, dtype, bits, block, mode) in enumerate(quant_cases()):
        cfg = zs.QuantConfig(bit_width=bits, block_size=block, mode=mode)
        vals = as_f64(arr, dtype)
        q = zs.quantize(zs.FlatTensor(vals), cfg)
        deq = zs.dequantize(q).values
        out[f"{i}_input"] = np.asarray(arr)
        out[f"{i}_codes"] = q.codes
        out[f"{i}_scales"] = q.scales
        out[f"{i}_deq"] = deq
        meta.append(dict(idx=i, name=name, dtype=dtype, bits=bits, block=block, mode=mode,
                         eff_block=q.config.block_size, n=len(vals),
                         payload=q.payload_bytes, metadata=q.metadata_bytes,
                         padding=q.padding_bytes, wire=q.wire_bytes))
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **out)
    print("quant cases:", len(meta))


# ---------------------------------------------------------------------------
# fused dequant -> reduce -> requant


def build_fused():
    rng = np.random.default_rng(41)
    out = {}
    meta = []
    for i in range(200):
        k = int(rng.integers(1, 6))
        n = int(rng.integers(1, 1200))
        in_bits = int(rng.choice([4, 8]))
        in_block = int(rng.choice([8, 64, 512]))
        out_bits = int(rng.choice([4, 8]))
        out_block = int(rng.choice([8, 64, 512]))
        in_cfg = zs.QuantConfig(bit_width=in_bits, block_size=in_block)
        out_cfg = zs.QuantConfig(bit_width=out_bits, block_size=out_block)
        scale = float(rng.uniform(0.1, 10))
        vals = [rng.normal(size=n) * scale for _ in range(k)]
        qs = [zs.quantize(zs.FlatTensor(v), in_cfg) for v in vals]
        fused = zs.fused_dequant_reduce_quant(qs, out_cfg)
        for j, q in enumerate(qs):
            out[f"{i}_in{j}_values"] = vals[j]
            out[f"{i}_in{j}_codes"] = q.codes
            out[f"{i}_in{j}_scales"] = q.scales
        out[f"{i}_codes"] = fused.codes
        out[f"{i}_scales"] = fused.scales
        meta.append(dict(idx=i, k=k, n=n, in_bits=in_bits, in_block=in_block,
                         out_bits=out_bits, out_block=out_block))
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "fused.npz"), **out)
    print("fused cases:", len(meta))


# ---------------------------------------------------------------------------
# collectives


def build_collectives():
    out = {}
    meta = {"reorder": [], "partition": [], "qwz": [], "groups": [], "qgz": [], "ring": []}

    for x, y, s in [(1, 1, 1), (2, 2, 1), (2, 3, 1), (2, 2, 2), (4, 2, 1), (4, 2, 4), (3, 2, 2), (4, 3, 2)]:
        p = zs.reorder_mapping(x, y, s)
        key = f"reorder_{x}_{y}_{s}"
        out[key + "_fwd"] = p.forward
        out[key + "_inv"] = p.inverse
        meta["reorder"].append([x, y, s])

    for total, world, group in [(10, 4, 2), (12, 4, 4), (30, 6, 3), (1300004864, 8, 4),
                                (50364416, 8, 4), (7, 8, 2), (0, 2, 1)]:
        spec = zs.PartitionSpec(total_elems=total, world=world, group_size=group)
        key = f"part_{total}_{world}_{group}"
        out[key + "_primary"] = np.array([spec.primary_range(r) for r in range(world)], dtype=np.int64)
        out[key + "_secondary"] = np.array([spec.secondary_range(r) for r in range(world)], dtype=np.int64)
        out[key + "_groups"] = np.array(spec.groups(), dtype=np.int64)
        meta["partition"].append([total, world, group])

    # qwZ: equal shards; blocks restart at each shard start
    qcases = [(2, 2, 32, 8, 8, "f64"), (1, 8, 5000, 8, 2048, "fp16"), (2, 4, 4099, 8, 2048, "fp16"),
              (2, 2, 1000, 4, 512, "fp32"), (1, 1, 3000, 8, 2048, "fp16"), (1, 3, 777, 8, 64, "bf16")]
    for i, (nodes, gpn, shard_len, bits, block, dtype) in enumerate(qcases):
        rng = np.random.default_rng(1000 + i)
        world = nodes * gpn
        raw = []
        for r in range(world):
            v = rng.normal(size=shard_len) * 0.02 * (1 + r)
            raw.append(v.astype(np.float16) if dtype == "fp16" else
                       bf16_bits_from_f32(v) if dtype == "bf16" else
                       v.astype(np.float32) if dtype == "fp32" else v)
        shards = [zs.FlatTensor(as_f64(a, dtype)) for a in raw]
        topo = zs.ClusterTopology(nodes=nodes, gpus_per_node=gpn)
        ledger = zs.TrafficLedger()
        res = zs.all_gather_qwz(shards, zs.QuantConfig(bit_width=bits, block_size=block), topo, ledger)
        for r in range(world):
            out[f"qwz{i}_in{r}"] = raw[r]
            out[f"qwz{i}_codes{r}"] = res.quantized[r].codes
            out[f"qwz{i}_scales{r}"] = res.quantized[r].scales
            assert np.array_equal(res.gathered[r].values, res.gathered[0].values)
        out[f"qwz{i}_gathered"] = res.gathered[0].values
        vol = {f"{lb}|{cls}": [b.payload, b.metadata, b.padding] for (lb, cls), b in ledger.volume.items()}
        meta["qwz"].append(dict(idx=i, nodes=nodes, gpn=gpn, shard_len=shard_len, bits=bits,
                                block=block, dtype=dtype, depth=res.codec_depth, volume=vol))

    # hpZ grouped gather
    for i, (nodes, gpn, shard_len) in enumerate([(2, 2, 5), (2, 4, 1000), (3, 2, 17)]):
        rng = np.random.default_rng(3000 + i)
        world = nodes * gpn
        raw = [rng.normal(size=shard_len).astype(np.float16) for _ in range(world)]
        topo = zs.ClusterTopology(nodes=nodes, gpus_per_node=gpn)
        spec = zs.build_partitions(shard_len * gpn, topo)
        ledger = zs.TrafficLedger()
        res = zs.all_gather_baseline([zs.FlatTensor(a.astype(np.float64)) for a in raw], topo, ledger,
                                     groups=spec.groups())
        for r in range(world):
            out[f"grp{i}_in{r}"] = raw[r]
            out[f"grp{i}_out{r}"] = res.gathered[r].values
        vol = {f"{lb}|{cls}": [b.payload, b.metadata, b.padding] for (lb, cls), b in ledger.volume.items()}
        phys = {f"{lb}|{cls}": [b.payload, b.messages] for (lb, cls), b in ledger.physical.items()}
        meta["groups"].append(dict(idx=i, nodes=nodes, gpn=gpn, shard_len=shard_len, volume=vol,
                                   physical=phys))

    # qgZ two-hop
    gcases = []
    for x, y, s in [(2, 2, 1), (2, 3, 2), (4, 2, 1), (4, 2, 4), (1, 2, 1), (2, 1, 1), (1, 1, 1), (4, 3, 2)]:
        gcases.append((x, y, s, 4, 8, None, None, True, "f64", 8))
    gcases += [
        (2, 2, 1, 4, 512, None, None, True, "bf16", 512),
        (4, 2, 2, 4, 512, None, None, True, "bf16", 1024),
        (2, 2, 1, 4, 8, 8, 8, True, "f64", 16),       # int8 intra, int4 inter
        (4, 2, 1, 4, 512, 8, 256, True, "bf16", 512),  # mixed blocks
        (2, 2, 1, 4, 8, None, None, False, "f64", 8),  # no reorder: misplacement
        (2, 2, 1, 8, 8, None, None, True, "fp32", 16),
        (4, 2, 1, 8, 64, 4, 32, True, "fp16", 128),
    ]
    for i, (x, y, s, bits, block, ibits, iblock, reorder, dtype, L) in enumerate(gcases):
        rng = np.random.default_rng(2000 + i)
        world = x * y
        n = s * world * L
        raw = []
        for r in range(world):
            v = rng.normal(size=n) * np.exp(rng.normal(size=n)) * (1e-3 if dtype == "bf16" else 2.0)
            raw.append(v.astype(np.float16) if dtype == "fp16" else
                       bf16_bits_from_f32(v) if dtype == "bf16" else
                       v.astype(np.float32) if dtype == "fp32" else v)
        inputs = [zs.FlatTensor(as_f64(a, dtype)) for a in raw]
        topo = zs.ClusterTopology(nodes=y, gpus_per_node=x)
        ledger = zs.TrafficLedger()
        cfg = zs.QuantConfig(bit_width=bits, block_size=block)
        icfg = zs.QuantConfig(bit_width=ibits, block_size=iblock) if ibits else None
        res = zs.qgz_2hop(inputs, cfg, topo, ledger, stages=s, intra_codec=icfg, reorder=reorder)
        for r in range(world):
            out[f"qgz{i}_in{r}"] = raw[r]
            out[f"qgz{i}_out{r}"] = res.shards[r].values
        # passthrough routing on the same inputs = ring fold (exact for integers)
        ints = [zs.FlatTensor(np.random.default_rng(9000 + i + r).integers(-40, 41, size=n).astype(np.float64))
                for r in range(world)]
        pt = zs.qgz_2hop(ints, zs.PassthroughCodec(), topo, zs.TrafficLedger(), stages=s, reorder=reorder)
        for r in range(world):
            out[f"qgz{i}_int_in{r}"] = ints[r].values
            out[f"qgz{i}_int_out{r}"] = pt.shards[r].values
        vol = {f"{lb}|{cls}": [b.payload, b.metadata, b.padding] for (lb, cls), b in ledger.volume.items()}
        phys = {f"{lb}|{cls}": [b.payload, b.messages] for (lb, cls), b in ledger.physical.items()}
        meta["qgz"].append(dict(idx=i, x=x, y=y, s=s, bits=bits, block=block, ibits=ibits, iblock=iblock,
                                reorder=reorder, dtype=dtype, L=L, n=n, depth=res.codec_depth,
                                volume=vol, physical=phys))

    # fp ring reduce-scatter baseline
    for i, (nodes, gpn, n) in enumerate([(1, 2, 2), (2, 2, 24), (2, 4, 4096)]):
        rng = np.random.default_rng(4000 + i)
        world = nodes * gpn
        ins = [zs.FlatTensor(rng.normal(size=n) * 7.0) for _ in range(world)]
        res = zs.reduce_scatter_ring(ins, zs.ClusterTopology(nodes=nodes, gpus_per_node=gpn), zs.TrafficLedger())
        for r in range(world):
            out[f"ring{i}_in{r}"] = ins[r].values
            out[f"ring{i}_out{r}"] = res.shards[r].values
        meta["ring"].append(dict(idx=i, nodes=nodes, gpn=gpn, n=n))

    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "collectives.npz"), **out)
    print("collective cases:", {k: len(v) for k, v in meta.items()})


def build_wire():
    """to_bytes / from_bytes (zs/quantizer.py:121-149): raw wire bytes and the
    values the reference decodes from them (fp16 wire scales)."""
    out, meta = {}, []
    rng = np.random.default_rng(5)
    for i, (n, bits, block) in enumerate([(777, 4, 64), (5000, 8, 2048), (1021, 4, 512), (64, 8, 64)]):
        q = zs.quantize(zs.FlatTensor(rng.normal(size=n) * 3), zs.QuantConfig(bit_width=bits, block_size=block))
        raw = q.to_bytes()
        back = zs.QuantizedTensor.from_bytes(raw)
        out[f"{i}_raw"] = np.frombuffer(raw, dtype=np.uint8)
        out[f"{i}_codes"] = q.codes
        out[f"{i}_scales"] = q.scales
        out[f"{i}_deq_from_bytes"] = zs.dequantize(back).values
        meta.append(dict(idx=i, n=n, bits=bits, block=block))
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "wire.npz"), **out)
    print("wire cases:", len(meta))


def build_volumes():
    """step_volumes CSV (ledger volume rows) for the ZeRO / ZeRO++ switches."""
    rows = []
    for nodes, gpn in [(2, 4), (8, 4), (2, 2)]:
        for qw, hp, qg in [(False, False, False), (True, True, True), (True, False, False),
                           (False, True, False), (False, False, True)]:
            cfg = zs.ZeroConfig(nodes=nodes, gpus_per_node=gpn, quantized_weight_gather=qw,
                                hierarchical_secondary_gather=hp, quantized_grad_reduce=qg)
            m = 1 << 20
            ledger, vols, _ = zs.step_volumes(cfg, m)
            rows.append(dict(nodes=nodes, gpn=gpn, qw=qw, hp=hp, qg=qg, m=m, csv=ledger.to_csv(m),
                             vols=vols))
    with open(os.path.join(HERE, "volumes.json"), "w") as f:
        json.dump(rows, f, indent=1)
    print("volume cases:", len(rows))


ENGINE_CASES = [
    # (name, ZeroConfig kwargs, task kwargs, passthrough codecs)
    ("plain", {}, {}, False),
    ("qwz", dict(quantized_weight_gather=True), {}, False),
    ("hpz", dict(hierarchical_secondary_gather=True), {}, False),
    ("qgz", dict(quantized_grad_reduce=True), {}, False),
    ("all_on", dict(quantized_weight_gather=True, hierarchical_secondary_gather=True, quantized_grad_reduce=True),
     {}, False),
    ("all_on_s2_2x4", dict(nodes=2, gpus_per_node=4, grad_stages=2, quantized_weight_gather=True,
                           hierarchical_secondary_gather=True, quantized_grad_reduce=True), {}, False),
    ("qgz_half_int8_intra", dict(quantized_grad_reduce=True, grad_quant_fraction=0.5,
                                 grad_intra_quant=("q", 8, 256)), {}, False),
    ("qgz_slice_scale_c09", dict(quantized_grad_reduce=True, grad_quant=("q", 4, 2560), seed=1),
     dict(noise_sigma=0.1, input_scale_range=16.0), False),
    ("routed_passthrough_c08", dict(quantized_weight_gather=True, hierarchical_secondary_gather=True,
                                    quantized_grad_reduce=True), {}, True),
]


def _engine_cfg(kw):
    kw = dict(kw)
    for k, v in list(kw.items()):
        if isinstance(v, tuple) and v and v[0] == "q":
            kw[k] = zs.QuantConfig(bit_width=v[1], block_size=v[2])
    return kw


def build_engine(steps=40):
    """Whole toy training runs of the reference TrainingEngine
    (zs/engine.py:256-452): per-step losses and volumes, final master weights."""
    import hashlib

    rows = []
    for name, zkw, tkw, passthrough in ENGINE_CASES:
        eng = zs.TrainingEngine(zs.ToyTaskConfig(**tkw), zs.ZeroConfig(steps=steps, **_engine_cfg(zkw)))
        if passthrough:
            eng.weight_codec = zs.PassthroughCodec()
            eng.grad_codec = zs.PassthroughCodec()
        rec = eng.train()
        rows.append(dict(name=name, zero=zkw, task=tkw, passthrough=passthrough, steps=steps,
                         losses=[float(s.loss).hex() for s in rec.steps],
                         volumes=[[repr(s.fwd_gather_volume), repr(s.bwd_gather_volume), repr(s.reduce_volume)]
                                  for s in rec.steps],
                         quantized_grads=[bool(s.quantized_grads) for s in rec.steps],
                         csv_sha256=hashlib.sha256(rec.to_csv().encode()).hexdigest(),
                         initial_loss=float(rec.initial_loss).hex(), final_loss=float(rec.final_loss).hex(),
                         diverged=rec.diverged, padded=rec.padded_params,
                         master_sha256=hashlib.sha256(eng.master.tobytes()).hexdigest()))
    with open(os.path.join(HERE, "engine.json"), "w") as f:
        json.dump(rows, f, indent=1)
    print("engine cases:", len(rows))


if __name__ == "__main__":
    which = sys.argv[1:] or ["quant", "fused", "collectives", "volumes", "wire", "engine"]
    for name in which:
        globals()["build_" + name]()
