"""CPU oracle for the ZeRO++ hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference algorithms in
``zerosim`` (``/root/reference/pkg/src/zerosim``).  It exists so that

* ``tests/`` can check the CUDA path bit-for-bit on seeded inputs,
* ``__graft_entry__.smoke()`` can check one small invocation, and
* ``bench.py`` can time the reference algorithm on the host (``cpu_baseline``
  and ``--impl reference``).

Nothing in the product package (``paper_2306_10209_b200``) imports it; the
product path has no CPU fallback.

Parity pinning: every function here is checked against golden vectors that
were produced by running the real reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's own known-answer tests (``pkg/tests/test_quantizer.py:51-77``,
``pkg/tests/test_collectives.py:193-201``); see ``tests/test_oracle.py``.

Numerics follow the reference exactly: values are carried in float64,
``scale = maxabs / qmax``, ``inv = qmax / maxabs`` (0 for an all-zero block),
``code = clip(rint(x * inv), -qmax, qmax)`` with numpy's round-half-to-even,
INT4 packed low nibble first, full-precision reductions folded left to right
from +0.0 in ascending source order.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SCALE_WIRE_BYTES = 2  # zs/quantizer.py:24 -- accounted width of one scale


# ---------------------------------------------------------------------------
# codec (zs/quantizer.py)


def qmax_of(bits: int) -> int:
    """zs/quantizer.py:57-59."""
    return (1 << (bits - 1)) - 1


def effective_block(bits: int, block: int, mode: str, n: int) -> int:
    """zs/quantizer.py:179-182: full_tensor -> one block of n rounded up to 8."""
    if mode == "full_tensor":
        return max(8, -(-n // 8) * 8)
    return block


def pack(codes: np.ndarray, bits: int) -> np.ndarray:
    """zs/quantizer.py:185-189: int8 two's complement, or two nibbles/byte low first."""
    u = codes.astype(np.int8).view(np.uint8)
    if bits == 8:
        return u.copy()
    u = u & 0x0F
    return (u[0::2] | (u[1::2] << 4)).astype(np.uint8)


def unpack(packed: np.ndarray, bits: int, count: int) -> np.ndarray:
    """zs/quantizer.py:192-201: signed codes as int64 (nibbles >= 8 sign-extend)."""
    packed = np.asarray(packed, dtype=np.uint8)
    if bits == 8:
        return packed.view(np.int8).astype(np.int64)[:count]
    out = np.empty(packed.size * 2, dtype=np.int64)
    out[0::2] = packed & 0x0F
    out[1::2] = packed >> 4
    out -= (out >= 8) * 16
    return out[:count]


def quantize(values, bits: int, block: int, mode: str = "blocked"):
    """zs/quantizer.py:204-228.

    Returns ``(codes uint8, scales float64, eff_block)``.  ``codes`` includes
    the zero padding of the last block.
    """
    x = np.asarray(values, dtype=np.float64).reshape(-1)
    if not np.all(np.isfinite(x)):  # zs/quantizer.py:73-74
        raise ValueError("non-finite input")
    n = x.size
    b = effective_block(bits, block, mode, n)
    nb = -(-n // b) if n else 0
    grid = np.zeros(nb * b, dtype=np.float64)
    grid[:n] = x
    grid = grid.reshape(nb, b)
    q = qmax_of(bits)
    m = np.abs(grid).max(axis=1) if nb else np.zeros(0)
    scales = m / q
    inv = np.zeros_like(m)
    np.divide(q, m, out=inv, where=m > 0)
    codes = np.clip(np.rint(grid * inv[:, None]), -q, q)
    return pack(codes.reshape(-1), bits), scales, b


def dequantize(codes, scales, n: int, bits: int, block: int) -> np.ndarray:
    """zs/quantizer.py:231-238 (raises ValueError where the reference raises
    IntegrityError on an out-of-range code)."""
    scales = np.asarray(scales, dtype=np.float64)
    nb = scales.size
    c = unpack(codes, bits, nb * block)
    if np.any(np.abs(c) > qmax_of(bits)):
        raise ValueError("code outside symmetric range")
    vals = c.reshape(nb, block).astype(np.float64) * scales[:, None]
    return vals.reshape(-1)[:n]


def fused_dequant_reduce_quant(inputs, out_bits: int, out_block: int, out_mode="blocked"):
    """zs/quantizer.py:241-258.  ``inputs`` = [(codes, scales, n, bits, block)]."""
    if not inputs:
        raise ValueError("fused reduce needs at least one input")
    n = inputs[0][2]
    acc = np.zeros(n, dtype=np.float64)
    for codes, scales, m, bits, block in inputs:
        acc += dequantize(codes, scales, m, bits, block)
    return quantize(acc, out_bits, out_block, out_mode)


def accounting(n: int, bits: int, block: int, mode: str = "blocked"):
    """(payload, metadata, padding) wire bytes -- zs/quantizer.py:103-115,
    zs/collectives.py:186-195."""
    b = effective_block(bits, block, mode, n)
    nb = -(-n // b) if n else 0
    payload = math.ceil(n * bits / 8)
    total = nb * b * bits // 8
    return payload, nb * SCALE_WIRE_BYTES, total - payload


# ---------------------------------------------------------------------------
# partitions and slice reordering


def balanced(total: int, parts: int, index: int):
    """zs/partitioner.py:52-56."""
    base, rem = divmod(total, parts)
    start = index * base + min(index, rem)
    return start, start + base + (1 if index < rem else 0)


def primary_range(total: int, world: int, rank: int):
    """zs/partitioner.py:58-61."""
    return balanced(total, world, rank)


def secondary_range(total: int, group_size: int, rank: int):
    """zs/partitioner.py:75-82."""
    return balanced(total, group_size, rank % group_size)


def reorder_mapping(x: int, y: int, s: int = 1):
    """zs/collectives.py:407-417: (forward, inverse) slice permutations."""
    t = x * y
    ids = np.arange(s * t)
    st, res = ids // t, ids % t
    forward = st * t + (res % x) * y + res // x
    inverse = st * t + (res % y) * x + res // y
    return forward, inverse


# ---------------------------------------------------------------------------
# collectives (zs/collectives.py), restated per rank without the simulated fabric


def all_gather_qwz(shards, bits: int, block: int, mode: str = "blocked"):
    """zs/collectives.py:244-282: every rank quantizes its shard once (blocks
    restart at the shard start); every rank decodes all W payloads, its own
    included, in rank order.  Returns (gathered f64, [(codes, scales, eff_block)])."""
    enc = [quantize(s, bits, block, mode) for s in shards]
    parts = [dequantize(c, sc, len(s), bits, b) for (c, sc, b), s in zip(enc, shards)]
    return np.concatenate(parts) if parts else np.zeros(0), enc


def all_gather_groups(shards, groups):
    """zs/collectives.py:202-241 (hpZ with groups): rank r receives the
    concatenation of its group's shards in member order."""
    out = {}
    for members in groups:
        cat = np.concatenate([np.asarray(shards[m], dtype=np.float64) for m in members])
        for m in members:
            out[m] = cat
    return [out[r] for r in range(len(shards))]


def reduce_scatter_ring(inputs, world: int):
    """zs/collectives.py:289-331: rank r gets the ascending-source fold of chunk r."""
    n = len(inputs[0])
    chunk = n // world
    acc = np.zeros(n, dtype=np.float64)
    for a in inputs:
        acc = acc + np.asarray(a, dtype=np.float64)
    return [acc[r * chunk:(r + 1) * chunk] for r in range(world)]


def qgz_send_layout(vals, x: int, y: int, s: int, stage: int, reorder: bool = True):
    """Hop-1 send buffer of one rank for one stage, layout [j][c][e].

    zs/collectives.py:509-518: message j (to local peer j) is the concat over
    c < Y of the slice at residue resid_at[j*Y + c] of this stage.
    """
    n = len(vals)
    t = x * y
    L = n // (s * t)
    part = s * L
    _, inverse = reorder_mapping(x, y, 1)
    resid_at = inverse if reorder else np.arange(t)
    out = np.empty(t * L, dtype=np.float64)
    for k in range(t):
        off = int(resid_at[k]) * part + stage * L
        out[k * L:(k + 1) * L] = vals[off:off + L]
    return out


def qgz_2hop(inputs, x: int, y: int, s: int, inter_bits: int, inter_block: int,
             intra_bits: int | None = None, intra_block: int | None = None,
             reorder: bool = True, return_hops: bool = False):
    """zs/collectives.py:464-569 for quantizing codecs, restated per rank.

    Per stage: hop-1 messages quantized with the intra config, every rank
    fuses the X messages it receives (ascending local source; dequantize,
    f64 fold, requantize with the inter config), slices the fused tensor into
    Y segments of L, and after the cross-node exchange folds the Y segments it
    receives (ascending node) in f64 from +0.0.
    Returns per-rank f64 partitions (and the intermediate wire tensors if
    ``return_hops``).
    """
    intra_bits = inter_bits if intra_bits is None else intra_bits
    intra_block = inter_block if intra_block is None else intra_block
    world = x * y
    vals = [np.asarray(v, dtype=np.float64) for v in inputs]
    n = len(vals[0])
    L = n // (s * world)
    outs = [np.empty(s * L, dtype=np.float64) for _ in range(world)]
    hops = []
    for st in range(s):
        # hop 1: encode messages
        send = []
        for r in range(world):
            buf = qgz_send_layout(vals[r], x, y, s, st, reorder)
            msgs = [quantize(buf[j * y * L:(j + 1) * y * L], intra_bits, intra_block)
                    for j in range(x)]
            send.append(msgs)
        # fuse at each receiver
        fused = []
        for r in range(world):
            node, loc = divmod(r, x)
            ins = [(send[node * x + src][loc][0], send[node * x + src][loc][1], y * L,
                    intra_bits, intra_block) for src in range(x)]
            fused.append(fused_dequant_reduce_quant(ins, inter_bits, inter_block))
        # hop 2 + final fold
        for r in range(world):
            node, loc = divmod(r, x)
            acc = np.zeros(L, dtype=np.float64)
            for c in range(y):
                codes, scales, _ = fused[c * x + loc]
                bpb = inter_block * inter_bits // 8
                b0, nb = node * L // inter_block, L // inter_block
                acc += dequantize(codes[b0 * bpb:(b0 + nb) * bpb], scales[b0:b0 + nb], L,
                                  inter_bits, inter_block)
            outs[r][st * L:(st + 1) * L] = acc
        if return_hops:
            hops.append((send, fused))
    return (outs, hops) if return_hops else outs


def qgz_2hop_slices(src, x: int, y: int, inter_bits: int, inter_block: int,
                    intra_bits: int | None = None, intra_block: int | None = None) -> np.ndarray:
    """One rank's qgZ output at sampled positions, from the W source ranks'
    inputs at the same positions (zs/collectives.py:464-569 with reordering on,
    restated through SURVEY Appendix A's index map).

    Rank r's output element ``st*L + e`` is
    ``fold_c'( dequant( requant_inter( fold_j'( dequant( quant_intra(
    grad_{c'*X + j'}[r*S*L + st*L + e] ))))))`` -- folds from +0.0 in ascending
    j' (local source) and c' (group).  Quantization blocks tile the slice
    grid, so ``src`` (shape (W, K)) may concatenate any number of sampled
    slices as long as each is a whole number of intra and inter blocks and
    block-aligned in the output partition.  Checked against qgz_2hop in
    tests/test_synth.py."""
    intra_bits = inter_bits if intra_bits is None else intra_bits
    intra_block = inter_block if intra_block is None else intra_block
    src = np.asarray(src, dtype=np.float64)
    k = src.shape[1]
    out = np.zeros(k, dtype=np.float64)
    for c in range(y):
        acc = np.zeros(k, dtype=np.float64)
        for j in range(x):
            codes, scales, _ = quantize(src[c * x + j], intra_bits, intra_block)
            acc += dequantize(codes, scales, k, intra_bits, intra_block)
        codes, scales, _ = quantize(acc, inter_bits, inter_block)
        out += dequantize(codes, scales, k, inter_bits, inter_block)
    return out


# ---------------------------------------------------------------------------
# multi-threaded drivers for the CPU baseline (bench.py only)


def _pool_map(fn, items, threads):
    if threads <= 1:
        return [fn(i) for i in items]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, items))


def qwz_roundtrip_threaded(shard: np.ndarray, bits: int, block: int, threads: int | None = None,
                           out_dtype=np.float16):
    """quantize -> dequantize of one shard split into block-aligned chunks over
    host threads (numpy releases the GIL inside its kernels).  Same values as
    ``dequantize(*quantize(shard))`` because blocks are independent."""
    threads = threads or os.cpu_count() or 1
    n = shard.size
    nb = -(-n // block)
    per = -(-nb // threads) * block
    starts = list(range(0, n, per)) or [0]
    out = np.empty(n, dtype=out_dtype)

    def work(s0):
        seg = shard[s0:s0 + per]
        c, sc, b = quantize(seg, bits, block)
        out[s0:s0 + seg.size] = dequantize(c, sc, seg.size, bits, b).astype(out_dtype)

    _pool_map(work, starts, threads)
    return out
