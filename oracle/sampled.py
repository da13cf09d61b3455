"""Sampled bitwise parity at full BASELINE sizes -- TEST INFRASTRUCTURE ONLY.

The GPU collectives run on multi-GB inputs generated on the device by
``oracle.synth.device``; these helpers pull a random sample of output blocks /
slices back to the host and recompute exactly those from the seeded inputs
with the oracle (``oracle.zpp_oracle``), comparing bit patterns (so -0.0 vs
+0.0 counts as a mismatch).  Used by the multi-GPU parity workers in
``tests/`` and by ``bench.py`` after its timed region (the line's ``parity``
key).  The product package never imports this module.

Seeds (one stream per rank and tensor):
* qwZ shard of rank r: ``seed_base + r``, kind "weight", fp16;
* qgZ gradient of rank q: ``seed_base + 1000 * q``, kind "grad", bf16.
"""

from __future__ import annotations

import numpy as np

from . import synth
from . import zpp_oracle as O

_BITS = {np.dtype(np.float16): np.uint16, np.dtype(np.float32): np.uint32, np.dtype(np.float64): np.uint64}


def _bits(a: np.ndarray) -> np.ndarray:
    return a.view(_BITS[a.dtype])


def _take(t, idx: np.ndarray) -> np.ndarray:
    """t[idx] for a CUDA tensor t and host int64 indices (gathered on the device)."""
    import torch

    i = torch.from_numpy(np.ascontiguousarray(idx.reshape(-1))).to(t.device)
    return t.index_select(0, i).cpu().numpy().reshape(idx.shape)


def qwz_check(out, world: int, shard_len: int, bits: int = 8, block: int = 2048, seed_base: int = 1000,
              samples: int = 4096, rng_seed: int = 0, out_dtype=np.float16, lo: int = 0, hi: int | None = None):
    """Check `samples` random whole quantization blocks of a qwZ-gathered
    buffer (rank order, shard_len per rank, blocks from each shard's start)
    against dequantize(quantize(shard)) of the seeded shards.  ``lo/hi``
    restrict the sample to gathered elements [lo, hi) of which `out` holds
    exactly that range (the hpZ gather's view).  Returns (elements checked,
    mismatching elements)."""
    total = world * shard_len
    hi = total if hi is None else hi
    nb_shard = -(-shard_len // block)
    rng = np.random.default_rng(rng_seed)
    # candidate blocks: whole blocks inside [lo, hi)
    first = [(r, b) for r in range(world) for b in (0, nb_shard - 1)]
    cand = rng.integers(0, world * nb_shard, size=samples)
    ranks, blks = cand // nb_shard, cand % nb_shard
    ranks = np.concatenate([ranks, [r for r, _ in first]])
    blks = np.concatenate([blks, [b for _, b in first]])
    checked = mism = 0
    for r in np.unique(ranks):
        sel = np.unique(blks[ranks == r])
        starts = r * shard_len + sel * block
        lens = np.minimum(block, shard_len - sel * block)
        keep = (starts >= lo) & (starts + lens <= hi)
        sel, starts, lens = sel[keep], starts[keep], lens[keep]
        if sel.size == 0:
            continue
        full = lens == block
        for group in (full, ~full):
            if not np.any(group):
                continue
            s_sel, s_starts, s_lens = sel[group], starts[group], lens[group]
            ln = int(s_lens[0])
            if not np.all(s_lens == ln):
                raise AssertionError("ragged blocks of different lengths")
            local = (s_sel * block)[:, None] + np.arange(ln)[None, :]
            x = synth.host_at(seed_base + int(r), local, "fp16", "weight")
            if ln == block:  # whole blocks tile a concatenation exactly
                codes, scales, _ = O.quantize(x.reshape(-1), bits, block)
                want = O.dequantize(codes, scales, x.size, bits, block).reshape(x.shape)
            else:  # the ragged last block of each shard, padded on its own
                want = np.stack([O.dequantize(*O.quantize(v, bits, block)[:2], ln, bits, block) for v in x])
            want = want.astype(out_dtype)
            got = _take(out, (s_starts - lo)[:, None] + np.arange(ln)[None, :])
            mism += int(np.count_nonzero(_bits(got) != _bits(want)))
            checked += got.size
    return checked, mism


def qgz_check(out, rank: int, world: int, group: int, n: int, stages: int = 1, inter=(4, 512), intra=None,
              seed_base: int = 2000, samples: int = 4096, rng_seed: int = 0, slice_len: int | None = None,
              valid: int | None = None):
    """Check `samples` random output slices (slice_len elements, default the
    larger block) of rank `rank`'s qgZ partition (n // world elements) against
    the per-slice oracle, bitwise in out's dtype.  ``valid``: inputs at bucket
    positions >= valid are the zero padding of a stream's tail bucket.
    Returns (checked, mismatches)."""
    intra = intra or inter
    x, y = group, world // group
    part = n // world
    sl = slice_len or max(inter[1], intra[1])
    n_sl = part // sl
    rng = np.random.default_rng(rng_seed + rank)
    pick = np.unique(np.concatenate([rng.integers(0, n_sl, size=min(samples, n_sl)), [0, n_sl - 1]]))
    pos = (pick[:, None] * sl + np.arange(sl)[None, :]).reshape(-1)
    src = np.stack([synth.host_at(seed_base + 1000 * q, rank * part + pos, "bf16", "grad") for q in range(world)])
    if valid is not None:
        src[:, rank * part + pos >= valid] = 0.0
    want = O.qgz_2hop_slices(src, x, y, inter[0], inter[1], intra[0], intra[1])
    got = _take(out, pos)
    want = want.astype(got.dtype)
    return got.size, int(np.count_nonzero(_bits(got) != _bits(want)))
