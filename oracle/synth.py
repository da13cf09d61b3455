"""Seeded counter-based synthetic inputs -- TEST INFRASTRUCTURE ONLY.

Element ``i`` of stream ``seed`` is a pure function of ``(seed, i)``, computed
with the same wrapping int64 and IEEE float32 operations by

* ``device(seed, lo, n, dtype)`` -- torch, any device (the inputs the GPU path
  consumes: tests and ``bench.py`` generate shards and gradient buckets on the
  GPU with it), and
* ``host(seed, lo, n, dtype)`` -- numpy (the oracle side),

so a parity check at full BASELINE sizes can recompute any rank's input at any
index on the host -- e.g. the W source slices behind one 512-element qgZ output
slice -- without materialising or transferring the
multi-GB tensors.  The two functions agree bit-for-bit (tests/test_synth.py).

Distributions (shape only; the parity tests do not depend on it):

* ``kind="weight"``: uniform magnitude times 2^-(0..3), times 0.04 -- about the
  N(0, 0.02^2) fp16 weights of SURVEY §8d config 2, with exact fp16 ties.
* ``kind="grad"``: uniform magnitude times 2^(-6..+1), times 1e-3 -- heavy
  tailed like N(0,1)*exp(N(0,1))*1e-3 (config 4), with many bf16 ties.

Nothing in the product package imports this module.
"""

from __future__ import annotations

import numpy as np

# splitmix64-style constants as signed int64 (torch has no uint64 arithmetic)
_C1 = -7046029254386353131  # 0x9E3779B97F4A7C15
_C2 = -4658895280553007687  # 0xBF58476D1CE4E5B9
_C3 = -7723592293110705685  # 0x94D049BB133111EB
# h >> k & _L[k] is the logical right shift of the 64-bit pattern
_L = {k: (1 << (64 - k)) - 1 for k in (27, 31, 32)}

# kind -> (scale, number of power-of-two steps, power-of-two table)
_KINDS = {"weight": (np.float32(0.04), 4, np.array([2.0 ** -k for k in range(4)], np.float32)),
          "grad": (np.float32(1e-3), 8, np.array([2.0 ** (k - 6) for k in range(8)], np.float32))}


def _mix_np(idx: np.ndarray, seed: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = idx * np.int64(_C1) + np.int64(seed * 1_000_003 + 12345)
        h = h ^ ((h >> 31) & _L[31])
        h = h * np.int64(_C2)
        h = h ^ ((h >> 27) & _L[27])
        h = h * np.int64(_C3)
        h = h ^ ((h >> 32) & _L[32])
    return h


def _values_np(h: np.ndarray, kind: str) -> np.ndarray:
    scale, n_exp, pow2 = _KINDS[kind]
    m = ((h >> 8) & 0xFFFF).astype(np.float32)          # 16-bit magnitude, exact in f32
    p = pow2[(h >> 24) & (n_exp - 1)]                    # power-of-two spread
    sgn = np.float32(1.0) - np.float32(2.0) * ((h >> 40) & 1).astype(np.float32)
    u = (m * np.float32(2.0) + np.float32(1.0)) * np.float32(2.0 ** -17)  # (0, 1), exact
    return (u * p * sgn) * scale                          # one rounding: the final multiply


def bf16_bits_from_f32(v: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bits, round to nearest even (torch's .bfloat16() for finite values)."""
    b = np.asarray(v, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def host(seed: int, lo: int, n: int, dtype: str = "fp16", kind: str = "weight") -> np.ndarray:
    """Elements [lo, lo+n) of stream `seed` as float64 values of `dtype`
    ('fp16', 'bf16' or 'fp32')."""
    idx = np.arange(lo, lo + n, dtype=np.int64)
    v = _values_np(_mix_np(idx, seed), kind)
    if dtype == "fp32":
        return v.astype(np.float64)
    if dtype == "fp16":
        return v.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        return (bf16_bits_from_f32(v).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    raise ValueError(dtype)


def host_at(seed: int, idx: np.ndarray, dtype: str = "fp16", kind: str = "weight") -> np.ndarray:
    """Like host() at arbitrary int64 indices (any shape)."""
    idx = np.asarray(idx, dtype=np.int64)
    v = _values_np(_mix_np(idx.reshape(-1), seed), kind)
    if dtype == "fp32":
        out = v.astype(np.float64)
    elif dtype == "fp16":
        out = v.astype(np.float16).astype(np.float64)
    elif dtype == "bf16":
        out = (bf16_bits_from_f32(v).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    else:
        raise ValueError(dtype)
    return out.reshape(idx.shape)


def device(seed: int, lo: int, n: int, dtype, kind: str = "weight", device=None, out=None, chunk: int = 1 << 26):
    """The same stream as host(), generated with torch ops (on `device`),
    written into `out` (a 1-D tensor of torch dtype `dtype`) chunk by chunk."""
    import torch

    if out is None:
        out = torch.empty(n, dtype=dtype, device=device)
    dev = out.device
    scale, n_exp, pow2 = _KINDS[kind]
    pow2 = torch.from_numpy(pow2).to(dev)
    for c0 in range(0, n, chunk):
        cn = min(chunk, n - c0)
        h = torch.arange(lo + c0, lo + c0 + cn, dtype=torch.int64, device=dev)
        h = h * _C1 + (seed * 1_000_003 + 12345)
        h = h ^ ((h >> 31) & _L[31])
        h = h * _C2
        h = h ^ ((h >> 27) & _L[27])
        h = h * _C3
        h = h ^ ((h >> 32) & _L[32])
        m = ((h >> 8) & 0xFFFF).to(torch.float32)
        p = pow2[(h >> 24) & (n_exp - 1)]
        sgn = 1.0 - 2.0 * ((h >> 40) & 1).to(torch.float32)
        del h
        u = (m * 2.0 + 1.0) * (2.0 ** -17)
        v = (u * p * sgn) * float(scale)
        out[c0:c0 + cn] = v.to(dtype)
    return out
