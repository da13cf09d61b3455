"""Loading helpers for the committed golden vectors (tests/golden/*.npz),
produced by the real reference with tests/golden/make_golden.py."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name: str):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    return z, meta


@functools.lru_cache(maxsize=None)
def volumes():
    with open(os.path.join(GOLDEN, "volumes.json")) as f:
        return json.load(f)


def bf16_bits_to_f64(b) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def as_f64(arr, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return bf16_bits_to_f64(arr)
    return np.asarray(arr).astype(np.float64)


def to_torch(arr, dtype: str, device="cuda"):
    """Golden input array -> torch tensor of the dtype the GPU path consumes."""
    import torch

    if dtype == "bf16":
        t = torch.from_numpy(np.asarray(arr, dtype=np.uint16).astype(np.int16)).view(torch.bfloat16)
    elif dtype == "fp16":
        t = torch.from_numpy(np.asarray(arr, dtype=np.float16))
    elif dtype == "fp32":
        t = torch.from_numpy(np.asarray(arr, dtype=np.float32))
    else:
        t = torch.from_numpy(np.asarray(arr, dtype=np.float64))
    return t.to(device)


def f64_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Correctly rounded f64 -> bf16 (as float64 values), ties to even."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    q = np.ldexp(1.0, np.maximum(e - 8, -133))
    with np.errstate(over="ignore", invalid="ignore"):  # sign(0) * inf; zeros are restored below
        r = np.rint(x / q) * q
        r = np.where(np.abs(r) > 3.3895313892515355e38, np.sign(x) * np.inf, r)
    return np.where(x == 0, x, r)


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """The reference's f64 values rounded once to the GPU output dtype."""
    if dtype == "f64":
        return np.asarray(x, dtype=np.float64)
    if dtype == "fp32":
        return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
    if dtype == "fp16":
        with np.errstate(over="ignore"):
            return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)
    return f64_to_bf16_rne(x)
