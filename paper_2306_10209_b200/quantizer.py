"""Blockwise symmetric INT8/INT4 codec on B200 -- drop-in for zs/quantizer.py.

Same names, argument meaning and exceptions as the reference
(``QuantConfig`` zs/quantizer.py:28-59, ``FlatTensor`` :62-83,
``QuantizedTensor`` :86-169, ``quantize`` :204-228, ``dequantize`` :231-238,
``fused_dequant_reduce_quant`` :241-258).  Values live on the GPU as torch
tensors; the arithmetic runs in libzpp.so (K0/K2/K4 in csrc/zpp_kernels.cuh).

Differences a caller can see, all deliberate:

* ``QuantizedTensor`` stores per-block ``absmax`` (fp32 when the input was
  fp16/bf16/fp32 -- exact -- or f64) instead of f64 scales; ``.scales`` returns
  the reference's f64 ``absmax / qmax`` bit-exactly.
* ``dequantize`` takes an optional output ``dtype`` (default float64, the
  reference's); every output element is the correctly rounded f64 value.
* ``FlatTensor`` keeps the caller's dtype instead of converting to f64 (fp16,
  bf16 and fp32 are exactly representable in f64, so codes are identical).
  Host (numpy) inputs are checked for finiteness at construction like the
  reference; device tensors are checked by the kernels (the device error word
  is raised as ``ValidationError`` when the op synchronises).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, IntegrityError, ValidationError

SCALE_WIRE_BYTES = 2  # zs/quantizer.py:24 -- accounted width of one wire scale
_HEADER = struct.Struct("<QBI")  # zs/quantizer.py:25

_DT = {torch.float32: _lib.F32, torch.float16: _lib.F16, torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise ValidationError(f"unsupported dtype {dt}; use float16, bfloat16, float32 or float64") from None


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2306_10209_b200 ops need a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass(frozen=True)
class QuantConfig:
    """Codec parameters (zs/quantizer.py:28-59).

    bit_width: 4 or 8.  block_size: elements per scale, a positive multiple of
    8.  mode: "blocked" or "full_tensor".  rounding: only "ties-to-even".
    """

    bit_width: int
    block_size: int = 2048
    mode: str = "blocked"
    rounding: str = "ties-to-even"

    def __post_init__(self):
        if self.bit_width not in (4, 8):
            raise ConfigError(f"bit_width must be 4 or 8, got {self.bit_width}")
        if self.block_size < 8 or self.block_size % 8 != 0:
            raise ConfigError(f"block_size must be a positive multiple of 8, got {self.block_size}")
        if self.mode not in ("blocked", "full_tensor"):
            raise ConfigError(f"unknown mode {self.mode!r}")
        if self.rounding != "ties-to-even":
            raise ConfigError(f"unsupported rounding {self.rounding!r}")

    @property
    def qmax(self) -> int:
        return (1 << (self.bit_width - 1)) - 1


class FlatTensor:
    """A 1-D tensor of real values plus its wire element width (zs/quantizer.py:62-83)."""

    def __init__(self, values, wire_element_bytes: int = 2):
        if isinstance(values, torch.Tensor):
            t = values
            if t.dim() != 1:
                raise ValidationError("FlatTensor expects a 1-D array")
            if t.dtype not in _DT:
                t = t.to(torch.float64)
            if not t.is_cuda and not bool(torch.isfinite(t).all()):
                raise ValidationError("FlatTensor values must be finite")
        else:
            arr = np.asarray(values, dtype=np.float64)
            if arr.ndim != 1:
                raise ValidationError("FlatTensor expects a 1-D array")
            if not np.all(np.isfinite(arr)):
                raise ValidationError("FlatTensor values must be finite")
            t = torch.from_numpy(np.ascontiguousarray(arr))
        if wire_element_bytes not in (2, 4):
            raise ValidationError("wire_element_bytes must be 2 or 4")
        self.values = t
        self.wire_element_bytes = wire_element_bytes

    def __len__(self) -> int:
        return int(self.values.numel())

    @property
    def wire_bytes(self) -> int:
        return len(self) * self.wire_element_bytes

    def cuda_values(self) -> torch.Tensor:
        v = self.values
        if not v.is_cuda:
            v = v.to(device(), non_blocking=False)
        return v.contiguous()


def as_flat(t) -> FlatTensor:
    return t if isinstance(t, FlatTensor) else FlatTensor(t)


@dataclass
class QuantizedTensor:
    """Packed codes plus per-block absmax for one quantized tensor (zs/quantizer.py:86-169).

    codes: uint8 device tensor, ``n_blocks * block_size * bit_width / 8`` bytes
    (block padding included).  absmax: float32 or float64 device tensor.
    """

    codes: torch.Tensor
    absmax: torch.Tensor
    original_len: int
    config: QuantConfig

    @property
    def n_blocks(self) -> int:
        return int(self.absmax.numel())

    @property
    def padded_len(self) -> int:
        return self.n_blocks * self.config.block_size

    @property
    def payload_bytes(self) -> int:
        return math.ceil(self.original_len * self.config.bit_width / 8)

    @property
    def metadata_bytes(self) -> int:
        return self.n_blocks * SCALE_WIRE_BYTES

    @property
    def padding_bytes(self) -> int:
        return self.padded_len * self.config.bit_width // 8 - self.payload_bytes

    @property
    def wire_bytes(self) -> int:
        return self.payload_bytes + self.metadata_bytes

    @property
    def absmax_code(self) -> int:
        return _lib.F64 if self.absmax.dtype == torch.float64 else _lib.F32

    @property
    def scales(self) -> torch.Tensor:
        """f64 per-block scales ``absmax / qmax``, bit-identical to the reference's."""
        out = torch.empty(self.n_blocks, dtype=torch.float64, device=self.absmax.device)
        if self.n_blocks:
            _lib.check(_lib.load().zpp_scales(self.absmax.data_ptr(), self.absmax_code, self.n_blocks,
                                              self.config.bit_width, out.data_ptr(), stream_ptr()), "scales")
        return out

    def to_wire(self) -> torch.Tensor:
        """Canonical wire layout (zs/quantizer.py:121-131) built on the device:
        a uint8 device tensor [header | fp16 scales | codes] (zpp_wire_pack)."""
        n_bytes = _HEADER.size + self.n_blocks * SCALE_WIRE_BYTES + int(self.codes.numel())
        out = torch.empty(n_bytes, dtype=torch.uint8, device=self.codes.device)
        _lib.check(_lib.load().zpp_wire_pack(self.codes.data_ptr(), self.absmax.data_ptr(), self.absmax_code,
                                             self.original_len, self.config.bit_width, self.config.block_size,
                                             out.data_ptr(), stream_ptr()), "to_bytes")
        return out

    def to_bytes(self) -> bytes:
        """Canonical wire layout (zs/quantizer.py:121-131): header, fp16 scales,
        codes -- packed on the device, one device-to-host copy."""
        return self.to_wire().cpu().numpy().tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes) -> "QuantizedTensor":
        """Parse the canonical wire layout (zs/quantizer.py:133-149).

        Wire scales are fp16; the tensor keeps them exactly as an f64 absmax of
        ``scale16 * qmax`` (exact in f64), from which every kernel recovers
        ``scale16`` bit-exactly (``RN64(scale16*qmax/qmax) == scale16``)."""
        original_len, cfg, n_blocks, scale_end = from_bytes_header(raw)
        dev = device()
        wire = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)  # one host-to-device copy
        codes = torch.empty(len(raw) - scale_end, dtype=torch.uint8, device=dev)
        absmax = torch.empty(n_blocks, dtype=torch.float64, device=dev)
        _lib.check(_lib.load().zpp_wire_unpack(wire.data_ptr(), original_len, cfg.bit_width, cfg.block_size,
                                               codes.data_ptr(), absmax.data_ptr(), stream_ptr()), "from_bytes")
        return cls(codes=codes, absmax=absmax, original_len=original_len, config=cfg)

    def slice_blocks(self, start: int, length: int) -> "QuantizedTensor":
        """Elements [start, start+length) as a zero-copy view (zs/quantizer.py:151-169)."""
        bs = self.config.block_size
        if start % bs or length % bs or start + length > self.original_len:
            raise ValidationError("slice_blocks requires block-aligned bounds")
        if self.original_len != self.padded_len:
            raise ValidationError("slice_blocks requires a block-aligned tensor")
        bpb = bs * self.config.bit_width // 8
        b0, nb = start // bs, length // bs
        return QuantizedTensor(codes=self.codes[b0 * bpb:(b0 + nb) * bpb], absmax=self.absmax[b0:b0 + nb],
                               original_len=length, config=self.config)


@dataclass
class QuantErrorStats:
    rmse: float
    max_abs_error: float
    per_block_bound_violations: int


def effective_block(cfg: QuantConfig, n: int) -> int:
    """zs/quantizer.py:179-182."""
    if cfg.mode == "full_tensor":
        return max(8, -(-n // 8) * 8)
    return cfg.block_size


def check_flag(flag: torch.Tensor, what: str):
    """Synchronise on the device error word and raise the reference's exception."""
    _lib.raise_for_flags(int(flag.item()), what)


def new_flag() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device())


def alloc_quantized(n: int, cfg: QuantConfig, absmax_dtype=torch.float32) -> QuantizedTensor:
    b = effective_block(cfg, n)
    nb = -(-n // b) if n else 0
    out_cfg = replace(cfg, block_size=b) if b != cfg.block_size else cfg
    codes = torch.empty(nb * b * cfg.bit_width // 8, dtype=torch.uint8, device=device())
    absmax = torch.empty(nb, dtype=absmax_dtype, device=device())
    return QuantizedTensor(codes=codes, absmax=absmax, original_len=n, config=out_cfg)


def quantize(t, cfg: QuantConfig, *, flag: torch.Tensor | None = None) -> QuantizedTensor:
    """K0 (zs/quantizer.py:204-228).  Bit-exact codes and scales.

    With ``flag=None`` the call synchronises and raises ``ValidationError`` on
    non-finite input like the reference; passing a device flag defers that check.
    """
    x = as_flat(t).cuda_values()
    n = int(x.numel())
    q = alloc_quantized(n, cfg, torch.float64 if x.dtype == torch.float64 else torch.float32)
    if n == 0:
        return q
    own = flag is None
    f = new_flag() if own else flag
    _lib.check(_lib.load().zpp_quantize(x.data_ptr(), dtype_code(x.dtype), n, q.config.bit_width,
                                        q.config.block_size, q.codes.data_ptr(), q.absmax.data_ptr(),
                                        f.data_ptr(), stream_ptr()), "quantize")
    if own:
        check_flag(f, "quantize")
    return q


def dequantize(q: QuantizedTensor, dtype: torch.dtype = torch.float64, *, out: torch.Tensor | None = None,
               flag: torch.Tensor | None = None) -> FlatTensor:
    """K4 (zs/quantizer.py:231-238): ``code * scale`` per element, padding dropped.

    Raises ``IntegrityError`` on an out-of-range code (-128 / -8).
    """
    n = q.original_len
    if out is None:
        out = torch.empty(n, dtype=dtype, device=q.codes.device if q.codes.is_cuda else device())
    if n:
        own = flag is None
        f = new_flag() if own else flag
        _lib.check(_lib.load().zpp_dequantize(q.codes.data_ptr(), q.absmax.data_ptr(), q.absmax_code, n,
                                              q.config.bit_width, q.config.block_size, out.data_ptr(),
                                              dtype_code(out.dtype), f.data_ptr(), stream_ptr()), "dequantize")
        if own:
            check_flag(f, "dequantize")
    ft = FlatTensor.__new__(FlatTensor)
    ft.values, ft.wire_element_bytes = out, 2
    return ft


def fused_dequant_reduce_quant(inputs, out_cfg: QuantConfig, *, flag: torch.Tensor | None = None) -> QuantizedTensor:
    """K2 (zs/quantizer.py:241-258): dequantize each input, fold left to right in
    f64 from +0.0, requantize -- bit-identical to the unfused composition.
    The result's absmax is f64 (exact), so its scales equal the reference's."""
    inputs = list(inputs)
    if not inputs:
        raise ValidationError("fused reduce needs at least one input")
    first = inputs[0]
    for q in inputs[1:]:
        if q.original_len != first.original_len or q.config != first.config:
            raise ValidationError("fused reduce inputs must share length and config")
    if len({q.absmax.dtype for q in inputs}) != 1:
        raise ValidationError("fused reduce inputs must share the absmax dtype")
    n = first.original_len
    out = alloc_quantized(n, out_cfg, torch.float64)
    if n == 0:
        return out
    lib = _lib.load()
    own = flag is None
    f = new_flag() if own else flag
    cp, _k1 = _lib.ptr_array([q.codes.data_ptr() for q in inputs])
    ap, _k2 = _lib.ptr_array([q.absmax.data_ptr() for q in inputs])
    ws_bytes = lib.zpp_drq_workspace_bytes(n, out.config.block_size)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device())
    _lib.check(lib.zpp_dequant_reduce_quant(cp, ap, first.absmax_code, len(inputs), n, first.config.bit_width,
                                            first.config.block_size, out.config.bit_width, out.config.block_size,
                                            out.codes.data_ptr(), out.absmax.data_ptr(), ws.data_ptr(), ws_bytes,
                                            f.data_ptr(), stream_ptr()), "fused_dequant_reduce_quant")
    if own:
        check_flag(f, "fused_dequant_reduce_quant")
    return out


def dequant_reduce(inputs, dtype: torch.dtype = torch.float64, *, post_scale: float = 1.0,
                   out: torch.Tensor | None = None, flag: torch.Tensor | None = None) -> torch.Tensor:
    """K3 (BlockCodec.reduce_final, zs/collectives.py:71-75): f64 fold of the
    decoded inputs in the given (ascending-source) order, from +0.0."""
    inputs = list(inputs)
    if not inputs:
        raise ValidationError("reduce needs at least one input")
    first = inputs[0]
    for q in inputs[1:]:
        if q.original_len != first.original_len or q.config != first.config or q.absmax.dtype != first.absmax.dtype:
            raise ValidationError("reduce inputs must share length, config and absmax dtype")
    n = first.original_len
    if out is None:
        out = torch.empty(n, dtype=dtype, device=device())
    if n:
        own = flag is None
        f = new_flag() if own else flag
        cp, _k1 = _lib.ptr_array([q.codes.data_ptr() for q in inputs])
        ap, _k2 = _lib.ptr_array([q.absmax.data_ptr() for q in inputs])
        _lib.check(_lib.load().zpp_dequant_reduce(cp, ap, first.absmax_code, len(inputs), n, first.config.bit_width,
                                                  first.config.block_size, out.data_ptr(), dtype_code(out.dtype),
                                                  float(post_scale), f.data_ptr(), stream_ptr()), "dequant_reduce")
        if own:
            check_flag(f, "dequant_reduce")
    return out


def quant_error_stats(t, cfg: QuantConfig) -> QuantErrorStats:
    """Round-trip error summary (zs/quantizer.py:261-272); a test aid, not hot path."""
    ft = as_flat(t)
    x = ft.cuda_values().to(torch.float64)
    q = quantize(ft, cfg)
    back = dequantize(q).values
    err = (back - x).abs()
    n = x.numel()
    if n == 0:
        return QuantErrorStats(0.0, 0.0, 0)
    bound = torch.repeat_interleave(q.scales, q.config.block_size)[:n] / 2.0
    return QuantErrorStats(rmse=float(torch.sqrt((err * err).mean())), max_abs_error=float(err.max()),
                           per_block_bound_violations=int((err > bound).sum()))


def from_bytes_header(raw: bytes):
    """Parse and validate the wire header (zs/quantizer.py:133-146); returns
    (original_len, QuantConfig, n_blocks, scale_end)."""
    if len(raw) < _HEADER.size:
        raise IntegrityError("payload shorter than header")
    original_len, bit_width, block_size = _HEADER.unpack_from(raw)
    try:
        cfg = QuantConfig(bit_width=bit_width, block_size=block_size)
    except ConfigError as e:
        raise IntegrityError(f"header describes invalid config: {e}") from e
    n_blocks = math.ceil(original_len / block_size) if original_len else 0
    scale_end = _HEADER.size + n_blocks * SCALE_WIRE_BYTES
    if len(raw) != scale_end + n_blocks * block_size * bit_width // 8:
        raise IntegrityError("payload length does not match header")
    return original_len, cfg, n_blocks, scale_end
