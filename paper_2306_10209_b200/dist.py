"""ZeRO++ collectives across GPUs: one process per GPU, NVLink P2P.

The single-process functions in ``collectives.py`` keep the reference's
whole-cluster signatures (zs/collectives.py).  This module is the same three
collectives run for real, one rank per GPU, on a symmetric device workspace
that every rank maps through CUDA IPC:

* ``Communicator.qwz_allgather``  qwZ (zs/collectives.py:244-282): K0 quantizes
  this rank's shard into its symmetric buffer, a device barrier, then ONE
  kernel pulls every rank's INT8 codes over NVLink and dequantizes them into
  the local fp16 output.  Optional hpZ write-through keeps this rank's
  secondary partition (zs/engine.py:364-367) in HBM.
* ``Communicator.hpz_allgather``  hpZ (zs/collectives.py:202-241, groups):
  group barrier, then a copy kernel pulls the group members' secondary shards.
* ``Communicator.qgz_reduce_scatter``  qgZ (zs/collectives.py:464-569): per
  stage K1 (reorder + quantize) -> group barrier -> K2 pulls the X intra-group
  messages over NVLink and requantizes -> cross barrier -> K3 pulls the Y
  hop-2 segments and folds them in f64.  With one group, K2 writes the final
  partition itself (hop 2 is a self-send).

``torch.distributed`` is plumbing only: it exchanges the 64-byte IPC handles
once and provides the NCCL comparators (``nccl_allgather`` /
``nccl_reduce_scatter``: the fp16/bf16 ZeRO-3 baseline collectives).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .errors import DeviceError, ValidationError
from .partitioner import PartitionSpec
from .quantizer import QuantConfig, device, dtype_code, stream_ptr

ALIGN = 256


def _align(x: int) -> int:
    return (x + ALIGN - 1) // ALIGN * ALIGN


def members(rank: int, world: int, group_size: int, scope: str) -> list[int]:
    """Ranks taking part in a barrier scope -- mirrors zpp_comm::members in
    csrc/zpp_comm.cu.  world: all ranks; group: consecutive ranks of this
    rank's group (zs/partitioner.py:67-73); cross: the ranks with this rank's
    local index in every group (qgZ hop 2)."""
    node, loc = divmod(rank, group_size)
    if scope == "world":
        return list(range(world))
    if scope == "group":
        return [node * group_size + j for j in range(group_size)]
    if scope == "cross":
        return [c * group_size + loc for c in range(world // group_size)]
    raise ValidationError(f"unknown scope {scope!r}")


@dataclass(frozen=True)
class SymLayout:
    """Byte offsets of each collective's region in the symmetric workspace."""

    qwz: int
    hpz: int
    qgz: int
    total: int

    @staticmethod
    def plan(qwz_bytes: int, hpz_bytes: int, qgz_bytes: int) -> "SymLayout":
        qwz = 0
        hpz = _align(qwz + qwz_bytes)
        qgz = _align(hpz + hpz_bytes)
        return SymLayout(qwz=qwz, hpz=hpz, qgz=qgz, total=_align(qgz + qgz_bytes))


def _check_buf(t: torch.Tensor, name: str, min_numel: int):
    """The C ABI takes raw pointers: insist on dense CUDA tensors of sufficient size."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValidationError(f"{name} must be a contiguous CUDA tensor")
    if t.numel() < min_numel:
        raise ValidationError(f"{name} has {t.numel()} elements, needs {min_numel}")


def exchange_handles(handle: bytes, group=None) -> bytes:
    """All-gather one fixed-size blob per rank (rank order) over torch.distributed."""
    if not (dist.is_available() and dist.is_initialized()):
        return handle
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return b"".join(out)


class Communicator:
    """NVLink peer-memory communicator for the fused ZeRO++ collectives.

    Sizes are fixed at construction (the symmetric workspace is allocated once):
    ``qwz_shard`` elements per rank for qwZ, ``hpz_sec`` secondary elements per
    rank (0 = hpZ off), ``qgz_elems`` gradient elements per call for qgZ.
    ``group_size`` is the reference's gpus_per_node (zs/topology.py:31-52); on
    one 8xB200 box the default 2 groups x 4 GPUs stand in for 2 nodes.
    """

    def __init__(self, *, group_size: int | None = None, qwz_shard: int = 0,
                 qwz_cfg: QuantConfig = QuantConfig(bit_width=8, block_size=2048), hpz_sec: int = 0,
                 hpz_dtype: torch.dtype = torch.float16, hpz_layers: int = 1, qgz_elems: int = 0, qgz_stages: int = 1,
                 qgz_cfg: QuantConfig = QuantConfig(bit_width=4, block_size=512),
                 qgz_intra_cfg: QuantConfig | None = None):
        self.lib = _lib.load()
        initialized = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank() if initialized else 0
        self.world = dist.get_world_size() if initialized else 1
        if group_size is None:
            group_size = min(self.world, 4) if self.world % min(self.world, 4) == 0 else self.world
        if self.world % group_size:
            raise ValidationError(f"group_size {group_size} must divide world {self.world}")
        self.group_size = group_size
        self.qwz_shard, self.qwz_cfg = qwz_shard, qwz_cfg
        self.hpz_sec, self.hpz_dtype = hpz_sec, hpz_dtype
        if hpz_layers < 1:
            raise ValidationError("hpz_layers must be >= 1")
        self.hpz_layers = hpz_layers
        self.qgz_elems, self.qgz_stages = qgz_elems, qgz_stages
        self.qgz_cfg = qgz_cfg
        self.qgz_intra_cfg = qgz_intra_cfg or qgz_cfg
        hpz_esz = torch.tensor([], dtype=hpz_dtype).element_size()
        # one secondary slot per layer (the backward gathers of a whole stack
        # read the secondaries the forward wrote, zs/engine.py:364-370)
        self._hpz_slot = self.lib.zpp_hpz_sym_bytes(hpz_sec, hpz_esz) if hpz_sec else 0
        self.layout = SymLayout.plan(
            self.lib.zpp_qwz_sym_bytes(qwz_shard, qwz_cfg.bit_width, qwz_cfg.block_size, self.world) if qwz_shard else 0,
            self._hpz_slot * hpz_layers,
            self.lib.zpp_qgz_sym_bytes(qgz_elems, self.world, qgz_stages, self.qgz_intra_cfg.bit_width,
                                       self.qgz_intra_cfg.block_size, qgz_cfg.bit_width, qgz_cfg.block_size)
            if qgz_elems else 0)
        device()  # fail loudly without a GPU
        h = ctypes.c_void_p()
        _lib.check(self.lib.zpp_comm_create(self.rank, self.world, group_size, max(self.layout.total, ALIGN),
                                            ctypes.byref(h)), "zpp_comm_create")
        self.handle = h
        mine = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        _lib.check(self.lib.zpp_comm_ipc_handle(h, mine), "zpp_comm_ipc_handle")
        allh = exchange_handles(mine.raw)
        buf = ctypes.create_string_buffer(allh, len(allh))
        rc = self.lib.zpp_comm_open_peers(h, buf)
        if rc != _lib.OK:
            err = _lib.last_error()
            self.lib.zpp_comm_destroy(h)
            self.handle = None
            raise DeviceError(
                f"zpp_comm_open_peers: {err}. The fused collectives need every peer's symmetric buffer mapped "
                "through CUDA IPC (cudaIpcOpenMemHandle), i.e. all ranks on one node with peer access between "
                "their GPUs (NVLink/NVSwitch) and no container or driver policy blocking IPC. Use the NCCL "
                "comparators (nccl_allgather / nccl_reduce_scatter) where that is not available.")
        self.flag = torch.zeros(1, dtype=torch.int32, device=device())
        self._broken = False
        if hpz_sec:
            base = self.lib.zpp_comm_sym_ptr(h, self.rank) + self.layout.hpz
            self._secondaries = [_wrap_device(base + i * self._hpz_slot, hpz_sec, hpz_dtype)
                                 for i in range(hpz_layers)]
            self._secondary = self._secondaries[0]
        else:
            self._secondaries = []
            self._secondary = None
        if initialized:
            dist.barrier()

    # -- collectives ---------------------------------------------------------

    def qwz_allgather(self, shard: torch.Tensor, out: torch.Tensor | None = None,
                      out_dtype: torch.dtype = torch.float16, write_secondary: bool = False,
                      out_stride: int = 0, next_shard: torch.Tensor | None = None, layer: int = 0) -> torch.Tensor:
        """qwZ: every rank ends with the concatenation (rank order) of every
        rank's dequantize(quantize(shard)) -- zs/collectives.py:244-282.

        ``out_stride`` (elements between consecutive ranks' segments, default
        the shard length) lets a caller gather piece k of every shard in place.
        ``next_shard`` (cross-layer prefetch): the next
        layer's shard is quantized on a side stream beside this gather; pass it
        as ``shard`` to the next call and leave it unchanged until then.
        ``layer`` selects the hpZ secondary slot the write-through fills."""
        self._usable()
        n = int(shard.numel())
        if n > self.qwz_shard:
            raise ValidationError(f"shard has {n} elements, communicator was sized for {self.qwz_shard}")
        stride = out_stride or n
        if stride < n:
            raise ValidationError(f"out_stride {stride} is smaller than the shard ({n})")
        _check_buf(shard, "shard", n)
        if out is None:
            out = torch.empty(stride * (self.world - 1) + n, dtype=out_dtype, device=shard.device)
        _check_buf(out, "out", stride * (self.world - 1) + n)
        sec_ptr, sec_lo, sec_len = None, 0, 0
        if write_secondary:
            if self._secondary is None:
                raise ValidationError("communicator has no hpZ secondary region")
            if out.dtype != self.hpz_dtype or stride != n:
                raise ValidationError("secondary write-through needs an unstrided gather of the hpZ dtype")
            spec = PartitionSpec(total_elems=n * self.world, world=self.world, group_size=self.group_size)
            sec_lo, sec_hi = spec.secondary_range(self.rank)
            if sec_hi - sec_lo != self.hpz_sec:
                raise ValidationError("secondary shard length does not match the communicator's hpz_sec")
            sec_len = sec_hi - sec_lo
            sec_ptr = self.secondary_of(layer).data_ptr()
        nxt, nlen = None, 0
        if next_shard is not None:
            nlen = int(next_shard.numel())
            if nlen > self.qwz_shard or next_shard.dtype != shard.dtype:
                raise ValidationError("next_shard must fit the communicator and match the shard's dtype")
            _check_buf(next_shard, "next_shard", nlen)
            nxt = next_shard.data_ptr()
        _lib.check(self.lib.zpp_qwz_allgather_next(self.handle, self.layout.qwz, shard.data_ptr(),
                                                   dtype_code(shard.dtype), n, self.qwz_cfg.bit_width,
                                                   self.qwz_cfg.block_size, out.data_ptr(), dtype_code(out.dtype),
                                                   stride, sec_ptr, sec_lo, sec_len, nxt, nlen, self.flag.data_ptr(),
                                                   stream_ptr()), "qwz_allgather")
        return out

    def qwz_allgather_layers(self, shards, outs=None, write_secondary: bool = False, prefetch: bool = True):
        """qwZ of a layer sequence (the forward pass of a ZeRO++ step,
        zs/engine.py:345-360): layer i is gathered while layer i+1 is
        quantized on the side stream (``prefetch``), and with
        ``write_secondary`` layer i's hpZ secondary goes to slot i."""
        outs = outs if outs is not None else [None] * len(shards)
        res = []
        for i, sh in enumerate(shards):
            nxt = shards[i + 1] if prefetch and i + 1 < len(shards) else None
            res.append(self.qwz_allgather(sh, out=outs[i], write_secondary=write_secondary, next_shard=nxt,
                                          layer=i if write_secondary else 0))
        return res

    def qwz_allgather_host(self, h_shard: torch.Tensor, h_out: torch.Tensor, chunks: int = 8,
                           d_shard: torch.Tensor | None = None, d_out: torch.Tensor | None = None):
        """qwZ between HOST buffers with transfer/compute overlap.

        The shard is split into ``chunks`` block-aligned pieces; piece k is one
        fused sub-collective (quantize piece k of every rank's shard, gather it
        in place), so H2D of piece k+1, the collective on piece k and D2H of
        piece k-1 run concurrently on three streams.  h_shard / h_out should be
        pinned.  Same values as ``qwz_allgather`` (blocks never straddle pieces)."""
        n = int(h_shard.numel())
        blk = self.qwz_cfg.block_size
        per = -(-(-(-n // chunks)) // blk) * blk
        if d_shard is None:
            d_shard = torch.empty(n, dtype=h_shard.dtype, device=device())
        if d_out is None:
            d_out = torch.empty(n * self.world, dtype=h_out.dtype, device=device())
        if not hasattr(self, "_h2d"):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
        main = torch.cuda.current_stream()
        self._h2d.wait_stream(main)
        self._d2h.wait_stream(main)
        pieces = [(k, min(per, n - k)) for k in range(0, n, per)]
        for k, cl in pieces:
            with torch.cuda.stream(self._h2d):
                d_shard[k:k + cl].copy_(h_shard[k:k + cl], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
            main.wait_event(ev)
            self.qwz_allgather(d_shard[k:k + cl], out=d_out[k:], out_stride=n)
            done = torch.cuda.Event()
            done.record(main)
            with torch.cuda.stream(self._d2h):
                self._d2h.wait_event(done)
                for r in range(self.world):
                    h_out[r * n + k:r * n + k + cl].copy_(d_out[r * n + k:r * n + k + cl], non_blocking=True)
        main.wait_stream(self._d2h)
        return h_out

    @property
    def secondary(self) -> torch.Tensor:
        """This rank's hpZ secondary partition, held in the symmetric workspace."""
        if self._secondary is None:
            raise ValidationError("communicator has no hpZ secondary region")
        return self._secondary

    def secondary_of(self, layer: int) -> torch.Tensor:
        """This rank's hpZ secondary partition of `layer` (slot in the symmetric workspace)."""
        if not self._secondaries:
            raise ValidationError("communicator has no hpZ secondary region")
        if not 0 <= layer < self.hpz_layers:
            raise ValidationError(f"layer {layer} outside the communicator's {self.hpz_layers} hpZ slots")
        return self._secondaries[layer]

    def hpz_allgather(self, out: torch.Tensor | None = None, layer: int = 0) -> torch.Tensor:
        """hpZ: gather the group's secondary shards (member order) over NVLink."""
        self._usable()
        if self._secondary is None:
            raise ValidationError("communicator has no hpZ secondary region")
        if not 0 <= layer < self.hpz_layers:
            raise ValidationError(f"layer {layer} outside the communicator's {self.hpz_layers} hpZ slots")
        if out is None:
            out = torch.empty(self.hpz_sec * self.group_size, dtype=self.hpz_dtype, device=device())
        _check_buf(out, "out", self.hpz_sec * self.group_size)
        if out.element_size() != self._secondary.element_size():
            raise ValidationError("hpZ output dtype must match the secondary shard's element size")
        _lib.check(self.lib.zpp_hpz_allgather(self.handle, self.layout.hpz + layer * self._hpz_slot, self.hpz_sec,
                                              self._secondary.element_size(), out.data_ptr(), self.flag.data_ptr(),
                                              stream_ptr()), "hpz_allgather")
        return out

    def qgz_reduce_scatter(self, grad: torch.Tensor, out: torch.Tensor | None = None,
                           out_dtype: torch.dtype = torch.float32, reorder: bool = True) -> torch.Tensor:
        """qgZ: this rank's partition (n/W elements) of the SUM over ranks,
        through two codec passes -- zs/collectives.py:464-569."""
        self._usable()
        n = int(grad.numel())
        if n != self.qgz_elems:
            raise ValidationError(f"gradient has {n} elements, communicator was sized for {self.qgz_elems}")
        return self._qgz(grad, n, out, out_dtype, reorder)

    def _qgz(self, grad, n, out, out_dtype, reorder):
        _check_buf(grad, "grad", n)
        if out is None:
            out = torch.empty(n // self.world, dtype=out_dtype, device=grad.device)
        _check_buf(out, "out", n // self.world)
        _lib.check(self.lib.zpp_qgz_reduce_scatter(self.handle, self.layout.qgz, grad.data_ptr(),
                                                   dtype_code(grad.dtype), n, self.qgz_stages, int(reorder),
                                                   self.qgz_intra_cfg.bit_width, self.qgz_intra_cfg.block_size,
                                                   self.qgz_cfg.bit_width, self.qgz_cfg.block_size, out.data_ptr(),
                                                   dtype_code(out.dtype), self.flag.data_ptr(), stream_ptr()),
                   "qgz_reduce_scatter")
        return out

    def stream_layout(self, n_total: int) -> tuple[int, int, int, int]:
        """(full buckets, tail elements, padded tail, output elements per rank)
        of a gradient stream of n_total elements cut into buckets of
        ``qgz_elems``; the tail is zero-padded to a multiple of
        W * S * max(intra block, inter block) (zs/engine.py:465-466)."""
        bucket = self.qgz_elems
        full, tail = divmod(n_total, bucket)
        align = self.world * self.qgz_stages * max(self.qgz_cfg.block_size, self.qgz_intra_cfg.block_size)
        tail_pad = -(-tail // align) * align
        return full, tail, tail_pad, (full * bucket + tail_pad) // self.world

    def qgz_reduce_scatter_stream(self, grads: torch.Tensor, out: torch.Tensor | None = None,
                                  out_dtype: torch.dtype = torch.float32, reorder: bool = True) -> torch.Tensor:
        """qgZ over a flat gradient stream in buckets of ``qgz_elems`` (the
        way ZeRO++ reduces a model's gradients, BASELINE configs[3]): bucket b
        is one qgz_2hop call (zs/collectives.py:464-569) and this rank's
        output is the concatenation of its partitions of every bucket.  The
        tail bucket is zero-padded as zs/engine.py:465-466 pads the whole
        tensor (one device copy into a staging buffer kept by the
        communicator).  The full buckets are one zpp_qgz_reduce_scatter_buckets
        call (same results as separate calls); with one group (hop 2 a
        self-send) K1 of bucket b+1 runs on the communicator's side stream
        beside the pulling K2 of bucket b, otherwise buckets run back to back
        (the measured better choice for each layout)."""
        self._usable()
        n_total = int(grads.numel())
        full, tail, tail_pad, n_out = self.stream_layout(n_total)
        _check_buf(grads, "grads", n_total)
        if out is None:
            out = torch.empty(n_out, dtype=out_dtype, device=grads.device)
        _check_buf(out, "out", n_out)
        bucket, w = self.qgz_elems, self.world
        if full:
            _lib.check(self.lib.zpp_qgz_reduce_scatter_buckets(
                self.handle, self.layout.qgz, grads.data_ptr(), dtype_code(grads.dtype), bucket, full,
                self.qgz_stages, int(reorder), self.qgz_intra_cfg.bit_width, self.qgz_intra_cfg.block_size,
                self.qgz_cfg.bit_width, self.qgz_cfg.block_size, out.data_ptr(), dtype_code(out.dtype),
                self.flag.data_ptr(), stream_ptr()), "qgz_reduce_scatter_stream")
        if tail:
            if getattr(self, "_tail_buf", None) is None or self._tail_buf.numel() != tail_pad \
                    or self._tail_buf.dtype != grads.dtype:
                self._tail_buf = torch.zeros(tail_pad, dtype=grads.dtype, device=grads.device)
            self._tail_buf[:tail].copy_(grads[full * bucket:])
            self._qgz(self._tail_buf, tail_pad, out[full * bucket // w:], out.dtype, reorder)
        return out

    TRACE_STAGES = ("begin", "quantize", "barrier", "gather", "K1", "K2", "K3")

    def trace(self, enable: bool = True) -> None:
        """Record timing events between the launches of each qwZ / qgZ call
        (diagnostics; read them with trace_read)."""
        _lib.check(self.lib.zpp_comm_trace(self.handle, 1 if enable else 0), "zpp_comm_trace")

    def trace_read(self) -> list[tuple[str, float]]:
        """[(stage just finished, ms since the last traced call began)]; waits
        for that call to finish."""
        ids = (ctypes.c_int * 32)()
        ms = (ctypes.c_float * 32)()
        n = self.lib.zpp_comm_trace_read(self.handle, ids, ms, 32)
        if n < 0:
            _lib.check(-n, "zpp_comm_trace_read")
        return [(self.TRACE_STAGES[ids[i]], float(ms[i])) for i in range(n)]

    def barrier(self, scope: str = "world", timeout_ms: int = 60000):
        code = {"world": 0, "group": 1, "cross": 2}[scope]
        _lib.check(self.lib.zpp_comm_barrier(self.handle, code, timeout_ms, self.flag.data_ptr(), stream_ptr()),
                   "barrier")

    def _usable(self):
        if self._broken:
            raise DeviceError("communicator stopped after a device-barrier timeout; call recover() on every rank")

    def check(self):
        """Synchronise and raise the reference's exception for any device-side
        condition seen since the last check (non-finite input, bad code, timeout).

        The collectives are stream-ordered and host-asynchronous: their outputs
        are only valid once check() has returned without raising.  After a
        TIMEOUT (a peer never reached a device barrier) every later data kernel
        on this communicator returns without touching its buffers, and the
        communicator refuses new calls until recover() has run on every rank."""
        v = int(self.flag.item())
        if v:
            if v & _lib.FLAG_TIMEOUT:
                self._broken = True
                self.flag.fill_(_lib.FLAG_TIMEOUT)
            else:
                self.flag.zero_()
            _lib.raise_for_flags(v, "zpp collective")

    def recover(self):
        """Collective re-initialisation after a barrier timeout: every rank
        drains its device, passes a host barrier, restarts its barrier epochs
        and double-buffer phases (zpp_comm_reset), clears its error word and
        passes a second host barrier.  Then the communicator is usable again."""
        torch.cuda.synchronize()
        if dist.is_available() and dist.is_initialized():
            dist.barrier()
        _lib.check(self.lib.zpp_comm_reset(self.handle), "zpp_comm_reset")
        self.flag.zero_()
        torch.cuda.synchronize()
        if dist.is_available() and dist.is_initialized():
            dist.barrier()
        self._broken = False

    def close(self):
        if getattr(self, "handle", None) is not None:
            torch.cuda.synchronize()
            if dist.is_available() and dist.is_initialized():
                dist.barrier()
            self.lib.zpp_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        # Garbage collection is not collective: peers may still be pulling from
        # this rank's symmetric buffer, so a multi-rank communicator that was
        # never close()d is leaked (with a warning) instead of freed.
        try:
            if getattr(self, "handle", None) is None:
                return
            if self.world == 1:
                self.lib.zpp_comm_destroy(self.handle)
            else:
                import warnings

                warnings.warn("zpp Communicator garbage-collected without close(): its symmetric buffer is leaked "
                              "(freeing it could fault peers still reading it)", ResourceWarning, stacklevel=2)
            self.handle = None
        except Exception:
            pass


class _DevBuf:
    """Minimal __cuda_array_interface__ wrapper so torch can view raw device memory."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype):
        typestr = {torch.float16: "<f2", torch.bfloat16: "<f2", torch.float32: "<f4", torch.float64: "<f8",
                   torch.uint8: "|u1"}[dtype]
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def _wrap_device(ptr: int, n: int, dtype: torch.dtype) -> torch.Tensor:
    t = torch.as_tensor(_DevBuf(ptr, n, torch.float16 if dtype == torch.bfloat16 else dtype), device=device())
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


# ---------------------------------------------------------------------------
# NCCL comparators (the ZeRO-3 baseline collectives)


def nccl_allgather(shard: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """fp16 ZeRO-3 weight all-gather (the baseline qwZ replaces)."""
    w = dist.get_world_size(group)
    if out is None:
        out = torch.empty(shard.numel() * w, dtype=shard.dtype, device=shard.device)
    dist.all_gather_into_tensor(out, shard, group=group)
    return out


def nccl_reduce_scatter(grad: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """bf16 ZeRO-3 gradient reduce-scatter (the baseline qgZ replaces)."""
    w = dist.get_world_size(group)
    if out is None:
        out = torch.empty(grad.numel() // w, dtype=grad.dtype, device=grad.device)
    dist.reduce_scatter_tensor(out, grad, group=group)
    return out


def make_groups(group_size: int):
    """(my group, my cross group) as torch.distributed process groups; every
    rank must call this collectively."""
    world, rank = dist.get_world_size(), dist.get_rank()
    mine = cross = None
    for g in range(world // group_size):
        pg = dist.new_group(list(range(g * group_size, (g + 1) * group_size)))
        if rank // group_size == g:
            mine = pg
    for loc in range(group_size):
        pg = dist.new_group([c * group_size + loc for c in range(world // group_size)])
        if rank % group_size == loc:
            cross = pg
    return mine, cross
