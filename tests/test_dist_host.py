"""Host-side logic of the multi-GPU layer on CPU: IPC-handle exchange over a
world-size-2 gloo group, barrier scopes and workspace layout."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_10209_b200.dist import SymLayout, exchange_handles, members


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank]) * 64
    allh = exchange_handles(blob)
    q.put((rank, allh))
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_handles_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert got[r] == bytes([0]) * 64 + bytes([1]) * 64


def test_barrier_scopes_match_reference_groups():
    # groups of consecutive ranks (zs/partitioner.py:67-73), cross = same local index
    assert members(5, 8, 4, "world") == list(range(8))
    assert members(5, 8, 4, "group") == [4, 5, 6, 7]
    assert members(5, 8, 4, "cross") == [1, 5]
    assert members(0, 2, 1, "cross") == [0, 1]
    assert members(1, 2, 2, "group") == [0, 1]
    with pytest.raises(Exception):
        members(0, 2, 1, "bogus")


def test_layout_regions_are_disjoint_and_aligned():
    lay = SymLayout.plan(1000, 3, 5000)
    assert lay.qwz == 0 and lay.hpz >= 1000 and lay.qgz >= lay.hpz + 3
    assert lay.hpz % 256 == 0 and lay.qgz % 256 == 0 and lay.total % 256 == 0
    assert lay.total >= lay.qgz + 5000


def test_exchange_handles_without_process_group():
    assert exchange_handles(b"x" * 64) == b"x" * 64


def test_stream_layout_pads_the_tail_like_the_reference():
    """Communicator.stream_layout (host arithmetic only): a 7B gradient stream
    in 256 MiB buckets is 52 full buckets plus a 20,678,144-element tail,
    zero-padded to a multiple of W * S * max(block) (zs/engine.py:465-466:
    20,680,704 at W = 8, S = 1, INT4/512); the output holds every
    bucket's partition followed by the padded tail's."""
    from types import SimpleNamespace

    from paper_2306_10209_b200.dist import Communicator
    from paper_2306_10209_b200.quantizer import QuantConfig

    cfg = QuantConfig(bit_width=4, block_size=512)
    for world, stages, want_pad in ((8, 1, 20_680_704), (4, 1, 20_678_656), (2, 2, 20_678_656), (1, 1, 20_678_144)):
        fake = SimpleNamespace(qgz_elems=134_217_728, world=world, qgz_stages=stages, qgz_cfg=cfg, qgz_intra_cfg=cfg)
        full, tail, tail_pad, n_out = Communicator.stream_layout(fake, 7_000_000_000)
        assert (full, tail) == (52, 20_678_144)
        assert tail_pad == want_pad and tail_pad % (world * stages * 512) == 0 and tail_pad >= tail
        assert n_out == (52 * 134_217_728 + tail_pad) // world
