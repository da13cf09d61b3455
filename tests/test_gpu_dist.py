"""Multi-GPU parity of the fused NVLink collectives (qwZ, hpZ, qgZ): torchrun
one process per GPU; every rank checks its outputs bit-exactly against the
CPU oracle (tests/dist_worker.py)."""

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(nproc, group, stages, env=None, worker="dist_worker.py", extra=()):
    for attempt in range(3):  # the free port can be taken between probing and binding
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(HERE, worker), "--group", str(group), *(["--stages", str(stages)] if stages else []),
               *extra]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env={**os.environ, **(env or {})})
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return r.stdout


def _run_large(nproc, group, env=None):
    """BASELINE shapes with sampled bitwise parity (tests/dist_large_worker.py)."""
    out = _run(nproc, group, 0, env=env, worker="dist_large_worker.py")
    assert "large parity ok" in out, out[-4000:]


@pytest.mark.parametrize("group", [1, 2])
def test_two_gpus(group):
    _run(2, group, 2)


def test_two_gpus_bucket_pipeline_forced():
    """2x1 (a second hop) with the bucket pipelining forced on (ZPP_QGZ_XB=2;
    by default only one-group layouts pipeline buckets) and the qwZ prefetch
    in share placement: the stream and layer cases of dist_worker stay
    bit-exact on the code paths the defaults skip at this shape."""
    _run(2, 1, 2, env={"ZPP_QGZ_XB": "2", "ZPP_QWZ_PREFETCH_MODE": "share"})


def test_four_gpus_2x2():
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, 2, 2)


def test_four_gpus_1x4():
    """One group of four (Y = 1: the hop-2 self-send fused into K2)."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, 4, 1)


@pytest.mark.parametrize("mode", ["push", "pull", "push-hop2push"])
def test_qgz_hop1_modes(mode):
    """Both hop-1 transports (K1 pushing with TMA bulk stores / K2 pulling)
    on the layouts whose default is the other one: 1xN defaults to pull, 2x2
    to push (see zpp_qgz_reduce_scatter); and with a pushed hop 1, hop 2
    pushed by K2 into the receivers' slots (ZPP_QGZ_HOP2=push, opt-in)."""
    n = torch.cuda.device_count()
    env = {"ZPP_QGZ_MODE": mode.split("-")[0]}
    if mode.endswith("hop2push"):
        env["ZPP_QGZ_HOP2"] = "push"
    _run(2, 2, 2, env=env)
    _run(2, 1, 2, env=env)
    if n >= 4:
        _run(4, 4, 1, env=env)
        _run(4, 2, 2, env=env)


def test_eight_gpus_2x4():
    if torch.cuda.device_count() < 8:
        pytest.skip("needs 8 GPUs")
    _run(8, 4, 1)


def _oversub_allowed():
    # Ranks whose kernels spin on one another's flags, time-sliced on one GPU,
    # have raised Xid 109 (context-switch timeout) on this pool's B200s
    # (B200_PROFILING.md).  These runs passed on 4 B200s during development
    # (profiles/r2/gpu_dist_large_r2.log); they stay opt-in.
    if os.environ.get("ZPP_ALLOW_OVERSUBSCRIBE") != "1":
        pytest.skip("oversubscribed ranks are opt-in (ZPP_ALLOW_OVERSUBSCRIBE=1)")


def test_eight_ranks_2x4_oversubscribed():
    """The driver's 8-GPU layout (2 groups x 4, K3 + cross barrier with X = 4)
    on a smaller box: two ranks per GPU, still one process per rank and peer
    memory through CUDA IPC (see ZPP_OVERSUBSCRIBE in dist_worker.py)."""
    _oversub_allowed()
    n = torch.cuda.device_count()
    if n < 2 or n >= 8:
        pytest.skip("needs 2..7 GPUs (8 run test_eight_gpus_2x4)")
    _run(8, 4, 1, env={"ZPP_OVERSUBSCRIBE": "1"})


# ---- the BASELINE shapes: 1.3B qwZ, 256 MiB qgZ bucket, GPT-13B layer ---------


@pytest.mark.parametrize("group", [1, 2])
def test_large_two_gpus(group):
    _run_large(2, group)


@pytest.mark.parametrize("group", [4, 2])
def test_large_four_gpus(group):
    """1x4 and 2x2 at the BASELINE shapes."""
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run_large(4, group)


def test_large_eight_gpus_2x4():
    if torch.cuda.device_count() < 8:
        pytest.skip("needs 8 GPUs")
    _run_large(8, 4)


def test_large_eight_ranks_2x4_oversubscribed():
    """The 2x4 layout at the BASELINE shapes, two ranks per GPU (see
    test_eight_ranks_2x4_oversubscribed)."""
    _oversub_allowed()
    n = torch.cuda.device_count()
    if n < 4 or n >= 8:
        pytest.skip("needs 4..7 GPUs (8 run test_large_eight_gpus_2x4)")
    _run_large(8, 4, env={"ZPP_OVERSUBSCRIBE": "1"})
