"""CPU checks of bench.py's output contract: the reference arm prints exactly
one JSON line on stdout with the keys the driver reads (the GPU arm shares
the same emitter, which reserves stdout for that line)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    env = {**os.environ, "RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def _bench_module():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_bench_layouts_follow_survey():
    """SURVEY 8d's hierarchy: two groups of W/2 GPUs (W = 8: 2x4, W = 4: 2x2,
    W = 2: 2x1); a 1-GPU world is one group of one."""
    b = _bench_module()
    assert [b.group_size_for(w) for w in (1, 2, 4, 8)] == [1, 1, 2, 4]


def test_qgz_byte_model():
    """qgz_bytes (the qgZ roofline's wire and HBM bytes): at W = 8
    (2x4) one 256 MiB bucket sends, per GPU, 3 INT4 hop-1 messages of Y*L
    elements with fp32 absmax and one hop-2 segment of L elements whose absmax
    is the f64 block max of the fold (8 B/block, which keeps hop 2 bit-exact;
    SURVEY's 59,637,760 B assumed a 4 B scale there): 59,768,832 B.  With one
    group hop 2 is a self-send and costs no wire."""
    b = _bench_module()
    L = 134_217_728 // 8
    wire, hbm = b.qgz_bytes(134_217_728, 8, 4)
    assert wire == 3 * (2 * L // 2 + 2 * L // 512 * 4) + (L // 2 + L // 512 * 8) == 59_768_832
    w1, _ = b.qgz_bytes(134_217_728, 4, 4)
    L4 = 134_217_728 // 4
    assert w1 == 3 * (L4 // 2 + L4 // 512 * 4)
    assert hbm > 2 * 134_217_728  # at least the bf16 read of the bucket
