"""The toy ZeRO++ training loop on the GPU collectives (paper_2306_10209_b200.engine):
whole runs bit-identical to the reference's TrainingEngine (golden fixtures made by
tests/golden/make_golden.py), plus the reference's acceptance checks c08
(passthrough routing changes nothing) and c09 (convergence envelope),
pkg/tests/test_acceptance.py:268-341."""

import hashlib
import json
import os
import time

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "engine.json")


def _cfg(zpp, kw):
    out = {}
    for k, v in kw.items():
        out[k] = zpp.QuantConfig(bit_width=v[1], block_size=v[2]) if isinstance(v, list) and v and v[0] == "q" else v
    return out


def _cases():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_training_run_matches_reference_bit_for_bit(case):
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200 import engine as E

    eng = E.TrainingEngine(E.ToyTaskConfig(**case["task"]), E.ZeroConfig(steps=case["steps"], **_cfg(zpp, case["zero"])))
    if case["passthrough"]:
        eng.weight_codec = zpp.PassthroughCodec()
        eng.grad_codec = zpp.PassthroughCodec()
    rec = eng.train()
    assert rec.padded_params == case["padded"]
    assert float(rec.initial_loss).hex() == case["initial_loss"]
    assert [float(s.loss).hex() for s in rec.steps] == case["losses"]
    assert [[repr(s.fwd_gather_volume), repr(s.bwd_gather_volume), repr(s.reduce_volume)] for s in rec.steps] \
        == case["volumes"]
    assert [bool(s.quantized_grads) for s in rec.steps] == case["quantized_grads"]
    assert hashlib.sha256(rec.to_csv().encode()).hexdigest() == case["csv_sha256"]  # incl. est_latency_s
    assert float(rec.final_loss).hex() == case["final_loss"] and rec.diverged == case["diverged"]
    assert hashlib.sha256(eng.master.tobytes()).hexdigest() == case["master_sha256"]


def test_c08_passthrough_routing_is_bit_identical():
    import numpy as np

    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200 import engine as E

    task = E.ToyTaskConfig()
    plain = E.TrainingEngine(task, E.ZeroConfig(steps=100))
    routed = E.TrainingEngine(task, E.ZeroConfig(steps=100, quantized_weight_gather=True,
                                                 hierarchical_secondary_gather=True, quantized_grad_reduce=True))
    routed.weight_codec = zpp.PassthroughCodec()
    routed.grad_codec = zpp.PassthroughCodec()
    a, b = plain.train(), routed.train()
    assert [s.loss for s in a.steps] == [s.loss for s in b.steps]
    assert np.array_equal(plain.master, routed.master)


def test_c09_convergence_envelope():
    import paper_2306_10209_b200 as zpp
    from paper_2306_10209_b200 import engine as E

    t0 = time.perf_counter()
    task = E.ToyTaskConfig(noise_sigma=0.1, input_scale_range=16.0)
    run = lambda **kw: E.train_toy(task, E.ZeroConfig(seed=1, **kw)).final_loss  # noqa: E731
    base = run()
    all_on = run(quantized_weight_gather=True, hierarchical_secondary_gather=True, quantized_grad_reduce=True)
    blocked = run(quantized_grad_reduce=True, grad_quant=zpp.QuantConfig(bit_width=4, block_size=512))
    coarse = zpp.QuantConfig(bit_width=4, block_size=2560)  # one scale per transmitted slice
    slice_scale = run(quantized_grad_reduce=True, grad_quant=coarse)
    sched = {f: run(quantized_grad_reduce=True, grad_quant=coarse, grad_quant_fraction=f) for f in (0.0, 0.5, 1.0)}
    assert abs(all_on - base) / base <= 0.05
    assert slice_scale > blocked
    assert sched[0.0] == base
    lo, hi = sorted((sched[0.0], sched[1.0]))
    assert lo <= sched[0.5] <= hi and sched[0.0] != sched[1.0]
    assert time.perf_counter() - t0 < 120.0
