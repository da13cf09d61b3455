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
    import engine_harness as E

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
    import engine_harness as E

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
    import engine_harness as E

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


SMALL = dict(in_dim=6, hidden=(16, 16), out_dim=4, eval_samples=64)


def test_one_rank_run_equals_a_direct_adam_loop():
    """World of one: the engine (fp16 weight/gradient boundaries, f64 Adam
    masters) equals the same loop written out directly (zs/engine.py:332-428)."""
    import numpy as np

    import engine_harness as E

    task = E.ToyTaskConfig(**SMALL)
    cfg = E.ZeroConfig(nodes=1, gpus_per_node=1, steps=20, seed=11)
    eng = E.TrainingEngine(task, cfg)
    rec = eng.train()
    dims = task.layer_dims()
    t_rng, i_rng, d_rng, _ = (np.random.default_rng(q) for q in np.random.SeedSequence(cfg.seed).spawn(4))
    teacher = E.init_params(dims, t_rng, scale=1.5)
    w = E.init_params(dims, i_rng, output_bias=task.output_offset)
    m1, m2, losses = np.zeros_like(w), np.zeros_like(w), []
    for t in range(1, cfg.steps + 1):
        x = d_rng.normal(size=(cfg.batch_per_rank, task.in_dim))
        t_out, _ = E.mlp_forward(teacher, x, dims)
        y = t_out + task.output_offset + task.noise_sigma * d_rng.normal(size=t_out.shape)
        loss, g = E.mlp_loss_and_grad(E.half_round(w), x, y, dims)
        losses.append(loss)
        g = E.half_round(g)
        m1 = cfg.adam_beta1 * m1 + (1 - cfg.adam_beta1) * g
        m2 = cfg.adam_beta2 * m2 + (1 - cfg.adam_beta2) * g ** 2
        w -= cfg.lr * (m1 / (1 - cfg.adam_beta1 ** t)) / (np.sqrt(m2 / (1 - cfg.adam_beta2 ** t)) + cfg.adam_eps)
    assert [s.loss for s in rec.steps] == losses
    assert np.array_equal(eng.master[:eng.m_params], w)


def test_hpz_moves_traffic_not_values():
    import numpy as np

    import engine_harness as E

    task = E.ToyTaskConfig(**SMALL)
    a = E.TrainingEngine(task, E.ZeroConfig(steps=8, seed=5))
    b = E.TrainingEngine(task, E.ZeroConfig(steps=8, seed=5, hierarchical_secondary_gather=True))
    ra, rb = a.train(), b.train()
    assert [s.loss for s in ra.steps] == [s.loss for s in rb.steps]
    assert np.array_equal(a.master, b.master)
    assert {s.bwd_gather_volume for s in ra.steps} == {1.0} and {s.bwd_gather_volume for s in rb.steps} == {0.0}


def test_switch_volumes_and_schedule():
    import paper_2306_10209_b200 as zpp
    import engine_harness as E

    task = E.ToyTaskConfig(**SMALL)
    for s in E.train_toy(task, E.ZeroConfig(steps=3, seed=2)).steps:
        assert (s.fwd_gather_volume, s.bwd_gather_volume, s.reduce_volume) == (1.0, 1.0, 1.0)
        assert s.est_latency_s > 0 and not (s.quantized_weights or s.secondary_gather or s.quantized_grads)
    full = E.ZeroConfig(steps=3, seed=2, quantized_weight_gather=True, hierarchical_secondary_gather=True,
                        quantized_grad_reduce=True, grad_quant=zpp.QuantConfig(bit_width=4, block_size=64))
    rec = E.train_toy(task, full)
    assert not rec.diverged
    for s in rec.steps:
        assert (s.fwd_gather_volume, s.bwd_gather_volume, s.reduce_volume) == (0.5, 0.0, 0.25)
    q64 = zpp.QuantConfig(bit_width=4, block_size=64)
    flags = lambda f, n: [s.quantized_grads for s in E.train_toy(  # noqa: E731
        task, E.ZeroConfig(steps=n, seed=1, quantized_grad_reduce=True, grad_quant_fraction=f, grad_quant=q64)).steps]
    assert flags(0.5, 10) == [False, True] * 5
    assert sum(flags(0.25, 8)) == 2 and not any(flags(0.0, 4))


def test_training_converges_and_divergence_is_flagged():
    import engine_harness as E

    task = E.ToyTaskConfig(**SMALL)
    rec = E.train_toy(task, E.ZeroConfig(steps=150, seed=7, lr=5e-3, quantized_weight_gather=True,
                                         hierarchical_secondary_gather=True, quantized_grad_reduce=True))
    assert not rec.diverged and rec.final_loss < 0.5 * rec.initial_loss
    bad = E.train_toy(task, E.ZeroConfig(steps=40, seed=0, lr=3e3))
    assert bad.diverged and len(bad.steps) <= 40
    lines = E.train_toy(task, E.ZeroConfig(steps=2, seed=3)).to_csv().strip().split("\n")
    assert lines[0].startswith("step,loss,") and len(lines) == 3 and lines[1].split(",")[-3:] == ["0", "0", "0"]
