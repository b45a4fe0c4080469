"""The shardsim-shaped Session API on the B200 runtime — tests written like
the reference's own tests/test_engine.py.  Multi-rank cases run in
tests/mp_worker.py (real GPUs); these cover config/API behaviour (CPU) and
world-1 numerics (GPU)."""
import numpy as np
import pytest

from oracle import shardsim_port as sp

SPEC3 = dict(dims=(4, 8, 8, 2))


def test_engine_config_validation():
    from paper_2304_11277_b200.plan import build_plan
    from paper_2304_11277_b200.session import EngineConfig, EngineError
    plan = build_plan(2, 2)
    with pytest.raises(EngineError):
        EngineConfig(plan=plan, reshard_after_forward="SOMETIMES")
    with pytest.raises(EngineError):
        EngineConfig(plan=plan, accumulation="maybe")
    with pytest.raises(EngineError):
        EngineConfig(plan=plan, accumulation_steps=3)
    with pytest.raises(EngineError):
        EngineConfig(plan=plan, rate_limit=0)
    with pytest.raises(EngineError):
        EngineConfig(plan=plan, init_path="lazy")


def test_execution_order_and_scaler():
    from paper_2304_11277_b200.session import (EngineError, ExecutionOrder, ScalerConfig,
                                               ShardedGradScaler)
    order = ExecutionOrder()
    order.record(0)
    order.record(2)
    assert order.backward_order() == [2, 0]
    with pytest.raises(EngineError):
        order.record(0)
    sc = ShardedGradScaler(ScalerConfig(init_scale=8.0, growth_interval=2))
    sc.update(found_inf=True)
    assert sc.scale == 4.0 and sc.steps_skipped == 1
    sc.update(False)
    sc.update(False)
    assert sc.scale == 8.0
    sc.scale = float("inf")
    with pytest.raises(EngineError):
        sc.update(False)


def test_data_semantics_match_reference_oracle():
    from paper_2304_11277_b200.data import ModelSpec, batch_stream, init_values
    spec = ModelSpec(**SPEC3)
    o = sp.eager_param_values(sp.MLPSpec(**SPEC3), 3)
    mine = init_values(spec, 3)
    assert all(np.array_equal(o[k], mine[k]) for k in o)
    a = list(batch_stream(5, 2, 8, 4, 2))
    b = list(sp.batch_stream(5, 2, 8, 4, 2))
    assert all(np.array_equal(x, y) for (x, _), (y, _) in zip(a, b))


def _session(**kw):
    from paper_2304_11277_b200.data import ModelSpec
    from paper_2304_11277_b200.plan import build_plan
    from paper_2304_11277_b200.session import EngineConfig, Session
    seed = kw.pop("seed", 0)
    spec = kw.pop("spec", ModelSpec(**SPEC3))
    return Session(spec, EngineConfig(plan=build_plan(1, 1), **kw), seed=seed)


@pytest.mark.gpu
@pytest.mark.parametrize("opt", ["sgd", "adam"])
def test_world1_session_bitwise_vs_oracle(opt):
    """Integer data + dyadic init keep every fp32 op exact, so the GPU
    session equals the oracle's fp32 restatement of Session.run bit-for-bit."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    sess = _session(seed=3, optimizer=opt)
    res = sess.run(steps=1, batch=8)
    exp, losses, stepped, _ = sp.sharded_train(sp.MLPSpec(**SPEC3), sp.Plan(1, 1), 3, 1, 8,
                                               optimizer=opt, full=np.float32, acc_dtype=np.float32)
    got = sess.gather_full_params()
    for k in exp:
        assert got[k].tobytes() == exp[k].astype(np.float32).tobytes(), k
    assert [r.stepped for r in res] == stepped
    assert abs(res[0].loss - losses[0]) < 1e-6


@pytest.mark.gpu
def test_world1_uniform_close_to_float64_reference():
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    sess = _session(seed=9)
    sess.run(steps=3, batch=8, regime="uniform")
    exp, *_ = sp.sharded_train(sp.MLPSpec(**SPEC3), sp.Plan(1, 1), 9, 3, 8, regime="uniform")
    got = sess.gather_full_params()
    assert max(float(np.abs(got[k] - exp[k]).max()) for k in exp) < 1e-6


@pytest.mark.gpu
def test_world1_scaler_injection_and_mixed():
    from paper_2304_11277_b200.session import PrecisionPolicy
    sess = _session(seed=1, use_scaler=True)
    sess.inject_inf = {(0, 1)}
    res = sess.run(steps=3, batch=8)
    assert [r.stepped for r in res] == [True, False, True]
    assert res[1].found_inf and res[1].scale == 65536.0 * 0.5
    exp, _, stepped, scales = sp.sharded_train(sp.MLPSpec(**SPEC3), sp.Plan(1, 1), 1, 3, 8,
                                               use_scaler=True, inject_inf={(0, 1)},
                                               full=np.float32, acc_dtype=np.float32)
    assert stepped == [r.stepped for r in res]
    got = sess.gather_full_params()
    assert max(float(np.abs(got[k] - exp[k]).max()) for k in exp) < 1e-6
    mixed = _session(seed=4, precision=PrecisionPolicy(mixed=True))
    mixed.run(steps=3, batch=8)
    ref, *_ = sp.sharded_train(sp.MLPSpec(**SPEC3), sp.Plan(1, 1), 4, 3, 8)
    g = mixed.gather_full_params()
    d = max(float(np.abs(g[k] - ref[k]).max()) for k in ref)
    assert 0 < d < 1e-2
    assert mixed.check_reduction_ordering() == []


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["with_comm", "no_comm"])
def test_world1_accumulation_matches_oracle(mode):
    sess = _session(seed=8, accumulation=mode, accumulation_steps=2)
    sess.run(steps=2, batch=8)
    exp, *_ = sp.sharded_train(sp.MLPSpec(**SPEC3), sp.Plan(1, 1), 8, 2, 8, accumulation=mode,
                               accumulation_steps=2, full=np.float32, acc_dtype=np.float32)
    got = sess.gather_full_params()
    assert max(float(np.abs(got[k] - exp[k]).max()) for k in exp) < 1e-6


@pytest.mark.gpu
def test_train_step_validates_micro_batches():
    from paper_2304_11277_b200.session import EngineError
    sess = _session()
    x, y = np.zeros((8, 4)), np.zeros((8, 2))
    with pytest.raises(EngineError):
        sess.train_step([(x, y), (x, y)])


@pytest.mark.gpu
def test_init_paths_bit_identical_and_resident_memory():
    """The reference's three materialisation paths (deferred_init.py:156-263,
    bound by test_acceptance.py:402-433): bit-identical shards; the
    whole-model path peaks at the full unsharded model on the device, the
    deferred and streamed paths at about one unit, and only the streamed path
    holds a host arena (the raw, unpadded model)."""
    from paper_2304_11277_b200.data import ModelSpec
    spec = ModelSpec(dims=(1024,) * 9, init="scaled_uniform")       # 8 units of ~1.05 M
    sess = {p: _session(spec=spec, seed=5, init_path=p) for p in ("deferred", "device", "streamed")}
    ref = sess["deferred"]
    for p in ("device", "streamed"):
        for a, b in zip(ref.rt.units, sess[p].rt.units):
            assert a.master.cpu().numpy().tobytes() == b.master.cpu().numpy().tobytes(), p
    vals = sp.eager_param_values(sp.MLPSpec(dims=(1024,) * 9, init="scaled_uniform"), 5)
    unit_bytes = max(l.psi for l in ref.layouts) * 4
    model_bytes = sum(l.psi for l in ref.layouts) * 4
    st = {p: s.init_stats for p, s in sess.items()}
    assert st["device"]["device_peak_bytes"] >= model_bytes
    for p in ("deferred", "streamed"):
        assert st[p]["device_peak_bytes"] < model_bytes / 2, (p, st[p])
        assert st[p]["device_peak_bytes"] >= unit_bytes
    assert st["streamed"]["host_arena_peak_elements"] == sum(l.raw_numel for l in ref.layouts)
    assert st["deferred"]["host_arena_peak_elements"] == 0
    for uid, lay in enumerate(ref.layouts):      # and they equal the oracle's replay
        exp = sp.shard(sp.flatten({k: v.astype(np.float32) for k, v in vals.items()}, lay, np.float32),
                       lay, 0)
        assert ref.rt.units[uid].master.cpu().numpy().tobytes() == exp.tobytes()
