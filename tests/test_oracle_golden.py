"""Pin the oracle (`oracle/`) against golden vectors produced by the real
reference (tests/golden/make_golden.py imports shardsim).  Bit-exact with the
reference's own dtypes (full = float64, low = float32)."""
import numpy as np
import pytest

from oracle import shardsim_port as sp
from oracle.bf16 import f32_to_bf16_bits, round_to_bf16

from tests.golden.make_golden import tiny_gpt_shapes


def test_two_unit_layouts_known_answer(golden):
    _, meta = golden
    shapes = [("a.weight", (2, 3)), ("a.bias", (2,)), ("b.weight", (3, 3))]
    lays = sp.build_unit_layouts(shapes, [["a.weight", "a.bias"], ["b.weight"]], 4)
    assert sp.dump_plan_lines(lays) == meta["two_unit_dump"]
    for lay, exp in zip(lays, meta["two_unit"]):
        assert [o.offset for o in lay.originals] == exp["offsets"]
        assert (lay.psi, lay.padding, lay.shard_numel) == (exp["psi"], exp["padding"], exp["shard"])


@pytest.mark.parametrize("f", [1, 2, 4, 8, 3, 7])
def test_tiny_gpt_layouts(golden, f):
    _, meta = golden
    shapes, units = tiny_gpt_shapes()
    lays = sp.build_unit_layouts(shapes, units, f)
    exp = meta["tiny_gpt"][str(f)]
    assert [l.psi for l in lays] == exp["psi"]
    assert [l.padding for l in lays] == exp["padding"]
    assert sp.dump_plan_lines(lays) == exp["dump"]
    if f == 2:
        assert exp["psi"] == [295424, 789760, 789760]   # SURVEY §8 tiny GPT


def test_spec3_dumps(golden):
    _, meta = golden
    spec = sp.MLPSpec(dims=(4, 8, 8, 2))
    for f, lines in meta["spec3_dump"].items():
        lays = sp.build_unit_layouts(spec.param_shapes(), spec.unit_param_names(), int(f))
        assert sp.dump_plan_lines(lays) == lines


def test_layout_errors():
    shapes = [("w", (2,)), ("v", (2,))]
    with pytest.raises(sp.SharedParameterError):
        sp.build_unit_layouts(shapes, [["w"], ["w", "v"]], 2)
    with pytest.raises(sp.FlatParamError):
        sp.build_unit_layouts(shapes, [["w"]], 2)


@pytest.mark.parametrize("w", [1, 2, 3, 4, 8])
def test_collectives_bit_exact(golden, w):
    arrays, _ = golden
    inputs = [arrays[f"coll/in/w{w}/r{r}"] for r in range(w)]
    n = inputs[0].size
    ag = sp.all_gather([x[: n // w] for x in inputs])
    rs = sp.reduce_scatter(inputs)
    ar = sp.all_reduce(inputs)
    for r in range(w):
        assert np.array_equal(ag, arrays[f"coll/ag/w{w}/out{r}"])
        assert rs[r].tobytes() == arrays[f"coll/rs/w{w}/out{r}"].tobytes()
        assert ar.tobytes() == arrays[f"coll/ar/w{w}/out{r}"].tobytes()


def test_ascending_order_known_answer():
    # test_collectives.py:111-122: ((0 + 1e16) + 1) + -1e16 == 0
    out = sp.all_reduce([np.array([1e16]), np.array([1.0]), np.array([-1e16])])
    assert out[0] == 0.0
    # SPEC.md:137 example
    rs = sp.reduce_scatter([np.array([1., 2, 3, 4]), np.array([10., 20, 30, 40])])
    assert rs[0].tolist() == [11, 22] and rs[1].tolist() == [33, 44]
    # SPEC.md:155 example: W=4, F=2 grads 1..4 -> 10
    out = sp.hybrid_reduce([np.full(2, float(r + 1)) for r in range(4)], sp.Plan(4, 2))
    assert all(o.tolist() == [10.0] for o in out)


def test_hybrid_all_w_f(golden):
    arrays, _ = golden
    for w in range(1, 9):
        for f in range(1, w + 1):
            if w % f:
                continue
            grads = [arrays[f"hyb/w{w}f{f}/in{r}"] for r in range(w)]
            out = sp.hybrid_reduce(grads, sp.Plan(w, f))
            for r in range(w):
                assert out[r].tobytes() == arrays[f"hyb/w{w}f{f}/out{r}"].tobytes(), (w, f, r)


@pytest.mark.parametrize("lr", [1e-3, 0.01])
def test_adam_float32_bit_exact(golden, lr):
    arrays, _ = golden
    p = arrays[f"adam/lr{lr}/p0"].copy()
    st = sp.adam_init(p.size, np.float32)
    for t in range(4):
        sp.adam_step(p, arrays[f"adam/lr{lr}/g{t}"], st, lr=lr)
        assert p.tobytes() == arrays[f"adam/lr{lr}/p{t + 1}"].tobytes()
        assert st["m"].tobytes() == arrays[f"adam/lr{lr}/m{t + 1}"].tobytes()
        assert st["v"].tobytes() == arrays[f"adam/lr{lr}/v{t + 1}"].tobytes()


def test_sgd_bit_exact(golden):
    arrays, _ = golden
    p = arrays["sgd/p0"].copy()
    sp.sgd_step(p, arrays["sgd/g"])
    assert p.tobytes() == arrays["sgd/p1"].tobytes()


SESSIONS = ["w4f2_sgd", "w2f2_adam", "w4f4_uniform", "w8f4_hybrid_adam", "w4f1_noshard",
            "w4f4_mixed", "w4f2_scaler_inject", "w4f2_accum_with", "w4f2_accum_no",
            "w2f2_multifwd", "w4f2_sum_nraf"]


@pytest.mark.parametrize("name", SESSIONS)
def test_sharded_train_matches_shardsim_session(golden, name):
    """The composed restatement reproduces shardsim's Session bit-for-bit."""
    arrays, meta = golden
    s = meta["sessions"][name]
    cfg = dict(s["cfg"])
    kw = {}
    if cfg.pop("precision", False):
        kw["mixed"] = True
    for k in ("optimizer", "use_scaler", "accumulation", "accumulation_steps",
              "forwards_per_micro", "loss_reduction"):
        if k in cfg:
            kw[k] = cfg[k]
    params, losses, stepped, scales = sp.sharded_train(
        sp.MLPSpec(dims=(4, 8, 8, 2)), sp.Plan(s["w"], s["f"]), s["seed"], s["steps"],
        s["batch"], regime=s.get("regime", "integer"),
        inject_inf={tuple(x) for x in s["inject"]}, **kw)
    for k, v in params.items():
        assert v.tobytes() == arrays[f"sess/{name}/{k}"].tobytes(), (name, k)
    assert losses == s["losses"]
    assert stepped == s["stepped"]
    if s["cfg"].get("use_scaler"):
        assert scales == s["scales"]


def test_local_train_matches_sharded(golden):
    arrays, _ = golden
    params, *_ = sp.sharded_train(sp.MLPSpec(dims=(4, 8, 8, 2)), sp.Plan(4, 2), 3, 4, 8)
    for k, v in params.items():
        assert v.tobytes() == arrays[f"local/w4f2/{k}"].tobytes()


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(10000).astype(np.float32) * 1e3,
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-40, -1e-40, 3.4e38, 1.00390625,
                  1.01171875, 65504.0], dtype=np.float32),
        (np.arange(1 << 16, dtype=np.uint32) << 16 | 0x8000).view(np.float32)])
    ours = f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    ok = ~np.isnan(x)
    assert np.array_equal(ours[ok], ref[ok])
    assert np.isnan(round_to_bf16(x[~ok])).all()
