"""Generate golden vectors from the REAL reference (`shardsim`).

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `/root/reference/pkg/src/shardsim` read-only and writes
`tests/golden/shardsim_golden.npz` + `tests/golden/shardsim_golden.json`.
The committed fixtures pin `oracle/` (tests/test_oracle_golden.py), which in
turn is the checker for the CUDA path.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# tiny GPT (d=256, L=2, V=1024, S=128, GPT-2 style, tied head in the root unit)
D, L, V, S = 256, 2, 1024, 128


def tiny_gpt_shapes():
    shapes = [("wte.weight", (V, D)), ("wpe.weight", (S, D))]
    units = [["wte.weight", "wpe.weight"]]
    for i in range(L):
        p = f"h.{i}."
        blk = [(p + "ln_1.weight", (D,)), (p + "ln_1.bias", (D,)),
               (p + "attn.c_attn.weight", (3 * D, D)), (p + "attn.c_attn.bias", (3 * D,)),
               (p + "attn.c_proj.weight", (D, D)), (p + "attn.c_proj.bias", (D,)),
               (p + "ln_2.weight", (D,)), (p + "ln_2.bias", (D,)),
               (p + "mlp.c_fc.weight", (4 * D, D)), (p + "mlp.c_fc.bias", (4 * D,)),
               (p + "mlp.c_proj.weight", (D, 4 * D)), (p + "mlp.c_proj.bias", (D,))]
        shapes += blk
        units.append([n for n, _ in blk])
    shapes += [("ln_f.weight", (D,)), ("ln_f.bias", (D,))]
    units[0] += ["ln_f.weight", "ln_f.bias"]
    return shapes, units


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import shardsim as ss  # noqa: E402

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": REF, "shardsim_version": ss.__version__}

    # -- layouts (flatparam.py:63-96, :238-247) ---------------------------
    shapes = [("a.weight", (2, 3)), ("a.bias", (2,)), ("b.weight", (3, 3))]
    units = [["a.weight", "a.bias"], ["b.weight"]]
    lays = ss.build_unit_layouts(shapes, units, 4)
    meta["two_unit_dump"] = ss.dump_plan_lines(lays)
    meta["two_unit"] = [{"offsets": [o.offset for o in l.originals], "psi": l.psi,
                         "padding": l.padding, "shard": l.shard_numel} for l in lays]
    gs, gu = tiny_gpt_shapes()
    meta["tiny_gpt"] = {}
    for f in (1, 2, 4, 8, 3, 7):
        ls = ss.build_unit_layouts(gs, gu, f)
        meta["tiny_gpt"][str(f)] = {"psi": [l.psi for l in ls], "padding": [l.padding for l in ls],
                                    "dump": ss.dump_plan_lines(ls)}
    spec3 = ss.ModelSpec(dims=(4, 8, 8, 2))
    meta["spec3_dump"] = {str(f): ss.dump_plan_lines(
        ss.build_unit_layouts(spec3.param_shapes(), spec3.unit_param_names(), f))
        for f in (1, 2, 4)}

    # -- collective values on float32 payloads (collectives.py:273-301) ----
    rng = np.random.default_rng(1234)
    for w in (1, 2, 3, 4, 8):
        n = 6 * w
        inputs = [rng.standard_normal(n).astype(np.float32) * np.float32(10.0 ** rng.integers(-3, 4))
                  for _ in range(w)]
        fab = ss.CollectiveFabric(ss.build_plan(w, w))
        def ag(rank):
            out = yield fab.all_gather_begin(rank, range(w), inputs[rank][: n // w])
            return out
        def rs(rank):
            out = yield fab.reduce_scatter_begin(rank, range(w), inputs[rank])
            return out
        def ar(rank):
            out = yield fab.all_reduce_begin(rank, range(w), inputs[rank])
            return out
        for kind, fn in (("ag", ag), ("rs", rs), ("ar", ar)):
            res = ss.run_symmetric(fab, fn)
            for r in range(w):
                arrays[f"coll/{kind}/w{w}/out{r}"] = np.asarray(res[r])
        for r in range(w):
            arrays[f"coll/in/w{w}/r{r}"] = inputs[r]

    # ascending order known-answer (test_collectives.py:111-122)
    # -- hybrid reduce for all (W <= 8, F | W), float32 (collectives.py:377-397)
    for w in range(1, 9):
        for f in range(1, w + 1):
            if w % f:
                continue
            plan = ss.build_plan(w, f)
            fab = ss.CollectiveFabric(plan)
            psi = 4 * f * w
            grads = [rng.standard_normal(psi).astype(np.float32) for _ in range(w)]
            res = ss.run_symmetric(fab, lambda rank: ss.hybrid_reduce_task(fab, rank, grads[rank]))
            for r in range(w):
                arrays[f"hyb/w{w}f{f}/in{r}"] = grads[r]
                arrays[f"hyb/w{w}f{f}/out{r}"] = np.asarray(res[r])

    # -- optimizers on float32 shards (numerics.py:239-296) ----------------
    for lr in (1e-3, 0.01):
        opt = ss.Adam(lr=lr)
        n = 257
        p = rng.uniform(-1, 1, n).astype(np.float32)
        arrays[f"adam/lr{lr}/p0"] = p.copy()
        st = opt.init_state(n, dtype="low")
        for t in range(4):
            g = (rng.standard_normal(n) * 10.0 ** (t - 2)).astype(np.float32)
            if t == 3:
                g[:5] = 0.0
            arrays[f"adam/lr{lr}/g{t}"] = g
            opt.step(p, g, st)
            arrays[f"adam/lr{lr}/p{t + 1}"] = p.copy()
            arrays[f"adam/lr{lr}/m{t + 1}"] = st["m"].copy()
            arrays[f"adam/lr{lr}/v{t + 1}"] = st["v"].copy()
    sgd = ss.SGD()
    p = rng.uniform(-1, 1, 64).astype(np.float32)
    g = rng.standard_normal(64).astype(np.float32)
    arrays["sgd/p0"], arrays["sgd/g"] = p.copy(), g
    sgd.step(p, g, {})
    arrays["sgd/p1"] = p

    # -- whole sessions (engine.py:296-597) ---------------------------------
    sessions = {
        "w4f2_sgd": dict(w=4, f=2, seed=3, steps=4, batch=8),
        "w2f2_adam": dict(w=2, f=2, seed=5, steps=3, batch=8, cfg={"optimizer": "adam"}),
        "w4f4_uniform": dict(w=4, f=4, seed=9, steps=3, batch=8, regime="uniform"),
        "w8f4_hybrid_adam": dict(w=8, f=4, seed=11, steps=3, batch=16, regime="uniform",
                                 cfg={"optimizer": "adam"}),
        "w4f1_noshard": dict(w=4, f=1, seed=2, steps=2, batch=8),
        "w4f4_mixed": dict(w=4, f=4, seed=4, steps=3, batch=8,
                           cfg={"precision": ss.PrecisionPolicy(mixed=True)}),
        "w4f2_scaler_inject": dict(w=4, f=2, seed=1, steps=3, batch=8,
                                   cfg={"use_scaler": True}, inject={(2, 1)}),
        "w4f2_accum_with": dict(w=4, f=2, seed=8, steps=3, batch=8,
                                cfg={"accumulation": ss.ACCUM_WITH_COMM, "accumulation_steps": 2}),
        "w4f2_accum_no": dict(w=4, f=2, seed=8, steps=3, batch=8,
                              cfg={"accumulation": ss.ACCUM_NO_COMM, "accumulation_steps": 2}),
        "w2f2_multifwd": dict(w=2, f=2, seed=2, steps=2, batch=8, cfg={"forwards_per_micro": 2}),
        "w4f2_sum_nraf": dict(w=4, f=2, seed=6, steps=2, batch=8,
                              cfg={"loss_reduction": "sum", "reshard_after_forward": ss.NRAF}),
    }
    meta["sessions"] = {}
    spec = ss.ModelSpec(dims=(4, 8, 8, 2))
    for name, s in sessions.items():
        cfg = dict(s.get("cfg", {}))
        sess = ss.Session(spec, ss.EngineConfig(plan=ss.build_plan(s["w"], s["f"]), **cfg),
                          seed=s["seed"])
        if "inject" in s:
            sess.inject_inf = set(s["inject"])
        res = sess.run(steps=s["steps"], batch=s["batch"], regime=s.get("regime", "integer"))
        params = sess.gather_full_params()
        for k, v in params.items():
            arrays[f"sess/{name}/{k}"] = v
        info = {k: v for k, v in s.items() if k not in ("cfg", "inject")}
        info["cfg"] = {k: (v.mixed if k == "precision" else v) for k, v in cfg.items()}
        info["inject"] = sorted(list(s.get("inject", [])))
        info["losses"] = [r.loss for r in res]
        info["stepped"] = [r.stepped for r in res]
        info["scales"] = [r.scale for r in res]
        meta["sessions"][name] = info

    # local_train oracle used by shardsim's own bitwise tests (engine.py:920)
    lt = ss.local_train(spec, 3, 4, 8, grad_slices=4, grad_block=2)
    for k, v in lt.params.items():
        arrays[f"local/w4f2/{k}"] = v

    np.savez_compressed(os.path.join(HERE, "shardsim_golden.npz"), **arrays)
    with open(os.path.join(HERE, "shardsim_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, ensure_ascii=False)
    print(f"wrote {len(arrays)} arrays")


if __name__ == "__main__":
    main()
