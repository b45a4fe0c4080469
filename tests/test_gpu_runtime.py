"""Single-GPU runtime tests: the FSDP wrapper around the tiny GPT at world 1.

The model compute is ordinary torch, so the forward/backward of the wrapped
model must equal an unwrapped bf16 copy bit-for-bit (same kernels on the same
inputs); the FSDP epilogue (write-back, / W, Adam on the arena) is checked
bit-exactly against the oracle."""
import numpy as np
import pytest
import torch

from oracle import shardsim_port as sp

pytestmark = pytest.mark.gpu


def build(cfg_name="tiny", **kw):
    from paper_2304_11277_b200.fsdp import FullyShardedDataParallel, MixedPrecision, ModuleWrapPolicy
    from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_
    cfg = CONFIGS[cfg_name]
    kw.setdefault("mixed_precision", MixedPrecision(param_dtype=torch.bfloat16))
    m = FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=0),
                                 auto_wrap_policy=ModuleWrapPolicy({Block}), **kw)
    ref = init_gpt_(GPT(cfg), seed=0).cuda().to(torch.bfloat16)
    return cfg, m, ref


def flat_grads_of(ref, lay):
    g = {n: p.grad.float().cpu().numpy() for n, p in ref.named_parameters()}
    return sp.writeback_grad(lay, g, np.float32)[0]


def test_wrapped_step_matches_unwrapped_and_oracle():
    # (the slot-starved num_slots=2 re-gather needs F > 1: tests/mp_worker.py
    # runs it at W = 2 / 4 / 8, on a 1-GPU box with the ranks sharing cuda:0)
    from paper_2304_11277_b200.workloads import synthetic_batch
    cfg, m, ref = build()
    x, y = synthetic_batch(cfg, 4, seed=3, device="cuda")
    loss = m(x, y)
    loss.backward()
    lref = ref(x, y)
    lref.backward()
    assert loss.item() == lref.item()
    before = [u.master.clone() for u in m.rt.units]
    grads = [m.rt.reduced_grad(i).clone() for i in range(len(m.rt.units))]
    # W = 1 bf16 payload: the reduced gradient lives in the bf16 arena (exact)
    assert all(u.grad_is_low for u in m.rt.units)
    for lay, g in zip(m.layouts, grads):
        exp = flat_grads_of(ref, lay)
        assert np.array_equal(g.cpu().numpy(), exp), f"unit {lay.unit_id} grad"
    m.optimizer(lr=1e-3).step()
    torch.cuda.synchronize()
    for b, g, u in zip(before, grads, m.rt.units):
        p = b.cpu().numpy().copy()
        sp.adam_step(p, g.cpu().numpy(), sp.adam_init(p.size, np.float32), lr=1e-3)
        assert u.master.cpu().numpy().tobytes() == p.tobytes()
        assert torch.equal(u.low, u.master.to(torch.bfloat16))


def test_two_steps_and_no_sync_accumulation():
    from paper_2304_11277_b200.workloads import synthetic_batch
    cfg, m, ref = build()
    opt = m.optimizer(lr=1e-3)
    losses = []
    for s in range(2):
        for k in range(2):
            x, y = synthetic_batch(cfg, 2, seed=10 * s + k, device="cuda")
            if k == 0:
                with m.no_sync():
                    l = m(x, y)
                    l.backward()
            else:
                l = m(x, y)
                l.backward()
            losses.append(l.item())
        opt.step()
    torch.cuda.synchronize()
    assert all(np.isfinite(losses))
    assert losses[2] < losses[0] + 1.0


def test_fp32_no_mixed_precision_step():
    from paper_2304_11277_b200.workloads import synthetic_batch
    cfg, m, _ = build(mixed_precision=None)
    x, y = synthetic_batch(cfg, 2, seed=5, device="cuda")
    l = m(x, y)
    l.backward()
    m.optimizer().step()
    torch.cuda.synchronize()
    assert np.isfinite(l.item())


def test_state_dict_roundtrips_and_trace_format():
    from paper_2304_11277_b200.workloads import GPT, init_gpt_, synthetic_batch
    cfg, a, _ = build()
    x, y = synthetic_batch(cfg, 2, seed=7, device="cuda")
    a(x, y).backward()
    a.optimizer(lr=1e-3).step()
    full = a.full_state_dict()
    shard = a.sharded_state_dict()
    # a model with a different init, loaded from the gathered state
    _, b, _ = build()
    ref = init_gpt_(GPT(cfg), seed=5)
    b.load_full_state_dict({k: v for k, v in ref.state_dict().items()})
    b.load_full_state_dict(full)
    with torch.no_grad():
        assert a(x, y).item() == b(x, y).item()
    for ua, ub in zip(a.rt.units, b.rt.units):
        assert torch.equal(ua.master, ub.master) and torch.equal(ua.low, ub.low)
    # sharded checkpoint restores optimizer state too: both continue identically
    b.load_sharded_state_dict(shard)
    for m in (a, b):
        m(x, y).backward()
        m.optimizer(lr=1e-3).step()
    torch.cuda.synchronize()
    for ua, ub in zip(a.rt.units, b.rt.units):
        assert torch.equal(ua.master, ub.master)
    lines = a.trace_lines()
    assert all(l.startswith("rank=0 seq=") and " kind=" in l and " bytes=" in l for l in lines)


def test_wrapper_grad_scaler_skips_nonfinite_step():
    from paper_2304_11277_b200.fsdp import ShardedGradScaler
    from paper_2304_11277_b200.workloads import synthetic_batch
    cfg, m, _ = build()
    sc = ShardedGradScaler(init_scale=1024.0)
    opt = m.optimizer(lr=1e-3)
    x, y = synthetic_batch(cfg, 2, seed=3, device="cuda")
    sc.scale(m(x, y)).backward()
    sc.step(opt)
    assert not sc.update() and sc.scale_value == 1024.0
    before = [u.master.clone() for u in m.rt.units]
    m.rt.inject_inf = {m.rt.step_count}          # poison unit 0's gradient this step
    sc.scale(m(x, y)).backward()
    sc.step(opt)
    assert sc.update() and sc.scale_value == 512.0 and sc.steps_skipped == 1
    for b, u in zip(before, m.rt.units):
        assert torch.equal(b, u.master)          # every shard skipped on device
    m.rt.inject_inf = set()
    sc.scale(m(x, y)).backward()
    sc.step(opt)
    assert not sc.update()
    assert m.rt.adam_steps == 2                  # the skipped step did not advance Adam's t


class _OddMLP(torch.nn.Module):
    """Root without parameters; units with odd, non-multiple-of-8 sizes and
    one unit whose parameter is never used (zero-filled gradient)."""

    def __init__(self):
        super().__init__()
        self.a = torch.nn.Linear(5, 7)
        self.b = torch.nn.Linear(7, 3)
        self.unused = torch.nn.Linear(3, 3)

    def forward(self, x):
        return self.b(torch.relu(self.a(x))).pow(2).mean()


def test_paramless_root_odd_sizes_unused_unit():
    import warnings
    from paper_2304_11277_b200.fsdp import FullyShardedDataParallel, ModuleWrapPolicy
    torch.manual_seed(0)
    ref = _OddMLP()
    m = FullyShardedDataParallel(_OddMLP().requires_grad_(True), auto_wrap_policy=ModuleWrapPolicy({torch.nn.Linear}),
                                 optimizer="sgd", lr=0.1)
    m.load_full_state_dict({k: v for k, v in ref.state_dict().items()})
    assert m.layouts[0].psi == 0 and [l.psi for l in m.layouts[1:]] == [42, 24, 12]
    x = torch.randn(4, 5, device="cuda")
    refc = _OddMLP().cuda()
    refc.load_state_dict(ref.state_dict())
    loss = m(x)
    loss.backward()
    m.optimizer().step()
    lr = refc(x)
    lr.backward()
    with torch.no_grad():
        for p in refc.parameters():
            if p.grad is not None:
                p -= 0.1 * p.grad
    sd = m.full_state_dict()
    for k, v in refc.state_dict().items():
        assert torch.allclose(sd[k], v, atol=1e-6), k
    assert torch.equal(sd["unused.weight"], refc.unused.weight)      # zero grad: unchanged


def test_optimizer_in_backward_identical():
    """Per-unit Adam on the reduce stream during backward == end-of-step launch."""
    from paper_2304_11277_b200.workloads import synthetic_batch
    cfg, a, _ = build()
    _, b, _ = build(optimizer_in_backward=True)
    for s in range(2):
        x, y = synthetic_batch(cfg, 2, seed=40 + s, device="cuda")
        for m in (a, b):
            l = m(x, y)
            l.backward()
            m.optimizer(lr=1e-3).step()
    torch.cuda.synchronize()
    for ua, ub in zip(a.rt.units, b.rt.units):
        assert torch.equal(ua.master, ub.master)
        assert torch.equal(ua.exp_avg_sq, ub.exp_avg_sq)
        assert torch.equal(ua.low, ub.low)
