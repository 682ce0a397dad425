"""ACCO round on the GPU engine vs the CPU oracle restatement of AccoEngine
(proj/src/protocols.cpp:437-709), which is itself pinned bitwise to the
reference on the reference's problems (tests/test_oracle_golden.py).

Bit-exact: micro-batch counts per stage, samples_cum, token indexing (through
the seeds). fp32 tolerance (north star): per-update theta / theta-tilde
rel <= 1e-5 (norm-wise) and full-dataset loss rel <= 1e-5."""
import numpy as np
import pytest

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import api

pytestmark = pytest.mark.gpu

MINI = dict(vocab=64, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3)
C1 = dict(vocab=256, d_model=128, n_layer=2, n_head=4, seq_len=64, n_samples=64, data_seed=1)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _oracle(method, cfg, opt, sim, T, schedule=None, theta0=None):
    gc = G.GPTConfig(**cfg)
    prob = G.LMProblem(gc)
    th0 = G.default_theta0(gc, sim.master_seed).astype(np.float32).astype(np.float64) if theta0 is None else theta0
    ocfg = O.OptimizerConfig(**{k: getattr(opt, k) for k in O.OptimizerConfig.__dataclass_fields__})
    osim = O.SimConfig(sim.n_workers, sim.batch_size, sim.n_grad_accumulation, False, sim.master_seed,
                       sim.warmup_rounds)

    def grad_fn(theta, stream):
        return prob.stochastic_grad(theta, stream, sim.batch_size)

    return O.run_method(method, grad_fn, th0, ocfg, osim, T, schedule=schedule, eval_fn=prob.value_and_grad)


def _compare(tr, ref, tol=1e-5):
    assert len(tr.records) == len(ref.records)
    for t, (r, o) in enumerate(zip(tr.records, ref.records)):
        assert r.update == o.update
        assert r.mb_main == o.mb_main and r.mb_estimate == o.mb_estimate
        assert r.samples_cum == o.samples_cum
        assert abs(r.loss - o.loss) <= tol * abs(o.loss), (t, r.loss, o.loss)
        assert _rel(tr.theta_history[t + 1], ref.theta_history[t + 1]) <= tol, t
        assert _rel(tr.estimate_history[t + 1], ref.estimate_history[t + 1]) <= tol, t
        assert abs(r.train_loss - o.train_loss) <= 1e-5 * abs(o.train_loss)


ADAMW = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95, scheduler="cosine")
SGD = api.OptimizerConfig(kind="sgd", learning_rate=0.5)


@pytest.mark.parametrize("n_workers,k", [(1, 1), (2, 1), (3, 2)])
@pytest.mark.parametrize("opt", [ADAMW, SGD], ids=["adamw", "sgd"])
def test_acco_floor_schedule_matches_oracle(cuda, n_workers, k, opt):
    sim = api.SimConfig(n_workers=n_workers, batch_size=4, n_grad_accumulation=k, master_seed=7)
    tr = api.run_protocol("acco", api.LMConfig(**MINI, precision="fp32", max_batch=8), opt, sim, 6)
    ref = _oracle("acco", MINI, opt, sim, 6)
    assert not tr.diverged
    _compare(tr, ref)
    # floor schedule = the reference's under free comm (round-0 estimate half is the bootstrap)
    assert tr.records[0].mb_estimate == [1] * n_workers
    assert all(r.mb_main == [k] * n_workers for r in tr.records)


def test_acco_replay_heterogeneous_counts(cuda):
    # per-stage counts of a straggler scenario (cf. test_protocols.cpp:242-252)
    sched = [([1, 1, 1], [3, 3, 1])] + [([3, 2, 1], [3, 3, 1])] * 4
    sim = api.SimConfig(n_workers=3, batch_size=2, master_seed=11, schedule="replay", replay=sched)
    tr = api.run_protocol("acco", api.LMConfig(**MINI, precision="fp32", max_batch=8), ADAMW, sim, 5)
    ref = _oracle("acco", MINI, ADAMW, sim, 5, schedule=sched)
    _compare(tr, ref)


@pytest.mark.parametrize("method", ["ddp", "zero1"])
def test_sync_baselines_match_oracle_ddp(cuda, method):
    sim = api.SimConfig(n_workers=2, batch_size=4, n_grad_accumulation=2, master_seed=5)
    tr = api.run_protocol(method, api.LMConfig(**MINI, precision="fp32", max_batch=8), ADAMW, sim, 5)
    ref = _oracle("ddp", MINI, ADAMW, sim, 5)
    _compare(tr, ref)


def test_acco_c1_config(cuda):
    """BASELINE.json config 1 shape: tiny GPT (2L, d=128, seq=64), 2 workers."""
    sim = api.SimConfig(n_workers=2, batch_size=8, master_seed=1, eval_every=1)
    tr = api.run_protocol("acco", api.LMConfig(**C1, precision="fp32", max_batch=8), ADAMW, sim, 3)
    ref = _oracle("acco", C1, ADAMW, sim, 3)
    _compare(tr, ref)


def test_adaptive_schedule_replays_on_oracle(cuda):
    """Adaptive (timing-driven) counts are logged; replaying them on the oracle
    reproduces the trajectory."""
    sim = api.SimConfig(n_workers=1, batch_size=4, n_grad_accumulation=1, master_seed=3, schedule="adaptive")
    tr = api.run_protocol("acco", api.LMConfig(**MINI, precision="fp32", max_batch=8), ADAMW, sim, 5)
    sched = O.schedule_from_records(tr.records)
    assert all(m >= 1 for r in tr.records for m in r.mb_main + r.mb_estimate)
    ref = _oracle("acco", MINI, ADAMW, sim, 5, schedule=sched)
    _compare(tr, ref)


def test_bf16_acco_tracks_oracle_loss(cuda):
    sim = api.SimConfig(n_workers=2, batch_size=4, master_seed=2)
    opt = api.OptimizerConfig(kind="adamw", learning_rate=3e-3, adam_beta2=0.95)
    tr = api.run_protocol("acco", api.LMConfig(**C1, precision="bf16", max_batch=8), opt, sim, 8)
    ref = _oracle("acco", C1, opt, sim, 8)
    for r, o in zip(tr.records, ref.records):
        assert abs(r.loss - o.loss) <= 2e-2 * abs(o.loss)
    assert tr.records[-1].loss < tr.records[0].loss


def test_engine_validation(cuda):
    m = api.LMConfig(**MINI, precision="fp32", max_batch=4)
    with pytest.raises(api.InvalidArgument):
        api.run_protocol("acco", m, ADAMW, api.SimConfig(batch_size=8), 2)  # exceeds workspace
    with pytest.raises(api.InvalidArgument):
        api.run_protocol("dpu", m, ADAMW, api.SimConfig(warmup_rounds=-1), 2)
    with pytest.raises(api.InvalidArgument):
        api.run_protocol("pipeline", m, ADAMW, api.SimConfig(), 2)
    with pytest.raises(api.InvalidArgument):
        api.run_protocol("acco", m, ADAMW, api.SimConfig(), 0)
    with pytest.raises(api.InvalidArgument):
        api.run_protocol("acco", m, ADAMW, api.SimConfig(n_workers=2, schedule="adaptive"), 2)


@pytest.mark.parametrize("method,n_workers,k,warmup", [("dpu", 1, 1, 0), ("dpu", 2, 2, 0), ("dpu", 2, 1, 2),
                                                       ("wp", 1, 1, 0), ("wp", 3, 2, 0)])
@pytest.mark.parametrize("opt", [ADAMW, SGD], ids=["adamw", "sgd"])
def test_delayed_baselines_match_oracle(cuda, method, n_workers, k, warmup, opt):
    """DPU / WP (protocols.cpp:340-425) on the same kernels: one pending bundle
    per worker consumed per update, seeds, warm-up rounds, discarded tail."""
    sim = api.SimConfig(n_workers=n_workers, batch_size=4, n_grad_accumulation=k, master_seed=13,
                        warmup_rounds=warmup, eval_every=1)
    tr = api.run_protocol(method, api.LMConfig(**MINI, precision="fp32", max_batch=8), opt, sim, 6)
    ref = _oracle(method, MINI, opt, sim, 6)
    assert not tr.diverged
    _compare(tr, ref)
    assert tr.issued_micro_batches == ref.issued_micro_batches
    assert tr.discarded_micro_batches == ref.discarded_micro_batches == k * n_workers
    for r, o in zip(tr.records, ref.records):
        assert abs(r.grad_sq_estimate - o.grad_sq_estimate) <= 1e-4 * abs(o.grad_sq_estimate)


@pytest.mark.parametrize("method", ["dpu", "wp", "acco", "zero1"])
def test_run_continues_across_calls(cuda, method):
    """Trainer.run(3) + run(3) == one 6-update run: the optimizer step, round
    numbering (seeds) and the DPU/WP pending bundle carry over."""
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine", total_steps=6)
    sim = api.SimConfig(n_workers=2, batch_size=4, n_grad_accumulation=1, master_seed=21)
    model = api.Model(api.LMConfig(**MINI, precision="fp32", max_batch=8))
    th0 = model.default_theta0(sim.master_seed)
    t = api.Trainer(method, model, opt, sim)
    t.set_theta(th0)
    r1, h1, _, _ = t.run(3, history=True)
    r2, h2, _, _ = t.run(3, history=True)
    ref = _oracle(method, MINI, opt, sim, 6, theta0=th0.astype(np.float64))
    hist = np.concatenate([h1, h2])
    for i in range(6):
        assert _rel(hist[i, 0], ref.theta_history[i + 1]) <= 1e-5, i
        assert _rel(hist[i, 1], ref.estimate_history[i + 1]) <= 1e-5, i
    assert [r.samples_cum for r in r1 + r2] == [o.samples_cum for o in ref.records]


def test_heterogeneity_multipliers_throttle_one_worker(cuda):
    """HeterogeneityProfile (protocols.hpp:19-27): worker_multipliers become a
    measured per-worker throttle; the math is unchanged (floor schedule) and
    the slow worker's micro-batch intervals are ~m x longer on the timeline."""
    cfg = dict(vocab=64, d_model=64, n_layer=2, n_head=2, seq_len=32, n_samples=32, data_seed=3)
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine")
    base = api.SimConfig(n_workers=2, batch_size=4, n_grad_accumulation=2, master_seed=7)
    slow = api.SimConfig(n_workers=2, batch_size=4, n_grad_accumulation=2, master_seed=7, worker_multipliers=[4.0, 1.0])
    lm = api.LMConfig(**cfg, precision="fp32", max_batch=4)
    ta = api.run_protocol("acco", lm, opt, base, 3)
    tb = api.run_protocol("acco", lm, opt, slow, 3)
    for t in range(3):
        assert np.array_equal(ta.theta_history[t + 1], tb.theta_history[t + 1])

    def mb_time(tr, w):
        iv = [i for i in tr.timeline if i.stream == "compute" and i.worker == w and i.kind == "microbatch"]
        return sum(i.t_end - i.t_start for i in iv) / max(1, sum(i.micro_batches for i in iv))

    r = mb_time(tb, 0) / mb_time(tb, 1)
    assert 2.5 < r < 6.0, r
