"""Pin the CPU oracle restatement against the REFERENCE (CPU, no GPU).

tests/golden/*.json were produced by oracle/golden_dump.cpp linked against the
reference accosim library built from /root/reference sources (oracle/Makefile).
Integer work (rng, shards, counts) must be bit-exact; the fp64 restatement is
required to reproduce the reference's trajectories *bitwise* as well, because it
follows the reference's operation order.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import accosim_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_rng_derive_and_streams():
    g = load("rng.json")
    for m, a, b, c, d, out in g["derive"]:
        assert O.derive(m, a, b, c, d) == out
    for e in g["streams"]:
        s = O.Stream(e["seed"])
        assert [s.next_u64() for _ in range(8)] == e["next_u64"]
        assert [s.uniform01() for _ in range(8)] == e["uniform01"]
        assert [s.gaussian() for _ in range(8)] == e["gaussian"]
        assert [s.below(n) for n in (1, 2, 10, 256, 50257, 4096)] == e["below"]
        # the vectorised counter form agrees with the sequential stream
        blk = O.stream_u64_block(e["seed"], 0, 8)
        assert [int(x) for x in blk] == e["next_u64"]


def test_shard_partition():
    for c in load("shard.json"):
        assert [list(r) for r in O.shard_partition(c["dim"], c["n"])] == c["ranges"]
    with pytest.raises(ValueError):
        O.shard_partition(4, 0)


def test_scheduled_lr():
    for c in load("lr.json"):
        cfg = O.OptimizerConfig.from_dict(c["cfg"])
        assert [O.scheduled_lr(cfg, t) for t in range(110)] == c["lr"]


def test_opt_step_bitwise():
    for c in load("optim.json"):
        cfg = O.OptimizerConfig.from_dict(c["cfg"])
        st = O.OptimizerState.for_range(cfg, 0, len(c["theta0"]))
        th = np.array(c["theta0"])
        for s, g in enumerate(c["grads"]):
            st, th = O.opt_step(st, th, np.array(g), cfg)
            assert th.tolist() == c["thetas"][s]
            assert st.m.tolist() == c["m"][s]
            assert st.v.tolist() == c["v"][s]
        assert c["sharded_max_abs_diff"] == 0.0


def test_opt_step_validation():
    cfg = O.OptimizerConfig(kind="sgd", learning_rate=0.1)
    with pytest.raises(ValueError):
        O.opt_step(O.OptimizerState.for_range(cfg, 0, 2), np.ones(1), np.ones(2), cfg)
    with pytest.raises(ValueError):
        O.opt_step(O.OptimizerState.for_range(cfg, 0, 1), np.ones(1), np.array([np.inf]), cfg)


def test_fabric_bitwise():
    for c in load("fabric.json"):
        layout = O.shard_partition(c["dim"], c["n"])
        ins = [np.array(x) for x in c["inputs"]]
        assert O.all_reduce(ins).tolist() == c["all_reduce"]
        assert O.all_reduce_counts(c["counts"]) == c["all_reduce_counts"]
        rs = O.reduce_scatter(ins, layout)
        assert [r.tolist() for r in rs] == c["reduce_scatter"]
        ag = O.all_gather(rs, layout)
        assert ag.tolist() == c["all_gather"]
        assert ag.tolist() == c["all_reduce"]  # RS o AG == AR bitwise


def _run_golden_case(c):
    p = O.AnalyticProblem(c["problem"])
    cfg = O.OptimizerConfig.from_dict(c["optimizer"])
    s = c["sim"]
    sim = O.SimConfig(s["n_workers"], s["batch_size"], s["n_grad_accumulation"], s["full_batch_gradients"],
                      s["master_seed"], s.get("warmup_rounds", 0))
    theta0 = np.array(c["theta_history"][0])
    bs, fb = sim.batch_size, sim.full_batch_gradients

    def grad_fn(theta, stream):
        return p.stochastic_grad(theta, stream, bs, fb)

    if c["method"] == "acco":
        sched = O.schedule_from_records(c["records"])
        return O.run_acco(grad_fn, theta0, cfg, sim, c["t_updates"], schedule=sched,
                          eval_fn=p.value_and_grad, smoothness=p.smoothness, optimum=p.optimum)
    return O.run_method(c["method"], grad_fn, theta0, cfg, sim, c["t_updates"], eval_fn=p.value_and_grad,
                        smoothness=p.smoothness, optimum=p.optimum)


@pytest.mark.parametrize("name", [c["name"] for c in load("protocols.json")])
def test_protocol_trajectories_bitwise(name):
    c = next(c for c in load("protocols.json") if c["name"] == name)
    tr = _run_golden_case(c)
    assert len(tr.theta_history) == len(c["theta_history"])
    for t, (a, b) in enumerate(zip(tr.theta_history, c["theta_history"])):
        assert a.tolist() == b, f"theta differs at update {t}"
    for t, (a, b) in enumerate(zip(tr.estimate_history, c["estimate_history"])):
        assert a.tolist() == b, f"estimate differs at update {t}"
    for r, g in zip(tr.records, c["records"]):
        assert r.update == g["update"]
        assert r.samples_cum == g["samples_cum"]
        assert r.loss == g["loss"]
        assert r.grad_sq == g["grad_sq"]
        assert r.grad_sq_estimate == g["grad_sq_estimate"]
        assert r.lyapunov == g["lyapunov"]
    for a, b in zip(tr.consumed_mean_grad, c["consumed_mean_grad"]):
        assert a.tolist() == b
    assert sum(sum(r.mb_main) + sum(r.mb_estimate) for r in tr.records) == c["consumed"]
    assert c["issued"] == c["consumed"] + c["discarded"]
    if c["method"] != "acco":  # (acco replays the consumed schedule; its discards are not replayed)
        assert tr.issued_micro_batches == c["issued"]
    if c["method"] in ("dpu", "wp"):
        assert tr.discarded_micro_batches == c["discarded"]
        for r, g in zip(tr.records, c["records"]):
            assert r.mb_main == g["mb_main"] and r.mb_estimate == g["mb_estimate"]


@pytest.mark.parametrize("name", ["acco_logistic_adamw_k2", "acco_mlp_adam_warmup_k3", "acco_single_worker"])
def test_floor_schedule_matches_reference_under_free_comm(name):
    c = next(c for c in load("protocols.json") if c["name"] == name)
    s = c["sim"]
    sched = O.floor_schedule(c["t_updates"], s["n_workers"], s["n_grad_accumulation"])
    assert sched == O.schedule_from_records(c["records"])


def test_heterogeneous_steady_state_counts():
    # proj/tests/test_protocols.cpp:242-252 analogue recorded from the reference
    c = next(c for c in load("protocols.json") if c["name"] == "acco_mlp_hetero")
    for r in c["records"][3:]:
        assert r["mb_main"] == [4, 4, 4, 1]
        assert r["mb_estimate"] == [4, 4, 4, 1]


@pytest.mark.parametrize("name", [c["name"] for c in load("divergence.json")])
def test_divergence_semantics_match_reference(name):
    """Diverging runs (divergence.json, written by the reference): the partial
    trace, the diverged flag and the non-finite last loss of
    test_protocols.cpp:328-336 for every method; a non-finite theta0 raises
    the reference's exception type (invalid_argument -> ValueError,
    logic_error -> ProtocolLogicError)."""
    c = next(c for c in load("divergence.json") if c["name"] == name)
    if "throws" in c:
        exc = ValueError if c["throws"] == "invalid_argument" else O.ProtocolLogicError
        nan_case = {"ddp": ("ddp", 2), "acco": ("acco", 2)}[c["method"]]
        with pytest.raises(exc, match=c["what"]):
            O.check_theta0(nan_case[0], np.array([1.0, np.nan, 0.5]), nan_case[1])
        return
    tr = _run_golden_case(c)
    assert tr.diverged == c["diverged"] is True
    assert len(tr.records) == len(c["records"]) < c["t_updates"]
    for r, g in zip(tr.records, c["records"]):
        if g["loss"] is None:  # json null = the reference's non-finite loss
            assert not np.isfinite(r.loss)
        else:
            assert r.loss == g["loss"]
    assert not np.isfinite(tr.records[-1].loss)
    for a, b in zip(tr.theta_history, c["theta_history"]):
        assert [x if np.isfinite(x) else None for x in a.tolist()] == b


def test_nan_loss_under_eval_is_divergence():
    """An evaluated NaN loss ends the run (protocols.cpp:164-167: !isfinite);
    NaN only means "not evaluated" when the cadence skipped the update."""
    p = O.AnalyticProblem(next(c for c in load("divergence.json") if c["name"] == "ddp_identity_sgd1e8")["problem"])
    cfg = O.OptimizerConfig(kind="sgd", learning_rate=0.1)
    sim = O.SimConfig(1, 1, 1, False, 1)
    calls = []

    def eval_fn(theta):
        calls.append(1)
        return (float("nan") if len(calls) > 2 else 1.0), np.zeros_like(theta)

    tr = O.run_ddp(lambda th, s: p.stochastic_grad(th, s, 1, False), np.array([1.0]), cfg, sim, 10, eval_fn=eval_fn)
    assert tr.diverged and len(tr.records) == 2
    calls.clear()  # cadence 3: updates 2 (finite) and 5 (NaN) are evaluated, the rest carry NaN
    tr = O.run_ddp(lambda th, s: p.stochastic_grad(th, s, 1, False), np.array([1.0]), cfg, sim, 10, eval_fn=eval_fn,
                   eval_every=3)
    assert tr.diverged and len(tr.records) == 6
    assert np.isnan(tr.records[0].loss) and tr.records[2].loss == 1.0
