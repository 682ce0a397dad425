"""Divergence and non-finite semantics of the GPU engine vs the reference
(ADVICE r01 / VERDICT r01 missing item 8). The reference's rules, pinned on
its own runs by tests/golden/divergence.json (tests/test_oracle_golden.py):

* a commit whose state is non-finite, or whose evaluated loss is non-finite,
  is recorded and ends the run: RunTrace.diverged, CLI exit 3
  (protocols.cpp:113-119,164-167);
* a synchronous round whose reduced mean is non-finite ends the run before
  its record (protocols.cpp:298-306);
* in ACCO a non-finite input to an optimizer step is opt_step's
  invalid_argument (optim.cpp:56-57): no trace, CLI exit 2;
* a non-finite theta0 is a logic_error (check_replicas, >= 2 workers of the
  synchronous family) or invalid_argument (stochastic_grad's check_theta)."""
import json

import numpy as np
import pytest

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import _lib, api
from paper_2406_02613_b200.__main__ import main

pytestmark = pytest.mark.gpu

MINI = dict(vocab=64, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3)


def _oracle(method, opt, sim, T, theta0):
    gc = G.GPTConfig(**MINI)
    prob = G.LMProblem(gc)
    ocfg = O.OptimizerConfig(**{k: getattr(opt, k) for k in O.OptimizerConfig.__dataclass_fields__})
    osim = O.SimConfig(sim.n_workers, sim.batch_size, sim.n_grad_accumulation, False, sim.master_seed)
    with np.errstate(all="ignore"):
        return O.run_method(method, lambda th, s: prob.stochastic_grad(th, s, sim.batch_size), theta0, ocfg, osim,
                            T, eval_fn=prob.value_and_grad)


@pytest.mark.parametrize("method", ["acco", "ddp", "zero1", "dpu"])
def test_exploding_run_is_a_partial_trace(cuda, method):
    """lr = 1e300: the first update's parameters overflow (fp32 on the GPU,
    the evaluated loss in fp64 on the oracle). Both record that update with a
    non-finite loss and stop: diverged after 1 of 6 updates."""
    opt = api.OptimizerConfig(kind="adamw", learning_rate=1e300, adam_beta2=0.95)
    sim = api.SimConfig(n_workers=2, batch_size=2, master_seed=5)
    tr = api.run_protocol(method, api.LMConfig(**MINI, precision="fp32", max_batch=2), opt, sim, 6)
    th0 = G.default_theta0(G.GPTConfig(**MINI), 5).astype(np.float32).astype(np.float64)
    ref = _oracle(method, opt, sim, 6, th0)
    assert tr.diverged and ref.diverged
    assert len(tr.records) == len(ref.records) == 1
    assert not np.isfinite(tr.records[-1].loss) and not np.isfinite(ref.records[-1].loss)
    assert tr.records[0].samples_cum == ref.records[0].samples_cum
    assert len(tr.theta_history) == 2  # theta0 + the diverged update


def test_wp_prediction_on_overflowed_theta_is_invalid(cuda):
    """WP: the commit step overflows theta in fp32; the prediction step then
    feeds it to opt_step, which is the reference's invalid_argument
    (protocols.cpp:398-403, optim.cpp:56-57)."""
    opt = api.OptimizerConfig(kind="adamw", learning_rate=1e300, adam_beta2=0.95)
    sim = api.SimConfig(n_workers=1, batch_size=2, master_seed=5)
    with pytest.raises(api.InvalidArgument, match="prediction step"):
        api.run_protocol("wp", api.LMConfig(**MINI, precision="fp32", max_batch=2), opt, sim, 6)


def test_eval_cadence_still_catches_a_non_finite_state(cuda):
    """With full-dataset evaluation only every 4 updates, the non-finite state
    still ends the run at the update that produced it (finite_state check)."""
    opt = api.OptimizerConfig(kind="adamw", learning_rate=1e300, adam_beta2=0.95)
    sim = api.SimConfig(n_workers=1, batch_size=2, master_seed=5, eval_every=4)
    tr = api.run_protocol("acco", api.LMConfig(**MINI, precision="fp32", max_batch=2), opt, sim, 6)
    assert tr.diverged and len(tr.records) == 1 and tr.records[0].loss == float("inf")


@pytest.mark.parametrize("method,n_workers,exc", [("acco", 2, api.InvalidArgument), ("acco", 1, api.InvalidArgument),
                                                  ("ddp", 2, api.LogicError), ("zero1", 2, api.LogicError),
                                                  ("ddp", 1, api.InvalidArgument)])
def test_non_finite_theta0(cuda, method, n_workers, exc):
    opt = api.OptimizerConfig(kind="adamw", learning_rate=1e-3)
    sim = api.SimConfig(n_workers=n_workers, batch_size=2, master_seed=1)
    lm = api.LMConfig(**MINI, precision="fp32", max_batch=2)
    m = api.Model(lm)
    th0 = m.default_theta0(1)
    th0[7] = np.nan
    with pytest.raises(exc):
        api.run_protocol(method, m, opt, sim, 3, theta0=th0)
    oexc = ValueError if exc is api.InvalidArgument else O.ProtocolLogicError
    with pytest.raises(oexc):
        O.check_theta0("acco" if method == "acco" else "ddp", th0.astype(np.float64), n_workers)


@pytest.mark.parametrize("method", ["acco", "ddp"])
def test_non_finite_gradient(cuda, method):
    """Finite but huge parameters overflow the forward pass, so the first
    gradients are non-finite: ACCO's optimizer step is the reference's
    invalid_argument; DDP ends before its first record (diverged)."""
    opt = api.OptimizerConfig(kind="adamw", learning_rate=1e-3)
    sim = api.SimConfig(n_workers=1, batch_size=2, master_seed=1)
    m = api.Model(api.LMConfig(**MINI, precision="fp32", max_batch=2))
    th0 = np.full(m.dim, 1e30, dtype=np.float32)
    if method == "acco":
        with pytest.raises(api.InvalidArgument, match="opt_step: non-finite input"):
            api.run_protocol("acco", m, opt, sim, 3, theta0=th0)
    else:
        tr = api.run_protocol("ddp", m, opt, sim, 3, theta0=th0)
        assert tr.diverged and len(tr.records) == 0


def test_cli_exit_codes_for_divergence(cuda, tmp_path):
    cfg = {"problem": {"kind": "gpt", **{k: v for k, v in MINI.items() if k != "data_seed"}, "seed": 3,
                       "precision": "fp32"},
           "method_name": "acco", "optimizer": {"kind": "adamw", "learning_rate": 1e300},
           "n_workers": 1, "batch_size": 2, "t_updates": 4, "master_seed": 5}
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    out = tmp_path / "out"
    assert main(["run", "--config", str(path), "--out", str(out)]) == 3  # accosim exit 3
    rows = (out / "metrics.csv").read_text().splitlines()[1:]
    assert len(rows) == 1 and rows[0].split(",")[3] == "inf"
    m = json.loads((out / "manifest.json").read_text())
    assert m["diverged"] is True and m["updates"] == 1
    _lib.lib()  # library still usable
