"""CPU restatement of the reference ACCO path — TEST INFRASTRUCTURE ONLY.

This module is the *checker* for the B200 library: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The product path (``paper_2406_02613_b200``) never calls it and fails loudly
without its CUDA library.

Restates, in fp64 with the reference's exact operation order (so trajectories
are bitwise equal on the reference's own problems, checked against
tests/golden/*.json produced by oracle/golden_dump.cpp from the reference):

  rng::splitmix64 / mix / derive / Stream     proj/include/accosim/rng.hpp:13-56
  shard_partition                             proj/include/accosim/shard.hpp:24-38
  scheduled_lr / opt_step / sharded_opt_step  proj/src/optim.cpp:37-119
  Fabric::{all_reduce,_counts,reduce_scatter,all_gather}  proj/src/collectives.cpp:36-91
  mean_over_samples + quadratic/logistic/mlp  proj/src/problems.cpp:103-192, 406-451
  make_batch / Bundle                         proj/src/protocols.cpp:56-82
  AccoEngine (phase algebra)                  proj/src/protocols.cpp:437-709
  SyncEngine::ddp_round                       proj/src/protocols.cpp:191-338
  TraceBuilder::commit (loss columns)         proj/src/protocols.cpp:107-169

The reference's discrete-event clock (simclock.cpp) is NOT restated: the
timing-dependent per-stage micro-batch counts are an *input* here — either the
floor-only schedule (exact under free comm and homogeneous workers, SURVEY.md
§7 "Hard parts") or a replay of counts logged by a run (reference or GPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional, Sequence

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

# ----------------------------------------------------------------------------- rng


def splitmix64_next(state: int):
    """rng.hpp:13-18; returns (output, new_state)."""
    state = (state + GOLDEN) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31), state


def mix(a: int, b: int) -> int:
    """rng.hpp:20-25."""
    h, _ = splitmix64_next(a & MASK64)
    s = h ^ ((b + GOLDEN + ((h << 6) & MASK64) + (h >> 2)) & MASK64)
    out, _ = splitmix64_next(s & MASK64)
    return out


def derive(master: int, a: int, b: int = 0, c: int = 0, d: int = 0) -> int:
    """rng.hpp:27-31."""
    return mix(mix(mix(mix(master & MASK64, a & MASK64), b & MASK64), c & MASK64), d & MASK64)


class Stream:
    """rng.hpp:33-56."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        out, self.state = splitmix64_next(self.state)
        return out

    def uniform01(self) -> float:
        return float((self.next_u64() >> 11) + 1) * 2.0 ** -53

    def gaussian(self) -> float:
        u1 = self.uniform01()
        u2 = self.uniform01()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * 3.14159265358979323846 * u2)

    def below(self, n: int) -> int:
        return self.next_u64() % n


def stream_u64_block(seed: int, start: int, count: int) -> np.ndarray:
    """Vectorised Stream(seed): draws start..start+count-1 (counter-based splitmix)."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & MASK64) + k * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform01_block(seed: int, start: int, count: int) -> np.ndarray:
    u = stream_u64_block(seed, start, count)
    return ((u >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53


def sample_indices(stream_seed: int, batch: int, n_samples: int) -> List[int]:
    """stochastic_grad's index draw (problems.cpp:442-444), with replacement."""
    s = Stream(stream_seed)
    return [s.below(n_samples) for _ in range(batch)]


# --------------------------------------------------------------------------- shards


def shard_partition(dim: int, n: int):
    """shard.hpp:24-38: remainder-first contiguous ranges [(lo, hi)]."""
    if n < 1:
        raise ValueError("shard_partition: need at least one worker")
    base, extra = divmod(dim, n)
    out, lo = [], 0
    for w in range(n):
        ln = base + (1 if w < extra else 0)
        out.append((lo, lo + ln))
        lo += ln
    return out


# ------------------------------------------------------------------------ optimizer


@dataclass
class OptimizerConfig:
    """optim.hpp:21-32 (defaults included)."""
    kind: str = "sgd"
    learning_rate: float = 0.0
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    weight_decay: float = 0.0
    scheduler: str = "constant"
    n_warmup_steps: int = 0
    total_steps: int = 0
    cosine_min_factor: float = 0.0

    @staticmethod
    def from_dict(d: dict) -> "OptimizerConfig":
        return OptimizerConfig(**{k: d[k] for k in OptimizerConfig.__dataclass_fields__ if k in d})


@dataclass
class OptimizerState:
    """optim.hpp:35-43."""
    step: int
    m: np.ndarray
    v: np.ndarray
    lo: int
    hi: int

    @staticmethod
    def for_range(cfg: OptimizerConfig, lo: int, hi: int) -> "OptimizerState":
        n = hi - lo
        return OptimizerState(0, np.zeros(n), np.zeros(n if cfg.kind != "sgd" else 0), lo, hi)

    def copy(self) -> "OptimizerState":
        return OptimizerState(self.step, self.m.copy(), self.v.copy(), self.lo, self.hi)


def scheduled_lr(cfg: OptimizerConfig, t: int) -> float:
    """optim.cpp:37-48."""
    peak = cfg.learning_rate
    warmup = cfg.n_warmup_steps
    if t < warmup:
        return peak * float(t + 1) / float(warmup)
    if cfg.scheduler == "constant":
        return peak
    floor = peak * cfg.cosine_min_factor
    span = cfg.total_steps - 1 - warmup
    if span <= 0:
        return peak
    x = float(t - warmup) / float(span)
    if x > 1.0:
        x = 1.0
    return floor + (peak - floor) * 0.5 * (1.0 + math.cos(3.14159265358979323846 * x))


def opt_step(state: OptimizerState, theta: np.ndarray, grad: np.ndarray, cfg: OptimizerConfig):
    """optim.cpp:50-92: pure transition; returns (new_state, new_theta)."""
    n = state.hi - state.lo
    if theta.shape[0] != n or grad.shape[0] != n:
        raise ValueError("opt_step: slice length mismatch")
    if not (np.all(np.isfinite(theta)) and np.all(np.isfinite(grad))):
        raise ValueError("opt_step: non-finite input")
    lr = scheduled_lr(cfg, state.step)
    st = state.copy()
    st.step += 1
    th = np.array(theta, dtype=np.float64, copy=True)
    if cfg.kind == "sgd":
        g = grad + cfg.weight_decay * th
        th -= lr * g
        return st, th
    b1, b2 = cfg.adam_beta1, cfg.adam_beta2
    corr1 = 1.0 - math.pow(b1, float(st.step))
    corr2 = 1.0 - math.pow(b2, float(st.step))
    g = np.array(grad, dtype=np.float64, copy=True)
    if cfg.kind == "adam":
        g = g + cfg.weight_decay * th
    st.m = b1 * st.m + (1.0 - b1) * g
    st.v = b2 * st.v + (1.0 - b2) * g * g
    m_hat = st.m / corr1
    v_hat = st.v / corr2
    update = m_hat / (np.sqrt(v_hat) + cfg.adam_eps)
    if cfg.kind == "adamw":
        update = update + cfg.weight_decay * th
    th = th - lr * update
    return st, th


def sharded_opt_step(states: List[OptimizerState], theta: np.ndarray, grad_shards, cfg, layout):
    """optim.cpp:94-119: per-worker opt_step on its shard, then all_gather."""
    if len(states) != len(layout) or len(grad_shards) != len(layout):
        raise ValueError("sharded_opt_step: layout/state mismatch")
    new_shards = []
    for w, (lo, hi) in enumerate(layout):
        st = states[w]
        if st.lo != lo or st.hi != hi:
            raise ValueError("sharded_opt_step: state covers wrong range")
        nxt, upd = opt_step(st, theta[lo:hi], grad_shards[w], cfg)
        states[w] = nxt
        new_shards.append(upd)
    return all_gather(new_shards, layout)


# ---------------------------------------------------------------------- collectives


def all_reduce(inputs: Sequence[np.ndarray]) -> np.ndarray:
    """collectives.cpp:36-46: ascending-worker sum."""
    out = np.array(inputs[0], dtype=np.float64, copy=True)
    for x in inputs[1:]:
        if x.shape != out.shape:
            raise ValueError("all_reduce: dimension mismatch")
        out += x
    return out


def all_reduce_counts(counts: Sequence[int]) -> int:
    return int(sum(counts))


def reduce_scatter(inputs: Sequence[np.ndarray], layout) -> List[np.ndarray]:
    """collectives.cpp:55-75: owner w gets sum over workers of [lo_w, hi_w)."""
    if len(inputs) != len(layout):
        raise ValueError("Fabric: expected one input per worker")
    out = []
    for lo, hi in layout:
        s = np.array(inputs[0][lo:hi], dtype=np.float64, copy=True)
        for x in inputs[1:]:
            s += x[lo:hi]
        out.append(s)
    return out


def all_gather(shards: Sequence[np.ndarray], layout) -> np.ndarray:
    """collectives.cpp:77-91."""
    dim = layout[-1][1] if layout else 0
    full = np.zeros(dim)
    for (lo, hi), s in zip(layout, shards):
        if len(s) != hi - lo:
            raise ValueError("all_gather: shard length mismatch")
        full[lo:hi] = s
    return full


# ------------------------------------------------------------------------- problems


def _dot_seq(a, b) -> float:
    s = 0.0
    for x, y in zip(a, b):
        s += x * y
    return s


class AnalyticProblem:
    """The reference's quadratic / logistic / mlp problems rebuilt from a golden
    dump (data arrays included) — protocol-parity fixtures only."""

    def __init__(self, d: dict):
        self.kind = d["kind"]
        self.dim = int(d["dim"])
        self.smoothness = d["smoothness"]
        self.noise_sigma = d.get("noise_sigma", 0.0)
        self.optimum = d.get("optimum")
        if self.kind == "quadratic":
            self.a = [list(map(float, d["a"][i * self.dim:(i + 1) * self.dim])) for i in range(self.dim)]
            self.b = list(map(float, d["b"]))
        else:
            self.n = int(d["n"])
            self.dim_x = int(d["dim_x"])
            self.x = [list(map(float, d["x"][k * self.dim_x:(k + 1) * self.dim_x])) for k in range(self.n)]
            self.y = list(map(float, d["y"]))
            self.n_in, self.hidden = int(d["n_in"]), int(d["hidden"])

    # problems.cpp:133-150
    def _eval_logistic(self, k, theta, grad):
        xk, yk = self.x[k], self.y[k]
        margin = _dot_seq(xk, theta)
        z = -yk * margin
        loss = z if z > 30.0 else math.log1p(math.exp(z))
        s = 1.0 / (1.0 + math.exp(-z))
        coef = -yk * s
        for j in range(self.dim_x):
            grad[j] += coef * xk[j]
        return loss

    # problems.cpp:152-192
    def _eval_mlp(self, k, theta, grad):
        h, ni = self.hidden, self.n_in
        xk = self.x[k]
        w1o, b1o, w2o = 0, h * ni, h * ni + h
        b2 = theta[w2o + h]
        out = b2
        z = [0.0] * h
        for i in range(h):
            s = theta[b1o + i]
            for j in range(ni):
                s += theta[w1o + i * ni + j] * xk[j]
            z[i] = math.tanh(s)
            out += theta[w2o + i] * z[i]
        err = out - self.y[k]
        grad[w2o + h] += err
        for i in range(h):
            zi = z[i]
            grad[w2o + i] += err * zi
            dz = err * theta[w2o + i] * (1.0 - zi * zi)
            grad[b1o + i] += dz
            for j in range(ni):
                grad[w1o + i * ni + j] += dz * xk[j]
        return 0.5 * err * err

    def _mean_over_samples(self, theta, idx):
        """problems.cpp:103-131: 64-sample chunks folded in order, then x 1/n."""
        theta = [float(t) for t in theta]
        n = len(idx)
        ev = self._eval_logistic if self.kind == "logistic" else self._eval_mlp
        grad = [0.0] * self.dim
        loss = 0.0
        for c in range(0, n, 64):
            g = [0.0] * self.dim
            lc = 0.0
            for i in range(c, min(n, c + 64)):
                lc += ev(idx[i], theta, g)
            for j in range(self.dim):
                grad[j] += 1.0 * g[j]
            loss += lc
        inv = 1.0 / float(n)
        return loss * inv, np.array([gj * inv for gj in grad])

    def value_and_grad(self, theta):
        """problems.cpp:406-417."""
        if self.kind == "quadratic":
            th = [float(t) for t in theta]
            at = [_dot_seq(row, th) for row in self.a]
            f = 0.5 * _dot_seq(th, at) - _dot_seq(self.b, th)
            return f, np.array([at[j] - self.b[j] for j in range(self.dim)])
        return self._mean_over_samples(theta, list(range(self.n)))

    def stochastic_grad(self, theta, stream: int, size: int, full_batch: bool):
        """problems.cpp:419-451 -> (mean_grad, sample_count, loss)."""
        if self.kind == "quadratic":
            f, g = self.value_and_grad(theta)
            if self.noise_sigma > 0.0:
                s = Stream(stream)
                g = np.array([gj + self.noise_sigma * s.gaussian() for gj in g])
            return g, size, f
        idx = list(range(self.n)) if full_batch else sample_indices(stream, size, self.n)
        loss, g = self._mean_over_samples(theta, idx)
        return g, len(idx), loss


# -------------------------------------------------------------------------- engines

TAG_INIT, TAG_MAIN, TAG_ESTIMATE = 1, 2, 3  # protocols.cpp:52-54


@dataclass
class SimConfig:
    """SimConfig (protocols.hpp:29-38) minus the simulated-time fields."""
    n_workers: int = 1
    batch_size: int = 1
    n_grad_accumulation: int = 1
    full_batch_gradients: bool = False
    master_seed: int = 1
    warmup_rounds: int = 0  # dpu: leading rounds with ddp semantics (protocols.hpp:33)


def make_batch_stream(sim: SimConfig, rnd: int, tag: int, worker: int, ordinal: int) -> int:
    """protocols.cpp:74-82."""
    return derive(sim.master_seed, worker, rnd, tag, ordinal)


class Bundle:
    """protocols.cpp:56-72: grad_sum += N * mean_grad; samples += N; micro += 1."""

    def __init__(self):
        self.grad_sum: Optional[np.ndarray] = None
        self.samples = 0
        self.micro = 0

    def add(self, grad: np.ndarray, count: int):
        if self.grad_sum is None:
            self.grad_sum = np.zeros(grad.shape[0])
        self.grad_sum += float(count) * grad
        self.samples += count
        self.micro += 1


GradFn = Callable[[np.ndarray, int], tuple]  # (theta, stream_seed) -> (mean_grad, count, loss)
EvalFn = Callable[[np.ndarray], tuple]       # theta -> (f, grad)


@dataclass
class Record:
    update: int
    loss: float
    grad_sq: float
    grad_sq_estimate: float
    lyapunov: Optional[float]
    samples_cum: int
    mb_main: List[int]
    mb_estimate: List[int]
    train_loss: float = float("nan")  # sample-weighted mean micro-batch loss (B200 addition)


@dataclass
class Trace:
    records: List[Record] = field(default_factory=list)
    theta_history: List[np.ndarray] = field(default_factory=list)
    estimate_history: List[np.ndarray] = field(default_factory=list)
    consumed_mean_grad: List[np.ndarray] = field(default_factory=list)
    issued_micro_batches: int = 0
    discarded_micro_batches: int = 0
    diverged: bool = False


def floor_schedule(t_updates: int, n_workers: int, k: int):
    """Per-update (mb_estimate[w], mb_main[w]) of the reference under a free
    fabric and homogeneous workers: round 0's estimate half is the 1-mb
    bootstrap, every other stage is exactly max(k, 1) micro-batches
    (protocols.cpp:542-573; test_protocols.cpp:216-228)."""
    k = max(k, 1)
    return [([1] * n_workers if t == 0 else [k] * n_workers, [k] * n_workers) for t in range(t_updates)]


class _Commit:
    """TraceBuilder::commit loss columns (protocols.cpp:107-169)."""

    def __init__(self, eval_fn: Optional[EvalFn], cfg: OptimizerConfig, smoothness=None,
                 optimum=None, eval_every: int = 1, lyapunov_eta: float = -1.0):
        self.eval_fn, self.cfg = eval_fn, cfg
        self.l, self.fstar = smoothness, optimum
        self.eval_every = eval_every
        self.eta = lyapunov_eta if lyapunov_eta > 0 else cfg.learning_rate
        self.samples_cum = 0

    def __call__(self, trace, update, theta, estimate, consumed, mb_main, mb_est, mean, train_loss):
        nan = float("nan")
        loss = gsq = gsq_e = nan
        lyap = None
        evaluated = False
        if not (np.all(np.isfinite(theta)) and np.all(np.isfinite(estimate))):
            # finite_state check (protocols.cpp:113-119): +inf whatever the cadence
            loss = gsq = gsq_e = float("inf")
            evaluated = True
        elif self.eval_fn is not None and self.eval_every > 0 and (update + 1) % self.eval_every == 0:
            evaluated = True
            loss, g = self.eval_fn(theta)
            le, ge = self.eval_fn(estimate)
            gsq = _dot_seq(g, g)
            gsq_e = _dot_seq(ge, ge)
            if self.fstar is not None:
                d = theta - estimate
                lyap = (loss - self.fstar) + self.eta * self.l * (le - self.fstar) + self.l * _dot_seq(d, d)
        self.samples_cum += consumed
        trace.records.append(Record(update, loss, gsq, gsq_e, lyap, self.samples_cum, list(mb_main),
                                    list(mb_est), train_loss))
        trace.theta_history.append(theta.copy())
        trace.estimate_history.append(estimate.copy())
        trace.consumed_mean_grad.append(mean)
        # NaN marks "not evaluated" under an eval cadence; an evaluated
        # non-finite loss (inf or NaN) is divergence (protocols.cpp:164-167)
        if evaluated and not math.isfinite(loss):
            trace.diverged = True
            return False
        return True


def _stage(grad_fn: GradFn, sim: SimConfig, params, w: int, rnd: int, tag: int, k: int, trace: Trace):
    b = Bundle()
    loss_sum = 0.0
    for j in range(k):
        g, n, loss = grad_fn(params, make_batch_stream(sim, rnd, tag, w, j))
        b.add(g, n)
        loss_sum += loss * n
        trace.issued_micro_batches += 1
    return b, loss_sum


def run_acco(grad_fn: GradFn, theta0: np.ndarray, cfg: OptimizerConfig, sim: SimConfig, t_updates: int,
             schedule=None, eval_fn: Optional[EvalFn] = None, smoothness=None, optimum=None,
             eval_every: int = 1) -> Trace:
    """AccoEngine's phase algebra (protocols.cpp:437-709) for a given per-update
    schedule [(mb_estimate[w], mb_main[w])]; default = floor schedule."""
    if cfg.total_steps == 0:
        cfg = replace(cfg, total_steps=t_updates)  # run_protocol, protocols.cpp:729
    n = sim.n_workers
    if schedule is None:
        schedule = floor_schedule(t_updates, n, sim.n_grad_accumulation)
    dim = theta0.shape[0]
    layout = shard_partition(dim, n)
    states = [OptimizerState.for_range(cfg, lo, hi) for lo, hi in layout]
    theta = np.array(theta0, dtype=np.float64, copy=True)
    estimate = theta.copy()
    trace = Trace()
    trace.theta_history.append(theta.copy())
    trace.estimate_history.append(estimate.copy())
    commit = _Commit(eval_fn, cfg, smoothness, optimum, eval_every)
    for t in range(t_updates):
        mb_est, mb_main = schedule[t]
        # ---- phase 2t: estimate (bundles computed at the previous estimate)
        est_b, est_loss = [], 0.0
        for w in range(n):
            if t == 0:
                b, ls = _stage(grad_fn, sim, theta0, w, 0, TAG_INIT, 1, trace)
            else:
                b, ls = _stage(grad_fn, sim, estimate, w, t, TAG_ESTIMATE, mb_est[w], trace)
            est_b.append(b)
            est_loss += ls
        total = all_reduce_counts([b.samples for b in est_b])
        shards = reduce_scatter([b.grad_sum for b in est_b], layout)
        retained, retained_total = [s.copy() for s in shards], total
        mean_shards = [s * (1.0 / float(total)) for s in shards]
        transient = [s.copy() for s in states]
        estimate = sharded_opt_step(transient, theta, mean_shards, cfg, layout)
        # ---- phase 2t+1: commit (bundles computed at theta^(t))
        main_b, main_loss = [], 0.0
        for w in range(n):
            b, ls = _stage(grad_fn, sim, theta, w, t, TAG_MAIN, mb_main[w], trace)
            main_b.append(b)
            main_loss += ls
        total = all_reduce_counts([b.samples for b in main_b])
        shards = reduce_scatter([b.grad_sum for b in main_b], layout)
        combined = total + retained_total
        mean_shards = []
        for s, e in zip(shards, retained):
            s = s + e
            mean_shards.append(s * (1.0 / float(combined)))
        theta = sharded_opt_step(states, theta, mean_shards, cfg, layout)
        mean_full = all_gather(mean_shards, layout)
        train_loss = (est_loss + main_loss) / combined
        mbm = [b.micro for b in main_b]
        mbe = [b.micro for b in est_b]
        if not commit(trace, t, theta, estimate, combined, mbm, mbe, mean_full, train_loss):
            break
    return trace


def run_ddp(grad_fn: GradFn, theta0: np.ndarray, cfg: OptimizerConfig, sim: SimConfig, t_updates: int,
            eval_fn: Optional[EvalFn] = None, smoothness=None, optimum=None, eval_every: int = 1) -> Trace:
    """SyncEngine::ddp_round + apply_and_commit (protocols.cpp:191-206, 298-338)."""
    if cfg.total_steps == 0:
        cfg = replace(cfg, total_steps=t_updates)
    n = sim.n_workers
    dim = theta0.shape[0]
    state = OptimizerState.for_range(cfg, 0, dim)
    theta = np.array(theta0, dtype=np.float64, copy=True)
    trace = Trace()
    trace.theta_history.append(theta.copy())
    trace.estimate_history.append(theta.copy())
    commit = _Commit(eval_fn, cfg, smoothness, optimum, eval_every)
    k = sim.n_grad_accumulation
    for r in range(t_updates):
        bundles, loss_sum = [], 0.0
        for w in range(n):
            b, ls = _stage(grad_fn, sim, theta, w, r, TAG_MAIN, k, trace)
            bundles.append(b)
            loss_sum += ls
        s = all_reduce([b.grad_sum for b in bundles])
        total = all_reduce_counts([b.samples for b in bundles])
        if total <= 0:
            raise RuntimeError("protocol: zero consumed samples")
        mean = s * (1.0 / float(total))
        if not np.all(np.isfinite(mean)):
            trace.diverged = True
            break
        state, theta = opt_step(state, theta, mean, cfg)
        if not commit(trace, r, theta, theta, total, [b.micro for b in bundles], [0] * n, mean,
                      loss_sum / total):
            break
    return trace


def _reduce_mean(bundles):
    """reduce_mean (protocols.cpp:191-206): AR of the sums, AR of the counts, x 1/total."""
    s = all_reduce([b.grad_sum for b in bundles])
    total = all_reduce_counts([b.samples for b in bundles])
    if total <= 0:
        raise RuntimeError("protocol: zero consumed samples")
    return s * (1.0 / float(total)), total


def _run_delayed(method: str, grad_fn: GradFn, theta0: np.ndarray, cfg: OptimizerConfig, sim: SimConfig,
                 t_updates: int, eval_fn: Optional[EvalFn] = None, smoothness=None, optimum=None,
                 eval_every: int = 1) -> Trace:
    """SyncEngine::dpu_round / wp_round (protocols.cpp:340-425), DPU's leading
    `warmup_rounds` as ddp_round (:235-238). One pending bundle per worker
    (computed in the previous round, or the Init-tag seed of :340-351) is
    consumed by each update; the last round's fresh bundles are discarded."""
    if cfg.total_steps == 0:
        cfg = replace(cfg, total_steps=t_updates)
    n = sim.n_workers
    dim = theta0.shape[0]
    state = OptimizerState.for_range(cfg, 0, dim)
    theta = np.array(theta0, dtype=np.float64, copy=True)
    estimate = theta.copy()
    trace = Trace()
    trace.theta_history.append(theta.copy())
    trace.estimate_history.append(estimate.copy())
    commit = _Commit(eval_fn, cfg, smoothness, optimum, eval_every)
    k = sim.n_grad_accumulation
    pending = None  # [(bundle, loss_sum)] per worker
    for r in range(t_updates):
        if method == "dpu" and r < sim.warmup_rounds:  # ddp_round
            fresh = [_stage(grad_fn, sim, theta, w, r, TAG_MAIN, k, trace) for w in range(n)]
            mean, total = _reduce_mean([b for b, _ in fresh])
            if not np.all(np.isfinite(mean)):
                trace.diverged = True
                break
            state, theta = opt_step(state, theta, mean, cfg)
            estimate = theta
            ok = commit(trace, r, theta, estimate, total, [b.micro for b, _ in fresh], [0] * n, mean,
                        sum(l for _, l in fresh) / total)
            if not ok:
                break
            continue
        if method == "dpu":
            if pending is None:  # seed_pending at the committed params
                pending = [_stage(grad_fn, sim, theta, w, r, TAG_INIT, 1, trace) for w in range(n)]
            params_for_compute = theta
            fresh = [_stage(grad_fn, sim, params_for_compute, w, r, TAG_MAIN, k, trace) for w in range(n)]
            consumed, pending = pending, fresh
            mean, total = _reduce_mean([b for b, _ in consumed])
            if not np.all(np.isfinite(mean)):
                trace.diverged = True
                break
            state, theta = opt_step(state, theta, mean, cfg)
            estimate = params_for_compute  # the applied gradients' params
        else:  # wp
            if pending is None:  # seed at the current prediction
                pending = [_stage(grad_fn, sim, estimate, w, r, TAG_INIT, 1, trace) for w in range(n)]
            consumed = pending
            mean, total = _reduce_mean([b for b, _ in consumed])
            if not np.all(np.isfinite(mean)):
                trace.diverged = True
                break
            state, theta = opt_step(state, theta, mean, cfg)
            _, estimate = opt_step(state.copy(), theta, mean, cfg)  # prediction on a throwaway copy
            pending = [_stage(grad_fn, sim, estimate, w, r, TAG_MAIN, k, trace) for w in range(n)]
        if not commit(trace, r, theta, estimate, total, [b.micro for b, _ in consumed], [0] * n, mean,
                      sum(l for _, l in consumed) / total):
            break
    trace.discarded_micro_batches = sum(b.micro for b, _ in pending) if pending else 0
    return trace


def run_dpu(grad_fn, theta0, cfg, sim, t_updates, **kw) -> Trace:
    return _run_delayed("dpu", grad_fn, theta0, cfg, sim, t_updates, **kw)


def run_wp(grad_fn, theta0, cfg, sim, t_updates, **kw) -> Trace:
    return _run_delayed("wp", grad_fn, theta0, cfg, sim, t_updates, **kw)


class ProtocolLogicError(RuntimeError):
    """std::logic_error of the reference (protocol invariants)."""


def check_theta0(method: str, theta0: np.ndarray, n_workers: int) -> None:
    """A non-finite theta0 fails where the reference first touches it: the
    synchronous rounds start with check_replicas (protocols.cpp:208-212,
    321-322; NaN != NaN across >= 2 replicas: logic_error), otherwise the first
    stochastic_grad's check_theta throws invalid_argument (problems.cpp:37-42)."""
    if np.all(np.isfinite(theta0)):
        return
    if method != "acco" and n_workers >= 2:
        raise ProtocolLogicError("protocol: parameter divergence across workers")
    raise ValueError("theta has non-finite entries")


def run_method(method: str, grad_fn, theta0, cfg, sim, t_updates, schedule=None, **kw) -> Trace:
    """run_protocol's dispatch (protocols.cpp:734-741)."""
    check_theta0(method, np.asarray(theta0), sim.n_workers)
    if method == "acco":
        return run_acco(grad_fn, theta0, cfg, sim, t_updates, schedule=schedule, **kw)
    if method in ("ddp", "zero1"):
        return run_ddp(grad_fn, theta0, cfg, sim, t_updates, **kw)
    if method in ("dpu", "wp"):
        return _run_delayed(method, grad_fn, theta0, cfg, sim, t_updates, **kw)
    raise ValueError(f"unknown method {method}")


def schedule_from_records(records) -> list:
    """Replay schedule from reference (golden) or GPU records."""
    return [(list(r["mb_estimate"]), list(r["mb_main"])) if isinstance(r, dict)
            else (list(r.mb_estimate), list(r.mb_main)) for r in records]
