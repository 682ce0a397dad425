"""Python host mirror of the reference trainer API over the C-ABI.

Mirrors, with the same names, argument meaning and error behaviour:
  OptimizerConfig / scheduled_lr        proj/include/accosim/optim.hpp:21-64
  SimConfig                             proj/include/accosim/protocols.hpp:29-38
  run_protocol -> RunTrace              proj/include/accosim/protocols.hpp:61-90
  parse_config (JSON schema)            proj/src/config.cpp:80-133
  shard_partition                       proj/include/accosim/shard.hpp:24-38
with the B200 additions: problem kind "gpt" (the LM plugin), precision,
schedule (floor / adaptive / replay), eval cadence, and NCCL multi-GPU via
:class:`Comm` (one process per GPU).

Errors: the reference's std::invalid_argument -> :class:`InvalidArgument`
(a ValueError), std::logic_error -> :class:`LogicError`; divergence is data
(``RunTrace.diverged``), as in the reference.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import AccoError, InvalidArgument, LogicError  # noqa: F401

METHODS = {"ddp": 0, "dpu": 1, "wp": 2, "acco": 3, "zero1": 4}
KINDS = {"sgd": 0, "adam": 1, "adamw": 2}
SCHEDULES = {"floor": 0, "adaptive": 1, "replay": 2}


class LMCfgC(C.Structure):
    _fields_ = [("vocab", C.c_int), ("d_model", C.c_int), ("n_layer", C.c_int), ("n_head", C.c_int),
                ("seq_len", C.c_int), ("n_samples", C.c_int), ("data_seed", C.c_uint64),
                ("precision", C.c_int), ("max_batch", C.c_int), ("host_data", C.c_int), ("arch", C.c_int),
                ("n_kv_head", C.c_int), ("d_ff", C.c_int), ("rope_base", C.c_double)]


class SimCfgC(C.Structure):
    _fields_ = [("n_workers", C.c_int), ("batch_size", C.c_int), ("n_grad_accumulation", C.c_int),
                ("warmup_rounds", C.c_int), ("master_seed", C.c_uint64), ("schedule", C.c_int),
                ("replay", C.POINTER(C.c_int32)), ("replay_len", C.c_int), ("eval_every", C.c_int),
                ("eval_batch", C.c_int), ("throttle_ns", C.POINTER(C.c_double)), ("comm_delay_ns", C.c_double),
                ("check_replicas", C.c_int), ("throttle_host", C.c_int), ("comm_standin_ctas", C.c_int),
                ("comm_standin_bytes", C.c_double)]


class RecordC(C.Structure):
    _fields_ = [("update", C.c_int), ("time_s", C.c_double), ("loss", C.c_double), ("grad_sq", C.c_double),
                ("grad_sq_estimate", C.c_double), ("lyapunov", C.c_double), ("samples_cum", C.c_longlong),
                ("train_loss", C.c_double)]


class StatsC(C.Structure):
    _fields_ = [("issued_micro_batches", C.c_longlong), ("consumed_micro_batches", C.c_longlong),
                ("discarded_micro_batches", C.c_longlong), ("wall_ms", C.c_double),
                ("compute_busy_ms", C.c_double), ("comm_busy_ms", C.c_double), ("comm_exposed_ms", C.c_double),
                ("opt_ms", C.c_double), ("opt_launches", C.c_int), ("diverged", C.c_int),
                ("h2d_bytes", C.c_longlong), ("d2h_bytes", C.c_longlong), ("n_records", C.c_int)]


class IntervalC(C.Structure):
    _fields_ = [("worker_id", C.c_int), ("stream", C.c_int), ("kind", C.c_int), ("micro_batches", C.c_int),
                ("t_start", C.c_double), ("t_end", C.c_double), ("bytes", C.c_longlong)]


IV_KINDS = ("init_grad", "microbatch", "all_reduce", "reduce_scatter", "optimizer", "all_gather")

_P = C.c_void_p
_lib.register({
    "acco_trainer_timeline": (C.c_int, [_P, C.POINTER(IntervalC), C.c_int, C.POINTER(C.c_int)]),
    "acco_peer_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "acco_peer_destroy": (C.c_int, [_P]),
    "acco_trainer_peer_blob_bytes": (C.c_longlong, [_P]),
    "acco_trainer_peer_export": (C.c_int, [_P, _P]),
    "acco_trainer_peer_connect": (C.c_int, [_P, _P]),
    "acco_model_create": (C.c_int, [C.POINTER(LMCfgC), C.POINTER(C.c_void_p)]),
    "acco_model_destroy": (C.c_int, [_P]),
    "acco_model_num_params": (C.c_longlong, [_P]),
    "acco_model_theta0": (C.c_int, [_P, C.c_uint64, _P]),
    "acco_model_dataset": (C.c_int, [_P, _P]),
    "acco_model_stochastic_grad": (C.c_int, [_P, _P, C.c_uint64, C.c_int, _P, _P, _P]),
    "acco_model_value_and_grad": (C.c_int, [_P, _P, C.POINTER(C.c_double), _P, _P]),
    "acco_model_time_micro_batch": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "acco_trainer_create": (C.c_int, [_P, C.POINTER(_lib.OptCfg), C.POINTER(SimCfgC), C.c_int, _P,
                                      C.POINTER(C.c_void_p)]),
    "acco_trainer_create_peer": (C.c_int, [_P, C.POINTER(_lib.OptCfg), C.POINTER(SimCfgC), C.c_int, _P,
                                           C.POINTER(C.c_void_p)]),
    "acco_trainer_destroy": (C.c_int, [_P]),
    "acco_trainer_set_theta": (C.c_int, [_P, _P]),
    "acco_trainer_get_theta": (C.c_int, [_P, C.c_int, _P]),
    "acco_trainer_run": (C.c_int, [_P, C.c_int, C.POINTER(RecordC), _P, _P, C.POINTER(StatsC)]),
    "acco_trainer_n_local": (C.c_int, [_P]),
})


# ------------------------------------------------------------------ optimizer
@dataclass
class OptimizerConfig:
    """optim.hpp:21-32 (same defaults)."""
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

    def to_c(self) -> _lib.OptCfg:
        if self.kind not in KINDS:
            raise InvalidArgument(_lib.INVALID, f"unknown optimizer kind: {self.kind}")
        if self.scheduler not in ("constant", "cosine"):
            raise InvalidArgument(_lib.INVALID, "config: scheduler must be constant or cosine")
        return _lib.OptCfg(KINDS[self.kind], self.learning_rate, self.adam_beta1, self.adam_beta2, self.adam_eps,
                           self.weight_decay, 1 if self.scheduler == "cosine" else 0, self.n_warmup_steps,
                           self.total_steps, self.cosine_min_factor)


def scheduled_lr(cfg: OptimizerConfig, t: int) -> float:
    """optim.cpp:37-48, evaluated by the library."""
    c = cfg.to_c()
    return _lib.lib().acco_scheduled_lr(C.byref(c), t)


def shard_partition(dim: int, n: int):
    """shard.hpp:24-38 via the library (bit-exact integer layout)."""
    if n < 1:
        raise InvalidArgument(_lib.INVALID, "shard_partition: need at least one worker")
    lo = (C.c_uint64 * n)()
    hi = (C.c_uint64 * n)()
    _lib.call("acco_shard_partition", dim, n, lo, hi)
    return [(int(lo[i]), int(hi[i])) for i in range(n)]


def sample_indices(stream_seed: int, batch: int, n_samples: int) -> List[int]:
    out = (C.c_int32 * batch)()
    _lib.call("acco_sample_indices", C.c_uint64(stream_seed), batch, n_samples, out)
    return list(out)


def derive(master: int, a: int, b: int = 0, c: int = 0, d: int = 0) -> int:
    return int(_lib.lib().acco_rng_derive(*(C.c_uint64(x & (2**64 - 1)) for x in (master, a, b, c, d))))


def launch_count() -> int:
    """Kernel launches issued by this library so far (process-wide)."""
    return int(_lib.lib().acco_launch_count())


PROF_CLASSES = ("gemm", "attention", "optimizer", "column_reduce", "layernorm", "cross_entropy", "embedding", "other")


def prof_enable(on: bool = True):
    _lib.lib().acco_prof_enable(int(on))
    if on:
        _lib.call("acco_prof_reset")


def prof_read() -> dict:
    """Per-class kernel time (CUDA events on the launching stream), work
    (algorithmic flops for gemm/attention, bytes for the optimizer), launches."""
    k = len(PROF_CLASSES)
    ms = (C.c_double * k)()
    work = (C.c_double * k)()
    n = (C.c_longlong * k)()
    _lib.call("acco_prof_read", ms, work, n)
    return {c: {"ms": ms[i], "work": work[i], "launches": int(n[i])} for i, c in enumerate(PROF_CLASSES)}


# ---------------------------------------------------------------------- model
@dataclass(frozen=True)
class LMConfig:
    """problem.kind == "gpt" (B200 addition to config.cpp's problem block)."""
    vocab: int = 256
    d_model: int = 128
    n_layer: int = 2
    n_head: int = 4
    seq_len: int = 64
    n_samples: int = 256
    data_seed: int = 1
    precision: str = "fp32"  # "fp32" (parity) or "bf16" (throughput)
    max_batch: int = 8
    host_data: bool = False  # data-loader path: per-micro-batch H2D of token rows
    arch: str = "gpt2"       # "gpt2" | "llama" (RMSNorm, RoPE, GQA, SwiGLU, untied head)
    n_kv_head: int = 0       # llama: KV heads (0 -> n_head)
    d_ff: int = 0            # llama: SwiGLU hidden (0 -> 4 * d_model)
    rope_base: float = 10000.0

    def to_c(self) -> LMCfgC:
        if self.precision not in ("fp32", "bf16"):
            raise InvalidArgument(_lib.INVALID, "lm config: precision must be fp32 or bf16")
        if self.arch not in ("gpt2", "llama"):
            raise InvalidArgument(_lib.INVALID, "lm config: arch must be gpt2 or llama")
        return LMCfgC(self.vocab, self.d_model, self.n_layer, self.n_head, self.seq_len, self.n_samples,
                      self.data_seed, 1 if self.precision == "bf16" else 0, self.max_batch, int(self.host_data),
                      1 if self.arch == "llama" else 0, self.n_kv_head, self.d_ff, float(self.rope_base))


class Model:
    """The LM plugin (owns device weights workspace and the token dataset)."""

    def __init__(self, cfg: LMConfig):
        self.cfg = cfg
        self._h = C.c_void_p()
        c = cfg.to_c()
        _lib.call("acco_model_create", C.byref(c), C.byref(self._h))
        self.dim = int(_lib.lib().acco_model_num_params(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().acco_model_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def time_micro_batch(self, batch: int, reps: int = 3) -> float:
        """Device time (ns) of one micro-batch of `batch` samples."""
        out = C.c_double()
        _lib.call("acco_model_time_micro_batch", self._h, batch, reps, C.byref(out))
        return out.value

    def default_theta0(self, master_seed: int) -> np.ndarray:
        out = np.empty(self.dim, dtype=np.float32)
        _lib.call("acco_model_theta0", self._h, C.c_uint64(master_seed), out.ctypes.data_as(C.c_void_p))
        return out

    def dataset(self) -> np.ndarray:
        out = np.empty((self.cfg.n_samples, self.cfg.seq_len + 1), dtype=np.int32)
        _lib.call("acco_model_dataset", self._h, out.ctypes.data_as(C.c_void_p))
        return out


# ---------------------------------------------------------------------- comm
class Comm:
    """NCCL communicator for one rank (one process per GPU). The unique id is
    exchanged over an existing torch.distributed group (any backend)."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist

        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _lib.call("acco_comm_unique_id", uid)
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        self._h = C.c_void_p()
        _lib.call("acco_comm_init_rank", world, rank, uid, device, C.byref(self._h))
        self.rank, self.world = rank, world

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().acco_comm_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h


class PeerComm:
    """Peer fabric for one rank (one process per GPU of one box): the comm
    phase as one fused kernel over NVLink peer memory (include/acco.h,
    csrc/peer.h) instead of NCCL. The IPC handles of every rank's buffers are
    all-gathered over an existing torch.distributed group when a Trainer is
    created on it."""

    kind = "peer"

    def __init__(self, rank: int, world: int, device: int, group=None):
        self._h = C.c_void_p()
        _lib.call("acco_peer_create", world, rank, device, C.byref(self._h))
        self.rank, self.world, self.group = rank, world, group

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().acco_peer_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def connect(self, trainer_handle) -> None:
        n = _lib.lib().acco_trainer_peer_blob_bytes(trainer_handle)
        blob = (C.c_ubyte * n)()
        _lib.call("acco_trainer_peer_export", trainer_handle, blob)
        if self.world > 1:
            import torch.distributed as dist

            parts = [None] * self.world
            dist.all_gather_object(parts, bytes(blob), group=self.group)
        else:
            parts = [bytes(blob)]
        allb = (C.c_ubyte * (n * self.world)).from_buffer_copy(b"".join(parts))
        _lib.call("acco_trainer_peer_connect", trainer_handle, allb)


# --------------------------------------------------------------------- trainer
@dataclass
class SimConfig:
    """protocols.hpp:29-38 (cost model / simulated time replaced by real
    streams), plus B200 execution keys."""
    n_workers: int = 1
    batch_size: int = 1
    n_grad_accumulation: int = 1
    warmup_rounds: int = 0
    full_batch_gradients: bool = False
    master_seed: int = 1
    worker_multipliers: Optional[Sequence[float]] = None
    # B200 keys
    schedule: str = "floor"
    replay: Optional[Sequence] = None  # [(mb_estimate[w], mb_main[w])] per update
    eval_every: int = 1
    eval_batch: int = 0
    throttle_ns: Optional[Sequence[float]] = None
    comm_delay_ns: float = 0.0  # emulated interconnect time per comm phase (single-GPU overlap study)
    check_replicas: bool = False  # debug: cross-rank replica checksum after every comm phase
    throttle_host: bool = False   # straggler by host sleep after each micro-batch (the paper's time.sleep)
    comm_standin_ctas: int = 0    # emulated interconnect: paced HBM copy on this many CTAs (0 = 1-thread spin)
    comm_standin_bytes: float = 0.0


@dataclass
class RoundRecord:
    """protocols.hpp:41-53 (+ train_loss)."""
    update: int
    time_s: float
    loss: float
    grad_sq: float
    grad_sq_estimate: float
    lyapunov: float
    samples_cum: int
    mb_main: List[int]
    mb_estimate: List[int]
    train_loss: float
    idle_frac: List[float] = field(default_factory=list)  # compute-stream idle per worker this window

    @property
    def micro_batches(self):
        return [a + b for a, b in zip(self.mb_main, self.mb_estimate)]


@dataclass
class RunTrace:
    """protocols.hpp:61-76."""
    records: List[RoundRecord] = field(default_factory=list)
    diverged: bool = False
    theta_history: List[np.ndarray] = field(default_factory=list)
    estimate_history: List[np.ndarray] = field(default_factory=list)
    issued_micro_batches: int = 0
    consumed_micro_batches: int = 0
    discarded_micro_batches: int = 0
    stats: dict = field(default_factory=dict)
    timeline: list = field(default_factory=list)  # csvio.Interval rows, CUDA-event times


class Trainer:
    def __init__(self, method: str, model: Model, opt: OptimizerConfig, sim: SimConfig, comm: Optional[Comm] = None):
        if method not in METHODS:
            raise InvalidArgument(_lib.INVALID, f"unknown method: {method}")
        if sim.full_batch_gradients:
            raise InvalidArgument(_lib.INVALID, "full_batch_gradients is not supported for the LM problem")
        if sim.worker_multipliers is not None and len(sim.worker_multipliers) != sim.n_workers:
            raise InvalidArgument(_lib.INVALID, "run_protocol: one multiplier per worker")
        self.method, self.model, self.opt, self.sim, self.comm = method, model, opt, sim, comm
        self._replay = None
        rp, rl = None, 0
        if sim.replay is not None:
            flat = []
            for est, main in sim.replay:
                flat += list(est) + list(main)
            self._replay = (C.c_int32 * len(flat))(*flat)
            rp, rl = self._replay, len(flat)
        self._thr = None
        thr = sim.throttle_ns
        if thr is None and sim.worker_multipliers is not None and any(m != 1.0 for m in sim.worker_multipliers):
            # HeterogeneityProfile (protocols.hpp:19-27): worker w's micro-batch lasts
            # m_w x the base time; on the GPU the slow worker spins (m_w - 1) x the
            # measured micro-batch time after each micro-batch (m_w < 1: no speed-up)
            t = model.time_micro_batch(sim.batch_size)
            thr = [max(0.0, m - 1.0) * t for m in sim.worker_multipliers]
        if thr is not None:
            self._thr = (C.c_double * sim.n_workers)(*thr)
        self.throttle_ns = thr
        s = SimCfgC(sim.n_workers, sim.batch_size, sim.n_grad_accumulation, sim.warmup_rounds, sim.master_seed,
                    SCHEDULES[sim.schedule], rp, rl, sim.eval_every, sim.eval_batch, self._thr,
                    float(sim.comm_delay_ns), int(sim.check_replicas), int(sim.throttle_host),
                    int(sim.comm_standin_ctas), float(sim.comm_standin_bytes))
        o = opt.to_c()
        self._h = C.c_void_p()
        if isinstance(comm, PeerComm):
            _lib.call("acco_trainer_create_peer", model.handle, C.byref(o), C.byref(s), METHODS[method],
                      comm.handle, C.byref(self._h))
            comm.connect(self._h)
        else:
            _lib.call("acco_trainer_create", model.handle, C.byref(o), C.byref(s), METHODS[method],
                      comm.handle if comm is not None else None, C.byref(self._h))
        self.n_local = _lib.lib().acco_trainer_n_local(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().acco_trainer_destroy(h)
            self._h = None

    def set_theta(self, theta: np.ndarray):
        th = np.ascontiguousarray(theta, dtype=np.float32)
        if th.shape != (self.model.dim,):
            raise InvalidArgument(_lib.INVALID, "run_protocol: theta0 dimension mismatch")
        _lib.call("acco_trainer_set_theta", self._h, th.ctypes.data_as(C.c_void_p))

    def theta(self, which: int = 0) -> np.ndarray:
        n = self.model.dim
        out = np.empty(n, dtype=np.float32)
        _lib.call("acco_trainer_get_theta", self._h, which, out.ctypes.data_as(C.c_void_p))
        return out

    def run(self, t_updates: int, history: bool = False):
        recs = (RecordC * t_updates)()
        nl = self.n_local
        counts = np.zeros((t_updates, 2, nl), dtype=np.int32)
        hist = np.zeros((t_updates, 2, self.model.dim), dtype=np.float32) if history else None
        st = StatsC()
        rc = _lib.lib().acco_trainer_run(self._h, t_updates, recs, counts.ctypes.data_as(C.c_void_p),
                                         hist.ctypes.data_as(C.c_void_p) if history else None, C.byref(st))
        diverged = rc == _lib.DIVERGED
        if rc not in (_lib.OK, _lib.DIVERGED):
            _lib.check(rc)
        # a diverged run keeps the records up to the divergence (the
        # reference's partial RunTrace, protocols.cpp:164-167)
        n_rec = st.n_records
        if hist is not None:
            hist = hist[:n_rec]
        out = []
        for i in range(n_rec):
            r = recs[i]
            out.append(RoundRecord(r.update, r.time_s, r.loss, r.grad_sq, r.grad_sq_estimate, r.lyapunov,
                                   r.samples_cum, counts[i, 1].tolist(), counts[i, 0].tolist(), r.train_loss))
        stats = {k: getattr(st, k) for k, _ in StatsC._fields_}
        return out, hist, stats, diverged

    def timeline(self):
        """timeline.csv rows of the last run() (CUDA-event times, seconds)."""
        from .csvio import Interval

        n = C.c_int(0)
        _lib.call("acco_trainer_timeline", self._h, None, 0, C.byref(n))
        buf = (IntervalC * max(n.value, 1))()
        _lib.call("acco_trainer_timeline", self._h, buf, n.value, C.byref(n))
        return [Interval(b.worker_id, "comm" if b.stream else "compute", IV_KINDS[b.kind], b.t_start, b.t_end,
                         b.micro_batches, b.bytes) for b in buf[:n.value]]


def run_protocol(method: str, problem, opt_cfg: OptimizerConfig, sim: SimConfig, t_updates: int,
                 theta0: Optional[np.ndarray] = None, comm: Optional[Comm] = None,
                 record_history: bool = True) -> RunTrace:
    """protocols.hpp:89-90 / protocols.cpp:713-742 on B200."""
    if t_updates < 1:
        raise InvalidArgument(_lib.INVALID, "run_protocol: t_updates >= 1")
    if sim.n_workers < 1:
        raise InvalidArgument(_lib.INVALID, "run_protocol: n_workers >= 1")
    if sim.batch_size < 1:
        raise InvalidArgument(_lib.INVALID, "run_protocol: batch_size >= 1")
    if sim.n_grad_accumulation < 1:
        raise InvalidArgument(_lib.INVALID, "run_protocol: n_grad_accumulation >= 1")
    if sim.warmup_rounds < 0:
        raise InvalidArgument(_lib.INVALID, "run_protocol: warmup_rounds >= 0")
    if sim.worker_multipliers is not None:
        if len(sim.worker_multipliers) != sim.n_workers:
            raise InvalidArgument(_lib.INVALID, "run_protocol: one multiplier per worker")
        if any(not (m > 0.0) for m in sim.worker_multipliers):
            raise InvalidArgument(_lib.INVALID, "run_protocol: multipliers > 0")
    if not (opt_cfg.learning_rate > 0.0):
        raise InvalidArgument(_lib.INVALID, "run_protocol: learning_rate > 0")
    if opt_cfg.total_steps == 0:
        opt_cfg = OptimizerConfig(**{**opt_cfg.__dict__, "total_steps": t_updates})
    model = problem if isinstance(problem, Model) else Model(problem)
    th0 = model.default_theta0(sim.master_seed) if theta0 is None else np.asarray(theta0, dtype=np.float32)
    if th0.shape != (model.dim,):
        raise InvalidArgument(_lib.INVALID, "run_protocol: theta0 dimension mismatch")
    tr = Trainer(method, model, opt_cfg, sim, comm)
    tr.set_theta(th0)
    recs, hist, stats, diverged = tr.run(t_updates, history=record_history)
    out = RunTrace(records=recs, diverged=diverged, stats=stats, timeline=tr.timeline())
    _fill_idle(out, sim, comm)
    out.issued_micro_batches = stats["issued_micro_batches"]
    out.consumed_micro_batches = stats["consumed_micro_batches"]
    out.discarded_micro_batches = stats["discarded_micro_batches"]
    if record_history:
        out.theta_history = [th0.copy()] + [hist[t, 0].copy() for t in range(len(recs))]
        out.estimate_history = [th0.copy()] + [hist[t, 1].copy() for t in range(len(recs))]
    return out


def _fill_idle(trace: RunTrace, sim: SimConfig, comm) -> None:
    """RoundRecord.idle_frac for every worker (NCCL mode: gathered from the ranks)."""
    from .csvio import idle_fractions

    if comm is None:
        rows = idle_fractions(trace.records, trace.timeline, range(sim.n_workers))
    elif comm.world == 1:
        rows = idle_fractions(trace.records, trace.timeline, [comm.rank])
    else:
        import torch.distributed as dist

        mine = idle_fractions(trace.records, trace.timeline, [comm.rank])
        allr = [None] * comm.world
        dist.all_gather_object(allr, [r[0] for r in mine])
        rows = [[allr[w][t] for w in range(comm.world)] for t in range(len(trace.records))]
    for r, row in zip(trace.records, rows):
        r.idle_frac = row


# ---------------------------------------------------------------------- config
@dataclass
class ExperimentConfig:
    """config.hpp:13-27."""
    problem: LMConfig
    method: str
    optimizer: OptimizerConfig
    sim: SimConfig
    t_updates: int
    output_dir: str = ""
    raw: dict = field(default_factory=dict)


def _get(j, k, default):
    return j[k] if k in j else default


def _req(j, k):
    if k not in j:
        raise InvalidArgument(_lib.INVALID, f"config: missing key '{k}'")
    return j[k]


def parse_config(j: dict) -> ExperimentConfig:
    """config.cpp:80-133 (same keys, defaults and validation); problem.kind
    must be "gpt" or "llama" on the B200 path (the analytic problems are CPU
    fixtures); "llama" adds n_kv_head, d_ff, rope_base."""
    p = _req(j, "problem")
    kind = _req(p, "kind")
    if kind not in ("gpt", "llama"):
        raise InvalidArgument(_lib.INVALID, f"unknown problem kind for the B200 path: {kind}")
    prob = LMConfig(vocab=_get(p, "vocab", 256), d_model=_get(p, "d_model", 128), n_layer=_get(p, "n_layer", 2),
                    n_head=_get(p, "n_head", 4), seq_len=_get(p, "seq_len", 64), n_samples=_get(p, "n_samples", 256),
                    data_seed=_get(p, "seed", 1), precision=_get(p, "precision", "fp32"),
                    max_batch=max(_get(j, "batch_size", 1), _get(p, "max_batch", 1)),
                    arch="llama" if kind == "llama" else "gpt2", n_kv_head=_get(p, "n_kv_head", 0),
                    d_ff=_get(p, "d_ff", 0), rope_base=_get(p, "rope_base", 10000.0))
    method = _req(j, "method_name")
    if method not in METHODS:
        raise InvalidArgument(_lib.INVALID, f"unknown method: {method}")
    o = _req(j, "optimizer")
    kind = _req(o, "kind")
    if kind not in KINDS:
        raise InvalidArgument(_lib.INVALID, f"unknown optimizer kind: {kind}")
    opt = OptimizerConfig(kind=kind, learning_rate=_req(o, "learning_rate"), weight_decay=_get(o, "weight_decay", 0.0),
                          adam_beta1=_get(o, "adam_beta1", 0.9), adam_beta2=_get(o, "adam_beta2", 0.999),
                          adam_eps=_get(o, "adam_eps", 1e-8), scheduler=_get(o, "scheduler", "constant"),
                          n_warmup_steps=_get(o, "n_warmup_steps", 0),
                          cosine_min_factor=_get(o, "cosine_min_factor", 0.0))
    if opt.scheduler not in ("constant", "cosine"):
        raise InvalidArgument(_lib.INVALID, "config: scheduler must be constant or cosine")
    if not (opt.learning_rate > 0.0):
        raise InvalidArgument(_lib.INVALID, "config: learning_rate > 0")
    if not (0.0 <= opt.adam_beta1 < 1.0 and 0.0 <= opt.adam_beta2 < 1.0):
        raise InvalidArgument(_lib.INVALID, "config: adam betas must lie in [0, 1)")
    if opt.weight_decay < 0.0:
        raise InvalidArgument(_lib.INVALID, "config: weight_decay >= 0")
    if opt.n_warmup_steps < 0:
        raise InvalidArgument(_lib.INVALID, "config: n_warmup_steps >= 0")
    sim = SimConfig(n_workers=_get(j, "n_workers", 1), batch_size=_get(j, "batch_size", 1),
                    n_grad_accumulation=_get(j, "n_grad_accumulation", 1), warmup_rounds=_get(j, "warmup_rounds", 0),
                    full_batch_gradients=_get(j, "full_batch_gradients", False), master_seed=_get(j, "master_seed", 1),
                    schedule=_get(j, "schedule", "floor"), eval_every=_get(j, "eval_every", 1),
                    check_replicas=bool(_get(j, "check_replicas", False)),
                    throttle_host=bool(_get(j, "throttle_host", False)))
    if "heterogeneity" in j:
        sim.worker_multipliers = _get(j["heterogeneity"], "worker_multipliers", None)
    t = _req(j, "t_updates")
    if t < 1:
        raise InvalidArgument(_lib.INVALID, "config: t_updates >= 1")
    if sim.n_workers < 1:
        raise InvalidArgument(_lib.INVALID, "config: n_workers >= 1")
    if sim.batch_size < 1:
        raise InvalidArgument(_lib.INVALID, "config: batch_size >= 1")
    if sim.n_grad_accumulation < 1:
        raise InvalidArgument(_lib.INVALID, "config: n_grad_accumulation >= 1")
    if sim.warmup_rounds < 0:
        raise InvalidArgument(_lib.INVALID, "config: warmup_rounds >= 0")
    if sim.worker_multipliers is not None:
        if len(sim.worker_multipliers) != sim.n_workers:
            raise InvalidArgument(_lib.INVALID, "config: worker_multipliers length must equal n_workers")
        if any(not (m > 0) for m in sim.worker_multipliers):
            raise InvalidArgument(_lib.INVALID, "config: worker_multipliers > 0")
    opt.total_steps = t  # config.cpp:131
    return ExperimentConfig(prob, method, opt, sim, t, _get(j, "output_dir", ""), dict(j))


def config_hash(j: dict) -> str:
    """config.cpp:147-157: FNV-1a over the canonical (nlohmann dump) serialisation."""
    import json

    s = json.dumps(j, separators=(",", ":"), sort_keys=True, ensure_ascii=False).encode()
    h = 0xCBF29CE484222325
    for c in s:
        h ^= c
        h = (h * 0x100000001B3) & (2**64 - 1)
    return f"{h:016x}"


# ------------------------------------------------------- config-level entry
class RunSummaryC(C.Structure):
    _fields_ = [("updates", C.c_int), ("diverged", C.c_int), ("final_loss", C.c_double),
                ("samples", C.c_longlong), ("wall_ms", C.c_double), ("out_dir", C.c_char * 1024)]


_lib.register({"acco_run": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(RunSummaryC)])})


def run_config(config: str, out_dir: str = "") -> tuple:
    """acco_run (include/acco.h): the reference CLI's `run` as one library call
    (load_config -> run_protocol -> write_run_outputs, proj/src/config.cpp:135-145,
    csvio.cpp:79-102). `config`: a JSON file path or JSON text. Returns
    (exit code, summary dict); 0 ok, 3 diverged (outputs written); invalid
    configs raise InvalidArgument (exit 2)."""
    s = RunSummaryC()
    rc = _lib.lib().acco_run(config.encode(), out_dir.encode(), C.byref(s))
    if rc not in (_lib.OK, _lib.DIVERGED):
        _lib.check(rc)
    return rc, {"updates": s.updates, "diverged": bool(s.diverged), "final_loss": s.final_loss,
                "samples": s.samples, "wall_ms": s.wall_ms, "out_dir": s.out_dir.decode()}


# ---------------------------------------------------------------- memory model
MEMORY_METHODS = ("ddp", "zero1", "zero2", "zero3", "slowmo", "diloco", "co2", "dpu", "wp", "acco")


def memory_model_bytes(method: str, k: float, n: float, psi: float) -> float:
    """Per-replica bytes (convergence.cpp:182-201; the paper's Table 1): bf16
    params + grads (2 + 2 B), optimizer K B/param (sharded by N where the
    method shards it); ACCO / DPU / WP add one bf16 communication buffer."""
    if not (k > 0.0) or not (n >= 1.0) or not (psi >= 1.0):
        raise InvalidArgument(_lib.INVALID, "memory_model: K > 0, N >= 1, psi >= 1 required")
    table = {"ddp": (2 + 2 + k), "zero1": (2 + 2 + k / n), "zero2": (2 + (2 + k) / n), "zero3": ((2 + 2 + k) / n),
             "slowmo": (2 + 2 + 2 * 2 + k), "diloco": (2 + 2 + 2 * 2 + k), "co2": (2 + 2 + 4 * 2 + k)}
    if method in ("dpu", "wp", "acco"):
        return (2 + 2 + 2 + k / n) * psi
    if method not in table:
        raise InvalidArgument(_lib.INVALID, f"memory_model: unknown method {method}")
    return table[method] * psi


def memory_reported_gb(b: float) -> int:
    """convergence.cpp:203-205."""
    return int(math.floor(b / 1e9 + 0.25))
