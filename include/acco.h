/*
 * acco.h — C-ABI of the B200-native ACCO library (libacco: _acco_b200.so).
 *
 * This is the drop-in boundary for the ACCO round of the reference simulator
 * `accosim` (/root/reference/proj). Every entry point below names the
 * reference interface it replaces (file:line). Conventions:
 *   - plain pointers and sizes only; no C++ / torch types;
 *   - device pointers are caller-owned unless a *_create/destroy pair owns them;
 *   - `stream` is a cudaStream_t passed as void*; ops are asynchronous on it;
 *   - every function returns a status code (below) and never throws; the
 *     message of the last failure on the calling thread is acco_last_error().
 *
 * Status codes mirror the accosim CLI exit codes
 * (/root/reference/proj/tools/accosim_main.cpp:30-33) plus two B200 codes.
 */
#ifndef ACCO_H_
#define ACCO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACCO_ABI_VERSION 2

#define ACCO_OK 0
#define ACCO_VERIFY_FAIL 1  /* accosim exit 1 */
#define ACCO_INVALID 2      /* std::invalid_argument, accosim exit 2 */
#define ACCO_DIVERGED 3     /* RunTrace.diverged, accosim exit 3 */
#define ACCO_CUDA_ERROR 4   /* CUDA / NCCL failure (B200 only) */
#define ACCO_LOGIC_ERROR 5  /* std::logic_error (protocol invariants) */

#define ACCO_DTYPE_F32 0
#define ACCO_DTYPE_BF16 1

const char* acco_last_error(void);
int acco_version(void);

/* Instrumentation (B200 only): number of this library's kernel launches so
 * far, and optional CUDA-event timing per kernel class on the launching
 * stream — class 0 GEMM (work = algorithmic flops), 1 attention (flops),
 * 2 fused optimizer (algorithmic bytes), 3 bias / LN-parameter column
 * reductions (bytes), 4 LayerNorm fwd/bwd (bytes), 5 cross-entropy (bytes),
 * 6 token gather / embedding (bytes), 7 other. */
#define ACCO_PROF_CLASSES 8
long long acco_launch_count(void);
void acco_prof_enable(int on);
int acco_prof_reset(void);
int acco_prof_read(double ms[ACCO_PROF_CLASSES], double work[ACCO_PROF_CLASSES],
                   long long launches[ACCO_PROF_CLASSES]);

/* ------------------------------------------------------------------ shards
 * shard_partition (proj/include/accosim/shard.hpp:24-38): contiguous
 * near-equal split, the first (dim mod n) ranges get one extra element. */
int acco_shard_partition(uint64_t dim, int n, uint64_t* lo_out, uint64_t* hi_out);

/* ------------------------------------------------------------------- rng
 * rng::derive / Stream (proj/include/accosim/rng.hpp:13-56) and the
 * micro-batch index draw of stochastic_grad (proj/src/problems.cpp:442-444).
 * Exposed so callers can pin token indexing bit-exactly. */
uint64_t acco_rng_derive(uint64_t master, uint64_t a, uint64_t b, uint64_t c, uint64_t d);
int acco_sample_indices(uint64_t stream_seed, int batch, int n_samples, int32_t* out);

/* -------------------------------------------------------------- optimizer
 * OptimizerConfig (proj/include/accosim/optim.hpp:21-32). kind: 0 sgd,
 * 1 adam, 2 adamw. scheduler: 0 constant, 1 cosine. */
typedef struct acco_opt_cfg {
    int kind;
    double learning_rate;
    double adam_beta1;
    double adam_beta2;
    double adam_eps;
    double weight_decay;
    int scheduler;
    int n_warmup_steps;
    long long total_steps;
    double cosine_min_factor;
} acco_opt_cfg;

/* scheduled_lr (proj/src/optim.cpp:37-48). */
double acco_scheduled_lr(const acco_opt_cfg* cfg, long long t);

/* OptimizerState (proj/include/accosim/optim.hpp:35-43) for one shard
 * [lo, hi), device resident: fp32 master params, first/second moments
 * (v unused for sgd, m unused for sgd). `step` is host state. */
typedef struct acco_shard_state {
    long long step;
    float* theta;
    float* m;
    float* v;
    uint64_t lo;
    uint64_t hi;
} acco_shard_state;

/* K6 — ACCO estimate branch (proj/src/protocols.cpp:647-658): the optimizer
 * step of opt_step (proj/src/optim.cpp:50-92) on a *transient* copy of the
 * shard state: theta_est = Opt(theta, gsum / total); m, v and step are NOT
 * written. `total` is read from device memory (the counts all-reduce output).
 * Output dtype is ACCO_DTYPE_F32 or ACCO_DTYPE_BF16 (the all-gather payload).
 * `nonfinite_flag` (device int, nullable) gets bit 0 (value 1) if any input is
 * non-finite — opt_step's std::invalid_argument (optim.cpp:56-57) — and bit 1
 * (value 2) if a new parameter is non-finite. */
int acco_opt_estimate(const acco_opt_cfg* cfg, const acco_shard_state* st, const float* gsum,
                      const int64_t* total_dev, void* theta_out, int out_dtype,
                      int* nonfinite_flag, void* stream);

/* K7 — ACCO commit branch (proj/src/protocols.cpp:659-707): persistent
 * step on the shard: mean = (gsum + g_retained) / (total + retained_total),
 * theta, m, v updated in place, step += 1 (host), theta also written to
 * theta_out (all-gather payload, may be NULL). g_retained / retained_total_dev
 * may be NULL (DDP / ZeRO-1: plain sharded_opt_step, optim.cpp:94-119). */
int acco_opt_commit(const acco_opt_cfg* cfg, acco_shard_state* st, const float* gsum,
                    const float* g_retained, const int64_t* total_dev,
                    const int64_t* retained_total_dev, void* theta_out, int out_dtype,
                    int* nonfinite_flag, void* stream);

/* -------------------------------------------------------------- collectives
 * Fabric (proj/include/accosim/collectives.hpp:31-49) over NCCL on
 * NVLink 5 / NVSwitch: one rank per process (one GPU). */
typedef struct acco_comm acco_comm;
int acco_comm_unique_id(unsigned char id_out[128]);
int acco_comm_init_rank(int nranks, int rank, const unsigned char id[128], int device,
                        acco_comm** out);
int acco_comm_destroy(acco_comm* comm);
int acco_comm_size(const acco_comm* comm);
int acco_comm_rank(const acco_comm* comm);
/* Fabric::all_reduce (collectives.cpp:36-46), fp32 sum. */
int acco_all_reduce_f32(acco_comm* comm, const float* send, float* recv, uint64_t count,
                        void* stream);
/* Fabric::all_reduce_counts (collectives.cpp:48-53), int64 sum. */
int acco_all_reduce_i64(acco_comm* comm, const int64_t* send, int64_t* recv, uint64_t count,
                        void* stream);
/* Fabric::reduce_scatter (collectives.cpp:55-75): send holds nranks*count
 * elements (owner-padded chunks), recv gets this rank's summed chunk. */
int acco_reduce_scatter_f32(acco_comm* comm, const float* send, float* recv, uint64_t count,
                            void* stream);
/* Fabric::all_gather (collectives.cpp:77-91): recv holds nranks*count. */
int acco_all_gather(acco_comm* comm, const void* send, void* recv, uint64_t count, int dtype,
                    void* stream);
/* Owner-padded layout for NCCL's equal-count RS/AG when dim mod n != 0:
 * chunk = ceil(dim/n); padded[w*chunk + j] <-> flat[lo_w + j] for
 * j < hi_w - lo_w (shard_partition ranges), zero padding otherwise.
 * pack: fp32 flat -> padded; unpack: padded -> flat (dtype F32 or BF16). */
int acco_pack_padded(const float* flat, float* padded, uint64_t dim, int n, void* stream);
int acco_unpack_padded(const void* padded, void* flat, uint64_t dim, int n, int dtype, void* stream);

/* ----------------------------------------------------------- raw GEMM (K1)
 * C[m,n] (op)= sum_k A(m,k) B(n,k); operands K-major (ptr[row*ld+k]) or
 * MN-major (ptr[k*ld+row]). dtype BF16 -> tcgen05/TMA kernel, F32 -> SIMT
 * parity kernel. epi_mode: 0 store(+bias+residual), 1 gelu (aux=pre-act),
 * 2 dgelu (C=acc*gelu'(aux)), 3 fp32 accumulate (C = beta*C + acc). */
int acco_gemm(const void* a, int64_t lda, int a_mn_major, const void* b, int64_t ldb,
              int b_mn_major, int m, int n, int k, int dtype, int epi_mode, void* c, int64_t ldc,
              const void* bias, const void* residual, int64_t ldr, void* aux, int64_t ld_aux,
              int beta, void* stream);
/* Weight-gradient GEMM with its bias gradient (bf16 operands, fp32 outputs):
 * C[m,n] (+)= sum_k A(m,k) B(n,k) and bias_grad[m] (+)= sum_k A(m,k) (the
 * column sums of dY for A = dY^T), '+' when beta = 1. The row sums come off
 * the tensor core (a ones-operand MMA in the first n-block's tiles), fused
 * into the same launch — the reference's Bundle::add of the bias entries
 * (/root/reference/proj/src/protocols.cpp:61-66) without a separate pass. */
int acco_gemm_bias_grad(const void* a, int64_t lda, int a_mn_major, const void* b, int64_t ldb,
                        int b_mn_major, int m, int n, int k, float* c, int64_t ldc, float* bias_grad,
                        int beta, void* stream);

/* ------------------------------------------------------ model plugin (LM)
 * The B200 gradient oracle for the GPT-style LM defined in
 * oracle/gpt_oracle.py, behind the Problem contract of
 * proj/include/accosim/problems.hpp:86-92. precision: ACCO_DTYPE_F32
 * (fp32-accurate parity mode) or ACCO_DTYPE_BF16 (tcgen05 throughput mode). */
typedef struct acco_lm_cfg {
    int vocab;
    int d_model;
    int n_layer;
    int n_head;
    int seq_len;
    int n_samples;
    uint64_t data_seed;
    int precision;
    int max_batch; /* samples per micro-batch the workspace is sized for */
    int host_data; /* 1: dataset stays in pinned host memory; every micro-batch's
                      token rows are copied host->device (data-loader path), and
                      every micro-batch loss is read back device->host */
    /* model family (BASELINE.json C4): 0 = GPT-2 block (configs C1-C3),
     * 1 = Llama block (RMSNorm, RoPE, grouped-query attention, SwiGLU, untied
     * head; oracle/gpt_oracle.py arch="llama") */
    int arch;
    int n_kv_head;    /* llama: KV heads (0 -> n_head) */
    int d_ff;         /* llama: SwiGLU hidden size (0 -> 4 * d_model) */
    double rope_base; /* llama: rotary base (0 -> 10000) */
} acco_lm_cfg;

typedef struct acco_model acco_model;
int acco_model_create(const acco_lm_cfg* cfg, acco_model** out);
int acco_model_destroy(acco_model* m);
long long acco_model_num_params(const acco_model* m);
/* default_theta0 (proj/src/problems.cpp:474-488 key) for the LM, host fp32 [psi]. */
int acco_model_theta0(const acco_model* m, uint64_t master_seed, float* host_out);
/* The synthetic token dataset, host int32 [n_samples][seq_len+1]. */
int acco_model_dataset(const acco_model* m, int32_t* host_out);
/* stochastic_grad (problems.cpp:419-451) fused with Bundle::add
 * (protocols.cpp:61-66): grad_acc[psi] += batch * (per-sample mean gradient)
 * at `params` (device, model precision); *loss_sum_dev (double) = sum of the
 * per-sample losses. Draws Stream(stream_seed).below(n_samples) x batch. */
int acco_model_stochastic_grad(acco_model* m, const void* params, uint64_t stream_seed, int batch,
                               float* grad_acc, double* loss_sum_dev, void* stream);
/* value_and_grad (problems.cpp:406-417) over the full dataset; blocking.
 * grad_out (device fp32 [psi]) may be NULL. */
int acco_model_value_and_grad(acco_model* m, const void* params, double* loss_out, float* grad_out,
                              void* stream);

/* Device time of one micro-batch (fwd + bwd + accumulate) of `batch` samples,
 * mean of `reps` (ns). Used to turn the reference's HeterogeneityProfile
 * multipliers (protocols.hpp:19-27) into per-worker throttles: a worker with
 * multiplier m spins (m - 1) x this after each micro-batch. */
int acco_model_time_micro_batch(acco_model* m, int batch, int reps, double* ns_out);

/* --------------------------------------------------------------- trainer
 * run_protocol (proj/include/accosim/protocols.hpp:89-90) on B200: one
 * process per GPU (comm != NULL, NCCL) or all workers as virtual workers on
 * one device (comm == NULL; device-side Fabric with the reference's fixed
 * ascending-worker reduction order). */
#define ACCO_METHOD_DDP 0
#define ACCO_METHOD_DPU 1 /* one-step-delayed update (protocols.cpp:357-379), warmup_rounds as DDP */
#define ACCO_METHOD_WP 2  /* weight prediction (protocols.cpp:383-424): commit + transient prediction step */
#define ACCO_METHOD_ACCO 3
#define ACCO_METHOD_ZERO1 4 /* B200 baseline: DDP semantics, RS + sharded step + AG */

#define ACCO_SCHED_FLOOR 0    /* every stage exactly max(k,1) micro-batches (round-0 estimate: 1) */
#define ACCO_SCHED_ADAPTIVE 1 /* accumulate until the in-flight phase completes (Alg. 1) */
#define ACCO_SCHED_REPLAY 2   /* per-update counts given in `replay` */

/* SimConfig (protocols.hpp:29-38) plus B200 execution keys. */
typedef struct acco_sim_cfg {
    int n_workers;
    int batch_size;
    int n_grad_accumulation;
    int warmup_rounds;
    uint64_t master_seed;
    int schedule;
    const int32_t* replay;      /* [t_updates][2][n_workers]: mb_estimate, mb_main */
    int replay_len;             /* number of int32 in replay */
    int eval_every;             /* full-dataset loss/grad every k updates; 0 = never */
    int eval_batch;             /* samples per evaluation chunk; 0 = model max_batch */
    const double* throttle_ns;  /* [n_workers] straggler delay per micro-batch, or NULL */
    /* Single-GPU emulation of an N-GPU interconnect: every comm phase spins this
     * many ns on the comm stream after the counts all-reduce (the NVLink time of
     * that phase's reduce-scatter + all-gather), so the overlap of ACCO vs the
     * synchronous baselines can be measured on one GPU. 0 = off. */
    double comm_delay_ns;
    /* Debug (the reference's check_replicas, protocols.cpp:208-212): after every
     * comm phase the ranks hash their theta / theta-tilde replicas, exchange
     * the hashes and compare; a mismatch fails the run with ACCO_LOGIC_ERROR.
     * One extra barrier per phase. 0 = off. */
    int check_replicas;
    /* Straggler emulation mode for throttle_ns: 0 = a spin kernel on the
     * worker's compute stream after each micro-batch (device time); 1 = the
     * paper's method (time.sleep): the host waits for the
     * micro-batch to complete, then sleeps, leaving the GPU idle. */
    int throttle_host;
    /* With comm_delay_ns > 0: 0 = the phase's emulated interconnect time is a
     * one-thread spin; > 0 = a paced HBM copy of comm_standin_bytes on this
     * many CTAs (NCCL's channel count), holding SMs like the real collectives. */
    int comm_standin_ctas;
    double comm_standin_bytes;
} acco_sim_cfg;

/* RoundRecord (protocols.hpp:41-53); NaN where not evaluated. */
typedef struct acco_record {
    int update;
    double time_s; /* measured seconds (CUDA events) since the start of the run call */
    double loss;
    double grad_sq;
    double grad_sq_estimate;
    double lyapunov;
    long long samples_cum;
    double train_loss; /* sample-weighted mean micro-batch loss (this rank) */
} acco_record;

typedef struct acco_run_stats {
    long long issued_micro_batches;
    long long consumed_micro_batches;
    long long discarded_micro_batches;
    double wall_ms;
    double compute_busy_ms;
    double comm_busy_ms;
    double comm_exposed_ms; /* comm busy time not overlapped by compute */
    double opt_ms;          /* fused optimizer kernel time, summed */
    int opt_launches;
    int diverged;
    long long h2d_bytes; /* host-data path: token rows shipped host->device */
    long long d2h_bytes; /* host-data path: per-micro-batch losses read back */
    int n_records;       /* valid rows of recs / mb_counts / theta_history: t_updates, or fewer
                            when the run diverged (the reference's partial RunTrace) */
} acco_run_stats;

typedef struct acco_trainer acco_trainer;
int acco_trainer_create(acco_model* model, const acco_opt_cfg* opt, const acco_sim_cfg* sim, int method,
                        acco_comm* comm, acco_trainer** out);
int acco_trainer_destroy(acco_trainer* t);
/* Replicates theta0 (host fp32 [psi]) and resets optimizer state. */
int acco_trainer_set_theta(acco_trainer* t, const float* host_theta);
/* which: 0 committed theta replica, 1 estimate replica, 2 this rank's fp32 master shard. */
int acco_trainer_get_theta(acco_trainer* t, int which, float* host_out);
/* Runs t_updates committed updates (continuing). recs: [t_updates];
 * Divergence, as the reference (protocols.cpp:113-119,164-167,298-306;
 * optim.cpp:56-57): a non-finite parameter state or evaluated loss at a commit
 * ends the run with that record (loss +inf for the state) and returns
 * ACCO_DIVERGED; a synchronous round whose reduced mean is non-finite ends it
 * before its record (ACCO_DIVERGED); in ACCO a non-finite input to either
 * optimizer step is the reference's opt_step invalid_argument: ACCO_INVALID,
 * no records. stats->n_records counts the valid rows.
 * mb_counts (nullable): [t_updates][2][n_local] (mb_estimate, mb_main);
 * theta_history (nullable, host fp32): [t_updates][2][psi] = theta^(t+1) and
 * theta-tilde^(t+1) after each commit (RunTrace.theta/estimate_history,
 * protocols.hpp:61-76). */
int acco_trainer_run(acco_trainer* t, int t_updates, acco_record* recs, int32_t* mb_counts,
                     float* theta_history, acco_run_stats* stats);
int acco_trainer_n_local(const acco_trainer* t);

/* ------------------------------------------------------- config-level run
 * The reference's CLI `run` path as one call: load_config / parse_config
 * (proj/src/config.cpp:80-145; `config` is a JSON file path, or the JSON text
 * itself when it starts with '{') -> run_protocol (protocols.hpp:89-90) on this
 * device (n_workers virtual workers) -> write_run_outputs (csvio.cpp:79-102:
 * metrics.csv, timeline.csv, manifest.json; the manifest and config hash are
 * the reference's byte for byte). out_dir NULL/"" -> the config's output_dir,
 * else $ACCOSIM_OUT/run_<config_hash> (accosim_main.cpp:35-40,57-58).
 * Returns the CLI exit code (accosim_main.cpp:30-33): ACCO_OK, ACCO_DIVERGED
 * (outputs written), ACCO_INVALID (bad config), plus ACCO_CUDA_ERROR /
 * ACCO_LOGIC_ERROR. problem.kind: "gpt" or "llama" (B200 LM problems). */
typedef struct acco_run_summary {
    int updates;       /* records written to metrics.csv */
    int diverged;
    double final_loss; /* the last record's loss (NaN when not evaluated) */
    long long samples; /* samples_cum of the last record */
    double wall_ms;    /* device time of the run */
    char out_dir[1024];
} acco_run_summary;
int acco_run(const char* config, const char* out_dir, acco_run_summary* summary);

/* ------------------------------------------------------------- peer fabric
 * B200-native alternative to NCCL for the comm phase: ONE fused kernel per
 * phase reads every rank's accumulator shard over NVLink peer memory (CUDA
 * IPC), folds them in ascending rank order (the reference Fabric's reduce
 * order, collectives.cpp:55-75), applies the optimizer step and stores the
 * new parameters into every rank's replica (all-gather fused in); the counts
 * all-reduce and the phase barriers are device flags. One process per GPU of
 * one box. Setup: create the fabric, create the trainer on it, export this
 * rank's blob, all-gather the blobs out of band (any host transport), connect. */
typedef struct acco_peer acco_peer;
int acco_peer_create(int nranks, int rank, int device, acco_peer** out);
int acco_peer_destroy(acco_peer* p);
int acco_trainer_create_peer(acco_model* model, const acco_opt_cfg* opt, const acco_sim_cfg* sim, int method,
                             acco_peer* peer, acco_trainer** out);
long long acco_trainer_peer_blob_bytes(const acco_trainer* t);
int acco_trainer_peer_export(const acco_trainer* t, void* blob);
/* blobs: [nranks][blob_bytes], rank order */
int acco_trainer_peer_connect(acco_trainer* t, const void* blobs);

/* timeline.csv rows of the last acco_trainer_run (Timeline/Interval,
 * proj/include/accosim/simclock.hpp; written by csvio.cpp:48-66), measured
 * with CUDA events on the compute / comm streams, seconds since the run start.
 * kind: ACCO_IV_* below (event_kind strings "init_grad", "microbatch",
 * "all_reduce", "reduce_scatter", "optimizer", "all_gather"). */
#define ACCO_IV_INIT_GRAD 0
#define ACCO_IV_MICROBATCH 1
#define ACCO_IV_ALL_REDUCE 2
#define ACCO_IV_REDUCE_SCATTER 3
#define ACCO_IV_OPTIMIZER 4
#define ACCO_IV_ALL_GATHER 5
typedef struct acco_interval {
    int worker_id;
    int stream; /* 0 compute, 1 comm */
    int kind;
    int micro_batches;
    double t_start;
    double t_end;
    long long bytes;
} acco_interval;
/* Copies up to cap rows into out (nullable); *n_out = total row count. */
int acco_trainer_timeline(const acco_trainer* t, acco_interval* out, int cap, int* n_out);

#ifdef __cplusplus
}
#endif

#endif /* ACCO_H_ */
