// Trainer engines: ACCO (proj/src/protocols.cpp:437-709) and the DDP
// (:191-338) / ZeRO-1 baselines, on real CUDA streams instead of the
// reference's discrete-event clock.
#pragma once

#include <vector>

#include "comm.h"
#include "peer.h"
#include "host_util.h"
#include "model.h"
#include "optim.h"

namespace acco {

enum Method : int { kDDP = 0, kDPU = 1, kWP = 2, kACCO = 3, kZeRO1 = 4 };
enum Schedule : int { kFloor = 0, kAdaptive = 1, kReplay = 2 };

struct SimCfg {
    int n_workers = 1;
    int batch_size = 1;
    int n_grad_accumulation = 1;
    int warmup_rounds = 0;
    uint64_t master_seed = 1;
    int schedule = kFloor;
    std::vector<int32_t> replay;     // [T][2][n_workers] (mb_estimate, mb_main)
    int eval_every = 0;              // 0: no full-dataset evaluation
    std::vector<double> throttle_ns; // per worker, extra ns after every micro-batch
    int eval_batch = 0;              // samples per evaluation chunk (0 = model max)
    double comm_delay_ns = 0;        // emulated interconnect time per comm phase (0 = off)
    int check_replicas = 0;          // debug: cross-rank replica checksum after every comm phase
    int throttle_host = 0;           // 1: throttle by a host sleep after the micro-batch completes
    // emulated interconnect: with comm_standin_ctas > 0 the comm_delay_ns of
    // a phase is spent by a paced HBM copy of comm_standin_bytes on that many
    // CTAs (2/3 before the optimizer: reduce-scatter, 1/3 after: all-gather)
    // instead of a one-thread spin
    int comm_standin_ctas = 0;
    double comm_standin_bytes = 0;
};

struct UpdateRecord {
    int update = 0;
    double time_s = 0;
    double loss = NAN, grad_sq = NAN, grad_sq_estimate = NAN, lyapunov = NAN;
    long long samples_cum = 0;
    double train_loss = NAN;
    std::vector<int> mb_main, mb_estimate;  // local workers
};

struct RunStats {
    long long issued = 0, consumed = 0, discarded = 0;
    double wall_ms = 0, compute_busy_ms = 0, comm_busy_ms = 0, comm_exposed_ms = 0;
    double opt_ms = 0;  // optimizer-kernel time summed over phases (device events)
    int opt_launches = 0;
    int diverged = 0;
    long long h2d_bytes = 0, d2h_bytes = 0;  // host-data path traffic during the run
    int n_records = 0;  // committed records (< t_updates when the run diverged)
};

// One timeline.csv row (simclock.hpp Interval; csvio.cpp:48-66), from CUDA
// events, seconds since the start of the run() call.
enum IntervalKind : int { kIvInitGrad = 0, kIvMicrobatch = 1, kIvAllReduce = 2, kIvReduceScatter = 3,
                          kIvOptimizer = 4, kIvAllGather = 5 };
struct Interval {
    int worker = 0;
    int stream = 0;  // 0 compute, 1 comm
    int kind = 0;
    double t_start = 0, t_end = 0;
    int micro_batches = 0;
    long long bytes = 0;
};

class Trainer {
public:
    Trainer(GPTModel* model, const OptConfig& cfg, const SimCfg& sim, int method, Comm* comm,
            PeerFabric* peer = nullptr);
    ~Trainer();
    Trainer(const Trainer&) = delete;
    Trainer& operator=(const Trainer&) = delete;

    void set_theta(const float* host_theta);
    void get_theta(int which, float* host_out);
    // Runs t_updates committed updates, continuing from the current state.
    // theta_hist (host, nullable): [t_updates][2][psi] fp32 — theta^(t+1) and
    // theta-tilde^(t+1) after each commit (RunTrace.theta/estimate_history).
    void run(int t_updates, std::vector<UpdateRecord>& recs, RunStats& st, float* theta_hist = nullptr);
    int n_local() const { return n_local_; }
    PeerFabric* peer() const { return peer_; }
    const std::vector<Interval>& timeline() const { return timeline_; }
    cudaStream_t compute_stream() const { return cs_; }

private:
    struct PhaseEvents;
    void alloc();
    void launch_phase(int p, int acc_q, int64_t* tot, PhaseEvents& ev, bool warm = false);
    FoldIO fold_sources(int acc_q, float* dst);
    void opt_gather(bool commit, FoldIO io, const float* ret, const int64_t* tot, const int64_t* ret_tot,
                    void* act_dst, void* ag_dst, cudaEvent_t after_opt);
    void run_acco(int T, std::vector<UpdateRecord>& recs, RunStats& st);
    void run_sync(int T, std::vector<UpdateRecord>& recs, RunStats& st);
    void snapshot(int t, bool est_is_theta);
    void fetch_history(int T, float* host);
    char* hist_dev_ = nullptr;
    int stage_len(int p, int w, bool boot) const;
    void build_timeline(int n_phases, const PhaseEvents& ev, cudaEvent_t base, bool sync_kind,
                        const std::vector<int>& stage_k, const std::vector<char>& stage_init,
                        const std::vector<char>& slot_used);
    std::vector<Interval> timeline_;
    void micro(int w, const void* params, uint64_t round, uint64_t tag, int ordinal, float* acc, double* loss_slot);
    void eval(const void* params, double* loss_slots, double* gsq_slot);
    void* theta_params() const { return theta_act_; }
    void check_replicas(int p, unsigned long long seq);
    uint64_t* hash_buf_ = nullptr;  // [2 local][kMaxPeers * 2 gathered]
    void* standin_buf_ = nullptr;   // comm stand-in source / destination (2 x bytes)
    void emulate_comm(double frac);
    // Blocking waits that cannot hang on a dead rank: in NCCL mode they poll the
    // communicator's async error state with a timeout (Comm::wait).
    void wait_event(cudaEvent_t e);
    void sync_streams();
    cudaEvent_t sync_ev_[3] = {nullptr, nullptr, nullptr};  // [2]: host-throttle micro-batch completion
    void* est_params() const { return est_act_; }

    GPTModel* model_;
    OptConfig cfg_;
    SimCfg sim_;
    int method_;
    Comm* comm_;
    PeerFabric* peer_ = nullptr;     // fused fold over NVLink peer memory instead of NCCL
    unsigned long long phase_seq_ = 0;  // comm phases issued so far (peer protocol sequence)
    void* rep_[2] = {nullptr, nullptr}; // registered replicas (DPU swaps theta_act_/est_act_ between them)
    int n_local_ = 1, world_ = 1, rank_ = 0;
    ShardLayout layout_;
    int64_t psi_ = 0, chunk_ = 0, own_n_ = 0, own_lo_ = 0;
    bool padded_ = false;
    cudaStream_t cs_ = nullptr, ms_ = nullptr;  // compute, comm
    // device state
    void* theta_act_ = nullptr;  // flat replica of theta (activation dtype)
    void* est_act_ = nullptr;    // flat replica of theta-tilde
    void* ag_theta_ = nullptr;   // padded all-gather buffers (== flat when not padded)
    void* ag_est_ = nullptr;
    float *master_ = nullptr, *m_ = nullptr, *v_ = nullptr;
    std::vector<float*> acc_;  // [n_local][2]
    float* pad_send_ = nullptr;
    float *g_ret_ = nullptr, *g_main_ = nullptr, *full_red_ = nullptr;
    int64_t* cnt_send_ = nullptr;
    int* phase_flags_ = nullptr;  // this run's per-phase optimizer non-finite bits (see optim.cu)
    int* cur_flag_ = nullptr;     // the phase being launched
    double* loss_ring_ = nullptr;
    double* loss_host_ = nullptr;  // pinned mirror of loss_ring_ (host-data path)
    long long d2h_bytes_ = 0;
    int loss_cap_ = 0;
    float* eval_grad_ = nullptr;
    double* eval_scratch_ = nullptr;
    long long step_ = 0;   // optimizer step (OptimizerState::step), shared by all shards
    long long update_ = 0; // committed updates so far (continues across run() calls)
    long long samples_cum_ = 0;
    long long mb_counter_ = 0;
    // DPU / WP: the bundle computed in the last round awaits its optimizer
    // step (SyncEngine::pending_, protocols.cpp:268); it survives run() calls
    bool theta0_nonfinite_ = false;  // set_theta saw a non-finite theta0 (raised by run())
    bool pending_valid_ = false;
    int pending_slot_ = 0;       // accumulator parity holding it
    int pending_k_ = 0;          // its micro-batches per worker
    double pending_loss_ = 0.0;  // its summed micro-batch losses (local workers)
};

}  // namespace acco
