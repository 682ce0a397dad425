// ACCO / DDP / ZeRO-1 trainer engines on two CUDA streams per GPU.
//
// ACCO (proj/src/protocols.cpp:437-709, Alg. 1 of PAPER.md:910-960): comm
// phase p consumes the accumulator each worker posts at the end of its
// stage p; even phases commit the estimate (transient optimizer copy), odd
// phases the full update. Stage p computes at the parameters produced by
// phase p-2 (theta-tilde for even p, theta for odd p) and may only *end* once
// phase p-1 is complete:
//
//   compute stream:  [stage p ..........][stage p+1 ............]
//   comm stream:            [phase p-1: AR(counts) RS -> fused AdamW -> AG]
//
// The reference's discrete-event clock is replaced by real streams; the
// reference's "keep accumulating until the collective completes" is either
// realised literally (adaptive schedule: the host polls the phase-done event
// after every micro-batch) or fixed (floor/replay schedules: the compute
// stream waits on the event before starting the next stage), which makes
// micro-batch counts bit-exact and replayable by the oracle.
#include "engine.h"
#include "gemm.h"
#include "lm_kernels.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <numeric>

namespace acco {

namespace {
constexpr uint64_t kTagInit = 1, kTagMain = 2, kTagEstimate = 3;  // protocols.cpp:52-54

struct EventArr {
    std::vector<cudaEvent_t> ev;
    void create(size_t n) {
        ev.assign(n, nullptr);
        for (auto& e : ev) ACCO_CUDA(cudaEventCreate(&e));
    }
    ~EventArr() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
    cudaEvent_t operator[](size_t i) const { return ev[i]; }
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    ACCO_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}
}  // namespace

struct Trainer::PhaseEvents {
    EventArr post, stage_start, start, cnt_done, rs_done, opt_done, done, mb;
    std::vector<long long> counts;  // [phase][local worker] samples posted
    int n_local = 1;
};

Trainer::Trainer(GPTModel* model, const OptConfig& cfg, const SimCfg& sim, int method, Comm* comm,
                 PeerFabric* peer)
    : model_(model), cfg_(cfg), sim_(sim), method_(method), comm_(comm), peer_(peer) {
    validate(cfg_);
    ACCO_REQUIRE(method == kACCO || method == kDDP || method == kZeRO1 || method == kDPU || method == kWP,
                 "method: unknown protocol");
    ACCO_REQUIRE(sim.warmup_rounds >= 0, "run_protocol: warmup_rounds >= 0");
    ACCO_REQUIRE(sim.n_workers >= 1, "run_protocol: n_workers >= 1");
    ACCO_REQUIRE(sim.batch_size >= 1, "run_protocol: batch_size >= 1");
    ACCO_REQUIRE(sim.n_grad_accumulation >= 1, "run_protocol: n_grad_accumulation >= 1");
    ACCO_REQUIRE(sim.batch_size <= model->cfg().max_batch, "batch_size exceeds the model's max_batch workspace");
    ACCO_REQUIRE(sim.throttle_ns.empty() || static_cast<int>(sim.throttle_ns.size()) == sim.n_workers,
                 "run_protocol: one multiplier per worker");
    ACCO_REQUIRE(!(comm_ && peer_), "trainer: NCCL communicator or peer fabric, not both");
    if (peer_) {
        world_ = peer_->size();
        rank_ = peer_->rank();
        n_local_ = 1;
        ACCO_REQUIRE(world_ == sim.n_workers, "peer fabric size must equal n_workers");
        ACCO_REQUIRE(method != kDDP, "peer fabric: sharded methods only (acco, zero1, dpu, wp)");
    } else if (comm_) {
        world_ = comm_->size();
        rank_ = comm_->rank();
        n_local_ = 1;
        ACCO_REQUIRE(world_ == sim.n_workers, "comm size must equal n_workers");
    } else {
        world_ = 1;
        rank_ = 0;
        n_local_ = sim.n_workers;
        ACCO_REQUIRE(n_local_ <= 16, "virtual workers: at most 16 per device");
        ACCO_REQUIRE(sim.schedule != kAdaptive || n_local_ == 1,
                     "adaptive schedule needs one worker per device (NCCL mode)");
    }
    // collectives beside compute (real ranks or an emulated interconnect):
    // CTA-pair GEMMs and the attention kernels take their work from queues
    // (the overlapping protocols only: DDP / ZeRO-1 run their collectives after
    // the backward, where the static schedules are faster)
    const bool beside = (world_ > 1 || sim.comm_delay_ns > 0 || sim.comm_standin_ctas > 0) &&
                        (method == kACCO || method == kDPU || method == kWP);
    gemm_set_pair_queue(beside);
    attention_set_dynamic(beside);  // the attention kernels' work items from a queue as well
    psi_ = model->num_params();
    layout_ = shard_partition(static_cast<uint64_t>(psi_), sim.n_workers);
    const bool sharded = (comm_ || peer_) && method_ != kDDP;
    if (sharded) {
        chunk_ = static_cast<int64_t>(layout_.chunk());
        padded_ = comm_ && psi_ % world_ != 0;  // NCCL's equal counts; the peer fold addresses [lo, hi) directly
        own_lo_ = static_cast<int64_t>(layout_.lo(rank_));
        own_n_ = static_cast<int64_t>(layout_.size(rank_));
    } else {
        chunk_ = psi_;
        padded_ = false;
        own_lo_ = 0;
        own_n_ = psi_;
    }
    int lo_prio = 0, hi_prio = 0;
    ACCO_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    // ACCO_COMM_PRIO: "low" puts the comm stream at the compute stream's priority,
    // "inverted" below it (A/B knob; default: comm high, compute low)
    int comm_prio = hi_prio, comp_prio = lo_prio;
    if (const char* e = std::getenv("ACCO_COMM_PRIO")) {
        if (std::string(e) == "low") comm_prio = lo_prio;
        if (std::string(e) == "inverted") std::swap(comm_prio, comp_prio);
    }
    ACCO_CUDA(cudaStreamCreateWithPriority(&cs_, cudaStreamNonBlocking, comp_prio));
    ACCO_CUDA(cudaStreamCreateWithPriority(&ms_, cudaStreamNonBlocking, comm_prio));
    for (auto& e : sync_ev_) ACCO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    alloc();
    if (peer_) {  // exported to the peers: accumulators, then the two replicas
        rep_[0] = theta_act_;
        rep_[1] = est_act_;
        std::vector<void*> bufs(acc_.begin(), acc_.end());
        bufs.push_back(rep_[0]);
        bufs.push_back(rep_[1]);
        peer_->register_buffers(bufs);
    }
}

Trainer::~Trainer() {
    cudaStreamSynchronize(cs_);
    cudaStreamSynchronize(ms_);
    void* bufs[] = {theta_act_, est_act_, master_, m_, v_, pad_send_, g_ret_, g_main_, cnt_send_,
                    loss_ring_, eval_grad_, eval_scratch_};
    for (void* b : bufs) cudaFree(b);
    if (ag_theta_ != theta_act_) cudaFree(ag_theta_);
    if (ag_est_ != est_act_) cudaFree(ag_est_);
    for (float* a : acc_) cudaFree(a);
    if (hash_buf_) cudaFree(hash_buf_);
    if (standin_buf_) cudaFree(standin_buf_);
    if (loss_host_) cudaFreeHost(loss_host_);
    for (auto& e : sync_ev_)
        if (e) cudaEventDestroy(e);
    cudaStreamDestroy(cs_);
    cudaStreamDestroy(ms_);
}

void Trainer::wait_event(cudaEvent_t e) {
    if (comm_)
        comm_->wait(e);
    else
        ACCO_CUDA(cudaEventSynchronize(e));
}

void Trainer::sync_streams() {
    ACCO_CUDA(cudaEventRecord(sync_ev_[0], ms_));
    ACCO_CUDA(cudaEventRecord(sync_ev_[1], cs_));
    wait_event(sync_ev_[0]);
    wait_event(sync_ev_[1]);
}

void Trainer::alloc() {
    const size_t e = model_->act_bytes();
    const size_t P = static_cast<size_t>(psi_);
    ACCO_CUDA(cudaMalloc(&theta_act_, P * e));
    ACCO_CUDA(cudaMalloc(&est_act_, P * e));
    if (comm_ && padded_) {
        ACCO_CUDA(cudaMalloc(&ag_theta_, static_cast<size_t>(chunk_) * world_ * e));
        ACCO_CUDA(cudaMalloc(&ag_est_, static_cast<size_t>(chunk_) * world_ * e));
        ACCO_CUDA(cudaMalloc(&pad_send_, static_cast<size_t>(chunk_) * world_ * 4));
    } else {
        ag_theta_ = theta_act_;
        ag_est_ = est_act_;
    }
    const size_t own_cap = static_cast<size_t>((comm_ || peer_) && method_ != kDDP ? chunk_ : psi_);
    ACCO_CUDA(cudaMalloc(&master_, own_cap * 4));
    if (cfg_.kind != 0) {
        ACCO_CUDA(cudaMalloc(&m_, own_cap * 4));
        ACCO_CUDA(cudaMalloc(&v_, own_cap * 4));
    }
    // accumulators: ACCO ping-pongs two per worker; with a single virtual
    // worker the estimate shard *is* the accumulator, so a third one keeps it
    // alive through the commit phase without a copy.
    const int nacc = method_ == kACCO ? (!comm_ && n_local_ == 1 ? 3 : 2) : (method_ == kDPU || method_ == kWP ? 2 : 1);
    for (int i = 0; i < n_local_ * nacc; ++i) {
        float* a = nullptr;
        ACCO_CUDA(cudaMalloc(&a, P * 4));
        ACCO_CUDA(cudaMemset(a, 0, P * 4));
        acc_.push_back(a);
    }
    if (comm_ || peer_ || n_local_ > 1) ACCO_CUDA(cudaMalloc(&g_ret_, own_cap * 4));  // retained estimate shard
    if (comm_) ACCO_CUDA(cudaMalloc(&g_main_, own_cap * 4));                  // reduce-scatter target
    ACCO_CUDA(cudaMalloc(&cnt_send_, 8));
    if (sim_.check_replicas) ACCO_CUDA(cudaMalloc(&hash_buf_, (2 + 2 * 64) * sizeof(uint64_t)));
    if (sim_.comm_standin_ctas > 0 && sim_.comm_standin_bytes > 0)
        ACCO_CUDA(cudaMalloc(&standin_buf_, 2 * (static_cast<size_t>(sim_.comm_standin_bytes) / 16 + 1) * 16));
    loss_cap_ = 1 << 16;
    ACCO_CUDA(cudaMalloc(&loss_ring_, loss_cap_ * sizeof(double)));
    if (model_->host_data()) ACCO_CUDA(cudaHostAlloc(&loss_host_, loss_cap_ * sizeof(double), cudaHostAllocDefault));
    if (sim_.eval_every > 0) {
        ACCO_CUDA(cudaMalloc(&eval_grad_, P * 4));
        ACCO_CUDA(cudaMalloc(&eval_scratch_, 512 * sizeof(double)));
    }
}

void Trainer::set_theta(const float* host) {
    const size_t P = static_cast<size_t>(psi_);
    theta0_nonfinite_ = false;
    for (size_t i = 0; i < P; ++i)
        if (!std::isfinite(host[i])) {
            theta0_nonfinite_ = true;
            break;
        }
    float* tmp = nullptr;
    ACCO_CUDA(cudaMalloc(&tmp, P * 4));
    ACCO_CUDA(cudaMemcpy(tmp, host, P * 4, cudaMemcpyHostToDevice));
    f32_to(tmp, theta_act_, model_->act_dtype(), psi_, cs_);
    f32_to(tmp, est_act_, model_->act_dtype(), psi_, cs_);
    ACCO_CUDA(cudaMemcpyAsync(master_, tmp + own_lo_, static_cast<size_t>(own_n_) * 4, cudaMemcpyDeviceToDevice, cs_));
    if (m_) {
        ACCO_CUDA(cudaMemsetAsync(m_, 0, static_cast<size_t>(own_n_) * 4, cs_));
        ACCO_CUDA(cudaMemsetAsync(v_, 0, static_cast<size_t>(own_n_) * 4, cs_));
    }
    ACCO_CUDA(cudaStreamSynchronize(cs_));
    ACCO_CUDA(cudaFree(tmp));
    step_ = 0;
    update_ = 0;
    samples_cum_ = 0;
    pending_valid_ = false;
}

void Trainer::get_theta(int which, float* host) {
    sync_streams();
    if (which == 2) {
        ACCO_CUDA(cudaMemcpy(host, master_, static_cast<size_t>(own_n_) * 4, cudaMemcpyDeviceToHost));
        return;
    }
    const void* src = which == 0 ? theta_act_ : est_act_;
    const size_t P = static_cast<size_t>(psi_);
    if (model_->act_dtype() == 0) {
        ACCO_CUDA(cudaMemcpy(host, src, P * 4, cudaMemcpyDeviceToHost));
    } else {
        std::vector<uint16_t> tmp(P);
        ACCO_CUDA(cudaMemcpy(tmp.data(), src, P * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < P; ++i) {
            uint32_t u = static_cast<uint32_t>(tmp[i]) << 16;
            std::memcpy(&host[i], &u, 4);
        }
    }
}

int Trainer::stage_len(int p, int w, bool boot) const {
    if (method_ != kACCO) return sim_.n_grad_accumulation;
    if (p == 0 && boot) return 1;  // bootstrap: one micro-batch at theta0 (protocols.cpp:468-474)
    if (sim_.schedule == kReplay) {
        const long long t = update_ + p / 2;
        const int half = p % 2;  // half 0: estimate, 1: main
        const int gw = (comm_ || peer_) ? rank_ : w;
        const size_t i = (static_cast<size_t>(t) * 2 + half) * sim_.n_workers + gw;
        ACCO_REQUIRE(i < sim_.replay.size(), "replay schedule shorter than the run");
        const int k = sim_.replay[i];
        ACCO_REQUIRE(k >= 1, "acco: empty accumulator at barrier");  // protocols.cpp:603
        return k;
    }
    return std::max(sim_.n_grad_accumulation, 1);
}

void Trainer::micro(int w, const void* params, uint64_t round, uint64_t tag, int ordinal, float* acc,
                    double* loss_slot) {
    const uint64_t gw = (comm_ || peer_) ? static_cast<uint64_t>(rank_) : static_cast<uint64_t>(w);
    const uint64_t seed = rng_derive(sim_.master_seed, gw, round, tag, static_cast<uint64_t>(ordinal));
    // the stage's first micro-batch overwrites the accumulator (Bundle::reset + add)
    model_->micro_batch(params, seed, 0, 0, sim_.batch_size, acc, loss_slot, cs_, ordinal > 0);
    if (loss_host_) {  // host-data path: every micro-batch loss is read back as it completes
        const ptrdiff_t slot = loss_slot - loss_ring_;
        ACCO_CUDA(cudaMemcpyAsync(loss_host_ + slot, loss_slot, sizeof(double), cudaMemcpyDeviceToHost, cs_));
        d2h_bytes_ += sizeof(double);
    }
    if (!sim_.throttle_ns.empty()) {
        const double ns = sim_.throttle_ns[static_cast<size_t>(gw)];
        if (sim_.throttle_host) {  // the paper's time.sleep: GPU idle while the worker sleeps
            if (ns > 0) {
                ACCO_CUDA(cudaEventRecord(sync_ev_[2], cs_));
                wait_event(sync_ev_[2]);
                std::this_thread::sleep_for(std::chrono::nanoseconds(static_cast<long long>(ns)));
            }
        } else {
            spin_ns(static_cast<uint64_t>(ns), cs_);
        }
    }
}

void Trainer::eval(const void* params, double* loss_slots, double* gsq_slot) {
    const int n = model_->cfg().n_samples;
    const int eb = sim_.eval_batch > 0 ? std::min(sim_.eval_batch, model_->cfg().max_batch) : model_->cfg().max_batch;
    ACCO_CUDA(cudaMemsetAsync(eval_grad_, 0, static_cast<size_t>(psi_) * 4, cs_));
    int ci = 0;
    for (int c = 0; c < n; c += eb, ++ci)
        model_->micro_batch(params, 0, 1, c, std::min(eb, n - c), eval_grad_, loss_slots + ci, cs_);
    scale_f32(eval_grad_, 1.0 / n, psi_, cs_);
    norm_sq(eval_grad_, psi_, gsq_slot, eval_scratch_, cs_);
}

// Gradient sources of one comm phase (accumulators with parity acc_q).
// NCCL: Fabric::reduce_scatter (collectives.cpp:55-75) into this rank's shard
// `dst` (DDP all-reduces in place, SyncEngine's reduce_mean,
// protocols.cpp:191-206) and the fold has that one source. Virtual workers:
// the fold reads every local accumulator itself, in ascending worker order
// (the reference's reduce order) — no separate reduction pass.
FoldIO Trainer::fold_sources(int acc_q, float* dst) {
    const int nacc = static_cast<int>(acc_.size()) / n_local_;
    auto acc_of = [&](int w) { return acc_[static_cast<size_t>(w) * nacc + acc_q % nacc]; };
    FoldIO io;
    if (peer_) {  // every rank's accumulator, this rank's shard, ascending rank order, over NVLink
        for (int r = 0; r < world_; ++r)
            io.src[r] = static_cast<const float*>(peer_->peer_buffer(r, acc_q % nacc)) + own_lo_;
        io.nsrc = world_;
        return io;
    }
    if (comm_ && method_ == kDDP) {
        comm_->all_reduce_f32(acc_of(0), acc_of(0), static_cast<size_t>(psi_), ms_);
        io.src[0] = acc_of(0);
        io.nsrc = 1;
        return io;
    }
    if (comm_) {
        const float* send = acc_of(0);
        if (padded_) {
            std::vector<uint64_t> lo, sz;
            for (int w = 0; w < world_; ++w) {
                lo.push_back(layout_.lo(w));
                sz.push_back(layout_.size(w));
            }
            pack_padded(send, pad_send_, lo.data(), sz.data(), world_, static_cast<uint64_t>(chunk_), ms_);
            send = pad_send_;
        }
        comm_->reduce_scatter_f32(send, dst, static_cast<size_t>(chunk_), ms_);
        io.src[0] = dst;
        io.nsrc = 1;
        return io;
    }
    for (int w = 0; w < n_local_; ++w) io.src[w] = acc_of(w);
    io.nsrc = n_local_;
    return io;
}

// Fused sharded optimizer step on this rank's shard (K6 transient estimate when
// !commit, K7 commit otherwise; optim.cpp:50-119) over the folded sources,
// then Fabric::all_gather (collectives.cpp:77-91) of the activation-dtype
// parameters into act_dst (NCCL) — or written straight into act_dst.
void Trainer::opt_gather(bool commit, FoldIO io, const float* ret, const int64_t* tot, const int64_t* ret_tot,
                         void* act_dst, void* ag_dst, cudaEvent_t after_opt) {
    const int act = model_->act_dtype();
    const size_t e = model_->act_bytes();
    if (peer_) {  // the new shard goes straight into every rank's replica (all-gather fused in)
        const int ri = act_dst == rep_[0] ? 0 : 1;
        for (int r = 0; r < world_; ++r)
            io.dst[r] = static_cast<char*>(peer_->peer_buffer(r, static_cast<int>(acc_.size()) + ri)) +
                        static_cast<size_t>(own_lo_) * e;
        io.ndst = world_;
        opt_fold(cfg_, step_, commit, io, ret, tot, ret_tot, master_, m_, v_, own_n_, act, cur_flag_, ms_);
        if (after_opt) ACCO_CUDA(cudaEventRecord(after_opt, ms_));
        return;
    }
    const bool sharded = comm_ && method_ != kDDP;
    void* out = sharded ? static_cast<char*>(ag_dst) + static_cast<size_t>(rank_) * chunk_ * e : act_dst;
    io.dst[0] = out;
    io.ndst = 1;
    opt_fold(cfg_, step_, commit, io, ret, tot, ret_tot, master_, m_, v_, own_n_, act, cur_flag_, ms_);
    if (after_opt) ACCO_CUDA(cudaEventRecord(after_opt, ms_));
    if (!sharded) return;
    comm_->all_gather(out, ag_dst, static_cast<size_t>(chunk_), act, ms_);
    if (padded_) {
        std::vector<uint64_t> lo, sz;
        for (int w = 0; w < world_; ++w) {
            lo.push_back(layout_.lo(w));
            sz.push_back(layout_.size(w));
        }
        unpack_padded(ag_dst, act_dst, static_cast<int>(e), lo.data(), sz.data(), world_,
                      static_cast<uint64_t>(chunk_), ms_);
    }
}

// Comm phase p on the comm stream: AR(counts) -> reduce -> optimizer -> AG
// (protocols.cpp:613-631 for ACCO; apply_and_commit / wp_round for the
// synchronous family). acc_q: parity of the accumulators consumed.
void Trainer::launch_phase(int p, int acc_q, int64_t* tot, PhaseEvents& ev, bool warm) {
    for (int w = 0; w < n_local_; ++w) ACCO_CUDA(cudaStreamWaitEvent(ms_, ev.post[static_cast<size_t>(p) * n_local_ + w], 0));
    ACCO_CUDA(cudaEventRecord(ev.start[p], ms_));
    long long local = 0;
    for (int w = 0; w < n_local_; ++w) local += ev.counts[static_cast<size_t>(p) * n_local_ + w];
    int64_t* totp = tot + p;
    // non-finite bits: one slot per ACCO phase; the synchronous family uses
    // slot 2r for the round's step and 2r+1 for WP's prediction step
    cur_flag_ = phase_flags_ + (method_ == kACCO ? p : 2 * p);
    // 1. Fabric::all_reduce_counts (collectives.cpp:48-53)
    const unsigned long long seq = ++phase_seq_;
    if (peer_) {  // post + wait for every rank's post; counts folded in rank order
        peer_->signal_post(seq, static_cast<int>(seq & 1), local, ms_);
        peer_->wait_posts(seq, static_cast<int>(seq & 1), totp, ms_);
    } else if (comm_) {
        fill_i64(cnt_send_, local, ms_);
        comm_->all_reduce_i64(cnt_send_, totp, 1, ms_);
    } else {
        fill_i64(totp, local, ms_);
    }
    ACCO_CUDA(cudaEventRecord(ev.cnt_done[p], ms_));
    emulate_comm(2.0 / 3.0);  // emulated interconnect: the reduce-scatter share
    if (method_ == kACCO) {
        const bool est = p % 2 == 0;
        FoldIO io = fold_sources(acc_q, est ? g_ret_ : g_main_);
        ACCO_CUDA(cudaEventRecord(ev.rs_done[p], ms_));
        if (est) {  // estimate on a transient copy of the shard state (protocols.cpp:652-658)
            // retain the folded shard for the commit (NCCL: the reduce-scatter already wrote it there)
            if (peer_ || (!comm_ && n_local_ > 1)) io.ret_out = g_ret_;
            opt_gather(false, io, nullptr, totp, nullptr, est_act_, ag_est_, ev.opt_done[p]);
        } else {    // commit with the retained estimate shard (protocols.cpp:661-670)
            const int nacc = static_cast<int>(acc_.size()) / n_local_;
            const float* ret =
                (comm_ || peer_ || n_local_ > 1) ? g_ret_ : acc_[static_cast<size_t>((acc_q + nacc - 1) % nacc)];
            opt_gather(true, io, ret, totp, totp - 1, theta_act_, ag_theta_, ev.opt_done[p]);
            ++step_;
        }
    } else {
        const FoldIO io = fold_sources(acc_q, g_main_);
        ACCO_CUDA(cudaEventRecord(ev.rs_done[p], ms_));
        if (method_ == kDPU && !warm) {
            // theta^(r+1) goes to the other replica: stage r still reads theta^(r),
            // which becomes the record's estimate (protocols.cpp:361-378)
            opt_gather(true, io, nullptr, totp, nullptr, est_act_, ag_est_, ev.opt_done[p]);
            ++step_;
            std::swap(theta_act_, est_act_);
            std::swap(ag_theta_, ag_est_);
        } else {
            opt_gather(true, io, nullptr, totp, nullptr, theta_act_, ag_theta_, ev.opt_done[p]);
            ++step_;
            // WP: prediction step from the updated state on a throwaway copy (protocols.cpp:398-403)
            if (method_ == kWP) {
                cur_flag_ = phase_flags_ + 2 * p + 1;
                opt_gather(false, io, nullptr, totp, nullptr, est_act_, ag_est_, nullptr);
            }
        }
    }
    emulate_comm(1.0 / 3.0);  // emulated interconnect: the all-gather share
    if (peer_) peer_->signal_done(seq, ms_);  // this rank's shard is in every replica
    if (sim_.check_replicas && (comm_ || peer_)) check_replicas(p, seq);
    ACCO_CUDA(cudaEventRecord(ev.done[p], ms_));
}

// Single-GPU study of the overlap (bench.py --emulate-comm-gpus): the phase's
// NVLink time comm_delay_ns, split 2:1 between the reduce-scatter (fp32) and
// the all-gather (bf16) byte volumes; a one-thread spin, or with
// comm_standin_ctas > 0 a paced copy that holds that many SMs and moves the
// bytes through HBM like NCCL's kernels.
void Trainer::emulate_comm(double frac) {
    if (!(sim_.comm_delay_ns > 0)) return;
    const uint64_t ns = static_cast<uint64_t>(sim_.comm_delay_ns * frac);
    if (sim_.comm_standin_ctas > 0 && standin_buf_) {
        const int64_t bytes = static_cast<int64_t>(sim_.comm_standin_bytes * frac) / 16 * 16;
        const size_t half = (static_cast<size_t>(sim_.comm_standin_bytes) / 16 + 1) * 16;
        comm_standin(standin_buf_, static_cast<char*>(standin_buf_) + half, bytes, sim_.comm_standin_ctas, ns, ms_);
    } else {
        spin_ns(ns, ms_);
    }
}

// check_replicas (protocols.cpp:208-212) across the ranks: after the phase's
// all-gather every rank's theta and theta-tilde replicas must be bitwise equal.
// Each rank hashes both, the hashes are exchanged (NCCL all-gather of 16 B, or
// the peer flag blocks) and compared on the device; a mismatch sets bit 2
// (value 4) of the phase's flag and run() throws logic_error. Debug mode
// (SimConfig.check_replicas): one extra barrier per phase.
void Trainer::check_replicas(int p, unsigned long long seq) {
    int* flag = phase_flags_ + (method_ == kACCO ? p : 2 * p);
    const size_t bytes = static_cast<size_t>(psi_) * model_->act_bytes();
    if (peer_) peer_->wait_done(seq, ms_);  // every rank's shard has landed in our replicas
    // fault injection for the tests: ACCO_DEBUG_CORRUPT=<rank>,<phase> perturbs
    // one parameter of that rank's replica before the check
    if (const char* c = std::getenv("ACCO_DEBUG_CORRUPT")) {
        int cr = -1, cp = -1;
        if (std::sscanf(c, "%d,%d", &cr, &cp) == 2 && cr == rank_ && cp == p)
            ACCO_CUDA(cudaMemsetAsync(theta_act_, 0x3f, 2, ms_));
    }
    replica_hash(theta_act_, static_cast<int64_t>(bytes), hash_buf_, ms_);
    replica_hash(est_act_, static_cast<int64_t>(bytes), hash_buf_ + 1, ms_);
    if (peer_) {
        peer_->check_hashes(seq, hash_buf_, flag, 4, ms_);
    } else {
        comm_->all_gather_u64(hash_buf_, hash_buf_ + 2, 2, ms_);
        hash_compare(hash_buf_ + 2, world_, 2, flag, 4, ms_);
    }
}

void Trainer::run(int T, std::vector<UpdateRecord>& recs, RunStats& st, float* theta_hist) {
    ACCO_REQUIRE(T >= 1, "run_protocol: t_updates >= 1");
    ACCO_REQUIRE(!peer_ || peer_->connected(), "peer fabric: connect the ranks before run()");
    if (peer_ && phase_seq_ > 0) peer_->wait_done(phase_seq_, cs_);  // peers finished writing our replicas
    if (cfg_.total_steps == 0) cfg_.total_steps = T;  // run_protocol, protocols.cpp:729
    if (theta0_nonfinite_ && update_ == 0) {
        // where the reference first touches theta0: the synchronous rounds'
        // check_replicas (NaN != NaN across >= 2 replicas, protocols.cpp:208-212),
        // else the first stochastic_grad's check_theta (problems.cpp:37-42)
        if (method_ != kACCO && sim_.n_workers >= 2)
            throw Error(kLogicError, "protocol: parameter divergence across workers");
        throw Error(kInvalidArg, "theta has non-finite entries");
    }
    recs.clear();
    st = RunStats{};
    if (theta_hist) ACCO_CUDA(cudaMalloc(&hist_dev_, static_cast<size_t>(T) * 2 * psi_ * model_->act_bytes()));
    ACCO_CUDA(cudaMalloc(&phase_flags_, static_cast<size_t>(2 * T) * sizeof(int)));
    ACCO_CUDA(cudaMemsetAsync(phase_flags_, 0, static_cast<size_t>(2 * T) * sizeof(int), cs_));
    const long long h2d0 = model_->h2d_bytes(), d2h0 = d2h_bytes_;
    try {
        if (method_ == kACCO)
            run_acco(T, recs, st);
        else
            run_sync(T, recs, st);
        if (peer_) {  // the replicas are final only when every rank's last phase is done
            peer_->wait_done(phase_seq_, cs_);
            ACCO_CUDA(cudaStreamSynchronize(cs_));
        }
        st.h2d_bytes = model_->h2d_bytes() - h2d0;
        st.d2h_bytes = d2h_bytes_ - d2h0;
        if (theta_hist) fetch_history(T, theta_hist);
    } catch (...) {
        if (hist_dev_) cudaFree(hist_dev_);
        hist_dev_ = nullptr;
        cudaFree(phase_flags_);
        phase_flags_ = cur_flag_ = nullptr;
        throw;
    }
    if (hist_dev_) cudaFree(hist_dev_);
    hist_dev_ = nullptr;
    cudaFree(phase_flags_);
    phase_flags_ = cur_flag_ = nullptr;
}

// after the commit of update t (comm stream): copy theta^(t+1), theta-tilde^(t+1)
void Trainer::snapshot(int t, bool est_is_theta) {
    if (!hist_dev_) return;
    if (peer_) peer_->wait_done(phase_seq_, ms_);  // every rank's shard of this phase has landed
    const size_t bytes = static_cast<size_t>(psi_) * model_->act_bytes();
    char* dst = hist_dev_ + static_cast<size_t>(t) * 2 * bytes;
    ACCO_CUDA(cudaMemcpyAsync(dst, theta_act_, bytes, cudaMemcpyDeviceToDevice, ms_));
    ACCO_CUDA(cudaMemcpyAsync(dst + bytes, est_is_theta ? theta_act_ : est_act_, bytes,
                              cudaMemcpyDeviceToDevice, ms_));
}

void Trainer::fetch_history(int T, float* host) {
    const size_t n = static_cast<size_t>(T) * 2 * psi_;
    if (model_->act_dtype() == 0) {
        ACCO_CUDA(cudaMemcpy(host, hist_dev_, n * 4, cudaMemcpyDeviceToHost));
        return;
    }
    std::vector<uint16_t> tmp(n);
    ACCO_CUDA(cudaMemcpy(tmp.data(), hist_dev_, n * 2, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) {
        uint32_t u = static_cast<uint32_t>(tmp[i]) << 16;
        std::memcpy(&host[i], &u, 4);
    }
}

namespace {

// comm busy time not covered by compute busy time (SURVEY.md §8d "exposed comm")
double exposed(const std::vector<std::pair<double, double>>& comm, std::vector<std::pair<double, double>> comp,
               double* comm_busy, double* comp_busy) {
    std::sort(comp.begin(), comp.end());
    std::vector<std::pair<double, double>> u;
    for (auto& iv : comp) {
        if (!u.empty() && iv.first <= u.back().second)
            u.back().second = std::max(u.back().second, iv.second);
        else
            u.push_back(iv);
    }
    double cb = 0, xb = 0, ex = 0;
    for (auto& iv : u) xb += iv.second - iv.first;
    for (auto& c : comm) {
        const double len = c.second - c.first;
        cb += len;
        double cov = 0;
        for (auto& iv : u) cov += std::max(0.0, std::min(c.second, iv.second) - std::max(c.first, iv.first));
        ex += std::max(0.0, len - cov);
    }
    *comm_busy = cb;
    *comp_busy = xb;
    return ex;
}

}  // namespace

// timeline.csv rows of the last run() (csvio.cpp:48-66; the reference's
// simulated intervals, protocols.cpp:278-289 and :536-537, :620-627, here from
// the CUDA events of the two streams). One compute interval per stage and
// worker; per comm phase: counts all-reduce, reduce(-scatter), optimizer,
// all-gather (sync_kind: DDP's single all-reduce).
void Trainer::build_timeline(int n_phases, const PhaseEvents& ev, cudaEvent_t base, bool sync_kind,
                             const std::vector<int>& stage_k, const std::vector<char>& stage_init,
                             const std::vector<char>& slot_used) {
    timeline_.clear();
    const int nl = n_local_;
    const size_t n_slots = slot_used.size();  // stage_k: [slot][local worker]
    auto wid = [&](int w) { return (comm_ || peer_) ? rank_ : w; };
    for (size_t q = 0; q < n_slots; ++q) {
        if (!slot_used[q]) continue;
        for (int w = 0; w < nl; ++w) {
            Interval iv;
            iv.worker = wid(w);
            iv.stream = 0;
            iv.kind = stage_init[q] ? kIvInitGrad : kIvMicrobatch;
            iv.t_start = elapsed(base, ev.stage_start[q * nl + w]) * 1e-3;
            iv.t_end = elapsed(base, ev.post[q * nl + w]) * 1e-3;
            iv.micro_batches = stage_k[q * nl + w];
            timeline_.push_back(iv);
        }
    }
    const long long psi = psi_;
    const long long grad_bytes = psi * 4, param_bytes = psi * static_cast<long long>(model_->act_bytes());
    const bool all_reduce = sync_kind && method_ == kDDP;
    for (int p = 0; p < n_phases; ++p) {
        const double t0 = elapsed(base, ev.start[p]) * 1e-3, t1 = elapsed(base, ev.cnt_done[p]) * 1e-3,
                     t2 = elapsed(base, ev.rs_done[p]) * 1e-3, t3 = elapsed(base, ev.opt_done[p]) * 1e-3,
                     t4 = elapsed(base, ev.done[p]) * 1e-3;
        for (int w = 0; w < nl; ++w) {
            timeline_.push_back({wid(w), 1, kIvAllReduce, t0, t1, 0, 8});
            timeline_.push_back({wid(w), 1, all_reduce ? kIvAllReduce : kIvReduceScatter, t1, t2, 0, grad_bytes});
            timeline_.push_back({wid(w), 1, kIvOptimizer, t2, t3, 0, 0});
            if (!all_reduce) timeline_.push_back({wid(w), 1, kIvAllGather, t3, t4, 0, param_bytes});
        }
    }
}

void Trainer::run_acco(int T, std::vector<UpdateRecord>& recs, RunStats& st) {
    const int NP = 2 * T;
    const int nl = n_local_;
    const int B = sim_.batch_size;
    const int nacc = static_cast<int>(acc_.size()) / nl;
    PhaseEvents ev;
    ev.n_local = nl;
    ev.post.create(static_cast<size_t>(NP) * nl);
    ev.stage_start.create(static_cast<size_t>(NP) * nl);
    ev.start.create(NP);
    ev.cnt_done.create(NP);
    ev.rs_done.create(NP);
    ev.opt_done.create(NP);
    ev.done.create(NP);
    ev.mb.create(4);
    ev.counts.assign(static_cast<size_t>(NP) * nl, 0);
    int64_t* tot = nullptr;
    ACCO_CUDA(cudaMalloc(&tot, NP * sizeof(int64_t)));
    const bool do_eval = sim_.eval_every > 0;
    const int n_eval_chunks = do_eval ? ceil_div(model_->cfg().n_samples,
                                                  sim_.eval_batch > 0 ? std::min(sim_.eval_batch, model_->cfg().max_batch)
                                                                      : model_->cfg().max_batch)
                                      : 0;
    double* eval_buf = nullptr;  // [T][2 (theta, est)][n_chunks + 1 (gsq)]
    if (do_eval) ACCO_CUDA(cudaMalloc(&eval_buf, static_cast<size_t>(T) * 2 * (n_eval_chunks + 1) * sizeof(double)));
    std::vector<int> mb_phase;  // phase of each micro-batch's loss slot
    std::vector<int> stage_len_rec(static_cast<size_t>(NP) * nl, 0);
    const long long mb0 = mb_counter_;
    cudaEvent_t base;
    ACCO_CUDA(cudaEventCreate(&base));
    ACCO_CUDA(cudaEventRecord(base, cs_));
    ACCO_CUDA(cudaStreamWaitEvent(ms_, base, 0));
    const uint64_t r0 = static_cast<uint64_t>(update_);
    const unsigned long long seq0 = phase_seq_;  // phase p carries peer sequence seq0 + p + 1
    // a continuing run() resumes with the estimate stage of round r0 (the
    // pipeline of the previous call drained at its last commit); a fresh run
    // bootstraps with one Init micro-batch at theta0
    const bool boot = update_ == 0;
    for (int p = 0; p < NP; ++p) {
        for (int w = 0; w < nl; ++w) {
            // stage p computes at the parameters of phase p-2 and reuses its accumulator
            if (p >= 2) {
                ACCO_CUDA(cudaStreamWaitEvent(cs_, ev.done[p - 2], 0));
                if (peer_) peer_->wait_done(seq0 + static_cast<unsigned long long>(p - 1), cs_);  // every rank's phase p-2
            }
            ACCO_CUDA(cudaEventRecord(ev.stage_start[static_cast<size_t>(p) * nl + w], cs_));
            float* acc = acc_[static_cast<size_t>(w) * nacc + p % nacc];
            const void* params;
            uint64_t round, tag;
            if (p == 0 && boot) {
                params = theta_act_, round = r0, tag = kTagInit;
            } else if (p % 2 == 1) {
                params = theta_act_, round = r0 + static_cast<uint64_t>((p - 1) / 2), tag = kTagMain;
            } else {
                params = est_act_, round = r0 + static_cast<uint64_t>(p / 2), tag = kTagEstimate;
            }
            int k = 0;
            const bool adaptive = sim_.schedule == kAdaptive && p >= 1;
            const int target = stage_len(p, w, boot);
            while (true) {
                if (!adaptive && k >= target) break;
                if (adaptive && k >= target) {
                    // floor met: the decision is taken when micro-batch k-1
                    // completes, as in on_mb_done (protocols.cpp:566-573) — hand
                    // off iff phase p-1 has completed, else accumulate another.
                    wait_event(ev.mb[(k - 1) % 4]);
                    if (cudaEventQuery(ev.done[p - 1]) == cudaSuccess) break;
                }
                // the loss ring holds every micro-batch loss of this run() until it ends:
                // fail before overwriting one (an adaptive schedule can run long stages)
                ACCO_REQUIRE(mb_counter_ - mb0 < loss_cap_,
                             "loss ring overflow: more than 65536 micro-batches in one run() call");
                const int slot = static_cast<int>(mb_counter_ % loss_cap_);
                micro(w, params, round, tag, k, acc, loss_ring_ + slot);
                ACCO_CUDA(cudaEventRecord(ev.mb[k % 4], cs_));
                mb_phase.push_back(p);
                ++mb_counter_;
                ++k;
            }
            stage_len_rec[static_cast<size_t>(p) * nl + w] = k;
            ev.counts[static_cast<size_t>(p) * nl + w] = static_cast<long long>(k) * B;
            ACCO_CUDA(cudaEventRecord(ev.post[static_cast<size_t>(p) * nl + w], cs_));
        }
        launch_phase(p, p, tot, ev);
        if (p % 2 == 1) snapshot((p - 1) / 2, false);
        if (do_eval && p % 2 == 1) {
            const int t = (p - 1) / 2;
            if ((static_cast<long long>(update_) + t + 1) % sim_.eval_every == 0) {
                ACCO_CUDA(cudaStreamWaitEvent(cs_, ev.done[p], 0));
                if (peer_) peer_->wait_done(seq0 + static_cast<unsigned long long>(p + 1), cs_);
                double* e0 = eval_buf + static_cast<size_t>(t) * 2 * (n_eval_chunks + 1);
                eval(theta_act_, e0, e0 + n_eval_chunks);
                eval(est_act_, e0 + n_eval_chunks + 1, e0 + 2 * n_eval_chunks + 1);
            }
        }
    }
    sync_streams();

    // ---- gather results
    std::vector<int64_t> tot_h(NP);
    ACCO_CUDA(cudaMemcpy(tot_h.data(), tot, NP * sizeof(int64_t), cudaMemcpyDeviceToHost));
    const long long nmb = mb_counter_ - mb0;
    ACCO_REQUIRE(nmb <= loss_cap_, "loss ring overflow: run fewer updates per call");
    std::vector<double> ring(static_cast<size_t>(loss_cap_));
    if (loss_host_)
        std::memcpy(ring.data(), loss_host_, ring.size() * sizeof(double));
    else
        ACCO_CUDA(cudaMemcpy(ring.data(), loss_ring_, ring.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> phase_loss(NP, 0.0);
    for (long long i = 0; i < nmb; ++i)
        phase_loss[static_cast<size_t>(mb_phase[static_cast<size_t>(i)])] += ring[static_cast<size_t>((mb0 + i) % loss_cap_)];
    std::vector<double> evh;
    if (do_eval) {
        evh.resize(static_cast<size_t>(T) * 2 * (n_eval_chunks + 1));
        ACCO_CUDA(cudaMemcpy(evh.data(), eval_buf, evh.size() * sizeof(double), cudaMemcpyDeviceToHost));
    }
    std::vector<int> pf(static_cast<size_t>(NP));
    ACCO_CUDA(cudaMemcpy(pf.data(), phase_flags_, NP * sizeof(int), cudaMemcpyDeviceToHost));
    // the reference's order of events: phase 2t (estimate), phase 2t+1
    // (commit), then TraceBuilder::commit of update t. A non-finite input to
    // either optimizer step throws invalid_argument out of run_protocol
    // (optim.cpp:56-57: no trace, CLI exit 2); a non-finite state or
    // evaluated loss at the commit ends the run with that record (loss = +inf
    // for a non-finite state, protocols.cpp:113-119,164-167: exit 3).
    for (int p = 0; p < NP; ++p)
        if (pf[static_cast<size_t>(p)] & 4)
            throw Error(kLogicError, "protocol: parameter divergence across workers (comm phase " +
                                         std::to_string(p) + " of this run)");
    int first_bad_input = -1;
    for (int p = 0; p < NP && first_bad_input < 0; ++p)
        if (pf[static_cast<size_t>(p)] & 1) first_bad_input = p;
    const int n = model_->cfg().n_samples;
    std::string invalid;  // thrown after this run's resources are released
    for (int t = 0; t < T; ++t) {
        if (first_bad_input >= 0 && first_bad_input <= 2 * t + 1) {
            invalid = "opt_step: non-finite input (update " + std::to_string(update_ + t) +
                      (first_bad_input % 2 == 0 ? ", estimate phase)" : ", commit phase)");
            break;
        }
        UpdateRecord r;
        r.update = static_cast<int>(update_) + t;
        r.time_s = elapsed(base, ev.done[2 * t + 1]) * 1e-3;
        const long long comb = tot_h[2 * t] + tot_h[2 * t + 1];
        samples_cum_ += comb;
        r.samples_cum = samples_cum_;
        long long local = 0;
        for (int w = 0; w < nl; ++w) {
            r.mb_estimate.push_back(stage_len_rec[static_cast<size_t>(2 * t) * nl + w]);
            r.mb_main.push_back(stage_len_rec[static_cast<size_t>(2 * t + 1) * nl + w]);
            local += ev.counts[static_cast<size_t>(2 * t) * nl + w] + ev.counts[static_cast<size_t>(2 * t + 1) * nl + w];
        }
        r.train_loss = (phase_loss[2 * t] + phase_loss[2 * t + 1]) / static_cast<double>(local);
        if (do_eval && (update_ + t + 1) % sim_.eval_every == 0) {
            const double* e0 = evh.data() + static_cast<size_t>(t) * 2 * (n_eval_chunks + 1);
            double l0 = 0, l1 = 0;
            for (int c = 0; c < n_eval_chunks; ++c) {
                l0 += e0[c];
                l1 += e0[n_eval_chunks + 1 + c];
            }
            r.loss = l0 / n;
            r.grad_sq = e0[n_eval_chunks];
            r.grad_sq_estimate = e0[2 * n_eval_chunks + 1];
        }
        const bool evaluated = do_eval && (update_ + t + 1) % sim_.eval_every == 0;
        const bool bad_state = ((pf[static_cast<size_t>(2 * t)] | pf[static_cast<size_t>(2 * t + 1)]) & 2) != 0;
        if (bad_state) r.loss = r.grad_sq = r.grad_sq_estimate = INFINITY;
        st.consumed += comb / B;
        recs.push_back(r);
        if (bad_state || (evaluated && !std::isfinite(r.loss))) {
            st.diverged = 1;
            break;
        }
    }
    st.n_records = static_cast<int>(recs.size());
    st.issued = nmb;
    // timeline: comm phases vs compute stages
    std::vector<std::pair<double, double>> comm_iv, comp_iv;
    for (int p = 0; p < NP; ++p) {
        comm_iv.emplace_back(elapsed(base, ev.start[p]), elapsed(base, ev.done[p]));
        st.opt_ms += elapsed(ev.rs_done[p], ev.opt_done[p]);
        for (int w = 0; w < nl; ++w)
            comp_iv.emplace_back(elapsed(base, ev.stage_start[static_cast<size_t>(p) * nl + w]),
                                 elapsed(base, ev.post[static_cast<size_t>(p) * nl + w]));
    }
    st.opt_launches = NP;
    st.comm_exposed_ms = exposed(comm_iv, comp_iv, &st.comm_busy_ms, &st.compute_busy_ms);
    {
        std::vector<char> init(static_cast<size_t>(NP), 0), used(static_cast<size_t>(NP), 1);
        init[0] = boot;
        build_timeline(NP, ev, base, false, stage_len_rec, init, used);
    }
    st.wall_ms = elapsed(base, ev.done[NP - 1]);
    update_ += T;
    cudaEventDestroy(base);
    cudaFree(tot);
    if (eval_buf) cudaFree(eval_buf);
    if (!invalid.empty()) throw Error(kInvalidArg, invalid);
}

// Synchronous family (SyncEngine, protocols.cpp:218-425). DDP / ZeRO-1: the
// round's bundles are computed at theta and applied at once. DPU: the bundle
// computed in round r-1 at theta^(r-1) is applied while round r's bundle is
// computed at theta^(r) (one-step delay; leading warmup_rounds as DDP). WP: the
// pending bundle is applied, a prediction step on a throwaway state copy gives
// theta-tilde, and round r's bundle is computed there. "slot q" = the bundle
// consumed by phase q; slot T holds the DPU/WP bundle left pending at the end.
void Trainer::run_sync(int T, std::vector<UpdateRecord>& recs, RunStats& st) {
    const int nl = n_local_;
    const int B = sim_.batch_size;
    const int k = sim_.n_grad_accumulation;
    const bool delayed_method = method_ == kDPU || method_ == kWP;
    const int NS = T + 1;  // slots
    PhaseEvents ev;
    ev.n_local = nl;
    ev.post.create(static_cast<size_t>(NS) * nl);
    ev.stage_start.create(static_cast<size_t>(NS) * nl);
    ev.start.create(T);
    ev.cnt_done.create(T);
    ev.rs_done.create(T);
    ev.opt_done.create(T);
    ev.done.create(T);
    ev.counts.assign(static_cast<size_t>(NS) * nl, 0);
    std::vector<int> slot_k(static_cast<size_t>(NS), 0);
    std::vector<char> slot_used(static_cast<size_t>(NS), 0), slot_init(static_cast<size_t>(NS), 0);
    int64_t* tot = nullptr;
    ACCO_CUDA(cudaMalloc(&tot, T * sizeof(int64_t)));
    const bool do_eval = sim_.eval_every > 0;
    const int n_eval_chunks = do_eval ? ceil_div(model_->cfg().n_samples,
                                                  sim_.eval_batch > 0 ? std::min(sim_.eval_batch, model_->cfg().max_batch)
                                                                      : model_->cfg().max_batch)
                                      : 0;
    double* eval_buf = nullptr;  // [T][2 (theta, est)][n_chunks + 1 (gsq)]
    if (do_eval) ACCO_CUDA(cudaMalloc(&eval_buf, static_cast<size_t>(T) * 2 * (n_eval_chunks + 1) * sizeof(double)));
    std::vector<char> est_is_theta(static_cast<size_t>(T), 1);
    std::vector<int> mb_slot;
    const long long mb0 = mb_counter_;
    cudaEvent_t base;
    ACCO_CUDA(cudaEventCreate(&base));
    ACCO_CUDA(cudaEventRecord(base, cs_));
    ACCO_CUDA(cudaStreamWaitEvent(ms_, base, 0));
    const double carried_loss = pending_valid_ ? pending_loss_ : 0.0;
    const unsigned long long seq0 = phase_seq_;  // round r's phase carries peer sequence seq0 + r + 1
    EventArr eval_ev;
    eval_ev.create(1);
    cudaEvent_t eval_done = eval_ev[0];
    if (pending_valid_) {  // bundle left pending by the previous run() call: already resident
        for (int w = 0; w < nl; ++w) {
            ACCO_CUDA(cudaEventRecord(ev.stage_start[static_cast<size_t>(w)], cs_));
            ACCO_CUDA(cudaEventRecord(ev.post[static_cast<size_t>(w)], cs_));
            ev.counts[static_cast<size_t>(w)] = static_cast<long long>(pending_k_) * B;
        }
        slot_k[0] = pending_k_;
        slot_used[0] = 1;
    }
    // one stage per local worker: n micro-batches at params into accumulator parity q, bundle slot `slot`
    auto stage = [&](int slot, int q, const void* params, uint64_t round, uint64_t tag, int n) {
        const int nacc = static_cast<int>(acc_.size()) / nl;
        for (int w = 0; w < nl; ++w) {
            ACCO_CUDA(cudaEventRecord(ev.stage_start[static_cast<size_t>(slot) * nl + w], cs_));
            float* acc = acc_[static_cast<size_t>(w) * nacc + q % nacc];
            for (int j = 0; j < n; ++j) {
                ACCO_REQUIRE(mb_counter_ - mb0 < loss_cap_,
                             "loss ring overflow: more than 65536 micro-batches in one run() call");
                const int ls = static_cast<int>(mb_counter_ % loss_cap_);
                micro(w, params, round, tag, j, acc, loss_ring_ + ls);
                mb_slot.push_back(slot);
                ++mb_counter_;
            }
            ev.counts[static_cast<size_t>(slot) * nl + w] = static_cast<long long>(n) * B;
            ACCO_CUDA(cudaEventRecord(ev.post[static_cast<size_t>(slot) * nl + w], cs_));
        }
        slot_k[static_cast<size_t>(slot)] = n;
        slot_used[static_cast<size_t>(slot)] = 1;
        slot_init[static_cast<size_t>(slot)] = tag == kTagInit;
    };
    for (int r = 0; r < T; ++r) {
        const uint64_t R = static_cast<uint64_t>(update_ + r);
        const bool warm = !delayed_method || (method_ == kDPU && static_cast<long long>(R) < sim_.warmup_rounds);
        if (r >= 1) {
            ACCO_CUDA(cudaStreamWaitEvent(cs_, ev.done[r - 1], 0));
            if (peer_) peer_->wait_done(seq0 + static_cast<unsigned long long>(r), cs_);
        }
        if (warm) {  // ddp_round (protocols.cpp:321-338)
            ACCO_REQUIRE(!pending_valid_, "dpu: warm-up round after the delayed rounds started");
            stage(r, 0, theta_act_, R, kTagMain, k);
            launch_phase(r, 0, tot, ev, true);
        } else if (method_ == kDPU) {  // dpu_round (protocols.cpp:357-379)
            if (!pending_valid_) {
                stage(r, 0, theta_act_, R, kTagInit, 1);  // seed_pending (:340-351)
                pending_slot_ = 0;
                pending_valid_ = true;
            }
            stage(r + 1, pending_slot_ ^ 1, theta_act_, R, kTagMain, k);
            launch_phase(r, pending_slot_, tot, ev, false);
            pending_slot_ ^= 1;
            est_is_theta[static_cast<size_t>(r)] = 0;
        } else {  // wp_round (protocols.cpp:383-424)
            if (!pending_valid_) {
                stage(r, 0, est_act_, R, kTagInit, 1);
                pending_slot_ = 0;
                pending_valid_ = true;
            }
            launch_phase(r, pending_slot_, tot, ev, false);
            ACCO_CUDA(cudaStreamWaitEvent(cs_, ev.done[r], 0));
            if (peer_) peer_->wait_done(seq0 + static_cast<unsigned long long>(r + 1), cs_);
            stage(r + 1, pending_slot_ ^ 1, est_act_, R, kTagMain, k);
            pending_slot_ ^= 1;
            est_is_theta[static_cast<size_t>(r)] = 0;
        }
        snapshot(r, est_is_theta[static_cast<size_t>(r)]);
        if (do_eval && (update_ + r + 1) % sim_.eval_every == 0) {
            ACCO_CUDA(cudaStreamWaitEvent(cs_, ev.done[r], 0));
            if (peer_) peer_->wait_done(seq0 + static_cast<unsigned long long>(r + 1), cs_);
            double* e0 = eval_buf + static_cast<size_t>(r) * 2 * (n_eval_chunks + 1);
            eval(theta_act_, e0, e0 + n_eval_chunks);
            if (!est_is_theta[static_cast<size_t>(r)]) eval(est_act_, e0 + n_eval_chunks + 1, e0 + 2 * n_eval_chunks + 1);
            // DPU's next phase overwrites est_act_ and only waits for the
            // (already posted) fresh stage: order it after the evaluation too
            ACCO_CUDA(cudaEventRecord(eval_done, cs_));
            ACCO_CUDA(cudaStreamWaitEvent(ms_, eval_done, 0));
        }
    }
    sync_streams();
    std::vector<int64_t> tot_h(T);
    ACCO_CUDA(cudaMemcpy(tot_h.data(), tot, T * sizeof(int64_t), cudaMemcpyDeviceToHost));
    const long long nmb = mb_counter_ - mb0;
    ACCO_REQUIRE(nmb <= loss_cap_, "loss ring overflow: run fewer updates per call");
    std::vector<double> ring(static_cast<size_t>(loss_cap_));
    if (loss_host_)
        std::memcpy(ring.data(), loss_host_, ring.size() * sizeof(double));
    else
        ACCO_CUDA(cudaMemcpy(ring.data(), loss_ring_, ring.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> sl(static_cast<size_t>(NS), 0.0);
    sl[0] = carried_loss;
    for (long long i = 0; i < nmb; ++i)
        sl[static_cast<size_t>(mb_slot[static_cast<size_t>(i)])] += ring[static_cast<size_t>((mb0 + i) % loss_cap_)];
    std::vector<double> evh;
    if (do_eval) {
        evh.resize(static_cast<size_t>(T) * 2 * (n_eval_chunks + 1));
        ACCO_CUDA(cudaMemcpy(evh.data(), eval_buf, evh.size() * sizeof(double), cudaMemcpyDeviceToHost));
    }
    std::vector<int> pf(static_cast<size_t>(2 * T));
    ACCO_CUDA(cudaMemcpy(pf.data(), phase_flags_, 2 * T * sizeof(int), cudaMemcpyDeviceToHost));
    for (int r = 0; r < T; ++r)
        if (pf[static_cast<size_t>(2 * r)] & 4)
            throw Error(kLogicError, "protocol: parameter divergence across workers (round " + std::to_string(r) +
                                         " of this run)");
    const int n = model_->cfg().n_samples;
    std::string invalid;  // thrown after this run's resources are released
    for (int r = 0; r < T; ++r) {
        // apply_and_commit (protocols.cpp:298-318): a non-finite mean ends the
        // run before the round's record; a non-finite new state or evaluated
        // loss ends it with the record (loss = +inf for the state). WP's
        // prediction opt_step on a non-finite theta throws invalid_argument
        // (protocols.cpp:398-403, optim.cpp:56-57).
        if (pf[static_cast<size_t>(2 * r)] & 1) {
            st.diverged = 1;
            break;
        }
        if (pf[static_cast<size_t>(2 * r + 1)] & 1) {
            invalid = "opt_step: non-finite input (update " + std::to_string(update_ + r) + ", prediction step)";
            break;
        }
        UpdateRecord rec;
        rec.update = static_cast<int>(update_) + r;
        rec.time_s = elapsed(base, ev.done[r]) * 1e-3;
        samples_cum_ += tot_h[r];
        rec.samples_cum = samples_cum_;
        const int kc = slot_k[static_cast<size_t>(r)];
        rec.train_loss = sl[static_cast<size_t>(r)] / static_cast<double>(static_cast<long long>(nl) * kc * B);
        for (int w = 0; w < nl; ++w) {
            rec.mb_main.push_back(kc);
            rec.mb_estimate.push_back(0);
        }
        if (do_eval && (update_ + r + 1) % sim_.eval_every == 0) {
            const double* e0 = evh.data() + static_cast<size_t>(r) * 2 * (n_eval_chunks + 1);
            double l0 = 0;
            for (int c = 0; c < n_eval_chunks; ++c) l0 += e0[c];
            rec.loss = l0 / n;
            rec.grad_sq = e0[n_eval_chunks];
            rec.grad_sq_estimate = est_is_theta[static_cast<size_t>(r)] ? rec.grad_sq : e0[2 * n_eval_chunks + 1];
        }
        const bool evaluated = do_eval && (update_ + r + 1) % sim_.eval_every == 0;
        const bool bad_state = ((pf[static_cast<size_t>(2 * r)] | pf[static_cast<size_t>(2 * r + 1)]) & 2) != 0;
        if (bad_state) rec.loss = rec.grad_sq = rec.grad_sq_estimate = INFINITY;
        st.consumed += tot_h[r] / B;
        recs.push_back(rec);
        if (bad_state || (evaluated && !std::isfinite(rec.loss))) {
            st.diverged = 1;
            break;
        }
    }
    st.n_records = static_cast<int>(recs.size());
    st.issued = nmb;
    if (delayed_method && pending_valid_) {
        pending_k_ = slot_k[static_cast<size_t>(T)];
        pending_loss_ = sl[static_cast<size_t>(T)];
        st.discarded = static_cast<long long>(pending_k_) * nl;  // if the run ended here (protocols.cpp:246)
    }
    std::vector<std::pair<double, double>> comm_iv, comp_iv;
    for (int r = 0; r < T; ++r) {
        comm_iv.emplace_back(elapsed(base, ev.start[r]), elapsed(base, ev.done[r]));
        st.opt_ms += elapsed(ev.rs_done[r], ev.opt_done[r]);
    }
    for (int q = 0; q < NS; ++q) {
        if (!slot_used[static_cast<size_t>(q)]) continue;
        for (int w = 0; w < nl; ++w)
            comp_iv.emplace_back(elapsed(base, ev.stage_start[static_cast<size_t>(q) * nl + w]),
                                 elapsed(base, ev.post[static_cast<size_t>(q) * nl + w]));
    }
    st.opt_launches = T * (method_ == kWP ? 2 : 1);
    st.comm_exposed_ms = exposed(comm_iv, comp_iv, &st.comm_busy_ms, &st.compute_busy_ms);
    {
        std::vector<int> k_sw;
        for (int q = 0; q < NS; ++q)
            for (int w = 0; w < nl; ++w) k_sw.push_back(slot_k[static_cast<size_t>(q)]);
        build_timeline(T, ev, base, true, k_sw, slot_init, slot_used);
    }
    st.wall_ms = elapsed(base, ev.done[T - 1]);
    update_ += T;
    cudaEventDestroy(base);
    cudaFree(tot);
    if (eval_buf) cudaFree(eval_buf);
    if (!invalid.empty()) throw Error(kInvalidArg, invalid);
}

}  // namespace acco
