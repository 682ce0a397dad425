// C-ABI of the model plugin and the trainer (include/acco.h).
#include "acco.h"
#include "capi_util.h"
#include "engine.h"
#include "lm_kernels.h"

#include <cmath>
#include <cstring>
#include <memory>

using namespace acco;

struct acco_model {
    std::unique_ptr<GPTModel> impl;
};

struct acco_trainer {
    std::unique_ptr<Trainer> impl;
};

struct acco_peer {
    std::unique_ptr<PeerFabric> impl;
};

namespace {
LMConfig to_lm(const acco_lm_cfg& c) {
    LMConfig l;
    l.vocab = c.vocab;
    l.d_model = c.d_model;
    l.n_layer = c.n_layer;
    l.n_head = c.n_head;
    l.seq_len = c.seq_len;
    l.n_samples = c.n_samples;
    l.data_seed = c.data_seed;
    l.precision = c.precision;
    l.max_batch = c.max_batch;
    l.host_data = c.host_data;
    l.arch = c.arch;
    l.n_kv_head = c.n_kv_head;
    l.d_ff = c.d_ff;
    l.rope_base = c.rope_base;
    return l;
}
SimCfg to_sim(const acco_sim_cfg* sim) {
    SimCfg s;
    s.n_workers = sim->n_workers;
    s.batch_size = sim->batch_size;
    s.n_grad_accumulation = sim->n_grad_accumulation;
    s.warmup_rounds = sim->warmup_rounds;
    s.master_seed = sim->master_seed;
    s.schedule = sim->schedule;
    ACCO_REQUIRE(s.schedule >= kFloor && s.schedule <= kReplay, "sim: unknown schedule");
    if (sim->replay && sim->replay_len > 0) s.replay.assign(sim->replay, sim->replay + sim->replay_len);
    ACCO_REQUIRE(s.schedule != kReplay || !s.replay.empty(), "sim: replay schedule requires counts");
    s.eval_every = sim->eval_every;
    s.eval_batch = sim->eval_batch;
    if (sim->throttle_ns) s.throttle_ns.assign(sim->throttle_ns, sim->throttle_ns + sim->n_workers);
    ACCO_REQUIRE(sim->comm_delay_ns >= 0.0, "sim: comm_delay_ns >= 0");
    s.comm_delay_ns = sim->comm_delay_ns;
    s.check_replicas = sim->check_replicas;
    s.throttle_host = sim->throttle_host;
    ACCO_REQUIRE(sim->comm_standin_ctas >= 0 && sim->comm_standin_bytes >= 0, "sim: comm stand-in sizes >= 0");
    s.comm_standin_ctas = sim->comm_standin_ctas;
    s.comm_standin_bytes = sim->comm_standin_bytes;
    return s;
}
}  // namespace

namespace acco {
// Device time of one micro-batch (fwd + bwd + accumulate), mean of `reps` (ns).
double time_micro_batch(GPTModel& g, int batch, int reps) {
    const int64_t n = g.num_params();
    const size_t eb = g.act_bytes();
    std::vector<float> th(static_cast<size_t>(n));
    lm_default_theta0(g.cfg(), 1, th.data());
    void* params = nullptr;
    float* grad = nullptr;
    double* slot = nullptr;
    ACCO_CUDA(cudaMalloc(&params, n * eb));
    ACCO_CUDA(cudaMalloc(&grad, n * sizeof(float)));
    ACCO_CUDA(cudaMalloc(&slot, sizeof(double)));
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ACCO_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    ACCO_CUDA(cudaEventCreate(&e0));
    ACCO_CUDA(cudaEventCreate(&e1));
    {
        float* tmp = nullptr;
        ACCO_CUDA(cudaMalloc(&tmp, n * sizeof(float)));
        ACCO_CUDA(cudaMemcpy(tmp, th.data(), n * sizeof(float), cudaMemcpyHostToDevice));
        f32_to(tmp, params, g.act_dtype(), n, s);
        ACCO_CUDA(cudaStreamSynchronize(s));
        cudaFree(tmp);
    }
    g.micro_batch(params, 1, 0, 0, batch, grad, slot, s, false);  // warm-up
    ACCO_CUDA(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) g.micro_batch(params, 2 + r, 0, 0, batch, grad, slot, s, r > 0);
    ACCO_CUDA(cudaEventRecord(e1, s));
    ACCO_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    ACCO_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    cudaFree(params);
    cudaFree(grad);
    cudaFree(slot);
    return 1e6 * ms / reps;
}
}  // namespace acco

extern "C" {

int acco_model_create(const acco_lm_cfg* cfg, acco_model** out) {
    return guarded([&] {
        ACCO_REQUIRE(cfg && out, "acco_model_create: null argument");
        *out = new acco_model{std::make_unique<GPTModel>(to_lm(*cfg))};
    });
}

int acco_model_destroy(acco_model* m) {
    return guarded([&] { delete m; });
}

long long acco_model_num_params(const acco_model* m) { return m ? m->impl->num_params() : -1; }

int acco_model_theta0(const acco_model* m, uint64_t master_seed, float* host_out) {
    return guarded([&] { lm_default_theta0(m->impl->cfg(), master_seed, host_out); });
}

int acco_model_dataset(const acco_model* m, int32_t* host_out) {
    return guarded([&] {
        std::vector<int32_t> d = lm_dataset(m->impl->cfg());
        std::memcpy(host_out, d.data(), d.size() * sizeof(int32_t));
    });
}

int acco_model_stochastic_grad(acco_model* m, const void* params, uint64_t stream_seed, int batch,
                               float* grad_acc, double* loss_sum_dev, void* stream) {
    return guarded([&] {
        m->impl->micro_batch(params, stream_seed, 0, 0, batch, grad_acc, loss_sum_dev,
                             static_cast<cudaStream_t>(stream));
    });
}

int acco_model_value_and_grad(acco_model* m, const void* params, double* loss_out, float* grad_out, void* stream) {
    return guarded([&] {
        GPTModel& g = *m->impl;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int n = g.cfg().n_samples, eb = g.cfg().max_batch;
        const int nch = ceil_div(n, eb);
        double* slots = nullptr;
        float* grad = grad_out;
        ACCO_CUDA(cudaMalloc(&slots, nch * sizeof(double)));
        if (!grad) ACCO_CUDA(cudaMalloc(&grad, g.num_params() * sizeof(float)));
        ACCO_CUDA(cudaMemsetAsync(grad, 0, g.num_params() * sizeof(float), s));
        int ci = 0;
        for (int c = 0; c < n; c += eb, ++ci) g.micro_batch(params, 0, 1, c, std::min(eb, n - c), grad, slots + ci, s);
        scale_f32(grad, 1.0 / n, g.num_params(), s);
        std::vector<double> h(static_cast<size_t>(nch));
        ACCO_CUDA(cudaMemcpyAsync(h.data(), slots, nch * sizeof(double), cudaMemcpyDeviceToHost, s));
        ACCO_CUDA(cudaStreamSynchronize(s));
        double l = 0;
        for (double v : h) l += v;
        *loss_out = l / n;
        cudaFree(slots);
        if (!grad_out) cudaFree(grad);
    });
}


int acco_model_time_micro_batch(acco_model* m, int batch, int reps, double* ns_out) {
    return guarded([&] {
        ACCO_REQUIRE(m && ns_out && reps >= 1, "acco_model_time_micro_batch: bad argument");
        *ns_out = time_micro_batch(*m->impl, batch, reps);
    });
}

int acco_trainer_create(acco_model* model, const acco_opt_cfg* opt, const acco_sim_cfg* sim, int method,
                        acco_comm* comm, acco_trainer** out) {
    return guarded([&] {
        ACCO_REQUIRE(model && opt && sim && out, "acco_trainer_create: null argument");
        *out = new acco_trainer{
            std::make_unique<Trainer>(model->impl.get(), from_c(*opt), to_sim(sim), method, comm_impl(comm))};
    });
}

int acco_peer_create(int nranks, int rank, int device, acco_peer** out) {
    return guarded([&] {
        ACCO_REQUIRE(out, "acco_peer_create: null argument");
        *out = new acco_peer{std::make_unique<PeerFabric>(nranks, rank, device)};
    });
}

int acco_peer_destroy(acco_peer* p) {
    return guarded([&] { delete p; });
}

int acco_trainer_create_peer(acco_model* model, const acco_opt_cfg* opt, const acco_sim_cfg* sim, int method,
                             acco_peer* peer, acco_trainer** out) {
    return guarded([&] {
        ACCO_REQUIRE(model && opt && sim && peer && out, "acco_trainer_create_peer: null argument");
        *out = new acco_trainer{std::make_unique<Trainer>(model->impl.get(), from_c(*opt), to_sim(sim), method,
                                                          nullptr, peer->impl.get())};
    });
}

long long acco_trainer_peer_blob_bytes(const acco_trainer* t) {
    return t && t->impl->peer() ? static_cast<long long>(t->impl->peer()->blob_bytes()) : -1;
}

int acco_trainer_peer_export(const acco_trainer* t, void* blob) {
    return guarded([&] {
        ACCO_REQUIRE(t && t->impl->peer() && blob, "acco_trainer_peer_export: not a peer-fabric trainer");
        t->impl->peer()->export_blob(blob);
    });
}

int acco_trainer_peer_connect(acco_trainer* t, const void* blobs) {
    return guarded([&] {
        ACCO_REQUIRE(t && t->impl->peer() && blobs, "acco_trainer_peer_connect: not a peer-fabric trainer");
        t->impl->peer()->connect(blobs);
    });
}

int acco_trainer_destroy(acco_trainer* t) {
    return guarded([&] { delete t; });
}

int acco_trainer_set_theta(acco_trainer* t, const float* host_theta) {
    return guarded([&] { t->impl->set_theta(host_theta); });
}

int acco_trainer_get_theta(acco_trainer* t, int which, float* host_out) {
    return guarded([&] {
        ACCO_REQUIRE(which >= 0 && which <= 2, "get_theta: which in {0,1,2}");
        t->impl->get_theta(which, host_out);
    });
}

int acco_trainer_n_local(const acco_trainer* t) { return t ? t->impl->n_local() : 0; }

int acco_trainer_timeline(const acco_trainer* t, acco_interval* out, int cap, int* n_out) {
    return guarded([&] {
        ACCO_REQUIRE(t && n_out, "acco_trainer_timeline: null argument");
        const auto& tl = t->impl->timeline();
        *n_out = static_cast<int>(tl.size());
        for (int i = 0; out && i < cap && i < static_cast<int>(tl.size()); ++i) {
            const auto& iv = tl[static_cast<size_t>(i)];
            out[i] = acco_interval{iv.worker, iv.stream, iv.kind, iv.micro_batches, iv.t_start, iv.t_end, iv.bytes};
        }
    });
}

int acco_trainer_run(acco_trainer* t, int t_updates, acco_record* recs, int32_t* mb_counts, float* theta_history,
                     acco_run_stats* stats) {
    int diverged = 0;
    int rc = guarded([&] {
        std::vector<UpdateRecord> r;
        RunStats st;
        t->impl->run(t_updates, r, st, theta_history);
        const int nl = t->impl->n_local();
        for (size_t i = 0; i < r.size(); ++i) {
            if (recs) {
                recs[i].update = r[i].update;
                recs[i].time_s = r[i].time_s;
                recs[i].loss = r[i].loss;
                recs[i].grad_sq = r[i].grad_sq;
                recs[i].grad_sq_estimate = r[i].grad_sq_estimate;
                recs[i].lyapunov = r[i].lyapunov;
                recs[i].samples_cum = r[i].samples_cum;
                recs[i].train_loss = r[i].train_loss;
            }
            if (mb_counts)
                for (int w = 0; w < nl; ++w) {
                    mb_counts[(i * 2 + 0) * nl + w] = r[i].mb_estimate[static_cast<size_t>(w)];
                    mb_counts[(i * 2 + 1) * nl + w] = r[i].mb_main[static_cast<size_t>(w)];
                }
        }
        if (stats) {
            stats->issued_micro_batches = st.issued;
            stats->consumed_micro_batches = st.consumed;
            stats->discarded_micro_batches = st.discarded;
            stats->wall_ms = st.wall_ms;
            stats->compute_busy_ms = st.compute_busy_ms;
            stats->comm_busy_ms = st.comm_busy_ms;
            stats->comm_exposed_ms = st.comm_exposed_ms;
            stats->opt_ms = st.opt_ms;
            stats->opt_launches = st.opt_launches;
            stats->diverged = st.diverged;
            stats->h2d_bytes = st.h2d_bytes;
            stats->d2h_bytes = st.d2h_bytes;
            stats->n_records = st.n_records;
        }
        if (st.diverged) diverged = 1;
    });
    if (rc == kOk && diverged) {
        set_last_error("run diverged: non-finite parameters or evaluated loss");
        return kDiverged;
    }
    return rc;
}

}  // extern "C"
