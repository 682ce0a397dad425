// The drop-in boundary exercised from C++ the way a reference maintainer
// would bind it: this program includes the REFERENCE's
// headers (accosim, /root/reference/proj/include) next to include/acco.h,
// links the reference's own library (oracle/_ref/libaccosim_ref.a, built from
// its sources by oracle/Makefile) and _acco_b200.so, converts the reference's
// types with the INTEGRATION.md shim, and checks the B200 entry points against
// the reference's functions on identical inputs:
//   rng::derive / Stream::below           vs acco_rng_derive / acco_sample_indices   (bit-exact)
//   shard_partition                       vs acco_shard_partition                    (bit-exact)
//   scheduled_lr                          vs acco_scheduled_lr                       (bit-exact)
//   opt_step (25 steps, sgd/adam/adamw)   vs acco_opt_commit on device               (fp32: rel <= 1e-6)
//   sharded_opt_step (N = 3, ragged)      vs acco_opt_commit per shard_partition range
//   opt_step on a transient copy          vs acco_opt_estimate (state untouched)
//   run_protocol ACCO / DDP record counts vs acco_trainer_run (mb_main / mb_estimate /
//                                            samples_cum, bit-exact; free fabric)
// Test infrastructure (tests/test_gpu_reference_dropin.py runs it on the GPU
// box). Prints one PASS/FAIL line per check; exit code = number of failures,
// the reference acceptance binary's convention.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "acco.h"
#include "accosim/collectives.hpp"
#include "accosim/optim.hpp"
#include "accosim/problems.hpp"
#include "accosim/protocols.hpp"
#include "accosim/rng.hpp"
#include "accosim/shard.hpp"

namespace {

int g_fail = 0;

void check(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++g_fail;
}

// accosim::OptimizerConfig -> acco_opt_cfg
acco_opt_cfg to_c(const accosim::OptimizerConfig& c) {
    return {static_cast<int>(c.kind), c.learning_rate, c.adam_beta1, c.adam_beta2, c.adam_eps, c.weight_decay,
            c.scheduler == accosim::LrSchedule::cosine ? 1 : 0, c.n_warmup_steps, c.total_steps,
            c.cosine_min_factor};
}

double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1e-300));
}

std::vector<double> gauss(uint64_t seed, size_t n, double scale) {
    accosim::rng::Stream s(seed);
    std::vector<double> v(n);
    for (double& x : v) x = scale * s.gaussian();
    return v;
}

struct DevShard {  // fp32 device state of one shard [lo, hi)
    float *theta = nullptr, *m = nullptr, *v = nullptr, *g = nullptr, *out = nullptr;
    int64_t* total = nullptr;
    size_t n = 0;
    explicit DevShard(const std::vector<double>& th) : n(th.size()) {
        std::vector<float> f(th.begin(), th.end());
        cudaMalloc(&theta, n * 4);
        cudaMalloc(&m, n * 4);
        cudaMalloc(&v, n * 4);
        cudaMalloc(&g, n * 4);
        cudaMalloc(&out, n * 4);
        cudaMalloc(&total, 8);
        cudaMemcpy(theta, f.data(), n * 4, cudaMemcpyHostToDevice);
        cudaMemset(m, 0, n * 4);
        cudaMemset(v, 0, n * 4);
        const int64_t one = 1;
        cudaMemcpy(total, &one, 8, cudaMemcpyHostToDevice);
    }
    ~DevShard() {
        cudaFree(theta), cudaFree(m), cudaFree(v), cudaFree(g), cudaFree(out), cudaFree(total);
    }
    void set_grad(const std::vector<double>& gd) {
        std::vector<float> f(gd.begin(), gd.end());
        cudaMemcpy(g, f.data(), n * 4, cudaMemcpyHostToDevice);
    }
    std::vector<double> get(const float* p) const {
        std::vector<float> f(n);
        cudaMemcpy(f.data(), p, n * 4, cudaMemcpyDeviceToHost);
        return std::vector<double>(f.begin(), f.end());
    }
};

accosim::OptimizerConfig opt_cfg(accosim::OptKind kind) {
    accosim::OptimizerConfig c;
    c.kind = kind;
    c.learning_rate = kind == accosim::OptKind::sgd ? 0.05 : 1e-3;
    c.weight_decay = 0.1;
    c.adam_beta2 = 0.95;
    c.scheduler = accosim::LrSchedule::cosine;
    c.n_warmup_steps = 3;
    c.total_steps = 25;
    c.cosine_min_factor = 0.1;
    return c;
}

}  // namespace

int main() {
    // ---- rng: seeds and micro-batch sample indices (token indexing)
    {
        bool ok = true;
        for (uint64_t m = 0; m < 50; ++m)
            ok &= acco_rng_derive(m, m + 1, 7, 2, m % 5) == accosim::rng::derive(m, m + 1, 7, 2, m % 5);
        const uint64_t seed = accosim::rng::derive(1, 0, 3, 2, 0);
        std::vector<int32_t> idx(64);
        ok &= acco_sample_indices(seed, 64, 4096, idx.data()) == ACCO_OK;
        accosim::rng::Stream s(seed);
        for (int i = 0; i < 64; ++i) ok &= idx[static_cast<size_t>(i)] == static_cast<int32_t>(s.below(4096));
        check(ok, "rng::derive / Stream::below == acco_rng_derive / acco_sample_indices");
    }
    // ---- shard_partition
    {
        bool ok = true;
        for (uint64_t dim : {0ull, 3ull, 5ull, 437760ull, 124439808ull, 1000003ull})
            for (int n : {1, 2, 3, 4, 8}) {
                const accosim::ShardLayout r = accosim::shard_partition(dim, n);
                std::vector<uint64_t> lo(static_cast<size_t>(n)), hi(static_cast<size_t>(n));
                ok &= acco_shard_partition(dim, n, lo.data(), hi.data()) == ACCO_OK;
                for (int w = 0; w < n; ++w) ok &= lo[w] == r.lo(w) && hi[w] == r.hi(w);
            }
        check(ok, "shard_partition == acco_shard_partition");
    }
    // ---- scheduled_lr
    {
        bool ok = true;
        for (auto k : {accosim::OptKind::sgd, accosim::OptKind::adamw}) {
            const accosim::OptimizerConfig c = opt_cfg(k);
            const acco_opt_cfg cc = to_c(c);
            for (long long t = 0; t < 30; ++t) ok &= acco_scheduled_lr(&cc, t) == accosim::scheduled_lr(c, t);
        }
        check(ok, "scheduled_lr == acco_scheduled_lr (bitwise)");
    }
    // ---- opt_step trajectories (persistent commit) for every optimizer kind
    for (auto kind : {accosim::OptKind::sgd, accosim::OptKind::adam, accosim::OptKind::adamw}) {
        const size_t d = 1000;
        const accosim::OptimizerConfig c = opt_cfg(kind);
        const acco_opt_cfg cc = to_c(c);
        std::vector<double> th = gauss(11, d, 0.5);
        // the reference and the device start from the same fp32-representable theta
        for (double& x : th) x = static_cast<float>(x);
        accosim::OptimizerState st = accosim::OptimizerState::for_range(c, 0, d);
        DevShard dev(th);
        acco_shard_state ds{0, dev.theta, dev.m, dev.v, 0, d};
        double worst = 0;
        for (int s = 0; s < 25; ++s) {
            std::vector<double> g = gauss(100 + s, d, 1.0);
            for (double& x : g) x = static_cast<float>(x);
            dev.set_grad(g);
            auto [next, upd] = accosim::opt_step(std::move(st), th, g, c);
            st = std::move(next);
            th = std::move(upd);
            acco_opt_commit(&cc, &ds, dev.g, nullptr, dev.total, nullptr, nullptr, ACCO_DTYPE_F32, nullptr, nullptr);
            cudaDeviceSynchronize();
            worst = std::max(worst, rel(dev.get(dev.theta), th));
        }
        char msg[160];
        std::snprintf(msg, sizeof msg, "opt_step x25 == acco_opt_commit (kind %d, worst rel %.2e <= 1e-6, step %lld)",
                      static_cast<int>(kind), worst, ds.step);
        check(worst <= 1e-6 && ds.step == st.step, msg);
    }
    // ---- sharded_opt_step (N = 3, ragged) vs per-shard commits; estimate on a transient copy
    {
        const size_t d = 1001;
        const int N = 3;
        const accosim::OptimizerConfig c = opt_cfg(accosim::OptKind::adamw);
        const acco_opt_cfg cc = to_c(c);
        std::vector<double> th = gauss(5, d, 0.3);
        for (double& x : th) x = static_cast<float>(x);
        const accosim::ShardLayout layout = accosim::shard_partition(d, N);
        std::vector<accosim::OptimizerState> states;
        for (int w = 0; w < N; ++w) states.push_back(accosim::OptimizerState::for_range(c, layout.lo(w), layout.hi(w)));
        accosim::Fabric fabric(N);
        std::vector<double> g = gauss(6, d, 1.0);
        for (double& x : g) x = static_cast<float>(x);
        std::vector<std::vector<double>> shards;
        for (int w = 0; w < N; ++w)
            shards.emplace_back(g.begin() + static_cast<long>(layout.lo(w)), g.begin() + static_cast<long>(layout.hi(w)));
        // estimate: the reference's transient copy (protocols.cpp:654)
        std::vector<accosim::OptimizerState> transient = states;
        const std::vector<double> est = accosim::sharded_opt_step(transient, th, shards, c, layout, fabric);
        const std::vector<double> ref = accosim::sharded_opt_step(states, th, shards, c, layout, fabric);
        std::vector<double> got_est(d), got(d);
        bool untouched = true;
        for (int w = 0; w < N; ++w) {
            std::vector<double> sl(th.begin() + static_cast<long>(layout.lo(w)), th.begin() + static_cast<long>(layout.hi(w)));
            DevShard dev(sl);
            dev.set_grad(shards[static_cast<size_t>(w)]);
            acco_shard_state ds{0, dev.theta, dev.m, dev.v, layout.lo(w), layout.hi(w)};
            acco_opt_estimate(&cc, &ds, dev.g, dev.total, dev.out, ACCO_DTYPE_F32, nullptr, nullptr);
            cudaDeviceSynchronize();
            const std::vector<double> e = dev.get(dev.out), th_after = dev.get(dev.theta), m_after = dev.get(dev.m);
            untouched &= ds.step == 0 && rel(th_after, sl) == 0.0;
            for (double x : m_after) untouched &= x == 0.0;
            acco_opt_commit(&cc, &ds, dev.g, nullptr, dev.total, nullptr, nullptr, ACCO_DTYPE_F32, nullptr, nullptr);
            cudaDeviceSynchronize();
            const std::vector<double> t = dev.get(dev.theta);
            for (size_t j = 0; j < t.size(); ++j) {
                got[layout.lo(w) + j] = t[j];
                got_est[layout.lo(w) + j] = e[j];
            }
        }
        check(rel(got, ref) <= 1e-6, "sharded_opt_step (N=3, ragged) == acco_opt_commit per shard");
        check(rel(got_est, est) <= 1e-6 && untouched, "transient-copy opt_step == acco_opt_estimate (state untouched)");
    }
    // ---- protocol record counts: run_protocol vs acco_trainer_run (free fabric, floor schedule)
    for (int method : {ACCO_METHOD_ACCO, ACCO_METHOD_DDP}) {
        accosim::SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 3;
        sim.n_grad_accumulation = 2;
        sim.master_seed = 9;
        const int T = 4;
        const accosim::Problem p = accosim::make_quadratic(3, 4, 0.2, 1.0, 0.1);
        accosim::OptimizerConfig oc = opt_cfg(accosim::OptKind::adamw);
        const accosim::RunTrace tr = accosim::run_protocol(
            method == ACCO_METHOD_ACCO ? accosim::Method::acco : accosim::Method::ddp, p, oc, sim, T);
        acco_lm_cfg lm{64, 32, 2, 2, 16, 32, 3, ACCO_DTYPE_F32, 3, 0, 0, 0, 0, 0.0};
        acco_model* model = nullptr;
        acco_model_create(&lm, &model);
        acco_sim_cfg s{2, 3, 2, 0, 9, ACCO_SCHED_FLOOR, nullptr, 0, 0, 0, nullptr, 0.0, 0, 0, 0, 0.0};
        oc.total_steps = T;
        const acco_opt_cfg cc = to_c(oc);
        acco_trainer* trn = nullptr;
        int rc = acco_trainer_create(model, &cc, &s, method, nullptr, &trn);
        std::vector<float> th0(static_cast<size_t>(acco_model_num_params(model)));
        acco_model_theta0(model, 9, th0.data());
        acco_trainer_set_theta(trn, th0.data());
        std::vector<acco_record> recs(T);
        std::vector<int32_t> counts(static_cast<size_t>(T) * 2 * 2);
        acco_run_stats st{};
        rc |= acco_trainer_run(trn, T, recs.data(), counts.data(), nullptr, &st);
        bool ok = rc == ACCO_OK && st.n_records == T && static_cast<int>(tr.records.size()) == T;
        for (int t = 0; ok && t < T; ++t) {
            const auto& r = tr.records[static_cast<size_t>(t)];
            ok &= recs[t].update == r.update && recs[t].samples_cum == r.samples_cum;
            for (int w = 0; w < 2; ++w)
                ok &= counts[(t * 2 + 0) * 2 + w] == r.mb_estimate[static_cast<size_t>(w)] &&
                      counts[(t * 2 + 1) * 2 + w] == r.mb_main[static_cast<size_t>(w)];
        }
        acco_trainer_destroy(trn);
        acco_model_destroy(model);
        check(ok, method == ACCO_METHOD_ACCO ? "run_protocol(acco) counts / samples_cum == acco_trainer_run"
                                             : "run_protocol(ddp) counts / samples_cum == acco_trainer_run");
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
