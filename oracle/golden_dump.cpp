// Golden-vector generator: runs the REFERENCE accosim library (built from its
// own sources by oracle/Makefile) and writes JSON fixtures to tests/golden/.
// Test infrastructure only. Each fixture pins one §8(a) row of SURVEY.md:
//   rng.json       rng::derive / Stream            (proj/include/accosim/rng.hpp:13-56)
//   shard.json     shard_partition                 (proj/include/accosim/shard.hpp:24-38)
//   lr.json        scheduled_lr                    (proj/src/optim.cpp:37-48)
//   optim.json     opt_step / sharded_opt_step     (proj/src/optim.cpp:50-119)
//   fabric.json    Fabric RS / AG / AR / counts    (proj/src/collectives.cpp:36-91)
//   protocols.json run_protocol ACCO/DDP/DPU/WP traces (proj/src/protocols.cpp:191-742)
//   io/            write_run_outputs of one run + the trace it was written from
//                  (proj/src/csvio.cpp:12-102, config.cpp:147-157)
//   memory.json    memory_model_bytes / memory_reported_gb (proj/src/convergence.cpp:182-205)
//   divergence.json partial traces / exceptions of diverging runs
//                  (protocols.cpp:113-119,164-167,298-306; optim.cpp:56-57;
//                  the case of proj/tests/test_protocols.cpp:328-336)
#include <cmath>
#include <cstdio>
#include <limits>
#include <fstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "accosim/collectives.hpp"
#include "accosim/config.hpp"
#include "accosim/convergence.hpp"
#include "accosim/csvio.hpp"
#include "accosim/optim.hpp"
#include "accosim/problems.hpp"
#include "accosim/protocols.hpp"
#include "accosim/rng.hpp"
#include "accosim/shard.hpp"

using namespace accosim;
using json = nlohmann::json;

static std::vector<double> rand_vec(std::uint64_t seed, int n, double scale) {
    rng::Stream s(seed);
    std::vector<double> v(static_cast<std::size_t>(n));
    for (double& x : v) x = scale * s.gaussian();
    return v;
}

static void write(const std::string& dir, const std::string& name, const json& j) {
    std::ofstream out(dir + "/" + name);
    out << j.dump() << "\n";
    std::printf("wrote %s/%s\n", dir.c_str(), name.c_str());
}

static json rng_fixture() {
    json j;
    json derives = json::array();
    for (std::uint64_t m : std::vector<std::uint64_t>{1ull, 7ull, 0xdeadbeefull, 0xffffffffffffffffull})
        for (std::uint64_t a : std::vector<std::uint64_t>{0ull, 1ull, 3ull})
            for (std::uint64_t b : std::vector<std::uint64_t>{0ull, 2ull, 17ull}) {
                std::uint64_t c = a + 1, d = b * 3;
                derives.push_back({m, a, b, c, d, rng::derive(m, a, b, c, d)});
            }
    j["derive"] = derives;
    json streams = json::array();
    for (std::uint64_t seed : std::vector<std::uint64_t>{0ull, 1ull, 42ull, rng::derive(1, 0, 0, 1, 0)}) {
        rng::Stream s(seed);
        json e;
        e["seed"] = seed;
        std::vector<std::uint64_t> u;
        for (int i = 0; i < 8; ++i) u.push_back(s.next_u64());
        e["next_u64"] = u;
        std::vector<double> un, ga;
        for (int i = 0; i < 8; ++i) un.push_back(s.uniform01());
        for (int i = 0; i < 8; ++i) ga.push_back(s.gaussian());
        e["uniform01"] = un;
        e["gaussian"] = ga;
        std::vector<std::uint64_t> bl;
        for (std::uint64_t n : std::vector<std::uint64_t>{1ull, 2ull, 10ull, 256ull, 50257ull, 4096ull}) bl.push_back(s.below(n));
        e["below"] = bl;
        streams.push_back(e);
    }
    j["streams"] = streams;
    return j;
}

static json shard_fixture() {
    json cases = json::array();
    std::vector<std::pair<std::size_t, int>> dn = {{4, 2},      {5, 2},        {3, 4},       {0, 3},
                                                   {437760, 2}, {124439808, 8}, {354823168, 8},
                                                   {10000001, 8}, {7, 3},      {1, 1},        {17, 5}};
    for (auto [d, n] : dn) {
        ShardLayout l = shard_partition(d, n);
        json r = json::array();
        for (int w = 0; w < n; ++w) r.push_back({l.lo(w), l.hi(w)});
        cases.push_back({{"dim", d}, {"n", n}, {"ranges", r}});
    }
    return cases;
}

static json cfg_json(const OptimizerConfig& c) {
    return {{"kind", to_string(c.kind)},
            {"learning_rate", c.learning_rate},
            {"adam_beta1", c.adam_beta1},
            {"adam_beta2", c.adam_beta2},
            {"adam_eps", c.adam_eps},
            {"weight_decay", c.weight_decay},
            {"scheduler", c.scheduler == LrSchedule::cosine ? "cosine" : "constant"},
            {"n_warmup_steps", c.n_warmup_steps},
            {"total_steps", c.total_steps},
            {"cosine_min_factor", c.cosine_min_factor}};
}

static json lr_fixture() {
    json cases = json::array();
    for (int sched = 0; sched < 2; ++sched)
        for (int warm : {0, 4})
            for (long long total : {1LL, 5LL, 101LL}) {
                OptimizerConfig c;
                c.learning_rate = 2.0;
                c.scheduler = sched ? LrSchedule::cosine : LrSchedule::constant;
                c.n_warmup_steps = warm;
                c.total_steps = total;
                c.cosine_min_factor = 0.1;
                std::vector<double> lrs;
                for (long long t = 0; t < 110; ++t) lrs.push_back(scheduled_lr(c, t));
                cases.push_back({{"cfg", cfg_json(c)}, {"lr", lrs}});
            }
    return cases;
}

static json optim_fixture() {
    json cases = json::array();
    int id = 0;
    for (OptKind kind : {OptKind::sgd, OptKind::adam, OptKind::adamw})
        for (double wd : {0.0, 0.05})
            for (int sched = 0; sched < 2; ++sched) {
                OptimizerConfig c;
                c.kind = kind;
                c.learning_rate = kind == OptKind::sgd ? 0.1 : 0.01;
                c.weight_decay = wd;
                c.adam_beta2 = 0.95;
                c.scheduler = sched ? LrSchedule::cosine : LrSchedule::constant;
                c.n_warmup_steps = sched ? 2 : 0;
                c.total_steps = 8;
                const int d = 11, steps = 6;
                std::vector<double> theta = rand_vec(rng::derive(5, id, 0), d, 1.0);
                json e;
                e["cfg"] = cfg_json(c);
                e["theta0"] = theta;
                json grads = json::array(), thetas = json::array(), ms = json::array(),
                     vs = json::array();
                OptimizerState st = OptimizerState::for_range(c, 0, d);
                // sharded path with 3 workers (remainder-first layout) must agree
                Fabric fabric(3);
                ShardLayout layout = shard_partition(d, 3);
                std::vector<OptimizerState> shards;
                for (int w = 0; w < 3; ++w)
                    shards.push_back(OptimizerState::for_range(c, layout.lo(w), layout.hi(w)));
                std::vector<double> theta_sh = theta;
                double worst = 0.0;
                for (int s = 0; s < steps; ++s) {
                    std::vector<double> g = rand_vec(rng::derive(6, id, s), d, 1.0);
                    if (s == 2) g[3] = 0.0;  // exact zero coordinate
                    grads.push_back(g);
                    auto [next, upd] = opt_step(std::move(st), theta, g, c);
                    st = std::move(next);
                    theta = std::move(upd);
                    thetas.push_back(theta);
                    ms.push_back(st.m);
                    vs.push_back(st.v);
                    std::vector<std::vector<double>> gs;
                    for (int w = 0; w < 3; ++w)
                        gs.emplace_back(g.begin() + static_cast<long>(layout.lo(w)),
                                        g.begin() + static_cast<long>(layout.hi(w)));
                    theta_sh = sharded_opt_step(shards, theta_sh, gs, c, layout, fabric);
                    for (int j = 0; j < d; ++j)
                        worst = std::max(worst, std::fabs(theta_sh[j] - theta[j]));
                }
                e["grads"] = grads;
                e["thetas"] = thetas;
                e["m"] = ms;
                e["v"] = vs;
                e["sharded_max_abs_diff"] = worst;
                cases.push_back(e);
                ++id;
            }
    return cases;
}

static json fabric_fixture() {
    json cases = json::array();
    for (auto [d, n] : std::vector<std::pair<int, int>>{{7, 3}, {4, 2}, {12, 5}, {3, 4}, {16, 1}, {9, 8}}) {
        Fabric f(n);
        ShardLayout layout = shard_partition(static_cast<std::size_t>(d), n);
        std::vector<std::vector<double>> in;
        std::vector<long long> counts;
        for (int w = 0; w < n; ++w) {
            in.push_back(rand_vec(rng::derive(42, d, w), d, 1.0));
            counts.push_back(3 * w + 1);
        }
        auto rs = f.reduce_scatter(in, layout);
        cases.push_back({{"dim", d},
                         {"n", n},
                         {"inputs", in},
                         {"counts", counts},
                         {"all_reduce", f.all_reduce(in)},
                         {"all_reduce_counts", f.all_reduce_counts(counts)},
                         {"reduce_scatter", rs},
                         {"all_gather", f.all_gather(rs, layout)}});
    }
    return cases;
}

static json problem_json(const Problem& p) {
    json j;
    j["kind"] = to_string(p.kind);
    j["dim"] = p.dim;
    j["smoothness"] = p.smoothness;
    j["noise_sigma"] = p.noise_sigma;
    if (p.optimum) j["optimum"] = *p.optimum;
    if (p.minimizer) j["minimizer"] = *p.minimizer;
    if (p.kind == ProblemKind::quadratic) {
        j["a"] = p.a;
        j["b"] = p.b;
    } else {
        j["n"] = p.data.n;
        j["dim_x"] = p.data.dim_x;
        j["x"] = p.data.x;
        j["y"] = p.data.y;
        j["n_in"] = p.mlp.n_in;
        j["hidden"] = p.mlp.hidden;
    }
    return j;
}

static json run_case(const std::string& name, Method m, const Problem& p, OptimizerConfig cfg,
                     const SimConfig& sim, int t, std::vector<double> theta0 = {}) {
    RunOptions opts;
    opts.record_details = true;
    opts.theta0 = std::move(theta0);
    RunTrace tr = run_protocol(m, p, cfg, sim, t, opts);
    if (cfg.total_steps == 0) cfg.total_steps = t;
    json j;
    j["name"] = name;
    j["method"] = to_string(m);
    j["problem"] = problem_json(p);
    j["optimizer"] = cfg_json(cfg);
    j["sim"] = {{"n_workers", sim.n_workers},
                {"batch_size", sim.batch_size},
                {"n_grad_accumulation", sim.n_grad_accumulation},
                {"warmup_rounds", sim.warmup_rounds},
                {"full_batch_gradients", sim.full_batch_gradients},
                {"master_seed", sim.master_seed},
                {"alpha_s", sim.cost.alpha_s},
                {"beta_s_per_byte", sim.cost.beta_s_per_byte},
                {"worker_multipliers", sim.hetero.multipliers}};
    j["t_updates"] = t;
    j["theta_history"] = tr.theta_history;
    j["estimate_history"] = tr.estimate_history;
    json recs = json::array();
    for (const RoundRecord& r : tr.records)
        recs.push_back({{"update", r.update},
                        {"time_s", r.time_s},
                        {"loss", r.loss},
                        {"grad_sq", r.grad_sq},
                        {"grad_sq_estimate", r.grad_sq_estimate},
                        {"lyapunov", std::isnan(r.lyapunov) ? json(nullptr) : json(r.lyapunov)},
                        {"samples_cum", r.samples_cum},
                        {"mb_main", r.mb_main},
                        {"mb_estimate", r.mb_estimate},
                        {"micro_batches", r.micro_batches},
                        {"idle_frac", r.idle_frac}});
    j["records"] = recs;
    j["issued"] = tr.issued_micro_batches;
    j["consumed"] = tr.consumed_micro_batches;
    j["discarded"] = tr.discarded_micro_batches;
    j["diverged"] = tr.diverged;
    j["consumed_mean_grad"] = tr.consumed_mean_grad;
    return j;
}

static json protocols_fixture() {
    json cases = json::array();
    auto sgd = [](double lr) {
        OptimizerConfig c;
        c.kind = OptKind::sgd;
        c.learning_rate = lr;
        return c;
    };
    auto adamw = [](double lr, double wd, bool cosine) {
        OptimizerConfig c;
        c.kind = OptKind::adamw;
        c.learning_rate = lr;
        c.weight_decay = wd;
        c.adam_beta2 = 0.95;
        c.scheduler = cosine ? LrSchedule::cosine : LrSchedule::constant;
        return c;
    };
    {
        SimConfig sim;
        sim.n_workers = 4;
        sim.batch_size = 8;
        sim.cost.alpha_s = 0.001;
        sim.cost.beta_s_per_byte = 1e-9;
        cases.push_back(run_case("acco_quadratic_cfg", Method::acco, make_quadratic(7, 10, 0.1, 1.0, 0.5),
                                 sgd(0.25), sim, 30));
    }
    {
        SimConfig sim;
        sim.n_workers = 3;
        sim.batch_size = 2;
        sim.cost.alpha_s = 0.3;
        sim.master_seed = 99;
        cases.push_back(run_case("acco_quadratic_comm", Method::acco, make_quadratic(55, 6, 0.2, 1.0, 0.7),
                                 sgd(0.15), sim, 12));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.cost.alpha_s = 0.25;
        sim.cost.beta_s_per_byte = 0.03125;
        cases.push_back(run_case("acco_two_mb_per_stage", Method::acco, make_quadratic(51, 4, 0.2, 1.0, 0.0),
                                 sgd(0.2), sim, 8));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 4;
        sim.n_grad_accumulation = 2;
        sim.master_seed = 11;
        cases.push_back(run_case("acco_logistic_adamw_k2", Method::acco, make_logistic(11, 64, 8),
                                 adamw(0.05, 0.01, false), sim, 15));
    }
    {
        SimConfig sim;
        sim.n_workers = 4;
        sim.batch_size = 8;
        sim.master_seed = 3;
        sim.hetero.multipliers = {1, 1, 1, 4};
        cases.push_back(run_case("acco_mlp_hetero", Method::acco, make_mlp(2024, 4, 8, 64, 0.1),
                                 adamw(0.0075, 0.0, true), sim, 20));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 3;
        sim.n_grad_accumulation = 3;
        sim.master_seed = 8;
        OptimizerConfig c = adamw(0.01, 0.1, true);
        c.kind = OptKind::adam;
        c.n_warmup_steps = 3;
        c.cosine_min_factor = 0.1;
        cases.push_back(run_case("acco_mlp_adam_warmup_k3", Method::acco, make_mlp(5, 3, 6, 48, 0.05),
                                 c, sim, 10));
    }
    {
        SimConfig sim;
        sim.batch_size = 4;
        cases.push_back(run_case("acco_single_worker", Method::acco, make_quadratic(3, 5, 0.2, 1.0, 0.3),
                                 sgd(0.2), sim, 10));
    }
    {
        SimConfig sim;
        sim.n_workers = 3;
        sim.batch_size = 2;
        sim.master_seed = 99;
        cases.push_back(run_case("ddp_quadratic", Method::ddp, make_quadratic(55, 6, 0.2, 1.0, 0.7),
                                 sgd(0.15), sim, 10));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 16;
        sim.n_grad_accumulation = 2;
        sim.master_seed = 21;
        cases.push_back(run_case("ddp_logistic_adamw_k2", Method::ddp, make_logistic(11, 64, 8),
                                 adamw(0.05, 0.01, true), sim, 10));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 8;
        sim.n_grad_accumulation = 2;
        sim.master_seed = 5;
        cases.push_back(run_case("ddp_mlp_adamw", Method::ddp, make_mlp(2024, 4, 8, 64, 0.1),
                                 adamw(0.0075, 0.0, false), sim, 10));
    }
    // one-step-delay baselines (protocols.cpp:340-425)
    {
        SimConfig sim;
        sim.n_workers = 3;
        sim.batch_size = 2;
        sim.master_seed = 99;
        cases.push_back(run_case("dpu_quadratic", Method::dpu, make_quadratic(55, 6, 0.2, 1.0, 0.7),
                                 sgd(0.15), sim, 10));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 4;
        sim.n_grad_accumulation = 2;
        sim.warmup_rounds = 3;
        sim.master_seed = 17;
        cases.push_back(run_case("dpu_logistic_adamw_warmup3", Method::dpu, make_logistic(11, 64, 8),
                                 adamw(0.05, 0.01, true), sim, 10));
    }
    {
        SimConfig sim;
        sim.n_workers = 3;
        sim.batch_size = 2;
        sim.master_seed = 99;
        cases.push_back(run_case("wp_quadratic", Method::wp, make_quadratic(55, 6, 0.2, 1.0, 0.7),
                                 sgd(0.15), sim, 10));
    }
    {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 8;
        sim.n_grad_accumulation = 2;
        sim.master_seed = 5;
        cases.push_back(run_case("wp_mlp_adamw", Method::wp, make_mlp(2024, 4, 8, 64, 0.1),
                                 adamw(0.0075, 0.1, true), sim, 10));
    }
    return cases;
}

// Diverging runs. json has no inf / NaN: non-finite losses and parameters are
// written as null (nlohmann's encoding).
static json divergence_fixture() {
    json cases = json::array();
    auto sgd = [](double lr) {
        OptimizerConfig c;
        c.kind = OptKind::sgd;
        c.learning_rate = lr;
        return c;
    };
    // proj/tests/test_protocols.cpp:328-336, for every method
    auto guarded_case = [&](const std::string& name, Method m, const Problem& p, OptimizerConfig cfg,
                            const SimConfig& sim, int t, std::vector<double> theta0) {
        try {
            cases.push_back(run_case(name, m, p, cfg, sim, t, std::move(theta0)));
        } catch (const std::invalid_argument& e) {
            cases.push_back({{"name", name}, {"method", to_string(m)}, {"throws", "invalid_argument"}, {"what", e.what()}});
        } catch (const std::logic_error& e) {
            cases.push_back({{"name", name}, {"method", to_string(m)}, {"throws", "logic_error"}, {"what", e.what()}});
        }
    };
    for (Method m : {Method::ddp, Method::dpu, Method::wp, Method::acco}) {
        SimConfig sim;
        guarded_case(std::string(to_string(m)) + "_identity_sgd1e8", m, make_identity_quadratic(1), sgd(1e8), sim,
                     200, {1.0});
    }
    // a non-finite theta0: the synchronous rounds see a non-finite mean (diverged,
    // no record); ACCO's optimizer step throws invalid_argument
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (Method m : {Method::ddp, Method::acco}) {
        SimConfig sim;
        sim.n_workers = 2;
        sim.batch_size = 2;
        guarded_case(std::string(to_string(m)) + "_nan_theta0", m, make_quadratic(3, 3, 0.2, 1.0, 0.1), sgd(0.1),
                     sim, 5, {1.0, nan, 0.5});
    }
    return cases;
}

static json io_fixture(const std::string& dir) {
    // the config of proj/tests/test_io.cpp:17-37
    json cfgj = {
        {"problem", {{"kind", "quadratic"}, {"dimension", 4}, {"l_smooth", 1.0},
                     {"mu", 0.2}, {"noise_sigma", 0.1}, {"seed", 5}}},
        {"method_name", "acco"},
        {"optimizer",
         {{"kind", "adamw"}, {"learning_rate", 0.01}, {"weight_decay", 0.1},
          {"adam_beta1", 0.9}, {"adam_beta2", 0.95}, {"scheduler", "cosine"},
          {"n_warmup_steps", 2}}},
        {"n_workers", 2},
        {"batch_size", 3},
        {"n_grad_accumulation", 1},
        {"warmup_rounds", 0},
        {"t_updates", 5},
        {"cost_model", {{"alpha_s", 0.1}, {"beta_s_per_byte", 1e-9}}},
        {"heterogeneity",
         {{"compute_s_per_microbatch", 1.0}, {"worker_multipliers", {1.0, 2.0}}}},
        {"master_seed", 11},
    };
    ExperimentConfig cfg = parse_config(cfgj);
    RunTrace tr = run_protocol(cfg.method, cfg.problem, cfg.optimizer, cfg.sim, cfg.t_updates);
    write_run_outputs(dir + "/io", cfg.raw, tr, cfg.sim.n_workers);
    json j;
    j["config"] = cfg.raw;
    j["config_hash"] = config_hash(cfg.raw);
    j["n_workers"] = cfg.sim.n_workers;
    j["diverged"] = tr.diverged;
    json recs = json::array();
    for (const RoundRecord& r : tr.records)
        recs.push_back({{"update", r.update}, {"time_s", r.time_s}, {"samples_cum", r.samples_cum},
                        {"loss", r.loss}, {"grad_sq", r.grad_sq},
                        {"lyapunov", std::isnan(r.lyapunov) ? json(nullptr) : json(r.lyapunov)},
                        {"idle_frac", r.idle_frac}});
    j["records"] = recs;
    json ivs = json::array();
    for (const Interval& iv : tr.timeline.intervals)
        ivs.push_back({iv.worker, to_string(iv.stream), iv.kind, iv.t_start, iv.t_end, iv.micro_batches, iv.bytes});
    j["intervals"] = ivs;
    // format_g17 samples (csvio.cpp:12-16) incl. the values the LM path emits
    json g17 = json::array();
    for (double v : {0.0, -0.0, 1.0, 0.1, 1e-300, 123456789.125, 3.0e22, -2.5e-7, 1.0 / 3.0, 6.02214076e23})
        g17.push_back({v, format_g17(v)});
    j["g17"] = g17;
    j["g17_nan"] = format_g17(std::numeric_limits<double>::quiet_NaN());
    j["g17_inf"] = format_g17(std::numeric_limits<double>::infinity());
    j["metrics_header_1"] = metrics_header(1);
    j["metrics_header_3"] = metrics_header(3);
    return j;
}

static json memory_fixture() {
    json rows = json::array();
    for (const char* m : {"ddp", "zero1", "zero2", "zero3", "slowmo", "diloco", "co2", "dpu", "wp", "acco"})
        for (double k : {12.0, 16.0})
            for (double n : {1.0, 8.0, 64.0})
                for (double psi : {124439808.0, 7.5e9}) {
                    double b = memory_model_bytes(memory_method_from(m), k, n, psi);
                    rows.push_back({{"method", m}, {"k", k}, {"n", n}, {"psi", psi}, {"bytes", b},
                                    {"gb", memory_reported_gb(b)}});
                }
    return rows;
}

int main(int argc, char** argv) {
    std::string dir = argc > 1 ? argv[1] : "../tests/golden";
    write(dir, "rng.json", rng_fixture());
    write(dir, "shard.json", shard_fixture());
    write(dir, "lr.json", lr_fixture());
    write(dir, "optim.json", optim_fixture());
    write(dir, "fabric.json", fabric_fixture());
    write(dir, "protocols.json", protocols_fixture());
    write(dir, "io_trace.json", io_fixture(dir));
    write(dir, "memory.json", memory_fixture());
    write(dir, "divergence.json", divergence_fixture());
    return 0;
}
