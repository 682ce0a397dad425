// CPU baseline of the ACCO optimizer round on the REFERENCE code (C5 in
// SURVEY.md §8(d)): the exact comm-phase call sequence of
// proj/src/protocols.cpp:644-670 — reduce_scatter, x 1/total, transient
// sharded_opt_step (estimate), reduce_scatter, + retained, x 1/combined,
// persistent sharded_opt_step (commit), all-gathers inside sharded_opt_step.
// Test/bench infrastructure only. Usage: ref_round_bench <psi> <n_workers> <reps>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "accosim/collectives.hpp"
#include "accosim/optim.hpp"
#include "accosim/rng.hpp"
#include "accosim/shard.hpp"
#include "accosim/vecmath.hpp"

using namespace accosim;

int main(int argc, char** argv) {
    std::size_t psi = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 10000000ull;
    int n = argc > 2 ? std::atoi(argv[2]) : 8;
    int reps = argc > 3 ? std::atoi(argv[3]) : 3;
    OptimizerConfig cfg;
    cfg.kind = OptKind::adamw;
    cfg.learning_rate = 6e-4;
    cfg.weight_decay = 0.1;
    cfg.adam_beta2 = 0.95;
    cfg.scheduler = LrSchedule::cosine;
    cfg.total_steps = 100;
    Fabric fabric(n);
    ShardLayout layout = shard_partition(psi, n);
    std::vector<OptimizerState> states;
    for (int w = 0; w < n; ++w) states.push_back(OptimizerState::for_range(cfg, layout.lo(w), layout.hi(w)));
    std::vector<double> theta(psi);
    rng::Stream g0(1);
    for (double& x : theta) x = 0.02 * g0.gaussian();
    std::vector<std::vector<double>> sums(static_cast<std::size_t>(n), std::vector<double>(psi));
    for (int w = 0; w < n; ++w) {
        rng::Stream g(rng::derive(2, static_cast<std::uint64_t>(w)));
        for (double& x : sums[static_cast<std::size_t>(w)]) x = g.gaussian();
    }
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        long long total = 8 * n;
        auto est = fabric.reduce_scatter(sums, layout);
        auto mean = est;
        for (auto& s : mean) vec::scale(s, 1.0 / static_cast<double>(total));
        std::vector<OptimizerState> transient = states;
        auto theta_est = sharded_opt_step(transient, theta, mean, cfg, layout, fabric);
        auto main = fabric.reduce_scatter(sums, layout);
        for (int w = 0; w < n; ++w) {
            auto& s = main[static_cast<std::size_t>(w)];
            const auto& e = est[static_cast<std::size_t>(w)];
            for (std::size_t j = 0; j < s.size(); ++j) s[j] += e[j];
            vec::scale(s, 1.0 / static_cast<double>(2 * total));
        }
        theta = sharded_opt_step(states, theta, main, cfg, layout, fabric);
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (dt < best) best = dt;
        if (theta_est.size() != psi) return 2;
    }
    std::printf("{\"psi\": %zu, \"n_workers\": %d, \"best_s\": %.6f, \"params_per_s\": %.1f}\n", psi, n,
                best, static_cast<double>(psi) / best);
    return 0;
}
