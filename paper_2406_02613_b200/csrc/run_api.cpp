// Config-level drop-in entry (SURVEY.md §8(b) "Trainer"): acco_run(config,
// out_dir, summary) = the reference's load_config / parse_config
// (proj/src/config.cpp:80-145) -> run_protocol (proj/src/protocols.cpp:713-742)
// -> write_run_outputs (proj/src/csvio.cpp:79-102), with the CLI's exit-code
// convention as the return value (proj/tools/accosim_main.cpp:30-33, 53-70).
//
// Host C++ only (compiled by the host compiler through nvcc). JSON is
// nlohmann/json — the library the reference itself parses and dumps with — so
// the echoed config, its FNV-1a hash and the manifest layout are the
// reference's byte for byte. The problem block takes the B200 kinds "gpt" /
// "llama" (the analytic problems are CPU parity fixtures, not GPU workloads);
// the execution keys match paper_2406_02613_b200/api.py parse_config.
#include <json.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "acco.h"
#include "capi_util.h"
#include "engine.h"

namespace acco {
namespace {

using json = nlohmann::json;

template <class T>
T get_or(const json& j, const char* key, T fallback) {  // config.cpp:10-14
    if (!j.contains(key)) return fallback;
    return j.at(key).get<T>();
}

template <class T>
T require(const json& j, const char* key) {  // config.cpp:16-21
    if (!j.contains(key)) throw std::invalid_argument(std::string("config: missing key '") + key + "'");
    return j.at(key).get<T>();
}

struct RunConfig {
    LMConfig lm;
    int method = kACCO;
    OptConfig opt;
    SimCfg sim;
    std::vector<double> multipliers;
    int t_updates = 0;
    std::string output_dir;
    json raw;
};

int method_from(const std::string& m) {
    if (m == "ddp") return kDDP;
    if (m == "dpu") return kDPU;
    if (m == "wp") return kWP;
    if (m == "acco") return kACCO;
    if (m == "zero1") return kZeRO1;
    throw std::invalid_argument("config: unknown method_name '" + m + "'");
}

RunConfig parse(const json& j) {
    RunConfig c;
    c.raw = j;
    const json& p = require<json>(j, "problem");
    const std::string kind = require<std::string>(p, "kind");
    if (kind != "gpt" && kind != "llama")
        throw std::invalid_argument("config: unknown problem kind for the B200 path: " + kind);
    c.lm.vocab = get_or<int>(p, "vocab", 256);
    c.lm.d_model = get_or<int>(p, "d_model", 128);
    c.lm.n_layer = get_or<int>(p, "n_layer", 2);
    c.lm.n_head = get_or<int>(p, "n_head", 4);
    c.lm.seq_len = get_or<int>(p, "seq_len", 64);
    c.lm.n_samples = get_or<int>(p, "n_samples", 256);
    c.lm.data_seed = get_or<uint64_t>(p, "seed", 1);
    const std::string prec = get_or<std::string>(p, "precision", "fp32");
    if (prec != "fp32" && prec != "bf16") throw std::invalid_argument("lm config: precision must be fp32 or bf16");
    c.lm.precision = prec == "bf16" ? 1 : 0;
    c.lm.max_batch = std::max(get_or<int>(j, "batch_size", 1), get_or<int>(p, "max_batch", 1));
    c.lm.arch = kind == "llama" ? 1 : 0;
    c.lm.n_kv_head = get_or<int>(p, "n_kv_head", 0);
    c.lm.d_ff = get_or<int>(p, "d_ff", 0);
    c.lm.rope_base = get_or<double>(p, "rope_base", 10000.0);
    c.method = method_from(require<std::string>(j, "method_name"));
    // parse_optimizer, config.cpp:51-76
    const json& o = require<json>(j, "optimizer");
    const std::string ok = require<std::string>(o, "kind");
    if (ok == "sgd") c.opt.kind = 0;
    else if (ok == "adam") c.opt.kind = 1;
    else if (ok == "adamw") c.opt.kind = 2;
    else throw std::invalid_argument("unknown optimizer kind: " + ok);
    c.opt.learning_rate = require<double>(o, "learning_rate");
    c.opt.weight_decay = get_or<double>(o, "weight_decay", 0.0);
    c.opt.adam_beta1 = get_or<double>(o, "adam_beta1", 0.9);
    c.opt.adam_beta2 = get_or<double>(o, "adam_beta2", 0.999);
    c.opt.adam_eps = get_or<double>(o, "adam_eps", 1e-8);
    const std::string sched = get_or<std::string>(o, "scheduler", "constant");
    if (sched == "constant") c.opt.scheduler = 0;
    else if (sched == "cosine") c.opt.scheduler = 1;
    else throw std::invalid_argument("config: scheduler must be constant or cosine");
    c.opt.n_warmup_steps = get_or<int>(o, "n_warmup_steps", 0);
    c.opt.cosine_min_factor = get_or<double>(o, "cosine_min_factor", 0.0);
    if (!(c.opt.learning_rate > 0.0)) throw std::invalid_argument("config: learning_rate > 0");
    if (c.opt.adam_beta1 < 0.0 || c.opt.adam_beta1 >= 1.0 || c.opt.adam_beta2 < 0.0 || c.opt.adam_beta2 >= 1.0)
        throw std::invalid_argument("config: adam betas must lie in [0, 1)");
    if (c.opt.weight_decay < 0.0) throw std::invalid_argument("config: weight_decay >= 0");
    if (c.opt.n_warmup_steps < 0) throw std::invalid_argument("config: n_warmup_steps >= 0");
    // simulation keys (config.cpp:86-128) + the B200 execution keys
    c.sim.n_workers = get_or<int>(j, "n_workers", 1);
    c.sim.batch_size = get_or<int>(j, "batch_size", 1);
    c.sim.n_grad_accumulation = get_or<int>(j, "n_grad_accumulation", 1);
    c.sim.warmup_rounds = get_or<int>(j, "warmup_rounds", 0);
    if (get_or<bool>(j, "full_batch_gradients", false))
        throw std::invalid_argument("full_batch_gradients is not supported for the LM problem");
    c.sim.master_seed = get_or<uint64_t>(j, "master_seed", 1);
    const std::string schedule = get_or<std::string>(j, "schedule", "floor");
    if (schedule == "floor") c.sim.schedule = kFloor;
    else if (schedule == "adaptive") c.sim.schedule = kAdaptive;
    else throw std::invalid_argument("config: schedule must be floor or adaptive");
    c.sim.eval_every = get_or<int>(j, "eval_every", 1);
    c.sim.check_replicas = get_or<bool>(j, "check_replicas", false) ? 1 : 0;
    c.sim.throttle_host = get_or<bool>(j, "throttle_host", false) ? 1 : 0;
    if (j.contains("heterogeneity"))
        c.multipliers = get_or<std::vector<double>>(j.at("heterogeneity"), "worker_multipliers", {});
    c.t_updates = require<int>(j, "t_updates");
    c.output_dir = get_or<std::string>(j, "output_dir", "");
    if (c.t_updates < 1) throw std::invalid_argument("config: t_updates >= 1");
    if (c.sim.n_workers < 1) throw std::invalid_argument("config: n_workers >= 1");
    if (c.sim.batch_size < 1) throw std::invalid_argument("config: batch_size >= 1");
    if (c.sim.n_grad_accumulation < 1) throw std::invalid_argument("config: n_grad_accumulation >= 1");
    if (c.sim.warmup_rounds < 0) throw std::invalid_argument("config: warmup_rounds >= 0");
    if (!c.multipliers.empty() && static_cast<int>(c.multipliers.size()) != c.sim.n_workers)
        throw std::invalid_argument("config: worker_multipliers length must equal n_workers");
    for (double m : c.multipliers)
        if (!(m > 0.0)) throw std::invalid_argument("config: worker_multipliers > 0");
    c.opt.total_steps = c.t_updates;  // config.cpp:131
    return c;
}

json load(const char* config) {  // load_config (config.cpp:135-145), or inline JSON text
    std::string s(config);
    const size_t i = s.find_first_not_of(" \t\r\n");
    try {
        if (i != std::string::npos && s[i] == '{') return json::parse(s);
        std::ifstream in(s);
        if (!in) throw std::invalid_argument("config: cannot open " + s);
        json j;
        in >> j;
        return j;
    } catch (const json::exception& e) {
        throw std::invalid_argument(std::string("config: invalid JSON: ") + e.what());
    }
}

std::string config_hash(const json& j) {  // config.cpp:147-157
    const std::string s = j.dump();
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char ch : s) {
        h ^= ch;
        h *= 0x100000001b3ull;
    }
    char buf[17];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
    return buf;
}

std::string g17(double v) {  // format_g17, csvio.cpp:12-16
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

void write_file(const std::string& path, const std::string& content) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + path);
    out << content;
}

const char* kIvNames[] = {"init_grad", "microbatch", "all_reduce", "reduce_scatter", "optimizer", "all_gather"};

}  // namespace
}  // namespace acco

using namespace acco;

extern "C" int acco_run(const char* config, const char* out_dir, acco_run_summary* summary) {
    int status = kOk;
    const int rc = guarded([&] {
        ACCO_REQUIRE(config, "acco_run: null config");
        RunConfig c;
        try {
            c = parse(load(config));
        } catch (const json::exception& e) {  // wrong value types: the reference CLI's exit 2
            throw std::invalid_argument(std::string("config: ") + e.what());
        }
        std::string dir = out_dir && *out_dir ? std::string(out_dir) : c.output_dir;
        if (dir.empty()) {  // accosim_main.cpp:35-40, 57-58
            const char* root = std::getenv("ACCOSIM_OUT");
            dir = std::string(root ? root : "out") + "/run_" + config_hash(c.raw);
        }
        GPTModel model(c.lm);
        if (!c.multipliers.empty() &&
            std::any_of(c.multipliers.begin(), c.multipliers.end(), [](double m) { return m != 1.0; })) {
            // HeterogeneityProfile (protocols.hpp:19-27) -> per-worker throttle of
            // (m - 1) x the measured micro-batch time
            const double t = time_micro_batch(model, c.sim.batch_size, 3);
            for (double m : c.multipliers) c.sim.throttle_ns.push_back(std::max(0.0, m - 1.0) * t);
        }
        Trainer trainer(&model, c.opt, c.sim, c.method, nullptr);
        std::vector<float> th0(static_cast<size_t>(model.num_params()));
        lm_default_theta0(c.lm, c.sim.master_seed, th0.data());
        trainer.set_theta(th0.data());
        std::vector<UpdateRecord> recs;
        RunStats st;
        trainer.run(c.t_updates, recs, st, nullptr);
        const auto& tl = trainer.timeline();
        // metrics.csv (csvio.cpp:18-46) with idle_frac from the measured compute intervals
        const int n = c.sim.n_workers;
        std::string m = "update,time_s,samples,loss,grad_norm_sq,lyapunov";
        for (int w = 0; w < n; ++w) m += ",idle_frac_w" + std::to_string(w);
        m += "\n";
        double prev = 0.0;
        for (const UpdateRecord& r : recs) {
            const double t = r.time_s, window = t - prev;
            m += std::to_string(r.update) + "," + g17(t) + "," + std::to_string(r.samples_cum) + "," + g17(r.loss) +
                 "," + g17(r.grad_sq) + "," + g17(r.lyapunov);
            for (int w = 0; w < n; ++w) {
                double busy = 0.0;
                for (const Interval& iv : tl)
                    if (iv.stream == 0 && iv.worker == w)
                        busy += std::max(0.0, std::min(iv.t_end, t) - std::max(iv.t_start, prev));
                m += "," + g17(window > 0 ? std::max(0.0, (window - busy) / window) : 0.0);
            }
            m += "\n";
            prev = t;
        }
        std::string tcsv = "worker_id,stream,event_kind,t_start,t_end,micro_batches,bytes\n";  // csvio.cpp:48-66
        for (const Interval& iv : tl)
            tcsv += std::to_string(iv.worker) + "," + (iv.stream ? "comm" : "compute") + "," + kIvNames[iv.kind] +
                    "," + g17(iv.t_start) + "," + g17(iv.t_end) + "," + std::to_string(iv.micro_batches) + "," +
                    std::to_string(iv.bytes) + "\n";
        std::filesystem::create_directories(dir);
        write_file(dir + "/metrics.csv", m);
        write_file(dir + "/timeline.csv", tcsv);
        json manifest;  // csvio.cpp:84-96
        manifest["tool"] = "accosim";
        manifest["version"] = "0.1.0";
        manifest["config"] = c.raw;
        manifest["config_hash"] = config_hash(c.raw);
        manifest["master_seed"] = c.raw.contains("master_seed") ? c.raw.at("master_seed") : json(1);
        manifest["diverged"] = st.diverged != 0;
        manifest["updates"] = recs.size();
        manifest["outputs"] = {"metrics.csv", "timeline.csv"};
        write_file(dir + "/manifest.json", manifest.dump(2) + "\n");
        if (summary) {
            std::memset(summary, 0, sizeof(*summary));
            summary->updates = static_cast<int>(recs.size());
            summary->diverged = st.diverged;
            summary->final_loss = recs.empty() ? NAN : recs.back().loss;
            summary->samples = recs.empty() ? 0 : recs.back().samples_cum;
            summary->wall_ms = st.wall_ms;
            std::snprintf(summary->out_dir, sizeof(summary->out_dir), "%s", dir.c_str());
        }
        if (st.diverged) status = kDiverged;  // accosim_main.cpp:65-68: exit 3
    });
    if (rc != kOk) return rc;
    if (status == kDiverged) set_last_error("run diverged");
    return status;
}
