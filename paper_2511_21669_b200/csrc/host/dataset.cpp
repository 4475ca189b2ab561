// dataset.cpp — see dataset.hpp.  Restates proj/src/awc/dataset.cpp and
// serialize_dataset (proj/src/awc/train.cpp:16-33); the simulations run as one
// device batch per call instead of a thread pool of engines.
#include "dataset.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <numeric>
#include <sstream>
#include <thread>

#include <json.hpp>

#include "../device/rng.cuh"

namespace dsd::host {

using cfg::Node;

namespace {

[[noreturn]] void config_error(const std::string& m) { throw Error(DSD_ERR_CONFIG, m); }

std::vector<double> doubles_from(const Node& node, const char* key, std::vector<double> dflt) {
    const Node* n = node.get(key);
    if (!n || n->null()) return dflt;
    std::vector<double> out;
    for (const auto& v : n->items) out.push_back(v.to_double());
    return out;
}

// Grid::interpolate (profile.cpp:20-27, 57-88) on a host profile grid
double interpolate(const ProfileTable::Grid& g, double batch, double context) {
    auto clamp = [](const std::vector<double>& a, double q) { return q < a.front() ? a.front() : (q > a.back() ? a.back() : q); };
    auto segment = [](const std::vector<double>& a, double q) -> size_t {
        if (a.size() == 1) return 0;
        size_t hi = static_cast<size_t>(std::upper_bound(a.begin(), a.end(), q) - a.begin());
        if (hi == 0) return 0;
        if (hi >= a.size()) return a.size() - 2;
        return hi - 1;
    };
    const double b = clamp(g.batch, batch), c = clamp(g.context, context);
    const size_t bi = segment(g.batch, b), ci = segment(g.context, c);
    const size_t bj = std::min(bi + 1, g.batch.size() - 1), cj = std::min(ci + 1, g.context.size() - 1);
    const double tb = (bj == bi) ? 0.0 : (b - g.batch[bi]) / (g.batch[bj] - g.batch[bi]);
    const double tc = (cj == ci) ? 0.0 : (c - g.context[ci]) / (g.context[cj] - g.context[ci]);
    const size_t n = g.context.size();
    auto at = [&](size_t i, size_t j) { return g.values[i * n + j]; };
    const double v = (1.0 - tb) * (1.0 - tc) * at(bi, ci) + (1.0 - tb) * tc * at(bi, cj) +
                     tb * (1.0 - tc) * at(bj, ci) + tb * tc * at(bj, cj);
    return v * g.calibration;
}

// Resolves one config per item on a thread pool (resolution is independent
// per item; the device batch is assembled in item order afterwards).
std::vector<Resolved> resolve_all(const std::vector<Node>& configs, const std::vector<uint64_t>& seeds,
                                  Caches* caches) {
    std::vector<Resolved> out(configs.size());
    std::vector<std::string> errors(configs.size());
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (;;) {
            const size_t i = next.fetch_add(1);
            if (i >= configs.size()) return;
            try {
                out[i] = resolve_config(configs[i], true, seeds[i], ".", caches, /*want_digest=*/false);
            } catch (const std::exception& e) {
                errors[i] = e.what();
            }
        }
    };
    unsigned nthreads = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
    if (configs.size() < 64) nthreads = 1;
    if (nthreads == 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nthreads; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
    }
    for (size_t i = 0; i < configs.size(); ++i)
        if (!errors[i].empty()) config_error(errors[i]);
    for (auto& r : out) r.bind();
    return out;
}

struct BatchOut {
    std::vector<dsd_replica_summary> sums;
    std::vector<double> probe;  // [n][DSD_PROBE_FIELDS]
};

// One device batch: replica i runs resolved[i] with seed = gen_seed = seeds[i]
// (the reference's seed override and its generate_synthetic(spec, s.seed)).
BatchOut run_probed(Runtime& rt, const std::vector<Resolved>& resolved, const std::vector<uint64_t>& seeds) {
    const size_t n = resolved.size();
    std::vector<dsd_scenario> sc(n);
    std::vector<dsd_replica> reps(n);
    for (size_t i = 0; i < n; ++i) {
        sc[i] = resolved[i].scen;
        reps[i] = dsd_replica{};
        reps[i].scenario = static_cast<uint32_t>(i);
        reps[i].seed = seeds[i];
        reps[i].gen_seed = seeds[i];
    }
    BatchOut o;
    o.sums.resize(n);
    o.probe.resize(n * DSD_PROBE_FIELDS);
    if (n == 0) return o;
    rt.prepare(sc.data(), n, reps.data(), n, false, /*feature_probe=*/true);
    rt.launch();
    rt.sync();
    rt.summaries(o.sums.data(), n);
    rt.probe(o.probe.data(), n);
    for (size_t i = 0; i < n; ++i)
        if (o.sums[i].status != DSD_OK)
            throw Error(DSD_ERR_RUNTIME, "engine capacity exceeded on the device (event heap / sequence arena)");
    return o;
}

}  // namespace

DatasetGrid DatasetGrid::from_node(const Node& node) {
    DatasetGrid g;
    if (!node.map()) return g;
    g.rtt_ms = doubles_from(node, "rtt_ms", g.rtt_ms);
    g.alpha = doubles_from(node, "alpha", g.alpha);
    g.load_factor = doubles_from(node, "load_factor", g.load_factor);
    if (const Node* d = node.get("drafts"); d && d->seq()) {
        g.drafts.clear();
        for (const auto& v : d->items) g.drafts.push_back(static_cast<int>(v.to_int()));
    }
    g.cost_ratio = doubles_from(node, "cost_ratio", g.cost_ratio);
    g.target_decode_ms = node.double_or("target_decode_ms", g.target_decode_ms);
    g.n_requests = static_cast<int>(node.int_or("n_requests", g.n_requests));
    g.seed = static_cast<uint64_t>(node.int_or("seed", static_cast<int64_t>(g.seed)));
    return g;
}

// build_scenarios (dataset.cpp:50-87)
std::vector<ScenarioSpec> build_scenarios(const DatasetGrid& grid) {
    std::vector<ScenarioSpec> out;
    uint64_t id = 0;
    for (double rtt : grid.rtt_ms)
        for (double alpha : grid.alpha)
            for (double load : grid.load_factor)
                for (int drafts : grid.drafts)
                    for (double c : grid.cost_ratio) {
                        ScenarioSpec s;
                        s.scenario_id = id++;
                        s.rtt_ms = rtt;
                        s.jitter_ms = rtt >= 4.0 ? rtt * 0.1 : 0.0;
                        s.alpha = alpha;
                        s.load_factor = load;
                        s.drafts = drafts;
                        s.target_decode_ms = grid.target_decode_ms;
                        s.cost_ratio = c;
                        s.n_requests = grid.n_requests;
                        s.seed = cfg::fnv1a64("scenario-" + std::to_string(s.scenario_id), grid.seed);
                        out.push_back(s);
                    }
    // 80/10/10 split on a seeded Fisher-Yates shuffle of the scenario order
    std::vector<size_t> order(out.size());
    std::iota(order.begin(), order.end(), 0);
    Rng shuffle;
    shuffle.seed(grid.seed, fnv1a64("scenario-split"));
    for (size_t i = order.size(); i > 1; --i) {
        const size_t j = static_cast<size_t>(shuffle.below(i));
        std::swap(order[i - 1], order[j]);
    }
    const size_t n_train = std::max<size_t>(out.empty() ? 0 : 1, (out.size() * 8) / 10);
    const size_t n_val = out.size() / 10;
    for (size_t rank = 0; rank < order.size(); ++rank)
        out[order[rank]].split = rank < n_train ? "train" : (rank < n_train + n_val ? "val" : "test");
    return out;
}

// serialize_scenarios / parse_scenarios (dataset.cpp:89-143)
std::string serialize_scenarios(const std::vector<ScenarioSpec>& scenarios) {
    using cfg::fmt_exact;
    std::string out;
    for (const auto& s : scenarios) {
        out += "{\"scenario_id\":" + std::to_string(s.scenario_id);
        out += ",\"split\":\"" + s.split + "\"";
        out += ",\"rtt_ms\":" + fmt_exact(s.rtt_ms);
        out += ",\"jitter_ms\":" + fmt_exact(s.jitter_ms);
        out += ",\"alpha\":" + fmt_exact(s.alpha);
        out += ",\"load_factor\":" + fmt_exact(s.load_factor);
        out += ",\"drafts\":" + std::to_string(s.drafts);
        out += ",\"targets\":" + std::to_string(s.targets);
        out += ",\"target_decode_ms\":" + fmt_exact(s.target_decode_ms);
        out += ",\"cost_ratio\":" + fmt_exact(s.cost_ratio);
        out += ",\"prompt_median\":" + fmt_exact(s.prompt_median);
        out += ",\"output_median\":" + fmt_exact(s.output_median);
        out += ",\"n_requests\":" + std::to_string(s.n_requests);
        out += ",\"seed\":" + std::to_string(s.seed);
        out += "}\n";
    }
    return out;
}

std::vector<ScenarioSpec> parse_scenarios(const std::string& text) {
    std::vector<ScenarioSpec> out;
    std::istringstream in(text);
    std::string line;
    int line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        nlohmann::json j = nlohmann::json::parse(line, nullptr, false);
        if (j.is_discarded()) config_error("scenario line " + std::to_string(line_no) + ": invalid JSON");
        try {
            ScenarioSpec s;
            s.scenario_id = j.at("scenario_id").get<uint64_t>();
            s.split = j.at("split").get<std::string>();
            s.rtt_ms = j.at("rtt_ms").get<double>();
            s.jitter_ms = j.at("jitter_ms").get<double>();
            s.alpha = j.at("alpha").get<double>();
            s.load_factor = j.at("load_factor").get<double>();
            s.drafts = j.at("drafts").get<int>();
            s.targets = j.at("targets").get<int>();
            s.target_decode_ms = j.at("target_decode_ms").get<double>();
            s.cost_ratio = j.at("cost_ratio").get<double>();
            s.prompt_median = j.at("prompt_median").get<double>();
            s.output_median = j.at("output_median").get<double>();
            s.n_requests = j.at("n_requests").get<int>();
            s.seed = j.at("seed").get<uint64_t>();
            out.push_back(s);
        } catch (const nlohmann::json::exception& e) {
            config_error("scenario line " + std::to_string(line_no) + ": " + e.what());
        }
    }
    return out;
}

// scenario_trace (dataset.cpp:125-147): the arrival rate for load_factor of a
// reference verify capacity (full batch of 8 at gamma 4, ~3 tokens committed)
double scenario_rate(const ScenarioSpec& s) {
    auto profile = synth_profile(s.target_decode_ms, s.cost_ratio, 0.05, 0.3, 0.2);
    const int g = profile->find("target-model", "cloud-gpu", 1);  // verify is decode-shaped
    if (g < 0) config_error("no profile entry for (target-model, cloud-gpu, decode)");
    // LatencyProfile::predict(Verify, BatchShape{8, 4, 128}) (profile.cpp:129-151)
    const double step_ms = interpolate(profile->grids[static_cast<size_t>(g)], 8.0 * 4.0, 128.0);
    const double tokens_per_s = 8.0 * 3.0 * 1000.0 / step_ms;
    return s.load_factor * tokens_per_s / s.output_median;
}

Node scenario_config(const ScenarioSpec& s, const std::string& window_kind, int gamma, const std::string& model_path) {
    Node cfgn;
    cfgn.kind = Node::Kind::Map;
    auto map = [] {
        Node m;
        m.kind = Node::Kind::Map;
        return m;
    };
    cfgn.put("targets", Node::of_int(s.targets));
    cfgn.put("drafts", Node::of_int(s.drafts));
    Node net = map();
    net.put("rtt_ms", Node::of_double(s.rtt_ms));
    net.put("jitter_ms", Node::of_double(s.jitter_ms));
    cfgn.put("network", std::move(net));
    Node pol = map();
    pol.put("routing", Node::of_string("jsq"));
    Node batching = map();
    batching.put("kind", Node::of_string("fifo"));
    batching.put("max_batch_size", Node::of_int(8));
    pol.put("batching", std::move(batching));
    Node window = map();
    window.put("kind", Node::of_string(window_kind));
    window.put("gamma", Node::of_int(gamma));
    if (!model_path.empty()) window.put("model", Node::of_string(model_path));
    pol.put("window", std::move(window));
    cfgn.put("policies", std::move(pol));
    Node prof = map(), synth = map();
    synth.put("target_decode_ms", Node::of_double(s.target_decode_ms));
    synth.put("cost_ratio", Node::of_double(s.cost_ratio));
    synth.put("batch_coef", Node::of_double(0.05));
    synth.put("context_coef", Node::of_double(0.3));
    prof.put("synth", std::move(synth));
    cfgn.put("latency_profile", std::move(prof));
    cfgn.put("seed", Node::of_int(static_cast<int64_t>(s.seed)));
    // scenario_trace's SyntheticSpec (dataset.cpp:135-146): the trace the
    // reference generates with generate_synthetic(spec, s.seed) and replays
    // trace-driven is this synthetic workload with gen_seed = s.seed
    Node w = map();
    w.put("mode", Node::of_string("poisson"));
    w.put("rate_rps", Node::of_double(scenario_rate(s)));
    w.put("n_requests", Node::of_int(s.n_requests));
    w.put("acceptance_rate", Node::of_double(s.alpha));
    w.put("prompt_median", Node::of_double(s.prompt_median));
    w.put("prompt_sigma", Node::of_double(0.3));
    w.put("output_median", Node::of_double(s.output_median));
    w.put("output_sigma", Node::of_double(0.3));
    w.put("gen_seed", Node::of_int(static_cast<int64_t>(s.seed)));
    cfgn.put("workload", std::move(w));
    return cfgn;
}

// score_candidates (dataset.cpp:208-230)
void score_candidates(std::vector<CandidateOutcome>& candidates, const ObjectiveWeights& weights) {
    auto norm = [&](auto getter) {
        double lo = 1e300, hi = -1e300;
        for (const auto& c : candidates) {
            lo = std::min(lo, getter(c));
            hi = std::max(hi, getter(c));
        }
        std::vector<double> out;
        for (const auto& c : candidates) out.push_back(hi > lo ? (getter(c) - lo) / (hi - lo) : 0.0);
        return out;
    };
    auto tpot_n = norm([](const CandidateOutcome& c) { return c.mean_tpot_ms; });
    auto ttft_n = norm([](const CandidateOutcome& c) { return c.mean_ttft_ms; });
    auto thr_n = norm([](const CandidateOutcome& c) { return c.throughput_rps; });
    for (size_t i = 0; i < candidates.size(); ++i)
        candidates[i].objective =
            weights.w_tpot * tpot_n[i] + weights.w_ttft * ttft_n[i] - weights.w_throughput * thr_n[i];
}

// pick_label (dataset.cpp:232-243): argmin objective, ties to the lower gamma
int pick_label(const std::vector<CandidateOutcome>& candidates) {
    int best = 0;
    for (int i = 1; i < static_cast<int>(candidates.size()); ++i) {
        const auto& c = candidates[static_cast<size_t>(i)];
        const auto& b = candidates[static_cast<size_t>(best)];
        if (c.objective < b.objective || (c.objective == b.objective && c.gamma < b.gamma)) best = i;
    }
    return candidates[static_cast<size_t>(best)].gamma;
}

// generate_dataset (dataset.cpp:188-206 run_candidate, 245-256
// sweep_scenario, 258-290): candidates static gamma 2..12 then fused
std::vector<ScenarioSweepResult> generate_dataset(Runtime& rt, const std::vector<ScenarioSpec>& scenarios,
                                                  const ObjectiveWeights& weights, Caches* caches) {
    constexpr int kCandidates = 12;
    std::vector<Node> configs;
    std::vector<uint64_t> seeds;
    configs.reserve(scenarios.size() * kCandidates);
    for (const auto& s : scenarios) {
        for (int gamma = 2; gamma <= 12; ++gamma) {
            configs.push_back(scenario_config(s, "static", gamma, ""));
            seeds.push_back(s.seed);
        }
        configs.push_back(scenario_config(s, "fused", 4, ""));
        seeds.push_back(s.seed);
    }
    const std::vector<Resolved> resolved = resolve_all(configs, seeds, caches);
    const BatchOut o = run_probed(rt, resolved, seeds);
    std::vector<ScenarioSweepResult> sweeps(scenarios.size());
    for (size_t k = 0; k < scenarios.size(); ++k) {
        ScenarioSweepResult& r = sweeps[k];
        r.scenario = scenarios[k];
        for (int j = 0; j < kCandidates; ++j) {
            const size_t i = k * kCandidates + static_cast<size_t>(j);
            const dsd_replica_summary& sm = o.sums[i];
            const double* pr = &o.probe[i * DSD_PROBE_FIELDS];
            CandidateOutcome c;
            c.fused = j == kCandidates - 1;
            c.gamma = c.fused ? 1 : j + 2;
            c.throughput_rps = sm.throughput_rps;
            c.mean_ttft_ms = sm.mean_ttft_ms;
            c.mean_tpot_ms = sm.mean_tpot_ms;
            // RunResult::mean_features (engine.cpp:660-664)
            for (int f = 0; f < 5; ++f) c.mean_features[f] = pr[5] > 0.0 ? pr[f] / pr[5] : pr[f];
            r.candidates.push_back(c);
        }
        score_candidates(r.candidates, weights);
        r.label_gamma = pick_label(r.candidates);
    }
    return sweeps;
}

// serialize_dataset (train.cpp:16-33) of generate_dataset's samples
std::string serialize_dataset(const std::vector<ScenarioSweepResult>& sweeps) {
    std::string out;
    for (const auto& sw : sweeps)
        for (const auto& c : sw.candidates) {
            out += "{\"scenario_id\":" + std::to_string(sw.scenario.scenario_id);
            out += ",\"split\":\"" + sw.scenario.split + "\"";
            out += ",\"features\":[";
            for (int f = 0; f < 5; ++f) {
                if (f) out += ',';
                out += cfg::fmt_exact(c.mean_features[static_cast<size_t>(f)]);
            }
            out += "],\"candidate_gamma\":" + std::to_string(c.gamma);
            out += ",\"candidate_mode\":\"" + std::string(c.fused ? "fused" : "distributed") + "\"";
            out += ",\"objective\":" + cfg::fmt_exact(c.objective);
            out += ",\"label_gamma\":" + std::to_string(sw.label_gamma);
            out += "}\n";
        }
    return out;
}

// eval_policy_on_scenarios (dataset.cpp:292-369)
PolicyEval eval_policy_on_scenarios(Runtime& rt, const std::vector<ScenarioSpec>& scenarios,
                                    const std::string& window_kind, int gamma, const std::string& model_path,
                                    Caches* caches) {
    PolicyEval eval;
    eval.policy = window_kind;
    if (scenarios.empty()) return eval;
    std::vector<Node> configs;
    std::vector<uint64_t> seeds;
    for (const auto& s : scenarios) {
        configs.push_back(scenario_config(s, window_kind, gamma, model_path));
        seeds.push_back(s.seed);
    }
    const std::vector<Resolved> resolved = resolve_all(configs, seeds, caches);
    const BatchOut o = run_probed(rt, resolved, seeds);
    for (size_t i = 0; i < scenarios.size(); ++i) {
        eval.mean_throughput_rps += o.sums[i].throughput_rps;
        eval.mean_ttft_ms += o.sums[i].mean_ttft_ms;
        eval.mean_tpot_ms += o.sums[i].mean_tpot_ms;
        // mean over the records' gamma sequences (fused counts as 1); every
        // request completes, so the per-iteration tally is the same multiset
        const double* pr = &o.probe[i * DSD_PROBE_FIELDS];
        eval.mean_chosen_gamma += pr[7] > 0.0 ? pr[6] / pr[7] : 0.0;
    }
    const double n = static_cast<double>(scenarios.size());
    eval.mean_throughput_rps /= n;
    eval.mean_ttft_ms /= n;
    eval.mean_tpot_ms /= n;
    eval.mean_chosen_gamma /= n;
    return eval;
}

}  // namespace dsd::host
