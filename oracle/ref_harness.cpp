// oracle/ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" shim around the UNMODIFIED reference library, which the
// recipe in oracle/Makefile compiles directly from /root/reference/proj/src
// into oracle/_ref/libspecsim_ref.so.  Nothing here re-implements reference
// behaviour: every entry point forwards to the reference's own public C++ API
//   resolve_config / run_simulation / aggregate_run   (proj/src/runner/runner.cpp:96-169)
//   SweepSpec::from_node / run_sweep / sweep_point_seed (proj/src/runner/sweep.cpp:16-162)
//   generate_synthetic / serialize_trace               (proj/src/workload/trace.cpp:104-187)
//   RngStream / net_delay / consume_acceptance         (proj/src/sim/rng.cpp, engine.cpp:10-32)
// so that pytest (ctypes), bench.py's reference arm and the golden-fixture
// script can drive the real reference.  Only tests/, bench.py's cpu_baseline
// leg and __graft_entry__.smoke() may load this library.

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "specsim/awc/dataset.hpp"
#include "specsim/awc/mlp.hpp"
#include "specsim/awc/train.hpp"
#include "specsim/engine/engine.hpp"
#include "specsim/errors.hpp"
#include "specsim/latency/profile.hpp"
#include "specsim/metrics/metrics.hpp"
#include "specsim/runner/runner.hpp"
#include "specsim/runner/sweep.hpp"
#include "specsim/sim/rng.hpp"
#include "specsim/util/fnv.hpp"
#include "specsim/util/yaml.hpp"
#include "specsim/workload/trace.hpp"

using namespace specsim;

namespace {

char* dup_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = '\0';
    return p;
}

void set_err(char* err, std::size_t errlen, const std::string& msg) {
    if (!err || errlen == 0) return;
    std::size_t n = std::min(errlen - 1, msg.size());
    std::memcpy(err, msg.data(), n);
    err[n] = '\0';
}

// Exception -> status code, mirroring tools/specsim_main.cpp:293-311.
template <typename F>
int guarded(char* err, std::size_t errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const ParseError& e) {
        set_err(err, errlen, std::string("parse error: ") + e.what());
        return 2;
    } catch (const ConfigError& e) {
        set_err(err, errlen, std::string("config error: ") + e.what());
        return 2;
    } catch (const ValidationError& e) {
        set_err(err, errlen, std::string("validation error: ") + e.what());
        return 2;
    } catch (const UnknownProfileKey& e) {
        set_err(err, errlen, std::string("profile error: ") + e.what());
        return 2;
    } catch (const CorruptModelFile& e) {
        set_err(err, errlen, std::string("model error: ") + e.what());
        return 2;
    } catch (const std::exception& e) {
        set_err(err, errlen, std::string("runtime error: ") + e.what());
        return 3;
    }
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

std::uint64_t ref_fnv1a64(const char* data, std::size_t n, std::uint64_t seed) {
    return fnv1a64(std::string_view(data, n), seed);
}

void ref_rng_u64(std::uint64_t seed, const char* label, std::uint64_t* out, std::size_t n) {
    RngStream rng(seed, label);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

void ref_rng_unit(std::uint64_t seed, const char* label, double* out, std::size_t n) {
    RngStream rng(seed, label);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_unit();
}

void ref_rng_uniform_below(std::uint64_t seed, const char* label, std::uint64_t bound,
                           std::uint64_t* out, std::size_t n) {
    RngStream rng(seed, label);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.uniform_below(bound);
}

void ref_rng_lognormal(std::uint64_t seed, const char* label, double mu, double sigma,
                       double* out, std::size_t n) {
    RngStream rng(seed, label);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.lognormal(mu, sigma);
}

void ref_rng_exponential(std::uint64_t seed, const char* label, double mean, double* out,
                         std::size_t n) {
    RngStream rng(seed, label);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.exponential(mean);
}

void ref_net_delay(double rtt_ms, double jitter_ms, std::uint64_t seed, std::int64_t* out,
                   std::size_t n) {
    LinkSpec link{rtt_ms, jitter_ms};
    RngStream rng(seed, "jitter");
    for (std::size_t i = 0; i < n; ++i) out[i] = net_delay(link, rng);
}

// consume_acceptance on a 0/1 byte vector; writes {accepted, consumed} per call.
int ref_consume_acceptance(const std::uint8_t* bits, std::size_t nbits, const int* gammas,
                           std::size_t ncalls, int* out_pairs) {
    std::vector<std::uint8_t> v(bits, bits + nbits);
    std::size_t cursor = 0;
    try {
        for (std::size_t i = 0; i < ncalls; ++i) {
            auto [a, c] = consume_acceptance(v, cursor, gammas[i]);
            out_pairs[2 * i] = a;
            out_pairs[2 * i + 1] = c;
        }
    } catch (const std::exception&) {
        return 2;
    }
    return 0;
}

// Grid::interpolate through LatencyProfile::predict on the synthetic profile.
double ref_predict_synth(double target_decode_ms, double cost_ratio, double batch_coef,
                         double context_coef, double prefill_ms_per_token, int draft, int op,
                         int batch, int tokens, std::int64_t context) {
    LatencyProfile p = synth_profile(default_synth_spec(target_decode_ms, cost_ratio, batch_coef,
                                                        context_coef, prefill_ms_per_token));
    BatchShape s{batch, tokens, context};
    return p.predict(static_cast<OpKind>(op), s, draft ? kDraftModel : kTargetModel,
                     draft ? kEdgeHardware : kCloudHardware)
        .latency_ms;
}

// generate_synthetic -> serialize_trace JSONL (trace.cpp:104-187).
int ref_gen_trace(double rate_rps, std::int64_t n_requests, double acceptance_rate,
                  const char* preset, double prompt_median, double prompt_sigma,
                  double output_median, double output_sigma, std::int64_t n_drafts,
                  std::uint64_t seed, char** jsonl, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        SyntheticSpec spec;
        spec.rate_rps = rate_rps;
        spec.n_requests = n_requests;
        spec.acceptance_rate = acceptance_rate;
        if (preset && *preset) {
            spec.lengths = length_preset(preset);
        } else {
            spec.lengths.prompt_median = prompt_median;
            spec.lengths.prompt_sigma = prompt_sigma;
            spec.lengths.output_median = output_median;
            spec.lengths.output_sigma = output_sigma;
        }
        spec.n_drafts = n_drafts;
        *jsonl = dup_string(serialize_trace(generate_synthetic(spec, seed)));
    });
}

// resolve_config + run_simulation + aggregate_run (runner.cpp:96-169).
// agg = {completed, throughput_rps, mean_ttft_ms, mean_tpot_ms}.
int ref_run_config(const char* yaml_text, const char* base_dir, int has_seed,
                   std::uint64_t seed, int strict, char** report, std::uint64_t* events,
                   std::int64_t* end_time, double* agg, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        yaml::Node cfg = yaml::parse_string(yaml_text);
        ResolvedConfig rc =
            resolve_config(cfg, strict != 0,
                           has_seed ? std::optional<std::uint64_t>(seed) : std::nullopt,
                           base_dir ? base_dir : ".");
        SimulationOutput out = run_simulation(rc);
        if (report) *report = dup_string(out.report_json);
        if (events) *events = out.result.events_processed;
        if (end_time) *end_time = out.result.end_time;
        RunAggregates a = aggregate_run(out.result);
        if (agg) {
            agg[0] = static_cast<double>(a.completed);
            agg[1] = a.throughput_rps;
            agg[2] = a.mean_ttft_ms;
            agg[3] = a.mean_tpot_ms;
        }
    });
}

// Same as ref_run_config but also returns the per-request CSV
// (emit_report_csv, metrics.cpp:280-302) and the engine event log.
int ref_run_config_full(const char* yaml_text, const char* base_dir, int has_seed,
                        std::uint64_t seed, char** report, char** csv, char** event_log,
                        std::uint64_t* events, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        yaml::Node cfg = yaml::parse_string(yaml_text);
        ResolvedConfig rc =
            resolve_config(cfg, true, has_seed ? std::optional<std::uint64_t>(seed) : std::nullopt,
                           base_dir ? base_dir : ".");
        EngineOptions opts;
        opts.collect_event_log = event_log != nullptr;
        SimulationOutput out = run_simulation(rc, opts);
        if (report) *report = dup_string(out.report_json);
        if (csv) *csv = dup_string(emit_report_csv(out.result.records));
        if (event_log) {
            std::string log;
            for (const auto& l : out.result.event_log) {
                log += l;
                log += '\n';
            }
            *event_log = dup_string(log);
        }
        if (events) *events = out.result.events_processed;
    });
}

// RunResult::busy_intervals (engine.hpp:37-48, recorded at engine.cpp:563-564)
// of one run as text, one interval per line: "<t|d> <server id> <start> <end>".
int ref_run_config_busy(const char* yaml_text, const char* base_dir, int has_seed, std::uint64_t seed,
                        char** busy, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        yaml::Node cfg = yaml::parse_string(yaml_text);
        ResolvedConfig rc =
            resolve_config(cfg, true, has_seed ? std::optional<std::uint64_t>(seed) : std::nullopt,
                           base_dir ? base_dir : ".");
        SimulationOutput out = run_simulation(rc, EngineOptions{});
        std::string text;
        for (const auto& b : out.result.busy_intervals) {
            text += b.role == Role::Target ? "t " : "d ";
            text += std::to_string(b.server_id) + " " + std::to_string(b.start) + " " + std::to_string(b.end) + "\n";
        }
        *busy = dup_string(text);
    });
}

// The stock run_sweep + sweep_summary_json/csv (sweep.cpp:87-199).
int ref_run_sweep(const char* sweep_yaml, const char* base_dir, int parallel,
                  const char* out_dir, char** summary_json, char** summary_csv, char* err,
                  std::size_t errlen) {
    return guarded(err, errlen, [&] {
        yaml::Node node = yaml::parse_string(sweep_yaml);
        SweepSpec spec = SweepSpec::from_node(node, base_dir ? base_dir : ".");
        SweepResult r = run_sweep(spec, parallel, out_dir ? out_dir : "");
        if (summary_json) *summary_json = dup_string(sweep_summary_json(r));
        if (summary_csv) *summary_csv = dup_string(sweep_summary_csv(r));
    });
}

std::uint64_t ref_sweep_point_seed(std::uint64_t base, const char* point_id, int rep) {
    return sweep_point_seed(base, point_id, rep);
}

static int sweep_worker_run(const char* sweep_yaml, const char* base_dir, int threads,
                            const std::int64_t* points, std::int64_t n_points, double* out, double* rows,
                            char* err, std::size_t errlen);

// Timing harness for the CPU baseline: the run_sweep worker (sweep.cpp:112-150)
// reproduced with event counting (run_sweep itself does not return
// RunResult::events_processed).  Runs the listed point indices (all when
// n_points == 0) on `threads` std::threads with an atomic job counter, each
// job = one point with all its repetitions, exactly as the reference worker.
// out = {events, replicas, wall_seconds, failed_points, run_simulation seconds,
// resolve_config (+ generate_synthetic) seconds}, the last two summed over threads.
int ref_sweep_bench(const char* sweep_yaml, const char* base_dir, int threads,
                    const std::int64_t* points, std::int64_t n_points, double* out, char* err,
                    std::size_t errlen) {
    return sweep_worker_run(sweep_yaml, base_dir, threads, points, n_points, out, nullptr, err, errlen);
}

// The same worker over every point, keeping each replica's result: rows
// [point * repetitions + rep][6] = {events_processed, end_time, completed,
// throughput_rps, mean_ttft_ms, mean_tpot_ms} (RunResult, engine.hpp:44-53;
// RunAggregates, runner.hpp:53-60).  A failed point's rows are all -1.
int ref_sweep_replicas(const char* sweep_yaml, const char* base_dir, int threads, double* rows, char* err,
                       std::size_t errlen) {
    double out[6];
    return sweep_worker_run(sweep_yaml, base_dir, threads, nullptr, 0, out, rows, err, errlen);
}

static int sweep_worker_run(const char* sweep_yaml, const char* base_dir, int threads,
                            const std::int64_t* points, std::int64_t n_points, double* out, double* rows,
                            char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        yaml::Node node = yaml::parse_string(sweep_yaml);
        SweepSpec spec = SweepSpec::from_node(node, base_dir ? base_dir : ".");
        const std::size_t total = spec.point_count();
        std::vector<std::size_t> jobs;
        if (n_points <= 0) {
            for (std::size_t i = 0; i < total; ++i) jobs.push_back(i);
        } else {
            for (std::int64_t i = 0; i < n_points; ++i) jobs.push_back(static_cast<std::size_t>(points[i]) % total);
        }
        // point ids (sweep.cpp:95-107)
        auto point_id_of = [&](std::size_t idx) {
            std::vector<std::string> parts;
            std::size_t rem = idx;
            std::vector<std::pair<std::string, std::string>> assignment;
            for (std::size_t a = spec.axes.size(); a-- > 0;) {
                const auto& [path, values] = spec.axes[a];
                const yaml::Node& v = values[rem % values.size()];
                rem /= values.size();
                assignment.emplace_back(path, v.is_scalar() ? v.as_string() : v.canonical());
            }
            for (const auto& [k, v] : assignment) parts.push_back(k + "=" + v);
            std::sort(parts.begin(), parts.end());
            std::string id;
            for (const auto& p : parts) {
                if (!id.empty()) id += ';';
                id += p;
            }
            return id.empty() ? std::string("base") : id;
        };
        std::atomic<std::size_t> next{0};
        std::atomic<std::uint64_t> events{0};
        std::atomic<std::int64_t> replicas{0}, failed{0};
        std::atomic<std::uint64_t> resolve_ns{0}, sim_ns{0};  // thread-summed: the sim-only split
        auto worker = [&]() {
            for (;;) {
                std::size_t j = next.fetch_add(1);
                if (j >= jobs.size()) return;
                std::size_t idx = jobs[j];
                try {
                    yaml::Node config = spec.base_config;
                    std::size_t rem = idx;
                    for (std::size_t a = spec.axes.size(); a-- > 0;) {
                        const auto& [path, values] = spec.axes[a];
                        yaml::set_path(config, path, values[rem % values.size()]);
                        rem /= values.size();
                    }
                    std::string pid = point_id_of(idx);
                    double thr = 0.0, ttft = 0.0, tpot = 0.0;
                    for (int rep = 0; rep < spec.repetitions; ++rep) {
                        std::uint64_t seed = sweep_point_seed(spec.base_seed, pid, rep);
                        const auto ta = std::chrono::steady_clock::now();
                        ResolvedConfig rc = resolve_config(config, true, seed, spec.base_dir);
                        const auto tb = std::chrono::steady_clock::now();
                        SimulationOutput o = run_simulation(rc);
                        const auto tc = std::chrono::steady_clock::now();
                        resolve_ns.fetch_add(static_cast<std::uint64_t>(
                            std::chrono::duration_cast<std::chrono::nanoseconds>(tb - ta).count()));
                        sim_ns.fetch_add(static_cast<std::uint64_t>(
                            std::chrono::duration_cast<std::chrono::nanoseconds>(tc - tb).count()));
                        RunAggregates agg = aggregate_run(o.result);
                        thr += agg.throughput_rps;
                        ttft += agg.mean_ttft_ms;
                        tpot += agg.mean_tpot_ms;
                        events.fetch_add(o.result.events_processed);
                        replicas.fetch_add(1);
                        if (rows) {
                            double* row = rows + (idx * static_cast<std::size_t>(spec.repetitions) + rep) * 6;
                            row[0] = static_cast<double>(o.result.events_processed);
                            row[1] = static_cast<double>(o.result.end_time);
                            row[2] = static_cast<double>(agg.completed);
                            row[3] = agg.throughput_rps;
                            row[4] = agg.mean_ttft_ms;
                            row[5] = agg.mean_tpot_ms;
                        }
                    }
                    volatile double sink = thr + ttft + tpot;
                    (void)sink;
                } catch (const std::exception&) {
                    failed.fetch_add(1);
                    if (rows)
                        for (int rep = 0; rep < spec.repetitions; ++rep)
                            for (int f = 0; f < 6; ++f)
                                rows[(idx * static_cast<std::size_t>(spec.repetitions) + rep) * 6 + f] = -1.0;
                }
            }
        };
        auto t0 = std::chrono::steady_clock::now();
        int width = std::max(1, threads);
        if (width == 1) {
            worker();
        } else {
            std::vector<std::thread> pool;
            for (int i = 0; i < width; ++i) pool.emplace_back(worker);
            for (auto& t : pool) t.join();
        }
        double secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out[0] = static_cast<double>(events.load());
        out[1] = static_cast<double>(replicas.load());
        out[2] = secs;
        out[3] = static_cast<double>(failed.load());
        out[4] = 1e-9 * static_cast<double>(sim_ns.load());
        out[5] = 1e-9 * static_cast<double>(resolve_ns.load());
    });
}

// A randomly initialised WC-DNN with a given normaliser, saved in the
// reference wc-dnn/1 format (mlp.cpp:192-235).  Lets tests exercise the AWC
// path without the multi-second dataset+train pipeline.
int ref_random_model(std::uint64_t seed, int hidden, int blocks, const double* lo,
                     const double* hi, const char* path, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        AwcModel m;
        WcDnn::Dims d;
        d.hidden = hidden;
        d.blocks = blocks;
        RngStream rng(seed, "init");
        m.net = WcDnn::random_init(d, rng);
        // put the output bias mid-range so predictions span several windows
        m.net.params()[m.net.param_count() - 1] = 4.0;
        for (int f = 0; f < 5; ++f) {
            m.norm.lo[f] = lo[f];
            m.norm.hi[f] = hi[f];
        }
        m.hyper.hidden = hidden;
        m.hyper.blocks = blocks;
        m.train_seed = seed;
        m.save(path);
    });
}

// The full reference AWC pipeline (dataset.cpp:277-315 + train.cpp:94-177):
// build_scenarios(DatasetGrid{}) -> generate_dataset -> train_wc_dnn.
int ref_train_model(const char* path, int parallel, int epochs, std::uint64_t seed,
                    double* maes, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        auto scenarios = build_scenarios(DatasetGrid{});
        auto samples = generate_dataset(scenarios, ObjectiveWeights{}, parallel);
        TrainHyper h;
        if (epochs > 0) h.epochs = epochs;
        TrainResult r = train_wc_dnn(samples, h, seed);
        r.model.save(path);
        if (maes) {
            maes[0] = r.train_mae;
            maes[1] = r.val_mae;
            maes[2] = r.test_mae;
        }
    });
}

// AwcModel::predict_gamma on one raw feature vector (mlp.cpp:173-176).
int ref_awc_predict(const char* model_path, const double* features, std::size_t n_rows,
                    double* out, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        AwcModel m = AwcModel::load(model_path);
        for (std::size_t i = 0; i < n_rows; ++i) {
            std::array<double, 5> f{};
            for (int k = 0; k < 5; ++k) f[static_cast<std::size_t>(k)] = features[i * 5 + static_cast<std::size_t>(k)];
            out[i] = m.predict_gamma(f);
        }
    });
}

// build_scenarios + serialize_scenarios (dataset.cpp:50-108) of a
// DatasetGrid YAML document (DatasetGrid::from_node; empty = defaults).
int ref_build_scenarios(const char* grid_yaml, char** scenarios_jsonl, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        DatasetGrid g;
        if (grid_yaml && *grid_yaml) g = DatasetGrid::from_node(yaml::parse_string(grid_yaml));
        *scenarios_jsonl = dup_string(serialize_scenarios(build_scenarios(g)));
    });
}

// `specsim gen-dataset` (specsim_main.cpp:97-112): generate_dataset over
// build_scenarios(grid) with ObjectiveWeights{}, serialize_dataset.
int ref_generate_dataset(const char* grid_yaml, int parallel, char** dataset_jsonl, char** scenarios_jsonl,
                         char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        DatasetGrid g;
        if (grid_yaml && *grid_yaml) g = DatasetGrid::from_node(yaml::parse_string(grid_yaml));
        auto scenarios = build_scenarios(g);
        auto samples = generate_dataset(scenarios, ObjectiveWeights{}, parallel);
        *dataset_jsonl = dup_string(serialize_dataset(samples));
        *scenarios_jsonl = dup_string(serialize_scenarios(scenarios));
    });
}

// eval_policy_on_scenarios (dataset.cpp:292-369) on the scenarios of a
// scenarios JSONL with the given split ("all" = every scenario).
int ref_eval_policy(const char* scenarios_jsonl, const char* split, const char* window_kind, int gamma,
                    const char* model_path, int parallel, double* out, char* err, std::size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<ScenarioSpec> selected;
        const std::string sp = split ? split : "all";
        for (const auto& sc : parse_scenarios(scenarios_jsonl))
            if (sp == "all" || sc.split == sp) selected.push_back(sc);
        if (selected.empty()) throw ConfigError("no scenarios with split '" + sp + "'");
        PolicyEval e = eval_policy_on_scenarios(selected, window_kind, gamma, model_path ? model_path : "", parallel);
        out[0] = e.mean_throughput_rps;
        out[1] = e.mean_ttft_ms;
        out[2] = e.mean_tpot_ms;
        out[3] = e.mean_chosen_gamma;
    });
}

}  // extern "C"
