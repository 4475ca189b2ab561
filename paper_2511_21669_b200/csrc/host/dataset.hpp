// dataset.hpp — AWC training-data generation and window-policy evaluation on
// the GPU engine: proj/include/specsim/awc/dataset.hpp and
// proj/src/awc/dataset.cpp.  Every (scenario, candidate) simulation of the
// reference's thread pool becomes one replica of a single device batch, run
// with the engine's feature probe.
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "../device/runtime.hpp"
#include "resolve.hpp"
#include "yaml.hpp"

namespace dsd::host {

// ScenarioSpec (dataset.hpp:14-30)
struct ScenarioSpec {
    uint64_t scenario_id = 0;
    std::string split;
    double rtt_ms = 10.0, jitter_ms = 0.0, alpha = 0.8, load_factor = 0.5;
    int drafts = 4, targets = 1;
    double target_decode_ms = 15.0, cost_ratio = 0.1, prompt_median = 24.0, output_median = 56.0;
    int n_requests = 36;
    uint64_t seed = 0;
};

// DatasetGrid (dataset.hpp:32-44) + DatasetGrid::from_node (dataset.cpp:33-48)
struct DatasetGrid {
    std::vector<double> rtt_ms = {2, 10, 30, 60, 100};
    std::vector<double> alpha = {0.3, 0.5, 0.7, 0.85, 0.95};
    std::vector<double> load_factor = {0.35, 0.8};
    std::vector<int> drafts = {2, 6};
    std::vector<double> cost_ratio = {0.05, 0.15};
    double target_decode_ms = 15.0;
    int n_requests = 36;
    uint64_t seed = 20240501;
    static DatasetGrid from_node(const cfg::Node& node);
};

struct ObjectiveWeights {  // dataset.hpp:55-59
    double w_tpot = 0.5, w_ttft = 0.2, w_throughput = 0.3;
};

struct CandidateOutcome {  // dataset.hpp:61-69
    int gamma = 2;  // 1 encodes fused
    bool fused = false;
    double throughput_rps = 0.0, mean_ttft_ms = 0.0, mean_tpot_ms = 0.0;
    std::array<double, 5> mean_features{};
    double objective = 0.0;
};

struct ScenarioSweepResult {  // dataset.hpp:71-75
    ScenarioSpec scenario;
    std::vector<CandidateOutcome> candidates;  // gamma 2..12 then fused
    int label_gamma = 2;
};

struct PolicyEval {  // dataset.hpp:101-108
    std::string policy;
    double mean_throughput_rps = 0.0, mean_ttft_ms = 0.0, mean_tpot_ms = 0.0, mean_chosen_gamma = 0.0;
};

std::vector<ScenarioSpec> build_scenarios(const DatasetGrid& grid);
std::string serialize_scenarios(const std::vector<ScenarioSpec>& scenarios);
std::vector<ScenarioSpec> parse_scenarios(const std::string& text);

// scenario_trace's arrival rate (dataset.cpp:125-133) and scenario_config
// (dataset.cpp:149-186) with the trace expressed as the equivalent synthetic
// workload section (same generator, seed and parameters)
double scenario_rate(const ScenarioSpec& s);
cfg::Node scenario_config(const ScenarioSpec& s, const std::string& window_kind, int gamma,
                          const std::string& model_path);

void score_candidates(std::vector<CandidateOutcome>& candidates, const ObjectiveWeights& weights);
int pick_label(const std::vector<CandidateOutcome>& candidates);

// generate_dataset (dataset.cpp:248-290): all scenarios x 12 candidates in one
// device batch; returns the per-scenario sweeps (samples are derived from them)
std::vector<ScenarioSweepResult> generate_dataset(Runtime& rt, const std::vector<ScenarioSpec>& scenarios,
                                                  const ObjectiveWeights& weights, Caches* caches);
// serialize_dataset (train.cpp:16-33) of the samples generate_dataset emits
std::string serialize_dataset(const std::vector<ScenarioSweepResult>& sweeps);

// eval_policy_on_scenarios (dataset.cpp:292-369): one replica per scenario
PolicyEval eval_policy_on_scenarios(Runtime& rt, const std::vector<ScenarioSpec>& scenarios,
                                    const std::string& window_kind, int gamma, const std::string& model_path,
                                    Caches* caches);

}  // namespace dsd::host
