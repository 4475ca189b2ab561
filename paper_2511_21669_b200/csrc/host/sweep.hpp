// sweep.hpp — the simulate-a-sweep driver on the GPU engine: SweepSpec
// (proj/include/specsim/runner/sweep.hpp:17-50, proj/src/runner/sweep.cpp:16-199)
// resolved once per point, all (point, repetition) replicas in one device batch.
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../device/runtime.hpp"
#include "resolve.hpp"
#include "uninit.hpp"
#include "yaml.hpp"

namespace dsd::host {

struct SweepSpec {
    cfg::Node base;
    std::string base_dir;
    uint64_t base_seed = 42;
    int repetitions = 1;
    std::vector<std::pair<std::string, std::vector<cfg::Node>>> axes;
    static SweepSpec from_node(const cfg::Node& node, const std::string& base_dir);
    size_t point_count() const;
};

struct ReplicaOrigin {
    int64_t first;   // point
    int32_t second;  // repetition
};

struct SweepPoint {
    std::vector<std::pair<std::string, std::string>> assignment;
    std::string point_id;
    bool failed = false;
    std::string error;
    double mean_throughput_rps = 0.0, mean_ttft_ms = 0.0, mean_tpot_ms = 0.0;
    std::vector<std::string> report_files;
};

uint64_t sweep_point_seed(uint64_t base_seed, const std::string& point_id, int repetition);
// config digest of point idx (the reference's per-run config_digest)
std::string point_digest(const SweepSpec& spec, size_t idx);

// Points resolved into scenarios + replicas (optionally one shard of them).
struct SweepBatch {
    SweepSpec spec;
    std::vector<SweepPoint> points;
    std::vector<Resolved> resolved;          // one per resolvable point
    std::vector<int64_t> point_scenario;     // point -> index in resolved, -1 when failed
    std::vector<dsd_scenario> scenarios;
    uvector<dsd_replica> replicas;
    uvector<ReplicaOrigin> replica_origin;  // replica -> (point, rep)
    size_t point_base = 0;  // points[i] is sweep point point_base + i
};

SweepBatch plan_sweep(const cfg::Node& node, const std::string& base_dir, int shard, int n_shards, Caches* caches);
// Points [lo, hi) of a parsed spec, every replica (no sharding).
SweepBatch plan_range(const SweepSpec& spec, size_t lo, size_t hi, Caches* caches);

// DSD_HOST_TIMING=1: phase durations of the host sweep path to stderr
class PhaseTimer {
  public:
    explicit PhaseTimer(const char* what);
    void lap(const char* phase);

  private:
    const char* what_;
    bool on_;
    double t_ = 0.0;
};

struct SweepTotals {
    double points = 0, replicas = 0, failed = 0, events = 0;
};

// Summary text split per point: the part known before the run (id and
// assignment) and, once the points are filled in, the results.
struct SummaryParts {
    std::vector<std::string> json, csv;
};
// `first`: the sweep index of points[0] (the separator before the first entry)
SummaryParts render_summary_prefixes(const std::vector<SweepPoint>& points, size_t first = 0);
// Both texts in one parallel pass (either may be null).
void assemble_summaries(const SummaryParts& parts, const std::vector<SweepPoint>& points, std::string* json,
                        std::string* csv);
std::string assemble_summary_json(const SummaryParts& parts, const std::vector<SweepPoint>& points);
std::string assemble_summary_csv(const SummaryParts& parts, const std::vector<SweepPoint>& points);

// run_sweep on the GPU; writes per-replica reports when out_dir is non-empty.
// With `parts`, the summary prefixes are rendered while the kernels run.
SweepTotals run_sweep(Runtime& rt, SweepBatch& b, const std::string& out_dir, SummaryParts* parts = nullptr);
// The two halves of run_sweep: enqueue the batch on rt; wait for it and fill
// the points' means (writing reports when out_dir is set) into `tot`.
void launch_batch(Runtime& rt, SweepBatch& b, bool reports);
void collect_batch(Runtime& rt, SweepBatch& b, const std::string& out_dir, SweepTotals& tot);
std::string sweep_summary_json(const std::vector<SweepPoint>& points);
std::string sweep_summary_csv(const std::vector<SweepPoint>& points);

}  // namespace dsd::host
