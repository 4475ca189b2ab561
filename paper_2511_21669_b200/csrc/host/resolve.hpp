// resolve.hpp — config document -> dsd_scenario (the reference's
// resolve_config, proj/src/runner/runner.cpp:96-134, plus auto_topology,
// proj/src/config/topology.cpp:179-250, and the profile/trace/model loaders).
// A Resolved owns every array its dsd_scenario view points to.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "dsdsim.h"
#include "yaml.hpp"

namespace dsd::host {

struct ProfileTable {  // LatencyProfile (profile.hpp:26-84)
    struct Grid {
        std::vector<double> batch, context, values;
        double calibration = 1.0;
    };
    std::map<std::tuple<std::string, std::string, int>, int> index;  // (model, hw, op) -> grid
    std::vector<Grid> grids;
    std::vector<dsd_grid> view;
    int find(const std::string& model, const std::string& hw, int op) const;
    void add(const std::string& model, const std::string& hw, int op, Grid g);
    void finalize();
};

struct TraceData {  // TraceRecord[] (trace.hpp:14-22)
    std::vector<int64_t> prompt, output, arrival, drafter, bits_offset;
    std::vector<uint8_t> bits;
    dsd_trace view{};
    void finalize();
};

struct AwcData {  // AwcModel (mlp.hpp:80-96)
    std::vector<double> params;
    dsd_awc_model view{};
};

struct Caches {
    std::mutex mu;
    std::map<std::string, std::shared_ptr<const ProfileTable>> profiles;
    std::map<std::string, std::shared_ptr<const AwcData>> models;
    std::map<std::string, std::shared_ptr<const TraceData>> traces;
};

struct Resolved {
    std::vector<int32_t> tgroup, dgroup;
    std::vector<dsd_link> links;
    std::vector<int32_t> tgrids, dgrids;
    std::shared_ptr<const ProfileTable> profile;
    std::shared_ptr<const AwcData> awc;
    std::shared_ptr<const TraceData> trace;
    uint64_t seed = 42;
    uint64_t gen_seed = 42;
    bool gen_seed_fixed = false;  // workload.gen_seed given explicitly
    std::string digest;
    dsd_scenario scen{};
    void bind();  // (re)points scen's arrays at the owned vectors
};

// Throws dsd::Error.  `caches` may be null.  `want_digest` = false leaves
// Resolved::digest empty (sweeps compute it only for report files).
Resolved resolve_config(const cfg::Node& config, bool strict, std::optional<uint64_t> seed_override,
                        const std::string& base_dir, Caches* caches, bool want_digest = true);

std::shared_ptr<const TraceData> load_trace_file(const std::string& path);
std::shared_ptr<const TraceData> parse_trace_text(const std::string& text);
std::shared_ptr<const ProfileTable> load_profile_file(const std::string& path);
std::shared_ptr<const AwcData> load_model_file(const std::string& path);
std::shared_ptr<const ProfileTable> synth_profile(double target_decode_ms, double cost_ratio,
                                                  double batch_coef, double context_coef,
                                                  double prefill_ms_per_token);
std::string join_path(const std::string& base, const std::string& path);

}  // namespace dsd::host
