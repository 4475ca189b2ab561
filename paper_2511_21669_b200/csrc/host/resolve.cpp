// resolve.cpp — configuration resolution for the GPU engine.  Restates the
// reference's host-side pipeline so the device receives exactly the inputs
// the reference Engine would:
//   auto_topology / parse_groups / parse_policies   proj/src/config/topology.cpp:13-250
//   profile_from / synth_profile / default_synth_spec runner.cpp:40-69, profile.cpp:192-278
//   resolve_config                                   runner.cpp:96-134
//   Engine::Impl ctor checks                         engine.cpp:165-195
//   load_trace / parse_trace / validate_record       trace.cpp:31-102
//   AwcModel::parse                                  mlp.cpp:238-287
// Error texts and their status class match the reference
// (ParseError/ConfigError/ValidationError/UnknownProfileKey/CorruptModelFile
// -> DSD_ERR_CONFIG; IoError and the rest -> DSD_ERR_RUNTIME).
#include "resolve.hpp"

#include <sys/stat.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <set>
#include <initializer_list>
#include <string_view>
#include <sstream>

#include <json.hpp>

#include "../device/runtime.hpp"

namespace dsd::host {

using cfg::Node;
using nlohmann::json;

namespace {

[[noreturn]] void config_error(const std::string& m) { throw Error(DSD_ERR_CONFIG, m); }
[[noreturn]] void io_error(const std::string& m) { throw Error(DSD_ERR_RUNTIME, m); }

const char* kTargetModel = "target-model";
const char* kCloudHw = "cloud-gpu";
const char* kDraftModel = "draft-model";
const char* kEdgeHw = "edge-gpu";

// (a handful of literal keys: a linear scan, no per-call allocation)
void check_keys(const Node& n, std::initializer_list<std::string_view> allowed, std::string_view where, bool strict) {
    if (!strict || !n.map()) return;
    for (const auto& f : n.fields)
        if (std::find(allowed.begin(), allowed.end(), std::string_view(f.first)) == allowed.end())
            config_error("unknown key '" + f.first + "' in " + std::string(where) + " (use lenient mode to ignore)");
}

struct Group {
    int count = 1;
    std::string model, hardware;
    int gpu_count = 1;
};

std::vector<Group> parse_groups(const Node& pool, bool draft, const std::string& where, bool strict) {
    const std::string dm = draft ? kDraftModel : kTargetModel;
    const std::string dh = draft ? kEdgeHw : kCloudHw;
    auto one = [&](const Node& g) {
        check_keys(g, {"count", "model", "hardware", "gpu_count"}, where, strict);
        Group grp;
        grp.count = static_cast<int>(g.int_or("count", 1));
        grp.model = g.string_or("model", dm);
        grp.hardware = g.string_or("hardware", dh);
        grp.gpu_count = static_cast<int>(g.int_or("gpu_count", 1));
        if (grp.count < 0) config_error(where + ": count must be >= 0");
        if (grp.gpu_count < 1) config_error(where + ": gpu_count must be >= 1");
        return grp;
    };
    std::vector<Group> out;
    if (pool.null()) return out;
    if (pool.kind == Node::Kind::Int) {
        Group g{static_cast<int>(pool.i), dm, dh, 1};
        if (g.count < 0) config_error(where + ": count must be >= 0");
        if (g.count > 0) out.push_back(g);
    } else if (pool.seq()) {
        for (const auto& g : pool.items) out.push_back(one(g));
    } else if (pool.map() && pool.has("groups")) {
        check_keys(pool, {"count", "groups"}, where, strict);
        for (const auto& g : pool.get("groups")->items) out.push_back(one(g));
        if (pool.has("count")) {
            int64_t declared = pool.int_or("count", 0), total = 0;
            for (const auto& g : out) total += g.count;
            if (declared != total)
                config_error(where + ": declared count " + std::to_string(declared) +
                             " does not match group total " + std::to_string(total));
        }
    } else if (pool.map()) {
        out.push_back(one(pool));
    } else {
        config_error(where + ": expected a count, a group, or a list of groups");
    }
    return out;
}

int routing_of(const std::string& s) {
    if (s == "random") return DSD_ROUTE_RANDOM;
    if (s == "rr" || s == "round_robin" || s == "round-robin") return DSD_ROUTE_ROUND_ROBIN;
    if (s == "jsq") return DSD_ROUTE_JSQ;
    config_error("unknown routing policy '" + s + "'");
}
int batching_of(const std::string& s) {
    if (s == "fifo") return DSD_BATCH_FIFO;
    if (s == "lab") return DSD_BATCH_LAB;
    config_error("unknown batching policy '" + s + "'");
}
int window_of(const std::string& s) {
    if (s == "static") return DSD_WINDOW_STATIC;
    if (s == "dynamic") return DSD_WINDOW_DYNAMIC;
    if (s == "awc") return DSD_WINDOW_AWC;
    if (s == "fused") return DSD_WINDOW_FUSED;
    config_error("unknown window policy '" + s + "'");
}

struct Policy {
    int routing = DSD_ROUTE_RANDOM, batching = DSD_BATCH_FIFO, max_batch = 8;
    int64_t window_us = 0;
    double sim_frac = 0.2;
    int window = DSD_WINDOW_STATIC, gamma = 4, gamma_min = 1, gamma_max = 12;
    std::string model_path;
    int queue_capacity = 64, draft_max_batch = 1;
};

Policy parse_policies(const Node& config, bool strict) {
    Policy p;
    const Node* pol = config.get("policies");
    if (!pol || pol->null()) return p;
    check_keys(*pol, {"routing", "batching", "window", "queue_capacity", "draft_max_batch"}, "policies", strict);
    p.routing = routing_of(pol->string_or("routing", "random"));
    if (const Node* b = pol->get("batching")) {
        if (b->scalar()) {
            p.batching = batching_of(b->to_string());
        } else if (b->map()) {
            check_keys(*b, {"kind", "max_batch_size", "batching_window_us", "similarity_fraction"},
                       "policies.batching", strict);
            p.batching = batching_of(b->string_or("kind", "fifo"));
            p.max_batch = static_cast<int>(b->int_or("max_batch_size", 8));
            p.window_us = b->int_or("batching_window_us", 0);
            p.sim_frac = b->double_or("similarity_fraction", 0.2);
        }
    }
    if (const Node* w = pol->get("window")) {
        if (w->scalar()) {
            p.window = window_of(w->to_string());
        } else if (w->map()) {
            check_keys(*w, {"kind", "gamma", "gamma_min", "gamma_max", "model"}, "policies.window", strict);
            p.window = window_of(w->string_or("kind", "static"));
            p.gamma = static_cast<int>(w->int_or("gamma", 4));
            p.gamma_min = static_cast<int>(w->int_or("gamma_min", 1));
            p.gamma_max = static_cast<int>(w->int_or("gamma_max", 12));
            p.model_path = w->string_or("model", "");
        }
    }
    p.queue_capacity = static_cast<int>(pol->int_or("queue_capacity", 64));
    p.draft_max_batch = static_cast<int>(pol->int_or("draft_max_batch", 1));
    if (p.max_batch < 1) config_error("batching.max_batch_size must be >= 1");
    if (p.sim_frac < 0.0) config_error("batching.similarity_fraction must be >= 0");
    if (p.gamma_min < 1 || p.gamma_max < p.gamma_min)
        config_error("window gamma bounds must satisfy 1 <= gamma_min <= gamma_max");
    if (p.window == DSD_WINDOW_STATIC && (p.gamma < p.gamma_min || p.gamma > p.gamma_max))
        config_error("static window gamma out of [gamma_min, gamma_max]");
    if (p.queue_capacity < 1) config_error("queue_capacity must be >= 1");
    return p;
}

struct Device {
    std::string model, hardware;
    int group;
};

struct Topology {
    std::vector<Device> targets, drafts;
    int n_tg = 0, n_dg = 0;
    dsd_link def{0.0, 0.0};
    std::vector<std::pair<std::pair<int, int>, dsd_link>> overrides;  // in declaration order
    Policy policy;
};

Topology auto_topology(const Node& config, bool strict) {
    if (!config.map()) config_error("config root must be a mapping");
    check_keys(config, {"targets", "drafts", "network", "policies", "workload", "seed", "latency_profile"},
               "config", strict);
    Topology t;
    static const Node kNull;
    const Node* tn = config.get("targets");
    const Node* dn = config.get("drafts");
    std::vector<Group> tgs = parse_groups(tn ? *tn : kNull, false, "targets", strict);
    std::vector<Group> dgs = parse_groups(dn ? *dn : kNull, true, "drafts", strict);
    for (size_t g = 0; g < tgs.size(); ++g)
        for (int i = 0; i < tgs[g].count; ++i) t.targets.push_back(Device{tgs[g].model, tgs[g].hardware, static_cast<int>(g)});
    for (size_t g = 0; g < dgs.size(); ++g)
        for (int i = 0; i < dgs[g].count; ++i) t.drafts.push_back(Device{dgs[g].model, dgs[g].hardware, static_cast<int>(g)});
    t.n_tg = static_cast<int>(tgs.size());
    t.n_dg = static_cast<int>(dgs.size());
    if (t.targets.empty()) config_error("target pool must be non-empty");
    if (const Node* net = config.get("network"); net && !net->null()) {
        check_keys(*net, {"rtt_ms", "jitter_ms", "overrides"}, "network", strict);
        t.def.rtt_ms = net->double_or("rtt_ms", 0.0);
        t.def.jitter_ms = net->double_or("jitter_ms", 0.0);
        if (const Node* ov = net->get("overrides"); ov && ov->seq()) {
            for (const auto& o : ov->items) {
                check_keys(o, {"draft_group", "target_group", "rtt_ms", "jitter_ms"}, "network.overrides", strict);
                int dg = static_cast<int>(o.int_or("draft_group", 0));
                int tg = static_cast<int>(o.int_or("target_group", 0));
                if (dg < 0 || dg >= t.n_dg || tg < 0 || tg >= t.n_tg)
                    config_error("network override references a group out of range");
                dsd_link l;
                l.rtt_ms = o.double_or("rtt_ms", t.def.rtt_ms);
                l.jitter_ms = o.double_or("jitter_ms", t.def.jitter_ms);
                t.overrides.push_back({{dg, tg}, l});
            }
        }
    }
    auto check_link = [](const dsd_link& l) {
        if (l.rtt_ms < 0.0 || l.jitter_ms < 0.0) config_error("link rtt_ms/jitter_ms must be >= 0");
        if (l.jitter_ms > l.rtt_ms) config_error("link jitter_ms must not exceed rtt_ms");
    };
    check_link(t.def);
    // the reference checks overrides in (draft_group, target_group) map order
    {
        std::map<std::pair<int, int>, dsd_link> m;
        for (const auto& kv : t.overrides) m[kv.first] = kv.second;
        for (const auto& kv : m) check_link(kv.second);
    }
    t.policy = parse_policies(config, strict);
    if (t.drafts.empty() && t.policy.window != DSD_WINDOW_FUSED)
        config_error("empty draft pool requires the fused window policy");
    return t;
}

std::string slurp(const std::string& path, const char* what) {
    std::ifstream in(path);
    if (!in) io_error(std::string("cannot open ") + what + " file: " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return buf.str();
}

int op_of(const std::string& s) {
    if (s == "prefill") return 0;
    if (s == "decode") return 1;
    if (s == "verify") return 2;
    config_error("profile: unknown op '" + s + "'");
}

}  // namespace

std::string join_path(const std::string& base, const std::string& path) {
    if (path.empty() || path.front() == '/' || base.empty() || base == ".") return path;
    return base + "/" + path;
}

// ---------------------------------------------------------------------------
// latency profiles
// ---------------------------------------------------------------------------
int ProfileTable::find(const std::string& model, const std::string& hw, int op) const {
    if (op == 2) op = 1;  // verify is decode-shaped (profile.cpp:103-118)
    auto it = index.find({model, hw, op});
    return it == index.end() ? -1 : it->second;
}

void ProfileTable::add(const std::string& model, const std::string& hw, int op, Grid g) {
    // LatencyProfile::add_grid checks (profile.cpp:90-101)
    auto check_axis = [](const std::vector<double>& a, const char* name) {
        if (a.empty()) config_error(std::string("profile grid: empty ") + name);
        for (size_t i = 1; i < a.size(); ++i)
            if (!(a[i] > a[i - 1])) config_error(std::string("profile grid: ") + name + " must be strictly increasing");
    };
    check_axis(g.batch, "batch axis");
    check_axis(g.context, "context axis");
    if (g.values.size() != g.batch.size() * g.context.size())
        config_error("profile grid: values size does not match axes");
    for (double v : g.values)
        if (!(v > 0.0)) config_error("profile grid: latencies must be positive");
    auto key = std::make_tuple(model, hw, op);
    auto it = index.find(key);
    if (it != index.end()) {
        grids[it->second] = std::move(g);
    } else {
        index[key] = static_cast<int>(grids.size());
        grids.push_back(std::move(g));
    }
}

void ProfileTable::finalize() {
    view.resize(grids.size());
    for (size_t i = 0; i < grids.size(); ++i) {
        view[i].n_batch = static_cast<int32_t>(grids[i].batch.size());
        view[i].n_context = static_cast<int32_t>(grids[i].context.size());
        view[i].batch_axis = grids[i].batch.data();
        view[i].context_axis = grids[i].context.data();
        view[i].values_ms = grids[i].values.data();
        view[i].calibration = grids[i].calibration;
    }
}

std::shared_ptr<const ProfileTable> synth_profile(double target_decode_ms, double cost_ratio, double batch_coef,
                                                  double context_coef, double prefill_ms_per_token) {
    // default_synth_spec + synth_profile (profile.cpp:221-278)
    if (!(cost_ratio > 0.0)) config_error("cost ratio must be positive");
    struct Entry {
        const char* model;
        const char* hw;
        double decode_base, prefill_per_token;
    };
    const Entry entries[2] = {{kTargetModel, kCloudHw, target_decode_ms, prefill_ms_per_token},
                              {kDraftModel, kEdgeHw, target_decode_ms * cost_ratio, prefill_ms_per_token * cost_ratio}};
    static const double kBatch[] = {1, 2, 4, 8, 16, 32, 64, 128, 256};
    static const double kCtx[] = {0, 64, 128, 256, 512, 1024, 2048, 4096};
    const double context_ref = 512.0;
    auto table = std::make_shared<ProfileTable>();
    for (const Entry& e : entries) {
        if (!(e.decode_base > 0.0) || !(e.prefill_per_token > 0.0))
            config_error("synth profile: base latencies must be positive");
        if (batch_coef < 0.0 || context_coef < 0.0)
            config_error("synth profile: coefficients must be non-negative");
        ProfileTable::Grid dec, pre;
        dec.batch.assign(std::begin(kBatch), std::end(kBatch));
        dec.context.assign(std::begin(kCtx), std::end(kCtx));
        pre.batch = dec.batch;
        pre.context = dec.context;
        for (double b : kBatch)
            for (double c : kCtx) {
                double batch_scale = 1.0 + batch_coef * (b - 1.0);
                dec.values.push_back(e.decode_base * batch_scale *
                                     (1.0 + context_coef * std::sqrt(c / context_ref)));
                pre.values.push_back(e.prefill_per_token * (c + 1.0) * batch_scale);
            }
        table->add(e.model, e.hw, 1, std::move(dec));
        table->add(e.model, e.hw, 0, std::move(pre));
    }
    table->finalize();
    return table;
}

std::shared_ptr<const ProfileTable> load_profile_file(const std::string& path) {
    const std::string text = slurp(path, "profile");
    json j = json::parse(text, nullptr, false);
    if (j.is_discarded() || !j.is_object() || !j.contains("entries")) config_error("profile: invalid JSON document");
    auto table = std::make_shared<ProfileTable>();
    try {
        for (const auto& e : j["entries"]) {
            ProfileTable::Grid g;
            g.calibration = e.value("calibration", 1.0);
            g.batch = e.at("batch_axis").get<std::vector<double>>();
            g.context = e.at("context_axis").get<std::vector<double>>();
            g.values = e.at("values_ms").get<std::vector<double>>();
            table->add(e.at("model").get<std::string>(), e.at("hardware").get<std::string>(),
                       op_of(e.at("op").get<std::string>()), std::move(g));
        }
    } catch (const json::exception& e) {
        io_error(e.what());
    }
    table->finalize();
    return table;
}

// ---------------------------------------------------------------------------
// traces
// ---------------------------------------------------------------------------
void TraceData::finalize() {
    view.n = static_cast<int64_t>(prompt.size());
    view.prompt_length = prompt.data();
    view.output_length = output.data();
    view.arrival_us = arrival.data();
    view.drafter_id = drafter.data();
    view.bits_offset = bits_offset.data();
    view.acceptance_bits = bits.data();
}

std::shared_ptr<const TraceData> parse_trace_text(const std::string& text) {
    auto t = std::make_shared<TraceData>();
    t->bits_offset.push_back(0);
    std::istringstream in(text);
    std::string line;
    int line_no = 0;
    const std::string lp = "trace line ";
    try {
        while (std::getline(in, line)) {
            ++line_no;
            if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
            const std::string ln = lp + std::to_string(line_no);
            json j = json::parse(line, nullptr, false);
            if (j.is_discarded() || !j.is_object()) config_error(ln + ": invalid JSON record");
            auto req_int = [&](const char* key) {
                auto it = j.find(key);
                if (it == j.end() || !it->is_number_integer())
                    config_error(ln + ": missing integer field '" + key + "'");
                return it->get<int64_t>();
            };
            int64_t prompt = req_int("prompt_length");
            int64_t output = req_int("output_length");
            auto at = j.find("arrival_time_ms");
            if (at == j.end() || !at->is_number()) config_error(ln + ": missing numeric field 'arrival_time_ms'");
            int64_t arrival = static_cast<int64_t>(std::llround(at->get<double>() * 1000.0));
            int64_t drafter = req_int("drafter_id");
            auto sq = j.find("acceptance_seq");
            if (sq == j.end() || !sq->is_array()) config_error(ln + ": missing array field 'acceptance_seq'");
            const size_t idx = t->prompt.size();
            std::vector<uint8_t> bits;
            bits.reserve(sq->size());
            for (const auto& b : *sq) {
                if (!b.is_number_integer()) config_error(ln + ": acceptance_seq must contain integers");
                bits.push_back(static_cast<uint8_t>(b.get<int>()));
            }
            // validate_record (trace.cpp:31-47)
            const std::string rw = "trace record " + std::to_string(idx) + ": field '";
            if (prompt < 1) config_error(rw + "prompt_length' must be >= 1");
            if (output < 0) config_error(rw + "output_length' must be >= 0");
            if (arrival < 0) config_error(rw + "arrival_time_ms' must be >= 0");
            if (drafter < 0) config_error(rw + "drafter_id' must be >= 0");
            if (output > 0 && bits.empty()) config_error(rw + "acceptance_seq' must be non-empty when output_length > 0");
            for (uint8_t b : bits)
                if (b > 1) config_error(rw + "acceptance_seq' contains a value other than 0/1");
            t->prompt.push_back(prompt);
            t->output.push_back(output);
            t->arrival.push_back(arrival);
            t->drafter.push_back(drafter);
            t->bits.insert(t->bits.end(), bits.begin(), bits.end());
            t->bits_offset.push_back(static_cast<int64_t>(t->bits.size()));
        }
    } catch (const json::exception& e) {
        io_error(e.what());
    }
    t->finalize();
    return t;
}

std::shared_ptr<const TraceData> load_trace_file(const std::string& path) {
    return parse_trace_text(slurp(path, "trace"));
}

// ---------------------------------------------------------------------------
// AWC model (wc-dnn/1, mlp.cpp:180-287)
// ---------------------------------------------------------------------------
std::shared_ptr<const AwcData> load_model_file(const std::string& path) {
    const std::string text = slurp(path, "model");
    json j = json::parse(text, nullptr, false);
    if (j.is_discarded() || !j.is_object()) config_error("model file is not valid JSON");
    auto m = std::make_shared<AwcData>();
    try {
        if (j.at("format").get<std::string>() != "wc-dnn/1") config_error("unsupported model format");
        int input = j.at("dims").at("input").get<int>();
        int hidden = j.at("dims").at("hidden").get<int>();
        int blocks = j.at("dims").at("blocks").get<int>();
        if (input < 1 || hidden < 1 || blocks < 0) config_error("invalid network dimensions");
        auto lo = j.at("normalizer").at("lo").get<std::vector<double>>();
        auto hi = j.at("normalizer").at("hi").get<std::vector<double>>();
        auto ls = j.at("normalizer").at("log_scale").get<std::vector<bool>>();
        if (lo.size() != 5 || hi.size() != 5 || ls.size() != 5)
            config_error("normalizer must have five entries");
        const auto& hp = j.at("hyperparams");
        (void)hp.at("lr").get<double>();
        (void)hp.at("weight_decay").get<double>();
        (void)hp.at("beta1").get<double>();
        (void)hp.at("beta2").get<double>();
        (void)hp.at("eps").get<double>();
        (void)hp.at("epochs").get<int>();
        (void)hp.at("batch_size").get<int>();
        (void)hp.at("seed").get<uint64_t>();
        m->params = j.at("weights").get<std::vector<double>>();
        const int64_t H = hidden, I = input;
        const int64_t expect = H * I + H + static_cast<int64_t>(blocks) * (2 * H * H + 2 * H) + H + 1;
        if (static_cast<int64_t>(m->params.size()) != expect) config_error("weight count does not match dims");
        std::string blob;
        for (double v : m->params) {
            blob += cfg::fmt_exact(v);
            blob += ';';
        }
        if (j.at("checksum").get<std::string>() != cfg::hex16(cfg::fnv1a64(blob)))
            config_error("model checksum mismatch");
        m->view.input = input;
        m->view.hidden = hidden;
        m->view.blocks = blocks;
        for (int f = 0; f < 5; ++f) {
            m->view.norm_lo[f] = lo[f];
            m->view.norm_hi[f] = hi[f];
            m->view.log_scale[f] = ls[f] ? 1 : 0;
        }
    } catch (const json::exception& e) {
        config_error(std::string("model file structure: ") + e.what());
    }
    m->view.params = m->params.data();
    return m;
}

// ---------------------------------------------------------------------------
// resolve_config
// ---------------------------------------------------------------------------
void Resolved::bind() {
    scen.target_group = tgroup.data();
    scen.draft_group = dgroup.empty() ? nullptr : dgroup.data();
    scen.links = links.data();
    scen.n_grids = static_cast<int32_t>(profile->view.size());
    scen.grids = profile->view.data();
    scen.target_grids = tgrids.data();
    scen.draft_grids = dgrids.empty() ? nullptr : dgrids.data();
    scen.awc = awc ? &awc->view : nullptr;
    scen.trace = trace ? &trace->view : nullptr;
}

namespace {

// Cache key of a file-backed input: its path plus size and modification
// time, so a model / trace / profile rewritten at the same path between two
// calls on one handle is read again (the reference re-reads every input on
// each resolve_config, runner.cpp:96-134).  A file that cannot be stat'ed
// keys by path alone (its loader reports the error).
std::string file_key(const std::string& path) {
    struct stat st;
    if (::stat(path.c_str(), &st) != 0) return path;
    return path + "|" + std::to_string(static_cast<long long>(st.st_size)) + "|" +
           std::to_string(static_cast<long long>(st.st_mtim.tv_sec)) + "." +
           std::to_string(static_cast<long long>(st.st_mtim.tv_nsec)) + "|" +
           std::to_string(static_cast<unsigned long long>(st.st_ino));
}

template <typename T, typename F>
std::shared_ptr<const T> cached(Caches* caches, std::map<std::string, std::shared_ptr<const T>> Caches::*slot,
                                const std::string& key, F&& make) {
    if (!caches) return make();
    {
        std::lock_guard<std::mutex> lk(caches->mu);
        auto& m = caches->*slot;
        auto it = m.find(key);
        if (it != m.end()) return it->second;
    }
    auto v = make();
    // planner threads that missed together share the first table inserted
    // (one copy of each latency grid in the device blob)
    std::lock_guard<std::mutex> lk(caches->mu);
    return (caches->*slot).emplace(key, std::move(v)).first->second;
}

}  // namespace

Resolved resolve_config(const Node& config, bool strict, std::optional<uint64_t> seed_override,
                        const std::string& base_dir, Caches* caches, bool want_digest) {
    Resolved rc;
    Topology topo = auto_topology(config, strict);
    // profile_from (runner.cpp:40-69)
    {
        const Node* node = config.get("latency_profile");
        if (!node || node->null())
            config_error("config requires 'latency_profile' (a path or an inline synth spec)");
        if (node->scalar()) {
            const std::string path = join_path(base_dir, node->to_string());
            rc.profile = cached(caches, &Caches::profiles, "file:" + file_key(path), [&] { return load_profile_file(path); });
        } else if (node->map() && node->has("synth")) {
            const Node& s = *node->get("synth");
            if (strict) {
                static const std::set<std::string> allowed = {"target_decode_ms", "cost_ratio", "batch_coef",
                                                              "context_coef", "prefill_ms_per_token"};
                if (s.map())
                    for (const auto& f : s.fields)
                        if (!allowed.count(f.first))
                            config_error("unknown key '" + f.first + "' in latency_profile.synth");
            }
            const double v[5] = {s.double_or("target_decode_ms", 20.0), s.double_or("cost_ratio", 0.1),
                                 s.double_or("batch_coef", 0.05), s.double_or("context_coef", 0.3),
                                 s.double_or("prefill_ms_per_token", 0.2)};
            // keyed by the five values' bit patterns (a sweep's points mostly
            // share one synth spec: the planner thread's last lookup is
            // reused without the cache lock)
            thread_local uint64_t last_bits[5];
            thread_local const Caches* last_caches = nullptr;
            thread_local std::shared_ptr<const ProfileTable> last_profile;
            uint64_t b[5];
            std::memcpy(b, v, sizeof(b));
            if (caches && last_caches == caches && last_profile && std::memcmp(b, last_bits, sizeof(b)) == 0) {
                rc.profile = last_profile;
            } else {
                char key[96];
                std::snprintf(key, sizeof(key), "synth:%016llx%016llx%016llx%016llx%016llx",
                              static_cast<unsigned long long>(b[0]), static_cast<unsigned long long>(b[1]),
                              static_cast<unsigned long long>(b[2]), static_cast<unsigned long long>(b[3]),
                              static_cast<unsigned long long>(b[4]));
                rc.profile = cached(caches, &Caches::profiles, key,
                                    [&] { return synth_profile(v[0], v[1], v[2], v[3], v[4]); });
                if (caches) {
                    std::memcpy(last_bits, b, sizeof(b));
                    last_caches = caches;
                    last_profile = rc.profile;
                }
            }
        } else {
            config_error("latency_profile must be a path or {synth: {...}}");
        }
    }
    const uint64_t cfg_seed = static_cast<uint64_t>(config.int_or("seed", 42));
    rc.seed = seed_override.value_or(cfg_seed);
    if (want_digest) rc.digest = cfg::hex16(cfg::fnv1a64(config.canonical()));
    const Policy& pol = topo.policy;
    if (pol.window == DSD_WINDOW_AWC && !topo.drafts.empty()) {
        if (pol.model_path.empty()) config_error("window policy 'awc' requires policies.window.model");
        const std::string path = join_path(base_dir, pol.model_path);
        rc.awc = cached(caches, &Caches::models, file_key(path), [&] { return load_model_file(path); });
    }
    dsd_scenario& s = rc.scen;
    s = dsd_scenario{};
    // workload (runner.cpp:103-133)
    const Node* w = config.get("workload");
    if (!w || w->null()) config_error("config requires a 'workload' section");
    if (strict && w->map()) {
        static const std::set<std::string> allowed = {"mode", "trace", "rate_rps", "n_requests", "acceptance_rate",
                                                      "preset", "gen_seed", "prompt_median", "prompt_sigma",
                                                      "output_median", "output_sigma"};
        for (const auto& f : w->fields)
            if (!allowed.count(f.first)) config_error("unknown key '" + f.first + "' in workload");
    }
    const std::string mode = w->string_or("mode", "trace");
    const int64_t n_drafts = static_cast<int64_t>(topo.drafts.size());
    rc.gen_seed = rc.seed;
    if (mode == "trace") {
        std::string path = w->string_or("trace", "");
        if (path.empty()) config_error("workload.mode=trace requires workload.trace");
        path = join_path(base_dir, path);
        rc.trace = cached(caches, &Caches::traces, file_key(path), [&] { return load_trace_file(path); });
        s.workload = DSD_WORKLOAD_TRACE;
    } else if (mode == "poisson") {
        double rate = w->double_or("rate_rps", 0.0);
        if (!(rate > 0.0)) config_error("workload.mode=poisson requires rate_rps > 0");
        if (w->has("trace")) {
            const std::string path = join_path(base_dir, w->string_or("trace", ""));
            rc.trace = cached(caches, &Caches::traces, file_key(path), [&] { return load_trace_file(path); });
            s.workload = DSD_WORKLOAD_TRACE_POISSON;
            s.rate_rps = rate;
        } else {
            s.workload = DSD_WORKLOAD_SYNTHETIC;
            s.rate_rps = rate;
            s.n_requests = w->int_or("n_requests", 0);
            s.acceptance_rate = w->double_or("acceptance_rate", 0.8);
            // LengthDist defaults / presets (trace.hpp:46-53, trace.cpp:125-143)
            double pm = 60.0, ps = 0.4, om = 90.0, os = 0.35;
            if (w->has("preset")) {
                const std::string p = w->string_or("preset", "");
                if (p == "gsm8k-like") { pm = 60.0; ps = 0.4; om = 90.0; os = 0.35; }
                else if (p == "cnndm-like") { pm = 600.0; ps = 0.5; om = 180.0; os = 0.4; }
                else if (p == "humaneval-like") { pm = 130.0; ps = 0.4; om = 160.0; os = 0.5; }
                else config_error("unknown length preset '" + p +
                                  "' (expected gsm8k-like, cnndm-like or humaneval-like)");
            }
            s.prompt_median = w->double_or("prompt_median", pm);
            s.prompt_sigma = w->double_or("prompt_sigma", ps);
            s.output_median = w->double_or("output_median", om);
            s.output_sigma = w->double_or("output_sigma", os);
            s.prompt_cap = 4096;
            s.output_cap = 2048;
            s.gen_n_drafts = std::max<int64_t>(1, n_drafts);
            rc.gen_seed = static_cast<uint64_t>(w->int_or("gen_seed", static_cast<int64_t>(rc.seed)));
            const Node* gs = w->get("gen_seed");
            rc.gen_seed_fixed = gs && !gs->null();
            // generate_synthetic preconditions (trace.cpp:146-153)
            if (!(s.acceptance_rate >= 0.0 && s.acceptance_rate <= 1.0))
                config_error("acceptance rate must lie in [0, 1]");
            if (!(s.rate_rps > 0.0) || !std::isfinite(s.rate_rps))
                config_error("poisson rate must be finite and positive");
            if (s.n_requests < 0) config_error("n_requests must be >= 0");
        }
    } else {
        config_error("workload.mode must be 'trace' or 'poisson'");
    }

    // expanded topology -> arrays
    s.n_targets = static_cast<int32_t>(topo.targets.size());
    s.n_drafts = static_cast<int32_t>(topo.drafts.size());
    s.n_target_groups = topo.n_tg;
    s.n_draft_groups = std::max(1, topo.n_dg);
    for (const auto& d : topo.targets) rc.tgroup.push_back(d.group);
    for (const auto& d : topo.drafts) rc.dgroup.push_back(d.group);
    rc.links.assign(static_cast<size_t>(s.n_draft_groups) * s.n_target_groups, topo.def);
    for (const auto& kv : topo.overrides)
        rc.links[static_cast<size_t>(kv.first.first) * s.n_target_groups + kv.first.second] = kv.second;
    const bool fused_everything = pol.window == DSD_WINDOW_FUSED || topo.drafts.empty();
    // Engine::Impl ctor (engine.cpp:170-189)
    for (const auto& d : topo.targets) {
        int pre = rc.profile->find(d.model, d.hardware, 0), dec = rc.profile->find(d.model, d.hardware, 1);
        if (pre < 0 || dec < 0)
            config_error("no latency profile for target (" + d.model + ", " + d.hardware + ")");
        rc.tgrids.push_back(pre);
        rc.tgrids.push_back(dec);
    }
    for (const auto& d : topo.drafts) {
        int pre = rc.profile->find(d.model, d.hardware, 0), dec = rc.profile->find(d.model, d.hardware, 1);
        if (!fused_everything && (pre < 0 || dec < 0))
            config_error("no latency profile for draft (" + d.model + ", " + d.hardware + ")");
        rc.dgrids.push_back(pre);
        rc.dgrids.push_back(dec);
    }
    if (!topo.drafts.empty() && rc.trace) {
        const TraceData& t = *rc.trace;
        for (size_t i = 0; i < t.drafter.size(); ++i)
            if (t.drafter[i] >= n_drafts)
                config_error("trace record " + std::to_string(i) + ": field 'drafter_id' " +
                             std::to_string(t.drafter[i]) + " out of range for draft pool of size " +
                             std::to_string(n_drafts));
    }
    s.routing = pol.routing;
    s.batching = pol.batching;
    s.max_batch_size = pol.max_batch;
    s.draft_max_batch = pol.draft_max_batch;
    s.batching_window_us = pol.window_us;
    s.similarity_fraction = pol.sim_frac;
    s.window_kind = pol.window;
    s.gamma = pol.gamma;
    s.gamma_min = pol.gamma_min;
    s.gamma_max = pol.gamma_max;
    s.queue_capacity = pol.queue_capacity;
    rc.bind();
    return rc;
}

}  // namespace dsd::host
