// capi.cpp — extern "C" boundary (include/dsdsim.h).  Every entry point
// converts dsd::Error / std::exception into a status code + message, so no
// exception crosses the ABI.
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../device/runtime.hpp"
#include "dsdsim.h"
#include "report.hpp"
#include "resolve.hpp"
#include "dataset.hpp"
#include "sweep.hpp"

struct dsd_handle {
    std::unique_ptr<dsd::Runtime> rt;
    dsd::host::Caches caches;
    std::unique_ptr<dsd::host::SweepBatch> prepared_sweep;
    // frees the last dsd_run_sweep's host batch off the caller's path
    std::thread reaper;
    ~dsd_handle() {
        if (reaper.joinable()) reaper.join();
    }
};

namespace {

void put_err(char* err, size_t errlen, const std::string& m) {
    if (!err || errlen == 0) return;
    size_t k = std::min(errlen - 1, m.size());
    std::memcpy(err, m.data(), k);
    err[k] = '\0';
}

template <typename F>
int guard(char* err, size_t errlen, F&& f) {
    try {
        f();
        if (err && errlen) err[0] = '\0';
        return DSD_OK;
    } catch (const dsd::Error& e) {
        put_err(err, errlen, e.what());
        return e.code;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return DSD_ERR_RUNTIME;
    }
}

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = '\0';
    return p;
}

void need(dsd_handle* h) {
    if (!h || !h->rt) throw dsd::Error(DSD_ERR_RUNTIME, "null dsd handle");
}

}  // namespace

extern "C" {

int dsd_abi_version(void) { return DSD_ABI_VERSION; }

void dsd_free(void* p) { std::free(p); }

int dsd_create(int device_ordinal, dsd_handle** out, char* err, size_t errlen) {
    return dsd_create_devices(&device_ordinal, 1, out, err, errlen);
}

int dsd_create_devices(const int* device_ordinals, int n_devices, dsd_handle** out, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        if (!out) throw dsd::Error(DSD_ERR_RUNTIME, "null output handle");
        if (n_devices < 1 || !device_ordinals) throw dsd::Error(DSD_ERR_RUNTIME, "empty device list");
        auto h = std::make_unique<dsd_handle>();
        h->rt = std::make_unique<dsd::Runtime>(std::vector<int>(device_ordinals, device_ordinals + n_devices));
        *out = h.release();
    });
}

int dsd_device_count(dsd_handle* h) { return (h && h->rt) ? static_cast<int>(h->rt->device_count()) : 0; }

int dsd_batch_shard_sizes(dsd_handle* h, int64_t* sizes, int cap) {
    if (!h || !h->rt) return 0;
    const std::vector<size_t> s = h->rt->shard_sizes();
    for (size_t k = 0; k < s.size() && static_cast<int>(k) < cap; ++k) sizes[k] = static_cast<int64_t>(s[k]);
    return static_cast<int>(s.size());
}

void dsd_destroy(dsd_handle* h) { delete h; }

int dsd_run_batch(dsd_handle* h, const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas,
                  size_t n, const dsd_run_opts* opts, dsd_replica_summary* summaries, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        h->rt->prepare(scenarios, n_scenarios, replicas, n, opts && opts->collect_records, opts && opts->feature_probe,
                       opts && opts->collect_event_log);
        h->rt->launch();
        h->rt->sync();
        if (summaries && n) h->rt->summaries(summaries, n);
    });
}

int dsd_fetch_records(dsd_handle* h, size_t replica, dsd_request_record* records, size_t records_cap,
                      int64_t* n_records, int32_t* gamma_seq, int32_t* committed_seq, size_t seq_cap, int64_t* n_seq,
                      int64_t* busy_us, size_t busy_cap, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        h->rt->fetch_records(replica, records, records_cap, n_records, gamma_seq, committed_seq, seq_cap, n_seq,
                             busy_us, busy_cap);
    });
}

int dsd_batch_prepare(dsd_handle* h, const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas,
                      size_t n, const dsd_run_opts* opts, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        h->rt->prepare(scenarios, n_scenarios, replicas, n, opts && opts->collect_records, opts && opts->feature_probe,
                       opts && opts->collect_event_log);
    });
}

int dsd_batch_launch(dsd_handle* h, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        h->rt->launch();
    });
}

int dsd_batch_sync(dsd_handle* h, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        h->rt->sync();
    });
}

int dsd_batch_summaries(dsd_handle* h, dsd_replica_summary* summaries, size_t n, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        h->rt->summaries(summaries, n);
    });
}

int dsd_batch_device_summaries(dsd_handle* h, void** dev_ptr, size_t* bytes) {
    if (!h || !h->rt || !dev_ptr || !bytes || h->rt->device_count() != 1) return DSD_ERR_RUNTIME;
    h->rt->device_summaries(dev_ptr, bytes);
    return DSD_OK;
}

void* dsd_stream(dsd_handle* h) { return (h && h->rt) ? h->rt->stream() : nullptr; }

int64_t dsd_last_launch_count(dsd_handle* h) { return (h && h->rt) ? h->rt->last_launch_count() : 0; }

int dsd_last_kernel_ms(dsd_handle* h, double* sim_kernel_ms, double* gen_kernel_ms, double* total_ms) {
    char err[8];
    return guard(err, sizeof(err), [&] {
        need(h);
        h->rt->last_kernel_ms(sim_kernel_ms, gen_kernel_ms, total_ms);
    });
}

int dsd_last_transfer_bytes(dsd_handle* h, int64_t* h2d_bytes, int64_t* d2h_bytes) {
    if (!h || !h->rt) return DSD_ERR_RUNTIME;
    h->rt->transfer_bytes(h2d_bytes, d2h_bytes);
    return DSD_OK;
}

int dsd_run_simulation(dsd_handle* h, const char* config_yaml, const char* base_dir, int strict, int has_seed,
                       uint64_t seed, char** report_json, char** report_csv, uint64_t* events_processed,
                       int64_t* end_time_us, double* agg, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        dsd::cfg::Node config = dsd::cfg::parse(config_yaml ? config_yaml : "");
        dsd::host::Resolved rc =
            dsd::host::resolve_config(config, strict != 0, has_seed ? std::optional<uint64_t>(seed) : std::nullopt,
                                      base_dir ? base_dir : ".", &h->caches);
        dsd_replica rep{};
        rep.scenario = 0;
        rep.seed = rc.seed;
        rep.gen_seed = rc.gen_seed;
        const bool need_records = report_json || report_csv;
        h->rt->prepare(&rc.scen, 1, &rep, 1, need_records);
        h->rt->launch();
        h->rt->sync();
        dsd::host::ReplicaOutput out;
        h->rt->summaries(&out.summary, 1);
        if (out.summary.status != DSD_OK)
            throw dsd::Error(DSD_ERR_RUNTIME, "engine capacity exceeded on the device (event heap / sequence arena)");
        if (need_records) {
            int64_t nrec = 0, nseq = 0;
            h->rt->fetch_records(0, nullptr, 0, &nrec, nullptr, nullptr, 0, &nseq, nullptr, 0);
            out.records.resize(static_cast<size_t>(nrec));
            out.gamma_seq.resize(static_cast<size_t>(nseq));
            out.committed_seq.resize(static_cast<size_t>(nseq));
            out.busy_us.resize(static_cast<size_t>(rc.scen.n_targets));
            h->rt->fetch_records(0, out.records.data(), out.records.size(), &nrec, out.gamma_seq.data(),
                                 out.committed_seq.data(), out.gamma_seq.size(), &nseq, out.busy_us.data(),
                                 out.busy_us.size());
            if (report_json) *report_json = dup(dsd::host::emit_report(out, rc.scen.n_targets, rc.digest, rc.seed));
            if (report_csv) *report_csv = dup(dsd::host::emit_report_csv(out));
        }
        if (events_processed) *events_processed = out.summary.events_processed;
        if (end_time_us) *end_time_us = out.summary.end_time_us;
        if (agg) {
            agg[0] = static_cast<double>(out.summary.completed);
            agg[1] = out.summary.throughput_rps;
            agg[2] = out.summary.mean_ttft_ms;
            agg[3] = out.summary.mean_tpot_ms;
        }
    });
}

static void event_log_out(dsd::Runtime& rt, size_t replica, char** event_log, dsd_busy_interval* intervals,
                          size_t cap, int64_t* n_intervals) {
    std::vector<char> el, bi;
    rt.fetch_event_log(replica, event_log ? &el : nullptr, (intervals || n_intervals) ? &bi : nullptr);
    if (event_log) *event_log = dup(dsd::host::render_event_log(el));
    if (intervals || n_intervals) {
        const std::vector<dsd_busy_interval> iv = dsd::host::decode_busy_intervals(bi);
        for (size_t k = 0; intervals && k < iv.size() && k < cap; ++k) intervals[k] = iv[k];
        if (n_intervals) *n_intervals = static_cast<int64_t>(iv.size());
    }
}

int dsd_fetch_event_log(dsd_handle* h, size_t replica, char** event_log, dsd_busy_interval* intervals, size_t cap,
                        int64_t* n_intervals, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        event_log_out(*h->rt, replica, event_log, intervals, cap, n_intervals);
    });
}

int dsd_run_simulation_traced(dsd_handle* h, const char* config_yaml, const char* base_dir, int strict, int has_seed,
                              uint64_t seed, char** report_json, char** event_log, dsd_busy_interval* intervals,
                              size_t cap, int64_t* n_intervals, uint64_t* events_processed, char* err,
                              size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        dsd::cfg::Node config = dsd::cfg::parse(config_yaml ? config_yaml : "");
        dsd::host::Resolved rc =
            dsd::host::resolve_config(config, strict != 0, has_seed ? std::optional<uint64_t>(seed) : std::nullopt,
                                      base_dir ? base_dir : ".", &h->caches);
        dsd_replica rep{};
        rep.seed = rc.seed;
        rep.gen_seed = rc.gen_seed;
        h->rt->prepare(&rc.scen, 1, &rep, 1, true, false, true);
        h->rt->launch();
        h->rt->sync();
        dsd::host::ReplicaOutput out;
        h->rt->summaries(&out.summary, 1);
        if (out.summary.status != DSD_OK)
            throw dsd::Error(DSD_ERR_RUNTIME, "engine capacity exceeded on the device (event heap / sequence arena)");
        if (report_json) {
            int64_t nrec = 0, nseq = 0;
            h->rt->fetch_records(0, nullptr, 0, &nrec, nullptr, nullptr, 0, &nseq, nullptr, 0);
            out.records.resize(static_cast<size_t>(nrec));
            out.gamma_seq.resize(static_cast<size_t>(nseq));
            out.committed_seq.resize(static_cast<size_t>(nseq));
            out.busy_us.resize(static_cast<size_t>(rc.scen.n_targets));
            h->rt->fetch_records(0, out.records.data(), out.records.size(), &nrec, out.gamma_seq.data(),
                                 out.committed_seq.data(), out.gamma_seq.size(), &nseq, out.busy_us.data(),
                                 out.busy_us.size());
            *report_json = dup(dsd::host::emit_report(out, rc.scen.n_targets, rc.digest, rc.seed));
        }
        event_log_out(*h->rt, 0, event_log, intervals, cap, n_intervals);
        if (events_processed) *events_processed = out.summary.events_processed;
    });
}

int dsd_run_sweep(dsd_handle* h, const char* sweep_yaml, const char* base_dir, const char* out_dir,
                  char** summary_json, char** summary_csv, double* totals, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        dsd::host::PhaseTimer tm("dsd_run_sweep");
        dsd::cfg::Node node = dsd::cfg::parse(sweep_yaml ? sweep_yaml : "");
        const std::string bdir = base_dir ? base_dir : ".";
        const std::string odir = out_dir ? out_dir : "";
        dsd::host::SweepSpec spec = dsd::host::SweepSpec::from_node(node, bdir);
        tm.lap("parse");
        dsd::host::SummaryParts parts;
        const bool text = summary_json || summary_csv;
        auto b = std::make_unique<dsd::host::SweepBatch>(dsd::host::plan_range(spec, 0, spec.point_count(), &h->caches));
        tm.lap("plan");
        const dsd::host::SweepTotals t = dsd::host::run_sweep(*h->rt, *b, odir, text ? &parts : nullptr);
        tm.lap("run");
        if (text) {
            std::string js, cs;
            dsd::host::assemble_summaries(parts, b->points, summary_json ? &js : nullptr,
                                          summary_csv ? &cs : nullptr);
            if (summary_json) *summary_json = dup(js);
            if (summary_csv) *summary_csv = dup(cs);
        }
        tm.lap("summary");
        // tens of thousands of small host objects: release them on a helper
        // thread (joined by the next call or dsd_destroy)
        if (h->reaper.joinable()) h->reaper.join();
        h->reaper = std::thread([bb = std::move(b),
                                 pp = std::make_unique<dsd::host::SummaryParts>(std::move(parts))]() mutable {
            bb.reset();
            pp.reset();
        });
        if (totals) {
            totals[0] = t.points;
            totals[1] = t.replicas;
            totals[2] = t.failed;
            totals[3] = t.events;
        }
    });
}

int dsd_prepare_sweep(dsd_handle* h, const char* sweep_yaml, const char* base_dir, int shard, int n_shards,
                      int64_t* n_replicas, int64_t* n_points, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        if (n_shards < 1 || shard < 0 || shard >= n_shards) throw dsd::Error(DSD_ERR_CONFIG, "bad shard index");
        dsd::cfg::Node node = dsd::cfg::parse(sweep_yaml ? sweep_yaml : "");
        auto b = std::make_unique<dsd::host::SweepBatch>(
            dsd::host::plan_sweep(node, base_dir ? base_dir : ".", shard, n_shards, &h->caches));
        h->rt->prepare(b->scenarios.data(), b->scenarios.size(), b->replicas.data(), b->replicas.size(), false);
        if (n_replicas) *n_replicas = static_cast<int64_t>(b->replicas.size());
        if (n_points) *n_points = static_cast<int64_t>(b->points.size());
        h->prepared_sweep = std::move(b);
    });
}

struct dsd_resolved {
    dsd::host::Resolved rc;
};

int dsd_resolve_config(const char* config_yaml, const char* base_dir, int strict, int has_seed, uint64_t seed,
                       dsd_resolved** out, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        dsd::cfg::Node config = dsd::cfg::parse(config_yaml ? config_yaml : "");
        auto r = std::make_unique<dsd_resolved>();
        r->rc = dsd::host::resolve_config(config, strict != 0, has_seed ? std::optional<uint64_t>(seed) : std::nullopt,
                                          base_dir ? base_dir : ".", nullptr);
        r->rc.bind();
        *out = r.release();
    });
}

const dsd_scenario* dsd_resolved_scenario(const dsd_resolved* r) { return &r->rc.scen; }

void dsd_resolved_replica(const dsd_resolved* r, dsd_replica* out) {
    *out = dsd_replica{};
    out->seed = r->rc.seed;
    out->gen_seed = r->rc.gen_seed;
}

const char* dsd_resolved_digest(const dsd_resolved* r) { return r->rc.digest.c_str(); }

void dsd_resolved_free(dsd_resolved* r) { delete r; }

struct dsd_sweep_plan {
    dsd::host::SweepBatch b;
};

int dsd_plan_sweep(const char* sweep_yaml, const char* base_dir, int shard, int n_shards, dsd_sweep_plan** out,
                   char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        if (n_shards < 1 || shard < 0 || shard >= n_shards) throw dsd::Error(DSD_ERR_CONFIG, "bad shard index");
        dsd::cfg::Node node = dsd::cfg::parse(sweep_yaml ? sweep_yaml : "");
        auto p = std::make_unique<dsd_sweep_plan>();
        dsd::host::Caches caches;  // profiles / traces / models shared by the sweep's points
        p->b = dsd::host::plan_sweep(node, base_dir ? base_dir : ".", shard, n_shards, &caches);
        for (size_t k = 0; k < p->b.resolved.size(); ++k) {
            p->b.resolved[k].bind();
            p->b.scenarios[k] = p->b.resolved[k].scen;
        }
        *out = p.release();
    });
}

size_t dsd_sweep_plan_scenarios(const dsd_sweep_plan* p, const dsd_scenario** scenarios) {
    if (scenarios) *scenarios = p->b.scenarios.data();
    return p->b.scenarios.size();
}

size_t dsd_sweep_plan_replicas(const dsd_sweep_plan* p, const dsd_replica** replicas) {
    if (replicas) *replicas = p->b.replicas.data();
    return p->b.replicas.size();
}

size_t dsd_sweep_plan_origin(const dsd_sweep_plan* p, int64_t* point, int32_t* repetition, size_t cap) {
    const auto& o = p->b.replica_origin;
    for (size_t k = 0; k < o.size() && k < cap; ++k) {
        if (point) point[k] = o[k].first;
        if (repetition) repetition[k] = o[k].second;
    }
    return o.size();
}

void dsd_sweep_plan_free(dsd_sweep_plan* p) { delete p; }

int dsd_emit_report(const dsd_replica_summary* summary, const dsd_request_record* records, size_t n_records,
                    const int32_t* gamma_seq, const int32_t* committed_seq, size_t n_seq, const int64_t* busy_us,
                    int n_targets, const char* digest, uint64_t seed, char** report_json, char** report_csv) {
    char err[8];
    return guard(err, sizeof(err), [&] {
        dsd::host::ReplicaOutput o;
        o.summary = *summary;
        o.records.assign(records, records + n_records);
        if (n_seq) {
            o.gamma_seq.assign(gamma_seq, gamma_seq + n_seq);
            o.committed_seq.assign(committed_seq, committed_seq + n_seq);
        }
        o.busy_us.assign(busy_us, busy_us + n_targets);
        if (report_json) *report_json = dup(dsd::host::emit_report(o, n_targets, digest ? digest : "", seed));
        if (report_csv) *report_csv = dup(dsd::host::emit_report_csv(o));
    });
}

uint64_t dsd_sweep_point_seed(uint64_t base_seed, const char* point_id, int repetition) {
    return dsd::host::sweep_point_seed(base_seed, point_id ? point_id : "", repetition);
}


int dsd_batch_probe(dsd_handle* h, double* out, size_t n, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        if (!out && n) throw dsd::Error(DSD_ERR_RUNTIME, "null output buffer");
        h->rt->probe(out, n);
    });
}

int dsd_build_scenarios(const char* grid_yaml, char** scenarios_jsonl, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        dsd::cfg::Node node = dsd::cfg::parse(grid_yaml ? grid_yaml : "");
        auto sc = dsd::host::build_scenarios(dsd::host::DatasetGrid::from_node(node));
        if (scenarios_jsonl) *scenarios_jsonl = dup(dsd::host::serialize_scenarios(sc));
    });
}

int dsd_generate_dataset(dsd_handle* h, const char* grid_yaml, const double* weights, char** dataset_jsonl,
                         char** scenarios_jsonl, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        dsd::cfg::Node node = dsd::cfg::parse(grid_yaml ? grid_yaml : "");
        auto sc = dsd::host::build_scenarios(dsd::host::DatasetGrid::from_node(node));
        dsd::host::ObjectiveWeights w;
        if (weights) {
            w.w_tpot = weights[0];
            w.w_ttft = weights[1];
            w.w_throughput = weights[2];
        }
        auto sweeps = dsd::host::generate_dataset(*h->rt, sc, w, &h->caches);
        if (dataset_jsonl) *dataset_jsonl = dup(dsd::host::serialize_dataset(sweeps));
        if (scenarios_jsonl) *scenarios_jsonl = dup(dsd::host::serialize_scenarios(sc));
    });
}

int dsd_eval_policy(dsd_handle* h, const char* scenarios_jsonl, const char* split, const char* window_kind,
                    int gamma, const char* model_path, double* out, char* err, size_t errlen) {
    return guard(err, errlen, [&] {
        need(h);
        const std::string sp = split ? split : "all";
        std::vector<dsd::host::ScenarioSpec> selected;
        for (const auto& s : dsd::host::parse_scenarios(scenarios_jsonl ? scenarios_jsonl : ""))
            if (sp == "all" || s.split == sp) selected.push_back(s);
        if (selected.empty()) throw dsd::Error(DSD_ERR_CONFIG, "no scenarios with split '" + sp + "'");
        auto e = dsd::host::eval_policy_on_scenarios(*h->rt, selected, window_kind ? window_kind : "static", gamma,
                                                      model_path ? model_path : "", &h->caches);
        if (out) {
            out[0] = e.mean_throughput_rps;
            out[1] = e.mean_ttft_ms;
            out[2] = e.mean_tpot_ms;
            out[3] = e.mean_chosen_gamma;
        }
    });
}

}  // extern "C"
