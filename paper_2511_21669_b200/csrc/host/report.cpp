// report.cpp — byte-identical report emission (see report.hpp for citations).
#include "report.hpp"

#include <cstring>

#include "../device/layout.cuh"

#include <algorithm>
#include <cmath>

#include "yaml.hpp"

namespace dsd::host {

void JsonOut::newline() {
    out_ += '\n';
    out_.append(2 * counts_.size(), ' ');
}

void JsonOut::pre_value() {
    if (after_key_) {
        after_key_ = false;
        return;
    }
    if (!counts_.empty()) {
        if (counts_.back()++ > 0) out_ += ',';
        newline();
    }
}

JsonOut& JsonOut::open_object() {
    pre_value();
    counts_.push_back(0);
    out_ += '{';
    return *this;
}

JsonOut& JsonOut::close_object() {
    bool items = counts_.back() > 0;
    counts_.pop_back();
    if (items) newline();
    out_ += '}';
    return *this;
}

JsonOut& JsonOut::open_array() {
    pre_value();
    counts_.push_back(0);
    out_ += '[';
    return *this;
}

JsonOut& JsonOut::close_array() {
    bool items = counts_.back() > 0;
    counts_.pop_back();
    if (items) newline();
    out_ += ']';
    return *this;
}

JsonOut& JsonOut::key(const std::string& k) {
    if (counts_.back()++ > 0) out_ += ',';
    newline();
    out_ += '"';
    cfg::json_escape(out_, k);
    out_ += "\": ";
    after_key_ = true;
    return *this;
}

JsonOut& JsonOut::str(const std::string& s) {
    pre_value();
    out_ += '"';
    cfg::json_escape(out_, s);
    out_ += '"';
    return *this;
}

JsonOut& JsonOut::i64(int64_t v) {
    pre_value();
    out_ += std::to_string(v);
    return *this;
}

JsonOut& JsonOut::u64(uint64_t v) {
    pre_value();
    out_ += std::to_string(v);
    return *this;
}

JsonOut& JsonOut::boolean(bool v) {
    pre_value();
    out_ += v ? "true" : "false";
    return *this;
}

JsonOut& JsonOut::null() {
    pre_value();
    out_ += "null";
    return *this;
}

JsonOut& JsonOut::fixed(double v, int decimals) {
    pre_value();
    out_ += cfg::fmt_fixed(v, decimals);
    return *this;
}

namespace {

double nearest_rank(std::vector<double> v, double q) {  // metrics.cpp:12-19
    std::sort(v.begin(), v.end());
    size_t rank = static_cast<size_t>(std::ceil(q * static_cast<double>(v.size())));
    if (rank == 0) rank = 1;
    return v[rank - 1];
}

struct Rec {
    const dsd_request_record* r;
    int64_t id;
    size_t seq_off;
    double ttft, e2e, tpot, ratio, arrival;
    bool has_tpot, has_ratio;
};

std::vector<Rec> finalize(const ReplicaOutput& out) {
    std::vector<Rec> recs;
    size_t off = 0;
    for (size_t i = 0; i < out.records.size(); ++i) {
        const dsd_request_record& r = out.records[i];
        const size_t my_off = off;
        off += static_cast<size_t>(r.n_iterations);
        if (r.completion_us < 0) continue;
        Rec x{};
        x.r = &r;
        x.id = static_cast<int64_t>(i);
        x.seq_off = my_off;
        x.arrival = static_cast<double>(r.arrival_us) / 1000.0;
        x.ttft = static_cast<double>(r.first_token_us - r.arrival_us) / 1000.0;
        x.e2e = static_cast<double>(r.completion_us - r.arrival_us) / 1000.0;
        x.has_tpot = r.output_length >= 2;
        if (x.has_tpot)
            x.tpot = (static_cast<double>(r.completion_us - r.first_token_us) / 1000.0) /
                     static_cast<double>(r.output_length - 1);
        x.has_ratio = r.proposed > 0;
        if (x.has_ratio) x.ratio = static_cast<double>(r.accepted) / static_cast<double>(r.proposed);
        recs.push_back(x);
    }
    return recs;
}

}  // namespace

std::string emit_report(const ReplicaOutput& out, int n_targets, const std::string& digest, uint64_t seed) {
    const std::vector<Rec> recs = finalize(out);
    const dsd_replica_summary& s = out.summary;
    JsonOut w;
    w.open_object();
    w.key("config_digest").str(digest);
    w.key("seed").u64(seed);
    w.key("system").open_object();
    const int64_t completed = static_cast<int64_t>(recs.size());
    w.key("completed").i64(completed);
    const bool has_dur = completed > 0 && s.last_completion_us > s.first_arrival_us;
    const int64_t dur = s.last_completion_us - s.first_arrival_us;
    w.key("duration_ms");
    if (has_dur) w.fixed(static_cast<double>(dur) / 1000.0, 3); else w.null();
    w.key("throughput_rps");
    if (has_dur) w.fixed(static_cast<double>(completed) / (static_cast<double>(dur) / 1e6), 6); else w.null();
    w.key("target_utilization").open_array();
    for (int t = 0; t < n_targets; ++t) {
        double u = 0.0;
        if (has_dur) {
            u = static_cast<double>(out.busy_us[static_cast<size_t>(t)]) / static_cast<double>(dur);
            u = std::clamp(u, 0.0, 1.0);
        }
        w.fixed(u, 6);
    }
    w.close_array();
    const double total_ms = static_cast<double>(s.net_queue_wait_total_us) / 1000.0;
    w.key("net_queue_delay_total_ms").fixed(total_ms, 3);
    w.key("net_queue_delay_mean_ms");
    if (s.net_queue_wait_count > 0) w.fixed(total_ms / static_cast<double>(s.net_queue_wait_count), 3); else w.null();
    std::vector<double> ttft, tpot, e2e;
    for (const Rec& r : recs) {
        ttft.push_back(r.ttft);
        e2e.push_back(r.e2e);
        if (r.has_tpot) tpot.push_back(r.tpot);
    }
    auto pct = [&](const char* name, const std::vector<double>& v) {
        w.key(name);
        if (v.empty()) {
            w.null();
            return;
        }
        w.open_object();
        w.key("p50").fixed(nearest_rank(v, 0.50), 3);
        w.key("p90").fixed(nearest_rank(v, 0.90), 3);
        w.key("p99").fixed(nearest_rank(v, 0.99), 3);
        w.close_object();
    };
    w.key("percentiles").open_object();
    pct("ttft_ms", ttft);
    pct("tpot_ms", tpot);
    pct("e2e_ms", e2e);
    w.close_object();
    w.close_object();
    w.key("requests").open_array();
    for (const Rec& x : recs) {
        const dsd_request_record& r = *x.r;
        w.open_object();
        w.key("request_id").u64(static_cast<uint64_t>(x.id));
        w.key("drafter_id").i64(r.drafter_id);
        w.key("target_id").i64(r.target_id);
        w.key("arrival_ms").fixed(x.arrival, 3);
        w.key("ttft_ms").fixed(x.ttft, 3);
        w.key("tpot_ms");
        if (x.has_tpot) w.fixed(x.tpot, 3); else w.null();
        w.key("e2e_latency_ms").fixed(x.e2e, 3);
        w.key("acceptance_ratio");
        if (x.has_ratio) w.fixed(x.ratio, 6); else w.null();
        w.key("prompt_length").i64(r.prompt_length);
        w.key("output_length").i64(r.output_length);
        w.key("gamma_sequence").open_array();
        for (int32_t k = 0; k < r.n_iterations; ++k) w.i64(out.gamma_seq[x.seq_off + static_cast<size_t>(k)]);
        w.close_array();
        w.key("committed_sequence").open_array();
        for (int32_t k = 0; k < r.n_iterations; ++k) w.i64(out.committed_seq[x.seq_off + static_cast<size_t>(k)]);
        w.close_array();
        w.close_object();
    }
    w.close_array();
    w.close_object();
    std::string s_out = w.take();
    s_out += '\n';
    return s_out;
}

std::string emit_report_csv(const ReplicaOutput& out) {
    const std::vector<Rec> recs = finalize(out);
    std::string o =
        "request_id,drafter_id,target_id,arrival_ms,ttft_ms,tpot_ms,e2e_latency_ms,"
        "acceptance_ratio,prompt_length,output_length,iterations\n";
    for (const Rec& x : recs) {
        const dsd_request_record& r = *x.r;
        o += std::to_string(x.id) + ',' + std::to_string(r.drafter_id) + ',' + std::to_string(r.target_id) + ',' +
             cfg::fmt_fixed(x.arrival, 3) + ',' + cfg::fmt_fixed(x.ttft, 3) + ',';
        if (x.has_tpot) o += cfg::fmt_fixed(x.tpot, 3);
        o += ',' + cfg::fmt_fixed(x.e2e, 3) + ',';
        if (x.has_ratio) o += cfg::fmt_fixed(x.ratio, 6);
        o += ',' + std::to_string(r.prompt_length) + ',' + std::to_string(r.output_length) + ',' +
             std::to_string(r.n_iterations) + '\n';
    }
    return o;
}

std::string render_event_log(const std::vector<char>& bytes) {
    // phase_name (engine.cpp:47-59) and the log_transition details
    static const char* phases[] = {"arrived", "routed", "queued_prefill", "speculating",
                                   "inflight_to_target", "verifying", "inflight_to_draft", "done"};
    static const char* details[] = {"routed", "speculating", "proposal_sent", "proposal_at_target", "verify_done",
                                    "done"};
    const size_t n = bytes.size() / sizeof(ElogRec);
    std::string out;
    out.reserve(n * 72);
    for (size_t k = 0; k < n; ++k) {
        ElogRec e;
        std::memcpy(&e, bytes.data() + k * sizeof(ElogRec), sizeof(e));
        out += "t_us=";
        out += std::to_string(e.t);
        out += " req=";
        out += std::to_string(e.req);
        out += " phase=";
        out += e.phase < 8 ? phases[e.phase] : "?";
        out += " server=d";
        out += std::to_string(e.draft);
        out += "/t";
        out += std::to_string(e.target);
        out += ' ';
        out += e.detail < 6 ? details[e.detail] : "?";
        out += '\n';
    }
    return out;
}

std::vector<dsd_busy_interval> decode_busy_intervals(const std::vector<char>& bytes) {
    const size_t n = bytes.size() / sizeof(BusyRec);
    std::vector<dsd_busy_interval> out(n);
    for (size_t k = 0; k < n; ++k) {
        BusyRec b;
        std::memcpy(&b, bytes.data() + k * sizeof(BusyRec), sizeof(b));
        out[k].role = b.server < 0 ? 1 : 0;
        out[k].server_id = b.server < 0 ? ~b.server : b.server;
        out[k].start_us = b.start;
        out[k].end_us = b.end;
    }
    return out;
}

}  // namespace dsd::host
