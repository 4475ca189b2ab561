// report.hpp — deterministic report emission from device records:
// MetricsCollector::system (proj/src/metrics/metrics.cpp:130-170),
// finalize_request (:172-201), emit_report (:203-278), emit_report_csv
// (:280-302), with the JsonWriter formatting of proj/src/util/json_writer.cpp.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "dsdsim.h"

namespace dsd::host {

// Pretty JSON writer with the reference's byte layout (2-space indent,
// "key": value, empty containers inline).
class JsonOut {
public:
    JsonOut& open_object();
    JsonOut& close_object();
    JsonOut& open_array();
    JsonOut& close_array();
    JsonOut& key(const std::string& k);
    JsonOut& str(const std::string& s);
    JsonOut& i64(int64_t v);
    JsonOut& u64(uint64_t v);
    JsonOut& boolean(bool v);
    JsonOut& null();
    JsonOut& fixed(double v, int decimals);
    std::string take() { return std::move(out_); }

private:
    void pre_value();
    void newline();
    std::string out_;
    std::vector<int> counts_;
    bool after_key_ = false;
};

struct ReplicaOutput {
    dsd_replica_summary summary{};
    std::vector<dsd_request_record> records;  // request-id order
    std::vector<int32_t> gamma_seq, committed_seq;
    std::vector<int64_t> busy_us;  // per target
};

std::string emit_report(const ReplicaOutput& r, int n_targets, const std::string& digest, uint64_t seed);
std::string emit_report_csv(const ReplicaOutput& r);

// RunResult::event_log (engine.cpp:213-219) from the device's ElogRec
// records, one line each, newline-terminated (specsim_main.cpp:65-72).
std::string render_event_log(const std::vector<char>& elog_records);
// BusyRec records -> dsd_busy_interval (role, server id, start, end).
std::vector<dsd_busy_interval> decode_busy_intervals(const std::vector<char>& busy_records);

}  // namespace dsd::host
