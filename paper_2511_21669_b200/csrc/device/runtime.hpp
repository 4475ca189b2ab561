// runtime.hpp — host-side owner of one GPU's replica batches (no CUDA types
// leak out of this header, so host C++ translation units build with g++).
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsdsim.h"

namespace dsd {

// Status-carrying error used across the host layer; code is DSD_ERR_CONFIG or
// DSD_ERR_RUNTIME (mirrors the reference's exception -> exit-code map,
// tools/specsim_main.cpp:293-311).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct RuntimeImpl;

class Runtime {
public:
    explicit Runtime(int device);
    ~Runtime();
    Runtime(const Runtime&) = delete;
    Runtime& operator=(const Runtime&) = delete;

    // Packs + uploads scenarios and replicas and sizes the workspace.
    // feature_probe: accumulate the per-replica probe sums (probe()).
    void prepare(const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas,
                 size_t n, bool collect_records, bool feature_probe = false);
    // Enqueues the staging + simulation kernels on the handle's stream.
    void launch();
    void sync();
    void summaries(dsd_replica_summary* out, size_t n);
    // The batch's summaries in a page-locked buffer the Runtime owns (valid
    // until the next call; no host allocation per batch).
    const dsd_replica_summary* host_summaries();
    void fetch_records(size_t replica, dsd_request_record* records, size_t cap, int64_t* n_records,
                       int32_t* gamma_seq, int32_t* committed_seq, size_t seq_cap, int64_t* n_seq,
                       int64_t* busy_us, size_t busy_cap);
    void device_summaries(void** ptr, size_t* bytes);
    // After a probed run: [n][kProbeFields] sums per replica (see Workspace::probe).
    void probe(double* out, size_t n);
    void* stream();
    int64_t last_launch_count() const;
    void last_kernel_ms(double* sim_ms, double* gen_ms, double* total_ms);
    size_t replica_count() const;
    void transfer_bytes(int64_t* h2d, int64_t* d2h) const;

private:
    std::unique_ptr<RuntimeImpl> impl_;
};

}  // namespace dsd
