// runtime.hpp — host-side owner of one GPU's replica batches (no CUDA types
// leak out of this header, so host C++ translation units build with g++).
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsdsim.h"
#include "../host/uninit.hpp"

namespace dsd {

// Status-carrying error used across the host layer; code is DSD_ERR_CONFIG or
// DSD_ERR_RUNTIME (mirrors the reference's exception -> exit-code map,
// tools/specsim_main.cpp:293-311).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct RuntimeImpl;
struct DevicePool;  // host threads of a multi-device Runtime (multi.cpp)

// One GPU: packs a batch into its scenario blob + workspace and runs the
// staging and simulation kernels on its own stream (runtime.cu).
class DeviceRuntime {
public:
    explicit DeviceRuntime(int device);
    ~DeviceRuntime();
    DeviceRuntime(const DeviceRuntime&) = delete;
    DeviceRuntime& operator=(const DeviceRuntime&) = delete;

    // Packs + uploads scenarios and replicas and sizes the workspace.
    // feature_probe: accumulate the per-replica probe sums (probe()).
    void prepare(const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas,
                 size_t n, bool collect_records, bool feature_probe = false, bool event_log = false);
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
    // After a run with event_log: the replica's log_transition records and
    // busy intervals in event order (ElogRec / BusyRec, layout.cuh).
    void fetch_event_log(size_t replica, std::vector<char>* elog, std::vector<char>* busy);
    void* stream();
    int device() const;
    int64_t last_launch_count() const;
    void last_kernel_ms(double* sim_ms, double* gen_ms, double* total_ms);
    size_t replica_count() const;
    void transfer_bytes(int64_t* h2d, int64_t* d2h) const;

private:
    std::unique_ptr<RuntimeImpl> impl_;
};

// The engine behind a dsd_handle: one or more GPUs driven from one host
// thread (multi.cpp).  A batch's replicas are dealt across the devices in
// cost order (shard_of_replicas) and every call below keeps the
// caller's replica numbering: summaries, records and probe sums come back in
// the order the replicas were given.  With one device it is a thin
// forwarder to its DeviceRuntime.
class Runtime {
public:
    explicit Runtime(int device);
    explicit Runtime(const std::vector<int>& devices);
    ~Runtime();
    Runtime(const Runtime&) = delete;
    Runtime& operator=(const Runtime&) = delete;

    void prepare(const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas,
                 size_t n, bool collect_records, bool feature_probe = false, bool event_log = false);
    void launch();
    void sync();
    void summaries(dsd_replica_summary* out, size_t n);
    const dsd_replica_summary* host_summaries();
    void fetch_records(size_t replica, dsd_request_record* records, size_t cap, int64_t* n_records,
                       int32_t* gamma_seq, int32_t* committed_seq, size_t seq_cap, int64_t* n_seq,
                       int64_t* busy_us, size_t busy_cap);
    // single-device handles only (the benchmark's NCCL gather reads it)
    void device_summaries(void** ptr, size_t* bytes);
    void probe(double* out, size_t n);
    void fetch_event_log(size_t replica, std::vector<char>* elog, std::vector<char>* busy);
    void* stream();  // device 0's stream
    int64_t last_launch_count() const;        // summed over the devices
    void last_kernel_ms(double* sim_ms, double* gen_ms, double* total_ms);  // max over the devices
    size_t replica_count() const;
    void transfer_bytes(int64_t* h2d, int64_t* d2h) const;  // summed
    size_t device_count() const { return devs_.size(); }
    int device(size_t k) const { return devs_[k]->device(); }
    // replicas of the prepared batch per device
    std::vector<size_t> shard_sizes() const;

private:
    template <class F>
    void each_device(F&& fn);
    std::vector<std::unique_ptr<DeviceRuntime>> devs_;
    std::unique_ptr<DevicePool> pool_;  // host threads of devices 1.. (none for one device)
    // prepared batch: replica -> (device, index on it); per device its replicas' global indices
    std::vector<int32_t> dev_of_;
    std::vector<uint32_t> local_of_;
    std::vector<std::vector<uint32_t>> global_of_;
    std::vector<std::vector<dsd_replica>> mine_;  // each device's replicas (storage kept across batches)
    host::uvector<dsd_replica_summary> gathered_;  // (no zero fill: every element is written)
    bool gathered_valid_ = false;
    size_t n_ = 0;
};

// Estimated cost (simulated events) of one replica of a scenario: N x (4 +
// 5 x median output / E[tokens per round]) for a synthetic workload with a
// static window (E = (1 - a^(g+1)) / (1 - a)), N x (4 + 5 x mean output)
// otherwise.  Only orders replicas; results never depend on it.
double replica_cost_estimate(const dsd_scenario& s);
// Shard of each replica when n replicas are spread over n_shards devices:
// replicas sorted by decreasing cost (ties: lower index first) are dealt in
// snake order 0..N-1, N-1..0, ..., so every shard gets the same count (+-1)
// and a near-equal share of the heavy replicas.
std::vector<int32_t> shard_of_replicas(const dsd_scenario* scenarios, const dsd_replica* replicas, size_t n,
                                       int n_shards);

}  // namespace dsd
