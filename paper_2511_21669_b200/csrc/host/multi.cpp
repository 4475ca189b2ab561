// multi.cpp — Runtime: one dsd_handle driving one or more GPUs from one host
// thread (include/dsdsim.h dsd_create_devices).  The reference's run_sweep
// spreads a sweep's (point, repetition) jobs over a thread pool
// (proj/src/runner/sweep.cpp:109-160); here the replicas of a batch are
// dealt across the devices in cost order and each device runs its share as
// one batch, the shares running concurrently (one stream per device).  The
// per-replica summaries come back into one host array in the caller's
// replica order - the gather of SURVEY §8(e) done as per-device D2H copies
// into page-locked memory, since one process owns every device here.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <numeric>
#include <thread>

#include "../device/runtime.hpp"

namespace dsd {

double replica_cost_estimate(const dsd_scenario& s) {
    double n = 0.0, out = 0.0;
    if (s.workload == DSD_WORKLOAD_SYNTHETIC) {
        n = static_cast<double>(s.n_requests);
        out = s.output_median;
    } else if (s.trace) {
        n = static_cast<double>(s.trace->n);
        double sum = 0.0;
        for (int64_t i = 0; i < s.trace->n; ++i) sum += static_cast<double>(s.trace->output_length[i]);
        out = s.trace->n > 0 ? sum / static_cast<double>(s.trace->n) : 0.0;
    }
    double tau = 1.0;
    if (s.workload == DSD_WORKLOAD_SYNTHETIC && s.window_kind == DSD_WINDOW_STATIC && s.n_drafts > 0) {
        const double a = s.acceptance_rate, g = s.gamma;
        tau = a < 1.0 ? (1.0 - std::pow(a, g + 1.0)) / (1.0 - a) : g + 1.0;
    }
    return n * (4.0 + 5.0 * out / std::max(tau, 1e-9));
}

std::vector<int32_t> shard_of_replicas(const dsd_scenario* sc, const dsd_replica* reps, size_t n, int n_shards) {
    std::vector<int32_t> shard(n, 0);
    if (n_shards <= 1 || n == 0) return shard;
    // cost per distinct scenario; replicas by decreasing cost = the
    // scenarios sorted by cost, then a counting sort of the replicas by their
    // scenario's rank (replica order within a rank).  One pass over the
    // replicas gathers the scenario count, the per-scenario replica counts
    // and whether each scenario's replicas are contiguous (memory-bound at a
    // million replicas: every pass over them costs ~3 ms)
    uint32_t ns = 0;
    std::vector<size_t> cnt;
    bool grouped = true;
    for (size_t k = 0; k < n; ++k) {
        const uint32_t t = reps[k].scenario;
        if (t >= ns) {
            ns = t + 1;
            cnt.resize(ns, 0);
        }
        ++cnt[t];
        grouped = grouped && (k == 0 || t >= reps[k - 1].scenario);
    }
    std::vector<double> sc_cost(ns, 0.0);
    for (uint32_t s = 0; s < ns; ++s)
        if (cnt[s]) sc_cost[s] = replica_cost_estimate(sc[s]);
    std::vector<uint32_t> sorder(ns), srank(ns);
    std::iota(sorder.begin(), sorder.end(), 0u);
    std::stable_sort(sorder.begin(), sorder.end(), [&](uint32_t a, uint32_t b) { return sc_cost[a] > sc_cost[b]; });
    // the deal position of the i-th replica in cost order: 0..N-1, N-1..0, ...
    const int32_t N = n_shards;
    auto snake = [N](size_t i, int32_t& pos, int32_t& dir) {
        const size_t round = i / static_cast<size_t>(N);
        const int32_t p = static_cast<int32_t>(i % static_cast<size_t>(N));
        dir = round % 2 == 0 ? 1 : -1;
        pos = dir > 0 ? p : N - 1 - p;
    };
    auto step = [N](int32_t& pos, int32_t& dir) {
        pos += dir;
        if (pos == N || pos < 0) {
            dir = -dir;
            pos += dir;
        }
    };
    // Fast path - every scenario's replicas contiguous and in scenario order,
    // as plan_sweep lays them out: each scenario's run is dealt from its
    // offset in cost order with sequential writes (a million-replica batch:
    // ~19 -> ~2 ms)
    if (grouped) {
        std::vector<size_t> first(static_cast<size_t>(ns) + 1, 0);  // replicas of scenario s: [first[s], first[s+1])
        for (uint32_t t = 0; t < ns; ++t) first[t + 1] = first[t] + cnt[t];
        size_t base = 0;
        for (uint32_t i = 0; i < ns; ++i) {
            const uint32_t sc_i = sorder[i];
            const size_t lo = first[sc_i], hi = first[sc_i + 1];
            if (lo == hi) continue;
            int32_t pos, dir;
            snake(base, pos, dir);
            for (size_t k = lo; k < hi; ++k) {
                shard[k] = pos;
                step(pos, dir);
            }
            base += hi - lo;
        }
        return shard;
    }
    for (uint32_t i = 0; i < ns; ++i) srank[sorder[i]] = i;
    std::vector<size_t> start(static_cast<size_t>(ns) + 1, 0);
    for (size_t k = 0; k < n; ++k) ++start[srank[reps[k].scenario] + 1];
    for (uint32_t i = 0; i < ns; ++i) start[i + 1] += start[i];
    std::vector<uint32_t> order(n);
    for (size_t k = 0; k < n; ++k) order[start[srank[reps[k].scenario]]++] = static_cast<uint32_t>(k);
    int32_t pos = 0, dir = 1;
    for (size_t i = 0; i < n; ++i) {
        shard[order[i]] = pos;
        step(pos, dir);
    }
    return shard;
}

// One persistent host thread per extra device (device 0 runs on the caller):
// a thread that makes its first CUDA call attaches to the device's context,
// which cost ~0.3 ms per device and call when every call spawned threads.
// run(fn) calls fn(k) for every device concurrently and rethrows the first
// exception once all have finished.
struct DevicePool {
    explicit DevicePool(size_t n) : n_(n) {
        for (size_t k = 1; k < n; ++k)
            th_.emplace_back([this, k] {
                uint64_t seen = 0;
                for (;;) {
                    const std::function<void(size_t)>* task;
                    {
                        std::unique_lock<std::mutex> lk(m_);
                        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                        if (stop_) return;
                        seen = gen_;
                        task = task_;
                    }
                    call(*task, k);
                    std::lock_guard<std::mutex> lk(m_);
                    if (++done_ == n_ - 1) done_cv_.notify_all();
                }
            });
    }
    ~DevicePool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(const std::function<void(size_t)>& fn) {
        {
            std::lock_guard<std::mutex> lk(m_);
            task_ = &fn;
            done_ = 0;
            first_ = nullptr;
            ++gen_;
        }
        cv_.notify_all();
        call(fn, 0);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return done_ == n_ - 1; });
        if (first_) std::rethrow_exception(first_);
    }

  private:
    void call(const std::function<void(size_t)>& fn, size_t k) {
        try {
            fn(k);
        } catch (...) {
            std::lock_guard<std::mutex> lk(m_);
            if (!first_) first_ = std::current_exception();
        }
    }
    size_t n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t)>* task_ = nullptr;
    uint64_t gen_ = 0;
    size_t done_ = 0;
    bool stop_ = false;
    std::exception_ptr first_;
};

Runtime::Runtime(int device) { devs_.push_back(std::make_unique<DeviceRuntime>(device)); }

Runtime::Runtime(const std::vector<int>& devices) {
    if (devices.empty()) throw Error(DSD_ERR_RUNTIME, "empty device list");
    for (size_t i = 0; i < devices.size(); ++i)
        for (size_t j = 0; j < i; ++j)
            if (devices[i] == devices[j]) throw Error(DSD_ERR_RUNTIME, "device listed twice");
    for (int d : devices) devs_.push_back(std::make_unique<DeviceRuntime>(d));
    if (devs_.size() > 1) pool_ = std::make_unique<DevicePool>(devs_.size());
    mine_.resize(devs_.size());
}

Runtime::~Runtime() = default;

// fn(k) for every device, concurrently (the persistent pool)
template <class F>
void Runtime::each_device(F&& fn) {
    if (!pool_) {
        fn(size_t{0});
        return;
    }
    const std::function<void(size_t)> task = fn;
    pool_->run(task);
}

void Runtime::prepare(const dsd_scenario* sc, size_t ns, const dsd_replica* reps, size_t n, bool collect,
                      bool feature_probe, bool event_log) {
    n_ = n;
    gathered_valid_ = false;
    if (devs_.size() == 1) {
        devs_[0]->prepare(sc, ns, reps, n, collect, feature_probe, event_log);
        return;
    }
    const size_t D = devs_.size();
    dev_of_ = shard_of_replicas(sc, reps, n, static_cast<int>(D));
    local_of_.resize(n);
    global_of_.resize(D);
    // every device's thread picks its replicas out of the deal (one scan of
    // the shard ids each, in parallel; a million-replica batch took ~15 ms
    // as one serial pass of push_backs)
    each_device([&](size_t d) {
        std::vector<uint32_t>& g = global_of_[d];
        g.clear();
        g.reserve(n / D + 1);
        const int32_t di = static_cast<int32_t>(d);
        for (size_t k = 0; k < n; ++k)
            if (dev_of_[k] == di) {
                local_of_[k] = static_cast<uint32_t>(g.size());
                g.push_back(static_cast<uint32_t>(k));
            }
        std::vector<dsd_replica>& mine = mine_[d];
        mine.resize(g.size());
        for (size_t j = 0; j < mine.size(); ++j) mine[j] = reps[g[j]];
        devs_[d]->prepare(sc, ns, mine.data(), mine.size(), collect, feature_probe, event_log);
    });
}

void Runtime::launch() {
    gathered_valid_ = false;
    if (devs_.size() == 1) {
        devs_[0]->launch();
        return;
    }
    // launch() computes the lane placement on the host while k_stage runs:
    // one host thread per device keeps the devices' launches overlapped
    each_device([&](size_t d) { devs_[d]->launch(); });
}

void Runtime::sync() {
    for (auto& d : devs_) d->sync();
}

const dsd_replica_summary* Runtime::host_summaries() {
    if (devs_.size() == 1) return devs_[0]->host_summaries();
    if (!gathered_valid_) {
        if (gathered_.size() != n_) gathered_.resize(n_);  // (kept across batches: no re-zeroing)
        each_device([&](size_t d) {
            const dsd_replica_summary* s = devs_[d]->host_summaries();
            const std::vector<uint32_t>& g = global_of_[d];
            for (size_t j = 0; j < g.size(); ++j) gathered_[g[j]] = s[j];
        });
        gathered_valid_ = true;
    }
    return gathered_.data();
}

void Runtime::summaries(dsd_replica_summary* out, size_t n) {
    if (devs_.size() == 1) {
        devs_[0]->summaries(out, n);
        return;
    }
    if (n > n_) throw Error(DSD_ERR_RUNTIME, "summary buffer larger than the batch");
    const dsd_replica_summary* s = host_summaries();
    std::copy(s, s + n, out);
}

void Runtime::fetch_records(size_t replica, dsd_request_record* records, size_t cap, int64_t* n_records,
                            int32_t* gamma_seq, int32_t* committed_seq, size_t seq_cap, int64_t* n_seq,
                            int64_t* busy_us, size_t busy_cap) {
    if (devs_.size() == 1) {
        devs_[0]->fetch_records(replica, records, cap, n_records, gamma_seq, committed_seq, seq_cap, n_seq, busy_us,
                                busy_cap);
        return;
    }
    if (replica >= n_) throw Error(DSD_ERR_RUNTIME, "replica index out of range");
    devs_[static_cast<size_t>(dev_of_[replica])]->fetch_records(local_of_[replica], records, cap, n_records,
                                                                 gamma_seq, committed_seq, seq_cap, n_seq, busy_us,
                                                                 busy_cap);
}

void Runtime::device_summaries(void** ptr, size_t* bytes) {
    if (devs_.size() != 1) throw Error(DSD_ERR_RUNTIME, "device summaries of a multi-device handle");
    devs_[0]->device_summaries(ptr, bytes);
}

void Runtime::probe(double* out, size_t n) {
    if (devs_.size() == 1) {
        devs_[0]->probe(out, n);
        return;
    }
    if (n > n_) n = n_;
    std::vector<std::vector<double>> part(devs_.size());
    each_device([&](size_t d) {
        part[d].resize(global_of_[d].size() * DSD_PROBE_FIELDS);
        devs_[d]->probe(part[d].data(), global_of_[d].size());
    });
    for (size_t k = 0; k < n; ++k) {
        const double* src = part[static_cast<size_t>(dev_of_[k])].data() + static_cast<size_t>(local_of_[k]) * DSD_PROBE_FIELDS;
        std::copy(src, src + DSD_PROBE_FIELDS, out + k * DSD_PROBE_FIELDS);
    }
}

void Runtime::fetch_event_log(size_t replica, std::vector<char>* elog, std::vector<char>* busy) {
    if (devs_.size() == 1) {
        devs_[0]->fetch_event_log(replica, elog, busy);
        return;
    }
    if (replica >= n_) throw Error(DSD_ERR_RUNTIME, "replica index out of range");
    devs_[static_cast<size_t>(dev_of_[replica])]->fetch_event_log(local_of_[replica], elog, busy);
}

void* Runtime::stream() { return devs_[0]->stream(); }

int64_t Runtime::last_launch_count() const {
    int64_t s = 0;
    for (const auto& d : devs_) s += d->last_launch_count();
    return s;
}

void Runtime::last_kernel_ms(double* sim_ms, double* gen_ms, double* total_ms) {
    double a = 0, b = 0, c = 0;
    for (auto& d : devs_) {
        double x = 0, y = 0, z = 0;
        d->last_kernel_ms(&x, &y, &z);
        a = std::max(a, x);
        b = std::max(b, y);
        c = std::max(c, z);
    }
    if (sim_ms) *sim_ms = a;
    if (gen_ms) *gen_ms = b;
    if (total_ms) *total_ms = c;
}

size_t Runtime::replica_count() const { return n_; }

void Runtime::transfer_bytes(int64_t* h2d, int64_t* d2h) const {
    int64_t a = 0, b = 0;
    for (const auto& d : devs_) {
        int64_t x = 0, y = 0;
        d->transfer_bytes(&x, &y);
        a += x;
        b += y;
    }
    if (h2d) *h2d = a;
    if (d2h) *d2h = b;
}

std::vector<size_t> Runtime::shard_sizes() const {
    if (devs_.size() == 1) return {n_};
    std::vector<size_t> s;
    for (const auto& g : global_of_) s.push_back(g.size());
    return s;
}

}  // namespace dsd
