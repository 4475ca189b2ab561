// sweep.cpp — run_sweep on the GPU engine (see sweep.hpp).  Point
// materialisation, seeds, file names and summaries follow
// proj/src/runner/sweep.cpp:16-199; the per-(point, rep) worker loop
// (:112-150) becomes one device batch of replicas.
#include "sweep.hpp"

#include <algorithm>
#include <charconv>
#include <numeric>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <cstdlib>
#include <thread>
#include <unistd.h>
#include <mutex>
#include <memory>
#include <functional>
#include <exception>
#include <condition_variable>

#include "report.hpp"

namespace dsd::host {

using cfg::Node;

SweepSpec SweepSpec::from_node(const Node& node, const std::string& base_dir) {
    SweepSpec spec;
    spec.base_dir = base_dir;
    const Node* base = node.get("base");
    if (base && base->scalar()) {
        std::string path = base->to_string();
        if (!path.empty() && path.front() != '/' && !base_dir.empty() && base_dir != ".") path = base_dir + "/" + path;
        spec.base = cfg::parse_file(path);
    } else if (const Node* inl = node.get("config")) {
        spec.base = *inl;
    } else {
        throw Error(DSD_ERR_CONFIG, "sweep spec requires 'base' (path) or 'config' (inline)");
    }
    spec.base_seed = static_cast<uint64_t>(node.int_or("seed", 42));
    spec.repetitions = static_cast<int>(node.int_or("repetitions", 1));
    if (spec.repetitions < 1) throw Error(DSD_ERR_CONFIG, "sweep repetitions must be >= 1");
    if (const Node* axes = node.get("axes"); axes && axes->map()) {
        for (const auto& f : axes->fields) {
            if (!f.second.seq() || f.second.items.empty())
                throw Error(DSD_ERR_CONFIG, "sweep axis '" + f.first + "' must be a non-empty list");
            spec.axes.emplace_back(f.first, f.second.items);
        }
    }
    return spec;
}

size_t SweepSpec::point_count() const {
    size_t n = 1;
    for (const auto& a : axes) n *= a.second.size();
    return n;
}

uint64_t sweep_point_seed(uint64_t base_seed, const std::string& point_id, int repetition) {
    if (point_id == "base" && repetition == 0) return base_seed;
    return cfg::fnv1a64(point_id + "#rep=" + std::to_string(repetition), base_seed ^ 0x9e3779b97f4a7c15ULL);
}

// sweep_point_seed for every repetition of one point: FNV-1a is a left fold,
// so the point id is hashed once and each repetition continues from there.
static void point_seeds(uint64_t base_seed, const std::string& point_id, int reps, std::vector<uint64_t>& out) {
    out.resize(static_cast<size_t>(reps));
    const uint64_t h = cfg::fnv1a64(point_id, base_seed ^ 0x9e3779b97f4a7c15ULL);
    for (int r = 0; r < reps; ++r) {
        if (r == 0 && point_id == "base") {
            out[0] = base_seed;
            continue;
        }
        // fnv1a64("#rep=" + to_string(r), h) without building the string
        char buf[32] = {'#', 'r', 'e', 'p', '='};
        const auto end = std::to_chars(buf + 5, buf + sizeof(buf), r).ptr;
        uint64_t x = h;
        for (const char* c = buf; c < end; ++c) {
            x ^= static_cast<unsigned char>(*c);
            x *= 0x100000001b3ULL;
        }
        out[static_cast<size_t>(r)] = x;
    }
}

namespace {

std::string point_id_of(const std::vector<std::pair<std::string, std::string>>& assignment) {
    std::vector<std::string> parts;
    for (const auto& kv : assignment) parts.push_back(kv.first + "=" + kv.second);
    std::sort(parts.begin(), parts.end());
    std::string id;
    for (const auto& p : parts) {
        if (!id.empty()) id += ';';
        id += p;
    }
    return id.empty() ? "base" : id;
}

std::string sanitize_filename(const std::string& s) {
    std::string out;
    for (char c : s)
        out += (std::isalnum(static_cast<unsigned char>(c)) || c == '-' || c == '_' || c == '=') ? c : '_';
    return out.size() > 120 ? out.substr(0, 120) : out;
}

}  // namespace

// The base config with point idx's axis values set (sweep.cpp:95-108).
static Node point_config(const SweepSpec& spec, size_t idx) {
    Node config = spec.base;
    size_t rem = idx;
    for (size_t a = spec.axes.size(); a-- > 0;) {
        const auto& values = spec.axes[a].second;
        cfg::set_path(config, spec.axes[a].first, values[rem % values.size()]);
        rem /= values.size();
    }
    return config;
}

std::string point_digest(const SweepSpec& spec, size_t idx) {
    return cfg::hex16(cfg::fnv1a64(point_config(spec, idx).canonical()));
}

// Host threads for the per-point loops (DSD_HOST_THREADS overrides).
static unsigned host_threads() {
    unsigned t = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
    if (const char* e = std::getenv("DSD_HOST_THREADS")) t = static_cast<unsigned>(std::max(1, std::atoi(e)));
    return t;
}

// Process-wide host worker threads for parallel_chunks: creating ~16 threads
// costs a few hundred microseconds, several times per sweep.  One parallel
// region at a time (a concurrent caller, e.g. a second handle on another
// thread, spawns its own threads instead); recreated in a forked child.
// Each region's task, counters and first exception live in a Region that
// late-waking workers hold by shared_ptr, so they can never run a stale task.
class HostPool {
  public:
    static HostPool* get(unsigned workers) {
        static std::mutex mu;
        static HostPool* pool = nullptr;
        std::lock_guard<std::mutex> lk(mu);
        if (!pool || pool->pid_ != getpid() || pool->workers_ < workers)
            pool = new HostPool(workers);  // lives for the process (a replaced pool's threads stay parked)
        return pool;
    }
    // task(0..tasks-1) on the workers and the caller; false when busy
    bool try_run(size_t tasks, const std::function<void(size_t)>& task) {
        std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
        if (!busy) return false;
        auto r = std::make_shared<Region>();
        r->task = &task;
        r->total = tasks;
        {
            std::lock_guard<std::mutex> lk(m_);
            region_ = r;
            ++gen_;
        }
        cv_.notify_all();
        work(*r);
        std::unique_lock<std::mutex> lk(r->m);
        r->cv.wait(lk, [&] { return r->finished == r->total; });
        if (r->err) std::rethrow_exception(r->err);
        return true;
    }

  private:
    struct Region {
        const std::function<void(size_t)>* task = nullptr;
        size_t total = 0;
        std::atomic<size_t> next{0};
        std::mutex m;
        std::condition_variable cv;
        size_t finished = 0;
        std::exception_ptr err;
    };
    static void work(Region& r) {
        size_t did = 0;
        for (size_t i; (i = r.next.fetch_add(1)) < r.total; ++did) {
            try {
                (*r.task)(i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(r.m);
                if (!r.err) r.err = std::current_exception();
            }
        }
        if (did == 0) return;
        std::lock_guard<std::mutex> lk(r.m);
        r.finished += did;
        if (r.finished == r.total) r.cv.notify_all();
    }
    explicit HostPool(unsigned workers) : workers_(workers), pid_(getpid()) {
        for (unsigned w = 0; w < workers; ++w)
            std::thread([this] {
                uint64_t seen = 0;
                for (;;) {
                    std::shared_ptr<Region> r;
                    {
                        std::unique_lock<std::mutex> lk(m_);
                        cv_.wait(lk, [&] { return gen_ != seen; });
                        seen = gen_;
                        r = region_;
                    }
                    work(*r);
                }
            }).detach();
    }
    unsigned workers_;
    pid_t pid_;
    std::mutex busy_, m_;
    std::condition_variable cv_;
    uint64_t gen_ = 0;
    std::shared_ptr<Region> region_;
};

// fn(begin, end) over contiguous chunks of [0, n), at least `grain` items per
// chunk; the calling thread takes part.
template <class F>
static void parallel_chunks(size_t n, size_t grain, F&& fn) {
    const size_t t = std::min<size_t>(host_threads(), std::max<size_t>(1, n / std::max<size_t>(grain, 1)));
    if (t <= 1) {
        fn(size_t{0}, n);
        return;
    }
    const std::function<void(size_t)> chunk = [&fn, n, t](size_t i) { fn(n * i / t, n * (i + 1) / t); };
    if (HostPool::get(static_cast<unsigned>(t - 1))->try_run(t, chunk)) return;
    std::vector<std::thread> pool;
    pool.reserve(t - 1);
    for (size_t i = 1; i < t; ++i) pool.emplace_back([&chunk, i] { chunk(i); });
    chunk(0);
    for (auto& th : pool) th.join();
}

// Points [lo, hi) of b.spec (local index i = point lo + i) resolved into
// scenarios and the replicas of one shard.
static void plan_points(SweepBatch& b, size_t lo, size_t hi, int shard, int n_shards, Caches* caches) {
    PhaseTimer tm("plan_sweep");
    const SweepSpec& spec = b.spec;
    const size_t n_points = hi - lo;
    b.point_base = lo;
    b.points.resize(n_points);
    // every point is materialised and resolved once, in parallel: assignment
    // and id, the config, its scenario (the digest is only computed when
    // report files are written) and the seeds of its repetitions
    std::vector<Resolved> res(n_points);
    std::vector<char> ok(n_points, 0);
    std::vector<std::vector<uint64_t>> seeds(n_points);
    // the axis values' text, once; and the order of the point id's sorted
    // "key=value" parts, which does not depend on the values when the keys
    // are distinct (a key that prefixes another compares on '=' vs its next
    // character)
    const size_t na = spec.axes.size();
    std::vector<std::vector<std::string>> vtext(na);
    for (size_t a = 0; a < na; ++a)
        for (const Node& v : spec.axes[a].second) vtext[a].push_back(v.scalar() ? v.to_string() : v.canonical());
    std::vector<size_t> id_order(na);
    std::iota(id_order.begin(), id_order.end(), size_t{0});
    std::sort(id_order.begin(), id_order.end(),
              [&](size_t x, size_t y) { return spec.axes[x].first + "=" < spec.axes[y].first + "="; });
    bool keys_distinct = true;
    for (size_t k = 1; k < na; ++k)
        if (spec.axes[id_order[k]].first == spec.axes[id_order[k - 1]].first) keys_distinct = false;
    std::atomic<size_t> next{0};
    auto worker = [&](size_t, size_t) {
        for (;;) {
            size_t idx = next.fetch_add(1);
            if (idx >= n_points) return;
            SweepPoint& p = b.points[idx];
            size_t rem = lo + idx;
            auto& asg = p.assignment;
            asg.resize(na);
            for (size_t a = na; a-- > 0;) {
                const size_t nv = spec.axes[a].second.size();
                asg[a] = {spec.axes[a].first, vtext[a][rem % nv]};
                rem /= nv;
            }
            if (keys_distinct && na > 0) {
                std::string& id = p.point_id;
                for (size_t k = 0; k < na; ++k) {
                    if (k) id += ';';
                    id += asg[id_order[k]].first;
                    id += '=';
                    id += asg[id_order[k]].second;
                }
            } else {
                p.point_id = point_id_of(asg);
            }
            point_seeds(spec.base_seed, p.point_id, spec.repetitions, seeds[idx]);
            try {
                res[idx] = resolve_config(point_config(spec, lo + idx), true, seeds[idx][0], spec.base_dir, caches,
                                          /*want_digest=*/false);
                ok[idx] = 1;
            } catch (const std::exception& e) {
                p.failed = true;
                p.error = e.what();
            }
        }
    };
    // one work-stealing worker per thread (points differ in cost)
    parallel_chunks(n_points < 64 ? 1 : std::min<size_t>(n_points, host_threads()), 1, worker);
    tm.lap("points");
    // resolved scenarios in point order, then the replicas: global replica
    // g = scenario * repetitions + rep (point-major)
    b.point_scenario.assign(n_points, -1);
    size_t n_ok = 0;
    for (size_t idx = 0; idx < n_points; ++idx)
        if (ok[idx]) b.point_scenario[idx] = static_cast<int64_t>(n_ok++);
    const size_t R = static_cast<size_t>(spec.repetitions);
    const size_t n_rep = n_ok * R;
    b.resolved.resize(n_ok);
    b.scenarios.resize(n_ok);
    b.replicas.resize(n_rep);
    b.replica_origin.resize(n_rep);
    parallel_chunks(n_points, 256, [&](size_t lo, size_t hi) {
        for (size_t idx = lo; idx < hi; ++idx) {
            const int64_t s = b.point_scenario[idx];
            if (s < 0) continue;
            Resolved& r = b.resolved[static_cast<size_t>(s)];
            r = std::move(res[idx]);
            r.bind();
            b.scenarios[static_cast<size_t>(s)] = r.scen;
            for (size_t rep = 0; rep < R; ++rep) {
                const size_t g = static_cast<size_t>(s) * R + rep;
                dsd_replica& x = b.replicas[g];
                x = dsd_replica{};
                x.scenario = static_cast<uint32_t>(s);
                x.seed = seeds[idx][rep];
                x.gen_seed = r.gen_seed_fixed ? r.gen_seed : x.seed;
                b.replica_origin[g] = {static_cast<int64_t>(idx), static_cast<int32_t>(rep)};
            }
        }
    });
    if (n_shards > 1) {
        // one shard: the replicas shard_of_replicas deals to it (the split a
        // multi-device handle makes), kept in point-major order
        const std::vector<int32_t> sh = shard_of_replicas(b.scenarios.data(), b.replicas.data(), n_rep, n_shards);
        size_t w = 0;
        for (size_t g = 0; g < n_rep; ++g) {
            if (sh[g] != shard) continue;
            b.replicas[w] = b.replicas[g];
            b.replica_origin[w] = b.replica_origin[g];
            ++w;
        }
        b.replicas.resize(w);
        b.replica_origin.resize(w);
    }
    tm.lap("replicas");
}

SweepBatch plan_sweep(const Node& node, const std::string& base_dir, int shard, int n_shards, Caches* caches) {
    SweepBatch b;
    b.spec = SweepSpec::from_node(node, base_dir);
    plan_points(b, 0, b.spec.point_count(), shard, n_shards, caches);
    return b;
}

SweepBatch plan_range(const SweepSpec& spec, size_t lo, size_t hi, Caches* caches) {
    SweepBatch b;
    b.spec = spec;
    plan_points(b, lo, hi, 0, 1, caches);
    return b;
}

PhaseTimer::PhaseTimer(const char* what) : what_(what), on_(std::getenv("DSD_HOST_TIMING") != nullptr) {
    if (on_) t_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void PhaseTimer::lap(const char* phase) {
    if (!on_) return;
    const double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    std::fprintf(stderr, "[dsd %s] %-10s %8.2f ms\n", what_, phase, t - t_);
    t_ = t;
}

void launch_batch(Runtime& rt, SweepBatch& b, bool reports) {
    PhaseTimer tm("run_sweep");
    if (b.replicas.empty()) return;
    rt.prepare(b.scenarios.data(), b.scenarios.size(), b.replicas.data(), b.replicas.size(), reports);
    tm.lap("prepare");
    rt.launch();
    tm.lap("launch");
}

void collect_batch(Runtime& rt, SweepBatch& b, const std::string& out_dir, SweepTotals& tot) {
    PhaseTimer tm("run_sweep");
    const bool reports = !out_dir.empty();
    const size_t n = b.replicas.size();
    const dsd_replica_summary* sums = nullptr;
    if (n > 0) {
        rt.sync();
        tm.lap("kernels");
        sums = rt.host_summaries();
        tm.lap("summaries");
    }
    const int R = b.spec.repetitions;
    std::vector<double> thr(b.points.size(), 0.0), ttft(b.points.size(), 0.0), tpot(b.points.size(), 0.0);
    std::vector<std::string> digest(reports ? b.points.size() : 0);  // config digests, on first use
    // replicas k in [lo, hi): a point's replicas are contiguous (plan_sweep
    // places them in (point, rep) order), so chunks that start and end on
    // point boundaries own their points and sum them in rep order
    auto accumulate = [&](size_t lo, size_t hi, SweepTotals& t) {
        for (size_t k = lo; k < hi; ++k) {
            const auto [p, rep] = b.replica_origin[k];
            SweepPoint& pt = b.points[static_cast<size_t>(p)];
            const dsd_replica_summary& s = sums[k];
            t.events += static_cast<double>(s.events_processed);
            t.replicas += 1;
            if (s.status != DSD_OK) {
                pt.failed = true;
                pt.error = "engine capacity exceeded on the device (event heap / sequence arena)";
                continue;
            }
            thr[p] += s.throughput_rps;
            ttft[p] += s.mean_ttft_ms;
            tpot[p] += s.mean_tpot_ms;
            if (reports) {
                const Resolved& r = b.resolved[static_cast<size_t>(b.point_scenario[p])];
                ReplicaOutput out;
                out.summary = s;
                int64_t nrec = 0, nseq = 0;
                rt.fetch_records(k, nullptr, 0, &nrec, nullptr, nullptr, 0, &nseq, nullptr, 0);
                out.records.resize(static_cast<size_t>(nrec));
                out.gamma_seq.resize(static_cast<size_t>(nseq));
                out.committed_seq.resize(static_cast<size_t>(nseq));
                out.busy_us.resize(static_cast<size_t>(r.scen.n_targets));
                rt.fetch_records(k, out.records.data(), out.records.size(), &nrec, out.gamma_seq.data(),
                                 out.committed_seq.data(), out.gamma_seq.size(), &nseq, out.busy_us.data(),
                                 out.busy_us.size());
                const std::string file =
                    out_dir + "/" + sanitize_filename(pt.point_id) + "_rep" + std::to_string(rep) + ".json";
                std::ofstream f(file, std::ios::binary);
                if (!f) throw Error(DSD_ERR_RUNTIME, "cannot write file: " + file);
                std::string& dg = digest[static_cast<size_t>(p)];
                if (dg.empty()) dg = point_digest(b.spec, b.point_base + static_cast<size_t>(p));
                f << emit_report(out, r.scen.n_targets, dg, b.replicas[k].seed);
                pt.report_files.push_back(file);
            }
        }
    };
    if (reports || n < 4096) {
        accumulate(0, n, tot);
    } else {
        std::vector<SweepTotals> part(host_threads());
        std::atomic<size_t> slot{0};
        parallel_chunks(n, 2048, [&](size_t lo, size_t hi) {
            auto boundary = [&](size_t k) {
                while (k > 0 && k < n && b.replica_origin[k].first == b.replica_origin[k - 1].first) ++k;
                return k;
            };
            SweepTotals& t = part[slot.fetch_add(1)];
            accumulate(boundary(lo), boundary(hi), t);
        });
        for (const SweepTotals& t : part) {  // integer-valued totals: any order is exact
            tot.events += t.events;
            tot.replicas += t.replicas;
        }
    }
    tm.lap(reports ? "reports" : "aggregate");
    for (size_t p = 0; p < b.points.size(); ++p) {
        SweepPoint& pt = b.points[p];
        tot.points += 1;
        if (pt.failed) {
            tot.failed += 1;
            continue;
        }
        pt.mean_throughput_rps = thr[p] / R;
        pt.mean_ttft_ms = ttft[p] / R;
        pt.mean_tpot_ms = tpot[p] / R;
    }
}

SweepTotals run_sweep(Runtime& rt, SweepBatch& b, const std::string& out_dir, SummaryParts* parts) {
    SweepTotals tot;
    const bool reports = !out_dir.empty();
    if (reports) std::filesystem::create_directories(out_dir);
    launch_batch(rt, b, reports);
    // the host is idle while the kernels run: render the summary text that
    // does not depend on the results
    {
        PhaseTimer tm("run_sweep");
        if (parts) *parts = render_summary_prefixes(b.points, b.point_base);
        tm.lap("prefixes");
    }
    collect_batch(rt, b, out_dir, tot);
    return tot;
}

// sweep_summary_json / sweep_summary_csv (sweep.cpp:164-199) in the layout
// JsonOut writes (2-space indent), split per point into the part that is
// known before the simulation (id, assignment) and the part that needs its
// results, so run_sweep renders the former while the kernels run.
SummaryParts render_summary_prefixes(const std::vector<SweepPoint>& points, size_t first) {
    SummaryParts parts;
    parts.json.resize(points.size());
    parts.csv.resize(points.size());
    for (size_t i = 0; i < points.size(); ++i) {
        const SweepPoint& p = points[i];
        std::string& j = parts.json[i];
        j += first + i ? ",\n    {\n      \"point\": \"" : "\n    {\n      \"point\": \"";
        cfg::json_escape(j, p.point_id);
        j += "\",\n      \"assignment\": {";
        for (size_t k = 0; k < p.assignment.size(); ++k) {
            j += k ? ",\n        \"" : "\n        \"";
            cfg::json_escape(j, p.assignment[k].first);
            j += "\": \"";
            cfg::json_escape(j, p.assignment[k].second);
            j += '"';
        }
        j += p.assignment.empty() ? "}" : "\n      }";
        j += ",\n      \"failed\": ";
        parts.csv[i] = "\"" + p.point_id + "\",";
    }
    return parts;
}

// The point's entry after its prefix; json and/or csv may be null.
static void render_point(const SummaryParts& parts, const SweepPoint& p, size_t i, std::string* j, std::string* c) {
    std::string thr, ttft, tpot;
    if (c || !p.failed) {
        thr = cfg::fmt_fixed(p.mean_throughput_rps, 6);
        ttft = cfg::fmt_fixed(p.mean_ttft_ms, 3);
        tpot = cfg::fmt_fixed(p.mean_tpot_ms, 3);
    }
    if (j) {
        *j += parts.json[i];
        if (p.failed) {
            *j += "true,\n      \"error\": \"";
            cfg::json_escape(*j, p.error);
            *j += "\"\n    }";
        } else {
            *j += "false,\n      \"throughput_rps\": ";
            *j += thr;
            *j += ",\n      \"mean_ttft_ms\": ";
            *j += ttft;
            *j += ",\n      \"mean_tpot_ms\": ";
            *j += tpot;
            *j += "\n    }";
        }
    }
    if (c) {
        *c += parts.csv[i];
        *c += p.failed ? "1," : "0,";
        *c += thr;
        *c += ',';
        *c += ttft;
        *c += ',';
        *c += tpot;
        *c += '\n';
    }
}

void assemble_summaries(const SummaryParts& parts, const std::vector<SweepPoint>& points, std::string* json,
                        std::string* csv) {
    const size_t n = points.size();
    // contiguous point ranges rendered in parallel, then concatenated
    const size_t chunks = std::max<size_t>(1, std::min<size_t>(host_threads(), n / 512));
    std::vector<std::string> cj(chunks), cc(chunks);
    parallel_chunks(chunks, 1, [&](size_t c0, size_t c1) {
        for (size_t c = c0; c < c1; ++c)
            for (size_t i = n * c / chunks; i < n * (c + 1) / chunks; ++i)
                render_point(parts, points[i], i, json ? &cj[c] : nullptr, csv ? &cc[c] : nullptr);
    });
    if (json) {
        size_t len = 32;
        for (const auto& x : cj) len += x.size();
        json->clear();
        json->reserve(len);
        *json += "{\n  \"points\": [";
        for (const auto& x : cj) *json += x;
        *json += points.empty() ? "]\n}\n" : "\n  ]\n}\n";
    }
    if (csv) {
        size_t len = 64;
        for (const auto& x : cc) len += x.size();
        csv->clear();
        csv->reserve(len);
        *csv += "point,failed,throughput_rps,mean_ttft_ms,mean_tpot_ms\n";
        for (const auto& x : cc) *csv += x;
    }
}

std::string assemble_summary_json(const SummaryParts& parts, const std::vector<SweepPoint>& points) {
    std::string out;
    assemble_summaries(parts, points, &out, nullptr);
    return out;
}

std::string assemble_summary_csv(const SummaryParts& parts, const std::vector<SweepPoint>& points) {
    std::string out;
    assemble_summaries(parts, points, nullptr, &out);
    return out;
}

std::string sweep_summary_json(const std::vector<SweepPoint>& points) {
    return assemble_summary_json(render_summary_prefixes(points), points);
}

std::string sweep_summary_csv(const std::vector<SweepPoint>& points) {
    return assemble_summary_csv(render_summary_prefixes(points), points);
}

}  // namespace dsd::host
