// pack.cpp — host-side validation and packing of a replica batch into the
// device layout of layout.cuh (scenario blob, capacities, replica arrays) and
// the workspace field layout.  Plain C++: shared by the CUDA runtime.
#include "pack.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <unordered_map>
#include <numeric>
#include <string>
#include <type_traits>

#include "layout.cuh"

namespace dsd {

namespace {

struct BlobBuilder {
    std::vector<char> data;
    std::unordered_map<const void*, int64_t> seen;
    // Arrays shared between scenarios (latency grids, traces, AWC weights)
    // are stored once, keyed by their host address; a scenario's own small
    // arrays (groups, grid indices) are simply appended.
    static constexpr size_t kDedupeMin = 256;
    int64_t put(const void* src, size_t bytes, bool dedupe = true) {
        dedupe = dedupe && bytes >= kDedupeMin;
        if (dedupe && src) {
            auto it = seen.find(src);
            if (it != seen.end()) return it->second;
        }
        size_t off = (data.size() + 15) & ~size_t(15);
        data.resize(off + std::max<size_t>(bytes, 1));
        if (bytes) std::memcpy(data.data() + off, src, bytes);
        if (dedupe && src) seen[src] = static_cast<int64_t>(off);
        return static_cast<int64_t>(off);
    }
    // a derived array (e.g. a re-laid-out copy) stored once per source `key`
    int64_t put_keyed(const void* key, const std::vector<double>& v) {
        auto it = seen.find(key);
        if (it != seen.end()) return it->second;
        const int64_t off = put(v.data(), sizeof(double) * v.size(), false);
        seen[key] = off;
        return off;
    }
};

[[noreturn]] void cfg_error(const std::string& m) { throw Error(DSD_ERR_CONFIG, m); }

int64_t awc_param_count(const dsd_awc_model& m);

// WcDnn parameters (the reference's flat layout, mlp.cpp:20-48) in the
// device's transposed layout: every weight matrix [rows][cols] stored as
// [cols][rows] (engine.cuh, awc_forward_warp); biases and the head as is.
std::vector<double> awc_transpose(const dsd_awc_model& m) {
    const int64_t H = m.hidden, I = m.input;
    std::vector<double> t(static_cast<size_t>(awc_param_count(m)));
    const double* p = m.params;
    int64_t o = 0;
    auto mat = [&](int64_t rows, int64_t cols) {
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t c = 0; c < cols; ++c) t[static_cast<size_t>(o + c * rows + r)] = p[o + r * cols + c];
        o += rows * cols;
    };
    auto vec = [&](int64_t n) {
        for (int64_t k = 0; k < n; ++k) t[static_cast<size_t>(o + k)] = p[o + k];
        o += n;
    };
    mat(H, I);
    vec(H);
    for (int b = 0; b < m.blocks; ++b) {
        mat(H, H);
        vec(H);
        mat(H, H);
        vec(H);
    }
    vec(H + 1);
    return t;
}

int64_t awc_param_count(const dsd_awc_model& m) {
    int64_t H = m.hidden, I = m.input;
    return H * I + H + static_cast<int64_t>(m.blocks) * (2 * H * H + 2 * H) + H + 1;
}

// Segment table of one axis for integer queries 0..Q, Q = ceil(axis.back())
// (larger queries clamp to the same entry).  Each entry is what
// Grid::interpolate computes for that query (profile.cpp:20-27, 64-84):
// clamp, upper_bound segment, weight (q - a[lo]) / (a[hi] - a[lo]).
int64_t axis_table(BlobBuilder& B, const double* axis, int n, int32_t* size) {
    const double back = axis[n - 1];
    if (!(back >= 0.0) || back > 65536.0) {
        *size = 0;
        return -1;
    }
    const int32_t q_max = static_cast<int32_t>(std::ceil(back));
    std::vector<AxisSeg> tab(static_cast<size_t>(q_max) + 1);
    for (int32_t q = 0; q <= q_max; ++q) {
        double v = static_cast<double>(q);
        if (v < axis[0]) v = axis[0];
        else if (v > back) v = back;
        int lo = 0;
        if (n > 1) {
            int hi = static_cast<int>(std::upper_bound(axis, axis + n, v) - axis);
            lo = hi == 0 ? 0 : (hi >= n ? n - 2 : hi - 1);
        }
        const int hi = std::min(lo + 1, n - 1);
        tab[static_cast<size_t>(q)] = AxisSeg{lo, hi, hi == lo ? 0.0 : (v - axis[lo]) / (axis[hi] - axis[lo])};
    }
    *size = q_max + 1;
    return B.put(tab.data(), sizeof(AxisSeg) * tab.size(), false);
}

}  // namespace

Packed pack_batch(const dsd_scenario* sc, size_t ns, const dsd_replica* reps, size_t n, bool probe) {
    Packed P;
    pack_batch_into(P, sc, ns, reps, n, probe);
    return P;
}

void pack_batch_into(Packed& P, const dsd_scenario* sc, size_t ns, const dsd_replica* reps, size_t n, bool probe) {
    if (ns == 0 && n > 0) cfg_error("batch has replicas but no scenarios");
    BlobBuilder B;
    B.data = std::move(P.blob);
    B.data.clear();
    B.data.reserve(256 * ns + (1u << 16));
    B.seen.reserve(64);
    std::vector<DevScenario>& ds = P.scen;
    ds.clear();
    ds.resize(ns);
    Caps& c = P.caps;
    c = Caps{};
    bool any_pairs = false;
    double last_pm_in = std::nan(""), last_pm = 0.0, last_om_in = std::nan(""), last_om = 0.0;
    std::vector<int64_t> scen_bw(ns, 0), scen_nr(ns, 0);
    std::map<const dsd_grid*, int64_t> grid_tables;
    const dsd_grid* last_grids = nullptr;
    auto last_git = grid_tables.end();
    for (size_t k = 0; k < ns; ++k) {
        const dsd_scenario& s = sc[k];
        DevScenario& d = ds[k];
        std::memset(&d, 0, sizeof(d));
        d.o_slat = -1;  // set by Runtime::prepare for specialised batches
        // error-message prefix, built only when a check fails
        const auto where = [k] { return "scenario " + std::to_string(k) + ": "; };
        if (s.n_targets < 1) cfg_error(where() + "target pool must be non-empty");
        if (s.n_drafts < 0) cfg_error(where() + "negative draft pool");
        if (s.n_target_groups < 1 || (s.n_drafts > 0 && s.n_draft_groups < 1))
            cfg_error(where() + "group counts must be >= 1");
        d.n_targets = s.n_targets;
        d.n_drafts = s.n_drafts;
        d.n_tg = s.n_target_groups;
        d.n_dg = std::max(1, s.n_draft_groups);
        d.fused_everything = (s.window_kind == DSD_WINDOW_FUSED || s.n_drafts == 0) ? 1 : 0;
        for (int i = 0; i < s.n_targets; ++i)
            if (s.target_group[i] < 0 || s.target_group[i] >= s.n_target_groups)
                cfg_error(where() + "target group out of range");
        for (int i = 0; i < s.n_drafts; ++i)
            if (s.draft_group[i] < 0 || s.draft_group[i] >= s.n_draft_groups)
                cfg_error(where() + "draft group out of range");
        int32_t zero = 0;
        d.o_tgroup = B.put(s.target_group, sizeof(int32_t) * s.n_targets);
        d.o_dgroup = s.n_drafts > 0 ? B.put(s.draft_group, sizeof(int32_t) * s.n_drafts)
                                    : B.put(&zero, sizeof(zero), false);
        if (!s.links) cfg_error(where() + "missing link table");
        {
            size_t nl = static_cast<size_t>(d.n_dg) * d.n_tg;
            for (size_t l = 0; l < nl; ++l) {
                if (s.n_drafts == 0 && l > 0) break;
                if (s.links[l].rtt_ms < 0.0 || s.links[l].jitter_ms < 0.0)
                    cfg_error("link rtt_ms/jitter_ms must be >= 0");
                if (s.links[l].jitter_ms > s.links[l].rtt_ms)
                    cfg_error("link jitter_ms must not exceed rtt_ms");
                // one-way delays are held as int32 microseconds on the device
                if (!(s.links[l].rtt_ms <= 2.0e6))
                    throw Error(DSD_ERR_RUNTIME, "link rtt_ms above the engine limit of 2e6 ms");
            }
            // device links carry the constant one-way delay of jitter-free links:
            // net_delay = llround((rtt/2 + U(-0, 0)) * 1000) = llround((rtt/2 + 0.0) * 1000)
            // (engine.cpp:10-15); when every link is jitter-free the jitter stream
            // is never observable, so the engine skips its draws.
            const size_t ndev = s.n_drafts > 0 ? nl : 1;
            DevLink dl_small[8];
            std::vector<DevLink> dl_big(ndev > 8 ? ndev : 0);
            DevLink* dl = ndev > 8 ? dl_big.data() : dl_small;
            bool jitter_free = true;
            for (size_t l = 0; l < ndev; ++l) {
                dl[l].rtt_ms = s.links[l].rtt_ms;
                dl[l].jitter_ms = s.links[l].jitter_ms;
                dl[l].fixed_us = std::llround((s.links[l].rtt_ms / 2.0 + 0.0) * 1000.0);
                if (s.links[l].jitter_ms != 0.0) jitter_free = false;
            }
            d.o_links = B.put(dl, sizeof(DevLink) * ndev, false);
            d.jitter_free = jitter_free ? 1 : 0;
        }
        // grids
        if (s.n_grids < 1 || !s.grids) cfg_error(where() + "latency profile has no grids");
        // (a sweep's scenarios share one profile: the last lookup first)
        auto git = (last_grids == s.grids) ? last_git : grid_tables.find(s.grids);
        if (git == grid_tables.end()) {
            std::vector<DevGrid> g(s.n_grids);
            for (int gi = 0; gi < s.n_grids; ++gi) {
                const dsd_grid& src = s.grids[gi];
                if (src.n_batch < 1 || src.n_context < 1)
                    cfg_error("profile grid: empty axis");
                for (int a = 1; a < src.n_batch; ++a)
                    if (!(src.batch_axis[a] > src.batch_axis[a - 1]))
                        cfg_error("profile grid: batch axis must be strictly increasing");
                for (int a = 1; a < src.n_context; ++a)
                    if (!(src.context_axis[a] > src.context_axis[a - 1]))
                        cfg_error("profile grid: context axis must be strictly increasing");
                g[gi].nb = src.n_batch;
                g[gi].nc = src.n_context;
                g[gi].o_batch = B.put(src.batch_axis, sizeof(double) * src.n_batch);
                g[gi].o_ctx = B.put(src.context_axis, sizeof(double) * src.n_context);
                g[gi].o_vals =
                    B.put(src.values_ms, sizeof(double) * src.n_batch * src.n_context);
                g[gi].calibration = src.calibration;
                g[gi].o_btab = axis_table(B, src.batch_axis, src.n_batch, &g[gi].nbt);
                g[gi].o_ctab = axis_table(B, src.context_axis, src.n_context, &g[gi].nct);
            }
            int64_t off = B.put(g.data(), sizeof(DevGrid) * g.size(), false);
            git = grid_tables.emplace(s.grids, off).first;
        }
        last_grids = s.grids;
        last_git = git;
        d.o_grids = git->second;
        d.n_grids = s.n_grids;
        for (int i = 0; i < s.n_targets; ++i)
            for (int op = 0; op < 2; ++op) {
                int32_t g = s.target_grids[2 * i + op];
                if (g < 0 || g >= s.n_grids)
                    cfg_error("no latency profile for target " + std::to_string(i));
            }
        d.o_tgrid = B.put(s.target_grids, sizeof(int32_t) * 2 * s.n_targets);
        if (s.n_drafts > 0) {
            if (!d.fused_everything)
                for (int i = 0; i < s.n_drafts; ++i)
                    for (int op = 0; op < 2; ++op) {
                        int32_t g = s.draft_grids[2 * i + op];
                        if (g < 0 || g >= s.n_grids)
                            cfg_error("no latency profile for draft " + std::to_string(i));
                    }
            d.o_dgrid = B.put(s.draft_grids, sizeof(int32_t) * 2 * s.n_drafts);
        } else {
            d.o_dgrid = B.put(&zero, sizeof(zero), false);
        }
        // policy
        if (s.routing < 0 || s.routing > 2) cfg_error("unhandled routing policy");
        if (s.batching < 0 || s.batching > 1) cfg_error("unknown batching policy");
        if (s.window_kind < 0 || s.window_kind > 3) cfg_error("unknown window policy");
        if (s.max_batch_size < 1) cfg_error("batching.max_batch_size must be >= 1");
        if (s.draft_max_batch < 1) cfg_error("predict: invalid batch shape (draft_max_batch < 1)");
        if (s.similarity_fraction < 0.0) cfg_error("batching.similarity_fraction must be >= 0");
        if (s.gamma_min < 1 || s.gamma_max < s.gamma_min)
            cfg_error("window gamma bounds must satisfy 1 <= gamma_min <= gamma_max");
        if (s.window_kind == DSD_WINDOW_STATIC && !d.fused_everything && s.gamma < 1)
            cfg_error("static window gamma must be >= 1");
        if (s.queue_capacity < 1) cfg_error("queue_capacity must be >= 1");
        d.routing = s.routing;
        d.batching = s.batching;
        d.max_batch = s.max_batch_size;
        d.draft_max_batch = s.draft_max_batch;
        d.batching_window_us = s.batching_window_us;
        d.sim_frac = s.similarity_fraction;
        d.window_kind = s.window_kind;
        d.gamma = s.gamma;
        d.gamma_min = s.gamma_min;
        d.gamma_max = s.gamma_max;
        d.queue_capacity = s.queue_capacity;
        d.pair_stats = ((!d.fused_everything && (s.window_kind == DSD_WINDOW_DYNAMIC ||
                                                  s.window_kind == DSD_WINDOW_AWC)) ||
                        (probe && s.n_drafts > 0))
                           ? 1
                           : 0;
        if (s.window_kind == DSD_WINDOW_AWC && !d.fused_everything) {
            if (!s.awc) cfg_error("awc window policy requires a trained model");
            const dsd_awc_model& m = *s.awc;
            if (m.input != 5) cfg_error("awc model input dimension must be 5");
            if (m.hidden < 1 || m.hidden > kMaxHidden || m.blocks < 0)
                cfg_error("awc model dimensions unsupported (hidden must be 1..64)");
            d.awc_hidden = m.hidden;
            d.awc_blocks = m.blocks;
            d.awc_input = m.input;
            d.o_awc_params = B.put_keyed(m.params, awc_transpose(m));
            for (int f = 0; f < 5; ++f) {
                d.awc_lo[f] = m.norm_lo[f];
                d.awc_hi[f] = m.norm_hi[f];
                d.awc_log[f] = m.log_scale[f] ? 1 : 0;
            }
        }
        if (d.pair_stats) any_pairs = true;
        if (d.window_kind == DSD_WINDOW_AWC && !d.fused_everything) c.awc = 1;
        // workload
        d.workload = s.workload;
        int64_t N = 0, bw = 0, lbound = 0;
        if (s.workload == DSD_WORKLOAD_SYNTHETIC) {
            // generate_synthetic preconditions (trace.cpp:146-153)
            if (!(s.acceptance_rate >= 0.0 && s.acceptance_rate <= 1.0))
                cfg_error("acceptance rate must lie in [0, 1]");
            if (!(s.rate_rps > 0.0) || !std::isfinite(s.rate_rps))
                cfg_error("poisson rate must be finite and positive");
            if (s.n_requests < 0) cfg_error("n_requests must be >= 0");
            if (s.gen_n_drafts < 1) cfg_error("n_drafts must be >= 1");
            if (s.n_drafts > 0 && s.gen_n_drafts > s.n_drafts)
                cfg_error("synthetic drafter range exceeds the draft pool");
            if (s.prompt_cap < 1 || s.output_cap < 1) cfg_error("length caps must be >= 1");
            d.n_requests = s.n_requests;
            d.rate_rps = s.rate_rps;
            d.mean_gap_ms = 1000.0 / s.rate_rps;
            d.alpha = s.acceptance_rate;
            // host libm, as the reference (trace.cpp:163-164); repeated medians reuse the last log
            if (s.prompt_median != last_pm_in || std::signbit(s.prompt_median) != std::signbit(last_pm_in)) {
                last_pm_in = s.prompt_median;
                last_pm = std::log(s.prompt_median);
            }
            if (s.output_median != last_om_in || std::signbit(s.output_median) != std::signbit(last_om_in)) {
                last_om_in = s.output_median;
                last_om = std::log(s.output_median);
            }
            d.p_mu = last_pm;
            d.o_mu = last_om;
            d.p_sigma = s.prompt_sigma;
            d.o_sigma = s.output_sigma;
            d.p_cap = s.prompt_cap;
            d.o_cap = s.output_cap;
            d.gen_n_drafts = s.gen_n_drafts;
            N = s.n_requests;
            bw = N * ((s.output_cap + 63) / 64);
            lbound = N * s.output_cap;
        } else if (s.workload == DSD_WORKLOAD_TRACE || s.workload == DSD_WORKLOAD_TRACE_POISSON) {
            if (!s.trace) cfg_error("trace workload without a trace");
            const dsd_trace& t = *s.trace;
            if (s.workload == DSD_WORKLOAD_TRACE_POISSON && !(s.rate_rps > 0.0))
                cfg_error("poisson arrival mode requires a positive rate");
            N = t.n;
            std::vector<int64_t> order(N);
            std::iota(order.begin(), order.end(), 0);
            bool sorted = true;
            for (int64_t i = 0; i < N; ++i) {
                // validate_record (trace.cpp:31-47) + validate_drafter_ids (:49-58)
                const std::string rw = "trace record " + std::to_string(i) + ": field ";
                if (t.prompt_length[i] < 1) cfg_error(rw + "'prompt_length' must be >= 1");
                if (t.output_length[i] < 0) cfg_error(rw + "'output_length' must be >= 0");
                if (t.arrival_us[i] < 0) cfg_error(rw + "'arrival_time_ms' must be >= 0");
                if (t.drafter_id[i] < 0) cfg_error(rw + "'drafter_id' must be >= 0");
                int64_t nb = t.bits_offset[i + 1] - t.bits_offset[i];
                if (t.output_length[i] > 0 && nb <= 0)
                    cfg_error(rw + "'acceptance_seq' must be non-empty when output_length > 0");
                if (s.n_drafts > 0 && t.drafter_id[i] >= s.n_drafts)
                    cfg_error(rw + "'drafter_id' " + std::to_string(t.drafter_id[i]) +
                              " out of range for draft pool of size " + std::to_string(s.n_drafts));
                if (t.prompt_length[i] > INT32_MAX || t.output_length[i] > INT32_MAX)
                    cfg_error(rw + "length exceeds engine limits");
                bw += (nb + 63) / 64;
                lbound += t.output_length[i];
                if (i > 0 && t.arrival_us[i] < t.arrival_us[i - 1]) sorted = false;
            }
            d.tr_n = N;
            d.rate_rps = s.rate_rps;
            d.o_tr_prompt = B.put(t.prompt_length, sizeof(int64_t) * N);
            d.o_tr_output = B.put(t.output_length, sizeof(int64_t) * N);
            d.o_tr_arrival = B.put(t.arrival_us, sizeof(int64_t) * N);
            d.o_tr_drafter = B.put(t.drafter_id, sizeof(int64_t) * N);
            d.o_tr_bitoff = B.put(t.bits_offset, sizeof(int64_t) * (N + 1));
            d.o_tr_bits = B.put(t.acceptance_bits, static_cast<size_t>(t.bits_offset[N]));
            if (s.workload == DSD_WORKLOAD_TRACE && !sorted) {
                std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
                    return t.arrival_us[a] < t.arrival_us[b];
                });
                d.o_tr_order = B.put(order.data(), sizeof(int64_t) * N, false);
                d.has_order = 1;
            }
        } else {
            cfg_error("unknown workload kind");
        }
        if (N >= (int64_t(1) << 26)) throw Error(DSD_ERR_RUNTIME, "too many requests per replica (engine limit 2^26)");
        if (lbound >= (int64_t(1) << 31) || bw >= (int64_t(1) << 31))
            throw Error(DSD_ERR_RUNTIME, "total output tokens per replica above the engine limit of 2^31");
        scen_nr[k] = N;
        scen_bw[k] = bw;
        c.nr = std::max(c.nr, N);
        c.ns = std::max<int64_t>(c.ns, s.n_targets + s.n_drafts);
        c.nt = std::max<int64_t>(c.nt, s.n_targets);
        if (d.pair_stats)
            c.np = std::max<int64_t>(c.np, static_cast<int64_t>(s.n_targets) * s.n_drafts);
    }
    (void)any_pairs;
    std::vector<uint32_t>& rs = P.rep_scen;
    std::vector<uint64_t>& seed = P.seed;
    std::vector<uint64_t>& gseed = P.gseed;
    rs.resize(n);
    seed.resize(n);
    gseed.resize(n);
    for (size_t i = 0; i < n; ++i) {
        if (reps[i].scenario >= ns) cfg_error("replica references an unknown scenario");
        rs[i] = reps[i].scenario;
        seed[i] = reps[i].seed;
        gseed[i] = reps[i].gen_seed;
        c.bw = std::max(c.bw, scen_bw[reps[i].scenario]);
    }
    c.nr = std::max<int64_t>(c.nr, 1);
    c.ns = std::max<int64_t>(c.ns, 1);
    c.nt = std::max<int64_t>(c.nt, 1);
    c.bw = std::max<int64_t>(c.bw, 1);
    c.hc = 2 * c.nr + 8 * c.ns + 64;
    c.n = static_cast<int64_t>(n);
    c.nwarps = (c.n + kLanes - 1) / kLanes;

    P.blob = std::move(B.data);
}

size_t layout_workspace(Workspace& W, const Caps& c, char* base) {
    W.c = c;
    const int64_t lanes = c.nwarps * kLanes;
    std::vector<std::pair<void**, size_t>> fields;
    auto field = [&](auto*& ptr, int64_t cap) {
        using T = std::remove_reference_t<decltype(*ptr)>;
        fields.emplace_back(reinterpret_cast<void**>(&ptr), sizeof(T) * static_cast<size_t>(cap * lanes));
    };
    // request records are replica-contiguous (not lane-interleaved): `lanes`
    // replicas x nr records of 128 bytes
    field(W.req, c.nr);
    field(W.srv, kServerFields * c.ns);
    field(W.v_busy_us, c.ns);
    field(W.route_state, 5);  // sized lanes x 5, indexed replica-contiguous
    if (c.np > 0) {
        field(W.t_tpot, c.nt * 50); field(W.t_tpos, c.nt); field(W.t_tcnt, c.nt);
        field(W.p_acc_ex, c.np * 20); field(W.p_acc_ac, c.np * 20); field(W.p_acc_pos, c.np);
        field(W.p_acc_cnt, c.np); field(W.p_rtt, c.np * 20); field(W.p_rtt_pos, c.np);
        field(W.p_rtt_cnt, c.np); field(W.p_gprev, c.np); field(W.p_dyn, c.np);
        field(W.p_sm_init, c.np); field(W.p_sm_ema, c.np); field(W.p_sm_low, c.np);
        field(W.p_sm_fused, c.np);
    }
    field(W.h_time, c.hc); field(W.h_key, c.hc);
    size_t off = 0;
    for (auto& f : fields) {
        if (base) *f.first = base + off;
        off += (f.second + 255) & ~size_t(255);
    }
    const size_t bits_bytes = sizeof(uint64_t) * static_cast<size_t>(c.bw) * static_cast<size_t>(std::max<int64_t>(c.n, 1));
    if (base) W.bits = reinterpret_cast<uint64_t*>(base + off);
    off += (bits_bytes + 255) & ~size_t(255);
    return off;
}

}  // namespace dsd
