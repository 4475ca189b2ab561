// engine.cuh — the per-replica discrete-event engine (one GPU thread = one
// replica), a B200-native restatement of the reference's hot loop
//   SimKernel::run_until   proj/src/sim/event_queue.cpp:28-42
//   Engine::Impl::handle   proj/src/engine/engine.cpp:249-646
// with the latency model (proj/src/latency/profile.cpp:20-151), the policies
// (proj/src/policies/policies.cpp), the metrics hooks (proj/src/metrics/metrics.cpp:40-128)
// and the AWC controller (proj/src/awc/{features,mlp,smoother}.cpp) inlined.
//
// Design:
//  * arrivals never enter the heap: they are a pre-ordered stream whose seq
//    (0..N-1) is below every dynamic event's, so the pop is a 2-way merge of
//    the arrival cursor and a small (time, seq) binary heap of dynamic events;
//  * work queues, running batches and draft session FIFOs are intrusive
//    linked lists through two work-item slots per request (a target prefill
//    and "the other" item), so no per-server capacity is needed;
//  * replica scalars (clock, seq counter, RNG states, totals) live in
//    registers for the whole run; everything else is warp-interleaved SoA.
// Bit-exactness: all floating point is compiled with -fmad=false and follows
// the reference's operation order (see comments at each site).
#pragma once
#include <cmath>
#include <cstdint>

#include "layout.cuh"
#include "rng.cuh"

namespace dsd {

struct Lane {
    int64_t w;
    int lane;
    template <typename T>
    DSD_HD T& at(T* base, int64_t cap, int64_t idx) const {
        return base[(w * cap + idx) * kLanes + lane];
    }
};

template <typename T>
DSD_HD const T* blob_ptr(const char* blob, int64_t off) {
    return reinterpret_cast<const T*>(blob + off);
}

// ---------------------------------------------------------------------------
// latency model: Grid::interpolate (profile.cpp:57-88) + predict (:129-151)
// ---------------------------------------------------------------------------
DSD_HD int segment_index(const double* axis, int n, double q) {
    // std::upper_bound then clamp to a valid [i, i+1] segment (profile.cpp:20-27)
    if (n == 1) return 0;
    int lo = 0, hi = n;  // first element > q
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (axis[mid] > q) hi = mid; else lo = mid + 1;
    }
    if (lo == 0) return 0;
    if (lo >= n) return n - 2;
    return lo - 1;
}

DSD_HD double grid_interpolate(const char* blob, const DevGrid& g, double batch, double context) {
    const double* ba = blob_ptr<double>(blob, g.o_batch);
    const double* ca = blob_ptr<double>(blob, g.o_ctx);
    const double* v = blob_ptr<double>(blob, g.o_vals);
    double b = batch, c = context;
    if (b < ba[0]) b = ba[0]; else if (b > ba[g.nb - 1]) b = ba[g.nb - 1];
    if (c < ca[0]) c = ca[0]; else if (c > ca[g.nc - 1]) c = ca[g.nc - 1];
    int bi = segment_index(ba, g.nb, b);
    int ci = segment_index(ca, g.nc, c);
    int bj = bi + 1 < g.nb - 1 ? bi + 1 : g.nb - 1;
    int cj = ci + 1 < g.nc - 1 ? ci + 1 : g.nc - 1;
    double tb = (bj == bi) ? 0.0 : (b - ba[bi]) / (ba[bj] - ba[bi]);
    double tc = (cj == ci) ? 0.0 : (c - ca[ci]) / (ca[cj] - ca[ci]);
    const int n = g.nc;
    // same association as the reference: ((a*b)*v) summed left to right
    double r = (1.0 - tb) * (1.0 - tc) * v[bi * n + ci] + (1.0 - tb) * tc * v[bi * n + cj] +
               tb * (1.0 - tc) * v[bj * n + ci] + tb * tc * v[bj * n + cj];
    return r * g.calibration;
}

// ---------------------------------------------------------------------------
// AWC: FeatureNormalizer::transform + WcDnn::forward (mlp.cpp:83-97,163-176)
// with Backend::matvec in the AVX2 summation order the reference auto-selects
// on AVX2 hosts (kernels_avx2.cpp:17-40, kernels_dispatch.cpp:21-26).
// ---------------------------------------------------------------------------
DSD_HD void matvec_avx2_order(const double* w, const double* x, const double* bias, double* y,
                              int rows, int cols) {
    const int tail = cols & ~3;
    for (int r = 0; r < rows; ++r) {
        const double* row = w + static_cast<int64_t>(r) * cols;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = 0;
        for (; c < tail; c += 4) {
            a0 = a0 + row[c] * x[c];
            a1 = a1 + row[c + 1] * x[c + 1];
            a2 = a2 + row[c + 2] * x[c + 2];
            a3 = a3 + row[c + 3] * x[c + 3];
        }
        double s = (a0 + a2) + (a1 + a3);  // hsum: lo+hi then unpackhi (kernels_avx2.cpp:17-23)
        for (; c < cols; ++c) s += row[c] * x[c];
        y[r] = bias[r] + s;
    }
}

DSD_HD double awc_predict(const char* blob, const DevScenario& S, const double raw[5]) {
    double x[5];
    for (int f = 0; f < 5; ++f) {
        double v = S.awc_log[f] ? log1p(raw[f]) : raw[f];
        double span = S.awc_hi[f] - S.awc_lo[f];
        x[f] = span > 0.0 ? (v - S.awc_lo[f]) / span : 0.0;
    }
    const int H = S.awc_hidden, I = S.awc_input;
    const double* p = blob_ptr<double>(blob, S.o_awc_params);
    double h[kMaxHidden], u[kMaxHidden], s[kMaxHidden];
    int64_t off = 0;
    matvec_avx2_order(p + off, x, p + off + H * I, h, H, I);
    off += static_cast<int64_t>(H) * I + H;
    for (int b = 0; b < S.awc_blocks; ++b) {
        const double* w1 = p + off;
        const double* b1 = w1 + static_cast<int64_t>(H) * H;
        const double* w2 = b1 + H;
        const double* b2 = w2 + static_cast<int64_t>(H) * H;
        matvec_avx2_order(w1, h, b1, u, H, H);
        for (int i = 0; i < H; ++i) {  // kernels::silu (kernels_scalar.cpp:65-70)
            double sg = 1.0 / (1.0 + exp(-u[i]));
            s[i] = u[i] * sg;
        }
        matvec_avx2_order(w2, s, b2, u, H, H);
        for (int i = 0; i < H; ++i) h[i] += u[i];
        off += 2 * static_cast<int64_t>(H) * H + 2 * H;
    }
    const double* w_out = p + off;
    double out = w_out[H];  // b_out
    for (int i = 0; i < H; ++i) out += w_out[i] * h[i];
    return out;
}

// ---------------------------------------------------------------------------
// the engine
// ---------------------------------------------------------------------------
struct Engine {
    const Workspace& W;
    const DevScenario& S;
    const char* blob;
    Lane L;
    int64_t rep;

    // replica scalars (registers)
    int64_t N;
    int64_t now = 0;
    uint32_t seq_next;      // next seq for schedule(); arrivals hold 0..N-1
    int64_t heap_n = 0;
    int64_t next_arr = 0;
    uint64_t processed = 0;
    Rng routing, jitter;
    uint64_t rr_counter = 0;
    int64_t first_arrival = -1, last_completion = -1;
    int64_t net_wait_total = 0, net_wait_count = 0;
    int64_t completed = 0;
    int32_t fail = kFailNone;
    int64_t seqbase = 0;
    int32_t T, D;

    DSD_HD Engine(const Workspace& w, const DevScenario& s, int64_t replica)
        : W(w), S(s), blob(w.blob), rep(replica) {
        L.w = replica / kLanes;
        L.lane = static_cast<int>(replica % kLanes);
        T = S.n_targets;
        D = S.n_drafts;
    }

    // ---- accessors ----
    DSD_HD int64_t nr() const { return W.c.nr; }
#define RQ(field, i) L.at(W.field, W.c.nr, (i))
#define SL(field, i) L.at(W.field, 2 * W.c.nr, (i))
#define SV(field, i) L.at(W.field, W.c.ns, (i))

    DSD_HD uint32_t phase(int64_t i) const { return RQ(r_flags, i) & 7u; }
    DSD_HD void set_phase(int64_t i, uint32_t p) {
        uint8_t& f = RQ(r_flags, i);
        f = static_cast<uint8_t>((f & ~7u) | p);
    }
    DSD_HD bool flag(int64_t i, int bit) const { return (RQ(r_flags, i) >> bit) & 1u; }
    DSD_HD void set_flag(int64_t i, int bit, bool v) {
        uint8_t& f = RQ(r_flags, i);
        f = static_cast<uint8_t>(v ? (f | (1u << bit)) : (f & ~(1u << bit)));
    }
    static constexpr int kDpd = 3, kTpd = 4, kFused = 5;

    DSD_HD int32_t draft_of(int64_t i) const { return D > 0 ? RQ(r_drafter, i) : -1; }

    // ---- event heap: SimKernel::schedule (event_queue.cpp:20-26) ----
    DSD_HD bool key_less(int64_t ta, uint64_t ka, int64_t tb, uint64_t kb) const {
        return ta < tb || (ta == tb && ka < kb);
    }
    DSD_HD void schedule(int64_t t, uint32_t info) {
        if (heap_n >= W.c.hc) {
            fail = kFailHeap;
            return;
        }
        uint64_t key = (static_cast<uint64_t>(seq_next) << 32) | info;
        ++seq_next;
        int64_t i = heap_n++;
        while (i > 0) {
            int64_t p = (i - 1) >> 1;
            int64_t pt = L.at(W.h_time, W.c.hc, p);
            uint64_t pk = L.at(W.h_key, W.c.hc, p);
            if (!key_less(t, key, pt, pk)) break;
            L.at(W.h_time, W.c.hc, i) = pt;
            L.at(W.h_key, W.c.hc, i) = pk;
            i = p;
        }
        L.at(W.h_time, W.c.hc, i) = t;
        L.at(W.h_key, W.c.hc, i) = key;
    }
    DSD_HD void heap_pop() {
        int64_t n = --heap_n;
        if (n == 0) return;
        int64_t t = L.at(W.h_time, W.c.hc, n);
        uint64_t k = L.at(W.h_key, W.c.hc, n);
        int64_t i = 0;
        for (;;) {
            int64_t c = 2 * i + 1;
            if (c >= n) break;
            int64_t ct = L.at(W.h_time, W.c.hc, c);
            uint64_t ck = L.at(W.h_key, W.c.hc, c);
            if (c + 1 < n) {
                int64_t dt = L.at(W.h_time, W.c.hc, c + 1);
                uint64_t dk = L.at(W.h_key, W.c.hc, c + 1);
                if (key_less(dt, dk, ct, ck)) {
                    c = c + 1;
                    ct = dt;
                    ck = dk;
                }
            }
            if (!key_less(ct, ck, t, k)) break;
            L.at(W.h_time, W.c.hc, i) = ct;
            L.at(W.h_key, W.c.hc, i) = ck;
            i = c;
        }
        L.at(W.h_time, W.c.hc, i) = t;
        L.at(W.h_key, W.c.hc, i) = k;
    }

    static DSD_HD uint32_t info(uint32_t kind, uint32_t msg, uint32_t id) {
        return kind | (msg << 3) | (id << 5);
    }

    // ---- network: net_delay (engine.cpp:10-15) ----
    DSD_HD int64_t net_delay(int32_t d, int32_t t) {
        const int32_t* dg = blob_ptr<int32_t>(blob, S.o_dgroup);
        const int32_t* tg = blob_ptr<int32_t>(blob, S.o_tgroup);
        const double* lk = blob_ptr<double>(blob, S.o_links) + 2 * (dg[d] * S.n_tg + tg[t]);
        double rtt = lk[0], jit = lk[1];
        double j = jitter.uniform(-jit / 2.0, jit / 2.0);
        double ms = rtt / 2.0 + j;
        if (ms < 0.0) ms = 0.0;
        return llround(ms * 1000.0);
    }
    DSD_HD double link_rtt(int32_t d, int32_t t) const {
        const int32_t* dg = blob_ptr<int32_t>(blob, S.o_dgroup);
        const int32_t* tg = blob_ptr<int32_t>(blob, S.o_tgroup);
        return blob_ptr<double>(blob, S.o_links)[2 * (dg[d] * S.n_tg + tg[t])];
    }

    // ---- metrics hooks (metrics.cpp:40-128) ----
    DSD_HD int64_t pair_of(int32_t d, int32_t t) const { return static_cast<int64_t>(d) * T + t; }

    DSD_HD double acceptance_recent(int64_t p) const {
        int32_t cnt = L.at(W.p_acc_cnt, W.c.np, p);
        int64_t ex = 0, ac = 0;
        for (int k = 0; k < cnt; ++k) {
            ex += L.at(W.p_acc_ex, W.c.np * 20, p * 20 + k);
            ac += L.at(W.p_acc_ac, W.c.np * 20, p * 20 + k);
        }
        if (ex == 0) return 0.5;
        return static_cast<double>(ac) / static_cast<double>(ex);
    }
    DSD_HD void on_verify(int32_t d, int32_t t, int ex, int ac) {
        if (!S.pair_stats) return;
        int64_t p = pair_of(d, t);
        int32_t& cnt = L.at(W.p_acc_cnt, W.c.np, p);
        int32_t& pos = L.at(W.p_acc_pos, W.c.np, p);
        int64_t slot;
        if (cnt < 20) {
            slot = cnt++;
        } else {
            slot = pos;
            pos = (pos + 1) % 20;
        }
        L.at(W.p_acc_ex, W.c.np * 20, p * 20 + slot) = ex;
        L.at(W.p_acc_ac, W.c.np * 20, p * 20 + slot) = ac;
    }
    DSD_HD void on_rtt_sample(int32_t d, int32_t t, double rtt_ms) {
        if (!S.pair_stats) return;
        int64_t p = pair_of(d, t);
        int32_t& cnt = L.at(W.p_rtt_cnt, W.c.np, p);
        int32_t& pos = L.at(W.p_rtt_pos, W.c.np, p);
        int64_t slot;
        if (cnt < 20) {
            slot = cnt++;
        } else {
            slot = pos;
            pos = (pos + 1) % 20;
        }
        L.at(W.p_rtt, W.c.np * 20, p * 20 + slot) = rtt_ms;
    }
    DSD_HD void on_gamma_chosen(int32_t d, int32_t t, int g) {
        if (!S.pair_stats) return;
        L.at(W.p_gprev, W.c.np, pair_of(d, t)) = g;
    }
    DSD_HD void push_tpot(int32_t t, double v) {
        if (!S.pair_stats) return;
        int32_t& cnt = L.at(W.t_tcnt, W.c.nt, t);
        int32_t& pos = L.at(W.t_tpos, W.c.nt, t);
        int64_t slot;
        if (cnt < 50) {
            slot = cnt++;
        } else {
            slot = pos;
            pos = (pos + 1) % 50;
        }
        L.at(W.t_tpot, W.c.nt * 50, static_cast<int64_t>(t) * 50 + slot) = v;
    }

    // ---- window policies: decide_window (engine.cpp:350-374) ----
    struct Decision {
        bool fused;
        int gamma;
    };
    DSD_HD Decision decide_window(int64_t i) {
        int32_t d = draft_of(i);
        if (d < 0) return Decision{true, 1};
        int32_t t = RQ(r_target, i);
        switch (S.window_kind) {
            case 0:  // window_static (policies.cpp:55-58)
                return Decision{false, S.gamma};
            case 1: {  // window_dynamic (policies.cpp:60-68)
                int64_t p = pair_of(d, t);
                double a = acceptance_recent(p);
                int32_t& g = L.at(W.p_dyn, W.c.np, p);
                if (a > 0.75 && g < S.gamma_max) {
                    ++g;
                } else if (a < 0.25 && g > S.gamma_min) {
                    --g;
                }
                return Decision{false, g};
            }
            case 2: {  // AWC: extract_features -> predict_gamma -> stabilized_decide
                int64_t p = pair_of(d, t);
                double f[5];
                // features.cpp:5-13
                double q = static_cast<double>(SV(v_open, t)) / static_cast<double>(S.queue_capacity);
                f[0] = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
                f[1] = acceptance_recent(p);
                int32_t rc = L.at(W.p_rtt_cnt, W.c.np, p);
                if (rc == 0) {
                    f[2] = link_rtt(d, t);
                } else {
                    double sum = 0.0;
                    for (int k = 0; k < rc; ++k) sum += L.at(W.p_rtt, W.c.np * 20, p * 20 + k);
                    f[2] = sum / static_cast<double>(rc);
                }
                int32_t tc = L.at(W.t_tcnt, W.c.nt, t);
                if (tc == 0) {
                    f[3] = 0.0;
                } else {
                    double sum = 0.0;
                    for (int k = 0; k < tc; ++k)
                        sum += L.at(W.t_tpot, W.c.nt * 50, static_cast<int64_t>(t) * 50 + k);
                    f[3] = sum / static_cast<double>(tc);
                }
                f[4] = static_cast<double>(L.at(W.p_gprev, W.c.np, p));
                double raw = awc_predict(blob, S, f);
                // stabilized_decide (smoother.cpp:8-37)
                const double gmin = static_cast<double>(S.gamma_min);
                const double gmax = static_cast<double>(S.gamma_max);
                double clamped = raw < gmin ? gmin : (gmax < raw ? gmax : raw);
                uint8_t& init = L.at(W.p_sm_init, W.c.np, p);
                double& ema = L.at(W.p_sm_ema, W.c.np, p);
                int32_t& low = L.at(W.p_sm_low, W.c.np, p);
                uint8_t& fz = L.at(W.p_sm_fused, W.c.np, p);
                const double ema_alpha = 0.4;
                if (!init) {
                    ema = clamped;
                    init = 1;
                } else {
                    ema = ema_alpha * clamped + (1.0 - ema_alpha) * ema;
                }
                if (!fz) {
                    if (ema <= 1.5) {
                        ++low;
                    } else {
                        low = 0;
                    }
                    if (low >= 2) fz = 1;
                } else if (ema > 1.5) {
                    fz = 0;
                    low = 0;
                }
                int g = static_cast<int>(floor(ema + 0.5));
                int gi_min = static_cast<int>(gmin), gi_max = static_cast<int>(gmax);
                g = g < gi_min ? gi_min : (gi_max < g ? gi_max : g);
                if (fz && g <= 1) return Decision{true, 1};
                return Decision{false, g > 1 ? g : 1};
            }
            default:
                return Decision{true, 1};
        }
    }

    // ---- work queues (intrusive lists through item slots) ----
    DSD_HD void push_item(int32_t v, int64_t slot, uint32_t op, int32_t tokens, bool via) {
        SL(s_op, slot) = static_cast<uint8_t>(op | (via ? 4u : 0u));
        SL(s_tok, slot) = tokens;
        SL(s_enq, slot) = now;
        SL(s_next, slot) = -1;
        int32_t& tail = SV(v_qtail, v);
        if (tail < 0) {
            SV(v_qhead, v) = static_cast<int32_t>(slot);
        } else {
            SL(s_next, tail) = static_cast<int32_t>(slot);
        }
        tail = static_cast<int32_t>(slot);
        try_dispatch(v, false);  // push_work (engine.cpp:473-476)
    }

    DSD_HD bool eligible(bool is_draft, uint32_t op, int64_t req) const {
        // item_eligible (engine.cpp:478-483)
        return is_draft || op == kOpPrefill || flag(req, kTpd);
    }

    DSD_HD int64_t work_len(uint32_t op, int64_t slot) const {
        if (op == kOpPrefill) return SL(s_tok, slot);
        int64_t req = slot >> 1;
        return static_cast<int64_t>(RQ(r_output, req)) - RQ(r_tokens, req);
    }

    // try_dispatch (engine.cpp:485-567)
    DSD_HD void try_dispatch(int32_t v, bool window_expired) {
        if (SV(v_busy, v) || SV(v_qhead, v) < 0) return;
        const bool is_draft = v >= T;
        int32_t kind = -1;
        int64_t ncand = 0;
        for (int32_t cur = SV(v_qhead, v); cur >= 0; cur = SL(s_next, cur)) {
            uint32_t op = SL(s_op, cur) & 3u;
            if (!eligible(is_draft, op, cur >> 1)) continue;
            if (kind < 0) kind = static_cast<int32_t>(op);
            if (static_cast<int32_t>(op) != kind) continue;
            ++ncand;
        }
        if (ncand == 0) return;
        const int64_t max_batch = is_draft ? S.draft_max_batch : S.max_batch;
        if (!is_draft && S.batching_window_us > 0 && !window_expired && ncand < max_batch) {
            if (!SV(v_armed, v)) {
                SV(v_armed, v) = 1;
                SV(v_armseq, v) = seq_next;  // stands in for ++window_gen (engine.cpp:512-517)
                schedule(now + S.batching_window_us, info(kEvBatchReady, 0, static_cast<uint32_t>(v)));
            }
            return;
        }
        SV(v_armed, v) = 0;

        const bool lab = !is_draft && S.batching == 1;
        int64_t head_len = 0;
        double band = 0.0;
        int64_t taken = 0;
        int64_t seen = 0;
        int32_t prev = -1;
        int32_t run_tail = -1;
        int32_t tok = 1;
        int64_t ctx = 0;
        for (int32_t cur = SV(v_qhead, v); cur >= 0;) {
            int32_t nxt = SL(s_next, cur);
            uint32_t opv = SL(s_op, cur);
            uint32_t op = opv & 3u;
            bool take = false;
            if (static_cast<int32_t>(op) == kind && eligible(is_draft, op, cur >> 1)) {
                if (!lab) {  // batch_fifo (policies.cpp:30-38)
                    take = taken < max_batch;
                } else {  // batch_lab (policies.cpp:40-53)
                    int64_t wl = work_len(op, cur);
                    if (seen == 0) {
                        head_len = wl;
                        band = S.sim_frac * static_cast<double>(head_len);
                        take = true;
                    } else if (taken < max_batch) {
                        double diff = fabs(static_cast<double>(wl - head_len));
                        take = diff <= band;
                    }
                }
                ++seen;
            }
            if (take) {
                ++taken;
                // unlink from the queue (stable removal)
                if (prev < 0) SV(v_qhead, v) = nxt; else SL(s_next, prev) = nxt;
                if (SV(v_qtail, v) == cur) SV(v_qtail, v) = prev;
                // append to the running batch
                SL(s_next, cur) = -1;
                if (run_tail < 0) SV(v_run, v) = cur; else SL(s_next, run_tail) = cur;
                run_tail = cur;
                // BatchShape (engine.cpp:544-552)
                int32_t t_i = SL(s_tok, cur);
                if (t_i > tok) tok = t_i;
                if (op != kOpPrefill) {
                    int64_t req = cur >> 1;
                    int64_t c = static_cast<int64_t>(RQ(r_prompt, req)) + RQ(r_tokens, req);
                    if (c > ctx) ctx = c;
                }
                if (opv & 4u) {
                    net_wait_total += now - SL(s_enq, cur);
                    ++net_wait_count;
                }
            } else {
                prev = cur;
            }
            cur = nxt;
        }
        // LatencyProfile::predict (profile.cpp:129-151) on the server's grids
        const int32_t* gi = is_draft ? blob_ptr<int32_t>(blob, S.o_dgrid) + 2 * (v - T)
                                     : blob_ptr<int32_t>(blob, S.o_tgrid) + 2 * v;
        const DevGrid* grids = blob_ptr<DevGrid>(blob, S.o_grids);
        double ms;
        if (kind == static_cast<int32_t>(kOpPrefill)) {
            ms = grid_interpolate(blob, grids[gi[0]], static_cast<double>(taken),
                                  static_cast<double>(tok));
        } else if (kind == static_cast<int32_t>(kOpDecode)) {
            ms = grid_interpolate(blob, grids[gi[1]], static_cast<double>(taken),
                                  static_cast<double>(ctx));
            ms *= tok;
        } else {
            ms = grid_interpolate(blob, grids[gi[1]], static_cast<double>(taken) * tok,
                                  static_cast<double>(ctx));
        }
        int64_t lat = llround(ms * 1000.0);
        if (lat < 1) lat = 1;
        SV(v_busy, v) = 1;
        SV(v_busy_us, v) += lat;
        schedule(now + lat, info(kEvComputeDone, 0, static_cast<uint32_t>(v)));
    }

    // ---- request lifecycle ----
    DSD_HD void record_gamma(int64_t i, int g) {
        int32_t& n = RQ(r_ng, i);
        if (W.collect) {
            int64_t o = seqbase + RQ(r_seqoff, i) + n;
            if (o < W.seq_cap) W.seq_gamma[o] = g; else fail = kFailSeq;
        }
        ++n;
    }
    DSD_HD void record_commit(int64_t i, int c) {
        int32_t& n = RQ(r_nc, i);
        if (W.collect) {
            int64_t o = seqbase + RQ(r_seqoff, i) + n;
            if (o < W.seq_cap) W.seq_commit[o] = c; else fail = kFailSeq;
        }
        ++n;
    }

    // activate_next_session (engine.cpp:332-339)
    DSD_HD void activate_next_session(int32_t d) {
        int32_t v = T + d;
        if (SV(v_active, v) >= 0 || SV(v_shead, v) < 0) return;
        int32_t i = SV(v_shead, v);
        SV(v_shead, v) = RQ(r_snext, i);
        if (SV(v_shead, v) < 0) SV(v_stail, v) = -1;
        SV(v_active, v) = i;
        push_item(v, 2 * static_cast<int64_t>(i) + 1, kOpPrefill, RQ(r_prompt, i), false);
    }

    // route (engine.cpp:315-330, policies.cpp:9-28)
    DSD_HD int32_t route() {
        switch (S.routing) {
            case 0:
                return static_cast<int32_t>(routing.below(static_cast<uint64_t>(T)));
            case 1:
                return static_cast<int32_t>(rr_counter++ % static_cast<uint64_t>(T));
            default: {
                int32_t best = 0;
                int32_t bd = SV(v_open, 0);
                for (int32_t t = 1; t < T; ++t) {
                    int32_t dt = SV(v_open, t);
                    if (dt < bd) {
                        best = t;
                        bd = dt;
                    }
                }
                return best;
            }
        }
    }

    // on_arrival (engine.cpp:289-313)
    DSD_HD void on_arrival(int64_t i) {
        RQ(r_arrival, i) = now;
        set_phase(i, kPhRouted);
        int32_t t = route();
        RQ(r_target, i) = t;
        ++SV(v_open, t);  // MetricsCollector::on_route
        if (first_arrival < 0 || now < first_arrival) first_arrival = now;
        set_phase(i, kPhQueuedPrefill);
        if (S.fused_everything) {
            set_flag(i, kFused, true);
            push_item(t, 2 * i, kOpPrefill, RQ(r_prompt, i), false);
        } else {
            int32_t d = RQ(r_drafter, i);
            int32_t v = T + d;
            RQ(r_snext, i) = -1;
            int32_t tail = SV(v_stail, v);
            if (tail < 0) SV(v_shead, v) = static_cast<int32_t>(i); else RQ(r_snext, tail) = static_cast<int32_t>(i);
            SV(v_stail, v) = static_cast<int32_t>(i);
            activate_next_session(d);
            int64_t delay = net_delay(d, t);
            schedule(now + delay, info(kEvNetArrive, kMsgPrompt, static_cast<uint32_t>(i)));
        }
    }

    // begin_iteration (engine.cpp:383-404)
    DSD_HD void begin_iteration(int64_t i, Decision dec) {
        if (phase(i) == kPhDone) return;
        int32_t d = draft_of(i);
        int32_t t = RQ(r_target, i);
        if (d >= 0 && t >= 0) on_gamma_chosen(d, t, dec.fused ? 1 : dec.gamma);
        int32_t ctx = RQ(r_prompt, i) + RQ(r_tokens, i);
        (void)ctx;
        if (dec.fused) {
            set_flag(i, kFused, true);
            record_gamma(i, 0);
            push_item(t, 2 * i + 1, kOpDecode, 1, false);
        } else {
            set_flag(i, kFused, false);
            record_gamma(i, dec.gamma);
            RQ(r_pgamma, i) = dec.gamma;
            set_phase(i, kPhSpeculating);
            push_item(T + d, 2 * i + 1, kOpDecode, dec.gamma, false);
        }
    }

    // finish_request (engine.cpp:449-468) + MetricsCollector::add_record
    DSD_HD void finish_request(int64_t i) {
        RQ(r_done, i) = now;
        if (RQ(r_first, i) < 0) RQ(r_first, i) = now;
        set_phase(i, kPhDone);
        int32_t t = RQ(r_target, i);
        --SV(v_open, t);
        int32_t out = RQ(r_output, i);
        if (out >= 2 && S.pair_stats) {
            double tpot = (static_cast<double>(now - RQ(r_first, i)) / 1000.0) /
                          static_cast<double>(out - 1);
            push_tpot(t, tpot);
        }
        if (now > last_completion) last_completion = now;
        ++completed;
        int32_t d = draft_of(i);
        if (d >= 0) {
            int32_t v = T + d;
            if (SV(v_active, v) == static_cast<int32_t>(i)) {
                SV(v_active, v) = -1;
                activate_next_session(d);
            }
        }
    }

    // commit_tokens (engine.cpp:437-447)
    DSD_HD void commit_tokens(int64_t i, int32_t raw) {
        int32_t remaining = RQ(r_output, i) - RQ(r_tokens, i);
        int32_t c = raw < remaining ? raw : remaining;
        RQ(r_tokens, i) += c;
        record_commit(i, c);
        if (RQ(r_first, i) < 0) RQ(r_first, i) = now;
        if (RQ(r_tokens, i) >= RQ(r_output, i)) finish_request(i);
    }

    // consume_acceptance (engine.cpp:17-32) on the packed bits
    DSD_HD void consume_acceptance(int64_t i, int gamma, int& accepted, int& consumed) {
        const uint64_t* bits = W.bits + rep * W.c.bw + RQ(r_bitoff, i);
        const int32_t nb = RQ(r_nbits, i);
        int32_t cur = RQ(r_cursor, i);
        accepted = 0;
        consumed = 0;
        while (consumed < gamma) {
            uint64_t b = (bits[cur >> 6] >> (cur & 63)) & 1u;
            cur = cur + 1 == nb ? 0 : cur + 1;
            ++consumed;
            if (b) {
                ++accepted;
            } else {
                break;
            }
        }
        RQ(r_cursor, i) = cur;
    }

    DSD_HD void send_proposal(int64_t i) {  // engine.cpp:591-597
        set_phase(i, kPhInFlightToTarget);
        int64_t dl = net_delay(RQ(r_drafter, i), RQ(r_target, i));
        RQ(r_outd, i) = dl;
        schedule(now + dl, info(kEvNetArrive, kMsgProposal, static_cast<uint32_t>(i)));
    }

    // on_target_item_done (engine.cpp:599-646)
    DSD_HD void on_target_item_done(int64_t i, uint32_t op, int32_t tokens) {
        if (op == kOpPrefill) {
            set_flag(i, kTpd, true);
            if (RQ(r_output, i) == 0) {
                if (phase(i) != kPhDone) finish_request(i);
                return;
            }
            if (flag(i, kFused) && S.fused_everything) begin_iteration(i, Decision{true, 1});
        } else if (op == kOpVerify) {
            int acc, cons;
            consume_acceptance(i, tokens, acc, cons);
            RQ(r_lcr, i) = acc + 1;
            RQ(r_prop, i) += cons;
            RQ(r_acc, i) += acc;
            int32_t d = RQ(r_drafter, i), t = RQ(r_target, i);
            on_verify(d, t, cons, acc);
            int64_t bd = net_delay(d, t);
            RQ(r_backd, i) = bd;
            set_phase(i, kPhInFlightToDraft);
            schedule(now + bd, info(kEvNetArrive, kMsgResult, static_cast<uint32_t>(i)));
        } else {
            commit_tokens(i, 1);
            if (phase(i) == kPhDone) return;
            if (S.fused_everything || draft_of(i) < 0) {
                begin_iteration(i, Decision{true, 1});
            } else {
                begin_iteration(i, decide_window(i));
            }
        }
    }

    // on_compute_done (engine.cpp:569-589)
    DSD_HD void on_compute_done(int32_t v) {
        SV(v_busy, v) = 0;
        int32_t cur = SV(v_run, v);
        SV(v_run, v) = -1;
        const bool is_draft = v >= T;
        while (cur >= 0) {
            int32_t nxt = SL(s_next, cur);
            uint32_t op = SL(s_op, cur) & 3u;
            int32_t tok = SL(s_tok, cur);
            int64_t i = cur >> 1;
            if (is_draft) {
                if (op == kOpPrefill) {
                    set_flag(i, kDpd, true);
                    if (RQ(r_output, i) > 0)
                        schedule(now, info(kEvIterStart, 0, static_cast<uint32_t>(i)));
                } else {
                    send_proposal(i);
                }
            } else {
                on_target_item_done(i, op, tok);
            }
            cur = nxt;
        }
        try_dispatch(v, false);
    }

    // on_net_arrive (engine.cpp:406-435)
    DSD_HD void on_net_arrive(uint32_t msg, int64_t i) {
        int32_t t = RQ(r_target, i);
        if (msg == kMsgPrompt) {
            push_item(t, 2 * i, kOpPrefill, RQ(r_prompt, i), true);
        } else if (msg == kMsgProposal) {
            set_phase(i, kPhVerifying);
            push_item(t, 2 * i + 1, kOpVerify, RQ(r_pgamma, i), true);
        } else {
            if (S.pair_stats) {
                on_rtt_sample(RQ(r_drafter, i), t,
                              static_cast<double>(RQ(r_outd, i) + RQ(r_backd, i)) / 1000.0);
            }
            commit_tokens(i, RQ(r_lcr, i));
            if (phase(i) != kPhDone) schedule(now, info(kEvIterStart, 0, static_cast<uint32_t>(i)));
        }
    }

    // ---- setup + SimKernel::run_until (event_queue.cpp:28-42) ----
    DSD_HD void init() {
        const uint64_t seed = W.rep_seed[rep];
        routing.seed(seed, kLabelRouting);
        jitter.seed(seed, kLabelJitter);
        N = (S.workload == 0) ? S.n_requests : S.tr_n;
        seq_next = static_cast<uint32_t>(N);
        if (W.collect) seqbase = W.rep_seqbase[rep];
        for (int64_t i = 0; i < N; ++i) {
            RQ(r_flags, i) = 0;
            RQ(r_target, i) = -1;
            RQ(r_tokens, i) = 0;
            RQ(r_cursor, i) = 0;
            RQ(r_first, i) = -1;
            RQ(r_done, i) = -1;
            RQ(r_pgamma, i) = 0;
            RQ(r_lcr, i) = 0;
            RQ(r_outd, i) = 0;
            RQ(r_backd, i) = 0;
            RQ(r_prop, i) = 0;
            RQ(r_acc, i) = 0;
            RQ(r_ng, i) = 0;
            RQ(r_nc, i) = 0;
            RQ(r_snext, i) = -1;
        }
        for (int32_t v = 0; v < T + D; ++v) {
            SV(v_qhead, v) = -1;
            SV(v_qtail, v) = -1;
            SV(v_run, v) = -1;
            SV(v_busy, v) = 0;
            SV(v_armed, v) = 0;
            SV(v_armseq, v) = 0;
            SV(v_busy_us, v) = 0;
            SV(v_active, v) = -1;
            SV(v_shead, v) = -1;
            SV(v_stail, v) = -1;
            SV(v_open, v) = 0;
        }
        if (S.pair_stats) {
            for (int32_t t = 0; t < T; ++t) {
                L.at(W.t_tcnt, W.c.nt, t) = 0;
                L.at(W.t_tpos, W.c.nt, t) = 0;
            }
            int64_t np = static_cast<int64_t>(T) * D;
            for (int64_t p = 0; p < np; ++p) {
                L.at(W.p_acc_cnt, W.c.np, p) = 0;
                L.at(W.p_acc_pos, W.c.np, p) = 0;
                L.at(W.p_rtt_cnt, W.c.np, p) = 0;
                L.at(W.p_rtt_pos, W.c.np, p) = 0;
                L.at(W.p_gprev, W.c.np, p) = S.gamma;
                L.at(W.p_dyn, W.c.np, p) = S.gamma;
                L.at(W.p_sm_init, W.c.np, p) = 0;
                L.at(W.p_sm_ema, W.c.np, p) = 0.0;
                L.at(W.p_sm_low, W.c.np, p) = 0;
                L.at(W.p_sm_fused, W.c.np, p) = 0;
            }
        }
    }

    DSD_HD int64_t arrival_index(int64_t k) const {
        if (S.has_order) return blob_ptr<int64_t>(blob, S.o_tr_order)[k];
        return k;
    }

    DSD_HD void run() {
        init();
        for (;;) {
            if (fail) break;
            const bool have_arr = next_arr < N;
            int64_t ai = 0, ta = 0;
            if (have_arr) {
                ai = arrival_index(next_arr);
                ta = RQ(r_arrival, ai);
            }
            if (heap_n == 0 && !have_arr) break;
            // arrivals hold seq 0..N-1: they win every time tie
            if (have_arr && (heap_n == 0 || ta <= L.at(W.h_time, W.c.hc, 0))) {
                ++next_arr;
                now = ta;
                ++processed;
                on_arrival(ai);
                continue;
            }
            const int64_t t = L.at(W.h_time, W.c.hc, 0);
            const uint64_t key = L.at(W.h_key, W.c.hc, 0);
            heap_pop();
            now = t;
            ++processed;
            const uint32_t inf = static_cast<uint32_t>(key);
            const uint32_t kind = inf & 7u;
            const uint32_t msg = (inf >> 3) & 3u;
            const uint32_t id = inf >> 5;
            switch (kind) {
                case kEvIterStart:
                    begin_iteration(id, decide_window(id));
                    break;
                case kEvNetArrive:
                    on_net_arrive(msg, id);
                    break;
                case kEvComputeDone:
                    on_compute_done(static_cast<int32_t>(id));
                    break;
                case kEvBatchReady: {
                    int32_t v = static_cast<int32_t>(id);
                    if (SV(v_armed, v) && SV(v_armseq, v) == static_cast<uint32_t>(key >> 32)) {
                        SV(v_armed, v) = 0;
                        try_dispatch(v, true);
                    }
                    break;
                }
                default:
                    break;
            }
        }
        finish();
    }

    // Engine::finish (engine.cpp:648-669) + aggregate_run (runner.cpp:153-169)
    DSD_HD void finish() {
        DevSummary s;
        s.events_processed = processed;
        s.end_time_us = now;
        s.completed = completed;
        s.first_arrival_us = first_arrival;
        s.last_completion_us = last_completion;
        s.net_queue_wait_total_us = net_wait_total;
        s.net_queue_wait_count = net_wait_count;
        s.n_requests = N;
        s.has_duration = (completed > 0 && last_completion > first_arrival) ? 1 : 0;
        s.throughput_rps = 0.0;
        if (s.has_duration) {
            int64_t dur = last_completion - first_arrival;
            s.throughput_rps = static_cast<double>(completed) / (static_cast<double>(dur) / 1e6);
        }
        double ttft = 0.0, tpot = 0.0;
        int64_t n_tpot = 0, n_rec = 0;
        for (int64_t i = 0; i < N; ++i) {  // records sorted by request id
            int64_t done = RQ(r_done, i);
            if (done < 0) continue;
            ++n_rec;
            int64_t first = RQ(r_first, i);
            ttft += static_cast<double>(first - RQ(r_arrival, i)) / 1000.0;
            int32_t out = RQ(r_output, i);
            if (out >= 2) {
                tpot += (static_cast<double>(done - first) / 1000.0) / static_cast<double>(out - 1);
                ++n_tpot;
            }
        }
        s.mean_ttft_ms = n_rec > 0 ? ttft / static_cast<double>(n_rec) : 0.0;
        s.mean_tpot_ms = n_tpot > 0 ? tpot / static_cast<double>(n_tpot) : 0.0;
        s.status = fail ? 3 : 0;
        W.summary[rep] = s;
        W.fail[rep] = fail;
    }
#undef RQ
#undef SL
#undef SV
};

// ---------------------------------------------------------------------------
// workload staging: generate_synthetic (trace.cpp:145-187), trace copy, and the
// engine's poisson re-sampling (engine.cpp:224-238).  One thread per replica.
// ---------------------------------------------------------------------------
DSD_HD void stage_workload(const Workspace& W, int64_t rep) {
    const DevScenario& S = W.scen[W.rep_scen[rep]];
    const char* blob = W.blob;
    Lane L;
    L.w = rep / kLanes;
    L.lane = static_cast<int>(rep % kLanes);
    const int64_t nr = W.c.nr;
    uint64_t* bits = W.bits + rep * W.c.bw;
    int64_t word = 0;
    int64_t lsum = 0;
    if (S.workload == 0) {
        const uint64_t gseed = W.rep_gen_seed[rep];
        Rng arrivals, bitrng, lengths, drafter;
        arrivals.seed(gseed, kLabelArrivals);
        bitrng.seed(gseed, kLabelAcceptBits);
        lengths.seed(gseed, kLabelLengths);
        drafter.seed(gseed, kLabelDrafter);
        double clock_ms = 0.0;
        const double alpha = S.alpha;
        for (int64_t n = 0; n < S.n_requests; ++n) {
            clock_ms += arrivals.exponential(S.mean_gap_ms);
            L.at(W.r_arrival, nr, n) = llround(clock_ms * 1000.0);
            int64_t p = llround(lengths.lognormal(S.p_mu, S.p_sigma));
            p = p < 1 ? 1 : (S.p_cap < p ? S.p_cap : p);
            int64_t o = llround(lengths.lognormal(S.o_mu, S.o_sigma));
            o = o < 1 ? 1 : (S.o_cap < o ? S.o_cap : o);
            L.at(W.r_prompt, nr, n) = static_cast<int32_t>(p);
            L.at(W.r_output, nr, n) = static_cast<int32_t>(o);
            L.at(W.r_drafter, nr, n) =
                static_cast<int32_t>(drafter.below(static_cast<uint64_t>(S.gen_n_drafts)));
            L.at(W.r_bitoff, nr, n) = static_cast<int32_t>(word);
            L.at(W.r_nbits, nr, n) = static_cast<int32_t>(o);
            L.at(W.r_seqoff, nr, n) = lsum;
            lsum += o;
            for (int64_t k = 0; k < o; k += 64) {
                int64_t m = o - k < 64 ? o - k : 64;
                uint64_t acc = 0;
                for (int64_t j = 0; j < m; ++j) {
                    uint64_t b = bitrng.unit() < alpha ? 1u : 0u;  // bernoulli (rng.cpp:64-66)
                    acc |= b << j;
                }
                bits[word++] = acc;
            }
        }
    } else {
        const int64_t* tp = blob_ptr<int64_t>(blob, S.o_tr_prompt);
        const int64_t* to = blob_ptr<int64_t>(blob, S.o_tr_output);
        const int64_t* ta = blob_ptr<int64_t>(blob, S.o_tr_arrival);
        const int64_t* td = blob_ptr<int64_t>(blob, S.o_tr_drafter);
        const int64_t* tb = blob_ptr<int64_t>(blob, S.o_tr_bitoff);
        const uint8_t* tbits = blob_ptr<uint8_t>(blob, S.o_tr_bits);
        Rng arrivals;
        arrivals.seed(W.rep_seed[rep], kLabelArrivals);
        double clock_ms = 0.0;
        for (int64_t n = 0; n < S.tr_n; ++n) {
            if (S.workload == 2) {
                clock_ms += arrivals.exponential(1000.0 / S.rate_rps);
                L.at(W.r_arrival, nr, n) = llround(clock_ms * 1000.0);
            } else {
                L.at(W.r_arrival, nr, n) = ta[n];
            }
            L.at(W.r_prompt, nr, n) = static_cast<int32_t>(tp[n]);
            L.at(W.r_output, nr, n) = static_cast<int32_t>(to[n]);
            L.at(W.r_drafter, nr, n) = static_cast<int32_t>(td[n]);
            L.at(W.r_bitoff, nr, n) = static_cast<int32_t>(word);
            const int64_t nb = tb[n + 1] - tb[n];
            L.at(W.r_nbits, nr, n) = static_cast<int32_t>(nb);
            L.at(W.r_seqoff, nr, n) = lsum;
            lsum += to[n];
            for (int64_t k = 0; k < nb; k += 64) {
                int64_t m = nb - k < 64 ? nb - k : 64;
                uint64_t acc = 0;
                for (int64_t j = 0; j < m; ++j)
                    acc |= static_cast<uint64_t>(tbits[tb[n] + k + j] & 1u) << j;
                bits[word++] = acc;
            }
        }
    }
}

}  // namespace dsd
