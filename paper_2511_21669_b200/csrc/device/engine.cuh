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
//  * replica scalars (clock, seq counter, RNG states, totals, the action
//    stack) live in registers for the whole run; per-request state is one
//    128-byte record per request; server state and the event heap are
//    warp-interleaved SoA (a warp's 32 replicas read one row per slot).
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

#ifndef DSD_SPEC_STACK
#define DSD_SPEC_STACK 2
#endif
// action-stack depth of the specialised kernel (2..4)
constexpr int kSpecStack = DSD_SPEC_STACK;

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

// Same result as grid_interpolate(blob, g, qb, qc) for integer queries, from
// the host-built segment tables: two table loads instead of two binary
// searches and two divisions.
DSD_HD double grid_interpolate_int(const char* blob, const DevGrid& g, int64_t qb, int64_t qc) {
    const AxisSeg sb = blob_ptr<AxisSeg>(blob, g.o_btab)[qb < g.nbt ? qb : g.nbt - 1];
    const AxisSeg sc = blob_ptr<AxisSeg>(blob, g.o_ctab)[qc < g.nct ? qc : g.nct - 1];
    const double* v = blob_ptr<double>(blob, g.o_vals);
    const int n = g.nc;
    const double tb = sb.t, tc = sc.t;
    double r = (1.0 - tb) * (1.0 - tc) * v[sb.lo * n + sc.lo] + (1.0 - tb) * tc * v[sb.lo * n + sc.hi] +
               tb * (1.0 - tc) * v[sb.hi * n + sc.lo] + tb * tc * v[sb.hi * n + sc.hi];
    return r * g.calibration;
}

// General (non-integer or table-less) query; out of line, it is cold.
DSD_HD_NOINLINE double grid_interpolate(const char* blob, const DevGrid& g, double batch, double context) {
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

// LatencyProfile::predict (profile.cpp:129-151) on one grid for an integer
// query, times `mult` tokens when mult > 0 (decode), as ms_to_us with the
// engine's 1 us floor (engine.cpp:553-557)
DSD_HD int64_t grid_latency_us(const char* blob, const DevGrid& g, int64_t qb, int64_t qc, int32_t mult) {
    double ms = g.o_btab >= 0 && g.o_ctab >= 0
                    ? grid_interpolate_int(blob, g, qb, qc)
                    : grid_interpolate(blob, g, static_cast<double>(qb), static_cast<double>(qc));
    if (mult > 0) ms *= mult;
    const int64_t lat = llround(ms * 1000.0);
    return lat < 1 ? 1 : lat;
}

// A session latency table of the specialised kernel (Workspace::spec_lat):
// draft decode grid, verify grid, gamma (>= 1), contexts [0, n), and its
// element offset (status word, pad, then n {draft, verify} pairs).
struct SpecLatJob {
    int64_t o_gd, o_gt, base;
    int32_t g1, n;
};
constexpr int32_t kSpecLatMax = 1 << 28;  // entries must stay below (32-bit relative times)

// ---------------------------------------------------------------------------
// AWC: FeatureNormalizer::transform + WcDnn::forward (mlp.cpp:83-97,163-176)
// with Backend::matvec in the AVX2 summation order the reference auto-selects
// on AVX2 hosts (kernels_avx2.cpp:17-40, kernels_dispatch.cpp:21-26).
//
// The blob holds the network in a TRANSPOSED flat layout (pack.cpp,
// awc_transpose): for each weight matrix, element (row r, column c) at
// [c * rows + r], biases and the head as in the reference's layout
// (mlp.cpp:20-48).  A warp evaluates a network cooperatively - lane l owns
// output rows l, l + 32 - so at every step of a dot product the 32 lanes read
// 32 consecutive weights (one 256-byte line, conflict-free in shared memory)
// while the input element is a broadcast.  Each row is still summed in the
// AVX2 order: 4 strided lane sums, (l0 + l2) + (l1 + l3), then the tail.
// ---------------------------------------------------------------------------
#ifndef DSD_AWC_FIXED
#define DSD_AWC_FIXED 0
#endif
// one output row r of a transposed [cols][rows] matrix against x
template <typename P>
DSD_HD double avx2_dot_t(const P* wt, int rows, int r, const double* x, int cols) {
    const int tail = cols & ~3;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = 0;
    for (; c < tail; c += 4) {
        a0 = a0 + wt[c * rows + r] * x[c];
        a1 = a1 + wt[(c + 1) * rows + r] * x[c + 1];
        a2 = a2 + wt[(c + 2) * rows + r] * x[c + 2];
        a3 = a3 + wt[(c + 3) * rows + r] * x[c + 3];
    }
    double s = (a0 + a2) + (a1 + a3);  // hsum: lo+hi then unpackhi (kernels_avx2.cpp:17-23)
    for (; c < cols; ++c) s += wt[c * rows + r] * x[c];
    return s;
}
// the same for compile-time widths (the trained shape): fully unrolled
template <int R, int C>
DSD_HD double avx2_dot_t_fixed(const double* wt, int r, const double* x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int c = 0; c < (C & ~3); c += 4) {
        a0 = a0 + wt[c * R + r] * x[c];
        a1 = a1 + wt[(c + 1) * R + r] * x[c + 1];
        a2 = a2 + wt[(c + 2) * R + r] * x[c + 2];
        a3 = a3 + wt[(c + 3) * R + r] * x[c + 3];
    }
    double s = (a0 + a2) + (a1 + a3);
#pragma unroll
    for (int c = C & ~3; c < C; ++c) s += wt[c * R + r] * x[c];
    return s;
}
// the WC-DNN shape the reference trains (TrainHyper: 5 features, 64 hidden)
constexpr int kAwcH = 64, kAwcI = 5;

// FeatureNormalizer::transform (mlp.cpp:163-170): raw features -> model input
DSD_HD void awc_normalize(const DevScenario& S, const double raw[5], double x[5]) {
    for (int f = 0; f < 5; ++f) {
        double v = S.awc_log[f] ? DSD_LOG1P(raw[f]) : raw[f];
        double span = S.awc_hi[f] - S.awc_lo[f];
        x[f] = span > 0.0 ? (v - S.awc_lo[f]) / span : 0.0;
    }
}

// Per-warp scratch of the cooperative AWC evaluation (shared memory): the
// requesting lanes' model inputs and results, the request flags, and the
// hidden vectors of the network being evaluated.
struct AwcWarpScratch {
    double x[kLanes][8];
    double raw[kLanes];
    double hv[kMaxHidden], sv[kMaxHidden];
    int32_t req[kLanes];
};

#ifdef __CUDACC__
// WcDnn::forward (mlp.cpp:83-97) of one network on a normalised input x,
// evaluated by the whole warp from the transposed weights `pt` (shared
// memory when the block staged them, else the blob); every lane of the warp
// must call it (converged).  Returns the raw prediction on every lane.
__device__ __forceinline__ double awc_forward_warp(const double* pt, const DevScenario* S, const double* x,
                                                   AwcWarpScratch* sc) {
    const int lane = threadIdx.x & (kLanes - 1);
    const int H = S->awc_hidden, I = S->awc_input;
    if (DSD_AWC_FIXED && H == kAwcH && I == kAwcI) {  // compile-time widths (the trained shape)
        constexpr int FH = kAwcH, FI = kAwcI;
#pragma unroll
        for (int k = 0; k < FH / kLanes; ++k) {
            const int r = lane + k * kLanes;
            sc->hv[r] = pt[FH * FI + r] + avx2_dot_t_fixed<FH, FI>(pt, r, x);
        }
        __syncwarp();
        int off = FH * FI + FH;
        for (int b = 0; b < S->awc_blocks; ++b) {
            const double* w1 = pt + off;
            const double* b1 = w1 + FH * FH;
            const double* w2 = b1 + FH;
            const double* b2 = w2 + FH * FH;
#pragma unroll
            for (int k = 0; k < FH / kLanes; ++k) {
                const int r = lane + k * kLanes;
                const double u = b1[r] + avx2_dot_t_fixed<FH, FH>(w1, r, sc->hv);
                const double sg = 1.0 / (1.0 + DSD_EXP(-u));  // kernels::silu (kernels_scalar.cpp:65-70)
                sc->sv[r] = u * sg;
            }
            __syncwarp();
            // (the products read sv; each lane updates only its own rows of hv)
#pragma unroll
            for (int k = 0; k < FH / kLanes; ++k) {
                const int r = lane + k * kLanes;
                sc->hv[r] += b2[r] + avx2_dot_t_fixed<FH, FH>(w2, r, sc->sv);
            }
            __syncwarp();
            off += 2 * FH * FH + 2 * FH;
        }
        double out = 0.0;
        if (lane == 0) {
            const double* w_out = pt + off;
            out = w_out[FH];  // b_out, then the sequential head (mlp.cpp:93-95)
            for (int i = 0; i < FH; ++i) out += w_out[i] * sc->hv[i];
        }
        __syncwarp();
        return __shfl_sync(0xffffffffu, out, 0);
    }
    for (int r = lane; r < H; r += kLanes) sc->hv[r] = pt[H * I + r] + avx2_dot_t(pt, H, r, x, I);
    __syncwarp();
    int off = H * I + H;
    for (int b = 0; b < S->awc_blocks; ++b) {
        const double* w1 = pt + off;
        const double* b1 = w1 + H * H;
        const double* w2 = b1 + H;
        const double* b2 = w2 + H * H;
        for (int r = lane; r < H; r += kLanes) {
            const double u = b1[r] + avx2_dot_t(w1, H, r, sc->hv, H);
            const double sg = 1.0 / (1.0 + DSD_EXP(-u));  // kernels::silu (kernels_scalar.cpp:65-70)
            sc->sv[r] = u * sg;
        }
        __syncwarp();
        for (int r = lane; r < H; r += kLanes) sc->hv[r] += b2[r] + avx2_dot_t(w2, H, r, sc->sv, H);
        __syncwarp();
        off += 2 * H * H + 2 * H;
    }
    double out = 0.0;
    if (lane == 0) {
        const double* w_out = pt + off;
        out = w_out[H];  // b_out, then the sequential head (mlp.cpp:93-95)
        for (int i = 0; i < H; ++i) out += w_out[i] * sc->hv[i];
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, out, 0);
}

// Serves every pending AWC request of the warp: one network at a time, each
// evaluated by all 32 lanes (idle and finished lanes included).  `staged`:
// the block's shared-memory copy of the weights at blob offset staged_off
// (or null); other models are read from the blob.
__device__ __forceinline__ void awc_serve_warp(const char* blob, const DevScenario* my_scen, AwcWarpScratch* sc,
                                               const double* staged, int64_t staged_off) {
    const int lane = threadIdx.x & (kLanes - 1);
    unsigned pending = __ballot_sync(0xffffffffu, sc->req[lane] != 0);
    while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        const DevScenario* S = reinterpret_cast<const DevScenario*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_scen), src));
        const double* pt = S->o_awc_params == staged_off && staged ? staged : blob_ptr<double>(blob, S->o_awc_params);
        const double raw = awc_forward_warp(pt, S, sc->x[src], sc);
        if (lane == src) {
            sc->raw[lane] = raw;
            sc->req[lane] = 0;
        }
        __syncwarp();
    }
}
#endif

// ---------------------------------------------------------------------------
// pair / target metric rings (MetricsCollector, metrics.cpp:40-128) and the
// AWC feature vector, as free functions over the workspace: the feature code
// runs out of line (AWC decisions and the feature probe only), which keeps it
// out of the event loop's instruction footprint
// ---------------------------------------------------------------------------
// warp-interleaved per-replica arrays in HBM (pair stats, busy export)
template <typename U>
DSD_HD U& il_at(U* base, int32_t rep, int64_t cap, int64_t idx) {
    return base[((static_cast<int64_t>(rep) >> 5) * cap + idx) * kLanes + (rep & 31)];
}

// acceptance_recent (metrics.cpp:93-108): ring sums in storage order
DSD_HD double acceptance_recent_at(const Workspace& W, int32_t rep, int64_t p) {
    int32_t cnt = il_at(W.p_acc_cnt, rep, W.c.np, p);
    int64_t ex = 0, ac = 0;
    for (int k = 0; k < cnt; ++k) {
        ex += il_at(W.p_acc_ex, rep, W.c.np * 20, p * 20 + k);
        ac += il_at(W.p_acc_ac, rep, W.c.np * 20, p * 20 + k);
    }
    if (ex == 0) return 0.5;
    return static_cast<double>(ac) / static_cast<double>(ex);
}

// extract_features (features.cpp:5-13) for pair p = (d, t): queue pressure
// (open requests of the target / queue capacity, clamped), recent
// acceptance, recent RTT (the link's nominal RTT before any sample), recent
// TPOT of the target, the pair's previous window
DSD_HD_NOINLINE void extract_features(const Workspace& W, int32_t rep, int64_t p, int32_t t, int32_t open_t,
                                      int32_t queue_capacity, double link_rtt_ms, double* f) {
    double q = static_cast<double>(open_t) / static_cast<double>(queue_capacity);
    f[0] = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
    f[1] = acceptance_recent_at(W, rep, p);
    int32_t rc = il_at(W.p_rtt_cnt, rep, W.c.np, p);
    if (rc == 0) {
        f[2] = link_rtt_ms;
    } else {
        double sum = 0.0;
        for (int k = 0; k < rc; ++k) sum += il_at(W.p_rtt, rep, W.c.np * 20, p * 20 + k);
        f[2] = sum / static_cast<double>(rc);
    }
    int32_t tc = il_at(W.t_tcnt, rep, W.c.nt, t);
    if (tc == 0) {
        f[3] = 0.0;
    } else {
        double sum = 0.0;
        for (int k = 0; k < tc; ++k) sum += il_at(W.t_tpot, rep, W.c.nt * 50, static_cast<int64_t>(t) * 50 + k);
        f[3] = sum / static_cast<double>(tc);
    }
    f[4] = static_cast<double>(il_at(W.p_gprev, rep, W.c.np, p));
}

// EngineOptions::feature_probe (engine.cpp:376-381, 660-664) plus the
// chosen-window tally eval_policy_on_scenarios reads from the records
// (dataset.cpp:344-351, fused counts as 1): per-replica sums in
// W.probe[rep][kProbeFields], accumulated in event order.  p < 0: the
// request has no draft server (no feature sample).
DSD_HD_NOINLINE void probe_iteration(const Workspace& W, int32_t rep, int64_t p, int32_t t, int32_t open_t,
                                     int32_t queue_capacity, double link_rtt_ms, int32_t chosen) {
    double* pr = W.probe + static_cast<int64_t>(rep) * kProbeFields;
    if (p >= 0) {
        double f[5];
        extract_features(W, rep, p, t, open_t, queue_capacity, link_rtt_ms, f);
        for (int k = 0; k < 5; ++k) pr[k] += f[k];
        pr[5] += 1.0;
    }
    pr[6] += static_cast<double>(chosen);
    pr[7] += 1.0;
}

// EngineOptions::collect_event_log: one log_transition (engine.cpp:213-219)
// and one busy interval (engine.cpp:563-564), appended to the replica's
// region in event order; out of line - only logged runs take these calls.
// A full region fails the replica like the sequence arena (kFailSeq).
DSD_HD_NOINLINE int32_t elog_append(const Workspace& W, int32_t rep, int64_t now, int64_t i, uint32_t phase,
                                    uint32_t detail, int32_t d, int32_t t) {
    int64_t& n = W.elog_n[rep];
    if (n >= W.elog_cap) return kFailSeq;
    ElogRec& e = W.elog[static_cast<int64_t>(rep) * W.elog_cap + n++];
    e.t = now;
    e.req = static_cast<int32_t>(i);
    e.draft = d;
    e.target = t;
    e.phase = static_cast<uint8_t>(phase);
    e.detail = static_cast<uint8_t>(detail);
    return kFailNone;
}
DSD_HD_NOINLINE int32_t busy_append(const Workspace& W, int32_t rep, int32_t server, int64_t start, int64_t end) {
    int64_t& n = W.busy_n[rep];
    if (n >= W.busy_cap) return kFailSeq;
    BusyRec& b = W.busy_iv[static_cast<int64_t>(rep) * W.busy_cap + n++];
    b.start = start;
    b.end = end;
    b.server = server;
    b.pad = 0;
    return kFailNone;
}

// ---------------------------------------------------------------------------
// the engine
//
// Control flow is continuation-passing: the reference's nested call chains
// (push_work -> try_dispatch, finish_request -> activate_next_session ->
// push_work, on_compute_done's per-item loop, ...) become small actions on a
// 4-deep register stack that the main loop pops before it takes the next
// event.  Every handler body therefore exists exactly once in the binary
// (the fully inlined direct-call version was ~28K SASS instructions and
// stalled on instruction fetch), and all schedule() calls still happen in the
// reference's order, so seq numbers - and with them the (time, seq) event
// order - are identical.  The deepest chain (compute-done item -> finish ->
// activate -> dispatch) needs 3 stack slots.
// ---------------------------------------------------------------------------
// Kinds are numbered in the order they follow each other inside one event's
// chain (pop -> handler -> ... -> dispatch -> send prompt), so the kernel's
// cyclic sweep over kinds usually carries a lane through a whole event per sweep.
enum : uint32_t {
    kActPop = 0,          // pop the next event (stack empty)
    kActArrival = 1,      // on_arrival(i)                     arg = i
    kActNetPrompt = 2,    // NetArrive handlers, by message:   arg = i
    kActNetProposal = 3,  //   kActNetPrompt + kMsg*
    kActNetResult = 4,
    kActBegin = 5,        // [decide_window] + begin_iteration  arg = i*2 + decide
    kActComputeDone = 6,  // on_compute_done(v)                arg = v
    kActItem = 7,         // one item of a finished batch      arg = slot
    kActFinish = 8,       // finish_request(i)                 arg = i
    kActActivate = 9,     // activate_next_session(d)          arg = d
    kActDispatch = 10,    // try_dispatch(v, expired)          arg = v*2 + expired
    kActSendPrompt = 11,  // ship the prompt to the verifier   arg = i
    kActBeginAwc = 12,    // AWC decision served -> begin       arg = i
    kActKinds = 13,
    kActNone = 15         // replica finished
};
// Actions are kind | arg << 4 (args < 2^28: requests < 2^26, slots < 2^27).

// Step kinds at which a lane's continuation chain stops and waits for the
// warp's next vote.  The selected lanes run their chain (popping events as
// they go) until they reach one of these, so the warp executes each of the
// frequent, costly handlers - dispatch, iteration start, batch items, the
// proposal and result arrivals - for all lanes that have it pending at once,
// while the cheap or rare steps (pops, arrivals, prompt shipping, compute
// completion, finish, activation) ride along inside the chains.  Making a
// rare kind a barrier starves it: the vote picks the kind most lanes have
// pending.  Measured on the C5 sweep (B200): {pop, dispatch} 170 ms, this set
// 85 ms, every kind 210 ms.
#ifndef DSD_BARRIER_KINDS
#define DSD_BARRIER_KINDS                                                                            \
    ((1u << kActDispatch) | (1u << kActBegin) | (1u << kActItem) | (1u << kActNetProposal) |         \
     (1u << kActNetResult) | (1u << kActBeginAwc) | (1u << kActNone))
#endif
constexpr uint32_t kBarrierKinds = DSD_BARRIER_KINDS;
// The generic shared-memory kernel (up to 4 servers; solo mode) and every AWC
// kernel: the session entry and the AWC continuation only.  Measured (B200)
// against the general set: a 8,192-replica dynamic-window sweep 57.1 -> 54.8
// ms, the 768-replica AWC sweep 157 -> 153 ms, 4,096 C3 replicas (HBM, AWC)
// 3.51 -> 2.87 s; the non-AWC HBM variant keeps the general set (the C2 sweep
// 512 -> 677 ms with this one).
#ifndef DSD_SMEM_BARRIER_KINDS
#define DSD_SMEM_BARRIER_KINDS ((1u << kActBegin) | (1u << kActBeginAwc) | (1u << kActNone))
#endif
constexpr uint32_t kSmemBarrierKinds = DSD_SMEM_BARRIER_KINDS;
// The specialised kernel's barrier: only the session loop's entry (Begin).
// The loop absorbs the steady state, so what remains between two loop runs
// is a short chain of per-request general events, which each lane now runs
// in one go: every warp round is one loop run + one chain for all lanes.
// Measured on the C5 sweep (B200): the general set 18.6 ms, {Begin} 14.2,
// {Begin, Dispatch} 14.2, {Begin, Item} 14.6.
#ifndef DSD_SPEC_BARRIER_KINDS
#define DSD_SPEC_BARRIER_KINDS ((1u << kActBegin) | (1u << kActNone))
#endif
constexpr uint32_t kSpecBarrierKinds = DSD_SPEC_BARRIER_KINDS;
DSD_HD bool is_barrier(uint32_t kind, bool spec, bool smem) {
    return ((spec ? kSpecBarrierKinds : smem ? kSmemBarrierKinds : kBarrierKinds) >> kind) & 1u;
}

struct Engine {
    // Register budget: everything below stays live across the whole event
    // loop, so only what nearly every step touches lives here; counters the
    // reference keeps incrementally (events processed, first arrival, last
    // completion, completed) are derived once in finish(), and the routing
    // stream / round-robin counter (random and rr routing only) live in HBM.
    const Workspace& W;
    const DevScenario& S;
    ReqRec* R;  // this replica's request records
    // shared-memory copies of the draft servers' active sessions (slot d =
    // draft d, lane stride kHotStride), or null: see rec()
    unsigned char* hotb;
    int32_t rep;
    int32_t N;
    int64_t now = 0;
    uint32_t seq_next;  // next seq for schedule(); arrivals hold 0..N-1
    int32_t heap_n = 0;
    int32_t next_arr = 0;
    int64_t next_arr_t = 0;  // arrival time of arrival next_arr (valid while next_arr < N)
    Rng jitter;
    int64_t net_wait_total = 0;
    int32_t net_wait_count = 0;
    int32_t fail = kFailNone;
    int32_t T, D;
    // action stack
    // slots hold kStackEmpty when unused (its kind bits read kActNone), so the
    // depth needs no counter
    static constexpr uint32_t kStackEmpty = 0xffffffffu;
    uint32_t st0 = kStackEmpty, st1 = kStackEmpty, st2 = kStackEmpty, st3 = kStackEmpty;
    int32_t item_server = -1;
    // the one event a step schedules (pend_t < 0: none); step() inserts it
    // at its end, so the heap insertion is inlined once
    int64_t pend_t = -1;
    uint32_t pend_info = 0;
    // per-warp state blocks (shared memory for small topologies, else HBM),
    // already offset by this lane: element k of a field is at base[k * 32]
    int32_t* sb;     // server fields [kServerFields][nsc]
    int64_t* htb;    // heap times [hcap]
    uint64_t* hkb;   // heap keys  [hcap]
    int32_t hcap;
    int32_t nsc;
    int32_t lst;  // lane stride of sb / htb / hkb (lstride())
    // hot scenario parameters: packed policy flags + the static window
    // fused_everything | pair_stats<<1 | lab<<2 | jitter_free<<3 | window<<4 | routing<<6 |
    // has_order<<8 | single_link<<9 | batching_window<<10
    uint32_t pflags;
    int32_t gamma_s, max_batch, dmax_batch;
    // Specialised instantiation for batches whose every scenario is a single
    // (target, draft) pair with a static window, FIFO batching, no batching
    // window, a jitter-free link, no pair statistics, no probe and no record
    // collection (Runtime::launch checks; the C5 sweep is one).  The kernel
    // passes a compile-time true, so T, D and the policy flags below become
    // constants and the generic paths fold away: a smaller, faster event loop.
    bool spec;
    bool smem_barriers = false;  // the generic shared-memory kernel's barrier set (kSmemBarrierKinds)
    int spec_limit;  // overflow limit of the specialised stack (a kernel template constant)
    static constexpr uint32_t kSpecFlags = (1u << 3) | (1u << 9);  // jitter_free | single_link
    // specialised kernel only: the four latency grids (target / draft x
    // prefill / decode-shaped) and the link's one-way delay, resolved once
    const DevGrid *g_tp = nullptr, *g_td = nullptr, *g_dp = nullptr, *g_dd = nullptr;
    int64_t link_us = 0;
    // the warp's cooperative AWC scratch (shared memory), null for batches
    // without AWC scenarios
    AwcWarpScratch* awc = nullptr;

    DSD_HD Engine(const Workspace& w, const DevScenario& s, int64_t replica, int32_t* server_base,
                  int64_t* heap_time_base, uint64_t* heap_key_base, int64_t heap_cap, int32_t server_cap,
                  unsigned char* hot_base = nullptr, bool specialized = false, AwcWarpScratch* awc_scratch = nullptr,
                  int spec_stack_limit = kSpecStack, int32_t lane_stride = kLanes, ReqRec* records = nullptr)
        : W(w), S(s), rep(static_cast<int32_t>(replica)), sb(server_base), htb(heap_time_base),
          hkb(heap_key_base), hcap(static_cast<int32_t>(heap_cap)), nsc(server_cap), lst(lane_stride),
          spec(specialized), spec_limit(spec_stack_limit) {
        R = records ? records : W.req + replica * W.c.nr;
        gamma_s = S.gamma;
        max_batch = S.max_batch;
        dmax_batch = S.draft_max_batch;
        if (spec) {
            T = 1;
            D = 1;
            hotb = hot_base;
            pflags = kSpecFlags;
            const int32_t* tg = blob_ptr<int32_t>(W.blob, S.o_tgrid);
            const int32_t* dg = blob_ptr<int32_t>(W.blob, S.o_dgrid);
            const DevGrid* grids = blob_ptr<DevGrid>(W.blob, S.o_grids);
            g_tp = grids + tg[0];
            g_td = grids + tg[1];
            g_dp = grids + dg[0];
            g_dd = grids + dg[1];
            link_us = blob_ptr<DevLink>(W.blob, S.o_links)[0].fixed_us;
            return;
        }
        T = S.n_targets;
        D = S.n_drafts;
        hotb = S.fused_everything ? nullptr : hot_base;
        awc = awc_scratch;
        pflags = static_cast<uint32_t>(S.fused_everything) | (static_cast<uint32_t>(S.pair_stats) << 1) |
                 (static_cast<uint32_t>(S.batching == 1) << 2) | (static_cast<uint32_t>(S.jitter_free) << 3) |
                 (static_cast<uint32_t>(S.window_kind) << 4) | (static_cast<uint32_t>(S.routing) << 6) |
                 (static_cast<uint32_t>(S.has_order != 0) << 8) |
                 (static_cast<uint32_t>(S.n_dg == 1 && S.n_tg == 1) << 9) |
                 (static_cast<uint32_t>(S.batching_window_us > 0) << 10);
    }
    DSD_HD bool hot() const { return spec || hotb != nullptr; }
    // this thread's lane in its warp (per-warp shared-memory slots); a
    // replica's index says nothing about it when the kernel runs a replica list
    static DSD_HD int hw_lane() {
#ifdef __CUDA_ARCH__
        return static_cast<int>(threadIdx.x & (kLanes - 1));
#else
        return 0;
#endif
    }
    DSD_HD bool collecting() const { return !spec && W.collect; }
    // log_transition (engine.cpp:213-219) of request i, whose phase was just set
    DSD_HD void log_tr(int64_t i, const ReqRec& r, uint32_t detail) {
        if (spec || !W.elog) return;
        const int32_t f = elog_append(W, rep, now, i, phase(r), detail, D > 0 ? r.drafter : -1, r.target);
        if (f) fail = f;
    }
    DSD_HD bool probing() const { return !spec && W.probe != nullptr; }
    DSD_HD bool fe() const { return pflags & 1u; }
    DSD_HD bool ps() const { return (pflags >> 1) & 1u; }
    DSD_HD bool lab_batching() const { return (pflags >> 2) & 1u; }
    DSD_HD bool jitter_free() const { return (pflags >> 3) & 1u; }
    DSD_HD uint32_t wkind() const { return (pflags >> 4) & 3u; }
    DSD_HD uint32_t routing_kind() const { return (pflags >> 6) & 3u; }
    DSD_HD bool has_order() const { return (pflags >> 8) & 1u; }
    DSD_HD bool single_link() const { return (pflags >> 9) & 1u; }
    DSD_HD bool batching_window() const { return (pflags >> 10) & 1u; }
    // warp-interleaved per-replica arrays in HBM (pair stats, busy export)
    template <typename U>
    DSD_HD U& IL(U* base, int64_t cap, int64_t idx) const {
        return base[((static_cast<int64_t>(rep) >> 5) * cap + idx) * kLanes + (rep & 31)];
    }

    // server fields (engine.cpp:70-84 Server, minus the queue/running vectors
    // which are intrusive lists through the request records).  Targets and
    // draft servers use disjoint fields, overlaid: targets keep the batching
    // window's arm sequence, open requests and busy time (only target busy
    // time is reported); draft servers keep the active session and the
    // session FIFO.
    enum : int {
        F_v_qhead = 0, F_v_qtail = 1, F_v_run = 2,
        F_v_flags = 3,  // busy | armed << 1
        F_v_armseq = 4, F_v_open = 5, F_v_busy_lo = 6, F_v_busy_hi = 7,  // targets
        F_v_active = 4, F_v_shead = 5, F_v_stail = 6                      // draft servers
    };
#define SV(field, i) sv(F_##field, (i))
    // (32-bit index math: server and heap blocks are far below 2^31 elements)
    // lane stride of the per-warp state blocks: kLanes when a warp's lanes
    // interleave their replicas, 1 in solo mode (one replica per block)
    DSD_HD int32_t lstride() const { return spec ? kLanes : lst; }
    DSD_HD int32_t& sv(int f, int32_t v) const { return sb[(f * nsc + v) * lstride()]; }
    // Server::busy_us (engine.cpp:562) as two 32-bit halves in the server block
    DSD_HD int64_t get_busy(int32_t v) const {
        return static_cast<int64_t>((static_cast<uint64_t>(static_cast<uint32_t>(SV(v_busy_hi, v))) << 32) |
                                    static_cast<uint32_t>(SV(v_busy_lo, v)));
    }
    DSD_HD void set_busy(int32_t v, int64_t x) {
        SV(v_busy_lo, v) = static_cast<int32_t>(static_cast<uint32_t>(x));
        SV(v_busy_hi, v) = static_cast<int32_t>(static_cast<uint32_t>(static_cast<uint64_t>(x) >> 32));
    }
    DSD_HD bool busy(int32_t v) const { return SV(v_flags, v) & 1; }
    DSD_HD bool armed(int32_t v) const { return SV(v_flags, v) & 2; }
    DSD_HD void set_busy_flag(int32_t v, bool b) { SV(v_flags, v) = (SV(v_flags, v) & ~1) | (b ? 1 : 0); }
    DSD_HD void set_armed(int32_t v, bool b) { SV(v_flags, v) = (SV(v_flags, v) & ~2) | (b ? 2 : 0); }
    DSD_HD int64_t& ht(int32_t k) const { return htb[k * lstride()]; }
    DSD_HD uint64_t& hk(int32_t k) const { return hkb[k * lstride()]; }

    // ---- action stack ----
    static DSD_HD uint32_t act(uint32_t kind, uint32_t arg) { return kind | (arg << 4); }
    // Depth 4 (st0..st3); the specialised kernel keeps kSpecStack slots (fewer
    // registers to shift and to merge at every join), and a replica that
    // would need more fails with kFailStack and runs again on the HBM variant.
    DSD_HD int stack_cap() const { return spec ? kSpecStack : 4; }
    DSD_HD void push_act(uint32_t a) {
        const int lim = spec ? spec_limit : 4;  // full when the limit's last slot is taken
        if ((lim <= 1 ? st0 : lim == 2 ? st1 : lim == 3 ? st2 : st3) != kStackEmpty) {
            fail = kFailStack;
            return;
        }
        if (stack_cap() > 3) st3 = st2;
        if (stack_cap() > 2) st2 = st1;
        st1 = st0;
        st0 = a;
    }
    DSD_HD uint32_t pop_act() {
        uint32_t a = st0;
        st0 = st1;
        st1 = stack_cap() > 2 ? st2 : kStackEmpty;
        if (stack_cap() > 2) st2 = stack_cap() > 3 ? st3 : kStackEmpty;
        if (stack_cap() > 3) st3 = kStackEmpty;
        return a;
    }

    // ---- request flags ----
    static constexpr int kDpd = 3, kTpd = 4, kFused = 5;
    static DSD_HD uint32_t phase(const ReqRec& r) { return r.flags & 7u; }
    static DSD_HD void set_phase(ReqRec& r, uint32_t p) { r.flags = static_cast<uint8_t>((r.flags & ~7u) | p); }
    static DSD_HD bool flag(const ReqRec& r, int bit) { return (r.flags >> bit) & 1u; }
    static DSD_HD void set_flag(ReqRec& r, int bit, bool v) {
        uint8_t f = r.flags;
        r.flags = static_cast<uint8_t>(v ? (f | (1u << bit)) : (f & ~(1u << bit)));
    }
    DSD_HD int32_t draft_of(int64_t i) const { return D > 0 ? rec(i).drafter : -1; }

    // ---- request records ----
    // On sm_100 a global store invalidates its line in L1, so a record that
    // is read-modify-written every step would cost an L2 round trip per step.
    // A draft server's active session (the request in its speculation loop,
    // which takes nearly all record traffic) is therefore moved into a
    // shared-memory slot while it is active: activate_next_session copies it
    // in, finish_request writes it back.  rec(i) is the only way the engine
    // touches a record; the slot is authoritative while i is active.
    DSD_HD ReqRec& slot(int32_t d) const {
        return *reinterpret_cast<ReqRec*>(hotb + static_cast<int64_t>(d) * kLanes * kHotStride);
    }
    DSD_HD ReqRec& rec(int64_t i) const {
        if (hot()) {
            for (int32_t d = 0; d < D; ++d)
                if (SV(v_active, T + d) == static_cast<int32_t>(i)) return slot(d);
        }
        return R[i];
    }
    static DSD_HD void copy_rec_inline(ReqRec& dst, const ReqRec& src) {
        uint64_t* d = reinterpret_cast<uint64_t*>(&dst);
        const uint64_t* s = reinterpret_cast<const uint64_t*>(&src);
        uint64_t v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = s[k];  // all loads first: one memory latency
#pragma unroll
        for (int k = 0; k < 16; ++k) d[k] = v[k];
    }
    // out of line in the generic kernel (its code size is the constraint);
    // runs twice per request (activation, write-back)
    static DSD_HD_NOINLINE void copy_rec_call(ReqRec& dst, const ReqRec& src) { copy_rec_inline(dst, src); }
    DSD_HD void copy_rec(ReqRec& dst, const ReqRec& src) const {
        if (spec) copy_rec_inline(dst, src); else copy_rec_call(dst, src);
    }
    // Specialised kernel: the active session's current acceptance-bit word,
    // bits[cursor >> 6], kept in the 8 bytes that pad its shared-memory slot
    // to kHotStride.  Refilled by an asynchronous global->shared copy when
    // the session activates and when its cursor moves to another word, so a
    // verify reads shared memory instead of a bit line that L1 (small next
    // to the shared-memory carveout) has usually evicted.
    DSD_HD uint64_t* slot_word() const { return reinterpret_cast<uint64_t*>(hotb + sizeof(ReqRec)); }
    DSD_HD void fetch_word(const ReqRec& r, int32_t cur) const {
#ifdef __CUDA_ARCH__
        // a refill still in flight (the previous session's last verify) must
        // land first: copies from one thread complete in no particular order
        wait_word();
        const uint64_t* src = W.bits + static_cast<int64_t>(rep) * W.c.bw + r.bitoff + (cur >> 6);
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(slot_word()));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
#else
        *slot_word() = W.bits[static_cast<int64_t>(rep) * W.c.bw + r.bitoff + (cur >> 6)];
#endif
    }
    static DSD_HD void wait_word() {
#ifdef __CUDA_ARCH__
        asm volatile("cp.async.wait_all;" ::: "memory");
#endif
    }
    // pulls a queued session's record towards L2 ahead of its activation
    DSD_HD void prefetch_l2(int32_t i) const {
#ifdef __CUDA_ARCH__
        if (i >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(R + i));
#else
        (void)i;
#endif
    }

    // ---- event heap: SimKernel::schedule (event_queue.cpp:20-26) ----
    static DSD_HD bool key_less(int64_t ta, uint64_t ka, int64_t tb, uint64_t kb) {
        return ta < tb || (ta == tb && ka < kb);
    }
    DSD_HD void defer(int64_t t, uint32_t inf) {
        pend_t = t;
        pend_info = inf;
    }
    DSD_HD void schedule(int64_t t, uint32_t info) {
        if (heap_n >= hcap) {
            fail = kFailHeap;
            return;
        }
        uint64_t key = (static_cast<uint64_t>(seq_next) << 32) | info;
        ++seq_next;
        int32_t i = heap_n++;
        while (i > 0) {
            int32_t p = (i - 1) >> 1;
            int64_t pt = ht(p);
            uint64_t pk = hk(p);
            if (!key_less(t, key, pt, pk)) break;
            ht(i) = pt;
            hk(i) = pk;
            i = p;
        }
        ht(i) = t;
        hk(i) = key;
    }
    DSD_HD void heap_pop() {
        int32_t n = --heap_n;
        if (n == 0) return;
        int64_t t = ht(n);
        uint64_t k = hk(n);
        int32_t i = 0;
        for (;;) {
            int32_t c = 2 * i + 1;
            if (c >= n) break;
            int64_t ct = ht(c);
            uint64_t ck = hk(c);
            if (c + 1 < n) {
                int64_t dt = ht(c + 1);
                uint64_t dk = hk(c + 1);
                if (key_less(dt, dk, ct, ck)) {
                    c = c + 1;
                    ct = dt;
                    ck = dk;
                }
            }
            if (!key_less(ct, ck, t, k)) break;
            ht(i) = ct;
            hk(i) = ck;
            i = c;
        }
        ht(i) = t;
        hk(i) = k;
    }
    static DSD_HD uint32_t info(uint32_t kind, uint32_t msg, uint32_t id) { return kind | (msg << 3) | (id << 5); }

    // ---- network: net_delay (engine.cpp:10-15) ----
    DSD_HD const DevLink& link(int32_t d, int32_t t) const {
        const DevLink* links = blob_ptr<DevLink>(W.blob, S.o_links);
        if (single_link()) return links[0];
        const int32_t* dg = blob_ptr<int32_t>(W.blob, S.o_dgroup);
        const int32_t* tg = blob_ptr<int32_t>(W.blob, S.o_tgroup);
        return links[dg[d] * S.n_tg + tg[t]];
    }
    DSD_HD int64_t net_delay(int32_t d, int32_t t) {
        if (spec) return link_us;  // one jitter-free link
        const DevLink& lk = link(d, t);
        if (jitter_free()) return lk.fixed_us;  // the jitter stream is unobservable
        double rtt = lk.rtt_ms, jit = lk.jitter_ms;
        double j = jitter.uniform(-jit / 2.0, jit / 2.0);
        double ms = rtt / 2.0 + j;
        if (ms < 0.0) ms = 0.0;
        return llround(ms * 1000.0);
    }

    // ---- metrics hooks (metrics.cpp:40-128) ----
    DSD_HD int64_t pair_of(int32_t d, int32_t t) const { return static_cast<int64_t>(d) * T + t; }
    // fixed-capacity ring insert: returns the storage slot (metrics.cpp:55-72)
    static DSD_HD int64_t ring_slot(int32_t& cnt, int32_t& pos, int cap) {
        if (cnt < cap) return cnt++;
        int64_t s = pos;
        pos = (pos + 1) % cap;
        return s;
    }
    DSD_HD void on_verify(int32_t d, int32_t t, int ex, int ac) {
        if (!ps()) return;
        int64_t p = pair_of(d, t);
        int64_t slot = ring_slot(IL(W.p_acc_cnt, W.c.np, p), IL(W.p_acc_pos, W.c.np, p), 20);
        IL(W.p_acc_ex, W.c.np * 20, p * 20 + slot) = ex;
        IL(W.p_acc_ac, W.c.np * 20, p * 20 + slot) = ac;
    }
    DSD_HD void on_rtt_sample(int32_t d, int32_t t, double rtt_ms) {
        if (!ps()) return;
        int64_t p = pair_of(d, t);
        int64_t slot = ring_slot(IL(W.p_rtt_cnt, W.c.np, p), IL(W.p_rtt_pos, W.c.np, p), 20);
        IL(W.p_rtt, W.c.np * 20, p * 20 + slot) = rtt_ms;
    }
    DSD_HD void push_tpot(int32_t t, double v) {
        if (!ps()) return;
        int64_t slot = ring_slot(IL(W.t_tcnt, W.c.nt, t), IL(W.t_tpos, W.c.nt, t), 50);
        IL(W.t_tpot, W.c.nt * 50, static_cast<int64_t>(t) * 50 + slot) = v;
    }

    // ---- window policies: decide_window (engine.cpp:350-374) ----
    struct Decision {
        bool fused;
        int gamma;
    };

    DSD_HD Decision decide_window(int64_t i) {
        const ReqRec& r = rec(i);
        int32_t d = D > 0 ? r.drafter : -1;
        if (d < 0) return Decision{true, 1};
        int32_t t = r.target;
        switch (wkind()) {
            case 0:  // window_static (policies.cpp:55-58)
                return Decision{false, gamma_s};
            case 1: {  // window_dynamic (policies.cpp:60-68)
                int64_t p = pair_of(d, t);
                double a = acceptance_recent_at(W, rep, p);
                int32_t& g = IL(W.p_dyn, W.c.np, p);
                if (a > 0.75 && g < S.gamma_max) {
                    ++g;
                } else if (a < 0.25 && g > S.gamma_min) {
                    --g;
                }
                return Decision{false, g};
            }
            case 2:  // AWC: begin() hands these to the warp (extract_features ->
                     // awc_serve_warp -> begin_awc); only batches with AWC
                     // scenarios run them, on the kAwc kernels, so this is
                     // unreachable - fail loudly rather than compile the
                     // per-lane network into every kernel
                fail = kFailAwcDims;
                return Decision{true, 1};
            default:
                return Decision{true, 1};
        }
    }
    // stabilized_decide (smoother.cpp:8-37) of the pair's smoother on a raw
    // AWC prediction
    DSD_HD Decision stabilized_decide(int64_t p, double raw) {
        const double gmin = static_cast<double>(S.gamma_min);
        const double gmax = static_cast<double>(S.gamma_max);
        double clamped = raw < gmin ? gmin : (gmax < raw ? gmax : raw);
        uint8_t& init = IL(W.p_sm_init, W.c.np, p);
        double& ema = IL(W.p_sm_ema, W.c.np, p);
        int32_t& low = IL(W.p_sm_low, W.c.np, p);
        uint8_t& fz = IL(W.p_sm_fused, W.c.np, p);
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

    // ---- work queues: intrusive lists through the records' item slots ----
    DSD_HD int32_t slot_next(int32_t s) const { return rec(s >> 1).next[s & 1]; }
    DSD_HD void set_slot_next(int32_t s, int32_t n) { rec(s >> 1).next[s & 1] = n; }

    // push_work (engine.cpp:473-476): append, then try_dispatch as the next action
    DSD_HD void enqueue(int32_t v, int64_t i, int k, uint32_t op, int32_t tokens, bool via) {
        ReqRec& r = rec(i);
        r.op[k] = static_cast<uint8_t>(op | (via ? 4u : 0u));
        if (k) r.tok1 = tokens;
        r.enq[k] = now;
        r.next[k] = -1;
        const int32_t slot = static_cast<int32_t>(2 * i + k);
        int32_t& tail = SV(v_qtail, v);
        if (tail < 0) {
            SV(v_qhead, v) = slot;
        } else {
            set_slot_next(tail, slot);
        }
        tail = slot;
        push_act(act(kActDispatch, static_cast<uint32_t>(v) * 2));
    }

    static DSD_HD bool eligible(bool is_draft, uint32_t op, const ReqRec& r) {
        // item_eligible (engine.cpp:478-483)
        return is_draft || op == kOpPrefill || flag(r, kTpd);
    }

    // try_dispatch (engine.cpp:485-567)
    DSD_HD void try_dispatch(int32_t v, bool window_expired) {
        if (busy(v) || SV(v_qhead, v) < 0) return;
        if (spec && (v == 1 ? dispatch_single_draft() : dispatch_single_target())) return;
        const bool is_draft = v >= T;
        const int64_t mb = is_draft ? dmax_batch : max_batch;
        int32_t kind = -1;
        // Only an armable batching window needs the candidate count before
        // anything is taken; otherwise the head kind is fixed by the first
        // eligible item of the single forming pass below.
        if (!is_draft && batching_window() && !window_expired) {
            int64_t ncand = 0;
            for (int32_t cur = SV(v_qhead, v); cur >= 0; cur = rec(cur >> 1).next[cur & 1]) {
                const ReqRec& rc = rec(cur >> 1);
                uint32_t op = rc.op[cur & 1] & 3u;
                if (!eligible(is_draft, op, rc)) continue;
                if (kind < 0) kind = static_cast<int32_t>(op);
                if (static_cast<int32_t>(op) != kind) continue;
                ++ncand;
            }
            if (ncand == 0) return;
            if (ncand < mb) {
                if (!armed(v)) {
                    set_armed(v, true);
                    SV(v_armseq, v) = seq_next;  // stands in for ++window_gen (engine.cpp:512-517)
                    defer(now + S.batching_window_us, info(kEvBatchReady, 0, static_cast<uint32_t>(v)));
                }
                return;
            }
            set_armed(v, false);
        }

        const bool lab = !is_draft && lab_batching();
        int64_t head_len = 0;
        double band = 0.0;
        int64_t taken = 0, seen = 0;
        int32_t prev = -1, run_tail = -1;
        int32_t tok = 1;
        int64_t ctx = 0;
        for (int32_t cur = SV(v_qhead, v); cur >= 0;) {
            const int64_t i = cur >> 1;
            const int k = cur & 1;
            ReqRec& r = rec(i);
            const int32_t nxt = r.next[k];
            const uint32_t opv = r.op[k];
            const uint32_t op = opv & 3u;
            bool take = false;
            const bool elig = eligible(is_draft, op, r);
            if (elig && kind < 0) kind = static_cast<int32_t>(op);
            if (static_cast<int32_t>(op) == kind && elig) {
                if (!lab) {  // batch_fifo (policies.cpp:30-38)
                    take = taken < mb;
                } else {     // batch_lab (policies.cpp:40-53)
                    int64_t wl = op == kOpPrefill ? static_cast<int64_t>(k ? r.tok1 : r.prompt)
                                                  : static_cast<int64_t>(r.output) - r.tokens;
                    if (seen == 0) {
                        head_len = wl;
                        band = S.sim_frac * static_cast<double>(head_len);
                        take = true;
                    } else if (taken < mb) {
                        double diff = fabs(static_cast<double>(wl - head_len));
                        take = diff <= band;
                    }
                }
                ++seen;
            }
            if (take) {
                ++taken;
                // stable removal from the queue, append to the running batch
                if (prev < 0) SV(v_qhead, v) = nxt; else set_slot_next(prev, nxt);
                if (SV(v_qtail, v) == cur) SV(v_qtail, v) = prev;
                r.next[k] = -1;
                if (run_tail < 0) SV(v_run, v) = cur; else set_slot_next(run_tail, cur);
                run_tail = cur;
                // BatchShape (engine.cpp:544-552)
                int32_t t_i = k ? r.tok1 : r.prompt;
                if (t_i > tok) tok = t_i;
                if (op != kOpPrefill) {
                    int64_t c = static_cast<int64_t>(r.prompt) + r.tokens;
                    if (c > ctx) ctx = c;
                }
                if (opv & 4u) {
                    net_wait_total += now - r.enq[k];
                    ++net_wait_count;
                }
            } else {
                prev = cur;
            }
            cur = nxt;
        }
        if (taken == 0) return;  // nothing eligible (the reference's empty candidate list)
        // LatencyProfile::predict (profile.cpp:129-151) on the server's grids
        const bool prefill = kind == static_cast<int32_t>(kOpPrefill);
        const bool decode = kind == static_cast<int32_t>(kOpDecode);
        // queries: (batch, prompt tokens) / (batch, context) / (batch*tokens, context)
        const int64_t qb = (prefill || decode) ? taken : taken * tok;
        const int64_t qc = prefill ? static_cast<int64_t>(tok) : ctx;
        const DevGrid* gp;
        if (spec) {
            gp = is_draft ? (prefill ? g_dp : g_dd) : (prefill ? g_tp : g_td);
        } else {
            const int32_t* gi = is_draft ? blob_ptr<int32_t>(W.blob, S.o_dgrid) + 2 * (v - T)
                                         : blob_ptr<int32_t>(W.blob, S.o_tgrid) + 2 * v;
            gp = blob_ptr<DevGrid>(W.blob, S.o_grids) + gi[prefill ? 0 : 1];
        }
        const DevGrid& g = *gp;
        double ms = g.o_btab >= 0 && g.o_ctab >= 0
                        ? grid_interpolate_int(W.blob, g, qb, qc)
                        : grid_interpolate(W.blob, g, static_cast<double>(qb), static_cast<double>(qc));
        if (decode) ms *= tok;
        int64_t lat = llround(ms * 1000.0);
        if (lat < 1) lat = 1;
        set_busy_flag(v, true);
        if (!is_draft) set_busy(v, get_busy(v) + lat);  // only target busy time is reported
        if (!spec && W.elog) {
            const int32_t f = busy_append(W, rep, is_draft ? ~(v - T) : v, now, now + lat);
            if (f) fail = f;
        }
        defer(now + lat, info(kEvComputeDone, 0, static_cast<uint32_t>(v)));
    }

    DSD_HD int64_t latency_us(const DevGrid& g, int64_t qb, int64_t qc, int32_t mult) const {
        return grid_latency_us(W.blob, g, qb, qc, mult);
    }

    // try_dispatch of the specialised kernel's target server when its queue
    // holds one item (with one draft server, only the active session has
    // work at the target): FIFO forming takes that item if it is eligible
    // (item_eligible) and nothing otherwise; same BatchShape, latency query,
    // rounding and busy time as the general pass with taken = 1.
    DSD_HD bool dispatch_single_target() {
        const int32_t cur = SV(v_qhead, 0);
        ReqRec& r = rec(cur >> 1);
        const int k = cur & 1;
        if (r.next[k] >= 0) return false;  // more than one item: the general path
        const uint32_t opv = r.op[k];
        const uint32_t op = opv & 3u;
        if (!eligible(false, op, r)) return true;  // nothing eligible: no batch
        SV(v_qhead, 0) = -1;
        SV(v_qtail, 0) = -1;
        SV(v_run, 0) = cur;
        const int32_t t_i = k ? r.tok1 : r.prompt;
        const int32_t tok = t_i > 1 ? t_i : 1;
        const bool prefill = op == kOpPrefill;
        const bool decode = op == kOpDecode;
        const int64_t ctx = prefill ? 0 : static_cast<int64_t>(r.prompt) + r.tokens;
        if (opv & 4u) {
            net_wait_total += now - r.enq[k];
            ++net_wait_count;
        }
        const int64_t qb = (prefill || decode) ? 1 : tok;
        const int64_t qc = prefill ? static_cast<int64_t>(tok) : (ctx > 0 ? ctx : 0);
        const int64_t lat = latency_us(*(prefill ? g_tp : g_td), qb, qc, decode ? tok : 0);
        set_busy_flag(0, true);
        set_busy(0, get_busy(0) + lat);
        defer(now + lat, info(kEvComputeDone, 0, 0u));
        return true;
    }

    // try_dispatch of the specialised kernel's draft server when its queue
    // holds one item (the active session's draft prefill or decode): the
    // general forming pass below reduces to taking that item (always
    // eligible, never via the network); same latency query and rounding.
    DSD_HD bool dispatch_single_draft() {
        const int32_t cur = SV(v_qhead, 1);
        ReqRec& r = rec(cur >> 1);
        const int k = cur & 1;
        if (r.next[k] >= 0) return false;  // more than one item: the general path
        const uint32_t op = r.op[k] & 3u;
        SV(v_qhead, 1) = -1;
        SV(v_qtail, 1) = -1;
        SV(v_run, 1) = cur;
        const int32_t t_i = k ? r.tok1 : r.prompt;
        const int32_t tok = t_i > 1 ? t_i : 1;
        const bool prefill = op == kOpPrefill;
        const int64_t ctx = prefill ? 0 : static_cast<int64_t>(r.prompt) + r.tokens;
        // qb = taken = 1 (prefill / decode); qc = prompt tokens / context
        const int64_t qc = prefill ? static_cast<int64_t>(tok) : (ctx > 0 ? ctx : 0);
        // decode: latency x tokens_per_request
        const int64_t lat = latency_us(*(prefill ? g_dp : g_dd), 1, qc, prefill ? 0 : tok);
        set_busy_flag(1, true);
        defer(now + lat, info(kEvComputeDone, 0, 1u));
        return true;
    }

    // ---- request lifecycle ----
    DSD_HD void record_gamma(ReqRec& r, int g) {
        int32_t n = r.ng;
        if (collecting()) {
            int64_t o = W.rep_seqbase[rep] + r.seqoff + n;
            if (o < W.seq_cap) W.seq_gamma[o] = g; else fail = kFailSeq;
        }
        r.ng = n + 1;
    }
    DSD_HD void record_commit(ReqRec& r, int c) {
        int32_t n = r.nc;
        if (collecting()) {
            int64_t o = W.rep_seqbase[rep] + r.seqoff + n;
            if (o < W.seq_cap) W.seq_commit[o] = c; else fail = kFailSeq;
        }
        r.nc = n + 1;
    }

    // activate_next_session (engine.cpp:332-339)
    DSD_HD void activate_next_session(int32_t d) {
        int32_t v = T + d;
        if (SV(v_active, v) >= 0 || SV(v_shead, v) < 0) return;
        int32_t i = SV(v_shead, v);
        const ReqRec& g = R[i];  // not active yet: the HBM record is current
        int32_t nx = g.snext;
        SV(v_shead, v) = nx;
        if (nx < 0) SV(v_stail, v) = -1;
        if (hot()) {
            copy_rec(slot(d), g);
            if (spec && g.nbits > 0) fetch_word(g, g.cursor);
            prefetch_l2(nx);  // the next session's copy-in is one activation away
        }
        SV(v_active, v) = i;
        enqueue(v, i, 1, kOpPrefill, g.prompt, false);
    }

    // route (engine.cpp:315-330, policies.cpp:9-28)
    DSD_HD int32_t route() {
        if (T <= 1) return 0;  // uniform_below(1) draws nothing; rr and jsq pick 0 too
        uint64_t* st = W.route_state + static_cast<int64_t>(rep) * 5;  // routing stream + rr counter
        switch (routing_kind()) {
            case 0: {
                Rng g{st[0], st[1], st[2], st[3]};
                const int32_t t = static_cast<int32_t>(g.below(static_cast<uint64_t>(T)));
                st[0] = g.s0;
                st[1] = g.s1;
                st[2] = g.s2;
                st[3] = g.s3;
                return t;
            }
            case 1:
                return static_cast<int32_t>(st[4]++ % static_cast<uint64_t>(T));
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
        ReqRec& r = R[i];  // a new arrival is never an active session
        set_phase(r, kPhRouted);
        int32_t t = route();
        r.target = t;
        ++SV(v_open, t);  // MetricsCollector::on_route
        log_tr(i, r, kLogRouted);
        set_phase(r, kPhQueuedPrefill);
        if (fe()) {
            set_flag(r, kFused, true);
            enqueue(t, i, 0, kOpPrefill, r.prompt, false);
        } else {
            int32_t d = r.drafter;
            int32_t v = T + d;
            r.snext = -1;
            int32_t tail = SV(v_stail, v);
            // queued sessions are not active: their HBM records are current
            if (tail < 0) SV(v_shead, v) = static_cast<int32_t>(i); else R[tail].snext = static_cast<int32_t>(i);
            SV(v_stail, v) = static_cast<int32_t>(i);
            // activate_next_session runs first, then net_delay + schedule
            push_act(act(kActSendPrompt, static_cast<uint32_t>(i)));
            push_act(act(kActActivate, static_cast<uint32_t>(d)));
        }
    }

    // [decide_window] + begin_iteration (engine.cpp:254-257, 383-404)
    DSD_HD void begin(int64_t i, bool decide) {
        if (decide && awc && wkind() == 2) {
            const ReqRec& r = rec(i);
            const int32_t d = D > 0 ? r.drafter : -1;
            if (d >= 0) {
                // AWC decision: park the model input and yield; the warp
                // evaluates the network cooperatively (awc_serve_warp) before
                // the continuation kActBeginAwc runs the smoother and the rest
                const int32_t t = r.target;
                // (the raw features go straight into the lane's shared-memory
                // input slot and are normalised in place: no local array)
                const int lane = hw_lane();
                double* xin = awc->x[lane];
                extract_features(W, rep, pair_of(d, t), t, SV(v_open, t), S.queue_capacity, link(d, t).rtt_ms, xin);
                awc_normalize(S, xin, xin);
                awc->req[lane] = 1;
                push_act(act(kActBeginAwc, static_cast<uint32_t>(i)));
                return;
            }
        }
        begin_with(i, decide ? decide_window(i) : Decision{true, 1});
    }
    // continuation of begin once the warp served the AWC request
    DSD_HD void begin_awc(int64_t i) {
        const ReqRec& r = rec(i);
        const Decision dec = stabilized_decide(pair_of(r.drafter, r.target), awc->raw[hw_lane()]);
        begin_with(i, dec);
    }
    DSD_HD void begin_with(int64_t i, const Decision& dec) {
        ReqRec& r = rec(i);
        if (phase(r) == kPhDone) return;
        int32_t d = D > 0 ? r.drafter : -1;
        int32_t t = r.target;
        if (probing())  // before the pair's previous window is overwritten
            probe_iteration(W, rep, d >= 0 ? pair_of(d, t) : -1, t, SV(v_open, t), S.queue_capacity,
                            d >= 0 ? link(d, t).rtt_ms : 0.0, dec.fused ? 1 : dec.gamma);
        if (d >= 0 && t >= 0 && ps()) IL(W.p_gprev, W.c.np, pair_of(d, t)) = dec.fused ? 1 : dec.gamma;
        if (dec.fused) {
            set_flag(r, kFused, true);
            record_gamma(r, 0);
            enqueue(t, i, 1, kOpDecode, 1, false);
        } else {
            set_flag(r, kFused, false);
            record_gamma(r, dec.gamma);
            r.pgamma = dec.gamma;
            set_phase(r, kPhSpeculating);
            log_tr(i, r, kLogSpeculating);
            enqueue(T + d, i, 1, kOpDecode, dec.gamma, false);
        }
    }

    // Specialised kernel: the active session's speculation loop run directly.
    // One iteration is five events - IterationStart (begin_iteration + the
    // draft's dispatch), the draft's ComputeDone (send_proposal), the
    // proposal's NetArrive (verify enqueued and dispatched), the target's
    // ComputeDone (consume_acceptance, the result sent back) and the result's
    // NetArrive (commit_tokens, the next IterationStart at the same time).
    // Each of them is scheduled by its predecessor, so it carries the largest
    // seq so far: it is the replica's next event exactly when its time is
    // below `ext`, the earliest of the next arrival (seq < N) and the heap top
    // (scheduled earlier).  While that holds no other event runs, the heap
    // and both servers' queues stay as they were, and the event is handled
    // here without a heap round trip, an action-stack round trip or a warp
    // vote; seq_next advances as its schedule() would.  The first event that
    // is not the earliest goes to the heap through defer() (the same seq),
    // and anything the loop does not cover (a busy or non-empty target, the
    // target prefill still pending, the request finishing) is handed to the
    // general handlers in the state they would have reached, so events,
    // seqs, timestamps and totals are identical to the step-by-step path.
    //
    // The request's evolving fields live in registers for the loop and are
    // written back once at its exit.  Both latency queries of an iteration
    // use the same context (prompt + tokens committed so far), and the
    // verify's acceptance draw only depends on the cursor, so the two
    // bilinear interpolations and the bit scan are independent chains the
    // scheduler overlaps; the batch-axis segments (batch 1 for the draft
    // decode, gamma for the verify) and the grids' constants are hoisted.
    DSD_HD void session_run(int64_t i) {
        ReqRec& r = rec(i);
        if (phase(r) == kPhDone) return;
        const int32_t g = gamma_s;
        const int32_t prompt = r.prompt, output = r.output, nb = r.nbits;
        // the scenario's latency table: lat[c] = {draft decode of g tokens,
        // verify of g tokens} at context c (status word 0: all below 2^28 us)
        const int2* lat = S.o_slat >= 0 ? reinterpret_cast<const int2*>(W.spec_lat + S.o_slat + 2) : nullptr;
        if (busy(1) || SV(v_qhead, 1) >= 0 || g > 63 || !lat || W.spec_lat[S.o_slat] != 0 ||
            link_us >= kSpecLatMax || prompt + output >= W.spec_lat[S.o_slat + 1] || nb < 1) {
            begin_with(i, Decision{false, gamma_s});  // outside the loop's steady state
            return;
        }
        int64_t ext = next_arr < N ? next_arr_t : INT64_MAX;
        if (heap_n > 0 && ht(0) < ext) ext = ht(0);
        // times relative to the entry: 32-bit, below xr <= 2^30, and every
        // step adds less than 2^28, so no sum overflows
        const int64_t base = now;
        const int32_t xr = ext - base < (1 << 30) ? static_cast<int32_t>(ext - base) : (1 << 30);
        const int32_t lk = static_cast<int32_t>(link_us);
        // the target's state cannot change inside the loop
        const bool target_ok = !busy(0) && SV(v_qhead, 0) < 0 && flag(r, kTpd);
        const uint64_t* bits = W.bits + static_cast<int64_t>(rep) * W.c.bw + r.bitoff;
        const int32_t nwords = (nb + 63) >> 6;
        int32_t tokens = r.tokens, cur = r.cursor, ng = r.ng, nc = r.nc, prop = r.prop, acc = r.acc, lcr = r.lcr;
        int64_t first = r.first;
        int64_t busy0 = get_busy(0);
        wait_word();  // the activation's refill of the slot word has landed
        // the acceptance words at the cursor and after it
        uint64_t w0 = *slot_word();
        uint64_t w1 = (cur >> 6) + 1 < nwords ? bits[(cur >> 6) + 1] : 0;
        int32_t nr = 0;  // now - base
        int32_t nw = 0;  // verifies dispatched (net_wait_count; their wait is 0)
        uint32_t seq = seq_next;
        int32_t t2 = 0;  // proposal arrival of the last iteration (verify enqueue time)
        int2 l = lat[prompt + tokens];
        int a_acc, a_cons;
        int32_t ncur;
        bool full;
        for (;;) {
            // consume_acceptance (engine.cpp:17-32) at the cursor: the run of
            // ones of the g bits there (cyclic over the request's nb bits),
            // capped at g - trailing ones of a 64-bit window with bit g forced
            {
                const int sh = cur & 63;
                uint64_t w = (w0 >> sh) | ((w1 << 1) << (63 - sh));  // bits cur.. (0 past the request's words)
                const int32_t n1 = nb - cur;                          // bits left before the wrap
                if (n1 < g) {
                    // the window wraps once (nb >= g): the request's first
                    // bits follow its last ones
                    if (nb >= g) {
                        w = (w & ((1ull << n1) - 1)) | (bits[0] << n1);
                    } else {  // shorter than the window: several wraps, bit by bit
                        uint64_t x = 0;
                        for (int32_t k = 0, c = cur; k < g; ++k, c = c + 1 == nb ? 0 : c + 1)
                            x |= ((bits[c >> 6] >> (c & 63)) & 1u) << k;
                        w = x;
                    }
                }
#ifdef __CUDA_ARCH__
                a_acc = __ffsll(static_cast<long long>(~w | (1ull << g))) - 1;
#else
                a_acc = __builtin_ctzll(~w | (1ull << g));
#endif
                a_cons = a_acc < g ? a_acc + 1 : g;
                ncur = cur + a_cons;
                while (ncur >= nb) ncur -= nb;  // (cursor + consumed) mod nbits
            }
            // the next iteration's context, and its latency pair loaded now so
            // the load overlaps this iteration's time checks
            const int32_t remaining = output - tokens;
            const int32_t committed = a_acc + 1 < remaining ? a_acc + 1 : remaining;
            const int32_t ntok = tokens + committed;
            const int2 lnext = ntok < output ? lat[prompt + ntok] : l;
            // IterationStart -> draft done -> proposal -> verify done -> result
            const int32_t t4 = nr + l.x + lk + l.y + lk;
            full = target_ok && t4 < xr;
            if (!full) break;
            // the whole iteration is the replica's next five events
            t2 = nr + l.x + lk;
            nr = t4;
            ++ng;
            ++nw;
            busy0 += l.y;
            if ((ncur >> 6) != (cur >> 6)) {  // the cursor moved to another word
                const int32_t wi = ncur >> 6;
                w0 = wi == (cur >> 6) + 1 ? w1 : bits[wi];
                w1 = wi + 1 < nwords ? bits[wi + 1] : 0;
            }
            cur = ncur;
            lcr = a_acc + 1;
            prop += a_cons;
            acc += a_acc;
            tokens = ntok;
            l = lnext;
            ++nc;
            if (first < 0) first = base + nr;
            seq += 4;
            if (tokens >= output) break;
            ++seq;  // IterationStart at now: scheduled, and the earliest event
        }
#ifdef DSD_REP_STATS
        if (W.rep_stats) W.rep_stats[3 * static_cast<int64_t>(rep) + 1] += static_cast<uint32_t>(nc - r.nc);
#endif
        // where the last iteration stopped: the first event that is not the
        // replica's earliest is left pending (defer), the handlers before it ran
        int stage = 5;   // 5: the request completed
        int64_t te = 0;  // the pending event's time
        if (!full) {
            const int32_t t1 = nr + l.x;
            const int32_t tp = t1 + lk;
            const int32_t t3 = tp + l.y;
            ++ng;  // begin_iteration ran
            if (!(t1 < xr)) {
                stage = 0;
                te = base + t1;
            } else if (!(tp < xr)) {
                stage = 1;
                te = base + tp;
                nr = t1;
                seq += 1;
            } else if (!target_ok) {
                stage = 2;
                nr = tp;
                seq += 2;
            } else if (!(t3 < xr)) {
                stage = 3;
                te = base + t3;
                t2 = tp;
                nr = tp;
                seq += 2;
                ++nw;
                busy0 += l.y;
            } else {
                stage = 4;
                te = base + t3 + lk;
                t2 = tp;
                nr = t3;
                seq += 3;
                ++nw;
                busy0 += l.y;
                if ((ncur >> 6) != (cur >> 6)) w0 = bits[ncur >> 6];
                cur = ncur;
                lcr = a_acc + 1;
                prop += a_cons;
                acc += a_acc;
            }
        }
        now = base + nr;
        seq_next = seq;
        // write-back: the record as the step-by-step handlers leave it
        r.tokens = tokens;
        r.cursor = cur;
        r.ng = ng;
        r.prop = prop;
        r.acc = acc;
        r.lcr = lcr;
        r.first = first;
        r.pgamma = g;
        r.tok1 = g;
        r.next[1] = -1;
        *slot_word() = w0;
        set_flag(r, kFused, false);
        net_wait_count += nw;
        set_busy(0, busy0);
        // both legs of a single jitter-free link: the proposal leg once a
        // draft decode finished, the result leg once a verify did
        if (stage >= 1 || nc > r.nc) r.outd = lk;
        if (stage >= 4 || nc > r.nc) r.backd = lk;
        r.nc = nc;
        r.op[1] = static_cast<uint8_t>(stage >= 3 ? (kOpVerify | 4u) : kOpDecode);
        // the item's enqueue time: the verify's (the proposal arrival) from
        // stage 3 on, else begin_iteration's (stage 2: enqueue() sets it)
        r.enq[1] = stage >= 3 ? base + t2 : (stage == 1 ? base + (nr - l.x) : now);
        switch (stage) {
            case 0:  // the draft is running the decode
                set_phase(r, kPhSpeculating);
                SV(v_run, 1) = static_cast<int32_t>(2 * i + 1);
                set_busy_flag(1, true);
                defer(te, info(kEvComputeDone, 0, 1u));
                break;
            case 1:  // the proposal is on the wire
                set_phase(r, kPhInFlightToTarget);
                defer(te, info(kEvNetArrive, kMsgProposal, static_cast<uint32_t>(i)));
                break;
            case 2:  // the verify waits for the target: the general enqueue + dispatch
                set_phase(r, kPhVerifying);
                enqueue(0, i, 1, kOpVerify, g, true);
                break;
            case 3:  // the target is running the verify
                set_phase(r, kPhVerifying);
                SV(v_run, 0) = static_cast<int32_t>(2 * i + 1);
                set_busy_flag(0, true);
                defer(te, info(kEvComputeDone, 0, 0u));
                break;
            case 4:  // the result is on the wire
                set_phase(r, kPhInFlightToDraft);
                defer(te, info(kEvNetArrive, kMsgResult, static_cast<uint32_t>(i)));
                break;
            default:  // the request is complete
                set_phase(r, kPhInFlightToDraft);
                push_act(act(kActFinish, static_cast<uint32_t>(i)));
                break;
        }
    }

    // finish_request (engine.cpp:449-468) + MetricsCollector::add_record
    DSD_HD void finish_request(int64_t i) {
        ReqRec& r = rec(i);
        r.done = now;
        if (r.first < 0) r.first = now;
        set_phase(r, kPhDone);
        log_tr(i, r, kLogDone);
        const int32_t t = r.target;
        --SV(v_open, t);
        if (r.output >= 2 && ps()) {
            double tpot = (static_cast<double>(now - r.first) / 1000.0) / static_cast<double>(r.output - 1);
            push_tpot(t, tpot);
        }
        int32_t d = D > 0 ? r.drafter : -1;
        if (d >= 0) {
            int32_t v = T + d;
            if (SV(v_active, v) == static_cast<int32_t>(i)) {
                if (hot()) copy_rec(R[i], slot(d));  // write the session back
                SV(v_active, v) = -1;
                push_act(act(kActActivate, static_cast<uint32_t>(d)));
            }
        }
    }

    // commit_tokens (engine.cpp:437-447); returns true when the request is done
    DSD_HD bool commit_tokens(ReqRec& r, int32_t raw) {
        int32_t remaining = r.output - r.tokens;
        int32_t c = raw < remaining ? raw : remaining;
        r.tokens += c;
        record_commit(r, c);
        if (r.first < 0) r.first = now;
        return r.tokens >= r.output;
    }

    // consume_acceptance (engine.cpp:17-32) on the packed bits
    DSD_HD void consume_acceptance(ReqRec& r, int gamma, int& accepted, int& consumed) {
        const uint64_t* bits = W.bits + static_cast<int64_t>(rep) * W.c.bw + r.bitoff;
        const int32_t nb = r.nbits;
        int32_t cur = r.cursor;
        const bool cached = spec && &r == &slot(0);  // the active session: its word is in the slot
        if (gamma > 0 && gamma <= 64 && cur + gamma <= nb) {
            // no wrap inside the window: the accepted prefix is the run of
            // trailing ones of the gamma bits at the cursor
            const int s = cur & 63;
            uint64_t w;
            if (cached) {
                wait_word();
                w = *slot_word() >> s;
            } else {
                w = bits[cur >> 6] >> s;
            }
            if (s + gamma > 64) w |= bits[(cur >> 6) + 1] << (64 - s);
            const uint64_t zeros = ~w;
#ifdef __CUDA_ARCH__
            const int ones = zeros ? __ffsll(static_cast<long long>(zeros)) - 1 : 64;
#else
            const int ones = zeros ? __builtin_ctzll(zeros) : 64;
#endif
            accepted = ones < gamma ? ones : gamma;
            consumed = accepted < gamma ? accepted + 1 : gamma;
            const int32_t old = cur;
            cur += consumed;
            cur = cur == nb ? 0 : cur;
            r.cursor = cur;
            if (cached && (cur >> 6) != (old >> 6)) fetch_word(r, cur);
            return;
        }
        accepted = 0;
        consumed = 0;
        const int32_t old = cur;
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
        r.cursor = cur;
        if (cached && (cur >> 6) != (old >> 6)) fetch_word(r, cur);
    }

    // one member of a finished batch (engine.cpp:573-587, 591-646)
    DSD_HD void item_done(int32_t slot) {
        const int64_t i = slot >> 1;
        const int k = slot & 1;
        ReqRec& r = rec(i);
        const int32_t nxt = r.next[k];
        const uint32_t op = r.op[k] & 3u;
        if (nxt >= 0) push_act(act(kActItem, static_cast<uint32_t>(nxt)));
        if (item_server >= T) {  // draft server
            if (op == kOpPrefill) {
                set_flag(r, kDpd, true);
                if (r.output > 0) defer(now, info(kEvIterStart, 0, static_cast<uint32_t>(i)));
            } else {  // send_proposal (engine.cpp:591-597)
                set_phase(r, kPhInFlightToTarget);
                log_tr(i, r, kLogProposalSent);
                int64_t dl = net_delay(r.drafter, r.target);
                r.outd = static_cast<int32_t>(dl);
                defer(now + dl, info(kEvNetArrive, kMsgProposal, static_cast<uint32_t>(i)));
            }
            return;
        }
        if (op == kOpPrefill) {
            set_flag(r, kTpd, true);
            if (r.output == 0) {
                if (phase(r) != kPhDone) push_act(act(kActFinish, static_cast<uint32_t>(i)));
            } else if (flag(r, kFused) && fe()) {
                push_act(act(kActBegin, static_cast<uint32_t>(i) * 2));
            }
        } else if (op == kOpVerify) {
            int acc, cons;
            consume_acceptance(r, r.tok1, acc, cons);
            r.lcr = acc + 1;
            r.prop += cons;
            r.acc += acc;
            on_verify(r.drafter, r.target, cons, acc);
            int64_t bd = net_delay(r.drafter, r.target);
            r.backd = static_cast<int32_t>(bd);
            set_phase(r, kPhInFlightToDraft);
            log_tr(i, r, kLogVerifyDone);
            defer(now + bd, info(kEvNetArrive, kMsgResult, static_cast<uint32_t>(i)));
        } else {  // fused decode step: commit one token, then the next iteration
            if (commit_tokens(r, 1)) {
                push_act(act(kActFinish, static_cast<uint32_t>(i)));
            } else {
                const bool decide = !(fe() || D == 0 || r.drafter < 0);
                push_act(act(kActBegin, static_cast<uint32_t>(i) * 2 + (decide ? 1u : 0u)));
            }
        }
    }

    // ---- setup + SimKernel::run_until (event_queue.cpp:28-42) ----
    DSD_HD void init() {
        const uint64_t seed = W.rep_seed[rep];
        if (T > 1 && routing_kind() <= 1) {  // the routing stream / rr counter live in HBM
            Rng g;
            g.seed(seed, kLabelRouting);
            uint64_t* st = W.route_state + static_cast<int64_t>(rep) * 5;
            st[0] = g.s0;
            st[1] = g.s1;
            st[2] = g.s2;
            st[3] = g.s3;
            st[4] = 0;
        }
        jitter.seed(seed, kLabelJitter);
        if (probing())
            for (int k = 0; k < kProbeFields; ++k) W.probe[static_cast<int64_t>(rep) * kProbeFields + k] = 0.0;
        if (!spec && W.elog) {
            W.elog_n[rep] = 0;
            W.busy_n[rep] = 0;
        }
        N = (S.workload == 0) ? S.n_requests : S.tr_n;
        seq_next = static_cast<uint32_t>(N);
        if (N > 0) next_arr_t = R[arrival_index(0)].arrival;
        for (int32_t v = 0; v < T + D; ++v) {
            SV(v_qhead, v) = -1;
            SV(v_qtail, v) = -1;
            SV(v_run, v) = -1;
            SV(v_flags, v) = 0;
            if (v < T) {
                SV(v_armseq, v) = 0;
                SV(v_open, v) = 0;
                set_busy(v, 0);
            } else {
                SV(v_active, v) = -1;
                SV(v_shead, v) = -1;
                SV(v_stail, v) = -1;
            }
        }
        if (ps()) {
            for (int32_t t = 0; t < T; ++t) {
                IL(W.t_tcnt, W.c.nt, t) = 0;
                IL(W.t_tpos, W.c.nt, t) = 0;
            }
            int64_t np = static_cast<int64_t>(T) * D;
            for (int64_t p = 0; p < np; ++p) {
                IL(W.p_acc_cnt, W.c.np, p) = 0;
                IL(W.p_acc_pos, W.c.np, p) = 0;
                IL(W.p_rtt_cnt, W.c.np, p) = 0;
                IL(W.p_rtt_pos, W.c.np, p) = 0;
                IL(W.p_gprev, W.c.np, p) = S.gamma;
                IL(W.p_dyn, W.c.np, p) = S.gamma;
                IL(W.p_sm_init, W.c.np, p) = 0;
                IL(W.p_sm_ema, W.c.np, p) = 0.0;
                IL(W.p_sm_low, W.c.np, p) = 0;
                IL(W.p_sm_fused, W.c.np, p) = 0;
            }
        }
    }

    DSD_HD int64_t arrival_index(int64_t k) const {
        if (has_order()) return blob_ptr<int64_t>(W.blob, S.o_tr_order)[k];
        return k;
    }

    // Kind of this replica's next step: the top action, else kActPop while
    // events remain, else kActNone.  The kernel's warp scheduler reads it.
    DSD_HD uint32_t next_kind() const {
        if (fail) return kActNone;
        return next_kind_unchecked();
    }
    // next_kind for the chain loop: a failed replica finishes the (at most two)
    // pending actions - every failure leaves the state bounded: a dropped push
    // or heap insertion, a guarded arena write - and stops at its next pop
    DSD_HD uint32_t next_kind_unchecked() const {
        if (st0 != kStackEmpty) return st0 & 15u;
        return (!fail && (next_arr < N || heap_n > 0)) ? static_cast<uint32_t>(kActPop)
                                                       : static_cast<uint32_t>(kActNone);
    }

    // SimKernel::run_until's pop (event_queue.cpp:28-42): a 2-way merge of the
    // arrival stream (seq 0..N-1, wins every time tie) with the dynamic heap.
    // The event's handler becomes the next action.
    DSD_HD void pop_event() {
        const bool have_arr = next_arr < N;
        if (have_arr && (heap_n == 0 || next_arr_t <= ht(0))) {
            const int64_t ai = arrival_index(next_arr);
            now = next_arr_t;
            ++next_arr;
            // the following arrival's time: not needed before the next pop,
            // so the load's latency hides behind this event
            if (next_arr < N) next_arr_t = R[arrival_index(next_arr)].arrival;
            push_act(act(kActArrival, static_cast<uint32_t>(ai)));
            return;
        }
        const int64_t t = ht(0);
        const uint64_t key = hk(0);
        heap_pop();
        now = t;
        const uint32_t inf = static_cast<uint32_t>(key);
        const uint32_t kind = inf & 7u;
        const uint32_t msg = (inf >> 3) & 3u;
        const uint32_t id = inf >> 5;
        if (kind == kEvIterStart) {
            push_act(act(kActBegin, id * 2 + 1));
        } else if (kind == kEvNetArrive) {
            push_act(act(kActNetPrompt + msg, id));
        } else if (kind == kEvComputeDone) {
            push_act(act(kActComputeDone, id));
        } else if (kind == kEvBatchReady) {  // engine.cpp:265-271
            const int32_t v = static_cast<int32_t>(id);
            if (armed(v) && SV(v_armseq, v) == static_cast<uint32_t>(key >> 32)) {
                set_armed(v, false);
                push_act(act(kActDispatch, static_cast<uint32_t>(v) * 2 + 1));
            }
        }
    }

    static DSD_HD uint32_t opaque(uint32_t x) {
#ifdef __CUDA_ARCH__
        asm volatile("" : "+r"(x));
#endif
        return x;
    }
    // the once-per-request steps
    DSD_HD void step_rare(uint32_t k, uint32_t arg) {
        switch (k) {
            case kActActivate: activate_next_session(static_cast<int32_t>(arg)); break;
            case kActFinish: finish_request(arg); break;
            case kActSendPrompt: {
                const ReqRec& r = rec(arg);
                int64_t delay = net_delay(r.drafter, r.target);
                defer(now + delay, info(kEvNetArrive, kMsgPrompt, arg));
                break;
            }
            case kActArrival: on_arrival(arg); break;
            case kActBeginAwc:
                if (!spec) begin_awc(arg);  // (no AWC in the specialised kernel)
                break;
            default: {  // kActNetPrompt: on_net_arrive (engine.cpp:406-435)
                const ReqRec& r = rec(arg);
                enqueue(r.target, arg, 0, kOpPrefill, r.prompt, true);
                break;
            }
        }
    }

    // Executes exactly one step of kind next_kind().
    DSD_HD void step() {
        if (st0 == kStackEmpty) {
            pop_event();
            // a handler that is not a vote barrier runs in the same step
            if (st0 == kStackEmpty || is_barrier(st0 & 15u, spec, smem_barriers)) return;
        }
        const uint32_t a = pop_act();
        const uint32_t arg = a >> 4;
        const uint32_t k = a & 15u;
        // the frequent kinds as a branch chain in C5 frequency order (dispatch,
        // batch item, compute done, iteration start, proposal, result), the
        // rare ones through a switch: no indirect jump on the hot path (each
        // test reads the kind through opaque() so the compiler cannot fold
        // the chain back into a jump table)
        if (opaque(k) == kActDispatch) {
            try_dispatch(static_cast<int32_t>(arg >> 1), arg & 1u);
        } else if (opaque(k) == kActItem) {
            item_done(static_cast<int32_t>(arg));
        } else if (opaque(k) == kActComputeDone) {  // on_compute_done (engine.cpp:569-589)
            const int32_t v = static_cast<int32_t>(arg);
            set_busy_flag(v, false);
            const int32_t head = SV(v_run, v);
            SV(v_run, v) = -1;
            push_act(act(kActDispatch, static_cast<uint32_t>(v) * 2));
            if (head >= 0) {
                item_server = v;
                push_act(act(kActItem, static_cast<uint32_t>(head)));
            }
        } else if (opaque(k) == kActBegin) {
            if (spec && W.session_fast && (arg & 1u))
                session_run(arg >> 1);
            else
                begin(arg >> 1, arg & 1u);
        } else if (opaque(k) == kActNetProposal) {
            ReqRec& r = rec(arg);
            set_phase(r, kPhVerifying);
            log_tr(arg, r, kLogProposalAtTarget);
            enqueue(r.target, arg, 1, kOpVerify, r.pgamma, true);
        } else if (opaque(k) == kActNetResult) {  // on_result_at_draft (engine.cpp:428-435)
            ReqRec& r = rec(arg);
            if (ps())
                on_rtt_sample(r.drafter, r.target, static_cast<double>(static_cast<int64_t>(r.outd) + r.backd) / 1000.0);
            if (commit_tokens(r, r.lcr)) {
                push_act(act(kActFinish, arg));
            } else {
                defer(now, info(kEvIterStart, 0, arg));
            }
        } else {
            step_rare(k, arg);
        }
        if (pend_t >= 0) {
            schedule(pend_t, pend_info);
            pend_t = -1;
        }
    }

    // Single-replica driver (host debug builds); the kernel interleaves the
    // steps of a warp's replicas with the warp scheduler instead.
    DSD_HD void run() {
        init();
        while (next_kind() != kActNone) step();
        finish();
    }

    // Engine::finish (engine.cpp:648-669) + aggregate_run (runner.cpp:153-169)
    DSD_HD void finish() {
        for (int32_t v = 0; v < T; ++v) IL(W.v_busy_us, W.c.ns, v) = get_busy(v);  // for the records export
        if (hot())  // sessions still active (a failed replica stops early): write them back
            for (int32_t d = 0; d < D; ++d) {
                const int32_t a = SV(v_active, T + d);
                if (a >= 0) copy_rec(R[a], slot(d));
            }
        DevSummary s;
        // every pop is one schedule() or one arrival (event_queue.cpp:38):
        // arrivals popped + dynamic events scheduled - still pending
        s.events_processed = static_cast<uint64_t>(next_arr) + (seq_next - static_cast<uint32_t>(N)) -
                             static_cast<uint64_t>(heap_n);
        s.end_time_us = now;
        s.net_queue_wait_total_us = net_wait_total;
        s.net_queue_wait_count = net_wait_count;
        s.n_requests = N;
        // MetricsCollector's first_arrival_ (min over routed arrivals),
        // last_completion_ and records_.size() (metrics.cpp:47-89)
        int64_t first_arrival = -1, last_completion = -1, completed = 0;
        for (int32_t k = 0; k < next_arr; ++k) {
            const int64_t a = R[k].arrival;
            if (first_arrival < 0 || a < first_arrival) first_arrival = a;
        }
        double ttft = 0.0, tpot = 0.0;
        int64_t n_tpot = 0, n_rec = 0;
        for (int64_t i = 0; i < N; ++i) {  // records sorted by request id
            const ReqRec& r = R[i];
            if (r.done < 0) continue;
            ++completed;
            if (r.done > last_completion) last_completion = r.done;
            ++n_rec;
            ttft += static_cast<double>(r.first - r.arrival) / 1000.0;
            if (r.output >= 2) {
                tpot += (static_cast<double>(r.done - r.first) / 1000.0) / static_cast<double>(r.output - 1);
                ++n_tpot;
            }
        }
        s.mean_ttft_ms = n_rec > 0 ? ttft / static_cast<double>(n_rec) : 0.0;
        s.mean_tpot_ms = n_tpot > 0 ? tpot / static_cast<double>(n_tpot) : 0.0;
        s.completed = completed;
        s.first_arrival_us = first_arrival;
        s.last_completion_us = last_completion;
        s.has_duration = (completed > 0 && last_completion > first_arrival) ? 1 : 0;
        s.throughput_rps = 0.0;
        if (s.has_duration) {
            int64_t dur = last_completion - first_arrival;
            s.throughput_rps = static_cast<double>(completed) / (static_cast<double>(dur) / 1e6);
        }
        s.status = fail ? 3 : 0;
        W.summary[rep] = s;
        W.fail[rep] = fail;
    }
#undef SV
};

// ---------------------------------------------------------------------------
// workload staging: generate_synthetic (trace.cpp:145-187), trace copy, and the
// engine's poisson re-sampling (engine.cpp:224-238).  One thread per replica;
// writes each request's complete initial record.
// ---------------------------------------------------------------------------
DSD_HD void init_record(ReqRec& out, int64_t arrival, int32_t prompt, int32_t output, int32_t drafter,
                        int32_t bitoff, int32_t nbits, int32_t seqoff) {
    // built in registers and written as eight 16-byte stores (records are
    // 128-byte aligned in HBM): each of a warp's lanes writes its own
    // replica's record, so per-field stores would cost a line per field
    union alignas(16) Staged {
        ReqRec r;
        uint4 v[sizeof(ReqRec) / 16];
    } u;
    ReqRec& r = u.r;
    r.arrival = arrival;
    r.first = -1;
    r.done = -1;
    r.enq[0] = 0;
    r.enq[1] = 0;
    r.prompt = prompt;
    r.output = output;
    r.drafter = drafter;
    r.target = -1;
    r.bitoff = bitoff;
    r.nbits = nbits;
    r.tokens = 0;
    r.cursor = 0;
    r.pgamma = 0;
    r.lcr = 0;
    r.outd = 0;
    r.backd = 0;
    r.prop = 0;
    r.acc = 0;
    r.ng = 0;
    r.nc = 0;
    r.snext = -1;
    r.seqoff = seqoff;
    r.next[0] = -1;
    r.next[1] = -1;
    r.tok1 = 0;
    r.flags = 0;
    r.op[0] = 0;
    r.op[1] = 0;
    r.pad = 0;
    uint4* dst = reinterpret_cast<uint4*>(&out);
#pragma unroll
    for (int k = 0; k < static_cast<int>(sizeof(ReqRec) / 16); ++k) dst[k] = u.v[k];
}

DSD_HD void stage_workload(const Workspace& W, int64_t rep) {
    const DevScenario& S = W.scen[W.rep_scen[rep]];
    const char* blob = W.blob;
    ReqRec* R = W.req + rep * W.c.nr;
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
        // bernoulli(alpha) = next_unit() < alpha (rng.cpp:64-66), with
        // next_unit() = (x >> 11) * 2^-53 exact: it holds iff the 53-bit
        // integer (x >> 11) < ceil(alpha * 2^53) (also exact), so each draw
        // is an integer compare instead of a conversion and a multiply
        const uint64_t accept_below = static_cast<uint64_t>(ceil(S.alpha * 0x1.0p53));
        for (int64_t n = 0; n < S.n_requests; ++n) {
            clock_ms += arrivals.exponential(S.mean_gap_ms);
            const int64_t arr = llround(clock_ms * 1000.0);
            int64_t p = llround(lengths.lognormal(S.p_mu, S.p_sigma));
            p = p < 1 ? 1 : (S.p_cap < p ? S.p_cap : p);
            int64_t o = llround(lengths.lognormal(S.o_mu, S.o_sigma));
            o = o < 1 ? 1 : (S.o_cap < o ? S.o_cap : o);
            const int32_t dr = static_cast<int32_t>(drafter.below(static_cast<uint64_t>(S.gen_n_drafts)));
            init_record(R[n], arr, static_cast<int32_t>(p), static_cast<int32_t>(o), dr, static_cast<int32_t>(word),
                        static_cast<int32_t>(o), static_cast<int32_t>(lsum));
            lsum += o;
            bits[word] = static_cast<uint64_t>(o);  // (stashed for the bit loop, which overwrites it)
            word += (o + 63) >> 6;                   // each request's bits start a word
        }
        // The acceptance bits (their own stream, so drawn after the records):
        // one loop over the replica's bit words.  Per-request loops held a
        // warp's lanes for the longest of their requests' outputs every time
        // (half the lanes idle); here a lane waits at most for the rest of
        // another lane's word.
        // (a request's output length comes from its stashed first word, loaded
        // a request ahead; the records' lines are not read back)
        const int64_t N = S.n_requests;
        int32_t rem = N > 0 ? static_cast<int32_t>(bits[0]) : 0;
        int32_t o_next = N > 1 ? static_cast<int32_t>(bits[(rem + 63) >> 6]) : 0;
        int64_t nn = 1;
        for (int64_t w = 0; w < word; ++w) {
            const int m = rem < 64 ? rem : 64;
            uint64_t acc = 0;
            for (int j = 0; j < m; ++j) {
                const uint64_t b = (bitrng.next() >> 11) < accept_below ? 1u : 0u;
                acc |= b << j;
            }
            bits[w] = acc;
            rem -= m;
            if (rem == 0) {
                rem = o_next;
                ++nn;
                o_next = nn < N ? static_cast<int32_t>(bits[w + 1 + ((rem + 63) >> 6)]) : 0;
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
            int64_t arr;
            if (S.workload == 2) {
                clock_ms += arrivals.exponential(1000.0 / S.rate_rps);
                arr = llround(clock_ms * 1000.0);
            } else {
                arr = ta[n];
            }
            const int64_t nb = tb[n + 1] - tb[n];
            init_record(R[n], arr, static_cast<int32_t>(tp[n]), static_cast<int32_t>(to[n]),
                        static_cast<int32_t>(td[n]), static_cast<int32_t>(word), static_cast<int32_t>(nb),
                        static_cast<int32_t>(lsum));
            lsum += to[n];
            for (int64_t k = 0; k < nb; k += 64) {
                int64_t m = nb - k < 64 ? nb - k : 64;
                uint64_t acc = 0;
                for (int64_t j = 0; j < m; ++j) acc |= static_cast<uint64_t>(tbits[tb[n] + k + j] & 1u) << j;
                bits[word++] = acc;
            }
        }
    }
}

}  // namespace dsd
