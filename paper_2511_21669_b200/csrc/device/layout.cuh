// layout.cuh — device-side data layout of a replica batch.
//
// HBM layout:
//   * one read-only "scenario blob": DevScenario headers + the arrays they
//     point to (group ids, link table, latency grids, AWC weights, traces),
//     shared by every replica of a scenario;
//   * one workspace of replica state in a warp-interleaved SoA layout: for a
//     field F with per-replica capacity C, replica r = 32*w + lane stores
//     element i at F[(w*C + i)*32 + lane].  A warp's 32 replicas therefore
//     touch one contiguous 32-element row whenever they access the same slot
//     (heap top, server state, per-replica scalars), which is the common case.
#pragma once
#include <cstdint>

namespace dsd {

constexpr int kLanes = 32;
constexpr int kMaxHidden = 64;  // AWC hidden width supported by the engine
// int32 fields per server (Engine::F_*; targets and draft servers use
// disjoint subsets, overlaid)
constexpr int kServerFields = 8;
// Shared-memory variant of the simulation kernel (<= kSmemServers servers):
// per-warp server state, the first heap slots and the draft servers' active
// sessions live in shared memory; a replica whose dynamic event heap outgrows
// it is re-run on the HBM variant.
constexpr int kSmemServers = 4;
constexpr int kProbeFields = 8;  // Workspace::probe entries per replica

// Event kinds (proj/include/specsim/sim/event_queue.hpp:12-18).
enum : uint32_t { kEvArrival = 0, kEvBatchReady = 1, kEvComputeDone = 2, kEvNetArrive = 3, kEvIterStart = 4 };
// NetArrive payload tags (engine.cpp:108-111).
enum : uint32_t { kMsgPrompt = 0, kMsgProposal = 1, kMsgResult = 2 };
// OpKind (profile.hpp:10).
enum : uint32_t { kOpPrefill = 0, kOpDecode = 1, kOpVerify = 2 };
// ReqPhase (engine.cpp:36-45).
enum : uint32_t {
    kPhArrived = 0, kPhRouted, kPhQueuedPrefill, kPhSpeculating, kPhInFlightToTarget,
    kPhVerifying, kPhInFlightToDraft, kPhDone
};

// Per-replica failure codes (summary.status carries DSD_ERR_RUNTIME, detail here).
enum : int32_t { kFailNone = 0, kFailHeap = 1, kFailAwcDims = 2, kFailSeq = 3, kFailStack = 4 };

// Segment of a clamped integer query on one grid axis: the bracketing
// indices and the interpolation weight, exactly as Grid::interpolate computes
// them (profile.cpp:57-88).  Latency queries are integers (batch size,
// batch*tokens, prompt or context tokens), so each axis gets a table indexed
// by the query, built on the host with the same formula.
struct AxisSeg {
    int32_t lo, hi;
    double t;
};

struct DevLink {  // LinkSpec (topology.hpp:25-30) + the jitter-free delay
    double rtt_ms, jitter_ms;
    int64_t fixed_us;
};

struct DevGrid {
    int32_t nb, nc;
    int64_t o_batch, o_ctx, o_vals;  // byte offsets into the blob (double arrays)
    double calibration;
    int64_t o_btab, o_ctab;          // AxisSeg tables (-1: query by binary search)
    int32_t nbt, nct;                // table sizes; queries >= size use the last entry
};

// A resolved scenario (dsd_scenario) in device form.  Offsets are bytes into
// the scenario blob.
struct DevScenario {
    int32_t n_targets, n_drafts, n_tg, n_dg;
    int32_t routing, batching, max_batch, draft_max_batch;
    int32_t window_kind, gamma, gamma_min, gamma_max;
    int32_t queue_capacity, fused_everything, workload, pair_stats;
    int64_t batching_window_us;
    double sim_frac;
    // workload
    int64_t n_requests;
    double rate_rps;
    double mean_gap_ms;  // 1000 / rate (generator) or re-sampling mean
    double alpha;
    double p_mu, p_sigma, o_mu, o_sigma;  // log(median) computed on the host with libm
    int64_t p_cap, o_cap, gen_n_drafts;
    // arrays
    int64_t o_tgroup, o_dgroup, o_links, o_tgrid, o_dgrid, o_grids;
    int32_t n_grids, awc_hidden;
    int32_t awc_blocks, awc_input;
    int64_t o_awc_params;
    double awc_lo[5], awc_hi[5];
    int32_t awc_log[5], has_order;
    int32_t jitter_free, pad0;  // every link has jitter 0: net_delay is DevLink::fixed_us
    // trace (TRACE / TRACE_POISSON)
    int64_t tr_n;
    int64_t o_tr_prompt, o_tr_output, o_tr_arrival, o_tr_drafter, o_tr_bitoff, o_tr_bits, o_tr_order;
    // specialised kernel: offset (int32 elements) of this scenario's session
    // latency table in Workspace::spec_lat, or -1 (Engine::session_run)
    int64_t o_slat;
};

// Per-batch capacities (max over the batch's scenarios).
struct Caps {
    int64_t nr;      // requests per replica
    int64_t ns;      // servers per replica (targets + drafts)
    int64_t nt;      // targets
    int64_t np;      // pairs with ring statistics (0 when no replica needs them)
    int64_t hc;      // event-heap capacity
    int64_t bw;      // acceptance-bit words per replica
    int64_t n;       // replicas
    int64_t nwarps;  // ceil(n / 32)
    int64_t awc;     // some scenario decides windows with the AWC model (cooperative scratch needed)
};

struct DevSummary {  // == dsd_replica_summary
    uint64_t events_processed;
    int64_t end_time_us, completed, first_arrival_us, last_completion_us;
    int64_t net_queue_wait_total_us, net_queue_wait_count, n_requests;
    double throughput_rps, mean_ttft_ms, mean_tpot_ms;
    int32_t has_duration, status;
};

// One log_transition line (engine.cpp:213-219), rendered on the host.
enum : uint8_t { kLogRouted = 0, kLogSpeculating, kLogProposalSent, kLogProposalAtTarget, kLogVerifyDone, kLogDone };
struct ElogRec {
    int64_t t;
    int32_t req, draft, target;
    uint8_t phase, detail, pad[2];
};
static_assert(sizeof(ElogRec) == 24, "event-log record layout");
// One BusyInterval (engine.hpp:37-42, engine.cpp:563-564): server = the
// target index, or ~(draft index) for a draft server.
struct BusyRec {
    int64_t start, end;
    int32_t server, pad;
};
static_assert(sizeof(BusyRec) == 24, "busy-interval record layout");

struct DevRecord {  // == dsd_request_record
    int64_t drafter_id, prompt_length, output_length, arrival_us, first_token_us, completion_us,
        proposed, accepted;
    int32_t target_id, n_iterations;
};

// Everything the engine keeps about one request (RequestState, engine.cpp:86-106,
// plus its two work-item slots) in a single 128-byte line, so the handful of
// fields an event touches cost one L1 line instead of one line per field.
// Work-item slot k of request i has id 2*i + k: k = 0 is the target prefill
// item, k = 1 is the request's other item (draft prefill / draft decode /
// verify / fused decode); a request never has two items of the same slot.
// Records are 128-byte aligned in HBM (one line each); the shared-memory
// copies of active sessions (Engine::rec) sit at a kHotStride lane stride,
// so the struct itself only asks for 8-byte alignment.
struct ReqRec {
    int64_t arrival;       // arrival event time (trace or re-sampled)
    int64_t first;         // first-token time, -1 before the first commit
    int64_t done;          // completion time, -1 while running
    int64_t enq[2];        // enqueue time of slot 0 / 1
    int32_t prompt, output;
    int32_t drafter, target;
    int32_t bitoff, nbits;  // packed acceptance bits: word offset, length
    int32_t tokens, cursor;  // tokens_done, accept cursor (mod nbits)
    int32_t pgamma, lcr;     // pending gamma, last committed raw
    int32_t outd, backd;     // the two legs of the last exchange (us)
    int32_t prop, acc;       // proposed_total, accepted_total
    int32_t ng, nc;          // gamma_sequence / committed_sequence lengths
    int32_t snext, seqoff;   // draft session FIFO link, sequence-arena offset
    int32_t next[2];         // work-queue / running-batch links of slot 0 / 1
    int32_t tok1;            // tokens of slot 1 (slot 0 always carries the prompt)
    uint8_t flags;           // phase | dpd<<3 | tpd<<4 | fused<<5
    uint8_t op[2];           // op | via_network<<2 of slot 0 / 1
    uint8_t pad;
};
static_assert(sizeof(ReqRec) == 128, "request record must be one 128-byte line");
constexpr int kHotStride = 136;  // 34 words: at most 2-way bank conflicts, 8-byte aligned

struct Workspace {
    Caps c;
    const char* blob;
    const DevScenario* scen;
    const uint32_t* rep_scen;  // [n]
    const uint64_t* rep_seed;  // [n]
    const uint64_t* rep_gen_seed;
    DevSummary* summary;  // [n]
    int32_t* fail;        // [n]
    // ---- per request: one 128-byte record, replica-contiguous [n][nr] ----
    ReqRec* req;
    // ---- per server (cap ns, interleaved): targets 0..T-1, drafts T.. ----
    // kServerFields int32 fields x ns servers per warp block (queue head/tail,
    // running batch, busy, armed, armed-event seq, active session, session
    // FIFO head/tail, open requests); used when the batch runs the HBM variant
    int32_t* srv;
    int64_t* v_busy_us;
    // routing stream (4 words) + round-robin counter, replica-contiguous [n][5];
    // touched only by random / rr routing over more than one target
    uint64_t* route_state;
    // ---- per target TPOT ring (cap nt*50) and per pair stats (cap np) ----
    double* t_tpot;
    int32_t* t_tpos;     // cap nt
    int32_t* t_tcnt;     // cap nt
    int32_t* p_acc_ex;   // cap np*20
    int32_t* p_acc_ac;   // cap np*20
    int32_t* p_acc_pos;  // cap np
    int32_t* p_acc_cnt;
    double* p_rtt;       // cap np*20
    int32_t* p_rtt_pos;
    int32_t* p_rtt_cnt;
    int32_t* p_gprev;
    int32_t* p_dyn;
    uint8_t* p_sm_init;
    double* p_sm_ema;
    int32_t* p_sm_low;
    uint8_t* p_sm_fused;
    // ---- event heap (cap hc, interleaved) ----
    int64_t* h_time;
    uint64_t* h_key;     // seq<<32 | info
    // ---- acceptance bits: replica-contiguous [n][bw] ----
    uint64_t* bits;
    // ---- optional feature probe (dsd_run_opts.feature_probe): [n][kProbeFields]
    // feature sums f0..f4, feature samples, chosen-window sum, decisions
    double* probe;
    // ---- optional step profile (DSD_STEP_STATS=1): [2k] cycles, [2k+1] count
    // per step kind, [32] warp iterations, [33] warp cycles, [34] max iterations
    unsigned long long* step_stats;
    // ... and per replica [n][3]: vote rounds it ran in, session-loop
    // iterations (builds with -DDSD_REP_STATS), cycles from init to finish
    unsigned long long* rep_stats;
    // solo mode (small batches of large topologies): one replica per block of
    // one warp, lane 0; its server state and an event heap of solo_hcap slots
    // in shared memory at lane stride 1, and (solo_rec) its request records too
    int32_t solo, solo_hcap, solo_rec, pad_solo;
    // AWC batches: blob offset / double count of the one WC-DNN (transposed
    // layout) the kAwc blocks stage into shared memory, or -1
    int64_t awc_stage_off;
    int32_t awc_stage_n;
    int32_t pad_awc;
    // specialised kernel: run the active session's speculation loop directly
    // (Engine::session_run); env DSD_SESSION_FAST=0 disables it
    int32_t session_fast;
    // session latency tables of the specialised kernel (built by k_spec_lat
    // at prepare): per (draft decode grid, verify grid, gamma) a status word
    // (0: every entry below 2^28 us), then for each context c in [0, n) the
    // pair {draft decode of gamma tokens at (1, c), verify at (gamma, c)} in
    // us - latency_us() of both queries, so looking one up is exact
    const int32_t* spec_lat;
    // ---- event log + busy intervals (optional, EngineOptions::collect_event_log):
    // per replica a region of elog_cap / busy_cap records at replica * cap,
    // filled in event order; counts in elog_n / busy_n
    ElogRec* elog;
    BusyRec* busy_iv;
    int64_t elog_cap, busy_cap;
    int64_t* elog_n;
    int64_t* busy_n;
    // ---- records (optional) ----
    int32_t collect;
    int64_t* rep_seqbase;  // [n] offset into the sequence arena
    int64_t seq_cap;
    int32_t* seq_gamma;
    int32_t* seq_commit;
};

}  // namespace dsd
