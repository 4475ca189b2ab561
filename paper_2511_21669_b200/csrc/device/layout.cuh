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
enum : int32_t { kFailNone = 0, kFailHeap = 1, kFailAwcDims = 2, kFailSeq = 3 };

struct DevGrid {
    int32_t nb, nc;
    int64_t o_batch, o_ctx, o_vals;  // byte offsets into the blob (double arrays)
    double calibration;
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
    // trace (TRACE / TRACE_POISSON)
    int64_t tr_n;
    int64_t o_tr_prompt, o_tr_output, o_tr_arrival, o_tr_drafter, o_tr_bitoff, o_tr_bits, o_tr_order;
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
};

struct DevSummary {  // == dsd_replica_summary
    uint64_t events_processed;
    int64_t end_time_us, completed, first_arrival_us, last_completion_us;
    int64_t net_queue_wait_total_us, net_queue_wait_count, n_requests;
    double throughput_rps, mean_ttft_ms, mean_tpot_ms;
    int32_t has_duration, status;
};

struct DevRecord {  // == dsd_request_record
    int64_t drafter_id, prompt_length, output_length, arrival_us, first_token_us, completion_us,
        proposed, accepted;
    int32_t target_id, n_iterations;
};

struct Workspace {
    Caps c;
    const char* blob;
    const DevScenario* scen;
    const uint32_t* rep_scen;  // [n]
    const uint64_t* rep_seed;  // [n]
    const uint64_t* rep_gen_seed;
    DevSummary* summary;  // [n]
    int32_t* fail;        // [n]
    // ---- per request (cap nr, interleaved) ----
    int32_t* r_prompt;
    int32_t* r_output;
    int64_t* r_arrival;
    int32_t* r_drafter;
    int32_t* r_bitoff;   // word offset into the replica's bit region
    int32_t* r_nbits;    // acceptance sequence length
    uint8_t* r_flags;    // phase | dpd<<3 | tpd<<4 | fused<<5
    int32_t* r_target;
    int32_t* r_tokens;
    int32_t* r_cursor;   // accept cursor modulo nbits
    int64_t* r_first;
    int64_t* r_done;     // completion time, -1 while running
    int32_t* r_pgamma;
    int32_t* r_lcr;      // last committed raw
    int64_t* r_outd;
    int64_t* r_backd;
    int32_t* r_prop;
    int32_t* r_acc;
    int32_t* r_ng;       // gamma_sequence length
    int32_t* r_nc;       // committed_sequence length
    int32_t* r_snext;    // draft session FIFO link
    int64_t* r_seqoff;   // offset of the request's sequences in the seq arena (records only)
    // ---- work-item slots (cap 2*nr, interleaved): slot 2i = target prefill, 2i+1 = other ----
    uint8_t* s_op;       // op | via_network<<2
    int32_t* s_tok;
    int64_t* s_enq;
    int32_t* s_next;
    // ---- per server (cap ns, interleaved): targets 0..T-1, drafts T.. ----
    int32_t* v_qhead;
    int32_t* v_qtail;
    int32_t* v_run;
    uint8_t* v_busy;
    uint8_t* v_armed;
    uint32_t* v_armseq;
    int64_t* v_busy_us;
    int32_t* v_active;
    int32_t* v_shead;
    int32_t* v_stail;
    int32_t* v_open;
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
    // ---- records (optional) ----
    int32_t collect;
    int64_t* rep_seqbase;  // [n] offset into the sequence arena
    int64_t seq_cap;
    int32_t* seq_gamma;
    int32_t* seq_commit;
};

}  // namespace dsd
