/*
 * dsdsim.h — C ABI of the B200-native DSD-Sim replica engine (libdsdsim.so).
 *
 * This is the drop-in boundary for the reference's simulate-a-sweep path
 * (arxiv 2511.21669 "specsim", /root/reference/proj).  The reference exposes
 * that path as a C++ class API, not an FFI; each entry point below names the
 * reference interface it replaces:
 *
 *   dsd_run_simulation  <- resolve_config + run_simulation + aggregate_run
 *                          (proj/include/specsim/runner/runner.hpp:36-60,
 *                           proj/src/runner/runner.cpp:96-169) and the
 *                          `specsim run` front end (tools/specsim_main.cpp:50-78)
 *   dsd_run_sweep       <- SweepSpec::from_node + run_sweep + sweep_summary_*
 *                          (proj/include/specsim/runner/sweep.hpp:17-50,
 *                           proj/src/runner/sweep.cpp:16-199) and `specsim sweep`
 *                          (tools/specsim_main.cpp:80-95)
 *   dsd_run_batch       <- N independent Engine(topology, profile, trace, mode,
 *                          seed, options, awc).run() calls
 *                          (proj/include/specsim/engine/engine.hpp:59-74);
 *                          a dsd_scenario is a ResolvedConfig (runner.hpp:20-28)
 *                          and a dsd_replica is one (scenario, seed) run
 *   dsd_fetch_records   <- RunResult::records / MetricsRecord
 *                          (engine.hpp:44-53, metrics.hpp:13-30)
 *
 * Conventions
 *   - Plain C types only; the caller owns every host buffer, the library owns
 *     device memory.  No callbacks, no exceptions cross the ABI.
 *   - Status codes mirror the reference CLI exit codes
 *     (tools/specsim_main.cpp:24-27, 293-311): DSD_OK, DSD_ERR_CONFIG (parse /
 *     config / validation / unknown profile key / corrupt model), DSD_ERR_RUNTIME.
 *     A human-readable message with the reference's error text is written to
 *     err[0..errlen).
 *   - A handle drives one or more CUDA devices (dsd_create_devices) and must
 *     be used from one host thread at a time (the reference Engine is
 *     single-threaded too).  The replicas of every batch / sweep
 *     are dealt across the handle's devices in cost order and run
 *     concurrently, one stream per device; results always come back in the
 *     caller's replica order, identical to a one-device run.  (One process
 *     per GPU, each with a one-device handle and dsd_prepare_sweep's shards,
 *     is the other way to use several GPUs.)
 *     Internally the sweep planning and summary loops run on a process-wide
 *     pool of host worker threads (DSD_HOST_THREADS), and dsd_run_sweep frees
 *     its host batch on a helper thread that the next call or dsd_destroy
 *     joins; neither is visible through the ABI.
 *   - There is no CPU fallback: every simulation runs in the sm_100a kernels.
 *     Creating a handle without a usable GPU fails with DSD_ERR_RUNTIME.
 */
#ifndef DSDSIM_H
#define DSDSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSD_ABI_VERSION 2

#define DSD_OK 0
#define DSD_ERR_CONFIG 2
#define DSD_ERR_RUNTIME 3

/* Policy enums: RoutingKind / BatchingKind / WindowKind
 * (proj/include/specsim/config/topology.hpp:32-34). */
enum { DSD_ROUTE_RANDOM = 0, DSD_ROUTE_ROUND_ROBIN = 1, DSD_ROUTE_JSQ = 2 };
enum { DSD_BATCH_FIFO = 0, DSD_BATCH_LAB = 1 };
enum { DSD_WINDOW_STATIC = 0, DSD_WINDOW_DYNAMIC = 1, DSD_WINDOW_AWC = 2, DSD_WINDOW_FUSED = 3 };

/* Workload kinds (runner.cpp:103-133):
 *   SYNTHETIC      mode: poisson without a trace file: generate_synthetic(spec,
 *                  gen_seed) on the device, then trace-driven arrivals.
 *   TRACE          mode: trace: the trace's arrival_us verbatim.
 *   TRACE_POISSON  mode: poisson with a trace file: trace records, arrivals
 *                  re-sampled from the engine's "arrivals" stream
 *                  (engine.cpp:224-238). */
enum { DSD_WORKLOAD_SYNTHETIC = 0, DSD_WORKLOAD_TRACE = 1, DSD_WORKLOAD_TRACE_POISSON = 2 };

/* One latency grid, LatencyProfile::Grid (proj/include/specsim/latency/profile.hpp:33-42). */
typedef struct dsd_grid {
    int32_t n_batch;
    int32_t n_context;
    const double* batch_axis;   /* [n_batch], strictly increasing */
    const double* context_axis; /* [n_context], strictly increasing */
    const double* values_ms;    /* [n_batch * n_context], row-major [batch][context] */
    double calibration;
} dsd_grid;

/* LinkSpec (topology.hpp:25-30). */
typedef struct dsd_link {
    double rtt_ms;
    double jitter_ms;
} dsd_link;

/* AwcModel (proj/include/specsim/awc/mlp.hpp:80-96): WcDnn parameters in the
 * reference's flat layout (mlp.cpp:20-48) plus the FeatureNormalizer. */
typedef struct dsd_awc_model {
    int32_t input;  /* must be 5 */
    int32_t hidden;
    int32_t blocks;
    int32_t reserved;
    const double* params; /* hidden*input + hidden + blocks*(2*hidden*hidden + 2*hidden) + hidden + 1 */
    double norm_lo[5];
    double norm_hi[5];
    int32_t log_scale[5];
} dsd_awc_model;

/* A workload trace, TraceRecord[] (proj/include/specsim/workload/trace.hpp:14-22). */
typedef struct dsd_trace {
    int64_t n;
    const int64_t* prompt_length; /* [n] */
    const int64_t* output_length; /* [n] */
    const int64_t* arrival_us;    /* [n] */
    const int64_t* drafter_id;    /* [n] */
    const int64_t* bits_offset;   /* [n+1] offsets into acceptance_bits */
    const uint8_t* acceptance_bits; /* concatenated 0/1 acceptance sequences */
} dsd_trace;

/* A fully resolved scenario == ResolvedConfig (runner.hpp:20-28) with the
 * expanded Topology (topology.hpp:68-91) flattened to arrays.  Arrays may be
 * shared between scenarios (they are uploaded once per distinct pointer). */
typedef struct dsd_scenario {
    /* expanded pools: device ids are array indices */
    int32_t n_targets;
    int32_t n_drafts;
    int32_t n_target_groups;
    int32_t n_draft_groups;
    const int32_t* target_group; /* [n_targets] declaration group */
    const int32_t* draft_group;  /* [n_drafts] */
    /* resolved per-(draft group, target group) link: the override when one is
     * declared, otherwise the default link (Topology::link, topology.cpp:172-177) */
    const dsd_link* links; /* [n_draft_groups * n_target_groups], row = draft group */
    /* latency grids and, per device, the (prefill, decode) grid indices of its
     * (model, hardware) key; -1 when the profile has no such entry */
    int32_t n_grids;
    const dsd_grid* grids;
    const int32_t* target_grids; /* [n_targets * 2] */
    const int32_t* draft_grids;  /* [n_drafts * 2] */
    /* PolicyConfig (topology.hpp:36-66) */
    int32_t routing;
    int32_t batching;
    int32_t max_batch_size;
    int32_t draft_max_batch;
    int64_t batching_window_us;
    double similarity_fraction;
    int32_t window_kind;
    int32_t gamma;
    int32_t gamma_min;
    int32_t gamma_max;
    int32_t queue_capacity;
    int32_t reserved0;
    const dsd_awc_model* awc; /* required when window_kind == AWC and n_drafts > 0 */
    /* workload */
    int32_t workload;
    int32_t reserved1;
    double rate_rps;        /* SYNTHETIC: generator rate; TRACE_POISSON: re-sampling rate */
    int64_t n_requests;     /* SYNTHETIC */
    double acceptance_rate; /* SYNTHETIC */
    double prompt_median, prompt_sigma, output_median, output_sigma; /* SYNTHETIC LengthDist */
    int64_t prompt_cap, output_cap;                                  /* SYNTHETIC LengthDist */
    int64_t gen_n_drafts;   /* SYNTHETIC: max(1, n_drafts) in the reference resolver */
    const dsd_trace* trace; /* TRACE / TRACE_POISSON */
} dsd_scenario;

/* One replica = one Engine run: scenario index, engine seed (streams
 * "routing", "jitter", "arrivals", engine.cpp:159-161) and the synthetic
 * generator seed (workload.gen_seed, default = seed, runner.cpp:123-125). */
typedef struct dsd_replica {
    uint32_t scenario;
    uint32_t reserved;
    uint64_t seed;
    uint64_t gen_seed;
} dsd_replica;

typedef struct dsd_run_opts {
    int32_t collect_records; /* keep per-request records + sequences for dsd_fetch_records */
    int32_t feature_probe;   /* EngineOptions::feature_probe (engine.hpp:34): per-replica AWC
                                feature sums, read back with dsd_batch_probe */
    int32_t collect_event_log; /* EngineOptions::collect_event_log (engine.hpp:32-35): the
                                  log_transition lines and RunResult::busy_intervals
                                  (engine.cpp:213-219, 563-564), read back with
                                  dsd_fetch_event_log; implies collect_records */
    int32_t reserved;
} dsd_run_opts;

/* BusyInterval (proj/include/specsim/engine/engine.hpp:37-42). */
typedef struct dsd_busy_interval {
    int32_t role; /* 0 = target (Role::Target), 1 = draft */
    int32_t server_id;
    int64_t start_us;
    int64_t end_us;
} dsd_busy_interval;

/* Per-replica result: RunResult scalars (engine.hpp:44-53), the SystemMetrics
 * fields that are not percentiles (metrics.hpp:38-47) and RunAggregates
 * (runner.hpp:53-60). */
typedef struct dsd_replica_summary {
    uint64_t events_processed;
    int64_t end_time_us;
    int64_t completed;
    int64_t first_arrival_us;   /* -1 when nothing arrived */
    int64_t last_completion_us; /* -1 when nothing completed */
    int64_t net_queue_wait_total_us;
    int64_t net_queue_wait_count;
    int64_t n_requests;
    double throughput_rps; /* 0 when undefined, as aggregate_run's value_or(0) */
    double mean_ttft_ms;
    double mean_tpot_ms;
    int32_t has_duration; /* SystemMetrics::duration_ms has a value */
    int32_t status;       /* DSD_OK or DSD_ERR_RUNTIME (capacity overflow) */
} dsd_replica_summary;

/* MetricsRecord inputs (metrics.hpp:13-30, finalize_request metrics.cpp:172-201). */
typedef struct dsd_request_record {
    int64_t drafter_id; /* -1 in fused-only deployments */
    int64_t prompt_length;
    int64_t output_length;
    int64_t arrival_us;
    int64_t first_token_us;
    int64_t completion_us; /* -1 if the request never finished */
    int64_t proposed;
    int64_t accepted;
    int32_t target_id;
    int32_t n_iterations; /* length of gamma_sequence == committed_sequence */
} dsd_request_record;

typedef struct dsd_handle dsd_handle;

/* Library / device management.  dsd_create(d) == dsd_create_devices(&d, 1).
 * dsd_create_devices replaces run_sweep's `parallelism` worker pool
 * (proj/src/runner/sweep.cpp:109-160) with a list of GPUs: every entry point
 * that takes the handle spreads its replicas over all of them. */
int dsd_abi_version(void);
int dsd_create(int device_ordinal, dsd_handle** out, char* err, size_t errlen);
int dsd_create_devices(const int* device_ordinals, int n_devices, dsd_handle** out, char* err, size_t errlen);
int dsd_device_count(dsd_handle* h);
/* Replicas of the prepared batch on each device (returns the device count). */
int dsd_batch_shard_sizes(dsd_handle* h, int64_t* sizes, int cap);
void dsd_destroy(dsd_handle* h);

/* Runs n replicas of the given scenarios on the handle's GPU (one Engine run
 * each).  summaries[n] is filled on success. */
int dsd_run_batch(dsd_handle* h, const dsd_scenario* scenarios, size_t n_scenarios,
                  const dsd_replica* replicas, size_t n, const dsd_run_opts* opts,
                  dsd_replica_summary* summaries, char* err, size_t errlen);

/* After a dsd_run_batch with collect_records: per-request records of one
 * replica (request-id order) and its flattened sequences.  busy_us[n_targets]
 * receives Server::busy_us per target (engine.cpp:562, feeds utilization).
 * gamma_seq/committed_seq receive sum(n_iterations) entries in request order.
 * Pass NULL for any output to skip it.  *n_records / *n_seq return the sizes. */
int dsd_fetch_records(dsd_handle* h, size_t replica, dsd_request_record* records,
                      size_t records_cap, int64_t* n_records, int32_t* gamma_seq,
                      int32_t* committed_seq, size_t seq_cap, int64_t* n_seq, int64_t* busy_us,
                      size_t busy_cap, char* err, size_t errlen);

/* After a dsd_run_batch with collect_event_log: RunResult::event_log of one
 * replica rendered exactly as the reference's log_transition lines, one per
 * line with a trailing newline (what `specsim run --event-log` writes,
 * tools/specsim_main.cpp:65-72; malloc'd, dsd_free), and its busy intervals
 * in dispatch order (intervals[0..cap), *n_intervals = the count). */
int dsd_fetch_event_log(dsd_handle* h, size_t replica, char** event_log, dsd_busy_interval* intervals,
                        size_t cap, int64_t* n_intervals, char* err, size_t errlen);

/* --- device-resident batch (for measurement: inputs stay in HBM) --------- */
/* Uploads scenarios + replicas once; dsd_batch_launch then runs the kernels
 * asynchronously on the handle's stream with no host<->device traffic;
 * dsd_batch_sync waits; dsd_batch_summaries copies the summaries back. */
int dsd_batch_prepare(dsd_handle* h, const dsd_scenario* scenarios, size_t n_scenarios,
                      const dsd_replica* replicas, size_t n, const dsd_run_opts* opts,
                      char* err, size_t errlen);
int dsd_batch_launch(dsd_handle* h, char* err, size_t errlen);
int dsd_batch_sync(dsd_handle* h, char* err, size_t errlen);
int dsd_batch_summaries(dsd_handle* h, dsd_replica_summary* summaries, size_t n, char* err,
                        size_t errlen);
/* Device pointer + byte size of the summary array of the prepared batch
 * (valid until the next prepare/destroy); lets a caller gather it with NCCL.
 * One-device handles only. */
int dsd_batch_device_summaries(dsd_handle* h, void** dev_ptr, size_t* bytes);
/* cudaStream_t of the handle, as an opaque pointer (for event timing). */
void* dsd_stream(dsd_handle* h);
/* Kernel launches issued by the last dsd_batch_launch / dsd_run_batch. */
int64_t dsd_last_launch_count(dsd_handle* h);
/* Duration (ms, CUDA events on the handle's stream) of the simulation kernel
 * of the last launch (the dominant kernel) and of the whole launch. */
int dsd_last_kernel_ms(dsd_handle* h, double* sim_kernel_ms, double* gen_kernel_ms,
                       double* total_ms);
/* Host->device bytes of the last prepare (scenario blob + headers + replica
 * table) and device->host bytes of the last summaries/records copy. */
int dsd_last_transfer_bytes(dsd_handle* h, int64_t* h2d_bytes, int64_t* d2h_bytes);

/* --- config-level entry points (the reference's C++ API, via YAML) -------- */

/* resolve_config(yaml, strict, seed_override, base_dir) + run_simulation +
 * aggregate_run.  report_json / report_csv (emit_report / emit_report_csv,
 * metrics.cpp:203-302) are malloc'd; free them with dsd_free.
 * agg = {completed, throughput_rps, mean_ttft_ms, mean_tpot_ms}. */
int dsd_run_simulation(dsd_handle* h, const char* config_yaml, const char* base_dir, int strict,
                       int has_seed, uint64_t seed, char** report_json, char** report_csv,
                       uint64_t* events_processed, int64_t* end_time_us, double* agg,
                       char* err, size_t errlen);

/* dsd_run_simulation with EngineOptions::collect_event_log: additionally the
 * run's event log text and busy intervals (as dsd_fetch_event_log) - the
 * `specsim run --event-log` path (tools/specsim_main.cpp:50-78). */
int dsd_run_simulation_traced(dsd_handle* h, const char* config_yaml, const char* base_dir, int strict,
                              int has_seed, uint64_t seed, char** report_json, char** event_log,
                              dsd_busy_interval* intervals, size_t cap, int64_t* n_intervals,
                              uint64_t* events_processed, char* err, size_t errlen);

/* SweepSpec::from_node + run_sweep + sweep_summary_json/csv.  When out_dir is
 * non-empty the per-replica reports are written there with the reference's
 * file names (sweep.cpp:134-140).  totals = {points, replicas, failed_points,
 * events_processed}.  Summaries are malloc'd (dsd_free). */
int dsd_run_sweep(dsd_handle* h, const char* sweep_yaml, const char* base_dir,
                  const char* out_dir, char** summary_json, char** summary_csv,
                  double* totals, char* err, size_t errlen);

/* Resolves a sweep spec into scenarios+replicas and prepares it on the
 * handle's device(s) (dsd_batch_prepare) without running it; returns the
 * replica count.  With n_shards > 1 only shard `shard` of the replicas is
 * kept - the cost-ordered deal dsd_create_devices makes (shard_of_replicas:
 * replicas by decreasing estimated cost, dealt 0..N-1, N-1..0, ...), in
 * point-major order - i.e. one GPU's share of the sweep when each GPU has
 * its own process.  Used by the benchmark to time the kernels with inputs
 * resident in HBM. */
int dsd_prepare_sweep(dsd_handle* h, const char* sweep_yaml, const char* base_dir, int shard,
                      int n_shards, int64_t* n_replicas, int64_t* n_points, char* err,
                      size_t errlen);

/* --- host-only helpers (no GPU needed) ----------------------------------- */

/* resolve_config (runner.cpp:96-134) without running: the dsd_scenario and
 * dsd_replica a config resolves to, plus its report digest.  The resolved
 * object owns every array the scenario points to. */
typedef struct dsd_resolved dsd_resolved;
int dsd_resolve_config(const char* config_yaml, const char* base_dir, int strict, int has_seed,
                       uint64_t seed, dsd_resolved** out, char* err, size_t errlen);
const dsd_scenario* dsd_resolved_scenario(const dsd_resolved* r);
void dsd_resolved_replica(const dsd_resolved* r, dsd_replica* out);
const char* dsd_resolved_digest(const dsd_resolved* r);
void dsd_resolved_free(dsd_resolved* r);

/* Resolves a sweep spec into scenarios + replicas without running it (the
 * object owns the arrays).  Replicas are point-major, repetition-minor; with
 * n_shards > 1 only the shard's replicas are kept (the cost-ordered deal),
 * exactly the set dsd_prepare_sweep(shard, n_shards) runs.  dsd_sweep_plan_origin
 * returns, per kept replica, its (point index, repetition). */
typedef struct dsd_sweep_plan dsd_sweep_plan;
int dsd_plan_sweep(const char* sweep_yaml, const char* base_dir, int shard, int n_shards,
                   dsd_sweep_plan** out, char* err, size_t errlen);
size_t dsd_sweep_plan_origin(const dsd_sweep_plan* p, int64_t* point, int32_t* repetition,
                             size_t cap);
size_t dsd_sweep_plan_scenarios(const dsd_sweep_plan* p, const dsd_scenario** scenarios);
size_t dsd_sweep_plan_replicas(const dsd_sweep_plan* p, const dsd_replica** replicas);
void dsd_sweep_plan_free(dsd_sweep_plan* p);

/* emit_report / emit_report_csv (metrics.cpp:203-302) from per-request
 * records in request-id order, flattened sequences and per-target busy time. */
int dsd_emit_report(const dsd_replica_summary* summary, const dsd_request_record* records,
                    size_t n_records, const int32_t* gamma_seq, const int32_t* committed_seq,
                    size_t n_seq, const int64_t* busy_us, int n_targets, const char* digest,
                    uint64_t seed, char** report_json, char** report_csv);

/* The canonical sweep seed derivation (sweep.cpp:51-57), exposed for tests. */
uint64_t dsd_sweep_point_seed(uint64_t base_seed, const char* point_id, int repetition);

/* After a batch prepared with dsd_run_opts.feature_probe: DSD_PROBE_FIELDS
 * doubles per replica - the sums of the AWC feature vector over the
 * iterations of requests with a draft server (features.cpp:5-13), their
 * count (RunResult::mean_features = sums / count, engine.cpp:660-664), the
 * sum of chosen windows (fused counted as 1) and the number of decisions. */
#define DSD_PROBE_FIELDS 8
int dsd_batch_probe(dsd_handle* h, double* out, size_t n, char* err, size_t errlen);

/* ---- AWC dataset generation and policy evaluation ----
 * build_scenarios (dataset.cpp:50-87) of a DatasetGrid YAML document
 * (DatasetGrid::from_node, dataset.cpp:33-48; NULL or "" = the defaults),
 * serialized as serialize_scenarios' JSONL (dataset.cpp:89-108).  Host only. */
int dsd_build_scenarios(const char* grid_yaml, char** scenarios_jsonl, char* err, size_t errlen);

/* generate_dataset (dataset.cpp:258-290) over build_scenarios(grid): every
 * scenario x 12 candidates (static gamma 2..12, fused) as one device batch
 * with the feature probe.  weights = {w_tpot, w_ttft, w_throughput} or NULL
 * for ObjectiveWeights{} (dataset.hpp:55-59).  Returns serialize_dataset's
 * JSONL (train.cpp:16-33) and the scenarios JSONL, as `specsim gen-dataset`
 * writes dataset.jsonl / scenarios.jsonl (specsim_main.cpp:97-112). */
int dsd_generate_dataset(dsd_handle* h, const char* grid_yaml, const double* weights, char** dataset_jsonl,
                         char** scenarios_jsonl, char* err, size_t errlen);

/* eval_policy_on_scenarios (dataset.cpp:292-369) on the scenarios of a
 * scenarios JSONL whose split matches ("all" = every scenario; none ->
 * DSD_ERR_CONFIG as specsim_main.cpp:131-138): window_kind static / dynamic /
 * awc / fused with gamma and (awc) the model path.  out[4] = mean
 * throughput_rps, mean_ttft_ms, mean_tpot_ms, mean chosen gamma. */
int dsd_eval_policy(dsd_handle* h, const char* scenarios_jsonl, const char* split, const char* window_kind,
                    int gamma, const char* model_path, double* out, char* err, size_t errlen);

void dsd_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* DSDSIM_H */
