/*
 * dsd_oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference simulator's hot path, used as the CPU checker for the GPU engine.
 * Only tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() may
 * load it; the product (libdsdsim.so) never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement against the
 * reference itself (oracle/_ref/libspecsim_ref.so, built from
 * /root/reference/proj/src) on the SURVEY Appendix C goldens and on policy
 * variants, byte for byte through the report renderer.
 *
 * Input is the same dsd_scenario / dsd_replica description the product's C ABI
 * takes (include/dsdsim.h); output is the same dsd_replica_summary and
 * dsd_request_record rows, so GPU-vs-oracle comparisons are direct.
 */
#ifndef DSD_ORACLE_H
#define DSD_ORACLE_H
#include "dsdsim.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Number of requests a replica of this scenario simulates. */
int64_t oracle_request_count(const dsd_scenario* s);

/* Upper bound of the flattened gamma/committed sequence length. */
int64_t oracle_sequence_bound(const dsd_scenario* s, const dsd_replica* r);

/* One Engine run (engine.cpp:680-685).  records[oracle_request_count] in
 * request-id order (completion_us == -1 if not finished), gamma/committed
 * flattened in request order (seq_cap entries available), busy_us[n_targets].
 * Any output pointer may be NULL.  Returns DSD_OK or DSD_ERR_*. */
int oracle_run(const dsd_scenario* s, const dsd_replica* r, dsd_replica_summary* summary,
               dsd_request_record* records, int32_t* gamma_seq, int32_t* committed_seq,
               int64_t seq_cap, int64_t* busy_us, char* err, size_t errlen);

/* Many replicas on `threads` host threads (0 = all cores). */
int oracle_run_batch(const dsd_scenario* scenarios, const dsd_replica* replicas, size_t n,
                     int threads, dsd_replica_summary* summaries, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif
