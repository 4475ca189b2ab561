// runtime.cu — packs resolved scenarios into a device blob, sizes the replica
// workspace, and launches the staging + simulation kernels for sm_100a.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <tuple>
#include <vector>

#include "engine.cuh"
#include "pack.hpp"
#include "runtime.hpp"

namespace dsd {

static_assert(sizeof(DevSummary) == sizeof(dsd_replica_summary), "summary layout");
static_assert(sizeof(DevRecord) == sizeof(dsd_request_record), "record layout");

#define DSD_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            throw Error(DSD_ERR_RUNTIME, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                             " at " #call);                                    \
    } while (0)

constexpr int kBlock = 64;

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// Replica lists: the first launch covers replicas 0..n-1 (list == nullptr);
// the overflow re-run covers the `*count` replicas in `list`.
__device__ __forceinline__ bool replica_of(const Workspace& W, const int32_t* list, const int32_t* count,
                                          int64_t t, int64_t& rep) {
    if (list) {  // a replica list (overflow re-run, lane placement); -1 = an idle lane
        if (t >= *count) return false;
        rep = list[t];
        return rep >= 0;
    }
    rep = t;
    return t < W.c.n;
}

__global__ void __launch_bounds__(kBlock) k_stage(Workspace W, int64_t* ltot, const int32_t* list,
                                                  const int32_t* count) {
    int64_t rep;
    if (!replica_of(W, list, count, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x, rep)) return;
    stage_workload(W, rep);
    if (ltot) {
        const DevScenario& S = W.scen[W.rep_scen[rep]];
        int64_t N = S.workload == 0 ? S.n_requests : S.tr_n;
        const ReqRec* R = W.req + rep * W.c.nr;
        ltot[rep] = N == 0 ? 0 : static_cast<int64_t>(R[N - 1].seqoff) + R[N - 1].output;
    }
}

// One thread per replica; each iteration the warp runs ONE kind of step, for
// the lanes whose next step is of that kind: the kind most lanes have pending
// (__match_any_sync + __reduce_max_sync).  Replicas are independent, so
// reordering steps across lanes is free, while lanes that wait for the
// popular kind fall into phase with each other - the warp executes one handler
// body per iteration instead of the union of all of them.  (Measured on the
// C5 sweep: majority + chaining to the next pop/dispatch beat a cyclic sweep
// over kinds and un-chained stepping.)
//
// kSmem: the warp's server state and the first `heap_cap` event-heap slots
// live in shared memory (small topologies, <= kSmemServers servers); a replica
// whose heap would outgrow them fails with kFailHeap and is re-run on the HBM
// variant (k_collect_overflow + k_stage + k_simulate<false>).
//
// __launch_bounds__(64, 8): <= 128 registers, so 8 blocks (16 warps) fit per
// SM and a 65,536-replica sweep (13.8 warps/SM on 148 SMs) is one wave.
// Shared memory per warp of the kSmem variant: server fields, heap slots, the
// active-session record slots (one per possible draft server, ns - 1) and
// their first acceptance-bit words.
__host__ __device__ inline int64_t smem_warp_bytes(int64_t ns, int64_t heap_cap, bool awc) {
    return static_cast<int64_t>(kServerFields) * ns * kLanes * 4 + heap_cap * kLanes * 16 +
           (ns - 1) * kLanes * kHotStride + (awc ? static_cast<int64_t>(sizeof(AwcWarpScratch)) : 0);
}

// kBarrierKinds (the vote barriers) is defined in engine.cuh.

#ifndef DSD_VOTE_MODE
#define DSD_VOTE_MODE 0
#endif
// The warp runs the pending kind with the highest score: lane count, ties to
// the higher kind number.
__device__ __forceinline__ unsigned vote_score(unsigned count, uint32_t kind) {
#if DSD_VOTE_MODE == 1
    return (count << 4) | (15u - kind);  // ties to the lower kind (decoded by vote_kind)
#elif DSD_VOTE_MODE == 2
    return ((kind == kActDispatch ? 2u * count : count) << 4) | kind;
#elif DSD_VOTE_MODE == 3
    return ((kind == kActBegin ? 2u * count : count) << 4) | kind;
#elif DSD_VOTE_MODE == 4
    return ((kind == kActItem ? 2u * count : count) << 4) | kind;
#elif DSD_VOTE_MODE == 5
    return ((kind == kActDispatch ? count + (count >> 1) : count) << 4) | kind;
#else
    return (count << 4) | kind;
#endif
}

__device__ __forceinline__ uint32_t vote_kind(unsigned best) {
#if DSD_VOTE_MODE == 1
    return 15u - (best & 15u);
#else
    return best & 15u;
#endif
}

#ifndef DSD_MIN_BLOCKS
#define DSD_MIN_BLOCKS 8
#endif
// the specialised kernel needs ~100 registers: more resident blocks per SM
// leave room for thin warps (placement_list) in one wave
#ifndef DSD_SPEC_MIN_BLOCKS
#define DSD_SPEC_MIN_BLOCKS 8
#endif
// kSpec: the single-pair specialisation (Engine::spec; kSmem only).
// kAwc: the batch has AWC scenarios (cooperative AWC scratch + serving); the
// other instantiations compile that code out.
// kSpecLimit: overflow limit of the specialised action stack (1 only in the
// test instantiation that forces the HBM re-run, DSD_SPEC_STACK_LIMIT=1).
// kAwc kernels run with blocks of up to kAwcMaxThreads threads: one block
// per SM shares one shared-memory copy of the WC-DNN weights (staging).
constexpr int kAwcMaxThreads = 512;
// event-heap slots of the specialised kernel's overflow re-run (45.6 KB per
// block of two warps: few replicas, so occupancy does not matter there)
constexpr int kSpecRerunHeap = 32;
// the generic shared-memory kernel's (up to 4 servers and their session slots:
// <= 50 KB per block)
constexpr int kGenRerunHeap = 16;
template <bool kSmem, bool kStats, bool kSpec = false, bool kAwc = false, int kSpecLimit = kSpecStack>
__global__ void __launch_bounds__(kAwc ? kAwcMaxThreads : kBlock,
                                  kAwc ? 1 : (kSpec ? DSD_SPEC_MIN_BLOCKS : DSD_MIN_BLOCKS))
    k_simulate(const __grid_constant__ Workspace W, const int32_t* list, const int32_t* count, int32_t smem_heap_cap) {
    int64_t rep = 0;
    // solo mode: replica = block, run by lane 0 (the other lanes help copy)
    const bool solo = kSmem && !kSpec && W.solo;
    const bool live = solo ? (threadIdx.x == 0 && replica_of(W, list, count, blockIdx.x, rep))
                           : replica_of(W, list, count, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x, rep);
    const int64_t r = live ? rep : 0;
    int32_t lstride = kLanes;
    ReqRec* srec = nullptr;
    int32_t* sbase;
    int64_t* hb;
    uint64_t* kb;
    int64_t hcap;
    int32_t nsc;
    unsigned char* hot = nullptr;
    AwcWarpScratch* awc = nullptr;
    extern __shared__ __align__(16) unsigned char smem_all[];
    // AWC batches whose scenarios share one model: the block stages its
    // (transposed) weights into shared memory once; the per-warp regions follow
    const double* awc_w = nullptr;
    unsigned char* smem = smem_all;
    if constexpr (kAwc) {
        if (W.awc_stage_off >= 0) {
            double* sw = reinterpret_cast<double*>(smem_all);
            const double* gw = reinterpret_cast<const double*>(W.blob + W.awc_stage_off);
            for (int32_t k = threadIdx.x; k < W.awc_stage_n; k += blockDim.x) sw[k] = gw[k];
            __syncthreads();
            awc_w = sw;
            smem = smem_all + ((static_cast<int64_t>(W.awc_stage_n) * 8 + 127) & ~int64_t(127));
        }
    }
    if (solo) {
        // [AWC scratch][servers 8 x ns int32][heap times][heap keys][records]
        unsigned char* blk = smem;
        if constexpr (kAwc) {
            awc = reinterpret_cast<AwcWarpScratch*>(blk);
            blk += (sizeof(AwcWarpScratch) + 15) & ~size_t(15);
        }
        nsc = static_cast<int32_t>(W.c.ns);
        hcap = W.solo_hcap;
        lstride = 1;
        sbase = reinterpret_cast<int32_t*>(blk);
        blk += (static_cast<int64_t>(kServerFields) * nsc * 4 + 15) & ~int64_t(15);
        hb = reinterpret_cast<int64_t*>(blk);
        kb = reinterpret_cast<uint64_t*>(blk + hcap * 8);
        blk += hcap * 16;
        int64_t sr = 0;  // the block's replica (every lane copies its records)
        const bool has = replica_of(W, list, count, blockIdx.x, sr);
        if (W.solo_rec && has) {
            srec = reinterpret_cast<ReqRec*>(blk);
            const DevScenario& S0 = W.scen[W.rep_scen[sr]];
            const int64_t nreq = S0.workload == 0 ? S0.n_requests : S0.tr_n;
            const uint4* src = reinterpret_cast<const uint4*>(W.req + sr * W.c.nr);
            uint4* dst = reinterpret_cast<uint4*>(srec);
            for (int64_t k = threadIdx.x; k < nreq * static_cast<int64_t>(sizeof(ReqRec) / 16); k += blockDim.x)
                dst[k] = src[k];
        }
        __syncwarp();
    } else if constexpr (kSmem) {
        const int lane = threadIdx.x % kLanes;
        nsc = kSpec ? 2 : static_cast<int32_t>(W.c.ns);
        hcap = smem_heap_cap;
        const int64_t srv_bytes = static_cast<int64_t>(kServerFields) * nsc * kLanes * 4;
        constexpr bool with_awc = kAwc;
        unsigned char* blk = smem + (threadIdx.x / kLanes) * smem_warp_bytes(nsc, hcap, with_awc);
        sbase = reinterpret_cast<int32_t*>(blk) + lane;
        hb = reinterpret_cast<int64_t*>(blk + srv_bytes) + lane;
        kb = reinterpret_cast<uint64_t*>(blk + srv_bytes + hcap * kLanes * 8) + lane;
        hot = blk + srv_bytes + hcap * kLanes * 16 + lane * kHotStride;
        if (with_awc)
            awc = reinterpret_cast<AwcWarpScratch*>(blk + srv_bytes + hcap * kLanes * 16 + (nsc - 1) * kLanes * kHotStride);
    } else {
        const int64_t w = r / kLanes, lane = r % kLanes;
        nsc = static_cast<int32_t>(W.c.ns);
        hcap = W.c.hc;
        sbase = W.srv + w * kServerFields * W.c.ns * kLanes + lane;
        hb = W.h_time + w * W.c.hc * kLanes + lane;
        kb = W.h_key + w * W.c.hc * kLanes + lane;
        if constexpr (kAwc) awc = reinterpret_cast<AwcWarpScratch*>(smem) + threadIdx.x / kLanes;
    }
    if constexpr (kAwc) awc->req[threadIdx.x % kLanes] = 0;
    Engine e(W, W.scen[W.rep_scen[r]], r, sbase, hb, kb, hcap, nsc, hot, kSpec, awc, kSpecLimit, lstride, srec);
    e.smem_barriers = (kSmem || kAwc) && !kSpec;
    if (live) e.init();
    uint32_t kind = live ? e.next_kind() : static_cast<uint32_t>(kActNone);
    // kStats: per-step-kind cycle profile (DSD_STEP_STATS=1), one block-level
    // accumulation, flushed once per block
    __shared__ unsigned long long blk_stats[kStats ? 2 * kActKinds : 1];
    long long t_start = 0;
    unsigned long long iters = 0, my_rounds = 0;
    if constexpr (kStats) {
        for (int k = threadIdx.x; k < 2 * kActKinds; k += blockDim.x) blk_stats[k] = 0;
        __syncthreads();
        t_start = clock64();
    }
    for (;;) {
        // AWC decisions requested during the last chains: the whole warp
        // evaluates each requester's network (warp-uniform branch)
        if constexpr (kAwc) awc_serve_warp(W.blob, &e.S, awc, awc_w, W.awc_stage_off);
        // the kind most lanes have pending (majority vote); a solo replica
        // without AWC decisions runs alone (the idle lanes leave)
        uint32_t sel;
        if (solo && !kAwc) {
            if (kind == kActNone) break;
            sel = kind;
        } else {
            const unsigned peers = __match_any_sync(0xffffffffu, kind);
            const unsigned score = kind == kActNone ? 0u : vote_score(static_cast<unsigned>(__popc(peers)), kind);
            const unsigned best = __reduce_max_sync(0xffffffffu, score);
            if (best == 0u) break;
            sel = vote_kind(best);
        }
        if constexpr (kStats) {  // warp rounds per selected kind (lanes per round = steps / rounds)
            if ((threadIdx.x & (kLanes - 1)) == 0) atomicAdd(&W.step_stats[40 + sel], 1ull);
        }
        if (kind == sel) {
            if constexpr (kStats) ++my_rounds;
            // the selected lanes run their continuation chain up to the next
            // barrier kind (kBarrierKinds)
            do {
                if constexpr (kStats) {
                    const long long t0 = clock64();
                    e.step();
                    const long long t1 = clock64();
                    atomicAdd(&blk_stats[2 * kind], static_cast<unsigned long long>(t1 - t0));
                    atomicAdd(&blk_stats[2 * kind + 1], 1ull);
                } else {
                    e.step();
                }
                kind = e.next_kind_unchecked();
            } while (!(((kSpec ? kSpecBarrierKinds : (kSmem || kAwc) ? kSmemBarrierKinds : kBarrierKinds) >> kind) & 1u));
            // (a failed replica stops at its next pop: next_kind_unchecked)
        }
        if constexpr (kStats) ++iters;
    }
    if constexpr (kStats) {
        if ((threadIdx.x % kLanes) == 0) {
            atomicAdd(&W.step_stats[32], iters);
            atomicAdd(&W.step_stats[33], static_cast<unsigned long long>(clock64() - t_start));
            atomicMax(&W.step_stats[34], iters);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < 2 * kActKinds; k += blockDim.x) atomicAdd(&W.step_stats[k], blk_stats[k]);
    }
    if (live) e.finish();
    if (solo && srec && W.collect) {  // the records export reads them from HBM
        __syncwarp();
        int64_t sr = 0;
        if (replica_of(W, list, count, blockIdx.x, sr) && W.fail[sr] == kFailNone) {
            const DevScenario& S0 = W.scen[W.rep_scen[sr]];
            const int64_t nreq = S0.workload == 0 ? S0.n_requests : S0.tr_n;
            const uint4* src = reinterpret_cast<const uint4*>(srec);
            uint4* dst = reinterpret_cast<uint4*>(W.req + sr * W.c.nr);
            for (int64_t k = threadIdx.x; k < nreq * static_cast<int64_t>(sizeof(ReqRec) / 16); k += blockDim.x)
                dst[k] = src[k];
        }
    }
    if constexpr (kStats) {
        if (live && W.rep_stats) {
            W.rep_stats[3 * rep] = my_rounds;
            W.rep_stats[3 * rep + 2] = static_cast<unsigned long long>(clock64() - t_start);
        }
    }
}

// Session latency tables of the specialised kernel (Workspace::spec_lat):
// one block row per table (blockIdx.y), contexts across threads.  Entry c is
// {grid_latency_us(draft decode grid, 1, c, g), grid_latency_us(verify
// grid, g, c, 0)} - the very calls dispatch_single_draft / _target make - so
// a lookup is exact; a table with an entry >= kSpecLatMax is marked unusable
// in its status word (session_run then takes the step-by-step path).
__global__ void k_spec_lat(const char* blob, const SpecLatJob* jobs, int32_t* lat) {
    const SpecLatJob j = jobs[blockIdx.y];
    int32_t* t = lat + j.base;
    const DevGrid& gd = *reinterpret_cast<const DevGrid*>(blob + j.o_gd);
    const DevGrid& gt = *reinterpret_cast<const DevGrid*>(blob + j.o_gt);
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < j.n;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t a = grid_latency_us(blob, gd, 1, c, j.g1);
        const int64_t b = grid_latency_us(blob, gt, j.g1, c, 0);
        if (a >= kSpecLatMax || b >= kSpecLatMax) atomicOr(&t[0], 1);
        t[2 + 2 * c] = static_cast<int32_t>(a);
        t[3 + 2 * c] = static_cast<int32_t>(b);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) t[1] = j.n;
}

// Collects the replicas whose shared-memory heap (or the specialised
// kernel's shorter action stack) overflowed.
__global__ void k_collect_overflow(Workspace W, int32_t* list, int32_t* count) {
    const int64_t rep = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (rep >= W.c.n) return;
    if (W.fail[rep] == kFailHeap || W.fail[rep] == kFailStack) list[atomicAdd(count, 1)] = static_cast<int32_t>(rep);
}

// Collects the replicas that failed with one failure code.
__global__ void k_collect_fail(Workspace W, int32_t code, int32_t* list, int32_t* count) {
    const int64_t rep = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (rep >= W.c.n) return;
    if (W.fail[rep] == code) list[atomicAdd(count, 1)] = static_cast<int32_t>(rep);
}

__global__ void k_export(Workspace W, DevRecord* rec, int64_t* busy) {
    int64_t rep = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (rep >= W.c.n) return;
    const DevScenario& S = W.scen[W.rep_scen[rep]];
    Lane L{rep / kLanes, static_cast<int>(rep % kLanes)};
    const int64_t nr = W.c.nr;
    int64_t N = S.workload == 0 ? S.n_requests : S.tr_n;
    const ReqRec* R = W.req + rep * nr;
    for (int64_t i = 0; i < N; ++i) {
        DevRecord r;
        r.drafter_id = S.n_drafts > 0 ? R[i].drafter : -1;
        r.prompt_length = R[i].prompt;
        r.output_length = R[i].output;
        r.arrival_us = R[i].arrival;
        r.first_token_us = R[i].first;
        r.completion_us = R[i].done;
        r.proposed = R[i].prop;
        r.accepted = R[i].acc;
        r.target_id = R[i].target;
        r.n_iterations = R[i].ng;
        rec[rep * nr + i] = r;
    }
    for (int32_t t = 0; t < S.n_targets; ++t) busy[rep * W.c.nt + t] = L.at(W.v_busy_us, W.c.ns, t);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t n) {
        if (n <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (n == 0) return;
        DSD_CUDA(cudaMalloc(&p, n));
        bytes = n;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct RuntimeImpl {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {};
    DevBuf blob, scen, reps, arena, summary, fail, ltot, seqbase, seqg, seqc, rec, busy, ovf, probe, slat, sjobs;
    DevBuf heap2, ovf2;  // retry_heap_overflows: the larger event heap, its replica list
    bool elog_on = false;  // the batch records the event log + busy intervals
    // AWC batches with one shared model: warps per block of the kAwc kernels
    // (0: weights not staged, blocks of kBlock threads) for the
    // shared-memory and the HBM variant; staged weight bytes (128-aligned)
    int awc_warps_smem = 0, awc_warps_hbm = 0;
    size_t awc_wbytes = 0;
    int smem_optin = 0;
    DevBuf elog, busyiv, elogn;
    // shared-memory heap slots per replica for small topologies (0 = always
    // run the HBM variant; env DSD_SMEM_HEAP overrides, for tests)
    // 7: with 8 server fields x 2 servers and one session slot a warp needs
    // 9.75 KB, so 8 blocks/SM fit the 164 KB carveout (L1 keeps 92 KB)
    int32_t smem_heap = 7;
    bool step_stats = false;  // env DSD_STEP_STATS=1: per-step-kind cycle profile to stderr
    // every scenario of the prepared batch fits the single-pair kernel
    // specialisation (Engine::spec); env DSD_SPECIALIZE=0 disables its use
    bool spec_ok = false;
    bool specialize = true;
    // shared-memory carveout of the kSmem kernels (% of the SM's maximum):
    // -1 = sized per launch (DeviceRuntime::launch), env DSD_CARVEOUT fixes it
    int carveout = -1;
    // lane placement of the simulation kernel: [count][thread -> replica or
    // -1] (empty: replica = thread index)
    DevBuf place;
    int64_t place_n = 0;
    bool place_pending = false;  // prepare() -> the next launch() computes the placement
    int lanes_per_warp = 32;  // env DSD_LANES_PER_WARP: replicas per warp (experiments)
    bool placement = true;    // cost-aware lane placement (env DSD_PLACEMENT=0 disables)
    bool spread = true;       // sparse batches over the whole wave (env DSD_SPREAD=0 disables)
    double spread_max = 2.5;  // ... up to this many dense warps per SM (env DSD_SPREAD_MAX)
    int sms = 148, smem_per_sm = 228 * 1024;
    DevBuf stats;
    Workspace W{};
    Packed packed;  // the last batch, host side (storage reused across batches)
    std::vector<int64_t> host_seqbase;
    std::vector<int64_t> host_ltot;
    size_t n = 0;
    bool collect = false;
    bool prepared = false;
    bool ran = false;
    int64_t launches = 0;
    int64_t h2d_bytes = 0, d2h_bytes = 0;
    bool spec_stack_limit1 = false;  // DSD_SPEC_STACK_LIMIT=1 (tests: force the HBM re-run)
    bool session_fast = true;        // Engine::session_run in the specialised kernel (DSD_SESSION_FAST=0: off)
    bool awc_stage = true;           // stage one shared WC-DNN per block in shared memory (DSD_AWC_STAGE=0: off)
    int solo = 1;  // solo mode (DSD_SOLO): 0 off, 1 topologies past kSmemServers, 2 any topology
    int solo_heap = 0;     // DSD_SOLO_HEAP: cap on its heap slots (tests: force the HBM re-run)
    bool solo_rec = true;  // DSD_SOLO_REC=0: keep the records in HBM
    bool smem_launch = false;
    bool spec_rerun = false;  // the last launch re-ran overflows in its shared-memory kernel first
    int rerun_heap = 0;       // ... with this many heap slots
    void* pinned = nullptr;  // host_summaries() buffer (page-locked)
    bool pinned_valid = false;  // it holds the last launch's summaries
    bool retried = false;       // sync() ran retry_heap_overflows for the last launch
    size_t pinned_bytes = 0;  // the last launch ran the shared-memory variant (+ HBM re-run)
    // records cache (filled lazily after a collect run)
    bool rec_cached = false;
    std::vector<DevRecord> h_rec;
    std::vector<int64_t> h_busy;
    std::vector<int32_t> h_seqg, h_seqc;
};

// Block shape of the HBM variant's launches: the AWC scratch per warp (and
// the staged weights) or nothing.
struct HbmCfg {
    unsigned threads;
    size_t smem;
};
// Warps per staged-AWC block for a launch of `threads` threads: at most
// `cap`, but few enough that the blocks cover every SM (one block per SM
// fits next to the staged weights).
static int awc_block_warps(const RuntimeImpl& R, int cap, int64_t threads) {
    const int64_t warps = (threads + kLanes - 1) / kLanes;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap, (warps + R.sms - 1) / R.sms)));
}
static HbmCfg hbm_cfg(const RuntimeImpl& R, int64_t threads) {
    if (!R.W.c.awc) return {static_cast<unsigned>(kBlock), 0};
    if (R.awc_warps_hbm > 0) {
        const int w = awc_block_warps(R, R.awc_warps_hbm, threads);
        return {static_cast<unsigned>(w * kLanes), R.awc_wbytes + static_cast<size_t>(w) * sizeof(AwcWarpScratch)};
    }
    return {static_cast<unsigned>(kBlock), (kBlock / kLanes) * sizeof(AwcWarpScratch)};
}

DeviceRuntime::DeviceRuntime(int device) : impl_(new RuntimeImpl) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw Error(DSD_ERR_RUNTIME, "no CUDA device available: the DSD engine has no CPU fallback");
    if (device < 0 || device >= count) throw Error(DSD_ERR_RUNTIME, "device ordinal out of range");
    impl_->device = device;
    DSD_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    DSD_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        throw Error(DSD_ERR_RUNTIME, std::string("device ") + prop.name + " is not sm_100-class");
    DSD_CUDA(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking));
    if (const char* h = std::getenv("DSD_SMEM_HEAP")) impl_->smem_heap = std::max(0, std::atoi(h));
    if (const char* s = std::getenv("DSD_STEP_STATS")) impl_->step_stats = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_SPEC_STACK_LIMIT")) impl_->spec_stack_limit1 = std::atoi(s) == 1;
    if (const char* s = std::getenv("DSD_SPECIALIZE")) impl_->specialize = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_SESSION_FAST")) impl_->session_fast = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_AWC_STAGE")) impl_->awc_stage = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_SOLO")) impl_->solo = std::atoi(s);
    if (const char* s = std::getenv("DSD_SOLO_HEAP")) impl_->solo_heap = std::max(0, std::atoi(s));
    if (const char* s = std::getenv("DSD_SOLO_REC")) impl_->solo_rec = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_PLACEMENT")) impl_->placement = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_SPREAD")) impl_->spread = std::atoi(s) != 0;
    if (const char* s = std::getenv("DSD_SPREAD_MAX")) impl_->spread_max = std::atof(s);
    if (const char* s = std::getenv("DSD_LANES_PER_WARP"))
        impl_->lanes_per_warp = std::max(1, std::min(kLanes, std::atoi(s)));
    if (const char* s = std::getenv("DSD_CARVEOUT")) {  // shared-memory share of the L1/smem array (%)
        impl_->carveout = std::atoi(s);
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<false, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      impl_->carveout));
    }
    DSD_CUDA(cudaDeviceGetAttribute(&impl_->sms, cudaDevAttrMultiProcessorCount, device));
    DSD_CUDA(cudaDeviceGetAttribute(&impl_->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
    DSD_CUDA(cudaDeviceGetAttribute(&impl_->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    for (auto& ev : impl_->ev) DSD_CUDA(cudaEventCreate(&ev));
}

DeviceRuntime::~DeviceRuntime() {
    if (!impl_) return;
    cudaSetDevice(impl_->device);
    if (impl_->stream) cudaStreamSynchronize(impl_->stream);
    if (impl_->pinned) cudaFreeHost(impl_->pinned);
    for (auto& ev : impl_->ev)
        if (ev) cudaEventDestroy(ev);
    if (impl_->stream) cudaStreamDestroy(impl_->stream);
}

void* DeviceRuntime::stream() { return impl_->stream; }
int DeviceRuntime::device() const { return impl_->device; }
int64_t DeviceRuntime::last_launch_count() const { return impl_->launches; }
size_t DeviceRuntime::replica_count() const { return impl_->n; }
void DeviceRuntime::transfer_bytes(int64_t* h2d, int64_t* d2h) const {
    if (h2d) *h2d = impl_->h2d_bytes;
    if (d2h) *d2h = impl_->d2h_bytes;
}

// Cost-aware lane placement.  A warp advances at the pace of
// its slowest lane, and the more lanes it carries the more vote rounds each
// of them waits through: measured on the heaviest C5 replica (gamma 1, alpha
// 0.5) alone, a warp of 1 / 2 / 4 / 8 / 16 lanes takes 1 / 1.68 / 2.54 /
// 3.54 / 4.57 x the time of a lone lane (kWarpSlow).  Replicas are sorted by
// an estimate of their cost - N x (150 + median output / E[tokens per round])
// in the specialised kernel (9 in the generic one, where every iteration's
// events are general steps too) for a synthetic workload with a static
// window, E = (1 - a^(g+1)) / (1 - a):
// a request's general event handling (~60 steps, ~13 us on a lone lane)
// against one session iteration (~66 ns) per round, fitted to lone-lane
// kernel times of C5's (gamma, alpha) corners (the earlier
// weight 9 ranked gamma-15 replicas as light and packed them 32 wide, a
// 9 ms warp in 1/8 of C5) - and each gets the widest warp that keeps
// cost x kWarpSlow[width] within a makespan T, the smallest T whose warps
// all fit one wave (`warp_cap`, binary search).  So a batch that leaves room
// (a strong-scaling shard, a small sweep) runs its heavy replicas one per
// warp, and a full one packs the light replicas 32 to a warp.  Sorting also
// makes warps homogeneous.  Returns [count][thread -> replica or -1], or
// nothing when the batch has no estimate or needs more than one wave.
// Placement only chooses which thread runs which replica: results are
// unchanged.
static std::vector<int32_t> placement_list(const Packed& P, size_t n, int64_t warp_cap, bool spec) {
    if (n < 2) return {};
    // a batch that nearly fills the wave densely is issue-bound, not
    // critical-path-bound: thin warps would only cost SIMT efficiency
    // (C5, 65,536 replicas on 2,368 warps: dense 13.2 ms, placed 13.7 ms)
    static const double max_fill = std::getenv("DSD_PLACE_MAX_FILL") ? std::atof(std::getenv("DSD_PLACE_MAX_FILL")) : 0.75;
    if (static_cast<double>(n) > max_fill * static_cast<double>(warp_cap * kLanes)) return {};
    std::vector<double> est(P.scen.size(), 0.0);
    // the specialised kernel runs a request's iterations in its session loop,
    // so the request's general steps weigh 150 iterations; the generic kernel
    // handles every iteration's events as general steps too: 9 (C2's
    // 16,384-replica sweep: 514 ms at 9, 572 ms at 150)
    static const char* env_cost = std::getenv("DSD_COST_REQ");
    const double cost_req = env_cost ? std::atof(env_cost) : (spec ? 150.0 : 9.0);
    for (size_t k = 0; k < P.scen.size(); ++k) {
        const DevScenario& d = P.scen[k];
        if (d.workload != 0 || d.n_drafts < 1 || d.fused_everything || d.window_kind != 0) return {};
        const double a = d.alpha, g = d.gamma;
        const double tau = a < 1.0 ? (1.0 - std::pow(a, g + 1.0)) / (1.0 - a) : g + 1.0;
        est[k] = static_cast<double>(d.n_requests) * (cost_req + std::exp(d.o_mu) / tau);
    }
    // replicas by decreasing estimate: sort the scenarios, then a counting
    // sort of the replicas by their scenario's rank (replica order within one)
    const size_t ns = P.scen.size();
    std::vector<int32_t> sorder(ns), srank(ns), start(ns + 1, 0);
    std::iota(sorder.begin(), sorder.end(), 0);
    std::stable_sort(sorder.begin(), sorder.end(), [&](int32_t x, int32_t y) { return est[x] > est[y]; });
    for (size_t i = 0; i < ns; ++i) srank[static_cast<size_t>(sorder[i])] = static_cast<int32_t>(i);
    for (size_t r = 0; r < n; ++r) ++start[static_cast<size_t>(srank[P.rep_scen[r]]) + 1];
    for (size_t i = 0; i < ns; ++i) start[i + 1] += start[i];
    // (cost, replica count) per scenario with replicas, in cost order: the
    // makespan search below runs over these groups, not the replicas
    std::vector<double> gcost;
    std::vector<int64_t> gcnt;
    for (size_t i = 0; i < ns; ++i)
        if (start[i + 1] > start[i]) {
            gcost.push_back(est[static_cast<size_t>(sorder[i])]);
            gcnt.push_back(start[i + 1] - start[i]);
        }
    std::vector<int32_t> order(n);
    for (size_t r = 0; r < n; ++r) order[static_cast<size_t>(start[static_cast<size_t>(srank[P.rep_scen[r]])]++)] = static_cast<int32_t>(r);
    std::vector<double> cost(n);
    for (size_t i = 0; i < n; ++i) cost[i] = est[P.rep_scen[static_cast<size_t>(order[i])]];
    static const int kWidth[6] = {1, 2, 4, 8, 16, 32};
    static const double kWarpSlow[6] = {1.0, 1.68, 2.54, 3.54, 4.57, 5.6};
    // width of replica i under makespan T (-1: does not fit even alone)
    auto width = [&](double c, double T) {
        int w = -1;
        for (int k = 0; k < 6; ++k)
            if (c * kWarpSlow[k] <= T) w = k;
        return w;
    };
    // warps needed: consecutive replicas (costs descending, widths
    // ascending) of one width share warps
    auto warps = [&](double T) {
        int64_t total = 0, run = 0;
        int cur = -2;
        for (size_t g = 0; g < gcost.size(); ++g) {
            const int w = width(gcost[g], T);
            if (w < 0) return INT64_MAX;
            if (w != cur) {
                if (cur >= 0) total += (run + kWidth[cur] - 1) / kWidth[cur];
                cur = w;
                run = 0;
            }
            run += gcnt[g];
        }
        return total + (run + kWidth[cur] - 1) / kWidth[cur];
    };
    double lo = cost[0], hi = cost[0] * kWarpSlow[5];
    if (warps(hi) > warp_cap) return {};
    for (int it = 0; it < 40; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (warps(mid) <= warp_cap) hi = mid; else lo = mid;
    }
    const double T = hi;
    if (width(cost[n - 1], T) == 5 && width(cost[0], T) == 5) return {};  // every warp full: the dense layout
    std::vector<int32_t> pl(1, 0);
    for (size_t i = 0; i < n;) {
        const int w = width(cost[i], T);
        size_t j = i;
        while (j < n && width(cost[j], T) == w) ++j;
        for (size_t k = i; k < j;) {
            for (int l = 0; l < kLanes; ++l) pl.push_back(l < kWidth[w] && k < j ? order[k++] : -1);
        }
        i = j;
    }
    pl[0] = static_cast<int32_t>(pl.size() - 1);
    return pl;
}

// Session latency tables for a specialised batch: one per distinct (draft
// decode grid, verify grid, gamma), covering every context a request of the
// scenarios can reach (prompt + output: the length caps of a synthetic
// workload, the longest trace record otherwise); sets each scenario's o_slat
// (-1: no table, the session loop stays off).  Returns the int32 elements.
static int64_t spec_lat_jobs(Packed& P, std::vector<SpecLatJob>& jobs) {
    std::map<std::tuple<int64_t, int64_t, int32_t>, size_t> key_job;
    std::vector<size_t> job_of(P.scen.size(), SIZE_MAX);
    for (size_t k = 0; k < P.scen.size(); ++k) {
        DevScenario& d = P.scen[k];
        d.o_slat = -1;
        int64_t maxctx = 0;
        if (d.workload == 0) {
            maxctx = d.p_cap + d.o_cap;
        } else {
            const int64_t* tp = reinterpret_cast<const int64_t*>(P.blob.data() + d.o_tr_prompt);
            const int64_t* to = reinterpret_cast<const int64_t*>(P.blob.data() + d.o_tr_output);
            for (int64_t q = 0; q < d.tr_n; ++q) maxctx = std::max(maxctx, tp[q] + to[q]);
        }
        if (maxctx < 0 || maxctx >= (1 << 20) || d.gamma > 63) continue;  // no table
        const int32_t* tg = reinterpret_cast<const int32_t*>(P.blob.data() + d.o_tgrid);
        const int32_t* dg = reinterpret_cast<const int32_t*>(P.blob.data() + d.o_dgrid);
        const int64_t o_gt = d.o_grids + static_cast<int64_t>(sizeof(DevGrid)) * tg[1];
        const int64_t o_gd = d.o_grids + static_cast<int64_t>(sizeof(DevGrid)) * dg[1];
        const int32_t g1 = std::max(1, d.gamma);
        auto it = key_job.emplace(std::make_tuple(o_gd, o_gt, g1), jobs.size()).first;
        if (it->second == jobs.size()) jobs.push_back(SpecLatJob{o_gd, o_gt, 0, g1, 0});
        SpecLatJob& j = jobs[it->second];
        j.n = std::max<int32_t>(j.n, static_cast<int32_t>(maxctx + 1));
        job_of[k] = it->second;
    }
    int64_t off = 0;
    for (SpecLatJob& j : jobs) {
        j.base = off;
        off += 2 + 2 * static_cast<int64_t>(j.n);
    }
    for (size_t k = 0; k < P.scen.size(); ++k)
        if (job_of[k] != SIZE_MAX) P.scen[k].o_slat = jobs[job_of[k]].base;
    return off;
}

void DeviceRuntime::prepare(const dsd_scenario* sc, size_t ns, const dsd_replica* reps, size_t n,
                      bool collect, bool feature_probe, bool event_log) {
    RuntimeImpl& R = *impl_;
    DSD_CUDA(cudaSetDevice(R.device));
    R.prepared = false;
    R.ran = false;
    R.rec_cached = false;
    R.pinned_valid = false;
    // DSD_HOST_TIMING=1: phase durations to stderr
    static const bool timing = std::getenv("DSD_HOST_TIMING") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!timing) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[dsd prepare] %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_prev).count());
        t_prev = t;
    };
    Packed& P = R.packed;
    pack_batch_into(P, sc, ns, reps, n, feature_probe);
    lap("pack");
    // tests: a smaller HBM event heap (forces retry_heap_overflows)
    if (const char* h = std::getenv("DSD_HEAP_CAP")) P.caps.hc = std::max<int64_t>(1, std::atoll(h));
    const Caps& c = P.caps;
    // every scenario fits the single-pair specialisation (Engine::spec)
    R.spec_ok = c.ns == 2;
    for (const DevScenario& d : P.scen)
        R.spec_ok = R.spec_ok && d.n_targets == 1 && d.n_drafts == 1 && !d.fused_everything && d.window_kind == 0 &&
                    d.batching == 0 && d.batching_window_us == 0 && d.jitter_free && d.n_dg == 1 && d.n_tg == 1 &&
                    !d.has_order && !d.pair_stats;
    std::vector<SpecLatJob> jobs;
    int64_t slat_elems = 0;
    if (R.spec_ok && R.session_fast) slat_elems = spec_lat_jobs(P, jobs);
    // ---- upload blob, scenarios, replicas ----
    R.blob.ensure(P.blob.size());
    DSD_CUDA(cudaMemcpyAsync(R.blob.p, P.blob.data(), P.blob.size(), cudaMemcpyHostToDevice, R.stream));
    R.scen.ensure(sizeof(DevScenario) * std::max<size_t>(ns, 1));
    if (ns) DSD_CUDA(cudaMemcpyAsync(R.scen.p, P.scen.data(), sizeof(DevScenario) * ns, cudaMemcpyHostToDevice, R.stream));
    const size_t rep_bytes = n * (sizeof(uint32_t) + 2 * sizeof(uint64_t)) + 64;
    R.reps.ensure(rep_bytes);
    char* rp = static_cast<char*>(R.reps.p);
    uint64_t* d_seed = reinterpret_cast<uint64_t*>(rp);
    uint64_t* d_gseed = d_seed + n;
    uint32_t* d_rs = reinterpret_cast<uint32_t*>(d_gseed + n);
    if (n) {
        DSD_CUDA(cudaMemcpyAsync(d_seed, P.seed.data(), 8 * n, cudaMemcpyHostToDevice, R.stream));
        DSD_CUDA(cudaMemcpyAsync(d_gseed, P.gseed.data(), 8 * n, cudaMemcpyHostToDevice, R.stream));
        DSD_CUDA(cudaMemcpyAsync(d_rs, P.rep_scen.data(), 4 * n, cudaMemcpyHostToDevice, R.stream));
    }
    R.h2d_bytes = static_cast<int64_t>(P.blob.size() + sizeof(DevScenario) * ns + 20 * n);
    R.d2h_bytes = 0;
    R.summary.ensure(sizeof(DevSummary) * std::max<size_t>(n, 1));
    R.fail.ensure(sizeof(int32_t) * std::max<size_t>(n, 1));

    // ---- workspace arena ----
    Workspace& W = R.W;
    W = Workspace{};
    lap("upload");
    const size_t total = layout_workspace(W, c, nullptr);
    if (total > R.arena.bytes) {  // growing: check the device has room (cudaMemGetInfo is not free)
        size_t free_b = 0, total_b = 0;
        DSD_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (total + (256u << 20) > free_b + R.arena.bytes)
            throw Error(DSD_ERR_RUNTIME, "replica workspace (" + std::to_string(total >> 20) +
                                             " MiB) exceeds free device memory");
    }
    R.arena.ensure(total);
    layout_workspace(W, c, static_cast<char*>(R.arena.p));
    W.blob = static_cast<const char*>(R.blob.p);
    W.scen = static_cast<const DevScenario*>(R.scen.p);
    W.rep_scen = d_rs;
    W.rep_seed = d_seed;
    W.rep_gen_seed = d_gseed;
    W.summary = static_cast<DevSummary*>(R.summary.p);
    W.fail = static_cast<int32_t*>(R.fail.p);
    W.collect = collect ? 1 : 0;
    W.session_fast = R.session_fast ? 1 : 0;
    // AWC: stage the WC-DNN into shared memory when every AWC scenario of the
    // batch uses one model and it fits next to at least one warp's state
    W.awc_stage_off = -1;
    W.awc_stage_n = 0;
    R.awc_warps_smem = R.awc_warps_hbm = 0;
    R.awc_wbytes = 0;
    if (c.awc && R.awc_stage) {
        int64_t off = -1, cnt = 0;
        bool one = true;
        for (const DevScenario& d : P.scen) {
            if (d.window_kind != 2 || d.fused_everything) continue;
            const int64_t k = static_cast<int64_t>(d.awc_hidden) * d.awc_input + d.awc_hidden +
                              static_cast<int64_t>(d.awc_blocks) * (2 * d.awc_hidden * d.awc_hidden + 2 * d.awc_hidden) +
                              d.awc_hidden + 1;
            if (off < 0) {
                off = d.o_awc_params;
                cnt = k;
            } else if (d.o_awc_params != off) {
                one = false;
            }
        }
        const size_t wb = (static_cast<size_t>(cnt) * 8 + 127) & ~size_t(127);
        // (the kernels' static shared memory - the step-stats counters - comes off the opt-in limit)
        const int64_t room = static_cast<int64_t>(R.smem_optin) - 1024 - static_cast<int64_t>(wb);
        if (one && off >= 0 && room > 0) {
            const int64_t sw = static_cast<int64_t>(smem_warp_bytes(c.ns <= kSmemServers ? c.ns : 2, R.smem_heap, true));
            R.awc_warps_hbm = static_cast<int>(std::min<int64_t>(16, room / static_cast<int64_t>(sizeof(AwcWarpScratch))));
            R.awc_warps_smem = c.ns <= kSmemServers && R.smem_heap > 0 ? static_cast<int>(std::min<int64_t>(16, room / sw)) : 0;
            if (R.awc_warps_hbm > 0 && (R.awc_warps_smem > 0 || !(c.ns <= kSmemServers && R.smem_heap > 0))) {
                W.awc_stage_off = off;
                W.awc_stage_n = static_cast<int32_t>(cnt);
                R.awc_wbytes = wb;
            } else {
                R.awc_warps_hbm = R.awc_warps_smem = 0;
            }
        }
    }
    if (feature_probe) {
        R.probe.ensure(sizeof(double) * kProbeFields * std::max<size_t>(n, 1));
        W.probe = static_cast<double*>(R.probe.p);
    }
    // session latency tables (specialised batches)
    W.spec_lat = nullptr;
    if (slat_elems > 0) {
        R.slat.ensure(sizeof(int32_t) * static_cast<size_t>(slat_elems));
        R.sjobs.ensure(sizeof(SpecLatJob) * jobs.size());
        DSD_CUDA(cudaMemsetAsync(R.slat.p, 0, sizeof(int32_t) * static_cast<size_t>(slat_elems), R.stream));
        DSD_CUDA(cudaMemcpyAsync(R.sjobs.p, jobs.data(), sizeof(SpecLatJob) * jobs.size(), cudaMemcpyHostToDevice,
                                 R.stream));
        int32_t nmax = 0;
        for (const SpecLatJob& j : jobs) nmax = std::max(nmax, j.n);
        const dim3 g(static_cast<unsigned>(std::min<int64_t>(64, (nmax + 255) / 256)), static_cast<unsigned>(jobs.size()));
        k_spec_lat<<<g, 256, 0, R.stream>>>(W.blob, static_cast<const SpecLatJob*>(R.sjobs.p),
                                            static_cast<int32_t*>(R.slat.p));
        DSD_CUDA(cudaGetLastError());
        W.spec_lat = static_cast<const int32_t*>(R.slat.p);
        R.h2d_bytes += static_cast<int64_t>(sizeof(SpecLatJob) * jobs.size());
    }
    // lane placement
    R.place_n = 0;
    // the lane placement is computed by launch() while k_stage runs
    R.place_pending = true;
    R.n = n;
    R.elog_on = event_log;
    collect = collect || event_log;  // the log's sizing uses the records' output totals
    R.collect = collect;
    if (collect) R.ltot.ensure(sizeof(int64_t) * std::max<size_t>(n, 1));
    lap("workspace");
    DSD_CUDA(cudaStreamSynchronize(R.stream));
    lap("sync");
    R.prepared = true;
}

// Lane placement of the prepared batch (placement_list, or the uniform
// DSD_LANES_PER_WARP layout), uploaded on the stream: launch() computes it on
// the host while k_stage runs, once per prepared batch.
static void place_lanes(RuntimeImpl& R) {
    R.place_pending = false;
    R.place_n = 0;
    const size_t n = R.n;
    const bool spec_launch = R.spec_ok && R.specialize && !R.collect && !R.W.probe;
    const int64_t max_blocks = spec_launch ? DSD_SPEC_MIN_BLOCKS : DSD_MIN_BLOCKS;
    // blocks one wave puts on an SM: the launch bounds, and for the
    // shared-memory variant its per-block shared memory
    int64_t per_sm = max_blocks;
    if (R.W.c.ns <= kSmemServers && R.smem_heap > 0) {
        const int64_t bytes = (kBlock / kLanes) * smem_warp_bytes(spec_launch ? 2 : R.W.c.ns, R.smem_heap,
                                                                  R.W.c.awc != 0);
        per_sm = std::max<int64_t>(1, std::min<int64_t>(max_blocks, R.smem_per_sm / (bytes + 1024)));
    }
    int64_t warp_cap = R.sms * per_sm * (kBlock / kLanes);
    if (R.W.c.awc && (R.W.c.ns <= kSmemServers && R.smem_heap > 0 ? R.awc_warps_smem : R.awc_warps_hbm) > 0)
        warp_cap = R.sms * (R.W.c.ns <= kSmemServers && R.smem_heap > 0 ? R.awc_warps_smem : R.awc_warps_hbm);
    std::vector<int32_t> pl = placement_list(R.packed, n, warp_cap, spec_launch);
    if (!pl.empty() && R.placement && R.lanes_per_warp == kLanes) {
        R.place.ensure(4 * pl.size());
        DSD_CUDA(cudaMemcpyAsync(R.place.p, pl.data(), 4 * pl.size(), cudaMemcpyHostToDevice, R.stream));
        R.place_n = static_cast<int64_t>(pl.size()) - 1;
    }
    // A batch that leaves the SMs underfilled when dense (at most 2.5 full
    // warps per SM) and that the cost-aware placement does not place (any
    // workload but synthetic static windows; e.g. the AWC dataset's 2,400
    // replicas = 75 warps on 148 SMs): spread it over the wave, ceil(n / warp
    // capacity) replicas per warp - every SM gets work and fewer lanes share a
    // warp's vote rounds.  Measured: dataset 118 -> 58 ms, a 768-replica AWC
    // sweep 1.97 -> 0.32 s, dynamic-window sweeps of 2,048 / 4,096 / 8,192 /
    // 12,288 replicas -24 / -20 / -9 / -2%, but 24,576 replicas +12%.
    int64_t lpw = R.lanes_per_warp;
    if (R.place_n == 0 && R.placement && lpw == kLanes && n > 0 && R.spread &&
        static_cast<double>(n) <= R.spread_max * R.sms * kLanes)
        lpw = std::max<int64_t>(1, (static_cast<int64_t>(n) + warp_cap - 1) / warp_cap);
    if (lpw < kLanes && n > 0) {
        const int64_t nw = (static_cast<int64_t>(n) + lpw - 1) / lpw;
        std::vector<int32_t> ul(static_cast<size_t>(nw * kLanes + 1), -1);
        ul[0] = static_cast<int32_t>(nw * kLanes);
        for (int64_t w = 0; w < nw; ++w)
            for (int64_t l = 0; l < lpw; ++l)
                if (w * lpw + l < static_cast<int64_t>(n)) ul[1 + w * kLanes + l] = static_cast<int32_t>(w * lpw + l);
        R.place.ensure(4 * ul.size());
        DSD_CUDA(cudaMemcpyAsync(R.place.p, ul.data(), 4 * ul.size(), cudaMemcpyHostToDevice, R.stream));
        R.place_n = nw * kLanes;
    }
}

// Solo mode: a batch of at most one wave of replicas whose server state
// does not fit the shared-memory variant's per-lane layout (more than
// kSmemServers servers: C2-C4) runs one replica per block of one warp, its
// servers and an event heap in shared memory at lane stride 1 and, when
// they fit next to the heap, the batch's staged WC-DNN weights (AWC) and all
// its request records.  The per-warp HBM layout would leave every dependent state access
// an L2 round trip for a lone replica.  A heap overflow hands the replica to
// the HBM re-run like the shared-memory variant's.
struct SoloCfg {
    bool on = false;
    int32_t hcap = 0;
    bool rec = false;
    bool stage = false;  // the block stages the batch's one WC-DNN (AWC)
    size_t bytes = 0;
};
static SoloCfg solo_cfg(const RuntimeImpl& R) {
    SoloCfg s;
    const Caps& c = R.W.c;
    if (R.solo == 0 || R.n == 0 || (R.solo == 1 && c.ns <= kSmemServers)) return s;
    const int64_t per_sm = (static_cast<int64_t>(R.n) + R.sms - 1) / R.sms;
    if (per_sm > 32) return s;  // one wave of one-warp blocks
    const int64_t budget =
        std::min<int64_t>(R.smem_optin, R.smem_per_sm / per_sm) - 1024;  // (static shared memory: the step stats)
    int64_t fixed = (c.awc ? ((static_cast<int64_t>(sizeof(AwcWarpScratch)) + 15) & ~int64_t(15)) : 0) +
                    ((static_cast<int64_t>(kServerFields) * c.ns * 4 + 15) & ~int64_t(15));
    // heap: 1,024 slots or 1 per server (C4-static/-AWC single runs peak below
    // 1,024; an overflow costs an HBM re-run, not a wrong result; a larger
    // heap takes L1 from the records: C4-AWC 7.10 s at 1,024 slots, 7.45 s
    // at 2,080)
    const int64_t hmin = std::min<int64_t>(R.solo_heap > 0 ? R.solo_heap : c.hc, std::max<int64_t>(1024, c.ns));
    if (fixed + 16 * hmin > budget) return s;
    // AWC: the staged weights when they fit too (every decision reads all of them)
    if (R.W.awc_stage_off >= 0 && fixed + static_cast<int64_t>(R.awc_wbytes) + 16 * hmin <= budget) {
        s.stage = true;
        fixed += static_cast<int64_t>(R.awc_wbytes);
    } else if (R.W.awc_stage_off >= 0) {
        // the HBM variant stages the weights once per block for several warps:
        // better than solo blocks that cannot (256 C3 replicas: 683 vs 740 ms)
        return s;
    }
    const int64_t recb = c.nr * static_cast<int64_t>(sizeof(ReqRec));
    s.rec = R.solo_rec && fixed + recb + 16 * hmin <= budget;
    // (records left in HBM: the heap stays at hmin, the rest of the array is L1 for them)
    s.hcap = static_cast<int32_t>(s.rec ? std::min<int64_t>(c.hc, (budget - fixed - recb) / 16) : hmin);
    if (R.solo_heap > 0) s.hcap = std::min(s.hcap, R.solo_heap);
    s.bytes = static_cast<size_t>(fixed + 16 * s.hcap + (s.rec ? recb : 0));
    s.on = true;
    return s;
}

void DeviceRuntime::launch() {
    RuntimeImpl& R = *impl_;
    if (!R.prepared) throw Error(DSD_ERR_RUNTIME, "launch without a prepared batch");
    DSD_CUDA(cudaSetDevice(R.device));
    static const bool timing = std::getenv("DSD_HOST_TIMING") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!timing) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[dsd launch] %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_prev).count());
        t_prev = t;
    };
    R.launches = 0;
    R.rec_cached = false;
    R.pinned_valid = false;
    R.retried = false;
    if (R.n == 0) {
        R.ran = true;
        return;
    }
    const unsigned grid = static_cast<unsigned>((R.n + kBlock - 1) / kBlock);
    if (R.W.c.awc) {
        for (auto k : {k_simulate<false, false, false, true>, k_simulate<false, true, false, true>,
                       k_simulate<true, false, false, true>, k_simulate<true, true, false, true>}) {
            cudaFuncAttributes fa;
            DSD_CUDA(cudaFuncGetAttributes(&fa, k));
            DSD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          R.smem_optin - static_cast<int>(fa.sharedSizeBytes)));
        }
    }
    DSD_CUDA(cudaEventRecord(R.ev[0], R.stream));
    k_stage<<<grid, kBlock, 0, R.stream>>>(R.W, R.collect ? static_cast<int64_t*>(R.ltot.p) : nullptr, nullptr,
                                           nullptr);
    DSD_CUDA(cudaGetLastError());
    ++R.launches;
    lap("stage");
    if (R.place_pending) place_lanes(R);
    lap("placement");
    // the HBM variant's only shared memory: the cooperative AWC scratch (and
    // the staged AWC weights); its carveout keeps just that (the rest of the
    // array is L1, which holds the replicas' state)
    // (the block shape of the HBM variant's main launch: the placement's thread count)
    const HbmCfg hcfg = hbm_cfg(R, R.place_n ? R.place_n : static_cast<int64_t>(R.n));
    const size_t hbm_smem = hcfg.smem;
    auto hgrid_of = [&](int64_t threads) { return static_cast<unsigned>((threads + hcfg.threads - 1) / hcfg.threads); };
    // sized for the blocks a launch of `g` blocks puts on an SM
    auto hbm_carveout = [&](unsigned g) {
        if (R.carveout >= 0) return;
        const int64_t per_sm = R.awc_warps_hbm > 0 ? 1 : std::min<int64_t>(DSD_MIN_BLOCKS, (g + R.sms - 1) / R.sms);
        const int64_t need = hbm_smem ? per_sm * (static_cast<int64_t>(hbm_smem) + 1024) : 0;
        const int pct = static_cast<int>(std::min<int64_t>(100, (100 * need + R.smem_per_sm - 1) / R.smem_per_sm));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<false, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<false, false, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    };
    hbm_carveout(hgrid_of(R.place_n ? R.place_n : static_cast<int64_t>(R.n)));
    if (R.collect) {
        // size the sequence arena exactly: prefix sum of per-replica output totals
        R.host_ltot.resize(R.n);
        DSD_CUDA(cudaMemcpyAsync(R.host_ltot.data(), R.ltot.p, 8 * R.n, cudaMemcpyDeviceToHost, R.stream));
        DSD_CUDA(cudaStreamSynchronize(R.stream));
        R.host_seqbase.resize(R.n);
        int64_t acc = 0;
        for (size_t i = 0; i < R.n; ++i) {
            R.host_seqbase[i] = acc;
            acc += R.host_ltot[i];
        }
        R.seqbase.ensure(8 * R.n);
        R.seqg.ensure(4 * std::max<int64_t>(acc, 1));
        R.seqc.ensure(4 * std::max<int64_t>(acc, 1));
        DSD_CUDA(cudaMemcpyAsync(R.seqbase.p, R.host_seqbase.data(), 8 * R.n, cudaMemcpyHostToDevice, R.stream));
        R.W.rep_seqbase = static_cast<int64_t*>(R.seqbase.p);
        R.W.seq_cap = acc;
        R.W.seq_gamma = static_cast<int32_t*>(R.seqg.p);
        R.W.seq_commit = static_cast<int32_t*>(R.seqc.p);
        R.W.elog = nullptr;
        R.W.busy_iv = nullptr;
        if (R.elog_on) {
            // every iteration commits >= 1 token, so a request logs at most
            // 4 x output + 2 transitions and dispatches at most 2 x output + 2
            // batch items
            int64_t lmax = 0;
            for (size_t i = 0; i < R.n; ++i) lmax = std::max(lmax, R.host_ltot[i]);
            const int64_t ecap = 4 * lmax + 2 * R.W.c.nr + 16, bcap = 2 * lmax + 2 * R.W.c.nr + 16;
            const size_t bytes = (sizeof(ElogRec) * ecap + sizeof(BusyRec) * bcap) * R.n;
            size_t free_b = 0, total_b = 0;
            DSD_CUDA(cudaMemGetInfo(&free_b, &total_b));
            if (bytes + (256u << 20) > free_b + R.elog.bytes + R.busyiv.bytes)
                throw Error(DSD_ERR_RUNTIME, "event log of the batch (" + std::to_string(bytes >> 20) +
                                                 " MiB) exceeds free device memory");
            R.elog.ensure(sizeof(ElogRec) * ecap * R.n);
            R.busyiv.ensure(sizeof(BusyRec) * bcap * R.n);
            R.elogn.ensure(2 * sizeof(int64_t) * R.n);
            R.W.elog = static_cast<ElogRec*>(R.elog.p);
            R.W.busy_iv = static_cast<BusyRec*>(R.busyiv.p);
            R.W.elog_cap = ecap;
            R.W.busy_cap = bcap;
            R.W.elog_n = static_cast<int64_t*>(R.elogn.p);
            R.W.busy_n = R.W.elog_n + R.n;
        }
    }
    if (R.step_stats) {
        R.stats.ensure((64 + 3 * R.n) * sizeof(unsigned long long));
        DSD_CUDA(cudaMemsetAsync(R.stats.p, 0, (64 + 3 * R.n) * sizeof(unsigned long long), R.stream));
        R.W.step_stats = static_cast<unsigned long long*>(R.stats.p);
        R.W.rep_stats = R.W.step_stats + 64;
    }
    lap("arena");
    DSD_CUDA(cudaEventRecord(R.ev[1], R.stream));
    const SoloCfg solo = solo_cfg(R);
    const bool smem = solo.on || (R.W.c.ns <= kSmemServers && R.smem_heap > 0);
    R.smem_launch = smem;
    if (solo.on) {
        Workspace Ws = R.W;
        Ws.solo = 1;
        Ws.solo_hcap = solo.hcap;
        Ws.solo_rec = solo.rec ? 1 : 0;
        if (!solo.stage) Ws.awc_stage_off = -1;
        auto k = R.W.c.awc ? (R.step_stats ? k_simulate<true, true, false, true> : k_simulate<true, false, false, true>)
                           : (R.step_stats ? k_simulate<true, true> : k_simulate<true, false>);
        cudaFuncAttributes fa;
        DSD_CUDA(cudaFuncGetAttributes(&fa, k));
        DSD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      R.smem_optin - static_cast<int>(fa.sharedSizeBytes)));
        int pct = R.carveout;
        if (pct < 0) {
            const int64_t per_sm = (static_cast<int64_t>(R.n) + R.sms - 1) / R.sms;
            pct = static_cast<int>(std::min<int64_t>(
                100, (100 * per_sm * (static_cast<int64_t>(solo.bytes) + 1024) + R.smem_per_sm - 1) / R.smem_per_sm));
        }
        DSD_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        k<<<static_cast<unsigned>(R.n), kLanes, solo.bytes, R.stream>>>(Ws, nullptr, nullptr, 0);
        DSD_CUDA(cudaGetLastError());
        ++R.launches;
    } else if (smem) {
        // AWC with staged weights: one block of awc_warps_smem warps per SM
        const unsigned sthreads =
            R.awc_warps_smem > 0
                ? static_cast<unsigned>(awc_block_warps(R, R.awc_warps_smem, R.place_n ? R.place_n : static_cast<int64_t>(R.n)) * kLanes)
                : kBlock;
        const size_t bytes = (R.awc_warps_smem > 0 ? R.awc_wbytes : 0) +
                             static_cast<size_t>(sthreads / kLanes) * smem_warp_bytes(R.W.c.ns, R.smem_heap, R.W.c.awc != 0);
        const int32_t* pcount = R.place_n ? static_cast<const int32_t*>(R.place.p) : nullptr;
        const int32_t* plist = R.place_n ? pcount + 1 : nullptr;
        const unsigned sgrid = static_cast<unsigned>(((R.place_n ? R.place_n : static_cast<int64_t>(R.n)) + sthreads - 1) / sthreads);
        const bool spec = R.spec_ok && R.specialize && !R.collect && !R.W.probe;
        // Carveout: just the shared memory of the blocks one wave puts on an
        // SM (1 KB of it reserved per block); the rest of the 256 KB array is
        // L1.  The driver's default sizes for the launch-bounds maximum (8
        // blocks) even when 65,536 replicas need 7 per SM, costing 32-64 KB of L1.
        int pct = R.carveout;
        if (pct < 0) {
            const int64_t per_sm = R.awc_warps_smem > 0 ? 1 : std::min<int64_t>(spec ? DSD_SPEC_MIN_BLOCKS : DSD_MIN_BLOCKS, (sgrid + R.sms - 1) / R.sms);
            const int64_t need = per_sm * (static_cast<int64_t>(bytes) + 1024);
            pct = static_cast<int>(std::min<int64_t>(100, (100 * need + R.smem_per_sm - 1) / R.smem_per_sm));
        }
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, false, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, false, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, true, true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, false, true, false, 1>,
                                      cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        if (spec && R.spec_stack_limit1)
            k_simulate<true, false, true, false, 1><<<sgrid, kBlock, bytes, R.stream>>>(R.W, plist, pcount, R.smem_heap);
        else if (spec)
            (R.step_stats ? k_simulate<true, true, true> : k_simulate<true, false, true>)<<<sgrid, kBlock, bytes, R.stream>>>(
                R.W, plist, pcount, R.smem_heap);
        else if (R.W.c.awc)
            (R.step_stats ? k_simulate<true, true, false, true> : k_simulate<true, false, false, true>)<<<sgrid, sthreads, bytes,
                                                                                                    R.stream>>>(
                R.W, plist, pcount, R.smem_heap);
        else
            (R.step_stats ? k_simulate<true, true> : k_simulate<true, false>)<<<sgrid, kBlock, bytes, R.stream>>>(
                R.W, plist, pcount, R.smem_heap);
        DSD_CUDA(cudaGetLastError());
        ++R.launches;
    }
    if (smem) {
        // replicas whose event heap outgrew shared memory (or the specialised
        // kernel's action stack) run again: a specialised batch first in the
        // same kernel with a kSpecRerunHeap-slot heap (a lone C5 replica takes
        // ~2 ms there and ~30 ms in the HBM variant), then whatever still fails
        // from HBM
        R.ovf.ensure(8 * (R.n + 1));
        int32_t* count = static_cast<int32_t*>(R.ovf.p);
        int32_t* list = count + 1;
        const unsigned g2 = static_cast<unsigned>((R.n + 255) / 256);
        const bool spec = !solo.on && R.spec_ok && R.specialize && !R.collect && !R.W.probe;
        // (the generic shared-memory kernel likewise, with a kGenRerunHeap-slot heap; not AWC)
        const bool gen = !solo.on && !spec && !R.W.c.awc;
        R.spec_rerun = spec || gen;
        R.rerun_heap = spec ? kSpecRerunHeap : kGenRerunHeap;
        if (spec || gen) {
            int32_t* count1 = count + R.n + 1;
            int32_t* list1 = count1 + 1;
            DSD_CUDA(cudaMemsetAsync(count1, 0, 4, R.stream));
            k_collect_overflow<<<g2, 256, 0, R.stream>>>(R.W, list1, count1);
            k_stage<<<grid, kBlock, 0, R.stream>>>(R.W, nullptr, list1, count1);
            if (spec) {
                const size_t rbytes = (kBlock / kLanes) * smem_warp_bytes(2, kSpecRerunHeap, false);
                k_simulate<true, false, true><<<grid, kBlock, rbytes, R.stream>>>(R.W, list1, count1, kSpecRerunHeap);
            } else {
                const size_t rbytes = (kBlock / kLanes) * smem_warp_bytes(R.W.c.ns, kGenRerunHeap, false);
                cudaFuncAttributes fa;
                DSD_CUDA(cudaFuncGetAttributes(&fa, k_simulate<true, false>));
                DSD_CUDA(cudaFuncSetAttribute(k_simulate<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              R.smem_optin - static_cast<int>(fa.sharedSizeBytes)));
                k_simulate<true, false><<<grid, kBlock, rbytes, R.stream>>>(R.W, list1, count1, kGenRerunHeap);
            }
            DSD_CUDA(cudaGetLastError());
            R.launches += 3;
        }
        DSD_CUDA(cudaMemsetAsync(count, 0, 4, R.stream));
        k_collect_overflow<<<g2, 256, 0, R.stream>>>(R.W, list, count);
        k_stage<<<grid, kBlock, 0, R.stream>>>(R.W, R.collect ? static_cast<int64_t*>(R.ltot.p) : nullptr, list,
                                                count);
        (R.W.c.awc ? (R.step_stats ? k_simulate<false, true, false, true> : k_simulate<false, false, false, true>)
                    : (R.step_stats ? k_simulate<false, true> : k_simulate<false, false>))<<<hgrid_of(static_cast<int64_t>(R.n)), hcfg.threads, hbm_smem, R.stream>>>(R.W, list, count, 0);
        DSD_CUDA(cudaGetLastError());
        R.launches += 3;
    } else {
        // (HBM state is indexed by replica, so a lane placement is just a thread -> replica list)
        const int32_t* pcount = R.place_n ? static_cast<const int32_t*>(R.place.p) : nullptr;
        const int32_t* plist = R.place_n ? pcount + 1 : nullptr;
        const unsigned hgrid = hgrid_of(R.place_n ? R.place_n : static_cast<int64_t>(R.n));
        hbm_carveout(hgrid);
        (R.W.c.awc ? (R.step_stats ? k_simulate<false, true, false, true> : k_simulate<false, false, false, true>)
                    : (R.step_stats ? k_simulate<false, true> : k_simulate<false, false>))<<<hgrid, hcfg.threads, hbm_smem, R.stream>>>(R.W, plist, pcount, 0);
        DSD_CUDA(cudaGetLastError());
        ++R.launches;
    }
    DSD_CUDA(cudaEventRecord(R.ev[2], R.stream));
    lap("simulate");
    R.ran = true;
}

// The HBM variant's event heap holds Caps::hc = 2 x requests + 8 x servers +
// 64 pending events per replica.  That covers every pending event but the
// stale BatchReady timers a full-batch dispatch leaves behind when it
// disarms a batching window (engine.cpp:508-519): a window much longer than
// the service time can pile them up past hc.  Replicas that overflowed
// (kFailHeap after the HBM pass) run again with the heap doubled, in a
// separate heap buffer and otherwise the same workspace, until none
// overflows or the device has no room left for a larger heap.
static void retry_heap_overflows(RuntimeImpl& R) {
    int64_t hc = R.W.c.hc;
    const unsigned grid = static_cast<unsigned>((R.n + kBlock - 1) / kBlock);
    for (;;) {
        R.ovf2.ensure(4 * (R.n + 1));
        int32_t* count = static_cast<int32_t*>(R.ovf2.p);
        int32_t* list = count + 1;
        DSD_CUDA(cudaMemsetAsync(count, 0, 4, R.stream));
        k_collect_fail<<<static_cast<unsigned>((R.n + 255) / 256), 256, 0, R.stream>>>(R.W, kFailHeap, list, count);
        int32_t nfail = 0;
        DSD_CUDA(cudaMemcpyAsync(&nfail, count, 4, cudaMemcpyDeviceToHost, R.stream));
        DSD_CUDA(cudaStreamSynchronize(R.stream));
        if (nfail == 0) return;
        hc *= 2;
        if (std::getenv("DSD_HOST_TIMING"))
            std::fprintf(stderr, "[dsd sync] event heap overflow: %d replicas again with a heap of %lld\n", nfail,
                         static_cast<long long>(hc));
        const size_t slots = static_cast<size_t>(R.W.c.nwarps) * kLanes * static_cast<size_t>(hc);
        const size_t bytes = slots * (sizeof(int64_t) + sizeof(uint64_t));
        if (bytes > R.heap2.bytes) {
            size_t free_b = 0, total_b = 0;
            DSD_CUDA(cudaMemGetInfo(&free_b, &total_b));
            if (bytes + (256u << 20) > free_b + R.heap2.bytes) return;  // the replicas stay failed
        }
        R.heap2.ensure(bytes);
        Workspace W2 = R.W;
        W2.c.hc = hc;
        W2.h_time = static_cast<int64_t*>(R.heap2.p);
        W2.h_key = reinterpret_cast<uint64_t*>(W2.h_time + slots);
        const HbmCfg hc_cfg = hbm_cfg(R, static_cast<int64_t>(R.n));
        k_stage<<<grid, kBlock, 0, R.stream>>>(W2, nullptr, list, count);
        (R.W.c.awc ? k_simulate<false, false, false, true> : k_simulate<false, false>)<<<
            static_cast<unsigned>((R.n + hc_cfg.threads - 1) / hc_cfg.threads), hc_cfg.threads, hc_cfg.smem,
            R.stream>>>(W2, list, count, 0);
        DSD_CUDA(cudaGetLastError());
        R.launches += 3;
    }
}

void DeviceRuntime::sync() {
    RuntimeImpl& R = *impl_;
    DSD_CUDA(cudaSetDevice(R.device));
    DSD_CUDA(cudaStreamSynchronize(R.stream));
    if (R.ran && R.n > 0 && !R.retried) {
        retry_heap_overflows(R);
        R.retried = true;
    }
    if (R.ran && R.n > 0 && R.smem_launch && std::getenv("DSD_HOST_TIMING")) {  // replicas the shared-memory kernel handed on
        int32_t rerun = 0, rerun1 = 0;
        DSD_CUDA(cudaMemcpy(&rerun, R.ovf.p, sizeof(rerun), cudaMemcpyDeviceToHost));
        if (R.spec_rerun) {
            DSD_CUDA(cudaMemcpy(&rerun1, static_cast<int32_t*>(R.ovf.p) + R.n + 1, sizeof(rerun1), cudaMemcpyDeviceToHost));
            std::fprintf(stderr, "[dsd sync] re-run in the shared-memory kernel (%d-slot heap): %d of %zu replicas\n",
                         R.rerun_heap, rerun1, R.n);
        }
        std::fprintf(stderr, "[dsd sync] re-run on the HBM variant: %d of %zu replicas\n", rerun, R.n);
    }
    if (R.step_stats && R.W.step_stats) {
        unsigned long long s[64];
        static_assert(40 + kActKinds <= 64, "step stats layout");
        DSD_CUDA(cudaMemcpy(s, R.stats.p, sizeof(s), cudaMemcpyDeviceToHost));
        if (const char* f = std::getenv("DSD_REP_STATS_FILE")) {  // per-replica [n][3], raw u64
            std::vector<unsigned long long> rs(3 * R.n);
            DSD_CUDA(cudaMemcpy(rs.data(), R.W.rep_stats, 8 * rs.size(), cudaMemcpyDeviceToHost));
            if (FILE* fp = std::fopen(f, "wb")) {
                std::fwrite(rs.data(), 8, rs.size(), fp);
                std::fclose(fp);
            }
        }
        static const char* names[] = {"pop", "arrival", "net_prompt", "net_proposal", "net_result", "begin",
                                      "compute_done", "item", "finish", "activate", "dispatch", "send_prompt"};
        unsigned long long steps = 0;
        for (int k = 0; k < kActKinds; ++k) steps += s[2 * k + 1];
        std::fprintf(stderr, "[dsd step stats] warp iterations %llu (max %llu), warp cycles %llu, lane steps %llu\n",
                     s[32], s[34], s[33], steps);
        for (int k = 0; k < kActKinds; ++k)
            if (s[2 * k + 1])
                std::fprintf(stderr, "  %-13s steps %12llu  avg cycles/step %8.1f  rounds %10llu  lanes/round %5.2f\n",
                             names[k], s[2 * k + 1], static_cast<double>(s[2 * k]) / static_cast<double>(s[2 * k + 1]),
                             s[40 + k], s[40 + k] ? static_cast<double>(s[2 * k + 1]) / s[40 + k] : 0.0);
    }
}

void DeviceRuntime::last_kernel_ms(double* sim_ms, double* gen_ms, double* total_ms) {
    RuntimeImpl& R = *impl_;
    float a = 0, b = 0;
    if (R.ran && R.n > 0) {
        DSD_CUDA(cudaEventSynchronize(R.ev[2]));
        DSD_CUDA(cudaEventElapsedTime(&a, R.ev[1], R.ev[2]));
        DSD_CUDA(cudaEventElapsedTime(&b, R.ev[0], R.ev[2]));
    }
    if (sim_ms) *sim_ms = a;
    if (total_ms) *total_ms = b;
    if (gen_ms) *gen_ms = b - a;
}

void DeviceRuntime::summaries(dsd_replica_summary* out, size_t n) {
    RuntimeImpl& R = *impl_;
    if (!R.ran) throw Error(DSD_ERR_RUNTIME, "no completed batch");
    if (n > R.n) throw Error(DSD_ERR_RUNTIME, "summary buffer larger than the batch");
    sync();  // (and the heap-overflow retries)
    if (n) DSD_CUDA(cudaMemcpyAsync(out, R.summary.p, sizeof(DevSummary) * n, cudaMemcpyDeviceToHost, R.stream));
    R.d2h_bytes += static_cast<int64_t>(sizeof(DevSummary) * n);
    DSD_CUDA(cudaStreamSynchronize(R.stream));
}

const dsd_replica_summary* DeviceRuntime::host_summaries() {
    RuntimeImpl& R = *impl_;
    if (!R.ran) throw Error(DSD_ERR_RUNTIME, "no completed batch");
    DSD_CUDA(cudaSetDevice(R.device));
    const size_t bytes = sizeof(DevSummary) * std::max<size_t>(R.n, 1);
    if (bytes > R.pinned_bytes) {  // grown, never shrunk: later batches touch no fresh pages
        if (R.pinned) DSD_CUDA(cudaFreeHost(R.pinned));
        R.pinned = nullptr;
        R.pinned_bytes = 0;
        DSD_CUDA(cudaMallocHost(&R.pinned, bytes));
        R.pinned_bytes = bytes;
    }
    if (R.pinned_valid) return static_cast<const dsd_replica_summary*>(R.pinned);
    sync();
    if (R.n) DSD_CUDA(cudaMemcpyAsync(R.pinned, R.summary.p, sizeof(DevSummary) * R.n, cudaMemcpyDeviceToHost, R.stream));
    R.d2h_bytes += static_cast<int64_t>(sizeof(DevSummary) * R.n);
    DSD_CUDA(cudaStreamSynchronize(R.stream));
    R.pinned_valid = true;
    return static_cast<const dsd_replica_summary*>(R.pinned);
}

static_assert(kProbeFields == DSD_PROBE_FIELDS, "probe layout must match include/dsdsim.h");
static_assert(sizeof(DevSummary) == sizeof(dsd_replica_summary), "summary layout must match include/dsdsim.h");

void DeviceRuntime::probe(double* out, size_t n) {
    RuntimeImpl& R = *impl_;
    if (!R.ran || !R.W.probe) throw Error(DSD_ERR_RUNTIME, "the batch did not run with the feature probe");
    if (n > R.n) n = R.n;
    sync();
    if (n) DSD_CUDA(cudaMemcpy(out, R.W.probe, sizeof(double) * kProbeFields * n, cudaMemcpyDeviceToHost));
}

void DeviceRuntime::fetch_event_log(size_t replica, std::vector<char>* elog, std::vector<char>* busy) {
    RuntimeImpl& R = *impl_;
    if (!R.ran || !R.elog_on) throw Error(DSD_ERR_RUNTIME, "the batch did not record an event log");
    if (replica >= R.n) throw Error(DSD_ERR_RUNTIME, "replica index out of range");
    sync();
    int64_t n[2] = {0, 0};
    DSD_CUDA(cudaMemcpy(&n[0], R.W.elog_n + replica, 8, cudaMemcpyDeviceToHost));
    DSD_CUDA(cudaMemcpy(&n[1], R.W.busy_n + replica, 8, cudaMemcpyDeviceToHost));
    if (elog) {
        elog->resize(sizeof(ElogRec) * static_cast<size_t>(n[0]));
        if (n[0])
            DSD_CUDA(cudaMemcpy(elog->data(), R.W.elog + static_cast<int64_t>(replica) * R.W.elog_cap, elog->size(),
                                cudaMemcpyDeviceToHost));
    }
    if (busy) {
        busy->resize(sizeof(BusyRec) * static_cast<size_t>(n[1]));
        if (n[1])
            DSD_CUDA(cudaMemcpy(busy->data(), R.W.busy_iv + static_cast<int64_t>(replica) * R.W.busy_cap,
                                busy->size(), cudaMemcpyDeviceToHost));
    }
}

void DeviceRuntime::device_summaries(void** ptr, size_t* bytes) {
    *ptr = impl_->summary.p;
    *bytes = sizeof(DevSummary) * impl_->n;
}

void DeviceRuntime::fetch_records(size_t replica, dsd_request_record* records, size_t cap,
                            int64_t* n_records, int32_t* gamma_seq, int32_t* committed_seq,
                            size_t seq_cap, int64_t* n_seq, int64_t* busy_us, size_t busy_cap) {
    RuntimeImpl& R = *impl_;
    if (!R.ran || !R.collect) throw Error(DSD_ERR_RUNTIME, "records were not collected for this batch");
    if (replica >= R.n) throw Error(DSD_ERR_RUNTIME, "replica index out of range");
    sync();  // (and the heap-overflow retries)
    const Caps& c = R.W.c;
    if (!R.rec_cached) {
        R.rec.ensure(sizeof(DevRecord) * static_cast<size_t>(c.nr) * R.n);
        R.busy.ensure(sizeof(int64_t) * static_cast<size_t>(c.nt) * R.n);
        const unsigned grid = static_cast<unsigned>((R.n + 127) / 128);
        k_export<<<grid, 128, 0, R.stream>>>(R.W, static_cast<DevRecord*>(R.rec.p), static_cast<int64_t*>(R.busy.p));
        DSD_CUDA(cudaGetLastError());
        R.h_rec.resize(static_cast<size_t>(c.nr) * R.n);
        R.h_busy.resize(static_cast<size_t>(c.nt) * R.n);
        R.h_seqg.resize(static_cast<size_t>(std::max<int64_t>(R.W.seq_cap, 1)));
        R.h_seqc.resize(R.h_seqg.size());
        DSD_CUDA(cudaMemcpyAsync(R.h_rec.data(), R.rec.p, sizeof(DevRecord) * R.h_rec.size(), cudaMemcpyDeviceToHost, R.stream));
        DSD_CUDA(cudaMemcpyAsync(R.h_busy.data(), R.busy.p, 8 * R.h_busy.size(), cudaMemcpyDeviceToHost, R.stream));
        if (R.W.seq_cap > 0) {
            DSD_CUDA(cudaMemcpyAsync(R.h_seqg.data(), R.seqg.p, 4 * R.W.seq_cap, cudaMemcpyDeviceToHost, R.stream));
            DSD_CUDA(cudaMemcpyAsync(R.h_seqc.data(), R.seqc.p, 4 * R.W.seq_cap, cudaMemcpyDeviceToHost, R.stream));
        }
        DSD_CUDA(cudaStreamSynchronize(R.stream));
        R.rec_cached = true;
    }
    const DevScenario& S = R.packed.scen[0];
    (void)S;
    // the batch's summaries come back once, in bulk (host_summaries), not one
    // blocking copy per call
    if (!R.pinned_valid) host_summaries();
    const int64_t N = static_cast<const dsd_replica_summary*>(R.pinned)[replica].n_requests;
    if (n_records) *n_records = N;
    const DevRecord* src = R.h_rec.data() + replica * c.nr;
    if (records) {
        for (int64_t i = 0; i < N && static_cast<size_t>(i) < cap; ++i)
            std::memcpy(&records[i], &src[i], sizeof(DevRecord));
    }
    int64_t total = 0;
    for (int64_t i = 0; i < N; ++i) total += src[i].n_iterations;
    if (n_seq) *n_seq = total;
    if (gamma_seq || committed_seq) {
        // per request the sequence starts at seqbase + prefix of output lengths
        int64_t w = 0, pref = 0;
        for (int64_t i = 0; i < N; ++i) {
            int64_t base = R.host_seqbase[replica] + pref;
            for (int32_t k = 0; k < src[i].n_iterations && static_cast<size_t>(w) < seq_cap; ++k, ++w) {
                if (gamma_seq) gamma_seq[w] = R.h_seqg[base + k];
                if (committed_seq) committed_seq[w] = R.h_seqc[base + k];
            }
            pref += src[i].output_length;
        }
    }
    if (busy_us) {
        for (size_t t = 0; t < busy_cap && t < static_cast<size_t>(c.nt); ++t)
            busy_us[t] = R.h_busy[replica * c.nt + t];
    }
}

}  // namespace dsd
