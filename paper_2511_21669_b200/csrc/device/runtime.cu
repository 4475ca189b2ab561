// runtime.cu — packs resolved scenarios into a device blob, sizes the replica
// workspace, and launches the staging + simulation kernels for sm_100a.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
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
__global__ void __launch_bounds__(kBlock) k_stage(Workspace W, int64_t* ltot) {
    int64_t rep = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (rep >= W.c.n) return;
    stage_workload(W, rep);
    if (ltot) {
        const DevScenario& S = W.scen[W.rep_scen[rep]];
        int64_t N = S.workload == 0 ? S.n_requests : S.tr_n;
        Lane L{rep / kLanes, static_cast<int>(rep % kLanes)};
        ltot[rep] = N == 0 ? 0 : L.at(W.r_seqoff, W.c.nr, N - 1) + L.at(W.r_output, W.c.nr, N - 1);
    }
}

__global__ void __launch_bounds__(kBlock) k_simulate(Workspace W) {
    int64_t rep = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (rep >= W.c.n) return;
    Engine e(W, W.scen[W.rep_scen[rep]], rep);
    e.run();
}

__global__ void k_export(Workspace W, DevRecord* rec, int64_t* busy) {
    int64_t rep = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (rep >= W.c.n) return;
    const DevScenario& S = W.scen[W.rep_scen[rep]];
    Lane L{rep / kLanes, static_cast<int>(rep % kLanes)};
    const int64_t nr = W.c.nr;
    int64_t N = S.workload == 0 ? S.n_requests : S.tr_n;
    for (int64_t i = 0; i < N; ++i) {
        DevRecord r;
        r.drafter_id = S.n_drafts > 0 ? L.at(W.r_drafter, nr, i) : -1;
        r.prompt_length = L.at(W.r_prompt, nr, i);
        r.output_length = L.at(W.r_output, nr, i);
        r.arrival_us = L.at(W.r_arrival, nr, i);
        r.first_token_us = L.at(W.r_first, nr, i);
        r.completion_us = L.at(W.r_done, nr, i);
        r.proposed = L.at(W.r_prop, nr, i);
        r.accepted = L.at(W.r_acc, nr, i);
        r.target_id = L.at(W.r_target, nr, i);
        r.n_iterations = L.at(W.r_ng, nr, i);
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
    DevBuf blob, scen, reps, arena, summary, fail, ltot, seqbase, seqg, seqc, rec, busy;
    Workspace W{};
    std::vector<DevScenario> host_scen;
    std::vector<int64_t> host_seqbase;
    std::vector<int64_t> host_ltot;
    size_t n = 0;
    bool collect = false;
    bool prepared = false;
    bool ran = false;
    int64_t launches = 0;
    // records cache (filled lazily after a collect run)
    bool rec_cached = false;
    std::vector<DevRecord> h_rec;
    std::vector<int64_t> h_busy;
    std::vector<int32_t> h_seqg, h_seqc;
};

Runtime::Runtime(int device) : impl_(new RuntimeImpl) {
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
    for (auto& ev : impl_->ev) DSD_CUDA(cudaEventCreate(&ev));
}

Runtime::~Runtime() {
    if (!impl_) return;
    cudaSetDevice(impl_->device);
    if (impl_->stream) cudaStreamSynchronize(impl_->stream);
    for (auto& ev : impl_->ev)
        if (ev) cudaEventDestroy(ev);
    if (impl_->stream) cudaStreamDestroy(impl_->stream);
}

void* Runtime::stream() { return impl_->stream; }
int64_t Runtime::last_launch_count() const { return impl_->launches; }
size_t Runtime::replica_count() const { return impl_->n; }

void Runtime::prepare(const dsd_scenario* sc, size_t ns, const dsd_replica* reps, size_t n,
                      bool collect) {
    RuntimeImpl& R = *impl_;
    DSD_CUDA(cudaSetDevice(R.device));
    R.prepared = false;
    R.ran = false;
    R.rec_cached = false;
    Packed P = pack_batch(sc, ns, reps, n);
    const Caps& c = P.caps;
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
    R.summary.ensure(sizeof(DevSummary) * std::max<size_t>(n, 1));
    R.fail.ensure(sizeof(int32_t) * std::max<size_t>(n, 1));

    // ---- workspace arena ----
    Workspace& W = R.W;
    W = Workspace{};
    const size_t total = layout_workspace(W, c, nullptr);
    size_t free_b = 0, total_b = 0;
    DSD_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (total > R.arena.bytes && total + (256u << 20) > free_b + R.arena.bytes)
        throw Error(DSD_ERR_RUNTIME, "replica workspace (" + std::to_string(total >> 20) +
                                         " MiB) exceeds free device memory");
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
    R.host_scen = std::move(P.scen);
    R.n = n;
    R.collect = collect;
    if (collect) R.ltot.ensure(sizeof(int64_t) * std::max<size_t>(n, 1));
    DSD_CUDA(cudaStreamSynchronize(R.stream));
    R.prepared = true;
}

void Runtime::launch() {
    RuntimeImpl& R = *impl_;
    if (!R.prepared) throw Error(DSD_ERR_RUNTIME, "launch without a prepared batch");
    DSD_CUDA(cudaSetDevice(R.device));
    R.launches = 0;
    R.rec_cached = false;
    if (R.n == 0) {
        R.ran = true;
        return;
    }
    const unsigned grid = static_cast<unsigned>((R.n + kBlock - 1) / kBlock);
    DSD_CUDA(cudaEventRecord(R.ev[0], R.stream));
    k_stage<<<grid, kBlock, 0, R.stream>>>(R.W, R.collect ? static_cast<int64_t*>(R.ltot.p) : nullptr);
    DSD_CUDA(cudaGetLastError());
    ++R.launches;
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
    }
    DSD_CUDA(cudaEventRecord(R.ev[1], R.stream));
    k_simulate<<<grid, kBlock, 0, R.stream>>>(R.W);
    DSD_CUDA(cudaGetLastError());
    ++R.launches;
    DSD_CUDA(cudaEventRecord(R.ev[2], R.stream));
    R.ran = true;
}

void Runtime::sync() {
    RuntimeImpl& R = *impl_;
    DSD_CUDA(cudaSetDevice(R.device));
    DSD_CUDA(cudaStreamSynchronize(R.stream));
}

void Runtime::last_kernel_ms(double* sim_ms, double* gen_ms, double* total_ms) {
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

void Runtime::summaries(dsd_replica_summary* out, size_t n) {
    RuntimeImpl& R = *impl_;
    if (!R.ran) throw Error(DSD_ERR_RUNTIME, "no completed batch");
    if (n > R.n) throw Error(DSD_ERR_RUNTIME, "summary buffer larger than the batch");
    DSD_CUDA(cudaSetDevice(R.device));
    if (n) DSD_CUDA(cudaMemcpyAsync(out, R.summary.p, sizeof(DevSummary) * n, cudaMemcpyDeviceToHost, R.stream));
    DSD_CUDA(cudaStreamSynchronize(R.stream));
}

void Runtime::device_summaries(void** ptr, size_t* bytes) {
    *ptr = impl_->summary.p;
    *bytes = sizeof(DevSummary) * impl_->n;
}

void Runtime::fetch_records(size_t replica, dsd_request_record* records, size_t cap,
                            int64_t* n_records, int32_t* gamma_seq, int32_t* committed_seq,
                            size_t seq_cap, int64_t* n_seq, int64_t* busy_us, size_t busy_cap) {
    RuntimeImpl& R = *impl_;
    if (!R.ran || !R.collect) throw Error(DSD_ERR_RUNTIME, "records were not collected for this batch");
    if (replica >= R.n) throw Error(DSD_ERR_RUNTIME, "replica index out of range");
    DSD_CUDA(cudaSetDevice(R.device));
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
    const DevScenario& S = R.host_scen[0];
    (void)S;
    dsd_replica_summary sm;
    DSD_CUDA(cudaMemcpy(&sm, static_cast<DevSummary*>(R.summary.p) + replica, sizeof(sm), cudaMemcpyDeviceToHost));
    const int64_t N = sm.n_requests;
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
