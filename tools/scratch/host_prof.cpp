// Host-side timing of the sweep planning and packing (no GPU): plan_range and
// pack_batch_into of the C5 sweep, repeated.  Scratch profiling harness:
//   g++ -O2 -std=c++17 -pg ... (see host_prof.sh)
#include <chrono>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "../../paper_2511_21669_b200/csrc/device/pack.hpp"
#include "../../paper_2511_21669_b200/csrc/host/sweep.hpp"

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "configs/c5_sweep_65536.yaml";
    const int iters = argc > 2 ? std::atoi(argv[2]) : 5;
    std::ifstream f(path);
    std::stringstream ss;
    ss << f.rdbuf();
    dsd::host::Caches caches;
    dsd::Packed P;
    for (int it = 0; it < iters; ++it) {
        auto t0 = std::chrono::steady_clock::now();
        auto node = dsd::cfg::parse(ss.str());
        auto spec = dsd::host::SweepSpec::from_node(node, "configs");
        auto b = dsd::host::plan_range(spec, 0, spec.point_count(), &caches);
        auto t1 = std::chrono::steady_clock::now();
        dsd::pack_batch_into(P, b.scenarios.data(), b.scenarios.size(), b.replicas.data(), b.replicas.size(), false);
        auto t2 = std::chrono::steady_clock::now();
        auto parts = dsd::host::render_summary_prefixes(b.points, 0);
        std::string js, cs;
        dsd::host::assemble_summaries(parts, b.points, &js, &cs);
        auto t3 = std::chrono::steady_clock::now();
        auto sh = dsd::shard_of_replicas(b.scenarios.data(), b.replicas.data(), b.replicas.size(), 4);
        auto t4 = std::chrono::steady_clock::now();
        std::printf("shard_of_replicas %.2f ms (%d)\n", std::chrono::duration<double, std::milli>(t4 - t3).count(), sh[7]);
        std::printf("plan %.2f ms  pack %.2f ms  summary %.2f ms  (%zu replicas)\n",
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count(),
                    std::chrono::duration<double, std::milli>(t3 - t2).count(), b.replicas.size());
    }
}
