// pack.hpp — host-side batch packing shared by the CUDA runtime.
#pragma once
#include <cstdint>
#include <vector>

#include "dsdsim.h"
#include "layout.cuh"
#include "runtime.hpp"

namespace dsd {

struct Packed {
    std::vector<char> blob;
    std::vector<DevScenario> scen;
    Caps caps{};
    std::vector<uint32_t> rep_scen;
    std::vector<uint64_t> seed, gseed;
};

// Validates the scenarios (reference error texts, DSD_ERR_CONFIG) and packs
// them into the scenario blob; computes the batch capacities.  `probe`: the
// batch runs with the feature probe, so every scenario with draft servers
// keeps the pair metric rings (the reference always does).
Packed pack_batch(const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas, size_t n,
                  bool probe = false);
// The same into P, reusing its vectors' storage (a Runtime packs every batch
// into one Packed, so repeated batches touch no fresh host pages).
void pack_batch_into(Packed& P, const dsd_scenario* scenarios, size_t n_scenarios, const dsd_replica* replicas,
                     size_t n, bool probe);

// Assigns the workspace field pointers inside [base, base + bytes) and
// returns bytes; with base == nullptr it only sizes.
size_t layout_workspace(Workspace& W, const Caps& c, char* base);

}  // namespace dsd
