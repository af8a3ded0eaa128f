// Interface of the level-synchronous traversal (traverse.cu).
#pragma once

#include <vector>

#include "hxf_internal.cuh"

struct TravInput {
    hxf_system* sys;
    hxf_pairs* bra;
    hxf_pairs* ket;
    hxf_density* dens;
    double tau;
    int mode;
    int sym;               // 0 naive, 1 fourfold, 2 eightfold (fourfold restricted to bra <= ket)
    int shard_level;       // < 0: whole tree
    int64_t shard_begin;
    int64_t shard_end;
    int64_t shard_stride;  // > 1: every stride-th task of [begin, end)
    const uint8_t* shard_mask;  // host; non-NULL: tasks t < shard_end with mask[t] != 0
    int frontier_only;     // stop at frontier_level and return its expand list
    int frontier_level;
    long long* counters;   // device C_NCOUNTERS
    unsigned long long* ledger;  // device LEDGER_LIMBS
    int root_level = 0;    // the traversal starts at the diagonal node (root_index, root_index)
    int root_index = 0;    // of this level (a diagonal subtree; 0, 0 = the tree root)
    TieLog ties{nullptr, nullptr, 0};   // device tie log (task stage), or disabled
};

struct TraversalResult {
    uint64_t* leaf;        // device leaf tasks (partition-leaf ids + live mask)
    int64_t n_leaf;
    uint64_t* frontier = nullptr;  // frontier_only: expand list at frontier_level
    int64_t n_frontier = 0;
    std::vector<int64_t> frontier_sizes;
};

TraversalResult traverse(const TravInput& in, cudaStream_t st);
