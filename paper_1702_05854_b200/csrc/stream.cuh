// Device-resident SampleStream (proj/src/sampler.cpp:383-501): decoded walks in deterministic
// (batch, seq) order in one dense pool, plus the per-batch cumulative accepted counts that
// counters_for needs.
#pragma once

#include <vector>

#include "common.cuh"

struct hsaw_gpu_stream {
    hsaw_gpu_ctx* ctx = nullptr;
    uint64_t uid = 0;  // process-unique id (caches keyed by stream must survive address reuse)
    uint64_t seed = 0;
    hsaw_sampler_cfg cfg{};

    // pool: walk w has edges [edge_off[w], edge_off[w+1]) and nodes
    // [edge_off[w] + w, edge_off[w+1] + w + 1)  (len + 1 nodes per walk, no padding)
    hsawgpu::DevVec<uint64_t> edge_off;  // accepted + 1
    hsawgpu::GrowVec<uint32_t> nodes;    // total_edges + accepted   (grown in place, see GrowVec)
    hsawgpu::GrowVec<uint32_t> edges;    // total_edges
    // Which item arrays the pool keeps (hsaw_gpu_stream_keep): a solve over edge candidates never
    // reads the node lists and vice versa; at the Twitter shape each array is tens of gigabytes.
    bool keep_nodes = true, keep_edges = true;
    hsawgpu::DevVec<uint64_t> tag_batch; // global batch index of each walk (worker id = seed + it)
    hsawgpu::DevVec<uint32_t> tag_seq;   // seq within the batch, assigned before decode drops
    uint64_t accepted = 0, total_edges = 0;

    // cumulative decoded count after each batch this stream ran, in the order it ran them
    hsawgpu::DevVec<uint64_t> accepted_after_batch;
    uint64_t local_batches = 0;
    uint64_t next_batch = 0;   // next global batch for ensure()
    uint64_t last_batch_end = 0;  // ranges must be increasing
    uint64_t grow = 4096;      // first-round size while nothing has been accepted yet

    // Partitioned sampling (hsaw_gpu_stream_restrict; proj/src/partition.cpp:183-268): start domain,
    // allowed mask, and the cumulative crossing count after each batch (host side, like the
    // reference's crossed_after vector)
    hsawgpu::DevVec<uint32_t> r_domain, r_cross;
    hsawgpu::DevVec<uint8_t> r_allowed;
    uint32_t r_ndomain = 0;
    std::vector<uint64_t> crossed_after_batch;

    hsawgpu::DevVec<uint64_t> stats;  // u64[8] + cursor scratch
    uint64_t dropped = 0;             // walks removed by the exact recheck
    bool collect_stats = false;       // K1 work counters (draws/picks/bytes): instrumentation only
    uint64_t replayed = 0;            // fused path: walks whose log overflowed (replayed by K2)
    double pairs_per_attempt = 0;     // fused path: running arena-volume estimate

};

// A fixed collection of item sets on the device (CoverageIndex input): the fixed-walk-set parity
// mode (hsaw_gpu_walkset_import) and the reverse-reachable node sets of the InfMax baselines.
struct hsaw_gpu_walkset {
    hsaw_gpu_ctx* ctx = nullptr;
    uint32_t limit = 0;
    uint64_t nsets = 0, nitems = 0;
    hsawgpu::DevVec<uint64_t> off;
    hsawgpu::DevVec<uint32_t> items;
};
