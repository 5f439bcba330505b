// Launch wrappers of the sampler kernels (sampler.cu), used by the C-ABI entry points in
// sampler.cu itself and by the sample stream (stream.cu). All pointers are device pointers.
#pragma once

#include "common.cuh"

namespace hsawgpu {

// index into the u64[8] stats block (hsaw_gpu.h: hsaw_gpu_encode_batches)
enum { ST_ATTEMPTS = 0, ST_DRAWS = 1, ST_STEPS = 2, ST_BYTES = 3, ST_ACCEPTED = 4,
       ST_DECODE_STEPS = 5, ST_DROPPED = 6, ST_SPARE = 7 };

void validate_cfg(const hsaw_sampler_cfg& cfg);

// K1: batches [first_worker, first_worker + nbatches) -> per-batch count + (seed, len) slots.
// d_stats: u64[8] accumulated (never reset here). d_cursor: one zeroed u64 of scratch.
// Optional recording: accepted walks are logged as (node, edge id) pairs into `arena` while K1
// generates them (one 32-byte sector store per four steps); out_log[slot] = first pair of the walk
// or record_overflow_marker() when the walk outgrew its chunk / the arena and must be replayed.
struct EncodeRecord {
    uint2* arena;
    uint32_t arena_cap;      // pairs, >= record_chunk_pairs()
    uint32_t* arena_cursor;  // one u32 of device scratch
    uint32_t* out_log;       // nbatches * batch_size entries
};
uint32_t record_chunk_pairs();
uint32_t record_overflow_marker();
uint64_t record_resident_lanes(hsaw_gpu_ctx* ctx);

void launch_encode(hsaw_gpu_ctx* ctx, const hsaw_sampler_cfg& cfg, uint64_t first_worker,
                   uint64_t nbatches, uint64_t* d_seed, uint32_t* d_len, uint32_t* d_count,
                   uint64_t* d_stats, uint64_t* d_cursor, const EncodeRecord* rec,
                   bool with_stats);
// Recording is built for the default SamplerConfig (Brent + window 2) only.
bool record_supported(const hsaw_sampler_cfg& cfg);

// K2: replay nwalks encoded walks into nodes/edges at edge_off (exclusive sum of lens).
// d_status[w]: 1 replayed, 2 mismatch. d_cursor: one zeroed u64 of scratch.
void launch_decode(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* d_seed,
                   const uint32_t* d_len, const uint64_t* d_edge_off, uint32_t* d_nodes,
                   uint32_t* d_edges, uint8_t* d_status, uint64_t* d_stats, uint64_t* d_cursor);

// K2b: exact self-avoidance recheck; sets d_status[w] = 0 for walks (status 1) whose node list
// is not pairwise distinct. Synchronises the stream; returns the number of walks dropped.
uint32_t launch_distinct_check(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* d_edge_off,
                               const uint32_t* d_nodes, uint8_t* d_status);

// Pair-log variants used by the fused stream path: replay of selected walks into pair logs, and
// the recheck reading nodes from d_pair_src[w][0..d_lens[w]].x.
void launch_decode_pairs(hsaw_gpu_ctx* ctx, uint64_t nsel, const uint32_t* d_sel,
                         const uint64_t* d_seed, const uint32_t* d_len, uint2* const* d_pair_dst,
                         uint8_t* d_status, uint64_t* d_stats, uint64_t* d_cursor,
                         bool on_side = false);
// on_side replays run beside the context stream until join_side_stream (called by the recheck
// after its main pass); that is safe for walks of more than this many edges
uint32_t distinct_check_defers_walks_longer_than();
void join_side_stream(hsaw_gpu_ctx* ctx);
uint32_t launch_distinct_check_pairs(hsaw_gpu_ctx* ctx, uint64_t nwalks,
                                     const uint2* const* d_pair_src, const uint32_t* d_lens,
                                     uint8_t* d_status);

}  // namespace hsawgpu
