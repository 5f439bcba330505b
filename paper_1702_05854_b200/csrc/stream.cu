// Sample stream: orchestration of K1 (encode) -> gather -> K2 (decode) -> K2b (exact recheck) ->
// deterministic compaction into the dense walk pool. Order contract (proj/src/sampler.cpp:452-460):
// walks are appended in (batch, seq) order — positions come from prefix sums, never from atomics —
// so prefixes of the pool are pure functions of (graph, suspects, seed) exactly as in the reference.
#include "stream.cuh"

#include <atomic>
#include <cmath>
#include <cstdlib>

#include "sampler.cuh"

using namespace hsawgpu;

namespace {

constexpr uint64_t kMaxChunkBatches = 1ull << 22;  // bounds per-chunk scratch (slots = 10x this)
constexpr uint64_t kArenaTargetBytes = 6ull << 30;  // soft bound of the K1 pair-log arena per chunk

// (batch, seq) slots -> dense encoded list in batch-major order. One thread per slot.
__global__ void gather_encoded(uint64_t nbatches, uint32_t l, uint64_t first_global_batch,
                               const uint32_t* __restrict__ count,
                               const uint32_t* __restrict__ first,
                               const uint64_t* __restrict__ slot_seed,
                               const uint32_t* __restrict__ slot_len, uint64_t* __restrict__ enc_seed,
                               uint32_t* __restrict__ enc_len, uint64_t* __restrict__ enc_batch,
                               uint32_t* __restrict__ enc_seq) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbatches * l) return;
    uint64_t b = i / l;
    uint32_t j = (uint32_t)(i - b * l);
    if (j >= count[b]) return;
    uint32_t dst = first[b] + j;
    enc_seed[dst] = slot_seed[i];
    enc_len[dst] = slot_len[i];
    enc_batch[dst] = first_global_batch + b;
    enc_seq[dst] = j;
}

// status -> (valid flag, valid length) for the two compaction scans; flags a replay mismatch.
__global__ void mark_valid(uint64_t nwalks, const uint8_t* __restrict__ status,
                           const uint32_t* __restrict__ enc_len, uint32_t* __restrict__ vflag,
                           uint32_t* __restrict__ vlen, uint32_t* __restrict__ mismatch) {
    uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w > nwalks) return;
    if (w == nwalks) {  // scan sentinels
        vflag[w] = 0;
        vlen[w] = 0;
        return;
    }
    uint8_t st = status[w];
    if (st == 2) atomicExch(mismatch, 1u);
    vflag[w] = st == 1;
    vlen[w] = st == 1 ? enc_len[w] : 0;
}

// One warp per decoded walk: copy it to its final place in the pool.
__global__ void compact_walks(uint64_t nwalks, const uint32_t* __restrict__ vflag,
                              const uint32_t* __restrict__ vidx, const uint64_t* __restrict__ voff,
                              const uint64_t* __restrict__ tmp_off,
                              const uint32_t* __restrict__ tmp_nodes,
                              const uint32_t* __restrict__ tmp_edges,
                              const uint32_t* __restrict__ enc_len,
                              const uint64_t* __restrict__ enc_batch,
                              const uint32_t* __restrict__ enc_seq, uint64_t base_walk,
                              uint64_t base_edge, uint64_t* __restrict__ edge_off,
                              uint32_t* __restrict__ nodes, uint32_t* __restrict__ edges,
                              uint64_t* __restrict__ tag_batch, uint32_t* __restrict__ tag_seq) {
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = warp; w < nwalks; w += nwarps) {
        if (!vflag[w]) continue;
        uint64_t dw = base_walk + vidx[w];
        uint64_t de = base_edge + voff[w];
        uint32_t len = enc_len[w];
        uint64_t se = tmp_off[w];
        if (lane == 0) {
            edge_off[dw] = de;
            tag_batch[dw] = enc_batch[w];
            tag_seq[dw] = enc_seq[w];
        }
        if (nodes)
            for (uint32_t i = lane; i <= len; i += 32) nodes[de + dw + i] = tmp_nodes[se + w + i];
        if (edges)
            for (uint32_t i = lane; i < len; i += 32) edges[de + i] = tmp_edges[se + i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        edge_off[base_walk + vidx[nwalks]] = base_edge + voff[nwalks];
}

// ---- fused path: K1 logged the walks as (node, edge id) pairs while generating them ------------
// (batch, seq) slots -> dense encoded list, plus where each walk's pair log lives. Walks whose log
// overflowed get a null source here and are marked for replay.
__global__ void gather_recorded(uint64_t nbatches, uint32_t l, uint64_t first_global_batch,
                                const uint32_t* __restrict__ count,
                                const uint32_t* __restrict__ first,
                                const uint64_t* __restrict__ slot_seed,
                                const uint32_t* __restrict__ slot_len,
                                const uint32_t* __restrict__ slot_log, const uint2* arena,
                                uint32_t overflow_marker, uint64_t* __restrict__ enc_seed,
                                uint32_t* __restrict__ enc_len, uint64_t* __restrict__ enc_batch,
                                uint32_t* __restrict__ enc_seq, const uint2** __restrict__ enc_src,
                                uint32_t* __restrict__ ovf_pairs) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nbatches * l) return;
    uint64_t b = i / l;
    uint32_t j = (uint32_t)(i - b * l);
    if (j >= count[b]) return;
    uint32_t dst = first[b] + j;
    uint32_t len = slot_len[i], lg = slot_log[i];
    enc_seed[dst] = slot_seed[i];
    enc_len[dst] = len;
    enc_batch[dst] = first_global_batch + b;
    enc_seq[dst] = j;
    bool ovf = lg == overflow_marker;
    enc_src[dst] = ovf ? nullptr : arena + lg;
    ovf_pairs[dst] = ovf ? ((len + 1 + 3) & ~3u) : 0;  // replay space, sector aligned
}

// Overflowed walks: point them at their slice of the replay buffer and list them for K2.
__global__ void place_overflow(uint64_t nwalks, const uint32_t* __restrict__ ovf_pairs,
                               const uint64_t* __restrict__ ovf_off, uint2* replay_base,
                               const uint2** __restrict__ enc_src, uint32_t* __restrict__ sel,
                               uint32_t* __restrict__ nsel, const uint32_t* __restrict__ enc_len) {
    uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwalks || ovf_pairs[w] == 0) return;
    enc_src[w] = replay_base + ovf_off[w];
    sel[atomicAdd(nsel, 1u)] = (uint32_t)w;  // order is irrelevant: each entry is independent work
    atomicMin(nsel + 1, enc_len[w]);         // shortest replayed walk (decides the overlap below)
}

// Pair logs -> final node / edge arrays of the pool. One warp per group of 32 encoded walks: each
// lane reads the metadata of one walk (coalesced), then the group's nodes are copied ITEM-parallel:
// the kept walks of a group are contiguous in the pool, so flat node index q of the group maps to
// pool position G + q, and its (walk, position) comes from a 5-step shuffle search over the group's
// node-count prefix. Every lane moves one item per step whatever the walk lengths are and the
// stores of a step are 32 consecutive words. nodes / edges may be null (array not kept).
constexpr int kU = 4;  // item steps in flight per lane (2: 3.03 ms per 390 M items at the Twitter shape)
__global__ void __launch_bounds__(256) compact_pairs(
    uint64_t nwalks, const uint32_t* __restrict__ vflag, const uint32_t* __restrict__ vidx,
    const uint64_t* __restrict__ voff, const uint2* const* __restrict__ enc_src,
    const uint32_t* __restrict__ enc_len, const uint64_t* __restrict__ enc_batch,
    const uint32_t* __restrict__ enc_seq, uint64_t base_walk, uint64_t base_edge,
    uint64_t* __restrict__ edge_off, uint32_t* __restrict__ nodes, uint32_t* __restrict__ edges,
    uint64_t* __restrict__ tag_batch, uint32_t* __restrict__ tag_seq) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t groups = (nwalks + 31) / 32;
    for (uint64_t grp = warp; grp < groups; grp += nwarps) {
        const uint64_t w = grp * 32 + lane;
        const bool valid = w < nwalks && vflag[w];
        uint32_t len = 0;
        const uint2* src = nullptr;
        uint64_t dw = 0, de = 0;
        if (valid) {
            len = enc_len[w];
            src = enc_src[w];
            dw = base_walk + vidx[w];
            de = base_edge + voff[w];
            edge_off[dw] = de;
            tag_batch[dw] = enc_batch[w];
            tag_seq[dw] = enc_seq[w];
        }
        const unsigned vmask = __ballot_sync(kFullMask, valid);
        if (!vmask) continue;
        const uint32_t cnt = valid ? len + 1 : 0;
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(kFullMask, incl, d);
            if (lane >= (uint32_t)d) incl += t;
        }
        const uint32_t start = incl - cnt;  // first flat node index of this lane's walk
        const uint32_t total = __shfl_sync(kFullMask, incl, 31);
        const int first = __ffs(vmask) - 1;
        const uint64_t G = __shfl_sync(kFullMask, (unsigned long long)(de + dw), first);   // pool node position of q = 0
        const uint64_t dw0 = __shfl_sync(kFullMask, (unsigned long long)dw, first);
        for (uint32_t q0 = 0; q0 < total; q0 += 32 * kU) {
            uint2 pr[kU];
            uint32_t ii[kU], jj[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                uint32_t j = 0;  // largest lane whose walk starts at or before q
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const uint32_t s_at = __shfl_sync(kFullMask, start, (j + step) & 31);
                    if (s_at <= q) j += step;
                }
                const uint32_t sj = __shfl_sync(kFullMask, start, j);
                const uint2* sp = reinterpret_cast<const uint2*>(
                    __shfl_sync(kFullMask, (unsigned long long)src, j));
                ii[u] = q - sj;
                jj[u] = j;
                if (q < total) pr[u] = __ldcs(sp + ii[u]);  // the log is read exactly once
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                if (q >= total) continue;
                if (nodes) nodes[G + q] = pr[u].x;
                if (edges && ii[u]) {
                    // walk j is the (rank of j among the kept lanes)-th kept walk of the group
                    const uint64_t dwj = dw0 + __popc(vmask & ((1u << jj[u]) - 1u));
                    edges[G + q - dwj - 1] = pr[u].y;
                }
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        edge_off[base_walk + vidx[nwalks]] = base_edge + voff[nwalks];
}

// accepted_after_batch (sampler.cpp:459) for the batches of this chunk.
// `first` is indexed by launch item: batches, or single attempts in the Philox mode, where a batch
// is `stride` consecutive items.
__global__ void batch_cumulative(uint64_t nbatches, const uint32_t* __restrict__ first,
                                 const uint32_t* __restrict__ vidx, uint64_t base_walk,
                                 uint64_t* __restrict__ out, uint32_t stride) {
    uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbatches) return;
    out[b] = base_walk + vidx[first[(b + 1) * stride]];
}

// Philox mode: the launch items were single attempts; turn (global attempt index, 0) into the
// stream's (batch, seq) tags: batch = attempt / l, seq = rank among the batch's accepted attempts.
__global__ void philox_tags(uint64_t nwalks, uint32_t l, uint64_t first_attempt, uint64_t first_batch,
                            const uint32_t* __restrict__ first, uint64_t* __restrict__ enc_batch,
                            uint32_t* __restrict__ enc_seq) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nwalks) return;
    const uint64_t item = enc_batch[i] - first_attempt;  // launch item of this walk
    const uint64_t b = item / l;
    enc_seq[i] = first[item] - first[b * l];
    enc_batch[i] = first_batch + b;
}

// first index with a[i] >= key, or n
__global__ void lower_bound_u64(const uint64_t* __restrict__ a, uint64_t n, uint64_t key,
                                uint64_t* __restrict__ out) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] >= key)
            hi = mid;
        else
            lo = mid + 1;
    }
    out[0] = lo;
    out[1] = lo < n ? a[lo] : 0;
}

inline int blocks_for(uint64_t items, int threads) {
    uint64_t b = (items + threads - 1) / threads;
    return (int)(b ? b : 1);
}

uint64_t read_u64(hsaw_gpu_ctx* ctx, const uint64_t* d) {
    HSAW_CUDA_CHECK(
        cudaMemcpyAsync(ctx->h_scalars, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return ctx->h_scalars[0];
}
uint32_t read_u32(hsaw_gpu_ctx* ctx, const uint32_t* d) {
    HSAW_CUDA_CHECK(
        cudaMemcpyAsync(ctx->h_scalars, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return *reinterpret_cast<uint32_t*>(ctx->h_scalars);
}

// Samples global batches [first_batch, first_batch + nb) (nb <= kMaxChunkBatches) and appends.
void sample_chunk(hsaw_gpu_stream* s, uint64_t first_batch, uint64_t nb) {
    hsaw_gpu_ctx* ctx = s->ctx;
    cudaStream_t st = ctx->stream;
    const uint32_t l = s->cfg.batch_size;
    const uint64_t slots = nb * l;
    if (slots > 0xFFFFFFF0ull) fail(HSAW_EINVAL, "stream: chunk too large for 32-bit walk ids");
    SamplerScratch& x = ctx->samp;  // chunk scratch is shared by all streams of the context

    // a restricted stream (partitioned sampling) hands its start domain / allowed mask to the
    // sampler launches of this chunk through the context
    struct RestrictGuard {
        hsaw_gpu_ctx* c;
        ~RestrictGuard() { c->restr = Restriction{}; }
    } guard{ctx};
    if (s->r_ndomain) {
        s->r_cross.ensure_scratch(nb);
        ctx->restr = Restriction{s->r_domain.p, s->r_ndomain, s->r_allowed.p, s->r_cross.p};
    }

    // ---- K1
    x.slot_seed.ensure_scratch(slots + 1);
    x.slot_len.ensure_scratch(slots + 1);
    x.count.ensure_scratch(nb + 1);
    x.first.ensure_scratch(nb + 1);
    HSAW_CUDA_CHECK(cudaMemsetAsync(x.count.p + nb, 0, 4, st));
    launch_encode(ctx, s->cfg, s->seed + first_batch, nb, x.slot_seed.p, x.slot_len.p,
                  x.count.p, s->stats.p, s->stats.p + 8, nullptr, s->collect_stats);
    if (s->r_ndomain) {  // crossings per batch -> cumulative, like crossed_after (partition.cpp:239-243)
        std::vector<uint32_t> cross(nb);
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(cross.data(), s->r_cross.p, nb * 4, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        uint64_t run = s->crossed_after_batch.empty() ? 0 : s->crossed_after_batch.back();
        for (uint64_t b = 0; b < nb; ++b) s->crossed_after_batch.push_back(run += cross[b]);
    }
    exclusive_sum_u32(ctx, x.count.p, x.first.p, nb + 1);
    const uint64_t E = read_u32(ctx, x.first.p + nb);  // encoded (heuristically accepted) walks

    uint64_t A = 0, VT = 0;
    x.vidx.ensure_scratch(E + 1);
    if (E > 0) {
        // ---- dense (batch, seq) order
        x.enc_seed.ensure_scratch(E);
        x.enc_len.ensure_scratch(E + 1);
        x.enc_batch.ensure_scratch(E);
        x.enc_seq.ensure_scratch(E);
        x.tmp_off.ensure_scratch(E + 1);
        {
            StageScope timer(ctx, HSAW_STAGE_COMPACT);
            gather_encoded<<<blocks_for(slots, 256), 256, 0, st>>>(
                nb, l, first_batch, x.count.p, x.first.p, x.slot_seed.p, x.slot_len.p,
                x.enc_seed.p, x.enc_len.p, x.enc_batch.p, x.enc_seq.p);
            check_launch(ctx, "gather_encoded");
            HSAW_CUDA_CHECK(cudaMemsetAsync(x.enc_len.p + E, 0, 4, st));
            exclusive_sum_u32_to_u64(ctx, x.enc_len.p, x.tmp_off.p, E + 1);
        }
        const uint64_t T = read_u64(ctx, x.tmp_off.p + E);  // edges of all encoded walks

        // ---- K2 + K2b
        x.tmp_nodes.ensure_scratch(T + E);
        x.tmp_edges.ensure_scratch(T + 1);
        x.status.ensure_scratch(E);
        launch_decode(ctx, E, x.enc_seed.p, x.enc_len.p, x.tmp_off.p, x.tmp_nodes.p,
                      x.tmp_edges.p, x.status.p, s->stats.p, s->stats.p + 8);
        s->dropped += launch_distinct_check(ctx, E, x.tmp_off.p, x.tmp_nodes.p, x.status.p);

        // ---- compaction offsets. The slot arrays are dead after the gather and hold
        // slots + 1 >= E + 1 entries, so they double as the valid-flag / valid-length scan inputs.
        uint32_t* vflag = x.slot_len.p;
        uint32_t* vlen = reinterpret_cast<uint32_t*>(x.slot_seed.p);
        x.voff.ensure_scratch(E + 1);
        uint32_t* mismatch = reinterpret_cast<uint32_t*>(s->stats.p + 9);
        HSAW_CUDA_CHECK(cudaMemsetAsync(mismatch, 0, 4, st));
        {
            StageScope timer(ctx, HSAW_STAGE_COMPACT);
            mark_valid<<<blocks_for(E + 1, 256), 256, 0, st>>>(E, x.status.p, x.enc_len.p, vflag,
                                                               vlen, mismatch);
            check_launch(ctx, "mark_valid");
            exclusive_sum_u32(ctx, vflag, x.vidx.p, E + 1);
            exclusive_sum_u32_to_u64(ctx, vlen, x.voff.p, E + 1);
        }
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(ctx->h_scalars + 1, x.voff.p + E, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(ctx->h_scalars + 2, mismatch, 4, cudaMemcpyDeviceToHost, st));
        A = read_u32(ctx, x.vidx.p + E);
        VT = ctx->h_scalars[1];
        if (*reinterpret_cast<uint32_t*>(ctx->h_scalars + 2) != 0)
            fail(HSAW_EDATA, "decode: replay disagreed with generation (internal error)");

        // ---- append to the pool
        s->edge_off.reserve(s->accepted + A + 1, st);
        if (s->keep_nodes) s->nodes.reserve(s->total_edges + VT + s->accepted + A, st);
        if (s->keep_edges) s->edges.reserve(s->total_edges + VT + 1, st);
        s->tag_batch.reserve(s->accepted + A + 1, st);
        s->tag_seq.reserve(s->accepted + A + 1, st);
        // one warp per group of 32 encoded walks, 8 warps per block
        int cblocks = (int)std::min<uint64_t>((E + 255) / 256, (uint64_t)ctx->sm_count * 16);
        {
            StageScope timer(ctx, HSAW_STAGE_COMPACT);
            compact_walks<<<cblocks, 256, 0, st>>>(
                E, vflag, x.vidx.p, x.voff.p, x.tmp_off.p, x.tmp_nodes.p, x.tmp_edges.p,
                x.enc_len.p, x.enc_batch.p, x.enc_seq.p, s->accepted, s->total_edges,
                s->edge_off.p, s->keep_nodes ? s->nodes.p : nullptr,
                s->keep_edges ? s->edges.p : nullptr, s->tag_batch.p, s->tag_seq.p);
            check_launch(ctx, "compact_walks");
        }
    } else {
        HSAW_CUDA_CHECK(cudaMemsetAsync(x.vidx.p, 0, 4, st));
        s->edge_off.reserve(s->accepted + 1, st);
        uint64_t te = s->total_edges;
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(s->edge_off.p + s->accepted, &te, 8, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    }

    // ---- per-batch cumulative counts
    s->accepted_after_batch.size = s->local_batches;
    s->accepted_after_batch.reserve(s->local_batches + nb, st);
    if (E > 0) {
        batch_cumulative<<<blocks_for(nb, 256), 256, 0, st>>>(
            nb, x.first.p, x.vidx.p, s->accepted, s->accepted_after_batch.p + s->local_batches, 1);
        check_launch(ctx, "batch_cumulative");
    } else {
        std::vector<uint64_t> flat(nb, s->accepted);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(s->accepted_after_batch.p + s->local_batches, flat.data(),
                                        nb * 8, cudaMemcpyHostToDevice, st));
    }
    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    collect_timings(ctx);

    s->accepted += A;
    s->total_edges += VT;
    s->local_batches += nb;
    s->edge_off.size = s->accepted + 1;
    s->nodes.size = s->keep_nodes ? s->total_edges + s->accepted : 0;
    s->edges.size = s->keep_edges ? s->total_edges : 0;
    s->tag_batch.size = s->accepted;
    s->tag_seq.size = s->accepted;
    s->accepted_after_batch.size = s->local_batches;
}

// Fused variant of sample_chunk: K1 records the walks while generating them, so the replay kernel
// only runs for walks that outgrew their log chunk. Same outputs, same order.
// The chunk is handled in two halves so that sample_range can pipeline: fused_launch_k1 queues K1
// (its outputs live in one of two scratch sets), fused_finish does everything after it. K1 of
// chunk i + 1 is queued on the context's second stream BEFORE chunk i is finished, so it runs
// beside K2b / the compaction of chunk i.
struct FusedLaunch {
    uint64_t first_batch = 0, nb = 0, ni = 0, slots = 0;
    uint32_t l = 0, ml = 0;
    bool philox = false;
    int buf = 0;         // scratch set holding K1's outputs (0: ctx->samp, 1: ctx->samp2)
    bool ahead = false;  // K1 was queued on ctx->ahead[buf]; ahead_done[buf] marks its end
};

static void ensure_ahead_stream(hsaw_gpu_ctx* ctx) {
    if (ctx->ahead[0]) return;
    for (auto& a : ctx->ahead) HSAW_CUDA_CHECK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    HSAW_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ahead_go, cudaEventDisableTiming));
    for (auto& e : ctx->ahead_done)
        HSAW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

FusedLaunch fused_launch_k1(hsaw_gpu_stream* s, uint64_t first_batch, uint64_t nb, int buf,
                            bool ahead) {
    hsaw_gpu_ctx* ctx = s->ctx;
    const uint32_t l = s->cfg.batch_size;
    const uint64_t slots = nb * l;
    if (slots > 0xFFFFFFF0ull) fail(HSAW_EINVAL, "stream: chunk too large for 32-bit walk ids");
    SamplerScratch& k = buf ? ctx->samp2 : ctx->samp;
    // Philox per-walk mode: the launch items are single attempts (ni items of ml = 1 attempt);
    // a batch is l consecutive items. Reference mode: items are batches.
    FusedLaunch fl;
    fl.first_batch = first_batch;
    fl.nb = nb;
    fl.l = l;
    fl.slots = slots;
    fl.philox = s->cfg.rng_mode == 1;
    fl.ni = fl.philox ? slots : nb;
    fl.ml = fl.philox ? 1u : l;
    fl.buf = buf;
    fl.ahead = ahead;
    const uint64_t ni = fl.ni;
    hsaw_sampler_cfg kcfg = s->cfg;
    kcfg.batch_size = fl.ml;
    const uint64_t first_item = fl.philox ? (s->seed + first_batch) * l : s->seed + first_batch;
    struct RngGuard {
        hsaw_gpu_ctx* c;
        ~RngGuard() {
            c->rng_mode = 0;
            c->k1_stream = nullptr;
        }
    } rng_guard{ctx};
    ctx->rng_mode = s->cfg.rng_mode;

    // ---- arena sizing: one open chunk per resident lane + the expected volume of accepted walks
    // (observed pairs per attempt so far, with slack). Too small is safe: overflow -> replay.
    const uint64_t chunk = record_chunk_pairs();
    const uint64_t lanes = std::min<uint64_t>(record_resident_lanes(ctx), nb);
    double per_attempt = s->pairs_per_attempt > 0 ? s->pairs_per_attempt : 24.0;
    uint64_t want = lanes * chunk + (uint64_t)((double)slots * per_attempt * 1.5) + 64 * chunk;
    want = std::min<uint64_t>(want, 0xFFFF0000ull);
    k.arena.ensure_scratch(want);
    uint32_t arena_cap = (uint32_t)std::min<uint64_t>(k.arena.cap, 0xFFFF0000ull);
    // test hook: a deliberately tiny arena exercises the "arena exhausted -> replay" path
    if (const char* env = std::getenv("HSAW_ARENA_MAX_PAIRS")) {
        uint64_t cap = std::strtoull(env, nullptr, 10);
        if (cap >= chunk && cap < arena_cap) arena_cap = (uint32_t)cap;
    }

    // ---- K1 (recording)
    k.slot_seed.ensure_scratch(slots + 1);
    k.slot_len.ensure_scratch(slots + 1);
    k.slot_log.ensure_scratch(slots + 1);
    k.count.ensure_scratch(ni + 1);
    k.first.ensure_scratch(ni + 1);
    k.k1_words.ensure_scratch(4);
    cudaStream_t st = ctx->stream;
    if (ahead) {
        // the buffers above were (re)allocated in the context stream's order: the second stream
        // starts behind that point (the context stream is idle here: the previous chunk's
        // finish ended with a synchronisation)
        ensure_ahead_stream(ctx);
        HSAW_CUDA_CHECK(cudaEventRecord(ctx->ahead_go, ctx->stream));
        st = ctx->ahead[buf];
        HSAW_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ahead_go, 0));
        ctx->k1_stream = st;
    }
    HSAW_CUDA_CHECK(cudaMemsetAsync(k.count.p + ni, 0, 4, st));
    uint32_t* arena_cursor = reinterpret_cast<uint32_t*>(k.k1_words.p + 1);
    EncodeRecord rec{k.arena.p, arena_cap, arena_cursor, k.slot_log.p};
    launch_encode(ctx, kcfg, first_item, ni, k.slot_seed.p, k.slot_len.p, k.count.p,
                  s->stats.p, k.k1_words.p, &rec, s->collect_stats);
    if (ahead) HSAW_CUDA_CHECK(cudaEventRecord(ctx->ahead_done[buf], st));
    return fl;
}

void fused_finish(hsaw_gpu_stream* s, const FusedLaunch& fl) {
    hsaw_gpu_ctx* ctx = s->ctx;
    cudaStream_t st = ctx->stream;
    const uint32_t l = fl.l, ml = fl.ml;
    const uint64_t slots = fl.slots, ni = fl.ni, nb = fl.nb, first_batch = fl.first_batch;
    const bool philox = fl.philox;
    SamplerScratch& x = ctx->samp;                       // post-processing scratch (one set)
    SamplerScratch& k = fl.buf ? ctx->samp2 : ctx->samp;  // K1's outputs
    struct RngGuard {
        hsaw_gpu_ctx* c;
        ~RngGuard() { c->rng_mode = 0; }
    } rng_guard{ctx};
    ctx->rng_mode = s->cfg.rng_mode;
    if (fl.ahead) HSAW_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ahead_done[fl.buf], 0));
    uint32_t* arena_cursor = reinterpret_cast<uint32_t*>(k.k1_words.p + 1);
    exclusive_sum_u32(ctx, k.count.p, k.first.p, ni + 1);
    HSAW_CUDA_CHECK(
        cudaMemcpyAsync(ctx->h_scalars + 1, arena_cursor, 4, cudaMemcpyDeviceToHost, st));
    const uint64_t E = read_u32(ctx, k.first.p + ni);
    const uint64_t arena_used = *reinterpret_cast<uint32_t*>(ctx->h_scalars + 1);
    (void)arena_used;

    uint64_t A = 0, VT = 0;
    x.vidx.ensure_scratch(E + 1);
    if (E > 0) {
        x.enc_seed.ensure_scratch(E);
        x.enc_len.ensure_scratch(E + 1);
        x.enc_batch.ensure_scratch(E);
        x.enc_seq.ensure_scratch(E);
        x.enc_src.ensure_scratch(E);
        x.ovf_pairs.ensure_scratch(E + 1);
        x.tmp_off.ensure_scratch(E + 1);
        x.status.ensure_scratch(E);
        uint32_t* nsel = reinterpret_cast<uint32_t*>(s->stats.p + 11);
        {
            StageScope timer(ctx, HSAW_STAGE_COMPACT);
            gather_recorded<<<blocks_for(slots, 256), 256, 0, st>>>(
                ni, ml, philox ? first_batch * l : first_batch, k.count.p, k.first.p, k.slot_seed.p,
                k.slot_len.p, k.slot_log.p, k.arena.p, record_overflow_marker(), x.enc_seed.p,
                x.enc_len.p, x.enc_batch.p, x.enc_seq.p,
                reinterpret_cast<const uint2**>(x.enc_src.p), x.ovf_pairs.p);
            check_launch(ctx, "gather_recorded");
            if (philox) {
                philox_tags<<<blocks_for(E, 256), 256, 0, st>>>(E, l, first_batch * l, first_batch,
                                                               k.first.p, x.enc_batch.p, x.enc_seq.p);
                check_launch(ctx, "philox_tags");
            }
            HSAW_CUDA_CHECK(cudaMemsetAsync(x.ovf_pairs.p + E, 0, 4, st));
            HSAW_CUDA_CHECK(cudaMemsetAsync(nsel, 0, 4, st));
            HSAW_CUDA_CHECK(cudaMemsetAsync(nsel + 1, 0xFF, 4, st));
            exclusive_sum_u32_to_u64(ctx, x.ovf_pairs.p, x.tmp_off.p, E + 1);
            // recorded walks are complete by construction
            HSAW_CUDA_CHECK(cudaMemsetAsync(x.status.p, 1, E, st));
        }
        const uint64_t OV = read_u64(ctx, x.tmp_off.p + E);  // pairs to replay (usually 0)
        if (OV > 0) {
            x.replay.ensure_scratch(OV);
            x.sel.ensure_scratch(E);
            place_overflow<<<blocks_for(E, 256), 256, 0, st>>>(
                E, x.ovf_pairs.p, x.tmp_off.p, x.replay.p,
                reinterpret_cast<const uint2**>(x.enc_src.p), x.sel.p, nsel, x.enc_len.p);
            check_launch(ctx, "place_overflow");
            const uint64_t both = read_u64(ctx, s->stats.p + 11);
            const uint64_t nreplay = (uint32_t)both;
            const uint32_t shortest = (uint32_t)(both >> 32);
            // The replay is a handful of single lanes chasing thousands of dependent steps each
            // (1.3 ms per chunk at the Twitter shape with the GPU idle). Walks that outgrew a log
            // chunk (> 1024 pairs) are beyond what K2b's main pass reads (it only queues them for
            // the mid / long passes), so the replay runs on a side stream beside that pass and
            // is joined right after it. Replays of SHORT walks (arena exhaustion) keep the
            // serial order.
            const bool overlap = distinct_check_defers_walks_longer_than() <= shortest;
            launch_decode_pairs(ctx, nreplay, x.sel.p, x.enc_seed.p, x.enc_len.p,
                                reinterpret_cast<uint2* const*>(x.enc_src.p), x.status.p,
                                s->stats.p, s->stats.p + 8, overlap);
            s->replayed += nreplay;
        }
        // ---- K2b on the pair logs
        s->dropped += launch_distinct_check_pairs(
            ctx, E, reinterpret_cast<const uint2* const*>(x.enc_src.p), x.enc_len.p, x.status.p);

        uint32_t* vflag = k.slot_len.p;  // slot arrays are dead after the gather (>= E + 1 entries)
        uint32_t* vlen = reinterpret_cast<uint32_t*>(k.slot_seed.p);
        x.voff.ensure_scratch(E + 1);
        uint32_t* mismatch = reinterpret_cast<uint32_t*>(s->stats.p + 9);
        HSAW_CUDA_CHECK(cudaMemsetAsync(mismatch, 0, 4, st));
        {
            StageScope timer(ctx, HSAW_STAGE_COMPACT);
            mark_valid<<<blocks_for(E + 1, 256), 256, 0, st>>>(E, x.status.p, x.enc_len.p, vflag,
                                                               vlen, mismatch);
            check_launch(ctx, "mark_valid");
            exclusive_sum_u32(ctx, vflag, x.vidx.p, E + 1);
            exclusive_sum_u32_to_u64(ctx, vlen, x.voff.p, E + 1);
        }
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(ctx->h_scalars + 1, x.voff.p + E, 8, cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(ctx->h_scalars + 2, mismatch, 4, cudaMemcpyDeviceToHost, st));
        A = read_u32(ctx, x.vidx.p + E);
        VT = ctx->h_scalars[1];
        if (*reinterpret_cast<uint32_t*>(ctx->h_scalars + 2) != 0)
            fail(HSAW_EDATA, "decode: replay disagreed with generation (internal error)");

        s->edge_off.reserve(s->accepted + A + 1, st);
        if (s->keep_nodes) s->nodes.reserve(s->total_edges + VT + s->accepted + A, st);
        if (s->keep_edges) s->edges.reserve(s->total_edges + VT + 1, st);
        s->tag_batch.reserve(s->accepted + A + 1, st);
        s->tag_seq.reserve(s->accepted + A + 1, st);
        // one warp per group of 32 encoded walks, 8 warps per block
        int cblocks = (int)std::min<uint64_t>((E + 255) / 256, (uint64_t)ctx->sm_count * 16);
        {
            StageScope timer(ctx, HSAW_STAGE_COMPACT);
            compact_pairs<<<cblocks, 256, 0, st>>>(
                E, vflag, x.vidx.p, x.voff.p, reinterpret_cast<const uint2* const*>(x.enc_src.p),
                x.enc_len.p, x.enc_batch.p, x.enc_seq.p, s->accepted, s->total_edges,
                s->edge_off.p, s->keep_nodes ? s->nodes.p : nullptr,
                s->keep_edges ? s->edges.p : nullptr, s->tag_batch.p, s->tag_seq.p);
            check_launch(ctx, "compact_pairs");
        }
    } else {
        HSAW_CUDA_CHECK(cudaMemsetAsync(x.vidx.p, 0, 4, st));
        s->edge_off.reserve(s->accepted + 1, st);
        uint64_t te = s->total_edges;
        HSAW_CUDA_CHECK(
            cudaMemcpyAsync(s->edge_off.p + s->accepted, &te, 8, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    }

    s->accepted_after_batch.size = s->local_batches;
    s->accepted_after_batch.reserve(s->local_batches + nb, st);
    if (E > 0) {
        batch_cumulative<<<blocks_for(nb, 256), 256, 0, st>>>(
            nb, k.first.p, x.vidx.p, s->accepted, s->accepted_after_batch.p + s->local_batches,
            philox ? l : 1u);  // launch items per batch
        check_launch(ctx, "batch_cumulative");
    } else {
        std::vector<uint64_t> flat(nb, s->accepted);
        HSAW_CUDA_CHECK(cudaMemcpyAsync(s->accepted_after_batch.p + s->local_batches, flat.data(),
                                        nb * 8, cudaMemcpyHostToDevice, st));
    }
    HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
    collect_timings(ctx);

    // Running estimate for the next chunk's arena: pairs that stay in the log are those of the
    // kept walks (plus the ones the recheck dropped and line padding, hence the slack). The arena
    // cursor itself is no measure: it advances a whole chunk per lane however little is logged.
    const double seen = 1.25 * (double)(VT + A + 8 * A) / (double)slots;
    s->pairs_per_attempt = s->pairs_per_attempt > 0 ? 0.5 * (s->pairs_per_attempt + seen) : seen;

    s->accepted += A;
    s->total_edges += VT;
    s->local_batches += nb;
    s->edge_off.size = s->accepted + 1;
    s->nodes.size = s->keep_nodes ? s->total_edges + s->accepted : 0;
    s->edges.size = s->keep_edges ? s->total_edges : 0;
    s->tag_batch.size = s->accepted;
    s->tag_seq.size = s->accepted;
    s->accepted_after_batch.size = s->local_batches;
}

void sample_chunk_fused(hsaw_gpu_stream* s, uint64_t first_batch, uint64_t nb) {
    fused_finish(s, fused_launch_k1(s, first_batch, nb, 0, false));
}

bool ctx_has_window(const hsaw_gpu_ctx* ctx) { return ctx->k1_window_on; }

bool fused_enabled() {
    static const bool on = [] {
        const char* env = std::getenv("HSAW_FUSED");
        return env ? std::atoi(env) != 0 : true;
    }();
    return on;
}

// Pipelined sampling (default; HSAW_PIPELINE=0 keeps the serial chunks): when a call spans more
// than one chunk, K1 of chunk i + 1 is queued on one of the context's two extra streams before
// chunk i is finished, so the tail of a K1 launch (its last lanes chase the longest walks for a
// millisecond or more while the SMs drain), K2b, the scans and the compaction of a chunk run
// beside the next chunk's walk generation. Measured at the Twitter shape (47 chunks of ~1.1 M
// batches per eSIA solve): sampling 1.114 -> 1.057 s. Cutting a call into SMALLER chunks to
// pipeline more (HSAW_PIPE_BATCHES, 0 = off; the tests use it) loses: a launch of 2^18 batches
// gives each lane two or three batches, most of the launch is tail, and K2b squeezed into the
// registers K1 leaves runs 5x slower (2^20 batches as 4 x 2^18: 24.3 ms against 22.9 serial).
// Results and their order do not change: chunks are finished strictly in batch order.
static uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* env = std::getenv(name);
    return env && *env ? std::strtoull(env, nullptr, 10) : dflt;
}

void sample_range(hsaw_gpu_stream* s, uint64_t first_batch, uint64_t nbatches) {
    if (first_batch < s->last_batch_end)
        fail(HSAW_EINVAL, "stream: batch ranges must be issued in increasing order");
    hsaw_gpu_ctx* ctx = s->ctx;
    if (s->cfg.rng_mode == 1 && s->r_ndomain != 0)
        fail(HSAW_EINVAL, "stream: the Philox mode does not combine with a restriction");
    const bool fused =
        (fused_enabled() || s->cfg.rng_mode == 1) && record_supported(s->cfg) && s->r_ndomain == 0;
    const uint64_t pipe_batches = env_u64("HSAW_PIPE_BATCHES", 0);
    auto chunk_batches = [&](uint64_t done) {
        uint64_t nb = std::min(nbatches - done, kMaxChunkBatches);
        // a chunk's slots carry 32-bit walk ids, and its pair-log arena (about 1.5x the expected
        // log volume) is kept to a few gigabytes: long walks (Twitter shape: 130 pairs per accepted
        // walk) get smaller chunks instead of a 25 GB arena
        const uint64_t bs = std::max<uint64_t>(s->cfg.batch_size, 1);
        nb = std::min(nb, std::max<uint64_t>(0xFFFFFFF0ull / bs, 1));
        const double per_attempt = s->pairs_per_attempt > 0 ? s->pairs_per_attempt : 24.0;
        const uint64_t arena_batches = (uint64_t)((double)(kArenaTargetBytes / 8) / (per_attempt * 1.5 * (double)bs));
        nb = std::min(nb, std::max<uint64_t>(arena_batches, 1ull << 14));
        if (pipe_batches > 0) nb = std::min(nb, pipe_batches);
        return nb;
    };
    const bool pipelined =
        fused && env_u64("HSAW_PIPELINE", 1) != 0 && chunk_batches(0) < nbatches;
    if (pipelined) {
        try {
            int buf = 0;
            uint64_t issued = chunk_batches(0);
            FusedLaunch cur = fused_launch_k1(s, first_batch, issued, buf, true);
            for (;;) {
                const bool more = issued < nbatches;
                FusedLaunch next;
                if (more) {
                    const uint64_t nb = chunk_batches(issued);
                    next = fused_launch_k1(s, first_batch + issued, nb, buf ^ 1, true);
                    issued += nb;
                }
                fused_finish(s, cur);
                s->last_batch_end = cur.first_batch + cur.nb;
                if (!more) break;
                cur = next;
                buf ^= 1;
            }
        } catch (...) {
            for (cudaStream_t a : ctx->ahead)  // a chunk sampled ahead may be in flight
                if (a) cudaStreamSynchronize(a);
            throw;
        }
    } else {
        uint64_t done = 0;
        while (done < nbatches) {
            const uint64_t nb = chunk_batches(done);
            if (fused)
                sample_chunk_fused(s, first_batch + done, nb);
            else
                sample_chunk(s, first_batch + done, nb);
            done += nb;
            s->last_batch_end = first_batch + done;
        }
    }
    s->last_batch_end = first_batch + nbatches;
    // sampling is over for this call: the graph lines K1 kept persisting go back to normal, the
    // greedy / coverage kernels that follow want the whole L2 for their counters
    if (ctx_has_window(s->ctx)) cudaCtxResetPersistingL2Cache();
}

void local_cut(const hsaw_gpu_stream* s, uint64_t min_count, uint64_t* idx, uint64_t* value) {
    hsaw_gpu_ctx* ctx = s->ctx;
    uint64_t* d_out = ctx->d_scalars;
    lower_bound_u64<<<1, 1, 0, ctx->stream>>>(s->accepted_after_batch.p, s->local_batches,
                                              min_count, d_out);
    check_launch(ctx, "lower_bound_u64");
    HSAW_CUDA_CHECK(
        cudaMemcpyAsync(ctx->h_scalars, d_out, 16, cudaMemcpyDeviceToHost, ctx->stream));
    HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    *idx = ctx->h_scalars[0];
    *value = ctx->h_scalars[1];
}

}  // namespace

extern "C" {

int hsaw_gpu_stream_create(hsaw_gpu_ctx* ctx, uint64_t seed, const hsaw_sampler_cfg* cfg,
                           hsaw_gpu_stream** out) {
    if (!ctx || !out) return HSAW_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&] {
        if (!cfg) fail(HSAW_EINVAL, "stream_create: null config");
        if (!ctx->g.nodes) fail(HSAW_EINVAL, "stream_create: no graph uploaded");
        validate_cfg(*cfg);
        auto* s = new hsaw_gpu_stream;
        static std::atomic<uint64_t> next_uid{1};
        s->uid = next_uid.fetch_add(1);
        s->ctx = ctx;
        s->seed = seed;
        s->cfg = *cfg;
        if (const char* env = std::getenv("HSAW_STATS")) s->collect_stats = std::atoi(env) != 0;
        try {
            s->stats.ensure_scratch(16);
            HSAW_CUDA_CHECK(cudaMemsetAsync(s->stats.p, 0, 16 * 8, ctx->stream));
            // recycle the walk-pool buffers of the previous stream on this context, if any
            PoolCache& pc = ctx->pool_cache;
            s->edge_off.swap(pc.edge_off);
            s->nodes.swap(pc.nodes);
            s->edges.swap(pc.edges);
            s->tag_batch.swap(pc.tag_batch);
            s->tag_seq.swap(pc.tag_seq);
            s->accepted_after_batch.swap(pc.accepted_after_batch);
            s->edge_off.size = s->nodes.size = s->edges.size = 0;
            s->tag_batch.size = s->tag_seq.size = s->accepted_after_batch.size = 0;
            s->edge_off.reserve(1024, ctx->stream);
            HSAW_CUDA_CHECK(cudaMemsetAsync(s->edge_off.p, 0, 8, ctx->stream));
            s->edge_off.size = 1;
            HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

void hsaw_gpu_stream_destroy(hsaw_gpu_stream* s) {
    if (!s) return;
    cudaSetDevice(s->ctx->device);
    current_stream() = s->ctx->stream;
    // hand the walk-pool buffers to the context for the next stream (keep the larger set)
    PoolCache& pc = s->ctx->pool_cache;
    if (s->nodes.cap + s->edges.cap >= pc.nodes.cap + pc.edges.cap) {
        pc.edge_off.swap(s->edge_off);
        pc.nodes.swap(s->nodes);
        pc.edges.swap(s->edges);
        pc.tag_batch.swap(s->tag_batch);
        pc.tag_seq.swap(s->tag_seq);
        pc.accepted_after_batch.swap(s->accepted_after_batch);
    }
    delete s;  // whatever is left goes back to the device pool in stream order
}

int hsaw_gpu_stream_ensure(hsaw_gpu_stream* s, uint64_t min_accepted) {
    if (!s) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        const uint64_t bs = s->cfg.batch_size;
        while (s->accepted < min_accepted) {
            // budget rule of sampler.cpp:396-404: floor(max_attempts / batch_size) batches overall
            uint64_t attempts_so_far = s->next_batch * bs;
            uint64_t budget_left =
                s->cfg.max_attempts > attempts_so_far ? s->cfg.max_attempts - attempts_so_far : 0;
            uint64_t max_batches = budget_left / bs;
            if (max_batches == 0)
                fail(HSAW_EBUDGET,
                     "attempt budget exhausted while sampling walks; suspects may be unreachable");
            // round size: only a speed knob (sampler.cpp:406-421) — pools are cut at whole-batch
            // prefixes by accepted count, so over-materialising never changes a result
            // A round of up to ~2^17 batches costs the same few hundred microseconds (one
            // resident wave of K1 plus the fixed host round trips), so when sampling is needed at
            // all, aim for at least kFloor walks: the early, small iterations of the doubling
            // loop then find their samples already there.
            constexpr uint64_t kFloor = 1ull << 18;
            uint64_t need = std::max(min_accepted, kFloor) - s->accepted;
            uint64_t batches;
            if (s->accepted == 0) {
                batches = s->grow;
                s->grow = std::min<uint64_t>(s->grow * 8, 1ull << 22);
            } else {
                // expected batches for the remainder plus ~4 sigma of the accepted count (a
                // shortfall only costs one more small round; the reference's 1.1 factor would
                // over-sample every call by 10 %)
                double rate = (double)s->accepted / (double)attempts_so_far;
                double est = (double)need / (rate * (double)bs);
                double sigma = std::sqrt((double)need / rate) / (double)bs;
                batches = (uint64_t)(est * 1.005 + 4.0 * sigma) + 16;
            }
            batches = std::max<uint64_t>(std::min(batches, max_batches), 1);
            sample_range(s, s->next_batch, batches);
            s->next_batch += batches;
        }
    });
}

int hsaw_gpu_stream_sample_range(hsaw_gpu_stream* s, uint64_t first_batch, uint64_t nbatches,
                                 uint64_t* accepted_in_range) {
    if (!s) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        uint64_t before = s->accepted;
        sample_range(s, first_batch, nbatches);
        if (first_batch + nbatches > s->next_batch) s->next_batch = first_batch + nbatches;
        if (accepted_in_range) *accepted_in_range = s->accepted - before;
    });
}

int hsaw_gpu_stream_size(const hsaw_gpu_stream* s, uint64_t* accepted, uint64_t* batches,
                         uint64_t* total_edges) {
    if (!s) return HSAW_EINVAL;
    if (accepted) *accepted = s->accepted;
    if (batches) *batches = s->local_batches;
    if (total_edges) *total_edges = s->total_edges;
    return HSAW_OK;
}

int hsaw_gpu_stream_counters(const hsaw_gpu_stream* s, uint64_t min_accepted, uint64_t* attempts,
                             uint64_t* accepted) {
    if (!s || !attempts || !accepted) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        if (min_accepted == 0) {  // sampler.cpp:474
            *attempts = 0;
            *accepted = 0;
            return;
        }
        uint64_t idx = 0, val = 0;
        local_cut(s, min_accepted, &idx, &val);
        if (idx >= s->local_batches)
            fail(HSAW_ERANGE, "sample stream target not materialized");  // sampler.cpp:477-478
        *attempts = (idx + 1) * s->cfg.batch_size;
        *accepted = val;
    });
}

int hsaw_gpu_stream_local_cut(const hsaw_gpu_stream* s, uint64_t min_local, uint64_t* nbatches,
                              uint64_t* accepted) {
    if (!s || !nbatches || !accepted) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        if (min_local == 0) {
            *nbatches = 0;
            *accepted = 0;
            return;
        }
        uint64_t idx = 0, val = 0;
        local_cut(s, min_local, &idx, &val);
        if (idx >= s->local_batches) fail(HSAW_ERANGE, "local cut beyond materialised batches");
        *nbatches = idx + 1;
        *accepted = val;
    });
}

int hsaw_gpu_stream_slice_edges(const hsaw_gpu_stream* s, uint64_t off, uint64_t cnt,
                                uint64_t* total_edges) {
    if (!s || !total_edges) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        if (off + cnt > s->accepted)
            fail(HSAW_ERANGE, "sample stream prefix not materialized");  // sampler.cpp:467-468
        hsaw_gpu_ctx* ctx = s->ctx;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[0], s->edge_off.p + off, 8,
                                        cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(&ctx->h_scalars[1], s->edge_off.p + off + cnt, 8,
                                        cudaMemcpyDeviceToHost, ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        *total_edges = ctx->h_scalars[1] - ctx->h_scalars[0];
    });
}

int hsaw_gpu_stream_export(const hsaw_gpu_stream* s, uint64_t off, uint64_t cnt,
                           uint64_t* edge_off, uint32_t* nodes, uint32_t* edges,
                           uint64_t* tag_worker, uint32_t* tag_seq) {
    if (!s || !edge_off) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        if (off + cnt > s->accepted)
            fail(HSAW_ERANGE, "sample stream prefix not materialized");
        cudaStream_t st = s->ctx->stream;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(edge_off, s->edge_off.p + off, (cnt + 1) * 8,
                                        cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        uint64_t e0 = edge_off[0], e1 = edge_off[cnt];
        if ((nodes && !s->keep_nodes) || (edges && !s->keep_edges))
            fail(HSAW_EINVAL, "stream_export: this stream does not keep that item array");
        if (nodes && (e1 - e0 + cnt))
            HSAW_CUDA_CHECK(cudaMemcpyAsync(nodes, s->nodes.p + e0 + off, (e1 - e0 + cnt) * 4,
                                            cudaMemcpyDeviceToHost, st));
        if (edges && e1 > e0)
            HSAW_CUDA_CHECK(cudaMemcpyAsync(edges, s->edges.p + e0, (e1 - e0) * 4,
                                            cudaMemcpyDeviceToHost, st));
        if (tag_worker && cnt)
            HSAW_CUDA_CHECK(cudaMemcpyAsync(tag_worker, s->tag_batch.p + off, cnt * 8,
                                            cudaMemcpyDeviceToHost, st));
        if (tag_seq && cnt)
            HSAW_CUDA_CHECK(cudaMemcpyAsync(tag_seq, s->tag_seq.p + off, cnt * 4,
                                            cudaMemcpyDeviceToHost, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i <= cnt; ++i) edge_off[i] -= e0;
        if (tag_worker)
            for (uint64_t i = 0; i < cnt; ++i) tag_worker[i] += s->seed;  // worker id = seed + batch
    });
}

int hsaw_gpu_stream_keep(hsaw_gpu_stream* s, int keep_nodes, int keep_edges) {
    if (!s) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        if (s->local_batches) fail(HSAW_EINVAL, "stream_keep: must be called before sampling");
        if (!keep_nodes && !keep_edges) fail(HSAW_EINVAL, "stream_keep: nothing to keep");
        s->keep_nodes = keep_nodes != 0;
        s->keep_edges = keep_edges != 0;
    });
}

int hsaw_gpu_stream_restrict(hsaw_gpu_stream* s, const uint32_t* domain, uint64_t ndomain,
                             const uint8_t* allowed) {
    if (!s) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        if (s->local_batches) fail(HSAW_EINVAL, "stream_restrict: must be called before sampling");
        if (!domain || !allowed || ndomain == 0 || ndomain > 0xFFFFFFFFull)
            fail(HSAW_EINVAL, "stream_restrict: empty start domain or null mask");
        const uint32_t n = s->ctx->g.n;
        for (uint64_t i = 0; i < ndomain; ++i)
            if (domain[i] >= n) fail(HSAW_EDATA, "stream_restrict: start node out of range");
        s->r_domain.ensure_scratch(ndomain);
        s->r_allowed.ensure_scratch(n);
        cudaStream_t st = s->ctx->stream;
        HSAW_CUDA_CHECK(cudaMemcpyAsync(s->r_domain.p, domain, ndomain * 4, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(cudaMemcpyAsync(s->r_allowed.p, allowed, n, cudaMemcpyHostToDevice, st));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(st));
        s->r_ndomain = (uint32_t)ndomain;
    });
}

int hsaw_gpu_stream_crossings(const hsaw_gpu_stream* s, uint64_t min_accepted, uint64_t* crossings) {
    if (!s || !crossings) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        *crossings = 0;
        if (min_accepted == 0 || s->r_ndomain == 0) return;
        uint64_t idx = 0, val = 0;
        local_cut(s, min_accepted, &idx, &val);
        if (idx >= s->local_batches) fail(HSAW_ERANGE, "sample stream target not materialized");
        *crossings = s->crossed_after_batch[idx];
    });
}

int hsaw_gpu_stream_collect_stats(hsaw_gpu_stream* s, int on) {
    if (!s) return HSAW_EINVAL;
    s->collect_stats = on != 0;
    return HSAW_OK;
}

int hsaw_gpu_stream_stats(const hsaw_gpu_stream* s, uint64_t* stats) {
    if (!s || !stats) return HSAW_EINVAL;
    return guarded(s->ctx, [&] {
        HSAW_CUDA_CHECK(cudaMemcpyAsync(s->ctx->h_scalars, s->stats.p, 64, cudaMemcpyDeviceToHost,
                                        s->ctx->stream));
        HSAW_CUDA_CHECK(cudaStreamSynchronize(s->ctx->stream));
        for (int i = 0; i < 8; ++i) stats[i] = s->ctx->h_scalars[i];
        if (!s->collect_stats) {  // work counters were not collected: fill what the host knows
            stats[hsawgpu::ST_ATTEMPTS] = s->local_batches * s->cfg.batch_size;
            stats[hsawgpu::ST_ACCEPTED] = s->accepted + s->dropped;
        }
        stats[hsawgpu::ST_DROPPED] = s->dropped;
        stats[hsawgpu::ST_SPARE] = s->replayed;  // walks that overflowed their log and were replayed
    });
}

}  // extern "C"
