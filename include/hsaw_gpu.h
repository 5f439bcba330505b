/*
 * hsaw_gpu.h — C-ABI of the B200-native HSAW sampling + greedy max-cover path.
 *
 * This is the drop-in boundary for the eSIA/nSIA hot path of arXiv 1702.05854 as implemented by
 * the reference library in /root/reference/proj. The reference has no FFI layer of its own: the
 * path sits behind plain C++ functions in namespace `hsaw`. Every entry point below names the
 * reference interface (file:line, relative to /root/reference/) whose work it takes over; the C++
 * host layer in paper_1702_05854_b200/host/ re-exposes the reference's own signatures on top of
 * these calls (see INTEGRATION.md for the binding a maintainer would add).
 *
 * Conventions
 *   - plain pointers and sizes only; host arrays are borrowed for the duration of a call;
 *     outputs are written to caller-allocated host buffers unless a parameter says "device".
 *   - every function returns an hsaw_status; hsaw_gpu_last_error() gives the message.
 *   - handles are single-owner and not thread-safe (like SampleStream/DecodeContext,
 *     proj/include/hsaw/sampler.hpp:85-163).
 *   - there is NO CPU fallback: without a CUDA device every call fails with HSAW_ECUDA.
 *   - ids are uint32 (NodeId/EdgeId, proj/include/hsaw/types.hpp:9-10), so m < 2^32.
 */
#ifndef HSAW_GPU_H
#define HSAW_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. 1..3 mirror the exception -> exit-code mapping of proj/src/cli.cpp:520-538 so the
 * host layer can rethrow the matching exception type. */
typedef enum hsaw_status {
    HSAW_OK = 0,
    HSAW_EINVAL = 1,  /* std::invalid_argument */
    HSAW_EDATA = 2,   /* hsaw::DataError (proj/include/hsaw/types.hpp:21) */
    HSAW_EBUDGET = 3, /* hsaw::SamplingError (types.hpp:26): attempt budget exhausted */
    HSAW_ERANGE = 4,  /* std::out_of_range: prefix/counters beyond what is materialised */
    HSAW_ECUDA = 5    /* CUDA runtime failure / no device */
} hsaw_status;

typedef struct hsaw_gpu_ctx hsaw_gpu_ctx;         /* one device + the uploaded graph */
typedef struct hsaw_gpu_stream hsaw_gpu_stream;   /* SampleStream, device resident */
typedef struct hsaw_gpu_walkset hsaw_gpu_walkset; /* fixed item sets (CoverageIndex input) */

/* SamplerConfig, proj/include/hsaw/sampler.hpp:48-55. */
typedef struct hsaw_sampler_cfg {
    int32_t heuristic;     /* 0 Brent (default), 1 Floyd, 2 None (CycleHeuristic, sampler.hpp:46) */
    uint32_t window;       /* exact short-cycle window, 0..8 (default 2) */
    uint32_t batch_size;   /* attempts chained per batch / worker id (default 10) */
    uint64_t max_attempts; /* stream budget (default 100000000) */
    /* 0 (default): the reference's stream — xorshift64* chained through each batch
     * (proj/src/sampler.cpp:267-290); every output is bit-exact with the reference.
     * 1: throughput mode, NOT the reference's walks: a counter-based Philox4x32-10 substream per
     * walk index, one independent attempt per lane with immediate refill. Same walk law (start,
     * live-edge pick, Brent + window 2, acceptance), same (batch, seq) bookkeeping with
     * batch = walk index / batch_size; parity is statistical only (hit rate, length distribution,
     * per-edge frequency, est_suspension; tests/test_gpu_philox.py states the tolerances).
     * Requires heuristic 0 and window 2. */
    uint32_t rng_mode;
} hsaw_sampler_cfg;

/* ItemKind, proj/include/hsaw/types.hpp:14. */
enum { HSAW_KIND_EDGE = 0, HSAW_KIND_NODE = 1 };

/* ---- context ------------------------------------------------------------------------------- */

/* Binds a CUDA device. cuda_stream: a cudaStream_t the caller owns (e.g. a torch stream) or NULL
 * to let the context create its own; all kernels of this context are launched on it. */
int hsaw_gpu_ctx_create(int device, void* cuda_stream, hsaw_gpu_ctx** out);
void hsaw_gpu_ctx_destroy(hsaw_gpu_ctx* ctx);
const char* hsaw_gpu_last_error(const hsaw_gpu_ctx* ctx);
/* The cudaStream_t kernels run on (for CUDA-event timing by the caller). */
void* hsaw_gpu_ctx_cuda_stream(const hsaw_gpu_ctx* ctx);
int hsaw_gpu_ctx_sync(hsaw_gpu_ctx* ctx);

/* Replaces the host-resident ProbGraph + SuspectSet the reference sampler reads
 * (proj/include/hsaw/graph.hpp:19-51 in_offsets/in_src/in_cum, :84-94 p_of). The arrays are the
 * reference's own: in_offsets u64[n+1], in_src u32[m], in_cum f64[m] (per-row sequential FP64
 * cumulative sums, proj/src/graph.cpp:158-192 — uploaded, never recomputed), p_of f64[n].
 * They are re-laid out on the device into 32-byte node records plus either the
 * compact arrays (packed in_src + 16-byte row headers, graphs whose headers fit in L2) or 32-byte
 * edge records (fat layout), all holding exact integer thresholds. HSAW_EDATA if a row's cumulative array decreases. */
int hsaw_gpu_graph_upload(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const uint64_t* in_offsets,
                          const uint32_t* in_src, const double* in_cum, const double* p_of);

/* Replaces build_graph (proj/src/graph.cpp:112-199, declared proj/include/hsaw/graph.hpp:123-125)
 * for WeightMode::Given (weight_mode 0, edge_w required) and ::InDegree (weight_mode 1, edge_w
 * ignored): the edge list (edge_u[i] -> edge_v[i]) is sorted on the device into the canonical
 * (target, source) order, edge id = CSR position, and every row's in_cum is the SEQUENTIAL FP64
 * sum the reference computes, so all outputs are bit-identical to the reference's ProbGraph
 * fields: in_offsets u64[n+1], in_src u32[ne], in_cum f64[ne], and optionally weight f64[ne],
 * edge_dst u32[ne] (NULL to skip). Data errors return HSAW_EDATA with the reference's messages
 * ("edge endpoint out of range", "self-loop u -> v", "weight w out of (0,1] on edge u -> v",
 * "duplicate edge u -> v", "in-weight sum s > 1 at node v", and validate()'s "graph: in-weight sum
 * ..." / "graph: cumulative weights not increasing ..."). WeightMode::RandomNormalized (one global
 * xorshift stream over all rows) is not built on the device: HSAW_EINVAL. */
int hsaw_gpu_csr_build(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                       const uint32_t* edge_v, const double* edge_w, int weight_mode,
                       uint64_t* out_in_offsets, uint32_t* out_in_src, double* out_in_cum,
                       double* out_weight, uint32_t* out_edge_dst);

/* build_graph + hsaw_gpu_graph_upload in one step, without the CSR ever visiting the host: the
 * edge list goes up (8 or 16 bytes per edge instead of 12 + 8 n / m), is sorted and summed on the
 * device and re-laid out for the walk kernels. Same errors as hsaw_gpu_csr_build. */
int hsaw_gpu_graph_build_upload(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t ne, const uint32_t* edge_u,
                                const uint32_t* edge_v, const double* edge_w, int weight_mode,
                                const double* p_of);

/* Text ingest: the parsing and id-remap half of load_edge_list (proj/src/graph.cpp:29-59 parse_line,
 * :201-241) on the device. `text` is the whole edge-list file. Lines are split at '\n', tokenised
 * at C-locale whitespace; blank and '#' lines are skipped; an edge line is "u v" or "u v w".
 * The device handles the plain grammar (unsigned decimal ids of <= 19 digits; weights
 * digits[.digits][e[+-]digits] with <= 19 significant digits in the normal range, converted to
 * the correctly rounded double std::stod returns). If any line is outside it (signs, hex floats,
 * inf/nan, overlong numbers, malformed lines, a missing weight when weight_required) nothing is
 * guessed: *host_line is set to the 1-based number of the first such line and no handle is
 * returned; the caller re-reads the file with the host parser, which words the errors.
 * weight_required: WeightMode::Given (:216-218). weight_values: also convert the weights (else they
 * are only validated and returned as 0.0, for modes that ignore them). On success *nedges edge
 * lines in file order, *nids distinct raw ids, *identity = raw ids are already 0..nids-1 (:236).
 * hsaw_gpu_edge_text_fetch copies out dense endpoints (rank of the raw id among the sorted ids,
 * :232-241), weights and the sorted raw ids (the node map, :254-260); every pointer nullable. */
typedef struct hsaw_gpu_edge_text hsaw_gpu_edge_text;
int hsaw_gpu_edge_text_parse(hsaw_gpu_ctx* ctx, const char* text, uint64_t bytes,
                             int weight_required, int weight_values, hsaw_gpu_edge_text** out,
                             uint64_t* nedges, uint64_t* nids, int* identity, uint64_t* host_line);
int hsaw_gpu_edge_text_fetch(hsaw_gpu_edge_text* el, uint32_t* edge_u, uint32_t* edge_v,
                             double* edge_w, uint64_t* raw_ids);
/* build_graph + hsaw_gpu_graph_upload on the parsed edges where they lie on the device: text file ->
 * graph resident and ready to sample, no host CSR and no host edge list. weight_mode 0 Given (the
 * parse must have converted the weights) / 1 InDegree; p_of NULL = no suspects yet. Same errors as
 * hsaw_gpu_csr_build. */
int hsaw_gpu_edge_text_install(hsaw_gpu_edge_text* el, int weight_mode, const double* p_of);
void hsaw_gpu_edge_text_free(hsaw_gpu_edge_text* el);

/* Binary ingest: the HSAW1 cache format (save_cache / load_cache, proj/src/graph.cpp:383-430).
 * `body` points at the bytes that follow the 21-byte header ("HSAW1", n, m as LE u64): (n + 1) u64
 * offsets, m u64-widened sources, m f64 bit patterns, all little endian, as they lie in the file
 * (any alignment). The device decodes them, runs load_cache's sequential per-row cumulative sums
 * (:417-424) and the checks of ProbGraph::validate() (:70-104, HSAW_EDATA with the reference's
 * message for the first offending row).
 * hsaw_gpu_cache_decode returns the ProbGraph arrays (out_weight / out_edge_dst nullable);
 * hsaw_gpu_graph_cache_upload installs the graph on the device without any host CSR (p_of NULL =
 * no suspects yet; hsaw_gpu_suspects_upload sets them later). */
int hsaw_gpu_cache_decode(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const void* body,
                          uint64_t* out_in_offsets, uint32_t* out_in_src, double* out_in_cum,
                          double* out_weight, uint32_t* out_edge_dst);
int hsaw_gpu_graph_cache_upload(hsaw_gpu_ctx* ctx, uint32_t n, uint32_t m, const void* body,
                                const double* p_of);

/* Bench inputs (no reference counterpart: the reference's only generator is the uniform
 * synth_graph, proj/src/graph.cpp:330-352; SURVEY.md §8d asks for R-MAT graphs of the named
 * shapes). Generates on the device the graph hsaw::rmat_graph_n (host/graph_io.cpp) defines,
 * bit-identical to it: quadrant probabilities (a, b, c, 1-a-b-c), ceil(log2 n) draws of one
 * xorshift64* stream (proj/include/hsaw/prng.hpp:41-53) per raw edge starting from `prg_state`
 * (the state after the generator's n-1 relabelling draws), endpoints relabelled through label[n]
 * (host array), self-loops / endpoints >= n / duplicates removed, rows in (target, source) order,
 * WeightMode::InDegree cumulative sums as build_graph forms them (graph.cpp:172-178). The CSR stays
 * on the device, held by the context; *out_m = edges kept.
 *   hsaw_gpu_held_csr_fetch    copies the reference-layout arrays out (any pointer nullable)
 *   hsaw_gpu_held_csr_install  = hsaw_gpu_graph_upload on the held arrays where they lie (p_of NULL =
 *                              no suspects yet); keep != 0 keeps the CSR for a later fetch
 *   hsaw_gpu_held_csr_drop     frees it */
int hsaw_gpu_rmat_build(hsaw_gpu_ctx* ctx, uint32_t n, uint64_t raw_edges, const uint32_t* label,
                        uint64_t prg_state, double a, double b, double c, uint64_t* out_m);
int hsaw_gpu_held_csr_fetch(hsaw_gpu_ctx* ctx, uint64_t* in_offsets, uint32_t* in_src,
                            double* in_cum);
int hsaw_gpu_held_csr_install(hsaw_gpu_ctx* ctx, const double* p_of, int keep);
void hsaw_gpu_held_csr_drop(hsaw_gpu_ctx* ctx);

/* Same, but p_of replaced later without re-uploading the CSR (new SuspectSet on the same graph). */
int hsaw_gpu_suspects_upload(hsaw_gpu_ctx* ctx, const double* p_of);
/* Bytes of device memory held by the uploaded graph. */
uint64_t hsaw_gpu_graph_bytes(const hsaw_gpu_ctx* ctx);
/* Device layout of the uploaded graph: 0 = fat 32-byte edge records; 21 / 32 =
 * compact arrays with 21-bit packed / 32-bit flagged sources; 1 = compact with plain sources
 * (HSAW_PACK=0); -1 = no graph. Diagnostic only: results never depend on it. */
int hsaw_gpu_graph_layout(const hsaw_gpu_ctx* ctx);
/* How the last hsaw_gpu_graph_upload moved in_cum: 0 copied from the host array, 1 regenerated on
 * the device after host threads verified, bit for bit, that every row holds the sequential
 * 1/in-degree sums of WeightMode::InDegree (proj/src/graph.cpp:172-178). Diagnostic. */
int hsaw_gpu_graph_upload_mode(const hsaw_gpu_ctx* ctx);
/* Bytes the last hsaw_gpu_graph_upload copied host -> device (the regenerated part of in_cum is
 * the difference to 8 (n + 1) + 12 m + 8 n). */
uint64_t hsaw_gpu_graph_upload_bytes(const hsaw_gpu_ctx* ctx);

/* ---- sampler: encode / decode (kernels K1, K2) ---------------------------------------------- */

/* thread_sample for a range of batches (proj/src/sampler.cpp:267-290; worker ids
 * first_worker_id + b, b in [0, nbatches)): out_count[b] accepted attempts of batch b, their
 * (seed, len) in out_seed/out_len[b * batch_size + seq]. Bit-exact with the reference stream.
 * stats (nullable) u64[8]: {attempts, draws, steps(picks), alg_bytes, accepted, 0, 0,
 * walk_items = sum of (len + 1) over the accepted walks}. */
int hsaw_gpu_encode_batches(hsaw_gpu_ctx* ctx, const hsaw_sampler_cfg* cfg,
                            uint64_t first_worker_id, uint64_t nbatches, uint64_t* out_seed,
                            uint32_t* out_len, uint32_t* out_count, uint64_t* stats);

/* Instrumentation only: the work counters of the same batch range without producing output
 * (u64[8] as above). Used by bench.py to attribute algorithmic bytes to timed launches whose
 * production kernels run with counters compiled out. */
int hsaw_gpu_encode_stats(hsaw_gpu_ctx* ctx, const hsaw_sampler_cfg* cfg, uint64_t first_worker_id,
                          uint64_t nbatches, uint64_t* stats);

/* DecodeContext::decode for an array of encoded walks (proj/src/sampler.cpp:295-338).
 * edge_off u64[nwalks+1] must be the exclusive prefix sum of lens. Walk w gets nodes
 * [edge_off[w]+w, edge_off[w+1]+w+1) and edges [edge_off[w], edge_off[w+1]).
 * out_status[w]: 1 decoded, 0 dropped (revisit found by the exact recheck), 2 replay mismatch
 * (the reference throws DataError, sampler.cpp:306-335). */
int hsaw_gpu_decode_walks(hsaw_gpu_ctx* ctx, uint64_t nwalks, const uint64_t* seeds,
                          const uint32_t* lens, const uint64_t* edge_off, uint32_t* out_nodes,
                          uint32_t* out_edges, uint8_t* out_status);

/* ---- sample stream (proj/src/sampler.cpp:383-501) ------------------------------------------- */

/* SampleStream ctor. Batch b of the stream uses worker id seed + b (sampler.cpp:430). */
int hsaw_gpu_stream_create(hsaw_gpu_ctx* ctx, uint64_t seed, const hsaw_sampler_cfg* cfg,
                           hsaw_gpu_stream** out);
/* Which item arrays the stream's pool keeps. A SampleStream holds nodes and edge_ids of every
 * walk (HsawSample, proj/include/hsaw/sampler.hpp:27-33); a solve over edge candidates only ever
 * indexes the edge ids and one over node candidates only the nodes (CoverageIndex,
 * proj/src/coverage.cpp:49-53), and at the Twitter shape each array is tens of gigabytes. Call
 * before sampling. Order, counters and every result are unaffected; greedy / coverage / export
 * calls that ask for a dropped array fail with HSAW_EINVAL. */
int hsaw_gpu_stream_keep(hsaw_gpu_stream* stream, int keep_nodes, int keep_edges);

/* Partitioned sampling: the per-part restricted stream of distributed_sample
 * (proj/src/partition.cpp:183-268; detail::sample_batch_restricted, proj/src/sampler.cpp:510-539;
 * WalkCursor::start with a domain, sampler.cpp:24-31; the crossing abort, sampler.cpp:196-199).
 * domain: the part's base nodes, ascending (start nodes are drawn from it); allowed: byte mask over
 * all n nodes (the part's h-hop extension). A walk that moves onto a node outside the mask without
 * hitting is aborted and counted as a crossing. Call before sampling; the caller creates the
 * stream with seed + part * 2^40 (partition.cpp:14,218). hsaw_gpu_stream_crossings gives the
 * crossings of the minimal whole-batch prefix reaching min_accepted (the reference's
 * crossed_after[cut_batches - 1]); hsaw_gpu_stream_counters gives its attempts and samples. */
int hsaw_gpu_stream_restrict(hsaw_gpu_stream* stream, const uint32_t* domain, uint64_t ndomain,
                             const uint8_t* allowed);
int hsaw_gpu_stream_crossings(const hsaw_gpu_stream* stream, uint64_t min_accepted,
                              uint64_t* crossings);
void hsaw_gpu_stream_destroy(hsaw_gpu_stream* s);

/* SampleStream::ensure (sampler.cpp:388-463): grow until >= min_accepted decoded samples exist.
 * HSAW_EBUDGET once floor(max_attempts / batch_size) batches did not suffice. */
int hsaw_gpu_stream_ensure(hsaw_gpu_stream* s, uint64_t min_accepted);

/* Multi-GPU building block: sample exactly the global batches [first_batch, first_batch +
 * nbatches) and append their decoded walks to this (rank-local) stream. Ranges must be issued in
 * increasing order. accepted_in_range: decoded walks they produced. */
int hsaw_gpu_stream_sample_range(hsaw_gpu_stream* s, uint64_t first_batch, uint64_t nbatches,
                                 uint64_t* accepted_in_range);

/* accepted = decoded walks held, batches = batches run, total_edges = sum of their lengths. */
int hsaw_gpu_stream_size(const hsaw_gpu_stream* s, uint64_t* accepted, uint64_t* batches,
                         uint64_t* total_edges);

/* SampleStream::counters_for (sampler.cpp:472-482): attempts/accepted of the minimal whole-batch
 * prefix reaching min_accepted. HSAW_ERANGE if not materialised. */
int hsaw_gpu_stream_counters(const hsaw_gpu_stream* s, uint64_t min_accepted, uint64_t* attempts,
                             uint64_t* accepted);

/* Rank-local variant for sharded streams: within the ranges this stream ran, the number of
 * batches (counted from its first local batch) needed to hold min_local decoded walks and the
 * decoded count at that batch. */
int hsaw_gpu_stream_local_cut(const hsaw_gpu_stream* s, uint64_t min_local, uint64_t* nbatches,
                              uint64_t* accepted);

/* SampleStream::prefix / to_pool (sampler.cpp:465-493) copied to the host: walks
 * [off, off + cnt). edge_off u64[cnt+1] (rebased to 0), nodes u32[E + cnt], edges u32[E] with
 * E = total edges of the slice (hsaw_gpu_stream_slice_edges). tags nullable. */
int hsaw_gpu_stream_slice_edges(const hsaw_gpu_stream* s, uint64_t off, uint64_t cnt,
                                uint64_t* total_edges);
int hsaw_gpu_stream_export(const hsaw_gpu_stream* s, uint64_t off, uint64_t cnt,
                           uint64_t* edge_off, uint32_t* nodes, uint32_t* edges,
                           uint64_t* tag_worker, uint32_t* tag_seq);

/* Turns the K1 work counters (draws, picks, algorithmic bytes) on or off for this stream. They
 * cost registers in the hot kernel, so they are off unless requested (or HSAW_STATS=1). */
int hsaw_gpu_stream_collect_stats(hsaw_gpu_stream* s, int on);

/* Sampler work counters accumulated over the stream's life (u64[8], as in encode_batches; [5] =
 * replay (K2) picks, [6] = walks dropped by the exact recheck, [7] = walks whose log overflowed
 * and were replayed). [1]-[3] stay 0 unless hsaw_gpu_stream_collect_stats is on. */
int hsaw_gpu_stream_stats(const hsaw_gpu_stream* s, uint64_t* stats);

/* ---- fixed walk sets (fixed-walk-set parity mode) ------------------------------------------- */

/* Raw item sets, as the CoverageIndex item-set constructor takes them
 * (proj/src/coverage.cpp:60-74): set i = items[set_off[i] .. set_off[i+1]). limit = id space
 * (g.m for edges, g.n for nodes). */
int hsaw_gpu_walkset_import(hsaw_gpu_ctx* ctx, uint32_t limit, uint64_t nsets,
                            const uint64_t* set_off, const uint32_t* items,
                            hsaw_gpu_walkset** out);
void hsaw_gpu_walkset_destroy(hsaw_gpu_walkset* w);

/* ---- greedy max-cover + coverage (kernels K3-K6) -------------------------------------------- */

/* CoverageIndex(kind, samples[off, off+cnt), cand) + greedy_max_cover(idx, k)
 * (proj/src/coverage.cpp:37-58, 91-138). Exactly one of stream / walkset is non-NULL; kind picks
 * edge ids or all nodes of the stream's walks (coverage.cpp:49-53) and is ignored for walksets.
 * cand_ids NULL = CandidateSet::all. solution u32[k] in selection order (ties and zero-gain
 * slots -> smallest id, coverage.cpp:101-106,155); coverage = sum of marginal gains.
 * HSAW_EINVAL if k exceeds the candidate count, HSAW_EDATA for a candidate id >= limit. */
int hsaw_gpu_greedy(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                    const hsaw_gpu_walkset* walkset, int kind, uint64_t off, uint64_t cnt,
                    const uint32_t* cand_ids, uint64_t ncand, uint32_t k, uint32_t* solution,
                    uint64_t* coverage);

/* CoverageIndex::coverage_of (proj/src/coverage.cpp:76-89) on walks [off, off+cnt): number of
 * distinct walks containing at least one of the candidate items in `items`. */
int hsaw_gpu_coverage_of(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                         const hsaw_gpu_walkset* walkset, int kind, uint64_t off, uint64_t cnt,
                         const uint32_t* cand_ids, uint64_t ncand, const uint32_t* items,
                         uint64_t nitems, uint64_t* coverage);

/* An upper bound of CoverageIndex::coverage_of(S) (proj/src/coverage.cpp:76-89) over EVERY set S of
 * at most k candidate items, on the walks [off, off + cnt): the sum of the k largest per-item
 * occurrence counts (capped at cnt). The doubling loop uses it on R'_t before running greedy:
 * check_solution (coverage.cpp:216-217) fails whenever Cov_R'(solution) < Lambda_1, so an iteration
 * whose bound is below Lambda_1 — and that is not the last one allowed by N_max — cannot pass
 * whatever greedy selects, and its greedy run and coverage counts are skipped. Results are
 * unchanged: only the final iteration's solution is ever reported (interdiction.cpp:36-61). */
int hsaw_gpu_coverage_upper_bound(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                                  const hsaw_gpu_walkset* walkset, int kind, uint64_t off,
                                  uint64_t cnt, const uint32_t* cand_ids, uint64_t ncand,
                                  uint32_t k, uint64_t* bound);

/* Building blocks of the sharded (multi-GPU) solve: walks are sharded over ranks by
 * batch range, so CoverageIndex / greedy_max_cover (proj/src/coverage.cpp:37-138) become: local
 * counts -> all-reduce (the caller's NCCL) -> every rank extracts from its LOCAL walks the items
 * that can still win -> all-gather of those reduced walks -> the single-GPU greedy run redundantly.
 * d_counts arguments are DEVICE pointers to `limit` u32 counters (limit = m for edges, n for nodes).
 *   hsaw_gpu_stream_histogram   occurrences of every candidate item in walks [off, off+cnt)
 *   hsaw_gpu_counts_bound       hsaw_gpu_coverage_upper_bound's answer from (all-reduced) counts
 *   hsaw_gpu_counts_threshold   the indexing threshold hsaw_gpu_greedy would choose for them
 *   hsaw_gpu_reduced_walks      walks [off, off+cnt) restricted to items with count >= min_count
 *                               (walks left empty are dropped), as a device walk set
 *   hsaw_gpu_walkset_copy_device / _from_device   lengths + items out of / into a walk set,
 *                               device to device (the all-gather buffers)
 *   hsaw_gpu_last_greedy_min_gain  smallest per-round gain of the last hsaw_gpu_greedy on this
 *                               context (0 if it ran out of positive gains): below min_count means
 *                               the reduced instance was not enough and the caller gathers all */
int hsaw_gpu_stream_histogram(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind,
                              uint64_t off, uint64_t cnt, const uint32_t* cand_ids, uint64_t ncand,
                              uint32_t* d_counts);
int hsaw_gpu_counts_bound(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit, uint32_t k,
                          uint64_t cap, uint64_t* bound);
int hsaw_gpu_counts_threshold(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit,
                              uint32_t* min_count);
/* hsaw_gpu_counts_threshold raised to ck_percent % of the k-th largest count (0: the plain rule):
 * an optimistic threshold, valid iff the greedy run on the reduced walks ends with
 * hsaw_gpu_last_greedy_min_gain >= it; callers step down 60 -> 30 -> 0 -> everything. */
int hsaw_gpu_counts_threshold_for(hsaw_gpu_ctx* ctx, const uint32_t* d_counts, uint32_t limit,
                                  uint32_t k, uint32_t ck_percent, uint32_t* min_count);
int hsaw_gpu_reduced_walks(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream, int kind, uint64_t off,
                           uint64_t cnt, const uint32_t* d_counts, uint32_t min_count,
                           hsaw_gpu_walkset** out, uint64_t* nsets, uint64_t* nitems);
int hsaw_gpu_walkset_copy_device(const hsaw_gpu_walkset* walkset, uint32_t* d_lens,
                                 uint32_t* d_items);
int hsaw_gpu_walkset_from_device(hsaw_gpu_ctx* ctx, uint32_t limit, uint64_t nsets,
                                 const uint32_t* d_lens, const uint32_t* d_items, uint64_t nitems,
                                 hsaw_gpu_walkset** out);
uint64_t hsaw_gpu_last_greedy_min_gain(const hsaw_gpu_ctx* ctx);
/* Device-buffer plumbing for a host that drives several contexts from one process (the C++
 * multi-device solve, host/multi.cpp): allocation on the context's device, copies between any two
 * device pointers (also across devices), and dst[i] += src[i] over u32 counters. */
int hsaw_gpu_device_alloc(hsaw_gpu_ctx* ctx, uint64_t bytes, void** out);
void hsaw_gpu_device_free(hsaw_gpu_ctx* ctx, void* p);
int hsaw_gpu_device_copy(hsaw_gpu_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int hsaw_gpu_counts_add(hsaw_gpu_ctx* ctx, uint32_t* d_dst, const uint32_t* d_src, uint64_t n);

/* ---- stepwise greedy for sharded (multi-GPU) solves ---------------------------------------- */

/* The rounds of greedy_max_cover split into steps so that ranks holding disjoint shards of R_t can
 * keep one replicated vector of marginal-gain counts:
 *   begin   local histogram of this rank's walks [off, off+cnt) into d_counts (DEVICE memory owned
 *           by the caller, u32[limit + 4], e.g. a torch tensor) + local inverted index;
 *           the caller then all-reduces d_counts (sum) across ranks, in place;
 *   select  argmax (largest count, smallest id) over d_counts -> host; identical on every rank;
 *   cover   marks this rank's uncovered walks containing `item` covered, decrements d_counts for
 *           their candidate items and appends every decremented item id to d_list (DEVICE, caller
 *           owned, capacity list_cap >= hsaw_gpu_rounds_occurrences); n_out = entries written;
 *   apply   replays a peer's decrement list (DEVICE pointer) on this rank's d_counts.
 * After each round every rank has applied every rank's list, so the replicas stay identical and
 * the selections equal the single-GPU greedy (proj/src/coverage.cpp:91-138) bit for bit. */
typedef struct hsaw_gpu_rounds hsaw_gpu_rounds;
int hsaw_gpu_rounds_begin(hsaw_gpu_ctx* ctx, const hsaw_gpu_stream* stream,
                          const hsaw_gpu_walkset* walkset, int kind, uint64_t off, uint64_t cnt,
                          const uint32_t* cand_ids, uint64_t ncand, uint32_t* d_counts,
                          hsaw_gpu_rounds** out);
uint64_t hsaw_gpu_rounds_occurrences(const hsaw_gpu_rounds* g);
int hsaw_gpu_rounds_select(hsaw_gpu_rounds* g, uint32_t* item, uint64_t* gain);
int hsaw_gpu_rounds_cover(hsaw_gpu_rounds* g, uint32_t item, uint32_t* d_list, uint64_t list_cap,
                          uint64_t* n_out);
int hsaw_gpu_rounds_apply(hsaw_gpu_rounds* g, const uint32_t* d_items, uint64_t n);
void hsaw_gpu_rounds_end(hsaw_gpu_rounds* g);

/* ---- paired LT forward simulation ----------------------------------------- */

/* The run loop of estimate_suspension (proj/src/evaluation.cpp:228-237) and lt_forward_simulate
 * (proj/include/hsaw/evaluation.hpp:25-26, evaluation.cpp:202-207) for `nruns` consecutive runs on
 * ONE xorshift64* stream: run i draws the seed set (members ascending) and one live in-edge per
 * node (draw_realization, :49-59) and counts the infected nodes on the original graph (full[i])
 * and on the residual graph without the removal set (residual[i]; count_infected, :65-108).
 * *prg_state is PrgState::state before the first run and is advanced exactly as the reference
 * would (nruns * (|V_I| + n) draws). kind: HSAW_KIND_EDGE / HSAW_KIND_NODE select what removal_ids
 * name (RemovalSet, evaluation.hpp:16-21; ids out of range: HSAW_EDATA); kind -1 = no removal
 * (residual, if given, repeats full). Results are bit-exact with the sequential reference. */
int hsaw_gpu_paired_runs(hsaw_gpu_ctx* ctx, int kind, const uint32_t* removal_ids, uint64_t nids,
                         uint64_t* prg_state, uint64_t nruns, uint32_t* full, uint32_t* residual);

/* PrgState::state after `draws` calls of prg_next (proj/include/hsaw/prng.hpp:41-48) without
 * making them: the state update is linear over GF(2), so this is a 64x64 bit-matrix power applied
 * to the state. Pure host arithmetic (no device needed); lets a caller address any run of a
 * simulation stream directly, e.g. to shard the runs of hsaw_gpu_paired_runs over several GPUs. */
uint64_t hsaw_gpu_prg_jump(uint64_t prg_state, uint64_t draws);

/* estimate_suspension (evaluation.hpp:36-39, evaluation.cpp:209-242): stopping-rule estimate of
 * the influence suspension of a removal set. Same argument checks and order (HSAW_EINVAL for
 * epsilon/delta outside (0,1), HSAW_EDATA for a bad id), same early return for an empty set, same
 * draw cap (10^9 draws), same value/capped/runs and the same final *prg_state. Runs are simulated
 * in device batches; the FP64 accumulation runs on the host one run at a time, in order. */
int hsaw_gpu_estimate_suspension(hsaw_gpu_ctx* ctx, int kind, const uint32_t* removal_ids,
                                 uint64_t nids, double epsilon, double delta, uint64_t* prg_state,
                                 double* value, int* capped, uint64_t* runs);

/* Reverse-reachable node sets of the InfMax baselines (rr_node_sets, proj/src/evaluation.cpp:169-191,
 * used by baseline(), :356-376): `count` sets drawn from the caller's sequential xorshift64* stream
 * — a uniform start node, then live in-edge picks until "no edge" or a pick lands on a node already
 * in the set; 1 + |set| draws each. Bit-exact with the reference's stream: the device evaluates the
 * set that would start at every stream position of a window and the chain of real starts is
 * followed through it. *prg_state is advanced past the last set. The sets come
 * back as a device walk set over node ids (limit = n), ready for hsaw_gpu_greedy /
 * hsaw_gpu_coverage_of; hsaw_gpu_walkset_export copies any walk set out (set_off u64[nsets + 1],
 * items; both nullable). */
int hsaw_gpu_rr_node_sets(hsaw_gpu_ctx* ctx, uint64_t* prg_state, uint32_t count,
                          hsaw_gpu_walkset** out, uint64_t* total_nodes);
int hsaw_gpu_walkset_export(const hsaw_gpu_walkset* walkset, uint64_t* set_off, uint32_t* items);

/* ---- instrumentation ------------------------------------------------------------------------ */

/* Number of kernel launches this context has issued since creation (bench.py "gpu_launches"). */
uint64_t hsaw_gpu_launch_count(const hsaw_gpu_ctx* ctx);

/* Device time per stage, measured with CUDA events recorded on the context stream directly around
 * the stage's kernels (so it is the kernels' own duration, not the host call's). */
enum {
    HSAW_STAGE_ENCODE = 0,   /* K1 encode_kernel */
    HSAW_STAGE_DECODE = 1,   /* K2 decode_kernel */
    HSAW_STAGE_DISTINCT = 2, /* K2b exact self-avoidance recheck */
    HSAW_STAGE_COMPACT = 3,  /* gather + scans + deterministic compaction */
    HSAW_STAGE_INDEX = 4,    /* K3 histogram + inverted index */
    HSAW_STAGE_ROUNDS = 5,   /* K4/K5 greedy rounds */
    HSAW_STAGE_COVERAGE = 6, /* K6 coverage_of */
    HSAW_STAGE_UPLOAD = 7,   /* graph transform kernels */
    HSAW_STAGE_SIMULATE = 8, /* paired forward simulation (realize + pointer jumping + counts) */
    HSAW_STAGE_COUNT = 9
};
/* ms[HSAW_STAGE_COUNT] accumulated milliseconds, count[HSAW_STAGE_COUNT] timed regions (both
 * nullable); reset != 0 zeroes the accumulators afterwards. Synchronises the stream. */
int hsaw_gpu_stage_times(hsaw_gpu_ctx* ctx, double* ms, uint64_t* count, int reset);

/* Process-wide device-allocation counters: out[0] host seconds spent in pool allocations,
 * out[1] calls, out[2] bytes requested (as doubles). */
void hsaw_gpu_debug_counters(double* out3);

#ifdef __cplusplus
}
#endif
#endif /* HSAW_GPU_H */
