/*
 * hsaw_host.h — C view of the C++ host layer (paper_1702_05854_b200/host/hsaw_b200.hpp).
 *
 * The host layer is C++ (namespace hsaw, same entry points as the reference's
 * /root/reference/proj/include/hsaw headers). These wrappers exist so that ctypes-based tests and
 * bench.py can drive it; they add no behaviour. Status codes as in hsaw_gpu.h: 0 ok, 1
 * std::invalid_argument, 2 hsaw::DataError, 3 hsaw::SamplingError, 4 std::out_of_range, 5 device.
 */
#ifndef HSAW_HOST_H
#define HSAW_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* hsawh_last_error(void);

/* ---- graphs (hsaw::ProbGraph handles) — proj/include/hsaw/graph.hpp:123-141 ---- */
int hsawh_graph_load_edge_list(const char* path, int weight_mode, uint64_t seed, int symmetrize,
                               const char* mapping_out, void** out);
int hsawh_graph_build(uint32_t n, uint64_t nedges, const uint32_t* u, const uint32_t* v,
                      const double* w, int weight_mode, uint64_t seed, void** out);
/* hsaw::build_graph_device: build_graph with the sort / sums / validation on the GPU
 * (hsaw_gpu_csr_build); weight_mode 0 Given, 1 InDegree. */
int hsawh_graph_build_device(uint32_t n, uint64_t nedges, const uint32_t* u, const uint32_t* v,
                             const double* w, int weight_mode, int device, void** out);
int hsawh_graph_synth(uint32_t n, uint32_t density, uint64_t seed, void** out);
int hsawh_graph_rmat(uint32_t scale, double edge_factor, uint64_t seed, void** out);
/* Bench inputs of any node count (hsaw::rmat_graph_n; rmat above = the power-of-two case), on the
 * host, or generated / sorted / summed on the GPU (hsaw::rmat_graph_device; lean: no weight /
 * edge_dst arrays). hsawh_graph_shell: a ProbGraph carrying only n and m, for callers that hold
 * the graph on the device alone. hsawh_graph_ptrs: borrowed views of the CSR arrays. */
int hsawh_graph_rmat_n(uint32_t n, uint64_t raw_edges, uint64_t seed, void** out);
int hsawh_graph_rmat_device(uint32_t n, uint64_t raw_edges, uint64_t seed, int device, int lean,
                            void** out);
int hsawh_graph_shell(uint32_t n, uint32_t m, void** out);
void hsawh_graph_ptrs(const void* g, const uint64_t** in_offsets, const uint32_t** in_src,
                      const double** in_cum);
int hsawh_graph_from_csr(uint32_t n, uint32_t m, const uint64_t* in_offsets,
                         const uint32_t* in_src, const double* in_cum, void** out);
int hsawh_graph_save_cache(const void* g, const char* path);
int hsawh_graph_load_cache(const char* path, void** out);
int hsawh_graph_save_edge_list(const void* g, const char* path);
int hsawh_graph_validate(const void* g);
void hsawh_graph_dims(const void* g, uint32_t* n, uint32_t* m);
/* any pointer may be NULL */
void hsawh_graph_copy(const void* g, uint64_t* in_offsets, uint32_t* in_src, double* in_cum,
                      double* weight, uint32_t* edge_dst);
void hsawh_graph_free(void* g);

/* ---- suspects: dense p_of[n] out — graph.hpp:129-132 ---- */
int hsawh_suspects_random(const void* g, uint32_t count, uint64_t seed, double* p_of);
int hsawh_suspects_random_n(uint32_t n, uint32_t count, uint64_t seed, double* p_of);
int hsawh_suspects_load(const char* path, const void* g, double* p_of);

/* ---- schedule / stopping rule — proj/include/hsaw/coverage.hpp:61-92 ---- */
/* out4 = {n_max, lambda, lambda1, (double)lambda_samples} */
int hsawh_schedule(uint64_t M, uint32_t k, double eps, double delta, double* out4,
                   uint32_t* t_max);
int hsawh_check(double cov_r, double cov_rp, double n_rp, uint64_t M, uint32_t k, double eps,
                double delta, uint32_t t, int* pass, double* eps_t);

/* ---- device graph (hsaw::DeviceGraph) ---- */
int hsawh_device_create(const void* g, const double* p_of, int device, void* cuda_stream,
                        void** out);
/* the same with a prebuilt hsaw::SuspectSet handle (hsawh_suspects_create), i.e. exactly the
 * arguments of hsaw::DeviceGraph(const ProbGraph&, const SuspectSet&, int device) */
int hsawh_suspects_create(const void* g, const double* p_of, void** out);
void hsawh_suspects_free(void* vi);
int hsawh_device_create_vi(const void* g, const void* vi, int device, void* cuda_stream,
                           void** out);
void hsawh_device_free(void* dg);
void* hsawh_device_ctx(const void* dg); /* the hsaw_gpu_ctx* underneath */

/* Binary ingest on the device (graph.hpp:139-141 load_cache): hsaw::load_cache_device returns the
 * same ProbGraph as load_cache; hsaw::DeviceGraph::from_cache goes file -> resident graph with no
 * host CSR (no suspects until hsawh_device_set_suspects). */
int hsawh_graph_load_cache_device(const char* path, int device, void** out);
/* hsaw::load_edge_list_device: load_edge_list (graph.hpp:126-128) with parse / remap / build on the
 * GPU; files outside the device parser's plain grammar go through the host parser unchanged. */
int hsawh_graph_load_edge_list_device(const char* path, int weight_mode, uint64_t seed,
                                      int symmetrize, const char* mapping_out, int device,
                                      void** out);
int hsawh_device_from_cache(const char* path, int device, void* cuda_stream, void** out);
/* hsaw::DeviceGraph::from_edge_list: text file -> resident graph; *out NULL when the file needs
 * the host loader (outside the device parser's plain grammar, RandomNormalized, empty). */
int hsawh_device_from_edge_list(const char* path, int weight_mode, int device, void* cuda_stream,
                                void** out);
/* hsaw::DeviceGraph::from_rmat: the R-MAT graph generated on the device and installed where it
 * lies. p_of dense f64[n] or NULL. *g_out: a ProbGraph handle — the lean host copy (in_offsets /
 * in_src / in_cum) when want_host, else a shell with n and m only. */
int hsawh_device_from_rmat(uint32_t n, uint64_t raw_edges, uint64_t seed, const double* p_of,
                           int device, void* cuda_stream, int want_host, void** dg_out,
                           void** g_out);
int hsawh_device_set_suspects(void* dg, const void* g, const double* p_of);

/* ---- eSIA / nSIA — proj/include/hsaw/interdiction.hpp:37-47 ---- */
typedef struct hsawh_result {
    uint32_t k, iterations;
    uint64_t coverage, samples_used, attempts;
    double est_suspension, wall_time_s, sample_s, greedy_s, check_s;
    int32_t passed_check;
} hsawh_result;
/* dg NULL: upload inside the call (timed in wall_time_s). kind 0 = esia, 1 = nsia. cand NULL =
 * all. json (nullable) receives to_json(result, false). */
int hsawh_interdict(const void* dg, const void* g, const double* p_of, int kind,
                    const uint32_t* cand, uint64_t ncand, uint32_t k, double eps, double delta,
                    uint64_t seed, uint32_t batch_size, uint64_t max_attempts, int device,
                    hsawh_result* out, uint32_t* solution, char* json, uint64_t json_cap);
/* Same with SamplerConfig::rng: 0 the reference's stream (bit-exact), 1 the device's Philox
 * per-walk throughput mode (statistical parity only; never implied). */
int hsawh_interdict_rng(const void* dg, const void* g, const double* p_of, int kind,
                    const uint32_t* cand, uint64_t ncand, uint32_t k, double eps, double delta,
                    uint64_t seed, uint32_t batch_size, uint64_t max_attempts, int device, int rng_mode,
                    hsawh_result* out, uint32_t* solution, char* json, uint64_t json_cap);

/* ---- `hsaw sample` equivalent: stream to `target`, return the counters — cli.cpp:267-290 ---- */
int hsawh_sample(const void* dg, uint64_t target, uint64_t seed, uint64_t max_attempts,
                 uint64_t* attempts, uint64_t* accepted);

/* ---- reference-signature stream_samples with the pool copied out (drop-in check) ---- */
int hsawh_stream_samples(const void* g, const double* p_of, uint64_t target, uint64_t seed,
                         uint32_t batch_size, uint64_t max_attempts, void** pool_out);
void hsawh_pool_stats(const void* pool, uint64_t* nsamples, uint64_t* attempts,
                      uint64_t* total_edges);
void hsawh_pool_copy(const void* pool, uint64_t* edge_off, uint32_t* nodes, uint32_t* edges,
                     uint64_t* tag_worker, uint32_t* tag_seq);
void hsawh_pool_free(void* pool);

/* ---- paired forward simulation — proj/include/hsaw/evaluation.hpp:25-39 ---- */
/* dg NULL: the reference signatures (g, vi) with the upload inside the call. *state is
 * PrgState::state, advanced as the reference advances it. kind 0 edge / 1 node removal. */
int hsawh_lt_forward_simulate(const void* dg, const void* g, const double* p_of, uint64_t* state,
                              uint32_t* infected);
int hsawh_estimate_suspension(const void* dg, const void* g, const double* p_of, int kind,
                              const uint32_t* ids, uint64_t nids, double eps, double delta,
                              uint64_t* state, double* value, int* capped, uint64_t* runs);

/* ---- CLI (proj/include/hsaw/cli.hpp) ---- */
/* esia / nsia with InterdictionOptions::devices: the multi-device solve of the C++ host layer
 * (graph replicated per device, walks sharded by batch range, NCCL all-reduce of the marginal-gain
 * counts; a repeated device id selects the in-process exchange). Same result for every list. */
int hsawh_interdict_devices(const void* g, const double* p_of, int kind, const uint32_t* cand,
                            uint64_t ncand, uint32_t k, double eps, double delta, uint64_t seed,
                            uint64_t max_attempts, const int* devices, uint32_t ndevices,
                            hsawh_result* out, uint32_t* solution);

/* Transport the multi-device solve would use for a device list: "nccl" (distinct devices,
 * libnccl.so.2 resolvable), "in-process exchange" (a repeated id) or "single device". */
void hsawh_multi_transport(const int* devices, uint32_t ndevices, char* out, uint64_t cap);

/* ---- partitioned sampling — proj/include/hsaw/partition.hpp:27-54 ---- */
/* partition_graph (method 0 Hash, 1 LabelProp, 2 ExternalFile with part_file) followed by
 * extend_partition(hops): assign_out u32[n], extended_out u8[p * n] part-major (nullable). */
int hsawh_partition(const void* g, uint32_t p, int method, uint64_t seed, const char* part_file,
                    uint32_t hops, uint32_t* assign_out, uint8_t* extended_out);
/* distributed_sample on a DeviceGraph: pool handle for hsawh_pool_*, targets u64[p]. */
int hsawh_distributed_sample(const void* dg, uint32_t n, uint32_t p, uint32_t hops,
                             const uint32_t* assign, const uint8_t* extended,
                             uint64_t total_target, uint64_t seed, uint32_t batch_size,
                             uint64_t max_attempts, void** pool_out, uint64_t* crossings,
                             uint64_t* attempts, double* crossing_fraction, uint64_t* targets);

/* ---- ranking baselines — proj/include/hsaw/evaluation.hpp:45-50 ---- */
/* baseline(): kind 0 Pagerank, 1 MaxDegree, 2 Randomized, 3 InfMaxV, 4 InfMaxVI; mode 0 edge,
 * 1 node; ids_out holds k ids; *state is the caller's PrgState, advanced as the reference does.
 * dg may be NULL (a DeviceGraph is then created for the InfMax kinds). */
int hsawh_baseline(const void* dg, const void* g, const double* p_of, int kind, int mode,
                   uint32_t k, uint64_t* state, uint32_t infmax_samples, uint32_t* ids_out);
/* rr_node_sets on the device: set_off u64[count + 1]; *total = nodes of all sets (items are only
 * written while they fit items_cap: call again with a larger buffer if *total > items_cap). */
int hsawh_rr_node_sets(const void* dg, uint64_t* state, uint32_t count, uint64_t* set_off,
                       uint32_t* items, uint64_t items_cap, uint64_t* total);

/* A double as the result JSON prints it (nlohmann::json::dump's number layout,
 * proj/src/interdiction.cpp:89-104). */
void hsawh_json_number(double x, char* out, uint64_t cap);
int hsawh_run_cli(int argc, const char** argv);

#ifdef __cplusplus
}
#endif
#endif /* HSAW_HOST_H */
