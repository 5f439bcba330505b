/* TEST INFRASTRUCTURE ONLY — see hsaw_oracle.h. Plain-C restatement of the reference hot path.
 * Compiled with -ffp-contract=off so every FP64 operation rounds exactly as the reference's
 * (g++ -O2 on x86-64: SSE2 doubles, no fused multiply-add). */
#include "hsaw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INVALID_NODE 0xFFFFFFFFu /* kInvalidNode, proj/include/hsaw/types.hpp:12 */

/* ------------------------------------------------------------------------------------------
 * prng — proj/include/hsaw/prng.hpp
 * ---------------------------------------------------------------------------------------- */

/* splitmix_next, prng.hpp:29-38 */
void orc_splitmix_next(uint64_t state, uint64_t* out_state, uint64_t* out_output) {
    uint64_t z = state + 0x9E3779B97F4A7C15ULL;
    uint64_t o = z;
    o ^= o >> 30;
    o *= 0xBF58476D1CE4E5B9ULL;
    o ^= o >> 27;
    o *= 0x94D049BB133111EBULL;
    o ^= o >> 31;
    *out_state = z;
    *out_output = o;
}

/* prg_next (xorshift64*), prng.hpp:41-48 */
uint64_t orc_prg_next(uint64_t* state) {
    uint64_t x = *state;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    *state = x;
    return x * 0x2545F4914F6CDD1DULL;
}

/* u01, prng.hpp:51-53 */
double orc_u01(uint64_t output) { return (double)(output >> 11) * 0x1.0p-53; }

/* pick_uniform_node, prng.hpp:57-61 */
uint32_t orc_pick_uniform_node(uint64_t* state, uint32_t n) {
    double r = orc_u01(orc_prg_next(state));
    uint32_t v = (uint32_t)(r * (double)n);
    return v < n ? v : n - 1;
}

/* seed_from_worker, prng.hpp:65-72 */
uint64_t orc_seed_from_worker(uint64_t worker_id) {
    uint64_t st = worker_id;
    for (;;) {
        uint64_t ns, out;
        orc_splitmix_next(st, &ns, &out);
        if (out != 0) return out;
        st = ns;
    }
}

/* ------------------------------------------------------------------------------------------
 * live-edge pick — proj/include/hsaw/graph.hpp:61-80
 * ---------------------------------------------------------------------------------------- */

static uint32_t ceil_log2_u64(uint64_t d) { /* d >= 1 */
    return d <= 1 ? 0u : (uint32_t)(64 - __builtin_clzll(d - 1));
}

/* Algorithmic bytes of one pick (stated in DESIGN.md):
 * d = 0: offsets pair (16); r >= total: + total read (24); success: + ceil(log2 d) probes of 8 B
 * + in_src (4). The p_of read (8) is added by the caller when resolve() runs. */
static uint64_t pick_bytes(uint64_t d, int success) {
    if (d == 0) return 16;
    if (!success) return 24;
    return 28 + 8ull * ceil_log2_u64(d);
}

int orc_pick_live_in_edge(uint64_t* state, const orc_graph* g, uint32_t v, uint32_t* src,
                          uint32_t* edge) {
    double r = orc_u01(orc_prg_next(state)); /* exactly one draw, graph.hpp:63 */
    uint64_t lo = g->in_offsets[v];
    uint64_t hi = g->in_offsets[v + 1];
    if (lo == hi || r >= g->in_cum[hi - 1]) return 0; /* graph.hpp:66 */
    if (hi - lo <= 16) {                               /* graph.hpp:67-70 */
        while (g->in_cum[lo] <= r) ++lo;
    } else { /* first cumulative entry > r, graph.hpp:72-78 */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (g->in_cum[mid] > r)
                hi = mid;
            else
                lo = mid + 1;
        }
    }
    *src = g->in_src[lo];
    *edge = (uint32_t)lo;
    return 1;
}

/* ------------------------------------------------------------------------------------------
 * one walk attempt — proj/src/sampler.cpp:16-204
 * ---------------------------------------------------------------------------------------- */

typedef struct { /* WalkCursor, sampler.cpp:16-62 */
    uint64_t s;
    uint32_t node;
    uint32_t edges;
} cursor;

/* WalkCursor::start, sampler.cpp:21-37: uniform over all nodes, or over the start domain */
static int cursor_start(cursor* c, const orc_graph* g, uint64_t* draws) {
    if (g->domain && g->ndomain) { /* sampler.cpp:26-31 */
        double r = orc_u01(orc_prg_next(&c->s));
        uint64_t idx = (uint64_t)(r * (double)g->ndomain);
        if (idx >= g->ndomain) idx = g->ndomain - 1;
        c->node = g->domain[idx];
    } else {
        c->node = orc_pick_uniform_node(&c->s, g->n);
    }
    ++*draws;
    if (g->p_of[c->node] > 0.0) {
        double r = orc_u01(orc_prg_next(&c->s));
        ++*draws;
        if (r <= g->p_of[c->node]) return 1; /* length-0 hit */
    }
    return 0;
}

/* WalkCursor::advance_edge, sampler.cpp:41-49. 0 stepped, 1 no edge, 2 length cap */
static int cursor_advance(cursor* c, const orc_graph* g, uint32_t* u, uint32_t* e, uint64_t len_cap,
                          uint64_t* draws, uint64_t* steps, uint64_t* bytes) {
    if (c->edges >= len_cap) return 2;
    uint64_t d = g->in_offsets[c->node + 1] - g->in_offsets[c->node];
    int ok = orc_pick_live_in_edge(&c->s, g, c->node, u, e);
    ++*draws;
    ++*steps;
    *bytes += pick_bytes(d, ok);
    return ok ? 0 : 1;
}

/* WalkCursor::resolve, sampler.cpp:53-61 */
static int cursor_resolve(cursor* c, const orc_graph* g, uint32_t u, uint64_t* draws,
                          uint64_t* bytes) {
    ++c->edges;
    *bytes += 8; /* p_of[u] */
    if (g->p_of[u] > 0.0) {
        double r = orc_u01(orc_prg_next(&c->s));
        ++*draws;
        if (r <= g->p_of[u]) return 1;
    }
    c->node = u;
    return 0;
}

typedef struct { /* WindowFilter, sampler.cpp:65-86 */
    uint32_t ring[8];
    uint32_t size, pos;
} window_t;

static void win_push(window_t* w, uint32_t u) {
    if (w->size == 0) return;
    w->ring[w->pos] = u;
    w->pos = (w->pos + 1) % w->size;
}
static void win_reset(window_t* w, uint32_t width, uint32_t v0) {
    w->size = width > 8 ? 8 : width;
    for (uint32_t i = 0; i < w->size; ++i) w->ring[i] = ORC_INVALID_NODE;
    w->pos = 0;
    win_push(w, v0);
}
static int win_contains(const window_t* w, uint32_t u) {
    for (uint32_t i = 0; i < w->size; ++i)
        if (w->ring[i] == u) return 1;
    return 0;
}

typedef struct { /* BrentState, sampler.cpp:90-109 */
    uint32_t anchor, power, lam;
} brent_t;

static int brent_check(brent_t* b, uint32_t u) {
    if (u == b->anchor) return 1;
    if (++b->lam == b->power) {
        b->anchor = u;
        b->power <<= 1;
        b->lam = 0;
    }
    return 0;
}

orc_attempt_result orc_attempt(const orc_graph* g, uint64_t* state, int heuristic, uint32_t window,
                               uint64_t len_cap) {
    orc_attempt_result res;
    memset(&res, 0, sizeof res);
    uint64_t snapshot = *state; /* sampler.cpp:155 */
    cursor hare = {*state, ORC_INVALID_NODE, 0};
    res.alg_bytes += 8; /* start-node p_of */
    if (cursor_start(&hare, g, &res.draws)) { /* sampler.cpp:157-164 */
        res.accepted = 1;
        res.len = 0;
        *state = hare.s;
        return res;
    }
    window_t win;
    win_reset(&win, window, hare.node); /* sampler.cpp:166-167 */
    brent_t brent = {hare.node, 1, 0};  /* sampler.cpp:168-169, 95-99 */
    /* FloydState, sampler.cpp:113-138: second cursor replaying the stream from the snapshot */
    cursor tortoise = {snapshot, ORC_INVALID_NODE, 0};
    uint64_t hare_pos = 0, scratch = 0;
    if (heuristic == 1) (void)cursor_start(&tortoise, g, &scratch);

    for (;;) { /* sampler.cpp:174-201 */
        uint32_t u = ORC_INVALID_NODE, e = 0;
        if (cursor_advance(&hare, g, &u, &e, len_cap, &res.draws, &res.steps, &res.alg_bytes) != 0)
            break; /* no edge or length cap */
        int cyc = win_contains(&win, u);
        if (!cyc && heuristic == 0) cyc = brent_check(&brent, u);
        if (!cyc && heuristic == 1) {
            ++hare_pos;
            if (hare_pos % 2 == 0) {
                uint32_t tu = ORC_INVALID_NODE, te = 0;
                (void)cursor_advance(&tortoise, g, &tu, &te, len_cap, &scratch, &scratch, &scratch);
                (void)cursor_resolve(&tortoise, g, tu, &scratch, &scratch);
                cyc = tortoise.node == u;
            }
        }
        if (cyc) {
            res.cycle_flagged = 1;
            break;
        }
        if (cursor_resolve(&hare, g, u, &res.draws, &res.alg_bytes)) {
            res.accepted = 1;
            res.len = hare.edges;
            break;
        }
        if (g->allowed && !g->allowed[u]) { /* sampler.cpp:196-199: continuing needs u's adjacency */
            res.crossed = 1;
            break;
        }
        win_push(&win, u);
    }
    *state = hare.s; /* sampler.cpp:202 */
    return res;
}

/* thread_sample, sampler.cpp:267-290; with a restriction in g also sample_batch_restricted's
 * attempt loop (sampler.cpp:520-536): *crossings counts the attempts that left the allowed set */
static uint32_t thread_sample_x(const orc_graph* g, uint64_t worker_id, uint32_t l,
                                const orc_cfg* cfg, uint64_t* seeds, uint32_t* lens,
                                uint64_t* stats4, uint64_t* crossings);
uint32_t orc_thread_sample(const orc_graph* g, uint64_t worker_id, uint32_t l, const orc_cfg* cfg,
                           uint64_t* seeds, uint32_t* lens, uint64_t* stats4) {
    return thread_sample_x(g, worker_id, l, cfg, seeds, lens, stats4, NULL);
}
static uint32_t thread_sample_x(const orc_graph* g, uint64_t worker_id, uint32_t l,
                                const orc_cfg* cfg, uint64_t* seeds, uint32_t* lens,
                                uint64_t* stats4, uint64_t* crossings) {
    uint64_t s = orc_seed_from_worker(worker_id);
    for (int i = 0; i < 8; ++i) (void)orc_prg_next(&s); /* burn-in */
    uint32_t count = 0;
    for (uint32_t i = 0; i < l; ++i) {
        uint64_t snapshot = s;
        orc_attempt_result r = orc_attempt(g, &s, cfg->heuristic, cfg->window, g->n);
        if (stats4) {
            stats4[0] += 1;
            stats4[1] += r.draws;
            stats4[2] += r.steps;
            stats4[3] += r.alg_bytes;
        }
        if (crossings && r.crossed) ++*crossings;
        if (r.accepted) {
            seeds[count] = snapshot;
            lens[count] = r.len;
            ++count;
        }
    }
    return count;
}

/* DecodeContext::decode_restricted with an empty domain, sampler.cpp:299-338 */
int orc_decode(const orc_graph* g, uint64_t seed, uint32_t len, uint32_t* mark, uint32_t epoch,
               uint32_t* nodes, uint32_t* edges) {
    if (seed == 0) return -2;
    cursor c = {seed, ORC_INVALID_NODE, 0};
    uint64_t scratch = 0;
    int start_hit = cursor_start(&c, g, &scratch);
    uint32_t nn = 0;
    nodes[nn++] = c.node;
    if (start_hit) return len != 0 ? -2 : 1;
    if (len == 0) return -2;
    mark[c.node] = epoch;
    for (;;) {
        uint32_t u = ORC_INVALID_NODE, e = 0;
        if (cursor_advance(&c, g, &u, &e, g->n, &scratch, &scratch, &scratch) != 0) return -2;
        if (mark[u] == epoch) return 0; /* missed cycle */
        int hit = cursor_resolve(&c, g, u, &scratch, &scratch);
        nodes[nn++] = u;
        edges[nn - 2] = e;
        if (hit) return c.edges != len ? -2 : 1;
        if (c.edges >= len) return -2;
        mark[u] = epoch;
    }
}

/* ------------------------------------------------------------------------------------------
 * stream / pool — proj/src/sampler.cpp:383-501
 * Batches are worker ids seed+0, seed+1, ...; samples are kept in (batch, seq) order and the pool
 * is cut at the first whole-batch prefix reaching the target (:472-493). The reference's round
 * sizing (:406-421) is "only a speed knob", so the restatement simply walks batch by batch.
 * ---------------------------------------------------------------------------------------- */

struct orc_pool {
    uint64_t nsamples, attempts, total_edges;
    uint64_t cap_samples, cap_items;
    uint64_t* edge_off; /* nsamples+1 */
    uint32_t* nodes;    /* total_edges + nsamples */
    uint32_t* edges;    /* total_edges */
    uint64_t* tag_worker;
    uint32_t* tag_seq;
    /* full stream bookkeeping for orc_interdict */
    uint64_t nbatches, cap_batches;
    uint64_t* accepted_after_batch;
    uint64_t* crossed_after_batch; /* restricted sampling: cumulative crossings per batch */
};

static void pool_reserve(orc_pool* p, uint64_t more_samples, uint64_t more_items) {
    if (p->nsamples + more_samples + 1 > p->cap_samples) {
        uint64_t c = p->cap_samples ? p->cap_samples : 1024;
        while (c < p->nsamples + more_samples + 1) c *= 2;
        p->edge_off = realloc(p->edge_off, c * 8);
        p->tag_worker = realloc(p->tag_worker, c * 8);
        p->tag_seq = realloc(p->tag_seq, c * 4);
        p->cap_samples = c;
    }
    uint64_t need = p->total_edges + p->nsamples + more_items + more_samples;
    if (need > p->cap_items) {
        uint64_t c = p->cap_items ? p->cap_items : 4096;
        while (c < need) c *= 2;
        p->nodes = realloc(p->nodes, c * 4);
        p->edges = realloc(p->edges, c * 4);
        p->cap_items = c;
    }
}

typedef struct {
    const orc_graph* g;
    orc_cfg cfg;
    uint64_t seed;
    uint32_t* mark;
    uint32_t epoch;
    uint64_t* enc_seed;
    uint32_t* enc_len;
    uint32_t* tmp_nodes;
    uint32_t* tmp_edges;
    uint64_t tmp_cap;
    orc_pool* pool;
} stream_t;

static int stream_init(stream_t* st, const orc_graph* g, uint64_t seed, const orc_cfg* cfg) {
    memset(st, 0, sizeof *st);
    st->g = g;
    st->cfg = *cfg;
    st->seed = seed;
    st->mark = calloc(g->n ? g->n : 1, 4);
    st->enc_seed = malloc(8ull * (cfg->batch_size ? cfg->batch_size : 1));
    st->enc_len = malloc(4ull * (cfg->batch_size ? cfg->batch_size : 1));
    st->pool = calloc(1, sizeof(orc_pool));
    return 0;
}

static void stream_free(stream_t* st, int keep_pool) {
    free(st->mark);
    free(st->enc_seed);
    free(st->enc_len);
    free(st->tmp_nodes);
    free(st->tmp_edges);
    if (!keep_pool) orc_pool_free(st->pool);
}

/* one batch = thread_sample + immediate decode, sampler.cpp:430-439, merged :452-460 */
static int stream_one_batch(stream_t* st) {
    orc_pool* p = st->pool;
    uint64_t wid = st->seed + p->nbatches;
    uint64_t crossings = 0;
    uint32_t cnt = thread_sample_x(st->g, wid, st->cfg.batch_size, &st->cfg, st->enc_seed,
                                   st->enc_len, NULL, &crossings);
    for (uint32_t i = 0; i < cnt; ++i) {
        uint64_t need = (uint64_t)st->enc_len[i] + 1;
        if (need > st->tmp_cap) {
            st->tmp_cap = need * 2;
            st->tmp_nodes = realloc(st->tmp_nodes, st->tmp_cap * 4);
            st->tmp_edges = realloc(st->tmp_edges, st->tmp_cap * 4);
        }
        if (++st->epoch == 0) { /* sampler.cpp:301-304 */
            memset(st->mark, 0, 4ull * st->g->n);
            st->epoch = 1;
        }
        int rc = orc_decode(st->g, st->enc_seed[i], st->enc_len[i], st->mark, st->epoch,
                            st->tmp_nodes, st->tmp_edges);
        if (rc < 0) return 2;
        if (rc == 0) continue; /* dropped by the exact recheck */
        uint32_t len = st->enc_len[i];
        pool_reserve(p, 1, len);
        uint64_t eo = p->total_edges, w = p->nsamples;
        p->edge_off[w] = eo;
        memcpy(p->nodes + eo + w, st->tmp_nodes, 4ull * (len + 1));
        memcpy(p->edges + eo, st->tmp_edges, 4ull * len);
        p->tag_worker[w] = wid;
        p->tag_seq[w] = i; /* seq assigned before decode drops, sampler.cpp:283-284 */
        p->total_edges += len;
        p->nsamples += 1;
        p->edge_off[p->nsamples] = p->total_edges;
    }
    if (p->nbatches + 1 > p->cap_batches) {
        p->cap_batches = p->cap_batches ? p->cap_batches * 2 : 1024;
        p->accepted_after_batch = realloc(p->accepted_after_batch, p->cap_batches * 8);
        p->crossed_after_batch = realloc(p->crossed_after_batch, p->cap_batches * 8);
    }
    p->crossed_after_batch[p->nbatches] =
        (p->nbatches ? p->crossed_after_batch[p->nbatches - 1] : 0) + crossings;
    p->accepted_after_batch[p->nbatches++] = p->nsamples;
    return 0;
}

/* SampleStream::ensure, sampler.cpp:388-463: grows until min_accepted samples exist; the attempt
 * budget allows floor(max_attempts / batch_size) batches in total, then SamplingError (:396-404). */
static int stream_ensure(stream_t* st, uint64_t min_accepted) {
    orc_pool* p = st->pool;
    pool_reserve(p, 0, 0);
    if (p->nsamples == 0) p->edge_off[0] = 0;
    while (p->nsamples < min_accepted) {
        uint64_t attempts_so_far = p->nbatches * st->cfg.batch_size;
        uint64_t budget_left =
            st->cfg.max_attempts > attempts_so_far ? st->cfg.max_attempts - attempts_so_far : 0;
        if (st->cfg.batch_size == 0 || budget_left / st->cfg.batch_size == 0) return 3;
        int rc = stream_one_batch(st);
        if (rc) return rc;
    }
    return 0;
}

/* counters_for, sampler.cpp:472-482 */
static int stream_counters(const stream_t* st, uint64_t min_accepted, uint64_t* attempts,
                           uint64_t* accepted) {
    const orc_pool* p = st->pool;
    if (min_accepted == 0) {
        *attempts = 0;
        *accepted = 0;
        return 0;
    }
    for (uint64_t b = 0; b < p->nbatches; ++b) { /* lower_bound over the cumulative counts */
        if (p->accepted_after_batch[b] >= min_accepted) {
            *attempts = (b + 1) * st->cfg.batch_size;
            *accepted = p->accepted_after_batch[b];
            return 0;
        }
    }
    return 4;
}

/* stream_samples = ensure + to_pool, sampler.cpp:484-501 */
int orc_stream_samples(const orc_graph* g, uint64_t target, uint64_t seed, const orc_cfg* cfg,
                       orc_pool** out) {
    stream_t st;
    stream_init(&st, g, seed, cfg);
    int rc = stream_ensure(&st, target);
    if (rc) {
        stream_free(&st, 0);
        return rc;
    }
    uint64_t attempts = 0, accepted = 0;
    stream_counters(&st, target, &attempts, &accepted);
    orc_pool* p = st.pool;
    /* to_pool keeps all samples of the minimal whole-batch prefix; ensure() here never runs past
     * that prefix, so accepted == nsamples. */
    p->attempts = attempts;
    p->nsamples = accepted;
    p->total_edges = p->edge_off[accepted];
    stream_free(&st, 1);
    *out = p;
    return 0;
}

/* one part of distributed_sample, partition.cpp:183-268 */
int orc_part_sample(const orc_graph* g, uint64_t target, uint64_t first_worker, const orc_cfg* cfg,
                    orc_pool** out, uint64_t* crossings, uint64_t* attempts) {
    stream_t st;
    stream_init(&st, g, first_worker, cfg);
    int rc = stream_ensure(&st, target);
    if (rc) {
        stream_free(&st, 0);
        return rc;
    }
    orc_pool* p = st.pool;
    uint64_t att = 0, acc = 0;
    *crossings = 0;
    if (target > 0) { /* cut at the minimal batch prefix reaching the quota, :245-262 */
        stream_counters(&st, target, &att, &acc);
        *crossings = p->crossed_after_batch[att / cfg->batch_size - 1];
    }
    p->attempts = att;
    p->nsamples = acc;
    p->total_edges = acc ? p->edge_off[acc] : 0;
    *attempts = att;
    stream_free(&st, 1);
    *out = p;
    return 0;
}

void orc_pool_stats(const orc_pool* p, uint64_t* nsamples, uint64_t* attempts,
                    uint64_t* total_edges) {
    *nsamples = p->nsamples;
    *attempts = p->attempts;
    *total_edges = p->total_edges;
}

void orc_pool_copy(const orc_pool* p, uint64_t* edge_off, uint32_t* nodes, uint32_t* edges,
                   uint64_t* tag_worker, uint32_t* tag_seq) {
    memcpy(edge_off, p->edge_off, 8 * (p->nsamples + 1));
    memcpy(nodes, p->nodes, 4 * (p->total_edges + p->nsamples));
    memcpy(edges, p->edges, 4 * p->total_edges);
    if (tag_worker) memcpy(tag_worker, p->tag_worker, 8 * p->nsamples);
    if (tag_seq) memcpy(tag_seq, p->tag_seq, 4 * p->nsamples);
}

void orc_pool_free(orc_pool* p) {
    if (!p) return;
    free(p->edge_off);
    free(p->nodes);
    free(p->edges);
    free(p->tag_worker);
    free(p->tag_seq);
    free(p->accepted_after_batch);
    free(p->crossed_after_batch);
    free(p);
}

/* ------------------------------------------------------------------------------------------
 * coverage index + greedy — proj/src/coverage.cpp:13-166
 * ---------------------------------------------------------------------------------------- */

typedef struct {
    uint32_t limit;
    uint64_t nsets;
    uint8_t* is_cand;    /* limit */
    uint32_t* cands;     /* ascending candidate ids, coverage.cpp:55-57 */
    uint64_t ncands;
    uint64_t* by_off;    /* limit+1: item -> sample ids (CSR form of by_item_) */
    uint32_t* by_sample; /* in insertion (sample id) order, like push_back at :33 */
} cov_index;

static void cov_free(cov_index* ix) {
    free(ix->is_cand);
    free(ix->cands);
    free(ix->by_off);
    free(ix->by_sample);
}

/* CoverageIndex raw item-set constructor, coverage.cpp:60-74 (candidate_mask :13-27).
 * status 2 when a candidate id is out of range (:18-20). */
static int cov_build(cov_index* ix, uint32_t limit, uint64_t nsets, const uint64_t* set_off,
                     const uint32_t* items, const uint32_t* cand_ids, uint64_t ncand) {
    memset(ix, 0, sizeof *ix);
    ix->limit = limit;
    ix->nsets = nsets;
    ix->is_cand = calloc(limit ? limit : 1, 1);
    if (cand_ids) {
        for (uint64_t i = 0; i < ncand; ++i) {
            if (cand_ids[i] >= limit) {
                cov_free(ix);
                return 2;
            }
            ix->is_cand[cand_ids[i]] = 1;
        }
    } else {
        memset(ix->is_cand, 1, limit);
    }
    ix->by_off = calloc((uint64_t)limit + 2, 8);
    for (uint64_t s = 0; s < nsets; ++s)
        for (uint64_t j = set_off[s]; j < set_off[s + 1]; ++j)
            if (items[j] < limit && ix->is_cand[items[j]]) ix->by_off[items[j] + 1]++;
    for (uint64_t i = 0; i < limit; ++i) ix->by_off[i + 1] += ix->by_off[i];
    ix->by_sample = malloc(4 * (ix->by_off[limit] ? ix->by_off[limit] : 1));
    uint64_t* fill = malloc(8 * ((uint64_t)limit + 1));
    memcpy(fill, ix->by_off, 8 * ((uint64_t)limit + 1));
    for (uint64_t s = 0; s < nsets; ++s)
        for (uint64_t j = set_off[s]; j < set_off[s + 1]; ++j)
            if (items[j] < limit && ix->is_cand[items[j]])
                ix->by_sample[fill[items[j]]++] = (uint32_t)s;
    free(fill);
    ix->cands = malloc(4 * ((uint64_t)limit ? limit : 1));
    for (uint32_t i = 0; i < limit; ++i)
        if (ix->is_cand[i]) ix->cands[ix->ncands++] = i;
    return 0;
}

/* coverage_of, coverage.cpp:76-89 */
static uint64_t cov_coverage_of(const cov_index* ix, const uint32_t* q, uint64_t nq) {
    uint8_t* covered = calloc(ix->nsets ? ix->nsets : 1, 1);
    uint64_t count = 0;
    for (uint64_t i = 0; i < nq; ++i) {
        uint32_t item = q[i];
        if (item >= ix->limit) continue;
        for (uint64_t j = ix->by_off[item]; j < ix->by_off[item + 1]; ++j) {
            uint32_t sid = ix->by_sample[j];
            if (!covered[sid]) {
                covered[sid] = 1;
                ++count;
            }
        }
    }
    free(covered);
    return count;
}

/* greedy_max_cover_naive, coverage.cpp:140-166 */
static void greedy_naive(const cov_index* ix, uint32_t k, uint32_t* solution, uint64_t* coverage) {
    uint8_t* covered = calloc(ix->nsets ? ix->nsets : 1, 1);
    uint8_t* selected = calloc((uint64_t)ix->limit + 1, 1);
    uint64_t cov = 0;
    for (uint32_t iter = 0; iter < k; ++iter) {
        uint64_t best_gain = 0;
        uint32_t best_item = ORC_INVALID_NODE;
        for (uint64_t c = 0; c < ix->ncands; ++c) {
            uint32_t item = ix->cands[c];
            if (selected[item]) continue;
            uint64_t gain = 0;
            for (uint64_t j = ix->by_off[item]; j < ix->by_off[item + 1]; ++j)
                if (!covered[ix->by_sample[j]]) ++gain;
            if (best_item == ORC_INVALID_NODE || gain > best_gain) { /* first max wins, :155 */
                best_gain = gain;
                best_item = item;
            }
        }
        solution[iter] = best_item;
        selected[best_item] = 1;
        cov += best_gain;
        for (uint64_t j = ix->by_off[best_item]; j < ix->by_off[best_item + 1]; ++j)
            covered[ix->by_sample[j]] = 1;
    }
    *coverage = cov;
    free(covered);
    free(selected);
}

/* greedy_max_cover (CELF), coverage.cpp:91-138: max-heap on (gain desc, item asc) with stamps */
typedef struct {
    uint64_t gain;
    uint32_t item, stamp;
} heap_entry;

static int entry_worse(const heap_entry* a, const heap_entry* b) { /* Worse, :101-106 */
    if (a->gain != b->gain) return a->gain < b->gain;
    return a->item > b->item;
}
static void heap_push(heap_entry* h, uint64_t* n, heap_entry e) {
    uint64_t i = (*n)++;
    h[i] = e;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (!entry_worse(&h[p], &h[i])) break;
        heap_entry t = h[p];
        h[p] = h[i];
        h[i] = t;
        i = p;
    }
}
static heap_entry heap_pop(heap_entry* h, uint64_t* n) {
    heap_entry top = h[0];
    h[0] = h[--(*n)];
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, best = i;
        if (l < *n && entry_worse(&h[best], &h[l])) best = l;
        if (r < *n && entry_worse(&h[best], &h[r])) best = r;
        if (best == i) break;
        heap_entry t = h[best];
        h[best] = h[i];
        h[i] = t;
        i = best;
    }
    return top;
}

static void greedy_lazy(const cov_index* ix, uint32_t k, uint32_t* solution, uint64_t* coverage) {
    heap_entry* heap = malloc(sizeof(heap_entry) * (ix->ncands + (uint64_t)k + 1));
    uint64_t hn = 0;
    for (uint64_t c = 0; c < ix->ncands; ++c) {
        uint32_t item = ix->cands[c];
        heap_entry e = {ix->by_off[item + 1] - ix->by_off[item], item, 0};
        heap_push(heap, &hn, e);
    }
    uint8_t* covered = calloc(ix->nsets ? ix->nsets : 1, 1);
    uint8_t* selected = calloc((uint64_t)ix->limit + 1, 1);
    uint64_t cov = 0;
    for (uint32_t iter = 0; iter < k; ++iter) {
        for (;;) {
            heap_entry top = heap_pop(heap, &hn);
            if (selected[top.item]) continue;
            if (top.stamp != iter) {
                uint64_t gain = 0;
                for (uint64_t j = ix->by_off[top.item]; j < ix->by_off[top.item + 1]; ++j)
                    if (!covered[ix->by_sample[j]]) ++gain;
                heap_entry e = {gain, top.item, iter};
                heap_push(heap, &hn, e);
                continue;
            }
            solution[iter] = top.item;
            selected[top.item] = 1;
            cov += top.gain;
            for (uint64_t j = ix->by_off[top.item]; j < ix->by_off[top.item + 1]; ++j)
                covered[ix->by_sample[j]] = 1;
            break;
        }
    }
    *coverage = cov;
    free(heap);
    free(covered);
    free(selected);
}

int orc_greedy(uint32_t limit, uint64_t nsets, const uint64_t* set_off, const uint32_t* items,
               const uint32_t* cand_ids, uint64_t ncand, uint32_t k, int lazy, uint32_t* solution,
               uint64_t* coverage) {
    cov_index ix;
    int rc = cov_build(&ix, limit, nsets, set_off, items, cand_ids, ncand);
    if (rc) return rc;
    if (k > ix.ncands) { /* coverage.cpp:93-94 / :142-143 */
        cov_free(&ix);
        return 1;
    }
    if (lazy)
        greedy_lazy(&ix, k, solution, coverage);
    else
        greedy_naive(&ix, k, solution, coverage);
    cov_free(&ix);
    return 0;
}

int orc_coverage_of(uint32_t limit, uint64_t nsets, const uint64_t* set_off, const uint32_t* items,
                    const uint32_t* cand_ids, uint64_t ncand, const uint32_t* query,
                    uint64_t nquery, uint64_t* coverage) {
    cov_index ix;
    int rc = cov_build(&ix, limit, nsets, set_off, items, cand_ids, ncand);
    if (rc) return rc;
    *coverage = cov_coverage_of(&ix, query, nquery);
    cov_free(&ix);
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * schedule + check — proj/src/coverage.cpp:168-231
 * ---------------------------------------------------------------------------------------- */

/* ln_choose, coverage.cpp:168-173 */
double orc_ln_choose(uint64_t M, uint64_t k) {
    double s = 0.0;
    for (uint64_t i = 1; i <= k; ++i) s += log((double)(M - k + i) / (double)i);
    return s;
}

/* compute_schedule_m, coverage.cpp:179-204; lambda_samples :175-177 */
int orc_schedule_m(uint64_t M, uint32_t k, double epsilon, double delta, orc_schedule* s) {
    if (!(epsilon > 0.0) || epsilon >= 1.0) return 1;
    if (!(delta > 0.0) || delta >= 1.0) return 1;
    if (k < 1 || k > M) return 1;
    s->epsilon = epsilon;
    s->delta = delta;
    s->k = k;
    double c = (2.0 - 1.0 / exp(1.0)) * (2.0 - 1.0 / exp(1.0));
    double a = 2.0 + 2.0 * epsilon / 3.0;
    double eps2 = epsilon * epsilon;
    s->n_max = c * a * (double)M * (log(6.0 / delta) + orc_ln_choose(M, k)) / ((double)k * eps2);
    double lambda0 = a * log(3.0 / delta) / eps2;
    double t = ceil(log2(2.0 * s->n_max / lambda0));
    s->t_max = t < 1.0 ? 1 : (uint32_t)t;
    s->lambda = a * log(3.0 * s->t_max / delta) / eps2;
    s->lambda1 = 1.0 + (1.0 + epsilon) * a * log(3.0 * s->t_max / delta) / eps2;
    s->lambda_samples = (uint64_t)ceil(s->lambda);
    return 0;
}

/* check_solution, coverage.cpp:212-231 (coverage counts supplied by the caller) */
int orc_check(double cov_r, double cov_rp, double n_rp, const orc_schedule* sched, uint32_t t,
              double* eps_t_out) {
    if (cov_rp < sched->lambda1) {
        *eps_t_out = INFINITY;
        return 0;
    }
    double eps = sched->epsilon;
    double pow2 = ldexp(1.0, (int)t - 1);
    double one_me = 1.0 - 1.0 / exp(1.0);
    double eps1 = cov_r / cov_rp - 1.0;
    double eps2 = eps * sqrt(n_rp * (1.0 + eps) / (pow2 * cov_rp));
    double eps3 =
        eps * sqrt(n_rp * (1.0 + eps) * (one_me - eps) / ((1.0 + eps / 3.0) * pow2 * cov_rp));
    double eps_t = (eps1 + eps2 + eps1 * eps2) * (one_me - eps) + one_me * eps3;
    *eps_t_out = eps_t;
    return eps_t <= eps;
}

/* ------------------------------------------------------------------------------------------
 * interdiction — proj/src/interdiction.cpp:12-87
 * ---------------------------------------------------------------------------------------- */

/* item sets of samples [off, off+cnt): edge ids (kind 0, coverage.cpp:50) or all nodes incl.
 * start and hit (kind 1, coverage.cpp:52), as CSR over a fresh copy. */
static void slice_sets(const orc_pool* p, int kind, uint64_t off, uint64_t cnt, uint64_t** set_off,
                       uint32_t** items) {
    uint64_t* so = malloc(8 * (cnt + 1));
    uint64_t total = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        uint64_t w = off + i, len = p->edge_off[w + 1] - p->edge_off[w];
        so[i] = total;
        total += kind == 0 ? len : len + 1;
    }
    so[cnt] = total;
    uint32_t* it = malloc(4 * (total ? total : 1));
    for (uint64_t i = 0; i < cnt; ++i) {
        uint64_t w = off + i, len = p->edge_off[w + 1] - p->edge_off[w];
        if (kind == 0)
            memcpy(it + so[i], p->edges + p->edge_off[w], 4 * len);
        else
            memcpy(it + so[i], p->nodes + p->edge_off[w] + w, 4 * (len + 1));
    }
    *set_off = so;
    *items = it;
}

int orc_interdict(const orc_graph* g, int kind, const uint32_t* cand_ids, uint64_t ncand,
                  uint32_t k, double eps, double delta, uint64_t seed, const orc_cfg* cfg,
                  orc_result* out, uint32_t* solution) {
    uint32_t limit = kind == 0 ? g->m : g->n;
    /* CandidateSet::validate, proj/src/graph.cpp:432-443; k range, interdiction.cpp:17-18 */
    uint64_t csize = cand_ids ? ncand : limit;
    if (csize == 0) return 2;
    if (cand_ids) {
        uint8_t* seen = calloc(limit ? limit : 1, 1);
        for (uint64_t i = 0; i < ncand; ++i) {
            if (cand_ids[i] >= limit || seen[cand_ids[i]]) {
                free(seen);
                return 2;
            }
            seen[cand_ids[i]] = 1;
        }
        free(seen);
    }
    if (k < 1 || k > csize) return 1;
    orc_schedule sched;
    int rc = orc_schedule_m(limit, k, eps, delta, &sched); /* compute_schedule, :206-210 */
    if (rc) return rc;
    uint64_t lam = sched.lambda_samples;

    stream_t st;
    stream_init(&st, g, seed, cfg);
    uint64_t size = 0, coverage = 0;
    uint32_t t = 0;
    int pass = 0;
    for (;;) { /* interdiction.cpp:36-47 */
        ++t;
        size = lam << (t - 1);
        rc = stream_ensure(&st, 2 * size);
        if (rc) {
            stream_free(&st, 0);
            return rc;
        }
        uint64_t *off_r, *off_rp;
        uint32_t *it_r, *it_rp;
        slice_sets(st.pool, kind, 0, size, &off_r, &it_r);
        slice_sets(st.pool, kind, size, size, &off_rp, &it_rp);
        rc = orc_greedy(limit, size, off_r, it_r, cand_ids, ncand, k, 1, solution, &coverage);
        uint64_t cov_r = 0, cov_rp = 0;
        if (!rc) rc = orc_coverage_of(limit, size, off_r, it_r, cand_ids, ncand, solution, k, &cov_r);
        if (!rc)
            rc = orc_coverage_of(limit, size, off_rp, it_rp, cand_ids, ncand, solution, k, &cov_rp);
        free(off_r);
        free(it_r);
        free(off_rp);
        free(it_rp);
        if (rc) {
            stream_free(&st, 0);
            return rc;
        }
        double eps_t;
        pass = orc_check((double)cov_r, (double)cov_rp, (double)size, &sched, t, &eps_t);
        if (pass || (double)size >= sched.n_max) break;
    }
    uint64_t attempts = 0, accepted = 0;
    stream_counters(&st, 2 * size, &attempts, &accepted); /* interdiction.cpp:54-55 */
    out->k = k;
    out->iterations = t;
    out->coverage = coverage;
    out->samples_used = 2 * size;
    out->attempts = attempts;
    out->passed_check = pass;
    double influence = (double)g->n * (double)accepted / (double)attempts; /* :57-59 */
    out->est_suspension = influence * (double)coverage / (double)size;     /* :60-61 */
    stream_free(&st, 0);
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * paired LT forward simulation — proj/src/evaluation.cpp:19-108,195-242
 * ---------------------------------------------------------------------------------------- */

#define ORC_NO_EDGE 0xFFFFFFFFu

typedef struct { /* SimContext, evaluation.cpp:20-46 */
    uint8_t* in_x;
    uint32_t* choice;
    uint8_t* node_gone;
    uint8_t* edge_gone;
    int8_t* status;
    uint32_t* stack;
} sim_ctx;

static int sim_init(sim_ctx* c, const orc_graph* g) {
    c->in_x = (uint8_t*)calloc(g->n ? g->n : 1, 1);
    c->choice = (uint32_t*)malloc(sizeof(uint32_t) * (g->n ? g->n : 1));
    c->node_gone = (uint8_t*)calloc(g->n ? g->n : 1, 1);
    c->edge_gone = (uint8_t*)calloc(g->m ? g->m : 1, 1);
    c->status = (int8_t*)malloc(g->n ? g->n : 1);
    c->stack = (uint32_t*)malloc(sizeof(uint32_t) * (g->n ? g->n : 1));
    return c->in_x && c->choice && c->node_gone && c->edge_gone && c->status && c->stack;
}

static void sim_free(sim_ctx* c) {
    free(c->in_x); free(c->choice); free(c->node_gone); free(c->edge_gone);
    free(c->status); free(c->stack);
}

/* SimContext::set_removal, evaluation.cpp:35-45. edge_dst[e] is the row that holds slot e
 * (build_graph, graph.cpp:150-192), recovered here from the offsets. */
static void sim_set_removal(sim_ctx* c, const orc_graph* g, int kind, const uint32_t* ids,
                            uint64_t nids) {
    if (kind == 0) {
        for (uint64_t i = 0; i < nids; ++i) c->edge_gone[ids[i]] = 1;
    } else {
        for (uint64_t i = 0; i < nids; ++i) c->node_gone[ids[i]] = 1;
        for (uint32_t v = 0; v < g->n; ++v)
            for (uint64_t e = g->in_offsets[v]; e < g->in_offsets[v + 1]; ++e)
                if (c->node_gone[g->in_src[e]] || c->node_gone[v]) c->edge_gone[e] = 1;
    }
}

/* draw_realization, evaluation.cpp:49-59: members ascending (the nodes with p_of > 0,
 * SuspectSet::from_members graph.cpp:266-283), then one pick per node ascending. */
static void sim_draw(const orc_graph* g, uint64_t* state, sim_ctx* c) {
    memset(c->in_x, 0, g->n);
    for (uint32_t v = 0; v < g->n; ++v)
        if (g->p_of[v] != 0.0)
            if (orc_u01(orc_prg_next(state)) <= g->p_of[v]) c->in_x[v] = 1;
    for (uint32_t v = 0; v < g->n; ++v) {
        uint32_t src, e;
        c->choice[v] = orc_pick_live_in_edge(state, g, v, &src, &e) ? e : ORC_NO_EDGE;
    }
}

/* count_infected, evaluation.cpp:65-108 */
static uint32_t sim_count(const orc_graph* g, sim_ctx* c, int residual) {
    const int8_t kUnknown = -1, kInProgress = -2;
    memset(c->status, kUnknown, g->n);
    uint32_t count = 0;
    for (uint32_t v0 = 0; v0 < g->n; ++v0) {
        if (c->status[v0] >= 0) {
            count += (uint32_t)c->status[v0];
            continue;
        }
        uint64_t sp = 0;
        uint32_t cur = v0;
        int8_t verdict;
        for (;;) {
            if (c->status[cur] >= 0) { verdict = c->status[cur]; break; }
            if (c->status[cur] == kInProgress) { verdict = 0; break; }
            if (residual && c->node_gone[cur]) { verdict = 0; break; }
            if (c->in_x[cur]) { verdict = 1; break; }
            uint32_t e = c->choice[cur];
            if (e == ORC_NO_EDGE || (residual && c->edge_gone[e])) { verdict = 0; break; }
            c->status[cur] = kInProgress;
            c->stack[sp++] = cur;
            cur = g->in_src[e];
        }
        if (c->status[cur] < 0) c->status[cur] = verdict;
        for (uint64_t i = 0; i < sp; ++i) c->status[c->stack[i]] = verdict;
        count += (uint32_t)verdict;
    }
    return count;
}

/* lt_forward_simulate, evaluation.cpp:202-207 */
uint32_t orc_lt_forward_simulate(const orc_graph* g, uint64_t* state) {
    sim_ctx c;
    if (!sim_init(&c, g)) { sim_free(&c); return 0; }
    sim_draw(g, state, &c);
    uint32_t r = sim_count(g, &c, 0);
    sim_free(&c);
    return r;
}

/* rr_node_sets, evaluation.cpp:169-191 */
int orc_rr_node_sets(const orc_graph* g, uint64_t* state, uint32_t count, uint64_t* set_off,
                     uint32_t* items, uint64_t items_cap) {
    uint32_t* mark = calloc(g->n ? g->n : 1, 4);
    uint64_t at = 0;
    int rc = 0;
    set_off[0] = 0;
    for (uint32_t i = 1; i <= count && !rc; ++i) {
        uint32_t v = orc_pick_uniform_node(state, g->n);
        if (at >= items_cap) { rc = 5; break; }
        items[at++] = v;
        mark[v] = i;
        for (;;) {
            uint32_t u = 0, e = 0;
            if (!orc_pick_live_in_edge(state, g, v, &u, &e)) break;
            if (mark[u] == i) break;
            v = u;
            if (at >= items_cap) { rc = 5; break; }
            items[at++] = v;
            mark[v] = i;
        }
        set_off[i] = at;
    }
    free(mark);
    return rc;
}

static int removal_valid(const orc_graph* g, int kind, const uint32_t* ids, uint64_t nids) {
    uint32_t limit = kind == 0 ? g->m : g->n; /* RemovalSet::validate, evaluation.cpp:195-200 */
    for (uint64_t i = 0; i < nids; ++i)
        if (ids[i] >= limit) return 0;
    return 1;
}

/* The paired runs of the estimate_suspension loop body (evaluation.cpp:233-236) for a fixed
 * number of runs: full[i] / residual[i] of run i on one shared stream. status 0 / 2. */
int orc_paired_runs(const orc_graph* g, int kind, const uint32_t* ids, uint64_t nids,
                    uint64_t* state, uint64_t nruns, uint32_t* full, uint32_t* residual) {
    if (!removal_valid(g, kind, ids, nids)) return 2;
    sim_ctx c;
    if (!sim_init(&c, g)) { sim_free(&c); return 4; }
    sim_set_removal(&c, g, kind, ids, nids);
    for (uint64_t r = 0; r < nruns; ++r) {
        sim_draw(g, state, &c);
        full[r] = sim_count(g, &c, 0);
        residual[r] = sim_count(g, &c, 1);
    }
    sim_free(&c);
    return 0;
}

/* estimate_suspension, evaluation.cpp:209-242. status 0 ok, 1 invalid argument, 2 DataError. */
int orc_estimate_suspension(const orc_graph* g, int kind, const uint32_t* ids, uint64_t nids,
                            double epsilon, double delta, uint64_t* state, orc_suspension* out) {
    if (!(epsilon > 0.0) || epsilon >= 1.0) return 1;
    if (!(delta > 0.0) || delta >= 1.0) return 1;
    if (!removal_valid(g, kind, ids, nids)) return 2;
    out->value = 0.0; out->capped = 0; out->runs = 0;
    if (nids == 0) return 0; /* :218 */

    sim_ctx c;
    if (!sim_init(&c, g)) { sim_free(&c); return 4; }
    sim_set_removal(&c, g, kind, ids, nids);

    double upsilon = 4.0 * (exp(1.0) - 2.0) * log(2.0 / delta) * (1.0 + epsilon) /
                     (epsilon * epsilon);
    uint64_t members = 0;
    for (uint32_t v = 0; v < g->n; ++v) members += g->p_of[v] != 0.0;
    uint64_t draws_per_run = members + g->n;
    uint64_t max_runs = 1000000000ull / draws_per_run; /* kDrawCap, :17 */
    if (max_runs < 1) max_runs = 1;

    double sum = 0.0;
    uint64_t runs = 0;
    while (sum < upsilon) {
        if (runs >= max_runs) {
            out->value = 0.0; out->capped = 1; out->runs = runs;
            sim_free(&c);
            return 0;
        }
        sim_draw(g, state, &c);
        uint32_t full = sim_count(g, &c, 0);
        uint32_t residual = sim_count(g, &c, 1);
        sum += (double)(full - residual) / (double)g->n;
        ++runs;
    }
    out->value = (double)g->n * upsilon / (double)runs;
    out->capped = 0;
    out->runs = runs;
    sim_free(&c);
    return 0;
}
