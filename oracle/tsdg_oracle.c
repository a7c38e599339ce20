/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (see tsdg_oracle.h).  Plain-C restatement
 * of the reference search path; each function cites the reference lines it
 * follows (paths relative to /root/reference/proj).  Compiled with
 * -ffp-contract=off: every fp32 op rounds separately, as in the reference's
 * sequential addss chain (vectors.hpp:36-49).
 */
#include "tsdg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define INVALID_ID 0xFFFFFFFFu
#define SEG_W 32u
#define LANES 32u

/* ---- common.hpp:22-61 ------------------------------------------------------ */
typedef struct { uint32_t id; float dist; } IdDist;

static inline int closer(IdDist a, IdDist b) {             /* common.hpp:22-25 */
    if (a.dist != b.dist) return a.dist < b.dist;
    return a.id < b.id;
}
static inline IdDist sentinel(void) { IdDist e = {INVALID_ID, INFINITY}; return e; }

uint64_t tsdg_o_mix64(uint64_t z) {                          /* common.hpp:27-31 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t rng_next(uint64_t* s) {               /* common.hpp:39-42 */
    *s += 0x9E3779B97F4A7C15ULL;
    return tsdg_o_mix64(*s);
}
static inline uint32_t rng_below(uint64_t* s, uint32_t n) {  /* common.hpp:45-47 */
    return (uint32_t)(rng_next(s) % n);
}
uint64_t tsdg_o_fork(uint64_t state, uint64_t index) {       /* common.hpp:55-57 */
    return tsdg_o_mix64(state ^ (0xD1B54A32D192ED03ULL * (index + 1)));
}

/* ---- vectors.hpp:36-49, vectors.cpp:10-16,36-43 ---------------------------- */
float tsdg_o_distance(const float* a, const float* b, uint32_t d, int metric) {
    float acc = 0.0f;
    if (metric == 0) {
        for (uint32_t i = 0; i < d; ++i) {
            const float diff = a[i] - b[i];
            acc += diff * diff;
        }
        return acc;
    }
    for (uint32_t i = 0; i < d; ++i) acc += a[i] * b[i];
    return metric == 1 ? 1.0f - acc : -acc;
}

static inline float dist_row(const tsdg_o_graph* g, const float* q, uint32_t v) {
    return tsdg_o_distance(q, g->base + (size_t)v * g->d, g->d, g->metric);
}

/* ---- diversify.cpp:34-42: partition_point(lambda < cut) ----------------------- */
static uint64_t prefix_len(const tsdg_o_graph* g, uint32_t u, uint32_t cut) {
    uint64_t lo = g->offsets[u], hi = g->offsets[u + 1];
    const uint64_t begin = lo;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (g->lambdas[mid] < cut) lo = mid + 1; else hi = mid;
    }
    return lo - begin;
}

/* ---- segmented.cpp:8-61 SegmentedQueue ------------------------------------- */
typedef struct {
    uint32_t m;
    IdDist* slot;      /* m x 32 */
    uint32_t* size;    /* m */
    uint64_t total, evictions;
} Queue;

static int queue_init(Queue* q, uint32_t m) {
    q->m = m;
    q->slot = (IdDist*)malloc(sizeof(IdDist) * (size_t)m * SEG_W);
    q->size = (uint32_t*)calloc(m, sizeof(uint32_t));
    q->total = q->evictions = 0;
    return q->slot && q->size ? 0 : 2;
}
static void queue_free(Queue* q) { free(q->slot); free(q->size); }

static void queue_push(Queue* q, uint32_t id, float dist) {  /* segmented.cpp:13-34 */
    const uint32_t s = id % q->m;
    IdDist* seg = q->slot + (size_t)s * SEG_W;
    IdDist e = {id, dist};
    if (q->size[s] == SEG_W) {
        if (!closer(e, seg[q->size[s] - 1])) { q->evictions++; return; }
        q->size[s]--; q->total--; q->evictions++;
    }
    uint32_t pos = 0;                          /* upper_bound by closer */
    while (pos < q->size[s] && !closer(e, seg[pos])) pos++;
    for (uint32_t i = q->size[s]; i > pos; --i) seg[i] = seg[i - 1];
    seg[pos] = e;
    q->size[s]++; q->total++;
}

static int queue_pop_min(Queue* q, IdDist* out) {            /* segmented.cpp:36-53 */
    uint32_t best_idx = q->m;
    IdDist best = sentinel();
    for (uint32_t s = 0; s < q->m; ++s) {
        if (q->size[s] != 0 && closer(q->slot[(size_t)s * SEG_W], best)) {
            best = q->slot[(size_t)s * SEG_W];
            best_idx = s;
        }
    }
    if (best_idx == q->m) return 0;
    IdDist* seg = q->slot + (size_t)best_idx * SEG_W;
    for (uint32_t i = 1; i < q->size[best_idx]; ++i) seg[i - 1] = seg[i];
    q->size[best_idx]--; q->total--;
    *out = best;
    return 1;
}

static int queue_contains(const Queue* q, uint32_t id) {     /* segmented.cpp:55-61 */
    const uint32_t s = id % q->m;
    const IdDist* seg = q->slot + (size_t)s * SEG_W;
    for (uint32_t i = 0; i < q->size[s]; ++i) if (seg[i].id == id) return 1;
    return 0;
}

/* ---- segmented.cpp:63-87 SegmentedVisited ---------------------------------- */
typedef struct { uint32_t m; uint32_t* slot; uint32_t* size; uint32_t* oldest; } Visited;

static int visited_init(Visited* v, uint32_t m) {
    v->m = m;
    v->slot = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m * SEG_W);
    v->size = (uint32_t*)calloc(m, sizeof(uint32_t));
    v->oldest = (uint32_t*)calloc(m, sizeof(uint32_t));
    return v->slot && v->size && v->oldest ? 0 : 2;
}
static void visited_free(Visited* v) { free(v->slot); free(v->size); free(v->oldest); }

static void visited_add(Visited* v, uint32_t id) {           /* segmented.cpp:68-79 */
    const uint32_t s = id % v->m;
    uint32_t* seg = v->slot + (size_t)s * SEG_W;
    for (uint32_t i = 0; i < v->size[s]; ++i) if (seg[i] == id) return;
    if (v->size[s] < SEG_W) { seg[v->size[s]++] = id; return; }
    seg[v->oldest[s]] = id;
    v->oldest[s] = (v->oldest[s] + 1) % SEG_W;
}
static int visited_contains(const Visited* v, uint32_t id) { /* segmented.cpp:81-87 */
    const uint32_t s = id % v->m;
    const uint32_t* seg = v->slot + (size_t)s * SEG_W;
    for (uint32_t i = 0; i < v->size[s]; ++i) if (seg[i] == id) return 1;
    return 0;
}

/* ---- segmented.cpp:89-111 TopK ---------------------------------------------- */
typedef struct { uint32_t k, n; IdDist* e; } TopK;

static int topk_init(TopK* t, uint32_t k) {
    t->k = k; t->n = 0;
    t->e = (IdDist*)malloc(sizeof(IdDist) * ((size_t)k + 2));
    return t->e ? 0 : 2;
}
static int topk_push(TopK* t, uint32_t id, float dist) {     /* segmented.cpp:94-101 */
    for (uint32_t i = 0; i < t->n; ++i) if (t->e[i].id == id) return 0;
    IdDist e = {id, dist};
    uint32_t pos = 0;
    while (pos < t->n && !closer(e, t->e[pos])) pos++;
    for (uint32_t i = t->n; i > pos; --i) t->e[i] = t->e[i - 1];
    t->e[pos] = e;
    t->n++;
    return 1;
}
static IdDist topk_furthest(const TopK* t) {                 /* segmented.cpp:108-111 */
    return t->n ? t->e[t->n - 1] : sentinel();
}

/* ---- unbounded stand-ins (bestfirst_search.cpp:14-47) ------------------------
 * std::set<(dist,id)> + unordered_set: a sorted array + an open-addressing set. */
typedef struct { uint32_t* keys; uint64_t cap, n; } IdSet;
static int idset_init(IdSet* s, uint64_t cap) {
    s->cap = cap; s->n = 0;
    s->keys = (uint32_t*)malloc(sizeof(uint32_t) * cap);
    if (!s->keys) return 2;
    memset(s->keys, 0xFF, sizeof(uint32_t) * cap);
    return 0;
}
static uint64_t idset_slot(const IdSet* s, uint32_t id) {
    uint64_t h = (tsdg_o_mix64(id) % s->cap);
    while (s->keys[h] != INVALID_ID && s->keys[h] != id) h = (h + 1) % s->cap;
    return h;
}
static int idset_contains(const IdSet* s, uint32_t id) { return s->keys[idset_slot(s, id)] == id; }
static int idset_grow(IdSet* s);
static void idset_insert(IdSet* s, uint32_t id) {
    uint64_t h = idset_slot(s, id);
    if (s->keys[h] == id) return;
    s->keys[h] = id; s->n++;
    if (s->n * 2 > s->cap) idset_grow(s);
}
static void idset_erase(IdSet* s, uint32_t id) {            /* backward-shift delete */
    uint64_t h = idset_slot(s, id);
    if (s->keys[h] != id) return;
    s->keys[h] = INVALID_ID; s->n--;
    uint64_t j = h;
    for (;;) {
        j = (j + 1) % s->cap;
        if (s->keys[j] == INVALID_ID) return;
        const uint64_t home = tsdg_o_mix64(s->keys[j]) % s->cap;
        const int wrap = (h <= j) ? (home <= h || home > j) : (home <= h && home > j);
        if (wrap) { s->keys[h] = s->keys[j]; s->keys[j] = INVALID_ID; h = j; }
    }
}
static int idset_grow(IdSet* s) {
    IdSet t;
    if (idset_init(&t, s->cap * 2) != 0) return 2;
    for (uint64_t i = 0; i < s->cap; ++i) if (s->keys[i] != INVALID_ID) idset_insert(&t, s->keys[i]);
    free(s->keys);
    *s = t;
    return 0;
}

typedef struct { IdDist* e; uint64_t n, cap; IdSet present; } UQueue;
static int uqueue_init(UQueue* q) {
    q->n = 0; q->cap = 256;
    q->e = (IdDist*)malloc(sizeof(IdDist) * q->cap);
    return q->e && idset_init(&q->present, 512) == 0 ? 0 : 2;
}
static void uqueue_push(UQueue* q, uint32_t id, float dist) {
    if (q->n == q->cap) { q->cap *= 2; q->e = (IdDist*)realloc(q->e, sizeof(IdDist) * q->cap); }
    IdDist e = {id, dist};
    /* kept sorted DESCENDING so pop_min takes the back */
    uint64_t pos = q->n;
    while (pos > 0 && closer(q->e[pos - 1], e)) { q->e[pos] = q->e[pos - 1]; pos--; }
    q->e[pos] = e;
    q->n++;
    idset_insert(&q->present, id);
}
static int uqueue_pop_min(UQueue* q, IdDist* out) {
    if (q->n == 0) return 0;
    *out = q->e[--q->n];
    idset_erase(&q->present, out->id);
    return 1;
}

/* ---- bestfirst_search.cpp:50-108 search_impl + :112-127 validation ---------- */
int tsdg_o_bestfirst(const tsdg_o_graph* g, const float* query, uint64_t rng_state,
                     const tsdg_o_bf_params* p, uint32_t* ids, float* dists, uint32_t* count,
                     uint64_t* stats3, uint64_t* trace2) {
    if (g->n == 0) return 1;
    if (p->k < 1 || p->hop_limit < 1 || p->m_segments < 1 || p->lambda_cut < 1 ||
        p->delta < 0.0f)
        return 1;
    uint64_t rng = rng_state;
    uint64_t evals = 0, examined = 0, expanded = 0;

    IdDist start = sentinel();
    for (uint32_t i = 0; i < 32; ++i) {                      /* :57-63 */
        const uint32_t v = rng_below(&rng, g->n);
        IdDist cand = {v, dist_row(g, query, v)};
        if (closer(cand, start)) start = cand;
    }
    evals += 32;

    TopK results;
    Queue queue;
    Visited visited;
    UQueue uq;
    IdSet uv;
    const int ub = p->unbounded != 0;
    int rc = topk_init(&results, p->k);
    if (ub) {
        if (!rc) rc = uqueue_init(&uq);
        if (!rc) rc = idset_init(&uv, 1024);
    } else {
        if (!rc) rc = queue_init(&queue, p->m_segments);
        if (!rc) rc = visited_init(&visited, p->m_segments);
    }
    if (rc) return 2;

    topk_push(&results, start.id, start.dist);               /* :68-69 */
    if (ub) uqueue_push(&uq, start.id, start.dist); else queue_push(&queue, start.id, start.dist);

    uint32_t t = 0;
    for (;;) {                                               /* :73-97 */
        const int empty = ub ? uq.n == 0 : queue.total == 0;
        if (empty || t >= p->hop_limit) break;
        ++t;
        IdDist popped;
        const int got = ub ? uqueue_pop_min(&uq, &popped) : queue_pop_min(&queue, &popped);
        if (!got) break;
        const uint32_t u = popped.id;
        if (popped.dist > topk_furthest(&results).dist + p->delta) break;   /* :79 */
        if (ub) idset_insert(&uv, u); else visited_add(&visited, u);
        expanded++;
        const uint64_t beg = g->offsets[u];
        const uint64_t len = prefix_len(g, u, p->lambda_cut);
        for (uint64_t j = 0; j < len; ++j) {                 /* :84-96 */
            const uint32_t e = g->targets[beg + j];
            examined++;
            const int seen = ub ? (idset_contains(&uv, e) || idset_contains(&uq.present, e))
                                : (visited_contains(&visited, e) || queue_contains(&queue, e));
            if (seen) continue;
            const float dist = dist_row(g, query, e);
            ++evals;
            if (dist < topk_furthest(&results).dist || results.n < p->k) {
                topk_push(&results, e, dist);
                if (ub) uqueue_push(&uq, e, dist); else queue_push(&queue, e, dist);
                if (results.n > p->k) results.n--;           /* pop_furthest */
            }
        }
    }

    if (stats3) {
        stats3[0] = t;
        stats3[1] = evals;
        stats3[2] = ub ? 0 : queue.evictions;
    }
    if (trace2) { trace2[0] = expanded; trace2[1] = examined; }
    *count = results.n;
    for (uint32_t i = 0; i < results.n; ++i) {
        ids[i] = results.e[i].id;
        if (dists) dists[i] = results.e[i].dist;
    }
    free(results.e);
    if (ub) { free(uq.e); free(uq.present.keys); free(uv.keys); }
    else { queue_free(&queue); visited_free(&visited); }
    return 0;
}

/* bestfirst_search.cpp:129-150: stream fork(q) of Rng64(seed) for query q. */
int tsdg_o_large_batch(const tsdg_o_graph* g, const float* queries, uint32_t nq,
                       uint64_t query_index_base, const tsdg_o_bf_params* p, uint32_t* ids,
                       float* dists, uint32_t* counts, uint64_t* stats) {
    for (uint32_t q = 0; q < nq; ++q) {
        uint32_t* qi = ids + (size_t)q * p->k;
        float* qd = dists ? dists + (size_t)q * p->k : NULL;
        for (uint32_t i = 0; i < p->k; ++i) { qi[i] = INVALID_ID; if (qd) qd[i] = INFINITY; }
        const int rc = tsdg_o_bestfirst(g, queries + (size_t)q * g->d,
                                        tsdg_o_fork(p->seed, query_index_base + q), p, qi, qd,
                                        counts + q, stats ? stats + 3 * (size_t)q : NULL, NULL);
        if (rc) return rc;
    }
    return 0;
}

/* ---- rank_list.cpp:8-18 lane_update ------------------------------------------ */
int tsdg_o_lane_update(uint32_t* slot_ids, float* slot_dists, const uint32_t* lanes,
                       const uint32_t* ids, const float* dists, uint32_t nb) {
    if (nb > LANES) return 1;
    for (uint32_t i = 0; i < nb; ++i) {
        if (lanes[i] >= LANES) return 1;
        if (dists[i] < slot_dists[lanes[i]]) {
            slot_ids[lanes[i]] = ids[i];
            slot_dists[lanes[i]] = dists[i];
        }
    }
    return 0;
}

static void sort_closer(IdDist* a, uint32_t n) {             /* insertion sort, total order */
    for (uint32_t i = 1; i < n; ++i) {
        IdDist x = a[i];
        uint32_t j = i;
        while (j > 0 && closer(x, a[j - 1])) { a[j] = a[j - 1]; j--; }
        a[j] = x;
    }
}

/* ---- rank_list.cpp:20-49 merge_halves ---------------------------------------- */
static int merge_halves(IdDist* rij, const IdDist* rtemp) {
    IdDist incoming[LANES];
    memcpy(incoming, rtemp, sizeof(incoming));
    sort_closer(incoming, LANES);
    IdDist pool[LANES + LANES / 2];
    memcpy(pool, rij, sizeof(IdDist) * LANES);
    uint32_t np = LANES;
    for (uint32_t i = 0; i < LANES / 2; ++i) {
        const IdDist e = incoming[i];
        if (e.id == INVALID_ID) break;
        uint32_t j = 0;
        while (j < np && pool[j].id != e.id) j++;
        if (j == np) pool[np++] = e;
        else if (closer(e, pool[j])) pool[j] = e;
    }
    sort_closer(pool, np);
    int changed = 0;
    for (uint32_t i = 0; i < LANES; ++i) {
        if (pool[i].id != rij[i].id || pool[i].dist != rij[i].dist) changed = 1;
        rij[i] = pool[i];
    }
    return changed;
}

int tsdg_o_merge_halves(uint32_t* rij_ids, float* rij_dists, const uint32_t* tmp_ids,
                        const float* tmp_dists, int* updated) {
    IdDist a[LANES], t[LANES];
    for (uint32_t i = 0; i < LANES; ++i) {
        a[i].id = rij_ids[i]; a[i].dist = rij_dists[i];
        t[i].id = tmp_ids[i]; t[i].dist = tmp_dists[i];
    }
    *updated = merge_halves(a, t);
    for (uint32_t i = 0; i < LANES; ++i) { rij_ids[i] = a[i].id; rij_dists[i] = a[i].dist; }
    return 0;
}

/* ---- greedy_search.cpp:12-25 select_start + :27-72 greedy_search_once -------- */
static uint32_t select_start(const tsdg_o_graph* g, const float* q, uint64_t* rng,
                             uint64_t* evals) {
    IdDist best = sentinel();
    for (uint32_t i = 0; i < 32; ++i) {
        const uint32_t v = rng_below(rng, g->n);
        IdDist cand = {v, dist_row(g, q, v)};
        if (closer(cand, best)) best = cand;
    }
    *evals += 32;
    return best.id;
}

static int greedy_once(const tsdg_o_graph* g, const float* query, uint64_t rng,
                       uint32_t hop_limit, uint32_t cut, IdDist* rij, uint64_t* hops,
                       uint64_t* evals) {
    if (cut < 1 || hop_limit < 1) return 1;
    if (g->n == 0) return 1;
    uint32_t u = select_start(g, query, &rng, evals);
    IdDist rtemp[LANES];
    for (uint32_t i = 0; i < LANES; ++i) rij[i] = sentinel();
    int improved = 1;
    uint32_t t = 0;
    while (improved && t < hop_limit) {
        ++t;
        for (uint32_t i = 0; i < LANES; ++i) rtemp[i] = sentinel();
        const uint64_t beg = g->offsets[u];
        const uint64_t len = prefix_len(g, u, cut);
        for (uint64_t j = 0; j < len; ++j) {   /* lane = position mod 32, strict < */
            const uint32_t v = g->targets[beg + j];
            const float dist = dist_row(g, query, v);
            const uint32_t lane = (uint32_t)(j % LANES);
            if (dist < rtemp[lane].dist) { rtemp[lane].id = v; rtemp[lane].dist = dist; }
        }
        *evals += len;
        const int updated = merge_halves(rij, rtemp);
        IdDist next = sentinel();
        for (uint32_t i = 0; i < LANES; ++i) if (closer(rtemp[i], next)) next = rtemp[i];
        if (next.id != INVALID_ID) u = next.id;
        improved = updated;
    }
    *hops += t;
    return 0;
}

int tsdg_o_greedy_once(const tsdg_o_graph* g, const float* query, uint64_t rng_state,
                       uint32_t hop_limit, uint32_t lambda_cut, uint32_t* ids32,
                       float* dists32, uint64_t* stats3) {
    IdDist r[LANES];
    uint64_t hops = 0, evals = 0;
    const int rc = greedy_once(g, query, rng_state, hop_limit, lambda_cut, r, &hops, &evals);
    if (rc) return rc;
    for (uint32_t i = 0; i < LANES; ++i) { ids32[i] = r[i].id; dists32[i] = r[i].dist; }
    if (stats3) { stats3[0] = hops; stats3[1] = evals; stats3[2] = 0; }
    return 0;
}

/* ---- greedy_search.cpp:74-127 small_batch_search(_one) ----------------------- */
int tsdg_o_small_batch(const tsdg_o_graph* g, const float* queries, uint32_t nq, uint32_t k,
                       const tsdg_o_greedy_params* p, uint32_t* ids, float* dists,
                       uint32_t* counts, uint64_t* stats) {
    if (k < 1 || p->t0 < 1 || (uint64_t)k > (uint64_t)LANES * p->t0) return 1;
    IdDist* pool = (IdDist*)malloc(sizeof(IdDist) * (size_t)p->t0 * LANES);
    if (!pool) return 2;
    for (uint32_t q = 0; q < nq; ++q) {
        const float* query = queries + (size_t)q * g->d;
        uint64_t hops = 0, evals = 0;
        uint32_t np = 0;
        for (uint32_t s = 0; s < p->t0; ++s) {
            IdDist r[LANES];
            const int rc = greedy_once(g, query, tsdg_o_fork(p->seed, s), p->hop_limit,
                                       p->lambda_cut, r, &hops, &evals);
            if (rc) { free(pool); return rc; }
            for (uint32_t i = 0; i < LANES; ++i) if (r[i].id != INVALID_ID) pool[np++] = r[i];
        }
        sort_closer(pool, np);
        uint32_t nu = 0;                                   /* std::unique by id */
        for (uint32_t i = 0; i < np; ++i) {
            if (nu > 0 && pool[nu - 1].id == pool[i].id) continue;
            pool[nu++] = pool[i];
        }
        uint32_t* qi = ids + (size_t)q * k;
        float* qd = dists ? dists + (size_t)q * k : NULL;
        counts[q] = nu < k ? nu : k;
        for (uint32_t i = 0; i < k; ++i) {
            qi[i] = i < counts[q] ? pool[i].id : INVALID_ID;
            if (qd) qd[i] = i < counts[q] ? pool[i].dist : INFINITY;
        }
        if (stats) { stats[3 * q] = hops; stats[3 * q + 1] = evals; stats[3 * q + 2] = 0; }
    }
    free(pool);
    return 0;
}

/* ---- op replays for pinning the segmented structures ------------------------ */
int tsdg_o_segmented_replay(uint32_t m, const uint8_t* ops, const uint32_t* ids,
                            const float* dists, uint32_t n_ops, uint32_t* out,
                            float* out_dist, uint64_t* sizes, uint64_t* evictions) {
    if (m < 1) return 1;
    Queue q;
    Visited v;
    if (queue_init(&q, m) || visited_init(&v, m)) return 2;
    for (uint32_t i = 0; i < n_ops; ++i) {
        out[i] = 0;
        out_dist[i] = 0.0f;
        if (ops[i] == 0) {
            if (!queue_contains(&q, ids[i])) { queue_push(&q, ids[i], dists[i]); out[i] = 1; }
        } else if (ops[i] == 1) {
            IdDist e;
            if (queue_pop_min(&q, &e)) { out[i] = e.id; out_dist[i] = e.dist; }
            else { out[i] = INVALID_ID; out_dist[i] = INFINITY; }
        } else if (ops[i] == 2) {
            visited_add(&v, ids[i]);
        } else {
            out[i] = (uint32_t)visited_contains(&v, ids[i]);
        }
        sizes[i] = q.total;
    }
    *evictions = q.evictions;
    queue_free(&q);
    visited_free(&v);
    return 0;
}

int tsdg_o_topk_replay(uint32_t k, const uint8_t* ops, const uint32_t* ids,
                       const float* dists, uint32_t n_ops, uint32_t* out,
                       uint32_t* final_ids, float* final_dists, uint32_t* final_n) {
    if (k < 1) return 1;
    TopK t;
    t.k = k; t.n = 0;
    t.e = (IdDist*)malloc(sizeof(IdDist) * ((size_t)n_ops + 2));
    if (!t.e) return 2;
    for (uint32_t i = 0; i < n_ops; ++i) {
        if (ops[i] == 0) out[i] = (uint32_t)topk_push(&t, ids[i], dists[i]);
        else { if (t.n == 0) { free(t.e); return 2; } t.n--; out[i] = 0; }
    }
    *final_n = t.n;
    for (uint32_t i = 0; i < t.n; ++i) { final_ids[i] = t.e[i].id; final_dists[i] = t.e[i].dist; }
    free(t.e);
    return 0;
}

/* ---- reference.cpp:96-111 exact_topk (stable sort by closer == sort by (dist,id)) */
int tsdg_o_exact_topk(const float* base, uint32_t n, const float* queries, uint32_t nq,
                      uint32_t d, uint32_t k, int metric, uint32_t* ids, float* dists) {
    IdDist* kept = (IdDist*)malloc(sizeof(IdDist) * ((size_t)k + 1));
    if (!kept) return 2;
    for (uint32_t q = 0; q < nq; ++q) {
        uint32_t nk = 0;
        for (uint32_t v = 0; v < n; ++v) {
            IdDist e = {v, tsdg_o_distance(queries + (size_t)q * d, base + (size_t)v * d, d, metric)};
            if (nk == k && !closer(e, kept[nk - 1])) continue;
            uint32_t pos = nk;
            while (pos > 0 && closer(e, kept[pos - 1])) { kept[pos] = kept[pos - 1]; pos--; }
            kept[pos] = e;
            if (nk < k) nk++;
        }
        for (uint32_t i = 0; i < k; ++i) {
            ids[(size_t)q * k + i] = i < nk ? kept[i].id : INVALID_ID;
            dists[(size_t)q * k + i] = i < nk ? kept[i].dist : INFINITY;
        }
    }
    free(kept);
    return 0;
}

/* knn_graph.cpp:64-86 brute_force_knn (BoundedPool, knn_graph.cpp:28-60): for every
 * node the k smallest (dist, id) over all other nodes; k already clamped by the
 * caller (clamp_k, knn_graph.cpp:17-26).  Output n x k ascending. */
int tsdg_o_brute_force_knn(const float* base, uint32_t n, uint32_t d, uint32_t k, int metric,
                           uint32_t* ids, float* dists) {
    if (n < 2 || k < 1 || k > n - 1) return 1;
    IdDist* kept = (IdDist*)malloc(sizeof(IdDist) * ((size_t)k + 1));
    if (!kept) return 2;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t nk = 0;
        for (uint32_t j = 0; j < n; ++j) {
            if (j == i) continue;
            IdDist e = {j, tsdg_o_distance(base + (size_t)i * d, base + (size_t)j * d, d, metric)};
            if (nk == k && !closer(e, kept[nk - 1])) continue;
            uint32_t pos = nk;
            while (pos > 0 && closer(e, kept[pos - 1])) { kept[pos] = kept[pos - 1]; pos--; }
            kept[pos] = e;
            if (nk < k) nk++;
        }
        for (uint32_t t = 0; t < k; ++t) {
            ids[(size_t)i * k + t] = kept[t].id;
            dists[(size_t)i * k + t] = kept[t].dist;
        }
    }
    free(kept);
    return 0;
}
