/*
 * Input preparation executable (NOT the search path, never timed): materialises a
 * dataset's files in the formats the REFERENCE reads, so the reference arm of
 * bench.py can load them through its own loaders (io.cpp:112-117 load_vectors,
 * diversify.cpp:274-306 load_tsdg) without mapping any library of this repository.
 *
 *   tsdg_prepare vectors lowlid|synthetic n nq d latent clusters spread seed noise \
 *                <base.fvecs> <queries.fvecs> [<fnv_base> <fnv_queries>]
 *       generate the seeded vectors (tools/datagen.c) and write them as fvecs;
 *       with checksums given, verify them first (generator drift).
 *   tsdg_prepare pack <graph.tsdg> <graph.pk>
 *       the transport form of a reference-built TSDG (format below, ~20 bits/edge)
 *   tsdg_prepare unpack <graph.pk> <base.fvecs> <out.tsdg> [row_offset]
 *       rebuild the TSDG file byte for byte: targets + lambdas from the pack,
 *       per-edge distances recomputed from the base rows in the reference's order;
 *       the result must match the original file's FNV-1a or nothing is written.
 *
 * Built by paper_2204_00824_b200/_build.py as _lib/tsdg_prepare (gcc, -fopenmp,
 * -ffp-contract=off, datagen.c linked in statically).
 */
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

int tsdg_make_synthetic_split(uint32_t n, uint32_t nq, uint32_t d, uint32_t clusters,
                              float spread, uint64_t seed, float* base, float* queries);
int tsdg_make_lowlid(uint32_t n, uint32_t nq, uint32_t d, uint32_t latent_dim,
                     uint32_t clusters, float spread, uint64_t seed, float noise, float* base,
                     float* queries);
uint64_t tsdg_fnv1a(const void* p, uint64_t nbytes);
void tsdg_edge_distances(const float* base, uint32_t n, uint32_t d, int metric,
                         const uint64_t* offsets, const uint32_t* targets, float* out);

static int die(const char* msg, const char* what) {
    fprintf(stderr, "tsdg_prepare: %s%s%s\n", msg, what ? ": " : "", what ? what : "");
    return 1;
}

static int write_fvecs(const char* path, const float* v, uint32_t n, uint32_t d) {
    char tmp[4096];
    snprintf(tmp, sizeof tmp, "%s.tmp%ld", path, (long)getpid());
    FILE* f = fopen(tmp, "wb");
    if (!f) return die("cannot open for writing", tmp);
    const int32_t dd = (int32_t)d;
    for (uint32_t i = 0; i < n; ++i) {
        if (fwrite(&dd, 4, 1, f) != 1 || fwrite(v + (size_t)i * d, 4, d, f) != d) {
            fclose(f);
            return die("write failed", tmp);
        }
    }
    if (fclose(f) != 0) return die("write failed", tmp);
    if (rename(tmp, path) != 0) return die("rename failed", path);
    return 0;
}

static int cmd_vectors(int argc, char** argv) {
    if (argc != 13 && argc != 15) return die("usage: vectors kind n nq d latent clusters spread seed noise base.fvecs queries.fvecs [fnv_base fnv_queries]", NULL);
    const char* kind = argv[2];
    const uint32_t n = (uint32_t)strtoul(argv[3], NULL, 10), nq = (uint32_t)strtoul(argv[4], NULL, 10);
    const uint32_t d = (uint32_t)strtoul(argv[5], NULL, 10), latent = (uint32_t)strtoul(argv[6], NULL, 10);
    const uint32_t clusters = (uint32_t)strtoul(argv[7], NULL, 10);
    const float spread = strtof(argv[8], NULL);
    const uint64_t seed = strtoull(argv[9], NULL, 10);
    const float noise = strtof(argv[10], NULL);
    float* base = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* q = (float*)malloc(sizeof(float) * (size_t)nq * d);
    if (!base || !q) return die("out of memory", NULL);
    int rc;
    if (strcmp(kind, "lowlid") == 0) rc = tsdg_make_lowlid(n, nq, d, latent, clusters, spread, seed, noise, base, q);
    else if (strcmp(kind, "synthetic") == 0) rc = tsdg_make_synthetic_split(n, nq, d, clusters, spread, seed, base, q);
    else return die("unknown kind", kind);
    if (rc != 0) return die("generator failed", kind);
    if (argc == 15) {
        char hb[32], hq[32];
        snprintf(hb, sizeof hb, "%016llx", (unsigned long long)tsdg_fnv1a(base, (uint64_t)n * d * 4));
        snprintf(hq, sizeof hq, "%016llx", (unsigned long long)tsdg_fnv1a(q, (uint64_t)nq * d * 4));
        if (strcmp(hb, argv[13]) != 0 || strcmp(hq, argv[14]) != 0)
            return die("generated vectors do not match the dataset checksums", argv[13]);
    }
    if (write_fvecs(argv[11], base, n, d) || write_fvecs(argv[12], q, nq, d)) return 1;
    free(base);
    free(q);
    return 0;
}

static float* read_fvecs(const char* path, uint32_t* n_out, uint32_t* d_out) {
    FILE* f = fopen(path, "rb");
    if (!f) return NULL;
    int32_t d = 0;
    if (fread(&d, 4, 1, f) != 1 || d <= 0) {
        fclose(f);
        return NULL;
    }
    fseek(f, 0, SEEK_END);
    const long size = ftell(f);
    fseek(f, 0, SEEK_SET);
    const size_t rec = 4 + 4 * (size_t)d;
    if (size < 0 || (size_t)size % rec != 0) {
        fclose(f);
        return NULL;
    }
    const uint32_t n = (uint32_t)((size_t)size / rec);
    float* v = (float*)malloc(sizeof(float) * (size_t)n * d);
    for (uint32_t i = 0; v && i < n; ++i) {
        int32_t di;
        if (fread(&di, 4, 1, f) != 1 || di != d || fread(v + (size_t)i * d, 4, d, f) != (size_t)d) {
            free(v);
            v = NULL;
        }
    }
    fclose(f);
    *n_out = n;
    *d_out = (uint32_t)d;
    return v;
}

/* ---- graph.pk: the transport form of a reference-built TSDG file ------------------
 *   "TSDGPK02" | u64 n | u64 E | u32 lbits | u32 dbytes | u64 fnv (of the original
 *   file) | u64 nbits | 27-byte TSDG header | n degrees (dbytes each, LE) | bitstream
 * Bitstream, LSB first, per node u: its targets sorted ascending, Rice-coded gaps
 * (first target, then differences - 1) with parameter k_u = floor(log2(n / (deg+1))),
 * then the lambda of each edge in that order (lbits each).  The fp32 distances are
 * not stored: they are recomputed from the base rows in the reference's sequential
 * order, and the reference's edge order (lambda, dist, target) (diversify.cpp:147,
 * 239-242) is restored by sorting on it.  The rebuilt file must match `fnv`. */
typedef struct {
    uint64_t* w;
    uint64_t cap, nbits;
} BitW;
static void bw_put(BitW* b, uint64_t v, uint32_t nb) { /* nb <= 32 */
    while (nb) {
        const uint64_t word = b->nbits >> 6, off = b->nbits & 63;
        if (word >= b->cap) {
            b->cap = b->cap ? 2 * b->cap : 1 << 20;
            b->w = (uint64_t*)realloc(b->w, 8 * b->cap);
        }
        if (off == 0) b->w[word] = 0;
        const uint32_t take = (uint32_t)(64 - off) < nb ? (uint32_t)(64 - off) : nb;
        b->w[word] |= (v & ((take == 64) ? ~0ull : ((1ull << take) - 1))) << off;
        v >>= take;
        nb -= take;
        b->nbits += take;
    }
}
typedef struct {
    const uint64_t* w;
    uint64_t pos, nbits;
} BitR;
static inline uint64_t br_get(BitR* b, uint32_t nb) {
    uint64_t v = 0;
    uint32_t got = 0;
    while (got < nb) {
        const uint64_t word = b->pos >> 6, off = b->pos & 63;
        const uint32_t take = (uint32_t)(64 - off) < nb - got ? (uint32_t)(64 - off) : nb - got;
        const uint64_t bits = (b->w[word] >> off) & ((take == 64) ? ~0ull : ((1ull << take) - 1));
        v |= bits << got;
        got += take;
        b->pos += take;
    }
    return v;
}
static inline uint32_t rice_k(uint64_t n, uint32_t deg) {
    uint64_t m = n / ((uint64_t)deg + 1);
    uint32_t k = 0;
    while ((2ull << k) <= m) ++k;
    return m ? k : 0;
}
static void rice_put(BitW* b, uint64_t g, uint32_t k) {
    uint64_t q = g >> k;
    while (q >= 32) {
        bw_put(b, 0xFFFFFFFFull, 32);
        q -= 32;
    }
    bw_put(b, (1ull << q) - 1, (uint32_t)q); /* q ones */
    bw_put(b, 0, 1);
    if (k) bw_put(b, g & ((1ull << k) - 1), k);
}
static uint64_t rice_get(BitR* b, uint32_t k) {
    uint64_t q = 0;
    while (br_get(b, 1)) ++q;
    return (q << k) | (k ? br_get(b, k) : 0);
}

typedef struct {
    uint32_t t;
    uint16_t lam;
    float dist;
} Edge;
static int cmp_target(const void* x, const void* y) {
    const Edge* a = (const Edge*)x;
    const Edge* b = (const Edge*)y;
    return a->t < b->t ? -1 : a->t > b->t;
}
static int cmp_edge_order(const void* x, const void* y) { /* (lambda, dist, target) */
    const Edge* a = (const Edge*)x;
    const Edge* b = (const Edge*)y;
    if (a->lam != b->lam) return a->lam < b->lam ? -1 : 1;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->t < b->t ? -1 : a->t > b->t;
}

static unsigned char* read_all(const char* path, size_t* size) {
    FILE* f = fopen(path, "rb");
    if (!f) return NULL;
    fseek(f, 0, SEEK_END);
    const long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    unsigned char* buf = (unsigned char*)malloc(sz > 0 ? (size_t)sz : 1);
    if (buf && fread(buf, 1, (size_t)sz, f) != (size_t)sz) {
        free(buf);
        buf = NULL;
    }
    fclose(f);
    *size = (size_t)sz;
    return buf;
}

static int cmd_pack(int argc, char** argv) {
    if (argc != 4) return die("usage: pack graph.tsdg out.pk", NULL);
    size_t size;
    unsigned char* raw = read_all(argv[2], &size);
    if (!raw || size < 27 || memcmp(raw, "TSDG", 4) != 0) return die("not a TSDG file", argv[2]);
    uint64_t n;
    memcpy(&n, raw + 8, 8);
    uint32_t* deg = (uint32_t*)malloc(4 * (n ? n : 1));
    size_t pos = 27;
    uint64_t E = 0;
    uint32_t maxdeg = 0, maxlam = 0;
    for (uint64_t u = 0; u < n; ++u) {
        if (pos + 4 > size) return die("truncated TSDG", argv[2]);
        memcpy(&deg[u], raw + pos, 4);
        for (uint32_t j = 0; j < deg[u]; ++j) {
            uint16_t l;
            memcpy(&l, raw + pos + 4 + 10 * (size_t)j + 4, 2);
            if (l > maxlam) maxlam = l;
        }
        pos += 4 + 10 * (size_t)deg[u];
        E += deg[u];
        if (deg[u] > maxdeg) maxdeg = deg[u];
    }
    if (pos != size) return die("trailing bytes in TSDG", argv[2]);
    uint32_t lbits = 1;
    while ((1u << lbits) <= maxlam) ++lbits;
    const uint32_t dbytes = maxdeg < 256 ? 1 : maxdeg < 65536 ? 2 : 4;
    BitW bw = {0};
    Edge* tmp = (Edge*)malloc(sizeof(Edge) * (maxdeg ? maxdeg : 1));
    pos = 27;
    for (uint64_t u = 0; u < n; ++u) {
        const uint32_t dg = deg[u];
        for (uint32_t j = 0; j < dg; ++j) {
            const unsigned char* r = raw + pos + 4 + 10 * (size_t)j;
            memcpy(&tmp[j].t, r, 4);
            memcpy(&tmp[j].lam, r + 4, 2);
        }
        qsort(tmp, dg, sizeof(Edge), cmp_target);
        const uint32_t k = rice_k(n, dg);
        uint64_t prev = 0;
        for (uint32_t j = 0; j < dg; ++j) {
            const uint64_t g = j == 0 ? tmp[j].t : (uint64_t)tmp[j].t - prev - 1;
            rice_put(&bw, g, k);
            prev = tmp[j].t;
        }
        for (uint32_t j = 0; j < dg; ++j) bw_put(&bw, tmp[j].lam, lbits);
        pos += 4 + 10 * (size_t)dg;
    }
    const uint64_t fnv = tsdg_fnv1a(raw, size);
    FILE* o = fopen(argv[3], "wb");
    if (!o) return die("cannot open for writing", argv[3]);
    const uint32_t hdr32[2] = {lbits, dbytes};
    fwrite("TSDGPK02", 1, 8, o);
    fwrite(&n, 8, 1, o);
    fwrite(&E, 8, 1, o);
    fwrite(hdr32, 4, 2, o);
    fwrite(&fnv, 8, 1, o);
    fwrite(&bw.nbits, 8, 1, o);
    fwrite(raw, 1, 27, o);
    for (uint64_t u = 0; u < n; ++u) fwrite(&deg[u], dbytes, 1, o);
    fwrite(bw.w, 1, (bw.nbits + 7) / 8, o);
    if (fclose(o) != 0) return die("write failed", argv[3]);
    free(raw);
    free(deg);
    free(tmp);
    free(bw.w);
    return 0;
}

static float edge_dist(const float* a, const float* b, uint32_t d, int metric) {
    /* vectors.hpp:36-49: sequential fp32 (built with -ffp-contract=off) */
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

/* unpack graph.pk base.fvecs out.tsdg [row_offset]: base rows [row_offset,
 * row_offset + n) of the fvecs file are the graph's nodes (a shard of a larger set). */
static int cmd_unpack(int argc, char** argv) {
    if (argc != 5 && argc != 6) return die("usage: unpack graph.pk base.fvecs out.tsdg [row_offset]", NULL);
    size_t size;
    unsigned char* pk = read_all(argv[2], &size);
    if (!pk || size < 72 || memcmp(pk, "TSDGPK02", 8) != 0) return die("not a graph pack", argv[2]);
    uint64_t n, E, fnv, nbits;
    uint32_t lbits, dbytes;
    memcpy(&n, pk + 8, 8);
    memcpy(&E, pk + 16, 8);
    memcpy(&lbits, pk + 24, 4);
    memcpy(&dbytes, pk + 28, 4);
    memcpy(&fnv, pk + 32, 8);
    memcpy(&nbits, pk + 40, 8);
    const unsigned char* hdr = pk + 48;
    const unsigned char* degp = pk + 75;
    const size_t bit_off = 75 + (size_t)n * dbytes;
    if (size < bit_off + (nbits + 7) / 8) return die("truncated pack", argv[2]);
    /* the bitstream as 64-bit words (copy: alignment + zero tail) */
    const uint64_t nw = (nbits + 63) / 64 + 1;
    uint64_t* words = (uint64_t*)calloc(nw, 8);
    if (!words) return die("out of memory", NULL);
    memcpy(words, pk + bit_off, (nbits + 7) / 8);
    uint32_t bn, bd;
    float* base = read_fvecs(argv[3], &bn, &bd);
    const uint64_t row0 = argc == 6 ? strtoull(argv[5], NULL, 10) : 0;
    if (!base || row0 + n > bn) return die("base vectors do not match the graph", argv[3]);
    const float* rows = base + (size_t)row0 * bd;
    const int metric = hdr[16];
    const size_t out_size = 27 + 4 * n + 10 * E;
    unsigned char* body = (unsigned char*)malloc(out_size);
    uint64_t* node_pos = (uint64_t*)malloc(8 * (n ? n : 1));
    uint64_t* bit_pos = (uint64_t*)malloc(8 * (n ? n : 1));
    uint32_t* deg = (uint32_t*)malloc(4 * (n ? n : 1));
    if (!body || !node_pos || !bit_pos || !deg) return die("out of memory", NULL);
    memcpy(body, hdr, 27);
    /* sequential pass: degrees, output offsets, and each node's bit offset (the
     * gaps must be decoded to skip a node; the lambdas are fixed width) */
    BitR br = {words, 0, nbits};
    uint64_t off = 27, e_total = 0;
    for (uint64_t u = 0; u < n; ++u) {
        uint32_t dg = 0;
        memcpy(&dg, degp + (size_t)u * dbytes, dbytes);
        deg[u] = dg;
        node_pos[u] = off;
        bit_pos[u] = br.pos;
        const uint32_t k = rice_k(n, dg);
        for (uint32_t j = 0; j < dg; ++j) rice_get(&br, k);
        br.pos += (uint64_t)dg * lbits;
        off += 4 + 10 * (uint64_t)dg;
        e_total += dg;
    }
    if (e_total != E || off != out_size || br.pos != nbits) return die("pack is inconsistent", argv[2]);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : bad)
    for (int64_t u = 0; u < (int64_t)n; ++u) {
        const uint32_t dg = deg[u];
        Edge* ed = (Edge*)malloc(sizeof(Edge) * (dg ? dg : 1));
        BitR r = {words, bit_pos[u], nbits};
        const uint32_t k = rice_k(n, dg);
        uint64_t prev = 0;
        for (uint32_t j = 0; j < dg; ++j) {
            const uint64_t g = rice_get(&r, k);
            const uint64_t t = j == 0 ? g : prev + 1 + g;
            ed[j].t = (uint32_t)t;
            prev = t;
            if (t >= n) bad = 1;
        }
        for (uint32_t j = 0; j < dg; ++j) ed[j].lam = (uint16_t)br_get(&r, lbits);
        if (!bad) {
            for (uint32_t j = 0; j < dg; ++j)
                ed[j].dist = edge_dist(rows + (size_t)u * bd, rows + (size_t)ed[j].t * bd, bd, metric);
            qsort(ed, dg, sizeof(Edge), cmp_edge_order);
            unsigned char* p = body + node_pos[u];
            memcpy(p, &dg, 4);
            for (uint32_t j = 0; j < dg; ++j) {
                memcpy(p + 4 + 10 * (size_t)j, &ed[j].t, 4);
                memcpy(p + 8 + 10 * (size_t)j, &ed[j].lam, 2);
                memcpy(p + 10 + 10 * (size_t)j, &ed[j].dist, 4);
            }
        }
        free(ed);
    }
    if (bad) return die("pack has an edge target out of range", argv[2]);
    if (tsdg_fnv1a(body, out_size) != fnv) return die("unpacked TSDG differs from the original (fnv)", argv[2]);
    char tmp[4096];
    snprintf(tmp, sizeof tmp, "%s.tmp%ld", argv[4], (long)getpid());
    FILE* o = fopen(tmp, "wb");
    if (!o || fwrite(body, 1, out_size, o) != out_size || fclose(o) != 0) return die("write failed", tmp);
    if (rename(tmp, argv[4]) != 0) return die("rename failed", argv[4]);
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 2 && strcmp(argv[1], "vectors") == 0) return cmd_vectors(argc, argv);
    if (argc >= 2 && strcmp(argv[1], "unpack") == 0) return cmd_unpack(argc, argv);
    if (argc >= 2 && strcmp(argv[1], "pack") == 0) return cmd_pack(argc, argv);
    return die("usage: tsdg_prepare vectors|pack|unpack ...", NULL);
}
