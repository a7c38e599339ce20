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
 *   tsdg_prepare unpack <graph.pk> <base.fvecs> <out.tsdg>
 *       rebuild a TSDG file from its packed transport form (tools/graph_pack.py):
 *       targets + lambdas from the pack, per-edge distances recomputed from the
 *       base rows in the reference's order; the result must match the original
 *       file's FNV-1a or nothing is written.
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

/* graph.pk (tools/graph_pack.py):
 *   "TSDGPK01" | u64 n | u64 E | u32 lbits | u32 nbytes | u64 fnv | 27-byte TSDG
 *   header | n x u32 degrees | E x nbytes little-endian (target << lbits | lambda) */
static int cmd_unpack(int argc, char** argv) {
    if (argc != 5) return die("usage: unpack graph.pk base.fvecs out.tsdg", NULL);
    FILE* f = fopen(argv[2], "rb");
    if (!f) return die("cannot open", argv[2]);
    char magic[8];
    uint64_t n, E, fnv;
    uint32_t lbits, nbytes;
    unsigned char hdr[27];
    if (fread(magic, 1, 8, f) != 8 || memcmp(magic, "TSDGPK01", 8) != 0 || fread(&n, 8, 1, f) != 1 ||
        fread(&E, 8, 1, f) != 1 || fread(&lbits, 4, 1, f) != 1 || fread(&nbytes, 4, 1, f) != 1 ||
        fread(&fnv, 8, 1, f) != 1 || fread(hdr, 1, 27, f) != 27 || nbytes > 8)
        return die("malformed pack", argv[2]);
    uint32_t* degs = (uint32_t*)malloc(4 * n);
    unsigned char* packed = (unsigned char*)malloc((size_t)E * nbytes);
    uint64_t* offsets = (uint64_t*)malloc(8 * (n + 1));
    uint32_t* targets = (uint32_t*)malloc(4 * (E ? E : 1));
    uint16_t* lambdas = (uint16_t*)malloc(2 * (E ? E : 1));
    float* dists = (float*)malloc(4 * (E ? E : 1));
    if (!degs || !packed || !offsets || !targets || !lambdas || !dists) return die("out of memory", NULL);
    if (fread(degs, 4, n, f) != n || fread(packed, nbytes, E, f) != E) return die("truncated pack", argv[2]);
    fclose(f);
    offsets[0] = 0;
    for (uint64_t u = 0; u < n; ++u) offsets[u + 1] = offsets[u] + degs[u];
    if (offsets[n] != E) return die("pack degree sum mismatch", argv[2]);
    for (uint64_t j = 0; j < E; ++j) {
        uint64_t v = 0;
        memcpy(&v, packed + (size_t)j * nbytes, nbytes);
        targets[j] = (uint32_t)(v >> lbits);
        lambdas[j] = (uint16_t)(v & ((1ull << lbits) - 1));
    }
    uint32_t bn, bd;
    float* base = read_fvecs(argv[3], &bn, &bd);
    if (!base || bn != n) return die("base vectors do not match the graph", argv[3]);
    const int metric = hdr[16];
    tsdg_edge_distances(base, (uint32_t)n, bd, metric, offsets, targets, dists);
    const size_t size = 27 + 4 * n + 10 * E;
    unsigned char* body = (unsigned char*)malloc(size);
    if (!body) return die("out of memory", NULL);
    memcpy(body, hdr, 27);
    size_t pos = 27;
    for (uint64_t u = 0; u < n; ++u) {
        memcpy(body + pos, &degs[u], 4);
        pos += 4;
        for (uint64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
            memcpy(body + pos, &targets[j], 4);
            memcpy(body + pos + 4, &lambdas[j], 2);
            memcpy(body + pos + 6, &dists[j], 4);
            pos += 10;
        }
    }
    if (tsdg_fnv1a(body, size) != fnv) return die("unpacked TSDG differs from the original (fnv)", argv[2]);
    char tmp[4096];
    snprintf(tmp, sizeof tmp, "%s.tmp%ld", argv[4], (long)getpid());
    FILE* o = fopen(tmp, "wb");
    if (!o || fwrite(body, 1, size, o) != size || fclose(o) != 0) return die("write failed", tmp);
    if (rename(tmp, argv[4]) != 0) return die("rename failed", argv[4]);
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 2 && strcmp(argv[1], "vectors") == 0) return cmd_vectors(argc, argv);
    if (argc >= 2 && strcmp(argv[1], "unpack") == 0) return cmd_unpack(argc, argv);
    return die("usage: tsdg_prepare vectors|unpack ...", NULL);
}
