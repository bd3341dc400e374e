/*
 * cksgen.c -- seeded, synthetic key-column generators for the five
 * BASELINE.json configs plus generic edge-case columns.
 *
 * This module is INPUT GENERATION ONLY. It holds none of the compressed key
 * sort's arithmetic (no distinction bits, no compression, no sorting); both the
 * CPU oracle (oracle/) and the CUDA path (paper_2009_11543_b200/) consume its
 * output through the Python wrapper cksgen/__init__.py.
 *
 * Randomness is counter-based: every draw is mix(seed, stream, counter), so a
 * row's content depends only on (seed, row) and rows are generated in parallel
 * with OpenMP while staying bit-for-bit deterministic.
 *
 * Recipes (SURVEY.md 8(d) readings; the paper's
 * workloads they stand in for are its Table 2 datasets):
 *   cfg1  n x 16 B bytes i.i.d. uniform, ~1% exact duplicates
 *   cfg2  n x 8 B big-endian uint64 = base + 4096*cluster + U[0,4096), 1000 clusters
 *   cfg3  n x 32 B title-like NUL-padded strings (lognormal length, Zipf first char)
 *   cfg4  n x 64 B URL-like NUL-padded strings (200 Zipf hosts + random path)
 *   cfg5  n x 32 B ACGT 32-mers from a 4n-base sequence with 10% copied repeats
 *   Zipf(s,n,m)  the paper's sensitivity-analysis family (Sec. 6.4):
 *         n-byte keys; in every 8-byte word the first m bytes hold one fixed ASCII
 *         character and the other 8-m bytes lower-case letters drawn from Zipf(s, 26)
 *         (rank 1 = 'a', ..., rank 26 = 'z'); 10 M keys in the paper
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---- counter-based RNG (splitmix64 finaliser) -------------------------- */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
    return mix64(mix64(seed * 0x9E3779B97F4A7C15ull + stream) ^ (ctr * 0xD1B54A32D192ED03ull));
}
/* per-row sequential stream: state seeded from (seed, stream, row) */
typedef struct { uint64_t s; } rowrng;
static inline uint64_t rr_next(rowrng* r) { r->s += 0x9E3779B97F4A7C15ull; return mix64(r->s); }
static inline double rr_unif(rowrng* r) { return (double)(rr_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint64_t rr_below(rowrng* r, uint64_t k) { return rr_next(r) % k; }

/* Zipf(s) over ranks 1..k: inverse CDF by binary search on a prebuilt table */
static void zipf_cdf(double s, int k, double* cdf) {
    double acc = 0.0;
    for (int r = 1; r <= k; r++) { acc += 1.0 / pow((double)r, s); cdf[r - 1] = acc; }
    for (int r = 0; r < k; r++) cdf[r] /= acc;
}
static inline int zipf_pick(const double* cdf, int k, double u) {
    int lo = 0, hi = k - 1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (u <= cdf[mid]) hi = mid; else lo = mid + 1; }
    return lo;
}

/* ---- cfg1 / generic: uniform bytes ------------------------------------- */
static void row_uniform(uint64_t seed, uint64_t i, uint32_t B, uint8_t* out) {
    uint32_t words = (B + 7) / 8;
    for (uint32_t w = 0; w < words; w++) {
        uint64_t v = draw(seed, 0, i * words + w);
        for (uint32_t b = 0; b < 8 && w * 8 + b < B; b++) out[w * 8 + b] = (uint8_t)(v >> (8 * b));
    }
}

/* ---- cfg3: title-like strings ------------------------------------------ */
static const char ALPHA64[] = "-0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZ_abcdefghijklmnopqrstuvwxyz";
typedef struct { double cdf[64]; char perm[64]; } title_tab;
static void title_init(uint64_t seed, title_tab* t) {
    zipf_cdf(1.1, 64, t->cdf);
    memcpy(t->perm, ALPHA64, 64);
    for (int k = 63; k > 0; k--) {                 /* seeded Fisher-Yates */
        int j = (int)(draw(seed, 5, (uint64_t)k) % (uint64_t)(k + 1));
        char c = t->perm[k]; t->perm[k] = t->perm[j]; t->perm[j] = c;
    }
}
static void row_title(uint64_t seed, uint64_t i, uint32_t B, const title_tab* t, uint8_t* out) {
    rowrng r = { draw(seed, 3, i) };
    double u1 = rr_unif(&r), u2 = rr_unif(&r);
    if (u1 < 1e-300) u1 = 1e-300;
    double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    double mu = log(18.0) - 0.18, sigma = 0.6;      /* mean exp(mu + sigma^2/2) = 18 */
    long len = lround(exp(mu + sigma * z));
    if (len < 1) len = 1;
    if (len > (long)B) len = (long)B;
    memset(out, 0, B);
    out[0] = (uint8_t)t->perm[zipf_pick(t->cdf, 64, rr_unif(&r))];
    for (long c = 1; c < len; c++) out[c] = (uint8_t)ALPHA64[rr_next(&r) & 63];
}

/* ---- cfg4: URL-like strings --------------------------------------------- */
#define NHOST 200
typedef struct { double cdf[NHOST]; char host[NHOST][40]; int hlen[NHOST]; } url_tab;
static void url_init(uint64_t seed, url_tab* t) {
    static const char* tld[4] = { ".com", ".org", ".net", ".io" };
    zipf_cdf(1.2, NHOST, t->cdf);
    for (int h = 0; h < NHOST; h++) {
        rowrng r = { draw(seed, 11, (uint64_t)h) };
        int total = 12 + (int)rr_below(&r, 19);          /* U[12,30] */
        const char* d = tld[rr_below(&r, 4)];
        int dl = (int)strlen(d);
        int lab = total - 8 - dl;
        if (lab < 1) lab = 1;
        int p = 0;
        memcpy(t->host[h], "https://", 8); p = 8;
        for (int c = 0; c < lab; c++) t->host[h][p++] = (char)('a' + rr_below(&r, 26));
        memcpy(t->host[h] + p, d, (size_t)dl); p += dl;
        t->hlen[h] = p;
    }
}
static void row_url(uint64_t seed, uint64_t i, uint32_t B, const url_tab* t, uint8_t* out) {
    static const char AN[] = "abcdefghijklmnopqrstuvwxyz0123456789";
    char buf[512];
    rowrng r = { draw(seed, 12, i) };
    int h = zipf_pick(t->cdf, NHOST, rr_unif(&r));
    int p = 0;
    memcpy(buf, t->host[h], (size_t)t->hlen[h]); p = t->hlen[h];
    int nseg = 2 + (int)rr_below(&r, 4);                 /* U{2..5} */
    for (int s = 0; s < nseg; s++) {
        buf[p++] = '/';
        int sl = 3 + (int)rr_below(&r, 8);              /* U{3..10} */
        for (int c = 0; c < sl; c++) buf[p++] = AN[rr_below(&r, 36)];
    }
    memset(out, 0, B);
    memcpy(out, buf, (size_t)(p < (int)B ? p : (int)B));
}

/* ---- duplicate injection: row i becomes a copy of row src's original ---- */
static inline int is_dup(uint64_t seed, uint64_t i, uint32_t dup_ppm) {
    return dup_ppm && (draw(seed, 1, i) % 1000000ull) < dup_ppm;
}
static inline uint64_t dup_src(uint64_t seed, uint64_t i, uint64_t n) { return draw(seed, 2, i) % n; }

/* ------------------------------------------------------------------------ */
/* Public entry points (ctypes). Return 0 on success, -1 on bad arguments.   */
/* ------------------------------------------------------------------------ */

/* uniform bytes, B arbitrary, dup_ppm parts-per-million exact duplicates (cfg1 family) */
int cksgen_uniform(uint64_t seed, uint64_t n, uint32_t B, uint32_t dup_ppm, uint8_t* out) {
    if (!out && n) return -1;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint64_t src = is_dup(seed, (uint64_t)i, dup_ppm) ? dup_src(seed, (uint64_t)i, n) : (uint64_t)i;
        row_uniform(seed, src, B, out + (uint64_t)i * B);
    }
    return 0;
}

/* cfg2 family: big-endian uint64 = base + 4096*cluster + U[0,4096) */
int cksgen_clusters(uint64_t seed, uint64_t n, uint32_t nclusters, uint32_t width, uint8_t* out) {
    if ((!out && n) || nclusters == 0 || width == 0) return -1;
    uint64_t base = draw(seed, 0, 0) >> 1;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint64_t c = draw(seed, 1, (uint64_t)i) % nclusters;
        uint64_t o = draw(seed, 2, (uint64_t)i) % width;
        uint64_t v = base + (uint64_t)width * c + o;
        for (int b = 0; b < 8; b++) out[(uint64_t)i * 8 + b] = (uint8_t)(v >> (56 - 8 * b));
    }
    return 0;
}

int cksgen_titles(uint64_t seed, uint64_t n, uint32_t B, uint32_t dup_ppm, uint8_t* out) {
    if ((!out && n) || B == 0) return -1;
    title_tab t; title_init(seed, &t);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint64_t src = is_dup(seed, (uint64_t)i, dup_ppm) ? dup_src(seed, (uint64_t)i, n) : (uint64_t)i;
        row_title(seed, src, B, &t, out + (uint64_t)i * B);
    }
    return 0;
}

int cksgen_urls(uint64_t seed, uint64_t n, uint32_t B, uint8_t* out) {
    if ((!out && n) || B == 0) return -1;
    url_tab* t = (url_tab*)malloc(sizeof(url_tab));
    if (!t) return -1;
    url_init(seed, t);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) row_url(seed, (uint64_t)i, B, t, out + (uint64_t)i * B);
    free(t);
    return 0;
}

/* cfg5 family: k-mers (B bytes) sampled from a G = 4n base ACGT sequence, 10% repeats */
int cksgen_genome(uint64_t seed, uint64_t n, uint32_t B, uint8_t* out) {
    if ((!out && n) || B == 0) return -1;
    if (n == 0) return 0;
    uint64_t G = 4 * n;
    if (G < (uint64_t)B + 8192) G = (uint64_t)B + 8192;
    uint8_t* seq = (uint8_t*)malloc(G);
    if (!seq) return -1;
    static const char ACGT[4] = { 'A', 'C', 'G', 'T' };
    #pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < (int64_t)((G + 31) / 32); w++) {
        uint64_t v = draw(seed, 20, (uint64_t)w);
        for (int b = 0; b < 32 && (uint64_t)w * 32 + b < G; b++) seq[w * 32 + b] = (uint8_t)ACGT[(v >> (2 * b)) & 3];
    }
    /* repeats: copy U[64,4096] segments until 10% of the bases were overwritten (sequential) */
    rowrng r = { draw(seed, 21, 0) };
    uint64_t over = 0;
    while (over < G / 10) {
        uint64_t len = 64 + rr_below(&r, 4033);
        if (len > G) len = G;
        uint64_t src = rr_below(&r, G - len + 1), dst = rr_below(&r, G - len + 1);
        memmove(seq + dst, seq + src, len);
        over += len;
    }
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint64_t st = draw(seed, 22, (uint64_t)i) % (G - B + 1);
        memcpy(out + (uint64_t)i * B, seq + st, B);
    }
    free(seq);
    return 0;
}

/* Zipf(s, B, m): every 8-byte word of a key = m copies of `fixed`, then
 * 8 - m letters 'a' + (rank - 1) with rank ~ Zipf(s, 26); a trailing partial word likewise */
int cksgen_zipf(uint64_t seed, uint64_t n, uint32_t B, double s, uint32_t m, uint8_t fixed, uint8_t* out) {
    if ((!out && n) || B == 0 || m > 8 || !(s > 0.0)) return -1;
    double cdf[26];
    zipf_cdf(s, 26, cdf);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        rowrng r = { draw(seed, 30, (uint64_t)i) };
        uint8_t* row = out + (uint64_t)i * B;
        for (uint32_t j = 0; j < B; j++)
            row[j] = (j % 8) < m ? fixed : (uint8_t)('a' + zipf_pick(cdf, 26, rr_unif(&r)));
    }
    return 0;
}

/* fill n keys of BASELINE config cfg (1..5) with key width B (fixed per config) */
int cksgen_config(int cfg, uint64_t seed, uint64_t n, uint8_t* out) {
    switch (cfg) {
        case 1: return cksgen_uniform(seed, n, 16, 10000, out);
        case 2: return cksgen_clusters(seed, n, 1000, 4096, out);
        case 3: return cksgen_titles(seed, n, 32, 5000, out);
        case 4: return cksgen_urls(seed, n, 64, out);
        case 5: return cksgen_genome(seed, n, 32, out);
        default: return -1;
    }
}
