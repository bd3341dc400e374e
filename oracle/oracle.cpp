/*
 * oracle.cpp -- plain, slow, obviously-correct CPU reference of the compressed
 * key sort hot path (arXiv 2009.11543, "Compressed Key Sort and Fast Index
 * Reconstruction"). TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2009_11543_b200/); neither includes the other.
 *
 * Citations are PAPER.md line numbers ("P:n") with their section.
 * Conventions:
 *   - a key is a byte string of B bytes; bit position p is bit (7 - p%8) of
 *     byte p/8, position 0 is the most significant bit (reading C4);
 *   - a mask/bitmap uses the same layout as a key (D-bitmap P:363);
 *   - the compressed key P = Compress(key) read as an unsigned integer whose
 *     most significant bit is the first selected position (reading C5),
 *     stored right-aligned as SoA u32 planes: planes[q*n + i] = bits
 *     [32q, 32q+32) of P_i, nplanes = ceil(m/32);
 *   - duplicates have no distinction bit (0xFFFF marker) and are ordered by
 *     row id (reading C3); the sorted order is (full key, row id).
 *
 * Every function below is a direct transcription of a definition or an
 * algorithm step of the paper; library std::sort is used as the sort step.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <numeric>
#include <omp.h>
#include <parallel/algorithm>

#define ORC_NONE 0xFFFFu

static inline int key_bit(const uint8_t* key, uint32_t p) {
    return (key[p >> 3] >> (7 - (p & 7))) & 1;
}
static inline void set_bit(uint8_t* mask, uint32_t p) { mask[p >> 3] |= (uint8_t)(0x80u >> (p & 7)); }

extern "C" {

/* D-bit(a, b): "the most significant bit position where the two keys differ"
 * (Sec. 3.1). Returns -1 when the keys are equal (reading C3).
 * Byte loop to find the first differing byte, then a bit loop inside it. */
int orc_dbit_pair(const uint8_t* a, const uint8_t* b, uint32_t B) {
    for (uint32_t j = 0; j < B; j++) {
        if (a[j] != b[j]) {
            for (uint32_t t = 0; t < 8; t++)
                if (key_bit(a, 8 * j + t) != key_bit(b, 8 * j + t)) return (int)(8 * j + t);
        }
    }
    return -1;
}

/* D_all: the set of D-bits of ALL key pairs (Theorem 1), O(n^2).
 * Used for tiny inputs (and cfg1) to pin the adjacency computation. */
void orc_dbits_all_pairs(const uint8_t* keys, uint64_t n, uint32_t B, uint8_t* mask_out, int threads) {
    memset(mask_out, 0, B);
    if (threads < 1) threads = 1;
    std::vector<std::vector<uint8_t>> part((size_t)threads, std::vector<uint8_t>(B, 0));
    #pragma omp parallel for num_threads(threads) schedule(dynamic, 64)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        std::vector<uint8_t>& m = part[(size_t)omp_get_thread_num()];
        for (uint64_t j = (uint64_t)i + 1; j < n; j++) {
            int d = orc_dbit_pair(keys + (uint64_t)i * B, keys + j * B, B);
            if (d >= 0) set_bit(m.data(), (uint32_t)d);
        }
    }
    for (int t = 0; t < threads; t++)
        for (uint32_t j = 0; j < B; j++) mask_out[j] |= part[(size_t)t][j];
}

/* Sorted order of the full keys: lexicographic binary comparison (P:174, P:308,
 * P:327), ties (exact duplicates) broken by row id (reading C3).
 * rid == NULL means row ids 0..n-1. perm_out[i] = row id of the i-th key.
 * threads > 1 uses libstdc++ parallel mode (__gnu_parallel::sort), the paper's
 * own GCC STL parallel-sort baseline. */
void orc_sort_keys(const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* rid,
                   uint32_t* perm_out, int threads) {
    std::vector<uint64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (uint64_t)0);
    auto rowid = [&](uint64_t i) -> uint32_t { return rid ? rid[i] : (uint32_t)i; };
    auto less = [&](uint64_t x, uint64_t y) {
        int c = memcmp(keys + x * B, keys + y * B, B);
        if (c != 0) return c < 0;
        return rowid(x) < rowid(y);
    };
    if (threads > 1) {
        omp_set_num_threads(threads);
        __gnu_parallel::sort(idx.begin(), idx.end(), less);
    } else {
        std::sort(idx.begin(), idx.end(), less);
    }
    for (uint64_t i = 0; i < n; i++) perm_out[i] = rowid(idx[i]);
}

/* D_i = D-bit(key_{i-1}, key_i) over the sorted order, and
 * D_adj = {D_1..D_n} (Theorem 1). perm gives the sorted order as row ids
 * that index `keys` (identity row ids). dbit_out[0] = 0xFFFF; equal adjacent
 * keys give 0xFFFF and no bit (reading C3). Either output may be NULL. */
void orc_adjacent_dbits(const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm,
                        uint16_t* dbit_out, uint8_t* mask_out) {
    if (mask_out) memset(mask_out, 0, B);
    if (n && dbit_out) dbit_out[0] = ORC_NONE;
    for (uint64_t i = 1; i < n; i++) {
        int d = orc_dbit_pair(keys + (uint64_t)perm[i - 1] * B, keys + (uint64_t)perm[i] * B, B);
        if (dbit_out) dbit_out[i] = d < 0 ? ORC_NONE : (uint16_t)d;
        if (d >= 0 && mask_out) set_bit(mask_out, (uint32_t)d);
    }
}

/* Variant bitmap: OR over keys of (key XOR reference key), reference = key_0
 * (Sec. 4.3 recompute step 3). */
void orc_variant_bitmap(const uint8_t* keys, uint64_t n, uint32_t B, uint8_t* mask_out) {
    memset(mask_out, 0, B);
    for (uint64_t i = 1; i < n; i++)
        for (uint32_t j = 0; j < B; j++) mask_out[j] |= (uint8_t)(keys[i * B + j] ^ keys[j]);
}

/* D+ (byte-occupancy superset, SURVEY F4 / DESIGN reading R2): for each byte
 * position j, the distinction bits of the SET of byte values occurring at j,
 * obtained by Theorem 1 applied to those values: sort the distinct values
 * and take the D-bit of each adjacent pair. D is a subset of D+ (every pair's
 * D-bit lies in the first byte where the pair differs, and both byte values occur
 * there), so D+ is an "extended distinction bit" set. */
void orc_byteocc_superset(const uint8_t* keys, uint64_t n, uint32_t B, uint8_t* mask_out) {
    memset(mask_out, 0, B);
    std::vector<uint8_t> seen(256);
    for (uint32_t j = 0; j < B; j++) {
        std::fill(seen.begin(), seen.end(), 0);
        for (uint64_t i = 0; i < n; i++) seen[keys[i * B + j]] = 1;
        int prev = -1;
        for (int v = 0; v < 256; v++) {
            if (!seen[(size_t)v]) continue;
            if (prev >= 0) {
                uint8_t a = (uint8_t)prev, b = (uint8_t)v;
                int d = orc_dbit_pair(&a, &b, 1);
                set_bit(mask_out, 8 * j + (uint32_t)d);
            }
            prev = v;
        }
    }
}

/* D-offset[i] = position of the (i+1)-st 1 in the bitmap. Returns m. */
uint32_t orc_doffset(const uint8_t* mask, uint32_t B, uint16_t* moff_out) {
    uint32_t m = 0;
    for (uint32_t p = 0; p < 8 * B; p++)
        if (key_bit(mask, p)) { if (moff_out) moff_out[m] = (uint16_t)p; m++; }
    return m;
}

/* Compress(key): "the concatenation of the bits of key in (extended)
 * distinction bit positions", bit loop over the mask positions in
 * increasing order; the t-th selected bit is P's bit (m-1-t). */
void orc_compress(const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* mask, uint32_t* planes) {
    uint32_t m = orc_doffset(mask, B, NULL);
    uint32_t np = (m + 31) / 32;
    memset(planes, 0, (size_t)np * n * 4);
    for (uint64_t i = 0; i < n; i++) {
        uint32_t t = 0;
        for (uint32_t p = 0; p < 8 * B; p++) {
            if (!key_bit(mask, p)) continue;
            uint32_t e = m - 1 - t;
            if (key_bit(keys + i * B, p)) planes[(uint64_t)(e >> 5) * n + i] |= 1u << (e & 31);
            t++;
        }
    }
}

/* Sec. 5.1 segmentation: 8-byte masks; the first starts at the byte
 * holding the first 1 of the bitmap, each next one at the byte holding the
 * first 1 after the previous mask. Writes start bytes and per-mask popcounts;
 * returns the number of masks. */
uint32_t orc_pext_segments(const uint8_t* mask, uint32_t B, uint32_t* start_out, uint32_t* bits_out) {
    uint32_t nseg = 0, j = 0;
    while (j < B) {
        if (mask[j] == 0) { j++; continue; }
        uint32_t bits = 0;
        for (uint32_t b = j; b < j + 8 && b < B; b++)
            for (uint32_t t = 0; t < 8; t++) bits += (mask[b] >> t) & 1;
        if (start_out) start_out[nseg] = j;
        if (bits_out) bits_out[nseg] = bits;
        nseg++;
        j += 8;
    }
    return nseg;
}

/* PEXT as defined for BMI2: the k-th set bit of `m` (counting from the
 * least significant) selects a source bit that becomes bit k of the result. */
static uint64_t soft_pext64(uint64_t x, uint64_t m) {
    uint64_t r = 0;
    int k = 0;
    for (int b = 0; b < 64; b++)
        if ((m >> b) & 1) { r |= ((x >> b) & 1ull) << k; k++; }
    return r;
}

/* Compress via the paper's Sec. 5.1 pipeline: split the bitmap into
 * 8-byte masks (step 1), PEXT each key word with its mask (step 2), concatenate
 * by shift + OR (step 3). Words are read big-endian so the selected bits keep
 * their significance (the paper's little-endian detail P:449 is an
 * implementation choice). Must equal orc_compress bit for bit (reading C7). */
void orc_compress_pext(const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* mask, uint32_t* planes) {
    uint32_t m = orc_doffset(mask, B, NULL);
    uint32_t np = (m + 31) / 32;
    std::vector<uint32_t> st(B + 1), cnt(B + 1);
    uint32_t nseg = orc_pext_segments(mask, B, st.data(), cnt.data());
    std::vector<uint32_t> acc(np + 2);
    for (uint64_t i = 0; i < n; i++) {
        std::fill(acc.begin(), acc.end(), 0u);          /* big integer, limb 0 least significant */
        const uint8_t* key = keys + i * B;
        for (uint32_t s = 0; s < nseg; s++) {
            uint64_t kw = 0, mw = 0;
            for (uint32_t b = 0; b < 8; b++) {
                uint32_t jb = st[s] + b;
                kw = (kw << 8) | (jb < B ? key[jb] : 0);
                mw = (mw << 8) | (jb < B ? mask[jb] : 0);
            }
            uint64_t ext = soft_pext64(kw, mw);
            uint32_t c = cnt[s];
            /* acc = (acc << c) | ext, limb by limb (c <= 64) */
            for (uint32_t sh = c; sh > 0;) {
                uint32_t step = sh > 31 ? 31 : sh;
                uint32_t carry = 0;
                for (uint32_t q = 0; q < acc.size(); q++) {
                    uint32_t nc = step ? (acc[q] >> (32 - step)) : 0;
                    acc[q] = (acc[q] << step) | carry;
                    carry = nc;
                }
                sh -= step;
            }
            acc[0] |= (uint32_t)ext;
            if (acc.size() > 1) acc[1] |= (uint32_t)(ext >> 32);
        }
        for (uint32_t q = 0; q < np; q++) planes[(uint64_t)q * n + i] = acc[q];
    }
}

/* Sort of the (compressed key, row id) pairs: order by P as an
 * unsigned integer (most significant plane first), ties by row id.
 * rid == NULL means 0..n-1; perm_out receives row ids. */
void orc_sort_packed(const uint32_t* planes, uint32_t np, uint64_t n, const uint32_t* rid,
                     uint32_t* perm_out, int threads) {
    std::vector<uint32_t> rec((size_t)n * (np + 1));     /* AoS copy: P most significant first, then rid */
    for (uint64_t i = 0; i < n; i++) {
        for (uint32_t q = 0; q < np; q++) rec[i * (np + 1) + q] = planes[(uint64_t)(np - 1 - q) * n + i];
        rec[i * (np + 1) + np] = rid ? rid[i] : (uint32_t)i;
    }
    std::vector<uint64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (uint64_t)0);
    auto less = [&](uint64_t x, uint64_t y) {
        const uint32_t* a = &rec[x * (np + 1)];
        const uint32_t* b = &rec[y * (np + 1)];
        for (uint32_t q = 0; q <= np; q++)
            if (a[q] != b[q]) return a[q] < b[q];
        return false;
    };
    if (threads > 1) {
        omp_set_num_threads(threads);
        __gnu_parallel::sort(idx.begin(), idx.end(), less);
    } else {
        std::sort(idx.begin(), idx.end(), less);
    }
    for (uint64_t i = 0; i < n; i++) perm_out[i] = rec[idx[i] * (np + 1) + np];
}

/* Rebuild-time recompute and leaf D-bits: over sorted compressed
 * keys, D_i = D-offset[D-bit(Compress(key_{i-1}), Compress(key_i))], where the
 * D-bit of two m-bit compressed keys is their first differing bit counting from
 * the most significant (bit m-1 of P is compressed position 0). Outputs the
 * exact D (subset of the sort mask) and the D_i (0xFFFF for i=0 / equal).
 * sorted_planes are SoA planes already in sorted order. */
void orc_adjacent_compressed(const uint32_t* sorted_planes, uint32_t m, uint64_t n,
                             const uint8_t* sort_mask, uint32_t B,
                             uint16_t* dbit_out, uint8_t* mask_out) {
    std::vector<uint16_t> moff(8 * B + 1);
    uint32_t mm = orc_doffset(sort_mask, B, moff.data());
    (void)mm;
    uint32_t np = (m + 31) / 32;
    if (mask_out) memset(mask_out, 0, B);
    if (n && dbit_out) dbit_out[0] = ORC_NONE;
    for (uint64_t i = 1; i < n; i++) {
        int t = -1;
        for (uint32_t c = 0; c < m && t < 0; c++) {         /* compressed position c = P bit (m-1-c) */
            uint32_t e = m - 1 - c;
            uint32_t a = (sorted_planes[(uint64_t)(e >> 5) * n + i - 1] >> (e & 31)) & 1;
            uint32_t b = (sorted_planes[(uint64_t)(e >> 5) * n + i] >> (e & 31)) & 1;
            if (a != b) t = (int)c;
        }
        (void)np;
        if (t < 0) { if (dbit_out) dbit_out[i] = ORC_NONE; continue; }
        uint16_t pos = moff[(size_t)t];
        if (dbit_out) dbit_out[i] = pos;
        if (mask_out) set_bit(mask_out, pos);
    }
}

/* Bottom-up bulk load (Sec. 5.3). Each node has `fanout` slots and is
 * filled with per = floor(fanout * fill) entries (reading C8). Levels are
 * stored leaves first, concatenated; level_nodes[l] nodes at level l.
 *   leaf node j, slot e:  rid = perm[j*per + e], dbit = D_{j*per+e} (leaf entry
 *                         D-bit vs the global predecessor; reading C9)
 *   inner node j, slot e: child c = j*per + e of the level below (global node
 *                         index), rid = row id of the highest key under c
 *                         (P:356), dbit = D-bit(highest key of the previous entry
 *                         at this level, highest key of c) computed DIRECTLY on
 *                         the full keys; 0xFFFF for c = 0 / equal.
 * Empty slots: rid/child 0xFFFFFFFF, dbit 0xFFFF. Returns the height (levels). */
/* Block-parallel index construction (Sec. 5.3): "n sort keys are divided into p
 * blocks ... Thread i constructs a subtree consisting of all sort keys in the i-th block.
 * When all the subtrees are constructed, they are merged into one tree ... we remove the root
 * nodes of the subtrees, and build the top layers of the whole tree by linking the children
 * of the root nodes of the subtrees."
 * blocks: consecutive ranges of the sorted order of sizes block_n[0..nblocks) (empty blocks
 * contribute nothing). Each block's subtree is the bottom-up bulk load of its keys (per
 * entries a node). The root's children are at level h-2 of a subtree of height h; blocks of
 * unequal heights (not in the paper, whose blocks are equal) keep their levels up to
 * l* = max(0, min_b h_b - 2), so every leaf stays at the same depth (reading R17). Level
 * l <= l* of the whole tree = the blocks' level-l nodes in block order; above l*, nodes of
 * per consecutive nodes up to one root. Entries as orc_bulkload: a leaf entry is a key
 * (row id, D_i); an inner entry is a child node (row id of its highest key, global child
 * node id, D-bit of its highest key against the highest key of the previous node of that
 * level -- across block borders -- computed from the keys; none for a level's first).
 * Output layout as orc_bulkload (levels concatenated, leaves first). Returns the height. */
uint32_t orc_bulkload_blocks(const uint32_t* perm, const uint16_t* dbit, uint64_t n, const uint64_t* block_n,
                             uint32_t nblocks, uint32_t fanout, uint32_t per, const uint8_t* keys, uint32_t B,
                             uint64_t* level_nodes_out, uint32_t* node_cnt, uint32_t* entry_rid,
                             uint32_t* entry_child, uint16_t* entry_dbit) {
    struct Node { uint64_t lo, hi; std::vector<uint64_t> ent; };  /* key range; entries (keys or child ids in level) */
    std::vector<std::vector<std::vector<Node>>> sub;             /* [block][level][node] */
    uint64_t start = 0;
    for (uint32_t b = 0; b < nblocks; b++) {
        const uint64_t nb = block_n[b];
        if (nb == 0) continue;
        std::vector<std::vector<Node>> lv(1);
        for (uint64_t x = start; x < start + nb; x += per) {    /* leaves of per keys */
            Node nd;
            nd.lo = x;
            nd.hi = std::min(x + per, start + nb) - 1;
            for (uint64_t k = nd.lo; k <= nd.hi; k++) nd.ent.push_back(k);
            lv[0].push_back(nd);
        }
        while (lv.back().size() > 1) {                          /* up to the subtree's root */
            const std::vector<Node>& below = lv.back();
            std::vector<Node> up;
            for (uint64_t j = 0; j < below.size(); j += per) {
                Node nd;
                const uint64_t j1 = std::min<uint64_t>(j + per, below.size());
                nd.lo = below[j].lo;
                nd.hi = below[j1 - 1].hi;
                for (uint64_t c = j; c < j1; c++) nd.ent.push_back(c);
                up.push_back(nd);
            }
            lv.push_back(up);
        }
        sub.push_back(lv);
        start += nb;
    }
    if (sub.empty()) return 0;
    size_t hmin = sub[0].size();
    for (auto& t : sub) hmin = std::min(hmin, t.size());
    const size_t lstar = hmin >= 2 ? hmin - 2 : 0;               /* the roots' children (equal heights) */
    /* the whole tree's levels 0..lstar: the blocks' levels concatenated; child ids rebased */
    std::vector<std::vector<Node>> all(lstar + 1);
    for (size_t l = 0; l <= lstar; l++) {
        uint64_t rebase = 0;                                     /* nodes of level l-1 in earlier blocks */
        for (size_t b = 0; b < sub.size(); b++) {
            for (const Node& nd : sub[b][l]) {
                Node c = nd;
                if (l > 0)
                    for (auto& e : c.ent) e += rebase;
                all[l].push_back(c);
            }
            if (l > 0) rebase += sub[b][l - 1].size();
        }
    }
    while (all.back().size() > 1) {                             /* the top layers */
        const std::vector<Node>& below = all.back();
        std::vector<Node> up;
        for (uint64_t j = 0; j < below.size(); j += per) {
            Node nd;
            const uint64_t j1 = std::min<uint64_t>(j + per, below.size());
            nd.lo = below[j].lo;
            nd.hi = below[j1 - 1].hi;
            for (uint64_t c = j; c < j1; c++) nd.ent.push_back(c);
            up.push_back(nd);
        }
        all.push_back(up);
    }
    uint64_t off = 0;
    for (size_t l = 0; l < all.size(); l++) {
        level_nodes_out[l] = all[l].size();
        const uint64_t below_off = l ? off - all[l - 1].size() : 0;
        for (uint64_t j = 0; j < all[l].size(); j++) {
            const Node& nd = all[l][j];
            const uint64_t node = off + j;
            node_cnt[node] = (uint32_t)nd.ent.size();
            for (uint32_t e = 0; e < fanout; e++) {
                const uint64_t slot = node * fanout + e;
                entry_rid[slot] = 0xFFFFFFFFu;
                entry_child[slot] = 0xFFFFFFFFu;
                entry_dbit[slot] = ORC_NONE;
                if (e >= nd.ent.size()) continue;
                const uint64_t x = nd.ent[e];
                if (l == 0) {
                    entry_rid[slot] = perm[x];
                    entry_dbit[slot] = dbit ? dbit[x] : (uint16_t)ORC_NONE;
                } else {
                    const Node& c = all[l - 1][x];
                    entry_rid[slot] = perm[c.hi];
                    entry_child[slot] = (uint32_t)(below_off + x);
                    if (x > 0) {
                        const Node& pv = all[l - 1][x - 1];
                        int d = orc_dbit_pair(keys + (uint64_t)perm[pv.hi] * B, keys + (uint64_t)perm[c.hi] * B, B);
                        entry_dbit[slot] = d < 0 ? (uint16_t)ORC_NONE : (uint16_t)d;
                    }
                }
            }
        }
        off += all[l].size();
    }
    return (uint32_t)all.size();
}

uint32_t orc_bulkload(const uint32_t* perm, const uint16_t* dbit, uint64_t n, uint32_t fanout,
                      uint32_t per, const uint8_t* keys, uint32_t B,
                      uint64_t* level_nodes_out, uint32_t* node_cnt, uint32_t* entry_rid,
                      uint32_t* entry_child, uint16_t* entry_dbit) {
    if (n == 0) return 0;
    std::vector<uint64_t> lv;            /* nodes per level */
    uint64_t cnt = n;
    do { cnt = (cnt + per - 1) / per; lv.push_back(cnt); } while (cnt > 1);
    uint64_t off = 0;
    uint64_t span = 1;                   /* sorted keys covered by one entry at this level */
    for (size_t l = 0; l < lv.size(); l++) {
        level_nodes_out[l] = lv[l];
        uint64_t entries = (l == 0) ? n : lv[l - 1];
        for (uint64_t j = 0; j < lv[l]; j++) {
            uint64_t node = off + j;
            uint32_t c = 0;
            for (uint32_t e = 0; e < fanout; e++) {
                uint64_t slot = node * fanout + e;
                uint64_t x = j * per + e;                 /* entry index within this level */
                if (e < per && x < entries) {
                    uint64_t hi = std::min((x + 1) * span, n) - 1;       /* highest sorted index */
                    entry_rid[slot] = perm[hi];
                    if (l == 0) {
                        entry_child[slot] = 0xFFFFFFFFu;
                        entry_dbit[slot] = dbit ? dbit[x] : (uint16_t)ORC_NONE;
                    } else {
                        uint64_t below = off - lv[l - 1];
                        entry_child[slot] = (uint32_t)(below + x);
                        if (x == 0) entry_dbit[slot] = ORC_NONE;
                        else {
                            uint64_t phi = x * span - 1;        /* highest sorted index of entry x-1 */
                            int d = orc_dbit_pair(keys + (uint64_t)perm[phi] * B, keys + (uint64_t)perm[hi] * B, B);
                            entry_dbit[slot] = d < 0 ? (uint16_t)ORC_NONE : (uint16_t)d;
                        }
                    }
                    c++;
                } else {
                    entry_rid[slot] = 0xFFFFFFFFu;
                    entry_child[slot] = 0xFFFFFFFFu;
                    entry_dbit[slot] = ORC_NONE;
                }
            }
            node_cnt[node] = c;
        }
        off += lv[l];
        span *= per;
    }
    return (uint32_t)lv.size();
}


/* ---- NEXT-3: the paper's index tree format (Sec. 4.2; Sec. 5.3) ----
 *
 * Node = 256 bytes. Leaf: 24-byte header, 8-byte next-node pointer, 14 entries of 16
 * bytes ("(256-32)/16 = 14"); an entry is a partial key, a distinction bit position,
 * an index key length and a record ID. Non-leaf: 24-byte header, 9 entries of 24
 * bytes = partial key, distinction bit position, key length, child pointer, pointer
 * to the highest key. Nodes are filled to floor(max fanout * fill).
 * Byte layout (little-endian, R16):
 *   header  u16 count | u16 level | u32 key_bytes | u64 highest key (record id) | u64 0
 *   leaf    u64 next leaf (node index, all-ones for the last) | 14 x {u32 pk | u16 dbit |
 *           u16 key_len | u64 record id}
 *   inner   9 x {u32 pk | u16 dbit | u16 key_len | u64 child node index | u64 highest key}
 * The partial key is the pk bits following the entry's distinction bit position D (P:335,
 * reading C14: positions D+1 .. D+pk; positions past the key are 0); with no distinction bit
 * (first key, equal keys) positions 0 .. pk-1 (reading R16). Bits are packed from bit 31 down.
 * Non-leaf entry: highest key of the child's subtree, its D-bit against the previous entry's
 * highest key at the same level, computed here directly on the full keys. Nodes are
 * numbered leaves first, then each level up. Returns the height. */
static uint32_t partial_key(const uint8_t* key, uint32_t B, int d, uint32_t pk) {
    uint32_t v = 0;
    uint32_t p0 = d < 0 ? 0u : (uint32_t)d + 1;
    for (uint32_t j = 0; j < pk; j++) {
        uint32_t p = p0 + j;
        uint32_t bit = p < 8 * B ? (uint32_t)key_bit(key, p) : 0u;
        v |= bit << (31 - j);
    }
    return v;
}
static void put16(uint8_t* o, uint16_t v) { memcpy(o, &v, 2); }
static void put32(uint8_t* o, uint32_t v) { memcpy(o, &v, 4); }
static void put64(uint8_t* o, uint64_t v) { memcpy(o, &v, 8); }

uint32_t orc_paper_tree(const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit,
                        uint32_t pk, uint32_t leaf_per, uint32_t inner_per, uint8_t* nodes) {
    if (n == 0) return 0;
    std::vector<uint64_t> lv;                         /* nodes per level */
    std::vector<uint64_t> cover;                      /* sorted keys per node of each level */
    uint64_t c = (n + leaf_per - 1) / leaf_per;
    lv.push_back(c);
    cover.push_back(leaf_per);
    while (c > 1) {
        c = (c + inner_per - 1) / inner_per;
        lv.push_back(c);
        cover.push_back(cover.back() * inner_per);
    }
    uint64_t total = 0;
    for (uint64_t x : lv) total += x;
    memset(nodes, 0, total * 256);
    auto key = [&](uint64_t sorted_idx) { return keys + (uint64_t)perm[sorted_idx] * B; };
    /* leaves */
    for (uint64_t j = 0; j < lv[0]; j++) {
        uint8_t* nd = nodes + j * 256;
        uint64_t k0 = j * leaf_per, k1 = std::min(k0 + leaf_per, n);
        put16(nd, (uint16_t)(k1 - k0));
        put16(nd + 2, 0);
        put32(nd + 4, B);
        put64(nd + 8, perm[k1 - 1]);
        put64(nd + 24, j + 1 < lv[0] ? j + 1 : ~0ull);
        for (uint64_t k = k0; k < k1; k++) {
            uint8_t* e = nd + 32 + (k - k0) * 16;
            int d = dbit[k] == ORC_NONE ? -1 : (int)dbit[k];
            put32(e, partial_key(key(k), B, d, pk));
            put16(e + 4, dbit[k]);
            put16(e + 6, (uint16_t)B);
            put64(e + 8, perm[k]);
        }
    }
    /* non-leaf levels */
    uint64_t off = lv[0], below = 0;
    for (size_t l = 1; l < lv.size(); l++) {
        for (uint64_t j = 0; j < lv[l]; j++) {
            uint8_t* nd = nodes + (off + j) * 256;
            uint64_t c0 = j * inner_per, c1 = std::min(c0 + inner_per, lv[l - 1]);
            uint64_t hi_last = std::min((c1) * cover[l - 1], n) - 1;
            put16(nd, (uint16_t)(c1 - c0));
            put16(nd + 2, (uint16_t)l);
            put32(nd + 4, B);
            put64(nd + 8, perm[hi_last]);
            for (uint64_t ch = c0; ch < c1; ch++) {
                uint8_t* e = nd + 24 + (ch - c0) * 24;
                uint64_t hi = std::min((ch + 1) * cover[l - 1], n) - 1;      /* highest key of child ch */
                int d = -1;
                if (ch > 0) {
                    uint64_t phi = ch * cover[l - 1] - 1;                       /* ... of child ch-1 */
                    d = orc_dbit_pair(key(phi), key(hi), B);
                }
                put32(e, partial_key(key(hi), B, d, pk));
                put16(e + 4, d < 0 ? (uint16_t)ORC_NONE : (uint16_t)d);
                put16(e + 6, (uint16_t)B);
                put64(e + 8, below + ch);
                put64(e + 16, perm[hi]);
            }
        }
        below = off;
        off += lv[l];
    }
    return (uint32_t)lv.size();
}

}  /* extern "C" */
