/*
 * cks.h -- C ABI of libcks.so, the B200 (sm_100a) compressed key sort.
 *
 * Paper: "Compressed Key Sort and Fast Index Reconstruction", arXiv 2009.11543.
 * Citations "P:n" are lines of the paper text with their section.
 *
 * CONVENTIONS (DESIGN.md Sec. 2 readings R3-R5, R8-R9)
 *   keys     device u8[n][key_bytes], row-major; byte 0 is most significant and bit
 *            position p is bit (7 - p%8) of byte p/8, position 0 = MSB.
 *            Row id of key i is i unless row ids are passed explicitly.
 *   mask     HOST u8[key_bytes] in the same bit layout as a key: 1 = (possibly) a
 *            distinction bit position (the D-bitmap). m = popcount(mask).
 *   packed   device u32[ceil(m/32)][n], structure-of-arrays "planes": plane q holds
 *            bits [32q, 32q+32) of P, where P = Compress(key) read as an
 *            unsigned m-bit integer whose MOST significant bit is the mask's first
 *            (smallest) position. m = 0 means zero planes.
 *   perm     device u32[n]; perm[i] = row id of the i-th smallest (key, row id).
 *   dbit     device u16[n]; dbit[i] = D_i = D-bit(sorted key_{i-1}, sorted key_i)
 *            (P:176), CKS_DBIT_NONE for i = 0 and for equal adjacent keys.
 *
 * OWNERSHIP  The caller allocates and owns every pointer it passes (device
 *            pointers may come from torch.empty(..., device="cuda")). The library
 *            never frees caller memory. A cks_ctx owns internal scratch, grown on
 *            demand and freed by cks_ctx_destroy; pointers it returns as "views"
 *            stay valid until the next call on the same context.
 * STREAMS    All device work is ordered on the context's stream (borrowed from the
 *            caller, e.g. torch.cuda.current_stream().cuda_stream; NULL = legacy
 *            default stream). Calls that return host results (masks, popcounts,
 *            heights) synchronise that stream before returning and say so.
 * ERRORS     Every call returns CKS_OK (0) or a positive error code:
 *              CKS_EINVAL  null pointer with n > 0, key_bytes not in [1, 512],
 *                          fanout < 2, fill not in (0, 1], floor(fanout*fill) < 2,
 *                          bits > 8*512, unknown kind;
 *              CKS_ERANGE  n >= 2^32 (row ids are u32); or, from cks_build /
 *                          cks_build_host[_batch] / cks_distinction_mask with the order
 *                          check on (cks_ctx_set_verify; by default whenever a prior mask
 *                          is passed), a sort mask that is not a superset of the true
 *                          distinction bits: Theorem 2 then does not hold and
 *                          the check finds an adjacent pair of the returned order out of
 *                          (key, row id) order. With the check off such a mask yields a
 *                          wrong permutation without an error;
 *              CKS_ENOMEM  scratch allocation failed;
 *              CKS_ECUDA   a CUDA runtime error (text in cks_last_error).
 *            Duplicated keys are NOT an error (reading R3). n = 0 is a valid no-op.
 *            m = 0 (n <= 1 or all keys equal) is valid: zero planes, identity perm.
 *            No call falls back to the CPU.
 */
#ifndef CKS_H
#define CKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKS_OK 0
#define CKS_EINVAL 1
#define CKS_ERANGE 2
#define CKS_ENOMEM 3
#define CKS_ECUDA 4

#define CKS_DBIT_NONE 0xFFFFu
#define CKS_MAX_KEY_BYTES 512u
#define CKS_MAX_LEVELS 40

/* superset masks for the first build (reading R2) */
#define CKS_SUPERSET_VARIANT 0   /* V: OR of key XOR key_0 */
#define CKS_SUPERSET_BYTEOCC 1   /* D+: per byte, D-bits of the set of occurring byte values */

typedef struct cks_ctx cks_ctx;

/* ---- context ---------------------------------------------------------------- */

/* Create a context on CUDA `device` using `stream` (cudaStream_t, may be NULL). */
int cks_ctx_create(int device, void* stream, cks_ctx** out);
int cks_ctx_destroy(cks_ctx* ctx);
/* Replace the borrowed stream used by subsequent calls. */
int cks_ctx_set_stream(cks_ctx* ctx, void* stream);
/* 1 = record per-stage CUDA events in cks_build (read with cks_ctx_stage_ms) and the dominant
 * kernel's own events (cks_ctx_kernel_stats). The event records sit between kernels that are
 * otherwise chained by programmatic dependent launch, so a timed build is slower (cfg5:
 * ~0.06 ms); bench.py times one build in ten this way. */
int cks_ctx_set_timing(cks_ctx* ctx, int enable);
/* How cks_build / cks_distinction_mask sort (the result is the same):
 *   CKS_SORT_SINGLE       one stable LSD sort over all m = |M| bits of P_M;
 *   CKS_SORT_PREFIX_AUTO  by distinguishing prefixes (NEXT-1) when m > 64 (default);
 *   CKS_SORT_PREFIX       by distinguishing prefixes whenever m > 0. */
#define CKS_SORT_SINGLE 0
#define CKS_SORT_PREFIX_AUTO 1
#define CKS_SORT_PREFIX 2
int cks_ctx_set_sort_mode(cks_ctx* ctx, int mode);
/* Width T of the first refinement round: 0 = chosen from a sample
 * (default), else a multiple of 8 in [8, 64]. The result does not depend on T (CKS_EINVAL
 * otherwise). */
int cks_ctx_set_round0_bits(cks_ctx* ctx, uint32_t bits);
/* Order check of cks_build / cks_build_host[_batch] / cks_distinction_mask results against the
 * key rows (one random row gather per key; returns CKS_ERANGE on a pair out of order, see
 * ERRORS). The paper's rebuild extracts with the current D-bitmap, which is only
 * correct while it contains every distinction bit; the check is complete because
 * the (key, row id) order is total and a sequence is sorted iff every adjacent pair is.
 *   CKS_VERIFY_OFF     never;
 *   CKS_VERIFY_PRIOR   when the caller passes a prior mask (default; the library's own
 *                      superset masks contain D by construction, reading R2). A sufficient
 *                      test runs first: the new keys' byte-occupancy superset D+ (reading R2:
 *                      D is inside it; marked by the rebuild's compress, or one sequential
 *                      pass), and when D+ lies inside the prior mask the order is right by
 *                      Theorem 2 and the row-gather check is skipped; a mask that
 *                      failed the test is remembered by the context, which then goes straight
 *                      to the row-gather check;
 *   CKS_VERIFY_ALWAYS  every build. */
#define CKS_VERIFY_OFF 0
#define CKS_VERIFY_PRIOR 1
#define CKS_VERIFY_ALWAYS 2
int cks_ctx_set_verify(cks_ctx* ctx, int mode);
/* The speculative first build (cks_build): 1 = on (default), 0 = every
 * first build runs its own superset pass before the compress. The result is the same either
 * way; a column whose row sample keeps missing byte values pays a second build when on. */
int cks_ctx_set_speculative_mask(cks_ctx* ctx, int enable);
/* First builds that took the speculative mask, and those of them run again by the full D+. */
int cks_ctx_speculation_stats(const cks_ctx* ctx, uint64_t* builds, uint64_t* retries);
/* Stage times (ms) of the last timed cks_build: a1 mask, a3 compress, a4 histograms+scan,
 * a5 LSD passes, a6 adjacency, a7 repack, a8 bulk load, total. Synchronises. Returns the
 * count written (0 if timing was off). */
int cks_ctx_stage_ms(cks_ctx* ctx, float* out, int max);
/* Number of kernels libcks launched since the context was created. */
uint64_t cks_ctx_launches(const cks_ctx* ctx);
/* Dominant kernel of the last timed cks_build (the warp-specialised LSD downsweep, one
 * launch per digit pass): summed CUDA-event time in ms on the context's stream, summed
 * algorithmic bytes (every stream of the pass read once and written once) and the number
 * of launches. Synchronises. Zeros when timing was off. */
int cks_ctx_kernel_stats(cks_ctx* ctx, double* ms, double* bytes, uint32_t* count);
/* Algorithmic bytes of the last cks_build / cks_build_host / cks_sort_prefix on this context:
 * the sum over every kernel it launched of the bytes that kernel must read and write at least
 * (each input stream read once, each output written once; DESIGN.md Sec. 6 lists the per-kernel
 * formulas). With the build's time this is the whole path's roofline, on the work actually
 * run (not on a formula for a full-width sort). Host-side, no synchronisation. */
int cks_ctx_path_bytes(const cks_ctx* ctx, double* bytes);
const char* cks_strerror(int code);
const char* cks_last_error(const cks_ctx* ctx);

/* ---- a1: superset mask -------------------------------------------------------------
 * One pass over the keys; writes the chosen superset M of the distinction bits
 * (kind = CKS_SUPERSET_VARIANT: variant bitmap V, P:365/P:413;
 *  kind = CKS_SUPERSET_BYTEOCC: D+ = union over byte positions j of the D-bits of the
 *  set of byte values occurring at j -- "extended distinction bit positions").
 * mask_out: host u8[key_bytes]; popcount_out: host, may be NULL. Synchronises. */
int cks_superset_mask(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes,
                      int kind, uint8_t* mask_out, uint32_t* popcount_out);

/* ---- exact D (first build; rebuild recompute) ------------------------
 * Exact distinction bits D = {D_1..D_{n}} over the sorted order (Theorem 1).
 * Runs: superset mask (or `prior_mask`, host u8[key_bytes], which MUST be a superset of
 * D, e.g. the previous D-bitmap; checked by default, CKS_ERANGE when it is not, see
 * cks_ctx_set_verify) -> compress -> ONE stable sort -> adjacency.
 * If perm_out (device u32[n]) is non-NULL it receives the permutation of that same sort.
 * mask_out: host u8[key_bytes]; popcount_out: host, may be NULL. Synchronises. */
int cks_distinction_mask(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes,
                         const uint8_t* prior_mask, uint8_t* mask_out, uint32_t* popcount_out,
                         uint32_t* perm_out);

/* ---- a2+a3: compress (Sec. 5.1) -------------------------------------------
 * packed_out[q][i] = plane q of Compress_mask(key_i), input row order.
 * mask: host u8[key_bytes]; packed_out: device u32[ceil(m/32)][n] (may be NULL if m=0).
 * Asynchronous. */
int cks_compress(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes,
                 const uint8_t* mask, uint32_t* packed_out);

/* ---- a4+a5: sort ------------------------------------------------------------
 * Stable LSD radix sort of (P, row id) by P, ties by row id (Theorem 2).
 * packed: device u32[ceil(packed_bits/32)][n] (not modified); packed_bits = m.
 * row_ids: device u32[n] or NULL (= 0..n-1). Non-NULL row ids are sorted first as the
 *   least significant digits, the paper's record-ID bits in the sort key.
 * perm_out: device u32[n]. sorted_packed_out: device planes like `packed`, or NULL.
 * Asynchronous. */
int cks_sort(cks_ctx* ctx, const uint32_t* packed, uint32_t packed_bits, uint64_t n,
             const uint32_t* row_ids, uint32_t* perm_out, uint32_t* sorted_packed_out);

/* ---- a6: adjacency / recompute ---------------------------------------------
 * Over sorted packed keys compressed with `sort_mask` (host u8[key_bytes], popcount =
 * packed_bits): D_i = D-offset[D-bit(Compress(key_{i-1}), Compress(key_i))] and the new
 * D-bitmap (a subset of sort_mask). mask_out: host u8[key_bytes];
 * popcount_out: host, may be NULL; dbit_out: device u16[n] or NULL. Synchronises. */
int cks_adjacent_dbits(cks_ctx* ctx, const uint32_t* sorted_packed, uint32_t packed_bits,
                       uint64_t n, const uint8_t* sort_mask, uint32_t key_bytes,
                       uint8_t* mask_out, uint32_t* popcount_out, uint16_t* dbit_out);

/* ---- NEXT-4: the sharded path -------------------------------------------
 * One process per GPU holds a shard of the key column; the pieces below are the per-shard
 * steps between the exchanges (the orchestration and the collectives are the caller's:
 * paper_2009_11543_b200/shard.py).
 *
 * cks_occupancy: a1's per-byte occupancy of this shard's keys -- bit (v & 31) of word
 * occ_out[j*8 + (v>>5)] set when byte value v occurs at byte position j (the set whose D-bits
 * form D+). occ_out: device u32[key_bytes*8], overwritten. Asynchronous. The union
 * over shards (bitwise OR; NCCL has no OR reduction, so: all-gather + cks_occupancy_mask)
 * is the occupancy of the whole column. */
int cks_occupancy(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes, uint32_t* occ_out);
/* The speculative mask of the sharded first build: cks_occupancy_sample
 * is the occupancy of `samples` rows strided over this shard (occ_out overwritten; keys of 8,
 * 16, 32 or 64 bytes, 16-byte aligned, else the whole shard's occupancy); cks_compress_marking
 * is cks_compress that also writes the shard's full occupancy to occ_out (overwritten) from the
 * same read of the keys (the same key widths; CKS_EINVAL otherwise). The union of the sampled
 * occupancies gives a mask M' inside the column's D+; when the union of the marked ones gives
 * the same D+, P_M' is the column's P_{D+}. Asynchronous. */
int cks_occupancy_sample(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes, uint32_t samples,
                         uint32_t* occ_out);
int cks_compress_marking(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes, const uint8_t* mask,
                         uint32_t* packed_out, uint32_t* occ_out);

/* cks_occupancy_mask: the superset mask of the union of `nocc` occupancies (device
 * u32[nocc][key_bytes*8], e.g. the all-gathered shard occupancies), n_total = keys over all
 * shards: kind CKS_SUPERSET_BYTEOCC -> D+ (as cks_superset_mask), CKS_SUPERSET_VARIANT -> V.
 * mask_out: host u8[key_bytes]; popcount_out: host, may be NULL. Synchronises. */
int cks_occupancy_mask(cks_ctx* ctx, const uint32_t* occ, uint32_t nocc, uint32_t key_bytes, uint64_t n_total,
                       int kind, uint8_t* mask_out, uint32_t* popcount_out);

/* cks_rank_sorted: for each query q (device u32[nq][np+1]: P's plane words 0..np-1 --
 * plane 0 least significant, as cks_compress -- then a row id) the number of elements of
 * a sorted (P, row id) sequence that are smaller than it (lower bound in the order of
 * Theorem 2 with the row-id tie-break). sorted_packed: device u32[np][n] (np =
 * ceil(packed_bits/32)), sorted_rid: device u32[n]; element i's row id is
 * rid_base + sorted_rid[i] (compared in 64 bits). ranks_out: device u64[nq].
 * Used to cut a locally sorted shard at the global splitters. Asynchronous. */
int cks_rank_sorted(cks_ctx* ctx, const uint32_t* sorted_packed, uint32_t packed_bits, uint64_t n,
                    const uint32_t* sorted_rid, uint64_t rid_base, const uint32_t* queries, uint32_t nq,
                    uint64_t* ranks_out);

/* cks_partition: stable partition of a shard's (P, row id) pairs by G-1 splitters (device
 * u32[G-1][np+1], the query layout of cks_rank_sorted, ascending): element i (row id
 * rid_base + i) goes to part d = the number of splitters <= (P_i, rid_base + i). Outputs, in
 * part order and within a part in input order: packed_out device u32[np][n], rid_out device
 * u32[n] (the row ids), counts_out device u64[G] (elements per part). One destination pass
 * plus one LSD digit pass on the part index (G <= 256). Since the parts keep the input
 * order, a receiver that concatenates the parts sent to it in source-rank order holds them in
 * row-id order, and a stable sort on P alone yields the (P, row id) order. Asynchronous. */
int cks_partition(cks_ctx* ctx, const uint32_t* packed, uint32_t packed_bits, uint64_t n, const uint32_t* splitters,
                  uint32_t parts, uint64_t rid_base, uint32_t* packed_out, uint32_t* rid_out, uint64_t* counts_out);

/* The fused partition-and-send (NEXT-4): the partition of cks_partition with
 * every part written straight into its receiver's buffer by the digit pass itself, instead of a
 * local partition followed by an all-to-all.
 * cks_partition_count: part of every element and the per-part counts (counts_out device
 * u64[parts]); keeps the partition input in the context for the send. The caller all-gathers
 * the counts (G x G), sizes the receive buffers and computes where its part starts in each.
 * cks_partition_send: the one stable digit pass on the part index of the last count on this
 * context; part d's planes go to dst_planes[d] + q * dst_pitch[d] (plane q, u32 elements from
 * this sender's start in receiver d's buffer) and its global row ids (rid_base + i) to
 * dst_rid[d]. dst_planes / dst_pitch / dst_rid are HOST arrays [parts] of DEVICE addresses:
 * peer pointers when the receiver is another GPU (cudaIpc / P2P; NVLink stores), plain device
 * pointers when it is on this one. Asynchronous; the receiver may read after the sender's
 * stream completes (the caller's barrier). */
int cks_partition_count(cks_ctx* ctx, const uint32_t* packed, uint32_t packed_bits, uint64_t n,
                        const uint32_t* splitters, uint32_t parts, uint64_t rid_base, uint64_t* counts_out);
int cks_partition_send(cks_ctx* ctx, uint32_t* const* dst_planes, const uint64_t* dst_pitch, uint32_t* const* dst_rid);

/* cks_sort_prefix: the first build's sort (a4-a6, by distinguishing prefixes as cks_build,
 * SURVEY 8(f) NEXT-1) on GIVEN compressed keys instead of key rows: packed = P_M, device
 * u32[ceil(m/32)][n] right-aligned as cks_compress, input order; sort_mask = M (host
 * u8[key_bytes], m = its popcount). Outputs: perm_out device u32[n] = input indices in
 * (P, index) order; dbit_out device u16[n] (D_i, first = CKS_DBIT_NONE); mask_out host
 * u8[key_bytes] = exact D of this sequence (a subset of M); popcount_out (may be NULL);
 * packed_out device u32[ceil(|D|/32)][n] = P_D in sorted order, or NULL to skip it. Used
 * after the sharded path's exchange (the received pairs are in row-id order, so the index
 * order is the row-id order). Synchronises. */
int cks_sort_prefix(cks_ctx* ctx, const uint32_t* packed, const uint8_t* sort_mask, uint32_t key_bytes, uint64_t n,
                    uint32_t* perm_out, uint16_t* dbit_out, uint8_t* mask_out, uint32_t* popcount_out,
                    uint32_t* packed_out);

/* cks_repack: P_D from P_M for D a subset of M (a7): packed_in device
 * u32[ceil(|M|/32)][n], packed_out device u32[ceil(|D|/32)][n], both right-aligned as
 * cks_compress, same element order. in_mask = M, out_mask = D: host u8[key_bytes].
 * Asynchronous (CKS_EINVAL if D is not a subset of M). */
int cks_repack(cks_ctx* ctx, const uint32_t* packed_in, const uint8_t* in_mask, const uint8_t* out_mask,
               uint32_t key_bytes, uint64_t n, uint32_t* packed_out);

/* ---- a8: bottom-up bulk load (Sec. 5.3) -----------------------------------------
 * Nodes have `fanout` slots filled with per_node = floor(fanout*fill) entries.
 * Level 0 = leaves; levels are concatenated leaves first (level_offset[l]).
 *   node_cnt[node]              entries used in the node
 *   entry_rid[node][fanout]     leaf: row id of the entry's key; inner: row id of the
 *                               highest key under the child
 *   entry_dbit[node][fanout]    leaf: D_i against the global predecessor;
 *                               inner: D-bit of the child's highest key vs the previous
 *                               entry's highest key at that level, computed as
 *                               the range-min of D_k (Lemma 1); CKS_DBIT_NONE for
 *                               the first entry of a level and for equal keys.
 *   entry_child[(node-level_offset[1])][fanout]  inner nodes only: global index of child
 * Empty slots hold 0xFFFFFFFF / CKS_DBIT_NONE. */
typedef struct {
    uint64_t n;
    uint32_t fanout;
    uint32_t per_node;
    uint32_t height;                          /* number of levels; 0 when n = 0 */
    uint32_t reserved;
    uint64_t level_nodes[CKS_MAX_LEVELS];
    uint64_t level_offset[CKS_MAX_LEVELS];
    uint64_t total_nodes;
    uint64_t inner_nodes;                     /* total_nodes - level_nodes[0] */
} cks_tree_shape;

typedef struct {
    uint32_t* node_cnt;                       /* device u32[total_nodes] */
    uint32_t* entry_rid;                      /* device u32[total_nodes*fanout] */
    uint16_t* entry_dbit;                     /* device u16[total_nodes*fanout] or NULL */
    uint32_t* entry_child;                    /* device u32[inner_nodes*fanout] or NULL */
} cks_tree;

/* Host-only arithmetic; no context needed. */
int cks_bulkload_shape(uint64_t n, uint32_t fanout, double fill, cks_tree_shape* out);

/* perm: device u32[n] (sorted row ids); dbit: device u16[n] D_i or NULL (then leaf and
 * inner D-bits are not produced: entry_dbit must be NULL too). Asynchronous. */
int cks_bulkload(cks_ctx* ctx, const uint32_t* perm, const uint16_t* dbit, uint64_t n,
                 uint32_t fanout, double fill, const cks_tree* out);

/* ---- NEXT-3: the paper's index tree format (Sec. 4.2; Sec. 5.3) -------
 * Nodes of 256 bytes, leaves first then each level up, numbered from 0; a node holds
 * floor(max fanout * fill) entries (leaf max 14, non-leaf max 9; fill 0.9 -> 12 / 8). Little-
 * endian layout:
 *   header (24 B)  u16 count | u16 level (0 = leaf) | u32 key_bytes | u64 highest key (record
 *                  id of the node's last key) | u64 0
 *   leaf           u64 next leaf (node index, all ones for the last leaf) at byte 24, then 14
 *                  entries of 16 B at 32 + 16 e: u32 partial key | u16 D_i | u16 key length |
 *                  u64 record id
 *   non-leaf       9 entries of 24 B at 24 + 24 e: u32 partial key | u16 D-bit | u16 key length
 *                  | u64 child node index | u64 highest key (record id)
 * Unused entries and bytes are 0. The partial key holds the pk_bits (<= 32) key bits at
 * positions D+1 .. D+pk (reading C14; 0 past the key), packed from bit 31 down, where D
 * is the entry's distinction bit position; with none (first key, equal keys) positions
 * 0 .. pk-1. A non-leaf entry's D-bit is that of its child's highest key against the previous
 * entry's highest key at the same level (CKS_DBIT_NONE for the first), equal to the
 * minimum D_k over the child's keys (Lemma 1).
 * cks_paper_tree_shape: host arithmetic; fanout = 14, per_node = leaf entries, reserved =
 * non-leaf entries. cks_paper_tree: keys device u8[n][key_bytes]; perm / dbit from cks_build;
 * nodes device u8[total_nodes][256]. Asynchronous. */
#define CKS_PTREE_NODE_BYTES 256
#define CKS_PTREE_LEAF_FANOUT 14
#define CKS_PTREE_INNER_FANOUT 9
int cks_paper_tree_shape(uint64_t n, double fill, cks_tree_shape* out);
int cks_paper_tree(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes, const uint32_t* perm,
                   const uint16_t* dbit, uint32_t pk_bits, double fill, uint8_t* nodes);

/* cks_paper_tree_ds: the same nodes (byte for byte), with every partial-key bit taken from the
 * source P:484-496 names instead of the key row:
 *   A  positions in packed_mask: from the sorted compressed planes (sorted_packed: device
 *      u32[ceil(|packed_mask|/32)][packed_pitch], right-aligned as cks_compress, in sorted order --
 *      e.g. cks_build_out.packed / packed_pitch with packed_mask = the exact D);
 *   B  invariant positions (0 in `variant`): from the reference key value (ref_key);
 *   C  the other variant positions: C(b), from the key row (keys; may be NULL when every variant
 *      position is in packed_mask, CKS_EINVAL otherwise), read only by entries whose window
 *      holds such a position.
 * variant / ref_key: host u8[key_bytes], the DS-metadata of the column (cks_build_out.variant /
 * ref_key). Asynchronous. */
int cks_paper_tree_ds(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes, const uint32_t* perm,
                      const uint16_t* dbit, const uint32_t* sorted_packed, uint64_t packed_pitch,
                      const uint8_t* packed_mask, const uint8_t* variant, const uint8_t* ref_key, uint32_t pk_bits,
                      double fill, uint8_t* nodes);

/* ---- P:502 block-parallel bulk load (the sharded path's a8, NEXT-4) ----------------------
 * "n sort keys are divided into p blocks ... thread i constructs a subtree consisting of all
 * sort keys in the i-th block. ... we remove the root nodes of the subtrees, and build the
 * top layers of the whole tree by linking the children of the root nodes".
 *
 * cks_bulkload_block: levels 0 .. levels-1 (levels = 0: all) of the subtree over one block:
 * perm / dbit = the block's slice of the global sorted order (D_i against the GLOBAL
 * predecessor). Layout and entries as cks_bulkload over the block's own shape, except that
 * with first_global = 0 (a block after the first) the first entry of every inner level takes
 * its child's minimum D_k like every other entry (its predecessor lives in the previous
 * block). top_min_out: device u16[nodes of the top built level] = minimum D_k under each of
 * those nodes (input of the merge), or NULL. height_out: levels built. Asynchronous. */
int cks_bulkload_block(cks_ctx* ctx, const uint32_t* perm, const uint16_t* dbit, uint64_t n, uint32_t fanout,
                       double fill, int first_global, uint32_t levels, cks_tree* out, uint16_t* top_min_out,
                       uint32_t* height_out);

/* cks_bulkload_top: the merged top over nchild child nodes = the blocks' top built levels
 * concatenated in block order (child_rid: device u32[nchild], row id of each child's highest
 * key; child_min: device u16[nchild], minimum D_k under each child). The first level above
 * them has ceil(nchild/per) nodes whose entries are the children (entry_child = index into
 * the child list; entry D-bit = child_min, CKS_DBIT_NONE for the first child), then upward
 * to one root as cks_bulkload. Node ids start at 0 on that first level; arrays sized for
 * cks_bulkload_shape(nchild, fanout, fill).total_nodes nodes (entry_child for all of them);
 * nchild <= 1 builds nothing (the one child is the root). height_out: levels built.
 * Asynchronous. */
int cks_bulkload_top(cks_ctx* ctx, const uint32_t* child_rid, const uint16_t* child_min, uint64_t nchild,
                     uint32_t fanout, double fill, cks_tree* out, uint32_t* height_out);

/* ---- fused first build: a1 -> a2 -> a3 -> a4 -> a5 -> a6 -> a7 -> a8 -----------------------
 * The benchmarked step. The superset mask M (or prior_mask) is compressed once; the sort
 * runs by distinguishing prefixes ("sort by distinguishing prefixes",
 * P:603): LSD over the first 64 bits of P_M for all keys, then only the keys still tied
 * with a neighbour are re-sorted by (run, next 64 bits), round after round. A pair's D-bit
 * comes from the round that separates it, so the exact D and the D_i fall out of the sort;
 * P_D in sorted order is then compressed from the key rows (or repacked from the sorted
 * chunk when one chunk held all of P_M); bulk load. cks_ctx_set_sort_mode(CKS_SORT_SINGLE)
 * selects the plain single sort over all m bits (one adjacency pass, repack skipped when
 * M = D). */
typedef struct {
    /* inputs (caller-owned buffers) */
    uint8_t* mask;            /* host u8[key_bytes]: receives exact D */
    uint32_t* perm;           /* device u32[n] */
    uint16_t* dbit;           /* device u16[n] or NULL (library scratch is used) */
    cks_tree tree;            /* device arrays, or node_cnt == NULL to skip the bulk load */
    uint32_t fanout;          /* bulk load fanout (>= 2) */
    double fill;               /* bulk load fill in (0, 1] */
    int superset_kind;        /* CKS_SUPERSET_BYTEOCC (default) or CKS_SUPERSET_VARIANT */
    /* outputs */
    uint32_t popcount;        /* |D| */
    uint32_t sort_bits;       /* |M|, the width the sort ran on */
    uint32_t height;          /* tree height (0 if skipped) */
    uint32_t passes;          /* LSD digit passes run */
    const uint32_t* packed;   /* VIEW (ctx-owned): sorted P_D planes; plane q at packed + q*packed_pitch */
    uint64_t packed_pitch;    /* plane stride of `packed` in u32 elements (>= n, padded for alignment) */
    uint32_t rounds;          /* prefix-refinement rounds run (0 = plain single sort) */
    uint32_t round0_bits;     /* width of the first refinement round (top bits of P_M) */
    uint64_t refined_keys;    /* keys re-sorted in rounds >= 1 (summed over rounds) */
    /* DS-metadata recompute at (re)build time, optional:  */
    uint8_t* variant;         /* host u8[key_bytes] or NULL: receives the variant bitmap V =
                                 OR over the keys of key XOR reference key; a first build
                                 takes it from the superset pass, a rebuild (prior mask) runs one
                                 more pass over the keys for it */
    uint8_t* ref_key;         /* host u8[key_bytes] or NULL: receives the reference key value,
                                 the key of row 0 ("an arbitrary index key") */
    /* NEXT-3, optional: the paper-format index tree (cks_paper_tree's layout, identical bytes)
     * built by the same call from the sorted order; partial-key bits from the sources of
     * P:484-496 chosen by ptree_source:
     *   CKS_PTREE_AUTO   DECODE when it applies, else ROWS (the default);
     *   CKS_PTREE_DECODE source A alone: on a first build the sort mask is D+, whose bits at a
     *                    byte position tell the byte values occurring there apart, so the
     *                    sorted P_{D+} determines every key bit (per-byte decode tables from the
     *                    superset pass; no row reads, no extra plane). Applies when the sort mask
     *                    holds the keys' D+ (a first build, D+ or V; a rebuild whose prior mask
     *                    the D+ test of CKS_VERIFY_PRIOR proved), the build keeps P_M sorted (at
     *                    most 96 mask bits, or the single-sort mode) and the tables (sum over
     *                    bytes of 2^|mask bits of the byte|) fit 64 KB; otherwise CKS_EINVAL;
     *   CKS_PTREE_ROWS   C(b): every bit from the key row (random row reads);
     *   CKS_PTREE_DS     A from the sorted P_D, B from the reference key for invariant bits, C(b)
     *                    rows only for the variant bits outside D;
     *   CKS_PTREE_CARRY  as DS, with C(a): the variant bits outside the sort mask that some
     *                    partial key needs are compressed into one more plane that rides through
     *                    the sort with P_M (when P_M has three planes and they fit one plane), so
     *                    the tree reads no rows.
     * cks_paper_tree_shape(n, ptree_fill) gives the node count. */
    uint8_t* ptree_nodes;     /* device u8[total_nodes][256] or NULL (no paper tree) */
    uint32_t ptree_pk;        /* partial key bits (<= 32) */
    uint32_t ptree_source;    /* CKS_PTREE_AUTO (0) / _ROWS (1) / _DS (2) / _CARRY (3) / _DECODE (4) */
    double ptree_fill;        /* fill factor in (0, 1] */
    uint8_t* sort_mask;       /* host u8[key_bytes] or NULL: receives the mask the sort ran on (the
                                 first build's D+ or V, the prior mask of a rebuild) */
} cks_build_out;

#define CKS_PTREE_AUTO 0
#define CKS_PTREE_ROWS 1
#define CKS_PTREE_DS 2
#define CKS_PTREE_CARRY 3
#define CKS_PTREE_DECODE 4

/* keys: device u8[n][key_bytes]; prior_mask: host u8[key_bytes] superset or NULL.
 * A prior mask must contain every distinction bit of THIS column (e.g. the D-bitmap of the
 * last build when no key was inserted since); with the default order check a mask
 * that does not returns CKS_ERANGE (see cks_ctx_set_verify).
 * Without a prior mask, columns of at least 2^20 keys of 32 or 64 bytes (16-byte aligned)
 * take the sort mask from a strided sample of 65536 rows and the compress marks every key's
 * byte occupancy on the way; the column's D+ is compared with the sample's at the end and the
 * build is run again by it when they differ. The result is the same as with a separate
 * superset pass; sort_bits reports the mask finally used.
 * Synchronises: after the superset mask, once per refinement round (to size the next
 * round), after the exact D is known, and after the order check when it runs. */
int cks_build(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t key_bytes,
              const uint8_t* prior_mask, cks_build_out* out);

/* Same as cks_build with HOST buffers: host_keys u8[n][key_bytes] (pinned or pageable)
 * is copied to ctx-owned device memory in chunks that overlap the superset-mask pass;
 * out->perm is a HOST u32[n] filled by a device->host copy; out->dbit and out->tree
 * must be NULL/skipped (device-side results stay in ctx scratch). Synchronises. */
int cks_build_host(cks_ctx* ctx, const uint8_t* host_keys, uint64_t n, uint32_t key_bytes,
                   const uint8_t* prior_mask, cks_build_out* out);

/* cks_build_host_batch: `count` fused builds of HOST key columns (pinned u8[n][key_bytes]
 * each, host_keys[i]), pipelined: column i+1 is copied to the device (copy stream) while
 * column i builds and column i-1's permutation returns (a second copy stream), so the two PCIe
 * directions and the build overlap; two device key buffers and two permutation buffers are
 * context-owned. outs[i] as cks_build_host (mask, perm = host u32[n]; dbit and tree NULL);
 * outs[i].packed is NULL on return. Synchronises at the end. */
int cks_build_host_batch(cks_ctx* ctx, const uint8_t* const* host_keys, uint32_t count, uint64_t n,
                         uint32_t key_bytes, const uint8_t* prior_mask, cks_build_out* outs);

#ifdef __cplusplus
}
#endif
#endif /* CKS_H */
