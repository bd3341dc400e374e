// cks_internal.h -- shared declarations of the libcks kernels and the host layer.
// Not part of the public ABI (that is include/cks.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define CKS_NONE_INTERNAL 0xFFFFu

// Checked build (-DCKS_CHECKED=1, lib/libcks_checked.so; the pool has no compute-sanitizer):
// device-side bounds assertions at the computed-index stores, poisoned scratch and canary
// bands after every scratch buffer (cks_api.cu). The product build compiles them out.
#if defined(CKS_CHECKED) && CKS_CHECKED
#include <assert.h>
#define CKS_DCHECK(c) assert(c)
#else
#define CKS_DCHECK(c) ((void)0)
#endif

namespace cks {

constexpr uint32_t kMaxKeyBytes = 512;
constexpr uint32_t kMaxBits = 8 * kMaxKeyBytes;
constexpr uint32_t kMaxWords = kMaxKeyBytes / 4;        // 32-bit words per key
constexpr uint32_t kMaxPlanes = kMaxBits / 32;          // u32 planes of a packed key
constexpr int kSortThreads = 256;                       // one thread per 8-bit digit value
constexpr int kRadix = 256;

// One step of the word-level bit gather (Sec. 5.1 PEXT, done in software):
// the bits of source word `src` selected by `mask` are moved to the low end of the
// word with five masked shifts (mv[s] selects the bits that move right by 2^s; the
// classic parallel-suffix compress), giving `cnt` bits. Steps are listed from the
// least significant end of P upward, so a thread just appends `cnt` bits each step.
struct GatherStep {
    uint32_t src;      // compress: 32-bit big-endian word index in the key; repack: plane index
    uint32_t mask;
    uint32_t mv[5];
    uint32_t cnt;
};

struct GatherPlan {
    uint32_t nsteps;
    uint32_t out_bits;     // total bits = sum cnt
    GatherStep step[kMaxWords > kMaxPlanes ? kMaxWords : kMaxPlanes];
};

// Raise a kernel's dynamic shared-memory limit on the current device to at least `bytes`.
// Never lowers it: one record per (device, kernel) shared by every launch site (cks_plan.cpp).
cudaError_t raise_smem_limit(const void* kernel, size_t bytes);

// Tuning knobs (cks_plan.cpp). Fixed defaults in the product build: the library reads no
// environment. Built with -DCKS_EXPERIMENTS=1 (CKS_EXPERIMENTS=1 python -m
// paper_2009_11543_b200._build) the timing-experiment variables CKS_LSD_ITEMS / _SLOTS /
// _CHUNK / _WS / _DEBUG (the last makes results WRONG), CKS_REF_CTA, CKS_NO_TILE_RUNS,
// CKS_NO_KERNEL_EVENTS and CKS_REFINE_LOG override them. Initialised once (std::call_once),
// read-only afterwards, so concurrent host threads see one consistent set.
struct Knobs {
    int lsd_items = 16;        // keys per thread of the LSD tile (8 or 16)
    int lsd_slots = 4;         // ring slots of the non-specialised downsweep
    int lsd_chunk = 0;         // tiles per upsweep CTA (0 = by size)
    int lsd_ws = 1;            // warp-specialised downsweep on full tiles
    int lsd_debug = 0;         // timing-only modes with wrong results (experiments build only)
    int ref_cta = 2048;        // longest run one CTA sorts in the refinement
    int spec_mask = 1;         // first build: mask from a row sample, occupancy marked by the compress
    bool no_tile_runs = false; // round-0 adjacency without in-tile run finishing
    bool no_kernel_events = false;
    bool refine_log = false;
};
const Knobs& knobs();

// Host-side planning (cks_plan.cpp).
void plan_compress(const uint8_t* mask, uint32_t key_bytes, GatherPlan* plan);
void move_masks_left(uint32_t mask, uint32_t mv[5]);
void plan_repack(const uint32_t* sub_words /* u32[np_in], bit b of word q = P_M bit 32q+b kept */,
                 uint32_t np_in, GatherPlan* plan);

// ---- kernel launchers (stream-ordered, return cudaGetLastError) ------------------
cudaError_t launch_occupancy(const uint8_t* keys, uint64_t n, uint32_t B, uint32_t* occ,
                             int sms, cudaStream_t st);
cudaError_t launch_occ_finalize(const uint32_t* occ, uint32_t B, uint64_t n, uint8_t* dplus,
                                uint8_t* variant, cudaStream_t st);
// First-round width of the refinement: compresses a strided sample of `samples` keys (power
// of two, <= 16384) with the compress plan, sorts their top-64-bit prefixes of P_M in one CTA
// and writes counts[w] = distinct prefixes of the top 8(w+1) bits, w = 0..7.
cudaError_t launch_prefix_sample(const uint8_t* keys, uint64_t n, uint32_t B, const GatherPlan* plan, uint32_t samples,
                                 uint32_t* counts, cudaStream_t st, const uint32_t* pm = nullptr,
                                 uint32_t np = 0, uint64_t pitch = 0);
// Planes are u32 SoA arrays: plane q of a packed array starts at ptr + q*pitch (pitch in
// elements; user buffers have pitch n, library scratch pads the pitch to 32 elements so every
// plane is 128-byte aligned for TMA).
// lead: P is stored shifted left by `lead` bits (left-aligned planes when lead = 32*np - m);
// rows != NULL: key i is keys[rows[i]] (compress in a given order).
cudaError_t launch_compress(const uint8_t* keys, uint64_t n, uint32_t B, const GatherPlan* dplan,
                            const GatherPlan* hplan, uint32_t out_planes, uint32_t* planes, uint64_t pitch,
                            int sms, cudaStream_t st, uint32_t lead = 0, const uint32_t* rows = nullptr,
                            uint32_t* occ = nullptr);
// occ != NULL (no row list): the compress also ORs every key byte's occupancy into occ
// (u32[B][8]) -- the fixed widths only (compress_marks_occupancy)
bool compress_marks_occupancy(const uint8_t* keys, uint32_t B);
// occupancy (u32[B][8], OR-ed in) of `samples` rows strided over the n keys (B in 8/16/32/64)
cudaError_t launch_occupancy_sample(const uint8_t* keys, uint64_t n, uint32_t B, uint32_t samples, uint32_t* occ,
                                    cudaStream_t st);
cudaError_t launch_repack(const uint32_t* in_planes, uint64_t in_pitch, uint64_t n, const GatherPlan* dplan,
                          uint32_t nsteps, uint32_t out_planes, uint32_t* out, uint64_t out_pitch, int sms,
                          cudaStream_t st, const uint32_t* rows = nullptr);
// Reduce-then-scan LSD pass (k_lsd.cu): upsweep -> chunk scan -> persistent downsweep.
struct LsdPassArgs {
    const uint32_t* in_planes;
    uint32_t* out_planes;
    const uint32_t* in_rid;      // NULL = implicit row id (input index)
    uint32_t* out_rid;
    uint64_t n;
    uint64_t in_pitch;
    uint64_t out_pitch;
    uint32_t nplanes;
    int32_t digit_plane;         // -1 = digit taken from the row id
    uint32_t shift;
    uint32_t* tile_off;          // u32[tiles][256] scratch
    uint32_t* chunk_tot;         // u32[chunks][256] scratch
    uint32_t* total;             // u32[256] scratch
    uint32_t chunk_tiles;        // set by the launcher
    uint32_t slots;              // set by the launcher
    uint32_t tma;                // set by the launcher
    uint32_t tile_begin;         // first tile this launch covers (set by the launcher)
    uint32_t debug;              // timing experiments only (CKS_LSD_DEBUG); results are wrong when set
    uint32_t rid_add;            // added to implicit row ids as they are written
    // scatter-to-parts (fused partition-and-send, k_lsd.cu SCATTER): stream k >= 1 of an element
    // of part d is written to part_dst[(k-1)*256 + d][its position - bbase[d]]; NULL = off
    uint32_t* const* part_dst;
    uint32_t* bbase;             // u32[256] bucket bases, written by the chunk scan when non-NULL
};
// optional side stream for the partial last tile (runs concurrently with the full tiles)
struct LsdAux {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    // timing of the dominant kernel (the warp-specialised downsweep): events recorded around
    // it when non-null; *ws_bytes receives its algorithmic bytes (0 if it did not run)
    cudaEvent_t ws_begin = nullptr, ws_end = nullptr;
    double* ws_bytes = nullptr;
};
cudaError_t launch_lsd_pass(const LsdPassArgs& a, int sms, cudaStream_t st, const LsdAux& aux, int* launches);
void lsd_sizes(uint64_t n, uint64_t* tiles, uint64_t* chunks);

cudaError_t launch_adjacent(const uint32_t* planes, uint64_t pitch, uint64_t n, uint32_t m, const uint16_t* moff,
                            uint32_t B, uint16_t* dbit_out, uint32_t* dacc /* u32[ceil(8B/32)] */,
                            int sms, cudaStream_t st);
cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t st);
// Order check (k_verify.cu): *first_bad = smallest sorted position i >= 1 whose pair
// (perm[i-1], perm[i]) is not in (key, row id) order, or all ones when there is none.
cudaError_t launch_verify_order(const uint8_t* keys, uint32_t B, const uint32_t* perm, uint64_t n,
                                unsigned long long* first_bad, int sms, cudaStream_t st);

// NEXT-1 prefix refinement (k_refine.cu)
uint64_t ref_tiles(uint64_t nr);
cudaError_t launch_part_dest(const uint32_t* planes, uint32_t np, uint64_t n, uint64_t pitch, const uint32_t* spl,
                             uint32_t nspl, uint64_t rid_base, uint32_t* dest, unsigned long long* counts, int sms,
                             cudaStream_t st);
cudaError_t launch_align_left(const uint32_t* in, uint64_t in_pitch, uint32_t np, uint64_t n, uint32_t lead,
                              uint32_t* out, uint64_t out_pitch, int sms, cudaStream_t st);
cudaError_t launch_add_base(uint32_t* a, uint64_t n, uint32_t base, int sms, cudaStream_t st);
cudaError_t launch_occ_union(const uint32_t* occ, uint32_t nocc, uint32_t words, uint32_t* out, cudaStream_t st);
cudaError_t launch_rank_sorted(const uint32_t* planes, uint32_t np, uint64_t n, const uint32_t* rid, uint64_t rid_base,
                               const uint32_t* q, uint32_t nq, unsigned long long* ranks, cudaStream_t st);
cudaError_t launch_ref_tile(const uint32_t* pm, uint64_t pitch, uint32_t np, int qtop, uint32_t fmask,
                            const uint16_t* moff, uint32_t* perm, uint16_t* dbit, uint32_t* carried, const uint32_t* lo,
                            const uint32_t* hi, uint64_t hpitch, uint64_t n, unsigned long long cmask, uint32_t B,
                            uint8_t* tie, uint32_t* dacc, uint32_t* handled, int sms, cudaStream_t st, uint8_t* any);
cudaError_t launch_ref_adj(const uint32_t* lo, const uint32_t* hi, const uint32_t* seg, const uint32_t* pos,
                           uint64_t nr, uint32_t cbase, const uint16_t* moff, uint32_t m, uint32_t B,
                           uint16_t* dbit, uint8_t* tie, uint32_t* dacc, bool round0, int sms, cudaStream_t st,
                           unsigned long long cmask = ~0ull);
// run_off / run_pos (NULL: not needed): list index and global position of each run's first key
cudaError_t launch_ref_compact(const uint8_t* tie, uint64_t nr, const uint32_t* pos, uint32_t* cnt, uint32_t* tot,
                               uint32_t* pos_next, uint32_t* seg_next, uint32_t* run_off, uint32_t* run_pos,
                               cudaStream_t st, const uint8_t* any = nullptr);
cudaError_t launch_ref_local(const uint32_t* pm, uint64_t pitch, uint32_t np, int qtop, const uint16_t* moff,
                             const uint32_t* run_pos, const uint32_t* seg, const uint32_t* run_off, uint64_t nseg,
                             uint64_t nn, uint32_t* perm, uint16_t* dbit, uint32_t* dacc, uint8_t* done, uint8_t* keep,
                             uint32_t* carried, uint32_t B, uint32_t* mlist, uint32_t* wlist, uint32_t* mcount, int sms,
                             cudaStream_t st, uint32_t fmask);
cudaError_t launch_ref_keep(const uint32_t* seg, const uint32_t* run_off, const uint8_t* done, uint64_t nn,
                            uint8_t* keep, int sms, cudaStream_t st);
cudaError_t launch_ref_gather(const uint32_t* pm, uint64_t pitch, uint32_t np, uint32_t o, const uint32_t* pos,
                              const uint32_t* seg, const uint32_t* perm, uint64_t nr, uint32_t* out, uint64_t opitch,
                              uint32_t* orid, int sms, cudaStream_t st);
// a refinement round without LSD passes when every long run holds at most kChunkCta keys
constexpr uint32_t kChunkCtaKeys = 4096;
cudaError_t launch_ref_cta_chunk(const uint32_t* pm, uint64_t pitch, uint32_t np, uint32_t o, const uint32_t* perm,
                                 const uint32_t* run_off, const uint32_t* run_pos, uint64_t nseg, uint64_t nn,
                                 uint32_t* out, uint64_t opitch, uint32_t* orid, int sms, cudaStream_t st);
cudaError_t launch_ref_refresh(const uint32_t* list, uint64_t nr, const uint32_t* perm, const uint32_t* pm,
                              uint64_t pitch, uint32_t np, uint32_t np0, uint32_t* sorted, uint64_t spitch, int sms,
                              cudaStream_t st);
cudaError_t launch_ref_put(uint32_t* perm, const uint32_t* pos, const uint32_t* rid, uint64_t nr, const uint32_t* pm,
                           uint64_t pitch, uint32_t np, uint32_t* carried, int sms, cudaStream_t st);
cudaError_t launch_fill_u16(uint16_t* out, uint64_t n, uint16_t v, cudaStream_t st);

struct BulkLevel {
    uint64_t entries;      // entries at this level (= n for leaves, nodes below otherwise)
    uint64_t nodes;
    uint64_t node_off;     // global node index of the first node of the level
    uint64_t below_off;    // global node index of the first node of the level below
    uint64_t span;         // sorted keys covered per entry
};
cudaError_t launch_bulk_leaves(const uint32_t* perm, const uint16_t* dbit, const BulkLevel& L,
                               uint32_t fanout, uint32_t per, uint32_t* node_cnt, uint32_t* rid,
                               uint16_t* edbit, uint16_t* rmin, int sms, cudaStream_t st);
cudaError_t launch_bulk_inner(const uint32_t* perm, const uint16_t* rmin_below, const BulkLevel& L,
                              uint64_t n, uint32_t fanout, uint32_t per, uint32_t* node_cnt,
                              uint32_t* rid, uint16_t* edbit, uint32_t* child, uint64_t inner_off,
                              uint16_t* rmin, int sms, cudaStream_t st, bool first_none = true);

// NEXT-3 paper-format index tree (k_ptree.cu). ds == NULL: partial keys from the key rows;
// else from the DS-metadata sources (sorted compressed planes, reference key, rows only for
// variant positions outside the planes' mask).
// Per window start p0 (= D + 1, 0 for none; 8B + 1 entries): the pk-bit window's positions in X
// and in Y, its invariant bits taken from the reference key, the variant positions in neither
// (read from the rows), and the rank in X / Y of the window's first position.
struct PtreeEnt {
    uint32_t wx, wy, refb, wc, rx, ry;
};
struct PtreeDs {
    const uint32_t* planes;    // sorted compressed planes: segment X (mask X) then Y (mask Y)
    uint64_t pitch;
    uint32_t np;
    uint32_t gx, gy;           // first bit of X / Y counted from the MSB of the np planes
    const PtreeEnt* ent;       // device table, 8B + 1 entries
};
// Per-level scratch of the tree build (every array sized by the leaf count + 16): the node
// minima of D_k (rmin), per node {partial key of its highest key at the node's minimum D-bit,
// highest key's row id} (sum) for the level above, and the plane words / row id of each leaf's
// highest key (hk, hr) captured by the leaf kernel.
struct PtreeWs {
    uint16_t* rmin[2];
    uint2* sum[2];
    uint4* hk;
    uint32_t* hr;
};
// partial keys decoded from the sorted P_{D+} alone (k_ptree.cu PkDec). pj: per byte j0 a uint4
// {g | c_i << (12 + 4 i), off_0 | off_1 << 16, off_2 | off_3 << 16, off_4} for the bytes j0 .. j0+4
// (g = first M bit of byte j0 from the MSB of the planes, c_i = M bits of byte j0+i, off_i = its
// values in dec; bytes past the key: c = 0, off = the zero byte at dec[dec_bytes - 1]).
cudaError_t launch_ptree_decode(uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit, uint32_t pk,
                                uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                                const uint64_t* level_offset, uint32_t height, uint8_t* nodes, const PtreeWs& ws,
                                int sms, cudaStream_t st, int* launches, const uint32_t* planes, uint64_t pitch,
                                uint32_t np, const uint4* pj, const uint8_t* dec, uint32_t dec_bytes);
cudaError_t launch_ptree(const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit,
                         uint32_t pk, uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                         const uint64_t* level_offset, uint32_t height, uint8_t* nodes, const PtreeWs& ws, int sms,
                         cudaStream_t st, int* launches, const PtreeDs* ds = nullptr);

}  // namespace cks
