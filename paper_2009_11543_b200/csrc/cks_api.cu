// cks_api.cu -- the C ABI of libcks.so (include/cks.h): argument checks, scratch
// management, host planning and the stream-ordered launch sequence of each call.
// Every step of the path runs in the kernels of k_*.cu; the host only plans (mask ->
// gather masks / D-offset table, a few hundred bytes) and orchestrates.
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/cks.h"
#include "cks_internal.h"

using namespace cks;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

enum Stage { ST_BEGIN = 0, ST_MASK, ST_COMPRESS, ST_HIST, ST_SORT, ST_ADJ, ST_REPACK, ST_BULK, ST_N };

}  // namespace

struct cks_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaStream_t d2h_stream = nullptr;    // cks_build_host_batch: results back while the next copies in
    cudaEvent_t bev[6] = {};              // cks_build_host_batch: keys in / build done / perm out, x2
    cudaStream_t aux_stream = nullptr;   // partial tail tile of an LSD pass
    cudaEvent_t aux_ev[2] = {};
    // dominant-kernel timing (cks_ctx_kernel_stats): event pairs around each warp-specialised
    // downsweep of the last timed build, and their algorithmic bytes
    static constexpr int kMaxKev = 128;
    cudaEvent_t kev[2 * kMaxKev] = {};
    double kbytes[kMaxKev] = {};
    int nkev = 0;
    char err[512] = {0};
    uint64_t launches = 0;
    bool timing = false;
    bool timed = false;
    cudaEvent_t ev[ST_N] = {};
    cudaEvent_t plan_ev[3] = {};      // guards the pinned staging slots
    // scratch
    DevBuf occ, occ_s, masks8, planeA, planeB, ridA, ridB, dacc, moff, dbit,
        rmin0, rmin1, plan[3], keys, perm_scratch, tile_off, chunk_tot, total,
        pm, pd, cmp, crid, crid2, posA, posB, posC, segA, segB, segC, runoff, runpos, runoff2, runpos2, tie, keep, done, mlist, wlist, rcnt, rtot,   // NEXT-1
        part_in, part_out,                                                 // NEXT-4
        anyt,                                                              // k_ref_reg: compaction tiles with ties left
        vbad,                                                              // k_verify_order result
        ptab,                                                              // cks_paper_tree_ds tables
        pdec,                                                              // decode tree tables
        rlist,                                                             // round 1's tied positions (a7)
        psum0, psum1, phk, phr,                                            // paper-tree level summaries
        part_ptrs,                                                         // cks_partition_send pointer table
        keys2, perm2;                                                      // cks_build_host_batch: 2nd buffers
    // pinned host staging
    GatherPlan* h_plan[3] = {};       // 0: compress, 1: repack, 2: partial-key bits (P_E)
    uint16_t* h_moff = nullptr;
    uint32_t* h_small = nullptr;      // 4 KiB: masks, dacc words
    uint32_t* h_tot = nullptr;        // refinement: (members, runs) of the next round
    int refine = CKS_SORT_PREFIX_AUTO; // first build by distinguishing prefixes (NEXT-1)
    uint32_t round0_bits = 0;         // forced width of refinement round 0 (0 = sampled)
    int verify = CKS_VERIFY_PRIOR;    // order check of the result against the key rows
    uint32_t* spec_occ = nullptr;     // speculative first build: the compress marks the occupancy here
    uint64_t spec_retries = 0;        // ... builds redone because the sample's mask fell short
    uint64_t spec_builds = 0;         // ... builds that took the speculative mask
    bool spec_on = true;              // cks_ctx_set_speculative_mask
    bool spec_pending = false;        // ... the full D+ / V are on their way to h_small + 4096
    std::vector<uint8_t> proof_mask;  // rebuild: prior mask whose D+ test rides on the compress
    cudaEvent_t spec_ev = nullptr;
    bool verify_now = false;          // ... for the build in progress
    std::vector<uint8_t> unproven;    // the last prior mask the D+ test could not prove
    double path_bytes = 0.0;          // algorithmic bytes of every kernel of the last build
    std::vector<uint8_t> pt_E;        // fused paper tree: partial-key bits appended to P_M (C(a))
    bool pt_on = false;
    uint32_t pt_npe = 0;              // planes actually appended by the last build_refine
    // where the last build left P_M in sorted order (carried / single sort), for the decode tree
    const uint32_t* spm = nullptr;
    uint64_t spm_pitch = 0;
    uint32_t spm_np = 0, spm_g0 = 0;
    PtreeEnt* h_ptab = nullptr;       // pinned staging of the paper tree's per-window table
    uint64_t ps_n = 0, ps_rid_base = 0; // cks_partition_count -> cks_partition_send state
    uint32_t ps_np = 0, ps_parts = 0;
    cudaEvent_t ptab_ev = nullptr;
    bool skip_packed = false;         // cks_sort_prefix without packed_out: no a7
};

namespace {

int fail(cks_ctx* c, int code, const char* fmt, ...) {
    if (c) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(c->err, sizeof(c->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, CKS_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                              \
    } while (0)

#define LAUNCH(expr)        \
    do {                    \
        ctx->launches++;    \
        CK(expr);           \
    } while (0)

// algorithmic bytes of a launch (what it must read + write at least), summed per build
#define BYTES(x) (ctx->path_bytes += (double)(x))

#define TRY(expr)                   \
    do {                            \
        int r_ = (expr);            \
        if (r_ != CKS_OK) return r_; \
    } while (0)

#if defined(CKS_CHECKED) && CKS_CHECKED
#define CKS_CHECKED_BUILD 1
constexpr size_t kGuardBytes = 4096;
constexpr int kPoison = 0xA5, kCanary = 0x5A;
#else
#define CKS_CHECKED_BUILD 0
#endif

int ensure(cks_ctx* ctx, DevBuf& b, size_t bytes, bool zero = false) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return CKS_OK;
    if (b.p) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
#if CKS_CHECKED_BUILD
    // checked build: no headroom, a canary band after the buffer and poisoned contents, so a
    // write past the end or a read of never-written scratch changes a result (check_guards)
    size_t cap = bytes;
    cudaError_t e = cudaMalloc(&b.p, cap + kGuardBytes);
#else
    size_t cap = bytes + bytes / 8;                          // a little headroom
    cudaError_t e = cudaMalloc(&b.p, cap);
#endif
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, CKS_ENOMEM, "cudaMalloc(%zu): %s", cap, cudaGetErrorString(e));
    }
    b.cap = cap;
#if CKS_CHECKED_BUILD
    CK(cudaMemsetAsync(b.p, kPoison, cap, ctx->stream));
    CK(cudaMemsetAsync((uint8_t*)b.p + cap, kCanary, kGuardBytes, ctx->stream));
#endif
    if (zero) CK(cudaMemsetAsync(b.p, 0, cap, ctx->stream));
    return CKS_OK;
}

template <class T>
T* as(DevBuf& b) { return reinterpret_cast<T*>(b.p); }

// speculative first build (build_common): sampled rows for the mask, smallest column
constexpr uint32_t kSpecSamples = 65536;
constexpr uint64_t kSpecMinKeys = 1u << 20;
constexpr uint32_t kSpecMinB = 32;                // (8-byte keys: cfg2 0.556 ms without, 0.560 with)
constexpr size_t kSpecHostOff = 4096;             // the full D+ and V in h_small (2B bytes)

// right after the speculative compress: the keys' D+ and V from the occupancy it marked, copied
// to the host behind the build (checked at its end without a stall)
int spec_enqueue(cks_ctx* ctx, uint64_t n, uint32_t B) {
    LAUNCH(launch_occ_finalize(as<uint32_t>(ctx->occ), B, n, as<uint8_t>(ctx->masks8), as<uint8_t>(ctx->masks8) + B,
                               ctx->stream));
    CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(ctx->h_small) + kSpecHostOff, ctx->masks8.p, (size_t)B * 2,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(ctx->spec_ev, ctx->stream));
    ctx->spec_pending = true;
    return CKS_OK;
}

// the paper tree's per-level scratch, sized by the leaf count
int ptree_ws(cks_ctx* ctx, uint64_t nleaves, PtreeWs* ws) {
    TRY(ensure(ctx, ctx->rmin0, (size_t)nleaves * 2 + 16));
    TRY(ensure(ctx, ctx->rmin1, (size_t)nleaves * 2 + 16));
    TRY(ensure(ctx, ctx->psum0, (size_t)nleaves * 8 + 16));
    TRY(ensure(ctx, ctx->psum1, (size_t)nleaves * 8 + 16));
    TRY(ensure(ctx, ctx->phk, (size_t)nleaves * 16 + 16));
    TRY(ensure(ctx, ctx->phr, (size_t)nleaves * 4 + 16));
    *ws = PtreeWs{{as<uint16_t>(ctx->rmin0), as<uint16_t>(ctx->rmin1)}, {as<uint2>(ctx->psum0), as<uint2>(ctx->psum1)},
                  as<uint4>(ctx->phk), as<uint32_t>(ctx->phr)};
    return CKS_OK;
}

// every scratch buffer of a context
#define CKS_SCRATCH_LIST(c)                                                                                      \
    {&c->occ, &c->occ_s, &c->masks8, &c->planeA, &c->planeB, &c->ridA, &c->ridB, &c->dacc, &c->moff, &c->dbit, &c->rmin0, \
     &c->rmin1, &c->plan[0], &c->plan[1], &c->plan[2], &c->keys, &c->perm_scratch, &c->tile_off, &c->chunk_tot, \
     &c->total, &c->pm, &c->pd, &c->cmp, &c->crid, &c->crid2, &c->posA, &c->posB, &c->posC, &c->segA, &c->segB,   \
     &c->segC, &c->runoff, &c->runpos, &c->runoff2, &c->runpos2, &c->tie, &c->keep, &c->done, &c->mlist,         \
     &c->wlist, &c->rcnt, &c->rtot, &c->part_in, &c->part_out, &c->anyt, &c->vbad, &c->keys2, &c->perm2,     \
     &c->ptab, &c->part_ptrs, &c->pdec, &c->psum0, &c->psum1, &c->phk, &c->phr, &c->rlist}

// checked build: the canary band after every scratch buffer must be intact after a call
// (synchronises); no-op otherwise
int check_guards(cks_ctx* ctx) {
#if CKS_CHECKED_BUILD
    CK(cudaStreamSynchronize(ctx->stream));
    static thread_local uint8_t host[kGuardBytes];
    DevBuf* bufs[] = CKS_SCRATCH_LIST(ctx);
    for (size_t i = 0; i < sizeof(bufs) / sizeof(bufs[0]); i++) {
        DevBuf* b = bufs[i];
        if (!b->p) continue;
        CK(cudaMemcpy(host, (uint8_t*)b->p + b->cap, kGuardBytes, cudaMemcpyDeviceToHost));
        for (size_t j = 0; j < kGuardBytes; j++)
            if (host[j] != (uint8_t)kCanary)
                return fail(ctx, CKS_ECUDA, "checked build: write past scratch buffer #%zu (cap %zu) at +%zu", i,
                            b->cap, j);
    }
#else
    (void)ctx;
#endif
    return CKS_OK;
}

uint32_t popcount_mask(const uint8_t* m, uint32_t B) {
    uint32_t c = 0;
    for (uint32_t j = 0; j < B; j++) c += (uint32_t)__builtin_popcount(m[j]);
    return c;
}

int check_keys(cks_ctx* ctx, const void* keys, uint64_t n, uint32_t B) {
    if (!ctx) return CKS_EINVAL;
    if (B < 1 || B > CKS_MAX_KEY_BYTES) return fail(ctx, CKS_EINVAL, "key_bytes %u not in [1,512]", B);
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n = %llu >= 2^32", (unsigned long long)n);
    if (n > 0 && !keys) return fail(ctx, CKS_EINVAL, "keys is NULL with n > 0");
    return CKS_OK;
}

void mark(cks_ctx* ctx, Stage s) {
    if (ctx->timing) cudaEventRecord(ctx->ev[s], ctx->stream);
}

// Upload a gather plan through pinned slot `slot` (waits for the slot's previous copy).
int upload_plan(cks_ctx* ctx, int slot, GatherPlan** dplan) {
    TRY(ensure(ctx, ctx->plan[slot], sizeof(GatherPlan)));
    size_t bytes = offsetof(GatherPlan, step) + sizeof(GatherStep) * ctx->h_plan[slot]->nsteps;
    CK(cudaMemcpyAsync(ctx->plan[slot].p, ctx->h_plan[slot], bytes, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->plan_ev[slot], ctx->stream));
    *dplan = as<GatherPlan>(ctx->plan[slot]);
    return CKS_OK;
}
int claim_slot(cks_ctx* ctx, int slot) {
    CK(cudaEventSynchronize(ctx->plan_ev[slot]));
    return CKS_OK;
}

// a1: superset mask into host `mask_out`; returns popcount via *m.
int run_superset(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, int kind,
                 uint8_t* mask_out, uint32_t* m, bool keys_ready = true, uint8_t* variant_out = nullptr) {
    if (kind != CKS_SUPERSET_VARIANT && kind != CKS_SUPERSET_BYTEOCC)
        return fail(ctx, CKS_EINVAL, "unknown superset kind %d", kind);
    TRY(ensure(ctx, ctx->occ, (size_t)B * 8 * 4));
    TRY(ensure(ctx, ctx->masks8, (size_t)B * 2));
    if (keys_ready) {
        CK(cudaMemsetAsync(ctx->occ.p, 0, (size_t)B * 8 * 4, ctx->stream));
        if (n) LAUNCH(launch_occupancy(keys, n, B, as<uint32_t>(ctx->occ), ctx->sms, ctx->stream));
        BYTES((double)n * B);
    }
    LAUNCH(launch_occ_finalize(as<uint32_t>(ctx->occ), B, n, as<uint8_t>(ctx->masks8),
                               as<uint8_t>(ctx->masks8) + B, ctx->stream));
    CK(cudaEventSynchronize(ctx->plan_ev[2]));
    CK(cudaMemcpyAsync(ctx->h_small, ctx->masks8.p, (size_t)B * 2, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const uint8_t* src = reinterpret_cast<const uint8_t*>(ctx->h_small) + (kind == CKS_SUPERSET_BYTEOCC ? 0 : B);
    memcpy(mask_out, src, B);
    if (variant_out) memcpy(variant_out, reinterpret_cast<const uint8_t*>(ctx->h_small) + B, B);
    *m = popcount_mask(mask_out, B);
    return CKS_OK;
}

inline uint64_t scratch_pitch(uint64_t n) { return (n + 31) & ~31ull; }

// a2 + a3
int run_compress(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* mask,
                 uint32_t* planes, uint64_t pitch, uint32_t lead = 0, const uint32_t* rows = nullptr,
                 uint32_t* occ = nullptr) {
    TRY(claim_slot(ctx, 0));
    plan_compress(mask, B, ctx->h_plan[0]);
    uint32_t m = ctx->h_plan[0]->out_bits, np = (m + 31) / 32;
    if (n == 0 || m == 0) return CKS_OK;
    GatherPlan* dplan;
    TRY(upload_plan(ctx, 0, &dplan));
    LAUNCH(launch_compress(keys, n, B, dplan, ctx->h_plan[0], np, planes, pitch, ctx->sms, ctx->stream, lead, rows,
                           occ));
    BYTES((double)n * (B + 4.0 * np + (rows ? 4.0 : 0.0)));
    return CKS_OK;
}

// a4 + a5. `in_planes` (np planes, stride in_pitch) is not modified. `in_rid` NULL = implicit
// ids; when non-NULL its rid_passes digits are sorted first. Sorted planes land in
// `final_planes` (stride final_pitch; NULL = ctx scratch), row ids in `final_rid`; the sorted
// planes' location is returned in *sorted_view / *sorted_pitch. Scratch plane buffers alternate
// so that the last pass writes the final buffers; the caller may have compressed into the
// scratch buffer the first pass does not write (see first_pass_out()).
uint32_t* first_pass_out(cks_ctx* ctx, uint32_t P) {
    return ((P - 1) & 1) ? as<uint32_t>(ctx->planeA) : as<uint32_t>(ctx->planeB);
}

// digit0: key digits below it are known to be constant (left-alignment padding, an absent
// plane) and are not sorted.
int run_sort(cks_ctx* ctx, const uint32_t* in_planes, uint64_t in_pitch, uint32_t np, uint32_t key_passes,
             uint64_t n, const uint32_t* in_rid, uint32_t rid_passes, uint32_t* final_planes,
             uint64_t final_pitch, uint32_t* final_rid, const uint32_t** sorted_view, uint64_t* sorted_pitch,
             uint32_t digit0 = 0, bool mark_stages = true) {
    if (digit0 > key_passes) digit0 = key_passes;
    const uint32_t Pfull = key_passes + (in_rid ? rid_passes : 0);
    const uint32_t P = Pfull - digit0;
    if (sorted_view) *sorted_view = in_planes;
    if (sorted_pitch) *sorted_pitch = in_pitch;
    if (n == 0) return CKS_OK;
    if (P == 0) {                                        // nothing to sort: identity order
        if (in_rid) CK(cudaMemcpyAsync(final_rid, in_rid, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        else LAUNCH(launch_iota(final_rid, n, ctx->stream));
        if (final_planes && np)
            CK(cudaMemcpy2DAsync(final_planes, final_pitch * 4, in_planes, in_pitch * 4, n * 4, np,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        return CKS_OK;
    }
    const uint64_t sp = scratch_pitch(n);
    const size_t pbytes = (size_t)np * sp * 4;
    TRY(ensure(ctx, ctx->planeA, pbytes));
    TRY(ensure(ctx, ctx->planeB, pbytes));
    TRY(ensure(ctx, ctx->ridA, sp * 4));
    TRY(ensure(ctx, ctx->ridB, sp * 4));
    uint64_t lsd_tiles = 0, lsd_chunks = 0;
    lsd_sizes(n, &lsd_tiles, &lsd_chunks);
    TRY(ensure(ctx, ctx->tile_off, (size_t)lsd_tiles * 256 * 4));
    TRY(ensure(ctx, ctx->chunk_tot, (size_t)lsd_chunks * 256 * 4));
    TRY(ensure(ctx, ctx->total, 256 * 4, /*zero=*/true));        // then kept zero by every downsweep
    if (mark_stages) mark(ctx, ST_HIST);

    const uint32_t* cur_p = in_planes;
    uint64_t cur_pitch = in_pitch;
    const uint32_t* cur_r = in_rid;
    for (uint32_t t = 0; t < P; t++) {
        const bool last = t == P - 1;
        const bool odd = ((P - 1 - t) & 1) != 0;
        uint32_t* out_p = odd ? as<uint32_t>(ctx->planeA) : (last && final_planes ? final_planes : as<uint32_t>(ctx->planeB));
        uint64_t out_pitch = (last && final_planes && !odd) ? final_pitch : sp;
        uint32_t* out_r = last ? final_rid : (odd ? as<uint32_t>(ctx->ridA) : as<uint32_t>(ctx->ridB));
        LsdPassArgs la;
        memset(&la, 0, sizeof(la));
        la.in_planes = cur_p;
        la.out_planes = out_p;
        la.in_rid = cur_r;
        la.out_rid = out_r;
        la.n = n;
        la.in_pitch = cur_pitch;
        la.out_pitch = out_pitch;
        la.nplanes = np;
        if (in_rid && t < rid_passes) {                  // row-id digits first (least significant)
            la.digit_plane = -1;
            la.shift = 8 * t;
        } else {
            const uint32_t p = (in_rid ? t - rid_passes : t) + digit0;
            la.digit_plane = (int32_t)(p >> 2);
            la.shift = 8 * (p & 3);
        }
        la.tile_off = as<uint32_t>(ctx->tile_off);
        la.chunk_tot = as<uint32_t>(ctx->chunk_tot);
        la.total = as<uint32_t>(ctx->total);
        LsdAux aux;
        aux.stream = ctx->aux_stream;
        aux.fork = ctx->aux_ev[0];
        aux.join = ctx->aux_ev[1];
        const int ke = ctx->nkev;
        if (ctx->timing && !knobs().no_kernel_events && ke < cks_ctx::kMaxKev) {
            aux.ws_begin = ctx->kev[2 * ke];
            aux.ws_end = ctx->kev[2 * ke + 1];
            ctx->kbytes[ke] = 0.0;
            aux.ws_bytes = &ctx->kbytes[ke];
        }
        int nl = 0;
        CK(launch_lsd_pass(la, ctx->sms, ctx->stream, aux, &nl));
        // upsweep reads the digit word; the downsweep reads every loaded stream and writes all
        BYTES(4.0 * n * (1 + (np + (cur_r ? 1 : 0)) + (np + 1)));
        if (aux.ws_bytes && ctx->kbytes[ke] > 0.0) ctx->nkev++;
        ctx->launches += (uint64_t)nl;
        cur_p = out_p;
        cur_pitch = out_pitch;
        cur_r = out_r;
    }
    if (sorted_view) *sorted_view = cur_p;
    if (sorted_pitch) *sorted_pitch = cur_pitch;
    return CKS_OK;
}

bool same_mask(const uint8_t* a, const uint8_t* b, uint32_t B) { return memcmp(a, b, B) == 0; }

constexpr uint32_t kSampleKeys = 4096;           // keys sorted to choose the round-0 width

// D-offset table of the sort mask: moff[t] = key position of the (t+1)-st mask bit.
int upload_moff(cks_ctx* ctx, const uint8_t* sort_mask, uint32_t B, uint32_t m) {
    TRY(ensure(ctx, ctx->moff, (size_t)(m + 1) * 2));
    CK(cudaEventSynchronize(ctx->plan_ev[1]));
    uint32_t t = 0;
    for (uint32_t p = 0; p < 8 * B; p++)
        if ((sort_mask[p >> 3] >> (7 - (p & 7))) & 1) ctx->h_moff[t++] = (uint16_t)p;
    if (t != m) return fail(ctx, CKS_EINVAL, "packed_bits %u != popcount(sort_mask) %u", m, t);
    if (m) CK(cudaMemcpyAsync(ctx->moff.p, ctx->h_moff, (size_t)m * 2, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->plan_ev[1], ctx->stream));
    return CKS_OK;
}

// D accumulated on the device (u32 words, key bit p = bit 31 - p%32 of word p/32) -> host mask
int read_dacc(cks_ctx* ctx, uint32_t B, uint8_t* mask_out) {
    const uint32_t nwords = (8 * B + 31) / 32;
    CK(cudaEventSynchronize(ctx->plan_ev[2]));
    CK(cudaMemcpyAsync(ctx->h_small, ctx->dacc.p, (size_t)nwords * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (uint32_t j = 0; j < B; j++) mask_out[j] = (uint8_t)(ctx->h_small[j >> 2] >> (24 - 8 * (j & 3)));
    return CKS_OK;
}

// a6: exact D from sorted planes compressed with `sort_mask` (host).
int run_adjacent(cks_ctx* ctx, const uint32_t* sorted, uint64_t pitch, uint32_t m, uint64_t n,
                 const uint8_t* sort_mask, uint32_t B, uint8_t* mask_out, uint16_t* dbit) {
    const uint32_t nwords = (8 * B + 31) / 32;
    TRY(ensure(ctx, ctx->dacc, (size_t)nwords * 4));
    TRY(upload_moff(ctx, sort_mask, B, m));
    CK(cudaMemsetAsync(ctx->dacc.p, 0, (size_t)nwords * 4, ctx->stream));
    if (n && m) {
        BYTES((double)n * (4.0 * ((m + 31) / 32) + (dbit ? 2.0 : 0.0)));
        LAUNCH(launch_adjacent(sorted, pitch, n, m, as<uint16_t>(ctx->moff), B, dbit, as<uint32_t>(ctx->dacc),
                               ctx->sms, ctx->stream));
    } else if (n && dbit) {
        LAUNCH(launch_fill_u16(dbit, n, (uint16_t)CKS_DBIT_NONE, ctx->stream));
    }
    return read_dacc(ctx, B, mask_out);
}

// Sub-mask of P_M bits that are exact-D positions, for the repack (a7). P_M bit of the
// compressed index t (0 = first mask position) is m - 1 - t + lead.
static void repack_words(const uint8_t* M, const uint8_t* D, uint32_t B, uint32_t m, uint32_t lead,
                         std::vector<uint32_t>& sub) {
    uint32_t t = 0;
    for (uint32_t p = 0; p < 8 * B; p++) {
        if (!((M[p >> 3] >> (7 - (p & 7))) & 1)) continue;
        const uint32_t b = m - 1 - t + lead;
        if ((D[p >> 3] >> (7 - (p & 7))) & 1) sub[b >> 5] |= 1u << (b & 31);
        t++;
    }
}

// NEXT-1: first build by distinguishing prefixes (k_refine.cu). Outputs perm, dbit, the
// exact D (out->mask) and P_D in sorted order (out->packed).
// keys == NULL: P_M is given instead (planes_in, right-aligned u32[np][n] as cks_compress).
// E != NULL (P_M of three planes, keys given): the partial-key bits E (C(a) of P:492) are
// compressed into one more plane appended below P_M and ride through the sort with it.
int build_refine(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* M, uint32_t m,
                 cks_build_out* out, uint16_t* dbit, const uint32_t* planes_in = nullptr, const uint8_t* E = nullptr) {
    const uint32_t npm = (m + 31) / 32, lead = 32 * npm - m;
    const uint32_t npe = (E && keys && !planes_in && npm == 3) ? 1u : 0u;   // appended planes (P_E)
    const uint32_t np = npm + npe;                               // planes sorted / carried
    ctx->pt_npe = npe;
    const uint64_t sp = scratch_pitch(n);
    const uint32_t nwords = (8 * B + 31) / 32;
    // a3: P_M left-aligned (the first mask position is bit 31 of the top plane), so chunk r
    // is planes np-1-2r (high word) and np-2-2r (low word)
    // given P_M that is already left-aligned with the scratch pitch (m a multiple of 32, n of 32;
    // e.g. the sharded path's received planes): sorted from where it is, read only
    const bool pm_given = planes_in && lead == 0 && sp == n && ((uintptr_t)planes_in & 15) == 0;
    uint32_t* pm = pm_given ? const_cast<uint32_t*>(planes_in) : nullptr;
    if (!pm_given) {
        TRY(ensure(ctx, ctx->pm, (size_t)np * sp * 4));
        pm = as<uint32_t>(ctx->pm);
    }
    // a2 + a3, and the width T of round 0: 8 bits more than the narrowest multiple of 8 bits
    // that separates a strided sample of the keys as well as the full 64-bit chunk does (fewer
    // round-0 passes; whatever still ties is finished by the later rounds -- the result is
    // exact for any T).
    // The sample is compressed and sorted on the side stream while the full compress runs.
    // cks_ctx_set_round0_bits forces T.
    GatherPlan* dplan = nullptr;
    if (!planes_in) {
        TRY(claim_slot(ctx, 0));
        plan_compress(M, B, ctx->h_plan[0]);
        TRY(upload_plan(ctx, 0, &dplan));
    }
    const int forced = (int)ctx->round0_bits;
    const bool sample = !(forced > 0 && forced <= 64 && (forced & 7) == 0) && npm >= 2 && n >= (1u << 16);
    TRY(ensure(ctx, ctx->rtot, 64));
    uint32_t* scnt = as<uint32_t>(ctx->rtot) + 4;
    if (planes_in) {                                             // given P_M: left-align it, then sample
        if (!pm_given) LAUNCH(launch_align_left(planes_in, n, np, n, lead, pm, sp, ctx->sms, ctx->stream));
        if (sample) {
            CK(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
            CK(cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_ev[0], 0));
            LAUNCH(launch_prefix_sample(nullptr, n, B, nullptr, kSampleKeys, scnt, ctx->aux_stream, pm, np, sp));
            CK(cudaMemcpyAsync(ctx->h_tot + 8, scnt, 32, cudaMemcpyDeviceToHost, ctx->aux_stream));
            CK(cudaEventRecord(ctx->aux_ev[1], ctx->aux_stream));
        }
    } else {
        if (sample) {
            CK(cudaEventRecord(ctx->aux_ev[0], ctx->stream));
            CK(cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_ev[0], 0));
            LAUNCH(launch_prefix_sample(keys, n, B, dplan, kSampleKeys, scnt, ctx->aux_stream));
            CK(cudaMemcpyAsync(ctx->h_tot + 8, scnt, 32, cudaMemcpyDeviceToHost, ctx->aux_stream));
            CK(cudaEventRecord(ctx->aux_ev[1], ctx->aux_stream));
        }
        LAUNCH(launch_compress(keys, n, B, dplan, ctx->h_plan[0], npm, pm + (uint64_t)npe * sp, sp, ctx->sms,
                               ctx->stream, lead, nullptr, ctx->spec_occ));
        if (ctx->spec_occ) TRY(spec_enqueue(ctx, n, B));
        if (npe) {                                               // P_E, left-aligned in plane 0
            TRY(claim_slot(ctx, 2));
            plan_compress(E, B, ctx->h_plan[2]);
            GatherPlan* eplan;
            TRY(upload_plan(ctx, 2, &eplan));
            const uint32_t me = ctx->h_plan[2]->out_bits;
            LAUNCH(launch_compress(keys, n, B, eplan, ctx->h_plan[2], 1, pm, sp, ctx->sms, ctx->stream, 32 - me));
            BYTES((double)n * (B + 4.0));
        }
    }
    mark(ctx, ST_COMPRESS);
    uint32_t T = forced > 0 && forced <= 64 && (forced & 7) == 0 ? (uint32_t)forced : 64;
    if (sample) {
        CK(cudaEventSynchronize(ctx->aux_ev[1]));
        // one byte of margin when P_M is read back by row id: a 4096-key sample misses the birthday
        // collisions that tie millions of keys at the narrowest separating width, and finishing
        // those by row is dearer than a pass (measured: cfg3 32 -> 40). With P_M carried (np == 3)
        // the tile kernel finishes short ties from the sorted planes for less than a pass costs
        // (measured, cfg5: T = 40 3.65 ms, 48 3.89 ms)
        const uint32_t margin = npm == 3 ? 0u : 1u;
        for (uint32_t w = 0; w < 8; w++)
            if (ctx->h_tot[8 + w] == ctx->h_tot[15]) {
                T = 8 * (w + 1 + margin) < 64 ? 8 * (w + 1 + margin) : 64;
                break;
            }
        CK(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));   // (scnt is reused below)
    }
    if (T > m) T = (m + 7) & ~7u;
    mark(ctx, ST_HIST);
    TRY(upload_moff(ctx, M, B, m));
    TRY(ensure(ctx, ctx->dacc, (size_t)nwords * 4));
    CK(cudaMemsetAsync(ctx->dacc.p, 0, (size_t)nwords * 4, ctx->stream));
    TRY(ensure(ctx, ctx->tie, n + 16));
    const uint16_t* moff = as<uint16_t>(ctx->moff);
    uint32_t* dacc = as<uint32_t>(ctx->dacc);
    uint8_t* tie = as<uint8_t>(ctx->tie);

    // round 0: every key by chunk 0. With three planes the third is carried through the
    // round-0 passes (4 more bytes per key per pass), which is cheaper than gathering the key
    // rows again at the end: P_M then comes out in sorted order (and stays so: the rounds
    // that reorder runs move its planes too).
    const bool carry = npm == 3;
    const uint32_t np0 = carry ? np : (np >= 2 ? 2 : 1);
    // round 0 sorts the top T bits of chunk 0 (the digits below them are skipped)
    const uint32_t dig0 = np <= 2 ? (lead / 8 > 4 * np0 - T / 8 ? lead / 8 : 4 * np0 - T / 8) : 4 * np0 - T / 8;
    const uint32_t* sorted0 = nullptr;
    uint64_t sp0 = sp;
    uint32_t* carried = nullptr;
    if (carry) {
        TRY(ensure(ctx, ctx->pd, (size_t)np * sp * 4));
        carried = as<uint32_t>(ctx->pd);
    }
    TRY(run_sort(ctx, pm + (uint64_t)(np - np0) * sp, sp, np0, 4 * np0, n, nullptr, 0, carried, sp, out->perm,
                 &sorted0, &sp0, dig0, false));
    if (carry) {                                                 // sorted P_M (+ P_E below) stays here
        ctx->spm = sorted0;
        ctx->spm_pitch = sp0;
        ctx->spm_np = np;
        ctx->spm_g0 = 0;
    }
    // round-0 adjacency; when rounds follow, fused with finishing the short runs inside a tile
    const bool no_tile = knobs().no_tile_runs;   // (experiments build only)
    const uint32_t* lo0 = np0 >= 2 ? sorted0 + (uint64_t)(np0 - 2) * sp0 : nullptr;
    const uint32_t* hi0 = sorted0 + (uint64_t)(np0 - 1) * sp0;
    TRY(ensure(ctx, ctx->rtot, 64));
    CK(cudaMemsetAsync(as<uint32_t>(ctx->rtot) + 2, 0, 4, ctx->stream));
    const bool tiled = T < m && carry && !no_tile && (int)np - (int)(T >> 5) <= 3;   // (P_M by row id: the compaction + k_ref_local path measured faster)
    if (tiled) {
        TRY(ensure(ctx, ctx->anyt, ref_tiles(n) + 16));
        CK(cudaMemsetAsync(ctx->anyt.p, 0, ref_tiles(n) + 16, ctx->stream));
        // reads the chunk (hi, lo), row ids and the carried words below the chunk; writes tie
        // flags and D_i (the reordered members' row ids and words are counted after the round)
        // (np == 3: chunk = planes 2, 1; the remaining words below the chunk add plane 0)
        BYTES((double)n * (8.0 + 4.0 + 4.0 + 3.0));
        LAUNCH(launch_ref_tile(pm, sp, np, (int)np - 1 - (int)(T >> 5), 0xFFFFFFFFu >> (T & 31), moff, out->perm, dbit,
                               carried, lo0, hi0, sp0, n, ~0ull << (64 - T), B, tie, dacc, as<uint32_t>(ctx->rtot) + 2,
                               ctx->sms, ctx->stream, as<uint8_t>(ctx->anyt)));
    } else {
        LAUNCH(launch_ref_adj(lo0, hi0, nullptr, nullptr, n, 0, moff, m, B, dbit, tie, dacc, true, ctx->sms,
                              ctx->stream, ~0ull << (64 - T)));
        BYTES((double)n * (4.0 * (np0 >= 2 ? 2 : 1) + 3.0));
    }
    out->round0_bits = T;
    out->rounds = 1;
    out->refined_keys = 0;
    out->passes = 4 * np0 - dig0;
    // rounds 1..: the tied runs. Short runs (and runs of equal keys) are finished in place by
    // comparing their remaining bits; the others are re-sorted by (run, chunk r).
    uint64_t nr = n;
    const uint32_t* pos = nullptr;                               // list of round r-1 (null: all keys)
    if (T < m) {
        DevBuf* pb[3] = {&ctx->posA, &ctx->posB, &ctx->posC};
        DevBuf* sb[3] = {&ctx->segA, &ctx->segB, &ctx->segC};
        for (int i = 0; i < 3; i++) {
            TRY(ensure(ctx, *pb[i], sp * 4));
            TRY(ensure(ctx, *sb[i], sp * 4));
        }
        TRY(ensure(ctx, ctx->runoff, sp * 4));
        TRY(ensure(ctx, ctx->runpos, sp * 4));
        TRY(ensure(ctx, ctx->runoff2, sp * 4));
        TRY(ensure(ctx, ctx->runpos2, sp * 4));
        TRY(ensure(ctx, ctx->keep, n + 16));
        TRY(ensure(ctx, ctx->done, n + 16));
        TRY(ensure(ctx, ctx->mlist, sp * 4));
        TRY(ensure(ctx, ctx->wlist, sp * 4));
        TRY(ensure(ctx, ctx->rcnt, (size_t)(ref_tiles(n) + 1) * 8));
        TRY(ensure(ctx, ctx->rtot, 64));
    }
    auto counts = [&](uint64_t* a, uint64_t* b) -> int {
        CK(cudaMemcpyAsync(ctx->h_tot, ctx->rtot.p, 12, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        *a = ctx->h_tot[0];
        *b = ctx->h_tot[1];
        if (ctx->h_tot[2]) {                                     // keys finished by the tile kernel
            out->refined_keys += ctx->h_tot[2];
            BYTES((double)ctx->h_tot[2] * (4.0 + 4.0 * (double)((int)np - (int)(T >> 5))));   // row ids + words
            CK(cudaMemsetAsync(as<uint32_t>(ctx->rtot) + 2, 0, 4, ctx->stream));
        }
        return CKS_OK;
    };
    const bool log = knobs().refine_log;          // (experiments build only)
    // a7 from the round-0 planes (below): they stay sorted except at round 1's tied positions,
    // which are saved here (when few) and refreshed at the end; an LSD round reuses their buffers
    bool lsd_refine = false, list1_ok = true;
    uint64_t nlist1 = 0;
    int li = -1;                                                 // buffer of the current list
    for (uint32_t r = 1; T + 64 * (r - 1) < m; r++) {
        const uint32_t o = T + 64 * (r - 1);                     // first P_M bit of this round's chunk
        const int ai = li == 0 ? 1 : 0;                          // (1)'s output
        const int bi = li < 0 ? 1 : 3 - li - ai;                 // (3)'s output, the next list
        uint32_t* posA_ = as<uint32_t>(ai == 0 ? ctx->posA : ai == 1 ? ctx->posB : ctx->posC);
        uint32_t* segA_ = as<uint32_t>(ai == 0 ? ctx->segA : ai == 1 ? ctx->segB : ctx->segC);
        uint32_t* posB_ = as<uint32_t>(bi == 0 ? ctx->posA : bi == 1 ? ctx->posB : ctx->posC);
        uint32_t* segB_ = as<uint32_t>(bi == 0 ? ctx->segA : bi == 1 ? ctx->segB : ctx->segC);
        // (1) the tied runs of the current list
        LAUNCH(launch_ref_compact(tie, nr, pos, as<uint32_t>(ctx->rcnt), as<uint32_t>(ctx->rtot), posA_, segA_,
                                  as<uint32_t>(ctx->runoff), as<uint32_t>(ctx->runpos), ctx->stream,
                                  r == 1 && tiled ? as<uint8_t>(ctx->anyt) : nullptr));
        uint64_t nn = 0, nseg = 0;
        TRY(counts(&nn, &nseg));
        BYTES((double)nr * (1.0 + (pos ? 4.0 : 0.0)) + (double)nn * 8.0 + (double)nseg * 8.0);
        if (nn == 0) break;
        if (r == 1 && !carry && keys) {
            list1_ok = nn <= n / 4;
            if (list1_ok) {
                TRY(ensure(ctx, ctx->rlist, nn * 4));
                CK(cudaMemcpyAsync(ctx->rlist.p, posA_, nn * 4, cudaMemcpyDeviceToDevice, ctx->stream));
                BYTES((double)nn * 8.0);
                nlist1 = nn;
            }
        }
        // (2) finish short runs and runs of equal keys in place
        const int qtop = (int)np - 1 - (int)(o >> 5);            // plane holding bit o
        LAUNCH(launch_ref_local(pm, sp, np, qtop, moff, as<uint32_t>(ctx->runpos), segA_, as<uint32_t>(ctx->runoff),
                                nseg, nn, out->perm,
                                dbit, dacc, as<uint8_t>(ctx->done), as<uint8_t>(ctx->keep), carried, B,
                                as<uint32_t>(ctx->mlist), as<uint32_t>(ctx->wlist), as<uint32_t>(ctx->rtot) + 12,
                                ctx->sms, ctx->stream, 0xFFFFFFFFu >> (o & 31)));
        BYTES((double)nseg * 8.0 + (double)nn * (4.0 + 4.0 * (double)(qtop + 1) + 2.0 + 1.0));
        // (3) the runs left for a round on the next 64 bits (none: done)
        CK(cudaMemcpyAsync(ctx->h_tot, as<uint32_t>(ctx->rtot) + 12, 16, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        const uint32_t maxlong = ctx->h_tot[3];
        uint64_t n2 = 0, nseg2 = 0;
        if (ctx->h_tot[1] > 0) {
            LAUNCH(launch_ref_keep(segA_, as<uint32_t>(ctx->runoff), as<uint8_t>(ctx->done), nn, as<uint8_t>(ctx->keep),
                                   ctx->sms, ctx->stream));
            LAUNCH(launch_ref_compact(as<uint8_t>(ctx->keep), nn, posA_, as<uint32_t>(ctx->rcnt),
                                      as<uint32_t>(ctx->rtot), posB_, segB_, as<uint32_t>(ctx->runoff2),
                                      as<uint32_t>(ctx->runpos2), ctx->stream));
            TRY(counts(&n2, &nseg2));
            BYTES((double)nn * 2.0 + (double)n2 * 8.0 + (double)nseg2 * 8.0);
        }
        if (log)
            fprintf(stderr, "[cks refine] round %u: %llu tied keys in %llu runs; %llu keys in %llu runs (longest %u) "
                    "left for the next chunk\n", r, (unsigned long long)nn, (unsigned long long)nseg,
                    (unsigned long long)n2, (unsigned long long)nseg2, maxlong);
        out->refined_keys += nn;
        if (n2 == 0) break;
        out->rounds = r + 1;
        // (4) the left runs by (run, 64-bit chunk at o): one CTA per run when every run fits,
        // else an LSD round over the compact list
        const uint64_t cp = scratch_pitch(n2);
        TRY(ensure(ctx, ctx->cmp, (size_t)3 * cp * 4));
        TRY(ensure(ctx, ctx->crid, cp * 4));
        TRY(ensure(ctx, ctx->crid2, cp * 4));
        const uint32_t* sv = nullptr;
        uint64_t svp = cp;
        if (maxlong <= kChunkCtaKeys) {
            LAUNCH(launch_ref_cta_chunk(pm, sp, np, o, out->perm, as<uint32_t>(ctx->runoff2), as<uint32_t>(ctx->runpos2),
                                        nseg2, n2, as<uint32_t>(ctx->cmp), cp, as<uint32_t>(ctx->crid2), ctx->sms,
                                        ctx->stream));
            sv = as<uint32_t>(ctx->cmp);
            BYTES((double)nseg2 * 8.0 + (double)n2 * (4.0 + 8.0 + 12.0 + 4.0));   // row, chunk by row -> chunk, row
        } else {
            lsd_refine = true;
            LAUNCH(launch_ref_gather(pm, sp, np, o, posB_, segB_, out->perm, n2, as<uint32_t>(ctx->cmp), cp,
                                     as<uint32_t>(ctx->crid), ctx->sms, ctx->stream));
            BYTES((double)n2 * (8.0 + 4.0 + 8.0 + 12.0 + 4.0));  // pos, seg, row, chunk by row -> list
            const uint32_t segbits = nseg2 > 1 ? 32u - (uint32_t)__builtin_clz((uint32_t)(nseg2 - 1)) : 0u;
            const uint32_t d0 = o + 64 > m ? (o + 64 - m) / 8 : 0;   // digits past the last mask bit are zero
            out->passes += 8 + (segbits + 7) / 8 - d0;
            TRY(run_sort(ctx, as<uint32_t>(ctx->cmp), cp, 3, 8 + (segbits + 7) / 8, n2, as<uint32_t>(ctx->crid), 0,
                         nullptr, 0, as<uint32_t>(ctx->crid2), &sv, &svp, d0, false));
        }
        LAUNCH(launch_ref_put(out->perm, posB_, as<uint32_t>(ctx->crid2), n2, pm, sp, np, carried, ctx->sms,
                              ctx->stream));
        BYTES((double)n2 * (8.0 + 4.0 + (carried ? 8.0 * np : 0.0)) + (double)n2 * (12.0 + 4.0 + 3.0));  // put + adj
        LAUNCH(launch_ref_adj(sv, sv + svp, sv + 2 * svp, posB_, n2, o, moff, m, B, dbit, tie, dacc, false, ctx->sms,
                              ctx->stream));
        pos = posB_;
        nr = n2;
        li = bi;
    }
    mark(ctx, ST_SORT);
    TRY(read_dacc(ctx, B, out->mask));
    out->popcount = popcount_mask(out->mask, B);
    mark(ctx, ST_ADJ);
    // a7: P_D in sorted order -- from the sorted chunk when one chunk held all of P_M,
    // otherwise compressed again from the key rows in sorted order
    const uint32_t npd = (out->popcount + 31) / 32;
    out->packed = nullptr;
    out->packed_pitch = sp;
    if (out->popcount > 0 && !ctx->skip_packed) {
        if (!carry) TRY(ensure(ctx, ctx->pd, (size_t)npd * sp * 4));
        uint32_t* pd = carry ? pm : as<uint32_t>(ctx->pd);       // (P_M in row order is no longer needed)
        if (carry && pm_given) {                                  // (the caller's planes are read only)
            TRY(ensure(ctx, ctx->pm, (size_t)np * sp * 4));
            pd = as<uint32_t>(ctx->pm);
        }
        const bool single = T >= m;                               // round 0 sorted all of P_M
        if ((single || carry) && lead == 0 && same_mask(out->mask, M, B)) {
            out->packed = sorted0 + (uint64_t)npe * sp0;           // (P_M's planes above the appended P_E)
            out->packed_pitch = sp0;
        } else if (single || carry) {
            std::vector<uint32_t> sub(np, 0);
            repack_words(M, out->mask, B, m, lead + 32 * npe, sub);
            TRY(claim_slot(ctx, 1));
            plan_repack(sub.data(), np, ctx->h_plan[1]);
            GatherPlan* dplan;
            TRY(upload_plan(ctx, 1, &dplan));
            LAUNCH(launch_repack(sorted0, sp0, n, dplan, ctx->h_plan[1]->nsteps, npd, pd, sp, ctx->sms, ctx->stream));
            BYTES((double)n * 4.0 * (np + npd));
            out->packed = pd;
        } else if (keys && !carry && !lsd_refine && list1_ok && np0 == 2 &&
                   [&] {                                          // every D bit in the round-0 planes
                       std::vector<uint32_t> sub(np, 0);
                       repack_words(M, out->mask, B, m, lead, sub);
                       for (uint32_t q = 0; q + np0 < np; q++)
                           if (sub[q]) return false;
                       return true;
                   }()) {
            // the round-0 sorted planes (top 64 bits of P_M) hold every D bit: refresh the
            // positions the refinement reordered from P_M by row, then repack -- no row gather
            uint32_t* s0 = const_cast<uint32_t*>(sorted0);
            if (nlist1) {
                LAUNCH(launch_ref_refresh(as<uint32_t>(ctx->rlist), nlist1, out->perm, pm, sp, np, np0, s0, sp0,
                                          ctx->sms, ctx->stream));
                BYTES((double)nlist1 * (4.0 + 4.0 + 8.0 * np0));
            }
            std::vector<uint32_t> sub(np, 0);
            repack_words(M, out->mask, B, m, lead, sub);
            TRY(claim_slot(ctx, 1));
            plan_repack(sub.data() + (np - np0), np0, ctx->h_plan[1]);
            GatherPlan* dplan;
            TRY(upload_plan(ctx, 1, &dplan));
            LAUNCH(launch_repack(s0, sp0, n, dplan, ctx->h_plan[1]->nsteps, npd, pd, sp, ctx->sms, ctx->stream));
            BYTES((double)n * 4.0 * (np0 + npd));
            out->packed = pd;
        } else if (keys) {
            TRY(run_compress(ctx, keys, n, B, out->mask, pd, sp, 0, out->perm));
            out->packed = pd;
        } else {                                                  // given P_M (row order): gather + repack
            std::vector<uint32_t> sub(np, 0);
            repack_words(M, out->mask, B, m, lead, sub);
            TRY(claim_slot(ctx, 1));
            plan_repack(sub.data(), np, ctx->h_plan[1]);
            GatherPlan* dplan;
            TRY(upload_plan(ctx, 1, &dplan));
            LAUNCH(launch_repack(pm, sp, n, dplan, ctx->h_plan[1]->nsteps, npd, pd, sp, ctx->sms, ctx->stream,
                                 out->perm));
            BYTES((double)n * 4.0 * (1 + np + npd));
            out->packed = pd;
        }
    }
    mark(ctx, ST_REPACK);
    return CKS_OK;
}

int tree_shape(uint64_t n, uint32_t fanout, double fill, cks_tree_shape* s) {
    if (!s || fanout < 2 || !(fill > 0.f) || fill > 1.f) return CKS_EINVAL;
    uint32_t per = (uint32_t)((double)fanout * (double)fill);
    if (per < 2) return CKS_EINVAL;
    memset(s, 0, sizeof(*s));
    s->n = n;
    s->fanout = fanout;
    s->per_node = per;
    uint64_t c = n, off = 0;
    uint32_t h = 0;
    while (c > 0) {
        c = (c + per - 1) / per;
        if (h >= CKS_MAX_LEVELS) return CKS_ERANGE;
        s->level_nodes[h] = c;
        s->level_offset[h] = off;
        off += c;
        h++;
        if (c <= 1) break;
    }
    s->height = h;
    s->total_nodes = off;
    if (off * (uint64_t)fanout >= (1ull << 32)) return CKS_ERANGE;   // kernels index slots in 32 bits
    s->inner_nodes = h ? off - s->level_nodes[0] : 0;
    return CKS_OK;
}

// a8
// first_global: the order's first entry is the global first (its levels' first entries get
// CKS_DBIT_NONE); otherwise (a later block) every inner entry takes its child's minimum.
// levels: build levels 0..levels-1 only (0 = all); top_min: minima of the top built level.
int run_bulkload(cks_ctx* ctx, const uint32_t* perm, const uint16_t* dbit, uint64_t n, uint32_t fanout,
                 double fill, const cks_tree* t, uint32_t* height, bool first_global = true, uint32_t levels = 0,
                 uint16_t* top_min = nullptr) {
    cks_tree_shape s;
    int rc = tree_shape(n, fanout, fill, &s);
    if (rc != CKS_OK) return fail(ctx, rc, "bad bulk-load shape (fanout %u, fill %f)", fanout, (double)fill);
    const uint32_t H = (levels == 0 || levels > s.height) ? s.height : levels;
    if (height) *height = H;
    if (n == 0) return CKS_OK;
    if (!t || !t->node_cnt || !t->entry_rid) return fail(ctx, CKS_EINVAL, "tree arrays are NULL");
    if (t->entry_dbit && !dbit) return fail(ctx, CKS_EINVAL, "entry_dbit requested without dbit");
    if (top_min && !dbit) return fail(ctx, CKS_EINVAL, "top_min requested without dbit");
    const uint32_t per = s.per_node;
    BulkLevel L{};
    L.entries = n;
    L.nodes = s.level_nodes[0];
    L.node_off = 0;
    L.span = 1;
    // per-node minima of D_k (rmin) ping-pong between two scratch buffers, level by level
    const bool mins = dbit && (H > 1 || top_min);
    if (mins) {
        TRY(ensure(ctx, ctx->rmin0, (size_t)s.level_nodes[0] * 2 + 16));
        TRY(ensure(ctx, ctx->rmin1, (size_t)s.level_nodes[0] * 2 + 16));
    }
    BYTES((double)n * (8.0 + (dbit ? 2.0 + (t->entry_dbit ? 2.0 : 0.0) : 0.0)) + (double)s.level_nodes[0] * 4.0);
    LAUNCH(launch_bulk_leaves(perm, dbit, L, fanout, per, t->node_cnt, t->entry_rid, t->entry_dbit,
                              mins ? as<uint16_t>(ctx->rmin0) : nullptr, ctx->sms, ctx->stream));
    const uint16_t* rbelow = mins ? as<uint16_t>(ctx->rmin0) : nullptr;
    uint64_t span = per;
    for (uint32_t l = 1; l < H; l++) {
        BulkLevel I{};
        I.entries = s.level_nodes[l - 1];
        I.nodes = s.level_nodes[l];
        I.node_off = s.level_offset[l];
        I.below_off = s.level_offset[l - 1];
        I.span = span;
        uint16_t* rout = mins ? ((l & 1) ? as<uint16_t>(ctx->rmin1) : as<uint16_t>(ctx->rmin0)) : nullptr;
        LAUNCH(launch_bulk_inner(perm, rbelow, I, n, fanout, per, t->node_cnt, t->entry_rid, t->entry_dbit,
                                 t->entry_child, s.level_offset[1], rout, ctx->sms, ctx->stream, first_global));
        rbelow = rout;
        span *= per;
    }
    if (top_min)
        CK(cudaMemcpyAsync(top_min, rbelow, (size_t)s.level_nodes[H - 1] * 2, cudaMemcpyDeviceToDevice, ctx->stream));
    return CKS_OK;
}

// P:502 merge: the levels above nchild child nodes (highest row id + minimum D_k of each);
// node ids start at 0 on the first built level.
int run_bulkload_top(cks_ctx* ctx, const uint32_t* child_rid, const uint16_t* child_min, uint64_t nchild,
                     uint32_t fanout, double fill, const cks_tree* t, uint32_t* height) {
    cks_tree_shape s;
    int rc = tree_shape(nchild, fanout, fill, &s);
    if (rc != CKS_OK) return fail(ctx, rc, "bad bulk-load shape (fanout %u, fill %f)", fanout, (double)fill);
    const uint32_t H = nchild > 1 ? s.height : 0;                 // levels over the children (one child: none)
    if (height) *height = H;
    if (nchild == 0) return CKS_OK;
    if (!t || !t->node_cnt || !t->entry_rid) return fail(ctx, CKS_EINVAL, "tree arrays are NULL");
    const uint32_t per = s.per_node;
    TRY(ensure(ctx, ctx->rmin0, (size_t)nchild * 2 + 16));
    TRY(ensure(ctx, ctx->rmin1, (size_t)nchild * 2 + 16));
    const uint16_t* rbelow = child_min;
    uint64_t span = 1, entries = nchild, below_off = 0, off = 0;
    for (uint32_t l = 0; l < H; l++) {
        BulkLevel I{};
        I.entries = entries;
        I.nodes = (entries + per - 1) / per;
        I.node_off = off;
        I.below_off = below_off;
        I.span = span;
        uint16_t* rout = (l & 1) ? as<uint16_t>(ctx->rmin1) : as<uint16_t>(ctx->rmin0);
        LAUNCH(launch_bulk_inner(child_rid, rbelow, I, nchild, fanout, per, t->node_cnt, t->entry_rid, t->entry_dbit,
                                 t->entry_child, 0, rout, ctx->sms, ctx->stream, true));
        rbelow = rout;
        below_off = I.node_off;
        off += I.nodes;
        entries = I.nodes;
        span *= per;
    }
    return CKS_OK;
}

// The order check (k_verify.cu) of the permutation just computed, when this build asks for it
// (ctx->verify_now): CKS_ERANGE if the sort mask was not a superset of the distinction bits.
int verify_if(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const cks_build_out* out) {
    if (!ctx->verify_now || !keys || n < 2) return CKS_OK;
    if (!ctx->proof_mask.empty() && ctx->spec_pending) {
        // rebuild: the D+ test on the occupancy the compress marked (finalised long ago)
        CK(cudaEventSynchronize(ctx->spec_ev));
        const uint8_t* dp = reinterpret_cast<const uint8_t*>(ctx->h_small) + kSpecHostOff;
        bool proven = true;
        for (uint32_t j = 0; j < B; j++) proven = proven && (dp[j] & ~ctx->proof_mask[j]) == 0;
        ctx->spec_pending = false;
        if (proven) return CKS_OK;
        ctx->unproven = ctx->proof_mask;
    }
    TRY(ensure(ctx, ctx->vbad, 16));
    LAUNCH(launch_verify_order(keys, B, out->perm, n, as<unsigned long long>(ctx->vbad), ctx->sms, ctx->stream));
    BYTES((double)n * (4.0 + B));
    CK(cudaEventSynchronize(ctx->plan_ev[2]));
    CK(cudaMemcpyAsync(ctx->h_small, ctx->vbad.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    unsigned long long bad;
    memcpy(&bad, ctx->h_small, 8);
    if (bad != ~0ull)
        return fail(ctx, CKS_ERANGE,
                    "the sort mask is not a superset of the distinction bits: sorted positions %llu and %llu are "
                    "out of (key, row id) order (Theorem 2 needs every D-bit in the mask, P:222-238)",
                    bad - 1, bad);
    return CKS_OK;
}

// Everything after the sort mask is known: a3 .. a8 on device keys.
// keys == NULL: P_M is given (planes_in, right-aligned u32[np][n]) -- cks_sort_prefix.
int build_from_mask(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* M,
                    uint32_t m, cks_build_out* out, const uint32_t* planes_in = nullptr) {
    const uint32_t np = (m + 31) / 32, k = (m + 7) / 8;
    out->sort_bits = m;
    out->passes = k;
    out->rounds = 0;
    out->refined_keys = 0;
    out->round0_bits = 0;
    uint16_t* dbit = out->dbit;
    if (!dbit && n) {
        TRY(ensure(ctx, ctx->dbit, n * 2));
        dbit = as<uint16_t>(ctx->dbit);
    }
    // 1 = auto: by prefixes whenever P_M is wider than one 64-bit chunk (m > 64); for m <= 64
    // round 0 would be the whole sort anyway
    if (n && m && (ctx->refine == 2 || (ctx->refine == 1 && m > 64))) {
        TRY(build_refine(ctx, keys, n, B, M, m, out, dbit, planes_in, ctx->pt_on ? ctx->pt_E.data() : nullptr));
        TRY(verify_if(ctx, keys, n, B, out));
        out->height = 0;
        if (out->tree.node_cnt) {
            cks_tree tr = out->tree;
            TRY(run_bulkload(ctx, out->perm, dbit, n, out->fanout, out->fill, &tr, &out->height));
        }
        mark(ctx, ST_BULK);
        return CKS_OK;
    }
    // a3: compress into whichever plane buffer the first LSD pass does not write
    const uint64_t sp = scratch_pitch(n);
    const size_t pbytes = (size_t)np * sp * 4;
    TRY(ensure(ctx, ctx->planeA, pbytes));
    TRY(ensure(ctx, ctx->planeB, pbytes));
    uint32_t* cbuf = k ? (first_pass_out(ctx, k) == as<uint32_t>(ctx->planeA) ? as<uint32_t>(ctx->planeB)
                                                                              : as<uint32_t>(ctx->planeA))
                       : as<uint32_t>(ctx->planeB);
    uint64_t cpitch = sp;
    if (planes_in) {                                              // given P_M: sort it in place of a compress
        cbuf = const_cast<uint32_t*>(planes_in);                  // (read only: the first pass writes elsewhere)
        cpitch = n;
    } else {
        TRY(run_compress(ctx, keys, n, B, M, cbuf, sp, 0, nullptr, ctx->spec_occ));
        if (ctx->spec_occ && n && m) TRY(spec_enqueue(ctx, n, B));
    }
    mark(ctx, ST_COMPRESS);
    // a4 + a5
    const uint32_t* sorted = nullptr;
    uint64_t spitch = sp;
    TRY(run_sort(ctx, cbuf, cpitch, np, k, n, nullptr, 0, nullptr, 0, out->perm, &sorted, &spitch));
    ctx->spm = sorted;                                           // right-aligned P_M in sorted order
    ctx->spm_pitch = spitch;
    ctx->spm_np = np;
    ctx->spm_g0 = 32 * np - m;
    mark(ctx, ST_SORT);
    // a6
    TRY(run_adjacent(ctx, sorted, spitch, m, n, M, B, out->mask, dbit));
    out->popcount = popcount_mask(out->mask, B);
    mark(ctx, ST_ADJ);
    // a7: repack P_M -> P_D
    out->packed = sorted;
    out->packed_pitch = spitch;
    if (!same_mask(out->mask, M, B) && out->popcount > 0 && !ctx->skip_packed) {
        std::vector<uint32_t> sub(np, 0);
        repack_words(M, out->mask, B, m, 0, sub);
        TRY(claim_slot(ctx, 1));
        plan_repack(sub.data(), np, ctx->h_plan[1]);
        GatherPlan* dplan;
        TRY(upload_plan(ctx, 1, &dplan));
        uint32_t* dst = (sorted == as<uint32_t>(ctx->planeA)) ? as<uint32_t>(ctx->planeB) : as<uint32_t>(ctx->planeA);
        BYTES((double)n * 4.0 * (np + (out->popcount + 31) / 32));
        LAUNCH(launch_repack(sorted, spitch, n, dplan, ctx->h_plan[1]->nsteps, (out->popcount + 31) / 32, dst, sp,
                             ctx->sms, ctx->stream));
        out->packed = dst;
        out->packed_pitch = sp;
    } else if (out->popcount == 0) {
        out->packed = nullptr;
    }
    mark(ctx, ST_REPACK);
    TRY(verify_if(ctx, keys, n, B, out));
    // a8
    out->height = 0;
    if (out->tree.node_cnt) {
        cks_tree tr = out->tree;
        TRY(run_bulkload(ctx, out->perm, dbit, n, out->fanout, out->fill, &tr, &out->height));
    }
    mark(ctx, ST_BULK);
    return CKS_OK;
}

// NEXT-3 tree with the paper's partial-key sources: segments X (mask X, first bit gx
// from the MSB of the np sorted planes) and Y (mask Y or NULL, first bit gy) give source A,
// `ref` source B (invariant = 0 in V), the key rows C(b) for the other variant positions.
int run_ptree_ds(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit,
                 const uint32_t* planes, uint64_t pitch, uint32_t np, const uint8_t* X, uint32_t gx, const uint8_t* Y,
                 uint32_t gy, const uint8_t* V, const uint8_t* ref, uint32_t pk, double fill, uint8_t* nodes) {
    bool need_rows = false;
    for (uint32_t j = 0; j < B; j++) need_rows |= (V[j] & ~X[j] & ~(Y ? Y[j] : 0)) != 0;
    if (n && (!perm || !dbit || !nodes || (need_rows && !keys)))
        return fail(ctx, CKS_EINVAL, "NULL perm, dbit, nodes, or keys (variant bits outside the planes)");
    cks_tree_shape s;
    const int rc = cks_paper_tree_shape(n, fill, &s);
    if (rc != CKS_OK) return fail(ctx, rc, "bad paper-tree shape (fill %f)", fill);
    if (n == 0) return CKS_OK;
    PtreeWs ws;
    TRY(ptree_ws(ctx, s.level_nodes[0], &ws));
    // per-window-start table (k_ptree.cu PkDs): for p0 = 0 .. 8B, the pk-bit window's X / Y /
    // invariant / row positions and the ranks of its first position in X and Y
    const uint32_t nb = 8 * B, nent = nb + 1;
    TRY(ensure(ctx, ctx->ptab, (size_t)nent * sizeof(PtreeEnt) + 16));
    if (!ctx->h_ptab) {
        CK(cudaMallocHost(&ctx->h_ptab, (size_t)(8 * CKS_MAX_KEY_BYTES + 1) * sizeof(PtreeEnt)));
        CK(cudaEventRecord(ctx->ptab_ev, ctx->stream));
    }
    CK(cudaEventSynchronize(ctx->ptab_ev));                     // the previous upload is done
    auto bit = [&](const uint8_t* m, uint32_t p) -> uint32_t {
        return (m && p < nb) ? (uint32_t)(m[p >> 3] >> (7 - (p & 7))) & 1u : 0u;
    };
    uint32_t rx = 0, ry = 0;
    for (uint32_t p0 = 0; p0 < nent; p0++) {
        PtreeEnt& e = ctx->h_ptab[p0];
        e = PtreeEnt{0, 0, 0, 0, rx, ry};
        for (uint32_t i = 0; i < pk && p0 + i < nb; i++) {
            const uint32_t p = p0 + i, b = 0x80000000u >> i;
            if (bit(X, p)) e.wx |= b;
            else if (bit(Y, p)) e.wy |= b;
            else if (bit(V, p)) e.wc |= b;
            else if (bit(ref, p)) e.refb |= b;
        }
        rx += bit(X, p0);
        ry += bit(Y, p0);
    }
    CK(cudaMemcpyAsync(ctx->ptab.p, ctx->h_ptab, (size_t)nent * sizeof(PtreeEnt), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->ptab_ev, ctx->stream));
    PtreeDs ds{planes, pitch, np, gx, gy, as<PtreeEnt>(ctx->ptab)};
    int nl = 0;
    CK(launch_ptree(keys, n, B, perm, dbit, pk, s.per_node, s.reserved, s.level_nodes, s.level_offset, s.height, nodes,
                    ws, ctx->sms, ctx->stream, &nl, &ds));
    ctx->launches += (uint64_t)nl;
    BYTES((double)n * (4.0 * np + 4.0 + 2.0) + (double)s.total_nodes * 256.0);
    return CKS_OK;
}

// The decode tree (k_ptree.cu PkDec): per byte j, the M-bit projection of every byte value
// occurring there (ctx->occ, from this build's superset pass) -> the value; M = D+ makes the
// projections distinct, so the sorted P_M alone gives every key bit.
int run_ptree_decode(cks_ctx* ctx, uint64_t n, uint32_t B, const uint8_t* M, const uint32_t* perm, const uint16_t* dbit,
                     uint32_t pk, double fill, uint8_t* nodes) {
    cks_tree_shape s;
    const int rc = cks_paper_tree_shape(n, fill, &s);
    if (rc != CKS_OK) return fail(ctx, rc, "bad paper-tree fill %f", fill);
    std::vector<uint32_t> occ((size_t)B * 8);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(occ.data(), ctx->occ.p, occ.size() * 4, cudaMemcpyDeviceToHost));
    // layout: pj uint4[B] (k_ptree.cu PkDec), then byte j's 2^c_j values at off[j], then one 0
    std::vector<uint32_t> rank(B + 5, 0), cnt(B + 5, 0), off(B + 5, 0);
    uint32_t r = 0, dec_bytes = 0;
    for (uint32_t j = 0; j < B; j++) {
        cnt[j] = (uint32_t)__builtin_popcount(M[j]);
        rank[j] = r;
        off[j] = dec_bytes;
        r += cnt[j];
        dec_bytes += 1u << cnt[j];
    }
    const uint32_t zero = dec_bytes++;                              // bytes past the key
    for (uint32_t j = B; j < B + 5; j++) off[j] = zero;
    if (dec_bytes > 65536u || ctx->spm_g0 + r > 4096u)
        return fail(ctx, CKS_EINVAL, "decode tables too large (%u bytes)", dec_bytes);
    const size_t tb = (size_t)B * 16 + dec_bytes;
    std::vector<uint8_t> h(tb, 0);
    uint32_t* pj = reinterpret_cast<uint32_t*>(h.data());
    for (uint32_t j = 0; j < B; j++) {
        uint32_t x = ctx->spm_g0 + rank[j];
        for (uint32_t i = 0; i < 5; i++) x |= cnt[j + i] << (12 + 4 * i);
        pj[4 * j + 0] = x;
        pj[4 * j + 1] = off[j] | off[j + 1] << 16;
        pj[4 * j + 2] = off[j + 2] | off[j + 3] << 16;
        pj[4 * j + 3] = off[j + 4];
    }
    uint8_t* dec = h.data() + (size_t)B * 16;
    for (uint32_t j = 0; j < B; j++) {
        const uint32_t mj = M[j];
        for (uint32_t v = 0; v < 256; v++) {
            if (!((occ[(size_t)j * 8 + (v >> 5)] >> (v & 31)) & 1u)) continue;
            uint32_t proj = 0;                                       // M bits of v, MSB first
            for (int b = 7; b >= 0; b--)
                if ((mj >> b) & 1u) proj = (proj << 1) | ((v >> b) & 1u);
            dec[off[j] + proj] = (uint8_t)v;
        }
    }
    TRY(ensure(ctx, ctx->pdec, tb + 16));
    CK(cudaMemcpy(ctx->pdec.p, h.data(), tb, cudaMemcpyHostToDevice));
    PtreeWs ws;
    TRY(ptree_ws(ctx, s.level_nodes[0], &ws));
    int nl = 0;
    CK(launch_ptree_decode(n, B, perm, dbit, pk, s.per_node, s.reserved, s.level_nodes, s.level_offset, s.height, nodes,
                           ws, ctx->sms, ctx->stream, &nl, ctx->spm, ctx->spm_pitch, ctx->spm_np,
                           as<uint4>(ctx->pdec), as<uint8_t>(ctx->pdec) + (size_t)B * 16, dec_bytes));
    ctx->launches += (uint64_t)nl;
    BYTES((double)n * (4.0 * ctx->spm_np + 4.0 + 2.0) + (double)s.total_nodes * 256.0);
    return CKS_OK;
}

int build_common(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* prior,
                 cks_build_out* out, bool keys_ready_for_mask) {
    std::vector<uint8_t> M(B, 0), V(B, 0);
    uint32_t m = 0;
    const bool ptree = out->ptree_nodes != nullptr && n > 0;
    const bool want_v = out->variant || ptree;
    // the speculative mask (first builds of large columns whose compress can mark occupancy;
    // V comes out of the same occupancy after the build -- not with the C(a) tree source, whose
    // carried plane needs V before the sort)
    ctx->proof_mask.clear();
    struct Reset {                                       // every exit: no marking request outlives the call
        cks_ctx* c;
        ~Reset() {
            c->spec_occ = nullptr;
            c->spec_pending = false;
            c->proof_mask.clear();
            c->verify_now = false;
        }
    } reset{ctx};
    const bool spec = !prior && keys && keys_ready_for_mask && knobs().spec_mask && ctx->spec_on &&
                      out->superset_kind == CKS_SUPERSET_BYTEOCC &&
                      !(ptree && out->ptree_source == CKS_PTREE_CARRY) &&
                      n >= kSpecMinKeys && B >= kSpecMinB && compress_marks_occupancy(keys, B);
    ctx->spec_occ = nullptr;
    bool proven = false;                                 // prior mask shown to contain D
    if (prior) {
        memcpy(M.data(), prior, B);
        m = popcount_mask(M.data(), B);
        // the order check of a prior mask (CKS_VERIFY_PRIOR): first the sufficient test D+ of
        // the new keys inside M (one sequential pass; D is inside D+, reading R2, so sorting by
        // M gives the full-key order, Theorem 2), skipped for a mask that failed it before
        const bool vprior = keys && n > 1 && ctx->verify == CKS_VERIFY_PRIOR;
        const bool try_proof = vprior && !(ctx->unproven.size() == B && memcmp(ctx->unproven.data(), prior, B) == 0);
        if (try_proof && !want_v && compress_marks_occupancy(keys, B)) {
            // the test rides on the compress: it marks the occupancy, the D+ is finalised behind
            // it, and the order check (verify_if, after the sort) first tests D+ inside M
            TRY(ensure(ctx, ctx->occ, (size_t)B * 8 * 4));
            TRY(ensure(ctx, ctx->masks8, (size_t)B * 2));
            CK(cudaMemsetAsync(ctx->occ.p, 0, (size_t)B * 8 * 4, ctx->stream));
            ctx->spec_occ = as<uint32_t>(ctx->occ);
            ctx->proof_mask.assign(prior, prior + B);
        } else if (want_v || try_proof) {
            // (rebuild: the new variant bitmap is the same pass, P:413 step 3)
            std::vector<uint8_t> Dp(B);
            uint32_t mp = 0;
            TRY(run_superset(ctx, keys, n, B, CKS_SUPERSET_BYTEOCC, Dp.data(), &mp, true, V.data()));
            if (vprior) {
                proven = true;
                for (uint32_t j = 0; j < B; j++) proven = proven && (Dp[j] & ~M[j]) == 0;
                if (!proven) ctx->unproven.assign(prior, prior + B);
            }
        }
    } else if (spec) {
        // speculative first build: M' = D+ of a strided row sample (a subset of the rows, so
        // M' is inside the keys' D+); the compress marks every key's bytes on the way, and the
        // full D+ is compared with M' after the build (below) -- the keys are read once for both
        TRY(ensure(ctx, ctx->occ_s, (size_t)B * 8 * 4));
        TRY(ensure(ctx, ctx->occ, (size_t)B * 8 * 4));
        TRY(ensure(ctx, ctx->masks8, (size_t)B * 2));
        CK(cudaMemsetAsync(ctx->occ_s.p, 0, (size_t)B * 8 * 4, ctx->stream));
        CK(cudaMemsetAsync(ctx->occ.p, 0, (size_t)B * 8 * 4, ctx->stream));
        LAUNCH(launch_occupancy_sample(keys, n, B, kSpecSamples, as<uint32_t>(ctx->occ_s), ctx->stream));
        BYTES((double)kSpecSamples * B);
        LAUNCH(launch_occ_finalize(as<uint32_t>(ctx->occ_s), B, n, as<uint8_t>(ctx->masks8),
                                   as<uint8_t>(ctx->masks8) + B, ctx->stream));
        CK(cudaEventSynchronize(ctx->plan_ev[2]));
        CK(cudaMemcpyAsync(ctx->h_small, ctx->masks8.p, B, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        memcpy(M.data(), ctx->h_small, B);
        m = popcount_mask(M.data(), B);
        ctx->spec_occ = as<uint32_t>(ctx->occ);
        ctx->spec_builds++;
    } else {
        int kind = out->superset_kind;
        TRY(run_superset(ctx, keys, n, B, kind, M.data(), &m, keys_ready_for_mask, V.data()));
    }
    if (out->variant && !spec) memcpy(out->variant, V.data(), B);
    if (out->ref_key) {                                  // the reference key (row 0's key)
        if (n) {
            CK(cudaEventSynchronize(ctx->plan_ev[2]));
            CK(cudaMemcpyAsync(ctx->h_small, keys, B, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            memcpy(out->ref_key, ctx->h_small, B);
        } else {
            memset(out->ref_key, 0, B);
        }
    }
    // NEXT-3 fused paper tree: DS-metadata V and the reference key, and the partial-key bits that
    // are variant but not in M (E, P:492 C(a)) -- appended to P_M when P_M is carried (3 planes)
    std::vector<uint8_t> ref(B, 0);
    ctx->pt_on = false;
    ctx->pt_npe = 0;
    ctx->spm = nullptr;
    if (ptree) {
        if (out->ptree_pk > 32) return fail(ctx, CKS_EINVAL, "ptree_pk %u > 32", out->ptree_pk);
        if (out->ptree_source > CKS_PTREE_DECODE)
            return fail(ctx, CKS_EINVAL, "unknown ptree_source %u", out->ptree_source);
        CK(cudaEventSynchronize(ctx->plan_ev[2]));
        CK(cudaMemcpyAsync(ctx->h_small, keys, B, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        memcpy(ref.data(), ctx->h_small, B);
        // E = variant positions outside M inside some window [q+1, q+pk] (q in M) or [0, pk)
        const uint32_t pk = out->ptree_pk, nb = 8 * B;
        std::vector<uint8_t> win(nb + 1, 0);
        int last = -1;                                           // last M position at or before p
        ctx->pt_E.assign(B, 0);
        uint32_t ne = 0;
        for (uint32_t p = 0; p < nb; p++) {
            const bool inM = (M[p >> 3] >> (7 - (p & 7))) & 1, inV = (V[p >> 3] >> (7 - (p & 7))) & 1;
            const bool inwin = p < pk || (last >= 0 && p <= (uint32_t)last + pk);
            if (inV && !inM && inwin) { ctx->pt_E[p >> 3] |= (uint8_t)(0x80u >> (p & 7)); ne++; }
            if (inM) last = (int)p;
        }
        ctx->pt_on = out->ptree_source == CKS_PTREE_CARRY && ne > 0 && ne <= 32;
    }
    mark(ctx, ST_MASK);
    ctx->verify_now =
        keys && (ctx->verify == CKS_VERIFY_ALWAYS || (ctx->verify == CKS_VERIFY_PRIOR && prior && !proven));
    ctx->spec_pending = false;
    int rc = build_from_mask(ctx, keys, n, B, M.data(), m, out);
    ctx->spec_occ = nullptr;
    ctx->proof_mask.clear();
    if (rc == CKS_OK && spec) {
        // the keys' D+ from the occupancy the compress marked: equal to M' -> the build stands
        // (M' holds D+ holds D: Theorem 2); else (the sample missed a byte value that adds a
        // D+ bit) build again by the full D+, no further pass over the keys for the mask
        std::vector<uint8_t> Mp(M);
        uint32_t mf = 0;
        if (ctx->spec_pending) {
            CK(cudaEventSynchronize(ctx->spec_ev));
            const uint8_t* h = reinterpret_cast<const uint8_t*>(ctx->h_small) + kSpecHostOff;
            memcpy(M.data(), h, B);
            memcpy(V.data(), h + B, B);
            mf = popcount_mask(M.data(), B);
        } else {                                                  // (nothing was compressed: m' = 0)
            TRY(run_superset(ctx, keys, n, B, CKS_SUPERSET_BYTEOCC, M.data(), &mf, true, V.data()));
        }
        ctx->spec_pending = false;
        if (out->variant) memcpy(out->variant, V.data(), B);
        if (mf != m || memcmp(M.data(), Mp.data(), B) != 0) {
            ctx->spec_retries++;
            m = mf;
            rc = build_from_mask(ctx, keys, n, B, M.data(), m, out);
        }
    }
    ctx->verify_now = false;
    ctx->pt_on = false;
    TRY(rc);
    if (out->sort_mask) memcpy(out->sort_mask, M.data(), B);
    if (ptree) {
        const uint16_t* db = out->dbit ? out->dbit : as<uint16_t>(ctx->dbit);
        // DECODE: every bit from the sorted P_{D+} (a first build's byte-occupancy mask)
        uint64_t dec_bytes = 1;                                   // the decode tables fit u16 offsets
        for (uint32_t j = 0; j < B; j++) dec_bytes += 1ull << __builtin_popcount(M[j]);
        // (the sort mask holds the keys' D+ -- a first build's D+ or V, or a prior mask the D+
        // test proved -- so its bits at byte j tell the byte values occurring there apart, and
        // ctx->occ is these keys' occupancy)
        const bool decodable = (!prior || proven) && ctx->spm && n && dec_bytes <= 65536u;
        uint32_t src = out->ptree_source;
        if (src == CKS_PTREE_AUTO) src = decodable ? CKS_PTREE_DECODE : CKS_PTREE_ROWS;
        if (src == CKS_PTREE_DECODE && !decodable)
            return fail(ctx, CKS_EINVAL, "ptree_source DECODE needs a sort mask holding the keys' D+ (a first build, or a proven prior mask) kept sorted");
        if (src == CKS_PTREE_DECODE) {
            TRY(run_ptree_decode(ctx, n, B, M.data(), out->perm, db, out->ptree_pk, out->ptree_fill, out->ptree_nodes));
        } else if (src == CKS_PTREE_ROWS) {                       // C(b) for every bit
            cks_tree_shape s;
            TRY(cks_paper_tree_shape(n, out->ptree_fill, &s) == CKS_OK ? CKS_OK
                    : fail(ctx, CKS_EINVAL, "bad paper-tree fill %f", out->ptree_fill));
            PtreeWs ws;
            TRY(ptree_ws(ctx, s.level_nodes[0], &ws));
            int nl = 0;
            CK(launch_ptree(keys, n, B, out->perm, db, out->ptree_pk, s.per_node, s.reserved, s.level_nodes,
                            s.level_offset, s.height, out->ptree_nodes, ws, ctx->sms, ctx->stream, &nl));
            ctx->launches += (uint64_t)nl;
        } else if (src == CKS_PTREE_CARRY && ctx->pt_npe) {                                       // A from the carried P_M | P_E, B, no rows
            const uint32_t npm = (m + 31) / 32;
            TRY(run_ptree_ds(ctx, keys, n, B, out->perm, db, as<uint32_t>(ctx->pd), scratch_pitch(n), npm + 1,
                             M.data(), 0, ctx->pt_E.data(), 32 * npm, V.data(), ref.data(), out->ptree_pk,
                             out->ptree_fill, out->ptree_nodes));
        } else {                                                 // A from P_D, B, C(b) from the rows
            const uint32_t npd = (out->popcount + 31) / 32;
            TRY(run_ptree_ds(ctx, keys, n, B, out->perm, db, out->packed, out->packed_pitch, npd, out->mask,
                             32 * npd - out->popcount, nullptr, 0, V.data(), ref.data(), out->ptree_pk,
                             out->ptree_fill, out->ptree_nodes));
        }
        mark(ctx, ST_BULK);
    }
    return check_guards(ctx);
}

}  // namespace

// ======================================================================================
extern "C" {

int cks_ctx_create(int device, void* stream, cks_ctx** out) {
    if (!out) return CKS_EINVAL;
    *out = nullptr;
    cks_ctx* ctx = new (std::nothrow) cks_ctx();
    if (!ctx) return CKS_ENOMEM;
    ctx->device = device;
    ctx->stream = (cudaStream_t)stream;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete ctx;
        return CKS_ECUDA;
    }
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    bool ok = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
    if (ok) ok = cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; i < 6 && ok; i++) ok = cudaEventCreateWithFlags(&ctx->bev[i], cudaEventDisableTiming) == cudaSuccess;
    if (ok) ok = cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; i < 2 && ok; i++) ok = cudaEventCreateWithFlags(&ctx->aux_ev[i], cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < 2 * cks_ctx::kMaxKev && ok; i++) ok = cudaEventCreate(&ctx->kev[i]) == cudaSuccess;
    for (int i = 0; i < ST_N && ok; i++) ok = cudaEventCreate(&ctx->ev[i]) == cudaSuccess;
    for (int i = 0; i < 3 && ok; i++) ok = cudaEventCreateWithFlags(&ctx->plan_ev[i], cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < 3 && ok; i++) ok = cudaMallocHost(&ctx->h_plan[i], sizeof(GatherPlan)) == cudaSuccess;
    if (ok) ok = cudaMallocHost(&ctx->h_moff, kMaxBits * 2) == cudaSuccess;
    if (ok) ok = cudaMallocHost(&ctx->h_small, 8192) == cudaSuccess;
    if (ok) ok = cudaMallocHost(&ctx->h_tot, 64) == cudaSuccess;
    if (ok) ok = cudaEventCreateWithFlags(&ctx->ptab_ev, cudaEventDisableTiming) == cudaSuccess;
    if (ok) ok = cudaEventCreateWithFlags(&ctx->spec_ev, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < 3 && ok; i++) ok = cudaEventRecord(ctx->plan_ev[i], ctx->stream) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        cks_ctx_destroy(ctx);
        return CKS_ECUDA;
    }
    *out = ctx;
    return CKS_OK;
}

int cks_ctx_destroy(cks_ctx* ctx) {
    if (!ctx) return CKS_EINVAL;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    DevBuf* bufs[] = CKS_SCRATCH_LIST(ctx);
    for (DevBuf* b : bufs)
        if (b->p) cudaFree(b->p);
    for (int i = 0; i < ST_N; i++)
        if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
    for (int i = 0; i < 3; i++)
        if (ctx->plan_ev[i]) cudaEventDestroy(ctx->plan_ev[i]);
    for (int i = 0; i < 3; i++)
        if (ctx->h_plan[i]) cudaFreeHost(ctx->h_plan[i]);
    if (ctx->h_moff) cudaFreeHost(ctx->h_moff);
    if (ctx->h_small) cudaFreeHost(ctx->h_small);
    if (ctx->h_tot) cudaFreeHost(ctx->h_tot);
    if (ctx->h_ptab) cudaFreeHost(ctx->h_ptab);
    if (ctx->ptab_ev) cudaEventDestroy(ctx->ptab_ev);
    if (ctx->spec_ev) cudaEventDestroy(ctx->spec_ev);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
    for (int i = 0; i < 6; i++)
        if (ctx->bev[i]) cudaEventDestroy(ctx->bev[i]);
    if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
    for (int i = 0; i < 2; i++)
        if (ctx->aux_ev[i]) cudaEventDestroy(ctx->aux_ev[i]);
    for (int i = 0; i < 2 * cks_ctx::kMaxKev; i++)
        if (ctx->kev[i]) cudaEventDestroy(ctx->kev[i]);
    delete ctx;
    return CKS_OK;
}

int cks_ctx_set_stream(cks_ctx* ctx, void* stream) {
    if (!ctx) return CKS_EINVAL;
    if ((cudaStream_t)stream != ctx->stream) {
        // keep the pinned staging guards valid on the new stream
        cudaStreamSynchronize(ctx->stream);
        ctx->stream = (cudaStream_t)stream;
        for (int i = 0; i < 3; i++) cudaEventRecord(ctx->plan_ev[i], ctx->stream);
    }
    return CKS_OK;
}

int cks_ctx_set_timing(cks_ctx* ctx, int enable) {
    if (!ctx) return CKS_EINVAL;
    ctx->timing = enable != 0;
    return CKS_OK;
}

int cks_ctx_set_sort_mode(cks_ctx* ctx, int mode) {
    if (!ctx || mode < CKS_SORT_SINGLE || mode > CKS_SORT_PREFIX) return CKS_EINVAL;
    ctx->refine = mode;
    return CKS_OK;
}

int cks_ctx_set_round0_bits(cks_ctx* ctx, uint32_t bits) {
    if (!ctx || bits > 64 || (bits & 7)) return CKS_EINVAL;
    ctx->round0_bits = bits;
    return CKS_OK;
}

int cks_ctx_set_speculative_mask(cks_ctx* ctx, int enable) {
    if (!ctx) return CKS_EINVAL;
    ctx->spec_on = enable != 0;
    return CKS_OK;
}

int cks_ctx_speculation_stats(const cks_ctx* ctx, uint64_t* builds, uint64_t* retries) {
    if (!ctx) return CKS_EINVAL;
    if (builds) *builds = ctx->spec_builds;
    if (retries) *retries = ctx->spec_retries;
    return CKS_OK;
}

int cks_ctx_set_verify(cks_ctx* ctx, int mode) {
    if (!ctx || mode < CKS_VERIFY_OFF || mode > CKS_VERIFY_ALWAYS) return CKS_EINVAL;
    ctx->verify = mode;
    return CKS_OK;
}

int cks_ctx_stage_ms(cks_ctx* ctx, float* out, int max) {
    if (!ctx || !out) return 0;
    if (!ctx->timed) return 0;
    cudaEventSynchronize(ctx->ev[ST_BULK]);
    int k = 0;
    for (int s = ST_MASK; s < ST_N && k < max; s++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[s - 1], ctx->ev[s]);
        out[k++] = ms;
    }
    if (k < max) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[ST_BEGIN], ctx->ev[ST_BULK]);
        out[k++] = ms;
    }
    return k;
}

uint64_t cks_ctx_launches(const cks_ctx* ctx) { return ctx ? ctx->launches : 0; }

int cks_ctx_kernel_stats(cks_ctx* ctx, double* ms, double* bytes, uint32_t* count) {
    if (!ctx || !ms || !bytes || !count) return CKS_EINVAL;
    *ms = 0.0;
    *bytes = 0.0;
    *count = 0;
    if (!ctx->timed) return CKS_OK;
    for (int i = 0; i < ctx->nkev; i++) {
        CK(cudaEventSynchronize(ctx->kev[2 * i + 1]));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ctx->kev[2 * i], ctx->kev[2 * i + 1]));
        *ms += t;
        *bytes += ctx->kbytes[i];
    }
    *count = (uint32_t)ctx->nkev;
    return CKS_OK;
}

int cks_ctx_path_bytes(const cks_ctx* ctx, double* bytes) {
    if (!ctx || !bytes) return CKS_EINVAL;
    *bytes = ctx->path_bytes;
    return CKS_OK;
}

const char* cks_strerror(int code) {
    switch (code) {
        case CKS_OK: return "ok";
        case CKS_EINVAL: return "invalid argument";
        case CKS_ERANGE: return "out of range";
        case CKS_ENOMEM: return "out of device memory";
        case CKS_ECUDA: return "CUDA error";
        default: return "unknown error";
    }
}

const char* cks_last_error(const cks_ctx* ctx) { return ctx ? ctx->err : "no context"; }

int cks_superset_mask(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, int kind,
                      uint8_t* mask_out, uint32_t* popcount_out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!mask_out) return fail(ctx, CKS_EINVAL, "mask_out is NULL");
    CK(cudaSetDevice(ctx->device));
    uint32_t m = 0;
    TRY(run_superset(ctx, keys, n, B, kind, mask_out, &m));
    if (popcount_out) *popcount_out = m;
    return CKS_OK;
}

int cks_occupancy(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, uint32_t* occ_out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!occ_out) return fail(ctx, CKS_EINVAL, "occ_out is NULL");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemsetAsync(occ_out, 0, (size_t)B * 8 * 4, ctx->stream));
    if (n) LAUNCH(launch_occupancy(keys, n, B, occ_out, ctx->sms, ctx->stream));
    return CKS_OK;
}

int cks_occupancy_sample(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, uint32_t samples,
                         uint32_t* occ_out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!occ_out) return fail(ctx, CKS_EINVAL, "occ_out is NULL");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemsetAsync(occ_out, 0, (size_t)B * 8 * 4, ctx->stream));
    if (n && compress_marks_occupancy(keys, B) && samples && samples < n) {
        LAUNCH(launch_occupancy_sample(keys, n, B, samples, occ_out, ctx->stream));
        BYTES((double)samples * B);
    } else if (n) {
        LAUNCH(launch_occupancy(keys, n, B, occ_out, ctx->sms, ctx->stream));
        BYTES((double)n * B);
    }
    return CKS_OK;
}

int cks_compress_marking(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* mask,
                         uint32_t* packed_out, uint32_t* occ_out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!mask || !occ_out) return fail(ctx, CKS_EINVAL, "mask or occ_out is NULL");
    if (n && !compress_marks_occupancy(keys, B))
        return fail(ctx, CKS_EINVAL, "cks_compress_marking needs 16-byte aligned keys of 8, 16, 32 or 64 bytes");
    const uint32_t m = popcount_mask(mask, B);
    if (n && m && !packed_out) return fail(ctx, CKS_EINVAL, "packed_out is NULL");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemsetAsync(occ_out, 0, (size_t)B * 8 * 4, ctx->stream));
    if (n && m) {
        TRY(run_compress(ctx, keys, n, B, mask, packed_out, n, 0, nullptr, occ_out));
    } else if (n) {                                               // (no planes: the occupancy alone)
        LAUNCH(launch_occupancy(keys, n, B, occ_out, ctx->sms, ctx->stream));
    }
    return check_guards(ctx);
}

int cks_occupancy_mask(cks_ctx* ctx, const uint32_t* occ, uint32_t nocc, uint32_t B, uint64_t n_total, int kind,
                       uint8_t* mask_out, uint32_t* popcount_out) {
    if (!ctx) return CKS_EINVAL;
    if (B < 1 || B > CKS_MAX_KEY_BYTES) return fail(ctx, CKS_EINVAL, "key_bytes %u not in [1,512]", B);
    if (!occ || nocc == 0 || !mask_out) return fail(ctx, CKS_EINVAL, "NULL occupancy or mask, or nocc = 0");
    CK(cudaSetDevice(ctx->device));
    TRY(ensure(ctx, ctx->occ, (size_t)B * 8 * 4));
    LAUNCH(launch_occ_union(occ, nocc, B * 8, as<uint32_t>(ctx->occ), ctx->stream));
    uint32_t m = 0;
    TRY(run_superset(ctx, nullptr, n_total, B, kind, mask_out, &m, /*keys_ready=*/false));
    if (popcount_out) *popcount_out = m;
    return check_guards(ctx);
}

int cks_rank_sorted(cks_ctx* ctx, const uint32_t* sorted_packed, uint32_t bits, uint64_t n, const uint32_t* sorted_rid,
                    uint64_t rid_base, const uint32_t* queries, uint32_t nq, uint64_t* ranks_out) {
    if (!ctx) return CKS_EINVAL;
    if (bits > kMaxBits) return fail(ctx, CKS_EINVAL, "packed_bits %u > %u", bits, kMaxBits);
    if (nq && (!queries || !ranks_out)) return fail(ctx, CKS_EINVAL, "NULL queries or ranks_out");
    if (n && nq && (!sorted_rid || (bits && !sorted_packed))) return fail(ctx, CKS_EINVAL, "NULL sorted input");
    CK(cudaSetDevice(ctx->device));
    LAUNCH(launch_rank_sorted(sorted_packed, (bits + 31) / 32, n, sorted_rid, rid_base, queries, nq,
                              reinterpret_cast<unsigned long long*>(ranks_out), ctx->stream));
    return check_guards(ctx);
}

int cks_partition(cks_ctx* ctx, const uint32_t* packed, uint32_t bits, uint64_t n, const uint32_t* splitters,
                  uint32_t parts, uint64_t rid_base, uint32_t* packed_out, uint32_t* rid_out, uint64_t* counts_out) {
    if (!ctx) return CKS_EINVAL;
    if (bits > kMaxBits) return fail(ctx, CKS_EINVAL, "packed_bits %u > %u", bits, kMaxBits);
    if (parts < 1 || parts > 256) return fail(ctx, CKS_EINVAL, "parts %u not in [1, 256]", parts);
    if (n >= (1ull << 32) || rid_base + n > (1ull << 32)) return fail(ctx, CKS_ERANGE, "row ids exceed u32");
    if (!counts_out || (parts > 1 && !splitters)) return fail(ctx, CKS_EINVAL, "NULL splitters or counts_out");
    if (n && (!rid_out || (bits && (!packed || !packed_out)))) return fail(ctx, CKS_EINVAL, "NULL buffer with n > 0");
    CK(cudaSetDevice(ctx->device));
    const uint32_t np = (bits + 31) / 32;
    if (parts == 1 || n == 0) {                                   // one part: the input order
        const unsigned long long cnt = n;
        CK(cudaMemsetAsync(counts_out, 0, (size_t)parts * 8, ctx->stream));
        CK(cudaMemcpyAsync(counts_out, &cnt, 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));                   // (&cnt is on the stack)
        if (n && np) CK(cudaMemcpyAsync(packed_out, packed, (size_t)np * n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        if (n) {
            LAUNCH(launch_iota(rid_out, n, ctx->stream));
            LAUNCH(launch_add_base(rid_out, n, (uint32_t)rid_base, ctx->sms, ctx->stream));
        }
        return CKS_OK;
    }
    // [part index, P planes] -> one LSD pass on the part index's low byte (stable)
    const uint64_t sp = scratch_pitch(n);
    TRY(ensure(ctx, ctx->part_in, (size_t)(np + 1) * sp * 4));
    TRY(ensure(ctx, ctx->part_out, (size_t)(np + 1) * sp * 4));
    uint32_t* in = as<uint32_t>(ctx->part_in);
    uint32_t* out = as<uint32_t>(ctx->part_out);
    LAUNCH(launch_part_dest(packed, np, n, n, splitters, parts - 1, rid_base, in,
                            reinterpret_cast<unsigned long long*>(counts_out), ctx->sms, ctx->stream));
    if (np) CK(cudaMemcpy2DAsync(in + sp, sp * 4, packed, n * 4, n * 4, np, cudaMemcpyDeviceToDevice, ctx->stream));
    TRY(run_sort(ctx, in, sp, np + 1, 1, n, nullptr, 0, out, sp, rid_out, nullptr, nullptr, 0, false));
    if (np) CK(cudaMemcpy2DAsync(packed_out, n * 4, out + sp, sp * 4, n * 4, np, cudaMemcpyDeviceToDevice, ctx->stream));
    LAUNCH(launch_add_base(rid_out, n, (uint32_t)rid_base, ctx->sms, ctx->stream));
    return check_guards(ctx);
}

int cks_partition_count(cks_ctx* ctx, const uint32_t* packed, uint32_t bits, uint64_t n, const uint32_t* splitters,
                        uint32_t parts, uint64_t rid_base, uint64_t* counts_out) {
    if (!ctx) return CKS_EINVAL;
    if (bits > kMaxBits) return fail(ctx, CKS_EINVAL, "packed_bits %u > %u", bits, kMaxBits);
    if (parts < 1 || parts > 256) return fail(ctx, CKS_EINVAL, "parts %u not in [1, 256]", parts);
    if (n >= (1ull << 32) || rid_base + n > (1ull << 32)) return fail(ctx, CKS_ERANGE, "row ids exceed u32");
    if (!counts_out || (parts > 1 && !splitters) || (n && bits && !packed))
        return fail(ctx, CKS_EINVAL, "NULL splitters, counts_out or packed");
    CK(cudaSetDevice(ctx->device));
    const uint32_t np = (bits + 31) / 32;
    const uint64_t sp = scratch_pitch(n);
    TRY(ensure(ctx, ctx->part_in, (size_t)(np + 1) * sp * 4));
    uint32_t* in = as<uint32_t>(ctx->part_in);
    CK(cudaMemsetAsync(counts_out, 0, (size_t)parts * 8, ctx->stream));
    if (n) {
        if (parts > 1) {
            LAUNCH(launch_part_dest(packed, np, n, n, splitters, parts - 1, rid_base, in,
                                    reinterpret_cast<unsigned long long*>(counts_out), ctx->sms, ctx->stream));
        } else {
            CK(cudaMemsetAsync(in, 0, n * 4, ctx->stream));
            const unsigned long long cnt = n;
            CK(cudaMemcpyAsync(counts_out, &cnt, 8, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));                   // (&cnt is on the stack)
        }
        if (np) CK(cudaMemcpy2DAsync(in + sp, sp * 4, packed, n * 4, n * 4, np, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ctx->ps_n = n;
    ctx->ps_np = np;
    ctx->ps_parts = parts;
    ctx->ps_rid_base = rid_base;
    return check_guards(ctx);
}

int cks_partition_send(cks_ctx* ctx, uint32_t* const* dst_planes, const uint64_t* dst_pitch, uint32_t* const* dst_rid) {
    if (!ctx) return CKS_EINVAL;
    const uint32_t parts = ctx->ps_parts, np = ctx->ps_np;
    const uint64_t n = ctx->ps_n;
    if (parts == 0) return fail(ctx, CKS_EINVAL, "cks_partition_send without cks_partition_count");
    if (!dst_rid || (np && (!dst_planes || !dst_pitch))) return fail(ctx, CKS_EINVAL, "NULL destination tables");
    CK(cudaSetDevice(ctx->device));
    ctx->ps_parts = 0;
    if (n == 0) return CKS_OK;
    // pointer table: stream k = 1..np is plane k-1, stream np+1 the row id; 256 parts per stream
    const size_t ptab = (size_t)(np + 1) * 256;
    TRY(ensure(ctx, ctx->part_ptrs, ptab * sizeof(uint32_t*) + 256 * 4 + 16));
    std::vector<uint32_t*> h(ptab, nullptr);
    for (uint32_t d = 0; d < parts; d++) {
        for (uint32_t q = 0; q < np; q++) h[(size_t)q * 256 + d] = dst_planes[d] + q * dst_pitch[d];
        h[(size_t)np * 256 + d] = dst_rid[d];
    }
    CK(cudaMemcpyAsync(ctx->part_ptrs.p, h.data(), ptab * sizeof(uint32_t*), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));                       // (h is on the stack)
    const uint64_t sp = scratch_pitch(n);
    uint64_t lsd_tiles = 0, lsd_chunks = 0;
    lsd_sizes(n, &lsd_tiles, &lsd_chunks);
    TRY(ensure(ctx, ctx->tile_off, (size_t)lsd_tiles * 256 * 4));
    TRY(ensure(ctx, ctx->chunk_tot, (size_t)lsd_chunks * 256 * 4));
    TRY(ensure(ctx, ctx->total, 256 * 4, /*zero=*/true));
    LsdPassArgs la;
    memset(&la, 0, sizeof(la));
    la.in_planes = as<uint32_t>(ctx->part_in);
    la.out_planes = as<uint32_t>(ctx->part_in);                  // (not written: every stream is scattered)
    la.out_rid = as<uint32_t>(ctx->part_in);
    la.n = n;
    la.in_pitch = sp;
    la.out_pitch = sp;
    la.nplanes = np + 1;
    la.digit_plane = 0;
    la.shift = 0;
    la.tile_off = as<uint32_t>(ctx->tile_off);
    la.chunk_tot = as<uint32_t>(ctx->chunk_tot);
    la.total = as<uint32_t>(ctx->total);
    la.rid_add = (uint32_t)ctx->ps_rid_base;
    la.part_dst = as<uint32_t* const>(ctx->part_ptrs);
    la.bbase = reinterpret_cast<uint32_t*>(as<uint8_t>(ctx->part_ptrs) + ptab * sizeof(uint32_t*));
    LsdAux aux;
    aux.stream = ctx->aux_stream;
    aux.fork = ctx->aux_ev[0];
    aux.join = ctx->aux_ev[1];
    int nl = 0;
    CK(launch_lsd_pass(la, ctx->sms, ctx->stream, aux, &nl));
    ctx->launches += (uint64_t)nl;
    BYTES((double)n * 4.0 * (1 + (np + 1) + (np + 1)));
    return check_guards(ctx);
}

int cks_sort_prefix(cks_ctx* ctx, const uint32_t* packed, const uint8_t* sort_mask, uint32_t B, uint64_t n,
                    uint32_t* perm_out, uint16_t* dbit_out, uint8_t* mask_out, uint32_t* popcount_out,
                    uint32_t* packed_out) {
    if (!ctx) return CKS_EINVAL;
    if (B < 1 || B > CKS_MAX_KEY_BYTES) return fail(ctx, CKS_EINVAL, "key_bytes %u not in [1,512]", B);
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n >= 2^32");
    if (!sort_mask || !mask_out) return fail(ctx, CKS_EINVAL, "mask pointer is NULL");
    const uint32_t m = popcount_mask(sort_mask, B);
    if (n && (!perm_out || !dbit_out || (m && !packed))) return fail(ctx, CKS_EINVAL, "NULL buffer with n > 0");
    CK(cudaSetDevice(ctx->device));
    ctx->timed = ctx->timing;
    ctx->nkev = 0;
    ctx->path_bytes = 0.0;
    mark(ctx, ST_BEGIN);
    cks_build_out o;
    memset(&o, 0, sizeof(o));
    o.mask = mask_out;
    o.perm = perm_out;
    o.dbit = dbit_out;
    o.fanout = 64;
    o.fill = 1.f;
    if (n == 0) {
        memset(mask_out, 0, B);
        if (popcount_out) *popcount_out = 0;
        return CKS_OK;
    }
    ctx->skip_packed = packed_out == nullptr;
    const int rc = build_from_mask(ctx, nullptr, n, B, sort_mask, m, &o, packed);
    ctx->skip_packed = false;
    TRY(rc);
    if (popcount_out) *popcount_out = o.popcount;
    if (packed_out && o.popcount && o.packed)
        CK(cudaMemcpy2DAsync(packed_out, n * 4, o.packed, o.packed_pitch * 4, n * 4, (o.popcount + 31) / 32,
                             cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return check_guards(ctx);
}

int cks_bulkload_block(cks_ctx* ctx, const uint32_t* perm, const uint16_t* dbit, uint64_t n, uint32_t fanout, double fill,
                       int first_global, uint32_t levels, cks_tree* out, uint16_t* top_min_out, uint32_t* height_out) {
    if (!ctx) return CKS_EINVAL;
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n >= 2^32");
    if (n && !perm) return fail(ctx, CKS_EINVAL, "perm is NULL");
    CK(cudaSetDevice(ctx->device));
    uint32_t h = 0;
    TRY(run_bulkload(ctx, perm, dbit, n, fanout, fill, out, &h, first_global != 0, levels, top_min_out));
    if (height_out) *height_out = h;
    return check_guards(ctx);
}

int cks_bulkload_top(cks_ctx* ctx, const uint32_t* child_rid, const uint16_t* child_min, uint64_t nchild,
                     uint32_t fanout, double fill, cks_tree* out, uint32_t* height_out) {
    if (!ctx) return CKS_EINVAL;
    if (nchild && (!child_rid || !child_min)) return fail(ctx, CKS_EINVAL, "NULL child arrays");
    CK(cudaSetDevice(ctx->device));
    uint32_t h = 0;
    TRY(run_bulkload_top(ctx, child_rid, child_min, nchild, fanout, fill, out, &h));
    if (height_out) *height_out = h;
    return check_guards(ctx);
}

int cks_repack(cks_ctx* ctx, const uint32_t* packed_in, const uint8_t* in_mask, const uint8_t* out_mask, uint32_t B,
               uint64_t n, uint32_t* packed_out) {
    if (!ctx) return CKS_EINVAL;
    if (B < 1 || B > CKS_MAX_KEY_BYTES) return fail(ctx, CKS_EINVAL, "key_bytes %u not in [1,512]", B);
    if (!in_mask || !out_mask) return fail(ctx, CKS_EINVAL, "mask pointer is NULL");
    for (uint32_t j = 0; j < B; j++)
        if (out_mask[j] & ~in_mask[j]) return fail(ctx, CKS_EINVAL, "out_mask is not a subset of in_mask (byte %u)", j);
    const uint32_t m = popcount_mask(in_mask, B), d = popcount_mask(out_mask, B);
    if (n == 0 || d == 0) return CKS_OK;
    if (!packed_in || !packed_out) return fail(ctx, CKS_EINVAL, "NULL packed buffer");
    CK(cudaSetDevice(ctx->device));
    const uint32_t np = (m + 31) / 32;
    std::vector<uint32_t> sub(np, 0);
    repack_words(in_mask, out_mask, B, m, 0, sub);
    TRY(claim_slot(ctx, 1));
    plan_repack(sub.data(), np, ctx->h_plan[1]);
    GatherPlan* dplan;
    TRY(upload_plan(ctx, 1, &dplan));
    LAUNCH(launch_repack(packed_in, n, n, dplan, ctx->h_plan[1]->nsteps, (d + 31) / 32, packed_out, n, ctx->sms,
                         ctx->stream));
    return check_guards(ctx);
}

int cks_compress(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* mask,
                 uint32_t* packed_out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!mask) return fail(ctx, CKS_EINVAL, "mask is NULL");
    uint32_t m = popcount_mask(mask, B);
    if (n && m && !packed_out) return fail(ctx, CKS_EINVAL, "packed_out is NULL");
    CK(cudaSetDevice(ctx->device));
    TRY(run_compress(ctx, keys, n, B, mask, packed_out, n));
    return check_guards(ctx);
}

int cks_sort(cks_ctx* ctx, const uint32_t* packed, uint32_t bits, uint64_t n, const uint32_t* row_ids,
             uint32_t* perm_out, uint32_t* sorted_packed_out) {
    if (!ctx) return CKS_EINVAL;
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n >= 2^32");
    if (bits > kMaxBits) return fail(ctx, CKS_EINVAL, "packed_bits %u > %u", bits, kMaxBits);
    if (n && (!perm_out || (bits && !packed))) return fail(ctx, CKS_EINVAL, "NULL buffer with n > 0");
    CK(cudaSetDevice(ctx->device));
    const uint32_t np = (bits + 31) / 32, k = (bits + 7) / 8;
    TRY(run_sort(ctx, packed, n, np, k, n, row_ids, 4, sorted_packed_out, n, perm_out, nullptr, nullptr));
    return check_guards(ctx);
}

int cks_adjacent_dbits(cks_ctx* ctx, const uint32_t* sorted_packed, uint32_t bits, uint64_t n,
                       const uint8_t* sort_mask, uint32_t B, uint8_t* mask_out, uint32_t* popcount_out,
                       uint16_t* dbit_out) {
    if (!ctx) return CKS_EINVAL;
    if (B < 1 || B > CKS_MAX_KEY_BYTES) return fail(ctx, CKS_EINVAL, "key_bytes %u not in [1,512]", B);
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n >= 2^32");
    if (n && bits && !sorted_packed) return fail(ctx, CKS_EINVAL, "sorted_packed is NULL");
    if (!sort_mask || !mask_out) return fail(ctx, CKS_EINVAL, "mask pointer is NULL");
    CK(cudaSetDevice(ctx->device));
    TRY(run_adjacent(ctx, sorted_packed, n, bits, n, sort_mask, B, mask_out, dbit_out));
    if (popcount_out) *popcount_out = popcount_mask(mask_out, B);
    return check_guards(ctx);
}

int cks_bulkload_shape(uint64_t n, uint32_t fanout, double fill, cks_tree_shape* out) {
    return tree_shape(n, fanout, fill, out);
}

int cks_paper_tree_shape(uint64_t n, double fill, cks_tree_shape* s) {
    if (!s || !(fill > 0.f) || fill > 1.f) return CKS_EINVAL;
    const uint32_t lp = (uint32_t)((double)CKS_PTREE_LEAF_FANOUT * (double)fill);
    const uint32_t ip = (uint32_t)((double)CKS_PTREE_INNER_FANOUT * (double)fill);
    if (lp < 2 || ip < 2) return CKS_EINVAL;
    memset(s, 0, sizeof(*s));
    s->n = n;
    s->fanout = CKS_PTREE_LEAF_FANOUT;
    s->per_node = lp;
    s->reserved = ip;                                    // entries per non-leaf node
    uint64_t c = n, off = 0, per = lp;
    uint32_t h = 0;
    while (c > 0) {
        c = (c + per - 1) / per;
        if (h >= CKS_MAX_LEVELS) return CKS_ERANGE;
        s->level_nodes[h] = c;
        s->level_offset[h] = off;
        off += c;
        h++;
        per = ip;
        if (c <= 1) break;
    }
    s->height = h;
    s->total_nodes = off;
    s->inner_nodes = h ? off - s->level_nodes[0] : 0;
    return CKS_OK;
}

int cks_paper_tree(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm,
                   const uint16_t* dbit, uint32_t pk_bits, double fill, uint8_t* nodes) {
    TRY(check_keys(ctx, keys, n, B));
    if (pk_bits > 32) return fail(ctx, CKS_EINVAL, "pk_bits %u > 32", pk_bits);
    if (n && (!perm || !dbit || !nodes)) return fail(ctx, CKS_EINVAL, "NULL perm, dbit or nodes with n > 0");
    cks_tree_shape s;
    const int rc = cks_paper_tree_shape(n, fill, &s);
    if (rc != CKS_OK) return fail(ctx, rc, "bad paper-tree shape (fill %f)", (double)fill);
    if (n == 0) return CKS_OK;
    CK(cudaSetDevice(ctx->device));
    PtreeWs ws;
    TRY(ptree_ws(ctx, s.level_nodes[0], &ws));
    int nl = 0;
    CK(launch_ptree(keys, n, B, perm, dbit, pk_bits, s.per_node, s.reserved, s.level_nodes, s.level_offset,
                    s.height, nodes, ws, ctx->sms, ctx->stream, &nl));
    ctx->launches += (uint64_t)nl;
    return check_guards(ctx);
}

int cks_paper_tree_ds(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm,
                      const uint16_t* dbit, const uint32_t* sorted_packed, uint64_t packed_pitch,
                      const uint8_t* packed_mask, const uint8_t* variant, const uint8_t* ref_key, uint32_t pk_bits,
                      double fill, uint8_t* nodes) {
    if (!ctx) return CKS_EINVAL;
    if (B < 1 || B > CKS_MAX_KEY_BYTES) return fail(ctx, CKS_EINVAL, "key_bytes %u not in [1,512]", B);
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n >= 2^32");
    if (pk_bits > 32) return fail(ctx, CKS_EINVAL, "pk_bits %u > 32", pk_bits);
    if (!packed_mask || !variant || !ref_key) return fail(ctx, CKS_EINVAL, "NULL DS-metadata mask or key");
    const uint32_t mx = popcount_mask(packed_mask, B);
    if (n && mx && (!sorted_packed || packed_pitch < n)) return fail(ctx, CKS_EINVAL, "NULL planes or pitch < n");
    CK(cudaSetDevice(ctx->device));
    const uint32_t np = (mx + 31) / 32;
    TRY(run_ptree_ds(ctx, keys, n, B, perm, dbit, sorted_packed, packed_pitch, np, packed_mask, 32 * np - mx, nullptr,
                     0, variant, ref_key, pk_bits, fill, nodes));
    return check_guards(ctx);
}

int cks_bulkload(cks_ctx* ctx, const uint32_t* perm, const uint16_t* dbit, uint64_t n, uint32_t fanout,
                 double fill, const cks_tree* out) {
    if (!ctx) return CKS_EINVAL;
    if (n >= (1ull << 32)) return fail(ctx, CKS_ERANGE, "n >= 2^32");
    if (n && !perm) return fail(ctx, CKS_EINVAL, "perm is NULL");
    CK(cudaSetDevice(ctx->device));
    TRY(run_bulkload(ctx, perm, dbit, n, fanout, fill, out, nullptr));
    return check_guards(ctx);
}

int cks_distinction_mask(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* prior,
                         uint8_t* mask_out, uint32_t* popcount_out, uint32_t* perm_out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!mask_out) return fail(ctx, CKS_EINVAL, "mask_out is NULL");
    CK(cudaSetDevice(ctx->device));
    cks_build_out o;
    memset(&o, 0, sizeof(o));
    o.mask = mask_out;
    o.superset_kind = CKS_SUPERSET_BYTEOCC;
    o.perm = perm_out;
    if (!perm_out && n) {                 // the last LSD pass still needs somewhere to put row ids
        TRY(ensure(ctx, ctx->perm_scratch, n * 4));
        o.perm = as<uint32_t>(ctx->perm_scratch);
    }
    TRY(build_common(ctx, keys, n, B, prior, &o, true));
    if (popcount_out) *popcount_out = o.popcount;
    return check_guards(ctx);
}

int cks_build(cks_ctx* ctx, const uint8_t* keys, uint64_t n, uint32_t B, const uint8_t* prior,
              cks_build_out* out) {
    TRY(check_keys(ctx, keys, n, B));
    if (!out || !out->mask || (n && !out->perm)) return fail(ctx, CKS_EINVAL, "NULL output");
    CK(cudaSetDevice(ctx->device));
    ctx->timed = ctx->timing;
    ctx->nkev = 0;
    ctx->path_bytes = 0.0;
    mark(ctx, ST_BEGIN);
    return build_common(ctx, keys, n, B, prior, out, true);
}

int cks_build_host(cks_ctx* ctx, const uint8_t* host_keys, uint64_t n, uint32_t B, const uint8_t* prior,
                   cks_build_out* out) {
    TRY(check_keys(ctx, host_keys, n, B));
    if (!out || !out->mask || (n && !out->perm)) return fail(ctx, CKS_EINVAL, "NULL output");
    if (out->dbit || out->tree.node_cnt) return fail(ctx, CKS_EINVAL, "cks_build_host: dbit/tree must be NULL");
    CK(cudaSetDevice(ctx->device));
    ctx->timed = ctx->timing;
    ctx->nkev = 0;
    ctx->path_bytes = 0.0;
    mark(ctx, ST_BEGIN);
    const size_t bytes = (size_t)n * B;
    TRY(ensure(ctx, ctx->keys, bytes));
    const uint8_t* dkeys = as<uint8_t>(ctx->keys);
    // H2D in chunks on the copy stream; the superset-mask pass of chunk c overlaps the
    // copy of chunk c+1 (occupancy is order-independent, so partial passes just OR).
    const bool want_mask = prior == nullptr;
    if (want_mask) {
        TRY(ensure(ctx, ctx->occ, (size_t)B * 8 * 4));
        CK(cudaMemsetAsync(ctx->occ.p, 0, (size_t)B * 8 * 4, ctx->stream));
    }
    uint64_t chunk_keys = ((64ull << 20) / B) & ~15ull;
    if (chunk_keys == 0) chunk_keys = 16;
    std::vector<cudaEvent_t> evs;
    for (uint64_t k0 = 0; k0 < n; k0 += chunk_keys) {
        uint64_t kc = std::min<uint64_t>(chunk_keys, n - k0);
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
        CK(cudaMemcpyAsync((void*)(dkeys + k0 * B), host_keys + k0 * B, kc * B, cudaMemcpyHostToDevice,
                           ctx->copy_stream));
        CK(cudaEventRecord(e, ctx->copy_stream));
        CK(cudaStreamWaitEvent(ctx->stream, e, 0));
        if (want_mask)
            LAUNCH(launch_occupancy(dkeys + k0 * B, kc, B, as<uint32_t>(ctx->occ), ctx->sms, ctx->stream));
    }
    uint32_t* host_perm = out->perm;
    cks_build_out o = *out;
    if (n) {
        TRY(ensure(ctx, ctx->perm_scratch, n * 4));
        o.perm = as<uint32_t>(ctx->perm_scratch);
    }
    int rc = build_common(ctx, dkeys, n, B, prior, &o, /*keys_ready_for_mask=*/false);
    if (rc == CKS_OK && n) {
        cudaError_t e = cudaMemcpyAsync(host_perm, o.perm, n * 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (e != cudaSuccess) rc = fail(ctx, CKS_ECUDA, "D2H perm: %s", cudaGetErrorString(e));
    }
    cudaError_t se = cudaStreamSynchronize(ctx->stream);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (rc == CKS_OK && se != cudaSuccess) rc = fail(ctx, CKS_ECUDA, "sync: %s", cudaGetErrorString(se));
    if (rc != CKS_OK) return rc;
    o.perm = host_perm;
    *out = o;
    return CKS_OK;
}

int cks_build_host_batch(cks_ctx* ctx, const uint8_t* const* host_keys, uint32_t count, uint64_t n, uint32_t B,
                         const uint8_t* prior, cks_build_out* outs) {
    if (!ctx) return CKS_EINVAL;
    if (count == 0) return CKS_OK;
    if (!host_keys || !outs) return fail(ctx, CKS_EINVAL, "NULL host_keys or outs");
    for (uint32_t i = 0; i < count; i++) {
        TRY(check_keys(ctx, host_keys[i], n, B));
        if (!outs[i].mask || (n && !outs[i].perm)) return fail(ctx, CKS_EINVAL, "NULL output (column %u)", i);
        if (outs[i].dbit || outs[i].tree.node_cnt) return fail(ctx, CKS_EINVAL, "batch: dbit/tree must be NULL");
    }
    CK(cudaSetDevice(ctx->device));
    const size_t bytes = (size_t)n * B;
    TRY(ensure(ctx, ctx->keys, bytes));
    TRY(ensure(ctx, ctx->keys2, bytes));
    TRY(ensure(ctx, ctx->perm_scratch, n * 4 + 16));
    TRY(ensure(ctx, ctx->perm2, n * 4 + 16));
    uint8_t* kb[2] = {as<uint8_t>(ctx->keys), as<uint8_t>(ctx->keys2)};
    uint32_t* pb[2] = {as<uint32_t>(ctx->perm_scratch), as<uint32_t>(ctx->perm2)};
    cudaEvent_t* in_ev = ctx->bev;          // [2] keys of column i in kb[i & 1]
    cudaEvent_t* done_ev = ctx->bev + 2;    // [2] build of the column in buffer b finished
    cudaEvent_t* out_ev = ctx->bev + 4;     // [2] perm of buffer b copied out
    // the copy of column i+1 runs (copy stream) while column i builds (library stream) and
    // column i-1's permutation goes back (d2h stream): H2D and D2H use both PCIe directions
    auto copy_in = [&](uint32_t i) -> int {
        const int b = (int)(i & 1);
        if (i >= 2) CK(cudaStreamWaitEvent(ctx->copy_stream, done_ev[b], 0));    // kb[b] free
        if (bytes) CK(cudaMemcpyAsync(kb[b], host_keys[i], bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
        CK(cudaEventRecord(in_ev[b], ctx->copy_stream));
        return CKS_OK;
    };
    TRY(copy_in(0));
    for (uint32_t i = 0; i < count; i++) {
        const int b = (int)(i & 1);
        if (i + 1 < count) TRY(copy_in(i + 1));
        CK(cudaStreamWaitEvent(ctx->stream, in_ev[b], 0));
        if (i >= 2) CK(cudaStreamWaitEvent(ctx->stream, out_ev[b], 0));             // pb[b] free
        ctx->timed = ctx->timing;
        ctx->nkev = 0;
        ctx->path_bytes = 0.0;
        mark(ctx, ST_BEGIN);
        cks_build_out o = outs[i];
        o.perm = pb[b];
        TRY(build_common(ctx, kb[b], n, B, prior, &o, /*keys_ready_for_mask=*/true));
        CK(cudaEventRecord(done_ev[b], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->d2h_stream, done_ev[b], 0));
        if (n) CK(cudaMemcpyAsync(outs[i].perm, pb[b], n * 4, cudaMemcpyDeviceToHost, ctx->d2h_stream));
        CK(cudaEventRecord(out_ev[b], ctx->d2h_stream));
        uint32_t* host_perm = outs[i].perm;
        outs[i] = o;
        outs[i].perm = host_perm;
        outs[i].packed = nullptr;                  // (device views of a reused buffer: not returned)
    }
    CK(cudaStreamSynchronize(ctx->d2h_stream));
    CK(cudaStreamSynchronize(ctx->copy_stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CKS_OK;
}

}  // extern "C"
