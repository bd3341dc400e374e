// k_lsd.cu -- a5: one stable LSD digit pass as reduce-then-scan ("sort the pairs").
//
// Three kernels per 8-bit digit, no inter-tile waiting:
//   k_upsweep    CTA per chunk of CT consecutive tiles: per-tile digit counts (per-warp
//                shared-memory bins), stored as within-chunk exclusive offsets
//                tile_off[tile][256]; chunk totals chunk_tot[chunk][256]; digit totals
//                accumulated into total[256] with one atomic per digit per chunk.
//   k_chunk_scan bucket base of every digit (exclusive scan of total[]) plus the exclusive
//                scan of chunk totals over chunks, in place: chunk_tot -> chunk_base.
//   k_downsweep  persistent CTAs over a static tile schedule (tile = blockIdx + i*grid).
//                All streams of the tile (digit word, other planes, row id) are fetched by
//                1-D TMA bulk copies into a ring of shared-memory slots that runs ahead
//                across tiles (the next tile of a CTA is known statically), so the loads of
//                the next tile overlap the work on this one. The digit is ranked per warp
//                (bit-plane ballots; the group leader reserves slots with a shared atomic,
//                applied in issue order: stable); the resulting tile permutation is stored
//                once as a u16 source index per output slot, and every stream is gathered
//                from its slot in that order and written in coalesced runs to
//                chunk_base[chunk][d] + tile_off[tile][d] + rank.
// Compared with a single-kernel "onesweep" pass this reads the digit words twice (+4 B/key)
// but has no decoupled look-back and no dynamic tile counter on the critical path.
#include <stdlib.h>

#include <type_traits>

#include "cks_internal.h"
#include "cks_ptx.cuh"

namespace cks {

namespace {

constexpr int kW = kSortThreads / 32;
// timing-only debug modes of the downsweep (wrong results): compiled in only with CKS_EXPERIMENTS
#if defined(CKS_EXPERIMENTS) && CKS_EXPERIMENTS
constexpr bool kLsdDebug = true;
#else
constexpr bool kLsdDebug = false;
#endif

// Programmatic dependent launch: the kernels of a pass are launched with programmatic stream
// serialisation, so a kernel's CTAs can be scheduled while its predecessor drains; each
// waits here before touching what the predecessor wrote.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t lt_mask() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t scan256(uint32_t v, uint32_t* s_warp) {      // exclusive
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t t = lane < kW ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < kW; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kW) s_warp[lane] = t;
    }
    __syncthreads();
    uint32_t r = (warp ? s_warp[warp - 1] : 0) + x - v;
    __syncthreads();
    return r;
}
// stream k of a pass: 0 = digit word, then the other planes in order, then the row id
__device__ __forceinline__ int stream_plane(int k, int dp, int np) {
    if (k == 0) return dp;
    int idx = k - 1;
    int others = np - (dp >= 0 ? 1 : 0);
    if (idx < others) return idx + ((dp >= 0 && idx >= dp) ? 1 : 0);
    return -1;
}

}  // namespace

// ---- upsweep ------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t digit_of(uint32_t w, uint32_t sel) {   // byte `sel` of w
    return __byte_perm(w, 0u, 0x4440u | sel);
}

template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads)
k_upsweep(const LsdPassArgs a) {
    constexpr int TILE = kSortThreads * ITEMS;
    constexpr int V = ITEMS / 4;                              // uint4 loads per thread per tile
    // cumulative per-warp bins, one set per tile parity: tile t's counts are bins[t&1] now
    // minus bins[t&1] two tiles ago, so no per-tile clearing and one barrier per tile
    __shared__ uint32_t bins[2][kW][kRadix];
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t n = a.n;
    const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
    const uint32_t t0 = blockIdx.x * a.chunk_tiles;
    const uint32_t t1 = min(t0 + a.chunk_tiles, ntiles);
    const uint32_t* src = a.digit_plane >= 0 ? a.in_planes + (uint64_t)a.digit_plane * a.in_pitch : a.in_rid;
    const uint32_t sel = a.shift >> 3;
    const bool vec = src && ((uintptr_t)src % 16 == 0);
#pragma unroll
    for (int p = 0; p < 2; p++)
#pragma unroll
        for (int k = 0; k < kW; k++) bins[p][k][tid] = 0;
    __syncthreads();
    uint32_t running = 0, prev[2] = {0u, 0u};
    uint4 w[2][V];                                            // tiles t+1 and t+2 in flight
    auto load = [&](uint32_t t, auto b) {                      // full, aligned tiles only
        const uint4* s4 = reinterpret_cast<const uint4*>(src + (uint64_t)t * TILE);
#pragma unroll
        for (int v = 0; v < V; v++) w[decltype(b)::value][v] = __ldg(s4 + v * kSortThreads + tid);
    };
    auto is_fast = [&](uint32_t t) { return vec && t < t1 && (uint64_t)(t + 1) * TILE <= n; };
    if (is_fast(t0)) load(t0, std::integral_constant<int, 0>{});
    if (is_fast(t0 + 1)) load(t0 + 1, std::integral_constant<int, 1>{});
    // one tile; P (the buffer / bin parity) is a compile-time constant so w stays in registers
    auto tile_step = [&](auto pc, uint32_t t) {
        constexpr int P = decltype(pc)::value;
        uint32_t* hb = bins[P][warp];
        if (is_fast(t)) {
            uint4 c[V];
#pragma unroll
            for (int v = 0; v < V; v++) c[v] = w[P][v];
            if (is_fast(t + 2)) load(t + 2, pc);              // two tiles ahead
#pragma unroll
            for (int v = 0; v < V; v++) {
                atomicAdd(&hb[digit_of(c[v].x, sel)], 1u);
                atomicAdd(&hb[digit_of(c[v].y, sel)], 1u);
                atomicAdd(&hb[digit_of(c[v].z, sel)], 1u);
                atomicAdd(&hb[digit_of(c[v].w, sel)], 1u);
            }
        } else {
            const uint64_t tb = (uint64_t)t * TILE;
            for (int i = 0; i < ITEMS; i++) {
                const uint64_t idx = tb + (uint64_t)i * kSortThreads + tid;
                if (idx < n) atomicAdd(&hb[digit_of(src ? __ldg(src + idx) : (uint32_t)idx, sel)], 1u);
            }
        }
        __syncthreads();
        uint32_t cum = 0;
#pragma unroll
        for (int k = 0; k < kW; k++) cum += bins[P][k][tid];
        a.tile_off[(uint64_t)t * kRadix + tid] = running;
        running += cum - prev[P];
        prev[P] = cum;
    };
    for (uint32_t t = t0; t < t1; t += 2) {
        tile_step(std::integral_constant<int, 0>{}, t);
        if (t + 1 < t1) tile_step(std::integral_constant<int, 1>{}, t + 1);
    }
    a.chunk_tot[(uint64_t)blockIdx.x * kRadix + tid] = running;
    if (running) atomicAdd(&a.total[tid], running);
}

// ---- chunk scan: CTA per group of 32 digits, warps split the chunks ------------------------
__global__ void __launch_bounds__(1024)
k_chunk_scan(const LsdPassArgs a, uint32_t nchunks) {
    __shared__ uint32_t s_part[32][33];
    __shared__ uint32_t s_base[32];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t d = blockIdx.x * 32 + lane;
    if (warp < 8) {                                          // bucket bases: a scan of all 256 totals
        const uint32_t v = a.total[threadIdx.x];             // (one load each; the earlier serial sum
        uint32_t x = v;                                      // of the lower digits' totals took up to
#pragma unroll                                               // 224 dependent L2 reads, ~10 us a pass)
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        s_part[warp][lane] = x - v;                          // exclusive inside the warp
        if (lane == 31) s_part[8][warp] = x;                 // warp total
    }
    __syncthreads();
    if (warp == (int)blockIdx.x) {                           // this CTA's 32 digits = warp blockIdx.x
        uint32_t run = 0;
        for (int w = 0; w < (int)blockIdx.x; w++) run += s_part[8][w];
        s_base[lane] = run + s_part[warp][lane];
        if (a.bbase) a.bbase[d] = s_base[lane];              // (scatter-to-parts passes)
    }
    __syncthreads();
    const uint32_t per = (nchunks + 31) / 32;
    const uint32_t c0 = warp * per, c1 = min(c0 + per, nchunks);
    // up to kKeep of the warp's chunk totals stay in registers for the write-back below (one
    // read of chunk_tot instead of two: cfg5 has 436 chunks, 14 a warp)
    constexpr uint32_t kKeep = 16;
    uint32_t keep[kKeep];
    uint32_t sum = 0;
#pragma unroll
    for (uint32_t i = 0; i < kKeep; i++) {
        keep[i] = c0 + i < c1 ? a.chunk_tot[(uint64_t)(c0 + i) * kRadix + d] : 0u;
        sum += keep[i];
    }
#pragma unroll 8
    for (uint32_t c = c0 + kKeep; c < c1; c++) sum += a.chunk_tot[(uint64_t)c * kRadix + d];
    s_part[warp][lane] = sum;
    __syncthreads();
    if (warp == 0) {
        uint32_t run = s_base[lane];
        for (int k = 0; k < 32; k++) {
            uint32_t v = s_part[k][lane];
            s_part[k][lane] = run;
            run += v;
        }
    }
    __syncthreads();
    uint32_t run = s_part[warp][lane];
#pragma unroll
    for (uint32_t i = 0; i < kKeep; i++)
        if (c0 + i < c1) {
            a.chunk_tot[(uint64_t)(c0 + i) * kRadix + d] = run;
            run += keep[i];
        }
#pragma unroll 8
    for (uint32_t c = c0 + kKeep; c < c1; c++) {
        uint32_t* p = a.chunk_tot + (uint64_t)c * kRadix + d;
        uint32_t v = *p;
        *p = run;
        run += v;
    }
}

// ---- downsweep ----------------------------------------------------------------------------
// Warp match of an NB-bit label: lanes whose label equals this lane's (bit-plane ballots;
// ptxas turns the bit tests into one R2P per 7 bits, so ~3 SASS per bit).
template <int NB>
__device__ __forceinline__ uint32_t match_bits(uint32_t d) {
    uint32_t peers = 0xFFFFFFFFu;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        uint32_t m;
        asm("{\n .reg .pred p;\n .reg .b32 t;\n and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n"
            " vote.sync.ballot.b32 %0, p, 0xffffffff;\n @!p not.b32 %0, %0;\n}"
            : "=r"(m) : "r"(d), "r"(1u << b));
        peers &= m;
    }
    return peers;
}

// SCATTER (the fused partition-and-send of the sharded path): stream 0 (the part index) is not
// written, and every other stream k of an element of part d goes to
// part_dst[(k-1)*256 + d][position - bucket base of d] -- each part straight into its receiver's
// buffer (a peer device pointer over NVLink when the receiver is another GPU).
__device__ __forceinline__ uint32_t* part_out(const LsdPassArgs& a, int k, uint32_t d, uint32_t pos) {
    return a.part_dst[(uint32_t)(k - 1) * 256u + d] + (pos - a.bbase[d]);
}

template <int ITEMS, bool SCATTER>
__global__ void __launch_bounds__(kSortThreads, ITEMS == 8 ? 3 : 2)
k_downsweep(const LsdPassArgs a) {
    constexpr int TILE = kSortThreads * ITEMS;
    constexpr int HW = kRadix + 8;                            // bin row (+ label 256 of tail lanes)
    extern __shared__ __align__(128) uint8_t s_dyn[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(s_dyn);                                   // [R][TILE]
    uint32_t* s_hist = ring + (size_t)a.slots * TILE;                                     // [kW][HW]
    uint16_t* s_src = reinterpret_cast<uint16_t*>(s_hist + kW * HW);                      // [TILE] byte offsets
    __shared__ uint32_t s_warp[kW];
    __shared__ uint32_t s_gb[kRadix];
    __shared__ __align__(8) uint64_t s_bar[16];

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = a.n;
    const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
    const uint32_t G = gridDim.x;
    if (blockIdx.x == 0 && tid < kRadix) a.total[tid] = 0;      // digit totals of the next pass's upsweep
    const int np = (int)a.nplanes, dp = a.digit_plane;
    const int S = np + 1;
    const bool implicit_rid = a.in_rid == nullptr;
    const int L = S - (implicit_rid ? 1 : 0);                   // loaded streams per tile
    const int R = (int)a.slots;
    const uint32_t sel = a.shift >> 3;
    const uint32_t nfull = a.tma ? (uint32_t)(n / TILE) : 0u;   // tiles [0, nfull) arrive by TMA

    auto src_of = [&](int k) -> const uint32_t* {
        int id = stream_plane(k, dp, np);
        return id >= 0 ? a.in_planes + (uint64_t)id * a.in_pitch : a.in_rid;
    };
    auto dst_of = [&](int k) -> uint32_t* {
        int id = stream_plane(k, dp, np);
        return id >= 0 ? a.out_planes + (uint64_t)id * a.out_pitch : a.out_rid;
    };

    uint32_t p_t = a.tile_begin + blockIdx.x;                    // producer (thread 0) cursor
    int p_k = 0, p_slot = 0;
    auto produce = [&]() {
        if (p_t < nfull) {
            proxy_fence();
            bulk_load(ring + (size_t)p_slot * TILE, src_of(p_k) + (uint64_t)p_t * TILE, TILE * 4, &s_bar[p_slot]);
        }
        if (++p_slot == R) p_slot = 0;
        if (++p_k == L) { p_k = 0; p_t += G; }
    };
    if (tid == 0) {
        for (int sl = 0; sl < R; sl++) bar_init(&s_bar[sl]);
        bar_fence_init();
        for (int sl = 0; sl < R; sl++) produce();
    }
    __syncthreads();

    int c_slot = 0, c_round = 0;
    const uint32_t wofs = warp * 32 * ITEMS;
    const uint32_t ltm = lt_mask();
    uint32_t* h = s_hist + warp * HW;

    // one tile; FULL = TILE keys delivered by TMA (the hot path), else the generic tail path
    auto tile_body = [&](auto full_tag, uint32_t tile) {
        constexpr bool FULL = decltype(full_tag)::value;
        const uint64_t base = (uint64_t)tile * TILE;
        const uint32_t tile_n = FULL ? (uint32_t)TILE : (uint32_t)min((uint64_t)TILE, n - base);
        const uint32_t goff = a.chunk_tot[(uint64_t)(tile / a.chunk_tiles) * kRadix + tid] +
                              a.tile_off[(uint64_t)tile * kRadix + tid];
        auto acquire = [&](int k) -> const uint32_t* {
            uint32_t* slot = ring + (size_t)c_slot * TILE;
            if (FULL) {
                bar_wait(&s_bar[c_slot], (uint32_t)c_round & 1u);
            } else {
                const uint32_t* src = src_of(k) + base;
                for (uint32_t i = tid; i < tile_n; i += kSortThreads) slot[i] = __ldg(src + i);
                __syncthreads();
            }
            return slot;
        };
        auto release = [&]() {                                   // after a __syncthreads
            if (tid == 0) produce();
            if (++c_slot == R) { c_slot = 0; c_round++; }
        };

        // ---- rank within the warp: warp-private bins (each warp clears its own row)
#pragma unroll
        for (int j = lane; j < HW; j += 32) h[j] = 0;
        __syncwarp();
        const uint32_t* dslot = acquire(0);
        uint32_t dg[ITEMS], pos[ITEMS];
        {
            uint32_t peers[ITEMS];
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                const uint32_t idx = wofs + i * 32 + lane;
                dg[i] = (FULL || idx < tile_n) ? digit_of(dslot[idx], sel) : 0x100u;
                peers[i] = match_bits<FULL ? 8 : 9>(dg[i]);
            }
            // the group's lowest lane (unique per label) reserves the group's places in the
            // warp-private bin (predicated atomics, all issued before any result is used; a
            // __syncwarp between items orders item i's reservations before item i+1's: stable),
            // then broadcasts
            uint32_t old[ITEMS];
            const uint32_t hbase = smem_addr(h);
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                const uint32_t lower = __popc(peers[i] & ltm);
                asm volatile("{\n .reg .pred p;\n setp.eq.u32 p, %1, 0;\n mov.u32 %0, 0;\n"
                             " @p atom.shared.add.u32 %0, [%2], %3;\n}"
                             : "=r"(old[i]) : "r"(lower), "r"(hbase + dg[i] * 4), "r"((uint32_t)__popc(peers[i]))
                             : "memory");
                pos[i] = lower;
                __syncwarp();                                    // item i's reservations before item i+1's
            }
#pragma unroll
            for (int i = 0; i < ITEMS; i++) pos[i] += __shfl_sync(0xFFFFFFFFu, old[i], __ffs(peers[i]) - 1);
        }
        __syncthreads();

        // ---- digit tid: warp offsets, tile-local base, global base
        {
            uint32_t c[kW], total = 0;
#pragma unroll
            for (int k = 0; k < kW; k++) { c[k] = s_hist[k * HW + tid]; total += c[k]; }
            const uint32_t excl = scan256(total, s_warp);
            // row k of the bins becomes the tile position of warp k's first key of digit tid;
            // slot p of digit tid goes to global position p + (goff - excl)
            uint32_t run = excl;
#pragma unroll
            for (int k = 0; k < kW; k++) { s_hist[k * HW + tid] = run; run += c[k]; }
            s_gb[tid] = goff - excl;
        }
        __syncthreads();
        // ---- tile permutation: slot p <- key (warp, item, lane), as a byte offset in a slot
#pragma unroll
        for (int i = 0; i < ITEMS; i++)
            if (FULL || dg[i] < 0x100u) s_src[pos[i] + h[dg[i]]] = (uint16_t)((wofs + i * 32 + lane) * 4);
        __syncthreads();
        uint32_t from[ITEMS], dest[ITEMS], dd[ITEMS];
        // ---- stream 0 (the digit word): gather in digit order; the gathered word's digit
        // gives the slot's global destination (consecutive slots share digits: no conflicts)
        {
            uint32_t* out = dst_of(0);
            const uint8_t* slot = reinterpret_cast<const uint8_t*>(dslot);
#pragma unroll
            for (int r = 0; r < ITEMS; r++) {
                const uint32_t s = r * kSortThreads + tid;
                if (FULL || s < tile_n) {
                    from[r] = s_src[s];
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(slot + from[r]);
                    dd[r] = digit_of(w, sel);
                    dest[r] = s + s_gb[dd[r]];
                    CKS_DCHECK(dest[r] < n);
                    if (!SCATTER) out[dest[r]] = w;
                }
            }
            __syncthreads();
            release();
        }
        // ---- the other streams: same gather, same destinations
        for (int k = 1; k < S; k++) {
            uint32_t* out = dst_of(k);
            if (k == S - 1 && implicit_rid) {
                const uint32_t b32 = (uint32_t)base + a.rid_add;
#pragma unroll
                for (int r = 0; r < ITEMS; r++)
                    if (FULL || r * kSortThreads + tid < tile_n) {
                        uint32_t* o = SCATTER ? part_out(a, k, dd[r], dest[r]) : out + dest[r];
                        *o = b32 + (from[r] >> 2);
                    }
                continue;
            }
            const uint8_t* slot = reinterpret_cast<const uint8_t*>(acquire(k));
#pragma unroll
            for (int r = 0; r < ITEMS; r++)
                if (FULL || r * kSortThreads + tid < tile_n) {
                    uint32_t* o = SCATTER ? part_out(a, k, dd[r], dest[r]) : out + dest[r];
                    *o = *reinterpret_cast<const uint32_t*>(slot + from[r]);
                }
            __syncthreads();
            release();
        }
    };

    for (uint32_t tile = a.tile_begin + blockIdx.x; tile < ntiles; tile += G) {
        if (tile < nfull) tile_body(std::true_type{}, tile);
        else tile_body(std::false_type{}, tile);
    }
}

// ---- warp-specialised downsweep (full TMA tiles) -------------------------------------------
// Three roles in one persistent CTA per SM, pipelined across the CTA's tiles:
//   producer warp  issues the 1-D TMA bulk loads of every stream of every tile, in order,
//                  into a ring of R slots (waits on the slot's `empty` barrier);
//   ranker warps   (16, 8 keys per lane) rank tile j's digit word and publish the tile
//                  permutation s_src[j&1] and global bases s_gb[j&1] (barrier `ranked[j&1]`);
//   writer warps   (8) gather every stream of tile j in digit order and store it in
//                  coalesced runs, releasing each slot (`empty`) as they go.
// So while the writers move tile j the rankers already work on tile j+1 and the producer
// keeps the next loads in flight: the store stream never waits for a ranking phase.
// Shapes (TILE keys, RW ranker warps, WW writer warps, CTAs per SM): ranking is
// latency-bound, so rankers get twice the warps of the writers.
//   WsShape<4096, 16, 8, 1>  one CTA of 800 threads per SM (default)
//   WsShape<2048,  8, 4, 2>  two CTAs of 416 threads per SM (CKS_LSD_ITEMS=8)
template <int TILE_, int RW_, int WW_, int MINB_>
struct WsShape {
    static constexpr int TILE = TILE_, RW = RW_, WW = WW_, MINB = MINB_;
    static constexpr int RT = RW * 32, WT = WW * 32;            // ranker / writer threads
    static constexpr int THREADS = (RW + WW + 1) * 32;          // + 1 producer warp
    static constexpr int RI = TILE / RT, WI = TILE / WT;        // keys per ranker lane / slots per writer
    static_assert(RT >= kRadix, "digit phase needs a thread per digit");
};
constexpr uint32_t kDigitSlots = 3;              // digit-word ring (ranked one tile ahead)

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_init_n(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// exclusive scan over the RW*32 ranker threads (named barrier 1)
template <int RW>
__device__ __forceinline__ uint32_t scan_rankers(uint32_t v, uint32_t* s_warp, uint32_t rt) {
    constexpr int kRW = RW, kRT = RW * 32;
    const uint32_t lane = rt & 31, warp = rt >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    named_sync(1, kRT);
    if (warp == 0) {
        uint32_t t = lane < (uint32_t)kRW ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < kRW; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= (uint32_t)o) t += y;
        }
        if (lane < (uint32_t)kRW) s_warp[lane] = t;
    }
    named_sync(1, kRT);
    uint32_t r = (warp ? s_warp[warp - 1] : 0) + x - v;
    named_sync(1, kRT);
    return r;
}

template <class SH, bool SCATTER>
__global__ void __launch_bounds__(SH::THREADS, SH::MINB)
k_downsweep_ws(const LsdPassArgs a, uint32_t nfull) {
    constexpr int TILE = SH::TILE, kRW = SH::RW, kWW = SH::WW, kRT = SH::RT, WI = SH::WI;
    constexpr int HW = kRadix + 8;
    extern __shared__ __align__(128) uint8_t s_dyn[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(s_dyn);                                   // [R][TILE]
    uint32_t* s_hist = ring + (size_t)(kDigitSlots + a.slots) * TILE;                     // [kRW][HW]
    uint16_t* s_src = reinterpret_cast<uint16_t*>(s_hist + kRW * HW);                     // [2][TILE]
    __shared__ uint32_t s_gb[2][kRadix];
    __shared__ uint32_t s_warp[kRW];
    __shared__ __align__(8) uint64_t s_full[kDigitSlots + 16];
    __shared__ __align__(8) uint64_t s_empty[kDigitSlots + 16];
    __shared__ __align__(8) uint64_t s_ranked[2];
    __shared__ __align__(8) uint64_t s_written[2];

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t G = gridDim.x;
    const int np = (int)a.nplanes, dp = a.digit_plane;
    const int S = np + 1;
    const bool implicit_rid = a.in_rid == nullptr;
    const uint32_t L = (uint32_t)(S - (implicit_rid ? 1 : 0));   // loaded streams per tile
    const uint32_t R = a.slots;                                  // data-ring slots
    const uint32_t sel = a.shift >> 3;
    const uint32_t my_tiles = blockIdx.x < nfull ? (nfull - blockIdx.x + G - 1) / G : 0;

    auto src_of = [&](int k) -> const uint32_t* {
        int id = stream_plane(k, dp, np);
        return id >= 0 ? a.in_planes + (uint64_t)id * a.in_pitch : a.in_rid;
    };
    auto dst_of = [&](int k) -> uint32_t* {
        int id = stream_plane(k, dp, np);
        return id >= 0 ? a.out_planes + (uint64_t)id * a.out_pitch : a.out_rid;
    };

    if (tid == 0) {
        for (uint32_t s = 0; s < kDigitSlots + R; s++) { bar_init_n(&s_full[s], 1); bar_init_n(&s_empty[s], kWW); }
        for (int b = 0; b < 2; b++) { bar_init_n(&s_ranked[b], kRW); bar_init_n(&s_written[b], kWW); }
        bar_fence_init();
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    if (blockIdx.x == 0 && tid < kRadix) a.total[tid] = 0;      // digit totals of the next pass's upsweep

    if (warp == kRW + kWW) {
        // ---------------- producer: digit words one tile ahead in their own 3-slot ring
        // (D0, D1, then after the data streams of tile j the digit word of tile j+2), the
        // other streams in order through the data ring
        if (lane == 0) {
            auto issue_digit = [&](uint32_t j) {
                const uint32_t s = j % kDigitSlots;
                if (j >= kDigitSlots) bar_wait(&s_empty[s], ((j / kDigitSlots) - 1) & 1u);
                proxy_fence();
                bulk_load(ring + (size_t)s * TILE, src_of(0) + (uint64_t)(blockIdx.x + j * G) * TILE, TILE * 4,
                          &s_full[s]);
            };
            uint32_t y = 0;                                  // data item counter
            for (uint32_t j = 0; j < my_tiles && j < 2; j++) issue_digit(j);
            for (uint32_t j = 0; j < my_tiles; j++) {
                const uint64_t off = (uint64_t)(blockIdx.x + j * G) * TILE;
                for (uint32_t k = 1; k < L; k++, y++) {
                    const uint32_t s = kDigitSlots + y % R;
                    if (y >= R) bar_wait(&s_empty[s], ((y / R) - 1) & 1u);
                    proxy_fence();
                    bulk_load(ring + (size_t)s * TILE, src_of((int)k) + off, TILE * 4, &s_full[s]);
                }
                if (j + 2 < my_tiles) issue_digit(j + 2);
            }
        }
        return;
    }

    if (warp < kRW) {
        // ---------------- rankers: thread rt < 256 is digit rt in the per-digit phases
        constexpr int RI = SH::RI;                               // keys per ranker lane
        const uint32_t rt = tid;
        const uint32_t wofs = warp * 32 * RI;
        const uint32_t ltm = lt_mask();
        uint32_t* h = s_hist + warp * HW;
        const uint32_t hbase = smem_addr(h);
        // global offsets of digit rt for a tile (upsweep output), loaded one tile ahead so the
        // global-load latency is hidden behind the ranking of the current tile
        uint32_t nc = 0, nt = 0;
        auto fetch = [&](uint32_t j) {
            if (rt < kRadix && j < my_tiles) {
                const uint32_t tile = blockIdx.x + j * G;
                nc = __ldg(a.chunk_tot + (uint64_t)(tile / a.chunk_tiles) * kRadix + rt);
                nt = __ldg(a.tile_off + (uint64_t)tile * kRadix + rt);
            }
        };
        fetch(0);
        for (uint32_t j = 0; j < my_tiles; j++) {
            const uint32_t buf = j & 1;
            const uint32_t goff = nc + nt;
            fetch(j + 1);
            const uint32_t* dslot = ring + (size_t)(j % kDigitSlots) * TILE;
#pragma unroll
            for (int q = lane; q < HW; q += 32) h[q] = 0;
            __syncwarp();
            bar_wait(&s_full[j % kDigitSlots], (j / kDigitSlots) & 1u);
            uint32_t dg[RI], pos[RI];
            {
                uint32_t peers[RI];
#pragma unroll
                for (int i = 0; i < RI; i++) {
                    dg[i] = digit_of(dslot[wofs + i * 32 + lane], sel);
                    peers[i] = match_bits<8>(dg[i]);
                }
                if constexpr (!SCATTER && SH::TILE == 4096) {
#pragma unroll
                    for (int i = 0; i < RI; i++) {
                        // every lane reads its digit's warp-private bin (peers read the same word:
                        // a broadcast), then the digit's leader advances it by the peer count -- a
                        // plain load and store instead of an atomic with return and a shuffle
                        const uint32_t lower = __popc(peers[i] & ltm);
                        const uint32_t o = h[dg[i]];
                        __syncwarp();                            // every read of item i before its writes
                        if (lower == 0) h[dg[i]] = o + (uint32_t)__popc(peers[i]);
                        pos[i] = lower + o;
                        __syncwarp();                            // item i's reservations before item i+1's
                    }
                } else {                                         // (ptxas C7600 on these shapes with the above)
                    uint32_t old[RI];
#pragma unroll
                    for (int i = 0; i < RI; i++) {
                        const uint32_t lower = __popc(peers[i] & ltm);
                        asm volatile("{\n .reg .pred p;\n setp.eq.u32 p, %1, 0;\n mov.u32 %0, 0;\n"
                                     " @p atom.shared.add.u32 %0, [%2], %3;\n}"
                                     : "=r"(old[i]) : "r"(lower), "r"(hbase + dg[i] * 4), "r"((uint32_t)__popc(peers[i]))
                                     : "memory");
                        pos[i] = lower;
                        __syncwarp();                            // item i's reservations before item i+1's
                    }
#pragma unroll
                    for (int i = 0; i < RI; i++) pos[i] += __shfl_sync(0xFFFFFFFFu, old[i], __ffs(peers[i]) - 1);
                }
            }
            named_sync(1, kRT);
            {
                uint32_t c[kRW], total = 0;
                if (rt < kRadix) {
#pragma unroll
                    for (int k = 0; k < kRW; k++) { c[k] = s_hist[k * HW + rt]; total += c[k]; }
                }
                const uint32_t excl = scan_rankers<kRW>(total, s_warp, rt);
                if (rt < kRadix) {
                    uint32_t run = excl;
#pragma unroll
                    for (int k = 0; k < kRW; k++) { s_hist[k * HW + rt] = run; run += c[k]; }
                    if (j >= 2) bar_wait(&s_written[buf], ((j >> 1) - 1) & 1u);   // writers done with tile j-2
                    s_gb[buf][rt] = goff - excl;
                }
            }
            named_sync(1, kRT);
            uint16_t* src = s_src + buf * TILE;
#pragma unroll
            for (int i = 0; i < RI; i++) {
                CKS_DCHECK(pos[i] + h[dg[i]] < (uint32_t)TILE);
                src[(kLsdDebug && (a.debug & 2)) ? wofs + i * 32 + lane : pos[i] + h[dg[i]]] =
                    (uint16_t)((wofs + i * 32 + lane) * 4);
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&s_ranked[buf]);
        }
        return;
    }

    // ---------------- writers: thread wt owns output slots r*WT + wt
    const uint32_t wt = tid - kRT;
    uint32_t y = 0;                                              // data item counter
    for (uint32_t j = 0; j < my_tiles; j++) {
        const uint32_t tile = blockIdx.x + j * G;
        const uint32_t buf = j & 1;
        bar_wait(&s_ranked[buf], (j >> 1) & 1u);
        const uint16_t* src = s_src + buf * TILE;
        uint32_t from[WI], dest[WI];
        uint8_t dd[SCATTER ? WI : 1];                           // SCATTER: the slot's part
#pragma unroll
        for (int r = 0; r < WI; r++) from[r] = src[r * SH::WT + wt];
        {
            const uint32_t slot = j % kDigitSlots;
            bar_wait(&s_full[slot], (j / kDigitSlots) & 1u);
            const uint8_t* sl = reinterpret_cast<const uint8_t*>(ring + (size_t)slot * TILE);
            uint32_t* out = dst_of(0);
#pragma unroll
            for (int r = 0; r < WI; r++) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(sl + from[r]);
                const uint32_t dg = digit_of(w, sel);
                dest[r] = (kLsdDebug && (a.debug & 1)) ? tile * (uint32_t)TILE + r * SH::WT + wt
                                                       : r * SH::WT + wt + s_gb[buf][dg];
                CKS_DCHECK(dest[r] < a.n);
                if (SCATTER) {
                    dd[r] = (uint8_t)dg;
                    dest[r] -= a.bbase[dg];                      // position inside the part
                } else {
                    out[dest[r]] = w;
                }
            }
            __syncwarp();
            if (lane == 0) { bar_arrive(&s_written[buf]); bar_arrive(&s_empty[slot]); }
        }
        for (int k = 1; k < S; k++) {
            uint32_t* out = dst_of(k);
            if (k == S - 1 && implicit_rid) {
                const uint32_t b32 = tile * (uint32_t)TILE + a.rid_add;
#pragma unroll
                for (int r = 0; r < WI; r++) {
                    uint32_t* o = SCATTER ? a.part_dst[(uint32_t)(k - 1) * 256u + dd[SCATTER ? r : 0]] + dest[r]
                                          : out + dest[r];
                    *o = b32 + (from[r] >> 2);
                }
                continue;
            }
            const uint32_t slot = kDigitSlots + y % R;
            bar_wait(&s_full[slot], (y / R) & 1u);
            y++;
            const uint8_t* sl = reinterpret_cast<const uint8_t*>(ring + (size_t)slot * TILE);
#pragma unroll
            for (int r = 0; r < WI; r++) {
                uint32_t* o = SCATTER ? a.part_dst[(uint32_t)(k - 1) * 256u + dd[SCATTER ? r : 0]] + dest[r]
                                      : out + dest[r];
                *o = *reinterpret_cast<const uint32_t*>(sl + from[r]);
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&s_empty[slot]);
        }
    }
}

// ---- launch ---------------------------------------------------------------------------------

// tiles per upsweep CTA: 32 for the largest lists (measured cfg5, 12.2 k tiles: 3.64 -> 3.60 ms),
// 16 below 8192 tiles (cfg3/cfg4 and the refinement's lists lose parallelism with 32)
static uint32_t chunk_for(uint64_t tiles) {
    if (knobs().lsd_chunk > 0) return (uint32_t)knobs().lsd_chunk;
    // three waves of upsweep CTAs over B200's 148 SMs with equal chunks (cfg5: 12,207 tiles ->
    // 28-tile chunks, 436 CTAs; fixed 32-tile chunks left a third wave of 86 CTAs on 148 SMs),
    // at least 8 tiles a chunk
    const uint64_t c = (tiles + 3 * 148 - 1) / (3 * 148);
    return c < 8 ? 8u : (uint32_t)c;
}

uint64_t lsd_tile_keys() { return (uint64_t)kSortThreads * knobs().lsd_items; }

void lsd_sizes(uint64_t n, uint64_t* tiles, uint64_t* chunks) {
    uint64_t t = lsd_tile_keys();
    *tiles = (n + t - 1) / t;
    const uint32_t c = chunk_for(*tiles);
    *chunks = (*tiles + c - 1) / c;
}

template <class... KArgs, class... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int ITEMS, bool SCATTER>
static cudaError_t lsd_pass(LsdPassArgs a, int sms, cudaStream_t st, const LsdAux& aux, int* launches) {
    constexpr int TILE = kSortThreads * ITEMS;
    const uint64_t tiles = (a.n + TILE - 1) / TILE;
    const uint64_t chunks = (tiles + a.chunk_tiles - 1) / a.chunk_tiles;
    // (a.total is zero: the previous pass's downsweep cleared it, or it was just allocated)
    launch_pdl(k_upsweep<ITEMS>, dim3((unsigned)chunks), dim3(kSortThreads), 0, st, a);
    launch_pdl(k_chunk_scan, dim3(kRadix / 32), dim3(1024), 0, st, a, (uint32_t)chunks);
    const int streams = (int)a.nplanes + 1 - (a.in_rid == nullptr ? 1 : 0);
    const uint64_t nfull = a.n / TILE;
    int nl = 2;
    if (knobs().lsd_ws && a.tma && nfull > 0) {
        // warp-specialised kernel over the full tiles, one persistent CTA per SM
        using SH = typename std::conditional<ITEMS == 8, WsShape<2048, 8, 4, 2>, WsShape<4096, 16, 8, 1>>::type;
        static_assert(SH::TILE == TILE, "the upsweep's tile is the downsweep's tile");
        constexpr size_t fixed = (size_t)SH::RW * (kRadix + 8) * 4 + (size_t)2 * TILE * 2;
        const size_t budget = SH::MINB == 2 ? 100u * 1024u : 200u * 1024u;
        const int max_slots = (int)((budget - fixed) / ((size_t)TILE * 4));
        int R = 2 * (streams - 1);                           // data ring: the non-digit streams
        if (R > max_slots - (int)kDigitSlots) R = max_slots - (int)kDigitSlots;
        if (R > 16) R = 16;
        if (R < 1) R = 1;
        LsdPassArgs w = a;
        w.slots = (uint32_t)R;
        const size_t smem = (size_t)(kDigitSlots + R) * TILE * 4 + fixed;
        raise_smem_limit((const void*)k_downsweep_ws<SH, SCATTER>, smem);
        const uint64_t gmax = (uint64_t)sms * SH::MINB;
        const uint64_t grid = nfull < gmax ? nfull : gmax;
        const bool tail = nfull != tiles;
        if (tail && aux.stream) {
            // the partial last tile runs concurrently on the aux stream (its offsets are
            // already known from the upsweep)
            LsdPassArgs tl = a;
            tl.tile_begin = (uint32_t)nfull;
            if ((int)tl.slots > 2 * streams) tl.slots = streams > 0 ? 2 * streams : 1;
            const size_t tsm = (size_t)tl.slots * TILE * 4 + kW * (kRadix + 8) * 4 + (size_t)TILE * 2;
            raise_smem_limit((const void*)k_downsweep<ITEMS, SCATTER>, tsm);
            cudaEventRecord(aux.fork, st);
            cudaStreamWaitEvent(aux.stream, aux.fork, 0);
            k_downsweep<ITEMS, SCATTER><<<1, kSortThreads, tsm, aux.stream>>>(tl);
            cudaEventRecord(aux.join, aux.stream);
            nl++;
        }
        if (aux.ws_begin) cudaEventRecord(aux.ws_begin, st);
        launch_pdl(k_downsweep_ws<SH, SCATTER>, dim3((unsigned)grid), dim3(SH::THREADS), smem, st, w, (uint32_t)nfull);
        if (aux.ws_end) cudaEventRecord(aux.ws_end, st);
        // algorithmic bytes: every loaded stream read once, every stream written once
        if (aux.ws_bytes) *aux.ws_bytes = (double)nfull * TILE * 4.0 * (double)(streams + (int)a.nplanes + 1);
        nl++;
        if (tail && aux.stream) cudaStreamWaitEvent(st, aux.join, 0);
        if (!tail || aux.stream) { *launches = nl; return cudaGetLastError(); }
        a.tile_begin = (uint32_t)nfull;                      // the partial last tile
    }
    if ((int)a.slots > 2 * streams) a.slots = streams > 0 ? 2 * streams : 1;
    size_t smem = (size_t)a.slots * TILE * 4 + kW * (kRadix + 8) * 4 + (size_t)TILE * 2;
    raise_smem_limit((const void*)k_downsweep<ITEMS, SCATTER>, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_downsweep<ITEMS, SCATTER>, kSortThreads, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (grid > tiles - a.tile_begin) grid = tiles - a.tile_begin;
    k_downsweep<ITEMS, SCATTER><<<(unsigned)grid, kSortThreads, smem, st>>>(a);
    nl++;
    *launches = nl;
    return cudaGetLastError();
}

cudaError_t launch_lsd_pass(const LsdPassArgs& args, int sms, cudaStream_t st, const LsdAux& aux, int* launches) {
    *launches = 0;
    if (args.n == 0) return cudaSuccess;
    const Knobs& kn = knobs();
    LsdPassArgs a = args;
    a.slots = (uint32_t)kn.lsd_slots;
    a.chunk_tiles = chunk_for((a.n + lsd_tile_keys() - 1) / lsd_tile_keys());
    a.debug = (uint32_t)kn.lsd_debug;
    a.tma = ((uintptr_t)a.in_planes % 16 == 0) && (a.in_pitch % 4 == 0) &&
            (a.in_rid == nullptr || (uintptr_t)a.in_rid % 16 == 0);
    if (a.part_dst) {
        if (a.in_rid || a.digit_plane != 0) return cudaErrorInvalidValue;   // (the partition pass only)
        return kn.lsd_items == 8 ? lsd_pass<8, true>(a, sms, st, aux, launches)
                                 : lsd_pass<16, true>(a, sms, st, aux, launches);
    }
    return kn.lsd_items == 8 ? lsd_pass<8, false>(a, sms, st, aux, launches)
                             : lsd_pass<16, false>(a, sms, st, aux, launches);
}

}  // namespace cks
