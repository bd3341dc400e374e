// k_ptree.cu -- NEXT-3: the paper's index tree format, built bottom-up from
// the sorted row ids and the D_i (Sec. 4.2; Sec. 5.3).
//
// Node = 256 bytes. Leaf: 24-byte header, 8-byte next pointer, 14 entries of 16 bytes
// {partial key, distinction bit position, key length, record id}; non-leaf: 24-byte
// header, 9 entries of 24 bytes {partial key, distinction bit position, key length, child,
// highest key}. Nodes hold floor(max fanout * fill) entries. The partial key
// is the pk bits of the key following the entry's distinction bit position (reading
// C14), from one of the paper's sources (the Pk* structs below): the key row
// (C(b)), the sorted compressed key + reference key + rows for what neither holds (A, B,
// C(b)), or the sorted P_{D+} alone (decode). A non-leaf entry's distinction bit position is
// that of its child's highest key against the previous entry's highest key = the
// minimum D_k over the child's keys (Lemma 1). Each level leaves, per node, a summary
// for the level above (that minimum, the partial key of the node's highest key at it, and the
// highest key's row id), so an inner entry is a sequential read of its child's summary.
// Byte layout: DESIGN.md R16 / include/cks.h.
#include <algorithm>

#include "cks_internal.h"

namespace cks {

namespace {
constexpr int kPtThreads = 128;

// pk (<= 32) bits of the B-byte key starting at bit position p0 (bit 0 = MSB of byte 0),
// left-aligned in a u32; positions past the key read as 0
__device__ __forceinline__ uint32_t key_bits(const uint8_t* key, uint32_t B, uint32_t p0, uint32_t pk) {
    if (pk == 0) return 0u;
    unsigned long long w = 0;                                     // 40-bit window from byte p0/8
    const uint32_t b0 = p0 >> 3;
#pragma unroll
    for (int i = 0; i < 5; i++) {
        const uint32_t j = b0 + i;
        w = (w << 8) | (j < B ? key[j] : 0u);
    }
    const uint32_t v = (uint32_t)(w >> (8 - (p0 & 7)));         // bits p0 .. p0+31 (window bits 0..31)
    return pk >= 32 ? v : v & ~(0xFFFFFFFFu >> pk);
}
__device__ __forceinline__ uint32_t pk_of(const uint8_t* keys, uint32_t B, uint32_t rid, uint16_t d, uint32_t pk) {
    return key_bits(keys + (uint64_t)rid * B, B, d == CKS_NONE_INTERNAL ? 0u : (uint32_t)d + 1, pk);
}
// the same with the 40-bit window read as two aligned 8-byte words (key rows 8-byte aligned,
// B % 8 == 0). A random row costs ~128 bytes of HBM traffic whichever way it is loaded
// (ncu: cached, L2-only, one or two requests; cudaLimitMaxL2FetchGranularity has no effect)
__device__ __forceinline__ unsigned long long bswap64(unsigned long long x) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((unsigned long long)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
}
__device__ __forceinline__ uint32_t pk_of8(const uint8_t* keys, uint32_t B, uint32_t rid, uint16_t d, uint32_t pk) {
    if (pk == 0) return 0u;
    const uint32_t p0 = d == CKS_NONE_INTERNAL ? 0u : (uint32_t)d + 1;
    const uint32_t w0 = (p0 >> 6);                                  // 8-byte word holding bit p0
    if (8 * w0 >= B) return 0u;
    const unsigned long long* row = reinterpret_cast<const unsigned long long*>(keys + (uint64_t)rid * B);
    const unsigned long long a = bswap64(__ldg(row + w0));           // big-endian: bit 0 = MSB
    const unsigned long long b = 8 * (w0 + 1) < B ? bswap64(__ldg(row + w0 + 1)) : 0ull;
    const uint32_t sh = p0 & 63;
    const unsigned long long v = sh ? (a << sh) | (b >> (64 - sh)) : a;
    const uint32_t top = (uint32_t)(v >> 32);
    return pk >= 32 ? top : top & ~(0xFFFFFFFFu >> pk);
}
}  // namespace

// Where a partial key's bits come from.
//   PkRows  every bit from the key row (C(b): dereference the record) -- any caller.
//   PkDs    A: from the sorted compressed planes the build produced (positions of `xmask`,
//           compressed index = rank in xmask), B: invariant positions (0 in the variant bitmap)
//           from the reference key, C(b): the remaining variant positions from the key row,
//           read only when the entry's window holds one.
struct PkRows {
    const uint8_t* keys;
    uint32_t B;
    bool w8;
    __host__ __device__ uint32_t smem_bytes() const { return 0u; }
    __device__ __forceinline__ PkRows stage(uint8_t*) const { return *this; }
    __device__ __forceinline__ void pre(uint64_t, uint32_t (&)[4]) const {}
    __device__ __forceinline__ uint32_t get(uint64_t /*k*/, uint32_t rid, uint16_t d, uint32_t pk,
                                            const uint32_t (&)[4]) const {
        return w8 ? pk_of8(keys, B, rid, d, pk) : pk_of(keys, B, rid, d, pk);
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk) const {
        const uint32_t w[4] = {0, 0, 0, 0};
        return get(k, rid, d, pk, w);
    }
};

struct PkDs {
    const uint8_t* keys;                 // rows for C(b) (may be NULL when V is inside X u Y)
    uint32_t B;
    bool w8;
    const uint32_t* planes;              // sorted compressed planes, plane np-1 most significant
    uint64_t pitch;
    uint32_t np;
    uint32_t gx, gy;                     // bit (from the MSB of the np planes) of segment X's / Y's
                                         // first compressed bit; X then Y (Y may be empty)
    const PtreeEnt* ent;                 // per window start p0 = D + 1 (0 for none), 8B + 1 entries
    __host__ __device__ uint32_t smem_bytes() const { return 0u; }
    __device__ __forceinline__ PkDs stage(uint8_t*) const { return *this; }
    // the plane words of sorted position k loaded ahead (np <= 4): the loads do not wait for the
    // per-window table lookup
    __device__ __forceinline__ void pre(uint64_t k, uint32_t (&w)[4]) const {
#pragma unroll
        for (int q = 0; q < 4; q++) w[q] = (np <= 4 && q < (int)np) ? __ldg(planes + (uint64_t)q * pitch + k) : 0u;
    }
    __device__ __forceinline__ static uint32_t pick(const uint32_t (&w)[4], int q) {
        return q == 0 ? w[0] : q == 1 ? w[1] : q == 2 ? w[2] : w[3];
    }
    // c (<= 32) bits of the planes from bit g (counted from the MSB), left-aligned
    __device__ __forceinline__ uint32_t field(uint64_t k, uint32_t g, uint32_t c, const uint32_t (&w)[4]) const {
        const int q = (int)np - 1 - (int)(g >> 5);
        CKS_DCHECK(q >= 0 && q < (int)np && k < pitch);
        const bool reg = np <= 4;
        const uint32_t a = reg ? pick(w, q) : __ldg(planes + (uint64_t)q * pitch + k);
        const uint32_t b = q >= 1 ? (reg ? pick(w, q - 1) : __ldg(planes + (uint64_t)(q - 1) * pitch + k)) : 0u;
        const uint32_t v = (g & 31) ? __funnelshift_l(b, a, g & 31) : a;
        return c >= 32 ? v : v & ~(0xFFFFFFFFu >> c);
    }
    // the left-aligned field's bits deposited, in order, at the set bits of m (software PDEP)
    __device__ __forceinline__ static uint32_t deposit(uint32_t f, uint32_t m) {
        uint32_t out = 0;
        while (m) {
            const uint32_t hb = 0x80000000u >> __clz(m);
            if (f & 0x80000000u) out |= hb;
            f <<= 1;
            m &= ~hb;
        }
        return out;
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk) const {
        uint32_t w[4];
        pre(k, w);
        return get(k, rid, d, pk, w);
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk,
                                            const uint32_t (&w)[4]) const {
        const uint32_t p0 = d == CKS_NONE_INTERNAL ? 0u : min((uint32_t)d + 1, 8 * B);
        const uint2 e0 = __ldg(reinterpret_cast<const uint2*>(ent + p0));
        const uint2 e1 = __ldg(reinterpret_cast<const uint2*>(ent + p0) + 1);
        const uint2 e2 = __ldg(reinterpret_cast<const uint2*>(ent + p0) + 2);
        // e0 = (wx, wy), e1 = (ref bits, wc), e2 = (rank x, rank y) -- all within the pk bits
        uint32_t out = e1.x;                                       // B: invariant bits
        if (e0.x) out |= deposit(field(k, gx + e2.x, (uint32_t)__popc(e0.x), w), e0.x);   // A
        if (e0.y) out |= deposit(field(k, gy + e2.y, (uint32_t)__popc(e0.y), w), e0.y);
        if (e1.y) out |= (w8 ? pk_of8(keys, B, rid, d, pk) : pk_of(keys, B, rid, d, pk)) & e1.y;   // C(b)
        return out;
    }
};

// Source A extended ("decode"): with M = D+ (a first build) the compressed key determines the
// whole key -- D+ at byte j is the D-bit set of the byte values occurring there, so their M-bit
// projections are distinct (Theorem 2 on the byte column, reading R2) and a per-byte table maps
// a projection back to the byte. Every partial-key bit comes from the sorted P_M: no rows, no
// extra plane. A window start in byte j0 needs bytes j0 .. j0+4, whose M bits are contiguous in
// P_M: one <= 40-bit field; the per-j0 entry (cks_internal.h) packs where it starts, how it
// splits into bytes and where each byte's values sit, so a key costs one 16-byte table read,
// the field's plane words and five byte lookups. Tables staged in shared memory per CTA.
template <int NP>                        // planes: 1..4 (words prefetched in registers) or 0 (any np)
struct PkDec {
    const uint32_t* planes;              // sorted P_M, plane np-1 most significant
    uint64_t pitch;
    uint32_t np, B;
    const uint4* pj;                     // [B] per window byte
    const uint8_t* dec;                  // byte values by (offset + projection); last byte 0
    uint32_t dec_bytes;
    __host__ __device__ uint32_t smem_bytes() const { return 16 * B + ((dec_bytes + 15) & ~15u); }
    __device__ __forceinline__ PkDec stage(uint8_t* sm) const {
        uint4* s_pj = reinterpret_cast<uint4*>(sm);
        uint8_t* s_dec = sm + 16 * B;
        for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) s_pj[i] = pj[i];
        for (uint32_t i = threadIdx.x; i < dec_bytes; i += blockDim.x) s_dec[i] = dec[i];
        __syncthreads();
        PkDec t = *this;
        t.pj = s_pj;
        t.dec = s_dec;
        return t;
    }
    __device__ __forceinline__ void pre(uint64_t k, uint32_t (&w)[4]) const {
        const uint32_t* p = planes + k;
#pragma unroll
        for (int q = 0; q < 4; q++) w[q] = q < NP ? __ldg(p + (uint64_t)q * pitch) : 0u;
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk,
                                            const uint32_t (&w)[4]) const {
        if (pk == 0) return 0u;
        const uint32_t p0 = d == CKS_NONE_INTERNAL ? 0u : (uint32_t)d + 1;
        if (p0 >= 8 * B) return 0u;
        const uint4 e = pj[p0 >> 3];
        const uint32_t g = e.x & 0xFFFu, sh = g & 31, top = g >> 5;   // word top from the MSB
        uint32_t a, b, c;                                              // words top, top+1, top+2
        if (NP > 0) {
            a = w[NP > 0 ? NP - 1 : 0];
            b = NP > 1 ? w[NP > 1 ? NP - 2 : 0] : 0u;
            c = NP > 2 ? w[NP > 2 ? NP - 3 : 0] : 0u;
#pragma unroll
            for (int s = 1; s < NP; s++)                               // shift the window down
                if (top >= (uint32_t)s) {
                    a = b;
                    b = c;
                    c = NP - 3 - s >= 0 ? w[NP - 3 - s >= 0 ? NP - 3 - s : 0] : 0u;
                }
        } else {
            const int q = (int)np - 1 - (int)top;
            const uint32_t* p = planes + k;
            a = q >= 0 ? __ldg(p + (uint64_t)q * pitch) : 0u;            // (np = 0: an empty mask)
            b = q >= 1 ? __ldg(p + (uint64_t)(q - 1) * pitch) : 0u;
            c = q >= 2 ? __ldg(p + (uint64_t)(q - 2) * pitch) : 0u;
        }
        uint32_t fh = __funnelshift_l(b, a, sh), fl = __funnelshift_l(c, b, sh);   // bits g .. g+63
        const uint32_t off[5] = {e.y & 0xFFFFu, e.y >> 16, e.z & 0xFFFFu, e.z >> 16, e.w};
        uint32_t cn = e.x >> 12, win = 0, last = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint32_t ci = cn & 15u;
            cn >>= 4;
            const uint32_t proj = __funnelshift_rc(fh, 0u, 32 - ci);     // top ci bits (0 for ci = 0)
            fh = __funnelshift_l(fl, fh, ci);
            fl <<= ci;
            const uint32_t v = dec[off[i] + proj];
            if (i < 4) win = (win << 8) | v;
            else last = v;
        }
        const uint32_t out = __funnelshift_l(last << 24, win, p0 & 7);   // bits p0 .. p0+31
        return pk >= 32 ? out : out & ~(0xFFFFFFFFu >> pk);
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk) const {
        uint32_t w[4];
        pre(k, w);
        return get(k, rid, d, pk, w);
    }
};

// leaves, thread per sorted key k (entry k % per of leaf k / per): the key-row reads of a
// warp are independent (a thread per node would walk its entries serially). The unused entry
// slots of a leaf are zeroed by its first threads (slot cnt + e); the thread of a leaf's highest
// key keeps that key's plane words and row id (hk, hr) for the level above.
template <class Src>
__global__ void __launch_bounds__(kPtThreads)
k_ptree_leaf_entries(const Src src0, uint64_t n, uint32_t B, const uint32_t* __restrict__ perm,
                     const uint16_t* __restrict__ dbit, uint32_t pk, uint32_t per, uint64_t nleaves,
                     uint8_t* __restrict__ nodes, uint4* __restrict__ hk, uint32_t* __restrict__ hr, uint32_t per_magic) {
    extern __shared__ __align__(16) uint8_t s_srctab[];
    const Src src = src0.stage(s_srctab);
    constexpr int U = 4;                                          // keys in flight per thread
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < n; k0 += U * T) {
        uint32_t rid[U], pkv[U], pw[U][4] = {};
        uint16_t d[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t k = k0 + u * T;
            rid[u] = k < n ? perm[k] : 0u;
            d[u] = k < n ? dbit[k] : (uint16_t)CKS_NONE_INTERNAL;
            if (k < n) src.pre(k, pw[u]);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            pkv[u] = k0 + u * T < n ? src.get(k0 + u * T, rid[u], d[u], pk, pw[u]) : 0u;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t k = k0 + u * T;
            if (k >= n) break;
            // j = k / per (n < 2^32): per_magic = floor(2^32 / per) is at most one short
            uint32_t jj = __umulhi((uint32_t)k, per_magic), e = (uint32_t)k - jj * per;
            if (e >= per) {
                jj++;
                e -= per;
            }
            const uint64_t j = jj;
            const uint64_t k1 = min(j * per + per, n);
            const uint32_t cnt = (uint32_t)(k1 - j * per);
            uint4* nd = reinterpret_cast<uint4*>(nodes + j * 256);
            nd[2 + e] = make_uint4(pkv[u], (uint32_t)d[u] | (B << 16), rid[u], 0u);   // 32 + 16 e
            for (uint32_t v = cnt + e; v < 14; v += cnt) nd[2 + v] = make_uint4(0, 0, 0, 0);
            if (e == 0) {                                         // header, next leaf
                const unsigned long long next = j + 1 < nleaves ? j + 1 : ~0ull;
                nd[0] = make_uint4(cnt, B, perm[k1 - 1], 0u);
                nd[1] = make_uint4(0u, 0u, (uint32_t)next, (uint32_t)(next >> 32));
            }
            if (hk && k == k1 - 1) {
                hk[j] = make_uint4(pw[u][0], pw[u][1], pw[u][2], pw[u][3]);
                hr[j] = rid[u];
            }
        }
    }
}

// per leaf: the minimum of D_k over its keys (the D-bit of its highest key against the previous
// leaf's, Lemma 1) and the partial key of its highest key at that position -- the leaf's entry
// one level up (the first leaf's at position 0). Thread per leaf, from hk/hr.
template <class Src>
__global__ void __launch_bounds__(kPtThreads)
k_ptree_leaf_sum(const Src src0, const uint16_t* __restrict__ dbit, uint64_t n, uint32_t pk, uint32_t per,
                 uint64_t nleaves, const uint4* __restrict__ hk, const uint32_t* __restrict__ hr,
                 uint16_t* __restrict__ rmin, uint2* __restrict__ sum) {
    extern __shared__ __align__(16) uint8_t s_srctab[];
    const Src src = src0.stage(s_srctab);
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nleaves; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k0 = j * per, k1 = min(k0 + per, n);
        uint16_t mn = CKS_NONE_INTERNAL;
        for (uint64_t k = k0; k < k1; k++) mn = dbit[k] < mn ? dbit[k] : mn;
        const uint4 h = hk[j];
        const uint32_t w[4] = {h.x, h.y, h.z, h.w};
        const uint32_t rid = hr[j];
        rmin[j] = mn;
        sum[j] = make_uint2(src.get(k1 - 1, rid, j == 0 ? (uint16_t)CKS_NONE_INTERNAL : mn, pk, w), rid);
    }
}

// level `level` (>= 1): a thread per entry slot (node j, entry e < 9), the entry read from the
// child's summary; the e = 0 thread writes the header and the node's minimum D_k and, below the
// root, the node's own summary (its highest key's partial key at that minimum: one random read
// of that key's planes per node)
template <class Src>
__global__ void __launch_bounds__(kPtThreads)
k_ptree_inner(const Src src0, uint64_t n, uint32_t B, uint32_t pk, uint32_t per, uint64_t nbelow,
              uint64_t cover_below, uint64_t below_off, uint64_t nnodes, uint64_t node_off, uint32_t level,
              const uint16_t* __restrict__ rmin_below, const uint2* __restrict__ sum_below, uint16_t* __restrict__ rmin,
              uint2* __restrict__ sum, uint8_t* __restrict__ nodes, const uint4* __restrict__ hk_below) {
    extern __shared__ __align__(16) uint8_t s_srctab[];
    const Src src = src0.stage(s_srctab);
    const uint64_t slots = nnodes * 9;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < slots; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = t < (1ull << 32) ? (uint64_t)((uint32_t)t / 9u) : t / 9;
        const uint32_t e = (uint32_t)(t - j * 9);
        uint2* w = reinterpret_cast<uint2*>(nodes + (node_off + j) * 256);
        const uint64_t c0 = j * per, c1 = min(c0 + per, nbelow);
        const uint32_t cnt = (uint32_t)(c1 - c0);
        uint2 a = make_uint2(0, 0), b = make_uint2(0, 0), c = make_uint2(0, 0);
        if (e < cnt) {
            const uint64_t ch = c0 + e;
            CKS_DCHECK(ch < nbelow);
            const uint2 s = __ldg(sum_below + ch);
            const uint16_t d = ch == 0 ? (uint16_t)CKS_NONE_INTERNAL : __ldg(rmin_below + ch);   // vs the previous entry
            const unsigned long long child = below_off + ch;
            a = make_uint2(s.x, (uint32_t)d | (B << 16));
            b = make_uint2((uint32_t)child, (uint32_t)(child >> 32));
            c = make_uint2(s.y, 0u);
        }
        w[3 + 3 * e] = a;                                         // 24 + 24 e
        w[4 + 3 * e] = b;
        w[5 + 3 * e] = c;
        if (e == 0) {
            uint16_t mn = CKS_NONE_INTERNAL;
            for (uint64_t ch = c0; ch < c1; ch++) {
                const uint16_t rm = __ldg(rmin_below + ch);
                mn = rm < mn ? rm : mn;
            }
            const uint32_t rid_hi = __ldg(&sum_below[c1 - 1].y);  // the node's highest key = its last child's
            w[0] = make_uint2(cnt | (level << 16), B);
            w[1] = make_uint2(rid_hi, 0u);
            w[2] = make_uint2(0u, 0u);
            w[30] = make_uint2(0u, 0u);                           // bytes 240..255
            w[31] = make_uint2(0u, 0u);
            rmin[j] = mn;
            if (sum) {
                uint64_t hi = c1 * cover_below;
                if (hi > n) hi = n;
                uint32_t wv[4];
                if (hk_below) {                                   // level 1: the last leaf kept its words
                    const uint4 h = __ldg(hk_below + c1 - 1);
                    wv[0] = h.x;
                    wv[1] = h.y;
                    wv[2] = h.z;
                    wv[3] = h.w;
                } else {
                    src.pre(hi - 1, wv);
                }
                sum[j] = make_uint2(src.get(hi - 1, rid_hi, j == 0 ? (uint16_t)CKS_NONE_INTERNAL : mn, pk, wv), rid_hi);
            }
        }
    }
}

static unsigned grid_pt(uint64_t work, int sms) {
    uint64_t g = (work + kPtThreads - 1) / kPtThreads;
    const uint64_t cap = (uint64_t)sms * 32;
    if (g > cap) g = cap;
    return (unsigned)(g ? g : 1);
}

template <class Src>
static cudaError_t run_ptree(const Src& src, uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit,
                             uint32_t pk, uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                             const uint64_t* level_offset, uint32_t height, uint8_t* nodes, const PtreeWs& ws, int sms,
                             cudaStream_t st, int* launches) {
    *launches = 0;
    if (n == 0 || height == 0) return cudaSuccess;
    const uint32_t smem = src.smem_bytes();
    if (smem > 48 * 1024) {
        raise_smem_limit((const void*)k_ptree_leaf_entries<Src>, smem);
        raise_smem_limit((const void*)k_ptree_leaf_sum<Src>, smem);
        raise_smem_limit((const void*)k_ptree_inner<Src>, smem);
    }
    const bool up = height > 1;
    k_ptree_leaf_entries<Src><<<grid_pt(n, sms), kPtThreads, smem, st>>>(
        src, n, B, perm, dbit, pk, leaf_per, level_nodes[0], nodes, up ? ws.hk : nullptr, ws.hr,
        (uint32_t)std::min<uint64_t>((1ull << 32) / leaf_per, 0xFFFFFFFFull));
    ++*launches;
    if (!up) return cudaGetLastError();
    k_ptree_leaf_sum<Src><<<grid_pt(level_nodes[0], sms), kPtThreads, smem, st>>>(
        src, dbit, n, pk, leaf_per, level_nodes[0], ws.hk, ws.hr, ws.rmin[0], ws.sum[0]);
    ++*launches;
    uint64_t cover = leaf_per;
    int cur = 0;
    for (uint32_t l = 1; l < height; l++) {
        k_ptree_inner<Src><<<grid_pt(level_nodes[l] * 9, sms), kPtThreads, smem, st>>>(
            src, n, B, pk, inner_per, level_nodes[l - 1], cover, level_offset[l - 1], level_nodes[l], level_offset[l],
            l, ws.rmin[cur], ws.sum[cur], ws.rmin[cur ^ 1], l + 1 < height ? ws.sum[cur ^ 1] : nullptr, nodes,
            l == 1 ? ws.hk : nullptr);
        ++*launches;
        cover *= inner_per;
        cur ^= 1;
    }
    return cudaGetLastError();
}

cudaError_t launch_ptree_decode(uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit, uint32_t pk,
                                uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                                const uint64_t* level_offset, uint32_t height, uint8_t* nodes, const PtreeWs& ws,
                                int sms, cudaStream_t st, int* launches, const uint32_t* planes, uint64_t pitch,
                                uint32_t np, const uint4* pj, const uint8_t* dec, uint32_t dec_bytes) {
#define CKS_PTREE_DEC(NP)                                                                                     \
    run_ptree(PkDec<NP>{planes, pitch, np, B, pj, dec, dec_bytes}, n, B, perm, dbit, pk, leaf_per, inner_per,      \
              level_nodes, level_offset, height, nodes, ws, sms, st, launches)
    switch (np) {
        case 1: return CKS_PTREE_DEC(1);
        case 2: return CKS_PTREE_DEC(2);
        case 3: return CKS_PTREE_DEC(3);
        case 4: return CKS_PTREE_DEC(4);
        default: return CKS_PTREE_DEC(0);
    }
#undef CKS_PTREE_DEC
}

cudaError_t launch_ptree(const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit,
                         uint32_t pk, uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                         const uint64_t* level_offset, uint32_t height, uint8_t* nodes, const PtreeWs& ws, int sms,
                         cudaStream_t st, int* launches, const PtreeDs* ds) {
    const bool w8 = B % 8 == 0 && ((uintptr_t)keys & 7) == 0;
    if (ds) {
        PkDs src{keys, B, w8, ds->planes, ds->pitch, ds->np, ds->gx, ds->gy, ds->ent};
        return run_ptree(src, n, B, perm, dbit, pk, leaf_per, inner_per, level_nodes, level_offset, height, nodes, ws,
                         sms, st, launches);
    }
    PkRows src{keys, B, w8};
    return run_ptree(src, n, B, perm, dbit, pk, leaf_per, inner_per, level_nodes, level_offset, height, nodes, ws, sms,
                     st, launches);
}

}  // namespace cks
