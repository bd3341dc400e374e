// k_ptree.cu -- NEXT-3: the paper's index tree format, built bottom-up from
// the sorted row ids and the D_i (Sec. 4.2; Sec. 5.3).
//
// Node = 256 bytes. Leaf: 24-byte header, 8-byte next pointer, 14 entries of 16 bytes
// {partial key, distinction bit position, key length, record id}; non-leaf: 24-byte
// header, 9 entries of 24 bytes {partial key, distinction bit position, key length, child,
// highest key}. Nodes hold floor(max fanout * fill) entries. The partial key
// is the pk bits of the key following the entry's distinction bit position (reading
// C14), read from the key row (option C(b) of P:491: dereference the record). A non-leaf
// entry's distinction bit position is that of its child's highest key against the previous
// entry's highest key = the minimum D_k over the child's keys (Lemma 1),
// carried up the levels as per-node minima. Byte layout: DESIGN.md R16 / include/cks.h.
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
// extra plane. Table: dec[j*256 + projection] = byte; rc[j] = rank of byte j's first M bit |
// (its M-bit count << 16).
struct PkDec {
    const uint32_t* planes;              // sorted P_M (bit g0 from the MSB of the np planes = its first bit)
    uint64_t pitch;
    uint32_t np, g0, B;
    const uint8_t* dec;                  // byte j's values at dec[off[j] + projection] (2^c_j entries)
    const uint32_t* rc;                  // rank of byte j's first M bit | c_j << 16
    const uint32_t* off;
    uint32_t dec_bytes;                  // table bytes; staged in shared memory per CTA (random
                                         // lane addresses: banks, not L1 wavefronts per line)
    __host__ __device__ uint32_t smem_bytes() const { return dec_bytes ? 8 * B + ((dec_bytes + 15) & ~15u) : 0u; }
    __device__ __forceinline__ PkDec stage(uint8_t* sm) const {
        if (!dec_bytes) return *this;
        uint32_t* src_rc = reinterpret_cast<uint32_t*>(sm);
        uint32_t* src_off = src_rc + B;
        uint8_t* src_dec = reinterpret_cast<uint8_t*>(src_off + B);
        for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) { src_rc[i] = rc[i]; src_off[i] = off[i]; }
        for (uint32_t i = threadIdx.x; i < dec_bytes; i += blockDim.x) src_dec[i] = dec[i];
        __syncthreads();
        PkDec t = *this;
        t.rc = src_rc;
        t.off = src_off;
        t.dec = src_dec;
        return t;
    }
    __device__ __forceinline__ void pre(uint64_t k, uint32_t (&w)[4]) const {
#pragma unroll
        for (int q = 0; q < 4; q++) w[q] = (np <= 4 && q < (int)np) ? __ldg(planes + (uint64_t)q * pitch + k) : 0u;
    }
    __device__ __forceinline__ static uint32_t pick(const uint32_t (&w)[4], int q) {
        return q == 0 ? w[0] : q == 1 ? w[1] : q == 2 ? w[2] : w[3];
    }
    // c (1..8) bits of the planes from bit g (counted from the MSB), right-aligned
    __device__ __forceinline__ uint32_t bits(uint64_t k, uint32_t g, uint32_t c, const uint32_t (&w)[4]) const {
        const int q = (int)np - 1 - (int)(g >> 5);
        const bool reg = np <= 4;
        const uint32_t a = reg ? pick(w, q) : __ldg(planes + (uint64_t)q * pitch + k);
        const uint32_t b = q >= 1 ? (reg ? pick(w, q - 1) : __ldg(planes + (uint64_t)(q - 1) * pitch + k)) : 0u;
        const uint32_t v = (g & 31) ? __funnelshift_l(b, a, g & 31) : a;
        return v >> (32 - c);
    }
    // the plane word q (from the prefetched words when np <= 4)
    __device__ __forceinline__ uint32_t word(uint64_t k, int q, const uint32_t (&w)[4]) const {
        if (q < 0) return 0u;
        return np <= 4 ? pick(w, q) : __ldg(planes + (uint64_t)q * pitch + k);
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk,
                                            const uint32_t (&w)[4]) const {
        if (pk == 0) return 0u;
        const uint32_t p0 = d == CKS_NONE_INTERNAL ? 0u : (uint32_t)d + 1;
        if (p0 >= 8 * B) return 0u;
        const uint32_t j0 = p0 >> 3;
        // the M bits of bytes j0 .. j0+4 are contiguous in P_M: one field of <= 40 bits
        uint32_t cnt[5], tot = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            cnt[i] = j0 + i < B ? rc[j0 + i] >> 16 : 0u;
            tot += cnt[i];
        }
        unsigned long long f = 0;                                  // left-aligned field
        if (tot) {
            const uint32_t g = g0 + (rc[j0] & 0xFFFFu);
            const int q = (int)np - 1 - (int)(g >> 5);
            const uint32_t a = word(k, q, w), b = word(k, q - 1, w), c = word(k, q - 2, w);
            const uint32_t sh = g & 31;
            const unsigned long long ab = ((unsigned long long)a << 32) | b;
            f = sh ? (ab << sh) | (c >> (32 - sh)) : ab;
        }
        unsigned long long win = 0;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const uint32_t c = cnt[i];
            const uint32_t proj = c ? (uint32_t)(f >> (64 - c)) : 0u;
            f <<= c;
            const uint32_t v = j0 + i < B ? (uint32_t)dec[off[j0 + i] + proj] : 0u;
            win = (win << 8) | v;
        }
        const uint32_t out = (uint32_t)(win >> (8 - (p0 & 7)));
        return pk >= 32 ? out : out & ~(0xFFFFFFFFu >> pk);
    }
    __device__ __forceinline__ uint32_t get(uint64_t k, uint32_t rid, uint16_t d, uint32_t pk) const {
        uint32_t w[4];
        pre(k, w);
        return get(k, rid, d, pk, w);
    }
};

// leaves, thread per sorted key k (entry k % per of leaf k / per): the key-row reads of a
// warp are independent (a thread per node would walk its entries serially)
template <class Src>
__global__ void __launch_bounds__(kPtThreads)
k_ptree_leaf_entries(const Src src0, uint64_t n, uint32_t B, const uint32_t* __restrict__ perm,
                     const uint16_t* __restrict__ dbit, uint32_t pk, uint32_t per, uint64_t nleaves,
                     uint8_t* __restrict__ nodes) {
    extern __shared__ __align__(16) uint8_t s_srctab[];
    const Src src = src0.stage(s_srctab);
    constexpr int U = 4;                                          // keys in flight per thread
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < n; k0 += U * T) {
        uint32_t rid[U], pkv[U], pw[U][4];
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
            const uint64_t j = (uint32_t)k / per;                 // (n < 2^32: 32-bit division)
            const uint32_t e = (uint32_t)(k - j * per);
            uint4* nd = reinterpret_cast<uint4*>(nodes + j * 256);
            nd[2 + e] = make_uint4(pkv[u], (uint32_t)d[u] | (B << 16), rid[u], 0u);   // 32 + 16 e
            if (e == 0) {                                         // header, next leaf, unused entries
                const uint64_t k1 = min(k + per, n);
                const unsigned long long next = j + 1 < nleaves ? j + 1 : ~0ull;
                nd[0] = make_uint4((uint32_t)(k1 - k), B, perm[k1 - 1], 0u);
                nd[1] = make_uint4(0u, 0u, (uint32_t)next, (uint32_t)(next >> 32));
                for (uint32_t v = (uint32_t)(k1 - k); v < 14; v++) nd[2 + v] = make_uint4(0, 0, 0, 0);
            }
        }
    }
}

// per-leaf minimum of D_k over its keys (the D-bit of its highest key against the previous
// leaf's, Lemma 1), thread per leaf
__global__ void __launch_bounds__(kPtThreads)
k_ptree_leaf_min(const uint16_t* __restrict__ dbit, uint64_t n, uint32_t per, uint64_t nleaves,
                 uint16_t* __restrict__ rmin) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nleaves; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k0 = j * per, k1 = min(k0 + per, n);
        uint16_t mn = CKS_NONE_INTERNAL;
        for (uint64_t k = k0; k < k1; k++) mn = dbit[k] < mn ? dbit[k] : mn;
        rmin[j] = mn;
    }
}

// level `level` (>= 1): a thread per entry slot (node j, entry e < 9): the child's highest key
// (a random sorted position) is read by many threads at once; the e = 0 thread also writes the
// header and the node's minimum D_k
template <class Src>
__global__ void __launch_bounds__(kPtThreads)
k_ptree_inner(const Src src0, uint64_t n, uint32_t B, const uint32_t* __restrict__ perm,
              uint32_t pk, uint32_t per, uint64_t nbelow, uint64_t cover_below, uint64_t below_off, uint64_t nnodes,
              uint64_t node_off, uint32_t level, const uint16_t* __restrict__ rmin_below, uint16_t* __restrict__ rmin,
              uint8_t* __restrict__ nodes) {
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
        auto hi_of = [&](uint64_t ch) {                              // the child's highest key
            uint64_t hk = (ch + 1) * cover_below;
            if (hk > n) hk = n;
            return hk - 1;
        };
        if (e < cnt) {
            const uint64_t ch = c0 + e, hi = hi_of(ch);
            CKS_DCHECK(hi < n && ch < nbelow);
            const uint32_t rid = __ldg(perm + hi);
            const uint16_t d = ch == 0 ? (uint16_t)CKS_NONE_INTERNAL : __ldg(rmin_below + ch);   // vs the previous entry
            const unsigned long long child = below_off + ch;
            a = make_uint2(src.get(hi, rid, d, pk), (uint32_t)d | (B << 16));
            b = make_uint2((uint32_t)child, (uint32_t)(child >> 32));
            c = make_uint2(rid, 0u);
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
            w[0] = make_uint2(cnt | (level << 16), B);
            w[1] = make_uint2(__ldg(perm + hi_of(c1 - 1)), 0u);
            w[2] = make_uint2(0u, 0u);
            w[30] = make_uint2(0u, 0u);                           // bytes 240..255
            w[31] = make_uint2(0u, 0u);
            rmin[j] = mn;
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
                             const uint64_t* level_offset, uint32_t height, uint8_t* nodes, uint16_t* rmin_a,
                             uint16_t* rmin_b, int sms, cudaStream_t st, int* launches) {
    *launches = 0;
    if (n == 0 || height == 0) return cudaSuccess;
    const uint32_t smem = src.smem_bytes();
    if (smem > 48 * 1024) {
        raise_smem_limit((const void*)k_ptree_leaf_entries<Src>, smem);
        raise_smem_limit((const void*)k_ptree_inner<Src>, smem);
    }
    k_ptree_leaf_entries<Src><<<grid_pt(n, sms), kPtThreads, smem, st>>>(src, n, B, perm, dbit, pk, leaf_per,
                                                                         level_nodes[0], nodes);
    k_ptree_leaf_min<<<grid_pt(level_nodes[0], sms), kPtThreads, 0, st>>>(dbit, n, leaf_per, level_nodes[0], rmin_a);
    *launches += 2;
    uint64_t cover = leaf_per;
    uint16_t* below = rmin_a;
    uint16_t* cur = rmin_b;
    for (uint32_t l = 1; l < height; l++) {
        k_ptree_inner<Src><<<grid_pt(level_nodes[l] * 9, sms), kPtThreads, smem, st>>>(
            src, n, B, perm, pk, inner_per, level_nodes[l - 1], cover, level_offset[l - 1], level_nodes[l],
            level_offset[l], l, below, cur, nodes);
        ++*launches;
        cover *= inner_per;
        uint16_t* t = below;
        below = cur;
        cur = t;
    }
    return cudaGetLastError();
}

cudaError_t launch_ptree_decode(uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit, uint32_t pk,
                                uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                                const uint64_t* level_offset, uint32_t height, uint8_t* nodes, uint16_t* rmin_a,
                                uint16_t* rmin_b, int sms, cudaStream_t st, int* launches, const uint32_t* planes,
                                uint64_t pitch, uint32_t np, uint32_t g0, const uint8_t* dec, const uint32_t* rc,
                                const uint32_t* off, uint32_t dec_bytes) {
    PkDec src{planes, pitch, np, g0, B, dec, rc, off, dec_bytes <= 96u * 1024u ? dec_bytes : 0u};
    return run_ptree(src, n, B, perm, dbit, pk, leaf_per, inner_per, level_nodes, level_offset, height, nodes, rmin_a,
                     rmin_b, sms, st, launches);
}

cudaError_t launch_ptree(const uint8_t* keys, uint64_t n, uint32_t B, const uint32_t* perm, const uint16_t* dbit,
                         uint32_t pk, uint32_t leaf_per, uint32_t inner_per, const uint64_t* level_nodes,
                         const uint64_t* level_offset, uint32_t height, uint8_t* nodes, uint16_t* rmin_a,
                         uint16_t* rmin_b, int sms, cudaStream_t st, int* launches, const PtreeDs* ds) {
    const bool w8 = B % 8 == 0 && ((uintptr_t)keys & 7) == 0;
    if (ds) {
        PkDs src{keys, B, w8, ds->planes, ds->pitch, ds->np, ds->gx, ds->gy, ds->ent};
        return run_ptree(src, n, B, perm, dbit, pk, leaf_per, inner_per, level_nodes, level_offset, height, nodes,
                         rmin_a, rmin_b, sms, st, launches);
    }
    PkRows src{keys, B, w8};
    return run_ptree(src, n, B, perm, dbit, pk, leaf_per, inner_per, level_nodes, level_offset, height, nodes, rmin_a,
                     rmin_b, sms, st, launches);
}

}  // namespace cks
