// cks_plan.cpp -- host-side planning of the bit gather (a2).
//
// For each 32-bit source word with a non-zero selection mask we precompute the five
// "move" masks of the parallel-suffix compress: at step k the selected bits that still
// have an odd number of unselected positions (in units of 2^k) below them move right by
// 2^k. Applying the five steps to (x & mask) leaves the selected bits, in order, in the
// low popcount(mask) bits -- what PEXT does in hardware.
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <utility>

#include "cks_internal.h"

namespace cks {

const Knobs& knobs() {
    static Knobs k;
    static std::once_flag once;
    std::call_once(once, [] {
#if defined(CKS_EXPERIMENTS) && CKS_EXPERIMENTS
        auto env = [](const char* name, int def) {
            const char* e = getenv(name);
            return e ? atoi(e) : def;
        };
        k.lsd_items = env("CKS_LSD_ITEMS", 16);
        if (k.lsd_items != 8 && k.lsd_items != 16) k.lsd_items = 16;
        k.lsd_slots = env("CKS_LSD_SLOTS", 4);
        if (k.lsd_slots < 1) k.lsd_slots = 1;
        if (k.lsd_slots > 16) k.lsd_slots = 16;
        k.lsd_chunk = env("CKS_LSD_CHUNK", 0);
        if (k.lsd_chunk < 0) k.lsd_chunk = 0;
        k.lsd_ws = env("CKS_LSD_WS", 1);
        k.lsd_debug = env("CKS_LSD_DEBUG", 0);
        k.ref_cta = env("CKS_REF_CTA", 2048);
        if (k.ref_cta < 0) k.ref_cta = 0;
        if (k.ref_cta > 2048) k.ref_cta = 2048;
        k.spec_mask = env("CKS_SPEC_MASK", 1);
        k.no_tile_runs = getenv("CKS_NO_TILE_RUNS") != nullptr;
        k.no_kernel_events = getenv("CKS_NO_KERNEL_EVENTS") != nullptr;
        k.refine_log = getenv("CKS_REFINE_LOG") != nullptr;
#endif
    });
    return k;
}

cudaError_t raise_smem_limit(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> limit;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = limit[{dev, kernel}];
    if (bytes <= cur) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

static void move_masks(uint32_t m, uint32_t mv[5]) {
    uint32_t mk = ~m << 1;                 // count unselected positions to the right
    for (int k = 0; k < 5; k++) {
        uint32_t mp = mk ^ (mk << 1);      // parallel suffix (prefix-from-the-right) parity
        mp ^= mp << 2;
        mp ^= mp << 4;
        mp ^= mp << 8;
        mp ^= mp << 16;
        uint32_t v = mp & m;               // bits that move by 2^k at this step
        mv[k] = v;
        m = (m ^ v) | (v >> (1u << k));
        mk &= ~mp;
    }
}

// mirror image: the selected bits end left-aligned (top popcount(m) bits), each step moving
// bits LEFT by 2^k, so a step is x + (x & mv) * (2^(2^k) - 1) -- one multiply-add
static uint32_t rev32(uint32_t x) {
    uint32_t r = 0;
    for (int i = 0; i < 32; i++) r |= ((x >> i) & 1u) << (31 - i);
    return r;
}

void move_masks_left(uint32_t m, uint32_t mv[5]) {
    uint32_t r[5];
    move_masks(rev32(m), r);
    for (int k = 0; k < 5; k++) mv[k] = rev32(r[k]);
}

static void add_step(GatherPlan* plan, uint32_t src, uint32_t mask) {
    GatherStep& s = plan->step[plan->nsteps++];
    s.src = src;
    s.mask = mask;
    move_masks(mask, s.mv);
    s.cnt = (uint32_t)__builtin_popcount(mask);
    plan->out_bits += s.cnt;
}

void plan_compress(const uint8_t* mask, uint32_t B, GatherPlan* plan) {
    memset(plan, 0, sizeof(GatherPlan));
    uint32_t words = (B + 3) / 4;
    for (int w = (int)words - 1; w >= 0; w--) {           // least significant end of P first
        uint32_t mw = 0;
        for (uint32_t b = 0; b < 4; b++) {
            uint32_t j = (uint32_t)w * 4 + b;
            mw = (mw << 8) | (j < B ? mask[j] : 0u);
        }
        if (mw) add_step(plan, (uint32_t)w, mw);
    }
}

void plan_repack(const uint32_t* sub_words, uint32_t np_in, GatherPlan* plan) {
    memset(plan, 0, sizeof(GatherPlan));
    for (uint32_t q = 0; q < np_in; q++)
        if (sub_words[q]) add_step(plan, q, sub_words[q]);
}

}  // namespace cks
