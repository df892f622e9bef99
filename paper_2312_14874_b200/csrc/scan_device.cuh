// scan_device.cuh -- device building blocks of the sm_100a look-back scan.
//
// What the reference does on the CPU, and what each piece here replaces:
//   * simd.py:55-72 vector_inclusive_scan: log2(w) shift-add rounds over w
//     lanes  ->  warp_inclusive_scan: 5 __shfl_up_sync rounds over 32 lanes.
//   * simd.py:75-101 horizontal kernel: block scan + running carry  ->  one
//     tile per CTA, carry obtained by decoupled look-back over predecessor
//     tiles' published aggregates / inclusive prefixes (replaces the
//     engine's barrier + ledger fold, engine.py:314, :329-331).
//   * core.py:40-48 accumulator typing: elements are widened to the acc type
//     (int64 / uint64 / double) before any addition.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ps {

constexpr unsigned FULL = 0xffffffffu;

// ---- accumulator traits ------------------------------------------------------
template <typename T> struct AccOf;
template <> struct AccOf<int32_t> { using type = int64_t; };
template <> struct AccOf<int64_t> { using type = int64_t; };
template <> struct AccOf<uint32_t> { using type = uint64_t; };
template <> struct AccOf<uint64_t> { using type = uint64_t; };
template <> struct AccOf<float> { using type = double; };
template <> struct AccOf<double> { using type = double; };

template <typename A> __device__ __forceinline__ A acc_from_bits(uint64_t b) {
    if constexpr (sizeof(A) == 8 && (A)0.5 != (A)0) return __longlong_as_double((long long)b);
    else return (A)b;
}
template <typename A> __device__ __forceinline__ uint64_t acc_to_bits(A v) {
    if constexpr ((A)0.5 != (A)0) return (uint64_t)__double_as_longlong(v);
    else return (uint64_t)v;
}

// ---- memory-model primitives for the tile descriptors --------------------------
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- 256-bit streaming global access (LDG.E.256 / STG.E.256 on sm_100a) -------
struct alignas(32) V256 {
    uint64_t w[4];
};
__device__ __forceinline__ V256 ldg256_stream(const void *p) {
    V256 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r.w[0]), "=l"(r.w[1]), "=l"(r.w[2]), "=l"(r.w[3])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void stg256_stream(void *p, const V256 &v) {
    asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v.w[0]),
                 "l"(v.w[1]), "l"(v.w[2]), "l"(v.w[3])
                 : "memory");
}

// ---- warp primitives ------------------------------------------------------------
template <typename A> __device__ __forceinline__ A shfl_up(A v, int d) {
    return __shfl_up_sync(FULL, v, d);
}
template <typename A> __device__ __forceinline__ A shfl_xor(A v, int d) {
    return __shfl_xor_sync(FULL, v, d);
}
template <typename A> __device__ __forceinline__ A shfl_down(A v, int d) {
    return __shfl_down_sync(FULL, v, d);
}
template <typename A> __device__ __forceinline__ A shfl_idx(A v, int src) {
    return __shfl_sync(FULL, v, src);
}
template <typename A> __device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}

// Descriptor status values (low 2 bits of the epoch-tagged status word).
constexpr uint64_t ST_A = 1;  // aggregate published
constexpr uint64_t ST_P = 2;  // inclusive prefix published

// One 16-byte descriptor per tile: {(epoch << 2) | status, value bits}.  It is
// written and read with single 128-bit strong accesses (st/ld.relaxed.gpu
// .b128 -> STG/LDG.E.128.STRONG.GPU), so a reader sees status and value
// together without fences: one L2 round trip per look-back window and no
// acquire-induced L1 invalidation.
struct Desc {
    ulonglong2 *d;
};

__device__ __forceinline__ ulonglong2 ld_desc(const ulonglong2 *p) {
    ulonglong2 v;
    asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
                 : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_desc(ulonglong2 *p, uint64_t word, uint64_t value) {
    asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.gpu.global.b128 [%0], t; }"
                 ::"l"(p), "l"(word), "l"(value) : "memory");
}

// In-kernel stall injection (stress tests only; max_ns == 0 disables it and the
// check is one predictable branch per site).  The GPU form of the reference's
// delay_hook (engine.py:91, test_engine.py "stalls must never corrupt the
// double-buffered sums"): a role of one CTA sleeps for a pseudo-random time at
// a hand-off point, chosen by hashing (seed, a, b, site) -- reproducible.
struct Stall {
    uint32_t seed;
    uint32_t prob;    // stall probability per site visit, in 1/1024 units
    uint32_t max_ns;  // stall length drawn from [0, max_ns)
    uint32_t pad;
};
__device__ __forceinline__ uint64_t stall_mix(uint64_t x) {  // splitmix64 finaliser
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ void maybe_stall(const Stall &s, uint64_t a, uint64_t b, uint32_t site) {
    if (s.max_ns == 0) return;
    const uint64_t h = stall_mix(((uint64_t)s.seed << 32) ^ (a * 0x9E3779B97F4A7C15ull) ^
                                 (b * 0xC2B2AE3D27D4EB4Full) ^ ((uint64_t)site << 56));
    if ((uint32_t)(h & 1023) >= s.prob) return;
    uint32_t ns = (uint32_t)((h >> 10) % s.max_ns);
    while (ns > 0) {
        const uint32_t d = ns > 500000u ? 500000u : ns;
        __nanosleep(d);
        ns -= d;
    }
}

// compile-time gate for the persistent kernels: their stress instantiation has
// the stall sites, the production one has none (not even the branch)
template <bool ON>
__device__ __forceinline__ void stall_site(const Stall &s, uint64_t a, uint64_t b, uint32_t site) {
    if constexpr (ON) maybe_stall(s, a, b, site);
}

// ---- cross-GPU mailbox (fused exchange of shard totals over NVLink) ----------------------
// Rank h's reduce publishes its total into slot h of every peer's mailbox
// (ps_publish_total); a scan that needs the carry of ranks 0..n-1 polls its
// own mailbox slots 0..n-1 from inside the kernel (only the warp that folds
// the seed waits; loads and reductions of the first regions proceed
// meanwhile).  A wait that exceeds ~10 s gives up and raises *timeout
// instead of hanging the GPU.
//
// Slot = 16 bytes {flag, value}.  Message passing in the PTX memory model at
// system scope (the writer is another GPU across NVLink / NVSwitch): the
// producer stores the value, then the flag word {epoch << 2 | 1} with
// st.release.sys; the consumer polls the flag with ld.acquire.sys and reads the
// value only after the flag matched.  Release/acquire orders the value before
// the flag across devices; nothing relies on a 16-byte store being single-copy
// atomic over the fabric.
struct Mailbox {
    const ulonglong2 *slots;  // this GPU's mailbox (written by peers)
    int n;                    // slots to wait for (the ranks before this one)
    uint32_t epoch;
    int *timeout;             // device flag, nullable
};
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const unsigned long long *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const unsigned long long *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// producer side: value first, then the flag that makes it visible
__device__ __forceinline__ void mailbox_post(ulonglong2 *slot, uint32_t epoch, uint64_t value) {
    st_relaxed_sys(&slot->y, value);
    st_release_sys(&slot->x, ((uint64_t)epoch << 2) | 1ull);
}
// consumer side: true (and *value) once the slot carries `epoch`
__device__ __forceinline__ bool mailbox_try(const ulonglong2 *slot, uint32_t epoch, uint64_t *value) {
    const uint64_t f = ld_acquire_sys(&slot->x);
    if ((f & ~3ull) != ((uint64_t)epoch << 2) || (f & 3ull) == 0) return false;
    *value = ld_relaxed_sys(&slot->y);
    return true;
}

__device__ __forceinline__ void publish(const Desc &d, int64_t tile, uint32_t epoch, uint64_t st, uint64_t bits) {
    st_desc(d.d + tile, ((uint64_t)epoch << 2) | st, bits);
}

// Warp-parallel decoupled look-back (one full warp).  Returns the exclusive
// prefix of `tile` within its segment [head, ...).  Lane j inspects tile
// base-j; only the lanes in front of the nearest P descriptor have to be
// valid, so older stragglers never stall a tile whose neighbour is done.
// The window slides back 32 tiles when it holds no P.  Tiles before `head`
// read as P with value 0 (the head tile publishes P itself).
#ifdef PS_TRACE
__device__ uint64_t *g_trace;   // development builds only (scripts/trace*.cu)
__device__ uint64_t *g_trace2;
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

template <typename A>
__device__ A lookback(const Desc &d, int64_t tile, int64_t head, uint32_t epoch, int lane) {
    const uint64_t want = (uint64_t)epoch << 2;
#ifdef PS_TRACE
    uint32_t n_windows = 0, n_polls = 0;
#endif
    A excl = (A)0;
    int64_t base = tile - 1;
    while (true) {
        const int64_t p = base - lane;
        const bool live = p >= head;
        ulonglong2 v = live ? ld_desc(d.d + p) : make_ulonglong2(want | ST_P, 0);
        unsigned pmask, need;
        int polls = 0;
        while (true) {
            const bool ok = (v.x & ~3ull) == want && (v.x & 3ull) != 0;
            pmask = __ballot_sync(FULL, ok && (v.x & 3ull) == ST_P);
            const unsigned xmask = __ballot_sync(FULL, !ok);
            need = pmask ? ((pmask & (0u - pmask)) - 1) : FULL;  // lanes before the first P
            if ((xmask & need) == 0) break;
            if (++polls > 8) __nanosleep(polls > 64 ? 128 : 32);
#ifdef PS_TRACE
            ++n_polls;
#endif
            if (!ok && ((need >> lane) & 1)) v = ld_desc(d.d + p);
        }
        const int first_p = pmask ? __ffs(pmask) - 1 : 32;
        A val = (A)0;
        if (live && lane <= first_p) val = acc_from_bits<A>(v.y);
        excl += warp_sum(val);
#ifdef PS_TRACE
        ++n_windows;
        if (pmask && g_trace && lane == 0) g_trace[tile * 8 + 5] = ((uint64_t)n_windows << 32) | n_polls;
#endif
        if (pmask) return excl;
        base -= 32;
    }
}

}  // namespace ps
