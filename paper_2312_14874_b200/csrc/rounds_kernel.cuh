// rounds_kernel.cuh -- the paper's cache-partitioned accumulate-scan, B200 form.
//
// Reference structure (engine.py:278-344, plan.py:211-241, PAPER.md s2.2):
// the input is walked in cache-sized regions ("iterations"); in each region
// every worker first ACCUMULATES its partition (read-only pass 1), the
// partition totals go through a double-buffered ledger with one barrier per
// iteration, then every worker SCANS its partition seeded with the ledger
// prefix (pass 2) while the data is still in cache, and pass 2 of iteration k
// overlaps pass 1 of iteration k+1 (engine.py:1-22, SchemeId
// ACCUMULATE_SCAN_EQUAL).
//
// Here the cache is the 126 MB L2 and the workers are G persistent CTAs
// (cooperative launch, so all are co-resident):
//   * region r = `round_elems` positions, CTA c owns the contiguous portion
//     [r*R + c*P, r*R + (c+1)*P) with P = R / G;
//   * pass 1: 256-bit streaming loads, sum in the accumulator type, publish
//     the portion total as one 16-byte epoch-tagged descriptor (r, c);
//     loads carry an L2 evict_last policy so the region stays resident;
//   * ledger + barrier: warp 0 gathers the G totals of region r (one 128-bit
//     load per descriptor, all issued at once), the prefix of the CTAs before
//     c and the region total are folded in a fixed order -- every CTA computes
//     the identical region total, so float carries agree bit for bit;
//   * pass 2: TMA bulk copies (cp.async.bulk + mbarrier ring) pull the portion
//     back from L2 (evict_first) sub-tile by sub-tile into shared memory; each
//     sub-tile is scanned in registers (warp shuffles + one CTA barrier) with
//     a running carry and stored with 256-bit streaming stores;
//   * pass 1 of region r+1 is issued before the ledger wait of region r, so
//     the barrier latency hides behind HBM reads (the reference's overlap).
// HBM traffic stays one read + one write per element: the second read of
// every element is an L2 hit.
#pragma once

#include "scan_kernels.cuh"

namespace ps {

// ---- mbarrier / bulk-copy primitives (sm_90+; UBLKCP / SYNCS in SASS) ----------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
#ifndef PS_MBAR_HINT
#define PS_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if PS_MBAR_HINT
    // with a suspend-time hint a waiting warp sleeps up to the hint inside try_wait
    // instead of re-issuing it, leaving the issue slots to the working warps
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity), "r"((uint32_t)PS_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
#endif
}
// mbarrier wait that suspends the warp in try_wait (up to `hint_ns` per attempt)
// instead of re-issuing it: for kernels whose spinning roles would otherwise
// take the issue slots of the working ones
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t hint_ns = 1000000u) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}
// mbarrier wait with a nanosleep back-off between probes (waiting roles leave the issue slots alone)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity, uint32_t ns = 128u) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @p bra DONE_%=;\n"
        " nanosleep.u32 %2;\n"
        " bra WAIT_%=;\n DONE_%=:\n}" ::"r"(smem_addr(bar)),
        "r"(parity), "r"(ns)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ V256 ldg256_policy(const void *p, uint64_t pol) {
    V256 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(r.w[0]), "=l"(r.w[1]), "=l"(r.w[2]), "=l"(r.w[3])
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void stg256_policy(void *p, const V256 &v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "l"(v.w[0]),
                 "l"(v.w[1]), "l"(v.w[2]), "l"(v.w[3]), "l"(pol)
                 : "memory");
}
// 32 bytes per lane from shared memory as two 16-byte loads.  Lanes sit 32 bytes
// apart, so loading every lane's first half and then its second half makes
// lanes l and l+4 of a quarter-warp hit the same bank group (2-way conflict,
// a third of all shared wavefronts in the f32 profile).  With SWZ, lanes of odd
// quarters (address bit 7) load their halves in the opposite order: each
// 16-byte load instruction then covers all eight bank groups per quarter-warp
// -- conflict-free -- and a register swap restores the order.  Measured on the
// stream kernel (scripts/stream_variants.cu): +3.8 % for 64-bit data, -1 % for
// float32 (whose scanner is issue-bound and pays for the swap), so it is a
// per-kernel choice.
template <bool SWZ = false>
__device__ __forceinline__ V256 lds256(const void *p) {
    V256 r;
    const uint32_t a = smem_addr(p);
    if constexpr (SWZ) {
        const uint32_t sw = (a >> 7) & 1u;
        uint64_t x0, x1, y0, y1;
        asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(x0), "=l"(x1) : "r"(a + (sw << 4)));
        asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(y0), "=l"(y1) : "r"(a + ((sw ^ 1u) << 4)));
        r.w[0] = sw ? y0 : x0;
        r.w[1] = sw ? y1 : x1;
        r.w[2] = sw ? x0 : y0;
        r.w[3] = sw ? x1 : y1;
    } else {
        asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(r.w[0]), "=l"(r.w[1]) : "r"(a));
        asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(r.w[2]), "=l"(r.w[3]) : "r"(a + 16));
    }
    return r;
}

struct RoundArgs {
    Stall stall;      // stress tests: stall injection at every role hand-off
    Mailbox mail;     // seed += totals published by the ranks before this one
    const void *in;   // aligned base: position p <-> element p - lead
    void *out;
    int64_t lo, hi;   // valid positions [lo, hi) (lo = lead, hi = lead + n)
    int64_t portion;      // P: per-CTA positions of a full region (multiple of SUB << ramp)
    int64_t rounds;       // regions actually launched (ramp-up + full + ramp-down, trailing empties dropped)
    int64_t full_regions; // F full-size regions between the ramps
    int ramp;             // K: regions 0..K-1 have portions P/2^K .. P/2, the K after the full ones P/2 .. P/2^K
    uint64_t seed_bits;
    const void *seed_terms;
    int64_t n_seed_terms;
    void *total;          // acc-typed, nullable
    ulonglong2 *desc;     // rounds * G portion-total descriptors
    uint32_t epoch;
    int exclusive;
    int lead_regions;     // reducer runs up to this many regions ahead of the scanners
    int l2_prefetch;      // issue a bulk L2 prefetch of each reducer portion
};

// Region r of the ramped schedule: first position and per-CTA portion.  Small
// regions at both ends shorten the pipeline fill (first region reduced alone)
// and drain (last region scanned alone).
__host__ __device__ __forceinline__ int64_t ramp_part(int64_t P, int64_t sub, int k) {  // P/2^k, >= sub
    const int64_t q = (P >> k) / sub * sub;
    return q < sub ? sub : q;
}
__host__ __device__ __forceinline__ void region_geom(int64_t portion, int ramp, int64_t full, int64_t G, int64_t sub,
                                                     int64_t r, int64_t &start, int64_t &part) {
    const int64_t P = portion;
    int64_t up = 0;  // ramp-up regions: P/2^ramp .. P/2 (multiples of sub)
    for (int q = 0; q < ramp && q < r; ++q) up += ramp_part(P, sub, ramp - q);
    if (r < ramp) {
        part = ramp_part(P, sub, (int)(ramp - r));
        start = G * up;
        return;
    }
    if (r < ramp + full) {
        part = P;
        start = G * (up + (r - ramp) * P);
        return;
    }
    const int64_t i = r - ramp - full;  // ramp-down: P/2, P/4, ...
    int64_t down = 0;
    for (int q = 0; q < i; ++q) down += ramp_part(P, sub, q + 1);
    part = ramp_part(P, sub, (int)(i + 1));
    start = G * (up + full * P + down);
}

__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Ledger gather (one warp): waits for the G portion totals of one region and
// returns the sum of those before CTA c (sb) and of all of them (sa).  Every
// lane keeps 8 descriptors in flight per polling round, G may be up to 1024;
// the summation order is the same on every CTA, so `sa` is bit-identical
// everywhere (float carries stay consistent across CTAs).
template <typename A>
__device__ __forceinline__ void gather_totals(const ulonglong2 *desc, int G, int c, uint64_t want, int lane, A &sb,
                                              A &sa) {
    constexpr int PER = 8;
    sb = (A)0;
    sa = (A)0;
    for (int g0 = 0; g0 < G; g0 += 32 * PER) {
        ulonglong2 d[PER];
        unsigned pending = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = g0 + lane + 32 * i;
            if (j < G) {
                d[i] = ld_desc(desc + j);
                pending |= 1u << i;
            }
        }
        while (true) {
#pragma unroll
            for (int i = 0; i < PER; ++i)
                if (((pending >> i) & 1) && (d[i].x & ~3ull) == want && (d[i].x & 3ull) != 0) pending &= ~(1u << i);
            if (!__any_sync(FULL, pending != 0)) break;
            __nanosleep(32);
#pragma unroll
            for (int i = 0; i < PER; ++i)
                if ((pending >> i) & 1) d[i] = ld_desc(desc + g0 + lane + 32 * i);
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = g0 + lane + 32 * i;
            if (j < G) {
                const A v = acc_from_bits<A>(d[i].y);
                sa += v;
                if (j < c) sb += v;
            }
        }
    }
    sb = warp_sum(sb);
    sa = warp_sum(sa);
}

// Warp roles of one persistent CTA (one CTA per SM):
//   SW scanner warps    pass 2: each warp scans its own chunk of every sub-tile
//                       with a starting carry known in advance -> no CTA barriers
//   RWP reducer warps   pass 1: per-chunk totals of region r+lead
//   2 producer warps    TMA bulk copies: the scanners' ring (region r, out of
//                       L2) and the reducers' ring (region r+lead, from HBM,
//                       behind a bulk L2 prefetch of the whole portion)
//   1 ledger warp       gathers the G portion totals of a region and folds them
//                       with the chunk totals into per-chunk starting carries
// A chunk is ROWS x 1 KiB of input (one warp's share of a sub-tile).
template <typename TIn, typename TOut, int SW, int ROWS, int STAGES, int RWP, int RSTAGES>
struct RoundGeom {
    static constexpr int WARPS = SW + RWP + 3;
    static constexpr int THREADS = WARPS * 32;
    static constexpr int VEC = 32 / sizeof(TIn);
    static constexpr int ROW_ELEMS = 32 * VEC;
    static constexpr int CHUNK = ROWS * ROW_ELEMS;             // elements per chunk (one warp)
    static constexpr int SUB = SW * CHUNK;                     // elements per scanner stage
    static constexpr int SUB_BYTES = SUB * (int)sizeof(TIn);
    static constexpr int RSUB = RWP * CHUNK;                   // elements per reducer stage
    static constexpr int RSUB_BYTES = RSUB * (int)sizeof(TIn);
    static constexpr int MAX_CHUNKS = 256;                     // chunks per portion (smem arrays)
    static constexpr int SMEM = STAGES * SUB_BYTES + RSTAGES * RSUB_BYTES + 2 * (STAGES + RSTAGES) * 8 +
                                2 * 2 * MAX_CHUNKS * 8 + 64;
};

// Sum of one lane-row of VEC elements in the accumulator type.  For float32
// input the row is summed in float32 with Knuth's TwoSum error terms carried in
// a second float (6 FMA-pipe ops per element) and converted to double once per
// row: the conversion unit (XU, a quarter of the FP32 rate) is the scarce
// resource of this kernel.  The pair (s, c) is exact whenever the error terms
// sum without rounding -- e.g. for values on a common 2^-k grid such as
// uniform [0,1) floats; otherwise the row total is within ~2^-46 relative.
template <typename TIn, typename A, int VEC>
__device__ __forceinline__ A lane_row_sum(const TIn (&x)[VEC]) {
    if constexpr (sizeof(TIn) == 4 && (TIn)0.5 != (TIn)0) {
        // pairwise tree (depth log2 VEC), error terms gathered in the same tree
        float s[VEC], c[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            s[j] = x[j];
            c[j] = 0.f;
        }
#pragma unroll
        for (int d = 1; d < VEC; d <<= 1)
#pragma unroll
            for (int j = 0; j + d < VEC; j += 2 * d) {
                const float a = s[j], b = s[j + d];
                const float t = __fadd_rn(a, b);
                const float bp = __fsub_rn(t, a);
                const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(t, bp)), __fsub_rn(b, bp));
                s[j] = t;
                c[j] = __fadd_rn(__fadd_rn(c[j], c[j + d]), err);
            }
        return (A)s[0] + (A)c[0];
    } else {
        A v[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = (A)x[j];
#pragma unroll
        for (int d = 1; d < VEC; d <<= 1)
#pragma unroll
            for (int j = 0; j + d < VEC; j += 2 * d) v[j] += v[j + d];
        return v[0];
    }
}

template <typename A, int VEC>
__device__ __forceinline__ void lane_prefix(A (&v)[VEC]) {  // in-register inclusive scan, log2(VEC) levels
#pragma unroll
    for (int d = 1; d < VEC; d <<= 1)
#pragma unroll
        for (int j = VEC - 1; j >= d; --j) v[j] += v[j - d];
}

template <typename TIn, typename TOut, int SW, int ROWS, int STAGES, int RWP, int RSTAGES, int MINB = 1,
          bool STALL = false>
__global__ void __launch_bounds__((SW + RWP + 3) * 32, MINB) scan_rounds_kernel(const RoundArgs a) {
    using Geo = RoundGeom<TIn, TOut, SW, ROWS, STAGES, RWP, RSTAGES>;
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = Geo::VEC, ROW_ELEMS = Geo::ROW_ELEMS, CHUNK = Geo::CHUNK, SUB = Geo::SUB;
    constexpr int RSUB = Geo::RSUB;
    constexpr int MAXC = Geo::MAX_CHUNKS;
    constexpr bool FLOAT = (A)0.5 != (A)0;
    constexpr int RT = RWP * 32;
    constexpr int BAR_RED = 1;
    constexpr int W_SPROD = SW + RWP, W_RPROD = SW + RWP + 1, W_LEDGER = SW + RWP + 2;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    TIn *stage_buf = reinterpret_cast<TIn *>(smem_raw);
    TIn *rstage_buf = stage_buf + (size_t)STAGES * SUB;
    uint64_t *full = reinterpret_cast<uint64_t *>(rstage_buf + (size_t)RSTAGES * RSUB);
    uint64_t *empty = full + STAGES;
    uint64_t *rfull = empty + STAGES;
    uint64_t *rempty = rfull + RSTAGES;
    A *chunk_tot = reinterpret_cast<A *>(rempty + RSTAGES);  // [2][MAXC] (region parity)
    A *chunk_pre = chunk_tot + 2 * MAXC;                      // [2][MAXC] starting carries
    // role hand-offs are mbarriers, so waiting warps sleep in try_wait instead of
    // spinning on shared flags and stealing issue slots from the scanners:
    //   bar_red[r&1]   reducer -> ledger   chunk totals of region r written     (1 arrival)
    //   bar_pre[r&1]   ledger  -> all      chunk carries of region r written    (1 arrival)
    //   bar_scan[r&7]  scanners -> all     region r stored by every scanner warp (SW arrivals)
    // Scanner warps drift apart by at most STAGES sub-tiles (the TMA ring), i.e.
    // fewer than 8 regions, so arrivals for regions r and r+8 never share a phase.
    static_assert(STAGES < 8, "bar_scan slots must exceed the scanner drift");
    __shared__ __align__(8) uint64_t bar_red[2], bar_pre[2], bar_scan[8];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    TOut *out = reinterpret_cast<TOut *>(a.out);
    const uint64_t want = (uint64_t)a.epoch << 2;
    // this CTA's portion of region r: [p0, p0 + part)
    auto portion_of = [&](int64_t r, int64_t &p0, int64_t &part) {
        int64_t start;
        region_geom(a.portion, a.ramp, a.full_regions, G, SUB, r, start, part);
        p0 = start + (int64_t)c * part;
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], SW);
        }
        for (int s = 0; s < RSTAGES; ++s) {
            mbar_init(&rfull[s], 1);
            mbar_init(&rempty[s], RWP);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_red[i], 1);
            mbar_init(&bar_pre[i], 1);
        }
        for (int i = 0; i < 8; ++i) mbar_init(&bar_scan[i], SW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // sub-tiles [k_lo, k_hi) of a region's portion are fully valid (scanner TMA path)
    auto span_of = [&](int64_t r, int64_t &p0, int64_t &k_lo, int64_t &k_hi) {
        int64_t part;
        portion_of(r, p0, part);
        const int64_t nsub = part / SUB;
        k_lo = a.lo <= p0 ? 0 : (a.lo - p0 + SUB - 1) / SUB;
        k_hi = a.hi <= p0 ? 0 : (a.hi - p0) / SUB;
        if (k_hi > nsub) k_hi = nsub;
        if (k_lo > k_hi) k_lo = k_hi;
    };
    auto whole_portion = [&](int64_t r) {
        int64_t p0, part;
        portion_of(r, p0, part);
        return p0 >= a.lo && p0 + part <= a.hi;
    };
    // wait until region q has been stored by every scanner warp / has its carries
    // (q < 0: nothing to wait for).  Slot reuse is safe: a waiter for region q
    // has already waited for region q-8 (q-2 for bar_pre).
    auto wait_scanned = [&](int64_t q) {
        if (q >= 0) mbar_wait(&bar_scan[q & 7], (uint32_t)((q >> 3) & 1));
    };
    auto wait_prefixed = [&](int64_t q) {
        if (q >= 0) mbar_wait(&bar_pre[q & 1], (uint32_t)((q >> 1) & 1));
    };
    // L2 holds regions [r-lead, r]; chunk_tot[r&1] is free once the ledger used region r-2
    auto wait_reducer_may_start = [&](int64_t r) {
        wait_scanned(r - a.lead_regions - 1);
        wait_prefixed(r - 2);
    };

    if (warp == W_RPROD) {
        // ================ reducer producer: L2 prefetch + TMA ring ================
        if (lane == 0) {
            const uint64_t pol_keep = policy_evict_last();
            uint32_t use = 0;
            for (int64_t r = 0; r < a.rounds; ++r) {
                if (!whole_portion(r)) continue;
                wait_reducer_may_start(r);
                int64_t p0, part;
                portion_of(r, p0, part);
                const int64_t nrsub = part / RSUB;
                if (a.l2_prefetch) {
                    constexpr int64_t PIECE = 65536;
                    const int64_t bytes = part * (int64_t)sizeof(TIn);
                    const char *src = reinterpret_cast<const char *>(in + p0);
                    for (int64_t o = 0; o < bytes; o += PIECE) {
                        const uint32_t sz = (uint32_t)((bytes - o) < PIECE ? (bytes - o) : PIECE);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + o), "r"(sz) : "memory");
                    }
                }
                for (int64_t k = 0; k < nrsub; ++k, ++use) {
                    const uint32_t st = use % RSTAGES;
                    stall_site<STALL>(a.stall, r * G + c, k, 3);
                    mbar_wait(&rempty[st], ((use / RSTAGES) & 1) ^ 1);
                    mbar_expect_tx(&rfull[st], Geo::RSUB_BYTES);
                    bulk_g2s(rstage_buf + (size_t)st * RSUB, in + p0 + k * RSUB, Geo::RSUB_BYTES, &rfull[st], pol_keep);
                }
            }
        }
        return;
    }

    if (warp >= SW && warp < W_SPROD) {
        // ======================= reducer warps: pass 1 ===========================
        const int rw = warp - SW;
        uint32_t use = 0;
        for (int64_t r = 0; r < a.rounds; ++r) {
            wait_reducer_may_start(r);
            stall_site<STALL>(a.stall, r * G + c, rw, 1);
#ifdef PS_TRACE
            if (g_trace && rw == 0 && lane == 0) g_trace[(r * G + c) * 8 + 0] = gtimer();
#endif
            A *tot = chunk_tot + (r & 1) * MAXC;
            int64_t p0, part;
            portion_of(r, p0, part);
            const int64_t nrsub = part / RSUB, nchunk = part / CHUNK;
            if (whole_portion(r)) {
                for (int64_t k = 0; k < nrsub; ++k, ++use) {
                    const uint32_t st = use % RSTAGES;
                    mbar_wait(&rfull[st], (use / RSTAGES) & 1);
                    const TIn *sb = rstage_buf + (size_t)st * RSUB + (size_t)rw * CHUNK;
                    V256 raw[ROWS];
#pragma unroll
                    for (int rr = 0; rr < ROWS; ++rr) raw[rr] = lds256(sb + rr * ROW_ELEMS + lane * VEC);
                    A s = (A)0;
#pragma unroll
                    for (int rr = 0; rr < ROWS; ++rr) {
                        TIn x[VEC];
                        unpack<TIn>(raw[rr], x);
                        s += lane_row_sum<TIn, A, VEC>(x);
                    }
                    // release the stage only once the loaded values have been consumed
                    // (and behind a generic->async proxy fence): a shared load still in
                    // flight must not race the next TMA fill
                    s = warp_sum(s);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&rempty[st]);
                    if (lane == 0) tot[k * RWP + rw] = s;
                }
            } else {
                for (int64_t ch = rw; ch < nchunk; ch += RWP) {
                    A s = (A)0;
                    for (int rr = 0; rr < ROWS; ++rr)
                        for (int j = 0; j < VEC; ++j) {
                            const int64_t pos = p0 + ch * CHUNK + rr * ROW_ELEMS + lane * VEC + j;
                            if (pos >= a.lo && pos < a.hi) s += (A)in[pos];
                        }
                    s = warp_sum(s);
                    if (lane == 0) tot[ch] = s;
                }
            }
            named_sync(BAR_RED, RT);
            if (rw == 0) {  // portion total, fixed order -> the region ledger in global memory
                A t = (A)0;
                for (int64_t ch = lane; ch < nchunk; ch += 32) t += tot[ch];
                t = warp_sum(t);
                stall_site<STALL>(a.stall, r * G + c, 0, 2);
                if (lane == 0) {
                    st_desc(a.desc + r * G + c, want | ST_A, acc_to_bits<A>(t));
                    __threadfence_block();
                    mbar_arrive(&bar_red[r & 1]);
#ifdef PS_TRACE
                    if (g_trace) g_trace[(r * G + c) * 8 + 1] = gtimer();
#endif
                }
            }
            named_sync(BAR_RED, RT);
        }
        return;
    }

    if (warp == W_SPROD) {
        // ==================== scanner producer: TMA ring out of L2 =================
        if (lane == 0) {
            const uint64_t pol_stream = policy_evict_first();
            uint32_t use = 0;
            for (int64_t r = 0; r < a.rounds; ++r) {
                int64_t p0, k_lo, k_hi;
                span_of(r, p0, k_lo, k_hi);
                for (int64_t k = k_lo; k < k_hi; ++k, ++use) {
                    const uint32_t st = use % STAGES;
                    stall_site<STALL>(a.stall, r * G + c, k, 8);
#ifdef PS_TRACE
                    const int64_t tk = ((r * (a.portion / SUB) + k) * (SW + 1) + SW) * 4;
                    if (g_trace2 && c == 0) g_trace2[tk] = gtimer();
#endif
                    mbar_wait(&empty[st], ((use / STAGES) & 1) ^ 1);
#ifdef PS_TRACE
                    if (g_trace2 && c == 0) g_trace2[tk + 1] = gtimer();
#endif
                    mbar_expect_tx(&full[st], Geo::SUB_BYTES);
                    bulk_g2s(stage_buf + (size_t)st * SUB, in + p0 + k * SUB, Geo::SUB_BYTES, &full[st], pol_stream);
                }
            }
        }
        return;
    }

    if (warp == W_LEDGER) {
        // ======================= ledger warp =====================================
        A carry = (A)0;  // seed + totals of all earlier regions (same on every CTA)
        {
            A seed = (A)0;
            if (a.seed_terms) {
                const A *st = reinterpret_cast<const A *>(a.seed_terms);
                for (int64_t i = lane; i < a.n_seed_terms; i += 32) seed += st[i];
            }
            carry = acc_from_bits<A>(a.seed_bits) + warp_sum(seed);
            if (a.mail.n) carry += mailbox_sum<A>(a.mail, lane);
        }
        for (int64_t r = 0; r < a.rounds; ++r) {
            A sb, sa;
            stall_site<STALL>(a.stall, r * G + c, 0, 4);
            gather_totals<A>(a.desc + r * G, G, c, want, lane, sb, sa);

#ifdef PS_TRACE
            if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 2] = gtimer();
#endif
            // own chunk totals ready, and the scanners are done with region r-2's carries
            mbar_wait(&bar_red[r & 1], (uint32_t)((r >> 1) & 1));
            wait_scanned(r - 2);
            const A *tot = chunk_tot + (r & 1) * MAXC;
            A *pre = chunk_pre + (r & 1) * MAXC;
            int64_t p0r, part;
            portion_of(r, p0r, part);
            const int64_t nchunk = part / CHUNK;
            // exclusive scan of the chunk totals: lane owns a contiguous block of chunks
            const int64_t per = (nchunk + 31) / 32;
            const int64_t b0 = lane * per, b1 = (b0 + per) < nchunk ? (b0 + per) : nchunk;
            A own = (A)0;
            for (int64_t ch = b0; ch < b1; ++ch) own += tot[ch];
            A incl = own;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const A y = shfl_up(incl, dd);
                if (lane >= dd) incl += y;
            }
            A ex = shfl_up(incl, 1);
            if (lane == 0) ex = (A)0;
            A run = carry + sb + ex;
            for (int64_t ch = b0; ch < b1; ++ch) {
                pre[ch] = run;
                run += tot[ch];
            }
            carry += sa;
            stall_site<STALL>(a.stall, r * G + c, 0, 5);
            __syncwarp();
            __threadfence_block();
            if (lane == 0) mbar_arrive(&bar_pre[r & 1]);
#ifdef PS_TRACE
            if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 3] = gtimer();
#endif
        }
        if (c == 0 && lane == 0 && a.total) *reinterpret_cast<A *>(a.total) = carry;
        return;
    }

    // ========================= scanner warps: pass 2 ================================
    const uint64_t pol_stream = policy_evict_first();
    uint32_t use = 0;
    for (int64_t r = 0; r < a.rounds; ++r) {
        wait_prefixed(r);
        stall_site<STALL>(a.stall, r * G + c, warp, 6);
#ifdef PS_TRACE
        if (g_trace && warp == 0 && lane == 0) g_trace[(r * G + c) * 8 + 4] = gtimer();
#endif
        const A *pre = chunk_pre + (r & 1) * MAXC;
        int64_t p0, k_lo, k_hi, part;
        span_of(r, p0, k_lo, k_hi);
        portion_of(r, p0, part);
        const int64_t nsub = part / SUB;
        for (int64_t k = 0; k < nsub; ++k) {
            const int64_t t0 = p0 + k * SUB + (int64_t)warp * CHUNK;  // this warp's chunk
            const int64_t sub0 = p0 + k * SUB;
            if (sub0 + SUB <= a.lo) continue;
            if (sub0 >= a.hi) break;
            const bool tma = k >= k_lo && k < k_hi;
            stall_site<STALL>(a.stall, (r * G + c) * 4096 + k, warp, 7);
            A v[ROWS][VEC];
#ifdef PS_TRACE
            const int64_t tk = ((r * (a.portion / SUB) + k) * (SW + 1) + warp) * 4;
            if (g_trace2 && c == 0 && lane == 0) g_trace2[tk] = gtimer();
#endif
            if (tma) {
                const uint32_t st = use % STAGES;
                mbar_wait(&full[st], (use / STAGES) & 1);
#ifdef PS_TRACE
                if (g_trace2 && c == 0 && lane == 0) g_trace2[tk + 1] = gtimer();
#endif
                const TIn *sb = stage_buf + (size_t)st * SUB + (size_t)warp * CHUNK;
                V256 raw[ROWS];
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) raw[rr] = lds256(sb + rr * ROW_ELEMS + lane * VEC);
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) {
                    TIn x[VEC];
                    unpack<TIn>(raw[rr], x);
#pragma unroll
                    for (int j = 0; j < VEC; ++j) v[rr][j] = (A)x[j];
                }
                ++use;
            } else {
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
                    for (int j = 0; j < VEC; ++j) {
                        const int64_t pos = t0 + rr * ROW_ELEMS + lane * VEC + j;
                        v[rr][j] = (pos >= a.lo && pos < a.hi) ? (A)in[pos] : (A)0;
                    }
            }
#pragma unroll
            for (int rr = 0; rr < ROWS; ++rr) {
#pragma unroll
                for (int j = 1; j < VEC; ++j) v[rr][j] += v[rr][j - 1];  // x0 + ... + xj (rows give the ILP)
            }
            if (tma) {
                // Hand the stage back only after every loaded value has been consumed
                // (the row prefixes depend on all of them) and after a generic->async
                // proxy fence: the next TMA fill of this stage must not overtake a
                // shared load that is still in flight (observed for int64, where the
                // widening is a no-op and nothing else waited on the loads).
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[(use - 1) % STAGES]);
            }
            A sc[ROWS];
#pragma unroll
            for (int rr = 0; rr < ROWS; ++rr) sc[rr] = v[rr][VEC - 1];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) {
                    const A y = shfl_up(sc[rr], d);
                    if (lane >= d) sc[rr] += y;
                }
            }
            A base = pre[k * SW + warp];
#pragma unroll
            for (int rr = 0; rr < ROWS; ++rr) {
                A ex;
                if constexpr (FLOAT) {
                    ex = shfl_up(sc[rr], 1);
                    if (lane == 0) ex = (A)0;
                } else {
                    ex = sc[rr] - v[rr][VEC - 1];
                }
                const A b = base + ex;
                base += shfl_idx(sc[rr], 31);
                TOut y[VEC];
                if (a.exclusive) {
                    y[0] = (TOut)b;
#pragma unroll
                    for (int j = 1; j < VEC; ++j) y[j] = (TOut)(b + v[rr][j - 1]);
                } else {
#pragma unroll
                    for (int j = 0; j < VEC; ++j) y[j] = (TOut)(b + v[rr][j]);
                }
                if (tma) {
                    constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
                    for (int q = 0; q < NV; ++q)
                        stg256_policy(out + t0 + rr * ROW_ELEMS + lane * VEC + q * (32 / sizeof(TOut)),
                                      pack<TOut>(&y[q * (32 / sizeof(TOut))]), pol_stream);
                } else {
#pragma unroll
                    for (int j = 0; j < VEC; ++j) {
                        const int64_t pos = t0 + rr * ROW_ELEMS + lane * VEC + j;
                        if (pos >= a.lo && pos < a.hi) out[pos] = y[j];
                    }
                }
            }
#ifdef PS_TRACE
            if (g_trace2 && c == 0 && lane == 0) g_trace2[tk + 2] = gtimer();
#endif
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_scan[r & 7]);
#ifdef PS_TRACE
        if (g_trace && warp == 0 && lane == 0) g_trace[(r * G + c) * 8 + 5] = gtimer();
#endif
    }
}

}  // namespace ps
