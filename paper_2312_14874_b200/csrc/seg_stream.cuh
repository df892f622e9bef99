// seg_stream.cuh -- CSR-segmented scans on the shared-memory-region
// accumulate-scan (the stream kernel's structure, stream_kernel.cuh).
//
// Segment s is in[off[s] .. off[s+1]); every segment restarts at zero and
// seg_totals[s] receives its sum (ps_scan_segmented).  The reference has no
// kernel of this shape: it is the general form of the per-chunk scans of
// simd.py:164-206 with chunk boundaries from an offsets array.  The look-back
// form (segmented.cuh) is bound by the carry chain's L2 round trips; here the
// data streams through shared memory exactly as for a plain 1-D scan -- one
// HBM read and one write per element -- and the segments only change the
// operator: the segmented sum on (head flag, value) pairs,
//     (f1, v1) . (f2, v2) = (f1 | f2,  f2 ? v2 : v1 + v2),
// applied by every role in a fixed order (deterministic float results).
//
// A pre-pass (seg_prepare_kernel) scatters the offsets into a head bitmap in
// global memory (1 bit per position) and computes, per CTA portion q (P
// positions of region r, q = r * G + c), the lower bound lb[q] of its start in
// the offsets and a flag for repeated offsets (empty segments) inside it.  Roles:
//   producer    TMA bulk copies of the portion and of its slice of the head bitmap
//               (plus the next 128 bits) into slot r % NBUF
//   head warp   per slot: counts of heads before every 32-position word (prefix
//               popcounts, for the segment index of a total) and the portion's
//               lb / flags (prefetched 32 regions at a time)
//   reducers    per-chunk segmented aggregates (f, v) from shared memory;
//               the portion aggregate -> the region's descriptor (flag in bit 62)
//   ledger      grid-wide gather of the region's G portion aggregates, segmented
//               fold -> one carry per chunk
//   scanners    segmented in-lane / warp scans of each chunk, the chunk carry
//               applied where no head precedes; each element followed by a head
//               (a segment's last element) writes the segment total
#pragma once
#ifndef PS_SEG_EXP
#define PS_SEG_EXP 0
#endif
#ifndef PS_SEG_SLEEP
#define PS_SEG_SLEEP 1
#endif
#if PS_SEG_SLEEP == 2
#define SEG_WAIT(bar, par) mbar_wait_backoff(bar, par)
#elif PS_SEG_SLEEP
#define SEG_WAIT(bar, par) mbar_wait_sleep(bar, par)
#else
#define SEG_WAIT(bar, par) mbar_wait(bar, par)
#endif
#ifndef PS_SEG_WIDE
#define PS_SEG_WIDE 1
#endif
#ifndef PS_SEG_RED_ROLLED
#define PS_SEG_RED_ROLLED 0
#endif
#ifndef PS_SEG_POLL_NS  // ledger: pause between polls of a region's descriptors
#define PS_SEG_POLL_NS 32
#endif
#ifndef PS_SEG_EARLY_ISSUE
#define PS_SEG_EARLY_ISSUE 0
#endif
#ifndef PS_SEG_WSPLIT  // scanner: separate copy of the row loop for whole portions
#define PS_SEG_WSPLIT 1
#endif
#ifndef PS_SEG_INCLEAR  // head warp clears the consumed bitmap slice (no memset after the launch)
#define PS_SEG_INCLEAR 1
#endif
#ifndef PS_SEG_RED_WSPLIT  // reducers: separate whole-portion copy (measured slower: code layout)
#define PS_SEG_RED_WSPLIT 0
#endif
#ifndef PS_SEG_UNROLL
#define PS_SEG_UNROLL 1
#endif
#ifdef PS_SEG_TRACE  // development builds only: per (region, CTA) timestamps of the role hand-offs
__device__ uint64_t *g_seg_trace;
#define SEG_TRACE(r, k)                                                                        \
    do {                                                                                       \
        if (g_seg_trace) {                                                                     \
            uint64_t t_;                                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
            g_seg_trace[((r) * gridDim.x + blockIdx.x) * 8 + (k)] = t_;                        \
        }                                                                                      \
    } while (0)
#else
#define SEG_TRACE(r, k) do { } while (0)
#endif

#include <type_traits>

#include "stream_kernel.cuh"

namespace ps {

constexpr int SEG_UNROLL = PS_SEG_UNROLL;  // scanner rows per loop body (code size vs ILP; measured)
constexpr uint64_t SEG_FLAG = 1ull << 62;  // descriptor word: the portion holds a segment head

struct SegStreamArgs {
    const void *in;   // aligned base: position p <-> element p - lead
    void *out;
    int64_t lo, hi;   // valid positions
    int64_t lead;
    int64_t portion;  // positions per CTA per region
    int64_t rounds;
    const int64_t *offsets;  // nseg + 1 entries
    int64_t nseg;
    const int64_t *lb;       // [rounds * G + 1]: lower_bound(offsets, q * P - lead) << 2
    const uint32_t *dupflag; // [rounds * G + 1]: nonzero if offsets repeat inside portion q
    const uint32_t *bitmap;  // head bitmap by position, rounds * G * P + 128 bits
    void *totals;            // acc-typed per segment, pre-zeroed; nullable
    ulonglong2 *desc;        // rounds * G descriptors (+ rounds * G more for integers: head info)
    uint32_t epoch;
    int exclusive;
    int inflight;
    int one;  // 1 (the opaque multiplier of add_widen)
};

// offsets of uniform segments (rows of `ucols` elements, ps_scan_batched's short rows) are
// computed, not read
__device__ __forceinline__ int64_t seg_off(const int64_t *off, int64_t ucols, int64_t t) {
    return off ? __ldg(off + t) : t * ucols;
}

// Pre-pass, one thread per offset t (0..nseg):
//   bitmap          bit (off[t] + lead) set (the terminal off[nseg] = n too);
//   dupflag[q]      4 if two offsets coincide inside portion q (empty segments);
//   lb[q] (q <= Q)  = first s in [0, nseg] with off[s] >= q * P - lead (nseg + 1 if none), stored
//                     << 2 so no word of it can pass for a published descriptor: thread t owns
//                     the portion boundaries in (off[t-1], off[t]] -- every boundary lies in
//                     exactly one such interval, so each lb entry is written once, without the
//                     chain of dependent loads a per-boundary search over the offsets costs
//                     (the first version galloped and bisected: ~10 round trips, 12 us).
// bitmap and dupflag must be zero on entry.
__global__ void seg_prepare_kernel(const int64_t *off, int64_t ucols, int64_t nseg, int64_t n, int64_t lead,
                                   int64_t P, int64_t Q, int64_t *lb, uint32_t *dupflag, uint32_t *bitmap) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t > nseg) return;
    const int64_t e = seg_off(off, ucols, t);
    const int64_t prev = t > 0 ? seg_off(off, ucols, t - 1) : -1;
    const int64_t pos = e + lead;
    const int ps = 63 - __clzll(P);  // P is a power of two (32 KiB of input elements)
    atomicOr(bitmap + (pos >> 5), 1u << (pos & 31));
    if (t > 0 && prev == e) atomicOr(dupflag + (pos >> ps), 4u);
    // boundaries q * P - lead in (prev, e]  (thread 0: all boundaries <= off[0])
    int64_t qlo = t > 0 ? ((prev + lead) >> ps) + 1 : 0;
    int64_t qhi = pos >> ps;
    if (qhi > Q) qhi = Q;
    for (int64_t q = qlo; q <= qhi; ++q) lb[q] = t << 2;
    if (t == nseg)  // boundaries past the end of the input
        for (int64_t q = qhi + 1; q <= Q; ++q) lb[q] = (nseg + 1) << 2;
}

// Segment totals of the instantiations with 8-byte (= accumulator-typed) outputs are read back
// from the scan's own output after the launch (the inclusive value of a segment's last
// element is its total: exact in two's complement for integers, the very float64 value the
// scanners would have stored for floats) instead of being scattered by the scanners: one
// 64-byte fetch per segment against a per-head loop on the scanners' serial path.  An
// exclusive scan keeps the last element in totals[] from before the launch (input and output
// may alias) and adds it to the last exclusive value.
template <typename TIn, typename A>
__global__ void seg_last_in_kernel(const TIn *in, const int64_t *off, int64_t ucols, int64_t nseg, A *tot) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nseg) return;
    const int64_t b = seg_off(off, ucols, t), e = seg_off(off, ucols, t + 1);
    tot[t] = e > b ? (A)in[e - 1] : (A)0;
}
template <typename TOut, typename A>
__global__ void seg_totals_gather_kernel(const TOut *out, const int64_t *off, int64_t ucols, int64_t nseg, A *tot,
                                         int exclusive) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nseg) return;
    const int64_t b = seg_off(off, ucols, t), e = seg_off(off, ucols, t + 1);
    A v = (A)0;
    if (e > b) {
        // one 8-byte element per segment out of a multi-GB array: fetch 64 bytes from DRAM into
        // L2, not the default 128 (ncu: 132 B of DRAM reads per segment before)
        if constexpr (sizeof(TOut) == 8) {
            uint64_t raw;
            asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(raw) : "l"(out + e - 1));
            v = (A) * reinterpret_cast<const TOut *>(&raw);
        } else {
            v = (A)out[e - 1];  // (instantiated, never launched: narrow outputs emit their totals in-kernel)
        }
        if (exclusive) v += tot[t];
    }
    tot[t] = v;
}

// acc + (A)x.  For 32-bit integer input under a 64-bit accumulator the widening is one
// IMAD.WIDE on the FMA pipe (multiplier `one` = 1 from the kernel arguments, opaque to
// ptxas, which would otherwise sign-extend on the ALU pipe): the kernel was bound by the ALU
// pipe (ncu: 61 % busy against 10 % for the FMA pipe).
template <typename A, typename TIn> __device__ __forceinline__ A add_widen(A acc, TIn x, int one) {
#if PS_SEG_WIDE
    if constexpr (sizeof(TIn) == 4 && sizeof(A) == 8 && (A)0.5 == (A)0) {
        A d;
        if constexpr ((TIn)-1 < (TIn)0)
            asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"((int)x), "r"(one), "l"(acc));
        else
            asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"((unsigned)x), "r"(one), "l"(acc));
        return d;
    }
#endif
    (void)one;
    return acc + (A)x;
}
// inclusive plain scan of a 64-bit integer across the warp: the adds are predicated on
// shfl.up's own "source lane in range" predicate (no lane compares)
template <typename A> __device__ __forceinline__ A warp_scan_pred(A v) {
    static_assert(sizeof(A) == 8, "64-bit accumulators");
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        asm volatile(
            "{\n .reg .pred q;\n .reg .b32 lo, hi, tl, th;\n .reg .b64 t;\n"
            " mov.b64 {lo, hi}, %0;\n"
            " shfl.sync.up.b32 tl|q, lo, %1, 0, 0xffffffff;\n"
            " shfl.sync.up.b32 th, hi, %1, 0, 0xffffffff;\n"
            " mov.b64 t, {tl, th};\n"
            " @q add.s64 %0, %0, t;\n}"
            : "+l"(v)
            : "r"(d));
    }
    return v;
}

// the two 16-byte descriptors of one portion of an integer scan (total; sum before the last
// head + head flag) sit side by side and are polled with ONE 256-bit strong load -- each
// half carries its own tag, so tearing between the halves is harmless.  Five loads per lane
// and region (as the 1-D kernel) instead of ten: the next region's gather can be in flight
// during the fold without its loads holding the scoreboards the fold's shuffles wait on.
__device__ __forceinline__ void ld_desc_pair(const ulonglong2 *p, ulonglong2 &a, ulonglong2 &b) {
    asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y)
                 : "l"(p)
                 : "memory");
}

template <typename A> struct SegPair {
    A v;
    uint32_t f;
};
template <typename A> __device__ __forceinline__ SegPair<A> seg_combine(const SegPair<A> &a, const SegPair<A> &b) {
    return SegPair<A>{b.f ? b.v : a.v + b.v, a.f | b.f};
}
template <typename A> __device__ __forceinline__ SegPair<A> seg_shfl_up(const SegPair<A> &p, int d) {
    return SegPair<A>{shfl_up(p.v, d), __shfl_up_sync(FULL, p.f, d)};
}
// inclusive segmented scan across the warp (lane order)
template <typename A> __device__ __forceinline__ SegPair<A> seg_warp_scan(SegPair<A> p, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const SegPair<A> y = seg_shfl_up(p, d);
        if (lane >= d) p = seg_combine(y, p);
    }
    return p;
}

struct SegMeta {       // per buffer slot, written by the head warp
    int64_t lb0, lb1;  // the portion's offsets: off[lb0 .. lb1)
    int32_t dup, next_head, live, pad;
};

template <typename TIn, int SW, int ROWS, int NBUF, int RWP>
struct SegStreamGeom {
    static constexpr int WARPS = SW + RWP + 3;  // + producer, ledger, head warp
    static constexpr int THREADS = WARPS * 32;
    static constexpr int VEC = 32 / sizeof(TIn);
    static constexpr int ROW_ELEMS = 32 * VEC;
    static constexpr int CHUNK = ROWS * ROW_ELEMS;
    static constexpr int MAXC = 16;
    static constexpr int64_t P = 32768 / sizeof(TIn);  // 32 KiB of input per CTA per region
    static constexpr int WORDS = (int)(P / 32);         // head bitmap words per portion
    static constexpr int BMW = WORDS + 4;               // per slot: + the next 128 positions (TMA: 16 B units)
    using Meta = SegMeta;
    static constexpr int SMEM_FIXED = NBUF * BMW * 4 + 5 * NBUF * 8 + 4 * NBUF * MAXC * 8 + 2 * 32 * GATHER_LP * 8 + 32 * GATHER_LP * 4 +
                                      2 * NBUF * MAXC * 4 + NBUF * 4 +
                                      NBUF * WORDS * 4 + NBUF * (int)sizeof(Meta) + 128;
    static constexpr int SMEM = (int)(NBUF * P * sizeof(TIn)) + SMEM_FIXED;
};

template <typename TIn, typename TOut, int SW, int ROWS, int NBUF, int RWP>
__global__ void __launch_bounds__((SW + RWP + 3) * 32, 1) seg_stream_kernel(const SegStreamArgs a) {
    using Geo = SegStreamGeom<TIn, SW, ROWS, NBUF, RWP>;
    using A = typename AccOf<TIn>::type;
    using Pair = SegPair<A>;
    using Meta = typename Geo::Meta;
    constexpr int VEC = Geo::VEC, ROW_ELEMS = Geo::ROW_ELEMS, CHUNK = Geo::CHUNK, MAXC = Geo::MAXC;
    constexpr int WORDS = Geo::WORDS, BMW = Geo::BMW;
    constexpr int64_t P = Geo::P;
    constexpr int64_t NCHUNK = P / CHUNK;
    constexpr uint32_t VMASK = (VEC == 32) ? 0xffffffffu : ((1u << VEC) - 1);
    constexpr int RT = RWP * 32;
    constexpr int BAR_RED = 1;
    constexpr int W_PROD = SW + RWP, W_LEDGER = SW + RWP + 1, W_HEAD = SW + RWP + 2;
    static_assert(NCHUNK <= MAXC && NCHUNK <= 32, "chunks per portion");
    // integers: "subtract the segment base" form -- out = S - B with S the plain running
    // sum and B = S before the last head at or before the element (exact in two's
    // complement); floats: the (flag, value) pair operator (no cancellation)
    constexpr bool SUB = (A)0.5 == (A)0;
    // scans with 64-bit outputs: totals are gathered after the launch (seg_totals_gather_kernel)
    constexpr bool EMIT = sizeof(TOut) != 8;  // 8-byte outputs are accumulator-typed: totals gathered from them
    static_assert(32 % VEC == 0, "a lane's head bits sit in one bitmap word");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    TIn *buf = reinterpret_cast<TIn *>(smem_raw);
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem_raw + (size_t)NBUF * P * sizeof(TIn));  // TMA'd
    uint64_t *bars = reinterpret_cast<uint64_t *>(bitmap + NBUF * BMW);
    uint64_t *full = bars;              // TMA landed            (1 arrival + tx)
    uint64_t *hdr = bars + NBUF;        // head counts and meta  (1)
    uint64_t *red = bars + 2 * NBUF;    // chunk aggregates      (1)
    uint64_t *pre = bars + 3 * NBUF;    // chunk carries         (1)
    uint64_t *freeb = bars + 4 * NBUF;  // scanners released it  (SW)
    A *chunk_tot = reinterpret_cast<A *>(bars + 5 * NBUF);
    A *chunk_pre = chunk_tot + NBUF * MAXC;
    A *chunk_plh = chunk_pre + NBUF * MAXC;  // SUB: chunk sum before its last head (reducers)
    A *chunk_B = chunk_plh + NBUF * MAXC;    // SUB: S before the last head preceding the chunk (ledger)
    A *led_S = chunk_B + NBUF * MAXC;          // SUB ledger: S at the start of every portion of the region
    A *led_H = led_S + 32 * GATHER_LP;         // ... and S before every portion's last head
    uint32_t *led_F = reinterpret_cast<uint32_t *>(led_H + 32 * GATHER_LP);  // transposition: head flags
    uint32_t *chunk_f = led_F + 32 * GATHER_LP;
    int32_t *chunk_lh = reinterpret_cast<int32_t *>(chunk_f + NBUF * MAXC);  // chunk-relative last head, -1: none (head warp)
    uint32_t *row_heads = reinterpret_cast<uint32_t *>(chunk_lh + NBUF * MAXC);  // per slot: bit k = row k holds a head
    int32_t *cntb = reinterpret_cast<int32_t *>(row_heads + NBUF);
    Meta *meta = reinterpret_cast<Meta *>(cntb + NBUF * WORDS);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    TOut *out = reinterpret_cast<TOut *>(a.out);
    const uint64_t want = (uint64_t)a.epoch << 2;

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&hdr[b], 1);
            mbar_init(&red[b], 1);
            mbar_init(&pre[b], 1);
            mbar_init(&freeb[b], SW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto par = [&](int64_t r) { return (uint32_t)((r / NBUF) & 1); };
    auto p0_of = [&](int64_t r) { return (r * G + c) * P; };
    auto whole = [&](int64_t r) {
        const int64_t p0 = p0_of(r);
        return p0 >= a.lo && p0 + P <= a.hi;
    };
    auto live = [&](int64_t r) {
        const int64_t p0 = p0_of(r);
        return p0 + P > a.lo && p0 < a.hi;
    };
    // head bits of the VEC positions at portion-relative position q0 (a multiple of VEC)
    auto heads_at = [&](const uint32_t *bm, int64_t q0) {
        return (bm[q0 >> 5] >> (q0 & 31)) & VMASK;
    };

    if (warp == W_PROD) {
        // ============================ producer ===================================
        // lane 0 issues the bulk copies; for the instantiations whose totals are gathered
        // (nothing reads a neighbour's head bits) the whole warp also clears the global
        // bitmap slice and repeat flag of a region once its slot has been released, so the
        // launch leaves the scratch clean without a 32 MB memset behind it
        constexpr bool CLEAR = !EMIT && PS_SEG_INCLEAR;
        auto clear_region = [&](int64_t r) {
            uint32_t *g = const_cast<uint32_t *>(a.bitmap) + (p0_of(r) >> 5);
            for (int k = lane * 4; k < WORDS; k += 128) *reinterpret_cast<uint4 *>(g + k) = make_uint4(0u, 0u, 0u, 0u);
            if (lane == 0) const_cast<uint32_t *>(a.dupflag)[r * G + c] = 0u;
            if (r == a.rounds - 1 && c == G - 1 && lane == 1) {  // past the last portion
                *reinterpret_cast<uint4 *>(g + WORDS) = make_uint4(0u, 0u, 0u, 0u);
                const_cast<uint32_t *>(a.dupflag)[a.rounds * G] = 0u;
            }
        };
        const uint64_t pol = policy_evict_first();
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            if (lane == 0) {
                if (r >= NBUF) SEG_WAIT(&freeb[b], par(r - NBUF));
                if (r >= a.inflight && a.inflight > 0 && a.inflight < NBUF)
                    SEG_WAIT(&full[(r - a.inflight) % NBUF], par(r - a.inflight));
                // the portion's slice of the head bitmap (+ the next 128 positions) always;
                // its data when the portion is whole (boundary portions read global memory)
                constexpr uint32_t BM_BYTES = (uint32_t)BMW * 4;
                const bool w = whole(r);
                const uint32_t bytes = w ? (uint32_t)(P * sizeof(TIn)) : 0u;
                mbar_expect_tx(&full[b], bytes + BM_BYTES);
                bulk_g2s(bitmap + b * BMW, a.bitmap + (p0_of(r) >> 5), BM_BYTES, &full[b], pol);
                SEG_TRACE(r, 0);
                if (w) {
                    constexpr uint32_t PIECE = 16384;
                    const char *src = reinterpret_cast<const char *>(in + p0_of(r));
                    char *dst = reinterpret_cast<char *>(buf + (size_t)b * P);
                    for (uint32_t o = 0; o < bytes; o += PIECE)
                        bulk_g2s(dst + o, src + o, bytes - o < PIECE ? bytes - o : PIECE, &full[b], pol);
                }
            }
            if constexpr (CLEAR) {
                __syncwarp();  // lane 0 has seen slot b released: region r - NBUF is done with
                if (r >= NBUF) clear_region(r - NBUF);
            }
        }
        if constexpr (CLEAR) {
            for (int64_t r = a.rounds > NBUF ? a.rounds - NBUF : 0; r < a.rounds; ++r) {
                if (lane == 0) SEG_WAIT(&freeb[r % NBUF], par(r));
                __syncwarp();
                clear_region(r);
            }
        }
        return;
    }

    if (warp == W_HEAD) {
        // ============================ head warp ==================================
        constexpr int PER = WORDS / 32;
        int64_t pf_lb0 = 0, pf_lb1 = 0;  // lane k: portion (r0 + k) of this CTA, prefetched
        uint32_t pf_dup = 0;
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            if ((r & 31) == 0) {  // one round trip per 32 regions
                const int64_t rk = r + lane;
                if (rk < a.rounds) {
                    const int64_t q = rk * G + c;
                    pf_lb0 = a.lb[q] >> 2;
                    pf_lb1 = a.lb[q + 1] >> 2;
                    pf_dup = a.dupflag[q];
                }
            }
            const int k = (int)(r & 31);
            const int64_t s0 = __shfl_sync(FULL, pf_lb0, k), s1 = __shfl_sync(FULL, pf_lb1, k);
            const uint32_t dup = __shfl_sync(FULL, pf_dup, k);
            if (r >= NBUF) SEG_WAIT(&freeb[b], par(r - NBUF));
            SEG_WAIT(&full[b], par(r));  // the bitmap slice has landed
            const uint32_t *bm = bitmap + b * BMW;
            int32_t *cb = cntb + b * WORDS;
            // lane k holds the bitmap words of row k of the portion (32 rows): the last head of
            // every chunk (ROWS consecutive rows), for the reducers and the ledger
            static_assert(PER * 32 == ROW_ELEMS, "one lane of the head warp per row");
            uint32_t wd[PER];
            int32_t last = -1;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                wd[j] = bm[lane * PER + j];
                if (wd[j]) last = (lane * PER + j) * 32 + (31 - __clz((int)wd[j]));
            }
            const uint32_t rowmask = __ballot_sync(FULL, last >= 0);
            if (lane == 0) row_heads[b] = rowmask;
#pragma unroll
            for (int d = 1; d < ROWS; d <<= 1) last = max(last, __shfl_xor_sync(FULL, last, d));
            if (lane % ROWS == 0 && lane / ROWS < NCHUNK)
                chunk_lh[b * MAXC + lane / ROWS] = last >= 0 ? last - (lane / ROWS) * CHUNK : -1;
            if constexpr (EMIT) {
                // heads before each 32-position word: exclusive scan of popcounts
                int32_t v[PER], run = 0;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    v[j] = run;
                    run += __popc(wd[j]);
                }
                int32_t incl = run;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int32_t y = __shfl_up_sync(FULL, incl, d);
                    if (lane >= d) incl += y;
                }
                const int32_t ex = incl - run;
#pragma unroll
                for (int j = 0; j < PER; ++j) cb[lane * PER + j] = ex + v[j];
            }
            if (lane == 0) {
                Meta m;
                m.lb0 = s0;
                m.lb1 = s1;
                m.dup = dup != 0;
                m.next_head = (int32_t)(bm[WORDS] & 1u);
                m.live = live(r);
                m.pad = 0;
                meta[b] = m;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr[b]);
        }
        return;
    }

    if (warp >= SW && warp < W_PROD) {
        // ============================ reducers ===================================
        const int rw = warp - SW;
        if constexpr (SUB) {
            // per chunk: plain sum, and the sum of the elements before its last head
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                SEG_WAIT(&full[b], par(r));
                if (rw == 0 && lane == 0) SEG_TRACE(r, 1);
                const TIn *sb = buf + (size_t)b * P;
                const uint32_t *bm = bitmap + b * BMW;
                const int64_t p0 = p0_of(r);
                const bool w = whole(r);
                const bool lv = w || live(r);
                for (int64_t ch = rw; ch < NCHUNK; ch += RWP) {
                    A s = (A)0, pl = (A)0;
                    int lastpos = -1;
#if PS_SEG_RED_ROLLED
                    if (lv && PS_SEG_EXP != 11) {
                        // the chunk's last head from the head bitmap alone, then one rolled pass
                        // over the rows (small code: the hot loops of all roles share the SM's
                        // instruction cache)
#pragma unroll
                        for (int rr = 0; rr < ROWS; ++rr) {
                            const int64_t q0 = ch * CHUNK + rr * ROW_ELEMS + lane * VEC;
                            const uint32_t hb = heads_at(bm, q0);
                            if (hb) lastpos = rr * ROW_ELEMS + lane * VEC + (31 - __clz((int)hb));
                        }
                        const int lh = __reduce_max_sync(FULL, lastpos);  // -1: none
                        const int lrow = lh >= 0 ? lh / ROW_ELEMS : -1;
                        const int lim = lh - lrow * ROW_ELEMS - lane * VEC;  // row lrow: this lane's elements j < lim
#pragma unroll 1
                        for (int rr = 0; rr < ROWS; ++rr) {
                            const int64_t q0 = ch * CHUNK + rr * ROW_ELEMS + lane * VEC;
                            TIn x[VEC];
                            if (w) {
                                unpack<TIn>(lds256<(sizeof(TIn) == 8)>(sb + q0), x);
                            } else {
#pragma unroll
                                for (int j = 0; j < VEC; ++j) {
                                    const int64_t pos = p0 + q0 + j;
                                    x[j] = (pos >= a.lo && pos < a.hi) ? in[pos] : (TIn)0;
                                }
                            }
                            A t = (A)x[0];
#pragma unroll
                            for (int j = 1; j < VEC; ++j) t = add_widen(t, x[j], a.one);
                            s += t;
                            if (rr < lrow) {
                                pl += t;
                            } else if (rr == lrow) {
#pragma unroll
                                for (int j = 0; j < VEC; ++j)
                                    if (j < lim) pl += (A)x[j];
                            }
                        }
                        if (lh >= 0) pl = warp_sum(pl);
                        lastpos = lh;
                    }
#else
                    auto reduce_chunk = [&](auto whole_c) {
                        constexpr bool W = decltype(whole_c)::value;
                        TIn x[ROWS][VEC];
                        A rs[ROWS];  // the lane's sum of each row
#pragma unroll
                        for (int rr = 0; rr < ROWS; ++rr) {
                            const int64_t q0 = ch * CHUNK + rr * ROW_ELEMS + lane * VEC;
                            if (W || w) {
                                unpack<TIn>(lds256<(sizeof(TIn) == 8)>(sb + q0), x[rr]);
                            } else {
#pragma unroll
                                for (int j = 0; j < VEC; ++j) {
                                    const int64_t pos = p0 + q0 + j;
                                    x[rr][j] = (pos >= a.lo && pos < a.hi) ? in[pos] : (TIn)0;
                                }
                            }
                            A t = (A)x[rr][0];
#pragma unroll
                            for (int j = 1; j < VEC; ++j)
                                if (PS_SEG_EXP != 15 || j == VEC - 1) t = add_widen(t, x[rr][j], a.one);
                            rs[rr] = t;
                            s += t;
                        }
                        SEG_WAIT(&hdr[b], par(r));  // the head warp's pass over the slot's bitmap
                        const int lh = PS_SEG_EXP == 16 ? -1 : chunk_lh[b * MAXC + ch];  // the chunk's last head (-1: none)
                        if (lh >= 0) {
                            // sum before the last head: whole rows before its row, and in that row
                            // (warp-uniform index) the elements before it
                            const int lrow = lh / ROW_ELEMS;
                            const int lim = lh - lrow * ROW_ELEMS - lane * VEC;  // this lane's elements j < lim
#pragma unroll
                            for (int rr = 0; rr < ROWS; ++rr) {
                                if (rr < lrow) {
                                    pl += rs[rr];
                                } else if (rr == lrow) {
#pragma unroll
                                    for (int j = 0; j < VEC; ++j)
                                        if (j < lim) pl += (A)x[rr][j];
                                }
                            }
                            pl = warp_sum(pl);
                        }
                        lastpos = lh;
                    };
                    if (lv && PS_SEG_EXP != 11) {
#if PS_SEG_RED_WSPLIT
                        if (w) reduce_chunk(std::true_type{});  // whole portions: no bounds logic in the hot copy
                        else reduce_chunk(std::false_type{});
#else
                        reduce_chunk(std::false_type{});
#endif
                    }
#endif
                    s = warp_sum(s);
                    if (lane == 0) {
                        chunk_tot[b * MAXC + ch] = s;
                        chunk_plh[b * MAXC + ch] = pl;
                        chunk_f[b * MAXC + ch] = lastpos >= 0;
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                named_sync(BAR_RED, RT);
                if (rw == 0) {
                    // the portion (lanes = chunks): total, and the sum before its last head
                    const A ct = lane < NCHUNK ? chunk_tot[b * MAXC + lane] : (A)0;
                    const uint32_t fb = __ballot_sync(FULL, lane < NCHUNK && chunk_f[b * MAXC + lane] != 0u);
                    const int kl = fb ? 31 - __clz((int)fb) : -1;
                    const A t = warp_sum(ct);
                    const A before = warp_sum(lane < kl ? ct : (A)0);
                    const A plh = before + (kl >= 0 ? chunk_plh[b * MAXC + kl] : (A)0);
                    if (lane == 0) {
                        ulonglong2 *rec = a.desc + 2 * (r * G + c);  // {total, sum before the last head}
                        st_desc(rec + 1, want | ST_A | (fb ? SEG_FLAG : 0ull), acc_to_bits<A>(plh));
                        st_desc(rec, want | ST_A, acc_to_bits<A>(t));
                        SEG_TRACE(r, 2);
                        mbar_arrive(&red[b]);
                    }
                }
                named_sync(BAR_RED, RT);
            }
            return;
        }
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            SEG_WAIT(&full[b], par(r));  // data and head bits (the reducers need no counts)
            if (rw == 0 && lane == 0) SEG_TRACE(r, 1);
            const TIn *sb = buf + (size_t)b * P;
            const uint32_t *bm = bitmap + b * BMW;
            const int64_t p0 = p0_of(r);
            const bool w = whole(r);
            const bool lv = w || live(r);
            if (lv) SEG_WAIT(&hdr[b], par(r));  // the chunks' last heads (head warp)
            for (int64_t ch = rw; ch < NCHUNK; ch += RWP) {
                // the chunk's aggregate under the segmented-sum operator: (any head, sum of the
                // elements from its last head on -- of all of them if it holds none).  The head
                // warp found the last head, so this is one masked sum: lanes, then one warp tree
                // (a fixed order: deterministic)
                A acc = (A)0;
                int lh = -1;
                if (lv) {
                    lh = chunk_lh[b * MAXC + ch];
                    const int lrow = lh >= 0 ? lh / ROW_ELEMS : -1;
                    const int lim = lh - lrow * ROW_ELEMS - lane * VEC;  // row lrow: this lane's elements j >= lim count
#pragma unroll 1
                    for (int rr = lrow > 0 ? lrow : 0; rr < ROWS; ++rr) {
                        const int64_t q0 = ch * CHUNK + rr * ROW_ELEMS + lane * VEC;
                        TIn x[VEC];
                        if (w) {
                            unpack<TIn>(lds256<(sizeof(TIn) == 8)>(sb + q0), x);
                        } else {
#pragma unroll
                            for (int j = 0; j < VEC; ++j) {
                                const int64_t pos = p0 + q0 + j;
                                x[j] = (pos >= a.lo && pos < a.hi) ? in[pos] : (TIn)0;
                            }
                        }
                        if (rr == lrow) {
#pragma unroll
                            for (int j = 0; j < VEC; ++j)
                                if (j < lim) x[j] = (TIn)0;
                        }
                        A v[VEC];
#pragma unroll
                        for (int j = 0; j < VEC; ++j) v[j] = (A)x[j];
#pragma unroll
                        for (int d = 1; d < VEC; d <<= 1)
#pragma unroll
                            for (int j = 0; j + d < VEC; j += 2 * d) v[j] += v[j + d];
                        acc += v[0];
                    }
                    acc = warp_sum(acc);
                }
                if (lane == 0) {
                    chunk_tot[b * MAXC + ch] = acc;
                    chunk_f[b * MAXC + ch] = lh >= 0;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_sync(BAR_RED, RT);
            if (rw == 0 && lane == 0) {
                Pair t{(A)0, 0u};
                for (int64_t ch = 0; ch < NCHUNK; ++ch) t = seg_combine(t, Pair{chunk_tot[b * MAXC + ch], chunk_f[b * MAXC + ch]});
                st_desc(a.desc + r * G + c, want | ST_A | (t.f ? SEG_FLAG : 0ull), acc_to_bits<A>(t.v));
                SEG_TRACE(r, 2);
                mbar_arrive(&red[b]);
            }
            named_sync(BAR_RED, RT);
        }
        return;
    }

    if (warp == W_LEDGER) {
        // ============================ ledger =====================================
        if constexpr (SUB) {
            // plain carries as the 1-D stream kernel, plus the running sum before the last
            // head seen so far (B), region by region.  Lane l holds GATHER_LP *consecutive*
            // portions (l * GATHER_LP + i): their in-lane prefix plus ONE warp scan of the lane
            // totals gives S at the start of every portion; the three lookups (this CTA's
            // portion, the last head-holding portion before it, the region's last one) go
            // through a small shared array.  (The first version kept portions lane + 32 i and
            // took four masked sums with butterfly reductions plus per-group shuffles: ~300
            // dependent instructions, 1.3-1.5 us per region -- the kernel's critical loop.)
            constexpr int LP = GATHER_LP;
            A carry = (A)0, bcarry = (A)0;
            ulonglong2 dn[LP], dh[LP];
            auto issue = [&](int64_t r) {
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    const int j = lane + 32 * i;  // coalesced polls; transposed through shared memory below
                    if (j < G) ld_desc_pair(a.desc + 2 * (r * G + j), dn[i], dh[i]);
                }
            };
            issue(0);
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                SEG_WAIT(&red[b], par(r));
                if (lane == 0) SEG_TRACE(r, 3);
                // chunks of this portion: exclusive prefix of the sums, and per chunk the
                // portion-relative S before the last head of an earlier chunk
                const A ct = lane < NCHUNK ? chunk_tot[b * MAXC + lane] : (A)0;
                const uint32_t cf = lane < NCHUNK ? chunk_f[b * MAXC + lane] : 0u;
                const A cpl = lane < NCHUNK ? chunk_plh[b * MAXC + lane] : (A)0;
                A cinc = ct;
#pragma unroll
                for (int d = 1; d < NCHUNK; d <<= 1) {  // lanes >= NCHUNK hold nothing anyone reads
                    const A y = shfl_up(cinc, d);
                    if (lane >= d) cinc += y;
                }
                const A cex = cinc - ct;
                const uint32_t cfb = __ballot_sync(FULL, cf != 0u);
                const uint32_t cbelow = cfb & ((1u << lane) - 1u);
                const A chead = shfl_idx(cex + cpl, cbelow ? 31 - __clz((int)cbelow) : 0);
                // the region's G portion totals and head infos
                {
                    unsigned pending = 0;
#pragma unroll
                    for (int i = 0; i < LP; ++i)
                        if (lane + 32 * i < G) pending |= 1u << i;
                    while (true) {
#pragma unroll
                        for (int i = 0; i < LP; ++i)
                            if (((pending >> i) & 1) && (dn[i].x & ~3ull) == want && (dn[i].x & 3ull) != 0 &&
                                (dh[i].x & ~(3ull | SEG_FLAG)) == want && (dh[i].x & 3ull) != 0)
                                pending &= ~(1u << i);
                        if (!__any_sync(FULL, pending != 0)) break;
                        __nanosleep(PS_SEG_POLL_NS);
#pragma unroll
                        for (int i = 0; i < LP; ++i)
                            if ((pending >> i) & 1) ld_desc_pair(a.desc + 2 * (r * G + lane + 32 * i), dn[i], dh[i]);
                    }
                }
                if (lane == 0) SEG_TRACE(r, 4);
                // transpose: lane l takes the LP consecutive portions l * LP + i
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    const int j = lane + 32 * i;
                    led_S[j] = j < G ? acc_from_bits<A>(dn[i].y) : (A)0;
                    led_H[j] = j < G ? acc_from_bits<A>(dh[i].y) : (A)0;
                    led_F[j] = j < G && (dh[i].x & SEG_FLAG) ? 1u : 0u;
                }
                __syncwarp();
                A sbef[LP], hv[LP];  // in-lane: sum of the lane's portions before i; sum before portion i's last head
                A run = (A)0;
                int best1 = -1, best2 = -1;  // last head-holding portion before c / of the region, among this lane's
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    const int j = lane * LP + i;
                    sbef[i] = run;
                    run += led_S[j];
                    hv[i] = led_H[j];
                    if (led_F[j]) {
                        best2 = j;
                        if (j < c) best1 = j;
                    }
                }
                __syncwarp();
#if PS_SEG_EARLY_ISSUE
                if (r + 1 < a.rounds) issue(r + 1);
#endif
                const A incl = warp_scan_pred(run);
                const A excl = incl - run, s_all = shfl_idx(incl, 31);
                const int j1 = __reduce_max_sync(FULL, best1), j2 = __reduce_max_sync(FULL, best2);
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    const A sp = excl + sbef[i];  // S (region-relative) at the start of portion l * LP + i
                    led_S[lane * LP + i] = sp;
                    led_H[lane * LP + i] = sp + hv[i];
                }
                __syncwarp();
                const A mine_pre = led_S[c], run_all = s_all;
                const bool has_before = j1 >= 0, has_last = j2 >= 0;
                const A head_before = has_before ? led_H[j1] : (A)0, head_last = has_last ? led_H[j2] : (A)0;
                const A s_start = carry + mine_pre;                        // S at this portion's start
                const A b_in = has_before ? carry + head_before : bcarry;  // B entering this portion
                if (lane < NCHUNK) {
                    chunk_pre[b * MAXC + lane] = s_start + cex;
                    chunk_B[b * MAXC + lane] = cbelow ? s_start + chead : b_in;
                }
                if (has_last) bcarry = carry + head_last;
                carry += run_all;
                __syncwarp();
                if (lane == 0) SEG_TRACE(r, 5);
                if (lane == 0) mbar_arrive(&pre[b]);
#if !PS_SEG_EARLY_ISSUE
                // the next region's gather only now: its pending loads would hold the scoreboards
                // the fold's shuffles wait on (measured: the fold then takes one L2 round trip)
                if (r + 1 < a.rounds) issue(r + 1);
#endif
            }
            return;
        }
        A carry = (A)0;  // the open segment's running sum at the region start
        ulonglong2 dn[GATHER_LP];
        desc_issue(dn, a.desc, G, lane);
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            SEG_WAIT(&red[b], par(r));
            if (lane == 0) SEG_TRACE(r, 3);
            // chunk aggregates of this portion: exclusive segmented scan across lanes
            const Pair cp = lane < NCHUNK ? Pair{chunk_tot[b * MAXC + lane], chunk_f[b * MAXC + lane]} : Pair{(A)0, 0u};
            const Pair cinc = seg_warp_scan(cp, lane);
            Pair cex = seg_shfl_up(cinc, 1);
            if (lane == 0) cex = Pair{(A)0, 0u};
            // the region's G portion aggregates (flag-masked tag compare)
            {
                unsigned pending = 0;
#pragma unroll
                for (int i = 0; i < GATHER_LP; ++i)
                    if (lane + 32 * i < G) pending |= 1u << i;
                while (true) {
#pragma unroll
                    for (int i = 0; i < GATHER_LP; ++i)
                        if (((pending >> i) & 1) && (dn[i].x & ~(3ull | SEG_FLAG)) == want && (dn[i].x & 3ull) != 0)
                            pending &= ~(1u << i);
                    if (!__any_sync(FULL, pending != 0)) break;
                    __nanosleep(PS_SEG_POLL_NS);
#pragma unroll
                    for (int i = 0; i < GATHER_LP; ++i)
                        if ((pending >> i) & 1) dn[i] = ld_desc(a.desc + r * G + lane + 32 * i);
                }
            }
            if (lane == 0) SEG_TRACE(r, 4);
            Pair gp[GATHER_LP];
#pragma unroll
            for (int i = 0; i < GATHER_LP; ++i)
                gp[i] = (lane + 32 * i < G) ? Pair{acc_from_bits<A>(dn[i].y), (dn[i].x & SEG_FLAG) ? 1u : 0u}
                                            : Pair{(A)0, 0u};
#if PS_SEG_EXP == 1
#pragma unroll
            for (int i = 0; i < GATHER_LP; ++i) gp[i].f = 0;
#endif
            if (r + 1 < a.rounds) desc_issue(dn, a.desc + (r + 1) * G, G, lane);
            // segmented scan of the G aggregates in portion order: per group of 32, then groups
            Pair run{(A)0, 0u}, mine{(A)0, 0u};
#pragma unroll
            for (int i = 0; i < GATHER_LP; ++i) {
                if (32 * i >= G) break;
                const Pair inc = seg_warp_scan(gp[i], lane);
                Pair ex = seg_shfl_up(inc, 1);
                if (lane == 0) ex = Pair{(A)0, 0u};
                const Pair before = seg_combine(run, ex);
                if ((c >> 5) == i) mine = before;                     // lane (c & 31) holds this CTA's prefix
                run = seg_combine(run, Pair{shfl_idx(inc.v, 31), __shfl_sync(FULL, inc.f, 31)});
            }
            const Pair cta_ex{shfl_idx(mine.v, c & 31), __shfl_sync(FULL, mine.f, c & 31)};
            const A portion_in = cta_ex.f ? cta_ex.v : carry + cta_ex.v;
            if (lane < NCHUNK) chunk_pre[b * MAXC + lane] = cex.f ? cex.v : portion_in + cex.v;
            carry = run.f ? run.v : carry + run.v;
            __syncwarp();
            if (lane == 0) SEG_TRACE(r, 5);
            if (lane == 0) mbar_arrive(&pre[b]);
        }
        return;
    }

    // ============================== scanners =======================================
    const uint64_t pol = policy_evict_first();
    A *tot = EMIT ? reinterpret_cast<A *>(a.totals) : nullptr;
    for (int64_t r = 0; r < a.rounds; ++r) {
        const int b = (int)(r % NBUF);
        SEG_WAIT(&full[b], par(r));
        SEG_WAIT(&hdr[b], par(r));
        const TIn *sb = buf + (size_t)b * P;
        const uint32_t *bm = bitmap + b * BMW;
        const int32_t *cb = cntb + b * WORDS;
        const int64_t p0 = p0_of(r);
        const bool w = whole(r);
        if (w || live(r)) {
            const Meta &m = meta[b];  // in shared memory (no local copy)
            // one lane-row's outputs and, at every head it holds, the total of the segment
            // that ends just before it (inc[j-1], or the lane's incoming value at j = 0);
            // the last segment of the input ends at the head at hi (the offset n), which is
            // inside a boundary portion or, when hi ends a portion, handled by its last lane
            auto store_row = [&](int64_t q0, const TOut (&y)[VEC]) {
                if (PS_SEG_EXP == 13 && a.exclusive != 77) return;  // ablation: no output stores
                if (w) {
                    constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
                    for (int k = 0; k < NV; ++k)
                        stg256_policy(out + p0 + q0 + k * (32 / sizeof(TOut)), pack<TOut>(&y[k * (32 / sizeof(TOut))]),
                                      pol);
                } else {
#pragma unroll
                    for (int j = 0; j < VEC; ++j) {
                        const int64_t pos = p0 + q0 + j;
                        if (pos >= a.lo && pos < a.hi) out[pos] = y[j];
                    }
                }
            };
            auto emit_totals = [&](int64_t q0, uint32_t hbits, const A (&inc)[VEC], A lane_prev) {
                uint32_t heads = hbits;
                // warp-uniform loop over the (usually single) head of each lane; the value is
                // picked by selects (static register indices)
                while (__any_sync(FULL, heads != 0u)) {
                    const int j = heads ? __ffs((int)heads) - 1 : 0;
                    A v = lane_prev;
#pragma unroll
                    for (int jj = 1; jj < VEC; ++jj)
                        if (jj == j) v = inc[jj - 1];
                    if (heads) {
                        const int64_t x = q0 + j;  // portion position of the head
                        int64_t sg;
                        if (!m.dup) {
                            sg = m.lb0 + cb[x >> 5] + __popc(bm[x >> 5] & ((1u << (x & 31)) - 1u)) - 1;
                        } else {
                            const int64_t e = p0 + x - a.lead;  // repeated offsets: lower bound by search
                            int64_t l = m.lb0, h = m.lb1;
                            while (l < h) {
                                const int64_t mid = (l + h) >> 1;
                                if (__ldg(a.offsets + mid) >= e) h = mid;
                                else l = mid + 1;
                            }
                            sg = l - 1;
                        }
                        if (sg >= 0) tot[sg] = v;
                    }
                    heads &= heads - 1u;
                }
            };
            // the input's last segment when hi ends this portion: its total is the last element's value
            const bool tail_tot = tot && p0 + P == a.hi && m.next_head;
            auto emit = [&](int64_t q0, uint32_t hbits, const A (&inc)[VEC], const TOut (&y)[VEC], A lane_prev) {
                store_row(q0, y);
                if constexpr (EMIT) {
                    if (!tot) return;
                    emit_totals(q0, hbits, inc, lane_prev);
                    if (tail_tot && q0 + VEC == P) tot[m.lb1 - 1] = inc[VEC - 1];
                }
            };
            for (int64_t ch = warp; ch < NCHUNK; ch += SW) {
                const int64_t c0 = ch * CHUNK;
                uint32_t hb[ROWS];
                if constexpr (SUB) {
                    // one row at a time (a rolled loop: the kernel's hot code has to fit the
                    // SM's instruction cache, see DESIGN): the plain in-lane and warp prefix sums
                    // of the 1-D stream kernel give S; a row without heads (a bit of the head
                    // warp's row mask: most rows unless segments are short) subtracts one base B
                    // for the whole row; a row with heads finds each element's base -- S before
                    // the last head at or before it.  Whole portions (all but the array's two
                    // ends) run a copy of the loop without any bounds logic.
                    if (warp == 0 && lane == 0 && ch == warp) SEG_TRACE(r, 6);
                    SEG_WAIT(&pre[b], par(r));  // the chunk's S and B (the ledger)
                    auto sub_rows = [&](auto whole_c) {
                        constexpr bool W = decltype(whole_c)::value;
                        A base = chunk_pre[b * MAXC + ch], bin = chunk_B[b * MAXC + ch];
                        const int one = a.one;
                        const uint32_t rh = PS_SEG_EXP == 12 ? 0u : row_heads[b] >> (ch * ROWS);
                        auto put = [&](int64_t q0, const TOut (&y)[VEC]) {
                            if constexpr (W) {
                                if (PS_SEG_EXP == 13 && a.exclusive != 77) return;  // ablation: no output stores
                                constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
                                for (int k = 0; k < NV; ++k)
                                    stg256_policy(out + p0 + q0 + k * (32 / sizeof(TOut)),
                                                  pack<TOut>(&y[k * (32 / sizeof(TOut))]), pol);
                            } else {
                                store_row(q0, y);
                            }
                        };
#pragma unroll SEG_UNROLL
                        for (int rr = 0; rr < ROWS; ++rr) {
                            const int64_t q0 = c0 + rr * ROW_ELEMS + lane * VEC;
                            TIn x[VEC];
                            if constexpr (W) {
                                unpack<TIn>(lds256<(sizeof(TIn) == 8)>(sb + q0), x);
                            } else {
#pragma unroll
                                for (int j = 0; j < VEC; ++j) {
                                    const int64_t pos = p0 + q0 + j;
                                    x[j] = (pos >= a.lo && pos < a.hi) ? in[pos] : (TIn)0;
                                }
                            }
                            A p[VEC];  // in-lane inclusive prefix
                            p[0] = (A)x[0];
#pragma unroll
                            for (int j = 1; j < VEC; ++j) p[j] = add_widen(p[j - 1], x[j], one);
                            const A sc = PS_SEG_EXP == 14 ? p[VEC - 1] * (lane + 1) : warp_scan_pred(p[VEC - 1]);  // 14: ablation
                            const A exs = sc - p[VEC - 1], rts = PS_SEG_EXP == 14 ? sc + lane : shfl_idx(sc, 31);
                            TOut y[VEC];
                            if (!((rh >> rr) & 1u)) {
                                const A d = base + exs - bin;  // the open segment's sum before this lane
                                if (a.exclusive) {
                                    y[0] = (TOut)d;
#pragma unroll
                                    for (int j = 1; j < VEC; ++j) y[j] = (TOut)(d + p[j - 1]);
                                } else {
#pragma unroll
                                    for (int j = 0; j < VEC; ++j) y[j] = (TOut)(d + p[j]);
                                }
                                put(q0, y);
                                if constexpr (EMIT)
                                    if (tail_tot && q0 + VEC == P) tot[m.lb1 - 1] = d + p[VEC - 1];
                            } else {
                                const uint32_t hbr = heads_at(bm, q0);
                                const uint32_t bh = __ballot_sync(FULL, hbr != 0u);
                                // o[j]: the sum since the lane's last head at or before j (since the
                                // lane's start before its first head); pb: the lane's sum before its last head
                                A pb = (A)0, o[VEC];
                                o[0] = p[0];
#pragma unroll
                                for (int j = 1; j < VEC; ++j) {
                                    if ((hbr >> j) & 1u) pb = p[j - 1];
                                    o[j] = p[j] - pb;
                                }
                                const A hrel = exs + pb;  // row-relative S before this lane's last head
                                const uint32_t below = bh & ((1u << lane) - 1u);
                                const A hsrc = shfl_idx(hrel, below ? 31 - __clz((int)below) : lane);
                                const A Bl = below ? base + hsrc : bin;
                                const A d = base + exs - Bl;
                                A inc[VEC];
                                uint32_t seen = 0;
#pragma unroll
                                for (int j = 0; j < VEC; ++j) {
                                    seen |= (hbr >> j) & 1u;
                                    inc[j] = seen ? o[j] : d + p[j];
                                }
                                if (a.exclusive) {
#pragma unroll
                                    for (int j = 0; j < VEC; ++j)
                                        y[j] = ((hbr >> j) & 1u) ? (TOut)0 : (TOut)(j == 0 ? d : inc[j - 1]);
                                } else {
#pragma unroll
                                    for (int j = 0; j < VEC; ++j) y[j] = (TOut)inc[j];
                                }
                                put(q0, y);
                                if constexpr (EMIT) {
                                    if (tot) {
                                        emit_totals(q0, hbr, inc, d);
                                        if (tail_tot && q0 + VEC == P) tot[m.lb1 - 1] = inc[VEC - 1];
                                    }
                                }
                                bin = base + shfl_idx(hrel, 31 - __clz((int)bh));
                            }
                            base += rts;
                        }
                    };
#if PS_SEG_WSPLIT
                    if (w) sub_rows(std::true_type{});
                    else sub_rows(std::false_type{});
#else
                    sub_rows(std::false_type{});
#endif
                    continue;
                }
                // floats: one row at a time (rolled: the hot loops of all roles have to fit the
                // instruction cache -- the unrolled form of this loop thrashed it, 1.7 stall
                // cycles per issue waiting for instructions).  A row without heads is the plain
                // scan of the 1-D kernel on top of the open segment's running sum; a row with
                // heads runs the (flag, value) pair operator
                if (warp == 0 && lane == 0 && ch == warp) SEG_TRACE(r, 6);
                SEG_WAIT(&pre[b], par(r));  // the chunk carries of region r (the ledger)
                A base = chunk_pre[b * MAXC + ch];
                const uint32_t rh = row_heads[b] >> (ch * ROWS);
#pragma unroll 1
                for (int rr = 0; rr < ROWS; ++rr) {
                    const int64_t q0 = c0 + rr * ROW_ELEMS + lane * VEC;
                    TIn x[VEC];
                    if (w) {
                        unpack<TIn>(lds256<(sizeof(TIn) == 8)>(sb + q0), x);
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) {
                            const int64_t pos = p0 + q0 + j;
                            x[j] = (pos >= a.lo && pos < a.hi) ? in[pos] : (TIn)0;
                        }
                    }
                    A v[VEC], inc[VEC];
                    TOut y[VEC];
                    if (!((rh >> rr) & 1u)) {
                        v[0] = (A)x[0];
#pragma unroll
                        for (int j = 1; j < VEC; ++j) v[j] = v[j - 1] + (A)x[j];
                        A sc = v[VEC - 1];
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const A t = shfl_up(sc, d);
                            if (lane >= d) sc += t;
                        }
                        A exs = shfl_up(sc, 1);
                        if (lane == 0) exs = (A)0;
                        const A lane_in = base + exs;
#pragma unroll
                        for (int j = 0; j < VEC; ++j) inc[j] = lane_in + v[j];
                        if (a.exclusive) {
                            y[0] = (TOut)lane_in;
#pragma unroll
                            for (int j = 1; j < VEC; ++j) y[j] = (TOut)inc[j - 1];
                        } else {
#pragma unroll
                            for (int j = 0; j < VEC; ++j) y[j] = (TOut)inc[j];
                        }
                        store_row(q0, y);
                        if constexpr (EMIT)
                            if (tail_tot && q0 + VEC == P) tot[m.lb1 - 1] = inc[VEC - 1];
                        base += shfl_idx(sc, 31);
                    } else {
                        const uint32_t hbr = heads_at(bm, q0);
                        // in-lane segmented prefix: v[j] = sum since the last head at or before j
                        // (or since the lane's first element if there is none)
                        A run = (A)0;
#pragma unroll
                        for (int j = 0; j < VEC; ++j) {
                            run = ((hbr >> j) & 1u) ? (A)x[j] : run + (A)x[j];
                            v[j] = run;
                        }
                        const Pair pinc = seg_warp_scan(Pair{run, hbr != 0u}, lane);
                        Pair ex = seg_shfl_up(pinc, 1);
                        if (lane == 0) ex = Pair{(A)0, 0u};
                        const Pair rt{shfl_idx(pinc.v, 31), __shfl_sync(FULL, pinc.f, 31)};
                        const A lane_in = ex.f ? ex.v : base + ex.v;  // sum before the lane's first element
                        uint32_t seen = 0;
#pragma unroll
                        for (int j = 0; j < VEC; ++j) {
                            seen |= (hbr >> j) & 1u;
                            inc[j] = seen ? v[j] : lane_in + v[j];
                        }
                        if (a.exclusive) {
#pragma unroll
                            for (int j = 0; j < VEC; ++j)
                                y[j] = ((hbr >> j) & 1u) ? (TOut)0 : (TOut)(j == 0 ? lane_in : inc[j - 1]);
                        } else {
#pragma unroll
                            for (int j = 0; j < VEC; ++j) y[j] = (TOut)inc[j];
                        }
                        emit(q0, hbr, inc, y, lane_in);
                        base = rt.f ? rt.v : base + rt.v;
                    }
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (warp == 0 && lane == 0) SEG_TRACE(r, 7);
        if (lane == 0) mbar_arrive(&freeb[b]);
    }
}

}  // namespace ps
