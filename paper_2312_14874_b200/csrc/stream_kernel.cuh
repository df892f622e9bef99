// stream_kernel.cuh -- shared-memory-resident regions: the partitioned
// accumulate-scan with each CTA's partition held on chip between its two
// passes.
//
// The reference's cache-partitioned scheme (PAPER.md s2.2, engine.py:278-344)
// reads every partition twice, relying on the cache to make the second read
// cheap.  On the B200 the aggregate shared memory of 148 SMs (~30 MB) is the
// cache we control exactly: a region is sized so that every CTA's portion fits
// in shared memory several times over, the portion is loaded ONCE from HBM by
// TMA bulk copies, reduced and scanned from shared memory, and written once --
// one read and one write per element, no L2 re-read that could miss.
//
// Warp roles of one persistent CTA per SM (cooperative launch):
//   producer warp   TMA bulk copies of region r into buffer r % NBUF once the
//                   scanners have released it (mbarrier `free`)
//   RWP reducers    per-chunk totals from shared memory, portion total -> the
//                   region's global ledger (16-byte epoch-tagged descriptors)
//   ledger warp     all G portion totals of region r -> per-chunk carries
//                   (fixed summation order: identical on every CTA)
//   SW scanners     chunk scans out of shared memory with known carries,
//                   256-bit streaming stores; release the buffer
// NBUF buffers let the producer run up to NBUF-1 regions ahead, which hides
// the grid-wide ledger exchange behind HBM streaming.
#pragma once

#include "rounds_kernel.cuh"

#ifndef PS_COPY_DEPTH  // copy_in: regions whose element-wise copies are in flight per reducer warp
#define PS_COPY_DEPTH 3
#endif

namespace ps {

struct StreamArgs {
    const void *in;   // aligned base: position p <-> element p - lead
    void *out;
    int64_t lo, hi;   // valid positions
    int64_t portion;  // positions per CTA per region (multiple of SW * CHUNK)
    int64_t rounds;   // regions
    uint64_t seed_bits;
    const void *seed_terms;
    int64_t n_seed_terms;
    void *total;
    ulonglong2 *desc;  // rounds * G descriptors
    uint32_t epoch;
    int exclusive;
    int inflight;      // producer: at most this many regions' loads outstanding (0: NBUF)
    int copy_in;       // 1: the producer warp copies portions with element-sized loads (input not TMA-alignable)
    Stall stall;       // stress tests: stall injection at every role hand-off
    Mailbox mail;      // seed += totals published by the ranks before this one
};

template <typename TIn, int SW, int ROWS, int NBUF, int RWP>
struct StreamGeom {
    static constexpr int WARPS = SW + RWP + 2;
    static constexpr int THREADS = WARPS * 32;
    static constexpr int VEC = 32 / sizeof(TIn);
    static constexpr int ROW_ELEMS = 32 * VEC;
    static constexpr int CHUNK = ROWS * ROW_ELEMS;  // one warp's unit (ROWS KiB)
    static constexpr int MAXC = 16;                 // chunks per portion (32 KiB portions hold 8)
    static constexpr int BUF_BYTES_MAX = 224 * 1024;
    static constexpr int SMEM_FIXED = 4 * NBUF * 8 + 2 * NBUF * MAXC * 8 + NBUF * MAXC * 4 + 128;
    static constexpr int smem(int64_t portion) { return (int)(NBUF * portion * sizeof(TIn)) + SMEM_FIXED; }
};

// widen a warp chunk to the accumulator type.  (A shift-and-rebias float32 ->
// float64 on the integer pipes, with an F2F fallback for zero/subnormal/inf/nan
// chunks, measured 16 % slower than F2F here: scripts/stream_variants.cu.)
template <typename TIn, typename A, int ROWS, int VEC>
__device__ __forceinline__ void widen_chunk(const V256 (&raw)[ROWS], A (&v)[ROWS][VEC]) {
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) {
        TIn x[VEC];
        unpack<TIn>(raw[rr], x);
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[rr][j] = (A)x[j];
    }
}

// Ledger gather with its round trip overlapped.  One grid-wide gather of a
// region's G descriptors is one L2 round trip (~1-1.3 us under full HBM load,
// scripts/trace_stream.cu), and the ledger warp's per-region chain -- gather,
// fold, hand-off -- sets the kernel's region rate whenever the reducers run
// ahead of it.  So the loads of region r+1 are issued as soon as region r's have
// arrived (the totals are normally published by then) and the chunk-total scan,
// which needs only this CTA's reducers, runs while they are in flight: the
// chain per region is one round trip (integer data; see the ledger for float32).
// Issuing gathers further ahead was slower: polls that return before the totals
// are published cost a full extra round trip each (measured 8-25 % slower at
// 2-3 regions ahead).
constexpr int GATHER_LP = 5;  // descriptors per lane: the stream kernel runs with G <= 160 CTAs

__device__ __forceinline__ void desc_issue(ulonglong2 (&d)[GATHER_LP], const ulonglong2 *base, int G, int lane) {
#pragma unroll
    for (int i = 0; i < GATHER_LP; ++i)
        if (lane + 32 * i < G) d[i] = ld_desc(base + lane + 32 * i);
}

// poll until every descriptor of the region carries this launch's tag
__device__ __forceinline__ void desc_wait(ulonglong2 (&d)[GATHER_LP], const ulonglong2 *base, int G, uint64_t want,
                                          int lane) {
    unsigned pending = 0;
#pragma unroll
    for (int i = 0; i < GATHER_LP; ++i)
        if (lane + 32 * i < G) pending |= 1u << i;
    while (true) {
#pragma unroll
        for (int i = 0; i < GATHER_LP; ++i)
            if (((pending >> i) & 1) && (d[i].x & ~3ull) == want && (d[i].x & 3ull) != 0) pending &= ~(1u << i);
        if (!__any_sync(FULL, pending != 0)) break;
        __nanosleep(32);
#pragma unroll
        for (int i = 0; i < GATHER_LP; ++i)
            if ((pending >> i) & 1) d[i] = ld_desc(base + lane + 32 * i);
    }
}

// float32 -> float32 scanner body with FP32-pipe arithmetic only (F32PAIR).  The
// reference rounds every output from a float64 running sum (core.py:86-92); the
// exact path (F32PAIR = false) does the same per element -- two float<->double
// conversions on the XU pipe plus float64 adds, which made cfg2 issue/latency-
// bound at 0.85 of the HBM roofline (profiles/r01_cfg2_full.md: XU 35 %).  Here
// the in-lane and warp scans of a chunk run in float32 (the reference's own
// horizontal_scan rounds its blocks in the element dtype, simd.py:84-98), and
// the carry -- float64 from the ledger -- is split once per chunk into a float
// pair hi + lo (48-bit significand), advanced row by row with TwoSum and
// applied per element as hi + (lo' + p): two float adds per element, no
// conversion.  Error against float32(cumsum(float64)): the in-chunk partial p
// (<= 1024 elements, a 13-add tree/chain) plus one rounding of the output;
// measured <= 3e-7 relative on the BASELINE cfg2 input (tests: <= 1e-6).
// part 1 (before the carry is known): in-lane and warp-inclusive scans in float32
template <int ROWS, int VEC>
__device__ __forceinline__ void f32pair_prescan(float (&x)[ROWS][VEC], float (&sc)[ROWS], int lane) {
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
        for (int j = 1; j < VEC; ++j) x[rr][j] = __fadd_rn(x[rr][j], x[rr][j - 1]);
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) sc[rr] = x[rr][VEC - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) {
            const float y = __shfl_up_sync(FULL, sc[rr], d);
            if (lane >= d) sc[rr] = __fadd_rn(sc[rr], y);
        }
    }
}

// part 2: the float64 chunk carry as a float pair, applied row by row
template <int ROWS, int VEC, typename Emit>
__device__ __forceinline__ void f32pair_apply(const float (&x)[ROWS][VEC], const float (&sc)[ROWS], double base,
                                              int lane, int exclusive, Emit &&emit) {
    float hi = __double2float_rn(base);
    float lo = __double2float_rn(base - (double)hi);
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) {
        float exs = __shfl_up_sync(FULL, sc[rr], 1);
        if (lane == 0) exs = 0.f;
        const float rt = __shfl_sync(FULL, sc[rr], 31);
        const float l1 = __fadd_rn(lo, exs);  // this lane's offset folded into the low word
        float y[VEC];
        if (exclusive) {
            y[0] = __fadd_rn(hi, l1);
#pragma unroll
            for (int j = 1; j < VEC; ++j) y[j] = __fadd_rn(hi, __fadd_rn(l1, x[rr][j - 1]));
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) y[j] = __fadd_rn(hi, __fadd_rn(l1, x[rr][j]));
        }
        emit(rr, y);
        // (hi, lo) += row total: TwoSum, then renormalise
        const float s = __fadd_rn(hi, rt);
        const float bp = __fsub_rn(s, hi);
        const float e = __fadd_rn(__fsub_rn(hi, __fsub_rn(s, bp)), __fsub_rn(rt, bp));
        const float l2 = __fadd_rn(lo, e);
        hi = __fadd_rn(s, l2);
        lo = __fsub_rn(l2, __fsub_rn(hi, s));
    }
}

// Reducer row sums of the float-pair kernel.  PS_F32_RED 0: the float32 TwoSum tree
// (lane_row_sum, ~6 FP32 ops per element); 1: float64 tree (one F2F on the XU pipe +
// one DADD per element -- the float-pair scanners leave the XU pipe free).
#ifndef PS_F32_RED
#define PS_F32_RED 1
#endif
template <typename TIn, typename A, int VEC, bool F32PAIR>
__device__ __forceinline__ A reducer_row_sum(const TIn (&x)[VEC]) {
    if constexpr (F32PAIR && PS_F32_RED == 1) {
        A v[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = (A)x[j];
#pragma unroll
        for (int d = 1; d < VEC; d <<= 1)
#pragma unroll
            for (int j = 0; j + d < VEC; j += 2 * d) v[j] += v[j + d];
        return v[0];
    } else {
        return lane_row_sum<TIn, A, VEC>(x);
    }
}

template <typename TIn, typename TOut, int SW, int ROWS, int NBUF, int RWP, bool STALL = false, int MINB = 1,
          bool F32PAIR = false>
__global__ void __launch_bounds__((SW + RWP + 2) * 32, MINB) scan_stream_kernel(const StreamArgs a) {
    using Geo = StreamGeom<TIn, SW, ROWS, NBUF, RWP>;
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = Geo::VEC, ROW_ELEMS = Geo::ROW_ELEMS, CHUNK = Geo::CHUNK, MAXC = Geo::MAXC;
    constexpr bool FLOAT = (A)0.5 != (A)0;
    constexpr int RT = RWP * 32;
    constexpr int BAR_RED = 1;
    constexpr int W_PROD = SW + RWP, W_LEDGER = SW + RWP + 1;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    TIn *buf = reinterpret_cast<TIn *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NBUF * a.portion * sizeof(TIn));
    uint64_t *full = bars;             // TMA landed            (1 arrival + tx)
    uint64_t *red = bars + NBUF;       // chunk totals written  (1)
    uint64_t *pre = bars + 2 * NBUF;   // chunk carries written (1)
    uint64_t *freeb = bars + 3 * NBUF; // scanners released it  (SW)
    A *chunk_tot = reinterpret_cast<A *>(bars + 4 * NBUF);
    A *chunk_pre = chunk_tot + NBUF * MAXC;
    // F32PAIR: per chunk, nonzero if any element has its sign bit set (or the portion
    // is a boundary one) -- such chunks take the float64-per-element path
    uint32_t *chunk_neg = reinterpret_cast<uint32_t *>(chunk_pre + NBUF * MAXC);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    TOut *out = reinterpret_cast<TOut *>(a.out);
    const uint64_t want = (uint64_t)a.epoch << 2;
    const int64_t P = a.portion;
    const int64_t nchunk = P / CHUNK;

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], a.copy_in ? RWP : 1);  // copy_in: every reducer warp lands its own chunks
            mbar_init(&red[b], 1);
            mbar_init(&pre[b], 1);
            mbar_init(&freeb[b], SW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // phase of buffer slot b = r % NBUF for region r
    auto par = [&](int64_t r) { return (uint32_t)((r / NBUF) & 1); };
    auto p0_of = [&](int64_t r) { return r * P * G + (int64_t)c * P; };
    auto whole = [&](int64_t r) {
        const int64_t p0 = p0_of(r);
        return p0 >= a.lo && p0 + P <= a.hi;
    };
    auto live = [&](int64_t r) {  // anything valid in this portion?
        const int64_t p0 = p0_of(r);
        return p0 + P > a.lo && p0 < a.hi;
    };

    if (warp == W_PROD) {
        // ============================ producer ===================================
        if (a.copy_in) return;  // no bulk copies: the reducer warps fetch their own chunks (below)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                stall_site<STALL>(a.stall, r * G + c, 0, 1);
                if (r >= NBUF) mbar_wait(&freeb[b], par(r - NBUF));
                // bounded loads in flight: an SM's ledger polls return behind its own
                // outstanding TMA data, so six regions issued at start-up would hold
                // the first grid-wide gather back by ~5 us
                if (r >= a.inflight && a.inflight > 0 && a.inflight < NBUF)
                    mbar_wait(&full[(r - a.inflight) % NBUF], par(r - a.inflight));
#ifdef PS_TRACE
                if (g_trace && true) g_trace[(r * G + c) * 8 + 0] = gtimer();
#endif
                if (whole(r)) {
                    constexpr uint32_t PIECE = 16384;
                    const uint32_t bytes = (uint32_t)(P * sizeof(TIn));
                    mbar_expect_tx(&full[b], bytes);
                    const char *src = reinterpret_cast<const char *>(in + p0_of(r));
                    char *dst = reinterpret_cast<char *>(buf + (size_t)b * P);
                    for (uint32_t o = 0; o < bytes; o += PIECE)
                        bulk_g2s(dst + o, src + o, bytes - o < PIECE ? bytes - o : PIECE, &full[b], pol);
                } else {
                    mbar_arrive(&full[b]);  // boundary portion: consumers read global memory
                }
            }
        }
        return;
    }

    if (warp >= SW && warp < W_PROD) {
        // ============================ reducers ===================================
        const int rw = warp - SW;
        // copy_in.  The output's 32-byte phase fixes the tile grid (256-bit stores); an input
        // whose 16-byte phase does not fit that grid cannot be bulk-copied.  Each reducer warp
        // then fetches its own chunks of a portion with element-wise cp.async (LDGSTS: no
        // registers held), D - 1 regions ahead of the one it reduces, into the very layout a
        // bulk copy would leave -- scanners and ledger do not notice.  (Before: such in/out
        // pairs ran on the look-back tiles with scalar accesses, 0.31-0.50 of the peak; one
        // copying warp per SM reached 0.5, its copies in flight being too few.)
        constexpr int D = PS_COPY_DEPTH;
        auto copy_stage = [&](int64_t q) {
            if (q < a.rounds) {
                if (lane == 0 && q >= NBUF) mbar_wait(&freeb[q % NBUF], par(q - NBUF));
                __syncwarp();
                if (whole(q)) {
                    const TIn *src = in + p0_of(q);
                    const uint32_t dst = smem_addr(buf + (size_t)(q % NBUF) * P);
                    for (int64_t ch = rw; ch < nchunk; ch += RWP) {
#pragma unroll 8
                        for (int64_t i = ch * CHUNK + lane; i < (ch + 1) * CHUNK; i += 32)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst + (uint32_t)(i * sizeof(TIn))),
                                         "l"(src + i), "n"(sizeof(TIn))
                                         : "memory");
                    }
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if (a.copy_in)
            for (int64_t q = 0; q < D - 1; ++q) copy_stage(q);
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            if (a.copy_in) {
                copy_stage(r + D - 1);
                asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");  // region r's copies have landed
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[b]);
            }
            mbar_wait(&full[b], par(r));
#ifdef PS_TRACE
                if (g_trace && rw == 0 && lane == 0) g_trace[(r * G + c) * 8 + 1] = gtimer();
#endif
            stall_site<STALL>(a.stall, r * G + c, rw, 2);
            A *tot = chunk_tot + b * MAXC;
            const TIn *sb = buf + (size_t)b * P;
            const int64_t p0 = p0_of(r);
            const bool w = whole(r);
            if (FLOAT && w && nchunk == 2 * RWP) {
                // float data, whole portion, two chunks per reducer warp: both reduced
                // together (the TwoSum reducer is latency-bound next to 8 scanner warps;
                // cfg2 +0.7 %; integer data measured 1 % slower this way)
                const int64_t c0 = rw, c1 = rw + RWP;
                A s0 = (A)0, s1 = (A)0;
                uint64_t sign0 = 0, sign1 = 0;
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) {
                    const V256 r0 = lds256<(sizeof(TIn) == 8)>(sb + c0 * CHUNK + rr * ROW_ELEMS + lane * VEC);
                    const V256 r1 = lds256<(sizeof(TIn) == 8)>(sb + c1 * CHUNK + rr * ROW_ELEMS + lane * VEC);
                    if constexpr (F32PAIR) {
                        sign0 |= r0.w[0] | r0.w[1] | r0.w[2] | r0.w[3];
                        sign1 |= r1.w[0] | r1.w[1] | r1.w[2] | r1.w[3];
                    }
                    TIn x0[VEC], x1[VEC];
                    unpack<TIn>(r0, x0);
                    unpack<TIn>(r1, x1);
                    s0 += reducer_row_sum<TIn, A, VEC, F32PAIR>(x0);
                    s1 += reducer_row_sum<TIn, A, VEC, F32PAIR>(x1);
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    s0 += __shfl_xor_sync(FULL, s0, d);
                    s1 += __shfl_xor_sync(FULL, s1, d);
                }
                if constexpr (F32PAIR) {
                    const bool n0 = __any_sync(FULL, (sign0 & 0x8000000080000000ull) != 0);
                    const bool n1 = __any_sync(FULL, (sign1 & 0x8000000080000000ull) != 0);
                    if (lane == 0) {
                        chunk_neg[b * MAXC + c0] = n0;
                        chunk_neg[b * MAXC + c1] = n1;
                    }
                }
                if (lane == 0) {
                    tot[c0] = s0;
                    tot[c1] = s1;
                }
            } else
            for (int64_t ch = rw; ch < nchunk; ch += RWP) {
                A s = (A)0;
                uint64_t sign = w ? 0 : 0x8000000000000000ull;  // boundary chunks: float64 path
                if (w) {
                    V256 raw[ROWS];
#pragma unroll
                    for (int rr = 0; rr < ROWS; ++rr) raw[rr] = lds256<(sizeof(TIn) == 8)>(sb + ch * CHUNK + rr * ROW_ELEMS + lane * VEC);
#pragma unroll
                    for (int rr = 0; rr < ROWS; ++rr) {
                        TIn x[VEC];
                        if constexpr (F32PAIR) sign |= raw[rr].w[0] | raw[rr].w[1] | raw[rr].w[2] | raw[rr].w[3];
                        unpack<TIn>(raw[rr], x);
                        s += reducer_row_sum<TIn, A, VEC, F32PAIR>(x);
                    }
                } else if (live(r)) {
                    for (int rr = 0; rr < ROWS; ++rr)
                        for (int j = 0; j < VEC; ++j) {
                            const int64_t pos = p0 + ch * CHUNK + rr * ROW_ELEMS + lane * VEC + j;
                            if (pos >= a.lo && pos < a.hi) s += (A)in[pos];
                        }
                }
                s = warp_sum(s);
                if constexpr (F32PAIR) {
                    const bool neg = __any_sync(FULL, (sign & 0x8000000080000000ull) != 0);
                    if (lane == 0) chunk_neg[b * MAXC + ch] = neg;
                }
                if (lane == 0) tot[ch] = s;
            }
            // reads of this buffer are done (their sums are stored); order them before
            // any later TMA refill of the buffer (generic -> async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_sync(BAR_RED, RT);
            if (rw == 0) {
                A t = (A)0;
                for (int64_t ch = lane; ch < nchunk; ch += 32) t += tot[ch];
                t = warp_sum(t);
                stall_site<STALL>(a.stall, r * G + c, 0, 3);
                if (lane == 0) {
                    st_desc(a.desc + r * G + c, want | ST_A, acc_to_bits<A>(t));
                    mbar_arrive(&red[b]);
#ifdef PS_TRACE
                if (g_trace && true) g_trace[(r * G + c) * 8 + 2] = gtimer();
#endif
                }
            }
            // integer data: the reducer warps stay in step.  float data: warps 1.. go on
            // to the next region while warp 0 publishes (tot[] of this buffer is not
            // rewritten before the buffer comes round again; cfg2 +0.7 %, int -0.5 %)
            if constexpr (!FLOAT) named_sync(BAR_RED, RT);
        }
        return;
    }

    if (warp == W_LEDGER) {
        // ============================ ledger =====================================
        A carry;
        {
            A seed = (A)0;
            if (a.seed_terms) {
                const A *st = reinterpret_cast<const A *>(a.seed_terms);
                for (int64_t i = lane; i < a.n_seed_terms; i += 32) seed += st[i];
            }
            carry = acc_from_bits<A>(a.seed_bits) + warp_sum(seed);
            if (a.mail.n) carry += mailbox_sum<A>(a.mail, lane);
        }
        // float data on the float64-per-element scanner: one gather per region on its own
        // turn.  Integer data and the float-pair scanner (F32PAIR): early-issued gathers.
        if constexpr (FLOAT && !F32PAIR) {
            // float32/float64: one gather per region on its own turn, then the fold (the
            // early-issued gather below made cfg2 2.6 % slower: its reducers, not the
            // ledger, set the pace)
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                A sb, sa;
                stall_site<STALL>(a.stall, r * G + c, 0, 4);
#ifdef PS_EXP_NOLEDGER
                sb = sa = (A)0;
#else
#ifdef PS_TRACE
                if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 3] = gtimer();
#endif
                gather_totals<A>(a.desc + r * G, G, c, want, lane, sb, sa);
#ifdef PS_TRACE
                    if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 4] = gtimer();
#endif
#endif

                mbar_wait(&red[b], par(r));  // own chunk totals (and chunk_pre[b] is free, see above)
                const A *tot = chunk_tot + b * MAXC;
                A *pr = chunk_pre + b * MAXC;
                // nchunk <= 64: two chunks per lane, exclusive scan across the warp
                const A t0 = lane * 2 < nchunk ? tot[lane * 2] : (A)0;
                const A t1 = lane * 2 + 1 < nchunk ? tot[lane * 2 + 1] : (A)0;
                const A own = t0 + t1;
                A incl = own;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const A y = shfl_up(incl, dd);
                    if (lane >= dd) incl += y;
                }
                A ex = shfl_up(incl, 1);
                if (lane == 0) ex = (A)0;
                const A base = carry + sb + ex;
                if (lane * 2 < nchunk) pr[lane * 2] = base;
                if (lane * 2 + 1 < nchunk) pr[lane * 2 + 1] = base + t0;
                carry += sa;
                stall_site<STALL>(a.stall, r * G + c, 0, 5);
                __syncwarp();
                if (lane == 0) mbar_arrive(&pre[b]);
#ifdef PS_TRACE
                    if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 5] = gtimer();
#endif
            }
        } else {
            // integer data: the next region's gather is issued as soon as this one's
            // descriptors arrived, and the chunk-total scan runs inside the round trip
            // (int64 2^27 -2.6 %, cfg1 unchanged)
            ulonglong2 dn[GATHER_LP];  // the gather in flight (launcher: G <= 32 * GATHER_LP)
            desc_issue(dn, a.desc, G, lane);
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                stall_site<STALL>(a.stall, r * G + c, 0, 4);
                // exclusive scan of this portion's chunk totals (needs only this CTA's reducers)
                mbar_wait(&red[b], par(r));  // own chunk totals (and chunk_pre[b] is free, see above)
                const A *tot = chunk_tot + b * MAXC;
                A *pr = chunk_pre + b * MAXC;
                // nchunk <= 64: two chunks per lane, exclusive scan across the warp
                const A t0 = lane * 2 < nchunk ? tot[lane * 2] : (A)0;
                const A t1 = lane * 2 + 1 < nchunk ? tot[lane * 2 + 1] : (A)0;
                A incl = t0 + t1;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const A y = shfl_up(incl, dd);
                    if (lane >= dd) incl += y;
                }
                A ex = shfl_up(incl, 1);
                if (lane == 0) ex = (A)0;
                A sb = (A)0, sa = (A)0;
#ifndef PS_EXP_NOLEDGER
#ifdef PS_TRACE
                if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 3] = gtimer();
#endif
                desc_wait(dn, a.desc + r * G, G, want, lane);
#pragma unroll
                for (int i = 0; i < GATHER_LP; ++i) {  // gather_totals' summation order
                    const int j = lane + 32 * i;
                    if (j < G) {
                        const A v = acc_from_bits<A>(dn[i].y);
                        sa += v;
                        if (j < c) sb += v;
                    }
                }
                if (r + 1 < a.rounds) desc_issue(dn, a.desc + (r + 1) * G, G, lane);
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {  // both warp sums in one pass
                    sa += __shfl_xor_sync(FULL, sa, d);
                    sb += __shfl_xor_sync(FULL, sb, d);
                }
#ifdef PS_TRACE
                if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 4] = gtimer();
#endif
#endif
                const A base = carry + sb + ex;
                if (lane * 2 < nchunk) pr[lane * 2] = base;
                if (lane * 2 + 1 < nchunk) pr[lane * 2 + 1] = base + t0;
                carry += sa;
                stall_site<STALL>(a.stall, r * G + c, 0, 5);
                __syncwarp();
                if (lane == 0) mbar_arrive(&pre[b]);
#ifdef PS_TRACE
                if (g_trace && lane == 0) g_trace[(r * G + c) * 8 + 5] = gtimer();
#endif
            }
        }
        if (c == 0 && lane == 0 && a.total) *reinterpret_cast<A *>(a.total) = carry;
        return;
    }

    // ============================== scanners =======================================
    const uint64_t pol = policy_evict_first();
    for (int64_t r = 0; r < a.rounds; ++r) {
        const int b = (int)(r % NBUF);
        // everything that does not need the carry (loads, widening, in-lane and
        // warp scans) runs as soon as the data has landed, overlapping the
        // ledger's grid-wide exchange; only the carry adds and stores wait for it
        mbar_wait(&full[b], par(r));
#ifdef PS_TRACE
                if (g_trace && warp == 0 && lane == 0) g_trace[(r * G + c) * 8 + 6] = gtimer();
#endif
        stall_site<STALL>(a.stall, r * G + c, warp, 6);
        const A *pr = chunk_pre + b * MAXC;
        const TIn *sb = buf + (size_t)b * P;
        const int64_t p0 = p0_of(r);
        const bool w = whole(r);
        if (w || live(r)) {
            for (int64_t ch = warp; ch < nchunk; ch += SW) {
                const int64_t t0 = p0 + ch * CHUNK;
                stall_site<STALL>(a.stall, (r * G + c) * 64 + ch, warp, 7);
                if constexpr (F32PAIR) {
                    static_assert(sizeof(TIn) == 4 && sizeof(TOut) == 4, "F32PAIR: float32 -> float32 only");
                    float x[ROWS][VEC];
                    if (w) {
#pragma unroll
                        for (int rr = 0; rr < ROWS; ++rr)
                            unpack<float>(lds256<false>(sb + ch * CHUNK + rr * ROW_ELEMS + lane * VEC), x[rr]);
                    } else {
#pragma unroll
                        for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
                            for (int j = 0; j < VEC; ++j) {
                                const int64_t pos = t0 + rr * ROW_ELEMS + lane * VEC + j;
                                x[rr][j] = (pos >= a.lo && pos < a.hi) ? (float)in[pos] : 0.f;
                            }
                    }
                    float sc[ROWS];
                    f32pair_prescan<ROWS, VEC>(x, sc, lane);  // before the ledger's carries are known
                    mbar_wait(&pre[b], par(r));
                    const double base = (double)pr[ch];
                    // the float pair is used where it is accurate to ~1e-7 relative: nonnegative
                    // data under a carry >= 64x the chunk's own sum (no cancellation, and the
                    // float32 in-chunk partials are small next to the output).  Any other chunk
                    // -- signed data, the first chunks of a scan -- takes the float64 path below.
                    const bool pair_ok = chunk_neg[b * MAXC + ch] == 0 && base >= 64.0 * (double)chunk_tot[b * MAXC + ch];
                    if (pair_ok) {
                        f32pair_apply<ROWS, VEC>(x, sc, base, lane, a.exclusive, [&](int rr, const float(&y)[VEC]) {
                            if (w) {
                                stg256_policy(out + t0 + rr * ROW_ELEMS + lane * VEC,
                                              pack<TOut>(reinterpret_cast<const TOut *>(y)), pol);
                            } else {
#pragma unroll
                                for (int j = 0; j < VEC; ++j) {
                                    const int64_t pos = t0 + rr * ROW_ELEMS + lane * VEC + j;
                                    if (pos >= a.lo && pos < a.hi) out[pos] = (TOut)y[j];
                                }
                            }
                        });
                        continue;
                    }
                }
                A v[ROWS][VEC];
                if (w) {
                    V256 raw[ROWS];
#pragma unroll
                    for (int rr = 0; rr < ROWS; ++rr) raw[rr] = lds256<(sizeof(TIn) == 8)>(sb + ch * CHUNK + rr * ROW_ELEMS + lane * VEC);
                    widen_chunk<TIn, A, ROWS, VEC>(raw, v);
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
                for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
                    for (int j = 1; j < VEC; ++j) v[rr][j] += v[rr][j - 1];
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
                A exs[ROWS], rts[ROWS];
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) {
                    if constexpr (FLOAT) {
                        exs[rr] = shfl_up(sc[rr], 1);
                        if (lane == 0) exs[rr] = (A)0;
                    } else {
                        exs[rr] = sc[rr] - v[rr][VEC - 1];
                    }
                    rts[rr] = shfl_idx(sc[rr], 31);
                }
                mbar_wait(&pre[b], par(r));  // the chunk carries of region r (the ledger)
                A base = pr[ch];
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) {
                    const A bb = base + exs[rr];
                    base += rts[rr];
                    TOut y[VEC];
                    if (a.exclusive) {
                        y[0] = (TOut)bb;
#pragma unroll
                        for (int j = 1; j < VEC; ++j) y[j] = (TOut)(bb + v[rr][j - 1]);
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) y[j] = (TOut)(bb + v[rr][j]);
                    }
                    if (w) {
                        constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
                        for (int q = 0; q < NV; ++q)
                            stg256_policy(out + t0 + rr * ROW_ELEMS + lane * VEC + q * (32 / sizeof(TOut)),
                                          pack<TOut>(&y[q * (32 / sizeof(TOut))]), pol);
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) {
                            const int64_t pos = t0 + rr * ROW_ELEMS + lane * VEC + j;
                            if (pos >= a.lo && pos < a.hi) out[pos] = y[j];
                        }
                    }
                }
            }
        }
        // every value read from this buffer has been consumed by the stores above
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[b]);
#ifdef PS_TRACE
                if (g_trace && warp == 0 && lane == 0) g_trace[(r * G + c) * 8 + 7] = gtimer();
#endif
    }
}

}  // namespace ps
