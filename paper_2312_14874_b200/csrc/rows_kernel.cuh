// rows_kernel.cuh -- many independent rows (batched scans, cfg4 "delta
// decoding"): every row is owned by one persistent CTA, so no carry ever
// crosses a CTA and nothing is exchanged through global memory.
//
// Reference semantics: the per-chunk scans of the vertical family
// (simd.py:164-206: chunk i scanned independently, seeded with a row seed,
// its running total written out) generalised to `rows` chunks of `cols`
// elements with a row stride.
//
// Per CTA: a producer warp streams (row, segment) work items into a ring of
// NBUF shared-memory buffers with TMA bulk copies; SW scanner warps first
// reduce the segment's chunks (4 KiB each) to totals, exchange them through
// shared memory (one named barrier), then scan their chunks with the carry
// (row seed + earlier segments + earlier chunks) and store with 256-bit
// streaming stores.  Each element is read from HBM once and written once.
#pragma once

#include <type_traits>

#include "stream_kernel.cuh"

namespace ps {

struct RowsArgs {
    const void *in;
    void *out;
    int64_t rows, cols, ld_in, ld_out;  // elements
    const void *row_seeds;              // acc-typed, nullable
    void *row_totals;                   // acc-typed, nullable
    int exclusive;
    int vec_out;                        // output rows are 32-byte aligned
    unsigned long long *ctr;            // [row ticket, producers done], zero between launches;
                                        // null: CTA c takes rows c, c + G, ...
    Stall stall;                        // stress tests: stall injection
};

template <typename TIn, int SW, int RPC, int NBUF, int NCH>
struct RowsGeom {
    static constexpr int THREADS = (SW + 1) * 32;
    static constexpr int VEC = 32 / sizeof(TIn);
    static constexpr int ROW_ELEMS = 32 * VEC;
    static constexpr int CHUNK = RPC * ROW_ELEMS;  // elements per chunk (RPC KiB)
    static constexpr int SEG = NCH * CHUNK;        // elements per work item
    static constexpr int SEG_BYTES = SEG * (int)sizeof(TIn);
    static constexpr int SMEM = NBUF * SEG_BYTES + 2 * NBUF * 8 + NBUF * NCH * 8 + NBUF * 16 + 64;
};

template <typename TIn, typename TOut, int SW, int RPC, int NBUF, int NCH, bool STALL = false>
__global__ void __launch_bounds__((SW + 1) * 32, RPC <= 2 ? 2 : 1) scan_rows_kernel(const RowsArgs a) {
    using Geo = RowsGeom<TIn, SW, RPC, NBUF, NCH>;
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = Geo::VEC, ROW_ELEMS = Geo::ROW_ELEMS, CHUNK = Geo::CHUNK, SEG = Geo::SEG;
    constexpr bool FLOAT = (A)0.5 != (A)0;
    constexpr int BAR_SCAN = 1;
    static_assert(NCH <= 32, "chunk totals are scanned by one warp");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    TIn *buf = reinterpret_cast<TIn *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NBUF * Geo::SEG_BYTES);
    uint64_t *freeb = full + NBUF;
    A *tot = reinterpret_cast<A *>(freeb + NBUF);  // [NBUF][NCH]
    int64_t *item_row = reinterpret_cast<int64_t *>(tot + NBUF * NCH);  // [NBUF]: row of the item (-1: end)
    int64_t *item_seg = item_row + NBUF;                                 // [NBUF]: its segment

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    TOut *out = reinterpret_cast<TOut *>(a.out);
    const int64_t nseg = (a.cols + SEG - 1) / SEG;

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&freeb[b], SW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == SW) {
        // =========================== producer ======================================
        // Rows are taken from a grid-wide ticket when a.ctr is given: an SM that
        // streams faster takes more rows (fixed shares leave the grid waiting for the
        // slowest SMs: scripts/sm_fairness.cu).  The next ticket is fetched while the
        // current row's loads are issued.
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const bool dyn = a.ctr != nullptr;
            int64_t item = 0;
            int64_t r = dyn ? (int64_t)atomicAdd(a.ctr, 1ull) : c;
            while (true) {
                const int64_t rn = r < a.rows ? (dyn ? (int64_t)atomicAdd(a.ctr, 1ull) : r + G) : r;
                for (int64_t sg = 0; sg < nseg; ++sg, ++item) {
                    const int b = (int)(item % NBUF);
                    stall_site<STALL>(a.stall, r, sg, 1);
                    if (item >= NBUF) mbar_wait(&freeb[b], (uint32_t)(((item / NBUF) - 1) & 1));
                    if (r >= a.rows) {  // end marker: the scanners stop at this item
                        item_row[b] = -1;
                        mbar_arrive(&full[b]);
                        break;
                    }
                    item_row[b] = r;
                    item_seg[b] = sg;
                    const int64_t e0 = sg * SEG;
                    const int64_t cnt = (a.cols - e0) < SEG ? (a.cols - e0) : SEG;
                    const uint32_t bytes = (uint32_t)(cnt * sizeof(TIn));
                    mbar_expect_tx(&full[b], bytes);
                    const char *src = reinterpret_cast<const char *>(in + r * a.ld_in + e0);
                    char *dst = reinterpret_cast<char *>(buf + (size_t)b * SEG);
                    for (uint32_t o = 0; o < bytes; o += 16384)
                        bulk_g2s(dst + o, src + o, bytes - o < 16384u ? bytes - o : 16384u, &full[b], pol);
                }
                if (r >= a.rows) break;
                r = rn;
            }
            if (dyn) {
                // the last producer to take its final ticket resets the counters for the
                // next launch on this scratch (stream order makes them visible to it)
                __threadfence();
                if (atomicAdd(a.ctr + 1, 1ull) == (unsigned long long)(G - 1)) {
                    a.ctr[0] = 0;
                    a.ctr[1] = 0;
                }
            }
        }
        return;
    }

    // ============================= scanner warps ===================================
    const uint64_t pol = policy_evict_first();
    const A *seeds = reinterpret_cast<const A *>(a.row_seeds);
    A *totals = reinterpret_cast<A *>(a.row_totals);
    A carry = (A)0;
    for (int64_t item = 0;; ++item) {
        {
            const int b = (int)(item % NBUF);
            mbar_wait(&full[b], (uint32_t)((item / NBUF) & 1));
            const int64_t r = item_row[b];
            if (r < 0) break;
            const int64_t sg = item_seg[b];
            stall_site<STALL>(a.stall, r * 4096 + sg, warp, 2);
            if (sg == 0) carry = seeds ? seeds[r] : (A)0;
            const TIn *sb = buf + (size_t)b * SEG;
            A *tb = tot + b * NCH;
            const int64_t e0 = sg * SEG;
            const int64_t cnt = (a.cols - e0) < SEG ? (a.cols - e0) : SEG;
            // ---- pass 1 over shared memory: chunk totals ----
            for (int ch = warp; ch < NCH; ch += SW) {
                A s = (A)0;
                if ((int64_t)(ch + 1) * CHUNK <= cnt) {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        TIn x[VEC];
                        unpack<TIn>(lds256(sb + ch * CHUNK + rr * ROW_ELEMS + lane * VEC), x);
                        s += lane_row_sum<TIn, A, VEC>(x);
                    }
                } else {
                    for (int rr = 0; rr < RPC; ++rr)
                        for (int j = 0; j < VEC; ++j) {
                            const int64_t k = (int64_t)ch * CHUNK + rr * ROW_ELEMS + lane * VEC + j;
                            if (k < cnt) s += (A)sb[k];
                        }
                }
                s = warp_sum(s);
                if (lane == 0) tb[ch] = s;
            }
            named_sync(BAR_SCAN, SW * 32);
            // ---- chunk carries: exclusive scan of the NCH totals (every warp, same order) ----
            const A t = lane < NCH ? tb[lane] : (A)0;
            A inc = t;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const A y = shfl_up(inc, d);
                if (lane >= d) inc += y;
            }
            A exs = shfl_up(inc, 1);
            if (lane == 0) exs = (A)0;
            const A seg_total = shfl_idx(inc, 31);
            // ---- pass 2: scan each chunk from its carry, store ----
            for (int ch = warp; ch < NCH; ch += SW) {
                const int64_t k0 = (int64_t)ch * CHUNK;
                if (k0 >= cnt) break;
                const bool fullc = k0 + CHUNK <= cnt;
                A v[RPC][VEC];
                if (fullc) {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        TIn x[VEC];
                        unpack<TIn>(lds256(sb + k0 + rr * ROW_ELEMS + lane * VEC), x);
#pragma unroll
                        for (int j = 0; j < VEC; ++j) v[rr][j] = (A)x[j];
                    }
                } else {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr)
#pragma unroll
                        for (int j = 0; j < VEC; ++j) {
                            const int64_t k = k0 + rr * ROW_ELEMS + lane * VEC + j;
                            v[rr][j] = k < cnt ? (A)sb[k] : (A)0;
                        }
                }
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr)
#pragma unroll
                    for (int j = 1; j < VEC; ++j) v[rr][j] += v[rr][j - 1];
                A sc[RPC];
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr) sc[rr] = v[rr][VEC - 1];
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        const A y = shfl_up(sc[rr], d);
                        if (lane >= d) sc[rr] += y;
                    }
                }
                A base = carry + shfl_idx(exs, ch);
                TOut *orow = out + r * a.ld_out + e0 + k0;
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr) {
                    A ex;
                    if constexpr (FLOAT) {
                        ex = shfl_up(sc[rr], 1);
                        if (lane == 0) ex = (A)0;
                    } else {
                        ex = sc[rr] - v[rr][VEC - 1];
                    }
                    const A bb = base + ex;
                    base += shfl_idx(sc[rr], 31);
                    TOut y[VEC];
                    if (a.exclusive) {
                        y[0] = (TOut)bb;
#pragma unroll
                        for (int j = 1; j < VEC; ++j) y[j] = (TOut)(bb + v[rr][j - 1]);
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) y[j] = (TOut)(bb + v[rr][j]);
                    }
                    if (fullc && a.vec_out) {
                        constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
                        for (int q = 0; q < NV; ++q)
                            stg256_policy(orow + rr * ROW_ELEMS + lane * VEC + q * (32 / sizeof(TOut)),
                                          pack<TOut>(&y[q * (32 / sizeof(TOut))]), pol);
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j)
                            if (k0 + rr * ROW_ELEMS + lane * VEC + j < cnt) orow[rr * ROW_ELEMS + lane * VEC + j] = y[j];
                    }
                }
            }
            carry += seg_total;
            // every value this warp read from buf[b] / tot[b] has been consumed: hand
            // its share back (the producer waits for all SW warps)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&freeb[b]);
            if (sg == nseg - 1 && totals && warp == 0 && lane == 0) totals[r] = carry;
        }
    }
}

// Short rows (cols <= SEG / 2): several whole rows per buffer.  Each row starts on
// a chunk boundary of the buffer (cpr chunks per row), the chunk totals are scanned
// segmented by row, and the rows' loads are one bulk copy each -- so a buffer still
// holds 32-64 KiB even for rows of a few KiB (65536 x 3000 int32 -> int64: one row
// per buffer ran at 0.35 of the HBM peak).  A separate kernel: the general
// bookkeeping costs the one-row-per-buffer kernel 7-16 %.
template <typename TIn, typename TOut, int SW, int RPC, int NBUF, int NCH, bool STALL = false>
__global__ void __launch_bounds__((SW + 1) * 32, RPC <= 2 ? 2 : 1) scan_rows_multi_kernel(const RowsArgs a) {
    using Geo = RowsGeom<TIn, SW, RPC, NBUF, NCH>;
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = Geo::VEC, ROW_ELEMS = Geo::ROW_ELEMS, CHUNK = Geo::CHUNK, SEG = Geo::SEG;
    constexpr bool FLOAT = (A)0.5 != (A)0;
    constexpr int BAR_SCAN = 1;
    static_assert(NCH <= 32, "chunk totals are scanned by one warp");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    TIn *buf = reinterpret_cast<TIn *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NBUF * Geo::SEG_BYTES);
    uint64_t *freeb = full + NBUF;
    A *tot = reinterpret_cast<A *>(freeb + NBUF);  // [NBUF][NCH]
    int64_t *item_row = reinterpret_cast<int64_t *>(tot + NBUF * NCH);  // [NBUF]: first row of the item (-1: end)
    int64_t *item_seg = item_row + NBUF;                                 // [NBUF]: segment | (rows << 32)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    TOut *out = reinterpret_cast<TOut *>(a.out);
    const int64_t nseg = (a.cols + SEG - 1) / SEG;
    // Short rows share an item: each row starts on a chunk boundary of the buffer
    // (cpr chunks per row), so up to NCH / cpr rows stream and scan together and a
    // buffer holds 48-64 KiB of data even for rows of a few KiB.
    const int cpr = nseg == 1 ? (int)((a.cols + CHUNK - 1) / CHUNK) : NCH;  // chunks per row in a buffer
    const int rpi = nseg == 1 ? NCH / cpr : 1;                              // rows per item

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&freeb[b], SW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == SW) {
        // =========================== producer ======================================
        // Rows are taken from a grid-wide ticket when a.ctr is given: an SM that
        // streams faster takes more rows (fixed shares leave the grid waiting for the
        // slowest SMs: scripts/sm_fairness.cu).  The next ticket is fetched while the
        // current item's loads are issued.
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const bool dyn = a.ctr != nullptr;
            int64_t item = 0;
            int64_t r = dyn ? (int64_t)atomicAdd(a.ctr, (unsigned long long)rpi) : c * rpi;
            while (true) {
                const int64_t rn = r < a.rows ? (dyn ? (int64_t)atomicAdd(a.ctr, (unsigned long long)rpi) : r + G * rpi) : r;
                const int k = r < a.rows ? (int)((a.rows - r) < rpi ? (a.rows - r) : rpi) : 0;
                for (int64_t sg = 0; sg < nseg; ++sg, ++item) {
                    const int b = (int)(item % NBUF);
                    stall_site<STALL>(a.stall, r, sg, 1);
                    if (item >= NBUF) mbar_wait(&freeb[b], (uint32_t)(((item / NBUF) - 1) & 1));
                    if (r >= a.rows) {  // end marker: the scanners stop at this item
                        item_row[b] = -1;
                        mbar_arrive(&full[b]);
                        break;
                    }
                    item_row[b] = r;
                    item_seg[b] = sg | ((int64_t)k << 32);
                    const int64_t e0 = sg * SEG;
                    const int64_t cnt = (a.cols - e0) < SEG ? (a.cols - e0) : SEG;
                    const uint32_t bytes = (uint32_t)(cnt * sizeof(TIn));
                    mbar_expect_tx(&full[b], bytes * (uint32_t)k);
                    for (int i = 0; i < k; ++i) {
                        const char *src = reinterpret_cast<const char *>(in + (r + i) * a.ld_in + e0);
                        char *dst = reinterpret_cast<char *>(buf + (size_t)b * SEG + (size_t)i * cpr * CHUNK);
                        for (uint32_t o = 0; o < bytes; o += 16384)
                            bulk_g2s(dst + o, src + o, bytes - o < 16384u ? bytes - o : 16384u, &full[b], pol);
                    }
                }
                if (r >= a.rows) break;
                r = rn;
            }
            if (dyn) {
                // the last producer to take its final ticket resets the counters for the
                // next launch on this scratch (stream order makes them visible to it)
                __threadfence();
                if (atomicAdd(a.ctr + 1, 1ull) == (unsigned long long)(G - 1)) {
                    a.ctr[0] = 0;
                    a.ctr[1] = 0;
                }
            }
        }
        return;
    }

    // ============================= scanner warps ===================================
    const uint64_t pol = policy_evict_first();
    const A *seeds = reinterpret_cast<const A *>(a.row_seeds);
    A *totals = reinterpret_cast<A *>(a.row_totals);
    A carry = (A)0;  // running total of the current row over its segments (nseg > 1)
    for (int64_t item = 0;; ++item) {
        const int b = (int)(item % NBUF);
        mbar_wait(&full[b], (uint32_t)((item / NBUF) & 1));
        const int64_t r0 = item_row[b];
        if (r0 < 0) break;
        const int64_t sg = item_seg[b] & 0xffffffff;
        const int k = (int)(item_seg[b] >> 32);
        stall_site<STALL>(a.stall, r0 * 4096 + sg, warp, 2);
        if (sg == 0 && nseg > 1) carry = seeds ? seeds[r0] : (A)0;
        const TIn *sb = buf + (size_t)b * SEG;
        A *tb = tot + b * NCH;
        const int64_t e0 = sg * SEG;
        const int64_t cnt = (a.cols - e0) < SEG ? (a.cols - e0) : SEG;  // elements per row in this item
        const int nch = k * cpr;                                         // chunks in use
        // chunk ch: row ch / cpr of the item, elements [lc CHUNK, lc CHUNK + CHUNK) of its segment
        auto chunk_len = [&](int ch) {
            const int64_t lc0 = (int64_t)(ch % cpr) * CHUNK;
            return lc0 >= cnt ? (int64_t)0 : ((cnt - lc0) < CHUNK ? (cnt - lc0) : (int64_t)CHUNK);
        };
        // every chunk of the buffer in use and full (cfg4-like rows): the chunk loops
        // have a static trip count and no length checks, so the compiler overlaps chunks
        const bool all_full = nch == NCH && cnt == (int64_t)cpr * CHUNK;
        // ---- pass 1 over shared memory: chunk totals ----
        auto pass1 = [&](auto full_tag) {
            constexpr bool FULLI = decltype(full_tag)::value;
            for (int ch = warp; ch < NCH; ch += SW) {
                if (!FULLI && ch >= nch) break;
                A s = (A)0;
                const int64_t len = FULLI ? (int64_t)CHUNK : chunk_len(ch);
                if (len == CHUNK) {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        TIn x[VEC];
                        unpack<TIn>(lds256(sb + ch * CHUNK + rr * ROW_ELEMS + lane * VEC), x);
                        s += lane_row_sum<TIn, A, VEC>(x);
                    }
                } else {  // a row's last chunk: whole lane vectors where valid
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        const int k0v = rr * ROW_ELEMS + lane * VEC;
                        if (k0v + VEC <= len) {
                            TIn x[VEC];
                            unpack<TIn>(lds256(sb + ch * CHUNK + k0v), x);
                            s += lane_row_sum<TIn, A, VEC>(x);
                        } else {
                            for (int j = 0; j < VEC; ++j)
                                if (k0v + j < len) s += (A)sb[(int64_t)ch * CHUNK + k0v + j];
                        }
                    }
                }
                s = warp_sum(s);
                if (lane == 0) tb[ch] = s;
            }
        };
        if (all_full) pass1(std::true_type{});
        else pass1(std::false_type{});
        named_sync(BAR_SCAN, SW * 32);
        // ---- chunk carries: exclusive scan of the chunk totals within each row
        //      (every warp, same order; a row's chunks are lanes [rs, rs + cpr)) ----
        const int rs = (lane / cpr) * cpr;
        const A t = lane < nch ? tb[lane] : (A)0;
        A inc = t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const A y = shfl_up(inc, d);
            if (lane - d >= rs) inc += y;
        }
        A exs = shfl_up(inc, 1);
        if (lane == rs) exs = (A)0;
        // ---- pass 2: scan each chunk from its carry, store ----
        auto pass2 = [&](auto full_tag) {
            constexpr bool FULLI = decltype(full_tag)::value;
            for (int ch = warp; ch < NCH; ch += SW) {
                if (!FULLI && ch >= nch) break;
                const int64_t len = FULLI ? (int64_t)CHUNK : chunk_len(ch);
                if (len == 0) continue;
                const int ri = ch / cpr;
                const int64_t k0 = (int64_t)(ch % cpr) * CHUNK;  // within the row's segment
                const bool fullc = len == CHUNK;
                A v[RPC][VEC];
                if (fullc) {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        TIn x[VEC];
                        unpack<TIn>(lds256(sb + (int64_t)ch * CHUNK + rr * ROW_ELEMS + lane * VEC), x);
#pragma unroll
                        for (int j = 0; j < VEC; ++j) v[rr][j] = (A)x[j];
                    }
                } else {  // a row's last chunk: whole lane vectors where valid
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        const int k0v = rr * ROW_ELEMS + lane * VEC;
                        if (k0v + VEC <= len) {
                            TIn x[VEC];
                            unpack<TIn>(lds256(sb + (int64_t)ch * CHUNK + k0v), x);
#pragma unroll
                            for (int j = 0; j < VEC; ++j) v[rr][j] = (A)x[j];
                        } else {
#pragma unroll
                            for (int j = 0; j < VEC; ++j)
                                v[rr][j] = k0v + j < len ? (A)sb[(int64_t)ch * CHUNK + k0v + j] : (A)0;
                        }
                    }
                }
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr)
#pragma unroll
                    for (int j = 1; j < VEC; ++j) v[rr][j] += v[rr][j - 1];
                A sc[RPC];
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr) sc[rr] = v[rr][VEC - 1];
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                    for (int rr = 0; rr < RPC; ++rr) {
                        const A y = shfl_up(sc[rr], d);
                        if (lane >= d) sc[rr] += y;
                    }
                }
                const A rc = nseg > 1 ? carry : (seeds ? seeds[r0 + ri] : (A)0);
                A base = rc + shfl_idx(exs, ch);
                TOut *orow = out + (r0 + ri) * a.ld_out + e0 + k0;
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr) {
                    A ex;
                    if constexpr (FLOAT) {
                        ex = shfl_up(sc[rr], 1);
                        if (lane == 0) ex = (A)0;
                    } else {
                        ex = sc[rr] - v[rr][VEC - 1];
                    }
                    const A bb = base + ex;
                    base += shfl_idx(sc[rr], 31);
                    TOut y[VEC];
                    if (a.exclusive) {
                        y[0] = (TOut)bb;
#pragma unroll
                        for (int j = 1; j < VEC; ++j) y[j] = (TOut)(bb + v[rr][j - 1]);
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) y[j] = (TOut)(bb + v[rr][j]);
                    }
                    if (a.vec_out) {  // 32-byte pieces wherever they are whole
                        constexpr int NV = VEC * sizeof(TOut) / 32, PE = 32 / sizeof(TOut);
#pragma unroll
                        for (int q = 0; q < NV; ++q) {
                            const int kq = rr * ROW_ELEMS + lane * VEC + q * PE;
                            if (fullc || kq + PE <= len) {
                                stg256_policy(orow + kq, pack<TOut>(&y[q * PE]), pol);
                            } else {
#pragma unroll
                                for (int j = 0; j < PE; ++j)
                                    if (kq + j < len) orow[kq + j] = y[q * PE + j];
                            }
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j)
                            if (rr * ROW_ELEMS + lane * VEC + j < len) orow[rr * ROW_ELEMS + lane * VEC + j] = y[j];
                    }
                }
            }
        };
        if (all_full) pass2(std::true_type{});
        else pass2(std::false_type{});
        // row totals: the inclusive chunk total at each row's last chunk
        if (nseg > 1) {
            carry += shfl_idx(inc, cpr - 1);
            if (sg == nseg - 1 && totals && warp == 0 && lane == 0) totals[r0] = carry;
        } else if (totals && warp == 0) {
            for (int ri = 0; ri < k; ++ri) {
                const A rt = shfl_idx(inc, ri * cpr + cpr - 1);
                if (lane == 0) totals[r0 + ri] = (seeds ? seeds[r0 + ri] : (A)0) + rt;
            }
        }
        // every value this warp read from buf[b] / tot[b] has been consumed: hand
        // its share back (the producer waits for all SW warps)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[b]);
    }
}

}  // namespace ps
