// scan_kernels.cuh -- the sm_100a kernels of the prefix-sum hot path.
//
//   scan_tiles_kernel  single-pass decoupled look-back scan (1-D and batched rows)
//                      <- core.py:86-92 _scan_kernel, simd.py:75-101 horizontal,
//                         core.py:109-115 exclusive shift (fused), simd.py:164-206
//                         vertical passes (row seeds / row totals)
//   reduce_kernel      read-only deterministic total  <- core.py:95-100 _accumulate_kernel
//   add_offset_kernel  buf += delta                   <- core.py:103-106 _increment_kernel
//
// Memory-bound by design (one read + one write per element).  Tile geometry:
// WARPS warps x ROWS rows x 32 lanes x VEC elements, VEC = 32 bytes of input
// per lane per row, so every load is one LDG.E.256 and a warp row is 1 KiB of
// contiguous input.  A thread keeps its ROWS x VEC inputs in registers from
// load to store; the tile's carry comes from the look-back, never from a
// second pass over HBM.
#pragma once

#include "scan_device.cuh"

namespace ps {

// Sum of the published totals of mailbox slots 0..m.n-1 (one full warp; the
// tree order is fixed, so every CTA of a rank folds the same value).
template <typename A>
__device__ A mailbox_sum(const Mailbox &m, int lane) {
    A v = (A)0;
    for (int j = lane; j < m.n; j += 32) {
        uint64_t bits = 0;
        if (!mailbox_try(m.slots + j, m.epoch, &bits)) {
            const uint64_t t0 = global_ns();
            while (true) {
                __nanosleep(100);
                if (mailbox_try(m.slots + j, m.epoch, &bits)) break;
                if (global_ns() - t0 > 10000000000ull) {
                    if (m.timeout) atomicExch(m.timeout, 1);
                    bits = 0;
                    break;
                }
            }
        }
        v += acc_from_bits<A>(bits);
    }
    return warp_sum(v);
}

struct ScanArgs {
    const void *in;
    void *out;
    int64_t rows;           // independent segments laid out as rows
    int64_t cols;           // elements per row
    int64_t ld_in, ld_out;  // row strides (elements)
    int64_t tiles_per_row;
    int64_t lead;           // masked leading elements so tiles start 32B-aligned
    uint64_t seed_bits;     // host part of the seed (acc bits)
    const void *seed_terms; // rows == 1: seed += sum(seed_terms[0..n_seed_terms))
    int64_t n_seed_terms;   // rows  > 1: seed_terms is per-row (n_seed_terms == rows)
    void *totals;           // acc-typed per-row totals (nullable)
    Desc desc;
    uint32_t epoch;
    int exclusive;
    int vec_ok;             // in/out row bases (minus lead) are 32B aligned
    int row_lead;           // rows > 1: lead and vec_ok per row from the row's own addresses
    int debug_flags;        // bit 0: skip the look-back (timing experiments only; wrong results)
    Stall stall;            // stress tests: stall injection at the publication points
    Mailbox mail;           // rows == 1: seed += totals published by the ranks before this one
};

template <typename T> __device__ __forceinline__ void unpack(const V256 &v, T (&x)[32 / sizeof(T)]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if constexpr (sizeof(T) == 8) {
            memcpy(&x[k], &v.w[k], 8);
        } else {
            const uint32_t lo = (uint32_t)v.w[k], hi = (uint32_t)(v.w[k] >> 32);
            memcpy(&x[2 * k], &lo, 4);
            memcpy(&x[2 * k + 1], &hi, 4);
        }
    }
}

// pack 32 bytes of T starting at y[0] into a V256 (register-only bit casts)
template <typename T> __device__ __forceinline__ V256 pack(const T *y) {
    V256 v;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if constexpr (sizeof(T) == 8) {
            memcpy(&v.w[k], &y[k], 8);
        } else {
            uint32_t lo, hi;
            memcpy(&lo, &y[2 * k], 4);
            memcpy(&hi, &y[2 * k + 1], 4);
            v.w[k] = (uint64_t)lo | ((uint64_t)hi << 32);
        }
    }
    return v;
}

template <typename TIn, typename TOut, int WARPS, int ROWS>
#ifndef PS_TILES_MINB
#define PS_TILES_MINB 4  // 4 CTAs per SM (64 registers): more tiles in flight hide the look-back; 2, 3, 5, 6 and no bound were slower
#endif
__global__ void __launch_bounds__(WARPS * 32, PS_TILES_MINB)
    scan_tiles_kernel(const ScanArgs a) {
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = 32 / sizeof(TIn);
    constexpr int ROW_ELEMS = 32 * VEC;
    constexpr int WARP_ELEMS = ROWS * ROW_ELEMS;
    constexpr int64_t TILE = (int64_t)WARPS * WARP_ELEMS;
    constexpr bool FLOAT = (A)0.5 != (A)0;

    __shared__ A s_warp[WARPS];
    __shared__ A s_base[WARPS];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // Tile ids follow blockIdx: CTAs are dispatched in increasing linear
    // order, so every predecessor a look-back waits on is already resident or
    // finished (the same forward-progress argument CUB's single-pass scan uses).
    const int64_t tile = blockIdx.x;
    const int64_t row = tile / a.tiles_per_row;
    const int64_t chunk = tile - row * a.tiles_per_row;
    const int64_t head = row * a.tiles_per_row;

    // tile-space coordinates: element c of the row sits at position c + lead
    int64_t lead = a.lead;
    bool vec = a.vec_ok;
    if (a.row_lead) {
        // each row's tiles start on the 32-byte boundary at or before the row start, so
        // rows whose length is not a multiple of 32 bytes still move with 256-bit
        // accesses; contiguous int32 -> int64 and same-size rows then also have their
        // output 32-byte aligned (checked per row)
        const uintptr_t ia = (uintptr_t)(reinterpret_cast<const TIn *>(a.in) + row * a.ld_in);
        lead = (int64_t)((ia & 31) / sizeof(TIn));
        const uintptr_t oa = (uintptr_t)(reinterpret_cast<TOut *>(a.out) + row * a.ld_out) - lead * sizeof(TOut);
        vec = (oa & 31) == 0;
    }
    const int64_t t0 = chunk * TILE;
    const int64_t lo = lead, hi = lead + a.cols;  // valid positions [lo, hi)
    const TIn *in = reinterpret_cast<const TIn *>(a.in) + row * a.ld_in - lead + t0;
    TOut *out = reinterpret_cast<TOut *>(a.out) + row * a.ld_out - lead + t0;
    const bool full = vec && t0 >= lo && t0 + TILE <= hi;
    // a lane's 32-byte vector of row r lies entirely inside the valid positions
    auto lane_vec = [&](int r) {
        const int64_t p = t0 + (int64_t)warp * WARP_ELEMS + lane * VEC + r * ROW_ELEMS;
        return vec && p >= lo && p + VEC <= hi;
    };
#ifdef PS_TRACE
    if (g_trace && threadIdx.x == 0) {
        g_trace[tile * 8 + 0] = gtimer();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace[tile * 8 + 6] = smid;
    }
#endif

    // ---- load: ROWS independent 256-bit loads per thread --------------------------
    TIn x[ROWS][VEC];
    const int64_t my0 = (int64_t)warp * WARP_ELEMS + lane * VEC;  // + r * ROW_ELEMS
    if (full) {
        V256 raw[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) raw[r] = ldg256_stream(in + my0 + r * ROW_ELEMS);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) unpack<TIn>(raw[r], x[r]);
    } else {  // edge tile: whole lane vectors where they are valid, masked elements elsewhere
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            if (lane_vec(r)) {
                unpack<TIn>(ldg256_stream(in + my0 + r * ROW_ELEMS), x[r]);
            } else {
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    const int64_t pos = t0 + my0 + r * ROW_ELEMS + j;
                    x[r][j] = (pos >= lo && pos < hi) ? in[my0 + r * ROW_ELEMS + j] : (TIn)0;
                }
            }
        }
    }

    // ---- per-lane sums, then ROWS interleaved warp scans (5 shuffle rounds) --------
    A lsum[ROWS], scan[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        A s = (A)x[r][0];
#pragma unroll
        for (int j = 1; j < VEC; ++j) s += (A)x[r][j];
        lsum[r] = s;
        scan[r] = s;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            const A y = shfl_up(scan[r], d);
            if (lane >= d) scan[r] += y;
        }
    }
    // lane-exclusive offset inside each warp row, and the row totals
    A lex[ROWS];
    A wrun = (A)0;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        A ex;
        if constexpr (FLOAT) {
            ex = shfl_up(scan[r], 1);
            if (lane == 0) ex = (A)0;
        } else {
            ex = scan[r] - lsum[r];
        }
        const A rtot = shfl_idx(scan[r], 31);
        lex[r] = wrun + ex;
        wrun += rtot;
    }
    if (lane == 0) s_warp[warp] = wrun;
#ifdef PS_TRACE
    if (g_trace && threadIdx.x == 0) g_trace[tile * 8 + 1] = gtimer();
#endif
    __syncthreads();
#ifdef PS_TRACE
    if (g_trace && threadIdx.x == 0) g_trace[tile * 8 + 2] = gtimer();
#endif

    // ---- warp 0: tile aggregate, publish, look-back, publish inclusive -------------
    if (warp == 0) {
        A wt = lane < WARPS ? s_warp[lane] : (A)0;
        A ws = wt;
#pragma unroll
        for (int d = 1; d < WARPS; d <<= 1) {
            const A y = shfl_up(ws, d);
            if (lane >= d) ws += y;
        }
        const A agg = shfl_idx(ws, WARPS - 1);
        A wex;
        if constexpr (FLOAT) {
            wex = shfl_up(ws, 1);
            if (lane == 0) wex = (A)0;
        } else {
            wex = ws - wt;
        }
        A excl;
        if (tile == head) {
            A seed = acc_from_bits<A>(a.seed_bits);
            if (a.seed_terms) {
                const A *st = reinterpret_cast<const A *>(a.seed_terms);
                if (a.rows > 1) {
                    seed += st[row];
                } else {
                    A acc = (A)0;
                    for (int64_t i = lane; i < a.n_seed_terms; i += 32) acc += st[i];
                    seed += warp_sum(acc);
                }
            }
            if (a.mail.n) seed += mailbox_sum<A>(a.mail, lane);
            excl = seed;
            if (lane == 0 && a.tiles_per_row > 1) publish(a.desc, tile, a.epoch, ST_P, acc_to_bits<A>(seed + agg));
        } else {
            maybe_stall(a.stall, tile, 0, 1);
            if (lane == 0) publish(a.desc, tile, a.epoch, ST_A, acc_to_bits<A>(agg));
            excl = (a.debug_flags & 1) ? (A)0 : lookback<A>(a.desc, tile, head, a.epoch, lane);
            maybe_stall(a.stall, tile, 0, 2);
            if (lane == 0 && chunk + 1 < a.tiles_per_row)
                publish(a.desc, tile, a.epoch, ST_P, acc_to_bits<A>(excl + agg));
        }
        if (lane < WARPS) s_base[lane] = excl + wex;
        if (lane == 0 && a.totals && chunk + 1 == a.tiles_per_row)
            reinterpret_cast<A *>(a.totals)[row] = excl + agg;
    }
    __syncthreads();
#ifdef PS_TRACE
    if (g_trace && threadIdx.x == 0) g_trace[tile * 8 + 3] = gtimer();
#endif

    // ---- add carries, convert, store -----------------------------------------------
    const A wbase = s_base[warp];
    if (full) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            A run = wbase + lex[r];
            TOut y[VEC];
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                if (a.exclusive) {
                    y[j] = (TOut)run;
                    run += (A)x[r][j];
                } else {
                    run += (A)x[r][j];
                    y[j] = (TOut)run;
                }
            }
            constexpr int NV = VEC * sizeof(TOut) / 32;  // 256-bit stores per lane-row
#pragma unroll
            for (int k = 0; k < NV; ++k)
                stg256_stream(out + my0 + r * ROW_ELEMS + k * (32 / sizeof(TOut)),
                              pack<TOut>(&y[k * (32 / sizeof(TOut))]));
        }
    } else {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            A run = wbase + lex[r];
            TOut y[VEC];
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const A before = run;
                run += (A)x[r][j];
                y[j] = (TOut)(a.exclusive ? before : run);
            }
            if (lane_vec(r)) {
                constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
                for (int k = 0; k < NV; ++k)
                    stg256_stream(out + my0 + r * ROW_ELEMS + k * (32 / sizeof(TOut)),
                                  pack<TOut>(&y[k * (32 / sizeof(TOut))]));
            } else {
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    const int64_t pos = t0 + my0 + r * ROW_ELEMS + j;
                    if (pos >= lo && pos < hi) out[my0 + r * ROW_ELEMS + j] = y[j];
                }
            }
        }
    }
#ifdef PS_TRACE
    if (g_trace && threadIdx.x == 0) g_trace[tile * 8 + 4] = gtimer();
#endif
}

// ---- deterministic read-only reduction ------------------------------------------------
struct ReduceArgs {
    const void *in;
    int64_t n;
    int64_t lead;           // elements before the first 32B boundary
    uint64_t seed_bits;
    const void *seed_terms;
    int64_t n_seed_terms;
    void *total;            // acc-typed
    uint64_t *partials;     // one per CTA (reduce_kernel) or per block (reduce_blocks_kernel)
    uint32_t *ticket;       // zero between launches (the last CTA resets it)
    unsigned long long *blk_ticket;  // reduce_blocks_kernel: next block, zero between launches
    int64_t blk_vecs;       // reduce_blocks_kernel: 32-byte vectors per block
};

template <typename A, int THREADS> __device__ __forceinline__ A block_sum(A v, A *smem) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    A r = (A)0;
    if (warp == 0) {
        r = lane < THREADS / 32 ? smem[lane] : (A)0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;  // valid in warp 0
}

template <typename TIn, int THREADS>
__global__ void __launch_bounds__(THREADS) reduce_kernel(const ReduceArgs a) {
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = 32 / sizeof(TIn);
    __shared__ A smem[THREADS / 32];
    __shared__ bool last;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    A acc = (A)0;
    const int64_t head = a.lead < a.n ? a.lead : a.n;
    const int64_t nvec = (a.n - head) / VEC;
    const int64_t tail0 = head + nvec * VEC;
    const int64_t tid = (int64_t)blockIdx.x * THREADS + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * THREADS;
    int64_t v = tid;
    for (; v + 3 * stride < nvec; v += 4 * stride) {  // 4 loads in flight per thread
        V256 r0 = ldg256_stream(in + head + v * VEC);
        V256 r1 = ldg256_stream(in + head + (v + stride) * VEC);
        V256 r2 = ldg256_stream(in + head + (v + 2 * stride) * VEC);
        V256 r3 = ldg256_stream(in + head + (v + 3 * stride) * VEC);
        TIn x0[VEC], x1[VEC], x2[VEC], x3[VEC];
        unpack<TIn>(r0, x0); unpack<TIn>(r1, x1); unpack<TIn>(r2, x2); unpack<TIn>(r3, x3);
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc += (A)x0[j];
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc += (A)x1[j];
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc += (A)x2[j];
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc += (A)x3[j];
    }
    for (; v < nvec; v += stride) {
        TIn x0[VEC];
        unpack<TIn>(ldg256_stream(in + head + v * VEC), x0);
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc += (A)x0[j];
    }
    if (tid < head) acc += (A)in[tid];
    if (tid < a.n - tail0) acc += (A)in[tail0 + tid];
    A bs = block_sum<A, THREADS>(acc, smem);
    if (threadIdx.x == 0) {
        st_relaxed_u64(a.partials + blockIdx.x, acc_to_bits<A>(bs));
        __threadfence();
        const uint32_t t = atomicAdd(a.ticket, 1u);
        last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last CTA: fixed-order sum of the partials (deterministic for floats)
    A p = (A)0;
    for (int64_t i = threadIdx.x; i < gridDim.x; i += THREADS) p += acc_from_bits<A>(ld_relaxed_u64(a.partials + i));
    p = block_sum<A, THREADS>(p, smem);
    if (threadIdx.x == 0) {
        A seed = acc_from_bits<A>(a.seed_bits);
        if (a.seed_terms) {
            const A *st = reinterpret_cast<const A *>(a.seed_terms);
            for (int64_t i = 0; i < a.n_seed_terms; ++i) seed += st[i];
        }
        *reinterpret_cast<A *>(a.total) = seed + p;
        *a.ticket = 0;
    }
}

// Blocks of blk_vecs vectors taken from a ticket (an SM that streams faster takes
// more of them; fixed grid-stride shares leave the grid waiting for the slowest
// SMs, scripts/sm_fairness.cu).  Each block's sum lands in partials[block] and
// the last CTA folds them in block order, so float totals stay run-to-run
// identical whichever CTA reduced which block.
template <typename TIn, int THREADS>
__global__ void __launch_bounds__(THREADS) reduce_blocks_kernel(const ReduceArgs a) {
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = 32 / sizeof(TIn);
    __shared__ A smem[THREADS / 32];
    __shared__ int64_t s_blk;
    __shared__ bool last;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    const int64_t head = a.lead < a.n ? a.lead : a.n;
    const int64_t nvec = (a.n - head) / VEC;
    const int64_t tail0 = head + nvec * VEC;
    const int64_t nblk = (nvec + a.blk_vecs - 1) / a.blk_vecs;
    if (threadIdx.x == 0) s_blk = (int64_t)atomicAdd(a.blk_ticket, 1ull);
    __syncthreads();
    int64_t blk = s_blk;
    while (blk < nblk) {
        __syncthreads();  // everyone has read s_blk
        if (threadIdx.x == 0) s_blk = (int64_t)atomicAdd(a.blk_ticket, 1ull);  // next one, in flight
        const int64_t v0 = blk * a.blk_vecs;
        const int64_t v1 = v0 + a.blk_vecs < nvec ? v0 + a.blk_vecs : nvec;
        A acc = (A)0;
        int64_t v = v0 + threadIdx.x;
        for (; v + 3 * THREADS < v1; v += 4 * THREADS) {
            V256 r0 = ldg256_stream(in + head + v * VEC);
            V256 r1 = ldg256_stream(in + head + (v + THREADS) * VEC);
            V256 r2 = ldg256_stream(in + head + (v + 2 * THREADS) * VEC);
            V256 r3 = ldg256_stream(in + head + (v + 3 * THREADS) * VEC);
            TIn x0[VEC], x1[VEC], x2[VEC], x3[VEC];
            unpack<TIn>(r0, x0); unpack<TIn>(r1, x1); unpack<TIn>(r2, x2); unpack<TIn>(r3, x3);
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc += (A)x0[j];
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc += (A)x1[j];
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc += (A)x2[j];
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc += (A)x3[j];
        }
        for (; v < v1; v += THREADS) {
            TIn x0[VEC];
            unpack<TIn>(ldg256_stream(in + head + v * VEC), x0);
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc += (A)x0[j];
        }
        const A bs = block_sum<A, THREADS>(acc, smem);  // ends with __syncthreads: s_blk is written
        if (threadIdx.x == 0) st_relaxed_u64(a.partials + blk, acc_to_bits<A>(bs));
        blk = s_blk;
    }
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(a.ticket, 1u);
        last = t == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last CTA: the blocks in order, then the unaligned head and tail elements
    A p = (A)0;
    for (int64_t i = threadIdx.x; i < nblk; i += THREADS) p += acc_from_bits<A>(ld_relaxed_u64(a.partials + i));
    if (threadIdx.x < head) p += (A)in[threadIdx.x];
    if (threadIdx.x < a.n - tail0) p += (A)in[tail0 + threadIdx.x];
    p = block_sum<A, THREADS>(p, smem);
    if (threadIdx.x == 0) {
        A seed = acc_from_bits<A>(a.seed_bits);
        if (a.seed_terms) {
            const A *st = reinterpret_cast<const A *>(a.seed_terms);
            for (int64_t i = 0; i < a.n_seed_terms; ++i) seed += st[i];
        }
        *reinterpret_cast<A *>(a.total) = seed + p;
        *a.ticket = 0;
        *a.blk_ticket = 0;
    }
}

// ---- buf[i] += delta ---------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) add_offset_kernel(T *buf, int64_t n, int64_t lead, uint64_t delta_bits,
                                                         const void *delta_terms, int64_t n_terms) {
    using A = typename AccOf<T>::type;
    constexpr int VEC = 32 / sizeof(T);
    A delta = acc_from_bits<A>(delta_bits);
    if (delta_terms) {
        const A *st = reinterpret_cast<const A *>(delta_terms);
        for (int64_t i = 0; i < n_terms; ++i) delta += st[i];
    }
    const int64_t head = lead < n ? lead : n;
    const int64_t nvec = (n - head) / VEC;
    const int64_t tail0 = head + nvec * VEC;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < nvec; v += stride) {
        T *p = buf + head + v * VEC;
        V256 raw;
        asm volatile("ld.global.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(raw.w[0]), "=l"(raw.w[1]), "=l"(raw.w[2]), "=l"(raw.w[3])
                     : "l"(p));
        T x[VEC];
        unpack<T>(raw, x);
#pragma unroll
        for (int j = 0; j < VEC; ++j) x[j] = (T)((A)x[j] + delta);
        stg256_stream(p, pack<T>(x));
    }
    if (tid < head) buf[tid] = (T)((A)buf[tid] + delta);
    if (tid < n - tail0) buf[tail0 + tid] = (T)((A)buf[tail0 + tid] + delta);
}

}  // namespace ps
