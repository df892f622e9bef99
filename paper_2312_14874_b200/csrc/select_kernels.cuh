// select_kernels.cuh -- stream compaction / stable partition on top of the
// exclusive offsets: the paper's motivating consumer of a
// prefix sum, "determine the new offsets of data items during a partitioning
// step ... from a previously constructed bitmap, and then used as the new index
// values" (parallel filtering).
//
// Three launches:
//   select_count_kernel    flags -> per-tile selected counts            (read flags; HBM-bound)
//   select_offsets_kernel  exclusive scan of the counts + total         (one CTA; n/1024 bytes)
//   select_scatter_kernel  flags + values -> out at the tile's offset   (read both, write out)
// A tile is 8 warps x 4 rows x 256 elements = 8192 elements.  Inside a tile the
// destination of every element is computed in registers (lane popcounts,
// warp scans of two packed 16-bit row counts, an 8-entry CTA scan), the tile
// is compacted into shared memory, and written back with coalesced stores.
// Order is preserved (stable) for the selected elements and, in partition
// mode, for the rejected ones, which follow all selected elements.
#pragma once

#include "scan_kernels.cuh"

namespace ps {

constexpr int SEL_WARPS = 8;
constexpr int SEL_ROWS = 4;
constexpr int SEL_VEC = 8;                                    // elements per lane per row
constexpr int SEL_ROW_ELEMS = 32 * SEL_VEC;                   // 256
constexpr int SEL_WARP_ELEMS = SEL_ROWS * SEL_ROW_ELEMS;      // 1024
constexpr int64_t SEL_TILE = SEL_WARPS * SEL_WARP_ELEMS;      // 8192
constexpr int SEL_THREADS = SEL_WARPS * 32;

// 8 consecutive elements of T starting at p (p aligned to 8 * sizeof(T) bytes
// for 4/8-byte T, 8 bytes for 1-byte T) -> raw 64-bit lanes
template <typename T>
__device__ __forceinline__ void load8(const T *p, T (&x)[SEL_VEC]) {
    if constexpr (sizeof(T) == 1) {
        const uint64_t w = __ldcs(reinterpret_cast<const unsigned long long *>(p));
        memcpy(x, &w, 8);
    } else if constexpr (sizeof(T) == 4) {
        const V256 v = ldg256_stream(p);
        unpack<T>(v, x);
    } else {
        const V256 a = ldg256_stream(p), b = ldg256_stream(p + 4);
        T lo[4], hi[4];
        unpack<T>(a, lo);
        unpack<T>(b, hi);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] = lo[j];
            x[4 + j] = hi[j];
        }
    }
}

template <typename T>
__device__ __forceinline__ bool is_set(const T &f) {
    // any nonzero bit pattern selects (a -0.0 float flag counts as set, like a bitmap)
    if constexpr (sizeof(T) == 1) {
        uint8_t b;
        memcpy(&b, &f, 1);
        return b != 0;
    } else if constexpr (sizeof(T) == 4) {
        uint32_t b;
        memcpy(&b, &f, 4);
        return b != 0;
    } else {
        uint64_t b;
        memcpy(&b, &f, 8);
        return b != 0;
    }
}

// tile counts: grid-stride over tiles, one int64 count per tile
template <typename TF>
__global__ void __launch_bounds__(SEL_THREADS) select_count_kernel(const TF *flags, int64_t n, int64_t ntiles,
                                                                    int vec_ok, long long *counts) {
    __shared__ int s_warp[SEL_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t t0 = t * SEL_TILE;
        int c = 0;
        if (vec_ok && t0 + SEL_TILE <= n) {
            TF f[SEL_ROWS][SEL_VEC];
#pragma unroll
            for (int r = 0; r < SEL_ROWS; ++r)
                load8<TF>(flags + t0 + warp * SEL_WARP_ELEMS + r * SEL_ROW_ELEMS + lane * SEL_VEC, f[r]);
#pragma unroll
            for (int r = 0; r < SEL_ROWS; ++r)
#pragma unroll
                for (int j = 0; j < SEL_VEC; ++j) c += is_set(f[r][j]) ? 1 : 0;
        } else {
            for (int64_t i = t0 + threadIdx.x; i < n && i < t0 + SEL_TILE; i += SEL_THREADS) c += is_set(flags[i]) ? 1 : 0;
        }
        c = __reduce_add_sync(FULL, (unsigned)c);
        if (lane == 0) s_warp[warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long tot = 0;
#pragma unroll
            for (int w = 0; w < SEL_WARPS; ++w) tot += s_warp[w];
            counts[t] = tot << 2;  // low 2 bits 0: never a published look-back descriptor tag
        }
        __syncthreads();
    }
}

// Exclusive scan of the tile counts in place by one CTA (8 bytes per 8192
// elements: 32768 counts = 256 KiB for 2^28 elements), total -> *total.  No look-back
// descriptors, so the select scratch never needs epoch tags.  Counts and offsets are
// kept shifted left by 2: a scratch shared with a later scan then holds no word whose
// status bits could pass for a published descriptor.
constexpr int SEL_SCAN_THREADS = 1024;
constexpr int SEL_SCAN_PER = 8;
__global__ void __launch_bounds__(SEL_SCAN_THREADS) select_offsets_kernel(long long *counts, int64_t ntiles,
                                                                           long long *total) {
    __shared__ long long s_warp[SEL_SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long carry = 0;
    for (int64_t b = 0; b < ntiles; b += (int64_t)SEL_SCAN_THREADS * SEL_SCAN_PER) {
        const int64_t i0 = b + (int64_t)threadIdx.x * SEL_SCAN_PER;
        long long x[SEL_SCAN_PER];
        long long own = 0;
#pragma unroll
        for (int j = 0; j < SEL_SCAN_PER; ++j) {
            x[j] = i0 + j < ntiles ? (counts[i0 + j] >> 2) : 0;
            own += x[j];
        }
        long long inc = own;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(FULL, inc, d);
            if (lane >= d) inc += y;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        long long wbase = 0, btot = 0;
        for (int w = 0; w < SEL_SCAN_THREADS / 32; ++w) {
            const long long v = s_warp[w];
            wbase += w < warp ? v : 0;
            btot += v;
        }
        long long run = carry + wbase + inc - own;
#pragma unroll
        for (int j = 0; j < SEL_SCAN_PER; ++j) {
            if (i0 + j < ntiles) counts[i0 + j] = run << 2;
            run += x[j];
        }
        carry += btot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// One CTA per tile.  offsets[t] = selected elements before tile t (exclusive
// scan of the counts), *total = all selected elements.
template <typename TV, typename TF, bool PARTITION>
__global__ void __launch_bounds__(SEL_THREADS) select_scatter_kernel(const TV *values, const TF *flags, int64_t n,
                                                                      int vec_ok, const long long *offsets,
                                                                      const long long *total, TV *out) {
    extern __shared__ __align__(16) unsigned char sel_smem[];
    TV *stage = reinterpret_cast<TV *>(sel_smem);  // [SEL_TILE]: selected first, then rejected
    __shared__ int s_warp[SEL_WARPS];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t = blockIdx.x;
    const int64_t t0 = t * SEL_TILE;
    const int64_t cnt = (n - t0) < SEL_TILE ? (n - t0) : SEL_TILE;
    const int64_t w0 = t0 + warp * SEL_WARP_ELEMS;

    TV v[SEL_ROWS][SEL_VEC];
    uint32_t m[SEL_ROWS];  // selection bits of the lane's 8 elements per row
    if (vec_ok && cnt == SEL_TILE) {
        TF f[SEL_ROWS][SEL_VEC];
#pragma unroll
        for (int r = 0; r < SEL_ROWS; ++r) {
            load8<TF>(flags + w0 + r * SEL_ROW_ELEMS + lane * SEL_VEC, f[r]);
            load8<TV>(values + w0 + r * SEL_ROW_ELEMS + lane * SEL_VEC, v[r]);
        }
#pragma unroll
        for (int r = 0; r < SEL_ROWS; ++r) {
            m[r] = 0;
#pragma unroll
            for (int j = 0; j < SEL_VEC; ++j) m[r] |= (is_set(f[r][j]) ? 1u : 0u) << j;
        }
    } else {
#pragma unroll
        for (int r = 0; r < SEL_ROWS; ++r) {
            m[r] = 0;
#pragma unroll
            for (int j = 0; j < SEL_VEC; ++j) {
                const int64_t i = w0 + r * SEL_ROW_ELEMS + lane * SEL_VEC + j;
                if (i < n) {
                    v[r][j] = values[i];
                    m[r] |= (is_set(flags[i]) ? 1u : 0u) << j;
                } else {
                    memset(&v[r][j], 0, sizeof(TV));
                }
            }
        }
    }

    // lane-exclusive prefixes of the row counts: rows (0,1) and (2,3) packed in 16-bit halves
    const uint32_t c0 = __popc(m[0]), c1 = __popc(m[1]), c2 = __popc(m[2]), c3 = __popc(m[3]);
    uint32_t p01 = c0 | (c1 << 16), p23 = c2 | (c3 << 16);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t a = __shfl_up_sync(FULL, p01, d), b = __shfl_up_sync(FULL, p23, d);
        if (lane >= d) {
            p01 += a;
            p23 += b;
        }
    }
    const uint32_t t01 = __shfl_sync(FULL, p01, 31), t23 = __shfl_sync(FULL, p23, 31);
    const uint32_t ex01 = p01 - (c0 | (c1 << 16)), ex23 = p23 - (c2 | (c3 << 16));
    const uint32_t rt0 = t01 & 0xffff, rt1 = t01 >> 16, rt2 = t23 & 0xffff, rt3 = t23 >> 16;
    // within-warp offset of each row's first selected element for this lane
    uint32_t rbase[SEL_ROWS];
    rbase[0] = ex01 & 0xffff;
    rbase[1] = rt0 + (ex01 >> 16);
    rbase[2] = rt0 + rt1 + (ex23 & 0xffff);
    rbase[3] = rt0 + rt1 + rt2 + (ex23 >> 16);
    const uint32_t wtot = rt0 + rt1 + rt2 + rt3;
    if (lane == 0) s_warp[warp] = (int)wtot;
    __syncthreads();
    int wbase = 0, sel_tile = 0;
#pragma unroll
    for (int w = 0; w < SEL_WARPS; ++w) {
        const int x = s_warp[w];
        wbase += w < warp ? x : 0;
        sel_tile += x;
    }

    // compact into shared memory: selected at [0, sel_tile), rejected after them
#pragma unroll
    for (int r = 0; r < SEL_ROWS; ++r) {
        uint32_t s = (uint32_t)wbase + rbase[r];
        // local element index of (r, lane, 0) inside the tile
        const uint32_t e0 = warp * SEL_WARP_ELEMS + r * SEL_ROW_ELEMS + lane * SEL_VEC;
#pragma unroll
        for (int j = 0; j < SEL_VEC; ++j) {
            const bool sel = (m[r] >> j) & 1u;
            if (sel) {
                stage[s] = v[r][j];
                ++s;
            } else if (PARTITION && (int64_t)(e0 + j) < cnt) {
                // rejected before this element inside the tile = e - (selected before it)
                stage[sel_tile + (e0 + j) - s] = v[r][j];
            }
        }
    }
    __syncthreads();

    const int64_t off = offsets[t] >> 2;
    for (int i = threadIdx.x; i < sel_tile; i += SEL_THREADS) out[off + i] = stage[i];
    if constexpr (PARTITION) {
        // rejected elements before this tile = t0 - off; all rejected follow the total
        const int64_t roff = *total + (t0 - off);
        const int rej = (int)cnt - sel_tile;
        for (int i = threadIdx.x; i < rej; i += SEL_THREADS) out[roff + i] = stage[sel_tile + i];
    }
}

}  // namespace ps
