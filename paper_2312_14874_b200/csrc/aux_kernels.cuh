// aux_kernels.cuh -- the smaller kernels behind the remaining reference entry
// points on the hot path:
//
//   shift_gather_kernel / shift_tiles_kernel
//       exclusive_from_inclusive (core.py:141-151, _shift_right_kernel
//       core.py:109-115) in place in one read + one write: the element each
//       tile needs from its predecessor is gathered first, then every tile
//       shifts itself through shared memory.
//   reduce_rows_kernel
//       per-chunk totals (simd.py:178-186 _vertical_pass1_accumulate).
//   add_rows_kernel
//       per-chunk increments (simd.py:189-195 _vertical_pass2_increment).
//   wrapped_block_total_kernel
//       the total the reference's horizontal kernel returns for uint32 data
//       (simd.py:84-99: each w-block is reduced in uint32 registers, so the
//       carried total only keeps every block's sum mod 2^32).
#pragma once

#include "scan_kernels.cuh"

namespace ps {

constexpr int SHIFT_THREADS = 256;
constexpr int SHIFT_ITEMS = 16;
constexpr int64_t SHIFT_TILE = SHIFT_THREADS * SHIFT_ITEMS;

template <typename T>
__global__ void shift_gather_kernel(const T *in, int64_t n, int64_t tiles, T *bound, T *last_out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 1 && t < tiles) bound[t] = in[t * SHIFT_TILE - 1];
    if (t == 0 && last_out) *last_out = in[n - 1];
}

template <typename T>
__global__ void __launch_bounds__(SHIFT_THREADS)
    shift_tiles_kernel(const T *in, T *out, int64_t n, const T *bound, uint64_t ident_bits) {
    __shared__ T tile[SHIFT_TILE];
    const int64_t base = (int64_t)blockIdx.x * SHIFT_TILE;
    const int64_t cnt = n - base < SHIFT_TILE ? n - base : SHIFT_TILE;
#pragma unroll
    for (int k = 0; k < SHIFT_ITEMS; ++k) {
        const int i = k * SHIFT_THREADS + threadIdx.x;
        if (i < cnt) tile[i] = in[base + i];
    }
    __syncthreads();  // the whole tile is read before any of it is overwritten
    T ident;
    memcpy(&ident, &ident_bits, sizeof(T));
    const T first = blockIdx.x == 0 ? ident : bound[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SHIFT_ITEMS; ++k) {
        const int i = k * SHIFT_THREADS + threadIdx.x;
        if (i < cnt) out[base + i] = i == 0 ? first : tile[i - 1];
    }
}

template <typename T, int THREADS>
__global__ void __launch_bounds__(THREADS)
    reduce_rows_kernel(const T *in, int64_t cols, int64_t ld, void *totals) {
    using A = typename AccOf<T>::type;
    __shared__ A smem[THREADS / 32];
    const T *row = in + (int64_t)blockIdx.x * ld;
    A acc = (A)0;
    for (int64_t c = threadIdx.x; c < cols; c += THREADS) acc += (A)row[c];
    acc = block_sum<A, THREADS>(acc, smem);
    if (threadIdx.x == 0) reinterpret_cast<A *>(totals)[blockIdx.x] = acc;
}

template <typename T>
__global__ void add_rows_kernel(T *buf, int64_t cols, int64_t ld, const void *deltas) {
    using A = typename AccOf<T>::type;
    const A d = reinterpret_cast<const A *>(deltas)[blockIdx.y];
    T *row = buf + (int64_t)blockIdx.y * ld;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x)
        row[c] = (T)((A)row[c] + d);
}

__global__ void wrapped_block_total_kernel(const uint32_t *in, int64_t n, int w, unsigned long long *total) {
    const int64_t nblk = n / w;
    unsigned long long acc = 0;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblk; b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int j = 0; j < w; ++j) s += in[b * w + j];  // wraps like the w-lane register
        acc += s;
    }
    if (blockIdx.x == 0)
        for (int64_t i = nblk * w + threadIdx.x; i < n; i += blockDim.x) acc += in[i];  // scalar tail
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(total, acc);
}

}  // namespace ps

namespace ps {

// ---- Blelloch tree step functions: up_sweep / down_sweep (simd.py:327-367) ---------------
// Element-typed arithmetic (uint32 wraps, float32 adds in float32) in exactly the
// reference's pairing, so float results are bit-identical.  Levels with stride
// below TREE_B run inside one CTA's shared-memory block; the top levels (a
// handful for any n) run one launch each.
constexpr int TREE_B = 2048;
constexpr int TREE_THREADS = 1024;

template <typename T>
__device__ __forceinline__ T tree_add(T a, T b) {
    return (T)(a + b);
}

template <typename T>
__global__ void __launch_bounds__(TREE_THREADS) tree_up_block_kernel(T *d, int64_t n, int64_t blk) {
    __shared__ T s[TREE_B];
    T *base = d + (int64_t)blockIdx.x * blk;
    for (int i = threadIdx.x; i < blk; i += TREE_THREADS) s[i] = base[i];
    __syncthreads();
    for (int stride = 1; stride < blk; stride *= 2) {
        const int step = stride * 2;
        for (int k = threadIdx.x; (int64_t)(k + 1) * step - 1 < blk; k += TREE_THREADS) {
            const int i = (k + 1) * step - 1;
            s[i] = tree_add(s[i], s[i - stride]);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < blk; i += TREE_THREADS) base[i] = s[i];
}

template <typename T>
__global__ void tree_up_level_kernel(T *d, int64_t n, int64_t stride) {
    const int64_t step = stride * 2;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; (k + 1) * step - 1 < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = (k + 1) * step - 1;
        d[i] = tree_add(d[i], d[i - stride]);
    }
}

template <typename T>
__global__ void tree_down_level_kernel(T *d, int64_t n, int64_t stride, int clear_root) {
    const int64_t step = stride * 2;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; (k + 1) * step - 1 < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = (k + 1) * step - 1;
        const T t = d[i - stride];
        const T top = (clear_root && i == n - 1) ? (T)0 : d[i];
        d[i - stride] = top;
        d[i] = tree_add(top, t);
    }
}

template <typename T>
__global__ void __launch_bounds__(TREE_THREADS) tree_down_block_kernel(T *d, int64_t n, int64_t blk, int clear_root) {
    __shared__ T s[TREE_B];
    T *base = d + (int64_t)blockIdx.x * blk;
    for (int i = threadIdx.x; i < blk; i += TREE_THREADS) s[i] = base[i];
    __syncthreads();
    if (clear_root && threadIdx.x == 0) s[blk - 1] = (T)0;  // n <= TREE_B: the root lives here
    __syncthreads();
    for (int stride = (int)(blk / 2); stride >= 1; stride /= 2) {
        const int step = stride * 2;
        for (int k = threadIdx.x; (int64_t)(k + 1) * step - 1 < blk; k += TREE_THREADS) {
            const int i = (k + 1) * step - 1;
            const T t = s[i - stride];
            s[i - stride] = s[i];
            s[i] = tree_add(s[i], t);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < blk; i += TREE_THREADS) base[i] = s[i];
}

}  // namespace ps
