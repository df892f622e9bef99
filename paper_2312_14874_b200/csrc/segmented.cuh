// segmented.cuh -- CSR-segmented look-back scan (many independent rows of
// arbitrary length packed back to back in one buffer).
//
// No reference kernel has this shape; it is the general form of the
// per-chunk scans of simd.py:164-206 (chunks = segments, totals_out = segment
// totals) with segment boundaries taken from an offsets array instead of a
// fixed stride.  The scan operator is the segmented sum on (head-flag, value)
// pairs:  (f1, v1) . (f2, v2) = (f1 | f2,  f2 ? v2 : v1 + v2).  A tile that
// contains a segment head can publish its inclusive value immediately (status
// P), so look-backs never cross a segment boundary.
#pragma once

#include "scan_kernels.cuh"

namespace ps {

struct SegArgs {
    const void *in;
    void *out;
    int64_t n;
    int64_t lead;
    const int64_t *offsets;  // nseg + 1 entries
    int64_t nseg;
    void *totals;  // acc-typed per segment (pre-zeroed by the host)
    const int64_t *tile_seg;  // [tiles]: segment holding each tile's first element (seg_tile_kernel)
    int64_t ucols;            // > 0: uniform segments of ucols elements (contiguous batched rows), no offsets
    Desc desc;
    uint32_t epoch;
    int exclusive;
    int vec_ok;
};

// last s in [0, nseg) with offsets[s] <= e (offsets[0] == 0 <= e)
__device__ __forceinline__ int64_t seg_of(const int64_t *off, int64_t nseg, int64_t e) {
    int64_t lo = 0, hi = nseg;  // invariant: off[lo] <= e, answer < hi
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= e) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Segment of every tile's first element, one thread per tile: a galloping search
// from the guess e * nseg / n (uniform segments: a couple of dependent loads), so
// the scan kernel needs no per-lane binary searches over the whole offsets array
// (each was ~log2(nseg) dependent L2 round trips under full load).
__global__ void seg_tile_kernel(const int64_t *off, int64_t nseg, int64_t n, int64_t lead, int64_t tile_elems,
                                int64_t tiles, int64_t *tile_seg) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= tiles) return;
    int64_t e = t * tile_elems - lead;
    if (e < 0) e = 0;
    if (e > n - 1) e = n - 1;
    // largest s in [0, nseg) with off[s] <= e (off[0] == 0 <= e)
    int64_t g = (int64_t)((double)e / (double)n * (double)nseg);
    if (g > nseg - 1) g = nseg - 1;
    if (g < 0) g = 0;
    int64_t lo, hi;  // invariant: off[lo] <= e, answer < hi
    if (__ldg(off + g) <= e) {
        lo = g;
        int64_t step = 1;
        while (lo + step < nseg && __ldg(off + lo + step) <= e) {
            lo += step;
            step <<= 1;
        }
        hi = lo + step < nseg ? lo + step : nseg;
    } else {
        hi = g;
        int64_t step = 1;
        while (hi - step > 0 && __ldg(off + hi - step) > e) {
            hi -= step;
            step <<= 1;
        }
        lo = hi - step > 0 ? hi - step : 0;
    }
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= e) lo = mid;
        else hi = mid;
    }
    // stored as lo << 2: the low two bits of every word stay 0, so no word of this
    // array can ever pass for a published look-back descriptor (status != 0) when a
    // later scan reuses the scratch with a small epoch
    tile_seg[t] = lo << 2;
}

constexpr int SEG_CACHE = 4096;  // offsets of one tile's segments kept in shared memory (2 CTAs/SM by registers anyway)

template <typename A> struct Pair {
    A v;
    int f;
};
template <typename A> __device__ __forceinline__ Pair<A> combine(Pair<A> a, Pair<A> b) {
    return Pair<A>{b.f ? b.v : a.v + b.v, a.f | b.f};
}

template <typename TIn, typename TOut, int WARPS, int ROWS>
__global__ void __launch_bounds__(WARPS * 32, PS_TILES_MINB) seg_scan_kernel(const SegArgs a) {
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = 32 / sizeof(TIn);
    constexpr int ROW_ELEMS = 32 * VEC;
    constexpr int WARP_ELEMS = ROWS * ROW_ELEMS;
    constexpr int64_t TILE = (int64_t)WARPS * WARP_ELEMS;
    static_assert(ROWS * VEC <= 32, "head mask is 32 bits");

    __shared__ A s_wv[WARPS];
    __shared__ int s_wf[WARPS];
    __shared__ A s_base[WARPS];
    __shared__ int64_t s_off[SEG_CACHE];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tile = blockIdx.x;
    const int64_t t0 = tile * TILE;
    const int64_t lo = a.lead, hi = a.lead + a.n;
    const TIn *in = reinterpret_cast<const TIn *>(a.in) - a.lead + t0;
    TOut *out = reinterpret_cast<TOut *>(a.out) - a.lead + t0;
    const bool full = a.vec_ok && t0 >= lo && t0 + TILE <= hi;
    const int64_t my0 = (int64_t)warp * WARP_ELEMS + lane * VEC;

    TIn x[ROWS][VEC];
    if (full) {
        V256 raw[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) raw[r] = ldg256_stream(in + my0 + r * ROW_ELEMS);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) unpack<TIn>(raw[r], x[r]);
    } else {
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const int64_t pos = t0 + my0 + r * ROW_ELEMS + j;
                x[r][j] = (pos >= lo && pos < hi) ? in[my0 + r * ROW_ELEMS + j] : (TIn)0;
            }
    }

    // this tile's segments are [s_lo, s_hi]; their offsets (s_lo .. s_hi + 1) are
    // cached in shared memory when they fit, so every lookup below is local
    int64_t s_lo, s_hi;
    if (a.ucols) {  // uniform segments: everything is arithmetic
        const int64_t e_first = t0 - a.lead > 0 ? t0 - a.lead : 0;
        const int64_t e_next = t0 + TILE - a.lead < a.n ? t0 + TILE - a.lead : a.n - 1;
        s_lo = e_first / a.ucols;
        s_hi = e_next / a.ucols;
    } else {
        s_lo = a.tile_seg[tile] >> 2;
        s_hi = tile + 1 < (int64_t)gridDim.x ? (a.tile_seg[tile + 1] >> 2) : a.nseg - 1;
    }
    const bool cached = !a.ucols && s_hi - s_lo + 2 <= SEG_CACHE;
    if (cached)
        for (int64_t i = threadIdx.x; i <= s_hi - s_lo + 1; i += blockDim.x) s_off[i] = __ldg(a.offsets + s_lo + i);
    __syncthreads();
    auto off_at = [&](int64_t sg) {
        if (a.ucols) return sg * a.ucols < a.n ? sg * a.ucols : a.n;
        return cached ? s_off[sg - s_lo] : __ldg(a.offsets + sg);
    };
    auto seg_at = [&](int64_t e) {  // largest s in [s_lo, s_hi] with off[s] <= e
        int64_t lo = s_lo, hi = s_hi + 1;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (off_at(mid) <= e) lo = mid;
            else hi = mid;
        }
        return lo;
    };

    // segment heads inside this thread's elements (bit r*VEC + j); element e
    // is a head iff it starts a non-empty segment: off[seg_of(e)] == e
    uint32_t heads = 0;
    int64_t seg0[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        const int64_t e0 = t0 + my0 + r * ROW_ELEMS - a.lead;  // element index of (r, 0)
        int64_t s = -1, nb = 0;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const int64_t e = e0 + j;
            if (e < 0 || e >= a.n) continue;
            if (s < 0) {
                s = seg_at(e);
                nb = off_at(s + 1);
                if (off_at(s) == e) heads |= 1u << (r * VEC + j);
                seg0[r] = s;
            } else if (e == nb) {
                while (off_at(s + 1) <= e) ++s;
                nb = off_at(s + 1);
                heads |= 1u << (r * VEC + j);
            }
        }
        if (s < 0) seg0[r] = 0;
    }

    // per-lane segmented sums, warp pair scans, row / warp combines
    Pair<A> lp[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        Pair<A> p{(A)0, 0};
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            if (heads & (1u << (r * VEC + j))) p = Pair<A>{(A)x[r][j], 1};
            else p.v += (A)x[r][j];
        }
        lp[r] = p;
    }
    Pair<A> sc[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) sc[r] = lp[r];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
            Pair<A> y{shfl_up(sc[r].v, d), shfl_up(sc[r].f, d)};
            if (lane >= d) sc[r] = combine(y, sc[r]);
        }
    }
    Pair<A> lex[ROWS];
    Pair<A> wrun{(A)0, 0};
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        Pair<A> ex{shfl_up(sc[r].v, 1), shfl_up(sc[r].f, 1)};
        if (lane == 0) ex = Pair<A>{(A)0, 0};
        const Pair<A> rt{shfl_idx(sc[r].v, 31), shfl_idx(sc[r].f, 31)};
        lex[r] = combine(wrun, ex);
        wrun = combine(wrun, rt);
    }
    if (lane == 0) {
        s_wv[warp] = wrun.v;
        s_wf[warp] = wrun.f;
    }
    __syncthreads();

    if (warp == 0) {
        // serial combine over WARPS (tiny), lane-parallel result
        Pair<A> run{(A)0, 0}, mine{(A)0, 0};
        for (int w = 0; w < WARPS; ++w) {
            if (lane == w) mine = run;
            run = combine(run, Pair<A>{s_wv[w], s_wf[w]});
        }
        const Pair<A> agg = run;
        A excl;
        if (tile == 0) {
            excl = (A)0;
            if (lane == 0) publish(a.desc, tile, a.epoch, ST_P, acc_to_bits<A>(agg.v));
        } else {
            if (lane == 0) publish(a.desc, tile, a.epoch, agg.f ? ST_P : ST_A, acc_to_bits<A>(agg.v));
            excl = lookback<A>(a.desc, tile, 0, a.epoch, lane);
            if (lane == 0 && !agg.f) publish(a.desc, tile, a.epoch, ST_P, acc_to_bits<A>(excl + agg.v));
        }
        if (lane < WARPS) s_base[lane] = mine.f ? mine.v : excl + mine.v;
    }
    __syncthreads();

    const A wbase = s_base[warp];
    A *tot = reinterpret_cast<A *>(a.totals);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
        A run = lex[r].f ? lex[r].v : wbase + lex[r].v;
        int64_t s = seg0[r];
        TOut y[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const bool h = heads & (1u << (r * VEC + j));
            const A before = h ? (A)0 : run;
            run = before + (A)x[r][j];
            y[j] = (TOut)(a.exclusive ? before : run);
            const int64_t e = t0 + my0 + r * ROW_ELEMS + j - a.lead;
            if (tot && e >= 0 && e < a.n) {
                if (h) {
                    while (off_at(s + 1) <= e) ++s;
                }
                if (e + 1 == off_at(s + 1)) tot[s] = run;
            }
        }
        if (full) {
            constexpr int NV = VEC * sizeof(TOut) / 32;
#pragma unroll
            for (int k = 0; k < NV; ++k)
                stg256_stream(out + my0 + r * ROW_ELEMS + k * (32 / sizeof(TOut)), pack<TOut>(&y[k * (32 / sizeof(TOut))]));
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const int64_t pos = t0 + my0 + r * ROW_ELEMS + j;
                if (pos >= lo && pos < hi) out[my0 + r * ROW_ELEMS + j] = y[j];
            }
        }
    }
}

inline size_t seg_align_up(size_t x, size_t al) { return (x + al - 1) / al * al; }

inline int64_t seg_tile_elems(int elem_bytes) { return (int64_t)8 * 4 * 32 * (32 / elem_bytes); }

inline size_t seg_scratch_bytes(int64_t n, int elem_bytes) {
    const int64_t tiles = (n + seg_tile_elems(elem_bytes) - 1) / seg_tile_elems(elem_bytes) + 1;
    return 256 + seg_align_up((size_t)tiles * 16, 256) + seg_align_up((size_t)tiles * 8, 256);
}

template <typename TIn, typename TOut>
int launch_segmented(const void *in, void *out, int64_t n, const int64_t *offsets, int64_t nseg, int exclusive,
                     void *totals, void *scratch, uint32_t epoch, cudaStream_t s, int64_t ucols = 0) {
    constexpr int64_t TILE = (int64_t)8 * 4 * 32 * (32 / sizeof(TIn));
    SegArgs a{};
    a.in = in;
    a.out = out;
    a.n = n;
    a.offsets = offsets;
    a.nseg = nseg;
    a.totals = totals;
    a.epoch = epoch;
    a.exclusive = exclusive;
    const uintptr_t ain = (uintptr_t)in % 32;
    int64_t lead = (ain % sizeof(TIn)) ? -1 : (int64_t)(ain / sizeof(TIn));
    bool vec = lead >= 0 && ((uintptr_t)out % 32) == (uintptr_t)((lead * sizeof(TOut)) % 32) &&
               (uintptr_t)out % sizeof(TOut) == 0 && lead * (int64_t)sizeof(TOut) < 32;
    a.vec_ok = vec;
    a.lead = vec ? lead : 0;
    const int64_t tiles = (a.lead + n + TILE - 1) / TILE;
    if (tiles > 0x7fffffffLL) return 2;
    a.desc.d = reinterpret_cast<ulonglong2 *>(static_cast<char *>(scratch) + 256);
    // tile -> first segment, after the descriptors (seg_scratch_bytes reserves tiles + 1 of each)
    const int64_t cap = (n + TILE - 1) / TILE + 1;
    int64_t *tile_seg = reinterpret_cast<int64_t *>(static_cast<char *>(scratch) + 256 + seg_align_up((size_t)cap * 16, 256));
    a.tile_seg = tile_seg;
    a.ucols = ucols;
    if (!ucols)
        seg_tile_kernel<<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(offsets, nseg, n, a.lead, TILE, tiles, tile_seg);
    seg_scan_kernel<TIn, TOut, 8, 4><<<(unsigned)tiles, 256, 0, s>>>(a);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : 1000 + (int)e;
}

}  // namespace ps
