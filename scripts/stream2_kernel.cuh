// scripts/stream2_kernel.cuh -- EXPERIMENT (dev tool, not in the library): the
// stream kernel without reducer warps.  The scanner warps compute their chunk's
// in-register scan as soon as the data lands, publish the chunk totals themselves
// (one named barrier per group), and finish (carry adds + stores) after the
// ledger; NG groups of SW scanner warps alternate regions so that one group's
// ledger wait overlaps the other's front half.  Each element is read from shared
// memory once and no TwoSum reducer runs.
#pragma once

#include "../paper_2312_14874_b200/csrc/stream_kernel.cuh"

namespace ps {

template <typename TIn, typename TOut, int SW, int ROWS, int NBUF, int NG>
struct Stream2Geom {
    static constexpr int WARPS = SW * NG + 2;
    static constexpr int THREADS = WARPS * 32;
    static constexpr int VEC = 32 / sizeof(TIn);
    static constexpr int ROW_ELEMS = 32 * VEC;
    static constexpr int CHUNK = ROWS * ROW_ELEMS;
    static constexpr int SMEM_FIXED = 4 * NBUF * 8 + 2 * NBUF * SW * 8 + 128;
    static constexpr int smem(int64_t portion) { return (int)(NBUF * portion * sizeof(TIn)) + SMEM_FIXED; }
};

template <typename TIn, typename TOut, int SW, int ROWS, int NBUF, int NG>
__global__ void __launch_bounds__((SW * NG + 2) * 32, 1) scan_stream2_kernel(const StreamArgs a) {
    using Geo = Stream2Geom<TIn, TOut, SW, ROWS, NBUF, NG>;
    using A = typename AccOf<TIn>::type;
    constexpr int VEC = Geo::VEC, ROW_ELEMS = Geo::ROW_ELEMS, CHUNK = Geo::CHUNK;
    constexpr bool FLOAT = (A)0.5 != (A)0;
    constexpr int W_PROD = SW * NG, W_LEDGER = SW * NG + 1;
    static_assert(NBUF % NG == 0, "a buffer must always serve the same group");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    TIn *buf = reinterpret_cast<TIn *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NBUF * a.portion * sizeof(TIn));
    uint64_t *full = bars, *red = bars + NBUF, *pre = bars + 2 * NBUF, *freeb = bars + 3 * NBUF;
    A *chunk_tot = reinterpret_cast<A *>(bars + 4 * NBUF);  // [NBUF][SW]
    A *chunk_pre = chunk_tot + NBUF * SW;                    // [NBUF][SW]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const TIn *in = reinterpret_cast<const TIn *>(a.in);
    TOut *out = reinterpret_cast<TOut *>(a.out);
    const uint64_t want = (uint64_t)a.epoch << 2;
    const int64_t P = a.portion;  // == SW * CHUNK

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&red[b], 1);
            mbar_init(&pre[b], 1);
            mbar_init(&freeb[b], SW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto par = [&](int64_t r) { return (uint32_t)((r / NBUF) & 1); };
    auto p0_of = [&](int64_t r) { return r * P * G + (int64_t)c * P; };
    auto whole = [&](int64_t r) {
        const int64_t p0 = p0_of(r);
        return p0 >= a.lo && p0 + P <= a.hi;
    };

    if (warp == W_PROD) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                if (r >= NBUF) mbar_wait(&freeb[b], par(r - NBUF));
                if (whole(r)) {
                    const uint32_t bytes = (uint32_t)(P * sizeof(TIn));
                    mbar_expect_tx(&full[b], bytes);
                    const char *src = reinterpret_cast<const char *>(in + p0_of(r));
                    char *dst = reinterpret_cast<char *>(buf + (size_t)b * P);
                    for (uint32_t o = 0; o < bytes; o += 16384)
                        bulk_g2s(dst + o, src + o, bytes - o < 16384u ? bytes - o : 16384u, &full[b], pol);
                } else {
                    mbar_arrive(&full[b]);
                }
            }
        }
        return;
    }

    if (warp == W_LEDGER) {
        A carry = acc_from_bits<A>(a.seed_bits);
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            A sb, sa;
            gather_totals<A>(a.desc + r * G, G, c, want, lane, sb, sa);
            mbar_wait(&red[b], par(r));
            const A t = lane < SW ? chunk_tot[b * SW + lane] : (A)0;
            A inc = t;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const A y = shfl_up(inc, d);
                if (lane >= d) inc += y;
            }
            A ex = shfl_up(inc, 1);
            if (lane == 0) ex = (A)0;
            if (lane < SW) chunk_pre[b * SW + lane] = carry + sb + ex;
            carry += sa;
            __syncwarp();
            if (lane == 0) mbar_arrive(&pre[b]);
        }
        if (c == 0 && lane == 0 && a.total) *reinterpret_cast<A *>(a.total) = carry;
        return;
    }

    // ---- scanner groups ----
    const int g = warp / SW, w = warp % SW;
    const uint64_t pol = policy_evict_first();
    for (int64_t r = g; r < a.rounds; r += NG) {
        const int b = (int)(r % NBUF);
        mbar_wait(&full[b], par(r));
        const TIn *sbuf = buf + (size_t)b * P;
        const int64_t p0 = p0_of(r);
        const bool wh = whole(r);
        const int64_t t0 = p0 + (int64_t)w * CHUNK;
        A v[ROWS][VEC];
        if (wh) {
            V256 raw[ROWS];
#pragma unroll
            for (int rr = 0; rr < ROWS; ++rr) raw[rr] = lds256<(sizeof(TIn) == 8)>(sbuf + w * CHUNK + rr * ROW_ELEMS + lane * VEC);
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
        A ctot = (A)0;
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) {
            if constexpr (FLOAT) {
                exs[rr] = shfl_up(sc[rr], 1);
                if (lane == 0) exs[rr] = (A)0;
            } else {
                exs[rr] = sc[rr] - v[rr][VEC - 1];
            }
            rts[rr] = shfl_idx(sc[rr], 31);
            ctot += rts[rr];
        }
        if (lane == 0) chunk_tot[b * SW + w] = ctot;
        named_sync(1 + g, SW * 32);
        if (w == 0) {  // the portion total -> the grid ledger
            A t = lane < SW ? chunk_tot[b * SW + lane] : (A)0;
            t = warp_sum(t);
            if (lane == 0) {
                st_desc(a.desc + r * G + c, want | ST_A, acc_to_bits<A>(t));
                mbar_arrive(&red[b]);
            }
        }
        mbar_wait(&pre[b], par(r));
        A base = chunk_pre[b * SW + w];
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
            if (wh) {
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
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[b]);
    }
}

}  // namespace ps
