// select_stream.cuh -- single-pass stream compaction: the flags-and-values form of
// the shared-memory-region accumulate-scan (stream_kernel.cuh).
//
// ps_select's three-launch path reads the flags twice (tile counts, then the
// scatter).  Here every region of flags + values is loaded ONCE by TMA into a
// shared-memory buffer of a persistent CTA; the reducers count the selected
// elements of each 512-element chunk, the ledger warp turns the grid's portion
// counts (16-byte epoch-tagged descriptors, as in the scan) into per-chunk output
// offsets, and the scanner warps compute each element's destination in
// registers, compact their chunk in place in shared memory and write it out
// with coalesced stores.  Order-preserving.  Compaction only: a stable
// partition needs the global count before the first rejected element can be
// placed, so it stays on the three-launch path.
#pragma once

#include "stream_kernel.cuh"
#include "select_kernels.cuh"

namespace ps {

struct SelectArgs {
    const void *values;
    const void *flags;
    void *out;
    int64_t n;
    int64_t portion;   // elements per CTA per region (SW chunks)
    int64_t rounds;
    long long *count;  // total selected (device, nullable)
    ulonglong2 *desc;  // rounds * G descriptors
    uint64_t want;     // descriptor tag: (~epoch << 32) | (epoch << 2) -- never matches a small count
    int inflight;      // producer: at most this many regions' loads outstanding (0: NBUF)
};

constexpr int SS_SW = 8, SS_RWP = 4, SS_ROWS = 2, SS_VEC = 8;
// one ledger warp.  (Measured and rejected: two or four ledger warps folding
// alternate regions, and one warp loading the descriptors of four regions per
// round trip -- the extra polling competes with the data streams.)
constexpr int SS_NL = 1;
constexpr int SS_ROW = 32 * SS_VEC;            // 256 elements
constexpr int SS_CHUNK = SS_ROWS * SS_ROW;     // 512 elements: one warp's unit
constexpr int SS_P = SS_SW * SS_CHUNK;         // 4096 elements per CTA per region
constexpr int SS_THREADS = (SS_SW + SS_RWP + 1 + SS_NL) * 32;

template <typename TV, typename TF>
struct SelectStreamGeom {
    static constexpr int FBYTES = SS_P * (int)sizeof(TF);
    static constexpr int VBYTES = SS_P * (int)sizeof(TV);
    static constexpr int BUF = FBYTES + VBYTES;  // multiples of 4 KiB
    static constexpr int NBUF = (196608 / BUF) > 8 ? 8 : (196608 / BUF);
    static constexpr int SMEM = NBUF * BUF + 4 * NBUF * 8 + 2 * NBUF * SS_SW * 8 + 128;
};

// 8 consecutive flags/values of one lane from shared memory
template <typename T>
__device__ __forceinline__ void lds8(const T *p, T (&x)[SS_VEC]) {
    if constexpr (sizeof(T) == 1) {
        uint64_t w;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(w) : "r"(smem_addr(p)));
        memcpy(x, &w, 8);
    } else if constexpr (sizeof(T) == 4) {
        unpack<T>(lds256(p), x);
    } else {
        T lo[4], hi[4];
        unpack<T>(lds256(p), lo);
        unpack<T>(lds256(p + 4), hi);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] = lo[j];
            x[4 + j] = hi[j];
        }
    }
}

template <typename TF>
__device__ __forceinline__ uint32_t flag_bits(const TF (&f)[SS_VEC]) {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < SS_VEC; ++j) m |= (is_set(f[j]) ? 1u : 0u) << j;
    return m;
}

template <typename TV, typename TF>
__global__ void __launch_bounds__(SS_THREADS, 1) select_stream_kernel(const SelectArgs a) {
    using Geo = SelectStreamGeom<TV, TF>;
    constexpr int NBUF = Geo::NBUF;
    constexpr int RT = SS_RWP * 32;
    constexpr int BAR_RED = 1;
    constexpr int W_PROD = SS_SW + SS_RWP, W_LEDGER = SS_SW + SS_RWP + 1;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NBUF * Geo::BUF);
    uint64_t *full = bars, *red = bars + NBUF, *pre = bars + 2 * NBUF, *freeb = bars + 3 * NBUF;
    long long *chunk_tot = reinterpret_cast<long long *>(bars + 4 * NBUF);  // [NBUF][SW]
    long long *chunk_pre = chunk_tot + NBUF * SS_SW;                          // [NBUF][SW]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const TV *values = reinterpret_cast<const TV *>(a.values);
    const TF *flags = reinterpret_cast<const TF *>(a.flags);
    TV *out = reinterpret_cast<TV *>(a.out);
    const int64_t P = SS_P;

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&red[b], 1);
            mbar_init(&pre[b], 1);
            mbar_init(&freeb[b], SS_SW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto par = [&](int64_t r) { return (uint32_t)((r / NBUF) & 1); };
    auto p0_of = [&](int64_t r) { return r * P * G + (int64_t)c * P; };
    auto fbuf = [&](int b) { return reinterpret_cast<TF *>(smem_raw + (size_t)b * Geo::BUF); };
    auto vbuf = [&](int b) { return reinterpret_cast<TV *>(smem_raw + (size_t)b * Geo::BUF + Geo::FBYTES); };

    if (warp == W_PROD) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t r = 0; r < a.rounds; ++r) {
                const int b = (int)(r % NBUF);
                if (r >= NBUF) mbar_wait(&freeb[b], par(r - NBUF));
                if (r >= a.inflight && a.inflight > 0 && a.inflight < NBUF)  // see scan_stream_kernel
                    mbar_wait(&full[(r - a.inflight) % NBUF], par(r - a.inflight));
                const int64_t p0 = p0_of(r);
                if (p0 + P <= a.n) {
                    mbar_expect_tx(&full[b], Geo::BUF);
                    const char *fs = reinterpret_cast<const char *>(flags + p0);
                    const char *vs = reinterpret_cast<const char *>(values + p0);
                    char *fd = reinterpret_cast<char *>(fbuf(b));
                    char *vd = reinterpret_cast<char *>(vbuf(b));
                    for (int o = 0; o < Geo::FBYTES; o += 16384)
                        bulk_g2s(fd + o, fs + o, (uint32_t)(Geo::FBYTES - o < 16384 ? Geo::FBYTES - o : 16384), &full[b],
                                 pol);
                    for (int o = 0; o < Geo::VBYTES; o += 16384)
                        bulk_g2s(vd + o, vs + o, (uint32_t)(Geo::VBYTES - o < 16384 ? Geo::VBYTES - o : 16384), &full[b],
                                 pol);
                } else {
                    mbar_arrive(&full[b]);  // partial / empty portion: consumers read global memory
                }
            }
        }
        return;
    }

    if (warp >= SS_SW && warp < W_PROD) {
        // ---------------- reducers: selected count per chunk, portion count --------------
        const int rw = warp - SS_SW;
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            mbar_wait(&full[b], par(r));
            long long *tot = chunk_tot + b * SS_SW;
            const int64_t p0 = p0_of(r);
            const bool whole = p0 + P <= a.n;
            for (int ch = rw; ch < SS_SW; ch += SS_RWP) {
                int cnt = 0;
#pragma unroll
                for (int rr = 0; rr < SS_ROWS; ++rr) {
                    const int e0 = ch * SS_CHUNK + rr * SS_ROW + lane * SS_VEC;
                    if (whole) {
                        TF f[SS_VEC];
                        lds8<TF>(fbuf(b) + e0, f);
                        cnt += __popc(flag_bits<TF>(f));
                    } else {
                        for (int j = 0; j < SS_VEC; ++j)
                            if (p0 + e0 + j < a.n && is_set(flags[p0 + e0 + j])) ++cnt;
                    }
                }
                cnt = (int)__reduce_add_sync(FULL, (unsigned)cnt);
                if (lane == 0) tot[ch] = cnt;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_sync(BAR_RED, RT);
            if (rw == 0) {
                long long t = lane < SS_SW ? tot[lane] : 0;
                t = (long long)__reduce_add_sync(FULL, (unsigned)t);  // <= 4096 per portion
                if (lane == 0) {
                    st_desc(a.desc + r * G + c, a.want | ST_A, (uint64_t)t);
                    mbar_arrive(&red[b]);
                }
            }
            named_sync(BAR_RED, RT);
        }
        return;
    }

    if (warp == W_LEDGER) {
        // ---------------- ledger: per-chunk output offsets -----------------------------
        long long carry = 0;
        // the next region's gather is issued as soon as this one's descriptors arrived
        // and the chunk scan runs inside the round trip (as in scan_stream_kernel)
        const bool overlap = G <= 32 * GATHER_LP;
        ulonglong2 dn[GATHER_LP];
        if (overlap) desc_issue(dn, a.desc, G, lane);
        for (int64_t r = 0; r < a.rounds; ++r) {
            const int b = (int)(r % NBUF);
            mbar_wait(&red[b], par(r));
            const long long *tot = chunk_tot + b * SS_SW;
            long long *pr = chunk_pre + b * SS_SW;
            const long long t = lane < SS_SW ? tot[lane] : 0;
            long long inc = t;
#pragma unroll
            for (int d = 1; d < SS_SW; d <<= 1) {
                const long long y = __shfl_up_sync(FULL, inc, d);
                if (lane >= d) inc += y;
            }
            long long sb = 0, sa = 0;
#ifndef PS_EXP_NOLEDGER
            if (overlap) {
                desc_wait(dn, a.desc + r * G, G, a.want, lane);
#pragma unroll
                for (int i = 0; i < GATHER_LP; ++i) {  // gather_totals' order
                    const int j = lane + 32 * i;
                    if (j < G) {
                        const long long v = (long long)dn[i].y;
                        sa += v;
                        if (j < c) sb += v;
                    }
                }
                if (r + 1 < a.rounds) desc_issue(dn, a.desc + (r + 1) * G, G, lane);
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    sa += __shfl_xor_sync(FULL, sa, d);
                    sb += __shfl_xor_sync(FULL, sb, d);
                }
            } else {
                gather_totals<long long>(a.desc + r * G, G, c, a.want, lane, sb, sa);
            }
#endif
            if (lane < SS_SW) pr[lane] = carry + sb + inc - t;
            carry += sa;
            __syncwarp();
            if (lane == 0) mbar_arrive(&pre[b]);
        }
        if (c == 0 && lane == 0 && a.count) *a.count = carry;
        return;
    }

    // ---------------- scanners: destinations, in-place compaction, coalesced writes ------
    for (int64_t r = 0; r < a.rounds; ++r) {
        const int b = (int)(r % NBUF);
        mbar_wait(&pre[b], par(r));
        const int64_t p0 = p0_of(r);
        const bool whole = p0 + P <= a.n;
        const int ch = warp;
        const long long base = chunk_pre[b * SS_SW + ch];
        TV v[SS_ROWS][SS_VEC];
        uint32_t m[SS_ROWS];
#pragma unroll
        for (int rr = 0; rr < SS_ROWS; ++rr) {
            const int e0 = ch * SS_CHUNK + rr * SS_ROW + lane * SS_VEC;
            if (whole) {
                TF f[SS_VEC];
                lds8<TF>(fbuf(b) + e0, f);
                lds8<TV>(vbuf(b) + e0, v[rr]);
                m[rr] = flag_bits<TF>(f);
            } else {
                m[rr] = 0;
#pragma unroll
                for (int j = 0; j < SS_VEC; ++j) {
                    const int64_t i = p0 + e0 + j;
                    if (i < a.n) {
                        v[rr][j] = values[i];
                        m[rr] |= (is_set(flags[i]) ? 1u : 0u) << j;
                    } else {
                        memset(&v[rr][j], 0, sizeof(TV));
                    }
                }
            }
        }
        // lane-exclusive offsets of the two rows, packed in 16-bit halves
        const uint32_t c0 = __popc(m[0]), c1 = __popc(m[1]);
        uint32_t p = c0 | (c1 << 16);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, p, d);
            if (lane >= d) p += y;
        }
        const uint32_t tot01 = __shfl_sync(FULL, p, 31);
        const uint32_t ex = p - (c0 | (c1 << 16));
        const uint32_t rt0 = tot01 & 0xffff, k = rt0 + (tot01 >> 16);
        // compact this chunk in place: every lane's values are in registers now
        TV *stage = vbuf(b) + ch * SS_CHUNK;
        __syncwarp();
        uint32_t s0 = ex & 0xffff, s1 = rt0 + (ex >> 16);
#pragma unroll
        for (int j = 0; j < SS_VEC; ++j) {
            if ((m[0] >> j) & 1u) stage[s0++] = v[0][j];
        }
#pragma unroll
        for (int j = 0; j < SS_VEC; ++j) {
            if ((m[1] >> j) & 1u) stage[s1++] = v[1][j];
        }
        __syncwarp();
        // coalesced write-out, four independent loads in flight per lane
        uint32_t i = lane;
        for (; i + 96 < k; i += 128) {
            const TV y0 = stage[i], y1 = stage[i + 32], y2 = stage[i + 64], y3 = stage[i + 96];
            out[base + i] = y0;
            out[base + i + 32] = y1;
            out[base + i + 64] = y2;
            out[base + i + 96] = y3;
        }
        for (; i < k; i += 32) out[base + i] = stage[i];
        // everything read from this buffer has been consumed; hand it back to the TMA
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[b]);
    }
}

}  // namespace ps
