// prefixscan_b200.cu -- C-ABI of libprefixscan_b200.so (see include/prefixscan_b200.h).
//
// Host side of the sm_100a scan path: argument validation (the reference's
// ValueError cases map to PS_ERR_*), dtype-pair dispatch, tile geometry,
// scratch carving, launches, and the pipelined host-buffer entry point.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>
#include <cstdio>
#include <type_traits>

#include "../../include/prefixscan_b200.h"
#include "scan_kernels.cuh"
#include "segmented.cuh"
#include "aux_kernels.cuh"
#include "rounds_kernel.cuh"
#include "stream_kernel.cuh"
#include "seg_stream.cuh"
#include "rows_kernel.cuh"
#include "select_kernels.cuh"
#include "select_stream.cuh"
#include "host_pipeline.h"

namespace ps {
namespace {

constexpr int SCAN_WARPS = 8;
constexpr int SCAN_ROWS = 4;
constexpr int REDUCE_THREADS = 512;

template <typename TIn> constexpr int64_t tile_elems() {
    return (int64_t)SCAN_WARPS * SCAN_ROWS * 32 * (32 / sizeof(TIn));
}

size_t dsize(int dt) {
    switch (dt) {
        case PS_DTYPE_INT32: case PS_DTYPE_UINT32: case PS_DTYPE_FLOAT32: return 4;
        case PS_DTYPE_INT64: case PS_DTYPE_UINT64: case PS_DTYPE_FLOAT64: return 8;
        default: return 0;
    }
}

bool pair_ok(int i, int o) {
    switch (i) {
        case PS_DTYPE_INT32: return o == PS_DTYPE_INT32 || o == PS_DTYPE_INT64;
        case PS_DTYPE_INT64: return o == PS_DTYPE_INT64;
        case PS_DTYPE_UINT32: return o == PS_DTYPE_UINT32 || o == PS_DTYPE_UINT64;
        case PS_DTYPE_UINT64: return o == PS_DTYPE_UINT64;
        case PS_DTYPE_FLOAT32: return o == PS_DTYPE_FLOAT32 || o == PS_DTYPE_FLOAT64;
        case PS_DTYPE_FLOAT64: return o == PS_DTYPE_FLOAT64;
        default: return false;
    }
}

int64_t tile_of_dtype(int dt) { return (int64_t)SCAN_WARPS * SCAN_ROWS * 32 * (int64_t)(32 / (dsize(dt) ? dsize(dt) : 4)); }

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// look-back scratch: 256 bytes of control words, then one 16-byte descriptor per tile
size_t desc_bytes(int64_t tiles) { return 256 + align_up((size_t)tiles * 16, 256); }

Desc carve_desc(void *scratch, int64_t tiles) {
    (void)tiles;
    Desc d;
    d.d = reinterpret_cast<ulonglong2 *>(static_cast<char *>(scratch) + 256);
    return d;
}

int cuda_rc(cudaError_t e) { return e == cudaSuccess ? PS_OK : PS_ERR_CUDA_BASE + (int)e; }

int launch_rc() { return cuda_rc(cudaGetLastError()); }

bool overlaps_partially(const void *a, size_t abytes, const void *b, size_t bbytes) {
    if (a == b) return false;
    const uintptr_t a0 = (uintptr_t)a, a1 = a0 + abytes, b0 = (uintptr_t)b, b1 = b0 + bbytes;
    return a0 < b1 && b0 < a1;
}

// ---- tuning (ps_set_tuning) ----------------------------------------------------------------
struct Tuning {
    int scan_kernel = 0;                    // 0 auto, 1 look-back, 2 cache-partitioned rounds
    int64_t round_bytes = 0;                // input + output bytes per L2 region (0 = per-dtype default)
    int64_t rounds_min_bytes = 32ll << 20;  // auto: stream kernel from this many input bytes (scripts/crossover.py)
    int64_t round_lead = 2;                 // regions the reducer warps may run ahead of the scanners
    int64_t round_ramp = 0;                 // ramp regions at each end (sizes P/2^k .. P/2); 0 = off
    int64_t round_prefetch = 0;             // bulk L2 prefetch of each reducer portion (1 = on)
    int rows_kernel = 0;                    // batched: 0 auto, 1 look-back tiles, 2 one CTA per row
    int stream_inflight = 2;                // stream kernel: regions' TMA loads outstanding per SM (0 = ring)
    int stream_copy_in = 1;                 // stream kernel for in/out pairs at different 32-byte phases (0: look-back tiles)
    int rows_dynamic = 1;                   // rows kernel: rows from a grid-wide ticket (0 = fixed shares)
    int reduce_blocks = 1;                  // ps_reduce: blocks from a ticket (0 = grid-stride shares)
    int add_chunked = 1;                    // ps_add_offset: one CTA per 64 KiB (0 = grid-stride shares)
    int rows_multi = 1;                     // rows kernel: several short rows per buffer (0 = one row per buffer)
    int tiles_row_lead = 1;                 // look-back tiles, batched: 32-byte tile grid per row (0 = shared lead)
    int seg_kernel = 0;                     // CSR segments: 0 auto, 1 look-back tiles, 2 shared-memory regions
    int float_exact = 0;                    // stream kernel float32 -> float32: 1 = float64 per element (bit-exact
                                            // to float32(cumsum(float64)) whenever the float64 sums are exact)
    Stall stall{};                          // stress tests: in-kernel stall injection (max_ns 0 = off)
};
// Per calling thread: a knob set by one host thread (a harness label, a stress
// test's stall injection) never changes the kernels another thread launches.
thread_local Tuning g_tune;

// rounds kernel: scanner warps, rows per warp, TMA stages, reducer warps, reducer lead (regions)
constexpr int RW = 8, RR = 4, RRED = 4;
// shared-memory split between the scanner ring (L2 re-reads) and the reducer
// ring (HBM reads): float32 rows need deeper reducer buffering (measured with
// scripts/trace_rounds.cu), the rest favours the scanner ring
template <typename TIn> struct RingSplit { static constexpr int RS = 5, RRS = 3; };
template <> struct RingSplit<float> { static constexpr int RS = 3, RRS = 6; };
#define RGEO RoundGeom<TIn, TOut, RW, RR, RingSplit<TIn>::RS, RRED, RingSplit<TIn>::RRS>
#define RKERN scan_rounds_kernel<TIn, TOut, RW, RR, RingSplit<TIn>::RS, RRED, RingSplit<TIn>::RRS>
#define RKERN_STALL scan_rounds_kernel<TIn, TOut, RW, RR, RingSplit<TIn>::RS, RRED, RingSplit<TIn>::RRS, 1, true>

struct DevInfo {
    int sms = 0;
};
DevInfo g_dev[64];

int device_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!g_dev[dev].sms) cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    return g_dev[dev].sms;
}

template <typename TIn, typename TOut>
int rounds_grid() {
    using Geo = RGEO;
    auto kern = RKERN;
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 0;
    if (!per_sm[dev]) {
        if (Geo::SMEM > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, Geo::THREADS, Geo::SMEM);
        per_sm[dev] = b > 0 ? b : -1;
    }
    return per_sm[dev] > 0 ? per_sm[dev] * device_sms() : 0;
}

// Region size (input + output bytes) of the rounds kernel, measured with
// scripts/sweep.cu: float32 rows are compute-heavier and prefer 48 MiB,
// integer paths 64 MiB (a larger share of the L2 per region).
template <typename TIn, typename TOut>
int64_t region_bytes() {
    if (g_tune.round_bytes > 0) return g_tune.round_bytes;
    return (sizeof(TIn) == 4 && (TIn)0.5 != (TIn)0) ? (48ll << 20) : (64ll << 20);
}

// geometry of the rounds kernel for n positions: grid, full-region portion,
// ramp, full-region count and launched regions (see region_geom)
struct RoundPlan {
    int64_t G, portion, full, rounds;
    int ramp;
};

template <typename TIn, typename TOut>
bool rounds_plan(int64_t positions, RoundPlan &p) {
    using Geo = RGEO;
    p.G = rounds_grid<TIn, TOut>();
    if (p.G <= 0) return false;
    p.ramp = (int)g_tune.round_ramp;
    const int64_t unit = Geo::SUB;
    int64_t want = region_bytes<TIn, TOut>() / (int64_t)(sizeof(TIn) + sizeof(TOut)) / p.G;
    p.portion = want / unit * unit;
    if (p.portion < unit) p.portion = unit;
    const int64_t cap = (int64_t)Geo::MAX_CHUNKS * Geo::CHUNK / unit * unit;
    if (p.portion > cap) p.portion = cap;
    const int64_t per_cta = (positions + p.G - 1) / p.G;
    int64_t ramps = 0;
    for (int k = 1; k <= p.ramp; ++k) ramps += 2 * ramp_part(p.portion, Geo::SUB, k);
    p.full = per_cta > ramps ? (per_cta - ramps + p.portion - 1) / p.portion : 0;
    // launch only regions that start before the end of the data
    const int64_t total = 2 * (int64_t)p.ramp + p.full;
    p.rounds = 0;
    for (int64_t r = 0; r < total; ++r) {
        int64_t start, part;
        region_geom(p.portion, p.ramp, p.full, p.G, Geo::SUB, r, start, part);
        if (start >= positions) break;
        p.rounds = r + 1;
    }
    return true;
}

template <typename TIn, typename TOut>
int launch_rounds(const void *in, void *out, int64_t n, int64_t lead, int exclusive, uint64_t seed_bits,
                  const void *seed_terms, int64_t n_seed_terms, void *total, void *scratch, size_t scratch_bytes,
                  uint32_t epoch, cudaStream_t s, const Mailbox *mail = nullptr) {
    using Geo = RGEO;
    RoundPlan pl;
    if (!rounds_plan<TIn, TOut>(lead + n, pl) || pl.G > 1024) return PS_ERR_CUDA_BASE + (int)cudaErrorLaunchFailure;
    const int64_t G = pl.G;
    if (!scratch || scratch_bytes < 256 + (size_t)(pl.rounds * G) * 16) return PS_ERR_SCRATCH;
    RoundArgs a{};
    a.stall = g_tune.stall;
    if (mail) a.mail = *mail;
    a.in = static_cast<const TIn *>(in) - lead;
    a.out = static_cast<TOut *>(out) - lead;
    a.lo = lead;
    a.hi = lead + n;
    a.portion = pl.portion;
    a.rounds = pl.rounds;
    a.full_regions = pl.full;
    a.ramp = pl.ramp;
    a.seed_bits = seed_bits;
    a.seed_terms = seed_terms;
    a.n_seed_terms = n_seed_terms;
    a.total = total;
    a.desc = reinterpret_cast<ulonglong2 *>(static_cast<char *>(scratch) + 256);
    a.epoch = epoch;
    a.exclusive = exclusive;
    a.lead_regions = (int)g_tune.round_lead;
    a.l2_prefetch = (int)g_tune.round_prefetch;
    void *params[] = {&a};
    const void *kern = (const void *)RKERN;
    if (a.stall.max_ns) {  // stress-test instantiation with the stall sites compiled in
        kern = (const void *)RKERN_STALL;
        if (Geo::SMEM > 48 * 1024) cudaFuncSetAttribute(RKERN_STALL, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
    }
    cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3((unsigned)G), dim3(Geo::THREADS), params, Geo::SMEM, s);
    return cuda_rc(e);
}

// ---- shared-memory-resident streaming kernel (stream_kernel.cuh) ---------------------------------
// measured with scripts/stream_variants.cu: six 32 KiB buffers per SM (regions of
// 4.6 MiB) hide the grid-wide ledger exchange; three 64 KiB buffers do not
#ifndef PS_SNBUF
#define PS_SNBUF 7
#endif
#ifndef PS_SRWP
#define PS_SRWP 4
#endif
#ifndef PS_SSW
#define PS_SSW 8
#endif
#ifndef PS_SROWS
#define PS_SROWS 4
#endif
constexpr int SSW = PS_SSW, SROWS = PS_SROWS, SNBUF = PS_SNBUF, SRWP = PS_SRWP;
#define SGEO StreamGeom<TIn, SSW, SROWS, SNBUF, SRWP>
#define SKERN scan_stream_kernel<TIn, TOut, SSW, SROWS, SNBUF, SRWP>
#define SKERN_STALL scan_stream_kernel<TIn, TOut, SSW, SROWS, SNBUF, SRWP, true>
// float32 -> float32 with FP32-pipe arithmetic (stream_kernel.cuh f32pair_*); the
// float64-per-element form stays selectable (tuning "float_exact" = 1)
#define SKERN_F32 scan_stream_kernel<TIn, TOut, SSW, SROWS, SNBUF, SRWP, false, 1, true>
#define SKERN_F32_STALL scan_stream_kernel<TIn, TOut, SSW, SROWS, SNBUF, SRWP, true, 1, true>

constexpr int STREAM_MAX_GRID = 32 * GATHER_LP;  // the ledger warp gathers <= 5 descriptors per lane

template <typename TIn, typename TOut>
int64_t stream_portion() {  // positions per CTA per region: NBUF buffers in ~200 KB
    constexpr int64_t unit = (int64_t)SSW * SGEO::CHUNK;
    int64_t p = (int64_t)SGEO::BUF_BYTES_MAX / SNBUF / (int64_t)sizeof(TIn) / unit * unit;
    if (p > (int64_t)SGEO::MAXC * SGEO::CHUNK) p = (int64_t)SGEO::MAXC * SGEO::CHUNK / unit * unit;
    return p < unit ? unit : p;
}

template <typename TIn, typename TOut>
int stream_grid() {
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 0;
    if (!per_sm[dev]) {
        const int smem = SGEO::smem(stream_portion<TIn, TOut>());
        cudaFuncSetAttribute(SKERN, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, SKERN, SGEO::THREADS, smem);
        per_sm[dev] = b > 0 ? b : -1;
    }
    return per_sm[dev] > 0 ? per_sm[dev] * device_sms() : 0;
}

template <typename TIn, typename TOut>
int launch_stream(const void *in, void *out, int64_t n, int64_t lead, int exclusive, uint64_t seed_bits,
                  const void *seed_terms, int64_t n_seed_terms, void *total, void *scratch, size_t scratch_bytes,
                  uint32_t epoch, cudaStream_t s, const Mailbox *mail = nullptr, bool copy_in = false) {
    const int64_t G = stream_grid<TIn, TOut>();
    if (G <= 0 || G > STREAM_MAX_GRID) return PS_ERR_CUDA_BASE + (int)cudaErrorLaunchFailure;
    const int64_t P = stream_portion<TIn, TOut>();
    const int64_t rounds = (lead + n + P * G - 1) / (P * G);
    if (!scratch || scratch_bytes < 256 + (size_t)(rounds * G) * 16) return PS_ERR_SCRATCH;
    StreamArgs a{};
    a.stall = g_tune.stall;
    if (mail) a.mail = *mail;
    a.in = static_cast<const TIn *>(in) - lead;
    a.out = static_cast<TOut *>(out) - lead;
    a.lo = lead;
    a.hi = lead + n;
    a.portion = P;
    a.rounds = rounds;
    a.seed_bits = seed_bits;
    a.seed_terms = seed_terms;
    a.n_seed_terms = n_seed_terms;
    a.total = total;
    a.desc = reinterpret_cast<ulonglong2 *>(static_cast<char *>(scratch) + 256);
    a.epoch = epoch;
    a.exclusive = exclusive;
    a.inflight = g_tune.stream_inflight;
    a.copy_in = copy_in ? 1 : 0;
    void *params[] = {&a};
    const void *kern = (const void *)SKERN;
    if (a.stall.max_ns) {  // stress-test instantiation with the stall sites compiled in
        kern = (const void *)SKERN_STALL;
        cudaFuncSetAttribute(SKERN_STALL, cudaFuncAttributeMaxDynamicSharedMemorySize, SGEO::smem(P));
    }
    if constexpr (std::is_same<TIn, float>::value && std::is_same<TOut, float>::value) {
        if (!g_tune.float_exact) {
            kern = a.stall.max_ns ? (const void *)SKERN_F32_STALL : (const void *)SKERN_F32;
            static bool attr[64] = {false};
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev >= 0 && dev < 64 && !attr[dev]) {
                cudaFuncSetAttribute(SKERN_F32, cudaFuncAttributeMaxDynamicSharedMemorySize, SGEO::smem(P));
                cudaFuncSetAttribute(SKERN_F32_STALL, cudaFuncAttributeMaxDynamicSharedMemorySize, SGEO::smem(P));
                attr[dev] = true;
            }
        }
    }
    cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3((unsigned)G), dim3(SGEO::THREADS), params, SGEO::smem(P), s);
    return cuda_rc(e);
}

// ---- CSR segments on shared-memory regions (seg_stream.cuh) ---------------------------------------
#ifndef PS_SEG_SW  // geometry overrides for scripts/build_variants.sh experiments
#define PS_SEG_SW 8
#endif
#ifndef PS_SEG_ROWS
#define PS_SEG_ROWS 4
#endif
#ifndef PS_SEG_NBUF
#define PS_SEG_NBUF 6
#endif
#ifndef PS_SEG_RWP
#define PS_SEG_RWP 4
#endif
constexpr int GSW = PS_SEG_SW, GROWS = PS_SEG_ROWS, GNBUF = PS_SEG_NBUF, GRWP = PS_SEG_RWP;
// 8-byte integer inputs: a 32-lane row is half the bytes of a 4-byte one for the same reducer
// work, and the reducers set the region rate -- eight reducer warps instead of four
// (2^27 int64, 16K / 1M segments: 424 / 540 -> 395 / 509 us; 4-byte and float inputs: +-0)
template <typename TIn> struct SegCfg { static constexpr int RWP = GRWP; };
template <> struct SegCfg<int64_t> { static constexpr int RWP = GRWP == 4 ? 8 : GRWP; };
template <> struct SegCfg<uint64_t> { static constexpr int RWP = GRWP == 4 ? 8 : GRWP; };
#define GGEO SegStreamGeom<TIn, GSW, GROWS, GNBUF, SegCfg<TIn>::RWP>
#define GKERN seg_stream_kernel<TIn, TOut, GSW, GROWS, GNBUF, SegCfg<TIn>::RWP>
constexpr int64_t SEG_STREAM_MAX_GRID = STREAM_MAX_GRID;

template <typename TIn, typename TOut>
int seg_stream_grid() {
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 0;
    if (!per_sm[dev]) {
        cudaFuncSetAttribute(GKERN, cudaFuncAttributeMaxDynamicSharedMemorySize, GGEO::SMEM);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, GKERN, GGEO::THREADS, GGEO::SMEM);
        per_sm[dev] = b > 0 ? b : -1;
    }
    return per_sm[dev] > 0 ? per_sm[dev] * device_sms() : 0;
}

// scratch of the region kernel: control words, one descriptor per (region, CTA),
// the portions' lower bounds and repeat flags, then the head bitmap (1 bit per
// position) -- the last two cleared before and after every call, so the scratch
// is left as the other entry points expect it (no stray words that could pass
// for a descriptor)
struct SegStreamLayout {
    int64_t Q;  // portions (rounds * G)
    size_t off_lb, off_dup, off_bm, bm_bytes, total;
};
SegStreamLayout seg_stream_layout(int64_t q_portions, int64_t P) {
    SegStreamLayout L{};
    L.Q = q_portions;
    L.off_lb = 256 + align_up((size_t)q_portions * 32, 256);  // integers: two descriptors per portion
    L.off_dup = L.off_lb + align_up((size_t)(q_portions + 1) * 8, 256);
    L.off_bm = L.off_dup + align_up((size_t)(q_portions + 1) * 4, 256);
    L.bm_bytes = align_up((size_t)((q_portions * P + 128 + 7) / 8), 256);
    L.total = L.off_bm + L.bm_bytes;
    return L;
}
size_t seg_stream_scratch_bytes(int64_t n, int elem_bytes) {
    const int64_t P = 32768 / elem_bytes;
    const int64_t q = (n + 32 + P - 1) / P + 2 * SEG_STREAM_MAX_GRID + 1;  // rounds * G <= ceil((lead + n) / P) + G
    return seg_stream_layout(q, P).total;
}

// returns -1 when the buffers do not suit the region kernel (caller falls back)
template <typename TIn, typename TOut>
int launch_seg_stream(const void *in, void *out, int64_t n, const int64_t *offsets, int64_t nseg, int exclusive,
                      void *totals, void *scratch, size_t scratch_bytes, uint32_t epoch, cudaStream_t s,
                      int64_t ucols = 0) {  // offsets == nullptr: nseg uniform segments of ucols elements
    const uintptr_t ain = (uintptr_t)in % 32;
    const int64_t lead = (ain % sizeof(TIn)) ? -1 : (int64_t)(ain / sizeof(TIn));
    const bool vec = lead >= 0 && ((uintptr_t)out % 32) == (uintptr_t)((lead * sizeof(TOut)) % 32) &&
                     (uintptr_t)out % sizeof(TOut) == 0 && lead * (int64_t)sizeof(TOut) < 32;
    if (!vec) return -1;
    const int64_t G = seg_stream_grid<TIn, TOut>();
    if (G <= 0 || G > SEG_STREAM_MAX_GRID) return -1;
    const int64_t P = GGEO::P;
    const int64_t rounds = (lead + n + P * G - 1) / (P * G);
    const SegStreamLayout L = seg_stream_layout(rounds * G, P);
    if (!scratch || scratch_bytes < L.total) return PS_ERR_SCRATCH;
    char *sc = static_cast<char *>(scratch);
    SegStreamArgs a{};
    a.in = static_cast<const TIn *>(in) - lead;
    a.out = static_cast<TOut *>(out) - lead;
    a.lo = lead;
    a.hi = lead + n;
    a.lead = lead;
    a.portion = P;
    a.rounds = rounds;
    a.offsets = offsets;
    a.nseg = nseg;
    int64_t *lb = reinterpret_cast<int64_t *>(sc + L.off_lb);
    uint32_t *dup = reinterpret_cast<uint32_t *>(sc + L.off_dup);
    uint32_t *bm = reinterpret_cast<uint32_t *>(sc + L.off_bm);
    a.lb = lb;
    a.dupflag = dup;
    a.bitmap = bm;
    using A = typename AccOf<TIn>::type;
    constexpr bool GATHER = sizeof(TOut) == 8;  // accumulator-typed output: totals read back from it
    a.totals = GATHER ? nullptr : totals;
    if (!GATHER && totals) {  // emitted by the scanners: empty segments keep the zero
        cudaError_t ze = cudaMemsetAsync(totals, 0, (size_t)nseg * 8, s);
        if (ze != cudaSuccess) return cuda_rc(ze);
    }
    if (GATHER && totals && exclusive)
        seg_last_in_kernel<TIn, A><<<(unsigned)((nseg + 255) / 256), 256, 0, s>>>(
            static_cast<const TIn *>(in), offsets, ucols, nseg, static_cast<A *>(totals));
    a.desc = reinterpret_cast<ulonglong2 *>(sc + 256);
    a.epoch = epoch;
    a.exclusive = exclusive;
    a.inflight = g_tune.stream_inflight;
    a.one = 1;
    const size_t clear = L.total - L.off_dup;  // repeat flags + bitmap
    cudaError_t e = cudaMemsetAsync(dup, 0, clear, s);
    if (e != cudaSuccess) return cuda_rc(e);
    const int64_t threads = nseg + 1;  // one per offset
    seg_prepare_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(offsets, ucols, nseg, n, lead, P, L.Q, lb, dup,
                                                                          bm);
    void *params[] = {&a};
#ifdef PS_SEG_TRACE
    static uint64_t *trace = nullptr;
    const size_t tbytes = (size_t)rounds * G * 8 * 8;
    static size_t tcap = 0;
    if (tcap < tbytes) {
        if (trace) cudaFree(trace);
        cudaMalloc(&trace, tbytes);
        tcap = tbytes;
        cudaMemcpyToSymbol(g_seg_trace, &trace, sizeof(trace));
    }
    cudaMemsetAsync(trace, 0, tbytes, s);
#endif
    e = cudaLaunchCooperativeKernel((const void *)GKERN, dim3((unsigned)G), dim3(GGEO::THREADS), params, GGEO::SMEM, s);
    if (e != cudaSuccess) return cuda_rc(e);
#ifdef PS_SEG_TRACE
    {
        std::vector<uint64_t> h(tbytes / 8);
        cudaMemcpyAsync(h.data(), trace, tbytes, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        FILE *f = std::fopen("gpurun_out/seg_trace.bin", "wb");
        if (f) {
            const int64_t hdr[2] = {rounds, G};
            std::fwrite(hdr, 8, 2, f);
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
#endif
    if (GATHER && PS_SEG_INCLEAR) {  // these instantiations cleared the repeat flags and the bitmap as they consumed them
        if (totals)
            seg_totals_gather_kernel<TOut, A><<<(unsigned)((nseg + 255) / 256), 256, 0, s>>>(
                static_cast<const TOut *>(out), offsets, ucols, nseg, static_cast<A *>(totals), exclusive);
        return launch_rc();
    }
    if (GATHER && totals)
        seg_totals_gather_kernel<TOut, A><<<(unsigned)((nseg + 255) / 256), 256, 0, s>>>(
            static_cast<const TOut *>(out), offsets, ucols, nseg, static_cast<A *>(totals), exclusive);
    return cuda_rc(cudaMemsetAsync(dup, 0, clear, s));
}

// ---- batched rows, one CTA per row (rows_kernel.cuh) ----------------------------------------------
// measured with scripts/rows_variants.cu: float32 rows are compute-heavier and run
// best as two independent 64 KiB CTAs per SM; integer rows as one 192 KiB CTA
template <typename TIn> struct RowsCfg { static constexpr int SW = 8, RPC = 4, NBUF = 3, NCH = 16; };
template <> struct RowsCfg<float> { static constexpr int SW = 8, RPC = 2, NBUF = 2, NCH = 16; };
#define WGEO RowsGeom<TIn, RowsCfg<TIn>::SW, RowsCfg<TIn>::RPC, RowsCfg<TIn>::NBUF, RowsCfg<TIn>::NCH>
#define WKERN scan_rows_kernel<TIn, TOut, RowsCfg<TIn>::SW, RowsCfg<TIn>::RPC, RowsCfg<TIn>::NBUF, RowsCfg<TIn>::NCH>
#define WKERN_STALL \
    scan_rows_kernel<TIn, TOut, RowsCfg<TIn>::SW, RowsCfg<TIn>::RPC, RowsCfg<TIn>::NBUF, RowsCfg<TIn>::NCH, true>
#define WMKERN scan_rows_multi_kernel<TIn, TOut, RowsCfg<TIn>::SW, RowsCfg<TIn>::RPC, RowsCfg<TIn>::NBUF, RowsCfg<TIn>::NCH>
#define WMKERN_STALL \
    scan_rows_multi_kernel<TIn, TOut, RowsCfg<TIn>::SW, RowsCfg<TIn>::RPC, RowsCfg<TIn>::NBUF, RowsCfg<TIn>::NCH, true>

template <typename TIn, typename TOut>
int rows_grid() {
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 0;
    if (!per_sm[dev]) {
        cudaFuncSetAttribute(WKERN, cudaFuncAttributeMaxDynamicSharedMemorySize, WGEO::SMEM);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, WKERN, WGEO::THREADS, WGEO::SMEM);
        per_sm[dev] = b > 0 ? b : -1;
    }
    return per_sm[dev] > 0 ? per_sm[dev] * device_sms() : 0;
}

// TMA row streaming needs 16-byte aligned row starts and row lengths
template <typename TIn, typename TOut>
bool rows_kernel_applies(const void *in, int64_t rows, int64_t cols, int64_t ld_in) {
    if (g_tune.rows_kernel == 1) return false;
    if ((uintptr_t)in % 16 || (cols * (int64_t)sizeof(TIn)) % 16 || (ld_in * (int64_t)sizeof(TIn)) % 16) return false;
    const int G = rows_grid<TIn, TOut>();
    if (G <= 0) return false;
    return g_tune.rows_kernel == 2 || rows >= 2 * (int64_t)G;
}

template <typename TIn, typename TOut>
int launch_rows(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out, int exclusive,
                const void *row_seeds, void *row_totals, void *scratch, size_t scratch_bytes, cudaStream_t s) {
    RowsArgs a{};
    // rows from a grid-wide ticket in the scratch's control words (zero between launches)
    if (g_tune.rows_dynamic && scratch && scratch_bytes >= 256) a.ctr = static_cast<unsigned long long *>(scratch);
    a.stall = g_tune.stall;
    a.in = in;
    a.out = out;
    a.rows = rows;
    a.cols = cols;
    a.ld_in = ld_in;
    a.ld_out = ld_out;
    a.row_seeds = row_seeds;
    a.row_totals = row_totals;
    a.exclusive = exclusive;
    a.vec_out = (uintptr_t)out % 32 == 0 && (ld_out * (int64_t)sizeof(TOut)) % 32 == 0;
    int64_t G = rows_grid<TIn, TOut>();
    if (G > rows) G = rows;
    // rows of at most half a buffer: several rows per buffer (scan_rows_multi_kernel)
    const bool multi = cols <= WGEO::SEG / 2 && g_tune.rows_multi;
    if (multi) {
        static bool attr[64] = {false};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 0 && dev < 64 && !attr[dev]) {
            cudaFuncSetAttribute(WMKERN, cudaFuncAttributeMaxDynamicSharedMemorySize, WGEO::SMEM);
            attr[dev] = true;
        }
    }
    if (a.stall.max_ns) {  // stress-test instantiation with the stall sites compiled in
        if (multi) {
            cudaFuncSetAttribute(WMKERN_STALL, cudaFuncAttributeMaxDynamicSharedMemorySize, WGEO::SMEM);
            WMKERN_STALL<<<(unsigned)G, WGEO::THREADS, WGEO::SMEM, s>>>(a);
        } else {
            cudaFuncSetAttribute(WKERN_STALL, cudaFuncAttributeMaxDynamicSharedMemorySize, WGEO::SMEM);
            WKERN_STALL<<<(unsigned)G, WGEO::THREADS, WGEO::SMEM, s>>>(a);
        }
    } else if (multi) {
        WMKERN<<<(unsigned)G, WGEO::THREADS, WGEO::SMEM, s>>>(a);
    } else {
        WKERN<<<(unsigned)G, WGEO::THREADS, WGEO::SMEM, s>>>(a);
    }
    return launch_rc();
}

// ---- scan (1-D and batched share one kernel) ----------------------------------------------
template <typename TIn, typename TOut>
int launch_scan(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
                int exclusive, uint64_t seed_bits, const void *seed_terms, int64_t n_seed_terms,
                void *totals, void *scratch, size_t scratch_bytes, uint32_t epoch, cudaStream_t s,
                const Mailbox *mail = nullptr) {
    constexpr int64_t TILE = tile_elems<TIn>();
    ScanArgs a{};
    a.stall = g_tune.stall;
    if (mail && rows == 1) a.mail = *mail;
    a.in = in;
    a.out = out;
    a.rows = rows;
    a.cols = cols;
    a.ld_in = ld_in;
    a.ld_out = ld_out;
    a.seed_bits = seed_bits;
    a.seed_terms = seed_terms;
    a.n_seed_terms = n_seed_terms;
    a.totals = totals;
    a.epoch = epoch;
    a.exclusive = exclusive;
    // alignment: tiles start on 32-byte boundaries of the input; the output
    // must sit at the same element phase for the 256-bit store path
    const uintptr_t ain = (uintptr_t)in % 32;
    int64_t lead = (ain % sizeof(TIn)) ? -1 : (int64_t)(ain / sizeof(TIn));
    bool vec = lead >= 0 && ((uintptr_t)out % 32) == (uintptr_t)((lead * sizeof(TOut)) % 32) &&
               (uintptr_t)out % sizeof(TOut) == 0;
    if (rows > 1) vec = vec && (ld_in * sizeof(TIn)) % 32 == 0 && (ld_out * sizeof(TOut)) % 32 == 0;
    if (vec && lead * (int64_t)sizeof(TOut) >= 32) vec = false;
    a.vec_ok = vec;
    a.lead = vec ? lead : 0;
    // batched rows on element-aligned buffers: lead and vector accesses decided per row
    // in the kernel (tiles_per_row then has room for the largest lead)
    int64_t max_lead = 0;
    if (rows > 1 && g_tune.tiles_row_lead && (uintptr_t)in % sizeof(TIn) == 0 && (uintptr_t)out % sizeof(TOut) == 0) {
        a.row_lead = 1;
        a.lead = 0;
        max_lead = 32 / (int64_t)sizeof(TIn) - 1;
    }
    const bool big = cols * (int64_t)sizeof(TIn) >= g_tune.rounds_min_bytes;
    if (rows == 1 && vec &&
        (g_tune.scan_kernel == 3 || (g_tune.scan_kernel == 0 && big && stream_grid<TIn, TOut>() <= STREAM_MAX_GRID)))
        return launch_stream<TIn, TOut>(in, out, cols, a.lead, exclusive, seed_bits, seed_terms, n_seed_terms, totals,
                                        scratch, scratch_bytes, epoch, s, mail);
    // in/out pairs at different 32-byte phases: the output decides the tile grid (256-bit
    // stores); the input is bulk-copied if some lead of that grid leaves it 16-byte aligned,
    // otherwise the producer warp copies it (stream_kernel.cuh, copy_in)
    if (rows == 1 && !vec && g_tune.stream_copy_in && (uintptr_t)in % sizeof(TIn) == 0 && (uintptr_t)out % sizeof(TOut) == 0 &&
        (g_tune.scan_kernel == 3 || (g_tune.scan_kernel == 0 && big && stream_grid<TIn, TOut>() <= STREAM_MAX_GRID))) {
        const int64_t ev_out = 32 / (int64_t)sizeof(TOut), vec_in = 32 / (int64_t)sizeof(TIn);
        const int64_t k = (int64_t)(((uintptr_t)out % 32) / sizeof(TOut));  // lead = k (mod ev_out)
        int64_t pick = k;
        bool tma = false;
        for (int64_t l = k; l < vec_in; l += ev_out)
            if (((uintptr_t)in - (uintptr_t)(l * (int64_t)sizeof(TIn))) % 16 == 0) {
                pick = l;
                tma = true;
                break;
            }
        return launch_stream<TIn, TOut>(in, out, cols, pick, exclusive, seed_bits, seed_terms, n_seed_terms, totals,
                                        scratch, scratch_bytes, epoch, s, mail, !tma);
    }
    if (rows == 1 && vec && g_tune.scan_kernel == 2)
        return launch_rounds<TIn, TOut>(in, out, cols, a.lead, exclusive, seed_bits, seed_terms, n_seed_terms, totals,
                                        scratch, scratch_bytes, epoch, s, mail);
    // many short contiguous rows without seeds: one flat segmented scan with uniform
    // segments (a look-back tile per row would leave most of each tile idle)
    if (rows > 1 && g_tune.tiles_row_lead && !seed_terms && seed_bits == 0 && !mail && ld_in == cols && ld_out == cols &&
        scratch) {
        // large batches, rows of any length that the rows kernel cannot stream (or short ones):
        // the shared-memory-region kernel with computed offsets -- one HBM read and write per
        // element (2^20 rows x 250 int32 -> int64: 0.31 -> 0.70 of the peak; 16384 x 16383: 0.80 -> 0.9+)
        if (g_tune.seg_kernel != 1 && rows * cols * (int64_t)sizeof(TIn) >= g_tune.rounds_min_bytes &&
            scratch_bytes >= seg_stream_scratch_bytes(rows * cols, (int)sizeof(TIn))) {
            const int rc = launch_seg_stream<TIn, TOut>(in, out, rows * cols, nullptr, rows, exclusive, totals, scratch,
                                                        scratch_bytes, epoch, s, cols);
            if (rc >= 0) return rc;
        }
        if (cols * 4 <= TILE && scratch_bytes >= seg_scratch_bytes(rows * cols, (int)sizeof(TIn)))
            return launch_segmented<TIn, TOut>(in, out, rows * cols, nullptr, rows, exclusive, totals, scratch, epoch, s,
                                               cols);
    }
    a.tiles_per_row = (a.lead + max_lead + cols + TILE - 1) / TILE;
    const int64_t tiles = rows * a.tiles_per_row;
    if (tiles > 0x7fffffffLL) return PS_ERR_ARG;
    if (a.tiles_per_row > 1) {
        if (!scratch || scratch_bytes < desc_bytes(tiles)) return PS_ERR_SCRATCH;
        a.desc = carve_desc(scratch, tiles);
    }
    scan_tiles_kernel<TIn, TOut, SCAN_WARPS, SCAN_ROWS><<<(unsigned)tiles, SCAN_WARPS * 32, 0, s>>>(a);
    return launch_rc();
}

// Mailbox layout on every GPU: 2 x n_peers 16-byte slots, slot (e & 1) * n_peers + h
// holds rank h's total of exchange epoch e.  Before publishing epoch e a rank
// waits until every rank has published e-1 (prev_epoch): each rank publishes
// e-1 only after its scan of e-2 has consumed its slots, so a slot of parity
// e & 1 is never overwritten while a slower rank may still read it.
__global__ void publish_total_kernel(const uint64_t *total, ulonglong2 *const *peer_mailboxes, int n_peers, int rank,
                                     uint32_t epoch, uint32_t prev_epoch, const ulonglong2 *own_mailbox,
                                     int *timeout) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32 && prev_epoch) {
        Mailbox prev{own_mailbox + (size_t)(prev_epoch & 1) * n_peers, n_peers, prev_epoch, timeout};
        (void)mailbox_sum<unsigned long long>(prev, lane);
    }
    __syncthreads();
    const int h = threadIdx.x;
    if (h < n_peers)
        mailbox_post(peer_mailboxes[h] + (size_t)(epoch & 1) * n_peers + rank, epoch, *total);
}

template <typename A> __global__ void mailbox_seed_kernel(A *total, uint64_t seed_bits, Mailbox m) {
    const A v = mailbox_sum<A>(m, threadIdx.x & 31);
    if (threadIdx.x == 0 && total) *total = acc_from_bits<A>(seed_bits) + v;
}

template <typename A> __global__ void fill_seed_kernel(A *dst, int64_t count, uint64_t seed_bits, const void *terms,
                                                       int64_t n_terms, int per_row) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    A v = acc_from_bits<A>(seed_bits);
    if (terms) {
        const A *t = reinterpret_cast<const A *>(terms);
        if (per_row) v += t[i];
        else for (int64_t k = 0; k < n_terms; ++k) v += t[k];
    }
    dst[i] = v;
}

#define PS_DISPATCH_PAIR(din, dout, CALL)                                                      \
    do {                                                                                        \
        if (din == PS_DTYPE_INT32 && dout == PS_DTYPE_INT32) { CALL(int32_t, int32_t); }        \
        else if (din == PS_DTYPE_INT32 && dout == PS_DTYPE_INT64) { CALL(int32_t, int64_t); }   \
        else if (din == PS_DTYPE_INT64 && dout == PS_DTYPE_INT64) { CALL(int64_t, int64_t); }   \
        else if (din == PS_DTYPE_UINT32 && dout == PS_DTYPE_UINT32) { CALL(uint32_t, uint32_t); } \
        else if (din == PS_DTYPE_UINT32 && dout == PS_DTYPE_UINT64) { CALL(uint32_t, uint64_t); } \
        else if (din == PS_DTYPE_UINT64 && dout == PS_DTYPE_UINT64) { CALL(uint64_t, uint64_t); } \
        else if (din == PS_DTYPE_FLOAT32 && dout == PS_DTYPE_FLOAT32) { CALL(float, float); }   \
        else if (din == PS_DTYPE_FLOAT32 && dout == PS_DTYPE_FLOAT64) { CALL(float, double); }  \
        else if (din == PS_DTYPE_FLOAT64 && dout == PS_DTYPE_FLOAT64) { CALL(double, double); } \
        else return PS_ERR_DTYPE;                                                               \
    } while (0)

#define PS_DISPATCH_ONE(dt, CALL)                                        \
    do {                                                                  \
        switch (dt) {                                                     \
            case PS_DTYPE_INT32: CALL(int32_t); break;                    \
            case PS_DTYPE_INT64: CALL(int64_t); break;                    \
            case PS_DTYPE_UINT32: CALL(uint32_t); break;                  \
            case PS_DTYPE_UINT64: CALL(uint64_t); break;                  \
            case PS_DTYPE_FLOAT32: CALL(float); break;                    \
            case PS_DTYPE_FLOAT64: CALL(double); break;                   \
            default: return PS_ERR_DTYPE;                                 \
        }                                                                 \
    } while (0)

// Empty input: totals (if requested) still receive the seed (core.py:152-156:
// a zero-length span returns the offset).
int write_seed_only(int din, void *totals, int64_t count, uint64_t seed_bits, const void *terms, int64_t n_terms,
                    int per_row, cudaStream_t s) {
    if (!totals || count == 0) return PS_OK;
    const unsigned blocks = (unsigned)((count + 255) / 256);
#define FILL(T)                                                                                     \
    fill_seed_kernel<typename AccOf<T>::type><<<blocks, 256, 0, s>>>(                               \
        reinterpret_cast<typename AccOf<T>::type *>(totals), count, seed_bits, terms, n_terms, per_row)
    PS_DISPATCH_ONE(din, FILL);
#undef FILL
    return launch_rc();
}

// ---- host-buffer pipeline (host_pipeline.h): device workspace layout ----------------------------
constexpr int NSLOT = host::NSLOT;

struct HostLayout {
    size_t in_slot, out_slot, scratch, total;  // byte sizes
    size_t off_in, off_out, off_scratch, off_carry;
};

HostLayout host_layout(int64_t chunk, int din, int dout) {
    HostLayout L{};
    L.in_slot = align_up((size_t)chunk * dsize(din), 256);
    L.out_slot = align_up((size_t)chunk * dsize(dout), 256);
    L.scratch = align_up(ps_scan_scratch_bytes(chunk, din, dout), 256);  // whichever kernel a chunk takes
    L.off_in = 0;
    L.off_out = L.off_in + NSLOT * L.in_slot;
    L.off_scratch = L.off_out + NSLOT * L.out_slot;
    L.off_carry = L.off_scratch + L.scratch;
    L.total = L.off_carry + 256;
    return L;
}

}  // namespace
}  // namespace ps

using namespace ps;

namespace ps {
namespace {
constexpr int64_t SELECT_STREAM_MIN = 1 << 22;  // elements; below this the 3-launch path wins (fill/drain)
thread_local int g_select_kernel = 0;            // 0 auto, 1 three launches, 2 single pass (per thread)

template <typename TV, typename TF>
int launch_select_stream(const void *values, const void *flags, int64_t n, void *out, void *count, void *scratch,
                         size_t scratch_bytes, uint32_t epoch, cudaStream_t s) {
    using Geo = SelectStreamGeom<TV, TF>;
    auto kern = select_stream_kernel<TV, TF>;
    static int per_sm[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return PS_ERR_CUDA_BASE + (int)cudaErrorInvalidDevice;
    if (!per_sm[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, SS_THREADS, Geo::SMEM);
        per_sm[dev] = b > 0 ? b : -1;
    }
    if (per_sm[dev] <= 0) return PS_ERR_CUDA_BASE + (int)cudaErrorLaunchFailure;
    int64_t G = (int64_t)per_sm[dev] * device_sms();
    if (G > 256) G = 256;
    SelectArgs a{};
    a.values = values;
    a.flags = flags;
    a.out = out;
    a.n = n;
    a.portion = SS_P;
    a.rounds = (n + SS_P * G - 1) / (SS_P * G);
    a.count = static_cast<long long *>(count);
    if (!scratch || scratch_bytes < 256 + (size_t)(a.rounds * G) * 16) return PS_ERR_SCRATCH;
    a.desc = reinterpret_cast<ulonglong2 *>(static_cast<char *>(scratch) + 256);
    // the high word makes a stale count (a small integer) in this scratch unmistakable for a tag
    a.want = ((uint64_t)(~epoch) << 32) | ((uint64_t)epoch << 2);
    a.inflight = g_tune.stream_inflight;
    void *params[] = {&a};
    return cuda_rc(cudaLaunchCooperativeKernel((const void *)kern, dim3((unsigned)G), dim3(SS_THREADS), params,
                                               Geo::SMEM, s));
}
}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int ps_version(void) { return 100; }

int ps_pair_supported(int dtype_in, int dtype_out) { return pair_ok(dtype_in, dtype_out) ? 1 : 0; }

const char *ps_error_string(int code) {
    switch (code) {
        case PS_OK: return "ok";
        case PS_ERR_DTYPE: return "unsupported dtype pair";
        case PS_ERR_ARG: return "invalid argument (size, pointer or leading dimension)";
        case PS_ERR_SCRATCH: return "scratch buffer missing or too small";
        case PS_ERR_EPOCH: return "epoch outside [1, PS_EPOCH_MAX]";
        case PS_ERR_OVERLAP: return "input and output partially overlap";
        default:
            if (code >= PS_ERR_CUDA_BASE) return cudaGetErrorString((cudaError_t)(code - PS_ERR_CUDA_BASE));
            return "unknown error";
    }
}

size_t ps_scan_scratch_bytes(int64_t n, int dtype_in, int dtype_out) {
    if (!pair_ok(dtype_in, dtype_out) || n < 0) return 0;
    const int64_t tile = tile_of_dtype(dtype_in);
    size_t bytes = desc_bytes((n + tile - 1) / tile + 1);  // +1: a misaligned start can add a tile
    // the cache-partitioned kernel needs one descriptor per (region, CTA): at most
    // 1024 persistent CTAs, regions of g_tune.round_bytes of input + output
    const int64_t traffic = n * (int64_t)(dsize(dtype_in) + dsize(dtype_out));
    const int64_t rbytes = g_tune.round_bytes > 0 ? g_tune.round_bytes : (48ll << 20);
    int64_t regions = traffic / rbytes + 2 + 2 * g_tune.round_ramp;
    size_t rb = 256 + (size_t)regions * 1024 * 16;
    // stream kernel: <= 256 CTAs, portions of >= 16 KiB of input per CTA and region
    const size_t sb = 256 + (size_t)(n * (int64_t)dsize(dtype_in) / (16ll << 10) + 2 * 256) * 16;
    if (sb > rb) rb = sb;
    return bytes > rb ? bytes : rb;
}

int ps_set_tuning(const char *key, int64_t value) {
    if (!key) return PS_ERR_ARG;
    if (!std::strcmp(key, "scan_kernel")) {
        if (value < 0 || value > 3) return PS_ERR_ARG;
        g_tune.scan_kernel = (int)value;
    } else if (!std::strcmp(key, "round_bytes")) {
        if (value != 0 && value < (1ll << 20)) return PS_ERR_ARG;
        g_tune.round_bytes = value;
    } else if (!std::strcmp(key, "round_lead")) {
        if (value < 1 || value > 8) return PS_ERR_ARG;
        g_tune.round_lead = value;
    } else if (!std::strcmp(key, "rows_kernel")) {
        if (value < 0 || value > 2) return PS_ERR_ARG;
        g_tune.rows_kernel = (int)value;
    } else if (!std::strcmp(key, "stream_copy_in")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.stream_copy_in = (int)value;
    } else if (!std::strcmp(key, "stream_inflight")) {
        if (value < 0 || value > 8) return PS_ERR_ARG;
        g_tune.stream_inflight = (int)value;
    } else if (!std::strcmp(key, "tiles_row_lead")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.tiles_row_lead = (int)value;
    } else if (!std::strcmp(key, "seg_kernel")) {
        if (value < 0 || value > 2) return PS_ERR_ARG;
        g_tune.seg_kernel = (int)value;
    } else if (!std::strcmp(key, "float_exact")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.float_exact = (int)value;
    } else if (!std::strcmp(key, "add_chunked")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.add_chunked = (int)value;
    } else if (!std::strcmp(key, "reduce_blocks")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.reduce_blocks = (int)value;
    } else if (!std::strcmp(key, "rows_multi")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.rows_multi = (int)value;
    } else if (!std::strcmp(key, "rows_dynamic")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.rows_dynamic = (int)value;
    } else if (!std::strcmp(key, "select_kernel")) {
        if (value < 0 || value > 2) return PS_ERR_ARG;
        g_select_kernel = (int)value;
    } else if (!std::strcmp(key, "stall_seed")) {
        if (value < 0 || value > 0xffffffffLL) return PS_ERR_ARG;
        g_tune.stall.seed = (uint32_t)value;
    } else if (!std::strcmp(key, "stall_prob")) {
        if (value < 0 || value > 1024) return PS_ERR_ARG;
        g_tune.stall.prob = (uint32_t)value;
    } else if (!std::strcmp(key, "stall_ns")) {
        if (value < 0 || value > 10000000) return PS_ERR_ARG;
        g_tune.stall.max_ns = (uint32_t)value;
    } else if (!std::strcmp(key, "round_prefetch")) {
        if (value < 0 || value > 1) return PS_ERR_ARG;
        g_tune.round_prefetch = value;
    } else if (!std::strcmp(key, "round_ramp")) {
        if (value < 0 || value > 4) return PS_ERR_ARG;
        g_tune.round_ramp = value;
    } else if (!std::strcmp(key, "rounds_min_bytes")) {
        if (value < 0) return PS_ERR_ARG;
        g_tune.rounds_min_bytes = value;
    } else {
        return PS_ERR_ARG;
    }
    return PS_OK;
}

int64_t ps_get_tuning(const char *key) {
    if (!key) return -1;
    if (!std::strcmp(key, "scan_kernel")) return g_tune.scan_kernel;
    if (!std::strcmp(key, "round_bytes")) return g_tune.round_bytes;
    if (!std::strcmp(key, "rounds_min_bytes")) return g_tune.rounds_min_bytes;
    if (!std::strcmp(key, "round_lead")) return g_tune.round_lead;
    if (!std::strcmp(key, "round_ramp")) return g_tune.round_ramp;
    if (!std::strcmp(key, "round_prefetch")) return g_tune.round_prefetch;
    if (!std::strcmp(key, "rows_kernel")) return g_tune.rows_kernel;
    if (!std::strcmp(key, "select_kernel")) return g_select_kernel;
    if (!std::strcmp(key, "stream_copy_in")) return g_tune.stream_copy_in;
    if (!std::strcmp(key, "stream_inflight")) return g_tune.stream_inflight;
    if (!std::strcmp(key, "rows_dynamic")) return g_tune.rows_dynamic;
    if (!std::strcmp(key, "rows_multi")) return g_tune.rows_multi;
    if (!std::strcmp(key, "reduce_blocks")) return g_tune.reduce_blocks;
    if (!std::strcmp(key, "add_chunked")) return g_tune.add_chunked;
    if (!std::strcmp(key, "tiles_row_lead")) return g_tune.tiles_row_lead;
    if (!std::strcmp(key, "float_exact")) return g_tune.float_exact;
    if (!std::strcmp(key, "seg_kernel")) return g_tune.seg_kernel;
    if (!std::strcmp(key, "stall_seed")) return g_tune.stall.seed;
    if (!std::strcmp(key, "stall_prob")) return g_tune.stall.prob;
    if (!std::strcmp(key, "stall_ns")) return g_tune.stall.max_ns;
    return -1;
}

int ps_scan(const void *in, void *out, int64_t n, int dtype_in, int dtype_out, int exclusive, uint64_t seed_bits,
            const void *seed_terms, int64_t n_seed_terms, void *total_out, void *scratch, size_t scratch_bytes,
            uint32_t epoch, void *stream) {
    if (!pair_ok(dtype_in, dtype_out)) return PS_ERR_DTYPE;
    if (n < 0 || n_seed_terms < 0 || (n > 0 && (!in || !out)) || (seed_terms == nullptr && n_seed_terms > 0))
        return PS_ERR_ARG;
    if (epoch == 0 || epoch > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) return write_seed_only(dtype_in, total_out, 1, seed_bits, seed_terms, n_seed_terms, 0, s);
    if (overlaps_partially(in, (size_t)n * dsize(dtype_in), out, (size_t)n * dsize(dtype_out))) return PS_ERR_OVERLAP;
    if (in == out && dsize(dtype_in) != dsize(dtype_out)) return PS_ERR_OVERLAP;
#define CALL(TI, TO)                                                                                          \
    return launch_scan<TI, TO>(in, out, 1, n, n, n, exclusive, seed_bits, seed_terms, n_seed_terms, total_out, \
                               scratch, scratch_bytes, epoch, s)
    PS_DISPATCH_PAIR(dtype_in, dtype_out, CALL);
#undef CALL
}

size_t ps_scan_batched_scratch_bytes(int64_t rows, int64_t cols, int dtype_in, int dtype_out) {
    if (!pair_ok(dtype_in, dtype_out) || rows < 0 || cols < 0) return 0;
    const int64_t tile = tile_of_dtype(dtype_in);
    size_t need = desc_bytes(rows * ((cols + tile - 1) / tile + 1));
    // short rows, and rows the rows kernel cannot stream (byte length not a multiple of 16), may
    // run as one segmented scan of the flat array
    if (rows > 1 && (cols * 4 <= tile || (cols * (int64_t)dsize(dtype_in)) % 16 != 0)) {
        const size_t a = seg_scratch_bytes(rows * cols, (int)dsize(dtype_in));
        const size_t b = seg_stream_scratch_bytes(rows * cols, (int)dsize(dtype_in));
        need = std::max(need, std::max(a, b));
    }
    return need;
}

int ps_scan_batched(const void *in, void *out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
                    int dtype_in, int dtype_out, int exclusive, const void *row_seeds, void *row_totals,
                    void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream) {
    if (!pair_ok(dtype_in, dtype_out)) return PS_ERR_DTYPE;
    if (rows < 0 || cols < 0 || ld_in < cols || ld_out < cols) return PS_ERR_ARG;
    if (epoch == 0 || epoch > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (rows == 0) return PS_OK;
    if (cols == 0) return write_seed_only(dtype_in, row_totals, rows, 0, row_seeds, rows, 1, s);
    if (!in || !out) return PS_ERR_ARG;
    if (in == out && (dsize(dtype_in) != dsize(dtype_out) || ld_in != ld_out)) return PS_ERR_OVERLAP;
    if (rows == 1) ld_in = ld_out = cols;
    // short contiguous rows of a large batch run as one segmented scan of the flat array on the
    // shared-memory-region kernel (launch_scan's uniform-segment route): a row per TMA item
    // leaves the rows kernel at 0.05-0.4 of the peak below ~2 KiB per row, the region kernel
    // holds 0.6-0.8 (scripts/short_rows_cross.py; crossover 2 KiB rows for integers, 1 KiB floats)
    const int64_t row_bytes = cols * (int64_t)dsize(dtype_in);
    const bool floats = dtype_in == PS_DTYPE_FLOAT32 || dtype_in == PS_DTYPE_FLOAT64;
    const bool flat_segments = rows > 1 && !row_seeds && ld_in == cols && ld_out == cols && g_tune.rows_kernel != 2 &&
                               g_tune.seg_kernel != 1 && g_tune.tiles_row_lead && row_bytes <= (floats ? 1024 : 2048) &&
                               rows * row_bytes >= g_tune.rounds_min_bytes && scratch &&
                               scratch_bytes >= seg_stream_scratch_bytes(rows * cols, (int)dsize(dtype_in)) &&
                               scratch_bytes >= seg_scratch_bytes(rows * cols, (int)dsize(dtype_in));
    // smaller batches of very short rows: the look-back tiles' uniform-segment scan (0.29-0.31 of
    // the peak at 2^22 int32 in rows of 64-256 columns, where a row per TMA item gives 0.05-0.18)
    const bool flat_small = rows > 1 && !row_seeds && ld_in == cols && ld_out == cols && g_tune.rows_kernel != 2 &&
                            g_tune.tiles_row_lead && row_bytes <= (floats ? 512 : 1024) && scratch &&
                            scratch_bytes >= seg_scratch_bytes(rows * cols, (int)dsize(dtype_in));
#define CALL(TI, TO)                                                                                            \
    if (rows > 1 && !flat_segments && !flat_small && rows_kernel_applies<TI, TO>(in, rows, cols, ld_in))        \
        return launch_rows<TI, TO>(in, out, rows, cols, ld_in, ld_out, exclusive, row_seeds, row_totals, scratch, \
                                   scratch_bytes, s);                                                           \
    return launch_scan<TI, TO>(in, out, rows, cols, ld_in, ld_out, exclusive, 0, row_seeds, row_seeds ? rows : 0, \
                               row_totals, scratch, scratch_bytes, epoch, s)
    PS_DISPATCH_PAIR(dtype_in, dtype_out, CALL);
#undef CALL
}

constexpr int64_t REDUCE_MAX_BLOCKS = 16384;  // block partials of reduce_blocks_kernel

size_t ps_reduce_scratch_bytes(int64_t n, int dtype_in) {
    (void)n;
    if (!dsize(dtype_in)) return 0;
    return 256 + 8 * (REDUCE_MAX_BLOCKS + 64);  // tickets + block (or CTA) partials
}

int ps_reduce(const void *in, int64_t n, int dtype_in, uint64_t seed_bits, const void *seed_terms,
              int64_t n_seed_terms, void *total_out, void *scratch, size_t scratch_bytes, void *stream) {
    if (!dsize(dtype_in)) return PS_ERR_DTYPE;
    if (n < 0 || !total_out || (n > 0 && !in)) return PS_ERR_ARG;
    if ((uintptr_t)in % dsize(dtype_in)) return PS_ERR_ARG;  // element-misaligned: not a typed array
    if (!scratch || scratch_bytes < ps_reduce_scratch_bytes(n, dtype_in)) return PS_ERR_SCRATCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t vec = 32 / (int64_t)dsize(dtype_in);
    int64_t want = (n / vec + REDUCE_THREADS * 4 - 1) / (REDUCE_THREADS * 4);
    int64_t grid = want < (int64_t)sms * 4 ? want : (int64_t)sms * 4;
    if (grid < 1) grid = 1;
    ReduceArgs a{};
    a.in = in;
    a.n = n;
    const uintptr_t ain = (uintptr_t)in % 32;
    a.lead = (int64_t)(((32 - ain) % 32) / dsize(dtype_in));
    a.seed_bits = seed_bits;
    a.seed_terms = seed_terms;
    a.n_seed_terms = n_seed_terms;
    a.total = total_out;
    a.ticket = static_cast<uint32_t *>(scratch);
    a.partials = reinterpret_cast<uint64_t *>(static_cast<char *>(scratch) + 256);
    a.blk_ticket = reinterpret_cast<unsigned long long *>(static_cast<char *>(scratch) + 8);
    // blocks from a ticket (>= 256 KiB each, <= REDUCE_MAX_BLOCKS of them)
    const int64_t nvec = n / vec;
    int64_t bv = (int64_t)REDUCE_THREADS * 16;
    if ((nvec + bv - 1) / bv > REDUCE_MAX_BLOCKS) bv = (nvec + REDUCE_MAX_BLOCKS - 1) / REDUCE_MAX_BLOCKS;
    a.blk_vecs = bv;
    if (g_tune.reduce_blocks && scratch_bytes >= 256 + 8 * (size_t)((nvec + bv - 1) / bv + 1)) {
#define CALL(T) reduce_blocks_kernel<T, REDUCE_THREADS><<<(unsigned)grid, REDUCE_THREADS, 0, s>>>(a)
        PS_DISPATCH_ONE(dtype_in, CALL);
#undef CALL
        return launch_rc();
    }
#define CALL(T) reduce_kernel<T, REDUCE_THREADS><<<(unsigned)grid, REDUCE_THREADS, 0, s>>>(a)
    PS_DISPATCH_ONE(dtype_in, CALL);
#undef CALL
    return launch_rc();
}

int ps_add_offset(void *buf, int64_t n, int dtype, uint64_t delta_bits, const void *delta_terms,
                  int64_t n_delta_terms, void *stream) {
    if (!dsize(dtype)) return PS_ERR_DTYPE;
    if (n < 0 || (n > 0 && !buf) || n_delta_terms < 0) return PS_ERR_ARG;
    if ((uintptr_t)buf % dsize(dtype)) return PS_ERR_ARG;  // element-misaligned: not a typed array
    if (n == 0) return PS_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uintptr_t ab = (uintptr_t)buf % 32;
    const int64_t lead = (int64_t)(((32 - ab) % 32) / dsize(dtype));
    const int64_t vec = 32 / (int64_t)dsize(dtype);
    int64_t want = (n / vec + 255) / 256;
    int64_t grid = want < (int64_t)sms * 8 ? want : (int64_t)sms * 8;
    if (g_tune.add_chunked) {
        // one CTA per 2048 vectors (64 KiB): the hardware hands blocks to whichever SM
        // is free, so faster SMs take more (grid-stride shares leave the grid waiting
        // for the slowest SMs)
        want = (n / vec + 2047) / 2048;
        grid = want > 0x7fffffffLL ? 0x7fffffffLL : want;
    }
    if (grid < 1) grid = 1;
#define CALL(T)                                                                                          \
    add_offset_kernel<T><<<(unsigned)grid, 256, 0, s>>>(static_cast<T *>(buf), n, lead, delta_bits, delta_terms, \
                                                        n_delta_terms)
    PS_DISPATCH_ONE(dtype, CALL);
#undef CALL
    return launch_rc();
}

size_t ps_scan_segmented_scratch_bytes(int64_t n, int dtype_in, int dtype_out) {
    if (!pair_ok(dtype_in, dtype_out) || n < 0) return 0;
    const size_t a = seg_scratch_bytes(n, (int)dsize(dtype_in)), b = seg_stream_scratch_bytes(n, (int)dsize(dtype_in));
    return a > b ? a : b;
}

int ps_scan_segmented(const void *in, void *out, int64_t n, const int64_t *seg_offsets, int64_t nseg,
                      int dtype_in, int dtype_out, int exclusive, void *seg_totals, void *scratch,
                      size_t scratch_bytes, uint32_t epoch, void *stream) {
    if (!pair_ok(dtype_in, dtype_out)) return PS_ERR_DTYPE;
    if (n < 0 || nseg < 0 || (nseg > 0 && !seg_offsets) || (n > 0 && (!in || !out))) return PS_ERR_ARG;
    if (epoch == 0 || epoch > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (nseg == 0) return PS_OK;
    // totals start from zero (empty segments keep it) -- except where the region kernel's
    // gather pass writes every entry itself (launch_seg_stream)
    auto zero_totals = [&]() -> int {
        return seg_totals ? cuda_rc(cudaMemsetAsync(seg_totals, 0, (size_t)nseg * 8, s)) : PS_OK;
    };
    if (n == 0) return zero_totals();
    if (overlaps_partially(in, (size_t)n * dsize(dtype_in), out, (size_t)n * dsize(dtype_out))) return PS_ERR_OVERLAP;
    if (in == out && dsize(dtype_in) != dsize(dtype_out)) return PS_ERR_OVERLAP;
    if (!scratch || scratch_bytes < seg_scratch_bytes(n, (int)dsize(dtype_in))) return PS_ERR_SCRATCH;
    // large inputs: the shared-memory-region kernel (one HBM read + write per element);
    // small ones, or buffers it cannot stream: the look-back tiles
    const bool big = n * (int64_t)dsize(dtype_in) >= g_tune.rounds_min_bytes;
    const bool regions = g_tune.seg_kernel == 2 || (g_tune.seg_kernel == 0 && big);
#define CALL(TI, TO)                                                                                           \
    {                                                                                                          \
        if (regions) {                                                                                         \
            const int rc = launch_seg_stream<TI, TO>(in, out, n, seg_offsets, nseg, exclusive, seg_totals,      \
                                                     scratch, scratch_bytes, epoch, s);                        \
            if (rc >= 0) return rc;                                                                            \
        }                                                                                                      \
        if (const int zrc = zero_totals()) return zrc;                                                         \
        return launch_segmented<TI, TO>(in, out, n, seg_offsets, nseg, exclusive, seg_totals, scratch, epoch, s); \
    }
    PS_DISPATCH_PAIR(dtype_in, dtype_out, CALL);
#undef CALL
}

size_t ps_shift_right_scratch_bytes(int64_t n, int dtype) {
    if (!dsize(dtype) || n < 0) return 0;
    return align_up((size_t)((n + SHIFT_TILE - 1) / SHIFT_TILE + 1) * 8, 256);
}

int ps_shift_right(const void *in, void *out, int64_t n, int dtype, uint64_t identity_bits, void *last_out,
                   void *scratch, size_t scratch_bytes, void *stream) {
    if (!dsize(dtype)) return PS_ERR_DTYPE;
    if (n < 0 || (n > 0 && (!in || !out))) return PS_ERR_ARG;
    if (n == 0) return PS_OK;
    if (overlaps_partially(in, (size_t)n * dsize(dtype), out, (size_t)n * dsize(dtype))) return PS_ERR_OVERLAP;
    if (!scratch || scratch_bytes < ps_shift_right_scratch_bytes(n, dtype)) return PS_ERR_SCRATCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t tiles = (n + SHIFT_TILE - 1) / SHIFT_TILE;
    if (tiles > 0x7fffffffLL) return PS_ERR_ARG;
#define CALL(T)                                                                                              \
    do {                                                                                                     \
        shift_gather_kernel<T><<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(                              \
            static_cast<const T *>(in), n, tiles, static_cast<T *>(scratch), static_cast<T *>(last_out));     \
        shift_tiles_kernel<T><<<(unsigned)tiles, SHIFT_THREADS, 0, s>>>(                                     \
            static_cast<const T *>(in), static_cast<T *>(out), n, static_cast<const T *>(scratch), identity_bits); \
    } while (0)
    PS_DISPATCH_ONE(dtype, CALL);
#undef CALL
    return launch_rc();
}

int ps_reduce_batched(const void *in, int64_t rows, int64_t cols, int64_t ld_in, int dtype_in, void *row_totals,
                      void *stream) {
    if (!dsize(dtype_in)) return PS_ERR_DTYPE;
    if (rows < 0 || cols < 0 || ld_in < cols || (rows > 0 && !row_totals) || (rows > 0 && cols > 0 && !in))
        return PS_ERR_ARG;
    if (rows == 0) return PS_OK;
    if (rows > 0x7fffffffLL) return PS_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
#define CALL(T) \
    reduce_rows_kernel<T, 256><<<(unsigned)rows, 256, 0, s>>>(static_cast<const T *>(in), cols, ld_in, row_totals)
    PS_DISPATCH_ONE(dtype_in, CALL);
#undef CALL
    return launch_rc();
}

int ps_add_offset_batched(void *buf, int64_t rows, int64_t cols, int64_t ld, int dtype, const void *row_deltas,
                          void *stream) {
    if (!dsize(dtype)) return PS_ERR_DTYPE;
    if (rows < 0 || cols < 0 || ld < cols || (rows > 0 && cols > 0 && (!buf || !row_deltas))) return PS_ERR_ARG;
    if (rows == 0 || cols == 0) return PS_OK;
    if (rows > 65535) return PS_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t gx = (cols + 255) / 256;
    if (gx > 1024) gx = 1024;
    dim3 grid((unsigned)gx, (unsigned)rows);
#define CALL(T) add_rows_kernel<T><<<grid, 256, 0, s>>>(static_cast<T *>(buf), cols, ld, row_deltas)
    PS_DISPATCH_ONE(dtype, CALL);
#undef CALL
    return launch_rc();
}

int ps_reduce_wrapped_blocks(const void *in, int64_t n, int w, uint64_t seed_bits, void *total_out, void *stream) {
    if (n < 0 || w < 1 || !total_out || (n > 0 && !in)) return PS_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    fill_seed_kernel<uint64_t><<<1, 32, 0, s>>>(static_cast<uint64_t *>(total_out), 1, seed_bits, nullptr, 0, 0);
    if (n > 0) {
        int64_t grid = (n / w + 255) / 256;
        if (grid > 148 * 8) grid = 148 * 8;
        if (grid < 1) grid = 1;
        wrapped_block_total_kernel<<<(unsigned)grid, 256, 0, s>>>(static_cast<const uint32_t *>(in), n, w,
                                                                  static_cast<unsigned long long *>(total_out));
    }
    return launch_rc();
}

size_t ps_scan_host_workspace_bytes(int64_t chunk_elems, int dtype_in, int dtype_out) {
    if (!pair_ok(dtype_in, dtype_out) || chunk_elems <= 0) return 0;
    return host_layout(chunk_elems, dtype_in, dtype_out).total;
}

int64_t ps_scan_host_epochs(int64_t n, int64_t chunk_elems) {
    if (n <= 0 || chunk_elems <= 0) return 1;
    return (n + chunk_elems - 1) / chunk_elems;
}

int ps_scan_host(const void *in_host, void *out_host, int64_t n, int dtype_in, int dtype_out, int exclusive,
                 uint64_t seed_bits, void *total_host, void *workspace, size_t workspace_bytes, int64_t chunk_elems,
                 uint32_t epoch, void *stream) {
    if (!pair_ok(dtype_in, dtype_out)) return PS_ERR_DTYPE;
    if (n < 0 || chunk_elems <= 0 || (n > 0 && (!in_host || !out_host))) return PS_ERR_ARG;
    const int64_t nchunks = ps_scan_host_epochs(n, chunk_elems);
    if (epoch == 0 || (uint64_t)epoch + (uint64_t)nchunks - 1 > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    const HostLayout L = host_layout(chunk_elems, dtype_in, dtype_out);
    if (!workspace || workspace_bytes < L.total) return PS_ERR_SCRATCH;
    cudaStream_t comp = static_cast<cudaStream_t>(stream);
    char *ws = static_cast<char *>(workspace);
    // two carry slots by chunk parity: chunk k seeds from slot (k-1)&1 and writes
    // its total to slot k&1, so no kernel reads the word another one writes
    char *carry = ws + L.off_carry;
    void *scratch = ws + L.off_scratch;
    if (n == 0) {
        if (total_host) std::memcpy(total_host, &seed_bits, 8);
        return PS_OK;
    }
    host::Pipe *P = nullptr;
    if (host::pipe_for_current_device(&P)) return PS_ERR_CUDA_BASE + (int)cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> guard(P->mu);
    cudaError_t e = P->init();
    if (e != cudaSuccess) return cuda_rc(e);
    const size_t bi = dsize(dtype_in), bo = dsize(dtype_out);
    auto chunk_of = [&](int64_t k) {
        const int64_t off = k * chunk_elems;
        const int64_t len = (n - off) < chunk_elems ? (n - off) : chunk_elems;
        return host::Chunk{(size_t)off * bi, (size_t)len * bi, (size_t)off * bo, (size_t)len * bo};
    };
    auto launch = [&](int64_t k, char *din, char *dout) {
        const int64_t off = k * chunk_elems;
        const int64_t len = (n - off) < chunk_elems ? (n - off) : chunk_elems;
        return ps_scan(din, dout, len, dtype_in, dtype_out, exclusive, k == 0 ? seed_bits : 0,
                       k == 0 ? nullptr : carry + 8 * ((k - 1) & 1), k == 0 ? 0 : 1, carry + 8 * (k & 1), scratch,
                       L.scratch, epoch + (uint32_t)k, comp);
    };
    int rc = host::run(*P, static_cast<const char *>(in_host), static_cast<char *>(out_host), nchunks,
                       (size_t)chunk_elems * bi, (size_t)chunk_elems * bo, ws + L.off_in, ws + L.off_out, L.in_slot,
                       L.out_slot, comp, chunk_of, launch, &e);
    if (rc > 0) return rc;
    if (rc < 0) return cuda_rc(e);
    if (total_host) {
        e = cudaMemcpy(total_host, carry + 8 * ((nchunks - 1) & 1), 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_rc(e);
    }
    return PS_OK;
}


// ---- host-buffer pipeline for batched rows (independent rows: no carry between chunks) ----
namespace ps {
namespace {
HostLayout host_layout_rows(int64_t chunk_rows, int64_t cols, int din, int dout) {
    HostLayout L{};
    const int64_t chunk = chunk_rows * cols;
    L.in_slot = align_up((size_t)chunk * dsize(din), 256);
    L.out_slot = align_up((size_t)chunk * dsize(dout), 256);
    L.scratch = align_up(ps_scan_batched_scratch_bytes(chunk_rows, cols, din, dout), 256);
    L.off_in = 0;
    L.off_out = L.off_in + NSLOT * L.in_slot;
    L.off_scratch = L.off_out + NSLOT * L.out_slot;
    L.off_carry = L.off_scratch + L.scratch;
    L.total = L.off_carry + 256;
    return L;
}
}  // namespace
}  // namespace ps

size_t ps_scan_batched_host_workspace_bytes(int64_t chunk_rows, int64_t cols, int dtype_in, int dtype_out) {
    if (!pair_ok(dtype_in, dtype_out) || chunk_rows <= 0 || cols <= 0) return 0;
    return host_layout_rows(chunk_rows, cols, dtype_in, dtype_out).total;
}

int ps_scan_batched_host(const void *in_host, void *out_host, int64_t rows, int64_t cols, int dtype_in,
                         int dtype_out, int exclusive, void *workspace, size_t workspace_bytes, int64_t chunk_rows,
                         uint32_t epoch, void *stream) {
    if (!pair_ok(dtype_in, dtype_out)) return PS_ERR_DTYPE;
    if (rows < 0 || cols < 0 || chunk_rows <= 0 || (rows > 0 && cols > 0 && (!in_host || !out_host)))
        return PS_ERR_ARG;
    const int64_t nchunks = ps_scan_host_epochs(rows, chunk_rows);
    if (epoch == 0 || (uint64_t)epoch + (uint64_t)nchunks - 1 > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    if (rows == 0 || cols == 0) return PS_OK;
    const HostLayout L = host_layout_rows(chunk_rows, cols, dtype_in, dtype_out);
    if (!workspace || workspace_bytes < L.total) return PS_ERR_SCRATCH;
    cudaStream_t comp = static_cast<cudaStream_t>(stream);
    char *ws = static_cast<char *>(workspace);
    void *scratch = ws + L.off_scratch;
    host::Pipe *P = nullptr;
    if (host::pipe_for_current_device(&P)) return PS_ERR_CUDA_BASE + (int)cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> guard(P->mu);
    cudaError_t e = P->init();
    if (e != cudaSuccess) return cuda_rc(e);
    const size_t bi = dsize(dtype_in), bo = dsize(dtype_out);
    auto rows_of = [&](int64_t k) { return (rows - k * chunk_rows) < chunk_rows ? (rows - k * chunk_rows) : chunk_rows; };
    auto chunk_of = [&](int64_t k) {
        const size_t e0 = (size_t)(k * chunk_rows * cols), elems = (size_t)(rows_of(k) * cols);
        return host::Chunk{e0 * bi, elems * bi, e0 * bo, elems * bo};
    };
    auto launch = [&](int64_t k, char *din, char *dout) {
        return ps_scan_batched(din, dout, rows_of(k), cols, cols, cols, dtype_in, dtype_out, exclusive, nullptr,
                               nullptr, scratch, L.scratch, epoch + (uint32_t)k, comp);
    };
    int rc = host::run(*P, static_cast<const char *>(in_host), static_cast<char *>(out_host), nchunks,
                       (size_t)(chunk_rows * cols) * bi, (size_t)(chunk_rows * cols) * bo, ws + L.off_in,
                       ws + L.off_out, L.in_slot, L.out_slot, comp, chunk_of, launch, &e);
    if (rc > 0) return rc;
    if (rc < 0) return cuda_rc(e);
    return PS_OK;
}

int ps_host_register(void *ptr, size_t bytes, int *registered) {
    if (registered) *registered = 0;
    if (!ptr || bytes == 0) return PS_OK;
    if (host::is_pinned(ptr, bytes)) return PS_OK;
    cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        return PS_OK;
    }
    if (e != cudaSuccess) return cuda_rc(e);
    if (registered) *registered = 1;
    return PS_OK;
}

int ps_host_unregister(void *ptr) {
    if (!ptr) return PS_OK;
    return cuda_rc(cudaHostUnregister(ptr));
}

int ps_host_is_pinned(const void *ptr) { return host::is_pinned(ptr, 1) ? 1 : 0; }

// ---- Blelloch tree step functions (simd.py:327-367) -------------------------------------------
int ps_tree_up_sweep(void *data, int64_t n, int dtype, void *root_out, void *stream) {
    if (!dsize(dtype)) return PS_ERR_DTYPE;
    if (n < 1 || (n & (n - 1)) || !data) return PS_ERR_ARG;  // power-of-two span (simd.py:370-372)
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t blk = n < TREE_B ? n : TREE_B;
    const int64_t nblk = n / blk;
    if (nblk > 0x7fffffffLL) return PS_ERR_ARG;
#define CALL(T)                                                                                                   \
    do {                                                                                                          \
        T *d = static_cast<T *>(data);                                                                            \
        tree_up_block_kernel<T><<<(unsigned)nblk, TREE_THREADS, 0, s>>>(d, n, blk);                                \
        for (int64_t st = blk; st < n; st *= 2) {                                                                 \
            const int64_t work = n / (2 * st);                                                                    \
            tree_up_level_kernel<T><<<(unsigned)((work + 255) / 256 < 148 * 16 ? (work + 255) / 256 : 148 * 16),     \
                                      256, 0, s>>>(d, n, st);                                                      \
        }                                                                                                         \
        if (root_out) cudaMemcpyAsync(root_out, d + n - 1, sizeof(T), cudaMemcpyDeviceToDevice, s);               \
    } while (0)
    PS_DISPATCH_ONE(dtype, CALL);
#undef CALL
    return launch_rc();
}

int ps_tree_down_sweep(void *data, int64_t n, int dtype, void *stream) {
    if (!dsize(dtype)) return PS_ERR_DTYPE;
    if (n < 1 || (n & (n - 1)) || !data) return PS_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t blk = n < TREE_B ? n : TREE_B;
    const int64_t nblk = n / blk;
    if (nblk > 0x7fffffffLL) return PS_ERR_ARG;
#define CALL(T)                                                                                                   \
    do {                                                                                                          \
        T *d = static_cast<T *>(data);                                                                            \
        int clear = 1;                                                                                            \
        for (int64_t st = n / 2; st >= blk; st /= 2) {                                                            \
            const int64_t work = n / (2 * st);                                                                    \
            tree_down_level_kernel<T><<<(unsigned)((work + 255) / 256 < 148 * 16 ? (work + 255) / 256 : 148 * 16),   \
                                        256, 0, s>>>(d, n, st, clear);                                             \
            clear = 0;                                                                                            \
        }                                                                                                         \
        tree_down_block_kernel<T><<<(unsigned)nblk, TREE_THREADS, 0, s>>>(d, n, blk, clear);                       \
    } while (0)
    PS_DISPATCH_ONE(dtype, CALL);
#undef CALL
    return launch_rc();
}

// ---- fused exchange of shard totals over NVLink (mailboxes) --------------------------------
int ps_publish_total(const void *total, void *const *peer_mailboxes, int n_peers, int rank, uint32_t epoch,
                     uint32_t prev_epoch, const void *own_mailbox, int *timeout_flag, void *stream) {
    if (!total || n_peers < 1 || n_peers > 1024 || rank < 0 || rank >= n_peers || !peer_mailboxes) return PS_ERR_ARG;
    if (prev_epoch && !own_mailbox) return PS_ERR_ARG;
    if (epoch == 0 || epoch > PS_EPOCH_MAX || prev_epoch > PS_EPOCH_MAX || (prev_epoch && prev_epoch == epoch))
        return PS_ERR_EPOCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int threads = ((n_peers + 31) / 32) * 32;
    publish_total_kernel<<<1, threads, 0, s>>>(static_cast<const uint64_t *>(total),
                                               reinterpret_cast<ulonglong2 *const *>(peer_mailboxes), n_peers, rank,
                                               epoch, prev_epoch, static_cast<const ulonglong2 *>(own_mailbox),
                                               timeout_flag);
    return launch_rc();
}

int ps_scan_mailbox(const void *in, void *out, int64_t n, int dtype_in, int dtype_out, int exclusive,
                    uint64_t seed_bits, const void *mailbox, int n_wait, uint32_t mail_epoch, int *timeout_flag,
                    void *total_out, void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream) {
    if (!pair_ok(dtype_in, dtype_out)) return PS_ERR_DTYPE;
    if (n < 0 || n_wait < 0 || (n > 0 && (!in || !out)) || (n_wait > 0 && !mailbox)) return PS_ERR_ARG;
    if (epoch == 0 || epoch > PS_EPOCH_MAX || mail_epoch == 0 || mail_epoch > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Mailbox m{static_cast<const ulonglong2 *>(mailbox), n_wait, mail_epoch, timeout_flag};
    if (n == 0) {
        if (!total_out) return PS_OK;
#define SEED(T) mailbox_seed_kernel<typename AccOf<T>::type><<<1, 32, 0, s>>>( \
        static_cast<typename AccOf<T>::type *>(total_out), seed_bits, m)
        PS_DISPATCH_ONE(dtype_in, SEED);
#undef SEED
        return launch_rc();
    }
    if (overlaps_partially(in, (size_t)n * dsize(dtype_in), out, (size_t)n * dsize(dtype_out))) return PS_ERR_OVERLAP;
    if (in == out && dsize(dtype_in) != dsize(dtype_out)) return PS_ERR_OVERLAP;
#define CALL(TI, TO)                                                                                          \
    return launch_scan<TI, TO>(in, out, 1, n, n, n, exclusive, seed_bits, nullptr, 0, total_out, scratch,    \
                               scratch_bytes, epoch, s, &m)
    PS_DISPATCH_PAIR(dtype_in, dtype_out, CALL);
#undef CALL
}

// ---- stream compaction / stable partition (select_kernels.cuh) -----------------------------
size_t ps_select_scratch_bytes(int64_t n) {
    if (n < 0) return 0;
    const int64_t ntiles = (n + SEL_TILE - 1) / SEL_TILE;
    const size_t counts = 256 + (size_t)ntiles * 8;
    const size_t desc = 256 + (size_t)(n / SS_P + 256 + 1) * 16;  // single-pass path: <= 256 CTAs
    return counts > desc ? counts : desc;
}


int ps_select(const void *values, const void *flags, int64_t n, int dtype_values, int dtype_flags, int partition,
              void *out, void *count_out, void *scratch, size_t scratch_bytes, uint32_t epoch, void *stream) {
    const size_t vb = dsize(dtype_values);
    const size_t fb = dtype_flags == PS_DTYPE_UINT8 ? 1 : dsize(dtype_flags);
    if (!vb || !fb) return PS_ERR_DTYPE;
    if (n < 0 || (partition != 0 && partition != 1)) return PS_ERR_ARG;
    if (epoch == 0 || epoch > PS_EPOCH_MAX) return PS_ERR_EPOCH;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        if (count_out) return cuda_rc(cudaMemsetAsync(count_out, 0, 8, s));
        return PS_OK;
    }
    if (!values || !flags || !out) return PS_ERR_ARG;
    const int64_t ntiles = (n + SEL_TILE - 1) / SEL_TILE;
    if (ntiles > 0x7fffffffLL) return PS_ERR_ARG;
    // out may hold up to n elements; it must not touch the inputs
    if (overlaps_partially(values, (size_t)n * vb, out, (size_t)n * vb) || values == out) return PS_ERR_OVERLAP;
    if (overlaps_partially(flags, (size_t)n * fb, out, (size_t)n * vb) || flags == out) return PS_ERR_OVERLAP;
    if (!scratch || scratch_bytes < ps_select_scratch_bytes(n)) return PS_ERR_SCRATCH;
    const bool aligned16 = (uintptr_t)values % 16 == 0 && (uintptr_t)flags % 16 == 0;
    // auto: the single pass pays off when re-reading the flags is expensive (4/8-byte
    // flags); byte flags re-read at 1 B/element and the three-launch path, with its
    // many small CTAs, is faster there (profiles/r01_select_bench.md)
    if (!partition && aligned16 && g_select_kernel != 1 &&
        (g_select_kernel == 2 || (n >= SELECT_STREAM_MIN && fb >= 4))) {
        long long *cnt = count_out ? static_cast<long long *>(count_out) : nullptr;
#define ONE(TV, TF) return launch_select_stream<TV, TF>(values, flags, n, out, cnt, scratch, scratch_bytes, epoch, s)
#define BY_F(TV)                        \
    do {                                \
        if (fb == 1) ONE(TV, uint8_t);  \
        if (fb == 4) ONE(TV, uint32_t); \
        ONE(TV, uint64_t);              \
    } while (0)
        if (vb == 4) BY_F(uint32_t);
        BY_F(uint64_t);
#undef BY_F
#undef ONE
    }
    char *base = static_cast<char *>(scratch);
    // (control word 16: words 0-1 are the rows kernel's row ticket when a scratch is shared)
    long long *total = count_out ? static_cast<long long *>(count_out) : reinterpret_cast<long long *>(base + 16);
    long long *counts = reinterpret_cast<long long *>(base + 256);
    const uintptr_t va = (uintptr_t)values, fa = (uintptr_t)flags;
    const int vec_ok = (va % 32 == 0) && (fb == 1 ? fa % 8 == 0 : fa % 32 == 0);
    int64_t grid = ntiles < 148 * 8 ? ntiles : 148 * 8;
    // 1) per-tile selected counts
#define COUNT(TF) \
    select_count_kernel<TF><<<(unsigned)grid, SEL_THREADS, 0, s>>>(static_cast<const TF *>(flags), n, ntiles, vec_ok, counts)
    if (fb == 1) COUNT(uint8_t);
    else if (fb == 4) COUNT(uint32_t);
    else COUNT(uint64_t);
#undef COUNT
    int rc = launch_rc();
    if (rc) return rc;
    // 2) exclusive offsets of the tiles + the selected total
    select_offsets_kernel<<<1, SEL_SCAN_THREADS, 0, s>>>(counts, ntiles, total);
    rc = launch_rc();
    if (rc) return rc;
    // 3) scatter through shared memory
    const size_t smem = (size_t)SEL_TILE * vb;
#define SCATTER(TV, TF, P)                                                                                    \
    do {                                                                                                       \
        auto k = select_scatter_kernel<TV, TF, P>;                                                             \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                       \
        k<<<(unsigned)ntiles, SEL_THREADS, smem, s>>>(static_cast<const TV *>(values), static_cast<const TF *>(flags), \
                                                      n, vec_ok, counts, total, static_cast<TV *>(out));       \
    } while (0)
#define BY_FLAG(TV, P)                                   \
    do {                                                 \
        if (fb == 1) SCATTER(TV, uint8_t, P);            \
        else if (fb == 4) SCATTER(TV, uint32_t, P);      \
        else SCATTER(TV, uint64_t, P);                   \
    } while (0)
    if (vb == 4) {
        if (partition) BY_FLAG(uint32_t, true);
        else BY_FLAG(uint32_t, false);
    } else {
        if (partition) BY_FLAG(uint64_t, true);
        else BY_FLAG(uint64_t, false);
    }
#undef BY_FLAG
#undef SCATTER
    return launch_rc();
}

}  // extern "C"
