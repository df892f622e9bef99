/*
 * oracle/scan_oracle.c -- CPU restatement of the reference prefix-sum path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("kind": "port") for bench.py.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_2312_14874_b200) never links or calls it.
 *
 * It restates, loop for loop, the numba kernels of the reference package
 * /root/reference/pkg/src/prefixscan (cited per function below), including
 * the accumulator typing numba infers for them:
 *
 *   element uint32  -> accumulator uint64  (core.py:40-48 coerce_offset -> np.uint64,
 *                                            uint64 + uint32 stays uint64)
 *   element float32 -> accumulator float64 (core.py:40-48 -> np.float64)
 *   element int32 / int64 -> accumulator float64: numba unifies
 *                      uint64 (the coerced offset) + signed int into float64
 *                      (signature (int64[],int64[],int64,int64,uint64)->float64),
 *                      so the reference is exact only while |running sum| < 2^53.
 *
 * Accumulators cross this ABI as 8 raw bytes: uint64 for uint32 data, IEEE
 * double for everything else.  Parity of this restatement is pinned against
 * golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures, tests/test_oracle.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#include "scan_oracle.h"

/* ---------------------------------------------------------------------------
 * Type plumbing.  T = element type, A = accumulator type (see header comment).
 * LOAD converts an element to the accumulator, STORE converts back the way
 * numba's setitem does (float64 -> int via truncating cast through int64).
 * ------------------------------------------------------------------------- */
#define CVT_U32(a) ((uint32_t)(a))
#define CVT_F32(a) ((float)(a))
#define CVT_I64(a) ((int64_t)(a))
#define CVT_I32(a) ((int32_t)(int64_t)(a))
#define CVT_F64(a) ((double)(a))

#define FOR_EACH_KIND(X)                  \
    X(u32, uint32_t, uint64_t, CVT_U32)   \
    X(f32, float, double, CVT_F32)        \
    X(i64, int64_t, double, CVT_I64)      \
    X(i32, int32_t, double, CVT_I32)      \
    X(f64, double, double, CVT_F64)

/* core.py:86-92 _scan_kernel: acc = offset; acc += src[i]; dst[i] = acc */
/* core.py:95-100 _accumulate_kernel */
/* core.py:103-106 _increment_kernel: buf[i] = buf[i] + delta */
/* core.py:109-115 _shift_right_kernel */
/* simd.py:75-101 _make_horizontal_kernel: per w-block Hillis-Steele rounds in
 *   the ELEMENT dtype, + acc, acc += v[w-1]; scalar tail */
/* simd.py:104-121 _make_simd_accumulate_kernel: w lane partials (acc dtype) */
#define DEFINE_KERNELS(K, T, A, CVT)                                                   \
    static A scan_##K(const T *src, T *dst, int64_t start, int64_t len, A offset) {    \
        A acc = offset;                                                                \
        for (int64_t i = start; i < start + len; ++i) {                                \
            acc = acc + (A)src[i];                                                     \
            dst[i] = CVT(acc);                                                         \
        }                                                                              \
        return acc;                                                                    \
    }                                                                                  \
    static A accumulate_##K(const T *src, int64_t start, int64_t len, A offset) {      \
        A acc = offset;                                                                \
        for (int64_t i = start; i < start + len; ++i) acc = acc + (A)src[i];           \
        return acc;                                                                    \
    }                                                                                  \
    static void increment_##K(T *buf, int64_t start, int64_t len, A delta) {           \
        for (int64_t i = start; i < start + len; ++i) buf[i] = CVT((A)buf[i] + delta); \
    }                                                                                  \
    static T shift_right_##K(T *buf, int64_t n, T identity) {                          \
        T last = buf[n - 1];                                                           \
        for (int64_t i = n - 1; i > 0; --i) buf[i] = buf[i - 1];                       \
        buf[0] = identity;                                                             \
        return last;                                                                   \
    }                                                                                  \
    /* W is a compile-time lane count so gcc keeps the w-vector in registers  \
     * and emits vector shifts/adds; the arithmetic (order, types) is the      \
     * reference's, unchanged.  Dispatched from horizontal_##K below. */        \
    static inline __attribute__((always_inline)) A horizontal_w_##K(           \
        const int W, const T *src, T *dst, int64_t start, int64_t len,          \
        A offset) {                                                             \
        A acc = offset;                                                         \
        T v[16];                                                                \
        int64_t end = start + len, b = start;                                   \
        while (b + W <= end) {                                                  \
            for (int j = 0; j < W; ++j) v[j] = src[b + j];                      \
            for (int sh = 1; sh < W; sh <<= 1)                                  \
                for (int j = W - 1; j >= sh; --j) v[j] = (T)(v[j] + v[j - sh]); \
            for (int j = 0; j < W; ++j) dst[b + j] = CVT((A)v[j] + acc);        \
            acc = acc + (A)v[W - 1];                                            \
            b += W;                                                             \
        }                                                                       \
        for (int64_t i = b; i < end; ++i) {                                     \
            acc = acc + (A)src[i];                                              \
            dst[i] = CVT(acc);                                                  \
        }                                                                       \
        return acc;                                                             \
    }                                                                           \
    static A horizontal_##K(int w, const T *src, T *dst, int64_t start,         \
                            int64_t len, A offset) {                            \
        switch (w) {                                                            \
            case 4: return horizontal_w_##K(4, src, dst, start, len, offset);   \
            case 8: return horizontal_w_##K(8, src, dst, start, len, offset);   \
            default: return horizontal_w_##K(16, src, dst, start, len, offset); \
        }                                                                       \
    }                                                                           \
    static inline __attribute__((always_inline)) A simd_accumulate_w_##K(      \
        const int W, const T *src, int64_t start, int64_t len) {                \
        A part[16];                                                             \
        for (int j = 0; j < W; ++j) part[j] = (A)0;                             \
        int64_t end = start + len, b = start;                                   \
        while (b + W <= end) {                                                  \
            for (int j = 0; j < W; ++j) part[j] = part[j] + (A)src[b + j];      \
            b += W;                                                             \
        }                                                                       \
        A acc = (A)0;                                                           \
        for (int j = 0; j < W; ++j) acc = acc + part[j];                        \
        for (int64_t i = b; i < end; ++i) acc = acc + (A)src[i];                \
        return acc;                                                             \
    }                                                                           \
    static A simd_accumulate_##K(int w, const T *src, int64_t start,            \
                                 int64_t len) {                                 \
        switch (w) {                                                            \
            case 4: return simd_accumulate_w_##K(4, src, start, len);           \
            case 8: return simd_accumulate_w_##K(8, src, start, len);           \
            default: return simd_accumulate_w_##K(16, src, start, len);         \
        }                                                                       \
    }                                                                           \
    /* simd.py:164-175 _vertical_pass1_scan: lane-chunk scans, lane 0 seeded */         \
    static void vp1_scan_##K(T *data, int64_t start, int64_t k, int w, A carry,        \
                             A *totals) {                                              \
        A run[16];                                                                     \
        for (int l = 0; l < w; ++l) run[l] = (A)0;                                     \
        run[0] = carry;                                                                \
        for (int64_t j = 0; j < k; ++j)                                                \
            for (int l = 0; l < w; ++l) {                                              \
                int64_t idx = start + (int64_t)l * k + j;                              \
                run[l] = run[l] + (A)data[idx];                                        \
                data[idx] = CVT(run[l]);                                               \
            }                                                                          \
        for (int l = 0; l < w; ++l) totals[l] = run[l];                                \
    }                                                                                  \
    /* simd.py:178-186 _vertical_pass1_accumulate */                                   \
    static void vp1_acc_##K(const T *data, int64_t start, int64_t k, int w,            \
                            A *totals) {                                               \
        A run[16];                                                                     \
        for (int l = 0; l < w; ++l) run[l] = (A)0;                                     \
        for (int64_t j = 0; j < k; ++j)                                                \
            for (int l = 0; l < w; ++l)                                                \
                run[l] = run[l] + (A)data[start + (int64_t)l * k + j];                 \
        for (int l = 0; l < w; ++l) totals[l] = run[l];                                \
    }                                                                                  \
    /* simd.py:189-195 _vertical_pass2_increment */                                    \
    static void vp2_inc_##K(T *data, int64_t start, int64_t k, int w, const A *offs) { \
        for (int64_t j = 0; j < k; ++j)                                                \
            for (int l = 0; l < w; ++l) {                                              \
                int64_t idx = start + (int64_t)l * k + j;                              \
                data[idx] = CVT((A)data[idx] + offs[l]);                               \
            }                                                                          \
    }                                                                                  \
    /* simd.py:198-206 _vertical_pass2_scan */                                         \
    static void vp2_scan_##K(T *data, int64_t start, int64_t k, int w,                 \
                             const A *offs) {                                          \
        A run[16];                                                                     \
        for (int l = 0; l < w; ++l) run[l] = offs[l];                                  \
        for (int64_t j = 0; j < k; ++j)                                                \
            for (int l = 0; l < w; ++l) {                                              \
                int64_t idx = start + (int64_t)l * k + j;                              \
                run[l] = run[l] + (A)data[idx];                                        \
                data[idx] = CVT(run[l]);                                               \
            }                                                                          \
    }                                                                                  \
    /* simd.py:326-334 _up_sweep (element dtype, in place) */                          \
    static T up_sweep_##K(T *data, int64_t start, int64_t len) {                       \
        for (int64_t stride = 1; stride < len; stride *= 2) {                          \
            int64_t step = stride * 2;                                                 \
            for (int64_t i = start + step - 1; i < start + len; i += step)             \
                data[i] = (T)(data[i] + data[i - stride]);                             \
        }                                                                              \
        return data[start + len - 1];                                                  \
    }                                                                                  \
    /* simd.py:337-347 _down_sweep */                                                  \
    static void down_sweep_##K(T *data, int64_t start, int64_t len) {                  \
        data[start + len - 1] = (T)0;                                                  \
        for (int64_t stride = len / 2; stride >= 1; stride /= 2) {                     \
            int64_t step = stride * 2;                                                 \
            for (int64_t i = start + step - 1; i < start + len; i += step) {           \
                T t = data[i - stride];                                                \
                data[i - stride] = data[i];                                            \
                data[i] = (T)(data[i] + t);                                            \
            }                                                                          \
        }                                                                              \
    }                                                                                  \
    /* simd.py:350-353 _add_back: (data + scratch) in element dtype, + offset (acc) */ \
    static void add_back_##K(T *data, const T *scratch, int64_t start, int64_t len,    \
                             A offset) {                                               \
        for (int64_t i = 0; i < len; ++i)                                              \
            data[start + i] = CVT((A)(T)(data[start + i] + scratch[i]) + offset);      \
    }

FOR_EACH_KIND(DEFINE_KERNELS)

/* ---------------------------------------------------------------------------
 * ABI helpers: 8-byte accumulator slots.
 * ------------------------------------------------------------------------- */
static int kind_of(int dtype) {
    switch (dtype) {
        case OR_DTYPE_UINT32: return 0;
        case OR_DTYPE_FLOAT32: return 1;
        case OR_DTYPE_INT64: return 2;
        case OR_DTYPE_INT32: return 3;
        case OR_DTYPE_FLOAT64: return 4;
        default: return -1;
    }
}

#define ACC_GET(K, p) (*(const K *)(p))
#define ACC_PUT(K, p, v) (*(K *)(p) = (v))

#define DISPATCH(dtype, MACRO)                                    \
    switch (kind_of(dtype)) {                                     \
        case 0: MACRO(u32, uint32_t, uint64_t); break;            \
        case 1: MACRO(f32, float, double); break;                 \
        case 2: MACRO(i64, int64_t, double); break;               \
        case 3: MACRO(i32, int32_t, double); break;               \
        case 4: MACRO(f64, double, double); break;                \
        default: return OR_ERR_DTYPE;                             \
    }

int or_scan(int dtype, const void *src, void *dst, int64_t start, int64_t len,
            const void *offset, void *total) {
#define M(K, T, A) ACC_PUT(A, total, scan_##K((const T *)src, (T *)dst, start, len, ACC_GET(A, offset)))
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_accumulate(int dtype, const void *src, int64_t start, int64_t len, void *total) {
#define M(K, T, A) ACC_PUT(A, total, accumulate_##K((const T *)src, start, len, (A)0))
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_increment(int dtype, void *buf, int64_t start, int64_t len, const void *delta) {
#define M(K, T, A) increment_##K((T *)buf, start, len, ACC_GET(A, delta))
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_shift_right(int dtype, void *buf, int64_t n, const void *identity_elem, void *last_elem) {
    if (n <= 0) return 0;
#define M(K, T, A) *(T *)last_elem = shift_right_##K((T *)buf, n, *(const T *)identity_elem)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

static int bad_w(int w) { return !(w == 4 || w == 8 || w == 16); }

int or_horizontal(int dtype, int w, const void *src, void *dst, int64_t start, int64_t len,
                  const void *offset, void *total) {
    if (bad_w(w)) return OR_ERR_ARG;
#define M(K, T, A) ACC_PUT(A, total, horizontal_##K(w, (const T *)src, (T *)dst, start, len, ACC_GET(A, offset)))
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_simd_accumulate(int dtype, int w, const void *src, int64_t start, int64_t len, void *total) {
    if (bad_w(w)) return OR_ERR_ARG;
#define M(K, T, A) ACC_PUT(A, total, simd_accumulate_##K(w, (const T *)src, start, len))
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_vertical_pass1_scan(int dtype, void *data, int64_t start, int64_t k, int w,
                           const void *carry, void *totals) {
    if (w < 1 || w > 16) return OR_ERR_ARG;
#define M(K, T, A) vp1_scan_##K((T *)data, start, k, w, ACC_GET(A, carry), (A *)totals)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_vertical_pass1_accumulate(int dtype, const void *data, int64_t start, int64_t k, int w,
                                 void *totals) {
    if (w < 1 || w > 16) return OR_ERR_ARG;
#define M(K, T, A) vp1_acc_##K((const T *)data, start, k, w, (A *)totals)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_vertical_pass2_increment(int dtype, void *data, int64_t start, int64_t k, int w,
                                const void *offsets) {
    if (w < 1 || w > 16) return OR_ERR_ARG;
#define M(K, T, A) vp2_inc_##K((T *)data, start, k, w, (const A *)offsets)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_vertical_pass2_scan(int dtype, void *data, int64_t start, int64_t k, int w,
                           const void *offsets) {
    if (w < 1 || w > 16) return OR_ERR_ARG;
#define M(K, T, A) vp2_scan_##K((T *)data, start, k, w, (const A *)offsets)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_up_sweep(int dtype, void *data, int64_t start, int64_t len, void *root_elem) {
    if (len <= 0) return OR_ERR_ARG;
#define M(K, T, A) *(T *)root_elem = up_sweep_##K((T *)data, start, len)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_down_sweep(int dtype, void *data, int64_t start, int64_t len) {
    if (len <= 0) return OR_ERR_ARG;
#define M(K, T, A) down_sweep_##K((T *)data, start, len)
    DISPATCH(dtype, M)
#undef M
    return 0;
}

int or_add_back(int dtype, void *data, const void *scratch, int64_t start, int64_t len,
                const void *offset) {
#define M(K, T, A) add_back_##K((T *)data, (const T *)scratch, start, len, ACC_GET(A, offset))
    DISPATCH(dtype, M)
#undef M
    return 0;
}

/* ---------------------------------------------------------------------------
 * Mixed-dtype composite (no reference entry point exists; SURVEY 8(c) gaps):
 * int32 flags/deltas -> int64 output = widening copy, then the reference's
 * int64 scan (core.py:86-92), then for exclusive mode the reference's
 * exclusive_from_inclusive (core.py:141-151) whose returned "last" is the total.
 * ------------------------------------------------------------------------- */
int or_scan_widen_i32_i64(const int32_t *src, int64_t *dst, int64_t n, int exclusive,
                          double offset, int64_t *total) {
    for (int64_t i = 0; i < n; ++i) dst[i] = (int64_t)src[i];
    double acc = scan_i64(dst, dst, 0, n, offset);
    if (exclusive) {
        int64_t ident = (int64_t)offset;
        if (n == 0) {
            *total = ident;
            return 0;
        }
        *total = shift_right_i64(dst, n, ident);
    } else {
        *total = (int64_t)acc;
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Engine port: plan.py:131-241 (compute_layout / compute_grid) and
 * engine.py:278-384 (_execute / _next_carry / _result_owner), with POSIX
 * threads and one barrier per iteration (engine.py:314).  This is the CPU
 * baseline the GPU path is timed against ("kind": "port").
 * ------------------------------------------------------------------------- */
enum { ROLE_SCAN = 0, ROLE_ACC = 1, ROLE_INC = 2 };

#define OR_MAXT 256
#define OR_MAXS (OR_MAXT + 2)

typedef struct { int thread, span, role, seeded; } item_t;
typedef struct {
    int nspans;
    int64_t start[OR_MAXS], len[OR_MAXS];
    int np1, np2;
    item_t p1[OR_MAXS], p2[OR_MAXS];
    int scheme; /* effective scheme (d0 == 0 collapses +1 -> equal, plan.py:149-152) */
} layout_t;

static int64_t align_down(int64_t x, int64_t w) { return (x / w) * w; }

/* plan.py:122-128 _single_thread_layout */
static void single_layout(layout_t *L, int64_t start, int64_t n, int scheme) {
    L->nspans = 1;
    L->start[0] = start;
    L->len[0] = n;
    L->scheme = scheme;
    if (scheme == OR_SCHEME_ACCUMULATE_SCAN_EQUAL || scheme == OR_SCHEME_ACCUMULATE_SCAN_PLUS_ONE) {
        L->np1 = 1; L->p1[0] = (item_t){0, 0, ROLE_ACC, 0};
        L->np2 = 1; L->p2[0] = (item_t){0, 0, ROLE_SCAN, 0};
    } else {
        L->np1 = 1; L->p1[0] = (item_t){0, 0, ROLE_SCAN, 1};
        L->np2 = 0;
    }
}

static void set_spans(layout_t *L, int64_t start, const int64_t *lens, int cnt) {
    int64_t pos = start;
    L->nspans = cnt;
    for (int i = 0; i < cnt; ++i) {
        L->start[i] = pos;
        L->len[i] = lens[i];
        pos += lens[i];
    }
}

/* plan.py:131-197 compute_layout */
static int compute_layout(layout_t *L, int64_t n, int m, int scheme, double d0, double d_last,
                          int64_t w, int64_t start, int need_last_total) {
    int64_t lens[OR_MAXS], base;
    if (m < 1 || m > OR_MAXT) return OR_ERR_ARG;
    if (w < 1) w = 1;
    int plus_one = scheme == OR_SCHEME_SCAN_INCREMENT_PLUS_ONE || scheme == OR_SCHEME_ACCUMULATE_SCAN_PLUS_ONE;
    if (plus_one && d0 == 0.0) {
        scheme = scheme == OR_SCHEME_SCAN_INCREMENT_PLUS_ONE ? OR_SCHEME_SCAN_INCREMENT_EQUAL
                                                             : OR_SCHEME_ACCUMULATE_SCAN_EQUAL;
        plus_one = 0;
    }
    if (plus_one) {
        if (scheme == OR_SCHEME_SCAN_INCREMENT_PLUS_ONE)
            base = align_down((int64_t)((double)n / ((double)m + d0)), w);
        else
            base = align_down((int64_t)((double)n / ((double)(m - 1) + d0 + d_last)), w);
    } else {
        base = align_down(n / m, w);
    }
    if (n < (int64_t)m * w || base == 0) {
        single_layout(L, start, n, scheme);
        return 0;
    }
    L->scheme = scheme;
    if (scheme == OR_SCHEME_SCAN_INCREMENT_EQUAL) {
        for (int j = 0; j < m - 1; ++j) lens[j] = base;
        lens[m - 1] = n - base * (m - 1);
        set_spans(L, start, lens, m);
        L->np1 = m;
        for (int j = 0; j < m; ++j) L->p1[j] = (item_t){j, j, ROLE_SCAN, j == 0};
        L->np2 = m - 1;
        for (int j = 1; j < m; ++j) L->p2[j - 1] = (item_t){j, j, ROLE_INC, 0};
    } else if (scheme == OR_SCHEME_ACCUMULATE_SCAN_EQUAL) {
        for (int j = 0; j < m - 1; ++j) lens[j] = base;
        lens[m - 1] = n - base * (m - 1);
        set_spans(L, start, lens, m);
        L->np1 = need_last_total ? m : m - 1;
        for (int j = 0; j < L->np1; ++j) L->p1[j] = (item_t){j, j, ROLE_ACC, 0};
        L->np2 = m;
        for (int j = 0; j < m; ++j) L->p2[j] = (item_t){j, j, ROLE_SCAN, 0};
    } else if (scheme == OR_SCHEME_SCAN_INCREMENT_PLUS_ONE) {
        for (int j = 0; j < m; ++j) lens[j] = base;
        lens[m] = n - base * m;
        set_spans(L, start, lens, m + 1);
        L->np1 = m;
        for (int j = 0; j < m; ++j) L->p1[j] = (item_t){j, j, ROLE_SCAN, j == 0};
        L->np2 = m;
        for (int j = 1; j < m; ++j) L->p2[j - 1] = (item_t){j, j, ROLE_INC, 0};
        L->p2[m - 1] = (item_t){0, m, ROLE_SCAN, 0};
    } else { /* ACCUMULATE_SCAN_PLUS_ONE */
        int64_t first = align_down((int64_t)(d0 * (double)base), w);
        lens[0] = first;
        for (int j = 1; j < m; ++j) lens[j] = base;
        lens[m] = n - first - base * (m - 1);
        if (lens[m] < 0) return OR_ERR_ARG;
        set_spans(L, start, lens, m + 1);
        L->np1 = m;
        L->p1[0] = (item_t){0, 0, ROLE_SCAN, 1};
        for (int j = 1; j < m; ++j) L->p1[j] = (item_t){j, j, ROLE_ACC, 0};
        L->np2 = m;
        for (int j = 1; j < m; ++j) L->p2[j - 1] = (item_t){j, j, ROLE_SCAN, 0};
        L->p2[m - 1] = (item_t){0, m, ROLE_SCAN, 0};
    }
    return 0;
}

typedef struct {
    int dtype, threads, simd_w;
    const void *src;
    void *dst;
    int64_t n;
    int niter;
    layout_t *layouts;
    pthread_barrier_t *barrier;
    double *ledger_d;     /* (2, OR_MAXS) float64 ledger for double-accumulator kinds */
    uint64_t *ledger_u;   /* (2, OR_MAXS) uint64 ledger for uint32 */
    uint64_t result_bits; /* accumulator bits of the grand total */
} engine_job_t;

typedef struct { engine_job_t *job; int wid; } worker_arg_t;

static int result_owner(const layout_t *L) {
    if (L->scheme == OR_SCHEME_ACCUMULATE_SCAN_EQUAL && L->np2) return L->p2[L->np2 - 1].thread;
    return 0;
}

#define ENGINE_WORKER(K, T, A, LEDGER)                                                             \
    static void engine_worker_##K(engine_job_t *job, int wid) {                                    \
        const T *src = (const T *)job->src;                                                        \
        T *dst = (T *)job->dst;                                                                    \
        int w = job->simd_w;                                                                       \
        A carry = (A)0;                                                                            \
        for (int k = 0; k < job->niter; ++k) {                                                     \
            const layout_t *L = &job->layouts[k];                                                  \
            A *row = (A *)job->LEDGER + (k % 2) * OR_MAXS;                                              \
            for (int t = 0; t < L->np1; ++t) { /* engine.py:295-307 pass 1 */                      \
                const item_t *it = &L->p1[t];                                                      \
                if (it->thread != wid) continue;                                                   \
                int64_t s = L->start[it->span], ln = L->len[it->span];                             \
                if (it->role == ROLE_SCAN) {                                                       \
                    A seed = it->seeded ? carry : (A)0;                                            \
                    row[it->span] = w ? horizontal_##K(w, src, dst, s, ln, seed)                   \
                                      : scan_##K(src, dst, s, ln, seed);                           \
                } else {                                                                           \
                    row[it->span] = w ? simd_accumulate_##K(w, src, s, ln)                         \
                                      : accumulate_##K(src, s, ln, (A)0);                          \
                }                                                                                  \
            }                                                                                      \
            pthread_barrier_wait(job->barrier); /* engine.py:314 */                                \
            int any_seeded = 0;                                                                    \
            for (int t = 0; t < L->np1; ++t) any_seeded |= L->p1[t].seeded;                        \
            A base = any_seeded ? (A)0 : carry; /* engine.py:323 */                                \
            int have_last = 0;                                                                     \
            A last_scan_total = (A)0;                                                              \
            for (int t = 0; t < L->np2; ++t) { /* engine.py:325-337 pass 2 */                      \
                const item_t *it = &L->p2[t];                                                      \
                if (it->thread != wid) continue;                                                   \
                int64_t s = L->start[it->span], ln = L->len[it->span];                             \
                A offset = base;                                                                   \
                for (int i = 0; i < it->span; ++i) offset = offset + row[i];                       \
                if (it->role == ROLE_INC) {                                                        \
                    if (ln) increment_##K(dst, s, ln, offset);                                     \
                } else {                                                                           \
                    last_scan_total = w ? horizontal_##K(w, src, dst, s, ln, offset)               \
                                        : scan_##K(src, dst, s, ln, offset);                       \
                    have_last = 1;                                                                 \
                }                                                                                  \
            }                                                                                      \
            /* engine.py:346-377 _next_carry */                                                    \
            if (L->scheme == OR_SCHEME_ACCUMULATE_SCAN_EQUAL) {                                    \
                if (L->np1 == L->nspans) {                                                         \
                    A acc = carry;                                                                 \
                    for (int i = 0; i < L->nspans; ++i) acc = acc + row[i];                        \
                    carry = acc;                                                                   \
                } else if (have_last && L->np2 && L->p2[L->np2 - 1].thread == wid) {               \
                    carry = last_scan_total;                                                       \
                }                                                                                  \
            } else if (L->scheme == OR_SCHEME_SCAN_INCREMENT_EQUAL) {                              \
                if (wid == 0) {                                                                    \
                    A acc = (A)0;                                                                  \
                    for (int i = 0; i < L->nspans; ++i) acc = acc + row[i];                        \
                    carry = acc;                                                                   \
                }                                                                                  \
            } else if (wid == 0) {                                                                 \
                if (have_last) {                                                                   \
                    carry = last_scan_total;                                                       \
                } else {                                                                           \
                    A acc = (A)0;                                                                  \
                    for (int i = 0; i < L->nspans; ++i) acc = acc + row[i];                        \
                    carry = acc;                                                                   \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        if (result_owner(&job->layouts[job->niter - 1]) == wid)                                    \
            memcpy(&job->result_bits, &carry, 8);                                                  \
    }

ENGINE_WORKER(u32, uint32_t, uint64_t, ledger_u)
ENGINE_WORKER(f32, float, double, ledger_d)
ENGINE_WORKER(i64, int64_t, double, ledger_d)
ENGINE_WORKER(i32, int32_t, double, ledger_d)
ENGINE_WORKER(f64, double, double, ledger_d)

static void *engine_thread(void *p) {
    worker_arg_t *a = (worker_arg_t *)p;
    switch (kind_of(a->job->dtype)) {
        case 0: engine_worker_u32(a->job, a->wid); break;
        case 1: engine_worker_f32(a->job, a->wid); break;
        case 2: engine_worker_i64(a->job, a->wid); break;
        case 3: engine_worker_i32(a->job, a->wid); break;
        case 4: engine_worker_f64(a->job, a->wid); break;
    }
    return NULL;
}

int or_engine_scan(int dtype, const void *src, void *dst, int64_t n, int threads, int scheme,
                   double d0, double d_last, int64_t block_len, int simd_w, void *total) {
    if (kind_of(dtype) < 0) return OR_ERR_DTYPE;
    if (threads < 1 || threads > OR_MAXT || block_len < 0) return OR_ERR_ARG;
    if (simd_w && bad_w(simd_w)) return OR_ERR_ARG;
    if (scheme < 0 || scheme > 3) return OR_ERR_ARG;
    /* plan.py:211-241 compute_grid */
    int64_t region_len = block_len > 0 ? block_len * threads : n;
    if (region_len <= 0) region_len = n > 1 ? n : 1;
    int64_t niter = n > 0 ? (n + region_len - 1) / region_len : 1;
    layout_t *layouts = (layout_t *)calloc((size_t)niter, sizeof(layout_t));
    if (!layouts) return OR_ERR_ARG;
    int64_t lane = simd_w ? simd_w : 16; /* ScanRequest.lane_width default (engine.py:87) */
    for (int64_t i = 0; i < niter; ++i) {
        int64_t rs = i * region_len;
        int64_t rl = n - rs < region_len ? n - rs : region_len;
        if (n == 0) { rs = 0; rl = 0; }
        int rc = compute_layout(&layouts[i], rl, threads, scheme, d0, d_last, lane, rs, i != niter - 1);
        if (rc) { free(layouts); return rc; }
    }
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)threads);
    double ledger_d[2 * OR_MAXS];
    uint64_t ledger_u[2 * OR_MAXS];
    memset(ledger_d, 0, sizeof ledger_d);
    memset(ledger_u, 0, sizeof ledger_u);
    engine_job_t job = {dtype, threads, simd_w, src, dst, n, (int)niter, layouts, &bar,
                        ledger_d, ledger_u, 0};
    pthread_t tids[OR_MAXT];
    worker_arg_t args[OR_MAXT];
    for (int t = 0; t < threads; ++t) {
        args[t].job = &job;
        args[t].wid = t;
        if (t) pthread_create(&tids[t], NULL, engine_thread, &args[t]);
    }
    engine_thread(&args[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    pthread_barrier_destroy(&bar);
    free(layouts);
    memcpy(total, &job.result_bits, 8);
    return 0;
}

/* Per-row batched composite used as the cfg4 CPU baseline: rows x cols int32
 * deltas widened to int64 and scanned per row (per-row
 * horizontal_scan on a thread pool).  Rows are split across `threads`. */
typedef struct {
    const int32_t *src; int64_t *dst; int64_t rows, cols, ld_in, ld_out; int w, threads, wid;
} rows_arg_t;

static void *rows_thread(void *p) {
    rows_arg_t *a = (rows_arg_t *)p;
    for (int64_t r = a->wid; r < a->rows; r += a->threads) {
        int64_t *d = a->dst + r * a->ld_out;
        const int32_t *s = a->src + r * a->ld_in;
        for (int64_t c = 0; c < a->cols; ++c) d[c] = (int64_t)s[c];
        if (a->w) horizontal_i64(a->w, d, d, 0, a->cols, 0.0);
        else scan_i64(d, d, 0, a->cols, 0.0);
    }
    return NULL;
}

int or_rows_scan_widen_i32_i64(const int32_t *src, int64_t *dst, int64_t rows, int64_t cols,
                               int64_t ld_in, int64_t ld_out, int threads, int simd_w) {
    if (threads < 1 || threads > OR_MAXT) return OR_ERR_ARG;
    if (simd_w && bad_w(simd_w)) return OR_ERR_ARG;
    pthread_t tids[OR_MAXT];
    rows_arg_t args[OR_MAXT];
    for (int t = 0; t < threads; ++t) {
        args[t] = (rows_arg_t){src, dst, rows, cols, ld_in, ld_out, simd_w, threads, t};
        if (t) pthread_create(&tids[t], NULL, rows_thread, &args[t]);
    }
    rows_thread(&args[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    return 0;
}
