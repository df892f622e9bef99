/* oracle/scan_oracle.h -- TEST INFRASTRUCTURE: CPU restatement of the reference
 * prefix-sum kernels (see scan_oracle.c).  Never linked by the product. */
#ifndef SCAN_ORACLE_H
#define SCAN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes: identical numbering to include/prefixscan_b200.h PS_DTYPE_* */
enum {
    OR_DTYPE_INT32 = 1,
    OR_DTYPE_INT64 = 2,
    OR_DTYPE_UINT32 = 3,
    OR_DTYPE_FLOAT32 = 5,
    OR_DTYPE_FLOAT64 = 6,
};

/* plan.py:24-37 SchemeId */
enum {
    OR_SCHEME_SCAN_INCREMENT_EQUAL = 0,
    OR_SCHEME_ACCUMULATE_SCAN_EQUAL = 1,
    OR_SCHEME_SCAN_INCREMENT_PLUS_ONE = 2,
    OR_SCHEME_ACCUMULATE_SCAN_PLUS_ONE = 3,
};

enum { OR_ERR_DTYPE = 1, OR_ERR_ARG = 2 };

/* accumulator slots are 8 bytes: uint64 for uint32 data, double otherwise */
int or_scan(int dtype, const void *src, void *dst, int64_t start, int64_t len,
            const void *offset, void *total);
int or_accumulate(int dtype, const void *src, int64_t start, int64_t len, void *total);
int or_increment(int dtype, void *buf, int64_t start, int64_t len, const void *delta);
int or_shift_right(int dtype, void *buf, int64_t n, const void *identity_elem, void *last_elem);
int or_horizontal(int dtype, int w, const void *src, void *dst, int64_t start, int64_t len,
                  const void *offset, void *total);
int or_simd_accumulate(int dtype, int w, const void *src, int64_t start, int64_t len, void *total);
int or_vertical_pass1_scan(int dtype, void *data, int64_t start, int64_t k, int w,
                           const void *carry, void *totals);
int or_vertical_pass1_accumulate(int dtype, const void *data, int64_t start, int64_t k, int w,
                                 void *totals);
int or_vertical_pass2_increment(int dtype, void *data, int64_t start, int64_t k, int w,
                                const void *offsets);
int or_vertical_pass2_scan(int dtype, void *data, int64_t start, int64_t k, int w,
                           const void *offsets);
int or_up_sweep(int dtype, void *data, int64_t start, int64_t len, void *root_elem);
int or_down_sweep(int dtype, void *data, int64_t start, int64_t len);
int or_add_back(int dtype, void *data, const void *scratch, int64_t start, int64_t len,
                const void *offset);
int or_scan_widen_i32_i64(const int32_t *src, int64_t *dst, int64_t n, int exclusive,
                          double offset, int64_t *total);
int or_engine_scan(int dtype, const void *src, void *dst, int64_t n, int threads, int scheme,
                   double d0, double d_last, int64_t block_len, int simd_w, void *total);
int or_rows_scan_widen_i32_i64(const int32_t *src, int64_t *dst, int64_t rows, int64_t cols,
                               int64_t ld_in, int64_t ld_out, int threads, int simd_w);

#ifdef __cplusplus
}
#endif
#endif
