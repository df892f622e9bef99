// scripts/sweep.cu -- kernel / geometry timing sweep through the public C-ABI
// (development tool; not part of the library).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/sweep scripts/sweep.cu \
//        -Lpaper_2312_14874_b200 -lprefixscan_b200 -Xlinker -rpath='$ORIGIN/../paper_2312_14874_b200'
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../include/prefixscan_b200.h"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
#define PK(x) do { int rc = (x); if (rc) { printf("ps error %d (%s) at %d\n", rc, ps_error_string(rc), __LINE__); exit(1); } } while (0)

static void *g_scratch;
static size_t g_scratch_bytes;
static uint32_t g_epoch;

static double time_scan(const void *in, void *out, int64_t n, int di, int dout, int excl, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w)
        PK(ps_scan(in, out, n, di, dout, excl, 0, nullptr, 0, nullptr, g_scratch, g_scratch_bytes, ++g_epoch, nullptr));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
        PK(ps_scan(in, out, n, di, dout, excl, 0, nullptr, 0, nullptr, g_scratch, g_scratch_bytes, ++g_epoch, nullptr));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

struct Case {
    const char *name;
    int64_t n;
    int di, dout, excl, ei, eo;
};

int main(int argc, char **argv) {
    const int64_t bytes = 1ll << 32;  // 4 GiB per buffer
    void *in, *out;
    CK(cudaMalloc(&in, bytes));
    CK(cudaMalloc(&out, bytes));
    CK(cudaMemset(in, 0, bytes));
    g_scratch_bytes = 256 << 20;
    CK(cudaMalloc(&g_scratch, g_scratch_bytes));
    CK(cudaMemset(g_scratch, 0, g_scratch_bytes));
    Case cases[] = {
        {"cfg1 i64", 1ll << 24, PS_DTYPE_INT64, PS_DTYPE_INT64, 0, 8, 8},
        {"cfg2 f32", 1ll << 28, PS_DTYPE_FLOAT32, PS_DTYPE_FLOAT32, 0, 4, 4},
        {"cfg3 i32>i64 ex", 1ll << 28, PS_DTYPE_INT32, PS_DTYPE_INT64, 1, 4, 8},
        {"2^28 i64", 1ll << 28, PS_DTYPE_INT64, PS_DTYPE_INT64, 0, 8, 8},
    };
    const int64_t rbs[] = {32ll << 20, 40ll << 20, 48ll << 20, 64ll << 20, 80ll << 20};
    for (const Case &c : cases) {
        PK(ps_set_tuning("scan_kernel", 1));
        double ms = time_scan(in, out, c.n, c.di, c.dout, c.excl, 10);
        double gb = (double)c.n * (c.ei + c.eo) / 1e9;
        printf("%-16s lookback            %8.1f us %7.1f GB/s\n", c.name, ms * 1e3, gb / (ms * 1e-3));
        PK(ps_set_tuning("scan_kernel", 3));
        ms = time_scan(in, out, c.n, c.di, c.dout, c.excl, 10);
        printf("%-16s stream (smem regions) %8.1f us %7.1f GB/s\n", c.name, ms * 1e3, gb / (ms * 1e-3));
        PK(ps_set_tuning("scan_kernel", 2));
        for (int lead : {1, 2})
            for (int64_t rb : rbs) {
                PK(ps_set_tuning("round_bytes", rb));
                PK(ps_set_tuning("round_lead", lead));
                ms = time_scan(in, out, c.n, c.di, c.dout, c.excl, 10);
                printf("%-16s rounds lead=%d R=%3lld MiB %8.1f us %7.1f GB/s\n", c.name, lead, (long long)(rb >> 20),
                       ms * 1e3, gb / (ms * 1e-3));
            }
        PK(ps_set_tuning("round_lead", 2));
        PK(ps_set_tuning("round_bytes", 0));
    }
    return 0;
}
