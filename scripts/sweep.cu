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
    struct Pair { const char *name; int di, dout, ei, eo; };
    const Pair pairs[] = {
        {"int32 -> int32", PS_DTYPE_INT32, PS_DTYPE_INT32, 4, 4},
        {"int32 -> int64", PS_DTYPE_INT32, PS_DTYPE_INT64, 4, 8},
        {"int64 -> int64", PS_DTYPE_INT64, PS_DTYPE_INT64, 8, 8},
        {"uint32 -> uint32", PS_DTYPE_UINT32, PS_DTYPE_UINT32, 4, 4},
        {"uint32 -> uint64", PS_DTYPE_UINT32, PS_DTYPE_UINT64, 4, 8},
        {"uint64 -> uint64", PS_DTYPE_UINT64, PS_DTYPE_UINT64, 8, 8},
        {"float32 -> float32", PS_DTYPE_FLOAT32, PS_DTYPE_FLOAT32, 4, 4},
        {"float32 -> float64", PS_DTYPE_FLOAT32, PS_DTYPE_FLOAT64, 4, 8},
        {"float64 -> float64", PS_DTYPE_FLOAT64, PS_DTYPE_FLOAT64, 8, 8},
    };
    if (argc > 1 && !strcmp(argv[1], "threshold")) {
        printf("| pair | n (bytes in) | look-back us | stream us | L2-rounds us |\n|---|---|---|---|---|\n");
        for (const Pair &p : pairs) {
            if (p.di != PS_DTYPE_INT64 && p.di != PS_DTYPE_FLOAT32 && !(p.di == PS_DTYPE_INT32 && p.dout == PS_DTYPE_INT64)) continue;
            for (int lg = 18; lg <= 25; ++lg) {
                const int64_t n = (1ll << lg) / p.ei * 4;  // 2^lg * 4 bytes of input
                double t[3];
                for (int k = 0; k < 3; ++k) {
                    PK(ps_set_tuning("scan_kernel", k == 0 ? 1 : (k == 1 ? 3 : 2)));
                    t[k] = time_scan(in, out, n, p.di, p.dout, 0, 20) * 1e3;
                }
                printf("| %s | %lld (%lld KiB) | %.1f | %.1f | %.1f |\n", p.name, (long long)n,
                       (long long)(n * p.ei >> 10), t[0], t[1], t[2]);
            }
        }
        PK(ps_set_tuning("scan_kernel", 0));
        return 0;
    }
    printf("| pair | n | auto kernel | us | GB/s | look-back GB/s | L2-rounds GB/s | stream GB/s |\n");
    printf("|---|---|---|---|---|---|---|---|\n");
    for (const Pair &p : pairs) {
        for (int lg : {20, 24, 28}) {
            const int64_t n = 1ll << lg;
            const double gb = (double)n * (p.ei + p.eo) / 1e9;
            PK(ps_set_tuning("scan_kernel", 0));
            const double ms = time_scan(in, out, n, p.di, p.dout, 0, 20);
            const bool big = n * p.ei >= ps_get_tuning("rounds_min_bytes");
            double k[3] = {0, 0, 0};
            if (lg == 28) {
                for (int i = 0; i < 3; ++i) {
                    PK(ps_set_tuning("scan_kernel", i + 1));
                    k[i] = gb / (time_scan(in, out, n, p.di, p.dout, 0, 10) * 1e-3);
                }
                PK(ps_set_tuning("scan_kernel", 0));
            }
            if (lg == 28)
                printf("| %s | 2^%d | %s | %.1f | %.0f | %.0f | %.0f | %.0f |\n", p.name, lg, big ? "stream" : "look-back",
                       ms * 1e3, gb / (ms * 1e-3), k[0], k[1], k[2]);
            else
                printf("| %s | 2^%d | %s | %.1f | %.0f | | | |\n", p.name, lg, big ? "stream" : "look-back", ms * 1e3,
                       gb / (ms * 1e-3));
        }
    }
    return 0;
}
