// scripts/sweep.cu -- tile-geometry / look-back timing sweep of scan_tiles_kernel
// on one GPU (development tool; not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/sweep scripts/sweep.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2312_14874_b200/csrc/scan_kernels.cuh"

using namespace ps;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void copy256(const V256 *in, V256 *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        stg256_stream(out + i, ldg256_stream(in + i));
}

template <typename TIn, typename TOut, int WARPS, int ROWS>
void run(const char *name, void *in, void *out, int64_t n, void *scratch, uint32_t &epoch, int flags, int reps) {
    constexpr int64_t TILE = (int64_t)WARPS * ROWS * 32 * (32 / sizeof(TIn));
    ScanArgs a{};
    a.in = in; a.out = out; a.rows = 1; a.cols = n; a.ld_in = n; a.ld_out = n;
    a.tiles_per_row = (n + TILE - 1) / TILE; a.vec_ok = 1; a.debug_flags = flags;
    char *p = (char *)scratch;
    a.desc.d = (ulonglong2 *)(p + 256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) { a.epoch = ++epoch; scan_tiles_kernel<TIn, TOut, WARPS, ROWS><<<(unsigned)a.tiles_per_row, WARPS * 32>>>(a); }
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) { a.epoch = ++epoch; scan_tiles_kernel<TIn, TOut, WARPS, ROWS><<<(unsigned)a.tiles_per_row, WARPS * 32>>>(a); }
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, scan_tiles_kernel<TIn, TOut, WARPS, ROWS>, WARPS * 32, 0);
    double gbs = (double)n * (sizeof(TIn) + sizeof(TOut)) / (ms * 1e-3) / 1e9;
    printf("%-10s W=%2d R=%d tile=%6lld occ=%d lookback=%s  %8.1f us  %7.1f GB/s\n", name, WARPS, ROWS, (long long)TILE,
           occ, (flags & 1) ? "off" : "on ", ms * 1e3, gbs);
}

template <typename TIn, typename TOut>
void family(const char *name, int64_t n, void *in, void *out, void *scratch, uint32_t &epoch) {
    for (int f : {0, 1}) {
        run<TIn, TOut, 4, 4>(name, in, out, n, scratch, epoch, f, 20);
        run<TIn, TOut, 8, 2>(name, in, out, n, scratch, epoch, f, 20);
        run<TIn, TOut, 8, 4>(name, in, out, n, scratch, epoch, f, 20);
        run<TIn, TOut, 8, 8>(name, in, out, n, scratch, epoch, f, 20);
        run<TIn, TOut, 16, 2>(name, in, out, n, scratch, epoch, f, 20);
        run<TIn, TOut, 16, 4>(name, in, out, n, scratch, epoch, f, 20);
    }
}

int main() {
    const int64_t bytes = 1ll << 31;  // 2 GiB per buffer
    void *in, *out, *scratch;
    CK(cudaMalloc(&in, bytes)); CK(cudaMalloc(&out, bytes)); CK(cudaMalloc(&scratch, 256 << 20));
    CK(cudaMemset(in, 0, bytes)); CK(cudaMemset(scratch, 0, 256 << 20));
    uint32_t epoch = 0;
    {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        int64_t nv = (1ll << 30) / 32;  // 1 GiB copy
        for (int g : {148 * 4, 148 * 8, 148 * 16}) {
            copy256<<<g, 256>>>((V256 *)in, (V256 *)out, nv);
            cudaEventRecord(e0);
            for (int r = 0; r < 20; ++r) copy256<<<g, 256>>>((V256 *)in, (V256 *)out, nv);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
            printf("copy256 grid=%d  %8.1f us  %7.1f GB/s\n", g, ms * 1e3, 2.0 * (1 << 30) / (ms * 1e-3) / 1e9);
        }
    }
    family<float, float>("cfg2 f32", 1ll << 28, in, out, scratch, epoch);
    family<int64_t, int64_t>("cfg1 i64", 1ll << 24, in, out, scratch, epoch);
    family<int64_t, int64_t>("2^27 i64", 1ll << 27, in, out, scratch, epoch);
    family<int32_t, int64_t>("cfg3 i32", 1ll << 28, in, out, scratch, epoch);
    return 0;
}
