// scripts/tiles_small.cu -- look-back tile geometry at small n (dev tool)
#include <cstdio>
#include <cstdlib>
#include "../paper_2312_14874_b200/csrc/scan_kernels.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename T, int WARPS, int ROWS>
void run(const char *name, void *in, void *out, int64_t n, void *scratch, uint32_t &epoch) {
    constexpr int64_t TILE = (int64_t)WARPS * ROWS * 32 * (32 / sizeof(T));
    ScanArgs a{};
    a.in = in; a.out = out; a.rows = 1; a.cols = n; a.ld_in = n; a.ld_out = n;
    a.tiles_per_row = (n + TILE - 1) / TILE; a.vec_ok = 1; a.lead = 0;
    a.desc.d = (ulonglong2 *)((char *)scratch + 256);
    const int64_t tiles = a.tiles_per_row;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) { a.epoch = ++epoch; scan_tiles_kernel<T, T, WARPS, ROWS><<<(unsigned)tiles, WARPS * 32>>>(a); }
    CK(cudaDeviceSynchronize());
    const int reps = 50;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) { a.epoch = ++epoch; scan_tiles_kernel<T, T, WARPS, ROWS><<<(unsigned)tiles, WARPS * 32>>>(a); }
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    printf("%-22s n=%-9lld tiles=%-6lld %7.2f us %7.1f GB/s\n", name, (int64_t)n, (int64_t)tiles, ms * 1e3,
           2.0 * n * sizeof(T) / (ms * 1e-3) / 1e9);
}

int main() {
    void *in, *out, *scratch;
    CK(cudaMalloc(&in, 1 << 28)); CK(cudaMalloc(&out, 1 << 28)); CK(cudaMalloc(&scratch, 16 << 20));
    CK(cudaMemset(in, 0, 1 << 28)); CK(cudaMemset(scratch, 0, 16 << 20));
    uint32_t epoch = 0;
    for (int64_t n : {1ll << 18, 1ll << 20, 1ll << 22}) {
        run<float, 8, 4>("f32 8w x4 rows", in, out, n, scratch, epoch);
        run<float, 8, 2>("f32 8w x2 rows", in, out, n, scratch, epoch);
        run<float, 8, 1>("f32 8w x1 row", in, out, n, scratch, epoch);
        run<float, 4, 2>("f32 4w x2 rows", in, out, n, scratch, epoch);
        run<int64_t, 8, 4>("i64 8w x4 rows", in, out, n, scratch, epoch);
        run<int64_t, 8, 1>("i64 8w x1 row", in, out, n, scratch, epoch);
    }
    return 0;
}
