// scripts/rows_variants.cu -- f32 compute-throughput experiment on the rows kernel (dev tool)
#include <cstdio>
#include <cstdlib>
#include "../paper_2312_14874_b200/csrc/rows_kernel.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename T, int SW, int RPC, int NBUF, int NCH>
void run(const char *name, void *in, void *out, int64_t rows, int64_t cols) {
    using Geo = RowsGeom<T, SW, RPC, NBUF, NCH>;
    auto k = scan_rows_kernel<T, T, SW, RPC, NBUF, NCH>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM));
    int per = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, Geo::THREADS, Geo::SMEM));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    RowsArgs a{};
    a.in = in; a.out = out; a.rows = rows; a.cols = cols; a.ld_in = cols; a.ld_out = cols; a.vec_out = 1;
    int G = per * sms;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<G, Geo::THREADS, Geo::SMEM>>>(a);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) k<<<G, Geo::THREADS, Geo::SMEM>>>(a);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
    printf("%-22s per_sm=%d  %7.1f us  %6.0f GB/s\n", name, per, ms * 1e3, 2.0 * rows * cols * sizeof(T) / (ms * 1e-3) / 1e9);
}

int main() {
    void *in, *out;
    CK(cudaMalloc(&in, 1ll << 30)); CK(cudaMalloc(&out, 1ll << 30)); CK(cudaMemset(in, 0, 1ll << 30));
    const int64_t rows = 16384, cols = 16384;
    run<float, 8, 2, 2, 16>("f32 8w rpc2 nbuf2", in, out, rows, cols);
    run<float, 8, 2, 3, 16>("f32 8w rpc2 nbuf3", in, out, rows, cols);
    run<float, 4, 2, 2, 16>("f32 4w rpc2 nbuf2", in, out, rows, cols);
    run<float, 8, 1, 2, 32>("f32 8w rpc1 nbuf2", in, out, rows, cols);
    run<float, 8, 2, 2, 8>("f32 8w rpc2 nch8", in, out, rows, cols);
    run<int, 8, 2, 2, 16>("i32 8w rpc2 nbuf2", in, out, rows, cols);
    run<int64_t, 8, 2, 2, 16>("i64 8w rpc2 nbuf2", in, out, rows, cols / 2);
    run<int64_t, 8, 4, 3, 16>("i64 8w rpc4 nbuf3", in, out, rows, cols / 2);
    return 0;
}
