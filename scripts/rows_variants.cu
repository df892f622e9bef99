// scripts/rows_variants.cu -- f32 compute-throughput experiment on the rows kernel (dev tool)
#include <cstdio>
#include <cstdlib>
#include "../paper_2312_14874_b200/csrc/rows_kernel.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename T, typename TO, int SW, int RPC, int NBUF, int NCH>
void run(const char *name, void *in, void *out, int64_t rows, int64_t cols) {
    using Geo = RowsGeom<T, SW, RPC, NBUF, NCH>;
    auto k = scan_rows_kernel<T, TO, SW, RPC, NBUF, NCH>;
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
    printf("%-22s per_sm=%d  %7.1f us  %6.0f GB/s\n", name, per, ms * 1e3, 1.0 * rows * cols * (sizeof(T) + sizeof(TO)) / (ms * 1e-3) / 1e9);
}

int main() {
    void *in, *out;
    CK(cudaMalloc(&in, 1ll << 30)); CK(cudaMalloc(&out, 1ll << 30)); CK(cudaMemset(in, 0, 1ll << 30));
    const int64_t rows = 16384, cols = 16384;
    run<int, int64_t, 8, 4, 3, 16>("i32>i64 nb3 nch16", in, out, rows, cols);
    run<int, int64_t, 8, 4, 6, 8>("i32>i64 nb6 nch8", in, out, rows, cols);
    run<int, int64_t, 8, 4, 4, 12>("i32>i64 nb4 nch12", in, out, rows, cols);
    run<int, int64_t, 8, 4, 8, 6>("i32>i64 nb8 nch6", in, out, rows, cols);
    run<int, int64_t, 8, 4, 12, 4>("i32>i64 nb12 nch4", in, out, rows, cols);
    run<float, float, 8, 2, 2, 16>("f32 rpc2 nb2 nch16", in, out, rows, cols);
    run<float, float, 8, 2, 4, 8>("f32 rpc2 nb4 nch8", in, out, rows, cols);
    run<float, float, 8, 4, 6, 8>("f32 rpc4 nb6 nch8", in, out, rows, cols);
    run<int, int64_t, 8, 4, 3, 16>("i32>i64 again", in, out, rows, cols);
    return 0;
}
