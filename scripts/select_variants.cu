// scripts/select_variants.cu -- single-pass select kernel timing (dev tool).  Build with
// -DPS_EXP_NOLEDGER to time it without the grid-wide ledger exchange (results wrong).
#include <cstdio>
#include <cstdlib>
#include "../paper_2312_14874_b200/csrc/select_stream.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename T>
__global__ void fillf(T *f, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f[i] = (T)((i * 2654435761ull >> 7) & 1);
}

template <typename TV, typename TF>
void run(const char *name, void *v, void *f, void *out, int64_t n, void *scratch, uint32_t &epoch) {
    using Geo = SelectStreamGeom<TV, TF>;
    auto kern = select_stream_kernel<TV, TF>;
    fillf<TF><<<1184, 256>>>((TF *)f, n);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM));
    const int G = 148;
    SelectArgs a{};
    a.values = v; a.flags = f; a.out = out; a.n = n; a.portion = SS_P;
    a.rounds = (n + SS_P * G - 1) / (SS_P * G);
    a.desc = (ulonglong2 *)((char *)scratch + 256);
    void *params[] = {&a};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 10; ++it) {
        ++epoch;
        a.want = ((uint64_t)(~epoch) << 32) | ((uint64_t)epoch << 2);
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(SS_THREADS), params, Geo::SMEM, 0));
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2 && ms < best) best = ms;
    }
    const double alg = (double)n * (sizeof(TV) + sizeof(TF)) + 0.5 * n * sizeof(TV);
    printf("%-16s NBUF=%d rounds=%lld: %.1f us  %.1f GB/s (alg, p=0.5)\n", name, Geo::NBUF, (long long)a.rounds,
           best * 1e3, alg / (best * 1e-3) / 1e9);
}

int main() {
    void *v, *f, *out, *scratch;
    CK(cudaMalloc(&v, 1ll << 31)); CK(cudaMalloc(&f, 1ll << 31)); CK(cudaMalloc(&out, 1ll << 31));
    CK(cudaMalloc(&scratch, 64 << 20)); CK(cudaMemset(scratch, 0, 64 << 20));
    uint32_t epoch = 0;
    const int64_t N = 1ll << 28;
    run<uint32_t, uint32_t>("i32_i32", v, f, out, N, scratch, epoch);
    run<uint32_t, uint8_t>("i32_u8", v, f, out, N, scratch, epoch);
    run<uint64_t, uint8_t>("i64_u8", v, f, out, N, scratch, epoch);
    return 0;
}
