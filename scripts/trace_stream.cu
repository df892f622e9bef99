// scripts/trace_stream.cu -- per-(region, CTA) timeline of scan_stream_kernel (dev tool).
// gpurun_out/trace_stream_<name>.bin: 8 uint64 per (region, CTA):
//   [0] TMA issued [1] data landed (reducer) [2] portion total published [3] ledger gather start
//   [4] gather done [5] carries ready [6] scanner warp 0 sees its data [7] scanner warp 0 done
#define PS_TRACE 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2312_14874_b200/csrc/stream_kernel.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename TIn, typename TOut, int SW, int ROWS, int NBUF, int RWP>
void run(const char *name, void *in, void *out, int64_t n, void *scratch, uint32_t &epoch) {
    using Geo = StreamGeom<TIn, SW, ROWS, NBUF, RWP>;
    auto kern = scan_stream_kernel<TIn, TOut, SW, ROWS, NBUF, RWP>;
    const int64_t unit = (int64_t)SW * Geo::CHUNK;
    const int64_t P = (32 << 10) / (int64_t)sizeof(TIn) / unit * unit;
    const int smem = Geo::smem(P);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t G = 148;
    StreamArgs a{};
    a.in = in; a.out = out; a.lo = 0; a.hi = n; a.portion = P;
    a.rounds = (n + P * G - 1) / (P * G);
    a.desc = (ulonglong2 *)((char *)scratch + 256);
    a.inflight = getenv("INFL") ? atoi(getenv("INFL")) : 2;
    void *params[] = {&a};
    for (int w = 0; w < 3; ++w) { a.epoch = ++epoch; CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(Geo::THREADS), params, smem, 0)); }
    CK(cudaDeviceSynchronize());
    uint64_t *tr; const size_t tb = (size_t)a.rounds * G * 64;
    CK(cudaMalloc(&tr, tb)); CK(cudaMemset(tr, 0, tb));
    CK(cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr)));
    a.epoch = ++epoch;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(Geo::THREADS), params, smem, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    uint64_t *nul = nullptr; CK(cudaMemcpyToSymbol(g_trace, &nul, sizeof(nul)));
    std::vector<uint64_t> h(tb / 8); CK(cudaMemcpy(h.data(), tr, tb, cudaMemcpyDeviceToHost));
    char path[256]; snprintf(path, sizeof path, "gpurun_out/trace_stream_%s.bin", name);
    FILE *f = fopen(path, "wb"); fwrite(h.data(), 8, h.size(), f); fclose(f);
    printf("%s: rounds=%lld  %.1f us  %.1f GB/s (traced)\n", name, (long long)a.rounds, ms * 1e3,
           (double)n * (sizeof(TIn) + sizeof(TOut)) / (ms * 1e-3) / 1e9);
    cudaFree(tr);
}

int main() {
    void *in, *out, *scratch;
    CK(cudaMalloc(&in, 1ll << 31)); CK(cudaMalloc(&out, 1ll << 31)); CK(cudaMalloc(&scratch, 64 << 20));
    CK(cudaMemset(in, 0, 1ll << 31)); CK(cudaMemset(scratch, 0, 64 << 20));
    uint32_t epoch = 0;
    run<float, float, 8, 4, 6, 4>("f32", in, out, 1ll << 28, scratch, epoch);
    run<int64_t, int64_t, 8, 4, 6, 4>("i64", in, out, 1ll << 27, scratch, epoch);
    run<int64_t, int64_t, 8, 4, 6, 4>("i64_cfg1", in, out, 1ll << 24, scratch, epoch);
    return 0;
}
