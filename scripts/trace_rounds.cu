// scripts/trace_rounds.cu -- per-(region, CTA) timeline of scan_rounds_kernel (dev tool).
// Build with -DNO_TRACE for timing only (no trace instrumentation compiled in).
// Environment: LEAD=<lead regions> PF=<1: L2 bulk prefetch of the reducer portion>.
// gpurun_out/trace_sub_<name>.bin: CTA 0's per-sub-tile scanner/producer timestamps
// (scripts/analyze_sub.py).
// gpurun_out/trace_rounds_<name>.bin: 8 uint64 per (region, CTA):
//   [0] reducer start [1] reducer published [2] scanner ledger start [3] ledger done [4] region scanned
#ifndef NO_TRACE
#define PS_TRACE 1
#endif
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2312_14874_b200/csrc/rounds_kernel.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename T>
__global__ void fill_kernel(T *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (T)(i % 3);
}

template <typename TIn, typename TOut, int SW, int ROWS, int STAGES, int RWP, int RSTAGES, int MINB = 1>
void run(const char *name, void *in, void *out, int64_t n, void *scratch, uint32_t &epoch, int64_t round_bytes) {
    using Geo = RoundGeom<TIn, TOut, SW, ROWS, STAGES, RWP, RSTAGES>;
    auto kern = scan_rounds_kernel<TIn, TOut, SW, ROWS, STAGES, RWP, RSTAGES, MINB>;
    fill_kernel<TIn><<<1184, 256>>>((TIn *)in, n);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM));
    int per = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, Geo::THREADS, Geo::SMEM));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int64_t G = (int64_t)per * sms;
    int64_t portion = round_bytes / (int64_t)sizeof(TIn) / G / Geo::SUB * Geo::SUB;
    if (portion < Geo::SUB) portion = Geo::SUB;
    RoundArgs a{};
    a.in = in; a.out = out; a.lo = 0; a.hi = n; a.portion = portion; a.lead_regions = getenv("LEAD") ? atoi(getenv("LEAD")) : 2; a.ramp = 0; a.l2_prefetch = getenv("PF") ? atoi(getenv("PF")) : 0;
    a.rounds = (n + portion * G - 1) / (portion * G); a.full_regions = a.rounds;
    a.desc = (ulonglong2 *)((char *)scratch + 256);
    uint64_t *tr; size_t tb = (size_t)a.rounds * G * 64;
    CK(cudaMalloc(&tr, tb)); CK(cudaMemset(tr, 0, tb));
    void *params[] = {&a};
    for (int w = 0; w < 3; ++w) { a.epoch = ++epoch; CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(Geo::THREADS), params, Geo::SMEM, 0)); }
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int it = 0; it < 10; ++it) {
            a.epoch = ++epoch;
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(Geo::THREADS), params, Geo::SMEM, 0));
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        // spot-check: input i%3 -> inclusive prefix known in closed form
        int bad = 0;
        for (int64_t i : {(int64_t)0, (int64_t)1, (int64_t)12345, n / 3, n / 2 + 7, n - 2, n - 1}) {
            TOut got; CK(cudaMemcpy(&got, (TOut *)out + i, sizeof(TOut), cudaMemcpyDeviceToHost));
            const int64_t m = i + 1, want = (m / 3) * 3 + (m % 3 == 2 ? 1 : 0);
            if ((double)got != (double)(TOut)want) ++bad;
        }
        printf("%s: best %.1f us  %.1f GB/s  check %s\n", name, best * 1e3,
               (double)n * (sizeof(TIn) + sizeof(TOut)) / (best * 1e-3) / 1e9, bad ? "FAIL" : "ok");
    }
#ifndef NO_TRACE
    CK(cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr)));
    uint64_t *tr2; size_t tb2 = (size_t)a.rounds * (portion / Geo::SUB) * (SW + 1) * 32;
    CK(cudaMalloc(&tr2, tb2)); CK(cudaMemset(tr2, 0, tb2));
    CK(cudaMemcpyToSymbol(g_trace2, &tr2, sizeof(tr2)));
    a.epoch = ++epoch;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(Geo::THREADS), params, Geo::SMEM, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    uint64_t *nul = nullptr; CK(cudaMemcpyToSymbol(g_trace, &nul, sizeof(nul)));
    std::vector<uint64_t> h(tb / 8); CK(cudaMemcpy(h.data(), tr, tb, cudaMemcpyDeviceToHost));
    char path[256]; snprintf(path, sizeof path, "gpurun_out/trace_rounds_%s.bin", name);
    FILE *f = fopen(path, "wb"); fwrite(h.data(), 8, h.size(), f); fclose(f);
    std::vector<uint64_t> h2(tb2 / 8); CK(cudaMemcpy(h2.data(), tr2, tb2, cudaMemcpyDeviceToHost));
    snprintf(path, sizeof path, "gpurun_out/trace_sub_%s.bin", name);
    f = fopen(path, "wb"); fwrite(h2.data(), 8, h2.size(), f); fclose(f);
    CK(cudaMemcpyToSymbol(g_trace2, &nul, sizeof(nul)));
    printf("%s: G=%lld per_sm=%d rounds=%lld portion=%lld  %.1f us  %.1f GB/s\n", name, (long long)G, per, (long long)a.rounds,
           (long long)portion, ms * 1e3, (double)n * (sizeof(TIn) + sizeof(TOut)) / (ms * 1e-3) / 1e9);
#endif
    cudaFree(tr);
}

int main() {
    void *in, *out, *scratch;
    CK(cudaMalloc(&in, 1ll << 32)); CK(cudaMalloc(&out, 1ll << 32)); CK(cudaMalloc(&scratch, 64 << 20));
    CK(cudaMemset(in, 0, 1ll << 32)); CK(cudaMemset(scratch, 0, 64 << 20));
    uint32_t epoch = 0;
    const int64_t N = 1ll << 28;
    // the shipped geometries (prefixscan_b200.cu RingSplit / region_bytes)
    run<float, float, 8, 4, 3, 4, 6>("f32_1cta", in, out, N, scratch, epoch, 24ll << 20);
    run<int64_t, int64_t, 8, 4, 5, 4, 3>("i64_1cta", in, out, N, scratch, epoch, 32ll << 20);
    run<int, int64_t, 8, 4, 5, 4, 3>("i32_1cta", in, out, N, scratch, epoch, 21ll << 20);
    return 0;
}
