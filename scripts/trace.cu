// scripts/trace.cu -- per-tile timeline of scan_tiles_kernel (development tool).
// Writes gpurun_out/trace_<name>.bin: 8 uint64 per tile
//   [0] entry  [1] data in registers  [2] after the CTA barrier  [3] carry known
//   [4] stores issued  [5] (look-back windows << 32 | polls)  [6] SM id
#define PS_TRACE 1
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2312_14874_b200/csrc/scan_kernels.cuh"

using namespace ps;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename TIn, typename TOut, int WARPS, int ROWS>
void run(const char *name, void *in, void *out, int64_t n, void *scratch, uint32_t &epoch) {
    constexpr int64_t TILE = (int64_t)WARPS * ROWS * 32 * (32 / sizeof(TIn));
    ScanArgs a{};
    a.in = in; a.out = out; a.rows = 1; a.cols = n; a.ld_in = n; a.ld_out = n;
    a.tiles_per_row = (n + TILE - 1) / TILE; a.vec_ok = 1;
    a.desc.d = (ulonglong2 *)((char *)scratch + 256);
    const int64_t tiles = a.tiles_per_row;
    uint64_t *tr;
    CK(cudaMalloc(&tr, tiles * 64));
    CK(cudaMemset(tr, 0, tiles * 64));
    for (int w = 0; w < 3; ++w) { a.epoch = ++epoch; scan_tiles_kernel<TIn, TOut, WARPS, ROWS><<<(unsigned)tiles, WARPS * 32>>>(a); }
    CK(cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr)));
    a.epoch = ++epoch;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    scan_tiles_kernel<TIn, TOut, WARPS, ROWS><<<(unsigned)tiles, WARPS * 32>>>(a);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    uint64_t *nul = nullptr;
    CK(cudaMemcpyToSymbol(g_trace, &nul, sizeof(nul)));
    std::vector<uint64_t> h(tiles * 8);
    CK(cudaMemcpy(h.data(), tr, tiles * 64, cudaMemcpyDeviceToHost));
    char path[256];
    snprintf(path, sizeof path, "gpurun_out/trace_%s.bin", name);
    FILE *f = fopen(path, "wb");
    fwrite(h.data(), 8, h.size(), f);
    fclose(f);
    printf("%s: %lld tiles, %.1f us traced launch\n", name, (long long)tiles, ms * 1e3);
    cudaFree(tr);
}

int main() {
    const int64_t bytes = 1ll << 31;
    void *in, *out, *scratch;
    CK(cudaMalloc(&in, bytes)); CK(cudaMalloc(&out, bytes)); CK(cudaMalloc(&scratch, 64 << 20));
    CK(cudaMemset(in, 0, bytes)); CK(cudaMemset(scratch, 0, 64 << 20));
    uint32_t epoch = 0;
    run<float, float, 8, 8>("f32_w8r8", in, out, 1ll << 28, scratch, epoch);
    run<float, float, 8, 4>("f32_w8r4", in, out, 1ll << 28, scratch, epoch);
    run<int64_t, int64_t, 8, 8>("i64cfg1_w8r8", in, out, 1ll << 24, scratch, epoch);
    return 0;
}
