// scripts/sm_fairness.cu -- are some SMs slower at streaming HBM than others? (dev tool)
// One CTA per SM copies 32 KiB tiles (TMA bulk load -> shared -> 256-bit STG) through a
// 6-deep ring.  static: CTA c owns tiles c, c+G, ... (the stream kernel's layout);
// dynamic: CTAs take tiles from a global atomic ticket.  Per-CTA finish times and SM ids
// show whether fixed equal shares leave the grid waiting for a few slow SMs.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../paper_2312_14874_b200/csrc/rounds_kernel.cuh"
using namespace ps;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int S = 6, B = 32768, INFL = 2;

__global__ void __launch_bounds__(288, 1) copy_ring(const char *in, char *out, int64_t ntiles, int dynamic,
                                                    unsigned long long *ticket, uint64_t *fin) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)S * B);
    uint64_t *empty = full + S;
    int64_t *tile_of = reinterpret_cast<int64_t *>(empty + S);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int G = gridDim.x;
    if (warp == 8) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int64_t next = dynamic ? (int64_t)atomicAdd(ticket, 1ull) : blockIdx.x;
            for (int64_t k = 0;; ++k) {
                const int st = (int)(k % S);
                const int64_t t = next;
                if (k >= S) mbar_wait(&empty[st], (uint32_t)(((k / S) - 1) & 1));
                if (k >= INFL) mbar_wait(&full[(k - INFL) % S], (uint32_t)(((k - INFL) / S) & 1));
                tile_of[st] = t < ntiles ? t : -1;
                if (t >= ntiles) { mbar_arrive(&full[st]); break; }
                next = dynamic ? (int64_t)atomicAdd(ticket, 1ull) : t + G;  // prefetch the next ticket
                mbar_expect_tx(&full[st], B);
                bulk_g2s(sm + (size_t)st * B, in + t * B, B / 2, &full[st], pol);
                bulk_g2s(sm + (size_t)st * B + B / 2, in + t * B + B / 2, B / 2, &full[st], pol);
            }
        }
        return;
    }
    const uint64_t pol = policy_evict_first();
    for (int64_t k = 0;; ++k) {
        const int st = (int)(k % S);
        mbar_wait(&full[st], (uint32_t)((k / S) & 1));
        const int64_t t = *(volatile int64_t *)&tile_of[st];
        if (t < 0) break;
        const char *sb = reinterpret_cast<const char *>(sm) + (size_t)st * B;
        for (int o = (warp * 32 + lane) * 32; o < B; o += 8 * 32 * 32) stg256_policy(out + t * B + o, lds256(sb + o), pol);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    __syncwarp();
    if (warp == 0 && lane == 0) {
        uint32_t smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        fin[blockIdx.x * 2] = t; fin[blockIdx.x * 2 + 1] = smid;
    }
}

int main() {
    const int64_t n = 1ll << 30;
    const int64_t ntiles = n / B;
    char *in, *out; unsigned long long *ticket; uint64_t *fin;
    CK(cudaMalloc(&in, n)); CK(cudaMalloc(&out, n)); CK(cudaMalloc(&ticket, 8)); CK(cudaMalloc(&fin, 4096 * 8));
    CK(cudaMemset(in, 1, n));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int smem = S * B + 2 * S * 8 + S * 8;
    CK(cudaFuncSetAttribute(copy_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep)
    for (int dyn = 0; dyn < 2; ++dyn) {
        float best = 1e30f;
        std::vector<uint64_t> h(sms * 2);
        for (int it = 0; it < 6; ++it) {
            CK(cudaMemset(ticket, 0, 8));
            cudaEventRecord(e0);
            copy_ring<<<sms, 288, smem>>>(in, out, ntiles, dyn, ticket, fin);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 1 && ms < best) { best = ms; CK(cudaMemcpy(h.data(), fin, sms * 16, cudaMemcpyDeviceToHost)); }
        }
        std::vector<uint64_t> f(sms);
        for (int i = 0; i < sms; ++i) f[i] = h[2 * i];
        const uint64_t mn = *std::min_element(f.begin(), f.end());
        std::vector<std::pair<uint64_t, int>> byf;
        for (int i = 0; i < sms; ++i) byf.push_back({f[i] - mn, (int)h[2 * i + 1]});
        std::sort(byf.begin(), byf.end());
        printf("%s: %.1f us  %.0f GB/s  finish spread (ns): p50 %llu p90 %llu max %llu  slowest SMs:", dyn ? "dynamic" : "static ",
               best * 1e3, 2.0 * n / (best * 1e-3) / 1e9, (unsigned long long)byf[sms / 2].first,
               (unsigned long long)byf[sms * 9 / 10].first, (unsigned long long)byf[sms - 1].first);
        for (int i = sms - 8; i < sms; ++i) printf(" %d", byf[i].second);
        printf("\n");
    }
    return 0;
}
