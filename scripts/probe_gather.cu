// Probe: achievable HBM throughput for gathering the decode step's selected
// 256-B K/V rows (config [2]: 64 x 8 rows of 32768 tokens, 2048 picked per row,
// ascending) with (a) LDG.128 into registers, (b) 1-D cp.async.bulk of whole
// rows into shared memory (mbarrier), (c) cp.async 16-B.  Reports GB/s of
// gathered bytes (K and V).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2510_07486_b200/csrc scripts/probe_gather.cu -o scripts/probe_gather_bin
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>

#include "tc.cuh"
using namespace asp::tc;

constexpr int ROWS = 64 * 8, L = 32768, K = 2048, D = 128;

__global__ void gather_ldg(const uint4 *kc, const uint4 *vc, const int *idx, unsigned *sink) {
    // one warp per 2 selected rows at a time (16 lanes x 16 B per row)
    unsigned acc = 0;
    const long total = (long)ROWS * K;
    const int lane = threadIdx.x & 31;
    for (long e = ((long)blockIdx.x * blockDim.x + threadIdx.x) / 16; e < total;
         e += (long)gridDim.x * blockDim.x / 16) {
        const int r = (int)(e / K);
        const long row = (long)r * L + idx[e];
        const uint4 a = __ldcs(kc + row * 16 + (lane & 15));
        const uint4 b = __ldcs(vc + row * 16 + (lane & 15));
        acc ^= a.x ^ a.y ^ b.z ^ b.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void gather_bulk(const char *kc, const char *vc, const int *idx, unsigned *sink, int stages) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    __shared__ uint64_t bars[16];
    if (threadIdx.x == 0) { for (int s = 0; s < stages; s++) mbar_init(smem_u32(&bars[s]), 1); fence_mbar_init(); }
    __syncthreads();
    const int per_tile = 128;                 // rows per stage per tensor
    const long total = (long)ROWS * K / per_tile;
    const long t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
    unsigned acc = 0;
    int s = 0;
    uint32_t ph = 0;
    for (long t = t0; t < t1; t++) {
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) mbar_arrive_expect_tx(smem_u32(&bars[s]), 2 * per_tile * 256);
            __syncwarp();
            for (int j = threadIdx.x; j < per_tile; j += 32) {
                const long e = t * per_tile + j;
                const int r = (int)(e / K);
                const long row = (long)r * L + idx[e];
                const uint32_t dk = base + s * 65536 + j * 256, dv = dk + 32768;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                             ::"r"(dk), "l"(kc + row * 256), "r"(smem_u32(&bars[s])) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                             ::"r"(dv), "l"(vc + row * 256), "r"(smem_u32(&bars[s])) : "memory");
            }
        }
        // consume the stage that is `stages-1` behind
        if (t - t0 >= stages - 1) {
            const int cs = (s + 1) % stages;
            const uint32_t cph = (cs <= s) ? ph : ph ^ 1;
            mbar_wait(smem_u32(&bars[cs]), cph);
            acc ^= *reinterpret_cast<volatile unsigned *>(sm + (base - smem_u32(sm)) + cs * 65536 + threadIdx.x * 4);
            __syncthreads();
        }
        if (++s == stages) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void gather_cpasync(const char *kc, const char *vc, const int *idx, unsigned *sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    const int per_tile = 128;
    const long total = (long)ROWS * K / per_tile;
    const long t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
    unsigned acc = 0;
    int s = 0;
    for (long t = t0; t < t1; t++) {
        for (int c = threadIdx.x; c < per_tile * 16; c += blockDim.x) {
            const int j = c / 16, ch = c % 16;
            const long e = t * per_tile + j;
            const int r = (int)(e / K);
            const long row = (long)r * L + idx[e];
            const uint32_t dk = base + s * 65536 + j * 256 + ch * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dk), "l"(kc + row * 256 + ch * 16) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dk + 32768), "l"(vc + row * 256 + ch * 16) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 2;" ::: "memory");
        if (++s == 3) s = 0;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    acc ^= *reinterpret_cast<volatile unsigned *>(sm + (base - smem_u32(sm)) + threadIdx.x * 4);
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    const size_t bytes = (size_t)ROWS * L * 256;
    char *kc, *vc;
    int *didx;
    unsigned *sink;
    cudaMalloc(&kc, bytes); cudaMalloc(&vc, bytes); cudaMalloc(&sink, 4);
    cudaMemset(kc, 1, bytes); cudaMemset(vc, 2, bytes);
    std::vector<int> idx((size_t)ROWS * K);
    srand(7);
    std::vector<int> perm(L);
    for (int r = 0; r < ROWS; r++) {
        for (int i = 0; i < L; i++) perm[i] = i;
        for (int i = 0; i < K; i++) std::swap(perm[i], perm[i + rand() % (L - i)]);
        std::sort(perm.begin(), perm.begin() + K);
        for (int i = 0; i < K; i++) idx[(size_t)r * K + i] = perm[i];
    }
    cudaMalloc(&didx, idx.size() * 4);
    cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double gbytes = 2.0 * ROWS * K * 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    char *junk; cudaMalloc(&junk, 512 << 20);
    auto timeit = [&](auto launch, const char *name) {
        float best = 1e9;
        for (int rep = 0; rep < 4; rep++) {
            cudaMemset(junk, rep, 512 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) best = ms < best ? ms : best;
        }
        printf("%-40s %8.1f us  %6.0f GB/s  (%s)\n", name, best * 1e3, gbytes / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int waves : {2, 4, 8, 16})
        timeit([&] { gather_ldg<<<sms * waves, 256>>>((const uint4 *)kc, (const uint4 *)vc, didx, sink); },
               waves == 2 ? "LDG.128 2 CTA/SM x256" : waves == 4 ? "LDG.128 4 CTA/SM x256" : waves == 8 ? "LDG.128 8 CTA/SM x256" : "LDG.128 16 CTA/SM x256");
    cudaFuncSetAttribute(gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int st : {2, 3})
        timeit([&] { gather_bulk<<<sms, 128, 1024 + st * 65536>>>(kc, vc, didx, sink, st); },
               st == 2 ? "cp.async.bulk 256B rows, 2x64KB stages" : "cp.async.bulk 256B rows, 3x64KB stages");
    cudaFuncSetAttribute(gather_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    timeit([&] { gather_cpasync<<<sms, 256, 1024 + 3 * 65536>>>(kc, vc, didx, sink); }, "cp.async 16B, 1 CTA/SM x256, 3 stages");
    timeit([&] { gather_cpasync<<<sms * 3, 256, 1024 + 3 * 65536 / 3>>>(kc, vc, didx, sink); }, "cp.async 16B (overlapping smem) 3 CTA/SM");
    return 0;
}
