// Probe: issue rate / cost of back-to-back tcgen05.mma kind::f16 (M = 128,
// cta_group::1) for several N, A and B from 128-B-swizzled K-major smem, one
// CTA per SM, one issuing thread.  Prints cycles per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2510_07486_b200/csrc scripts/probe_mma_rate.cu -o scripts/probe_mma_bin
#include <cuda.h>
#include <stdio.h>

#include "tc.cuh"
using namespace asp::tc;

__device__ __forceinline__ void mma_bf16_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int N, int M>
__global__ void mma_rate(int iters, int chains, unsigned long long *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(sm + (base - smem_u32(sm)))[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&holder));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x < 32) {                      // whole warp, elect.sync inside the asm
        constexpr uint32_t idesc = idesc_bf16_f32(M, N);
        const long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            for (int kk = 0; kk < 8; kk++)
                for (int c = 0; c < chains; c++) {
                    const int r = kk / 4, ko = (kk % 4) * 32;
                    mma_bf16_warp(tmem + c * N, desc_sw128_kmajor(base + r * 16384 + ko),
                                  desc_sw128_kmajor(base + 32768 + r * (N * 128) + ko), idesc, kk > 0);
                }
        }
        if (threadIdx.x == 0) mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        const long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, int M = 128>
void run(int chains, unsigned long long *d_out) {
    const int iters = 200;
    cudaFuncSetAttribute(mma_rate<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    mma_rate<N, M><<<148, 128, 100 * 1024>>>(iters, chains, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long cyc;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    const double per = (double)cyc / (iters * 8.0 * chains);
    printf("M=%3d N=%3d chains=%d: %.1f cycles/MMA  (%.1f cycles per 128x16 A slice-step) %s\n", M, N, chains,
           per, per, cudaGetErrorString(e));
}

int main() {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    for (int chains : {1, 2, 3, 4, 6, 8, 12}) run<32>(chains, d);
    for (int chains : {1, 3, 6}) run<32, 64>(chains, d);
    for (int chains : {1, 2}) run<256>(chains, d);
    return 0;
}
