// Probe: tcgen05.mma with an MN-major (token-major) A operand in the 128-B
// swizzled canonical layout -- which descriptor field (LBO/SBO) is the
// MN-block stride.  Also probes TMA tile::gather4 into a SW128 tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include
//        -I paper_2510_07486_b200/csrc scripts/probe_mn_major.cu -o /tmp/probe -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#include "tc.cuh"
using namespace asp::tc;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}

// A: V tile [128 tok][128 d] bf16 global, token-major.  P: [16][128 tok].
__global__ void probe(const __nv_bfloat16 *V, const __nv_bfloat16 *P, float *out, int variant) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    unsigned char *g = sm + (base - smem_u32(sm));
    // A regions: r in {0,1}: d 64r..64r+63, [tok][128B] swizzled
    for (int c = threadIdx.x; c < 128 * 16; c += blockDim.x) {
        int tok = c / 16, ch = c % 16;            // 16 chunks of 8 d per token row (256 B)
        int r = ch / 8, cc = ch % 8;
        uint4 v = *reinterpret_cast<const uint4 *>(V + tok * 128 + ch * 8);
        *reinterpret_cast<uint4 *>(g + r * 16384 + tok * 128 + ((cc ^ (tok & 7)) * 16)) = v;
    }
    // B: P [16 n][128 tok] K-major: regions of 64 tok, [n][128B]
    unsigned char *gb = g + 32768;
    for (int c = threadIdx.x; c < 16 * 16; c += blockDim.x) {
        int n = c / 16, ch = c % 16;
        int r = ch / 8, cc = ch % 8;
        uint4 v = *reinterpret_cast<const uint4 *>(P + n * 128 + ch * 8);
        *reinterpret_cast<uint4 *>(gb + r * 2048 + n * 128 + ((cc ^ (n & 7)) * 16)) = v;
    }
    fence_proxy_async_smem();
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc<32>(smem_u32(&holder));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        uint32_t idesc = idesc_bf16_f32(128, 16) | (1u << 15);   // A MN-major
        for (int k = 0; k < 8; k++) {
            uint32_t lbo = variant == 0 ? 16384 : 1024, sbo = variant == 0 ? 1024 : 16384;
            uint64_t ad = desc_sw128(base + k * 2048, lbo, sbo);
            uint64_t bd = desc_sw128(base + 32768 + (k / 4) * 2048 + (k % 4) * 32, 16, 1024);
            mma_bf16(tmem, ad, bd, idesc, k > 0);
        }
        mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    int w = threadIdx.x / 32;
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(w * 32) << 16), r);
    tmem_wait_ld();
    for (int n = 0; n < 16; n++) out[(w * 32 + (threadIdx.x & 31)) * 16 + n] = __uint_as_float(r[n]);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<32>(tmem);
}

// gather4 probe: gather 128 rows (given indices) of a [rows][128] bf16 matrix into SW128 regions
__global__ void probe_gather(const __grid_constant__ CUtensorMap map, const int *idx,
                             __nv_bfloat16 *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    unsigned char *g = sm + (base - smem_u32(sm));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(smem_u32(&bar), 32768);
        for (int grp = 0; grp < 32; grp++)
            for (int r = 0; r < 2; r++) {
                uint32_t dst = base + r * 16384 + grp * 512;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                    "l"(reinterpret_cast<uint64_t>(&map)), "r"(r * 64), "r"(idx[grp * 4]),
                    "r"(idx[grp * 4 + 1]), "r"(idx[grp * 4 + 2]), "r"(idx[grp * 4 + 3]),
                    "r"(smem_u32(&bar))
                    : "memory");
            }
    }
    mbar_wait(smem_u32(&bar), 0);
    // un-swizzle back to [128][128]
    for (int c = threadIdx.x; c < 128 * 16; c += blockDim.x) {
        int tok = c / 16, ch = c % 16, r = ch / 8, cc = ch % 8;
        *reinterpret_cast<uint4 *>(out + tok * 128 + ch * 8) =
            *reinterpret_cast<uint4 *>(g + r * 16384 + tok * 128 + ((cc ^ (tok & 7)) * 16));
    }
}

int main() {
    std::vector<__nv_bfloat16> V(128 * 128), P(16 * 128);
    std::vector<float> Vf(128 * 128), Pf(16 * 128);
    srand(1);
    for (int i = 0; i < 128 * 128; i++) { Vf[i] = (rand() % 17 - 8) / 8.0f; V[i] = __float2bfloat16(Vf[i]); }
    for (int i = 0; i < 16 * 128; i++) { Pf[i] = (rand() % 9) / 16.0f; P[i] = __float2bfloat16(Pf[i]); }
    __nv_bfloat16 *dV, *dP; float *dO;
    cudaMalloc(&dV, V.size() * 2); cudaMalloc(&dP, P.size() * 2); cudaMalloc(&dO, 128 * 16 * 4);
    cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int variant = 0; variant < 2; variant++) {
        cudaMemset(dO, 0, 128 * 16 * 4);
        probe<<<1, 128, 64 * 1024>>>(dV, dP, dO, variant);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> O(128 * 16);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int d = 0; d < 128; d++)
            for (int n = 0; n < 16; n++) {
                double ref = 0;
                for (int t = 0; t < 128; t++) ref += (double)Vf[t * 128 + d] * Pf[n * 128 + t];
                maxerr = fmax(maxerr, fabs(ref - O[d * 16 + n]));
            }
        printf("MN-major variant %d (%s): err=%s max_abs_err=%g\n", variant,
               variant == 0 ? "LBO=MN-block 16K, SBO=1K" : "LBO=1K, SBO=16K", cudaGetErrorString(e),
               maxerr);
    }
    // gather4
    int rows = 1000;
    std::vector<__nv_bfloat16> M(rows * 128);
    for (int i = 0; i < rows * 128; i++) M[i] = __float2bfloat16((float)((i * 7) % 251));
    std::vector<int> idx(128);
    for (int i = 0; i < 128; i++) idx[i] = (i * 37 + 11) % rows;
    __nv_bfloat16 *dM, *dOut; int *dIdx;
    cudaMalloc(&dM, M.size() * 2); cudaMalloc(&dOut, 128 * 128 * 2); cudaMalloc(&dIdx, 128 * 4);
    cudaMemcpy(dM, M.data(), M.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dIdx, idx.data(), 128 * 4, cudaMemcpyHostToDevice);
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap map;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dM, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode gather map: %d\n", (int)r);
    cudaFuncSetAttribute(probe_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    probe_gather<<<1, 128, 40 * 1024>>>(map, dIdx, dOut);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<__nv_bfloat16> O(128 * 128);
    cudaMemcpy(O.data(), dOut, O.size() * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < 128; t++)
        for (int d = 0; d < 128; d++)
            if (__bfloat162float(O[t * 128 + d]) != __bfloat162float(M[idx[t] * 128 + d])) bad++;
    printf("gather4: err=%s mismatches=%d of %d\n", cudaGetErrorString(e), bad, 128 * 128);
    return 0;
}
