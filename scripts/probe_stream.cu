// Probe: achievable HBM read bandwidth on this B200 for streaming a 4.3 GB
// bf16 [rows][128] matrix (the Qwen3-32B K cache) with (a) TMA 2-D tiles in
// an mbarrier ring (variants: stages, rows per box, CTAs per SM) and (b) plain
// 128-bit loads.  No compute: this is the ceiling the score kernel chases.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2510_07486_b200/csrc scripts/probe_stream.cu -o scripts/probe_stream_bin
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>

#include "tc.cuh"
using namespace asp::tc;

__global__ void tma_stream(const __grid_constant__ CUtensorMap map, long tiles, int rows_per_tile,
                           int stages, unsigned *sink) {
    extern __shared__ unsigned char sm[];
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    const uint32_t stage_bytes = rows_per_tile * 256;
    const uint32_t bar0 = base + stages * stage_bytes;
    const long start = tiles * blockIdx.x / gridDim.x, end = tiles * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; s++) { mbar_init(bar0 + 16 * s, 1); mbar_init(bar0 + 16 * s + 8, 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (long i = start; i < end; i++) {
            mbar_wait(bar0 + 16 * s + 8, ph ^ 1);
            mbar_arrive_expect_tx(bar0 + 16 * s, stage_bytes);
            for (int r = 0; r < 2; r++)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                    " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(base + s * stage_bytes + r * rows_per_tile * 128),
                    "l"(reinterpret_cast<uint64_t>(&map)), "r"(r * 64), "r"((int)(i * rows_per_tile)),
                    "r"(bar0 + 16 * s), "l"(kEvictFirst)
                    : "memory");
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        unsigned acc = 0;
        for (long i = start; i < end; i++) {
            mbar_wait(bar0 + 16 * s, ph);
            acc += *reinterpret_cast<volatile unsigned *>(sm + (base - smem_u32(sm)) + s * stage_bytes);
            mbar_arrive(bar0 + 16 * s + 8);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
        if (acc == 0x12345678u) *sink = acc;
    }
}

__global__ void ldg_stream(const uint4 *p, long n, unsigned *sink) {
    unsigned acc = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    const long rows = 64L * 8 * 32768;               // Qwen3-32B K cache rows
    const size_t bytes = rows * 256;
    void *buf;
    unsigned *sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    int cfgs[][3] = {{128, 6, 1}, {128, 4, 2}, {128, 3, 2}, {256, 3, 1}, {64, 12, 1}, {128, 6, 1},
                     {64, 6, 2}, {256, 2, 2}, {128, 8, 1}};
    for (auto &c : cfgs) {
        const int rpt = c[0], stages = c[1], cps = c[2];
        CUtensorMap map;
        cuuint64_t dims[2] = {128, (cuuint64_t)rows};
        cuuint64_t strides[1] = {256};
        cuuint32_t box[2] = {64, (cuuint32_t)rpt};
        cuuint32_t es[2] = {1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int smem = 1024 + stages * rpt * 256 + 16 * stages;
        const long tiles = rows / rpt;
        float best = 1e9;
        for (int rep = 0; rep < 4; rep++) {
            cudaEventRecord(e0);
            tma_stream<<<sms * cps, 64, smem>>>(map, tiles, rpt, stages, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) best = ms < best ? ms : best;
        }
        printf("TMA rows/tile=%3d stages=%2d ctas/sm=%d smem=%6d: %.1f us  %.0f GB/s  (%s)\n", rpt,
               stages, cps, smem, best * 1e3, bytes / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int bs : {256, 512, 1024}) {
        for (int waves : {1, 2, 4, 8}) {
            float best = 1e9;
            for (int rep = 0; rep < 4; rep++) {
                cudaEventRecord(e0);
                ldg_stream<<<sms * waves * (2048 / bs), bs>>>((const uint4 *)buf, bytes / 16, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) best = ms < best ? ms : best;
            }
            printf("LDG bs=%4d grid=%6d: %.1f us  %.0f GB/s\n", bs, sms * waves * (2048 / bs),
                   best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
