// tcgen05.mma kind::f16 issue-rate probe: one CTA per SM, one thread issues
// back-to-back M=128 MMAs from shared memory with K-major operands in the
// SWIZZLE_32B layout (one 32-byte row per K16 step, what the forward /
// adjoint stages use) or the SWIZZLE_128B layout (128-byte rows, K16 slices
// at +32 B), N = 128 or 256.  Prints cycles per MMA and the implied dense
// fp16 TFLOP/s for the whole GPU at the measured clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2103_06393_b200/csrc/tm_sm100.cuh"

using namespace tmb::sm100;

constexpr int ITERS = 4096;

template <int SW, int N>
__global__ void __launch_bounds__(128, 1) rate(unsigned long long* cyc, int ka) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    unsigned char* sA = sm;              // 128 rows x 64 K fp16 = 16 KB
    unsigned char* sB = sm + 16384;      // 256 rows x 64 K fp16 = 32 KB
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 32768);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc(tslot, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_f16(128, N);
        uint64_t A[4], B[4];
        for (int k = 0; k < 4; ++k) {
            if (SW == 32) {
                A[k] = umma_smem_desc(smem_u32(sA + k * 4096), 256, 6);
                B[k] = umma_smem_desc(smem_u32(sB + k * 8192), 256, 6);
            } else {
                A[k] = umma_smem_desc(smem_u32(sA) + 32 * k, 1024, 2);
                B[k] = umma_smem_desc(smem_u32(sB) + 32 * k, 1024, 2);
            }
        }
        const long long t0 = clock64();
        for (int it = 0; it < ITERS; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_f16(tmem + (ka ? 0u : 256u * (k & 1)), A[k], B[k], idesc, 1);
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
        const long long t1 = clock64();
        cyc[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int SW, int N>
void run(unsigned long long* d, int ka) {
    const size_t smem = 1024 + 16384 + 32768 + 64;
    cudaFuncSetAttribute(rate<SW, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rate<SW, N><<<148, 128, smem>>>(d, ka);
    cudaEventRecord(e0);
    rate<SW, N><<<148, 128, smem>>>(d, ka);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += double(h[i]) / 148;
    const double nmma = double(ITERS) * 4;
    const double flops = 148.0 * nmma * 2.0 * 128 * N * 16;
    printf("SW%-3d N=%d acc=%s: %.1f clk/MMA (ideal %.1f), %.0f TFLOP/s (event %.3f ms), clock %.0f MHz\n", SW, N,
           ka ? "same" : "alt", avg / nmma, 128.0 * N * 16 / 4096.0, flops / (ms * 1e-3) / 1e12, ms,
           avg / (ms * 1e-3) / 1e6);
    printf("  err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * sizeof(unsigned long long));
    for (int rep = 0; rep < 2; ++rep) {
        run<32, 256>(d, 1);
        run<128, 256>(d, 1);
        run<32, 128>(d, 1);
        run<128, 128>(d, 1);
        run<32, 256>(d, 0);
        run<128, 256>(d, 0);
    }
    return 0;
}
