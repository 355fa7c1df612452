// Test-only probe of the sm_100a building blocks used by the tensor-core
// kernels: thread-written SW32 K-major A tiles, TMA-loaded SW32 B tiles,
// tcgen05.mma kind::tf32 (M=128, N=256) with the negate-A bit, TMEM load.
// D[m][n] = sum_k A[m][k] B[n][k]; compared with a host fp64 product.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../../paper_2103_06393_b200/csrc/tm_sm100.cuh"
#include "../../paper_2103_06393_b200/csrc/tm_tmap.h"

using namespace tmb::sm100;

constexpr int M = 128, N = 256, K = 32, KS = 8, NST = K / KS;

__global__ void __launch_bounds__(192, 1) probe(const __grid_constant__ CUtensorMap bmap, const float* A, float* D,
                                                int negate) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = sm;                      // NST x (M x 32 B)
    unsigned char* sB = sm + NST * M * 32;       // NST x (N x 32 B)
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + NST * N * 32);
    uint64_t* done = full + NST;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1 + 4);
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
        if (elect_one()) {
            for (int s = 0; s < NST; ++s) {
                mbar_arrive_expect_tx(&full[s], N * 32);
                tma_load_3d(sB + s * N * 32, &bmap, &full[s], s * KS, 0, 0);
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            const uint32_t idesc = umma_idesc_tf32(M, N, negate != 0, false);
            for (int s = 0; s < NST; ++s) {
                mbar_wait(&full[s], 0);
                tc_fence_after();
                const uint64_t ad = umma_smem_desc(smem_u32(sA + s * M * 32), 256, 6);
                const uint64_t bd = umma_smem_desc(smem_u32(sB + s * N * 32), 256, 6);
                mma_tf32(tmem, ad, bd, idesc, s > 0);
            }
            mma_commit(done);
        }
        __syncwarp();
    } else {
        const int q = warp % 4;
        const int row = q * 32 + lane;
        for (int s = 0; s < NST; ++s) {
            for (int k = 0; k < KS; ++k)
                *reinterpret_cast<float*>(sA + s * M * 32 + sw_offset(row, k, 32)) = A[row * K + s * KS + k];
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        }
        mbar_wait(done, 0);
        tc_fence_after();
        for (int c = 0; c < N; c += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (uint32_t(q * 32) << 16) + c, v);
            tmem_ld_wait();
            for (int i = 0; i < 32; ++i) D[row * N + c + i] = __uint_as_float(v[i]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

static float tf32r(float x) {  // host round-to-nearest-even to tf32
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & ~0x1FFFu;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(7);
    for (auto& a : A) a = tf32r(float(rand()) / RAND_MAX - 0.5f);
    for (auto& b : B) b = tf32r(float(rand()) / RAND_MAX - 0.5f);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap bmap = tmb::make_tmap_3d_f32(dB, K, N, 1, K * 4, uint64_t(K) * N * 4, KS, N, CU_TENSOR_MAP_SWIZZLE_32B);
    const int smem = 1024 + NST * (M + N) * 32 + 256;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int bad = 0;
    for (int neg = 0; neg < 2; ++neg) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 192, smem>>>(bmap, dA, dD, neg);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("kernel error: %s\n", cudaGetErrorString(e));
            return 2;
        }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double num = 0, den = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * B[n * K + k];
                if (neg) s = -s;
                num += (D[m * N + n] - s) * (D[m * N + n] - s);
                den += s * s;
            }
        const double rel = std::sqrt(num / den);
        printf("umma_probe negate=%d rel_err=%.3e D[0]=%f D[last]=%f\n", neg, rel, D[0], D[M * N - 1]);
        if (!(rel < 1e-6)) bad = 1;
    }
    printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
    return bad;
}
