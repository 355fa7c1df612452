// Shared-memory wavefront cost of the producer access patterns (run under
// ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o smem_probe tools/smem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

// mode 0: LDS.64, 4 distinct addresses (lane & 3), 32 B stride (V pattern)
// mode 1: LDS.64, 8 distinct addresses (lane >> 2), odd row stride (U2 pattern)
// mode 2: LDS.128, 4 distinct addresses (lane & 3), contiguous 64 B
// mode 3: LDS.128, 8 distinct addresses (lane >> 2), contiguous 128 B
// mode 4: LDS.64, 1 address (warp-uniform)
// mode 5: LDS.64, 32 distinct contiguous
// mode 6: STS.U16, 16 distinct banks (producer split store)
// mode 7: LDS.128, 16 distinct addresses (lane >> 1), contiguous 256 B
// mode 8: LDS.64, 4 distinct (lane >> 3), 32 B stride;  mode 9: LDS.64, 8 distinct (lane & 7)
// mode 10: LDS.64, 2 distinct (lane & 1);  mode 11: LDS.128, 4 distinct (lane >> 3)
// mode 12: STS.U16 in the forward producer's swizzled A-stage pattern;  mode 13: LDS.64 by lane >> 4
// mode 14: STS.32 in the swizzled pattern;  mode 15: LDS.64, 4 distinct by (lane >> 2) & 3
// modes 16-19: a quad = 2 rows x 2 c lane mapping: V load, U2 load, A-stage STS.U16 at even / odd K
// mode 20: the current mapping's STS.U16 at odd K
template <int MODE>
__global__ void probe(float* out, int salt) {
    __shared__ __align__(16) float2 buf[4096];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = make_float2(float(i), float(i ^ salt));
    __syncthreads();
    float acc = 0.f;
    int off = 0;
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
        off = (off + 64 + salt) & 1023;
        if (MODE == 0) {
            const float2 v = buf[off + 4 * (lane & 3)];
            acc += v.x * v.y;
        } else if (MODE == 1) {
            const float2 v = buf[off + 9 * (lane >> 2)];
            acc += v.x * v.y;
        } else if (MODE == 2) {
            const float4 v = reinterpret_cast<const float4*>(buf)[(off >> 1) + (lane & 3)];
            acc += v.x * v.y + v.z * v.w;
        } else if (MODE == 3) {
            const float4 v = reinterpret_cast<const float4*>(buf)[(off >> 1) + (lane >> 2)];
            acc += v.x * v.y + v.z * v.w;
        } else if (MODE == 4) {
            const float2 v = buf[off];
            acc += v.x * v.y;
        } else if (MODE == 5) {
            const float2 v = buf[off + lane];
            acc += v.x * v.y;
        } else if (MODE == 6) {
            unsigned short* p = reinterpret_cast<unsigned short*>(buf) + 2 * off;
            p[(lane >> 2) * 16 + (lane & 3)] = static_cast<unsigned short>(it + lane);
        } else if (MODE == 8) {
            const float2 v = buf[off + 4 * (lane >> 3)];
            acc += v.x * v.y;
        } else if (MODE == 9) {
            const float2 v = buf[off + 9 * (lane & 7)];
            acc += v.x * v.y;
        } else if (MODE == 10) {
            const float2 v = buf[off + 4 * (lane & 1)];
            acc += v.x * v.y;
        } else if (MODE == 11) {
            const float4 v = reinterpret_cast<const float4*>(buf)[(off >> 1) + (lane >> 3)];
            acc += v.x * v.y + v.z * v.w;
        } else if (MODE == 12) {
            unsigned char* p = reinterpret_cast<unsigned char*>(buf) + 8 * off;
            const int row = lane >> 2;
            *reinterpret_cast<unsigned short*>(p + row * 32 + (((lane & 3) * 2) ^ ((row & 4) << 2))) =
                static_cast<unsigned short>(it + lane);
        } else if (MODE == 13) {
            const float2 v = buf[off + 4 * (lane >> 4)];
            acc += v.x * v.y;
        } else if (MODE == 14) {
            unsigned char* p = reinterpret_cast<unsigned char*>(buf) + 8 * off;
            const int row = lane >> 2;
            *reinterpret_cast<unsigned*>(p + row * 32 + (((lane & 3) * 4) ^ ((row & 4) << 2))) = unsigned(it + lane);
        } else if (MODE == 15) {
            const float2 v = buf[off + 4 * ((lane >> 2) & 3)];
            acc += v.x * v.y;
        } else if (MODE >= 16 && MODE <= 20) {
            // quad = 2 rows x 2 c: rowlane = 2 ((lane >> 2) & 3) + (lane & 1), hq = 2 (lane >> 4) + ((lane >> 1) & 1)
            const int rl = 2 * ((lane >> 2) & 3) + (lane & 1), hq = 2 * (lane >> 4) + ((lane >> 1) & 1);
            if (MODE == 16) {
                const float2 v = buf[off + 4 * hq];
                acc += v.x * v.y;
            } else if (MODE == 17) {
                const float2 v = buf[off + 9 * rl];
                acc += v.x * v.y;
            } else {
                unsigned char* p = reinterpret_cast<unsigned char*>(buf) + 8 * off;
                const int row = MODE == 20 ? (lane >> 2) : rl;
                const int K = (MODE == 20 ? (lane & 3) : hq) + (MODE == 18 ? 0 : 1);
                *reinterpret_cast<unsigned short*>(p + row * 32 + ((K * 2) ^ ((row & 4) << 2))) =
                    static_cast<unsigned short>(it + lane);
            }
        } else if (MODE == 7) {
            const float4 v = reinterpret_cast<const float4*>(buf)[(off >> 1) + (lane >> 1)];
            acc += v.x * v.y + v.z * v.w;
        }
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + buf[lane].x;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 128 * sizeof(float));
    probe<0><<<148, 128>>>(out, 0);
    probe<1><<<148, 128>>>(out, 0);
    probe<2><<<148, 128>>>(out, 0);
    probe<3><<<148, 128>>>(out, 0);
    probe<4><<<148, 128>>>(out, 0);
    probe<5><<<148, 128>>>(out, 0);
    probe<6><<<148, 128>>>(out, 0);
    probe<7><<<148, 128>>>(out, 0);
    probe<8><<<148, 128>>>(out, 0);
    probe<9><<<148, 128>>>(out, 0);
    probe<10><<<148, 128>>>(out, 0);
    probe<11><<<148, 128>>>(out, 0);
    probe<12><<<148, 128>>>(out, 0);
    probe<13><<<148, 128>>>(out, 0);
    probe<14><<<148, 128>>>(out, 0);
    probe<15><<<148, 128>>>(out, 0);
    probe<16><<<148, 128>>>(out, 0);
    probe<17><<<148, 128>>>(out, 0);
    probe<18><<<148, 128>>>(out, 0);
    probe<19><<<148, 128>>>(out, 0);
    probe<20><<<148, 128>>>(out, 0);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
