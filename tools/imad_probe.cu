// imad_probe.cu -- issue cost of the Philox multiply on sm_100a, by form:
// IMAD.WIDE.U32 with the multiplier as an immediate (what ptxas emits for the
// Philox constants) or in a register, alone and in a full round (+ 2 LOP3),
// and a round next to 4 independent FFMAs.  Clocks per warp-unit per SM
// sub-partition (32 warps/SM, 8 independent chains per thread), as
// tools/mix_probe.cu.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/imad_probe tools/imad_probe.cu
//   /tmp/imad_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 128;

// MODE 0: 2 IMAD.WIDE (imm) per unit; 1: 2 IMAD.WIDE (reg multiplier);
// 2: round (imm); 3: round (reg multiplier); 4: round (imm) + 4 FFMA;
// 5: round (reg) + 4 FFMA
template <int MODE>
__global__ void __launch_bounds__(1024, 1) probe(uint32_t seed, uint32_t m0, uint32_t m1, long long* cycles,
                                                 uint32_t* sink) {
    uint32_t x[kChains], y[kChains], z[kChains], v[kChains];
    float f[kChains][4];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        x[c] = seed * (threadIdx.x + 1) + c;
        y[c] = x[c] * 3u;
        z[c] = x[c] ^ 0x55u;
        v[c] = x[c] + 9u;
#pragma unroll
        for (int k = 0; k < 4; ++k) f[c][k] = 1.0f + 1e-3f * (float)(x[c] + k);
    }
    const bool reg = (MODE == 1 || MODE == 3 || MODE == 5);
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            uint64_t p0, p1;
            if (reg) {
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p0) : "r"(x[c]), "r"(m0));
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p1) : "r"(z[c]), "r"(m1));
            } else {
                asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(p0) : "r"(x[c]));
                asm volatile("mul.wide.u32 %0, %1, 0xCD9E8D57;" : "=l"(p1) : "r"(z[c]));
            }
            if (MODE <= 1) {
                x[c] = (uint32_t)(p0 >> 32) + (uint32_t)p1;
                z[c] = (uint32_t)(p1 >> 32) + (uint32_t)p0;
            } else {
                uint32_t nx, nz;
                asm volatile("lop3.b32 %0, %1, %2, 0x9E3779B9, 0x96;" : "=r"(nx) : "r"((uint32_t)(p1 >> 32)), "r"(y[c]));
                asm volatile("lop3.b32 %0, %1, %2, 0xBB67AE85, 0x96;" : "=r"(nz) : "r"((uint32_t)(p0 >> 32)), "r"(v[c]));
                y[c] = (uint32_t)p1;
                v[c] = (uint32_t)p0;
                x[c] = nx;
                z[c] = nz;
            }
            if (MODE >= 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, %1;" : "+f"(f[c][k]) : "f"(f[c][(k + 1) % 4]));
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c)
        acc ^= x[c] ^ y[c] ^ z[c] ^ v[c] ^ __float_as_uint(f[c][0] + f[c][1] + f[c][2] + f[c][3]);
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
double clocks_per_unit(int sms, long long* cyc, uint32_t* sink) {
    probe<MODE><<<sms, 1024>>>(7u, 0xD2511F53u, 0xCD9E8D57u, cyc, sink);
    probe<MODE><<<sms, 1024>>>(7u, 0xD2511F53u, 0xCD9E8D57u, cyc, sink);
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int b = 0; b < sms; ++b) mx = cyc[b] > mx ? cyc[b] : mx;
    return (double)mx / (32.0 * kIters * kChains / 4.0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc;
    uint32_t* sink;
    cudaMallocManaged(&cyc, sms * sizeof(long long));
    cudaMallocManaged(&sink, 4);
    printf("clocks per warp-unit per SMSP\n");
    printf("  2 IMAD.WIDE (imm) + 2 IADD        %.2f\n", clocks_per_unit<0>(sms, cyc, sink));
    printf("  2 IMAD.WIDE (reg) + 2 IADD        %.2f\n", clocks_per_unit<1>(sms, cyc, sink));
    printf("  round, multiplier imm             %.2f\n", clocks_per_unit<2>(sms, cyc, sink));
    printf("  round, multiplier reg             %.2f\n", clocks_per_unit<3>(sms, cyc, sink));
    printf("  round (imm) + 4 FFMA              %.2f\n", clocks_per_unit<4>(sms, cyc, sink));
    printf("  round (reg) + 4 FFMA              %.2f\n", clocks_per_unit<5>(sms, cyc, sink));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
