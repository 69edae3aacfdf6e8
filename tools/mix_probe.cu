// mix_probe.cu -- how the fused kernel's two instruction streams share an SM
// sub-partition on sm_100a: Philox4x32 rounds (IMAD.WIDE.U32 + LOP3) and fp32
// FFMA chains, alone, interleaved in one thread, and split across warps.
// Reports clocks per "unit" per SMSP (32 warps per SM, 8 independent chains
// per thread), a unit being one Philox round plus K FFMAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix_probe tools/mix_probe.cu
//   /tmp/mix_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 128;

__device__ __forceinline__ void round(uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& v) {
    uint64_t p0, p1;
    asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(p0) : "r"(x));
    asm volatile("mul.wide.u32 %0, %1, 0xCD9E8D57;" : "=l"(p1) : "r"(z));
    uint32_t nx, nz;
    asm volatile("lop3.b32 %0, %1, %2, 0x9E3779B9, 0x96;" : "=r"(nx) : "r"((uint32_t)(p1 >> 32)), "r"(y));
    asm volatile("lop3.b32 %0, %1, %2, 0xBB67AE85, 0x96;" : "=r"(nz) : "r"((uint32_t)(p0 >> 32)), "r"(v));
    y = (uint32_t)p1;
    v = (uint32_t)p0;
    x = nx;
    z = nz;
}

__device__ __forceinline__ void round_hilo(uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& v) {
    uint32_t h0, l0, h1, l1;
    asm volatile("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(h0) : "r"(x));
    asm volatile("mul.lo.u32 %0, %1, 0xD2511F53;" : "=r"(l0) : "r"(x));
    asm volatile("mul.hi.u32 %0, %1, 0xCD9E8D57;" : "=r"(h1) : "r"(z));
    asm volatile("mul.lo.u32 %0, %1, 0xCD9E8D57;" : "=r"(l1) : "r"(z));
    uint32_t nx, nz;
    asm volatile("lop3.b32 %0, %1, %2, 0x9E3779B9, 0x96;" : "=r"(nx) : "r"(h1), "r"(y));
    asm volatile("lop3.b32 %0, %1, %2, 0xBB67AE85, 0x96;" : "=r"(nz) : "r"(h0), "r"(v));
    y = l1;
    v = l0;
    x = nx;
    z = nz;
}

// MODE 0: rounds only; 1: K FFMAs only; 2: round + K FFMAs in every thread;
// 3: even warps rounds (x2), odd warps 2K FFMAs (the same total work as 2);
// 4: rounds as IMAD.HI + IMAD pairs; 5: FMULs only (K per unit)
template <int MODE, int K>
__global__ void __launch_bounds__(1024, 1) probe(uint32_t seed, long long* cycles, uint32_t* sink) {
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
    const bool even = ((threadIdx.x >> 5) & 1) == 0;
    __syncthreads();
    const long long t0 = clock64();
    if (MODE == 3) {
        if (even) {
#pragma unroll 4
            for (int it = 0; it < kIters; ++it)
#pragma unroll
                for (int c = 0; c < kChains; ++c) {
                    round(x[c], y[c], z[c], v[c]);
                    round(x[c], y[c], z[c], v[c]);
                }
        } else {
#pragma unroll 4
            for (int it = 0; it < kIters; ++it)
#pragma unroll
                for (int c = 0; c < kChains; ++c)
#pragma unroll
                    for (int k = 0; k < 2 * K; ++k)
                        asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, %1;" : "+f"(f[c][k % 4]) : "f"(f[c][(k + 1) % 4]));
        }
    }
#pragma unroll 4
    for (int it = 0; it < (MODE == 3 ? 0 : kIters); ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (MODE == 0 || MODE == 2) round(x[c], y[c], z[c], v[c]);
            if (MODE == 1 || MODE == 2) {
#pragma unroll
                for (int k = 0; k < K; ++k)
                    asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, %1;" : "+f"(f[c][k % 4]) : "f"(f[c][(k + 1) % 4]));
            }
            if (MODE == 4) round_hilo(x[c], y[c], z[c], v[c]);
            if (MODE >= 6) {  // a round plus K instructions of one other type, same warp
                round(x[c], y[c], z[c], v[c]);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (MODE == 6) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(f[c][k % 4]) : "f"(f[c][(k + 1) % 4]));
                    if (MODE == 7) asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, %1;" : "+f"(f[c][k % 4]) : "f"(f[c][(k + 1) % 4]));
                    if (MODE == 8) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f[c][k % 4]));
                    if (MODE == 9) asm volatile("lop3.b32 %0, %0, %1, 0x1234567, 0x96;" : "+r"(v[c]) : "r"(y[c]));
                    if (MODE == 10) {
                        uint32_t t = __float_as_uint(f[c][k % 4]);
                        asm volatile("add.u32 %0, %0, %1;" : "+r"(t) : "r"(x[c]));
                        f[c][k % 4] = __uint_as_float(t);
                    }
                    if (MODE == 11) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c][k % 4]) : "f"(f[c][(k + 1) % 4]), "f"(f[c][(k + 2) % 4]));
                }
            }
            if (MODE == 5) {
#pragma unroll
                for (int k = 0; k < K; ++k)
                    asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(f[c][k % 4]) : "f"(f[c][(k + 1) % 4]));
            }
        }
    }
    __syncthreads();  // the unit ends when every warp of the block is done
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c)
        acc ^= x[c] ^ y[c] ^ z[c] ^ v[c] ^ __float_as_uint(f[c][0] + f[c][1] + f[c][2] + f[c][3]);
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE, int K>
double clocks_per_unit(int sms, long long* cyc, uint32_t* sink) {
    probe<MODE, K><<<sms, 1024>>>(7u, cyc, sink);
    probe<MODE, K><<<sms, 1024>>>(7u, cyc, sink);
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int b = 0; b < sms; ++b) mx = cyc[b] > mx ? cyc[b] : mx;
    const double units_per_smsp = 32.0 * kIters * kChains / 4.0;  // per warp-unit
    return (double)mx / units_per_smsp;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc;
    uint32_t* sink;
    cudaMallocManaged(&cyc, sms * sizeof(long long));
    cudaMallocManaged(&sink, 4);
    printf("clocks per warp-unit per SMSP (unit = 1 Philox round [2 IMAD.WIDE + 2 LOP3] and/or K FFMA)\n");
    printf("  round only                 %.2f\n", clocks_per_unit<0, 0>(sms, cyc, sink));
    printf("  4 FFMA only                %.2f\n", clocks_per_unit<1, 4>(sms, cyc, sink));
    printf("  8 FFMA only                %.2f\n", clocks_per_unit<1, 8>(sms, cyc, sink));
    printf("  round + 2 FFMA, same warp  %.2f\n", clocks_per_unit<2, 2>(sms, cyc, sink));
    printf("  round + 4 FFMA, same warp  %.2f\n", clocks_per_unit<2, 4>(sms, cyc, sink));
    printf("  round + 8 FFMA, same warp  %.2f\n", clocks_per_unit<2, 8>(sms, cyc, sink));
    printf("  round | 2 FFMA, split warps %.2f\n", clocks_per_unit<3, 2>(sms, cyc, sink));
    printf("  round | 4 FFMA, split warps %.2f\n", clocks_per_unit<3, 4>(sms, cyc, sink));
    printf("  round | 8 FFMA, split warps %.2f\n", clocks_per_unit<3, 8>(sms, cyc, sink));
    printf("  round as IMAD.HI + IMAD     %.2f\n", clocks_per_unit<4, 0>(sms, cyc, sink));
    printf("  4 FMUL only                %.2f\n", clocks_per_unit<5, 4>(sms, cyc, sink));
    printf("  round + 4 FMUL             %.2f\n", clocks_per_unit<6, 4>(sms, cyc, sink));
    printf("  round + 4 FFMA (immediate) %.2f\n", clocks_per_unit<7, 4>(sms, cyc, sink));
    printf("  round + 4 FFMA (3 regs)    %.2f\n", clocks_per_unit<11, 4>(sms, cyc, sink));
    printf("  round + 2 MUFU.RSQ         %.2f\n", clocks_per_unit<8, 2>(sms, cyc, sink));
    printf("  round + 4 LOP3             %.2f\n", clocks_per_unit<9, 4>(sms, cyc, sink));
    printf("  round + 4 IADD3            %.2f\n", clocks_per_unit<10, 4>(sms, cyc, sink));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
