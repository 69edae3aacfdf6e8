// pipe_probe.cu -- measured issue rates of the instruction types the fused
// kernels are made of, on sm_100a: warp-instructions per clock per SMSP with
// 32 warps per SM and 8 independent dependency chains per thread.  Grounds the
// instruction-issue roofline of the compute-bound kernels (DESIGN.md s.6.4).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu
//   /tmp/pipe_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 256;

#define BODY_U32(...)                                                        \
    _Pragma("unroll 16") for (int it = 0; it < kIters; ++it) {               \
        _Pragma("unroll") for (int c = 0; c < kChains; ++c) { __VA_ARGS__; } \
    }

template <int OP>
__global__ void __launch_bounds__(1024, 1) probe(uint32_t seed, long long* cycles, uint32_t* sink) {
    uint32_t x[kChains];
    float f[kChains];
    double d[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        x[c] = seed * (threadIdx.x + 1) + c;
        f[c] = 1.0f + 1e-3f * (float)x[c];
        d[c] = 1.0 + 1e-3 * (double)x[c];
    }
    __syncthreads();
    const long long t0 = clock64();
    if (OP == 0) {  // FFMA, register operands
        BODY_U32(asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c + 1) % kChains]), "f"(f[(c + 2) % kChains])))
    } else if (OP == 1) {  // IMAD (mad.lo.u32, register operands)
        BODY_U32(asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(x[(c + 1) % kChains]), "r"(x[(c + 2) % kChains])))
    } else if (OP == 2) {  // IMAD.WIDE.U32 + the 64-bit add ptxas splits off (IADD3 + IADD3.X)
        uint64_t w[kChains];
#pragma unroll
        for (int c = 0; c < kChains; ++c) w[c] = x[c];
        BODY_U32(asm volatile("mad.wide.u32 %0, %1, 0xD2511F53, %0;" : "+l"(w[c]) : "r"((uint32_t)w[c])))
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32);
    } else if (OP == 12) {  // one Philox4x32 round on 2 independent counters per chain pair:
        // 2 IMAD.WIDE.U32 (immediate) + 2 LOP3 (3-input, constant key) per counter
        uint32_t y[kChains], z[kChains], v[kChains];
#pragma unroll
        for (int c = 0; c < kChains; ++c) { y[c] = x[c] * 3u; z[c] = x[c] ^ 0x55u; v[c] = x[c] + 9u; }
        BODY_U32({
            uint64_t p0, p1;
            asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(p0) : "r"(x[c]));
            asm volatile("mul.wide.u32 %0, %1, 0xCD9E8D57;" : "=l"(p1) : "r"(z[c]));
            uint32_t nx, nz;
            asm volatile("lop3.b32 %0, %1, %2, 0x9E3779B9, 0x96;" : "=r"(nx) : "r"((uint32_t)(p1 >> 32)), "r"(y[c]));
            asm volatile("lop3.b32 %0, %1, %2, 0xBB67AE85, 0x96;" : "=r"(nz) : "r"((uint32_t)(p0 >> 32)), "r"(v[c]));
            y[c] = (uint32_t)p1; v[c] = (uint32_t)p0; x[c] = nx; z[c] = nz;
        })
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] ^= y[c] ^ z[c] ^ v[c];
    } else if (OP == 8) {  // FFMA with an immediate operand
        BODY_U32(asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, %1;" : "+f"(f[c]) : "f"(f[(c + 1) % kChains])))
    } else if (OP == 9) {  // LOP3 with a constant operand (Philox key xor)
        BODY_U32(asm volatile("lop3.b32 %0, %0, %1, 0x9E3779B9, 0x96;" : "+r"(x[c]) : "r"(x[(c + 1) % kChains])))
    } else if (OP == 10) {  // MUFU.RSQ
        BODY_U32(asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f[c])))
    } else if (OP == 11) {  // I2FP.F32.U32
        BODY_U32({ float t; asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(t) : "r"(x[c])); x[c] = __float_as_uint(t) >> 3; })
    } else if (OP == 3) {  // LOP3 (3-input xor, Philox key mixing)
        BODY_U32(asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(x[(c + 1) % kChains]), "r"(x[(c + 3) % kChains])))
    } else if (OP == 4) {  // MUFU.EX2
        BODY_U32(asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[c])))
    } else if (OP == 5) {  // DFMA
        BODY_U32(asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(d[(c + 1) % kChains]), "d"(d[(c + 2) % kChains])))
    } else if (OP == 6) {  // IADD3 (add.u32, register operands)
        BODY_U32(asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(x[(c + 1) % kChains])))
    } else if (OP == 7) {  // FMUL
        BODY_U32(asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(f[c]) : "f"(f[(c + 1) % kChains])))
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= x[c] ^ __float_as_uint(f[c]) ^ (uint32_t)__double_as_longlong(d[c]);
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
double rate(int sms, long long* cyc, uint32_t* sink) {
    probe<OP><<<sms, 1024>>>(7u, cyc, sink);  // warm
    probe<OP><<<sms, 1024>>>(7u, cyc, sink);
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int b = 0; b < sms; ++b) mx = cyc[b] > mx ? cyc[b] : mx;
    const double warp_inst_per_sm = 32.0 * kIters * kChains;  // 32 warps per SM (one 1024-thread block)
    return warp_inst_per_sm / (double)mx / 4.0;                // per SMSP per clock
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc;
    uint32_t* sink;
    cudaMallocManaged(&cyc, sms * sizeof(long long));
    cudaMallocManaged(&sink, 4);
    printf("warp-instructions per clock per SMSP (32 warps/SM, 8 chains/thread):\n");
    printf("  FFMA          %.3f\n", rate<0>(sms, cyc, sink));
    printf("  FMUL          %.3f\n", rate<7>(sms, cyc, sink));
    printf("  IMAD          %.3f\n", rate<1>(sms, cyc, sink));
    printf("  IMAD.WIDE+2 IADD3 %.3f (per triple)\n", rate<2>(sms, cyc, sink));
    printf("  LOP3          %.3f\n", rate<3>(sms, cyc, sink));
    printf("  IADD3         %.3f\n", rate<6>(sms, cyc, sink));
    printf("  FFMA imm      %.3f\n", rate<8>(sms, cyc, sink));
    printf("  LOP3 const    %.3f\n", rate<9>(sms, cyc, sink));
    printf("  MUFU.RSQ      %.3f\n", rate<10>(sms, cyc, sink));
    printf("  I2FP+SHF pair %.3f (per pair)\n", rate<11>(sms, cyc, sink));
    printf("  Philox round  %.3f (rounds per clock per SMSP; 2 IMAD.WIDE + 2 LOP3 each)\n", rate<12>(sms, cyc, sink));
    printf("  MUFU.EX2      %.3f\n", rate<4>(sms, cyc, sink));
    printf("  DFMA          %.3f\n", rate<5>(sms, cyc, sink));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
