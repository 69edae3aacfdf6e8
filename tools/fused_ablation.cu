// fused_ablation.cu -- where the fused config-4 kernel's time goes: the same
// loop shape as philox_kernel<cap, pdf, 8> (256-thread blocks, persistent grid
// of occupancy x SMs, 8 samples per thread, four 256-bit output stores) with
// parts of the per-sample work removed.
//   A  Philox words only (two blocks, six words -> four floats)
//   B  Philox + config-4 input generation (c4_inputs_fp32)
//   C  the product: Philox + inputs + cap_fp32 + pdf + flag
//   D  inputs from a cheap integer hash (3 IMAD + shifts) instead of Philox:
//      the float part of C alone
//   E  words from the hash, C's float part, Philox of an unrelated counter
//      XORed into one output (C's work with the Philox rounds decoupled)
// Not product code: includes the library's device header for the arithmetic.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/abl tools/fused_ablation.cu
//   /tmp/abl
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2306_05044_b200/csrc/vndf_device.cuh"

using namespace vndf;

__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

__device__ __forceinline__ uint4 hash4(uint64_t i) {
    const uint32_t a = (uint32_t)i * 0x9E3779B9u, b = (uint32_t)i * 0x85EBCA6Bu, c = (uint32_t)i * 0xC2B2AE35u;
    return make_uint4(a ^ (b >> 15), b ^ (c >> 13), c ^ (a >> 16), a + b);
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) abl(uint64_t n, float* hx, float* hy, float* hz, float* pd,
                                              unsigned* flags_out, const __grid_constant__ PhiloxKeys ks) {
    const uint64_t nch = n / 8;
    unsigned fl = 0;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = c * 8;
        float ox[8], oy[8], oz[8], op[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t ctr = base | (uint64_t)j;
            uint4 X, Y;
            if (MODE == 0 || MODE == 1 || MODE == 2) {
                philox_pair_ks(ks, ctr, X, Y);
            } else {
                X = hash4(ctr);
                Y = hash4(ctr ^ 0x5555u);
            }
            if (MODE == 0) {
                ox[j] = __uint_as_float(X.x ^ Y.x);
                oy[j] = __uint_as_float(X.y ^ Y.y);
                oz[j] = __uint_as_float(X.z);
                op[j] = __uint_as_float(X.w);
                continue;
            }
            const Inputs in = c4_inputs_fp32(X, Y);
            if (MODE == 1) {
                ox[j] = in.wx + in.ax;
                oy[j] = in.wy + in.ay;
                oz[j] = in.wz + in.v1;
                op[j] = in.u2 + in.q;
                continue;
            }
            Sample o;
            fl |= (unsigned)cap_fp32<true, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, o);
            ox[j] = o.x;
            oy[j] = o.y;
            oz[j] = o.z;
            op[j] = o.pdf;
            if (MODE == 4) {
                uint4 P, Q;
                philox_pair_ks(ks, ctr + 0x100000000ull, P, Q);
                op[j] = __uint_as_float(__float_as_uint(op[j]) ^ (P.x ^ P.y ^ P.z ^ P.w ^ Q.x ^ Q.y));
            }
        }
        st8(hx + base, ox);
        st8(hy + base, oy);
        st8(hz + base, oz);
        st8(pd + base, op);
    }
    if (fl == 0x7fffffffu) flags_out[0] = fl;
}

template <int MODE>
void run(const char* name, uint64_t n, float* o[4], unsigned* f, const PhiloxKeys& ks) {
    int occ = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, abl<MODE>, 256, 0);
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, abl<MODE>);
    const int grid = sms * occ;
    for (int k = 0; k < 3; ++k) abl<MODE><<<grid, 256>>>(n, o[0], o[1], o[2], o[3], f, ks);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int k = 0; k < 10; ++k) abl<MODE><<<grid, 256>>>(n, o[0], o[1], o[2], o[3], f, ks);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    // clocks per warp of 32 samples per SM sub-partition at 1965 MHz
    const double cyc = ms * 1e-3 * 1965e6 * sms * 4 / (n / 32.0);
    printf("  %-44s %7.2f Gsamples/s  %6.1f SMSP-clk per warp-sample  (%d regs, %d blocks/SM)\n", name,
           n / (ms * 1e6), cyc, at.numRegs, occ);
}

int main() {
    const uint64_t n = 1ull << 28;
    float* o[4];
    for (auto& p : o) cudaMalloc(&p, n * sizeof(float));
    unsigned* f;
    cudaMalloc(&f, 4);
    PhiloxKeys ks;
    uint32_t k0 = 3, k1 = 0;
    for (int r = 0; r < 10; ++r) {
        ks.k0[r] = k0;
        ks.k1[r] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    printf("fused config-4 kernel ablation, 2^28 samples, 8 per thread, 256-thread blocks:\n");
    run<0>("A Philox words only", n, o, f, ks);
    run<1>("B Philox + input generation", n, o, f, ks);
    run<2>("C Philox + inputs + cap + pdf (product)", n, o, f, ks);
    run<3>("D hash + inputs + cap + pdf (float part)", n, o, f, ks);
    run<4>("E D + Philox of another counter", n, o, f, ks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
