// fix_latency.cu -- dependent latency (clock cycles, one thread) of the float64
// fix-up of a flagged sample and of the double-precision primitives it is made
// of: what a latency-bound launch (config 1) pays per flagged sample.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fixlat tools/fix_latency.cu
//   /tmp/fixlat
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2306_05044_b200/csrc/vndf_device.cuh"

using namespace vndf;

constexpr int kReps = 64;

template <int OP>
__global__ void lat(const double* in, double* out, long long* cyc) {
    double x = in[threadIdx.x], y = in[threadIdx.x + 1];
    float fx = (float)x;
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < kReps; ++r) {
        if (OP == 0) x = rsqrt(x + 1.0) ;
        if (OP == 1) x = sqrt(x + 1.0);
        if (OP == 2) { double s, c; sincospi(x, &s, &c); x = s + c; }
        if (OP == 3) x = y / (x + 1.0);
        if (OP == 4) x = fma(x, y, 0.5);
        if (OP == 5) {
            const float4 f = cap_fp64_d(x, 0.3, 0.2, 0.5, 0.4, 0.25, 0.999);
            x = 0.1 + 1e-3 * (double)(f.x + f.y + f.z + f.w);
        }
        if (OP == 6) {  // the fp32 sampler, for scale
            Sample o;
            cap_fp32<true>(fx, 0.3f, 0.2f, 0.5f, 0.4f, -0.25f, 0.999f, 0.001f, o);
            fx = 0.1f + 1e-3f * (o.x + o.y + o.z + o.pdf);
        }
    }
    const long long t1 = clock64();
    out[threadIdx.x] = x + fx;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// First (cold instruction cache) vs second call of the out-of-line recomputation
// the streamed kernels make (cap_fp64), one thread of a fresh launch.
__global__ void cold_warm(const double* in, double* out, long long* cyc) {
    float x = (float)in[threadIdx.x];
    long long t[3];
    t[0] = clock64();
    const float4 a = cap_fp64(x, 0.3f, 0.2f, 0.5f, 0.4f, 0.25f, 0.999f);
    x = 0.1f + 1e-3f * (a.x + a.y + a.z + a.w);
    t[1] = clock64();
    const float4 b = cap_fp64(x, 0.3f, 0.2f, 0.5f, 0.4f, 0.25f, 0.999f);
    x = 0.1f + 1e-3f * (b.x + b.y + b.z + b.w);
    t[2] = clock64();
    out[threadIdx.x] = x;
    cyc[0] = t[1] - t[0];
    cyc[1] = t[2] - t[1];
}

template <int OP>
void run(const char* name, const double* in, double* out, long long* cyc) {
    lat<OP><<<1, 1>>>(in, out, cyc);
    lat<OP><<<1, 1>>>(in, out, cyc);
    cudaDeviceSynchronize();
    printf("  %-40s %8.1f clk\n", name, (double)cyc[0] / kReps);
}

int main() {
    double *in, *out;
    long long* cyc;
    cudaMallocManaged(&in, 64 * sizeof(double));
    cudaMallocManaged(&out, 64 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    for (int i = 0; i < 64; ++i) in[i] = 0.3 + 0.01 * i;
    printf("dependent latency per call, one thread (clock64), sm_100a:\n");
    run<4>("DFMA", in, out, cyc);
    run<0>("rsqrt(double) (+ DADD)", in, out, cyc);
    run<1>("sqrt(double) (+ DADD)", in, out, cyc);
    run<2>("sincospi(double) (+ DADD)", in, out, cyc);
    run<3>("division (double) (+ DADD)", in, out, cyc);
    run<5>("cap_fp64_d (the fix-up arithmetic)", in, out, cyc);
    run<6>("cap_fp32 + pdf (the fp32 sampler)", in, out, cyc);
    cudaMallocManaged(&cyc, 2 * sizeof(long long));
    cold_warm<<<1, 1>>>(in, out, cyc);
    cudaDeviceSynchronize();
    printf("  %-40s %8lld clk (first call, cold) / %lld clk (second)\n", "cap_fp64 out of line", cyc[0], cyc[1]);
    return 0;
}
