// synth.cu -- seeded synthetic INPUT generators for the BASELINE.json configs.
//
// Test / bench infrastructure shared by both sides of the parity tests: it
// holds none of the method's arithmetic (no stretch, no cap, no pdf), only the
// input recipes of DESIGN.md section 5.  Counter-based (Philox4x32-10), so any
// index range can be regenerated: sample i uses X = Philox(ctr (i_lo, i_hi, 0, 0),
// key (seed_lo, seed_hi)), Y = same with ctr.z = 1, u(w) = (w >> 8) 2^-24.
//
// recipe 0  fixed wi and alpha (params), u1 = u(Y0), u2 = u(Y1)
// recipe 1  config 1: wi uniform upper hemisphere, ax = ay = 0.5
// recipe 2  config 2: wi cosine-weighted, ax, ay log-uniform [0.01, 1]
// recipe 3  config 3: wi uniform upper hemisphere, ax, ay log-uniform [0.001, 1]
// recipe 5  config 5: path-tracer edge mix (grazing / back side / upper, alpha
//           from {1e-3, 0.05, 0.3, 1}, u = 0 and rim injections)
#include <cuda_runtime.h>
#include <cstdint>

namespace {

__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k.x, (uint32_t)p1,
                       (uint32_t)(p0 >> 32) ^ c.w ^ k.y, (uint32_t)p0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ float uf(uint32_t w) { return __uint2float_rn(w >> 8) * 0x1p-24f; }

__device__ __forceinline__ float log_uniform(float u, float lo_log2, float span_log2) {
    return exp2f(lo_log2 + u * span_log2);
}

struct Planes {
    float *wx, *wy, *wz, *ax, *ay, *u1, *u2;
};

__global__ void synth_kernel(int recipe, uint64_t seed, uint64_t first, int64_t n, Planes p,
                             float fx, float fy, float fz, float fax, float fay) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t i = first + (uint64_t)k;
        const uint4 X = philox(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0u, 0u), key);
        const uint4 Y = philox(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 1u, 0u), key);
        float wx = fx, wy = fy, wz = fz, ax = fax, ay = fay;
        float u1 = uf(Y.x), u2 = uf(Y.y);
        if (recipe != 0) {
            const float ua = uf(X.x);
            float sp, cp;
            sincospif(2.0f * uf(X.y), &sp, &cp);
            float z, r;
            if (recipe == 2) {            // cosine-weighted
                r = sqrtf(ua);
                z = sqrtf(1.0f - ua);
            } else if (recipe == 5) {     // edge mix
                const float v = uf(Y.z);
                if (v < 0.4f) z = 1e-4f + ua * (0.05f - 1e-4f);
                else if (v < 0.6f) z = -(1.0f - ua);
                else z = 1.0f - ua;
                r = sqrtf(fmaxf((1.0f - z) * (1.0f + z), 0.0f));
            } else {                      // uniform upper hemisphere
                z = 1.0f - ua;
                r = sqrtf(ua * (2.0f - ua));
            }
            wx = r * cp;
            wy = r * sp;
            wz = z;
            if (recipe == 1) {
                ax = ay = 0.5f;
            } else if (recipe == 2) {
                ax = log_uniform(uf(X.z), -6.64385618977f, 6.64385618977f);
                ay = log_uniform(uf(X.w), -6.64385618977f, 6.64385618977f);
            } else if (recipe == 3) {
                ax = log_uniform(uf(X.z), -9.96578428466f, 9.96578428466f);
                ay = log_uniform(uf(X.w), -9.96578428466f, 9.96578428466f);
            } else {
                const float T[4] = {1e-3f, 0.05f, 0.3f, 1.0f};
                ax = T[X.z >> 30];
                ay = T[X.w >> 30];
                const uint32_t b = Y.w;
                if ((b & 0x3Fu) == 0u) u1 = 0.0f;
                if (((b >> 6) & 0x3Fu) == 0u) u2 = 0.0f;
                if (((b >> 12) & 0x3Fu) == 0u) u2 = 1.0f - 0x1p-24f;
            }
        }
        p.wx[k] = wx; p.wy[k] = wy; p.wz[k] = wz;
        p.ax[k] = ax; p.ay[k] = ay;
        p.u1[k] = u1; p.u2[k] = u2;
    }
}

}  // namespace

extern "C" int synth_fill(int recipe, uint64_t seed, uint64_t first, int64_t n,
                          float* wx, float* wy, float* wz, float* ax, float* ay, float* u1, float* u2,
                          const float* fixed /* wi.xyz, ax, ay for recipe 0, else NULL */,
                          cudaStream_t stream) {
    if (n < 0) return 1;
    if (n == 0) return 0;
    if (!(recipe == 0 || recipe == 1 || recipe == 2 || recipe == 3 || recipe == 5)) return 1;
    if (recipe == 0 && !fixed) return 1;
    Planes p{wx, wy, wz, ax, ay, u1, u2};
    float f[5] = {0, 0, 1, 1, 1};
    if (fixed)
        for (int k = 0; k < 5; ++k) f[k] = fixed[k];
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = (n + 255) / 256;
    const int grid = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
    synth_kernel<<<grid, 256, 0, stream>>>(recipe, seed, first, n, p, f[0], f[1], f[2], f[3], f[4]);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
