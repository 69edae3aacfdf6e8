// vndf.cu -- libvndf: sm_100a kernels and the C ABI declared in include/vndf.h.
//
// Citations: "P:n" = PAPER.md line n (arXiv 2306.05044).
// describes each kernel, its roofline and its algorithmic bytes per sample.
//
// Kernels
//   stream_kernel<METHOD, PDF, V>   streamed SoA sampling (cap or Heitz), V
//                                   samples per thread per step loaded with
//                                   one V*32-bit vector load per plane
//                                   (V = 8: LDG.E.256 / STG.E.256 on sm_100a),
//                                   persistent grid-stride loop, inline float64
//                                   fix-up of flagged cap samples.
//   philox_kernel<METHOD, PDF, V>   fused Philox4x32-10 input generation +
//                                   sampling + pdf, stores only.
//   philox_words_kernel             raw Philox words (bit-exactness audit).
//   count_*_kernel                  diagnostics: how many samples get fixed up.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>
#include <cmath>

#include "vndf_device.cuh"
#include "../../include/vndf.h"

using namespace vndf;

namespace {

// kCapNative: the paper's native below-horizon handling (NEXT-3, no flip)
enum Method { kCap = 0, kHeitz = 1, kCapNative = 2 };

struct StreamArgs {
    const float* wx;
    const float* wy;
    const float* wz;
    const float* ax;
    const float* ay;
    const float* u1;
    const float* u2;
    float* hx;
    float* hy;
    float* hz;
    float* pdf;
};

// ---------------------------------------------------------------- memory ops
// Streaming loads: read-only path, no L1 allocation (each byte is read once).
template <int V>
struct Vec {
    float v[V];
};

template <int V>
__device__ __forceinline__ Vec<V> ld_stream(const float* p);

template <>
__device__ __forceinline__ Vec<1> ld_stream<1>(const float* p) {
    Vec<1> r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r.v[0]) : "l"(p));
    return r;
}
template <>
__device__ __forceinline__ Vec<2> ld_stream<2>(const float* p) {
    Vec<2> r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.v[0]), "=f"(r.v[1]) : "l"(p));
    return r;
}
template <>
__device__ __forceinline__ Vec<4> ld_stream<4>(const float* p) {
    Vec<4> r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                 : "l"(p));
    return r;
}
template <>
__device__ __forceinline__ Vec<8> ld_stream<8>(const float* p) {
    Vec<8> r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]),
                   "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}

template <int V>
__device__ __forceinline__ void st_stream(float* p, const Vec<V>& r);

template <>
__device__ __forceinline__ void st_stream<1>(float* p, const Vec<1>& r) {
    asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(r.v[0]) : "memory");
}
template <>
__device__ __forceinline__ void st_stream<2>(float* p, const Vec<2>& r) {
    asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]) : "memory");
}
template <>
__device__ __forceinline__ void st_stream<4>(float* p, const Vec<4>& r) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
                 "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3])
                 : "memory");
}
template <>
__device__ __forceinline__ void st_stream<8>(float* p, const Vec<8>& r) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]),
                 "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}

// ------------------------------------------- programmatic dependent launch --
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------ TMA bulk copy into shared memory --
// One elected thread arms an mbarrier with the expected byte count and issues
// cp.async.bulk (global -> shared, SASS UBLKCP); every thread waits on the
// barrier's phase 0.  `bytes` must be a multiple of 16, both addresses 16-byte
// aligned.
__device__ __forceinline__ void bulk_load_shared(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                                 uint64_t* bar) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(d), "l"(gmem_src), "r"(bytes), "r"(b)
                     : "memory");
    }
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(b)
            : "memory");
    }
}

// ------------------------------------------------------------ one sample --
// fp32 sample; returns the conditioning flag (always false for Heitz).
template <int METHOD, bool PDF>
__device__ __forceinline__ bool sample_one(float wx, float wy, float wz, float ax, float ay, float u1,
                                           float u2, Sample& o) {
    const float v1 = u1 - 0.5f;  // exact for u1 on the 2^-24 grid and for u1 >= 1/4
    if (METHOD == kCap) return cap_fp32<PDF>(wx, wy, wz, ax, ay, v1, u2, 1.0f - u2, o);
    if (METHOD == kCapNative) return cap_fp32<PDF, kFrameNative>(wx, wy, wz, ax, ay, v1, u2, 1.0f - u2, o);
    heitz_fp32<PDF>(wx, wy, wz, ax, ay, v1, u2, o);
    return false;
}

__device__ __forceinline__ void fix_one(const StreamArgs& a, bool pdf, int64_t i, bool flip) {
    cap_fix_stream(a.wx, a.wy, a.wz, a.ax, a.ay, a.u1, a.u2, a.hx, a.hy, a.hz, pdf ? a.pdf : nullptr, i, flip);
}

// ------------------------------------------------------- streamed kernel --
// Chunk c covers samples [c V, c V + V).  Full chunks go through the vector
// path (one chunk per thread by default, grid-stride if the grid is capped);
// the n mod V tail is done by the first threads of the grid with scalar
// accesses.  Flagged samples are pushed to a block-level shared-memory queue
// and recomputed in float64 after a block barrier, one per thread, so a
// block's few fix-ups (~3.5 per 1024 samples in config 5) run side by side
// instead of serialising their warps; the vector loop itself stays call-free.
// A queue overflow (only possible with a capped, grid-stride grid) falls back
// to fixing in the thread that found it.
constexpr int kBlockFixCap = 512;

#ifndef VNDF_STREAM_MINB
#define VNDF_STREAM_MINB 1
#endif

template <int METHOD, bool PDF, int V>
__global__ void __launch_bounds__(256, VNDF_STREAM_MINB) stream_kernel(StreamArgs a, int64_t n) {
    __shared__ int64_t fix_idx[METHOD != kHeitz ? kBlockFixCap : 1];
    __shared__ int fix_count;
    if (METHOD != kHeitz && threadIdx.x == 0) fix_count = 0;
    // Programmatic dependent launch: let the next kernel on the stream be
    // scheduled once every block of this grid is running, and wait for the
    // previous grid (its completion and memory flush) before touching memory.
    pdl_launch_dependents();
    pdl_wait();
    if (METHOD != kHeitz) __syncthreads();
    auto defer = [&](int64_t i) {
        const int slot = atomicAdd(&fix_count, 1);
        if (slot < kBlockFixCap) fix_idx[slot] = i;
        else fix_one(a, PDF, i, METHOD == kCap);
    };
    const int64_t nchunks = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t c = tid; c < nchunks; c += stride) {
        const int64_t i = c * V;
        const Vec<V> wx = ld_stream<V>(a.wx + i), wy = ld_stream<V>(a.wy + i),
                     wz = ld_stream<V>(a.wz + i), ax = ld_stream<V>(a.ax + i),
                     ay = ld_stream<V>(a.ay + i), u1 = ld_stream<V>(a.u1 + i),
                     u2 = ld_stream<V>(a.u2 + i);
        Vec<V> hx, hy, hz, pd;
        unsigned flags = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            Sample o;
            const bool f = sample_one<METHOD, PDF>(wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j],
                                                   u1.v[j], u2.v[j], o);
            flags |= (unsigned)f << j;
            hx.v[j] = o.x;
            hy.v[j] = o.y;
            hz.v[j] = o.z;
            pd.v[j] = o.pdf;
        }
        st_stream<V>(a.hx + i, hx);
        st_stream<V>(a.hy + i, hy);
        st_stream<V>(a.hz + i, hz);
        if (PDF) st_stream<V>(a.pdf + i, pd);
        if (METHOD != kHeitz && __builtin_expect(flags != 0, 0)) {
            do {
                const int j = __ffs(flags) - 1;
                flags &= flags - 1;
                defer(i + j);
            } while (flags);
        }
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            Sample o;
            const bool f = sample_one<METHOD, PDF>(a.wx[i], a.wy[i], a.wz[i], a.ax[i], a.ay[i],
                                                   a.u1[i], a.u2[i], o);
            a.hx[i] = o.x;
            a.hy[i] = o.y;
            a.hz[i] = o.z;
            if (PDF) a.pdf[i] = o.pdf;
            if (METHOD != kHeitz && f) defer(i);
        }
    }
    if (METHOD != kHeitz) {
        __syncthreads();
        const int m = min(fix_count, kBlockFixCap);
        for (int t = threadIdx.x; t < m; t += blockDim.x) fix_one(a, PDF, fix_idx[t], METHOD == kCap);
    }
}

// ----------------------------------------------------- fused Philox kernel --
// Deferred float64 fix-up queue of the fused kernel (compute-bound: inline
// fp64 work would diverge the warp and its call would inflate the register
// allocation).  Flagged local indices are appended with one (warp-aggregated)
// atomic each (~0.4% of samples); a second kernel recomputes them with all
// lanes busy.  If the queue overflowed (count > cap), the fix-up kernel
// rescans every sample's flag instead: always correct, slower only then.
struct FixQueue {
    unsigned long long* count;
    uint64_t* idx;
    uint64_t cap;
};

template <int METHOD, bool PDF>
__device__ __forceinline__ Sample philox_one(uint64_t seed, uint64_t first, uint64_t k,
                                             const FixQueue& fq, const float2* __restrict__ tab) {
    const Inputs in = c4_inputs_fp32(philox_sample(seed, first + k), tab);
    Sample o;
    if (METHOD == kCap) {
        // config-4 inputs are on the upper hemisphere (wi.z = 1 - u > 0): no flip
        const bool flag = cap_fp32<PDF, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.v1, in.u2, in.q, o);
        if (__builtin_expect(flag, 0)) {
            const unsigned long long slot = atomicAdd(fq.count, 1ull);
            if (slot < fq.cap) fq.idx[slot] = k;
        }
    } else {
        heitz_fp32<PDF, false>(in.wx, in.wy, in.wz, in.ax, in.ay, in.v1, in.u2, o);
    }
    return o;
}

__global__ void __launch_bounds__(128) philox_fixup_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                            FixQueue fq, const float2* __restrict__ gtab,
                                                            float* __restrict__ hx,
                                                            float* __restrict__ hy, float* __restrict__ hz,
                                                            float* __restrict__ pdf) {
    const uint64_t count = *fq.count;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (count <= fq.cap) {
        for (uint64_t t = t0; t < count; t += stride) {
            const uint64_t k = fq.idx[t];
            const float4 f = cap_philox_fp64(seed, first + k);
            hx[k] = f.x;
            hy[k] = f.y;
            hz[k] = f.z;
            if (pdf) pdf[k] = f.w;
        }
        return;
    }
    for (uint64_t k = t0; k < (uint64_t)n; k += stride) {  // overflow: rescan
        const Inputs in = c4_inputs_fp32(philox_sample(seed, first + k), gtab);
        Sample o;
        if (cap_fp32<true, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.v1, in.u2, in.q, o)) {
            const float4 f = cap_philox_fp64(seed, first + k);
            hx[k] = f.x;
            hy[k] = f.y;
            hz[k] = f.z;
            if (pdf) pdf[k] = f.w;
        }
    }
}

#ifndef VNDF_PHILOX_MINB
#define VNDF_PHILOX_MINB 1
#endif
#ifndef VNDF_PHILOX_V
#define VNDF_PHILOX_V 4
#endif

template <int METHOD, bool PDF, int V>
__global__ void __launch_bounds__(256, VNDF_PHILOX_MINB) philox_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                     float* __restrict__ hxp, float* __restrict__ hyp,
                                                     float* __restrict__ hzp, float* __restrict__ pdfp,
                                                     FixQueue fq, const float2* __restrict__ gtab) {
    // Stage the 64 KB sin/cos table of the incidence azimuth in shared memory
    // with one TMA bulk copy (cp.async.bulk, completion on an mbarrier).
    extern __shared__ __align__(16) float2 tab[];
    __shared__ __align__(8) uint64_t tab_bar;
    bulk_load_shared(tab, gtab, kSinCosTableEntries * sizeof(float2), &tab_bar);
    const int64_t nchunks = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t c = tid; c < nchunks; c += stride) {
        const int64_t i = c * V;
        Vec<V> hx, hy, hz, pd;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const Sample o = philox_one<METHOD, PDF>(seed, first, (uint64_t)(i + j), fq, tab);
            hx.v[j] = o.x;
            hy.v[j] = o.y;
            hz.v[j] = o.z;
            pd.v[j] = o.pdf;
        }
        st_stream<V>(hxp + i, hx);
        st_stream<V>(hyp + i, hy);
        st_stream<V>(hzp + i, hz);
        if (PDF) st_stream<V>(pdfp + i, pd);
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            const Sample o = philox_one<METHOD, PDF>(seed, first, (uint64_t)i, fq, tab);
            hxp[i] = o.x;
            hyp[i] = o.y;
            hzp[i] = o.z;
            if (PDF) pdfp[i] = o.pdf;
        }
    }
}

__global__ void __launch_bounds__(256) philox_words_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                           uint32_t block, uint4* __restrict__ out) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t i = first + (uint64_t)k;
        out[k] = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), block, 0u), key);
    }
}

// ------------------------------------------------------------ diagnostics --
__device__ __forceinline__ void warp_count(bool flag, unsigned long long* count) {
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(count, (unsigned long long)__popc(m));
}

__global__ void __launch_bounds__(256) count_stream_kernel(StreamArgs a, int64_t n,
                                                           unsigned long long* count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rounds = (n + stride - 1) / stride;  // uniform trip count for the ballot
    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t i = start + r * stride;
        bool flag = false;
        if (i < n) {
            Sample o;
            const float u2 = a.u2[i];
            flag = cap_fp32<true>(a.wx[i], a.wy[i], a.wz[i], a.ax[i], a.ay[i], a.u1[i] - 0.5f, u2,
                                  1.0f - u2, o);
        }
        warp_count(flag, count);
    }
}

__global__ void __launch_bounds__(256) count_philox_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                           const float2* __restrict__ gtab,
                                                           unsigned long long* count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rounds = (n + stride - 1) / stride;
    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t i = start + r * stride;
        bool flag = false;
        if (i < n) {
            const Inputs in = c4_inputs_fp32(philox_sample(seed, first + (uint64_t)i), gtab);
            Sample o;
            flag = cap_fp32<true, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.v1, in.u2, in.q, o);
        }
        warp_count(flag, count);
    }
}

// ------------------------------------------------- NEXT-4: standalone pdf --
struct PdfArgs {
    const float* hx;
    const float* hy;
    const float* hz;
    const float* wx;
    const float* wy;
    const float* wz;
    const float* ax;
    const float* ay;
    float* pdf;
};

// 32 B in (h, wi, alpha), 4 B out per sample; HBM-bound.
template <int V>
__global__ void __launch_bounds__(256) pdf_kernel(PdfArgs a, int64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t nchunks = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t c = tid; c < nchunks; c += stride) {
        const int64_t i = c * V;
        const Vec<V> hx = ld_stream<V>(a.hx + i), hy = ld_stream<V>(a.hy + i), hz = ld_stream<V>(a.hz + i),
                     wx = ld_stream<V>(a.wx + i), wy = ld_stream<V>(a.wy + i), wz = ld_stream<V>(a.wz + i),
                     ax = ld_stream<V>(a.ax + i), ay = ld_stream<V>(a.ay + i);
        Vec<V> pd;
#pragma unroll
        for (int j = 0; j < V; ++j)
            pd.v[j] = vndf_pdf_fp32(hx.v[j], hy.v[j], hz.v[j], wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j]);
        st_stream<V>(a.pdf + i, pd);
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) a.pdf[i] = vndf_pdf_fp32(a.hx[i], a.hy[i], a.hz[i], a.wx[i], a.wy[i], a.wz[i], a.ax[i], a.ay[i]);
    }
}

// ------------------------------------------ NEXT-2: reflection sampling --
struct ReflectArgs {
    const float* wx;
    const float* wy;
    const float* wz;
    const float* ax;
    const float* ay;
    const float* u1;
    const float* u2;
    float* ox;
    float* oy;
    float* oz;
    float* pdf;
    float* weight;
};

// Streamed: 28 B in, 20 B out per sample (wo.xyz, pdf Eq. 20, weight G2/G1).
template <int V>
__global__ void __launch_bounds__(256) reflect_kernel(ReflectArgs a, int64_t n) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t nchunks = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t c = tid; c < nchunks; c += stride) {
        const int64_t i = c * V;
        const Vec<V> wx = ld_stream<V>(a.wx + i), wy = ld_stream<V>(a.wy + i),
                     wz = ld_stream<V>(a.wz + i), ax = ld_stream<V>(a.ax + i),
                     ay = ld_stream<V>(a.ay + i), u1 = ld_stream<V>(a.u1 + i),
                     u2 = ld_stream<V>(a.u2 + i);
        Vec<V> ox, oy, oz, pd, wt;
        unsigned flags = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            Reflected r;
            const bool f = cap_reflect_fp32(wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j], u1.v[j] - 0.5f,
                                            u2.v[j], 1.0f - u2.v[j], r);
            flags |= (unsigned)f << j;
            ox.v[j] = r.x;
            oy.v[j] = r.y;
            oz.v[j] = r.z;
            pd.v[j] = r.pdf;
            wt.v[j] = r.weight;
        }
        st_stream<V>(a.ox + i, ox);
        st_stream<V>(a.oy + i, oy);
        st_stream<V>(a.oz + i, oz);
        st_stream<V>(a.pdf + i, pd);
        st_stream<V>(a.weight + i, wt);
        while (__builtin_expect(flags != 0, 0)) {
            const int j = __ffs(flags) - 1;
            flags &= flags - 1;
            cap_reflect_fix_stream(a.wx, a.wy, a.wz, a.ax, a.ay, a.u1, a.u2, a.ox, a.oy, a.oz, a.pdf,
                                   a.weight, i + j);
        }
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            Reflected r;
            const float u2 = a.u2[i];
            const bool f = cap_reflect_fp32(a.wx[i], a.wy[i], a.wz[i], a.ax[i], a.ay[i], a.u1[i] - 0.5f, u2,
                                            1.0f - u2, r);
            a.ox[i] = r.x;
            a.oy[i] = r.y;
            a.oz[i] = r.z;
            a.pdf[i] = r.pdf;
            a.weight[i] = r.weight;
            if (f)
                cap_reflect_fix_stream(a.wx, a.wy, a.wz, a.ax, a.ay, a.u1, a.u2, a.ox, a.oy, a.oz, a.pdf,
                                       a.weight, i);
        }
    }
}

// White-furnace estimator, Eq. 19 with L = 1: for a fixed (wa, alpha), sample j
// (u1 = u(W0), u2 = u(W1) of Philox block (counter j, key seed)) contributes
// its weight f_r |cos| / PDF = G2/G1.  Per-thread float64 sums, fixed-order
// block reduction, per-block partials; a one-block pass adds the partials in
// block order (deterministic for a given grid).
template <int METHOD>
__global__ void __launch_bounds__(256) furnace_kernel(float wx, float wy, float wz, float ax, float ay,
                                                      uint64_t seed, uint64_t first, int64_t n,
                                                      double* __restrict__ partials) {
    double s1 = 0.0, s2 = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const uint4 W = philox_sample(seed, first + (uint64_t)j);
        const float v1 = fmaf(fw(W.x), 0x1p-24f, -0.5f);
        const float f2 = fw(W.y);
        Reflected r;
        if (METHOD == kCap) {
            if (cap_reflect_fp32(wx, wy, wz, ax, ay, v1, f2 * 0x1p-24f, fmaf(f2, -0x1p-24f, 1.0f), r)) {
                r.weight = cap_reflect_weight_fp64(wx, wy, wz, ax, ay, u01d(W.x), u01d(W.y));
            }
        } else {
            heitz_reflect_fp32(wx, wy, wz, ax, ay, v1, f2 * 0x1p-24f, r);
        }
        s1 += r.weight;
        s2 += (double)r.weight * r.weight;
    }
    __shared__ double sh1[8], sh2[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_down_sync(0xffffffffu, s1, o);
        s2 += __shfl_down_sync(0xffffffffu, s2, o);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sh1[warp] = s1;
        sh2[warp] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a1 = 0.0, a2 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a1 += sh1[w];
            a2 += sh2[w];
        }
        partials[2 * blockIdx.x] = a1;
        partials[2 * blockIdx.x + 1] = a2;
    }
}

__global__ void __launch_bounds__(256) furnace_finish_kernel(const double* __restrict__ partials, int blocks,
                                                            double* out) {
    // fixed-order reduction (deterministic for a given grid): strided partial
    // sums per thread, then a shared-memory tree
    __shared__ double r1[256], r2[256];
    double a1 = 0.0, a2 = 0.0;
    for (int b = threadIdx.x; b < blocks; b += blockDim.x) {
        a1 += partials[2 * b];
        a2 += partials[2 * b + 1];
    }
    r1[threadIdx.x] = a1;
    r2[threadIdx.x] = a2;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            r1[threadIdx.x] += r1[threadIdx.x + w];
            r2[threadIdx.x] += r2[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = r1[0];
        out[1] = r2[0];
    }
}

// ------------------------------------ NEXT-3: GPU histograms for chi-square --
// Samples a fixed (wi, alpha) n times (u1 = u(W0), u2 = u(W1) of Philox block
// (counter j, key seed)) and bins, in shared memory, either
//   mode 0: h in (theta in [0, pi/2), phi in [0, 2 pi))  (compare with Eq. 1 masses)
//   mode 1: the std-space reflected direction c = reflect(ws, normalize(M^T h'))
//           in (u_z = (c.z + ws.z)/(1 + ws.z), phi_c / 2 pi): uniform by Eq. 10.
// METHOD: kCap / kHeitz (reading R4 frame) or kCapNative.  Cap samples flagged
// by the conditioning test are recomputed in float64 first, as in the product
// kernels.  Counts are ADDED to counts[nt * nphi] (uint64).
template <int METHOD>
__global__ void __launch_bounds__(256) histogram_kernel(int mode, float wx, float wy, float wz, float ax,
                                                        float ay, uint64_t seed, uint64_t first, int64_t n,
                                                        int nt, int nphi, unsigned long long* counts) {
    extern __shared__ unsigned int bins[];
    const int nb = nt * nphi;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) bins[b] = 0u;
    __syncthreads();
    const bool native = METHOD == kCapNative;
    const float s = (!native && wz < 0.0f) ? -1.0f : 1.0f;
    // std-space incidence (for mode 1)
    const float tx = ax * wx, ty = ay * wy;
    const float iL = s * rsqrtf(fmaf(tx, tx, fmaf(ty, ty, wz * wz)));
    const float wsx = tx * iL, wsy = ty * iL, wsz = wz * iL;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const uint4 W = philox_sample(seed, first + (uint64_t)j);
        const float v1 = fmaf(fw(W.x), 0x1p-24f, -0.5f);
        const float f2 = fw(W.y);
        const float u2 = f2 * 0x1p-24f, q = fmaf(f2, -0x1p-24f, 1.0f);
        Sample o;
        if (METHOD == kHeitz) {
            heitz_fp32<false>(wx, wy, wz, ax, ay, v1, u2, o);
        } else {
            const bool f = native ? cap_fp32<false, kFrameNative>(wx, wy, wz, ax, ay, v1, u2, q, o)
                                  : cap_fp32<false>(wx, wy, wz, ax, ay, v1, u2, q, o);
            if (f) {
                const float4 d = cap_fp64(wx, wy, wz, ax, ay, fw(W.x) * 0x1p-24f, u2, !native);
                o.x = d.x;
                o.y = d.y;
                o.z = d.z;
            }
        }
        int ib;
        if (mode == 0) {
            const float th = acosf(fminf(fmaxf(o.z, -1.0f), 1.0f));
            float ph = atan2f(o.y, o.x);
            if (ph < 0.0f) ph += 6.28318530717958648f;
            const int it = min(max((int)(th * (float)nt * 0.636619772367581343f), 0), nt - 1);
            const int ip = min(max((int)(ph * (float)nphi * 0.159154943091895336f), 0), nphi - 1);
            ib = it * nphi + ip;
        } else {
            // h' = s h (sampling frame), hs ~ M^T h'
            float hx = s * o.x / ax, hy = s * o.y / ay, hz = s * o.z;
            const float ih = rsqrtf(fmaf(hx, hx, fmaf(hy, hy, hz * hz)));
            hx *= ih; hy *= ih; hz *= ih;
            const float d = 2.0f * fmaf(hx, wsx, fmaf(hy, wsy, hz * wsz));
            const float cx = fmaf(d, hx, -wsx), cy = fmaf(d, hy, -wsy), cz = fmaf(d, hz, -wsz);
            const float uz = (cz + wsz) / (1.0f + wsz);
            float ph = atan2f(cy, cx);
            if (ph < 0.0f) ph += 6.28318530717958648f;
            const int it = min(max((int)(uz * (float)nt), 0), nt - 1);
            const int ip = min(max((int)(ph * (float)nphi * 0.159154943091895336f), 0), nphi - 1);
            ib = it * nphi + ip;
        }
        atomicAdd(&bins[ib], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        if (bins[b]) atomicAdd(&counts[b], (unsigned long long)bins[b]);
}

// ------------------------------------- NEXT-1: sampler-only microbenchmark --
// The paper's GPU methodology: each lane calls Listing 1 `iters`
// times.  Lane t draws its incidence and roughness once from the config-4
// recipe (Philox block of index t).  Iteration k uses the integer Weyl
// sequence u1 = u(s1 + k A1), u2 = u(s2 + k A2) (s1 = W0, s2 = W1) and then
// rotates wi about z by a fixed angle with explicitly rounded fp32 operations
// (so every call does the full Listing 1 -- nothing is loop-invariant -- and
// the host oracle can replay the exact fp32 incidences).  h.x + 2 h.y + 3 h.z
// is summed into a per-lane checksum (the sink).  No pdf, no flag, no fix-up.
// VARIANT 0 = cap (production fp32 arithmetic), 1 = Heitz (Listing 2),
// 2 = Listing 3 literal.
constexpr uint32_t kWeyl1 = 0x9E3779B9u, kWeyl2 = 0x7F4A7C15u;
constexpr float kRotC = 0.764842187f, kRotS = 0.644217687f;  // cos, sin of 0.7 rad (fp32)

template <int VARIANT>
__global__ void __launch_bounds__(256) microbench_kernel(uint64_t seed, int64_t lanes, int iters,
                                                         const float2* __restrict__ gtab,
                                                         float* __restrict__ checksum) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= lanes) return;
    const uint4 W = philox_sample(seed, (uint64_t)t);
    const Inputs in = c4_inputs_fp32(W, gtab);
    uint32_t x1 = W.x, x2 = W.y;
    float wx = in.wx, wy = in.wy;
    float acc = 0.0f;
#pragma unroll 4
    for (int k = 0; k < iters; ++k) {
        const float v1 = fmaf(fw(x1), 0x1p-24f, -0.5f);
        const float f2 = fw(x2);
        Sample o;
        if (VARIANT == 0) {
            cap_fp32<false, kFrameUpper>(wx, wy, in.wz, in.ax, in.ay, v1, f2 * 0x1p-24f,
                                   fmaf(f2, -0x1p-24f, 1.0f), o);
        } else if (VARIANT == 1) {
            heitz_fp32<false, false>(wx, wy, in.wz, in.ax, in.ay, v1, f2 * 0x1p-24f, o);
        } else {
            cap_literal_fp32(wx, wy, in.wz, in.ax, in.ay, v1, f2 * 0x1p-24f, o);
        }
        acc += o.x + 2.0f * o.y + 3.0f * o.z;
        x1 += kWeyl1;
        x2 += kWeyl2;
        const float rx = __fmaf_rn(kRotC, wx, -__fmul_rn(kRotS, wy));
        const float ry = __fmaf_rn(kRotC, wy, __fmul_rn(kRotS, wx));
        wx = rx;
        wy = ry;
    }
    checksum[t] = acc;
}

// =============================================================== host side ==
thread_local int g_last_cuda_error = 0;

struct LaunchPrefs {
    int vector_width = 0;   // 0 = widest the alignment allows
    int block_size = 0;     // 0 = 256
    int blocks_per_sm = 0;  // 0 = occupancy
};
std::mutex g_mu;
LaunchPrefs g_prefs;
std::map<std::tuple<int, const void*, int>, int> g_occ;  // (device, kernel, block) -> blocks/SM
std::map<int, int> g_sms;

vndf_status cuda_fail(cudaError_t e) {
    g_last_cuda_error = (int)e;
    return VNDF_ERR_CUDA;
}

LaunchPrefs prefs() {
    std::lock_guard<std::mutex> lk(g_mu);
    return g_prefs;
}

// Launch with the programmatic-stream-serialization attribute (PDL): the
// kernel may start while the previous kernel on the stream drains; it calls
// griddepcontrol.wait before its first memory access, so stream order holds.
// Disabled with vector_width/block_size knobs untouched via VNDF_NO_PDL=1.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    static const bool off = [] {
        const char* v = getenv("VNDF_NO_PDL");
        return v && v[0] == '1';
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Persistent grid: min(work, SMs x resident blocks per SM).
// persistent: default grid policy of the kernel family when no preference is
// set (streamed kernels: one chunk per thread, measured faster on B200 for
// HBM-bound work; fused Philox: persistent, occupancy-limited).
cudaError_t grid_for(const void* kernel, int block, int64_t work_items, int* grid, bool persistent = true,
                     size_t smem = 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int sms = 0, occ = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_sms.find(dev);
        if (it != g_sms.end()) sms = it->second;
        auto jt = g_occ.find(std::make_tuple(dev, kernel, block));
        if (jt != g_occ.end()) occ = jt->second;
    }
    if (sms == 0) {
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        std::lock_guard<std::mutex> lk(g_mu);
        g_sms[dev] = sms;
    }
    if (occ == 0) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        std::lock_guard<std::mutex> lk(g_mu);
        g_occ[std::make_tuple(dev, kernel, block)] = occ;
    }
    const LaunchPrefs p = prefs();
    if (p.blocks_per_sm > 0) occ = std::min(occ, p.blocks_per_sm);
    const int64_t need = std::max<int64_t>(1, (work_items + block - 1) / block);
    // blocks_per_sm == -1: one work item per thread (non-persistent grid)
    const bool one_per_thread = p.blocks_per_sm < 0 || (p.blocks_per_sm == 0 && !persistent);
    const int64_t cap = one_per_thread ? (int64_t)INT32_MAX : (int64_t)sms * occ;
    *grid = (int)std::min<int64_t>(need, cap);
    return cudaSuccess;
}

// Library-private, stream-ordered memory pool per device for transient
// buffers (the fix-up queue): its release threshold is unlimited, so after the
// first call an allocation is a pool hit instead of a fresh mapping, without
// touching the caller's default pool settings.
std::map<int, cudaMemPool_t> g_pools;

cudaError_t queue_alloc(void** p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_pools.find(dev);
        if (it != g_pools.end()) pool = it->second;
    }
    if (!pool) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        e = cudaMemPoolCreate(&pool, &props);
        if (e != cudaSuccess) return e;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_pools.find(dev);
        if (it != g_pools.end()) {
            cudaMemPoolDestroy(pool);
            pool = it->second;
        } else {
            g_pools[dev] = pool;
        }
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// Opt a kernel into > 48 KB of dynamic shared memory, once per (device, kernel):
// function attributes are per device, a process may drive several.
std::map<std::pair<int, const void*>, bool> g_smem_attr;

cudaError_t allow_dynamic_smem(const void* kernel, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    const auto key = std::make_pair(dev, kernel);
    if (g_smem_attr.count(key)) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) g_smem_attr[key] = true;
    return e;
}

// Octant table of (sin, cos)(2 pi j / 2^16), j = 0 .. 8192, for the config-4
// incidence azimuth: built on the host in float64 (correctly rounded to fp32),
// uploaded once per device, kept for the life of the process (64 KB).
std::map<int, float2*> g_sincos_tab;

cudaError_t sincos_table(float2** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_sincos_tab.find(dev);
    if (it != g_sincos_tab.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    std::vector<float2> h(kSinCosTableEntries);
    for (int j = 0; j < kSinCosTableEntries; ++j) {
        const int jj = j < 8193 ? j : 8192;  // padding entry repeats the last one
        const double a = 2.0 * 3.14159265358979323846 * (double)jj / 65536.0;
        h[j] = make_float2((float)sin(a), (float)cos(a));
    }
    float2* d = nullptr;
    e = cudaMalloc((void**)&d, h.size() * sizeof(float2));
    if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (d) cudaFree(d);
        return e;
    }
    g_sincos_tab[dev] = d;
    *out = d;
    return cudaSuccess;
}

int block_size(int dflt = 256) {
    const int b = prefs().block_size;
    return b > 0 ? b : dflt;
}

bool aligned(const void* p, uintptr_t a) { return ((uintptr_t)p % a) == 0; }

bool overlaps(const void* a, const void* b, int64_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + (uintptr_t)bytes && y < x + (uintptr_t)bytes;
}

// Validate a streamed call: all inputs non-NULL, required outputs non-NULL,
// everything 4-byte aligned, no output overlapping an input or an output.
vndf_status validate_stream(const StreamArgs& a, bool need_pdf, int64_t n) {
    if (n < 0) return VNDF_ERR_INVALID_ARGUMENT;
    const void* in[7] = {a.wx, a.wy, a.wz, a.ax, a.ay, a.u1, a.u2};
    const void* out[4] = {a.hx, a.hy, a.hz, a.pdf};
    const int nout = a.pdf ? 4 : 3;
    for (auto p : in)
        if (!p || !aligned(p, 4)) return VNDF_ERR_INVALID_ARGUMENT;
    for (int k = 0; k < 3; ++k)
        if (!out[k] || !aligned(out[k], 4)) return VNDF_ERR_INVALID_ARGUMENT;
    if (need_pdf && !a.pdf) return VNDF_ERR_INVALID_ARGUMENT;
    if (a.pdf && !aligned(a.pdf, 4)) return VNDF_ERR_INVALID_ARGUMENT;
    const int64_t bytes = n * (int64_t)sizeof(float);
    if (n > 0) {
        for (int k = 0; k < nout; ++k) {
            for (auto p : in)
                if (overlaps(out[k], p, bytes)) return VNDF_ERR_INVALID_ARGUMENT;
            for (int l = k + 1; l < nout; ++l)
                if (overlaps(out[k], out[l], bytes)) return VNDF_ERR_INVALID_ARGUMENT;
        }
    }
    return VNDF_OK;
}

int widest_vector(const StreamArgs& a) {
    const void* all[11] = {a.wx, a.wy, a.wz, a.ax, a.ay, a.u1, a.u2, a.hx, a.hy, a.hz, a.pdf};
    int v = 8;
    for (auto p : all) {
        if (!p) continue;
        if (!aligned(p, 32)) v = std::min(v, 4);
        if (!aligned(p, 16)) v = 1;
    }
    const int cap = prefs().vector_width;
    if (cap == 1) v = 1;
    if (cap == 4) v = std::min(v, 4);
    return v;
}

template <int METHOD, bool PDF, int V>
vndf_status launch_stream_v(const StreamArgs& a, int64_t n, cudaStream_t s) {
    const void* k = (const void*)stream_kernel<METHOD, PDF, V>;
    const int block = block_size(128);
    int grid = 0;
    cudaError_t e = grid_for(k, block, std::max<int64_t>(n / V, 1), &grid, /*persistent=*/false);
    if (e != cudaSuccess) return cuda_fail(e);
    e = launch_pdl(stream_kernel<METHOD, PDF, V>, grid, block, s, a, n);
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

template <int METHOD, bool PDF>
vndf_status launch_stream(const StreamArgs& a, int64_t n, cudaStream_t s) {
    switch (widest_vector(a)) {
        case 8: return launch_stream_v<METHOD, PDF, 8>(a, n, s);
        case 4: return launch_stream_v<METHOD, PDF, 4>(a, n, s);
        default: return launch_stream_v<METHOD, PDF, 1>(a, n, s);
    }
}

StreamArgs make_args(const float* wx, const float* wy, const float* wz, const float* ax,
                     const float* ay, const float* u1, const float* u2, float* hx, float* hy,
                     float* hz, float* pdf) {
    StreamArgs a;
    a.wx = wx; a.wy = wy; a.wz = wz; a.ax = ax; a.ay = ay; a.u1 = u1; a.u2 = u2;
    a.hx = hx; a.hy = hy; a.hz = hz; a.pdf = pdf;
    return a;
}

vndf_status validate_philox_out(int64_t n, float* hx, float* hy, float* hz, float* pdf) {
    if (n < 0 || !hx || !hy || !hz) return VNDF_ERR_INVALID_ARGUMENT;
    float* out[4] = {hx, hy, hz, pdf};
    const int nout = pdf ? 4 : 3;
    for (int k = 0; k < nout; ++k)
        if (!aligned(out[k], 4)) return VNDF_ERR_INVALID_ARGUMENT;
    const int64_t bytes = n * (int64_t)sizeof(float);
    if (n > 0)
        for (int k = 0; k < nout; ++k)
            for (int l = k + 1; l < nout; ++l)
                if (overlaps(out[k], out[l], bytes)) return VNDF_ERR_INVALID_ARGUMENT;
    return VNDF_OK;
}

template <int METHOD, bool PDF, int V>
vndf_status launch_philox_v(uint64_t seed, uint64_t first, int64_t n, float* hx, float* hy, float* hz,
                            float* pdf, cudaStream_t s) {
    const void* k = (const void*)philox_kernel<METHOD, PDF, V>;
    const int block = block_size();
    const size_t smem = kSinCosTableEntries * sizeof(float2);
    cudaError_t e = allow_dynamic_smem(k, smem);
    if (e != cudaSuccess) return cuda_fail(e);
    int grid = 0;
    e = grid_for(k, block, std::max<int64_t>(n / V, 1), &grid, true, smem);
    if (e != cudaSuccess) return cuda_fail(e);
    FixQueue fq{nullptr, nullptr, 0};
    void* qbuf = nullptr;
    if (METHOD == kCap) {
        // stream-ordered transient queue: [count | cap indices]
        fq.cap = (uint64_t)std::min<int64_t>(std::max<int64_t>(n / 128, 1 << 16), (int64_t)1 << 26);
        e = queue_alloc(&qbuf, sizeof(unsigned long long) + fq.cap * sizeof(uint64_t), s);
        if (e != cudaSuccess) return cuda_fail(e);
        fq.count = (unsigned long long*)qbuf;
        fq.idx = (uint64_t*)((char*)qbuf + sizeof(unsigned long long));
        e = cudaMemsetAsync(fq.count, 0, sizeof(unsigned long long), s);
        if (e != cudaSuccess) {
            cudaFreeAsync(qbuf, s);
            return cuda_fail(e);
        }
    }
    float2* gtab = nullptr;
    e = sincos_table(&gtab);
    if (e != cudaSuccess) {
        if (qbuf) cudaFreeAsync(qbuf, s);
        return cuda_fail(e);
    }
    philox_kernel<METHOD, PDF, V><<<grid, block, smem, s>>>(seed, first, n, hx, hy, hz, pdf, fq, gtab);
    e = cudaGetLastError();
    if (e == cudaSuccess && METHOD == kCap) {
        // one thread per queue slot up to SMs x 32 blocks; blocks past the
        // device-side count exit at once
        int sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t fix_blocks = std::min<int64_t>(((int64_t)fq.cap + 127) / 128, (int64_t)std::max(sms, 1) * 32);
        philox_fixup_kernel<<<(int)fix_blocks, 128, 0, s>>>(seed, first, n, fq, gtab, hx, hy, hz, pdf);
        e = cudaGetLastError();
    }
    if (qbuf) {
        const cudaError_t ef = cudaFreeAsync(qbuf, s);
        if (e == cudaSuccess) e = ef;
    }
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

template <int METHOD>
vndf_status launch_philox(uint64_t seed, uint64_t first, int64_t n, float* hx, float* hy, float* hz,
                          float* pdf, cudaStream_t s) {
    vndf_status st = validate_philox_out(n, hx, hy, hz, pdf);
    if (st != VNDF_OK || n == 0) return st;
    constexpr int PV = VNDF_PHILOX_V;
    bool v4 = aligned(hx, 4 * PV) && aligned(hy, 4 * PV) && aligned(hz, 4 * PV) && (!pdf || aligned(pdf, 4 * PV));
    if (prefs().vector_width == 1) v4 = false;
    if (pdf) {
        return v4 ? launch_philox_v<METHOD, true, PV>(seed, first, n, hx, hy, hz, pdf, s)
                  : launch_philox_v<METHOD, true, 1>(seed, first, n, hx, hy, hz, pdf, s);
    }
    return v4 ? launch_philox_v<METHOD, false, PV>(seed, first, n, hx, hy, hz, pdf, s)
              : launch_philox_v<METHOD, false, 1>(seed, first, n, hx, hy, hz, pdf, s);
}

// ------------------------------------------------ host-path staging cache --
// The blocking host entry point streams a batch through two device staging
// sets of kStagingChunk samples (11 planes each: 7 in, 4 out), round-robin
// over kStagingSets streams, so chunk c's H2D copy overlaps chunk c-1's
// kernel and chunk c-2's D2H copy (PCIe is full duplex).
// One staging area per device is kept after first use (3 x 1 Mi x 44 B =
// 138 MB) so repeated calls pay no allocation; a concurrent second caller on
// the same device gets a private area that is freed when it returns.
constexpr int64_t kStagingChunk = (int64_t)1 << 20;
constexpr int kStagingSets = 3;

struct Staging {
    int device = 0;
    float* buf = nullptr;
    cudaStream_t s[kStagingSets] = {};
    cudaEvent_t ev[1 + kStagingSets] = {};
    bool busy = false;
    bool cached = false;
};
std::map<int, Staging*> g_staging;

cudaError_t destroy_staging(Staging* sg) {
    cudaError_t first = cudaSuccess;
    auto keep = [&](cudaError_t e) { if (first == cudaSuccess) first = e; };
    for (auto x : sg->s)
        if (x) keep(cudaStreamDestroy(x));
    for (auto x : sg->ev)
        if (x) keep(cudaEventDestroy(x));
    if (sg->buf) keep(cudaFree(sg->buf));
    delete sg;
    return first;
}

cudaError_t create_staging(int dev, Staging** out) {
    Staging* sg = new Staging();
    sg->device = dev;
    cudaError_t e = cudaMalloc((void**)&sg->buf, (size_t)kStagingSets * 11 * kStagingChunk * sizeof(float));
    for (int k = 0; k < kStagingSets && e == cudaSuccess; ++k)
        e = cudaStreamCreateWithFlags(&sg->s[k], cudaStreamNonBlocking);
    for (int k = 0; k < 1 + kStagingSets && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&sg->ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        destroy_staging(sg);
        return e;
    }
    *out = sg;
    return cudaSuccess;
}

cudaError_t acquire_staging(int dev, Staging** out) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_staging.find(dev);
        if (it != g_staging.end() && !it->second->busy) {
            it->second->busy = true;
            *out = it->second;
            return cudaSuccess;
        }
    }
    Staging* sg = nullptr;
    cudaError_t e = create_staging(dev, &sg);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    sg->busy = true;
    if (g_staging.find(dev) == g_staging.end()) {
        sg->cached = true;
        g_staging[dev] = sg;
    }
    *out = sg;
    return cudaSuccess;
}

void release_staging(Staging* sg) {
    if (sg->cached) {
        std::lock_guard<std::mutex> lk(g_mu);
        sg->busy = false;
        return;
    }
    destroy_staging(sg);
}

}  // namespace

// ================================================================== C ABI ==
extern "C" {

vndf_status vndf_sample_cap(const float* wi_x, const float* wi_y, const float* wi_z,
                            const float* alpha_x, const float* alpha_y, const float* u1,
                            const float* u2, float* h_x, float* h_y, float* h_z, int64_t n,
                            vndf_stream_t stream) {
    const StreamArgs a = make_args(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, nullptr);
    vndf_status st = validate_stream(a, false, n);
    if (st != VNDF_OK || n == 0) return st;
    return launch_stream<kCap, false>(a, n, (cudaStream_t)stream);
}

vndf_status vndf_sample_cap_pdf(const float* wi_x, const float* wi_y, const float* wi_z,
                                const float* alpha_x, const float* alpha_y, const float* u1,
                                const float* u2, float* h_x, float* h_y, float* h_z, float* pdf,
                                int64_t n, vndf_stream_t stream) {
    const StreamArgs a = make_args(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf);
    vndf_status st = validate_stream(a, true, n);
    if (st != VNDF_OK || n == 0) return st;
    return launch_stream<kCap, true>(a, n, (cudaStream_t)stream);
}

vndf_status vndf_sample_cap_pdf_native(const float* wi_x, const float* wi_y, const float* wi_z,
                                       const float* alpha_x, const float* alpha_y, const float* u1,
                                       const float* u2, float* h_x, float* h_y, float* h_z, float* pdf,
                                       int64_t n, vndf_stream_t stream) {
    const StreamArgs a = make_args(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf);
    vndf_status st = validate_stream(a, false, n);
    if (st != VNDF_OK || n == 0) return st;
    return pdf ? launch_stream<kCapNative, true>(a, n, (cudaStream_t)stream)
               : launch_stream<kCapNative, false>(a, n, (cudaStream_t)stream);
}

vndf_status vndf_sample_heitz2018(const float* wi_x, const float* wi_y, const float* wi_z,
                                  const float* alpha_x, const float* alpha_y, const float* u1,
                                  const float* u2, float* h_x, float* h_y, float* h_z, float* pdf,
                                  int64_t n, vndf_stream_t stream) {
    const StreamArgs a = make_args(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf);
    vndf_status st = validate_stream(a, false, n);
    if (st != VNDF_OK || n == 0) return st;
    return pdf ? launch_stream<kHeitz, true>(a, n, (cudaStream_t)stream)
               : launch_stream<kHeitz, false>(a, n, (cudaStream_t)stream);
}

vndf_status vndf_sample_cap_philox(uint64_t seed, uint64_t first_index, int64_t n, float* h_x,
                                   float* h_y, float* h_z, float* pdf, vndf_stream_t stream) {
    return launch_philox<kCap>(seed, first_index, n, h_x, h_y, h_z, pdf, (cudaStream_t)stream);
}

vndf_status vndf_sample_heitz2018_philox(uint64_t seed, uint64_t first_index, int64_t n, float* h_x,
                                         float* h_y, float* h_z, float* pdf, vndf_stream_t stream) {
    return launch_philox<kHeitz>(seed, first_index, n, h_x, h_y, h_z, pdf, (cudaStream_t)stream);
}

vndf_status vndf_philox4x32_10(uint64_t seed, uint64_t first_index, int64_t n, uint32_t block,
                               uint32_t* words, vndf_stream_t stream) {
    if (n < 0 || !words || !aligned(words, 16)) return VNDF_ERR_INVALID_ARGUMENT;
    if (n == 0) return VNDF_OK;
    int grid = 0;
    cudaError_t e = grid_for((const void*)philox_words_kernel, 256, n, &grid);
    if (e != cudaSuccess) return cuda_fail(e);
    philox_words_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, first_index, n, block,
                                                                 (uint4*)words);
    e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_count_fixups(const float* wi_x, const float* wi_y, const float* wi_z,
                              const float* alpha_x, const float* alpha_y, const float* u1,
                              const float* u2, int64_t n, uint64_t* count, vndf_stream_t stream) {
    if (n < 0 || !count || !aligned(count, 8)) return VNDF_ERR_INVALID_ARGUMENT;
    const void* in[7] = {wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2};
    for (auto p : in)
        if (!p || !aligned(p, 4)) return VNDF_ERR_INVALID_ARGUMENT;
    if (n == 0) return VNDF_OK;
    const StreamArgs a = make_args(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, nullptr, nullptr,
                                   nullptr, nullptr);
    int grid = 0;
    cudaError_t e = grid_for((const void*)count_stream_kernel, 256, n, &grid);
    if (e != cudaSuccess) return cuda_fail(e);
    count_stream_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a, n, (unsigned long long*)count);
    e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_count_fixups_philox(uint64_t seed, uint64_t first_index, int64_t n, uint64_t* count,
                                     vndf_stream_t stream) {
    if (n < 0 || !count || !aligned(count, 8)) return VNDF_ERR_INVALID_ARGUMENT;
    if (n == 0) return VNDF_OK;
    int grid = 0;
    cudaError_t e = grid_for((const void*)count_philox_kernel, 256, n, &grid);
    if (e != cudaSuccess) return cuda_fail(e);
    float2* gtab = nullptr;
    e = sincos_table(&gtab);
    if (e != cudaSuccess) return cuda_fail(e);
    count_philox_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, first_index, n, gtab,
                                                                 (unsigned long long*)count);
    e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_sample_cap_pdf_host(const float* wi_x, const float* wi_y, const float* wi_z,
                                     const float* alpha_x, const float* alpha_y, const float* u1,
                                     const float* u2, float* h_x, float* h_y, float* h_z, float* pdf,
                                     int64_t n, vndf_stream_t stream) {
    const StreamArgs host = make_args(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf);
    vndf_status st = validate_stream(host, true, n);
    if (st != VNDF_OK || n == 0) return st;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    Staging* sg = nullptr;
    e = acquire_staging(dev, &sg);
    if (e != cudaSuccess) return cuda_fail(e);
    cudaStream_t user = (cudaStream_t)stream;
    vndf_status result = VNDF_OK;
    // order after prior work on the caller's stream
    e = cudaEventRecord(sg->ev[0], user);
    for (int k = 0; k < kStagingSets && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(sg->s[k], sg->ev[0], 0);
    const float* hin[7] = {wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2};
    float* hout[4] = {h_x, h_y, h_z, pdf};
    for (int64_t off = 0, c = 0; off < n && e == cudaSuccess && result == VNDF_OK; off += kStagingChunk, ++c) {
        const int64_t m = std::min<int64_t>(kStagingChunk, n - off);
        cudaStream_t s = sg->s[c % kStagingSets];
        float* base = sg->buf + (size_t)(c % kStagingSets) * 11 * kStagingChunk;
        float* d[11];
        for (int k = 0; k < 11; ++k) d[k] = base + (size_t)k * kStagingChunk;
        const size_t bytes = (size_t)m * sizeof(float);
        for (int k = 0; k < 7 && e == cudaSuccess; ++k)
            e = cudaMemcpyAsync(d[k], hin[k] + off, bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) break;
        const StreamArgs da = make_args(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10]);
        result = launch_stream<kCap, true>(da, m, s);
        for (int k = 0; k < 4 && e == cudaSuccess && result == VNDF_OK; ++k)
            e = cudaMemcpyAsync(hout[k] + off, d[7 + k], bytes, cudaMemcpyDeviceToHost, s);
    }
    // join both pipeline streams back into the caller's stream, then block
    for (int k = 0; k < kStagingSets; ++k) {
        cudaEventRecord(sg->ev[1 + k], sg->s[k]);
        cudaStreamWaitEvent(user, sg->ev[1 + k], 0);
    }
    const cudaError_t es = cudaStreamSynchronize(user);
    if (e == cudaSuccess) e = es;
    release_staging(sg);
    if (result != VNDF_OK) return result;
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_release_host_staging(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaError_t first = cudaSuccess;
    for (auto& kv : g_staging) {
        Staging* sg = kv.second;
        if (sg->busy) return VNDF_ERR_INVALID_ARGUMENT;
    }
    for (auto& kv : g_staging) {
        cudaError_t e = destroy_staging(kv.second);
        if (first == cudaSuccess) first = e;
    }
    g_staging.clear();
    return first == cudaSuccess ? VNDF_OK : cuda_fail(first);
}

vndf_status vndf_sample_cap_reflect(const float* wi_x, const float* wi_y, const float* wi_z,
                                    const float* alpha_x, const float* alpha_y, const float* u1,
                                    const float* u2, float* wo_x, float* wo_y, float* wo_z, float* pdf,
                                    float* weight, int64_t n, vndf_stream_t stream) {
    if (n < 0) return VNDF_ERR_INVALID_ARGUMENT;
    const void* in[7] = {wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2};
    const void* out[5] = {wo_x, wo_y, wo_z, pdf, weight};
    for (auto p : in)
        if (!p || !aligned(p, 4)) return VNDF_ERR_INVALID_ARGUMENT;
    for (auto p : out)
        if (!p || !aligned(p, 4)) return VNDF_ERR_INVALID_ARGUMENT;
    const int64_t bytes = n * (int64_t)sizeof(float);
    for (int k = 0; k < 5; ++k) {
        for (auto p : in)
            if (n > 0 && overlaps(out[k], p, bytes)) return VNDF_ERR_INVALID_ARGUMENT;
        for (int l = k + 1; l < 5; ++l)
            if (n > 0 && overlaps(out[k], out[l], bytes)) return VNDF_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return VNDF_OK;
    ReflectArgs a{wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, wo_x, wo_y, wo_z, pdf, weight};
    int v = 8;
    for (auto p : in) v = std::min(v, aligned(p, 32) ? 8 : aligned(p, 16) ? 4 : 1);
    for (auto p : out) v = std::min(v, aligned(p, 32) ? 8 : aligned(p, 16) ? 4 : 1);
    if (prefs().vector_width == 1) v = 1;
    if (prefs().vector_width == 4) v = std::min(v, 4);
    const int block = block_size(128);
    int grid = 0;
    cudaError_t e = cudaSuccess;
    cudaStream_t s = (cudaStream_t)stream;
    switch (v) {
        case 8:
            e = grid_for((const void*)reflect_kernel<8>, block, std::max<int64_t>(n / 8, 1), &grid, false);
            if (e == cudaSuccess) e = launch_pdl(reflect_kernel<8>, grid, block, s, a, n);
            break;
        case 4:
            e = grid_for((const void*)reflect_kernel<4>, block, std::max<int64_t>(n / 4, 1), &grid, false);
            if (e == cudaSuccess) e = launch_pdl(reflect_kernel<4>, grid, block, s, a, n);
            break;
        default:
            e = grid_for((const void*)reflect_kernel<1>, block, n, &grid, false);
            if (e == cudaSuccess) e = launch_pdl(reflect_kernel<1>, grid, block, s, a, n);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_pdf(const float* h_x, const float* h_y, const float* h_z, const float* wi_x,
                     const float* wi_y, const float* wi_z, const float* alpha_x, const float* alpha_y,
                     float* pdf, int64_t n, vndf_stream_t stream) {
    if (n < 0 || !pdf || !aligned(pdf, 4)) return VNDF_ERR_INVALID_ARGUMENT;
    const void* in[8] = {h_x, h_y, h_z, wi_x, wi_y, wi_z, alpha_x, alpha_y};
    for (auto p : in) {
        if (!p || !aligned(p, 4)) return VNDF_ERR_INVALID_ARGUMENT;
        if (n > 0 && overlaps(pdf, p, n * (int64_t)sizeof(float))) return VNDF_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return VNDF_OK;
    PdfArgs a{h_x, h_y, h_z, wi_x, wi_y, wi_z, alpha_x, alpha_y, pdf};
    int v = aligned(pdf, 32) ? 8 : aligned(pdf, 16) ? 4 : 1;
    for (auto p : in) v = std::min(v, aligned(p, 32) ? 8 : aligned(p, 16) ? 4 : 1);
    if (prefs().vector_width == 1) v = 1;
    if (prefs().vector_width == 4) v = std::min(v, 4);
    const int block = block_size(128);
    int grid = 0;
    cudaError_t e = cudaSuccess;
    cudaStream_t s = (cudaStream_t)stream;
    switch (v) {
        case 8:
            e = grid_for((const void*)pdf_kernel<8>, block, std::max<int64_t>(n / 8, 1), &grid, false);
            if (e == cudaSuccess) e = launch_pdl(pdf_kernel<8>, grid, block, s, a, n);
            break;
        case 4:
            e = grid_for((const void*)pdf_kernel<4>, block, std::max<int64_t>(n / 4, 1), &grid, false);
            if (e == cudaSuccess) e = launch_pdl(pdf_kernel<4>, grid, block, s, a, n);
            break;
        default:
            e = grid_for((const void*)pdf_kernel<1>, block, n, &grid, false);
            if (e == cudaSuccess) e = launch_pdl(pdf_kernel<1>, grid, block, s, a, n);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_furnace(int method, float wi_x, float wi_y, float wi_z, float alpha_x, float alpha_y,
                         uint64_t seed, uint64_t first_index, int64_t n, double* sums,
                         vndf_stream_t stream) {
    if (n < 0 || !sums || !aligned(sums, 8) || (method != 0 && method != 1)) return VNDF_ERR_INVALID_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        const cudaError_t e = cudaMemsetAsync(sums, 0, 2 * sizeof(double), s);
        return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
    }
    const void* k = method == 0 ? (const void*)furnace_kernel<kCap> : (const void*)furnace_kernel<kHeitz>;
    int grid = 0;
    cudaError_t e = grid_for(k, 256, n, &grid, true);
    if (e != cudaSuccess) return cuda_fail(e);
    void* part = nullptr;
    e = queue_alloc(&part, (size_t)grid * 2 * sizeof(double), s);
    if (e != cudaSuccess) return cuda_fail(e);
    if (method == 0)
        furnace_kernel<kCap><<<grid, 256, 0, s>>>(wi_x, wi_y, wi_z, alpha_x, alpha_y, seed, first_index, n,
                                                  (double*)part);
    else
        furnace_kernel<kHeitz><<<grid, 256, 0, s>>>(wi_x, wi_y, wi_z, alpha_x, alpha_y, seed, first_index,
                                                    n, (double*)part);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        furnace_finish_kernel<<<1, 256, 0, s>>>((const double*)part, grid, sums);
        e = cudaGetLastError();
    }
    const cudaError_t ef = cudaFreeAsync(part, s);
    if (e == cudaSuccess) e = ef;
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_histogram(int method, int mode, float wi_x, float wi_y, float wi_z, float alpha_x,
                           float alpha_y, uint64_t seed, uint64_t first_index, int64_t n, int nt, int nphi,
                           uint64_t* counts, vndf_stream_t stream) {
    if (n < 0 || !counts || !aligned(counts, 8) || method < 0 || method > 2 || (mode != 0 && mode != 1) ||
        nt < 1 || nphi < 1 || (int64_t)nt * nphi > 8192)
        return VNDF_ERR_INVALID_ARGUMENT;
    if (n == 0) return VNDF_OK;
    const size_t smem = (size_t)nt * nphi * sizeof(unsigned int);
    const void* k = method == 0 ? (const void*)histogram_kernel<kCap>
                  : method == 1 ? (const void*)histogram_kernel<kHeitz>
                                : (const void*)histogram_kernel<kCapNative>;
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
    if (e != cudaSuccess) return cuda_fail(e);
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms * std::max(occ, 1));
    cudaStream_t s = (cudaStream_t)stream;
    auto* c = (unsigned long long*)counts;
    if (method == 0)
        histogram_kernel<kCap><<<grid, 256, smem, s>>>(mode, wi_x, wi_y, wi_z, alpha_x, alpha_y, seed, first_index, n, nt, nphi, c);
    else if (method == 1)
        histogram_kernel<kHeitz><<<grid, 256, smem, s>>>(mode, wi_x, wi_y, wi_z, alpha_x, alpha_y, seed, first_index, n, nt, nphi, c);
    else
        histogram_kernel<kCapNative><<<grid, 256, smem, s>>>(mode, wi_x, wi_y, wi_z, alpha_x, alpha_y, seed, first_index, n, nt, nphi, c);
    e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_microbench(int method, uint64_t seed, int64_t lanes, int iters, float* checksum,
                            vndf_stream_t stream) {
    if (lanes < 0 || iters < 0 || !checksum || !aligned(checksum, 4) || method < 0 || method > 2)
        return VNDF_ERR_INVALID_ARGUMENT;
    if (lanes == 0) return VNDF_OK;
    const int block = 256;
    const int64_t grid = (lanes + block - 1) / block;
    if (grid > INT32_MAX) return VNDF_ERR_INVALID_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    float2* gtab = nullptr;
    cudaError_t e = sincos_table(&gtab);
    if (e != cudaSuccess) return cuda_fail(e);
    switch (method) {
        case 0: microbench_kernel<0><<<(int)grid, block, 0, s>>>(seed, lanes, iters, gtab, checksum); break;
        case 1: microbench_kernel<1><<<(int)grid, block, 0, s>>>(seed, lanes, iters, gtab, checksum); break;
        default: microbench_kernel<2><<<(int)grid, block, 0, s>>>(seed, lanes, iters, gtab, checksum); break;
    }
    e = cudaGetLastError();
    return e == cudaSuccess ? VNDF_OK : cuda_fail(e);
}

vndf_status vndf_set_launch_config(int vector_width, int block_size, int blocks_per_sm) {
    if (!(vector_width == 0 || vector_width == 1 || vector_width == 4 || vector_width == 8))
        return VNDF_ERR_INVALID_ARGUMENT;
    if (!(block_size == 0 || (block_size >= 64 && block_size <= 256 && block_size % 32 == 0)))
        return VNDF_ERR_INVALID_ARGUMENT;
    if (blocks_per_sm < -1) return VNDF_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(g_mu);
    g_prefs.vector_width = vector_width;
    g_prefs.block_size = block_size;
    g_prefs.blocks_per_sm = blocks_per_sm;
    return VNDF_OK;
}

const char* vndf_status_string(vndf_status status) {
    switch (status) {
        case VNDF_OK: return "VNDF_OK";
        case VNDF_ERR_INVALID_ARGUMENT: return "VNDF_ERR_INVALID_ARGUMENT";
        case VNDF_ERR_CUDA: return "VNDF_ERR_CUDA";
        case VNDF_ERR_NOT_IMPLEMENTED: return "VNDF_ERR_NOT_IMPLEMENTED";
    }
    return "VNDF_ERR_UNKNOWN";
}

int vndf_last_cuda_error(void) { return g_last_cuda_error; }

int vndf_version(void) { return 100; }

}  // extern "C"
