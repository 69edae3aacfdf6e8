// kernels_philox.cuh -- fused Philox4x32-10 kernels (config 4) and their fused
// reflection twins (NEXT-2), the deferred fix-up queues and kernels, raw Philox
// words, fix-up counters.
// Part of libvndf's single translation unit (included by vndf.cu inside its
// anonymous namespace); see vndf.cu for the kernel list and DESIGN.md s.6.
#pragma once

// Uniform conversion of the cap kernel: 0 = SHF (ALU pipe), 1 = IMAD.HI shifts
// (fw_hi, FMA pipe).  The FMA datapath is the fused kernel's bound (DESIGN.md
// s.6.5), so 0: 145.7 vs 141.8 Gsamples/s with 1 (tools/variants.py).
#ifndef VNDF_CAP_FW_HI
#define VNDF_CAP_FW_HI 0
#endif

// ----------------------------------------------------- fused Philox kernel --
// Deferred float64 fix-up of the fused kernels (compute-bound: an in-thread
// float64 recomputation in the sample loop diverges the warp -- measured 138
// against 147 Gsamples/s at config 4, profiles/r2/fused_variants_r2.txt).
// Flagged local indices (~0.05% of the config-4 samples) are queued per block
// (BlockQueue below) and recomputed by the whole block at the end of its
// sample loop; a block queue's overflow goes to a global queue that the fix-up
// kernel drains, and if that overflowed too (count > cap) the fix-up kernel
// rescans every sample's flag: always correct, slower only then.

// Config-4 inputs of Philox counter ctr (both blocks, SURVEY s.8(d)).
template <bool FW_HI>
__device__ __forceinline__ Inputs c4_inputs_ks(const PhiloxKeys& ks, uint64_t ctr) {
    uint4 X, Y;
    philox_pair_ks(ks, ctr, X, Y);
    return c4_inputs_fp32<FW_HI>(X, Y);
}

__device__ __forceinline__ Inputs c4_inputs_seed(uint64_t seed, uint64_t ctr) {
    return c4_inputs_fp32(philox_block(seed, ctr, 0u), philox_block(seed, ctr, 1u));
}

// In-kernel input recipes of the fused sample kernels: kRecipeC4 = BASELINE
// config 4 (upper hemisphere, log-uniform alpha), kRecipeC5 = config 5 (edge
// mix: grazing, below-horizon and upper incidence, alpha from a 4-value set,
// u = 0 and rim injections).
constexpr int kRecipeC4 = 4, kRecipeC5 = 5;

template <int RECIPE>
__device__ __forceinline__ Inputs recipe_inputs_seed(uint64_t seed, uint64_t ctr) {
    const uint4 X = philox_block(seed, ctr, 0u), Y = philox_block(seed, ctr, 1u);
    return RECIPE == kRecipeC5 ? c5_inputs_fp32(X, Y) : c4_inputs_fp32(X, Y);
}

// Float64 recomputation of a flagged fused sample: config 4 from the exact
// uniforms (c4_inputs_fp64), config 5 from its fp32 inputs (the streamed
// kernels' fix-up of the same inputs).
template <int RECIPE>
__device__ __forceinline__ float4 recipe_cap_fp64(uint64_t seed, uint64_t ctr) {
    if (RECIPE == kRecipeC4) return cap_philox_fp64(seed, ctr);
    const Inputs in = recipe_inputs_seed<RECIPE>(seed, ctr);
    return cap_fp64(in.wx, in.wy, in.wz, in.ax, in.ay, in.v1 + 0.5f, in.u2, true);
}

// Block-level fix-up queue of the fused kernels.  Flagged local indices are
// collected in shared memory (a warp, or in the edge mix each flagged lane,
// reserves its slots with one shared-memory atomic); the sample kernel recomputes them at the end of the block
// (block_queue_fix), the reflection kernel publishes them to the global queue
// with one global atomic per block (block_queue_flush).  Round 1's global
// atomic per flagged warp-chunk stalled the warp on the L2 round trip of its
// return value in the ~12% of warp-chunks that hold a flagged sample (the
// shared-memory queue measured +0.9% at config 4).  Samples past the block's slots
// go to the global queue directly (correct, slower: a persistent block meets
// ~1.8k flagged samples at 2^30 samples per call, so only calls far larger
// than config 4 reach it; test hook VNDF_DEBUG_BLOCK_QUEUE).
constexpr int kBlockQueue = 4096;
struct BlockQueue {
    uint64_t idx[kBlockQueue];
    unsigned count;
    unsigned long long base;
};

__device__ __forceinline__ void block_queue_init(BlockQueue& bq) {
    if (threadIdx.x == 0) bq.count = 0u;
    __syncthreads();
}

// Appends the flagged samples of a V-sample chunk (bit j of `bits`: local
// index i + j), warp-cooperatively: the branch is warp-uniform (no divergent
// branch in the sample loop, so ptxas keeps the Philox round keys in uniform
// registers), one shared atomic per warp reserves the warp's slots, lanes
// place their samples by an exclusive prefix sum of their counts.
// LANE: the flagged lanes alone take their slots with one shared atomic each
// (a divergent branch): faster where flags are frequent and the loop diverges
// anyway (the config-5 edge mix, 0.21% flagged, ~40% of warp-chunks hold a
// flagged sample: 117.8 vs 115.2 Gsamples/s), marginally slower at config 4
// (155.8 vs 156.0; profiles/r2/fused_variants_r2.txt).
template <int V, bool LANE>
__device__ __forceinline__ void queue_flags(const FixQueue& fq, BlockQueue& bq, unsigned bits, uint64_t i) {
    if (LANE) {
        if (bits) {
            unsigned slot = atomicAdd(&bq.count, (unsigned)__popc(bits));
            while (bits) {
                const int j = __ffs(bits) - 1;
                bits &= bits - 1u;
                if (slot < fq.bcap) {
                    bq.idx[slot] = i + (uint64_t)j;
                } else {  // block queue full: straight to the global queue
                    const unsigned long long g = atomicAdd(fq.count, 1ull);
                    if (g < fq.cap) fq.idx[g] = i + (uint64_t)j;
                }
                ++slot;
            }
        }
        return;
    }
    const unsigned act = __activemask();
    if (!__any_sync(act, bits != 0u)) return;
    const unsigned lane = threadIdx.x & 31u;
    const int leader = __ffs(act) - 1;
    const unsigned c = (unsigned)__popc(bits);
    unsigned incl = c;  // inclusive prefix sum over the active lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(act, incl, d);
        if (lane >= (unsigned)d && ((act >> (lane - d)) & 1u)) incl += t;
    }
    const unsigned total = __shfl_sync(act, incl, 31 - __clz(act));
    unsigned base = 0;
    if ((int)lane == leader) base = atomicAdd(&bq.count, total);
    base = __shfl_sync(act, base, leader);
    unsigned slot = base + incl - c;
    while (bits) {
        const int j = __ffs(bits) - 1;
        bits &= bits - 1u;
        if (slot < fq.bcap) {
            bq.idx[slot] = i + (uint64_t)j;
        } else {  // block queue full: straight to the global queue
            const unsigned long long g = atomicAdd(fq.count, 1ull);
            if (g < fq.cap) fq.idx[g] = i + (uint64_t)j;
        }
        ++slot;
    }
}

// Recomputes the block's queued samples in float64 where the block's work
// ends, all threads of the block busy (all call it once, after their sample
// loop) -- no second launch for them; samples past the block queue went to
// the global queue and the fix-up kernel.
#ifndef VNDF_PHILOX_BLOCK_FIX
#define VNDF_PHILOX_BLOCK_FIX 1  // 0: publish the block queue to the fix-up kernel (0.9% slower at config 4)
#endif
template <int RECIPE>
__device__ __forceinline__ void block_queue_fix(const FixQueue& fq, BlockQueue& bq, uint64_t seed, uint64_t first,
                                                float* hx, float* hy, float* hz, float* pdf) {
    __syncthreads();
    const unsigned cnt = min(bq.count, fq.bcap);
    for (unsigned t = threadIdx.x; t < cnt; t += blockDim.x) {
        const uint64_t k = bq.idx[t];
        const float4 f = recipe_cap_fp64<RECIPE>(seed, first + k);
        hx[k] = f.x;
        hy[k] = f.y;
        hz[k] = f.z;
        if (pdf) pdf[k] = f.w;
    }
}

// Publishes the block's queue (all threads of the block call it once).
__device__ __forceinline__ void block_queue_flush(const FixQueue& fq, BlockQueue& bq) {
    __syncthreads();
    const unsigned cnt = min(bq.count, fq.bcap);
    if (threadIdx.x == 0) bq.base = cnt ? atomicAdd(fq.count, (unsigned long long)cnt) : 0ull;
    __syncthreads();
    for (unsigned t = threadIdx.x; t < cnt; t += blockDim.x) {
        const unsigned long long g = bq.base + t;
        if (g < fq.cap) fq.idx[g] = bq.idx[t];
    }
}

// One sample from its two blocks of Philox words; returns the conditioning
// flag (always false for Heitz).
template <int METHOD, bool PDF, int RECIPE>
__device__ __forceinline__ bool sample_words(uint4 X, uint4 Y, Sample& o) {
    if (RECIPE == kRecipeC5) {
        // edge mix: back-side incidence is flipped (reading R4), as in the streamed kernels
        const Inputs in = c5_inputs_fp32(X, Y);
        if (METHOD == kCap) return cap_fp32<PDF>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, o);
        heitz_fp32<PDF>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, o);
        return false;
    }
    const Inputs in = c4_inputs_fp32<VNDF_CAP_FW_HI && METHOD == kCap>(X, Y);
    if (METHOD == kCap) {
        // config-4 inputs are on the upper hemisphere (wi.z = 1 - u > 0): no flip
        return cap_fp32<PDF, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, o);
    }
    heitz_fp32<PDF, false>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, o);
    return false;
}

// ctr = first + k, the Philox counter of local sample k
template <int METHOD, bool PDF, int RECIPE = kRecipeC4>
__device__ __forceinline__ bool philox_one(const PhiloxKeys& ks, uint64_t ctr, Sample& o) {
    uint4 X, Y;
    philox_pair_ks(ks, ctr, X, Y);
    return sample_words<METHOD, PDF, RECIPE>(X, Y, o);
}

template <int RECIPE>
__global__ void __launch_bounds__(128) philox_fixup_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                            FixQueue fq, float* __restrict__ hx,
                                                            float* __restrict__ hy, float* __restrict__ hz,
                                                            float* __restrict__ pdf) {
    const uint64_t count = *fq.count;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto fix = [&](uint64_t k) {
        const float4 f = recipe_cap_fp64<RECIPE>(seed, first + k);
        hx[k] = f.x;
        hy[k] = f.y;
        hz[k] = f.z;
        if (pdf) pdf[k] = f.w;
    };
    if (count <= fq.cap) {
        for (uint64_t t = t0; t < count; t += stride) fix(fq.idx[t]);
        return;
    }
    for (uint64_t k = t0; k < (uint64_t)n; k += stride) {  // overflow: rescan
        const Inputs in = recipe_inputs_seed<RECIPE>(seed, first + k);
        Sample o;
        const bool f = RECIPE == kRecipeC5
                           ? cap_fp32<true>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, o)
                           : cap_fp32<true, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, o);
        if (f) fix(k);
    }
}

// Persistent grid (SMs x resident blocks); 8 samples per thread (one 256-bit
// store per output plane); 512-thread blocks, one per SM at ~123 registers
// (1.4% faster than two 256-thread blocks with the same 16 warps per SM).
// Block sizes / resident blocks per SM are build knobs swept on B200
// (tools/build_variant.py + tools/variants.py, profiles/r2/fused_variants_r2.txt).
#ifndef VNDF_PHILOX_BLOCK_CAP
#define VNDF_PHILOX_BLOCK_CAP 512
#endif
#ifndef VNDF_PHILOX_BLOCK_HEITZ
#define VNDF_PHILOX_BLOCK_HEITZ 512
#endif
#ifndef VNDF_PHILOX_MINB_CAP
#define VNDF_PHILOX_MINB_CAP 1
#endif
#ifndef VNDF_PHILOX_MINB_HEITZ
#define VNDF_PHILOX_MINB_HEITZ 1
#endif
#ifndef VNDF_PHILOX_V_CAP
#define VNDF_PHILOX_V_CAP 8
#endif
#ifndef VNDF_PHILOX_V_HEITZ
#define VNDF_PHILOX_V_HEITZ 8
#endif
template <int METHOD>
struct PhiloxLaunch {
    static constexpr int kBlock = METHOD == kCap ? VNDF_PHILOX_BLOCK_CAP : VNDF_PHILOX_BLOCK_HEITZ;
    static constexpr int kMinBlocks = METHOD == kCap ? VNDF_PHILOX_MINB_CAP : VNDF_PHILOX_MINB_HEITZ;
    static constexpr int kV = METHOD == kCap ? VNDF_PHILOX_V_CAP : VNDF_PHILOX_V_HEITZ;
};

// ALIGNED: first is a multiple of V, so the counters of a chunk share their
// high word and differ only in the low bits (no 64-bit add per sample).
template <int METHOD, bool PDF, int V, bool ALIGNED, int RECIPE = kRecipeC4>
__global__ void __launch_bounds__(PhiloxLaunch<METHOD>::kBlock, PhiloxLaunch<METHOD>::kMinBlocks)
    philox_kernel(uint64_t seed, uint64_t first, int64_t n, float* __restrict__ hxp, float* __restrict__ hyp,
                  float* __restrict__ hzp, float* __restrict__ pdfp, FixQueue fq,
                  const __grid_constant__ PhiloxKeys ks) {
    __shared__ BlockQueue bq;
    if (METHOD == kCap) block_queue_init(bq);
    const int64_t nchunks = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t c = tid; c < nchunks; c += stride) {
        const int64_t i = c * V;
        const uint64_t base = first + (uint64_t)i;
        // aligned chunks: round 0's product M0 i_lo once per chunk (philox_pair_r0)
        const uint64_t p0 = (uint64_t)0xD2511F53u * (uint32_t)base;
        Vec<V> hx, hy, hz, pd;
        unsigned flags = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            Sample o;
            if (ALIGNED && V <= 8) {
                uint4 X, Y;
                philox_pair_r0(ks, p0 + (uint64_t)0xD2511F53u * (uint32_t)j, (uint32_t)(base >> 32), X, Y);
                flags |= (unsigned)sample_words<METHOD, PDF, RECIPE>(X, Y, o) << j;
            } else {
                const uint64_t ctr = ALIGNED ? (base | (uint64_t)j) : base + (uint64_t)j;
                flags |= (unsigned)philox_one<METHOD, PDF, RECIPE>(ks, ctr, o) << j;
            }
            hx.v[j] = o.x;
            hy.v[j] = o.y;
            hz.v[j] = o.z;
            pd.v[j] = o.pdf;
        }
        st_stream<V>(hxp + i, hx);
        st_stream<V>(hyp + i, hy);
        st_stream<V>(hzp + i, hz);
        if (PDF) st_stream<V>(pdfp + i, pd);
        if (METHOD == kCap) queue_flags<V, RECIPE == kRecipeC5>(fq, bq, flags, (uint64_t)i);
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            Sample o;
            const bool f = philox_one<METHOD, PDF, RECIPE>(ks, first + (uint64_t)i, o);
            hxp[i] = o.x;
            hyp[i] = o.y;
            hzp[i] = o.z;
            if (PDF) pdfp[i] = o.pdf;
            if (METHOD == kCap && f) {
                const unsigned long long slot = atomicAdd(fq.count, 1ull);
                if (slot < fq.cap) fq.idx[slot] = (uint64_t)i;
            }
        }
    }
    if (METHOD == kCap) {
        if (VNDF_PHILOX_BLOCK_FIX)
            block_queue_fix<RECIPE>(fq, bq, seed, first, hxp, hyp, hzp, PDF ? pdfp : nullptr);
        else
            block_queue_flush(fq, bq);
    }
}

// ------------------------------------------- fused Philox reflection (NEXT-2) --
// Config-4 inputs generated in-kernel, then appendix steps (1)-(2):
// wo = reflect(wi, h), the Eq. 20 pdf and the G2/G1 weight; 20 B written per
// sample.  The cap kernel defers its ill-conditioned samples to the same
// global queue + float64 fix-up kernel as philox_kernel.
struct ReflectOut {
    float *ox, *oy, *oz, *pdf, *weight;
};

template <int METHOD>
__device__ __forceinline__ bool philox_reflect_one(const PhiloxKeys& ks, uint64_t ctr, Reflected& r) {
    const Inputs in = c4_inputs_ks<VNDF_CAP_FW_HI && METHOD == kCap>(ks, ctr);
    if (METHOD == kCap) return cap_reflect_fp32<false>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, r);
    heitz_reflect_fp32<false>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, r);
    return false;
}

template <int METHOD, int V, bool ALIGNED>
__global__ void __launch_bounds__(PhiloxLaunch<METHOD>::kBlock, PhiloxLaunch<METHOD>::kMinBlocks)
    philox_reflect_kernel(uint64_t first, int64_t n, ReflectOut out, FixQueue fq,
                          const __grid_constant__ PhiloxKeys ks) {
    __shared__ BlockQueue bq;
    if (METHOD == kCap) block_queue_init(bq);
    const int64_t nchunks = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t c = tid; c < nchunks; c += stride) {
        const int64_t i = c * V;
        const uint64_t base = first + (uint64_t)i;
        Vec<V> ox, oy, oz, pd, wg;
        unsigned flags = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint64_t ctr = ALIGNED ? (base | (uint64_t)j) : base + (uint64_t)j;
            Reflected r;
            flags |= (unsigned)philox_reflect_one<METHOD>(ks, ctr, r) << j;
            ox.v[j] = r.x;
            oy.v[j] = r.y;
            oz.v[j] = r.z;
            pd.v[j] = r.pdf;
            wg.v[j] = r.weight;
        }
        st_stream<V>(out.ox + i, ox);
        st_stream<V>(out.oy + i, oy);
        st_stream<V>(out.oz + i, oz);
        st_stream<V>(out.pdf + i, pd);
        st_stream<V>(out.weight + i, wg);
        if (METHOD == kCap) queue_flags<V, false>(fq, bq, flags, (uint64_t)i);
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            Reflected r;
            const bool f = philox_reflect_one<METHOD>(ks, first + (uint64_t)i, r);
            out.ox[i] = r.x;
            out.oy[i] = r.y;
            out.oz[i] = r.z;
            out.pdf[i] = r.pdf;
            out.weight[i] = r.weight;
            if (METHOD == kCap && f) {
                const unsigned long long slot = atomicAdd(fq.count, 1ull);
                if (slot < fq.cap) fq.idx[slot] = (uint64_t)i;
            }
        }
    }
    if (METHOD == kCap) block_queue_flush(fq, bq);
}

__global__ void __launch_bounds__(128) philox_reflect_fixup_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                                    FixQueue fq, ReflectOut out) {
    const uint64_t count = *fq.count;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto fix = [&](uint64_t k) {
        double r[5];
        cap_reflect_philox_fp64(seed, first + k, r);
        out.ox[k] = (float)r[0];
        out.oy[k] = (float)r[1];
        out.oz[k] = (float)r[2];
        out.pdf[k] = (float)r[3];
        out.weight[k] = (float)r[4];
    };
    if (count <= fq.cap) {
        for (uint64_t t = t0; t < count; t += stride) fix(fq.idx[t]);
        return;
    }
    for (uint64_t k = t0; k < (uint64_t)n; k += stride) {  // overflow: rescan
        const Inputs in = c4_inputs_seed(seed, first + k);
        Reflected r;
        if (cap_reflect_fp32<false>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, r)) fix(k);
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
            flag = cap_fp32<true>(a.wx[i], a.wy[i], a.wz[i], a.ax[i], a.ay[i], phi_reduced(a.u1[i]), u2,
                                  1.0f - u2, o);
        }
        warp_count(flag, count);
    }
}

__global__ void __launch_bounds__(256) count_philox_kernel(uint64_t seed, uint64_t first, int64_t n,
                                                           unsigned long long* count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t rounds = (n + stride - 1) / stride;
    for (int64_t r = 0; r < rounds; ++r) {
        const int64_t i = start + r * stride;
        bool flag = false;
        if (i < n) {
            const Inputs in = c4_inputs_seed(seed, first + (uint64_t)i);
            Sample o;
            flag = cap_fp32<true, kFrameUpper>(in.wx, in.wy, in.wz, in.ax, in.ay, in.p1, in.u2, in.q, o);
        }
        warp_count(flag, count);
    }
}
