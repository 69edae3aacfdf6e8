// kernels_next.cuh -- the SURVEY 8(f) NEXT rows: standalone pdf (NEXT-4), reflection
// sampling and the white-furnace estimator (NEXT-2), device histograms
// (NEXT-3), the sampler-only microbenchmark (NEXT-1).
// Part of libvndf's single translation unit (included by vndf.cu inside its
// anonymous namespace); see vndf.cu for the kernel list and DESIGN.md s.6.
#pragma once

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
#pragma unroll
        for (int j = 0; j < V; ++j) {
            Reflected r;
            // a flagged sample is recomputed in float64 at once from its registers
            if (cap_reflect_fp32(wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j], phi_reduced(u1.v[j]), u2.v[j],
                                 1.0f - u2.v[j], r))
                r = cap_reflect_fp64(wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j], u1.v[j], u2.v[j]);
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
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            const float wx = a.wx[i], wy = a.wy[i], wz = a.wz[i], ax = a.ax[i], ay = a.ay[i], u1 = a.u1[i],
                        u2 = a.u2[i];
            Reflected r;
            if (cap_reflect_fp32(wx, wy, wz, ax, ay, phi_reduced(u1), u2, 1.0f - u2, r))
                r = cap_reflect_fp64(wx, wy, wz, ax, ay, u1, u2);
            a.ox[i] = r.x;
            a.oy[i] = r.y;
            a.oz[i] = r.z;
            a.pdf[i] = r.pdf;
            a.weight[i] = r.weight;
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
        const float p1 = phi_reduced_w(fw(W.x));
        const float f2 = fw(W.y);
        Reflected r;
        if (METHOD == kCap) {
            if (cap_reflect_fp32(wx, wy, wz, ax, ay, p1, f2 * 0x1p-24f, fmaf(f2, -0x1p-24f, 1.0f), r)) {
                r.weight = cap_reflect_weight_fp64(wx, wy, wz, ax, ay, u01d(W.x), u01d(W.y));
            }
        } else {
            heitz_reflect_fp32(wx, wy, wz, ax, ay, p1, f2 * 0x1p-24f, r);
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
        const float p1 = phi_reduced_w(fw(W.x));
        const float f2 = fw(W.y);
        const float u2 = f2 * 0x1p-24f, q = fmaf(f2, -0x1p-24f, 1.0f);
        Sample o;
        if (METHOD == kHeitz) {
            heitz_fp32<false>(wx, wy, wz, ax, ay, p1, u2, o);
        } else {
            const bool f = native ? cap_fp32<false, kFrameNative>(wx, wy, wz, ax, ay, p1, u2, q, o)
                                  : cap_fp32<false>(wx, wy, wz, ax, ay, p1, u2, q, o);
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
// recipe (Philox blocks X, Y of index t).  Iteration k uses the integer Weyl
// sequence u1 = u(s1 + k A1), u2 = u(s2 + k A2) (s1 = Y0, s2 = Y1, the words
// of the recipe's u1, u2) and then rotates wi about z by a fixed angle with
// explicitly rounded fp32 operations (so every call does the full Listing 1 --
// nothing is loop-invariant -- and the host oracle can replay the exact fp32
// incidences).  h.x + 2 h.y + 3 h.z is summed into a per-lane checksum (the
// sink).  No pdf, no fix-up.  VARIANT 0 = cap (production fp32 arithmetic),
// 1 = Heitz (Listing 2), 2 = Listing 3 literal.
// TRACE (vndf_microbench_trace, tests only): also writes every call's
// (h.x, h.y, h.z, flag) to trace[4 (t iters + k) ..], flag = the cap's
// conditioning flag (1.0f: this call would be recomputed in float64 by the
// production kernels; always 0 for variants 1 and 2).
constexpr uint32_t kWeyl1 = 0x9E3779B9u, kWeyl2 = 0x7F4A7C15u;
constexpr float kRotC = 0.764842187f, kRotS = 0.644217687f;  // cos, sin of 0.7 rad (fp32)

template <int VARIANT, bool TRACE>
__global__ void __launch_bounds__(256) microbench_kernel(uint64_t seed, int64_t lanes, int iters,
                                                         float* __restrict__ checksum, float4* __restrict__ trace) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= lanes) return;
    const uint4 X = philox_block(seed, (uint64_t)t, 0u), Y = philox_block(seed, (uint64_t)t, 1u);
    const Inputs in = c4_inputs_fp32(X, Y);
    uint32_t x1 = Y.x, x2 = Y.y;
    float wx = in.wx, wy = in.wy;
    float acc = 0.0f;
#pragma unroll 4
    for (int k = 0; k < iters; ++k) {
        const float p1 = phi_reduced_w(fw(x1));
        const float f2 = fw(x2);
        Sample o;
        bool flag = false;
        if (VARIANT == 0) {
            flag = cap_fp32<false, kFrameUpper>(wx, wy, in.wz, in.ax, in.ay, p1, f2 * 0x1p-24f,
                                                fmaf(f2, -0x1p-24f, 1.0f), o);
        } else if (VARIANT == 1) {
            heitz_fp32<false, false>(wx, wy, in.wz, in.ax, in.ay, p1, f2 * 0x1p-24f, o);
        } else {
            cap_literal_fp32(wx, wy, in.wz, in.ax, in.ay, p1, f2 * 0x1p-24f, o);
        }
        if (TRACE) trace[t * (int64_t)iters + k] = make_float4(o.x, o.y, o.z, flag ? 1.0f : 0.0f);
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
