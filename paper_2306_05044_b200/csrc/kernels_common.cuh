// kernels_common.cuh -- device helpers shared by the kernels: argument structs, streaming
// vector loads/stores, programmatic dependent launch, the per-sample dispatch.
// Part of libvndf's single translation unit (included by vndf.cu inside its
// anonymous namespace); see vndf.cu for the kernel list and DESIGN.md s.6.
#pragma once

// kCapNative: the paper's native below-horizon handling (NEXT-3, no flip)
enum Method { kCap = 0, kHeitz = 1, kCapNative = 2 };

// A device queue of sample indices for deferred float64 fix-ups: a counter
// and `cap` slots (library pool memory, one per call).
struct FixQueue {
    unsigned long long* count;
    uint64_t* idx;
    uint64_t cap;
    unsigned bcap;  // shared-memory block queue slots used (fused kernels, <= kBlockQueue)
};

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
// L2 eviction priority of the 256-bit streaming accesses (PTX allows the
// .L2::evict_* qualifiers on 256-bit accesses only) (measured on B200,
// tools/stream_variants.py): inputs evict-last (the block-level fix-ups re-read
// a few of them), outputs evict-first (written once, never re-read): +1.7% on
// config 2, +5% on config 5 against the default evict-normal.
#ifndef VNDF_LD_L2
#define VNDF_LD_L2 ".L2::evict_last"
#endif
#ifndef VNDF_ST_L2
#define VNDF_ST_L2 ".L2::evict_first"
#endif

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
    asm volatile("ld.global.nc.L1::no_allocate" VNDF_LD_L2 ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
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
    asm volatile("st.global.L1::no_allocate" VNDF_ST_L2 ".v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]),
                 "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}

// ------------------------------------------- programmatic dependent launch --
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------ one sample --
// fp32 sample; returns the conditioning flag (always false for Heitz).
template <int METHOD, bool PDF>
__device__ __forceinline__ bool sample_one(float wx, float wy, float wz, float ax, float ay, float u1,
                                           float u2, Sample& o) {
    const float p1 = phi_reduced(u1);  // u1 - 1/2 exact for u1 on the 2^-24 grid and for u1 >= 1/4
    if (METHOD == kCap) return cap_fp32<PDF>(wx, wy, wz, ax, ay, p1, u2, 1.0f - u2, o);
    if (METHOD == kCapNative) return cap_fp32<PDF, kFrameNative>(wx, wy, wz, ax, ay, p1, u2, 1.0f - u2, o);
    heitz_fp32<PDF>(wx, wy, wz, ax, ay, p1, u2, o);
    return false;
}

// Float64 recomputation of a flagged sample from its fp32 inputs (flip: the
// flip frame of reading R4, else the native frame).
// INLINE: the float64 arithmetic inlined (cap_fp64_d) rather than called
// out of line (cap_fp64).
template <bool INLINE>
__device__ __forceinline__ Sample fix_regs(float wx, float wy, float wz, float ax, float ay, float u1, float u2,
                                           bool flip) {
    const float4 f = INLINE ? cap_fp64_d(wx, wy, wz, ax, ay, u1, u2, flip) : cap_fp64(wx, wy, wz, ax, ay, u1, u2, flip);
    Sample o;
    o.x = f.x;
    o.y = f.y;
    o.z = f.z;
    o.pdf = f.w;
    return o;
}
