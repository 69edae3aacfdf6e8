// vndf_device.cuh -- per-sample device arithmetic of libvndf (sm_100a).
//
// Citations: "P:n" = PAPER.md line n (arXiv 2306.05044 LaTeX source).
// This file is the product path.  It shares nothing with oracle/ (the float64
// CPU oracle used only by the tests).
//
// Layout of the arithmetic:
//   * the spherical-cap sampler is Listing 1 + Listing 3 rewritten in an
//     algebraically identical, cancellation-free fp32 form;
//   * each sample carries a conditioning flag; flagged samples are recomputed
//     in float64 (cap_fp64) so the 2e-5 / 1e-4 contract holds on every sample;
//   * the Heitz-2018 baseline is Listing 2 taken literally, with the same
//     primitive functions (same harness) and no fix-up.
#pragma once

#include <cstdint>

namespace vndf {

constexpr float kPiF = 3.14159265358979323846f;
constexpr double kPiD = 3.14159265358979323846;

// ---------------------------------------------------------------------------
// Conditioning flag thresholds ("error budget").
// Error model: the fp32 half vector hs = c + ws carries an absolute error
// e S, e a few 1e-7 (fp32 rounding and MUFU sin/cos ~3.6e-7 relative to the
// summands) and S the size of the summands, S <= sqrt(2 (sin^2 theta + rs^2))
// with rs = |ws.xy|; the unstretch multiplies it by at most max(ax, ay) and
// divides by |m| = |diag(ax, ay, 1) hs|, so |dh| ~ e A with A = max(a) S / |m|;
// the pdf |m|^3 / (pi ax ay a |hs|^2) carries ~3 e A + 2 e B, B = S / |hs|.
// Calibrated on the B200 against the float64 oracle with the fix-up disabled
// (tools/calibrate_scaled.py, 2^23 samples of configs 1, 2, 3, 5 and config 5
// in the native frame): with A <= 40 and B <= 60 (S = st + rs) the worst
// errors were |dh| = 5.6e-6 and pdf rel = 4.0e-5 (tolerances 2e-5 / 1e-4);
// the kernels test the same thresholds with the upper bound S^2 <=
// 2 (sin^2 + rs^2) (slightly more conservative).  Fix-up rates: 0.02-0.2%
// (flip frame), 0.3% (config 5, native frame).  Samples outside
//     |m|^2 >= max(a)^2 S^2 / 40^2   and   |hs|^2 >= S^2 / 60^2
// are recomputed in float64.
// The fused kernel (kFrameUpper, config 4) keeps the earlier scale-free test
// (A = max(a)/|m| <= 30, B = 1/|hs| <= 40; calibrated with tools/calibrate_flags.py):
// its inputs never reach the small-S regime and it saves two instructions.
constexpr float kFlagA = 30.0f;            // scale-free A <= 30 (kFrameUpper)
constexpr float kFlagHs = 1.0f / 1600.0f;  // scale-free B <= 40 (kFrameUpper)
constexpr float kFlagMS = 2.0f / 1600.0f;  // scaled: m2 < max(a)^2 * 2 (sin2 + rs2) / 40^2
constexpr float kFlagHsS = 2.0f / 3600.0f; // scaled: hs2 < 2 (sin2 + rs2) / 60^2

// ---------------------------------------------------------------------------
// Explicit single-instruction SFU approximations (MUFU.RSQ / SQRT / RCP).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// sin(2 pi u), cos(2 pi u) for u in [0, 1): phi = 2 pi u1 (Listing 3,
// Listing 2).  The samplers take the reduced angle p = 2 pi v of the
// exactly reduced v = u - 1/2 in [-1/2, 1/2) (exact on the 2^-24 grid of the
// uniforms, and for u >= 1/4 generally), so MUFU.SIN / MUFU.COS run on
// |p| <= pi where their absolute error is ~2^-21.4; sin(2 pi u) = -sin(p),
// same for cos.  p = fl(fl(2 pi) v), one rounding; from a 24-bit integer f
// (u = f 2^-24) one FFMA forms the same bits (phi_reduced_w).
constexpr float k2PiF = 6.28318530717958648f;
__device__ __forceinline__ float phi_reduced(float u) { return (u - 0.5f) * k2PiF; }
// fl(2 pi) 2^-24 and fl(2 pi) / 2 are exact, so this is fl(fl(2 pi) (f 2^-24 - 1/2)),
// the bits of phi_reduced(f 2^-24), in one FFMA instead of an FFMA and an FMUL.
__device__ __forceinline__ float phi_reduced_w(float f) { return fmaf(f, k2PiF * 0x1p-24f, -0.5f * k2PiF); }
__device__ __forceinline__ void sincos_reduced(float p, float* s, float* c) {
    float sv, cv;
    __sincosf(p, &sv, &cv);
    *s = -sv;
    *c = -cv;
}

struct Sample {
    float x, y, z, pdf;
};

// ---------------------------------------------------------------------------
// Spherical-cap VNDF sample, fp32 (Listing 1 P:415-427 + Listing 3
// P:523-539), plus the Eq. 1 pdf.  Returns the conditioning flag.
//
// Cancellation-free algebra (identical in exact arithmetic to Listing 3):
//   a = 1 + ws.z,  q = 1 - u2,  z = q a - ws.z
//   hs.z = z + ws.z = q a                                  (no cancel)
//   1 - z = u2 a,  1 + z = q a + (1 - ws.z) = q a + rs^2 / a,
//   rs^2 = ws.x^2 + ws.y^2 = (1 - ws.z)(1 + ws.z)
//   sin^2(theta) = (1 - z)(1 + z) = u2 (q a^2 + rs^2)
// pdf: with |c| = |ws| = 1, hs.ws = |hs|^2 / 2, so Eq. 1 with Eq. 2-4
//   D_vis = 2 (hs.ws) |m|^3 / (pi a ax ay |hs|^4) = |m|^3 / (pi a ax ay |hs|^2),
//   m = diag(ax, ay, 1) hs (the unnormalised output).
// ---------------------------------------------------------------------------
// p1 = 2 pi (u1 - 1/2) and q = 1 - u2 are passed precomputed (they are free when the
// uniforms are generated in-kernel from integer words).  FRAME selects the
// handling of the incidence frame (kFrameFlip / kFrameUpper / kFrameNative).
// The shared body of the cap kernels: steps (1)-(3) up to the unnormalised
// outputs, kept as named intermediates for the pdf / reflection epilogues.
struct CapCore {
    float s;              // flip sign (reading R4)
    float L2;             // |M^-1 w|^2 of the (possibly non-unit) input w
    float wz_u;           // s * w.z (upper-frame z of the input)
    float a;              // 1 + ws.z
    float hx, hy, hz;     // hs = c + ws (std space, unnormalised)
    float mx, my;         // m = diag(ax, ay, 1) hs
    float m2, invN;       // |m|^2, 1/|m|
    float hs2;            // |hs|^2
    float s2;             // sin^2(theta) + |ws.xy|^2 (size of the summands of hs)
};

// Frames of the incidence: kFrameFlip = reading R4 (wi.z < 0 is flipped);
// kFrameUpper = inputs known to have wi.z >= 0 (config 4); kFrameNative = the
// paper's native below-horizon handling (NEXT-3), where ws.z may be negative.
constexpr int kFrameFlip = 0, kFrameUpper = 1, kFrameNative = 2;

template <int FRAME>
__device__ __forceinline__ CapCore cap_core(float wx, float wy, float wz, float ax, float ay, float p1,
                                            float u2, float q) {
    CapCore k;
    k.s = (FRAME == kFrameFlip && wz < 0.0f) ? -1.0f : 1.0f;  // reading R4 (flip)
    // (1) warp to the hemisphere configuration: ws = M^-1 w / |M^-1 w|
    const float tx = ax * wx, ty = ay * wy;
    k.L2 = fmaf(tx, tx, fmaf(ty, ty, wz * wz));
    const float sinvL = k.s * rsqrt_approx(k.L2);
    const float wsx = tx * sinvL, wsy = ty * sinvL, wsz = wz * sinvL;
    k.wz_u = k.s * wz;
    // (2) sample the spherical cap z in (-ws.z, 1], phi = 2 pi u1
    const float rs2 = fmaf(wsx, wsx, wsy * wsy);
    // a = 1 + ws.z; for ws.z < 0 (native frame only) 1 + ws.z cancels, use the
    // identity 1 + ws.z = (1 - ws.z^2) / (1 - ws.z) = rs^2 / (1 - ws.z)
    k.a = (FRAME == kFrameNative && wsz < 0.0f) ? rs2 * rcp_approx(1.0f - wsz) : 1.0f + wsz;
    k.hz = q * k.a;
    const float sin2 = u2 * fmaf(k.hz, k.a, rs2);
    const float st = sqrt_approx(sin2);
    float sp, cp;
    sincos_reduced(p1, &sp, &cp);
    // half vector hs = c + ws, not normalised
    k.hx = fmaf(st, cp, wsx);
    k.hy = fmaf(st, sp, wsy);
    // (3) warp back with M^-T = diag(ax, ay, 1)
    k.mx = ax * k.hx;
    k.my = ay * k.hy;
    k.m2 = fmaf(k.mx, k.mx, fmaf(k.my, k.my, k.hz * k.hz));
    k.invN = rsqrt_approx(k.m2);
    k.hs2 = fmaf(k.hx, k.hx, fmaf(k.hy, k.hy, k.hz * k.hz));
    k.s2 = sin2 + rs2;  // S^2 / 2 of the error model (scaled conditioning test)
    return k;
}

template <int FRAME>
__device__ __forceinline__ bool cap_flag(const CapCore& k, float ax, float ay) {
#ifdef VNDF_NO_FIXUP  // calibration builds only (tools/calibrate_*.py)
    return false;
#else
    const float amax = fmaxf(ax, ay);
    // A = max(a)/|m| > 30 from the 1/|m| the normalisation already has: one
    // multiply fewer on the fused kernel's FMA datapath than m2 < max(a)^2/900
    if (FRAME == kFrameUpper) return (amax * k.invN > kFlagA) | (k.hs2 < kFlagHs);
    return (k.m2 < kFlagMS * (amax * amax) * k.s2) | (k.hs2 < kFlagHsS * k.s2);
#endif
}

template <bool PDF, int FRAME = kFrameFlip>
__device__ __forceinline__ bool cap_fp32(float wx, float wy, float wz, float ax, float ay,
                                         float p1, float u2, float q, Sample& o) {
    const CapCore k = cap_core<FRAME>(wx, wy, wz, ax, ay, p1, u2, q);
    // normalise and flip back
    const float t = k.s * k.invN;
    o.x = k.mx * t;
    o.y = k.my * t;
    o.z = k.hz * t;
    if (PDF) {
        const float num = k.m2 * (k.m2 * k.invN);            // |m|^3
        const float den = (kPiF * ax * ay) * k.a * k.hs2;
        o.pdf = num * rcp_approx(den);
    }
    return cap_flag<FRAME>(k, ax, ay);
}

// ---------------------------------------------------------------------------
// NEXT-2: reflection sampling (appendix steps (1)-(2)), its pdf
// (Eq. 20) and the sample weight f_r cos / pdf = G2 / G1 (Eq. 11
// with F = 1 and Eq. 13-17).  With unit w' = s w/|w|, L = |M^-1 w'|, z_i = w'.z:
//   w'.h' = L |hs|^2 / (2 |m|)          (ws.hs = |hs|^2 / 2 on the cap)
//   wo = 2 (w.h) h - w                  (Eq. 5)
//   pdf_o = D_vis / (4 w.h) = |m|^4 / (2 pi ax ay (1 + ws.z) L |hs|^4)
//   G2/G1 = z_o (z_i + L) / (L z_o + L_o z_i) if z_o > 0 else 0,
//           L_o = |M^-1 wo'|            (height-correlated Smith, via Lambda)
// ---------------------------------------------------------------------------
struct Reflected {
    float x, y, z, pdf, weight;
};

template <bool FLIP = true>
__device__ __forceinline__ bool cap_reflect_fp32(float wx, float wy, float wz, float ax, float ay,
                                                 float p1, float u2, float q, Reflected& o) {
    const CapCore k = cap_core<FLIP ? kFrameFlip : kFrameUpper>(wx, wy, wz, ax, ay, p1, u2, q);
    const float inv_w = rsqrt_approx(fmaf(wx, wx, fmaf(wy, wy, wz * wz)));
    const float L = k.L2 * rsqrt_approx(k.L2) * inv_w;       // |M^-1 w| / |w|
    const float t = k.s * k.invN;
    const float hx = k.mx * t, hy = k.my * t, hz = k.hz * t;  // h (output frame)
    const float dot = 0.5f * L * k.hs2 * k.invN;              // w_unit . h >= 0
    const float d2 = 2.0f * dot;
    o.x = fmaf(d2, hx, -wx * inv_w);
    o.y = fmaf(d2, hy, -wy * inv_w);
    o.z = fmaf(d2, hz, -wz * inv_w);
    const float m4 = k.m2 * k.m2, hs4 = k.hs2 * k.hs2;
    o.pdf = m4 * rcp_approx((2.0f * kPiF * ax * ay) * k.a * L * hs4);
    const float zi = k.wz_u * inv_w, zo = k.s * o.z;
    const float Lo = sqrt_approx(fmaf(ax * o.x, ax * o.x, fmaf(ay * o.y, ay * o.y, o.z * o.z)));
    const float wgt = zo * (zi + L) * rcp_approx(fmaf(L, zo, Lo * zi));
    o.weight = zo > 0.0f ? wgt : 0.0f;
    return cap_flag<FLIP ? kFrameFlip : kFrameUpper>(k, ax, ay);
}

// ---------------------------------------------------------------------------
// Float64 recomputation of one cap sample (the fix-up).  Same algebra as
// cap_fp32 in double (sincospi, sqrt, rsqrt) up to m and hs; the final
// normalisation and the pdf in fp32 (see below).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 cap_fp64_d(double wx, double wy, double wz, double ax, double ay,
                                             double u1, double u2, bool flip = true) {
    // Normalisations by rsqrt (61 cycles dependent) instead of sqrt + divide
    // (151): the recomputation's latency is what a one-wave launch exposes.
    // rsqrt is ~1 ulp in double, far below the 1e-9 this path needs.
    const double s = (flip && wz < 0.0) ? -1.0 : 1.0;
    const double tx = ax * wx, ty = ay * wy;
    const double iL = s * rsqrt(tx * tx + ty * ty + wz * wz);
    const double wsx = tx * iL, wsy = ty * iL, wsz = wz * iL;
    const double rs2 = wsx * wsx + wsy * wsy;
    double a;  // 1 + ws.z; native frame below the horizon: rs^2 / (1 - ws.z), no cancellation
    if (!flip && wsz < 0.0)
        a = rs2 / (1.0 - wsz);
    else
        a = 1.0 + wsz;
    const double q = 1.0 - u2;
    const double hz = q * a;
    const double st = sqrt(u2 * (hz * a + rs2));
    double sp, cp;
    sincospi(2.0 * u1, &sp, &cp);
    const double hx = fma(st, cp, wsx), hy = fma(st, sp, wsy);
    const double mx = ax * hx, my = ay * hy;
    const double m2 = mx * mx + my * my + hz * hz;
    const double hs2 = hx * hx + hy * hy + hz * hz;
    // The cancellation is behind us: m and hs carry float64 accuracy, and the
    // normalisation and the pdf are products and quotients of them -- well
    // conditioned -- so they run in fp32 (MUFU rsqrt / rcp, relative error
    // ~1e-7, far inside 2e-5 / 1e-4) instead of a dependent float64 rsqrt and
    // division (~230 of the recomputation's 575 clocks, tools/fix_latency.cu).
    // An exact power-of-two scale 2^-k brings |hs|^2 into [1, 4) (and |m|^2,
    // <= max(1, a)^2 |hs|^2, with it), so nothing under- or overflows fp32;
    // pdf = |m|^3 / (pi ax ay a |hs|^2) then carries the factor 2^k.
    const int k = (((__double2hiint(hs2) >> 20) & 0x7ff) - 1023) >> 1;  // floor(floor(log2 |hs|^2) / 2)
    const double sc = __hiloint2double((1023 - k) << 20, 0);           // 2^-k
    const float mxs = (float)(mx * sc), mys = (float)(my * sc), hzs = (float)(hz * sc);
    const float m2s = (float)(m2 * sc * sc), hs2s = (float)(hs2 * sc * sc);
    const float iN = rsqrt_approx(m2s);
    const float t = (float)s * iN;
    const float den = (kPiF * (float)ax * (float)ay) * (float)a * hs2s;
    const float pdf = m2s * (m2s * iN) * rcp_approx(den) * __int_as_float((127 + k) << 23);
    return make_float4(mxs * t, mys * t, hzs * t, pdf);
}

// Float64 reflection sample (fix-up of cap_reflect_fp32), same formulas.
__device__ __forceinline__ void cap_reflect_fp64_d(double wx, double wy, double wz, double ax, double ay,
                                                   double u1, double u2, double out[5]) {
    const double s = (wz < 0.0) ? -1.0 : 1.0;
    const double inw = s * rsqrt(wx * wx + wy * wy + wz * wz);
    const double ux = wx * inw, uy = wy * inw, uz = wz * inw;          // w'
    const double tx = ax * ux, ty = ay * uy;
    const double L2 = tx * tx + ty * ty + uz * uz;
    const double iL = rsqrt(L2), L = L2 * iL;
    const double wsx = tx * iL, wsy = ty * iL, wsz = uz * iL;
    const double a = 1.0 + wsz, q = 1.0 - u2;
    const double hz = q * a;
    const double st = sqrt(u2 * (hz * a + wsx * wsx + wsy * wsy));
    double sp, cp;
    sincospi(2.0 * u1, &sp, &cp);
    const double hx = fma(st, cp, wsx), hy = fma(st, sp, wsy);
    const double mx = ax * hx, my = ay * hy;
    const double m2 = mx * mx + my * my + hz * hz, iN = rsqrt(m2);
    const double hs2 = hx * hx + hy * hy + hz * hz;
    const double h0 = mx * iN, h1 = my * iN, h2 = hz * iN;            // h' (upper frame)
    const double dot = ux * h0 + uy * h1 + uz * h2;
    const double ox = 2.0 * dot * h0 - ux, oy = 2.0 * dot * h1 - uy, oz = 2.0 * dot * h2 - uz;
    const double Lo = sqrt(ax * ax * ox * ox + ay * ay * oy * oy + oz * oz);
    out[0] = s * ox;
    out[1] = s * oy;
    out[2] = s * oz;
    out[3] = m2 * m2 / (2.0 * kPiD * ax * ay * a * L * hs2 * hs2);
    out[4] = oz > 0.0 ? oz * (uz + L) / (L * oz + Lo * uz) : 0.0;
}

// Out-of-line float64 weight of one reflection sample (furnace fix-up).
__device__ __noinline__ float cap_reflect_weight_fp64(float wx, float wy, float wz, float ax, float ay,
                                                      double u1, double u2) {
    double r[5];
    cap_reflect_fp64_d(wx, wy, wz, ax, ay, u1, u2, r);
    return (float)r[4];
}

// Float64 recomputation of a flagged reflection sample from its fp32 inputs
// (out of line: the streamed reflection kernel's vector loop keeps its registers).
__device__ __noinline__ Reflected cap_reflect_fp64(float wx, float wy, float wz, float ax, float ay, float u1,
                                                   float u2) {
    double r[5];
    cap_reflect_fp64_d(wx, wy, wz, ax, ay, u1, u2, r);
    Reflected o;
    o.x = (float)r[0];
    o.y = (float)r[1];
    o.z = (float)r[2];
    o.pdf = (float)r[3];
    o.weight = (float)r[4];
    return o;
}

// Out-of-line entry for the streamed kernels: widening happens in here, so the
// fp32 hot path carries no conversions for it.
__device__ __noinline__ float4 cap_fp64(float wx, float wy, float wz, float ax, float ay, float u1,
                                        float u2, bool flip = true) {
    return cap_fp64_d(wx, wy, wz, ax, ay, u1, u2, flip);
}

// ---------------------------------------------------------------------------
// NEXT-4: the VNDF pdf, Eq. 1, at a caller-provided h.  With
// k = M^T h = (hx/ax, hy/ay, hz) and L = |M^-1 w| (reading R4 for w.z < 0),
// Eq. 1-4 reduce exactly to
//   D_vis(h, w) = 2 max(0, h.w) |h|^3 / (pi ax ay (L + s w.z) |k|^4)  if s h.z > 0, else 0,
// invariant to the scale of h and w.  Every factor is a product or a sum of
// squares (relative accuracy) except h.w, which is accumulated in float64.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float vndf_pdf_fp32(float hx, float hy, float hz, float wx, float wy, float wz,
                                               float ax, float ay) {
    const float s = (wz < 0.0f) ? -1.0f : 1.0f;
    const double dot = fma((double)hx, (double)wx, fma((double)hy, (double)wy, (double)hz * (double)wz));
    const float tx = ax * wx, ty = ay * wy;
    const float L2 = fmaf(tx, tx, fmaf(ty, ty, wz * wz));
    const float L = L2 * rsqrt_approx(L2);
    const float iax = rcp_approx(ax), iay = rcp_approx(ay);
    const float kx = hx * iax, ky = hy * iay;
    const float k2 = fmaf(kx, kx, fmaf(ky, ky, hz * hz));
    const float h2 = fmaf(hx, hx, fmaf(hy, hy, hz * hz));
    const float h3 = h2 * (h2 * rsqrt_approx(h2));
    const float num = 2.0f * (float)fmax(dot, 0.0) * h3;
    const float den = (kPiF * ax * ay) * (L + s * wz) * (k2 * k2);
    return (s * hz > 0.0f) ? num * rcp_approx(den) : 0.0f;
}

// ---------------------------------------------------------------------------
// Listing 1 around Listing 3 taken LITERALLY in fp32:
//   z = fma(1 - u.y, 1 + wi.z, -wi.z); sinTheta = sqrt(clamp(1 - z z, 0, 1)).
// Used only by the sampler-only microbenchmark (NEXT-1) to compare the
// paper's own fp32 code with Listing 2 in the paper's methodology; the
// production kernels use cap_fp32 (same cost class, no cancellation).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cap_literal_fp32(float wx, float wy, float wz, float ax, float ay,
                                                 float p1, float u2, Sample& o) {
    const float tx = ax * wx, ty = ay * wy;
    const float invL = rsqrt_approx(fmaf(tx, tx, fmaf(ty, ty, wz * wz)));
    const float wsx = tx * invL, wsy = ty * invL, wsz = wz * invL;
    float sp, cp;
    sincos_reduced(p1, &sp, &cp);
    const float z = fmaf(1.0f - u2, 1.0f + wsz, -wsz);
    const float st = sqrt_approx(fminf(fmaxf(fmaf(-z, z, 1.0f), 0.0f), 1.0f));
    const float hx = fmaf(st, cp, wsx), hy = fmaf(st, sp, wsy), hz = z + wsz;
    const float mx = ax * hx, my = ay * hy;
    const float invN = rsqrt_approx(fmaf(mx, mx, fmaf(my, my, hz * hz)));
    o.x = mx * invN;
    o.y = my * invN;
    o.z = hz * invN;
}

// ---------------------------------------------------------------------------
// Heitz-2018 baseline, fp32: Listing 1 around Listing 2 taken
// literally, with the same SFU primitives as the cap kernel.
// pdf: Eq. 1 for a unit std-space normal hs:
//   D_vis = 2 max(hs.ws, 0) |m|^3 / (pi a ax ay |hs|^4).
// ---------------------------------------------------------------------------
template <bool PDF, bool FLIP = true>
__device__ __forceinline__ void heitz_fp32(float wx, float wy, float wz, float ax, float ay,
                                           float p1, float u2, Sample& o) {
    const float s = (FLIP && wz < 0.0f) ? -1.0f : 1.0f;
    const float tx = ax * wx, ty = ay * wy;
    const float L2 = fmaf(tx, tx, fmaf(ty, ty, wz * wz));
    const float sinvL = s * rsqrt_approx(L2);
    const float wsx = tx * sinvL, wsy = ty * sinvL, wsz = wz * sinvL;
    // orthonormal basis (with special case if cross product is 0)
    const float tmp = wsx * wsx + wsy * wsy;
    float w1x = 1.0f, w1y = 0.0f;
    if (tmp > 0.0f) {
        const float it = rsqrt_approx(tmp);
        w1x = -wsy * it;
        w1y = wsx * it;
    }
    // w2 = cross(ws, w1) with w1.z = 0
    const float w2x = -wsz * w1y, w2y = wsz * w1x, w2z = wsx * w1y - wsy * w1x;
    // parameterization of the cross section
    float sp, cp;
    sincos_reduced(p1, &sp, &cp);
    const float r = sqrt_approx(u2);
    const float t1 = r * cp;
    float t2 = r * sp;
    const float sh = (1.0f + wsz) * 0.5f;
    t2 = (1.0f - sh) * sqrt_approx(1.0f - t1 * t1) + sh * t2;
    const float ti = sqrt_approx(fmaxf(1.0f - t1 * t1 - t2 * t2, 0.0f));
    // reprojection onto hemisphere
    const float hx = t1 * w1x + t2 * w2x + ti * wsx;
    const float hy = t1 * w1y + t2 * w2y + ti * wsy;
    const float hz = t2 * w2z + ti * wsz;
    // warp back
    const float mx = ax * hx, my = ay * hy;
    const float m2 = fmaf(mx, mx, fmaf(my, my, hz * hz));
    const float invN = rsqrt_approx(m2);
    const float t = s * invN;
    o.x = mx * t;
    o.y = my * t;
    o.z = hz * t;
    if (PDF) {
        const float hs2 = fmaf(hx, hx, fmaf(hy, hy, hz * hz));
        const float dotp = fmaxf(fmaf(hx, wsx, fmaf(hy, wsy, hz * wsz)), 0.0f);
        const float num = 2.0f * dotp * m2 * (m2 * invN);
        const float den = (kPiF * ax * ay) * (1.0f + wsz) * (hs2 * hs2);
        o.pdf = num * rcp_approx(den);
    }
}

// Heitz-2018 counterpart of cap_reflect_fp32 (same harness, for the furnace
// comparison): h from Listing 2, then w.h directly, the general Eq. 20 form
// pdf_h / (4 w.h) and the same G2/G1 weight.
template <bool FLIP = true>
__device__ __forceinline__ void heitz_reflect_fp32(float wx, float wy, float wz, float ax, float ay,
                                                   float p1, float u2, Reflected& o) {
    Sample h;
    heitz_fp32<true, FLIP>(wx, wy, wz, ax, ay, p1, u2, h);
    const float inv_w = rsqrt_approx(fmaf(wx, wx, fmaf(wy, wy, wz * wz)));
    const float ux = wx * inv_w, uy = wy * inv_w, uz = wz * inv_w;
    const float dot = fmaxf(fmaf(ux, h.x, fmaf(uy, h.y, uz * h.z)), 0.0f);
    const float d2 = 2.0f * dot;
    o.x = fmaf(d2, h.x, -ux);
    o.y = fmaf(d2, h.y, -uy);
    o.z = fmaf(d2, h.z, -uz);
    o.pdf = h.pdf * rcp_approx(4.0f * dot);
    const float s = (FLIP && wz < 0.0f) ? -1.0f : 1.0f;
    const float zi = s * uz, zo = s * o.z;
    const float L = sqrt_approx(fmaf(ax * ux, ax * ux, fmaf(ay * uy, ay * uy, uz * uz)));
    const float Lo = sqrt_approx(fmaf(ax * o.x, ax * o.x, fmaf(ay * o.y, ay * o.y, o.z * o.z)));
    const float wgt = zo * (zi + L) * rcp_approx(fmaf(L, zo, Lo * zi));
    o.weight = zo > 0.0f ? wgt : 0.0f;
}


// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11), counter-based: no state, any index.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mul_hilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mul_hilo(0xD2511F53u, c.x, hi0, lo0);
        mul_hilo(0xCD9E8D57u, c.z, hi1, lo1);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// Config-4 inputs from TWO Philox4x32-10 blocks per sample (counter = sample
// index, key = seed, vndf.h, DESIGN.md s.5 reading R12):
//   X = Philox(ctr (i_lo, i_hi, 0, 0)), Y = Philox(ctr (i_lo, i_hi, 1, 0))
//   wi: z = 1 - u(X0), r = sqrt(u(X0) (2 - u(X0))), phi = 2 pi u(X1)  (uniform upper hemisphere)
//   ax = 0.01 * 100^u(X2), ay = 0.01 * 100^u(X3)                      (log-uniform [0.01, 1])
//   u1 = u(Y0), u2 = u(Y1)                                            (the method's uniforms)
// with u(w) = (w >> 8) 2^-24 (24 bits each).
constexpr float kLog2_100F = 6.64385618977472436f;
constexpr double kLog2_100D = 6.64385618977472436;

// Inputs of one sample in the form the samplers take: p1 = 2 pi (u1 - 1/2)
// (sincos_reduced), q = 1 - u2 (exact); v1 = u1 - 1/2 (exact) for the float64
// recomputation.
struct Inputs {
    float wx, wy, wz, ax, ay, v1, p1, u2, q;
};

// Integer multiply-add / high multiply pinned to IMAD (FMA pipe): left to
// itself the compiler turns x * 2^k + c into SHF/IADD3/LEA on the ALU pipe.
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t imad_hi(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// The 24-bit integer of a word, as float: u(w) = fw(w) 2^-24 exactly.
__device__ __forceinline__ float fw(uint32_t w) { return __uint2float_rn(w >> 8); }
// The same value with the shift as a high multiply (FMA-heavy pipe, see imad),
// for kernels short of ALU-pipe issue (VNDF_CAP_FW_HI).
__device__ __forceinline__ float fw_hi(uint32_t w) { return __uint2float_rn(imad_hi(w, 1u << 24)); }
template <bool HI>
__device__ __forceinline__ float fw_t(uint32_t w) { return HI ? fw_hi(w) : fw(w); }

// The per-round Philox keys of a seed, precomputed on the host and passed as a
// __grid_constant__ kernel parameter: the round XORs then read them from the
// constant bank (LOP3 ... c[0x0][...]) instead of occupying 20 registers.
struct PhiloxKeys {
    uint32_t k0[10], k1[10];
};

inline PhiloxKeys philox_keys(uint64_t seed) {
    PhiloxKeys ks;
    uint32_t a = (uint32_t)seed, b = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        ks.k0[r] = a;
        ks.k1[r] = b;
        a += 0x9E3779B9u;
        b += 0xBB67AE85u;
    }
    return ks;
}

// One Philox round in plain C (no inline asm), so that the compiler folds the
// constant counter words (c.z = block, c.w = 0) and shares the rounds that the
// two blocks of one sample have in common: both blocks multiply the same
// c.x in round 0, and their states differ in one word after it.
__device__ __forceinline__ uint4 philox_round(uint4 c, uint32_t k0, uint32_t k1) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    return make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1,
                      (uint32_t)p0);
}

// Blocks 0 and 1 of sample counter i with the precomputed keys.
__device__ __forceinline__ void philox_pair_ks(const PhiloxKeys& ks, uint64_t i, uint4& X, uint4& Y) {
    uint4 x = make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0u, 0u);
    uint4 y = make_uint4((uint32_t)i, (uint32_t)(i >> 32), 1u, 0u);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        x = philox_round(x, ks.k0[r], ks.k1[r]);
        y = philox_round(y, ks.k0[r], ks.k1[r]);
    }
    X = x;
    Y = y;
}

// The same two blocks from round 0's shared product p0 = M0 i_lo (64-bit) and
// i_hi.  Round 0 of counter (i_lo, i_hi, b, 0) leaves x = (i_hi ^ k0, lo(M1 b),
// hi(p0) ^ k1, lo(p0)) with M1 b = 0 (b = 0) or M1 (b = 1), so after it the
// blocks differ in one word; rounds 1-9 as in philox_pair_ks.  For the counters
// base + j of a chunk with base = 0 mod 8 and j < 8 (no carry into i_hi),
// M0 (base_lo + j) = M0 base_lo + M0 j exactly: one IMAD.WIDE per chunk and a
// 64-bit add per sample replace a multiply per sample on the FMA datapath.
__device__ __forceinline__ void philox_pair_r0(const PhiloxKeys& ks, uint64_t p0, uint32_t i_hi, uint4& X,
                                               uint4& Y) {
    uint4 x = make_uint4(i_hi ^ ks.k0[0], 0u, (uint32_t)(p0 >> 32) ^ ks.k1[0], (uint32_t)p0);
    uint4 y = make_uint4(i_hi ^ ks.k0[0], 0xCD9E8D57u, (uint32_t)(p0 >> 32) ^ ks.k1[0], (uint32_t)p0);
#pragma unroll
    for (int r = 1; r < 10; ++r) {
        x = philox_round(x, ks.k0[r], ks.k1[r]);
        y = philox_round(y, ks.k0[r], ks.k1[r]);
    }
    X = x;
    Y = y;
}

__device__ __forceinline__ uint4 philox_block(uint64_t seed, uint64_t i, uint32_t block) {
    return philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), block, 0u),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// Block 0 only (furnace and histogram kernels: u1 = u(W0), u2 = u(W1)).
__device__ __forceinline__ uint4 philox_sample(uint64_t seed, uint64_t i) { return philox_block(seed, i, 0u); }

// sin and cos of phi = 2 pi u(w) for the 24-bit uniform of a word, with
// relative accuracy in each component (the incidence needs it: the stretch
// multiplies an absolute error of wi.x, wi.y by up to max(a)/|M^-1 wi|, large
// at grazing incidence; MUFU.SIN/COS, absolute error 2^-21.4, would not do).
// Exact integer reduction: with k = w >> 8 and r the low 22 bits of k read as
// a signed number (r in [-2^21, 2^21)), k = q 2^22 + r and
//   phi = q pi/2 + theta,  theta = 2 pi r 2^-24,  |theta| <= pi/4;
// r 2^10 is the int32 (w & ~0xFF) << 2, converted exactly; theta takes one
// rounding.  sin/cos(theta) by fp32 polynomials fitted for relative error on
// [0, pi/4] (tools/sincos_fit.py: <= 1.95 / 1.44 ulp over all 2^22 reduced
// arguments); the quadrant q = (k + 2^21) >> 22 swaps them (q odd) and sets
// the signs: sin negative for q = 2, 3; cos negative for q = 1, 2.
__device__ __forceinline__ void sincos_2pi_u24(uint32_t w, float* s, float* c) {
    const int32_t ir = (int32_t)((w & 0xFFFFFF00u) << 2);             // r 2^10
    const float th = __int2float_rn(ir) * 0x1.921fb6p-32f;             // 2 pi 2^-34 (fp32)
    const float x = th * th;
    float ps = fmaf(x, -1.951729937e-04f, 8.332177997e-03f);
    ps = fmaf(x, ps, -1.666665524e-01f);
    const float sn = fmaf(th * x, ps, th);
    float pc = fmaf(x, 2.438356933e-05f, -1.388668199e-03f);
    pc = fmaf(x, pc, 4.166661948e-02f);
    pc = fmaf(x, pc, -0.5f);
    const float cs = fmaf(x, pc, 1.0f);
    const uint32_t q0 = w + 0x20000000u;   // bits 31:30 = q
    const uint32_t q1 = w + 0x60000000u;   // bits 31:30 = q + 1
    const bool odd = (q0 & 0x40000000u) != 0u;
    const float a = odd ? cs : sn, b = odd ? sn : cs;
    *s = __uint_as_float(__float_as_uint(a) ^ (q0 & 0x80000000u));
    *c = __uint_as_float(__float_as_uint(b) ^ (q1 & 0x80000000u));
}

// FW_HI: convert the 24-bit uniforms with fw_hi (bit-identical to fw).
template <bool FW_HI = false>
__device__ __forceinline__ Inputs c4_inputs_fp32(uint4 X, uint4 Y) {
    Inputs in;
    const float fa = fw_t<FW_HI>(X.x);
    const float ua = fa * 0x1p-24f;
    const float z = fmaf(fa, -0x1p-24f, 1.0f);          // 1 - ua, exact
    const float r = sqrt_approx(fmaf(ua, z, ua));       // sqrt(ua (1 + z)) = sqrt(ua (2 - ua)), one rounding
    float sp, cp;
    sincos_2pi_u24(X.y, &sp, &cp);
    in.wx = r * cp;
    in.wy = r * sp;
    in.wz = z;
    // 0.01 * 100^u = 2^((u - 1) log2 100); u log2 100 = fw (2^-24 log2 100) exactly
    in.ax = ex2_approx(fmaf(fw_t<FW_HI>(X.z), kLog2_100F * 0x1p-24f, -kLog2_100F));
    in.ay = ex2_approx(fmaf(fw_t<FW_HI>(X.w), kLog2_100F * 0x1p-24f, -kLog2_100F));
    const float f1 = fw_t<FW_HI>(Y.x);
    in.v1 = fmaf(f1, 0x1p-24f, -0.5f);
    in.p1 = phi_reduced_w(f1);
    const float f2 = fw_t<FW_HI>(Y.y);
    in.u2 = f2 * 0x1p-24f;
    in.q = fmaf(f2, -0x1p-24f, 1.0f);
    return in;
}

// Config-5 inputs (BASELINE config 5, path-tracer edge mix; DESIGN.md s.5
// recipe 5) from the two words blocks of a sample, in the recipe's fp32
// operations, so the fused edge kernels sample exactly the fp32 inputs that
// the streamed kernels read from planes generated by the same recipe:
//   category v = u(Y2): v < 0.4 grazing z = 1e-4 + u(X0) (0.05 - 1e-4),
//   v < 0.6 back side z = -(1 - u(X0)), else upper z = 1 - u(X0);
//   phi = 2 pi u(X1), r = sqrt(max((1 - z)(1 + z), 0));
//   alpha_x = T[X2 >> 30], alpha_y = T[X3 >> 30], T = {1e-3, 0.05, 0.3, 1};
//   u1 = u(Y0), u2 = u(Y1); Y3 bits 0-5 = 0 -> u1 = 0, bits 6-11 = 0 -> u2 = 0,
//   bits 12-17 = 0 -> u2 = 1 - 2^-24 (the rim; a later rule wins).
__device__ __forceinline__ float alpha_edge(uint32_t w) {
    // two selects on the index bits (a compare chain compiled to divergent branches)
    const bool b0 = (w >> 30) & 1u, b1 = (w >> 31) != 0u;
    const float lo = b0 ? 0.05f : 1e-3f, hi = b0 ? 1.0f : 0.3f;
    return b1 ? hi : lo;
}

__device__ __forceinline__ Inputs c5_inputs_fp32(uint4 X, uint4 Y) {
    const float ua = __uint2float_rn(X.x >> 8) * 0x1p-24f;
    float sp, cp;
    sincospif(2.0f * (__uint2float_rn(X.y >> 8) * 0x1p-24f), &sp, &cp);
    const float v = __uint2float_rn(Y.z >> 8) * 0x1p-24f;
    // branch-free: all three categories, then selects
    const float z_graze = 1e-4f + ua * (0.05f - 1e-4f), z_upper = 1.0f - ua;
    const float z = v < 0.4f ? z_graze : v < 0.6f ? -z_upper : z_upper;
    const float r = sqrtf(fmaxf((1.0f - z) * (1.0f + z), 0.0f));
    float u1 = __uint2float_rn(Y.x >> 8) * 0x1p-24f, u2 = __uint2float_rn(Y.y >> 8) * 0x1p-24f;
    if ((Y.w & 0x3Fu) == 0u) u1 = 0.0f;
    if (((Y.w >> 6) & 0x3Fu) == 0u) u2 = 0.0f;
    if (((Y.w >> 12) & 0x3Fu) == 0u) u2 = 1.0f - 0x1p-24f;
    Inputs in;
    in.wx = r * cp;
    in.wy = r * sp;
    in.wz = z;
    in.ax = alpha_edge(X.z);
    in.ay = alpha_edge(X.w);
    in.v1 = u1 - 0.5f;  // exact: u1 is on the 2^-24 grid
    in.p1 = in.v1 * k2PiF;
    in.u2 = u2;
    in.q = 1.0f - u2;
    return in;
}

__device__ __forceinline__ double u01d(uint32_t w) { return (double)(w >> 8) * 0x1p-24; }

// The config-4 inputs of a sample in double from the exact uniforms:
// in = (wi.x, wi.y, wi.z, alpha_x, alpha_y, u1, u2) (vndf.h recipe).
__device__ __forceinline__ void c4_inputs_fp64(uint4 X, uint4 Y, double in[7]) {
    const double ua = u01d(X.x);
    const double r = sqrt(ua * (2.0 - ua));
    double sp, cp;
    sincospi(2.0 * u01d(X.y), &sp, &cp);
    in[0] = r * cp;
    in[1] = r * sp;
    in[2] = 1.0 - ua;
    in[3] = exp2((u01d(X.z) - 1.0) * kLog2_100D);
    in[4] = exp2((u01d(X.w) - 1.0) * kLog2_100D);
    in[5] = u01d(Y.x);
    in[6] = u01d(Y.y);
}

__device__ __forceinline__ void c4_inputs_fp64(uint64_t seed, uint64_t i, double in[7]) {
    c4_inputs_fp64(philox_block(seed, i, 0u), philox_block(seed, i, 1u), in);
}

// Float64 fix-up for a config-4 sample: regenerate the words, build the inputs
// in double from the exact uniforms, sample in double.
__device__ __noinline__ float4 cap_philox_fp64(uint64_t seed, uint64_t i) {
    double in[7];
    c4_inputs_fp64(seed, i, in);
    return cap_fp64_d(in[0], in[1], in[2], in[3], in[4], in[5], in[6]);
}

// The same for the reflection outputs (wo.xyz, Eq. 20 pdf, G2/G1 weight).
__device__ __noinline__ void cap_reflect_philox_fp64(uint64_t seed, uint64_t i, double out[5]) {
    double in[7];
    c4_inputs_fp64(seed, i, in);
    cap_reflect_fp64_d(in[0], in[1], in[2], in[3], in[4], in[5], in[6], out);
}

}  // namespace vndf
