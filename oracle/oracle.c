/*
 * oracle.c -- plain, slow, obviously-correct float64 CPU oracle for the
 * GGX VNDF spherical-cap sampler of arXiv 2306.05044.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path under paper_2306_05044_b200/ and it never includes or links it.
 *
 * Citations: "P:n" is /root/reference/PAPER.md line n (the paper's LaTeX
 * source), "S:n" is /root/reference/SPEC.md line n.  Every routine below
 * follows the cited passage step by step in the paper's order and notation;
 * all arithmetic is IEEE float64 (the fp32 inputs are widened exactly).
 *
 * Readings of the paper taken here (listed in DESIGN.md section 3):
 *   R1  M^-1 = diag(ax, ay, 1) warps directions to the hemisphere
 *       configuration; normals are warped back with M^-T = diag(ax, ay, 1)
 *       (Listing 1).
 *   R2  u1 drives the azimuth, u2 the cap height / disk radius (P:440-441,
 *       P:528-529).
 *   R4  incidence below the horizon (wi.z < 0; BASELINE config 5) is sampled
 *       on the flipped hemisphere: s = (wi.z < 0 ? -1 : +1) (so -0 -> +1),
 *       w = s*wi, h = s*sample(w), pdf(h | wi) := pdf(s*h | s*wi).
 *   R6  the pdf at grazing incidence uses no division by wi.z (Eq. 1 form).
 *
 * Pinning status (see tests/test_oracle_*.py): every function here is pinned
 * by a closed form, a textbook formula, a library routine, a normalisation
 * integral, a brute-force sampler or a chi-square test; see DESIGN.md s.4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <quadmath.h>

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  Not in the   */
/* paper: BASELINE config 4 asks for "in-kernel Philox4x32-10 (key=seed,    */
/* counter=sample index)"; S:43-48 asks for a counter-based generator.      */
/* Pinned by the Random123 known-answer vectors and by the CUDA toolkit's   */
/* curand_Philox4x32_10 host routine (tests/test_oracle_philox.py).         */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                       uint32_t out[4])
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (round < 9) { k0 += W0; k1 += W1; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox block b of sample index i under seed: counter (i_lo, i_hi, b, 0),
 * key (seed_lo, seed_hi).  DESIGN.md s.5 (input recipe). */
void orc_philox_block(uint64_t seed, uint64_t index, uint32_t block,
                      uint32_t out[4])
{
    uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), block, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

/* uniform in [0,1): (w >> 8) * 2^-24, exact in binary32 and binary64 */
double orc_u01(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }

/* ------------------------------------------------------------------------ */
/* Small vector helpers (plain float64).                                    */
/* ------------------------------------------------------------------------ */
typedef struct { double x, y, z; } v3;
static v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static double len(v3 a) { return sqrt(dot(a, a)); }
static v3 scale(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 normalize(v3 a) { return scale(a, 1.0 / len(a)); }
static v3 cross(v3 a, v3 b)
{
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double clampd(double v, double lo, double hi)
{
    return v < lo ? lo : (v > hi ? hi : v);
}

/* ------------------------------------------------------------------------ */
/* Hemisphere samplers (std space: the unit hemisphere configuration).      */
/* ------------------------------------------------------------------------ */

/* Listing 3, the paper's spherical-cap sampler, line by line:
 *   phi = 2 pi u.x
 *   z   = fma(1 - u.y, 1 + wi.z, -wi.z)   cap in (-wi.z, 1]
 *   sinTheta = sqrt(clamp(1 - z*z, 0, 1))
 *   c = (sinTheta cos phi, sinTheta sin phi, z)
 *   h = c + wi, returned WITHOUT normalisation
 * (the deferred normalisation is done by Listing 1). */
static v3 hemisphere_cap(double u1, double u2, v3 wi)
{
    double phi = 2.0 * ORC_PI * u1;
    double z = fma(1.0 - u2, 1.0 + wi.z, -wi.z);
    double sin_theta = sqrt(clampd(1.0 - z * z, 0.0, 1.0));
    double x = sin_theta * cos(phi);
    double y = sin_theta * sin(phi);
    v3 c = mk(x, y, z);
    v3 h = add(c, wi);
    return h;
}

/* Listing 2, Heitz's cross-section sampler as refactored in the
 * paper, line by line.  Also returns ti for conditioning gates. */
static v3 hemisphere_heitz(double u1, double u2, v3 wi, double *ti_out)
{
    double tmp = wi.x * wi.x + wi.y * wi.y;
    v3 w1 = tmp > 0.0 ? scale(mk(-wi.y, wi.x, 0.0), 1.0 / sqrt(tmp))
                      : mk(1.0, 0.0, 0.0);
    v3 w2 = cross(wi, w1);
    double phi = 2.0 * ORC_PI * u1;
    double r = sqrt(u2);
    double t1 = r * cos(phi);
    double t2 = r * sin(phi);
    double s = (1.0 + wi.z) / 2.0;
    t2 = (1.0 - s) * sqrt(1.0 - t1 * t1) + s * t2;
    double ti = sqrt(fmax(1.0 - t1 * t1 - t2 * t2, 0.0));
    v3 wm = add(add(scale(w1, t1), scale(w2, t2)), scale(wi, ti));
    if (ti_out) *ti_out = ti;
    return wm;
}

/* The hemisphere samplers alone, with NO flip, i.e. the paper's native
 * handling of any wi.z in (-1, 1] (Fig. 4 theta_i = 130 deg).
 * h_out is Listing 3's unnormalised c + wi, or Listing 2's wm. */
void orc_sample_hemisphere(int method, double u1, double u2, const double wi[3],
                           double h_out[3])
{
    v3 w = mk(wi[0], wi[1], wi[2]);
    v3 h = method == 0 ? hemisphere_cap(u1, u2, w) : hemisphere_heitz(u1, u2, w, NULL);
    h_out[0] = h.x; h_out[1] = h.y; h_out[2] = h.z;
}

/* ------------------------------------------------------------------------ */
/* Listing 1: stretch, sample the hemisphere, unstretch.        */
/* method 0 = spherical cap (Listing 3), 1 = Heitz cross section (Listing 2) */
/* Flip reading R4 applied around it.                                       */
/* ------------------------------------------------------------------------ */
void orc_sample_vndf(int method, const double wi_in[3], double ax, double ay,
                     double u1, double u2, double h_out[3], double *ti_out)
{
    double s = (wi_in[2] < 0.0) ? -1.0 : 1.0;                     /* R4 */
    v3 wi = mk(s * wi_in[0], s * wi_in[1], s * wi_in[2]);
    /* warp to the hemisphere configuration: M^-1 wi / |M^-1 wi| */
    v3 wi_std = normalize(mk(wi.x * ax, wi.y * ay, wi.z));
    /* sample the hemisphere */
    v3 wm_std = method == 0 ? hemisphere_cap(u1, u2, wi_std)
                            : hemisphere_heitz(u1, u2, wi_std, ti_out);
    if (method == 0 && ti_out) *ti_out = NAN;
    /* warp back to the ellipsoid configuration with M^-T */
    v3 wm = normalize(mk(wm_std.x * ax, wm_std.y * ay, wm_std.z));
    h_out[0] = s * wm.x; h_out[1] = s * wm.y; h_out[2] = s * wm.z;
}

/* NEXT-3: the paper's NATIVE handling of incidence below the horizon (Fig. 4,
 * theta_i = 130 deg): Listing 1 + Listing 3 (or 2) applied as
 * printed to any wi with wi_std.z > -1 -- no flip.  The cap is (-ws.z, 1],
 * which for ws.z < 0 lies above z = |ws.z|.
 * Evaluated in binary128 (__float128): with wi nearly straight below and small
 * alpha, ws.z = -1 + 1e-8 and Listing 3's h.z = z + wi.z is a
 * difference of two numbers within 1e-15 of 1 -- beyond binary64, not beyond
 * binary128 (reading R17).  Same literal steps as above. */
typedef __float128 q128;
void orc_sample_vndf_native(int method, const double wi_in[3], double ax_d, double ay_d,
                            double u1_d, double u2_d, double h_out[3])
{
    if (method != 0) {  /* Listing 2 needs no extra precision here (tests compare distributions) */
        v3 wi = mk(wi_in[0], wi_in[1], wi_in[2]);
        v3 wi_std = normalize(mk(wi.x * ax_d, wi.y * ay_d, wi.z));
        v3 wm_std = hemisphere_heitz(u1_d, u2_d, wi_std, NULL);
        v3 wm = normalize(mk(wm_std.x * ax_d, wm_std.y * ay_d, wm_std.z));
        h_out[0] = wm.x; h_out[1] = wm.y; h_out[2] = wm.z;
        return;
    }
    const q128 PI = M_PIq;
    q128 ax = ax_d, ay = ay_d, u1 = u1_d, u2 = u2_d;
    /* warp to the hemisphere configuration */
    q128 tx = wi_in[0] * ax, ty = wi_in[1] * ay, tz = wi_in[2];
    q128 L = sqrtq(tx * tx + ty * ty + tz * tz);
    q128 wx = tx / L, wy = ty / L, wz = tz / L;
    /* Listing 3 */
    q128 phi = 2 * PI * u1;
    q128 z = fmaq(1 - u2, 1 + wz, -wz);
    q128 st2 = 1 - z * z;
    if (st2 < 0) st2 = 0;
    if (st2 > 1) st2 = 1;
    q128 st = sqrtq(st2);
    q128 hx = st * cosq(phi) + wx, hy = st * sinq(phi) + wy, hz = z + wz;
    /* warp back with M^-T */
    q128 mx = hx * ax, my = hy * ay, mz = hz;
    q128 N = sqrtq(mx * mx + my * my + mz * mz);
    h_out[0] = (double)(mx / N); h_out[1] = (double)(my / N); h_out[2] = (double)(mz / N);
}

/* ------------------------------------------------------------------------ */
/* VNDF pdf, Eq. 1-4, written as defined.                      */
/* ------------------------------------------------------------------------ */
double orc_sigma_std(double zi) { return (1.0 + zi) / 2.0; }          /* Eq. 4 */
double orc_D_std(double zm) { return zm > 0.0 ? 1.0 / ORC_PI : 0.0; } /* Eq. 3 */

/* Eq. 2: D_vis,std(wm, wi) = max(wm.wi, 0) D_std(wm) / sigma_std(wi) */
double orc_Dvis_std(const double wm[3], const double wi[3])
{
    v3 m = mk(wm[0], wm[1], wm[2]), i = mk(wi[0], wi[1], wi[2]);
    return fmax(dot(m, i), 0.0) * orc_D_std(m.z) / orc_sigma_std(i.z);
}

/* Eq. 1 for wi with wi.z >= 0:
 *   D_vis(wm, wi) = D_vis,std(M^T wm/|M^T wm|, M^-1 wi/|M^-1 wi|)
 *                   * |det M^T| / |M^T wm|^3,
 * M^T = diag(1/ax, 1/ay, 1), M^-1 = diag(ax, ay, 1), |det M^T| = 1/(ax ay). */
static double vndf_pdf_upper(v3 wm, v3 wi, double ax, double ay)
{
    v3 MTwm = mk(wm.x / ax, wm.y / ay, wm.z);
    v3 Miwi = mk(wi.x * ax, wi.y * ay, wi.z);
    double nMT = len(MTwm);
    v3 a = scale(MTwm, 1.0 / nMT), b = normalize(Miwi);
    double A[3] = {a.x, a.y, a.z}, B[3] = {b.x, b.y, b.z};
    double detMT = 1.0 / (ax * ay);
    return orc_Dvis_std(A, B) * fabs(detMT) / (nMT * nMT * nMT);
}

/* pdf(h | wi) with reading R4 (flip) */
double orc_pdf_vndf(const double h[3], const double wi[3], double ax, double ay)
{
    double s = (wi[2] < 0.0) ? -1.0 : 1.0;
    return vndf_pdf_upper(mk(s * h[0], s * h[1], s * h[2]),
                          mk(s * wi[0], s * wi[1], s * wi[2]), ax, ay);
}

/* Eq. 1 as defined for any wi (no flip): sigma_std(z_i) = (1 + z_i)/2 holds
 * on [-1, 1] (Eq. 4) -- the native below-horizon pdf (NEXT-3). */
double orc_pdf_vndf_native(const double h[3], const double wi[3], double ax, double ay)
{
    return vndf_pdf_upper(mk(h[0], h[1], h[2]), mk(wi[0], wi[1], wi[2]), ax, ay);
}

/* Eq. 12: GGX NDF D(wm) = D_std(M^T wm/|.|) |det M^T| / |M^T wm|^4 */
double orc_D_ggx(const double wm[3], double ax, double ay)
{
    v3 MTwm = mk(wm[0] / ax, wm[1] / ay, wm[2]);
    double n = len(MTwm);
    return orc_D_std(MTwm.z / n) * (1.0 / (ax * ay)) / (n * n * n * n);
}

/* Eq. 16-17: G1(wm, wi) = G1,std(M^T wm/|.|, M^-1 wi/|.|),
 * G1,std = chi+(wi.wm) z_i / sigma_std(wi)   (arguments in std space) */
double orc_G1(const double wm[3], const double wi[3], double ax, double ay)
{
    v3 m = normalize(mk(wm[0] / ax, wm[1] / ay, wm[2]));
    v3 i = normalize(mk(wi[0] * ax, wi[1] * ay, wi[2]));
    double chi = dot(i, m) > 0.0 ? 1.0 : 0.0;
    return chi * i.z / orc_sigma_std(i.z);
}

/* The north-star form G1(wi) max(0, wi.h) D(h) / wi.z (BASELINE north_star;
 * Heitz 2014 definition of the VNDF; Eq. 12 and Eq. 16-17).  Needs wi.z != 0.
 * Flip reading R4 applied.  Used to cross-check Eq. 1. */
double orc_pdf_vndf_g1d(const double h[3], const double wi[3], double ax, double ay)
{
    double s = (wi[2] < 0.0) ? -1.0 : 1.0;
    double hh[3] = {s * h[0], s * h[1], s * h[2]};
    double ww[3] = {s * wi[0], s * wi[1], s * wi[2]};
    double wdoth = ww[0] * hh[0] + ww[1] * hh[1] + ww[2] * hh[2];
    return orc_G1(hh, ww, ax, ay) * fmax(0.0, wdoth) * orc_D_ggx(hh, ax, ay) / ww[2];
}

/* ------------------------------------------------------------------------ */
/* Reflection machinery of the proof (section 3.2).                         */
/* ------------------------------------------------------------------------ */
/* Eq. 5: wo = 2 (wm.wi) wm - wi */
void orc_reflect(const double wi[3], const double wm[3], double wo[3])
{
    double d = wm[0] * wi[0] + wm[1] * wi[1] + wm[2] * wi[2];
    for (int k = 0; k < 3; ++k) wo[k] = 2.0 * d * wm[k] - wi[k];
}
/* Eq. 6: wh = (wi + wo) / |wi + wo| */
void orc_half_vector(const double wi[3], const double wo[3], double wh[3])
{
    v3 h = normalize(mk(wi[0] + wo[0], wi[1] + wo[1], wi[2] + wo[2]));
    wh[0] = h.x; wh[1] = h.y; wh[2] = h.z;
}
/* Eq. 8: |d wh / d wo| = 1 / (4 |wo.wh|) */
double orc_reflect_jacobian(const double wo[3], const double wh[3])
{
    return 1.0 / (4.0 * fabs(wo[0] * wh[0] + wo[1] * wh[1] + wo[2] * wh[2]));
}
/* Eq. 10: f_p(wo, wi) = 1/(2 pi (1 + z_i)) if z_h > 0, else 0 */
double orc_cap_density(const double wo[3], const double wi[3])
{
    double hz = wi[2] + wo[2];  /* z of the (unnormalised) half vector */
    double n = sqrt((wi[0] + wo[0]) * (wi[0] + wo[0]) +
                    (wi[1] + wo[1]) * (wi[1] + wo[1]) + hz * hz);
    if (!(n > 0.0) || !(hz / n > 0.0)) return 0.0;
    return 1.0 / (2.0 * ORC_PI * (1.0 + wi[2]));
}

/* ------------------------------------------------------------------------ */
/* Brute-force ray-cast sampler from the DEFINITION of the VNDF (*/
/* Fig. 2): the normals where parallel rays (direction -wi) first hit the   */
/* ellipsoid M * (unit upper hemisphere), M = diag(1/ax, 1/ay, 1)           */
/* (P:363-380).  Rays start on a disk perpendicular to wi that covers the   */
/* ellipsoid's projection; a ray that misses, or first hits the ellipsoid   */
/* below z = 0 (the truncated part), is rejected.  The normal of the surface */
/* ax^2 x^2 + ay^2 y^2 + z^2 = 1 at P is normalize(ax^2 P.x, ay^2 P.y, P.z). */
/* Randomness: Philox block (trial, 2) of `seed` (independent of the u's).  */
/* Returns the number of trials used.                                       */
/* ------------------------------------------------------------------------ */
static uint64_t raycast(int flip, const double wi_in[3], double ax, double ay,
                        uint64_t seed, uint64_t first_trial, double h_out[3])
{
    double s = (flip && wi_in[2] < 0.0) ? -1.0 : 1.0;
    v3 wi = normalize(mk(s * wi_in[0], s * wi_in[1], s * wi_in[2]));
    /* orthonormal basis e1, e2 perpendicular to wi */
    v3 helper = fabs(wi.z) < 0.9 ? mk(0, 0, 1) : mk(1, 0, 0);
    v3 e1 = normalize(cross(helper, wi));
    v3 e2 = cross(wi, e1);
    double R = fmax(fmax(1.0 / ax, 1.0 / ay), 1.0);   /* bounding radius */
    for (uint64_t trial = first_trial;; ++trial) {
        uint32_t w[4];
        orc_philox_block(seed, trial, 2u, w);
        /* uniform point on the disk of radius R by rejection from the square */
        double d1 = (2.0 * ((double)w[0] * (1.0 / 4294967296.0)) - 1.0) * R;
        double d2 = (2.0 * ((double)w[1] * (1.0 / 4294967296.0)) - 1.0) * R;
        if (d1 * d1 + d2 * d2 > R * R) continue;
        v3 o = add(scale(e1, d1), scale(e2, d2));
        /* ray p(t) = o - t wi; solve |A p|^2 = 1 with A = diag(ax, ay, 1) */
        v3 Ao = mk(ax * o.x, ay * o.y, o.z), Aw = mk(ax * wi.x, ay * wi.y, wi.z);
        double qa = dot(Aw, Aw), qb = -2.0 * dot(Ao, Aw), qc = dot(Ao, Ao) - 1.0;
        double disc = qb * qb - 4.0 * qa * qc;
        if (disc < 0.0) continue;                       /* miss */
        double t = (-qb - sqrt(disc)) / (2.0 * qa);     /* first hit along -wi */
        v3 P = add(o, scale(wi, -t));
        if (P.z < 0.0) continue;                        /* truncated half */
        v3 n = normalize(mk(ax * ax * P.x, ay * ay * P.y, P.z));
        h_out[0] = s * n.x; h_out[1] = s * n.y; h_out[2] = s * n.z;
        return trial - first_trial + 1;
    }
}

uint64_t orc_sample_raycast(const double wi_in[3], double ax, double ay,
                            uint64_t seed, uint64_t first_trial, double h_out[3])
{
    return raycast(1, wi_in, ax, ay, seed, first_trial, h_out);
}

/* Native (no flip): rays travel along -wi even when wi points below the
 * horizon; a ray counts if its first hit on the full ellipsoid is on the kept
 * upper half (P:353-358 definition, NEXT-3). */
uint64_t orc_batch_raycast_native(const double wi[3], double ax, double ay, uint64_t seed,
                                  int64_t n, double *hx, double *hy, double *hz)
{
    uint64_t trial = 0;
    for (int64_t k = 0; k < n; ++k) {
        double h[3];
        trial += raycast(0, wi, ax, ay, seed, trial, h);
        hx[k] = h[0]; hy[k] = h[1]; hz[k] = h[2];
    }
    return trial;
}

void orc_batch_pdf_native(int64_t n, const double *hx, const double *hy, const double *hz,
                          const double wi[3], double ax, double ay, double *out)
{
    for (int64_t k = 0; k < n; ++k) {
        double h[3] = {hx[k], hy[k], hz[k]};
        out[k] = orc_pdf_vndf_native(h, wi, ax, ay);
    }
}

void orc_batch_sample_native(int method, int64_t n, const float *wx, const float *wy,
                             const float *wz, const float *ax, const float *ay,
                             const float *u1, const float *u2, double *hx, double *hy,
                             double *hz, double *pdf)
{
    for (int64_t k = 0; k < n; ++k) {
        double wi[3] = {wx[k], wy[k], wz[k]}, h[3];
        orc_sample_vndf_native(method, wi, ax[k], ay[k], u1[k], u2[k], h);
        hx[k] = h[0]; hy[k] = h[1]; hz[k] = h[2];
        if (pdf) pdf[k] = orc_pdf_vndf_native(h, wi, ax[k], ay[k]);
    }
}

/* ------------------------------------------------------------------------ */
/* Config-4 input recipe (DESIGN.md s.5 reading R12), in  */
/* float64 from the exact integers of TWO Philox blocks per sample --       */
/* "key=seed, counter=sample index" (BASELINE.json config 4):               */
/*   X = Philox(counter (i_lo, i_hi, 0, 0), key (seed_lo, seed_hi))          */
/*   Y = Philox(counter (i_lo, i_hi, 1, 0), key (seed_lo, seed_hi))          */
/*   wi uniform on the upper hemisphere (A12 / R16):                        */
/*      ua = u(X0), z = 1 - ua, r = sqrt(ua (2 - ua)), phi = 2 pi u(X1)     */
/*   ax = 0.01 * 100^u(X2), ay = 0.01 * 100^u(X3)   (log-uniform [0.01, 1]) */
/*   u1 = u(Y0), u2 = u(Y1)                  (the method's uniforms) */
/* Every uniform carries 24 bits (u(w) = (w >> 8) 2^-24).                   */
/* ------------------------------------------------------------------------ */
void orc_c4_inputs(uint64_t seed, uint64_t index, double out[7])
{
    uint32_t X[4], Y[4];
    orc_philox_block(seed, index, 0u, X);
    orc_philox_block(seed, index, 1u, Y);
    double ua = orc_u01(X[0]);
    double z = 1.0 - ua;
    double r = sqrt(ua * (2.0 - ua));
    double phi = 2.0 * ORC_PI * orc_u01(X[1]);
    out[0] = r * cos(phi);
    out[1] = r * sin(phi);
    out[2] = z;
    out[3] = 0.01 * pow(100.0, orc_u01(X[2]));
    out[4] = 0.01 * pow(100.0, orc_u01(X[3]));
    out[5] = orc_u01(Y[0]);
    out[6] = orc_u01(Y[1]);
}

/* The recipe over an index list: out7[7k .. 7k+6] (tests: distribution pins). */
void orc_batch_c4_inputs(uint64_t seed, int64_t n, const uint64_t *indices, double *out7)
{
    for (int64_t k = 0; k < n; ++k) orc_c4_inputs(seed, indices[k], out7 + 7 * k);
}

/* ------------------------------------------------------------------------ */
/* NEXT-2: BRDF importance sampling with the VNDF (appendix).  */
/* Height-correlated Smith G2, Eq. 13-14:                       */
/*   G2 = Gi Go / (Gi + Go - Gi Go), Gk = G1(wm, wk) (Eq. 15-17).            */
/* ------------------------------------------------------------------------ */
double orc_G2(const double wm[3], const double wi[3], const double wo[3], double ax, double ay)
{
    double gi = orc_G1(wm, wi, ax, ay), go = orc_G1(wm, wo, ax, ay);
    double den = gi + go - gi * go;
    return den > 0.0 ? gi * go / den : 0.0;
}

/* Eq. 11 times cos(theta_o), with F = 1 (the Fresnel term is not
 * defined by the paper; reading in DESIGN.md s.3): for wi.z > 0,
 *   f_r |cos theta_o| = G2(wh, wi, wo) D(wh) / (4 cos theta_i), wo.z > 0,
 * 0 below the horizon (reflection only). wh = half vector (Eq. 6). */
double orc_brdf_cos(const double wi[3], const double wo[3], double ax, double ay)
{
    if (!(wo[2] > 0.0) || !(wi[2] > 0.0)) return 0.0;
    double wh[3];
    orc_half_vector(wi, wo, wh);
    return orc_G2(wh, wi, wo, ax, ay) * orc_D_ggx(wh, ax, ay) / (4.0 * wi[2]);
}

/* Eq. 20: PDF(wb, wa) = G1(wm, wa) D(wm) / (4 cos theta_a), with
 * wm the half vector of (wa, wb), wa.z > 0. */
double orc_pdf_reflect(const double wa[3], const double wb[3], double ax, double ay)
{
    double wm[3];
    orc_half_vector(wa, wb, wm);
    double d = wm[0] * wa[0] + wm[1] * wa[1] + wm[2] * wa[2];
    if (!(d > 0.0)) return 0.0;
    return orc_G1(wm, wa, ax, ay) * orc_D_ggx(wm, ax, ay) / (4.0 * wa[2]);
}

/* The appendix's two sampling steps, with reading R4 for
 * wa.z < 0: (1) wm by Listing 1 (method 0 cap, 1 Heitz); (2) wb = reflect(wa,
 * wm) (Eq. 5).  out = (wb.xyz, PDF Eq. 20, weight = f_r |cos theta_b| / PDF
 * (= G2/G1 analytically)), evaluated in the upper frame s*wa. */
void orc_sample_reflect(int method, const double wa_in[3], double ax, double ay, double u1,
                        double u2, double out[5])
{
    double s = (wa_in[2] < 0.0) ? -1.0 : 1.0;
    double n = sqrt(wa_in[0] * wa_in[0] + wa_in[1] * wa_in[1] + wa_in[2] * wa_in[2]);
    double wa[3] = {s * wa_in[0] / n, s * wa_in[1] / n, s * wa_in[2] / n};
    double wm[3], wb[3];
    orc_sample_vndf(method, wa, ax, ay, u1, u2, wm, NULL);      /* step (1) */
    orc_reflect(wa, wm, wb);                                    /* step (2), Eq. 5 */
    double pdf = orc_pdf_reflect(wa, wb, ax, ay);               /* Eq. 20 */
    out[0] = s * wb[0]; out[1] = s * wb[1]; out[2] = s * wb[2];
    out[3] = pdf;
    out[4] = pdf > 0.0 ? orc_brdf_cos(wa, wb, ax, ay) / pdf : 0.0;  /* Eq. 19 summand, L = 1 */
}

void orc_batch_sample_reflect(int method, int64_t n, const float *wx, const float *wy,
                              const float *wz, const float *ax, const float *ay,
                              const float *u1, const float *u2, double *out5)
{
    for (int64_t k = 0; k < n; ++k) {
        double wa[3] = {wx[k], wy[k], wz[k]};
        orc_sample_reflect(method, wa, ax[k], ay[k], u1[k], u2[k], out5 + 5 * k);
    }
}

/* Fixed wa, alpha; arrays of wb (quadrature helpers for the pins). */
void orc_batch_pdf_reflect(int64_t n, const double wa[3], double ax, double ay, const double *bx,
                           const double *by, const double *bz, double *out)
{
    for (int64_t k = 0; k < n; ++k) {
        double wb[3] = {bx[k], by[k], bz[k]};
        out[k] = orc_pdf_reflect(wa, wb, ax, ay);
    }
}

void orc_batch_brdf_cos(int64_t n, const double wa[3], double ax, double ay, const double *bx,
                        const double *by, const double *bz, double *out)
{
    for (int64_t k = 0; k < n; ++k) {
        double wb[3] = {bx[k], by[k], bz[k]};
        out[k] = orc_brdf_cos(wa, wb, ax, ay);
    }
}

/* White-furnace Monte Carlo estimator, Eq. 19 with L = 1:
 * I = (1/N) sum_j f_r |cos| / PDF over N reflection samples of a fixed
 * (wa, alpha); sample j uses u1 = u(W0), u2 = u(W1) of the Philox block
 * (counter j, key seed).  Returns sum and sum of squares of the summands. */
void orc_furnace(int method, const double wa[3], double ax, double ay, uint64_t seed,
                 uint64_t first, int64_t n, double out2[2])
{
    double sum = 0.0, sq = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        uint32_t W[4];
        orc_philox_block(seed, first + (uint64_t)j, 0u, W);
        double r[5];
        orc_sample_reflect(method, wa, ax, ay, orc_u01(W[0]), orc_u01(W[1]), r);
        sum += r[4];
        sq += r[4] * r[4];
    }
    out2[0] = sum;
    out2[1] = sq;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1 sampler-only microbenchmark (the paper's GPU methodology: */
/* Listing 1 called `iters` times per lane), replayed for lane t: inputs of  */
/* the config-4 recipe of index t; iteration k: u1 = u(Y0 + k A1), u2 =      */
/* u(Y1 + k A2) (32-bit wrap; Y = Philox block 1, whose words give u1, u2 of  */
/* the recipe); h by the chosen listing in float64 from the                  */
/* CURRENT fp32 incidence; checksum += h.x + 2 h.y + 3 h.z; then the fp32    */
/* rotation of (wi.x, wi.y) about z with single roundings (vndf.h):          */
/* x' = fmaf(c, x, -(s*y)), y' = fmaf(c, y, s*x).  The incidence sequence is */
/* fp32 by definition of the benchmark; the method arithmetic is float64.    */
/* method: 0 = cap, 1 = Heitz, 2 = cap (Listing 3 literal: same math).       */
/* trace (nullable): receives h of every call, trace[3k .. 3k+2].           */
/* ------------------------------------------------------------------------ */
static double microbench_lane(int method, uint64_t seed, uint64_t lane, int iters, double *trace)
{
    double in[7];
    orc_c4_inputs(seed, lane, in);
    uint32_t Y[4];
    orc_philox_block(seed, lane, 1u, Y);
    uint32_t x1 = Y[0], x2 = Y[1];
    float wx = (float)in[0], wy = (float)in[1], wz = (float)in[2];
    double ax = (double)(float)in[3], ay = (double)(float)in[4];
    const float c = 0.764842187f, s = 0.644217687f;
    double acc = 0.0;
    for (int k = 0; k < iters; ++k) {
        double wi[3] = {wx, wy, wz}, h[3];
        orc_sample_vndf(method == 1 ? 1 : 0, wi, ax, ay, orc_u01(x1), orc_u01(x2), h, NULL);
        if (trace) {
            trace[3 * k] = h[0];
            trace[3 * k + 1] = h[1];
            trace[3 * k + 2] = h[2];
        }
        acc += h[0] + 2.0 * h[1] + 3.0 * h[2];
        x1 += 0x9E3779B9u;
        x2 += 0x7F4A7C15u;
        float sy = s * wy, sx = s * wx;
        float rx = fmaf(c, wx, -sy);
        float ry = fmaf(c, wy, sx);
        wx = rx;
        wy = ry;
    }
    return acc;
}

double orc_microbench_lane(int method, uint64_t seed, uint64_t lane, int iters)
{
    return microbench_lane(method, seed, lane, iters, NULL);
}

void orc_batch_microbench(int method, uint64_t seed, int64_t lanes, int iters, double *out)
{
    for (int64_t t = 0; t < lanes; ++t) out[t] = orc_microbench_lane(method, seed, (uint64_t)t, iters);
}

/* Per-call h of lanes [0, lanes): trace[(t iters + k) 3 + c]. */
void orc_batch_microbench_trace(int method, uint64_t seed, int64_t lanes, int iters, double *trace)
{
    for (int64_t t = 0; t < lanes; ++t)
        microbench_lane(method, seed, (uint64_t)t, iters, trace + (size_t)t * (size_t)iters * 3u);
}

/* ------------------------------------------------------------------------ */
/* Batched drivers (std::thread-like partition over contiguous ranges).     */
/* ------------------------------------------------------------------------ */
typedef struct {
    int method;
    int64_t lo, hi;
    /* streamed inputs (fp32 planes) or Philox (seed + index list) */
    const float *wx, *wy, *wz, *ax, *ay, *u1, *u2;
    uint64_t seed;
    const uint64_t *idx;
    double *hx, *hy, *hz, *pdf, *aux;
    double *out5; /* non-NULL: reflection outputs (orc_sample_reflect) instead of h */
} job_t;

static void run_one(const job_t *j, int64_t k)
{
    double wi[3], a_x, a_y, u1, u2, h[3], ti;
    if (j->idx) {
        double in[7];
        orc_c4_inputs(j->seed, j->idx[k], in);
        wi[0] = in[0]; wi[1] = in[1]; wi[2] = in[2];
        a_x = in[3]; a_y = in[4]; u1 = in[5]; u2 = in[6];
    } else {
        wi[0] = j->wx[k]; wi[1] = j->wy[k]; wi[2] = j->wz[k];
        a_x = j->ax[k]; a_y = j->ay[k]; u1 = j->u1[k]; u2 = j->u2[k];
    }
    if (j->out5) {
        orc_sample_reflect(j->method, wi, a_x, a_y, u1, u2, j->out5 + 5 * k);
        return;
    }
    orc_sample_vndf(j->method, wi, a_x, a_y, u1, u2, h, &ti);
    j->hx[k] = h[0]; j->hy[k] = h[1]; j->hz[k] = h[2];
    if (j->pdf) j->pdf[k] = orc_pdf_vndf(h, wi, a_x, a_y);
    if (j->aux) j->aux[k] = ti;
}

static void *run_range(void *arg)
{
    const job_t *j = (const job_t *)arg;
    for (int64_t k = j->lo; k < j->hi; ++k) run_one(j, k);
    return NULL;
}

static void run_parallel(job_t base, int64_t n, int threads)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if ((int64_t)threads > n) threads = (int)(n > 0 ? n : 1);
    pthread_t tid[256];
    job_t jobs[256];
    int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = base;
        jobs[t].lo = (int64_t)t * chunk;
        jobs[t].hi = jobs[t].lo + chunk < n ? jobs[t].lo + chunk : n;
        if (jobs[t].lo > n) jobs[t].lo = n;
    }
    if (threads == 1) { run_range(&jobs[0]); return; }
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, run_range, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* Streamed inputs: n samples from fp32 SoA planes.  pdf / aux may be NULL.
 * aux receives Listing 2's ti (method 1) or NaN (method 0). */
void orc_batch_sample(int method, int64_t n,
                      const float *wx, const float *wy, const float *wz,
                      const float *ax, const float *ay,
                      const float *u1, const float *u2,
                      double *hx, double *hy, double *hz, double *pdf,
                      double *aux, int threads)
{
    job_t b;
    memset(&b, 0, sizeof b);
    b.method = method;
    b.wx = wx; b.wy = wy; b.wz = wz; b.ax = ax; b.ay = ay; b.u1 = u1; b.u2 = u2;
    b.hx = hx; b.hy = hy; b.hz = hz; b.pdf = pdf; b.aux = aux;
    run_parallel(b, n, threads);
}

/* Config-4 (Philox) samples at an explicit list of global indices. */
void orc_batch_sample_philox(int method, uint64_t seed, int64_t n,
                             const uint64_t *indices,
                             double *hx, double *hy, double *hz, double *pdf,
                             double *aux, int threads)
{
    job_t b;
    memset(&b, 0, sizeof b);
    b.method = method; b.seed = seed; b.idx = indices;
    b.hx = hx; b.hy = hy; b.hz = hz; b.pdf = pdf; b.aux = aux;
    run_parallel(b, n, threads);
}

/* Reflection sampling (orc_sample_reflect) on config-4 (Philox) inputs at an
 * explicit list of global indices: out5[5k .. 5k+4] = wo.xyz, pdf, weight. */
void orc_batch_sample_reflect_philox(int method, uint64_t seed, int64_t n, const uint64_t *indices,
                                     double *out5, int threads)
{
    job_t b;
    memset(&b, 0, sizeof b);
    b.method = method; b.seed = seed; b.idx = indices; b.out5 = out5;
    run_parallel(b, n, threads);
}

/* Eq. 1 pdf over arrays (float64 directions, fp32 roughness/incidence). */
void orc_batch_pdf(int64_t n, const double *hx, const double *hy, const double *hz,
                   const double *wx, const double *wy, const double *wz,
                   const double *ax, const double *ay, double *pdf)
{
    for (int64_t k = 0; k < n; ++k) {
        double h[3] = {hx[k], hy[k], hz[k]}, wi[3] = {wx[k], wy[k], wz[k]};
        pdf[k] = orc_pdf_vndf(h, wi, ax[k], ay[k]);
    }
}

/* Raw Philox words of block `block` for an index list (4 words per index). */
void orc_batch_philox_words(uint64_t seed, int64_t n, const uint64_t *indices,
                            uint32_t block, uint32_t *words)
{
    for (int64_t k = 0; k < n; ++k) orc_philox_block(seed, indices[k], block, words + 4 * k);
}

/* Brute-force samples for a fixed (wi, alpha): n samples, trials counted. */
uint64_t orc_batch_raycast(const double wi[3], double ax, double ay, uint64_t seed,
                           int64_t n, double *hx, double *hy, double *hz)
{
    uint64_t trial = 0;
    for (int64_t k = 0; k < n; ++k) {
        double h[3];
        trial += orc_sample_raycast(wi, ax, ay, seed, trial, h);
        hx[k] = h[0]; hy[k] = h[1]; hz[k] = h[2];
    }
    return trial;
}
