/*
 * vndf.h -- C ABI of libvndf: batched GGX visible-normal (VNDF) sampling by
 * the spherical-cap construction of arXiv 2306.05044, on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source.
 *
 * The operation (per sample k, all fp32, SoA planes):
 *   inputs  wi_k = (wi_x, wi_y, wi_z)[k]  incident direction, need not be unit
 *                                          (Listing 1 normalises after the
 *                                          stretch)
 *           alpha_x[k], alpha_y[k] > 0     GGX roughness, M^-1 = diag(ax, ay, 1)
 *
 *           u1[k], u2[k] in [0, 1)         two uniforms
 *   outputs h_k = (h_x, h_y, h_z)[k]       unit visible normal, distributed as
 *                                          the VNDF D_vis(h, wi) of Eq. 1
 *           pdf[k]                         D_vis(h_k, wi_k), Eq. 1
 *                                          = G1(wi) max(0, wi.h) D(h) / wi.z
 *                                          (Eq. 12, 16-17)
 *   method  Listing 1 around Listing 3 (spherical cap:
 *           phi = 2 pi u1, z uniform on (-wi_std.z, 1] from u2, h_std = c +
 *           wi_std, normalised after the unstretch), or around
 *           Listing 2 (Heitz 2018 cross section) for the baseline.
 *   below-horizon incidence (wi.z < 0; -0.0 counts as upper): sampled on the
 *           flipped hemisphere, h = s * sample(s * wi), s = -1, and
 *           pdf(h | wi) = pdf(s h | s wi)   (reading R4).
 *
 * Accuracy contract (BASELINE.json north_star): against the float64 oracle on
 * identical inputs, max |dh| <= 2e-5 per component and |dpdf|/pdf <= 1e-4 for
 * the spherical-cap entry points, on every sample in the domain alpha in
 * [1e-3, 1], |wi| in [0.5, 2], u in [0, 1).  Ill-conditioned samples are
 * detected in-kernel and recomputed in float64.  The
 * Heitz baseline is the literal fp32 Listing 2 and carries no such guarantee.
 *
 * Ownership and behaviour (all entry points):
 *   - Every pointer argument of the sampling calls is a CUDA DEVICE pointer
 *     (except the *_host call), owned by the caller; the library never frees
 *     or retains it.  Buffers hold n fp32 elements (words: 4n uint32).
 *   - Any 4-byte aligned pointer is accepted.  When all planes of a call are
 *     32-byte aligned a 256-bit vector path runs, 16-byte aligned a 128-bit
 *     path, otherwise a scalar path; results are identical.
 *   - Calls only ENQUEUE work on `stream` (NULL = legacy default stream) and
 *     return; outputs are valid once the caller synchronises the stream.
 *     The *_host call is the exception: it is blocking.
 *   - The device calls never synchronise and never copy host data, so every
 *     device call, including the first one in the process, can be captured
 *     into a CUDA graph (stream capture).  (The very first libvndf call of a
 *     process starts the CUDA runtime inside the library, which waits for
 *     work already queued on the device; vndf_init does that up front.)  Replays recompute from the captured
 *     buffers.  The device a call runs on is the device of `stream` (the
 *     current device for the NULL stream); all its buffers must live there.
 *   - Thread-safe.  Global state, per device, created on first use and kept
 *     for the life of the process: cached device attributes and launch
 *     configurations, a private stream-ordered memory pool for transient
 *     fix-up queues (released with vndf_release_host_staging), and the host
 *     entry points' staging area (see vndf_release_host_staging).
 *   - Outputs are a pure function of the inputs (of seed and global index for
 *     the Philox calls): independent of grid, stream, vector path or chunking.
 *
 * Errors:
 *   n == 0                         -> VNDF_OK, nothing enqueued
 *   n < 0, required pointer NULL,  -> VNDF_ERR_INVALID_ARGUMENT, nothing
 *   an output aliasing an input      enqueued
 *   or another output, pointer not
 *   4-byte aligned
 *   CUDA launch / runtime failure  -> VNDF_ERR_CUDA; vndf_last_cuda_error()
 *                                     returns the cudaError_t (thread-local)
 *   Outside the per-sample domain the result is unspecified but never traps.
 */
#ifndef VNDF_H_
#define VNDF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same type as cudaStream_t / CUstream; NULL is the legacy default stream. */
typedef struct CUstream_st *vndf_stream_t;

typedef enum {
    VNDF_OK = 0,
    VNDF_ERR_INVALID_ARGUMENT = 1,
    VNDF_ERR_CUDA = 2,
    VNDF_ERR_NOT_IMPLEMENTED = 3
} vndf_status;

/* Spherical-cap sampling, h only (BASELINE config 3: 28 B in, 12 B out per
 * sample).  Listing 1 + Listing 3. */
vndf_status vndf_sample_cap(const float *wi_x, const float *wi_y, const float *wi_z,
                            const float *alpha_x, const float *alpha_y,
                            const float *u1, const float *u2,
                            float *h_x, float *h_y, float *h_z,
                            int64_t n, vndf_stream_t stream);

/* Spherical-cap sampling plus the VNDF pdf of each sample, Eq. 1
 * (BASELINE configs 1, 2, 5: 28 B in, 16 B out per sample). */
vndf_status vndf_sample_cap_pdf(const float *wi_x, const float *wi_y, const float *wi_z,
                                const float *alpha_x, const float *alpha_y,
                                const float *u1, const float *u2,
                                float *h_x, float *h_y, float *h_z, float *pdf,
                                int64_t n, vndf_stream_t stream);

/* The paper's NATIVE handling of incidence below the horizon (NEXT-3; Fig. 4,
 * theta_i = 130 deg): Listing 1 + Listing 3 applied as printed to
 * any wi (no flip), the cap being (-ws.z, 1]; h is always an upper-hemisphere
 * normal visible from wi, pdf = Eq. 1 with sigma_std = (1 + z_i)/2 (Eq. 4).
 * Identical to vndf_sample_cap_pdf for wi.z >= 0.  pdf may be NULL. */
vndf_status vndf_sample_cap_pdf_native(const float *wi_x, const float *wi_y, const float *wi_z,
                                       const float *alpha_x, const float *alpha_y,
                                       const float *u1, const float *u2,
                                       float *h_x, float *h_y, float *h_z, float *pdf,
                                       int64_t n, vndf_stream_t stream);

/* Same-harness baseline: Listing 1 around Heitz's cross-section sampler,
 * Listing 2, literal fp32.  pdf may be NULL (h only). */
vndf_status vndf_sample_heitz2018(const float *wi_x, const float *wi_y, const float *wi_z,
                                  const float *alpha_x, const float *alpha_y,
                                  const float *u1, const float *u2,
                                  float *h_x, float *h_y, float *h_z, float *pdf,
                                  int64_t n, vndf_stream_t stream);

/* Fused in-kernel Philox4x32-10 (BASELINE config 4: key = seed, counter =
 * sample index).  Sample k of the call has global index
 * i = first_index + k (modulo 2^64) and TWO Philox blocks, key (seed_lo, seed_hi):
 *   X = Philox(counter (i_lo, i_hi, 0, 0)),  Y = Philox(counter (i_lo, i_hi, 1, 0));
 * with u(w) = (w >> 8) 2^-24 (24 bits):
 *   wi uniform on the upper hemisphere: z = 1 - u(X0), r = sqrt(u(X0) (2 - u(X0))),
 *      phi = 2 pi u(X1), wi = (r cos phi, r sin phi, z);
 *   alpha_x = 0.01 * 100^u(X2), alpha_y = 0.01 * 100^u(X3);
 *   u1 = u(Y0), u2 = u(Y1).
 * Outputs h and pdf (16 B per sample); pdf may be NULL. */
vndf_status vndf_sample_cap_philox(uint64_t seed, uint64_t first_index, int64_t n,
                                   float *h_x, float *h_y, float *h_z, float *pdf,
                                   vndf_stream_t stream);

/* Heitz-2018 baseline on the same Philox inputs. pdf may be NULL. */
vndf_status vndf_sample_heitz2018_philox(uint64_t seed, uint64_t first_index, int64_t n,
                                         float *h_x, float *h_y, float *h_z, float *pdf,
                                         vndf_stream_t stream);

/* Fused in-kernel Philox4x32-10 on BASELINE config 5's path-tracer edge mix
 * (north_star: the fused variant "evidenced by ... warp-divergence counters on
 * grazing and below-horizon inputs").  Same counters and key as
 * vndf_sample_cap_philox, u(w) = (w >> 8) 2^-24; the incidence category is
 * v = u(Y2): v < 0.4 grazing z = 1e-4 + u(X0) (0.05 - 1e-4); v < 0.6 back
 * side z = -(1 - u(X0)); else upper z = 1 - u(X0); phi = 2 pi u(X1),
 * r = sqrt(max((1 - z)(1 + z), 0)); alpha_x = T[X2 >> 30], alpha_y = T[X3 >> 30],
 * T = {1e-3, 0.05, 0.3, 1}; u1 = u(Y0), u2 = u(Y1), then Y3 bits 0-5 = 0 ->
 * u1 = 0, bits 6-11 = 0 -> u2 = 0, bits 12-17 = 0 -> u2 = 1 - 2^-24 (a later
 * rule wins).  These are, bit for bit, the fp32 inputs of the config-5
 * recipe (DESIGN.md s.5); back-side incidence is flipped (reading R4) and the
 * outputs equal vndf_sample_cap_pdf / vndf_sample_heitz2018 on those inputs.
 * Outputs h and pdf (16 B per sample); pdf may be NULL. */
vndf_status vndf_sample_cap_philox_edge(uint64_t seed, uint64_t first_index, int64_t n,
                                        float *h_x, float *h_y, float *h_z, float *pdf,
                                        vndf_stream_t stream);

/* Heitz-2018 baseline on the same config-5 Philox inputs. pdf may be NULL. */
vndf_status vndf_sample_heitz2018_philox_edge(uint64_t seed, uint64_t first_index, int64_t n,
                                              float *h_x, float *h_y, float *h_z, float *pdf,
                                              vndf_stream_t stream);

/* Raw Philox4x32-10 words of block `block` for global indices
 * first_index .. first_index + n - 1: words[4k .. 4k+3] (test / audit).
 * words: device pointer to 4n uint32, 16-byte aligned (one uint4 per index). */
vndf_status vndf_philox4x32_10(uint64_t seed, uint64_t first_index, int64_t n,
                               uint32_t block, uint32_t *words, vndf_stream_t stream);

/* End-to-end form of vndf_sample_cap_pdf on HOST buffers; pdf may be NULL
 * (h only: the end-to-end form of vndf_sample_cap, BASELINE config 3).
 * - If all eleven buffers are page-locked and mapped into the device's address
 *   space (cudaHostAlloc / cudaMallocHost / torch pin_memory(); mapped by
 *   default under unified addressing), the kernel reads the inputs and writes
 *   the outputs across the host link in place (zero-copy), on `stream`.
 * - Otherwise (pageable memory) the batch is streamed through the GPU in
 *   chunks of 2 Mi samples on three library-owned streams (copies from and
 *   to pageable memory are staged by the driver and complete synchronously,
 *   so chunks overlap little: pin the buffers for throughput).  Device staging
 *   (3 x 2 Mi x 44 B = 277 MB per device) is allocated on first use and kept
 *   for later calls; vndf_release_host_staging() frees it.
 * BLOCKING: returns when the outputs are in host memory.  Work is ordered
 * after prior work on `stream`.  Results are bit-identical to
 * vndf_sample_cap_pdf on the same inputs. */
vndf_status vndf_sample_cap_pdf_host(const float *wi_x, const float *wi_y, const float *wi_z,
                                     const float *alpha_x, const float *alpha_y,
                                     const float *u1, const float *u2,
                                     float *h_x, float *h_y, float *h_z, float *pdf,
                                     int64_t n, vndf_stream_t stream);

/* End-to-end form of vndf_sample_cap_philox (BASELINE config 4) writing HOST
 * buffers h_x, h_y, h_z, pdf (pdf may be NULL); the inputs are generated in
 * the kernel, so nothing crosses the link host -> device.  Chunks of 2 Mi
 * samples are computed into the device staging of vndf_sample_cap_pdf_host and
 * copied device -> host with cudaMemcpyAsync on three library streams, so with
 * page-locked outputs (cudaHostAlloc / torch pin_memory()) the DMA of chunk c
 * overlaps the kernel of chunk c + 1: 3.35 Gsamples/s = 0.99 of a plain
 * device -> host copy on the B200 box, where the SMs writing mapped pinned
 * memory directly (zero-copy) reached 3.16 (tools/e2e_c4_probe.py).  Pageable
 * outputs work too; their copies complete synchronously and do not overlap.
 * BLOCKING; ordered after prior work on `stream`; results bit-identical to
 * vndf_sample_cap_philox with the same seed and first_index. */
vndf_status vndf_sample_cap_philox_host(uint64_t seed, uint64_t first_index, int64_t n,
                                        float *h_x, float *h_y, float *h_z, float *pdf,
                                        vndf_stream_t stream);

/* Frees the cached staging of the host entry points on every device and
 * trims the library's fix-up-queue memory pools to zero (it waits for the
 * devices to go idle first).  VNDF_ERR_INVALID_ARGUMENT if a host call is in
 * flight on another thread. */
vndf_status vndf_release_host_staging(void);

/* Diagnostic: number of samples the spherical-cap kernels would route to the
 * float64 recomputation for these inputs; ADDS the count to *count (device
 * pointer to one uint64).  Does not write samples. */
vndf_status vndf_count_fixups(const float *wi_x, const float *wi_y, const float *wi_z,
                              const float *alpha_x, const float *alpha_y,
                              const float *u1, const float *u2,
                              int64_t n, uint64_t *count, vndf_stream_t stream);

/* Diagnostic: same for the fused Philox inputs. */
vndf_status vndf_count_fixups_philox(uint64_t seed, uint64_t first_index, int64_t n,
                                     uint64_t *count, vndf_stream_t stream);

/* BRDF importance sampling with the VNDF, the appendix's two steps
 * (P:1048-1055): (1) h by Listing 1 + Listing 3 (as vndf_sample_cap_pdf),
 * (2) wo = reflect(w, h) = 2 (w.h) h - w with w = wi/|wi| (Eq. 5).  Outputs
 * wo (3 planes), pdf = PDF(wo, w) of Eq. 20 = D_vis(h)/(4 w.h),
 * and weight = f_r |cos theta_o| / pdf = G2/G1 (Eq. 11 with F = 1, Eq. 13-17;
 * 0 when wo is below the horizon).  Below-horizon incidence: reading R4 (the
 * reflection stays on the incident side).  28 B in, 20 B out per sample.
 * Accuracy against the float64 oracle: |d wo| <= 6e-5 per component, pdf
 * relative 1e-4, |d weight| <= 1e-4 (DESIGN.md s.6.5). */
vndf_status vndf_sample_cap_reflect(const float *wi_x, const float *wi_y, const float *wi_z,
                                    const float *alpha_x, const float *alpha_y,
                                    const float *u1, const float *u2,
                                    float *wo_x, float *wo_y, float *wo_z, float *pdf, float *weight,
                                    int64_t n, vndf_stream_t stream);

/* Fused form of vndf_sample_cap_reflect on the config-4 inputs of
 * vndf_sample_cap_philox (wi, alpha_x, alpha_y, u1, u2 of sample j drawn from
 * the Philox block of counter first_index + j, key seed): no inputs read,
 * 20 B written per sample (wo.xyz, Eq. 20 pdf, G2/G1 weight).  All five
 * device pointers required, 4-byte aligned, non-overlapping.  Same accuracy
 * contract as vndf_sample_cap_reflect; ill-conditioned samples are recomputed
 * in float64 from the same Philox words (transient stream-ordered queue). */
vndf_status vndf_sample_cap_reflect_philox(uint64_t seed, uint64_t first_index, int64_t n,
                                           float *wo_x, float *wo_y, float *wo_z, float *pdf,
                                           float *weight, vndf_stream_t stream);

/* Heitz-2018 (Listing 2) baseline of vndf_sample_cap_reflect_philox on the
 * same inputs (literal fp32, no fix-up; for the speed ratio). */
vndf_status vndf_sample_heitz2018_reflect_philox(uint64_t seed, uint64_t first_index, int64_t n,
                                                 float *wo_x, float *wo_y, float *wo_z, float *pdf,
                                                 float *weight, vndf_stream_t stream);

/* The VNDF pdf alone, Eq. 1, at caller-provided directions (e.g.
 * for multiple-importance-sampling weights): pdf[k] = D_vis(h_k, wi_k)
 * with reading R4 for wi.z < 0; 0 for back-facing h or h below the (flipped)
 * horizon.  h and wi need not be unit (the pdf is scale invariant).  32 B in,
 * 4 B out per sample; relative accuracy 1e-4 against the float64 oracle at the
 * same fp32 inputs. */
vndf_status vndf_pdf(const float *h_x, const float *h_y, const float *h_z,
                     const float *wi_x, const float *wi_y, const float *wi_z,
                     const float *alpha_x, const float *alpha_y, float *pdf,
                     int64_t n, vndf_stream_t stream);

/* White-furnace Monte Carlo estimator, Eq. 19 with L = 1: for a
 * fixed incidence wi and roughness, sample j = first_index .. first_index+n-1
 * uses u1 = u(W0), u2 = u(W1) of the Philox block (counter j, key seed) and
 * contributes its weight f_r |cos| / PDF.  Writes sums[0] = sum of weights,
 * sums[1] = sum of squared weights (float64, DEVICE pointer); the estimate is
 * sums[0]/n, its variance sums[1]/n - (sums[0]/n)^2.  method 0 = spherical cap,
 * 1 = Heitz 2018.  Deterministic for a given device and n. */
vndf_status vndf_furnace(int method, float wi_x, float wi_y, float wi_z, float alpha_x, float alpha_y,
                         uint64_t seed, uint64_t first_index, int64_t n, double *sums,
                         vndf_stream_t stream);

/* Distribution audit (NEXT-3): n samples of a fixed (wi, alpha), u1 = u(W0),
 * u2 = u(W1) of the Philox block (counter j, key seed), binned on the device.
 * method: 0 = spherical cap (reading R4), 1 = Heitz 2018, 2 = cap, native
 * below-horizon handling.  mode 0: h in nt x nphi bins of (theta in [0, pi/2),
 * phi in [0, 2 pi)) (expected masses: Eq. 1); mode 1: the std-space reflected
 * direction c = reflect(ws, normalize(M^T h)) in bins of ((c.z + ws.z)/(1 + ws.z),
 * phi_c/(2 pi)) -- uniform by Eq. 10.  Counts are ADDED to
 * counts[nt * nphi] (device uint64), row-major in theta / z.  nt * nphi <= 8192.
 * Per-block partial counts are 32-bit: VNDF_ERR_INVALID_ARGUMENT if one block
 * would bin 2^32 or more samples (n above ~6e11 on a B200); split the call. */
vndf_status vndf_histogram(int method, int mode, float wi_x, float wi_y, float wi_z,
                           float alpha_x, float alpha_y, uint64_t seed, uint64_t first_index,
                           int64_t n, int nt, int nphi, uint64_t *counts, vndf_stream_t stream);

/* Sampler-only microbenchmark in the paper's GPU methodology (P:814-817:
 * "calls Listing 1 64 times per lane").  Lane t (0 <= t < lanes) draws wi and
 * (alpha_x, alpha_y) once from the config-4 recipe of index t (seed), then for
 * k = 0 .. iters-1 samples h with u1 = u(Y0 + k 0x9E3779B9), u2 = u(Y1 + k
 * 0x7F4A7C15) (32-bit wrap-around; Y = that lane's Philox block 1), adds
 * h.x + 2 h.y + 3 h.z to an fp32 checksum, and rotates wi about z:
 * (x, y) <- (fma(c, x, -(s y)), fma(c, y, s x)) with c = 0.764842187f,
 * s = 0.644217687f, every operation rounded to fp32 (so no call is
 * loop-invariant).  checksum[t] is written once per lane.
 * method: 0 = spherical cap (Listing 3, production fp32 arithmetic, no fix-up),
 *         1 = Heitz 2018 (Listing 2), 2 = Listing 3 taken literally.
 * No pdf.  checksum: device pointer to `lanes` floats. */
vndf_status vndf_microbench(int method, uint64_t seed, int64_t lanes, int iters, float *checksum,
                            vndf_stream_t stream);

/* vndf_microbench that also records every call (tests, element-wise parity of
 * NEXT-1): trace[4 (t iters + k) + c] = (h.x, h.y, h.z, flag) of call k of
 * lane t, flag = 1.0f when the spherical-cap conditioning test marks the call
 * (the production kernels would recompute it in float64; always 0 for methods
 * 1 and 2).  trace: device pointer to 4 lanes iters floats, 16-byte aligned;
 * checksum as for vndf_microbench (must not overlap trace). */
vndf_status vndf_microbench_trace(int method, uint64_t seed, int64_t lanes, int iters, float *checksum,
                                  float *trace, vndf_stream_t stream);

/* Tuning knobs (process-wide, all threads; 0 = each kernel family's default).
 * Results do not depend on them (test_launch_configurations_bit_identical,
 * test_default_shapes_across_sizes).
 *   vector_width in {0, 1, 4, 8}: caps the vector path of the sampling
 *     kernels (1 = scalar accesses; the fused kernels honour 1 only).  The
 *     streamed default depends on the call size, in samples per SM: <= 512
 *     1 sample per thread x 64 threads, <= 2048 1 x 256, <= 262144 4 x 128,
 *     else 8 x 128 (latency-bound small calls, HBM-bound large ones).
 *   block_size 0 or 64..256 (multiple of 32): threads per block of the
 *     sampling kernels (defaults: as above streamed, 512 fused).
 *   blocks_per_sm: 0 = default grid (streamed: one vector chunk per thread;
 *     fused: persistent, SMs x resident blocks); >= 1 = persistent grid-stride grid
 *     of SMs x min(blocks_per_sm, occupancy) blocks; -1 = one chunk per thread. */
vndf_status vndf_set_launch_config(int vector_width, int block_size, int blocks_per_sm);

/* Initialises the library's CUDA state on `device` (-1 = the current device)
 * and waits for it: the CUDA runtime's one-time start-up in this process
 * (loading libvndf's kernels into the context waits for the work already
 * queued on the device: tools/first_call_probe.py), the cached device
 * attributes and the fix-up queue pool.  Optional: the first call of any
 * entry point does the same implicitly.  After it, calls only enqueue. */
vndf_status vndf_init(int device);

/* Static description of a status code. */
const char *vndf_status_string(vndf_status status);

/* cudaError_t behind the last VNDF_ERR_CUDA returned on this thread. */
int vndf_last_cuda_error(void);

/* ABI version: 100 * major + minor. */
int vndf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VNDF_H_ */
