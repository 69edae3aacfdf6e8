/*
 * c_demo.c -- the libvndf C ABI used from plain C (no Python, no torch):
 * sample 2^20 GGX visible normals by the spherical cap (vndf_sample_cap_pdf),
 * then through the fused Philox entry point, device and host (end to end),
 * and print a checksum.
 *
 *   gcc -std=c99 -O2 examples/c_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2306_05044_b200 -lvndf -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2306_05044_b200 -o c_demo -lm
 *
 * (libvndf.so is built by __graft_entry__.build(); link it by path as
 * paper_2306_05044_b200/libvndf.so or via -lvndf with a symlink.)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "vndf.h"

#define CHECK(x)                                                                         \
    do {                                                                                 \
        vndf_status s_ = (x);                                                            \
        if (s_ != VNDF_OK) {                                                             \
            fprintf(stderr, "%s failed: %s (cuda %d)\n", #x, vndf_status_string(s_),     \
                    vndf_last_cuda_error());                                             \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

int main(void)
{
    const int64_t n = (int64_t)1 << 20;
    const size_t bytes = (size_t)n * sizeof(float);
    float *h_in[7], *d_in[7], *d_out[4], *h_out[4];
    for (int k = 0; k < 7; ++k) {
        h_in[k] = (float *)malloc(bytes);
        if (cudaMalloc((void **)&d_in[k], bytes) != cudaSuccess) return 1;
    }
    for (int k = 0; k < 4; ++k) {
        h_out[k] = (float *)malloc(bytes);
        if (cudaMalloc((void **)&d_out[k], bytes) != cudaSuccess) return 1;
    }
    /* a simple deterministic input set: upper-hemisphere incidence, alpha in [0.05, 1] */
    uint32_t x = 12345u;
    for (int64_t i = 0; i < n; ++i) {
        x = x * 1664525u + 1013904223u; float a = (float)(x >> 8) * 0x1p-24f;
        x = x * 1664525u + 1013904223u; float b = (float)(x >> 8) * 0x1p-24f;
        float z = 1.0f - a, r = sqrtf(a * (2.0f - a));
        h_in[0][i] = r * cosf(6.2831853f * b);
        h_in[1][i] = r * sinf(6.2831853f * b);
        h_in[2][i] = z;
        x = x * 1664525u + 1013904223u; h_in[3][i] = 0.05f + 0.95f * (float)(x >> 8) * 0x1p-24f;
        x = x * 1664525u + 1013904223u; h_in[4][i] = 0.05f + 0.95f * (float)(x >> 8) * 0x1p-24f;
        x = x * 1664525u + 1013904223u; h_in[5][i] = (float)(x >> 8) * 0x1p-24f;
        x = x * 1664525u + 1013904223u; h_in[6][i] = (float)(x >> 8) * 0x1p-24f;
    }
    for (int k = 0; k < 7; ++k) cudaMemcpy(d_in[k], h_in[k], bytes, cudaMemcpyHostToDevice);

    CHECK(vndf_sample_cap_pdf(d_in[0], d_in[1], d_in[2], d_in[3], d_in[4], d_in[5], d_in[6],
                              d_out[0], d_out[1], d_out[2], d_out[3], n, NULL));
    if (cudaDeviceSynchronize() != cudaSuccess) return 1;
    for (int k = 0; k < 4; ++k) cudaMemcpy(h_out[k], d_out[k], bytes, cudaMemcpyDeviceToHost);

    double max_norm_err = 0.0, min_dot = 1.0, checksum = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double hx = h_out[0][i], hy = h_out[1][i], hz = h_out[2][i];
        double nrm = sqrt(hx * hx + hy * hy + hz * hz);
        if (fabs(nrm - 1.0) > max_norm_err) max_norm_err = fabs(nrm - 1.0);
        double d = hx * h_in[0][i] + hy * h_in[1][i] + hz * h_in[2][i];
        if (d < min_dot) min_dot = d;
        checksum += hx + 2.0 * hy + 3.0 * hz + 1e-3 * h_out[3][i];
    }
    printf("vndf_sample_cap_pdf: n=%lld max| |h|-1 |=%.2e min(wi.h)=%.3e checksum=%.6f\n",
           (long long)n, max_norm_err, min_dot, checksum);

    CHECK(vndf_sample_cap_philox(3, 0, n, d_out[0], d_out[1], d_out[2], d_out[3], NULL));
    if (cudaDeviceSynchronize() != cudaSuccess) return 1;
    cudaMemcpy(h_out[2], d_out[2], bytes, cudaMemcpyDeviceToHost);
    double zsum = 0.0;
    for (int64_t i = 0; i < n; ++i) zsum += h_out[2][i];
    printf("vndf_sample_cap_philox: mean h.z=%.6f\n", zsum / (double)n);

    /* the same samples end to end into plain malloc'd host memory (the host
       entry point stages chunks through device memory and copies them back) */
    float *e_out[4];
    for (int k = 0; k < 4; ++k) e_out[k] = (float *)malloc(bytes);
    CHECK(vndf_sample_cap_philox_host(3, 0, n, e_out[0], e_out[1], e_out[2], e_out[3], NULL));
    int64_t mismatches = 0;
    for (int64_t i = 0; i < n; ++i) mismatches += e_out[2][i] != h_out[2][i];
    printf("vndf_sample_cap_philox_host: %lld of %lld h.z differ from the device call\n",
           (long long)mismatches, (long long)n);
    for (int k = 0; k < 4; ++k) free(e_out[k]);
    if (mismatches) return 3;
    printf("status strings: %s / %s, ABI version %d\n", vndf_status_string(VNDF_OK),
           vndf_status_string(VNDF_ERR_INVALID_ARGUMENT), vndf_version());
    for (int k = 0; k < 7; ++k) { cudaFree(d_in[k]); free(h_in[k]); }
    for (int k = 0; k < 4; ++k) { cudaFree(d_out[k]); free(h_out[k]); }
    return (max_norm_err < 1e-5 && min_dot > -1e-5) ? 0 : 2;
}
