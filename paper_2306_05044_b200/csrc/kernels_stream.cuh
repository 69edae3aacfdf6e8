// kernels_stream.cuh -- streamed (HBM-bound) sampling kernel with in-thread float64
// fix-ups.
// Part of libvndf's single translation unit (included by vndf.cu inside its
// anonymous namespace); see vndf.cu for the kernel list and DESIGN.md s.6.
#pragma once

// ------------------------------------------------------- streamed kernel --
// Chunk c covers samples [c V, c V + V).  Full chunks go through the vector
// path (one chunk per thread by default, grid-stride if the grid is capped);
// the n mod V tail is done by the first threads of the grid with scalar
// accesses.  A flagged sample is recomputed in float64 at once, in the thread
// that found it, from the inputs it holds in registers: inlined in the 1- and
// 4-sample loops that small, latency-bound calls use (config 1 at 4-sample
// chunks: 1.89 -> 1.72 us per launch, the call's ~80 clocks and the scheduling
// barrier it puts in the loop gone), an out-of-line call (cap_fp64) in the
// 8-sample loop (inlined there it measured 3% slower at 2^20 samples).  Round 1 pushed
// flagged samples to a shared-memory queue, recomputed after a block barrier
// from a reload of their inputs; inline is faster wherever it was measured
// (config 5: 7.12 vs 6.86 TB/s; config 1: 2.54 vs 2.81 us per launch -- the
// barrier and the L2 round trip of the reload were on the critical path;
// profiles/r2/stream_fixup_r2.txt).
#ifndef VNDF_STREAM_MINB
#define VNDF_STREAM_MINB 1
#endif
#ifndef VNDF_STREAM_BOUND
#define VNDF_STREAM_BOUND 256
#endif

template <int METHOD, bool PDF, int V>
__global__ void __launch_bounds__(VNDF_STREAM_BOUND, VNDF_STREAM_MINB) stream_kernel(StreamArgs a, int64_t n) {
    // Programmatic dependent launch: let the next kernel on the stream be
    // scheduled once every block of this grid is running, and wait for the
    // previous grid (its completion and memory flush) before touching memory.
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
        Vec<V> hx, hy, hz, pd;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            Sample o;
            if (sample_one<METHOD, PDF>(wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j], u1.v[j], u2.v[j], o))
                o = fix_regs<(V <= 4)>(wx.v[j], wy.v[j], wz.v[j], ax.v[j], ay.v[j], u1.v[j], u2.v[j], METHOD == kCap);
            hx.v[j] = o.x;
            hy.v[j] = o.y;
            hz.v[j] = o.z;
            pd.v[j] = o.pdf;
        }
        st_stream<V>(a.hx + i, hx);
        st_stream<V>(a.hy + i, hy);
        st_stream<V>(a.hz + i, hz);
        if (PDF) st_stream<V>(a.pdf + i, pd);
    }
    if (V > 1) {
        const int64_t i = nchunks * V + tid;
        if (i < n) {
            const float wx = a.wx[i], wy = a.wy[i], wz = a.wz[i], ax = a.ax[i], ay = a.ay[i], u1 = a.u1[i],
                        u2 = a.u2[i];
            Sample o;
            if (sample_one<METHOD, PDF>(wx, wy, wz, ax, ay, u1, u2, o))
                o = fix_regs<false>(wx, wy, wz, ax, ay, u1, u2, METHOD == kCap);
            a.hx[i] = o.x;
            a.hy[i] = o.y;
            a.hz[i] = o.z;
            if (PDF) a.pdf[i] = o.pdf;
        }
    }
}
