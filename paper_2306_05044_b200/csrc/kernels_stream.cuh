// kernels_stream.cuh -- streamed (HBM-bound) sampling kernel with the block-level float64
// fix-up queue.
// Part of libvndf's single translation unit (included by vndf.cu inside its
// anonymous namespace); see vndf.cu for the kernel list and DESIGN.md s.6.
#pragma once

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
#ifndef VNDF_STREAM_BOUND
#define VNDF_STREAM_BOUND 256
#endif

template <int METHOD, bool PDF, int V>
__global__ void __launch_bounds__(VNDF_STREAM_BOUND, VNDF_STREAM_MINB) stream_kernel(StreamArgs a, int64_t n) {
    __shared__ int64_t fix_idx[METHOD != kHeitz ? kBlockFixCap : 1];
    __shared__ int fix_count;
    if (METHOD != kHeitz && threadIdx.x == 0) fix_count = 0;
    // Programmatic dependent launch: let the next kernel on the stream be
    // scheduled once every block of this grid is running, and wait for the
    // previous grid (its completion and memory flush) before touching memory.
    pdl_launch_dependents();
    pdl_wait();
    if (METHOD != kHeitz) __syncthreads();
    const int qcap = min(a.fix_cap, kBlockFixCap);
    auto defer = [&](int64_t i) {
        const int slot = atomicAdd(&fix_count, 1);
        if (slot < qcap) fix_idx[slot] = i;
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
        const int m = min(fix_count, qcap);
        for (int t = threadIdx.x; t < m; t += blockDim.x) fix_one(a, PDF, fix_idx[t], METHOD == kCap);
    }
}
