// bw_probe.cu -- achievable HBM bandwidth for the streamed kernels' exact access
// pattern, with no arithmetic: read R fp32 SoA planes, write W planes, 8 floats
// per plane per thread with the same 256-bit L2-hinted loads/stores, one chunk
// per thread, 128-thread blocks.  The number a sampling kernel with the same
// (R, W) is measured against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu
//   /tmp/bw_probe            # prints GB/s for (7,4), (7,3), (8,4) at 2^24 and 2^26 samples
#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

struct V8 {
    float v[8];
};

__device__ __forceinline__ V8 ld8(const float* p) {
    V8 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                   "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st8(float* p, const V8& r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :
                 : "l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]),
                   "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}

template <int R, int W>
__global__ void __launch_bounds__(128) probe(const float* const* in, float* const* out, long n) {
    extern __shared__ char occupancy_limiter[];
    const long c = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c * 8 >= n) return;
    V8 a[R];
#pragma unroll
    for (int k = 0; k < R; ++k) a[k] = ld8(in[k] + c * 8);
#pragma unroll
    for (int w = 0; w < W; ++w) {
        V8 o;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            // every input plane feeds every output (so no load is dead)
            float acc = (float)(w + 1);
#pragma unroll
            for (int k = 0; k < R; ++k) acc = fmaf(acc, 0.5f, a[k].v[j]);
            o.v[j] = acc;
        }
        st8(out[w] + c * 8, o);
    }
}

template <int R, int W>
double run(long n, const float* const* din, float* const* dout, int blocks_per_sm) {
    const int grid = (int)((n / 8 + 127) / 128);
    // limit residency with dynamic shared memory (228 KB per SM)
    const int smem = blocks_per_sm > 0 ? (227 * 1024) / blocks_per_sm - 1024 : 0;
    cudaFuncSetAttribute(probe<R, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int i = 0; i < 10; ++i) probe<R, W><<<grid, 128, smem>>>(din, dout, n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = n >= (1L << 26) ? 50 : 200;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) probe<R, W><<<grid, 128, smem>>>(din, dout, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return (double)(R + W) * 4.0 * n / (ms / reps * 1e-3) / 1e9;
}

int main(int argc, char** argv) {
    // mode "one73": a single 7-read / 3-write launch at 2^26 (for an ncu capture)
    if (argc > 1 && std::string(argv[1]) == "one73") {
        const long n = 1L << 26;
        std::vector<float*> bufs(10);
        for (auto& p : bufs) cudaMalloc(&p, n * sizeof(float));
        const float** din;
        float** dout;
        cudaMallocManaged(&din, 8 * sizeof(float*));
        cudaMallocManaged(&dout, 4 * sizeof(float*));
        for (int k = 0; k < 7; ++k) din[k] = bufs[k];
        for (int k = 0; k < 3; ++k) dout[k] = bufs[7 + k];
        cudaDeviceSynchronize();
        probe<7, 3><<<(int)((n / 8 + 127) / 128), 128>>>(din, dout, n);
        cudaDeviceSynchronize();
        return 0;
    }
    // mode "stagger": planes carved from one slab with a per-plane stagger
    if (argc > 1 && std::string(argv[1]) == "stagger") {
        for (long n : {1L << 24, 1L << 26}) {
            for (long stagger : {0L, 256L, 4096L, 65536L, 1L << 20, 3L << 20}) {
                float* slab = nullptr;
                const size_t plane = n * sizeof(float) + stagger;
                cudaMalloc(&slab, 12 * plane + 4096);
                cudaMemset(slab, 0, 12 * plane + 4096);
                const float** din;
                float** dout;
                cudaMallocManaged(&din, 8 * sizeof(float*));
                cudaMallocManaged(&dout, 4 * sizeof(float*));
                char* base = (char*)slab;
                for (int k = 0; k < 8; ++k) din[k] = (const float*)(base + k * plane);
                for (int k = 0; k < 4; ++k) dout[k] = (float*)(base + (8 + k) * plane);
                cudaDeviceSynchronize();
                printf("n=2^%d stagger %8ld B: (7,4) %5.0f  (7,3) %5.0f  (8,4) %5.0f GB/s\n", n == (1L << 24) ? 24 : 26,
                       stagger, run<7, 4>(n, din, dout, 0), run<7, 3>(n, din, dout, 0), run<8, 4>(n, din, dout, 0));
                cudaFree(slab);
                cudaFree(din);
                cudaFree(dout);
            }
        }
        return 0;
    }

    for (long n : {1L << 24, 1L << 26}) {
        // one allocation per plane of exactly n floats, as torch.empty would make them
        std::vector<float*> bufs(12);
        for (auto& p : bufs) {
            cudaMalloc(&p, n * sizeof(float));
            cudaMemset(p, 0, n * sizeof(float));
        }
        const float** din;
        float** dout;
        cudaMallocManaged(&din, 8 * sizeof(float*));
        cudaMallocManaged(&dout, 4 * sizeof(float*));
        for (int k = 0; k < 8; ++k) din[k] = bufs[k];
        for (int k = 0; k < 4; ++k) dout[k] = bufs[8 + k];
        cudaDeviceSynchronize();
        for (int bps : {0, 16, 8, 4}) {
            printf("n=2^%d blocks/SM %-3s  read 7 / write 4: %5.0f GB/s   read 7 / write 3: %5.0f GB/s   "
                   "read 8 / write 4: %5.0f GB/s\n",
                   n == (1L << 24) ? 24 : 26, bps ? std::to_string(bps).c_str() : "max",
                   run<7, 4>(n, din, dout, bps), run<7, 3>(n, din, dout, bps), run<8, 4>(n, din, dout, bps));
        }
        for (auto p : bufs) cudaFree(p);
        cudaFree(din);
        cudaFree(dout);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
