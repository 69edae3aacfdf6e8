// tma_probe.cu -- the streamed kernels' access pattern (read R fp32 SoA planes,
// write W) with the loads staged through shared memory by TMA bulk copies
// (cp.async.bulk + mbarrier ring, one producer warp) instead of per-thread
// 256-bit loads; no arithmetic.  Compared with tools/bw_probe.cu to decide
// whether TMA staging can lift the HBM-bound kernels.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe.bin tools/tma_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

struct Planes {
    const float* in[8];
    float* out[4];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(0x14F0000000000000ull)  // evict-first policy
        : "memory");
}

__device__ __forceinline__ void st8(float* p, const float* v) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// CW consumer warps (8 samples per thread per tile) + 1 producer warp.
template <int R, int W, int STAGES, int CW>
__global__ void __launch_bounds__((CW + 1) * 32) tma_probe(Planes p, long n) {
    constexpr int TILE = CW * 32 * 8;
    extern __shared__ __align__(128) float sm[];  // [STAGES][R][TILE]
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long ntiles = n / TILE;
    if (warp == CW) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], R * TILE * 4);
#pragma unroll
                for (int k = 0; k < R; ++k) bulk_g2s(sm + ((size_t)s * R + k) * TILE, p.in[k] + t * TILE, TILE * 4, &full[s]);
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }
    int s = 0;
    uint32_t ph = 0;
    const int tid = threadIdx.x;  // 0 .. CW*32-1
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&full[s], ph);
        float a[R][8];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const float4* q = reinterpret_cast<const float4*>(sm + ((size_t)s * R + k) * TILE + tid * 8);
            const float4 x = q[0], y = q[1];
            a[k][0] = x.x; a[k][1] = x.y; a[k][2] = x.z; a[k][3] = x.w;
            a[k][4] = y.x; a[k][5] = y.y; a[k][6] = y.z; a[k][7] = y.w;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            float o[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // every input plane feeds every output
                float acc = (float)(w + 1);
#pragma unroll
                for (int k = 0; k < R; ++k) acc = fmaf(acc, 0.5f, a[k][j]);
                o[j] = acc;
            }
            st8(p.out[w] + t * TILE + tid * 8, o);
        }
        if (++s == STAGES) {
            s = 0;
            ph ^= 1;
        }
    }
}

template <int R, int W, int STAGES, int CW>
double run(long n, const Planes& p, int blocks_per_sm) {
    constexpr int TILE = CW * 32 * 8;
    const size_t smem = (size_t)STAGES * R * TILE * 4;
    cudaFuncSetAttribute(tma_probe<R, W, STAGES, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * blocks_per_sm;
    for (int i = 0; i < 10; ++i) tma_probe<R, W, STAGES, CW><<<grid, (CW + 1) * 32, smem>>>(p, n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = n >= (1L << 26) ? 50 : 200;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) tma_probe<R, W, STAGES, CW><<<grid, (CW + 1) * 32, smem>>>(p, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return (double)(R + W) * 4.0 * n / (ms / reps * 1e-3) / 1e9;
}

int main() {
    for (long n : {1L << 24, 1L << 26}) {
        std::vector<float*> bufs(12);
        for (auto& q : bufs) {
            cudaMalloc(&q, n * sizeof(float));
            cudaMemset(q, 0, n * sizeof(float));
        }
        Planes p;
        for (int k = 0; k < 8; ++k) p.in[k] = bufs[k];
        for (int k = 0; k < 4; ++k) p.out[k] = bufs[8 + k];
        cudaDeviceSynchronize();
        const int e = n == (1L << 24) ? 24 : 26;
        printf("n=2^%d 4 cw, 4 st, 2/SM: (7,4) %5.0f  (7,3) %5.0f GB/s\n", e, run<7, 4, 4, 4>(n, p, 2), run<7, 3, 4, 4>(n, p, 2));
        printf("n=2^%d 4 cw, 3 st, 2/SM: (7,4) %5.0f  (7,3) %5.0f GB/s\n", e, run<7, 4, 3, 4>(n, p, 2), run<7, 3, 3, 4>(n, p, 2));
        printf("n=2^%d 8 cw, 3 st, 1/SM: (7,4) %5.0f  (7,3) %5.0f GB/s\n", e, run<7, 4, 3, 8>(n, p, 1), run<7, 3, 3, 8>(n, p, 1));
        printf("n=2^%d 2 cw, 6 st, 3/SM: (7,4) %5.0f  (7,3) %5.0f GB/s\n", e, run<7, 4, 6, 2>(n, p, 3), run<7, 3, 6, 2>(n, p, 3));
        printf("n=2^%d 4 cw, 6 st, 1/SM: (7,4) %5.0f  (7,3) %5.0f GB/s\n", e, run<7, 4, 6, 4>(n, p, 1), run<7, 3, 6, 4>(n, p, 1));
        for (auto q : bufs) cudaFree(q);
    }
    return 0;
}
