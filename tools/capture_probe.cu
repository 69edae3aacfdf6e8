// capture_probe.cu -- which CUDA runtime calls are legal inside a stream capture
// (cudaStreamCaptureModeGlobal, torch's default) in a fresh process, i.e. with
// no device state built yet.  Each candidate runs in its own capture.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cp tools/capture_probe.cu && /tmp/cp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_probe(float* p) { if (p) p[threadIdx.x] = 1.0f; }

template <typename F>
void probe(const char* name, F f) {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    cudaError_t e = f(s);
    cudaGraph_t g = nullptr;
    cudaError_t ee = cudaStreamEndCapture(s, &g);
    printf("%-44s call: %-40s end: %s\n", name, cudaGetErrorName(e), cudaGetErrorName(ee));
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(s);
}

int main() {
    cudaFree(0);  // context
    probe("cudaStreamIsCapturing", [](cudaStream_t s) {
        cudaStreamCaptureStatus c; return cudaStreamIsCapturing(s, &c); });
    probe("cudaStreamGetDevice", [](cudaStream_t s) { int d; return cudaStreamGetDevice(s, &d); });
    probe("cudaDeviceGetAttribute(SM count)", [](cudaStream_t) {
        int v; return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0); });
    probe("cudaOccupancyMaxActiveBlocks (first use)", [](cudaStream_t) {
        int o; return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_probe, 256, 0); });
    probe("cudaMemPoolCreate", [](cudaStream_t) {
        cudaMemPoolProps p = {};
        p.allocType = cudaMemAllocationTypePinned;
        p.location.type = cudaMemLocationTypeDevice;
        p.location.id = 0;
        cudaMemPool_t pool;
        return cudaMemPoolCreate(&pool, &p); });
    static cudaMemPool_t pool = nullptr;
    {
        cudaMemPoolProps p = {};
        p.allocType = cudaMemAllocationTypePinned;
        p.location.type = cudaMemLocationTypeDevice;
        p.location.id = 0;
        cudaMemPoolCreate(&pool, &p);
    }
    probe("cudaMallocFromPoolAsync (private pool)", [](cudaStream_t s) {
        void* q; cudaError_t e = cudaMallocFromPoolAsync(&q, 1 << 20, pool, s);
        if (e == cudaSuccess) e = cudaFreeAsync(q, s);
        return e; });
    probe("cudaMallocAsync (default pool)", [](cudaStream_t s) {
        void* q; cudaError_t e = cudaMallocAsync(&q, 1 << 20, s);
        if (e == cudaSuccess) e = cudaFreeAsync(q, s);
        return e; });
    probe("kernel launch", [](cudaStream_t s) {
        k_probe<<<1, 32, 0, s>>>(nullptr); return cudaGetLastError(); });
    return 0;
}
