// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw tools/l2bw.cu  (run on the B200)
// L2-resident streaming throughput: read-only (16 B loads, coalesced) and scattered 8-byte
// stores into an L2-resident array; reports bytes of 32-byte sectors per cycle and TB/s.
#include <cstdio>
#include <cstdint>
__global__ void rd(const double2* __restrict__ a, size_t n, int reps, double* out) {
    double s = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
            double2 v = __ldcg(a + i);
            s += v.x + v.y;
        }
    if (s == 12345.0) out[0] = s;
}
__global__ void scat(double* a, size_t n, int reps) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
            size_t j = (i * 2654435761ull + r) % n; // scattered
            a[j] = (double)i;
        }
}
int main() {
    const size_t bytes = 32ull << 20; // 32 MB: L2-resident
    double2* a; cudaMalloc(&a, bytes); cudaMemset(a, 0, bytes);
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t n = bytes / 16;
    const int reps = 50;
    for (int w = 0; w < 2; ++w) rd<<<sms * 4, 512>>>(a, n, 2, o);
    cudaEventRecord(e0); rd<<<sms * 4, 512>>>(a, n, reps, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tb = (double)bytes * reps / (ms * 1e-3) / 1e12;
    printf("L2 read stream: %.2f TB/s = %.0f B/cycle at %d MHz\n", tb, tb * 1e12 / (1965e6), clk / 1000);
    const size_t n8 = bytes / 8;
    for (int w = 0; w < 2; ++w) scat<<<sms * 4, 512>>>((double*)a, n8, 1);
    cudaEventRecord(e0); scat<<<sms * 4, 512>>>((double*)a, n8, 10); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double gs = (double)n8 * 10 / (ms * 1e-3) / 1e9;
    printf("scattered 8-B stores (L2-resident): %.1f G stores/s = %.2f TB/s of 32-B sectors\n", gs, gs * 32 / 1e3);
    return 0;
}
