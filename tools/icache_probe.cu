// Probe: cycles for one warp to run N straight-line instructions, cold vs
// relaunched (does the SM instruction cache survive across launches?), and
// after an L2 flush.
#include <cstdio>
#include <cuda_runtime.h>
template <int N>
__global__ void straight(float *out, long long *cyc, float a) {
    long long t0;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    float x = a + (float)(t0 & 1) * 0.f, y = a * 2.f, z = a * 3.f, w = a * 4.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        x = x * 1.0001f + y;
        y = y * 0.9999f + z;
        z = z * 1.0002f + w;
        w = w * 0.9998f + x;
    }
    long long t1;
    float sink = x + y + z + w;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) : "f"(sink) : "memory");
    if (threadIdx.x == 0) { out[blockIdx.x] = x + y + z + w; cyc[blockIdx.x] = t1 - t0; }
}
__global__ void flush(const float4 *b, size_t n, float *o) {
    float s = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += b[i].x;
    if (s == 12345.f) o[0] = s;
}
template <int N>
void run(float *out, long long *cyc, float4 *fb, size_t fn) {
    long long h[4];
    for (int rep = 0; rep < 4; ++rep) {
        if (rep == 3) { flush<<<592, 512>>>(fb, fn, out); }
        straight<N><<<1, 32>>>(out, cyc, 1.f);
        cudaMemcpy(&h[rep], cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("N=%6d (~%6d instr, %4d KB): launch1 %7lld cyc  launch2 %7lld  launch3 %7lld  after-L2-flush %7lld  (%.1f cyc/instr cold)\n",
           N, 4 * N * 1, 4 * N * 16 / 1024, h[0], h[1], h[2], h[3], (double)h[0] / (4.0 * N));
}
int main() {
    float *out; long long *cyc; float4 *fb;
    cudaMalloc(&out, 4096); cudaMalloc(&cyc, 4096);
    size_t fn = (512ull << 20) / 16; cudaMalloc(&fb, fn * 16); cudaMemset(fb, 0, fn * 16);
    run<64>(out, cyc, fb, fn);
    run<256>(out, cyc, fb, fn);
    run<512>(out, cyc, fb, fn);
    run<1024>(out, cyc, fb, fn);
    run<2048>(out, cyc, fb, fn);
    run<4096>(out, cyc, fb, fn);
    return 0;
}
