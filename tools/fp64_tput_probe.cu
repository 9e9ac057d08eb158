// Probe: f64 issue throughput (DADD / DMUL / mixed, independent chains) and
// F2F f32->f64, per SM per cycle, 8 and 16 warps per SM, on a B200.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void tput(double *out, long long *cyc, int n) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-9 + j;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = threadIdx.x * 1e-3f + j;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) a[j] = __dadd_rn(a[j], 1e-300);
            if (OP == 1) a[j] = __dmul_rn(a[j], 0.9999999);
            if (OP == 2) a[j] = __dadd_rn(a[j], __dmul_rn((double)f[j], 1.0000001));
            if (OP == 3) a[j] = __fma_rn(a[j], 0.9999999, 1e-300);
            if (OP == 4) { f[j] = f[j] * 1.0001f + 1.0f; }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j] + f[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char *name, int threads, double *o, long long *c) {
    const int n = 2048;
    long long h[148];
    tput<OP><<<148, threads>>>(o, c, n);
    tput<OP><<<148, threads>>>(o, c, n);
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double ops = (double)threads * n * 8 * (OP == 2 ? 3 : 1);  // OP 2: F2F + DMUL + DADD
    printf("%-28s %4d thr/SM: %7.1f lane-ops/clk/SM\n", name, threads, ops / h[0]);
}

int main() {
    double *o;
    long long *c;
    cudaMalloc(&o, 148 * 1024 * 8);
    cudaMalloc(&c, 148 * 8);
    for (int t : {256, 512, 1024}) {
        run<0>("dadd", t, o, c);
        run<1>("dmul", t, o, c);
        run<2>("f2f+dmul+dadd (3 ops)", t, o, c);
        run<3>("dfma", t, o, c);
        run<4>("ffma (f32)", t, o, c);
    }
    return 0;
}
