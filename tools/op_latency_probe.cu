// Probe: dependent-chain latency (cycles per op) of the f64 / warp ops the
// certification tail is built from, single warp, on a B200.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ double nl_exp(double x) { return exp(x); }
__device__ __noinline__ double nl_log(double x) { return log(x); }

template <int OP>
__global__ void chain(double *out, long long *cyc, double seed, int n) {
    double x = seed + threadIdx.x * 1e-9;
    unsigned u = __double_as_longlong(x);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
        if (OP == 0) x = __dadd_rn(x, 1e-300);
        if (OP == 1) x = __dmul_rn(x, 0.999999999);
        if (OP == 2) x = fmax(x, -x);
        if (OP == 3) x = __shfl_xor_sync(0xffffffffu, x, 1);
        if (OP == 4) u = __shfl_xor_sync(0xffffffffu, u, 1);
        if (OP == 5) u = __reduce_max_sync(0xffffffffu, u);
        if (OP == 6) x = exp(x) * 1e-3;
        if (OP == 7) x = nl_exp(x) * 1e-3;
        if (OP == 8) x = log(x + 2.0);
        if (OP == 9) x = (double)(float)x;
        if (OP == 10) x = __ddiv_rn(1.0, x + 1.5);
        if (OP == 11) { __syncwarp(); x = __dadd_rn(x, 1e-300); }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = x + u;
}

template <int OP>
void run(const char *name, double *o, long long *c) {
    const int n = 4096;
    long long h;
    for (int r = 0; r < 2; ++r) {
        chain<OP><<<1, 32>>>(o, c, 0.5, n);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cyc/op\n", name, (double)h / n);
}

__global__ void smemtest(long long *cyc) {
    __shared__ double buf[1024];
    __shared__ int flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    buf[threadIdx.x] = 0;
}

int main() {
    double *o;
    long long *c;
    cudaMalloc(&o, 4096);
    cudaMalloc(&c, 64);
    run<0>("dadd", o, c);
    run<1>("dmul", o, c);
    run<2>("fmax f64", o, c);
    run<3>("shfl.bfly f64", o, c);
    run<4>("shfl.bfly u32", o, c);
    run<5>("redux.max u32", o, c);
    run<6>("exp f64 (inline)", o, c);
    run<7>("exp f64 (noinline call)", o, c);
    run<8>("log f64", o, c);
    run<9>("f64->f32->f64", o, c);
    run<10>("ddiv", o, c);
    run<11>("syncwarp+dadd", o, c);
    long long h;
    smemtest<<<1, 256>>>(c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cyc/op\n", "__syncthreads (8 warps)", (double)h / 1024);
    return 0;
}
