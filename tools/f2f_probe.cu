// Probe: f32->f64 conversion throughput (F2F.F64.F32) vs an integer-op
// widening, per SM per cycle, 8 warps/SM, data-dependent inputs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double widen_int(float f) {  // exact for normals and zero
    const unsigned b = __float_as_uint(f);
    const unsigned e = b & 0x7f800000u;
    unsigned hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + 0x38000000u);
    unsigned lo = b << 29;
    if (e == 0u) { hi = b & 0x80000000u; lo = 0u; }  // +-0 (denormals would need F2F)
    return __hiloint2double((int)hi, (int)lo);
}

template <int OP>
__global__ void conv(const float *in, double *out, long long *cyc, int n) {
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = in[(threadIdx.x * 8 + j) & 1023];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const double x = OP == 0 ? (double)f[j] : widen_int(f[j]);
            acc[j] = __dadd_rn(acc[j], x);
            f[j] = __uint_as_float(__float_as_uint(f[j]) ^ 0x1u);  // data-dependent: no hoisting
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *in;
    double *o;
    long long *c, h;
    cudaMalloc(&in, 4096 * 4);
    cudaMalloc(&o, 148 * 1024 * 8);
    cudaMalloc(&c, 148 * 8);
    float hin[1024];
    for (int i = 0; i < 1024; ++i) hin[i] = 1.0f + i * 0.37f;
    cudaMemcpy(in, hin, sizeof(hin), cudaMemcpyHostToDevice);
    for (int op = 0; op < 2; ++op)
        for (int t : {256, 512}) {
            const int n = 2048;
            for (int r = 0; r < 2; ++r) {
                if (op == 0) conv<0><<<148, t>>>(in, o, c, n);
                else conv<1><<<148, t>>>(in, o, c, n);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("%-22s %4d thr/SM: %6.1f conversions(+dadd)/clk/SM\n", op ? "int-op widening" : "F2F.F64.F32", t,
                   (double)t * n * 8 / h);
        }
    return 0;
}
