// Probe: dependent-load latency on a B200 after an L2 flush, to separate HBM
// latency from TLB (page-walk) cost, and the cost of a 148-CTA grid barrier.
//   chase<stride>: one thread walks N dependent loads `stride` bytes apart in a
//   1 GiB buffer (stride 64 KiB: same 2 MiB page 32 times; 2 MiB: a new page
//   every load), timed in cycles.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void flush(const float4 *b, size_t n, float *o) {
    float s = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        s += __ldcg(b + i).x;
    if (s == 12345.f) o[0] = s;
}

// buf holds at offset i*stride the offset of the next hop
__global__ void chase(const char *buf, long long stride, int n, long long *out) {
    long long off = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) off = __ldcg(reinterpret_cast<const long long *>(buf + off));
    long long t1 = clock64();
    out[0] = t1 - t0;
    out[1] = off;
}

__global__ void init_chain(char *buf, long long stride, int n) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += gridDim.x * blockDim.x)
        *reinterpret_cast<long long *>(buf + (long long)i * stride) = (long long)(i + 1) * stride;
}

// grid barrier round trips: every CTA arrives; measure per-barrier cycles (CTA 0)
__global__ void gbar(unsigned *bar, int reps, long long *out) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned gen;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
            const unsigned t = atomicAdd(bar, 1u);
            if (t == gridDim.x - 1) {
                bar[0] = 0;
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
            } else {
                unsigned g2;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g2) : "l"(bar + 1) : "memory");
                } while (g2 == gen);
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / reps;
}

int main() {
    const size_t BYTES = 1ull << 30;
    char *buf;
    float4 *fb;
    float *o;
    long long *out, h[2];
    unsigned *bar;
    cudaMalloc(&buf, BYTES);
    size_t fn = (512ull << 20) / 16;
    cudaMalloc(&fb, fn * 16);
    cudaMemset(fb, 0, fn * 16);
    cudaMalloc(&o, 64);
    cudaMalloc(&out, 64);
    cudaMalloc(&bar, 64);
    cudaMemset(bar, 0, 64);
    const long long strides[] = {128, 4096, 65536, 1 << 21, 1 << 22};
    for (long long st : strides) {
        const int n = (int)std::min<long long>(256, BYTES / st - 1);
        init_chain<<<64, 256>>>(buf, st, n);
        for (int rep = 0; rep < 3; ++rep) {
            flush<<<592, 512>>>(fb, fn, o);
            chase<<<1, 1>>>(buf, st, n, out);
            cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            long long warm = 0;
            chase<<<1, 1>>>(buf, st, n, out);
            cudaMemcpy(&warm, out, 8, cudaMemcpyDeviceToHost);
            printf("stride %8lld: %3d hops cold %6.0f cyc/hop, warm (L2) %6.0f cyc/hop\n", st, n, (double)h[0] / n,
                   (double)warm / n);
        }
    }
    for (int threads : {32, 256}) {
        gbar<<<148, threads>>>(bar, 100, out);
        cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("grid barrier 148 CTAs x %d threads: %lld cyc\n", threads, h[0]);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
