// Probe 2: the same gather as gather_probe.cu but through cp.async into
// shared memory (like k_lp_fused's windows), to separate the cost of the
// staging mechanism from the access pattern.  (diagnostic tool only)
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ inline void cp16(void* dst, const void* src) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

template <int PER>
__global__ void k_gather_cp(const int* nbr, const double* w, const double* X, long long ne, int C, double* out) {
    extern __shared__ double sm[];
    double* my = sm + (size_t)threadIdx.x * PER * 10;
    double acc = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x * PER;
    for (long long p0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * PER; p0 < ne; p0 += stride) {
        int v[PER];
        double wt[PER];
#pragma unroll
        for (int j = 0; j < PER; j++) {
            v[j] = p0 + j < ne ? __ldcs(nbr + p0 + j) : 0;
            wt[j] = p0 + j < ne ? __ldcs(w + p0 + j) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < PER; j++)
            for (int c = 0; c < C; c += 2) cp16(my + j * C + c, X + (long long)v[j] * C + c);
        asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
        for (int j = 0; j < PER; j++) {
            double s = 0.0;
            for (int c = 0; c < C; c++) s += my[j * C + c];
            acc += s * wt[j];
        }
    }
    if (acc == 12345.678) out[0] = acc;
}

int main() {
    long long n = 1000000, deg = 28;
    int C = 10;
    long long ne = n * deg;
    std::vector<int> h(ne);
    srand(1);
    for (long long i = 0; i < ne; i++) h[i] = (int)(((long long)rand() * 65536LL + rand()) % n);
    int* nbr; double *w, *X, *out;
    cudaMalloc(&nbr, ne * 4); cudaMalloc(&w, ne * 8); cudaMalloc(&X, n * C * 8); cudaMalloc(&out, 8);
    cudaMemcpy(nbr, h.data(), ne * 4, cudaMemcpyHostToDevice);
    cudaMemset(w, 0, ne * 8); cudaMemset(X, 0, n * C * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, int per, int threads, int blocks) {
        size_t smem = (size_t)threads * per * 10 * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int it = 0; it < 2; it++) kern<<<blocks, threads, smem>>>(nbr, w, X, ne, C, out);
        cudaEventRecord(a);
        for (int it = 0; it < 5; it++) kern<<<blocks, threads, smem>>>(nbr, w, X, ne, C, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("cp.async PER=%d threads=%d blocks=%d smem=%zu: %.3f ms = %.1f G entries/s %s\n", per, threads, blocks,
               smem, ms, ne / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    };
    run(k_gather_cp<1>, 1, 256, 148 * 8);
    run(k_gather_cp<2>, 2, 256, 148 * 4);
    run(k_gather_cp<2>, 2, 256, 148 * 3);
    run(k_gather_cp<4>, 4, 128, 148 * 4);
    return 0;
}
