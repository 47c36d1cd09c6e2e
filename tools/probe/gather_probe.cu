// Upper-bound probe for the LP kernel's memory pattern: 1M rows x ~28 random
// neighbours, fp64 label vectors of C=10 columns (80 B) gathered per entry.
// Thread-per-entry gather with plenty of independent loads: how many entries
// per second can a B200 gather for this layout?  (diagnostic tool only)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_gather(const int* nbr, const double* w, const double* X, long long ne, int C, double* out) {
    double acc = 0.0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < ne; p += (long long)gridDim.x * blockDim.x) {
        int v = __ldcs(nbr + p);
        double wt = __ldcs(w + p);
        const double2* xv = (const double2*)(X + (long long)v * C);
        double s = 0.0;
        for (int c = 0; c < C / 2; c++) {
            double2 x = xv[c];
            s += x.x + x.y;
        }
        acc += s * wt;
    }
    if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
    long long n = 1000000, deg = 28;
    int C = 10;
    long long ne = n * deg;
    std::vector<int> h_nbr(ne);
    srand(1);
    for (long long i = 0; i < ne; i++) h_nbr[i] = (int)(((long long)rand() * 65536LL + rand()) % n);
    int* nbr; double *w, *X, *out;
    cudaMalloc(&nbr, ne * 4); cudaMalloc(&w, ne * 8); cudaMalloc(&X, n * C * 8); cudaMalloc(&out, 8);
    cudaMemcpy(nbr, h_nbr.data(), ne * 4, cudaMemcpyHostToDevice);
    cudaMemset(w, 0, ne * 8); cudaMemset(X, 0, n * C * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks : {148 * 8, 148 * 16, 148 * 32}) {
        for (int it = 0; it < 2; it++) k_gather<<<blocks, 256>>>(nbr, w, X, ne, C, out);
        cudaEventRecord(a);
        for (int it = 0; it < 5; it++) k_gather<<<blocks, 256>>>(nbr, w, X, ne, C, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("blocks %d: %.3f ms per %lld entries = %.1f G entries/s = %.0f GB/s (92 B/entry)\n", blocks, ms, ne,
               ne / (ms * 1e6), ne * 92.0 / (ms * 1e6));
    }
    return 0;
}
