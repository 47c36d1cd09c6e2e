// DADD / DMUL dependent-chain latency and the LDS->DADD loop on sm_100a
// (diagnostic).  nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false
#include <cstdio>
__global__ void chain(double* out, long long* cyc, int n, double a) {
    double x = a, y = a * 0.5, z = a * 0.25, w = a * 0.125;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) x = __dadd_rn(x, a);
    long long t1 = clock64();
    for (int i = 0; i < n; i++) {
        x = __dadd_rn(x, a);
        y = __dadd_rn(y, a);
        z = __dadd_rn(z, a);
        w = __dadd_rn(w, a);
    }
    long long t2 = clock64();
    for (int i = 0; i < n; i++) x = __dmul_rn(x, 1.0000001);
    long long t3 = clock64();
    out[threadIdx.x] = x + y + z + w;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
    }
}
int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 1024 * 8);
    cudaMallocManaged(&c, 64);
    const int n = 100000;
    for (int threads : {32, 128}) {
        chain<<<1, threads>>>(o, c, n, 1.0);
        cudaDeviceSynchronize();
        printf("threads=%d dadd chain %.2f cyc/op, 4 chains %.2f cyc/step, dmul chain %.2f cyc/op\n", threads,
               (double)c[0] / n, (double)c[1] / n, (double)c[2] / n);
    }
    return 0;
}
