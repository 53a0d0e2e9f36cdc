// FP64 issue-rate probe on the B200 (the router's f64 work): DFMA, F2F.F64.F32
// and FFMA throughput with 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, int iters, double a) {
    double s[8];
    for (int j = 0; j < 8; ++j) s[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = fma(s[j], a, 1.0);
    double t = 0; for (int j = 0; j < 8; ++j) t += s[j];
    if (t == 12345.0) out[0] = t;
}
__global__ void k_f2f(double* out, int iters, float a) {
    double s[8]; float f[8];
    for (int j = 0; j < 8; ++j) { s[j] = 0; f[j] = threadIdx.x * a + j; }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) { f[j] += a; s[j] = static_cast<double>(f[j]); }
    double t = 0; for (int j = 0; j < 8; ++j) t += s[j];
    if (t == 12345.0) out[0] = t;
}
__global__ void k_ffma(float* out, int iters, float a) {
    float s[8];
    for (int j = 0; j < 8; ++j) s[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = fmaf(s[j], a, 1.0f);
    float t = 0; for (int j = 0; j < 8; ++j) t += s[j];
    if (t == 12345.0f) out[0] = t;
}
__global__ void k_dfma1(double* out, int iters, double a) {   // one chain: latency
    double s = threadIdx.x;
    for (int i = 0; i < iters; ++i) s = fma(s, a, 1.0);
    if (s == 12345.0) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    const double ops = double(blocks) * threads * iters * 8;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(d, iters, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("DFMA  %.2f T/s (%.1f per clk per SM at 1.965 GHz)\n", ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(e0); k_f2f<<<blocks, threads>>>(d, iters, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("F2F   %.2f T/s (%.1f per clk per SM) [+FADD each]\n", ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(e0); k_ffma<<<blocks, threads>>>((float*)d, iters, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("FFMA  %.2f T/s (%.1f per clk per SM)\n", ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(e0); k_dfma1<<<148, 32>>>(d, iters * 8, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("DFMA dependent-chain latency %.1f cycles\n", ms * 1e-3 * 1.965e9 / (iters * 8));
    }
    return 0;
}
