// Throughput of the instruction classes the frame gather uses (B200, sm_100a):
// F2F.F64.F32, I2F.F64, F2I.F64 (rounding conversions), DADD, DFMA, FFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu xu.cu && ./xu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096, CH = 8;

__global__ void k_f2f(const float* in, double* out) {
    float v[CH]; long long acc[CH];
    for (int c = 0; c < CH; c++) { v[c] = in[threadIdx.x + c]; acc[c] = 0; }
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) { acc[c] ^= __double_as_longlong((double)v[c]); v[c] = __int_as_float(__float_as_int(v[c]) + 1); }
    double s = 0; for (int c = 0; c < CH; c++) s += (double)acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_i2f(const int* in, double* out) {
    int v[CH]; long long acc[CH];
    for (int c = 0; c < CH; c++) { v[c] = in[threadIdx.x + c]; acc[c] = 0; }
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) { acc[c] ^= __double_as_longlong((double)v[c]); v[c] += 1; }
    double s = 0; for (int c = 0; c < CH; c++) s += (double)acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f2i(const double* in, double* out) {
    double v[CH]; int acc[CH];
    for (int c = 0; c < CH; c++) { v[c] = in[threadIdx.x + c]; acc[c] = 0; }
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) { acc[c] += __double2int_rd(v[c]); v[c] = __longlong_as_double(__double_as_longlong(v[c]) ^ 1); }
    double s = 0; for (int c = 0; c < CH; c++) s += acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(const double* in, double* out) {
    double v[CH];
    for (int c = 0; c < CH; c++) v[c] = in[threadIdx.x + c];
    const double d = in[0] * 1e-30;
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) v[c] = __dadd_rn(v[c], d);
    double s = 0; for (int c = 0; c < CH; c++) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(const double* in, double* out) {
    double v[CH];
    for (int c = 0; c < CH; c++) v[c] = in[threadIdx.x + c];
    const double d = in[0] * 1e-30, m = 1.0 + in[1] * 1e-30;
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) v[c] = __fma_rn(v[c], m, d);
    double s = 0; for (int c = 0; c < CH; c++) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(const double* in, double* out) {
    float v[CH];
    for (int c = 0; c < CH; c++) v[c] = (float)in[threadIdx.x + c];
    const float d = (float)in[0] * 1e-30f, m = 1.0f + (float)in[1] * 1e-30f;
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) v[c] = fmaf(v[c], m, d);
    double s = 0; for (int c = 0; c < CH; c++) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_frnd(const double* in, double* out) {
    double v[CH]; long long acc[CH];
    for (int c = 0; c < CH; c++) { v[c] = in[threadIdx.x + c] + 0.5; acc[c] = 0; }
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) { acc[c] ^= __double_as_longlong(floor(v[c])); v[c] = __longlong_as_double(__double_as_longlong(v[c]) + 1); }
    double s = 0; for (int c = 0; c < CH; c++) s += (double)acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_d2f(const double* in, double* out) {
    double v[CH]; int acc[CH];
    for (int c = 0; c < CH; c++) { v[c] = in[threadIdx.x + c] + 0.5; acc[c] = 0; }
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) { acc[c] ^= __float_as_int((float)v[c]); v[c] = __longlong_as_double(__double_as_longlong(v[c]) + (1ll << 30)); }
    double s = 0; for (int c = 0; c < CH; c++) s += (double)acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_lop(const double* in, double* out) {
    int v[CH];
    for (int c = 0; c < CH; c++) v[c] = (int)in[threadIdx.x + c];
    const int m = (int)in[0] + 0x1234;
    for (int i = 0; i < ITERS; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) v[c] = (v[c] ^ m) + c;
    double s = 0; for (int c = 0; c < CH; c++) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class F, class T>
void run(const char* name, F kern, T* in, double* out, int sms) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256;
    kern<<<blocks, threads>>>(in, out);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(in, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = (double)blocks * threads * ITERS * CH;
    const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
    printf("%-8s %8.3f ms  %7.1f thread-ops/clk/SM  (%.1f warp-instr/clk/SM)\n", name, ms, per_clk_sm, per_clk_sm / 32);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* fin; int* iin; double* din; double* out;
    cudaMalloc(&fin, 4096 * 4); cudaMalloc(&iin, 4096 * 4); cudaMalloc(&din, 4096 * 8);
    cudaMalloc(&out, (size_t)sms * 8 * 256 * 8);
    cudaMemset(fin, 0, 4096 * 4); cudaMemset(iin, 0, 4096 * 4); cudaMemset(din, 0, 4096 * 8);
    run("F2F.F64", k_f2f, fin, out, sms);
    run("I2F.F64", k_i2f, iin, out, sms);
    run("F2I.F64", k_f2i, din, out, sms);
    run("DADD", k_dadd, din, out, sms);
    run("DFMA", k_dfma, din, out, sms);
    run("FFMA", k_ffma, din, out, sms);
    run("FRND.F64", k_frnd, din, out, sms);
    run("F2F.F32.F64", k_d2f, din, out, sms);
    run("IADD+LOP", k_lop, din, out, sms);
    return 0;
}
