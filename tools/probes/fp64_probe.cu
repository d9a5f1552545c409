// Throughput of FP64 on sm_100a: DMMA m8n8k4 vs DFMA, many independent chains.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
    double c[CH][2];
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
    double s = 0;
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
    double c[CH];
    for (int i = 0; i < CH; ++i) c[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) c[i] = fma(c[i], a, b);
    double s = 0;
    for (int i = 0; i < CH; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_cvt(double* out, int iters, const float* in) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = in[(threadIdx.x + i) & 255];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i] = acc[i] + (double)x[i];   // F2F + DADD
            x[i] = __int_as_float(__float_as_int(x[i]) ^ 1);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            k_dmma<4><<<148, warps * 32>>>(out, iters, 1.0000001, 0.999999);
            cudaEventRecord(e0);
            k_dmma<4><<<148, warps * 32>>>(out, iters, 1.0000001, 0.999999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = 148.0 * warps * iters * 4 * 512.0;   // 8x8x4 x 2 flops per warp-DMMA
            if (rep) printf("DMMA  warps/SM=%2d chains=4: %.3f ms  %.1f TFLOP/s  (%.1f cyc/DMMA/SMSP at 1.9GHz)\n", warps, ms,
                            fl / ms / 1e9, ms * 1e-3 * 1.9e9 / (warps / 4.0 * iters * 4));
        }
        for (int rep = 0; rep < 2; ++rep) {
            k_dfma<8><<<148, warps * 32>>>(out, iters, 1.0000001, 0.999999);
            cudaEventRecord(e0);
            k_dfma<8><<<148, warps * 32>>>(out, iters, 1.0000001, 0.999999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = 148.0 * warps * 32 * iters * 8 * 2.0;
            if (rep) printf("DFMA  warps/SM=%2d chains=8: %.3f ms  %.1f TFLOP/s\n", warps, ms, fl / ms / 1e9);
        }
    }
    {
        float* in;
        cudaMalloc(&in, 256 * 4);
        cudaMemset(in, 0, 256 * 4);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_cvt<<<148, 512>>>(out, iters, in);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double ops = 148.0 * 512 * iters * 8;
            if (rep) printf("F2F.F64.F32+DADD: %.3f ms  %.1f G conv/s  (%.2f per clk per SM at 1.9 GHz)\n", ms,
                            ops / ms / 1e6, ops / (ms * 1e-3) / 1.9e9 / 148);
        }
    }
    for (int ch : {1, 2, 4}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (ch == 1) k_dmma<1><<<148, 128>>>(out, iters, 1.0000001, 0.999999);
            if (ch == 2) k_dmma<2><<<148, 128>>>(out, iters, 1.0000001, 0.999999);
            if (ch == 4) k_dmma<4><<<148, 128>>>(out, iters, 1.0000001, 0.999999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = 148.0 * 4 * iters * ch * 512.0;
            if (rep) printf("DMMA 4 warps/SM chains=%d: %.1f TFLOP/s\n", ch, fl / ms / 1e9);
        }
    }
    // latency: one chain, one warp
    k_dmma<1><<<1, 32>>>(out, iters, 1.0000001, 0.999999);
    cudaEventRecord(e0);
    k_dmma<1><<<1, 32>>>(out, iters, 1.0000001, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA dependent-chain latency ~ %.1f ns/op\n", ms * 1e6 / iters);
    return 0;
}
