// Error of the tensor-core gate's 32-column chunk sums (csrc/gate.cu gate_fwd_mma_kernel): two
// chained mma.sync m16n8k16 bf16 -> f32 from a zero accumulator, against the exact (f64) sum of
// the same bf16 products.  Prints, per input family, max |D - exact| / sum|products| over all
// (expert, token) chunk results -- the constant kGateEps (2^-17) must bound it with margin.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/gate_err_probe tools/probes/gate_err_probe.cu
#include <cuda_bf16.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// one warp per problem: W (16 x 32 bf16, row-major), X (8 x 32 bf16, row-major); out 16 x 8 f32
__global__ void chunk(const uint16_t* w, const uint16_t* x, float* out, int problems) {
    const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (p >= problems) return;
    const int g = lane >> 2, q = lane & 3;
    const uint4 wa = *reinterpret_cast<const uint4*>(w + (size_t)p * 512 + g * 32 + 8 * q);
    const uint4 wb = *reinterpret_cast<const uint4*>(w + (size_t)p * 512 + (g + 8) * 32 + 8 * q);
    const uint4 xv = *reinterpret_cast<const uint4*>(x + (size_t)p * 256 + g * 32 + 8 * q);
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    mma(d, wa.x, wb.x, wa.y, wb.y, xv.x, xv.y);
    mma(d, wa.z, wb.z, wa.w, wb.w, xv.z, xv.w);
    for (int i = 0; i < 4; ++i) {
        const int e = g + 8 * (i >> 1), t = 2 * q + (i & 1);
        out[(size_t)p * 128 + e * 8 + t] = d[i];
    }
}

static uint16_t to_bf16(float f) {   // round to nearest even
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static double from_bf16(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    const int P = 1 << 16;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::uniform_real_distribution<double> ud(0.0, 1.0);
    const char* names[5] = {"normal", "log-uniform 2^-20..2^20", "cancelling pairs", "one large + small",
                            "equal magnitudes, random signs"};
    uint16_t *dw, *dx;
    float* dout;
    cudaMalloc(&dw, (size_t)P * 512 * 2);
    cudaMalloc(&dx, (size_t)P * 256 * 2);
    cudaMalloc(&dout, (size_t)P * 128 * 4);
    std::vector<uint16_t> w((size_t)P * 512), x((size_t)P * 256);
    std::vector<float> out((size_t)P * 128);
    printf("{");
    for (int fam = 0; fam < 5; ++fam) {
        auto gen = [&](int i) -> double {
            switch (fam) {
                case 0: return nd(rng);
                case 1: return (ud(rng) < 0.5 ? -1 : 1) * std::exp2(-20.0 + 40.0 * ud(rng));
                case 2: return (i & 1 ? -1 : 1) * (1.0 + std::ldexp(ud(rng), -6)) * std::exp2(std::floor(8 * ud(rng)));
                case 3: return (i % 32 == 0) ? 4096.0 * (1 + ud(rng)) : std::ldexp(nd(rng), -8);
                default: return (ud(rng) < 0.5 ? -1 : 1) * (1.0 + std::ldexp(std::floor(128 * ud(rng)), -7));
            }
        };
        for (size_t i = 0; i < w.size(); ++i) w[i] = to_bf16((float)gen((int)i));
        for (size_t i = 0; i < x.size(); ++i) x[i] = to_bf16((float)gen((int)i));
        cudaMemcpy(dw, w.data(), w.size() * 2, cudaMemcpyHostToDevice);
        cudaMemcpy(dx, x.data(), x.size() * 2, cudaMemcpyHostToDevice);
        chunk<<<P / 8, 256>>>(dw, dx, dout, P);
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0.0, worst_ulp = 0.0;
        for (int p = 0; p < P; ++p)
            for (int e = 0; e < 16; ++e)
                for (int t = 0; t < 8; ++t) {
                    double ex = 0.0, ab = 0.0, mx = 0.0;
                    for (int c = 0; c < 32; ++c) {
                        const double pr = from_bf16(w[(size_t)p * 512 + e * 32 + c]) * from_bf16(x[(size_t)p * 256 + t * 32 + c]);
                        ex += pr;   // f64 sum: error <= 2^-48 sum|p|, far below the ratios measured
                        ab += std::fabs(pr);
                        mx = std::fmax(mx, std::fabs(pr));
                    }
                    const double err = std::fabs((double)out[(size_t)p * 128 + e * 8 + t] - ex);
                    if (ab > 0) worst = std::fmax(worst, err / ab);
                    if (mx > 0) worst_ulp = std::fmax(worst_ulp, err / (mx * std::ldexp(1.0, -23)));
                }
        printf("%s\"%s\": {\"max_err_over_abs_sum\": %.3e, \"log2\": %.2f, \"max_err_in_ulps_of_max_product\": %.2f}",
               fam ? ", " : "", names[fam], worst, worst > 0 ? std::log2(worst) : -999.0, worst_ulp);
    }
    printf(", \"kGateEps\": %.3e, \"chunks_per_family\": %d}\n", std::ldexp(1.0, -17), P * 128);
    return 0;
}
