// Does cp.async.bulk (global -> shared, mbarrier completion) read a PEER GPU's memory over
// NVLink, and how fast?  One process, GPUs 0 and 1 with peer access enabled: GPU 0 gathers
// rows of a buffer on GPU 1 (and, for comparison, on GPU 0) through per-warp bulk-copy rings
// and writes them to a local buffer; the result is checked byte for byte.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peer_bulk_probe peer_bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kRow = 1024;      // bytes per bulk copy (512 bf16)
constexpr int kStages = 8;
constexpr int kWarps = 8;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kWarps * 32) gather(const char* __restrict__ src, char* __restrict__ dst, long long rows,
                                                      const int* __restrict__ perm) {
    extern __shared__ __align__(128) char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    char* ring = sm + warp * kStages * kRow;
    __shared__ __align__(8) uint64_t bars[kWarps][kStages];
    if (lane == 0)
        for (int s = 0; s < kStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bars[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long w = (long long)blockIdx.x * kWarps + warp, nw = (long long)gridDim.x * kWarps;
    const long long mine = w < rows ? (rows - 1 - w) / nw + 1 : 0;
    auto issue = [&](long long i) {
        const int st = (int)(i % kStages);
        const long long r = w + i * nw;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bars[warp][st])), "r"(kRow) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(ring + st * kRow)),
                     "l"(src + (long long)perm[r] * kRow), "r"(kRow), "r"(saddr(&bars[warp][st])) : "memory");
    };
    if (lane == 0)
        for (long long i = 0; i < mine && i < kStages - 1; ++i) issue(i);
    for (long long i = 0; i < mine; ++i) {
        if (lane == 0 && i + kStages - 1 < mine) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(i + kStages - 1);
        }
        const int st = (int)(i % kStages);
        const uint32_t par = (uint32_t)((i / kStages) & 1);
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(saddr(&bars[warp][st])), "r"(par) : "memory");
        const long long r = w + i * nw;
        const int4* s4 = reinterpret_cast<const int4*>(ring + st * kRow);
        int4* d4 = reinterpret_cast<int4*>(dst + r * kRow);
        for (int c = lane; c < kRow / 16; c += 32) d4[c] = s4[c];
        __syncwarp();
    }
}

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) { printf("{\"error\": \"needs 2 GPUs\"}\n"); return 0; }
    const long long rows = 64 * 1024;   // 64 MB
    const size_t bytes = rows * kRow;
    char *a1 = nullptr, *a0 = nullptr, *d0 = nullptr;
    int* perm = nullptr;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&a1, bytes));
    std::vector<unsigned char> h(bytes);
    for (size_t i = 0; i < bytes; ++i) h[i] = (unsigned char)((i * 2654435761u) >> 13);
    CK(cudaMemcpy(a1, h.data(), bytes, cudaMemcpyHostToDevice));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMalloc(&a0, bytes));
    CK(cudaMalloc(&d0, bytes));
    CK(cudaMemcpy(a0, h.data(), bytes, cudaMemcpyHostToDevice));
    std::vector<int> p(rows);
    for (long long i = 0; i < rows; ++i) p[i] = (int)((i * 40503) % rows);   // scattered rows
    CK(cudaMalloc(&perm, rows * sizeof(int)));
    CK(cudaMemcpy(perm, p.data(), rows * sizeof(int), cudaMemcpyHostToDevice));
    const int smem = kWarps * kStages * kRow;
    CK(cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{");
    for (int which = 0; which < 2; ++which) {
        const char* src = which ? a1 : a0;
        for (int ctas_per_sm : {1, 2, 3}) {
            const int grid = 148 * ctas_per_sm;
            CK(cudaMemset(d0, 0, bytes));
            gather<<<grid, kWarps * 32, smem>>>(src, d0, rows, perm);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                gather<<<grid, kWarps * 32, smem>>>(src, d0, rows, perm);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            std::vector<unsigned char> out(bytes);
            CK(cudaMemcpy(out.data(), d0, bytes, cudaMemcpyDeviceToHost));
            long long bad = 0;
            for (long long r = 0; r < rows; ++r)
                for (int c = 0; c < kRow; ++c) bad += out[r * kRow + c] != h[(long long)p[r] * kRow + c];
            printf("%s\"%s_ctas%d\": {\"GBs\": %.1f, \"mismatched_bytes\": %lld}", (which || ctas_per_sm > 1) ? ", " : "",
                   which ? "peer" : "local", ctas_per_sm, bytes / (best * 1e-3) / 1e9, bad);
        }
    }
    printf("}\n");
    return 0;
}
