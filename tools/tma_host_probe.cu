// Probe: random 512-byte row gather from a pinned host table (UVA) into HBM, by
//  (a) SM loads: one warp per row, 16-byte vectors (the K4 gather's host-tier path), and
//  (b) TMA bulk copies: one elected lane per CTA issues cp.async.bulk global->shared
//      (mbarrier complete_tx) for R rows, then bulk shared->global stores; a 32-thread
//      CTA keeps R rows in flight with almost no issue slots or registers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_host_probe.cu
// Run:   /tmp/tma_probe [table_GiB] [rows]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

constexpr int kRowBytes = 512;

__global__ void k_gather_sm(const uint4* __restrict__ table, const uint32_t* __restrict__ ids, uint64_t rows,
                            uint4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < rows; r += nw) {
        const uint64_t src = (uint64_t)ids[r] * (kRowBytes / 16);
        out[r * (kRowBytes / 16) + lane] = table[src + lane];  // 32 lanes x 16 B = 512 B
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// issue-bound filler shaped like the hop kernel (6 x 256-thread CTAs per SM, 40 regs)
__global__ void __launch_bounds__(256, 6) k_spin(uint32_t iters, uint32_t* sink) {
    uint32_t a = threadIdx.x, b = blockIdx.x;
    for (uint32_t i = 0; i < iters; ++i) {
        a = a * 1664525u + b;
        b = min(a ^ b, b + 7u);
    }
    if (a == 0x12345678u) sink[0] = b;
}

template <int R>
__global__ void __launch_bounds__(32) k_gather_tma(const char* __restrict__ table, const uint32_t* __restrict__ ids,
                                                   uint64_t rows, char* __restrict__ out) {
    __shared__ __align__(128) char buf[R][kRowBytes];
    __shared__ __align__(8) uint64_t bar[R];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < R; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase = 0;
    const uint64_t step = (uint64_t)gridDim.x * R;
    for (uint64_t r0 = (uint64_t)blockIdx.x * R; r0 < rows; r0 += step) {
        const int n = (int)((rows - r0) < (uint64_t)R ? (rows - r0) : (uint64_t)R);
        for (int s = 0; s < n; ++s) {
            const char* src = table + (uint64_t)ids[r0 + s] * kRowBytes;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                         "r"(kRowBytes));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(buf[s])),
                "l"(src), "r"(kRowBytes), "r"(smem_u32(&bar[s]))
                : "memory");
        }
        for (int s = 0; s < n; ++s) {
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(smem_u32(&bar[s])), "r"(phase)
                    : "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (r0 + s) * kRowBytes),
                         "r"(smem_u32(buf[s])), "r"(kRowBytes)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        phase ^= 1;
        // slots that got no load this round keep their phase: only full rounds repeat
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const double gib = argc > 1 ? atof(argv[1]) : 16.0;
    const uint64_t rows = argc > 2 ? strtoull(argv[2], 0, 10) : (1ull << 21);
    const uint64_t table_rows = (uint64_t)(gib * (1ull << 30)) / kRowBytes;
    char* host = nullptr;
    CK(cudaHostAlloc(&host, table_rows * kRowBytes, cudaHostAllocMapped));
    for (uint64_t i = 0; i < table_rows * kRowBytes; i += 4096) host[i] = (char)i;  // touch
    char* dtable = nullptr;
    CK(cudaHostGetDevicePointer((void**)&dtable, host, 0));
    uint32_t* hid = (uint32_t*)malloc(rows * 4);
    uint64_t x = 88172645463325252ull;
    for (uint64_t i = 0; i < rows; ++i) {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        hid[i] = (uint32_t)(x % table_rows);
    }
    uint32_t* ids;
    char* out;
    CK(cudaMalloc(&ids, rows * 4));
    CK(cudaMalloc(&out, rows * kRowBytes));
    CK(cudaMemcpy(ids, hid, rows * 4, cudaMemcpyHostToDevice));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto run = [&](const char* name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        ms /= 3;
        printf("%-34s %8.3f ms  %6.1f GB/s  %6.1f Mrows/s\n", name, ms, rows * kRowBytes / (ms * 1e6),
               rows / (ms * 1e3));
    };
    printf("table %.1f GiB pinned (cudaHostAlloc), %llu random 512-byte rows, %d SMs\n", gib,
           (unsigned long long)rows, sms);
    for (int ctas : {1, 4, 16})
        run(ctas == 16 ? "SM loads, 16 x 256-thread CTAs/SM" : ctas == 4 ? "SM loads, 4 x 256-thread CTAs/SM"
                                                                         : "SM loads, 1 x 256-thread CTA/SM",
            [&] { k_gather_sm<<<sms * ctas, 256>>>((const uint4*)dtable, ids, rows, (uint4*)out); });
    run("TMA, 1 x 32-thread CTA/SM, R=32", [&] { k_gather_tma<32><<<sms, 32>>>(dtable, ids, rows, out); });
    run("TMA, 2 x 32-thread CTAs/SM, R=32", [&] { k_gather_tma<32><<<sms * 2, 32>>>(dtable, ids, rows, out); });
    run("TMA, 4 x 32-thread CTAs/SM, R=32", [&] { k_gather_tma<32><<<sms * 4, 32>>>(dtable, ids, rows, out); });
    run("TMA, 4 x 32-thread CTAs/SM, R=64", [&] { k_gather_tma<64><<<sms * 4, 32>>>(dtable, ids, rows, out); });
    // the host-row gather concurrent with other work on a second stream: HBM copies
    // (memory-bound) or a spin kernel that keeps every SM's issue slots busy
    {
        cudaStream_t s1, s2;
        CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        char *big_a, *big_b;
        const size_t big = 8ull << 30;
        CK(cudaMalloc(&big_a, big));
        CK(cudaMalloc(&big_b, big));
        for (int mode = 0; mode < 3; ++mode) {
            if (mode == 2)  // the filler reserves the whole carveout for shared memory: room for TMA CTAs
                CK(cudaFuncSetAttribute(k_spin, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            cudaEvent_t h0, h1;
            CK(cudaEventCreate(&h0));
            CK(cudaEventCreate(&h1));
            CK(cudaDeviceSynchronize());
            for (int i = 0; i < 6; ++i) {
                if (mode == 0)
                    CK(cudaMemcpyAsync(big_b, big_a, big, cudaMemcpyDeviceToDevice, s2));
                else
                    k_spin<<<sms * 6, 256, 0, s2>>>(4000000u, (uint32_t*)big_b);
            }
            CK(cudaEventRecord(h0, s1));
            k_gather_tma<32><<<sms * 2, 32, 0, s1>>>(dtable, ids, rows, out);
            CK(cudaEventRecord(h1, s1));
            CK(cudaDeviceSynchronize());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, h0, h1));
            printf("TMA host gather while %-28s %8.3f ms  %6.1f GB/s\n",
                   mode == 0 ? "8 GB D2D copies run:" : mode == 1 ? "SMs spin (hop-like occupancy):" : "SMs spin, carveout 100% smem:", ms, rows * kRowBytes / (ms * 1e6));
        }
    }
    // correctness of the TMA copy against the table
    char* check = (char*)malloc(rows * kRowBytes);
    CK(cudaMemcpy(check, out, rows * kRowBytes, cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (uint64_t i = 0; i < rows; i += 997)
        for (int k = 0; k < kRowBytes; k += 64) bad += check[i * kRowBytes + k] != host[(uint64_t)hid[i] * kRowBytes + k];
    printf("TMA rows checked against the table: %s\n", bad ? "MISMATCH" : "ok");
    return 0;
}
