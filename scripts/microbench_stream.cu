// microbench_stream.cu — read bandwidth of streaming patterns on one B200
// (perf experiment; not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_stream.cu && ./mb
// Patterns: (1) LDG.128 grid-stride with register double buffering,
// (2) cp.async.bulk ring: STAGES x BYTES per block, consumer sums the stage.
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile("{\n .reg .pred P1;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W_%=;\n }" ::"r"(
                     smem_u32(bar)), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(256, 2) ldg_kernel(const float4* __restrict__ a, size_t n4, float* out) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * 256 * 4;
    size_t i = (size_t)blockIdx.x * 256 * 4 + threadIdx.x;
    float4 v[4], w[4];
    bool have = i + 3 * 256 < n4;
    if (have)
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(a + i + u * 256);
    while (have) {
        const size_t j = i + stride;
        const bool more = j + 3 * 256 < n4;
        if (more)
            for (int u = 0; u < 4; ++u) w[u] = __ldcs(a + j + u * 256);
        for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        i = j;
        have = more;
        for (int u = 0; u < 4; ++u) v[u] = w[u];
    }
    if (acc == 123.f) out[0] = acc;
}

template <int STAGES, int BYTES>
__global__ void __launch_bounds__(256) tma_kernel(const float4* __restrict__ a, size_t n4, float* out) {
    extern __shared__ __align__(128) float4 ring[];
    __shared__ unsigned long long full[STAGES], empty[STAGES];
    constexpr int V = BYTES / 16;
    const size_t nchunks = n4 / V;
    const unsigned mine = blockIdx.x < nchunks ? (unsigned)((nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned issued = 0;
    auto produce = [&](unsigned upto) {
        while (issued < upto && issued < mine) {
            const unsigned st = issued % STAGES;
            if (issued >= STAGES) mbar_wait(&empty[st], ((issued / STAGES) - 1) & 1);
            mbar_expect_tx(&full[st], BYTES);
            bulk_g2s(&ring[st * V], a + (size_t)(blockIdx.x + (size_t)issued * gridDim.x) * V, BYTES, &full[st]);
            ++issued;
        }
    };
    if (threadIdx.x == 0) produce(STAGES);
    float acc = 0.f;
    for (unsigned i = 0; i < mine; ++i) {
        if (threadIdx.x == 0) produce(i + STAGES);
        const unsigned st = i % STAGES;
        mbar_wait(&full[st], (i / STAGES) & 1);
        for (int k = threadIdx.x; k < V; k += 256) {
            const float4 v = ring[st * V + k];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[st]);
    }
    if (acc == 123.f) out[0] = acc;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

template <int STAGES, int BYTES>
void run_tma(const float4* d, size_t n4, float* out, int sms, int per_sm) {
    const int smem = STAGES * BYTES;
    cudaFuncSetAttribute(tma_kernel<STAGES, BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const float ms = timeit([&] { tma_kernel<STAGES, BYTES><<<sms * per_sm, 256, smem>>>(d, n4, out); });
    printf("tma  stages=%d bytes=%6d blocks/SM=%d : %.3f ms  %.0f GB/s\n", STAGES, BYTES, per_sm, ms,
           n4 * 16.0 / ms / 1e6);
}

int main() {
    const size_t bytes = 16ull << 30;
    const size_t n4 = bytes / 16;
    float4* d;
    float* out;
    cudaMalloc(&d, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(d, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per_sm = 2; per_sm <= 4; per_sm += 2) {
        const float ms = timeit([&] { ldg_kernel<<<sms * per_sm, 256>>>(d, n4, out); });
        printf("ldg  4xfloat4 dbl-buf blocks/SM=%d : %.3f ms  %.0f GB/s\n", per_sm, ms, n4 * 16.0 / ms / 1e6);
    }
    run_tma<4, 16384>(d, n4, out, sms, 2);
    run_tma<4, 16384>(d, n4, out, sms, 3);
    run_tma<8, 16384>(d, n4, out, sms, 1);
    run_tma<6, 16384>(d, n4, out, sms, 2);
    run_tma<4, 32768>(d, n4, out, sms, 1);
    run_tma<3, 32768>(d, n4, out, sms, 2);
    run_tma<8, 8192>(d, n4, out, sms, 2);
    run_tma<12, 8192>(d, n4, out, sms, 2);
    run_tma<16, 4096>(d, n4, out, sms, 2);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
