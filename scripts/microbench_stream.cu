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


// K2-structure mimic: super-tiles of 8 x 16 KiB sub-tiles, 4-stage ring.
// F_TICKET: dynamic atomic ticket per super-tile (else static round robin)
// F_SYNC:   4 __syncthreads per super-tile (else 1, needed to publish s_next)
// F_LB:     warp 0 reads 256 status words (8/lane, relaxed.gpu) + publishes one
template <int F_TICKET, int F_SYNC, int F_LB>
__global__ void __launch_bounds__(256, 2) k2mimic(const float4* __restrict__ a, unsigned ntiles, unsigned* ticket,
                                                  unsigned long long* status, float* out) {
    constexpr int STAGES = 4, V = 1024, SUB = 8;
    extern __shared__ __align__(128) float4 ring[];
    __shared__ unsigned long long full[STAGES], empty[STAGES];
    __shared__ unsigned s_next;
    __shared__ unsigned long long s_pre;
    const unsigned kProd = 224;
    unsigned issued = 0, ptile = 0, pnext = 0xffffffffu, pk = 0;
    unsigned static_t = blockIdx.x;
    auto get_ticket = [&]() -> unsigned {
        if (F_TICKET) return atomicAdd(ticket, 1u);
        const unsigned t = static_t;
        static_t += gridDim.x;
        return t;
    };
    auto produce = [&](unsigned upto) {
        while (issued < upto) {
            const unsigned kk = issued / SUB;
            unsigned t;
            if (kk == pk) t = ptile;
            else {
                if (pnext == 0xffffffffu) { pnext = get_ticket(); s_next = pnext; }
                t = pnext;
            }
            if (t >= ntiles) return;
            const unsigned st = issued % STAGES;
            if (issued >= STAGES) mbar_wait(&empty[st], ((issued / STAGES) - 1) & 1);
            mbar_expect_tx(&full[st], 16384);
            bulk_g2s(&ring[st * V], a + (size_t)t * V * SUB + (issued % SUB) * V, 16384, &full[st]);
            ++issued;
        }
    };
    if (threadIdx.x == kProd) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        ptile = get_ticket();
        s_next = ptile;
        produce(STAGES);
    }
    __syncthreads();
    unsigned tile = s_next;
    float acc = 0.f;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned k = 0;; ++k) {
        const bool have = tile < ntiles;
        if (have) {
            for (int sub = 0; sub < SUB; ++sub) {
                const unsigned seq = k * SUB + sub;
                if (threadIdx.x == kProd) produce(seq + STAGES);
                mbar_wait(&full[seq % STAGES], (seq / STAGES) & 1);
                for (int u = 0; u < 4; ++u) {
                    const float4 v = ring[(seq % STAGES) * V + u * 256 + threadIdx.x];
                    acc += v.x + v.y + v.z + v.w;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[seq % STAGES]);
            }
            if (threadIdx.x == kProd) {
                if (pnext == 0xffffffffu) { pnext = get_ticket(); s_next = pnext; }
                produce((k + 1) * SUB + STAGES);
            }
        }
        __syncthreads();
        const unsigned next = have ? s_next : 0xffffffffu;
        if (F_SYNC) __syncthreads();
        if (F_LB && have && warp == 0) {
            // F_LB: 1 = 8 x 8B/lane contiguous, 2 = 1 x 8B/lane, 3 = 8 x 4B/lane,
            //       4 = 8 x 8B/lane one word per 128B line, 5 = one word per 32B sector,
            //       6 = two-level: 1 tile word + 1 group word per lane, atomicAdd group
            constexpr int STR = F_LB == 4 ? 16 : (F_LB == 5 ? 4 : 1);
            constexpr int R = (F_LB == 2 || F_LB == 6) ? 1 : 8;
            if (lane == 0) {
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(status + (size_t)tile * STR), "l"((unsigned long long)k) : "memory");
                if (F_LB == 6) atomicAdd(status + (1u << 22) + (tile >> 5), 1ull);
            }
            unsigned long long s = 0;
            for (int r = 0; r < R; ++r) {
                const long long j = (long long)tile - 1 - (r * 32 + lane);
                unsigned long long x = 0;
                if (j >= 0) {
                    if (F_LB == 3) {
                        unsigned y;
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(y) : "l"(reinterpret_cast<unsigned*>(status) + j) : "memory");
                        x = y;
                    } else {
                        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(status + (size_t)j * STR) : "memory");
                    }
                }
                if (F_LB == 6) {
                    const long long gj = (long long)(tile >> 5) - 1 - lane;
                    unsigned long long y = 0;
                    if (gj >= 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(y) : "l"(status + (1u << 22) + gj) : "memory");
                    x += y;
                }
                s += x;
            }
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) s_pre = s;
        }
        if (F_SYNC) __syncthreads();
        if (F_SYNC) __syncthreads();
        if (!have) break;
        tile = next;
        if (threadIdx.x == kProd) { pk += 1; ptile = pnext; pnext = 0xffffffffu; }
    }
    if (acc == 123.f) out[0] = acc + (float)s_pre;
}

template <int T, int S, int L>
void run_mimic(const float4* d, size_t n4, unsigned* ticket, unsigned long long* status, float* out, int sms) {
    const int smem = 4 * 16384;
    cudaFuncSetAttribute(k2mimic<T, S, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const unsigned ntiles = (unsigned)(n4 / 8192);
    const float ms = timeit([&] {
        cudaMemsetAsync(ticket, 0, 4);
        k2mimic<T, S, L><<<sms * 2, 256, smem>>>(d, ntiles, ticket, status, out);
    });
    printf("mimic ticket=%d sync=%d lookback=%d : %.3f ms  %.0f GB/s\n", T, S, L, ms, n4 * 16.0 / ms / 1e6);
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
    setvbuf(stdout, nullptr, _IONBF, 0);
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

    unsigned* ticket;
    unsigned long long* status;
    cudaMalloc(&ticket, 4);
    cudaMalloc(&status, (8u << 22) * 8);
    cudaMemset(status, 0, (8u << 22) * 8);
    run_mimic<1, 1, 0>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 1>(d, n4, ticket, status, out, sms);
    run_mimic<0, 1, 1>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 2>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 3>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 4>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 5>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 6>(d, n4, ticket, status, out, sms);
    run_mimic<1, 1, 1>(d, n4, ticket, status, out, sms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
