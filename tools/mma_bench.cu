// Microbenchmark: issue rate of tcgen05.mma.kind::tf32 (cta_group::1, M=128,
// K=8) by one elected thread, A from TMEM ("ts") or shared memory ("ss"),
// N = 64/128/256, issuing thread chosen by `lane == 0` or by elect.sync.
// Reports cycles per MMA (clock64 around ITER MMAs + commit + wait).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\t@P1 mov.b32 %0, 1;\n\t}" : "+r"(pred));
    return pred != 0;
}

template <int N, bool ATMEM, bool ELECT>
__global__ void __launch_bounds__(128, 1) bench(long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 0.001f * (i & 255);
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t sb = smem_u32(smem);
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        bool leader = ELECT ? elect_one() : (lane == 0);
        t0 = clock64();
        if (leader) {
            for (int i = 0; i < iters; ++i) {
                const uint32_t d = tmem + 256;
                const uint64_t bd = desc(sb + 32768 + (i & 7) * 256, 128, 256);
                if (ATMEM) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(tmem + 8 * (i & 15)), "l"(bd), "r"(idesc), "r"((uint32_t)(i > 0)) : "memory");
                } else {
                    const uint64_t ad = desc(sb + (i & 7) * 256, 128, 256);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(i > 0)) : "memory");
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
        if (lane == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool ATMEM, bool ELECT>
void run(const char *name, long long *d, int iters, int grid) {
    auto k = bench<N, ATMEM, ELECT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<grid, 128, 64 * 1024>>>(d, iters);
    cudaDeviceSynchronize();
    k<<<grid, 128, 64 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += h[i];
    avg /= grid;
    printf("%-28s N=%3d iters=%d grid=%d: %.1f cycles/MMA  (%s)\n", name, N, iters, grid, avg / iters, cudaGetErrorString(e));
}

int main() {
    long long *d;
    cudaMalloc(&d, sizeof(long long) * 148);
    const int it = 4096;
    for (int grid : {1, 148}) {
        run<64, true, false>("ts lane0", d, it, grid);
        run<64, true, true>("ts elect", d, it, grid);
        run<128, true, true>("ts elect", d, it, grid);
        run<256, true, true>("ts elect", d, it, grid);
        run<64, false, true>("ss elect", d, it, grid);
        run<128, false, true>("ss elect", d, it, grid);
        run<256, false, true>("ss elect", d, it, grid);
    }
    return 0;
}
