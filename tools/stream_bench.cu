// Memory-pipeline micro-benchmark for the mode-H tensor-core pass (not part of
// the library).  It keeps apply_tcb's memory behaviour and drops its
// arithmetic: a persistent CTA per SM walks tiles of 2^(K+7) amplitudes (the
// 7 lowest bits plus K "target" bits, i.e. 2^K blocks of 1 KB), a producer
// warp group moves each K-half of a tile into a shared-memory ring with
// cp.async.bulk (one 1 KB copy per block), and NC consumer warps read a slot,
// release it, and write the same amplitudes back in place with 16-byte
// streaming stores.  Variants: ring depth (NS), consumer warps (NC), copy
// granularity (BLK bytes per cp.async.bulk; blocks of a contiguous tile part
// merge when the target bits allow it).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/stream_bench tools/stream_bench.cu
//   tools/stream_bench <log2 amplitudes> <reps> <targets, e.g. 8,9,10,20,21,22>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// store policy: 0 = st.global.cs (evict-first), 1 = st.global (default write-back)
template <int SP = 0>
__device__ __forceinline__ void st_cs(void *p, uint4 v) {
    if (SP == 0)
        asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else
        asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

struct P {
    uint64_t ntiles, tmask, step, base0[1];
    int ncopy;                 // copies per slot
    uint32_t cbytes;           // bytes per copy
    uint64_t coff[64];         // byte offset of copy j of K-half h: coff[h * ncopy + j]
    int pos[13], npos;
};

__device__ __forceinline__ uint64_t dep(uint64_t t, const P &p) {
    for (int i = 0; i < p.npos; ++i) { const int s = p.pos[i]; t = ((t >> s) << (s + 1)) | (t & ((1ull << s) - 1)); }
    return t;
}

__device__ unsigned long long g_fin[1024], g_start[1024];
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template <int NS, int NC, int NPW, int SP>
__global__ void __launch_bounds__((NC + NPW) * 32, 1) stream(char *psi, const __grid_constant__ P p, uint32_t slot_bytes) {
    if (threadIdx.x == 0) g_start[blockIdx.x] = gtime();
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sb = smem_u32(smem), bar = sb + NS * slot_bytes;
    auto rfull = [&](int s) { return bar + 8 * s; };
    auto rempty = [&](int s) { return bar + 8 * (NS + s); };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(rfull(s), 1); mbar_init(rempty(s), NC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t G = gridDim.x;
    const uint64_t tm = p.tmask, st = dep(G, p);
    if (warp >= NC) {          // producers: warp w handles K-half (w - NC) % 2 when NPW == 2
        const int pw = warp - NC;
        uint64_t base = dep(blockIdx.x, p) * 8;
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += G, ++it) {
            for (int h = (NPW == 1 ? 0 : pw); h < 2; h += NPW) {
                const uint32_t si = 2 * it + h;
                const int s = si % NS;
                mbar_wait(rempty(s), ((si / NS) & 1) ^ 1);
                if (lane == 0) mbar_arrive_tx(rfull(s), slot_bytes);
                __syncwarp();
                for (int j = lane; j < p.ncopy; j += 32)
                    bulk_g2s(sb + s * slot_bytes + j * p.cbytes, psi + base + p.coff[h * p.ncopy + j], p.cbytes, rfull(s));
            }
            base = (((base >> 3) | tm) + st & ~tm) * 8;
        }
    } else {
        uint64_t base = dep(blockIdx.x, p) * 8;
        uint32_t it = 0;
        constexpr int PER = 32 * 1024 / (NC * 32 * 16);     // 16-byte pieces per lane per 32 KB slot
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += G, ++it) {
            for (int h = 0; h < 2; ++h) {
                const uint32_t si = 2 * it + h;
                const int s = si % NS;
                mbar_wait(rfull(s), (si / NS) & 1);
                uint4 v[PER];
                uint32_t off[PER];
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    off[i] = ((i * NC + warp) * 32 + lane) * 16;
                    v[i] = *reinterpret_cast<const uint4 *>(smem + s * slot_bytes + off[i]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(rempty(s));
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const uint32_t j = off[i] / p.cbytes, r = off[i] % p.cbytes;
                    st_cs<SP>(psi + base + p.coff[h * p.ncopy + j] + r, v[i]);
                }
            }
            base = (((base >> 3) | tm) + st & ~tm) * 8;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) g_fin[blockIdx.x] = gtime();
}

// dynamic scheduling: a scheduler warp claims tiles (the first statically,
// then G + atomicAdd(ctr)) into a Q-entry shared queue that producers and
// consumers read in order; the counter resets itself when the last CTA exits
template <int NS, int NC>
__global__ void __launch_bounds__((NC + 3) * 32, 1) stream_dyn(char *psi, const __grid_constant__ P p, uint32_t slot_bytes,
                                                            unsigned long long *ctr) {
    constexpr int Q = 8;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sb = smem_u32(smem), bar = sb + NS * slot_bytes;
    auto rfull = [&](int s) { return bar + 8 * s; };
    auto rempty = [&](int s) { return bar + 8 * (NS + s); };
    auto qfull = [&](int q) { return bar + 8 * (2 * NS + q); };
    auto qempty = [&](int q) { return bar + 8 * (2 * NS + Q + q); };
    uint64_t *tq = reinterpret_cast<uint64_t *>(smem + NS * slot_bytes + 8 * (2 * NS + 2 * Q));
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(rfull(s), 1); mbar_init(rempty(s), NC); }
        for (int q = 0; q < Q; ++q) { mbar_init(qfull(q), 1); mbar_init(qempty(q), NC + 2); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t G = gridDim.x;
    auto next = [&](uint32_t it) -> uint64_t {      // tile of iteration it (all roles but the scheduler)
        const int q = it % Q;
        mbar_wait(qfull(q), (it / Q) & 1);
        const uint64_t t = *(volatile uint64_t *)&tq[q];
        __syncwarp();
        if (lane == 0) mbar_arrive(qempty(q));
        return t;
    };
    if (warp == NC + 2) {
        if (lane == 0) {
            for (uint32_t it = 0;; ++it) {
                const int q = it % Q;
                mbar_wait(qempty(q), ((it / Q) & 1) ^ 1);
                const uint64_t t = it == 0 ? blockIdx.x : G + atomicAdd(ctr, 1ull);
                tq[q] = t;
                mbar_arrive(qfull(q));
                if (t >= p.ntiles) break;
            }
        }
    } else if (warp >= NC) {
        const int h = warp - NC;
        for (uint32_t it = 0;; ++it) {
            const uint64_t t = next(it);
            if (t >= p.ntiles) break;
            const uint64_t base = dep(t, p) * 8;
            const uint32_t si = 2 * it + h;
            const int s = si % NS;
            mbar_wait(rempty(s), ((si / NS) & 1) ^ 1);
            if (lane == 0) mbar_arrive_tx(rfull(s), slot_bytes);
            __syncwarp();
            for (int j = lane; j < p.ncopy; j += 32)
                bulk_g2s(sb + s * slot_bytes + j * p.cbytes, psi + base + p.coff[h * p.ncopy + j], p.cbytes, rfull(s));
        }
    } else {
        constexpr int PER = 32 * 1024 / (NC * 32 * 16);
        for (uint32_t it = 0;; ++it) {
            const uint64_t t = next(it);
            if (t >= p.ntiles) break;
            const uint64_t base = dep(t, p) * 8;
            for (int h = 0; h < 2; ++h) {
                const uint32_t si = 2 * it + h;
                const int s = si % NS;
                mbar_wait(rfull(s), (si / NS) & 1);
                uint4 v[PER];
                uint32_t off[PER];
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    off[i] = ((i * NC + warp) * 32 + lane) * 16;
                    v[i] = *reinterpret_cast<const uint4 *>(smem + s * slot_bytes + off[i]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(rempty(s));
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const uint32_t j = off[i] / p.cbytes, r = off[i] % p.cbytes;
                    st_cs<0>(psi + base + p.coff[h * p.ncopy + j] + r, v[i]);
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        g_fin[blockIdx.x] = gtime();
        if (atomicAdd(ctr + 1, 1ull) == G - 1) {     // last CTA out: reset for the next launch
            ctr[0] = 0;
            ctr[1] = 0;
        }
    }
}

template <int NS, int NC>
float run_dyn(char *psi, const P &p, int reps, int sms) {
    const uint32_t slot = 32 * 1024;
    const int smem = NS * slot + 16 * NS + 16 * 8 + 8 * 8 + 64;
    CK(cudaFuncSetAttribute(stream_dyn<NS, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long *ctr;
    CK(cudaMalloc(&ctr, 16));
    CK(cudaMemset(ctr, 0, 16));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ms;
    for (int r = 0; r <= reps; ++r) {
        cudaEventRecord(a);
        stream_dyn<NS, NC><<<sms, (NC + 3) * 32, smem>>>(psi, p, slot, ctr);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float x;
        cudaEventElapsedTime(&x, a, b);
        if (r) ms.push_back(x);
    }
    {   // CTA start / finish spread of the last launch
        unsigned long long f[1024], st0[1024];
        cudaMemcpyFromSymbol(f, g_fin, sizeof(unsigned long long) * sms);
        cudaMemcpyFromSymbol(st0, g_fin, sizeof(unsigned long long) * sms);
        unsigned long long smin = ~0ull, smax = 0, fmin = ~0ull, fmax = 0;
        for (int i = 0; i < sms; ++i) {
            smin = std::min(smin, st0[i]); smax = std::max(smax, st0[i]);
            fmin = std::min(fmin, f[i]); fmax = std::max(fmax, f[i]);
        }
        std::vector<double> fin;
        for (int i = 0; i < sms; ++i) fin.push_back((f[i] - smin) * 1e-6);
        std::sort(fin.begin(), fin.end());
        printf("{\"dyn_spread_ms\": %.3f, \"finish_ms\": {\"min\": %.3f, \"p10\": %.3f, \"p50\": %.3f, \"p90\": %.3f, \"max\": %.3f}}\n",
               (smax - smin) * 1e-6, fin[0], fin[sms / 10], fin[sms / 2], fin[sms * 9 / 10], fin[sms - 1]);
    }
    cudaFree(ctr);
    float s = 0;
    for (int r = reps / 2; r < reps; ++r) s += ms[r];
    return s / (reps - reps / 2);
}

// reference: a plain in-place read + write of the whole array, 16 B per thread
template <int SP>
__global__ void plain(uint4 *psi, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = psi[i];
        st_cs<SP>(psi + i, v);
    }
}
// reference 2: non-persistent, one 4 x 16 B unit per thread (the SIMT apply kernel's shape)
template <int SP>
__global__ void plain4(uint4 *psi, size_t n16) {
    const size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x);
    const size_t w = i >> 5, l = i & 31;
    uint4 v[4];
    for (int j = 0; j < 4; ++j) v[j] = psi[(w * 4 + j) * 32 + l];
    for (int j = 0; j < 4; ++j) st_cs<SP>(psi + (w * 4 + j) * 32 + l, v[j]);
}

// reference 3: persistent, U x 16 B per thread per iteration (all loads issued before the stores)
template <int U>
__global__ void plainP(uint4 *psi, size_t n16) {
    const size_t chunk = (size_t)blockDim.x * U;               // 16-byte units per block-iteration
    for (size_t b = blockIdx.x; b * chunk < n16; b += gridDim.x) {
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = psi[b * chunk + j * blockDim.x + threadIdx.x];
#pragma unroll
        for (int j = 0; j < U; ++j) st_cs<0>(psi + b * chunk + j * blockDim.x + threadIdx.x, v[j]);
    }
}

template <int NS, int NC, int NPW, int SP = 0>
float run(char *psi, const P &p, int reps, int sms) {
    const uint32_t slot = 32 * 1024;
    const int smem = NS * slot + 16 * NS + 64;
    CK(cudaFuncSetAttribute(stream<NS, NC, NPW, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream<NS, NC, NPW, SP><<<sms, (NC + NPW) * 32, smem>>>(psi, p, slot);
    CK(cudaDeviceSynchronize());
    std::vector<float> ms;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        stream<NS, NC, NPW, SP><<<sms, (NC + NPW) * 32, smem>>>(psi, p, slot);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float x;
        cudaEventElapsedTime(&x, a, b);
        ms.push_back(x);
    }
    float s = 0;
    for (int r = reps / 2; r < reps; ++r) s += ms[r];
    {   // CTA start / finish spread of the last launch
        unsigned long long f[1024], st0[1024];
        cudaMemcpyFromSymbol(f, g_fin, sizeof(unsigned long long) * sms);
        cudaMemcpyFromSymbol(st0, g_start, sizeof(unsigned long long) * sms);
        unsigned long long smin = ~0ull, smax = 0, fmin = ~0ull, fmax = 0;
        for (int i = 0; i < sms; ++i) {
            smin = std::min(smin, st0[i]); smax = std::max(smax, st0[i]);
            fmin = std::min(fmin, f[i]); fmax = std::max(fmax, f[i]);
        }
        std::vector<double> fin;
        for (int i = 0; i < sms; ++i) fin.push_back((f[i] - smin) * 1e-6);
        std::sort(fin.begin(), fin.end());
        printf("{\"cta_start_spread_ms\": %.3f, \"finish_ms\": {\"min\": %.3f, \"p10\": %.3f, \"p50\": %.3f, \"p90\": %.3f, \"max\": %.3f}}\n",
               (smax - smin) * 1e-6, fin[0], fin[sms / 10], fin[sms / 2], fin[sms * 9 / 10], fin[sms - 1]);
    }
    return s / (reps - reps / 2);
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 32;
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    std::vector<int> tg;
    {
        const char *s = argc > 3 ? argv[3] : "8,9,10,20,21,22";
        while (*s) { tg.push_back(atoi(s)); while (*s && *s != ',') ++s; if (*s) ++s; }
    }
    const int K = (int)tg.size();
    size_t bytes = (size_t)8 << n;
    char *psi;
    CK(cudaMalloc(&psi, bytes));
    CK(cudaMemset(psi, 0, bytes));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // tile bits: targets + the 7 lowest non-target bits
    std::vector<int> pos = tg;
    for (int b = 0, c = 0; c < 7; ++b) {
        bool t = false;
        for (int x : tg) t |= x == b;
        if (!t) { pos.push_back(b); ++c; }
    }
    std::sort(pos.begin(), pos.end());
    P p;
    memset(&p, 0, sizeof(p));
    p.npos = (int)pos.size();
    for (int i = 0; i < p.npos; ++i) { p.pos[i] = pos[i]; p.tmask |= 1ull << pos[i]; }
    p.ntiles = 1ull << (n - K - 7);
    const int hi = *std::max_element(tg.begin(), tg.end());
    for (int var = 0; var < 9; ++var) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float tot = 0;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(a);
            if (var == 0) plain<0><<<sms * 4, 512>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 1) plain<1><<<sms * 4, 512>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 2) plain4<0><<<(unsigned)(bytes / 16 / 4 / 128), 128>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 3) plain4<1><<<(unsigned)(bytes / 16 / 4 / 128), 128>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 4) plainP<4><<<sms * 8, 256>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 5) plainP<8><<<sms * 8, 256>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 6) plainP<16><<<sms * 4, 256>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 7) plainP<8><<<sms * 2, 512>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            if (var == 8) plainP<32><<<sms, 512>>>(reinterpret_cast<uint4 *>(psi), bytes / 16);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float x;
            cudaEventElapsedTime(&x, a, b);
            if (r >= reps / 2) tot += x;
        }
        const float ms = tot / (reps - reps / 2);
        const char *nm[9] = {"plain grid-stride .cs", "plain grid-stride default", "plain4 one-shot .cs", "plain4 one-shot default",
                             "persistent U4 8x256/SM", "persistent U8 8x256/SM", "persistent U16 4x256/SM", "persistent U8 2x512/SM", "persistent U32 1x512/SM"};
        printf("{\"n\": %d, \"variant\": \"%s\", \"ms\": %.3f, \"gbs\": %.1f}\n", n, nm[var], ms, 2.0 * bytes / ms / 1e6);
    }
    for (int gran : {1024, 2048, 4096}) {
        // copies of `gran` bytes: the block bits 0..6 plus target bits 7.. contiguous from bit 7
        int cb = 7;                     // amplitude bits covered by one copy
        while ((8 << cb) < gran) {
            bool t = false;
            for (int x : tg) t |= x == cb;
            if (!t || cb == hi) break;
            ++cb;
        }
        if ((8 << cb) != gran) continue;
        std::vector<int> rest;          // targets not inside a copy, except the half bit (hi)
        for (int x : tg) if (x >= cb && x != hi) rest.push_back(x);
        p.cbytes = gran;
        p.ncopy = 1 << rest.size();
        if (p.ncopy * gran != 32 * 1024) continue;
        for (int h = 0; h < 2; ++h)
            for (int j = 0; j < p.ncopy; ++j) {
                uint64_t a = h ? (1ull << hi) : 0;
                for (size_t i = 0; i < rest.size(); ++i) if ((j >> i) & 1) a |= 1ull << rest[i];
                p.coff[h * p.ncopy + j] = a * 8;
            }
        struct V { const char *name; float (*f)(char *, const P &, int, int); };
        V vs[] = {{"NS4 NC4 NP2 .cs", run<4, 4, 2, 0>}, {"NS4 NC4 NP2 default", run<4, 4, 2, 1>},
                  {"NS4 NC8 NP2 default", run<4, 8, 2, 1>}, {"dynamic NS4 NC4", run_dyn<4, 4>},
                  {"dynamic NS4 NC8", run_dyn<4, 8>}, {"dynamic NS6 NC8", run_dyn<6, 8>}};
        for (auto &v : vs) {
            const float ms = v.f(psi, p, reps, sms);
            printf("{\"n\": %d, \"targets\": \"%s\", \"copy_bytes\": %d, \"variant\": \"%s\", \"ms\": %.3f, \"gbs\": %.1f}\n", n,
                   argc > 3 ? argv[3] : "8,9,10,20,21,22", gran, v.name, ms, 2.0 * bytes / ms / 1e6);
            fflush(stdout);
        }
    }
    return 0;
}
