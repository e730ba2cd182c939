// Tensor-core apply pass for complex64 k = 5, 6 (tcgen05, TMEM, sm_100a).
//
// Why tensor cores here: a k-qubit pass costs 8 * 2^k real flops per
// amplitude against 16 bytes of HBM traffic (AI = 2^(k-1) flop/B).  At k = 5, 6
// that is 16-32 flop/B, above the FP32 SIMT ridge (~11.5 flop/B at 1965 MHz),
// so the SIMT kernel cannot keep up with HBM; the per-tile complex matvec is a
// real dense contraction.
//
// Formulation (one tile = 64 gather sets of a 6-target gate; a 5-target gate is
// widened on the host to 6 targets as U (x) I on a spare non-target bit, which
// is exact):
//   D[m][n] = sum_kk A[m][kk] * B[kk][n]
//   A = real embedding of U, interleaved: A[2r+e][2c+f] = [[Ur,-Ui],[Ui,Ur]]_{ef}
//       (128 x 128 fp32, held in TMEM for the whole persistent CTA)
//   B = the tile: B[2c+f][n] = (re, im)_f of amplitude c of gather set n
//       (K-major in shared memory: each set's 128 reals are the natural
//        interleaved complex layout, no transpose)
//   D = the output tile, rows 2r+e = (re, im) of w_r, in TMEM.
// Precision: 3xTF32: A = Ahi + Alo (split on the host from
// fp64), B = Bhi + Blo (cvt.rna.tf32 in the kernel), D = Alo.Bhi + Ahi.Blo +
// Ahi.Bhi with FP32 accumulation in TMEM.  Plain 1xTF32 fails the 1e-4 bound.
//
// Warp roles (persistent, one CTA per SM, static round-robin tiles):
//   warps 0-3  epilogue: TMEM -> registers (tcgen05.ld) -> re/im pair shuffle
//              -> global stores (in place); also load A into TMEM at start.
//   warp  4    MMA issuer: one elected lane issues 48 tcgen05.mma per tile.
//   warps 5-12 converters: global loads of the tile (coalesced along sets),
//              split hi/lo, st.shared into the 3-stage B ring.
// Synchronisation: mbarriers full/empty (converters <-> MMA, smem ring) and
// tfull/tempty (MMA <-> epilogue, double-buffered TMEM accumulator).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <vector>

#include "hq_internal.h"

namespace hq {

namespace tc {

constexpr int N = 64;                    // gather sets per tile (MMA N)
constexpr int M = 128;                   // rows of A / D (2 * 64)
constexpr int KD = 128;                  // reduction length in reals
constexpr int STAGES = 3;
constexpr int HALF = N * KD * 4;         // bytes of the hi (or lo) part of a stage: 32 KB
constexpr int STAGE_BYTES = 2 * HALF;    // 64 KB
constexpr int NUM_EPI = 4;
constexpr int NUM_CONV = 8;
constexpr int MMA_WARP = NUM_EPI;
constexpr int CONV0 = NUM_EPI + 1;
constexpr int THREADS = (NUM_EPI + 1 + NUM_CONV) * 32;
constexpr int BAR_BYTES = 128;
constexpr int SMEM = STAGES * STAGE_BYTES + BAR_BYTES;
constexpr int TMEM_COLS = 512;
// TMEM columns: A_hi [0,128), A_lo [128,256); accumulator buffer d (0, 1):
// main [256+128d, 320+128d) = Ahi.Bhi, corr [320+128d, 384+128d) = Alo.Bhi + Ahi.Blo.
// Keeping the small correction terms in their own accumulator shortens the
// chain of FP32 accumulations on the main term (16 instead of 48 MMAs).

struct Params {
    uint64_t off[64];      // amplitude offset of canonical target pattern c
    uint32_t setoff[64];   // amplitude offset of set n inside a tile
    int pos[12];           // ascending bit positions of targets + set bits
    uint64_t ntiles;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // K-major, SWIZZLE_NONE canonical layout ((8,n),2):((1,SBO),LBO) in 16 B
    // units; version 1 (Blackwell) at bits [46,48).
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// One lane of the warp, chosen by elect.sync: the compiler then knows the
// issuing predicate is warp-uniform and emits UTCHMMA without a waterfall loop
// (measured: 32 vs 68 cycles per M128 N64 K8 tf32 MMA, tools/mma_bench.cu).
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\t@P1 mov.b32 %0, 1;\n\t}"
                 : "+r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

#define TC_REGS32(v)                                                                            \
    "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),        \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), \
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),           \
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),           \
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
#define TC_IN32(v)                                                                               \
    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),      \
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),       \
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),     \
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),     \
        "r"(v[29]), "r"(v[30]), "r"(v[31])
#define TC_LIST32                                                                                 \
    "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, " \
    "%20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}"

__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " TC_LIST32 ", [%32];"
                 : TC_REGS32(v)
                 : "r"(addr));
}

__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                 "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, "
                 "%18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(addr),
                 TC_IN32(v)
                 : "memory");
}

__device__ __forceinline__ uint64_t tile_base(uint64_t t, const Params &P) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        const int s = P.pos[i];
        t = ((t >> s) << (s + 1)) | (t & ((1ull << s) - 1));
    }
    return t;
}

__global__ void __launch_bounds__(THREADS, 1)
apply_tc6(float2 *__restrict__ psi, const __grid_constant__ Params P,
          const float *__restrict__ Areal /* [2][128][128]: hi then lo */) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + STAGES * STAGE_BYTES;
    // barrier layout: full[3], empty[3], tfull[2], tempty[2], tmem slot
    auto full_bar = [&](int s) { return bar0 + 8 * s; };
    auto empty_bar = [&](int s) { return bar0 + 8 * (STAGES + s); };
    auto tfull_bar = [&](int d) { return bar0 + 8 * (2 * STAGES + d); };
    auto tempty_bar = [&](int d) { return bar0 + 8 * (2 * STAGES + 2 + d); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4));

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), NUM_CONV);
            mbar_init(empty_bar(s), 1);
        }
        for (int d = 0; d < 2; ++d) {
            mbar_init(tfull_bar(d), 1);
            mbar_init(tempty_bar(d), NUM_EPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // A (hi, lo) into TMEM: warp q writes lanes 32q..32q+31 (row m of A).
    if (warp < NUM_EPI) {
        const int m = warp * 32 + lane;
#pragma unroll 1
        for (int ch = 0; ch < 8; ++ch) {
            uint32_t v[32];
            const float *src = Areal + (ch >> 2) * (M * KD) + m * KD + (ch & 3) * 32;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__ldg(src + i));
            tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + ch * 32, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const uint32_t A_HI = tmem, A_LO = tmem + 128;
    const uint64_t ntiles = P.ntiles;

    if (warp == MMA_WARP) {
        // idesc: F32 accumulate, A/B TF32, K-major, N = 64, M = 128
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(M >> 4) << 24);
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int s = it % STAGES;
            const uint32_t sp = (it / STAGES) & 1;
            const int d = it & 1;
            const uint32_t dp = (it >> 1) & 1;
            mbar_wait(tempty_bar(d), dp ^ 1);
            mbar_wait(full_bar(s), sp);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t Dm = tmem + 256 + 128 * d;
                const uint32_t Dc = Dm + 64;
                const uint32_t bhi = sbase + s * STAGE_BYTES;
                const uint64_t dhi = smem_desc(bhi, 1024, 128);
                const uint64_t dlo = smem_desc(bhi + HALF, 1024, 128);
                // K-chunk j covers reals 8j..8j+7 = two 16-byte core columns
                // (start address + 2048 B = +128 in the 16-byte address field);
                // LBO (next core column along K) = 1024 B, SBO (next 8 sets) = 128 B.
#pragma unroll
                for (int j = 0; j < KD / 8; ++j)
                    mma_ts(Dc, A_LO + 8 * j, dhi + 128 * j, idesc, j > 0);
#pragma unroll
                for (int j = 0; j < KD / 8; ++j)
                    mma_ts(Dc, A_HI + 8 * j, dlo + 128 * j, idesc, 1);
#pragma unroll
                for (int j = 0; j < KD / 8; ++j)
                    mma_ts(Dm, A_HI + 8 * j, dhi + 128 * j, idesc, j > 0);
                mma_commit(empty_bar(s));
                mma_commit(tfull_bar(d));
            }
            __syncwarp();
        }
    } else if (warp >= CONV0) {
        const int ct = (warp - CONV0) * 32 + lane;     // 0..255
        const int n = ct & 63;
        const int cp0 = ct >> 6;                       // 0..3
        const uint32_t soff = P.setoff[n];
        uint64_t offa[8], offb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            offa[i] = P.off[2 * (cp0 + 4 * i)] + soff;
            offb[i] = P.off[2 * (cp0 + 4 * i) + 1] + soff;
        }
        // software pipeline: the loads of tile it+1 are in flight while tile it
        // is converted and stored (two register buffers, 64 KB per SM in flight)
        float2 a0[8], b0[8], a1[8], b1[8];
        auto load = [&](uint64_t tt, float2 (&a)[8], float2 (&b)[8]) {
            const uint64_t base = tile_base(tt, P);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a[i] = psi[base + offa[i]];
                b[i] = psi[base + offb[i]];
            }
        };
        auto store = [&](uint32_t it, const float2 (&a)[8], const float2 (&b)[8]) {
            const int s = it % STAGES;
            const uint32_t sp = (it / STAGES) & 1;
            mbar_wait(empty_bar(s), sp ^ 1);
            uint8_t *hi = smem + s * STAGE_BYTES;
            uint8_t *lo = hi + HALF;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int cp = cp0 + 4 * i;
                const float2 x = a[i], y = b[i];
                uint4 h, l;
                h.x = to_tf32(x.x);
                h.y = to_tf32(x.y);
                h.z = to_tf32(y.x);
                h.w = to_tf32(y.y);
                l.x = __float_as_uint(x.x - __uint_as_float(h.x));
                l.y = __float_as_uint(x.y - __uint_as_float(h.y));
                l.z = __float_as_uint(y.x - __uint_as_float(h.z));
                l.w = __float_as_uint(y.y - __uint_as_float(h.w));
                *reinterpret_cast<uint4 *>(hi + cp * 1024 + n * 16) = h;
                *reinterpret_cast<uint4 *>(lo + cp * 1024 + n * 16) = l;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(full_bar(s));
        };
        const uint64_t G = gridDim.x;
        uint64_t t = blockIdx.x;
        uint32_t it = 0;
        if (t < ntiles) load(t, a0, b0);
        while (t < ntiles) {
            if (t + G < ntiles) load(t + G, a1, b1);
            store(it, a0, b0);
            t += G;
            ++it;
            if (t >= ntiles) break;
            if (t + G < ntiles) load(t + G, a0, b0);
            store(it, a1, b1);
            t += G;
            ++it;
        }
    } else {
        // epilogue warps 0..3: TMEM lanes 32q..32q+31 = rows m = 2r + e
        const int m = warp * 32 + lane;
        const int r = m >> 1, e = m & 1;
        const uint64_t offr = P.off[r];
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int d = it & 1;
            const uint32_t dp = (it >> 1) & 1;
            mbar_wait(tfull_bar(d), dp);
            tc_fence_after();
            uint32_t v0[32], v1[32], c0[32], c1[32];
            const uint32_t D = tmem + 256 + 128 * d + ((uint32_t)(warp * 32) << 16);
            tmem_ld32(D, v0);
            tmem_ld32(D + 32, v1);
            tmem_ld32(D + 64, c0);
            tmem_ld32(D + 96, c1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(d));
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v0[j] = __float_as_uint(__uint_as_float(v0[j]) + __uint_as_float(c0[j]));
                v1[j] = __float_as_uint(__uint_as_float(v1[j]) + __uint_as_float(c1[j]));
            }
            const uint64_t base = tile_base(t, P) + offr;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t x0 = j < 16 ? v0[2 * j] : v1[2 * j - 32];
                const uint32_t x1 = j < 16 ? v0[2 * j + 1] : v1[2 * j + 1 - 32];
                const uint32_t snd = e ? x0 : x1;
                const uint32_t rcv = __shfl_xor_sync(0xffffffffu, snd, 1);
                float2 o;
                o.x = __uint_as_float(e ? rcv : x0);
                o.y = __uint_as_float(e ? x1 : rcv);
                psi[base + P.setoff[2 * j + e]] = o;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

}  // namespace tc

// ------------------------------------------------------------------ host side

static inline float tf32_round_host(double x) {
    // round-to-nearest (ties away) to 10 explicit mantissa bits, as cvt.rna.tf32
    float f = (float)x;
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return f;
    u = (u + 0x1000u) & 0xffffe000u;
    memcpy(&f, &u, 4);
    return f;
}

bool tc_applicable(int dtype, const ApplyDesc &d) {
    return dtype == HQ_C64 && (d.k == 5 || d.k == 6) && d.n_local >= 16;
}

// Build the device payload (A hi/lo, 2 x 128 x 128 fp32) and kernel params
// from the canonical fp64 U (canonical order: U-index bit i <-> d.p[i]).
void tc_prepare(const ApplyDesc &d, const double *Ucanon, std::vector<char> &payload,
                std::vector<char> &params) {
    int p6[6];
    std::vector<double> U6;
    const int K = 6, D6 = 64;
    if (d.k == 6) {
        for (int i = 0; i < 6; ++i) p6[i] = d.p[i];
        U6.assign(Ucanon, Ucanon + 2 * D6 * D6);
    } else {
        // widen: U6 = U (x) I on the lowest non-target bit e
        int e = 0;
        for (;; ++e) {
            bool t = false;
            for (int i = 0; i < d.k; ++i) t |= d.p[i] == e;
            if (!t) break;
        }
        int j = 0;   // position of e in the sorted target list
        while (j < d.k && d.p[j] < e) ++j;
        for (int i = 0, s = 0; i < 6; ++i) p6[i] = i == j ? e : d.p[s++];
        const int D5 = 32;
        U6.assign(2 * D6 * D6, 0.0);
        auto drop = [&](int x) { return ((x >> (j + 1)) << j) | (x & ((1 << j) - 1)); };
        for (int r = 0; r < D6; ++r)
            for (int c = 0; c < D6; ++c) {
                if (((r >> j) & 1) != ((c >> j) & 1)) continue;
                const int r5 = drop(r), c5 = drop(c);
                U6[2 * (r * D6 + c)] = Ucanon[2 * (r5 * D5 + c5)];
                U6[2 * (r * D6 + c) + 1] = Ucanon[2 * (r5 * D5 + c5) + 1];
            }
    }
    // interleaved real embedding, split hi/lo
    payload.assign(2 * tc::M * tc::KD * sizeof(float), 0);
    float *hi = reinterpret_cast<float *>(payload.data());
    float *lo = hi + tc::M * tc::KD;
    for (int r = 0; r < D6; ++r)
        for (int c = 0; c < D6; ++c) {
            const double ur = U6[2 * (r * D6 + c)], ui = U6[2 * (r * D6 + c) + 1];
            const double blk[2][2] = {{ur, -ui}, {ui, ur}};
            for (int e = 0; e < 2; ++e)
                for (int f = 0; f < 2; ++f) {
                    const double x = blk[e][f];
                    const float h = tf32_round_host(x);
                    const float l = tf32_round_host(x - (double)h);
                    hi[(2 * r + e) * tc::KD + 2 * c + f] = h;
                    lo[(2 * r + e) * tc::KD + 2 * c + f] = l;
                }
        }
    // params
    params.assign(sizeof(tc::Params), 0);
    tc::Params &P = *reinterpret_cast<tc::Params *>(params.data());
    for (int c = 0; c < 64; ++c) {
        uint64_t o = 0;
        for (int i = 0; i < K; ++i)
            if ((c >> i) & 1) o |= 1ull << p6[i];
        P.off[c] = o;
    }
    int setbits[6], ns = 0;
    for (int b = 0; ns < 6; ++b) {
        bool t = false;
        for (int i = 0; i < 6; ++i) t |= p6[i] == b;
        if (!t) setbits[ns++] = b;
    }
    for (int n = 0; n < 64; ++n) {
        uint32_t o = 0;
        for (int i = 0; i < 6; ++i)
            if ((n >> i) & 1) o |= 1u << setbits[i];
        P.setoff[n] = o;
    }
    int all[12];
    for (int i = 0; i < 6; ++i) { all[i] = p6[i]; all[6 + i] = setbits[i]; }
    for (int i = 1; i < 12; ++i) {
        int x = all[i], k = i - 1;
        while (k >= 0 && all[k] > x) { all[k + 1] = all[k]; --k; }
        all[k + 1] = x;
    }
    for (int i = 0; i < 12; ++i) P.pos[i] = all[i];
    P.ntiles = 1ull << (d.n_local - 12);
}

int tc_launch(void *psi, const void *params, const void *dev_payload, void *stream) {
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(tc::apply_tc6, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const tc::Params &P = *reinterpret_cast<const tc::Params *>(params);
    uint64_t grid = P.ntiles < (uint64_t)sms ? P.ntiles : (uint64_t)sms;
    tc::apply_tc6<<<(unsigned)grid, tc::THREADS, tc::SMEM, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<float2 *>(psi), P, reinterpret_cast<const float *>(dev_payload));
    return (int)cudaGetLastError();
}

}  // namespace hq
