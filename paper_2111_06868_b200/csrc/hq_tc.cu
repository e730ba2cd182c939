// Tensor-core apply pass for complex64 k = 5, 6 (tcgen05, TMEM, sm_100a).
//
// Why tensor cores here: a k-qubit pass costs 8 * 2^k real flops per
// amplitude against 16 bytes of HBM traffic (AI = 2^(k-1) flop/B).  At k = 5, 6
// that is 16-32 flop/B, above the FP32 SIMT ridge (~11.5 flop/B at 1965 MHz),
// so the SIMT kernel cannot keep up with HBM; the per-tile complex matvec is a
// real dense contraction.
//
// Two orientations of the same contraction, both with FP16 operands
// (tcgen05.mma kind::f16, K = 16 per MMA), FP32 accumulation in TMEM and a
// 3-term split product D = Alo.Bhi + Ahi.Blo + Ahi.Bhi:
//   mode H (apply_tcb): lane = gather set.  A = the tile in TMEM (packed
//     f16x2, column c = amplitude c of the set), B = real embedding of U in
//     shared memory, B[2c+f][2r+e] = [[Ur,-Ui],[Ui,Ur]]_{ef}; each epilogue
//     thread owns a whole output gather set.  Used whenever the highest target
//     is at bit >= 7 and at most three targets sit in bits 0..3.
//   mode L (apply_tcL): lane = output real.  A = real embedding of U in TMEM,
//     B = the tile in shared memory (K-major SWIZZLE_128B, row = gather set).
//     Used for gathers concentrated in the lowest bits.
// Precision: each operand is carried as hi + lo with
// 11-bit significands (~22 bits together, FP32-class; a single-term TF32/FP16
// product fails the 1e-4 bound).  The FP16 range is handled by exact
// power-of-two scaling: U 2^ue (host, per gate) and psi 2^ea with ea chosen by
// the runtime from its rigorous bound on max |amplitude| (the tracked state
// norm), so that every scaled amplitude is <= 2^14 < 65504; amplitudes 2^-28
// below the bound and smaller lose relative precision gracefully (absolute
// error <= 2^-38 of the bound).
//
// Both kernels are persistent (one CTA per SM, static round-robin tiles) and
// warp-specialised: epilogue warps (TMEM -> registers -> global stores), one
// MMA-issuing warp (elect.sync), converter warps (shared memory -> FP16 hi/lo
// -> TMEM or swizzled shared memory) and TMA bulk-copy producer warps; mbarrier
// pairs hand every ring slot, A buffer and accumulator between the roles.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <type_traits>
#include <vector>

#include "hq_internal.h"

namespace hq {

namespace tc {

constexpr int M = 128;                   // gather sets per tile (MMA M = TMEM lanes)
constexpr int SETBITS = 7;
constexpr int NUM_EPI = 4;
constexpr int NUM_CONV = 8;
constexpr int MMA_WARP = NUM_EPI;
constexpr int CONV0 = NUM_EPI + 1;
constexpr int THREADS = (NUM_EPI + 1 + NUM_CONV) * 32;
constexpr int BAR_BYTES = 128;
// mode H: 8 converter warps (2 per TMEM lane quarter, each owning one K-half
// of its gather set)
constexpr int H_NUM_CONV = 8;

struct Params {
    uint64_t off[64];      // amplitude offset of canonical target pattern c
    uint32_t setoff[128];  // amplitude offset of set n inside a tile
    int pos[13];           // ascending bit positions of targets + set bits
    int k;
    int ue;                // B = U * 2^ue (host scaling into the fp16 range)
    int ea;                // A = psi * 2^ea (runtime: from the amplitude bound)
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

// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint expires) instead of spinning on the issue slots.
// In apply_tcb the converters wait ~40% of the time for bulk copies; spinning
// cost ~16% of all issued instructions (ncu source view) and power under the
// 1 kW cap.
#ifndef HQ_DEVICE_CHECKS
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(0x100000u)
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
#else
// Checked build (-DHQ_DEVICE_CHECKS, lib/libhq_check.so): every mbarrier wait
// carries a watchdog.  A phase that does not complete within ~2^33 cycles
// (several seconds) is a synchronisation bug (a missing arrive, a wrong
// parity, an expect-tx byte count that never lands): report and trap instead
// of hanging the GPU.  (compute-sanitizer is not available on the GPU pool.)
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __noinline__ void mbar_watchdog(uint32_t bar, uint32_t parity) {
    printf("hq device check: mbarrier wait timeout (block %d thread %d smem 0x%x parity %u)\n", blockIdx.x,
           threadIdx.x, bar, parity);
    __trap();
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    const long long t0 = clock64();
    while (!mbar_try(bar, parity))
        if (clock64() - t0 > (1ll << 33)) mbar_watchdog(bar, parity);
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) { mbar_wait(bar, parity); }
#endif

// Checked build: every global store / bulk-copy source of the tensor-core
// kernels must lie inside one of the buffers the pass may touch.
#ifdef HQ_DEVICE_CHECKS
__device__ __noinline__ void hq_range_fail(const void *p, uint32_t need, int where) {
    printf("hq device check %d: %u-byte access at %p outside the pass's buffers (block %d thread %d)\n", where, need,
           p, blockIdx.x, threadIdx.x);
    __trap();
}
__device__ __forceinline__ bool in_buf(const void *p, uint32_t need, uint64_t base, uint64_t bytes) {
    const uint64_t a = reinterpret_cast<uint64_t>(p);
    return base && a >= base && a + need <= base + bytes;
}
#define HQ_CHECK_IN(p, need, base, bytes, where) \
    do { if (!in_buf((p), (need), (uint64_t)(base), (bytes))) hq_range_fail((p), (need), (where)); } while (0)
#define HQ_CHECK_OUT(p, need, psi, om, bytes, where)                                                     \
    do {                                                                                                  \
        bool ok_ = false;                                                                                 \
        if (!(om).active) ok_ = in_buf((p), (need), (uint64_t)(psi), (bytes));                            \
        else for (int i_ = 0; i_ < 8; ++i_) ok_ |= in_buf((p), (need), (om).dst[i_], (bytes));            \
        if (!ok_) hq_range_fail((p), (need), (where));                                                    \
    } while (0)
#else
#define HQ_CHECK_IN(p, need, base, bytes, where) ((void)0)
#define HQ_CHECK_OUT(p, need, psi, om, bytes, where) ((void)0)
#endif

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

// D (+)= A B with A in TMEM (packed f16x2 per 32-bit column), B from a
// shared-memory descriptor; FP16 operands, FP32 accumulator (kind::f16; the
// instruction descriptor's A/B format fields are 0 = F16, bit 4 = F32 D).
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                        uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
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

__device__ __forceinline__ void tmem_st1(uint32_t addr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t addr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// 2^e as two float factors (each a normal power of two for |e| <= 252), so
// that x * f.x * f.y == x * 2^e exactly whenever the result is normal.  Kept
// branch-free and tiny: the converter applies it to every real of a tile.
__device__ __forceinline__ float2 pow2_factors(int e) {
    e = max(-252, min(252, e));
    const int a = e >> 1, b = e - (e >> 1);
    return make_float2(__int_as_float((127 + a) << 23), __int_as_float((127 + b) << 23));
}

// floor(log2(x)) + 1 for x > 0 (frexp exponent), including subnormals
__device__ __forceinline__ int frexp_exp(float x) {
    const uint32_t b = __float_as_uint(x);
    const int f = (int)((b >> 23) & 0xff);
    if (f != 0) return f - 126;
    return (int)((__float_as_uint(x * 18446744073709551616.0f) >> 23) & 0xff) - 126 - 64;
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(addr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
                 "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(addr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                 "r"(v[15])
                 : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                 "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, "
                 "%18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(addr),
                 TC_IN32(v)
                 : "memory");
}

template <int NPOS>
__device__ __forceinline__ uint64_t tile_base(uint64_t t, const Params &P) {
#pragma unroll
    for (int i = 0; i < NPOS; ++i) {
        const int s = P.pos[i];
        t = ((t >> s) << (s + 1)) | (t & ((1ull << s) - 1));
    }
    return t;
}

// Tile bases of a persistent CTA's tiles t, t + G, t + 2G, ...: the base is
// the tile index deposited into the non-tile bits, so stepping it by G is an
// addition in that masked space (carries ripple through the tile bits, which
// are forced to 1): base' = ((base | tilemask) + dep(G)) & ~tilemask.
struct TileWalk {
    uint64_t base, step, tmask;
    __device__ __forceinline__ void next() { base = ((base | tmask) + step) & ~tmask; }
};

template <int NPOS>
__device__ __forceinline__ TileWalk tile_walk(const Params &P) {
    uint64_t tm = 0;
#pragma unroll
    for (int i = 0; i < NPOS; ++i) tm |= 1ull << P.pos[i];
    return TileWalk{tile_base<NPOS>(blockIdx.x, P), tile_base<NPOS>(gridDim.x, P), tm};
}

// ------------------------------------------------------------------ mode H
// A tile (128 gather sets) spans 13 (K = 6) "tile bits": the targets and
// the 7 lowest non-target bits, so physical bits 0..6 are always tile bits and
// the tile is a union of 2^(K + 7 - 7) contiguous 1 KB blocks (128
// amplitudes, bits 0..6), whatever the placement.  One producer warp moves
// them with cp.async.bulk (the TMA engine's 1-D bulk copy, completion counted
// in bytes on an mbarrier) into an NS-deep ring of K-half slots; the K-half
// bit is the highest target, required to be >= 7 so a block never straddles
// halves.  Shared memory holds a slot in tile-index order (tile bits
// ascending, the half bit removed); converter thread (set n, pattern c) reads
// slot index nidx[n] | cidx[c].  No per-thread address arithmetic or LDGSTS,
// up to NS - 1 slots in flight while one is converted, and the A operand is
// double-buffered in TMEM so conversion of tile i+1 overlaps the MMAs of tile i.
//   warps 0-3 epilogue, 4 MMA, 5-12 converters, 13 producer.
// TMEM columns: A buffer a, half h: hi [a*KD + h*KD/2, + KD/4), lo the next
// KD/4; accumulator d: [2*KD + d*N, 2*KD + (d+1)*N).
constexpr int BK_PROD = NUM_EPI + 1 + H_NUM_CONV;
constexpr int bk_threads(int np) { return (BK_PROD + np) * 32; }   // np producer warps

template <int K, int NS> struct CfgB {
    static constexpr int D = 1 << K;
    static constexpr int KD = 2 * D;
    static constexpr int N = KD;
    static constexpr int HA = D / 2;
    static constexpr int B_BYTES = N * KD * 2;
    static constexpr int SLOT_BYTES = M * HA * 8;              // one K-half of a tile
    static constexpr int NBLK = SLOT_BYTES / 1024;             // 1 KB blocks per slot
    static constexpr int NSLOT = NS;
    static constexpr int RING = 2 * B_BYTES;
    static constexpr int BARS = RING + NSLOT * SLOT_BYTES;
    static constexpr int SMEM = BARS + 256;
    static constexpr int TMEM_COLS = 4 * KD;                   // 2 A buffers + 2 accumulators
    static constexpr int LBO = N * 16;
};

struct ParamsB {
    Params h;
    uint64_t off8[64];     // byte offset of canonical target pattern c (= 8 * off[c])
    uint64_t boff[2][32];  // amplitude offset (from the tile base) of block j of K-half h
    uint32_t cidx8[32];    // byte offset in a slot of pattern c (low K-1 bits of c)
    uint16_t nidx[128];    // slot index of gather set n (pattern 0)
    int diag;              // diagnostics (WRONG results; builds with -DHQ_TC_DIAG_BUILD only): 1 no MMA,
                           // 2 no conversion, 4 no stores
    int swz;               // 1: blocks arrive by 2-D TMA with SWIZZLE_128B; nidx/cidx8 are pre-swizzled
    int pair;              // 1: the lowest target is bit 0, patterns (2j, 2j+1) are one 16-byte load / store
    int xpair;             // 1: bit 0 is not a target and is lane bit 0: lane pairs swap one
                           //    output each so that every store is 16 bytes
};

// apply+pack output of mode H (a separate kernel argument of the PK
// instantiation only, so the in-place kernel's parameters stay as they were):
// byte offsets of the permuted pattern / set parts without the selector bits,
// and those bits
struct PackB {
    OutMap om;
    uint64_t poff8[64];
    uint64_t psoff8[128];
    uint8_t tpat[64];
    uint8_t tset[128];
};
struct NoPack {};
__device__ __forceinline__ const OutMap &pk_om(const PackB &x) { return x.om; }
__device__ __forceinline__ OutMap pk_om(const NoPack &) { return OutMap{}; }

// SWIZZLE_128B as seen from a slot index (8-byte amplitudes): byte address
// bits [4:6] ^= bits [7:9], i.e. index bits [1:3] ^= [4:6].  Linear over GF(2),
// so swz(nidx | cidx) = swz(nidx) ^ swz(cidx) for the disjoint set / pattern bits.
__host__ __device__ constexpr uint32_t swz128(uint32_t s) { return s ^ (((s >> 4) & 7u) << 1); }

__device__ __forceinline__ void tma_g2s_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void st_cs_f1(void *p, float v) {       // streaming store (evict-first)
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cs_f2(void *p, float2 v) {     // streaming store (evict-first)
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

__device__ __forceinline__ void st_cs_f4(void *p, float2 a, float2 b) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)
                 : "memory");
}
__device__ __forceinline__ void st_cs_f8(void *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ uint64_t f2_as_u64(float2 v) {
    return (uint64_t)__float_as_uint(v.x) | ((uint64_t)__float_as_uint(v.y) << 32);
}
__device__ __forceinline__ float2 u64_as_f2(uint64_t u) {
    return make_float2(__uint_as_float((uint32_t)u), __uint_as_float((uint32_t)(u >> 32)));
}
__device__ __forceinline__ uint64_t mul_f32x2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t sub_f32x2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// PK: apply+pack variant (out-of-place through P.om), instantiated separately
// so the in-place epilogue carries no output-map code.
template <int K, int NS, int NP, bool DIAG = false, bool PK = false>
__global__ void __launch_bounds__(bk_threads(NP), 1)
apply_tcb(float2 *__restrict__ psi, const __grid_constant__ ParamsB P,
          const __half *__restrict__ Breal /* [2][N][KD]: hi then lo, row n = output real */,
          const __grid_constant__ CUtensorMap tmap /* psi as [rows][16 amplitudes], box 8 rows, SWIZZLE_128B (P.swz) */,
          const __grid_constant__ std::conditional_t<PK, PackB, NoPack> X) {
    // even NS only: odd rings (a slot shared by both K-halves) failed with a
    // launch error at n >= 32 in the ring experiments; not pursued
    static_assert(NS % 2 == 0, "slot parity = K-half needs an even ring");
    using C = CfgB<K, NS>;
    constexpr int KD = C::KD, N = C::N, HA = C::HA, NSLOT = C::NSLOT;
    constexpr int NPOS = K + SETBITS;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + C::BARS;
    auto afull = [&](int a, int h) { return bar0 + 8 * (2 * a + h); };
    auto aempty = [&](int a, int h) { return bar0 + 8 * (4 + 2 * a + h); };
    auto tfull = [&](int d) { return bar0 + 8 * (8 + d); };
    auto tempty = [&](int d) { return bar0 + 8 * (10 + d); };
    auto rfull = [&](int s) { return bar0 + 8 * (12 + s); };
    auto rempty = [&](int s) { return bar0 + 8 * (12 + NSLOT + s); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::BARS + 8 * (12 + 2 * NSLOT));
    auto wait = [&](uint32_t bar, uint32_t parity) { mbar_wait_sleep(bar, parity); };

    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(bar0 + 8 * i, 4);              // afull: 4 converter warps
            mbar_init(bar0 + 8 * (4 + i), 1);        // aempty: MMA commit
        }
        for (int d = 0; d < 2; ++d) {
            mbar_init(tfull(d), 1);
            mbar_init(tempty(d), NUM_EPI);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(rfull(s), 1);                  // producer arrive.expect_tx + bytes
            mbar_init(rempty(s), 4);                 // 4 converter warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 2 * N * KD / 8; i += bk_threads(NP)) {
        const int part = i / (N * KD / 8);
        const int r = i % (N * KD / 8);
        const int n = r / (KD / 8), kq = r % (KD / 8);
        const uint4 v = *reinterpret_cast<const uint4 *>(Breal + part * N * KD + n * KD + 8 * kq);
        *reinterpret_cast<uint4 *>(smem + part * C::B_BYTES + kq * C::LBO + n * 16) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint64_t ntiles = P.h.ntiles;
    const uint64_t G = gridDim.x;

    if (warp >= BK_PROD) {
        // NP = 1: one warp fills slots in sidx order.  NP >= 2: producer warp
        // p fills the K-half h = p % 2 slots (sidx = 2 * it + h), blocks
        // [sub * NB, (sub + 1) * NB) of each slot, sub = p / 2; the sub = 0
        // warp posts the byte count (a copy may complete before it: the
        // mbarrier's tx-count may go transiently negative, and the phase
        // cannot complete while that arrival is pending).
        const int p = warp - BK_PROD;
        constexpr int NPH = NP == 1 ? 1 : NP / 2;
        constexpr int NB = C::NBLK / NPH;
        const int sub = NP == 1 ? 0 : p / 2;
        uint32_t it = 0;
        TileWalk tw = tile_walk<NPOS>(P.h);
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it, tw.next()) {
            const uint64_t tbo = tw.base;
            const float2 *tb = psi + tbo;
#pragma unroll 1
            for (int h = NP == 1 ? 0 : p % 2; h < (NP == 1 ? 2 : p % 2 + 1); ++h) {
                const uint32_t sidx = 2 * it + h;
                const int s = sidx % NSLOT;
                wait(rempty(s), ((sidx / NSLOT) & 1) ^ 1);
                if (sub == 0 && lane == 0) mbar_arrive_tx(rfull(s), C::SLOT_BYTES);
                __syncwarp();
                if (lane < NB) {
                    const int j = sub * NB + lane;
                    HQ_CHECK_IN(tb + P.boff[h][j], 1024, psi, P.h.ntiles << (K + SETBITS + 3), 1);
                    if (P.swz)   // row = 16 amplitudes; a 1 KB block is 8 rows, swizzled on arrival
                        tma_g2s_2d(sbase + C::RING + s * C::SLOT_BYTES + j * 1024, &tmap, 0,
                                   (int)((tbo + P.boff[h][j]) >> 4), rfull(s));
                    else
                        bulk_g2s(sbase + C::RING + s * C::SLOT_BYTES + j * 1024, tb + P.boff[h][j], 1024, rfull(s));
                }
            }
        }
    } else if (warp == MMA_WARP) {
        const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(M >> 4) << 24);
        const uint64_t dbhi = smem_desc(sbase, C::LBO, 128);
        const uint64_t dblo = smem_desc(sbase + C::B_BYTES, C::LBO, 128);
        constexpr int JH = KD / 32;
        constexpr uint32_t DSTEP = (2 * C::LBO) >> 4;
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it) {
            const int d = it & 1;                      // accumulator and A buffer
            const uint32_t ph = (it >> 1) & 1;
            const uint32_t Dt = tmem + 2 * KD + d * N;
            const uint32_t a0 = tmem + d * KD, a1 = a0 + KD / 2;
            mbar_wait(tempty(d), ph ^ 1);
            mbar_wait(afull(d, 0), ph);
            tc_fence_after();
            // Accumulation order matters for accuracy: the tensor core rounds
            // the FP32 accumulator coarsely at every MMA, so the error grows
            // with the number of MMAs that add into an accumulator of full
            // magnitude.  Issue all correction terms (Alo.Bhi, Ahi.Blo; ~2^-11
            // of the result) first, then the main terms Ahi.Bhi.
            const bool no_mma = DIAG && (P.diag & 1);   // diagnostics only: wrong results
            if (elect_one() && !no_mma) {
#pragma unroll 1
                for (int jj = 0; jj < JH; ++jj) {
                    const uint32_t jk = jj * DSTEP;
                    mma_f16(Dt, a0 + KD / 4 + 8 * jj, dbhi + jk, idesc, jj != 0);
                    mma_f16(Dt, a0 + 8 * jj, dblo + jk, idesc, 1);
                }
            }
            __syncwarp();
            mbar_wait(afull(d, 1), ph);
            tc_fence_after();
            if (elect_one()) {
                if (!no_mma) {
#pragma unroll 1
                    for (int jj = 0; jj < JH; ++jj) {
                        const uint32_t jk = (JH + jj) * DSTEP;
                        mma_f16(Dt, a1 + KD / 4 + 8 * jj, dbhi + jk, idesc, 1);
                        mma_f16(Dt, a1 + 8 * jj, dblo + jk, idesc, 1);
                    }
#pragma unroll 1
                    for (int jj = 0; jj < JH; ++jj)
                        mma_f16(Dt, a0 + 8 * jj, dbhi + jj * DSTEP, idesc, 1);
                }
                mma_commit(aempty(d, 0));
                if (!no_mma) {
#pragma unroll 1
                    for (int jj = 0; jj < JH; ++jj)
                        mma_f16(Dt, a1 + 8 * jj, dbhi + (JH + jj) * DSTEP, idesc, 1);
                }
                mma_commit(aempty(d, 1));
                mma_commit(tfull(d));
            }
            __syncwarp();
        }
    } else if (warp >= CONV0) {
        const int h = (warp - CONV0) >> 2;
        const int q = warp & 3;
        const int n = q * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const float sA = __int_as_float((127 + max(-126, min(127, P.h.ea))) << 23);
        const uint64_t sA2 = f2_as_u64(make_float2(sA, sA));
        const uint32_t nb8 = (uint32_t)P.nidx[n] * 8;
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it) {
            const int a = it & 1;
            const uint32_t sidx = 2 * it + h;
            const int s = sidx % NSLOT;
            // read the whole K-half of this set into registers and hand the
            // slot back before converting, so the producer can refill it
            // while this warp waits for the A buffer and converts
            wait(rfull(s), (sidx / NSLOT) & 1);
            const char *sraw = reinterpret_cast<const char *>(smem + C::RING + s * C::SLOT_BYTES);
            uint64_t v[HA];
            // nb8 ^ cidx8: with P.swz both are pre-swizzled; without, their bits are disjoint (^ == |)
            if (P.pair) {
#pragma unroll
                for (int c = 0; c < HA; c += 2) {
                    const uint4 w = *reinterpret_cast<const uint4 *>(sraw + (nb8 ^ P.cidx8[c]));
                    v[c] = (uint64_t)w.x | ((uint64_t)w.y << 32);
                    v[c + 1] = (uint64_t)w.z | ((uint64_t)w.w << 32);
                }
            } else {
#pragma unroll
                for (int c = 0; c < HA; ++c) v[c] = *reinterpret_cast<const uint64_t *>(sraw + (nb8 ^ P.cidx8[c]));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(rempty(s));
            wait(aempty(a, h), ((it >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t chi = tmem + a * KD + h * (KD / 2) + lane_addr, clo = chi + KD / 4;
            constexpr int CH = HA < 16 ? HA : 16;
#pragma unroll
            for (int c0 = 0; c0 < HA; c0 += CH) {
                uint32_t hi[CH], lo[CH];
#pragma unroll
                for (int i = 0; i < CH; ++i) {
                    if (DIAG && (P.diag & 2)) {         // diagnostics only: raw bits, no conversion
                        hi[i] = (uint32_t)v[c0 + i];
                        lo[i] = (uint32_t)(v[c0 + i] >> 32);
                        continue;
                    }
                    const uint64_t x = mul_f32x2(v[c0 + i], sA2);
                    const float2 xf = u64_as_f2(x);
                    const __half2 h2 = __floats2half2_rn(xf.x, xf.y);
                    const uint64_t r = sub_f32x2(x, f2_as_u64(__half22float2(h2)));
                    const float2 rf = u64_as_f2(r);
                    const __half2 l2 = __floats2half2_rn(rf.x, rf.y);
                    hi[i] = *reinterpret_cast<const uint32_t *>(&h2);
                    lo[i] = *reinterpret_cast<const uint32_t *>(&l2);
                }
                if constexpr (CH == 16) {
                    tmem_st16(chi + c0, hi);
                    tmem_st16(clo + c0, lo);
                } else {
                    tmem_st8(chi + c0, hi);
                    tmem_st8(clo + c0, lo);
                }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(afull(a, h));
        }
    } else {
        // epilogue: warp q reads TMEM lanes 32q.. = gather sets n
        const int n = warp * 32 + lane;
        const uint64_t soff8 = (uint64_t)P.h.setoff[n] * 8;
        const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
        const float2 sf = pow2_factors(-(max(-126, min(127, P.h.ea)) + P.h.ue));
        const uint64_t f1 = f2_as_u64(make_float2(sf.x, sf.x)), f2 = f2_as_u64(make_float2(sf.y, sf.y));
        uint32_t it = 0;
        TileWalk tw = tile_walk<NPOS>(P.h);
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it, tw.next()) {
            const int d = it & 1;
            wait(tfull(d), (it >> 1) & 1);
            tc_fence_after();
            char *pb = reinterpret_cast<char *>(psi + tw.base) + soff8;
            // apply+pack: the output index is om_swap(input index), split into a
            // buffer selector (tile | set | pattern parts) and an offset
            uint32_t tsel = 0;
            uint64_t obase = 0;
            if constexpr (PK) {
                const uint64_t y = om_swap(tw.base, X.om);
                tsel = ((uint32_t)(y >> X.om.tsh) & X.om.tmask) | X.tset[n];
                obase = ((y & ~((uint64_t)X.om.tmask << X.om.tsh)) | X.om.add) * 8 + X.psoff8[n];
            }
            auto saddr = [&](int c) -> char * {
                if constexpr (PK) return reinterpret_cast<char *>(X.om.dst[tsel | X.tpat[c]]) + obase + X.poff8[c];
                else return pb + P.off8[c];
            };
            const uint32_t Dt = tmem + 2 * KD + d * N + lane_addr;
#pragma unroll 2
            for (int ch = 0; ch < N / 32; ++ch) {
                uint32_t v[32];
                tmem_ld32(Dt + 32 * ch, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (ch == N / 32 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty(d));   // accumulator drained
                }
                if (P.pair) {
                    // bit 0 is a target: patterns 2j, 2j+1 of this set are adjacent
                    // amplitudes, one 16-byte store (full sectors per warp store)
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const uint64_t x0 = (uint64_t)v[2 * i] | ((uint64_t)v[2 * i + 1] << 32);
                        const uint64_t x1 = (uint64_t)v[2 * i + 2] | ((uint64_t)v[2 * i + 3] << 32);
                        const float2 o0 = u64_as_f2(mul_f32x2(mul_f32x2(x0, f1), f2));
                        const float2 o1 = u64_as_f2(mul_f32x2(mul_f32x2(x1, f1), f2));
                        if (DIAG && (P.diag & 4)) continue;
                        HQ_CHECK_OUT(saddr(16 * ch + i), 16, psi, pk_om(X), P.h.ntiles << (K + SETBITS + 3), 2);
                        st_cs_f4(saddr(16 * ch + i), o0, o1);
                    }
                    continue;
                }
                if (P.xpair) {
                    // bit 0 is a set bit and the lane parity: for the pattern pair
                    // (2j, 2j+1) the even lane (set s) stores (s, 2j), (s^1, 2j) and
                    // the odd lane (s, 2j+1), (s^1, 2j+1), adjacent amplitudes, one
                    // 16-byte store each after one 64-bit shuffle
                    const bool odd = lane & 1;
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const uint64_t x0 = (uint64_t)v[2 * i] | ((uint64_t)v[2 * i + 1] << 32);
                        const uint64_t x1 = (uint64_t)v[2 * i + 2] | ((uint64_t)v[2 * i + 3] << 32);
                        const uint64_t y0 = mul_f32x2(mul_f32x2(x0, f1), f2);
                        const uint64_t y1 = mul_f32x2(mul_f32x2(x1, f1), f2);
                        const uint64_t r = __shfl_xor_sync(0xffffffffu, odd ? y0 : y1, 1);
                        if (DIAG && (P.diag & 4)) continue;
                        HQ_CHECK_OUT(saddr(16 * ch + i + (odd ? 1 : 0)) - (odd ? 8 : 0), 16, psi, pk_om(X),
                                     P.h.ntiles << (K + SETBITS + 3), 3);
                        st_cs_f4(saddr(16 * ch + i + (odd ? 1 : 0)) - (odd ? 8 : 0), u64_as_f2(odd ? r : y0),
                                 u64_as_f2(odd ? y1 : r));
                    }
                    continue;
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint64_t x = (uint64_t)v[2 * i] | ((uint64_t)v[2 * i + 1] << 32);
                    const float2 o = u64_as_f2(mul_f32x2(mul_f32x2(x, f1), f2));
                    if (DIAG && (P.diag & 4)) continue; // diagnostics only: no stores
                    HQ_CHECK_OUT(saddr(16 * ch + i), 8, psi, pk_om(X), P.h.ntiles << (K + SETBITS + 3), 4);
                    st_cs_f2(saddr(16 * ch + i), o);
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
    }
}


// ------------------------------------------------------------------ mode L
// Orientation for gathers whose targets include the lowest physical bits
// (there a gather set is a short contiguous run, so "lanes = sets" loads and
// stores are strided).  The roles swap: A = real embedding of U in TMEM
// (lane = output real 2r+e), B = the tile in shared memory (K-major,
// SWIZZLE_128B, row = gather set, 64 sets per tile), D = output tile in TMEM
// (lane = output real, column = set).  Same arithmetic as mode H: FP16 hi/lo
// operands (kind::f16, K = 16 per MMA), A = U 2^ue from the host, B = psi 2^ea
// from the runtime's amplitude bound, 3-term product with the correction
// terms issued first, FP32 accumulation.
// Mode L's tile (6 targets + the 6 lowest non-target bits) always contains
// physical bits 0..6 (mode L is only chosen when some target is below bit 7),
// so the tile is 32 contiguous 1 KB blocks; a producer warp moves them with
// cp.async.bulk into an L_NR-slot raw ring in tile-index order, and the
// converter warps read it conflict-free, split, and write swizzled half2.
// k = 5 gates are widened to 6 targets on the host (U (x) I, exact): by the
// tcgen05 pacing law (B300_MICROARCH.md, floor = max(M,128) N / 256 cycles per
// MMA) a native M = 64 k = 5 pass costs the same tensor cycles per amplitude.
//   warps 0-7 epilogue (two per TMEM lane quarter, one per half of the 64
//   columns), 8 MMA, 9-16 converters, 17 producer.  The epilogue was the
//   bottleneck with four warps and re/im shuffles (ncu source view: the MMA
//   warp waited on the accumulator, the converters on the MMA): now each lane
//   stores its own real component, one 4-byte store per set.
// TMEM columns: A hi [0,64), A lo [64,128) (packed f16x2, column c = input
// amplitude c), accumulator d: [128 + 64 d, 192 + 64 d).

constexpr int L_NS = 64;                          // gather sets per tile (MMA N)
constexpr int L_STAGES = 2;
constexpr int L_ATOMCOL = (L_NS / 8) * 1024;      // bytes per 64-half (128 B) atom column
constexpr int L_HALF = 2 * L_ATOMCOL;             // 16 KB: hi (or lo) of one stage (K = 128 halves)
constexpr int L_STAGE = 2 * L_HALF;
constexpr int L_RAW = NUM_CONV * 32 * 16 * 8;     // one tile of raw amplitudes (32 KB)
constexpr int L_NR = 3;                           // raw ring slots
// warps 0-7 epilogue (warp w: TMEM lane quarter w % 4, columns [32 (w / 4), +32)),
// 8 MMA, 9-16 converters, 17 producer
constexpr int L_EPI = 8;
constexpr int L_MMA = L_EPI;
constexpr int L_CONV0 = L_EPI + 1;
constexpr int LB_PROD = L_CONV0 + NUM_CONV;
constexpr int LB_THREADS = (LB_PROD + 1) * 32;
constexpr int L_BARS = L_STAGES * L_STAGE + L_NR * L_RAW;
constexpr int LB_SMEM = L_BARS + BAR_BYTES;
constexpr int L_TMEM_COLS = 512;                  // K = 6: A 128 + D 2 x 64; K = 5: A 64 + D 2 x 128 (from 128)

struct ParamsL {
    uint64_t off[64];      // amplitude offset of canonical target pattern c
    uint32_t setoff[128];  // amplitude offset of set n inside a tile (64 sets at k = 6, 128 at k = 5)
    uint64_t boff[32];     // amplitude offset of 1 KB block j of a tile (tile bits >= 7 of j << 7)
    int pos[12];           // ascending bit positions of the tile (targets + set bits)
    int nbit[12];          // tile bit i -> set-index bit (or -1)
    int cbit[12];          // tile bit i -> canonical target bit (or -1)
    int ue;                // A = U * 2^ue (host scaling into the fp16 range)
    int ea;                // B = psi * 2^ea (runtime: from the amplitude bound)
    int k;                 // 6, or 5 (native M = 64 kernel)
    uint64_t ntiles;
};

// apply+pack output of mode L (PK instantiation only): amplitude offsets of
// the permuted pattern / set parts without the selector bits, and those bits
struct PackL {
    OutMap om;
    uint64_t poff[64];
    uint64_t psetoff[128];
    uint8_t tpat[64];
    uint8_t tset[128];
};

// tcgen05.ld .16x32bx2: a warp reads 16 TMEM lanes (the M = 64 accumulator
// layout uses lanes 0-15 of each 32-lane quarter); threads 0-15 get columns
// [c, c + 32) of lanes 0..15, threads 16-31 columns [c + 32, c + 64)
__device__ __forceinline__ void tmem_ld16x2_32(uint32_t addr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x32.b32 " TC_LIST32 ", [%32], 32;"
                 : TC_REGS32(v)
                 : "r"(addr));
}

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
    // K-major SWIZZLE_128B: rows of 128 B, 8-row atoms (SBO = 1024 B), LBO unused (1)
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__device__ __forceinline__ uint64_t tile_base12(uint64_t t, const ParamsL &P) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
        const int s = P.pos[i];
        t = ((t >> s) << (s + 1)) | (t & ((1ull << s) - 1));
    }
    return t;
}


// K = 6: M = 128 output reals, N = 64 sets.  K = 5 (native, no U (x) I
// widening): M = 64 output reals, N = 128 sets, K = 64 input reals -- half
// the tensor MACs per amplitude, which under the 1 kW cap is what sets the
// clock.  The M = 64 A operand and accumulator occupy TMEM lanes 0-15 of
// each 32-lane quarter (row m -> lane m % 16 + 32 (m / 16)).
template <int K, bool PK>      // PK: apply+pack variant (see apply_tcb)
__global__ void __launch_bounds__(LB_THREADS, 1)
apply_tcL(float2 *__restrict__ psi, const __grid_constant__ ParamsL P,
          const uint32_t *__restrict__ Apack /* [2][128][64] half2: hi then lo, row = output real */,
          const __grid_constant__ std::conditional_t<PK, PackL, NoPack> X) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + L_BARS;
    auto full_bar = [&](int s) { return bar0 + 8 * s; };
    auto empty_bar = [&](int s) { return bar0 + 8 * (L_STAGES + s); };
    auto tfull_bar = [&](int d) { return bar0 + 8 * (2 * L_STAGES + d); };
    auto tempty_bar = [&](int d) { return bar0 + 8 * (2 * L_STAGES + 2 + d); };
    auto rfull = [&](int r) { return bar0 + 8 * (2 * L_STAGES + 4 + r); };
    auto rempty = [&](int r) { return bar0 + 8 * (2 * L_STAGES + 4 + L_NR + r); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + L_BARS + 8 * (2 * L_STAGES + 4 + 2 * L_NR));
    const uint32_t raw0 = sbase + L_STAGES * L_STAGE;
    auto wait = [&](uint32_t bar, uint32_t parity) { mbar_wait_sleep(bar, parity); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < L_STAGES; ++s) {
            mbar_init(full_bar(s), NUM_CONV);
            mbar_init(empty_bar(s), 1);
        }
        for (int d = 0; d < 2; ++d) {
            mbar_init(tfull_bar(d), 1);
            mbar_init(tempty_bar(d), L_EPI);
        }
        for (int r = 0; r < L_NR; ++r) {
            mbar_init(rfull(r), 1);
            mbar_init(rempty(r), NUM_CONV);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == L_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(L_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // A (U hi, lo as packed half2) into TMEM: warp q writes lanes 32q..32q+31
    constexpr int ACOLS = K == 6 ? 64 : 32;           // 32-bit columns per term (K reals / 2)
    if (warp < 4) {
        // K = 6: lane 32q + l holds row 32q + l; K = 5: lanes 32q + l, l < 16,
        // hold rows 16q + l (M = 64 layout), the other lanes zeros
        const int m = K == 6 ? warp * 32 + lane : (lane < 16 ? warp * 16 + lane : -1);
#pragma unroll 1
        for (int ch = 0; ch < 2 * ACOLS / 32; ++ch) {
            uint32_t v[32];
            const int term = ch / (ACOLS / 32), cc = ch % (ACOLS / 32);
            const uint32_t *src = Apack + term * (128 * 64) + (m < 0 ? 0 : m) * 64 + cc * 32;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = m < 0 ? 0u : __ldg(src + i);
            tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + ch * 32, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t A_HI = tmem, A_LO = tmem + ACOLS;
    constexpr int NSET = K == 6 ? 64 : 128;           // MMA N (sets per tile)
    constexpr uint32_t D0 = 128;                      // accumulator d at columns [D0 + NSET d, + NSET)
    const uint64_t ntiles = P.ntiles;
    const uint64_t G = gridDim.x;
    uint64_t tmask = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i) tmask |= 1ull << P.pos[i];
    TileWalk tw{tile_base12(blockIdx.x, P), tile_base12(G, P), tmask};

    if (warp == LB_PROD) {
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it, tw.next()) {
            const int r = it % L_NR;
            wait(rempty(r), ((it / L_NR) & 1) ^ 1);
            if (lane == 0) mbar_arrive_tx(rfull(r), L_RAW);
            __syncwarp();
            HQ_CHECK_IN(psi + tw.base + P.boff[lane], 1024, psi, P.ntiles << 15, 5);
            bulk_g2s(raw0 + r * L_RAW + lane * 1024, psi + tw.base + P.boff[lane], 1024, rfull(r));
        }
    } else if (warp == L_MMA) {
        // idesc: F32 accumulate, A/B F16, both K-major; K = 6: M = 128 output
        // reals, N = 64 sets; K = 5: M = 64, N = 128
        constexpr uint32_t MM = K == 6 ? 128 : 64;
        const uint32_t idesc = (1u << 4) | ((uint32_t)(NSET >> 3) << 17) | ((MM >> 4) << 24);
        constexpr int NJ = K == 6 ? 8 : 4;            // K-chunks of 16 halves
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it) {
            const int s = it % L_STAGES;
            const uint32_t sp = (it / L_STAGES) & 1;
            const int d = it & 1;
            const uint32_t dp = (it >> 1) & 1;
            mbar_wait(tempty_bar(d), dp ^ 1);
            mbar_wait(full_bar(s), sp);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t D = tmem + D0 + NSET * d;
                const uint32_t bhi = sbase + s * L_STAGE, blo = bhi + L_HALF;
                // K-chunk j (16 halves = 32 B): atom column j/4, +32 B inside the 128-B row;
                // correction terms first, main terms last (accuracy, see apply_tcb)
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const uint32_t o = (j >> 2) * L_ATOMCOL + (j & 3) * 32;
                    mma_f16(D, A_LO + 8 * j, smem_desc_sw128(bhi + o), idesc, j > 0);
                    mma_f16(D, A_HI + 8 * j, smem_desc_sw128(blo + o), idesc, 1);
                }
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const uint32_t o = (j >> 2) * L_ATOMCOL + (j & 3) * 32;
                    mma_f16(D, A_HI + 8 * j, smem_desc_sw128(bhi + o), idesc, 1);
                }
                mma_commit(empty_bar(s));
                mma_commit(tfull_bar(d));
            }
            __syncwarp();
        }
    } else if (warp >= L_CONV0) {
        // thread -> tile-local amplitude index tl = lane | (cw << 5) | (i << 8), i = 0..15
        const int cw = warp - L_CONV0;
        uint32_t n_base = 0, c_base = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int bit = b < 5 ? (lane >> b) & 1 : (cw >> (b - 5)) & 1;
            if (bit) {
                if (P.nbit[b] >= 0) n_base |= 1u << P.nbit[b];
                if (P.cbit[b] >= 0) c_base |= 1u << P.cbit[b];
            }
        }
        // byte offset of (set n, amplitude c) in a K-major SWIZZLE_128B half2
        // stage: atom column c / 32, row n, 16-byte chunk (c / 4) % 8 ^ n % 8
        uint32_t sdst[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint32_t n = n_base, c = c_base;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((i >> b) & 1) {
                    if (P.nbit[8 + b] >= 0) n |= 1u << P.nbit[8 + b];
                    if (P.cbit[8 + b] >= 0) c |= 1u << P.cbit[8 + b];
                }
            const uint32_t r8 = n & 7, ch = (c >> 2) & 7;
            // atom column c / 32 spans the NSET rows (K = 5 has one atom column)
            sdst[i] = (c >> 5) * (NSET / 8) * 1024 + (n >> 3) * 1024 + r8 * 128 + ((ch ^ r8) << 4) + (c & 3) * 4;
        }
        const float sA = __int_as_float((127 + max(-126, min(127, P.ea))) << 23);
        const uint64_t sA2 = f2_as_u64(make_float2(sA, sA));
        const int ct = cw * 32 + lane;
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it) {
            const int r = it % L_NR;
            wait(rfull(r), (it / L_NR) & 1);
            const uint64_t *raw = reinterpret_cast<const uint64_t *>(smem + L_STAGES * L_STAGE + r * L_RAW) + ct;
            uint64_t v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = raw[i * 256];
            __syncwarp();
            if (lane == 0) mbar_arrive(rempty(r));
            const int s = it % L_STAGES;
            const uint32_t sp = (it / L_STAGES) & 1;
            wait(empty_bar(s), sp ^ 1);
            uint8_t *hi = smem + s * L_STAGE;
            uint8_t *lo = hi + L_HALF;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint64_t x = mul_f32x2(v[i], sA2);
                const float2 xf = u64_as_f2(x);
                const __half2 h2 = __floats2half2_rn(xf.x, xf.y);
                const float2 rf = u64_as_f2(sub_f32x2(x, f2_as_u64(__half22float2(h2))));
                const __half2 l2 = __floats2half2_rn(rf.x, rf.y);
                *reinterpret_cast<__half2 *>(hi + sdst[i]) = h2;
                *reinterpret_cast<__half2 *>(lo + sdst[i]) = l2;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(full_bar(s));
        }
    } else {
        // epilogue warp w (0..7), TMEM lane quarter q = w % 4, column half
        // hc = w / 4.  K = 6: lane l holds output real m = 32q + l (m = 2r + e)
        // for the 32 sets [32 hc, +32).  K = 5: a .16x32bx2 load gives lanes
        // l < 16 of the quarter (rows m = 16q + l % 16) to both thread halves,
        // sets [64 hc + 32 (l / 16), +32).  Each lane stores its own real
        // component, one 4-byte store per set (a full line per warp store when
        // the lowest targets are the lowest bits), no re/im shuffles.
        const int q = warp & 3, hc = warp >> 2;
        const int m = K == 6 ? q * 32 + lane : q * 16 + (lane & 15);
        const int r = m >> 1, e = m & 1;
        const int nbase = K == 6 ? 32 * hc : 64 * hc + 32 * (lane >> 4);
        const uint64_t rb = 2 * P.off[r] + e;                  // float offset of (r, e) in a set
        // set offsets are GF(2)-linear in the set index (disjoint bits), so
        // setoff[nbase + j] = setoff[nbase] + setoff[j], j a compile-time index
        const uint64_t rbh = rb + 2 * (uint64_t)P.setoff[nbase];
        uint64_t sb[5];
#pragma unroll
        for (int b = 0; b < 5; ++b) sb[b] = 2 * (uint64_t)P.setoff[1 << b];
        // 2^-(ea + ue) as one factor when it is a normal float, else two
        const int se = -(max(-126, min(127, P.ea)) + P.ue);
        const float2 sf = pow2_factors(se);
        const bool one = se >= -126 && se <= 127;
        const float s1 = one ? __int_as_float((127 + se) << 23) : 1.0f;
        float *const psif = reinterpret_cast<float *>(psi);
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < ntiles; t += G, ++it, tw.next()) {
            const int d = it & 1;
            const uint32_t dp = (it >> 1) & 1;
            wait(tfull_bar(d), dp);
            tc_fence_after();
            uint32_t v[32];
            if constexpr (K == 6)
                tmem_ld32(tmem + D0 + NSET * d + 32 * hc + ((uint32_t)(q * 32) << 16), v);
            else
                tmem_ld16x2_32(tmem + D0 + NSET * d + 64 * hc + ((uint32_t)(q * 32) << 16), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(d));
            if (one) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * s1);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * sf.x * sf.y);
            }
            if constexpr (!PK) {
                float *pb = psif + 2 * tw.base + rbh;
                // set j's offset from the five single-bit offsets (linearity):
                // five tile-invariant values instead of 32 held in registers
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    uint64_t o = 0;
#pragma unroll
                    for (int b = 0; b < 5; ++b)
                        if ((j >> b) & 1) o += sb[b];
                    HQ_CHECK_IN(pb + o, 4, psi, P.ntiles << 15, 6);
                    st_cs_f1(pb + o, __uint_as_float(v[j]));
                }
            } else {                  // apply+pack (see apply_tcb)
                const uint64_t y = om_swap(tw.base, X.om);
                const uint32_t tsel = ((uint32_t)(y >> X.om.tsh) & X.om.tmask) | X.tpat[r];
                const uint64_t ob = ((y & ~((uint64_t)X.om.tmask << X.om.tsh)) | X.om.add) + X.poff[r];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int sn = nbase + j;
                    float *dst = reinterpret_cast<float *>(X.om.dst[tsel | X.tset[sn]]);
                    HQ_CHECK_OUT(dst + 2 * (ob + X.psetoff[sn]) + e, 4, psi, X.om, P.ntiles << 15, 7);
                    dst[2 * (ob + X.psetoff[sn]) + e] = __uint_as_float(v[j]);
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == L_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L_TMEM_COLS));
    }
}

}  // namespace tc

// ------------------------------------------------------------------ host side

// complex64 k = 5, 6 run on the tensor cores, and k = 4 too, widened to a
// k = 5 gate (U (x) I on one more bit, exact): measured under the 1 kW cap the
// SIMT k = 4 pass is power-bound at 0.78-0.91 of the HBM peak (64 FMA per
// amplitude on the FP32 pipe), a k = 5 tensor-core pass runs at 0.81-0.95.
bool tc_applicable(int dtype, const ApplyDesc &d) {
    const int kk = d.k == 4 ? 5 : d.k;              // the widened k = 4 runs as k = 5
    return dtype == HQ_C64 && d.k >= 4 && d.k <= 6 && d.n_local >= kk + tc::SETBITS + 3;
}

// U (x) I: a k-qubit canonical gate as a (k+1)-qubit one with the extra
// physical bit e (not a target) as an identity factor; exact.
static void widen_gate(const ApplyDesc &d, const double *U, int e, ApplyDesc &w, std::vector<double> &Uw) {
    const int k = d.k, D = 1 << k, k1 = k + 1, D1 = 1 << k1;
    int j = 0;
    while (j < k && d.p[j] < e) ++j;                // canonical position of e
    w = d;
    w.k = k1;
    for (int i = 0, s = 0; i < k1; ++i) w.p[i] = i == j ? e : d.p[s++];
    Uw.assign((size_t)2 * D1 * D1, 0.0);
    auto drop = [&](int x) { return ((x >> (j + 1)) << j) | (x & ((1 << j) - 1)); };
    for (int r = 0; r < D1; ++r)
        for (int c = 0; c < D1; ++c) {
            if (((r >> j) & 1) != ((c >> j) & 1)) continue;
            Uw[2 * (r * D1 + c)] = U[2 * (drop(r) * D + drop(c))];
            Uw[2 * (r * D1 + c) + 1] = U[2 * (drop(r) * D + drop(c)) + 1];
        }
}

// Mode L (U in TMEM, tile in shared memory) when the targets crowd the lowest
// bits, where mode H's lanes-are-sets layout gives strided accesses, and
// whenever every target is below bit 7 (mode H's bulk-copy blocks need the
// K-half bit above bits 0..6).  Measured on a B200 (bench_sweep.py, n = 32
// dense state, same box, round 1): mode H wins with bits 0 and 1 as the only
// low targets and with three low targets that leave bit 0 or bit 1 free;
// mode L wins with four or more targets in bits 0..3 and with bits 0, 1 and a
// third low bit.
static bool tc_use_mode_l(const ApplyDesc &d) {
    int low = 0;
    bool b0 = false, b1 = false;
    for (int i = 0; i < d.k; ++i) {
        low += d.p[i] < 4;
        b0 |= d.p[i] == 0;
        b1 |= d.p[i] == 1;
    }
    return low >= 4 || (b0 && b1 && low >= 3) || d.p[d.k - 1] < 7;
}

// U 2^ue with max |U| 2^ue in [2^14, 2^15): the FP16 range of the U operand
static int u_scale_exp(const double *U, int k) {
    const int D = 1 << k;
    double umax = 0.0;
    for (int i = 0; i < 2 * D * D; ++i) umax = std::max(umax, std::fabs(U[i]));
    int ex = 0;
    if (umax > 0) std::frexp(umax, &ex);
    return umax > 0 ? 15 - ex : 0;
}

// fp64 x -> FP16 hi + lo (hi = RN(x), lo = RN(x - hi))
static void split_f16(double x, __half &hi, __half &lo) {
    hi = __double2half(x);
    lo = __double2half(x - (double)__half2float(hi));
}

static void tc_prepare_l(const ApplyDesc &d, const double *Ucanon, std::vector<char> &payload,
                         std::vector<char> &params) {
    // k = 6, or k = 5 on the native M = 64 kernel (no widening)
    const int K = d.k, D = 1 << K, NSET = K == 6 ? 64 : 128, NSB = 12 - K;
    const int ue = u_scale_exp(Ucanon, K);
    // A = interleaved real embedding (row = output real 2r+e, column kk = input
    // real 2c+f) times 2^ue, FP16 hi and lo, packed two halves (f = 0, 1) per
    // 32-bit word: [2][128 rows][64 words] (k = 5: rows < 64, words < 32)
    payload.assign(2 * 128 * 64 * sizeof(uint32_t), 0);
    __half *hi = reinterpret_cast<__half *>(payload.data());
    __half *lo = hi + 128 * 128;
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            const double ur = Ucanon[2 * (r * D + c)], ui = Ucanon[2 * (r * D + c) + 1];
            const double blk[2][2] = {{ur, -ui}, {ui, ur}};
            for (int e = 0; e < 2; ++e)
                for (int f = 0; f < 2; ++f) {
                    const int idx = (2 * r + e) * 128 + 2 * c + f;
                    split_f16(std::ldexp(blk[e][f], ue), hi[idx], lo[idx]);
                }
        }
    params.assign(sizeof(tc::ParamsL) + 1, 0);
    params.back() = 'L';
    tc::ParamsL &P = *reinterpret_cast<tc::ParamsL *>(params.data());
    P.k = K;
    P.ue = ue;
    P.ea = 14;             // set per launch by the runtime (tc_set_amp_bound)
    for (int c = 0; c < D; ++c) {
        uint64_t o = 0;
        for (int i = 0; i < K; ++i)
            if ((c >> i) & 1) o |= 1ull << d.p[i];
        P.off[c] = o;
    }
    int setbits[7], ns = 0;
    for (int b = 0; ns < NSB; ++b) {
        bool t = false;
        for (int i = 0; i < K; ++i) t |= d.p[i] == b;
        if (!t) setbits[ns++] = b;
    }
    for (int n = 0; n < NSET; ++n) {
        uint32_t o = 0;
        for (int i = 0; i < NSB; ++i)
            if ((n >> i) & 1) o |= 1u << setbits[i];
        P.setoff[n] = o;
    }
    int all[12];
    for (int i = 0; i < K; ++i) all[i] = d.p[i];
    for (int i = 0; i < NSB; ++i) all[K + i] = setbits[i];
    std::sort(all, all + 12);
    for (int i = 0; i < 12; ++i) {
        P.pos[i] = all[i];
        P.nbit[i] = P.cbit[i] = -1;
        for (int j = 0; j < NSB; ++j)
            if (setbits[j] == all[i]) P.nbit[i] = j;
        for (int j = 0; j < K; ++j)
            if (d.p[j] == all[i]) P.cbit[i] = j;
    }
    // physical bits 0..6 are tile bits 0..6 (some target is below bit 7 in
    // mode L), so a tile is 32 contiguous 1 KB blocks
    for (int j = 0; j < 32; ++j) {
        uint64_t o = 0;
        for (int b = 7; b < 12; ++b)
            if (((uint64_t)j << 7 >> b) & 1) o |= 1ull << P.pos[b];
        P.boff[j] = o;
    }
    P.ntiles = 1ull << (d.n_local - 12);
}

// Build the device payload (B = real embedding of U times 2^ue, FP16 hi and
// lo, [N][KD] each, row n = output real) and the kernel parameter block from
// the canonical fp64 U (canonical order: U-index bit i <-> d.p[i]).
void tc_prepare(const ApplyDesc &d0, const double *Ucanon0, std::vector<char> &payload,
                std::vector<char> &params) {
    ApplyDesc d = d0;
    const double *Ucanon = Ucanon0;
    std::vector<double> Uw;
    if (d0.k == 4) {
        // widen with the lowest non-target bit >= 4 (adds no low target, so
        // the mode rule sees the same low bits)
        int e = 4;
        for (;; ++e) {
            bool t = false;
            for (int i = 0; i < 4; ++i) t |= d0.p[i] == e;
            if (!t) break;
        }
        widen_gate(d0, Ucanon0, e, d, Uw);
        Ucanon = Uw.data();
    }
    if (tc_use_mode_l(d)) {
        tc_prepare_l(d, Ucanon, payload, params);
        return;
    }
    const int K = d.k, D = 1 << K, KD = 2 * D, N = KD;
    const int ue = u_scale_exp(Ucanon, K);
    payload.assign((size_t)2 * N * KD * sizeof(__half), 0);
    __half *hi = reinterpret_cast<__half *>(payload.data());
    __half *lo = hi + N * KD;
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            const double ur = Ucanon[2 * (r * D + c)], ui = Ucanon[2 * (r * D + c) + 1];
            // output real 2r+e, input real 2c+f: [[ur, -ui], [ui, ur]]_{ef}
            const double blk[2][2] = {{ur, -ui}, {ui, ur}};
            for (int e = 0; e < 2; ++e)
                for (int f = 0; f < 2; ++f) {
                    const int idx = (2 * r + e) * KD + 2 * c + f;
                    split_f16(std::ldexp(blk[e][f], ue), hi[idx], lo[idx]);
                }
        }
    params.assign(sizeof(tc::ParamsB) + 1, 0);
    params.back() = 'B';
    tc::ParamsB &B = *reinterpret_cast<tc::ParamsB *>(params.data());
    tc::Params &P = B.h;
    P.k = K;
    P.ue = ue;
    P.ea = 14;             // set per launch by the runtime (tc_set_amp_bound)
    for (int c = 0; c < D; ++c) {
        uint64_t o = 0;
        for (int i = 0; i < K; ++i)
            if ((c >> i) & 1) o |= 1ull << d.p[i];
        P.off[c] = o;
    }
    int setbits[tc::SETBITS], ns = 0;
    for (int b = 0; ns < tc::SETBITS; ++b) {
        bool t = false;
        for (int i = 0; i < K; ++i) t |= d.p[i] == b;
        if (!t) setbits[ns++] = b;
    }
    for (int n = 0; n < tc::M; ++n) {
        uint32_t o = 0;
        for (int i = 0; i < tc::SETBITS; ++i)
            if ((n >> i) & 1) o |= 1u << setbits[i];
        P.setoff[n] = o;
    }
    int all[13], na = 0;
    for (int i = 0; i < K; ++i) all[na++] = d.p[i];
    for (int i = 0; i < tc::SETBITS; ++i) all[na++] = setbits[i];
    std::sort(all, all + na);
    for (int i = 0; i < na; ++i) P.pos[i] = all[i];
    P.ntiles = 1ull << (d.n_local - K - tc::SETBITS);
    // the highest target is at bit >= 7 (tc_use_mode_l): the K-half bit lies
    // above the 1 KB blocks of bits 0..6
    for (int c = 0; c < D; ++c) B.off8[c] = P.off[c] * 8;
    auto tpos = [&](int phys) { return (int)(std::find(all, all + na, phys) - all); };
    const int hp = tpos(d.p[K - 1]);
    auto slot_of = [&](uint64_t ti) { return (ti & ((1ull << hp) - 1)) | ((ti >> (hp + 1)) << hp); };
    // Targets in bits 0..3 (measured on the 34q circuit, tools/pass_times.py,
    // same box):
    //  * bit 0 a target: patterns (2j, 2j+1) are adjacent, so converters
    //    load and the epilogue stores 16 bytes (pair): 61 -> 47 ms per pass;
    //  * bit 1 the lowest target (k = 6): 2-D TMA with SWIZZLE_128B removes the
    //    2-way bank conflicts of the converter loads (61 -> 58 ms).  The
    //    swizzled copies are slower elsewhere (no low target 57 -> 60 ms, a
    //    k = 5 pass with targets 3, 4, 6 56 -> 80 ms), so only this case uses them.
    B.swz = K == 6 && d.p[0] == 1;
    B.pair = d.p[0] == 0;
    B.xpair = 0;
    // Converter lanes (n bits 0..4) are 5 of the 7 set bits.  With one
    // target in bits 0..3 the ascending choice puts a warp's 8-byte reads
    // on 8 of 16 bank pairs (2-way conflicts); with the swizzled slot
    // another choice of lane bits, or 16-byte pattern pairs when bit 0 is
    // a target, reaches all of them.  Pick the conflict-minimal choice,
    // the ascending one on ties (it keeps the epilogue stores contiguous).
    int order[tc::SETBITS];
    for (int i = 0; i < tc::SETBITS; ++i) order[i] = setbits[i];
    if (B.swz) {
        auto slot_idx = [&](int n, const int *sb) {
            uint64_t ti = 0;
            for (int i = 0; i < tc::SETBITS; ++i)
                if ((n >> i) & 1) ti |= 1ull << tpos(sb[i]);
            return tc::swz128((uint32_t)slot_of(ti));
        };
        auto wavefronts = [&](const int *sb) {
            const int words = B.pair ? 4 : 2;
            int cnt[32] = {0};
            uint32_t seen[32][32];
            for (int l = 0; l < 32; ++l) {
                const uint32_t w0 = slot_idx(l, sb) * 2;
                for (int w = 0; w < words; ++w) {
                    const uint32_t word = w0 + w, bank = word & 31;
                    bool dup = false;
                    for (int i = 0; i < cnt[bank]; ++i) dup |= seen[bank][i] == word;
                    if (!dup) seen[bank][cnt[bank]++] = word;
                }
            }
            return *std::max_element(cnt, cnt + 32);
        };
        int best = wavefronts(order);
        for (int m = 0; m < (1 << tc::SETBITS); ++m) {
            if (__builtin_popcount(m) != 5) continue;
            int cand[tc::SETBITS], nc = 0;
            for (int i = 0; i < tc::SETBITS; ++i)
                if ((m >> i) & 1) cand[nc++] = setbits[i];
            for (int i = 0; i < tc::SETBITS; ++i)
                if (!((m >> i) & 1)) cand[nc++] = setbits[i];
            const int w = wavefronts(cand);
            if (w < best) {
                best = w;
                std::copy(cand, cand + tc::SETBITS, order);
            }
        }
        for (int n = 0; n < tc::M; ++n) {
            uint32_t o = 0;
            for (int i = 0; i < tc::SETBITS; ++i)
                if ((n >> i) & 1) o |= 1u << order[i];
            P.setoff[n] = o;
        }
    }
    // Every pass with bit 0 free, bit 0 being the set bit of lane bit 0: lane
    // pairs swap one output each so that every store is 16 bytes (halving the
    // epilogue's store instructions).
    if (d.p[0] != 0 && order[0] == 0) B.xpair = 1;
    for (int n = 0; n < tc::M; ++n) {
        uint64_t ti = 0;
        for (int i = 0; i < tc::SETBITS; ++i)
            if ((n >> i) & 1) ti |= 1ull << tpos(order[i]);
        B.nidx[n] = (uint16_t)(B.swz ? tc::swz128((uint32_t)slot_of(ti)) : slot_of(ti));
    }
    for (int c = 0; c < D / 2; ++c) {
        uint64_t ti = 0;
        for (int i = 0; i < K - 1; ++i)
            if ((c >> i) & 1) ti |= 1ull << tpos(d.p[i]);
        B.cidx8[c] = (uint32_t)(B.swz ? tc::swz128((uint32_t)slot_of(ti)) : slot_of(ti)) * 8;
    }
    for (int h = 0; h < 2; ++h)
        for (int j = 0; j < D / 2; ++j) {
            const uint64_t x = (uint64_t)j << 7;
            const uint64_t ti = (x & ((1ull << hp) - 1)) | ((uint64_t)h << hp) | ((x >> hp) << (hp + 1));
            uint64_t o = 0;
            for (int i = 0; i < na; ++i)
                if ((ti >> i) & 1) o |= 1ull << all[i];
            B.boff[h][j] = o;
        }
#ifdef HQ_TC_DIAG_BUILD
    static const char *dg = getenv("HQ_TC_DIAG");
    B.diag = dg ? atoi(dg) : 0;
#endif
}

// psi (2^nl complex64) as a 2-D FP32 tensor [2^(nl-4) rows][32 floats] (128 B
// rows), box 8 rows = one 1 KB block, SWIZZLE_128B; the driver entry point is
// looked up once (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static int tc_encode_rows_map(CUtensorMap *map, void *psi, int nl) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f) return e != cudaSuccess ? (int)e : (int)cudaErrorNotSupported;
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    const cuuint64_t dims[2] = {32, 1ull << (nl - 4)};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {32, 8};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, psi, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Ring depth NS = 4 K-half slots and NP = 2 producer warps: measured on the
// 34q bench circuit in the sustained (power-capped) regime
// (tools/pass_times.py, round 1): (4, 2) beats (4, 1), (8, *) and the
// earlier cp.async kernel (3.91 s vs 4.28 s and 4.08 s).
template <int K, bool DIAG = false, bool PK = false>
static int tc_launch_b(void *psi, const tc::ParamsB &P, const std::conditional_t<PK, tc::PackB, tc::NoPack> &X,
                       const void *dev_payload, cudaStream_t st) {
    constexpr int NS = 4, NP = 2;
    using C = tc::CfgB<K, NS>;
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = smem_attr_once(tc::apply_tcb<K, NS, NP, DIAG, PK>, C::SMEM, attr);
    if (e != cudaSuccess) return (int)e;
    const int sms = sm_count();
    const uint64_t grid = P.h.ntiles < (uint64_t)sms ? P.h.ntiles : (uint64_t)sms;
    alignas(64) CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (P.swz) {
        int nl = K + tc::SETBITS;
        while ((1ull << (nl - K - tc::SETBITS)) < P.h.ntiles) ++nl;
        const int r = tc_encode_rows_map(&map, psi, nl);
        if (r) return r;
    }
    tc::apply_tcb<K, NS, NP, DIAG, PK><<<(unsigned)grid, tc::bk_threads(NP), C::SMEM, st>>>(
        reinterpret_cast<float2 *>(psi), P, reinterpret_cast<const __half *>(dev_payload), map, X);
    return (int)cudaGetLastError();
}

template <int K, bool PK>
static int tc_launch_l(void *psi, const tc::ParamsL &P, const std::conditional_t<PK, tc::PackL, tc::NoPack> &X,
                       const void *dev_payload, cudaStream_t st) {
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = smem_attr_once(tc::apply_tcL<K, PK>, tc::LB_SMEM, attr);
    if (e != cudaSuccess) return (int)e;
    const int sms = sm_count();
    const uint64_t grid = P.ntiles < (uint64_t)sms ? P.ntiles : (uint64_t)sms;
    tc::apply_tcL<K, PK><<<(unsigned)grid, tc::LB_THREADS, tc::LB_SMEM, st>>>(
        reinterpret_cast<float2 *>(psi), P, reinterpret_cast<const uint32_t *>(dev_payload), X);
    return (int)cudaGetLastError();
}

// apply+pack: write the pass out of place through the output map o (the
// tile part is permuted in the kernel, once per tile; the pattern and set
// parts here).  Bits 0 and 1 must stay in place (16-byte pattern pairs and
// lane-pair stores, whole 32-byte sectors).
bool tc_set_output(std::vector<char> &params, const OutSpec &o) {
    if (params.empty()) return false;
    const char tag = params.back();
    if (!o.active) return tag == 'B' || tag == 'L';
    OutMap m{};
    m.active = 1;
    m.npairs = o.npairs;
    for (int i = 0; i < o.npairs; ++i) {
        if (o.pa[i] < PACK_MIN_BIT || o.pb[i] < PACK_MIN_BIT) return false;
        m.pa[i] = o.pa[i];
        m.pb[i] = o.pb[i];
    }
    if (o.tmask && o.tsh < PACK_MIN_BIT) return false;
    m.tsh = o.tmask ? o.tsh : 0;
    m.tmask = o.tmask;
    m.add = o.add;
    for (int t = 0; t < 8; ++t) m.dst[t] = reinterpret_cast<uint64_t>(o.dst[t]);
    const uint64_t strip = ~((uint64_t)m.tmask << m.tsh);
    auto split = [&](uint64_t x, uint64_t &low, uint8_t &sel) {
        const uint64_t y = om_swap(x, m);
        sel = (uint8_t)((y >> m.tsh) & m.tmask);
        low = y & strip;
    };
    // layout of a packed block: [Params][Pack][tag], tag 'P' (mode H) / 'Q' (mode L)
    if (tag == 'B' || tag == 'P') {
        const tc::ParamsB B = *reinterpret_cast<const tc::ParamsB *>(params.data());
        tc::PackB X{};
        X.om = m;
        for (int c = 0; c < (1 << B.h.k); ++c) {
            uint64_t lo;
            split(B.h.off[c], lo, X.tpat[c]);
            X.poff8[c] = lo * 8;
        }
        for (int n = 0; n < tc::M; ++n) {
            uint64_t lo;
            split(B.h.setoff[n], lo, X.tset[n]);
            X.psoff8[n] = lo * 8;
        }
        params.assign(sizeof(tc::ParamsB) + sizeof(tc::PackB) + 1, 0);
        memcpy(params.data(), &B, sizeof B);
        memcpy(params.data() + sizeof B, &X, sizeof X);
        params.back() = 'P';
        return true;
    }
    if (tag == 'L' || tag == 'Q') {
        const tc::ParamsL L = *reinterpret_cast<const tc::ParamsL *>(params.data());
        tc::PackL X{};
        X.om = m;
        for (int c = 0; c < (1 << L.k); ++c) split(L.off[c], X.poff[c], X.tpat[c]);
        for (int n = 0; n < (L.k == 5 ? 128 : 64); ++n) split(L.setoff[n], X.psetoff[n], X.tset[n]);
        params.assign(sizeof(tc::ParamsL) + sizeof(tc::PackL) + 1, 0);
        memcpy(params.data(), &L, sizeof L);
        memcpy(params.data() + sizeof L, &X, sizeof X);
        params.back() = 'Q';
        return true;
    }
    return false;
}

// Both modes scale the state into the FP16 range by 2^ea with
// max |psi| 2^ea <= 2^14, from the runtime's rigorous bound on max |amplitude|.
void tc_set_amp_bound(std::vector<char> &params, double bound) {
    if (params.empty()) return;
    int ex = 0;
    if (bound > 0 && std::isfinite(bound)) std::frexp(bound, &ex);   // bound < 2^ex
    const int ea = std::max(-126, std::min(127, 14 - ex));
    const char tag = params.back();
    if (tag == 'B' || tag == 'P') reinterpret_cast<tc::ParamsB *>(params.data())->h.ea = ea;
    else if (tag == 'L' || tag == 'Q') reinterpret_cast<tc::ParamsL *>(params.data())->ea = ea;
}

// params: a tc::ParamsB (mode H) or tc::ParamsL (mode L) block followed by
// one tag byte ('B' or 'L').
int tc_launch(void *psi, const void *params, size_t params_size, const void *dev_payload,
              void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const char *pb = reinterpret_cast<const char *>(params);
    const char tag = pb[params_size - 1];
    if (tag == 'L') {
        const tc::ParamsL &L = *reinterpret_cast<const tc::ParamsL *>(pb);
        return L.k == 5 ? tc_launch_l<5, false>(psi, L, tc::NoPack{}, dev_payload, st)
                        : tc_launch_l<6, false>(psi, L, tc::NoPack{}, dev_payload, st);
    }
    if (tag == 'Q') {
        const tc::ParamsL &L = *reinterpret_cast<const tc::ParamsL *>(pb);
        const tc::PackL &X = *reinterpret_cast<const tc::PackL *>(pb + sizeof(tc::ParamsL));
        return L.k == 5 ? tc_launch_l<5, true>(psi, L, X, dev_payload, st)
                        : tc_launch_l<6, true>(psi, L, X, dev_payload, st);
    }
    const tc::ParamsB &B = *reinterpret_cast<const tc::ParamsB *>(pb);
    if (tag == 'P') {
        const tc::PackB &X = *reinterpret_cast<const tc::PackB *>(pb + sizeof(tc::ParamsB));
        return B.h.k == 5 ? tc_launch_b<5, false, true>(psi, B, X, dev_payload, st)
                          : tc_launch_b<6, false, true>(psi, B, X, dev_payload, st);
    }
    if (tag != 'B') return (int)cudaErrorInvalidValue;
#ifdef HQ_TC_DIAG_BUILD
    if (B.diag) return B.h.k == 5 ? tc_launch_b<5, true>(psi, B, tc::NoPack{}, dev_payload, st)
                                  : tc_launch_b<6, true>(psi, B, tc::NoPack{}, dev_payload, st);
#endif
    return B.h.k == 5 ? tc_launch_b<5>(psi, B, tc::NoPack{}, dev_payload, st)
                      : tc_launch_b<6>(psi, B, tc::NoPack{}, dev_payload, st);
}

}  // namespace hq
