// SIMT apply kernels (sm_100a) and the small state kernels (init, norm,
// permute, gather/scatter).
//
// The operation: for every
// outer index o in [0, 2^(n_l-k)) take the gather set of 2^k amplitudes whose
// index agrees with o off the k target bits, and replace it by U times it.
// Each pass streams the whole shard through HBM once (read + write), so the
// kernels are built for bandwidth:
//
//  * apply_reg<R,K,T0,KL>  (k <= 4): each warp owns 32 lanes x 2^|R| amplitudes.
//    Lanes cover physical bits [LB, LB+5) with 16-byte vectors (c64: two
//    amplitudes per vector, bit 0 in-thread; c128: one), so every load/store
//    instruction of a warp is a fully coalesced 512-byte access.  Target bits
//    above the lane range are register bits (direct loads at stride 2^p).
//    Targets inside the lane range are moved into registers with warp shuffles
//    (a lane-bit <-> register-bit transpose against a spare high bit), which
//    is the GPU counterpart of the paper's "qubits are swapped to fully exploit
//    AVX instructions".  U travels in the kernel's parameter space
//    (constant bank), so every complex MAC is 4 FFMA/DFMA with a constant
//    operand and no load instruction.
//  * apply_gen<R,K> (any k <= 6, any placement, small n): one thread per
//    gather set, U from global memory (L1 broadcast).  Correctness fallback.
//
// Canonical target order: the host permutes U so that U-index bit i <-> the
// i-th smallest physical target bit (exact: a permutation of rows/columns).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "hq_internal.h"

namespace hq {

template <typename R> struct C2;
template <> struct C2<float> { using T = float2; };
template <> struct C2<double> { using T = double2; };

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int s) {
    const uint64_t lo = x & ((1ull << s) - 1);
    return ((x >> s) << (s + 1)) | lo;
}

// Checked build (-DHQ_DEVICE_CHECKS, lib/libhq_check.so): every SIMT store
// must land inside the buffer of the pass (in place: the shard; apply+pack:
// one of the output-map buffers).
#ifdef HQ_DEVICE_CHECKS
#include <cstdio>
__device__ __noinline__ void hq_store_fail(uint64_t idx, uint64_t lim, int where) {
    printf("hq device check %d: store index %llu >= %llu (block %d thread %d)\n", where,
           (unsigned long long)idx, (unsigned long long)lim, blockIdx.x, threadIdx.x);
    __trap();
}
#define HQ_CHECK_IDX(idx, lim, where) \
    do { if ((uint64_t)(idx) >= (uint64_t)(lim)) hq_store_fail((idx), (lim), (where)); } while (0)
#else
#define HQ_CHECK_IDX(idx, lim, where) ((void)0)
#endif

// ------------------------------------------------------------------ fast SIMT kernel

struct RegParams {
    uint64_t voff[32];   // offset (in 16-byte vectors) of each register vector
    uint64_t nunits;     // number of threads with work (= 32 * warps)
    int S[6];            // ascending insertion positions in warp space (count K-T0)
    int la[5];           // lane bit (0..4) of each lane target, canonical order
};

// apply+pack output of the SIMT kernel (positions in load units): pvoff[v] =
// om_swap(voff[v]) without the selector bits, tv[v] = its selector bits.  A
// separate kernel argument that only the PK instantiation carries: a larger
// RegParams alone raised the in-place kernel from 80 to 127 registers.
struct RegPack {
    OutMap om;
    uint64_t pvoff[32];
    uint8_t tv[32];
};
struct NoPack {};

template <typename R, int K> struct UParam {
    typename C2<R>::T u[1 << K][1 << K];
};

// Complex multiply-accumulate acc += u * v.  For complex64 this is two packed
// FFMA2 (fma.rn.f32x2, sm_100) instructions: (ar, ai) += (ur, ur) * (vr, vi)
// and (ar, ai) += (-ui, ui) * (vi, vr); ptxas folds the broadcast, swap and
// negation into FFMA2 operand modifiers and takes u from a uniform register.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float2 unpk2(unsigned long long r) {
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}

template <int D>
__device__ __forceinline__ void matvec(const float2 (&u)[D][D], const float2 *v, float2 *out) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
        unsigned long long acc = 0ull;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            acc = ffma2(pk2(u[r][c].x, u[r][c].x), pk2(v[c].x, v[c].y), acc);
            acc = ffma2(pk2(-u[r][c].y, u[r][c].y), pk2(v[c].y, v[c].x), acc);
        }
        out[r] = unpk2(acc);
    }
}

template <int D>
__device__ __forceinline__ void matvec(const double2 (&u)[D][D], const double2 *v, double2 *out) {
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double ar = 0, ai = 0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            ar = fma(u[r][c].x, v[c].x, ar);
            ar = fma(-u[r][c].y, v[c].y, ar);
            ai = fma(u[r][c].x, v[c].y, ai);
            ai = fma(u[r][c].y, v[c].x, ai);
        }
        out[r].x = ar;
        out[r].y = ai;
    }
}

// lane bit la <-> register bit e transpose (an involution) over the NR registers
template <typename V, int NR>
__device__ __forceinline__ void lane_transpose(V *x, int la, int e, int lane) {
    const bool hi = (lane >> la) & 1;
#pragma unroll
    for (int j0 = 0; j0 < NR; ++j0) {
        if (j0 & (1 << e)) continue;
        const int j1 = j0 | (1 << e);
        V snd;
        snd.x = hi ? x[j0].x : x[j1].x;
        snd.y = hi ? x[j0].y : x[j1].y;
        V rcv;
        rcv.x = __shfl_xor_sync(0xffffffffu, snd.x, 1 << la);
        rcv.y = __shfl_xor_sync(0xffffffffu, snd.y, 1 << la);
        if (hi) x[j0] = rcv; else x[j1] = rcv;
    }
}

// VEC = amplitudes per load: 2 (complex64 as float4, physical bit 0 in-thread)
// or 1 (complex64 as float2 / complex128 as double2).  T0: bit 0 is a target
// (VEC == 2 only).  KL: number of targets inside the lane bit range.
// PK: apply+pack variant (out-of-place through P.om); a separate
// instantiation so the in-place kernel keeps its register budget (the
// runtime branch cost 80 -> 128 registers and occupancy at k = 4).
template <typename R, int VEC, int K, int T0, int KL, bool PK>
__global__ void __launch_bounds__(128)
apply_reg(typename C2<R>::T *__restrict__ psi, const __grid_constant__ RegParams P,
          const __grid_constant__ UParam<R, K> U,
          const __grid_constant__ std::conditional_t<PK, RegPack, NoPack> X) {
    using V = typename C2<R>::T;
    constexpr int NB0 = (VEC == 2 && !T0) ? 1 : 0;              // bit 0 as non-target register bit
    constexpr int NR = 1 << (K + NB0);                           // amplitudes per thread
    constexpr int P0 = T0 ? 0 : K;                               // register bit holding phys bit 0
    constexpr int NV = NR / VEC;                                 // loads per thread
    constexpr int NS = K - T0;                                   // register phys bits above lanes

    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= P.nunits) return;
    const int lane = threadIdx.x & 31;
    uint64_t w = tid >> 5;
#pragma unroll
    for (int i = 0; i < NS; ++i) w = insert_zero(w, P.S[i]);
    const uint64_t base = (w << 5) | (uint64_t)lane;             // in load units

    V x[NR];
    if constexpr (VEC == 2) {
        const float4 *src = reinterpret_cast<const float4 *>(psi);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int j0 = ((v >> P0) << (P0 + 1)) | (v & ((1 << P0) - 1));
            const int j1 = j0 | (1 << P0);
            const float4 t = src[base + P.voff[v]];
            x[j0] = make_float2(t.x, t.y);
            x[j1] = make_float2(t.z, t.w);
        }
    } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) x[v] = psi[base + P.voff[v]];
    }

#pragma unroll
    for (int i = 0; i < KL; ++i) lane_transpose<V, NR>(x, P.la[i], T0 + i, lane);

#pragma unroll
    for (int s = 0; s < (1 << NB0); ++s) {
        V out[1 << K];
        matvec<1 << K>(U.u, x + (s << K), out);
#pragma unroll
        for (int r = 0; r < (1 << K); ++r) x[r | (s << K)] = out[r];
    }

#pragma unroll
    for (int i = KL - 1; i >= 0; --i) lane_transpose<V, NR>(x, P.la[i], T0 + i, lane);

    if constexpr (PK) {
        // apply+pack: out-of-place, bit-permuted (and buffer-selected) output
        const uint64_t yb = om_swap(base, X.om);
        const uint32_t tb = (uint32_t)(yb >> X.om.tsh) & X.om.tmask;
        const uint64_t lb = (yb & ~((uint64_t)X.om.tmask << X.om.tsh)) | X.om.add;
        if constexpr (VEC == 2) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int j0 = ((v >> P0) << (P0 + 1)) | (v & ((1 << P0) - 1));
                const int j1 = j0 | (1 << P0);
                float4 *dst = reinterpret_cast<float4 *>(X.om.dst[tb | X.tv[v]]);
                HQ_CHECK_IDX(lb | X.pvoff[v], P.nunits * NV, 11);
                dst[lb | X.pvoff[v]] = make_float4(x[j0].x, x[j0].y, x[j1].x, x[j1].y);
            }
        } else {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                HQ_CHECK_IDX(lb | X.pvoff[v], P.nunits * NV, 12);
                reinterpret_cast<V *>(X.om.dst[tb | X.tv[v]])[lb | X.pvoff[v]] = x[v];
            }
        }
    } else if constexpr (VEC == 2) {
        float4 *dst = reinterpret_cast<float4 *>(psi);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int j0 = ((v >> P0) << (P0 + 1)) | (v & ((1 << P0) - 1));
            const int j1 = j0 | (1 << P0);
            HQ_CHECK_IDX(base + P.voff[v], P.nunits * NV, 13);
            dst[base + P.voff[v]] = make_float4(x[j0].x, x[j0].y, x[j1].x, x[j1].y);
        }
    } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            HQ_CHECK_IDX(base + P.voff[v], P.nunits * NV, 14);
            psi[base + P.voff[v]] = x[v];
        }
    }
}

// ------------------------------------------------------------------ generic kernel

struct GenParams {
    uint64_t off[64];    // amplitude offset of U-index c (canonical order)
    uint64_t nsets;      // 2^(n_l - k)
    int s[6];            // ascending target bits
    OutMap om;           // out-of-place output (om.active), amplitude units
};

// output element for amplitude index x (in place, or through the output map)
template <typename V>
__device__ __forceinline__ V *gen_out(V *psi, uint64_t x, const OutMap &om) {
    if (!om.active) return psi + x;
    const uint64_t y = om_swap(x, om);
    const uint32_t t = (uint32_t)(y >> om.tsh) & om.tmask;
    return reinterpret_cast<V *>(om.dst[t]) + ((y & ~((uint64_t)om.tmask << om.tsh)) | om.add);
}

template <typename R, int K>
__global__ void __launch_bounds__(128)
apply_gen(typename C2<R>::T *__restrict__ psi, const __grid_constant__ GenParams P,
          const typename C2<R>::T *__restrict__ Ud) {
    using V = typename C2<R>::T;
    constexpr int D = 1 << K;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < P.nsets;
         o += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = o;
#pragma unroll
        for (int j = 0; j < K; ++j) base = insert_zero(base, P.s[j]);
        V v[D];
#pragma unroll
        for (int c = 0; c < D; ++c) v[c] = psi[base + P.off[c]];
        for (int r = 0; r < D; ++r) {
            R ar = 0, ai = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const V u = __ldg(&Ud[r * D + c]);
                ar = fma(u.x, v[c].x, ar);
                ar = fma(-u.y, v[c].y, ar);
                ai = fma(u.x, v[c].y, ai);
                ai = fma(u.y, v[c].x, ai);
            }
            V w;
            w.x = ar;
            w.y = ai;
            *gen_out(psi, base + P.off[r], P.om) = w;
        }
    }
}

// Small-state variant of the generic kernel: one warp per gather set (the
// set is staged in shared memory, lanes own output rows), so that a pass over
// a few thousand amplitudes is not a handful of serial threads.
template <typename R, int K>
__global__ void __launch_bounds__(128)
apply_gen_warp(typename C2<R>::T *__restrict__ psi, const __grid_constant__ GenParams P,
               const typename C2<R>::T *__restrict__ Ud) {
    using V = typename C2<R>::T;
    constexpr int D = 1 << K;
    __shared__ V sv[4][D];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t o = (uint64_t)blockIdx.x * 4 + w;
    if (o >= P.nsets) return;
    uint64_t base = o;
#pragma unroll
    for (int j = 0; j < K; ++j) base = insert_zero(base, P.s[j]);
    for (int c = lane; c < D; c += 32) sv[w][c] = psi[base + P.off[c]];
    __syncwarp();
    for (int r = lane; r < D; r += 32) {
        R ar = 0, ai = 0;
        for (int c = 0; c < D; ++c) {
            const V u = __ldg(&Ud[r * D + c]);
            const V v = sv[w][c];
            ar = fma(u.x, v.x, ar);
            ar = fma(-u.y, v.y, ar);
            ai = fma(u.x, v.y, ai);
            ai = fma(u.y, v.x, ai);
        }
        V out;
        out.x = ar;
        out.y = ai;
        *gen_out(psi, base + P.off[r], P.om) = out;
    }
}

// ------------------------------------------------------------------ pair gather (row f1)
// One thread per local gather set of the k-1 local targets: reads the
// 2^(k-1) amplitudes of the set from this rank and from its partner (peer
// memory over NVLink), forms the full 2^k input (canonical bit k-1 = the
// global target: this rank holds half `half`), and writes the 2^(k-1)
// outputs of its own half into dst.  NVLink-bound (one partner shard read per
// pass); used only for isolated global accesses.
template <typename R, int K>
__global__ void __launch_bounds__(128)
apply_pair_gather(const typename C2<R>::T *__restrict__ me, const typename C2<R>::T *__restrict__ peer,
                  typename C2<R>::T *__restrict__ dst, const __grid_constant__ GenParams P, int half,
                  const typename C2<R>::T *__restrict__ Ud) {
    using V = typename C2<R>::T;
    constexpr int D = 1 << K, H = D / 2;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < P.nsets;
         o += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = o;
#pragma unroll
        for (int j = 0; j < K - 1; ++j) base = insert_zero(base, P.s[j]);
        V v[D];
#pragma unroll
        for (int c = 0; c < H; ++c) {
            v[c | (half * H)] = me[base + P.off[c]];
            v[c | ((1 - half) * H)] = peer[base + P.off[c]];
        }
        for (int r = 0; r < H; ++r) {
            const int row = r | (half * H);
            R ar = 0, ai = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const V u = __ldg(&Ud[row * D + c]);
                ar = fma(u.x, v[c].x, ar);
                ar = fma(-u.y, v[c].y, ar);
                ai = fma(u.x, v[c].y, ai);
                ai = fma(u.y, v[c].x, ai);
            }
            V w;
            w.x = ar;
            w.y = ai;
            HQ_CHECK_IDX(base + P.off[r], P.nsets << (K - 1), 15);
            dst[base + P.off[r]] = w;
        }
    }
}

template <typename R>
static cudaError_t launch_pg(const void *me, const void *peer, void *dst, const GenParams &P, int K, int half,
                             const void *dU, cudaStream_t st) {
    using V = typename C2<R>::T;
    uint64_t blocks = (P.nsets + 127) / 128;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    if (blocks == 0) blocks = 1;
    const V *a = reinterpret_cast<const V *>(me), *b = reinterpret_cast<const V *>(peer);
    V *o = reinterpret_cast<V *>(dst);
    const V *u = reinterpret_cast<const V *>(dU);
    switch (K) {
        case 1: apply_pair_gather<R, 1><<<(unsigned)blocks, 128, 0, st>>>(a, b, o, P, half, u); break;
        case 2: apply_pair_gather<R, 2><<<(unsigned)blocks, 128, 0, st>>>(a, b, o, P, half, u); break;
        case 3: apply_pair_gather<R, 3><<<(unsigned)blocks, 128, 0, st>>>(a, b, o, P, half, u); break;
        case 4: apply_pair_gather<R, 4><<<(unsigned)blocks, 128, 0, st>>>(a, b, o, P, half, u); break;
        case 5: apply_pair_gather<R, 5><<<(unsigned)blocks, 128, 0, st>>>(a, b, o, P, half, u); break;
        case 6: apply_pair_gather<R, 6><<<(unsigned)blocks, 128, 0, st>>>(a, b, o, P, half, u); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int launch_pair_gather(int dtype, const void *psi_me, const void *psi_peer, void *dst, const ApplyDesc &d,
                       int half, const void *dev_U, void *stream) {
    // d.k = number of targets including the global one; d.p[0..k-2] local (ascending)
    GenParams gp{};
    const int kl = d.k - 1;
    for (int c = 0; c < (1 << kl); ++c) {
        uint64_t o = 0;
        for (int i = 0; i < kl; ++i)
            if ((c >> i) & 1) o |= 1ull << d.p[i];
        gp.off[c] = o;
    }
    for (int i = 0; i < kl; ++i) gp.s[i] = d.p[i];
    gp.nsets = 1ull << (d.n_local - kl);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const cudaError_t e = dtype == HQ_C64 ? launch_pg<float>(psi_me, psi_peer, dst, gp, d.k, half, dev_U, st)
                                          : launch_pg<double>(psi_me, psi_peer, dst, gp, d.k, half, dev_U, st);
    return (int)e;
}

// ------------------------------------------------------------------ dispatch

namespace {

constexpr int kThreads = 128;

template <typename R, int VEC, int K, int T0, int KL>
cudaError_t launch_reg_t(void *psi, const RegParams &P, const RegPack *X, const void *host_U, cudaStream_t st) {
    UParam<R, K> U;
    memcpy(&U, host_U, sizeof(U));
    const uint64_t blocks = (P.nunits + kThreads - 1) / kThreads;
    if (X)
        apply_reg<R, VEC, K, T0, KL, true><<<(unsigned)blocks, kThreads, 0, st>>>(
            reinterpret_cast<typename C2<R>::T *>(psi), P, U, *X);
    else
        apply_reg<R, VEC, K, T0, KL, false><<<(unsigned)blocks, kThreads, 0, st>>>(
            reinterpret_cast<typename C2<R>::T *>(psi), P, U, NoPack{});
    return cudaGetLastError();
}

template <typename R, int VEC, int K, int T0>
cudaError_t launch_reg_kl(int KL, void *psi, const RegParams &P, const RegPack *X, const void *hU, cudaStream_t st) {
    switch (KL) {
        case 0: return launch_reg_t<R, VEC, K, T0, 0>(psi, P, X, hU, st);
        case 1: if constexpr (K - T0 >= 1) return launch_reg_t<R, VEC, K, T0, 1>(psi, P, X, hU, st); break;
        case 2: if constexpr (K - T0 >= 2) return launch_reg_t<R, VEC, K, T0, 2>(psi, P, X, hU, st); break;
        case 3: if constexpr (K - T0 >= 3) return launch_reg_t<R, VEC, K, T0, 3>(psi, P, X, hU, st); break;
        case 4: if constexpr (K - T0 >= 4) return launch_reg_t<R, VEC, K, T0, 4>(psi, P, X, hU, st); break;
        default: break;
    }
    return cudaErrorInvalidValue;
}

template <int K>
cudaError_t launch_reg_f(int VEC, int T0, int KL, void *psi, const RegParams &P, const RegPack *X, const void *hU,
                         cudaStream_t st) {
    if (VEC == 2) {
        if (T0) return launch_reg_kl<float, 2, K, 1>(KL, psi, P, X, hU, st);
        if constexpr (K <= 3) return launch_reg_kl<float, 2, K, 0>(KL, psi, P, X, hU, st);
        return cudaErrorInvalidValue;
    }
    return launch_reg_kl<float, 1, K, 0>(KL, psi, P, X, hU, st);
}

template <typename R>
cudaError_t launch_gen(int K, void *psi, const GenParams &P, const void *dU, cudaStream_t st) {
    using V = typename C2<R>::T;
    if (P.nsets <= (1ull << 15)) {
        const unsigned blocks = (unsigned)((P.nsets + 3) / 4);
        V *p = reinterpret_cast<V *>(psi);
        const V *u = reinterpret_cast<const V *>(dU);
        switch (K) {
            case 1: apply_gen_warp<R, 1><<<blocks, 128, 0, st>>>(p, P, u); break;
            case 2: apply_gen_warp<R, 2><<<blocks, 128, 0, st>>>(p, P, u); break;
            case 3: apply_gen_warp<R, 3><<<blocks, 128, 0, st>>>(p, P, u); break;
            case 4: apply_gen_warp<R, 4><<<blocks, 128, 0, st>>>(p, P, u); break;
            case 5: apply_gen_warp<R, 5><<<blocks, 128, 0, st>>>(p, P, u); break;
            case 6: apply_gen_warp<R, 6><<<blocks, 128, 0, st>>>(p, P, u); break;
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    uint64_t blocks = (P.nsets + kThreads - 1) / kThreads;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    if (blocks == 0) blocks = 1;
    V *p = reinterpret_cast<V *>(psi);
    const V *u = reinterpret_cast<const V *>(dU);
    switch (K) {
        case 1: apply_gen<R, 1><<<(unsigned)blocks, kThreads, 0, st>>>(p, P, u); break;
        case 2: apply_gen<R, 2><<<(unsigned)blocks, kThreads, 0, st>>>(p, P, u); break;
        case 3: apply_gen<R, 3><<<(unsigned)blocks, kThreads, 0, st>>>(p, P, u); break;
        case 4: apply_gen<R, 4><<<(unsigned)blocks, kThreads, 0, st>>>(p, P, u); break;
        case 5: apply_gen<R, 5><<<(unsigned)blocks, kThreads, 0, st>>>(p, P, u); break;
        case 6: apply_gen<R, 6><<<(unsigned)blocks, kThreads, 0, st>>>(p, P, u); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// Plan the register kernel for this placement; returns false if it does not
// apply (then the generic kernel runs).  VEC: 2 for complex64 when bit 0 is a
// target or k <= 3 (float4 access, two gather sets per thread when bit 0 is
// not a target), else 1 (float2 / double2 access, one gather set per thread).
bool plan_reg(int dtype, const ApplyDesc &d, RegParams &P, int &VEC, int &T0, int &KL) {
    const int K = d.k;
    if (K > 4) return false;
    const bool t0 = dtype == HQ_C64 && d.p[0] == 0;
    VEC = (dtype == HQ_C64 && (t0 || K <= 3)) ? 2 : 1;
    const int LB = VEC == 2 ? 1 : 0;
    const int lane_hi = LB + 5;                    // lane bits [LB, LB+5)
    T0 = (VEC == 2 && t0) ? 1 : 0;
    KL = 0;
    for (int i = T0; i < K; ++i)
        if (d.p[i] < lane_hi) ++KL;
    const int used = lane_hi + (K - T0);
    if (d.n_local - used < 8) return false;       // too small to fill a GPU
    int extras[5], ne = 0;
    for (int b = lane_hi; ne < KL && b < d.n_local; ++b) {
        bool tgt = false;
        for (int i = 0; i < K; ++i) tgt |= d.p[i] == b;
        if (!tgt) extras[ne++] = b;
    }
    if (ne < KL) return false;
    // register bit -> physical bit (load-phase meaning)
    int regphys[7];
    int nreg = 0;
    if (T0) regphys[nreg++] = 0;
    for (int i = 0; i < KL; ++i) regphys[nreg++] = extras[i];
    for (int i = T0 + KL; i < K; ++i) regphys[nreg++] = d.p[i];
    const int NB0 = (VEC == 2 && !T0) ? 1 : 0;
    if (NB0) regphys[nreg++] = 0;                 // register bit K
    const int P0 = T0 ? 0 : K;
    const int NR = 1 << (K + NB0);
    for (int v = 0; v < NR / VEC; ++v) {
        int j0 = v;
        if (VEC == 2) j0 = ((v >> P0) << (P0 + 1)) | (v & ((1 << P0) - 1));
        uint64_t off = 0;
        for (int b = 0; b < nreg; ++b)
            if ((j0 >> b) & 1) off |= 1ull << (regphys[b] - LB);
        P.voff[v] = off;
    }
    int S[6], ns = 0;
    for (int b = 0; b < nreg; ++b)
        if (regphys[b] >= lane_hi) S[ns++] = regphys[b] - lane_hi;
    for (int i = 1; i < ns; ++i) {
        int x = S[i], j = i - 1;
        while (j >= 0 && S[j] > x) { S[j + 1] = S[j]; --j; }
        S[j + 1] = x;
    }
    if (ns != K - T0) return false;
    for (int i = 0; i < ns; ++i) P.S[i] = S[i];
    for (int i = 0; i < KL; ++i) P.la[i] = d.p[T0 + i] - LB;
    P.nunits = 1ull << (d.n_local - LB - ns);     // threads = 32 lanes x warps
    return true;
}

}  // namespace

// ------------------------------------------------------------------ complex128, k = 5, 6: FP64 tiles
// At k = 5, 6 a complex128 pass costs 2^(k-2) = 8, 16 flop/B: above the FP64
// ridge (~6 flop/B), so the bound is the FP64 pipe (<= ~0.7 / ~0.36 of the
// HBM roofline), and tcgen05 has no f64 kind.  The pass is then a small ZGEMM
// per tile: out (64 sets x D) = in (64 sets x D) . U^T.
//   * U^T staged once per persistent CTA in shared memory, Us[c][r] = U[r][c];
//   * the tile's inputs In[c][set] (set-contiguous: the 16 lanes of a
//     half-warp read 16 consecutive sets, conflict-free) double-buffered with
//     cp.async, the next tile loading while this one is computed;
//   * 256 threads, each 4 sets x D/16 rows of complex accumulators (k = 6:
//     64 DFMA per 8 shared loads); stores for a fixed row are 16 consecutive
//     sets.
// In place: a tile's outputs are exactly its inputs' amplitudes.
constexpr int ZT_SETS = 64;

template <int K>
__global__ void __launch_bounds__(256, K == 6 ? 1 : 2)
apply_ztile(double2 *__restrict__ psi, const __grid_constant__ GenParams P, const double2 *__restrict__ U,
            uint64_t ntiles) {
    constexpr int D = 1 << K, RJ = D / 16;       // rows per thread
    extern __shared__ __align__(16) double2 zsm[];
    double2 *Us = zsm;                           // [D][D]: Us[c][r] = U[r][c]
    double2 *In = zsm + D * D;                   // [2][D][ZT_SETS]
    const int tid = threadIdx.x;
    for (int i = tid; i < D * D; i += 256) {
        const int r = i / D, c = i % D;
        Us[c * D + r] = U[i];
    }
    auto base_of = [&](uint64_t o) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int b = P.s[i];
            o = ((o >> b) << (b + 1)) | (o & ((1ull << b) - 1));
        }
        return o;
    };
    const int lset = tid & (ZT_SETS - 1), lc0 = tid >> 6;          // loader: one set, c = lc0 + 4m
    auto prefetch = [&](uint64_t t, int buf) {
        const double2 *src = psi + base_of(t * ZT_SETS + lset);
        const uint32_t dst0 = (uint32_t)__cvta_generic_to_shared(In + buf * D * ZT_SETS + lset);
#pragma unroll
        for (int m = 0; m < D / 4; ++m) {
            const int c = lc0 + 4 * m;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + (uint32_t)(c * ZT_SETS) * 16),
                         "l"(src + P.off[c])
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int tx = tid & 15, ty = tid >> 4;
    const uint64_t G = gridDim.x;
    uint64_t t = blockIdx.x;
    if (t < ntiles) prefetch(t, 0);
    for (int it = 0; t < ntiles; t += G, ++it) {
        const int buf = it & 1;
        if (t + G < ntiles) {
            prefetch(t + G, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double2 *in = In + buf * D * ZT_SETS;
        double2 acc[4][RJ];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < RJ; ++j) acc[i][j] = make_double2(0.0, 0.0);
#pragma unroll 4
        for (int c = 0; c < D; ++c) {
            double2 a[4], b[RJ];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = in[c * ZT_SETS + tx + 16 * i];
#pragma unroll
            for (int j = 0; j < RJ; ++j) b[j] = Us[c * D + ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < RJ; ++j) {
                    acc[i][j].x = fma(a[i].x, b[j].x, acc[i][j].x);
                    acc[i][j].x = fma(-a[i].y, b[j].y, acc[i][j].x);
                    acc[i][j].y = fma(a[i].x, b[j].y, acc[i][j].y);
                    acc[i][j].y = fma(a[i].y, b[j].x, acc[i][j].y);
                }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double2 *dst = psi + base_of(t * ZT_SETS + tx + 16 * i);
#pragma unroll
            for (int j = 0; j < RJ; ++j) dst[P.off[ty + 16 * j]] = acc[i][j];
        }
        __syncthreads();        // every thread is done with In[buf] before it is refilled
    }
}

template <int K>
static cudaError_t launch_ztile(void *psi, const GenParams &P, const void *dU, cudaStream_t st) {
    constexpr int D = 1 << K;
    constexpr size_t smem = sizeof(double2) * (D * D + 2 * D * ZT_SETS);
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = smem_attr_once(apply_ztile<K>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const uint64_t ntiles = P.nsets / ZT_SETS;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t per = K == 6 ? 1 : 2;
    const uint64_t grid = ntiles < per * sms ? ntiles : per * sms;
    apply_ztile<K><<<(unsigned)grid, 256, smem, st>>>(reinterpret_cast<double2 *>(psi), P,
                                                      reinterpret_cast<const double2 *>(dU), ntiles);
    return cudaGetLastError();
}

// OutSpec (amplitude bit positions) -> OutMap in units of 2^lb amplitudes.
// False when a swapped bit, the selector or the added offset falls inside a
// unit (such a map would split a vector).
static bool out_map(const OutSpec &o, int lb, OutMap &m) {
    m = OutMap{};
    if (!o.active) return true;
    m.active = 1;
    m.npairs = o.npairs;
    for (int i = 0; i < o.npairs; ++i) {
        if (o.pa[i] < lb || o.pb[i] < lb) return false;
        m.pa[i] = o.pa[i] - lb;
        m.pb[i] = o.pb[i] - lb;
    }
    if (o.tmask && o.tsh < lb) return false;
    if (o.add & ((1ull << lb) - 1)) return false;
    m.tsh = o.tmask ? o.tsh - lb : 0;
    m.tmask = o.tmask;
    m.add = o.add >> lb;
    for (int t = 0; t < 8; ++t) m.dst[t] = reinterpret_cast<uint64_t>(o.dst[t]);
    return true;
}

static bool reg_out_tables(const RegParams &rp, RegPack &X, int VEC, int K, int T0, const OutSpec *out) {
    const int LB = VEC == 2 ? 1 : 0;
    if (!out_map(out ? *out : OutSpec{}, LB, X.om)) return false;
    if (!X.om.active) return true;
    const int NB0 = (VEC == 2 && !T0) ? 1 : 0;
    const int NV = (1 << (K + NB0)) / VEC;
    for (int v = 0; v < NV; ++v) {
        const uint64_t y = om_swap(rp.voff[v], X.om);
        X.tv[v] = (uint8_t)((y >> X.om.tsh) & X.om.tmask);
        X.pvoff[v] = y & ~((uint64_t)X.om.tmask << X.om.tsh);
    }
    return true;
}

bool apply_supports_out(int dtype, const ApplyDesc &d, const OutSpec &o) {
    RegParams rp;
    int VEC = 1, T0 = 0, KL = 0;
    RegPack X;
    if (plan_reg(dtype, d, rp, VEC, T0, KL)) return reg_out_tables(rp, X, VEC, d.k, T0, &o);
    if (dtype == HQ_C128 && d.k >= 5 && (1ull << (d.n_local - d.k)) >= (1ull << 12)) return false;   // apply_ztile
    OutMap m;
    return out_map(o, 0, m);
}

int launch_apply(int dtype, void *psi, const ApplyDesc &d, const void *host_U, const void *dev_U,
                 void *stream, int *launches, const OutSpec *out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    RegParams rp;
    int VEC = 1, T0 = 0, KL = 0;
    cudaError_t e;
    if (host_U && plan_reg(dtype, d, rp, VEC, T0, KL)) {
        RegPack X;
        if (!reg_out_tables(rp, X, VEC, d.k, T0, out)) return (int)cudaErrorInvalidValue;
        const RegPack *xp = X.om.active ? &X : nullptr;
        if (dtype == HQ_C64) {
            switch (d.k) {
                case 1: e = launch_reg_f<1>(VEC, T0, KL, psi, rp, xp, host_U, st); break;
                case 2: e = launch_reg_f<2>(VEC, T0, KL, psi, rp, xp, host_U, st); break;
                case 3: e = launch_reg_f<3>(VEC, T0, KL, psi, rp, xp, host_U, st); break;
                default: e = launch_reg_f<4>(VEC, T0, KL, psi, rp, xp, host_U, st); break;
            }
        } else {
            switch (d.k) {
                case 1: e = launch_reg_kl<double, 1, 1, 0>(KL, psi, rp, xp, host_U, st); break;
                case 2: e = launch_reg_kl<double, 1, 2, 0>(KL, psi, rp, xp, host_U, st); break;
                case 3: e = launch_reg_kl<double, 1, 3, 0>(KL, psi, rp, xp, host_U, st); break;
                default: e = launch_reg_kl<double, 1, 4, 0>(KL, psi, rp, xp, host_U, st); break;
            }
        }
    } else {
        GenParams gp;
        for (int c = 0; c < (1 << d.k); ++c) {
            uint64_t o = 0;
            for (int i = 0; i < d.k; ++i)
                if ((c >> i) & 1) o |= 1ull << d.p[i];
            gp.off[c] = o;
        }
        for (int i = 0; i < d.k; ++i) gp.s[i] = d.p[i];
        gp.nsets = 1ull << (d.n_local - d.k);
        if (!dev_U) return (int)cudaErrorInvalidValue;
        if (!out_map(out ? *out : OutSpec{}, 0, gp.om)) return (int)cudaErrorInvalidValue;
        if (dtype == HQ_C128 && d.k >= 5 && gp.nsets >= (1ull << 12)) {
            if (gp.om.active) return (int)cudaErrorInvalidValue;     // in place only
            e = d.k == 5 ? launch_ztile<5>(psi, gp, dev_U, st) : launch_ztile<6>(psi, gp, dev_U, st);
        }
        else
            e = dtype == HQ_C64 ? launch_gen<float>(d.k, psi, gp, dev_U, st)
                                : launch_gen<double>(d.k, psi, gp, dev_U, st);
    }
    if (launches) ++*launches;
    return (int)e;
}

bool apply_needs_dev_U(int dtype, const ApplyDesc &d) {
    RegParams rp;
    int VEC, T0, KL;
    return !plan_reg(dtype, d, rp, VEC, T0, KL);
}

// ------------------------------------------------------------------ small states: whole circuit in shared memory
// For n_local <= 12 (c64) / 11 (c128) the whole shard fits in shared memory
// twice (64 KB), so one CTA runs every pass of a compiled circuit with the
// state resident: out[x] = sum_c U[r(x)][c] in[base(x) | off[c]] per op,
// ping-ponging between two shared buffers, one HBM read and one write in
// total.  The launch-bound small-n case then costs one launch instead of one
// per pass (CUDA graph replay was ~16 us per pass at 12 qubits).
template <typename R>
__global__ void __launch_bounds__(1024, 1)
circuit_smem(typename C2<R>::T *__restrict__ psi, int nl, const SmemOp *__restrict__ ops, int nops,
             const typename C2<R>::T *__restrict__ mats) {
    using V = typename C2<R>::T;
    extern __shared__ __align__(16) unsigned char zbuf[];
    const int N = 1 << nl;
    V *a = reinterpret_cast<V *>(zbuf);
    V *b = a + N;
    V *Ut = b + N;                                    // U^T of the current op: Ut[c * D + r]
    int *offs = reinterpret_cast<int *>(Ut + 64 * 64);
    for (int i = threadIdx.x; i < N; i += blockDim.x) a[i] = psi[i];
    for (int o = 0; o < nops; ++o) {
        const SmemOp op = ops[o];
        const int K = op.k, D = 1 << K;
        const V *U = mats + op.uoff;
        __syncthreads();                              // previous op done with Ut / offs / a
        for (int i = threadIdx.x; i < D * D; i += blockDim.x) Ut[(i % D) * D + i / D] = U[i];
        for (int c = threadIdx.x; c < D; c += blockDim.x) {
            int off = 0;
            for (int i = 0; i < K; ++i) off |= ((c >> i) & 1) << op.p[i];
            offs[c] = off;
        }
        __syncthreads();
        // output j = set * D + r: lanes run over r, so the inputs of a set are
        // warp broadcasts and U^T columns are consecutive
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
            const int r = j & (D - 1);
            int base = j >> K;
            for (int i = 0; i < K; ++i) {
                const int s = op.p[i];
                base = ((base >> s) << (s + 1)) | (base & ((1 << s) - 1));
            }
            R re = 0, im = 0;
            for (int c = 0; c < D; ++c) {
                const V u = Ut[c * D + r];
                const V v = a[base | offs[c]];
                re = fma(u.x, v.x, re);
                re = fma(-u.y, v.y, re);
                im = fma(u.x, v.y, im);
                im = fma(u.y, v.x, im);
            }
            V y;
            y.x = re;
            y.y = im;
            b[base | offs[r]] = y;
        }
        V *t = a;
        a = b;
        b = t;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) psi[i] = a[i];
}

int launch_circuit_smem(int dtype, void *psi, int nl, const SmemOp *dev_ops, int nops, const void *dev_mats,
                        void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t es = dtype == HQ_C64 ? 8 : 16;
    const size_t smem = (2 * es << nl) + es * 64 * 64 + 64 * sizeof(int);
    const int threads = nl >= 10 ? 1024 : (1 << nl) < 32 ? 32 : (1 << nl);
    if (dtype == HQ_C64) {
        static std::atomic<uint64_t> attr{0};
        cudaError_t e = smem_attr_once(circuit_smem<float>, (int)((2 * 8 << SMEM_CIRCUIT_MAX_NL_C64) + 8 * 64 * 64 + 256), attr);
        if (e != cudaSuccess) return (int)e;
        circuit_smem<float><<<1, threads, smem, st>>>((float2 *)psi, nl, dev_ops, nops, (const float2 *)dev_mats);
    } else {
        static std::atomic<uint64_t> attr{0};
        cudaError_t e = smem_attr_once(circuit_smem<double>, (int)((2 * 16 << SMEM_CIRCUIT_MAX_NL_C128) + 16 * 64 * 64 + 256), attr);
        if (e != cudaSuccess) return (int)e;
        circuit_smem<double><<<1, threads, smem, st>>>((double2 *)psi, nl, dev_ops, nops, (const double2 *)dev_mats);
    }
    return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ small kernels

template <typename V>
__global__ void set_one_kernel(V *psi, int64_t idx) {
    V one;
    one.x = 1;
    one.y = 0;
    psi[idx] = one;
}

int launch_init_basis(int dtype, void *psi, uint64_t n_amps, int64_t idx, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t es = dtype == HQ_C64 ? 8 : 16;
    cudaError_t e = cudaMemsetAsync(psi, 0, es * n_amps, st);
    if (e != cudaSuccess) return (int)e;
    if (idx >= 0) {
        if (dtype == HQ_C64) set_one_kernel<float2><<<1, 1, 0, st>>>((float2 *)psi, idx);
        else set_one_kernel<double2><<<1, 1, 0, st>>>((double2 *)psi, idx);
        e = cudaGetLastError();
    }
    return (int)e;
}

// Sum of |psi_i|^2 in fp64 per block (deterministic: fixed block count and
// order, host sum of the partials).  16-byte loads (two complex64 amplitudes
// or one complex128), four independent loads in flight per thread per
// iteration: a read-only stream at ~6.5 TB/s (one 8-byte load per iteration
// read 34q at 4.8 TB/s).
template <typename V>
__global__ void __launch_bounds__(256) norm_partial_kernel(const V *__restrict__ psi, uint64_t n,
                                                           double *__restrict__ part) {
    constexpr int PER = sizeof(V) == 8 ? 2 : 1;          // amplitudes per 16-byte load
    const uint64_t nv = n / PER;                          // 16-byte vectors
    const float4 *v4 = reinterpret_cast<const float4 *>(psi);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    auto add = [&](const float4 &w) {
        if constexpr (PER == 2) {
            acc += (double)w.x * (double)w.x + (double)w.y * (double)w.y;
            acc += (double)w.z * (double)w.z + (double)w.w * (double)w.w;
        } else {
            const double2 d = *reinterpret_cast<const double2 *>(&w);
            acc += d.x * d.x + d.y * d.y;
        }
    };
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nv; i += 4 * stride) {
        const float4 a = __ldcs(v4 + i), b = __ldcs(v4 + i + stride), c = __ldcs(v4 + i + 2 * stride),
                     d = __ldcs(v4 + i + 3 * stride);
        add(a);
        add(b);
        add(c);
        add(d);
    }
    for (; i < nv; i += stride) add(__ldcs(v4 + i));
    if (PER == 2 && (n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {   // odd count (n < 2 amplitudes)
        const V t = psi[n - 1];
        acc += (double)t.x * (double)t.x + (double)t.y * (double)t.y;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

int launch_norm_partials(int dtype, const void *psi, uint64_t n_amps, double *dev_partial,
                         int max_blocks, void *stream, int *nblocks_out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t nv = dtype == HQ_C64 ? n_amps / 2 : n_amps;
    uint64_t blocks = (nv + 4 * 256 - 1) / (4 * 256);
    if (blocks > (uint64_t)max_blocks) blocks = max_blocks;
    if (blocks == 0) blocks = 1;
    if (dtype == HQ_C64)
        norm_partial_kernel<float2><<<(unsigned)blocks, 256, 0, st>>>((const float2 *)psi, n_amps, dev_partial);
    else
        norm_partial_kernel<double2><<<(unsigned)blocks, 256, 0, st>>>((const double2 *)psi, n_amps, dev_partial);
    *nblocks_out = (int)blocks;
    return (int)cudaGetLastError();
}

struct PermParams {
    int npairs;
    int a[6];
    int b[6];
};

template <typename V>
__global__ void permute_kernel(const V *__restrict__ src, V *__restrict__ dst, uint64_t n,
                               const __grid_constant__ PermParams P) {
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t y = x;
        for (int i = 0; i < P.npairs; ++i) {
            const uint64_t ba = (x >> P.a[i]) & 1, bb = (x >> P.b[i]) & 1;
            y &= ~((1ull << P.a[i]) | (1ull << P.b[i]));
            y |= (ba << P.b[i]) | (bb << P.a[i]);
        }
        dst[y] = src[x];
    }
}

int launch_permute(int dtype, const void *src, void *dst, uint64_t n_amps, int npairs, const int *a,
                   const int *b, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    PermParams P;
    P.npairs = npairs;
    for (int i = 0; i < npairs && i < 6; ++i) { P.a[i] = a[i]; P.b[i] = b[i]; }
    uint64_t blocks = (n_amps + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    if (dtype == HQ_C64)
        permute_kernel<float2><<<(unsigned)blocks, 256, 0, st>>>((const float2 *)src, (float2 *)dst, n_amps, P);
    else
        permute_kernel<double2><<<(unsigned)blocks, 256, 0, st>>>((const double2 *)src, (double2 *)dst, n_amps, P);
    return (int)cudaGetLastError();
}

struct MapParams {
    int bitmap[64];
    int n, n_local, rank;
};

template <typename V, bool GATHER>
__global__ void gather_scatter_kernel(V *psi, V *buf, uint64_t first, uint64_t count,
                                      const __grid_constant__ MapParams P) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = first + j;
        uint64_t phys = 0;
        for (int b = 0; b < P.n; ++b) phys |= ((i >> b) & 1) << P.bitmap[b];
        if ((int)(phys >> P.n_local) != P.rank) continue;
        const uint64_t off = phys & ((1ull << P.n_local) - 1);
        if (GATHER) buf[j] = psi[off];
        else psi[off] = buf[j];
    }
}

static int launch_gs(bool gather, int dtype, void *psi, void *buf, uint64_t first, uint64_t count,
                     int n, int n_local, const int *bitmap, int my_rank, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    MapParams P;
    for (int b = 0; b < n; ++b) P.bitmap[b] = bitmap[b];
    P.n = n;
    P.n_local = n_local;
    P.rank = my_rank;
    uint64_t blocks = (count + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    if (blocks == 0) return 0;
    if (dtype == HQ_C64) {
        if (gather) gather_scatter_kernel<float2, true><<<(unsigned)blocks, 256, 0, st>>>((float2 *)psi, (float2 *)buf, first, count, P);
        else gather_scatter_kernel<float2, false><<<(unsigned)blocks, 256, 0, st>>>((float2 *)psi, (float2 *)buf, first, count, P);
    } else {
        if (gather) gather_scatter_kernel<double2, true><<<(unsigned)blocks, 256, 0, st>>>((double2 *)psi, (double2 *)buf, first, count, P);
        else gather_scatter_kernel<double2, false><<<(unsigned)blocks, 256, 0, st>>>((double2 *)psi, (double2 *)buf, first, count, P);
    }
    return (int)cudaGetLastError();
}

int launch_gather(int dtype, const void *psi, void *dst, uint64_t first, uint64_t count, int n,
                  int n_local, const int *bitmap, int my_rank, void *stream) {
    return launch_gs(true, dtype, const_cast<void *>(psi), dst, first, count, n, n_local, bitmap, my_rank, stream);
}

int launch_scatter(int dtype, void *psi, const void *src, uint64_t first, uint64_t count, int n,
                   int n_local, const int *bitmap, int my_rank, void *stream) {
    return launch_gs(false, dtype, psi, const_cast<void *>(src), first, count, n, n_local, bitmap, my_rank, stream);
}

}  // namespace hq
