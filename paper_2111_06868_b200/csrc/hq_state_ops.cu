// State preparation and measurement kernels:
// token product states, projection
// and Born probabilities for measurement.
//
// All masks are PHYSICAL bit masks of the local index; the runtime maps
// logical qubits through pi and handles the rank (global) bits on the host.
// Each kernel is one streaming pass over the shard: init writes 8/16 B per
// amplitude, project reads+writes, probabilities reads.
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <type_traits>

#include "hq_internal.h"

namespace hq {

namespace {

template <typename V>
__global__ void __launch_bounds__(256) init_tokens_kernel(V *__restrict__ psi, uint64_t n_amps,
                                                          uint64_t fix_mask, uint64_t fix_val,
                                                          uint64_t minus_mask, double mag) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_amps;
         i += (uint64_t)gridDim.x * blockDim.x) {
        V v;
        v.y = 0;
        if ((i & fix_mask) != fix_val) {
            v.x = 0;
        } else {
            const int neg = __popcll(i & minus_mask) & 1;
            v.x = (decltype(v.x))(neg ? -mag : mag);
        }
        psi[i] = v;
    }
}

// Zero the amplitudes outside (i & mask) == val and sum |psi|^2 of the kept
// ones in fp64 per block (keep_all: keep everything).  16-byte vectors (two
// complex64 amplitudes or one complex128), four per thread per iteration
// (round 1's one 8-byte element per iteration ran at ~1 TB/s).
template <typename V>
__global__ void __launch_bounds__(256) project_kernel(V *__restrict__ psi, uint64_t n_amps,
                                                      uint64_t mask, uint64_t val, int keep_all,
                                                      double *__restrict__ part) {
    constexpr int PER = sizeof(V) == 8 ? 2 : 1;
    float4 *v4 = reinterpret_cast<float4 *>(psi);
    const uint64_t nv = n_amps / PER, S = (uint64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    auto kept = [&](uint64_t i) { return keep_all || (i & mask) == val; };
    // vectors whose amplitudes are all projected out are written (zeros)
    // without being read; the others are read, summed, and written only when
    // one of their two amplitudes goes
    auto dead = [&](uint64_t j) { return PER == 2 ? !kept(2 * j) && !kept(2 * j + 1) : !kept(j); };
    auto sum = [&](uint64_t j, float4 &w) -> bool {
        if constexpr (PER == 2) {
            bool dirty = false;
            if (kept(2 * j)) acc += (double)w.x * w.x + (double)w.y * w.y;
            else { w.x = w.y = 0.f; dirty = true; }
            if (kept(2 * j + 1)) acc += (double)w.z * w.z + (double)w.w * w.w;
            else { w.z = w.w = 0.f; dirty = true; }
            return dirty;
        } else {
            const double2 d = *reinterpret_cast<const double2 *>(&w);
            acc += d.x * d.x + d.y * d.y;
            return false;
        }
    };
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; j + 3 * S < nv; j += 4 * S) {
        float4 w[4];
        bool d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {            // all loads first
            d[u] = dead(j + u * S);
            if (!d[u]) w[u] = v4[j + u * S];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (d[u]) v4[j + u * S] = zero;
            else if (sum(j + u * S, w[u])) v4[j + u * S] = w[u];
        }
    }
    for (; j < nv; j += S) {
        if (dead(j)) {
            v4[j] = zero;
            continue;
        }
        float4 w = v4[j];
        if (sum(j, w)) v4[j] = w;
    }
    if (PER == 2 && (n_amps & 1) && blockIdx.x == 0 && threadIdx.x == 0) {   // a lone amplitude (n = 0)
        const uint64_t i = n_amps - 1;
        if (keep_all || (i & mask) == val) acc += (double)psi[i].x * psi[i].x + (double)psi[i].y * psi[i].y;
        else psi[i].x = psi[i].y = 0;
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

// psi *= s: 16-byte vectors, four per thread per iteration; complex64
// scales in FP32 (the factor's rounding is below the storage precision)
template <typename V>
__global__ void __launch_bounds__(256) scale_kernel(V *__restrict__ psi, uint64_t n_amps, double s) {
    constexpr int PER = sizeof(V) == 8 ? 2 : 1;
    float4 *v4 = reinterpret_cast<float4 *>(psi);
    const uint64_t nv = n_amps / PER, S = (uint64_t)gridDim.x * blockDim.x;
    const float sf = (float)s;
    auto scale = [&](float4 w) {
        if constexpr (PER == 2) {
            w.x *= sf;
            w.y *= sf;
            w.z *= sf;
            w.w *= sf;
        } else {
            double2 d = *reinterpret_cast<double2 *>(&w);
            d.x *= s;
            d.y *= s;
            w = *reinterpret_cast<float4 *>(&d);
        }
        return w;
    };
    uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; j + 3 * S < nv; j += 4 * S) {
        float4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = v4[j + u * S];          // all loads first
#pragma unroll
        for (int u = 0; u < 4; ++u) v4[j + u * S] = scale(w[u]);
    }
    for (; j < nv; j += S) v4[j] = scale(v4[j]);
    if (PER == 2 && (n_amps & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        psi[n_amps - 1].x *= sf;
        psi[n_amps - 1].y *= sf;
    }
}

template <typename V>
__global__ void __launch_bounds__(256) scale_complex_kernel(V *__restrict__ psi, uint64_t n_amps, double re,
                                                            double im) {
    using T = decltype(V::x);
    const T sr = (T)re, si = (T)im;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_amps;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const V v = psi[i];
        V o;
        o.x = sr * v.x - si * v.y;
        o.y = sr * v.y + si * v.x;
        psi[i] = o;
    }
}

// hist[c][y] = sum of |psi_i|^2 over chunk c of the amplitudes whose
// outcome bits (the bits of i at positions pos[0..nq), pos[0] = MSB of y)
// equal y.  Outcome bits at positions >= PROB_LOW are "high": block (c, yh)
// walks only the amplitudes with high outcome bits yh (i = r with zeros
// inserted at the high positions, OR yh's bits), so reads stay contiguous;
// the (at most PROB_LOW) low outcome bits vary inside a thread's reads and
// select one of 2^nlow register accumulators.  No atomics (round 1's
// per-amplitude shared-memory atomics serialised on the few bins of a
// 1-qubit measurement: 80 GB/s at 32q).
constexpr int PROB_LOW = 4;

template <typename V, int NLOW>
__global__ void __launch_bounds__(256) prob_kernel(const V *__restrict__ psi, uint64_t n_amps,
                                                   const __grid_constant__ ProbParams P,
                                                   double *__restrict__ hist) {
    constexpr int NBL = 1 << NLOW;
    const int yh = blockIdx.y;
    // split the outcome bits: low (position < PROB_LOW) and high; y = bits
    // pos[0..nq) with pos[0] the MSB
    int hpos[16], nh = 0, lpos[PROB_LOW], lj[PROB_LOW], hj[16];
    int nl = 0;
    for (int j = 0; j < P.nq; ++j) {
        if (P.pos[j] < PROB_LOW) { lpos[nl] = P.pos[j]; lj[nl] = j; ++nl; }
        else { hpos[nh] = P.pos[j]; hj[nh] = j; ++nh; }
    }
    // high bits of this block's outcome (yh: bit nh-1-t <-> hpos[t]), and the
    // ascending high positions for zero insertion
    uint64_t yb = 0;
    int spos[16];
    for (int t = 0; t < nh; ++t) {
        if ((yh >> (nh - 1 - t)) & 1) yb |= 1ull << hpos[t];
        spos[t] = hpos[t];
    }
    for (int x = 1; x < nh; ++x)
        for (int z = x; z > 0 && spos[z - 1] > spos[z]; --z) {
            const int tmp = spos[z];
            spos[z] = spos[z - 1];
            spos[z - 1] = tmp;
        }
    const uint64_t nrest = n_amps >> nh;
    double acc[NBL];
#pragma unroll
    for (int b = 0; b < NBL; ++b) acc[b] = 0.0;
    auto index = [&](uint64_t r) {
        for (int t = 0; t < nh; ++t) {
            const int sp = spos[t];
            r = ((r >> sp) << (sp + 1)) | (r & ((1ull << sp) - 1));
        }
        return r | yb;
    };
    auto add = [&](uint64_t i, const V &v) {
        const double p = (double)v.x * (double)v.x + (double)v.y * (double)v.y;
        int lb = 0;
        for (int t = 0; t < nl; ++t) lb |= (int)((i >> lpos[t]) & 1) << t;
#pragma unroll
        for (int b = 0; b < NBL; ++b) acc[b] += b == lb ? p : 0.0;
    };
    // four independent loads in flight per thread (a single load per
    // iteration left the pass latency-bound)
    const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
    uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; r + 3 * S < nrest; r += 4 * S) {
        const uint64_t i0 = index(r), i1 = index(r + S), i2 = index(r + 2 * S), i3 = index(r + 3 * S);
        const V v0 = __ldcs(psi + i0), v1 = __ldcs(psi + i1), v2 = __ldcs(psi + i2), v3 = __ldcs(psi + i3);
        add(i0, v0);
        add(i1, v1);
        add(i2, v2);
        add(i3, v3);
    }
    for (; r < nrest; r += S) {
        const uint64_t i0 = index(r);
        add(i0, psi[i0]);
    }
    __shared__ double red[8][NBL];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int b = 0; b < NBL; ++b) {
        double a = acc[b];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[warp][b] = a;
    }
    __syncthreads();
    if (threadIdx.x < (1 << nl)) {
        const int lb = threadIdx.x;
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][lb];
        int y = 0;                                   // full outcome from (yh, lb)
        for (int q = 0; q < nh; ++q)
            if ((yh >> (nh - 1 - q)) & 1) y |= 1 << (P.nq - 1 - hj[q]);
        for (int q = 0; q < nl; ++q)
            if ((lb >> q) & 1) y |= 1 << (P.nq - 1 - lj[q]);
        hist[(size_t)blockIdx.x * (1 << P.nq) + y] = t;
    }
}

unsigned grid_for(uint64_t n) {
    uint64_t b = (n + 255) / 256;
    if (b > 148ull * 8) b = 148ull * 8;
    return (unsigned)(b ? b : 1);
}

// Sum of the diagonal of an N-qubit density matrix stored as the 2N-qubit
// vec(rho): logical index (i, i) = i * 2^N + i, mapped to physical bits by
// bitmap (logical bit -> physical bit); only amplitudes of this rank count.
template <typename V>
__global__ void __launch_bounds__(256) dm_trace_kernel(const V *__restrict__ psi, int N, int n_local,
                                                       int rank, const __grid_constant__ DmParams P,
                                                       double2 *__restrict__ part) {
    double re = 0.0, im = 0.0;
    const uint64_t cnt = 1ull << N;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t li = (i << N) | i;
        uint64_t phys = 0;
        for (int b = 0; b < 2 * N; ++b) phys |= ((li >> b) & 1) << P.bitmap[b];
        if ((int)(phys >> n_local) != rank) continue;
        const V v = psi[phys & ((1ull << n_local) - 1)];
        re += (double)v.x;
        im += (double)v.y;
    }
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    __shared__ double2 red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_double2(re, im);
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 t = make_double2(0.0, 0.0);
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t.x += red[w].x; t.y += red[w].y; }
        part[blockIdx.x] = t;
    }
}

// rho[a][b] = sum over gather sets of psi_a conj(psi_b) (upper triangle,
// fp64 accumulation); one gather set per thread per step, consecutive
// threads on consecutive sets (coalesced unless bit 0 is a target).
// Batched form (row f3, shots along the top physical bits): blockIdx.y is
// the shot, whose amplitudes are [shot * shot_amps, (shot + 1) * shot_amps);
// partials go to part[shot][block][2E].  shot_amps = 0: one unbatched state.
template <typename V, int K>
__global__ void __launch_bounds__(256) reduced_dm_kernel(const V *__restrict__ psi, uint64_t nsets,
                                                         const __grid_constant__ RdmParams P,
                                                         double *__restrict__ part, uint64_t shot_amps) {
    constexpr int D = 1 << K, E = D * (D + 1) / 2;
    psi += (uint64_t)blockIdx.y * shot_amps;
    part += (size_t)blockIdx.y * gridDim.x * 2 * E;
    double acc[2 * E];
#pragma unroll
    for (int e = 0; e < 2 * E; ++e) acc[e] = 0.0;
    auto base_of = [&](uint64_t o) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int s = P.pos[i];
            o = ((o >> s) << (s + 1)) | (o & ((1ull << s) - 1));
        }
        return o;
    };
    auto accumulate = [&](const V (&v)[D]) {
        int e = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b, ++e) {
                const double ra = v[a].x, ia = v[a].y, rb = v[b].x, ib = v[b].y;
                acc[2 * e] += ra * rb + ia * ib;
                acc[2 * e + 1] += ia * rb - ra * ib;
            }
    };
    // two gather sets per iteration: 2 * 2^K independent loads in flight
    const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
    uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; o + S < nsets; o += 2 * S) {
        const uint64_t b0 = base_of(o), b1 = base_of(o + S);
        V v0[D], v1[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            v0[a] = __ldcs(psi + b0 + P.off[a]);
            v1[a] = __ldcs(psi + b1 + P.off[a]);
        }
        accumulate(v0);
        accumulate(v1);
    }
    if (o < nsets) {
        const uint64_t b0 = base_of(o);
        V v0[D];
#pragma unroll
        for (int a = 0; a < D; ++a) v0[a] = psi[b0 + P.off[a]];
        accumulate(v0);
    }
    __shared__ double red[8][2 * E];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int e = 0; e < 2 * E; ++e) {
        double x = acc[e];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (l == 0) red[w][e] = x;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * E; e += blockDim.x) {
        double t = 0.0;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) t += red[j][e];
        part[(size_t)blockIdx.x * 2 * E + e] = t;
    }
}

template <typename V>
int reduced_dm_dispatch(const V *psi, uint64_t nsets, const RdmParams &P, double *part, dim3 g,
                        cudaStream_t st, uint64_t shot_amps) {
    if (P.k == 1) reduced_dm_kernel<V, 1><<<g, 256, 0, st>>>(psi, nsets, P, part, shot_amps);
    else if (P.k == 2) reduced_dm_kernel<V, 2><<<g, 256, 0, st>>>(psi, nsets, P, part, shot_amps);
    else reduced_dm_kernel<V, 3><<<g, 256, 0, st>>>(psi, nsets, P, part, shot_amps);
    return (int)cudaGetLastError();
}

// psi <- M_shot psi on the k <= 3 targets, M_shot = mats[shot] (row-major
// D x D in the state dtype, canonical target order), shot = physical index
// >> sys_bits.  One thread per gather set; a block's sets share a shot (the
// matrices stay in L1).
template <typename V, int K>
__global__ void __launch_bounds__(256) apply_batched_kernel(V *__restrict__ psi, uint64_t nsets,
                                                            const __grid_constant__ RdmParams P,
                                                            const V *__restrict__ mats, int sys_bits) {
    constexpr int D = 1 << K;
    using T = decltype(V::x);
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < nsets;
         o += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = o;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int s = P.pos[i];
            base = ((base >> s) << (s + 1)) | (base & ((1ull << s) - 1));
        }
        const V *M = mats + (size_t)(base >> sys_bits) * D * D;
        V x[D];
#pragma unroll
        for (int c = 0; c < D; ++c) x[c] = psi[base + P.off[c]];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            T re = 0, im = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const V m = M[r * D + c];
                re += m.x * x[c].x - m.y * x[c].y;
                im += m.x * x[c].y + m.y * x[c].x;
            }
            V y;
            y.x = re;
            y.y = im;
            psi[base + P.off[r]] = y;
        }
    }
}

}  // namespace

int launch_reduced_dm(int dtype, const void *psi, uint64_t n_amps, const RdmParams &P, double *dev_part,
                      void *stream, int *nblocks_out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t nsets = n_amps >> P.k;
    unsigned g = grid_for(nsets);
    if (g > (unsigned)RDM_MAX_BLOCKS) g = RDM_MAX_BLOCKS;
    *nblocks_out = (int)g;
    if (dtype == HQ_C64) return reduced_dm_dispatch((const float2 *)psi, nsets, P, dev_part, dim3(g), st, 0);
    return reduced_dm_dispatch((const double2 *)psi, nsets, P, dev_part, dim3(g), st, 0);
}

int launch_reduced_dm_batched(int dtype, const void *psi, uint64_t shot_amps, int nshots, const RdmParams &P,
                              double *dev_part, int max_parts, void *stream, int *nblocks_out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t nsets = shot_amps >> P.k;
    unsigned g = grid_for(nsets);
    const unsigned cap = (unsigned)std::max(1, max_parts / nshots);
    if (g > cap) g = cap;
    if (g > 64) g = 64;
    *nblocks_out = (int)g;
    const dim3 grid(g, (unsigned)nshots);
    if (dtype == HQ_C64) return reduced_dm_dispatch((const float2 *)psi, nsets, P, dev_part, grid, st, shot_amps);
    return reduced_dm_dispatch((const double2 *)psi, nsets, P, dev_part, grid, st, shot_amps);
}

int launch_apply_batched(int dtype, void *psi, uint64_t n_amps, const RdmParams &P, const void *dev_mats,
                         int sys_bits, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t nsets = n_amps >> P.k;
    const unsigned g = grid_for(nsets);
    if (dtype == HQ_C64) {
        float2 *p = (float2 *)psi;
        const float2 *m = (const float2 *)dev_mats;
        if (P.k == 1) apply_batched_kernel<float2, 1><<<g, 256, 0, st>>>(p, nsets, P, m, sys_bits);
        else if (P.k == 2) apply_batched_kernel<float2, 2><<<g, 256, 0, st>>>(p, nsets, P, m, sys_bits);
        else apply_batched_kernel<float2, 3><<<g, 256, 0, st>>>(p, nsets, P, m, sys_bits);
    } else {
        double2 *p = (double2 *)psi;
        const double2 *m = (const double2 *)dev_mats;
        if (P.k == 1) apply_batched_kernel<double2, 1><<<g, 256, 0, st>>>(p, nsets, P, m, sys_bits);
        else if (P.k == 2) apply_batched_kernel<double2, 2><<<g, 256, 0, st>>>(p, nsets, P, m, sys_bits);
        else apply_batched_kernel<double2, 3><<<g, 256, 0, st>>>(p, nsets, P, m, sys_bits);
    }
    return (int)cudaGetLastError();
}

int launch_dm_trace(int dtype, const void *psi, int N, int n_local, int rank, const DmParams &P,
                    double2 *dev_part, int max_blocks, void *stream, int *nblocks_out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    unsigned g = grid_for(1ull << N);
    if (g > (unsigned)max_blocks) g = max_blocks;
    if (dtype == HQ_C64)
        dm_trace_kernel<float2><<<g, 256, 0, st>>>((const float2 *)psi, N, n_local, rank, P, dev_part);
    else
        dm_trace_kernel<double2><<<g, 256, 0, st>>>((const double2 *)psi, N, n_local, rank, P, dev_part);
    *nblocks_out = (int)g;
    return (int)cudaGetLastError();
}

int launch_init_tokens(int dtype, void *psi, uint64_t n_amps, uint64_t fix_mask, uint64_t fix_val,
                       uint64_t minus_mask, double mag, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == HQ_C64)
        init_tokens_kernel<float2><<<grid_for(n_amps), 256, 0, st>>>((float2 *)psi, n_amps, fix_mask,
                                                                     fix_val, minus_mask, mag);
    else
        init_tokens_kernel<double2><<<grid_for(n_amps), 256, 0, st>>>((double2 *)psi, n_amps, fix_mask,
                                                                      fix_val, minus_mask, mag);
    return (int)cudaGetLastError();
}

int launch_project(int dtype, void *psi, uint64_t n_amps, uint64_t mask, uint64_t val, int keep_all,
                   double *dev_partial, int max_blocks, void *stream, int *nblocks_out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    unsigned g = grid_for(n_amps);
    if (g > (unsigned)max_blocks) g = max_blocks;
    if (dtype == HQ_C64)
        project_kernel<float2><<<g, 256, 0, st>>>((float2 *)psi, n_amps, mask, val, keep_all, dev_partial);
    else
        project_kernel<double2><<<g, 256, 0, st>>>((double2 *)psi, n_amps, mask, val, keep_all, dev_partial);
    *nblocks_out = (int)g;
    return (int)cudaGetLastError();
}

int launch_scale(int dtype, void *psi, uint64_t n_amps, double s, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == HQ_C64) scale_kernel<float2><<<grid_for(n_amps), 256, 0, st>>>((float2 *)psi, n_amps, s);
    else scale_kernel<double2><<<grid_for(n_amps), 256, 0, st>>>((double2 *)psi, n_amps, s);
    return (int)cudaGetLastError();
}

int launch_scale_complex(int dtype, void *psi, uint64_t n_amps, double re, double im, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == HQ_C64)
        scale_complex_kernel<float2><<<grid_for(n_amps), 256, 0, st>>>((float2 *)psi, n_amps, re, im);
    else
        scale_complex_kernel<double2><<<grid_for(n_amps), 256, 0, st>>>((double2 *)psi, n_amps, re, im);
    return (int)cudaGetLastError();
}

// max_blocks: chunks per high outcome (the histogram has max_blocks << nq slots)
int launch_probabilities(int dtype, const void *psi, uint64_t n_amps, const ProbParams &P,
                         double *dev_hist, int max_blocks, void *stream, int *nblocks_out) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int nlow = 0;
    for (int j = 0; j < P.nq; ++j) nlow += P.pos[j] < PROB_LOW;
    const int nh = P.nq - nlow;
    const uint64_t nrest = n_amps >> nh;
    uint64_t gx = (nrest + 255) / 256;
    const uint64_t target = std::max<uint64_t>(1, (148ull * 8) >> nh);   // ~8 blocks per SM in all
    if (gx > target) gx = target;
    if (gx > (uint64_t)max_blocks) gx = max_blocks;
    if (gx == 0) gx = 1;
    const dim3 grid((unsigned)gx, 1u << nh);
#define HQ_PROB(NL)                                                                                  \
    do {                                                                                             \
        if (dtype == HQ_C64)                                                                         \
            prob_kernel<float2, NL><<<grid, 256, 0, st>>>((const float2 *)psi, n_amps, P, dev_hist);  \
        else                                                                                         \
            prob_kernel<double2, NL><<<grid, 256, 0, st>>>((const double2 *)psi, n_amps, P, dev_hist); \
    } while (0)
    switch (nlow) {
        case 0: HQ_PROB(0); break;
        case 1: HQ_PROB(1); break;
        case 2: HQ_PROB(2); break;
        case 3: HQ_PROB(3); break;
        default: HQ_PROB(4); break;
    }
#undef HQ_PROB
    *nblocks_out = (int)gx;
    return (int)cudaGetLastError();
}

}  // namespace hq
