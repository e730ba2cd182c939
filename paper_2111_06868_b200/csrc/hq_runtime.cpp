// C-ABI runtime: state objects, validation, the op-stream executor (apply /
// remap / permute), norm and amplitude I/O.  See include/hq.h for the
// contract of every exported function.
//
// Layout in HBM: each rank r holds physical indices
// [r 2^(n_l), (r+1) 2^(n_l)) of the 2^n amplitudes as one contiguous array of
// interleaved complex (float2 for HQ_C64, double2 for HQ_C128), 256-byte
// aligned.  The logical->physical qubit map pi starts as q -> n-1-q (so the
// physical index equals the logical index, reading C1) and changes only when
// the distributed schedule remaps global qubits.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <chrono>
#include <thread>
#include <vector>

#include "hq_internal.h"

namespace hq {

static thread_local std::string g_err;

hq_status set_error(hq_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

void clear_error() { g_err.clear(); }

}  // namespace hq

using namespace hq;

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return set_error(_e == cudaErrorMemoryAllocation ? HQ_ERR_OOM : HQ_ERR_CUDA, \
                             "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__,  \
                             __LINE__);                                                 \
    } while (0)

#define NCCL_TRY(expr)                                                                   \
    do {                                                                                 \
        ncclResult_t _r = (expr);                                                        \
        if (_r != ncclSuccess)                                                           \
            return set_error(HQ_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(_r), \
                             __FILE__, __LINE__);                                        \
    } while (0)

enum Mode { MODE_SINGLE = 0, MODE_RANK = 1, MODE_VIRTUAL = 2, MODE_MULTI = 3 };

// Device staging area for gate matrices (generic kernels read U from HBM).
struct Arena {
    char *dev = nullptr;
    char *host = nullptr;   // pinned
    size_t cap = 0, off = 0;
};

struct Shard {
    int device = 0;
    int rank = 0;
    void *psi = nullptr;
    void *buf = nullptr;          // receive / permute scratch (G > 1)
    bool own_psi = true;
    bool own_buf = true;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    ncclComm_t comm = nullptr;
    double *d_part = nullptr;     // norm partials
    double *h_part = nullptr;     // pinned
    double *d_red = nullptr;      // reduced-density-matrix partials (lazy)
    double *h_red = nullptr;      // pinned
    size_t red_cap = 0;           // doubles in d_red / h_red
    double *d_ar = nullptr;       // all-reduce scratch (rank mode), AR_CAP doubles
    double *h_ar = nullptr;       // pinned
    Arena arena;
    // profiling events, created on this shard's device (an event must be
    // recorded on a stream of the device it was created on)
    std::vector<cudaEvent_t> ev_pool;
};

// Synchronise a shard's stream.  With an NCCL communicator (rank mode, or one
// process driving several devices) the wait polls ncclCommGetAsyncError, so a
// peer that died or a broken link surfaces as HQ_ERR_NCCL -- the communicator
// is aborted -- instead of a host thread blocked forever in
// cudaStreamSynchronize behind a collective that never completes (SURVEY §5
// "failure detection").  Without one it is cudaStreamSynchronize.
static hq_status sync_shard(Shard &s) {
    if (!s.comm) {
        CUDA_TRY(cudaStreamSynchronize(s.stream));
        return HQ_OK;
    }
    for (unsigned spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s.stream);
        if (q == cudaSuccess) return HQ_OK;
        if (q != cudaErrorNotReady)
            return set_error(q == cudaErrorMemoryAllocation ? HQ_ERR_OOM : HQ_ERR_CUDA, "stream: %s",
                             cudaGetErrorString(q));
        ncclResult_t ar = ncclSuccess;
        const ncclResult_t r = ncclCommGetAsyncError(s.comm, &ar);
        if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
            ncclCommAbort(s.comm);
            s.comm = nullptr;
            return set_error(HQ_ERR_NCCL, "NCCL asynchronous error (communicator aborted): %s",
                             ncclGetErrorString(r != ncclSuccess ? r : ar));
        }
        if (spin >= 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}
#define SYNC_TRY(shard)                             \
    do {                                            \
        const hq_status _rc = sync_shard(shard);    \
        if (_rc) return _rc;                        \
    } while (0)

constexpr int AR_CAP = 1024;      // largest host all-reduce: 2^10 outcome probabilities

struct ProfEvent {
    cudaEvent_t a, b;
    uint64_t bytes;
    int path;
    int shard;
};

struct ProfAcc {
    uint64_t count = 0;
    double total = 0, max = 0;
    uint64_t bytes = 0;
};

struct hq_state {
    int n = 0, m = 0, nl = 0;
    hq_dtype dtype = HQ_C64;
    size_t es = 8;
    int world = 1;
    int mode = MODE_SINGLE;
    std::vector<Shard> sh;
    std::vector<int> pi;          // logical qubit -> physical bit
    std::vector<int> pi_init;     // layout restored by hq_state_init_basis
    // Rigorous upper bound on ||psi||_2 (hence on every |amplitude|), kept
    // through every pass from per-gate spectral-norm bounds; the FP16 tensor-
    // core path scales the state into range with it.  < 0: unknown.
    double amp_bound = -1.0;
    hq_stats stats{};
    bool profiling = false;
    std::vector<ProfEvent> prof;  // pending
    ProfAcc acc[3];               // per kernel family (PATH_REG, PATH_GEN, PATH_TC)
    // fused remap (row f1): the apply pass before a packed
    // remap writes every element straight into its destination rank's
    // exchange buffer (peer memory over NVLink), so the exchange needs no
    // separate transfer.  p2p: every peer's buffers are addressable.
    int remap_mode = HQ_REMAP_FUSED | HQ_REMAP_GATHER;
    bool p2p = false;
    std::vector<void *> peer_base[2];   // rank mode: IPC-mapped original [psi, buf] of every rank
    uint64_t swaps = 0;                 // psi <-> buf exchanges so far (the same on every rank)
    int *d_bar = nullptr;               // rank mode: one-int all-reduce used as a stream barrier
    std::vector<cudaEvent_t> bar_ev;    // multi-device mode: one event per shard for barriers
};

struct Fold {
    int consumed = 0;
    bool fused = false;
    bool with_perm = false;
    const Op *rem = nullptr;
    OutSpec tmpl;
};

struct hq_circuit {
    hq_state *owner = nullptr;
    std::vector<int> pi_start, pi_end;
    std::vector<Op> ops;
    std::vector<long long> op_uoff;        // per APPLY op: byte offset of its payload (-1: none)
    std::vector<struct Prep> prep;         // per op (APPLY)
    // row f1: APPLY ops with global targets, one Prep (and payload offset)
    // per shard; empty for the others
    std::vector<std::vector<struct Prep>> cprep;
    std::vector<std::vector<long long>> cuoff;
    std::vector<double> cgnorm;            // spectral bound of the whole U
    std::vector<Fold> fold;                // per APPLY op: ops folded into it (apply+pack, fused remap)
    std::vector<char *> dev_U;             // per shard: all payloads
    // small single-shard states: the whole op stream in one shared-memory CTA
    SmemOp *small_ops = nullptr;
    void *small_mats = nullptr;
    int small_nops = 0;
    int small_dev = 0;
    std::vector<int> dev_of;               // per shard: its device (destroy must not read the state)
    uint64_t passes = 0, remaps = 0, permutes = 0, packs = 0, gathers = 0;
    // CUDA graph of the whole op stream (single-shard states, profiling off):
    // captured on the first run, replayed while the capture key matches.
    cudaGraphExec_t graph = nullptr;
    std::vector<int> graph_ea;             // TC input-scale exponents baked into the graph
    cudaStream_t graph_stream = nullptr;
    void *graph_psi = nullptr;
    uint64_t graph_launches = 0;
};

// ------------------------------------------------------------------ helpers

static int ilog2(int x) {
    int l = 0;
    while ((1 << l) < x) ++l;
    return l;
}

// Host<->device copy on a shard stream that also counts the bytes in the
// state's statistics (the bench's e2e byte counts come from here).
static cudaError_t copy_async(hq_stats &stats, void *dst, const void *src, size_t bytes, cudaMemcpyKind kind,
                              cudaStream_t stream) {
    if (kind == cudaMemcpyHostToDevice) stats.h2d_bytes += bytes;
    if (kind == cudaMemcpyDeviceToHost) stats.d2h_bytes += bytes;
    return cudaMemcpyAsync(dst, src, bytes, kind, stream);
}

static hq_status arena_init(Shard &s, size_t cap) {
    CUDA_TRY(cudaSetDevice(s.device));
    CUDA_TRY(cudaMalloc((void **)&s.arena.dev, cap));
    CUDA_TRY(cudaMallocHost((void **)&s.arena.host, cap));
    s.arena.cap = cap;
    s.arena.off = 0;
    return HQ_OK;
}

// Copy `bytes` of host data to the device arena (stream-ordered); returns the
// device pointer.  When full, synchronise the stream and restart.
static hq_status arena_push(hq_state *st, Shard &s, const void *src, size_t bytes, void **dev_out) {
    const size_t a = (bytes + 255) & ~(size_t)255;
    if (a > s.arena.cap) return set_error(HQ_ERR_ARG, "matrix larger than staging arena");
    if (s.arena.off + a > s.arena.cap) {
        SYNC_TRY(s);
        s.arena.off = 0;
    }
    memcpy(s.arena.host + s.arena.off, src, bytes);
    CUDA_TRY(copy_async(st->stats, s.arena.dev + s.arena.off, s.arena.host + s.arena.off, bytes,
                        cudaMemcpyHostToDevice, s.stream));
    *dev_out = s.arena.dev + s.arena.off;
    s.arena.off += a;
    return HQ_OK;
}

static hq_status shard_alloc(hq_state *st, Shard &s, bool need_buf, bool make_stream) {
    CUDA_TRY(cudaSetDevice(s.device));
    const size_t bytes = st->es << st->nl;
    if (make_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        s.own_stream = true;
    }
    if (!s.psi) {
        cudaError_t e = cudaMalloc(&s.psi, bytes);
        if (e != cudaSuccess) {
            s.psi = nullptr;
            return set_error(HQ_ERR_OOM, "cudaMalloc(%zu) for the state shard failed: %s", bytes,
                             cudaGetErrorString(e));
        }
        s.own_psi = true;
    }
    if (need_buf && !s.buf) {
        cudaError_t e = cudaMalloc(&s.buf, bytes);
        if (e != cudaSuccess) {
            s.buf = nullptr;
            return set_error(HQ_ERR_OOM, "cudaMalloc(%zu) for the exchange buffer failed: %s",
                             bytes, cudaGetErrorString(e));
        }
        s.own_buf = true;
    }
    CUDA_TRY(cudaMalloc((void **)&s.d_part, sizeof(double) * 148 * 16));
    CUDA_TRY(cudaMallocHost((void **)&s.h_part, sizeof(double) * 148 * 16));
    return arena_init(s, (size_t)64 << 20);
}

static void shard_free(Shard &s) {
    cudaSetDevice(s.device);
    // a borrowed stream may already be destroyed by its owner: only our own
    // stream is synchronised here (cudaFree below synchronises the device)
    if (s.own_stream && s.stream) cudaStreamSynchronize(s.stream);
    if (s.own_psi && s.psi) cudaFree(s.psi);
    if (s.own_buf && s.buf) cudaFree(s.buf);
    if (s.d_part) cudaFree(s.d_part);
    if (s.h_part) cudaFreeHost(s.h_part);
    if (s.d_red) cudaFree(s.d_red);
    if (s.h_red) cudaFreeHost(s.h_red);
    if (s.d_ar) cudaFree(s.d_ar);
    if (s.h_ar) cudaFreeHost(s.h_ar);
    for (auto e : s.ev_pool) cudaEventDestroy(e);
    if (s.arena.dev) cudaFree(s.arena.dev);
    if (s.arena.host) cudaFreeHost(s.arena.host);
    if (s.comm) ncclCommDestroy(s.comm);
    if (s.own_stream && s.stream) cudaStreamDestroy(s.stream);
    s = Shard{};
    cudaGetLastError();        // teardown errors must not surface in a later launch check
}

static hq_status check_device() {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0)
        return set_error(HQ_ERR_NO_DEVICE,
                         "no CUDA device visible (%s); this library has no CPU fallback",
                         e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    return HQ_OK;
}

static hq_state *new_state(int n, hq_dtype dtype, int world) {
    hq_state *st = new (std::nothrow) hq_state();
    if (!st) return nullptr;
    st->n = n;
    st->dtype = dtype;
    st->es = dtype == HQ_C64 ? 8 : 16;
    st->world = world;
    st->m = ilog2(world);
    st->nl = n - st->m;
    st->pi.resize(n);
    for (int q = 0; q < n; ++q) st->pi[q] = n - 1 - q;
    st->pi_init = st->pi;
    return st;
}

static hq_status validate_common(int n, hq_dtype dtype, int G) {
    if (n < 1 || n > 40) return set_error(HQ_ERR_ARG, "n=%d not in [1,40]", n);
    if (dtype != HQ_C64 && dtype != HQ_C128) return set_error(HQ_ERR_ARG, "bad dtype %d", (int)dtype);
    if (G < 1 || (G & (G - 1))) return set_error(HQ_ERR_NGPUS, "G=%d is not a power of two", G);
    if (G > 1 && n - ilog2(G) < 6)
        return set_error(HQ_ERR_NGPUS, "n - log2(G) = %d < 6 local qubits", n - ilog2(G));
    return HQ_OK;
}

// ------------------------------------------------------------------ peer access (fused remaps)

// Single process, several devices: enable peer access between every pair.
static void setup_p2p_multi(hq_state *st) {
    bool ok = true;
    for (auto &a : st->sh)
        for (auto &b : st->sh) {
            if (a.device == b.device) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, a.device, b.device);
            if (!can) { ok = false; continue; }
            cudaSetDevice(a.device);
            cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ok = false;
        }
    cudaGetLastError();
    st->bar_ev.assign(st->sh.size(), nullptr);
    for (size_t r = 0; r < st->sh.size(); ++r) {
        cudaSetDevice(st->sh[r].device);
        if (cudaEventCreateWithFlags(&st->bar_ev[r], cudaEventDisableTiming) != cudaSuccess) ok = false;
    }
    st->p2p = ok;
}

// One process per GPU: map every rank's two exchange buffers into this process
// with CUDA IPC (handles of the allocations holding psi and buf, all-gathered
// over NCCL).  Any failure on any rank (e.g. buffers from a VMM allocator,
// which IPC cannot export) leaves fused remaps off on every rank, and the
// remaps go through the NCCL exchange.
using GetAddrRangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
static bool alloc_base(void *p, void **base) {
    static GetAddrRangeFn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return false;
        fn = reinterpret_cast<GetAddrRangeFn>(f);
    }
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
    *base = reinterpret_cast<void *>(b);
    return true;
}

static void setup_p2p_rank(hq_state *st) {
    Shard &s = st->sh[0];
    const int W = st->world;
    struct Rec {
        cudaIpcMemHandle_t h[2];
        uint64_t off[2];
        int ok;
        int pad;
    };
    Rec mine;
    memset(&mine, 0, sizeof mine);
    mine.ok = 1;
    void *ptrs[2] = {s.psi, s.buf};
    for (int i = 0; i < 2; ++i) {
        void *base = nullptr;
        if (!alloc_base(ptrs[i], &base) || cudaIpcGetMemHandle(&mine.h[i], base) != cudaSuccess) {
            mine.ok = 0;
            continue;
        }
        mine.off[i] = (uint64_t)((char *)ptrs[i] - (char *)base);
    }
    cudaGetLastError();
    cudaSetDevice(s.device);
    Rec *d = nullptr;
    std::vector<Rec> all(W);
    bool ok = cudaMalloc((void **)&d, sizeof(Rec) * W) == cudaSuccess &&
              cudaMemcpy(d + s.rank, &mine, sizeof mine, cudaMemcpyHostToDevice) == cudaSuccess &&
              ncclAllGather(d + s.rank, d, sizeof(Rec), ncclChar, s.comm, s.stream) == ncclSuccess &&
              cudaStreamSynchronize(s.stream) == cudaSuccess &&
              cudaMemcpy(all.data(), d, sizeof(Rec) * W, cudaMemcpyDeviceToHost) == cudaSuccess;
    if (d) cudaFree(d);
    for (int r = 0; r < W && ok; ++r) ok = all[r].ok != 0;
    st->peer_base[0].assign(W, nullptr);
    st->peer_base[1].assign(W, nullptr);
    int local_ok = ok ? 1 : 0;
    for (int r = 0; r < W && local_ok; ++r) {
        if (r == s.rank) {
            st->peer_base[0][r] = s.psi;
            st->peer_base[1][r] = s.buf;
            continue;
        }
        for (int i = 0; i < 2 && local_ok; ++i) {
            void *b = nullptr;
            if (cudaIpcOpenMemHandle(&b, all[r].h[i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) local_ok = 0;
            else st->peer_base[i][r] = (char *)b + all[r].off[i];
        }
    }
    cudaGetLastError();
    // every rank must agree (a rank that could not map its peers turns fusion off everywhere)
    int *dk = nullptr;
    int agree = 0;
    if (cudaMalloc((void **)&st->d_bar, sizeof(int)) == cudaSuccess &&
        cudaMemset(st->d_bar, 0, sizeof(int)) == cudaSuccess && cudaMalloc((void **)&dk, sizeof(int)) == cudaSuccess &&
        cudaMemcpy(dk, &local_ok, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
        ncclAllReduce(dk, dk, 1, ncclInt, ncclMin, s.comm, s.stream) == ncclSuccess &&
        cudaStreamSynchronize(s.stream) == cudaSuccess)
        cudaMemcpy(&agree, dk, sizeof(int), cudaMemcpyDeviceToHost);
    if (dk) cudaFree(dk);
    cudaGetLastError();
    st->p2p = agree == 1;
}

static void release_p2p(hq_state *st) {
    if (st->mode == MODE_RANK && !st->sh.empty()) {
        cudaSetDevice(st->sh[0].device);
        for (size_t r = 0; r < st->peer_base[0].size(); ++r) {
            if ((int)r == st->sh[0].rank) continue;
            for (int i = 0; i < 2; ++i)
                if (st->peer_base[i][r]) {
                    // the mapping was opened at the allocation base; psi/buf offsets are
                    // recomputed from the base the handle maps
                    void *b = nullptr;
                    if (alloc_base(st->peer_base[i][r], &b)) cudaIpcCloseMemHandle(b);
                }
        }
    }
    for (size_t r = 0; r < st->bar_ev.size(); ++r)
        if (st->bar_ev[r]) {
            cudaSetDevice(st->sh[r].device);
            cudaEventDestroy(st->bar_ev[r]);
        }
    if (st->d_bar) cudaFree(st->d_bar);
    cudaGetLastError();
}

// ------------------------------------------------------------------ create / destroy

extern "C" hq_status hq_state_create(int n, hq_dtype dtype, int ngpus, hq_state **out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!out) return set_error(HQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    hq_status rc = validate_common(n, dtype, ngpus);
    if (rc) return rc;
    if ((rc = check_device())) return rc;
    int cnt = 0;
    CUDA_TRY(cudaGetDeviceCount(&cnt));
    if (ngpus > cnt) return set_error(HQ_ERR_NGPUS, "ngpus=%d > %d visible devices", ngpus, cnt);
    hq_state *st = new_state(n, dtype, ngpus);
    if (!st) return set_error(HQ_ERR_OOM, "host allocation failed");
    st->mode = ngpus == 1 ? MODE_SINGLE : MODE_MULTI;
    st->sh.resize(ngpus);
    int cur = 0;
    cudaGetDevice(&cur);
    for (int r = 0; r < ngpus; ++r) {
        st->sh[r].device = ngpus == 1 ? cur : r;
        st->sh[r].rank = r;
        if ((rc = shard_alloc(st, st->sh[r], ngpus > 1, true))) {
            for (auto &s : st->sh) shard_free(s);
            delete st;
            return rc;
        }
    }
    if (ngpus > 1) {
        std::vector<ncclComm_t> comms(ngpus);
        std::vector<int> devs(ngpus);
        for (int r = 0; r < ngpus; ++r) devs[r] = r;
        ncclResult_t nr = ncclCommInitAll(comms.data(), ngpus, devs.data());
        if (nr != ncclSuccess) {
            for (auto &s : st->sh) shard_free(s);
            delete st;
            return set_error(HQ_ERR_NCCL, "ncclCommInitAll: %s", ncclGetErrorString(nr));
        }
        for (int r = 0; r < ngpus; ++r) st->sh[r].comm = comms[r];
        setup_p2p_multi(st);
    }
    cudaSetDevice(cur);
    *out = st;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_nccl_unique_id(void *out128) {
    HQ_ABI_BEGIN
    clear_error();
    if (!out128) return set_error(HQ_ERR_ARG, "out is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    memcpy(out128, &id, sizeof id);
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_create_rank(int n, hq_dtype dtype, int world_size, int rank,
                                          int device, const void *nccl_id, hq_state **out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!out) return set_error(HQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    hq_status rc = validate_common(n, dtype, world_size);
    if (rc) return rc;
    if (rank < 0 || rank >= world_size) return set_error(HQ_ERR_ARG, "rank %d not in [0,%d)", rank, world_size);
    if (world_size > 1 && !nccl_id) return set_error(HQ_ERR_ARG, "nccl_id is NULL");
    if ((rc = check_device())) return rc;
    hq_state *st = new_state(n, dtype, world_size);
    if (!st) return set_error(HQ_ERR_OOM, "host allocation failed");
    st->mode = world_size == 1 ? MODE_SINGLE : MODE_RANK;
    st->sh.resize(1);
    st->sh[0].device = device;
    st->sh[0].rank = rank;
    if ((rc = shard_alloc(st, st->sh[0], world_size > 1, true))) {
        shard_free(st->sh[0]);
        delete st;
        return rc;
    }
    if (world_size > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof id);
        cudaSetDevice(device);
        ncclResult_t nr = ncclCommInitRank(&st->sh[0].comm, world_size, id, rank);
        if (nr != ncclSuccess) {
            shard_free(st->sh[0]);
            delete st;
            return set_error(HQ_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(nr));
        }
        setup_p2p_rank(st);
    }
    *out = st;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_create_rank_from_buffers(int n, hq_dtype dtype, int world_size, int rank,
                                                       const void *nccl_id, void *psi_device, void *buf_device,
                                                       void *stream, hq_state **out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!out || !psi_device) return set_error(HQ_ERR_ARG, "NULL argument");
    *out = nullptr;
    hq_status rc = validate_common(n, dtype, world_size);
    if (rc) return rc;
    if (rank < 0 || rank >= world_size) return set_error(HQ_ERR_ARG, "rank %d not in [0,%d)", rank, world_size);
    if (world_size > 1 && (!nccl_id || !buf_device))
        return set_error(HQ_ERR_ARG, "world_size > 1 needs nccl_id and a receive buffer");
    if ((rc = check_device())) return rc;
    for (void *p : {psi_device, buf_device}) {
        if (!p) continue;
        if (((uintptr_t)p) & 255) return set_error(HQ_ERR_ARG, "buffer not 256-byte aligned");
        cudaPointerAttributes at;
        CUDA_TRY(cudaPointerGetAttributes(&at, p));
        if (at.type != cudaMemoryTypeDevice) return set_error(HQ_ERR_ARG, "buffer is not device memory");
    }
    cudaPointerAttributes at;
    CUDA_TRY(cudaPointerGetAttributes(&at, psi_device));
    hq_state *st = new_state(n, dtype, world_size);
    if (!st) return set_error(HQ_ERR_OOM, "host allocation failed");
    st->mode = world_size == 1 ? MODE_SINGLE : MODE_RANK;
    st->sh.resize(1);
    Shard &sh = st->sh[0];
    sh.device = at.device;
    sh.rank = rank;
    sh.psi = psi_device;
    sh.own_psi = false;
    if (world_size > 1) {
        sh.buf = buf_device;
        sh.own_buf = false;
    }
    sh.stream = reinterpret_cast<cudaStream_t>(stream);
    sh.own_stream = false;
    if ((rc = shard_alloc(st, sh, false, false))) {
        shard_free(sh);
        delete st;
        return rc;
    }
    if (world_size > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof id);
        cudaSetDevice(sh.device);
        ncclResult_t nr = ncclCommInitRank(&sh.comm, world_size, id, rank);
        if (nr != ncclSuccess) {
            shard_free(sh);
            delete st;
            return set_error(HQ_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(nr));
        }
        setup_p2p_rank(st);
    }
    *out = st;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_create_virtual(int n, hq_dtype dtype, int nshards, hq_state **out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!out) return set_error(HQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    hq_status rc = validate_common(n, dtype, nshards);
    if (rc) return rc;
    if ((rc = check_device())) return rc;
    hq_state *st = new_state(n, dtype, nshards);
    if (!st) return set_error(HQ_ERR_OOM, "host allocation failed");
    st->mode = MODE_VIRTUAL;
    st->p2p = true;                      // every shard buffer lives on this device
    st->sh.resize(nshards);
    int cur = 0;
    cudaGetDevice(&cur);
    for (int r = 0; r < nshards; ++r) {
        st->sh[r].device = cur;
        st->sh[r].rank = r;
        const bool mk = r == 0;
        if (!mk) { st->sh[r].stream = st->sh[0].stream; st->sh[r].own_stream = false; }
        if ((rc = shard_alloc(st, st->sh[r], nshards > 1, mk))) {
            for (auto &s : st->sh) shard_free(s);
            delete st;
            return rc;
        }
    }
    *out = st;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_create_from_buffers(int n, hq_dtype dtype, void *psi_device,
                                                  void *stream, hq_state **out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!out || !psi_device) return set_error(HQ_ERR_ARG, "NULL argument");
    *out = nullptr;
    hq_status rc = validate_common(n, dtype, 1);
    if (rc) return rc;
    if ((rc = check_device())) return rc;
    if (((uintptr_t)psi_device) & 15) return set_error(HQ_ERR_ARG, "psi buffer not 16-byte aligned");
    cudaPointerAttributes at;
    CUDA_TRY(cudaPointerGetAttributes(&at, psi_device));
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
        return set_error(HQ_ERR_ARG, "psi is not device memory");
    hq_state *st = new_state(n, dtype, 1);
    if (!st) return set_error(HQ_ERR_OOM, "host allocation failed");
    st->mode = MODE_SINGLE;
    st->sh.resize(1);
    Shard &s = st->sh[0];
    s.device = at.device;
    s.psi = psi_device;
    s.own_psi = false;
    s.stream = reinterpret_cast<cudaStream_t>(stream);
    s.own_stream = false;
    if ((rc = shard_alloc(st, s, false, false))) {
        shard_free(s);
        delete st;
        return rc;
    }
    *out = st;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_destroy(hq_state *st) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return HQ_OK;
    for (auto &p : st->prof) {
        cudaSetDevice(st->sh[p.shard].device);
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    release_p2p(st);
    // virtual shards share shard 0's stream: free others first
    for (size_t i = st->sh.size(); i-- > 0;) shard_free(st->sh[i]);
    delete st;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_set_remap_mode(hq_state *st, int mode, int *fused_available) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    if (mode & ~(HQ_REMAP_FUSED | HQ_REMAP_GATHER)) return set_error(HQ_ERR_ARG, "bad remap mode %d", mode);
    st->remap_mode = mode;
    if (fused_available) *fused_available = st->p2p ? 1 : 0;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_invalidate_bound(hq_state *st) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    st->amp_bound = -1.0;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_set_layout(hq_state *st, const int32_t *pi) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !pi) return set_error(HQ_ERR_ARG, "NULL argument");
    std::vector<int> seen(st->n, 0), v(st->n);
    for (int q = 0; q < st->n; ++q) {
        if (pi[q] < 0 || pi[q] >= st->n || seen[pi[q]]++)
            return set_error(HQ_ERR_ARG, "layout is not a permutation of [0, %d)", st->n);
        v[q] = pi[q];
    }
    st->pi = v;
    st->pi_init = v;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_get_layout(const hq_state *st, int32_t *pi_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !pi_out) return set_error(HQ_ERR_ARG, "NULL argument");
    for (int q = 0; q < st->n; ++q) pi_out[q] = st->pi[q];
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_set_stream(hq_state *st, void *stream) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    if (st->mode == MODE_MULTI) return set_error(HQ_ERR_STATE, "set_stream not supported for multi-device states");
    Shard &s0 = st->sh[0];
    CUDA_TRY(cudaSetDevice(s0.device));
    if (s0.stream) SYNC_TRY(s0);
    if (s0.own_stream && s0.stream) cudaStreamDestroy(s0.stream);
    for (auto &s : st->sh) {
        s.stream = reinterpret_cast<cudaStream_t>(stream);
        s.own_stream = false;
    }
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_state_info(const hq_state *st, int *n, int *dtype, int *world,
                                   int *local_shards, int *first_rank) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    if (n) *n = st->n;
    if (dtype) *dtype = (int)st->dtype;
    if (world) *world = st->world;
    if (local_shards) *local_shards = (int)st->sh.size();
    if (first_rank) *first_rank = st->sh[0].rank;
    return HQ_OK;
    HQ_ABI_END
}

// ------------------------------------------------------------------ executor

// Canonicalise: sort targets by physical bit ascending and permute U so that
// U-index bit i <-> i-th smallest target (exact), keep it in fp64.
static void canonical_U64(const double *U, int k, const int *phys, ApplyDesc &d,
                          std::vector<double> &out, int nl) {
    int order[6];
    for (int j = 0; j < k; ++j) order[j] = j;
    std::sort(order, order + k, [&](int a, int b) { return phys[a] < phys[b]; });
    d.k = k;
    d.n_local = nl;
    for (int i = 0; i < k; ++i) d.p[i] = phys[order[i]];
    // canonical bit i corresponds to user target order[i], whose user U bit is k-1-order[i]
    const int D = 1 << k;
    std::vector<int> map(D);
    for (int c = 0; c < D; ++c) {
        int u = 0;
        for (int i = 0; i < k; ++i)
            if ((c >> i) & 1) u |= 1 << (k - 1 - order[i]);
        map[c] = u;
    }
    out.resize((size_t)2 * D * D);
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            out[2 * (r * D + c)] = U[2 * (map[r] * D + map[c])];
            out[2 * (r * D + c) + 1] = U[2 * (map[r] * D + map[c]) + 1];
        }
}

enum { PATH_REG = 0, PATH_GEN = 1, PATH_TC = 2 };

struct Prep {
    ApplyDesc d;
    double gnorm = 1.0;          // upper bound on the spectral norm of U
    int path = PATH_GEN;
    std::vector<char> hostU;     // canonical U in the state dtype (RN from fp64)
    std::vector<char> payload;   // bytes the kernel reads from device memory
    std::vector<char> params;    // TC parameter block
    bool scalar = false;         // row f1: every target global -> a phase sre + i sim
    double sre = 1.0, sim = 0.0;
};

// Upper bound on ||U||_2: sqrt of the Gershgorin bound on lambda_max(U^H U)
// (max_i sum_j |(U^H U)_ij|), times a small slack for the FP32 rounding of the
// pass.  Tight (1 + ~1e-15) for unitary U; rigorous for any U.
static double spectral_bound(const double *U, int k) {
    const int D = 1 << k;
    double worst = 0.0;
    for (int i = 0; i < D; ++i) {
        double row = 0.0;
        for (int j = 0; j < D; ++j) {
            double re = 0.0, im = 0.0;     // (U^H U)_ij = sum_r conj(U_ri) U_rj
            for (int r = 0; r < D; ++r) {
                const double ar = U[2 * (r * D + i)], ai = -U[2 * (r * D + i) + 1];
                const double br = U[2 * (r * D + j)], bi = U[2 * (r * D + j) + 1];
                re += ar * br - ai * bi;
                im += ar * bi + ai * br;
            }
            row += std::sqrt(re * re + im * im);
        }
        worst = std::max(worst, row);
    }
    return std::sqrt(worst) * (1.0 + 1e-5);
}

static void prepare(hq_dtype dt, const double *U, int k, const int *phys, int nl, Prep &p) {
    p.scalar = false;
    std::vector<double> Uc;
    canonical_U64(U, k, phys, p.d, Uc, nl);
    p.gnorm = spectral_bound(Uc.data(), k);
    const int D = 1 << k;
    const size_t es = dt == HQ_C64 ? 8 : 16;
    p.hostU.resize(es * D * D);
    for (size_t i = 0; i < (size_t)2 * D * D; ++i) {
        if (dt == HQ_C64) reinterpret_cast<float *>(p.hostU.data())[i] = (float)Uc[i];
        else reinterpret_cast<double *>(p.hostU.data())[i] = Uc[i];
    }
    p.payload.clear();
    p.params.clear();
    if (tc_applicable((int)dt, p.d)) {
        p.path = PATH_TC;
        tc_prepare(p.d, Uc.data(), p.payload, p.params);
    } else if (!apply_needs_dev_U((int)dt, p.d)) {
        p.path = PATH_REG;
    } else {
        p.path = PATH_GEN;
        p.payload = p.hostU;
    }
}

static hq_status prof_begin(hq_state *st, Shard &s, ProfEvent &pe) {
    if (!st->profiling) return HQ_OK;
    CUDA_TRY(cudaSetDevice(s.device));
    auto take = [&]() {
        cudaEvent_t e;
        if (!s.ev_pool.empty()) { e = s.ev_pool.back(); s.ev_pool.pop_back(); }
        else cudaEventCreate(&e);
        return e;
    };
    pe.a = take();
    pe.b = take();
    pe.shard = (int)(&s - st->sh.data());
    CUDA_TRY(cudaEventRecord(pe.a, s.stream));
    return HQ_OK;
}

static hq_status prof_end(hq_state *st, Shard &s, ProfEvent &pe, uint64_t bytes, int path) {
    if (!st->profiling) return HQ_OK;
    CUDA_TRY(cudaEventRecord(pe.b, s.stream));
    pe.bytes = bytes;
    pe.path = path;
    st->prof.push_back(pe);
    return HQ_OK;
}

static hq_status ensure_bound(hq_state *st);

// apply+pack: the scheduler's PERMUTE right after an APPLY is
// folded into that pass, which then reads psi and writes the bit-permuted
// result into the exchange buffer (no extra HBM pass).  True when the
// prepared pass can do so; o receives the output map (dst set per shard).
static bool pack_spec(const hq_state *st, const Prep &p, const Op &perm, OutSpec &o) {
    if (p.scalar || perm.kind != OP_PERMUTE || perm.nbits < 1 || perm.nbits > 6) return false;
    o = OutSpec{};
    o.active = true;
    o.npairs = perm.nbits;
    for (int i = 0; i < perm.nbits; ++i) {
        o.pa[i] = perm.bits[2 * i];
        o.pb[i] = perm.bits[2 * i + 1];
        if (o.pa[i] < PACK_MIN_BIT || o.pb[i] < PACK_MIN_BIT) return false;
    }
    for (auto &sh : st->sh)
        if (!sh.buf) return false;
    if (p.path == PATH_TC) {
        std::vector<char> tmp = p.params;
        return tc_set_output(tmp, o);
    }
    return apply_supports_out((int)st->dtype, p.d, o);
}

static hq_status exec_apply(hq_state *st, Shard &s, const Prep &p, const void *dU, const OutSpec *pack = nullptr,
                           bool fused_remap = false) {
    CUDA_TRY(cudaSetDevice(s.device));
    ProfEvent pe{};
    hq_status rc = HQ_OK;
    std::vector<char> params;
    OutSpec o;
    if (pack) {
        o = *pack;
        if (!fused_remap) o.dst[0] = s.buf;      // apply+pack: this shard's own exchange buffer
    }
    if (p.path == PATH_TC) {
        if ((rc = ensure_bound(st))) return rc;
        params = p.params;
        tc_set_amp_bound(params, st->amp_bound);
        if (pack && !tc_set_output(params, o)) return set_error(HQ_ERR_STATE, "internal: pack not supported");
    }
    if ((rc = prof_begin(st, s, pe))) return rc;
    int launches = 0;
    int e;
    if (p.path == PATH_TC) {
        e = tc_launch(s.psi, params.data(), params.size(), dU, s.stream);
        launches = 1;
    } else {
        e = launch_apply((int)st->dtype, s.psi, p.d, p.hostU.data(), dU, s.stream, &launches, pack ? &o : nullptr);
    }
    if (e != cudaSuccess)
        return set_error(HQ_ERR_CUDA, "apply kernel launch failed: %s", cudaGetErrorString((cudaError_t)e));
    const uint64_t bytes = (uint64_t)2 * (st->es << st->nl);
    if ((rc = prof_end(st, s, pe, bytes, p.path))) return rc;
    if (pack && !fused_remap) {
        std::swap(s.psi, s.buf);
        std::swap(s.own_psi, s.own_buf);
    }
    st->stats.passes++;
    st->stats.kernel_launches += launches;
    st->stats.hbm_bytes += bytes;
    return HQ_OK;
}

// ------------------------------------------------------------------ row f1: global-diagonal gates
// The scheduler leaves a gate on its global targets when U is block-diagonal
// in them (block_diag_in): rank r then applies the block V_x, x = r's values
// of those bits, to the local targets; with no local target V_x is a phase.
static bool op_conditioned(const hq_state *st, const Op &op) {
    for (int j = 0; j < op.nbits; ++j)
        if (op.bits[j] >= st->nl) return true;
    return false;
}

static void prepare_cond(const hq_state *st, const GateRef &g, const Op &op, int rank, Prep &p) {
    const int k = g.k, D = 1 << k;
    int lb[6], lu[6], kl = 0, fixval = 0;
    for (int j = 0; j < k; ++j) {
        const int ub = k - 1 - j, b = op.bits[j];
        if (b >= st->nl) {
            if ((rank >> (b - st->nl)) & 1) fixval |= 1 << ub;
        } else {
            lb[kl] = b;
            lu[kl] = ub;
            ++kl;
        }
    }
    p.scalar = kl == 0;
    if (p.scalar) {
        p.sre = g.U[2 * (fixval * D + fixval)];
        p.sim = g.U[2 * (fixval * D + fixval) + 1];
        p.gnorm = std::hypot(p.sre, p.sim) * (1.0 + 1e-5);
        p.payload.clear();
        return;
    }
    const int d = 1 << kl;
    auto expand = [&](int a) {
        int x = fixval;
        for (int t = 0; t < kl; ++t)
            if ((a >> (kl - 1 - t)) & 1) x |= 1 << lu[t];
        return x;
    };
    std::vector<double> V((size_t)2 * d * d);
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            const size_t src = 2 * ((size_t)expand(r) * D + expand(c));
            V[2 * (r * d + c)] = g.U[src];
            V[2 * (r * d + c) + 1] = g.U[src + 1];
        }
    prepare(st->dtype, V.data(), kl, lb, st->nl, p);
}

static hq_status exec_prep(hq_state *st, Shard &s, const Prep &p, const void *dU, const OutSpec *pack = nullptr) {
    if (!p.scalar) return exec_apply(st, s, p, dU, pack, false);
    if (p.sre == 1.0 && p.sim == 0.0) return HQ_OK;
    CUDA_TRY(cudaSetDevice(s.device));
    int e = launch_scale_complex((int)st->dtype, s.psi, 1ull << st->nl, p.sre, p.sim, s.stream);
    if (e) return set_error(HQ_ERR_CUDA, "phase launch: %s", cudaGetErrorString((cudaError_t)e));
    st->stats.passes++;
    st->stats.kernel_launches++;
    st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
    return HQ_OK;
}

static hq_status exec_permute(hq_state *st, const Op &op) {
    int a[6], b[6];
    for (int i = 0; i < op.nbits; ++i) { a[i] = op.bits[2 * i]; b[i] = op.bits[2 * i + 1]; }
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        int e = launch_permute((int)st->dtype, s.psi, s.buf, 1ull << st->nl, op.nbits, a, b, s.stream);
        if (e != cudaSuccess)
            return set_error(HQ_ERR_CUDA, "permute launch failed: %s", cudaGetErrorString((cudaError_t)e));
        std::swap(s.psi, s.buf);
        std::swap(s.own_psi, s.own_buf);
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
    }
    st->swaps++;
    st->stats.permutes++;
    return HQ_OK;
}

// REMAP: swap global (rank) bits g_i with local bits l_i.  Element x of rank
// r goes to the peer p whose g-bits equal x's l-bits, landing at x with its
// l-bits replaced by r's g-bits.  This is symmetric: for each peer p (index t
// = p's g-bits), rank r sends the runs of x whose l-bits equal t and receives
// p's runs into the same offsets.  The runs: x = pdep(rho << lmin, ~Lmask) |
// pdep(t, Lmask), length 2^lmin amplitudes (one run per peer after a pack).
// remap_transfers lists them for one rank; the executor and hq_remap_plan
// (host-only, used by the gloo test) share it.
struct Transfer {
    int peer;
    uint64_t off, len;      // amplitudes: send [off, off+len) of this shard, receive into the same range
};

static bool remap_transfers(int nl, int m, const Op &op, int rank, std::vector<Transfer> &out) {
    out.clear();
    const int mp = op.nbits;
    int gsh[6], lb[6];
    uint64_t lmask = 0;
    int lmin = 64;
    for (int i = 0; i < mp; ++i) {
        gsh[i] = op.bits[2 * i] - nl;
        lb[i] = op.bits[2 * i + 1];
        if (lb[i] < 0 || lb[i] >= nl || gsh[i] < 0 || gsh[i] >= m) return false;
        lmask |= 1ull << lb[i];
        lmin = std::min(lmin, lb[i]);
    }
    const uint64_t runlen = 1ull << lmin;
    const uint64_t nruns = 1ull << (nl - mp - lmin);
    for (int t = 0; t < (1 << mp); ++t) {
        int p = rank;
        for (int i = 0; i < mp; ++i) p = (p & ~(1 << gsh[i])) | (((t >> i) & 1) << gsh[i]);
        for (uint64_t rho = 0; rho < nruns; ++rho) {
            uint64_t x = 0, src = rho << lmin;
            int b = 0;
            for (int pos = 0; pos < nl; ++pos) {
                if ((lmask >> pos) & 1) {
                    int i = 0;
                    while (lb[i] != pos) ++i;
                    x |= (uint64_t)((t >> i) & 1) << pos;
                } else {
                    x |= ((src >> b) & 1) << pos;
                    ++b;
                }
            }
            out.push_back({p, x, runlen});
        }
    }
    return true;
}

static hq_status exec_remap(hq_state *st, const Op &op) {
    std::vector<std::vector<Transfer>> plan(st->sh.size());
    for (size_t r = 0; r < st->sh.size(); ++r)
        if (!remap_transfers(st->nl, st->m, op, st->sh[r].rank, plan[r]))
            return set_error(HQ_ERR_STATE, "internal: bad remap bits");
    if (st->mode == MODE_VIRTUAL) {
        // shard r's run [off, off+len) lands in the peer's buffer at the run
        // of r's g-bits: the peer's own transfer list pairs them the same way
        // (symmetry), so copy r -> p at the offset p uses for peer r
        // shard r's run (t, rho) lands in the peer's buffer at the run offset
        // of (u, rho), u = r's swapped rank bits (offsets depend only on (t, rho))
        for (size_t r = 0; r < st->sh.size(); ++r) {
            Shard &s = st->sh[r];
            const size_t nruns = plan[r].size() >> op.nbits;
            int u = 0;
            for (int i = 0; i < op.nbits; ++i) u |= ((s.rank >> (op.bits[2 * i] - st->nl)) & 1) << i;
            for (size_t i = 0; i < plan[r].size(); ++i) {
                const Transfer &x = plan[r][i];
                Shard &d = st->sh[x.peer];
                const uint64_t doff = plan[r][(size_t)u * nruns + i % nruns].off;
                CUDA_TRY(cudaMemcpyAsync((char *)d.buf + doff * st->es, (const char *)s.psi + x.off * st->es,
                                         x.len * st->es, cudaMemcpyDeviceToDevice, s.stream));
                if (d.rank != s.rank) st->stats.link_bytes += x.len * st->es;
            }
        }
    } else {
        NCCL_TRY(ncclGroupStart());
        for (size_t r = 0; r < st->sh.size(); ++r) {
            Shard &s = st->sh[r];
            cudaSetDevice(s.device);
            for (const Transfer &x : plan[r]) {
                const char *src = (const char *)s.psi + x.off * st->es;
                char *dst = (char *)s.buf + x.off * st->es;     // from the peer: its runs for our g-bits land here
                const size_t bytes = x.len * st->es;
                if (x.peer == s.rank) {
                    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s.stream));
                } else {
                    NCCL_TRY(ncclSend(src, bytes, ncclChar, x.peer, s.comm, s.stream));
                    NCCL_TRY(ncclRecv(dst, bytes, ncclChar, x.peer, s.comm, s.stream));
                    st->stats.link_bytes += bytes;
                }
            }
        }
        NCCL_TRY(ncclGroupEnd());
    }
    for (auto &s : st->sh) {
        std::swap(s.psi, s.buf);
        std::swap(s.own_psi, s.own_buf);
    }
    st->swaps++;
    st->stats.remaps++;
    return HQ_OK;
}

extern "C" hq_status hq_remap_plan(int n, int m, const hq_op *op, int rank, int32_t *peer_out, uint64_t *off_out,
                                   uint64_t *len_out, size_t cap, size_t *count) {
    HQ_ABI_BEGIN
    clear_error();
    if (!op || !count) return set_error(HQ_ERR_ARG, "NULL argument");
    if (op->kind != OP_REMAP || m < 1 || n - m < 1 || rank < 0 || rank >= (1 << m) || op->nbits < 1 || op->nbits > 6)
        return set_error(HQ_ERR_ARG, "not a REMAP op of an n=%d, m=%d state / bad rank", n, m);
    Op o{OP_REMAP, -1, op->nbits, {0}};
    for (int t = 0; t < 12; ++t) o.bits[t] = op->bits[t];
    std::vector<Transfer> v;
    if (!remap_transfers(n - m, m, o, rank, v)) return set_error(HQ_ERR_ARG, "bad remap bits");
    *count = v.size();
    if (cap < v.size()) return peer_out ? set_error(HQ_ERR_RANGE, "cap %zu < %zu transfers", cap, v.size()) : HQ_OK;
    for (size_t i = 0; i < v.size(); ++i) {
        if (peer_out) peer_out[i] = v[i].peer;
        if (off_out) off_out[i] = v[i].off;
        if (len_out) len_out[i] = v[i].len;
    }
    return HQ_OK;
    HQ_ABI_END
}

static hq_status validate_gates(const hq_state *st, const hq_gate *g, size_t ng,
                                std::vector<GateRef> &refs) {
    refs.resize(ng);
    for (size_t i = 0; i < ng; ++i) {
        const hq_gate &x = g[i];
        if (x.k < 1 || x.k > 6) return set_error(HQ_ERR_K, "gate %zu: k=%d not in [1,6]", i, x.k);
        if (x.k > st->nl)
            return set_error(HQ_ERR_K, "gate %zu: k=%d > %d local qubits", i, x.k, st->nl);
        if (!x.U) return set_error(HQ_ERR_ARG, "gate %zu: U is NULL", i);
        refs[i].k = x.k;
        refs[i].U = x.U;
        for (int j = 0; j < x.k; ++j) {
            const int q = x.qubits[j];
            if (q < 0 || q >= st->n)
                return set_error(HQ_ERR_QUBIT, "gate %zu: qubit %d not in [0,%d)", i, q, st->n);
            for (int l = 0; l < j; ++l)
                if (x.qubits[l] == q) return set_error(HQ_ERR_DUP_QUBIT, "gate %zu: repeated qubit %d", i, q);
            refs[i].q[j] = q;
        }
    }
    return HQ_OK;
}

// ------------------------------------------------------------------ apply+pack and fused remaps
// How an APPLY op executes together with the ops after it:
//   consumed 0: alone, in place;
//   consumed 1, !fused: the PERMUTE after it folded in (apply+pack);
//   fused: [PERMUTE +] REMAP folded in (fused remap): the pass writes every
//   element into its destination rank's exchange buffer, peer memory over
//   NVLink (the remap's local bits must be the top nin local bits, which the
//   scheduler's pack guarantees).
static bool out_supported(const hq_state *st, const Prep &p, const OutSpec &o) {
    if (p.scalar) return false;
    if (p.path == PATH_TC) {
        std::vector<char> tmp = p.params;
        return tc_set_output(tmp, o);
    }
    return apply_supports_out((int)st->dtype, p.d, o);
}

static Fold plan_fold(const hq_state *st, const Prep &p, const std::vector<Op> &ops, size_t i) {
    Fold f;
    size_t j = i + 1;
    const Op *perm = (j < ops.size() && ops[j].kind == OP_PERMUTE) ? &ops[j] : nullptr;
    if (perm) ++j;
    const Op *rem = (j < ops.size() && ops[j].kind == OP_REMAP) ? &ops[j] : nullptr;
    for (auto &sh : st->sh)
        if (!sh.buf) return f;
    if (rem && (st->remap_mode & HQ_REMAP_FUSED) && st->p2p && rem->nbits >= 1 && rem->nbits <= 3) {
        bool top = true;
        for (int t = 0; t < rem->nbits; ++t) top &= rem->bits[2 * t + 1] == st->nl - rem->nbits + t;
        OutSpec o;
        o.active = true;
        if (perm) {
            o.npairs = perm->nbits;
            for (int t = 0; t < perm->nbits; ++t) {
                o.pa[t] = perm->bits[2 * t];
                o.pb[t] = perm->bits[2 * t + 1];
                top &= o.pa[t] >= PACK_MIN_BIT && o.pb[t] >= PACK_MIN_BIT;
            }
        }
        o.tsh = st->nl - rem->nbits;
        o.tmask = (1u << rem->nbits) - 1;
        for (int t = 0; t < 8; ++t) o.dst[t] = st->sh[0].buf;    // placeholders for the support check
        if (top && out_supported(st, p, o)) {
            f.consumed = (perm ? 1 : 0) + 1;
            f.fused = true;
            f.with_perm = perm != nullptr;
            f.rem = rem;
            f.tmpl = o;
            return f;
        }
    }
    if (perm && pack_spec(st, p, *perm, f.tmpl)) {
        f.consumed = 1;
        f.with_perm = true;
    }
    return f;
}

// the rank whose rank bits gsh[i] equal t's bits i (the others as r's)
static int remap_peer(const Op &rem, int nl, int r, int t) {
    int p = r;
    for (int i = 0; i < rem.nbits; ++i) {
        const int g = rem.bits[2 * i] - nl;
        p = (p & ~(1 << g)) | (((t >> i) & 1) << g);
    }
    return p;
}

static int remap_bits(const Op &rem, int nl, int r) {
    int t = 0;
    for (int i = 0; i < rem.nbits; ++i) t |= ((r >> (rem.bits[2 * i] - nl)) & 1) << i;
    return t;
}

// the current exchange buffer of rank p, as addressable from this process
static void *peer_buf(const hq_state *st, int p) {
    if (st->mode != MODE_RANK) return st->sh[p].buf;
    if (p == st->sh[0].rank) return st->sh[0].buf;
    return st->peer_base[(st->swaps & 1) ? 0 : 1][p];
}

// All shards' streams reach this point before any continues (fused remaps
// write into peers' buffers, which must be free before and complete after).
// the current state buffer of rank p, as addressable from this process
static const void *peer_psi(const hq_state *st, int p) {
    if (st->mode != MODE_RANK) return st->sh[p].psi;
    if (p == st->sh[0].rank) return st->sh[0].psi;
    return st->peer_base[(st->swaps & 1) ? 1 : 0][p];
}

static bool use_gather(const hq_state *st) {
    return st->m > 0 && st->p2p && (st->remap_mode & HQ_REMAP_GATHER);
}

static hq_status peer_barrier(hq_state *st) {
    if (st->mode == MODE_RANK) {
        Shard &s = st->sh[0];
        CUDA_TRY(cudaSetDevice(s.device));
        NCCL_TRY(ncclAllReduce(st->d_bar, st->d_bar, 1, ncclInt, ncclSum, s.comm, s.stream));
    } else if (st->mode == MODE_MULTI) {
        for (size_t r = 0; r < st->sh.size(); ++r) {
            CUDA_TRY(cudaSetDevice(st->sh[r].device));
            CUDA_TRY(cudaEventRecord(st->bar_ev[r], st->sh[r].stream));
        }
        for (size_t r = 0; r < st->sh.size(); ++r) {
            CUDA_TRY(cudaSetDevice(st->sh[r].device));
            for (size_t q = 0; q < st->sh.size(); ++q)
                if (q != r) CUDA_TRY(cudaStreamWaitEvent(st->sh[r].stream, st->bar_ev[q], 0));
        }
    }
    return HQ_OK;        // virtual shards share one stream
}

// Execute an APPLY with its fold.  get(r) -> (prep, device payload) of shard r.
template <class Get>
static hq_status run_apply(hq_state *st, const Fold &f, Get get) {
    hq_status rc;
    const size_t G = st->sh.size();
    if (!f.fused) {
        for (size_t r = 0; r < G; ++r) {
            auto pr = get(r);
            if ((rc = exec_prep(st, st->sh[r], *pr.first, pr.second, f.consumed ? &f.tmpl : nullptr))) return rc;
        }
        if (f.consumed) {
            st->swaps++;
            st->stats.packs++;
        }
        return HQ_OK;
    }
    // fused remap: every shard's output map from the peer buffers as they are now
    std::vector<OutSpec> os(G, f.tmpl);
    for (size_t r = 0; r < G; ++r) {
        const int rank = st->sh[r].rank;
        os[r].add = (uint64_t)remap_bits(*f.rem, st->nl, rank) << os[r].tsh;
        for (int t = 0; t < (1 << f.rem->nbits); ++t) os[r].dst[t] = peer_buf(st, remap_peer(*f.rem, st->nl, rank, t));
    }
    if ((rc = peer_barrier(st))) return rc;
    for (size_t r = 0; r < G; ++r) {
        auto pr = get(r);
        if ((rc = exec_apply(st, st->sh[r], *pr.first, pr.second, &os[r], true))) return rc;
    }
    if ((rc = peer_barrier(st))) return rc;
    for (auto &s : st->sh) {
        std::swap(s.psi, s.buf);
        std::swap(s.own_psi, s.own_buf);
    }
    st->swaps++;
    st->stats.remaps++;
    st->stats.remaps_fused++;
    if (f.with_perm) st->stats.packs++;
    const uint64_t chunk = (st->es << st->nl) >> f.rem->nbits;
    st->stats.link_bytes += (uint64_t)G * (((uint64_t)1 << f.rem->nbits) - 1) * chunk;
    return HQ_OK;
}

// OP_GATHER (row f1): the gate's one global target stays global; the rank
// pair that differs in it computes the gate over peer memory, each writing
// its half into its exchange buffer (out of place: the partner reads this
// rank's state during the pass), between two barriers.
static void prepare_gather(hq_dtype dt, const double *U, int k, const int *phys, int nl, Prep &p) {
    std::vector<double> Uc;
    canonical_U64(U, k, phys, p.d, Uc, nl);     // the global bit sorts last: canonical bit k-1
    p.gnorm = spectral_bound(Uc.data(), k);
    const int D = 1 << k;
    const size_t es = dt == HQ_C64 ? 8 : 16;
    p.hostU.resize(es * D * D);
    for (size_t i = 0; i < (size_t)2 * D * D; ++i) {
        if (dt == HQ_C64) reinterpret_cast<float *>(p.hostU.data())[i] = (float)Uc[i];
        else reinterpret_cast<double *>(p.hostU.data())[i] = Uc[i];
    }
    p.payload = p.hostU;
    p.params.clear();
    p.path = PATH_GEN;
    p.scalar = false;
}

template <class GetU>
static hq_status exec_gather(hq_state *st, const Prep &p, GetU dU_of) {
    hq_status rc;
    const int gsh = p.d.p[p.d.k - 1] - st->nl;
    if (gsh < 0 || gsh >= st->m) return set_error(HQ_ERR_STATE, "internal: gather without a global target");
    if ((rc = peer_barrier(st))) return rc;
    for (size_t r = 0; r < st->sh.size(); ++r) {
        Shard &s = st->sh[r];
        CUDA_TRY(cudaSetDevice(s.device));
        const int half = (s.rank >> gsh) & 1, partner = s.rank ^ (1 << gsh);
        int e = launch_pair_gather((int)st->dtype, s.psi, peer_psi(st, partner), s.buf, p.d, half, dU_of(r), s.stream);
        if (e) return set_error(HQ_ERR_CUDA, "pair gather launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
        st->stats.link_bytes += st->es << st->nl;
    }
    if ((rc = peer_barrier(st))) return rc;
    for (auto &s : st->sh) {
        std::swap(s.psi, s.buf);
        std::swap(s.own_psi, s.own_buf);
    }
    st->swaps++;
    st->stats.passes++;
    st->stats.gathers++;
    if (st->amp_bound >= 0) st->amp_bound *= p.gnorm;
    return HQ_OK;
}

// Run an op stream with matrices either host-side (converted on the fly and
// staged through the arena) or precompiled (circuit).
static hq_status run_ops(hq_state *st, const std::vector<GateRef> &refs, const std::vector<Op> &ops) {
    Prep p;
    std::vector<void *> dUs(st->sh.size());
    for (size_t i = 0; i < ops.size(); ++i) {
        const Op &op = ops[i];
        hq_status rc = HQ_OK;
        if (op.kind == OP_APPLY) {
            const GateRef &g = refs[op.gate];
            if (op_conditioned(st, op)) {
                for (size_t r = 0; r < st->sh.size(); ++r) {
                    Shard &s = st->sh[r];
                    prepare_cond(st, g, op, s.rank, p);
                    void *dU = nullptr;
                    if (!p.payload.empty() && (rc = arena_push(st, s, p.payload.data(), p.payload.size(), &dU)))
                        return rc;
                    if ((rc = exec_prep(st, s, p, dU))) return rc;
                }
                if (st->amp_bound >= 0) st->amp_bound *= spectral_bound(g.U, g.k);
                continue;
            }
            prepare(st->dtype, g.U, g.k, op.bits, st->nl, p);
            const Fold f = plan_fold(st, p, ops, i);
            for (size_t r = 0; r < st->sh.size(); ++r) {
                dUs[r] = nullptr;
                if (!p.payload.empty() && (rc = arena_push(st, st->sh[r], p.payload.data(), p.payload.size(), &dUs[r])))
                    return rc;
            }
            if ((rc = run_apply(st, f, [&](size_t r) { return std::make_pair((const Prep *)&p, (const void *)dUs[r]); })))
                return rc;
            i += f.consumed;
            if (st->amp_bound >= 0) st->amp_bound *= p.gnorm;
        } else if (op.kind == OP_GATHER) {
            const GateRef &g = refs[op.gate];
            prepare_gather(st->dtype, g.U, g.k, op.bits, st->nl, p);
            for (size_t r = 0; r < st->sh.size(); ++r) {
                dUs[r] = nullptr;
                if ((rc = arena_push(st, st->sh[r], p.payload.data(), p.payload.size(), &dUs[r]))) return rc;
            }
            rc = exec_gather(st, p, [&](size_t r) { return (const void *)dUs[r]; });
        } else if (op.kind == OP_REMAP) {
            rc = exec_remap(st, op);
        } else {
            rc = exec_permute(st, op);
        }
        if (rc) return rc;
    }
    return HQ_OK;
}

extern "C" hq_status hq_apply_matrix(hq_state *st, const double *U, const int32_t *qubits, int k) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !U || !qubits) return set_error(HQ_ERR_ARG, "NULL argument");
    if (k < 1 || k > 6) return set_error(HQ_ERR_K, "k=%d not in [1,6]", k);
    hq_gate g;
    g.k = k;
    for (int j = 0; j < 6; ++j) g.qubits[j] = j < k ? qubits[j] : -1;
    g.U = U;
    return hq_apply_circuit(st, &g, 1);
    HQ_ABI_END
}

extern "C" hq_status hq_apply_circuit(hq_state *st, const hq_gate *gates, size_t ng) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || (!gates && ng)) return set_error(HQ_ERR_ARG, "NULL argument");
    std::vector<GateRef> refs;
    hq_status rc = validate_gates(st, gates, ng, refs);
    if (rc) return rc;
    std::vector<Op> ops;
    std::vector<int> pi = st->pi;
    schedule(st->n, st->m, refs, pi, ops, use_gather(st));
    rc = run_ops(st, refs, ops);
    if (rc) return rc;
    st->pi = pi;
    return HQ_OK;
    HQ_ABI_END
}

// ------------------------------------------------------------------ circuits

static hq_status circuit_compile(hq_state *st, hq_circuit *c, const std::vector<GateRef> &refs) {
    c->pi_start = st->pi;
    c->pi_end = st->pi;
    schedule(st->n, st->m, refs, c->pi_end, c->ops, use_gather(st));
    c->prep.assign(c->ops.size(), Prep{});
    c->op_uoff.assign(c->ops.size(), -1);
    c->cprep.assign(c->ops.size(), {});
    c->cuoff.assign(c->ops.size(), {});
    c->cgnorm.assign(c->ops.size(), 1.0);
    c->fold.assign(c->ops.size(), Fold{});
    size_t total = 0;
    c->passes = c->remaps = c->permutes = c->packs = c->gathers = 0;
    for (size_t i = 0; i < c->ops.size(); ++i) {
        const Op &op = c->ops[i];
        bool folded = false;          // consumed by an earlier APPLY's fold
        for (size_t b = 1; b <= 2 && b <= i && !folded; ++b)
            folded = c->ops[i - b].kind == OP_APPLY && (size_t)c->fold[i - b].consumed >= b;
        if (folded) {
            if (op.kind == OP_REMAP) c->remaps++;
            continue;
        }
        if (op.kind == OP_APPLY) {
            const GateRef &g = refs[op.gate];
            if (op_conditioned(st, op)) {
                const size_t G = st->sh.size();
                c->cprep[i].assign(G, Prep{});
                c->cuoff[i].assign(G, -1);
                c->cgnorm[i] = spectral_bound(g.U, g.k);
                for (size_t r = 0; r < G; ++r) {
                    prepare_cond(st, g, op, st->sh[r].rank, c->cprep[i][r]);
                    if (!c->cprep[i][r].payload.empty()) {
                        c->cuoff[i][r] = (long long)total;
                        total += (c->cprep[i][r].payload.size() + 255) & ~(size_t)255;
                    }
                }
                c->passes++;
                continue;
            }
            prepare(st->dtype, g.U, g.k, op.bits, st->nl, c->prep[i]);
            if (!c->prep[i].payload.empty()) {
                c->op_uoff[i] = (long long)total;
                total += (c->prep[i].payload.size() + 255) & ~(size_t)255;
            }
            c->fold[i] = plan_fold(st, c->prep[i], c->ops, i);
            if (c->fold[i].fused) c->fold[i].rem = nullptr;     // re-pointed at run time (ops may move)
            if (c->fold[i].with_perm) c->packs++;
            c->passes++;
        } else if (op.kind == OP_GATHER) {
            const GateRef &g = refs[op.gate];
            prepare_gather(st->dtype, g.U, g.k, op.bits, st->nl, c->prep[i]);
            c->op_uoff[i] = (long long)total;
            total += (c->prep[i].payload.size() + 255) & ~(size_t)255;
            c->passes++;
            c->gathers++;
        } else if (op.kind == OP_REMAP) {
            c->remaps++;
        } else {
            c->permutes++;
        }
    }
    for (size_t r = 0; r < c->dev_U.size(); ++r)
        if (c->dev_U[r]) {
            cudaSetDevice(c->dev_of[r]);
            cudaFree(c->dev_U[r]);
        }
    c->dev_U.assign(st->sh.size(), nullptr);
    c->dev_of.resize(st->sh.size());
    for (size_t r = 0; r < st->sh.size(); ++r) c->dev_of[r] = st->sh[r].device;
    // small states: one CTA runs every pass with the shard in shared memory
    {
        // measured (tools/small_timing.py): one CTA beats the per-pass graph
        // for n_local <= 10 with >= 2 passes (8q: 16.5 vs 28.7 us, 10q: 45 vs
        // 55 us); at 11-12 qubits the multi-SM passes win (12q: 132 vs 237 us)
        const int maxnl = std::min(10, st->dtype == HQ_C64 ? SMEM_CIRCUIT_MAX_NL_C64 : SMEM_CIRCUIT_MAX_NL_C128);
        bool ok = st->sh.size() == 1 && st->m == 0 && st->nl <= maxnl && c->ops.size() >= 2 && c->remaps == 0 &&
                  c->permutes == 0;
        if (ok) {
            std::vector<SmemOp> ops;
            std::vector<char> mats;
            for (size_t i = 0; i < c->ops.size(); ++i) {
                const Prep &p = c->prep[i];
                SmemOp o{};
                o.k = p.d.k;
                o.mask = 0;
                for (int j = 0; j < p.d.k; ++j) { o.p[j] = p.d.p[j]; o.mask |= 1 << p.d.p[j]; }
                o.uoff = (int)(mats.size() / st->es);
                mats.insert(mats.end(), p.hostU.begin(), p.hostU.end());
                ops.push_back(o);
            }
            Shard &s0 = st->sh[0];
            CUDA_TRY(cudaSetDevice(s0.device));
            CUDA_TRY(cudaMalloc((void **)&c->small_ops, sizeof(SmemOp) * ops.size()));
            CUDA_TRY(cudaMalloc(&c->small_mats, mats.size()));
            CUDA_TRY(cudaMemcpy(c->small_ops, ops.data(), sizeof(SmemOp) * ops.size(), cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(c->small_mats, mats.data(), mats.size(), cudaMemcpyHostToDevice));
            c->small_nops = (int)ops.size();
            c->small_dev = s0.device;
        }
    }
    if (total == 0) return HQ_OK;
    std::vector<char> blob(total, 0);
    for (size_t i = 0; i < c->ops.size(); ++i) {
        if (c->op_uoff[i] >= 0)
            memcpy(blob.data() + c->op_uoff[i], c->prep[i].payload.data(), c->prep[i].payload.size());
        for (size_t r = 0; r < c->cuoff[i].size(); ++r)
            if (c->cuoff[i][r] >= 0)
                memcpy(blob.data() + c->cuoff[i][r], c->cprep[i][r].payload.data(), c->cprep[i][r].payload.size());
    }
    for (size_t r = 0; r < st->sh.size(); ++r) {
        Shard &s = st->sh[r];
        if (r > 0 && st->mode == MODE_VIRTUAL) { c->dev_U[r] = nullptr; continue; }
        CUDA_TRY(cudaSetDevice(s.device));
        CUDA_TRY(cudaMalloc((void **)&c->dev_U[r], total));
        CUDA_TRY(cudaMemcpy(c->dev_U[r], blob.data(), total, cudaMemcpyHostToDevice));
    }
    return HQ_OK;
}

extern "C" hq_status hq_circuit_create(hq_state *st, const hq_gate *gates, size_t ng, hq_circuit **out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !out || (!gates && ng)) return set_error(HQ_ERR_ARG, "NULL argument");
    *out = nullptr;
    std::vector<GateRef> refs;
    hq_status rc = validate_gates(st, gates, ng, refs);
    if (rc) return rc;
    hq_circuit *c = new (std::nothrow) hq_circuit();
    if (!c) return set_error(HQ_ERR_OOM, "host allocation failed");
    c->owner = st;
    if ((rc = circuit_compile(st, c, refs))) {
        hq_circuit_destroy(c);
        return rc;
    }
    *out = c;
    return HQ_OK;
    HQ_ABI_END
}

static hq_status circuit_run_ops(hq_state *st, hq_circuit *c) {
    for (size_t i = 0; i < c->ops.size(); ++i) {
        const Op &op = c->ops[i];
        hq_status rc = HQ_OK;
        if (op.kind == OP_APPLY) {
            const bool cond = !c->cprep[i].empty();
            auto get = [&](size_t r) {
                const char *base = c->dev_U[st->mode == MODE_VIRTUAL ? 0 : r];
                const long long off = cond ? c->cuoff[i][r] : c->op_uoff[i];
                const void *dU = (base && off >= 0) ? base + off : nullptr;
                return std::make_pair((const Prep *)(cond ? &c->cprep[i][r] : &c->prep[i]), dU);
            };
            Fold f = c->fold[i];
            if (f.fused) f.rem = &c->ops[i + f.consumed];
            if ((rc = run_apply(st, f, get))) return rc;
            if (st->amp_bound >= 0) st->amp_bound *= cond ? c->cgnorm[i] : c->prep[i].gnorm;
            i += f.consumed;
        } else if (op.kind == OP_GATHER) {
            rc = exec_gather(st, c->prep[i], [&](size_t r) {
                const char *base = c->dev_U[st->mode == MODE_VIRTUAL ? 0 : r];
                return (const void *)(base + c->op_uoff[i]);
            });
        } else if (op.kind == OP_REMAP) {
            rc = exec_remap(st, op);
        } else {
            rc = exec_permute(st, op);
        }
        if (rc) return rc;
    }
    return HQ_OK;
}

extern "C" hq_status hq_circuit_run(hq_state *st, hq_circuit *c) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !c) return set_error(HQ_ERR_ARG, "NULL argument");
    if (c->owner != st) return set_error(HQ_ERR_STATE, "circuit was compiled for another state");
    if (st->pi != c->pi_start)
        return set_error(HQ_ERR_STATE, "state qubit layout differs from the one the circuit was compiled for");
    hq_status rc;
    if (c->small_ops && !st->profiling) {
        Shard &s0 = st->sh[0];
        CUDA_TRY(cudaSetDevice(s0.device));
        int e = launch_circuit_smem((int)st->dtype, s0.psi, st->nl, c->small_ops, c->small_nops, c->small_mats,
                                    s0.stream);
        if (e) return set_error(HQ_ERR_CUDA, "circuit_smem launch: %s", cudaGetErrorString((cudaError_t)e));
        for (size_t i = 0; i < c->ops.size(); ++i)
            if (st->amp_bound >= 0) st->amp_bound *= c->prep[i].gnorm;
        st->stats.passes += c->passes;
        st->stats.kernel_launches += 1;
        st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
        st->pi = c->pi_end;
        return HQ_OK;
    }
    bool has_cond = false;
    for (auto &cp : c->cprep) has_cond |= !cp.empty();
    // rank-dependent (row f1) ops keep their own per-launch scales and bounds:
    // such circuits run op by op
    const bool graphable = st->sh.size() == 1 && !st->profiling && c->remaps == 0 && c->permutes == 0 &&
                           !c->ops.empty() && !has_cond;
    if (!graphable) {
        if ((rc = circuit_run_ops(st, c))) return rc;
        st->pi = c->pi_end;
        return HQ_OK;
    }
    Shard &s0 = st->sh[0];
    CUDA_TRY(cudaSetDevice(s0.device));
    bool has_tc = false;
    for (auto &p : c->prep) has_tc |= p.path == PATH_TC;
    if (has_tc && (rc = ensure_bound(st))) return rc;     // sync happens outside the capture
    const double bound0 = st->amp_bound;
    // the FP16 input scales the TC passes would use from this bound
    std::vector<int> ea;
    if (has_tc) {
        double b = bound0;
        for (size_t i = 0; i < c->ops.size(); ++i) {
            if (c->ops[i].kind != OP_APPLY) continue;
            if (c->prep[i].path == PATH_TC) {
                int ex = 0;
                std::frexp(b, &ex);
                ea.push_back(ex);
            }
            b *= c->prep[i].gnorm;
        }
    }
    if (c->graph && (c->graph_stream != s0.stream || c->graph_psi != s0.psi || c->graph_ea != ea)) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
    }
    if (!c->graph) {
        // capture: the op stream's launches on the state's stream become one graph
        if (!s0.stream) {           // the legacy default stream cannot be captured
            if ((rc = circuit_run_ops(st, c))) return rc;
            st->pi = c->pi_end;
            return HQ_OK;
        }
        const hq_stats before = st->stats;
        CUDA_TRY(cudaStreamBeginCapture(s0.stream, cudaStreamCaptureModeThreadLocal));
        rc = circuit_run_ops(st, c);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(s0.stream, &g);
        if (rc) { if (g) cudaGraphDestroy(g); return rc; }
        if (e != cudaSuccess) return set_error(HQ_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&c->graph, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) { c->graph = nullptr; return set_error(HQ_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e)); }
        c->graph_stream = s0.stream;
        c->graph_psi = s0.psi;
        c->graph_ea = ea;
        c->graph_launches = st->stats.kernel_launches - before.kernel_launches;
        st->amp_bound = bound0;     // the capture advanced it; the replay below does so again
        st->stats = before;
    }
    CUDA_TRY(cudaGraphLaunch(c->graph, s0.stream));
    for (size_t i = 0; i < c->ops.size(); ++i)
        if (c->ops[i].kind == OP_APPLY && st->amp_bound >= 0) st->amp_bound *= c->prep[i].gnorm;
    st->stats.passes += c->passes;
    st->stats.kernel_launches += c->graph_launches;
    st->stats.hbm_bytes += c->passes * (uint64_t)2 * (st->es << st->nl);
    st->pi = c->pi_end;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_circuit_info(const hq_circuit *c, uint64_t *passes, uint64_t *remaps,
                                     uint64_t *permutes) {
    HQ_ABI_BEGIN
    clear_error();
    if (!c) return set_error(HQ_ERR_ARG, "NULL circuit");
    if (passes) *passes = c->passes;
    if (remaps) *remaps = c->remaps;
    if (permutes) *permutes = c->permutes;      // standalone PERMUTE passes (folded ones excluded)
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_circuit_destroy(hq_circuit *c) {
    HQ_ABI_BEGIN
    if (!c) return HQ_OK;
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->small_ops || c->small_mats) {
        cudaSetDevice(c->small_dev);
        if (c->small_ops) cudaFree(c->small_ops);
        if (c->small_mats) cudaFree(c->small_mats);
    }
    // the owning state may already be gone (destroy order is the caller's):
    // use the devices recorded at compile time, never c->owner
    for (size_t r = 0; r < c->dev_U.size(); ++r)
        if (c->dev_U[r]) {
            cudaSetDevice(c->dev_of[r]);
            cudaFree(c->dev_U[r]);
        }
    delete c;
    cudaGetLastError();
    return HQ_OK;
    HQ_ABI_END
}

// ------------------------------------------------------------------ state I/O

static bool pi_identity(const hq_state *st) {
    for (int q = 0; q < st->n; ++q)
        if (st->pi[q] != st->n - 1 - q) return false;
    return true;
}

// physical index of logical index i
static uint64_t phys_of(const hq_state *st, uint64_t i) {
    uint64_t p = 0;
    for (int q = 0; q < st->n; ++q) p |= ((i >> (st->n - 1 - q)) & 1) << st->pi[q];
    return p;
}

extern "C" hq_status hq_state_init_basis(hq_state *st, uint64_t x) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    if (st->n < 64 && x >= (1ull << st->n)) return set_error(HQ_ERR_RANGE, "basis index out of range");
    // the whole state is overwritten: restore the chosen initial layout
    st->pi = st->pi_init;
    st->amp_bound = 1.0;
    const uint64_t p = phys_of(st, x);
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        const int64_t idx = (int)(p >> st->nl) == s.rank ? (int64_t)(p & ((1ull << st->nl) - 1)) : -1;
        int e = launch_init_basis((int)st->dtype, s.psi, 1ull << st->nl, idx, s.stream);
        if (e != cudaSuccess) return set_error(HQ_ERR_CUDA, "init launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches += idx >= 0 ? 1 : 0;
    }
    return HQ_OK;
    HQ_ABI_END
}

static hq_status range_check(const hq_state *st, uint64_t first, uint64_t count) {
    const uint64_t N = 1ull << st->n;
    if (first > N || count > N - first) return set_error(HQ_ERR_RANGE, "amplitude range outside [0, 2^n)");
    return HQ_OK;
}

static hq_status io_amplitudes(hq_state *st, uint64_t first, uint64_t count, void *host, bool get) {
    hq_status rc = range_check(st, first, count);
    if (rc) return rc;
    if (count == 0) return HQ_OK;
    const size_t es = st->es;
    const bool ident = pi_identity(st);
    std::vector<int> bitmap(st->n);
    for (int q = 0; q < st->n; ++q) bitmap[st->n - 1 - q] = st->pi[q];
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        if (ident) {
            // logical == physical: contiguous intersection with this shard
            const uint64_t lo = (uint64_t)s.rank << st->nl, hi = lo + (1ull << st->nl);
            const uint64_t a = std::max(first, lo), b = std::min(first + count, hi);
            if (a >= b) continue;
            char *h = (char *)host + (a - first) * es;
            char *d = (char *)s.psi + (a - lo) * es;
            if (get) CUDA_TRY(copy_async(st->stats, h, d, (b - a) * es, cudaMemcpyDeviceToHost, s.stream));
            else CUDA_TRY(copy_async(st->stats, d, h, (b - a) * es, cudaMemcpyHostToDevice, s.stream));
            SYNC_TRY(s);
            continue;
        }
        // general: gather/scatter through a device temp in slices
        const uint64_t slice = std::min<uint64_t>(count, 1ull << 24);
        void *tmp = nullptr;
        CUDA_TRY(cudaMalloc(&tmp, slice * es));
        std::vector<char> h(slice * es);
        for (uint64_t off = 0; off < count; off += slice) {
            const uint64_t c = std::min(slice, count - off);
            // which entries are owned by this shard
            std::vector<uint64_t> own;
            for (uint64_t j = 0; j < c; ++j)
                if ((int)(phys_of(st, first + off + j) >> st->nl) == s.rank) own.push_back(j);
            if (own.empty()) continue;
            int e;
            if (get) {
                e = launch_gather((int)st->dtype, s.psi, tmp, first + off, c, st->n, st->nl, bitmap.data(), s.rank, s.stream);
                if (e) { cudaFree(tmp); return set_error(HQ_ERR_CUDA, "gather launch failed"); }
                cudaError_t ce = copy_async(st->stats, h.data(), tmp, c * es, cudaMemcpyDeviceToHost, s.stream);
                if (!ce) ce = cudaStreamSynchronize(s.stream);
                if (ce) { cudaFree(tmp); return set_error(HQ_ERR_CUDA, "gather copy: %s", cudaGetErrorString(ce)); }
                for (uint64_t j : own) memcpy((char *)host + (off + j) * es, h.data() + j * es, es);
            } else {
                memcpy(h.data(), (const char *)host + off * es, c * es);
                cudaError_t ce = copy_async(st->stats, tmp, h.data(), c * es, cudaMemcpyHostToDevice, s.stream);
                if (ce) { cudaFree(tmp); return set_error(HQ_ERR_CUDA, "scatter copy: %s", cudaGetErrorString(ce)); }
                e = launch_scatter((int)st->dtype, s.psi, tmp, first + off, c, st->n, st->nl, bitmap.data(), s.rank, s.stream);
                if (e) { cudaFree(tmp); return set_error(HQ_ERR_CUDA, "scatter launch failed"); }
                ce = cudaStreamSynchronize(s.stream);
                if (ce) { cudaFree(tmp); return set_error(HQ_ERR_CUDA, "scatter: %s", cudaGetErrorString(ce)); }
            }
            st->stats.kernel_launches++;
        }
        cudaFree(tmp);
    }
    return HQ_OK;
}

extern "C" hq_status hq_get_amplitudes(hq_state *st, uint64_t first, uint64_t count, void *host_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || (!host_out && count)) return set_error(HQ_ERR_ARG, "NULL argument");
    return io_amplitudes(st, first, count, host_out, true);
    HQ_ABI_END
}

extern "C" hq_status hq_set_amplitudes(hq_state *st, uint64_t first, uint64_t count, const void *host_in) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || (!host_in && count)) return set_error(HQ_ERR_ARG, "NULL argument");
    st->amp_bound = -1.0;    // recomputed (hq_norm) before the next pass that needs it
    return io_amplitudes(st, first, count, const_cast<void *>(host_in), false);
    HQ_ABI_END
}

extern "C" hq_status hq_norm(hq_state *st, double *out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !out) return set_error(HQ_ERR_ARG, "NULL argument");
    double total = 0.0;
    // enqueue every shard's partial sums and their copy-back first, then
    // synchronise, so the devices of a multi-device state work concurrently
    std::vector<int> nbs(st->sh.size(), 0);
    for (size_t i = 0; i < st->sh.size(); ++i) {
        Shard &s = st->sh[i];
        CUDA_TRY(cudaSetDevice(s.device));
        int e = launch_norm_partials((int)st->dtype, s.psi, 1ull << st->nl, s.d_part, 148 * 16, s.stream, &nbs[i]);
        if (e) return set_error(HQ_ERR_CUDA, "norm launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += st->es << st->nl;
        CUDA_TRY(copy_async(st->stats, s.h_part, s.d_part, sizeof(double) * nbs[i], cudaMemcpyDeviceToHost, s.stream));
    }
    for (size_t i = 0; i < st->sh.size(); ++i) {
        Shard &s = st->sh[i];
        CUDA_TRY(cudaSetDevice(s.device));
        SYNC_TRY(s);
        double acc = 0.0;
        for (int b = 0; b < nbs[i]; ++b) acc += s.h_part[b];
        total += acc;
    }
    if (st->mode == MODE_RANK) {
        Shard &s = st->sh[0];
        s.h_part[0] = total;
        CUDA_TRY(copy_async(st->stats, s.d_part, s.h_part, sizeof(double), cudaMemcpyHostToDevice, s.stream));
        NCCL_TRY(ncclAllReduce(s.d_part, s.d_part, 1, ncclDouble, ncclSum, s.comm, s.stream));
        CUDA_TRY(copy_async(st->stats, s.h_part, s.d_part, sizeof(double), cudaMemcpyDeviceToHost, s.stream));
        SYNC_TRY(s);
        total = s.h_part[0];
    }
    *out = sqrt(total);
    st->amp_bound = *out * (1.0 + 1e-6) + 1e-300;
    return HQ_OK;
    HQ_ABI_END
}

static hq_status ensure_bound(hq_state *st) {
    if (st->amp_bound >= 0) return HQ_OK;
    double nrm = 0.0;
    return hq_norm(st, &nrm);
}

// ------------------------------------------------------------------ f4: tokens, projection, measurement

static hq_status validate_targets(const hq_state *st, const int32_t *qubits, int nq, int maxq) {
    if (!qubits || nq < 1 || nq > maxq) return set_error(HQ_ERR_ARG, "nq=%d not in [1,%d]", nq, maxq);
    for (int j = 0; j < nq; ++j) {
        if (qubits[j] < 0 || qubits[j] >= st->n) return set_error(HQ_ERR_QUBIT, "qubit %d not in [0,%d)", qubits[j], st->n);
        for (int l = 0; l < j; ++l)
            if (qubits[l] == qubits[j]) return set_error(HQ_ERR_DUP_QUBIT, "repeated qubit %d", qubits[j]);
    }
    return HQ_OK;
}

extern "C" hq_status hq_state_init_tokens(hq_state *st, const char *tokens) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !tokens) return set_error(HQ_ERR_ARG, "NULL argument");
    const size_t len = strlen(tokens);
    if (len != 1 && len != (size_t)st->n)
        return set_error(HQ_ERR_ARG, "token string has %zu characters; need 1 or n=%d", len, st->n);
    for (size_t i = 0; i < len; ++i)
        if (tokens[i] != '0' && tokens[i] != '1' && tokens[i] != '+' && tokens[i] != '-')
            return set_error(HQ_ERR_ARG, "token '%c' not in {0,1,+,-} (tensor-network-only or invalid)", tokens[i]);
    st->pi = st->pi_init;
    for (auto &s : st->sh) {
        uint64_t fix_mask = 0, fix_val = 0, minus = 0;
        int npm = 0;
        bool zero = false;
        double sign = 1.0;
        for (int q = 0; q < st->n; ++q) {
            const char t = tokens[len == 1 ? 0 : q];
            const int p = st->pi[q];
            if (p < st->nl) {
                if (t == '0' || t == '1') {
                    fix_mask |= 1ull << p;
                    if (t == '1') fix_val |= 1ull << p;
                } else {
                    ++npm;
                    if (t == '-') minus |= 1ull << p;
                }
            } else {
                const int rb = (s.rank >> (p - st->nl)) & 1;
                if (t == '0' || t == '1') zero |= rb != (t == '1');
                else {
                    ++npm;
                    if (t == '-' && rb) sign = -sign;
                }
            }
        }
        double mag = sign * std::pow(2.0, -0.5 * npm);
        if (zero) { fix_mask = 1; fix_val = 2; }      // never matches: all-zero shard
        CUDA_TRY(cudaSetDevice(s.device));
        int e = launch_init_tokens((int)st->dtype, s.psi, 1ull << st->nl, fix_mask, fix_val, minus, mag, s.stream);
        if (e) return set_error(HQ_ERR_CUDA, "init_tokens launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
    }
    st->amp_bound = 1.0 + 1e-12;
    return HQ_OK;
    HQ_ABI_END
}

// Sum `count` host doubles over the ranks (rank mode): one ncclAllReduce
// through a persistent device scratch (allocated on first use).
// Grow a shard's reduction scratch (device + pinned host) to >= cap doubles.
static hq_status ensure_red(Shard &s, size_t cap) {
    if (s.red_cap >= cap) return HQ_OK;
    if (s.d_red) cudaFree(s.d_red);
    if (s.h_red) cudaFreeHost(s.h_red);
    s.d_red = nullptr;
    s.h_red = nullptr;
    s.red_cap = 0;
    CUDA_TRY(cudaMalloc((void **)&s.d_red, sizeof(double) * cap));
    CUDA_TRY(cudaMallocHost((void **)&s.h_red, sizeof(double) * cap));
    s.red_cap = cap;
    return HQ_OK;
}

static hq_status allreduce_host(hq_state *st, double *v, int count) {
    if (st->mode != MODE_RANK) return HQ_OK;
    if (count > AR_CAP) return set_error(HQ_ERR_ARG, "internal: all-reduce of %d > %d doubles", count, AR_CAP);
    Shard &s = st->sh[0];
    CUDA_TRY(cudaSetDevice(s.device));
    if (!s.d_ar) {
        CUDA_TRY(cudaMalloc((void **)&s.d_ar, sizeof(double) * AR_CAP));
        CUDA_TRY(cudaMallocHost((void **)&s.h_ar, sizeof(double) * AR_CAP));
    }
    memcpy(s.h_ar, v, sizeof(double) * count);
    CUDA_TRY(copy_async(st->stats, s.d_ar, s.h_ar, sizeof(double) * count, cudaMemcpyHostToDevice, s.stream));
    NCCL_TRY(ncclAllReduce(s.d_ar, s.d_ar, count, ncclDouble, ncclSum, s.comm, s.stream));
    CUDA_TRY(copy_async(st->stats, s.h_ar, s.d_ar, sizeof(double) * count, cudaMemcpyDeviceToHost, s.stream));
    SYNC_TRY(s);
    memcpy(v, s.h_ar, sizeof(double) * count);
    return HQ_OK;
}

extern "C" hq_status hq_project(hq_state *st, const int32_t *qubits, const int32_t *bits, int nq,
                                int renormalize, double *norm_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !bits) return set_error(HQ_ERR_ARG, "NULL argument");
    hq_status rc = validate_targets(st, qubits, nq, st->n);
    if (rc) return rc;
    for (int j = 0; j < nq; ++j)
        if (bits[j] != 0 && bits[j] != 1) return set_error(HQ_ERR_ARG, "bits[%d]=%d not 0/1", j, bits[j]);
    double total = 0.0;
    for (auto &s : st->sh) {
        uint64_t mask = 0, val = 0;
        bool zero = false;
        for (int j = 0; j < nq; ++j) {
            const int p = st->pi[qubits[j]];
            if (p < st->nl) {
                mask |= 1ull << p;
                if (bits[j]) val |= 1ull << p;
            } else {
                zero |= ((s.rank >> (p - st->nl)) & 1) != bits[j];
            }
        }
        if (zero) { mask = 0; val = 1; }           // (i & 0) != 1: zero the shard
        CUDA_TRY(cudaSetDevice(s.device));
        int nb = 0;
        int e = launch_project((int)st->dtype, s.psi, 1ull << st->nl, mask, val, 0, s.d_part, 148 * 16, s.stream, &nb);
        if (e) return set_error(HQ_ERR_CUDA, "project launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
        CUDA_TRY(copy_async(st->stats, s.h_part, s.d_part, sizeof(double) * nb, cudaMemcpyDeviceToHost, s.stream));
        SYNC_TRY(s);
        double acc = 0.0;
        for (int b = 0; b < nb; ++b) acc += s.h_part[b];
        total += acc;
    }
    if ((rc = allreduce_host(st, &total, 1))) return rc;
    const double nrm = std::sqrt(total);
    if (norm_out) *norm_out = nrm;
    if (!renormalize) return HQ_OK;            // amp_bound unchanged: projection never grows the norm
    if (nrm < 1e-14) return set_error(HQ_ERR_RANGE, "projected norm %.3e < 1e-14 (ZeroNormProjection)", nrm);
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        int e = launch_scale((int)st->dtype, s.psi, 1ull << st->nl, 1.0 / nrm, s.stream);
        if (e) return set_error(HQ_ERR_CUDA, "scale launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
    }
    st->amp_bound = 1.0 + 1e-6;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_probabilities(hq_state *st, const int32_t *qubits, int nq, double *probs_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !probs_out) return set_error(HQ_ERR_ARG, "NULL argument");
    hq_status rc = validate_targets(st, qubits, nq, 10);
    if (rc) return rc;
    const int nout = 1 << nq;
    std::vector<double> probs(nout, 0.0);
    for (auto &s : st->sh) {
        ProbParams P;
        int loc[16], nloc = 0;      // local measured qubits, in qubits[] order
        for (int j = 0; j < nq; ++j)
            if (st->pi[qubits[j]] < st->nl) loc[nloc++] = j;
        P.nq = nloc;
        for (int t = 0; t < nloc; ++t) P.pos[t] = st->pi[qubits[loc[t]]];
        const int nb_max = 148 * 8;
        CUDA_TRY(cudaSetDevice(s.device));
        if ((rc = ensure_red(s, (size_t)nb_max << nloc))) return rc;     // persistent scratch
        int nb = 0;
        int e = launch_probabilities((int)st->dtype, s.psi, 1ull << st->nl, P, s.d_red, nb_max, s.stream, &nb);
        if (e) return set_error(HQ_ERR_CUDA, "probabilities launch: %s", cudaGetErrorString((cudaError_t)e));
        CUDA_TRY(copy_async(st->stats, s.h_red, s.d_red, sizeof(double) * ((size_t)nb << nloc),
                            cudaMemcpyDeviceToHost, s.stream));
        SYNC_TRY(s);
        const double *h = s.h_red;
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += st->es << st->nl;
        // local outcome y (bits of the local measured qubits) -> full outcome x
        int gx = 0;       // bits of global measured qubits for this shard
        for (int j = 0; j < nq; ++j) {
            const int p = st->pi[qubits[j]];
            if (p >= st->nl) gx |= ((s.rank >> (p - st->nl)) & 1) << (nq - 1 - j);
        }
        for (int y = 0; y < (1 << nloc); ++y) {
            double acc = 0.0;
            for (int b = 0; b < nb; ++b) acc += h[((size_t)b << nloc) + y];
            int x = gx;
            for (int t = 0; t < nloc; ++t)
                if ((y >> (nloc - 1 - t)) & 1) x |= 1 << (nq - 1 - loc[t]);
            probs[x] += acc;
        }
    }
    if ((rc = allreduce_host(st, probs.data(), nout))) return rc;
    for (int x = 0; x < nout; ++x) probs_out[x] = probs[x];
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_measure(hq_state *st, const int32_t *qubits, int nq, double u, uint64_t *outcome_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !outcome_out) return set_error(HQ_ERR_ARG, "NULL argument");
    if (!(u >= 0.0 && u < 1.0)) return set_error(HQ_ERR_ARG, "u=%g not in [0,1)", u);
    hq_status rc = validate_targets(st, qubits, nq, 10);
    if (rc) return rc;
    std::vector<double> p(1u << nq);
    if ((rc = hq_probabilities(st, qubits, nq, p.data()))) return rc;
    double total = 0.0;
    for (double v : p) total += v;
    if (!(total > 0.0)) return set_error(HQ_ERR_RANGE, "zero state cannot be measured");
    const double target = u * total;
    double cum = 0.0;
    int x = (int)p.size() - 1;
    for (int i = 0; i < (int)p.size(); ++i) {
        cum += p[i];
        if (target < cum && p[i] > 0.0) { x = i; break; }
    }
    while (x > 0 && p[x] == 0.0) --x;               // u at the very top: last non-zero outcome
    std::vector<int32_t> bits(nq);
    for (int j = 0; j < nq; ++j) bits[j] = (x >> (nq - 1 - j)) & 1;
    double nrm = 0.0;
    if ((rc = hq_project(st, qubits, bits.data(), nq, 1, &nrm))) return rc;
    *outcome_out = (uint64_t)x;
    return HQ_OK;
    HQ_ABI_END
}

// ------------------------------------------------------------------ f3: reduced density matrices, trajectories

// Bring every qubit of `qubits` to a local physical bit with the scheduler's
// remaps (as a gate on them would), without applying anything.
static hq_status ensure_local(hq_state *st, const int32_t *qubits, int k) {
    bool local = true;
    for (int j = 0; j < k; ++j) local &= st->pi[qubits[j]] < st->nl;
    if (local) return HQ_OK;
    std::vector<GateRef> refs(1);
    refs[0].k = k;
    refs[0].U = nullptr;
    for (int j = 0; j < k; ++j) refs[0].q[j] = qubits[j];
    std::vector<Op> ops;
    std::vector<int> pi = st->pi;
    schedule(st->n, st->m, refs, pi, ops);
    for (const Op &op : ops) {
        hq_status rc = HQ_OK;
        if (op.kind == OP_REMAP) rc = exec_remap(st, op);
        else if (op.kind == OP_PERMUTE) rc = exec_permute(st, op);
        if (rc) return rc;
    }
    st->pi = pi;
    return HQ_OK;
}

extern "C" hq_status hq_reduced_dm(hq_state *st, const int32_t *qubits, int k, double *rho_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !rho_out) return set_error(HQ_ERR_ARG, "NULL argument");
    if (k < 1 || k > 3) return set_error(HQ_ERR_K, "k=%d not in [1,3]", k);
    hq_status rc = validate_targets(st, qubits, k, 3);
    if (rc) return rc;
    if (k > st->nl) return set_error(HQ_ERR_K, "k=%d > %d local qubits", k, st->nl);
    if ((rc = ensure_local(st, qubits, k))) return rc;
    const int D = 1 << k, E = D * (D + 1) / 2;
    RdmParams P;
    P.k = k;
    int pos[3];
    for (int j = 0; j < k; ++j) pos[j] = st->pi[qubits[j]];
    for (int a = 0; a < D; ++a) {
        uint64_t o = 0;
        for (int j = 0; j < k; ++j)
            if ((a >> (k - 1 - j)) & 1) o |= 1ull << pos[j];
        P.off[a] = o;
    }
    std::sort(pos, pos + k);
    for (int j = 0; j < 3; ++j) P.pos[j] = j < k ? pos[j] : 0;
    std::vector<double> acc(2 * E, 0.0);
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        if ((rc = ensure_red(s, (size_t)RDM_MAX_BLOCKS * RDM_MAX_ENTRIES))) return rc;
        int nb = 0;
        int e = launch_reduced_dm((int)st->dtype, s.psi, 1ull << st->nl, P, s.d_red, s.stream, &nb);
        if (e) return set_error(HQ_ERR_CUDA, "reduced_dm launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
        st->stats.hbm_bytes += st->es << st->nl;
        CUDA_TRY(copy_async(st->stats, s.h_red, s.d_red, sizeof(double) * 2 * E * nb, cudaMemcpyDeviceToHost, s.stream));
        SYNC_TRY(s);
        for (int b = 0; b < nb; ++b)
            for (int x = 0; x < 2 * E; ++x) acc[x] += s.h_red[(size_t)b * 2 * E + x];
    }
    if ((rc = allreduce_host(st, acc.data(), 2 * E))) return rc;
    for (int a = 0, e = 0; a < D; ++a)
        for (int b = a; b < D; ++b, ++e) {
            rho_out[2 * (a * D + b)] = acc[2 * e];
            rho_out[2 * (a * D + b) + 1] = acc[2 * e + 1];
            rho_out[2 * (b * D + a)] = acc[2 * e];
            rho_out[2 * (b * D + a) + 1] = -acc[2 * e + 1];
        }
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_kraus_sample(hq_state *st, const double *const *K, int nkraus, const int32_t *qubits,
                                     int k, double u, int *chosen_out, double *probs_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !K || !chosen_out || nkraus < 1) return set_error(HQ_ERR_ARG, "NULL argument or no Kraus operators");
    if (!(u >= 0.0 && u < 1.0)) return set_error(HQ_ERR_ARG, "u=%g not in [0,1)", u);
    if (k < 1 || k > 3) return set_error(HQ_ERR_K, "k=%d not in [1,3]", k);
    for (int i = 0; i < nkraus; ++i)
        if (!K[i]) return set_error(HQ_ERR_ARG, "K[%d] is NULL", i);
    const int D = 1 << k;
    std::vector<double> rho((size_t)2 * D * D);
    hq_status rc = hq_reduced_dm(st, qubits, k, rho.data());
    if (rc) return rc;
    // p_i = ||K_i psi||^2 = Tr(K_i rho K_i^H) = sum_{a,b,c} K[a][b] rho[b][c] conj(K[a][c])
    std::vector<double> p(nkraus, 0.0);
    double total = 0.0;
    for (int i = 0; i < nkraus; ++i) {
        const double *A = K[i];
        double acc = 0.0;
        for (int a = 0; a < D; ++a)
            for (int b = 0; b < D; ++b) {
                const double kr = A[2 * (a * D + b)], ki = A[2 * (a * D + b) + 1];
                if (kr == 0.0 && ki == 0.0) continue;
                for (int c = 0; c < D; ++c) {
                    const double rr = rho[2 * (b * D + c)], ri = rho[2 * (b * D + c) + 1];
                    const double cr = A[2 * (a * D + c)], ci = -A[2 * (a * D + c) + 1];
                    // real part of K[a][b] * rho[b][c] * conj(K[a][c])
                    const double tr = kr * rr - ki * ri, ti = kr * ri + ki * rr;
                    acc += tr * cr - ti * ci;
                }
            }
        p[i] = std::max(acc, 0.0);
        total += p[i];
    }
    if (probs_out)
        for (int i = 0; i < nkraus; ++i) probs_out[i] = p[i];
    double pmax = 0.0;
    for (double v : p) pmax = std::max(pmax, v);
    if (!(pmax >= 1e-14)) return set_error(HQ_ERR_RANGE, "all branch probabilities < 1e-14 (ZeroNormBranch)");
    const double target = u * total;
    double cum = 0.0;
    int x = nkraus - 1;
    for (int i = 0; i < nkraus; ++i) {
        cum += p[i];
        if (target < cum && p[i] > 0.0) { x = i; break; }
    }
    while (x > 0 && p[x] == 0.0) --x;
    std::vector<double> Ks((size_t)2 * D * D);
    const double sc = 1.0 / std::sqrt(p[x]);
    for (int i = 0; i < 2 * D * D; ++i) Ks[i] = K[x][i] * sc;
    if ((rc = hq_apply_matrix(st, Ks.data(), qubits, k))) return rc;
    st->amp_bound = 1.0 + 1e-3;       // ||K_x psi|| / sqrt(p_x) = 1 up to the rounding of p_x
    *chosen_out = x;
    return HQ_OK;
    HQ_ABI_END
}

// Batched trajectories: 2^nb shots in one state, shot = logical qubits
// 0..nb-1 (they must sit on the top physical bits of a single shard), the
// system on qubits nb..n-1.
static hq_status batch_check(hq_state *st, int nb, const int32_t *qubits, int k) {
    if (st->sh.size() != 1) return set_error(HQ_ERR_STATE, "batched trajectories need a single-shard state");
    if (nb < 0 || nb > 16 || nb >= st->n) return set_error(HQ_ERR_ARG, "nb=%d not in [0, min(16, n))", nb);
    for (int q = 0; q < nb; ++q)
        if (st->pi[q] != st->n - 1 - q)
            return set_error(HQ_ERR_STATE, "batch qubit %d is not on physical bit %d (set a layout that keeps "
                                           "qubits 0..nb-1 on the top bits)", q, st->n - 1 - q);
    if (k < 1 || k > 3) return set_error(HQ_ERR_K, "k=%d not in [1,3]", k);
    hq_status rc = validate_targets(st, qubits, k, 3);
    if (rc) return rc;
    for (int j = 0; j < k; ++j)
        if (qubits[j] < nb) return set_error(HQ_ERR_QUBIT, "target %d is a batch qubit (< nb=%d)", qubits[j], nb);
    return HQ_OK;
}

static RdmParams rdm_params(const hq_state *st, const int32_t *qubits, int k) {
    RdmParams P;
    P.k = k;
    int pos[3];
    for (int j = 0; j < k; ++j) pos[j] = st->pi[qubits[j]];
    for (int a = 0; a < (1 << k); ++a) {
        uint64_t o = 0;
        for (int j = 0; j < k; ++j)
            if ((a >> (k - 1 - j)) & 1) o |= 1ull << pos[j];
        P.off[a] = o;
    }
    std::sort(pos, pos + k);
    for (int j = 0; j < 3; ++j) P.pos[j] = j < k ? pos[j] : 0;
    return P;
}

extern "C" hq_status hq_reduced_dm_batched(hq_state *st, int nb, const int32_t *qubits, int k, double *rho_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !rho_out) return set_error(HQ_ERR_ARG, "NULL argument");
    hq_status rc = batch_check(st, nb, qubits, k);
    if (rc) return rc;
    const int D = 1 << k, E = D * (D + 1) / 2, S = 1 << nb;
    const RdmParams P = rdm_params(st, qubits, k);
    Shard &s = st->sh[0];
    CUDA_TRY(cudaSetDevice(s.device));
    const size_t cap = (size_t)std::max(RDM_MAX_BLOCKS, S * 4) * RDM_MAX_ENTRIES;
    if ((rc = ensure_red(s, cap))) return rc;
    int nblk = 0;
    int e = launch_reduced_dm_batched((int)st->dtype, s.psi, 1ull << (st->n - nb), S, P, s.d_red,
                                      (int)(cap / (2 * E)), s.stream, &nblk);
    if (e) return set_error(HQ_ERR_CUDA, "reduced_dm_batched launch: %s", cudaGetErrorString((cudaError_t)e));
    st->stats.kernel_launches++;
    st->stats.hbm_bytes += st->es << st->nl;
    CUDA_TRY(copy_async(st->stats, s.h_red, s.d_red, sizeof(double) * 2 * E * nblk * S, cudaMemcpyDeviceToHost, s.stream));
    SYNC_TRY(s);
    for (int sh = 0; sh < S; ++sh) {
        double acc[2 * 36] = {0};
        for (int b = 0; b < nblk; ++b)
            for (int x = 0; x < 2 * E; ++x) acc[x] += s.h_red[((size_t)sh * nblk + b) * 2 * E + x];
        double *rho = rho_out + (size_t)sh * 2 * D * D;
        for (int a = 0, q = 0; a < D; ++a)
            for (int b = a; b < D; ++b, ++q) {
                rho[2 * (a * D + b)] = acc[2 * q];
                rho[2 * (a * D + b) + 1] = acc[2 * q + 1];
                rho[2 * (b * D + a)] = acc[2 * q];
                rho[2 * (b * D + a) + 1] = -acc[2 * q + 1];
            }
    }
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_reduced_dm_batched_sum(hq_state *st, int nb, const int32_t *qubits, int k, int nlive,
                                               double *rho_sum) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !rho_sum) return set_error(HQ_ERR_ARG, "NULL argument");
    if (nb < 0 || nb > 16 || nlive < 0 || nlive > (1 << nb)) return set_error(HQ_ERR_ARG, "nlive=%d not in [0, 2^nb]", nlive);
    if (k < 1 || k > 3) return set_error(HQ_ERR_K, "k=%d not in [1,3]", k);
    const int D = 1 << k;
    std::vector<double> rho((size_t)(1 << nb) * 2 * D * D);
    hq_status rc = hq_reduced_dm_batched(st, nb, qubits, k, rho.data());
    if (rc) return rc;
    std::vector<double> acc((size_t)2 * D * D, 0.0);
    for (int sh = 0; sh < nlive; ++sh) {
        const double *r = rho.data() + (size_t)sh * 2 * D * D;
        double tr = 0.0;
        for (int a = 0; a < D; ++a) tr += r[2 * (a * D + a)];
        if (!(tr > 0.0)) return set_error(HQ_ERR_RANGE, "shot %d: reduced density matrix has zero trace", sh);
        for (int i = 0; i < 2 * D * D; ++i) acc[i] += r[i] / tr;
    }
    for (int i = 0; i < 2 * D * D; ++i) rho_sum[i] = acc[i];
    return HQ_OK;
    HQ_ABI_END
}

// p_i = Re Tr(K_i rho K_i^H) for one shot
static double branch_weight(const double *A, const double *rho, int D) {
    double acc = 0.0;
    for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
            const double kr = A[2 * (a * D + b)], ki = A[2 * (a * D + b) + 1];
            if (kr == 0.0 && ki == 0.0) continue;
            for (int c = 0; c < D; ++c) {
                const double rr = rho[2 * (b * D + c)], ri = rho[2 * (b * D + c) + 1];
                const double cr = A[2 * (a * D + c)], ci = -A[2 * (a * D + c) + 1];
                const double tr = kr * rr - ki * ri, ti = kr * ri + ki * rr;
                acc += tr * cr - ti * ci;
            }
        }
    return std::max(acc, 0.0);
}

extern "C" hq_status hq_kraus_sample_batched(hq_state *st, int nb, const double *const *K, int nkraus,
                                             const int32_t *qubits, int k, const double *u, int32_t *chosen_out,
                                             double *probs_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !K || !u || !chosen_out || nkraus < 1) return set_error(HQ_ERR_ARG, "NULL argument or no Kraus operators");
    hq_status rc = batch_check(st, nb, qubits, k);
    if (rc) return rc;
    for (int i = 0; i < nkraus; ++i)
        if (!K[i]) return set_error(HQ_ERR_ARG, "K[%d] is NULL", i);
    const int S = 1 << nb, D = 1 << k;
    for (int sh = 0; sh < S; ++sh)
        if (!(u[sh] >= 0.0 && u[sh] < 1.0)) return set_error(HQ_ERR_ARG, "u[%d]=%g not in [0,1)", sh, u[sh]);
    std::vector<double> rho((size_t)S * 2 * D * D);
    if ((rc = hq_reduced_dm_batched(st, nb, qubits, k, rho.data()))) return rc;
    // choose every shot's branch first (all-or-nothing: no state change on error)
    std::vector<int> pick(S);
    std::vector<double> scale(S), p(nkraus);
    const double w = 1.0 / S;        // each shot keeps norm^2 1/S: the state norm stays 1
    for (int sh = 0; sh < S; ++sh) {
        double total = 0.0, pmax = 0.0;
        for (int i = 0; i < nkraus; ++i) {
            p[i] = branch_weight(K[i], rho.data() + (size_t)sh * 2 * D * D, D);
            total += p[i];
            pmax = std::max(pmax, p[i]);
        }
        if (probs_out)
            for (int i = 0; i < nkraus; ++i) probs_out[(size_t)sh * nkraus + i] = p[i];
        if (!(pmax >= 1e-14 * w)) return set_error(HQ_ERR_RANGE, "shot %d: all branch probabilities ~0 (ZeroNormBranch)", sh);
        const double target = u[sh] * total;
        double cum = 0.0;
        int x = nkraus - 1;
        for (int i = 0; i < nkraus; ++i) {
            cum += p[i];
            if (target < cum && p[i] > 0.0) { x = i; break; }
        }
        while (x > 0 && p[x] == 0.0) --x;
        pick[sh] = x;
        scale[sh] = std::sqrt(w / p[x]);
    }
    // per-shot matrices K_x * scale in the state dtype, in qubits[] index order
    Shard &s = st->sh[0];
    std::vector<char> mats((size_t)S * D * D * st->es);
    for (int sh = 0; sh < S; ++sh) {
        const double *A = K[pick[sh]];
        for (int i = 0; i < 2 * D * D; ++i) {
            const double v = A[i] * scale[sh];
            if (st->dtype == HQ_C64) reinterpret_cast<float *>(mats.data())[(size_t)sh * 2 * D * D + i] = (float)v;
            else reinterpret_cast<double *>(mats.data())[(size_t)sh * 2 * D * D + i] = v;
        }
        chosen_out[sh] = pick[sh];
    }
    void *dm = nullptr;
    if ((rc = arena_push(st, s, mats.data(), mats.size(), &dm))) return rc;
    const RdmParams P = rdm_params(st, qubits, k);
    int e = launch_apply_batched((int)st->dtype, s.psi, 1ull << st->nl, P, dm, st->n - nb, s.stream);
    if (e) return set_error(HQ_ERR_CUDA, "apply_batched launch: %s", cudaGetErrorString((cudaError_t)e));
    st->stats.passes++;
    st->stats.kernel_launches++;
    st->stats.hbm_bytes += (uint64_t)2 * (st->es << st->nl);
    st->amp_bound = 1.0 + 1e-3;
    return HQ_OK;
    HQ_ABI_END
}

// ------------------------------------------------------------------ f2: density matrices

extern "C" hq_status hq_dm_superop(const double *const *K, int nkraus, int k, double *S_out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!K || !S_out || nkraus < 1) return set_error(HQ_ERR_ARG, "NULL argument or no Kraus operators");
    if (k < 1 || k > 3) return set_error(HQ_ERR_K, "k=%d not in [1,3] (superoperator has 2k <= 6 targets)", k);
    const int d = 1 << k, D = d * d;
    for (int i = 0; i < 2 * D * D; ++i) S_out[i] = 0.0;
    for (int m = 0; m < nkraus; ++m) {
        if (!K[m]) return set_error(HQ_ERR_ARG, "K[%d] is NULL", m);
        const double *A = K[m];
        // S[(r, c), (r', c')] += A[r][r'] * conj(A[c][c'])
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c)
                for (int rp = 0; rp < d; ++rp)
                    for (int cp = 0; cp < d; ++cp) {
                        const double ar = A[2 * (r * d + rp)], ai = A[2 * (r * d + rp) + 1];
                        const double br = A[2 * (c * d + cp)], bi = -A[2 * (c * d + cp) + 1];
                        const int row = r * d + c, col = rp * d + cp;
                        S_out[2 * (row * D + col)] += ar * br - ai * bi;
                        S_out[2 * (row * D + col) + 1] += ar * bi + ai * br;
                    }
    }
    return HQ_OK;
    HQ_ABI_END
}

static hq_status dm_check(const hq_state *st, const int32_t *qubits, int k) {
    if (st->n % 2) return set_error(HQ_ERR_STATE, "density-matrix calls need an even number of qubits (n=%d)", st->n);
    const int N = st->n / 2;
    if (!qubits) return set_error(HQ_ERR_ARG, "qubits is NULL");
    for (int j = 0; j < k; ++j) {
        if (qubits[j] < 0 || qubits[j] >= N) return set_error(HQ_ERR_QUBIT, "qubit %d not in [0,%d)", qubits[j], N);
        for (int l = 0; l < j; ++l)
            if (qubits[l] == qubits[j]) return set_error(HQ_ERR_DUP_QUBIT, "repeated qubit %d", qubits[j]);
    }
    return HQ_OK;
}

extern "C" hq_status hq_dm_apply_kraus(hq_state *st, const double *const *K, int nkraus,
                                       const int32_t *qubits, int k) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    hq_status rc = dm_check(st, qubits, k);
    if (rc) return rc;
    if (k < 1 || k > 3) return set_error(HQ_ERR_K, "k=%d not in [1,3]", k);
    std::vector<double> S((size_t)2 << (4 * k));
    if ((rc = hq_dm_superop(K, nkraus, k, S.data()))) return rc;
    const int N = st->n / 2;
    int32_t q2[6];
    for (int j = 0; j < k; ++j) { q2[j] = qubits[j]; q2[k + j] = qubits[j] + N; }
    return hq_apply_matrix(st, S.data(), q2, 2 * k);
    HQ_ABI_END
}

extern "C" hq_status hq_dm_apply_unitary(hq_state *st, const double *U, const int32_t *qubits, int k) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !U) return set_error(HQ_ERR_ARG, "NULL argument");
    hq_status rc = dm_check(st, qubits, k);
    if (rc) return rc;
    if (k < 1 || k > 6) return set_error(HQ_ERR_K, "k=%d not in [1,6]", k);
    const int N = st->n / 2, d = 1 << k;
    if (k <= 3) {
        const double *K[1] = {U};
        return hq_dm_apply_kraus(st, K, 1, qubits, k);
    }
    std::vector<double> Uc((size_t)2 * d * d);
    for (int i = 0; i < d * d; ++i) { Uc[2 * i] = U[2 * i]; Uc[2 * i + 1] = -U[2 * i + 1]; }
    int32_t qc[6];
    for (int j = 0; j < k; ++j) qc[j] = qubits[j] + N;
    hq_gate g[2];
    g[0].k = k; g[1].k = k;
    for (int j = 0; j < 6; ++j) { g[0].qubits[j] = j < k ? qubits[j] : -1; g[1].qubits[j] = j < k ? qc[j] : -1; }
    g[0].U = U;
    g[1].U = Uc.data();
    return hq_apply_circuit(st, g, 2);
    HQ_ABI_END
}

extern "C" hq_status hq_dm_trace(hq_state *st, double *re, double *im) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !re || !im) return set_error(HQ_ERR_ARG, "NULL argument");
    if (st->n % 2) return set_error(HQ_ERR_STATE, "density-matrix calls need an even number of qubits");
    const int N = st->n / 2;
    DmParams P;
    for (int q = 0; q < st->n; ++q) P.bitmap[st->n - 1 - q] = st->pi[q];
    double t[2] = {0.0, 0.0};
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        int nb = 0;
        int e = launch_dm_trace((int)st->dtype, s.psi, N, st->nl, s.rank, P,
                                reinterpret_cast<double2 *>(s.d_part), 148 * 8, s.stream, &nb);
        if (e) return set_error(HQ_ERR_CUDA, "dm_trace launch: %s", cudaGetErrorString((cudaError_t)e));
        st->stats.kernel_launches++;
        CUDA_TRY(copy_async(st->stats, s.h_part, s.d_part, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, s.stream));
        SYNC_TRY(s);
        for (int b = 0; b < nb; ++b) { t[0] += s.h_part[2 * b]; t[1] += s.h_part[2 * b + 1]; }
    }
    hq_status rc = allreduce_host(st, t, 2);
    if (rc) return rc;
    *re = t[0];
    *im = t[1];
    return HQ_OK;
    HQ_ABI_END
}

// ------------------------------------------------------------------ diagnostics

extern "C" const char *hq_last_error(void) { return g_err.c_str(); }

extern "C" hq_status hq_sync(hq_state *st) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    for (auto &s : st->sh) {
        CUDA_TRY(cudaSetDevice(s.device));
        SYNC_TRY(s);
    }
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_stats_get(const hq_state *st, hq_stats *out) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st || !out) return set_error(HQ_ERR_ARG, "NULL argument");
    *out = st->stats;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_stats_reset(hq_state *st) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    st->stats = hq_stats{};
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_profile_enable(hq_state *st, int on) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    st->profiling = on != 0;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_kernel_times(hq_state *st, int path, uint64_t *count, double *total_ms,
                                     double *max_ms, uint64_t *bytes) {
    HQ_ABI_BEGIN
    clear_error();
    if (!st) return set_error(HQ_ERR_ARG, "state is NULL");
    if (path < -1 || path > 2) return set_error(HQ_ERR_ARG, "path %d not in [-1, 2]", path);
    for (auto &p : st->prof) {
        CUDA_TRY(cudaEventSynchronize(p.b));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
        ProfAcc &a = st->acc[p.path];
        a.count++;
        a.total += ms;
        a.max = std::max(a.max, (double)ms);
        a.bytes += p.bytes;
        st->sh[p.shard].ev_pool.push_back(p.a);
        st->sh[p.shard].ev_pool.push_back(p.b);
    }
    st->prof.clear();
    ProfAcc r;
    for (int i = 0; i < 3; ++i) {
        if (path >= 0 && i != path) continue;
        r.count += st->acc[i].count;
        r.total += st->acc[i].total;
        r.max = std::max(r.max, st->acc[i].max);
        r.bytes += st->acc[i].bytes;
        st->acc[i] = ProfAcc{};
    }
    if (count) *count = r.count;
    if (total_ms) *total_ms = r.total;
    if (max_ms) *max_ms = r.max;
    if (bytes) *bytes = r.bytes;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" const char *hq_version(void) { return "hq-b200 0.1 (sm_100a)"; }
