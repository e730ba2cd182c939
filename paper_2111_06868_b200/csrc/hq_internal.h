// Internal declarations shared by the host runtime (.cpp) and the kernels (.cu).
// Product code only: nothing here is shared with oracle/.
#pragma once

#include <atomic>
#include <exception>
#include <new>
#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "hq.h"

namespace hq {

// ------------------------------------------------------------------ errors
hq_status set_error(hq_status st, const char *fmt, ...);

// Every C ABI entry point runs inside this guard: an exception (a host
// allocation failure in a std container, or anything else) never crosses the
// extern "C" boundary; it becomes an hq_status with a message.
#define HQ_ABI_BEGIN try {
#define HQ_ABI_END                                                                   \
    }                                                                                \
    catch (const std::bad_alloc &) {                                                 \
        return ::hq::set_error(HQ_ERR_OOM, "host allocation failed");                \
    }                                                                                \
    catch (const std::exception &e_) {                                               \
        return ::hq::set_error(HQ_ERR_STATE, "internal error: %s", e_.what());       \
    }                                                                                \
    catch (...) {                                                                    \
        return ::hq::set_error(HQ_ERR_STATE, "internal error");                      \
    }
void clear_error();

// ------------------------------------------------------------------ launch helpers
// The dynamic shared-memory limit of a kernel is a per-device setting: raise
// it once per (kernel, device), tracked in a per-kernel device bitmask (a
// multi-device state launches the same kernel on several devices).
template <class Kern>
inline cudaError_t smem_attr_once(Kern kernel, int bytes, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// ------------------------------------------------------------------ planner (hq_plan.cpp)
struct GateRef {            // validated view of an hq_gate
    int k;
    int q[6];
    const double *U;        // 2*4^k doubles
};

// Greedy fusion (reading C7).  group_of[i] = group index in first-member order.
// Returns number of groups.
size_t fuse_groups(const std::vector<GateRef> &g, int kmax, std::vector<int32_t> &group_of);

// Build fused gates: ascending support, U = U_last...U_first (fp64, interleaved).
struct FusedGate {
    int k;
    int q[6];
    std::vector<double> U;  // 2*4^k
};
void fuse_build(const std::vector<GateRef> &g, int kmax, std::vector<FusedGate> &out, bool blocks = false);

// Distributed schedule (hq_schedule semantics).  pi: logical->physical, in/out.
enum OpKind { OP_APPLY = 0, OP_REMAP = 1, OP_PERMUTE = 2, OP_GATHER = 3 };
struct Op {
    int kind;
    int gate;
    int nbits;
    int bits[12];
};
// APPLY ops may carry global target bits (>= n - m): the scheduler emits them
// only for gates block-diagonal in those targets (block_diag_in), and rank r
// applies the block selected by its rank bits to the local targets (row f1).
// gather = true: a gate that needs exactly one global qubit local, which no
// gate in the lookahead window needs again, runs as OP_GATHER (pair gather
// over peer memory, no remap) instead of triggering a remap.
void schedule(int n, int m, const std::vector<GateRef> &g, std::vector<int> &pi,
              std::vector<Op> &ops, bool gather = false);
// Lowest physical bit a scheduler PERMUTE (pack) may move: bits 0 and 1 stay in
// place so that every apply+pack write still fills whole 32-byte sectors.
constexpr int PACK_MIN_BIT = 2;
// OP_GATHER only when the global qubit's next local need is further than this
// many gates away (or never): then bringing it in by a remap would buy nothing
constexpr int GATHER_LOOKAHEAD = 32;
bool block_diag_in(const double *U, int k, int umask);
uint64_t local_need(const GateRef &gt);

// Layout planner: logical->physical map of the local qubits minimising the
// estimated pass cost of `g` (hq_plan_layout).
double layout_pass_cost(int dtype, int k, const int *bits);
void plan_layout(int n, int m, int dtype, const std::vector<GateRef> &g, std::vector<int> &pi);

// ------------------------------------------------------------------ kernels (hq_apply.cu)
// Target description handed to the kernel launchers: k physical bit
// positions in CANONICAL order (ascending), and U already permuted so that
// U-index bit i <-> canonical target i (LSB first).  U in the state dtype.
struct ApplyDesc {
    int k;
    int p[6];               // ascending physical bit positions (< n_local)
    int n_local;
};

// Out-of-place output of an apply pass (apply+pack): the
// amplitude computed for input index x is written at output index
//   y = x with the bit pairs (pa[i], pb[i]) exchanged,
//   t = (y >> tsh) & tmask            (selects the output buffer dst[t]),
//   dst[t][(y & ~(tmask << tsh)) | add].
// apply+pack alone: one buffer (tmask = 0, add = 0).  The kernels take the
// positions in their own index units (amplitudes, or 16-byte vectors for the
// complex64 SIMT kernel).  active = 0: in place.
struct OutMap {
    uint64_t dst[8];
    uint64_t add;
    int active;
    int npairs;
    int pa[6], pb[6];
    int tsh;
    uint32_t tmask;
};

__host__ __device__ inline uint64_t om_swap(uint64_t x, const OutMap &m) {
    for (int i = 0; i < m.npairs; ++i) {
        const uint64_t d = ((x >> m.pa[i]) ^ (x >> m.pb[i])) & 1;
        x ^= (d << m.pa[i]) | (d << m.pb[i]);
    }
    return x;
}

// Host description of an out-of-place output (amplitude bit positions).
struct OutSpec {
    bool active = false;
    int npairs = 0;
    int pa[6] = {0}, pb[6] = {0};
    int tsh = 0;
    uint32_t tmask = 0;
    void *dst[8] = {nullptr};
    uint64_t add = 0;
};

// Device-side matrix: U in dtype, row-major, interleaved, 4^k complex.
// host_U (dtype, same layout) is also given so small matrices travel in the
// kernel's parameter space; dev_U may be null if host path suffices.
struct KernelStatus {
    int launches;
};

// Launch one apply pass on `psi` (2^n_local amplitudes).  Returns cudaError_t
// as int.  stream is a cudaStream_t.
int launch_apply(int dtype, void *psi, const ApplyDesc &d, const void *host_U,
                 const void *dev_U, void *stream, int *launches, const OutSpec *out = nullptr);
// Pair gather (OP_GATHER, row f1): a gate whose canonical target k-1 is a
// global (rank) bit, applied on the rank pair that differs in it.  Each rank
// reads its own shard and its partner's (peer memory) and writes its half of
// the outputs, rows with canonical bit k-1 = half, into dst (out of place).
// d: the k-1 local targets (canonical, ascending); dev_U: canonical D x D.
int launch_pair_gather(int dtype, const void *psi_me, const void *psi_peer, void *dst, const ApplyDesc &d,
                       int half, const void *dev_U, void *stream);

// Whether launch_apply can write this pass out of place through an OutSpec
// (every kernel but the complex128 k = 5, 6 tile kernel).
bool apply_supports_out(int dtype, const ApplyDesc &d, const OutSpec &o);

// Whether launch_apply needs dev_U (true when U cannot travel as a kernel
// parameter for this (dtype, k, placement)).
bool apply_needs_dev_U(int dtype, const ApplyDesc &d);

// Whole compiled circuit in one CTA with the shard resident in shared memory
// (n_local <= 12 for c64, <= 11 for c128).  ops[i]: k canonical targets at
// ascending physical bits p[], mask = OR of their bits, U at mats + uoff
// (canonical D x D, state dtype).
struct SmemOp {
    int k;
    int p[6];
    int mask;
    int uoff;              // in complex elements
};
constexpr int SMEM_CIRCUIT_MAX_NL_C64 = 12;
constexpr int SMEM_CIRCUIT_MAX_NL_C128 = 11;
int launch_circuit_smem(int dtype, void *psi, int nl, const SmemOp *dev_ops, int nops, const void *dev_mats,
                        void *stream);

// tcgen05 tensor-core path (hq_tc.cu): complex64, k = 5 or 6 (5 is widened to
// 6 exactly as U (x) I).  tc_prepare builds the device payload (real-embedded
// A hi/lo, 128 KB) and the kernel parameter block from the canonical fp64 U.
bool tc_applicable(int dtype, const ApplyDesc &d);
void tc_prepare(const ApplyDesc &d, const double *Ucanon, std::vector<char> &payload,
                std::vector<char> &params);
int tc_launch(void *psi, const void *params, size_t params_size, const void *dev_payload,
              void *stream);
// Fill the output-map tables of a tensor-core parameter block (apply+pack);
// returns false when this block cannot write out of place with that map.
bool tc_set_output(std::vector<char> &params, const OutSpec &o);
// Set the FP16 input scale of a mode-H parameter block from a rigorous upper
// bound on max |amplitude| of the state the pass will read.
void tc_set_amp_bound(std::vector<char> &params, double bound);

// psi = 0, then psi[idx] = 1 if idx >= 0.
int launch_init_basis(int dtype, void *psi, uint64_t n_amps, int64_t idx, void *stream);
// partial sums of |psi|^2 into dev_partial[0..nblocks), returns nblocks used.
int launch_norm_partials(int dtype, const void *psi, uint64_t n_amps, double *dev_partial,
                         int max_blocks, void *stream, int *nblocks_out);
// out-of-place local bit permutation: dst[perm(x)] = src[x] where perm swaps
// bit a[i] <-> b[i] for i < npairs.
int launch_permute(int dtype, const void *src, void *dst, uint64_t n_amps, int npairs,
                   const int *a, const int *b, void *stream);
// gather: dst[j] = psi[phys(first + j)] for the amplitudes this shard owns;
// phys() maps logical index -> physical index by the bit map `bitmap`
// (bitmap[logical_bit] = physical_bit, n entries), returns only those with
// rank == my_rank (others left untouched in dst, mask written as 0/1).
int launch_gather(int dtype, const void *psi, void *dst, uint64_t first, uint64_t count,
                  int n, int n_local, const int *bitmap, int my_rank, void *stream);
int launch_scatter(int dtype, void *psi, const void *src, uint64_t first, uint64_t count,
                   int n, int n_local, const int *bitmap, int my_rank, void *stream);

// ------------------------------------------------------------------ state ops (hq_state_ops.cu)
struct ProbParams {
    int nq;
    int pos[16];            // physical bit of outcome bit nq-1-j (pos[0] = MSB of x)
};
int launch_init_tokens(int dtype, void *psi, uint64_t n_amps, uint64_t fix_mask, uint64_t fix_val,
                       uint64_t minus_mask, double mag, void *stream);
int launch_project(int dtype, void *psi, uint64_t n_amps, uint64_t mask, uint64_t val, int keep_all,
                   double *dev_partial, int max_blocks, void *stream, int *nblocks_out);
int launch_scale(int dtype, void *psi, uint64_t n_amps, double s, void *stream);
int launch_scale_complex(int dtype, void *psi, uint64_t n_amps, double re, double im, void *stream);
int launch_probabilities(int dtype, const void *psi, uint64_t n_amps, const ProbParams &P,
                         double *dev_hist, int max_blocks, void *stream, int *nblocks_out);
struct DmParams {
    int bitmap[64];          // logical index bit -> physical bit
};
int launch_dm_trace(int dtype, const void *psi, int N, int n_local, int rank, const DmParams &P,
                    double2 *dev_part, int max_blocks, void *stream, int *nblocks_out);
// Reduced density matrix of k <= 3 local targets (row-major upper triangle,
// entry e of (a, b >= a) in row order; a's MSB = qubits[0]).
struct RdmParams {
    uint64_t off[8];         // amplitude offset of target pattern a
    int pos[3];              // ascending physical bits of the targets
    int k;
};
constexpr int RDM_MAX_BLOCKS = 148 * 4;
constexpr int RDM_MAX_ENTRIES = 2 * 36;  // doubles per block partial (k = 3)
int launch_reduced_dm(int dtype, const void *psi, uint64_t n_amps, const RdmParams &P, double *dev_part,
                      void *stream, int *nblocks_out);
// Batched trajectories (shots along the top physical bits): per-shot reduced
// density matrices (partials [shot][block][2E], blocks <= max_parts / nshots,
// <= 64) and a per-shot matrix apply (mats[shot], D x D in the state dtype).
int launch_reduced_dm_batched(int dtype, const void *psi, uint64_t shot_amps, int nshots, const RdmParams &P,
                              double *dev_part, int max_parts, void *stream, int *nblocks_out);
int launch_apply_batched(int dtype, void *psi, uint64_t n_amps, const RdmParams &P, const void *dev_mats,
                         int sys_bits, void *stream);

}  // namespace hq
