/*
 * hq.h -- C ABI of the B200-native HybridQ state-vector core.
 *
 * What it computes (the one hot path of HybridQ, arXiv 2111.06868):
 *   apply a dense, possibly fused, k-qubit gate matrix U (2^k x 2^k complex,
 *   1 <= k <= 6) to a 2^n complex amplitude vector on an arbitrary ordered
 *   set of target qubits -- the "matrix-vector multiplication of quantum
 *   states ... similar syntax of numpy.dot" of PAPER.md P:87-91, implemented
 *   there as the C++/AVX core of P:641-656 (SPEC.md S:238-246 apply_matrix,
 *   S:274-282 simulate_statevector).  Gates are fused on the host into
 *   blocks of <= kmax qubits (P:499-504 utils.compress: hq_fuse, the greedy
 *   rule of the paper's example, or hq_fuse_blocks, the block planner) before
 *   they reach the GPU.
 *
 * Conventions:
 *   - Amplitude index: qubit q is bit n-1-q (qubit 0 = most significant bit).
 *     Reading C1, pinned by the Grover listing P:403-422.
 *   - Matrices: 2*4^k doubles, interleaved (re, im), row-major; qubits[0] is
 *     the most significant bit of U's row/column index; psi' = U psi.
 *     Reading C2.  Target order matters (C3).  U need not be
 *     unitary (C4): no renormalisation happens inside apply.
 *   - Host amplitude buffers: interleaved complex in the state dtype
 *     (HQ_C64: 2 x float32, HQ_C128: 2 x float64), LOGICAL order (C14)
 *     whatever permutation the library uses internally.
 *
 * Ownership and threading:
 *   - The library owns all device memory it allocates, its streams and its
 *     NCCL communicators.  hq_state_create_from_buffers() borrows caller
 *     memory (e.g. torch tensors) that must outlive the state.
 *   - Every pointer argument is borrowed for the duration of the call only;
 *     matrices are copied (and rounded once, fp64 -> dtype, round-to-nearest)
 *     before the call returns.
 *   - Mutating calls are asynchronous and stream-ordered on the state's
 *     stream(s); hq_norm, hq_get_amplitudes, hq_sync synchronise.
 *   - A state is exclusively owned during mutation and is not thread-safe
 *     (SPEC S:295).
 *
 * Errors: every call returns hq_status; HQ_OK == 0.  No exception crosses the
 * ABI.  Arguments are validated before any device work is enqueued, so on an
 * argument error the state is unchanged.  hq_last_error() returns a
 * thread-local human-readable message for the last failing call.
 */
#ifndef HQ_H
#define HQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hq_status {
    HQ_OK = 0,
    HQ_ERR_ARG = 1,         /* NULL pointer, bad n / dtype / count / kmax        */
    HQ_ERR_NGPUS = 2,       /* ngpus not a power of two, too many, n - log2 G < 6 */
    HQ_ERR_OOM = 3,         /* device or pinned host allocation failed           */
    HQ_ERR_CUDA = 4,        /* a CUDA runtime call failed (message in last_error) */
    HQ_ERR_NCCL = 5,        /* an NCCL call failed                               */
    HQ_ERR_QUBIT = 6,       /* target qubit not in [0, n)          */
    HQ_ERR_DUP_QUBIT = 7,   /* repeated target qubit  ("distinct")    */
    HQ_ERR_K = 8,           /* k < 1, k > 6, k > local qubits, or k > kmax       */
    HQ_ERR_RANGE = 9,       /* basis index / amplitude range outside 2^n         */
    HQ_ERR_STATE = 10,      /* operation not valid for this state (e.g. mode)    */
    HQ_ERR_NO_DEVICE = 11   /* no CUDA device: the library has no CPU fallback   */
} hq_status;

typedef enum hq_dtype {
    HQ_C64 = 0,   /* complex64: FP32 storage; FP32 FMA (k<=4), 3-term FP16/TF32 tcgen05 (k=5,6) */
    HQ_C128 = 1   /* complex128: FP64 storage and FP64 FMA                            */
} hq_dtype;

/* Opaque state: the 2^n amplitudes, sharded over G = 2^m ranks on the top m
 * physical bits, plus the logical->physical qubit map pi. */
typedef struct hq_state hq_state;

/* A (possibly fused) gate: k targets, qubits[0..k-1] valid, U = 2*4^k doubles
 * (interleaved, row-major).  U is borrowed for the duration of the call. */
typedef struct hq_gate {
    int32_t k;
    int32_t qubits[6];
    const double *U;
} hq_gate;

/* A circuit uploaded once to the device(s) and replayable (compile once, run
 * many): scheduled op stream + device-resident matrices. */
typedef struct hq_circuit hq_circuit;

typedef struct hq_stats {
    uint64_t passes;          /* apply kernels launched (all shards)              */
    uint64_t remaps;          /* global<->local qubit swaps (all-to-all exchanges) */
    uint64_t permutes;        /* standalone local bit-permutation passes           */
    uint64_t kernel_launches; /* all library kernels launched on this rank         */
    uint64_t hbm_bytes;       /* algorithmic HBM bytes of those kernels (this rank) */
    uint64_t link_bytes;      /* bytes sent to peers by remaps (this rank)         */
    uint64_t h2d_bytes;       /* host->device bytes the library copied (this rank) */
    uint64_t d2h_bytes;       /* device->host bytes the library copied (this rank) */
    uint64_t packs;           /* PERMUTEs folded into an apply pass (apply+pack)   */
    uint64_t remaps_fused;    /* remaps done inside the preceding apply pass       */
    uint64_t gathers;         /* gates applied across a rank pair (GATHER ops)     */
} hq_stats;

/* ------------------------------------------------------------------ create */

/* Single-process state on ngpus devices (0..ngpus-1 of the current process).
 * ngpus = 1: the current CUDA device.  ngpus > 1: one shard per device, NCCL
 * communicator from ncclCommInitAll.  Requires ngpus a power of two <= the
 * visible device count and n - log2(ngpus) >= 6 (so any k<=6 gate can be made
 * local).  n in [1, 40].  The state is NOT initialised: call
 * hq_state_init_basis or hq_set_amplitudes.
 * Errors: HQ_ERR_ARG, HQ_ERR_NGPUS, HQ_ERR_OOM, HQ_ERR_CUDA, HQ_ERR_NCCL,
 * HQ_ERR_NO_DEVICE. */
hq_status hq_state_create(int n, hq_dtype dtype, int ngpus, hq_state **out);

/* One process per GPU (torchrun): this process holds shard `rank` of
 * `world_size` (a power of two) on CUDA device `device`.  nccl_id points to
 * the 128-byte ncclUniqueId produced by hq_nccl_unique_id() on rank 0 and
 * broadcast by the caller (e.g. torch.distributed); it may be NULL when
 * world_size == 1.  Collective: every rank must call it. */
hq_status hq_state_create_rank(int n, hq_dtype dtype, int world_size, int rank,
                               int device, const void *nccl_id, hq_state **out);

/* Writes a fresh 128-byte ncclUniqueId into out128. */
hq_status hq_nccl_unique_id(void *out128);

/* Test mode: G = nshards (power of two) "virtual" shards as separate buffers
 * on ONE device, remaps done by device-to-device copies on one stream.  Same
 * scheduler, same pi map and same kernels as the multi-GPU path; used to check
 * the distribution logic bit-exactly on a single GPU. */
hq_status hq_state_create_virtual(int n, hq_dtype dtype, int nshards, hq_state **out);

/* Borrowed-memory variant of the 1-GPU state (e.g. torch.empty buffers):
 * psi = 2^n amplitudes in dtype (16-byte aligned), stream = a cudaStream_t (or
 * NULL for the legacy default stream).  Memory must outlive the state.
 * Amplitude-bound rule (both borrowed-buffer constructors): the library keeps
 * a rigorous bound on ||psi||_2 that the complex64 tensor-core passes use to
 * scale amplitudes into the FP16 range.  It is updated by every library call
 * that writes the state.  A caller that writes the borrowed memory itself
 * (e.g. psi_t.mul_(8) or copy_ between calls) MUST call
 * hq_state_invalidate_bound (or hq_norm) before the next apply; otherwise
 * scaled amplitudes may overflow FP16 (inf/NaN results). */
hq_status hq_state_create_from_buffers(int n, hq_dtype dtype, void *psi_device,
                                       void *stream, hq_state **out);

/* Borrowed-memory variant of hq_state_create_rank (PyTorch allocates the
 * memory, the library never frees it): psi = this rank's shard of
 * 2^(n - log2 world_size) amplitudes and, for world_size > 1, buf = a receive
 * buffer of the same size (both device memory, 256-byte aligned, e.g.
 * torch.empty on the rank's device); stream = a cudaStream_t or NULL.  Remaps
 * swap the roles of psi and buf, so both must outlive the state.  Collective
 * for world_size > 1 (ncclCommInitRank).  Errors: HQ_ERR_ARG, HQ_ERR_NGPUS,
 * HQ_ERR_NCCL, HQ_ERR_CUDA. */
hq_status hq_state_create_rank_from_buffers(int n, hq_dtype dtype, int world_size, int rank,
                                            const void *nccl_id, void *psi_device, void *buf_device,
                                            void *stream, hq_state **out);

/* Qubit layout (the logical->physical bit map pi, pi[q] = physical index bit
 * of logical qubit q).  The default is pi[q] = n-1-q, i.e. physical index ==
 * logical index.  A layout is a permutation of [0, n); it changes only where
 * the amplitudes live in HBM, never what get/set_amplitudes return (always
 * logical order, C14).  hq_state_set_layout makes the given layout the one
 * hq_state_init_basis restores; the amplitudes are UNDEFINED after the call
 * until hq_state_init_basis or a full hq_set_amplitudes.  In a multi-rank
 * state every rank must set the same layout (the top log2 G physical bits are
 * the rank bits).  Errors: HQ_ERR_ARG (not a permutation). */
hq_status hq_state_set_layout(hq_state *s, const int32_t *pi);
hq_status hq_state_get_layout(const hq_state *s, int32_t *pi_out);

/* How a remap (global<->local qubit swap) moves data between ranks (mode =
 * OR of the flags; default HQ_REMAP_FUSED | HQ_REMAP_GATHER):
 *   HQ_REMAP_FUSED: when the scheduler has packed the evictees on
 *     the top local bits and the apply pass before the remap can write out
 *     of place, that pass writes every element directly into its destination
 *     rank's exchange buffer (peer memory: CUDA IPC in one-process-per-GPU
 *     states, peer access in multi-device states, the other shards' buffers
 *     for virtual shards), with a stream barrier across ranks before and
 *     after; the exchange costs no separate transfer or HBM pass.  Used only
 *     when every rank could map every peer (else the exchange path runs).
 *   HQ_REMAP_GATHER: a gate whose one global target is not needed local
 *     again within the lookahead runs as a pair gather over peer memory (each
 *     rank of the pair reads its partner's shard) instead of a remap.
 *   HQ_REMAP_EXCHANGE (0): always a separate exchange (grouped NCCL send/recv,
 *     or device copies for virtual shards) after the pass, and no gathers.
 * fused_available (may be NULL) receives 1 when peer buffers are mapped. */
#define HQ_REMAP_EXCHANGE 0
#define HQ_REMAP_FUSED 1
#define HQ_REMAP_GATHER 2
hq_status hq_state_set_remap_mode(hq_state *s, int mode, int *fused_available);

/* Forget the tracked amplitude bound (see the rule above): the next pass that
 * needs it recomputes it with one norm pass.  Never changes the amplitudes. */
hq_status hq_state_invalidate_bound(hq_state *s);

/* Frees everything the library owns.  NULL is accepted. */
hq_status hq_state_destroy(hq_state *s);

/* Replace the stream used for shard 0 of this process (caller-owned
 * cudaStream_t; must outlive its use).  Synchronises the old stream first. */
hq_status hq_state_set_stream(hq_state *s, void *stream);

/* n, dtype, world size G, ranks held by this process, first rank held. */
hq_status hq_state_info(const hq_state *s, int *n, int *dtype, int *world,
                        int *local_shards, int *first_rank);

/* ------------------------------------------------------------------ state */

/* psi = |x>: x read with qubit 0 as the most significant bit (C1).
 * x >= 2^n -> HQ_ERR_RANGE.  (SPEC S:229-236.) */
hq_status hq_state_init_basis(hq_state *s, uint64_t x);

/* Copy `count` amplitudes starting at LOGICAL index `first` into host_out
 * (interleaved, state dtype).  Synchronises.  In a multi-rank state each rank
 * writes only the amplitudes it owns and leaves the others untouched; call
 * hq_gather_amplitudes-style logic at the caller if needed.
 * Range outside [0, 2^n) -> HQ_ERR_RANGE.  (SPEC S:241.) */
hq_status hq_get_amplitudes(hq_state *s, uint64_t first, uint64_t count, void *host_out);

/* Inverse of hq_get_amplitudes: explicit-array initial state.
 * Each rank takes the amplitudes it owns from host_in. */
hq_status hq_set_amplitudes(hq_state *s, uint64_t first, uint64_t count, const void *host_in);

/* ||psi||_2 (not squared; reading C13), FP64 accumulation for both dtypes,
 * reduced over all ranks.  Synchronises.  (SPEC S:221.) */
hq_status hq_norm(hq_state *s, double *out);

/* Product initial state from tokens: a
 * NUL-terminated string of n characters over {0, 1, +, -} (character j is
 * qubit j), or a single character broadcast to every qubit (as the paper's
 * initial_state='+' benchmark).  '+' = (|0>+|1>)/sqrt2,
 * '-' = (|0>-|1>)/sqrt2.  '.' and letters are tensor-network-only tokens
 * and any other character is rejected with HQ_ERR_ARG.  Like
 * init_basis it restores the state's initial layout. */
hq_status hq_state_init_tokens(hq_state *s, const char *tokens);

/* Projection: zero every
 * amplitude whose qubit qubits[j] is not bits[j] (0/1), j < nq; if
 * renormalize, rescale to unit norm.  norm_out (may be NULL) receives the norm
 * of the projected state before renormalisation.  With renormalize and a
 * projected norm < 1e-14 the call returns HQ_ERR_RANGE (SPEC ZeroNormProjection)
 * leaving the projected, unnormalised state. */
hq_status hq_project(hq_state *s, const int32_t *qubits, const int32_t *bits, int nq,
                     int renormalize, double *norm_out);

/* Born probabilities of the 2^nq outcomes of measuring
 * qubits[0..nq) (1 <= nq <= 10): probs_out[x] = sum of |psi_i|^2 over the
 * indices whose measured qubits read x, qubits[0] the MSB of x (C1).  FP64,
 * reduced over all ranks; not normalised (the sum is ||psi||^2).  Synchronises. */
hq_status hq_probabilities(hq_state *s, const int32_t *qubits, int nq, double *probs_out);

/* Measurement: draw the outcome x from the
 * Born distribution with the caller's uniform random number u in [0, 1) (the
 * random numbers the method draws are inputs), then collapse: project onto x
 * and renormalise.  *outcome_out = x (qubits[0] = MSB). */
hq_status hq_measure(hq_state *s, const int32_t *qubits, int nq, double u, uint64_t *outcome_out);

/* ------------------------------------------------------------------ trajectories
 * Noise by pure-state sampling of the Kraus operators (PAPER P:1032-1041
 * "pure state sampling of the Kraus operators"; SURVEY row
 * f3).  Each shot owns a state; batches of shots shard across GPUs with no
 * data-path collective (paper_2111_06868_b200/trajectories.py). */

/* Reduced density matrix of qubits[0..k) (1 <= k <= 3):
 * rho[a][b] = sum_r psi[a, r] conj(psi[b, r]), a, b in [0, 2^k) with
 * qubits[0] the MSB (C1), r over the other qubits; trace = ||psi||^2.
 * rho_out: 2*4^k doubles (interleaved complex, row-major), FP64 accumulation
 * over all ranks (one read pass).  If a target is a global qubit the library
 * first remaps as hq_apply_matrix would (the layout changes, the state does
 * not).  Errors: HQ_ERR_ARG, HQ_ERR_K, HQ_ERR_QUBIT, HQ_ERR_DUP_QUBIT.
 * Synchronises. */
hq_status hq_reduced_dm(hq_state *s, const int32_t *qubits, int k, double *rho_out);

/* One trajectory step of the Kraus channel {K_i} (i < nkraus) on qubits[0..k)
 * (1 <= k <= 3), K[i] = 2*4^k doubles as U in hq_apply_matrix:
 * p_i = ||K_i psi||^2 = Tr(K_i rho_T K_i^dagger) (rho_T from hq_reduced_dm),
 * i = the first index with u * sum(p) < p_0 + ... + p_i (u in [0, 1) is the
 * caller's uniform random number), then psi <- K_i psi / sqrt(p_i) (one apply
 * pass).  *chosen_out = i; probs_out (nkraus doubles, may be NULL) = p.
 * On a multi-rank state the call is collective and every rank must pass the
 * same u (p is all-reduced, so every rank then picks the same branch).
 * Errors: HQ_ERR_RANGE if every p_i < 1e-14 (ZeroNormBranch; state
 * unchanged), else as hq_reduced_dm.  Synchronises. */
hq_status hq_kraus_sample(hq_state *s, const double *const *K, int nkraus, const int32_t *qubits, int k,
                          double u, int *chosen_out, double *probs_out);

/* Batched trajectories: 2^nb shots in ONE single-shard state.  Logical
 * qubits 0..nb-1 index the shot (they must sit on the top physical bits,
 * pi[q] = n-1-q, as in the default layout) and qubits nb..n-1 hold each shot's
 * system, so one apply pass of a gate on system qubits advances every shot.
 * 0 <= nb <= 16; targets must be system qubits.  Errors: HQ_ERR_STATE
 * (sharded state or batch qubits moved), HQ_ERR_ARG, HQ_ERR_K, HQ_ERR_QUBIT.
 *
 * hq_reduced_dm_batched: rho_out[shot] (2^nb blocks of 2*4^k doubles) = the
 * reduced density matrix of qubits[0..k) within that shot's block, unnormalised
 * (trace = the block's squared norm).  One read pass.  Synchronises.
 *
 * hq_kraus_sample_batched: one trajectory step per shot with its own uniform
 * u[shot] (same rule as hq_kraus_sample); shot s becomes
 * K_i psi_s * sqrt(2^-nb / p_i), so every block keeps squared norm 2^-nb and
 * the state norm stays 1.  chosen_out[shot] = i; probs_out (2^nb x nkraus,
 * may be NULL) = the unnormalised p_i.  One read pass + one apply pass (a
 * per-shot matrix).  HQ_ERR_RANGE if some shot has every p_i ~ 0 (state
 * unchanged).  Synchronises. */
hq_status hq_reduced_dm_batched(hq_state *s, int nb, const int32_t *qubits, int k, double *rho_out);
/* Sum over the first nlive shots of each shot's reduced density matrix
 * normalised to unit trace: rho_sum = sum_s rho_s / Tr(rho_s) (2*4^k doubles),
 * the trajectory average's numerator.  Same
 * read pass as hq_reduced_dm_batched.  HQ_ERR_RANGE if a live shot has zero
 * trace.  Synchronises. */
hq_status hq_reduced_dm_batched_sum(hq_state *s, int nb, const int32_t *qubits, int k, int nlive,
                                    double *rho_sum);
hq_status hq_kraus_sample_batched(hq_state *s, int nb, const double *const *K, int nkraus,
                                  const int32_t *qubits, int k, const double *u, int32_t *chosen_out,
                                  double *probs_out);

/* ------------------------------------------------------------------ density matrices
 * Density-matrix evolution by doubling (PAPER P:286-289 MatrixSuperGate "using
 * a matrix-vector multiplication", "a super circuit [becomes] a
 * regular circuit" on 2N qubits): an N-qubit density matrix rho
 * is the 2N-qubit state vec(rho) with vec(rho)[i 2^N + j] = rho[i][j], i.e.
 * logical qubits 0..N-1 index the rows and N..2N-1 the columns.  The state
 * must have an even number of qubits n = 2N.  Channels run through the same
 * apply kernels as any gate. */

/* Superoperator of the Kraus map rho -> sum_m K_m rho K_m^dagger on k qubits
 * (1 <= k <= 3): S = sum_m K_m (x) conj(K_m), a 2k-qubit matrix whose targets
 * are (qubits, qubits + N) in that order.  K[m] = 2*4^k doubles (interleaved,
 * row-major); S_out = 2*16^k doubles.  Host-only. */
hq_status hq_dm_superop(const double *const *K, int nkraus, int k, double *S_out);

/* rho -> U rho U^dagger on qubits[0..k) (1 <= k <= 3: one fused 2k-qubit pass;
 * 4 <= k <= 6: two passes, U on the row qubits and conj(U) on the columns). */
hq_status hq_dm_apply_unitary(hq_state *s, const double *U, const int32_t *qubits, int k);

/* rho -> sum_m K_m rho K_m^dagger on qubits[0..k), 1 <= k <= 3 (one 2k-qubit
 * superoperator pass; the channel need not be trace preserving). */
hq_status hq_dm_apply_kraus(hq_state *s, const double *const *K, int nkraus, const int32_t *qubits,
                            int k);

/* tr(rho) (complex, FP64 accumulation over the 2^N diagonal entries, all
 * ranks).  Synchronises. */
hq_status hq_dm_trace(hq_state *s, double *re, double *im);

/* ------------------------------------------------------------------ apply */

/* psi <- (U embedded on qubits) psi.
 * U: 2*4^k doubles (interleaved, row-major, qubits[0] = MSB of U's index).
 * Errors (state unchanged): HQ_ERR_ARG (NULL), HQ_ERR_K (k<1, k>6, k > n - m),
 * HQ_ERR_QUBIT, HQ_ERR_DUP_QUBIT.  If a target is a global (rank) qubit the
 * library first remaps (all-to-all) so that every target is local -- unless
 * U is block-diagonal in its global targets (exact zeros off the blocks:
 * controlled phases, CZ, ZZ, RZ and their products): then
 * every rank applies, with no communication, the block its rank bits select
 * to the local targets (a complex phase when every target is global). */
hq_status hq_apply_matrix(hq_state *s, const double *U, const int32_t *qubits, int k);

/* Apply an (already fused) gate list in order, leftmost first.
 * All gates are validated before any work is enqueued.  Remaps are scheduled
 * here with next-use (Belady) lookahead over the whole list. */
hq_status hq_apply_circuit(hq_state *s, const hq_gate *gates, size_t ngates);

/* Compile once, run many: validate + schedule + upload matrices of `gates`
 * for state s (the circuit is bound to s's layout: n, dtype, G).  Running it
 * applies exactly what hq_apply_circuit(s, gates, ngates) would. */
hq_status hq_circuit_create(hq_state *s, const hq_gate *gates, size_t ngates,
                            hq_circuit **out);
hq_status hq_circuit_run(hq_state *s, hq_circuit *c);
/* passes, remaps and local permutes in the compiled op stream. */
hq_status hq_circuit_info(const hq_circuit *c, uint64_t *passes, uint64_t *remaps,
                          uint64_t *permutes);
hq_status hq_circuit_destroy(hq_circuit *c);

/* ------------------------------------------------------------------ planner */

/* Greedy gate fusion (PAPER P:499-504 `compress` + P:493-494
 * `to_matrix_gate`; reading C7): gate g joins the earliest-created group G
 * with |supp(G) u supp(g)| <= kmax such that no non-member gate between G's
 * first member and g touches a qubit of g; otherwise it opens a new group.
 * Groups are emitted in first-member order; each fused gate acts on its
 * ascending support with U = U_last ... U_first (fp64).
 * kmax in [1, 6] and >= every input arity, else HQ_ERR_K.
 * *out is allocated by the library (free with hq_free_gates). */
hq_status hq_fuse(const hq_gate *in, size_t ngates, int kmax, hq_gate **out, size_t *nout);

/* Block planner (the paper's `compress` bounds the block size only,
 * P:499-504, so any partition into convex blocks of <= kmax qubits is the
 * same circuit): blocks are built front to back over the gate
 * DAG, each the maximal set of gates on a <= kmax-qubit set that can run as
 * one pass at that point, the set chosen by a short greedy lookahead over a
 * per-width pass-cost model (two settings on host threads, the cheaper plan
 * kept).  34q d20 at kmax = 6: 36 fused gates (hq_fuse:
 * 80).  Members of a block keep their list order; each fused gate acts on
 * its ascending support with U = U_last ... U_first (fp64).  Same
 * arguments, ownership and errors as hq_fuse. */
hq_status hq_fuse_blocks(const hq_gate *in, size_t ngates, int kmax, hq_gate **out, size_t *nout);
hq_status hq_free_gates(hq_gate *gates, size_t ngates);

/* Grouping only: group_of[i] = index (first-member order) of the fused group
 * of input gate i; *ngroups = number of groups.  group_of has ngates slots. */
hq_status hq_fuse_plan(const hq_gate *in, size_t ngates, int kmax, int32_t *group_of,
                       size_t *ngroups);

/* Host-only view of the distributed schedule (for tests): for an n-qubit
 * state on G = 2^m ranks, the op stream hq_apply_circuit would execute.
 * The stream is cut into segments, each a maximal run of gates whose
 * must-be-local qubits fit on the n - m local bits; one REMAP at each segment
 * boundary swaps the incoming globals with the local qubits of furthest next
 * use (Belady), which a PERMUTE first packs onto the top local bits (the
 * executor folds that PERMUTE into the preceding apply pass: apply+pack).
 * ops[i] = {kind, gate, nbits, bits[12]}:
 *   kind 0 APPLY  : gate index `gate`, bits[0..k-1] = physical target bits of
 *                   qubits[0..k-1]; a bit >= n - m is a global target of a
 *                   gate block-diagonal in its global targets (row f1): rank
 *                   r applies the block its rank bits select;
 *   kind 1 REMAP  : swap global bit bits[2i] with local bit bits[2i+1],
 *                   i < nbits (all-to-all among 2^nbits ranks);
 *   kind 2 PERMUTE: local bit swap bits[2i] <-> bits[2i+1], i < nbits;
 *   kind 3 GATHER : gate `gate` with bits as for APPLY, exactly one of them
 *                   global and not block-diagonal: the rank pair that differs
 *                   in it computes the gate over peer memory (row f1), no
 *                   remap; only with flags & HQ_SCHED_GATHER (the executor
 *                   asks for it when peer buffers are mapped).
 * pi_out (n entries, may be NULL) receives the final logical->physical map. */
typedef struct hq_op {
    int32_t kind;
    int32_t gate;
    int32_t nbits;
    int32_t bits[12];
} hq_op;
hq_status hq_schedule(int n, int m, const hq_gate *gates, size_t ngates,
                      hq_op **ops, size_t *nops, int32_t *pi_out);
/* The same from a given initial layout pi_in (n entries, a permutation; e.g.
 * hq_plan_layout's; NULL = default), as a state with that layout would execute
 * it; flags: HQ_SCHED_GATHER allows GATHER ops for isolated global accesses. */
#define HQ_SCHED_GATHER 1
hq_status hq_schedule_from(int n, int m, const hq_gate *gates, size_t ngates, const int32_t *pi_in,
                           int flags, hq_op **ops, size_t *nops, int32_t *pi_out);
hq_status hq_free_ops(hq_op *ops);
/* Host-only: the transfers a REMAP op makes for `rank` of an n-qubit state on
 * 2^m ranks, exactly as the executor issues them (grouped NCCL send/recv, or
 * device copies): transfer i sends amplitudes [off_out[i], off_out[i] +
 * len_out[i]) of this rank's shard to rank peer_out[i] and receives that
 * peer's run into the same range of the exchange buffer (peer == rank: a
 * local copy).  *count receives the number of transfers; with cap < count
 * (or NULL arrays) only *count is written (HQ_ERR_RANGE if the arrays are
 * given but too small).  Used by the multi-process CPU test. */
hq_status hq_remap_plan(int n, int m, const hq_op *op, int rank, int32_t *peer_out, uint64_t *off_out,
                        uint64_t *len_out, size_t cap, size_t *count);

/* Layout planner (the GPU counterpart of the paper's "qubits are swapped to
 * fully exploit AVX instructions"): a local search over the
 * logical->physical map of the n-m local qubits that lowers the summed
 * estimated pass cost of `gates` for dtype (HQ_C64 / HQ_C128).  The cost model
 * penalises targets in the warp-lane bits of the
 * SIMT kernel and tensor-core gathers spanning more than 16 8-MB regions.
 * With m > 0 it also picks the m qubits that start global: those outside the
 * first segment of the distributed schedule with the furthest next use, so
 * the first segment needs no remap.
 * pi_out receives n entries; cost_before / cost_after (may be NULL) the
 * model's totals for the default and the returned layout. */
hq_status hq_plan_layout(int n, int m, int dtype, const hq_gate *gates, size_t ngates,
                         int32_t *pi_out, double *cost_before, double *cost_after);

/* ------------------------------------------------------------------ diagnostics */

/* Thread-local message for the last failing call on this thread ("" if none). */
const char *hq_last_error(void);
/* Block until all work enqueued on the state's streams has completed. */
hq_status hq_sync(hq_state *s);
hq_status hq_stats_get(const hq_state *s, hq_stats *out);
hq_status hq_stats_reset(hq_state *s);
/* Per-launch timing of apply kernels with CUDA events on the launching
 * stream (off by default).  hq_kernel_times synchronises and returns, for the
 * launches of kernel family `path` since profiling was enabled / that path was
 * last read: count, total and max milliseconds, and algorithmic bytes
 * (2 x shard bytes per pass).  path: -1 all apply kernels, 0 SIMT register
 * kernel (apply_reg), 1 generic kernel (apply_gen), 2 tensor-core kernel
 * (apply_tc). */
hq_status hq_profile_enable(hq_state *s, int on);
hq_status hq_kernel_times(hq_state *s, int path, uint64_t *count, double *total_ms,
                          double *max_ms, uint64_t *bytes);
/* Library version string. */
const char *hq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HQ_H */
