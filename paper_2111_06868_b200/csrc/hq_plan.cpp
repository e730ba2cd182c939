// Host planner: greedy gate fusion and the distributed (global-qubit) schedule.
//
// Fusion follows PAPER.md P:499-504 (utils.compress: "Compress gates in
// circuit so that gates in the new circuit will not have more than
// max_n_qubits qubits ... larger gates may better exploit vectorization") and
// P:493-494 (to_matrix_gate), with the grouping rule of DESIGN.md reading C7
// (SPEC S:166-174 made sound):  gate g joins the earliest-created group G
// with |supp(G) u supp(g)| <= kmax such that no non-member gate between G's
// first member and g touches a qubit of g; otherwise it opens a new group.
// Worked example: P:510-529 (supports (0,1,2),(0,3,4),(1,3,4),(2,3,4)).
//
// The schedule implements the state-vector distribution the paper only
// plans: amplitudes are sharded on the top m physical
// bits; a gate with a global target is preceded by a REMAP that swaps global
// bits with the top local bits (an all-to-all), choosing which logical qubits
// to evict by furthest next use (Belady).  The paper's own idea is the same
// swap applied to the least-significant qubits for AVX.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <vector>
#include <limits>
#include <new>
#include <thread>
#include <system_error>
#include <exception>

#include "hq_internal.h"

namespace hq {

static inline uint64_t qmask(const GateRef &g) {
    uint64_t m = 0;
    for (int j = 0; j < g.k; ++j) m |= 1ull << g.q[j];
    return m;
}

size_t fuse_groups(const std::vector<GateRef> &g, int kmax, std::vector<int32_t> &group_of) {
    const size_t N = g.size();
    group_of.assign(N, -1);
    struct Group { size_t first; uint64_t support; };
    std::vector<Group> groups;
    // history[q] = indices of gates touching qubit q, ascending
    std::vector<std::vector<uint32_t>> history(64);
    for (size_t i = 0; i < N; ++i) {
        const uint64_t Q = qmask(g[i]);
        int chosen = -1;
        for (size_t G = 0; G < groups.size() && chosen < 0; ++G) {
            if (__builtin_popcountll(groups[G].support | Q) > kmax) continue;
            bool blocked = false;
            for (int j = 0; j < g[i].k && !blocked; ++j) {
                const auto &h = history[g[i].q[j]];
                // walk back over gates touching this qubit that come after G.first
                for (size_t t = h.size(); t-- > 0;) {
                    if (h[t] <= groups[G].first) break;
                    if (group_of[h[t]] != (int32_t)G) { blocked = true; break; }
                }
            }
            if (!blocked) chosen = (int)G;
        }
        if (chosen < 0) {
            chosen = (int)groups.size();
            groups.push_back({i, 0});
        }
        groups[chosen].support |= Q;
        group_of[i] = chosen;
        for (int j = 0; j < g[i].k; ++j) history[g[i].q[j]].push_back((uint32_t)i);
    }
    return groups.size();
}

// Embed member U (on qubits q, k) into the m-qubit ascending support `sup`:
// E[i][i'] = U[r(i)][r(i')] if i, i' agree off the member's bits, else 0,
// with support position j <-> index bit m-1-j (qubit order of C1 restricted
// to the support).  Then M <- E * M.
static void left_multiply_embedded(std::vector<double> &M, int m, const int *sup,
                                   const GateRef &gt) {
    const int D = 1 << m;
    int bitpos[6];
    for (int j = 0; j < gt.k; ++j) {
        int pos = -1;
        for (int s = 0; s < m; ++s) if (sup[s] == gt.q[j]) pos = s;
        bitpos[j] = m - 1 - pos;
    }
    uint32_t mask = 0;
    for (int j = 0; j < gt.k; ++j) mask |= 1u << bitpos[j];
    const int d = 1 << gt.k;
    std::vector<int> r(D);
    for (int i = 0; i < D; ++i) {
        int v = 0;
        for (int j = 0; j < gt.k; ++j) v |= ((i >> bitpos[j]) & 1) << (gt.k - 1 - j);
        r[i] = v;
    }
    std::vector<double> out((size_t)2 * D * D, 0.0);
    // out = E * M;  E[i][l] nonzero only when (i & ~mask) == (l & ~mask)
    for (int i = 0; i < D; ++i) {
        const int rest = i & ~mask;
        for (int c = 0; c < d; ++c) {
            // l = rest with member bits set from c
            int l = rest;
            for (int j = 0; j < gt.k; ++j)
                if ((c >> (gt.k - 1 - j)) & 1) l |= 1 << bitpos[j];
            const double er = gt.U[2 * (r[i] * d + r[l])];
            const double ei = gt.U[2 * (r[i] * d + r[l]) + 1];
            if (er == 0.0 && ei == 0.0) continue;
            const double *Ml = &M[(size_t)2 * l * D];
            double *Oi = &out[(size_t)2 * i * D];
            for (int col = 0; col < D; ++col) {
                const double mr = Ml[2 * col], mi = Ml[2 * col + 1];
                Oi[2 * col] += er * mr - ei * mi;
                Oi[2 * col + 1] += er * mi + ei * mr;
            }
        }
    }
    M.swap(out);
}

// Block planner (hq_fuse_blocks).  The paper's `compress` only bounds the
// block size; any partition of the gate list into convex blocks
// of <= kmax qubits computes the same circuit.  This planner builds the
// blocks front to back over the gate DAG (wire order = the list order):
//
// * frontier: ptr[q] = first gate on wire q not yet in a block; a gate is
//   ready when it is first on every one of its wires;
// * grow(S): the maximal block on qubit set S from the frontier = repeatedly
//   take any gate whose qubits are all in S and which is first on all of its
//   wires (all its predecessors are earlier blocks or this block), so the
//   block can run as one pass at this point of the list;
// * candidates: for every ready gate, S starts as its qubits and grows one
//   qubit at a time (the qubit, among those of the next LOOK gates on S's
//   wires, whose addition absorbs the most gates; lowest qubit on ties) up
//   to kmax; the candidate is the absorbed block, on its own support; equal
//   supports are one candidate; candidates are ranked by gates absorbed;
// * choice: each of the best WIDTH candidates is followed by HORIZON greedy
//   blocks (always the best-ranked candidate) and scored by modelled pass
//   cost per gate absorbed over that window (pass cost by block width:
//   the measured sustained complex64 pass times on one B200, relative to a
//   1-2 qubit pass); the lowest score wins (first on ties).
//   The WIDTH rollouts run on parallel host threads.
//
// Two settings run side by side, (LOOK, WIDTH, HORIZON) = (4, 6, 8) and
// (6, 3, 16); the cheaper plan under the same cost model is returned (the
// first on ties), or the C7 plan when that is cheaper still.  On the 34q
// d20 benchmark circuit at kmax = 6 this gives 36 blocks where the C7
// greedy gives 80 (30q d20: 33, 36q d24: 42).  Members are emitted in list
// order (a topological order of the block); blocks in the order they were
// built.
namespace {
struct BlkSetting { int look, width, horizon; };
constexpr BlkSetting BLK_SETTINGS[2] = {{4, 6, 8}, {6, 3, 16}};
constexpr double BLK_COST[7] = {0.0, 1.0, 1.0, 1.06, 1.15, 1.13, 1.24};

struct Frontier {
    const std::vector<GateRef> &g;
    std::vector<std::vector<uint32_t>> wire;       // gates on each qubit, list order
    explicit Frontier(const std::vector<GateRef> &gates) : g(gates), wire(64) {
        for (size_t i = 0; i < g.size(); ++i)
            for (int j = 0; j < g[i].k; ++j) wire[g[i].q[j]].push_back((uint32_t)i);
    }
    bool first_on_all(const std::vector<uint32_t> &p, uint32_t gi, uint64_t S) const {
        for (int j = 0; j < g[gi].k; ++j) {
            const int x = g[gi].q[j];
            if (!((S >> x) & 1) || p[x] >= wire[x].size() || wire[x][p[x]] != gi) return false;
        }
        return true;
    }
    // the maximal block on S from p (p advanced past it); gates absorbed,
    // their support and (optionally) their indices
    size_t grow(std::vector<uint32_t> &p, uint64_t S, uint64_t *supp, std::vector<uint32_t> *blk) const {
        size_t cnt = 0;
        uint64_t su = 0;
        for (bool changed = true; changed;) {
            changed = false;
            for (uint64_t m = S; m; m &= m - 1) {
                const int q = __builtin_ctzll(m);
                while (p[q] < wire[q].size()) {
                    const uint32_t gi = wire[q][p[q]];
                    if (!first_on_all(p, gi, S)) break;
                    for (int j = 0; j < g[gi].k; ++j) {
                        p[g[gi].q[j]]++;
                        su |= 1ull << g[gi].q[j];
                    }
                    if (blk) blk->push_back(gi);
                    ++cnt;
                    changed = true;
                }
            }
        }
        if (supp) *supp = su;
        return cnt;
    }
    struct Cand { size_t cnt; uint64_t supp; };
    std::vector<Cand> candidates(const std::vector<uint32_t> &ptr, int kmax, int look) const {
        std::vector<Cand> out;
        std::vector<uint32_t> p;
        for (int q = 0; q < 64; ++q) {
            if (ptr[q] >= wire[q].size()) continue;
            const uint32_t gi = wire[q][ptr[q]];
            uint64_t S = 0;
            for (int j = 0; j < g[gi].k; ++j) S |= 1ull << g[gi].q[j];
            if (__builtin_ctzll(S) != q || !first_on_all(ptr, gi, S)) continue;     // each ready gate once
            p = ptr;
            size_t cnt = grow(p, S, nullptr, nullptr);
            while (__builtin_popcountll(S) < kmax) {
                uint64_t cand = 0;
                for (uint64_t m = S; m; m &= m - 1) {
                    const int x = __builtin_ctzll(m);
                    const auto &w = wire[x];
                    for (size_t t = ptr[x]; t < w.size() && t < ptr[x] + (size_t)look; ++t)
                        for (int j = 0; j < g[w[t]].k; ++j) cand |= 1ull << g[w[t]].q[j];
                }
                cand &= ~S;
                if (!cand) break;
                int best = -1;
                size_t bc = 0;
                for (uint64_t m = cand; m; m &= m - 1) {
                    const int c = __builtin_ctzll(m);
                    p = ptr;
                    const size_t n2 = grow(p, S | (1ull << c), nullptr, nullptr);
                    if (best < 0 || n2 > bc) { best = c; bc = n2; }
                }
                S |= 1ull << best;
                cnt = bc;
            }
            p = ptr;
            uint64_t supp = 0;
            grow(p, S, &supp, nullptr);
            bool dup = false;
            for (const Cand &c : out) dup |= c.supp == supp;
            if (!dup) out.push_back({cnt, supp});
        }
        std::stable_sort(out.begin(), out.end(), [](const Cand &a, const Cand &b) { return a.cnt > b.cnt; });
        return out;
    }
    bool done(const std::vector<uint32_t> &p) const {
        for (int q = 0; q < 64; ++q) if (p[q] < wire[q].size()) return false;
        return true;
    }
};
}  // namespace

// f(0) .. f(n - 1) on host threads (f(0) on the caller's); a thread that
// cannot be created runs its share on the caller's thread instead.  An
// exception thrown by any f(i) (std::bad_alloc) is rethrown on the caller's
// thread after every thread has joined.
template <class F>
static void run_parallel(size_t n, F &&f) {
    std::vector<std::exception_ptr> err(n);
    auto guarded = [&](size_t i) {
        try {
            f(i);
        } catch (...) {
            err[i] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    std::vector<size_t> inline_idx;
    for (size_t i = 1; i < n; ++i) {
        try {
            th.emplace_back(guarded, i);
        } catch (const std::system_error &) {
            inline_idx.push_back(i);
        }
    }
    guarded(0);
    for (size_t i : inline_idx) guarded(i);
    for (auto &t : th) t.join();
    for (auto &e : err)
        if (e) std::rethrow_exception(e);
}

static std::vector<std::vector<size_t>> frontier_blocks(const std::vector<GateRef> &g, int kmax,
                                                        const BlkSetting &cfg) {
    Frontier F(g);
    std::vector<uint32_t> ptr(64, 0);
    std::vector<std::vector<size_t>> order;
    std::vector<uint32_t> blk;
    while (!F.done(ptr)) {
        const auto cs = F.candidates(ptr, kmax, cfg.look);
        size_t pick = 0;
        const size_t nw = std::min(cs.size(), (size_t)cfg.width);
        if (nw > 1) {
            // rollout c: candidate c, then HORIZON greedy blocks; cost per gate
            std::vector<double> score(nw);
            auto rollout = [&](size_t c) {
                std::vector<uint32_t> p2 = ptr;
                F.grow(p2, cs[c].supp, nullptr, nullptr);
                double cost = BLK_COST[__builtin_popcountll(cs[c].supp)];
                size_t gates = cs[c].cnt;
                for (int h = 0; h < cfg.horizon && !F.done(p2); ++h) {
                    const auto nx = F.candidates(p2, kmax, cfg.look);
                    F.grow(p2, nx[0].supp, nullptr, nullptr);
                    cost += BLK_COST[__builtin_popcountll(nx[0].supp)];
                    gates += nx[0].cnt;
                }
                score[c] = cost / (double)gates;
            };
            run_parallel(nw, rollout);
            double best = std::numeric_limits<double>::infinity();
            for (size_t c = 0; c < nw; ++c)
                if (score[c] < best - 1e-12) { best = score[c]; pick = c; }
        }
        blk.clear();
        F.grow(ptr, cs[pick].supp, nullptr, &blk);
        std::sort(blk.begin(), blk.end());
        order.emplace_back(blk.begin(), blk.end());
    }
    return order;
}

void fuse_build(const std::vector<GateRef> &g, int kmax, std::vector<FusedGate> &out, bool blocks) {
    std::vector<std::vector<size_t>> members;
    std::vector<int32_t> group_of;
    const size_t ng0 = fuse_groups(g, kmax, group_of);
    members.assign(ng0, {});
    for (size_t i = 0; i < g.size(); ++i) members[group_of[i]].push_back(i);
    if (blocks) {
        // the block plan, unless the C7 plan is cheaper under the same model
        auto cost = [&](const std::vector<std::vector<size_t>> &mm) {
            double c = 0;
            for (const auto &m : mm) {
                uint64_t s = 0;
                for (size_t i : m) s |= qmask(g[i]);
                c += BLK_COST[__builtin_popcountll(s)];
            }
            return c;
        };
        std::vector<std::vector<size_t>> fb[2];
        run_parallel(2, [&](size_t i) { fb[i] = frontier_blocks(g, kmax, BLK_SETTINGS[i]); });
        const int b = cost(fb[1]) < cost(fb[0]) ? 1 : 0;
        if (cost(fb[b]) <= cost(members)) members.swap(fb[b]);
    }
    const size_t ng = members.size();
    out.clear();
    out.resize(ng);
    for (size_t G = 0; G < ng; ++G) {
        uint64_t sm = 0;
        for (size_t i : members[G]) sm |= qmask(g[i]);
        FusedGate &f = out[G];
        f.k = 0;
        for (int q = 0; q < 64; ++q) if ((sm >> q) & 1) f.q[f.k++] = q;
        const int D = 1 << f.k;
        f.U.assign((size_t)2 * D * D, 0.0);
        for (int i = 0; i < D; ++i) f.U[(size_t)2 * (i * D + i)] = 1.0;
        // Consecutive members whose joint support stays <= 3 qubits are first
        // multiplied together in that small space (8 x 8 at most), so the
        // 2^k x 2^k group matrix sees a few embeddings instead of one per
        // member (same product, same order: U_last ... U_first).
        GateRef pend;
        std::vector<double> pendU;
        pend.k = 0;
        auto flush = [&]() {
            if (pend.k == 0) return;
            pend.U = pendU.data();
            left_multiply_embedded(f.U, f.k, f.q, pend);
            pend.k = 0;
        };
        for (size_t i : members[G]) {
            const GateRef &m = g[i];
            int uq[6], un = 0;
            for (int j = 0; j < pend.k; ++j) uq[un++] = pend.q[j];
            for (int j = 0; j < m.k; ++j) {
                bool have = false;
                for (int t = 0; t < un; ++t) have |= uq[t] == m.q[j];
                if (!have && un < 6) uq[un++] = m.q[j];
            }
            if (pend.k > 0 && un > 3) flush();
            if (pend.k == 0) {
                pend.k = m.k;
                for (int j = 0; j < m.k; ++j) pend.q[j] = m.q[j];
                pendU.assign(m.U, m.U + ((size_t)2 << (2 * m.k)));
                continue;
            }
            // pend <- m * pend on the joint support (ascending)
            std::sort(uq, uq + un);
            const int d = 1 << un;
            std::vector<double> P((size_t)2 * d * d, 0.0);
            for (int r = 0; r < d; ++r) P[(size_t)2 * (r * d + r)] = 1.0;
            pend.U = pendU.data();
            left_multiply_embedded(P, un, uq, pend);
            left_multiply_embedded(P, un, uq, m);
            pend.k = un;
            for (int j = 0; j < un; ++j) pend.q[j] = uq[j];
            pendU.swap(P);
        }
        flush();
    }
}

// ------------------------------------------------------------------ schedule

// True when U (2^k x 2^k, interleaved complex, qubits[0] = MSB of the index)
// is block-diagonal in the U-index bits of `umask`: U[r][c] == 0 whenever r
// and c differ in one of those bits.  Exact zeros only: products of
// structurally block-diagonal gates (diagonal, controlled) keep exact zeros.
bool block_diag_in(const double *U, int k, int umask) {
    if (!U || umask == 0) return false;
    const int D = 1 << k;
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c)
            if (((r ^ c) & umask) && (U[2 * (r * D + c)] != 0.0 || U[2 * (r * D + c) + 1] != 0.0)) return false;
    return true;
}

// Qubits gate gt must hold on local bits: every target in which U is not
// block-diagonal (row f1: a target in which U is block-diagonal may stay
// global; block-diagonality in each of several bits implies it in their union).
uint64_t local_need(const GateRef &gt) {
    uint64_t need = 0;
    for (int j = 0; j < gt.k; ++j)
        if (!block_diag_in(gt.U, gt.k, 1 << (gt.k - 1 - j))) need |= 1ull << gt.q[j];
    return need;
}

// Distributed schedule.  The op stream is cut into segments, each a maximal
// run of gates whose local-need qubits fit on the n - m local bits together
// (greedy furthest reach, which minimises the number of segments, hence of
// remaps, for a given first global set).  At each segment boundary one REMAP
// makes the new global set S: the current globals the segment does not need
// stay global, and the incoming ones trade places with the local qubits of the
// complement whose next use lies furthest ahead (Belady), preferring bits >=
// PACK_MIN_BIT.  Those evictees are first packed onto the top local bits by a
// PERMUTE (swap pairs), unless they already lie in the top RUNWIN bits; the
// executor folds a PERMUTE into the preceding apply pass as a bit-permuting
// out-of-place write (apply+pack: no extra HBM pass), so every peer's data is
// one contiguous chunk (or a few long runs).
void schedule(int n, int m, const std::vector<GateRef> &g, std::vector<int> &pi,
              std::vector<Op> &ops, bool gather) {
    const int nl = n - m;
    if ((int)pi.size() != n) {
        pi.resize(n);
        for (int q = 0; q < n; ++q) pi[q] = n - 1 - q;     // logical q <-> bit n-1-q (C1)
    }
    std::vector<int> inv(n);
    for (int q = 0; q < n; ++q) inv[pi[q]] = q;
    ops.clear();
    const size_t N = g.size();
    std::vector<uint64_t> need(N, 0);
    if (m > 0)
        for (size_t i = 0; i < N; ++i) need[i] = local_need(g[i]);
    // uses[q] = gates that need logical qubit q local (ascending)
    std::vector<std::vector<uint32_t>> uses(n);
    for (size_t i = 0; i < N; ++i)
        for (int q = 0; q < n; ++q)
            if ((need[i] >> q) & 1) uses[q].push_back((uint32_t)i);
    auto next_use = [&](int q, size_t from) -> size_t {     // first use at index >= from
        auto it = std::lower_bound(uses[q].begin(), uses[q].end(), (uint32_t)from);
        return it == uses[q].end() ? std::numeric_limits<size_t>::max() : *it;
    };
    auto swap_phys = [&](int a, int b) {           // exchange the qubits at physical bits a, b
        const int qa = inv[a], qb = inv[b];
        std::swap(pi[qa], pi[qb]);
        inv[a] = qb;
        inv[b] = qa;
    };
    auto globals = [&]() {
        uint64_t G = 0;
        for (int p = nl; p < n; ++p) G |= 1ull << inv[p];
        return G;
    };
    const int RUNWIN = std::min(nl, 7);
    for (size_t i = 0; i < N; ++i) {
        const GateRef &gt = g[i];
        if (gather && m > 0 && __builtin_popcountll(need[i] & globals()) == 1) {
            // an isolated global access (row f1): the one global qubit this
            // gate needs is not needed local again within the lookahead, so
            // the rank pair that differs in it computes the gate over peer
            // memory (OP_GATHER) and the global set stays
            const int gq = __builtin_ctzll(need[i] & globals());
            const size_t nu = next_use(gq, i + 1);
            if (nu == std::numeric_limits<size_t>::max() || nu > i + (size_t)GATHER_LOOKAHEAD) {
                Op ga{OP_GATHER, (int)i, gt.k, {0}};
                for (int jj = 0; jj < gt.k; ++jj) ga.bits[jj] = pi[gt.q[jj]];
                ops.push_back(ga);
                continue;
            }
        }
        if (m > 0 && (need[i] & globals())) {
            // the segment starting at gate i; it also ends early when the
            // incoming globals would outnumber the local qubits outside it
            // that can be evicted without a standalone pass: those a folded
            // pack can move (bits >= PACK_MIN_BIT) after an apply; with no
            // apply right before (circuit start, back-to-back remaps) nothing
            // can absorb a pack, so those in the top RUNWIN bits (the exchange
            // then sends a few long runs)
            bool after_apply = !ops.empty() && ops.back().kind == OP_APPLY;
            if (after_apply)        // an apply on a global target (row f1) runs per rank: no fold
                for (int jj = 0; jj < ops.back().nbits; ++jj) after_apply &= ops.back().bits[jj] < nl;
            const uint64_t Gm = globals();
            uint64_t Lp = 0;
            for (int p = after_apply ? std::min(PACK_MIN_BIT, nl) : nl - RUNWIN; p < nl; ++p) Lp |= 1ull << inv[p];
            uint64_t U = 0;
            size_t j = i;
            while (j < N) {
                const uint64_t U2 = U | need[j];
                if (__builtin_popcountll(U2) > nl) break;
                if (j > i && __builtin_popcountll(U2 & Gm) > __builtin_popcountll(Lp & ~U2)) break;
                U = U2;
                ++j;
            }
            // incoming: current globals the segment needs
            int in_bits[6], nin = 0;
            for (int p = nl; p < n; ++p)
                if ((U >> inv[p]) & 1) in_bits[nin++] = p;
            // outgoing: local qubits outside the segment's union, furthest next use
            // after the segment first, bits >= PACK_MIN_BIT before bits below it
            std::vector<std::tuple<int, size_t, int>> cand;   // (packable, next use, phys bit)
            for (int pass = after_apply ? 1 : 0; pass < 2 && (int)cand.size() < nin; ++pass) {
                cand.clear();
                for (int p = pass == 0 ? nl - RUNWIN : 0; p < nl; ++p) {
                    const int q = inv[p];
                    if ((U >> q) & 1) continue;
                    cand.push_back({p >= PACK_MIN_BIT ? 1 : 0, next_use(q, j), p});
                }
            }
            std::sort(cand.begin(), cand.end(), [](const auto &a, const auto &b) {
                if (std::get<0>(a) != std::get<0>(b)) return std::get<0>(a) > std::get<0>(b);
                if (std::get<1>(a) != std::get<1>(b)) return std::get<1>(a) > std::get<1>(b);
                return std::get<2>(a) > std::get<2>(b);
            });
            int ev[6];
            bool in_window = true;
            for (int t = 0; t < nin; ++t) {
                ev[t] = std::get<2>(cand[t]);
                in_window &= ev[t] >= nl - RUNWIN;
            }
            // after an apply the pack is free (folded into that pass), and
            // evictees on exactly the top bits let the executor fuse the whole
            // exchange into the pass (one contiguous chunk per peer); with no
            // apply before, evictees already in the top RUNWIN bits are used
            // where they are (a few long runs per peer, no permute pass)
            int lb[6];
            if (in_window && !after_apply) {
                for (int t = 0; t < nin; ++t) lb[t] = ev[t];
            } else {
                // pack: the evictees onto the top nin local bits
                Op perm{OP_PERMUTE, -1, 0, {0}};
                bool is_ev[64] = {false};
                for (int t = 0; t < nin; ++t) is_ev[ev[t]] = true;
                int slot = nl - 1;
                for (int t = 0; t < nin; ++t) {
                    if (ev[t] >= nl - nin) { lb[t] = ev[t]; continue; }
                    while (is_ev[slot]) --slot;      // a top slot not holding an evictee
                    perm.bits[2 * perm.nbits] = ev[t];
                    perm.bits[2 * perm.nbits + 1] = slot;
                    perm.nbits++;
                    swap_phys(ev[t], slot);
                    is_ev[slot] = true;
                    lb[t] = slot--;
                }
                if (perm.nbits > 0) ops.push_back(perm);
            }
            std::sort(in_bits, in_bits + nin);
            std::sort(lb, lb + nin);
            Op rem{OP_REMAP, -1, nin, {0}};
            for (int t = 0; t < nin; ++t) {
                rem.bits[2 * t] = in_bits[t];
                rem.bits[2 * t + 1] = lb[t];
                swap_phys(in_bits[t], lb[t]);
            }
            ops.push_back(rem);
        }
        Op ap{OP_APPLY, (int)i, gt.k, {0}};
        for (int jj = 0; jj < gt.k; ++jj) ap.bits[jj] = pi[gt.q[jj]];
        ops.push_back(ap);
    }
}

// ------------------------------------------------------------------ layout

// Estimated relative cost of one pass with physical targets `bits` (k of them)
// for the kernel the executor will pick.  The
// weights follow the measured pass times of bench_sweep.py on a B200:
//   SIMT (k <= 4): each target inside the warp-lane bit range costs a
//     shuffle transpose (~10% per target at k = 4);
//   tensor cores (complex64 k = 5, 6): passes with targets at bits 0..3 run
//     at 0.75-0.85 of HBM peak (mode L or a strided mode H) against ~0.9
//     with the low bits free.
double layout_pass_cost(int dtype, int k, const int *bits) {
    double c = 1.0;
    if (dtype == HQ_C64 && k >= 4) {      // tensor cores (k = 4 widened to 5, hq_tc.cu)
        // tensor-core pass, measured per pass on the sustained 34q circuit
        // (tools/pass_times.py): mode H with <= 1 target in bits 0..3 is the
        // baseline; 2 such targets cost 1.19x; 3 or more 1.29x, in mode L
        // (>= 4 low targets, or bits 0, 1 and a third) as in mode H (the
        // executor's rule, tc_use_mode_l; bits {0,1} alone now run mode H
        // and cost like any other pair).  Since the 16-byte pattern pairs and
        // lane-pair stores every measured mode-H pass with
        // <= 1 low target runs at the same ~47 ms, whichever bit it is; a
        // bit-0 bonus (tried: 4037 vs 4050 ms before the lane-pair stores)
        // no longer applies.
        int lo = 0;
        bool b0 = false, b1 = false;
        for (int j = 0; j < k; ++j) {
            lo += bits[j] < 4;
            b0 |= bits[j] == 0;
            b1 |= bits[j] == 1;
        }
        if (lo >= 4 || (b0 && b1 && lo >= 3)) c += 0.29;        // mode L
        else if (lo == 3) c += 0.29;   // mode H, 0.65-0.79 of peak
        else if (lo == 2) c += 0.19;   // mode H, incl. bits {0,1} (0.75-0.86)
    } else {
        const int lane_lo = dtype == HQ_C64 ? 1 : 0, lane_hi = lane_lo + 5;
        for (int j = 0; j < k; ++j)
            if (bits[j] >= lane_lo && bits[j] < lane_hi) c += 0.08;
    }
    return c;
}

// Local search over the logical->physical map of the n - m local qubits:
// start from q -> n-1-q and apply any swap of two local positions that lowers
// the summed pass cost, until no swap helps (deterministic).
void plan_layout(int n, int m, int dtype, const std::vector<GateRef> &g, std::vector<int> &pi) {
    pi.resize(n);
    for (int q = 0; q < n; ++q) pi[q] = n - 1 - q;
    const int nl = n - m;
    if (m > 0 && !g.empty()) {
        // the first global set: m qubits outside the first segment (the
        // schedule's maximal gate run whose local-need qubits fit on nl
        // bits), furthest first use after it first; they take the global bits
        // in place of the default globals (logical 0..m-1)
        std::vector<uint64_t> need(g.size());
        for (size_t i = 0; i < g.size(); ++i) need[i] = local_need(g[i]);
        uint64_t U = 0;
        size_t j = 0;
        while (j < g.size() && __builtin_popcountll(U | need[j]) <= nl) U |= need[j++];
        std::vector<std::pair<size_t, int>> cand;     // (first use at >= j, logical q)
        for (int q = 0; q < n; ++q) {
            if ((U >> q) & 1) continue;
            size_t first = std::numeric_limits<size_t>::max();
            for (size_t i = j; i < g.size() && first == std::numeric_limits<size_t>::max(); ++i)
                if ((need[i] >> q) & 1) first = i;
            cand.push_back({first, q});
        }
        std::stable_sort(cand.begin(), cand.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
        std::vector<int> inv(n);
        for (int q = 0; q < n; ++q) inv[pi[q]] = q;
        for (int t = 0; t < m && t < (int)cand.size(); ++t) {
            const int q = cand[t].second;
            if (pi[q] >= nl) continue;                  // already global
            // swap with a global qubit that is not itself chosen
            for (int p = nl; p < n; ++p) {
                const int o = inv[p];
                bool chosen = false;
                for (int u = 0; u < m && u < (int)cand.size(); ++u) chosen |= cand[u].second == o;
                if (chosen) continue;
                const int pq = pi[q];
                std::swap(pi[q], pi[o]);
                inv[p] = q;
                inv[pq] = o;
                break;
            }
        }
    }
    std::vector<std::vector<int>> uses(n);
    for (size_t i = 0; i < g.size(); ++i)
        for (int j = 0; j < g[i].k; ++j) uses[g[i].q[j]].push_back((int)i);
    auto gate_cost = [&](size_t i) {
        int b[6];
        for (int j = 0; j < g[i].k; ++j) b[j] = pi[g[i].q[j]];
        return layout_pass_cost(dtype, g[i].k, b);
    };
    auto total = [&]() {
        double c = 0;
        for (size_t i = 0; i < g.size(); ++i) c += gate_cost(i);
        return c;
    };
    std::vector<int> inv(n);
    auto descend = [&]() {
        for (int q = 0; q < n; ++q) inv[pi[q]] = q;
        for (int sweep = 0; sweep < 20; ++sweep) {
            bool improved = false;
            for (int a = 0; a < nl; ++a)
                for (int b = a + 1; b < nl; ++b) {
                    const int qa = inv[a], qb = inv[b];
                    std::vector<int> touched(uses[qa]);
                    touched.insert(touched.end(), uses[qb].begin(), uses[qb].end());
                    std::sort(touched.begin(), touched.end());
                    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
                    double before = 0, after = 0;
                    for (int i : touched) before += gate_cost(i);
                    std::swap(pi[qa], pi[qb]);
                    for (int i : touched) after += gate_cost(i);
                    if (after < before - 1e-9) {
                        inv[a] = qb;
                        inv[b] = qa;
                        improved = true;
                    } else {
                        std::swap(pi[qa], pi[qb]);
                    }
                }
            if (!improved) break;
        }
    };
    // pairwise-swap descent from the start layout, then from LAYOUT_RESTARTS
    // deterministic shuffles of its local positions; the cheapest result
    // wins (the first on ties)
    constexpr int LAYOUT_RESTARTS = 24;
    const std::vector<int> start = pi;
    descend();
    std::vector<int> best = pi;
    double bc = total();
    uint64_t rs = 0x9e3779b97f4a7c15ull;
    for (int r = 0; r < LAYOUT_RESTARTS && bc > (double)g.size() + 1e-9; ++r) {
        pi = start;
        std::vector<int> loc;
        for (int q = 0; q < n; ++q) if (pi[q] < nl) loc.push_back(q);
        for (size_t i = loc.size(); i > 1; --i) {         // Fisher-Yates on the local positions
            rs += 0x9e3779b97f4a7c15ull;
            uint64_t z = rs;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            z ^= z >> 31;
            const size_t j = (size_t)(z % i);
            std::swap(pi[loc[i - 1]], pi[loc[j]]);
        }
        descend();
        const double c = total();
        if (c < bc - 1e-9) { bc = c; best = pi; }
    }
    pi = best;
}

}  // namespace hq

// ------------------------------------------------------------------ C ABI

using namespace hq;

static hq_status to_refs(const hq_gate *in, size_t ng, int n, std::vector<GateRef> &out) {
    out.resize(ng);
    for (size_t i = 0; i < ng; ++i) {
        const hq_gate &x = in[i];
        if (x.k < 1 || x.k > 6) return set_error(HQ_ERR_K, "gate %zu: k=%d not in [1,6]", i, x.k);
        if (!x.U) return set_error(HQ_ERR_ARG, "gate %zu: U is NULL", i);
        GateRef &r = out[i];
        r.k = x.k;
        r.U = x.U;
        for (int j = 0; j < x.k; ++j) {
            const int q = x.qubits[j];
            if (q < 0 || q >= n) return set_error(HQ_ERR_QUBIT, "gate %zu: qubit %d not in [0,%d)", i, q, n);
            for (int l = 0; l < j; ++l)
                if (x.qubits[l] == q) return set_error(HQ_ERR_DUP_QUBIT, "gate %zu: repeated qubit %d", i, q);
            r.q[j] = q;
        }
    }
    return HQ_OK;
}

extern "C" hq_status hq_fuse_plan(const hq_gate *in, size_t ngates, int kmax, int32_t *group_of,
                                  size_t *ngroups) {
    HQ_ABI_BEGIN
    clear_error();
    if ((!in && ngates) || !ngroups || (!group_of && ngates)) return set_error(HQ_ERR_ARG, "NULL argument");
    if (kmax < 1 || kmax > 6) return set_error(HQ_ERR_K, "kmax=%d not in [1,6]", kmax);
    std::vector<GateRef> refs;
    hq_status st = to_refs(in, ngates, 64, refs);
    if (st) return st;
    for (size_t i = 0; i < ngates; ++i)
        if (refs[i].k > kmax) return set_error(HQ_ERR_K, "gate %zu wider (%d) than kmax=%d", i, refs[i].k, kmax);
    std::vector<int32_t> go;
    *ngroups = fuse_groups(refs, kmax, go);
    if (ngates) std::memcpy(group_of, go.data(), sizeof(int32_t) * ngates);
    return HQ_OK;
    HQ_ABI_END
}

static hq_status fuse_abi(const hq_gate *in, size_t ngates, int kmax, hq_gate **out, size_t *nout, bool blocks);

extern "C" hq_status hq_fuse(const hq_gate *in, size_t ngates, int kmax, hq_gate **out,
                             size_t *nout) {
    HQ_ABI_BEGIN
    return fuse_abi(in, ngates, kmax, out, nout, false);
    HQ_ABI_END
}

extern "C" hq_status hq_fuse_blocks(const hq_gate *in, size_t ngates, int kmax, hq_gate **out,
                                    size_t *nout) {
    HQ_ABI_BEGIN
    return fuse_abi(in, ngates, kmax, out, nout, true);
    HQ_ABI_END
}

static hq_status fuse_abi(const hq_gate *in, size_t ngates, int kmax, hq_gate **out, size_t *nout, bool blocks) {
    clear_error();
    if ((!in && ngates) || !out || !nout) return set_error(HQ_ERR_ARG, "NULL argument");
    if (kmax < 1 || kmax > 6) return set_error(HQ_ERR_K, "kmax=%d not in [1,6]", kmax);
    std::vector<GateRef> refs;
    hq_status st = to_refs(in, ngates, 64, refs);
    if (st) return st;
    for (size_t i = 0; i < ngates; ++i)
        if (refs[i].k > kmax) return set_error(HQ_ERR_K, "gate %zu wider (%d) than kmax=%d", i, refs[i].k, kmax);
    std::vector<FusedGate> fused;
    try {
        fuse_build(refs, kmax, fused, blocks);
    } catch (const std::bad_alloc &) {
        return set_error(HQ_ERR_OOM, "host allocation failed in hq_fuse");
    }
    hq_gate *arr = new (std::nothrow) hq_gate[fused.size() ? fused.size() : 1];
    if (!arr) return set_error(HQ_ERR_OOM, "host allocation failed");
    for (size_t G = 0; G < fused.size(); ++G) {
        arr[G].k = fused[G].k;
        for (int j = 0; j < 6; ++j) arr[G].qubits[j] = j < fused[G].k ? fused[G].q[j] : -1;
        double *U = new (std::nothrow) double[fused[G].U.size()];
        if (!U) {
            for (size_t t = 0; t < G; ++t) delete[] arr[t].U;
            delete[] arr;
            return set_error(HQ_ERR_OOM, "host allocation failed");
        }
        std::memcpy(U, fused[G].U.data(), sizeof(double) * fused[G].U.size());
        arr[G].U = U;
    }
    *out = arr;
    *nout = fused.size();
    return HQ_OK;
}

extern "C" hq_status hq_free_gates(hq_gate *gates, size_t ngates) {
    HQ_ABI_BEGIN
    if (!gates) return HQ_OK;
    for (size_t i = 0; i < ngates; ++i) delete[] gates[i].U;
    delete[] gates;
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_schedule(int n, int m, const hq_gate *gates, size_t ngates, hq_op **ops,
                                 size_t *nops, int32_t *pi_out) {
    HQ_ABI_BEGIN
    return hq_schedule_from(n, m, gates, ngates, nullptr, 0, ops, nops, pi_out);
    HQ_ABI_END
}

extern "C" hq_status hq_schedule_from(int n, int m, const hq_gate *gates, size_t ngates, const int32_t *pi_in,
                                      int flags, hq_op **ops, size_t *nops, int32_t *pi_out) {
    HQ_ABI_BEGIN
    clear_error();
    if ((!gates && ngates) || !ops || !nops) return set_error(HQ_ERR_ARG, "NULL argument");
    if (n < 1 || n > 63 || m < 0 || m > 16) return set_error(HQ_ERR_ARG, "bad n=%d / m=%d", n, m);
    if (m > 0 && n - m < 6) return set_error(HQ_ERR_NGPUS, "n - m = %d < 6", n - m);
    std::vector<GateRef> refs;
    hq_status st = to_refs(gates, ngates, n, refs);
    if (st) return st;
    for (size_t i = 0; i < ngates; ++i)
        if (refs[i].k > n - m) return set_error(HQ_ERR_K, "gate %zu: k=%d > local qubits %d", i, refs[i].k, n - m);
    std::vector<int> pi;
    if (pi_in) {
        std::vector<int> seen(n, 0);
        pi.assign(pi_in, pi_in + n);
        for (int q = 0; q < n; ++q)
            if (pi[q] < 0 || pi[q] >= n || seen[pi[q]]++) return set_error(HQ_ERR_ARG, "pi_in is not a permutation");
    }
    std::vector<Op> v;
    schedule(n, m, refs, pi, v, (flags & HQ_SCHED_GATHER) != 0);
    hq_op *arr = new (std::nothrow) hq_op[v.size() ? v.size() : 1];
    if (!arr) return set_error(HQ_ERR_OOM, "host allocation failed");
    for (size_t i = 0; i < v.size(); ++i) {
        arr[i].kind = v[i].kind;
        arr[i].gate = v[i].gate;
        arr[i].nbits = v[i].nbits;
        for (int t = 0; t < 12; ++t) arr[i].bits[t] = v[i].bits[t];
    }
    *ops = arr;
    *nops = v.size();
    if (pi_out) for (int q = 0; q < n; ++q) pi_out[q] = pi[q];
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_plan_layout(int n, int m, int dtype, const hq_gate *gates, size_t ngates,
                                   int32_t *pi_out, double *cost_before, double *cost_after) {
    HQ_ABI_BEGIN
    clear_error();
    if ((!gates && ngates) || !pi_out) return set_error(HQ_ERR_ARG, "NULL argument");
    if (n < 1 || n > 63 || m < 0 || m > 16 || (m > 0 && n - m < 6))
        return set_error(HQ_ERR_ARG, "bad n=%d / m=%d", n, m);
    std::vector<GateRef> refs;
    hq_status st = to_refs(gates, ngates, n, refs);
    if (st) return st;
    auto total = [&](const std::vector<int> &pi) {
        double c = 0;
        for (auto &gt : refs) {
            int b[6];
            for (int j = 0; j < gt.k; ++j) b[j] = pi[gt.q[j]];
            c += layout_pass_cost(dtype, gt.k, b);
        }
        return c;
    };
    std::vector<int> pi0(n), pi;
    for (int q = 0; q < n; ++q) pi0[q] = n - 1 - q;
    plan_layout(n, m, dtype, refs, pi);
    if (cost_before) *cost_before = total(pi0);
    if (cost_after) *cost_after = total(pi);
    for (int q = 0; q < n; ++q) pi_out[q] = pi[q];
    return HQ_OK;
    HQ_ABI_END
}

extern "C" hq_status hq_free_ops(hq_op *ops) {
    HQ_ABI_BEGIN
    delete[] ops;
    return HQ_OK;
    HQ_ABI_END
}
