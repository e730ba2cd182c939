/*
 * ORACLE -- test infrastructure only.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load, call or execute anything under oracle/.  The
 * product path (paper_2111_06868_b200/, include/) never does, and shares no
 * code, header, table or helper with this file.
 *
 * What it computes: the plain definition of applying a k-qubit gate U to a
 * 2^n amplitude vector on ordered target qubits, gate by gate, unfused, fp64
 * (SURVEY.md §8(c) "Definition"):
 *
 *   psi'[i] = sum_{c=0}^{2^k-1} U[r(i)][c] * psi[i with target bits := c]
 *
 *   - PAPER.md P:87-91 and P:641-656: the state-vector core is a matrix-vector
 *     multiplication on the target axes, "a similar syntax of numpy.dot".
 *   - SPEC.md S:238-246: apply_matrix, psi <- (M embedded on qubits) psi.
 *   - Bit order (reading C1, pinned by the Grover listing P:403-422): qubit q
 *     is index bit n-1-q (qubit 0 = most significant bit).
 *   - Matrix order (reading C2): U is row-major, qubits[0] is the
 *     most significant bit of U's row/column index.
 *
 * Algorithm, step by step (SURVEY.md §8(c) "Oracle algorithm"):
 *   1. b_j = n-1-q_j; off[c] = sum_j bit_(k-1-j)(c) * 2^(b_j).
 *   2. sort the b_j ascending for zero-bit insertion.
 *   3. for every outer index o in [0, 2^(n-k)) (OpenMP, static schedule):
 *        base = o with zero bits inserted at the sorted b_j;
 *        v[c] = psi[base + off[c]];
 *        w[r] = sum_c U[r][c] * v[c], c ascending, complex product written
 *               out as (ar*br - ai*bi, ar*bi + ai*br);
 *        psi[base + off[r]] = w[r].
 * Each output is produced by one thread in a fixed order, so results are
 * bit-identical for any thread count (pin P15).  Compile with
 * -ffp-contract=off so no FMA contraction changes the rounding.
 *
 * Layout: psi is 2*2^n doubles, interleaved (re, im).  U is 2*4^k doubles,
 * interleaved, row-major.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_KMAX 10

/* return codes */
#define OR_OK 0
#define OR_ERR_K 1
#define OR_ERR_QUBIT 2
#define OR_ERR_DUP 3

int oracle_apply(double *psi, int n, const double *U, const int *qubits, int k)
{
    if (k < 1 || k > ORACLE_KMAX || k > n) return OR_ERR_K;
    int b[ORACLE_KMAX], s[ORACLE_KMAX];
    for (int j = 0; j < k; ++j) {
        if (qubits[j] < 0 || qubits[j] >= n) return OR_ERR_QUBIT;
        for (int l = 0; l < j; ++l)
            if (qubits[l] == qubits[j]) return OR_ERR_DUP;
        b[j] = n - 1 - qubits[j];
        s[j] = b[j];
    }
    /* step 1: offsets; qubits[0] <-> MSB of c */
    const int d = 1 << k;
    uint64_t off[1 << ORACLE_KMAX];
    for (int c = 0; c < d; ++c) {
        uint64_t o = 0;
        for (int j = 0; j < k; ++j)
            if ((c >> (k - 1 - j)) & 1) o |= (uint64_t)1 << b[j];
        off[c] = o;
    }
    /* step 2: sort bit positions ascending (insertion sort) */
    for (int j = 1; j < k; ++j) {
        int x = s[j], l = j - 1;
        while (l >= 0 && s[l] > x) { s[l + 1] = s[l]; --l; }
        s[l + 1] = x;
    }
    /* step 3 */
    const int64_t N = (int64_t)1 << (n - k);
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < N; ++o) {
        uint64_t base = (uint64_t)o;
        for (int j = 0; j < k; ++j) {            /* insert a zero at s[j] */
            uint64_t lo = base & (((uint64_t)1 << s[j]) - 1);
            base = ((base >> s[j]) << (s[j] + 1)) | lo;
        }
        double vr[1 << ORACLE_KMAX], vi[1 << ORACLE_KMAX];
        for (int c = 0; c < d; ++c) {
            vr[c] = psi[2 * (base + off[c])];
            vi[c] = psi[2 * (base + off[c]) + 1];
        }
        for (int r = 0; r < d; ++r) {
            double wr = 0.0, wi = 0.0;
            for (int c = 0; c < d; ++c) {
                double ar = U[2 * (r * d + c)], ai = U[2 * (r * d + c) + 1];
                double pr = ar * vr[c] - ai * vi[c];
                double pi = ar * vi[c] + ai * vr[c];
                wr = wr + pr;
                wi = wi + pi;
            }
            psi[2 * (base + off[r])] = wr;
            psi[2 * (base + off[r]) + 1] = wi;
        }
    }
    return OR_OK;
}

/* ||psi||_2 with a fixed blocked summation (blocks of 2^16 amplitudes summed
 * in parallel, block sums added serially) so the result does not depend on
 * the thread count (reading C13: the norm, not its square). */
double oracle_norm(const double *psi, int n)
{
    const int64_t N = (int64_t)1 << n;
    const int64_t B = 1 << 16;
    const int64_t nb = (N + B - 1) / B;
    double *part = (double *)malloc(sizeof(double) * (size_t)nb);
    if (!part) return -1.0;
#pragma omp parallel for schedule(static)
    for (int64_t blk = 0; blk < nb; ++blk) {
        double acc = 0.0;
        int64_t e = (blk + 1) * B < N ? (blk + 1) * B : N;
        for (int64_t i = blk * B; i < e; ++i)
            acc = acc + (psi[2 * i] * psi[2 * i] + psi[2 * i + 1] * psi[2 * i + 1]);
        part[blk] = acc;
    }
    double tot = 0.0;
    for (int64_t blk = 0; blk < nb; ++blk) tot = tot + part[blk];
    free(part);
    return sqrt(tot);
}

/* psi = |x>, zero elsewhere (parallel first touch). */
void oracle_init_basis(double *psi, int n, uint64_t x)
{
    const int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < 2 * N; ++i) psi[i] = 0.0;
    psi[2 * x] = 1.0;
}

void oracle_set_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
