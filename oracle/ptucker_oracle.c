/*
 * ptucker_oracle.c -- plain, slow, FP64 CPU oracle of P-Tucker's row-wise ALS.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py
 * (its cpu_baseline leg and `--impl reference`) may load this library.  The
 * product path (paper_1710_02261_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Every function follows the paper (arXiv 1710.02261, /root/reference/PAPER.md,
 * cited as P:<line>) step by step in the paper's order and notation:
 *   - init ~ U[0,1)                         Alg. 2 line 1
 *   - mode slices Omega^(n)_{i_n}            Table 2
 *   - delta (Eq. 12)                         P:549-552, Alg. 3 lines 8-10 P:596-599
 *   - B (Eq. 10), c (Eq. 11)                 P:541-548, Alg. 3 line 13 P:605
 *   - row rule a = c [B + lambda I]^-1 (Eq. 9), Alg. 3 lines 14-15 P:607-608
 *   - reconstruction (Eq. 4), error (Eq. 5)  P:331-341, Alg. 2 line 4 P:499
 *   - loss (Eq. 6)
 *   - QR + core update (Eq. 7-8)             P:470-479, Alg. 2 lines 8-11 P:504-508
 *   - P-Tucker-Approx: partial error R(beta) (Eq. 13) and core truncation
 *     (Alg. 4)                               P:656-700, Alg. 2 lines 5-6 P:500-502
 *   - P-Tucker-Cache: cache table Pres, delta from it, its update
 *     (Alg. 3 TOP branch)
 * Readings where the paper is silent are listed in DESIGN.md ("Readings").
 *
 * Pins (tests/test_oracle_pins.py) check every function here against values
 * and identities the paper and the mathematics fix; see DESIGN.md "Oracle".
 * Parity unpinned: or_uniform (the init RNG; the paper only says "random real
 * values between 0 and 1") is pinned to the published SplitMix64 test
 * vector and to the survey's known-answer table, not to the paper.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXN 16

/* ------------------------------------------------------------------------ */
/* Init RNG (reading R2 in DESIGN.md): counter-based SplitMix64.             */
/* z = mix64(seed*0x9E3779B97F4A7C15 + (stream+1)*0xD1B54A32D192ED03 + idx)   */
/* stream 0 = core G (idx = C-order index), stream 1+n = A^(n) (idx = i*J+j)  */
/* ------------------------------------------------------------------------ */
uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t or_rng_word(uint64_t seed, uint64_t stream, uint64_t idx) {
    return or_mix64(seed * 0x9E3779B97F4A7C15ULL + (stream + 1) * 0xD1B54A32D192ED03ULL + idx);
}

/* prec 1: f64 = (z>>11) * 2^-53; prec 0: f32 = (z>>40) * 2^-24 (exact in f32). */
double or_uniform(uint64_t seed, uint64_t stream, uint64_t idx, int prec) {
    uint64_t z = or_rng_word(seed, stream, idx);
    if (prec == 1) return (double)(z >> 11) * (1.0 / 9007199254740992.0);
    return (double)(float)((double)(z >> 40) * (1.0 / 16777216.0));
}

/* Alg. 2 line 1: "initialize factor matrices A^(n) and core tensor G"
 * with "random real values between 0 and 1". */
void or_init(int N, const int64_t* dims, const int32_t* J, uint64_t seed, int prec,
             double* G, double* A_all) {
    int64_t gsize = 1;
    for (int n = 0; n < N; ++n) gsize *= J[n];
    for (int64_t b = 0; b < gsize; ++b) G[b] = or_uniform(seed, 0, (uint64_t)b, prec);
    int64_t off = 0;
    for (int n = 0; n < N; ++n) {
        int64_t cnt = dims[n] * (int64_t)J[n];
        for (int64_t t = 0; t < cnt; ++t) A_all[off + t] = or_uniform(seed, (uint64_t)(1 + n), (uint64_t)t, prec);
        off += cnt;
    }
}

static void factor_offsets(int N, const int64_t* dims, const int32_t* J, int64_t* off) {
    off[0] = 0;
    for (int n = 0; n < N; ++n) off[n + 1] = off[n] + dims[n] * (int64_t)J[n];
}

static int64_t core_size(int N, const int32_t* J) {
    int64_t s = 1;
    for (int n = 0; n < N; ++n) s *= J[n];
    return s;
}

/* ------------------------------------------------------------------------ */
/* Mode slices Omega^(n)_{i_n} (Table 2: "observable entries whose nth */
/* mode's index is i_n").  Stable counting sort: within a slice, entries keep */
/* their input order (reading R25).  row_ptr has I_n+1 entries.               */
/* ------------------------------------------------------------------------ */
int or_mode_index(int N, int64_t nnz, const int32_t* coords, const int64_t* dims, int n,
                  int64_t* row_ptr, int64_t* perm) {
    int64_t I = dims[n];
    for (int64_t i = 0; i <= I; ++i) row_ptr[i] = 0;
    for (int64_t e = 0; e < nnz; ++e) {
        int32_t i = coords[e * N + n];
        if (i < 0 || i >= I) return 1;
        row_ptr[i + 1] += 1;
    }
    for (int64_t i = 0; i < I; ++i) row_ptr[i + 1] += row_ptr[i];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(I > 0 ? I : 1));
    for (int64_t i = 0; i < I; ++i) fill[i] = row_ptr[i];
    for (int64_t e = 0; e < nnz; ++e) {
        int32_t i = coords[e * N + n];
        perm[fill[i]++] = e;
    }
    free(fill);
    return 0;
}

/* nnz-balanced contiguous row blocks:
 * b_0 = 0, b_W = I, b_g = lower_bound(row_ptr, ceil(g*nnz/W)). */
void or_partition(const int64_t* row_ptr, int64_t I, int world, int64_t* bounds) {
    int64_t nnz = row_ptr[I];
    bounds[0] = 0;
    for (int g = 1; g < world; ++g) {
        int64_t target = (g * nnz + world - 1) / world;
        int64_t r = 0;
        while (r <= I && row_ptr[r] < target) ++r; /* plain linear lower_bound */
        if (r > I) r = I;
        bounds[g] = r;
    }
    bounds[world] = I;
}

/* ------------------------------------------------------------------------ */
/* Eq. 12, Alg. 3 lines 8-10, default (MOP) branch:  */
/*   for beta = (j_1..j_N) in G:  delta(j_n) += G_beta * prod_{k!=n} a^(k)_{i_k j_k} */
/* A literal loop over every core entry in C order, N-1 multiplies each.      */
/* ------------------------------------------------------------------------ */
void or_delta(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
              const int32_t* coord, int n, double* delta) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    int64_t gsize = core_size(N, J);
    int jj[OR_MAXN];
    for (int k = 0; k < N; ++k) jj[k] = 0;
    for (int j = 0; j < J[n]; ++j) delta[j] = 0.0;
    for (int64_t b = 0; b < gsize; ++b) {
        double prod = G[b];
        for (int k = 0; k < N; ++k) {
            if (k == n) continue;
            prod *= A_all[off[k] + (int64_t)coord[k] * J[k] + jj[k]];
        }
        delta[jj[n]] += prod;
        /* advance the C-order odometer (last mode fastest) */
        for (int k = N - 1; k >= 0; --k) {
            if (++jj[k] < J[k]) break;
            jj[k] = 0;
        }
    }
}

/* Eq. 4: x_hat = sum_beta G_beta prod_n a^(n)_{i_n j_n}. */
double or_predict(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                  const int32_t* coord) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    int64_t gsize = core_size(N, J);
    int jj[OR_MAXN];
    for (int k = 0; k < N; ++k) jj[k] = 0;
    double s = 0.0;
    for (int64_t b = 0; b < gsize; ++b) {
        double prod = G[b];
        for (int k = 0; k < N; ++k) prod *= A_all[off[k] + (int64_t)coord[k] * J[k] + jj[k]];
        s += prod;
        for (int k = N - 1; k >= 0; --k) {
            if (++jj[k] < J[k]) break;
            jj[k] = 0;
        }
    }
    return s;
}

/* Eq. 10-11, Alg. 3 line 13: over the entries of
 * Omega^(n)_{row} in slice order, B += delta delta^T (full J x J), c += x delta.
 * sumsq = sum x^2 is returned as well (used only for the SSE identity check). */
void or_row_system(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                   const int32_t* coords, const double* vals, int n, const int64_t* row_ptr,
                   const int64_t* perm, int64_t row, double* B, double* c, double* sumsq) {
    int Jn = J[n];
    double delta[64];
    for (int t = 0; t < Jn * Jn; ++t) B[t] = 0.0;
    for (int t = 0; t < Jn; ++t) c[t] = 0.0;
    double s2 = 0.0;
    for (int64_t p = row_ptr[row]; p < row_ptr[row + 1]; ++p) {
        int64_t e = perm[p];
        or_delta(N, J, G, A_all, dims, coords + e * N, n, delta);
        double x = vals[e];
        for (int j1 = 0; j1 < Jn; ++j1) {
            for (int j2 = 0; j2 < Jn; ++j2) B[j1 * Jn + j2] += delta[j1] * delta[j2];
            c[j1] += x * delta[j1];
        }
        s2 += x * x;
    }
    if (sumsq) *sumsq = s2;
}

/* Eq. 9, Alg. 3 lines 14-15: a = c [B + lambda I]^-1.
 * "find the inverse matrix" is read as a Cholesky solve (reading R12): the
 * matrix is symmetric positive definite for lambda > 0, so
 * a^T = (B + lambda I)^-1 c^T.  Returns 0, or 2 on a non-positive pivot. */
int or_solve(int Jn, const double* B, const double* c, double lambda, double* a) {
    double L[64 * 64];
    double y[64];
    for (int i = 0; i < Jn; ++i)
        for (int j = 0; j < Jn; ++j) L[i * Jn + j] = B[i * Jn + j] + (i == j ? lambda : 0.0);
    /* Cholesky: M = L L^T, L lower-triangular (overwrite lower part). */
    for (int j = 0; j < Jn; ++j) {
        double d = L[j * Jn + j];
        for (int k = 0; k < j; ++k) d -= L[j * Jn + k] * L[j * Jn + k];
        if (!(d > 0.0) || !isfinite(d)) return 2;
        d = sqrt(d);
        L[j * Jn + j] = d;
        for (int i = j + 1; i < Jn; ++i) {
            double s = L[i * Jn + j];
            for (int k = 0; k < j; ++k) s -= L[i * Jn + k] * L[j * Jn + k];
            L[i * Jn + j] = s / d;
        }
    }
    /* L y = c */
    for (int i = 0; i < Jn; ++i) {
        double s = c[i];
        for (int k = 0; k < i; ++k) s -= L[i * Jn + k] * y[k];
        y[i] = s / L[i * Jn + i];
    }
    /* L^T a = y */
    for (int i = Jn - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < Jn; ++k) s -= L[k * Jn + i] * a[k];
        a[i] = s / L[i * Jn + i];
    }
    return 0;
}

/* Alg. 3 lines 6-15 for one row: delta per entry, B and c, solve,
 * write the row.  An empty slice gives B = 0, c = 0 and hence a = 0 (reading R5). */
int or_update_row(int N, const int32_t* J, const double* G, double* A_all, const int64_t* dims,
                  const int32_t* coords, const double* vals, int n, const int64_t* row_ptr,
                  const int64_t* perm, int64_t row, double lambda) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    int Jn = J[n];
    double B[64 * 64], c[64], a[64];
    or_row_system(N, J, G, A_all, dims, coords, vals, n, row_ptr, perm, row, B, c, NULL);
    int rc = or_solve(Jn, B, c, lambda, a);
    if (rc) return rc;
    for (int j = 0; j < Jn; ++j) A_all[off[n] + row * Jn + j] = a[j];
    return 0;
}

/* Alg. 3 line 6: "for i_n = 1..I_n, in parallel".  Rows are
 * independent, so the result does not depend on the order or on the
 * thread count.  OpenMP dynamic scheduling is the paper's own. */
int or_update_mode(int N, const int32_t* J, const double* G, double* A_all, const int64_t* dims,
                   const int32_t* coords, const double* vals, int n, const int64_t* row_ptr,
                   const int64_t* perm, double lambda, int nthreads) {
    int64_t I = dims[n];
    int bad = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
#endif
    for (int64_t i = 0; i < I; ++i) {
        if (or_update_row(N, J, G, A_all, dims, coords, vals, n, row_ptr, perm, i, lambda)) bad |= 1;
    }
    (void)nthreads;
    return bad ? 2 : 0;
}

/* Eq. 5, Alg. 2 line 4: SSE over Omega in input order.
 * Fixed 4096-entry chunks are summed in order so the value is independent of
 * the thread count (P:726-728 aggregates per-thread partials). */
double or_sse(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
              const int32_t* coords, const double* vals, int64_t nnz, int nthreads) {
    const int64_t CH = 4096;
    int64_t nch = (nnz + CH - 1) / CH;
    double* part = (double*)calloc((size_t)(nch > 0 ? nch : 1), sizeof(double));
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t ch = 0; ch < nch; ++ch) {
        double s = 0.0;
        int64_t e1 = (ch + 1) * CH < nnz ? (ch + 1) * CH : nnz;
        for (int64_t e = ch * CH; e < e1; ++e) {
            double r = vals[e] - or_predict(N, J, G, A_all, dims, coords + e * N);
            s += r * r;
        }
        part[ch] = s;
    }
    (void)nthreads;
    double tot = 0.0;
    for (int64_t ch = 0; ch < nch; ++ch) tot += part[ch];
    free(part);
    return tot;
}

/* Eq. 6: L = SSE + lambda * sum_n ||A^(n)||_F^2. */
double or_loss(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
               const int32_t* coords, const double* vals, int64_t nnz, double lambda, int nthreads) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    double reg = 0.0;
    for (int64_t t = 0; t < off[N]; ++t) reg += A_all[t] * A_all[t];
    return or_sse(N, J, G, A_all, dims, coords, vals, nnz, nthreads) + lambda * reg;
}

/* ------------------------------------------------------------------------ */
/* Eq. 7: A = Q R, Q column-orthonormal, R upper triangular.      */
/* Householder thin QR (reading R13), signs fixed so diag(R) > 0, which makes */
/* Q and R unique for full-rank A.  A: I x J row-major (overwritten by Q).    */
/* Returns 0, 1 if I < J, 2 if a column is (numerically) dependent.           */
/* ------------------------------------------------------------------------ */
int or_thin_qr(int64_t I, int Jn, double* A, double* R) {
    if (I < Jn) return 1;
    double* W = (double*)malloc(sizeof(double) * (size_t)(I * Jn));  /* working copy -> R */
    double* V = (double*)malloc(sizeof(double) * (size_t)(I * Jn));  /* reflector v_k in column k */
    double* Q = (double*)calloc((size_t)(I * Jn), sizeof(double));
    double* vnorm = (double*)calloc((size_t)Jn, sizeof(double));   /* v_k^T v_k */
    double anorm = 0.0;
    for (int64_t t = 0; t < I * Jn; ++t) { W[t] = A[t]; anorm = fmax(anorm, fabs(A[t])); }
    for (int k = 0; k < Jn; ++k) {
        /* v_k = x - alpha e_k with x = W[k:, k], alpha = -sign(x_k) ||x|| */
        double nrm = 0.0;
        for (int64_t i = k; i < I; ++i) nrm += W[i * Jn + k] * W[i * Jn + k];
        nrm = sqrt(nrm);
        double alpha = W[(int64_t)k * Jn + k] >= 0 ? -nrm : nrm;
        for (int64_t i = 0; i < I; ++i) V[i * Jn + k] = (i >= k) ? W[i * Jn + k] : 0.0;
        V[(int64_t)k * Jn + k] -= alpha;
        double vn = 0.0;
        for (int64_t i = k; i < I; ++i) vn += V[i * Jn + k] * V[i * Jn + k];
        vnorm[k] = vn;
        /* W <- (I - 2 v v^T / v^T v) W on columns k..J-1 */
        if (vn > 0.0) {
            for (int c = k; c < Jn; ++c) {
                double d = 0.0;
                for (int64_t i = k; i < I; ++i) d += V[i * Jn + k] * W[i * Jn + c];
                double f = 2.0 * d / vn;
                for (int64_t i = k; i < I; ++i) W[i * Jn + c] -= f * V[i * Jn + k];
            }
        }
    }
    /* R = upper J x J block of W */
    int rc = 0;
    for (int i = 0; i < Jn; ++i)
        for (int j = 0; j < Jn; ++j) R[i * Jn + j] = (j >= i) ? W[(int64_t)i * Jn + j] : 0.0;
    for (int k = 0; k < Jn; ++k)
        if (fabs(R[k * Jn + k]) <= 1e-12 * (anorm > 0 ? anorm : 1.0)) rc = 2; /* rank deficient */
    /* Q = H_0 H_1 ... H_{J-1} [I_J; 0]: apply the reflectors in reverse order. */
    for (int j = 0; j < Jn; ++j) Q[(int64_t)j * Jn + j] = 1.0;
    for (int k = Jn - 1; k >= 0; --k) {
        if (vnorm[k] <= 0.0) continue;
        for (int c = 0; c < Jn; ++c) {
            double d = 0.0;
            for (int64_t i = k; i < I; ++i) d += V[i * Jn + k] * Q[i * Jn + c];
            double f = 2.0 * d / vnorm[k];
            for (int64_t i = k; i < I; ++i) Q[i * Jn + c] -= f * V[i * Jn + k];
        }
    }
    /* sign fix so diag(R) > 0 (reading R13): negate row k of R and column k of Q */
    for (int k = 0; k < Jn; ++k) {
        if (R[k * Jn + k] < 0) {
            for (int j = 0; j < Jn; ++j) R[k * Jn + j] = -R[k * Jn + j];
            for (int64_t i = 0; i < I; ++i) Q[i * Jn + k] = -Q[i * Jn + k];
        }
    }
    for (int64_t t = 0; t < I * Jn; ++t) A[t] = Q[t];
    free(vnorm);
    free(W);
    free(V);
    free(Q);
    return rc;
}

/* Eq. 2 with U = R (J_n x J_n), as used by Eq. 8:
 * (G x_n R)_{j_1..k..j_N} = sum_{j} G_{j_1..j..j_N} r_{k j}. */
void or_core_mode_product(int N, const int32_t* J, double* G, int n, const double* R) {
    int64_t outer = 1, inner = 1;
    for (int k = 0; k < n; ++k) outer *= J[k];
    for (int k = n + 1; k < N; ++k) inner *= J[k];
    int Jn = J[n];
    double* col = (double*)malloc(sizeof(double) * (size_t)Jn);
    for (int64_t o = 0; o < outer; ++o) {
        for (int64_t in = 0; in < inner; ++in) {
            for (int j = 0; j < Jn; ++j) col[j] = G[(o * Jn + j) * inner + in];
            for (int k = 0; k < Jn; ++k) {
                double s = 0.0;
                for (int j = 0; j < Jn; ++j) s += col[j] * R[k * Jn + j];
                G[(o * Jn + k) * inner + in] = s;
            }
        }
    }
    free(col);
}

/* Alg. 2 lines 8-11: for n = 1..N: A^(n) -> Q R; A^(n) <- Q;
 * G <- G x_n R.  R_all receives the N R-factors (J_n x J_n each, concatenated). */
int or_orthogonalize(int N, const int32_t* J, double* G, double* A_all, const int64_t* dims, double* R_all) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    int64_t roff = 0;
    int rc = 0;
    for (int n = 0; n < N; ++n) {
        double* R = R_all + roff;
        int r = or_thin_qr(dims[n], J[n], A_all + off[n], R);
        if (r == 1) return 1;
        if (r) rc = 2;
        or_core_mode_product(N, J, G, n, R);
        roff += (int64_t)J[n] * J[n];
    }
    return rc;
}

/* ------------------------------------------------------------------------ */
/* P-Tucker-Approx: partial reconstruction error and truncation. */
/* ------------------------------------------------------------------------ */

/* Eq. 13, second line, Alg. 4 lines 1-2: for every core
 * entry beta with present[beta] != 0,
 *   R(beta) = sum_alpha t_beta (-2 X_alpha + t_beta + 2 sum_{gamma != beta} t_gamma),
 *   t_gamma = G_gamma prod_n a^(n)_{i_n j_n}   (gamma over the core, C order);
 * absent entries (truncated earlier: G_gamma = 0) get R = 0.  Per observed entry the
 * t_gamma are formed once and sum_{gamma != beta} t_gamma = x_hat - t_beta with
 * x_hat = sum_gamma t_gamma (Eq. 4) -- the "one shared pass" of reading R27.
 * Entries are taken in input order in fixed 4096-entry chunks whose partial
 * sums are added in chunk order (independent of the thread count). */
void or_partial_errors(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                       const int32_t* coords, const double* vals, int64_t nnz, const uint8_t* present,
                       double* R, int nthreads) {
    const int64_t CH = 4096;
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    const int64_t gsize = core_size(N, J);
    const int64_t nch = (nnz + CH - 1) / CH;
    double* part = (double*)calloc((size_t)(nch > 0 ? nch : 1) * (size_t)gsize, sizeof(double));
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t ch = 0; ch < nch; ++ch) {
        double* t = (double*)malloc((size_t)gsize * sizeof(double));
        double* Rc = part + ch * gsize;
        int64_t e1 = (ch + 1) * CH < nnz ? (ch + 1) * CH : nnz;
        for (int64_t e = ch * CH; e < e1; ++e) {
            const int32_t* coord = coords + e * N;
            int jj[OR_MAXN];
            for (int k = 0; k < N; ++k) jj[k] = 0;
            double xhat = 0.0;
            for (int64_t b = 0; b < gsize; ++b) {
                double prod = G[b];
                for (int k = 0; k < N; ++k) prod *= A_all[off[k] + (int64_t)coord[k] * J[k] + jj[k]];
                t[b] = prod;
                xhat += prod;
                for (int k = N - 1; k >= 0; --k) {
                    if (++jj[k] < J[k]) break;
                    jj[k] = 0;
                }
            }
            const double x = vals[e];
            for (int64_t b = 0; b < gsize; ++b)
                if (present[b]) Rc[b] += t[b] * (-2.0 * x + t[b] + 2.0 * (xhat - t[b]));
        }
        free(t);
    }
    (void)nthreads;
    for (int64_t b = 0; b < gsize; ++b) {
        double s = 0.0;
        for (int64_t ch = 0; ch < nch; ++ch) s += part[ch * gsize + b];
        R[b] = present[b] ? s : 0.0;
    }
    free(part);
}

/* Alg. 4 lines 3-4: among the present entries, sort R(beta) in
 * descending order (ties: ascending C-order index, reading R28) and remove the
 * top floor(p |G|) of them, never leaving fewer than one (reading R29): G_beta = 0,
 * present[beta] = 0.  |G| counts the present entries.  Returns the number removed. */
static const double* g_trunc_R;
static int trunc_cmp(const void* a, const void* b) {
    const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
    if (g_trunc_R[i] > g_trunc_R[j]) return -1;
    if (g_trunc_R[i] < g_trunc_R[j]) return 1;
    return i < j ? -1 : (i > j ? 1 : 0);
}

int64_t or_truncate(int64_t gsize, double* G, uint8_t* present, const double* R, double p) {
    int64_t n = 0;
    for (int64_t b = 0; b < gsize; ++b) n += present[b] != 0;
    int64_t k = (int64_t)floor(p * (double)n);
    if (k > n - 1) k = n - 1;
    if (k <= 0) return 0;
    int64_t* idx = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t m = 0;
    for (int64_t b = 0; b < gsize; ++b)
        if (present[b]) idx[m++] = b;
    g_trunc_R = R;
    qsort(idx, (size_t)n, sizeof(int64_t), trunc_cmp);
    for (int64_t r = 0; r < k; ++r) {
        G[idx[r]] = 0.0;
        present[idx[r]] = 0;
    }
    free(idx);
    return k;
}

/* Eq. 4 for n query coordinates (prediction of missing entries). */
void or_predict_many(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                     const int32_t* coords, int64_t n, double* out) {
    for (int64_t q = 0; q < n; ++q) out[q] = or_predict(N, J, G, A_all, dims, coords + q * N);
}

/* Held-out test RMSE (§4.4): sqrt( sum_q (x_q - x_hat_q)^2 / n ), n >= 1. */
double or_test_rmse(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                    const int32_t* coords, const double* vals, int64_t n) {
    double s = 0.0;
    for (int64_t q = 0; q < n; ++q) {
        double r = vals[q] - or_predict(N, J, G, A_all, dims, coords + q * N);
        s += r * r;
    }
    return sqrt(s / (double)n);
}

/* ------------------------------------------------------------------------ */
/* P-Tucker-Cache (TOP), Alg. 3 with the cache table Pres in R^{|Omega| x |G|} */
/* (P:581-626), literally:                                         */
/*   lines 1-4  : Pres[alpha][beta] = G_beta prod_{k=1..N} a^(k)_{i_k j_k}    */
/*   line 12    : delta(j_n) += Pres[alpha][beta] / a^(n)_{i_n j_n}           */
/*                (when a^(n)_{i_n j_n} = 0: as MOP, line 10)          */
/*   lines 16-19: after A^(n) is updated, Pres[alpha][beta] =                 */
/*                Pres[alpha][beta] / a_old^(n)_{i_n j_n} x a_new^(n)_{i_n j_n}*/
/*                (a_old = 0: recomputed as in lines 1-4)              */
/* Pres is row-major |Omega| x |G| with beta in C order.                      */
/* ------------------------------------------------------------------------ */
static void pres_entry(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                       const int32_t* coord, double* out /* [|G|] */) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    int64_t gsize = core_size(N, J);
    int jj[OR_MAXN];
    for (int k = 0; k < N; ++k) jj[k] = 0;
    for (int64_t b = 0; b < gsize; ++b) {
        double prod = G[b];
        for (int k = 0; k < N; ++k) prod *= A_all[off[k] + (int64_t)coord[k] * J[k] + jj[k]];
        out[b] = prod;
        for (int k = N - 1; k >= 0; --k) {
            if (++jj[k] < J[k]) break;
            jj[k] = 0;
        }
    }
}

/* Alg. 3 lines 1-4. */
void or_pres_init(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                  const int32_t* coords, int64_t nnz, double* pres, int nthreads) {
    const int64_t gsize = core_size(N, J);
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t e = 0; e < nnz; ++e) pres_entry(N, J, G, A_all, dims, coords + e * N, pres + e * gsize);
    (void)nthreads;
}

/* Alg. 3 lines 9-12, TOP branch: delta of entry e for mode n from Pres. */
void or_delta_cache(int N, const int32_t* J, const double* G, const double* A_all, const int64_t* dims,
                    const int32_t* coord, const double* pres_e, int n, double* delta) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    int64_t gsize = core_size(N, J);
    int jj[OR_MAXN];
    for (int k = 0; k < N; ++k) jj[k] = 0;
    for (int j = 0; j < J[n]; ++j) delta[j] = 0.0;
    for (int64_t b = 0; b < gsize; ++b) {
        const double a = A_all[off[n] + (int64_t)coord[n] * J[n] + jj[n]];
        if (a != 0.0) {
            delta[jj[n]] += pres_e[b] / a;                   /* line 12 */
        } else {                                              /* line 10 */
            double prod = G[b];
            for (int k = 0; k < N; ++k) {
                if (k == n) continue;
                prod *= A_all[off[k] + (int64_t)coord[k] * J[k] + jj[k]];
            }
            delta[jj[n]] += prod;
        }
        for (int k = N - 1; k >= 0; --k) {
            if (++jj[k] < J[k]) break;
            jj[k] = 0;
        }
    }
}

/* Alg. 3 lines 6-15 for every row of mode n with the TOP delta, then lines 16-19
 * (P:610-619): Pres rescaled by a_new / a_old (recomputed where a_old = 0).
 * pres: |Omega| x |G| (updated in place).  Returns 0 or 2 (non-positive pivot). */
int or_update_mode_cache(int N, const int32_t* J, const double* G, double* A_all, const int64_t* dims,
                         const int32_t* coords, const double* vals, int64_t nnz, int n, const int64_t* row_ptr,
                         const int64_t* perm, double lambda, double* pres, int nthreads) {
    int64_t off[OR_MAXN + 1];
    factor_offsets(N, dims, J, off);
    const int64_t gsize = core_size(N, J);
    const int Jn = J[n];
    const int64_t I = dims[n];
    double* old = (double*)malloc(sizeof(double) * (size_t)(I * Jn));
    memcpy(old, A_all + off[n], sizeof(double) * (size_t)(I * Jn));
    int bad = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(| : bad)
#endif
    for (int64_t i = 0; i < I; ++i) {
        double B[64 * 64], c[64], a[64], delta[64];
        for (int t = 0; t < Jn * Jn; ++t) B[t] = 0.0;
        for (int t = 0; t < Jn; ++t) c[t] = 0.0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const int64_t e = perm[p];
            or_delta_cache(N, J, G, A_all, dims, coords + e * N, pres + e * gsize, n, delta);
            const double x = vals[e];
            for (int j1 = 0; j1 < Jn; ++j1) {
                for (int j2 = 0; j2 < Jn; ++j2) B[j1 * Jn + j2] += delta[j1] * delta[j2];
                c[j1] += x * delta[j1];
            }
        }
        if (or_solve(Jn, B, c, lambda, a)) bad |= 1;
        else for (int j = 0; j < Jn; ++j) A_all[off[n] + i * Jn + j] = a[j];
    }
    /* lines 16-19: every entry's cache row, the mode-n factor value swapped */
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t e = 0; e < nnz; ++e) {
        const int32_t* coord = coords + e * N;
        double* pe = pres + e * gsize;
        int recompute = 0;
        int jj[OR_MAXN];
        for (int k = 0; k < N; ++k) jj[k] = 0;
        for (int64_t b = 0; b < gsize; ++b) {
            const double ao = old[(int64_t)coord[n] * Jn + jj[n]];
            const double an = A_all[off[n] + (int64_t)coord[n] * Jn + jj[n]];
            if (ao != 0.0) pe[b] = pe[b] / ao * an;
            else recompute = 1;
            for (int k = N - 1; k >= 0; --k) {
                if (++jj[k] < J[k]) break;
                jj[k] = 0;
            }
        }
        if (recompute) pres_entry(N, J, G, A_all, dims, coord, pe);
    }
    free(old);
    (void)nthreads;
    return bad ? 2 : 0;
}
