// update_generic.cu -- row update for any order N <= kMaxN and core size J <= 16 (the
// shapes without a compiled (N, J) kernel: the order-scaling workload of P:1013-1014,
// N = 3..10, J = 3, I = 100, |Omega| = 10^3, and any J outside {2,3,4,5,8,10}).
//
// Unequal core dimensions J_1..J_N (Alg. 2 input) run here too.
// One thread per SELL-32 lane (row segment) of mode n, everything in fp64:
//   delta(j) = sum over the other modes' indices k of G[beta(k, beta_n = j)] prod_{m != n} a^(m)_{i_m k_m}
// (Eq. 12, evaluated as written: J^(N-1) products of N-1 factors, each
// feeding J FMAs), B += delta delta^T, c += x delta, sum x^2 (Eq. 10-11), then the
// Cholesky solve a = c [B + lambda I]^-1 (Eq. 9) and the row's SSE by the identity
// of update.cuh (fused Eq. 5), or the heavy-row partial record.  These shapes are
// tiny (|Omega| = 10^3): the kernel favours generality over speed.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace pt {
namespace {

constexpr int kGJ = 16;  // max J of the generic kernel

__device__ __forceinline__ int upi(int i, int j, int J) { return i * J - i * (i - 1) / 2 + (j - i); }

// CACHE (P-Tucker-Cache, Alg. 3 line 12): delta(j_n) = sum over beta with beta_n = j_n
// of Pres[alpha][beta] / a^(n)_{i_n j_n}, the division taken once per j (the same sum); a
// factor value of exactly 0 takes the product loop instead.  Pres is |Omega| x |G|
// (beta in C order), alpha = the slot's input entry id (ModeIndex::sid).
// SPARSE (P-Tucker-Approx's truncated core): delta over the coordinate
// list of the present core entries only (C order, each packed as 4-bit digits beta_0..beta_{N-1}
// plus its C-order index): O(N |G|) per entry instead of the dense J^(N-1) (J + N - 1).  The
// list is in C order and the product is formed in the same mode order as the dense loop, so
// for every j the terms arrive in the dense order minus exact zeros: bit-identical deltas.
struct SparseCore {
    const uint64_t* digits = nullptr;  // packed beta digits (4 bits per mode, mode 0 lowest), this mode's order
    const int64_t* index = nullptr;    // C-order index of the entry in G
    const int32_t* off = nullptr;      // [33] lane l's entries: [off[l], off[l+1]) (see below)
};

// One WARP per SELL lane (row segment): the 32 lanes split the delta loop of each entry --
// dense: combination t of the other modes' indices (C order) to lane t mod 32; sparse: the
// mode's list is ordered by (t mod 32, C order) so each lane takes the same terms, in the
// same order, as in the dense loop (bit-identical); cache: beta to lane beta mod 32 -- then
// a fixed xor butterfly (every lane ends with the same bits) and the normal equations, kept
// identical in every lane; lane 0 writes.  The order-scaling shapes (|Omega| = 10^3, J^(N-1)
// up to 19,683 terms per component) ran one thread per segment before: 32x the parallelism.
template <typename TS, bool CACHE, bool SPARSE = false>
__global__ void __launch_bounds__(128) k_update_gen(const UpdateParams<TS> p, int N, const JDims jd,
                                                    const double* __restrict__ pres, const int32_t* __restrict__ sid,
                                                    int64_t gsize, const SparseCore sp = SparseCore()) {
    const int64_t nl = p.nslices * kWarp;
    const int lane = threadIdx.x & 31;
    const int n = p.n;
    const int J = jd.j[n];  // J_n: size of delta, B and c of this mode
    // stride of beta_m in the C-order core, and J of the k-th other mode (ascending)
    int64_t stride[kMaxN];
    int Jo[kMaxN - 1];
    {
        int64_t s = 1;
        for (int m = N - 1; m >= 0; --m) {
            stride[m] = s;
            s *= jd.j[m];
        }
        for (int k = 0; k < N - 1; ++k) Jo[k] = jd.j[k < n ? k : k + 1];
    }
    int64_t ncomb = 1;
    for (int k = 0; k < N - 1; ++k) ncomb *= Jo[k];
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t slot = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); slot < nl; slot += nw) {
        const int row = p.lane_row[slot];
        if (row < 0) continue;
        const int len = p.lane_len[slot];
        const int64_t base = p.slice_off[slot >> 5] + (slot & 31);
        double B[kGJ * (kGJ + 1) / 2], c[kGJ], s2 = 0.0;
        for (int q = 0; q < J * (J + 1) / 2; ++q) B[q] = 0.0;
        for (int q = 0; q < J; ++q) c[q] = 0.0;
        for (int e = 0; e < len; ++e) {
            const int64_t es = base + (int64_t)e * kWarp;
            const double x = (double)p.sv[es];
            const TS* rows[kMaxN - 1];
            for (int k = 0; k < N - 1; ++k) {
                PT_CHK(p.sc[k][es] >= 0 && p.sc[k][es] < p.dim_other[k]);
                rows[k] = p.A[k] + (int64_t)p.sc[k][es] * p.lda;
            }
            double d[kGJ];
            for (int j = 0; j < J; ++j) d[j] = 0.0;
            bool mop = !CACHE;  // product loop (P-Tucker) for every j, or only where a^(n)_{i_n j} = 0
            unsigned zero_j = 0;
            if constexpr (CACHE) {
                const double* pr = pres + (int64_t)sid[es] * gsize;
                const TS* an = p.An + (int64_t)row * p.lda;  // a^(n)_{i_n .} before this update
                for (int64_t b = lane; b < gsize; b += 32) d[(int)((b / stride[n]) % J)] += pr[b];
                for (int j = 0; j < J; ++j)
                    for (int o = 16; o > 0; o >>= 1) d[j] += __shfl_xor_sync(0xffffffffu, d[j], o);
                for (int j = 0; j < J; ++j) {
                    const double a = (double)an[j];
                    if (a != 0.0) d[j] /= a;
                    else {
                        d[j] = 0.0;
                        zero_j |= 1u << j;
                        mop = true;
                    }
                }
            }
            // this lane's partial sums of the product loop (dense or sparse), reduced below
            double dp[kGJ];
            for (int j = 0; j < J; ++j) dp[j] = 0.0;
            if constexpr (SPARSE) {
                mop = false;
                for (int64_t q = sp.off[lane]; q < sp.off[lane + 1]; ++q) {
                    const uint64_t dg = sp.digits[q];
                    double prod = 1.0;
                    for (int k = 0; k < N - 1; ++k) {
                        const int m = k < n ? k : k + 1;
                        prod *= (double)rows[k][(int)((dg >> (4 * m)) & 15u)];
                    }
                    const int jn = (int)((dg >> (4 * n)) & 15u);
                    dp[jn] = fma((double)p.Gp[sp.index[q]], prod, dp[jn]);
                }
            }
            for (int64_t t = lane; mop && t < ncomb; t += 32) {
                // the other modes' indices k_0..k_{N-2} (ascending mode order) of combination t
                int kk[kMaxN - 1];
                {
                    int64_t r = t;
                    for (int k = N - 2; k >= 0; --k) {
                        kk[k] = (int)(r % Jo[k]);
                        r /= Jo[k];
                    }
                }
                double prod = 1.0;
                int64_t gb = 0;
                for (int k = 0; k < N - 1; ++k) {
                    const int m = k < n ? k : k + 1;  // the mode of the k-th other row
                    prod *= (double)rows[k][kk[k]];
                    gb += kk[k] * stride[m];
                }
                for (int j = 0; j < J; ++j)
                    if (!CACHE || ((zero_j >> j) & 1u)) dp[j] = fma((double)p.Gp[gb + j * stride[n]], prod, dp[j]);
            }
            if (SPARSE || mop) {
                for (int j = 0; j < J; ++j) {
                    double v = dp[j];
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    d[j] += v;
                }
            }
            for (int i = 0; i < J; ++i) {
                c[i] = fma(x, d[i], c[i]);
                for (int j = i; j < J; ++j) B[upi(i, j, J)] = fma(d[i], d[j], B[upi(i, j, J)]);
            }
            s2 = fma(x, x, s2);
        }
        if (lane != 0) continue;  // every lane holds the same B, c, s2: lane 0 writes
        const int64_t pidx = p.lane_pidx[slot];
        if (pidx >= 0) {
            const int stp = p.lane_pstride[slot];
            const int NB = J * (J + 1) / 2;
            double* dst = p.partials + pidx;
            for (int q = 0; q < NB; ++q) dst[(int64_t)q * stp] = B[q];
            for (int q = 0; q < J; ++q) dst[(int64_t)(NB + q) * stp] = c[q];
            dst[(int64_t)(NB + J) * stp] = s2;
            continue;
        }
        // Cholesky of B + lambda I (upper triangle overwritten by L^T), then the two solves
        bool ok = true;
        double inv[kGJ], y[kGJ], a[kGJ];
        for (int j = 0; j < J; ++j) {
            double dj = B[upi(j, j, J)] + p.lambda;
            for (int k = 0; k < j; ++k) dj = fma(-B[upi(k, j, J)], B[upi(k, j, J)], dj);
            ok = ok && (dj > 0.0);
            inv[j] = 1.0 / sqrt(fmax(dj, 1e-300));
            for (int i = j + 1; i < J; ++i) {
                double s = B[upi(j, i, J)];
                for (int k = 0; k < j; ++k) s = fma(-B[upi(k, i, J)], B[upi(k, j, J)], s);
                B[upi(j, i, J)] = s * inv[j];
            }
        }
        for (int i = 0; i < J; ++i) {
            double s = c[i];
            for (int k = 0; k < i; ++k) s = fma(-B[upi(k, i, J)], y[k], s);
            y[i] = s * inv[i];
        }
        for (int i = J - 1; i >= 0; --i) {
            double s = y[i];
            for (int k = i + 1; k < J; ++k) s = fma(-B[upi(i, k, J)], a[k], s);
            a[i] = s * inv[i];
        }
        if (!ok) {
            atomicCAS(p.fail, 0, row + 1);
            for (int j = 0; j < J; ++j) a[j] = 0.0;
        }
        PT_CHK(row < p.dim_n);
        TS* out = p.An + (int64_t)row * p.lda;
        double sse = s2, ac = 0.0, aa = 0.0, ec = 0.0;
        for (int j = 0; j < J; ++j) {
            const TS st = (TS)a[j];
            out[j] = st;
            const double at = (double)st;
            sse = fma(-2.0 * at, c[j], sse);
            ac = fma(a[j], c[j], ac);
            aa = fma(a[j], a[j], aa);
            ec = fma(at - a[j], c[j] - p.lambda * a[j], ec);
        }
        p.sse_row[row] = sse + ac - p.lambda * aa + 2.0 * ec;  // SSE of the stored row (update.cuh)
        push_row(p.peers, out, row, p.lda * (int)sizeof(TS));
    }
}

}  // namespace

// The generic kernel reads the core in plain C order: p.Gp must be G itself.
template <typename TS>
void launch_gen_t(const UpdateParams<TS>& p, int N, const JDims& J, int nsm, cudaStream_t st, const double* pres,
                  const int32_t* sid, int64_t gsize, const uint64_t* sp_digits, const int64_t* sp_index,
                  const int32_t* sp_off) {
    const int64_t nl = p.nslices * kWarp;  // lanes = warps of the kernel, 4 per block
    int grid = (int)((nl + 3) / 4);
    if (grid > nsm * 32) grid = nsm * 32;
    if (grid <= 0) return;
    if (pres) {
        k_update_gen<TS, true><<<grid, 128, 0, st>>>(p, N, J, pres, sid, gsize);
    } else if (sp_digits) {
        SparseCore sc;
        sc.digits = sp_digits;
        sc.index = sp_index;
        sc.off = sp_off;
        k_update_gen<TS, false, true><<<grid, 128, 0, st>>>(p, N, J, nullptr, nullptr, gsize, sc);
    } else {
        k_update_gen<TS, false><<<grid, 128, 0, st>>>(p, N, J, nullptr, nullptr, gsize);
    }
}

void launch_update_generic(const void* params, int elem_bytes, int N, const JDims& J, int nsm, cudaStream_t st,
                           const double* pres, const int32_t* sid, const uint64_t* sp_digits, const int64_t* sp_index,
                           const int32_t* sp_off) {
    int64_t gsize = 1;
    for (int m = 0; m < N; ++m) gsize *= J.j[m];
    if (elem_bytes == 8)
        launch_gen_t(*reinterpret_cast<const UpdateParams<double>*>(params), N, J, nsm, st, pres, sid, gsize,
                     sp_digits, sp_index, sp_off);
    else
        launch_gen_t(*reinterpret_cast<const UpdateParams<float>*>(params), N, J, nsm, st, pres, sid, gsize,
                     sp_digits, sp_index, sp_off);
}

bool generic_shape_ok(int N, int J) { return N >= 2 && N <= kMaxN && J >= 1 && J <= kGJ; }

}  // namespace pt
