// approx.cu -- P-Tucker-Approx: partial reconstruction error R(beta) of
// every core entry (Eq. 13) for the core truncation of Alg. 4.
//
// Eq. 13's second line, t_beta(alpha) (-2 X_alpha + t_beta + 2 sum_{gamma != beta} t_gamma)
// with t_gamma = G_gamma K_gamma(alpha), K_gamma(alpha) = prod_n a^(n)_{i_n gamma_n} and
// sum_{gamma != beta} t_gamma = x_hat - t_beta, is  2 G_beta K_beta e_alpha - G_beta^2 K_beta^2
// with e_alpha = x_hat_alpha - X_alpha.  Summed over Omega:
//     R(beta) = 2 G_beta U_beta - G_beta^2 V_beta,
//     U = sum_alpha e_alpha K(alpha),   V = sum_alpha K(alpha)^2   (J^N each).
// Grouping the entries by their mode-0 segment s (this rank's SELL segments of
// mode 0, row i_s) splits K = a^(0)_{i_s} (x) K'(alpha) with K' over the other modes:
//     U[j0, b'] = sum_s a^(0)_{i_s j0}   W_s[b'],    W_s  = sum_{alpha in s} e_alpha K'(alpha)
//     V[j0, b'] = sum_s a^(0)_{i_s j0}^2 W2_s[b'],   W2_s = sum_{alpha in s} K'(alpha)^2
// so the per-entry work is J^(N-1) (not J^N) and the J x J^(N-1) outer sums over
// segments are a small reduction.  x_hat_alpha = sum_b' K'_b' H_s[b'] with
// H_s = a^(0)_{i_s} G_(0) (once per segment).  Everything is fp64 (the scores rank
// the core entries; the oracle computes them in fp64 too).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace pt {
namespace {

constexpr int kApproxWarps = 8;  // warps per block of k_approx_seg (one SELL segment per warp at a time)

// One warp per SELL segment of mode 0 (pad lanes: zero outputs).  The segment's
// entries go in batches of 32: lane l gathers entry l's rows (modes 1..N-1, fp64) into
// shared memory and computes its e = x_hat - X (J^(N-1) FMAs against H); then the
// batch's entries are accumulated into W, W2 with the b' split over the lanes (no
// global loads in that inner loop).
template <typename TS, int N, int J>
#ifndef PT_APPROX_MINB
#define PT_APPROX_MINB 2
#endif
__global__ void __launch_bounds__(kApproxWarps * 32, PT_APPROX_MINB) k_approx_seg(
    int64_t nlanes, const int64_t* slice_off, const int32_t* lane_row,
    const int32_t* lane_len, const int32_t* const* sc, const TS* sv, const TS* const* A, int lda,
    const double* G64, double* A0seg, double* W, double* W2, double* Eslot) {
    // dynamic shared memory, per warp: H[K1] (padded to 8 doubles), the batch's rows
    // [32][N-1][J] (fp64) and e[32]
    extern __shared__ double smem[];
    constexpr int K1 = ipow(J, N - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k1p = (K1 + 7) / 8 * 8;
    constexpr int rstride = (N - 1) * J;  // staged rows of one entry (fp64)
    double* H = smem + warp * (k1p + 32 * rstride + 32);
    double* Rw = H + k1p;               // Rw[entry * rstride + (n-1) * J + j]
    double* Ew = Rw + 32 * rstride;     // Ew[entry]
    // Eslot[slot]: e of each entry, computed in the first chunk pass (K1 > 256) and reused
    for (int64_t seg = (int64_t)blockIdx.x * kApproxWarps + warp; seg < nlanes;
         seg += (int64_t)gridDim.x * kApproxWarps) {
        const int row = lane_row[seg];
        const int len = row >= 0 ? lane_len[seg] : 0;
        double* w = W + seg * K1;
        double* w2 = W2 + seg * K1;
        if (row < 0) {
            for (int b = lane; b < K1; b += 32) w[b] = w2[b] = 0.0;
            if (lane < J) A0seg[seg * J + lane] = 0.0;
            continue;
        }
        const int64_t base = slice_off[seg >> 5] + (seg & 31);
        // a^(0) of the segment's row and H = a0 G_(0)
        if (lane < J) A0seg[seg * J + lane] = (double)A[0][(int64_t)row * lda + lane];
        for (int b = lane; b < K1; b += 32) {
            double h = 0.0;
            for (int j = 0; j < J; ++j) h = fma((double)A[0][(int64_t)row * lda + j], G64[(int64_t)j * K1 + b], h);
            H[b] = h;
        }
        __syncwarp();
        // K'_b' of a staged entry: b' = (b_1, ..., b_{N-1}) in C order
        auto kprod = [&](int b, const double* r) {
            double k = 1.0;
            for (int n = N - 1; n >= 1; --n) {
                k *= r[(n - 1) * J + b % J];
                b /= J;
            }
            return k;
        };
        // W, W2 accumulators of this lane's b' (b' = lane + 32 m), kept in registers over the
        // whole segment when K1 <= 256, else swept in chunks of 256 (re-gathering the entries)
        constexpr int MB = (K1 < 256 ? K1 : 256) / 32 + ((K1 < 256 ? K1 : 256) % 32 != 0);  // b' per lane per chunk
        for (int b0 = 0; b0 < K1; b0 += 256) {
            double acc[MB], acc2[MB];
            int ix[MB][N - 1];  // this lane's b' = b0 + lane + 32 m as row offsets (n - 1) * J + b_n
#pragma unroll
            for (int m = 0; m < MB; ++m) {
                acc[m] = acc2[m] = 0.0;
                int b = b0 + lane + 32 * m;
                b = b < K1 ? b : 0;
#pragma unroll
                for (int n = N - 1; n >= 1; --n) {
                    ix[m][n - 1] = (n - 1) * J + b % J;
                    b /= J;
                }
            }
            // order 3: lane (g, b2) = (lane / J, lane % J) accumulates W[b1][b2], W2[b1][b2] for
            // all b1 over the batch entries q = g (mod 32 / J): each r2 value is loaded once and
            // the r1 row is a broadcast read (about half the shared-memory loads per b')
            constexpr int NG3 = 32 / J;
            const int g3 = lane / J, c3 = lane % J;
            double a3[N == 3 ? J : 1], a3s[N == 3 ? J : 1];
            if constexpr (N == 3) {
#pragma unroll
                for (int b1 = 0; b1 < J; ++b1) a3[b1] = a3s[b1] = 0.0;
            }
            for (int e0 = 0; e0 < len; e0 += 32) {
                const int e = e0 + lane;
                double* r = Rw + lane * rstride;
                if (e < len) {
                    const int64_t slot = base + (int64_t)e * 32;
                    for (int n = 1; n < N; ++n) {
                        const TS* rowp = A[n] + (int64_t)sc[n - 1][slot] * lda;
                        for (int j = 0; j < J; ++j) r[(n - 1) * J + j] = (double)rowp[j];
                    }
                    if (b0 > 0) {  // later chunk pass: e from the first
                        Ew[lane] = Eslot[slot];
                    } else {
                    // x_hat as a contraction chain of H with the staged rows (innermost mode first)
                    double xh = 0.0;
                    if constexpr (N == 2) {
#pragma unroll
                        for (int b1 = 0; b1 < J; ++b1) xh = fma(H[b1], r[b1], xh);
                    } else if constexpr (N == 3) {  // x_hat = sum_b1 r1[b1] sum_b2 H[b1][b2] r2[b2]
#pragma unroll
                        for (int b1 = 0; b1 < J; ++b1) {
                            double t = 0.0;
#pragma unroll
                            for (int b2 = 0; b2 < J; ++b2) t = fma(H[b1 * J + b2], r[J + b2], t);
                            xh = fma(r[b1], t, xh);
                        }
                    } else if constexpr (N == 4) {
                        for (int b1 = 0; b1 < J; ++b1) {
                            double t1 = 0.0;
#pragma unroll
                            for (int b2 = 0; b2 < J; ++b2) {
                                double t2 = 0.0;
#pragma unroll
                                for (int b3 = 0; b3 < J; ++b3) t2 = fma(H[(b1 * J + b2) * J + b3], r[2 * J + b3], t2);
                                t1 = fma(r[J + b2], t2, t1);
                            }
                            xh = fma(r[b1], t1, xh);
                        }
                    } else if constexpr (N == 5) {
                        for (int b1 = 0; b1 < J; ++b1) {
                            double t1 = 0.0;
                            for (int b2 = 0; b2 < J; ++b2) {
                                double t2 = 0.0;
#pragma unroll
                                for (int b3 = 0; b3 < J; ++b3) {
                                    double t3 = 0.0;
#pragma unroll
                                    for (int b4 = 0; b4 < J; ++b4)
                                        t3 = fma(H[((b1 * J + b2) * J + b3) * J + b4], r[3 * J + b4], t3);
                                    t2 = fma(r[2 * J + b3], t3, t2);
                                }
                                t1 = fma(r[J + b2], t2, t1);
                            }
                            xh = fma(r[b1], t1, xh);
                        }
                    } else {
                        for (int b = 0; b < K1; ++b) xh = fma(kprod(b, r), H[b], xh);
                    }
                    Ew[lane] = xh - (double)sv[slot];
                    if (K1 > 256) Eslot[slot] = Ew[lane];
                    }
                }
                __syncwarp();
                const int cnt = len - e0 < 32 ? len - e0 : 32;
                if constexpr (N == 3) {
                    if (g3 < NG3) {
                        for (int q = g3; q < cnt; q += NG3) {
                            const double* rq = Rw + q * rstride;
                            const double ee = Ew[q];
                            const double r2 = rq[J + c3];
#pragma unroll
                            for (int b1 = 0; b1 < J; ++b1) {
                                const double k = rq[b1] * r2;
                                a3[b1] = fma(ee, k, a3[b1]);
                                a3s[b1] = fma(k, k, a3s[b1]);
                            }
                        }
                    }
                    __syncwarp();
                    continue;
                }
                for (int q = 0; q < cnt; ++q) {
                    const double* rq = Rw + q * rstride;
                    const double ee = Ew[q];
#pragma unroll
                    for (int m = 0; m < MB; ++m) {
                        const int b = b0 + lane + 32 * m;
                        if (b < K1) {
                            double k = rq[ix[m][0]];
#pragma unroll
                            for (int n = 1; n < N - 1; ++n) k *= rq[ix[m][n]];
                            acc[m] = fma(ee, k, acc[m]);
                            acc2[m] = fma(k, k, acc2[m]);
                        }
                    }
                }
                __syncwarp();
            }
            if constexpr (N == 3) {
                // add the groups' partials (group 0 collects, groups in order) and store
#pragma unroll
                for (int q = 1; q < NG3; ++q) {
#pragma unroll
                    for (int b1 = 0; b1 < J; ++b1) {
                        const double o = __shfl_down_sync(0xffffffffu, a3[b1], q * J);
                        const double o2 = __shfl_down_sync(0xffffffffu, a3s[b1], q * J);
                        if (g3 == 0) {
                            a3[b1] += o;
                            a3s[b1] += o2;
                        }
                    }
                }
                if (g3 == 0) {
#pragma unroll
                    for (int b1 = 0; b1 < J; ++b1) {
                        w[b1 * J + c3] = a3[b1];
                        w2[b1 * J + c3] = a3s[b1];
                    }
                }
                continue;
            }
#pragma unroll
            for (int m = 0; m < MB; ++m) {
                const int b = b0 + lane + 32 * m;
                if (b < K1) {
                    w[b] = acc[m];
                    w2[b] = acc2[m];
                }
            }
        }
        __syncwarp();
    }
}

// U[j0*K1 + b'] = sum_s A0seg[s][j0] W[s][b'],  V = sum_s A0seg[s][j0]^2 W2[s][b'];
// blockIdx.y = a contiguous range of segments (per-range partials, fixed-order sum).
template <int J>
__global__ void k_approx_outer(int K1, int64_t nseg, int64_t per, const double* A0seg, const double* W,
                               const double* W2, double* part) {
    // thread per b' (all J values of j0 at once, so W and W2 are read once);
    // blockIdx.y = a contiguous range of segments (per-range partials, fixed-order sum)
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= K1) return;
    const int64_t nout = (int64_t)J * K1;
    const int64_t s0 = (int64_t)blockIdx.y * per, s1 = s0 + per < nseg ? s0 + per : nseg;
    double u[J], v[J];
#pragma unroll
    for (int j0 = 0; j0 < J; ++j0) u[j0] = v[j0] = 0.0;
    for (int64_t s = s0; s < s1; ++s) {
        const double w = W[s * K1 + b], w2 = W2[s * K1 + b];
#pragma unroll
        for (int j0 = 0; j0 < J; ++j0) {
            const double a = A0seg[s * J + j0];
            u[j0] = fma(a, w, u[j0]);
            v[j0] = fma(a * a, w2, v[j0]);
        }
    }
#pragma unroll
    for (int j0 = 0; j0 < J; ++j0) {
        part[((int64_t)blockIdx.y * 2 + 0) * nout + (int64_t)j0 * K1 + b] = u[j0];
        part[((int64_t)blockIdx.y * 2 + 1) * nout + (int64_t)j0 * K1 + b] = v[j0];
    }
}

__global__ void k_approx_sum(int64_t nout, int nsplit, const double* part, double* UV) {
    const int64_t out = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (out >= nout) return;
    double u = 0.0, v = 0.0;
    for (int y = 0; y < nsplit; ++y) {
        u += part[((int64_t)y * 2 + 0) * nout + out];
        v += part[((int64_t)y * 2 + 1) * nout + out];
    }
    UV[out] = u;
    UV[nout + out] = v;
}

template <typename TS>
__global__ void k_to_f64(const TS* in, double* out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}

// Shapes without a compiled (N, J) (order > 5, other J): U and V straight from their
// definition, one thread per core entry beta looping over this rank's entries of the
// device COO (mode-0 row in [row_lo, row_hi)); e_alpha = x_hat_alpha - X_alpha with
// x_hat from k_predict (xhat[]).  Entries are staged in shared memory per chunk.
constexpr int kLitChunk = 128;
template <typename TS>
__global__ void __launch_bounds__(256) k_approx_literal(int N, const JDims jd, int64_t gsize, const TS* const* A, int lda,
                                                        const int32_t* coords, const TS* vals, const double* xhat,
                                                        int64_t n, int64_t row_lo, int64_t row_hi, double* UV) {
    __shared__ int32_t cs[kLitChunk * kMaxN];
    __shared__ double es[kLitChunk];
    __shared__ int keep[kLitChunk];
    const int64_t beta = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int bn[kMaxN];
    {
        int64_t b = beta < gsize ? beta : 0;
        for (int m = N - 1; m >= 0; --m) {
            bn[m] = (int)(b % jd.j[m]);
            b /= jd.j[m];
        }
    }
    double u = 0.0, v = 0.0;
    for (int64_t q0 = 0; q0 < n; q0 += kLitChunk) {
        const int cnt = n - q0 < kLitChunk ? (int)(n - q0) : kLitChunk;
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * N; t += blockDim.x) cs[t] = coords[q0 * N + t];
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
            const int32_t i0 = coords[(q0 + t) * N];
            keep[t] = i0 >= row_lo && i0 < row_hi;
            es[t] = xhat[q0 + t] - (double)vals[q0 + t];
        }
        __syncthreads();
        if (beta >= gsize) continue;
        for (int t = 0; t < cnt; ++t) {
            if (!keep[t]) continue;
            double k = 1.0;
            for (int m = 0; m < N; ++m) k *= (double)A[m][(int64_t)cs[t * N + m] * lda + bn[m]];
            u = fma(es[t], k, u);
            v = fma(k, k, v);
        }
    }
    if (beta < gsize) {
        UV[beta] = u;
        UV[gsize + beta] = v;
    }
}

}  // namespace

void launch_approx_literal(int N, const JDims& J, int elem_bytes, const void* const* d_A, int lda, const int32_t* coords,
                           const void* vals, const double* xhat, int64_t n, int64_t row_lo, int64_t row_hi,
                           double* UV, cudaStream_t st) {
    int64_t gsize = 1;
    for (int m = 0; m < N; ++m) gsize *= J.j[m];
    const unsigned grid = (unsigned)((gsize + 255) / 256);
    if (elem_bytes == 8)
        k_approx_literal<double><<<grid, 256, 0, st>>>(N, J, gsize, (const double* const*)d_A, lda, coords,
                                                       (const double*)vals, xhat, n, row_lo, row_hi, UV);
    else
        k_approx_literal<float><<<grid, 256, 0, st>>>(N, J, gsize, (const float* const*)d_A, lda, coords,
                                                      (const float*)vals, xhat, n, row_lo, row_hi, UV);
}

bool approx_shape_ok(int N, int J) {
#define PT_APPROX_OK(NN, JJ) \
    if (N == NN && J == JJ) return true;
    PT_NJ_LIST(PT_APPROX_OK)
#undef PT_APPROX_OK
    return false;
}

// U, V (J^N each, C order over the core) of this rank's entries of mode 0 into UV[2*J^N].
// Scratch: A0seg [nlanes*J], W, W2 [nlanes*K1], Eslot [nslots], part [2*nsplit*J^N], G64 [J^N].
void launch_approx_uv(int N, int J, int elem_bytes, int64_t nslices, const int64_t* slice_off,
                      const int32_t* lane_row, const int32_t* lane_len, const int32_t* const* d_sc, const void* sv,
                      const void* const* d_A, int lda, const void* G, double* G64, double* A0seg, double* W,
                      double* W2, double* Eslot, double* part, int nsplit, double* UV, int nsm, cudaStream_t st) {
    int K1 = 1;
    for (int n = 1; n < N; ++n) K1 *= J;
    const int64_t gsize = (int64_t)K1 * J;
    const int64_t nlanes = nslices * 32;
    if (elem_bytes == 8) k_to_f64<double><<<64, 256, 0, st>>>((const double*)G, G64, gsize);
    else k_to_f64<float><<<64, 256, 0, st>>>((const float*)G, G64, gsize);
    if (nlanes > 0) {
        int grid = (int)((nlanes + kApproxWarps - 1) / kApproxWarps);
        if (grid > nsm * 8) grid = nsm * 8;
        const size_t smem = (size_t)kApproxWarps * ((K1 + 7) / 8 * 8 + 32 * (N - 1) * J + 32) * sizeof(double);
#define PT_APPROX_CASE(NN, JJ)                                                                                     \
    if (N == NN && J == JJ) {                                                                                      \
        if (elem_bytes == 8) {                                                                                     \
            cudaFuncSetAttribute(k_approx_seg<double, NN, JJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            k_approx_seg<double, NN, JJ><<<grid, kApproxWarps * 32, smem, st>>>(                                   \
                nlanes, slice_off, lane_row, lane_len, d_sc, (const double*)sv, (const double* const*)d_A, lda, G64, \
                A0seg, W, W2, Eslot);                                                                              \
        } else {                                                                                                   \
            cudaFuncSetAttribute(k_approx_seg<float, NN, JJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            k_approx_seg<float, NN, JJ><<<grid, kApproxWarps * 32, smem, st>>>(                                    \
                nlanes, slice_off, lane_row, lane_len, d_sc, (const float*)sv, (const float* const*)d_A, lda, G64,  \
                A0seg, W, W2, Eslot);                                                                              \
        }                                                                                                          \
    }
        PT_NJ_LIST(PT_APPROX_CASE)
#undef PT_APPROX_CASE
    }
    const int64_t per = nlanes > 0 ? (nlanes + nsplit - 1) / nsplit : 1;
    dim3 g2((unsigned)((K1 + 127) / 128), (unsigned)nsplit);
    switch (J) {
#define PT_OUTER_CASE(JJ) \
    case JJ: k_approx_outer<JJ><<<g2, 128, 0, st>>>(K1, nlanes, per, A0seg, W, W2, part); break;
        PT_OUTER_CASE(2) PT_OUTER_CASE(3) PT_OUTER_CASE(4) PT_OUTER_CASE(5) PT_OUTER_CASE(8) PT_OUTER_CASE(10)
#undef PT_OUTER_CASE
        default: break;  // not reached: launch_approx_uv is called for compiled (N, J) only
    }
    k_approx_sum<<<(unsigned)((gsize + 127) / 128), 128, 0, st>>>(gsize, nsplit, part, UV);
}

}  // namespace pt

// ---------------------------------------------------------------------------
// Alg. 4 on the device: scores R(beta) = 2 G U - G^2 V of the present entries (NaN for
// truncated ones), then the top-k present entries by R (descending; ties by ascending
// C-order index, reading R28) are zeroed in G and marked absent.  The order comes from
// a stable radix sort of order-preserving 64-bit keys (absent entries key 0, below any
// real score), so the removed set is exactly the reading's.
// ---------------------------------------------------------------------------
#include <cub/cub.cuh>

namespace pt {
namespace {

template <typename TS>
__global__ void k_core_scores(int64_t gsize, const TS* G, const double* UV, const uint8_t* present, double* R,
                              uint64_t* key, int64_t* idx) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < gsize; b += (int64_t)gridDim.x * blockDim.x) {
        const double g = (double)G[b];
        const bool on = present[b] != 0;
        const double r = on ? 2.0 * g * UV[b] - g * g * UV[gsize + b] : __longlong_as_double(0x7ff8000000000000LL);
        R[b] = r;
        if (key) {
            // order-preserving map of a finite double to uint64 (negatives: all bits flipped,
            // non-negatives: sign bit set); absent entries 0
            const uint64_t u = (uint64_t)__double_as_longlong(r);
            key[b] = on ? ((u >> 63) ? ~u : (u | 0x8000000000000000ULL)) : 0ULL;
            idx[b] = b;
        }
    }
}

template <typename TS>
__global__ void k_zero_top(int64_t k, const int64_t* order, TS* G, uint8_t* present) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = order[r];
        G[b] = TS(0);
        present[b] = 0;
    }
}

}  // namespace

// R[gsize] on the device from UV (and, when key != null, the sort keys + identity indices).
void launch_core_scores(int64_t gsize, int elem_bytes, const void* G, const double* UV, const uint8_t* present,
                        double* R, uint64_t* key, int64_t* idx, cudaStream_t st) {
    const unsigned grid = (unsigned)std::min<int64_t>((gsize + 255) / 256, 148 * 16);
    if (elem_bytes == 8) k_core_scores<double><<<grid, 256, 0, st>>>(gsize, (const double*)G, UV, present, R, key, idx);
    else k_core_scores<float><<<grid, 256, 0, st>>>(gsize, (const float*)G, UV, present, R, key, idx);
}

// Scratch bytes for core_truncate_select (keys/indices in and out + CUB temp).
size_t core_select_temp_bytes(int64_t gsize) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                              (const int64_t*)nullptr, (int64_t*)nullptr, (int)gsize);
    return tb;
}

// Zero the k first entries of the (descending, stable) order of key: G[b] = 0, present[b] = 0.
cudaError_t launch_core_truncate(int64_t gsize, int64_t k, const uint64_t* key, const int64_t* idx, uint64_t* key_out,
                                 int64_t* idx_out, void* temp, size_t temp_bytes, int elem_bytes, void* G,
                                 uint8_t* present, cudaStream_t st) {
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, key, key_out, idx, idx_out, (int)gsize,
                                                              0, 64, st);
    if (e != cudaSuccess) return e;
    if (k <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((k + 255) / 256, 148 * 16);
    if (elem_bytes == 8) k_zero_top<double><<<grid, 256, 0, st>>>(k, idx_out, (double*)G, present);
    else k_zero_top<float><<<grid, 256, 0, st>>>(k, idx_out, (float*)G, present);
    return cudaGetLastError();
}

}  // namespace pt
