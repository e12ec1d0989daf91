// predict.cu -- Eq. 4 for query coordinates (prediction of missing
// entries; the held-out RMSE of §4.4):
//     x_hat = sum_beta G_beta prod_n a^(n)_{i_n beta_n},
// one thread per query, fp64 over the dense core (truncated entries are zero).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace pt {
namespace {

template <typename TS>
__global__ void k_predict(int N, const JDims jd, int64_t gsize, const TS* __restrict__ G, const TS* const* __restrict__ A,
                          int lda, const int32_t* __restrict__ coords, const TS* __restrict__ vals, int64_t n,
                          double* __restrict__ out, int residual_sq, int64_t row_lo, int64_t row_hi) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        if (residual_sq && (coords[q * N] < row_lo || coords[q * N] >= row_hi)) {  // another rank's mode-0 rows
            out[q] = 0.0;
            continue;
        }
        // the query's factor rows in fp64
        double r[kMaxN][16];
        for (int k = 0; k < N; ++k) {
            const TS* row = A[k] + (int64_t)coords[q * N + k] * lda;
            for (int j = 0; j < jd.j[k]; ++j) r[k][j] = (double)row[j];
        }
        const int JL = jd.j[N - 1];
        // depth-first over beta in C order: prod of the first N-1 factors, then a dot over beta_N
        int jj[kMaxN] = {0};
        double s = 0.0;
        for (int64_t b = 0; b < gsize; b += JL) {
            double pre = 1.0;
            for (int k = 0; k < N - 1; ++k) pre *= r[k][jj[k]];
            double dot = 0.0;
            for (int j = 0; j < JL; ++j) dot = fma((double)G[b + j], r[N - 1][j], dot);
            s = fma(pre, dot, s);
            for (int k = N - 2; k >= 0; --k) {
                if (++jj[k] < jd.j[k]) break;
                jj[k] = 0;
            }
        }
        if (residual_sq) {
            const double e = (double)vals[q] - s;
            out[q] = e * e;
        } else {
            out[q] = s;
        }
    }
}

}  // namespace

// out[q] = x_hat (residual_sq = 0) or (x - x_hat)^2 (1, 0 outside mode-0 rows [row_lo, row_hi))
// for n queries (device buffers).
void launch_predict(int N, const JDims& J, int elem_bytes, const void* G, const void* const* d_A, int lda,
                    const int32_t* coords, const void* vals, int64_t n, double* out, int residual_sq, int nsm,
                    cudaStream_t st, int64_t row_lo, int64_t row_hi) {
    if (n <= 0) return;
    int64_t gsize = 1;
    for (int k = 0; k < N; ++k) gsize *= J.j[k];
    int grid = (int)((n + 127) / 128);
    if (grid > nsm * 16) grid = nsm * 16;
    if (elem_bytes == 8)
        k_predict<double><<<grid, 128, 0, st>>>(N, J, gsize, (const double*)G, (const double* const*)d_A, lda, coords,
                                                (const double*)vals, n, out, residual_sq, row_lo, row_hi);
    else
        k_predict<float><<<grid, 128, 0, st>>>(N, J, gsize, (const float*)G, (const float* const*)d_A, lda, coords,
                                               (const float*)vals, n, out, residual_sq, row_lo, row_hi);
}

}  // namespace pt
