// cache.cu -- P-Tucker-Cache (the paper's time-optimised variant, Alg. 3 TOP branch,
// P:581-626): the cache table Pres in R^{|Omega| x |G|},
//   lines 1-4  : Pres[alpha][beta] = G_beta prod_{k=1..N} a^(k)_{i_k j_k}
//   lines 16-19: after A^(n) is updated, Pres[alpha][beta] = Pres[alpha][beta] / a_old * a_new
//                (a_old = 0: the product recomputed)
// (line 12, delta from Pres, is the CACHE instantiation of update_generic.cu).  One thread
// per (alpha, beta), fp64; the table lives in HBM (|Omega| |G| 8 bytes: c1 10 MB, c2 8 GB,
// the order-10 scaling shape of P:1070 472 MB).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace pt {
namespace {

template <typename TS>
__device__ __forceinline__ double pres_product(int N, const JDims& jd, const TS* G, const TS* const* A, int lda,
                                               const int32_t* coord, int64_t b) {
    double prod = (double)G[b];
    for (int m = N - 1; m >= 0; --m) {
        const int jm = (int)(b % jd.j[m]);
        b /= jd.j[m];
        prod *= (double)A[m][(int64_t)coord[m] * lda + jm];
    }
    return prod;
}

template <typename TS>
__global__ void k_pres_init(int N, const JDims jd, int64_t gsize, const TS* __restrict__ G, const TS* const* A,
                            int lda, const int32_t* __restrict__ coords, int64_t nnz, double* __restrict__ pres) {
    const int64_t total = nnz * gsize;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t / gsize, b = t % gsize;
        pres[t] = pres_product(N, jd, G, A, lda, coords + e * N, b);
    }
}

template <typename TS>
__global__ void k_pres_update(int N, const JDims jd, int64_t gsize, int n, int64_t stride_n, const TS* __restrict__ G,
                              const TS* const* A, int lda, const TS* __restrict__ A_old,
                              const int32_t* __restrict__ coords, int64_t nnz, double* __restrict__ pres) {
    const int64_t total = nnz * gsize;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t / gsize, b = t % gsize;
        const int32_t* coord = coords + e * N;
        const int jn = (int)((b / stride_n) % jd.j[n]);
        const int64_t at = (int64_t)coord[n] * lda + jn;
        const double ao = (double)A_old[at], an = (double)A[n][at];
        pres[t] = ao != 0.0 ? pres[t] / ao * an : pres_product(N, jd, G, A, lda, coord, b);
    }
}

int grid_of(int64_t total) {
    const int64_t g = (total + 255) / 256;
    return (int)(g < 148 * 32 ? (g > 0 ? g : 1) : 148 * 32);
}

}  // namespace

void launch_pres_init(int N, const JDims& J, int elem_bytes, const void* G, const void* const* d_A, int lda,
                      const int32_t* coords, int64_t nnz, double* pres, cudaStream_t st) {
    int64_t gsize = 1;
    for (int m = 0; m < N; ++m) gsize *= J.j[m];
    const int grid = grid_of(nnz * gsize);
    if (elem_bytes == 8)
        k_pres_init<double><<<grid, 256, 0, st>>>(N, J, gsize, (const double*)G, (const double* const*)d_A, lda, coords,
                                                  nnz, pres);
    else
        k_pres_init<float><<<grid, 256, 0, st>>>(N, J, gsize, (const float*)G, (const float* const*)d_A, lda, coords,
                                                 nnz, pres);
}

void launch_pres_update(int N, const JDims& J, int elem_bytes, int n, const void* G, const void* const* d_A, int lda,
                        const void* A_old, const int32_t* coords, int64_t nnz, double* pres, cudaStream_t st) {
    int64_t gsize = 1, stride_n = 1;
    for (int m = 0; m < N; ++m) gsize *= J.j[m];
    for (int m = n + 1; m < N; ++m) stride_n *= J.j[m];
    const int grid = grid_of(nnz * gsize);
    if (elem_bytes == 8)
        k_pres_update<double><<<grid, 256, 0, st>>>(N, J, gsize, n, stride_n, (const double*)G,
                                                    (const double* const*)d_A, lda, (const double*)A_old, coords, nnz,
                                                    pres);
    else
        k_pres_update<float><<<grid, 256, 0, st>>>(N, J, gsize, n, stride_n, (const float*)G, (const float* const*)d_A,
                                                   lda, (const float*)A_old, coords, nnz, pres);
}

}  // namespace pt
