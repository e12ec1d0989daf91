// kernels.cuh -- host-side launch wrappers of the small kernels (kernels.cu, index.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace pt {

// ---- init (Alg. 2 line 1; reading R2: counter-based SplitMix64) ----
void launch_init_uniform(void* out, int elem_bytes, int64_t rows, int J, int ld, uint64_t seed, uint64_t stream,
                         cudaStream_t st);
// ---- core permuted for mode n: Gp[(k_0..k_{N-3})][gblk] with block [k_{N-2}][j] ----
void launch_permute_core(const void* G, void* Gp, int elem_bytes, int N, int J, int n, cudaStream_t st);
// ---- heavy rows: reduce the segment partials in a fixed order and solve (Eq. 9) ----
void launch_heavy_finalize(int64_t nheavy, const int32_t* hrow, const int32_t* hnseg, const int64_t* hpbase,
                           const double* partials, double* rec, int J, double lambda, void* An, int elem_bytes,
                           int lda, double* sse_row, int* fail, cudaStream_t st, const PeerRows& peers,
                           int64_t max_seg, int64_t min_seg = 0);  // max segments of a heavy row (<= 64: one fused launch)
// ---- ptucker_init input validation on the device: bad[0] = first out-of-range coordinate
// (entry * 16 + mode), bad[1] = first non-finite value (all bits set = none), part[grid] =
// per-block sums of x^2 ----
void launch_validate_coo(const int32_t* coords, const void* vals, int elem_bytes, int64_t nnz, int N,
                         const int64_t* dims, int64_t* bad, double* part, int grid, cudaStream_t st);
// ---- deterministic sum of x[0..n) (fixed 256-block tree) into *out (device) ----
void launch_sum(const double* x, int64_t n, double* part256, double* out, cudaStream_t st);
// ---- QR (Eq. 7) by CholeskyQR2 in fp64, and G <- G x_n R (Eq. 8) ----
void launch_gram(const void* A, int elem_bytes, bool a_is_f64_scratch, int64_t I, int J, int lda, double* part,
                 double* W, cudaStream_t st);
void launch_chol_upper(const double* W, int J, double* R, int* fail, int fail_code, cudaStream_t st);
void launch_apply_rinv(const void* A, int a_bytes, int lda_a, void* Q, int q_bytes, int lda_q, int64_t I, int J,
                       const double* R, cudaStream_t st);
void launch_mat_upper_mul(const double* R2, const double* R1, double* R, int J, cudaStream_t st);
void launch_core_mode_product(const void* G, void* Gout, int elem_bytes, int N, const JDims& J, int n, const double* R,
                              cudaStream_t st);
// ---- small-mode precontraction for order-4 tensors with two small modes (smp.cu) ----
void launch_smp_table2(const void* G, const void* As1, const void* As2, int lda, int64_t I1, int64_t I2, int J, int n,
                       int r, int s1, int s2, double* T64, void* T32, int elem_bytes, cudaStream_t st);
// mode: 0 = fp32 table in smem, 1 = fp64 table from L2, 2 = hybrid (fp64 for single-segment rows)
bool launch_smp2_update(const void* params, int elem_bytes, int J, const double* T64, const void* T32,
                        int64_t tab_elems, int ir, int is1, int is2, int I2, int mode, int nsm, cudaStream_t st);
// order-4 mode with ONE small other mode s: table of order-3 cores, one per row of s
void launch_smp_table1(const void* G, const void* As, int lda, int64_t Is, int J, int n, int a, int b, int s, void* T,
                       int elem_bytes, cudaStream_t st);
bool launch_table_update(const void* params, int elem_bytes, int J, int nsm, cudaStream_t st);
// ---- P-Tucker-Approx scores (approx.cu): U = sum e K, V = sum K^2 over this rank's mode-0 entries ----
void launch_approx_uv(int N, int J, int elem_bytes, int64_t nslices, const int64_t* slice_off,
                      const int32_t* lane_row, const int32_t* lane_len, const int32_t* const* d_sc, const void* sv,
                      const void* const* d_A, int lda, const void* G, double* G64, double* A0seg, double* W,
                      double* W2, double* Eslot, double* part, int nsplit, double* UV, int nsm, cudaStream_t st);
// ---- Eq. 4 predictions of query coordinates (predict.cu) ----
void launch_predict(int N, const JDims& J, int elem_bytes, const void* G, const void* const* d_A, int lda,
                    const int32_t* coords, const void* vals, int64_t n, double* out, int residual_sq, int nsm,
                    cudaStream_t st, int64_t row_lo = 0, int64_t row_hi = INT64_MAX);
// ---- index build helpers (index.cu) ----
void launch_extract_col(const int32_t* coords, int64_t nnz, int N, int n, int32_t* keys, int32_t* iota,
                        cudaStream_t st);
void launch_row_ptr(const int32_t* sorted_keys, int64_t nnz, int64_t I, int64_t* row_ptr, cudaStream_t st);

}  // namespace pt
