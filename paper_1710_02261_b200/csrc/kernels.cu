// kernels.cu -- small kernels around the hot path: init RNG, core permutation,
// heavy-row finalize, deterministic sums, CholeskyQR2 and the core update.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"
#include "kernels.cuh"
#include "update.cuh"

namespace pt {

int g_pdl = 0;  // option "pdl" (internal.cuh): off, measured slower under graph replay

// ---------------------------------------------------------------------------
// Init (Alg. 2 line 1; "random real values between 0 and 1").
// Reading R2: z = mix64(seed*0x9E3779B97F4A7C15 + (stream+1)*0xD1B54A32D192ED03 + idx),
// mix64 = SplitMix64 finaliser; f64 = (z>>11)*2^-53, f32 = (z>>40)*2^-24.
// stream 0 = core (idx = C-order index), stream 1+n = A^(n) (idx = i*J + j).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_finalize(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void k_init_uniform(T* out, int64_t rows, int J, int ld, uint64_t seed, uint64_t stream) {
    const int64_t total = rows * J;
    const uint64_t base = seed * 0x9E3779B97F4A7C15ull + (stream + 1) * 0xD1B54A32D192ED03ull;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z = splitmix_finalize(base + (uint64_t)t);
        const int64_t i = t / J, j = t % J;
        T v;
        if constexpr (sizeof(T) == 8) v = (T)((double)(z >> 11) * 0x1.0p-53);
        else v = (T)((float)(z >> 40) * 0x1.0p-24f);
        out[i * ld + j] = v;
    }
}

void launch_init_uniform(void* out, int elem_bytes, int64_t rows, int J, int ld, uint64_t seed, uint64_t stream,
                         cudaStream_t st) {
    const int64_t total = rows * J;
    int grid = (int)((total + 255) / 256);
    if (grid > 148 * 32) grid = 148 * 32;
    if (grid < 1) grid = 1;
    if (elem_bytes == 8) k_init_uniform<double><<<grid, 256, 0, st>>>((double*)out, rows, J, ld, seed, stream);
    else k_init_uniform<float><<<grid, 256, 0, st>>>((float*)out, rows, J, ld, seed, stream);
}

// ---------------------------------------------------------------------------
// Core permuted for mode n (Eq. 12 groups beta by beta_n = j): the other modes
// m_0 < ... < m_{N-2} become k_0..k_{N-2}; Gp[o][k_{N-2}][j] with o the
// row-major index of (k_0..k_{N-3}); each J x J block padded to gblk.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_permute_core(const T* G, T* Gp, int N, int J, int n, int GB, int64_t nblocks) {
    const int64_t total = nblocks * GB;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = t / GB;
        const int w = (int)(t % GB);
        if (w >= J * J) { Gp[t] = T(0); continue; }
        int k[kMaxN];
        k[N - 2] = w / J;
        const int j = w % J;
        int64_t rem = o;
        for (int l = N - 3; l >= 0; --l) { k[l] = (int)(rem % J); rem /= J; }
        // assemble beta in C order
        int64_t beta = 0;
        int l = 0;
        for (int m = 0; m < N; ++m) {
            const int bm = (m == n) ? j : k[l++];
            beta = beta * J + bm;
        }
        Gp[t] = G[beta];
    }
}

void launch_permute_core(const void* G, void* Gp, int elem_bytes, int N, int J, int n, cudaStream_t st) {
    int64_t nblocks = 1;
    for (int l = 0; l < N - 2; ++l) nblocks *= J;
    const int GB = gblk(J, elem_bytes);
    const int64_t total = nblocks * GB;
    const int grid = (int)((total + 255) / 256);
    if (elem_bytes == 8) k_permute_core<double><<<grid, 256, 0, st>>>((const double*)G, (double*)Gp, N, J, n, GB, nblocks);
    else k_permute_core<float><<<grid, 256, 0, st>>>((const float*)G, (float*)Gp, N, J, n, GB, nblocks);
}

// ---------------------------------------------------------------------------
// Generic small fp64 Cholesky solve (runtime J <= 16), used once per heavy row.
// ---------------------------------------------------------------------------
__device__ bool chol_solve_rt(const double* rec, int J, double lam, double* a) {
    double L[16][16];
    double y[16];
    int q = 0;
    for (int i = 0; i < J; ++i)
        for (int j = i; j < J; ++j) { L[j][i] = rec[q]; ++q; }  // lower part holds M[j][i] = B[i][j]
    const double* c = rec + q;
    bool ok = true;
    for (int j = 0; j < J; ++j) {
        double d = L[j][j] + lam;
        for (int k = 0; k < j; ++k) d = fma(-L[j][k], L[j][k], d);
        ok = ok && (d > 0.0);
        const double l = sqrt(fmax(d, 1e-300));
        L[j][j] = l;
        const double il = 1.0 / l;
        for (int i = j + 1; i < J; ++i) {
            double s = L[i][j];
            for (int k = 0; k < j; ++k) s = fma(-L[i][k], L[j][k], s);
            L[i][j] = s * il;
        }
    }
    for (int i = 0; i < J; ++i) {
        double s = c[i];
        for (int k = 0; k < i; ++k) s = fma(-L[i][k], y[k], s);
        y[i] = s / L[i][i];
    }
    for (int i = J - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < J; ++k) s = fma(-L[k][i], a[k], s);
        a[i] = s / L[i][i];
    }
    return ok;
}

// Heavy rows: the partial records of a row's segments are stored component-major
// (partials[pbase + p*nseg + s]).  Stage 1: one warp per (row, component): lane l adds
// segments l, l+32, ... into four interleaved accumulators (more loads in flight),
// combined in a fixed order, then a fixed xor-butterfly -- the result depends only on
// the row's own segments (F9).  Stage 2: one thread per row solves in registers.
// Rows with at most kSmallSeg segments: one thread per (row, component), the segments
// added in order (many short heavy rows, e.g. a small seg_len); longer rows: a warp each.
constexpr int kSmallSeg = 64;
__global__ void __launch_bounds__(256) k_heavy_sum_small(int64_t nheavy, int PW, const int32_t* hnseg,
                                                         const int64_t* hpbase, const double* partials,
                                                         double* rec) {
    pdl_trigger_early();
    pdl_wait_trigger();
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nheavy * PW;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = w / PW;
        const int nseg = hnseg[h];
        if (nseg > kSmallSeg) continue;
        const int p = (int)(w % PW);
        const double* src = partials + hpbase[h] + (int64_t)p * nseg;
        double acc = 0.0;
        for (int s = 0; s < nseg; ++s) acc += src[s];
        rec[w] = acc;
    }
}

__global__ void __launch_bounds__(256) k_heavy_sum(int64_t nheavy, int PW, const int32_t* hnseg,
                                                   const int64_t* hpbase, const double* partials, double* rec) {
    pdl_trigger_early();
    pdl_wait_trigger();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nheavy * PW; w += nw) {
        const int64_t h = w / PW;
        const int p = (int)(w % PW);
        const int nseg = hnseg[h];
        if (nseg <= kSmallSeg) continue;
        const double* src = partials + hpbase[h] + (int64_t)p * nseg;
        // eight interleaved accumulators (eight loads in flight per lane: the sum is latency-bound,
        // c3's table-mode rows have ~7,800 segments), combined in a fixed order
        double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        int s = lane;
        for (; s + 224 < nseg; s += 256) {
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] += __ldcg(src + s + 32 * u);
        }
        for (; s < nseg; s += 32) a[0] += __ldcg(src + s);
        double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) rec[w] = acc;
    }
}

// JC > 0: the solve in registers (chol_solve<JC>, update.cuh); JC = 0: runtime J <= 16.
template <typename T, int JC>
__device__ __forceinline__ void heavy_solve_row(const double* rec, int J, int row, double lambda, T* An, int lda,
                                                double* sse_row, int* fail, const PeerRows& peers);

template <typename T, int JC>
__global__ void __launch_bounds__(128) k_heavy_solve(int64_t nheavy, const int32_t* hrow, const double* recs, int J,
                                                     double lambda, T* An, int lda, double* sse_row, int* fail,
                                                     const PeerRows peers) {
    pdl_trigger_early();
    pdl_wait_trigger();
    const int PW = J * (J + 1) / 2 + J + 1;
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nheavy; h += (int64_t)gridDim.x * blockDim.x)
        heavy_solve_row<T, JC>(recs + h * PW, J, hrow[h], lambda, An, lda, sse_row, fail, peers);
}

// Heavy rows with at most kSmallSeg segments each, one launch (small tensors whose
// automatic S makes most rows heavy: c1, c2): a thread per row sums its segments' records
// in segment order -- the additions of k_heavy_sum_small, so the same bits -- straight into
// registers (segments outer, the PW independent components inner: PW loads in flight per
// segment) and solves.  (Round 2's warp per row with lane 0 solving ran 31 us per c2 mode:
// 5.6 waves of one serial solve per warp.)
template <typename T, int JC>
__global__ void __launch_bounds__(64) k_heavy_thread(int64_t nheavy, const int32_t* hrow, const int32_t* hnseg,
                                                     const int64_t* hpbase, const double* partials, double lambda,
                                                     T* An, int lda, double* sse_row, int* fail, const PeerRows peers) {
    pdl_trigger_early();
    pdl_wait_trigger();
    constexpr int NB = JC * (JC + 1) / 2;
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nheavy; h += (int64_t)gridDim.x * blockDim.x) {
        const int nseg = hnseg[h];
        const double* src = partials + hpbase[h];
        double B[NB], c[JC], s2 = 0.0;
#pragma unroll
        for (int q = 0; q < NB; ++q) B[q] = 0.0;
#pragma unroll
        for (int q = 0; q < JC; ++q) c[q] = 0.0;
        for (int s = 0; s < nseg; ++s) {
#pragma unroll
            for (int q = 0; q < NB; ++q) B[q] += __ldg(src + (int64_t)q * nseg + s);
#pragma unroll
            for (int q = 0; q < JC; ++q) c[q] += __ldg(src + (int64_t)(NB + q) * nseg + s);
            s2 += __ldg(src + (int64_t)(NB + JC) * nseg + s);
        }
        const int row = hrow[h];
        double a[JC];
        const bool ok = chol_solve<JC>(B, c, lambda, a);
        if (!ok) {
            atomicCAS(fail, 0, row + 1);
#pragma unroll
            for (int j = 0; j < JC; ++j) a[j] = 0.0;
        }
        T* out = An + (int64_t)row * lda;
        double sse = s2, ac = 0.0, aa = 0.0, ec = 0.0;
#pragma unroll
        for (int j = 0; j < JC; ++j) {
            const T st = T(a[j]);
            out[j] = st;
            const double at = double(st);
            sse = fma(-2.0 * at, c[j], sse);
            ac = fma(a[j], c[j], ac);
            aa = fma(a[j], a[j], aa);
            ec = fma(at - a[j], c[j] - lambda * a[j], ec);
        }
        sse_row[row] = sse + (ac - lambda * aa + 2.0 * ec);  // heavy_solve_row's expression
        push_row(peers, out, row, lda * (int)sizeof(T));
    }
}

// Few such heavy rows (c1: 100 per mode, fewer than the GPU's thread slots would fill): a
// warp per row, lane l summing components
// l, l + 32, ... over the row's segments in order -- the additions of k_heavy_sum_small, so
// the same bits -- into shared memory, then lane 0 solves from there.
template <typename T, int JC>
__global__ void __launch_bounds__(128) k_heavy_warp(int64_t nheavy, const int32_t* hrow, const int32_t* hnseg,
                                                    const int64_t* hpbase, const double* partials, double lambda,
                                                    T* An, int lda, double* sse_row, int* fail, const PeerRows peers) {
    pdl_trigger_early();
    pdl_wait_trigger();
    constexpr int PW = JC * (JC + 1) / 2 + JC + 1;
    __shared__ double rec[4][PW];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t h = (int64_t)blockIdx.x * 4 + w; h < nheavy; h += (int64_t)gridDim.x * 4) {
        const int nseg = hnseg[h];
        const double* src = partials + hpbase[h];
        for (int q = lane; q < PW; q += 32) {
            const double* sq = src + (int64_t)q * nseg;
            double acc = 0.0;
            for (int s = 0; s < nseg; ++s) acc += sq[s];
            rec[w][q] = acc;
        }
        __syncwarp();
        if (lane == 0) heavy_solve_row<T, JC>(rec[w], JC, hrow[h], lambda, An, lda, sse_row, fail, peers);
        __syncwarp();
    }
}

// Eq. 9 (Cholesky) for one heavy row from its summed record, the stored row, its SSE by
// the identity of update.cuh, and the push into the peer replicas.
template <typename T, int JC>
__device__ __forceinline__ void heavy_solve_row(const double* rec, int J, int row, double lambda, T* An, int lda,
                                                double* sse_row, int* fail, const PeerRows& peers) {
    {
        double a[16];
        bool ok;
        if constexpr (JC > 0) {
            double B[JC * (JC + 1) / 2], c[JC], x[JC];
#pragma unroll
            for (int q = 0; q < JC * (JC + 1) / 2; ++q) B[q] = rec[q];
#pragma unroll
            for (int q = 0; q < JC; ++q) c[q] = rec[JC * (JC + 1) / 2 + q];
            ok = chol_solve<JC>(B, c, lambda, x);
#pragma unroll
            for (int q = 0; q < JC; ++q) a[q] = x[q];
        } else {
            ok = chol_solve_rt(rec, J, lambda, a);
        }
        // compile-time J when instantiated for one (the fused record stays in registers)
        const int Jr = JC > 0 ? JC : J;
        if (!ok) {
            atomicCAS(fail, 0, row + 1);
#pragma unroll
            for (int j = 0; j < Jr; ++j) a[j] = 0.0;
        }
        const int NB = Jr * (Jr + 1) / 2;
        const double* c = rec + NB;
        double sse = rec[NB + Jr], ac = 0.0, aa = 0.0, ec = 0.0;
        PT_CHK(row >= 0);
        T* out = An + (int64_t)row * lda;
#pragma unroll
        for (int j = 0; j < Jr; ++j) {
            const T st = T(a[j]);
            out[j] = st;
            const double at = double(st);
            sse = fma(-2.0 * at, c[j], sse);
            ac = fma(a[j], c[j], ac);
            aa = fma(a[j], a[j], aa);
            ec = fma(at - a[j], c[j] - lambda * a[j], ec);
        }
        sse_row[row] = sse + (ac - lambda * aa + 2.0 * ec);  // the update kernels' expression (same bits inline)
        push_row(peers, out, row, lda * (int)sizeof(T));
    }
}

void launch_heavy_finalize(int64_t nheavy, const int32_t* hrow, const int32_t* hnseg, const int64_t* hpbase,
                           const double* partials, double* rec, int J, double lambda, void* An, int elem_bytes,
                           int lda, double* sse_row, int* fail, cudaStream_t st, const PeerRows& peers,
                           int64_t max_seg, int64_t min_seg) {
    if (nheavy <= 0) return;
    if (max_seg <= kSmallSeg && (J == 2 || J == 3 || J == 4 || J == 5 || J == 8 || J == 10)) {
        // many rows: a thread per row (c2: 31 -> 15 us per mode); few rows: a warp per row (c1: the
        // thread version's one-thread serial sums ran 23 us against 8.6); the same bits either way
        if (nheavy < 148 * 16) {
            const unsigned gw = (unsigned)std::min<int64_t>((nheavy + 3) / 4, 148 * 32);
#define PT_HFW(JC)                                                                                               \
    if (elem_bytes == 8)                                                                                         \
        launch_pdl(k_heavy_warp<double, JC>, gw, 128, 0, st, nheavy, hrow, hnseg, hpbase, partials, lambda, (double*)An,   \
                                                     lda, sse_row, fail, peers);                                 \
    else                                                                                                         \
        launch_pdl(k_heavy_warp<float, JC>, gw, 128, 0, st, nheavy, hrow, hnseg, hpbase, partials, lambda, (float*)An,     \
                                                    lda, sse_row, fail, peers);
            switch (J) {
                case 2: PT_HFW(2) break;
                case 3: PT_HFW(3) break;
                case 4: PT_HFW(4) break;
                case 5: PT_HFW(5) break;
                case 8: PT_HFW(8) break;
                default: PT_HFW(10) break;
            }
#undef PT_HFW
            return;
        }
        const unsigned gf = (unsigned)std::min<int64_t>((nheavy + 63) / 64, 148 * 16);
#define PT_HFF(JC)                                                                                               \
    if (elem_bytes == 8)                                                                                         \
        launch_pdl(k_heavy_thread<double, JC>, gf, 64, 0, st, nheavy, hrow, hnseg, hpbase, partials, lambda, (double*)An,  \
                                                      lda, sse_row, fail, peers);                                \
    else                                                                                                         \
        launch_pdl(k_heavy_thread<float, JC>, gf, 64, 0, st, nheavy, hrow, hnseg, hpbase, partials, lambda, (float*)An,    \
                                                     lda, sse_row, fail, peers);
        switch (J) {
            case 2: PT_HFF(2) break;
            case 3: PT_HFF(3) break;
            case 4: PT_HFF(4) break;
            case 5: PT_HFF(5) break;
            case 8: PT_HFF(8) break;
            default: PT_HFF(10) break;
        }
#undef PT_HFF
        return;
    }
    const int PW = J * (J + 1) / 2 + J + 1;
    const int64_t nitems = nheavy * PW;
    const unsigned g0 = (unsigned)std::min<int64_t>((nitems + 255) / 256, 148 * 32);
    if (min_seg <= kSmallSeg)  // (some heavy rows short enough for a thread per component)
        launch_pdl(k_heavy_sum_small, g0, 256, 0, st, nheavy, PW, hnseg, hpbase, partials, rec);
    const unsigned g1 = (unsigned)std::min<int64_t>((nitems + 7) / 8, 148 * 32);
    launch_pdl(k_heavy_sum, g1, 256, 0, st, nheavy, PW, hnseg, hpbase, partials, rec);
    const unsigned g2 = (unsigned)std::min<int64_t>((nheavy + 127) / 128, 148 * 16);
#define PT_HF(JC)                                                                                                  \
    if (elem_bytes == 8)                                                                                           \
        launch_pdl(k_heavy_solve<double, JC>, g2, 128, 0, st, nheavy, hrow, rec, J, lambda, (double*)An, lda, sse_row, fail, peers); \
    else                                                                                                           \
        launch_pdl(k_heavy_solve<float, JC>, g2, 128, 0, st, nheavy, hrow, rec, J, lambda, (float*)An, lda, sse_row, fail, peers);
    switch (J) {
        case 2: PT_HF(2) break;
        case 3: PT_HF(3) break;
        case 4: PT_HF(4) break;
        case 5: PT_HF(5) break;
        case 8: PT_HF(8) break;
        case 10: PT_HF(10) break;
        default: PT_HF(0) break;
    }
#undef PT_HF
}

// ---------------------------------------------------------------------------
// Deterministic sum: 256 fixed blocks over contiguous chunks, fixed smem tree,
// then one block over the 256 partials.  Independent of the device and run.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_tree_sum(double v, double* sm) {
    sm[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    return sm[0];
}

__global__ void __launch_bounds__(256) k_sum_stage1(const double* x, int64_t n, double* part) {
    pdl_trigger_early();
    pdl_wait_trigger();
    __shared__ double sm[256];
    const int64_t chunk = (n + 255) / 256;
    const int64_t b0 = blockIdx.x * chunk;
    const int64_t b1 = b0 + chunk < n ? b0 + chunk : n;
    double acc = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += 256) acc += x[i];
    const double s = block_tree_sum(acc, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_sum_stage2(const double* part, double* out) {
    pdl_trigger_early();
    pdl_wait_trigger();
    __shared__ double sm[256];
    const double s = block_tree_sum(part[threadIdx.x], sm);
    if (threadIdx.x == 0) *out = s;
}

void launch_sum(const double* x, int64_t n, double* part256, double* out, cudaStream_t st) {
    launch_pdl(k_sum_stage1, 256, 256, 0, st, x, n, part256);
    launch_pdl(k_sum_stage2, 1, 256, 0, st, part256, out);
}

// ---------------------------------------------------------------------------
// QR (Eq. 7) by CholeskyQR2 in fp64:
//   W = A^T A, R1 = chol(W)^T, Q1 = A R1^-1; W2 = Q1^T Q1, R2 = chol(W2)^T,
//   Q = Q1 R2^-1, R = R2 R1 (diag > 0 by construction).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_gram_stage1(const T* A, int64_t I, int J, int lda, double* part) {
    // block b covers rows [b*chunk, (b+1)*chunk); rows staged in smem tiles of 64
    __shared__ double tile[64][17];
    const int NB = J * (J + 1) / 2;
    const int64_t chunk = (I + 255) / 256;
    const int64_t r0 = blockIdx.x * chunk;
    const int64_t r1 = r0 + chunk < I ? r0 + chunk : I;
    int pi = 0, pj = 0;
    {
        int q = threadIdx.x, i = 0;
        while (i < J && q >= J - i) { q -= J - i; ++i; }
        pi = i;
        pj = i + q;
    }
    double acc = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += 64) {
        const int nt = (int)((r1 - t0) < 64 ? (r1 - t0) : 64);
        __syncthreads();
        for (int w = threadIdx.x; w < nt * J; w += 256) {
            const int r = w / J, j = w % J;
            tile[r][j] = double(A[(t0 + r) * lda + j]);
        }
        __syncthreads();
        if ((int)threadIdx.x < NB)
            for (int r = 0; r < nt; ++r) acc = fma(tile[r][pi], tile[r][pj], acc);
    }
    if ((int)threadIdx.x < NB) part[(int64_t)blockIdx.x * NB + threadIdx.x] = acc;
}

__global__ void k_gram_stage2(const double* part, int J, double* W) {
    const int NB = J * (J + 1) / 2;
    const int q = threadIdx.x;
    if (q >= NB) return;
    double acc = 0.0;
    for (int b = 0; b < 256; ++b) acc += part[(int64_t)b * NB + q];
    int i = 0, r = q;
    while (r >= J - i) { r -= J - i; ++i; }
    const int j = i + r;
    W[i * J + j] = acc;
    W[j * J + i] = acc;
}

void launch_gram(const void* A, int elem_bytes, bool /*unused*/, int64_t I, int J, int lda, double* part, double* W,
                 cudaStream_t st) {
    if (elem_bytes == 8) k_gram_stage1<double><<<256, 256, 0, st>>>((const double*)A, I, J, lda, part);
    else k_gram_stage1<float><<<256, 256, 0, st>>>((const float*)A, I, J, lda, part);
    k_gram_stage2<<<1, 256, 0, st>>>(part, J, W);
}

// R = L^T with W = L L^T (upper triangular, positive diagonal).
__global__ void k_chol_upper(const double* W, int J, double* R, int* fail, int fail_code) {
    if (threadIdx.x != 0) return;
    double L[16][16];
    double wmax = 0.0;
    for (int i = 0; i < J; ++i) wmax = fmax(wmax, W[i * J + i]);
    bool ok = true;
    for (int j = 0; j < J; ++j) {
        double d = W[j * J + j];
        for (int k = 0; k < j; ++k) d = fma(-L[j][k], L[j][k], d);
        if (!(d > 1e-24 * wmax)) ok = false;  // |R_kk| <= 1e-12 max|A| : rank deficient
        const double l = sqrt(fmax(d, 1e-300));
        L[j][j] = l;
        for (int i = j + 1; i < J; ++i) {
            double s = W[i * J + j];
            for (int k = 0; k < j; ++k) s = fma(-L[i][k], L[j][k], s);
            L[i][j] = s / l;
        }
    }
    for (int i = 0; i < J; ++i)
        for (int j = 0; j < J; ++j) R[i * J + j] = (j >= i) ? L[j][i] : 0.0;
    if (!ok) atomicCAS(fail, 0, fail_code);
}

void launch_chol_upper(const double* W, int J, double* R, int* fail, int fail_code, cudaStream_t st) {
    k_chol_upper<<<1, 32, 0, st>>>(W, J, R, fail, fail_code);
}

// Q = A R^-1 row by row: x R = a  =>  x_j = (a_j - sum_{k<j} x_k R[k][j]) / R[j][j]
template <typename TA, typename TQ>
__global__ void k_apply_rinv(const TA* A, int lda_a, TQ* Q, int lda_q, int64_t I, int J, const double* R) {
    __shared__ double Rs[16 * 16];
    for (int t = threadIdx.x; t < J * J; t += blockDim.x) Rs[t] = R[t];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
        double x[16];
        for (int j = 0; j < J; ++j) {
            double s = double(A[i * lda_a + j]);
            for (int k = 0; k < j; ++k) s = fma(-x[k], Rs[k * J + j], s);
            x[j] = s / Rs[j * J + j];
        }
        for (int j = 0; j < J; ++j) Q[i * lda_q + j] = TQ(x[j]);
    }
}

void launch_apply_rinv(const void* A, int a_bytes, int lda_a, void* Q, int q_bytes, int lda_q, int64_t I, int J,
                       const double* R, cudaStream_t st) {
    int grid = (int)((I + 255) / 256);
    if (grid > 148 * 8) grid = 148 * 8;
    if (grid < 1) grid = 1;
    if (a_bytes == 8 && q_bytes == 8)
        k_apply_rinv<double, double><<<grid, 256, 0, st>>>((const double*)A, lda_a, (double*)Q, lda_q, I, J, R);
    else if (a_bytes == 4 && q_bytes == 8)
        k_apply_rinv<float, double><<<grid, 256, 0, st>>>((const float*)A, lda_a, (double*)Q, lda_q, I, J, R);
    else if (a_bytes == 8 && q_bytes == 4)
        k_apply_rinv<double, float><<<grid, 256, 0, st>>>((const double*)A, lda_a, (float*)Q, lda_q, I, J, R);
    else
        k_apply_rinv<float, float><<<grid, 256, 0, st>>>((const float*)A, lda_a, (float*)Q, lda_q, I, J, R);
}

__global__ void k_mat_upper_mul(const double* R2, const double* R1, double* R, int J) {
    const int t = threadIdx.x;
    if (t >= J * J) return;
    const int i = t / J, j = t % J;
    double s = 0.0;
    for (int k = 0; k < J; ++k) s = fma(R2[i * J + k], R1[k * J + j], s);
    R[t] = s;
}

void launch_mat_upper_mul(const double* R2, const double* R1, double* R, int J, cudaStream_t st) {
    k_mat_upper_mul<<<1, 256, 0, st>>>(R2, R1, R, J);
}

// Eq. 2 with U = R (Eq. 8): G'[..k..] = sum_j R[k][j] G[..j..]   (fp64 accumulation)
template <typename T>
__global__ void k_core_mode_product(const T* G, T* Gout, int N, const JDims jd, int n, const double* R) {
    int64_t inner = 1, total = 1;
    const int J = jd.j[n];  // R is J_n x J_n
    for (int m = n + 1; m < N; ++m) inner *= jd.j[m];
    for (int m = 0; m < N; ++m) total *= jd.j[m];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t in = t % inner;
        const int k = (int)((t / inner) % J);
        const int64_t o = t / (inner * J);
        double s = 0.0;
        for (int j = 0; j < J; ++j) s = fma(R[k * J + j], double(G[(o * J + j) * inner + in]), s);
        Gout[t] = T(s);
    }
}

void launch_core_mode_product(const void* G, void* Gout, int elem_bytes, int N, const JDims& J, int n,
                              const double* R, cudaStream_t st) {
    int64_t total = 1;
    for (int m = 0; m < N; ++m) total *= J.j[m];
    const int grid = (int)((total + 255) / 256);
    if (elem_bytes == 8) k_core_mode_product<double><<<grid, 256, 0, st>>>((const double*)G, (double*)Gout, N, J, n, R);
    else k_core_mode_product<float><<<grid, 256, 0, st>>>((const float*)G, (float*)Gout, N, J, n, R);
}

// Rows of a J = 10 fp32 factor (48-byte padded) split for the tensor-core kernel's
// gathers: 32-byte heads and 8-byte tails, 40 of 48 bytes per row, so the two tables a
// mode update gathers from (80 MB at c5) fit the L2 set-aside.
__global__ void k_pack_rows10(const float* __restrict__ A, int64_t I, int lda, float4* __restrict__ head,
                              float2* __restrict__ tail) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
        const float4* r = reinterpret_cast<const float4*>(A + i * lda);
        head[2 * i] = r[0];
        head[2 * i + 1] = r[1];
        tail[i] = *reinterpret_cast<const float2*>(A + i * lda + 8);
    }
}

void launch_pack_rows10(const float* A, int64_t I, int lda, float* head, float* tail, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>((I + 255) / 256, 148 * 16);
    if (grid > 0)
        k_pack_rows10<<<grid, 256, 0, st>>>(A, I, lda, reinterpret_cast<float4*>(head), reinterpret_cast<float2*>(tail));
}

// ---------------------------------------------------------------------------
// Input validation of ptucker_init on the device: the first entry with a coordinate out
// of range (key entry * 16 + mode, the lowest mode of that entry) and the first entry with
// a non-finite value, by atomicMin; per-block sums of x^2 over a fixed grid (the host adds
// the block sums in order: a deterministic sqrt(sum x^2) for reading R30).
// ---------------------------------------------------------------------------
struct DimsArg {
    int64_t d[kMaxN];
};
template <typename T>
__global__ void __launch_bounds__(256) k_validate_coo(const int32_t* __restrict__ coords, const T* __restrict__ vals,
                                                      int64_t nnz, int N, const DimsArg dims,
                                                      unsigned long long* bad, double* part) {
    __shared__ double sm[256];
    double sq = 0.0;
    unsigned long long bc = ~0ull, bv = ~0ull;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        for (int n = 0; n < N; ++n) {
            const int32_t c = coords[e * N + n];
            if (c < 0 || c >= dims.d[n]) {
                bc = min(bc, (unsigned long long)(e * 16 + n));
                break;
            }
        }
        const double v = (double)vals[e];
        if (!isfinite(v)) bv = min(bv, (unsigned long long)e);
        else sq += v * v;
    }
    if (bc != ~0ull) atomicMin(bad, bc);
    if (bv != ~0ull) atomicMin(bad + 1, bv);
    sm[threadIdx.x] = sq;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

void launch_validate_coo(const int32_t* coords, const void* vals, int elem_bytes, int64_t nnz, int N,
                         const int64_t* dims, int64_t* bad, double* part, int grid, cudaStream_t st) {
    DimsArg da;
    for (int n = 0; n < kMaxN; ++n) da.d[n] = n < N ? dims[n] : 0;
    cudaMemsetAsync(bad, 0xFF, 2 * sizeof(int64_t), st);  // all bits set = no offending entry
    if (elem_bytes == 8)
        k_validate_coo<double><<<grid, 256, 0, st>>>(coords, (const double*)vals, nnz, N, da,
                                                     reinterpret_cast<unsigned long long*>(bad), part);
    else
        k_validate_coo<float><<<grid, 256, 0, st>>>(coords, (const float*)vals, nnz, N, da,
                                                    reinterpret_cast<unsigned long long*>(bad), part);
}

}  // namespace pt
