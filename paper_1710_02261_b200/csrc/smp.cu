// smp.cu -- small-mode precontraction (SMP) for order-4 tensors with two small modes
// (the MovieLens-shaped c3: 138,000 x 27,000 x 21 x 24).
//
// Eq. 12 for mode n with other modes {r, s1, s2}, where s1 < s2 have
// few rows:
//   delta(j) = sum_{k_r} a_r[k_r] * T[i_s1][i_s2][k_r][j],
//   T[i1][i2][k_r][j] = sum_{k1,k2} G[..j..k_r..k1..k2..] a_s1[i1][k1] a_s2[i2][k2].
// T depends only on the small modes' factors, which do not change while mode n
// (a large mode) is updated, so it is built once per mode update (I_s1*I_s2*J^2
// values, 504 x 100 for c3) and every entry then costs J^2 FMAs instead of
// J^4 + J^3 + J^2 (the per-entry minimum WITHOUT sharing).  This
// is the same sum regrouped; T is accumulated in fp64 and stored in the
// context precision, the per-entry stage runs in fp64.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"
#include "update.cuh"

namespace pt {
namespace smp {

// ---- table build: one thread per output T[i1][i2][k_r][j], fp64 accumulation ----
template <typename TS, typename TT>
__global__ void k_table2(const TS* __restrict__ G, const TS* __restrict__ As1, const TS* __restrict__ As2, int lda,
                         int64_t I1, int64_t I2, int J, int n, int r, int s1, int s2, TT* __restrict__ T) {
    const int64_t total = I1 * I2 * J * J;
    int strideG[4];
    {
        int st = 1;
        for (int m = 3; m >= 0; --m) { strideG[m] = st; st *= J; }
    }
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t % J);
        const int kr = (int)((t / J) % J);
        const int64_t blk = t / (J * J);
        const int64_t i2 = blk % I2, i1 = blk / I2;
        const TS* a1 = As1 + i1 * lda;
        const TS* a2 = As2 + i2 * lda;
        const int64_t base = (int64_t)j * strideG[n] + (int64_t)kr * strideG[r];
        double acc = 0.0;
        for (int k1 = 0; k1 < J; ++k1) {
            double inner = 0.0;
            for (int k2 = 0; k2 < J; ++k2)
                inner = fma(double(G[base + (int64_t)k1 * strideG[s1] + (int64_t)k2 * strideG[s2]]), double(a2[k2]), inner);
            acc = fma(double(a1[k1]), inner, acc);
        }
        T[t] = TT(acc);
    }
}

// ---- row update: lane per row segment (SELL-32, as k_update), per entry
//      delta = a_r^T T[i_s1][i_s2] in fp64; B, c, solve as in k_update ----
// Table source (MODE): 0 = fp32 copy in shared memory; 1 = the fp64 table read
// from global memory (L2-resident, 8*I_s1*I_s2*J^2 bytes) -- exact to fp64 but
// ~4x the time; 2 = hybrid: the fp64 table for single-segment rows of at most
// kSmpLight entries (the light, ill-conditioned rows that dominate the fp32 table's
// rounding error), the fp32 shared-memory copy for all other rows (c3 modes 0/1:
// 1.96/1.64 -> 1.27/0.93 ms; worst sampled full-size row error 6.2e-7 -> 1.5e-6).
#ifndef PT_SMP_LIGHT
#define PT_SMP_LIGHT 32
#endif
constexpr int kSmpLight = PT_SMP_LIGHT;  // hybrid: fp64 table only for single-segment rows this short
#ifndef PT_SMP_THREADS
#define PT_SMP_THREADS kUpdThreads
#endif
constexpr int kSmpThreads = PT_SMP_THREADS;  // one CTA per SM (the fp32 table fills shared memory)
template <typename TS, int J, int MODE>
__global__ void __launch_bounds__(kSmpThreads, 1) k_update_smp2(const UpdateParams<TS> p, const double* __restrict__ T64,
                                                               const TS* __restrict__ T32, int64_t tab_elems, int ir,
                                                               int is1, int is2, int I2) {
    constexpr int NB = J * (J + 1) / 2;
    using V = typename Vec16<TS>::type;
    constexpr int VN = Vec16<TS>::n;
    constexpr int BLK = J * J;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TS* ts = reinterpret_cast<TS*>(smem_raw);
    if constexpr (MODE != 1) {
        const V* src = reinterpret_cast<const V*>(T32);
        V* dst = reinterpret_cast<V*>(ts);
        for (int64_t i = threadIdx.x; i < tab_elems / VN; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & (kWarp - 1);
    for (;;) {
        int s = 0;
        if (lane == 0) s = (int)atomicAdd(p.work, 1u);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= p.nslices) break;
        const int64_t slot = (int64_t)s * kWarp + lane;
        const int row = p.lane_row[slot];
        const int len = p.lane_len[slot];
        const int iters = p.slice_len[s];
        const int64_t base = p.slice_off[s] + lane;
        const bool use64 = MODE == 1 || (MODE == 2 && p.lane_pidx[slot] < 0 && len <= kSmpLight);
        double B[NB], c[J], s2 = 0.0;
#pragma unroll
        for (int q = 0; q < NB; ++q) B[q] = 0.0;
#pragma unroll
        for (int q = 0; q < J; ++q) c[q] = 0.0;
        // the gathered row a_r one entry ahead, the coordinates and value two ahead (the
        // row's address is known an iteration before it is requested: no dependent stall)
        int cr = 0, c1 = 0, c2 = 0;
        TS x = TS(0);
        TS ar[J];
        int mr = 0, m1 = 0, m2 = 0;  // entry e + 1
        TS mx = TS(0);
        auto load = [&](int e, int& r_, int& a_, int& b_, TS& x_) {
            const int64_t idx = base + (int64_t)e * kWarp;
            r_ = __ldg(p.sc[ir] + idx);
            a_ = __ldg(p.sc[is1] + idx);
            b_ = __ldg(p.sc[is2] + idx);
            x_ = __ldg(p.sv + idx);
            PT_CHK(r_ >= 0 && r_ < p.dim_other[ir] && a_ >= 0 && a_ < p.dim_other[is1] && b_ >= 0 &&
                   b_ < p.dim_other[is2]);
        };
        if (iters > 0) {
            load(0, cr, c1, c2, x);
            load_row<TS, J>(p.A[ir] + (int64_t)cr * p.lda, ar);
        }
        if (iters > 1) load(1, mr, m1, m2, mx);
        for (int e = 0; e < iters; ++e) {
            int nr = mr, n1 = m1, n2 = m2;
            TS nx = mx;
            TS nar[J];
            if (e + 1 < iters) load_row<TS, J>(p.A[ir] + (int64_t)nr * p.lda, nar);
            if (e + 2 < iters) load(e + 2, mr, m1, m2, mx);
            const int64_t boff = ((int64_t)c1 * I2 + c2) * BLK;
            double d[J];
#pragma unroll
            for (int j = 0; j < J; ++j) d[j] = 0.0;
            if (use64) {
                const double* tb = T64 + boff;
                if constexpr (BLK % 4 == 0) {
                    // the block (BLK doubles, 32-byte aligned: BLK * 8 is a multiple of 32) in
                    // 256-bit loads: a quarter of the LSU requests of 8-byte loads (the fp64-table
                    // path was LSU-throttled, profiles/r02/smp2_c3_mode0_full.txt)
#pragma unroll
                    for (int q = 0; q < BLK / 4; ++q) {
                        double v[4];
                        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                                     : "l"(tb + 4 * q));
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int kj = 4 * q + u, k = kj / J, j = kj % J;
                            d[j] = fma(double(ar[k]), v[u], d[j]);
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < J; ++k) {
                        const double ak = double(ar[k]);
#pragma unroll
                        for (int j = 0; j < J; ++j) d[j] = fma(ak, __ldg(tb + k * J + j), d[j]);
                    }
                }
            } else {
                const TS* tb = ts + boff;
#pragma unroll
                for (int k = 0; k < J; ++k) {
                    const double ak = double(ar[k]);
                    // odd j: the table value widened exactly by three integer operations into
                    // t * 2^-896 (f2d_scaled below), paired with ak * 2^896 (exact); even j on
                    // the XU (latency-bound kernel: neither pipe saturates)
                    const double aks = ak * 0x1p896;
#pragma unroll
                    for (int j = 0; j < J; ++j) {
#ifndef PT_SMP_F2D_XU
                        if constexpr (std::is_same<TS, float>::value)
                            d[j] = (j & 1) ? fma(aks, f2d_scaled896(tb[k * J + j]), d[j])
                                           : fma(ak, double(tb[k * J + j]), d[j]);
                        else
#endif
                            d[j] = fma(ak, double(tb[k * J + j]), d[j]);
                    }
                }
            }
            if (e < len) {  // inactive lanes (beyond their segment) skip the update
                const double xd = double(x);
#pragma unroll
                for (int i = 0; i < J; ++i) {
                    c[i] = fma(xd, d[i], c[i]);
#pragma unroll
                    for (int j = i; j < J; ++j) B[up_idx(i, j, J)] = fma(d[i], d[j], B[up_idx(i, j, J)]);
                }
                s2 = fma(xd, xd, s2);
            }
            cr = nr; c1 = n1; c2 = n2; x = nx;
#pragma unroll
            for (int j = 0; j < J; ++j) ar[j] = nar[j];
        }
        if (row < 0) continue;
        const int64_t pidx = p.lane_pidx[slot];
        if (pidx < 0) {
            double a[J];
            const bool ok = chol_solve<J>(B, c, p.lambda, a);
            if (!ok) {
                atomicCAS(p.fail, 0, row + 1);
#pragma unroll
                for (int j = 0; j < J; ++j) a[j] = 0.0;
            }
            PT_CHK(row < p.dim_n);
            TS* out = p.An + (int64_t)row * p.lda;
            double sse = s2, ac = 0.0, aa = 0.0, ec = 0.0;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const TS st = TS(a[j]);
                out[j] = st;
                const double at = double(st);
                sse = fma(-2.0 * at, c[j], sse);
                ac = fma(a[j], c[j], ac);
                aa = fma(a[j], a[j], aa);
                ec = fma(at - a[j], c[j] - p.lambda * a[j], ec);
            }
            p.sse_row[row] = sse + ac - p.lambda * aa + 2.0 * ec;
            push_row(p.peers, out, row, p.lda * (int)sizeof(TS));
        } else {
            const int stp = p.lane_pstride[slot];
            double* dst = p.partials + pidx;
#pragma unroll
            for (int q = 0; q < NB; ++q) dst[(int64_t)q * stp] = B[q];
#pragma unroll
            for (int q = 0; q < J; ++q) dst[(int64_t)(NB + q) * stp] = c[q];
            dst[(int64_t)(NB + J) * stp] = s2;
        }
    }
}

// ---- one small other mode s: T[i][k_a][k_b][j] = sum_k G[..j..k_a..k_b..k..] a_s[i][k],
//      laid out as a core permuted for an order-3 problem (blocks [k_a][gblk] with
//      gblk = [k_b][j] padded), one block per small-mode row i ----
template <typename TS>
__global__ void k_table1(const TS* __restrict__ G, const TS* __restrict__ As, int lda, int64_t Is, int J, int n,
                         int a, int b, int sm, int GB, TS* __restrict__ T) {
    const int64_t total = Is * J * GB;
    int strideG[4];
    {
        int st = 1;
        for (int m = 3; m >= 0; --m) { strideG[m] = st; st *= J; }
    }
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(t % GB);
        const int ka = (int)((t / GB) % J);
        const int64_t i = t / ((int64_t)GB * J);
        if (w >= J * J) { T[t] = TS(0); continue; }
        const int kb = w / J, j = w % J;
        const TS* as = As + i * lda;
        const int64_t base = (int64_t)j * strideG[n] + (int64_t)ka * strideG[a] + (int64_t)kb * strideG[b];
        double acc = 0.0;
        for (int k = 0; k < J; ++k) acc = fma(double(G[base + (int64_t)k * strideG[sm]]), double(as[k]), acc);
        T[t] = TS(acc);
    }
}

template <typename TS, int J>
int launch_table_update(const UpdateParams<TS>& p, int nsm, cudaStream_t st) {
    using TF = TS;
    auto k = k_update<TS, TF, 3, J, 1, false, true>;
    const size_t smem = gp_smem_bytes(p.gp_elems, sizeof(TS)) + (kUpdThreads / kWarp) * Stage<TS, 3, J>::BYTES_PER_WARP;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kUpdThreads, smem);
    if (nb < 1) nb = 1;
    k<<<nsm * nb, kUpdThreads, smem, st>>>(p);
    return 0;
}

template <typename TS, int J, int MODE>
int launch_smp2(const UpdateParams<TS>& p, const double* T64, const TS* T32, int64_t tab_elems, int ir, int is1,
                int is2, int I2, int nsm, cudaStream_t st) {
    auto k = k_update_smp2<TS, J, MODE>;
    const size_t smem = MODE == 1 ? 0 : (size_t)tab_elems * sizeof(TS);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kSmpThreads, smem);
    if (nb < 1) nb = 1;
    k<<<nsm * nb, kSmpThreads, smem, st>>>(p, T64, T32, tab_elems, ir, is1, is2, I2);
    return 0;
}

}  // namespace smp

// Host entry points (declared in kernels.cuh).
__global__ void k_round_table(const double* T64, float* T32, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        T32[t] = float(T64[t]);
}

void launch_smp_table2(const void* G, const void* As1, const void* As2, int lda, int64_t I1, int64_t I2, int J, int n,
                       int r, int s1, int s2, double* T64, void* T32, int elem_bytes, cudaStream_t st) {
    const int64_t total = I1 * I2 * J * J;
    int grid = (int)((total + 255) / 256);
    if (elem_bytes == 8)
        smp::k_table2<double, double><<<grid, 256, 0, st>>>((const double*)G, (const double*)As1, (const double*)As2, lda,
                                                            I1, I2, J, n, r, s1, s2, T64);
    else
        smp::k_table2<float, double><<<grid, 256, 0, st>>>((const float*)G, (const float*)As1, (const float*)As2, lda, I1,
                                                           I2, J, n, r, s1, s2, T64);
    if (T32) k_round_table<<<grid, 256, 0, st>>>(T64, (float*)T32, total);
}

void launch_smp_table1(const void* G, const void* As, int lda, int64_t Is, int J, int n, int a, int b, int s, void* T,
                       int elem_bytes, cudaStream_t st) {
    const int GB = gblk(J, elem_bytes);
    const int64_t total = Is * J * GB;
    const int grid = (int)((total + 255) / 256);
    if (elem_bytes == 8)
        smp::k_table1<double><<<grid, 256, 0, st>>>((const double*)G, (const double*)As, lda, Is, J, n, a, b, s, GB,
                                                    (double*)T);
    else
        smp::k_table1<float><<<grid, 256, 0, st>>>((const float*)G, (const float*)As, lda, Is, J, n, a, b, s, GB,
                                                   (float*)T);
}

bool launch_table_update(const void* params, int elem_bytes, int J, int nsm, cudaStream_t st) {
#define PT_TU(JJ)                                                                                              \
    case JJ:                                                                                                  \
        if (elem_bytes == 4)                                                                                  \
            smp::launch_table_update<float, JJ>(*reinterpret_cast<const UpdateParams<float>*>(params), nsm, st); \
        else                                                                                                  \
            smp::launch_table_update<double, JJ>(*reinterpret_cast<const UpdateParams<double>*>(params), nsm, st); \
        return true;
    switch (J) {
        PT_TU(2) PT_TU(3) PT_TU(4) PT_TU(5) PT_TU(8) PT_TU(10)
    }
#undef PT_TU
    return false;
}

bool launch_smp2_update(const void* params, int elem_bytes, int J, const double* T64, const void* T32,
                        int64_t tab_elems, int ir, int is1, int is2, int I2, int mode, int nsm, cudaStream_t st) {
#define PT_S2(JJ)                                                                                                 \
    case JJ:                                                                                                     \
        if (elem_bytes == 4) {                                                                                   \
            const auto& p = *reinterpret_cast<const UpdateParams<float>*>(params);                               \
            const float* t32 = (const float*)T32;                                                                \
            if (mode == 1) smp::launch_smp2<float, JJ, 1>(p, T64, t32, tab_elems, ir, is1, is2, I2, nsm, st);     \
            else if (mode == 2) smp::launch_smp2<float, JJ, 2>(p, T64, t32, tab_elems, ir, is1, is2, I2, nsm, st); \
            else smp::launch_smp2<float, JJ, 0>(p, T64, t32, tab_elems, ir, is1, is2, I2, nsm, st);               \
        } else {                                                                                                 \
            const auto& p = *reinterpret_cast<const UpdateParams<double>*>(params);                              \
            smp::launch_smp2<double, JJ, 1>(p, T64, nullptr, tab_elems, ir, is1, is2, I2, nsm, st);              \
        }                                                                                                        \
        return true;
    switch (J) {
        PT_S2(2) PT_S2(3) PT_S2(4) PT_S2(5) PT_S2(8) PT_S2(10)
    }
#undef PT_S2
    return false;
}

}  // namespace pt
