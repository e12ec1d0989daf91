// update.cuh -- the fused row-update kernel of P-Tucker (Alg. 3 lines 6-15).
//
// One warp owns a slice of 32 row segments (rows sorted by length, SELL-32
// layout); each LANE streams the entries of its own segment and, per entry,
//   (1) gathers the N-1 other factor rows a^(k)_{i_k}                  (Eq. 12)
//   (2) contracts the core with them as a depth-first TTV chain,
//       delta(j) = sum_{k_0} a0[k_0] ( ... sum_{k_{N-2}} G'[k..][j] a_{N-2}[k_{N-2}] )
//       -- exactly Eq. 12's sum over beta with beta_n = j, regrouped so every
//       core element is used once per entry (J^N + ... + J^2 FMAs instead of
//       the paper's N*J^N); the core sits in shared memory and every
//       lane reads the same element at the same time (broadcast LDS.128);
//   (3) accumulates B += delta delta^T (upper triangle), c += x delta and
//       sum x^2 in fp64 registers                                 (Eq. 10-11)
// and at the end of the segment either solves a = c [B + lambda I]^-1 by an
// in-register fp64 Cholesky (Eq. 9) and stores the row plus its SSE by the
// identity sum x^2 - 2 a.c + a B a^T (fused Eq. 5), or -- for segments of a
// heavy row -- writes its partial (B, c, sum x^2) for k_heavy_finalize.
//
// The LITERAL variant (mode 0 only) reuses (1)-(2) and accumulates the
// residual (x - a^(0)_{i_0} . delta)^2 per lane instead: the literal Eq. 5 pass.
#pragma once
#include <type_traits>

#include "internal.cuh"

namespace pt {

// The permuted core of the mode being updated, when it fits the 64 KB constant
// bank: every lane of a warp reads the same element at the same time, so the
// compiler feeds the FFMAs from uniform registers (LDCU.128 -> FFMA R,R,UR,R)
// without spending per-thread registers or shared-memory bandwidth on it.
// One copy per translation unit (static); filled by set_core_constant().
static __constant__ __align__(16) unsigned char c_core[65536];

// L64 = N - 3 at order 5 (policy F32-C2).  With the core offset computed from the level-0 loop
// counter nvcc addressed the constant bank through a per-thread register there
// (LDC R, c[0x3][R]: every core read a per-thread constant load, 5.1 ms per c4 mode);
// PT_C2_SMEM = 1 moved the core to shared memory for this policy (3.2 ms).  PT_C2_LOOP = 1
// (default) keeps it in the constant bank and walks it with a pointer of its own, levels 0
// and 1 as runtime loops: the reads are LDCU c[0x3][UR] again (2.60 ms; F32-C 2.74).
// PT_C2_LOOP = 2 unrolls level 1 (same time, 5x the code); 3 unrolls levels 0 and 1 (LDCU.128
// reads, but 124 KB of code and spills: 3.15 ms).
#ifndef PT_C2_SMEM
#define PT_C2_SMEM 0
#endif
#ifndef PT_C2_LOOP
#define PT_C2_LOOP 1
#endif
template <typename TS, int N, int J, int L64 = -1>
struct CoreInConst {
    static constexpr bool value = (size_t)ipow(J, N - 2) * gblk(J, sizeof(TS)) * sizeof(TS) <= sizeof(c_core) &&
                                  !(PT_C2_SMEM && N == 5 && L64 == N - 3);
};

// float -> double by integer operations (ALU pipe) instead of the quarter-rate XU
// conversion: exact for normal floats of either sign; zero or subnormal inputs become
// +-2^-127 (1 + m) (absolute error < 1.2e-38).  Used for half of the fp32 -> fp64
// conversions between TTV levels so that neither pipe saturates.
__device__ __forceinline__ double f2d_alu(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t hi = ((uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu) + 0x38000000u;
    return __hiloint2double((int)hi, (int)(u << 29));
}
// float -> double scaled by 2^-896 in three integer operations (no exponent rebias): exact for
// every finite float, zero and subnormals included (the fp64 bias replaces the fp32 one);
// the caller multiplies the other factor by 2^896 (exact).  Same construction as
// update_tc.cu's f2d_scaled.
__device__ __forceinline__ double f2d_scaled896(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t hi = (uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu;
    return __hiloint2double((int)hi, (int)(u << 29));
}
// TO(x) for the level outputs.  The ALU kernel is issue-bound at two CTAs per SM (c4:
// issue active 75%), so the one-instruction XU conversion wins over f2d_alu's four
// (c4 3.46 -> 2.78 ms per mode); -DPT_F2D_ALU puts half of them on the ALU pipe.
template <typename TO, typename TI>
__device__ __forceinline__ TO widen(TI x, int j) {
    if constexpr (std::is_same<TO, double>::value && std::is_same<TI, float>::value) {
#ifdef PT_F2D_ALU
        return (j & 1) ? f2d_alu(x) : double(x);
#else
        (void)j;
        return double(x);
#endif
    } else {
        return TO(x);
    }
}

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

template <typename T>
__device__ __forceinline__ void unpack(const typename Vec16<T>::type& v, T* e);
template <>
__device__ __forceinline__ void unpack<float>(const float4& v, float* e) { e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w; }
template <>
__device__ __forceinline__ void unpack<double>(const double2& v, double* e) { e[0] = v.x; e[1] = v.y; }

// Innermost TTV stage over one padded J x J core block g = [k][j]:
//   r[j] = sum_k g[k][j] * ak[k]   (sequential in k for each j; J independent chains)
template <typename TS, int J, typename TAcc, typename TA>
__device__ __forceinline__ void ttv_inner(const TS* __restrict__ g, const TA (&ak)[J], TAcc (&r)[J]) {
    using V = typename Vec16<TS>::type;
    constexpr int VN = Vec16<TS>::n;
    constexpr int NV = (J * J + VN - 1) / VN;
    const V* gv = reinterpret_cast<const V*>(g);
#pragma unroll
    for (int j = 0; j < J; ++j) r[j] = TAcc(0);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        TS e[VN];
        unpack<TS>(gv[q], e);
#pragma unroll
        for (int u = 0; u < VN; ++u) {
            const int idx = q * VN + u;
            if (idx < J * J) {
                const int k = idx / J, j = idx % J;
                r[j] = fma(TAcc(e[u]), TAcc(ak[k]), r[j]);
            }
        }
    }
}

// Precision policy: the innermost TTV stage (level
// N-2, J^N of the J^N + ... + J^2 FMAs) always runs in TF; outer level L
// accumulates in fp64 when L < L64 (L64 = number of outer levels in fp64,
// counted from level 0: 0 = "F32-A", 1 = "F32-B", N-2 = "F32-C").
template <typename TF, int L, int L64>
using LevelT = typename std::conditional<(L < L64) || std::is_same<TF, double>::value, double, TF>::type;

// Outer levels L = 1 .. N-3 of the chain (compile-time unrolled).  a_out[L] is
// the raw row of the L-th other mode, a_in the innermost row.  The child block
// stride of level L is J^(N-3-L) padded blocks.
template <typename TS, typename TF, int N, int J, int L64, int L>
__device__ __forceinline__ void ttv_level(const TS* __restrict__ g, const TF (&a_in)[J],
                                          const TS (&a_out)[N - 1][J], LevelT<TF, L, L64> (&r)[J]) {
    using TO = LevelT<TF, L, L64>;
    constexpr int GB = gblk(J, sizeof(TS));
    constexpr int sub = ipow(J, N - 3 - L) * GB;
#pragma unroll
    for (int j = 0; j < J; ++j) r[j] = TO(0);
#pragma unroll
    for (int k = 0; k < J; ++k) {
        TO t[J];
        if constexpr (L + 1 == N - 2) {
            TF ti[J];
            ttv_inner<TS, J, TF, TF>(g + k * sub, a_in, ti);
#pragma unroll
            for (int j = 0; j < J; ++j) t[j] = widen<TO>(ti[j], j);
        } else {
            LevelT<TF, L + 1, L64> tc[J];
            ttv_level<TS, TF, N, J, L64, L + 1>(g + k * sub, a_in, a_out, tc);
#pragma unroll
            for (int j = 0; j < J; ++j) t[j] = TO(tc[j]);
        }
        const TO ak = TO(a_out[L][k]);
#pragma unroll
        for (int j = 0; j < J; ++j) r[j] = fma(ak, t[j], r[j]);
    }
}

// delta for one entry, in LevelT<TF, 0, L64>.  For N >= 4 level 0 is a runtime
// loop reading a0[k] from the entry's staged row in smem.
template <typename TS, typename TF, int N, int J, int L64>
__device__ __forceinline__ void compute_delta(const TS* __restrict__ g, const TF (&a_in)[J],
                                              const TS (&a_out)[N - 1][J], const TS* __restrict__ a0row,
                                              LevelT<TF, 0, L64> (&d)[J]) {
    using TO = LevelT<TF, 0, L64>;
    constexpr int GB = gblk(J, sizeof(TS));
    if constexpr (N == 2) {
        ttv_inner<TS, J, TO, TF>(g, a_in, d);
    } else if constexpr (N == 3) {
#pragma unroll
        for (int j = 0; j < J; ++j) d[j] = TO(0);
        auto level0 = [&](int k) {
            TF t[J];
            ttv_inner<TS, J, TF, TF>(g + k * GB, a_in, t);
            const TO ak = TO(a_out[0][k]);
#pragma unroll
            for (int j = 0; j < J; ++j) d[j] = fma(ak, widen<TO>(t[j], j), d[j]);
        };
        if constexpr (sizeof(TS) == 8 && J >= 8) {
            // fp64 with J >= 8: the fully unrolled k loop held ~2 core blocks of doubles beside
            // the 55-double B and spilled 472 bytes (round 1); one block at a time does not.
            // a0[k] comes from the staged row (a register array indexed by a runtime k would
            // go to local memory)
            constexpr int VN = Vec16<TS>::n;
#pragma unroll 1
            for (int k = 0; k < J; ++k) {
                TF t[J];
                ttv_inner<TS, J, TF, TF>(g + k * GB, a_in, t);
                const TO ak = TO(a0row[(k / VN) * (kWarp * VN) + (k % VN)]);
#pragma unroll
                for (int j = 0; j < J; ++j) d[j] = fma(ak, widen<TO>(t[j], j), d[j]);
            }
        } else {
#pragma unroll
            for (int k = 0; k < J; ++k) level0(k);
        }
    } else if constexpr (PT_C2_LOOP && N == 5 && L64 == N - 3 && sizeof(TS) == 4) {
        // F32-C2 at order 5: levels 0 and 1 as runtime loops (a0[k0], a1[k1] from the staged
        // rows), so the unrolled body is one level-2 block (J^3 + J^2 fp32 FMAs) whose core
        // offset is a loop counter; same products in the same order as the unrolled level 1
        constexpr int sub0 = ipow(J, N - 3) * GB, sub1 = ipow(J, N - 4) * GB;
        constexpr int VN = Vec16<TS>::n;
        constexpr int NQ = factor_ld(J, sizeof(TS)) * (int)sizeof(TS) / 16;  // Stage<TS, N, J>::NQ
        const TS* a1row = a0row + NQ * kWarp * VN;
#pragma unroll
        for (int j = 0; j < J; ++j) d[j] = TO(0);
        static_assert(sub0 == J * sub1, "level-1 blocks are contiguous");
        const TS* gp = g;  // walks the core block by block (its own counter: uniform datapath)
        const TS* const gend = g + J * sub0;
#if PT_C2_LOOP == 3
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int k0 = 0; PT_C2_LOOP == 3 ? k0 < J : gp != gend; ++k0) {
            TO t1[J];
#pragma unroll
            for (int j = 0; j < J; ++j) t1[j] = TO(0);
#if PT_C2_LOOP >= 2
#pragma unroll
#else
#pragma unroll 1
#endif
            for (int k1 = 0; k1 < J; ++k1, gp += sub1) {
                TF t2[J];
                ttv_level<TS, TF, N, J, L64, 2>(gp, a_in, a_out, t2);
                const TO ak1 = TO(a1row[(k1 / VN) * (kWarp * VN) + (k1 % VN)]);
#pragma unroll
                for (int j = 0; j < J; ++j) t1[j] = fma(ak1, TO(t2[j]), t1[j]);
            }
            const TO ak0 = TO(a0row[(k0 / VN) * (kWarp * VN) + (k0 % VN)]);
#pragma unroll
            for (int j = 0; j < J; ++j) d[j] = fma(ak0, t1[j], d[j]);
        }
    } else {
        constexpr int sub = ipow(J, N - 3) * GB;
#pragma unroll
        for (int j = 0; j < J; ++j) d[j] = TO(0);
#pragma unroll 1
        for (int k = 0; k < J; ++k) {
            LevelT<TF, 1, L64> t[J];
            ttv_level<TS, TF, N, J, L64, 1>(g + k * sub, a_in, a_out, t);
            constexpr int VN = Vec16<TS>::n;
            const TO ak = TO(a0row[(k / VN) * (kWarp * VN) + (k % VN)]);  // lane-interleaved stage layout
#pragma unroll
            for (int j = 0; j < J; ++j) d[j] = fma(ak, TO(t[j]), d[j]);
        }
    }
}

__host__ __device__ constexpr int up_idx(int i, int j, int J) { return i * J - i * (i - 1) / 2 + (j - i); }

// Heavy rows finished inside the update kernel (p.seg_done set; rows of at most 64
// segments): the lane that stores a segment's partial (B, c, sum x^2) counts it in
// seg_done[row]; the lane whose count completes the row (a multiple of its segment count:
// the counters are never reset) sums the row's partials in segment order -- the additions
// of k_heavy_warp, so the same bits -- and then solves the row like a one-segment row.
// Replaces the separate finalize launch (c2: 31 us per mode).
template <int J>
__device__ __forceinline__ bool heavy_take_row(int32_t* seg_done, const int64_t* row_pbase, const double* partials,
                                               int row, int nseg, double (&B)[J * (J + 1) / 2], double (&c)[J],
                                               double& s2) {
    constexpr int NB = J * (J + 1) / 2;
    __threadfence();  // this lane's partial stores before its count
    const int old = atomicAdd(seg_done + row, 1);
    if ((old + 1) % nseg != 0) return false;
    __threadfence();  // every other segment's partial (counted before) is visible
    const double* src = partials + row_pbase[row];
#pragma unroll
    for (int q = 0; q < NB + J + 1; ++q) {
        double acc = 0.0;
        for (int s = 0; s < nseg; ++s) acc += __ldcg(src + (int64_t)q * nseg + s);
        if (q < NB) B[q < NB ? q : 0] = acc;
        else if (q < NB + J) c[q < NB + J && q >= NB ? q - NB : 0] = acc;
        else s2 = acc;
    }
    return true;
}

// In-register fp64 Cholesky solve of a (B + lam I) = c (Eq. 9).  B is the
// packed upper triangle; it is overwritten by L^T.  Returns false on a
// non-positive (or NaN) pivot.
template <int J>
__device__ __forceinline__ bool chol_solve(double (&B)[J * (J + 1) / 2], const double (&c)[J], double lam,
                                           double (&a)[J]) {
    bool ok = true;
    double inv[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        double dj = B[up_idx(j, j, J)] + lam;
#pragma unroll
        for (int k = 0; k < j; ++k) dj = fma(-B[up_idx(k, j, J)], B[up_idx(k, j, J)], dj);
        ok = ok && (dj > 0.0);
        const double l = sqrt(fmax(dj, 1e-300));
        inv[j] = 1.0 / l;
#pragma unroll
        for (int i = j + 1; i < J; ++i) {
            double s = B[up_idx(j, i, J)];
#pragma unroll
            for (int k = 0; k < j; ++k) s = fma(-B[up_idx(k, i, J)], B[up_idx(k, j, J)], s);
            B[up_idx(j, i, J)] = s * inv[j];  // L[i][j]
        }
    }
    double y[J];
#pragma unroll
    for (int i = 0; i < J; ++i) {
        double s = c[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s = fma(-B[up_idx(k, i, J)], y[k], s);
        y[i] = s * inv[i];
    }
#pragma unroll
    for (int i = J - 1; i >= 0; --i) {
        double s = y[i];
#pragma unroll
        for (int k = i + 1; k < J; ++k) s = fma(-B[up_idx(i, k, J)], a[k], s);
        a[i] = s * inv[i];
    }
    return ok;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(PENDING) : "memory"); }

// Per-warp staging ring (2 stages) of the gathered factor rows of one entry
// per lane: 16-byte chunk (stage, k, q) of lane l at ((stage*NR + k)*NQ + q)*32 + l,
// so both the cp.async writes and the LDS.128 reads of a warp are conflict-free.
template <typename TS, int N, int J>
struct Stage {
    static constexpr int NR = N - 1;
    static constexpr int NQ = factor_ld(J, sizeof(TS)) * (int)sizeof(TS) / 16;
    static constexpr int CHUNKS_PER_WARP = 2 * NR * NQ * kWarp;
    static constexpr size_t BYTES_PER_WARP = (size_t)CHUNKS_PER_WARP * 16;
};

template <typename TS, int J>
__device__ __forceinline__ void load_row(const TS* __restrict__ row, TS (&out)[J]) {
    using V = typename Vec16<TS>::type;
    constexpr int VN = Vec16<TS>::n;
    constexpr int NV = (J + VN - 1) / VN;
    const V* rv = reinterpret_cast<const V*>(row);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        TS e[VN];
        unpack<TS>(__ldg(rv + q), e);
#pragma unroll
        for (int u = 0; u < VN; ++u)
            if (q * VN + u < J) out[q * VN + u] = e[u];
    }
}

template <typename TS, int J, typename TR>
__device__ __forceinline__ void stage_row(const uint4* __restrict__ chunk0, TR (&out)[J]) {
    using V = typename Vec16<TS>::type;
    constexpr int VN = Vec16<TS>::n;
    constexpr int NV = (J + VN - 1) / VN;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const V v = *reinterpret_cast<const V*>(chunk0 + q * kWarp);
        TS e[VN];
        unpack<TS>(v, e);
#pragma unroll
        for (int u = 0; u < VN; ++u)
            if (q * VN + u < J) out[q * VN + u] = TR(e[u]);
    }
}

__host__ __device__ inline size_t gp_smem_bytes(int gp_elems, int esz) { return ((size_t)gp_elems * esz + 15) / 16 * 16; }

// TABLE: the "core" is a table of blocks in shared memory (small-mode
// precontraction, smp.cu) and each lane contracts with block lane_aux[slot].
// CTAs per SM the update kernel is compiled for: small J keeps its fp64 normal
// equations in <= 128 registers, so two CTAs (16 warps) hide the core-load latency
// (c4: 8 warps per SM left the FFMAs waiting on their LDS.128 operands).
#ifndef PT_UPD_MINB_SMALLJ
#define PT_UPD_MINB_SMALLJ 2
#endif
constexpr int upd_min_blocks(int J, int esz) { return (J <= 5 && esz == 4) ? PT_UPD_MINB_SMALLJ : 1; }

template <typename TS, typename TF, int N, int J, int L64, bool LITERAL, bool TABLE = false>
__global__ void __launch_bounds__(kUpdThreads, upd_min_blocks(J, (int)sizeof(TS))) k_update(const UpdateParams<TS> p) {
    using TD = LevelT<TF, 0, L64>;  // type of delta
    constexpr int NB = J * (J + 1) / 2;
    using V = typename Vec16<TS>::type;
    constexpr int VN = Vec16<TS>::n;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool GC = CoreInConst<TS, N, J, L64>::value && !TABLE;
    const TS* gs;
    if constexpr (GC) {
        gs = reinterpret_cast<const TS*>(c_core);
    } else {
        TS* gsm = reinterpret_cast<TS*>(smem_raw);
        const V* src = reinterpret_cast<const V*>(p.Gp);
        V* dst = reinterpret_cast<V*>(gsm);
        for (int i = threadIdx.x; i < p.gp_elems / VN; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
        gs = gsm;
    }
    const int lane = threadIdx.x & (kWarp - 1);
    using ST = Stage<TS, N, J>;
    constexpr int NR = ST::NR, NQ = ST::NQ;
    uint4* stg = reinterpret_cast<uint4*>(smem_raw + (GC ? 0 : gp_smem_bytes(p.gp_elems, sizeof(TS)))) +
                 (threadIdx.x / kWarp) * ST::CHUNKS_PER_WARP + lane;
    // cp.async the N-1 gathered rows of an entry into stage st
    auto issue_rows = [&](int st, const int (&crd)[NR]) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            PT_CHK(crd[k] >= 0 && crd[k] < p.dim_other[k]);
            const char* src = reinterpret_cast<const char*>(p.A[k] + (int64_t)crd[k] * p.lda);
#pragma unroll
            for (int q = 0; q < NQ; ++q) cp_async16(stg + ((st * NR + k) * NQ + q) * kWarp, src + 16 * q);
        }
        cp_async_commit();
    };

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
        const TS* gl = gs;
        if constexpr (TABLE) gl = gs + (int64_t)p.lane_aux[slot] * p.aux_stride;

        double B[NB], c[J], s2 = 0.0;
#pragma unroll
        for (int q = 0; q < NB; ++q) B[q] = 0.0;
#pragma unroll
        for (int q = 0; q < J; ++q) c[q] = 0.0;
        TS arow[J];
        if constexpr (LITERAL) {
            if (row >= 0) load_row<TS, J>(p.An + (int64_t)row * p.lda, arow);
            else {
#pragma unroll
                for (int q = 0; q < J; ++q) arow[q] = TS(0);
            }
        }

        // software pipeline: coordinates two entries ahead (registers), gathered
        // rows one entry ahead (cp.async into the 2-stage smem ring)
        int crd0[NR], crd1[NR];
        TS x0 = TS(0), x1 = TS(0);
#pragma unroll
        for (int k = 0; k < NR; ++k) crd0[k] = crd1[k] = 0;
        if (iters > 0) {
#pragma unroll
            for (int k = 0; k < NR; ++k) crd0[k] = __ldg(p.sc[k] + base);
            x0 = __ldg(p.sv + base);
            issue_rows(0, crd0);
        }
        if (iters > 1) {
#pragma unroll
            for (int k = 0; k < NR; ++k) crd1[k] = __ldg(p.sc[k] + base + kWarp);
            x1 = __ldg(p.sv + base + kWarp);
        }
        for (int e = 0; e < iters; ++e) {
            const int st = e & 1;
            if (e + 1 < iters) issue_rows(st ^ 1, crd1);
            int crd2[NR];
            TS x2 = TS(0);
            if (e + 2 < iters) {
                const int64_t idx2 = base + (int64_t)(e + 2) * kWarp;
#pragma unroll
                for (int k = 0; k < NR; ++k) crd2[k] = __ldg(p.sc[k] + idx2);
                x2 = __ldg(p.sv + idx2);
            } else {
#pragma unroll
                for (int k = 0; k < NR; ++k) crd2[k] = 0;
            }
            if (e + 1 < iters) cp_async_wait<1>();
            else cp_async_wait<0>();
            const TS x = x0;
            TF a_in[J];
            TS a_out[N - 1][J];
            stage_row<TS, J>(stg + ((st * NR + (NR - 1)) * NQ) * kWarp, a_in);
#pragma unroll
            for (int k = (N >= 4 ? 1 : 0); k < N - 2; ++k) stage_row<TS, J>(stg + ((st * NR + k) * NQ) * kWarp, a_out[k]);
            if constexpr (N >= 4) {
#pragma unroll
                for (int j = 0; j < J; ++j) a_out[0][j] = TS(0);
            }
            TD d[J];
            compute_delta<TS, TF, N, J, L64>(gl, a_in, a_out,
                                            reinterpret_cast<const TS*>(stg + (st * NR) * NQ * kWarp), d);
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                crd0[k] = crd1[k];
                crd1[k] = crd2[k];
            }
            x0 = x1;
            x1 = x2;
            const bool act = e < len;
            if constexpr (!LITERAL) {
                double dd[J];
#pragma unroll
                for (int j = 0; j < J; ++j) dd[j] = act ? double(d[j]) : 0.0;
                const double xd = act ? double(x) : 0.0;
#pragma unroll
                for (int i = 0; i < J; ++i) {
                    c[i] = fma(xd, dd[i], c[i]);
#pragma unroll
                    for (int j = i; j < J; ++j) B[up_idx(i, j, J)] = fma(dd[i], dd[j], B[up_idx(i, j, J)]);
                }
                s2 = fma(xd, xd, s2);
            } else {
                double xh = 0.0;
#pragma unroll
                for (int j = 0; j < J; ++j) xh = fma(double(d[j]), double(arow[j]), xh);
                const double r = act ? double(x) - xh : 0.0;
                s2 = fma(r, r, s2);
            }
        }

        if constexpr (LITERAL) {
            p.lit_part[slot] = s2;
        } else {
            if (row < 0) continue;
            const int64_t pidx = p.lane_pidx[slot];
            bool solve = pidx < 0;
            if (!solve) {
                const int st = p.lane_pstride[slot];
                double* dst = p.partials + pidx;
#pragma unroll
                for (int q = 0; q < NB; ++q) dst[(int64_t)q * st] = B[q];
#pragma unroll
                for (int q = 0; q < J; ++q) dst[(int64_t)(NB + q) * st] = c[q];
                dst[(int64_t)(NB + J) * st] = s2;
                if (p.seg_done) solve = heavy_take_row<J>(p.seg_done, p.row_pbase, p.partials, row, st, B, c, s2);
            }
            if (solve) {
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
                TS st[J];
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    st[j] = TS(a[j]);
                    const double at = double(st[j]);
                    const double eps = at - a[j];
                    sse = fma(-2.0 * at, c[j], sse);
                    ac = fma(a[j], c[j], ac);
                    aa = fma(a[j], a[j], aa);
                    ec = fma(eps, c[j] - p.lambda * a[j], ec);
                }
                // SSE of the stored row (Eq. 5 restricted to the row):
                // s2 - 2 a~.c + a~ B a~^T with a~ B a~^T = a.c - lam|a|^2 + 2 eps.(c - lam a) + O(eps^2)
                sse += ac - p.lambda * aa + 2.0 * ec;
                constexpr int LD = factor_ld(J, sizeof(TS));
#pragma unroll
                for (int q = 0; q < LD / VN; ++q) {
                    TS e4[VN];
#pragma unroll
                    for (int u = 0; u < VN; ++u) e4[u] = (q * VN + u < J) ? st[(q * VN + u) < J ? q * VN + u : 0] : TS(0);
                    V v;
                    if constexpr (VN == 4) v = make_float4(e4[0], e4[1], e4[2], e4[3]);
                    else v = make_double2(e4[0], e4[1]);
                    reinterpret_cast<V*>(out)[q] = v;
                    for (int r = 0; r < p.peers.n; ++r)  // multi-GPU push into the peer replicas
                        reinterpret_cast<V*>(static_cast<char*>(p.peers.base[r]) +
                                             (int64_t)row * p.lda * (int64_t)sizeof(TS))[q] = v;
                }
                p.sse_row[row] = sse;
            }
        }
    }
}

template <typename TS, typename TF, int N, int J, int L64>
void launch_update(const void* params, bool literal, int grid, cudaStream_t st) {
    const UpdateParams<TS>& p = *reinterpret_cast<const UpdateParams<TS>*>(params);
    const size_t smem = (CoreInConst<TS, N, J, L64>::value ? 0 : gp_smem_bytes(p.gp_elems, sizeof(TS))) +
                        (kUpdThreads / kWarp) * Stage<TS, N, J>::BYTES_PER_WARP;
    if (CoreInConst<TS, N, J, L64>::value)
        cudaMemcpyToSymbolAsync(c_core, p.Gp, (size_t)p.gp_elems * sizeof(TS), 0, cudaMemcpyDeviceToDevice, st);
    if (literal) {
        auto k = k_update<TS, TF, N, J, L64, true>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, kUpdThreads, smem, st>>>(p);
    } else {
        auto k = k_update<TS, TF, N, J, L64, false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, kUpdThreads, smem, st>>>(p);
    }
}

template <typename TS, typename TF, int N, int J, int L64>
int occupancy_update(bool literal, size_t gp_bytes) {
    const size_t smem = (CoreInConst<TS, N, J, L64>::value ? 0 : gp_bytes) + (kUpdThreads / kWarp) * Stage<TS, N, J>::BYTES_PER_WARP;
    int nb = 0;
    if (literal) {
        auto k = k_update<TS, TF, N, J, L64, true>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kUpdThreads, smem);
    } else {
        auto k = k_update<TS, TF, N, J, L64, false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kUpdThreads, smem);
    }
    return nb;
}

}  // namespace pt
