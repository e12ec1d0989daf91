// update_tc.cu -- row update for order-3 fp32 tensors with the innermost TTV
// stage on the 5th-generation tensor cores (tcgen05, kind::tf32, TMEM
// accumulators).
//
// For mode n with other modes m0 < m1, Eq. 12 regrouped as a TTV
// chain is   delta(j) = sum_k0 a0[k0] * t[k0][j],   t[k0][j] = sum_k1 a1[k1] G'[k0][k1][j].
// The inner stage, over the 128 entries a CTA holds at a time, is a dense GEMM
//     T (128 x J^2) = A1 (128 x J) * Bt^T,   Bt[(k0,j)][k1] = G'[k0][k1][j],
// with B = the core, shared by every entry.  It runs as 3xTF32 (a = a_hi + a_lo,
// small products first: lo*hi, hi*lo, hi*hi) so its accuracy matches an fp32
// FMA chain (tools/tc_probe.cu), accumulating in TMEM.  Each thread owns one
// TMEM lane = one entry of its own row segment (the SELL-32 layout of the ALU
// kernel, 4 slices per CTA), reads its J^2 outputs back with tcgen05.ld and
// finishes level 0 (fp64 under F32-B), B += delta delta^T, c += x delta (fp64,
// Eq. 10-11) and the Cholesky solve (Eq. 9) in registers.  The MMA for the next
// entry is issued before the epilogue of the current one (double-buffered A
// tiles and TMEM accumulators); the next rows are gathered by cp.async two
// entries ahead.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "update.cuh"

namespace pt {
namespace tc {

constexpr int kThreads = 128;  // one TMEM lane per thread; 4 warps = 4 SELL slices

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_NONE canonical layout (8-row x 16-byte core matrices): 32-bit
// element (r, k) of a [rows x KP] tile, in floats.
template <int KP>
__device__ __forceinline__ int kmaj(int r, int k) {
    return (((r >> 3) * (KP / 4) + (k >> 2)) * 128 + (r & 7) * 16 + (k & 3) * 4) / 4;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // sm100 descriptor version; base offset 0; SWIZZLE_NONE
    return d;
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}


__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld4_nowait(uint32_t addr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int J>
struct Shape {
    static constexpr int KP = (J + 7) / 8 * 8;             // K padded to the tf32 MMA K-step (8)
    static constexpr int KSTEPS = KP / 8;
    static constexpr int NP = (J * J + 15) / 16 * 16;      // N padded to 16 (M = 128)
    static constexpr int TCOLS = 2 * NP <= 32 ? 32 : (2 * NP <= 64 ? 64 : (2 * NP <= 128 ? 128 : (2 * NP <= 256 ? 256 : 512)));
    static constexpr int LD = factor_ld(J, 4);             // padded factor row (floats)
    static constexpr int NQ = LD / 4;                       // 16-byte chunks per factor row
    static constexpr int KQ = KP / 4;                       // 16-byte chunks per A row
    static constexpr int STAGES = 3;                        // gather/A-tile pipeline depth
    // shared memory map (bytes)
    static constexpr int B_BYTES = NP * KP * 4;                     // one of B_hi / B_lo
    static constexpr int A_BYTES = kThreads * KP * 4;               // one of A_hi / A_lo (per stage)
    static constexpr int RING_CHUNKS = STAGES * 2 * NQ * kThreads;  // the gathered rows a0, a1
    static constexpr int OFF_BHI = 0;
    static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
    static constexpr int OFF_A = OFF_BLO + B_BYTES;                 // [stage][hi,lo]
    static constexpr int OFF_RING = OFF_A + STAGES * 2 * A_BYTES;
    static constexpr int OFF_BAR = OFF_RING + RING_CHUNKS * 16;     // mbarriers: acc_full[2]
    static constexpr int OFF_MISC = OFF_BAR + 32;                   // tmem base, group id, arrival counters
    static constexpr int SMEM = OFF_MISC + 32;
};

// Split of the innermost factor into tf32 hi/lo parts (3xTF32 operand), K-padded:
// out rows of KP floats, hi = tf32_rna(a), lo = tf32_rna(a - hi), zeros for k >= J.
__global__ void k_split_tf32(const float* __restrict__ A, int64_t I, int lda, int J, int KP, float* __restrict__ hi,
                             float* __restrict__ lo) {
    const int64_t total = I * KP;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / KP;
        const int k = (int)(t % KP);
        const float v = k < J ? A[i * lda + k] : 0.f;
        const float h = tf32_rna(v);
        hi[t] = h;
        lo[t] = tf32_rna(v - h);
    }
}

// G0 = level-0 terms summed in fp32 before each fp64 accumulation (1: every term
// converted, the F32-B policy; 2: pairs -- half the fp32->fp64 conversions).
template <int J, bool LAST64, int G0>
__global__ void __launch_bounds__(kThreads, 2) k_update_tc(const UpdateParams<float> p) {
    using SH = Shape<J>;
    constexpr int KP = SH::KP, NP = SH::NP, NQ = SH::NQ, KQ = SH::KQ, ST = SH::STAGES;
    constexpr int NB = J * (J + 1) / 2;
    constexpr int GB = gblk(J, 4);
    using TD = typename std::conditional<LAST64, double, float>::type;
    extern __shared__ __align__(1024) unsigned char sm[];
    float* sBhi = reinterpret_cast<float*>(sm + SH::OFF_BHI);
    float* sBlo = reinterpret_cast<float*>(sm + SH::OFF_BLO);
    uint4* ring = reinterpret_cast<uint4*>(sm + SH::OFF_RING);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + SH::OFF_BAR);
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + SH::OFF_MISC);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

    // ---- B = core (hi/lo tf32 split), K-major: Bt[(k0, j)][k1] = G'[k0][k1][j] ----
    for (int i = t; i < NP * KP; i += kThreads) {
        const int c = i / KP, k1 = i % KP;
        float v = 0.f;
        if (c < J * J && k1 < J) v = p.Gp[(c / J) * GB + k1 * J + (c % J)];
        const float h = tf32_rna(v);
        sBhi[kmaj<KP>(c, k1)] = h;
        sBlo[kmaj<KP>(c, k1)] = tf32_rna(v - h);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&misc[0])),
                     "n"(SH::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // K-padding chunks (k >= 4*NQ) of every A tile are zero once and never rewritten
#pragma unroll
    for (int st = 0; st < ST * 2; ++st)
#pragma unroll
        for (int q = NQ; q < KQ; ++q)
            *reinterpret_cast<float4*>(sm + SH::OFF_A + st * SH::A_BYTES + kmaj<KP>(t, 4 * q) * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar[0])), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar[1])), "r"(1));
        for (int q = 0; q < ST; ++q) misc[2 + q] = 0;  // arrival counters of the A stages
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = misc[0];
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bhi = smem_u32(sBhi), blo = smem_u32(sBlo);
    const uint32_t a_base = smem_u32(sm + SH::OFF_A);
    uint32_t ntile = 0;  // tiles issued so far by this CTA (mbarrier phases, buffer parity)

    // ring chunk (stage, row k, q) of this thread: k = 0 the level-0 row a0, k = 1 the innermost row a1
    auto ring_at = [&](int st, int k, int q) -> uint4* { return ring + ((st * 2 + k) * NQ + q) * kThreads + t; };
    auto issue = [&](int st, int c0, int c1) {
        const char* s0 = reinterpret_cast<const char*>(p.A[0] + (int64_t)c0 * p.lda);
        const char* s1 = reinterpret_cast<const char*>(p.A[1] + (int64_t)c1 * p.lda);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            cp_async16(ring_at(st, 0, q), s0 + 16 * q);
            cp_async16(ring_at(st, 1, q), s1 + 16 * q);
        }
    };
    // A row of stage st from the gathered a1: hi = a rounded to tf32 (nearest, ties away:
    // two integer ops), lo = a - hi (exact; the tensor core truncates it to tf32, an
    // error <= 2^-23 |a|).  Padding k in [J, 4*NQ) is zero in the padded factor rows.
    auto build_a = [&](int st) {
        unsigned char* dh = sm + SH::OFF_A + (st * 2 + 0) * SH::A_BYTES;
        unsigned char* dl = sm + SH::OFF_A + (st * 2 + 1) * SH::A_BYTES;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const uint4 r = *ring_at(st, 1, q);
            const uint32_t w[4] = {r.x, r.y, r.z, r.w};
            uint32_t h[4];
            float l[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                h[u] = (w[u] + 0x1000u) & 0xFFFFE000u;
                l[u] = __uint_as_float(w[u]) - __uint_as_float(h[u]);
            }
            *reinterpret_cast<uint4*>(dh + kmaj<KP>(t, 4 * q) * 4) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(dl + kmaj<KP>(t, 4 * q) * 4) = make_float4(l[0], l[1], l[2], l[3]);
        }
    };
    // 3xTF32 into TMEM buffer `buf` from A stage `st`: lo*hi, hi*lo, hi*hi (small terms first)
    auto issue_mma = [&](int st, int buf) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ahi = a_base + (st * 2 + 0) * SH::A_BYTES, alo = a_base + (st * 2 + 1) * SH::A_BYTES;
        const uint32_t d = tmem + buf * NP;
        const uint32_t as[3] = {alo, ahi, ahi}, bs[3] = {bhi, blo, bhi};
        uint32_t acc = 0;
#pragma unroll
        for (int pr = 0; pr < 3; ++pr)
#pragma unroll
            for (int ks = 0; ks < SH::KSTEPS; ++ks) {
                // LBO: next 16-byte K chunk = next core matrix (128 B); SBO: next 8 rows
                mma_tf32(d, umma_desc(as[pr] + ks * 256, 128, KP * 32), umma_desc(bs[pr] + ks * 256, 128, KP * 32),
                         idesc, acc);
                acc = 1;
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&mbar[buf])) : "memory");
    };
    // This thread's A row of stage st has landed: make it visible to the tensor
    // core's async proxy and count the arrival; the LAST of the 128 threads issues
    // the MMAs, so no thread blocks on the others here (acq_rel atomic: the issuer
    // observes every row and every completed tcgen05.ld of the TMEM buffer).
    auto arrive_a = [&](int st, int buf) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        uint32_t old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&misc[2 + st])) : "memory");
        if (old == kThreads - 1) {
            misc[2 + st] = 0;
            issue_mma(st, buf);
        }
    };

    for (;;) {
        __syncthreads();
        if (t == 0) misc[1] = atomicAdd(p.work, 1u);
        __syncthreads();
        const int64_t s0 = (int64_t)misc[1] * 4;
        if (s0 >= p.nslices) break;
        const int64_t s = s0 + warp;
        const bool vs = s < p.nslices;
        const int64_t slot = s * kWarp + lane;
        const int row = vs ? p.lane_row[slot] : -1;
        const int len = vs ? p.lane_len[slot] : 0;
        const int iters = p.slice_len[s0];
        const int mylen = vs ? p.slice_len[s] : 0;
        const int64_t base = vs ? p.slice_off[s] + lane : 0;

        double B[NB], c[J], s2 = 0.0;
#pragma unroll
        for (int q = 0; q < NB; ++q) B[q] = 0.0;
#pragma unroll
        for (int q = 0; q < J; ++q) c[q] = 0.0;

        if (iters > 0) {
            // coordinates/values run 3 entries ahead of use (register queue q0 -> q1 -> q2),
            // rows 2 ahead (cp.async ring of 3 stages, stage = entry % 3)
            int ca0 = 0, cb0 = 0, ca1 = 0, cb1 = 0, ca2 = 0, cb2 = 0;
            float x0 = 0.f, x1 = 0.f, x2 = 0.f;
            auto load_crd = [&](int e, int& a, int& b, float& x) {
                const bool v = e < mylen;
                const int64_t idx = base + (int64_t)e * kWarp;
                a = v ? __ldg(p.sc[0] + idx) : 0;
                b = v ? __ldg(p.sc[1] + idx) : 0;
                x = v ? __ldg(p.sv + idx) : 0.f;
            };
            load_crd(0, ca0, cb0, x0);
            load_crd(1, ca1, cb1, x1);
            load_crd(2, ca2, cb2, x2);
            const int st0 = (int)(ntile % ST);
            issue(st0, ca0, cb0);
            cp_async_commit();
            if (iters > 1) issue((st0 + 1) % ST, ca1, cb1);
            cp_async_commit();
            cp_async_wait<1>();
            build_a(st0);
            arrive_a(st0, ntile & 1);
            for (int e = 0; e < iters; ++e) {
                const uint32_t tile = ntile + e;
                const int rs = (int)(tile % ST), rs1 = (int)((tile + 1) % ST), rs2 = (int)((tile + 2) % ST);
                if (e + 2 < iters) issue(rs2, ca2, cb2);
                cp_async_commit();
                const float x = x0;
                // advance the coordinate queue: entry e+1 -> q0, e+2 -> q1, load e+3 -> q2
                ca0 = ca1; cb0 = cb1; x0 = x1;
                ca1 = ca2; cb1 = cb2; x1 = x2;
                load_crd(e + 3, ca2, cb2, x2);
                if (e + 1 < iters) {
                    cp_async_wait<1>();
                    build_a(rs1);
                    arrive_a(rs1, (tile + 1) & 1);
                }
                // ---- epilogue of entry e ----
                float a0f[J];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(ring_at(rs, 0, q));
                    const float w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * q + u < J) a0f[4 * q + u] = w[u];
                }
                mbar_wait(smem_u32(&mbar[tile & 1]), (tile >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                TD d[J];
#pragma unroll
                for (int j = 0; j < J; ++j) d[j] = TD(0);
                const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (tile & 1) * NP;
                // level 0: d[j] = sum_k0 a0[k0] t[k0][j]; t[k0][j] is TMEM column k0*J + j
                if constexpr (G0 == 2 && LAST64 && J == 10) {
                    // pairs (k0, k0+1) = columns [20p, 20p+20): summed in fp32, one fp64 accumulation
#pragma unroll
                    for (int pp = 0; pp < J / 2; ++pp) {
                        float v[16], w[4];
                        tmem_ld16_nowait(taddr + pp * 20, v);
                        tmem_ld4_nowait(taddr + pp * 20 + 16, w);
                        tmem_wait_ld();
                        float t1[J];
#pragma unroll
                        for (int j = 0; j < J; ++j) t1[j] = (J + j < 16) ? v[J + j] : w[J + j - 16];
#pragma unroll
                        for (int j = 0; j < J; ++j)
                            d[j] = d[j] + TD(fmaf(a0f[2 * pp + 1], t1[j], a0f[2 * pp] * v[j]));
                    }
                } else {
                constexpr int NCH = (J * J + 31) / 32;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    float v[32];
                    if (ch * 32 + 16 >= J * J) {
                        float v16[16];
                        tmem_ld16(taddr + ch * 32, v16);
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = v16[i];
                    } else {
                        tmem_ld32(taddr + ch * 32, v);
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int cc = ch * 32 + i;
                        if (cc >= J * J) continue;
                        const int k0 = cc / J, j = cc % J;
                        if constexpr (!LAST64) d[j] = fmaf(a0f[k0], v[i], d[j]);
                        else d[j] = fma(TD(a0f[k0]), TD(v[i]), d[j]);
                    }
                }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                const bool act = e < len;
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
            }
            cp_async_wait<0>();
            ntile += iters;
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
            float* out = p.An + (int64_t)row * p.lda;
            double sse = s2, ac = 0.0, aa = 0.0, ec = 0.0;
            float stv[SH::LD];
#pragma unroll
            for (int j = 0; j < SH::LD; ++j) stv[j] = 0.f;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                stv[j] = float(a[j]);
                const double at = double(stv[j]);
                sse = fma(-2.0 * at, c[j], sse);
                ac = fma(a[j], c[j], ac);
                aa = fma(a[j], a[j], aa);
                ec = fma(at - a[j], c[j] - p.lambda * a[j], ec);
            }
            sse += ac - p.lambda * aa + 2.0 * ec;  // SSE of the stored row (see update.cuh)
#pragma unroll
            for (int q = 0; q < SH::NQ; ++q)
                reinterpret_cast<float4*>(out)[q] = make_float4(stv[4 * q], stv[4 * q + 1], stv[4 * q + 2], stv[4 * q + 3]);
            p.sse_row[row] = sse;
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
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(SH::TCOLS));
}

template <int J, bool LAST64>
void launch_tc(const void* params, bool literal, int grid, cudaStream_t st) {
    (void)literal;
    const UpdateParams<float>& p = *reinterpret_cast<const UpdateParams<float>*>(params);
    if (p.l0_group == 2 && LAST64) {
        auto k = k_update_tc<J, LAST64, 2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Shape<J>::SMEM);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        k<<<grid, kThreads, Shape<J>::SMEM, st>>>(p);
    } else {
        auto k = k_update_tc<J, LAST64, 1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Shape<J>::SMEM);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        k<<<grid, kThreads, Shape<J>::SMEM, st>>>(p);
    }
}

template <int J, bool LAST64>
int occupancy_tc(bool literal, size_t gp_bytes) {
    (void)literal;
    (void)gp_bytes;
    auto k = k_update_tc<J, LAST64, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Shape<J>::SMEM);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    // Resident CTAs per SM from the kernel's own resource use (the occupancy API
    // under-reports this kernel on sm_100a): registers, shared memory, TMEM.
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    int dev = 0, smem_sm = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs = (fa.numRegs + 7) / 8 * 8;
    const int by_regs = regs_sm / (regs * kThreads);
    const int by_smem = smem_sm / (Shape<J>::SMEM + 1024);
    int nb = by_regs < by_smem ? by_regs : by_smem;
    const int tm = 512 / Shape<J>::TCOLS;  // TMEM: every resident CTA allocates TCOLS of the 512 columns
    if (getenv("PTUCKER_DEBUG"))
        fprintf(stderr, "[ptucker] tc occupancy J=%d smem=%d regs=%d: by_regs=%d by_smem=%d tmem=%d\n", J,
                Shape<J>::SMEM, fa.numRegs, by_regs, by_smem, tm);
    return nb < tm ? nb : tm;
}

}  // namespace tc

#define PT_TC_J_LIST(X) X(2) X(3) X(4) X(5) X(8) X(10)

namespace {
#define PT_TC_ENTRY(J) {0, 0, 3, J, &tc::launch_tc<J, false>, &tc::occupancy_tc<J, false>}, \
                       {0, 1, 3, J, &tc::launch_tc<J, true>, &tc::occupancy_tc<J, true>},
const UpdateKernel kTcTable[] = {PT_TC_J_LIST(PT_TC_ENTRY)};
#undef PT_TC_ENTRY
}  // namespace

// Host: tf32 hi/lo split of the innermost factor (rows of KP floats) for the A operand.
int tc_kp(int J) {
    switch (J) {
        case 2: return tc::Shape<2>::KP;
        case 3: return tc::Shape<3>::KP;
        case 4: return tc::Shape<4>::KP;
        case 5: return tc::Shape<5>::KP;
        case 8: return tc::Shape<8>::KP;
        case 10: return tc::Shape<10>::KP;
    }
    return 0;
}

void launch_tc_split(const float* A, int64_t I, int lda, int J, float* hi, float* lo, cudaStream_t st) {
    const int KP = tc_kp(J);
    const int64_t total = I * KP;
    int grid = (int)((total + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    tc::k_split_tf32<<<grid, 256, 0, st>>>(A, I, lda, J, KP, hi, lo);
}

const UpdateKernel* find_update_kernel_tc(int l64, int J) {
    const int want = l64 > 0 ? 1 : 0;
    for (const auto& k : kTcTable)
        if (k.J == J && k.l64 == want) return &k;
    return nullptr;
}

}  // namespace pt
