// update_tc.cu -- row update for order-3 fp32 tensors with the innermost TTV
// stage on the 5th-generation tensor cores (tcgen05, kind::tf32, TMEM
// accumulators), warp-specialised.
//
// For mode n with other modes m0 < m1, Eq. 12 regrouped as a TTV
// chain is   delta(j) = sum_k0 a0[k0] * t[k0][j],   t[k0][j] = sum_k1 a1[k1] G'[k0][k1][j].
// The inner stage, over the 128 entries a CTA holds at a time ("tile"), is a
// dense GEMM
//     T (128 x J^2) = A1 (128 x J) * Bt^T,   Bt[(k0,j)][k1] = G'[k0][k1][j],
// with B = the core, shared by every entry.  It runs as 3xTF32 (a = a_hi + a_lo,
// small products first: lo*hi, hi*lo, hi*hi) so its accuracy matches an fp32
// FMA chain (tools/tc_probe.cu), accumulating in TMEM.
//
// CTA = 4 warps, two CTAs per SM (255 registers per thread; TMEM columns
// [0, TCOLS) of each CTA hold two accumulator buffers).  Thread t owns TMEM lane
// t and row segment t of the current group of 4 SELL-32 slices,
// and streams its own entries through two per-thread cp.async rings in shared
// memory: the coordinates/value kCPref tiles ahead, the two gathered factor
// rows kRPref tiles ahead (no cross-thread handshake: each thread reads only
// what it fetched).  Per tile k a thread
//   (a) splits its gathered a1 row of tile k+1 into tf32 hi/lo rows of the A
//       operand; the last of the 4 warps to do so issues that tile's MMAs
//       (double-buffered A stages and TMEM accumulators), so the MMA of tile
//       k+1 runs while
//   (b) the epilogue of tile k reads t[k0][j] from TMEM, finishes level 0 in
//       fp64 (F32-B), accumulates B += delta delta^T, c += x delta, sum x^2
//       (fp64, Eq. 10-11), and at the end of the segment solves
//       a = c [B + lambda I]^-1 (Cholesky, Eq. 9) and stores the row with its
//       SSE (fused Eq. 5).
// Groups are assigned statically (serpentine over the CTAs; SELL groups are
// sorted by length, so neighbouring CTAs get near-equal work), so every thread
// knows its whole tile sequence and the rings run ahead across group
// boundaries.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "update.cuh"

namespace pt {
namespace tc {

constexpr int kThreads = 128;  // = TMEM lanes = segments per group (4 SELL slices)
constexpr int kCPref = 7;      // coordinates fetched this many tiles ahead of their epilogue
constexpr int kCRing = 8;      // coordinate ring slots (> kCPref)
constexpr int kRPref = 3;      // factor rows gathered this many tiles ahead
constexpr int kRRing = 4;      // row ring slots (> kRPref)
static_assert(kCRing > kCPref && kRRing > kRPref && kCPref > 2 * kRPref - 1, "ring depths");

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

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(bar) : "memory");
}
// arrive once every cp.async this thread issued so far has landed (count pre-set in init)
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
// L2 cache policies: the SELL entry stream is read once per mode (evict first);
// the gathered factor rows are re-read ~|Omega|/I times per mode (evict last)
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async4_hint(void* smem, const void* gmem, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "l"(pol)
                 : "memory");
}

// 16 TMEM columns of this warp's 32 lanes (32x32b shape: thread i <- lane i).
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
// wait for this thread's outstanding tcgen05.ld; the registers are tied to the
// wait so that no use of them can be scheduled before it
__device__ __forceinline__ void tmem_wait16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
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
    static constexpr int NCH = (J * J + 15) / 16;           // 16-column TMEM chunks holding t
    // shared memory map (bytes)
    static constexpr int B_BYTES = NP * KP * 4;             // one of B_hi / B_lo
    static constexpr int A_BYTES = kThreads * KP * 4;       // one of A_hi / A_lo (per stage)
    static constexpr int CSLOT = 3 * kThreads * 4;          // coordinate ring slot: c0[128], c1[128], x[128]
    static constexpr int RSLOT = 2 * NQ * kThreads * 16;    // row ring slot: a0, a1 rows, chunk-major
    static constexpr int OFF_BHI = 0;
    static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
    static constexpr int OFF_A = OFF_BLO + B_BYTES;         // [stage 0,1][hi,lo]
    static constexpr int OFF_CRD = OFF_A + 2 * 2 * A_BYTES;
    static constexpr int OFF_ROW = OFF_CRD + kCRing * CSLOT;
    static constexpr int OFF_BAR = OFF_ROW + kRRing * RSLOT;  // acc_full[2]
    static constexpr int OFF_MISC = OFF_BAR + 2 * 8;          // tmem base, A-stage arrival counters[2], tiles
    static constexpr int SMEM = OFF_MISC + 16;
};

// Split of the innermost factor into tf32 hi/lo parts (3xTF32 operand), K-padded
// (diagnostic helper kept for tools/; the update kernel splits in place).
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

// Static serpentine assignment of groups (4 slices each) to CTAs.
struct Sched {
    int64_t ngroups, r;
    int G, b;
    __device__ int64_t group() const { return r * G + ((r & 1) ? (G - 1 - b) : b); }
    __device__ bool valid() const { return group() < ngroups; }
};

// Segment data of the current group for one thread.
struct Seg {
    int iters;     // tiles of the group (longest slice = its first)
    int row, len;  // segment row (-1: pad lane) and length
    int64_t slot;  // SELL lane slot (partials)
};

// This thread's slice of a group, for the coordinate cursor.
struct SliceMeta {
    int iters, slen;
    int64_t off;
    bool valid;
};

// G0 (level-0 grouping, LAST64 only): 1 = every a0[k0] t[k0][j] product and the sum
// in fp64 (F32-B); g > 1 = partial sums over runs of g consecutive k0 in fp32
// (one rounded product, then FMAs), each partial converted to fp64 once and the
// partials summed in fp64: ceil(J/g) instead of J^2 fp32->fp64 conversions per
// entry (F2F runs on the quarter-rate XU pipe; tools/level0_emulation.py measures
// the row error of each g).
template <int J, bool LAST64, int G0>
__global__ void __launch_bounds__(kThreads, 2) k_update_tc(const UpdateParams<float> p) {
    using SH = Shape<J>;
    constexpr int KP = SH::KP, NP = SH::NP, NQ = SH::NQ, KQ = SH::KQ;
    constexpr int NB = J * (J + 1) / 2;
    constexpr int GB = gblk(J, 4);
    using TD = typename std::conditional<LAST64, double, float>::type;
    extern __shared__ __align__(1024) unsigned char sm[];
    float* sBhi = reinterpret_cast<float*>(sm + SH::OFF_BHI);
    float* sBlo = reinterpret_cast<float*>(sm + SH::OFF_BLO);
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + SH::OFF_MISC);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t bar0 = smem_u32(sm + SH::OFF_BAR);
    auto acc_bar = [&](int b) { return bar0 + 8u * b; };
    // coordinate ring slot s: c0, c1, x of this thread's entry
    auto crd = [&](int s, int a) -> uint32_t* {
        return reinterpret_cast<uint32_t*>(sm + SH::OFF_CRD + s * SH::CSLOT) + a * kThreads + t;
    };
    // row ring slot s: chunk q of row k (0: a0, 1: a1) of this thread's entry
    auto rowc = [&](int s, int k, int q) -> uint4* {
        return reinterpret_cast<uint4*>(sm + SH::OFF_ROW + s * SH::RSLOT) + ((k * NQ + q) * kThreads + t);
    };

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
    for (int st = 0; st < 4; ++st)
#pragma unroll
        for (int q = NQ; q < KQ; ++q)
            *reinterpret_cast<float4*>(sm + SH::OFF_A + st * SH::A_BYTES + kmaj<KP>(t, 4 * q) * 4) =
                make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t ngroups = (p.nslices + 3) / 4;
    const Sched s0{ngroups, 0, (int)gridDim.x, (int)blockIdx.x};
    if (warp == 1) {
        // tiles of this CTA = sum of the iteration counts of its groups
        uint32_t n = 0;
        for (int64_t r = lane;; r += kWarp) {
            Sched q = s0;
            q.r = r;
            if (!q.valid()) break;
            n += (uint32_t)__ldg(p.slice_len + q.group() * 4);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        if (lane == 0) misc[3] = n;
    }
    if (t == 0) {
        mbar_init(acc_bar(0), 1);
        mbar_init(acc_bar(1), 1);
        misc[1] = misc[2] = 0;  // arrival counters of the two A stages
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = misc[0];
    const uint32_t total = misc[3];

    // ------------------------------------------------------------------
    // Coordinate cursor: walks this thread's entries kCPref tiles ahead of
    // the epilogue and cp.asyncs c0, c1, x into the coordinate ring.
    // ------------------------------------------------------------------
    auto load_meta = [&](const Sched& q, SliceMeta& m) {
        m.valid = q.valid();
        if (!m.valid) return;
        const int64_t g0 = q.group() * 4, sl = g0 + warp;
        const bool v = sl < p.nslices;
        m.iters = __ldg(p.slice_len + g0);
        m.slen = v ? __ldg(p.slice_len + sl) : 0;
        m.off = v ? __ldg(p.slice_off + sl) + lane : 0;
    };
    Sched cs = s0;
    SliceMeta cm, cn;  // cursor group, next group
    load_meta(cs, cm);
    {
        Sched q = cs;
        ++q.r;
        load_meta(q, cn);
    }
    int ce = 0;
    bool cend = !cm.valid || cm.iters == 0;
    const uint64_t pol_stream = policy_evict_first(), pol_rows = policy_evict_last();
    uint32_t ck = 0;  // tile index of the cursor
    auto issue_crd = [&]() {
        if (cend) return;
        const int s = (int)(ck % kCRing);
        const bool v = ce < cm.slen;
        const int64_t idx = cm.off + (int64_t)ce * kWarp;
        if (v) {
            cp_async4_hint(crd(s, 0), p.sc[0] + idx, pol_stream);
            cp_async4_hint(crd(s, 1), p.sc[1] + idx, pol_stream);
            cp_async4_hint(crd(s, 2), p.sv + idx, pol_stream);
        } else {
            *crd(s, 0) = 0u;  // padding entry: gather row 0 (its result is masked)
            *crd(s, 1) = 0u;
        }
        ++ck;
        if (++ce == cm.iters) {
            ce = 0;
            if (!cn.valid || cn.iters == 0) {
                cend = true;  // groups are sorted by length: nothing follows an empty group
            } else {
                cm = cn;
                ++cs.r;
                Sched q = cs;
                ++q.r;
                load_meta(q, cn);
            }
        }
    };
    // rows of tile k (its coordinates have landed): cp.async a0, a1 into row slot k % kRRing
    auto issue_rows = [&](uint32_t k) {
        const int s = (int)(k % kRRing), cslot = (int)(k % kCRing);
        const int c0 = (int)*crd(cslot, 0), c1 = (int)*crd(cslot, 1);
        const char* r0 = reinterpret_cast<const char*>(p.A[0] + (int64_t)c0 * p.lda);
        const char* r1 = reinterpret_cast<const char*>(p.A[1] + (int64_t)c1 * p.lda);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            cp_async16_hint(rowc(s, 0, q), r0 + 16 * q, pol_rows);
            cp_async16_hint(rowc(s, 1, q), r1 + 16 * q, pol_rows);
        }
    };
    // Step s (s = -kCPref .. total-1): coordinates of tile s+kCPref, rows of tile
    // s+kRPref, one cp.async group per step (groups are numbered by step).
    auto step = [&](int s) {
        issue_crd();
        const int kr = s + kRPref;
        // coordinates of tile kr were committed at step kr - kCPref
        cp_async_wait<kCPref - kRPref - 1>();
        if (kr >= 0 && kr < (int)total) issue_rows((uint32_t)kr);
        cp_async_commit();
    };

    const uint32_t idesc =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t bhi = smem_u32(sBhi), blo = smem_u32(sBlo);
    const uint32_t a_base = smem_u32(sm + SH::OFF_A);
    const uint32_t tm_lane = tmem + ((uint32_t)(warp * 32) << 16);

    // 3xTF32 into TMEM buffer `buf` from A stage `buf`: lo*hi, hi*lo, hi*hi (small terms first)
    auto issue_mma = [&](int buf) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ahi = a_base + (buf * 2 + 0) * SH::A_BYTES, alo = a_base + (buf * 2 + 1) * SH::A_BYTES;
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
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(acc_bar(buf))
                     : "memory");
    };
    // Tile k (its rows have landed): write this thread's A row of stage k&1
    // (hi = a rounded to tf32 by two integer ops, lo = a - hi exact; the tensor
    // core truncates lo to tf32, an error <= 2^-23 |a|), make it visible to the
    // async proxy and count the arrival (one per warp); the lane 0 of the LAST
    // warp issues the MMAs (acq_rel atomic: it observes every row and every
    // completed tcgen05.ld of the TMEM buffer it overwrites).
    auto prepare = [&](uint32_t k, auto&& after_split) {
        const int s = (int)(k % kRRing), st = (int)(k & 1);
        unsigned char* dh = sm + SH::OFF_A + (st * 2 + 0) * SH::A_BYTES;
        unsigned char* dl = sm + SH::OFF_A + (st * 2 + 1) * SH::A_BYTES;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const uint4 r = *rowc(s, 1, q);
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
        after_split();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        // one arrival per warp (its lanes are ordered before lane 0 by the warp barrier)
        if (lane == 0) {
            uint32_t old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old)
                         : "r"(smem_u32(&misc[1 + st]))
                         : "memory");
            if (old == kThreads / kWarp - 1) {
                misc[1 + st] = 0;
                issue_mma(st);
            }
        }
    };
    auto load_seg = [&](const Sched& s, Seg& g) {
        const int64_t g0 = s.group() * 4;
        const int64_t sl = g0 + warp;
        g.slot = sl * kWarp + lane;
        const bool v = sl < p.nslices;
        g.iters = __ldg(p.slice_len + g0);
        g.row = v ? __ldg(p.lane_row + g.slot) : -1;
        g.len = v ? __ldg(p.lane_len + g.slot) : 0;
    };
    double B[NB], c[J], s2;
    auto zero = [&]() {
#pragma unroll
        for (int q = 0; q < NB; ++q) B[q] = 0.0;
#pragma unroll
        for (int q = 0; q < J; ++q) c[q] = 0.0;
        s2 = 0.0;
    };
    // end of a segment: solve and store (Eq. 9 + fused Eq. 5), or write the heavy-row partial
    auto finalize = [&](const Seg& g) {
        if (g.row < 0) return;
        const int64_t pidx = p.lane_pidx[g.slot];
        if (pidx < 0) {
            double a[J];
            const bool ok = chol_solve<J>(B, c, p.lambda, a);
            if (!ok) {
                atomicCAS(p.fail, 0, g.row + 1);
#pragma unroll
                for (int j = 0; j < J; ++j) a[j] = 0.0;
            }
            float* out = p.An + (int64_t)g.row * p.lda;
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
            p.sse_row[g.row] = sse;
        } else {
            const int stp = p.lane_pstride[g.slot];
            double* dst = p.partials + pidx;
#pragma unroll
            for (int q = 0; q < NB; ++q) dst[(int64_t)q * stp] = B[q];
#pragma unroll
            for (int q = 0; q < J; ++q) dst[(int64_t)(NB + q) * stp] = c[q];
            dst[(int64_t)(NB + J) * stp] = s2;
        }
    };

    Sched sc = s0;
    if (sc.valid()) {
        Seg cur, nxt;
        load_seg(sc, cur);
        Sched sn = sc;
        ++sn.r;
        const bool tiles = total > 0;
        zero();
        if (tiles) {
            bool nvalid = sn.valid();
            if (nvalid) load_seg(sn, nxt);
            for (int s = -kCPref; s < 0; ++s) step(s);
            cp_async_wait<kRPref - 1>();  // rows of tile 0 (committed at step -kRPref)
            prepare(0, []() {});
            int e = 0;
            // optional per-phase clock trace (tools/trace_tc.py): CTA 0, lane 0 of each warp, tiles [64, 128)
            long long* const trb = (p.trace && blockIdx.x == 0 && lane == 0) ? p.trace + warp * 512 : nullptr;
            auto mark = [&](uint32_t k, int ph) {
                if (trb && k >= 64 && k < 128) trb[(k - 64) * 8 + ph] = clock64();
            };
            for (uint32_t k = 0; k < total; ++k) {
                mark(k, 0);
                step((int)k);
                mark(k, 1);
                if (k + 1 < total) {
                    cp_async_wait<kRPref - 1>();  // rows of tile k+1 (committed at step k+1-kRPref)
                    mark(k, 2);
                    prepare(k + 1, [&]() { mark(k, 3); });
                }
                mark(k, 4);
                // ---- epilogue of tile k ----
                const int s = (int)(k % kRRing), buf = (int)(k & 1);
                // an inactive lane (entry beyond its segment) gets a0 = 0, hence delta = 0
                // (the gathered rows are always real factor rows, never stale data)
                const bool act = e < cur.len;
                float a0f[J];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(rowc(s, 0, q));
                    const float w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * q + u < J) a0f[4 * q + u] = act ? w[u] : 0.f;
                }
                const float x = __uint_as_float(*crd((int)(k % kCRing), 2));
                mbar_wait(acc_bar(buf), (k >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                mark(k, 5);
                // level 0: d[j] = sum_k0 a0[k0] t[k0][j]; t[k0][j] is TMEM column k0*J + j
                TD d[J];
                float pf[J];  // fp32 partial sums (G0 > 1)
#pragma unroll
                for (int j = 0; j < J; ++j) d[j] = TD(0);
                const uint32_t taddr = tm_lane + buf * NP;
                uint32_t rb[2][16];
                tmem_ld16(taddr, rb[0]);
#pragma unroll
                for (int ch = 0; ch < SH::NCH; ++ch) {
                    tmem_wait16(rb[ch & 1]);
                    if (ch + 1 < SH::NCH) tmem_ld16(taddr + (ch + 1) * 16, rb[(ch + 1) & 1]);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int cc = ch * 16 + i;
                        if (cc >= J * J) continue;
                        const int k0 = cc / J, j = cc % J;
                        const float tv = __uint_as_float(rb[ch & 1][i]);
                        if constexpr (!LAST64) {
                            d[j] = fmaf(a0f[k0], tv, d[j]);
                        } else if constexpr (G0 == 1) {
                            d[j] = fma(TD(a0f[k0]), TD(tv), d[j]);
                        } else {
                            if (k0 % G0 == 0) pf[j] = a0f[k0] * tv;
                            else pf[j] = fmaf(a0f[k0], tv, pf[j]);
                            if (k0 % G0 == G0 - 1 || k0 == J - 1) d[j] = d[j] + TD(pf[j]);
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mark(k, 6);
                double dd[J];
#pragma unroll
                for (int j = 0; j < J; ++j) dd[j] = double(d[j]);
                const double xd = act ? double(x) : 0.0;
#pragma unroll
                for (int i = 0; i < J; ++i) {
                    c[i] = fma(xd, dd[i], c[i]);
#pragma unroll
                    for (int j = i; j < J; ++j) B[up_idx(i, j, J)] = fma(dd[i], dd[j], B[up_idx(i, j, J)]);
                }
                s2 = fma(xd, xd, s2);
                mark(k, 7);
                if (++e == cur.iters) {
                    finalize(cur);
                    zero();
                    e = 0;
                    sc = sn;
                    ++sn.r;
                    if (nvalid) {
                        cur = nxt;
                        nvalid = sn.valid();
                        if (nvalid) load_seg(sn, nxt);
                    }
                }
            }
            cp_async_wait<0>();
        }
        // the groups after the last one with entries are empty (sorted by length):
        // their rows get a = 0 and SSE 0
        for (; sc.valid(); ++sc.r) {
            load_seg(sc, cur);
            zero();
            finalize(cur);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(SH::TCOLS));
}

template <int J, bool LAST64, int G0>
void launch_tc_g(const UpdateParams<float>& p, int grid, cudaStream_t st) {
    auto k = k_update_tc<J, LAST64, G0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Shape<J>::SMEM);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    k<<<grid, kThreads, Shape<J>::SMEM, st>>>(p);
}

template <int J, bool LAST64>
void launch_tc(const void* params, bool literal, int grid, cudaStream_t st) {
    (void)literal;
    const UpdateParams<float>& p = *reinterpret_cast<const UpdateParams<float>*>(params);
    if constexpr (!LAST64) {
        launch_tc_g<J, false, 1>(p, grid, st);
    } else {
        if (p.l0_group == 1) launch_tc_g<J, true, 1>(p, grid, st);
        else if (p.l0_group == 2) launch_tc_g<J, true, 2>(p, grid, st);
        else launch_tc_g<J, true, 5>(p, grid, st);
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
