// update_tc.cu -- row update for order-3 fp32 tensors with the innermost TTV
// stage on the 5th-generation tensor cores (tcgen05, kind::tf32, TMEM
// accumulators), warp-specialised.
//
// For mode n with other modes m0 < m1, Eq. 12 regrouped as a TTV
// chain is   delta(j) = sum_k0 a0[k0] * t[k0][j],   t[k0][j] = sum_k1 a1[k1] G'[k0][k1][j].
// The inner stage, over 128 entries at a time ("tile"), is a dense GEMM
//     T (128 x J^2) = A1 (128 x J) * Bt^T,   Bt[(k0,j)][k1] = G'[k0][k1][j],
// with B = the core, shared by every entry.  It runs as 3xTF32 (a = a_hi + a_lo,
// small products first: lo*hi, hi*lo, hi*hi) so its accuracy matches an fp32
// FMA chain (tools/tc_probe.cu), accumulating in TMEM.
//
// One CTA per SM, 16 warps.  Warps w, w+4 (level 0) and w+8 (normal equations)
// serve TMEM lane quarter w: thread t owns TMEM lane 32w+t = row segment 32w+t
// of the current group of 4 SELL-32 slices.
//   warps 0-7   LEVEL 0 (kRegL0 registers via setmaxnreg; warps w and w+4 take
//               alternate tiles).  At tile k a warp first writes the A rows of its
//               tile k + kNA into TMEM (tf32 hi/lo split of the gathered a1 row)
//               and copies that tile's a0 row and x into its own stash, releasing
//               the row-ring slot early; then for tile k it loads the J^2 columns
//               t[k0][j] from TMEM (kBCH chunks per wait), finishes level 0 (fp64
//               per term, or fp32 partial sums of G0 terms added in fp64) and hands
//               delta (fp64) and x to warp w+8 through a shared-memory ring.
//   warps 8-11  NORMAL EQUATIONS (kRegNE registers): B += delta delta^T, c += x delta,
//               sum x^2 in fp64 registers (Eq. 10-11), and at the end of the
//               segment a = c [B + lambda I]^-1 (Cholesky, Eq. 9) and the row's SSE
//               (fused Eq. 5).
//   warps 14, 12, 13  LOADERS (tiles k = 0, 1, 2 mod kLoaders): stream the SELL
//               coordinates/values into a coordinate ring (cp.async, kCPref own
//               tiles ahead) and gather the two factor rows of every entry into a
//               kRing-slot row ring (cp.async).  The gathers are bound by the
//               L1TEX request rate of 16-byte lanes at distinct rows; three warps
//               on three sub-partitions keep it fed.
//   warp 15     MMA: lane 0 issues a tile's MMAs into one of kNT TMEM accumulators.
// Splitting level 0 from the normal equations keeps each role's registers small
// enough for two level-0 warps per SM sub-partition (the XU conversions of one
// overlap the waits of the other) and lets the XU and fp64 pipes work on
// different tiles concurrently.
// Groups are assigned statically (serpentine over the CTAs; SELL groups are
// sorted by length, so neighbouring CTAs get near-equal work), so every role
// knows the CTA's whole tile sequence in advance.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "update.cuh"

namespace pt {
namespace tc {

constexpr int kE = 128;                      // TMEM lanes = segments per group (4 slices)
constexpr int kThreads = 16 * 32;            // 2 level-0 WGs, normal-equation WG, loader/MMA WG
// PT_NOSTASH: the level-0 warps read a0, x and the scale exponent straight from the row-ring
// slot when they reduce the tile (the slot is released then, not at the split), instead of a
// copy into a per-warp stash at the split: 18 KB less shared-memory traffic per tile; the ring
// holds kNA more tiles
#ifndef PT_NOSTASH
#define PT_NOSTASH 1
#endif
#ifndef PT_RING
#define PT_RING (PT_NOSTASH ? 10 : 6)
#endif
constexpr int kRing = PT_RING;                     // row ring slots (tiles between loader and level 0)
constexpr bool kNoStash = PT_NOSTASH != 0;
constexpr int kCPref = 7;                    // loader: coordinates fetched this many tiles ahead of the gathers
#ifndef PT_LOADERS
#define PT_LOADERS 3
#endif
constexpr int kLoaders = PT_LOADERS;         // loader warps (14, 12, 13): tiles k = lp (mod kLoaders)
static_assert(kLoaders >= 1 && kLoaders <= 3, "loader warps");
constexpr int kCRing = 8 * kLoaders;                    // coordinate ring slots (> kCPref)
#ifndef PT_NT
#define PT_NT 3
#endif
#ifndef PT_NA
#define PT_NA 4
#endif
constexpr int kNT = PT_NT;                   // TMEM accumulator buffers
constexpr int kNA = PT_NA;                   // TMEM A buffers (the level-0 warps write A kNA tiles ahead)
constexpr int kStash = kNA / 2 + 1;          // a0/x stash slots per level-0 warp (its tiles k, k+2, .., k+kNA)
#ifndef PT_KD
#define PT_KD 4
#endif
constexpr int kD = PT_KD;                        // delta ring slots (level 0 -> normal equations)
// delta handoff through hardware named barriers (bar.arrive by the level-0 warp, bar.sync by
// the normal-equation warp; ids 1 + 4 kD): the waiting warp blocks in hardware instead of
// polling its mbarrier -- those polls were ~40% of the kernel's issued instructions
// (profiles/r02/tc_f16_c5_full.txt: the d_full retry loop and the row-ring wait)
#ifndef PT_NBAR
#define PT_NBAR 0
#endif
constexpr bool kNbar = PT_NBAR != 0;
#ifndef PT_SPLIT_LATE
#define PT_SPLIT_LATE 0
#endif
constexpr bool kSplitLate = PT_SPLIT_LATE != 0;  // level-0 warps split tile k + kNA after (not before) tile k
static_assert(!kNbar || 1 + 4 * kD <= 16, "named barriers: 4 quarters x kD slots + barrier 0");
constexpr int kRegLaunch = 65536 / kThreads / 8 * 8;  // registers per thread at launch (128)
#ifndef PT_REG_L0
#define PT_REG_L0 136
#endif
#ifndef PT_REG_NE
#define PT_REG_NE 192
#endif
#ifndef PT_BCH
#define PT_BCH 4
#endif
constexpr int kRegL0 = PT_REG_L0;            // setmaxnreg: level-0 warpgroups
constexpr int kRegNE = PT_REG_NE;            //             normal-equation warpgroup
#ifndef PT_REG_P
#define PT_REG_P 48
#endif
constexpr int kRegP = PT_REG_P;              //             loader/MMA warpgroup
#ifndef PT_L0_XU_MOD
#define PT_L0_XU_MOD 2
#endif
#ifndef PT_A0_INT
#define PT_A0_INT 0
#endif
constexpr int kXuMod = PT_L0_XU_MOD;         // level 0 (G0 = 1): every kXuMod-th t converted on the XU pipe, the rest by integer ops
// level 0 (G0 = 1), conversion scheme 1: the t[k0][.] of the k0 in kXuMask are converted on
// the XU pipe, the others by three integer operations into t * 2^-896 (f2d_scaled), whose
// a0[k0] is pre-multiplied by 2^896 (exact); scheme 0 = the kXuMod interleave of f2d_int
#ifndef PT_L0_CONV
#define PT_L0_CONV 1
#endif
#ifndef PT_XU_MASK
#define PT_XU_MASK 0x049
#endif
constexpr int kL0Conv = PT_L0_CONV;
#ifndef PT_ACC_EARLY
#define PT_ACC_EARLY 1
#endif
constexpr bool kAccEarly = PT_ACC_EARLY != 0;
// 3xTF32 as ONE K-sweep: A = [a_lo | a_hi | a_hi] and B = [b_hi ; b_lo ; b_hi] along K
// (the small products lo*hi and hi*lo first, then hi*hi)
// (3J columns padded to the K-step), so every MMA K-step carries useful products:
// J = 10 takes 4 MMAs (K = 32) per tile instead of 3 x 2 (K = 16 each, 10 used)
#ifndef PT_KCAT
#define PT_KCAT 1
#endif
constexpr bool kKcat = PT_KCAT != 0;
// The same three products with fp16 operands (kind::f16: K = 16 per MMA at twice the tf32
// rate).  An fp16 value carries the same 11 significant bits as tf32, so a = hi + lo keeps
// 22 bits either way; the narrower exponent range is handled by exact power-of-two
// scalings: every gathered a1 row by 2^sA (its largest |element| to [2^14, 2^15)) and the
// core by 2^sG (the same for max |G|), undone exactly in fp64 by the level-0 weights
// (a0 * 2^-(sA+sG)).  An element far below its row's (or the core's) maximum loses
// relative precision to fp16 subnormals, but its absolute error stays below 2^-38 of that
// maximum, far under the 2^-22 of the split itself.
#ifndef PT_F16
#define PT_F16 1
#endif
constexpr bool kF16 = PT_F16 != 0 && kKcat;
#ifndef PT_DFULL1
#define PT_DFULL1 1
#endif
constexpr bool kDfull1 = PT_DFULL1 != 0;  // delta handoff: one arrival per level-0 warp (else one per lane)
#ifndef PT_LOADER_SLEEP
#define PT_LOADER_SLEEP 0
#endif
#ifndef PT_NE_SLEEP
#define PT_NE_SLEEP 0
#endif
constexpr uint32_t kLoaderSleep = PT_LOADER_SLEEP;  // ns between polls of the loaders' slot waits (0: suspend-hint try_wait)
constexpr uint32_t kNeSleep = PT_NE_SLEEP;          // ns between polls of the normal-equation warps' delta waits  // release the accumulator once its last TMEM chunk is in registers
constexpr unsigned kXuMask = PT_XU_MASK;
constexpr bool kA0Int = PT_A0_INT != 0;      // a0 converted by integer ops too
constexpr int kBCH = PT_BCH;                      // level 0: TMEM chunks per load batch (registers)
static_assert(kCRing > kLoaders * kCPref, "ring depths");
// setmaxnreg moves registers inside the CTA's launch allocation: the increases
// must be covered by the helpers' release, or they wait forever
static_assert(4 * kWarp * (2 * kRegL0 + kRegNE + kRegP) <= kRegLaunch * kThreads, "register pool");

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

// A operand in tensor memory (lane = row, K along columns), B from shared memory
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
// packed fp32 pairs (FFMA2 / FADD2): two level-0 columns per instruction
__device__ __forceinline__ uint64_t fma_f32x2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t add_f32x2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t sub_f32x2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t pack_f32x2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ void mma_f16_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
// two floats -> packed f16x2 (round to nearest), a in the low half (the lower K index)
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}
// power-of-two scale exponent that takes a largest magnitude with float bits mb (sign
// cleared) to [2^14, 2^15); 0 for an all-zero set; clamped to [-60, 120] so 2^s is a normal
// float and the level-0 weight 2^(896 - sA - sG) a normal double
__device__ __forceinline__ int f16_scale_exp(uint32_t mb) {
    if (mb == 0u) return 0;
    const int e = (int)(mb >> 23);  // biased exponent (0: subnormal)
    const int s = 141 - e;
    return s > 120 ? 120 : (s < -60 ? -60 : s);
}
__device__ __forceinline__ float exp2f_int(int s) { return __uint_as_float((uint32_t)(127 + s) << 23); }
__device__ __forceinline__ double exp2d_int(int s) { return __hiloint2double((1023 + s) << 20, 0); }
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// float -> double with integer operations (SHF, LOP3, IADD3 and a shift) instead of
// the XU conversion: exact for normal floats of either sign; a zero or subnormal
// input becomes +-2^-127 * (1 + m) (an absolute error below 1.2e-38, irrelevant
// next to the O(1) terms of the level-0 sums it feeds).  Inputs here are finite
// tensor-core outputs.
__device__ __forceinline__ double f2d_int(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t hi = ((uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu) + 0x38000000u;
    return __hiloint2double((int)hi, (int)(u << 29));
}

// float -> double scaled by 2^-896, in three integer operations (SHF, LOP3, SHL): the
// fp32 exponent field e8 is placed unchanged in the fp64 exponent field, i.e. the fp64
// bias 1023 replaces the fp32 bias 127 without the +896 rebias.  Exact for every finite
// float: normal f -> f * 2^-896 (a normal double, >= 2^-1022), zero -> +-0, and a
// subnormal f = 0.m * 2^-126 -> the subnormal double 0.m * 2^-1022 = f * 2^-896.
__device__ __forceinline__ double f2d_scaled(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t hi = (uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu;
    return __hiloint2double((int)hi, (int)(u << 29));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(0x989680u)  // suspend up to 10 ms (woken by the phase change): waiters do not spin on issue slots
            : "memory");
    }
}
// Wait with a nanosleep back-off between polls: for the roles with slack (loaders far
// ahead of the ring, normal-equation warps behind level 0), so their polling does not take
// issue slots from the level-0 warps of the same sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, uint32_t ns) {
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) break;
        __nanosleep(ns);
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
__device__ __forceinline__ void cp_async8_hint(void* smem, const void* gmem, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "l"(pol)
                 : "memory");
}
// the same through L1 (.ca): a hot factor row (Zipf-skewed modes, p.rows_l1) is served by
// each SM's L1 instead of hammering the one L2 slice that holds it (c3 table modes 2.36 ->
// 1.07 ms); with uniform rows (c5) L1 allocation only thrashes (4.1 -> 7.0 ms)
__device__ __forceinline__ void cp_async16_l1(void* smem, const void* gmem, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
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
    static constexpr int KSTEP = kF16 ? 16 : 8;             // K per MMA (kind::f16 / kind::tf32)
    static constexpr int KC = (3 * J + KSTEP - 1) / KSTEP * KSTEP;  // concatenated K (kKcat): [lo | hi | hi]
    static constexpr int KCSTEPS = KC / KSTEP;
    static constexpr int ACOLS = kKcat ? (kF16 ? KC / 2 : KC) : 2 * KP;  // TMEM columns of one A buffer
    static constexpr int NP = (J * J + 15) / 16 * 16;      // N padded to 16 (M = 128)
    static constexpr int LD = factor_ld(J, 4);             // padded factor row (floats)
    static constexpr int NQ = LD / 4;                       // 16-byte chunks per factor row
    static constexpr int KQ = KP / 4;                       // 16-byte chunks per A row
    static constexpr int NCH = (J * J + 15) / 16;           // 16-column TMEM chunks holding t
    // TMEM (all 512 columns): accumulators [b*NP, (b+1)*NP), A buffers at ACOL + a*ACOLS
    // (hi, then lo; or the concatenated [hi | lo | hi])
    static constexpr int ACOL = kNT * NP;
    static constexpr int TCOLS = 512;
    static_assert(ACOL + kNA * ACOLS <= TCOLS, "TMEM columns");
    // shared memory map (bytes)
    static constexpr int B_BYTES = kKcat ? NP * KC * 4 / 2 : NP * KP * 4;  // one of B_hi / B_lo (kKcat: half of B)
    static constexpr int RSLOT = 2 * NQ * kE * 16 + kE * 4 + (kNoStash ? kE * 4 : 0);  // rows a0, a1 (chunk-major), x (, scale)
    static constexpr int CSLOT = 3 * kE * 4;                // coordinate ring slot: c0, c1, x
    static constexpr int JD = (J + 1) / 2 * 2;              // delta doubles per lane (even: 16-byte pairs)
    static constexpr int DSLOT = JD * kE * 8 + kE * 4;      // delta ring slot: delta[u][j] (fp64), x[u]
    static constexpr int OFF_BHI = 0;
    static constexpr int OFF_BLO = OFF_BHI + B_BYTES;
    static constexpr int OFF_MISC = OFF_BLO + (kF16 ? 0 : B_BYTES);  // tmem base, tiles (fp16: B is one array)
    static constexpr int OFF_ROW = (OFF_MISC + 64 + 127) / 128 * 128;
    static constexpr int OFF_CRD = OFF_ROW + kRing * RSLOT;
    static constexpr int OFF_DEL = OFF_CRD + kCRing * CSLOT;
    // a0/x stash of the level-0 warps (copied out of the row ring when the A rows are
    // split, kNA tiles before the tile is reduced): [warp 0..7][kStash][NQ][32] uint4 + [32] x
    // (+ [32] int: the lane's fp16 scale exponent sA + sG)
    static constexpr int STSLOT = NQ * kWarp * 16 + kWarp * 4 + kWarp * 4;
    static constexpr int OFF_STASH = OFF_DEL + kD * DSLOT;
    static constexpr int OFF_BAR = (OFF_STASH + (kNoStash ? 0 : 8 * kStash * STSLOT) + 7) / 8 * 8;
    // raw_full[kRing], raw_empty[kRing], acc_full[kNT], acc_empty[kNT], a_full[kNA], d_full[4][kD], d_empty[4][kD],
    // a_empty[kNA]
    static constexpr int NBAR = 2 * kRing + 2 * kNT + 2 * kNA + 8 * kD + 1;  // + b_free (table mode)
    static constexpr int SMEM = OFF_BAR + NBAR * 8;
};

// kKcat: B = [b_hi ; b_lo ; b_hi] along K (Shape::KC rows of K), K-major canonical layout,
// b = the core block G'[(k0, j)][k1] = T[k0*GB + k1*J + j]; rows c >= J^2 and K padding 0.
template <int J>
__device__ __forceinline__ void load_bcat(const float* T, float* sB, int t0, int nt) {
    constexpr int NP = (J * J + 15) / 16 * 16, KC = (3 * J + 7) / 8 * 8, GB = gblk(J, 4);
    for (int i = t0; i < NP * KC; i += nt) {
        const int c = i / KC, k = i % KC;
        float v = 0.f;
        if (c < J * J && k < 3 * J) {
            const int k1 = k % J;
            const float g = T[(c / J) * GB + k1 * J + (c % J)];
            const float hv = tf32_rna(g);
            v = (k >= J && k < 2 * J) ? tf32_rna(g - hv) : hv;  // [b_hi ; b_lo ; b_hi]
        }
        sB[kmaj<KC>(c, k)] = v;
    }
}

// kF16: the same B in fp16 from the core block scaled by 2^sG: K-major canonical layout of
// 16-bit elements (core matrix = 8 rows x 8 elements), element (c, k) at byte
// ((c/8)*(KC/8) + k/8)*128 + (c%8)*16 + (k%8)*2.
template <int J>
__device__ __forceinline__ void load_bcat16(const float* T, unsigned char* sB, int t0, int nt, int sG) {
    constexpr int NP = (J * J + 15) / 16 * 16, KC = (3 * J + 15) / 16 * 16, GB = gblk(J, 4);
    const float sc = exp2f_int(sG);
    for (int i = t0; i < NP * KC; i += nt) {
        const int c = i / KC, k = i % KC;
        __half v = __float2half_rn(0.f);
        if (c < J * J && k < 3 * J) {
            const int k1 = k % J;
            const float g = T[(c / J) * GB + k1 * J + (c % J)] * sc;
            const __half hv = __float2half_rn(g);
            v = (k >= J && k < 2 * J) ? __float2half_rn(g - __half2float(hv)) : hv;  // [b_hi ; b_lo ; b_hi]
        }
        *reinterpret_cast<__half*>(sB + ((c >> 3) * (KC / 8) + (k >> 3)) * 128 + (c & 7) * 16 + (k & 7) * 2) = v;
    }
}

// Static serpentine assignment of groups (4 slices each) to CTAs.
struct Sched {
    int ngroups, r;
    int G, b;
    __device__ int group() const { return r * G + ((r & 1) ? (G - 1 - b) : b); }
    __device__ bool valid() const { return group() < ngroups; }
};

// Segment data of the current group for one normal-equation thread.
struct Seg {
    int iters;     // tiles of the group (longest slice = its first)
    int row, len;  // segment row (-1: pad lane) and length
    int slot;      // SELL lane slot (partials)
};

__device__ __forceinline__ void setmaxnreg_ne() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegNE)); }
__device__ __forceinline__ void setmaxnreg_l0() {
    if constexpr (kRegL0 > kRegLaunch) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegL0));
    else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegL0));
}
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegP)); }

// G0 (level-0 grouping, LAST64 only): 1 = every a0[k0] t[k0][j] product and the sum
// in fp64 (F32-B); g > 1 = partial sums over runs of g consecutive k0 in fp32
// (one rounded product, then FMAs), each partial converted to fp64 once and the
// partials summed in fp64: J*ceil(J/g) instead of J^2 fp32->fp64 conversions per
// entry (F2F runs on the quarter-rate XU pipe; tools/l0_row_errors.py and
// tools/level0_emulation.py measure the row error of each g).
// TBL: table mode (order-4 one-small-mode tables, p.aux_stride > 0): the core block B is
// swapped per i_s class by the MMA warp (a separate instantiation: the runtime check
// cost the plain kernel ~2%).
template <int J, bool LAST64, int G0, bool TBL = false>
__global__ void __launch_bounds__(kThreads, 1) k_update_tc(const UpdateParams<float> p) {
    using SH = Shape<J>;
    constexpr int KP = SH::KP, NP = SH::NP, NQ = SH::NQ, KQ = SH::KQ, NCH = SH::NCH;
    constexpr int NB = J * (J + 1) / 2;
    constexpr int GB = gblk(J, 4);
    using TD = typename std::conditional<LAST64, double, float>::type;
    extern __shared__ __align__(1024) unsigned char sm[];
    float* sBhi = reinterpret_cast<float*>(sm + SH::OFF_BHI);
    float* sBlo = reinterpret_cast<float*>(sm + SH::OFF_BLO);
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + SH::OFF_MISC);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w4 = warp & 3;                 // slice of the group = TMEM lane quarter of the warp
    const int te = w4 * kWarp + lane;        // TMEM lane = segment of the group
    const uint32_t bar0 = smem_u32(sm + SH::OFF_BAR);
    auto raw_full = [&](int s) { return bar0 + 8u * s; };
    auto raw_empty = [&](int s) { return bar0 + 8u * (kRing + s); };
    auto acc_full = [&](int b) { return bar0 + 8u * (2 * kRing + b); };
    auto acc_empty = [&](int b) { return bar0 + 8u * (2 * kRing + kNT + b); };
    auto a_full = [&](int a) { return bar0 + 8u * (2 * kRing + 2 * kNT + a); };
    auto d_full = [&](int w, int s) { return bar0 + 8u * (2 * kRing + 2 * kNT + kNA + w * kD + s); };
    auto d_empty = [&](int w, int s) { return bar0 + 8u * (2 * kRing + 2 * kNT + kNA + 4 * kD + w * kD + s); };
    auto a_empty = [&](int a) { return bar0 + 8u * (2 * kRing + 2 * kNT + kNA + 8 * kD + a); };
    const uint32_t b_free = bar0 + 8u * (2 * kRing + 2 * kNT + 2 * kNA + 8 * kD);  // all MMAs so far done
    // row ring slot s: chunk q of row k (0: a0, 1: a1) of segment u; x of segment u
    auto rowc = [&](int s, int k, int q, int u) -> uint4* {
        return reinterpret_cast<uint4*>(sm + SH::OFF_ROW + s * SH::RSLOT) + ((k * NQ + q) * kE + u);
    };
    auto rowx = [&](int s, int u) -> float* {
        return reinterpret_cast<float*>(sm + SH::OFF_ROW + s * SH::RSLOT + 2 * NQ * kE * 16) + u;
    };
    auto rowscale = [&](int s, int u) -> int* {  // kNoStash: the lane's fp16 scale exponent (split -> level 0)
        return reinterpret_cast<int*>(sm + SH::OFF_ROW + s * SH::RSLOT + 2 * NQ * kE * 16 + kE * 4) + u;
    };
    // coordinate ring slot s: c0, c1, x (a = 0, 1, 2) of segment u
    auto crd = [&](int s, int a, int u) -> uint32_t* {
        return reinterpret_cast<uint32_t*>(sm + SH::OFF_CRD + s * SH::CSLOT) + a * kE + u;
    };
    // delta ring slot s: delta[j] of segment u (fp64), x of segment u
    // lane u's delta contiguous (JD doubles): 16-byte stores/loads; the lane stride JD*8
    // bytes (an odd multiple of 16 for J = 10) keeps a quarter-warp's 16-byte accesses
    // on distinct banks
    auto dslot2 = [&](int s, int q, int u) -> double2* {
        return reinterpret_cast<double2*>(sm + SH::OFF_DEL + s * SH::DSLOT) + u * (SH::JD / 2) + q;
    };
    auto dslot_x = [&](int s, int u) -> float* {
        return reinterpret_cast<float*>(sm + SH::OFF_DEL + s * SH::DSLOT + SH::JD * kE * 8) + u;
    };
    const int ngroups = (int)((p.nslices + 3) / 4);  // nslices * 32 < 2^31 (nnz <= INT32_MAX)
    const Sched s0{ngroups, 0, (int)gridDim.x, (int)blockIdx.x};

    // ---------------------------------------------------------------- setup
    pdl_trigger_early();  // the next grid may be placed on the SMs this one vacates
    if constexpr (NQ == 3) {
        // packed J = 10 gathers write 8 of chunk 2's 16 bytes: the rest (row padding) stays zero
        for (int i = threadIdx.x; i < kRing * 2 * kE; i += kThreads) {
            const int sl = i / (2 * kE), k = (i / kE) % 2, u = i % kE;
            float* c2 = reinterpret_cast<float*>(rowc(sl, k, 2, u));
            c2[2] = 0.f;
            c2[3] = 0.f;
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&misc[0])),
                     "n"(SH::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 14) {
        if (lane == 0) {
            for (int s = 0; s < kRing; ++s) {
                mbar_init(raw_full(s), 2 * kWarp);  // loader lanes: cp.async completion + plain arrive (x)
                mbar_init(raw_empty(s), 4);         // the 4 level-0 warps of the tile (split: a1 to TMEM, a0/x to the stash)
            }
            for (int b = 0; b < kNT; ++b) {
                mbar_init(acc_full(b), 1);   // tcgen05.commit
                mbar_init(acc_empty(b), 4);  // level-0 warps done reading the accumulator
            }
            for (int a = 0; a < kNA; ++a) {
                mbar_init(a_full(a), 4);   // the 4 level-0 warps of the tile wrote their A rows
                mbar_init(a_empty(a), 1);  // tcgen05.commit: the MMAs reading A buffer a completed
                if (a == 0) mbar_init(b_free, 1);  // table mode: tcgen05.commit before a core-block switch
            }
            for (int w = 0; w < 4; ++w)
                for (int s = 0; s < kD; ++s) {
                    mbar_init(d_full(w, s), kDfull1 ? 1 : kWarp);  // lane 0 of level-0 warp w after a __syncwarp (its delta stores)
                    mbar_init(d_empty(w, s), 1);     // normal-equation warp 4+w read the slot
                }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    }
    // PDL: everything above touches only this CTA's shared memory and TMEM; the core, the
    // index and the factors may have been written by the preceding grid
    pdl_wait_trigger();
    // B = core (hi/lo tf32 split), K-major: Bt[(k0, j)][k1] = G'[k0][k1][j]
    int sG = 0;  // kF16: core scale exponent (max |G| over every block this launch reads)
    if constexpr (kF16) {
        if (threadIdx.x == 0) misc[2] = 0u;
        __syncthreads();
        uint32_t mb = 0u;
        for (int i = threadIdx.x; i < p.gp_elems; i += kThreads) mb = max(mb, __float_as_uint(p.Gp[i]) & 0x7FFFFFFFu);
        mb = __reduce_max_sync(0xffffffffu, mb);
        if (lane == 0) atomicMax(&misc[2], mb);
        __syncthreads();
        sG = f16_scale_exp(misc[2]);
        load_bcat16<J>(p.Gp, reinterpret_cast<unsigned char*>(sBhi), threadIdx.x, kThreads, sG);
    } else if constexpr (kKcat) {
        load_bcat<J>(p.Gp, sBhi, threadIdx.x, kThreads);
    } else {
    for (int i = threadIdx.x; i < NP * KP; i += kThreads) {
        const int c = i / KP, k1 = i % KP;
        float v = 0.f;
        if (c < J * J && k1 < J) v = p.Gp[(c / J) * GB + k1 * J + (c % J)];
        const float hv = tf32_rna(v);
        sBhi[kmaj<KP>(c, k1)] = hv;
        sBlo[kmaj<KP>(c, k1)] = tf32_rna(v - hv);
    }
    }
    if (warp == 14) {
        // tiles of this CTA = sum of the iteration counts of its groups
        uint32_t n = 0;
        for (int r = lane;; r += kWarp) {
            Sched q = s0;
            q.r = r;
            if (!q.valid()) break;
            n += (uint32_t)__ldg(p.slice_len + q.group() * 4);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        if (lane == 0) misc[1] = n;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = misc[0];
    const uint32_t total = misc[1];

    if (warp >= 12) {
        setmaxnreg_dec();
        // loader warps 14, 12, 13 (the first kLoaders of them; 15 issues the MMAs)
        const int lslot = warp == 14 ? 0 : (warp == 12 ? 1 : (warp == 13 ? 2 : 3));
        if (lslot < kLoaders) {
            // ======================================================== loader(s)
            const uint32_t lp = (uint32_t)lslot;  // this loader's tiles: k = lp (mod kLoaders)
            // J = 10 with packed gather tables (option "pack_gathers"): 2.5x less DRAM traffic,
            // but the 8-byte tail copies make the update ~10% slower
            const bool kPacked = J == 10 && p.gmain[0] != nullptr;
            const bool rows_l1 = p.rows_l1 != 0;
            const uint64_t pol_stream = policy_evict_first(), pol_rows = policy_evict_last();
            // coordinate cursor (tile kc): this lane's 4 segments u = lane + 32 i, i = slice of the group
            Sched pc = s0;
            int pe = 0, piters = 0, plen[4];
            int64_t poff[4];
            bool pend = total == 0;
            auto load_group = [&]() {
                const int64_t g0 = (int64_t)pc.group() * 4;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool v = g0 + i < p.nslices;
                    plen[i] = v ? __ldg(p.slice_len + g0 + i) : 0;
                    poff[i] = v ? __ldg(p.slice_off + g0 + i) + lane : 0;
                }
                piters = plen[0];
                pe = 0;
                if (piters == 0) pend = true;  // groups are sorted by length: nothing follows an empty group
            };
            if (!pend) load_group();
            uint32_t kc = 0;
            auto advance = [&]() {
                ++kc;
                if (++pe == piters) {
                    ++pc.r;
                    if (pc.valid()) load_group();
                    else pend = true;
                }
            };
            // coordinates of this loader's next tile (the cursor walks every tile)
            auto issue_crd = [&]() {
                while (!pend && kc % kLoaders != lp) advance();
                if (pend) return;
                const int s = (int)(kc % kCRing);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int u = lane + kWarp * i;
                    const int64_t idx = poff[i] + (int64_t)pe * kWarp;
                    if (pe < plen[i]) {
                        cp_async4_hint(crd(s, 0, u), p.sc[0] + idx, pol_stream);
                        cp_async4_hint(crd(s, 1, u), p.sc[1] + idx, pol_stream);
                        cp_async4_hint(crd(s, 2, u), p.sv + idx, pol_stream);
                    } else {
                        *crd(s, 0, u) = 0u;  // padding entry: gather row 0 (its result is masked)
                        *crd(s, 1, u) = 0u;
                    }
                }
                advance();
            };
            for (int s = 0; s < kCPref; ++s) {
                issue_crd();
                cp_async_commit();
            }
#if defined(PT_TRACE) && defined(PT_TRACE_LOADER)
            long long* const trl = (p.trace && blockIdx.x == 0 && lane == 0) ? p.trace + 6 * 512 : nullptr;
#else
            constexpr long long* trl = nullptr;  // loader trace off: the 40-register loader must not spill
#endif
            for (uint32_t k = lp; k < total; k += kLoaders) {
                const int s = (int)(k % kRing), cs = (int)(k % kCRing);
                const bool tl = trl && k >= 64 && k < 128;
                if (tl) trl[(k - 64) * 8 + 0] = clock64();
                if (k >= (uint32_t)kRing) {
                    if constexpr (kLoaderSleep > 0) mbar_wait_sleep(raw_empty(s), ((k / kRing) + 1) & 1, kLoaderSleep);
                    else mbar_wait(raw_empty(s), ((k / kRing) + 1) & 1);
                }
                if (tl) trl[(k - 64) * 8 + 1] = clock64();
                cp_async_wait<kCPref - 1>();  // coordinates of tile k (committed kCPref groups ago)
                if (tl) trl[(k - 64) * 8 + 2] = clock64();
                if (kPacked) {
                    // J = 10 packed tables: 32-byte head (2 chunks) + 8-byte tail per row; the
                    // upper half of chunk 2 stays zero (set once at setup)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int u = lane + kWarp * i;
                        const int64_t c0 = (int)*crd(cs, 0, u), c1 = (int)*crd(cs, 1, u);
                        const char* h0 = reinterpret_cast<const char*>(p.gmain[0] + c0 * 8);
                        const char* h1 = reinterpret_cast<const char*>(p.gmain[1] + c1 * 8);
                        cp_async16_hint(rowc(s, 0, 0, u), h0, pol_rows);
                        cp_async16_hint(rowc(s, 1, 0, u), h1, pol_rows);
                        cp_async16_hint(rowc(s, 0, 1, u), h0 + 16, pol_rows);
                        cp_async16_hint(rowc(s, 1, 1, u), h1 + 16, pol_rows);
                        cp_async8_hint(rowc(s, 0, 2, u), p.gtail[0] + c0 * 2, pol_rows);
                        cp_async8_hint(rowc(s, 1, 2, u), p.gtail[1] + c1 * 2, pol_rows);
                        *rowx(s, u) = __uint_as_float(*crd(cs, 2, u));
                    }
                } else if (rows_l1) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int u = lane + kWarp * i;
                    const char* r0 = reinterpret_cast<const char*>(p.A[0] + (int64_t)(int)*crd(cs, 0, u) * p.lda);
                    const char* r1 = reinterpret_cast<const char*>(p.A[1] + (int64_t)(int)*crd(cs, 1, u) * p.lda);
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        cp_async16_l1(rowc(s, 0, q, u), r0 + 16 * q, pol_rows);
                        cp_async16_l1(rowc(s, 1, q, u), r1 + 16 * q, pol_rows);
                    }
                    *rowx(s, u) = __uint_as_float(*crd(cs, 2, u));
                }
                } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int u = lane + kWarp * i;
#if defined(PT_EXP_SMALLGATHER)  // experiment (wrong results): rows of a 4096-row window (L2-resident)
                    const char* r0 = reinterpret_cast<const char*>(p.A[0] + (int64_t)((int)*crd(cs, 0, u) & 4095) * p.lda);
                    const char* r1 = reinterpret_cast<const char*>(p.A[1] + (int64_t)((int)*crd(cs, 1, u) & 4095) * p.lda);
#elif defined(PT_EXP_NOGATHER)  // experiment (wrong results): no row gathers at all
                    if (true) { *rowx(s, u) = 0.f; continue; }
                    const char* r0 = reinterpret_cast<const char*>(p.A[0]);
                    const char* r1 = reinterpret_cast<const char*>(p.A[1]);
#else
                    PT_CHK((int)*crd(cs, 0, u) >= 0 && (int)*crd(cs, 0, u) < p.dim_other[0]);
                    PT_CHK((int)*crd(cs, 1, u) >= 0 && (int)*crd(cs, 1, u) < p.dim_other[1]);
                    const char* r0 = reinterpret_cast<const char*>(p.A[0] + (int64_t)(int)*crd(cs, 0, u) * p.lda);
                    const char* r1 = reinterpret_cast<const char*>(p.A[1] + (int64_t)(int)*crd(cs, 1, u) * p.lda);
#endif
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        cp_async16_hint(rowc(s, 0, q, u), r0 + 16 * q, pol_rows);
                        cp_async16_hint(rowc(s, 1, q, u), r1 + 16 * q, pol_rows);
                    }
                    *rowx(s, u) = __uint_as_float(*crd(cs, 2, u));
                }
                }
                cp_async_mbar_arrive(raw_full(s));  // fires when this lane's rows have landed
                mbar_arrive(raw_full(s));           // x (plain stores), release
                if (tl) trl[(k - 64) * 8 + 3] = clock64();
                issue_crd();
                cp_async_commit();
                if (tl) trl[(k - 64) * 8 + 4] = clock64();
            }
            cp_async_wait<0>();
        } else if (warp == 15) {
            // ====================================================== MMA issue (lane 0)
            // Table mode (order-4 small-mode tables, p.aux_stride > 0): the core block B is
            // T[i_s] of the group's class (every group has one i_s, index aux_groups); at a
            // class change the warp waits for all issued MMAs (b_free), rewrites B hi/lo and
            // makes it visible to the tensor core before the group's first MMA.
            constexpr bool tbl = TBL;
            Sched gs = s0;
            int g_left = 0, cur_aux = 0, g_aux = 0;
            uint32_t bpar = 0;
            auto next_group = [&]() {  // first group (from gs on) with tiles; its tile count
                while (gs.valid()) {
                    const int it = __ldg(p.slice_len + gs.group() * 4);
                    if (it > 0) return it;
                    ++gs.r;
                }
                return 0;
            };
            if constexpr (tbl) {
                g_left = next_group();
                if (gs.valid()) g_aux = __ldg(p.lane_aux + (int64_t)gs.group() * 128);
            }
            // instruction descriptor: D f32 (bits 4-5), A/B format (bits 7-9, 10-12: tf32 = 2,
            // f16 = 0), both K-major, N >> 3 (bits 17-22), M >> 4 (bits 24-28)
            const uint32_t idesc = (1u << 4) | (kF16 ? 0u : (2u << 7) | (2u << 10)) | ((uint32_t)(NP >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
            // B descriptors (K-major, SWIZZLE_NONE; LBO: next 16-byte K chunk = next core
            // matrix (128 B); SBO: next 8 rows), per K-step of 8
            uint64_t dbhi[SH::KSTEPS], dblo[SH::KSTEPS], dbc[SH::KCSTEPS];
#pragma unroll
            for (int ks = 0; ks < SH::KSTEPS; ++ks) {
                dbhi[ks] = umma_desc(smem_u32(sBhi) + ks * 256, 128, KP * 32);
                dblo[ks] = umma_desc(smem_u32(sBlo) + ks * 256, 128, KP * 32);
            }
#pragma unroll
            for (int ks = 0; ks < SH::KCSTEPS; ++ks)  // a K-step = 2 core matrices (32 bytes of K) either way
                dbc[ks] = umma_desc(smem_u32(sBhi) + ks * 256, 128, SH::KC * (kF16 ? 16 : 32));
            // optional trace (tools/trace_tc.py): CTA 0, tiles [64, 128)
#ifdef PT_TRACE
            long long* const trm = (p.trace && blockIdx.x == 0) ? p.trace + 4 * 512 : nullptr;
#else
            constexpr long long* trm = nullptr;
#endif
            // table mode: the whole warp runs the loop in lockstep (lane 0 issues); otherwise
            // lane 0 alone (a diverged remainder of the warp must not spin beside it)
            for (uint32_t k = 0; (tbl || lane == 0) && k < total; ++k) {
                const int a = (int)(k % kNA), b = (int)(k % kNT);
                if constexpr (tbl) {
                    if (g_left == 0) {  // next group: its class, loaded once
                        ++gs.r;
                        g_left = next_group();
                        g_aux = __ldg(p.lane_aux + (int64_t)gs.group() * 128);
                    }
                    const int aux = g_aux;
                    if (aux != cur_aux) {
                        if (lane == 0)
                            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                             b_free)
                                         : "memory");
                        mbar_wait(b_free, bpar);
                        bpar ^= 1u;
                        const float* T = p.Gp + (int64_t)aux * p.aux_stride;
                        if constexpr (kF16) {
                            load_bcat16<J>(T, reinterpret_cast<unsigned char*>(sBhi), lane, kWarp, sG);
                        } else if constexpr (kKcat) {
                            load_bcat<J>(T, sBhi, lane, kWarp);
                        } else {
#pragma unroll 8
                        for (int i = lane; i < NP * KP; i += kWarp) {
                            const int c = i / KP, k1 = i % KP;
                            float v = 0.f;
                            if (c < J * J && k1 < J) v = T[(c / J) * GB + k1 * J + (c % J)];
                            const float hv = tf32_rna(v);
                            sBhi[kmaj<KP>(c, k1)] = hv;
                            sBlo[kmaj<KP>(c, k1)] = tf32_rna(v - hv);
                        }
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        cur_aux = aux;
                    }
                    --g_left;
                }
                const bool tr = trm && lane == 0 && k >= 64 && k < 128;
                if (tr) trm[(k - 64) * 8 + 0] = clock64();
                mbar_wait(a_full(a), (k / kNA) & 1);  // A rows of tile k written
                if (tr) trm[(k - 64) * 8 + 1] = clock64();
                if (k >= (uint32_t)kNT) mbar_wait(acc_empty(b), ((k / kNT) + 1) & 1);  // accumulator b read (tile k-kNT)
                if (tr) trm[(k - 64) * 8 + 2] = clock64();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                // 3xTF32: lo*hi, hi*lo, hi*hi (small terms first)
                const uint32_t d = tmem + b * NP;
                const uint32_t ahi = tmem + SH::ACOL + a * SH::ACOLS;
                [[maybe_unused]] const uint32_t alo = ahi + KP;
                uint32_t acc = 0;
#ifdef PT_EXP_NOMMA  // experiment (wrong results): one MMA per tile instead of 3 x KSTEPS
                mma_tf32_ta(d, ahi, dbhi[0], idesc, 0);
#else
                // (braces around both branches: a discarded `else` followed by a #pragma-annotated
                // loop once swallowed the next statement, the accumulator commit, and the kernel hung)
                if constexpr (kKcat) {
#pragma unroll
                    for (int ks = 0; ks < SH::KCSTEPS; ++ks) {  // 8 TMEM columns of A per K-step
                        if constexpr (kF16) mma_f16_ta(d, ahi + 8 * ks, dbc[ks], idesc, acc);
                        else mma_tf32_ta(d, ahi + 8 * ks, dbc[ks], idesc, acc);
                        acc = 1;
                    }
                } else {
#pragma unroll
                    for (int pr = 0; pr < 3; ++pr) {
#pragma unroll
                        for (int ks = 0; ks < SH::KSTEPS; ++ks) {
                            mma_tf32_ta(d, (pr == 0 ? alo : ahi) + 8 * ks, pr == 1 ? dblo[ks] : dbhi[ks], idesc, acc);
                            acc = 1;
                        }
                    }
                }
#endif
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 acc_full(b))
                             : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 a_empty(a))
                             : "memory");
                }
                if (tr) {
                    trm[(k - 64) * 8 + 3] = clock64();
                    if (p.trace[8 * 512 - 1] == 1) {  // latency probe: wait for this tile's MMAs
                        mbar_wait(acc_full(b), (k / kNT) & 1);
                        trm[(k - 64) * 8 + 4] = clock64();
                    }
                }
                if constexpr (tbl) __syncwarp();
            }
        }
    } else if (warp < 8) {
        // ================================================================ level 0
        setmaxnreg_l0();
        const uint32_t par = (uint32_t)(warp >> 2);  // this warp takes the tiles k = par (mod 2)
        unsigned char* const stash = sm + SH::OFF_STASH + warp * kStash * SH::STSLOT;
        const uint32_t tm_lane = tmem + ((uint32_t)(w4 * 32) << 16);
#ifdef PT_TRACE
        long long* const trb = (p.trace && blockIdx.x == 0 && lane == 0 && warp < 4) ? p.trace + warp * 512 : nullptr;
#else
        constexpr long long* trb = nullptr;
#endif
        auto mark = [&](uint32_t k, int ph) {
            if (trb && k >= 64 && k < 192) trb[((k - 64) >> 1) * 8 + ph] = clock64();
        };
        // Tile k: once its rows have landed and MMA k - kNA (the last reader of A buffer
        // k % kNA) has completed, write this thread's A row into TMEM lane te of that
        // buffer (hi = a rounded to tf32 by two integer ops, lo = a - hi exact; the
        // tensor core truncates lo to tf32, an error <= 2^-21 |a|; columns k >= J are
        // zero) and arrive (one arrival per warp) for the MMA warp.
        auto split = [&](uint32_t k) {
            const int s = (int)(k % kRing);
            mbar_wait(raw_full(s), (k / kRing) & 1);
            if (k >= (uint32_t)kNA) mark(k - kNA, 7);
            // A buffer k % kNA was last read by MMA k - kNA (its own barrier: each phase
            // is one use of the buffer, so this wait can never be two phases behind)
            if (k >= (uint32_t)kNA) mbar_wait(a_empty((int)(k % kNA)), ((k / kNA) + 1) & 1);
            uint32_t hi[16], lo[16];
            int sA = 0;  // kF16: row scale exponent
#pragma unroll
            for (int q = 0; q < KQ; ++q) {
                uint32_t wv[4] = {0u, 0u, 0u, 0u};
                if (q < NQ) {
                    const uint4 r = *rowc(s, 1, q, te);
                    wv[0] = r.x, wv[1] = r.y, wv[2] = r.z, wv[3] = r.w;
                }
#pragma unroll
                for (int v = 0; v < 4; ++v) hi[4 * q + v] = wv[v];
            }
            if constexpr (kF16) {
                uint32_t mb = 0u;
#pragma unroll
                for (int i = 0; i < J; ++i) mb = max(mb, hi[i] & 0x7FFFFFFFu);
                sA = f16_scale_exp(mb);
                const float sc = exp2f_int(sA);
#pragma unroll
                for (int i = 0; i < J; ++i) hi[i] = __float_as_uint(__uint_as_float(hi[i]) * sc);  // exact
            }
#pragma unroll
            for (int i = 0; i < 4 * KQ; ++i) {
                // hi = the value rounded to 11 significant bits (nearest, ties away), lo = the exact
                // remainder; fp16 holds hi exactly (after the scaling) and rounds lo to nearest, the
                // tensor core truncates a tf32 lo
                const uint32_t w = hi[i];
                const uint32_t hh = (w + 0x1000u) & 0xFFFFE000u;
                hi[i] = hh;
                lo[i] = __float_as_uint(__uint_as_float(w) - __uint_as_float(hh));
            }
            // a0 and x of the tile go to this warp's stash: the ring slot is free once split
            if constexpr (kNoStash) {
                if constexpr (kF16) *rowscale(s, te) = sA + sG;
            } else {
                const int st = (int)((k >> 1) % kStash);
                unsigned char* sb = stash + st * SH::STSLOT;
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    reinterpret_cast<uint4*>(sb)[q * kWarp + lane] = *rowc(s, 0, q, te);
                reinterpret_cast<float*>(sb + NQ * kWarp * 16)[lane] = *rowx(s, te);
                if constexpr (kF16) reinterpret_cast<int*>(sb + NQ * kWarp * 16 + kWarp * 4)[lane] = sA + sG;
            }
            const uint32_t ta = tm_lane + SH::ACOL + (k % kNA) * SH::ACOLS;
            if constexpr (kF16) {
                // [a_lo | a_hi | a_hi | 0] over KC fp16 elements, two per TMEM column (lower K
                // index in the low half), against [b_hi ; b_lo ; b_hi]
                float v[SH::KC];
#pragma unroll
                for (int i = 0; i < SH::KC; ++i)
                    v[i] = __uint_as_float(i < J ? lo[i] : (i < 2 * J ? hi[i - J] : (i < 3 * J ? hi[i - 2 * J] : 0u)));
                uint32_t w[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) w[c] = 2 * c + 1 < SH::KC ? pack_h2(v[2 * c], v[2 * c + 1]) : 0u;
                if constexpr (SH::ACOLS == 16) tmem_st16(ta, w);
                else tmem_st8(ta, w);
            } else if constexpr (kKcat) {
                // [a_lo | a_hi | a_hi | 0] over KC columns (against [b_hi ; b_lo ; b_hi]: the two
                // small products first, as in the 3-sweep order -- big-first doubled the worst
                // full-size c5 row error to 1.9e-5), stored 16 (or 8) at a time
                uint32_t v[SH::KC];
#pragma unroll
                for (int i = 0; i < SH::KC; ++i)
                    v[i] = i < J ? lo[i] : (i < 2 * J ? hi[i - J] : (i < 3 * J ? hi[i - 2 * J] : 0u));
#pragma unroll
                for (int c0 = 0; c0 < SH::KC; c0 += 16) {
                    uint32_t w[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) w[i] = c0 + i < SH::KC ? v[c0 + i] : 0u;
                    if (c0 + 16 <= SH::KC) tmem_st16(ta + c0, w);
                    else tmem_st8(ta + c0, w);
                }
            } else if constexpr (KP == 16) {
                tmem_st16(ta, hi);
                tmem_st16(ta + KP, lo);
            } else {
                tmem_st8(ta, hi);
                tmem_st8(ta + KP, lo);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(a_full((int)(k % kNA)));
                if constexpr (!kNoStash) mbar_arrive(raw_empty(s));
            }
        };
        // this warp writes the A rows of its own tiles (kNA is even: tile k + kNA has
        // the parity of k), kNA tiles ahead of the one it reduces
        static_assert(kNA % 2 == 0, "level-0 warps split their own tiles");
        for (uint32_t k = par; k < (uint32_t)kNA && k < total; k += 2) split(k);
        for (uint32_t k = par; k < total; k += 2) {
            const int b = (int)(k % kNT), s = (int)(k % kRing);
            mark(k, 0);
            if (!kSplitLate && k + kNA < total) split(k + kNA);
            mark(k, 6);
            mbar_wait(acc_full(b), (k / kNT) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            mark(k, 1);
            // the first kBCH chunks of t in flight (the rest follow once those are consumed)
            uint32_t rb[kBCH][16];
            const uint32_t taddr = tm_lane + b * NP;
#pragma unroll
            for (int ch = 0; ch < kBCH && ch < NCH; ++ch) tmem_ld16(taddr + ch * 16, rb[ch]);
            // a0 and x of tile k from this warp's stash (written by this thread in split(k)), or
            // (kNoStash) from the ring slot itself, which is released here
            const unsigned char* sbk = stash + (int)((k >> 1) % kStash) * SH::STSLOT;
            float a0f[J];
            float x;
            int ssc;  // kF16: t arrives scaled by 2^ssc (row and core scalings), undone in the weights
            if constexpr (kNoStash) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const uint4 v = *rowc(s, 0, q, te);
                    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * q + u < J) a0f[4 * q + u] = __uint_as_float(wv[u]);
                }
                x = *rowx(s, te);
                ssc = kF16 ? *rowscale(s, te) : 0;
                __syncwarp();
                if (lane == 0) mbar_arrive(raw_empty(s));
            } else {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const float4 v = reinterpret_cast<const float4*>(sbk)[q * kWarp + lane];
                    const float wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * q + u < J) a0f[4 * q + u] = wv[u];
                }
                x = reinterpret_cast<const float*>(sbk + NQ * kWarp * 16)[lane];
                ssc = kF16 ? reinterpret_cast<const int*>(sbk + NQ * kWarp * 16 + kWarp * 4)[lane] : 0;
            }
            mark(k, 2);
#pragma unroll
            for (int ch = 0; ch < kBCH && ch < NCH; ++ch) tmem_wait16(rb[ch]);
            mark(k, 3);
            // level 0: d[j] = sum_k0 a0[k0] t[k0][j]; t[k0][j] is TMEM column k0*J + j
            TD d[J];
            float pf[J];  // fp32 partial sums (G0 > 1)
            double a0d[J];
            // (G0 == 1, fp64: folded into a0 exactly; the other paths scale delta at the end)
            constexpr bool kFold = LAST64 && G0 == 1 && kL0Conv == 1;
            const double wsc_int = kF16 ? exp2d_int(896 - ssc) : 0x1p896, wsc_xu = kF16 ? exp2d_int(-ssc) : 1.0;
#pragma unroll
            for (int q = 0; q < J; ++q) {
                a0d[q] = kA0Int ? f2d_int(a0f[q]) : double(a0f[q]);
                // scheme 1: a0[k0] * 2^896 pairs with f2d_scaled(t) = t * 2^-896 (both exact)
                if (kFold && !((kXuMask >> q) & 1u)) a0d[q] *= wsc_int;
                else if (kFold && kF16) a0d[q] *= wsc_xu;
            }
#pragma unroll
            for (int j = 0; j < J; ++j) d[j] = TD(0);
            // G0 == 0 (l0_group 0): level 0 in fp32 pairs (FFMA2 / FADD2, columns j, j + 1) with
            // Kahan compensation: y = a0 t + cn (the product exact inside the FMA, one rounding),
            // s' = s + y, cn = (s - s') + y; delta_j = s_j + cn_j in fp64 (exact widenings) --
            // one rounding per product instead of none (fp64 level 0), and no growth with k0
            static_assert(G0 != 0 || (LAST64 && J % 2 == 0), "compensated level 0: fp64 delta, even J");
            uint64_t ks[G0 == 0 ? J / 2 : 1], kc[G0 == 0 ? J / 2 : 1];
            if constexpr (G0 == 0) {
#pragma unroll
                for (int q = 0; q < J / 2; ++q) ks[q] = kc[q] = 0ull;
            }
#pragma unroll
            for (int cc = 0; cc < J * J; ++cc) {
                const int k0 = cc / J, j = cc % J;
                if (cc % (16 * kBCH) == 0 && cc > 0) {  // next batch of chunks
#pragma unroll
                    for (int q = 0; q < kBCH; ++q)
                        if (cc / 16 + q < NCH) tmem_ld16(taddr + (cc / 16 + q) * 16, rb[q]);
#pragma unroll
                    for (int q = 0; q < kBCH; ++q)
                        if (cc / 16 + q < NCH) tmem_wait16(rb[q]);
                    if (kAccEarly && cc / 16 + kBCH >= NCH) {
                        // the last batch is in registers: accumulator b is free for MMA k + kNT
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive(acc_empty(b));
                    }
                }
                const float tv = __uint_as_float(rb[(cc / 16) % kBCH][cc % 16]);
                if constexpr (G0 == 0) {
                    if (j % 2 == 0) {
                        const uint64_t aa = pack_f32x2(a0f[k0], a0f[k0]);
                        const uint64_t tt = (uint64_t)rb[(cc / 16) % kBCH][cc % 16] |
                                            ((uint64_t)rb[((cc + 1) / 16) % kBCH][(cc + 1) % 16] << 32);
                        const int q = j / 2;
                        const uint64_t y = fma_f32x2(aa, tt, kc[q]);
                        const uint64_t s1 = add_f32x2(ks[q], y);
                        kc[q] = add_f32x2(sub_f32x2(ks[q], s1), y);
                        ks[q] = s1;
                    }
                    continue;
                }
#ifdef PT_EXP_NOL0  // experiment (wrong results): level-0 arithmetic reduced to one fp32 add per term
                if (true) {
                    pf[j] = (k0 == 0 ? 0.f : pf[j]) + tv;
                    if (k0 == J - 1) d[j] = TD(pf[j]);
                } else
#endif
                if constexpr (!LAST64) {
                    d[j] = fmaf(a0f[k0], tv, d[j]);
                } else if constexpr (G0 == 1) {
                    // half of the fp32 -> fp64 conversions by integer ops on the ALU pipe, the
                    // other half on the (quarter-rate) XU pipe, so neither pipe saturates
                    if constexpr (kL0Conv == 1)
                        d[j] = fma(a0d[k0], ((kXuMask >> k0) & 1u) ? TD(tv) : f2d_scaled(tv), d[j]);
                    else
                        d[j] = fma(a0d[k0], (cc % kXuMod == 0) ? TD(tv) : f2d_int(tv), d[j]);
                } else {
                    if (k0 % G0 == 0) pf[j] = a0f[k0] * tv;
                    else pf[j] = fmaf(a0f[k0], tv, pf[j]);
                    if (k0 % G0 == G0 - 1 || k0 == J - 1) d[j] = d[j] + TD(pf[j]);
                }
            }
            if (!(kAccEarly && NCH > kBCH)) {
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(acc_empty(b));
            }
            if constexpr (G0 == 0) {
#pragma unroll
                for (int q = 0; q < J / 2; ++q) {
                    d[2 * q] = TD(__uint_as_float((uint32_t)ks[q])) + TD(__uint_as_float((uint32_t)kc[q]));
                    d[2 * q + 1] = TD(__uint_as_float((uint32_t)(ks[q] >> 32))) + TD(__uint_as_float((uint32_t)(kc[q] >> 32)));
                }
            }
            if constexpr (kF16 && !kFold) {
                // (fp32: in two steps, 2^-ssc can leave the float range)
                const TD u = LAST64 ? TD(exp2d_int(-ssc)) : TD(exp2f_int(-(ssc / 2)));
                const TD u2 = LAST64 ? TD(1) : TD(exp2f_int(-(ssc - ssc / 2)));
#pragma unroll
                for (int j = 0; j < J; ++j) d[j] = d[j] * u * u2;
            }
            mark(k, 4);
            // hand delta (fp64) and x to normal-equation warp 8 + w4
            const int ds = (int)(k % kD);
            if (k >= (uint32_t)kD) mbar_wait(d_empty(w4, ds), ((k / kD) + 1) & 1);
#pragma unroll
            for (int q = 0; q < SH::JD / 2; ++q)
                *dslot2(ds, q, te) = make_double2(double(d[2 * q]), 2 * q + 1 < J ? double(d[2 * q + 1]) : 0.0);
            *dslot_x(ds, te) = x;
            // one arrival per warp, not per lane: every arrival wakes the CTA's sleeping waiters
            // (NANOSLEEP.SYNCS), and 128 per tile dominated their polling
            if constexpr (kNbar) {
                __threadfence_block();
                __syncwarp();
                asm volatile("bar.arrive %0, %1;" ::"r"(1 + w4 * kD + ds), "n"(2 * kWarp) : "memory");
            } else if constexpr (kDfull1) {
                __syncwarp();
                if (lane == 0) mbar_arrive(d_full(w4, ds));
            } else {
                mbar_arrive(d_full(w4, ds));
            }
            mark(k, 5);
            // late split: tile k + kNA's rows get one more level-0 phase to land (the early
            // split waited for them: the row-ring wait was the hottest polling loop)
            if (kSplitLate && k + kNA < total) split(k + kNA);
        }
    } else {
        // ====================================================== normal equations
        setmaxnreg_ne();
        const uint32_t tm_lane = tmem + ((uint32_t)(w4 * 32) << 16);
        auto load_seg = [&](const Sched& s, Seg& g) {
            const int64_t g0 = (int64_t)s.group() * 4;
            const int64_t sl = g0 + w4;
            g.slot = (int)(sl * kWarp + lane);
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
            bool solve = pidx < 0;
            if (!solve) {
                const int stp = p.lane_pstride[g.slot];
                double* dst = p.partials + pidx;
#pragma unroll
                for (int q = 0; q < NB; ++q) dst[(int64_t)q * stp] = B[q];
#pragma unroll
                for (int q = 0; q < J; ++q) dst[(int64_t)(NB + q) * stp] = c[q];
                dst[(int64_t)(NB + J) * stp] = s2;
                if (p.seg_done) solve = heavy_take_row<J>(p.seg_done, p.row_pbase, p.partials, g.row, stp, B, c, s2);
            }
            if (solve) {
                double a[J];
                const bool ok = chol_solve<J>(B, c, p.lambda, a);
                if (!ok) {
                    atomicCAS(p.fail, 0, g.row + 1);
#pragma unroll
                    for (int j = 0; j < J; ++j) a[j] = 0.0;
                }
                float* out = p.An + (int64_t)g.row * p.lda;  // (no PT_CHK here: it made the 192-register role spill)
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
                for (int q = 0; q < SH::NQ; ++q) {
                    const float4 v = make_float4(stv[4 * q], stv[4 * q + 1], stv[4 * q + 2], stv[4 * q + 3]);
                    reinterpret_cast<float4*>(out)[q] = v;
                    for (int r = 0; r < p.peers.n; ++r)  // multi-GPU push into the peer replicas (NVLink)
                        reinterpret_cast<float4*>(static_cast<char*>(p.peers.base[r]) +
                                                  (int64_t)g.row * p.lda * 4)[q] = v;
                }
                p.sse_row[g.row] = sse;
            }
        };
        Sched sc = s0;
        if (sc.valid()) {
            Seg cur, nxt;
            load_seg(sc, cur);
            Sched sn = sc;
            ++sn.r;
            bool nvalid = sn.valid();
            if (nvalid) load_seg(sn, nxt);
            zero();
            int e = 0;
#ifdef PT_TRACE
            long long* const trn = (p.trace && blockIdx.x == 0 && lane == 0 && w4 == 0) ? p.trace + 5 * 512 : nullptr;
#else
            constexpr long long* trn = nullptr;
#endif
            auto markn = [&](uint32_t k, int ph) {
                if (trn && k >= 64 && k < 128) trn[(k - 64) * 8 + ph] = clock64();
            };
            for (uint32_t k = 0; k < total; ++k) {
                const int ds = (int)(k % kD);
                markn(k, 0);
                markn(k, 1);
                if constexpr (kNbar) asm volatile("bar.sync %0, %1;" ::"r"(1 + w4 * kD + ds), "n"(2 * kWarp) : "memory");
                else if constexpr (kNeSleep > 0) mbar_wait_sleep(d_full(w4, ds), (k / kD) & 1, kNeSleep);
                else mbar_wait(d_full(w4, ds), (k / kD) & 1);
                markn(k, 2);
                double dd[J];
#pragma unroll
                for (int q = 0; q < SH::JD / 2; ++q) {
                    const double2 v = *dslot2(ds, q, te);
                    dd[2 * q] = v.x;
                    if (2 * q + 1 < J) dd[2 * q + 1] = v.y;
                }
                const float x = *dslot_x(ds, te);
                __syncwarp();
                if (lane == 0) mbar_arrive(d_empty(w4, ds));
                // an inactive lane (entry beyond its segment: only in a group's tail) skips the
                // update; the branch is warp-uniform almost always, so no per-entry selects
#ifdef PT_EXP_NONE  // experiment (wrong results): normal equations reduced to c += x delta
                if (e < cur.len) {
                    const double xd = double(x);
#pragma unroll
                    for (int i = 0; i < J; ++i) c[i] = fma(xd, dd[i], c[i]);
                } else
#endif
                if (e < cur.len) {
                    const double xd = double(x);
#pragma unroll
                    for (int i = 0; i < J; ++i) {
                        c[i] = fma(xd, dd[i], c[i]);
#pragma unroll
                        for (int j = i; j < J; ++j) B[up_idx(i, j, J)] = fma(dd[i], dd[j], B[up_idx(i, j, J)]);
                    }
                    s2 = fma(xd, xd, s2);
                }
                markn(k, 3);
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
            // the groups after the last one with entries are empty (sorted by length):
            // their rows get a = 0 and SSE 0
            for (; sc.valid(); ++sc.r) {
                load_seg(sc, cur);
                zero();
                finalize(cur);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(SH::TCOLS));
}

template <int J, bool LAST64, int G0, bool TBL = false>
void launch_tc_g(const UpdateParams<float>& p, int grid, cudaStream_t st) {
    auto k = k_update_tc<J, LAST64, G0, TBL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Shape<J>::SMEM);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    launch_pdl(k, grid, kThreads, Shape<J>::SMEM, st, p);
}

template <int J, bool LAST64>
void launch_tc(const void* params, bool literal, int grid, cudaStream_t st) {
    (void)literal;
    const UpdateParams<float>& p = *reinterpret_cast<const UpdateParams<float>*>(params);
    if constexpr (!LAST64) {
        launch_tc_g<J, false, 1>(p, grid, st);
    } else {
        if (p.aux_stride > 0) launch_tc_g<J, true, 1, true>(p, grid, st);  // table mode
        else if (p.l0_group == 1) launch_tc_g<J, true, 1>(p, grid, st);
        else if (p.l0_group == 2) launch_tc_g<J, true, 2>(p, grid, st);
        else if (p.l0_group == 0) {
            if constexpr (J % 2 == 0) launch_tc_g<J, true, 0>(p, grid, st);
            else launch_tc_g<J, true, 1>(p, grid, st);  // (odd J: no column pairs; fp64 level 0)
        }
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
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (getenv("PTUCKER_DEBUG")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, k);
        fprintf(stderr, "[ptucker] tc J=%d smem=%d regs=%d (one CTA of %d threads per SM)\n", J, Shape<J>::SMEM,
                fa.numRegs, kThreads);
    }
    // one CTA per SM: it allocates all 512 TMEM columns
    return Shape<J>::SMEM + 1024 <= smem_sm ? 1 : 0;
}

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
