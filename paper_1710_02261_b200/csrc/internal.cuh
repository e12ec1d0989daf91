// internal.cuh -- shared declarations of the B200 P-Tucker library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace pt {

constexpr int kMaxN = 10;     // orders N = 2..10 (templated kernels for 2..5, update_generic.cu beyond)
constexpr int kWarp = 32;
constexpr int kUpdThreads = 256;  // update kernel CTA size (8 warps, one slice per warp at a time)

// Packed normal-equation record of one row (segment): upper triangle of B
// (J(J+1)/2), c (J), sum x^2 (1) -- all fp64 (Eq. 10-11).
__host__ __device__ constexpr int rec_width(int J) { return J * (J + 1) / 2 + J + 1; }
// Padded row stride of a factor in elements (16-byte rows for vector loads).
__host__ __device__ constexpr int factor_ld(int J, int elem_bytes) {
    return elem_bytes == 4 ? (J + 3) / 4 * 4 : (J + 1) / 2 * 2;
}
// Permuted core block: the innermost (k_{N-2}, j) J x J block, padded to 16 bytes.
__host__ __device__ constexpr int gblk(int J, int elem_bytes) {
    return elem_bytes == 4 ? (J * J + 3) / 4 * 4 : (J * J + 1) / 2 * 2;
}
__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// Checked builds (-DPT_CHECKED, tools/checked_build.sh; compute-sanitizer is closed on this
// pool): index and row bounds asserted in the kernels, a violation traps the kernel.
#ifdef PT_CHECKED
#define PT_CHK(c)           \
    do {                    \
        if (!(c)) __trap(); \
    } while (0)
#else
#define PT_CHK(c) \
    do {          \
    } while (0)
#endif

// Core dimensionality J_1..J_N (Alg. 2 input) for the kernels that accept
// unequal J_n (generic path, predictions, QR core update, Approx literal scores).
struct JDims {
    int j[kMaxN] = {0};
};
inline JDims jdims_uniform(int N, int J) {
    JDims d;
    for (int m = 0; m < N; ++m) d.j[m] = J;
    return d;
}

// Multi-GPU row exchange by push: the other ranks' replicas of A^(n),
// opened from their CUDA IPC handles (ptucker_open_peers).  Every kernel that stores a
// solved row of A^(n) also stores it into each peer replica (NVLink P2P stores), so the
// exchange overlaps the update; a barrier per mode (NCCL) orders it before the next mode.
constexpr int kMaxPeers = 7;
struct PeerRows {
    int n = 0;                          // peers (world - 1), 0: no push
    void* base[kMaxPeers] = {nullptr};  // peer replica of A^(n), same row stride as the local one
};
// Programmatic dependent launch (PDL, option "pdl"): the kernels of a sweep (mode updates,
// heavy-row finalize, error sums) are launched with programmatic stream serialization, so a
// kernel's CTAs are placed on the SMs its predecessor's CTAs vacate and run their prologue
// (TMEM allocation, barrier setup) while the predecessor's tail drains.  Every kernel launched
// this way calls pdl_wait() before it reads anything a predecessor writes: griddepcontrol.wait
// returns once the preceding grid has completed and its stores are visible (immediately when
// the launch carried no programmatic dependency).  pdl_trigger() lets the next grid launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// where a kernel lets its dependent launch: at its start (PT_PDL_LATE 0) or once its own
// pdl_wait() has returned (PT_PDL_LATE 1, the default: see DESIGN.md §9 for the A/B)
#ifndef PT_PDL_LATE
#define PT_PDL_LATE 1
#endif
__device__ __forceinline__ void pdl_trigger_early() {
    if constexpr (!PT_PDL_LATE) pdl_trigger();
}
__device__ __forceinline__ void pdl_wait_trigger() {
    pdl_wait();
    if constexpr (PT_PDL_LATE) pdl_trigger();
}
extern int g_pdl;  // option "pdl" (default 0)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Copy the row just stored at `local` (row_bytes, a multiple of 16) into every peer
// replica at the same row.  The reads return this thread's own stores.
__device__ __forceinline__ void push_row(const PeerRows& pr, const void* local, int64_t row, int row_bytes) {
    if (pr.n == 0) return;
    const uint4* src = reinterpret_cast<const uint4*>(local);
    for (int q = 0; q < row_bytes / 16; ++q) {
        const uint4 v = src[q];
#pragma unroll
        for (int r = 0; r < kMaxPeers; ++r)  // constant indices: the parameter struct stays in param space
            if (r < pr.n) reinterpret_cast<uint4*>(static_cast<char*>(pr.base[r]) + row * row_bytes)[q] = v;
    }
}

// Arguments of the fused row-update kernel for mode n over this rank's
// length-sorted segments (SELL-32 layout).
template <typename TS>
struct UpdateParams {
    int n;                        // mode being updated
    int64_t nslices;              // slices of 32 segments
    const int64_t* slice_off;     // [nslices] first slot of slice s; entry e of lane l at slice_off + e*32 + l
    const int32_t* slice_len;     // [nslices] iterations of slice s (= longest segment, lane 0)
    const int32_t* lane_row;      // [nslices*32] row of the segment in that lane (-1: pad lane)
    const int32_t* lane_len;      // [nslices*32] entries of that segment
    const int64_t* lane_pidx;     // [nslices*32] heavy rows: first partial slot (-1: segment is the whole row)
    const int32_t* lane_pstride;  // [nslices*32] heavy rows: stride between partial components (= #segments of the row)
    const int32_t* lane_aux;      // [nslices*32] small-mode table block of the segment (TABLE kernels only)
    int64_t aux_stride;           // elements per table block
    const int32_t* sc[kMaxN - 1]; // SELL coordinates of the other modes (ascending mode order)
    const TS* sv;                 // SELL values
    const TS* A[kMaxN - 1];       // the other factors, same order, row stride lda
    TS* An;                       // A^(n), written
    int lda;
    const TS* Gp;                 // core permuted for mode n: [outer J^(N-2)][gblk] with block = [k_{N-2}][j]
    int gp_elems;                 // elements of Gp (smem copy)
    double lambda;
    double* partials;             // heavy-row partial records, component-major per row
    double* sse_row;              // [I_n] per-row SSE by the identity (fused error, Eq. 5)
    double* lit_part;             // literal error mode: [nslices*32] per-lane SSE (else null)
    int* fail;                    // numeric failure flag (row+1)
    unsigned int* work;           // dynamic slice counter (reset to 0 before launch)
    int policy;                   // runtime copy of the precision policy (info only)
    long long* trace;             // optional per-phase clock trace (tools; null in production)
    const float* gmain[2];        // tensor-core kernel, J = 10: the two gathered factors with rows split
    const float* gtail[2];        //   into 32-byte heads (floats 0..7) and packed 8-byte tails (8..9)
    int l0_group;                 // tensor-core kernel: level-0 terms summed in fp32 before fp64 (1 or 2)
    int rows_l1;                  // gather factor rows through L1 (skewed gathered modes: hot rows)
    PeerRows peers;               // multi-GPU push: the other ranks' replicas of A^(n) (n = 0: none)
    int64_t dim_other[kMaxN - 1]; // I of the other modes (same order as A[]) -- bounds checks
    int64_t dim_n;                // I_n
    int32_t* seg_done;            // heavy rows solved in the update kernel: per-row segment counters (null: off)
    const int64_t* row_pbase;     //   per-row first partial (heavy rows of this mode)
};

using UpdateLauncher = void (*)(const void* params, bool literal, int grid, cudaStream_t st);
using UpdateOccupancy = int (*)(bool literal, size_t smem);

struct UpdateKernel {
    int prec, l64, N, J;  // l64: outer TTV levels in fp64 (precision policy)
    UpdateLauncher launch;
    UpdateOccupancy occupancy;
};

// Registries filled by the instantiation units (update_f32a.cu: l64 = 0,
// update_f32b.cu: l64 = 1, update_f32c.cu: l64 = N-2 for N >= 4, update_f64.cu).
const UpdateKernel* update_kernels_f32a(int* count);
const UpdateKernel* update_kernels_f32b(int* count);
const UpdateKernel* update_kernels_f32c(int* count);
const UpdateKernel* update_kernels_f32c2(int* count);  // order 5, l64 = 2 (policy 3)
const UpdateKernel* update_kernels_f64(int* count);
// Returns nullptr when (prec, l64, N, J) was not compiled.
const UpdateKernel* find_update_kernel(int prec, int l64, int N, int J);
// Tensor-core variant (fp32, N = 3): innermost TTV stage on tcgen05 (update_tc.cu).
const UpdateKernel* find_update_kernel_tc(int l64, int J);
int tc_kp(int J);  // K padding of the tensor-core A operand (floats per split row)
// J = 10 gather tables of the tensor-core kernel (kernels.cu): head[i] = A[i][0..8), tail[i] = A[i][8..10)
void launch_pack_rows10(const float* A, int64_t I, int lda, float* head, float* tail, cudaStream_t st);

// Generic-order kernel (update_generic.cu): any N <= kMaxN, J <= 16, fp64; p.Gp = G in C order.
void launch_update_generic(const void* params, int elem_bytes, int N, const JDims& J, int nsm, cudaStream_t st,
                           const double* pres = nullptr, const int32_t* sid = nullptr,
                           const uint64_t* sp_digits = nullptr, const int64_t* sp_index = nullptr,
                           const int32_t* sp_off = nullptr);
// P-Tucker-Cache (cache.cu): the cache table Pres (|Omega| x |G|, fp64) over the device COO
void launch_pres_init(int N, const JDims& J, int elem_bytes, const void* G, const void* const* d_A, int lda,
                      const int32_t* coords, int64_t nnz, double* pres, cudaStream_t st);
void launch_pres_update(int N, const JDims& J, int elem_bytes, int n, const void* G, const void* const* d_A, int lda,
                        const void* A_old, const int32_t* coords, int64_t nnz, double* pres, cudaStream_t st);
bool generic_shape_ok(int N, int J);
bool approx_shape_ok(int N, int J);  // approx.cu segment kernels instantiated for (N, J)
// Alg. 4 on the device (approx.cu): scores from U, V; stable top-k truncation
void launch_core_scores(int64_t gsize, int elem_bytes, const void* G, const double* UV, const uint8_t* present,
                        double* R, uint64_t* key, int64_t* idx, cudaStream_t st);
size_t core_select_temp_bytes(int64_t gsize);
cudaError_t launch_core_truncate(int64_t gsize, int64_t k, const uint64_t* key, const int64_t* idx, uint64_t* key_out,
                                 int64_t* idx_out, void* temp, size_t temp_bytes, int elem_bytes, void* G,
                                 uint8_t* present, cudaStream_t st);
// U, V of Eq. 13 from their definition over a device COO (shapes without a compiled (N, J))
void launch_approx_literal(int N, const JDims& J, int elem_bytes, const void* const* d_A, int lda, const int32_t* coords,
                           const void* vals, const double* xhat, int64_t n, int64_t row_lo, int64_t row_hi,
                           double* UV, cudaStream_t st);
void launch_tc_split(const float* A, int64_t I, int lda, int J, float* hi, float* lo, cudaStream_t st);

// (N, J) pairs compiled: N = 2..5, J in {2,3,4,5,8,10}, J^N <= 10^4.
#define PT_NJ_LIST(X) \
    X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 8) X(2, 10) \
    X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 8) X(3, 10) \
    X(4, 2) X(4, 3) X(4, 4) X(4, 5) X(4, 8) X(4, 10) \
    X(5, 2) X(5, 3) X(5, 4) X(5, 5)
#define PT_NJ_LIST_N45(X) \
    X(4, 2) X(4, 3) X(4, 4) X(4, 5) X(4, 8) X(4, 10) \
    X(5, 2) X(5, 3) X(5, 4) X(5, 5)

}  // namespace pt
