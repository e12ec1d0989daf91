/*
 * ptucker.h -- C-ABI of the B200-native P-Tucker row-wise ALS hot path.
 *
 * Method: Oh, Park, Sael, Kang, "Scalable Tucker Factorization for Sparse
 * Tensors - Algorithms and Discoveries" (arXiv 1710.02261).  P:<line> cites
 * /root/reference/PAPER.md.  Readings of the paper (R#) are listed in DESIGN.md.
 *
 * Conventions
 *  - Indices are 0-based (the paper's 1-based notation, stops here).
 *  - "host" pointers are plain CPU memory owned by the caller; every call that
 *    takes one copies synchronously before returning, so the caller may free it.
 *  - The library owns all device memory (one context per process, one GPU per
 *    process: the device current at ptucker_init).  Not thread-safe.
 *  - Precision: PTUCKER_F32 stores values, factors and core in fp32 (the
 *    per-entry contraction runs in fp32, the normal equations B, c and the
 *    solve in fp64); PTUCKER_F64 is fp64 throughout.
 *  - Factor A^(n) host layout: I_n x J_n row-major.  Core host layout: C order
 *    J_1 x ... x J_N (last mode fastest).  Both in the context precision.
 *  - Every function returns PTUCKER_OK (0) or an error code; the message of the
 *    last failure is ptucker_last_error().  Kernel launches are stream-ordered:
 *    a numeric failure inside a kernel (non-positive Cholesky pivot) is
 *    reported by the next synchronising call (ptucker_error, ptucker_get_*,
 *    ptucker_orthogonalize, ptucker_synchronize, ptucker_finalize) as
 *    PTUCKER_ENUMERIC with the (mode, row) in the message.
 */
#ifndef PTUCKER_H
#define PTUCKER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PTUCKER_OK = 0,
    PTUCKER_EINVAL = 1,    /* bad argument (shape, range, non-finite value, lambda <= 0, unsupported (N, J)) */
    PTUCKER_ENUMERIC = 2,  /* non-positive pivot in a row solve, rank-deficient factor in QR */
    PTUCKER_ERESOURCE = 3, /* device allocation failed */
    PTUCKER_ECUDA = 4,     /* CUDA runtime error (message has the driver text) */
    PTUCKER_ENCCL = 5,     /* NCCL error */
    PTUCKER_ESTATE = 6     /* call out of order (e.g. update before init) */
};
enum { PTUCKER_F32 = 0, PTUCKER_F64 = 1 };

/* Library version (major*10000 + minor*100 + patch). */
int32_t ptucker_version(void);

/* Message of the last failing call in this thread ("" if none). */
const char* ptucker_last_error(void);

/* ---------------- multi-GPU bootstrap (skip both when world == 1) --------
 * ptucker_get_unique_id: rank 0 creates an NCCL unique id (128 bytes, host);
 * the caller broadcasts the bytes (e.g. torch.distributed) and every rank then
 * calls ptucker_comm_init(rank, world, id) before ptucker_init (a call while a
 * context is initialised returns PTUCKER_ESTATE: the row blocks of every mode are
 * fixed at init for the world size seen then).  Rows of each
 * mode are then split into nnz-balanced contiguous blocks (see
 * ptucker_partition_rows); each rank updates its block and the blocks are
 * all-gathered over NVLink after each mode (the paper aggregates "all updated
 * rows from all threads", Fig. 3 caption P:517-518). */
int ptucker_get_unique_id(uint8_t out[128]);
int ptucker_comm_init(int32_t rank, int32_t world, const uint8_t id[128]);

/* Row exchange by push (S5, "aggregates all updated rows from all threads", Fig. 3
 * caption P:517-518), after ptucker_init on every rank:
 *  ptucker_peer_handles: writes this rank's N CUDA IPC handles (64 bytes each, A^(0..N-1)
 *    in mode order) into out (host, cap >= 64*N bytes); EINVAL if cap is too small.
 *  ptucker_open_peers: handles = the world ranks' outputs concatenated in rank order
 *    (host, world*64*N bytes, e.g. all-gathered with torch.distributed); opens the other
 *    ranks' replicas (cudaIpcOpenMemHandle, peer access over NVLink).  From then on every
 *    kernel that solves a row of A^(n) also stores it into each peer's replica, so the
 *    exchange overlaps the update; ptucker_update_mode ends with a one-int NCCL all-reduce
 *    that orders all ranks' pushes before the next mode (with no communicator -- ranks
 *    emulated as processes in tests -- the caller must synchronise and barrier between
 *    modes).  world must equal the context's world (communicator or emulate_world);
 *    at most 8 ranks.  ECUDA if a handle cannot be opened (then the NCCL all-gather-v of
 *    ptucker_update_mode stays in use).  The handles are closed by ptucker_finalize /
 *    the next ptucker_init. */
int ptucker_peer_handles(uint8_t* out, int32_t cap);
int ptucker_open_peers(const uint8_t* handles, int32_t world);

/* Pure host helper (no GPU needed): nnz-balanced contiguous row blocks.
 * row_ptr: host, I+1 int64 prefix counts of a mode's slices.  bounds: host,
 * world+1 int64 output; bounds[0] = 0, bounds[world] = I and bounds[g] is the
 * first row r with row_ptr[r] >= ceil(g*nnz/world).  Rows are never split. */
int ptucker_partition_rows(const int64_t* row_ptr, int64_t I, int32_t world, int64_t* bounds);

/* Use this CUDA stream (a cudaStream_t passed as void*, e.g.
 * torch.cuda.current_stream().cuda_stream) for all later work.  NULL selects
 * the library's own non-blocking stream (the default). */
int ptucker_set_stream(void* cuda_stream);

/* Alg. 2 line 1: set up the problem of Def. "Sparse Tucker
 * Factorization".
 *  coords    host, nnz x order int32, row-major, 0-based; coords[e*order+n] in [0, dims[n])
 *  vals      host, nnz values; vals_dtype selects the context precision
 *  vals_dtype PTUCKER_F32 | PTUCKER_F64
 *  nnz       1 <= nnz <= INT32_MAX (duplicate coordinates are accepted: multiset,
 *            reading R14); EINVAL outside
 *  order     2 <= N <= 10
 *  dims      host, N int64, each 1 <= I_n <= INT32_MAX
 *  core_dims host, N int32, J_1..J_N (Alg. 2 input): each 1 <= J_n <= 16 and
 *            prod J_n <= 2^26 (EINVAL otherwise).  Compiled fast paths for equal J_n: N in
 *            2..5 with J in {2,3,4,5,8,10} (tensor cores for N = 3 fp32, and for order-4
 *            modes with one small other mode); unequal J_n and any other (N, J) run the
 *            generic kernel (update_generic.cu: delta by Eq. 12 as written).  Factors are
 *            I_n x J_n and the core J_1 x ... x J_N (C order) in every getter/setter
 *  lambda    > 0 (makes B + lambda I positive definite)
 *  seed      init RNG seed: G and every A^(n) ~ U[0,1) (reading R2)
 * Copies the COO to the device, draws the init, builds every mode's slice
 * index Omega^(n)_{i_n} on the device (stable radix sort -> CSR ->
 * length-sorted segments) and this rank's row blocks.  Replaces any previous
 * context's data (the communicator is kept). */
int ptucker_init(const int32_t* coords, const void* vals, int32_t vals_dtype, int64_t nnz, int32_t order,
                 const int64_t* dims, const int32_t* core_dims, double lambda, uint64_t seed);

/* Alg. 3 lines 6-15 for mode n (0-based): every row i of A^(n)
 * owned by this rank becomes a_i = c_i [B_i + lambda I]^-1 (Eq. 9-12,
 * P:536-552), with empty rows set to 0; then, when world > 1, the row blocks
 * are all-gathered so every rank holds the whole A^(n).  Stream-ordered:
 * returns after enqueueing. */
int ptucker_update_mode(int32_t n);

/* One full ALS iteration (Alg. 2 line 3: update A^(1..N) by Alg. 3):
 * ptucker_update_mode(0..N-1) in ascending order. */
int ptucker_sweep(void);

/* Eq. 5: sqrt of sum over Omega of (x - x_hat)^2 for the current
 * state, summed over ranks (host *out, synchronises).  After an update_mode it
 * uses the per-row identity sum x^2 - 2 a.c + a B a^T of the rows just solved
 * (fused); otherwise it runs the literal per-entry pass. */
int ptucker_error(double* out);
/* Same quantity, always by the literal per-entry pass (Eq. 4-5). */
int ptucker_error_literal(double* out);

/* Alg. 2 lines 8-11: for n = 1..N, A^(n) = Q^(n) R^(n) with
 * diag(R) > 0, A^(n) <- Q^(n), G <- G x_n R^(n) (Eq. 7-8).
 * Requires I_n >= J_n; a rank-deficient A^(n) gives PTUCKER_ENUMERIC. */
int ptucker_orthogonalize(void);

/* P-Tucker-Approx.  Partial reconstruction error of every core entry,
 * Eq. 13: R(beta) = sum over Omega of t_beta (-2 X + t_beta + 2 sum_{gamma!=beta}
 * t_gamma), t_gamma = G_gamma prod_n a^(n)_{i_n gamma_n}, for the current state, summed over
 * ranks.  out: host, prod J doubles in C order; NaN for entries already truncated.
 * Computed in fp64 (approx.cu); synchronises. */
int ptucker_core_scores(double* out);
/* Alg. 4 with readings R28/R29: scores as above, then the
 * floor(p * |G|) present entries with the largest R (ties: lower C-order index) are set to
 * zero and marked truncated, never leaving fewer than one; *removed (may be null) receives
 * the count.  p in (0, 1) else PTUCKER_EINVAL.  Alg. 2 runs it after each iteration's error
 * (P:500-502); the final ptucker_orthogonalize makes G dense again. */
int ptucker_truncate_core(double p, int64_t* removed);
/* Number of core entries not truncated (|G| of Alg. 4). */
int ptucker_core_nnz(int64_t* nnz);

/* Eq. 4, "predict values of missing entries": x_hat for n query
 * coordinates.  coords: host, n x N int32 (row-major, in range else PTUCKER_EINVAL);
 * out: host, n doubles.  fp64 over the dense core; synchronises. */
int ptucker_predict(const int32_t* coords, int64_t n, double* out);
/* Held-out test RMSE (§4.4): sqrt(sum (x - x_hat)^2 / n) over n test entries
 * (host coords n x N int32, host vals n of vals_dtype = the context's precision); n >= 1. */
int ptucker_test_rmse(const int32_t* coords, const void* vals, int32_t vals_dtype, int64_t n, double* out);

/* Alg. 2 from the current state: e_0 = error; repeat { ptucker_sweep (line 3);
 * e_t = error (line 4, Eq. 5); if approx_p > 0, ptucker_truncate_core(approx_p) (lines 5-6) }
 * until t == max_iters, |e_t - e_{t-1}| < tol * e_{t-1} or e_t <= tol * ||x|| (reading R30,
 * ||x|| = sqrt of the sum of squares of the observed values); then
 * ptucker_orthogonalize if `orthogonalize` (lines 8-11).  errors: host, max_iters + 1 doubles
 * (e_0 .. e_T, may be null); *iters = T (may be null).  tol >= 0, 0 <= approx_p < 1. */
int ptucker_run(int32_t max_iters, double tol, double approx_p, int32_t orthogonalize, double* errors,
                int32_t* iters);

/* State access (host buffers of exactly I_n*J_n or prod J elements, context precision). */
int ptucker_get_factor(int32_t n, void* out);
int ptucker_set_factor(int32_t n, const void* in);
int ptucker_get_core(void* out);
int ptucker_set_core(const void* in);

/* Test hook: mode n's slice index.  row_ptr: host, I_n+1 int64; perm: host,
 * nnz int64 (entry ids sorted by coordinate n, ties in input order). */
int ptucker_get_mode_index(int32_t n, int64_t* row_ptr, int64_t* perm);
/* This context's row blocks of mode n: host, world+1 int64. */
int ptucker_get_partition(int32_t n, int64_t* bounds);

/* Options (set after init unless noted):
 *  "policy"       precision of the fp32 contraction: -1 = automatic
 *                 (default: every outer TTV stage in fp64; F32-C2 for N = 5, J = 5), 0 = F32-A (all fp32), 1 = F32-B
 *                 (outermost stage fp64), 2 = F32-C (all outer stages fp64), 3 = F32-C2 (order 5:
 *                 every outer stage in fp64 but the innermost one's parent: J^3 instead of J^4
 *                 fp32 -> fp64 conversions per entry; other orders: as 2)
 *  "tc"           1 = order-3 fp32 updates run the innermost contraction on the tcgen05 tensor
 *                 cores (3xTF32, default); 0 = the all-ALU kernel
 *  "smp"          1 = small-mode precontraction where it applies (order 4, two other modes with
 *                 <= 64 rows whose table fits on chip; default), 0 = off
 *  "smp_table"    two-small-mode table for fp32 data: 0 = fp32 copy in shared memory, 1 = fp64
 *                 table read from L2, 2 = hybrid: fp64 for single-segment rows (default)
 *  "emulate_world", "emulate_rank"  (before init, no communicator): build and update only
 *                 this rank's row blocks of a `world`-way partition, without the exchange
 *                 (tests of the partitioned path on one GPU)
 *  "sparse_core"  P-Tucker-Approx on the generic path (after ptucker_truncate_core): -1 = the
 *                 delta runs over the coordinate list of the present core entries when its
 *                 N |G| operations per entry beat the dense J^(N-1) (J_n + N - 1) (default), 1 =
 *                 always when the core is truncated, 0 = dense.  Bit-identical results either way
 *  "cache"        1 = P-Tucker-Cache (Alg. 3 TOP branch; read by the next ptucker_init): a cache
 *                 table Pres of |Omega| x |G| fp64 products G_beta prod_k a^(k) (lines 1-4), delta
 *                 read from it (line 12; a factor value of exactly 0 takes the product loop,
 *                 P:639), the table rescaled by a_new / a_old after every mode (lines 16-19) and
 *                 rebuilt after set_factor / set_core / QR / truncation.  Runs on the generic
 *                 path; ERESOURCE at init when |Omega| |G| 8 bytes exceed 80% of free device
 *                 memory (c1: 10 MB, c2: 8 GB; c3-c5 do not fit).  0 = P-Tucker (default)
 *  "exchange"     multi-GPU replica refresh: 1 = push from the kernels when peers are open
 *                 (default), 0 = NCCL all-gather-v (grouped broadcasts) after each mode
 *  "graph"        1 = ptucker_sweep records its launches once as a CUDA graph and replays it
 *                 (default); the graph is dropped by any option change, init, finalize,
 *                 QR and ptucker_open_peers; not used while time_kernels is on.  0 = direct
 *  "pdl"          1 = programmatic dependent launch: the tensor-core update, the heavy-row
 *                 finalize and the error-sum kernels are launched with programmatic stream
 *                 serialization, so each one's CTAs start (TMEM allocation, barrier setup) on
 *                 the SMs its predecessor vacates and wait in griddepcontrol.wait for the
 *                 predecessor's results; bit-identical results, but measured slower under
 *                 the sweep's CUDA graph (c2 0.26 -> 0.37 ms per iteration, c1 and c5
 *                 unchanged).  Process-wide (all contexts).  0 = plain stream order (default)
 *  "seg_len"      segment length S of the index (before init): -1 = automatic (default: the
 *                 power of two >= |Omega| / (SMs x 128) in [8, 256]), else 1..2^20
 *  "time_kernels" 1 = bracket every kernel launch with CUDA events (ptucker_kernel_stats)
 *  "fin_inline"   1 = rows cut into 2..64 segments (heavy rows) are solved inside the
 *                 tensor-core / ALU / table update kernels by the lane that stores the row's
 *                 last partial (same additions, same bits as the finalize launch); measured
 *                 slower (c1 0.10 -> 0.19, c2 0.33 -> 0.38 ms per iteration: one lane's serial
 *                 sum and solve lengthen the kernel's tail).  0 = a separate finalize launch
 *                 (default).  Modes with longer rows, the SMP and the generic kernels always
 *                 use the finalize launch
 *  "l0_group"     tensor-core kernel, F32-B: level-0 terms summed in fp32 in runs of g before
 *                 the fp64 sum (1 = every term in fp64, default; 2; 5 fails the 1e-5 row bound;
 *                 0 = packed fp32 pairs with Kahan compensation, even J: worst full-size c5 row
 *                 5.8e-6, no faster)
 *  "l2_persist_mb" L2 set-aside (MB) for the evict_last factor-row gathers: -1 = the device
 *                 maximum (default; applied at init, released by ptucker_finalize), 0 = leave
 *                 the driver default.  Side effect: cudaLimitPersistingL2CacheSize is a
 *                 process-wide (context) limit, so other work in the same process (torch)
 *                 runs with that much less normal L2 while the context lives, and
 *                 ptucker_finalize calls cudaCtxResetPersistingL2Cache, which also resets
 *                 lines other code marked persisting
 *  "tc_table"     1 = order-4 fp32 modes with one small other mode run the tensor-core kernel on
 *                 the per-i_s core blocks (default; set BEFORE init: it orders the index); 0 = ALU
 *  "rows_l1"      tensor-core gathers of factor rows: -1 = through L1 when a gathered mode has a
 *                 row with >= 1% of the entries (default, automatic), 1 = always, 0 = L2 only
 *  "pack_gathers" 1 = J = 10 tensor-core updates gather from packed 40-byte row tables (DRAM
 *                 reads 5.1 -> 2.1 GB per c5 update, ~10% slower); 0 = the factors (default)
 *  "trace"        1 = per-phase clock marks of the tensor-core kernel (builds with -DPT_TRACE) */
int ptucker_set_option(const char* key, int64_t value);

/* Device time (CUDA events on the library stream) accumulated for kernel
 * `name` ("update", "finalize", "sse_reduce", "allgather", ...) since the last
 * reset, with the launch count; synchronises. */
int ptucker_kernel_stats(const char* name, double* total_ms, int64_t* launches);
int ptucker_reset_kernel_stats(void);

/* JSON description of the context (sizes, segments, kernel variant); host buffer. */
int ptucker_info(char* buf, int32_t len);

/* Tools only: copy the per-phase clock trace recorded while option "trace" is on
 * (host buffer of n int64; layout documented in tools/trace_tc.py). */
int ptucker_debug_trace(long long* out, int32_t n);

/* Wait for all enqueued work; reports deferred numeric failures. */
int ptucker_synchronize(void);

/* Free all device memory and the communicator. */
int ptucker_finalize(void);

#ifdef __cplusplus
}
#endif
#endif /* PTUCKER_H */
