// abi.cu -- the C-ABI (include/ptucker.h): context, validation, orchestration of
// the kernels per call, NCCL exchange between ranks, state access.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/ptucker.h"
#include "index.cuh"
#include "internal.cuh"
#include "kernels.cuh"

namespace pt {

const UpdateKernel* find_update_kernel(int prec, int l64, int N, int J) {
    int cnt = 0;
    if (prec == PTUCKER_F32 && N <= 3 && l64 > 1) l64 = 1;  // N = 3 has a single outer level
    const UpdateKernel* t = prec == PTUCKER_F64 ? update_kernels_f64(&cnt)
                            : (l64 == 0 ? update_kernels_f32a(&cnt)
                                        : (l64 == 1 ? update_kernels_f32b(&cnt)
                                                    : (N == 5 && l64 == 2 ? update_kernels_f32c2(&cnt)
                                                                          : update_kernels_f32c(&cnt))));
    for (int i = 0; i < cnt; ++i)
        if (t[i].N == N && t[i].J == J) return &t[i];
    return nullptr;
}

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) {                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? PTUCKER_ERESOURCE : PTUCKER_ECUDA,        \
                        "%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));           \
        }                                                                                           \
    } while (0)

#define NK(x)                                                                                    \
    do {                                                                                         \
        ncclResult_t r_ = (x);                                                                   \
        if (r_ != ncclSuccess)                                                                   \
            return fail(PTUCKER_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #x, ncclGetErrorString(r_)); \
    } while (0)

struct Pending {
    std::string name;
    int mode;
    cudaEvent_t a, b;
};

struct Ctx {
    bool inited = false;
    int device = -1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    int emu_rank = 0, emu_world = 1;  // options "emulate_rank"/"emulate_world": partition without a communicator
    // problem
    int N = 0, J = 0, prec = 0, esz = 4;  // J: max_n J_n (equal J_n: the J of the compiled paths)
    JDims Jv;                             // J_1..J_N (unequal J_n run the generic path)
    bool ujn = false;                     // unequal J_n
    int64_t nnz = 0;
    int64_t dims[kMaxN] = {0};
    double xnorm = 0.0;  // sqrt(sum x^2) over Omega (convergence floor of ptucker_run)
    double lambda = 0.0;
    uint64_t seed = 0;
    int lda = 0, gp_elems = 0;
    int policy = -1;    // -1 = automatic per order; else outer fp64 levels
    int seg_len = -1;       // option "seg_len" (S); -1 = automatic (resolve_seg_len)
    int seg_len_eff = 256;  // the S of the current index
    DeviceArena arena, scratch;
    void* A[kMaxN] = {nullptr};
    void* G = nullptr;
    void* Gtmp = nullptr;
    void* Gp[kMaxN] = {nullptr};
    ModeIndex mi[kMaxN];
    double* sse_row[kMaxN] = {nullptr};
    double* lit_part = nullptr;
    double* red_part = nullptr;  // 256
    double* red_out = nullptr;   // 4
    double* qr = nullptr;        // W, W2, R1, R2, R (J*J each) + gram partials (256*NB)
    double* qd = nullptr;        // I_max x J fp64 scratch for CholeskyQR2 (lazy)
    int* d_fail = nullptr;       // row + 1 of a failed solve
    int* d_qrfail = nullptr;     // mode + 1 of a failed QR
    unsigned int* d_work = nullptr;
    int sse_mode = -1;           // mode whose per-row SSE describes the current state
    int last_fail_mode = -1;
    const UpdateKernel* kern = nullptr;      // row update (tensor-core variant when available)
    const UpdateKernel* kern_alu = nullptr;  // ALU kernel (literal error pass, and updates when tc = 0)
    bool generic = false;                    // no compiled (N, J): update_generic.cu + device COO for the error
    int32_t* coo_c = nullptr;                // generic shapes: the input COO kept on the device
    void* coo_v = nullptr;
    int use_tc = 1;                          // option "tc"
    int l0_group = 1;                        // option "l0_group" (tensor-core kernel, F32-B)
    int fin_inline = 0;                      // option "fin_inline": heavy rows (<= 64 segments) solved in the update kernel
    bool inline_used = false;                // the last update launch finished its heavy rows itself
    int64_t l2_persist_mb = -1;              // option "l2_persist_mb": L2 set-aside for evict_last lines (-1 = max)
    int pack_gathers = 0;                    // option "pack_gathers": J = 10 tensor-core gathers from packed tables
    int rows_l1[kMaxN] = {0};                // per updated mode: gather rows through L1 (skewed other modes)
    int rows_l1_opt = -1;                    // option "rows_l1": -1 = automatic (row skew), 0 / 1 = forced
    int tc_table = 1;                        // option "tc_table": order-4 one-small-mode tables on the tensor cores
    float* pk_head[2] = {nullptr, nullptr};  // tensor-core kernel, J = 10: packed gather tables
    float* pk_tail[2] = {nullptr, nullptr};
    int use_smp = 1;                         // option "smp"
    int smp_tab = 2;                         // option "smp_table": 0 fp32 smem, 1 fp64 L2, 2 hybrid (default)
    struct Smp {
        int kind = 0;                        // 2: order-4 mode with two small other modes (smp.cu)
        int r = 0, s1 = 0, s2 = 0;           // global mode ids
        int ir = 0, is1 = 0, is2 = 0;        // ordinals among the other modes (SELL/param order)
        int64_t elems = 0;                   // table elements
    } smp[kMaxN];
    void* smp_T = nullptr;                   // device table (largest over modes), fp64
    void* smp_T32 = nullptr;                 // fp32 copy of a kind-2 table
    // P-Tucker-Approx (approx.cu): presence of the core entries (C order) and lazy scratch
    uint8_t* d_present = nullptr;            // [J^N] core entries not truncated (Alg. 4), device
    int64_t n_present = 0;                   // their count (host bookkeeping of the truncation)
    double* ax_R = nullptr;                  // [J^N] scores R(beta)
    uint64_t *ax_key = nullptr, *ax_key2 = nullptr;  // selection sort keys (in/out)
    int64_t *ax_idx = nullptr, *ax_idx2 = nullptr;   // selection sort values (in/out)
    void* ax_tmp = nullptr;
    size_t ax_tmp_bytes = 0;
    double *ax_G64 = nullptr, *ax_A0 = nullptr, *ax_W = nullptr, *ax_W2 = nullptr, *ax_E = nullptr,
           *ax_part = nullptr, *ax_UV = nullptr;
    void** ax_ptrs = nullptr;  // device: sc[0..N-2] of mode 0, then A[0..N-1]
    // multi-GPU push exchange (ptucker_open_peers): the other ranks' replicas of every A^(n)
    void* peer_A[kMaxN][kMaxPeers] = {{nullptr}};
    int npeer = 0;
    int exchange = 1;            // option "exchange": 1 = push when peers are open, 0 = NCCL all-gather-v
    int* d_barrier = nullptr;    // 1 int: the NCCL all-reduce that orders the pushes before the next mode
    int nsm = 148;
    int grid_upd = 0, grid_lit = 0;
    int64_t launches = 0;        // kernels this library launched since init (gpu_launches evidence)
    long long* trace = nullptr;  // option "trace": device buffer of per-phase clocks (tools/)
    // P-Tucker-Cache (option "cache", before init): the cache table Pres (|Omega| x |G| fp64)
    int use_cache = 0;             // the option (read by ptucker_init)
    bool cache_on = false;         // this context runs P-Tucker-Cache
    double* pres = nullptr;
    void* cache_old = nullptr;     // A^(n) before its update (lines 16-19 divide by it)
    void** cache_ptrs = nullptr;   // device: A[0..N-1]
    bool pres_stale = false;       // factors / core changed outside the ALS sweep: rebuild Pres
    // P-Tucker-Approx on the generic path: coordinate list of the present core entries (C
    // order) for the sparse-core delta (option "sparse_core": -1 auto, 0 dense, 1 sparse)
    int sparse_core = -1;
    uint64_t* sp_digits = nullptr;  // [N][|G|] per mode, ordered by (t mod 32, C order), t = the
    int64_t* sp_index = nullptr;    //   entry's index over the other modes (update_generic.cu)
    int32_t* sp_off = nullptr;      // [N][33] each lane's range
    int64_t sp_n = -1;             // -1: no list (the core is dense)
    // CUDA graph of a whole sweep (option "graph"): captured at the first ptucker_sweep
    // and replayed while the launch parameters stay valid (invalidate_graph)
    int use_graph = 1;
    cudaGraphExec_t graph_exec = nullptr;
    int64_t graph_launches = 0;  // kernels in the captured sweep
    // timing
    bool time_kernels = false;
    std::vector<Pending> pending;
    std::map<std::string, std::pair<double, int64_t>> stats;
};

Ctx g;
double g_xnorm_pending = 0.0;

void close_peers() {
    for (int n = 0; n < kMaxN; ++n)
        for (int r = 0; r < kMaxPeers; ++r) {
            if (g.peer_A[n][r]) cudaIpcCloseMemHandle(g.peer_A[n][r]);
            g.peer_A[n][r] = nullptr;
        }
    g.npeer = 0;
}

bool pushing() { return g.npeer > 0 && g.exchange == 1; }

// A captured sweep bakes in pointers (G for the small-mode tables, the packed gather tables,
// the peer replicas) and the kernel choice: any option change, init, finalize, QR (which
// swaps G) or a new peer set drops it.
void invalidate_graph() {
    if (g.graph_exec) cudaGraphExecDestroy(g.graph_exec);
    g.graph_exec = nullptr;
}


cudaStream_t S() { return g.stream; }

template <class F>
int timed(const char* name, F&& f, int mode = -1) {
    if (!g.time_kernels) return f();
    Pending p;
    p.name = name;
    p.mode = mode;
    CK(cudaEventCreate(&p.a));
    CK(cudaEventCreate(&p.b));
    CK(cudaEventRecord(p.a, S()));
    const int rc = f();
    CK(cudaEventRecord(p.b, S()));
    g.pending.push_back(p);
    return rc;
}

int fold_stats() {
    for (auto& p : g.pending) {
        CK(cudaEventSynchronize(p.b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p.a, p.b));
        auto& s = g.stats[p.name];
        s.first += ms;
        s.second += 1;
        if (p.mode >= 0) {
            auto& sm = g.stats[p.name + "_m" + std::to_string(p.mode)];
            sm.first += ms;
            sm.second += 1;
        }
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g.pending.clear();
    return PTUCKER_OK;
}

int check_fail_flags() {
    int h[2] = {0, 0};
    CK(cudaMemcpyAsync(&h[0], g.d_fail, sizeof(int), cudaMemcpyDeviceToHost, S()));
    CK(cudaMemcpyAsync(&h[1], g.d_qrfail, sizeof(int), cudaMemcpyDeviceToHost, S()));
    CK(cudaStreamSynchronize(S()));
    if (h[0] != 0) {
        CK(cudaMemsetAsync(g.d_fail, 0, sizeof(int), S()));
        CK(cudaStreamSynchronize(S()));
        return fail(PTUCKER_ENUMERIC, "non-positive pivot in the row solve of mode %d, row %d", g.last_fail_mode,
                    h[0] - 1);
    }
    if (h[1] != 0) {
        CK(cudaMemsetAsync(g.d_qrfail, 0, sizeof(int), S()));
        CK(cudaStreamSynchronize(S()));
        return fail(PTUCKER_ENUMERIC, "rank-deficient factor A^(%d) in QR", h[1] - 1);
    }
    return PTUCKER_OK;
}

int sync_and_check() {
    CK(cudaStreamSynchronize(S()));
    CK(cudaGetLastError());
    return check_fail_flags();
}

int require_init() {
    if (!g.inited) return fail(PTUCKER_ESTATE, "ptucker_init has not been called");
    int dev = -1;
    CK(cudaGetDevice(&dev));
    if (dev != g.device) CK(cudaSetDevice(g.device));
    return PTUCKER_OK;
}

template <typename TS>
UpdateParams<TS> make_params(int n, bool literal) {
    UpdateParams<TS> p;
    memset(&p, 0, sizeof(p));
    const ModeIndex& m = g.mi[n];
    p.n = n;
    p.nslices = m.nslices;
    p.slice_off = m.slice_off;
    p.slice_len = m.slice_len;
    p.lane_row = m.lane_row;
    p.lane_len = m.lane_len;
    p.lane_pidx = m.lane_pidx;
    p.lane_pstride = m.lane_pstride;
    p.lane_aux = m.lane_aux;
    int l = 0;
    for (int k = 0; k < g.N; ++k) {
        if (k == n) continue;
        p.sc[l] = m.sc[l];
        p.A[l] = (const TS*)g.A[k];
        p.dim_other[l] = g.dims[k];
        ++l;
    }
    p.sv = (const TS*)m.sv;
    p.An = (TS*)g.A[n];
    p.dim_n = g.dims[n];
    p.lda = g.lda;
    p.Gp = (const TS*)g.Gp[n];
    p.gp_elems = g.gp_elems;
    p.lambda = g.lambda;
    p.partials = m.partials;
    p.sse_row = g.sse_row[n];
    p.lit_part = literal ? g.lit_part : nullptr;
    p.fail = g.d_fail;
    p.work = g.d_work;
    p.policy = g.policy;
    p.trace = g.trace;
    p.gmain[0] = g.pk_head[0];
    p.gmain[1] = g.pk_head[1];
    p.gtail[0] = g.pk_tail[0];
    p.gtail[1] = g.pk_tail[1];
    p.l0_group = g.l0_group;
    p.rows_l1 = g.rows_l1[n];
    if (!literal && g.fin_inline && m.nheavy > 0 && m.hmaxseg <= 64) {
        // (pointers offset by the block's first row: the kernels index them by global row)
        p.seg_done = m.seg_done - m.hr0;
        p.row_pbase = m.row_pbase - m.hr0;
    }
    if (pushing()) {
        p.peers.n = g.npeer;
        for (int r = 0; r < g.npeer; ++r) p.peers.base[r] = g.peer_A[n][r];
    }
    return p;
}

int launch_update_kernel(int n, bool literal) {
    const int grid = literal ? g.grid_lit : g.grid_upd;
    g.inline_used = false;
    if (g.mi[n].nslices == 0) return PTUCKER_OK;
    const Ctx::Smp& sp = g.smp[n];
    // the dynamic slice counter of the ALU / SMP kernels; the tensor-core kernel schedules
    // statically, and without the memset between it and the previous kernel its launch keeps
    // the programmatic (PDL) edge
    const bool smp2 = !literal && g.use_smp && sp.kind == 2 &&
                      !(g.prec == PTUCKER_F32 && g.smp_tab != 1 && sp.elems * 4 > 200 * 1024);
    const bool tc_main = !literal && !g.generic && !(g.use_smp && sp.kind == 1) && !smp2 && g.kern != g.kern_alu;
    const bool tc_table = !literal && !smp2 && g.use_smp && sp.kind == 1 && g.mi[n].aux_groups && g.use_tc &&
                          g.prec != PTUCKER_F64 && find_update_kernel_tc(1, g.J) != nullptr;
    if (!tc_main && !tc_table) CK(cudaMemsetAsync(g.d_work, 0, sizeof(unsigned int), S()));
    if (smp2) {
        // small-mode precontraction: T from the (unchanged) small-mode factors, then J^2 per entry
        const int mode = g.prec == PTUCKER_F64 ? 1 : g.smp_tab;
        launch_smp_table2(g.G, g.A[sp.s1], g.A[sp.s2], g.lda, g.dims[sp.s1], g.dims[sp.s2], g.J, n, sp.r, sp.s1, sp.s2,
                          (double*)g.smp_T, mode == 1 ? nullptr : g.smp_T32, g.esz, S());
        bool ok;
        if (g.prec == PTUCKER_F64) {
            UpdateParams<double> p = make_params<double>(n, false);
            p.seg_done = nullptr;  // (the SMP kernel leaves its heavy rows to the finalize launch)
            ok = launch_smp2_update(&p, 8, g.J, (const double*)g.smp_T, nullptr, sp.elems, sp.ir, sp.is1, sp.is2,
                                    (int)g.dims[sp.s2], 1, g.nsm, S());
        } else {
            UpdateParams<float> p = make_params<float>(n, false);
            p.seg_done = nullptr;
            ok = launch_smp2_update(&p, 4, g.J, (const double*)g.smp_T, g.smp_T32, sp.elems, sp.ir, sp.is1, sp.is2,
                                    (int)g.dims[sp.s2], mode, g.nsm, S());
        }
        if (!ok) return fail(PTUCKER_EINVAL, "no SMP kernel for J=%d", g.J);
        g.launches += 2;
        CK(cudaGetLastError());
        return PTUCKER_OK;
    }
    if (!literal && g.use_smp && sp.kind == 1) {
        // one small mode: table of order-3 cores T[i_s], then an order-3 TTV per entry
        launch_smp_table1(g.G, g.A[sp.s1], g.lda, g.dims[sp.s1], g.J, n, sp.r, sp.s2, sp.s1, g.smp_T, g.esz, S());
        const int GBk = gblk(g.J, g.esz);
        bool ok;
        auto fill = [&](auto& p) {
            using TSp = typename std::remove_const<typename std::remove_pointer<decltype(p.sv)>::type>::type;
            p.sc[0] = g.mi[n].sc[sp.ir];
            p.sc[1] = g.mi[n].sc[sp.is2];
            p.A[0] = (const TSp*)g.A[sp.r];
            p.A[1] = (const TSp*)g.A[sp.s2];
            p.dim_other[0] = g.dims[sp.r];
            p.dim_other[1] = g.dims[sp.s2];
            p.Gp = (const TSp*)g.smp_T;
            p.gp_elems = (int)sp.elems;
            p.aux_stride = (int64_t)g.J * GBk;
        };
        // the lanes of an aux-grouped index are in (i_s, length) order, which the ALU table
        // kernel also accepts (it reads lane_aux per lane): option tc = 0 takes that kernel
        const UpdateKernel* ktc = g.mi[n].aux_groups && g.use_tc ? find_update_kernel_tc(1, g.J) : nullptr;
        if (g.prec == PTUCKER_F64) {
            UpdateParams<double> p = make_params<double>(n, false);
            fill(p);
            g.inline_used = p.seg_done != nullptr;
            ok = launch_table_update(&p, 8, g.J, g.nsm, S());
        } else if (ktc) {  // tensor-core kernel with the group's table block as the core
            UpdateParams<float> p = make_params<float>(n, false);
            fill(p);
            p.gmain[0] = p.gmain[1] = p.gtail[0] = p.gtail[1] = nullptr;
            g.inline_used = p.seg_done != nullptr;
            ktc->launch(&p, false, g.nsm, S());
            ok = true;
        } else {
            UpdateParams<float> p = make_params<float>(n, false);
            fill(p);
            g.inline_used = p.seg_done != nullptr;
            ok = launch_table_update(&p, 4, g.J, g.nsm, S());
        }
        if (!ok) return fail(PTUCKER_EINVAL, "no table kernel for J=%d", g.J);
        g.launches += 2;
        CK(cudaGetLastError());
        return PTUCKER_OK;
    }
    g.launches += 1;
    if (g.generic) {
        if (literal) return fail(PTUCKER_EINVAL, "internal: no literal pass for generic shapes");
        if (g.cache_on) {
            if (g.pres_stale) {  // factors or core were set / orthogonalized / truncated: lines 1-4 again
                launch_pres_init(g.N, g.Jv, g.esz, g.G, (const void* const*)g.cache_ptrs, g.lda, g.coo_c, g.nnz,
                                 g.pres, S());
                g.pres_stale = false;
                g.launches += 1;
            }
            // a_old of lines 16-19
            CK(cudaMemcpyAsync(g.cache_old, g.A[n], (size_t)g.dims[n] * g.lda * g.esz, cudaMemcpyDeviceToDevice, S()));
        }
        const double* pres = g.cache_on ? g.pres : nullptr;
        // sparse-core delta (truncated core): when its O(N |G|) beats the dense J^(N-1) (J_n + N - 1)
        bool sparse = false;
        if (!pres && g.sp_n >= 0 && g.sparse_core != 0) {
            double dense = (double)(g.Jv.j[n] + g.N - 1);
            for (int m = 0; m < g.N; ++m)
                if (m != n) dense *= g.Jv.j[m];
            sparse = g.sparse_core == 1 || (double)g.sp_n * g.N < dense;
        }
        int64_t gsz = 1;
        for (int m = 0; m < g.N; ++m) gsz *= g.Jv.j[m];
        const uint64_t* spd = sparse ? g.sp_digits + (int64_t)n * gsz : nullptr;
        const int64_t* spi = sparse ? g.sp_index + (int64_t)n * gsz : nullptr;
        const int32_t* spo = sparse ? g.sp_off + n * 33 : nullptr;
        if (g.prec == PTUCKER_F64) {
            UpdateParams<double> p = make_params<double>(n, false);
            p.Gp = (const double*)g.G;
            p.seg_done = nullptr;  // (the generic kernel leaves its heavy rows to the finalize launch)
            launch_update_generic(&p, 8, g.N, g.Jv, g.nsm, S(), pres, g.mi[n].sid, spd, spi, spo);
        } else {
            UpdateParams<float> p = make_params<float>(n, false);
            p.Gp = (const float*)g.G;
            p.seg_done = nullptr;
            launch_update_generic(&p, 4, g.N, g.Jv, g.nsm, S(), pres, g.mi[n].sid, spd, spi, spo);
        }
        CK(cudaGetLastError());
        return PTUCKER_OK;
    }
    const UpdateKernel* k = literal ? g.kern_alu : g.kern;

    if (g.prec == PTUCKER_F64) {
        UpdateParams<double> p = make_params<double>(n, literal);
        g.inline_used = p.seg_done != nullptr;
        k->launch(&p, literal, grid, S());
    } else {
        const bool packed = g.pack_gathers && !literal && k != g.kern_alu && g.J == 10;
        if (packed) {  // tensor-core kernel: pack the two gathered factors (L2-resident gathers)
            if (!g.pk_head[0]) {
                int64_t imax = 0;
                for (int m = 0; m < g.N; ++m) imax = std::max<int64_t>(imax, g.dims[m]);
                for (int t = 0; t < 2; ++t) {
                    CK(g.arena.alloc((void**)&g.pk_head[t], (size_t)imax * 8 * sizeof(float)));
                    CK(g.arena.alloc((void**)&g.pk_tail[t], (size_t)imax * 2 * sizeof(float)));
                }
            }
            int t = 0;
            for (int m = 0; m < g.N; ++m) {
                if (m == n) continue;
                launch_pack_rows10((const float*)g.A[m], g.dims[m], g.lda, g.pk_head[t], g.pk_tail[t], S());
                ++t;
            }
            g.launches += 2;
        }
        UpdateParams<float> p = make_params<float>(n, literal);
        if (!packed) p.gmain[0] = p.gmain[1] = p.gtail[0] = p.gtail[1] = nullptr;
        g.inline_used = p.seg_done != nullptr;
        k->launch(&p, literal, grid, S());
    }
    CK(cudaGetLastError());
    return PTUCKER_OK;
}

int rebuild_gp() {
    if (g.generic) return PTUCKER_OK;
    for (int n = 0; n < g.N; ++n) launch_permute_core(g.G, g.Gp[n], g.esz, g.N, g.J, n, S());
    g.launches += g.N;
    CK(cudaGetLastError());
    return PTUCKER_OK;
}

// outer TTV levels in fp64 for the current policy.  auto = every outer level
// (F32-B for N = 3, F32-C for N >= 4): the one-level F32-B and the all-fp32
// F32-A both exceed the 1e-5 row bound on measured configs.
int policy_l64() {
    if (g.prec == PTUCKER_F64) return 1;
    const int all = g.N >= 4 ? g.N - 2 : 1;
    if (g.policy == 3) return g.N >= 5 ? g.N - 3 : all;  // F32-C2 (order 5): all outer levels but the innermost's parent
    if (g.policy >= 0) return g.policy == 2 ? all : g.policy;
    // automatic: order 5 with J = 5 (c4) takes F32-C2 -- J^3 instead of J^4 fp32 -> fp64
    // conversions per entry, worst full-size row 2.5e-6 of the 1e-5 bound (F32-C: 1.1e-6),
    // 2.60 against 2.74 ms per mode once its core reads go through the uniform datapath
    // (profiles/r02/ab_c4_f32c2.txt); other order-5 J keep F32-C (no full-size evidence)
    if (g.N == 5 && g.J == 5) return g.N - 3;
    return all;
}

int choose_kernel() {
    const int last64 = policy_l64();
    int nsm0 = 148;
    CK(cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, g.device));
    if (g.generic) {  // update_generic.cu
        g.kern = g.kern_alu = nullptr;
        g.nsm = nsm0;
        g.grid_upd = g.grid_lit = nsm0;
        return PTUCKER_OK;
    }
    g.kern_alu = find_update_kernel(g.prec, last64, g.N, g.J);
    if (!g.kern_alu) return fail(PTUCKER_EINVAL, "no compiled kernel for N=%d J=%d", g.N, g.J);
    g.kern = g.kern_alu;
    if (g.use_tc && g.prec == PTUCKER_F32 && g.N == 3) {
        const UpdateKernel* k = find_update_kernel_tc(last64, g.J);
        if (k) g.kern = k;
    }
    int nsm = 148;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g.device));
    g.nsm = nsm;
    const size_t smem = ((size_t)g.gp_elems * g.esz + 15) / 16 * 16;  // + staging ring (added per kernel)
    int occ = g.kern->occupancy(false, smem);
    int occl = g.kern_alu->occupancy(true, smem);
    CK(cudaGetLastError());
    if (occ < 1 || occl < 1) return fail(PTUCKER_ERESOURCE, "update kernel does not fit on an SM (smem %zu B)", smem);
    g.grid_upd = nsm * occ;
    g.grid_lit = nsm * occl;
    return PTUCKER_OK;
}

void free_all() {
    invalidate_graph();
    close_peers();
    g.d_barrier = nullptr;
    g.arena.release_all();
    g.scratch.release_all();
    g.scratch.free_chunks();
    for (int n = 0; n < kMaxN; ++n) {
        g.mi[n] = ModeIndex();
        g.A[n] = nullptr;
        g.Gp[n] = nullptr;
        g.sse_row[n] = nullptr;
    }
    g.G = g.Gtmp = nullptr;
    g.smp_T = nullptr;
    g.smp_T32 = nullptr;
    g.pk_head[0] = g.pk_head[1] = g.pk_tail[0] = g.pk_tail[1] = nullptr;
    for (int n = 0; n < kMaxN; ++n) g.rows_l1[n] = 0;
    g.lit_part = g.red_part = g.red_out = g.qr = g.qd = nullptr;
    g.ax_G64 = g.ax_A0 = g.ax_W = g.ax_W2 = g.ax_E = g.ax_part = g.ax_UV = nullptr;
    g.ax_ptrs = nullptr;
    g.d_present = nullptr;
    g.n_present = 0;
    g.ax_R = nullptr;
    g.ax_key = g.ax_key2 = nullptr;
    g.ax_idx = g.ax_idx2 = nullptr;
    g.ax_tmp = nullptr;
    g.ax_tmp_bytes = 0;
    g.coo_c = nullptr;
    g.coo_v = nullptr;
    g.pres = nullptr;
    g.cache_old = nullptr;
    g.cache_ptrs = nullptr;
    g.pres_stale = false;
    g.cache_on = false;
    g.sp_digits = nullptr;
    g.sp_index = nullptr;
    g.sp_off = nullptr;
    g.sp_n = -1;
    g.generic = false;
    g.d_fail = g.d_qrfail = nullptr;
    g.d_work = nullptr;
    g.launches = 0;
    g.inited = false;
    g.sse_mode = -1;
}

void partition_rows(const int64_t* row_ptr, int64_t I, int world, int64_t* bounds) {
    const int64_t nnz = row_ptr[I];
    bounds[0] = 0;
    for (int w = 1; w < world; ++w) {
        const int64_t target = (w * nnz + world - 1) / world;
        bounds[w] = std::lower_bound(row_ptr, row_ptr + I + 1, target) - row_ptr;
        if (bounds[w] > I) bounds[w] = I;
    }
    bounds[world] = I;
}

}  // namespace
}  // namespace pt

using namespace pt;

extern "C" {

int32_t ptucker_version(void) { return 100; }

const char* ptucker_last_error(void) { return g_err.c_str(); }

int ptucker_get_unique_id(uint8_t out[128]) {
    if (!out) return fail(PTUCKER_EINVAL, "null id buffer");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return PTUCKER_OK;
}

int ptucker_comm_init(int32_t rank, int32_t world, const uint8_t id[128]) {
    if (world < 1 || rank < 0 || rank >= world) return fail(PTUCKER_EINVAL, "bad rank/world %d/%d", rank, world);
    // the row blocks of every mode (m.bounds, the SELL index of this rank) are fixed by
    // ptucker_init for the world it saw: a communicator must come first
    if (g.inited) return fail(PTUCKER_ESTATE, "ptucker_comm_init must precede ptucker_init (or follow ptucker_finalize)");
    if (g.comm) {
        ncclCommDestroy(g.comm);
        g.comm = nullptr;
    }
    g.rank = rank;
    g.world = world;
    if (world > 1) {
        if (!id) return fail(PTUCKER_EINVAL, "null id");
        ncclUniqueId uid;
        memcpy(&uid, id, 128);
        NK(ncclCommInitRank(&g.comm, world, uid, rank));
    }
    return PTUCKER_OK;
}

int ptucker_partition_rows(const int64_t* row_ptr, int64_t I, int32_t world, int64_t* bounds) {
    if (!row_ptr || !bounds || I < 0 || world < 1) return fail(PTUCKER_EINVAL, "bad partition arguments");
    partition_rows(row_ptr, I, world, bounds);
    return PTUCKER_OK;
}

int ptucker_set_stream(void* cuda_stream) {
    if (g.own_stream && g.stream) cudaStreamDestroy(g.stream);
    g.own_stream = false;
    g.stream = (cudaStream_t)cuda_stream;
    if (!g.stream) {
        CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
        g.own_stream = true;
    }
    return PTUCKER_OK;
}

// L2 set-aside for lines accessed with the evict_last policy (the factor-row gathers of
// the tensor-core kernel, reused across the entries of a mode update): with the device
// maximum (79 MB on B200) a c5 update reads 5.1 GB from DRAM instead of 8.0 GB
// (profiles/r01/l2_persist_c5.txt); 0 leaves the driver default.
int apply_l2_persist() {
    if (g.l2_persist_mb == 0) return PTUCKER_OK;
    int mx = 0;
    CK(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, g.device));
    const size_t want =
        g.l2_persist_mb < 0 ? (size_t)mx : std::min<size_t>((size_t)g.l2_persist_mb << 20, (size_t)mx);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
    return PTUCKER_OK;
}

// Factor-row gathers of mode n's update through L1 when a gathered (other) mode is
// skewed: its most frequent row holds >= 1% of the entries (a Zipf head row), so one L2
// slice would serve a large share of all gathers; uniform modes keep the L2-only path.
int rows_l1_auto(int n) {
    if (g.rows_l1_opt >= 0) return g.rows_l1_opt;
    if (!g.inited && g.mi[0].h_row_ptr.empty()) return 0;
    for (int m = 0; m < g.N; ++m) {
        if (m == n) continue;
        const std::vector<int64_t>& rp = g.mi[m].h_row_ptr;
        int64_t mx = 0;
        for (size_t i = 0; i + 1 < rp.size(); ++i) mx = std::max<int64_t>(mx, rp[i + 1] - rp[i]);
        if (g.nnz > 0 && mx * 100 >= g.nnz) return 1;
    }
    return 0;
}

int ptucker_set_option(const char* key, int64_t value) {
    if (!key) return fail(PTUCKER_EINVAL, "null key");
    const std::string k = key;
    invalidate_graph();
    if (k == "pdl") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "pdl must be 0 or 1");
        g_pdl = (int)value;
        return PTUCKER_OK;
    }
    if (k == "graph") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "graph must be 0 or 1");
        g.use_graph = (int)value;
        return PTUCKER_OK;
    }
    if (k == "policy") {
        if (value < -1 || value > 3) return fail(PTUCKER_EINVAL, "policy must be -1 (auto), 0, 1, 2 or 3");
        g.policy = (int)value;
        if (g.inited) return choose_kernel();
        return PTUCKER_OK;
    }
    if (k == "seg_len") {
        if (value != -1 && (value < 1 || value > (1 << 20))) return fail(PTUCKER_EINVAL, "seg_len out of range");
        if (g.inited) return fail(PTUCKER_ESTATE, "seg_len must be set before ptucker_init");
        g.seg_len = (int)value;
        return PTUCKER_OK;
    }
    if (k == "tc_table") {
        if (g.inited) return fail(PTUCKER_ESTATE, "tc_table must be set before ptucker_init");
        g.tc_table = value != 0;
        return PTUCKER_OK;
    }
    if (k == "rows_l1") {
        if (value < -1 || value > 1) return fail(PTUCKER_EINVAL, "rows_l1 must be -1, 0 or 1");
        g.rows_l1_opt = (int)value;
        for (int n = 0; n < g.N; ++n) g.rows_l1[n] = rows_l1_auto(n);
        return PTUCKER_OK;
    }
    if (k == "pack_gathers") {
        g.pack_gathers = value != 0;
        return PTUCKER_OK;
    }
    if (k == "l2_persist_mb") {
        g.l2_persist_mb = value;
        return g.inited ? apply_l2_persist() : PTUCKER_OK;
    }
    if (k == "fin_inline") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "fin_inline must be 0 or 1");
        g.fin_inline = (int)value;
        return PTUCKER_OK;
    }
    if (k == "l0_group") {
        if (value != 0 && value != 1 && value != 2 && value != 5) return fail(PTUCKER_EINVAL, "l0_group must be 0, 1, 2 or 5");
        g.l0_group = (int)value;
        return PTUCKER_OK;
    }
    if (k == "tc") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "tc must be 0 or 1");
        g.use_tc = (int)value;
        if (g.inited) return choose_kernel();
        return PTUCKER_OK;
    }
    if (k == "emulate_world" || k == "emulate_rank") {
        if (g.inited) return fail(PTUCKER_ESTATE, "%s must be set before ptucker_init", key);
        if (g.comm) return fail(PTUCKER_ESTATE, "a communicator is active");
        if (k == "emulate_world") {
            if (value < 1 || value > 1024) return fail(PTUCKER_EINVAL, "emulate_world out of range");
            g.emu_world = (int)value;
        } else {
            if (value < 0) return fail(PTUCKER_EINVAL, "emulate_rank out of range");
            g.emu_rank = (int)value;
        }
        if (g.emu_rank >= g.emu_world) g.emu_rank = 0;
        return PTUCKER_OK;
    }
    if (k == "trace") {
        if (value) {
            if (!g.trace) CK(cudaMalloc((void**)&g.trace, 8 * 512 * sizeof(long long)));
            CK(cudaMemset(g.trace, 0, 8 * 512 * sizeof(long long)));
            if (value == 2) {  // tensor-core kernel: the MMA warp also waits for each traced tile (latency probe)
                const long long one = 1;
                CK(cudaMemcpy(g.trace + 8 * 512 - 1, &one, sizeof(one), cudaMemcpyHostToDevice));
            }
        } else if (g.trace) {
            cudaFree(g.trace);
            g.trace = nullptr;
        }
        return PTUCKER_OK;
    }
    if (k == "smp_table") {
        if (value < 0 || value > 2) return fail(PTUCKER_EINVAL, "smp_table must be 0, 1 or 2");
        g.smp_tab = (int)value;
        return PTUCKER_OK;
    }
    if (k == "smp") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "smp must be 0 or 1");
        g.use_smp = (int)value;
        return PTUCKER_OK;
    }
    if (k == "sparse_core") {
        if (value < -1 || value > 1) return fail(PTUCKER_EINVAL, "sparse_core must be -1 (auto), 0 or 1");
        g.sparse_core = (int)value;
        return PTUCKER_OK;
    }
    if (k == "cache") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "cache must be 0 or 1");
        g.use_cache = (int)value;  // takes effect at the next ptucker_init
        return PTUCKER_OK;
    }
    if (k == "exchange") {
        if (value != 0 && value != 1) return fail(PTUCKER_EINVAL, "exchange must be 0 (NCCL all-gather) or 1 (push)");
        g.exchange = (int)value;
        return PTUCKER_OK;
    }
    if (k == "time_kernels") {
        g.time_kernels = value != 0;
        return PTUCKER_OK;
    }
    return fail(PTUCKER_EINVAL, "unknown option '%s'", key);
}

namespace {
// PTUCKER_DEBUG: phase times of ptucker_init on stderr
struct PhaseClock {
    bool on = getenv("PTUCKER_DEBUG") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(const char* what, cudaStream_t st = nullptr) {
        if (!on) return;
        if (st) cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[ptucker] init %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};
}  // namespace

int ptucker_init(const int32_t* coords, const void* vals, int32_t vals_dtype, int64_t nnz, int32_t order,
                 const int64_t* dims, const int32_t* core_dims, double lambda, uint64_t seed) {
    // ---- validation (synchronous, EINVAL) ----
    PhaseClock pc;
    if (!coords || !vals || !dims || !core_dims) return fail(PTUCKER_EINVAL, "null argument");
    if (vals_dtype != PTUCKER_F32 && vals_dtype != PTUCKER_F64) return fail(PTUCKER_EINVAL, "bad vals_dtype");
    if (order < 2 || order > kMaxN) return fail(PTUCKER_EINVAL, "order %d not in 2..%d", order, kMaxN);
    if (nnz < 1 || nnz > INT32_MAX) return fail(PTUCKER_EINVAL, "nnz %lld out of range", (long long)nnz);
    if (!(lambda > 0.0) || !std::isfinite(lambda)) return fail(PTUCKER_EINVAL, "lambda must be > 0");
    bool ujn = false;
    int J = 0;  // max_n J_n
    for (int n = 0; n < order; ++n) {
        if (dims[n] < 1 || dims[n] > INT32_MAX) return fail(PTUCKER_EINVAL, "dims[%d] out of range", n);
        if (core_dims[n] < 1 || core_dims[n] > 16) return fail(PTUCKER_EINVAL, "core_dims[%d] must be in 1..16", n);
        ujn = ujn || core_dims[n] != core_dims[0];
        J = std::max(J, (int)core_dims[n]);
    }
    {
        double gs = 1.0;
        for (int n = 0; n < order; ++n) gs *= core_dims[n];
        if (gs > (double)(1 << 26)) return fail(PTUCKER_EINVAL, "core of %g entries exceeds 2^26", gs);
    }
    const int esz = vals_dtype == PTUCKER_F64 ? 8 : 4;
    {
        if (!ujn && !find_update_kernel(vals_dtype, 1, order, J) && !generic_shape_ok(order, J))
            return fail(PTUCKER_EINVAL, "(N=%d, J=%d): J must be <= 16", order, J);
    }
    // ---- the COO on the device, validated there (coordinates in range, values finite:
    // the first offending entry; sum of x^2 for reading R30) before the previous context is
    // released, so an invalid call leaves it intact.  (Round 1 scanned on the host threads:
    // ~40 ms of c5's init.)
    if (!g.stream) {
        CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
        g.own_stream = true;
    }
    DeviceArena input;
    int32_t* d_coords = nullptr;
    void* d_vals = nullptr;
    CK(input.alloc((void**)&d_coords, (size_t)nnz * order * sizeof(int32_t)));
    CK(input.alloc(&d_vals, (size_t)nnz * esz));
    CK(cudaMemcpyAsync(d_coords, coords, (size_t)nnz * order * sizeof(int32_t), cudaMemcpyHostToDevice, S()));
    CK(cudaMemcpyAsync(d_vals, vals, (size_t)nnz * esz, cudaMemcpyHostToDevice, S()));
    pc.lap("H2D of the COO input", S());
    {
        int64_t* d_val = nullptr;  // [0] first bad coordinate key (entry * 16 + mode), [1] first bad value
        double* d_part = nullptr;  // per-block sums of x^2 (fixed grid: a deterministic total)
        const int vgrid = 148 * 8;
        CK(input.alloc((void**)&d_val, 2 * sizeof(int64_t)));
        CK(input.alloc((void**)&d_part, vgrid * sizeof(double)));
        launch_validate_coo(d_coords, d_vals, esz, nnz, order, dims, d_val, d_part, vgrid, S());
        CK(cudaGetLastError());
        int64_t hv[2];
        std::vector<double> hp(vgrid);
        CK(cudaMemcpyAsync(hv, d_val, sizeof(hv), cudaMemcpyDeviceToHost, S()));
        CK(cudaMemcpyAsync(hp.data(), d_part, vgrid * sizeof(double), cudaMemcpyDeviceToHost, S()));
        CK(cudaStreamSynchronize(S()));
        const uint64_t none = ~0ull;  // all bits set: no offending entry
        if ((uint64_t)hv[0] != none)
            return fail(PTUCKER_EINVAL, "coordinate %d of entry %lld out of range", (int)((uint64_t)hv[0] % 16),
                        (long long)((uint64_t)hv[0] / 16));
        if ((uint64_t)hv[1] != none)
            return fail(PTUCKER_EINVAL, "value of entry %lld is not finite", (long long)hv[1]);
        double xx = 0.0;
        for (double v : hp) xx += v;
        g_xnorm_pending = std::sqrt(xx);
    }
    pc.lap("validation (device)", S());
    // ---- fresh context ----
    free_all();
    CK(cudaGetDevice(&g.device));
    g.N = order;
    g.J = J;
    g.ujn = ujn;
    g.Jv = JDims();
    for (int n = 0; n < order; ++n) g.Jv.j[n] = core_dims[n];
    // unequal J_n: the generic kernel (delta by Eq. 12 as written, any J_n <= 16)
    // P-Tucker-Cache runs on the generic path (delta from the cache table, any shape)
    g.cache_on = g.use_cache != 0;
    g.generic = g.cache_on || ujn || find_update_kernel(vals_dtype, 1, order, J) == nullptr;
    g.xnorm = g_xnorm_pending;
    g.prec = vals_dtype;
    g.esz = esz;
    g.nnz = nnz;
    g.lambda = lambda;
    g.seed = seed;
    for (int n = 0; n < order; ++n) g.dims[n] = dims[n];
    g.lda = factor_ld(J, esz);  // every factor padded to max_n J_n (rows beyond J_n stay zero)
    int64_t nblk = 1;
    for (int l = 0; l < order - 2; ++l) nblk *= J;
    g.gp_elems = g.generic ? 0 : (int)(nblk * gblk(J, esz));  // generic kernel reads G itself
    DeviceArena& A = g.arena;
    CK(A.alloc((void**)&g.d_fail, sizeof(int)));
    CK(A.alloc((void**)&g.d_qrfail, sizeof(int)));
    CK(A.alloc((void**)&g.d_work, sizeof(unsigned int)));
    CK(A.alloc((void**)&g.d_barrier, sizeof(int)));
    CK(cudaMemsetAsync(g.d_barrier, 0, sizeof(int), S()));
    CK(A.alloc((void**)&g.red_part, 256 * sizeof(double)));
    CK(A.alloc((void**)&g.red_out, 4 * sizeof(double)));
    CK(A.alloc((void**)&g.qr, (5 * 256 + 256 * 256) * sizeof(double)));
    CK(cudaMemsetAsync(g.d_fail, 0, sizeof(int), S()));
    CK(cudaMemsetAsync(g.d_qrfail, 0, sizeof(int), S()));
    // ---- init (Alg. 2 line 1) ----
    int64_t gsize = 1;
    for (int n = 0; n < order; ++n) gsize *= g.Jv.j[n];
    CK(A.alloc(&g.G, gsize * esz));
    CK(A.alloc(&g.Gtmp, gsize * esz));
    launch_init_uniform(g.G, esz, 1, (int)gsize, (int)gsize, seed, 0, S());
    for (int n = 0; n < order; ++n) {
        CK(A.alloc(&g.A[n], dims[n] * g.lda * esz));
        CK(cudaMemsetAsync(g.A[n], 0, dims[n] * g.lda * esz, S()));
        launch_init_uniform(g.A[n], esz, dims[n], g.Jv.j[n], g.lda, seed, (uint64_t)(1 + n), S());  // idx = i*J_n + j
        if (!g.generic) CK(A.alloc(&g.Gp[n], (size_t)g.gp_elems * esz));
        CK(A.alloc((void**)&g.sse_row[n], dims[n] * sizeof(double)));
        CK(cudaMemsetAsync(g.sse_row[n], 0, dims[n] * sizeof(double), S()));
    }
    CK(A.alloc((void**)&g.d_present, (size_t)gsize));
    CK(cudaMemsetAsync(g.d_present, 1, (size_t)gsize, S()));
    g.n_present = gsize;
    int rc = rebuild_gp();
    if (rc) return rc;
    // ---- small-mode precontraction plans, order 4 only ----
    {
        int64_t tmax = 0;
        const int GBk = gblk(J, esz);
        for (int n = 0; n < order; ++n) {
            g.smp[n] = Ctx::Smp();
            if (order != 4 || g.generic) continue;
            int oth[3], c = 0;
            for (int m = 0; m < order; ++m)
                if (m != n) oth[c++] = m;
            int nsmall = 0;
            for (int x = 0; x < 3; ++x) nsmall += dims[oth[x]] <= 64;
            Ctx::Smp& sp = g.smp[n];
            if (nsmall == 2) {
                // kind 2: two small other modes -> J^2 fp64 per entry against T[i_s1][i_s2]
                int r = 0;
                for (int x = 0; x < 3; ++x)
                    if (dims[oth[x]] > 64) r = x;
                const int a = r == 0 ? 1 : 0, b = 3 - r - a;
                const int64_t elems = dims[oth[a]] * dims[oth[b]] * (int64_t)J * J;
                if (elems * 8 <= (64 << 20)) {  // fp64 table in L2 (the fp32 shared-memory variant needs <= 200 KB)
                    sp.kind = 2;
                    sp.r = oth[r]; sp.s1 = oth[a]; sp.s2 = oth[b];
                    sp.ir = r; sp.is1 = a; sp.is2 = b;
                    sp.elems = elems;
                }
            } else if (nsmall == 1) {
                // kind 1: one small other mode -> order-3 TTV against the block T[i_s] of the segment
                int sx = 0;
                for (int x = 0; x < 3; ++x)
                    if (dims[oth[x]] <= 64) sx = x;
                const int a = sx == 0 ? 1 : 0, b = sx == 2 ? 1 : 2;
                const int64_t elems = dims[oth[sx]] * (int64_t)J * GBk;
                // the index groups each row by the small mode with a 32-bit composite key
                // i_n * I_s + i_s (index.cu k_composite_key): it must fit
                const bool key32 = dims[n] * dims[oth[sx]] < ((int64_t)1 << 32);
                if (elems * esz <= 128 * 1024 && key32) {
                    sp.kind = 1;
                    sp.s1 = oth[sx]; sp.r = oth[a]; sp.s2 = oth[b];   // r, s2 = the two large modes (a < b)
                    sp.is1 = sx; sp.ir = a; sp.is2 = b;
                    sp.elems = elems;
                }
            }
            if (sp.kind) tmax = std::max(tmax, sp.elems);
        }
        if (tmax > 0) CK(A.alloc(&g.smp_T, (size_t)tmax * 8));
        if (tmax > 0) CK(A.alloc(&g.smp_T32, (size_t)tmax * 4));
    }
    pc.lap("allocation + factor init", S());
    // ---- device index of every mode ----
    if (!g.comm) {  // no communicator: a single rank, or an emulated rank of a partition (tests)
        g.world = g.emu_world;
        g.rank = g.emu_rank;
    }
    {
        // automatic S (option seg_len = -1): at least one full 128-lane group per SM, i.e.
        // S = the power of two >= |Omega| / (SMs * 128), clamped to [8, 256].  Small tensors
        // (c1, c2) get short segments so every SM has work (their multi-segment rows are
        // reduced by the heavy-row finalize); large ones keep S = 256.  It depends only on
        // |Omega| and the device (not on the rank count), so factors stay bit-identical for
        // any number of GPUs (F9).
        int nsm_dev = 148;
        CK(cudaDeviceGetAttribute(&nsm_dev, cudaDevAttrMultiProcessorCount, g.device));
        if (g.seg_len > 0) {
            g.seg_len_eff = g.seg_len;
        } else {
            const int64_t want = (nnz + (int64_t)nsm_dev * 128 - 1) / ((int64_t)nsm_dev * 128);
            int sl = 8;
            while (sl < want && sl < 256) sl *= 2;
            g.seg_len_eff = sl;
        }
    }
#ifndef PT_SCRATCH_BUMP
#define PT_SCRATCH_BUMP 1
#endif
    g.scratch.bump = PT_SCRATCH_BUMP != 0;  // index-build temporaries: rewound chunks, freed after the builds
    for (int n = 0; n < order; ++n) {
        ModeIndex& m = g.mi[n];
        CK(build_mode_csr(d_coords, nnz, order, n, dims[n], m, g.arena, g.scratch, S()));
        pc.lap("CSR (sort, row_ptr)", S());
        m.bounds.assign((size_t)g.world + 1, 0);
        partition_rows(m.h_row_ptr.data(), dims[n], g.world, m.bounds.data());
        const int smode = g.smp[n].kind == 1 ? g.smp[n].s1 : -1;  // group each row by the small mode
        m.Is = smode >= 0 ? dims[smode] : 1;
        // kind-1 modes on the tensor cores: lanes in (i_s, length) order, one i_s per group
        const bool aux_groups = smode >= 0 && g.tc_table && g.use_tc && vals_dtype == PTUCKER_F32 &&
                                find_update_kernel_tc(1, J) != nullptr;
        // Per-mode S for the tensor-core kernel (automatic S only): its 128-lane groups are
        // assigned to the CTAs statically, so with few long groups the CTA with one group more
        // than the average sets the time (c3's table modes: 624 groups of ~256 tiles on 148
        // CTAs, 5 vs 4.2); take the largest S <= the global one that gives >= 8 groups per SM,
        // when one down to 32 does (c3 modes 2/3: S = 128, update 1.085 -> 1.045 ms; S = 64 was
        // slower, 1.12 ms, its heavy-row partials doubling the finalize).  Computed from all
        // rows (not this rank's block), so it does not depend on the number of GPUs.
        int S_n = g.seg_len_eff;
        const bool on_tc = !g.generic && vals_dtype == PTUCKER_F32 && g.use_tc &&
                           ((order == 3 && find_update_kernel_tc(1, J) != nullptr) || aux_groups);
        if (g.seg_len < 0 && on_tc) {
            int nsm_dev = 148;
            CK(cudaDeviceGetAttribute(&nsm_dev, cudaDevAttrMultiProcessorCount, g.device));
            for (int Sc = g.seg_len_eff; Sc >= 32; Sc /= 2) {
                int64_t segs = 0;
                for (int64_t r = 0; r < dims[n]; ++r) {
                    const int64_t len = m.h_row_ptr[r + 1] - m.h_row_ptr[r];
                    segs += len == 0 ? 1 : (len + Sc - 1) / Sc;
                }
                if (segs / 128 >= 8 * (int64_t)nsm_dev) {
                    S_n = Sc;
                    break;
                }
            }
        }
        m.seg_len = S_n;
        CK(build_mode_sell(d_coords, d_vals, esz, nnz, order, n, g.Jv.j[n], S_n, m.bounds[g.rank],
                           m.bounds[g.rank + 1], smode, m, g.arena, g.scratch, S(), aux_groups, g.cache_on));
        {   // most segments of one of this rank's rows (the heavy-row finalize picks its kernels by it)
            // exact, from the index (a small-mode-grouped row has a segment per class it meets)
            std::vector<int32_t> hn((size_t)m.nheavy);
            if (m.nheavy > 0)
                CK(cudaMemcpyAsync(hn.data(), m.hnseg, sizeof(int32_t) * m.nheavy, cudaMemcpyDeviceToHost, S()));
            CK(cudaStreamSynchronize(S()));
            int64_t mx = 1, mn = 0;
            for (int32_t v : hn) {
                mx = std::max<int64_t>(mx, v);
                mn = mn == 0 ? v : std::min<int64_t>(mn, v);
            }
            m.hmaxseg = mx;
            m.hminseg = mn;  // fewest segments of a heavy row (0: none)
        }
        pc.lap("SELL segments + scatter", S());
    }
    CK(A.alloc((void**)&g.lit_part, std::max<int64_t>(g.mi[0].nslices * 32, 1) * sizeof(double)));
    CK(cudaStreamSynchronize(S()));
    g.scratch.free_chunks();
    pc.lap("scratch free");

    CK(cudaStreamSynchronize(S()));
    if (g.generic) {
        // the literal error of generic shapes runs over the COO (update_generic.cu has no literal pass)
        CK(g.arena.alloc((void**)&g.coo_c, (size_t)nnz * order * sizeof(int32_t)));
        CK(g.arena.alloc(&g.coo_v, (size_t)nnz * esz));
        CK(cudaMemcpyAsync(g.coo_c, d_coords, (size_t)nnz * order * sizeof(int32_t), cudaMemcpyDeviceToDevice, S()));
        CK(cudaMemcpyAsync(g.coo_v, d_vals, (size_t)nnz * esz, cudaMemcpyDeviceToDevice, S()));
        CK(cudaStreamSynchronize(S()));
    }
    if (g.cache_on) {
        // Alg. 3 lines 1-4: the table for every entry (every rank holds all of it:
        // each mode's rows need the entries of that mode's row block)
        const double bytes = (double)nnz * (double)gsize * 8.0;
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        if (bytes > 0.8 * (double)fr)
            return fail(PTUCKER_ERESOURCE, "P-Tucker-Cache table of %.3g GB (|Omega| x |G| doubles) exceeds device memory",
                        bytes / 1e9);
        CK(g.arena.alloc((void**)&g.pres, (size_t)bytes));
        int64_t imax = 0;
        for (int n = 0; n < order; ++n) imax = std::max<int64_t>(imax, dims[n]);
        CK(g.arena.alloc(&g.cache_old, (size_t)imax * g.lda * esz));
        CK(g.arena.alloc((void**)&g.cache_ptrs, kMaxN * sizeof(void*)));
        CK(cudaMemcpyAsync(g.cache_ptrs, g.A, kMaxN * sizeof(void*), cudaMemcpyHostToDevice, S()));
        launch_pres_init(order, g.Jv, esz, g.G, (const void* const*)g.cache_ptrs, g.lda, g.coo_c, nnz, g.pres, S());
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(S()));
    }
    input.release_all();
    g.inited = true;
    rc = choose_kernel();
    if (rc) {
        g.inited = false;
        return rc;
    }
    rc = apply_l2_persist();
    if (rc) return rc;
    for (int n = 0; n < order; ++n) g.rows_l1[n] = rows_l1_auto(n);
    g.sse_mode = -1;
    return PTUCKER_OK;
}

int ptucker_peer_handles(uint8_t* out, int32_t cap) {
    int rc = require_init();
    if (rc) return rc;
    if (!out || cap < g.N * 64) return fail(PTUCKER_EINVAL, "need %d bytes", g.N * 64);
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    for (int n = 0; n < g.N; ++n) {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, g.A[n]));  // A^(n) is its own cudaMalloc (DeviceArena)
        memcpy(out + 64 * n, &h, 64);
    }
    return PTUCKER_OK;
}

int ptucker_open_peers(const uint8_t* handles, int32_t world) {
    int rc = require_init();
    if (rc) return rc;
    if (!handles || world != g.world) return fail(PTUCKER_EINVAL, "handles of %d ranks expected", g.world);
    if (g.world - 1 > kMaxPeers) return fail(PTUCKER_EINVAL, "at most %d peers", kMaxPeers);
    close_peers();
    invalidate_graph();
    int k = 0;
    for (int r = 0; r < world; ++r) {
        if (r == g.rank) continue;
        for (int n = 0; n < g.N; ++n) {
            cudaIpcMemHandle_t h;
            memcpy(&h, handles + 64 * ((size_t)r * g.N + n), 64);
            const cudaError_t e = cudaIpcOpenMemHandle(&g.peer_A[n][k], h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                g.peer_A[n][k] = nullptr;
                close_peers();
                cudaGetLastError();
                return fail(PTUCKER_ECUDA, "cudaIpcOpenMemHandle(rank %d, A^(%d)): %s", r, n, cudaGetErrorString(e));
            }
        }
        ++k;
    }
    g.npeer = k;
    return PTUCKER_OK;
}

int ptucker_update_mode(int32_t n) {
    int rc = require_init();
    if (rc) return rc;
    if (n < 0 || n >= g.N) return fail(PTUCKER_EINVAL, "mode %d out of range", n);
    g.last_fail_mode = n;
    rc = timed("update", [&]() -> int { return launch_update_kernel(n, false); }, n);
    if (rc) return rc;
    ModeIndex& m = g.mi[n];
    if (m.nheavy > 0 && !g.inline_used) {
        rc = timed("finalize", [&]() -> int {
            PeerRows pr;
            if (pushing()) {
                pr.n = g.npeer;
                for (int r = 0; r < g.npeer; ++r) pr.base[r] = g.peer_A[n][r];
            }
            launch_heavy_finalize(m.nheavy, m.hrow, m.hnseg, m.hpbase, m.partials, m.hrec, g.Jv.j[n], g.lambda, g.A[n], g.esz,
                                  g.lda, g.sse_row[n], g.d_fail, S(), pr, m.hmaxseg, m.hminseg);
            g.launches += 3;
            CK(cudaGetLastError());
            return PTUCKER_OK;
        }, n);
        if (rc) return rc;
    }
    if (g.world > 1 && pushing()) {
        // the rows already sit in every replica (pushed by the kernels above); an all-reduce
        // of one int orders every rank's pushes before any rank's next mode.  Without a
        // communicator (tests: ranks as processes on one GPU) the caller orders the ranks.
        if (g.comm) {
            rc = timed("allgather", [&]() -> int {
                NK(ncclAllReduce(g.d_barrier, g.d_barrier, 1, ncclInt32, ncclSum, g.comm, S()));
                return PTUCKER_OK;
            });
            if (rc) return rc;
        }
    } else if (g.world > 1 && g.comm) {
        rc = timed("allgather", [&]() -> int {
            // all-gather-v of the row blocks (grouped broadcasts, in place)
            const ncclDataType_t dt = g.prec == PTUCKER_F64 ? ncclDouble : ncclFloat;
            NK(ncclGroupStart());
            for (int r = 0; r < g.world; ++r) {
                const int64_t b0 = m.bounds[r], b1 = m.bounds[r + 1];
                if (b1 <= b0) continue;
                char* p = (char*)g.A[n] + (size_t)b0 * g.lda * g.esz;
                NK(ncclBroadcast(p, p, (size_t)(b1 - b0) * g.lda, dt, r, g.comm, S()));
            }
            NK(ncclGroupEnd());
            return PTUCKER_OK;
        });
        if (rc) return rc;
    }
    if (g.cache_on) {
        // Alg. 3 lines 16-19: every entry's cache row with the new A^(n) (all ranks
        // hold the refreshed replica by now)
        rc = timed("cache_update", [&]() -> int {
            launch_pres_update(g.N, g.Jv, g.esz, n, g.G, (const void* const*)g.cache_ptrs, g.lda, g.cache_old, g.coo_c,
                               g.nnz, g.pres, S());
            g.launches += 1;
            CK(cudaGetLastError());
            return PTUCKER_OK;
        }, n);
        if (rc) return rc;
    }
    g.sse_mode = n;
    return PTUCKER_OK;
}

int ptucker_sweep(void) {
    int rc = require_init();
    if (rc) return rc;
    // replay the captured sweep (one graph launch instead of ~2-5 launches per mode); kernel
    // timing (time_kernels) needs the per-launch events, so it runs the sweep directly
    const bool graphs = g.use_graph && !g.time_kernels && !g.cache_on;  // Cache: table rebuilds are host-decided
    if (graphs && g.graph_exec) {
        CK(cudaGraphLaunch(g.graph_exec, S()));
        g.launches += g.graph_launches;
        g.last_fail_mode = g.N - 1;
        g.sse_mode = g.N - 1;
        return PTUCKER_OK;
    }
    cudaGraph_t graph = nullptr;
    const int64_t l0 = g.launches;
    if (graphs) CK(cudaStreamBeginCapture(S(), cudaStreamCaptureModeRelaxed));
    for (int n = 0; n < g.N; ++n) {
        rc = ptucker_update_mode(n);
        if (rc) {
            if (graphs) {
                cudaStreamEndCapture(S(), &graph);
                if (graph) cudaGraphDestroy(graph);
                cudaGetLastError();
            }
            return rc;
        }
    }
    if (graphs) {
        CK(cudaStreamEndCapture(S(), &graph));
        const cudaError_t e = cudaGraphInstantiate(&g.graph_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            g.graph_exec = nullptr;
            return fail(PTUCKER_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
        }
        g.graph_launches = g.launches - l0;
        CK(cudaGraphLaunch(g.graph_exec, S()));  // the capture recorded the work; run it once
    }
    return PTUCKER_OK;
}

static int finish_error(double* out) {
    if (g.world > 1 && g.comm) NK(ncclAllReduce(g.red_out, g.red_out, 1, ncclDouble, ncclSum, g.comm, S()));
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, g.red_out, sizeof(double), cudaMemcpyDeviceToHost, S()));
    int rc = sync_and_check();
    if (rc) return rc;
    *out = std::sqrt(std::max(h, 0.0));
    return PTUCKER_OK;
}

int ptucker_error_literal(double* out) {
    int rc = require_init();
    if (rc) return rc;
    if (!out) return fail(PTUCKER_EINVAL, "null out");
    if (g.generic) {  // (x - x_hat)^2 over this rank's mode-0 rows of the device COO, then the same reduction
        void** d_A = nullptr;
        double* d_r = nullptr;
        DeviceArena tmp;
        CK(tmp.alloc((void**)&d_A, kMaxN * sizeof(void*)));
        CK(tmp.alloc((void**)&d_r, (size_t)g.nnz * sizeof(double)));
        CK(cudaMemcpyAsync(d_A, g.A, kMaxN * sizeof(void*), cudaMemcpyHostToDevice, S()));
        launch_predict(g.N, g.Jv, g.esz, g.G, (const void* const*)d_A, g.lda, g.coo_c, g.coo_v, g.nnz, d_r, 1, g.nsm,
                       S(), g.mi[0].r0, g.mi[0].r1);
        launch_sum(d_r, g.nnz, g.red_part, g.red_out, S());
        g.launches += 3;
        CK(cudaGetLastError());
        return finish_error(out);  // synchronises before tmp is freed
    }
    rc = timed("literal", [&]() -> int { return launch_update_kernel(0, true); });
    if (rc) return rc;
    rc = timed("error_reduce", [&]() -> int {
        launch_sum(g.lit_part, g.mi[0].nslices * 32, g.red_part, g.red_out, S());
        g.launches += 2;
        CK(cudaGetLastError());
        return PTUCKER_OK;
    });
    if (rc) return rc;
    return finish_error(out);
}

int ptucker_error(double* out) {
    int rc = require_init();
    if (rc) return rc;
    if (!out) return fail(PTUCKER_EINVAL, "null out");
    if (g.sse_mode < 0) return ptucker_error_literal(out);
    const ModeIndex& m = g.mi[g.sse_mode];
    rc = timed("error_reduce", [&]() -> int {
        launch_sum(g.sse_row[g.sse_mode] + m.r0, m.r1 - m.r0, g.red_part, g.red_out, S());
        g.launches += 2;
        CK(cudaGetLastError());
        return PTUCKER_OK;
    });
    if (rc) return rc;
    return finish_error(out);
}

int ptucker_orthogonalize(void) {
    int rc = require_init();
    if (rc) return rc;
    invalidate_graph();  // swaps G and Gtmp
    g.pres_stale = true;
    g.sp_n = -1;         // G x_n R is dense
    const int J = g.J;  // max_n J_n (scratch sizes)
    for (int n = 0; n < g.N; ++n)
        if (g.dims[n] < g.Jv.j[n]) return fail(PTUCKER_EINVAL, "orthogonalize needs I_%d >= J_%d", n, n);
    if (!g.qd) {
        int64_t imax = 0;
        for (int n = 0; n < g.N; ++n) imax = std::max(imax, g.dims[n]);
        CK(g.arena.alloc((void**)&g.qd, (size_t)imax * J * sizeof(double)));
    }
    double* W = g.qr;
    double* R1 = W + 256;
    double* R2 = R1 + 256;
    double* R = R2 + 256;
    double* part = g.qr + 5 * 256;
    rc = timed("qr", [&]() -> int {
        for (int n = 0; n < g.N; ++n) {
            const int64_t I = g.dims[n];
            const int Jn = g.Jv.j[n];
            launch_gram(g.A[n], g.esz, false, I, Jn, g.lda, part, W, S());
            launch_chol_upper(W, Jn, R1, g.d_qrfail, n + 1, S());
            launch_apply_rinv(g.A[n], g.esz, g.lda, g.qd, 8, Jn, I, Jn, R1, S());
            launch_gram(g.qd, 8, true, I, Jn, Jn, part, W, S());
            launch_chol_upper(W, Jn, R2, g.d_qrfail, n + 1, S());
            launch_apply_rinv(g.qd, 8, Jn, g.A[n], g.esz, g.lda, I, Jn, R2, S());
            launch_mat_upper_mul(R2, R1, R, Jn, S());
            launch_core_mode_product(g.G, g.Gtmp, g.esz, g.N, g.Jv, n, R, S());
            g.launches += 9;
            std::swap(g.G, g.Gtmp);
        }
        CK(cudaGetLastError());
        return rebuild_gp();
    });
    if (rc) return rc;
    g.sse_mode = -1;
    {
        int64_t gs = 1;
        for (int n = 0; n < g.N; ++n) gs *= g.Jv.j[n];
        CK(cudaMemsetAsync(g.d_present, 1, (size_t)gs, S()));  // G x_n R is dense again
        g.n_present = gs;
    }
    return sync_and_check();
}

int ptucker_get_factor(int32_t n, void* out) {
    int rc = require_init();
    if (rc) return rc;
    if (n < 0 || n >= g.N || !out) return fail(PTUCKER_EINVAL, "bad mode or buffer");
    const size_t rb = (size_t)g.Jv.j[n] * g.esz;  // I_n x J_n, row-major
    CK(cudaMemcpy2DAsync(out, rb, g.A[n], (size_t)g.lda * g.esz, rb, g.dims[n], cudaMemcpyDeviceToHost, S()));
    return sync_and_check();
}

int ptucker_set_factor(int32_t n, const void* in) {
    int rc = require_init();
    if (rc) return rc;
    if (n < 0 || n >= g.N || !in) return fail(PTUCKER_EINVAL, "bad mode or buffer");
    const size_t rb = (size_t)g.Jv.j[n] * g.esz;
    CK(cudaMemcpy2DAsync(g.A[n], (size_t)g.lda * g.esz, in, rb, rb, g.dims[n], cudaMemcpyHostToDevice, S()));
    g.sse_mode = -1;
    g.pres_stale = true;
    CK(cudaStreamSynchronize(S()));
    return PTUCKER_OK;
}

int ptucker_get_core(void* out) {
    int rc = require_init();
    if (rc) return rc;
    if (!out) return fail(PTUCKER_EINVAL, "null buffer");
    int64_t gsize = 1;
    for (int n = 0; n < g.N; ++n) gsize *= g.Jv.j[n];
    CK(cudaMemcpyAsync(out, g.G, gsize * g.esz, cudaMemcpyDeviceToHost, S()));
    return sync_and_check();
}

int ptucker_set_core(const void* in) {
    int rc = require_init();
    if (rc) return rc;
    if (!in) return fail(PTUCKER_EINVAL, "null buffer");
    int64_t gsize = 1;
    for (int n = 0; n < g.N; ++n) gsize *= g.Jv.j[n];
    CK(cudaMemcpyAsync(g.G, in, gsize * g.esz, cudaMemcpyHostToDevice, S()));
    rc = rebuild_gp();
    if (rc) return rc;
    g.sse_mode = -1;
    g.pres_stale = true;
    g.sp_n = -1;
    CK(cudaMemsetAsync(g.d_present, 1, (size_t)gsize, S()));  // a pushed core is dense (no truncation history)
    g.n_present = gsize;
    CK(cudaStreamSynchronize(S()));
    return PTUCKER_OK;
}

// ---------------------------------------------------------------- P-Tucker-Approx
namespace {
// R(beta) (Eq. 13) of every core entry into R (C order; NaN for truncated entries).
int compute_core_scores(bool with_keys) {
    const int N = g.N, J = g.J;
    int64_t K1 = 1;
    for (int n = 1; n < N; ++n) K1 *= g.Jv.j[n];
    const int64_t gsize = K1 * g.Jv.j[0];
    // segment ranges of the outer reduction: ~256 segments each (enough blocks to fill the
    // GPU: 3.8 ms at a fixed 256 ranges for c5's 10^6 segments), at most 4096 ranges
    const int nsplit = (int)std::min<int64_t>(4096, std::max<int64_t>(256, g.mi[0].nslices * 32 / 256));
    const ModeIndex& m = g.mi[0];
    if (g.ujn || !approx_shape_ok(N, J)) {  // generic shapes: U, V by definition over the device COO
        if (!g.coo_c) return fail(PTUCKER_EINVAL, "internal: no device COO for the generic Approx scores");
        if (!g.ax_UV) {
            CK(g.arena.alloc((void**)&g.ax_ptrs, kMaxN * sizeof(void*)));
            CK(g.arena.alloc((void**)&g.ax_E, (size_t)g.nnz * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_UV, 2 * gsize * sizeof(double)));
            CK(cudaMemcpyAsync(g.ax_ptrs, g.A, kMaxN * sizeof(void*), cudaMemcpyHostToDevice, S()));
        }
        int rc = timed("approx_scores", [&]() -> int {
            launch_predict(N, g.Jv, g.esz, g.G, (const void* const*)g.ax_ptrs, g.lda, g.coo_c, g.coo_v, g.nnz, g.ax_E, 0,
                           g.nsm, S());
            launch_approx_literal(N, g.Jv, g.esz, (const void* const*)g.ax_ptrs, g.lda, g.coo_c, g.coo_v, g.ax_E, g.nnz,
                                  m.r0, m.r1, g.ax_UV, S());
            g.launches += 2;
            CK(cudaGetLastError());
            return PTUCKER_OK;
        });
        if (rc) return rc;
    } else {
        const int64_t nlanes = m.nslices * 32;
        if (!g.ax_UV) {
            CK(g.arena.alloc((void**)&g.ax_G64, gsize * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_A0, std::max<int64_t>(nlanes, 1) * J * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_W, std::max<int64_t>(nlanes, 1) * K1 * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_W2, std::max<int64_t>(nlanes, 1) * K1 * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_E, std::max<int64_t>(m.nslots, 1) * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_part, (size_t)2 * nsplit * gsize * sizeof(double)));
            CK(g.arena.alloc((void**)&g.ax_ptrs, 2 * kMaxN * sizeof(void*)));
            CK(g.arena.alloc((void**)&g.ax_UV, 2 * gsize * sizeof(double)));
            void* h[2 * kMaxN] = {nullptr};
            for (int k = 0; k < N - 1; ++k) h[k] = m.sc[k];
            for (int k = 0; k < N; ++k) h[kMaxN + k] = g.A[k];
            CK(cudaMemcpyAsync(g.ax_ptrs, h, sizeof(h), cudaMemcpyHostToDevice, S()));
    }
    int rc = timed("approx_scores", [&]() -> int {
        launch_approx_uv(N, J, g.esz, m.nslices, m.slice_off, m.lane_row, m.lane_len, (const int32_t* const*)g.ax_ptrs,
                         m.sv, (const void* const*)(g.ax_ptrs + kMaxN), g.lda, g.G, g.ax_G64, g.ax_A0, g.ax_W,
                         g.ax_W2, g.ax_E, g.ax_part, nsplit, g.ax_UV, g.nsm, S());
        g.launches += m.nslices > 0 ? 4 : 3;
        CK(cudaGetLastError());
        return PTUCKER_OK;
    });
    if (rc) return rc;
    }
    if (g.world > 1 && g.comm) NK(ncclAllReduce(g.ax_UV, g.ax_UV, (size_t)(2 * gsize), ncclDouble, ncclSum, g.comm, S()));
    // R (and the selection keys) on the device
    if (!g.ax_R) {
        CK(g.arena.alloc((void**)&g.ax_R, gsize * sizeof(double)));
        CK(g.arena.alloc((void**)&g.ax_key, gsize * sizeof(uint64_t)));
        CK(g.arena.alloc((void**)&g.ax_key2, gsize * sizeof(uint64_t)));
        CK(g.arena.alloc((void**)&g.ax_idx, gsize * sizeof(int64_t)));
        CK(g.arena.alloc((void**)&g.ax_idx2, gsize * sizeof(int64_t)));
        g.ax_tmp_bytes = core_select_temp_bytes(gsize);
        CK(g.arena.alloc(&g.ax_tmp, std::max<size_t>(g.ax_tmp_bytes, 16)));
    }
    launch_core_scores(gsize, g.esz, g.G, g.ax_UV, g.d_present, g.ax_R, with_keys ? g.ax_key : nullptr,
                       with_keys ? g.ax_idx : nullptr, S());
    g.launches += 1;
    CK(cudaGetLastError());
    return PTUCKER_OK;
}
}  // namespace

int ptucker_core_scores(double* out) {
    int rc = require_init();
    if (rc) return rc;
    if (!out) return fail(PTUCKER_EINVAL, "null buffer");
    rc = compute_core_scores(false);
    if (rc) return rc;
    int64_t gsize = 1;
    for (int n = 0; n < g.N; ++n) gsize *= g.Jv.j[n];
    CK(cudaMemcpyAsync(out, g.ax_R, gsize * sizeof(double), cudaMemcpyDeviceToHost, S()));
    CK(cudaStreamSynchronize(S()));
    return PTUCKER_OK;
}

int ptucker_truncate_core(double p, int64_t* removed) {
    int rc = require_init();
    if (rc) return rc;
    if (!(p > 0.0 && p < 1.0)) return fail(PTUCKER_EINVAL, "truncation rate p must be in (0, 1)");
    rc = compute_core_scores(true);
    if (rc) return rc;
    int64_t gsize = 1;
    for (int n = 0; n < g.N; ++n) gsize *= g.Jv.j[n];
    const int64_t n = g.n_present;
    int64_t k = (int64_t)std::floor(p * (double)n);  // reading R29: floor(p |G|), at least one entry stays
    if (k > n - 1) k = n - 1;
    if (k < 0) k = 0;
    if (k > 0) {
        // reading R28: descending R, ties by ascending C-order index (stable device sort)
        CK(launch_core_truncate(gsize, k, g.ax_key, g.ax_idx, g.ax_key2, g.ax_idx2, g.ax_tmp, g.ax_tmp_bytes, g.esz,
                                g.G, g.d_present, S()));
        g.launches += 2;
        g.n_present -= k;
        g.pres_stale = true;  // G changed (P-Tucker-Cache: the table is rebuilt before the next update)
        rc = rebuild_gp();
        if (rc) return rc;
        g.sse_mode = -1;
        if (g.generic) {  // the coordinate list of the present entries, C order (sparse-core delta)
            std::vector<uint8_t> pres_h((size_t)gsize);
            CK(cudaMemcpyAsync(pres_h.data(), g.d_present, (size_t)gsize, cudaMemcpyDeviceToHost, S()));
            CK(cudaStreamSynchronize(S()));
            // per mode n: the present entries grouped by lane (t mod 32, t = the index over the
            // other modes, the dense loop's lane split) and in C order within a lane
            std::vector<uint64_t> dg((size_t)(g.N * gsize));
            std::vector<int64_t> ix((size_t)(g.N * gsize));
            std::vector<int32_t> off((size_t)(g.N * 33));
            int64_t np = 0;
            for (int n = 0; n < g.N; ++n) {
                std::vector<std::vector<int64_t>> per(32);
                for (int64_t b = 0; b < gsize; ++b) {
                    if (!pres_h[b]) continue;
                    int64_t r = b, t = 0, mul = 1;
                    for (int m = g.N - 1; m >= 0; --m) {
                        const int dgt = (int)(r % g.Jv.j[m]);
                        r /= g.Jv.j[m];
                        if (m != n) {
                            t += dgt * mul;
                            mul *= g.Jv.j[m];
                        }
                    }
                    per[t % 32].push_back(b);
                }
                int64_t w = 0;
                for (int l = 0; l < 32; ++l) {
                    off[n * 33 + l] = (int32_t)w;
                    for (int64_t b : per[l]) {
                        uint64_t code = 0;
                        int64_t r = b;
                        for (int m = g.N - 1; m >= 0; --m) {
                            code |= (uint64_t)(r % g.Jv.j[m]) << (4 * m);
                            r /= g.Jv.j[m];
                        }
                        dg[(size_t)(n * gsize + w)] = code;
                        ix[(size_t)(n * gsize + w)] = b;
                        ++w;
                    }
                }
                off[n * 33 + 32] = (int32_t)w;
                np = w;
            }
            if (!g.sp_digits) {
                CK(g.arena.alloc((void**)&g.sp_digits, (size_t)(g.N * gsize) * sizeof(uint64_t)));
                CK(g.arena.alloc((void**)&g.sp_index, (size_t)(g.N * gsize) * sizeof(int64_t)));
                CK(g.arena.alloc((void**)&g.sp_off, (size_t)(g.N * 33) * sizeof(int32_t)));
            }
            CK(cudaMemcpyAsync(g.sp_digits, dg.data(), dg.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, S()));
            CK(cudaMemcpyAsync(g.sp_index, ix.data(), ix.size() * sizeof(int64_t), cudaMemcpyHostToDevice, S()));
            CK(cudaMemcpyAsync(g.sp_off, off.data(), off.size() * sizeof(int32_t), cudaMemcpyHostToDevice, S()));
            CK(cudaStreamSynchronize(S()));
            g.sp_n = np;
            invalidate_graph();
        }
    }
    if (removed) *removed = k;
    return PTUCKER_OK;
}

int ptucker_core_nnz(int64_t* nnz) {
    int rc = require_init();
    if (rc) return rc;
    if (!nnz) return fail(PTUCKER_EINVAL, "null out");
    *nnz = g.n_present;
    return PTUCKER_OK;
}

// ---------------------------------------------------------------- prediction, held-out RMSE, driver
namespace {
int predict_common(const int32_t* coords, const void* vals, int vals_dtype, int64_t n, double* out, bool rmse) {
    if (!coords || !out || (rmse && !vals) || n < 0) return fail(PTUCKER_EINVAL, "null argument or n < 0");
    if (rmse && n == 0) return fail(PTUCKER_EINVAL, "empty test set");
    if (rmse && vals_dtype != g.prec) return fail(PTUCKER_EINVAL, "test values must have the context's precision");
    for (int64_t q = 0; q < n; ++q)
        for (int k = 0; k < g.N; ++k) {
            const int32_t c = coords[q * g.N + k];
            if (c < 0 || c >= g.dims[k])
                return fail(PTUCKER_EINVAL, "coordinate %d of query %lld out of range", k, (long long)q);
        }
    if (n == 0) return PTUCKER_OK;
    DeviceArena tmp;
    int32_t* d_c = nullptr;
    void* d_v = nullptr;
    double* d_o = nullptr;
    void** d_A = nullptr;
    CK(tmp.alloc((void**)&d_c, (size_t)n * g.N * sizeof(int32_t)));
    CK(tmp.alloc((void**)&d_o, (size_t)n * sizeof(double)));
    CK(tmp.alloc((void**)&d_A, kMaxN * sizeof(void*)));
    CK(cudaMemcpyAsync(d_c, coords, (size_t)n * g.N * sizeof(int32_t), cudaMemcpyHostToDevice, S()));
    CK(cudaMemcpyAsync(d_A, g.A, kMaxN * sizeof(void*), cudaMemcpyHostToDevice, S()));
    if (rmse) {
        CK(tmp.alloc(&d_v, (size_t)n * g.esz));
        CK(cudaMemcpyAsync(d_v, vals, (size_t)n * g.esz, cudaMemcpyHostToDevice, S()));
    }
    launch_predict(g.N, g.Jv, g.esz, g.G, (const void* const*)d_A, g.lda, d_c, d_v, n, d_o, rmse ? 1 : 0, g.nsm, S());
    g.launches += 1;
    CK(cudaGetLastError());
    if (rmse) {
        launch_sum(d_o, n, g.red_part, g.red_out, S());
        g.launches += 2;
        double s = 0.0;
        CK(cudaMemcpyAsync(&s, g.red_out, sizeof(double), cudaMemcpyDeviceToHost, S()));
        CK(cudaStreamSynchronize(S()));
        *out = std::sqrt(s / (double)n);
    } else {
        CK(cudaMemcpyAsync(out, d_o, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, S()));
        CK(cudaStreamSynchronize(S()));
    }
    return PTUCKER_OK;
}
}  // namespace

int ptucker_predict(const int32_t* coords, int64_t n, double* out) {
    int rc = require_init();
    if (rc) return rc;
    return predict_common(coords, nullptr, g.prec, n, out, false);
}

int ptucker_test_rmse(const int32_t* coords, const void* vals, int32_t vals_dtype, int64_t n, double* out) {
    int rc = require_init();
    if (rc) return rc;
    return predict_common(coords, vals, vals_dtype, n, out, true);
}

int ptucker_run(int32_t max_iters, double tol, double approx_p, int32_t orthogonalize, double* errors,
                int32_t* iters) {
    int rc = require_init();
    if (rc) return rc;
    if (max_iters < 0 || !(tol >= 0.0) || approx_p < 0.0 || approx_p >= 1.0)
        return fail(PTUCKER_EINVAL, "bad max_iters, tol or approx_p");
    double e = 0.0;
    rc = ptucker_error(&e);
    if (rc) return rc;
    if (errors) errors[0] = e;
    int t = 0;
    while (t < max_iters) {
        rc = ptucker_sweep();  // Alg. 2 line 3
        if (rc) return rc;
        double et = 0.0;
        rc = ptucker_error(&et);  // line 4 (Eq. 5)
        if (rc) return rc;
        ++t;
        if (errors) errors[t] = et;
        if (approx_p > 0.0) {  // lines 5-6 (P-Tucker-Approx)
            rc = ptucker_truncate_core(approx_p, nullptr);
            if (rc) return rc;
        }
        // reading R30: converged when the error changed by less than tol relative to the
        // previous error, or is itself below tol of the data's norm (a perfect fit)
        const bool conv = std::fabs(et - e) < tol * e || et <= tol * g.xnorm;
        e = et;
        if (conv) break;
    }
    if (iters) *iters = t;
    if (orthogonalize) {  // lines 8-11
        rc = ptucker_orthogonalize();
        if (rc) return rc;
    }
    return PTUCKER_OK;
}


int ptucker_get_mode_index(int32_t n, int64_t* row_ptr, int64_t* perm) {
    int rc = require_init();
    if (rc) return rc;
    if (n < 0 || n >= g.N || !row_ptr || !perm) return fail(PTUCKER_EINVAL, "bad mode or buffer");
    const ModeIndex& m = g.mi[n];
    memcpy(row_ptr, m.h_row_ptr.data(), sizeof(int64_t) * (size_t)(m.I + 1));
    std::vector<int32_t> p32((size_t)g.nnz);
    CK(cudaMemcpyAsync(p32.data(), m.perm, sizeof(int32_t) * (size_t)g.nnz, cudaMemcpyDeviceToHost, S()));
    CK(cudaStreamSynchronize(S()));
    for (int64_t e = 0; e < g.nnz; ++e) perm[e] = p32[(size_t)e];
    return PTUCKER_OK;
}

int ptucker_get_partition(int32_t n, int64_t* bounds) {
    int rc = require_init();
    if (rc) return rc;
    if (n < 0 || n >= g.N || !bounds) return fail(PTUCKER_EINVAL, "bad mode or buffer");
    memcpy(bounds, g.mi[n].bounds.data(), sizeof(int64_t) * g.mi[n].bounds.size());
    return PTUCKER_OK;
}

int ptucker_kernel_stats(const char* name, double* total_ms, int64_t* launches) {
    if (!name || !total_ms || !launches) return fail(PTUCKER_EINVAL, "null argument");
    int rc = fold_stats();
    if (rc) return rc;
    auto it = g.stats.find(name);
    *total_ms = it == g.stats.end() ? 0.0 : it->second.first;
    *launches = it == g.stats.end() ? 0 : it->second.second;
    return PTUCKER_OK;
}

int ptucker_reset_kernel_stats(void) {
    int rc = fold_stats();
    g.stats.clear();
    return rc;
}

int ptucker_info(char* buf, int32_t len) {
    if (!buf || len <= 0) return fail(PTUCKER_EINVAL, "bad buffer");
    std::string s = "{";
    char tmp[512];
    {
        std::string jl = "\"core_dims\": [";
        for (int n = 0; n < g.N; ++n) jl += (n ? ", " : "") + std::to_string(g.Jv.j[n]);
        s += jl + "], ";
    }
    int comm_ranks = 0;  // size of the library's NCCL communicator (0: none)
    if (g.comm && ncclCommCount(g.comm, &comm_ranks) != ncclSuccess) comm_ranks = -1;
    snprintf(tmp, sizeof(tmp), "\"cache\": %s, ", g.cache_on ? "true" : "false");
    s += tmp;
    snprintf(tmp, sizeof(tmp), "\"comm_ranks\": %d, \"peers\": %d, \"exchange\": \"%s\", ", comm_ranks, g.npeer,
             g.world == 1 ? "none" : (pushing() ? "push" : (g.comm ? "nccl_allgather" : "none")));
    s += tmp;
    snprintf(tmp, sizeof(tmp),
             "\"inited\": %s, \"N\": %d, \"J\": %d, \"prec\": \"%s\", \"policy\": \"%s\", \"nnz\": %lld, "
             "\"lambda\": %.17g, \"seg_len\": %d, \"rank\": %d, \"world\": %d, \"grid_update\": %d, "
             "\"threads_per_cta\": %d, \"smem_core_bytes\": %d, \"kernel_launches\": %lld, \"tensor_cores\": %s, \"generic\": %s, \"modes\": [",
             g.inited ? "true" : "false", g.N, g.J, g.prec == PTUCKER_F64 ? "f64" : "f32",
             g.prec == PTUCKER_F64 ? "F64" : (policy_l64() == 0 ? "F32-A" : (policy_l64() == 1 ? "F32-B" : (g.N >= 5 && policy_l64() == g.N - 3 ? "F32-C2" : "F32-C"))), (long long)g.nnz, g.lambda, g.seg_len_eff,
             g.rank, g.world, g.grid_upd, kUpdThreads, g.gp_elems * g.esz, (long long)g.launches,
             (g.kern && g.kern != g.kern_alu) ? "true" : "false", g.generic ? "true" : "false");
    s += tmp;
    for (int n = 0; n < g.N; ++n) {
        const ModeIndex& m = g.mi[n];
        snprintf(tmp, sizeof(tmp),
                 "%s{\"I\": %lld, \"rows\": [%lld, %lld], \"segments\": %lld, \"slices\": %lld, \"slots\": %lld, "
                 "\"heavy_rows\": %lld, \"smp\": %d, \"tc_table\": %s, \"seg_len\": %d}",
                 n ? ", " : "", (long long)m.I, (long long)m.r0, (long long)m.r1, (long long)m.nsegments,
                 (long long)m.nslices, (long long)m.nslots, (long long)m.nheavy, g.use_smp ? g.smp[n].kind : 0,
                 m.aux_groups ? "true" : "false", m.seg_len);
        s += tmp;
    }
    s += "]}";
    snprintf(buf, (size_t)len, "%s", s.c_str());
    return (int)s.size() < len ? PTUCKER_OK : fail(PTUCKER_EINVAL, "buffer too small (%zu)", s.size() + 1);
}

int ptucker_debug_trace(long long* out, int32_t n) {
    if (!g.trace || !out || n <= 0) return fail(PTUCKER_EINVAL, "no trace");
    CK(cudaMemcpy(out, g.trace, sizeof(long long) * std::min<int32_t>(n, 8 * 512), cudaMemcpyDeviceToHost));
    return PTUCKER_OK;
}

int ptucker_synchronize(void) {
    int rc = require_init();
    if (rc) return rc;
    return sync_and_check();
}

int ptucker_finalize(void) {
    if (g.inited) {
        cudaStreamSynchronize(S());
        fold_stats();
        if (g.l2_persist_mb != 0) {  // give the L2 set-aside back
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
            cudaCtxResetPersistingL2Cache();
        }
    }
    free_all();
    if (g.comm) {
        ncclCommDestroy(g.comm);
        g.comm = nullptr;
    }
    g.world = 1;
    g.rank = 0;
    g.emu_world = 1;
    g.emu_rank = 0;
    if (g.own_stream && g.stream) cudaStreamDestroy(g.stream);
    g.stream = nullptr;
    g.own_stream = false;
    return PTUCKER_OK;
}

}  // extern "C"
