// index.cu -- device-side build of the mode-slice index Omega^(n)_{i_n} (P:257,
// P:566) and of the SELL-32 segment layout the update kernel streams.
//
//   1. keys = coords[:, n]; stable LSD radix sort of (key, entry id) -> perm
//      (ties keep input order, reading R25); row_ptr by boundary scan.
//   2. This rank's row block [r0, r1) (nnz-balanced, see ptucker_partition_rows).
//   3. Every row becomes ceil(len/S) segments of <= S entries (S = seg_len;
//      an empty row is one segment of length 0, which solves to a = 0).  Rows
//      with more than one segment are "heavy": their segments write partial
//      (B, c, sum x^2) records that k_heavy_sum / k_heavy_solve reduce in a fixed order.
//   4. Segments are stably sorted by length (descending) and cut into slices
//      of 32 -- one warp per slice, one lane per segment, so lanes of a warp
//      do near-equal work (the paper's load balancing concern).
//   5. Entries are scattered into SELL-32 order: entry e of lane l of slice s
//      at slot slice_off[s] + e*32 + l, so a warp's loads are coalesced.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "index.cuh"
#include "internal.cuh"
#include "kernels.cuh"

namespace pt {

__global__ void k_extract_col(const int32_t* coords, int64_t nnz, int N, int n, int32_t* keys, int32_t* iota) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = coords[e * N + n];
        iota[e] = (int32_t)e;
    }
}

void launch_extract_col(const int32_t* coords, int64_t nnz, int N, int n, int32_t* keys, int32_t* iota,
                        cudaStream_t st) {
    int grid = (int)((nnz + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_extract_col<<<grid, 256, 0, st>>>(coords, nnz, N, n, keys, iota);
}

__global__ void k_iota(int32_t* out, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = (int32_t)e;
}

static int grid_for(int64_t n);

// row_ptr[i] = first position whose key >= i (sorted keys); row_ptr[I] = nnz.
__global__ void k_row_ptr(const int32_t* sk, int64_t nnz, int64_t I, int64_t* row_ptr) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = (e == 0) ? -1 : sk[e - 1];
        const int64_t cur = (e == nnz) ? I : sk[e];
        for (int64_t r = prev + 1; r <= cur; ++r) row_ptr[r] = e;
    }
}

void launch_row_ptr(const int32_t* sorted_keys, int64_t nnz, int64_t I, int64_t* row_ptr, cudaStream_t st) {
    int grid = (int)((nnz + 256) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_row_ptr<<<grid, 256, 0, st>>>(sorted_keys, nnz, I, row_ptr);
}

// Segments are cut inside "groups": a group is a row (Is = 1) or, for a mode
// updated with a small-mode table, a (row, i_s) pair, so that
// every segment has one i_s and a warp's lanes mostly share one table block.
// Per group of the block: number of segments (an empty ROW keeps one empty
// segment in its first group, which solves to a = 0).
__global__ void k_group_count(const int64_t* group_ptr, int64_t g0, int64_t ngroups, int64_t Is, int S,
                              int64_t* nseg_g) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ngroups; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t G = g0 + t;
        const int64_t len = group_ptr[G + 1] - group_ptr[G];
        const int64_t row = G / Is;
        const bool first = (G % Is) == 0;
        const int64_t row_len = group_ptr[(row + 1) * Is] - group_ptr[row * Is];
        nseg_g[t] = len > 0 ? (len + S - 1) / S : ((first && row_len == 0) ? 1 : 0);
    }
}

// Per row of the block: segments of the row (its groups are contiguous), heavy flag.
__global__ void k_row_count(const int64_t* seg_start_g, int64_t nrows, int64_t Is, int64_t* nseg_r, int64_t* hflag,
                            int64_t* hseg) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ns = seg_start_g[(t + 1) * Is] - seg_start_g[t * Is];
        nseg_r[t] = ns;
        hflag[t] = ns > 1 ? 1 : 0;
        hseg[t] = ns > 1 ? ns : 0;
    }
}

__global__ void k_heavy_list(int64_t r0, int64_t nrows, int PW, const int64_t* nseg_r, const int64_t* hidx,
                             const int64_t* hbase, int32_t* hrow, int32_t* hnseg, int64_t* hpbase,
                             int64_t* row_pbase) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows; t += (int64_t)gridDim.x * blockDim.x) {
        if (nseg_r[t] > 1) {
            hrow[hidx[t]] = (int32_t)(r0 + t);
            hnseg[hidx[t]] = (int32_t)nseg_r[t];
            hpbase[hidx[t]] = hbase[t] * PW;
        }
        row_pbase[t] = nseg_r[t] > 1 ? hbase[t] * PW : -1;
    }
}

__global__ void k_group_fill(const int64_t* group_ptr, int64_t g0, int64_t ngroups, int64_t Is, int S, int PW,
                             const int64_t* seg_start_g, const int64_t* nseg_r, const int64_t* hbase, int32_t* seg_row,
                             int64_t* seg_src, int32_t* seg_aux, int32_t* seg_len, uint32_t* seg_key,
                             int64_t* seg_pidx, int32_t* seg_pstride) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ngroups; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t G = g0 + t;
        const int64_t len = group_ptr[G + 1] - group_ptr[G];
        const int64_t rl = t / Is;                       // row index within the block
        const int64_t ns = seg_start_g[t + 1] - seg_start_g[t];
        const int64_t nsr = nseg_r[rl];
        const bool heavy = nsr > 1;
        for (int64_t s = 0; s < ns; ++s) {
            const int64_t sid = seg_start_g[t] + s;
            const int64_t in_row = sid - seg_start_g[rl * Is];
            const int64_t l = len - s * S < S ? len - s * S : S;
            seg_row[sid] = (int32_t)(G / Is);
            seg_src[sid] = group_ptr[G] + s * S;
            seg_aux[sid] = (int32_t)(G % Is);
            seg_len[sid] = (int32_t)(l > 0 ? l : 0);
            seg_key[sid] = (uint32_t)(S - (l > 0 ? l : 0));  // ascending key = descending length
            seg_pidx[sid] = heavy ? hbase[rl] * PW + in_row : -1;
            seg_pstride[sid] = heavy ? (int32_t)nsr : 0;
        }
    }
}

__global__ void k_slices(const int32_t* order, int64_t nseg, int64_t nslices, const int32_t* seg_row,
                         const int64_t* seg_src, const int32_t* seg_aux, const int32_t* seg_len,
                         const int64_t* seg_pidx, const int32_t* seg_pstride, int32_t* slice_len,
                         int64_t* slice_slots, int32_t* lane_row, int32_t* lane_len, int64_t* lane_pidx,
                         int32_t* lane_pstride, int64_t* lane_src, int32_t* lane_aux) {
    const int64_t total = nslices * 32;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        if (t < nseg) {
            const int32_t sid = order[t];
            lane_row[t] = seg_row[sid];
            lane_len[t] = seg_len[sid];
            lane_pidx[t] = seg_pidx[sid];
            lane_pstride[t] = seg_pstride[sid];
            lane_src[t] = seg_src[sid];
            lane_aux[t] = seg_aux[sid];
        } else {
            lane_row[t] = -1;
            lane_len[t] = 0;
            lane_pidx[t] = -1;
            lane_pstride[t] = 0;
            lane_src[t] = 0;
            lane_aux[t] = 0;
        }
        if ((t & 31) == 0) {
            const int32_t l = (t < nseg) ? seg_len[order[t]] : 0;
            slice_len[t >> 5] = l;
            slice_slots[t >> 5] = (int64_t)l * 32;
        }
    }
}

template <typename TS>
__global__ void k_sell_fill(int64_t nslices, const int64_t* slice_off, const int32_t* lane_row,
                            const int32_t* lane_len, const int64_t* lane_src, const int32_t* perm,
                            const int32_t* coords, const TS* vals, int N, int n, int32_t* const* sc, TS* sv,
                            int32_t* sid) {
    const int64_t total = nslices * 32;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t row = lane_row[t];
        if (row < 0) continue;
        const int32_t len = lane_len[t];
        const int64_t src0 = lane_src[t];
        const int64_t dst0 = slice_off[t >> 5] + (t & 31);
        // four entries at a time: their entry ids, then all their loads, then the stores (the
        // stores could alias the loads as far as the compiler knows: one entry per iteration
        // serialised two dependent DRAM latencies)
        constexpr int U = 4;
        for (int32_t e0 = 0; e0 < len; e0 += U) {
            int64_t src[U];
#pragma unroll
            for (int u = 0; u < U; ++u) src[u] = e0 + u < len ? __ldg(perm + src0 + e0 + u) : -1;
            int32_t cv[U][kMaxN];
            TS xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (src[u] < 0) continue;
                int l = 0;
                for (int m = 0; m < N; ++m) {
                    if (m == n) continue;
                    cv[u][l++] = __ldg(coords + src[u] * N + m);
                }
                xv[u] = __ldg(vals + src[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (src[u] < 0) continue;
                const int64_t dst = dst0 + (int64_t)(e0 + u) * 32;
                for (int l = 0; l < N - 1; ++l) sc[l][dst] = cv[u][l];
                sv[dst] = xv[u];
                if (sid) sid[dst] = (int32_t)src[u];  // input entry id (P-Tucker-Cache: the row of Pres)
            }
        }
    }
}

__global__ void k_composite_key(const int32_t* coords, int64_t nnz, int N, int n, int s, int64_t Is, uint32_t* keys,
                                int32_t* iota) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = (uint32_t)((int64_t)coords[e * N + n] * Is + coords[e * N + s]);
        iota[e] = (int32_t)e;
    }
}

__global__ void k_group_ptr(const uint32_t* sk, int64_t nnz, int64_t G, int64_t* gp) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = (e == 0) ? -1 : (int64_t)sk[e - 1];
        const int64_t cur = (e == nnz) ? G : (int64_t)sk[e];
        for (int64_t r = prev + 1; r <= cur; ++r) gp[r] = e;
    }
}

static int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (int)g;
}

#define IB_CHECK(x)                                  \
    do {                                             \
        cudaError_t e_ = (x);                        \
        if (e_ != cudaSuccess) return e_;            \
    } while (0)

template <typename T>
static cudaError_t dalloc(T** p, int64_t n, DeviceArena& arena) {
    return arena.alloc((void**)p, (size_t)(n > 0 ? n : 1) * sizeof(T));
}

cudaError_t build_mode_csr(const int32_t* d_coords, int64_t nnz, int N, int n, int64_t I, ModeIndex& mi,
                           DeviceArena& arena, DeviceArena& scratch, cudaStream_t st) {
    int32_t *keys = nullptr, *keys_sorted = nullptr, *iota = nullptr;
    IB_CHECK(dalloc(&keys, nnz, scratch));
    IB_CHECK(dalloc(&keys_sorted, nnz, scratch));
    IB_CHECK(dalloc(&iota, nnz, scratch));
    IB_CHECK(dalloc(&mi.perm, nnz, arena));
    IB_CHECK(dalloc(&mi.row_ptr, I + 1, arena));
    launch_extract_col(d_coords, nnz, N, n, keys, iota, st);
    int bits = 1;
    while ((int64_t(1) << bits) < I) ++bits;
    size_t tb = 0;
    IB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_sorted, iota, mi.perm, (int)nnz, 0, bits, st));
    void* tmp = nullptr;
    IB_CHECK(scratch.alloc(&tmp, tb));
    IB_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_sorted, iota, mi.perm, (int)nnz, 0, bits, st));
    launch_row_ptr(keys_sorted, nnz, I, mi.row_ptr, st);
    mi.I = I;
    mi.h_row_ptr.resize((size_t)I + 1);
    IB_CHECK(cudaMemcpyAsync(mi.h_row_ptr.data(), mi.row_ptr, sizeof(int64_t) * (size_t)(I + 1),
                             cudaMemcpyDeviceToHost, st));
    IB_CHECK(cudaStreamSynchronize(st));
    scratch.release_all();
    return cudaSuccess;
}

template <typename T>
static cudaError_t exclusive_sum(const T* in, T* out, int64_t n, DeviceArena& scratch, cudaStream_t st) {
    size_t tb = 0;
    IB_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, st));
    void* tmp = nullptr;
    IB_CHECK(scratch.alloc(&tmp, tb));
    IB_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, (int)n, st));
    return cudaSuccess;
}

// aux-major segment order (tensor-core table kernel): key = (i_s, descending length), the
// empty segments of empty rows last; per-class counts for the padded lane layout.
__global__ void k_aux_key(int64_t nS, const int32_t* seg_aux, const int32_t* seg_len, int64_t Is, int S,
                          uint32_t* seg_key) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nS; t += (int64_t)gridDim.x * blockDim.x) {
        const int l = seg_len[t];
        seg_key[t] = l == 0 ? (uint32_t)(Is * (S + 1)) : (uint32_t)(seg_aux[t] * (S + 1) + (S - l));
    }
}
__global__ void k_class_count(int64_t nS, const int32_t* seg_aux, const int32_t* seg_len, int64_t Is,
                              unsigned long long* cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nS; t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + (seg_len[t] == 0 ? Is : seg_aux[t]), 1ull);
}
// Lanes of the padded aux-major layout: class a occupies lanes [ps[a], ps[a+1]) (its count
// rounded up to 128 = one group of 4 slices, so no group spans two classes; the empty class
// last, unpadded); real lanes take sorted positions cs[a] + r, the rest are pad lanes.
__global__ void k_slices_aux(const int32_t* order, int64_t nslices, int nclass, const int64_t* ps, const int64_t* cs,
                             const int64_t* cnt, const int32_t* seg_row, const int64_t* seg_src, const int32_t* seg_aux,
                             const int32_t* seg_len, const int64_t* seg_pidx, const int32_t* seg_pstride,
                             int32_t* slice_len, int64_t* slice_slots, int32_t* lane_row, int32_t* lane_len,
                             int64_t* lane_pidx, int32_t* lane_pstride, int64_t* lane_src, int32_t* lane_aux) {
    const int64_t total = nslices * 32;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int a = 0;
        while (a + 1 < nclass && t >= ps[a + 1]) ++a;
        const int64_t r = t - ps[a];
        int32_t l = 0;
        if (r < cnt[a] && t < ps[nclass]) {
            const int32_t sid = order[cs[a] + r];
            l = seg_len[sid];
            lane_row[t] = seg_row[sid];
            lane_len[t] = l;
            lane_pidx[t] = seg_pidx[sid];
            lane_pstride[t] = seg_pstride[sid];
            lane_src[t] = seg_src[sid];
            lane_aux[t] = seg_aux[sid];
        } else {
            lane_row[t] = -1;
            lane_len[t] = 0;
            lane_pidx[t] = -1;
            lane_pstride[t] = 0;
            lane_src[t] = 0;
            lane_aux[t] = a < nclass - 1 ? a : 0;  // the class's table block (pad lanes of a group)
        }
        if ((t & 31) == 0) {
            slice_len[t >> 5] = l;
            slice_slots[t >> 5] = (int64_t)l * 32;
        }
    }
}

cudaError_t build_mode_sell(const int32_t* d_coords, const void* d_vals, int elem_bytes, int64_t nnz, int N, int n,
                            int J, int S, int64_t r0, int64_t r1, int smode, ModeIndex& mi, DeviceArena& arena,
                            DeviceArena& scratch, cudaStream_t st, bool aux_groups, bool with_sid) {
    const int PW = rec_width(J);
    const int64_t nrows = r1 - r0;
    // PTUCKER_DEBUG=2: phase times of this function on stderr (synchronising)
    const bool dbg = getenv("PTUCKER_DEBUG") && getenv("PTUCKER_DEBUG")[0] == '2';
    auto t_last = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[ptucker]   sell %-24s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    mi.r0 = r0;
    mi.r1 = r1;
    // ---- groups: rows, or (row, i_s) pairs for a small-mode table ----
    const int64_t Is = smode >= 0 ? mi.Is : 1;
    const int64_t* group_ptr = mi.row_ptr;
    const int32_t* perm = mi.perm;
    if (smode >= 0) {
        uint32_t *k_in = nullptr, *k_out = nullptr;
        int32_t *iota = nullptr, *perm2 = nullptr;
        int64_t* gptr = nullptr;
        IB_CHECK(dalloc(&k_in, nnz, scratch));
        IB_CHECK(dalloc(&k_out, nnz, scratch));
        IB_CHECK(dalloc(&iota, nnz, scratch));
        IB_CHECK(dalloc(&perm2, nnz, scratch));
        IB_CHECK(dalloc(&gptr, mi.I * Is + 1, scratch));
        k_composite_key<<<grid_for(nnz), 256, 0, st>>>(d_coords, nnz, N, n, smode, Is, k_in, iota);
        int bits = 1;
        while ((int64_t(1) << bits) < mi.I * Is) ++bits;
        size_t tb = 0;
        IB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, iota, perm2, (int)nnz, 0, bits, st));
        void* tmp = nullptr;
        IB_CHECK(scratch.alloc(&tmp, tb));
        IB_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, iota, perm2, (int)nnz, 0, bits, st));
        k_group_ptr<<<grid_for(nnz + 1), 256, 0, st>>>(k_out, nnz, mi.I * Is, gptr);
        group_ptr = gptr;
        perm = perm2;
    }
    lap("groups (small-mode sort)");
    const int64_t g0 = r0 * Is, ngroups = nrows * Is;
    // ---- 3. segments ----
    int64_t *nseg_g = nullptr, *seg_start_g = nullptr, *nseg_r = nullptr, *hflag = nullptr, *hseg = nullptr,
            *hidx = nullptr, *hbase = nullptr;
    IB_CHECK(dalloc(&nseg_g, ngroups + 1, scratch));
    IB_CHECK(dalloc(&seg_start_g, ngroups + 1, scratch));
    IB_CHECK(dalloc(&nseg_r, nrows + 1, scratch));
    IB_CHECK(dalloc(&hflag, nrows + 1, scratch));
    IB_CHECK(dalloc(&hseg, nrows + 1, scratch));
    IB_CHECK(dalloc(&hidx, nrows + 1, scratch));
    IB_CHECK(dalloc(&hbase, nrows + 1, scratch));
    IB_CHECK(cudaMemsetAsync(nseg_g, 0, sizeof(int64_t) * (ngroups + 1), st));
    IB_CHECK(cudaMemsetAsync(nseg_r, 0, sizeof(int64_t) * (nrows + 1), st));
    IB_CHECK(cudaMemsetAsync(hflag, 0, sizeof(int64_t) * (nrows + 1), st));
    IB_CHECK(cudaMemsetAsync(hseg, 0, sizeof(int64_t) * (nrows + 1), st));
    if (ngroups > 0) k_group_count<<<grid_for(ngroups), 256, 0, st>>>(group_ptr, g0, ngroups, Is, S, nseg_g);
    IB_CHECK(exclusive_sum(nseg_g, seg_start_g, ngroups + 1, scratch, st));
    if (nrows > 0) k_row_count<<<grid_for(nrows), 256, 0, st>>>(seg_start_g, nrows, Is, nseg_r, hflag, hseg);
    IB_CHECK(exclusive_sum(hflag, hidx, nrows + 1, scratch, st));
    IB_CHECK(exclusive_sum(hseg, hbase, nrows + 1, scratch, st));
    int64_t tot[3];
    IB_CHECK(cudaMemcpyAsync(&tot[0], seg_start_g + ngroups, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IB_CHECK(cudaMemcpyAsync(&tot[1], hidx + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IB_CHECK(cudaMemcpyAsync(&tot[2], hbase + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IB_CHECK(cudaStreamSynchronize(st));
    const int64_t nS = tot[0];
    mi.nheavy = tot[1];
    mi.npartial_doubles = tot[2] * PW;
    mi.nsegments = nS;

    lap("segment counts");
    int32_t *seg_row, *seg_aux, *seg_len, *seg_pstride;
    int64_t *seg_src, *seg_pidx;
    uint32_t *seg_key, *seg_key_sorted;
    int32_t *seg_iota, *order;
    IB_CHECK(dalloc(&seg_row, nS, scratch));
    IB_CHECK(dalloc(&seg_aux, nS, scratch));
    IB_CHECK(dalloc(&seg_len, nS, scratch));
    IB_CHECK(dalloc(&seg_pstride, nS, scratch));
    IB_CHECK(dalloc(&seg_src, nS, scratch));
    IB_CHECK(dalloc(&seg_pidx, nS, scratch));
    IB_CHECK(dalloc(&seg_key, nS, scratch));
    IB_CHECK(dalloc(&seg_key_sorted, nS, scratch));
    IB_CHECK(dalloc(&seg_iota, nS, scratch));
    IB_CHECK(dalloc(&order, nS, scratch));
    IB_CHECK(dalloc(&mi.hrow, mi.nheavy, arena));
    IB_CHECK(dalloc(&mi.hnseg, mi.nheavy, arena));
    IB_CHECK(dalloc(&mi.hpbase, mi.nheavy, arena));
    IB_CHECK(dalloc(&mi.partials, mi.npartial_doubles, arena));
    IB_CHECK(dalloc(&mi.hrec, mi.nheavy * PW, arena));
    mi.hr0 = r0;
    if (mi.nheavy > 0) {
        IB_CHECK(dalloc(&mi.seg_done, nrows, arena));
        IB_CHECK(dalloc(&mi.row_pbase, nrows, arena));
        IB_CHECK(cudaMemsetAsync(mi.seg_done, 0, sizeof(int32_t) * nrows, st));
    }
    if (nrows > 0 && mi.nheavy > 0)
        k_heavy_list<<<grid_for(nrows), 256, 0, st>>>(r0, nrows, PW, nseg_r, hidx, hbase, mi.hrow, mi.hnseg, mi.hpbase,
                                                      mi.row_pbase);
    if (ngroups > 0)
        k_group_fill<<<grid_for(ngroups), 256, 0, st>>>(group_ptr, g0, ngroups, Is, S, PW, seg_start_g, nseg_r, hbase,
                                                        seg_row, seg_src, seg_aux, seg_len, seg_key, seg_pidx,
                                                        seg_pstride);
    lap("segment fill + allocs");
    // ---- 4. stable sort of segments by length (descending); aux-major when requested ----
    aux_groups = aux_groups && smode >= 0;
    if (aux_groups && nS > 0) k_aux_key<<<grid_for(nS), 256, 0, st>>>(nS, seg_aux, seg_len, Is, S, seg_key);
    {
        if (nS > 0) k_iota<<<grid_for(nS), 256, 0, st>>>(seg_iota, nS);
        int bits = 1;
        const int64_t kmax = aux_groups ? Is * (S + 1) : S;
        while ((int64_t(1) << bits) <= kmax) ++bits;
        size_t tb = 0;
        IB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, seg_key, seg_key_sorted, seg_iota, order, (int)nS, 0,
                                                 bits, st));
        void* tmp = nullptr;
        IB_CHECK(scratch.alloc(&tmp, tb));
        IB_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, seg_key, seg_key_sorted, seg_iota, order, (int)nS, 0, bits,
                                                 st));
    }
    lap("segment sort");
    // padded class layout (aux_groups): counts -> host -> lane offsets
    const int nclass = (int)Is + 1;
    std::vector<int64_t> h_cnt(nclass, 0), h_cs(nclass + 1, 0), h_ps(nclass + 1, 0);
    int64_t *d_ps = nullptr, *d_cs = nullptr, *d_cnt = nullptr;
    if (aux_groups) {
        unsigned long long* cnt_u = nullptr;
        IB_CHECK(dalloc(&cnt_u, nclass, scratch));
        IB_CHECK(cudaMemsetAsync(cnt_u, 0, sizeof(unsigned long long) * nclass, st));
        if (nS > 0) k_class_count<<<grid_for(nS), 256, 0, st>>>(nS, seg_aux, seg_len, Is, cnt_u);
        IB_CHECK(cudaMemcpyAsync(h_cnt.data(), cnt_u, sizeof(int64_t) * nclass, cudaMemcpyDeviceToHost, st));
        IB_CHECK(cudaStreamSynchronize(st));
        for (int a = 0; a < nclass; ++a) {
            h_cs[a + 1] = h_cs[a] + h_cnt[a];
            h_ps[a + 1] = h_ps[a] + (a < nclass - 1 ? (h_cnt[a] + 127) / 128 * 128 : h_cnt[a]);
        }
        IB_CHECK(dalloc(&d_ps, nclass + 1, scratch));
        IB_CHECK(dalloc(&d_cs, nclass + 1, scratch));
        IB_CHECK(dalloc(&d_cnt, nclass, scratch));
        IB_CHECK(cudaMemcpyAsync(d_ps, h_ps.data(), sizeof(int64_t) * (nclass + 1), cudaMemcpyHostToDevice, st));
        IB_CHECK(cudaMemcpyAsync(d_cs, h_cs.data(), sizeof(int64_t) * (nclass + 1), cudaMemcpyHostToDevice, st));
        IB_CHECK(cudaMemcpyAsync(d_cnt, h_cnt.data(), sizeof(int64_t) * nclass, cudaMemcpyHostToDevice, st));
    }
    mi.nslices = aux_groups ? (h_ps[nclass] + 31) / 32 : (nS + 31) / 32;
    mi.aux_groups = aux_groups;
    const int64_t nlanes = mi.nslices * 32;
    int64_t *slice_slots = nullptr, *lane_src = nullptr;
    IB_CHECK(dalloc(&slice_slots, mi.nslices + 1, scratch));
    IB_CHECK(dalloc(&lane_src, nlanes, scratch));
    IB_CHECK(dalloc(&mi.slice_len, mi.nslices, arena));
    IB_CHECK(dalloc(&mi.slice_off, mi.nslices + 1, arena));
    IB_CHECK(dalloc(&mi.lane_row, nlanes, arena));
    IB_CHECK(dalloc(&mi.lane_len, nlanes, arena));
    IB_CHECK(dalloc(&mi.lane_pidx, nlanes, arena));
    IB_CHECK(dalloc(&mi.lane_pstride, nlanes, arena));
    IB_CHECK(dalloc(&mi.lane_aux, nlanes, arena));
    IB_CHECK(cudaMemsetAsync(slice_slots, 0, sizeof(int64_t) * (mi.nslices + 1), st));
    if (nlanes > 0 && aux_groups)
        k_slices_aux<<<grid_for(nlanes), 256, 0, st>>>(order, mi.nslices, nclass, d_ps, d_cs, d_cnt, seg_row, seg_src,
                                                       seg_aux, seg_len, seg_pidx, seg_pstride, mi.slice_len,
                                                       slice_slots, mi.lane_row, mi.lane_len, mi.lane_pidx,
                                                       mi.lane_pstride, lane_src, mi.lane_aux);
    else if (nlanes > 0)
        k_slices<<<grid_for(nlanes), 256, 0, st>>>(order, nS, mi.nslices, seg_row, seg_src, seg_aux, seg_len, seg_pidx,
                                                   seg_pstride, mi.slice_len, slice_slots, mi.lane_row, mi.lane_len,
                                                   mi.lane_pidx, mi.lane_pstride, lane_src, mi.lane_aux);
    IB_CHECK(exclusive_sum(slice_slots, mi.slice_off, mi.nslices + 1, scratch, st));
    IB_CHECK(cudaMemcpyAsync(&mi.nslots, mi.slice_off + mi.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    IB_CHECK(cudaStreamSynchronize(st));
    lap("slices");
    // ---- 5. SELL scatter ----
    for (int k = 0; k < N - 1; ++k) {
        IB_CHECK(dalloc(&mi.sc[k], mi.nslots, arena));
        IB_CHECK(cudaMemsetAsync(mi.sc[k], 0, sizeof(int32_t) * (size_t)(mi.nslots > 0 ? mi.nslots : 1), st));
    }
    IB_CHECK(arena.alloc(&mi.sv, (size_t)(mi.nslots > 0 ? mi.nslots : 1) * elem_bytes));
    IB_CHECK(cudaMemsetAsync(mi.sv, 0, (size_t)(mi.nslots > 0 ? mi.nslots : 1) * elem_bytes, st));
    int32_t** d_sc = nullptr;
    IB_CHECK(dalloc(&d_sc, kMaxN, scratch));
    IB_CHECK(cudaMemcpyAsync(d_sc, mi.sc, sizeof(int32_t*) * kMaxN, cudaMemcpyHostToDevice, st));
    if (with_sid) {
        IB_CHECK(dalloc(&mi.sid, mi.nslots, arena));
        IB_CHECK(cudaMemsetAsync(mi.sid, 0, sizeof(int32_t) * (size_t)(mi.nslots > 0 ? mi.nslots : 1), st));
    }
    if (nlanes > 0) {
        if (elem_bytes == 8)
            k_sell_fill<double><<<grid_for(nlanes), 256, 0, st>>>(mi.nslices, mi.slice_off, mi.lane_row, mi.lane_len,
                                                                  lane_src, perm, d_coords, (const double*)d_vals, N, n,
                                                                  d_sc, (double*)mi.sv, mi.sid);
        else
            k_sell_fill<float><<<grid_for(nlanes), 256, 0, st>>>(mi.nslices, mi.slice_off, mi.lane_row, mi.lane_len,
                                                                 lane_src, perm, d_coords, (const float*)d_vals, N, n,
                                                                 d_sc, (float*)mi.sv, mi.sid);
    }
    IB_CHECK(cudaGetLastError());
    lap("SELL scatter");
    IB_CHECK(cudaStreamSynchronize(st));
    scratch.release_all();
    lap("scratch release");
    return cudaSuccess;
}

}  // namespace pt
