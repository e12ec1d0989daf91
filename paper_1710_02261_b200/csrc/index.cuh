// index.cuh -- device index of one mode (CSR + SELL-32 segments) and a tiny arena.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace pt {

// Device allocations owned by a context (freed together).
struct DeviceArena {
    std::vector<void*> ptrs;
    // bump mode (the index-build scratch): sub-allocations from a few large chunks that are
    // kept between the builds (release_all only rewinds them; free_chunks returns them) --
    // the per-temporary cudaMalloc / cudaFree of round 2 cost ~8 ms of each c5 mode's build
    // (a stream-ordered pool was as fast in isolation but its first growth inside a process
    // that had freed a previous context took 0.2-0.7 s on some boxes)
    bool bump = false;
    struct Chunk {
        char* base;
        size_t size, used;
    };
    std::vector<Chunk> chunks;
    cudaError_t alloc(void** p, size_t bytes) {
        if (bump) {
            const size_t b = ((bytes > 0 ? bytes : 1) + 255) & ~(size_t)255;
            for (Chunk& c : chunks)
                if (c.size - c.used >= b) {
                    *p = c.base + c.used;
                    c.used += b;
                    return cudaSuccess;
                }
            const size_t sz = b > ((size_t)1 << 30) ? b : ((size_t)1 << 30);
            char* base = nullptr;
            const cudaError_t e = cudaMalloc((void**)&base, sz);
            if (e != cudaSuccess) {
                *p = nullptr;
                return e;
            }
            chunks.push_back({base, sz, b});
            *p = base;
            return cudaSuccess;
        }
        cudaError_t e = cudaMalloc(p, bytes > 0 ? bytes : 1);
        if (e == cudaSuccess) ptrs.push_back(*p);
        else *p = nullptr;
        return e;
    }
    // the caller has synchronised the stream that used the memory
    void release_all() {
        for (void* p : ptrs) cudaFree(p);
        ptrs.clear();
        for (Chunk& c : chunks) c.used = 0;
    }
    void free_chunks() {
        for (Chunk& c : chunks) cudaFree(c.base);
        chunks.clear();
    }
    ~DeviceArena() {
        release_all();
        free_chunks();
    }
};

struct ModeIndex {
    int64_t I = 0;
    // CSR of Omega^(n) over all rows
    int32_t* perm = nullptr;       // [nnz] entry ids sorted by coordinate n (stable)
    int64_t* row_ptr = nullptr;    // [I+1]
    std::vector<int64_t> h_row_ptr;
    // this rank's row block and its SELL-32 segments
    int64_t r0 = 0, r1 = 0;
    int64_t nsegments = 0, nslices = 0, nslots = 0;
    int32_t* slice_len = nullptr;
    int64_t* slice_off = nullptr;
    int32_t* lane_row = nullptr;
    int32_t* lane_len = nullptr;
    int64_t* lane_pidx = nullptr;
    int32_t* lane_pstride = nullptr;
    int32_t* lane_aux = nullptr;     // small-mode index i_s of the segment (SMP table block), else 0
    int64_t Is = 1;                  // rows of the grouping small mode (1 = none)
    bool aux_groups = false;         // lanes in (i_s, length) order, each class padded to 128 lanes
    int32_t* sc[kMaxN] = {nullptr};  // coordinates of the other modes, SELL order
    void* sv = nullptr;              // values, SELL order
    // heavy rows (more than one segment)
    int64_t nheavy = 0, npartial_doubles = 0;
    int64_t hmaxseg = 0;             // most segments of one row (host; set by ptucker_init)
    int64_t hminseg = 0;             // fewest segments of a heavy row (host; 0: no heavy row)
    int seg_len = 0;                 // the segment length S of this mode's index
    int32_t* hrow = nullptr;
    int32_t* hnseg = nullptr;
    int64_t* hpbase = nullptr;
    double* partials = nullptr;
    double* hrec = nullptr;          // [nheavy][PW] summed records (heavy-row finalize scratch)
    int64_t hr0 = 0;                 // first row of this rank's block (seg_done / row_pbase index row - hr0)
    int32_t* seg_done = nullptr;     // [rows of the block] heavy-row segment counters (in-kernel finalize)
    int64_t* row_pbase = nullptr;    // [rows of the block] first partial of a heavy row (else unused)
    int32_t* sid = nullptr;          // [nslots] input entry id per SELL slot (P-Tucker-Cache only)
    std::vector<int64_t> bounds;     // world+1 row-block bounds
};

cudaError_t build_mode_csr(const int32_t* d_coords, int64_t nnz, int N, int n, int64_t I, ModeIndex& mi,
                           DeviceArena& arena, DeviceArena& scratch, cudaStream_t st);
cudaError_t build_mode_sell(const int32_t* d_coords, const void* d_vals, int elem_bytes, int64_t nnz, int N, int n,
                            int J, int S, int64_t r0, int64_t r1, int smode, ModeIndex& mi, DeviceArena& arena,
                            DeviceArena& scratch, cudaStream_t st, bool aux_groups = false, bool with_sid = false);

}  // namespace pt
