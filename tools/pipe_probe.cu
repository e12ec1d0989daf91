// pipe_probe.cu -- per-SM throughput of the arithmetic pipes the row-update
// kernels use (B200, sm_100a): FFMA, FADD, DFMA, cvt.f64.f32 (F2F), integer
// LOP3/IADD3/SHF, and tcgen05.ld (TMEM -> registers).  Each kernel runs many
// independent chains on every SM at full occupancy; throughput is reported in
// thread-operations per SM per clock, with the clock measured in the kernel
// (clock64 over globaltimer).  These numbers are the peaks of the "alu"
// rooflines in bench.py.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_probe tools/pipe_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ void record(unsigned long long* clk, uint64_t c0, uint64_t t0) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = clock64() - c0;
        clk[1] = gtime() - t0;
    }
}

__global__ void k_ffma(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    float a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = fmaf(a[i], s, 0.5f);
    float r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    record(clk, c0, t0);
}

__global__ void k_fadd(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    float a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = a[i] + s;
    float r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    record(clk, c0, t0);
}

__global__ void k_dfma(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    double a[CH];
    const double ds = s;
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = fma(a[i], ds, 0.5);
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)r;
    record(clk, c0, t0);
}

// cvt.f64.f32 feeding a DADD (the DADD is on the fp64 pipe, 4x faster than
// the measured conversion rate, so the loop measures the conversion)
__global__ void k_f2f(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    float f[CH];
    double a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        f[i] = threadIdx.x * 1e-3f + i * s;
        a[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] += (double)f[i];
#pragma unroll
        for (int i = 0; i < CH; ++i) f[i] = __int_as_float(__float_as_int(f[i]) + 1);  // a new value every iteration
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)r;
    record(clk, c0, t0);
}

// baseline of k_f2f without the conversion (DADD + LOP3 only)
__global__ void k_dadd_lop(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    float f[CH];
    double a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        f[i] = threadIdx.x * 1e-3f + i * s;
        a[i] = 0;
    }
    double d[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) d[i] = f[i];
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] += d[i];
#pragma unroll
        for (int i = 0; i < CH; ++i) f[i] = __int_as_float(__float_as_int(f[i]) + 1);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i] + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)r;
    record(clk, c0, t0);
}

// float -> double by integer ops (exact for normal floats): hi = (asr(u,3) & 0x8FFFFFFF) + 0x38000000, lo = u << 29
__global__ void k_f2f_int(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    float f[CH];
    double a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        f[i] = threadIdx.x * 1e-3f + i * s + 1.0f;
        a[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            const uint32_t u = __float_as_uint(f[i]);
            const uint32_t hi = ((uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu) + 0x38000000u;
            const uint32_t lo = u << 29;
            a[i] += __hiloint2double((int)hi, (int)lo);
        }
#pragma unroll
        for (int i = 0; i < CH; ++i) f[i] = __int_as_float(__float_as_int(f[i]) + 1);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)r;
    record(clk, c0, t0);
}

__global__ void k_lop3(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    uint32_t a[CH];
    const uint32_t m = __float_as_uint(s);
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = (a[i] ^ m) & (a[i] | 0x1234u);
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)r;
    record(clk, c0, t0);
}

__global__ void k_iadd3(float* out, float s, unsigned long long* clk) {
    const uint64_t c0 = clock64(), t0 = gtime();
    uint32_t a[CH];
    const uint32_t m = __float_as_uint(s);
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = a[i] + m + 7u;
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)r;
    record(clk, c0, t0);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tcgen05.ld.32x32b.x32 (+ wait) per warp, summing the words (FADD cost 32/ld)
__global__ void k_tmem_ld(float* out, float s, unsigned long long* clk) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t addr = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    const uint64_t c0 = clock64(), t0 = gtime();
    float acc = 0.f;
    for (int it = 0; it < ITERS / 8; ++it) {
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
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) x ^= r[i];
        acc += __uint_as_float(x & 0x3F800000u);
    }
    record(clk, c0, t0);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + s;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

typedef void (*K)(float*, float, unsigned long long*);

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    unsigned long long* clk;
    cudaMalloc(&out, sizeof(float) * nsm * 4 * 1024);
    cudaMalloc(&clk, 16);
    struct T {
        const char* name;
        K k;
        int threads, blocks_per_sm;
        double ops_per_iter;  // thread-ops per loop iteration
        int iters;
    } tests[] = {
        {"ffma", k_ffma, 512, 4, CH, ITERS},
        {"fadd", k_fadd, 512, 4, CH, ITERS},
        {"dfma", k_dfma, 512, 4, CH, ITERS},
        {"f2f.f64.f32 (+dadd)", k_f2f, 512, 4, CH, ITERS},
        {"dadd+lop3 (f2f baseline)", k_dadd_lop, 512, 4, CH, ITERS},
        {"f2f by int ops (+dadd)", k_f2f_int, 512, 4, CH, ITERS},
        {"lop3", k_lop3, 512, 4, 2 * CH, ITERS},
        {"iadd3", k_iadd3, 512, 4, CH, ITERS},
        {"tmem ld x32 words", k_tmem_ld, 256, 1, 32, ITERS / 8},
    };
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (auto& t : tests) {
        const int grid = nsm * t.blocks_per_sm;
        t.k<<<grid, t.threads>>>(out, 1.0001f, clk);  // warm-up
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) t.k<<<grid, t.threads>>>(out, 1.0001f, clk);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        if (e != cudaSuccess) {
            printf("%s: %s\n", t.name, cudaGetErrorString(e));
            return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[2];
        cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
        const double ghz = (double)h[0] / (double)h[1];
        const double ops = (double)grid * t.threads * t.iters * t.ops_per_iter * 5;
        const double per_ns = ops / (ms * 1e6);
        printf("{\"op\": \"%s\", \"thread_ops_per_sm_per_clk\": %.2f, \"sm_ghz\": %.3f, \"tera_ops_per_s\": %.2f}\n", t.name,
               per_ns / (ghz * nsm), ghz, per_ns / 1e3);
    }
    return 0;
}
