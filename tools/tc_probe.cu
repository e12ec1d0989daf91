// tc_probe.cu -- standalone check of the tcgen05 kind::tf32 path used by the
// tensor-core row-update kernel: K-major SWIZZLE_NONE (interleaved core
// matrices) smem descriptors, instruction descriptor, TMEM alloc/ld, mbarrier
// commit; and the accuracy of 1xTF32 / 3xTF32 against fp64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tools/tc_probe.cu && ./tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, NN = 112, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major interleave layout: element (row r, k) of a [rows x 16] tf32 tile
__device__ __forceinline__ int kmaj_off(int r, int k) { return (((r >> 3) * 4 + (k >> 2)) * 128 + (r & 7) * 16 + (k & 3) * 4) / 4; }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__global__ void k_probe(const float* A, const float* B, float* C, int mode) {
    __shared__ __align__(128) float sA_hi[M * K], sA_lo[M * K], sB_hi[NN * K], sB_lo[NN * K];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    for (int k = 0; k < K; ++k) {
        float a = A[t * K + k];
        if (mode >= 3) {  // raw fp32 as "hi" (the tensor core truncates), lo = a - trunc(a) unrounded
            sA_hi[kmaj_off(t, k)] = a;
            sA_lo[kmaj_off(t, k)] = a - trunc_tf32(a);
        } else {
            float h = to_tf32(a);
            sA_hi[kmaj_off(t, k)] = h;
            sA_lo[kmaj_off(t, k)] = to_tf32(a - h);
        }
    }
    for (int i = t; i < NN * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        float b = B[r * K + k];
        if (mode >= 3) {
            sB_hi[kmaj_off(r, k)] = b;
            sB_lo[kmaj_off(r, k)] = b - trunc_tf32(b);
        } else {
            float h = to_tf32(b);
            sB_hi[kmaj_off(r, k)] = h;
            sB_lo[kmaj_off(r, k)] = to_tf32(b - h);
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    if (t == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const float* As[4] = {sA_lo, sA_hi, sA_lo, sA_hi};
        const float* Bs[4] = {sB_lo, sB_lo, sB_hi, sB_hi};
        const int first = mode == 0 ? 3 : (mode == 1 || mode == 3 ? 1 : 0);
        const int nprod = 4;
        int issued = 0;
        for (int p = first; p < nprod; ++p)
            for (int ks = 0; ks < K / 8; ++ks) {
                uint64_t da = make_desc(smem_u32(As[p]) + ks * 256, 128, 512);
                uint64_t db = make_desc(smem_u32(Bs[p]) + ks * 256, 128, 512);
                uint32_t acc = issued > 0 ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tbase),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
                ++issued;
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
    }
    // wait phase 0
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
                         : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < NN; c0 += 16) {
        uint32_t v[16];
        const uint32_t addr = tbase + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) C[t * NN + c0 + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

int main() {
    std::vector<float> A(M * K), B(NN * K), C(M * NN);
    uint64_t s = 12345;
    auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (float)((s >> 40) * (1.0 / 16777216.0)); };
    for (auto& x : A) x = rnd();
    for (auto& x : B) x = rnd();
    for (int k = 10; k < K; ++k) { for (int r = 0; r < M; ++r) A[r * K + k] = 0; for (int r = 0; r < NN; ++r) B[r * K + k] = 0; }
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 4; ++mode) {
        cudaMemset(dC, 0, C.size() * 4);
        k_probe<<<1, 128>>>(dA, dB, dC, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0, fp32max = 0;
        for (int r = 0; r < M; ++r)
            for (int n = 0; n < NN; ++n) {
                double ref = 0; float f32 = 0;
                for (int k = 0; k < K; ++k) { ref += (double)A[r * K + k] * B[n * K + k]; f32 = fmaf(A[r * K + k], B[n * K + k], f32); }
                maxrel = fmax(maxrel, fabs(C[r * NN + n] - ref) / fabs(ref));
                fp32max = fmax(fp32max, fabs(f32 - ref) / fabs(ref));
            }
        printf("mode %s: max rel err vs fp64 %.3e (sequential fp32 FMA: %.3e); C[0]=%g C[last]=%g\n",
               mode == 3 ? "3xTF32 raw-hi/trunc small-first" : (mode == 2 ? "4xTF32 small-first" : (mode ? "3xTF32 small-first" : "1xTF32")), maxrel, fp32max, C[0], C[M * NN - 1]);
    }
    return 0;
}
