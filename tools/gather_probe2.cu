// Random-row gather probe, second edition: where does a warp's row fetch spend
// its time?  Variants of the walk's access pattern (whole 4 KB rows at random
// ids), each on a large region (5.2 GB: HBM + TLB misses) and a small one
// (64 MB: L2-resident), so the LSU path can be told apart from DRAM:
//   ldg<R>     R rows per step through registers (8 LDG.128 per lane per row)
//   pf<G>      bulk L2 prefetch of G rows, then the rows two at a time (ldg<2>)
//   tma<S>     cp.async.bulk rows into a per-warp smem ring of S slots, LDS reads
// Prints GB/s and the time per row per warp.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gp2 tools/gather_probe2.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ unsigned row_id(unsigned w, int it, int r, unsigned n) {
    return hash32(w * 7919u + it * 104729u + r * 31u + 12345u) % n;
}

template <int R>
__global__ void k_ldg(const float4* __restrict__ X, unsigned n, int nv, int iters, float* out) {
    const int lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v[R][8];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float4* row = X + (size_t)row_id(w, it, r, n) * nv;
#pragma unroll
            for (int j = 0; j < 8; ++j) v[r][j] = __ldg(row + lane + 32 * j);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += v[r][j].x + v[r][j].y + v[r][j].z + v[r][j].w;
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    }
    if (acc == 12345.f) out[0] = acc;
}

// G rows per group: bulk L2 prefetch of all of them, then pairs through registers
template <int G>
__global__ void k_pf(const float4* __restrict__ X, unsigned n, int nv, int iters, float* out) {
    const int lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        if (lane < G) {
            const float4* row = X + (size_t)row_id(w, it, lane, n) * nv;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"(nv * 16) : "memory");
        }
        for (int g = 0; g < G; g += 2) {
            float4 v[2][8];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const float4* row = X + (size_t)row_id(w, it, g + r, n) * nv;
#pragma unroll
                for (int j = 0; j < 8; ++j) v[r][j] = __ldg(row + lane + 32 * j);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc += v[r][j].x + v[r][j].y + v[r][j].z + v[r][j].w;
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
                 : "memory");
}

// per-warp ring of S slots (4 KB each); rows stream continuously: slot refilled as soon as consumed
template <int S>
__global__ void k_tma(const float4* __restrict__ X, unsigned n, int nv, int iters, float* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float4* ring = reinterpret_cast<float4*>(smem) + (size_t)wib * S * nv;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)wpb * S * nv * 16) + wib * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int total = iters;  // rows per warp
    if (lane == 0)
        for (int s = 0; s < S && s < total; ++s) {
            mbar_expect(bars + s, nv * 16);
            bulk_g2s(ring + (size_t)s * nv, X + (size_t)row_id(w, s, 0, n) * nv, nv * 16, bars + s);
        }
    float acc = 0.f;
    for (int t = 0; t < total; ++t) {
        const int s = t % S;
        mbar_wait(bars + s, (t / S) & 1);
        const float4* row = ring + (size_t)s * nv;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 v = row[lane + 32 * j];
            acc += v.x + v.y + v.z + v.w;
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        __syncwarp();
        if (lane == 0 && t + S < total) {
            mbar_expect(bars + s, nv * 16);
            bulk_g2s(ring + (size_t)s * nv, X + (size_t)row_id(w, t + S, 0, n) * nv, nv * 16, bars + s);
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

template <class F>
void timeit(const char* name, int sms, int wps, int rows_per_iter, int iters, int nv, F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(4);
    cudaEventRecord(a);
    launch(iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double rows = (double)sms * wps * iters * rows_per_iter;
    cudaError_t e = cudaGetLastError();
    printf("%-10s warps/SM=%2d  %8.1f GB/s  %.3f us/row/warp  (%.2f ms)%s\n", name, wps, rows * nv * 16 / (ms * 1e-3) / 1e9,
           ms * 1e3 / (iters * rows_per_iter), ms, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char** argv) {
    const unsigned nfull = 1281167;
    const int dp = 1024, nv = dp / 4;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float4* X = nullptr;
    float* out = nullptr;
    cudaMalloc(&X, (size_t)nfull * dp * 4);
    cudaMalloc(&out, 4);
    cudaMemset(X, 0, (size_t)nfull * dp * 4);
    for (unsigned n : {nfull, 16384u}) {
        printf("---- region: %u rows (%.0f MB)\n", n, n * 4096.0 / 1e6);
        const int iters = 256;
        for (int wps : {4, 8, 16}) {
            const int blocks = sms * wps / 4;
            timeit("ldg<1>", sms, wps, 1, iters, nv, [&](int it) { k_ldg<1><<<blocks, 128>>>(X, n, nv, it, out); });
            timeit("ldg<2>", sms, wps, 2, iters / 2, nv, [&](int it) { k_ldg<2><<<blocks, 128>>>(X, n, nv, it, out); });
            timeit("pf<8>", sms, wps, 8, iters / 8, nv, [&](int it) { k_pf<8><<<blocks, 128>>>(X, n, nv, it, out); });
        }
        for (int wps : {4, 8, 12, 16}) {
            const int blocks = sms * wps / 4;
            {
                const size_t sm = 4 * 2 * 4096 + 4 * 2 * 8;
                cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                timeit("tma<2>", sms, wps, 1, iters, nv, [&](int it) { k_tma<2><<<blocks, 128, sm>>>(X, n, nv, it, out); });
            }
            if (wps <= 12) {
                const size_t sm = 4 * 4 * 4096 + 4 * 4 * 8;
                cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                timeit("tma<4>", sms, wps, 1, iters, nv, [&](int it) { k_tma<4><<<blocks, 128, sm>>>(X, n, nv, it, out); });
            }
            if (wps <= 4) {
                const size_t sm = 4 * 8 * 4096 + 4 * 8 * 8;
                cudaFuncSetAttribute(k_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                timeit("tma<8>", sms, wps, 1, iters, nv, [&](int it) { k_tma<8><<<blocks, 128, sm>>>(X, n, nv, it, out); });
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
