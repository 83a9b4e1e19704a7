// Random-row gather probe: the access pattern of the beam walk's fp32 screens
// (warp-cooperative reads of whole 4 KB rows at random ids from a 5.2 GB point
// matrix), measured alone.  Each warp reads R rows at a time (R x 8 LDG.128 per
// lane in flight), reduces them, and moves on; grid = SMs x warps-per-SM.
// Prints GB/s of row bytes for each (rows in flight, warps per SM).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gather_probe tools/gather_probe.cu
//   /tmp/gather_probe [n_rows=1281167] [dp=1024]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int R>
__global__ void gather(const float4* __restrict__ X, int n, int nv, int iters, float* out) {
    const int lane = threadIdx.x & 31;
    const unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v[R][8];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const unsigned id = hash32(w * 7919u + it * 104729u + r * 31u) % (unsigned)n;
            const float4* row = X + (size_t)id * nv;
#pragma unroll
            for (int j = 0; j < 8; ++j) v[r][j] = __ldg(row + lane + 32 * j);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += v[r][j].x + v[r][j].y + v[r][j].z + v[r][j].w;
        // a short dependent phase between row groups, as the walk has
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    }
    if (acc == 12345.f) out[0] = acc;
}

template <int R>
void run(const float4* X, int n, int nv, int sms, int wps, float* out) {
    const int threads = 128;
    const int warps = sms * wps;
    const int blocks = warps / 4;
    const int iters = 64;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<R><<<blocks, threads>>>(X, n, nv, 4, out);
    cudaEventRecord(a);
    gather<R><<<blocks, threads>>>(X, n, nv, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)warps * iters * R * nv * 16.0;
    printf("rows_in_flight=%d warps_per_sm=%2d  %8.1f GB/s  (%.3f ms)\n", R, wps, bytes / (ms * 1e-3) / 1e9, ms);
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 1281167;
    const int dp = argc > 2 ? atoi(argv[2]) : 1024;
    const int nv = dp / 4;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float4* X = nullptr;
    float* out = nullptr;
    cudaMalloc(&X, (size_t)n * dp * 4);
    cudaMalloc(&out, 4);
    cudaMemset(X, 0, (size_t)n * dp * 4);
    for (int wps : {8, 16, 24, 32}) {
        run<1>(X, n, nv, sms, wps, out);
        run<2>(X, n, nv, sms, wps, out);
        if (wps <= 16) run<4>(X, n, nv, sms, wps, out);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
