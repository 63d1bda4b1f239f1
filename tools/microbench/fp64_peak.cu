// FP64 roofline microbenchmarks for B200 (sm_100a).
// MEASURED_PEAKS.json carries no FP64 entry, so this fixes the FP64 denominator
// for the Jacobi / QR rooflines: DFMA throughput, DMMA (mma.sync m8n8k4 f64)
// throughput, and the latency/throughput of the primitives the Jacobi kernels
// are built from (DFMA chain, 64-bit warp shuffle, DDIV/DSQRT chains, LDS.64).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void shfl_tput(double* out, int iters) {
  double v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_xor_sync(0xffffffffu, v[i], 1 << (i & 3));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void lds_tput(double* out, int iters) {
  __shared__ double sm[8 * 256 + 64];
  for (int i = threadIdx.x; i < 8 * 256 + 64; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s = 0;
  int base = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s += sm[(base + i * 256 + it) & 2047];
  }
  if (s == 12345.678) out[0] = s;
}

// single-warp latency of dependent chains
__global__ void lat_kernel(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // shuffle chain
  t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __shfl_xor_sync(0xffffffffu, x, 1);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // div chain
  t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = a / (x + b);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // sqrt chain
  t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = sqrt(x + b);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // rsqrt chain
  t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = rsqrt(x + b);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // hypot chain
  t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = hypot(1.0, x) * a;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  out[threadIdx.x] = x;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", p.name, p.multiProcessorCount, clk_khz);
  double* d_out;
  long long* d_cyc;
  CK(cudaMalloc(&d_out, 1 << 20));
  CK(cudaMalloc(&d_cyc, 64 * sizeof(long long)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  float ms;
  // DFMA
  {
    int iters = 20000, threads = 256, blocks = sms * 8;
    for (int rep = 0; rep < 2; ++rep) dfma_tput<8><<<blocks, threads>>>(d_out, iters / 10, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_tput<8><<<blocks, threads>>>(d_out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf(", \"dfma_tflops\": %.3f", flops / ms / 1e9);
  }
  // DMMA
  {
    int iters = 4000, threads = 256, blocks = sms * 8;
    for (int rep = 0; rep < 2; ++rep) dmma_tput<<<blocks, threads>>>(d_out, iters / 10);
    cudaEventRecord(e0);
    dmma_tput<<<blocks, threads>>>(d_out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (threads / 32) * blocks;
    printf(", \"dmma_tflops\": %.3f", flops / ms / 1e9);
  }
  // SHFL (64-bit = 2 SHFL each)
  {
    int iters = 10000, threads = 256, blocks = sms * 8;
    shfl_tput<<<blocks, threads>>>(d_out, iters / 10);
    cudaEventRecord(e0);
    shfl_tput<<<blocks, threads>>>(d_out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 8.0 * iters * (threads / 32) * blocks;  // 64-bit warp shuffles
    printf(", \"shfl64_warp_per_ns\": %.3f, \"shfl64_per_sm_per_ns\": %.4f", n / ms / 1e6, n / ms / 1e6 / sms);
  }
  // LDS.64
  {
    int iters = 10000, threads = 256, blocks = sms * 8;
    lds_tput<<<blocks, threads>>>(d_out, iters / 10);
    cudaEventRecord(e0);
    lds_tput<<<blocks, threads>>>(d_out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 8.0 * 8 * iters * threads * (double)blocks;
    printf(", \"lds64_TBps\": %.3f, \"lds64_B_per_sm_per_ns\": %.2f", bytes / ms / 1e9, bytes / ms / 1e6 / sms);
  }
  // latencies
  {
    int iters = 1000;
    lat_kernel<<<1, 32>>>(d_out, d_cyc, 10, 0.999, 1e-3);
    lat_kernel<<<1, 32>>>(d_out, d_cyc, iters, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    long long cyc[8];
    cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    const char* names[6] = {"dfma", "shfl64", "ddiv", "dsqrt", "drsqrt", "hypot"};
    for (int i = 0; i < 6; ++i) printf(", \"lat_%s_cyc\": %.1f", names[i], cyc[i] / (16.0 * iters));
  }
  printf("}\n");
  return 0;
}
