// Latency of the building blocks of a Jacobi step on one warp (dependent chains, clock64).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../../paper_1707_05141_b200/csrc rot_latency.cu -o rot_latency
#include <cstdio>
#include "common.cuh"
#include "jacobi_reg.cuh"

using namespace bf;

__global__ void k_rot(double* out, long long* cyc, int iters) {
  double gpp = 1.5 + threadIdx.x * 1e-3, gpq = 0.3, gqq = 0.9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double c, s, t;
    jacobi_rotation_t(gpp, gpq, gqq, c, s, t);
    gpq = 0.3 + 1e-3 * s;  // dependent chain
    gpp = 1.5 + 1e-3 * c;
  }
  long long t1 = clock64();
  out[threadIdx.x] = gpp + gpq;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
}

__global__ void k_shfl(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
}

__global__ void k_lds(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x;
  __syncwarp();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = (int)sm[idx & 31] & 31;
  long long t1 = clock64();
  out[threadIdx.x] = idx;
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
}

__global__ void k_dfma(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
}

__global__ void k_bar(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("bar.sync 1, 64;" ::: "memory");
    x += 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k_rot<<<1, 32>>>(out, cyc, 1000);
    k_shfl<<<1, 32>>>(out, cyc, 1000);
    k_lds<<<1, 32>>>(out, cyc, 1000);
    k_dfma<<<1, 32>>>(out, cyc, 1000);
    k_bar<<<1, 64>>>(out, cyc, 1000);
    cudaDeviceSynchronize();
  }
  printf("{\"rotation_chain_cyc\": %lld, \"shfl64_add_cyc\": %lld, \"lds_dep_cyc\": %lld, \"dfma_dep_cyc\": %lld, "
         "\"bar64_cyc\": %lld}\n", cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
  return 0;
}
