// Pipe-throughput microbenchmarks for the SFU roofline denominator (MUFU.EX2),
// FP32 add, FP64 add, f64->f32 conversion, and a cluster-barrier round trip.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define ITERS 4096
__global__ void k_ex2(float* out, float seed) {
  float a0 = seed + threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < ITERS; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a4)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a5));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a6)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a7));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_fadd(float* out, float seed) {
  float a[8]; for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
  float b = seed * 0.5f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(b));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(double* out, double seed) {
  double a[8]; for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
  double b = seed * 0.5;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("add.f64 %0, %0, %1;" : "+d"(a[j]) : "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_cvt(float* out, double seed) {
  double a[8]; float f[8];
  for (int j = 0; j < 8; ++j) { a[j] = seed + j + threadIdx.x; f[j] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { float x; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(x) : "d"(a[j])); f[j] += x; }
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster(int* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int buf[8];
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) {
      int* peer = cl.map_shared_rank(buf, (cl.block_rank() + 1) % 8);
      peer[cl.block_rank()] = i;
    }
    cl.sync();
    acc += buf[(cl.block_rank() + 7) % 8];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_bar(int* out, int iters) {
  __shared__ int buf[32];
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) buf[threadIdx.x] = i + threadIdx.x;
    __syncthreads();
    acc += buf[(threadIdx.x + 1) & 31];
    __syncthreads();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d}\n", p.name, p.multiProcessorCount, clk_khz);
  int sms = p.multiProcessorCount;
  float* fo; double* dout; int* io;
  cudaMalloc(&fo, sizeof(float) * sms * 8 * 1024); cudaMalloc(&dout, sizeof(double) * sms * 8 * 1024);
  cudaMalloc(&io, sizeof(int) * sms * 8 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  int grid = sms * 4, blk = 512;
  double ops = double(grid) * blk * ITERS * 8;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); k_ex2<<<grid, blk>>>(fo, 0.001f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\": \"ex2.approx.f32\", \"Gops\": %.1f, \"per_sm_per_ns\": %.3f}\n", ops / ms / 1e6, ops / ms / 1e6 / sms);
    cudaEventRecord(a); k_fadd<<<grid, blk>>>(fo, 0.001f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\": \"add.f32\", \"Gops\": %.1f, \"per_sm_per_ns\": %.3f}\n", ops / ms / 1e6, ops / ms / 1e6 / sms);
    cudaEventRecord(a); k_dadd<<<grid, blk>>>(dout, 0.001); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\": \"add.f64\", \"Gops\": %.1f, \"per_sm_per_ns\": %.3f}\n", ops / ms / 1e6, ops / ms / 1e6 / sms);
    cudaEventRecord(a); k_cvt<<<grid, blk>>>(fo, 0.001); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"op\": \"cvt.f32.f64\", \"Gops\": %.1f, \"per_sm_per_ns\": %.3f}\n", ops / ms / 1e6, ops / ms / 1e6 / sms);
  }
  int iters = 100000;
  cudaEventRecord(a); k_cluster<<<8, 128>>>(io, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"op\": \"cluster8 dsmem store + cluster.sync\", \"ns_per_iter\": %.1f, \"err\": \"%s\"}\n", ms * 1e6 / iters, cudaGetErrorString(cudaGetLastError()));
  cudaEventRecord(a); k_bar<<<1, 256>>>(io, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"op\": \"2x __syncthreads (256 thr)\", \"ns_per_iter\": %.1f}\n", ms * 1e6 / iters);
  cudaEventRecord(a); k_bar<<<1, 1024>>>(io, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"op\": \"2x __syncthreads (1024 thr)\", \"ns_per_iter\": %.1f}\n", ms * 1e6 / iters);
  return 0;
}
