// Dependent-chain latency (cycles per op) of the operations on the semi-CRF critical path.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* cyc, int n) {
  __shared__ float sm[64];
  float v = threadIdx.x * 1e-3f + 1.0f;
  if (threadIdx.x < 64) sm[threadIdx.x] = v;
  __syncthreads();
  long long t0, t1;
  // SHFL.BFLY chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) v += __shfl_xor_sync(0xffffffff, v, 1 + (i & 15));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // LDS chain (address depends on previous value)
  int idx = threadIdx.x & 31;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { float w = sm[idx]; idx = ((int)w + i) & 31; v += w; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // MUFU.EX2 chain
  float e = v * 1e-6f;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(e)); e *= 1e-3f; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // FADD chain
  float f = v;
  t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("add.f32 %0, %0, 0f3F800000;" : "+f"(f));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // DADD chain
  double d = v;
  t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("add.f64 %0, %0, 0d3FF0000000000000;" : "+d"(d));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // redux.sync.max.f32 (sm_100a)
  float r = v;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { float o; asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(o) : "f"(r)); r = o - 1.0f + threadIdx.x * 1e-7f; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // cvt f64->f32 chain
  double dd = d;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { float fx; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(fx) : "d"(dd)); dd = (double)fx + 1.0; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  // clock64 overhead
  t0 = clock64();
  long long acc = 0;
  for (int i = 0; i < n; ++i) acc += clock64();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  out[threadIdx.x] = v + e + f + (float)d + r + (float)dd + (float)(acc & 1);
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64 * 8);
  const char* names[] = {"shfl.bfly+fadd", "lds (dep addr)+fadd", "ex2+fmul", "fadd", "dadd", "redux.max.f32+fadd", "cvt.f32.f64+cvt+dadd", "clock64+add"};
  for (int warps : {1, 4, 12}) {
    k<<<1, 32 * warps>>>(o, c, 2000);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("warps=%d (%s)\n", warps, cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 8; ++i) printf("  %-24s %lld cycles/iter\n", names[i], h[i]);
  }
}
