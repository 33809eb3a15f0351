// DSMEM hand-off latency: CTA 0 and CTA r of a cluster bounce a counter through st.async +
// mbarrier complete_tx (mode 0) or st.shared::cluster + mbarrier.arrive.release.cluster (mode 1).
// Optional background load: the other warps of every CTA run an FMA loop (busy = 1).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_pingpong tools/dsmem_pingpong.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n}"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}

__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, int mode, int busy, long long* out, float* sink) {
  __shared__ uint64_t bar;
  __shared__ float val;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  cl.sync();
  if (tid == 0) {
    const uint32_t lb = smem_u32(&bar);
    const uint32_t rb = mapa(lb, rank ^ 1), rv = mapa(smem_u32(&val), rank ^ 1);
    uint32_t par = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4;" ::"r"(lb) : "memory");
      if (rank == 0 || i > 0) {
        // send
        if (mode == 0) {
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(rv),
                       "r"(i), "r"(rb) : "memory");
        } else {
          asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(rv), "r"(i) : "memory");
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
        }
      }
      while (!try_wait(lb, par)) {
      }
      par ^= 1;
      if (rank == 1 && i == iters - 1) {
        if (mode == 0) {
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(rv),
                       "r"(i), "r"(rb) : "memory");
        } else {
          asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(rv), "r"(i) : "memory");
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
        }
      }
    }
    long long t1 = clock64();
    if (rank == 0) out[0] = (t1 - t0) / iters;
  } else if (busy && tid >= 32) {
    float a = tid, b = 1.0001f;
    for (int i = 0; i < iters * 200; ++i) a = a * b + 0.5f;
    sink[blockIdx.x * blockDim.x + tid] = a;
  }
  cl.sync();
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 1 << 20);
  for (int mode = 0; mode < 2; ++mode)
    for (int busy = 0; busy < 2; ++busy) {
      pingpong<<<2, 512>>>(2000, mode, busy, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("mode %s busy %d: round trip %lld cycles (%s)\n", mode == 0 ? "st.async+complete_tx" : "st+arrive.release",
             busy, h, cudaGetErrorString(e));
    }
  return 0;
}
