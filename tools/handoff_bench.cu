// Intra-CTA hand-off latency between two warps: named barriers (bar.arrive -> bar.sync),
// a shared-memory flag spin (st.volatile / ld.volatile), and an mbarrier (arrive -> try_wait).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/handoff_bench tools/handoff_bench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void pingpong(int iters, int mode, long long* out) {
  __shared__ volatile int flag[2];
  __shared__ uint64_t mb[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    flag[0] = flag[1] = -1;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(su32(&mb[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(su32(&mb[1])));
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {  // named barriers: warp 0 arrives id 1, warp 1 syncs id 1; back on id 2
      if (warp == 0) {
        asm volatile("bar.arrive 1, 64;" ::: "memory");
        asm volatile("bar.sync 2, 64;" ::: "memory");
      } else {
        asm volatile("bar.sync 1, 64;" ::: "memory");
        asm volatile("bar.arrive 2, 64;" ::: "memory");
      }
    } else if (mode == 1) {  // flag spin
      if (warp == 0) {
        if (lane == 0) flag[0] = i;
        while (flag[1] != i) {
        }
      } else {
        while (flag[0] != i) {
        }
        if (lane == 0) flag[1] = i;
      }
    } else {  // mbarrier, count 32 (one warp), parity = i & 1
      const uint32_t par = i & 1;
      uint32_t ok;
      if (warp == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&mb[0])) : "memory");
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}"
                       : "=r"(ok) : "r"(su32(&mb[1])), "r"(par) : "memory");
        } while (!ok);
      } else {
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}"
                       : "=r"(ok) : "r"(su32(&mb[0])), "r"(par) : "memory");
        } while (!ok);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&mb[1])) : "memory");
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const char* names[] = {"named barrier arrive->sync", "smem flag spin", "mbarrier arrive->try_wait"};
  for (int m = 0; m < 3; ++m) {
    pingpong<<<1, 64>>>(10000, m, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-30s round trip %lld cycles (%s)\n", names[m], h, cudaGetErrorString(e));
  }
  return 0;
}
