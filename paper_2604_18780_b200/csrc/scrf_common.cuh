// Shared device helpers for the streaming semi-CRF kernels (sm_100a).
//
// Numerics: every log-domain quantity is carried in
// base 2 (inputs scaled by log2(e) on load, results scaled back by ln 2), so the
// inner loops use the MUFU ex2/lg2 instructions directly. Large, label-dependent
// magnitudes (prefix sums S, running normalisers) are split into a (hi, lo) pair
// of the working type R so that the per-term difference S[t]-S[t-k] keeps
// fp64-level absolute accuracy while the term arithmetic stays in fp32.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace scrf {

namespace cg = cooperative_groups;

constexpr double kLog2e = 1.4426950408889634;
constexpr double kLn2 = 0.6931471805599453;
constexpr double kNegInfRef = -1.0e9;          // reference sentinel (_numerics.py:18)
constexpr double kGuard = kNegInfRef + 1.0;    // reference guard (_numerics.py:59-75)
constexpr double kGuardL2 = kGuard * kLog2e;   // the guard in log2 units
constexpr double kClampLimit = 1.0e6;          // reference CLAMP_LIMIT (_numerics.py:23)

template <typename R>
struct Mth;

template <>
struct Mth<float> {
  static __device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float ninf() { return -CUDART_INF_F; }
  static __device__ __forceinline__ float tiny() { return 1e-30f; }
};

template <>
struct Mth<double> {
  static __device__ __forceinline__ double ex2(double x) { return exp2(x); }
  static __device__ __forceinline__ double lg2(double x) { return log2(x); }
  static __device__ __forceinline__ double ninf() { return -CUDART_INF; }
  static __device__ __forceinline__ double tiny() { return 1e-290; }
};

template <typename R>
struct Vec2;
template <>
struct Vec2<float> {
  using T = float2;
};
template <>
struct Vec2<double> {
  using T = double2;
};

// (hi, lo) split of an fp64 value into the working type.
template <typename R>
__device__ __forceinline__ void split(double v, R& hi, R& lo) {
  hi = (R)v;
  lo = isfinite(v) ? (R)(v - (double)hi) : (R)0;
}

// log-sum-exp partial: value = m + log2(s)
template <typename R>
__device__ __forceinline__ void ms_merge(R& m, R& s, R m2, R s2) {
  R M = fmax(m, m2);
  if (M == Mth<R>::ninf()) {
    m = M;
    s = (R)0;
    return;
  }
  s = s * Mth<R>::ex2(m - M) + s2 * Mth<R>::ex2(m2 - M);
  m = M;
}

template <typename R>
__device__ __forceinline__ R ms_value(R m, R s) {
  return (m == Mth<R>::ninf() || !(s > (R)0)) ? Mth<R>::ninf() : m + Mth<R>::lg2(s);
}

// Reductions over aligned lane groups of width W (power of two <= 32). Each
// butterfly level merges (lower lane, upper lane) in that order in both partners,
// so every lane of the group ends with the bit-identical result.
template <typename R>
__device__ __forceinline__ void group_ms(R& m, R& s, int W) {
  const int lane = threadIdx.x & 31;
  for (int off = W >> 1; off > 0; off >>= 1) {
    R m2 = __shfl_xor_sync(0xffffffffu, m, off, W);
    R s2 = __shfl_xor_sync(0xffffffffu, s, off, W);
    if (lane & off) {
      R tm = m, ts = s;
      m = m2;
      s = s2;
      m2 = tm;
      s2 = ts;
    }
    ms_merge(m, s, m2, s2);
  }
}

template <typename T>
__device__ __forceinline__ T group_sum(T v, int W) {
  for (int off = W >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, W);
  return v;
}

template <typename T>
__device__ __forceinline__ T group_max(T v, int W) {
  for (int off = W >> 1; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off, W));
  return v;
}

// ----------------------------------------------------------------------------
// Cluster exchange without cluster barriers.
//
// Each CTA owns two mbarriers per exchanged vector (one per position parity). A
// producer lane sends its label's value to every CTA of the cluster with
// st.async ... mbarrier::complete_tx (async proxy: no release fence, so the
// sender's in-flight global loads / stores never stall it); the receiving CTA
// arms its barrier with expect_tx(C * sizeof(R)) and all its threads wait on
// the barrier's phase parity. Parity double-buffering is WAR-safe because a peer
// can only send position t+2 after receiving our position t+1, which we publish
// after finishing every read of position t.

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_init(uint32_t a, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity);

// Spin in C++ around try_wait (acquire at cluster scope: the data arrives through
// st.async from peer CTAs). A spin loop written inside one asm block deadlocked for
// clusters of >= 12 CTAs on B200; this form does not.
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  while (!mbar_try(a, parity)) {
  }
}

// bounded wait (debug builds of the sweep): returns false after ~2^spin polls
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void st_async(uint32_t dst, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void st_async(uint32_t dst, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(dst),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}

// One exchanged vector of C values of type T (double-buffered by parity).
template <typename T>
struct Xchg {
  T* buf;          // [2][C] local buffer
  uint64_t* bar;   // [2] local mbarriers
  uint32_t phase;  // bit p = parity of the next wait on bar[p]
  int C;

  __device__ void init(int tid) {
    if (tid == 0) {
      mbar_init(smem_u32(&bar[0]), 1);
      mbar_init(smem_u32(&bar[1]), 1);
      mbar_fence_init();
    }
    phase = 0;
  }
  // one thread per CTA, once per use of parity p, before waiting on it
  __device__ __forceinline__ void arm(int p) { mbar_expect(smem_u32(&bar[p]), (uint32_t)(C * sizeof(T))); }
  // send value v for label c to ranks r = first, first+stride, ... < G
  __device__ __forceinline__ void send(int p, int c, T v, int first, int stride, int G) {
    const uint32_t la = smem_u32(&buf[p * C + c]);
    const uint32_t lb = smem_u32(&bar[p]);
    for (int r = first; r < G; r += stride) st_async(mapa_u32(la, r), v, mapa_u32(lb, r));
  }
  __device__ __forceinline__ const T* wait(int p) {
    mbar_wait(smem_u32(&bar[p]), (phase >> p) & 1u);
    phase ^= (1u << p);
    return buf + p * C;
  }
};

// Launch geometry shared by forward, replay and backward so that replay is a
// bit-identical re-execution of the forward (same label slice, same per-thread
// duration subsets, same reduction trees).
struct Geometry {
  int G;      // CTAs per cluster (label slices)
  int Cgm;    // max labels per CTA = ceil(C / G)
  int TPL;    // threads per label (power of two, >= 1)
  int NT;     // threads per CTA
  int WPL;    // warps per label (TPL / 32, or 1 when TPL <= 32)
  int GW;     // lane-group width for intra-warp reductions = min(TPL, 32)
};

__host__ __device__ inline int label_lo(int rank, int C, int G) { return (int)(((long long)rank * C) / G); }

}  // namespace scrf
