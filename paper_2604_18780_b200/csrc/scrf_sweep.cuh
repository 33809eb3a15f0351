// Streaming semi-CRF message sweeps on B200 (sm_100a): the alpha (forward) and the
// beta (backward) recursions of the reference's hot path,
//   streaming_forward  (pkg/src/streamcrf/streaming.py:155-229)  -> direction 0
//   streaming_backward (pkg/src/streamcrf/streaming.py:264-408)  -> direction 1 (beta part)
// in the exact factorised form:
//   alpha:  Y[t,c] = alpha[t,c] = LSE_k (gamma[t-k,c] + h[t-k,k,c]),  X[t,c] = gamma[t,c] = LSE_c' (alpha[t,c'] + T[c',c])
//   beta:   Y[t,c] = delta[t,c] = LSE_k (h[t,k,c] + beta[t+k,c]),     X[t,c'] = beta[t,c'] = LSE_c (T[c',c] + delta[t,c])
// Both are one generic recursion over a sweep position p (alpha: t = p, beta: t = L - p):
//   r[p,c]  = n_p + X^[p,c] + Q[p,c]                   ("source" value, kept in a ring)
//   Y[p,c]  = log2 sum_{k=1..min(K,p)} 2^(r[p-k,c] + O[p,c] + B[k-1,c])
//   n_p     = n_{p-1} + max_c (Y[p,c] - n_{p-1});  Y^ = Y - n_p;  X^[p,x] = LSE_y (Y^[p,y] + Tm[y,x])
// with O/Q the per-position prefix-sum terms (alpha: O = S[t]+Pe[t-1], Q = -S[t]+Ps[t];
// beta: O = -S[t]+Ps[t], Q = S[t]+Pe[t-1]) and Tm = T (alpha) or T^T (beta). Everything is
// carried in base 2 (MUFU ex2/lg2); n_p is fp64, r is an fp32 (hi, lo) pair so that the
// prefix-sum differences keep fp64-level absolute accuracy.
//
// Execution layout (one thread-block cluster per (sequence, direction)):
//   head CTA
//     chain warp(s)  lane = label. Step p: merge the prepared partial (durations >= 3) with
//                    the k = 1, 2 terms, max-normalise (redux), C x C transition in exp space
//                    (smem-broadcast GEMV on FMA), publish. The only sequential dependency.
//     near warps     iteration p (one step of slack): source r[p-3] into the ring (and to the
//                    tails), durations 3..kc of target p, merge of the tails' partial.
//     aux warp(s)    lane = label: cp.async staging of input rows, fp64 prefix-sum terms,
//                    edge terms of the k = 1, 2 durations, per-position outputs, bookkeeping.
//   tail CTAs        (G-1, label slices, one warp per label) durations kc+1..K. Sources are
//                    pushed to them with st.async; they run kc-2 positions ahead of the head
//                    and push (max, sum) partials back with st.async + mbarrier complete_tx.
// Outputs per position (linear in T, compact): Y^ and X^ (working type) and n (fp64).
#pragma once

#include "scrf_common.cuh"

namespace scrf {

constexpr int kSlots = 32;      // head <-> tail mbarrier ring depth (power of two, > kNear + 12)
constexpr int kNear = 16;       // durations handled by the head when the cluster has tails
constexpr int kStage = 32;      // staged positions (power of two)
constexpr int kNring = 64;      // chain normaliser ring n_p (power of two, > kNear + 8)
constexpr int kAhead = 12;      // staging distance (positions)
constexpr float kSlack = 60.f;  // shared-reference LSE slack (log2 units)

// named barrier ids (0 is __syncthreads)
constexpr int BAR_A = 1;   // 1..4: chain -> near/aux (position q published), id 1 + (q & 3)
constexpr int BAR_B = 5;   // 5..8: near -> chain (partial of target p ready), id 5 + (p & 3)
constexpr int BAR_CH = 9;  // chain-internal (C > 32)
constexpr int BAR_CH2 = 10;
constexpr int BAR_NG = 11; // 11, 12: near group-internal

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename R>
__device__ __forceinline__ void st_async_pair(uint32_t dst, R x, R y, uint32_t bar);
template <>
__device__ __forceinline__ void st_async_pair<float>(uint32_t dst, float x, float y, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(dst), "f"(x),
               "f"(y), "r"(bar)
               : "memory");
}
template <>
__device__ __forceinline__ void st_async_pair<double>(uint32_t dst, double x, double y, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst), "d"(x),
               "d"(y), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t dst, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(dst), "d"(v), "r"(bar)
               : "memory");
}

template <typename R>
__device__ __forceinline__ R warp_max(R v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <>
__device__ __forceinline__ float warp_max<float>(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// ----------------------------------------------------------------------------
// geometry and arguments

template <typename R>
struct Vec4;
template <>
struct Vec4<float> {
  using T = float4;
};
template <>
struct Vec4<double> {
  using T = double4;
};

struct SweepGeo {
  int G;      // CTAs per cluster: head + G-1 tails
  int kc;     // head durations 1..kc (K when G == 1)
  int KRm;    // head source ring: power-of-two slots - 1
  int KTm;    // tail source ring: power-of-two slots - 1
  int NCW;    // chain warps (ceil(C/32))
  int NAS;    // aux warp sets of NCW warps: 2 = separate source and edge roles, 1 = merged
  int NNW;    // near warps
  int NG;     // near groups (2 or 4): group g owns the targets p with p % NG == g
  int PubS;   // slots of the position-indexed head rings (16: edge batches of 4, 8: per-step edge)
  int TWb;    // blocked tails: warps per label (1, or 2 taking alternate groups of 4 targets)
  int NOW;    // output warps (1 with separate edge warps: they write Y^, X^, n, max shift)
  int GWn;    // near threads per label (power of two <= 32)
  int NWt;    // tail warps
  int WPL;    // tail warps per label (each pushes its own partial)
  int TBlk;   // blocked tails (exp-space source blocks, FMA): 1 = one label per warp, 8 / 16 = that
              // many lanes per label (32 / TBlk labels per warp: more labels per tail); 0 = exact
  int PsRow;  // staged row holding Ps[t] (0 = no proj_start)
  int PeRow;  // staged row holding Pe[t-1] (0 = no proj_end)
  int CgMax;  // max labels per tail
  int NT;     // block size (max over roles)
  int Msm;    // exp-space transition matrix staged in shared memory
  unsigned long long wperm;  // head warp placement: 4 bits per physical warp = the role (logical
                             // warp) it runs; 0 = identity (SMSP of a warp = its index mod 4)
};

// logical head thread index of this thread (role layout is defined on logical warps)
__device__ __forceinline__ int head_ltid(const SweepGeo& g) {
  const int w = threadIdx.x >> 5;
  const int lw = g.wperm ? (int)((g.wperm >> (4 * w)) & 15) : w;
  return (lw << 5) | (threadIdx.x & 31);
}

// One window replay (sublinear-memory mode, streaming.py:232-261 recompute_alpha and its beta
// twin): a sweep over local positions p = 0 .. steps with absolute position t = t0 + p (alpha)
// or t0 - p (beta), whose first `nforce` positions are forced to the stored messages
// (Y^ and n rows fY/fN from frow on) instead of being computed; outputs go to window rows
// out_row + (t - t_lo).
struct SweepTask {
  int b, dir, t0, steps, nforce, t_lo;
  int fstep;      // forced row of local position p: frow + fstep * p
  long long frow, out_row;
  int ck_phase;   // alpha: t0 % delta (checkpoint counter at local position 0)
  double n_ref;   // alpha: checkpoint normaliser in effect after t0 (log2 units)
};

template <typename R>
struct SweepArgs {
  const double* S;
  const int64_t* lengths;
  const double* trans;
  const double* dur;
  const double* ps;
  const double* pe;
  int B, T, K, C;
  SweepGeo geo;
  int dirs;  // 1 = alpha only, 2 = beta only, 3 = both (cluster c -> b = c >> 1, dir = c & 1)
  // per-position outputs, indexed by true position t: [B][T+1][C] and [B][T+1]
  R* Y[2];
  R* X[2];
  double* n[2];
  double* logZ;      // [B] nats (alpha)
  double* logZb;     // [B] nats (beta: LSE_c beta[0,c], consistency value)
  int32_t* dead_at;  // [B]
  int32_t* clamp;    // [B] alpha positions whose max message leaves the reference's +-CLAMP_LIMIT (or null)
  R* amx;            // [B][T+1] full mode, alpha: per-position max shift (-inf: dead position), or null
  double* N;         // [B][n_ckpt] reference checkpoint normalisers
  int delta, n_ckpt;
  // storage mode of the per-position outputs Y^, X^, n:
  //   0 = every position at row b*(T+1) + t (full mode, linear memory);
  //   1 = checkpoint rows only (sublinear mode, pass 1): alpha rows of the last mA positions of
  //       every delta-period (+ t = 0), beta rows of [jW, t_top(j)] for every interior window
  //       boundary jW (ck_row_* below); Y^ and n only
  int store;
  int mA, W, nW;            // store == 1 geometry
  const SweepTask* tasks;   // replay mode (one task per cluster) or null
  const R* fY[2];           // forced Y^ rows of the replay tasks
  const double* fN[2];      // forced n rows
  long long* trace;  // debug: [256][16] clock64 stamps of cluster 0 (chain lane 0: 0..7, near thread 0: 8..15)
  int trace_from;    // first traced position
  int* hang;         // debug: watchdog record {block, thread, site, index} (first writer wins), or null
  // full mode: per-cluster progress of the stored rows, [B*2 + dir][kProgSlots] (or null). Slot w
  // of writer warp w holds q + 1 once every row the warp writes for local positions <= q is
  // globally visible (L + 1 when it is done); the overlapped posterior passes wait on the
  // minimum over the writers (prog_wait_kernel, scrf_capi.cu).
  int* prog;
  // streamed input (full mode; or null): S rows [j << gate_shift, (j+1) << gate_shift) of every
  // sequence are on the device once gate[j] != 0 (set by the caller's copy stream,
  // scrf_gate_set); gate[ngate] = 1 records a wait that timed out
  const int* gate;
  int gate_shift, ngate;
};

constexpr int kProgSlots = 8;

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// publish "rows of local positions < v written by this warp are visible" (whole warp calls)
__device__ __forceinline__ void prog_publish(int* slot, int v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    *(volatile int*)slot = v;
  }
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// cross-CTA latency trace (debug, globaltimer ns, cluster 0): a.trace + 1088*16 + 8*pos +
// {0: source pos sent, 1: tail saw source pos, 2: tail sent partial of target pos, 3: near
// received partial of pos, 4: chain passed B(pos), 5: chain arrived A(pos), 6: near group
// passed A(pos-4), 7: edge batch of A(pos) done}
#ifndef SCRF_TRACE
#define SCRF_GT(slot, pos) \
  do {                     \
  } while (0)
#else
#define SCRF_GT(slot, pos)                                                                            \
  do {                                                                                              \
    if (a.trace && (pos) >= a.trace_from && (pos) < a.trace_from + 256)                             \
      a.trace[1088 * 16 + ((pos) - a.trace_from) * 8 + (slot)] = gtimer();                          \
  } while (0)
#endif

// mbarrier wait with an optional watchdog (a.hang != null): after ~1e8 polls record where
// and trap instead of hanging the device. The watchdog is out of line: the hot loops that wait
// carry only the plain wait (their instruction footprint matters, see the tail GATE note).
__device__ __noinline__ void sweep_wait_watchdog(int* hang, uint32_t bar, uint32_t parity, int site, int idx) {
  for (long long i = 0; i < 100000000LL; ++i)
    if (mbar_try(bar, parity)) return;
  if (atomicCAS(hang, 0, 1) == 0) {
    hang[1] = blockIdx.x;
    hang[2] = threadIdx.x;
    hang[3] = site;
    hang[4] = idx;
    __threadfence_system();
  }
  __trap();
}
// OOL: the watchdog path as a call (MODE 3 instantiations: -1.2 ms of sweep at c4) or inline
// (the other modes measure faster with it inline: instruction layout of their hot loops)
template <bool OOL, typename A>
__device__ __forceinline__ void sweep_wait(const A& a, uint32_t bar, uint32_t parity, int site, int idx) {
  if (!a.hang) {
#ifdef SCRF_EXP_BACKOFF
    if (site == 2) {
      while (!mbar_try(bar, parity)) __nanosleep(SCRF_EXP_BACKOFF);
      return;
    }
#endif
    mbar_wait(bar, parity);
    return;
  }
  if (OOL) {
    sweep_wait_watchdog(a.hang, bar, parity, site, idx);
    return;
  }
  for (long long i = 0; i < 100000000LL; ++i)
    if (mbar_try(bar, parity)) return;
  if (atomicCAS(a.hang, 0, 1) == 0) {
    a.hang[1] = blockIdx.x;
    a.hang[2] = threadIdx.x;
    a.hang[3] = site;
    a.hang[4] = idx;
    __threadfence_system();
  }
  __trap();
}

// per-label row strides padded to an odd number of elements (conflict-free across labels)
__host__ __device__ inline int ring_stride(int mask) { return mask + 2; }
__host__ __device__ inline int b2_stride(int kc) { return kc | 1; }

__host__ __device__ inline int tail_lo(int r, int C, int G) { return (int)(((long long)(r - 1) * C) / (G - 1)); }

struct HeadLayout {
  size_t M, Xmax, B2, ring, stg, oq, own, pubY, pubX, pubA, nring, part, hh, h3, ew, wmax, tpart, tbar, total;
};
struct TailLayout {
  size_t ring, B2, nslot, tbar, stg, wtab, bx, total;
};

// blocked tails: exp-space source blocks of 32 held in registers (one block per lane)
constexpr int kBlk = 32;
// Edge work (the (O, Q) terms of each position, fp64 log2, read by the source warps (Q) and
// near groups (O); the duration 1..4 edge terms read by the chain; the per-position outputs):
//  - batched (NAS == 2, separate edge warps): at A(q), q % 4 == 0, targets q+kLead ..
//    q+kLead+3 and the outputs of positions q-3 .. q; position rings of 16 slots;
//  - per step (NAS == 1, done by the source warps): at A(q), target q+5 and the outputs of
//    position q; position rings of 8 slots.
// Input rows are prefetched into registers one batch (or four steps) ahead.
constexpr int kLead = 8;
__host__ __device__ inline int edge_lead(const SweepGeo& g) { return g.PubS == 16 ? kLead : 5; }
// w table length: windows read durations up to K + 35
__host__ __device__ inline int blk_wlen(int kc, int K) { return ((K < 1024 + kc ? K : 1024 + kc) + 64 + 1) & ~1; }
// w is stored in rows of 32 elements with a row stride of 34: lanes read windows that start
// 32*j elements apart, which the skew spreads over all banks (pairs never straddle a row)
__host__ __device__ inline int blk_wrow() { return 34; }
__host__ __device__ inline int blk_wphys(int e) { return (e >> 5) * 34 + (e & 31); }
__host__ __device__ inline int blk_wsize(int kc, int K) { return (blk_wlen(kc, K) / 32 + 2) * 34; }

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

// tail staging slots per position: one per (warp, label the warp handles) for the exact
// tails (warps sharing a label run at different paces), one per label for the blocked tails
__host__ __device__ inline int tail_lpw(const SweepGeo& g) {
  const int lstep = g.NWt / (g.WPL > 0 ? g.WPL : 1);
  return lstep > 0 ? (g.CgMax + lstep - 1) / lstep : 1;
}
__host__ __device__ inline int tail_stage_slots(const SweepGeo& g) {
  return g.TBlk ? g.CgMax : g.NWt * tail_lpw(g);
}

template <typename R>
__host__ __device__ inline HeadLayout head_layout(int K, int C, const SweepGeo& g) {
  HeadLayout L;
  size_t o = 0;
  const size_t Cw = C < 32 ? 32 : C;
  L.M = o;     o += g.Msm ? a16((size_t)C * C * sizeof(R)) : 0;
  L.Xmax = o;  o += a16((size_t)C * sizeof(R));
  L.B2 = o;    o += a16((size_t)C * b2_stride(g.kc) * sizeof(R));
  L.ring = o;  o += a16((size_t)C * ring_stride(g.KRm) * 2 * sizeof(R));
  L.stg = o;   // the head stages nothing in shared memory (edge rows are prefetched into registers)
  L.oq = o;    o += a16((size_t)g.PubS * C * sizeof(double2));
  L.own = o;   o += a16((size_t)C * sizeof(int2));
  L.pubY = o;  o += a16((size_t)g.PubS * C * sizeof(R));
  L.pubX = o;  o += a16((size_t)g.PubS * C * sizeof(R));
  L.pubA = o;  o += a16(g.PubS * sizeof(R));
  L.nring = o; o += a16(kNring * sizeof(double));
  L.part = o;  o += a16((size_t)4 * C * 2 * sizeof(R));
  L.hh = o;    o += a16((size_t)g.PubS * C * 4 * sizeof(R));
  L.h3 = o;
  L.ew = o;    o += a16(Cw * sizeof(R));
  L.wmax = o;  o += a16(32 * sizeof(R));
  L.tpart = o; o += a16((size_t)kSlots * g.WPL * C * 2 * sizeof(R));
  L.tbar = o;  o += a16(kSlots * sizeof(uint64_t));
  L.total = o;
  return L;
}

template <typename R>
__host__ __device__ inline TailLayout tail_layout(int K, int C, const SweepGeo& g) {
  TailLayout L;
  size_t o = 0;
  L.ring = o;  o += a16((size_t)g.CgMax * (g.KTm + 1) * 2 * sizeof(R));
  L.B2 = o;    o += g.TBlk ? 0 : a16((size_t)g.CgMax * K * sizeof(R));
  L.nslot = o; o += a16(kSlots * sizeof(double));
  L.tbar = o;  o += a16(kSlots * sizeof(uint64_t));
  L.stg = o;   o += a16((size_t)kStage * 2 * tail_stage_slots(g) * sizeof(double));
  L.wtab = o;  o += g.TBlk ? a16((size_t)g.CgMax * 2 * blk_wsize(g.kc, K) * sizeof(R)) : 0;
  L.bx = o;    o += g.TBlk ? a16((size_t)g.CgMax * (kBlk + 1) * sizeof(R)) : 0;
  L.total = o;
  return L;
}

template <typename R>
__host__ __device__ inline size_t sweep_smem_bytes(int K, int C, const SweepGeo& g) {
  size_t h = head_layout<R>(K, C, g).total;
  size_t t = g.G > 1 ? tail_layout<R>(K, C, g).total : 0;
  return h > t ? h : t;
}

// ----------------------------------------------------------------------------
// small numerics

template <typename R>
__device__ __forceinline__ void split2(double v, R& hi, R& lo) {
  hi = (R)v;
  lo = (v > -CUDART_INF && v < CUDART_INF) ? (R)(v - (double)hi) : (R)0;
}

// merge (m2, s2) into (m, s) (value = m + log2 s)
template <typename R>
__device__ __forceinline__ void lse_merge(R& m, R& s, R m2, R s2) {
  if (!(s2 > (R)0) || m2 == Mth<R>::ninf()) return;
  if (!(s > (R)0) || m == Mth<R>::ninf()) {
    m = m2;
    s = s2;
    return;
  }
  if (m2 > m) {
    s = s * Mth<R>::ex2(m - m2) + s2;
    m = m2;
  } else {
    s = s + s2 * Mth<R>::ex2(m2 - m);
  }
}

// log2(2^m s + 2^x2 + 2^x1)
template <typename R>
__device__ __forceinline__ R lse3(R m, R s, R x2, R x1) {
  const R mm = (s > (R)0) ? m : Mth<R>::ninf();
  const R M = fmax(mm, fmax(x2, x1));
  if (M == Mth<R>::ninf()) return M;
  R sum = Mth<R>::ex2(x2 - M) + Mth<R>::ex2(x1 - M);
  if (mm != Mth<R>::ninf()) sum += s * Mth<R>::ex2(mm - M);
  return M + Mth<R>::lg2(sum);
}

// Sum of 2^(term - mref) over ring terms k = k0, k0+kstep, ... <= kmax, with
// term = (rg[slot].x + e_hi) + (rg[slot].y + e_lo) + b2[k-1] and slot of k0 = slot0,
// stepping back kstep slots per term (power-of-two ring: mask). Tracks the largest
// exponent so the caller can fall back to the exact path.
template <typename R>
__device__ __forceinline__ void ring_sum(const typename Vec2<R>::T* rg, int mask, const R* b2, int k0, int kstep,
                                         int kmax, int slot0, R e_hi, R e_lo, R mref, R& sum, R& dmax) {
  R a0 = 0, a1 = 0, a2 = 0, a3 = 0, d0 = Mth<R>::ninf(), d1 = Mth<R>::ninf();
  int k = k0, slot = slot0;
  const R c_lo = e_lo - mref;  // (r.x + e_hi) + (r.y + e_lo - mref) + b
  for (; k + 3 * kstep <= kmax; k += 4 * kstep) {
    const auto r0 = rg[slot];
    const auto r1 = rg[(slot - kstep) & mask];
    const auto r2 = rg[(slot - 2 * kstep) & mask];
    const auto r3 = rg[(slot - 3 * kstep) & mask];
    slot = (slot - 4 * kstep) & mask;
    const R x0 = ((r0.x + e_hi) + (r0.y + c_lo)) + b2[k - 1];
    const R x1 = ((r1.x + e_hi) + (r1.y + c_lo)) + b2[k + kstep - 1];
    const R x2 = ((r2.x + e_hi) + (r2.y + c_lo)) + b2[k + 2 * kstep - 1];
    const R x3 = ((r3.x + e_hi) + (r3.y + c_lo)) + b2[k + 3 * kstep - 1];
    d0 = fmax(d0, fmax(x0, x1));
    d1 = fmax(d1, fmax(x2, x3));
    a0 += Mth<R>::ex2(x0);
    a1 += Mth<R>::ex2(x1);
    a2 += Mth<R>::ex2(x2);
    a3 += Mth<R>::ex2(x3);
  }
  for (; k <= kmax; k += kstep) {
    const auto r0 = rg[slot];
    slot = (slot - kstep) & mask;
    const R x0 = ((r0.x + e_hi) + (r0.y + c_lo)) + b2[k - 1];
    d0 = fmax(d0, x0);
    a0 += Mth<R>::ex2(x0);
  }
  sum += (a0 + a1) + (a2 + a3);
  dmax = fmax(dmax, fmax(d0, d1));
}

template <typename R>
__device__ __forceinline__ R gsum(R v, int W) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    if (off < W) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// exact (own-maximum) version of ring_sum including the optional reference term; the
// caller reduces (m, s) across the lane group with group_ms.
template <typename R>
__device__ __noinline__ typename Vec2<R>::T ring_exact(const typename Vec2<R>::T* rg, int mask, const R* b2, int k0,
                                                       int kstep, int kmax, int slot0, R e_hi, R e_lo, R mref,
                                                       bool self_term) {
  R m = self_term ? mref : Mth<R>::ninf();
  int slot = slot0;
  for (int k = k0; k <= kmax; k += kstep) {
    const auto r0 = rg[slot];
    m = fmax(m, (r0.x + e_hi) + (r0.y + e_lo) + b2[k - 1]);
    slot = (slot - kstep) & mask;
  }
  R s = 0;
  if (m != Mth<R>::ninf()) {
    if (self_term) s = Mth<R>::ex2(mref - m);
    slot = slot0;
    for (int k = k0; k <= kmax; k += kstep) {
      const auto r0 = rg[slot];
      s += Mth<R>::ex2(((r0.x + e_hi) + (r0.y + e_lo) + b2[k - 1]) - m);
      slot = (slot - kstep) & mask;
    }
  }
  typename Vec2<R>::T out;
  out.x = m;
  out.y = s;
  return out;
}

// group-reduced LSE over the ring terms of one label (lane group of width W)
template <typename R>
__device__ __forceinline__ void ring_lse(const typename Vec2<R>::T* rg, int mask, const R* b2, int k0, int kstep,
                                         int kmax, int slot0, R e_hi, R e_lo, R mref, bool self_term, int W, R& m,
                                         R& s) {
  s = self_term ? (R)1 : (R)0;
  R dmax = Mth<R>::ninf();
  bool slow = (mref == Mth<R>::ninf()) && (self_term || k0 <= kmax);
  if (!slow) ring_sum<R>(rg, mask, b2, k0, kstep, kmax, slot0, e_hi, e_lo, mref, s, dmax);
  slow = slow || dmax > (R)kSlack;
  m = mref;
  if (__any_sync(0xffffffffu, slow)) {
    const auto ms = ring_exact<R>(rg, mask, b2, k0, kstep, kmax, slot0, e_hi, e_lo, mref, self_term);
    m = ms.x;
    s = ms.y;
    group_ms(m, s, W);
  } else {
    s = gsum(s, W);
  }
}

// ----------------------------------------------------------------------------
// per-sweep context

struct SweepCtx {
  int b, dir, L, rank;  // L: local steps (positions 0 .. L)
  int t0;               // absolute position of local position 0 (alpha: 0, beta: L_b in full sweeps)
  int Lb;               // true length of sequence b
  const double* S;   // row base of sequence b: S + b*(T+1)*C
  const double* ps;  // proj_start rows of b or null
  const double* pe;
  const SweepTask* task;  // replay task or null
  __device__ __forceinline__ int tpos(int p) const { return dir == 0 ? t0 + p : t0 - p; }
};

// checkpoint rows (store == 1). Alpha: t = 0 -> row 0; else period i = ceil(t / delta),
// e = i*delta - t, stored iff e < mA at row 1 + (i-1)*mA + (mA-1-e). Beta: boundary j =
// floor(t / W) >= 1 with jW < L, stored iff t <= t_top(j) at row (j-1)*(K+32) + t - jW.
__host__ __device__ inline int ck_ttop(int j, int W, int K, int L) {
  const int need = j * W + K - 1;
  return need >= L ? L : L - 32 * ((L - need) / 32);
}
// alpha rows per sequence: t = 0, the last mA positions of every delta-period, and the last mA
// positions before L (the ring the reference holds past L, for the checkpoint view)
__host__ __device__ inline long long ck_rows_alpha(int T, int delta, int mA) {
  return 1 + (long long)((T + delta - 1) / delta) * mA + mA;
}
__device__ __forceinline__ long long ck_row(int dir, int t, int L, int K, int delta, int mA, int W) {
  if (dir == 0) {
    if (t == 0) return 0;
    const int i = (t + delta - 1) / delta;
    const int e = i * delta - t;
    return e < mA ? 1 + (long long)(i - 1) * mA + (mA - 1 - e) : -1;
  }
  const int j = t / W;
  if (j < 1 || j * W >= L || t > ck_ttop(j, W, K, L)) return -1;
  return (long long)(j - 1) * (K + 32) + (t - j * W);
}

// ----------------------------------------------------------------------------
// head CTA
//
// Hand-offs (q = position just published by the chain):
//   chain  step p : needs part(p) [near, frame n_{p-3}] and hh(p) = (h1, h2) [aux];
//                   adds the k = 1, 2 terms itself; publishes Y^[p], X^[p], n_p; arrives A(p).
//   near   iter p : waits A(p-3); writes the source r[p-3] into the ring (and to its
//                   tail); sums durations 3..kc (+ tail partial) of target p; arrives B(p).
//   aux    iter q : waits A(q); outputs of q, bookkeeping; (O, Q) of q+5 and hh(q+4);
//                   stages the input rows of position q+kAhead with cp.async.

template <typename R>
struct HeadPtr {
  using R2 = typename Vec2<R>::T;
  R* M;
  R* Xmax;
  R* B2;
  R2* ring;
  double* stg;
  double2* oq;
  int2* own;
  R* pubY;
  R* pubX;
  R* pubA;
  double* nring;
  R2* part;
  typename Vec4<R>::T* hh;
  R* ew;
  R* wmax;
  R2* tpart;
  uint64_t* tbar;
};

template <typename R>
__device__ HeadPtr<R> head_ptrs(unsigned char* base, const HeadLayout& L) {
  using R2 = typename Vec2<R>::T;
  HeadPtr<R> h;
  h.M = (R*)(base + L.M);
  h.Xmax = (R*)(base + L.Xmax);
  h.B2 = (R*)(base + L.B2);
  h.ring = (R2*)(base + L.ring);
  h.stg = (double*)(base + L.stg);
  h.oq = (double2*)(base + L.oq);
  h.own = (int2*)(base + L.own);
  h.pubY = (R*)(base + L.pubY);
  h.pubX = (R*)(base + L.pubX);
  h.pubA = (R*)(base + L.pubA);
  h.nring = (double*)(base + L.nring);
  h.part = (R2*)(base + L.part);
  h.hh = (typename Vec4<R>::T*)(base + L.hh);
  h.ew = (R*)(base + L.ew);
  h.wmax = (R*)(base + L.wmax);
  h.tpart = (R2*)(base + L.tpart);
  h.tbar = (uint64_t*)(base + L.tbar);
  return h;
}

// staged rows per position: S[t], then Ps[t] and Pe[t-1] when present
__host__ __device__ inline int stg_rows(const SweepGeo& g) { return 1 + (g.PsRow > 0) + (g.PeRow > 0); }

// fp64 (O, Q) of label c at sweep position p from the raw staged rows (log2 units)
__device__ __forceinline__ double2 oq_of(const SweepCtx& x, const SweepGeo& g, int C, const double* stg, int p, int c) {
  const double* d = stg + (size_t)(p & (kStage - 1)) * stg_rows(g) * C;
  const double s = d[c] * kLog2e;
  const double psv = g.PsRow ? d[g.PsRow * C + c] * kLog2e : 0.0;
  const double pev = g.PeRow ? d[g.PeRow * C + c] * kLog2e : 0.0;
  return x.dir == 0 ? make_double2(s + pev, -s + psv) : make_double2(-s + psv, s + pev);
}

// Streamed input: wait until the rows of local positions p0 .. p1 (and one row beyond each end:
// rows are not cache-line aligned, so a line fetched with an edge row may hold bytes of its
// neighbour) are on the device. The readers of S call it before they cross into rows not yet
// checked, 512 rows at a time: the edge warps (or the source warps when they do the edge work)
// every 256 positions, each tail thread when its next staged target passes its threshold.
// Gives up after 2 s (records gate[ngate] = 1) rather than hang on a caller bug.
template <typename R>
__device__ __noinline__ void gate_span_wait(const SweepArgs<R>& a, const SweepCtx& x, int p0, int p1) {
  int t0 = x.tpos(p0), t1 = x.tpos(p1);
  if (t0 > t1) {
    const int tt = t0;
    t0 = t1;
    t1 = tt;
  }
  t0 = t0 > 0 ? t0 - 1 : 0;
  t1 = t1 < a.T ? t1 + 1 : a.T;
  const int j0 = t0 >> a.gate_shift, j1 = t1 >> a.gate_shift;
  for (int j = j0; j <= j1; ++j) {
    const long long s = gtimer();
    while (ld_acquire_i32(a.gate + j) == 0) {
      if (ld_acquire_i32(a.gate + a.ngate) != 0) return;
      if (gtimer() - s > 2000000000LL) {
        atomicExch((int*)a.gate + a.ngate, 1);
        return;
      }
      __nanosleep(256);
    }
  }
}

// raw rows S[t], Ps[t], Pe[t-1] of label c at sweep position p into its staging slot
template <bool ASYNC>
__device__ __forceinline__ void stage_label(const SweepCtx& x, const SweepGeo& g, int T, int C, double* stg, int p,
                                            int c) {
  const int t = x.tpos(p);
  double* d = stg + (size_t)(p & (kStage - 1)) * stg_rows(g) * C + c;
  const double* s0 = x.S + (size_t)t * C + c;
  if (ASYNC) cp_async8(d, s0); else d[0] = __ldg(s0);
  if (g.PsRow) {
    double* dd = d + g.PsRow * C;
    if (t < T) {
      if (ASYNC) cp_async8(dd, x.ps + (size_t)t * C + c); else *dd = __ldg(x.ps + (size_t)t * C + c);
    } else {
      *dd = 0.0;
    }
  }
  if (g.PeRow) {
    double* dd = d + g.PeRow * C;
    if (t >= 1) {
      if (ASYNC) cp_async8(dd, x.pe + (size_t)(t - 1) * C + c); else *dd = __ldg(x.pe + (size_t)(t - 1) * C + c);
    } else {
      *dd = 0.0;
    }
  }
}

// edge terms of target u for label c from the (O, Q) ring: hk = O[u] + Q[u-k] + B[k-1] for
// k = 1..4 (-inf when the duration is infeasible), written as one 4-vector (prologue targets)
template <typename R>
__device__ __forceinline__ void head_edge(int C, int K, const double2* oq, const R* B2, int kc, int u, int c,
                                          typename Vec4<R>::T* hh, int pm) {
  const double O = oq[(size_t)(u & pm) * C + c].x;
  const R* b2 = B2 + (size_t)c * b2_stride(kc);
  R v[4];
#pragma unroll
  for (int k = 1; k <= 4; ++k) {
    v[k - 1] = Mth<R>::ninf();
    if (u >= k && K >= k) v[k - 1] = (R)(O + oq[(size_t)((u - k) & pm) * C + c].y + (double)b2[k - 1]);
  }
  typename Vec4<R>::T w;
  w.x = v[0];
  w.y = v[1];
  w.z = v[2];
  w.w = v[3];
  hh[(size_t)(u & pm) * C + c] = w;
}

// raw input rows of label c at sweep position p: S[t], Ps[t] (0 past the end), Pe[t-1] (0 at
// t = 0); zeros past L. Same values stage_label writes.
struct EdgeRows {
  double s, ps, pe;
};
__device__ __forceinline__ EdgeRows load_rows(const SweepCtx& x, const SweepGeo& g, int T, int C, int L, int p, int c) {
  EdgeRows r{0.0, 0.0, 0.0};
  if (p <= L) {
    const int t = x.tpos(p);
    r.s = __ldg(x.S + (size_t)t * C + c);
    if (g.PsRow && t < T) r.ps = __ldg(x.ps + (size_t)t * C + c);
    if (g.PeRow && t >= 1) r.pe = __ldg(x.pe + (size_t)(t - 1) * C + c);
  }
  return r;
}
// (O, Q) from raw rows (same arithmetic as oq_of)
__device__ __forceinline__ double2 oq_rows(const SweepCtx& x, const SweepGeo& g, const EdgeRows& r) {
  const double s = r.s * kLog2e;
  const double psv = g.PsRow ? r.ps * kLog2e : 0.0;
  const double pev = g.PeRow ? r.pe * kLog2e : 0.0;
  return x.dir == 0 ? make_double2(s + pev, -s + psv) : make_double2(-s + psv, s + pev);
}

// row of the per-position outputs of absolute position t, or -1 when it is not stored
template <typename R>
__device__ __forceinline__ long long out_row(const SweepArgs<R>& a, const SweepCtx& x, int t) {
  if (x.task) return x.task->out_row + (t - x.task->t_lo);
  if (a.store == 0) return (long long)x.b * (a.T + 1) + t;
  const long long r = ck_row(x.dir, t, x.Lb, a.K, a.delta, a.mA, a.W);
  if (r < 0) return -1;
  return (x.dir == 0 ? (long long)x.b * ck_rows_alpha(a.T, a.delta, a.mA) : (long long)x.b * a.nW * (a.K + 32)) + r;
}

template <typename R, int MODE>
__device__ __forceinline__ void put_out(const SweepArgs<R>& a, const SweepCtx& x, int t, int c, bool act, R y, R xv,
                                        double n, R am) {
  const int C = a.C;
  if (MODE == 0 || MODE == 3) {  // full mode: every position, row b*(T+1)+t
    const long long row = (long long)x.b * (a.T + 1) + t;
    if (act) {
      a.Y[x.dir][row * C + c] = y;
      a.X[x.dir][row * C + c] = xv;
    }
    if (c == 0) {
      a.n[x.dir][row] = n;
      if (x.dir == 0 && a.amx) a.amx[row] = am;
    }
    return;
  }
  const long long row = out_row(a, x, t);
  if (row >= 0) {
    if (act) {
      a.Y[x.dir][row * C + c] = y;
      if (a.X[x.dir]) a.X[x.dir][row * C + c] = xv;
    }
    if (c == 0) a.n[x.dir][row] = n;
  }
  if (a.store == 1 && !x.task && x.dir == 0 && t > x.Lb - a.mA) {  // final-ring rows of the checkpoint view
    const long long r2 = (long long)x.b * ck_rows_alpha(a.T, a.delta, a.mA) + 1 +
                         (long long)((a.T + a.delta - 1) / a.delta) * a.mA + (t - (x.Lb - a.mA + 1));
    if (act) a.Y[0][r2 * C + c] = y;
    if (c == 0) a.n[0][r2] = n;
  }
}

// edge-batch state of one label: Q of the four positions before the next batch's targets and
// the prefetched rows of those targets
struct EdgeState {
  double qh[4];     // qh[i] = Q[u0 - 4 + i], u0 = the next (first) target
  EdgeRows rw[4];   // rows of targets u0 + i
};
__device__ __forceinline__ void edge_init(const SweepCtx& x, const SweepGeo& g, const double2* oq, int T, int C, int L,
                                          int c, EdgeState& e) {
  const int lead = edge_lead(g);
#pragma unroll
  for (int i = 0; i < 4; ++i) e.qh[i] = oq[(size_t)(lead - 4 + i) * C + c].y;
#pragma unroll
  for (int i = 0; i < 4; ++i) e.rw[i] = load_rows(x, g, T, C, L, lead + i, c);
}

// Per-step edge work at A(q) (PubS == 8) for label c: (O, Q) and edge terms of target q+5,
// outputs of position q; rows of target q+9 prefetched into the register FIFO.
template <typename R, int MODE>
__device__ __forceinline__ void edge_step(const SweepArgs<R>& a, const SweepCtx& x, const HeadPtr<R>& h, int q, int c,
                                          bool act, const R* b2c, EdgeState& e) {
  const SweepGeo& g = a.geo;
  const int C = a.C, K = a.K, T = a.T, L = x.L;
  const int pm = g.PubS - 1;
  const int u = q + edge_lead(g);
  if (act && u <= L) {
    const double2 v = oq_rows(x, g, e.rw[0]);
#pragma unroll
    for (int i = 0; i < 3; ++i) e.rw[i] = e.rw[i + 1];
    e.rw[3] = load_rows(x, g, T, C, L, u + 4, c);
    h.oq[(size_t)(u & pm) * C + c] = v;
    const R ninf = Mth<R>::ninf();
    typename Vec4<R>::T w;
    w.x = K >= 1 ? (R)(v.x + e.qh[3] + (double)b2c[0]) : ninf;
    w.y = K >= 2 ? (R)(v.x + e.qh[2] + (double)b2c[1]) : ninf;
    w.z = K >= 3 ? (R)(v.x + e.qh[1] + (double)b2c[2]) : ninf;
    w.w = K >= 4 ? (R)(v.x + e.qh[0] + (double)b2c[3]) : ninf;
    h.hh[(size_t)(u & pm) * C + c] = w;
#pragma unroll
    for (int i = 0; i < 3; ++i) e.qh[i] = e.qh[i + 1];
    e.qh[3] = v.y;
  }
  const int sl = q & pm;
  const int cs = act ? c : 0;
  put_out<R, MODE>(a, x, x.tpos(q), c, act, h.pubY[sl * C + cs], h.pubX[sl * C + cs], h.nring[q & (kNring - 1)], h.pubA[sl]);
}

// per-position outputs (Y^, X^, n, max shift) of positions q-3 .. q from the published rings
template <typename R, int MODE>
__device__ __forceinline__ void edge_outputs(const SweepArgs<R>& a, const SweepCtx& x, const HeadPtr<R>& h, int q, int c,
                                             bool act) {
  const int C = a.C;
  const int cs = act ? c : 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pos = q - 3 + i;
    if (pos >= 0) {
      const int sl = pos & 15;
      put_out<R, MODE>(a, x, x.tpos(pos), c, act, h.pubY[sl * C + cs], h.pubX[sl * C + cs], h.nring[pos & (kNring - 1)],
                 h.pubA[sl]);
    }
  }
}

// One edge batch at A(q) (q % 4 == 0) for label c: (O, Q) and edge terms hk = O[u] + Q[u-k] +
// B[k-1] (k = 1..4) of targets u = q+kLead .. q+kLead+3, the outputs Y^, X^, n, max shift of
// positions q-3 .. q, and the register prefetch of the next batch's rows.
template <typename R, int MODE>
__device__ __forceinline__ void edge_batch(const SweepArgs<R>& a, const SweepCtx& x, const HeadPtr<R>& h, int q, int c,
                                           bool act, const R* b2c, EdgeState& e, bool outputs) {
  const SweepGeo& g = a.geo;
  const int C = a.C, K = a.K, T = a.T, L = x.L;
  if (act) {
    const int u0 = q + kLead;
    double2 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = oq_rows(x, g, e.rw[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) e.rw[i] = load_rows(x, g, T, C, L, u0 + 4 + i, c);  // next batch
    double qa[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      qa[i] = e.qh[i];
      qa[4 + i] = v[i].y;
    }
    const R ninf = Mth<R>::ninf();
    const double b0 = (double)b2c[0], b1 = (double)b2c[1], b2 = (double)b2c[2], b3 = (double)b2c[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = u0 + i;
      if (u <= L) {
        h.oq[(size_t)(u & 15) * C + c] = v[i];
        typename Vec4<R>::T w;
        w.x = K >= 1 ? (R)(v[i].x + qa[3 + i] + b0) : ninf;
        w.y = K >= 2 ? (R)(v[i].x + qa[2 + i] + b1) : ninf;
        w.z = K >= 3 ? (R)(v[i].x + qa[1 + i] + b2) : ninf;
        w.w = K >= 4 ? (R)(v[i].x + qa[0 + i] + b3) : ninf;
        h.hh[(size_t)(u & 15) * C + c] = w;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) e.qh[i] = qa[4 + i];
  }
  if (outputs) edge_outputs<R, MODE>(a, x, h, q, c, act);
}

// log2(2^m s + sum_k 2^xk), k = 1..4
template <typename R>
__device__ __forceinline__ R lse5(R m, R s, R x4, R x3, R x2, R x1) {
  const R mm = (s > (R)0) ? m : Mth<R>::ninf();
  const R M = fmax(fmax(mm, x4), fmax(fmax(x3, x2), x1));
  if (M == Mth<R>::ninf()) return M;
  R sum = (Mth<R>::ex2(x4 - M) + Mth<R>::ex2(x3 - M)) + (Mth<R>::ex2(x2 - M) + Mth<R>::ex2(x1 - M));
  if (mm != Mth<R>::ninf()) sum += s * Mth<R>::ex2(mm - M);
  return M + Mth<R>::lg2(sum);
}

// the reference's guard in the reference frame (rare: only reachable with a max shift below -1e8);
// out of line so that its fp64 arithmetic is not if-converted onto the chain's critical path
__device__ __noinline__ bool guard_dead(double n_prev, double am, double n_ref) { return (n_prev + am) - n_ref <= kGuardL2; }

// exact log-space transition pass (rare: underflowing exp-space sums)
template <typename R>
__device__ __noinline__ R gemv_exact(const double* trans, int dir, int C, int NCW, R* ew, R yh, bool act, int c, bool slow,
                                     R out) {
  const int nch = NCW * 32;
  if (NCW > 1) nbar_sync(BAR_CH, nch);
  if (act) ew[c] = yh;
  if (NCW > 1)
    nbar_sync(BAR_CH2, nch);
  else
    __syncwarp();
  const int cc = act ? c : 0;
  R mm = Mth<R>::ninf();
  for (int y = 0; y < C; ++y) {
    const double tv = dir == 0 ? trans[(size_t)y * C + cc] : trans[(size_t)cc * C + y];
    mm = fmax(mm, ew[y] + (R)(tv * kLog2e));
  }
  R ss = 0;
  if (mm != Mth<R>::ninf())
    for (int y = 0; y < C; ++y) {
      const double tv = dir == 0 ? trans[(size_t)y * C + cc] : trans[(size_t)cc * C + y];
      ss += Mth<R>::ex2(ew[y] + (R)(tv * kLog2e) - mm);
    }
  if (NCW > 1)
    nbar_sync(BAR_CH, nch);
  else
    __syncwarp();
  if (slow) out = (mm == Mth<R>::ninf()) ? mm : mm + Mth<R>::lg2(ss);
  return out;
}

// Barrier bookkeeping. A(q): id 1 + (q & 3); the chain arrives; the source and edge warps and
// the near group (q & 1) sync; count NA. B(p): id 5 + (p & 3); near group (p & 1) arrives, the
// chain syncs; count NB. Every id is used with one count only.

// ======================= chain warps =======================
template <typename R, bool CW1, int MODE>
__device__ void head_chain(const SweepArgs<R>& a, const SweepCtx& x, HeadPtr<R>& h, int NA, int NAE, int NB) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, L = x.L;
  // physical thread index: the chain warps never move (head_wperm keeps warps 0 .. NCW-1 in
  // place; a logical index here costs ~1.5 % of the step in re-materialised address math)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = warp * 32 + lane;
  const bool act = c < C;
  const int nch = g.NCW * 32;
  auto Mval = [&](int y) -> R {
    if (g.Msm) return h.M[y * C + c];
    const double tv = x.dir == 0 ? a.trans[(size_t)y * C + c] : a.trans[(size_t)c * C + y];
    return Mth<R>::ex2((R)(tv * kLog2e) - h.Xmax[c]);
  };
  R Mreg[CW1 ? 32 : 1];
  if (CW1) {
#pragma unroll
    for (int y = 0; y < 32; ++y) Mreg[y] = (act && y < C) ? Mval(y) : (R)0;
  }
  // The exp-space GEMV sum of label x is >= M[y*][x] (the frame's maximal label y* has Y^ = 0
  // exactly), so when every column's smallest factor is >= 2^-90 the sum can never fall below
  // the 1e-30 fallback threshold (a dead position sums to 0 and gives -inf on both paths): the
  // per-step vote for the exact path is then skipped (C <= 32; the outcome is unchanged).
  bool may_underflow = true;
  if (CW1) {
    R mn = (R)1;
#pragma unroll
    for (int y = 0; y < 32; ++y)
      if (y < C) mn = fmin(mn, Mreg[y]);
    may_underflow = __any_sync(0xffffffffu, act && !(mn >= (R)8.077935669463161e-28));  // 2^-90
  }
  const R xmax = act ? h.Xmax[c] : (R)0;
  // X^[x] = xmax[x] + log2 sum_y 2^(yh[y]) M[y][x]
  auto gemv = [&](R yh) -> R {
    const R e = act ? Mth<R>::ex2(yh) : (R)0;
    R s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (CW1) {
      h.ew[lane] = e;  // lanes >= C hold 0 and their Mreg rows are 0
      __syncwarp();
#pragma unroll
      for (int y = 0; y < 32; y += 4) {
        const R e0 = h.ew[y], e1 = h.ew[y + 1], e2 = h.ew[y + 2], e3 = h.ew[y + 3];
        s0 += e0 * Mreg[y];
        s1 += e1 * Mreg[y + 1];
        s2 += e2 * Mreg[y + 2];
        s3 += e3 * Mreg[y + 3];
      }
      __syncwarp();
    } else {
      if (act) h.ew[c] = e;
      nbar_sync(BAR_CH2, nch);
      if (act) {
        int y = 0;
        if (g.Msm) {  // M column of this label in shared memory: loads pipelined 8 deep
          const R* Mc = h.M + c;
#pragma unroll 2
          for (; y + 8 <= C; y += 8) {
            s0 += h.ew[y] * Mc[(size_t)y * C];
            s1 += h.ew[y + 1] * Mc[(size_t)(y + 1) * C];
            s2 += h.ew[y + 2] * Mc[(size_t)(y + 2) * C];
            s3 += h.ew[y + 3] * Mc[(size_t)(y + 3) * C];
            s0 += h.ew[y + 4] * Mc[(size_t)(y + 4) * C];
            s1 += h.ew[y + 5] * Mc[(size_t)(y + 5) * C];
            s2 += h.ew[y + 6] * Mc[(size_t)(y + 6) * C];
            s3 += h.ew[y + 7] * Mc[(size_t)(y + 7) * C];
          }
          for (; y < C; ++y) s0 += h.ew[y] * Mc[(size_t)y * C];
        } else {
          for (; y + 4 <= C; y += 4) {
            s0 += h.ew[y] * Mval(y);
            s1 += h.ew[y + 1] * Mval(y + 1);
            s2 += h.ew[y + 2] * Mval(y + 2);
            s3 += h.ew[y + 3] * Mval(y + 3);
          }
          for (; y < C; ++y) s0 += h.ew[y] * Mval(y);
        }
      }
      nbar_sync(BAR_CH, nch);
    }
    const R sum = (s0 + s1) + (s2 + s3);
    R out = xmax + Mth<R>::lg2(sum);
    const bool slow = act && !(sum >= (R)1e-30);
    if (may_underflow && __any_sync(0xffffffffu, slow)) out = gemv_exact<R>(a.trans, x.dir, C, g.NCW, h.ew, yh, act, c, slow, out);
    return out;
  };
  auto chain_max = [&](R y) -> R {
    R am = warp_max(act ? y : Mth<R>::ninf());
    if (!CW1) {
      if (lane == 0) h.wmax[warp] = am;
      nbar_sync(BAR_CH, nch);
      am = h.wmax[0];
      for (int w = 1; w < g.NCW; ++w) am = fmax(am, h.wmax[w]);
    }
    return am;
  };

  // replay: the first nforce positions take the stored messages (Y^, n) instead of the
  // computed ones; X^ (the transition GEMV) and everything downstream are recomputed, so the
  // replay reproduces the sweep that stored them (same positions mod 32, same arithmetic).
  // Forced rows are prefetched one position ahead.
  const SweepTask* tk = (MODE == 2) ? x.task : nullptr;
  const int nforce = (MODE == 2) ? tk->nforce : 0;
  const int cs = act ? c : 0;
  const R* fY = (MODE == 2) ? a.fY[x.dir] + (long long)tk->frow * C + cs : nullptr;
  const double* fN = (MODE == 2) ? a.fN[x.dir] + tk->frow : nullptr;
  const long long fsC = (MODE == 2) ? (long long)tk->fstep * C : 0;
  const int fs1 = (MODE == 2) ? tk->fstep : 0;
  R fq = Mth<R>::ninf();
  double nq = 0.0;
  if ((MODE == 2) && nforce > 0) {
    fq = act ? fY[0] : Mth<R>::ninf();
    nq = fN[0];
  }
  // position 0: alpha[0] = 0 (virtual source) / beta[L] = 0, or the first forced position
  const R yh0 = nforce > 0 ? fq : (x.dir == 0 ? (R)0 : Mth<R>::ninf());
  const double n0 = nforce > 0 ? nq : 0.0;
  if ((MODE == 2) && nforce > 1) {
    fq = act ? fY[fsC] : Mth<R>::ninf();
    nq = fN[fs1];
  }
  R x1h = (nforce > 0 || x.dir == 0) ? gemv(nforce > 0 ? yh0 : (R)0) : (R)0;  // X^[p-1]
  R x2h = Mth<R>::ninf();                    // X^[p-2]
  R x3h = Mth<R>::ninf();                    // X^[p-3]
  R x4h = Mth<R>::ninf();                    // X^[p-4]
  if (act) {
    h.pubY[c] = yh0;
    h.pubX[c] = x1h;
  }
  if (tid == 0) {
    h.pubA[0] = 0;
    h.nring[0] = n0;
  }
  nbar_arrive(BAR_A + 0, NA + NAE);
  R a1 = 0, a2 = 0, a3 = 0;  // frame shifts amax_{p-1}, amax_{p-2}, amax_{p-3}
  double n_prev = n0;
  // alpha: checkpoint normaliser in effect (log2) and the position counter since the last
  // checkpoint (streaming.py:205-214); beta: 0 (absolute frame)
  double n_ref = (MODE == 2) ? tk->n_ref : 0.0;
  int ck_cnt = (MODE == 2) ? tk->ck_phase : 0;
  // reference bookkeeping of the alpha sweep (streaming.py:194-229): in the full mode a
  // post-pass reads it off the stored per-position messages (book_kernel); the checkpoint-row
  // (sublinear) sweep stores too few positions for that, so its chain keeps it
  const bool sbook = MODE == 1 && x.dir == 0;
  int dmin = -1, n_clamp = 0;
  if (sbook && tid == 0 && a.N) a.N[(size_t)x.b * a.n_ckpt] = 0.0;
  const R2* partc = h.part + cs;
  const typename Vec4<R>::T* hhc = h.hh + cs;
  const int pubm = g.PubS - 1;
  for (int p = 1; p <= L; ++p) {
#ifdef SCRF_TRACE
    long long* tr = (a.trace && blockIdx.x == 0 && tid == 0 && p >= a.trace_from && p < a.trace_from + 256) ? a.trace + (p - a.trace_from) * 16 : nullptr;
#else
    constexpr long long* tr = nullptr;
#endif
    if (tr) tr[0] = clock64();
    nbar_sync(BAR_B + (p & 3), NB);
    if (blockIdx.x == 0 && tid == 0) SCRF_GT(4, p);
    bool dead;
    R yh, am;
    double n_p;
    if ((MODE == 2) && p < nforce) {
      yh = fq;
      n_p = nq;
      am = (R)(n_p - n_prev);  // the stored sweep's shift (exact: n_p = n_prev + (double)am there)
      dead = false;
      if (p + 1 < nforce) {
        fq = act ? fY[(p + 1) * fsC] : Mth<R>::ninf();
        nq = fN[(p + 1) * fs1];
      }
    } else {
      R y = Mth<R>::ninf();
      if (act) {
        const R2 pm = partc[(p & 3) * C];  // durations >= 5, frame n_{p-4}
        const auto hv = hhc[(p & pubm) * C];  // edge terms of durations 1..4
        const R s12 = a2 + a1, s123 = a3 + s12;
        y = lse5(pm.x - s123, pm.y, x4h + hv.w - s123, x3h + hv.z - s12, x2h + hv.y - a1, x1h + hv.x);
      }
      if (tr) tr[1] = clock64();
      am = chain_max(y);
      // the reference's guard (_numerics.py:59-75): a position whose every message is at or below
      // NEG_INF + 1 in the reference frame (alpha: relative to the checkpoint normaliser in effect,
      // streaming.py:194-214; beta: absolute, streaming.py:316-355) is masked, i.e. -inf here
      dead = (am == Mth<R>::ninf());
      // (a max shift below -1e8 is the only way to reach the 1e9-wide guard: exact test only then)
      if (am < (R)-1e8) dead = dead || guard_dead(n_prev, (double)am, n_ref);
      yh = dead ? Mth<R>::ninf() : y - am;
      n_p = dead ? n_prev : n_prev + (double)am;
    }
    // everything but X^[p] is published before the GEMV so those stores overlap it
    if (act) h.pubY[(p & pubm) * C + c] = yh;
    if (tid == 0) {
      h.pubA[p & pubm] = dead ? Mth<R>::ninf() : am;
      h.nring[p & (kNring - 1)] = n_p;
    }
    const R xh = gemv(yh);
    if (tr) tr[2] = clock64();
    if (act) h.pubX[(p & pubm) * C + c] = xh;
    nbar_arrive(BAR_A + (p & 3), NA + ((p & 3) == 0 ? NAE : 0));
    if (blockIdx.x == 0 && tid == 0) SCRF_GT(5, p);
    if (tr) tr[3] = clock64();
    if (sbook) {  // sparse alpha sweep: reference bookkeeping in registers (see below)
      dmin = (dead && dmin < 0) ? p : dmin;
      n_clamp += (!dead && fabs(n_p - n_ref) > kClampLimit * kLog2e) ? 1 : 0;
    }
    if (x.dir == 0 && ++ck_cnt == a.delta) {  // checkpoint shift at t % delta == 0 (live, alive only)
      ck_cnt = 0;
      if (!dead) n_ref = n_p;
      if (sbook && tid == 0 && a.N && p / a.delta < a.n_ckpt) a.N[(size_t)x.b * a.n_ckpt + p / a.delta] = n_ref * kLn2;
    }
    x4h = x3h;
    x3h = x2h;
    x2h = x1h;
    x1h = xh;
    a3 = a2;
    a2 = a1;
    a1 = dead ? (R)0 : am;
    n_prev = n_p;
  }
  if (sbook) {
    // logZ = n_L + log2 sum_c 2^(Y^[L,c]) (nats); the reference raises only when the final
    // log-partition is at or below the guard, naming the first dead position (streaming.py:216-229)
    R sm = act ? Mth<R>::ex2(h.pubY[(L & pubm) * C + c]) : (R)0;
    for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
    if (g.NCW > 1) {
      if (lane == 0) h.wmax[warp] = sm;
      nbar_sync(BAR_CH, g.NCW * 32);
      sm = 0;
      for (int w = 0; w < g.NCW; ++w) sm += h.wmax[w];
    }
    if (tid == 0) {
      const double lz = (sm > (R)0) ? (n_prev + (double)Mth<R>::lg2(sm)) * kLn2 : -CUDART_INF;
      if (a.logZ) a.logZ[x.b] = lz;
      if (a.N)
        for (int i = L / a.delta + 1; i < a.n_ckpt; ++i) a.N[(size_t)x.b * a.n_ckpt + i] = n_ref * kLn2;  // frozen past L
      if (a.dead_at) a.dead_at[x.b] = (lz - n_ref * kLn2 > kGuard) ? -1 : (dmin >= 0 ? dmin : L);
      if (a.clamp) a.clamp[x.b] = n_clamp;
    }
  }
}

// ======================= near warps =======================
// NG groups of NNW/NG warps; group gi owns the targets p with p % NG == gi. Iteration p
// waits A(p-4) and sums durations 5..kc of target p from the source ring (sources <= p-5,
// written by the source warps) plus the tail partial (durations kc+1..K), in frame n_{p-4};
// then arrives B(p).
template <typename R, bool TAILS, int MODE>
__device__ void head_near(const SweepArgs<R>& a, const SweepCtx& x, HeadPtr<R>& h, int NA, int NAE, int NB) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, L = x.L;
  const int kc = g.kc, KRm = g.KRm;
  const int ntid = head_ltid(g) - g.NCW * 32;
  const int NG = g.NG;
  const int ngw = g.NNW / NG;          // warps per group
  const int gi = (ntid >> 5) / ngw;    // group
  const int gtid = ntid - gi * ngw * 32;
  const int GW = g.GWn;
  const int c = gtid / GW, j = gtid % GW;  // one label per lane group
  const bool act = c < C;
  const int cs = act ? c : 0;
  const R2* ringc = h.ring + (size_t)cs * ring_stride(KRm);
  const R* b2c = h.B2 + (size_t)cs * b2_stride(kc);
  const R2* tpartc = h.tpart + cs;
  R2* partc = h.part + cs;
  R bk[kNear - 4];  // duration biases 5..kNear (log2) of this label
#pragma unroll
  for (int i = 0; i < kNear - 4; ++i) bk[i] = (5 + i <= kc) ? b2c[4 + i] : Mth<R>::ninf();
  for (int p = gi == 0 ? NG : gi; p <= L + 4; p += NG) {
#ifdef SCRF_TRACE
    long long* tr = (a.trace && blockIdx.x == 0 && gtid == 0 && p >= a.trace_from && p < a.trace_from + 256)
                        ? ((p & 1) == 0 ? a.trace + (p - a.trace_from) * 16 + 8 : a.trace + 832 * 16 + (p - a.trace_from) * 16)
                        : nullptr;
#else
    constexpr long long* tr = nullptr;
#endif
    if (tr) tr[0] = clock64();
    if (p >= 4) nbar_sync(BAR_A + ((p - 4) & 3), NA + (((p - 4) & 3) == 0 ? NAE : 0));
    if (tr) tr[1] = clock64();
    if (blockIdx.x == 0 && gtid == 0) SCRF_GT(6, p);
    if (p > L) continue;
    const int q = p - 4;
    const int kmax = min(kc, p);
    R m = Mth<R>::ninf(), s = 0;
    double n_q = 0.0;
    if (q >= 1) {
      n_q = h.nring[q & (kNring - 1)];
      R e_hi = 0, e_lo = 0, mref = Mth<R>::ninf();
      if (act && kmax >= 5) {
        split2(h.oq[(size_t)(p & (g.PubS - 1)) * C + cs].x - n_q, e_hi, e_lo);
        const R2 r5 = ringc[(q - 1) & KRm];
        mref = (r5.x + e_hi) + (r5.y + e_lo) + b2c[4];
      }
      if (tr) tr[2] = clock64();
      if (TAILS && GW == 1 && kmax == kNear) {
        // steady state, durations 5..kNear fully unrolled and branch-free: all ring loads
        // in flight at once (inactive lanes compute on label 0 and are ignored)
        constexpr int NK = kNear - 4;
        R xv[NK];
#pragma unroll
        for (int i = 0; i < NK; ++i) {
          const R2 rr = ringc[(q - 1 - i) & KRm];  // source p - 5 - i, duration 5 + i
          xv[i] = ((rr.x + e_hi) + (rr.y + e_lo)) + bk[i];
        }
        R t4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          t4[i] = xv[i];
#pragma unroll
          for (int k2 = i + 4; k2 < NK; k2 += 4) t4[i] = fmax(t4[i], xv[k2]);
        }
        const R xm = fmax(fmax(t4[0], t4[1]), fmax(t4[2], t4[3]));
        R a4[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < NK; ++i) a4[i & 3] += Mth<R>::ex2(xv[i] - xm);
        m = xm;
        s = (xm == Mth<R>::ninf()) ? (R)0 : (a4[0] + a4[1]) + (a4[2] + a4[3]);
      } else {
        // durations 6..kmax from the ring (k = 5 is the shared reference)
        ring_lse<R>(ringc, KRm, b2c, 6 + j, GW, act ? kmax : 0, (q - 2 - j) & KRm, e_hi, e_lo, mref,
                    j == 0 && act && kmax >= 5, GW, m, s);
      }
      if (tr) tr[3] = clock64();
    }
    if (TAILS && p >= kc + 1) {
      const int pi = p - kc - 1;
      const int sl = pi & (kSlots - 1);
      if (tr) tr[5] = clock64();
      sweep_wait<MODE == 3>(a, smem_u32(&h.tbar[sl]), (uint32_t)((pi / kSlots) & 1), 1, p);
      if (blockIdx.x == 0 && gtid == 0) SCRF_GT(3, p);
      if (tr) tr[6] = clock64();
      if (act && j == 0) {
        const double d = n_q - h.nring[pi & (kNring - 1)];  // tail frame n_{p-kc-1} -> n_{p-4}
        R d_hi, d_lo;
        split2(d, d_hi, d_lo);
        const R2* tp = tpartc + (size_t)sl * g.WPL * C;
        R tm = tp[0].x, ts = tp[0].y;
        for (int w = 1; w < g.WPL; ++w) lse_merge(tm, ts, tp[w * C].x, tp[w * C].y);
        lse_merge(m, s, (tm - d_hi) - d_lo, ts);
      }
      if (gtid == 0 && p + kSlots <= L) mbar_expect(smem_u32(&h.tbar[sl]), (uint32_t)(g.WPL * C * 2 * sizeof(R)));
    }
    if (act && j == 0) {
      R2 pm;
      pm.x = m;
      pm.y = s;
      partc[(p & 3) * C] = pm;
    }
    if (tr) tr[4] = clock64();
    nbar_arrive(BAR_B + (p & 3), NB);
  }
}

// ======================= source warps (lane = label) =======================
// Iteration q waits A(q): source r[q] = n_q + X^[q] + Q[q] into the ring (read by the near
// groups from iteration q+5 on) and to the tail owning the label; n_q to every tail. With
// NAS == 1 also the edge batches; otherwise only the outputs of the last L % 4 positions
// (the edge batches cover positions <= 4 floor(L/4)).
template <typename R, bool TAILS, int MODE>
__device__ void head_src(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, HeadPtr<R>& h,
                         const TailLayout& TL, int NA, int NAE, int wbase, bool do_edge) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, T = a.T, L = x.L;
  const int KRm = g.KRm, KTm = g.KTm;
  const int c = head_ltid(g) - wbase * 32;  // label
  const bool act = c < C;
  const int cs = act ? c : 0;
  const R* pXc = h.pubX + cs;
  R2* ringc = h.ring + (size_t)cs * ring_stride(KRm);
  const int nsend_max = L - g.kc - 1;  // last source any tail needs
  uint32_t t_ring = 0, t_bar = 0, t_nslot = 0, t_nbar = 0;
  const bool nsender = TAILS && c >= 32 * g.NCW - (g.G - 1);
  if (TAILS) {
    const int2 ow = h.own[cs];
    t_ring = mapa_u32(smem_u32(smem + TL.ring) + (uint32_t)((size_t)ow.y * (KTm + 1) * 2 * sizeof(R)), ow.x);
    t_bar = mapa_u32(smem_u32(smem + TL.tbar), ow.x);
    if (nsender) {
      const int rt = c - (32 * g.NCW - (g.G - 1)) + 1;
      t_nslot = mapa_u32(smem_u32(smem + TL.nslot), rt);
      t_nbar = mapa_u32(smem_u32(smem + TL.tbar), rt);
    }
  }
  EdgeState es;
  const R* b2c = h.B2 + (size_t)cs * b2_stride(g.kc);
  if (do_edge) edge_init(x, g, h.oq, T, C, L, cs, es);
  const int Lq = L & ~3;  // last position written by an edge batch
  // progress slot: source warp w is writer 1 + w beside the output warp, or writer w
  int* pslot = (a.prog && !x.task)
                   ? a.prog + (size_t)(x.b * 2 + x.dir) * kProgSlots + (c >> 5) + (do_edge ? 0 : 1)
                   : nullptr;
  if (pslot && !do_edge) prog_publish(pslot, Lq + 1);  // only the positions after Lq are this warp's
  for (int q = 0; q <= L; ++q) {
    if (MODE == 3 && do_edge && (q & 255) == 0) {  // streamed input (edge work here): next 512 rows
      if ((threadIdx.x & 31) == 0) gate_span_wait(a, x, q, min(q + 512, L));
      __syncwarp();
    }
#ifdef SCRF_TRACE
    // source-warp phases (cluster 0, lane 0): [0] loop top, [1] after A(q), [2] ring written, [3] sends issued
    long long* trs = (a.trace && blockIdx.x == 0 && c == 0 && q >= a.trace_from && q < a.trace_from + 256)
                         ? a.trace + 1344 * 16 + (q - a.trace_from) * 4
                         : nullptr;
    if (trs) trs[0] = clock64();
#endif
    nbar_sync(BAR_A + (q & 3), NA + ((q & 3) == 0 ? NAE : 0));
#ifdef SCRF_TRACE
    if (trs) trs[1] = clock64();
#endif
    const double n_q = h.nring[q & (kNring - 1)];
    const int sl = q & (g.PubS - 1);
    if (act) {
      const R X = pXc[sl * C];
      const double r = (X == Mth<R>::ninf()) ? -CUDART_INF : n_q + ((double)X + h.oq[(size_t)sl * C + c].y);
      R2 v;
      split2(r, v.x, v.y);
      ringc[q & KRm] = v;
#ifdef SCRF_TRACE
      if (trs) trs[2] = clock64();
#endif
      if (TAILS && q <= nsend_max)
        st_async_pair<R>(t_ring + (uint32_t)((q & KTm) * 2 * sizeof(R)), v.x, v.y,
                         t_bar + (uint32_t)((q & (kSlots - 1)) * sizeof(uint64_t)));
    }
    if (blockIdx.x == 0 && c == 0) SCRF_GT(0, q);
#ifdef SCRF_TRACE
    if (trs) trs[3] = clock64();
#endif
#ifdef SCRF_TRACE
    if (a.trace && blockIdx.x == 0 && c == 0 && q >= a.trace_from && q < a.trace_from + 256)
      a.trace[576 * 16 + (q - a.trace_from) * 16] = clock64();  // source q sent (head clock)
#endif
    if (TAILS && nsender && q <= nsend_max)
      st_async_f64(t_nslot + (uint32_t)((q & (kSlots - 1)) * sizeof(double)), n_q,
                   t_nbar + (uint32_t)((q & (kSlots - 1)) * sizeof(uint64_t)));
    if (do_edge) edge_step<R, MODE>(a, x, h, q, c, act, b2c, es);
    if (!do_edge && q > Lq)  // outputs of the positions after the last edge batch
      put_out<R, MODE>(a, x, x.tpos(q), c, act, h.pubY[sl * C + cs], pXc[sl * C], n_q, h.pubA[sl]);
    if (pslot && do_edge && (q & 255) == 255) prog_publish(pslot, q + 1);

    if (x.dir == 1 && q == L && c == 0 && !x.task) {
      const R* pX = h.pubX + sl * C;
      R mx = Mth<R>::ninf();
      for (int cc = 0; cc < C; ++cc) mx = fmax(mx, pX[cc]);
      R ssum = 0;
      if (mx != Mth<R>::ninf())
        for (int cc = 0; cc < C; ++cc) ssum += Mth<R>::ex2(pX[cc] - mx);
      a.logZb[x.b] = (mx == Mth<R>::ninf()) ? -CUDART_INF : (n_q + (double)mx + (double)Mth<R>::lg2(ssum)) * kLn2;
    }
  }
  if (pslot) prog_publish(pslot, L + 1);
}

// ======================= edge warps (lane = label), NAS == 2 =======================
// Sync A(q) for q % 4 == 0 only (barrier id 1 counts the edge warps) and run the edge batch.
template <typename R, int MODE>
__device__ void head_edge_role(const SweepArgs<R>& a, const SweepCtx& x, HeadPtr<R>& h, int NA, int NAE, int wbase) {
  const SweepGeo& g = a.geo;
  const int C = a.C, T = a.T, L = x.L;
  const int c = head_ltid(g) - wbase * 32;
  const bool act = c < C;
  const int cs = act ? c : 0;
  const R* b2c = h.B2 + (size_t)cs * b2_stride(g.kc);
  EdgeState es;
  edge_init(x, g, h.oq, T, C, L, cs, es);
  for (int q = 0; q <= L; q += 4) {
    if (MODE == 3 && (q & 255) == 0) {  // streamed input: the rows of the next 512 positions
      if ((threadIdx.x & 31) == 0) gate_span_wait(a, x, q, min(q + 512, L));
      __syncwarp();
    }
    nbar_sync(BAR_A + 0, NA + NAE);
    edge_batch<R, MODE>(a, x, h, q, c, act, b2c, es, g.NOW == 0);
    if (blockIdx.x == 0 && c == 0) SCRF_GT(7, q);
  }
}

// ======================= output warp (lane = label), NOW == 1 =======================
// Joins A(q) for q % 4 == 0 like the edge warps and writes the outputs of positions q-3 .. q,
// so the edge batch (on the critical path through that barrier) carries no HBM stores.
template <typename R, int MODE>
__device__ void head_out_role(const SweepArgs<R>& a, const SweepCtx& x, HeadPtr<R>& h, int NA, int NAE, int wbase) {
  const int C = a.C, L = x.L;
  const int c = head_ltid(a.geo) - wbase * 32;
  const bool act = c < C;
  int* pslot = (a.prog && !x.task) ? a.prog + (size_t)(x.b * 2 + x.dir) * kProgSlots : nullptr;
  for (int q = 0; q <= L; q += 4) {
    nbar_sync(BAR_A + 0, NA + NAE);
    edge_outputs<R, MODE>(a, x, h, q, c, act);
    if (pslot && (q & 255) == 252) prog_publish(pslot, q + 1);
  }
  if (pslot) prog_publish(pslot, L + 1);
}

template <typename R, bool TAILS, bool CW1, int MODE>
__device__ void head_main(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                          const TailLayout& TL) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int K = a.K, C = a.C, T = a.T, L = x.L;
  const int tid = threadIdx.x, warp = head_ltid(a.geo) >> 5;
  const int NAUX = g.NAS * g.NCW;                            // source (+ edge) warps
  const int NA = (2 * g.NCW + g.NNW / g.NG) * 32;            // chain + source + one near group
  const int NB = (g.NCW + g.NNW / g.NG) * 32;                // chain + one near group
  const int NAE = g.NAS == 2 ? (g.NCW + g.NOW) * 32 : 0;     // edge + output warps (A(q), q % 4 == 0 only)
  const int NH = (g.NCW + g.NNW + NAUX + g.NOW) * 32;        // all head threads
  HeadPtr<R> h = head_ptrs<R>(smem, HL);
  const int kc = g.kc;

  // ---- tables, (O, Q) of the first positions
  if (tid < NH) {
    for (int i = tid; i < C; i += NH) {
      double m = -CUDART_INF;
      for (int y = 0; y < C; ++y) {
        const double tv = x.dir == 0 ? a.trans[(size_t)y * C + i] : a.trans[(size_t)i * C + y];
        m = fmax(m, tv * kLog2e);
      }
      h.Xmax[i] = (R)m;
    }
    for (int i = tid; i < C * kc; i += NH) {
      const int cc = i / kc, k = i % kc;
      h.B2[(size_t)cc * b2_stride(kc) + k] = (R)(a.dur[(size_t)k * C + cc] * kLog2e);
    }
    for (int i = tid; i < C * ring_stride(g.KRm); i += NH) {
      R2 v;
      v.x = Mth<R>::ninf();
      v.y = 0;
      h.ring[i] = v;
    }
    if (TAILS && tid < kSlots) mbar_init(smem_u32(&h.tbar[tid]), 1);
    for (int i = tid; i < edge_lead(g) * C; i += NH) {  // (O, Q) of positions 0 .. lead-1
      const int u = i / C, cc = i % C;
      h.oq[(size_t)u * C + cc] = oq_rows(x, g, load_rows(x, g, T, C, L, u, cc));
    }
  }
  __syncthreads();
  if (tid < NH) {
    if (g.Msm)
      for (int i = tid; i < C * C; i += NH) {
        const int y = i / C, xx = i % C;
        const double tv = x.dir == 0 ? a.trans[(size_t)y * C + xx] : a.trans[(size_t)xx * C + y];
        h.M[i] = Mth<R>::ex2((R)(tv * kLog2e) - h.Xmax[xx]);
      }
    for (int i = tid; i < edge_lead(g) * C; i += NH) {  // edge terms of targets 1 .. lead-1
      const int u = i / C, cc = i % C;
      if (u >= 1 && u <= L) head_edge<R>(C, K, h.oq, h.B2, kc, u, cc, h.hh, g.PubS - 1);
    }
    for (int cc = tid; cc < C; cc += NH) {  // tail owning label cc and its index there
      int rt = 0, cl = 0;
      if (TAILS) {
        rt = 1;
        while (rt + 1 < g.G && tail_lo(rt + 1, C, g.G) <= cc) ++rt;
        cl = cc - tail_lo(rt, C, g.G);
      }
      h.own[cc] = make_int2(rt, cl);
    }
    if (TAILS && tid == 0) {
      mbar_fence_init();
      for (int q = 0; q < kSlots; ++q) mbar_expect(smem_u32(&h.tbar[q]), (uint32_t)(g.WPL * C * 2 * sizeof(R)));
    }
  }
  __syncthreads();
  if (TAILS) cluster_sync_all();

  if (warp < g.NCW)
    head_chain<R, CW1, MODE>(a, x, h, NA, NAE, NB);
  else if (warp < g.NCW + g.NNW)
    head_near<R, TAILS, MODE>(a, x, h, NA, NAE, NB);
  else if (warp < 2 * g.NCW + g.NNW)
    head_src<R, TAILS, MODE>(a, x, smem, h, TL, NA, NAE, g.NCW + g.NNW, g.NAS == 1);
  else if (g.NAS == 2 && warp < 3 * g.NCW + g.NNW)
    head_edge_role<R, MODE>(a, x, h, NA, NAE, 2 * g.NCW + g.NNW);
  else if (g.NOW && warp < NH / 32)
    head_out_role<R, MODE>(a, x, h, NA, NAE, 3 * g.NCW + g.NNW);
}

// ----------------------------------------------------------------------------
// tail CTA: durations kc+1..K of a label slice (one warp per label), ahead of the chain

// GATE: streamed input (MODE 3): the tails check the input gates before staging new rows. A
// template parameter so that the other modes carry no gate code (their tail loops are measurably
// faster without it: c4 MODE 0 sweep 33.8 -> 33.4 ms)
template <typename R, bool GATE>
__device__ void tail_loop(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                          const TailLayout& TL, int lo, int Cg) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int K = a.K, C = a.C, T = a.T, L = x.L, kc = g.kc, KTm = g.KTm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const R2* ring = (const R2*)(smem + TL.ring);
  const R* B2 = (const R*)(smem + TL.B2);
  const double* nslot = (const double*)(smem + TL.nslot);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  double* stg = (double*)(smem + TL.stg);
  // own rows of target u (S[t] and Pe[t-1] (alpha) / Ps[t] (beta)) for label cl
  // each warp stages its own copy (warps sharing a label run at different paces)
  const int NWs = tail_stage_slots(g), LPW = tail_lpw(g);
  const int WPL_ = g.WPL, lstep_ = g.NWt / WPL_, cl0_ = warp / WPL_;
  int gnext = 0;  // streamed input: rows below local position gnext are known to be on the device
  auto stage = [&](int u, int cl) {
    if (GATE && u >= gnext) {
      gate_span_wait(a, x, u, min(u + 512, x.L));
      gnext = u + 256;
    }
    const int t = x.tpos(u), c = lo + cl;
    double* d = stg + ((size_t)(u & (kStage - 1)) * NWs + warp * LPW + (cl - cl0_) / lstep_) * 2;
    cp_async8(d, x.S + (size_t)t * C + c);
    if (x.dir == 0 && x.pe && t >= 1)
      cp_async8(d + 1, x.pe + (size_t)(t - 1) * C + c);
    else if (x.dir == 1 && x.ps && t < T)
      cp_async8(d + 1, x.ps + (size_t)t * C + c);
    else
      d[1] = 0.0;
  };
  const int WPL = g.WPL;
  const int part = warp % WPL;         // k sub-range of this warp
  const int cl0 = warp / WPL;          // first label of this warp
  const int lstep = g.NWt / WPL;       // label stride across warps
  const int u0 = kc + 1;
  for (int i = 0; i < kAhead; ++i) {
    if (lane == 0 && u0 + i <= L)
      for (int cl = cl0; cl < Cg; cl += lstep) stage(u0 + i, cl);
    cp_async_commit();
  }
  const uint32_t hbar = mapa_u32(smem_u32(smem + HL.tbar), 0);
  const uint32_t hpart = mapa_u32(smem_u32(smem + HL.tpart), 0);
  int sn = 0;  // ring slot of the newest source s_new = u - kc - 1
  for (int u = u0; u <= L; ++u) {
    const int s_new = u - kc - 1;
#ifdef SCRF_TRACE
    long long* tr = (a.trace && blockIdx.x == 1 && threadIdx.x == 0 && u >= a.trace_from && u < a.trace_from + 256) ? a.trace + 256 * 16 + (u - a.trace_from) * 16 : nullptr;
#else
    constexpr long long* tr = nullptr;
#endif
    if (tr) tr[0] = clock64();
    cp_async_wait<kAhead - 1>();
    __syncwarp();
    if (tr) tr[1] = clock64();
    sweep_wait<GATE>(a, smem_u32(&tbar[s_new & (kSlots - 1)]), (uint32_t)((s_new / kSlots) & 1), 2, u);
    if (tr) tr[2] = clock64();
    if (threadIdx.x == 0 && s_new + kSlots <= L - kc - 1)
      mbar_expect(smem_u32(&tbar[s_new & (kSlots - 1)]), (uint32_t)(Cg * 2 * sizeof(R) + sizeof(double)));
    const double F = nslot[s_new & (kSlots - 1)];
    const int kmax = min(K, u);
    for (int cl = cl0; cl < Cg; cl += lstep) {
      const R2* rg = ring + (size_t)cl * (KTm + 1);
      const R* b2 = B2 + (size_t)cl * K;
      const double* d = stg + ((size_t)(u & (kStage - 1)) * NWs + warp * LPW + (cl - cl0) / lstep) * 2;
      const double s2 = d[0] * kLog2e, o2 = d[1] * kLog2e;
      const double O = x.dir == 0 ? s2 + o2 : -s2 + o2;
      R e_hi, e_lo;
      split2(O - F, e_hi, e_lo);
      const R2 r0 = rg[sn];
      const R mref = (r0.x + e_hi) + (r0.y + e_lo) + b2[kc];
      R m, s;
      const int ko = lane + 32 * part;
      ring_lse<R>(rg, KTm, b2, kc + 2 + ko, 32 * WPL, kmax, (sn - 1 - ko) & KTm, e_hi, e_lo, mref, ko == 0, 32, m, s);
      if (tr) tr[3] = clock64();
      if (lane == 0) {
        const uint32_t off = (uint32_t)((((size_t)(s_new & (kSlots - 1)) * WPL + part) * C + lo + cl) * 2 * sizeof(R));
        st_async_pair<R>(hpart + off, m, s, hbar + (uint32_t)((s_new & (kSlots - 1)) * sizeof(uint64_t)));
      }
    }
    if (lane == 0 && u + kAhead <= L)
      for (int cl = cl0; cl < Cg; cl += lstep) stage(u + kAhead, cl);
    cp_async_commit();
    sn = (sn + 1) & KTm;
  }
  cp_async_wait<0>();
}


// Blocked tail (TBlk). For target u the tail's durations kc+1..K are the sources
// s in [u-K, u-kc-1]. Sources form blocks of 32 (block j = [32j, 32j+31]); a complete
// block is kept as z[i] = 2^(r[32j+i] - G_j) (G_j = its largest source) in the registers of
// lane j % 32, and contributes 2^(G_j + e[u] + Bmax) * sum_i z[i] * w[u - 32j - i] to target
// u, with w[k] = 2^(B[k-1] - Bmax) (0 outside kc+1..K). Targets are processed in groups of
// four (one window load of 35 w values feeds 4 x 32 FMAs); the newest, incomplete block is
// summed term by term. Each target's partial is in the frame n_{u-kc-1} of its newest
// source. Needs kc + 32 <= K <= 1024 + kc.
template <typename R, bool GATE>
__device__ void tail_loop_blocked(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                                  const TailLayout& TL, int lo, int Cg) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, T = a.T, L = x.L, kc = g.kc, KTm = g.KTm, K = a.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TWb = g.TWb;
  const int cl = warp / TWb, par = warp % TWb;  // label; which of the label's warps
  // tails of an uneven label split own fewer than CgMax labels: their spare warps must not run
  // (they would send partials into another tail's label slots and break the head's byte count)
  if (cl >= Cg) return;
  const R2* rg = (const R2*)(smem + TL.ring) + (size_t)cl * (KTm + 1);
  const double* nslot = (const double*)(smem + TL.nslot);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  double* stg = (double*)(smem + TL.stg);
  const int WSZ = blk_wsize(kc, K);
  const R* wt = (const R*)(smem + TL.wtab) + (size_t)cl * 2 * WSZ;
  const R* bx = (const R*)(smem + TL.bx) + (size_t)cl * (kBlk + 1);
  const R bmax = bx[kBlk];
  int gnext = 0;  // streamed input: rows below local position gnext are known to be on the device
  auto stage = [&](int u) {
    if (GATE && u >= gnext) {
      gate_span_wait(a, x, u, min(u + 512, x.L));
      gnext = u + 256;
    }
    const int t = x.tpos(u), c = lo + cl;
    double* d = stg + ((size_t)(u & (kStage - 1)) * g.CgMax + cl) * 2;
    cp_async8(d, x.S + (size_t)t * C + c);
    if (x.dir == 0 && x.pe && t >= 1)
      cp_async8(d + 1, x.pe + (size_t)(t - 1) * C + c);
    else if (x.dir == 1 && x.ps && t < T)
      cp_async8(d + 1, x.ps + (size_t)t * C + c);
    else
      d[1] = 0.0;
  };
  // one lane per target (lanes 0..3) stages / computes / sends; results are broadcast
  const int li = lane & 3;
  const int gstep = 4 * TWb;          // this warp's groups: ub = u0 + 4 par + gstep i
  const int u0 = kc + 1 + 4 * par;
  const int nahead = TWb == 1 ? 3 : 2;  // staging distance in own groups (12 / 16 targets)
  for (int gq = 0; gq < nahead; ++gq) {
    if (lane < 4 && u0 + gstep * gq + li <= L) stage(u0 + gstep * gq + li);
    cp_async_commit();
  }
  const uint32_t hbar = mapa_u32(smem_u32(smem + HL.tbar), 0);
  const uint32_t hpart = mapa_u32(smem_u32(smem + HL.tpart), 0);
  R zr[kBlk];
#pragma unroll
  for (int i = 0; i < kBlk; ++i) zr[i] = 0;
  R Gh = Mth<R>::ninf(), Gl = 0;
  int jown = -1;   // block whose z this lane holds
  int jlast = -1;  // newest block loaded by this warp
  int snext = 0;   // first source this warp has not waited for
#ifdef SCRF_TRACE
  long long st_wait = 0, st_loop = 0, st_slow = 0;
  const long long st_t0 = clock64();
#endif
  for (int ub = u0; ub <= L; ub += gstep) {
    const int sb = ub - kc - 1;          // newest source of target ub (multiple of 4)
    const int nt = min(4, L - ub + 1);   // targets in this group
#ifdef SCRF_TRACE
    long long* tr = (a.trace && blockIdx.x == 1 && threadIdx.x == 0 && ub >= a.trace_from && ub < a.trace_from + 4 * 256)
                        ? a.trace + 256 * 16 + ((ub - a.trace_from) / 4) * 16
                        : nullptr;
#else
    constexpr long long* tr = nullptr;
#endif
    if (tr) tr[0] = clock64();
    if (TWb == 1)
      cp_async_wait<2>();
    else
      cp_async_wait<1>();
    __syncwarp();
    if (tr) tr[9] = clock64();
    // the group's sources sb .. sb+nt-1 (and their normalisers)
#ifdef SCRF_TRACE
    const long long w0 = clock64();
    if (a.trace && blockIdx.x == 1 && threadIdx.x == 0 && sb + 3 >= a.trace_from && sb + 3 < a.trace_from + 256) {
      a.trace[1312 * 16 + (sb + 3 - a.trace_from) * 2] = gtimer();  // tail starts waiting for sb..sb+3
      a.trace[1312 * 16 + (sb + 3 - a.trace_from) * 2 + 1] =
          mbar_try(smem_u32(&tbar[(sb + 3) & (kSlots - 1)]), (uint32_t)(((sb + 3) / kSlots) & 1)) ? 1 : 2;
    }
#endif
    // every source up to this group's newest (the other warp's group too: block loads need
    // them); warp 0 re-arms each slot for its next use
    const int s0 = snext;
    for (int s = s0; s < sb + nt; ++s) {
      sweep_wait<GATE>(a, smem_u32(&tbar[s & (kSlots - 1)]), (uint32_t)((s / kSlots) & 1), 2, s);
      if (threadIdx.x == 0 && blockIdx.x == 1) SCRF_GT(1, s);
    }
    snext = sb + nt;
#ifdef SCRF_TRACE
    if (ub >= 1000) st_wait += clock64() - w0;
#endif
    if (tr) tr[1] = clock64();
    R eh[4], el[4];
    {
      R h = 0, l = 0;
      if (lane < nt) {
        const int u = ub + lane;
        const double F = nslot[(sb + lane) & (kSlots - 1)];
        const double* d = stg + ((size_t)(u & (kStage - 1)) * g.CgMax + cl) * 2;
        const double s2 = d[0] * kLog2e, o2 = d[1] * kLog2e;
        split2((x.dir == 0 ? s2 + o2 : -s2 + o2) - F, h, l);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        eh[i] = __shfl_sync(0xffffffffu, h, i);
        el[i] = __shfl_sync(0xffffffffu, l, i);
      }
    }
    __syncwarp();
    if (tr) tr[4] = clock64();
    if (warp == 0 && lane < snext - s0) {
      const int s = s0 + lane;
      if (s + kSlots <= L - kc - 1)
        mbar_expect(smem_u32(&tbar[s & (kSlots - 1)]), (uint32_t)(Cg * 2 * sizeof(R) + sizeof(double)));
    }
    // newest complete block: z = 2^(r - G) into the registers of its owner lane
    if (sb >= kBlk && (sb >> 5) - 1 > jlast) {
      const int jb = (sb >> 5) - 1;
      const R2 r = rg[(jb * kBlk + lane) & KTm];
      const R gh = warp_max(r.x);
      const unsigned bal = __ballot_sync(0xffffffffu, r.x == gh);
      const R gl = __shfl_sync(0xffffffffu, r.y, __ffs(bal) - 1);
      const R z = (gh == Mth<R>::ninf() || r.x == Mth<R>::ninf()) ? (R)0 : Mth<R>::ex2((r.x - gh) + (r.y - gl));
      const bool own = lane == (jb & 31);
#pragma unroll
      for (int i = 0; i < kBlk; ++i) {
        const R v = __shfl_sync(0xffffffffu, z, i);
        if (own) zr[i] = v;
      }
      if (own) {
        Gh = gh;
        Gl = gl;
        jown = jb;
      }
      jlast = jb;
    }
    // newest incomplete block: sources [base, sb+i] for target i, term by term
    const int base = sb & ~(kBlk - 1);
    R xe[4];
    {
      const int s = base + lane;
      const R2 r = rg[s & KTm];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        xe[i] = Mth<R>::ninf();
        if (i < nt && s <= sb + i) xe[i] = (r.x + eh[i]) + (r.y + el[i]) + bx[ub + i - s - kc - 1];
      }
    }
    if (tr) tr[5] = clock64();
    // complete block owned by this lane: 4 x 32 FMAs against one window of w
    R pb[4] = {0, 0, 0, 0};
    bool have = false;
    int d0 = 0;
    if (jown >= 0 && Gh != Mth<R>::ninf()) {
      d0 = ub - jown * kBlk;     // duration of the block's source 0 for target ub
      const int wb = d0 - (kBlk - 1);  // window start: durations wb .. wb+34
      if (wb <= K) {
        have = true;
        const int m = wb & 1;
        const R* wc = wt + (size_t)m * WSZ;  // copy m holds w[y - m] at y (skewed rows)
        const int e0 = wb + m;               // even
        const int r0 = e0 >> 5, c0 = e0 & 31;
        R wv[kBlk + 4];
#pragma unroll
        for (int t2 = 0; t2 < (kBlk + 4) / 2; ++t2) {
          const int cc = c0 + 2 * t2;  // column within row r0 (may run into rows r0+1, r0+2)
          const int ph = r0 * 34 + cc + (cc >= 32 ? 2 : 0) + (cc >= 64 ? 2 : 0);
          const auto w2 = *(const typename Vec2<R>::T*)(wc + ph);
          wv[2 * t2] = w2.x;
          wv[2 * t2 + 1] = w2.y;
        }
        // target i, source j: duration d0 + i - j = wb + (31 - j) + i  ->  wv[31 - j + i]
#pragma unroll
        for (int jj = 0; jj < kBlk; ++jj) {
          const R z = zr[jj];
          pb[0] += z * wv[31 - jj];
          pb[1] += z * wv[32 - jj];
          pb[2] += z * wv[33 - jj];
          pb[3] += z * wv[34 - jj];
        }
      }
    }
    if (tr) tr[2] = clock64();
    // shared reference per target: the exact term of the newest source (lane (sb+i) & 31 of
    // the incomplete block) or, when the block just completed, the newest complete block
    R Mv[4], Sv[4], xbv[4];
    const int jnew = (sb >> 5) - 1;  // newest complete block
    bool slow = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      xbv[i] = (have && pb[i] > (R)0) ? ((Gh + eh[i]) + (Gl + el[i])) + bmax : Mth<R>::ninf();
      const int refl = (sb & (kBlk - 1)) + i <= kBlk - 1 ? ((sb + i) & (kBlk - 1)) : 0;
      const R rx = __shfl_sync(0xffffffffu, xe[i], refl);
      const R rb = __shfl_sync(0xffffffffu, xbv[i], jnew & 31);
      const R M = fmax(rx, rb);
      Mv[i] = M;
      slow |= (fmax(xbv[i], xe[i]) > M + (R)kSlack) || (M == Mth<R>::ninf() && fmax(xbv[i], xe[i]) != Mth<R>::ninf());
    }
    if (__any_sync(0xffffffffu, slow)) {
#ifdef SCRF_TRACE
      ++st_slow;
#endif
#pragma unroll
      for (int i = 0; i < 4; ++i) Mv[i] = warp_max(fmax(xbv[i], xe[i]));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const R M = Mv[i];
      R sm = 0;
      if (M != Mth<R>::ninf()) {
        if (xbv[i] != Mth<R>::ninf()) sm += pb[i] * Mth<R>::ex2(xbv[i] - M);
        if (xe[i] != Mth<R>::ninf()) sm += Mth<R>::ex2(xe[i] - M);
      }
      Sv[i] = sm;
    }
    if (tr) tr[6] = clock64();
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) Sv[i] += __shfl_xor_sync(0xffffffffu, Sv[i], off);
    }
    if (tr) tr[7] = clock64();
    {
      R mi = Mv[0], si = Sv[0];
#pragma unroll
      for (int i = 1; i < 4; ++i)
        if (li == i) {
          mi = Mv[i];
          si = Sv[i];
        }
      if (lane < nt) {
        const int sl = (sb + lane) & (kSlots - 1);
        const uint32_t off = (uint32_t)(((size_t)sl * C + lo + cl) * 2 * sizeof(R));
        st_async_pair<R>(hpart + off, mi, si, hbar + (uint32_t)(sl * sizeof(uint64_t)));
        if (warp == 0 && blockIdx.x == 1) SCRF_GT(2, ub + lane);
      }
      if (lane < 4 && ub + gstep * nahead + lane <= L) stage(ub + gstep * nahead + lane);
    }
    cp_async_commit();
    if (tr) tr[8] = clock64();
    if (tr) tr[3] = clock64();
#ifdef SCRF_TRACE
    if (ub < 1000) st_loop = clock64();
#endif
  }
#ifdef SCRF_TRACE
  // per-warp totals over targets >= 1000 (cluster 0): source-wait cycles, loop cycles, slow groups
  if (a.trace && blockIdx.x < g.G && lane == 0) {
    long long* o = a.trace + 1216 * 16 + ((blockIdx.x - 1) * 16 + warp) * 4;
    o[0] = st_wait;
    o[1] = clock64() - st_loop;
    o[2] = st_slow;
    o[3] = clock64() - st_t0;
  }
#endif
  cp_async_wait<0>();
}

// Blocked tail with several labels per warp (TBlk = LB lanes per label, 32 / LB labels per warp):
// the arithmetic of tail_loop_blocked, for durations short enough that at most LB complete source
// blocks are live (LB >= (K - kc - 1) / 32 + 1). A label's lane group holds one block per lane
// (block j in sub-lane j % LB), and the newest, incomplete block's 32 sources are spread over
// the group, 32 / LB per lane. Lets the exp-space tails serve 43-label slices (config 5: C = 128
// over 3 tails, where one label per warp would need 43 warps).
template <typename R, int LB, bool GATE>
__device__ void tail_loop_blocked_ml(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem,
                                     const HeadLayout& HL, const TailLayout& TL, int lo, int Cg) {
  using R2 = typename Vec2<R>::T;
  constexpr int P = 32 / LB;    // labels per warp
  constexpr int Q = kBlk / LB;  // sources of a 32-block per sub-lane
  const SweepGeo& g = a.geo;
  const int C = a.C, T = a.T, L = x.L, kc = g.kc, KTm = g.KTm, K = a.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pg = lane / LB, sl = lane % LB, gbase = pg * LB;
  const int cl = warp * P + pg;
  const bool lact = cl < Cg;  // groups past the tail's labels stay warp-synchronous but send nothing
  const int clc = lact ? cl : 0;
  const R2* rg = (const R2*)(smem + TL.ring) + (size_t)clc * (KTm + 1);
  const double* nslot = (const double*)(smem + TL.nslot);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  double* stg = (double*)(smem + TL.stg);
  const int WSZ = blk_wsize(kc, K);
  const R* wt = (const R*)(smem + TL.wtab) + (size_t)clc * 2 * WSZ;
  const R* bx = (const R*)(smem + TL.bx) + (size_t)clc * (kBlk + 1);
  const R bmax = bx[kBlk];
  int gnext = 0;  // streamed input: rows below local position gnext are known to be on the device
  auto stage = [&](int u) {
    if (GATE && u >= gnext) {
      gate_span_wait(a, x, u, min(u + 512, x.L));
      gnext = u + 256;
    }
    const int t = x.tpos(u), c = lo + clc;
    double* d = stg + ((size_t)(u & (kStage - 1)) * g.CgMax + clc) * 2;
    cp_async8(d, x.S + (size_t)t * C + c);
    if (x.dir == 0 && x.pe && t >= 1)
      cp_async8(d + 1, x.pe + (size_t)(t - 1) * C + c);
    else if (x.dir == 1 && x.ps && t < T)
      cp_async8(d + 1, x.ps + (size_t)t * C + c);
    else
      d[1] = 0.0;
  };
  // sub-lanes 0..3 of each label group stage / compute / send targets ub + sl
  const int u0 = kc + 1;
  constexpr int nahead = 3;
  for (int gq = 0; gq < nahead; ++gq) {
    if (lact && sl < 4 && u0 + 4 * gq + sl <= L) stage(u0 + 4 * gq + sl);
    cp_async_commit();
  }
  const uint32_t hbar = mapa_u32(smem_u32(smem + HL.tbar), 0);
  const uint32_t hpart = mapa_u32(smem_u32(smem + HL.tpart), 0);
  R zr[kBlk];
#pragma unroll
  for (int i = 0; i < kBlk; ++i) zr[i] = 0;
  R Gh = Mth<R>::ninf(), Gl = 0;
  int jown = -1, jlast = -1, snext = 0;
  for (int ub = u0; ub <= L; ub += 4) {
    const int sb = ub - kc - 1;         // newest source of target ub (a multiple of 4)
    const int nt = min(4, L - ub + 1);  // targets in this group
    cp_async_wait<2>();
    __syncwarp();
    const int s0 = snext;
    for (int s = s0; s < sb + nt; ++s) sweep_wait<GATE>(a, smem_u32(&tbar[s & (kSlots - 1)]), (uint32_t)((s / kSlots) & 1), 2, s);
    snext = sb + nt;
    R eh[4], el[4];
    {
      R h = 0, l = 0;
      if (lact && sl < nt) {
        const int u = ub + sl;
        const double F = nslot[(sb + sl) & (kSlots - 1)];
        const double* d = stg + ((size_t)(u & (kStage - 1)) * g.CgMax + clc) * 2;
        const double s2 = d[0] * kLog2e, o2 = d[1] * kLog2e;
        split2((x.dir == 0 ? s2 + o2 : -s2 + o2) - F, h, l);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        eh[i] = __shfl_sync(0xffffffffu, h, gbase + i);
        el[i] = __shfl_sync(0xffffffffu, l, gbase + i);
      }
    }
    __syncwarp();
    if (warp == 0 && lane < snext - s0) {
      const int s = s0 + lane;
      if (s + kSlots <= L - kc - 1)
        mbar_expect(smem_u32(&tbar[s & (kSlots - 1)]), (uint32_t)(Cg * 2 * sizeof(R) + sizeof(double)));
    }
    // newest complete block: z = 2^(r - G) (G its largest source; first one in source order
    // supplies the lo part) into the registers of its owner sub-lane jb % LB
    if (sb >= kBlk && (sb >> 5) - 1 > jlast) {
      const int jb = (sb >> 5) - 1;
      R2 r[Q];
      R gh = Mth<R>::ninf();
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        r[q] = rg[(jb * kBlk + sl + LB * q) & KTm];
        gh = fmax(gh, r[q].x);
      }
#pragma unroll
      for (int o = LB / 2; o > 0; o >>= 1) gh = fmax(gh, __shfl_xor_sync(0xffffffffu, gh, o));
      int ic = 1 << 30;
      R glc = 0;
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (ic == (1 << 30) && r[q].x == gh) {
          ic = sl + LB * q;
          glc = r[q].y;
        }
#pragma unroll
      for (int o = LB / 2; o > 0; o >>= 1) {
        const int oi = __shfl_xor_sync(0xffffffffu, ic, o);
        const R og = __shfl_xor_sync(0xffffffffu, glc, o);
        if (oi < ic) {
          ic = oi;
          glc = og;
        }
      }
      const R gl = glc;
      R z[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q)
        z[q] = (gh == Mth<R>::ninf() || r[q].x == Mth<R>::ninf()) ? (R)0 : Mth<R>::ex2((r[q].x - gh) + (r[q].y - gl));
      const bool own = sl == (jb & (LB - 1));
#pragma unroll
      for (int i = 0; i < kBlk; ++i) {
        const R v = __shfl_sync(0xffffffffu, z[i / LB], gbase + (i % LB));
        if (own) zr[i] = v;
      }
      if (own) {
        Gh = gh;
        Gl = gl;
        jown = jb;
      }
      jlast = jb;
    }
    // newest incomplete block: sources s = base + sl + LB q, term by term
    const int base = sb & ~(kBlk - 1);
    R xe[4][Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int s = base + sl + LB * q;
      const R2 r = rg[s & KTm];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        xe[i][q] = Mth<R>::ninf();
        if (i < nt && s <= sb + i) xe[i][q] = (r.x + eh[i]) + (r.y + el[i]) + bx[ub + i - s - kc - 1];
      }
    }
    // complete block owned by this sub-lane: 4 x 32 FMAs against one window of w
    R pb[4] = {0, 0, 0, 0};
    bool have = false;
    if (jown >= 0 && Gh != Mth<R>::ninf()) {
      const int d0 = ub - jown * kBlk;  // duration of the block's source 0 for target ub
      const int wb = d0 - (kBlk - 1);   // window start: durations wb .. wb+34
      if (wb <= K) {
        have = true;
        const int m = wb & 1;
        const R* wc = wt + (size_t)m * WSZ;
        const int e0 = wb + m;
        const int r0 = e0 >> 5, c0 = e0 & 31;
        R wv[kBlk + 4];
#pragma unroll
        for (int t2 = 0; t2 < (kBlk + 4) / 2; ++t2) {
          const int cc = c0 + 2 * t2;
          const int ph = r0 * 34 + cc + (cc >= 32 ? 2 : 0) + (cc >= 64 ? 2 : 0);
          const auto w2 = *(const typename Vec2<R>::T*)(wc + ph);
          wv[2 * t2] = w2.x;
          wv[2 * t2 + 1] = w2.y;
        }
#pragma unroll
        for (int jj = 0; jj < kBlk; ++jj) {
          const R zz = zr[jj];
          pb[0] += zz * wv[31 - jj];
          pb[1] += zz * wv[32 - jj];
          pb[2] += zz * wv[33 - jj];
          pb[3] += zz * wv[34 - jj];
        }
      }
    }
    // shared reference per target: the exact term of its newest source or the newest complete
    // block's value, whichever is larger; exact group maximum when a term would overflow it
    R Mv[4], Sv[4], xbv[4], xm[4];
    const int jnew = (sb >> 5) - 1;
    bool slow = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      xbv[i] = (have && pb[i] > (R)0) ? ((Gh + eh[i]) + (Gl + el[i])) + bmax : Mth<R>::ninf();
      xm[i] = xbv[i];
#pragma unroll
      for (int q = 0; q < Q; ++q) xm[i] = fmax(xm[i], xe[i][q]);
      const int ii = (sb & (kBlk - 1)) + i;  // index of source sb + i in the incomplete block (<= 31)
      R mine = Mth<R>::ninf();
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (ii / LB == q) mine = xe[i][q];
      const R rx = __shfl_sync(0xffffffffu, mine, gbase + (ii % LB));
      const R rb = __shfl_sync(0xffffffffu, xbv[i], gbase + (jnew & (LB - 1)));
      const R M = fmax(rx, rb);
      Mv[i] = M;
      slow |= (xm[i] > M + (R)kSlack) || (M == Mth<R>::ninf() && xm[i] != Mth<R>::ninf());
    }
    if (__any_sync(0xffffffffu, slow)) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        R v = xm[i];
#pragma unroll
        for (int o = LB / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        Mv[i] = v;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const R M = Mv[i];
      R sm = 0;
      if (M != Mth<R>::ninf()) {
        if (xbv[i] != Mth<R>::ninf()) sm += pb[i] * Mth<R>::ex2(xbv[i] - M);
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (xe[i][q] != Mth<R>::ninf()) sm += Mth<R>::ex2(xe[i][q] - M);
      }
      Sv[i] = sm;
    }
#pragma unroll
    for (int o = LB / 2; o > 0; o >>= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) Sv[i] += __shfl_xor_sync(0xffffffffu, Sv[i], o);
    }
    {
      R mi = Mv[0], si = Sv[0];
#pragma unroll
      for (int i = 1; i < 4; ++i)
        if (sl == i) {
          mi = Mv[i];
          si = Sv[i];
        }
      if (lact && sl < nt) {
        const int slt = (sb + sl) & (kSlots - 1);
        const uint32_t off = (uint32_t)(((size_t)slt * C + lo + cl) * 2 * sizeof(R));
        st_async_pair<R>(hpart + off, mi, si, hbar + (uint32_t)(slt * sizeof(uint64_t)));
      }
      if (lact && sl < 4 && ub + 4 * nahead + sl <= L) stage(ub + 4 * nahead + sl);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
}

template <typename R, int MODE>
__device__ void tail_main(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                          const TailLayout& TL) {
  const SweepGeo& g = a.geo;
  const int K = a.K, C = a.C;
  const int tid = threadIdx.x;
  const int lo = tail_lo(x.rank, C, g.G), Cg = tail_lo(x.rank + 1, C, g.G) - lo;
  R* B2 = (R*)(smem + TL.B2);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  if (g.TBlk) {
    const int WLEN = blk_wlen(g.kc, K);
    R* bx = (R*)(smem + TL.bx);
    R* wt = (R*)(smem + TL.wtab);
    for (int cl = tid; cl < Cg; cl += blockDim.x) {  // per-label max duration bias and near-duration table
      double m = -CUDART_INF;
      for (int k = g.kc + 1; k <= K; ++k) m = fmax(m, a.dur[(size_t)(k - 1) * C + lo + cl] * kLog2e);
      bx[(size_t)cl * (kBlk + 1) + kBlk] = (R)m;
      for (int i = 0; i < kBlk; ++i) {
        const int k = g.kc + 1 + i;
        bx[(size_t)cl * (kBlk + 1) + i] = k <= K ? (R)(a.dur[(size_t)(k - 1) * C + lo + cl] * kLog2e) : Mth<R>::ninf();
      }
    }
    __syncthreads();
    const int WSZ = blk_wsize(g.kc, K);
    for (int i = tid; i < Cg * 2 * WLEN; i += blockDim.x) {
      const int cl = i / (2 * WLEN), r = i % (2 * WLEN), m = r / WLEN, y = r % WLEN;
      const int k = y - m;  // copy m holds w[y - m]
      R v = 0;
      if (k >= g.kc + 1 && k <= K) {
        const R bm = bx[(size_t)cl * (kBlk + 1) + kBlk];
        v = Mth<R>::ex2((R)(a.dur[(size_t)(k - 1) * C + lo + cl] * kLog2e) - bm);
      }
      wt[((size_t)cl * 2 + m) * WSZ + blk_wphys(y)] = v;
    }
  } else {
    for (int i = tid; i < Cg * K; i += blockDim.x) {
      const int cl = i / K, k = i % K;
      B2[i] = (R)(a.dur[(size_t)k * C + lo + cl] * kLog2e);
    }
  }
  if (tid < kSlots) mbar_init(smem_u32(&tbar[tid]), 1);
  __syncthreads();
  if (tid == 0) {
    mbar_fence_init();
    for (int q = 0; q < kSlots; ++q) mbar_expect(smem_u32(&tbar[q]), (uint32_t)(Cg * 2 * sizeof(R) + sizeof(double)));
  }
  __syncthreads();
  cluster_sync_all();
  if ((tid >> 5) < g.NWt) {
    if (g.TBlk == 8)
      tail_loop_blocked_ml<R, 8, MODE == 3>(a, x, smem, HL, TL, lo, Cg);
    else if (g.TBlk == 16)
      tail_loop_blocked_ml<R, 16, MODE == 3>(a, x, smem, HL, TL, lo, Cg);
    else if (g.TBlk)
      tail_loop_blocked<R, MODE == 3>(a, x, smem, HL, TL, lo, Cg);
    else
      tail_loop<R, MODE == 3>(a, x, smem, HL, TL, lo, Cg);
  }
}

// ----------------------------------------------------------------------------

// MODE: 0 = full sweep (every position stored), 1 = checkpoint-row sweep (sublinear pass 1,
// bookkeeping in the chain), 2 = window replay (SweepTask per cluster, forced start)
template <typename R, bool TAILS, bool CW1, int MODE>
__global__ void __launch_bounds__(512) sweep_kernel(SweepArgs<R> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SweepGeo& g = a.geo;
  const int ci = blockIdx.x / g.G;
  SweepCtx x;
  x.task = nullptr;
  if (MODE == 2) {
    x.task = a.tasks + ci;
    x.b = x.task->b;
    x.dir = x.task->dir;
  } else if (a.dirs == 3) {
    x.b = ci >> 1;
    x.dir = ci & 1;
  } else {
    x.b = ci;
    x.dir = a.dirs == 1 ? 0 : 1;
  }
  x.rank = blockIdx.x % g.G;
  x.Lb = (int)a.lengths[x.b];
  if (x.task) {
    x.L = x.task->steps;
    x.t0 = x.task->t0;
    if (x.L < 0) return;  // empty task (sequence shorter than the window): the whole cluster exits
  } else {
    x.L = x.Lb;
    x.t0 = x.dir == 0 ? 0 : x.Lb;
  }
  x.S = a.S + (size_t)x.b * (a.T + 1) * a.C;
  x.ps = a.ps ? a.ps + (size_t)x.b * a.T * a.C : nullptr;
  x.pe = a.pe ? a.pe + (size_t)x.b * a.T * a.C : nullptr;
  if (MODE == 3) {  // streamed input: the first rows every CTA may read before the loop
    if (threadIdx.x == 0) gate_span_wait(a, x, 0, min(x.L, 320));
    __syncthreads();
  }
  const HeadLayout HL = head_layout<R>(a.K, a.C, g);
  const TailLayout TL = tail_layout<R>(a.K, a.C, g);
#ifdef SCRF_TRACE
  // globaltimer offset calibration (cluster 0): head thread 0 and tail 1 thread 0 ping-pong
  // 64 times through global flags at a.trace + 1280*16 (sends, echoes, receives)
  if (a.trace && TAILS && blockIdx.x < 2 && threadIdx.x == 0) {
    volatile long long* cb = a.trace + 1280 * 16;
    for (int i = 0; i < 64; ++i) {
      if (blockIdx.x == 0) {
        cb[i] = gtimer();
        __threadfence();
        while (cb[64 + i] == 0) {
        }
        cb[128 + i] = gtimer();
      } else {
        while (cb[i] == 0) {
        }
        cb[64 + i] = gtimer();
        __threadfence();
      }
    }
  }
#endif
  if (x.rank == 0)
    head_main<R, TAILS, CW1, MODE>(a, x, smem, HL, TL);
  else if (TAILS)
    tail_main<R, MODE>(a, x, smem, HL, TL);
  if (TAILS) cluster_sync_all();
}

// ----------------------------------------------------------------------------
// Reference bookkeeping of a full-mode alpha sweep (streaming.py:194-229) from the stored
// per-position normalisers n_t and max shifts (off the latency-bound chain): checkpoint
// normalisers N_i (shift = max_c alpha at i*delta, applied only while the sequence is alive,
// frozen past L), the first dead position (the chain marks it with a max shift of -inf), the
// positions where the reference would clamp the max message to +-1e6 relative to the
// normaliser in effect (_numerics.py:41-56), and logZ = LSE_c alpha[L,c]; the reference raises
// only when the final log-partition is dead. One block per sequence.
template <typename R>
__global__ void __launch_bounds__(1024) book_kernel(const R* Ya, const double* na, const R* amx, const int64_t* lengths,
                                                   int T, int C, int delta, int n_ckpt, double* N, int32_t* dead_at,
                                                   double* logZ, int32_t* clamp) {
  const int b = blockIdx.x;
  const int L = (int)lengths[b];
  const size_t rb = (size_t)b * (T + 1);
  double* Nb = N + (size_t)b * n_ckpt;  // N in effect from checkpoint i on
  __shared__ int dmin, ncl;
  if (threadIdx.x == 0) {
    double N_cur = 0.0;
    Nb[0] = 0.0;
    for (int i = 1; i < n_ckpt; ++i) {
      const long long q = (long long)i * delta;
      if (q <= L && amx[rb + q] != Mth<R>::ninf()) N_cur = na[rb + q] * kLn2;
      Nb[i] = N_cur;
    }
    dmin = 0x7fffffff;
    ncl = 0;
  }
  __syncthreads();
  int best = 0x7fffffff, cl = 0;
  for (int q = 1 + threadIdx.x; q <= L; q += blockDim.x) {
    if (amx[rb + q] == Mth<R>::ninf()) {
      best = min(best, q);
    } else {
      int i = (q - 1) / delta;  // normaliser in effect before the shift at q
      if (i >= n_ckpt) i = n_ckpt - 1;
      if (fabs(na[rb + q] * kLn2 - Nb[i]) > kClampLimit) ++cl;
    }
  }
  atomicMin(&dmin, best);
  atomicAdd(&ncl, cl);
  __syncthreads();
  if (threadIdx.x < 32) {
    R s = 0;
    for (int c = threadIdx.x; c < C; c += 32) s += Mth<R>::ex2(Ya[(rb + L) * C + c]);
    s = group_sum(s, 32);
    if (threadIdx.x == 0) {
      const double lz = (s > (R)0) ? (na[rb + L] + (double)Mth<R>::lg2(s)) * kLn2 : -CUDART_INF;
      logZ[b] = lz;
      const double Nfin = Nb[n_ckpt - 1 < (L / delta) ? n_ckpt - 1 : (L / delta)];
      dead_at[b] = (lz - Nfin > kGuard) ? -1 : (dmin == 0x7fffffff ? L : dmin);
      if (clamp) clamp[b] = ncl;
    }
  }
}

}  // namespace scrf
