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

constexpr int kSlots = 16;      // head <-> tail mbarrier ring depth (power of two, > kNear)
constexpr int kNear = 16;       // durations handled by the head when the cluster has tails
constexpr int kStage = 16;      // staged positions (power of two)
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

struct SweepGeo {
  int G;      // CTAs per cluster: head + G-1 tails
  int kc;     // head durations 1..kc (K when G == 1)
  int KRm;    // head source ring: power-of-two slots - 1
  int KTm;    // tail source ring: power-of-two slots - 1
  int NCW;    // chain warps (ceil(C/32)); aux warps = NCW
  int NNW;    // near warps
  int GWn;    // near threads per label (power of two <= 32)
  int NWt;    // tail warps
  int WPL;    // tail warps per label (each pushes its own partial)
  int TBlk;   // 1: blocked tails (exp-space source blocks, FMA); 0: exact per-term tails
  int PsRow;  // staged row holding Ps[t] (0 = no proj_start)
  int PeRow;  // staged row holding Pe[t-1] (0 = no proj_end)
  int CgMax;  // max labels per tail
  int NT;     // block size (max over roles)
  int Msm;    // exp-space transition matrix staged in shared memory
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
  double* N;         // [B][n_ckpt] reference checkpoint normalisers
  int delta, n_ckpt;
  long long* trace;  // debug: [256][16] clock64 stamps of cluster 0 (chain lane 0: 0..7, near thread 0: 8..15)
  int trace_from;    // first traced position
  int* hang;         // debug: watchdog record {block, thread, site, index} (first writer wins), or null
};

// mbarrier wait with an optional watchdog (a.hang != null): after ~1e8 polls record where
// and trap instead of hanging the device.
template <typename A>
__device__ __forceinline__ void sweep_wait(const A& a, uint32_t bar, uint32_t parity, int site, int idx) {
  if (!a.hang) {
    mbar_wait(bar, parity);
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
__host__ __device__ inline int blk_wlen(int kc) { return (1024 + 64 + kc + 1) & ~1; }
// w is stored in rows of 32 elements with a row stride of 34: lanes read windows that start
// 32*j elements apart, which the skew spreads over all banks (pairs never straddle a row)
__host__ __device__ inline int blk_wrow() { return 34; }
__host__ __device__ inline int blk_wphys(int e) { return (e >> 5) * 34 + (e & 31); }
__host__ __device__ inline int blk_wsize(int kc) { return (blk_wlen(kc) / 32 + 2) * 34; }

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
  L.ring = o;  o += a16((size_t)2 * C * ring_stride(g.KRm) * 2 * sizeof(R));  // one ring per near group
  L.stg = o;   o += a16((size_t)kStage * (1 + (g.PsRow > 0) + (g.PeRow > 0)) * C * sizeof(double));
  L.oq = o;    o += a16((size_t)kStage * C * 2 * sizeof(double));
  L.own = o;   o += a16((size_t)C * sizeof(int2));
  L.pubY = o;  o += a16((size_t)8 * C * sizeof(R));
  L.pubX = o;  o += a16((size_t)8 * C * sizeof(R));
  L.pubA = o;  o += a16(8 * sizeof(R));
  L.nring = o; o += a16(kNring * sizeof(double));
  L.part = o;  o += a16((size_t)4 * C * 2 * sizeof(R));
  L.hh = o;    o += a16((size_t)8 * C * 2 * sizeof(R));
  L.h3 = o;    o += a16((size_t)8 * C * sizeof(R));
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
  L.wtab = o;  o += g.TBlk ? a16((size_t)g.CgMax * 2 * blk_wsize(g.kc) * sizeof(R)) : 0;
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
  int b, dir, L, rank;
  const double* S;   // row base of sequence b: S + b*(T+1)*C
  const double* ps;  // proj_start rows of b or null
  const double* pe;
  __device__ __forceinline__ int tpos(int p) const { return dir == 0 ? p : L - p; }
};

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
  R2* hh;
  R* h3;
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
  h.hh = (R2*)(base + L.hh);
  h.h3 = (R*)(base + L.h3);
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

// edge terms of target u for label c: hk = O[u] + Q[u-k] + B[k-1] for k = 1, 2, 3
template <typename R>
__device__ __forceinline__ void head_edge(int C, int K, const double2* oq, const R* B2, int kc, int u, int c,
                                          typename Vec2<R>::T* hh, R* h3) {
  const double O = oq[(size_t)(u & (kStage - 1)) * C + c].x;
  const R* b2 = B2 + (size_t)c * b2_stride(kc);
  typename Vec2<R>::T v;
  v.x = (R)(O + oq[(size_t)((u - 1) & (kStage - 1)) * C + c].y + (double)b2[0]);
  v.y = (u >= 2 && K >= 2) ? (R)(O + oq[(size_t)((u - 2) & (kStage - 1)) * C + c].y + (double)b2[1]) : Mth<R>::ninf();
  hh[(size_t)(u & 7) * C + c] = v;
  h3[(size_t)(u & 7) * C + c] =
      (u >= 3 && K >= 3) ? (R)(O + oq[(size_t)((u - 3) & (kStage - 1)) * C + c].y + (double)b2[2]) : Mth<R>::ninf();
}

// log2(2^m s + 2^x3 + 2^x2 + 2^x1)
template <typename R>
__device__ __forceinline__ R lse4(R m, R s, R x3, R x2, R x1) {
  const R mm = (s > (R)0) ? m : Mth<R>::ninf();
  const R M = fmax(fmax(mm, x3), fmax(x2, x1));
  if (M == Mth<R>::ninf()) return M;
  R sum = (Mth<R>::ex2(x3 - M) + Mth<R>::ex2(x2 - M)) + Mth<R>::ex2(x1 - M);
  if (mm != Mth<R>::ninf()) sum += s * Mth<R>::ex2(mm - M);
  return M + Mth<R>::lg2(sum);
}

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

// Barrier bookkeeping. A(q): id 1 + (q & 3); the chain arrives, the aux warps and the near
// group (q & 1) sync; count NA. B(p): id 5 + (p & 3); near group (p & 1) arrives, the chain
// syncs; count NB. Every id is used with one count only.

// ======================= chain warps =======================
template <typename R, bool CW1>
__device__ void head_chain(const SweepArgs<R>& a, const SweepCtx& x, HeadPtr<R>& h, int NA, int NB) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, L = x.L;
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
  const R xmax = act ? h.Xmax[c] : (R)0;
  // X^[x] = xmax[x] + log2 sum_y 2^(yh[y]) M[y][x]
  auto gemv = [&](R yh) -> R {
    const R e = act ? Mth<R>::ex2(yh) : (R)0;
    R s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (CW1) {
      h.ew[lane] = e;
      __syncwarp();
#pragma unroll
      for (int y = 0; y < 32; y += 4) {
        if (y < C) {
          const R e0 = h.ew[y], e1 = h.ew[y + 1], e2 = h.ew[y + 2], e3 = h.ew[y + 3];
          s0 += e0 * Mreg[y];
          s1 += e1 * Mreg[y + 1];
          s2 += e2 * Mreg[y + 2];
          s3 += e3 * Mreg[y + 3];
        }
      }
      __syncwarp();
    } else {
      if (act) h.ew[c] = e;
      nbar_sync(BAR_CH2, nch);
      if (act) {
        int y = 0;
        for (; y + 4 <= C; y += 4) {
          s0 += h.ew[y] * Mval(y);
          s1 += h.ew[y + 1] * Mval(y + 1);
          s2 += h.ew[y + 2] * Mval(y + 2);
          s3 += h.ew[y + 3] * Mval(y + 3);
        }
        for (; y < C; ++y) s0 += h.ew[y] * Mval(y);
      }
      nbar_sync(BAR_CH, nch);
    }
    const R sum = (s0 + s1) + (s2 + s3);
    R out = xmax + Mth<R>::lg2(sum);
    const bool slow = act && !(sum >= (R)1e-30);
    if (__any_sync(0xffffffffu, slow)) out = gemv_exact<R>(a.trans, x.dir, C, g.NCW, h.ew, yh, act, c, slow, out);
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

  // position 0: alpha[0] = 0 (virtual source) / beta[L] = 0
  const R yh0 = x.dir == 0 ? (R)0 : Mth<R>::ninf();
  R x1h = x.dir == 0 ? gemv((R)0) : (R)0;  // X^[p-1]
  R x2h = Mth<R>::ninf();                    // X^[p-2]
  R x3h = Mth<R>::ninf();                    // X^[p-3]
  if (act) {
    h.pubY[c] = yh0;
    h.pubX[c] = x1h;
  }
  if (tid == 0) {
    h.pubA[0] = 0;
    h.nring[0] = 0.0;
  }
  nbar_arrive(BAR_A + 0, NA);
  R a1 = 0, a2 = 0, a3 = 0;  // frame shifts amax_{p-1}, amax_{p-2}, amax_{p-3}
  double n_prev = 0.0;
  const int cs = act ? c : 0;
  const R2* partc = h.part + cs;
  const R2* hhc = h.hh + cs;
  const R* h3c = h.h3 + cs;
  for (int p = 1; p <= L; ++p) {
    long long* tr = (a.trace && blockIdx.x == 0 && tid == 0 && p >= a.trace_from && p < a.trace_from + 256) ? a.trace + (p - a.trace_from) * 16 : nullptr;
    if (tr) tr[0] = clock64();
    nbar_sync(BAR_B + (p & 3), NB);
    R y = Mth<R>::ninf();
    if (act) {
      const R2 pm = partc[(p & 3) * C];  // frame n_{p-4}
      const R2 hv = hhc[(p & 7) * C];
      const R hv3 = h3c[(p & 7) * C];
      const R s12 = a2 + a1;
      y = lse4(pm.x - a3 - s12, pm.y, x3h + hv3 - s12, x2h + hv.y - a1, x1h + hv.x);
    }
    if (tr) tr[1] = clock64();
    const R am = chain_max(y);
    const bool dead = (am == Mth<R>::ninf());
    const R yh = dead ? Mth<R>::ninf() : y - am;
    const double n_p = dead ? n_prev : n_prev + (double)am;
    const R xh = gemv(yh);
    if (tr) tr[2] = clock64();
    if (act) {
      h.pubY[(p & 7) * C + c] = yh;
      h.pubX[(p & 7) * C + c] = xh;
    }
    if (tid == 0) {
      h.pubA[p & 7] = am;
      h.nring[p & (kNring - 1)] = n_p;
    }
    nbar_arrive(BAR_A + (p & 3), NA);
    if (tr) tr[3] = clock64();
    x3h = x2h;
    x2h = x1h;
    x1h = xh;
    a3 = a2;
    a2 = a1;
    a1 = dead ? (R)0 : am;
    n_prev = n_p;
  }
}

// ======================= near warps =======================
// Two groups of NNW/2 warps; group gi owns the targets p with (p & 1) == gi. Iteration p
// waits A(p-4), appends the sources p-5, p-4 to the group's ring, sums durations 4..kc of
// target p (+ the tail partial, durations kc+1..K) in frame n_{p-4}, and arrives B(p).
template <typename R, bool TAILS>
__device__ void head_near(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, HeadPtr<R>& h,
                          const TailLayout& TL, int NA, int NB) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, L = x.L;
  const int kc = g.kc, KRm = g.KRm, KTm = g.KTm;
  const int ntid = threadIdx.x - g.NCW * 32;
  const int ngw = g.NNW >> 1;          // warps per group
  const int gi = (ntid >> 5) / ngw;    // group
  const int gtid = ntid - gi * ngw * 32;
  const int gthr = ngw * 32;
  const int GW = g.GWn;
  const int c = gtid / GW, j = gtid % GW;  // one label per lane group
  const bool act = c < C;
  const int cs = act ? c : 0;
  const int nsend_max = L - kc - 1;  // last source any tail needs
  R2* ringc = h.ring + ((size_t)gi * C + cs) * ring_stride(KRm);
  const R* b2c = h.B2 + (size_t)cs * b2_stride(kc);
  const R b4 = kc >= 4 ? b2c[3] : (R)0;
  const double2* oqc = h.oq + cs;
  const R* pubXc = h.pubX + cs;
  const R2* tpartc = h.tpart + cs;
  R2* partc = h.part + cs;
  // remote (tail) addresses for this label's sources and the n messages
  uint32_t t_ring = 0, t_bar = 0, t_nslot = 0, t_nbar = 0;
  const bool nsender = TAILS && gtid >= gthr - (g.G - 1);
  if (TAILS) {
    const int2 ow = h.own[cs];
    t_ring = mapa_u32(smem_u32(smem + TL.ring) + (uint32_t)((size_t)ow.y * (KTm + 1) * 2 * sizeof(R)), ow.x);
    t_bar = mapa_u32(smem_u32(smem + TL.tbar), ow.x);
    if (nsender) {
      const int rt = gtid - (gthr - (g.G - 1)) + 1;
      t_nslot = mapa_u32(smem_u32(smem + TL.nslot), rt);
      t_nbar = mapa_u32(smem_u32(smem + TL.tbar), rt);
    }
  }
  auto source = [&](int q) -> R2 {  // r[q] = n_q + X^[q] + Q[q] as an fp32 (hi, lo) pair
    const R X = pubXc[(q & 7) * C];
    const double r = (X == Mth<R>::ninf()) ? -CUDART_INF
                                            : h.nring[q & (kNring - 1)] + ((double)X + oqc[(size_t)(q & (kStage - 1)) * C].y);
    R2 v;
    split2(r, v.x, v.y);
    return v;
  };
  for (int p = gi == 0 ? 2 : 1; p <= L + 4; p += 2) {
    long long* tr = (a.trace && blockIdx.x == 0 && ntid == 0 && p >= a.trace_from && p < a.trace_from + 256) ? a.trace + (p - a.trace_from) * 16 + 8 : nullptr;
    if (tr) tr[0] = clock64();
    if (p >= 4) nbar_sync(BAR_A + ((p - 4) & 3), NA);
    if (tr) tr[1] = clock64();
    if (p > L) continue;
    const int q = p - 4;  // newest source; frame n_q
    const int kmax = min(kc, p);
    R m = Mth<R>::ninf(), s = 0;
    double n_q = 0.0;
    if (q >= 0) {
      n_q = h.nring[q & (kNring - 1)];
      R2 r4;
      r4.x = Mth<R>::ninf();
      r4.y = 0;
      R e_hi = 0, e_lo = 0;
      if (act) {
        r4 = source(q);
        split2(oqc[(size_t)(p & (kStage - 1)) * C].x - n_q, e_hi, e_lo);
        if (tr) tr[7] = clock64();
        if (j == 0) {
          ringc[q & KRm] = r4;
          if (q >= 1) ringc[(q - 1) & KRm] = source(q - 1);
          if (TAILS && q <= nsend_max)
            st_async_pair<R>(t_ring + (uint32_t)((q & KTm) * 2 * sizeof(R)), r4.x, r4.y,
                             t_bar + (uint32_t)((q & (kSlots - 1)) * sizeof(uint64_t)));
        }
      }
      if (TAILS && nsender && q <= nsend_max)
        st_async_f64(t_nslot + (uint32_t)((q & (kSlots - 1)) * sizeof(double)), n_q,
                     t_nbar + (uint32_t)((q & (kSlots - 1)) * sizeof(uint64_t)));
      nbar_sync(BAR_NG + gi, gthr);  // the group's ring holds sources <= q
      if (tr) tr[2] = clock64();
      const R mref = (act && kmax >= 4) ? (r4.x + e_hi) + (r4.y + e_lo) + b4 : Mth<R>::ninf();
      // durations 5..kmax from the ring (k = 4 is the shared reference)
      ring_lse<R>(ringc, KRm, b2c, 5 + j, GW, act ? kmax : 0, (q - 1 - j) & KRm, e_hi, e_lo, mref,
                  j == 0 && act && kmax >= 4, GW, m, s);
      if (tr) tr[3] = clock64();
    }
    if (TAILS && p >= kc + 1) {
      const int pi = p - kc - 1;
      const int sl = pi & (kSlots - 1);
      if (tr) tr[5] = clock64();
      sweep_wait(a, smem_u32(&h.tbar[sl]), (uint32_t)((pi / kSlots) & 1), 1, p);
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

// ======================= aux warps =======================
template <typename R>
__device__ void head_aux(const SweepArgs<R>& a, const SweepCtx& x, HeadPtr<R>& h, int NA) {
  const SweepGeo& g = a.geo;
  const int K = a.K, C = a.C, T = a.T, L = x.L;
  const int c = threadIdx.x - (g.NCW + g.NNW) * 32;  // lane = label
  const bool act = c < C;
  const size_t rowbase = (size_t)x.b * (T + 1);
  R* Yo = a.Y[x.dir] + rowbase * C + (act ? c : 0);
  R* Xo = a.X[x.dir] + rowbase * C + (act ? c : 0);
  double* no = a.n[x.dir] + rowbase;
  const int tstep = x.dir == 0 ? 1 : -1;
  double N_cur = 0.0;
  int dead_at = -1;
  int to_ck = 0;  // positions until the next checkpoint boundary
  const bool book = (x.dir == 0) && c == 0;
  const R* pYc = h.pubY + (act ? c : 0);
  const R* pXc = h.pubX + (act ? c : 0);
  int t = x.tpos(0);
  for (int q = 0; q <= L; ++q, t += tstep) {
    cp_async_wait<6>();  // own rows of position q+5 (issued at iteration q-7)
    nbar_sync(BAR_A + (q & 3), NA);
    const double n_q = h.nring[q & (kNring - 1)];
    if (act) {
      Yo[(size_t)t * C] = pYc[(q & 7) * C];
      Xo[(size_t)t * C] = pXc[(q & 7) * C];
      if (q + 5 <= L) h.oq[(size_t)((q + 5) & (kStage - 1)) * C + c] = oq_of(x, g, C, h.stg, q + 5, c);
      if (q + 4 <= L) head_edge<R>(C, K, h.oq, h.B2, g.kc, q + 4, c, h.hh, h.h3);
      if (q + kAhead <= L) stage_label<true>(x, g, T, C, h.stg, q + kAhead, c);
    }
    cp_async_commit();
    if (c == 0) no[t] = n_q;
    if (book) {
      // reference bookkeeping in nats (streaming.py:194-225): dead check and checkpoint shifts
      const R am = h.pubA[q & 7];
      const bool dead = (am == Mth<R>::ninf());
      const double amax_abs = dead ? -CUDART_INF : n_q * kLn2;
      const bool at_ck = (to_ck == 0);
      if (q >= 1) {
        if (dead_at < 0 && !(amax_abs - N_cur > kGuard)) dead_at = q;
        if (at_ck && amax_abs - N_cur > kGuard) N_cur = amax_abs;
        if (at_ck && q / a.delta < a.n_ckpt) a.N[(size_t)x.b * a.n_ckpt + q / a.delta] = N_cur;
      } else {
        a.N[(size_t)x.b * a.n_ckpt] = 0.0;
      }
      to_ck = at_ck ? a.delta - 1 : to_ck - 1;
      if (q == L) {
        const R* pY = h.pubY + (q & 7) * C;
        R ssum = 0;
        if (!dead)
          for (int cc = 0; cc < C; ++cc) ssum += Mth<R>::ex2(pY[cc]);
        const double lz = dead ? -CUDART_INF : (n_q + (double)Mth<R>::lg2(ssum)) * kLn2;
        a.logZ[x.b] = lz;
        if (!(lz - N_cur > kGuard) && dead_at < 0) dead_at = L;
        for (int i = L / a.delta + 1; i < a.n_ckpt; ++i) a.N[(size_t)x.b * a.n_ckpt + i] = N_cur;
        a.dead_at[x.b] = dead_at;
      }
    }
    if (x.dir == 1 && q == L && c == 0) {
      const R* pX = h.pubX + (q & 7) * C;
      R mx = Mth<R>::ninf();
      for (int cc = 0; cc < C; ++cc) mx = fmax(mx, pX[cc]);
      R ssum = 0;
      if (mx != Mth<R>::ninf())
        for (int cc = 0; cc < C; ++cc) ssum += Mth<R>::ex2(pX[cc] - mx);
      a.logZb[x.b] = (mx == Mth<R>::ninf()) ? -CUDART_INF : (n_q + (double)mx + (double)Mth<R>::lg2(ssum)) * kLn2;
    }
  }
  cp_async_wait<0>();
}

template <typename R, bool TAILS, bool CW1>
__device__ void head_main(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                          const TailLayout& TL) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int K = a.K, C = a.C, T = a.T, L = x.L;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int NA = (2 * g.NCW + (g.NNW >> 1)) * 32;  // chain + aux + one near group
  const int NB = (g.NCW + (g.NNW >> 1)) * 32;      // chain + one near group
  const int NH = (2 * g.NCW + g.NNW) * 32;         // all head threads
  HeadPtr<R> h = head_ptrs<R>(smem, HL);
  const int kc = g.kc;

  // ---- tables and synchronous staging of positions 0 .. kAhead-1
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
    for (int i = tid; i < 2 * C * ring_stride(g.KRm); i += NH) {
      R2 v;
      v.x = Mth<R>::ninf();
      v.y = 0;
      h.ring[i] = v;
    }
    if (TAILS && tid < kSlots) mbar_init(smem_u32(&h.tbar[tid]), 1);
    for (int i = tid; i < kAhead * C; i += NH) {
      const int q = i / C, cc = i % C;
      if (q <= L) stage_label<false>(x, g, T, C, h.stg, q, cc);
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
    for (int i = tid; i < 5 * C; i += NH) {  // (O, Q) of positions 0..4
      const int q = i / C, cc = i % C;
      if (q <= L) h.oq[(size_t)q * C + cc] = oq_of(x, g, C, h.stg, q, cc);
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
  }
  __syncthreads();
  if (tid < NH) {
    for (int i = tid; i < 3 * C; i += NH) {  // edge terms of targets 1..3
      const int u = 1 + i / C, cc = i % C;
      if (u <= L) head_edge<R>(C, K, h.oq, h.B2, kc, u, cc, h.hh, h.h3);
    }
    if (TAILS && tid == 0) {
      mbar_fence_init();
      for (int q = 0; q < kSlots; ++q) mbar_expect(smem_u32(&h.tbar[q]), (uint32_t)(g.WPL * C * 2 * sizeof(R)));
    }
  }
  __syncthreads();
  if (TAILS) cluster_sync_all();

  if (warp < g.NCW)
    head_chain<R, CW1>(a, x, h, NA, NB);
  else if (warp < g.NCW + g.NNW)
    head_near<R, TAILS>(a, x, smem, h, TL, NA, NB);
  else if (warp < 2 * g.NCW + g.NNW)
    head_aux<R>(a, x, h, NA);
}

// ----------------------------------------------------------------------------
// tail CTA: durations kc+1..K of a label slice (one warp per label), ahead of the chain

template <typename R>
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
  auto stage = [&](int u, int cl) {
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
    long long* tr = (a.trace && blockIdx.x == 1 && threadIdx.x == 0 && u >= a.trace_from && u < a.trace_from + 256) ? a.trace + 256 * 16 + (u - a.trace_from) * 16 : nullptr;
    if (tr) tr[0] = clock64();
    cp_async_wait<kAhead - 1>();
    __syncwarp();
    if (tr) tr[1] = clock64();
    sweep_wait(a, smem_u32(&tbar[s_new & (kSlots - 1)]), (uint32_t)((s_new / kSlots) & 1), 2, u);
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
template <typename R>
__device__ void tail_loop_blocked(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                                  const TailLayout& TL, int lo, int Cg) {
  using R2 = typename Vec2<R>::T;
  const SweepGeo& g = a.geo;
  const int C = a.C, T = a.T, L = x.L, kc = g.kc, KTm = g.KTm, K = a.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = warp;  // one label per warp
  const R2* rg = (const R2*)(smem + TL.ring) + (size_t)cl * (KTm + 1);
  const double* nslot = (const double*)(smem + TL.nslot);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  double* stg = (double*)(smem + TL.stg);
  const int WSZ = blk_wsize(kc);
  const R* wt = (const R*)(smem + TL.wtab) + (size_t)cl * 2 * WSZ;
  const R* bx = (const R*)(smem + TL.bx) + (size_t)cl * (kBlk + 1);
  const R bmax = bx[kBlk];
  auto stage = [&](int u) {
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
  const int u0 = kc + 1;
  // staging runs 3 groups (12 targets) ahead; one commit group per 4 targets
  for (int gq = 0; gq < 3; ++gq) {
    if (lane == 0)
      for (int i = 0; i < 4; ++i)
        if (u0 + 4 * gq + i <= L) stage(u0 + 4 * gq + i);
    cp_async_commit();
  }
  const uint32_t hbar = mapa_u32(smem_u32(smem + HL.tbar), 0);
  const uint32_t hpart = mapa_u32(smem_u32(smem + HL.tpart), 0);
  R zr[kBlk];
#pragma unroll
  for (int i = 0; i < kBlk; ++i) zr[i] = 0;
  R Gh = Mth<R>::ninf(), Gl = 0;
  int jown = -1;
  for (int ub = u0; ub <= L; ub += 4) {
    const int sb = ub - kc - 1;          // newest source of target ub (multiple of 4)
    const int nt = min(4, L - ub + 1);   // targets in this group
    long long* tr = (a.trace && blockIdx.x == 1 && threadIdx.x == 0 && ub >= a.trace_from && ub < a.trace_from + 4 * 256)
                        ? a.trace + 256 * 16 + ((ub - a.trace_from) / 4) * 16
                        : nullptr;
    if (tr) tr[0] = clock64();
    cp_async_wait<2>();
    __syncwarp();
    // the group's sources sb .. sb+nt-1 (and their normalisers)
    for (int i = 0; i < nt; ++i) {
      const int s = sb + i;
      sweep_wait(a, smem_u32(&tbar[s & (kSlots - 1)]), (uint32_t)((s / kSlots) & 1), 2, s);
    }
    if (tr) tr[1] = clock64();
    R eh[4], el[4];
    double Fi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      eh[i] = 0;
      el[i] = 0;
      Fi[i] = 0.0;
      if (i < nt) {
        const int u = ub + i;
        Fi[i] = nslot[(sb + i) & (kSlots - 1)];
        const double* d = stg + ((size_t)(u & (kStage - 1)) * g.CgMax + cl) * 2;
        const double s2 = d[0] * kLog2e, o2 = d[1] * kLog2e;
        split2((x.dir == 0 ? s2 + o2 : -s2 + o2) - Fi[i], eh[i], el[i]);
      }
    }
    __syncwarp();
    if (threadIdx.x == 0)
      for (int i = 0; i < nt; ++i) {
        const int s = sb + i;
        if (s + kSlots <= L - kc - 1)
          mbar_expect(smem_u32(&tbar[s & (kSlots - 1)]), (uint32_t)(Cg * 2 * sizeof(R) + sizeof(double)));
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
    R Mv[4], Sv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const R xb = (have && pb[i] > (R)0) ? ((Gh + eh[i]) + (Gl + el[i])) + bmax : Mth<R>::ninf();
      const R M = warp_max(fmax(xb, xe[i]));
      R sm = 0;
      if (M != Mth<R>::ninf()) {
        if (xb != Mth<R>::ninf()) sm += pb[i] * Mth<R>::ex2(xb - M);
        if (xe[i] != Mth<R>::ninf()) sm += Mth<R>::ex2(xe[i] - M);
      }
      Mv[i] = M;
      Sv[i] = sm;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) Sv[i] += __shfl_xor_sync(0xffffffffu, Sv[i], off);
    }
    if (lane == 0) {
      for (int i = 0; i < nt; ++i) {
        const int sl = (sb + i) & (kSlots - 1);
        const uint32_t off = (uint32_t)(((size_t)sl * C + lo + cl) * 2 * sizeof(R));
        st_async_pair<R>(hpart + off, Mv[i], Sv[i], hbar + (uint32_t)(sl * sizeof(uint64_t)));
      }
      for (int i = 0; i < 4; ++i)
        if (ub + 12 + i <= L) stage(ub + 12 + i);
    }
    cp_async_commit();
    // block (sb+3)/32 completes after this group: frame = its largest source, z to its owner lane
    if (nt == 4 && ((sb + 3) & (kBlk - 1)) == kBlk - 1) {
      const int jb = (sb + 3) >> 5;
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
    }
    if (tr) tr[3] = clock64();
  }
  cp_async_wait<0>();
}

template <typename R>
__device__ void tail_main(const SweepArgs<R>& a, const SweepCtx& x, unsigned char* smem, const HeadLayout& HL,
                          const TailLayout& TL) {
  const SweepGeo& g = a.geo;
  const int K = a.K, C = a.C;
  const int tid = threadIdx.x;
  const int lo = tail_lo(x.rank, C, g.G), Cg = tail_lo(x.rank + 1, C, g.G) - lo;
  R* B2 = (R*)(smem + TL.B2);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  if (g.TBlk) {
    const int WLEN = blk_wlen(g.kc);
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
    const int WSZ = blk_wsize(g.kc);
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
    if (g.TBlk)
      tail_loop_blocked<R>(a, x, smem, HL, TL, lo, Cg);
    else
      tail_loop<R>(a, x, smem, HL, TL, lo, Cg);
  }
}

// ----------------------------------------------------------------------------

template <typename R, bool TAILS, bool CW1>
__global__ void __launch_bounds__(512) sweep_kernel(SweepArgs<R> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SweepGeo& g = a.geo;
  const int ci = blockIdx.x / g.G;
  SweepCtx x;
  if (a.dirs == 3) {
    x.b = ci >> 1;
    x.dir = ci & 1;
  } else {
    x.b = ci;
    x.dir = a.dirs == 1 ? 0 : 1;
  }
  x.rank = blockIdx.x % g.G;
  x.L = (int)a.lengths[x.b];
  x.S = a.S + (size_t)x.b * (a.T + 1) * a.C;
  x.ps = a.ps ? a.ps + (size_t)x.b * a.T * a.C : nullptr;
  x.pe = a.pe ? a.pe + (size_t)x.b * a.T * a.C : nullptr;
  const HeadLayout HL = head_layout<R>(a.K, a.C, g);
  const TailLayout TL = tail_layout<R>(a.K, a.C, g);
  if (x.rank == 0)
    head_main<R, TAILS, CW1>(a, x, smem, HL, TL);
  else if (TAILS)
    tail_main<R>(a, x, smem, HL, TL);
  if (TAILS) cluster_sync_all();
}

}  // namespace scrf
