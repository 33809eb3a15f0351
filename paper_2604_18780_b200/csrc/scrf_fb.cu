// Streaming semi-CRF forward / backward on B200 (sm_100a).
//
// Replaces the reference's hot path `pkg/src/streamcrf/streaming.py`:
//   streaming_forward  (:155-229)  -> fwd_kernel
//   recompute_alpha    (:232-261)  -> fwd_sweep<MODE_REPLAY> inside bwd_kernel
//   streaming_backward (:264-408)  -> bwd_kernel + finalize_kernel + reduce_partials_kernel
//   finalize_marginals (diagnostics.py:54-79) -> finalize_kernel / boundary_kernel
//
// Algorithm: the exact factorisation of the reference recursion
//   gamma[s,c] = LSE_c' (alpha[s,c'] + T[c',c])              (C^2 per position)
//   alpha[t,c] = LSE_k  (gamma[t-k,c] + h[t,k,c])             (K*C per position)
// with h = S[t,c]-S[t-k,c] + B[k-1,c] (+Ps[t-k,c] + Pe[t-1,c]); the backward is the
// mirror image (delta = LSE_k(h + beta[t+k]); beta[t,c'] = LSE_c(T[c',c] + delta[t,c]))
// and the joint marginals mu[b,k,c,c'] the reference materialises are consumed in
// their two contracted forms:
//   M[t,k,c]     = sum_c' mu = exp(gamma[t,c] + h + beta[t+k,c] - logZ)   (durations, S, coverage)
//   grad_T[c',c] = sum_t exp(alpha[t,c'] + T[c',c] + delta[t,c] - logZ).
//
// Parallel layout: one thread-block cluster per sequence; CTA r owns a label slice.
// The K-term sum of a label only needs that label's history, so the ring of
// per-source terms g[s,c] lives in the owning CTA's shared memory (label-major,
// (hi, lo) pairs -> one conflict-free LDS.64 per term). The only cross-CTA traffic
// per position is the C-vector of new messages, sent with st.async + mbarrier
// (scrf_common.cuh). The K-1 durations k >= 2 of position t+1 do not depend on
// position t, so they are summed while the exchange of position t is in flight.
//
// Inner-loop numerics: every thread of a label uses the same reference value
// m_ref = term(k = 2) (computable by all of them), so the K-term log-sum-exp is a
// single pass of ex2(x - m_ref) with plain-sum reductions; an exact own-max path
// takes over only if some term exceeds m_ref by more than kRefSlack (log2 units).
#include <stdint.h>

#include "scrf_common.cuh"

namespace scrf {

constexpr float kRefSlack = 60.f;

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

// ----------------------------------------------------------------------------
// kernel arguments

template <typename R>
struct Ckpt {
  // per (b, i): ring of g (hi, lo) [K][C], alpha-hat of the K ring positions [K][C],
  // normaliser of the K ring positions [K], header {n_{t0-1}, n_{t0}}
  R* g_hi;
  R* g_lo;
  R* alpha;
  double* n;
  double* hdr;
};

template <typename R>
struct Args {
  const double* S;
  const int64_t* lengths;
  const double* trans;
  const double* dur;
  const double* ps;
  const double* pe;
  int B, T, K, C, delta, n_ckpt;
  Geometry geo;
  Ckpt<R> ck;
  // forward outputs
  double* logZ;
  double* N;
  int32_t* dead_at;
  R* tail_alpha;  // [B][K][C]
  double* tail_n; // [B][K]
  // backward inputs / outputs
  const double* logZ_in;
  const double* upstream;
  R* ws_alpha;    // [B][delta+1][C]
  R* ws_gamma;    // [B][delta+1][C]
  double* ws_n;   // [B][G][delta+1]
  R* start_g;     // [B][T+1][C]  mass of segments starting at t
  R* end_g;       // [B][T+1][C]  mass of segments ending at t
  double* gT_part;  // [B][C][C]
  double* gB_part;  // [B][K][C]
  long long* trace;  // optional [256][8] phase timestamps of CTA 0, thread 0 (debug builds)
};

template <typename R>
__device__ __forceinline__ size_t ck_off(const Args<R>& a, int b, int i) {
  return ((size_t)b * a.n_ckpt + i);
}

// ----------------------------------------------------------------------------
// per-CTA context

struct Ctx {
  int b, rank, c0, Cg, L;
  int tid, cl, j, lane, warp, jj;  // jj = index within the label's first lane group
  int wl;                           // warp index within the label
  int cls;                          // cl if active else 0 (safe shared-memory index)
  bool active;                      // cl < Cg
  bool gl;                          // j < GW: label's first lane group (warp-uniform predicate)
  bool glane;                       // gl && active
  const double* S;                  // S + b*(T+1)*C
  const double* ps;                 // proj_start row base for b (or null)
  const double* pe;
};

template <typename R>
struct FwdSmem {
  typename Vec2<R>::T* ring;  // [Cgm][K]  g (hi, lo)
  R* B2;                      // [Cgm][K]  duration bias * log2e
  R* T2c;                     // [C][Cgm]  T2[c'][c] - Tcmax[c]
  R* Tcmax;                   // [Cgm]
  R* a_all;                   // [2][C]    exchanged messages (relative to the target frame)
  uint64_t* a_bar;            // [2]
  R* part;                    // [2][Cgm][WPL][2]  (m, s) bulk partials
};

template <typename R>
struct BwdSmem {
  typename Vec2<R>::T* vr;  // [Cgm][K]  beta-side terms v[e,c] (hi, lo)
  R* T2r;                   // [Cgm][C]  T2[c'][c] - Trmax[c'] (own rows c')
  R* T2o;                   // [Cgm][C]  T2 own rows (grad_T exponent)
  R* Trmax;                 // [Cgm]
  R* d_all;                 // [2][C]
  uint64_t* d_bar;          // [2]
  R* bpart;                 // [2][Cgm][WPL][3]  (m, s, msum)
  R* end_acc;               // [Cgm][K+1]
  R* end1;                  // [Cgm][K+1]
  R* gBs;                   // [Cgm][K]
  R* gTs;                   // [Cgm][C]
};

__device__ __forceinline__ double S2(const Ctx& x, int C, int t, int c) { return __ldg(x.S + (size_t)t * C + c) * kLog2e; }
__device__ __forceinline__ double PS2(const Ctx& x, int C, int t, int c) { return x.ps ? __ldg(x.ps + (size_t)t * C + c) * kLog2e : 0.0; }
__device__ __forceinline__ double PE2(const Ctx& x, int C, int t, int c) {
  return (x.pe && t >= 0) ? __ldg(x.pe + (size_t)t * C + c) * kLog2e : 0.0;
}

// ----------------------------------------------------------------------------
// shared-memory carving (byte counts mirror the carve functions exactly)

__host__ __device__ inline size_t r16(size_t n) { return (n + 15) & ~(size_t)15; }

template <typename R>
__host__ __device__ inline size_t fwd_smem_bytes(int K, int C, const Geometry& g) {
  const size_t KC = (size_t)K * g.Cgm;
  return r16(KC * 2 * sizeof(R)) + r16(KC * sizeof(R)) + r16((size_t)C * g.Cgm * sizeof(R)) +
         r16(g.Cgm * sizeof(R)) + r16(2 * (size_t)C * sizeof(R)) + r16(16) +
         r16(4 * (size_t)g.Cgm * g.WPL * sizeof(R));
}

template <typename R>
__host__ __device__ inline size_t bwd_extra_smem_bytes(int K, int C, const Geometry& g) {
  const size_t KC = (size_t)K * g.Cgm;
  return r16(KC * 2 * sizeof(R)) + 2 * r16((size_t)g.Cgm * C * sizeof(R)) + r16(g.Cgm * sizeof(R)) +
         r16(2 * (size_t)C * sizeof(R)) + r16(16) + r16(6 * (size_t)g.Cgm * g.WPL * sizeof(R)) +
         2 * r16((size_t)(K + 1) * g.Cgm * sizeof(R)) + r16(KC * sizeof(R)) + r16((size_t)g.Cgm * C * sizeof(R));
}

template <typename T>
__device__ __forceinline__ T* carve(unsigned char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += (count * sizeof(T) + 15) & ~(size_t)15;
  return r;
}

template <typename R>
__device__ void carve_fwd(unsigned char*& p, int K, int C, const Geometry& g, FwdSmem<R>& s) {
  using R2 = typename Vec2<R>::T;
  s.ring = carve<R2>(p, (size_t)K * g.Cgm);
  s.B2 = carve<R>(p, (size_t)K * g.Cgm);
  s.T2c = carve<R>(p, (size_t)C * g.Cgm);
  s.Tcmax = carve<R>(p, g.Cgm);
  s.a_all = carve<R>(p, 2 * (size_t)C);
  s.a_bar = carve<uint64_t>(p, 2);
  s.part = carve<R>(p, 4 * (size_t)g.Cgm * g.WPL);
}

template <typename R>
__device__ void carve_bwd(unsigned char*& p, int K, int C, const Geometry& g, BwdSmem<R>& s) {
  using R2 = typename Vec2<R>::T;
  s.vr = carve<R2>(p, (size_t)K * g.Cgm);
  s.T2r = carve<R>(p, (size_t)g.Cgm * C);
  s.T2o = carve<R>(p, (size_t)g.Cgm * C);
  s.Trmax = carve<R>(p, g.Cgm);
  s.d_all = carve<R>(p, 2 * (size_t)C);
  s.d_bar = carve<uint64_t>(p, 2);
  s.bpart = carve<R>(p, 6 * (size_t)g.Cgm * g.WPL);
  s.end_acc = carve<R>(p, (size_t)(K + 1) * g.Cgm);
  s.end1 = carve<R>(p, (size_t)(K + 1) * g.Cgm);
  s.gBs = carve<R>(p, (size_t)K * g.Cgm);
  s.gTs = carve<R>(p, (size_t)g.Cgm * C);
}

template <typename R>
__device__ Ctx make_ctx(const Args<R>& a, const cg::cluster_group& cl) {
  Ctx x;
  const Geometry& g = a.geo;
  x.rank = (int)cl.block_rank();
  x.b = (int)(blockIdx.x / g.G);
  x.c0 = label_lo(x.rank, a.C, g.G);
  x.Cg = label_lo(x.rank + 1, a.C, g.G) - x.c0;
  x.L = (int)a.lengths[x.b];
  x.tid = threadIdx.x;
  x.cl = x.tid / g.TPL;
  x.j = x.tid % g.TPL;
  x.lane = x.tid & 31;
  x.warp = x.tid >> 5;
  x.wl = x.j >> 5;
  x.jj = x.j;
  x.active = x.cl < x.Cg;
  x.cls = x.active ? x.cl : 0;
  x.gl = x.j < g.GW;
  x.glane = x.active && x.gl;
  x.S = a.S + (size_t)x.b * (a.T + 1) * a.C;
  x.ps = a.ps ? a.ps + (size_t)x.b * a.T * a.C : nullptr;
  x.pe = a.pe ? a.pe + (size_t)x.b * a.T * a.C : nullptr;
  return x;
}

// Load per-label constant tables (log2 domain).
template <typename R>
__device__ void load_fwd_tables(const Args<R>& a, const Ctx& x, FwdSmem<R>& s) {
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C;
  for (int i = x.tid; i < K * g.Cgm; i += g.NT) {
    const int cc = i / K, k = i % K;
    s.B2[i] = (cc < x.Cg) ? (R)(a.dur[(size_t)k * C + x.c0 + cc] * kLog2e) : (R)0;
  }
  for (int c = x.tid; c < g.Cgm; c += g.NT) {
    double m = -CUDART_INF;
    if (c < x.Cg)
      for (int cp = 0; cp < C; ++cp) m = fmax(m, a.trans[(size_t)cp * C + x.c0 + c] * kLog2e);
    s.Tcmax[c] = (R)m;
  }
  __syncthreads();
  for (int i = x.tid; i < C * g.Cgm; i += g.NT) {
    const int cp = i / g.Cgm, c = i % g.Cgm;
    s.T2c[i] = (c < x.Cg) ? (R)(a.trans[(size_t)cp * C + x.c0 + c] * kLog2e) - s.Tcmax[c] : (R)0;
  }
}

template <typename R>
__device__ void load_bwd_tables(const Args<R>& a, const Ctx& x, BwdSmem<R>& s) {
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C;
  for (int r = x.tid; r < g.Cgm; r += g.NT) {
    double m = -CUDART_INF;
    if (r < x.Cg)
      for (int c = 0; c < C; ++c) m = fmax(m, a.trans[(size_t)(x.c0 + r) * C + c] * kLog2e);
    s.Trmax[r] = (R)m;
  }
  __syncthreads();
  for (int i = x.tid; i < g.Cgm * C; i += g.NT) {
    const int r = i / C, c = i % C;
    const R t2 = (r < x.Cg) ? (R)(a.trans[(size_t)(x.c0 + r) * C + c] * kLog2e) : (R)0;
    s.T2o[i] = t2;
    s.T2r[i] = (r < x.Cg) ? t2 - s.Trmax[r] : (R)0;
    s.gTs[i] = (R)0;
  }
  for (int i = x.tid; i < (K + 1) * g.Cgm; i += g.NT) {
    s.end_acc[i] = (R)0;
    s.end1[i] = (R)0;
  }
  for (int i = x.tid; i < K * g.Cgm; i += g.NT) s.gBs[i] = (R)0;
}

// gamma-tilde of own label `cl` from alpha-hat values (<= 0), by the label's first lane group.
template <typename R>
__device__ __forceinline__ R gamma_from_alpha(const R* ahat, const R* T2c, const R* Tcmax, int C, int Cgm, int cl,
                                              int jj, int GW) {
  R s = 0;
  for (int cp = jj; cp < C; cp += GW) s += Mth<R>::ex2(ahat[cp] + T2c[(size_t)cp * Cgm + cl]);
  s = group_sum(s, GW);
  if (s < Mth<R>::tiny()) {  // underflow of the bounded sum: exact max path
    R m = Mth<R>::ninf();
    for (int cp = jj; cp < C; cp += GW) m = fmax(m, ahat[cp] + T2c[(size_t)cp * Cgm + cl]);
    m = group_max(m, GW);
    if (m == Mth<R>::ninf()) return m;
    R s2 = 0;
    for (int cp = jj; cp < C; cp += GW) s2 += Mth<R>::ex2(ahat[cp] + T2c[(size_t)cp * Cgm + cl] - m);
    s2 = group_sum(s2, GW);
    return Tcmax[cl] + m + Mth<R>::lg2(s2);
  }
  return Tcmax[cl] + Mth<R>::lg2(s);
}

// ----------------------------------------------------------------------------
// bulk (durations k >= 2) partial of one target / source
//
// Thread j of a label owns durations k = 2 + j + i*TPL. All threads share the
// reference m_ref = term(k = 2). Returns the lane-group-reduced (m, s[, msum]):
// m == m_ref on the fast path.

template <typename R>
__device__ __forceinline__ R fwd_term(const typename Vec2<R>::T& r, R e_hi, R e_lo, R b2) {
  return (r.x + e_hi) + (r.y + e_lo) + b2;
}

template <typename R>
__device__ __forceinline__ void fwd_bulk(const Args<R>& a, const Ctx& x, const FwdSmem<R>& s, int tt, int slot2,
                                         R e_hi, R e_lo, R& m_out, R& s_out) {
  using R2 = typename Vec2<R>::T;
  const Geometry& g = a.geo;
  const int K = a.K;
  const int kmax = min(K, tt);
  const R2* rg = s.ring + (size_t)x.cls * K;
  const R* b2 = s.B2 + (size_t)x.cls * K;
  R mref = Mth<R>::ninf(), sum = 0, dmax = Mth<R>::ninf();
  bool slow = false;
  const int k0 = 2 + x.j;
  const int stepK = g.TPL % K;
  int slot0 = slot2 - x.j % K;
  if (slot0 < 0) slot0 += K;
  if (kmax >= 2) {
    mref = fwd_term<R>(rg[slot2], e_hi, e_lo, b2[1]);
    slow = (mref == Mth<R>::ninf());
    if (x.active && !slow && k0 <= kmax) {
      int slot = slot0;
      R acc0 = 0, acc1 = 0;
      int k = k0;
      for (; k + g.TPL <= kmax; k += 2 * g.TPL) {
        const R x0 = fwd_term<R>(rg[slot], e_hi, e_lo, b2[k - 1]) - mref;
        slot -= stepK;
        if (slot < 0) slot += K;
        const R x1 = fwd_term<R>(rg[slot], e_hi, e_lo, b2[k + g.TPL - 1]) - mref;
        slot -= stepK;
        if (slot < 0) slot += K;
        dmax = fmax(dmax, fmax(x0, x1));
        acc0 += Mth<R>::ex2(x0);
        acc1 += Mth<R>::ex2(x1);
      }
      if (k <= kmax) {
        const R x0 = fwd_term<R>(rg[slot], e_hi, e_lo, b2[k - 1]) - mref;
        dmax = fmax(dmax, x0);
        acc0 += Mth<R>::ex2(x0);
      }
      sum = acc0 + acc1;
      slow = dmax > (R)kRefSlack;
    }
  }
  R m = mref;
  if (__any_sync(0xffffffffu, slow)) {
    // exact path: own maximum over the thread's durations
    m = Mth<R>::ninf();
    sum = 0;
    if (x.active && k0 <= kmax) {
      int slot = slot0;
      for (int k = k0; k <= kmax; k += g.TPL) {
        m = fmax(m, fwd_term<R>(rg[slot], e_hi, e_lo, b2[k - 1]));
        slot -= stepK;
        if (slot < 0) slot += K;
      }
      if (m != Mth<R>::ninf()) {
        slot = slot0;
        for (int k = k0; k <= kmax; k += g.TPL) {
          sum += Mth<R>::ex2(fwd_term<R>(rg[slot], e_hi, e_lo, b2[k - 1]) - m);
          slot -= stepK;
          if (slot < 0) slot += K;
        }
      }
    }
    group_ms(m, sum, g.GW);
  } else {
    sum = group_sum(sum, g.GW);
  }
  m_out = m;
  s_out = sum;
}

// ----------------------------------------------------------------------------
// per-position input staging
//
// Every position needs a handful of fp64 inputs per own label (prefix sums and
// projections, and in the backward the replayed window values). They are staged
// in chunks of P positions: chunk q+2 is loaded into registers while chunk q is
// consumed, then parked in one of two shared-memory chunk buffers.
//   E0[t,c] = S2[t,c] + Pe2[t-1,c]     (forward target term, backward v[t] base)
//   G0[t,c] = -S2[t,c] + Ps2[t,c]      (forward g[t] base, backward w[t] base)
// backward only: gam[t,c] = gamma~, ahat[t,c] = alpha-hat, n[t] (window store).

constexpr int kStageMax = 2;

template <typename R>
struct StageSmem {
  double* E0;  // [2][P][Cgm]
  double* G0;
  R* gam;      // [2][P][Cgm]
  R* ahat;
  double* n;   // [2][P]
};

__host__ __device__ inline int stage_chunk(const Geometry& g) {
  int P = 64;
  while (P > 2 && P * g.Cgm > g.NT * kStageMax) P >>= 1;
  return P;
}

template <typename R>
__host__ __device__ inline size_t stage_smem_bytes(const Geometry& g) {
  const size_t P = stage_chunk(g);
  return 2 * r16(2 * P * g.Cgm * 8) + 2 * r16(2 * P * g.Cgm * sizeof(R)) + r16(2 * P * 8);
}

template <typename R>
__device__ void carve_stage(unsigned char*& p, const Geometry& g, StageSmem<R>& st) {
  const size_t P = stage_chunk(g);
  st.E0 = carve<double>(p, 2 * P * g.Cgm);
  st.G0 = carve<double>(p, 2 * P * g.Cgm);
  st.gam = carve<R>(p, 2 * P * g.Cgm);
  st.ahat = carve<R>(p, 2 * P * g.Cgm);
  st.n = carve<double>(p, 2 * P);
}

template <typename R, bool BWD>
struct Stager {
  int P, lgP, tb, dir, win_t0;
  double rE[kStageMax], rG[kStageMax], rn[2];
  R rg[kStageMax], ra[kStageMax];

  __device__ __forceinline__ int pos(int q, int i) const { return tb + dir * (q * P + i); }

  __device__ __forceinline__ void load(const Args<R>& a, const Ctx& x, int q) {
    const int n = P * x.Cg;
#pragma unroll
    for (int r = 0; r < kStageMax; ++r) {
      const int e = x.tid + r * a.geo.NT;
      rE[r] = 0.0;
      rG[r] = 0.0;
      rg[r] = (R)0;
      ra[r] = (R)0;
      if (e < n) {
        const int i = e / x.Cg, cc = e % x.Cg, c = x.c0 + cc;
        const int t = pos(q, i);
        if (t >= 0 && t <= a.T) {
          const double s2 = __ldg(x.S + (size_t)t * a.C + c) * kLog2e;
          rE[r] = s2 + PE2(x, a.C, t - 1, c);
          rG[r] = -s2 + ((t < a.T) ? PS2(x, a.C, t, c) : 0.0);
          if (BWD && t >= win_t0 && t <= win_t0 + a.delta) {
            const size_t row = (size_t)x.b * (a.delta + 1) + (t - win_t0);
            rg[r] = a.ws_gamma[row * a.C + c];
            ra[r] = a.ws_alpha[row * a.C + c];
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {  // P <= 64 <= 2 * NT positions
      rn[r] = 0.0;
      const int i = x.tid + r * a.geo.NT;
      if (BWD && i < P) {
        const int t = pos(q, i);
        if (t >= win_t0 && t <= win_t0 + a.delta && t >= 0 && t <= a.T)
          rn[r] = a.ws_n[((size_t)x.b * a.geo.G + x.rank) * (a.delta + 1) + (t - win_t0)];
      }
    }
  }

  __device__ __forceinline__ void store(const Args<R>& a, const Ctx& x, StageSmem<R>& st, int q) {
    const int n = P * x.Cg;
    const int buf = q & 1;
    const int Cgm = a.geo.Cgm;
#pragma unroll
    for (int r = 0; r < kStageMax; ++r) {
      const int e = x.tid + r * a.geo.NT;
      if (e < n) {
        const int i = e / x.Cg, cc = e % x.Cg;
        const size_t k = ((size_t)buf * P + i) * Cgm + cc;
        st.E0[k] = rE[r];
        st.G0[k] = rG[r];
        if (BWD) {
          st.gam[k] = rg[r];
          st.ahat[k] = ra[r];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = x.tid + r * a.geo.NT;
      if (BWD && i < P) st.n[buf * P + i] = rn[r];
    }
  }

  // shared-memory row of position t (P is a power of two)
  __device__ __forceinline__ int row(int t) const {
    const int d = dir * (t - tb);
    return (((d >> lgP) & 1) << lgP) + (d & (P - 1));
  }
  __device__ __forceinline__ size_t idx(int t, int cl, int Cgm) const { return (size_t)row(t) * Cgm + cl; }

  // prime chunks 0 and 1 in shared memory and chunk 2 in registers (ends with a barrier)
  __device__ void begin(const Args<R>& a, const Ctx& x, StageSmem<R>& st, int tb_, int dir_, int win) {
    P = stage_chunk(a.geo);
    lgP = 31 - __clz(P);
    tb = tb_;
    dir = dir_;
    win_t0 = win;
    load(a, x, 0);
    store(a, x, st, 0);
    load(a, x, 1);
    store(a, x, st, 1);
    load(a, x, 2);
    __syncthreads();
  }

  // call at the top of the iteration that processes position t (before any use)
  __device__ __forceinline__ void advance(const Args<R>& a, const Ctx& x, StageSmem<R>& st, int t) {
    const int d = dir * (t - tb);
    if (d > 0 && (d & (P - 1)) == 0) {
      const int q = d >> lgP;
      store(a, x, st, q + 1);
      load(a, x, q + 2);
    }
  }
};

// ----------------------------------------------------------------------------
// forward sweep (shared by the forward kernel and the backward's replay)

enum { MODE_FWD = 0, MODE_REPLAY = 1 };

struct FwdBook {
  // forward-mode bookkeeping (rank 0, thread 0)
  double N_cur;
  int dead_at;
};

template <typename R>
__device__ __forceinline__ void store_part(const Geometry& g, const Ctx& x, R* part, int par, R m, R s) {
  if (!x.active) return;
  const bool first = (g.TPL >= 32) ? (x.lane == 0) : (x.j == 0);
  if (first) {
    const size_t i = (((size_t)par * g.Cgm + x.cl) * g.WPL + x.wl) * 2;
    part[i] = m;
    part[i + 1] = s;
  }
}

// merge of the stored per-warp partials by the label's first lane group
template <typename R>
__device__ __forceinline__ void merge_parts(const Geometry& g, const Ctx& x, const R* part, int par, R& m, R& s) {
  m = Mth<R>::ninf();
  s = 0;
  if (x.active && x.jj < g.WPL) {
    const size_t i = (((size_t)par * g.Cgm + x.cl) * g.WPL + x.jj) * 2;
    m = part[i];
    s = part[i + 1];
  }
  if (g.WPL > 1) {
    // fast path: every warp used the shared reference
    const R m0 = __shfl_sync(0xffffffffu, m, 0, g.GW);
    const bool same = (x.jj >= g.WPL) || (m == m0);
    if (__all_sync(0xffffffffu, same)) {
      s = group_sum(s, g.GW);
      m = m0;
    } else {
      group_ms(m, s, g.GW);
    }
  } else {
    // single partial per label: every lane of the group needs it (each sends to other ranks)
    m = __shfl_sync(0xffffffffu, m, 0, g.GW);
    s = __shfl_sync(0xffffffffu, s, 0, g.GW);
  }
}

// log2(exp2(m) * s + exp2(x1)) without overflow
template <typename R>
__device__ __forceinline__ R add_term(R m, R s, R x1) {
  if (m == Mth<R>::ninf() || !(s > (R)0)) return x1;
  if (x1 == Mth<R>::ninf()) return m + Mth<R>::lg2(s);
  const R d = x1 - m;
  if (d <= (R)kRefSlack) return m + Mth<R>::lg2(s + Mth<R>::ex2(d));
  return x1 + Mth<R>::lg2((R)1 + s * Mth<R>::ex2(-d));
}

// Runs targets t = t_begin+1 .. t_end. Preconditions: ring holds g[s] for
// s in (t_begin-K, t_begin]; Fcur = frame of target t_begin+1; n_prev = n_{t_begin}.
template <typename R, int MODE>
__device__ void fwd_sweep(const Args<R>& a, const Ctx& x, FwdSmem<R>& s, StageSmem<R>& st, Xchg<R>& xa, int t_begin,
                          int t_end, double Fcur, double n_prev, FwdBook& bk, int win_t0) {
  using R2 = typename Vec2<R>::T;
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C, Cgm = g.Cgm;
  const int c = x.c0 + x.cls;
  if (t_end <= t_begin) return;
  Stager<R, false> sg;
  sg.begin(a, x, st, t_begin, +1, 0);
  R2* ring = s.ring + (size_t)x.cls * K;

  // slots of positions t-1 and t-2 for the current target t (incremental mod K)
  int sl1 = t_begin % K;            // (t-1) mod K for t = t_begin+1
  int sl2 = (t_begin + K - 1) % K;  // (t-2) mod K
  int next_ck = (t_begin / a.delta + 1) * a.delta;

  // e for target t_begin+1, bulk partial for it
  R e_hi, e_lo;
  split(st.E0[sg.idx(t_begin + 1, x.cls, Cgm)] - Fcur, e_hi, e_lo);
  {
    R m, sm;
    fwd_bulk(a, x, s, t_begin + 1, sl2, e_hi, e_lo, m, sm);
    store_part(g, x, s.part, (t_begin + 1) & 1, m, sm);
  }
  __syncthreads();

  for (int t = t_begin + 1; t <= t_end; ++t) {
    const int par = t & 1;
    long long* tr = (a.trace && blockIdx.x == 0 && x.tid == 0 && t - t_begin <= 256) ? a.trace + (t - t_begin - 1) * 8 : nullptr;
    if (tr) tr[0] = clock64();
    sg.advance(a, x, st, t);
    if (x.tid == 0) xa.arm(par);
    // (A) critical: bulk partials + the k = 1 term -> a[t]; send it to the cluster
    if (x.gl) {
      R m, sm;
      merge_parts(g, x, s.part, par, m, sm);
      if (tr) tr[1] = clock64();
      const R x1 = fwd_term<R>(ring[sl1], e_hi, e_lo, s.B2[(size_t)x.cls * K]);
      const R av = add_term(m, sm, x1);
      if (x.active) xa.send(par, c, av, x.jj, g.GW, g.G);
    }
    if (tr) tr[2] = clock64();
    // (C) bulk for target t+1 (frame n_{t-1} = n_prev) while the exchange is in flight
    const double Fnext = n_prev;
    R en_hi = 0, en_lo = 0;
    if (t < t_end) {
      split(st.E0[sg.idx(t + 1, x.cls, Cgm)] - Fnext, en_hi, en_lo);
      R m, sm;
      fwd_bulk(a, x, s, t + 1, sl1, en_hi, en_lo, m, sm);
      store_part(g, x, s.part, (t + 1) & 1, m, sm);
    }
    // (E) normaliser, gamma, ring write
    if (tr) tr[3] = clock64();
    const R* aa = xa.wait(par);
    if (tr) tr[4] = clock64();
    R amax = Mth<R>::ninf();
    for (int i = x.lane; i < C; i += 32) amax = fmax(amax, aa[i]);
    amax = group_max(amax, 32);
    if (tr) tr[5] = clock64();
    const bool dead = (amax == Mth<R>::ninf());
    const double n_t = dead ? Fcur : Fcur + (double)amax;
    const int slt = (sl1 + 1 == K) ? 0 : sl1 + 1;  // t mod K
    if (x.gl) {
      const R ahat_own = dead ? Mth<R>::ninf() : aa[c] - amax;
      R gam = Mth<R>::ninf();
      if (!dead) {
        R ssum = 0;
        for (int cp = x.jj; cp < C; cp += g.GW) ssum += Mth<R>::ex2((aa[cp] - amax) + s.T2c[(size_t)cp * Cgm + x.cls]);
        ssum = group_sum(ssum, g.GW);
        if (ssum < Mth<R>::tiny()) {
          R mm = Mth<R>::ninf();
          for (int cp = x.jj; cp < C; cp += g.GW) mm = fmax(mm, (aa[cp] - amax) + s.T2c[(size_t)cp * Cgm + x.cls]);
          mm = group_max(mm, g.GW);
          R s2 = 0;
          if (mm != Mth<R>::ninf())
            for (int cp = x.jj; cp < C; cp += g.GW)
              s2 += Mth<R>::ex2((aa[cp] - amax) + s.T2c[(size_t)cp * Cgm + x.cls] - mm);
          s2 = group_sum(s2, g.GW);
          gam = (mm == Mth<R>::ninf()) ? mm : s.Tcmax[x.cls] + mm + Mth<R>::lg2(s2);
        } else {
          gam = s.Tcmax[x.cls] + Mth<R>::lg2(ssum);
        }
      }
      if (tr) tr[6] = clock64();
      if (x.active && x.jj == 0) {
        const double gv = (gam == Mth<R>::ninf()) ? -CUDART_INF : n_t + (double)gam + st.G0[sg.idx(t, x.cl, Cgm)];
        R2 v;
        split(gv, v.x, v.y);
        ring[slt] = v;
        if (MODE == MODE_FWD) {
          a.tail_alpha[((size_t)x.b * K + slt) * C + c] = ahat_own;
        } else {
          const size_t r = (size_t)x.b * (a.delta + 1) + (t - win_t0);
          a.ws_alpha[r * C + c] = ahat_own;
          a.ws_gamma[r * C + c] = gam;
        }
      }
    }
    const bool at_ck = (t == next_ck);
    if (at_ck) next_ck += a.delta;
    if (MODE == MODE_REPLAY && x.tid == 0) a.ws_n[((size_t)x.b * g.G + x.rank) * (a.delta + 1) + (t - win_t0)] = n_t;
    if (MODE == MODE_FWD && x.rank == 0) {
      if (x.tid == 0) {
        a.tail_n[(size_t)x.b * K + slt] = n_t;
        // reference bookkeeping in nats: shifted-frame dead check and checkpoint shift
        const double amax_abs = dead ? -CUDART_INF : n_t * kLn2;
        if (bk.dead_at < 0 && !(amax_abs - bk.N_cur > kGuard)) bk.dead_at = t;
        if (at_ck && amax_abs - bk.N_cur > kGuard) bk.N_cur = amax_abs;
        if (at_ck && t / a.delta < a.n_ckpt) a.N[(size_t)x.b * a.n_ckpt + t / a.delta] = bk.N_cur;
      }
      if (t == x.L && x.warp == 0) {
        R ssum = 0;
        if (!dead)
          for (int i = x.lane; i < C; i += 32) ssum += Mth<R>::ex2(aa[i] - amax);
        ssum = group_sum(ssum, 32);
        if (x.lane == 0) {
          const double lz = (dead ? -CUDART_INF : n_t + (double)Mth<R>::lg2(ssum)) * kLn2;
          a.logZ[x.b] = lz;
          if (!(lz - bk.N_cur > kGuard) && bk.dead_at < 0) bk.dead_at = x.L;
        }
      }
    }
    Fcur = Fnext;
    n_prev = n_t;
    e_hi = en_hi;
    e_lo = en_lo;
    sl2 = sl1;
    sl1 = slt;
    if (tr) tr[7] = clock64();
    __syncthreads();
    if (MODE == MODE_FWD && at_ck && t / a.delta < a.n_ckpt) {
      // snapshot ring + tail for checkpoint i = t / delta
      const int i = t / a.delta;
      const size_t base = ck_off(a, x.b, i);
      for (int q = x.tid; q < K * x.Cg; q += g.NT) {
        const int slot = q / x.Cg, cc = q % x.Cg;
        const size_t gi = (base * K + slot) * C + x.c0 + cc;
        const R2 v = s.ring[(size_t)cc * K + slot];
        a.ck.g_hi[gi] = v.x;
        a.ck.g_lo[gi] = v.y;
        a.ck.alpha[gi] = a.tail_alpha[((size_t)x.b * K + slot) * C + x.c0 + cc];
      }
      if (x.rank == 0) {
        for (int q = x.tid; q < K; q += g.NT) a.ck.n[base * K + q] = a.tail_n[(size_t)x.b * K + q];
        if (x.tid == 0) {
          a.ck.hdr[base * 2 + 0] = Fcur;  // = n_{t-1}: frame of target t+1
          a.ck.hdr[base * 2 + 1] = n_t;
        }
      }
      __syncthreads();
    }
  }
}

// ----------------------------------------------------------------------------
// forward kernel

template <typename R>
__device__ void ck_copy_ring(const Args<R>& a, const Ctx& x, const FwdSmem<R>& s, int i, bool alpha_from_tail) {
  using R2 = typename Vec2<R>::T;
  const int K = a.K, C = a.C;
  const size_t base = ck_off(a, x.b, i);
  for (int q = x.tid; q < K * x.Cg; q += a.geo.NT) {
    const int slot = q / x.Cg, cc = q % x.Cg;
    const size_t gi = (base * K + slot) * C + x.c0 + cc;
    const R2 v = s.ring[(size_t)cc * K + slot];
    a.ck.g_hi[gi] = v.x;
    a.ck.g_lo[gi] = v.y;
    a.ck.alpha[gi] = alpha_from_tail ? a.tail_alpha[((size_t)x.b * K + slot) * C + x.c0 + cc]
                                     : (slot == 0 ? (R)0 : Mth<R>::ninf());
  }
}

template <typename R>
__global__ void __launch_bounds__(1024) fwd_kernel(Args<R> a) {
  using R2 = typename Vec2<R>::T;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* p = smem_raw;
  FwdSmem<R> s;
  StageSmem<R> st;
  carve_fwd<R>(p, a.K, a.C, a.geo, s);
  carve_stage<R>(p, a.geo, st);
  Ctx x = make_ctx(a, cl);
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C, Cgm = g.Cgm;
  load_fwd_tables(a, x, s);
  // tail: position 0 has alpha = 0, every other slot is "never written"
  for (int q = x.tid; q < K * x.Cg; q += g.NT) {
    const int slot = q / x.Cg, cc = q % x.Cg;
    a.tail_alpha[((size_t)x.b * K + slot) * C + x.c0 + cc] = slot == 0 ? (R)0 : Mth<R>::ninf();
  }
  if (x.rank == 0)
    for (int q = x.tid; q < K; q += g.NT) a.tail_n[(size_t)x.b * K + q] = q == 0 ? 0.0 : -CUDART_INF;
  for (int q = x.tid; q < K * Cgm; q += g.NT) {
    R2 v;
    v.x = Mth<R>::ninf();
    v.y = 0;
    s.ring[q] = v;
  }
  __syncthreads();
  // position 0: alpha = 0 for every label (virtual source)
  const int c = x.c0 + x.cls;
  if (x.gl) {
    R ssum = 0;
    for (int cp = x.jj; cp < C; cp += g.GW) ssum += Mth<R>::ex2((R)0 + s.T2c[(size_t)cp * Cgm + x.cls]);
    ssum = group_sum(ssum, g.GW);
    const R gam = s.Tcmax[x.cls] + Mth<R>::lg2(ssum);
    if (x.active && x.jj == 0) {
      const double gv = (double)gam - S2(x, C, 0, c) + PS2(x, C, 0, c);
      R2 v;
      split(gv, v.x, v.y);
      s.ring[(size_t)x.cl * K] = v;
    }
  }
  __syncthreads();
  // checkpoint 0 = initial ring
  ck_copy_ring(a, x, s, 0, false);
  if (x.rank == 0) {
    const size_t base = ck_off(a, x.b, 0);
    for (int q = x.tid; q < K; q += g.NT) a.ck.n[base * K + q] = q == 0 ? 0.0 : -CUDART_INF;
    if (x.tid == 0) {
      a.ck.hdr[base * 2 + 0] = 0.0;
      a.ck.hdr[base * 2 + 1] = 0.0;
      a.N[(size_t)x.b * a.n_ckpt] = 0.0;
    }
  }
  FwdBook bk;
  bk.N_cur = 0.0;
  bk.dead_at = -1;
  Xchg<R> xa;
  xa.buf = s.a_all;
  xa.bar = s.a_bar;
  xa.C = C;
  xa.init(x.tid);
  cl.sync();
  fwd_sweep<R, MODE_FWD>(a, x, s, st, xa, 0, x.L, 0.0, 0.0, bk, 0);
  // checkpoints past the sequence end hold the frozen ring at L
  for (int i = x.L / a.delta + 1; i < a.n_ckpt; ++i) {
    ck_copy_ring(a, x, s, i, true);
    if (x.rank == 0) {
      const size_t base = ck_off(a, x.b, i);
      for (int q = x.tid; q < K; q += g.NT) a.ck.n[base * K + q] = a.tail_n[(size_t)x.b * K + q];
      if (x.tid == 0) a.N[(size_t)x.b * a.n_ckpt + i] = bk.N_cur;
    }
  }
  if (x.rank == 0 && x.tid == 0) a.dead_at[x.b] = bk.dead_at;
  cl.sync();
}

// ----------------------------------------------------------------------------
// backward kernel: per window (last to first) replay alpha, then sweep beta down

template <typename R>
__device__ void flush_grads(const Args<R>& a, const Ctx& x, BwdSmem<R>& sb) {
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C;
  __syncthreads();
  for (int q = x.tid; q < K * x.Cg; q += g.NT) {
    const int cc = q / K, k = q % K;
    const R v = sb.gBs[(size_t)cc * K + k];
    if (v != (R)0) {
      a.gB_part[((size_t)x.b * K + k) * C + x.c0 + cc] += (double)v;
      sb.gBs[(size_t)cc * K + k] = (R)0;
    }
  }
  for (int q = x.tid; q < x.Cg * C; q += g.NT) {
    const int r = q / C, cc = q % C;
    const R v = sb.gTs[r * C + cc];
    if (v != (R)0) {
      a.gT_part[((size_t)x.b * C + x.c0 + r) * C + cc] += (double)v;
      sb.gTs[r * C + cc] = (R)0;
    }
  }
  __syncthreads();
}

// Per-source values of own label: w = G0[t] - F'; Gam = (F' + n_t - logZ2) + gamma~[t]
template <typename R>
struct SrcVals {
  R w_hi, w_lo, gam;
};

template <typename R>
__device__ __forceinline__ R bwd_term(const typename Vec2<R>::T& v, const SrcVals<R>& s, R b2) {
  return (v.x + s.w_hi) + (v.y + s.w_lo) + b2;
}

// bulk for source ts (durations 2 <= k <= min(K, L - ts)); vslot2 = (ts+2) mod K,
// eslot2 = (ts+2) mod (K+1). Consumes every M[ts,k,c] (grad_B, end accumulators).
template <typename R>
__device__ __forceinline__ void bwd_bulk(const Args<R>& a, const Ctx& x, BwdSmem<R>& sb, const R* B2all, int ts,
                                         int vslot2, int eslot2, const SrcVals<R>& v, R& m_out, R& s_out, R& ms_out) {
  using R2 = typename Vec2<R>::T;
  const Geometry& g = a.geo;
  const int K = a.K;
  const int kmax = min(K, x.L - ts);
  const R2* vr = sb.vr + (size_t)x.cls * K;
  const R* b2 = B2all + (size_t)x.cls * K;
  R* gB = sb.gBs + (size_t)x.cls * K;
  R* ea = sb.end_acc + (size_t)x.cls * (K + 1);
  R mref = Mth<R>::ninf(), sum = 0, msum = 0, dmax = Mth<R>::ninf();
  bool slow = false;
  const int k0 = 2 + x.j;
  const int stepK = g.TPL % K, stepE = g.TPL % (K + 1);
  int slot0 = vslot2 + x.j % K;
  if (slot0 >= K) slot0 -= K;
  int eslot0 = eslot2 + x.j % (K + 1);
  if (eslot0 >= K + 1) eslot0 -= K + 1;
  if (kmax >= 2) {
    mref = bwd_term<R>(vr[vslot2], v, b2[1]);
    slow = (mref == Mth<R>::ninf());
    if (x.active && !slow && k0 <= kmax) {
      // pass 1 (no stores): largest exponent relative to the shared reference
      int slot = slot0;
      for (int k = k0; k <= kmax; k += g.TPL) {
        dmax = fmax(dmax, bwd_term<R>(vr[slot], v, b2[k - 1]) - mref);
        slot += stepK;
        if (slot >= K) slot -= K;
      }
      slow = dmax > (R)kRefSlack;
    }
  }
  const bool any_slow = __any_sync(0xffffffffu, slow);
  if (x.active && k0 <= kmax) {
    if (!slow) {
      const R F = Mth<R>::ex2(mref + v.gam);
      int slot = slot0, es = eslot0;
      for (int k = k0; k <= kmax; k += g.TPL) {
        const R e = Mth<R>::ex2(bwd_term<R>(vr[slot], v, b2[k - 1]) - mref);
        const R M = e * F;
        sum += e;
        msum += M;
        gB[k - 1] += M;
        ea[es] += M;
        slot += stepK;
        if (slot >= K) slot -= K;
        es += stepE;
        if (es >= K + 1) es -= K + 1;
      }
    } else {
      // exact path: own maximum, direct marginals
      R m = Mth<R>::ninf();
      int slot = slot0;
      for (int k = k0; k <= kmax; k += g.TPL) {
        m = fmax(m, bwd_term<R>(vr[slot], v, b2[k - 1]));
        slot += stepK;
        if (slot >= K) slot -= K;
      }
      slot = slot0;
      int es = eslot0;
      for (int k = k0; k <= kmax; k += g.TPL) {
        const R y = bwd_term<R>(vr[slot], v, b2[k - 1]);
        if (m != Mth<R>::ninf()) sum += Mth<R>::ex2(y - m);
        const R M = Mth<R>::ex2(y + v.gam);
        msum += M;
        gB[k - 1] += M;
        ea[es] += M;
        slot += stepK;
        if (slot >= K) slot -= K;
        es += stepE;
        if (es >= K + 1) es -= K + 1;
      }
      mref = m;
    }
  }
  R m = mref;
  if (any_slow) {
    group_ms(m, sum, g.GW);
  } else {
    sum = group_sum(sum, g.GW);
  }
  msum = group_sum(msum, g.GW);
  m_out = m;
  s_out = sum;
  ms_out = msum;
}

template <typename R>
__device__ __forceinline__ void store_bpart(const Geometry& g, const Ctx& x, R* bp, int par, R m, R s, R ms) {
  if (!x.active) return;
  const bool first = (g.TPL >= 32) ? (x.lane == 0) : (x.j == 0);
  if (first) {
    const size_t i = (((size_t)par * g.Cgm + x.cl) * g.WPL + x.wl) * 3;
    bp[i] = m;
    bp[i + 1] = s;
    bp[i + 2] = ms;
  }
}

template <typename R>
__global__ void __launch_bounds__(1024) bwd_kernel(Args<R> a) {
  using R2 = typename Vec2<R>::T;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* p = smem_raw;
  FwdSmem<R> s;
  BwdSmem<R> sb;
  StageSmem<R> st;
  carve_fwd<R>(p, a.K, a.C, a.geo, s);
  carve_bwd<R>(p, a.K, a.C, a.geo, sb);
  carve_stage<R>(p, a.geo, st);
  Ctx x = make_ctx(a, cl);
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C, Cgm = g.Cgm, L = x.L;
  const int c = x.c0 + x.cls;
  load_fwd_tables(a, x, s);
  load_bwd_tables(a, x, sb);
  Xchg<R> xa, xd;
  xa.buf = s.a_all;
  xa.bar = s.a_bar;
  xa.C = C;
  xa.init(x.tid);
  xd.buf = sb.d_all;
  xd.bar = sb.d_bar;
  xd.C = C;
  xd.init(x.tid);
  __syncthreads();
  cl.sync();
  const double logZ2 = a.logZ_in[x.b] * kLog2e;
  R2* vr = sb.vr + (size_t)x.cls * K;

  // beta ring: only v[L] is live initially (beta[L] = 0)
  if (x.active && x.j == 0) {
    R2 v;
    split(S2(x, C, L, c) + PE2(x, C, L - 1, c), v.x, v.y);
    vr[L % K] = v;
  }
  double Fp_cur = 0.0;   // frame of source t (= nd_{t+2})
  double nd_prev = 0.0;  // nd_{t+1}
  int steps_since_flush = 0;
  FwdBook bk;
  bk.N_cur = 0;
  bk.dead_at = -1;

  const int i_last = (L - 1) / a.delta;  // window holding source L-1
  for (int i = i_last; i >= 0; --i) {
    const int t0 = i * a.delta;
    const int t1 = min((i + 1) * a.delta, L);
    // ---- replay alpha over [t0, t1] from checkpoint i
    const size_t base = ck_off(a, x.b, i);
    __syncthreads();
    for (int q = x.tid; q < K * Cgm; q += g.NT) {
      const int cc = q / K, slot = q % K;
      if (cc < x.Cg) {
        const size_t gi = (base * K + slot) * C + x.c0 + cc;
        R2 v;
        v.x = a.ck.g_hi[gi];
        v.y = a.ck.g_lo[gi];
        s.ring[q] = v;
      }
    }
    // alpha-hat at t0 for all labels (into the exchange buffer, parity of t0)
    for (int q = x.tid; q < C; q += g.NT) s.a_all[(t0 & 1) * C + q] = a.ck.alpha[(base * K + (t0 % K)) * C + q];
    __syncthreads();
    const double n_t0 = a.ck.hdr[base * 2 + 1];
    const double n_t0m1 = a.ck.hdr[base * 2 + 0];
    if (x.gl) {
      const R* ah = s.a_all + (t0 & 1) * C;
      const R gam = gamma_from_alpha(ah, s.T2c, s.Tcmax, C, Cgm, x.cls, x.jj, g.GW);
      if (x.active && x.jj == 0) {
        const size_t r = (size_t)x.b * (a.delta + 1);
        a.ws_alpha[r * C + c] = ah[c];
        a.ws_gamma[r * C + c] = gam;
      }
    }
    if (x.tid == 0) a.ws_n[((size_t)x.b * g.G + x.rank) * (a.delta + 1)] = n_t0;
    __syncthreads();
    fwd_sweep<R, MODE_REPLAY>(a, x, s, st, xa, t0, t1, (t0 == 0) ? 0.0 : n_t0m1, n_t0, bk, t0);
    __syncthreads();
    cl.sync();

    // ---- beta sweep over sources t = t1-1 .. t0
    Stager<R, true> sg;
    sg.begin(a, x, st, t1 - 1, -1, t0);
    auto src = [&](int ts, double Fp) {
      SrcVals<R> v;
      const size_t k = sg.idx(ts, x.cls, Cgm);
      split(st.G0[k] - Fp, v.w_hi, v.w_lo);
      v.gam = (R)(Fp + st.n[sg.row(ts)] - logZ2) + st.gam[k];
      return v;
    };
    // slots of t+1, t+2 in the beta ring (mod K) and the end ring (mod K+1), source t = t1-1
    int vs1 = t1 % K, vs2 = (t1 + 1) % K;
    int es1 = t1 % (K + 1), es2 = (t1 + 1) % (K + 1);
    SrcVals<R> cur = src(t1 - 1, Fp_cur);
    {
      R m, sm, ms;
      bwd_bulk(a, x, sb, s.B2, t1 - 1, vs2, es2, cur, m, sm, ms);
      store_bpart(g, x, sb.bpart, (t1 - 1) & 1, m, sm, ms);
    }
    __syncthreads();
    for (int t = t1 - 1; t >= t0; --t) {
      const int par = t & 1;
      sg.advance(a, x, st, t);
      if (x.tid == 0) xd.arm(par);
      // (A) critical k = 1 term for source t
      if (x.gl) {
        R m = Mth<R>::ninf(), sm = 0, ms = 0;
        if (x.active && x.jj < g.WPL) {
          const size_t q = (((size_t)par * Cgm + x.cl) * g.WPL + x.jj) * 3;
          m = sb.bpart[q];
          sm = sb.bpart[q + 1];
          ms = sb.bpart[q + 2];
        }
        if (g.WPL > 1) {
          const R m0 = __shfl_sync(0xffffffffu, m, 0, g.GW);
          const bool same = (x.jj >= g.WPL) || (m == m0);
          if (__all_sync(0xffffffffu, same)) {
            sm = group_sum(sm, g.GW);
            m = m0;
          } else {
            group_ms(m, sm, g.GW);
          }
          ms = group_sum(ms, g.GW);
        } else {
          m = __shfl_sync(0xffffffffu, m, 0, g.GW);
          sm = __shfl_sync(0xffffffffu, sm, 0, g.GW);
          ms = __shfl_sync(0xffffffffu, ms, 0, g.GW);
        }
        const R y1 = bwd_term<R>(vr[vs1], cur, s.B2[(size_t)x.cls * K]);
        const R M1 = Mth<R>::ex2(y1 + cur.gam);
        const R dv = add_term(m, sm, y1);
        if (x.active && x.jj == 0) {
          sb.end1[(size_t)x.cl * (K + 1) + es1] = M1;
          sb.gBs[(size_t)x.cl * K] += M1;
          a.start_g[((size_t)x.b * (a.T + 1) + t) * C + c] = ms + M1;
        }
        if (x.active) xd.send(par, c, dv, x.jj, g.GW, g.G);
      }
      // (C) bulk for source t-1 (frame nd_{t+1}) while the exchange is in flight
      SrcVals<R> nxt = cur;
      if (t - 1 >= t0) {
        nxt = src(t - 1, nd_prev);
        R m, sm, ms;
        bwd_bulk(a, x, sb, s.B2, t - 1, vs1, es1, nxt, m, sm, ms);
        store_bpart(g, x, sb.bpart, (t - 1) & 1, m, sm, ms);
      }
      // (E) beta at t, grad_T, v[t], end emission
      const R* dd = xd.wait(par);
      R dmax = Mth<R>::ninf();
      for (int q = x.lane; q < C; q += 32) dmax = fmax(dmax, dd[q]);
      dmax = group_max(dmax, 32);
      const bool dead = (dmax == Mth<R>::ninf());
      const double nd_t = dead ? Fp_cur : Fp_cur + (double)dmax;
      const int vs0 = (vs1 == 0) ? K - 1 : vs1 - 1;  // t mod K
      const int es0 = (es1 == 0) ? K : es1 - 1;      // t mod (K+1)
      if (x.gl && !dead) {
        const size_t k = sg.idx(t, x.cls, Cgm);
        const double n_t = st.n[sg.row(t)];
        const R Zt = (R)(n_t + nd_t - logZ2);
        const R ahat = st.ahat[k];
        R ssum = 0;
        for (int q = x.jj; q < C; q += g.GW) {
          const R dh = dd[q] - dmax;
          ssum += Mth<R>::ex2(sb.T2r[(size_t)x.cls * C + q] + dh);
          if (x.active && ahat != Mth<R>::ninf())
            sb.gTs[(size_t)x.cls * C + q] += Mth<R>::ex2(ahat + sb.T2o[(size_t)x.cls * C + q] + dh + Zt);
        }
        ssum = group_sum(ssum, g.GW);
        R bt;
        if (ssum < Mth<R>::tiny()) {
          R mm = Mth<R>::ninf();
          for (int q = x.jj; q < C; q += g.GW) mm = fmax(mm, sb.T2r[(size_t)x.cls * C + q] + (dd[q] - dmax));
          mm = group_max(mm, g.GW);
          R s2 = 0;
          if (mm != Mth<R>::ninf())
            for (int q = x.jj; q < C; q += g.GW) s2 += Mth<R>::ex2(sb.T2r[(size_t)x.cls * C + q] + (dd[q] - dmax) - mm);
          s2 = group_sum(s2, g.GW);
          bt = (mm == Mth<R>::ninf()) ? mm : sb.Trmax[x.cls] + mm + Mth<R>::lg2(s2);
        } else {
          bt = sb.Trmax[x.cls] + Mth<R>::lg2(ssum);
        }
        if (x.active && x.jj == 0 && t >= 1) {
          const double vv = (bt == Mth<R>::ninf()) ? -CUDART_INF : st.E0[k] + nd_t + (double)bt;
          R2 v;
          split(vv, v.x, v.y);
          vr[vs0] = v;
        }
      }
      if (x.active && x.j == 0) {
        const int e = t + K;  // complete after source t: emit
        if (e <= L) {
          const int es = (es0 == 0) ? K : es0 - 1;  // (t + K) mod (K+1) = (t - 1) mod (K+1)
          R* ea = sb.end_acc + (size_t)x.cl * (K + 1);
          a.end_g[((size_t)x.b * (a.T + 1) + e) * C + c] = ea[es] + sb.end1[(size_t)x.cl * (K + 1) + es];
          ea[es] = (R)0;
        }
      }
      Fp_cur = nd_prev;
      nd_prev = nd_t;
      cur = nxt;
      vs2 = vs1;
      vs1 = vs0;
      es2 = es1;
      es1 = es0;
      __syncthreads();
      if (++steps_since_flush >= 256) {
        flush_grads(a, x, sb);
        steps_since_flush = 0;
      }
    }
    cl.sync();
  }
  // remaining ends e in [1, min(K-1, L)]
  __syncthreads();
  if (x.active && x.j == 0) {
    for (int e = 1; e <= min(K - 1, L); ++e) {
      const int es = e % (K + 1);
      a.end_g[((size_t)x.b * (a.T + 1) + e) * C + c] =
          sb.end_acc[(size_t)x.cl * (K + 1) + es] + sb.end1[(size_t)x.cl * (K + 1) + es];
    }
  }
  flush_grads(a, x, sb);
  cl.sync();
}

// ----------------------------------------------------------------------------
// finalize: start/end masses -> grad_S, grad_P*, marginals (diagnostics.py:54-79)
//
// One thread per (b, c): sequential fp64 scan over t (coverage cumsum).

template <typename R>
__global__ void finalize_kernel(const R* start_g, const R* end_g, const int64_t* lengths, const double* upstream, int B,
                                int T, int C, double* grad_S, double* grad_Ps, double* grad_Pe, double* pos) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * C) return;
  const int b = idx / C, c = idx % C;
  const int L = (int)lengths[b];
  const double up = upstream ? upstream[b] : 1.0;
  const size_t rb = (size_t)b * (T + 1);
  double cov = 0.0;
  for (int t = 0; t <= T; ++t) {
    const double st = (t < L) ? (double)start_g[(rb + t) * C + c] : 0.0;
    const double en = (t >= 1 && t <= L) ? (double)end_g[(rb + t) * C + c] : 0.0;
    grad_S[(rb + t) * C + c] = up * (en - st);
    if (t < T) {
      if (grad_Ps) grad_Ps[((size_t)b * T + t) * C + c] = up * st;
      cov += st - en;
      pos[((size_t)b * T + t) * C + c] = (t < L) ? fmin(fmax(cov, 0.0), 1.0) : 0.0;
    }
    if (t >= 1 && grad_Pe) grad_Pe[((size_t)b * T + t - 1) * C + c] = up * en;
  }
}

// boundary posterior + expected segment count, one block per b
template <typename R>
__global__ void boundary_kernel(const R* start_g, const int64_t* lengths, int B, int T, int C, double* boundary,
                                double* count) {
  const int b = blockIdx.x;
  const int L = (int)lengths[b];
  const size_t rb = (size_t)b * (T + 1);
  double acc = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    double s = 0.0;
    if (t < L)
      for (int c = 0; c < C; ++c) s += (double)start_g[(rb + t) * C + c];
    acc += s;
    boundary[(size_t)b * T + t] = (t < L) ? fmin(fmax(s, 0.0), 1.0) : 0.0;
  }
  __shared__ double red[1024];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) count[b] = red[0];
}

// fixed-order batch reduction of per-sequence partials (bit-reproducible)
__global__ void reduce_partials_kernel(const double* part, const double* upstream, int B, size_t n, double* out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int b = 0; b < B; ++b) acc += (upstream ? upstream[b] : 1.0) * part[(size_t)b * n + i];
  out[i] = acc;
}

template __global__ void fwd_kernel<float>(Args<float>);
template __global__ void fwd_kernel<double>(Args<double>);
template __global__ void bwd_kernel<float>(Args<float>);
template __global__ void bwd_kernel<double>(Args<double>);

}  // namespace scrf
