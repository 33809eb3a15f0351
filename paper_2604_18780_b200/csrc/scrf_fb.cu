// Streaming semi-CRF forward / backward on B200 (sm_100a).
//
// Replaces the reference's hot path `pkg/src/streamcrf/streaming.py`:
//   streaming_forward  (:155-229)  -> fwd_kernel
//   recompute_alpha    (:232-261)  -> fwd_sweep<REPLAY> inside bwd_kernel
//   streaming_backward (:264-408)  -> bwd_kernel + finalize_kernel + reduce_kernel
//   finalize_marginals (diagnostics.py:54-79) -> finalize_kernel
//
// Algorithm: the exact factorisation of the reference recursion
//   gamma[s,c] = LSE_c' (alpha[s,c'] + T[c',c])              (C^2 per position)
//   alpha[t,c] = LSE_k  (gamma[t-k,c] + h[t,k,c])             (K*C per position)
// with h = S[t,c]-S[t-k,c] + B[k-1,c] (+Ps[t-k,c] + Pe[t-1,c]); the backward is the
// mirror image (delta = LSE_k(h + beta[t+k]); beta[t,c'] = LSE_c(T[c',c] + delta[t,c]))
// and every joint marginal the reference materialises as mu[b,k,c,c'] is consumed
// in its two contracted forms:
//   M[t,k,c]     = sum_c' mu = exp(gamma[t,c] + h + beta[t+k,c] - logZ)   (durations, S, coverage)
//   grad_T[c',c] = sum_t exp(alpha[t,c'] + T[c',c] + delta[t,c] - logZ).
//
// Parallel layout: one thread-block cluster per sequence; CTA r of the cluster owns
// a contiguous label slice. The K-term sum of a label only needs that label's
// history, so the ring of per-source terms g[s,c] lives in the owning CTA's shared
// memory; the only cross-CTA traffic per position is the C-vector of new messages
// (DSMEM stores + one split cluster barrier). The bulk of the K*C work for position
// t+1 (durations k >= 2, which do not depend on position t) is computed between the
// barrier's arrive and wait, hiding the cluster round trip.
#include <stdint.h>

#include "scrf_common.cuh"

namespace scrf {

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
  R* tail_alpha;      // [B][K][C]
  double* tail_n;     // [B][K]
  // backward inputs / outputs
  const double* logZ_in;
  const double* upstream;
  R* ws_alpha;       // [B][delta+1][C]
  R* ws_gamma;       // [B][delta+1][C]
  double* ws_n;      // [B][G][delta+1]
  R* start_g;        // [B][T+1][C]  mass of segments starting at t (working type)
  R* end_g;          // [B][T+1][C]  mass of segments ending at t
  double* gT_part;   // [B][C][C]
  double* gB_part;   // [B][K][C]
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
  R* ring_hi;  // [K][Cgm]
  R* ring_lo;
  R* B2;       // [K][Cgm]  duration bias * log2e
  R* T2c;      // [C][Cgm]  T2[c'][c] - Tcmax[c]
  R* Tcmax;    // [Cgm]
  R* a_all;    // [2][C]    exchanged messages (relative to the target frame)
  uint64_t* a_bar;  // [2]   mbarriers of the a_all exchange
  R* part_m;   // [2][Cgm][WPL]
  R* part_s;
};

template <typename R>
struct BwdSmem {
  R* vr_hi;    // [K][Cgm]  beta-side terms v[e,c]
  R* vr_lo;
  R* T2r;      // [Cgm][C]  T2[c'][c] - Trmax[c'] (own rows c')
  R* Trmax;    // [Cgm]
  R* T2o;      // [Cgm][C]  T2 own rows (grad_T exponent)
  R* d_all;    // [2][C]
  uint64_t* d_bar;  // [2]
  R* bpart;    // [2][Cgm][WPL][3]
  R* end_acc;  // [K+1][Cgm]
  R* end1;     // [K+1][Cgm]
  R* gBs;      // [K][Cgm]
  R* gTs;      // [Cgm][C]
};

__device__ __forceinline__ double ld_or0(const double* p, size_t i) { return p ? __ldg(p + i) : 0.0; }

// S[b,t,c] * log2e etc.
__device__ __forceinline__ double S2(const Ctx& x, int C, int t, int c) { return __ldg(x.S + (size_t)t * C + c) * kLog2e; }
__device__ __forceinline__ double PS2(const Ctx& x, int C, int t, int c) { return x.ps ? __ldg(x.ps + (size_t)t * C + c) * kLog2e : 0.0; }
__device__ __forceinline__ double PE2(const Ctx& x, int C, int t, int c) {
  return (x.pe && t >= 0) ? __ldg(x.pe + (size_t)t * C + c) * kLog2e : 0.0;
}

// ----------------------------------------------------------------------------
// shared-memory carving

__host__ __device__ inline size_t r16(size_t n) { return (n + 15) & ~(size_t)15; }

// byte counts mirror carve_fwd / carve_bwd exactly (each chunk rounded to 16 B)
template <typename R>
__host__ __device__ inline size_t fwd_smem_bytes(int K, int C, const Geometry& g) {
  const size_t KC = (size_t)K * g.Cgm;
  return 3 * r16(KC * sizeof(R)) + r16((size_t)C * g.Cgm * sizeof(R)) + r16(g.Cgm * sizeof(R)) +
         r16(2 * (size_t)C * sizeof(R)) + r16(16) + 2 * r16(2 * (size_t)g.Cgm * g.WPL * sizeof(R));
}

template <typename R>
__host__ __device__ inline size_t bwd_extra_smem_bytes(int K, int C, const Geometry& g) {
  const size_t KC = (size_t)K * g.Cgm;
  return 2 * r16(KC * sizeof(R)) + 2 * r16((size_t)g.Cgm * C * sizeof(R)) + r16(g.Cgm * sizeof(R)) +
         r16(2 * (size_t)C * sizeof(R)) + r16(16) + r16(6 * (size_t)g.Cgm * g.WPL * sizeof(R)) +
         2 * r16((size_t)(K + 1) * g.Cgm * sizeof(R)) + r16(KC * sizeof(R)) +
         r16((size_t)g.Cgm * C * sizeof(R));
}

template <typename T>
__device__ __forceinline__ T* carve(unsigned char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += (count * sizeof(T) + 15) & ~(size_t)15;
  return r;
}

template <typename R>
__device__ void carve_fwd(unsigned char*& p, int K, int C, const Geometry& g, FwdSmem<R>& s) {
  s.ring_hi = carve<R>(p, (size_t)K * g.Cgm);
  s.ring_lo = carve<R>(p, (size_t)K * g.Cgm);
  s.B2 = carve<R>(p, (size_t)K * g.Cgm);
  s.T2c = carve<R>(p, (size_t)C * g.Cgm);
  s.Tcmax = carve<R>(p, g.Cgm);
  s.a_all = carve<R>(p, 2 * (size_t)C);
  s.a_bar = carve<uint64_t>(p, 2);
  s.part_m = carve<R>(p, 2 * (size_t)g.Cgm * g.WPL);
  s.part_s = carve<R>(p, 2 * (size_t)g.Cgm * g.WPL);
}

template <typename R>
__device__ void carve_bwd(unsigned char*& p, int K, int C, const Geometry& g, BwdSmem<R>& s) {
  s.vr_hi = carve<R>(p, (size_t)K * g.Cgm);
  s.vr_lo = carve<R>(p, (size_t)K * g.Cgm);
  s.T2r = carve<R>(p, (size_t)g.Cgm * C);
  s.T2o = carve<R>(p, (size_t)g.Cgm * C);
  s.Trmax = carve<R>(p, g.Cgm);
  s.d_all = carve<R>(p, 2 * (size_t)C);
  s.d_bar = carve<uint64_t>(p, 2);
  s.bpart = carve<R>(p, 2 * 3 * (size_t)g.Cgm * g.WPL);
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
  x.jj = x.j;  // meaningful when glane
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
    int k = i / g.Cgm, c = i % g.Cgm;
    s.B2[i] = (c < x.Cg) ? (R)(a.dur[(size_t)k * C + x.c0 + c] * kLog2e) : (R)0;
  }
  // column max of T for own labels
  for (int c = x.tid; c < g.Cgm; c += g.NT) {
    double m = -CUDART_INF;
    if (c < x.Cg)
      for (int cp = 0; cp < C; ++cp) m = fmax(m, a.trans[(size_t)cp * C + x.c0 + c] * kLog2e);
    s.Tcmax[c] = (R)m;
  }
  __syncthreads();
  for (int i = x.tid; i < C * g.Cgm; i += g.NT) {
    int cp = i / g.Cgm, c = i % g.Cgm;
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
    int r = i / C, c = i % C;
    R t2 = (r < x.Cg) ? (R)(a.trans[(size_t)(x.c0 + r) * C + c] * kLog2e) : (R)0;
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

// gamma-tilde of own label `cl` from exchanged alpha-hat values (relative, <= 0).
// Executed by the label's first lane group (width GW); result valid in all its lanes.
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

// Bulk (durations k >= 2) partial for target `tt` of own label: thread j owns k = 1 + j + i*TPL.
template <typename R>
__device__ __forceinline__ void fwd_bulk(const Args<R>& a, const Ctx& x, const FwdSmem<R>& s, int tt, R e_hi, R e_lo,
                                         R& m_out, R& s_out) {
  const Geometry& g = a.geo;
  const int K = a.K, Cgm = g.Cgm;
  const int kmax = min(K, tt);
  R m = Mth<R>::ninf(), sum = 0;
  int k0 = 1 + x.j;
  if (k0 == 1) k0 += g.TPL;  // k = 1 is the critical term
  if (x.active && k0 <= kmax) {
    const int step = g.TPL % K;
    int slot0 = (tt - k0) % K;
    int slot = slot0;
    for (int k = k0; k <= kmax; k += g.TPL) {
      R v = (s.ring_hi[slot * Cgm + x.cl] + e_hi) + (s.ring_lo[slot * Cgm + x.cl] + e_lo) + s.B2[(k - 1) * Cgm + x.cl];
      m = fmax(m, v);
      slot -= step;
      if (slot < 0) slot += K;
    }
    if (m != Mth<R>::ninf()) {
      slot = slot0;
      for (int k = k0; k <= kmax; k += g.TPL) {
        R v = (s.ring_hi[slot * Cgm + x.cl] + e_hi) + (s.ring_lo[slot * Cgm + x.cl] + e_lo) + s.B2[(k - 1) * Cgm + x.cl];
        sum += Mth<R>::ex2(v - m);
        slot -= step;
        if (slot < 0) slot += K;
      }
    }
  }
  group_ms(m, sum, g.GW);
  m_out = m;
  s_out = sum;
}

template <typename R>
__device__ __forceinline__ void store_part(const Geometry& g, const Ctx& x, R* pm, R* ps, int par, R m, R s) {
  // called by all threads after group reduction; one lane per (label, warp) stores
  if (!x.active) return;
  const int wl = x.j / 32;
  const bool first = (g.TPL >= 32) ? (x.lane == 0) : (x.j == 0);
  if (first) {
    size_t i = ((size_t)par * g.Cgm + x.cl) * g.WPL + wl;
    pm[i] = m;
    ps[i] = s;
  }
}

// ----------------------------------------------------------------------------
// per-position input staging
//
// Every position needs a handful of fp64 inputs per own label (prefix sums and
// projections, and in the backward the replayed window values). Loading them on
// the critical path costs a full HBM/L2 round trip per position, so they are
// staged in chunks of P positions: chunk q+2 is loaded into registers while chunk
// q is consumed, then parked in one of two shared-memory chunk buffers.
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
  int P, tb, dir, win_t0;
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
    // per-position normaliser: P <= 64 <= 2 * NT positions, at most two per thread
#pragma unroll
    for (int r = 0; r < 2; ++r) {
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

  // shared-memory index of (t, own label cl) / of position t
  __device__ __forceinline__ size_t idx(int t, int cl, int Cgm) const {
    const int d = dir * (t - tb);
    const int q = d / P, i = d - q * P;
    return ((size_t)(q & 1) * P + i) * Cgm + cl;
  }
  __device__ __forceinline__ int nidx(int t) const {
    const int d = dir * (t - tb);
    const int q = d / P, i = d - q * P;
    return (q & 1) * P + i;
  }

  // prime chunks 0 and 1 in shared memory and chunk 2 in registers (ends with a barrier)
  __device__ void begin(const Args<R>& a, const Ctx& x, StageSmem<R>& st, int tb_, int dir_, int win) {
    P = stage_chunk(a.geo);
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
    if (d > 0 && d % P == 0) {
      const int q = d / P;
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

// Runs targets t = t_begin+1 .. t_end. Preconditions: ring holds g[s] for
// s in (t_begin-K, t_begin]; Fcur = frame of target t_begin+1; n_prev = n_{t_begin}.
template <typename R, int MODE>
__device__ void fwd_sweep(const Args<R>& a, const Ctx& x, FwdSmem<R>& s, StageSmem<R>& st, Xchg<R>& xa,
                          int t_begin, int t_end, double Fcur, double n_prev, FwdBook& bk, int win_t0) {
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C, Cgm = g.Cgm;
  const int c = x.c0 + (x.active ? x.cl : 0);
  if (t_end <= t_begin) return;
  Stager<R, false> sg;
  sg.begin(a, x, st, t_begin, +1, 0);

  // e for target t_begin+1
  R e_hi, e_lo;
  {
    double e = st.E0[sg.idx(t_begin + 1, x.cls, Cgm)] - Fcur;
    split(e, e_hi, e_lo);
  }
  {
    R m, sm;
    fwd_bulk(a, x, s, t_begin + 1, e_hi, e_lo, m, sm);
    store_part(g, x, s.part_m, s.part_s, (t_begin + 1) & 1, m, sm);
  }
  __syncthreads();

  for (int t = t_begin + 1; t <= t_end; ++t) {
    const int par = t & 1;
    sg.advance(a, x, st, t);
    if (x.tid == 0) xa.arm(par);
    // (A) critical: merge bulk partials (lane-parallel tree) with the k = 1 term, publish a[t]
    if (x.gl) {
      R m = Mth<R>::ninf(), sm = 0;
      if (x.active && x.jj < g.WPL) {
        size_t i = ((size_t)par * Cgm + x.cl) * g.WPL + x.jj;
        m = s.part_m[i];
        sm = s.part_s[i];
      }
      group_ms(m, sm, g.GW);
      const int slot = (t - 1) % K;
      R v1 = (s.ring_hi[slot * Cgm + x.cls] + e_hi) + (s.ring_lo[slot * Cgm + x.cls] + e_lo) + s.B2[x.cls];
      ms_merge(m, sm, v1, (R)1);
      R av = ms_value(m, sm);
      if (x.active) xa.send(par, c, av, x.jj, g.GW, g.G);
    }
    // (C) bulk for target t+1 (frame n_{t-1} = n_prev)
    const double Fnext = n_prev;
    R en_hi = 0, en_lo = 0;
    if (t < t_end) {
      double e = st.E0[sg.idx(t + 1, x.cls, Cgm)] - Fnext;
      split(e, en_hi, en_lo);
      R m, sm;
      fwd_bulk(a, x, s, t + 1, en_hi, en_lo, m, sm);
      store_part(g, x, s.part_m, s.part_s, (t + 1) & 1, m, sm);
    }
    // (E) normaliser, gamma, ring write
    const R* aa = xa.wait(par);
    R amax = Mth<R>::ninf();
    for (int i = x.lane; i < C; i += 32) amax = fmax(amax, aa[i]);
    amax = group_max(amax, 32);
    const bool dead = (amax == Mth<R>::ninf());
    const double n_t = dead ? Fcur : Fcur + (double)amax;
    if (x.gl) {
      R ahat_own = dead ? Mth<R>::ninf() : aa[c] - amax;
      R gam;
      if (dead) {
        gam = Mth<R>::ninf();
      } else {
        // alpha-hat row in registers is read straight from the exchange buffer
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
      if (x.active && x.jj == 0) {
        double gv = (gam == Mth<R>::ninf()) ? -CUDART_INF : n_t + (double)gam + st.G0[sg.idx(t, x.cl, Cgm)];
        R hi, lo;
        split(gv, hi, lo);
        const int slot = t % K;
        s.ring_hi[slot * Cgm + x.cl] = hi;
        s.ring_lo[slot * Cgm + x.cl] = lo;
        if (MODE == MODE_FWD) {
          a.tail_alpha[((size_t)x.b * K + slot) * C + c] = ahat_own;
        } else {
          const size_t r = (size_t)x.b * (a.delta + 1) + (t - win_t0);
          a.ws_alpha[r * C + c] = ahat_own;
          a.ws_gamma[r * C + c] = gam;
        }
      }
    }
    if (MODE == MODE_REPLAY && x.tid == 0) a.ws_n[((size_t)x.b * g.G + x.rank) * (a.delta + 1) + (t - win_t0)] = n_t;
    if (MODE == MODE_FWD && x.rank == 0) {
      if (x.tid == 0) {
        a.tail_n[(size_t)x.b * K + t % K] = n_t;
        // reference bookkeeping in nats: shifted-frame dead check and checkpoint shift
        const double amax_abs = dead ? -CUDART_INF : n_t * kLn2;
        if (bk.dead_at < 0 && !(amax_abs - bk.N_cur > kGuard)) bk.dead_at = t;
        if (t % a.delta == 0 && amax_abs - bk.N_cur > kGuard) bk.N_cur = amax_abs;
        if (t % a.delta == 0 && t / a.delta < a.n_ckpt) a.N[(size_t)x.b * a.n_ckpt + t / a.delta] = bk.N_cur;
      }
      if (t == x.L && x.warp == 0) {
        R ssum = 0;
        if (!dead)
          for (int i = x.lane; i < C; i += 32) ssum += Mth<R>::ex2(aa[i] - amax);
        ssum = group_sum(ssum, 32);
        if (x.lane == 0) {
          double lz2 = dead ? -CUDART_INF : n_t + (double)Mth<R>::lg2(ssum);
          double lz = lz2 * kLn2;
          a.logZ[x.b] = lz;
          if (!(lz - bk.N_cur > kGuard) && bk.dead_at < 0) bk.dead_at = x.L;
        }
      }
    }
    Fcur = Fnext;
    n_prev = n_t;
    e_hi = en_hi;
    e_lo = en_lo;
    __syncthreads();
    if (MODE == MODE_FWD && t % a.delta == 0 && t / a.delta < a.n_ckpt) {
      // snapshot ring + tail for checkpoint i = t / delta
      const int i = t / a.delta;
      const size_t base = ck_off(a, x.b, i);
      for (int q = x.tid; q < K * x.Cg; q += g.NT) {
        int slot = q / x.Cg, cc = q % x.Cg;
        size_t gi = (base * K + slot) * C + x.c0 + cc;
        a.ck.g_hi[gi] = s.ring_hi[slot * Cgm + cc];
        a.ck.g_lo[gi] = s.ring_lo[slot * Cgm + cc];
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
__global__ void __launch_bounds__(1024) fwd_kernel(Args<R> a) {
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
    int slot = q / x.Cg, cc = q % x.Cg;
    a.tail_alpha[((size_t)x.b * K + slot) * C + x.c0 + cc] = slot == 0 ? (R)0 : Mth<R>::ninf();
  }
  if (x.rank == 0)
    for (int q = x.tid; q < K; q += g.NT) a.tail_n[(size_t)x.b * K + q] = q == 0 ? 0.0 : -CUDART_INF;
  for (int q = x.tid; q < K * Cgm; q += g.NT) {
    s.ring_hi[q] = Mth<R>::ninf();
    s.ring_lo[q] = 0;
  }
  __syncthreads();
  // position 0: alpha = 0 for every label (virtual source)
  const int c = x.c0 + (x.active ? x.cl : 0);
  if (x.gl) {
    R ssum = 0;
    for (int cp = x.jj; cp < C; cp += g.GW) ssum += Mth<R>::ex2((R)0 + s.T2c[(size_t)cp * Cgm + x.cls]);
    ssum = group_sum(ssum, g.GW);
    R gam = s.Tcmax[x.cls] + Mth<R>::lg2(ssum);
    if (x.active && x.jj == 0) {
      double gv = (double)gam - S2(x, C, 0, c) + PS2(x, C, 0, c);
      R hi, lo;
      split(gv, hi, lo);
      s.ring_hi[x.cl] = hi;
      s.ring_lo[x.cl] = lo;
    }
  }
  __syncthreads();
  // checkpoint 0 = initial ring
  {
    const size_t base = ck_off(a, x.b, 0);
    for (int q = x.tid; q < K * x.Cg; q += g.NT) {
      int slot = q / x.Cg, cc = q % x.Cg;
      size_t gi = (base * K + slot) * C + x.c0 + cc;
      a.ck.g_hi[gi] = s.ring_hi[slot * Cgm + cc];
      a.ck.g_lo[gi] = s.ring_lo[slot * Cgm + cc];
      a.ck.alpha[gi] = slot == 0 ? (R)0 : Mth<R>::ninf();
    }
    if (x.rank == 0) {
      for (int q = x.tid; q < K; q += g.NT) a.ck.n[base * K + q] = q == 0 ? 0.0 : -CUDART_INF;
      if (x.tid == 0) {
        a.ck.hdr[base * 2 + 0] = 0.0;
        a.ck.hdr[base * 2 + 1] = 0.0;
        a.N[(size_t)x.b * a.n_ckpt] = 0.0;
      }
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
  const int i_first = x.L / a.delta + 1;
  for (int i = i_first; i < a.n_ckpt; ++i) {
    const size_t base = ck_off(a, x.b, i);
    for (int q = x.tid; q < K * x.Cg; q += g.NT) {
      int slot = q / x.Cg, cc = q % x.Cg;
      size_t gi = (base * K + slot) * C + x.c0 + cc;
      a.ck.g_hi[gi] = s.ring_hi[slot * Cgm + cc];
      a.ck.g_lo[gi] = s.ring_lo[slot * Cgm + cc];
      a.ck.alpha[gi] = a.tail_alpha[((size_t)x.b * K + slot) * C + x.c0 + cc];
    }
    if (x.rank == 0) {
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
    int k = q / x.Cg, cc = q % x.Cg;
    R v = sb.gBs[k * g.Cgm + cc];
    if (v != (R)0) {
      a.gB_part[((size_t)x.b * K + k) * C + x.c0 + cc] += (double)v;
      sb.gBs[k * g.Cgm + cc] = (R)0;
    }
  }
  for (int q = x.tid; q < x.Cg * C; q += g.NT) {
    int r = q / C, cc = q % C;
    R v = sb.gTs[r * C + cc];
    if (v != (R)0) {
      a.gT_part[((size_t)x.b * C + x.c0 + r) * C + cc] += (double)v;
      sb.gTs[r * C + cc] = (R)0;
    }
  }
  __syncthreads();
}

// Per-source values of own label: w = -S2[t] + Ps2[t] - F', Gam = (F' + n_t - logZ2) + gamma~[t]
template <typename R>
struct SrcVals {
  R w_hi, w_lo, gam;
};

// bulk for source ts (durations k >= 2, k <= min(K, L - ts))
template <typename R>
__device__ __forceinline__ void bwd_bulk(const Args<R>& a, const Ctx& x, BwdSmem<R>& sb, const R* B2, int ts,
                                         const SrcVals<R>& v, R& m_out, R& s_out, R& ms_out) {
  const Geometry& g = a.geo;
  const int K = a.K, Cgm = g.Cgm;
  const int kmax = min(K, x.L - ts);
  R m = Mth<R>::ninf(), sum = 0, msum = 0;
  int k0 = 1 + x.j;
  if (k0 == 1) k0 += g.TPL;
  if (x.active && k0 <= kmax) {
    const int step = g.TPL % K;
    const int stepE = g.TPL % (K + 1);
    const int slot0 = (ts + k0) % K;
    const int eslot0 = (ts + k0) % (K + 1);
    int slot = slot0;
    for (int k = k0; k <= kmax; k += g.TPL) {
      R y = (sb.vr_hi[slot * Cgm + x.cl] + v.w_hi) + (sb.vr_lo[slot * Cgm + x.cl] + v.w_lo) + B2[(k - 1) * Cgm + x.cl];
      m = fmax(m, y);
      slot += step;
      if (slot >= K) slot -= K;
    }
    slot = slot0;
    int eslot = eslot0;
    for (int k = k0; k <= kmax; k += g.TPL) {
      R y = (sb.vr_hi[slot * Cgm + x.cl] + v.w_hi) + (sb.vr_lo[slot * Cgm + x.cl] + v.w_lo) + B2[(k - 1) * Cgm + x.cl];
      if (m != Mth<R>::ninf()) sum += Mth<R>::ex2(y - m);
      R M = Mth<R>::ex2(y + v.gam);
      msum += M;
      sb.gBs[(k - 1) * Cgm + x.cl] += M;
      sb.end_acc[eslot * Cgm + x.cl] += M;
      slot += step;
      if (slot >= K) slot -= K;
      eslot += stepE;
      if (eslot >= K + 1) eslot -= K + 1;
    }
  }
  group_ms(m, sum, g.GW);
  msum = group_sum(msum, g.GW);
  m_out = m;
  s_out = sum;
  ms_out = msum;
}

template <typename R>
__device__ __forceinline__ void store_bpart(const Geometry& g, const Ctx& x, R* bp, int par, R m, R s, R ms) {
  if (!x.active) return;
  const int wl = x.j / 32;
  const bool first = (g.TPL >= 32) ? (x.lane == 0) : (x.j == 0);
  if (first) {
    size_t i = (((size_t)par * g.Cgm + x.cl) * g.WPL + wl) * 3;
    bp[i] = m;
    bp[i + 1] = s;
    bp[i + 2] = ms;
  }
}

template <typename R>
__global__ void __launch_bounds__(1024) bwd_kernel(Args<R> a) {
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
  const int c = x.c0 + (x.active ? x.cl : 0);
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
  const double up = a.upstream ? a.upstream[x.b] : 1.0;

  // beta ring: only v[L] is live initially (beta[L] = 0)
  if (x.active && x.j == 0) {
    double vL = S2(x, C, L, c) + PE2(x, C, L - 1, c);
    R hi, lo;
    split(vL, hi, lo);
    sb.vr_hi[(L % K) * Cgm + x.cl] = hi;
    sb.vr_lo[(L % K) * Cgm + x.cl] = lo;
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
      int slot = q / Cgm, cc = q % Cgm;
      if (cc < x.Cg) {
        size_t gi = (base * K + slot) * C + x.c0 + cc;
        s.ring_hi[q] = a.ck.g_hi[gi];
        s.ring_lo[q] = a.ck.g_lo[gi];
      }
    }
    // alpha-hat at t0 for all labels (into the exchange buffer, parity of t0)
    for (int q = x.tid; q < C; q += g.NT) s.a_all[(t0 & 1) * C + q] = (R)a.ck.alpha[(base * K + (t0 % K)) * C + q];
    __syncthreads();
    const double n_t0 = a.ck.hdr[base * 2 + 1];
    const double n_t0m1 = a.ck.hdr[base * 2 + 0];
    if (x.gl) {
      const R* ah = s.a_all + (t0 & 1) * C;
      R gam = gamma_from_alpha(ah, s.T2c, s.Tcmax, C, Cgm, x.cls, x.jj, g.GW);
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
    // all CTAs must finish the replay (they exchange through a_all) before we reuse barriers
    cl.sync();

    // ---- beta sweep over sources t = t1-1 .. t0
    Stager<R, true> sg;
    sg.begin(a, x, st, t1 - 1, -1, t0);
    auto src = [&](int ts, double Fp) {
      SrcVals<R> v;
      const size_t k = sg.idx(ts, x.cls, Cgm);
      split(st.G0[k] - Fp, v.w_hi, v.w_lo);
      v.gam = (R)(Fp + st.n[sg.nidx(ts)] - logZ2) + st.gam[k];
      return v;
    };
    SrcVals<R> cur = src(t1 - 1, Fp_cur);
    {
      R m, sm, ms;
      bwd_bulk(a, x, sb, s.B2, t1 - 1, cur, m, sm, ms);
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
          size_t q = (((size_t)par * Cgm + x.cl) * g.WPL + x.jj) * 3;
          m = sb.bpart[q];
          sm = sb.bpart[q + 1];
          ms = sb.bpart[q + 2];
        }
        group_ms(m, sm, g.GW);
        ms = group_sum(ms, g.GW);
        const int slot = (t + 1) % K;
        R y1 = (sb.vr_hi[slot * Cgm + x.cls] + cur.w_hi) + (sb.vr_lo[slot * Cgm + x.cls] + cur.w_lo) + s.B2[x.cls];
        R M1 = Mth<R>::ex2(y1 + cur.gam);
        ms_merge(m, sm, y1, (R)1);
        ms += M1;
        R dv = ms_value(m, sm);
        if (x.active && x.jj == 0) {
          sb.end1[((t + 1) % (K + 1)) * Cgm + x.cl] = M1;
          sb.gBs[x.cl] += M1;
          a.start_g[((size_t)x.b * (a.T + 1) + t) * C + c] = ms;
        }
        if (x.active) xd.send(par, c, dv, x.jj, g.GW, g.G);
      }
      // (C) bulk for source t-1 (frame nd_{t+1})
      SrcVals<R> nxt = cur;
      if (t - 1 >= t0) {
        nxt = src(t - 1, nd_prev);
        R m, sm, ms;
        bwd_bulk(a, x, sb, s.B2, t - 1, nxt, m, sm, ms);
        store_bpart(g, x, sb.bpart, (t - 1) & 1, m, sm, ms);
      }
      // (E) beta at t, grad_T, v[t], end emission
      const R* dd = xd.wait(par);
      R dmax = Mth<R>::ninf();
      for (int q = x.lane; q < C; q += 32) dmax = fmax(dmax, dd[q]);
      dmax = group_max(dmax, 32);
      const bool dead = (dmax == Mth<R>::ninf());
      const double nd_t = dead ? Fp_cur : Fp_cur + (double)dmax;
      if (x.gl && !dead) {
        const size_t k = sg.idx(t, x.cls, Cgm);
        const double n_t = st.n[sg.nidx(t)];
        const R Zt = (R)(n_t + nd_t - logZ2);
        const R ahat = st.ahat[k];
        R ssum = 0;
        for (int q = x.jj; q < C; q += g.GW) {
          const R dh = dd[q] - dmax;
          ssum += Mth<R>::ex2(sb.T2r[(size_t)x.cls * C + q] + dh);
          if (x.active && ahat != Mth<R>::ninf()) sb.gTs[(size_t)x.cls * C + q] += Mth<R>::ex2(ahat + sb.T2o[(size_t)x.cls * C + q] + dh + Zt);
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
          double vv = (bt == Mth<R>::ninf()) ? -CUDART_INF : st.E0[k] + nd_t + (double)bt;
          R hi, lo;
          split(vv, hi, lo);
          sb.vr_hi[(t % K) * Cgm + x.cl] = hi;
          sb.vr_lo[(t % K) * Cgm + x.cl] = lo;
        }
      }
      if (x.active && x.j == 0) {
        const int e = t + K;
        if (e <= L) {
          const int es = e % (K + 1);
          a.end_g[((size_t)x.b * (a.T + 1) + e) * C + c] = sb.end_acc[es * Cgm + x.cl] + sb.end1[es * Cgm + x.cl];
          sb.end_acc[es * Cgm + x.cl] = (R)0;
        }
      }
      Fp_cur = nd_prev;
      nd_prev = nd_t;
      cur = nxt;
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
      a.end_g[((size_t)x.b * (a.T + 1) + e) * C + c] = sb.end_acc[es * Cgm + x.cl] + sb.end1[es * Cgm + x.cl];
    }
  }
  flush_grads(a, x, sb);
  (void)up;
  cl.sync();
}

// ----------------------------------------------------------------------------
// finalize: start/end masses -> grad_S, grad_P*, marginals (diagnostics.py:54-79)
//
// One thread per (b, c): sequential fp64 scan over t (coverage cumsum).

template <typename R>
__global__ void finalize_kernel(const R* start_g, const R* end_g, const int64_t* lengths,
                                const double* upstream, int B, int T, int C, double* grad_S, double* grad_Ps,
                                double* grad_Pe, double* pos) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * C) return;
  int b = idx / C, c = idx % C;
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
      double pm = (t < L) ? fmin(fmax(cov, 0.0), 1.0) : 0.0;
      pos[((size_t)b * T + t) * C + c] = pm;
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
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
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
