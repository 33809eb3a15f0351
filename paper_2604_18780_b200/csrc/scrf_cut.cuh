// Cut normalisers: exact-identity drift correction of the fp32 message sweeps (sm_100a).
//
// Every segmentation of [0, L) either has a boundary at t or one segment [s, e) with
// s < t < e, so for every boundary t (Appendix A identities; the reference's
// coverage bookkeeping, streaming.py:357-380, relies on the same fact):
//
//   U_t = sum_c E[t,c] + sum_c sum_{s < t < e <= s+K} mu(s, e-s, c) = 1,
//   E[t,c] = 2^(alpha[t,c] + beta[t,c] - Z),  mu = 2^(ra[s,c] + rb[e,c] + B[e-s-1,c])   (log2 units)
//
// with ra = gamma - S + Ps (alpha side) and rb = beta + S + Pe - Z (beta side), as in the
// grad_B pass (scrf_post.cuh). At t = 0 the identity is sum_c A[0,c] = 1, at t = L it is
// sum_c E[L,c] = 1.
//
// The fp32 sweeps carry a slowly varying frame error eps_t (a random walk plus a small
// per-step bias of the fp32/MUFU arithmetic, up to ~1e-4 relative at T = 1e5): every mass
// computed at boundary t is off by the factor (1 + eps_t), and U_t measures exactly that
// factor. The posterior passes divide the masses by U interpolated (in log space) between
// cut points every `d` positions; the residual is the walk's excursion between two cuts.
//
// Cost per interior cut and label: K(K-1)/2 terms, evaluated in exp space on the FMA pipe
// (a_s = 2^(ra[s] - Ra), b_e = 2^(rb[e] - Rb), w_k = 2^(B[k] - Bmax): 2K + K ex2, K^2/2 FMA)
// with per-block fp64 accumulation. Terms that underflow fp32 in a factor are below
// 2^-126 of a term bound that is itself <= 1 up to the duration-bias range: negligible.
#pragma once

#include "scrf_common.cuh"

namespace scrf {

constexpr int kCutSG = 8;   // sources per thread (register window over w)
constexpr int kCutEC = 64;  // targets per work item
constexpr int kCutCG = 4;   // labels per CTA

template <typename R>
struct CutArgs {
  const double* S;
  const int64_t* lengths;
  const double* dur;
  const double* ps;
  const double* pe;
  const double* logZ;  // (B,) nats
  int B, T, K, C;
  const R *Ya, *Xa, *Yb, *Xb;  // message rows as in PostArgs (alpha b*rowsA + t - tA0, beta b*rowsB + t - tB0)
  const double *na, *nb;
  int rowsA, tA0, rowsB, tB0;
  int w0, w1;                  // positions of this pass
  int d;                       // cut spacing
  int ncut;                    // cut slots per sequence: w0, w0 + d, ..., and min(w1, L) (last used slot)
  double* U;                   // [B][ncut][C] per-label contributions to U_t
  const int* tcut;             // probe mode: one cut per sequence at tcut[b] (slot 0), or null
  // pass mode: the pass's transposed source / target values (PostArgs::RA / RB, post_prep_kernel)
  // and the duration weights w[c][i] = 2^(B[i - kCutEC - 1, c] - Bmax[c]) (cut_w_kernel)
  const double *RA, *RB;
  int t_lo, NR;
  const R* Wt;
  const double* Bmax;
};

// per-label duration weights of the cut kernel (independent of the cut): Wt[c][i], i in [0, 2K +
// 2 kCutEC), k = i - kCutEC, w = 2^(B[k-1,c] - Bmax[c]) for k in 1..K, else 0
template <typename R>
__global__ void cut_w_kernel(const double* dur, int K, int C, R* Wt, double* Bmax) {
  __shared__ double red[8];
  const int c = blockIdx.x;
  double bm = -CUDART_INF;
  for (int k = threadIdx.x; k < K; k += blockDim.x) bm = fmax(bm, dur[(size_t)k * C + c] * kLog2e);
  for (int o = 16; o > 0; o >>= 1) bm = fmax(bm, __shfl_xor_sync(0xffffffffu, bm, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = bm;
  __syncthreads();
  bm = -CUDART_INF;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) bm = fmax(bm, red[i]);
  const int NW = 2 * K + 2 * kCutEC;
  for (int i = threadIdx.x; i < NW; i += blockDim.x) {
    const int k = i - kCutEC;
    Wt[(size_t)c * NW + i] =
        (bm > -CUDART_INF && k >= 1 && k <= K) ? Mth<R>::ex2((R)(dur[(size_t)(k - 1) * C + c] * kLog2e - bm)) : (R)0;
  }
  if (threadIdx.x == 0) Bmax[c] = bm;
}

// cut slots of a pass [w0, w1) for a sequence of length L: t_j = w0 + j d for j <= J =
// (tend - 1 - w0) / d, t_{J+1} = tend = min(w1, L)
__host__ __device__ inline int cut_J(int w0, int tend, int d) { return tend > w0 ? (tend - 1 - w0) / d : 0; }
__host__ __device__ inline int cut_count(int w0, int tend, int d) { return cut_J(w0, tend, d) + 2; }
__host__ __device__ inline int cut_pos(int j, int w0, int tend, int d) {
  return j <= cut_J(w0, tend, d) ? w0 + j * d : tend;
}
__host__ __device__ inline int cut_slots(int w0, int w1, int d) { return d > 0 ? (w1 - w0 - 1) / d + 2 : 0; }

// w is stored skewed (one pad word per 8): the lanes of a warp read w at indices 8 apart
// (consecutive source groups), which the skew spreads over distinct banks
__host__ __device__ inline int cut_wphys(int x) { return x + (x >> 3); }

template <typename R>
__host__ __device__ inline size_t cut_smem(int K) {
  // per label: a[K + kCutSG] (sources t-K+1 .. t-1, padded), b[K + kCutEC] (targets), w[2K + 2 kCutEC]
  return (size_t)kCutCG * ((K + kCutSG) + (K + kCutEC) + cut_wphys(2 * K + 2 * kCutEC)) * sizeof(R) +
         (size_t)(K / kCutSG + K / kCutEC + 4) + 64;
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];  // fixed order
  return s;
}

__device__ __forceinline__ double block_max_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = -CUDART_INF;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = fmax(s, red[i]);
  return s;
}

// grid (cut slot j, label group, b), 256 threads
template <typename R>
__global__ void __launch_bounds__(256, 3) cut_kernel(CutArgs<R> a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double red[8];
  const int j = blockIdx.x, cg = blockIdx.y, b = blockIdx.z;
  const int C = a.C, T = a.T, K = a.K;
  const int L = (int)a.lengths[b];
  int t;
  if (a.tcut) {
    if (j > 0) return;
    t = a.tcut[b];
  } else {
    if (L < a.w0) return;
    const int tend = min(a.w1, L);
    if (j >= cut_count(a.w0, tend, a.d)) return;
    t = cut_pos(j, a.w0, tend, a.d);
  }
  const int c0 = cg * kCutCG;
  const int Cn = min(kCutCG, C - c0);
  const size_t rb0 = (size_t)b * (T + 1);
  const size_t ra0 = (size_t)b * a.rowsA - a.tA0;  // alpha row of t: ra0 + t
  const size_t rbb = (size_t)b * a.rowsB - a.tB0;  // beta row of t: rbb + t
  // log2 Z reference of the masses; without logZ (probe mode) the frames of the cut itself
  const double Z2 = a.logZ ? a.logZ[b] * kLog2e : a.na[ra0 + t] + a.nb[rbb + t];
  const int NA = K + kCutSG, NBv = K + kCutEC, NW = 2 * K + 2 * kCutEC, NWp = cut_wphys(NW);
  R* sa = (R*)sm;                      // [CG][NA]   a[s], s = t-K+1+i
  R* sb = sa + (size_t)kCutCG * NA;    // [CG][NBv]  b[e], e = t+1+i
  R* sw = sb + (size_t)kCutCG * NBv;   // [CG][NW]   w[k], k = i - kCutEC (k in 1..K nonzero)
  const int nsg = (K - 1 + kCutSG - 1) / kCutSG;
  const int nec = (K - 1 + kCutEC - 1) / kCutEC;
  unsigned char* nzA = (unsigned char*)(sw + (size_t)kCutCG * cut_wphys(2 * K + 2 * kCutEC));  // [nsg]
  unsigned char* nzB = nzA + nsg;                                                             // [nec]
  const int s_lo = t - K + 1;
  for (int cl = 0; cl < Cn; ++cl) {
    const int c = c0 + cl;
    // point term: E[t,c] (interior, t = L) or A[0,c] (t = 0), fp64
    double pt = 0.0;
    if (threadIdx.x == 0) {
      const size_t oa = (ra0 + t) * C + c, ob = (rbb + t) * C + c;
      const double f = a.na[ra0 + t] + a.nb[rbb + t] - Z2;
      const R y = t == 0 ? a.Xa[oa] : a.Ya[oa];
      const R x = t == 0 ? a.Yb[ob] : a.Xb[ob];
      if (y > Mth<R>::ninf() && x > Mth<R>::ninf()) pt = exp2(f + (double)y + (double)x);
    }
    double cross = 0.0;
    if (t > 0 && t < L && K >= 2) {
      // log2 source / target values (fp64), their maxima as references
      double ra_max = -CUDART_INF, rb_max = -CUDART_INF, bm = -CUDART_INF;
      const double* rA = a.RA ? a.RA + ((size_t)b * C + c) * a.NR - a.t_lo : nullptr;  // index: position
      const double* rB = a.RB ? a.RB + ((size_t)b * C + c) * a.NR - a.t_lo : nullptr;
      auto src = [&](int s) -> double {  // ra[s] (-inf: no source)
        if (s < 0) return -CUDART_INF;
        if (rA) return rA[s];
        const R xa = a.Xa[(ra0 + s) * C + c];
        if (!(xa > Mth<R>::ninf())) return -CUDART_INF;
        return a.na[ra0 + s] + (double)xa - a.S[(rb0 + s) * C + c] * kLog2e +
               ((a.ps && s < T) ? a.ps[((size_t)b * T + s) * C + c] * kLog2e : 0.0);
      };
      auto tgt = [&](int e) -> double {  // rb[e] (-inf: no target)
        if (e > L) return -CUDART_INF;
        if (rB) return rB[e];
        const R xb = a.Xb[(rbb + e) * C + c];
        if (!(xb > Mth<R>::ninf())) return -CUDART_INF;
        return a.nb[rbb + e] + (double)xb + a.S[(rb0 + e) * C + c] * kLog2e +
               (a.pe ? a.pe[((size_t)b * T + e - 1) * C + c] * kLog2e : 0.0) - Z2;
      };
      for (int i = threadIdx.x; i < K - 1; i += blockDim.x) {
        ra_max = fmax(ra_max, src(s_lo + i));
        rb_max = fmax(rb_max, tgt(t + 1 + i));
      }
      if (a.Bmax) {
        bm = a.Bmax[c];
      } else {
        for (int k = threadIdx.x; k < K; k += blockDim.x) bm = fmax(bm, a.dur[(size_t)k * C + c] * kLog2e);
      }
      ra_max = block_max_d(ra_max, red);
      rb_max = block_max_d(rb_max, red);
      if (!a.Bmax) bm = block_max_d(bm, red);
      R* A = sa + (size_t)cl * NA;
      R* Bv = sb + (size_t)cl * NBv;
      R* W = sw + (size_t)cl * NWp;
      const bool live = ra_max > -CUDART_INF && rb_max > -CUDART_INF && bm > -CUDART_INF;
      for (int i = threadIdx.x; i < NA; i += blockDim.x) {
        R v = 0;
        if (live && i < K - 1) {
          const double ra = src(s_lo + i);
          if (ra > -CUDART_INF) v = Mth<R>::ex2((R)(ra - ra_max));
        }
        A[i] = v;
      }
      for (int i = threadIdx.x; i < NBv; i += blockDim.x) {
        R v = 0;
        if (live && i < K - 1) {
          const double rv = tgt(t + 1 + i);
          if (rv > -CUDART_INF) v = Mth<R>::ex2((R)(rv - rb_max));
        }
        Bv[i] = v;
      }
      if (a.Wt) {
        const R* wg = a.Wt + (size_t)c * NW;
        for (int i = threadIdx.x; i < NW; i += blockDim.x) W[cut_wphys(i)] = live ? wg[i] : (R)0;
      } else {
        for (int i = threadIdx.x; i < NW; i += blockDim.x) {
          const int k = i - kCutEC;
          W[cut_wphys(i)] = (live && k >= 1 && k <= K) ? Mth<R>::ex2((R)(a.dur[(size_t)(k - 1) * C + c] * kLog2e - bm)) : (R)0;
        }
      }
      __syncthreads();
      // sum_{s,e} a_s b_e w_{e-s}: item = (source group of kCutSG, target chunk of kCutEC).
      // Groups whose a (or chunks whose b) all underflowed contribute exactly 0 and are skipped:
      // path mass decays geometrically away from the cut, so few items remain on real data.
      for (int i = threadIdx.x; i < nsg + nec; i += blockDim.x) {
        bool nz = false;
        if (i < nsg) {
          for (int r = 0; r < kCutSG; ++r) nz |= A[i * kCutSG + r] != (R)0;
          nzA[i] = nz;
        } else {
          const int q = i - nsg;
          for (int u = 0; u < kCutEC; ++u) nz |= Bv[q * kCutEC + u] != (R)0;
          nzB[q] = nz;
        }
      }
      __syncthreads();
      double acc = 0.0;
      // lanes of a warp take consecutive source groups of one target chunk (b[e] reads are
      // broadcasts, w reads conflict-free through the skew); chunks entirely past the
      // duration limit (e - s > K for every pair) are skipped
      for (int it = threadIdx.x; it < nsg * nec; it += blockDim.x) {
        const int q = it / nsg, g = it % nsg;
        if (q * kCutEC > g * kCutSG + kCutSG - 1 || !nzA[g] || !nzB[q]) continue;
        const int i0 = g * kCutSG;   // sources s = s_lo + i0 + r, r < kCutSG
        const int e0 = q * kCutEC;   // targets e = t + 1 + e0 + u
        // k = e - s = (t + 1 + e0 + u) - (s_lo + i0 + r) = K + e0 + u - i0 - r
        const int kb = K + e0 - i0;  // k of (u = 0, r = 0)
        R sr[kCutSG];
#pragma unroll
        for (int r = 0; r < kCutSG; ++r) sr[r] = 0;
        // sub-blocks of 16 targets, fully unrolled: the window of w values the 16 x kCutSG
        // terms need sits in registers (no shifting), one b load per target
        constexpr int kU = 16;
#pragma unroll 1
        for (int u0 = 0; u0 < kCutEC; u0 += kU) {
          R wb[kCutSG - 1 + kU];  // wb[j] = w[kb + u0 - (kCutSG - 1) + j]
#pragma unroll
          for (int jj = 0; jj < kCutSG - 1 + kU; ++jj) wb[jj] = W[cut_wphys(kb + u0 - (kCutSG - 1) + jj + kCutEC)];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const R bv = Bv[e0 + u0 + u];
#pragma unroll
            for (int r = 0; r < kCutSG; ++r) sr[r] = fma(bv, wb[u - r + kCutSG - 1], sr[r]);
          }
        }
        double tot = 0.0;
#pragma unroll
        for (int r = 0; r < kCutSG; ++r) tot += (double)A[i0 + r] * (double)sr[r];
        acc += tot;
      }
      acc = block_sum_d(acc, red);
      if (live && acc > 0.0) cross = acc * exp2(ra_max + rb_max + bm);
      __syncthreads();
    }
    if (threadIdx.x == 0) a.U[((size_t)b * a.ncut + j) * C + c] = pt + cross;
  }
}

// log2 correction of boundary t: -lerp_j(log2 U_j) with U summed over labels in fixed order;
// 0 when the cut totals are not sane (|log2 U| > 1e-2: nothing to correct reliably)
__device__ __forceinline__ double cut_log2U(const double* U, int C) {
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += U[c];
  const double l = s > 0.0 ? log2(s) : 0.0;
  return fabs(l) <= 1e-2 ? l : 0.0;
}

}  // namespace scrf

namespace scrf {

// per-position log2 correction corr[b][t - w0] = -lerp(log2 U) between the enclosing cut slots
// (0 past L); grid (chunks of 256 positions of [w0, w1), B). Also counts the beta positions
// whose (absolute, unnormalised in the reference) message max leaves +-CLAMP_LIMIT (the
// reference would clamp them, _numerics.py:41-56).
template <typename R>
__global__ void __launch_bounds__(256) cut_corr_kernel(const int64_t* lengths, int C, int w0, int w1, int d, int ncut,
                                                       const double* U, double* corr, const R* Xb, const double* nb,
                                                       int rowsB, int tB0, int32_t* clampB) {
  const int b = blockIdx.y;
  const int t = w0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= w1) return;
  const int L = (int)lengths[b];
  if (clampB && t < L) {
    const size_t rt = (size_t)b * rowsB + t - tB0;
    R m = Mth<R>::ninf();
    for (int c = 0; c < C; ++c) m = fmax(m, Xb[rt * C + c]);
    if (m > Mth<R>::ninf() && fabs((nb[rt] + (double)m) * kLn2) > kClampLimit) atomicAdd(&clampB[b], 1);
  }
  double v = 0.0;
  if (d > 0 && t <= L) {
    const int tend = min(w1, L);
    const int J = cut_J(w0, tend, d);
    const int j = min((t - w0) / d, J);
    const int t0 = cut_pos(j, w0, tend, d), t1 = cut_pos(j + 1, w0, tend, d);
    const double* Ub = U + (size_t)b * ncut * C;
    const double l0 = cut_log2U(Ub + (size_t)j * C, C);
    const double l1 = cut_log2U(Ub + (size_t)(j + 1) * C, C);
    const double f = t1 > t0 ? (double)(t - t0) / (double)(t1 - t0) : 0.0;
    v = -(l0 + (l1 - l0) * f);
  }
  if (corr) corr[(size_t)b * (w1 - w0) + t - w0] = v;
}

}  // namespace scrf

namespace scrf {

// Exclusive prefix of the coverage chunk totals of a pass [w0, w1), re-anchored at every cut
// point: the coverage of cell t_j - 1 is exactly E[t_j,c] + (segments of label c crossing t_j),
// the per-label cut contribution U[b][j][c] (divided by the cut total, the frame correction at
// t_j), so the running sum restarts there and fp32 rounding accumulates over <= d positions
// only. Chunk starts coincide with cut points (CH divides d). The first chunk starts from the
// anchor at w0 (0 at w0 = 0; the running coverage of the previous pass if the anchor is not
// sane); the coverage at the end of the pass is left in carry[b][c]. One thread per (b, c).
__global__ void cut_prefix_kernel(const int64_t* lengths, int B, int C, int nch, int CH, int w0, int w1, int d,
                                  int ncut, const double* U, double* tot, double* carry) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * C) return;
  const int b = i / C, c = i % C;
  const int L = (int)lengths[b];
  const int tend = min(w1, L);
  const int J = cut_J(w0, tend, d);
  const double* Ub = U + (size_t)b * ncut * C;
  double* base = tot + (size_t)b * nch * C + c;
  double run = (w0 == 0 || !carry) ? 0.0 : carry[(size_t)b * C + c];
  // batches of 16 chunk totals loaded before any store (the loads pipeline instead of
  // serialising behind the stores to the same array)
  constexpr int kQB = 16;
  for (int qb = 0; qb < nch; qb += kQB) {
    double v[kQB];
#pragma unroll
    for (int i = 0; i < kQB; ++i) v[i] = qb + i < nch ? base[(size_t)(qb + i) * C] : 0.0;
#pragma unroll
    for (int i = 0; i < kQB; ++i) {
      const int q = qb + i;
      if (q >= nch) break;
      const int t0 = w0 + q * CH;
      if (t0 > 0 && t0 < tend && (t0 - w0) % d == 0 && (t0 - w0) / d <= J) {
        const int j = (t0 - w0) / d;
        double s = 0.0;
        for (int cc = 0; cc < C; ++cc) s += Ub[(size_t)j * C + cc];
        const double l = s > 0.0 ? log2(s) : 1.0;
        if (fabs(l) <= 1e-2) run = Ub[(size_t)j * C + c] / s;
      }
      base[(size_t)q * C] = run;
      run += v[i];
    }
  }
  if (carry) carry[(size_t)b * C + c] = run;
}

}  // namespace scrf

namespace scrf {

// Provisional log-partition of each sequence from one cut (the overlapped posterior passes run
// before either sweep has finished, so the final log Z is not known yet). With the frame
// reference Z_f = n_alpha[t] + n_beta[t] (log2) the cut total is U_t(Z_f) = 2^(Z - Z_f) exactly,
// so Z~ = Z_f + log2 U_t(Z_f) is log Z up to the frame drift the cut normalisers measure and
// remove anyway: every mass of a pass is divided by U interpolated between its cuts, which
// makes the pass outputs independent of the Z reference up to rounding.
//   probe position: the cut point nearest the middle of the sequence (both sweeps reach it first)
__host__ __device__ inline int probe_pos(int L, int d) { return d * ((L / 2) / d); }

__global__ void probe_pos_kernel(const int64_t* lengths, int B, int d, int* tcut) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) tcut[b] = probe_pos((int)lengths[b], d);
}

template <typename R>
__global__ void probe_finish_kernel(const int64_t* lengths, int B, int C, const int* tcut, const double* na,
                                    const double* nb, int rowsA, int tA0, int rowsB, int tB0, const double* U,
                                    double* Zt) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int t = tcut[b];
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += U[(size_t)b * C + c];
  const double zf = na[(size_t)b * rowsA + t - tA0] + nb[(size_t)b * rowsB + t - tB0];
  Zt[b] = s > 0.0 ? (zf + log2(s)) * kLn2 : -CUDART_INF;
}

}  // namespace scrf
