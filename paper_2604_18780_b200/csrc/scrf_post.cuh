// Posterior passes on B200 (sm_100a): everything the reference's backward derives from
// the joint segment marginals mu[b,s,k,c,c'] (pkg/src/streamcrf/streaming.py:357-395,
// diagnostics.py:54-79), computed data-parallel from the per-position messages the two
// sweeps stored (scrf_sweep.cuh). Exact identities used (log2 units, Z = logZ):
//   end mass   E[t,c] = sum_{k,c'} mu(seg ending at t)  = 2^(alpha[t,c] + beta[t,c] - Z)
//   start mass A[t,c] = sum_{k,c'} mu(seg starting at t) = 2^(gamma[t,c] + delta[t,c] - Z)
//   grad_T[c',c] = sum_t 2^(alpha[t,c'] + T[c',c] + delta[t,c] - Z)
//   grad_B[k,c]  = sum_s 2^(ra[s,c] + rb[s+k,c] - Z + B[k-1,c])
// with ra = gamma - S + Ps (alpha-side source value) and rb = beta + S + Pe (beta side).
// grad_S[t] = E[t] - A[t]; grad_Ps[t] = A[t]; grad_Pe[t-1] = E[t]; position marginals are
// the running sum of A - E (coverage difference array); boundary posterior = sum_c A[t,c].
// All batch/segment reductions are fixed-order (bit-reproducible), as in the reference.
#pragma once

#include "scrf_common.cuh"

namespace scrf {

template <typename R>
struct PostArgs {
  const double* S;
  const int64_t* lengths;
  const double* trans;
  const double* dur;
  const double* ps;
  const double* pe;
  const double* upstream;  // (B,) or null
  const double* logZ;      // (B,) nats
  int B, T, K, C;
  const R *Ya, *Xa, *Yb, *Xb;  // message rows: alpha side b*rowsA + t - tA0, beta side b*rowsB + t - tB0
  const double *na, *nb;
  int rowsA, tA0, rowsB, tB0;
  int w0, w1;                  // positions [w0, w1) of this pass (full mode: [0, T+1))
  const double* corr;          // [B][w1-w0] log2 frame correction from the cut normalisers (scrf_cut.cuh) or null
  // outputs
  double* grad_S;  // (B, T+1, C)
  double* grad_Ps; // (B, T, C) or null
  double* grad_Pe; // (B, T, C) or null
  double* pos;     // (B, T, C)
  double* bnd;     // (B, T)
  // chunk partials
  int CH, nch;        // positions per chunk, chunks per sequence in [w0, w1)
  double* tot;        // [B][nch][C]  chunk totals of (A - E)
  double* cntp;       // [B][nch]
  double* gTp;        // [B][nch][C][C]
  int SCB, nchB;      // grad_B: sources per CTA, CTAs per sequence (sources in [w0, w1))
  int CGB;            // labels per grad_B CTA
  double* gBp;        // [B][nchB][K][C]
  // partial-array placement: cntp / gTp chunk ch of sequence b at b*pnch + pq0 + ch, gBp
  // micro-chunk m at b*pnchB + pm0 + m (a window of a sequence-wide partial array; the final
  // sums then run over the whole sequence in one fixed order whatever the windowing)
  int pq0, pnch, pm0, pnchB;
  // log2 source / target values of the pass (post_prep_kernel), transposed per label:
  //   RA[b][c][s - t_lo] = na[s] + Xa[s,c] - S[s,c] + Ps[s,c]          (s in [w0 - K + 1, w1 - 1])
  //   RB[b][c][u - t_lo] = nb[u] + Xb[u,c] + S[u,c] + Pe[u-1,c] - Z    (u in [w0 + 1, w1 + K - 1])
  // (log2 units, -inf outside those ranges, past L or where the message is -inf)
  double *RA, *RB;
  int t_lo, NR;
  float gb_range;     // exp-space grad_B: detrended range above which a block takes the exact path
};

template <typename R>
__device__ __forceinline__ size_t rowA(const PostArgs<R>& a, int b, int t) { return (size_t)b * a.rowsA + (t - a.tA0); }
template <typename R>
__device__ __forceinline__ size_t rowB(const PostArgs<R>& a, int b, int t) { return (size_t)b * a.rowsB + (t - a.tB0); }

__host__ __device__ inline int post_chunk(int C) {
  int ch = 256;
  while (ch > 16 && (size_t)ch * C > 4096) ch >>= 1;
  return ch;
}

// pass 1: per (b, chunk) of CH positions: masses, grad_S / grad_P, local coverage scan,
// boundary posterior, chunk totals, count and grad_T partials.
// Transposed log2 source / target rows of a pass (PostArgs::RA / RB), shared by the cut and
// grad_B kernels: each value is computed once, read row-major (coalesced over labels) and
// written label-major (coalesced over positions) through a shared-memory tile. Grid
// (ceil(NR / 32), B), 256 threads, smem 2 * C * 33 doubles.
constexpr int kPrepRows = 32;
template <typename R>
__global__ void __launch_bounds__(256) post_prep_kernel(PostArgs<R> a) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* tA = (double*)sm;                       // [C][kPrepRows + 1]
  double* tB = tA + (size_t)a.C * (kPrepRows + 1);
  const int b = blockIdx.y, C = a.C, T = a.T, K = a.K;
  const int r0 = blockIdx.x * kPrepRows;
  const int L = (int)a.lengths[b];
  const double Z2 = a.logZ[b] * kLog2e;
  const int aLo = a.w0 - K + 1, aHi = a.w1 - 1;  // source range
  const int bLo = a.w0 + 1, bHi = a.w1 + K - 1;  // target range
  const size_t rs0 = (size_t)b * (T + 1);
  for (int i = threadIdx.x; i < kPrepRows * C; i += blockDim.x) {
    const int r = i / C, c = i % C;
    const int t = a.t_lo + r0 + r;
    double va = -CUDART_INF, vb = -CUDART_INF;
    if (r0 + r < a.NR && t >= 0 && t <= L) {
      const double sv = a.S[(rs0 + t) * C + c] * kLog2e;
      if (t >= aLo && t <= aHi) {
        const size_t oa = rowA(a, b, t);
        const R xa = a.Xa[oa * C + c];
        if (xa > Mth<R>::ninf())
          va = a.na[oa] + (double)xa - sv + ((a.ps && t < T) ? a.ps[((size_t)b * T + t) * C + c] * kLog2e : 0.0);
      }
      if (t >= bLo && t <= bHi && t >= 1) {
        const size_t ob = rowB(a, b, t);
        const R xb = a.Xb[ob * C + c];
        if (xb > Mth<R>::ninf())
          vb = a.nb[ob] + (double)xb + sv + (a.pe ? a.pe[((size_t)b * T + t - 1) * C + c] * kLog2e : 0.0) - Z2;
      }
    }
    tA[(size_t)c * (kPrepRows + 1) + r] = va;
    tB[(size_t)c * (kPrepRows + 1) + r] = vb;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPrepRows * C; i += blockDim.x) {
    const int c = i / kPrepRows, r = i % kPrepRows;
    if (r0 + r < a.NR) {
      const size_t o = ((size_t)b * C + c) * a.NR + r0 + r;
      a.RA[o] = tA[(size_t)c * (kPrepRows + 1) + r];
      a.RB[o] = tB[(size_t)c * (kPrepRows + 1) + r];
    }
  }
}
__host__ __device__ inline size_t post_prep_smem(int C) { return (size_t)2 * C * (kPrepRows + 1) * sizeof(double); }

template <typename R>
__global__ void __launch_bounds__(256) post_pos_kernel(PostArgs<R> a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.y, ch = blockIdx.x;
  const int C = a.C, T = a.T, CH = a.CH;
  const int L = (int)a.lengths[b];
  const int t0 = a.w0 + ch * CH;
  const int nt = min(CH, a.w1 - t0);
  double* dA = (double*)sm;                 // [CH][C] start mass
  double* dE = dA + (size_t)CH * C;         // [CH][C] end mass
  R* sYa = (R*)(dE + (size_t)CH * C);       // [CH][C]
  R* sYb = sYa + (size_t)CH * C;            // [CH][C]
  double* sf = (double*)(sm + ((2 * (size_t)CH * C * sizeof(double) + 2 * (size_t)CH * C * sizeof(R) + 15) & ~(size_t)15));
  __shared__ double red[256];
  const double Z2 = a.logZ[b] * kLog2e;
  const double up = a.upstream ? a.upstream[b] : 1.0;
  const size_t rb = (size_t)b * (T + 1);
  const int W = a.w1 - a.w0;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int t = t0 + i;
    sf[i] = (t <= L) ? a.na[rowA(a, b, t)] + a.nb[rowB(a, b, t)] - Z2 + (a.corr ? a.corr[(size_t)b * W + t - a.w0] : 0.0)
                     : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nt * C; e += blockDim.x) {
    const int i = e / C, c = e % C, t = t0 + i;
    const size_t o = (rb + t) * C + c;
    double A = 0.0, E = 0.0;
    R ya = Mth<R>::ninf(), yb = Mth<R>::ninf();
    if (t <= L) {
      const size_t oa = rowA(a, b, t) * C + c, ob = rowB(a, b, t) * C + c;
      const R f = (R)sf[i];
      ya = a.Ya[oa];
      if (t < L) {
        yb = a.Yb[ob];
        A = (double)Mth<R>::ex2(f + a.Xa[oa] + yb);
      }
      if (t >= 1) E = (double)Mth<R>::ex2(f + ya + a.Xb[ob]);
    }
    dA[e] = A;
    dE[e] = E;
    sYa[e] = ya;
    sYb[e] = yb;
    a.grad_S[o] = up * (E - A);
    if (t < T) {
      if (a.grad_Ps) a.grad_Ps[((size_t)b * T + t) * C + c] = up * A;
    }
    if (t >= 1 && a.grad_Pe) a.grad_Pe[((size_t)b * T + t - 1) * C + c] = up * E;
  }
  __syncthreads();
  // boundary posterior and count
  double cnt = 0.0;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int t = t0 + i;
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += dA[(size_t)i * C + c];
    cnt += s;
    if (t < T) a.bnd[(size_t)b * T + t] = (t < L) ? fmin(fmax(s, 0.0), 1.0) : 0.0;
  }
  red[threadIdx.x] = cnt;
  // local coverage scan per label (sequential over the chunk, fp64)
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    double cov = 0.0;
    for (int i = 0; i < nt; ++i) {
      const int t = t0 + i;
      cov += dA[(size_t)i * C + c] - dE[(size_t)i * C + c];
      if (t < T) a.pos[((size_t)b * T + t) * C + c] = cov;  // carried in pass 2
    }
    a.tot[((size_t)b * a.nch + ch) * C + c] = cov;
  }
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.cntp[(size_t)b * a.pnch + a.pq0 + ch] = red[0];
  // grad_T partial: sum over t < L of 2^(f_t + Ya[t,c'] + T2[c',c] + Yb[t,c])
  for (int pidx = threadIdx.x; pidx < C * C; pidx += blockDim.x) {
    const int cp = pidx / C, c = pidx % C;
    const R t2 = (R)(a.trans[pidx] * kLog2e);
    R acc0 = 0, acc1 = 0;
    int i = 0;
    for (; i + 1 < nt; i += 2) {
      acc0 += Mth<R>::ex2((R)sf[i] + sYa[(size_t)i * C + cp] + t2 + sYb[(size_t)i * C + c]);
      acc1 += Mth<R>::ex2((R)sf[i + 1] + sYa[(size_t)(i + 1) * C + cp] + t2 + sYb[(size_t)(i + 1) * C + c]);
    }
    if (i < nt) acc0 += Mth<R>::ex2((R)sf[i] + sYa[(size_t)i * C + cp] + t2 + sYb[(size_t)i * C + c]);
    a.gTp[((size_t)b * a.pnch + a.pq0 + ch) * C * C + pidx] = (double)(acc0 + acc1);
  }
}

template <typename R>
__host__ __device__ inline size_t post_pos_smem(int C, int CH) {
  return ((2 * (size_t)CH * C * sizeof(double) + 2 * (size_t)CH * C * sizeof(R) + 15) & ~(size_t)15) +
         (size_t)CH * sizeof(double);
}

// pass 2: add the carry of the preceding chunks to the local coverage, clip, zero padding
// chunk totals -> exclusive prefix over chunks, in place: one warp per (b, c); each lane
// sums a run of consecutive chunks, a warp scan of the run totals gives every run's start
// (fixed order, deterministic)
__global__ void __launch_bounds__(256) post_prefix_kernel(int B, int C, int nch, double* tot) {
  const int wid = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wid >= B * C) return;
  const int b = wid / C, c = wid % C;
  double* base = tot + (size_t)b * nch * C + c;
  const int per = (nch + 31) / 32, q0 = lane * per;
  double loc = 0.0;
  for (int i = 0; i < per; ++i)
    if (q0 + i < nch) loc += base[(size_t)(q0 + i) * C];
  double incl = loc;
  for (int off = 1; off < 32; off <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  double run = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) run = 0.0;
  for (int i = 0; i < per; ++i)
    if (q0 + i < nch) {
      const double v = base[(size_t)(q0 + i) * C];
      base[(size_t)(q0 + i) * C] = run;
      run += v;
    }
}

// pass 2: add the carry of the preceding chunks (tot holds exclusive prefixes after
// post_prefix_kernel) to the local coverage, clip, zero padding
__global__ void post_carry_kernel(const int64_t* lengths, int B, int T, int C, int CH, int nch, int w0, int w1,
                                  const double* tot, double* __restrict__ pos) {
  const int b = blockIdx.y, ch = blockIdx.x;
  const int L = (int)lengths[b];
  const int tend = min(w1, T);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const double carry = tot[((size_t)b * nch + ch) * C + c];
    const int t0 = w0 + ch * CH;
    for (int i = 0; i < CH; i += 4) {
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + i + j;
        v[j] = (i + j < CH && t < tend) ? pos[((size_t)b * T + t) * C + c] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + i + j;
        if (i + j < CH && t < tend) pos[((size_t)b * T + t) * C + c] = (t < L) ? fmin(fmax(v[j] + carry, 0.0), 1.0) : 0.0;
      }
    }
  }
}

// grad_B partial: CTA (b, source range, label group). A thread owns a window of kGBJ
// consecutive durations k0..k0+kGBJ-1 of one label and slides it along the sources: per
// source it loads ra[s] (a warp broadcast) and the one new rb[s+k0+kGBJ-1]; the other
// kGBJ-1 values are the previous source's, shifted in registers. ra[s] / rb[u] are staged
// per sub-chunk of kGBSub sources as (hi, lo) pairs in the working type (rb rows skewed by
// one pair per 16 so lanes kGBJ pairs apart hit distinct banks); terms are
// (ra_hi + rb_hi) + (ra_lo + rb_lo) + B2[k-1], one ex2 each.
constexpr int kGBSub = 128;
constexpr int kGBMicro = 1024;  // grad_B partial granularity (sources); a multiple of kGBSub
constexpr int kGBJ = 4;
constexpr int kGBW = 2;  // windows per thread (host keeps CG * ceil(K / kGBJ) <= kGBW * 512)
__host__ __device__ inline int gb_skew(int ui) { return ui + (ui >> 4); }
__host__ __device__ inline int gb_row(int K) { return gb_skew(kGBSub + K + kGBJ) + 1; }

template <typename R>
__global__ void __launch_bounds__(512) post_gradB_kernel(PostArgs<R> a) {
  using R2 = typename Vec2<R>::T;
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.z, cg = blockIdx.y, sb = blockIdx.x;
  const int C = a.C, T = a.T, K = a.K, CG = a.CGB;
  const int L = (int)a.lengths[b];
  const int c0 = cg * CG;
  const int Cn = min(CG, C - c0);
  const int nU = kGBSub + K + kGBJ;  // rb for u = s0+1 .. s0+nU (window over-read is -inf)
  const int rowU = gb_row(K);
  R2* sa = (R2*)sm;                      // [CG][kGBSub]
  R2* sbv = sa + (size_t)CG * kGBSub;    // [CG][rowU] (skewed)
  R* B2 = (R*)(sbv + (size_t)CG * rowU); // [CG][K]
  for (int i = threadIdx.x; i < Cn * K; i += blockDim.x) {
    const int cl = i / K, k = i % K;
    B2[i] = (R)(a.dur[(size_t)k * C + c0 + cl] * kLog2e);
  }
  const int nkb = (K + kGBJ - 1) / kGBJ;
  const int nwin = Cn * nkb;
  double acc[kGBW][kGBJ];
#pragma unroll
  for (int w = 0; w < kGBW; ++w)
#pragma unroll
    for (int j = 0; j < kGBJ; ++j) acc[w][j] = 0.0;
  const int sbeg = a.w0 + sb * a.SCB;
  const int W = a.w1 - a.w0;
  const int nmic = a.SCB / kGBMicro;
  __syncthreads();
  // partials per micro-chunk of kGBMicro sources (a fixed grid, independent of the batch size
  // and of how CTAs are laid out: per-sequence sums are bit-identical under batch sharding)
  for (int mi = 0; mi < nmic; ++mi) {
  const int slot_m = sb * nmic + mi;
  if (slot_m >= a.nchB) break;
  const int send = min(min(sbeg + (mi + 1) * kGBMicro, a.w1), L);  // sources s < L in [w0, w1)
#pragma unroll
  for (int w = 0; w < kGBW; ++w)
#pragma unroll
    for (int j = 0; j < kGBJ; ++j) acc[w][j] = 0.0;
  for (int s0 = sbeg + mi * kGBMicro; s0 < send; s0 += kGBSub) {
    __syncthreads();
    const int ns = min(kGBSub, send - s0);
    for (int i = threadIdx.x; i < Cn * kGBSub; i += blockDim.x) {
      const int cl = i / kGBSub, si = i % kGBSub, s = s0 + si, c = c0 + cl;
      R2 v;
      v.x = Mth<R>::ninf();
      v.y = 0;
      if (si < ns) {
        const double ra = a.RA[((size_t)b * C + c) * a.NR + (s - a.t_lo)] +
                          (a.corr ? a.corr[(size_t)b * W + s - a.w0] : 0.0);
        split2(ra, v.x, v.y);
      }
      sa[(size_t)cl * kGBSub + si] = v;
    }
    for (int i = threadIdx.x; i < Cn * nU; i += blockDim.x) {
      const int cl = i / nU, ui = i % nU, u = s0 + 1 + ui, c = c0 + cl;
      R2 v;
      v.x = Mth<R>::ninf();
      v.y = 0;
      if (u <= L && u < a.w1 + K && ui < kGBSub + K)  // (beta rows of a window end at w1 + K - 1)
        split2(a.RB[((size_t)b * C + c) * a.NR + (u - a.t_lo)], v.x, v.y);
      sbv[(size_t)cl * rowU + gb_skew(ui)] = v;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kGBW; ++w) {
      const int idx = threadIdx.x + w * blockDim.x;
      if (idx < nwin) {
        const int cl = idx / nkb, k0 = (idx % nkb) * kGBJ + 1;
        const R2* A = sa + (size_t)cl * kGBSub;
        const R2* Bv = sbv + (size_t)cl * rowU;
        const int ub = k0 - 1;  // u = s + k -> ui = si + k - 1
        R bk[kGBJ];
        R2 wv[kGBJ];
#pragma unroll
        for (int j = 0; j < kGBJ; ++j) {
          bk[j] = (k0 + j <= K) ? B2[(size_t)cl * K + k0 - 1 + j] : Mth<R>::ninf();
          if (j < kGBJ - 1) wv[j] = Bv[gb_skew(ub + j)];
        }
        R sj[kGBJ];
#pragma unroll
        for (int j = 0; j < kGBJ; ++j) sj[j] = 0;
#pragma unroll 4
        for (int si = 0; si < ns; ++si) {
          wv[kGBJ - 1] = Bv[gb_skew(si + ub + kGBJ - 1)];
          const R2 x = A[si];
#pragma unroll
          for (int j = 0; j < kGBJ; ++j) sj[j] += Mth<R>::ex2(((x.x + wv[j].x) + (x.y + wv[j].y)) + bk[j]);
#pragma unroll
          for (int j = 0; j < kGBJ - 1; ++j) wv[j] = wv[j + 1];
        }
#pragma unroll
        for (int j = 0; j < kGBJ; ++j) acc[w][j] += (double)sj[j];
      }
    }
  }
#pragma unroll
  for (int w = 0; w < kGBW; ++w) {
    const int idx = threadIdx.x + w * blockDim.x;
    if (idx < nwin) {
      const int cl = idx / nkb, k0 = (idx % nkb) * kGBJ;
#pragma unroll
      for (int j = 0; j < kGBJ; ++j)
        if (k0 + j < K) a.gBp[(((size_t)b * a.pnchB + a.pm0 + slot_m) * K + k0 + j) * C + c0 + cl] = acc[w][j];
    }
  }
  }  // micro-chunks
}

// grad_B partial in exp space (fp32 working type): CTA (b, source range, label group), one warp
// per (label, pass of 128 durations). Per block of 32 sources the source values are detrended by
// the block's slope lam (alpha grows at ~lam per position, the beta side falls at the same rate):
//   d_i = (ra[s0+i] - r0) - lam i,     e_v = (rb[s0+kb+v] + r0) + lam v     (r0 = the block's first ra)
//   term(s0+i, k) = 2^(d_i + e_v - lam (k - kb) + B[k-1]),  v = i + k - kb
// so with x_i = 2^(d_i - Gd), y_v = 2^(e_v - Ge) a block contributes
//   2^(Gd + Ge - lam (k - kb) + B[k-1]) * sum_i x_i y_{i+k-kb}
// -- 32 FMA per term group of a lane (4 durations x 32 sources from one 35-value y window)
// instead of one ex2 per term. Blocks whose detrended range exceeds kGBRange take the exact
// per-term path. x and y are lifted by 2^60 each, so factors down to 2^-120 of their block
// maximum stay normal fp32 and their products (<= 2^125 summed) neither overflow nor flush.
constexpr int kGBD = 8;                 // durations per lane
constexpr int kGBPass = 32 * kGBD;      // durations per warp item
constexpr float kGBRange = 180.f;
constexpr float kGBLift = 60.f;  // x and y carry 2^60 each: products of +-126-wide factors stay normal
__host__ __device__ inline int gbb_npass(int K) { return (K + kGBPass - 1) / kGBPass; }
__host__ __device__ inline int gbb_nU(int K) { return kGBSub + gbb_npass(K) * kGBPass + 32; }
__host__ __device__ inline int gbb_row(int K) { return gb_skew(gbb_nU(K)) + 1; }
constexpr int kGBNV = kGBPass + 32;     // target window per item (v < kGBPass + 31, padded)
constexpr int kGBBWarp = 32 + 32 + 2 * kGBNV;  // per-warp scratch: x, d, y window, e (floats)

__host__ __device__ inline size_t post_gradB_blk_smem(int K, int CG) {
  return (size_t)CG * kGBSub * 2 * sizeof(float) + (size_t)CG * gbb_row(K) * 2 * sizeof(float) +
         (size_t)CG * gbb_npass(K) * kGBPass * sizeof(float) + (size_t)16 * kGBBWarp * sizeof(float) + 64;
}

#ifndef SCRF_GBB_MINB
#define SCRF_GBB_MINB 1
#endif
__global__ void __launch_bounds__(512, SCRF_GBB_MINB) post_gradB_blk_kernel(PostArgs<float> a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.z, cg = blockIdx.y, sb = blockIdx.x;
  const int C = a.C, T = a.T, K = a.K, CG = a.CGB;
  const int L = (int)a.lengths[b];
  const int c0 = cg * CG;
  const int Cn = min(CG, C - c0);
  const int npass = gbb_npass(K);
  const int nU = gbb_nU(K);
  const int rowU = gbb_row(K);
  const int KP = npass * kGBPass;
  float2* sa = (float2*)sm;                          // [CG][kGBSub]
  float2* sbv = sa + (size_t)CG * kGBSub;            // [CG][rowU] (skewed)
  float* B2 = (float*)(sbv + (size_t)CG * rowU);     // [CG][KP], -inf past K
  float* wsc = (float*)(((uintptr_t)(B2 + (size_t)CG * KP) + 15) & ~(uintptr_t)15);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xs = wsc + (size_t)warp * kGBBWarp;  // [32]
  float* ds = xs + 32;                        // [32]
  float* yw = ds + 32;                        // [kGBNV] (16-byte aligned)
  float* es = yw + kGBNV;                     // [kGBNV]
  const int W = a.w1 - a.w0;
  for (int i = threadIdx.x; i < Cn * KP; i += blockDim.x) {
    const int cl = i / KP, k = i % KP;
    B2[i] = k < K ? (float)(a.dur[(size_t)k * C + c0 + cl] * kLog2e) : -CUDART_INF_F;
  }
  const int nitems = Cn * npass;
  double acc[2][kGBD];
#pragma unroll
  for (int w = 0; w < 2; ++w)
#pragma unroll
    for (int j = 0; j < kGBD; ++j) acc[w][j] = 0.0;
  const int sbeg = a.w0 + sb * a.SCB;
  const int nmic = a.SCB / kGBMicro;
  __syncthreads();
  for (int mi = 0; mi < nmic; ++mi) {  // micro-chunks (see post_gradB_kernel)
  const int slot_m = sb * nmic + mi;
  if (slot_m >= a.nchB) break;
  const int send = min(min(sbeg + (mi + 1) * kGBMicro, a.w1), L);
#pragma unroll
  for (int w = 0; w < 2; ++w)
#pragma unroll
    for (int j = 0; j < kGBD; ++j) acc[w][j] = 0.0;
  for (int s0 = sbeg + mi * kGBMicro; s0 < send; s0 += kGBSub) {
    __syncthreads();
    const int ns = min(kGBSub, send - s0);
    static_assert((kGBSub & (kGBSub - 1)) == 0, "kGBSub: power of two");
    for (int i = threadIdx.x; i < Cn * kGBSub; i += blockDim.x) {
      const int cl = i / kGBSub, si = i & (kGBSub - 1), s = s0 + si, c = c0 + cl;
      float2 v = make_float2(-CUDART_INF_F, 0.f);
      if (si < ns) {
        const double ra = a.RA[((size_t)b * C + c) * a.NR + (s - a.t_lo)] +
                          (a.corr ? a.corr[(size_t)b * W + s - a.w0] : 0.0);
        split2(ra, v.x, v.y);
      }
      sa[(size_t)cl * kGBSub + si] = v;
    }
    // targets u = s0 + 1 + ui of this sub-chunk: rb for ui < kGBSub + K - 1, -inf beyond (window
    // over-read). Consecutive sub-chunks of a CTA overlap in all but kGBSub of them: after the
    // first, the kept ones move down by kGBSub in place and only the new kGBSub are loaded.
    auto tgt = [&](int cl, int ui) -> float2 {
      const int u = s0 + 1 + ui;
      float2 v = make_float2(-CUDART_INF_F, 0.f);
      if (u <= L && u < a.w1 + K && ui < kGBSub + K - 1)  // (beta rows of a window end at w1 + K - 1)
        split2(a.RB[((size_t)b * C + c0 + cl) * a.NR + (u - a.t_lo)], v.x, v.y);
      return v;
    };
    if (s0 == sbeg) {
      for (int i = threadIdx.x; i < Cn * nU; i += blockDim.x) {
        const int cl = i / nU, ui = i % nU;
        sbv[(size_t)cl * rowU + gb_skew(ui)] = tgt(cl, ui);
      }
    } else {
      const int nk = K - 1;  // kept per label: ui in [0, K - 1) <- [kGBSub, kGBSub + K - 1)
      constexpr int kR = 8;
      for (int base = 0; base < Cn * nk; base += kR * 512) {
        float2 keep[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int i = base + r * 512 + (int)threadIdx.x;
          if (i < Cn * nk) {
            const int cl = i / nk, ui = i - cl * nk;
            keep[r] = sbv[(size_t)cl * rowU + gb_skew(ui + kGBSub)];
          }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int i = base + r * 512 + (int)threadIdx.x;
          if (i < Cn * nk) {
            const int cl = i / nk, ui = i - cl * nk;
            sbv[(size_t)cl * rowU + gb_skew(ui)] = keep[r];
          }
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < Cn * kGBSub; i += blockDim.x) {
        const int cl = i / kGBSub, ui = nk + (i & (kGBSub - 1));
        sbv[(size_t)cl * rowU + gb_skew(ui)] = tgt(cl, ui);
      }
    }
    __syncthreads();
#pragma unroll
    for (int slot = 0; slot < 2; ++slot) {  // static slot index: acc stays in registers
      const int it = warp + 16 * slot;
      if (it >= nitems) break;
      const int cl = it / npass, pass = it % npass;
      const int kb = pass * kGBPass + 1;  // durations kb .. kb + kGBPass - 1 (lane owns kb + kGBD lane + j)
      const float2* A = sa + (size_t)cl * kGBSub;
      const float2* Bv = sbv + (size_t)cl * rowU;
      const float* b2 = B2 + (size_t)cl * KP;
      float bk[kGBD];
#pragma unroll
      for (int j = 0; j < kGBD; ++j) bk[j] = b2[kb - 1 + kGBD * lane + j];
      for (int jb = 0; jb * 32 < ns; ++jb) {
        // sources of the block, detrended
        const float2 r = A[jb * 32 + lane];
        const bool fin = r.x != -CUDART_INF_F;
        const unsigned fm = __ballot_sync(0xffffffffu, fin);
        if (!fm) continue;
        const int f0 = __ffs(fm) - 1;
        const float r0x = __shfl_sync(0xffffffffu, r.x, f0), r0y = __shfl_sync(0xffffffffu, r.y, f0);
        // targets u = s0 + 32 jb + kb + v, v in [0, kGBPass + 31): e'_v = rb + r0
        float ev[kGBNV / 32];
        int vlo = 1 << 30, vhi = -1;
        float elo = 0.f, ehi = 0.f;
#pragma unroll
        for (int m = 0; m < kGBNV / 32; ++m) {
          const int v = lane + 32 * m;
          ev[m] = -CUDART_INF_F;
          if (v < kGBPass + 31) {
            const float2 q = Bv[gb_skew(jb * 32 + kb - 1 + v)];
            if (q.x != -CUDART_INF_F) {
              ev[m] = (q.x + r0x) + (q.y + r0y);
              if (v < vlo) {
                vlo = v;
                elo = ev[m];
              }
              vhi = v;
              ehi = ev[m];
            }
          }
        }
        // slope of the window (beta falls as alpha grows): detrend both sides with it
        for (int o = 16; o > 0; o >>= 1) {
          const int vl2 = __shfl_xor_sync(0xffffffffu, vlo, o), vh2 = __shfl_xor_sync(0xffffffffu, vhi, o);
          const float el2 = __shfl_xor_sync(0xffffffffu, elo, o), eh2 = __shfl_xor_sync(0xffffffffu, ehi, o);
          if (vl2 < vlo) {
            vlo = vl2;
            elo = el2;
          }
          if (vh2 > vhi) {
            vhi = vh2;
            ehi = eh2;
          }
        }
        if (vhi < 0) continue;  // every target of this pass is past L
        const float lam = vhi > vlo ? -(ehi - elo) / (float)(vhi - vlo) : 0.f;
        const float d = fin ? ((r.x - r0x) + (r.y - r0y)) - lam * (float)lane : -CUDART_INF_F;
        float gd = d, dmin = fin ? d : CUDART_INF_F;
        for (int o = 16; o > 0; o >>= 1) {
          gd = fmaxf(gd, __shfl_xor_sync(0xffffffffu, gd, o));
          dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        }
        xs[lane] = fin ? Mth<float>::ex2((d - gd) + kGBLift) : 0.f;
        ds[lane] = d;
        // detrended targets e_v = e'_v + lam v
        float ge = -CUDART_INF_F, emin = CUDART_INF_F;
#pragma unroll
        for (int m = 0; m < kGBNV / 32; ++m) {
          if (ev[m] != -CUDART_INF_F) {
            ev[m] += lam * (float)(lane + 32 * m);
            emin = fminf(emin, ev[m]);
          }
          ge = fmaxf(ge, ev[m]);
        }
        for (int o = 16; o > 0; o >>= 1) {
          ge = fmaxf(ge, __shfl_xor_sync(0xffffffffu, ge, o));
          emin = fminf(emin, __shfl_xor_sync(0xffffffffu, emin, o));
        }
        if (ge == -CUDART_INF_F) continue;  // every target of this pass is past L
#pragma unroll
        for (int m = 0; m < kGBNV / 32; ++m) {
          const int v = lane + 32 * m;
          yw[v] = ev[m] != -CUDART_INF_F ? Mth<float>::ex2((ev[m] - ge) + kGBLift) : 0.f;
          es[v] = ev[m];
        }
        __syncwarp();
        const bool exact = (gd - dmin > a.gb_range) || (ge - emin > a.gb_range);
        float out[kGBD];
#pragma unroll
        for (int j = 0; j < kGBD; ++j) out[j] = 0.f;
        if (!exact) {
          // lane: durations kb + kGBD lane + j, sum_i x_i y_{i + kGBD lane + j}
          float y[32 + kGBD];
          const float4* y4 = (const float4*)(yw + kGBD * lane);
#pragma unroll
          for (int q = 0; q < (32 + kGBD) / 4; ++q) {
            const float4 t4 = y4[q];
            y[4 * q] = t4.x;
            y[4 * q + 1] = t4.y;
            y[4 * q + 2] = t4.z;
            y[4 * q + 3] = t4.w;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float xi = xs[i];
#pragma unroll
            for (int j = 0; j < kGBD; ++j) out[j] = fmaf(xi, y[i + j], out[j]);
          }
#pragma unroll
          for (int j = 0; j < kGBD; ++j) {
            // the 2^-120 of the lift is applied in fp64 (the fp32 product could flush)
            const float E = (gd + ge) - lam * (float)(kGBD * lane + j) + bk[j];
            if (out[j] > 0.f && E != -CUDART_INF_F)
              acc[slot][j] += (double)out[j] * (double)Mth<float>::ex2(E) * 0x1p-120;
          }
        } else {
#pragma unroll 4
          for (int i = 0; i < 32; ++i) {
            const float di = ds[i];
            if (di == -CUDART_INF_F) continue;
#pragma unroll
            for (int j = 0; j < kGBD; ++j) {
              const float e = es[i + kGBD * lane + j];
              if (e != -CUDART_INF_F) out[j] += Mth<float>::ex2((di + e) - lam * (float)(kGBD * lane + j) + bk[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < kGBD; ++j) acc[slot][j] += (double)out[j];
        }
        __syncwarp();
      }
    }
  }
#pragma unroll
  for (int slot = 0; slot < 2; ++slot) {
    const int it = warp + 16 * slot;
    if (it >= nitems) break;
    const int cl = it / npass, pass = it % npass;
#pragma unroll
    for (int j = 0; j < kGBD; ++j) {
      const int k = pass * kGBPass + kGBD * lane + j;  // duration k + 1
      if (k < K) a.gBp[(((size_t)b * a.pnchB + a.pm0 + slot_m) * K + k) * C + c0 + cl] = acc[slot][j];
    }
  }
  }  // micro-chunks
}

template <typename R>
__host__ __device__ inline size_t post_gradB_smem(int K, int CG) {
  return (size_t)CG * kGBSub * 2 * sizeof(R) + (size_t)CG * gb_row(K) * 2 * sizeof(R) + (size_t)CG * K * sizeof(R) + 16;
}

// fixed-order reductions: per-sequence partials (unscaled) and batch totals (upstream-weighted)
__global__ void post_reduce_kernel(int B, int n, int nparts, const double* parts, const double* upstream,
                                   double* per_seq, double* total) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double tot = 0.0;
  for (int b = 0; b < B; ++b) {
    double s = 0.0;
    for (int q = 0; q < nparts; ++q) s += parts[((size_t)b * nparts + q) * n + i];
    if (per_seq) per_seq[(size_t)b * n + i] = s;
    tot += (upstream ? upstream[b] : 1.0) * s;
  }
  if (total) total[i] = tot;
}

// Same sums, parallel over the parts: block (32 outputs x 8 warps); warp w sums parts
// w, w+8, ... in order and the 8 warp sums are added in warp order (a fixed order, so the
// result is deterministic and independent of scheduling).
__global__ void __launch_bounds__(256) post_reduce2_kernel(int B, int n, int nparts, const double* parts,
                                                           const double* upstream, double* per_seq, double* total) {
  __shared__ double ws[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const bool ok = i < n;
  double tot = 0.0;
  for (int b = 0; b < B; ++b) {
    double s0 = 0.0, s1 = 0.0;
    const double* pb = parts + (size_t)b * nparts * n + i;
    int q = w;
    for (; q + 8 < nparts; q += 16) {
      if (ok) {
        s0 += pb[(size_t)q * n];
        s1 += pb[(size_t)(q + 8) * n];
      }
    }
    if (q < nparts && ok) s0 += pb[(size_t)q * n];
    ws[w][lane] = s0 + s1;
    __syncthreads();
    if (w == 0) {
      double sb = 0.0;
#pragma unroll
      for (int v = 0; v < 8; ++v) sb += ws[v][lane];
      if (ok && per_seq) per_seq[(size_t)b * n + i] = sb;
      tot = __dadd_rn(tot, __dmul_rn(upstream ? upstream[b] : 1.0, sb));
    }
    __syncthreads();
  }
  if (w == 0 && ok && total) total[i] = tot;
}

__global__ void post_count_kernel(int B, int nch, const double* cntp, double* count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int q = 0; q < nch; ++q) s += cntp[(size_t)b * nch + q];
  count[b] = s;
}

}  // namespace scrf
