// Exact max-plus Viterbi on B200 (sm_100a): bit-identical to the reference's
// `streaming_viterbi` (pkg/src/streamcrf/streaming.py:411-470).
//
// The reference scores every candidate as cand = fl(fl(prev[t-k,c'] + T[c',c]) + h[t,k,c])
// with h = fl(fl(fl(S[t,c] - S[t-k,c]) + B[k-1,c]) (+ Ps[t-k,c]) (+ Pe[t-1,c])), and takes
// the first maximum of the reversed-duration flattening (largest k, then smallest c').
// fp64 addition is correctly rounded and monotone, so with
//   gmax[s,c] = max_c' fl(prev[s,c'] + T[c',c])         (argmax: smallest c')
// the reference's best value at (t, k) is exactly fl(gmax[t-k,c] + h). That turns the
// K*C^2 scan into K*C + C^2 fp64 adds per position. The only subtlety is a c' smaller
// than the argmax whose fl(prev + T) is strictly smaller but rounds to the same value
// after "+ h"; gsec[s,c] (the best value over c' < argmax) detects that case exactly and
// a rare re-scan over the (global) message history picks the reference's c'.
//
// Layout mirrors the forward kernel: one cluster per sequence, CTA r owns a label slice.
#include <stdint.h>

#include "scrf_common.cuh"

namespace scrf {

struct VitArgs {
  const double* S;
  const int64_t* lengths;
  const double* trans;
  const double* dur;
  const double* ps;
  const double* pe;
  int B, T, K, C;
  Geometry geo;
  double* dvring;   // [B][K][C] message history (for the tie re-scan)
  int32_t* bp;      // [B][T+1][C] (k << 16) | c'
  double* score;    // [B]
  int32_t* seg_start;
  int32_t* seg_end;
  int32_t* seg_label;
  int32_t* seg_count;
};

// per-position inputs (raw fp64 S[t], Ps[t], Pe[t-1] of own labels) staged in chunks of P
__host__ __device__ inline int vit_chunk(const Geometry& g) {
  int P = 64;
  while (P > 2 && P * g.Cgm > g.NT * 2) P >>= 1;
  return P;
}

__host__ __device__ inline size_t vit_smem_bytes(int K, int C, const Geometry& g, bool has_ps) {
  auto r16 = [](size_t n) { return (n + 15) & ~(size_t)15; };
  const size_t KC = (size_t)K * g.Cgm;
  size_t n = 0;
  n += 3 * r16(KC * sizeof(double));  // gmax, gsec, S ring
  n += has_ps ? r16(KC * sizeof(double)) : 0;
  n += r16(KC * sizeof(double));      // duration bias
  n += r16(KC * sizeof(int32_t));     // argmax
  n += r16((size_t)C * g.Cgm * sizeof(double));  // T columns
  n += r16(2 * (size_t)C * sizeof(double)) + r16(16);  // exchange + mbarriers
  n += 3 * r16(2 * (size_t)vit_chunk(g) * g.Cgm * sizeof(double));  // staged S, Ps, Pe rows
  return n;
}

__device__ __forceinline__ void vit_merge(double& v, int& k, double v2, int k2) {
  // larger value wins; on equal values the larger duration wins (reference tie rule)
  if (v2 > v || (v2 == v && k2 > k)) {
    v = v2;
    k = k2;
  }
}

__global__ void __launch_bounds__(1024) vit_kernel(VitArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geometry& g = a.geo;
  const int K = a.K, C = a.C, Cgm = g.Cgm;
  unsigned char* p = smem_raw;
  auto take = [&](size_t bytes) {
    unsigned char* r = p;
    p += (bytes + 15) & ~(size_t)15;
    return r;
  };
  const size_t KC = (size_t)K * Cgm;
  double* gmax = (double*)take(KC * 8);
  double* gsec = (double*)take(KC * 8);
  double* sring = (double*)take(KC * 8);
  double* psring = a.ps ? (double*)take(KC * 8) : nullptr;
  double* Bd = (double*)take(KC * 8);
  int32_t* garg = (int32_t*)take(KC * 4);
  double* Tcol = (double*)take((size_t)C * Cgm * 8);
  double* xall = (double*)take(2 * (size_t)C * 8);
  uint64_t* xbar = (uint64_t*)take(16);
  const int P = vit_chunk(g);
  double* stS = (double*)take(2 * (size_t)P * Cgm * 8);
  double* stPs = (double*)take(2 * (size_t)P * Cgm * 8);
  double* stPe = (double*)take(2 * (size_t)P * Cgm * 8);

  const int rank = (int)cl.block_rank();
  const int b = blockIdx.x / g.G;
  const int c0 = label_lo(rank, C, g.G);
  const int Cg = label_lo(rank + 1, C, g.G) - c0;
  const int L = (int)a.lengths[b];
  const int tid = threadIdx.x;
  const int cl_ = tid / g.TPL, j = tid % g.TPL;
  const bool active = cl_ < Cg;
  const int cls = active ? cl_ : 0;
  const bool gl = j < g.GW;
  const int c = c0 + cls;
  const double* S = a.S + (size_t)b * (a.T + 1) * C;
  const double* ps = a.ps ? a.ps + (size_t)b * a.T * C : nullptr;
  const double* pe = a.pe ? a.pe + (size_t)b * a.T * C : nullptr;
  // this CTA's private copy of the full message history (for the tie re-scan)
  double* dvr = a.dvring + ((size_t)b * g.G + rank) * K * C;
  int32_t* bp = a.bp + (size_t)b * (a.T + 1) * C;

  // chunk q holds positions [q*P, (q+1)*P); registers carry chunk q+2 while q is consumed
  double rS[2], rPs[2], rPe[2];
  auto vload = [&](int q) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + r * g.NT;
      rS[r] = rPs[r] = rPe[r] = 0.0;
      if (e < P * Cg) {
        const int i = e / Cg, cc = e % Cg, t = q * P + i;
        if (t <= a.T) {
          rS[r] = __ldg(S + (size_t)t * C + c0 + cc);
          rPs[r] = (ps && t < a.T) ? __ldg(ps + (size_t)t * C + c0 + cc) : 0.0;
          rPe[r] = (pe && t >= 1) ? __ldg(pe + (size_t)(t - 1) * C + c0 + cc) : 0.0;
        }
      }
    }
  };
  auto vstore = [&](int q) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + r * g.NT;
      if (e < P * Cg) {
        const int i = e / Cg, cc = e % Cg;
        const size_t k = ((size_t)(q & 1) * P + i) * Cgm + cc;
        stS[k] = rS[r];
        stPs[k] = rPs[r];
        stPe[k] = rPe[r];
      }
    }
  };
  auto vidx = [&](int t, int cc) { return ((size_t)((t / P) & 1) * P + (t % P)) * Cgm + cc; };
  vload(0);
  vstore(0);
  vload(1);
  vstore(1);
  vload(2);

  for (int i = tid; i < (int)KC; i += g.NT) {
    int k = i / Cgm, cc = i % Cgm;
    Bd[i] = (cc < Cg) ? a.dur[(size_t)k * C + c0 + cc] : 0.0;
  }
  for (int i = tid; i < C * Cgm; i += g.NT) {
    int cp = i / Cgm, cc = i % Cgm;
    Tcol[i] = (cc < Cg) ? a.trans[(size_t)cp * C + c0 + cc] : 0.0;
  }
  __syncthreads();

  // gamma step for position s from exchanged messages xv[0..C)
  auto gamma_step = [&](const double* xv, int s) {
    if (!gl) return;
    double best = -CUDART_INF;
    int arg = 0x7fffffff;
    for (int cp = j; cp < C; cp += g.GW) {
      double v = __dadd_rn(xv[cp], Tcol[(size_t)cp * Cgm + cls]);
      if (v > best || (v == best && cp < arg)) {
        best = v;
        arg = cp;
      }
    }
    for (int off = g.GW >> 1; off > 0; off >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, off, g.GW);
      int oa = __shfl_xor_sync(0xffffffffu, arg, off, g.GW);
      if (ob > best || (ob == best && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    double sec = -CUDART_INF;
    for (int cp = j; cp < C && cp < arg; cp += g.GW) sec = fmax(sec, __dadd_rn(xv[cp], Tcol[(size_t)cp * Cgm + cls]));
    sec = group_max(sec, g.GW);
    if (active && j == 0) {
      const int slot = s % K;
      gmax[slot * Cgm + cls] = best;
      gsec[slot * Cgm + cls] = sec;
      garg[slot * Cgm + cls] = arg;
      sring[slot * Cgm + cls] = stS[vidx(s, cls)];
      if (psring) psring[slot * Cgm + cls] = stPs[vidx(s, cls)];
    }
  };

  Xchg<double> xv;
  xv.buf = xall;
  xv.bar = xbar;
  xv.C = C;
  xv.init(tid);
  // position 0: every label starts from the virtual source with message 0
  for (int i = tid; i < C; i += g.NT) {
    xall[i] = 0.0;
    dvr[i] = 0.0;
  }
  __syncthreads();
  gamma_step(xall, 0);
  __syncthreads();
  cl.sync();

  for (int t = 1; t <= L; ++t) {
    const int par = t & 1;
    const int kmax = min(K, t);
    double best = -CUDART_INF;
    int bk = 0;
    if (t % P == 0) {  // entering chunk q = t / P: park chunk q+1, prefetch chunk q+2
      vstore(t / P + 1);
      vload(t / P + 2);
      __syncthreads();
    }
    if (tid == 0) xv.arm(par);
    const double St = stS[vidx(t, cls)];
    const double Pet = stPe[vidx(t, cls)];
    if (active) {
      for (int k = 1 + j; k <= kmax; k += g.TPL) {
        const int slot = (t - k) % K;
        double h = __dadd_rn(__dadd_rn(St, -sring[slot * Cgm + cls]), Bd[(k - 1) * Cgm + cls]);
        if (psring) h = __dadd_rn(h, psring[slot * Cgm + cls]);
        if (pe) h = __dadd_rn(h, Pet);
        double cand = __dadd_rn(gmax[slot * Cgm + cls], h);
        vit_merge(best, bk, cand, k);
      }
    }
    // reduce within lane groups, then across warps of the label through xall scratch
    for (int off = g.GW >> 1; off > 0; off >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, best, off, g.GW);
      int okk = __shfl_xor_sync(0xffffffffu, bk, off, g.GW);
      vit_merge(best, bk, ov, okk);
    }
    if (g.WPL > 1) {
      __shared__ double wv[32];
      __shared__ int wk[32];
      const int warp = tid >> 5, lane = tid & 31;
      if (lane == 0) {
        wv[warp] = best;
        wk[warp] = bk;
      }
      __syncthreads();
      if (gl) {
        const int w0 = cl_ * g.WPL;
        for (int w = 0; w < g.WPL; ++w) vit_merge(best, bk, wv[w0 + w], wk[w0 + w]);
      }
      __syncthreads();
    }
    if (active && j == 0) {
      const int s = t - bk;
      const int slot = s % K;
      double h = __dadd_rn(__dadd_rn(St, -sring[slot * Cgm + cls]), Bd[(bk - 1) * Cgm + cls]);
      if (psring) h = __dadd_rn(h, psring[slot * Cgm + cls]);
      if (pe) h = __dadd_rn(h, Pet);
      int src = garg[slot * Cgm + cls];
      const double sec = gsec[slot * Cgm + cls];
      if (src > 0 && sec != -CUDART_INF && __dadd_rn(sec, h) == best) {
        // rare: an earlier source ties after rounding; re-scan in reference order
        const double* prev = (s == 0) ? nullptr : dvr + (size_t)slot * C;
        for (int cp = 0; cp < src; ++cp) {
          const double pv = prev ? prev[cp] : 0.0;
          if (__dadd_rn(__dadd_rn(pv, a.trans[(size_t)cp * C + c]), h) == best) {
            src = cp;
            break;
          }
        }
      }
      bp[(size_t)t * C + c] = (bk << 16) | src;
      xv.send(par, c, best, 0, 1, g.G);
    }
    const double* xin = xv.wait(par);
    for (int i = tid; i < C; i += g.NT) dvr[(size_t)(t % K) * C + i] = xin[i];
    gamma_step(xin, t);
    __syncthreads();
  }
  __threadfence();
  cl.sync();
  if (rank == 0 && tid == 0) {
    const double* fin = xall + (L & 1) * C;
    // final label: smallest argmax of the messages at L (streaming.py:458-460)
    int cbest = 0;
    for (int cc = 1; cc < C; ++cc)
      if (fin[cc] > fin[cbest]) cbest = cc;
    if (L == 0) cbest = 0;
    a.score[b] = fin[cbest];
    int32_t* st = a.seg_start + (size_t)b * a.T;
    int32_t* en = a.seg_end + (size_t)b * a.T;
    int32_t* lb = a.seg_label + (size_t)b * a.T;
    int n = 0, t = L, cc = cbest;
    while (t > 0) {
      const int32_t v = bp[(size_t)t * C + cc];
      const int k = v >> 16;
      st[n] = t - k;
      en[n] = t;
      lb[n] = cc;
      ++n;
      cc = v & 0xffff;
      t -= k;
    }
    for (int i = 0; i < n / 2; ++i) {
      int32_t x0 = st[i], x1 = en[i], x2 = lb[i];
      st[i] = st[n - 1 - i];
      en[i] = en[n - 1 - i];
      lb[i] = lb[n - 1 - i];
      st[n - 1 - i] = x0;
      en[n - 1 - i] = x1;
      lb[n - 1 - i] = x2;
    }
    a.seg_count[b] = n;
  }
}

}  // namespace scrf
