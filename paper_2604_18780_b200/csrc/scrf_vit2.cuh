// Exact max-plus Viterbi, head + tails cluster (sm_100a); bit-identical to the reference's
// `streaming_viterbi` (pkg/src/streamcrf/streaming.py:411-470).
//
// Same arithmetic as scrf_viterbi.cu (see its header): the best value of duration k for target
// t is fl(gmax[t-k,c] + h(t,k,c)) with h = fl(fl(fl(S[t,c] - S[t-k,c]) + B[k-1,c]) (+ Ps[t-k,c])
// (+ Pe[t-1,c])), ties go to the largest k; gmax[s,c] = max_c' fl(v[s,c'] + T[c',c]) with the
// smallest c' on ties, and gsec (best over c' < argmax) flags the rare rounding tie that needs a
// re-scan of the message history in the reference's order.
//
// One cluster per sequence:
//  * head CTA (rank 0), lane = label (NCW warps): per position t it takes the max over
//    durations 1..kn from a ring of the last R sources, merges the tails' best over kn+1..K,
//    resolves the source label (tie check / re-scan), writes the packed backpointer and the
//    message, computes gamma (gmax, argmax, gsec) of position t and pushes it to the tails;
//  * tail CTAs (ranks 1..G-1, label slices, TW warps per label taking alternate targets):
//    the exact max over durations kn+1..K of each target, from a ring of K sources per label,
//    returned with the tie-check verdict. Hand-offs use st.async + mbarrier complete_tx in both
//    directions (no cluster barriers in the loop).
#pragma once

#include <cstdio>

#include "scrf_common.cuh"

namespace scrf {

constexpr int kVSrc = 32;  // source mbarrier slots per tail

struct V2Geo {
  int G;     // CTAs per cluster (1 = head only)
  int NCW;   // head warps (32 labels each)
  int R;     // head ring positions (power of two); near durations kn = R / 2 (or K when G == 1)
  int kn;    // durations handled by the head
  int CgMax; // max labels per tail
  int TW;    // tail warps per label
  int KR;    // tail source ring positions (>= K + 8; any length, indexed incrementally)
  int NT;    // threads per CTA
};

struct V2Args {
  const double* S;
  const int64_t* lengths;
  const double* trans;
  const double* dur;
  const double* ps;
  const double* pe;
  int B, T, K, C;
  V2Geo geo;
  double* hist;   // [B][T+1][C] messages (tie re-scans)
  int32_t* bp;    // [B][T+1][C] (k << 16) | c'
  double* score;  // [B]
  int32_t* seg_start;
  int32_t* seg_end;
  int32_t* seg_label;
  int32_t* seg_count;
};

__host__ __device__ inline int v2_tail_lo(int rank, int C, int G) { return (int)(((long long)(rank - 1) * C) / (G - 1)); }
__host__ __device__ inline size_t v2_a16(size_t x) { return (x + 15) & ~(size_t)15; }

struct V2Head {
  size_t hg, hs, hP, hS, ha, Tm, vsm, part, tbar, gpb, gpa, total;
};
// warps sharing the head's gamma (every warp of the head CTA) and whether they are more than
// the label warps
__host__ __device__ inline int v2_gamma_warps(const V2Geo& g) { return g.NT / 32; }
// (worth its two extra barriers per position only when each label scans many c': measured
// c5 (C = 128) 188.8 -> 132.2 ms, c4 (C = 24) 192.4 -> 198.8 ms, c3 (C = 39) unchanged)
__host__ __device__ inline bool v2_par_gamma(const V2Geo& g) { return g.G > 1 && g.NCW >= 3 && g.NT / 32 > g.NCW; }
__host__ __device__ inline V2Head v2_head_layout(int C, const V2Geo& g, bool has_ps) {
  V2Head L;
  size_t o = 0;
  const size_t RC = (size_t)g.R * g.NCW * 32;  // ring columns padded to the head's lanes
  L.hg = o;   o += v2_a16(RC * 8);
  L.hs = o;   o += v2_a16(RC * 8);
  L.hS = o;   o += v2_a16(RC * 8);
  L.hP = o;   o += has_ps ? v2_a16(RC * 8) : 0;
  L.ha = o;   o += v2_a16(RC * 4);
  L.Tm = o;   o += v2_a16((size_t)C * C * 8);
  L.vsm = o;  o += v2_a16((size_t)2 * C * 8);
  L.part = o; o += g.G > 1 ? v2_a16((size_t)g.R * C * 16) : 0;
  L.tbar = o; o += v2_a16((size_t)g.R * 8);
  const size_t NPG = v2_par_gamma(g) ? (size_t)v2_gamma_warps(g) * g.NCW * 32 : 0;
  L.gpb = o;  o += v2_a16(NPG * 16);  // per (gamma warp, label): best and sec of its c' range
  L.gpa = o;  o += v2_a16(NPG * 4);   // and its first argmax
  L.total = o;
  return L;
}
struct V2Tail {
  size_t gs, sp, ga, bd, tbar, total;
};
__host__ __device__ inline V2Tail v2_tail_layout(int K, const V2Geo& g) {
  V2Tail L;
  size_t o = 0;
  const size_t KR = (size_t)g.KR * g.CgMax;
  L.gs = o;   o += v2_a16(KR * 16);  // (gmax, gsec)
  L.sp = o;   o += v2_a16(KR * 16);  // (S, Ps)
  L.ga = o;   o += v2_a16(KR * 4);   // argmax
  L.bd = o;   o += v2_a16((size_t)K * g.CgMax * 8);
  L.tbar = o; o += v2_a16((size_t)kVSrc * 8);
  L.total = o;
  return L;
}
__host__ __device__ inline size_t v2_smem_bytes(int K, int C, const V2Geo& g, bool has_ps) {
  const size_t h = v2_head_layout(C, g, has_ps).total;
  const size_t t = g.G > 1 ? v2_tail_layout(K, g).total : 0;
  return h > t ? h : t;
}

// reference tie rule for durations: larger value, ties to the larger k
__device__ __forceinline__ void v2_merge(double& v, int& k, double v2, int k2) {
  if (v2 > v || (v2 == v && k2 > k)) {
    v = v2;
    k = k2;
  }
}

__device__ __forceinline__ void v2_st_async_d2(uint32_t dst, double x, double y, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(dst), "d"(x),
               "d"(y), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void v2_st_async_i(uint32_t dst, int v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst), "r"(v), "r"(bar)
               : "memory");
}

// h(t, k, c) in the reference's order
__device__ __forceinline__ double v2_h(double St, double Ss, double Bk, double Pss, double Pet, bool ps, bool pe) {
  double h = __dadd_rn(__dadd_rn(St, -Ss), Bk);
  if (ps) h = __dadd_rn(h, Pss);
  if (pe) h = __dadd_rn(h, Pet);
  return h;
}

// ---------------------------------------------------------------------------- head
template <int NK>  // near candidates per step (>= kn)
__device__ void v2_head(const V2Args& a, unsigned char* smem, const V2Tail& TL, int b) {
  const V2Geo& g = a.geo;
  const int C = a.C, K = a.K, T = a.T;
  const int L = (int)a.lengths[b];
  const V2Head HL = v2_head_layout(C, g, a.ps != nullptr);
  double* hg = (double*)(smem + HL.hg);
  double* hs = (double*)(smem + HL.hs);
  double* hS = (double*)(smem + HL.hS);
  double* hP = a.ps ? (double*)(smem + HL.hP) : nullptr;
  int* ha = (int*)(smem + HL.ha);
  double* Tm = (double*)(smem + HL.Tm);
  double* vsm = (double*)(smem + HL.vsm);
  double2* part = (double2*)(smem + HL.part);
  uint64_t* tbar = (uint64_t*)(smem + HL.tbar);
  const int tid = threadIdx.x;
  const int NH = g.NCW * 32;
  const int Rm = g.R - 1, kn = g.kn;
  const bool tails = g.G > 1;
  const bool hps = a.ps != nullptr, hpe = a.pe != nullptr;
  const double* S = a.S + (size_t)b * (T + 1) * C;
  const double* ps = hps ? a.ps + (size_t)b * T * C : nullptr;
  const double* pe = hpe ? a.pe + (size_t)b * T * C : nullptr;
  double* hist = a.hist + (size_t)b * (T + 1) * C;
  int32_t* bp = a.bp + (size_t)b * (T + 1) * C;

  for (int i = tid; i < C * C; i += blockDim.x) Tm[i] = a.trans[i];
  if (tails && tid < g.R) mbar_init(smem_u32(&tbar[tid]), 1);
  __syncthreads();
  if (tails && tid == 0) {
    mbar_fence_init();
    for (int i = 0; i < g.R; ++i) mbar_expect(smem_u32(&tbar[i]), (uint32_t)(C * 16));
  }
  __syncthreads();
  if (tails) cluster_sync_all();
  // gamma over c' split across every warp of the head CTA: warp w scans c' in its range for
  // every label, then the label lanes join the ranges in order (the sequential scan's result
  // exactly: a later range wins only with a strictly larger value; its sec is the larger of
  // the earlier ranges' best and its own)
  const bool par = v2_par_gamma(g);
  const int GH = v2_gamma_warps(g), NPG = GH * 32;
  double2* gpb = (double2*)(smem + HL.gpb);
  int* gpa = (int*)(smem + HL.gpa);
  auto gamma_part = [&](int t) {
    const double* v = vsm + (t & 1) * C;
    const int w = tid >> 5, lane = tid & 31;
    const int CH = (C + GH - 1) / GH, c0 = w * CH, c1 = min(C, c0 + CH);
    for (int cw = 0; cw < g.NCW; ++cw) {
      const int lc = cw * 32 + lane;
      const int lcs = lc < C ? lc : 0;
      double best = -CUDART_INF, sec = -CUDART_INF;
      int arg = c0;
      for (int cp = c0; cp < c1; ++cp) {
        const double x = __dadd_rn(v[cp], Tm[(size_t)cp * C + lcs]);
        if (x > best) {
          sec = best;
          best = x;
          arg = cp;
        }
      }
      gpb[(size_t)w * NH + lc] = make_double2(best, sec);
      gpa[(size_t)w * NH + lc] = arg;
    }
  };
  if (tid >= NH) {
    if (!par) return;
    for (int t = 0; t <= L; ++t) {  // helper warps: the gamma ranges of every position
      asm volatile("bar.sync 2, %0;" ::"r"(NPG) : "memory");
      gamma_part(t);
      asm volatile("bar.sync 3, %0;" ::"r"(NPG) : "memory");
    }
    return;
  }

  const int c = tid;
  const bool act = c < C;
  const int cs = act ? c : 0;
  double bkr[NK];  // duration biases 1..kn of this label
#pragma unroll
  for (int i = 0; i < NK; ++i) bkr[i] = (i < kn) ? a.dur[(size_t)i * C + cs] : 0.0;
  // destination of this label's sources in its tail
  uint32_t t_gs = 0, t_sp = 0, t_ga = 0, t_bar = 0;
  if (tails) {
    int rt = 1;
    while (rt + 1 < g.G && v2_tail_lo(rt + 1, C, g.G) <= cs) ++rt;
    const int cl = cs - v2_tail_lo(rt, C, g.G);
    const size_t KR = (size_t)g.KR;
    t_gs = mapa_u32(smem_u32(smem + TL.gs) + (uint32_t)(cl * KR * 16), rt);
    t_sp = mapa_u32(smem_u32(smem + TL.sp) + (uint32_t)(cl * KR * 16), rt);
    t_ga = mapa_u32(smem_u32(smem + TL.ga) + (uint32_t)(cl * KR * 4), rt);
    t_bar = mapa_u32(smem_u32(smem + TL.tbar), rt);
  }
  const int nsrc_max = L - kn - 1;  // last source any tail needs
  auto sync_head = [&]() {
    if (g.NCW == 1)
      __syncwarp();
    else
      asm volatile("bar.sync 1, %0;" ::"r"(NH) : "memory");
  };
  // gamma of position t from the messages in vsm[(t & 1) * C ..]; ring slot t & Rm; push to tail
  // gmax = first maximum over c' of fl(v[c'] + T[c',c]) (smallest c' on ties) and gsec = the
  // best value over c' < argmax (the value the maximum replaced last)
  auto gamma = [&](int t, double St, double Pst) {
    const double* v = vsm + (t & 1) * C;
    double best = -CUDART_INF, sec = -CUDART_INF;
    int arg = 0;
    if (par) {
      asm volatile("bar.sync 2, %0;" ::"r"(NPG) : "memory");
      gamma_part(t);
      asm volatile("bar.sync 3, %0;" ::"r"(NPG) : "memory");
      best = gpb[c].x;
      sec = gpb[c].y;
      arg = gpa[c];
      for (int w = 1; w < GH; ++w) {
        const double2 pv = gpb[(size_t)w * NH + c];
        if (pv.x > best) {
          sec = best > pv.y ? best : pv.y;
          best = pv.x;
          arg = gpa[(size_t)w * NH + c];
        }
      }
    } else
    for (int c0 = 0; c0 < C; c0 += 8) {  // 8 independent loads + adds, then the ordered scan
      double x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cp = min(c0 + j, C - 1);
        x[j] = __dadd_rn(v[cp], Tm[(size_t)cp * C + cs]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c0 + j < C && x[j] > best) {
          sec = best;
          best = x[j];
          arg = c0 + j;
        }
    }
    {
      // every lane owns a ring column (padded to NH), so inactive lanes never read another
      // lane's slot
      const int r = t & Rm;
      hg[r * NH + c] = best;
      hs[r * NH + c] = sec;
      ha[r * NH + c] = arg;
      hS[r * NH + c] = St;
      if (hP) hP[r * NH + c] = Pst;
    }
    if (act) {
      if (tails && t <= nsrc_max) {
        const uint32_t sl = (uint32_t)(t % g.KR);
        const uint32_t bar = t_bar + (uint32_t)((t & (kVSrc - 1)) * 8);
        v2_st_async_d2(t_gs + sl * 16, best, sec, bar);
        v2_st_async_d2(t_sp + sl * 16, St, Pst, bar);
        v2_st_async_i(t_ga + sl * 4, arg, bar);
      }
    }
  };

  // position 0: every label starts from the virtual source with message 0
  if (act) {
    vsm[c] = 0.0;
    hist[c] = 0.0;
  }
  sync_head();
  gamma(0, act ? S[cs] : 0.0, (act && hps) ? ps[cs] : 0.0);
  // register prefetch of S[t], Pe[t-1], Ps[t] four positions ahead
  double fS[4], fPe[4], fPs[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = 1 + i;
    fS[i] = (act && t <= L) ? __ldg(S + (size_t)t * C + cs) : 0.0;
    fPe[i] = (act && hpe && t <= L) ? __ldg(pe + (size_t)(t - 1) * C + cs) : 0.0;
    fPs[i] = (act && hps && t <= L && t < T) ? __ldg(ps + (size_t)t * C + cs) : 0.0;
  }
#ifdef SCRF_VIT_PROF
  long long ph[6] = {0, 0, 0, 0, 0, 0}, c0 = 0, c1 = 0;
#define VPH(i) do { c1 = clock64(); ph[i] += c1 - c0; c0 = c1; } while (0)
#else
#define VPH(i) do {} while (0)
#endif
  for (int t = 1; t <= L; ++t) {
#ifdef SCRF_VIT_PROF
    c0 = clock64();
#endif
    const double St = fS[0], Pet = fPe[0], Pst = fPs[0];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      fS[i] = fS[i + 1];
      fPe[i] = fPe[i + 1];
      fPs[i] = fPs[i + 1];
    }
    {
      const int tn = t + 4;
      fS[3] = (act && tn <= L) ? __ldg(S + (size_t)tn * C + cs) : 0.0;
      fPe[3] = (act && hpe && tn <= L) ? __ldg(pe + (size_t)(tn - 1) * C + cs) : 0.0;
      fPs[3] = (act && hps && tn <= L && tn < T) ? __ldg(ps + (size_t)tn * C + cs) : 0.0;
    }
    // durations 1..kn from the ring
    // durations 1..kn from the ring (ties to the larger k)
    double best = -CUDART_INF, hb = 0.0;
    int bk = 0;
    const int kmax = min(kn, t);
    // all ring reads and adds first (slots of absent durations hold stale but readable values)
    double cv[NK], hv[NK];
#pragma unroll
    for (int i = 0; i < NK; ++i) {
      const int r = (t - i - 1) & Rm;
      hv[i] = v2_h(St, hS[r * NH + c], bkr[i], hP ? hP[r * NH + c] : 0.0, Pet, hps, hpe);
      cv[i] = __dadd_rn(hg[r * NH + c], hv[i]);
    }
#pragma unroll
    for (int i = 0; i < NK; ++i) {
      const int k = i + 1;
      if (k <= kmax && (cv[i] > best || (cv[i] == best && k > bk))) {
        best = cv[i];
        bk = k;
        hb = hv[i];
      }
    }
    VPH(0);
    int src = 0;
    bool flag = false;
    if (bk > 0) {
      const int r = (t - bk) & Rm;
      src = ha[r * NH + c];
      const double sec = hs[r * NH + c];
      flag = src > 0 && sec != -CUDART_INF && __dadd_rn(sec, hb) == best;
    }
    VPH(1);
    // durations kn+1..K from the tails
    if (tails && t > kn && K > kn) {
      const int pi = t - kn - 1;
      const int sl = pi & Rm;
      mbar_wait(smem_u32(&tbar[sl]), (uint32_t)((pi / g.R) & 1));
      const double2 pv = part[sl * C + cs];
      const int pk = __double_as_longlong(pv.y) & 0xffffffff;
      const int kT = (pk >> 16) & 0x7fff;
      if (pv.x > best || (pv.x == best && kT > bk)) {
        best = pv.x;
        bk = kT;
        src = pk & 0xffff;
        flag = (pk >> 31) & 1;
      }
      if (tid == 0 && t + g.R <= L) mbar_expect(smem_u32(&tbar[sl]), (uint32_t)(C * 16));
    }
    VPH(2);
    if (act && flag) {
      // rare: an earlier source label ties after rounding; re-scan in the reference's order
      const int s = t - bk;
      const double h = v2_h(St, S[(size_t)s * C + c], a.dur[(size_t)(bk - 1) * C + c],
                            hps ? ps[(size_t)s * C + c] : 0.0, Pet, hps, hpe);
      for (int cp = 0; cp < src; ++cp) {
        const double pv = s == 0 ? 0.0 : hist[(size_t)s * C + cp];
        if (__dadd_rn(__dadd_rn(pv, Tm[(size_t)cp * C + c]), h) == best) {
          src = cp;
          break;
        }
      }
    }
    if (act) {
      bp[(size_t)t * C + c] = (bk << 16) | src;
      hist[(size_t)t * C + c] = best;
      vsm[(t & 1) * C + c] = best;
    }
    sync_head();
    VPH(3);
    gamma(t, St, Pst);
    VPH(4);
  }
#ifdef SCRF_VIT_PROF
  if (b == 0 && tid == 0)
    printf("vit2 head cycles/step: near %.0f, flag %.0f, tail wait+merge %.0f, fix+store+sync %.0f, gamma+send %.0f\n",
           (double)ph[0] / L, (double)ph[1] / L, (double)ph[2] / L, (double)ph[3] / L, (double)ph[4] / L);
#endif
  sync_head();
  if (tid == 0) {
    const double* fin = vsm + (L & 1) * C;
    // final label: smallest argmax of the messages at L (streaming.py:458-460)
    int cbest = 0;
    for (int cc = 1; cc < C; ++cc)
      if (fin[cc] > fin[cbest]) cbest = cc;
    a.score[b] = fin[cbest];
    int32_t* st = a.seg_start + (size_t)b * T;
    int32_t* en = a.seg_end + (size_t)b * T;
    int32_t* lb = a.seg_label + (size_t)b * T;
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

// ---------------------------------------------------------------------------- tail
__device__ void v2_tail(const V2Args& a, unsigned char* smem, const V2Tail& TL, int b, int rank) {
  const V2Geo& g = a.geo;
  const int C = a.C, K = a.K, T = a.T;
  const int L = (int)a.lengths[b];
  const int lo = v2_tail_lo(rank, C, g.G), Cg = v2_tail_lo(rank + 1, C, g.G) - lo;
  const double2* GS = (const double2*)(smem + TL.gs);
  const double2* SP = (const double2*)(smem + TL.sp);
  const int* GA = (const int*)(smem + TL.ga);
  double* Bd = (double*)(smem + TL.bd);
  uint64_t* tbar = (uint64_t*)(smem + TL.tbar);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kn = g.kn, KR = g.KR;
  const bool hps = a.ps != nullptr, hpe = a.pe != nullptr;
  for (int i = tid; i < Cg * K; i += blockDim.x) {
    const int cl = i / K, k = i % K;
    Bd[i] = a.dur[(size_t)k * C + lo + cl];
  }
  if (tid < kVSrc) mbar_init(smem_u32(&tbar[tid]), 1);
  __syncthreads();
  if (tid == 0) {
    mbar_fence_init();
    for (int i = 0; i < kVSrc; ++i) mbar_expect(smem_u32(&tbar[i]), (uint32_t)(Cg * 36));
  }
  __syncthreads();
  cluster_sync_all();
  if (warp >= Cg * g.TW) return;
  const int cl = warp / g.TW, par = warp % g.TW;
  const int c = lo + cl;
  const double2* gsc = GS + (size_t)cl * KR;
  const double2* spc = SP + (size_t)cl * KR;
  const int* gac = GA + (size_t)cl * KR;
  const double* bdc = Bd + (size_t)cl * K;
  const double* S = a.S + (size_t)b * (T + 1) * C;
  const double* pe = hpe ? a.pe + (size_t)b * T * C : nullptr;
  const uint32_t hpart = mapa_u32(smem_u32(smem + v2_head_layout(C, g, hps).part), 0);
  const uint32_t hbar = mapa_u32(smem_u32(smem + v2_head_layout(C, g, hps).tbar), 0);
  const int nsrc_max = L - kn - 1;
  const int t0 = kn + 1 + par, tstep = g.TW;
  // register prefetch of S[t], Pe[t-1] four own targets ahead
  double fS[4], fPe[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + i * tstep;
    fS[i] = t <= L ? __ldg(S + (size_t)t * C + c) : 0.0;
    fPe[i] = (hpe && t <= L) ? __ldg(pe + (size_t)(t - 1) * C + c) : 0.0;
  }
  int snext = 0;
  for (int t = t0; t <= L; t += tstep) {
    const double St = fS[0], Pet = fPe[0];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      fS[i] = fS[i + 1];
      fPe[i] = fPe[i + 1];
    }
    {
      const int tn = t + 4 * tstep;
      fS[3] = tn <= L ? __ldg(S + (size_t)tn * C + c) : 0.0;
      fPe[3] = (hpe && tn <= L) ? __ldg(pe + (size_t)(tn - 1) * C + c) : 0.0;
    }
    // sources up to t-kn-1 (every source: both warps of a label read all of them)
    const int snew = t - kn - 1;
    for (int s = snext; s <= snew; ++s) {
      mbar_wait(smem_u32(&tbar[s & (kVSrc - 1)]), (uint32_t)((s / kVSrc) & 1));
      if (warp == 0 && lane == 0 && s + kVSrc <= nsrc_max)
        mbar_expect(smem_u32(&tbar[s & (kVSrc - 1)]), (uint32_t)(Cg * 36));
    }
    snext = snew + 1;
    double best = -CUDART_INF;
    int bk = 0;
    const int kmax = min(K, t);
    int r = (t - (kn + 1 + lane)) % KR;  // ring slot of source t-k, stepping down by 32
    if (r < 0) r += KR;
#pragma unroll 4
    for (int k = kn + 1 + lane; k <= kmax; k += 32) {
      const double2 gv = gsc[r], sv = spc[r];
      r -= 32;
      if (r < 0) r += KR;
      const double h = v2_h(St, sv.x, bdc[k - 1], sv.y, Pet, hps, hpe);
      v2_merge(best, bk, __dadd_rn(gv.x, h), k);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, off);
      const int ok = __shfl_xor_sync(0xffffffffu, bk, off);
      v2_merge(best, bk, ov, ok);
    }
    if (lane == 0) {
      int src = 0, flag = 0;
      if (bk > 0) {
        const int r = (t - bk) % KR;
        src = gac[r];
        const double sec = gsc[r].y;
        const double h = v2_h(St, spc[r].x, bdc[bk - 1], spc[r].y, Pet, hps, hpe);
        flag = (src > 0 && sec != -CUDART_INF && __dadd_rn(sec, h) == best) ? 1 : 0;
      }
      const int pk = (flag << 31) | (bk << 16) | src;
      const int pi = t - kn - 1;
      const uint32_t sl = (uint32_t)(pi & (g.R - 1));
      v2_st_async_d2(hpart + (uint32_t)((sl * C + c) * 16), best, __longlong_as_double((long long)(unsigned)pk),
                     hbar + sl * 8);
    }
  }
}

// NTMAX: thread bound of the instantiation (256 leaves the head 255 registers for its
// candidate arrays; 512 when the tails need 16 warps)
template <int NTMAX, int NK>
__global__ void __launch_bounds__(NTMAX) vit2_kernel(V2Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const V2Geo& g = a.geo;
  const int b = blockIdx.x / g.G, rank = blockIdx.x % g.G;
  const V2Tail TL = v2_tail_layout(a.K, g);
  if (rank == 0)
    v2_head<NK>(a, smem, TL, b);
  else
    v2_tail(a, smem, TL, b, rank);
  if (g.G > 1) cluster_sync_all();
}

}  // namespace scrf
