// C ABI of libscrf.so (declared in include/scrf.h): geometry selection, buffer
// layout and kernel launches. Host code only; kernels live in scrf_sweep.cuh, scrf_post.cuh and
// scrf_viterbi.cu (compiled into this translation unit so templates instantiate once).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/scrf.h"
#include "scrf_sweep.cuh"
#include "scrf_post.cuh"
#include "scrf_cut.cuh"
#include "scrf_viterbi.cu"
#include "scrf_vit2.cuh"

using namespace scrf;

namespace {

thread_local int g_launches = 0;
// optional events recorded around the next main kernel launch (forward / backward / Viterbi)
thread_local cudaEvent_t g_ev_start = nullptr;
thread_local cudaEvent_t g_ev_stop = nullptr;
thread_local cudaEvent_t g_ev_pos = nullptr;  // recorded once the per-position outputs are final
thread_local long long* g_trace = nullptr;  // debug: clock64 phase stamps of the next sweep
int* g_hang = nullptr;                        // debug: watchdog record (SCRF_WATCHDOG=1)

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}
int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p *= 2;
  return p;
}

int smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0)
      v = 227 * 1024;
  }
  return v;
}

int num_sms() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  }
  return v;
}

Geometry make_geo(int G, int K, int C) {
  Geometry g;
  g.G = G;
  g.Cgm = (C + G - 1) / G;
  int tpl = env_int("SCRF_TPL", 0);
  if (tpl <= 0) {
    // ~8 durations per thread, at most 1024 threads per CTA
    tpl = pow2_ceil(K / 8 > 0 ? K / 8 : 1);
    int cap = pow2_floor(1024 / g.Cgm > 0 ? 1024 / g.Cgm : 1);
    if (tpl > cap) tpl = cap;
  }
  g.TPL = tpl;
  g.GW = tpl < 32 ? tpl : 32;
  g.WPL = tpl >= 32 ? tpl / 32 : 1;
  int nt = g.Cgm * tpl;
  g.NT = (nt + 31) / 32 * 32;
  return g;
}

int choose_vit_geo(int B, int K, int C, bool has_ps, Geometry* out) {
  const size_t limit = (size_t)smem_optin();
  int forced = env_int("SCRF_G", 0);
  const int cands[] = {1, 2, 4, 8, 16};
  int gmin = 0;
  for (int G : cands) {
    if (G > C && G > 1) break;
    if (forced && G != forced) continue;
    Geometry g = make_geo(G, K, C);
    if (g.NT <= 1024 && vit_smem_bytes(K, C, g, has_ps) + 1024 <= limit) {
      gmin = G;
      break;
    }
  }
  if (!gmin) return SCRF_ECONFIG;
  int G = gmin;
  if (!forced)
    while (G * 2 <= 8 && G * 2 <= C && (long long)B * G * 2 <= num_sms()) G *= 2;
  *out = make_geo(G, K, C);
  return SCRF_OK;
}

int check_problem(const scrf_problem* p) {
  if (!p || !p->S || !p->lengths || !p->transition || !p->duration_bias) return SCRF_ENULL;
  if (p->B < 1 || p->T < 1 || p->K < 1 || p->C < 1) return SCRF_EDIM;
  if (p->T > (1LL << 30) || p->C > 1024 || p->K > 65535 || p->B > (1 << 20)) return SCRF_EDIM;
  return SCRF_OK;
}

int64_t n_ckpt_of(int64_t T, int64_t delta) { return (T + delta - 1) / delta; }

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// ---------------------------------------------------------------------------
// sweep geometry (scrf_sweep.cuh): head-only CTA when the duration range is small,
// otherwise a head + label-slice tails cluster sized to one wave of the chip.

int choose_sweep_geo(int B, int K, int C, int prec, int ndirs, bool has_ps, bool has_pe, SweepGeo* out) {
  const size_t limit = (size_t)smem_optin();
  SweepGeo g;
  memset(&g, 0, sizeof(g));
  g.TWb = 1;
  g.PsRow = has_ps ? 1 : 0;
  g.PeRow = has_pe ? (has_ps ? 2 : 1) : 0;
  g.NCW = (C + 31) / 32;
  if (g.NCW > 4) return SCRF_ECONFIG;  // C <= 128 (head roles fit one 512-thread CTA)
  g.Msm = (size_t)C * C * (prec ? 8 : 4) <= 65536 ? 1 : 0;
  g.NAS = g.NCW == 1 ? 2 : 1;  // separate source and edge warps when they fit
  g.NG = g.NCW == 1 ? 4 : 2;   // near groups (each owns every NG-th target)
  g.PubS = g.NAS == 2 ? 16 : 8; // batched edge warps / per-step edge in the source warps
  g.NOW = g.NAS == 2 ? 1 : 0;   // output warp beside the edge warps
  const int maxg = (16 - g.NCW - g.NAS * g.NCW - g.NOW) / g.NG;  // warps per near group
  // near lane-group width: SIMT runs each label's fp64 bookkeeping for the whole warp, so
  // use one lane per label unless a label has many ring terms (>= 16 per lane)
  auto near_gw = [&](int terms) {
    int gw = 1;
    while (gw < 32 && terms / (gw * 2) >= 16) gw *= 2;
    int env = env_int("SCRF_NEAR_GW", 0);
    if (env > 0) gw = env;
    while (gw > 1 && (C * gw + 31) / 32 > maxg) gw >>= 1;
    return gw;
  };
  const int forced = env_int("SCRF_SWEEP_G", 0);
  bool one = (long long)K * C <= 6144 || K <= kNear + 1;
  if (forced) one = (forced == 1) || K <= kNear + 1;
  if (one) {
    g.G = 1;
    g.kc = K;
    g.KRm = pow2_ceil(K) - 1;
    g.KTm = 0;
    g.WPL = 1;
    g.TBlk = 0;
    g.GWn = near_gw(K > 5 ? K - 5 : 1);
    g.NNW = g.NG * ((C * g.GWn + 31) / 32);
    g.NT = (g.NCW + g.NAS * g.NCW + g.NNW + g.NOW) * 32;
    size_t sm = prec ? sweep_smem_bytes<double>(K, C, g) : sweep_smem_bytes<float>(K, C, g);
    if (g.NNW <= g.NG * maxg && sm <= limit) {
      *out = g;
      return SCRF_OK;
    }
    if (K <= kNear + 1) return SCRF_ECONFIG;
  }
  g.kc = kNear;
  g.KRm = pow2_ceil(kNear) - 1;
  g.KTm = pow2_ceil(K) - 1;
  g.GWn = near_gw(kNear - 5);
  g.NNW = g.NG * ((C * g.GWn + 31) / 32);
  // blocked tails (one or two warps per label, <= 16 labels per tail) when the duration range
  // allows; at most 8 tails (8 x 16 labels covers C <= 128). (Larger clusters used to hang
  // because of spare warps in tails of an uneven label split; fixed in tail_loop_blocked.)
  bool blk = env_int("SCRF_TAIL_EXACT", 0) == 0 && K >= kNear + 33 && K <= 1024 + kNear;
  // blocked tails: <= 8 (8 x 16 labels covers C <= 128); exact tails may need up to 15 when their
  // K-long rings crowd shared memory (cluster of 16, non-portable size)
  auto max_tails = [&](bool blocked) { const int m = blocked ? 8 : 15; return C < m ? C : m; };
  auto start_tails = [&](bool blocked) {
    int t = forced > 1 ? forced - 1 : (blocked ? (C + 7) / 8 : (int)(((long long)K * C + 3499) / 3500));
    if (t > max_tails(blocked)) t = max_tails(blocked);
    if (t < 1) t = 1;
    if (!forced)
      while (t > 1 && (long long)B * ndirs * (1 + t) > num_sms()) --t;
    return t;
  };
  bool found = false;
  for (int pass = 0; pass < 2 && !found; ++pass) {
    // pass 0: blocked tails if eligible; pass 1: exact per-term tails
    if (pass == 1) {
      if (!blk) break;
      blk = false;
    }
    for (int tails = start_tails(blk); tails <= max_tails(blk); ++tails) {
      g.G = 1 + tails;
      g.CgMax = (C + tails - 1) / tails;
      g.WPL = 1;
      g.TBlk = (blk && g.CgMax <= 16) ? 1 : 0;
      g.TWb = (g.TBlk && g.CgMax * 2 <= 16) ? 2 : 1;  // two warps per label when they fit
      g.KTm = g.TBlk ? 63 : pow2_ceil(K) - 1;
      if (!g.TBlk)
        while (g.WPL < 4 && g.CgMax * g.WPL * 2 <= 16) g.WPL *= 2;
      g.NWt = g.CgMax * g.WPL < 16 ? g.CgMax * g.WPL : 16 / g.WPL * g.WPL;
      if (g.TBlk) g.NWt = g.CgMax * g.TWb;
      const int head_nt = (g.NCW + g.NAS * g.NCW + g.NNW + g.NOW) * 32;
      g.NT = head_nt > g.NWt * 32 ? head_nt : g.NWt * 32;
      size_t sm = prec ? sweep_smem_bytes<double>(K, C, g) : sweep_smem_bytes<float>(K, C, g);
      if (sm <= limit) {
        found = true;
        break;
      }
    }
  }
  if (!found) return SCRF_ECONFIG;
  *out = g;
  return SCRF_OK;
}

// forward state ("checkpoint buffer"): per-position alpha-side messages
struct FLayout {
  size_t Y, X, n, clamp, total;
};
FLayout f_layout(const scrf_problem* p, int prec) {
  FLayout L;
  const size_t rs = prec ? 8 : 4;
  const size_t npos = (size_t)p->B * (p->T + 1);
  size_t o = 0;
  L.Y = o;
  o += al(npos * p->C * rs);
  L.X = o;
  o += al(npos * p->C * rs);
  L.n = o;
  o += al(npos * 8);
  L.clamp = o;
  o += al(p->B * 4);
  L.total = o;
  return L;
}

struct PostGeo {
  int CH, nch, CGB, SCB, nchB;
};

PostGeo post_geo(const scrf_problem* p, int prec) {
  PostGeo q;
  const int C = (int)p->C, K = (int)p->K, T = (int)p->T, B = (int)p->B;
  q.CH = post_chunk(C);
  q.nch = (T + 1 + q.CH - 1) / q.CH;
  int cg = 4096 / K;
  if (cg < 1) cg = 1;
  if (cg > C) cg = C;
  const size_t limit = (size_t)smem_optin();
  while (cg > 1 && (prec ? post_gradB_smem<double>(K, cg) : post_gradB_smem<float>(K, cg)) > limit) --cg;
  while (cg > 1 && (long long)cg * ((K + kGBJ - 1) / kGBJ) > (long long)kGBW * 512) --cg;
  q.CGB = cg;
  const int ngc = (C + cg - 1) / cg;
  long long want = 4LL * num_sms();
  long long per = (want + (long long)ngc * B - 1) / ((long long)ngc * B);
  if (per < 1) per = 1;
  int scb = (int)((T + per - 1) / per);
  scb = (scb + kGBSub - 1) / kGBSub * kGBSub;
  if (scb < kGBSub) scb = kGBSub;
  q.SCB = scb;
  q.nchB = (T + scb - 1) / scb;
  return q;
}

// backward work buffer: beta-side messages + partials
struct BLayout {
  size_t Y, X, n, logZb, tot, cntp, gTp, gBp, gTs, gBs, cutU, corr, clamp, total;
};

// cut-normaliser spacing (scrf_cut.cuh): 0 disables the correction (SCRF_CUT_D=0, debugging)
int cut_spacing() { return env_int("SCRF_CUT_D", 512); }
int cut_slots(int64_t T, int d) { return d > 0 ? (int)((T - 1) / d) + 2 : 0; }
BLayout b_layout(const scrf_problem* p, int prec) {
  BLayout L;
  const size_t rs = prec ? 8 : 4;
  const size_t B = p->B, C = p->C, K = p->K;
  const size_t npos = B * (p->T + 1);
  const PostGeo q = post_geo(p, prec);
  size_t o = 0;
  L.Y = o;     o += al(npos * C * rs);
  L.X = o;     o += al(npos * C * rs);
  L.n = o;     o += al(npos * 8);
  L.logZb = o; o += al(B * 8);
  L.tot = o;   o += al(B * q.nch * C * 8);
  L.cntp = o;  o += al(B * q.nch * 8);
  L.gTp = o;   o += al(B * q.nch * C * C * 8);
  L.gBp = o;   o += al(B * q.nchB * K * C * 8);
  L.gTs = o;   o += al(B * C * C * 8);
  L.gBs = o;   o += al(B * K * C * 8);
  const int d = cut_spacing();
  L.cutU = o;  o += d > 0 ? al(B * (size_t)cut_slots(p->T, d) * C * 8) : 0;
  L.corr = o;  o += d > 0 ? al(B * (p->T + 1) * 8) : 0;
  L.clamp = o; o += al(B * 4);
  L.total = o;
  return L;
}

// Cluster launch with one CTA per SM: the recurrence CTAs are latency bound, and a second
// resident CTA (another cluster's tail) would share their issue slots, so the dynamic shared
// memory request is padded past half of the SM's capacity.
template <typename Kern, typename ArgT>
cudaError_t launch_cl(Kern kern, int G, int nclusters, int NT, size_t smem, cudaStream_t st, ArgT arg, bool record) {
  const size_t half = (size_t)smem_optin() / 2 + 1024;
  if (smem < half) smem = half;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (G > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(nclusters * G, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  if (record && g_ev_start) cudaEventRecord(g_ev_start, st);
  e = cudaLaunchKernelEx(&cfg, kern, arg);
  if (record && g_ev_stop) cudaEventRecord(g_ev_stop, st);
  return e;
}

template <typename R>
int run_sweep(const scrf_problem* p, int dirs, int64_t delta, const void* fstate, void* work, double* logZ, double* N,
              int32_t* dead_at, cudaStream_t st) {
  const int nd = dirs == 3 ? 2 : 1;
  SweepGeo g;
  int rc = choose_sweep_geo((int)p->B, (int)p->K, (int)p->C, sizeof(R) == 8, nd, p->proj_start != nullptr,
                            p->proj_end != nullptr, &g);
  if (rc) return rc;
  SweepArgs<R> a;
  memset(&a, 0, sizeof(a));
  a.S = p->S;
  a.lengths = p->lengths;
  a.trans = p->transition;
  a.dur = p->duration_bias;
  a.ps = p->proj_start;
  a.pe = p->proj_end;
  a.B = (int)p->B;
  a.T = (int)p->T;
  a.K = (int)p->K;
  a.C = (int)p->C;
  a.geo = g;
  a.dirs = dirs;
  const FLayout F = f_layout(p, sizeof(R) == 8);
  unsigned char* fb = (unsigned char*)fstate;
  a.Y[0] = (R*)(fb + F.Y);
  a.X[0] = (R*)(fb + F.X);
  a.n[0] = (double*)(fb + F.n);
  a.clamp = (dirs & 1) ? (int32_t*)(fb + F.clamp) : nullptr;
  if (work) {
    const BLayout W = b_layout(p, sizeof(R) == 8);
    unsigned char* wb = (unsigned char*)work;
    a.Y[1] = (R*)(wb + W.Y);
    a.X[1] = (R*)(wb + W.X);
    a.n[1] = (double*)(wb + W.n);
    a.logZb = (double*)(wb + W.logZb);
  }
  a.logZ = logZ;
  a.dead_at = dead_at;
  a.N = N;
  a.delta = (int)delta;
  a.n_ckpt = (int)n_ckpt_of(p->T, delta);
  a.trace = g_trace;
  a.trace_from = env_int("SCRF_TRACE_FROM", 64);
  if (env_int("SCRF_WATCHDOG", 0)) {
    if (!g_hang) {
      cudaMallocManaged(&g_hang, 8 * sizeof(int));
      memset(g_hang, 0, 8 * sizeof(int));
    }
    a.hang = g_hang;
  }
  const size_t smem = sweep_smem_bytes<R>(a.K, a.C, g);
  const bool tails = g.G > 1, cw1 = g.NCW == 1;
  cudaError_t e;
  if (tails && cw1)
    e = launch_cl(sweep_kernel<R, true, true>, g.G, a.B * nd, g.NT, smem, st, a, true);
  else if (tails)
    e = launch_cl(sweep_kernel<R, true, false>, g.G, a.B * nd, g.NT, smem, st, a, true);
  else if (cw1)
    e = launch_cl(sweep_kernel<R, false, true>, g.G, a.B * nd, g.NT, smem, st, a, true);
  else
    e = launch_cl(sweep_kernel<R, false, false>, g.G, a.B * nd, g.NT, smem, st, a, true);
  return (int)e;
}

template <typename R>
int run_post(const scrf_problem* p, const void* fstate, void* work, const double* logZ, const double* upstream,
             double* grad_S, double* grad_T, double* grad_B, double* gPs, double* gPe, double* pos, double* bnd,
             double* cnt, cudaStream_t st) {
  const PostGeo q = post_geo(p, sizeof(R) == 8);
  const FLayout F = f_layout(p, sizeof(R) == 8);
  const BLayout W = b_layout(p, sizeof(R) == 8);
  const unsigned char* fb = (const unsigned char*)fstate;
  unsigned char* wb = (unsigned char*)work;
  PostArgs<R> a;
  memset(&a, 0, sizeof(a));
  a.S = p->S;
  a.lengths = p->lengths;
  a.trans = p->transition;
  a.dur = p->duration_bias;
  a.ps = p->proj_start;
  a.pe = p->proj_end;
  a.upstream = upstream;
  a.logZ = logZ;
  a.B = (int)p->B;
  a.T = (int)p->T;
  a.K = (int)p->K;
  a.C = (int)p->C;
  a.Ya = (const R*)(fb + F.Y);
  a.Xa = (const R*)(fb + F.X);
  a.na = (const double*)(fb + F.n);
  a.Yb = (const R*)(wb + W.Y);
  a.Xb = (const R*)(wb + W.X);
  a.nb = (const double*)(wb + W.n);
  a.grad_S = grad_S;
  a.grad_Ps = gPs;
  a.grad_Pe = gPe;
  a.pos = pos;
  a.bnd = bnd;
  a.CH = q.CH;
  a.nch = q.nch;
  a.tot = (double*)(wb + W.tot);
  a.cntp = (double*)(wb + W.cntp);
  a.gTp = (double*)(wb + W.gTp);
  a.SCB = q.SCB;
  a.nchB = q.nchB;
  a.CGB = q.CGB;
  a.gBp = (double*)(wb + W.gBp);
  const int B = a.B, C = a.C, K = a.K, T = a.T;
  cudaError_t e;
  const int cd = cut_spacing();
  if (cd > 0) {
    // cut normalisers, then the per-position frame correction the passes below apply
    CutArgs<R> ca;
    memset(&ca, 0, sizeof(ca));
    ca.S = p->S;
    ca.lengths = p->lengths;
    ca.dur = p->duration_bias;
    ca.ps = p->proj_start;
    ca.pe = p->proj_end;
    ca.logZ = logZ;
    ca.B = B;
    ca.T = T;
    ca.K = K;
    ca.C = C;
    ca.Ya = a.Ya;
    ca.Xa = a.Xa;
    ca.Yb = a.Yb;
    ca.Xb = a.Xb;
    ca.na = a.na;
    ca.nb = a.nb;
    ca.d = cd;
    ca.ncut = cut_slots(T, cd);
    ca.U = (double*)(wb + W.cutU);
    const size_t sm = cut_smem<R>(K);
    e = cudaFuncSetAttribute(cut_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    cut_kernel<R><<<dim3(ca.ncut, (C + kCutCG - 1) / kCutCG, B), 256, sm, st>>>(ca);
    a.corr = (const double*)(wb + W.corr);
  }
  {
    // per-position frame correction (when enabled) and the beta-side clamp-event count
    e = cudaMemsetAsync(wb + W.clamp, 0, (size_t)B * 4, st);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    cut_corr_kernel<R><<<dim3((T + 1 + 255) / 256, B), 256, 0, st>>>(
        p->lengths, T, C, cd, cd > 0 ? cut_slots(T, cd) : 0, cd > 0 ? (const double*)(wb + W.cutU) : nullptr,
        cd > 0 ? (double*)(wb + W.corr) : nullptr, a.Xb, a.nb, (int32_t*)(wb + W.clamp));
  }
  {
    const size_t sm = post_pos_smem<R>(C, q.CH);
    e = cudaFuncSetAttribute(post_pos_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    post_pos_kernel<R><<<dim3(q.nch, B), 256, sm, st>>>(a);
    ++g_launches;
    ++g_launches;
    if (cd > 0 && cd % q.CH == 0)
      cut_prefix_kernel<<<(B * C + 127) / 128, 128, 0, st>>>(p->lengths, B, C, q.nch, q.CH, cd, cut_slots(T, cd),
                                                           (const double*)(wb + W.cutU), a.tot);
    else
      post_prefix_kernel<<<(B * C + 7) / 8, 256, 0, st>>>(B, C, q.nch, a.tot);
    post_carry_kernel<<<dim3(q.nch, B), 64, 0, st>>>(p->lengths, B, T, C, q.CH, q.nch, a.tot, pos);
    if (g_ev_pos) cudaEventRecord(g_ev_pos, st);
  }
  {
    // one CTA holds every duration window of its label group (K <= kGBW * 512 * kGBJ = 4096)
    if ((long long)q.CGB * ((K + kGBJ - 1) / kGBJ) > (long long)kGBW * 512) return SCRF_ECONFIG;
    const size_t sm = post_gradB_smem<R>(K, q.CGB);
    e = cudaFuncSetAttribute(post_gradB_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    post_gradB_kernel<R><<<dim3(q.nchB, (C + q.CGB - 1) / q.CGB, B), 512, sm, st>>>(a);
  }
  {
    const int nT = C * C, nB = K * C;
    ++g_launches;
    post_reduce2_kernel<<<(nT + 31) / 32, 256, 0, st>>>(B, nT, q.nch, a.gTp, upstream, (double*)(wb + W.gTs), grad_T);
    ++g_launches;
    post_reduce2_kernel<<<(nB + 31) / 32, 256, 0, st>>>(B, nB, q.nchB, a.gBp, upstream, (double*)(wb + W.gBs), grad_B);
    ++g_launches;
    post_count_kernel<<<(B + 127) / 128, 128, 0, st>>>(B, q.nch, a.cntp, cnt);
  }
  return (int)cudaGetLastError();
}

// reference-format checkpoint view (streaming.py:49-67): ring after the shift at i*delta
template <typename R>
__global__ void export_kernel(const R* Ya, const double* na, const double* N, const int64_t* lengths, int B, int T,
                              int nck, int K, int C, int delta, double* omega) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)B * nck * K * C;
  if (i >= total) return;
  const int c = (int)(i % C);
  const int slot = (int)((i / C) % K);
  const int ck = (int)((i / ((size_t)C * K)) % nck);
  const int b = (int)(i / ((size_t)C * K * nck));
  const int L = (int)lengths[b];
  long long e = (long long)ck * delta;
  if (e > L) e = L;
  long long s = e - (((e - slot) % K) + K) % K;
  if (s < 0) {
    omega[i] = kNegInfRef;
    return;
  }
  const size_t o = ((size_t)b * (T + 1) + s);
  const R y = Ya[o * C + c];
  if (!(y > -INFINITY)) {
    omega[i] = kNegInfRef;
    return;
  }
  const double v = (na[o] + (double)y) * kLn2 - N[(size_t)b * nck + ck];
  omega[i] = v <= kGuard ? kNegInfRef : v;
}
__global__ void clamp_sum_kernel(int B, const int32_t* a, const int32_t* b, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) out[i] = a[i] + (b ? b[i] : 0);
}
}  // namespace

extern "C" {

int64_t scrf_default_delta(int64_t T, int64_t K) {
  if (T < 1) return 1;
  int64_t d = (int64_t)llround(sqrt((double)T * (double)K));
  if (d < 1) d = 1;
  if (d > T) d = T;
  return d;
}

int scrf_checkpoint_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  *bytes = f_layout(p, precision).total;
  return SCRF_OK;
}

int scrf_forward(const scrf_problem* p, int64_t delta, int precision, double* logZ, double* N, int32_t* dead_at,
                 void* ckpt, size_t ckpt_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  if (!logZ || !N || !dead_at || !ckpt) return SCRF_ENULL;
  if (ckpt_bytes < f_layout(p, precision).total) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  return precision ? run_sweep<double>(p, 1, delta, ckpt, nullptr, logZ, N, dead_at, st)
                   : run_sweep<float>(p, 1, delta, ckpt, nullptr, logZ, N, dead_at, st);
}

int scrf_backward_work_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  *bytes = b_layout(p, precision).total;
  return SCRF_OK;
}

static int check_bwd_args(const scrf_problem* p, int64_t delta, const double* logZ, const void* ckpt, double* grad_S,
                          double* grad_T, double* grad_B, double* pos, double* bnd, double* cnt, void* work) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  if (!logZ || !ckpt || !grad_S || !grad_T || !grad_B || !pos || !bnd || !cnt || !work) return SCRF_ENULL;
  return SCRF_OK;
}

int scrf_backward(const scrf_problem* p, int64_t delta, int precision, const double* logZ, const void* ckpt,
                  const double* upstream, double* grad_S, double* grad_T, double* grad_B, double* grad_P_start,
                  double* grad_P_end, double* position_marginals, double* boundary_posterior,
                  double* expected_segment_count, void* work, size_t work_bytes, void* stream) {
  g_launches = 0;
  int rc = check_bwd_args(p, delta, logZ, ckpt, grad_S, grad_T, grad_B, position_marginals, boundary_posterior,
                          expected_segment_count, work);
  if (rc) return rc;
  if (work_bytes < b_layout(p, precision).total) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  rc = precision ? run_sweep<double>(p, 2, delta, ckpt, work, nullptr, nullptr, nullptr, st)
                 : run_sweep<float>(p, 2, delta, ckpt, work, nullptr, nullptr, nullptr, st);
  if (rc) return rc;
  return precision ? run_post<double>(p, ckpt, work, logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end,
                                      position_marginals, boundary_posterior, expected_segment_count, st)
                   : run_post<float>(p, ckpt, work, logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end,
                                     position_marginals, boundary_posterior, expected_segment_count, st);
}

int scrf_posterior(const scrf_problem* p, int64_t delta, int precision, const double* upstream, double* logZ, double* N,
                   int32_t* dead_at, void* ckpt, size_t ckpt_bytes, double* grad_S, double* grad_T, double* grad_B,
                   double* grad_P_start, double* grad_P_end, double* position_marginals, double* boundary_posterior,
                   double* expected_segment_count, void* work, size_t work_bytes, void* stream) {
  g_launches = 0;
  int rc = check_bwd_args(p, delta, logZ, ckpt, grad_S, grad_T, grad_B, position_marginals, boundary_posterior,
                          expected_segment_count, work);
  if (rc) return rc;
  if (!N || !dead_at) return SCRF_ENULL;
  if (ckpt_bytes < f_layout(p, precision).total || work_bytes < b_layout(p, precision).total) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  rc = precision ? run_sweep<double>(p, 3, delta, ckpt, work, logZ, N, dead_at, st)
                 : run_sweep<float>(p, 3, delta, ckpt, work, logZ, N, dead_at, st);
  if (rc) return rc;
  const int n0 = g_launches;
  rc = precision ? run_post<double>(p, ckpt, work, logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end,
                                    position_marginals, boundary_posterior, expected_segment_count, st)
                 : run_post<float>(p, ckpt, work, logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end,
                                   position_marginals, boundary_posterior, expected_segment_count, st);
  (void)n0;
  return rc;
}

int scrf_backward_partials(const scrf_problem* p, int64_t delta, int precision, const void* work,
                           double* grad_T_partial, double* grad_B_partial, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  (void)delta;
  const BLayout W = b_layout(p, precision);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned char* w = (const unsigned char*)work;
  cudaError_t e = cudaMemcpyAsync(grad_T_partial, w + W.gTs, (size_t)p->B * p->C * p->C * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(grad_B_partial, w + W.gBs, (size_t)p->B * p->K * p->C * 8, cudaMemcpyDeviceToDevice, st);
  return (int)e;
}

int scrf_beta_logz(const scrf_problem* p, int precision, const void* work, double* logZb, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  const BLayout W = b_layout(p, precision);
  return (int)cudaMemcpyAsync(logZb, (const unsigned char*)work + W.logZb, (size_t)p->B * 8, cudaMemcpyDeviceToDevice,
                              (cudaStream_t)stream);
}

static size_t vit_dvr_bytes(const scrf_problem* p, const Geometry& g) { return al((size_t)p->B * g.G * p->K * p->C * 8); }

// head + tails Viterbi (scrf_vit2.cuh): head-only when K <= 16, otherwise the head keeps
// durations 1..R/2 (R = 32, 16 or 8, the largest whose rings fit next to the C x C transition
// table) and ceil(C (K - kn) / 4000) tails (<= 16 labels each, two warps per label when they fit)
int choose_vit2_geo(int B, int K, int C, bool has_ps, V2Geo* out) {
  if (env_int("SCRF_VIT_OLD", 0)) return SCRF_ECONFIG;
  const size_t limit = (size_t)smem_optin();
  V2Geo g;
  memset(&g, 0, sizeof(g));
  g.NCW = (C + 31) / 32;
  if (g.NCW > 16) return SCRF_ECONFIG;
  g.TW = 1;
  g.KR = 8;
  if (K <= 16) {
    g.G = 1;
    g.R = 32;
    g.kn = K;
    g.NT = g.NCW * 32;
    if (v2_smem_bytes(K, C, g, has_ps) > limit) return SCRF_ECONFIG;
    *out = g;
    return SCRF_OK;
  }
  for (int R = 8; R >= 8; R >>= 1) {  // near durations 1..4: the head's fp64 compares are its bottleneck
    g.R = R;
    g.kn = R / 2;
    int nt = (int)(((long long)C * (K - g.kn) + 3999) / 4000);
    const int ntmin = (C + 15) / 16;
    if (nt < ntmin) nt = ntmin;
    if (nt > 15) nt = 15;
    if (nt > C) nt = C;
    while (nt > ntmin && (long long)B * (1 + nt) > num_sms()) --nt;
    g.G = 1 + nt;
    g.CgMax = (C + nt - 1) / nt;
    if (g.CgMax > 16) continue;
    g.TW = g.CgMax * 2 <= 16 ? 2 : 1;
    g.KR = K + 8;
    const int nth = g.NCW * 32, ntt = g.CgMax * g.TW * 32;
    g.NT = nth > ntt ? nth : ntt;
    if (g.NT > 512) continue;
    if (v2_smem_bytes(K, C, g, has_ps) <= limit) {
      *out = g;
      return SCRF_OK;
    }
  }
  return SCRF_ECONFIG;
}

int scrf_viterbi_work_bytes(const scrf_problem* p, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  V2Geo g2;
  if (choose_vit2_geo((int)p->B, (int)p->K, (int)p->C, p->proj_start != nullptr, &g2) == SCRF_OK) {
    *bytes = al((size_t)p->B * (p->T + 1) * p->C * 8) + al((size_t)p->B * (p->T + 1) * p->C * 4);
    return SCRF_OK;
  }
  Geometry g;
  rc = choose_vit_geo((int)p->B, (int)p->K, (int)p->C, p->proj_start != nullptr, &g);
  if (rc) return rc;
  *bytes = vit_dvr_bytes(p, g) + al((size_t)p->B * (p->T + 1) * p->C * 4);
  return SCRF_OK;
}

int scrf_viterbi(const scrf_problem* p, double* score, int32_t* seg_start, int32_t* seg_end, int32_t* seg_label,
                 int32_t* seg_count, void* work, size_t work_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (!score || !seg_start || !seg_end || !seg_label || !seg_count || !work) return SCRF_ENULL;
  size_t need = 0;
  scrf_viterbi_work_bytes(p, &need);
  if (work_bytes < need) return SCRF_EWORK;
  V2Geo g2;
  if (choose_vit2_geo((int)p->B, (int)p->K, (int)p->C, p->proj_start != nullptr, &g2) == SCRF_OK) {
    V2Args a;
    memset(&a, 0, sizeof(a));
    a.S = p->S;
    a.lengths = p->lengths;
    a.trans = p->transition;
    a.dur = p->duration_bias;
    a.ps = p->proj_start;
    a.pe = p->proj_end;
    a.B = (int)p->B;
    a.T = (int)p->T;
    a.K = (int)p->K;
    a.C = (int)p->C;
    a.geo = g2;
    unsigned char* w = (unsigned char*)work;
    a.hist = (double*)w;
    a.bp = (int32_t*)(w + al((size_t)p->B * (p->T + 1) * p->C * 8));
    a.score = score;
    a.seg_start = seg_start;
    a.seg_end = seg_end;
    a.seg_label = seg_label;
    a.seg_count = seg_count;
    const size_t smem = v2_smem_bytes(a.K, a.C, g2, a.ps != nullptr);
    cudaError_t e;
    auto kern = g2.NT <= 256 ? (g2.kn <= 4 ? vit2_kernel<256, 4> : g2.kn <= 8 ? vit2_kernel<256, 8> : vit2_kernel<256, 16>)
                             : (g2.kn <= 4 ? vit2_kernel<512, 4> : g2.kn <= 8 ? vit2_kernel<512, 8> : vit2_kernel<512, 16>);
    if (g2.G > 1) {
      e = launch_cl(kern, g2.G, a.B, g2.NT, smem, (cudaStream_t)stream, a, true);
    } else {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) {
        ++g_launches;
        if (g_ev_start) cudaEventRecord(g_ev_start, (cudaStream_t)stream);
        kern<<<a.B, g2.NT, smem, (cudaStream_t)stream>>>(a);
        e = cudaGetLastError();
        if (g_ev_stop) cudaEventRecord(g_ev_stop, (cudaStream_t)stream);
      }
    }
    return (int)e;
  }
  Geometry g;
  rc = choose_vit_geo((int)p->B, (int)p->K, (int)p->C, p->proj_start != nullptr, &g);
  if (rc) return rc;
  VitArgs a;
  memset(&a, 0, sizeof(a));
  a.S = p->S;
  a.lengths = p->lengths;
  a.trans = p->transition;
  a.dur = p->duration_bias;
  a.ps = p->proj_start;
  a.pe = p->proj_end;
  a.B = (int)p->B;
  a.T = (int)p->T;
  a.K = (int)p->K;
  a.C = (int)p->C;
  a.geo = g;
  unsigned char* w = (unsigned char*)work;
  a.dvring = (double*)w;
  a.bp = (int32_t*)(w + vit_dvr_bytes(p, g));
  a.score = score;
  a.seg_start = seg_start;
  a.seg_end = seg_end;
  a.seg_label = seg_label;
  a.seg_count = seg_count;
  size_t smem = vit_smem_bytes(a.K, a.C, g, a.ps != nullptr);
  cudaError_t e = launch_cl(vit_kernel, g.G, a.B, g.NT, smem, (cudaStream_t)stream, a, true);
  return (int)e;
}

int scrf_export_checkpoints(const scrf_problem* p, int64_t delta, int precision, const void* ckpt, const double* N,
                            double* omega, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  const FLayout F = f_layout(p, precision);
  const unsigned char* base = (const unsigned char*)ckpt;
  const int nck = (int)n_ckpt_of(p->T, delta);
  size_t total = (size_t)p->B * nck * p->K * p->C;
  ++g_launches;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (precision)
    export_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>((const double*)(base + F.Y), (const double*)(base + F.n), N,
                                                                  p->lengths, (int)p->B, (int)p->T, nck, (int)p->K,
                                                                  (int)p->C, (int)delta, omega);
  else
    export_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)(base + F.Y), (const double*)(base + F.n), N,
                                                                 p->lengths, (int)p->B, (int)p->T, nck, (int)p->K,
                                                                 (int)p->C, (int)delta, omega);
  return (int)cudaGetLastError();
}

int scrf_clamp_events(const scrf_problem* p, int precision, const void* ckpt, const void* work, int32_t* events,
                      void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (!ckpt || !events) return SCRF_ENULL;
  const FLayout F = f_layout(p, precision);
  cudaStream_t st = (cudaStream_t)stream;
  ++g_launches;
  clamp_sum_kernel<<<(unsigned)((p->B + 127) / 128), 128, 0, st>>>(
      (int)p->B, (const int32_t*)((const unsigned char*)ckpt + F.clamp),
      work ? (const int32_t*)((const unsigned char*)work + b_layout(p, precision).clamp) : nullptr, events);
  return (int)cudaGetLastError();
}

int scrf_last_launch_count(void) { return g_launches; }

int scrf_debug_hang(int* out5) {
  if (!g_hang) return 0;
  for (int i = 0; i < 5; ++i) out5[i] = g_hang[i];
  return g_hang[0];
}

void scrf_debug_trace(void* buf) { g_trace = (long long*)buf; }

void scrf_profile_events(void* start, void* stop) {
  g_ev_start = (cudaEvent_t)start;
  g_ev_stop = (cudaEvent_t)stop;
}

void scrf_position_outputs_event(void* event) { g_ev_pos = (cudaEvent_t)event; }

}  // extern "C"
