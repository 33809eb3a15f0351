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
// optional events recorded once the per-position outputs of window i (scrf_window_plan order) are final
thread_local cudaEvent_t* g_win_ev = nullptr;
thread_local int g_win_nev = 0;
// streamed input gate of the next full-mode sweeps (scrf_input_gate)
thread_local const int* g_gate = nullptr;
thread_local int g_gate_n = 0, g_gate_shift = 12;
thread_local long long* g_trace = nullptr;  // debug: clock64 phase stamps of the next sweep
int* g_hang = nullptr;                        // debug: watchdog record (SCRF_WATCHDOG=1)

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// SCRF_WPERM=<hex digits>: digit i = the head role (logical warp) physical warp i runs
// (placement experiment: which roles share an SM sub-partition); must be a permutation
unsigned long long head_wperm(int nwarps, int ncw, bool one_chain) {
  const char* v = getenv("SCRF_WPERM");
  // default for the 8-warp head (chain, 4 near groups, source, edge, output): the output warp on
  // the chain's sub-partition and the last near group beside the third (c4: sweep -2.5 %,
  // profiles/r02_head_attribution.txt); the edge warp's fp64 bursts stay off the chain's SMSP
  if (!v && one_chain && nwarps == 8) v = "01237564";
  if (!v || (int)strlen(v) != nwarps || nwarps > 16) return 0;
  unsigned long long m = 0;
  int seen = 0;
  for (int i = 0; i < nwarps; ++i) {
    const int d = (v[i] >= 'a') ? v[i] - 'a' + 10 : v[i] - '0';
    if (d < 0 || d >= nwarps || (seen >> d) & 1) return 0;
    if (i < ncw && d != i) return 0;  // the chain warps stay on warps 0 .. NCW-1
    seen |= 1 << d;
    m |= (unsigned long long)d << (4 * i);
  }
  for (int i = nwarps; i < 16; ++i) m |= (unsigned long long)i << (4 * i);  // warps beyond the head roles
  return m;
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
      g.wperm = head_wperm(g.NCW + g.NAS * g.NCW + g.NNW + g.NOW, g.NCW, g.NCW == 1 && g.NOW == 1);
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
      if (blk && !g.TBlk && env_int("SCRF_TAIL_ML", 1)) {
        // several labels per warp: LB lanes per label hold the <= LB live complete blocks
        const int nblk = (K - kNear - 1) / 32 + 1;
        int LB = 8;
        while (LB < nblk) LB *= 2;
        if (LB <= 16 && (g.CgMax + 32 / LB - 1) / (32 / LB) <= 16) g.TBlk = LB;
      }
      g.TWb = (g.TBlk == 1 && g.CgMax * 2 <= 16) ? 2 : 1;  // two warps per label when they fit
      g.KTm = g.TBlk ? 63 : pow2_ceil(K) - 1;
      if (!g.TBlk)
        while (g.WPL < 4 && g.CgMax * g.WPL * 2 <= 16) g.WPL *= 2;
      g.NWt = g.CgMax * g.WPL < 16 ? g.CgMax * g.WPL : 16 / g.WPL * g.WPL;
      if (g.TBlk == 1) g.NWt = g.CgMax * g.TWb;
      if (g.TBlk > 1) g.NWt = (g.CgMax + 32 / g.TBlk - 1) / (32 / g.TBlk);
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
  g.wperm = head_wperm(g.NCW + g.NAS * g.NCW + g.NNW + g.NOW, g.NCW, g.NCW == 1 && g.NOW == 1);
  *out = g;
  return SCRF_OK;
}

// ---------------------------------------------------------------------------
// buffer layouts

// full-mode forward state ("checkpoint buffer"): per-position alpha-side messages
struct FLayout {
  size_t Y, X, n, amx, clamp, total;
};
FLayout f_layout(const scrf_problem* p, int prec) {
  FLayout L;
  const size_t rs = prec ? 8 : 4;
  const size_t npos = (size_t)p->B * (p->T + 1);
  size_t o = 0;
  L.Y = o;     o += al(npos * p->C * rs);
  L.X = o;     o += al(npos * p->C * rs);
  L.n = o;     o += al(npos * 8);
  L.amx = o;   o += al(npos * rs);
  L.clamp = o; o += al(p->B * 4);
  L.total = o;
  return L;
}

// sublinear mode geometry: alpha checkpoint rows keep the last mA = min(K + 32, delta) positions
// of every delta-period (covering the reference's omega snapshots and the warm-up of a replay
// window); replay windows are W positions, a multiple of delta with W >= K + 32; beta
// checkpoint rows hold K + 32 positions above every interior window boundary
struct SparseGeo {
  int mA, W, nW, nWin;
  long long rowsAlpha, rowsBeta;  // per sequence
  int rowsWin;                    // rows of a replay window buffer per sequence
};
SparseGeo sparse_geo(const scrf_problem* p, int64_t delta) {
  SparseGeo g;
  const int K = (int)p->K, T = (int)p->T, d = (int)delta;
  g.mA = K + 32 < d ? K + 32 : d;
  g.W = d >= K + 32 ? d : d * ((K + 32 + d - 1) / d);
  g.nW = (T + g.W - 1) / g.W - 1;
  if (g.nW < 0) g.nW = 0;
  g.nWin = (T + 1 + g.W - 1) / g.W;
  g.rowsAlpha = ck_rows_alpha(T, d, g.mA);
  g.rowsBeta = (long long)g.nW * (K + 32);
  g.rowsWin = g.W + K + 33;
  return g;
}

// sparse forward state: alpha checkpoint rows (Y^, n) + clamp counts
struct SLayout {
  size_t Y, n, clamp, total;
};
SLayout s_layout(const scrf_problem* p, int64_t delta, int prec) {
  SLayout L;
  const size_t rs = prec ? 8 : 4;
  const SparseGeo g = sparse_geo(p, delta);
  const size_t rows = (size_t)p->B * g.rowsAlpha;
  size_t o = 0;
  L.Y = o;     o += al(rows * p->C * rs);
  L.n = o;     o += al(rows * 8);
  L.clamp = o; o += al(p->B * 4);
  L.total = o;
  return L;
}

struct PostGeo {
  int CH, nch, CGB, SCB, nchB;
};

// grad_B in exp space for the fp32 working type (SCRF_GRADB_EXACT=1: one ex2 per term)
bool gradB_blocked() { return env_int("SCRF_GRADB_EXACT", 0) == 0; }

// posterior-pass geometry for passes of at most Wn positions
PostGeo post_geo(const scrf_problem* p, int prec, int Wn) {
  PostGeo q;
  const int C = (int)p->C, K = (int)p->K, B = (int)p->B;
  q.CH = post_chunk(C);
  q.nch = (Wn + q.CH - 1) / q.CH;
  const size_t limit = (size_t)smem_optin();
  int cg;
  if (prec == 0 && gradB_blocked()) {
    // exp-space blocked kernel: one warp per (label, 128 durations), <= 2 items per warp
    cg = 16 / gbb_npass(K);
    if (cg < 1) cg = 1;
    if (cg > C) cg = C;
    while (cg > 1 && post_gradB_blk_smem(K, cg) > limit) --cg;
  } else {
    cg = 4096 / K;
    if (cg < 1) cg = 1;
    if (cg > C) cg = C;
    while (cg > 1 && (prec ? post_gradB_smem<double>(K, cg) : post_gradB_smem<float>(K, cg)) > limit) --cg;
    while (cg > 1 && (long long)cg * ((K + kGBJ - 1) / kGBJ) > (long long)kGBW * 512) --cg;
  }
  q.CGB = cg;
  const int ngc = (C + cg - 1) / cg;
  // blocked grad_B: one full wave at one CTA per SM (128 registers, no spills); exact kernel:
  // ~4 CTAs per SM
  const bool blk = prec == 0 && gradB_blocked();
  long long want = (blk ? 1LL : 4LL) * num_sms();
  long long per = blk ? want / ((long long)ngc * B) : (want + (long long)ngc * B - 1) / ((long long)ngc * B);
  if (per < 1) per = 1;
  // CTA source ranges are whole micro-chunks; partials are kept per micro-chunk (the
  // per-sequence grad_B sum order depends on T only, not on B: sharding stays bit-identical)
  const int nmic = (Wn + kGBMicro - 1) / kGBMicro;
  int mper = (int)((nmic + per - 1) / per);
  if (mper < 1) mper = 1;
  q.SCB = mper * kGBMicro;
  q.nchB = nmic;
  return q;
}

// cut-normaliser spacing (scrf_cut.cuh): 0 disables the correction (SCRF_CUT_D=0, debugging)
int cut_spacing() { return env_int("SCRF_CUT_D", 512); }

// Full-mode posterior passes (see run_full_post_win): SCRF_OVERLAP 1 = windows concurrent with
// the sweeps (default), 0 = the same windows after the sweeps, -1 = one pass after the sweeps.
int ovl_ws() { return env_int("SCRF_OVL_WS", 4096); }
int ovl_mode(const scrf_problem* p) {
  const int m = env_int("SCRF_OVERLAP", 1);
  const int ws = ovl_ws();
  if (m < 0 || cut_spacing() <= 0 || ws <= 0 || ws % kGBMicro || ws % cut_spacing()) return -1;
  if ((long long)p->T + 1 < 4LL * ws) return -1;  // too short to gain from windows
  if ((long long)p->T + 1 > 4096LL * ws) return -1;
  return m > 0 ? 1 : 0;
}

// per-pass partials and the running per-sequence accumulators
struct PLayout {
  size_t logZb, tot, cntp, gTp, gBp, cutU, corr, carry, clamp, accT, accB, accN, Zt, tcut, prog, status, RA, RB, Wt,
      Bmax, total;
  int prepNR;  // rows of RA / RB per (sequence, label): the longest pass + 2K - 1
  int nprep;   // RA / RB sets (2: concurrent windows on two side streams)
};
PLayout p_layout(const scrf_problem* p, int prec, int Wn, size_t o, int passWn = 0) {
  PLayout L;
  if (passWn <= 0) passWn = Wn;
  const size_t B = p->B, C = p->C, K = p->K;
  const PostGeo q = post_geo(p, prec, Wn);
  const int d = cut_spacing();
  L.logZb = o; o += al(B * 8);
  L.tot = o;   o += al(B * q.nch * C * 8);
  L.cntp = o;  o += al(B * q.nch * 8);
  L.gTp = o;   o += al(B * q.nch * C * C * 8);
  L.gBp = o;   o += al(B * q.nchB * K * C * 8);
  // (windowed full-mode passes keep each window's cut slots apart: 2 extra slots per window)
  const size_t xslots = passWn < Wn ? 2 * ((size_t)Wn / kGBMicro + 2) : 0;
  L.cutU = o;  o += d > 0 ? al(B * ((size_t)cut_slots(0, Wn, d) + xslots) * C * 8) : 0;
  L.corr = o;  o += d > 0 ? al(B * (size_t)Wn * 8) : 0;
  L.carry = o; o += al(B * C * 8);
  L.clamp = o; o += al(B * 4);
  L.accT = o;  o += al(B * C * C * 8);
  L.accB = o;  o += al(B * K * C * 8);
  L.accN = o;  o += al(B * 8);
  L.Zt = o;    o += al(B * 8);
  L.tcut = o;  o += al(B * 4);
  L.prog = o;  o += al(B * 2 * kProgSlots * 4);
  L.status = o; o += al(4);
  L.prepNR = passWn + 2 * (int)K - 1;
  L.nprep = passWn < Wn ? 2 : 1;  // windowed: one set per side stream
  L.RA = o;    o += al(B * C * (size_t)L.prepNR * 8 * L.nprep);
  L.RB = o;    o += al(B * C * (size_t)L.prepNR * 8 * L.nprep);
  L.Wt = o;    o += al(C * (2 * K + 2 * kCutEC) * 8);
  L.Bmax = o;  o += al(C * 8);
  L.total = o;
  return L;
}

// full-mode backward work buffer: beta-side messages + pass buffers
struct BLayout {
  size_t Y, X, n, total;
  PLayout P;
};
BLayout b_layout(const scrf_problem* p, int prec) {
  BLayout L;
  const size_t rs = prec ? 8 : 4;
  const size_t C = p->C;
  const size_t npos = (size_t)p->B * (p->T + 1);
  size_t o = 0;
  L.Y = o; o += al(npos * C * rs);
  L.X = o; o += al(npos * C * rs);
  L.n = o; o += al(npos * 8);
  // windowed passes (ovl_mode >= 0) need pass rows for one window only
  L.P = p_layout(p, prec, (int)p->T + 1, o, ovl_mode(p) >= 0 ? ovl_ws() : (int)p->T + 1);
  L.total = L.P.total;
  return L;
}

// windows replayed per launch (sublinear mode): enough clusters to fill the chip once
int win_par(const scrf_problem* p, int G, int nWin) {
  int P = env_int("SCRF_WIN_PAR", 0);
  if (P <= 0) {
    P = num_sms() / (2 * (int)p->B * G);
    if (P < 1) P = 1;
  }
  return P < nWin ? P : nWin;
}

// sparse backward work: beta checkpoint rows, replay window buffers (alpha and beta sides),
// replay tasks, pass buffers
struct WLayout {
  size_t bY, bn, aY, aX, an, wY, wX, wn, tasks, total;
  PLayout P;
  SparseGeo g;
  int Pw;
};
WLayout w_layout(const scrf_problem* p, int64_t delta, int prec, int G) {
  WLayout L;
  const size_t rs = prec ? 8 : 4;
  const size_t B = p->B, C = p->C;
  L.g = sparse_geo(p, delta);
  L.Pw = win_par(p, G, L.g.nWin);
  const size_t rb = B * (size_t)L.g.rowsBeta;
  // two sets of window rows: the posterior passes of one replay launch run on a side stream
  // while the next launch replays into the other set (run_sparse_post)
  const size_t rw = (size_t)2 * L.Pw * B * L.g.rowsWin;
  size_t o = 0;
  L.bY = o;    o += al((rb ? rb : 1) * C * rs);
  L.bn = o;    o += al((rb ? rb : 1) * 8);
  L.aY = o;    o += al(rw * C * rs);
  L.aX = o;    o += al(rw * C * rs);
  L.an = o;    o += al(rw * 8);
  L.wY = o;    o += al(rw * C * rs);
  L.wX = o;    o += al(rw * C * rs);
  L.wn = o;    o += al(rw * 8);
  L.tasks = o; o += al((size_t)2 * L.Pw * B * sizeof(SweepTask));
  L.P = p_layout(p, prec, L.g.W, o);
  L.total = L.P.total;
  return L;
}

// Cluster launch with one CTA per SM: the recurrence CTAs are latency bound, and a second
// resident CTA (another cluster's tail) would share their issue slots, so the dynamic shared
// memory request is padded past half of the SM's capacity.
template <typename Kern, typename ArgT>
cudaError_t launch_cl(Kern kern, int G, int nclusters, int NT, size_t smem, cudaStream_t st, ArgT arg, bool record) {
  const size_t half = (size_t)smem_optin() / 2 + 1024;
  if (smem < half && !env_int("SCRF_NO_PAD", 0)) smem = half;
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

// What one sweep launch reads and writes (untyped; run_sweep casts to the working type).
struct SweepIO {
  int dirs;                  // 1 alpha, 2 beta, 3 both (no tasks)
  int store;                 // 0 every position at row b*(T+1)+t; 1 checkpoint rows
  void* Y[2];
  void* X[2];
  double* n[2];
  const SweepTask* tasks;    // replay mode
  int ntasks;
  const void* fY[2];
  const double* fN[2];
  double* logZ;
  double* logZb;
  double* N;
  int32_t* dead_at;
  int32_t* clamp;
  void* amx;                 // full-mode alpha: per-position max shift (book_kernel input)
  int* prog;                 // full mode: row progress for the overlapped passes (or null)
  bool record;               // profiling events around this launch
};

template <typename R>
int sweep_geo_of(const scrf_problem* p, SweepGeo* g) {
  // geometry from (B, both directions) in every mode so that replays use the pass-1 geometry
  return choose_sweep_geo((int)p->B, (int)p->K, (int)p->C, sizeof(R) == 8, 2, p->proj_start != nullptr,
                          p->proj_end != nullptr, g);
}

template <typename R>
int run_sweep(const scrf_problem* p, int64_t delta, const SweepIO& io, cudaStream_t st) {
  SweepGeo g;
  int rc = io.dirs == 3 || io.tasks || io.store ? sweep_geo_of<R>(p, &g)
                                    : choose_sweep_geo((int)p->B, (int)p->K, (int)p->C, sizeof(R) == 8, 1,
                                                       p->proj_start != nullptr, p->proj_end != nullptr, &g);
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
  a.dirs = io.dirs;
  for (int d = 0; d < 2; ++d) {
    a.Y[d] = (R*)io.Y[d];
    a.X[d] = (R*)io.X[d];
    a.n[d] = io.n[d];
    a.fY[d] = (const R*)io.fY[d];
    a.fN[d] = io.fN[d];
  }
  a.logZ = io.logZ;
  a.logZb = io.logZb;
  a.dead_at = io.dead_at;
  a.N = io.N;
  a.clamp = io.store == 1 ? io.clamp : nullptr;
  a.amx = (R*)io.amx;
  a.delta = (int)delta;
  a.n_ckpt = (int)n_ckpt_of(p->T, delta);
  a.store = io.store;
  if (io.store == 1 || io.tasks) {
    const SparseGeo sg = sparse_geo(p, delta);
    a.mA = sg.mA;
    a.W = sg.W;
    a.nW = sg.nW;
  }
  a.tasks = io.tasks;
  a.prog = io.prog;
  if (!io.tasks && io.store == 0 && g_gate) {
    a.gate = g_gate;
    a.gate_shift = g_gate_shift;
    a.ngate = g_gate_n;
  }
  a.trace = g_trace;
  a.trace_from = env_int("SCRF_TRACE_FROM", 64);
  if (env_int("SCRF_WATCHDOG", 0)) {
    if (!g_hang) {
      cudaMallocManaged(&g_hang, 8 * sizeof(int));
      memset(g_hang, 0, 8 * sizeof(int));
    }
    a.hang = g_hang;
  }
  const int ncl = io.tasks ? io.ntasks : a.B * (io.dirs == 3 ? 2 : 1);
  const size_t smem = sweep_smem_bytes<R>(a.K, a.C, g);
  const bool tails = g.G > 1, cw1 = g.NCW == 1;
  cudaError_t e;
  const int mode = io.tasks ? 2 : (io.store ? 1 : (a.gate ? 3 : 0));  // 3: full mode, streamed input
#define SCRF_LAUNCH_SWEEP(M)                                                                              \
  (tails && cw1 ? launch_cl(sweep_kernel<R, true, true, M>, g.G, ncl, g.NT, smem, st, a, io.record)      \
   : tails    ? launch_cl(sweep_kernel<R, true, false, M>, g.G, ncl, g.NT, smem, st, a, io.record)     \
   : cw1      ? launch_cl(sweep_kernel<R, false, true, M>, g.G, ncl, g.NT, smem, st, a, io.record)     \
              : launch_cl(sweep_kernel<R, false, false, M>, g.G, ncl, g.NT, smem, st, a, io.record))
  e = mode == 2   ? SCRF_LAUNCH_SWEEP(2)
      : mode == 1 ? SCRF_LAUNCH_SWEEP(1)
      : mode == 3 ? SCRF_LAUNCH_SWEEP(3)
                  : SCRF_LAUNCH_SWEEP(0);
#undef SCRF_LAUNCH_SWEEP
  if (e != cudaSuccess) return (int)e;
  if (!io.tasks && io.store == 0 && (io.dirs & 1)) {
    // full mode: the reference bookkeeping of the alpha sweep from the stored rows
    ++g_launches;
    book_kernel<R><<<a.B, 1024, 0, st>>>(a.Y[0], a.n[0], a.amx, p->lengths, a.T, a.C, a.delta, a.n_ckpt, a.N,
                                        a.dead_at, a.logZ, io.clamp);
    e = cudaGetLastError();
  }
  return (int)e;
}

// message rows a posterior pass reads
struct MsgView {
  const void *Ya, *Xa, *Yb, *Xb;
  const double *na, *nb;
  int rowsA, tA0, rowsB, tB0;
};

struct PostOut {
  const double* logZ;
  const double* upstream;
  double *grad_S, *grad_T, *grad_B, *gPs, *gPe, *pos, *bnd, *cnt;
};

// running per-sequence sums of the pass partials, in a fixed order (pass order, then part order)
__global__ void acc_kernel(int B, int n, int nparts, const double* parts, double* acc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * n) return;
  const int b = i / n, k = i % n;
  double s = 0.0;
  for (int q = 0; q < nparts; ++q) s += parts[((size_t)b * nparts + q) * n + k];
  acc[i] += s;
}

// One posterior pass over positions [w0, w1): cut normalisers, frame correction, masses /
// grad_S / grad_P / boundary / coverage (re-anchored at the cuts), grad_T, grad_B, and the
// accumulation of the pass's transition / duration / count partials.
// How a pass places its partials. Default (sublinear windows, single full pass): pass-local
// partial arrays summed into the running accumulators at the end of the pass. Sequence-wide
// (full-mode windows): the pass writes its chunks of sequence-wide partial arrays and the sums
// run once after the last window (acc_parts), in the same order as one single pass.
struct PassOpt {
  const double* Z = nullptr;  // log Z reference of the masses (null: PostOut::logZ)
  bool seqwide = false;
  int pnch = 0, pnchB = 0;    // sequence-wide chunk / micro-chunk counts
  cudaEvent_t pos_ev = nullptr;  // recorded once this pass's per-position outputs are final
  // scratch placement of concurrent windows (doubles): frame correction, chunk totals, cut
  // slots; RA / RB set; duration weights of the cut kernel already in place (cut_w_kernel)
  size_t corr_off = 0, tot_off = 0, cut_off = 0;
  int prep_set = 0;
  bool w_ready = false;
};

template <typename R>
int run_pass(const scrf_problem* p, const MsgView& m, int w0, int w1, const PostOut& out, unsigned char* wb,
             const PLayout& PL, bool last, cudaStream_t st, const PassOpt& opt = PassOpt()) {
  const int Wn = w1 - w0;
  const PostGeo q = post_geo(p, sizeof(R) == 8, Wn);
  PostArgs<R> a;
  memset(&a, 0, sizeof(a));
  a.S = p->S;
  a.lengths = p->lengths;
  a.trans = p->transition;
  a.dur = p->duration_bias;
  a.ps = p->proj_start;
  a.pe = p->proj_end;
  a.upstream = out.upstream;
  a.logZ = opt.Z ? opt.Z : out.logZ;
  a.B = (int)p->B;
  a.T = (int)p->T;
  a.K = (int)p->K;
  a.C = (int)p->C;
  a.Ya = (const R*)m.Ya;
  a.Xa = (const R*)m.Xa;
  a.na = m.na;
  a.Yb = (const R*)m.Yb;
  a.Xb = (const R*)m.Xb;
  a.nb = m.nb;
  a.rowsA = m.rowsA;
  a.tA0 = m.tA0;
  a.rowsB = m.rowsB;
  a.tB0 = m.tB0;
  a.w0 = w0;
  a.w1 = w1;
  a.grad_S = out.grad_S;
  a.grad_Ps = out.gPs;
  a.grad_Pe = out.gPe;
  a.pos = out.pos;
  a.bnd = out.bnd;
  a.CH = q.CH;
  a.nch = q.nch;
  a.tot = (double*)(wb + PL.tot) + opt.tot_off;
  a.cntp = (double*)(wb + PL.cntp);
  a.gTp = (double*)(wb + PL.gTp);
  a.SCB = q.SCB;
  a.nchB = q.nchB;
  a.CGB = q.CGB;
  a.gBp = (double*)(wb + PL.gBp);
  if (opt.seqwide) {
    if (w0 % q.CH || w0 % kGBMicro) return SCRF_ECONFIG;
    a.pq0 = w0 / q.CH;
    a.pnch = opt.pnch;
    a.pm0 = w0 / kGBMicro;
    a.pnchB = opt.pnchB;
  } else {
    a.pq0 = 0;
    a.pnch = q.nch;
    a.pm0 = 0;
    a.pnchB = q.nchB;
  }
  a.gb_range = (float)env_int("SCRF_GB_RANGE", (int)kGBRange);
  const int B = a.B, C = a.C, K = a.K;
  cudaError_t e;
  // the pass's source / target values, once (shared by the cut and grad_B kernels)
  a.t_lo = w0 - K + 1;
  a.NR = Wn + 2 * K - 1;
  if (a.NR > PL.prepNR) return SCRF_EWORK;
  if (opt.prep_set >= PL.nprep) return SCRF_EWORK;
  a.RA = (double*)(wb + PL.RA) + (size_t)opt.prep_set * B * C * PL.prepNR;
  a.RB = (double*)(wb + PL.RB) + (size_t)opt.prep_set * B * C * PL.prepNR;
  {
    const size_t sm = post_prep_smem(C);
    e = cudaFuncSetAttribute(post_prep_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    post_prep_kernel<R><<<dim3((a.NR + kPrepRows - 1) / kPrepRows, B), 256, sm, st>>>(a);
  }
  const int cd = cut_spacing();
  const int ncut = cut_slots(w0, w1, cd);
  if (cd > 0) {
    if (!opt.w_ready) {
      ++g_launches;
      cut_w_kernel<R><<<C, 256, 0, st>>>(p->duration_bias, K, C, (R*)(wb + PL.Wt), (double*)(wb + PL.Bmax));
    }
    CutArgs<R> ca;
    memset(&ca, 0, sizeof(ca));
    ca.S = p->S;
    ca.lengths = p->lengths;
    ca.dur = p->duration_bias;
    ca.ps = p->proj_start;
    ca.pe = p->proj_end;
    ca.logZ = a.logZ;
    ca.B = B;
    ca.T = a.T;
    ca.K = K;
    ca.C = C;
    ca.Ya = a.Ya;
    ca.Xa = a.Xa;
    ca.Yb = a.Yb;
    ca.Xb = a.Xb;
    ca.na = a.na;
    ca.nb = a.nb;
    ca.rowsA = m.rowsA;
    ca.tA0 = m.tA0;
    ca.rowsB = m.rowsB;
    ca.tB0 = m.tB0;
    ca.w0 = w0;
    ca.w1 = w1;
    ca.d = cd;
    ca.ncut = ncut;
    ca.U = (double*)(wb + PL.cutU) + opt.cut_off;
    ca.RA = a.RA;
    ca.RB = a.RB;
    ca.t_lo = a.t_lo;
    ca.NR = a.NR;
    ca.Wt = (const R*)(wb + PL.Wt);
    ca.Bmax = (const double*)(wb + PL.Bmax);
    const size_t sm = cut_smem<R>(K);
    e = cudaFuncSetAttribute(cut_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    cut_kernel<R><<<dim3(ncut, (C + kCutCG - 1) / kCutCG, B), 256, sm, st>>>(ca);
    a.corr = (const double*)(wb + PL.corr) + opt.corr_off;
  }
  // per-position frame correction (when enabled) and the beta-side clamp-event count
  ++g_launches;
  cut_corr_kernel<R><<<dim3((Wn + 255) / 256, B), 256, 0, st>>>(
      p->lengths, C, w0, w1, cd, ncut, cd > 0 ? (const double*)(wb + PL.cutU) + opt.cut_off : nullptr,
      cd > 0 ? (double*)(wb + PL.corr) + opt.corr_off : nullptr, a.Xb, a.nb, m.rowsB, m.tB0, (int32_t*)(wb + PL.clamp));
  {
    const size_t sm = post_pos_smem<R>(C, q.CH);
    e = cudaFuncSetAttribute(post_pos_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    post_pos_kernel<R><<<dim3(q.nch, B), 256, sm, st>>>(a);
    ++g_launches;
    if (cd > 0 && cd % q.CH == 0)
      cut_prefix_kernel<<<(B * C + 127) / 128, 128, 0, st>>>(p->lengths, B, C, q.nch, q.CH, w0, w1, cd, ncut,
                                                           (const double*)(wb + PL.cutU) + opt.cut_off, a.tot,
                                                           opt.seqwide ? nullptr : (double*)(wb + PL.carry));
    else if (w0 == 0 && !opt.seqwide)
      post_prefix_kernel<<<(B * C + 7) / 8, 256, 0, st>>>(B, C, q.nch, a.tot);
    else
      return SCRF_ECONFIG;  // windowed passes need the cut normalisers
    ++g_launches;
    post_carry_kernel<<<dim3(q.nch, B), 64, 0, st>>>(p->lengths, B, a.T, C, q.CH, q.nch, w0, w1, a.tot, out.pos);
    if (last && g_ev_pos) cudaEventRecord(g_ev_pos, st);
    if (opt.pos_ev) cudaEventRecord(opt.pos_ev, st);
  }
  if (sizeof(R) == 4 && gradB_blocked()) {
    if ((long long)q.CGB * gbb_npass(K) > 32) return SCRF_ECONFIG;
    const size_t sm = post_gradB_blk_smem(K, q.CGB);
    e = cudaFuncSetAttribute(post_gradB_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    post_gradB_blk_kernel<<<dim3((q.nchB * kGBMicro + q.SCB - 1) / q.SCB, (C + q.CGB - 1) / q.CGB, B), 512, sm, st>>>(
        *reinterpret_cast<const PostArgs<float>*>(&a));
  } else {
    // one CTA holds every duration window of its label group (K <= kGBW * 512 * kGBJ = 4096)
    if ((long long)q.CGB * ((K + kGBJ - 1) / kGBJ) > (long long)kGBW * 512) return SCRF_ECONFIG;
    const size_t sm = post_gradB_smem<R>(K, q.CGB);
    e = cudaFuncSetAttribute(post_gradB_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    post_gradB_kernel<R><<<dim3((q.nchB * kGBMicro + q.SCB - 1) / q.SCB, (C + q.CGB - 1) / q.CGB, B), 512, sm, st>>>(a);
  }
  if (!opt.seqwide) {
    const int nT = C * C, nB = K * C;
    ++g_launches;
    acc_kernel<<<(B * nT + 255) / 256, 256, 0, st>>>(B, nT, q.nch, a.gTp, (double*)(wb + PL.accT));
    ++g_launches;
    acc_kernel<<<(B * nB + 255) / 256, 256, 0, st>>>(B, nB, q.nchB, a.gBp, (double*)(wb + PL.accB));
    ++g_launches;
    acc_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, 1, q.nch, a.cntp, (double*)(wb + PL.accN));
  }
  return (int)cudaGetLastError();
}

// zero the running accumulators / clamp counts before the first pass
int pass_begin(const scrf_problem* p, unsigned char* wb, const PLayout& PL, cudaStream_t st) {
  const size_t B = p->B, C = p->C, K = p->K;
  cudaError_t e = cudaMemsetAsync(wb + PL.accT, 0, B * C * C * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(wb + PL.accB, 0, B * K * C * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(wb + PL.accN, 0, B * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(wb + PL.clamp, 0, B * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(wb + PL.carry, 0, B * C * 8, st);
  return (int)e;
}

// batch totals (upstream-weighted, fixed order) of the accumulated partials
int pass_finish(const scrf_problem* p, unsigned char* wb, const PLayout& PL, const PostOut& out, cudaStream_t st) {
  const int B = (int)p->B, C = (int)p->C, K = (int)p->K;
  const int nT = C * C, nB = K * C;
  ++g_launches;
  post_reduce2_kernel<<<(nT + 31) / 32, 256, 0, st>>>(B, nT, 1, (const double*)(wb + PL.accT), out.upstream, nullptr,
                                                     out.grad_T);
  ++g_launches;
  post_reduce2_kernel<<<(nB + 31) / 32, 256, 0, st>>>(B, nB, 1, (const double*)(wb + PL.accB), out.upstream, nullptr,
                                                     out.grad_B);
  ++g_launches;
  post_count_kernel<<<(B + 127) / 128, 128, 0, st>>>(B, 1, (const double*)(wb + PL.accN), out.cnt);
  return (int)cudaGetLastError();
}

template <typename R>
int run_full_post(const scrf_problem* p, const void* fstate, void* work, const PostOut& out, cudaStream_t st) {
  const FLayout F = f_layout(p, sizeof(R) == 8);
  const BLayout W = b_layout(p, sizeof(R) == 8);
  const unsigned char* fb = (const unsigned char*)fstate;
  unsigned char* wb = (unsigned char*)work;
  MsgView m;
  m.Ya = fb + F.Y;
  m.Xa = fb + F.X;
  m.na = (const double*)(fb + F.n);
  m.Yb = wb + W.Y;
  m.Xb = wb + W.X;
  m.nb = (const double*)(wb + W.n);
  m.rowsA = m.rowsB = (int)p->T + 1;
  m.tA0 = m.tB0 = 0;
  int rc = pass_begin(p, wb, W.P, st);
  if (rc) return rc;
  rc = run_pass<R>(p, m, 0, (int)p->T + 1, out, wb, W.P, true, st);
  if (rc) return rc;
  return pass_finish(p, wb, W.P, out, st);
}

// ---------------------------------------------------------------------------
// Full mode, windowed posterior passes overlapped with the sweeps.
//
// Position t has both of its messages once the alpha sweep has passed t and the beta sweep has
// come down to t, so a window [w0, w1) can run its pass once alpha is through w1 and beta
// through w0 -- for windows around the middle, while the sweeps are still working on the rest
// of the sequence. The sweep clusters occupy one CTA on 4 B SMs; the passes run on a second
// (low-priority) stream on the remaining SMs, each window behind prog_wait_kernel, which spins
// on the row progress the sweeps' writer warps publish (SweepArgs::prog). The final log Z is not
// known until the sweeps end, so the masses use a provisional log Z from one cut normaliser at
// the middle of each sequence (probe_finish_kernel); the cut normalisers divide it out again
// (scrf_cut.cuh). Windows are aligned to 4096 positions, so every chunk / micro-chunk / cut is
// the one a single pass over [0, T] uses, and the transition / duration / count partials are
// kept sequence-wide and summed once at the end in the single-pass order: the result does not
// depend on the window size or on whether the windows ran concurrently (SCRF_OVERLAP=0 runs the
// same windows after the sweeps, for the bit-identity test).


// one CTA: returns once every swept direction of every sequence has published its rows through
// alpha t <= tA / beta t >= tB (probe: the probe cut of each sequence). Gives up after 20 s
// (sets *status), so a broken sweep cannot hang the stream.
__global__ void prog_wait_kernel(const int* prog, const int64_t* lengths, int B, int nw, int dirs, int tA, int tB,
                                 int probe_d, int* status) {
  for (int i = threadIdx.x; i < 2 * B; i += blockDim.x) {
    const int b = i >> 1, dir = i & 1;
    if (!((dirs >> dir) & 1)) continue;
    const int L = (int)lengths[b];
    int a0 = tA, b0 = tB;
    if (probe_d > 0) a0 = b0 = probe_pos(L, probe_d);
    const int need = dir == 0 ? min(L, max(a0, 0)) + 1 : L - min(L, max(b0, 0)) + 1;
    const int* sl = prog + (size_t)i * kProgSlots;
    const long long t0 = gtimer();
    for (;;) {
      int mn = 0x7fffffff;
      for (int w = 0; w < nw; ++w) mn = min(mn, ld_acquire_i32(sl + w));
      if (mn >= need) break;
      if (gtimer() - t0 > 20000000000LL) {
        atomicExch(status, 1);
        break;
      }
      __nanosleep(500);
    }
  }
}

struct OvlWin {
  int w0, w1;
  long long ready;
};

// windows of [0, T] in the order the sweeps complete them
int ovl_windows(const scrf_problem* p, OvlWin* w, int cap) {
  const int ws = ovl_ws();
  const int T = (int)p->T;
  int n = 0;
  for (int w0 = 0; w0 <= T && n < cap; w0 += ws) {
    const int w1 = w0 + ws < T + 1 ? w0 + ws : T + 1;
    w[n].w0 = w0;
    w[n].w1 = w1;
    w[n].ready = (long long)(w1 > T - w0 ? w1 : T - w0) * 2 + (w0 > T / 2 ? 1 : 0);
    ++n;
  }
  for (int i = 1; i < n; ++i)  // insertion sort by completion step
    for (int j = i; j > 0 && w[j].ready < w[j - 1].ready; --j) {
      const OvlWin t = w[j];
      w[j] = w[j - 1];
      w[j - 1] = t;
    }
  return n;
}

// writer warps per sweep cluster (SweepArgs::prog slots): output + source warp, or the source warps
int prog_writers(int C) { return C <= 32 ? 2 : (C + 31) / 32; }

// two low-priority side streams per device: the windows left and right of the middle run on
// their own streams (independent scratch), so the passes of both flanks overlap each other too
struct SideStream {
  cudaStream_t s[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr, probe = nullptr, join[2] = {nullptr, nullptr};
  cudaEvent_t sp_rep[2] = {nullptr, nullptr}, sp_pass[2] = {nullptr, nullptr};  // sublinear passes
};
SideStream& side_stream() {
  static SideStream ss[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& x = ss[dev & 63];
  if (!x.s[0]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (int i = 0; i < 2; ++i) {
      cudaStreamCreateWithPriority(&x.s[i], cudaStreamNonBlocking, lo);
      cudaEventCreateWithFlags(&x.join[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&x.sp_rep[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&x.sp_pass[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.probe, cudaEventDisableTiming);
  }
  return x;
}

__global__ void gate_set_kernel(int* gate, int j) {
  __threadfence();
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(gate + j), "r"(1) : "memory");
}

// Under lazy module loading (torch's default) the first launch of a kernel loads it, and the
// load waits for the kernels running on the device: a kernel that a running sweep waits on
// (gate_set_kernel) would deadlock, and the overlapped passes would serialise behind the sweep.
// Load every kernel those paths launch up front.
template <typename R>
void preload_post_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, probe_finish_kernel<R>);
  cudaFuncGetAttributes(&fa, cut_kernel<R>);
  cudaFuncGetAttributes(&fa, cut_w_kernel<R>);
  cudaFuncGetAttributes(&fa, cut_corr_kernel<R>);
  cudaFuncGetAttributes(&fa, post_prep_kernel<R>);
  cudaFuncGetAttributes(&fa, post_pos_kernel<R>);
  cudaFuncGetAttributes(&fa, post_gradB_kernel<R>);
  cudaFuncGetAttributes(&fa, book_kernel<R>);
}
void preload_concurrent_kernels() {
  static bool done = false;
  if (done) return;
  done = true;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gate_set_kernel);
  cudaFuncGetAttributes(&fa, prog_wait_kernel);
  cudaFuncGetAttributes(&fa, probe_pos_kernel);
  cudaFuncGetAttributes(&fa, cut_prefix_kernel);
  cudaFuncGetAttributes(&fa, post_prefix_kernel);
  cudaFuncGetAttributes(&fa, post_carry_kernel);
  cudaFuncGetAttributes(&fa, post_gradB_blk_kernel);
  cudaFuncGetAttributes(&fa, acc_kernel);
  cudaFuncGetAttributes(&fa, post_reduce2_kernel);
  cudaFuncGetAttributes(&fa, post_count_kernel);
  preload_post_kernels<float>();
  preload_post_kernels<double>();
}

// before the sweeps: zero the accumulators and the progress slots, fork the side stream
int ovl_begin(const scrf_problem* p, unsigned char* wb, const PLayout& PL, int mode, cudaStream_t st) {
  preload_concurrent_kernels();
  int rc = pass_begin(p, wb, PL, st);
  if (rc) return rc;
  cudaError_t e = cudaMemsetAsync(wb + PL.prog, 0, (size_t)p->B * 2 * kProgSlots * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(wb + PL.status, 0, 4, st);
  if (e == cudaSuccess && mode == 1) {
    SideStream& ss = side_stream();
    if (!ss.s[0] || !ss.s[1]) return (int)cudaErrorUnknown;
    e = cudaEventRecord(ss.fork, st);
  }
  return (int)e;
}

template <typename R>
int fill_cut_args(const scrf_problem* p, const MsgView& m, const double* Z, CutArgs<R>* ca) {
  memset(ca, 0, sizeof(*ca));
  ca->S = p->S;
  ca->lengths = p->lengths;
  ca->dur = p->duration_bias;
  ca->ps = p->proj_start;
  ca->pe = p->proj_end;
  ca->logZ = Z;
  ca->B = (int)p->B;
  ca->T = (int)p->T;
  ca->K = (int)p->K;
  ca->C = (int)p->C;
  ca->Ya = (const R*)m.Ya;
  ca->Xa = (const R*)m.Xa;
  ca->Yb = (const R*)m.Yb;
  ca->Xb = (const R*)m.Xb;
  ca->na = m.na;
  ca->nb = m.nb;
  ca->rowsA = m.rowsA;
  ca->tA0 = m.tA0;
  ca->rowsB = m.rowsB;
  ca->tB0 = m.tB0;
  return 0;
}

// the windowed passes (after ovl_begin and the sweep launch on st); dirs = the directions the
// sweep in flight computes (their progress is waited on in mode 1)
template <typename R>
int run_full_post_win(const scrf_problem* p, const void* fstate, void* work, const PostOut& out, int mode, int dirs,
                      cudaStream_t st) {
  const FLayout F = f_layout(p, sizeof(R) == 8);
  const BLayout W = b_layout(p, sizeof(R) == 8);
  const unsigned char* fb = (const unsigned char*)fstate;
  unsigned char* wb = (unsigned char*)work;
  MsgView m;
  m.Ya = fb + F.Y;
  m.Xa = fb + F.X;
  m.na = (const double*)(fb + F.n);
  m.Yb = wb + W.Y;
  m.Xb = wb + W.X;
  m.nb = (const double*)(wb + W.n);
  m.rowsA = m.rowsB = (int)p->T + 1;
  m.tA0 = m.tB0 = 0;
  const int B = (int)p->B, C = (int)p->C;
  const int d = cut_spacing();
  const PostGeo qall = post_geo(p, sizeof(R) == 8, (int)p->T + 1);
  // mode 1: windows left / right of the middle on side streams 0 / 1; mode 0: all on st
  cudaStream_t sw[2] = {st, st};
  SideStream* ss = nullptr;
  if (mode == 1) {
    ss = &side_stream();
    sw[0] = ss->s[0];
    sw[1] = ss->s[1];
    cudaError_t e = cudaStreamWaitEvent(sw[0], ss->fork, 0);
    if (e != cudaSuccess) return (int)e;
  }
  const int nw = prog_writers(C);
  int* status = (int*)(wb + W.P.status);
  // provisional log Z from the middle cut of each sequence, and the cut kernel's duration
  // weights, on side stream 0; side stream 1 starts after them
  if (mode == 1) {
    ++g_launches;
    prog_wait_kernel<<<1, 256, 0, sw[0]>>>((const int*)(wb + W.P.prog), p->lengths, B, nw, dirs, 0, 0, d, status);
  }
  ++g_launches;
  probe_pos_kernel<<<(B + 127) / 128, 128, 0, sw[0]>>>(p->lengths, B, d, (int*)(wb + W.P.tcut));
  {
    CutArgs<R> ca;
    fill_cut_args<R>(p, m, nullptr, &ca);
    ca.d = d;
    ca.ncut = 1;
    ca.U = (double*)(wb + W.P.cutU);
    ca.tcut = (const int*)(wb + W.P.tcut);
    const size_t sm = cut_smem<R>((int)p->K);
    cudaError_t e = cudaFuncSetAttribute(cut_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return (int)e;
    ++g_launches;
    cut_kernel<R><<<dim3(1, (C + kCutCG - 1) / kCutCG, B), 256, sm, sw[0]>>>(ca);
  }
  ++g_launches;
  probe_finish_kernel<R><<<(B + 127) / 128, 128, 0, sw[0]>>>(p->lengths, B, C, (const int*)(wb + W.P.tcut), m.na, m.nb,
                                                           m.rowsA, m.tA0, m.rowsB, m.tB0,
                                                           (const double*)(wb + W.P.cutU), (double*)(wb + W.P.Zt));
  ++g_launches;
  cut_w_kernel<R><<<C, 256, 0, sw[0]>>>(p->duration_bias, (int)p->K, C, (R*)(wb + W.P.Wt), (double*)(wb + W.P.Bmax));
  if (mode == 1) {
    cudaError_t e = cudaEventRecord(ss->probe, sw[0]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sw[1], ss->probe, 0);
    if (e != cudaSuccess) return (int)e;
  }
  OvlWin win[4096];
  const int nwin = ovl_windows(p, win, 4096);
  const int ws = ovl_ws();
  PassOpt opt;
  opt.Z = (const double*)(wb + W.P.Zt);
  opt.seqwide = true;
  opt.pnch = qall.nch;
  opt.pnchB = qall.nchB;
  opt.w_ready = true;
  for (int i = 0; i < nwin; ++i) {
    const int w0 = win[i].w0, w1 = win[i].w1;
    const int side = (long long)(w0 + w1) > (long long)p->T + 1 ? 1 : 0;
    opt.pos_ev = i < g_win_nev ? g_win_ev[i] : nullptr;
    // disjoint scratch per window (positions, chunks and cut slots of the window itself)
    opt.corr_off = (size_t)B * w0;
    opt.tot_off = (size_t)(w0 / qall.CH) * B * C;
    opt.cut_off = (size_t)(w0 / d + 2 * (w0 / ws)) * B * C;
    opt.prep_set = side;
    if (mode == 1) {
      ++g_launches;
      prog_wait_kernel<<<1, 256, 0, sw[side]>>>((const int*)(wb + W.P.prog), p->lengths, B, nw, dirs, w1 + 1,
                                                w0 - 1, 0, status);
    }
    int rc = run_pass<R>(p, m, w0, w1, out, wb, W.P, false, sw[side], opt);
    if (rc) return rc;
  }
  if (mode == 1) {
    for (int i = 0; i < 2; ++i) {
      cudaError_t e = cudaEventRecord(ss->join[i], sw[i]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ss->join[i], 0);
      if (e != cudaSuccess) return (int)e;
    }
  }
  if (g_ev_pos) cudaEventRecord(g_ev_pos, st);  // every window's per-position outputs are final
  // the sequence-wide sums, in the single-pass order
  const int nT = C * C, nB = (int)p->K * C;
  ++g_launches;
  acc_kernel<<<(B * nT + 255) / 256, 256, 0, st>>>(B, nT, qall.nch, (const double*)(wb + W.P.gTp),
                                                   (double*)(wb + W.P.accT));
  ++g_launches;
  acc_kernel<<<(B * nB + 255) / 256, 256, 0, st>>>(B, nB, qall.nchB, (const double*)(wb + W.P.gBp),
                                                   (double*)(wb + W.P.accB));
  ++g_launches;
  acc_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, 1, qall.nch, (const double*)(wb + W.P.cntp),
                                              (double*)(wb + W.P.accN));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  return pass_finish(p, wb, W.P, out, st);
}

// replay tasks of windows j0 .. j0+P-1 (all sequences, both directions); see SweepTask
__global__ void build_tasks_kernel(const int64_t* lengths, const double* N, int B, int T, int K, int delta, int n_ckpt,
                                   int mA, int W, int nW, long long rowsAlpha, int rowsWin, int j0, int P,
                                   SweepTask* tasks) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * B * P) return;
  const int dir = i & 1, b = (i >> 1) % B, wi = (i >> 1) / B, j = j0 + wi;
  const int L = (int)lengths[b];
  const int w0 = j * W, w1 = min((j + 1) * W, T + 1);
  SweepTask tk;
  tk.b = b;
  tk.dir = dir;
  tk.fstep = 1;
  tk.frow = 0;
  tk.nforce = 0;
  tk.ck_phase = 0;
  tk.n_ref = 0.0;
  tk.out_row = (long long)(wi * B + b) * rowsWin;
  if (w0 > L) {
    tk.t0 = 0;
    tk.steps = -1;
    tk.t_lo = 0;
  } else if (dir == 0) {
    const int tend = min(w1, L);
    const int t0 = j == 0 ? 0 : ((w0 - K + 1) & ~31);
    tk.t0 = t0;
    tk.t_lo = t0;
    tk.steps = tend - t0;
    if (j > 0) {
      tk.nforce = w0 - t0 + 1;
      // checkpoint row of t0 (ck_row, alpha); rows ascend with t over [t0, w0]
      const int ip = (t0 + delta - 1) / delta, e = ip * delta - t0;
      tk.frow = (long long)b * rowsAlpha + (t0 == 0 ? 0 : 1 + (long long)(ip - 1) * mA + (mA - 1 - e));
    }
    tk.ck_phase = t0 % delta;
    tk.n_ref = N[(size_t)b * n_ckpt + t0 / delta] * kLog2e;
  } else {
    tk.t_lo = w0;
    const int ttop = w1 >= L ? L : ck_ttop(j + 1, W, K, L);
    if (ttop == L) {  // the window's beta rows reach L: start at beta[L] = 0 like the full sweep
      tk.t0 = L;
      tk.steps = L - w0;
    } else {
      tk.t0 = ttop;
      tk.steps = ttop - w0;
      tk.nforce = ttop - w1 + 1;
      tk.frow = ((long long)b * nW + j) * (K + 32) + (ttop - w1);
      tk.fstep = -1;
    }
  }
  tasks[i] = tk;
}

// sparse posterior passes: replay windows (P per launch) from the checkpoint rows and run the
// posterior pass of each window
template <typename R>
int run_sparse_post(const scrf_problem* p, int64_t delta, const void* ckpt, const double* N, void* work,
                    const PostOut& out, cudaStream_t st) {
  SweepGeo geo;
  int rc = sweep_geo_of<R>(p, &geo);
  if (rc) return rc;
  const size_t rs = sizeof(R);
  const WLayout WL = w_layout(p, delta, sizeof(R) == 8, geo.G);
  const SLayout SL = s_layout(p, delta, sizeof(R) == 8);
  const SparseGeo& g = WL.g;
  const unsigned char* cb = (const unsigned char*)ckpt;
  unsigned char* wb = (unsigned char*)work;
  const int B = (int)p->B, C = (int)p->C, K = (int)p->K, T = (int)p->T;
  const size_t wstride = (size_t)B * g.rowsWin;  // rows per replayed window
  SweepTask* tasks = (SweepTask*)(wb + WL.tasks);
  rc = pass_begin(p, wb, WL.P, st);
  if (rc) return rc;
  // replay launch i writes window-row set i & 1 on st; its passes run in order on side stream 0
  // (after the launch) while launch i + 1 replays into the other set; launch i + 2 waits for
  // the passes of launch i (set reuse). SCRF_SPARSE_OVL=0: everything on st.
  const bool ovl = env_int("SCRF_SPARSE_OVL", 1) != 0;
  if (ovl) preload_concurrent_kernels();
  SideStream* ss = ovl ? &side_stream() : nullptr;
  cudaStream_t sp = ovl ? ss->s[0] : st;
  if (ovl) {
    cudaError_t e = cudaEventRecord(ss->fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sp, ss->fork, 0);
    if (e != cudaSuccess) return (int)e;
  }
  const size_t setrows = (size_t)WL.Pw * wstride;  // rows of one window-row set
  for (int j0 = 0, bi = 0; j0 < g.nWin; j0 += WL.Pw, ++bi) {
    const int P = g.nWin - j0 < WL.Pw ? g.nWin - j0 : WL.Pw;
    const int set = bi & 1;
    const size_t so = set * setrows;
    if (ovl && bi >= 2) {
      cudaError_t e = cudaStreamWaitEvent(st, ss->sp_pass[set], 0);
      if (e != cudaSuccess) return (int)e;
    }
    ++g_launches;
    build_tasks_kernel<<<(2 * B * P + 127) / 128, 128, 0, st>>>(p->lengths, N, B, T, K, (int)delta,
                                                                (int)n_ckpt_of(p->T, delta), g.mA, g.W, g.nW,
                                                                g.rowsAlpha, g.rowsWin, j0, P, tasks);
    SweepIO io;
    memset(&io, 0, sizeof(io));
    io.dirs = 3;
    io.tasks = tasks;
    io.ntasks = 2 * B * P;
    io.Y[0] = wb + WL.aY + so * C * rs;
    io.X[0] = wb + WL.aX + so * C * rs;
    io.n[0] = (double*)(wb + WL.an) + so;
    io.Y[1] = wb + WL.wY + so * C * rs;
    io.X[1] = wb + WL.wX + so * C * rs;
    io.n[1] = (double*)(wb + WL.wn) + so;
    io.fY[0] = cb + SL.Y;
    io.fN[0] = (const double*)(cb + SL.n);
    io.fY[1] = wb + WL.bY;
    io.fN[1] = (const double*)(wb + WL.bn);
    rc = run_sweep<R>(p, delta, io, st);
    if (rc) return rc;
    if (ovl) {
      cudaError_t e = cudaEventRecord(ss->sp_rep[set], st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(sp, ss->sp_rep[set], 0);
      if (e != cudaSuccess) return (int)e;
    }
    for (int wi = 0; wi < P; ++wi) {
      const int j = j0 + wi;
      const int w0 = j * g.W, w1 = (j + 1) * g.W < T + 1 ? (j + 1) * g.W : T + 1;
      MsgView m;
      const size_t ro = so + (size_t)wi * wstride;
      m.Ya = wb + WL.aY + ro * C * rs;
      m.Xa = wb + WL.aX + ro * C * rs;
      m.na = (const double*)(wb + WL.an) + ro;
      m.Yb = wb + WL.wY + ro * C * rs;
      m.Xb = wb + WL.wX + ro * C * rs;
      m.nb = (const double*)(wb + WL.wn) + ro;
      m.rowsA = m.rowsB = g.rowsWin;
      m.tA0 = j == 0 ? 0 : ((w0 - K + 1) & ~31);
      m.tB0 = w0;
      rc = run_pass<R>(p, m, w0, w1, out, wb, WL.P, j == g.nWin - 1, sp);
      if (rc) return rc;
    }
    if (ovl) {
      cudaError_t e = cudaEventRecord(ss->sp_pass[set], sp);
      if (e != cudaSuccess) return (int)e;
    }
  }
  if (ovl) {
    cudaError_t e = cudaEventRecord(ss->join[0], sp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ss->join[0], 0);
    if (e != cudaSuccess) return (int)e;
  }
  return pass_finish(p, wb, WL.P, out, st);
}

// sparse pass 1: alpha and/or beta sweeps storing checkpoint rows only
template <typename R>
int run_sparse_sweeps(const scrf_problem* p, int64_t delta, int dirs, void* ckpt, void* work, double* logZ,
                      double* N, int32_t* dead_at, cudaStream_t st, bool record) {
  SweepIO io;
  memset(&io, 0, sizeof(io));
  io.dirs = dirs;
  io.store = 1;
  io.record = record;
  if (dirs & 1) {
    const SLayout SL = s_layout(p, delta, sizeof(R) == 8);
    unsigned char* cb = (unsigned char*)ckpt;
    io.Y[0] = cb + SL.Y;
    io.n[0] = (double*)(cb + SL.n);
    io.clamp = (int32_t*)(cb + SL.clamp);
    io.logZ = logZ;
    io.N = N;
    io.dead_at = dead_at;
  }
  if (dirs & 2) {
    SweepGeo geo;
    int rc = sweep_geo_of<R>(p, &geo);
    if (rc) return rc;
    const WLayout WL = w_layout(p, delta, sizeof(R) == 8, geo.G);
    unsigned char* wb = (unsigned char*)work;
    io.Y[1] = wb + WL.bY;
    io.n[1] = (double*)(wb + WL.bn);
    io.logZb = (double*)(wb + WL.P.logZb);
  }
  return run_sweep<R>(p, delta, io, st);
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
// checkpoint view from the sparse alpha rows (same semantics as export_kernel)
template <typename R>
__global__ void export_sparse_kernel(const R* Y, const double* n, const double* N, const int64_t* lengths, int B,
                                     int T, int nck, int K, int C, int delta, int mA, long long rowsAlpha,
                                     double* omega) {
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
  const long long s = e - (((e - slot) % K) + K) % K;
  if (s < 0) {
    omega[i] = kNegInfRef;
    return;
  }
  long long row;
  if (s > L - mA) {
    row = 1 + (long long)((T + delta - 1) / delta) * mA + (s - (L - mA + 1));
  } else if (s == 0) {
    row = 0;
  } else {
    const long long ip = (s + delta - 1) / delta, ee = ip * delta - s;
    row = 1 + (ip - 1) * mA + (mA - 1 - ee);
  }
  row += (long long)b * rowsAlpha;
  const R y = Y[row * C + c];
  if (!(y > -INFINITY)) {
    omega[i] = kNegInfRef;
    return;
  }
  const double v = (n[row] + (double)y) * kLn2 - N[(size_t)b * nck + ck];
  omega[i] = v <= kGuard ? kNegInfRef : v;
}

// forced rows of a recompute_alpha replay: positions tf0 .. t0 from the snapshot's ring slots
// (alpha relative to N_i, nats; values at or below the guard are masked), and the task
template <typename R>
__global__ void ra_prep_kernel(const double* omega, const int64_t* lengths, int B, int K, int C, int t0, int t1,
                               int tf0, int rows, R* fY, double* fN, SweepTask* tasks) {
  const int b = blockIdx.x;
  const int L = (int)lengths[b];
  const double* om = omega + (size_t)b * K * C;
  __shared__ double red[4];
  double nprev = 0.0;
  for (int t = tf0; t <= t0; ++t) {
    const int slot = t % K;
    double m = -CUDART_INF;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      const double v = om[(size_t)slot * C + c];
      if (v > kGuard) m = fmax(m, v);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
    __syncthreads();
    const double nt = m > -CUDART_INF ? m * kLog2e : nprev;
    const size_t r = (size_t)b * K + (t - tf0);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      const double v = om[(size_t)slot * C + c];
      fY[r * C + c] = v > kGuard ? (R)(v * kLog2e - nt) : Mth<R>::ninf();
    }
    if (threadIdx.x == 0) fN[r] = nt;
    nprev = nt;
  }
  if (threadIdx.x == 0) {
    SweepTask tk;
    tk.b = b;
    tk.dir = 0;
    tk.t0 = tf0;
    const int tend = t1 < L ? t1 : L;
    tk.steps = tend > t0 ? tend - tf0 : -1;
    tk.nforce = t0 - tf0 + 1;
    tk.t_lo = tf0;
    tk.fstep = 1;
    tk.frow = (long long)b * K;
    tk.out_row = (long long)b * rows;
    tk.ck_phase = 0;   // delta is passed as 2^30: no checkpoint shift inside a replay window
    tk.n_ref = 0.0;    // snapshot frame: masked at or below the guard relative to N_i
    tasks[b] = tk;
  }
}

// block[b, t - t0, c] (snapshot frame, nats): replayed rows for t <= L; past L the ring slot
// t % K keeps the last position <= L of that slot (replayed, or the snapshot's own)
template <typename R>
__global__ void ra_block_kernel(const double* omega, const int64_t* lengths, int B, int K, int C, int t0, int t1,
                                int tf0, int rows, const R* oY, const double* on, double* block) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = t1 - t0 + 1;
  if (i >= (size_t)B * nt * C) return;
  const int c = (int)(i % C);
  const int j = (int)((i / C) % nt);
  const int b = (int)(i / ((size_t)C * nt));
  const int L = (int)lengths[b];
  int t = t0 + j;
  if (t > L) t -= K * ((t - L + K - 1) / K);
  double v;
  if (j == 0 || t <= t0) {
    v = omega[((size_t)b * K + (t0 + j) % K) * C + c];
  } else {
    const size_t r = (size_t)b * rows + (t - tf0);
    const R y = oY[r * C + c];
    v = (y > Mth<R>::ninf()) ? (on[r] + (double)y) * kLn2 : kNegInfRef;
  }
  block[i] = v;
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

#define SCRF_DISPATCH(prec, call) ((prec) ? call<double> : call<float>)

int scrf_forward(const scrf_problem* p, int64_t delta, int precision, double* logZ, double* N, int32_t* dead_at,
                 void* ckpt, size_t ckpt_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  if (!logZ || !N || !dead_at || !ckpt) return SCRF_ENULL;
  const FLayout F = f_layout(p, precision);
  if (ckpt_bytes < F.total) return SCRF_EWORK;
  unsigned char* fb = (unsigned char*)ckpt;
  SweepIO io;
  memset(&io, 0, sizeof(io));
  io.dirs = 1;
  io.Y[0] = fb + F.Y;
  io.X[0] = fb + F.X;
  io.n[0] = (double*)(fb + F.n);
  io.amx = fb + F.amx;
  io.clamp = (int32_t*)(fb + F.clamp);
  io.logZ = logZ;
  io.N = N;
  io.dead_at = dead_at;
  io.record = true;
  return SCRF_DISPATCH(precision, run_sweep)(p, delta, io, (cudaStream_t)stream);
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

static PostOut post_out(const double* logZ, const double* upstream, double* grad_S, double* grad_T, double* grad_B,
                        double* gPs, double* gPe, double* pos, double* bnd, double* cnt) {
  PostOut o;
  o.logZ = logZ;
  o.upstream = upstream;
  o.grad_S = grad_S;
  o.grad_T = grad_T;
  o.grad_B = grad_B;
  o.gPs = gPs;
  o.gPe = gPe;
  o.pos = pos;
  o.bnd = bnd;
  o.cnt = cnt;
  return o;
}

// full-mode beta sweep into the backward work buffer (dirs 2) or both sweeps (dirs 3)
static int full_sweeps(const scrf_problem* p, int64_t delta, int precision, int dirs, void* ckpt, void* work,
                       double* logZ, double* N, int32_t* dead_at, cudaStream_t st, bool progress = false) {
  const FLayout F = f_layout(p, precision);
  const BLayout W = b_layout(p, precision);
  unsigned char* fb = (unsigned char*)ckpt;
  unsigned char* wb = (unsigned char*)work;
  SweepIO io;
  memset(&io, 0, sizeof(io));
  io.dirs = dirs;
  io.record = true;
  if (dirs & 1) {
    io.Y[0] = fb + F.Y;
    io.X[0] = fb + F.X;
    io.n[0] = (double*)(fb + F.n);
    io.amx = fb + F.amx;
    io.clamp = (int32_t*)(fb + F.clamp);
    io.logZ = logZ;
    io.N = N;
    io.dead_at = dead_at;
  }
  io.Y[1] = wb + W.Y;
  io.X[1] = wb + W.X;
  io.n[1] = (double*)(wb + W.n);
  io.logZb = (double*)(wb + W.P.logZb);
  io.prog = progress ? (int*)(wb + W.P.prog) : nullptr;
  return SCRF_DISPATCH(precision, run_sweep)(p, delta, io, st);
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
  const PostOut o = post_out(logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end, position_marginals,
                             boundary_posterior, expected_segment_count);
  const int om = ovl_mode(p);
  if (om >= 0) {
    rc = ovl_begin(p, (unsigned char*)work, b_layout(p, precision).P, om, st);
    if (rc) return rc;
  }
  rc = full_sweeps(p, delta, precision, 2, (void*)ckpt, work, nullptr, nullptr, nullptr, st, om == 1);
  if (rc) return rc;
  if (om >= 0) return SCRF_DISPATCH(precision, run_full_post_win)(p, ckpt, work, o, om, 2, st);
  return SCRF_DISPATCH(precision, run_full_post)(p, ckpt, work, o, st);
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
  const PostOut o = post_out(logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end, position_marginals,
                             boundary_posterior, expected_segment_count);
  const int om = ovl_mode(p);
  if (om >= 0) {
    rc = ovl_begin(p, (unsigned char*)work, b_layout(p, precision).P, om, st);
    if (rc) return rc;
  }
  rc = full_sweeps(p, delta, precision, 3, ckpt, work, logZ, N, dead_at, st, om == 1);
  if (rc) return rc;
  if (om >= 0) return SCRF_DISPATCH(precision, run_full_post_win)(p, ckpt, work, o, om, 3, st);
  return SCRF_DISPATCH(precision, run_full_post)(p, ckpt, work, o, st);
}

int scrf_backward_partials(const scrf_problem* p, int64_t delta, int precision, const void* work,
                           double* grad_T_partial, double* grad_B_partial, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  (void)delta;
  const PLayout P = b_layout(p, precision).P;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned char* w = (const unsigned char*)work;
  cudaError_t e = cudaMemcpyAsync(grad_T_partial, w + P.accT, (size_t)p->B * p->C * p->C * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(grad_B_partial, w + P.accB, (size_t)p->B * p->K * p->C * 8, cudaMemcpyDeviceToDevice, st);
  return (int)e;
}

// ---------------------------------------------------------------------------
// sublinear-memory mode

static int sparse_G(const scrf_problem* p, int precision) {
  SweepGeo g;
  int rc = precision ? sweep_geo_of<double>(p, &g) : sweep_geo_of<float>(p, &g);
  return rc ? -1 : g.G;
}

int scrf_sparse_checkpoint_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  *bytes = s_layout(p, delta, precision).total;
  return SCRF_OK;
}

int scrf_sparse_backward_work_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  const int G = sparse_G(p, precision);
  if (G < 0) return SCRF_ECONFIG;
  *bytes = w_layout(p, delta, precision, G).total;
  return SCRF_OK;
}

int scrf_forward_sparse(const scrf_problem* p, int64_t delta, int precision, double* logZ, double* N, int32_t* dead_at,
                        void* ckpt, size_t ckpt_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  if (!logZ || !N || !dead_at || !ckpt) return SCRF_ENULL;
  if (ckpt_bytes < s_layout(p, delta, precision).total) return SCRF_EWORK;
  return SCRF_DISPATCH(precision, run_sparse_sweeps)(p, delta, 1, ckpt, nullptr, logZ, N, dead_at,
                                                      (cudaStream_t)stream, true);
}

int scrf_backward_sparse(const scrf_problem* p, int64_t delta, int precision, const double* logZ, const double* N,
                         const void* ckpt, const double* upstream, double* grad_S, double* grad_T, double* grad_B,
                         double* grad_P_start, double* grad_P_end, double* position_marginals,
                         double* boundary_posterior, double* expected_segment_count, void* work, size_t work_bytes,
                         void* stream) {
  g_launches = 0;
  int rc = check_bwd_args(p, delta, logZ, ckpt, grad_S, grad_T, grad_B, position_marginals, boundary_posterior,
                          expected_segment_count, work);
  if (rc) return rc;
  if (!N) return SCRF_ENULL;
  size_t need = 0;
  rc = scrf_sparse_backward_work_bytes(p, delta, precision, &need);
  if (rc) return rc;
  if (work_bytes < need) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  rc = SCRF_DISPATCH(precision, run_sparse_sweeps)(p, delta, 2, nullptr, work, nullptr, nullptr, nullptr, st, true);
  if (rc) return rc;
  const PostOut o = post_out(logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end, position_marginals,
                             boundary_posterior, expected_segment_count);
  return SCRF_DISPATCH(precision, run_sparse_post)(p, delta, ckpt, N, work, o, st);
}

int scrf_posterior_sparse(const scrf_problem* p, int64_t delta, int precision, const double* upstream, double* logZ,
                          double* N, int32_t* dead_at, void* ckpt, size_t ckpt_bytes, double* grad_S, double* grad_T,
                          double* grad_B, double* grad_P_start, double* grad_P_end, double* position_marginals,
                          double* boundary_posterior, double* expected_segment_count, void* work, size_t work_bytes,
                          void* stream) {
  g_launches = 0;
  int rc = check_bwd_args(p, delta, logZ, ckpt, grad_S, grad_T, grad_B, position_marginals, boundary_posterior,
                          expected_segment_count, work);
  if (rc) return rc;
  if (!N || !dead_at) return SCRF_ENULL;
  size_t need = 0;
  rc = scrf_sparse_backward_work_bytes(p, delta, precision, &need);
  if (rc) return rc;
  if (ckpt_bytes < s_layout(p, delta, precision).total || work_bytes < need) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  rc = SCRF_DISPATCH(precision, run_sparse_sweeps)(p, delta, 3, ckpt, work, logZ, N, dead_at, st, true);
  if (rc) return rc;
  const PostOut o = post_out(logZ, upstream, grad_S, grad_T, grad_B, grad_P_start, grad_P_end, position_marginals,
                             boundary_posterior, expected_segment_count);
  return SCRF_DISPATCH(precision, run_sparse_post)(p, delta, ckpt, N, work, o, st);
}

int scrf_backward_partials_sparse(const scrf_problem* p, int64_t delta, int precision, const void* work,
                                  double* grad_T_partial, double* grad_B_partial, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  const int G = sparse_G(p, precision);
  if (G < 0) return SCRF_ECONFIG;
  const PLayout P = w_layout(p, delta, precision, G).P;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned char* w = (const unsigned char*)work;
  cudaError_t e = cudaMemcpyAsync(grad_T_partial, w + P.accT, (size_t)p->B * p->C * p->C * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(grad_B_partial, w + P.accB, (size_t)p->B * p->K * p->C * 8, cudaMemcpyDeviceToDevice, st);
  return (int)e;
}

int scrf_beta_logz_sparse(const scrf_problem* p, int64_t delta, int precision, const void* work, double* logZb,
                          void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  const int G = sparse_G(p, precision);
  if (G < 0) return SCRF_ECONFIG;
  const PLayout P = w_layout(p, delta, precision, G).P;
  return (int)cudaMemcpyAsync(logZb, (const unsigned char*)work + P.logZb, (size_t)p->B * 8, cudaMemcpyDeviceToDevice,
                              (cudaStream_t)stream);
}

int scrf_beta_logz(const scrf_problem* p, int precision, const void* work, double* logZb, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  const BLayout W = b_layout(p, precision);
  return (int)cudaMemcpyAsync(logZb, (const unsigned char*)work + W.P.logZb, (size_t)p->B * 8, cudaMemcpyDeviceToDevice,
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
      work ? (const int32_t*)((const unsigned char*)work + b_layout(p, precision).P.clamp) : nullptr, events);
  return (int)cudaGetLastError();
}

int scrf_clamp_events_sparse(const scrf_problem* p, int64_t delta, int precision, const void* ckpt, const void* work,
                             int32_t* events, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (!ckpt || !events) return SCRF_ENULL;
  const SLayout S = s_layout(p, delta, precision);
  const int G = sparse_G(p, precision);
  if (G < 0) return SCRF_ECONFIG;
  cudaStream_t st = (cudaStream_t)stream;
  ++g_launches;
  clamp_sum_kernel<<<(unsigned)((p->B + 127) / 128), 128, 0, st>>>(
      (int)p->B, (const int32_t*)((const unsigned char*)ckpt + S.clamp),
      work ? (const int32_t*)((const unsigned char*)work + w_layout(p, delta, precision, G).P.clamp) : nullptr, events);
  return (int)cudaGetLastError();
}

int scrf_export_checkpoints_sparse(const scrf_problem* p, int64_t delta, int precision, const void* ckpt,
                                   const double* N, double* omega, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  const SLayout S = s_layout(p, delta, precision);
  const SparseGeo g = sparse_geo(p, delta);
  const unsigned char* base = (const unsigned char*)ckpt;
  const int nck = (int)n_ckpt_of(p->T, delta);
  const size_t total = (size_t)p->B * nck * p->K * p->C;
  ++g_launches;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (precision)
    export_sparse_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const double*)(base + S.Y), (const double*)(base + S.n), N, p->lengths, (int)p->B, (int)p->T, nck,
        (int)p->K, (int)p->C, (int)delta, g.mA, g.rowsAlpha, omega);
  else
    export_sparse_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const float*)(base + S.Y), (const double*)(base + S.n), N, p->lengths, (int)p->B, (int)p->T, nck,
        (int)p->K, (int)p->C, (int)delta, g.mA, g.rowsAlpha, omega);
  return (int)cudaGetLastError();
}

// recompute_alpha (streaming.py:232-261) on the device: forced rows from the snapshot, a replay
// task per sequence, the block in the snapshot frame
struct RALayout {
  size_t fY, fN, oY, oX, on, tasks, total;
  int rows;  // output rows per sequence
};
static RALayout ra_layout(const scrf_problem* p, int precision, int64_t t0, int64_t t1) {
  RALayout L;
  const size_t rs = precision ? 8 : 4;
  const size_t B = p->B, C = p->C, K = p->K;
  const int64_t tf0 = t0 - K + 1 > 0 ? t0 - K + 1 : 0;
  L.rows = (int)(t1 - tf0 + 1);
  size_t o = 0;
  L.fY = o;    o += al(B * K * C * rs);
  L.fN = o;    o += al(B * K * 8);
  L.oY = o;    o += al(B * (size_t)L.rows * C * rs);
  L.oX = o;    o += al(B * (size_t)L.rows * C * rs);
  L.on = o;    o += al(B * (size_t)L.rows * 8);
  L.tasks = o; o += al(B * sizeof(SweepTask));
  L.total = o;
  return L;
}

int scrf_recompute_alpha_work_bytes(const scrf_problem* p, int64_t t_start, int64_t t_end, int precision,
                                    size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (t_start < 0 || t_end < t_start || t_end > p->T) return SCRF_EDIM;
  *bytes = ra_layout(p, precision, t_start, t_end).total;
  return SCRF_OK;
}

int scrf_recompute_alpha(const scrf_problem* p, int precision, const double* omega_i, int64_t t_start, int64_t t_end,
                         double* block, void* work, size_t work_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (!omega_i || !block || !work) return SCRF_ENULL;
  if (t_start < 0 || t_end < t_start || t_end > p->T) return SCRF_EDIM;
  const RALayout RL = ra_layout(p, precision, t_start, t_end);
  if (work_bytes < RL.total) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* wb = (unsigned char*)work;
  const int B = (int)p->B, K = (int)p->K, C = (int)p->C;
  const int t0 = (int)t_start, t1 = (int)t_end;
  const int tf0 = t0 - K + 1 > 0 ? t0 - K + 1 : 0;
  ++g_launches;
  if (precision)
    ra_prep_kernel<double><<<B, 128, 0, st>>>(omega_i, p->lengths, B, K, C, t0, t1, tf0, RL.rows,
                                              (double*)(wb + RL.fY), (double*)(wb + RL.fN),
                                              (SweepTask*)(wb + RL.tasks));
  else
    ra_prep_kernel<float><<<B, 128, 0, st>>>(omega_i, p->lengths, B, K, C, t0, t1, tf0, RL.rows,
                                             (float*)(wb + RL.fY), (double*)(wb + RL.fN),
                                             (SweepTask*)(wb + RL.tasks));
  if (t1 > t0) {
    SweepIO io;
    memset(&io, 0, sizeof(io));
    io.dirs = 1;
    io.tasks = (const SweepTask*)(wb + RL.tasks);
    io.ntasks = B;
    io.Y[0] = wb + RL.oY;
    io.X[0] = wb + RL.oX;
    io.n[0] = (double*)(wb + RL.on);
    io.fY[0] = wb + RL.fY;
    io.fN[0] = (const double*)(wb + RL.fN);
    rc = SCRF_DISPATCH(precision, run_sweep)(p, (int64_t)1 << 30, io, st);
    if (rc) return rc;
  }
  const size_t total = (size_t)B * (t1 - t0 + 1) * C;
  ++g_launches;
  if (precision)
    ra_block_kernel<double><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        omega_i, p->lengths, B, K, C, t0, t1, tf0, RL.rows, (const double*)(wb + RL.oY), (const double*)(wb + RL.on),
        block);
  else
    ra_block_kernel<float><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        omega_i, p->lengths, B, K, C, t0, t1, tf0, RL.rows, (const float*)(wb + RL.oY), (const double*)(wb + RL.on),
        block);
  return (int)cudaGetLastError();
}

int scrf_reduce_partials(int64_t B, int64_t n, const double* parts, const double* upstream, double* out,
                         void* stream) {
  if (B < 1 || n < 1) return SCRF_EDIM;
  if (!parts || !out) return SCRF_ENULL;
  ++g_launches;
  post_reduce2_kernel<<<(unsigned)((n + 31) / 32), 256, 0, (cudaStream_t)stream>>>((int)B, (int)n, 1, parts, upstream,
                                                                                     nullptr, out);
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

int scrf_input_gate(const int32_t* gate, int ngate, int shift) {
  if (gate && (ngate < 1 || shift < 0 || shift > 30)) return SCRF_EDIM;
  if (gate) preload_concurrent_kernels();
  g_gate = gate;
  g_gate_n = gate ? ngate : 0;
  g_gate_shift = shift;
  return SCRF_OK;
}

int scrf_upload_rows(void* dst, const void* src, int64_t B, int64_t rows, int64_t row_bytes, int64_t r0, int64_t r1,
                     int32_t* gate, int j, void* stream) {
  if (!dst || !src) return SCRF_ENULL;
  if (B < 1 || rows < 1 || row_bytes < 1 || r0 < 0 || r1 > rows || r1 <= r0) return SCRF_EDIM;
  const size_t pitch = (size_t)rows * row_bytes;
  cudaError_t e = cudaMemcpy2DAsync((char*)dst + r0 * row_bytes, pitch, (const char*)src + r0 * row_bytes, pitch,
                                    (size_t)(r1 - r0) * row_bytes, (size_t)B, cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return (int)e;
  if (gate) {
    if (j < 0) return SCRF_EDIM;
    gate_set_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(gate, j);
    e = cudaGetLastError();
  }
  return (int)e;
}

int scrf_gate_set(int32_t* gate, int j, void* stream) {
  if (!gate) return SCRF_ENULL;
  if (j < 0) return SCRF_EDIM;
  gate_set_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(gate, j);
  return (int)cudaGetLastError();
}

void scrf_window_events(void** events, int n) {
  g_win_ev = (cudaEvent_t*)events;
  g_win_nev = events ? n : 0;
}

int scrf_window_plan(const scrf_problem* p, int32_t* w0, int32_t* w1, int cap) {
  if (check_problem(p) || ovl_mode(p) < 0) return 0;
  OvlWin win[4096];
  const int n = ovl_windows(p, win, 4096);
  if (n > cap) return -n;
  for (int i = 0; i < n; ++i) {
    w0[i] = win[i].w0;
    w1[i] = win[i].w1;
  }
  return n;
}

}  // extern "C"
