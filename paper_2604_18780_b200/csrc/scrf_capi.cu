// C ABI of libscrf.so (declared in include/scrf.h): geometry selection, buffer
// layout and kernel launches. Host code only; kernels live in scrf_fb.cu and
// scrf_viterbi.cu (compiled into this translation unit so templates instantiate once).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/scrf.h"
#include "scrf_fb.cu"
#include "scrf_viterbi.cu"

using namespace scrf;

namespace {

thread_local int g_launches = 0;
// optional events recorded around the next main kernel launch (forward / backward / Viterbi)
thread_local cudaEvent_t g_ev_start = nullptr;
thread_local cudaEvent_t g_ev_stop = nullptr;
thread_local long long* g_trace = nullptr;  // debug: phase timestamps of the forward

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

size_t fb_smem(const Geometry& g, int K, int C, int precision) {
  return precision ? fwd_smem_bytes<double>(K, C, g) + bwd_extra_smem_bytes<double>(K, C, g) + stage_smem_bytes<double>(g)
                   : fwd_smem_bytes<float>(K, C, g) + bwd_extra_smem_bytes<float>(K, C, g) + stage_smem_bytes<float>(g);
}

// Geometry shared by forward and backward (the replay must re-execute the forward
// bit for bit, so both kernels use the same label slices and thread mapping).
int choose_fb_geo(int B, int K, int C, int precision, Geometry* out) {
  const size_t limit = (size_t)smem_optin();
  int forced = env_int("SCRF_G", 0);
  const int cands[] = {1, 2, 4, 8, 16};
  int gmin = 0;
  for (int G : cands) {
    if (G > C && G > 1) break;
    if (forced && G != forced) continue;
    Geometry g = make_geo(G, K, C);
    if (g.NT <= 1024 && fb_smem(g, K, C, precision) <= limit) {
      gmin = G;
      break;
    }
  }
  if (!gmin) return SCRF_ECONFIG;
  int G = gmin;
  if (!forced) {
    // widen the cluster while the batch still fits on the chip (portable sizes)
    while (G * 2 <= 8 && G * 2 <= C && (long long)B * G * 2 <= num_sms()) G *= 2;
  }
  *out = make_geo(G, K, C);
  return SCRF_OK;
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

// checkpoint buffer layout (offsets in bytes, 256-aligned)
struct CkLayout {
  size_t hdr_geo, g_hi, g_lo, alpha, n, hdr, tail_alpha, tail_n, total;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

CkLayout ck_layout(const scrf_problem* p, int64_t delta, int precision) {
  CkLayout L;
  const size_t rs = precision ? 8 : 4;
  const size_t nck = (size_t)n_ckpt_of(p->T, delta);
  const size_t ring = (size_t)p->B * nck * p->K * p->C;
  size_t o = 0;
  L.hdr_geo = o;
  o += al(sizeof(Geometry) + 64);
  L.g_hi = o;
  o += al(ring * rs);
  L.g_lo = o;
  o += al(ring * rs);
  L.alpha = o;
  o += al(ring * rs);
  L.n = o;
  o += al((size_t)p->B * nck * p->K * 8);
  L.hdr = o;
  o += al((size_t)p->B * nck * 2 * 8);
  L.tail_alpha = o;
  o += al((size_t)p->B * p->K * p->C * rs);
  L.tail_n = o;
  o += al((size_t)p->B * p->K * 8);
  L.total = o;
  return L;
}

struct WorkLayout {
  size_t ws_alpha, ws_gamma, ws_n, start, end, gT, gB, total;
};

WorkLayout work_layout(const scrf_problem* p, int64_t delta, const Geometry& g, int precision) {
  WorkLayout W;
  size_t o = 0;
  const size_t win = (size_t)p->B * (delta + 1) * p->C;
  const size_t rs = precision ? 8 : 4;
  W.ws_alpha = o;
  o += al(win * rs);
  W.ws_gamma = o;
  o += al(win * rs);
  W.ws_n = o;
  o += al((size_t)p->B * g.G * (delta + 1) * 8);
  W.start = o;
  o += al((size_t)p->B * (p->T + 1) * p->C * rs);
  W.end = o;
  o += al((size_t)p->B * (p->T + 1) * p->C * rs);
  W.gT = o;
  o += al((size_t)p->B * p->C * p->C * 8);
  W.gB = o;
  o += al((size_t)p->B * p->K * p->C * 8);
  W.total = o;
  return W;
}

template <typename Kern, typename ArgT>
cudaError_t launch_cluster(Kern kern, const Geometry& g, int B, size_t smem, cudaStream_t st, ArgT arg) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (g.G > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(B * g.G, 1, 1);
  cfg.blockDim = dim3(g.NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  if (g_ev_start) cudaEventRecord(g_ev_start, st);
  e = cudaLaunchKernelEx(&cfg, kern, arg);
  if (g_ev_stop) cudaEventRecord(g_ev_stop, st);
  return e;
}

template <typename R>
void fill_args(Args<R>& a, const scrf_problem* p, int64_t delta, const Geometry& g, void* ckpt) {
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
  a.delta = (int)delta;
  a.n_ckpt = (int)n_ckpt_of(p->T, delta);
  a.geo = g;
  CkLayout L = ck_layout(p, delta, sizeof(R) == 8);
  unsigned char* base = (unsigned char*)ckpt;
  a.ck.g_hi = (R*)(base + L.g_hi);
  a.ck.g_lo = (R*)(base + L.g_lo);
  a.ck.alpha = (R*)(base + L.alpha);
  a.ck.n = (double*)(base + L.n);
  a.ck.hdr = (double*)(base + L.hdr);
  a.tail_alpha = (R*)(base + L.tail_alpha);
  a.tail_n = (double*)(base + L.tail_n);
}

template <typename R>
int run_forward(const scrf_problem* p, int64_t delta, double* logZ, double* N, int32_t* dead_at, void* ckpt,
                cudaStream_t st) {
  Geometry g;
  int rc = choose_fb_geo((int)p->B, (int)p->K, (int)p->C, sizeof(R) == 8, &g);
  if (rc) return rc;
  Args<R> a;
  fill_args(a, p, delta, g, ckpt);
  a.trace = g_trace;
  a.logZ = logZ;
  a.N = N;
  a.dead_at = dead_at;
  size_t smem = fwd_smem_bytes<R>(a.K, a.C, g) + stage_smem_bytes<R>(g);
  return (int)launch_cluster(fwd_kernel<R>, g, a.B, smem, st, a);
}

template <typename R>
int run_backward(const scrf_problem* p, int64_t delta, const double* logZ, const void* ckpt, const double* upstream,
                 double* grad_S, double* grad_T, double* grad_B, double* gPs, double* gPe, double* pos, double* bnd,
                 double* cnt, void* work, size_t work_bytes, cudaStream_t st) {
  Geometry g;
  int rc = choose_fb_geo((int)p->B, (int)p->K, (int)p->C, sizeof(R) == 8, &g);
  if (rc) return rc;
  WorkLayout W = work_layout(p, delta, g, sizeof(R) == 8);
  if (work_bytes < W.total) return SCRF_EWORK;
  Args<R> a;
  fill_args(a, p, delta, g, (void*)ckpt);
  unsigned char* w = (unsigned char*)work;
  a.logZ_in = logZ;
  a.upstream = upstream;
  a.ws_alpha = (R*)(w + W.ws_alpha);
  a.ws_gamma = (R*)(w + W.ws_gamma);
  a.ws_n = (double*)(w + W.ws_n);
  a.start_g = (R*)(w + W.start);
  a.end_g = (R*)(w + W.end);
  a.gT_part = (double*)(w + W.gT);
  a.gB_part = (double*)(w + W.gB);
  cudaError_t e = cudaMemsetAsync(w + W.start, 0, W.total - W.start, st);
  if (e != cudaSuccess) return (int)e;
  size_t smem = fwd_smem_bytes<R>(a.K, a.C, g) + bwd_extra_smem_bytes<R>(a.K, a.C, g) + stage_smem_bytes<R>(g);
  e = launch_cluster(bwd_kernel<R>, g, a.B, smem, st, a);
  if (e != cudaSuccess) return (int)e;
  const int B = a.B, T = a.T, C = a.C, K = a.K;
  {
    int n = B * C, blk = 128;
    ++g_launches;
    finalize_kernel<R><<<(n + blk - 1) / blk, blk, 0, st>>>(a.start_g, a.end_g, p->lengths, upstream, B, T, C, grad_S, gPs,
                                                         gPe, pos);
    ++g_launches;
    boundary_kernel<R><<<B, 256, 0, st>>>(a.start_g, p->lengths, B, T, C, bnd, cnt);
    size_t nT = (size_t)C * C, nB = (size_t)K * C;
    ++g_launches;
    reduce_partials_kernel<<<(unsigned)((nT + 255) / 256), 256, 0, st>>>(a.gT_part, upstream, B, nT, grad_T);
    ++g_launches;
    reduce_partials_kernel<<<(unsigned)((nB + 255) / 256), 256, 0, st>>>(a.gB_part, upstream, B, nB, grad_B);
  }
  return (int)cudaGetLastError();
}

template <typename A>
__global__ void export_kernel(const A* alpha, const double* n, const double* N, int B, int nck, int K, int C,
                              double* omega) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t total = (size_t)B * nck * K * C;
  if (i >= total) return;
  size_t bi = i / ((size_t)K * C);  // (b, ckpt)
  size_t slot = (i / C) % K;
  A av = alpha[i];
  double nv = n[bi * K + slot];
  if (!(av > -INFINITY) || !(nv > -INFINITY)) {
    omega[i] = kNegInfRef;
    return;
  }
  double v = ((double)av + nv) * kLn2 - N[bi];
  omega[i] = v <= kGuard ? kNegInfRef : v;
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
  *bytes = ck_layout(p, delta, precision).total;
  return SCRF_OK;
}

int scrf_forward(const scrf_problem* p, int64_t delta, int precision, double* logZ, double* N, int32_t* dead_at,
                 void* ckpt, size_t ckpt_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  if (!logZ || !N || !dead_at || !ckpt) return SCRF_ENULL;
  if (ckpt_bytes < ck_layout(p, delta, precision).total) return SCRF_EWORK;
  cudaStream_t st = (cudaStream_t)stream;
  return precision ? run_forward<double>(p, delta, logZ, N, dead_at, ckpt, st)
                   : run_forward<float>(p, delta, logZ, N, dead_at, ckpt, st);
}

int scrf_backward_work_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  Geometry g;
  rc = choose_fb_geo((int)p->B, (int)p->K, (int)p->C, precision, &g);
  if (rc) return rc;
  *bytes = work_layout(p, delta, g, precision).total;
  return SCRF_OK;
}

int scrf_backward(const scrf_problem* p, int64_t delta, int precision, const double* logZ, const void* ckpt,
                  const double* upstream, double* grad_S, double* grad_T, double* grad_B, double* grad_P_start,
                  double* grad_P_end, double* position_marginals, double* boundary_posterior,
                  double* expected_segment_count, void* work, size_t work_bytes, void* stream) {
  g_launches = 0;
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  if (!logZ || !ckpt || !grad_S || !grad_T || !grad_B || !position_marginals || !boundary_posterior ||
      !expected_segment_count || !work)
    return SCRF_ENULL;
  cudaStream_t st = (cudaStream_t)stream;
  return precision ? run_backward<double>(p, delta, logZ, ckpt, upstream, grad_S, grad_T, grad_B, grad_P_start,
                                          grad_P_end, position_marginals, boundary_posterior, expected_segment_count,
                                          work, work_bytes, st)
                   : run_backward<float>(p, delta, logZ, ckpt, upstream, grad_S, grad_T, grad_B, grad_P_start,
                                         grad_P_end, position_marginals, boundary_posterior, expected_segment_count,
                                         work, work_bytes, st);
}

int scrf_backward_partials(const scrf_problem* p, int64_t delta, int precision, const void* work,
                           double* grad_T_partial, double* grad_B_partial, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  Geometry g;
  rc = choose_fb_geo((int)p->B, (int)p->K, (int)p->C, precision, &g);
  if (rc) return rc;
  WorkLayout W = work_layout(p, delta, g, precision);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned char* w = (const unsigned char*)work;
  cudaError_t e = cudaMemcpyAsync(grad_T_partial, w + W.gT, (size_t)p->B * p->C * p->C * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(grad_B_partial, w + W.gB, (size_t)p->B * p->K * p->C * 8, cudaMemcpyDeviceToDevice, st);
  return (int)e;
}

static size_t vit_dvr_bytes(const scrf_problem* p, const Geometry& g) { return al((size_t)p->B * g.G * p->K * p->C * 8); }

int scrf_viterbi_work_bytes(const scrf_problem* p, size_t* bytes) {
  int rc = check_problem(p);
  if (rc) return rc;
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
  cudaError_t e = launch_cluster(vit_kernel, g, a.B, smem, (cudaStream_t)stream, a);
  return (int)e;
}

int scrf_export_checkpoints(const scrf_problem* p, int64_t delta, int precision, const void* ckpt, const double* N,
                            double* omega, void* stream) {
  int rc = check_problem(p);
  if (rc) return rc;
  if (delta < 1) return SCRF_EDELTA;
  CkLayout L = ck_layout(p, delta, precision);
  const unsigned char* base = (const unsigned char*)ckpt;
  const int nck = (int)n_ckpt_of(p->T, delta);
  size_t total = (size_t)p->B * nck * p->K * p->C;
  ++g_launches;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (precision)
    export_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const double*)(base + L.alpha), (const double*)(base + L.n), N, (int)p->B, nck, (int)p->K, (int)p->C, omega);
  else
    export_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const float*)(base + L.alpha), (const double*)(base + L.n), N, (int)p->B, nck, (int)p->K, (int)p->C, omega);
  return (int)cudaGetLastError();
}

int scrf_last_launch_count(void) { return g_launches; }

void scrf_debug_trace(void* buf) { g_trace = (long long*)buf; }

void scrf_profile_events(void* start, void* stop) {
  g_ev_start = (cudaEvent_t)start;
  g_ev_stop = (cudaEvent_t)stop;
}

}  // extern "C"
