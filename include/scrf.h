/* C ABI of the B200 streaming semi-CRF library (libscrf.so).
 *
 * This is the drop-in boundary for the reference's hot path,
 * `pkg/src/streamcrf/streaming.py` (streamcrf 0.1.0). Each entry point replaces
 * one reference function; the Python mirror (paper_2604_18780_b200.streaming)
 * keeps the reference's names and dataclasses and calls these through ctypes.
 *
 * Two working-memory modes of the same kernels:
 *   sublinear (the reference's design): the forward keeps only checkpoint
 *     rows (the reference's snapshots Omega every delta positions plus replay warm-up rows,
 *     O(sqrt(T K) C)); the backward replays alpha (and beta) window by window from them.
 *       scrf_forward_sparse   <- streaming_forward (streaming.py:155-229), forward_logZ (:707-722)
 *       scrf_backward_sparse  <- streaming_backward (streaming.py:264-408) incl. the alpha replay
 *                                (:332-336) and finalize_marginals (diagnostics.py:54-79)
 *       scrf_posterior_sparse <- posterior (streaming.py:725-746) in sublinear memory
 *       scrf_recompute_alpha  <- recompute_alpha (streaming.py:232-261)
 *       scrf_export_checkpoints_sparse <- CheckpointSet(omega, N, delta) (streaming.py:49-67)
 *   full: every position's messages are kept (O(T C) working memory), no replay; fastest.
 *       scrf_forward / scrf_backward / scrf_posterior / scrf_export_checkpoints
 *   scrf_viterbi   <- streaming_viterbi   (streaming.py:411-470) + decode (:749-762)
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer owned by the caller; optional
 *     inputs may be NULL. Shapes: S (B, T+1, C) fp64; lengths (B,) int64 with
 *     1 <= L_b <= T; transition (C, C) [c_prev, c_new]; duration_bias (K, C)
 *     [k-1, c]; proj_start / proj_end (B, T, C) fp64 or NULL.
 *   - Work buffers are sized by the matching *_bytes query; their contents on entry do not
 *     matter (every region is written before it is read, accumulators are cleared on the
 *     call's stream). No hidden allocations. The only process state is debug/profiling
 *     hooks (scrf_profile_events, scrf_position_outputs_event, scrf_debug_*), per thread.
 *   - `stream` is a cudaStream_t (passed as void*); all work is stream-ordered; no entry
 *     point synchronises with the host (tracebacks and segment lists stay on the device).
 *   - Return: 0 ok; < 0 invalid argument (see SCRF_E*); > 0 a cudaError_t.
 *   - precision: 0 = fp32 working type (production), 1 = fp64 working type
 *     (validation instantiation of the same algorithm).
 */
#ifndef SCRF_H_
#define SCRF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCRF_OK 0
#define SCRF_EDIM (-1)        /* B, T, K or C out of range */
#define SCRF_EDELTA (-2)      /* checkpoint interval < 1 */
#define SCRF_EWORK (-3)       /* work buffer too small */
#define SCRF_ECONFIG (-4)     /* no launch geometry fits shared memory */
#define SCRF_ENULL (-5)       /* required pointer is NULL */

typedef struct scrf_problem {
  const double* S;              /* (B, T+1, C) */
  const int64_t* lengths;       /* (B,) */
  const double* transition;     /* (C, C) */
  const double* duration_bias;  /* (K, C) */
  const double* proj_start;     /* (B, T, C) or NULL */
  const double* proj_end;       /* (B, T, C) or NULL */
  int64_t B, T, K, C;
} scrf_problem;

/* Checkpoint interval the reference uses: clamp(round(sqrt(T*K)), 1, T)
 * (streaming.py:101-109). */
int64_t scrf_default_delta(int64_t T, int64_t K);

/* Size of the opaque checkpoint buffer for (problem dims, delta, precision). */
int scrf_checkpoint_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes);

/* Forward pass: logZ (B,) in nats, reference-format normalisers N (B, n_ckpt),
 * dead_at (B,) = -1 or the first position at which every message fell below
 * the reference guard (caller raises the reference's ValueError), and the
 * opaque checkpoint buffer consumed by scrf_backward. */
int scrf_forward(const scrf_problem* p, int64_t delta, int precision, double* logZ, double* N,
                 int32_t* dead_at, void* ckpt, size_t ckpt_bytes, void* stream);

/* Size of the backward work buffer. */
int scrf_backward_work_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes);

/* Backward pass from scrf_forward's checkpoints. upstream (B,) scales the
 * gradients only (NULL = ones). Outputs (all device, fp64):
 *   grad_S (B, T+1, C); grad_T (C, C); grad_B (K, C);
 *   grad_P_start, grad_P_end (B, T, C) or NULL (only computed if non-NULL);
 *   position_marginals (B, T, C); boundary_posterior (B, T); expected_segment_count (B,).
 * Transition / duration gradients are reduced over the batch in a fixed order
 * (bit-reproducible). */
int scrf_backward(const scrf_problem* p, int64_t delta, int precision, const double* logZ,
                  const void* ckpt, const double* upstream, double* grad_S, double* grad_T,
                  double* grad_B, double* grad_P_start, double* grad_P_end,
                  double* position_marginals, double* boundary_posterior,
                  double* expected_segment_count, void* work, size_t work_bytes, void* stream);

/* posterior(cum, params, delta, upstream) in one call: the forward outputs of
 * scrf_forward (logZ, N, dead_at, ckpt) and the backward outputs of scrf_backward.
 * The alpha and beta message sweeps are independent and run concurrently. */
int scrf_posterior(const scrf_problem* p, int64_t delta, int precision, const double* upstream,
                   double* logZ, double* N, int32_t* dead_at, void* ckpt, size_t ckpt_bytes,
                   double* grad_S, double* grad_T, double* grad_B, double* grad_P_start,
                   double* grad_P_end, double* position_marginals, double* boundary_posterior,
                   double* expected_segment_count, void* work, size_t work_bytes, void* stream);

/* logZ recomputed from the beta sweep (LSE_c beta[0,c]; virtual source), (B,) nats:
 * a consistency value for tests, copied out of `work` after scrf_backward/posterior. */
int scrf_beta_logz(const scrf_problem* p, int precision, const void* work, double* logZb, void* stream);

/* Per-sequence (unreduced) transition / duration gradient partials, for the
 * multi-GPU path that reduces across ranks in a fixed order: after
 * scrf_backward, copies (B, C, C) and (B, K, C) fp64 partials out of `work`. */
int scrf_backward_partials(const scrf_problem* p, int64_t delta, int precision, const void* work,
                           double* grad_T_partial, double* grad_B_partial, void* stream);

/* Viterbi work buffer size. */
int scrf_viterbi_work_bytes(const scrf_problem* p, size_t* bytes);

/* Exact fp64 max-plus Viterbi with the reference's operation order and tie
 * rules. Outputs: score (B,); per sequence b the segments are written at
 * seg_start/seg_end/seg_label[b*T + j], j < seg_count[b] (in order). */
int scrf_viterbi(const scrf_problem* p, double* score, int32_t* seg_start, int32_t* seg_end,
                 int32_t* seg_label, int32_t* seg_count, void* work, size_t work_bytes,
                 void* stream);

/* Reference-format view of the checkpoints: omega (B, n_ckpt, K, C) fp64, ring
 * snapshots after the shift at i*delta with the reference's slot layout and
 * the sentinel -1e9 for never-written slots. */
int scrf_export_checkpoints(const scrf_problem* p, int64_t delta, int precision, const void* ckpt,
                            const double* N, double* omega, void* stream);

/* ---- sublinear-memory mode ------------------------------------------------------------ */

/* Size of the sparse checkpoint buffer (alpha checkpoint rows, O(sqrt(T K) C)). */
int scrf_sparse_checkpoint_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes);

/* Size of the sparse backward work buffer: beta checkpoint rows, the replay window buffers
 * (a few windows of ~max(delta, K+32) positions) and the per-pass partials. */
int scrf_sparse_backward_work_bytes(const scrf_problem* p, int64_t delta, int precision, size_t* bytes);

/* Forward keeping only checkpoint rows; same outputs as scrf_forward (logZ, N, dead_at). */
int scrf_forward_sparse(const scrf_problem* p, int64_t delta, int precision, double* logZ, double* N,
                        int32_t* dead_at, void* ckpt, size_t ckpt_bytes, void* stream);

/* Backward from scrf_forward_sparse's checkpoint rows and normalisers N: a beta sweep storing
 * beta checkpoint rows, then window by window the alpha and beta replays and the posterior
 * pass of the window. Outputs as scrf_backward. */
int scrf_backward_sparse(const scrf_problem* p, int64_t delta, int precision, const double* logZ,
                         const double* N, const void* ckpt, const double* upstream, double* grad_S,
                         double* grad_T, double* grad_B, double* grad_P_start, double* grad_P_end,
                         double* position_marginals, double* boundary_posterior,
                         double* expected_segment_count, void* work, size_t work_bytes, void* stream);

/* Both, with the alpha and beta checkpoint sweeps concurrent (scrf_posterior's signature). */
int scrf_posterior_sparse(const scrf_problem* p, int64_t delta, int precision, const double* upstream,
                          double* logZ, double* N, int32_t* dead_at, void* ckpt, size_t ckpt_bytes,
                          double* grad_S, double* grad_T, double* grad_B, double* grad_P_start,
                          double* grad_P_end, double* position_marginals, double* boundary_posterior,
                          double* expected_segment_count, void* work, size_t work_bytes, void* stream);

/* Sparse twins of scrf_backward_partials / scrf_beta_logz / scrf_clamp_events /
 * scrf_export_checkpoints. */
int scrf_backward_partials_sparse(const scrf_problem* p, int64_t delta, int precision, const void* work,
                                  double* grad_T_partial, double* grad_B_partial, void* stream);
int scrf_beta_logz_sparse(const scrf_problem* p, int64_t delta, int precision, const void* work,
                          double* logZb, void* stream);
int scrf_clamp_events_sparse(const scrf_problem* p, int64_t delta, int precision, const void* ckpt,
                             const void* work, int32_t* events, void* stream);
int scrf_export_checkpoints_sparse(const scrf_problem* p, int64_t delta, int precision, const void* ckpt,
                                   const double* N, double* omega, void* stream);

/* recompute_alpha(omega_i, n_i, cum, params, t_start, t_end): omega_i (B, K, C) fp64 device
 * snapshot in the reference's ring-slot layout (values relative to N_i, sentinel -1e9 for
 * empty slots); block (B, t_end - t_start + 1, C) fp64 in the same frame; block[:, 0] is the
 * snapshot slot of t_start and positions past L_b hold their ring slot, as the reference. */
int scrf_recompute_alpha_work_bytes(const scrf_problem* p, int64_t t_start, int64_t t_end, int precision,
                                    size_t* bytes);
int scrf_recompute_alpha(const scrf_problem* p, int precision, const double* omega_i, int64_t t_start,
                         int64_t t_end, double* block, void* work, size_t work_bytes, void* stream);

/* The fixed-order batch reduction of per-sequence partials: out[i] = sum over b = 0..B-1, in
 * order, of upstream[b] * parts[b][i] (upstream NULL = ones), one rounding per multiply and per
 * add. scrf_backward / scrf_posterior finish with exactly this reduction over their
 * *_partials, so a batch sharded across ranks (all-gather the partials in batch order, then
 * this call) reproduces the single-GPU grad_T / grad_B bit for bit (the reference reduces in a
 * fixed order too, streaming.py:389-395). */
int scrf_reduce_partials(int64_t B, int64_t n, const double* parts, const double* upstream, double* out,
                         void* stream);

/* Clamp-event count per sequence (B,) int32 after scrf_forward (ckpt) and optionally
 * scrf_backward / scrf_posterior (work, or NULL): positions whose max alpha message relative
 * to the checkpoint normaliser, or max (unnormalised) beta message, leaves +-1e6 -- where the
 * reference's clamp_log (_numerics.py:41-56) would clip. The kernels do not clip (exact fp64
 * normalisers); callers reject inputs with a non-zero count (ClampSemanticsError). */
int scrf_clamp_events(const scrf_problem* p, int precision, const void* ckpt, const void* work,
                      int32_t* events, void* stream);

/* Number of kernel launches issued by the last call on this thread (for the
 * benchmark's gpu_launches claim). */
int scrf_last_launch_count(void);

/* Record the given cudaEvent_t pair (or NULL, NULL to disable) immediately before and
 * after the main cluster kernel of every subsequent scrf_forward / scrf_backward /
 * scrf_viterbi call on this thread, on the call's stream. Used by bench.py to time the
 * dominant kernel live (no profiler). */
void scrf_profile_events(void* start, void* stop);

/* Record the given cudaEvent_t (or NULL to disable) on the call's stream as soon as the
 * per-position outputs of every subsequent scrf_backward / scrf_posterior call on this thread
 * are final (grad_S, grad_P*, position marginals, boundary posterior), before the duration-
 * gradient pass. Lets a caller start their device-to-host copies on another stream while the
 * remaining pass runs. */
void scrf_position_outputs_event(void* event);

/* Full-memory posterior / backward at long T run their posterior passes in windows of
 * positions, concurrently with the sweeps (SCRF_OVERLAP, SCRF_OVL_WS). Writes the windows
 * [w0[i], w1[i]) in the order the passes complete them and returns their number (0: one pass
 * after the sweeps; -n: cap < n). Windows cover boundaries 0..T; a window's per-position
 * outputs are grad_S rows [w0, w1) and grad_P*, position marginals, boundary posterior rows
 * [w0, min(w1, T)). */
int scrf_window_plan(const scrf_problem* p, int32_t* w0, int32_t* w1, int cap);

/* events[i] (cudaEvent_t, or events = NULL to disable) is recorded, on the library's side
 * stream, as soon as the per-position outputs of window i of every subsequent full-memory
 * scrf_posterior / scrf_backward call on this thread are final -- for device-to-host copies
 * of each window while the sweeps still run (the numpy posterior() facade does this). */
void scrf_window_events(void** events, int n);

/* Streamed input for the next full-memory scrf_posterior / scrf_backward / scrf_forward calls on
 * this thread (gate = NULL to disable): the sweeps start before S is on the device and read the
 * rows [j << shift, (j+1) << shift) of every sequence only once gate[j] != 0. gate is a device
 * int32 array of ngate + 1 entries, zeroed by the caller before the call; the caller copies the
 * row chunks on another stream and marks each with scrf_gate_set on that stream after its copy
 * (chunk order: the alpha sweep consumes chunks from 0 up, the beta sweep from ngate-1 down).
 * gate[ngate] becomes 1 if a sweep waited more than 2 s for a chunk (the sweeps then stop waiting
 * and read whatever is there: a caller bug). Ps / Pe must be on the device before the call. Returns SCRF_EDIM for a
 * bad ngate / shift. */
int scrf_input_gate(const int32_t* gate, int ngate, int shift);

/* Launch, on `stream`, a one-thread kernel that release-stores gate[j] = 1 (after the chunk
 * copies queued before it on that stream). */
int scrf_gate_set(int32_t* gate, int j, void* stream);

/* Rows [r0, r1) of B row-major blocks of `rows` rows of row_bytes each (e.g. S: rows = T + 1,
 * row_bytes = 8 C), host (pinned) -> device, as one 2-D copy on `stream`; then, if gate is not
 * NULL, scrf_gate_set(gate, j). */
int scrf_upload_rows(void* dst, const void* src, int64_t B, int64_t rows, int64_t row_bytes, int64_t r0, int64_t r1,
                     int32_t* gate, int j, void* stream);

/* Debug: if non-NULL, the next sweep writes clock64() phase stamps of cluster 0 for
 * positions 64..319 into buf (int64 [256][16]: chain lane 0 in 0..7, near thread 0 in 8..15). */
void scrf_debug_trace(void* buf);

/* Debug: with SCRF_WATCHDOG=1 in the environment, sweep mbarrier waits trap after ~1e8
 * polls instead of hanging; this returns 1 and {flag, block, thread, site, index} if one fired. */
int scrf_debug_hang(int* out5);

#ifdef __cplusplus
}
#endif
#endif /* SCRF_H_ */
