/*
 * rnntg.h — C ABI of the B200-native RNN-T / TDT greedy decoder.
 *
 * This is the drop-in boundary for the reference's decoder interface
 * (/root/reference/proj/include/rnntsim/decoders.hpp:56-130 and
 * model.hpp:92-161).  Plain pointers, sizes and int status codes only; the
 * C++ shim in include/rnntsim_cuda.hpp maps these 1:1 back onto the
 * reference's types and exceptions (errors.hpp:23-85).
 *
 * Object model (mirrors the reference ownership rules, decoders.hpp:100-113):
 *   rnntg_model    immutable device weights ("DecoderModel"); shareable by
 *                  many decoders on the same device, must outlive them.
 *   rnntg_decoder  one captured decode program for (algo, batch, max_frames,
 *                  max_symbols) -- the analogue of CapturedDecoder.  Owns a
 *                  CUDA stream, a cudaGraphExec with conditional WHILE nodes
 *                  (or the persistent kernel), and static device buffers.
 *                  Not thread-safe; one host thread per decoder.
 *
 * Every entry point returns RNNTG_OK (0) or a status code; the message of
 * the last failure on the calling thread is available from
 * rnntg_last_error().  There is no CPU fallback: without a CUDA device every
 * compute entry point returns RNNTG_E_CUDA.
 */
#ifndef RNNTG_H
#define RNNTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RNNTG_ABI_VERSION 1
#define RNNTG_MAX_LAYERS 4
#define RNNTG_MAX_DURATIONS 16

/* Status codes, 1:1 with the reference exception classes (errors.hpp). */
typedef enum {
  RNNTG_OK = 0,
  RNNTG_E_VALUE = 1,       /* ValueError: ms<1, B/T<1, bad dims (decoders.cpp:126,170) */
  RNNTG_E_DIMENSION = 2,   /* DimensionError: shapes, out_len range (decoders.cpp:127-141) */
  RNNTG_E_DTYPE = 3,       /* DtypeError */
  RNNTG_E_INDEX = 4,       /* IndexError: label id out of range (tensor.cpp:499-502) */
  RNNTG_E_STATE = 5,       /* StateError: TDT without a head, uninitialized decoder */
  RNNTG_E_STRUCTURE = 6,   /* StructureError: graph construction rejected */
  RNNTG_E_RUNAWAY = 7,     /* RunawayLoopError: device loop cap hit (engine.cpp:284-291) */
  RNNTG_E_CUDA = 8,        /* CUDA runtime / driver failure, or no device */
  RNNTG_E_ALLOC = 9        /* device or pinned allocation failed */
} rnntg_status;

typedef enum { RNNTG_CELL_TANH = 0, RNNTG_CELL_LSTM = 1, RNNTG_CELL_SCRIPTED = 2 } rnntg_cell;

/* DecodeAlgo (decoders.hpp:97). */
typedef enum {
  RNNTG_ALGO_FRAME_SYNC = 0,      /* greedy_decode_sync_free / FrameSync graph */
  RNNTG_ALGO_LABEL_LOOP = 1,      /* label_looping_decode / LabelLoop graph */
  RNNTG_ALGO_TDT_LABEL_LOOP = 2   /* tdt_label_looping_decode / TdtLabelLoop graph */
} rnntg_algo;

/* How the loops run on the device. */
typedef enum {
  RNNTG_EXEC_GRAPH = 0,       /* CUDA graph, nested conditional WHILE nodes; loop bodies = the
                                 tcgen05 step kernel (one decision per launch) when the model fits
                                 it, else the FFMA step kernels of RNNTG_EXEC_GRAPH_FFMA */
  RNNTG_EXEC_PERSISTENT = 1,  /* one cooperative persistent kernel, in-kernel loops (FFMA) */
  RNNTG_EXEC_TENSOR = 2,      /* persistent kernel on tcgen05 tensor cores, role-specialised CTAs */
  RNNTG_EXEC_HOSTLOOP = 3,    /* sync-requiring baseline (greedy_decode_baseline, decoders.cpp:546-563):
                                 the graph's kernels driven by a host loop with a device->host flag
                                 read + synchronise per step; rnntg_launch blocks until done */
  RNNTG_EXEC_GRAPH_FFMA = 4   /* CUDA graph with conditional WHILE nodes over the FFMA step kernels
                                 (joint, per-layer prediction, pred_proj: 4 nodes per inner step) */
} rnntg_exec;

/* RnntDims (model.hpp:31-40) + the prediction-network cell.
 * tanh: the reference NeuralModel (1 layer, embed may differ from hidden).
 * lstm: `layers` stacked LSTM layers, gates i,f,g,o, state [h0,c0,h1,c1,...]. */
typedef struct {
  int32_t vocab;          /* labels excluding blank; blank index == vocab */
  int32_t embed;
  int32_t hidden;
  int32_t layers;
  int32_t cell;           /* rnntg_cell */
  int32_t joint;
  int32_t feature;
  int32_t num_durations;  /* 0 = no duration head */
  int32_t durations[RNNTG_MAX_DURATIONS];  /* ascending, first 0 or 1 */
} rnntg_dims;

typedef struct rnntg_model rnntg_model;
typedef struct rnntg_decoder rnntg_decoder;

/* Per-decode counters (decode_joint_evals analogue, decoders.cpp:641-643). */
typedef struct {
  int64_t joint_evals;    /* joint-step launches (inner iterations) */
  int64_t pred_steps;     /* prediction-network steps */
  int64_t outer_iters;    /* frame-loop / label-loop outer iterations */
  int64_t emitted;        /* total emitted labels */
  float gpu_ms;           /* device time of the last launch (events) */
} rnntg_stats;

const char* rnntg_last_error(void);
int rnntg_abi_version(void);
/* Number of CUDA devices visible (0 on a host without a GPU). */
int rnntg_device_count(void);

/* Table-lookup model on the device (the reference's ScriptedModel,
 * model.hpp:168-230 / model.cpp:417-615) so the planted-trace schedule tests
 * run on the GPU schedules.  The prediction state is the running emission
 * count (run_prediction: hidden' = hidden + 1); the joint puts logit 10 on the
 * planted label of (utterance b, frame t, emission u) and 0 elsewhere
 * (logits_at), TDT also on the duration class of duration_at(b, t, u).
 *   labels   [batch][frames][umax]  planted label of emission u (vocab = blank
 *            for u past the frame's list); u >= umax or u < 0 is blank
 *   fs_arr   [batch][frames + 1]    emissions before frame t on a frame-sync
 *            schedule (frame_sync_arrival; t >= frames uses entry frames)
 *   dur_arr  [batch][frames]        emissions on arrival at frame t on a
 *            duration schedule, -1 if never reached (duration_arrival)
 *   dur_val  [batch][frames][umax + 1]  duration_at(b, t, min(u, umax));
 *            NULL (and num_durations 0) without a duration head
 * Decoders over a scripted model run on RNNTG_EXEC_GRAPH or
 * RNNTG_EXEC_HOSTLOOP (the persistent executors return RNNTG_E_VALUE). */
rnntg_status rnntg_model_create_scripted(int device, int vocab, int batch, int frames, int umax,
                                         const int32_t* labels, const int32_t* fs_arr,
                                         const int32_t* dur_arr, int num_durations,
                                         const int32_t* durations, const int32_t* dur_val,
                                         rnntg_model** out);

/* Weights in the reference's parameter order and [in,out] row-major layout
 * (model.hpp:44-59; the LSTM extension keeps the order with one
 * (w_ih, w_hh, bias) triple per layer):
 *   tanh: embedding[V+1,E], w_ih[E,H], w_hh[H,H], bias[H],
 *         enc_proj[F,J], pred_proj[H,J], out_proj[J,V+1] (, dur_proj[J,D])
 *   lstm: embedding[V+1,E], {w_ih_l[in,4H], w_hh_l[H,4H], bias_l[4H]}xL,
 *         enc_proj[F,J], pred_proj[H,J], out_proj[J,V+1] (, dur_proj[J,D])
 * Host pointers; the library repacks (padding, gate interleave, tf32 split)
 * without changing any per-output k-order of the reference math. */
rnntg_status rnntg_model_create(int device, const rnntg_dims* dims,
                                const float* const* weights, int num_weights,
                                rnntg_model** out);
rnntg_status rnntg_model_destroy(rnntg_model* m);

/* build_decode_graph (decoders.cpp:589-627): allocate static buffers and
 * capture the program for (algo, batch, max_frames, max_symbols). */
rnntg_status rnntg_decoder_create(rnntg_model* m, int algo, int exec, int batch,
                                  int max_frames, int max_symbols,
                                  rnntg_decoder** out);
rnntg_status rnntg_decoder_destroy(rnntg_decoder* d);
/* Emission capacity per utterance (max_frames * max_symbols, decoders.cpp:197). */
int rnntg_decoder_capacity(const rnntg_decoder* d);

/* bind_decode_inputs (decoders.cpp:202-207): validate and copy x[B,T,F]
 * (float32) and out_len[B] (int32 in [0,T]) from HOST memory (async; pinned
 * memory makes it truly asynchronous). */
rnntg_status rnntg_bind(rnntg_decoder* d, const float* x, const int32_t* out_len);
/* Same, from DEVICE pointers already resident on the decoder's device.  The
 * lengths are checked on the device in stream order (no host round trip): an
 * entry outside [0, T] is clamped for the decode and reported as
 * RNNTG_E_DIMENSION by the next rnntg_sync / rnntg_read. */
rnntg_status rnntg_bind_device(rnntg_decoder* d, const float* x_dev,
                               const int32_t* out_len_dev);
/* One graph launch (replay_decode's single host launch, decoders.cpp:629-639). */
rnntg_status rnntg_launch(rnntg_decoder* d);
rnntg_status rnntg_sync(rnntg_decoder* d);
/* read_emissions (decoders.cpp:97-122): counts[B], and per utterance up to
 * `cap` entries of tokens/frames/scores/durations in [B,cap] row-major
 * arrays (any pointer may be NULL).  Durations are the TDT duration value
 * of each emission (0 for RNN-T). */
rnntg_status rnntg_read(rnntg_decoder* d, int32_t* counts, int32_t* tokens,
                        int32_t* frames, float* scores, int32_t* durations,
                        int cap);
rnntg_status rnntg_get_stats(rnntg_decoder* d, rnntg_stats* s);
/* Host-side work of the last decode, for the reference's TimingReport
 * (engine.hpp:119-128): device->host synchronisations the host waited on
 * (rnntg_sync and, for RNNTG_EXEC_HOSTLOOP, one per inner step), host launch
 * calls (kernels + graph launches) and graph launches.  Counted since the last
 * rnntg_launch; read after rnntg_read / rnntg_sync. */
rnntg_status rnntg_host_counts(rnntg_decoder* d, int64_t* syncs, int64_t* launches, int64_t* graph_launches);
/* The decoder's CUDA stream (cudaStream_t), for callers that overlap work. */
void* rnntg_decoder_stream(rnntg_decoder* d);

/* Kernel-level step entry points (test_model.cpp:224-270 analogues).
 * joint: f[B,F], g[B,H] (h_top rows) -> logp[B,V+1] (and dur_logp[B,D] if
 * the model has a duration head and dur_logp != NULL), computed by the same
 * encoder-projection, predictor-projection and joint-step kernels the
 * decoder launches.  prediction: labels[B], state[B,W] -> state_out[B,W]. */
rnntg_status rnntg_step_joint(rnntg_model* m, int batch, const float* f,
                              const float* g, float* logp, float* dur_logp);
rnntg_status rnntg_step_prediction(rnntg_model* m, int batch,
                                   const int32_t* labels, const float* state,
                                   float* state_out);

/* Profiling hook for bench.py's roofline: launch one of the decoder's own
 * kernels standalone `reps` times on the decoder stream, with the decoder's
 * buffers (after a decode), every row live; *avg_ms = mean CUDA-event time.
 * which: 0 = K1 encoder projection, 1+l = prediction layer l,
 *        8 = pred_proj, 9 = joint step. */
rnntg_status rnntg_time_kernel(rnntg_decoder* d, int which, int reps, float* avg_ms);

/* Tensor executor event trace (RNNTG_PROF=1): [16 events][64 steps] globaltimer ns. */
rnntg_status rnntg_debug_trace(rnntg_decoder* d, unsigned long long* out, int n);
/* Logit-level parity of the tensor-core executor (test_model.cpp:224-270
 * analogue): runs one decode of the bound inputs with the J tiles' fp32
 * logits of decision step `step` (group row order = batch order) copied to
 * out[B][V1 + D] (vocab + blank, then the duration logits).  Rows that make
 * no decision at that step keep 0.  Tensor executor, B <= 256 only. */
rnntg_status rnntg_debug_logits(rnntg_decoder* d, int step, float* out);
/* Persistent executor phase profile (CTA 0, ns per phase, accumulated since
 * the last call; needs RNNTG_PROF=1 at decoder creation). */
rnntg_status rnntg_debug_profile(rnntg_decoder* d, unsigned long long* out16);

/* GPU idle fraction of the work issued between begin and end, from CUPTI
 * kernel activity records (graph kernel nodes reported individually):
 * busy = union of kernel intervals, span = first kernel start -> last end;
 * idle = 1 - busy / span (the reference's TimingReport.idle_fraction,
 * engine.cpp:329-366, measured on the device). */
rnntg_status rnntg_trace_begin(void);
rnntg_status rnntg_trace_end(double* busy_ms, double* span_ms, int64_t* kernels);

/* Encoder projection only (K1): fp[M,J] = x[M,F] @ enc_proj, host buffers. */
rnntg_status rnntg_enc_proj(rnntg_model* m, int rows, const float* x, float* fp);

#ifdef __cplusplus
}
#endif
#endif
