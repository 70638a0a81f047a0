/*
 * rnnt_oracle.h — CPU restatement of the reference RNN-T greedy decode path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA decoder
 * in paper_2406_03791_b200/csrc.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product path never does.
 *
 * It restates, in plain C with the reference's fixed-order fp32 arithmetic
 * (compile with -O2 -ffp-contract=off, glibc libm expf/logf/tanhf), the
 * functions the reference's rnnt-sim keeps in
 *   /root/reference/proj/src/tensor.cpp   (Rng, matmul, argmax, log_softmax)
 *   /root/reference/proj/src/model.cpp    (init_params, prediction, joint)
 *   /root/reference/proj/src/decoders.cpp (scalar_reference_decode[_tdt])
 *   /root/reference/proj/tests/decode_test_util.hpp (make_random_case)
 * plus the LSTM prediction network the BASELINE configs need, which the
 * reference lacks and which this repo defines as an oracle
 * extension.  Parity of the restatement is pinned
 * bit-for-bit against the compiled reference (oracle/_ref, see Makefile) and
 * the committed digests in tests/golden/.
 */
#ifndef RNNT_ORACLE_H
#define RNNT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_LAYERS 8
#define ORC_MAX_DURATIONS 16

enum { ORC_CELL_TANH = 0, ORC_CELL_LSTM = 1 };

/* RnntDims (model.hpp:31-40) + cell/layers (LSTM extension). */
typedef struct {
  int32_t vocab, embed, hidden, layers, cell, joint, feature;
  int32_t num_durations;
  int32_t durations[ORC_MAX_DURATIONS];
} orc_dims;

/* splitmix64 Rng (tensor.cpp:633-653). */
typedef struct { uint64_t state; } orc_rng;
uint64_t orc_rng_next(orc_rng* r);
float orc_rng_uniform(orc_rng* r, float lo, float hi);
int32_t orc_rng_uniform_int(orc_rng* r, int32_t n);

/* Parameter tensors in reference fill order (model.cpp:81-108):
 *  tanh : embedding[V1,E], w_ih[E,H], w_hh[H,H], bias[H],
 *         enc_proj[F,J], pred_proj[H,J], out_proj[J,V1] (, dur_proj[J,D])
 *  lstm : embedding[V1,E], {w_ih_l[in_l,4H], w_hh_l[H,4H], bias_l[4H]} x L,
 *         enc_proj[F,J], pred_proj[H,J], out_proj[J,V1] (, dur_proj[J,D])
 * All [in,out] row-major (x @ W).  Returns -1 on invalid dims. */
int orc_num_params(const orc_dims* d);
int orc_param_size(const orc_dims* d, int i, int64_t* rows, int64_t* cols);
int orc_validate_dims(const orc_dims* d);
int orc_state_width(const orc_dims* d);
int orc_init_params(uint64_t seed, const orc_dims* d, float* const* out);

/* One prediction step for `batch` rows: labels[b], state[b,W] -> state_out
 * (model.cpp:163-176 tanh; LSTM extension).  g is h_top of state_out. */
void orc_prediction(const orc_dims* d, const float* const* p, int batch,
                    const int32_t* labels, const float* state, float* state_out);
/* Joint log-probabilities (model.cpp:178-213): logp[b,V1], dur_logp[b,D]
 * (dur_logp may be NULL).  g points at h_top rows with stride g_stride. */
void orc_joint(const orc_dims* d, const float* const* p, int batch,
               const float* f, const float* g, int64_t g_stride, float* logp,
               float* dur_logp);

/* Decision record of the step-recording scalar decoder. */
typedef struct {
  int32_t t, k, dur_idx, dur;
  float v;        /* logp of k */
  float margin;   /* top1 - top2 of token logp */
  float dur_margin;
} orc_decision;

/* scalar_reference_decode (decoders.cpp:670-701) when tdt==0 and
 * scalar_reference_decode_tdt (703-755) when tdt==1, over one utterance
 * features[T,F].  Emissions go to tokens/frames/scores/durs (capacity cap,
 * any may be NULL); decisions (optional, capacity dcap) record every argmax
 * step.  Returns the emission count; *ndec gets the decision count and
 * *total the double-accumulated total_score (decoders.cpp:699-700). */
int orc_decode_utt(const orc_dims* d, const float* const* p,
                   const float* features, int frames, int out_len,
                   int max_symbols, int tdt, int32_t* tokens, int32_t* frm,
                   float* scores, int32_t* durs, int cap, orc_decision* dec,
                   int dcap, int* ndec, double* total);

/* make_random_case (decode_test_util.hpp:38-59): fills dims/batch/frames/ms
 * and returns the params seed.  Then orc_random_case_inputs fills
 * x[batch,frames,feature] and out_len[batch]. */
uint64_t orc_random_case_header(uint64_t seed, int with_durations,
                                orc_dims* d, int* batch, int* frames,
                                int* max_symbols);
void orc_random_case_inputs(uint64_t seed, float* x, int32_t* out_len);

/* Uniform fill helper: n floats from Rng(seed) in [lo,hi). */
void orc_fill_uniform(uint64_t seed, float lo, float hi, float* out, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
